"""Device-side statistical tests: the reference's four stat tests over GPU-generated streams.

Mirrors proj/include/twistsieve/stat_tests.hpp (TestSpec :18-33, TestResult :35-42, the desk
specs and named_spec of proj/src/stat_tests.cpp:52-103, run_test :313-319) and the campaign cell
of proj/src/sieve.cpp:116-183 (one fresh stream per (status, seed, test), rows ordered
(status, seed, test), per-row errors). The words are generated and counted on the GPU
(csrc/mtgp_stat.cu); the counts -> statistic / p-value step and the numerics are the C-ABI's
host half (csrc/stat_host.cpp). Everything goes through libmtgp_b200.so; nothing here computes a
test result in Python.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace
from typing import List, Optional, Sequence

import numpy as np

from . import mtgp

TEST_IDS = {"gap": 0, "hamming_indep": 1, "collision_over": 2, "random_walk": 3}
ID_NAMES = {v: k for k, v in TEST_IDS.items()}
ALIASES = {"hamming": "hamming_indep", "opso": "collision_over", "walk": "random_walk"}
CLASSES = ("correct", "suspect", "disastrous")  # PValueClass, classify.hpp:11
STAT_EXHAUSTED = 2
EXHAUSTED_MSG = "insufficient stream"  # StreamExhausted::what(), word_source.hpp:15-17


@dataclass
class TestSpec:
    """stat_tests.hpp:18-33; only the fields a given test reads are meaningful for it."""
    test_id: str
    N: int = 1
    n: int = 0
    r: int = 0
    alpha: float = 0.0
    beta: float = 0.0
    s: int = 0
    L: int = 0
    d: int = 0
    l: int = 0  # noqa: E741
    t: int = 0

    def to_c(self) -> mtgp.StatSpecC:
        c = mtgp.StatSpecC()
        c.test = TEST_IDS.get(self.test_id, -1)
        c.N, c.n, c.r, c.s, c.L, c.d, c.l, c.t = self.N, self.n, self.r, self.s, self.L, self.d, self.l, self.t
        c.alpha, c.beta = self.alpha, self.beta
        return c

    def validate(self) -> None:
        """TestSpec::validate (stat_tests.cpp:7-30) plus the test's pre-read checks."""
        if self.test_id not in TEST_IDS:
            raise mtgp.MtgpInvalidArgument(mtgp.MTGP_EINVAL, f"unknown test id: {self.test_id}")
        lib = mtgp.load_library()
        mtgp._check(lib, lib.mtgp_stat_validate(C.byref(self.to_c())))

    def describe(self) -> str:
        """TestSpec::describe (stat_tests.cpp:32-50)."""
        if self.test_id == "gap":
            return f"gap(n={self.n},r={self.r},alpha={self.alpha:.9g},beta={self.beta:.9g})"
        if self.test_id == "hamming_indep":
            return f"hamming_indep(n={self.n},r={self.r},s={self.s},L={self.L},d={self.d})"
        if self.test_id == "collision_over":
            return f"collision_over(n={self.n},r={self.r},s={self.s},t={self.t or 2 * self.s})"
        return f"random_walk(n={self.n},r={self.r},l={self.l})"


@dataclass
class TestResult:
    """stat_tests.hpp:35-42, plus the per-row error string of the campaign (sieve.hpp ResultRow)
    and the number of stream words the test consumed."""
    spec: TestSpec
    statistic: float = 0.0
    p_value: float = 0.0
    classification: str = "correct"
    degenerate: bool = False
    error: str = ""
    words_used: int = 0

    def is_error(self) -> bool:
        return bool(self.error)


# -- desk-scale specs (stat_tests.cpp:52-96)
def desk_gap_spec() -> TestSpec:
    return TestSpec("gap", n=1000000, r=25, alpha=0.0, beta=1.0 / 32.0)


def desk_hamming_spec() -> TestSpec:
    return TestSpec("hamming_indep", n=100000, r=25, s=5, L=1200, d=0)


def desk_opso_spec() -> TestSpec:
    return TestSpec("collision_over", n=32768, r=0, s=11, t=22)


def desk_walk_spec() -> TestSpec:
    return TestSpec("random_walk", n=100000, r=0, l=128)


def desk_battery() -> List[TestSpec]:
    return [desk_gap_spec(), desk_hamming_spec(), desk_opso_spec(), desk_walk_spec()]


def named_spec(name: str) -> TestSpec:
    """stat_tests.cpp:98-104: canonical ids plus the aliases hamming / opso / walk."""
    name = ALIASES.get(name, name)
    table = {"gap": desk_gap_spec, "hamming_indep": desk_hamming_spec, "collision_over": desk_opso_spec,
             "random_walk": desk_walk_spec}
    if name not in table:
        raise mtgp.MtgpInvalidArgument(mtgp.MTGP_EINVAL, f"unknown test name: {name}")
    return table[name]()


def _result(spec: TestSpec, r: mtgp.StatResultC) -> TestResult:
    if r.error == STAT_EXHAUSTED:
        return TestResult(spec, error=EXHAUSTED_MSG, words_used=r.words_used)
    return TestResult(spec, r.statistic, r.p_value, CLASSES[r.classification], bool(r.degenerate), "",
                      r.words_used)


def run_on_context(ctx: "mtgp.MtgpContext", spec: TestSpec) -> List[TestResult]:
    """run_test(spec) on every stream of `ctx` (GPU), from the current position."""
    spec.validate()
    out = (mtgp.StatResultC * ctx.n_sets)()
    mtgp._check(ctx.lib, ctx.lib.mtgp_stat_run(ctx.h, C.byref(spec.to_c()), out))
    return [_result(spec, out[s]) for s in range(ctx.n_sets)]


def counts_len(spec: TestSpec) -> int:
    lib = mtgp.load_library()
    n = C.c_uint64()
    mtgp._check(lib, lib.mtgp_stat_counts_len(C.byref(spec.to_c()), C.byref(n)))
    return n.value


def finish_counts(spec: TestSpec, counts: Sequence[int]) -> TestResult:
    """The host half alone (CPU): TestResult from a test's integer counts (layout in
    include/mtgp_b200.h, mtgp_stat_finish)."""
    lib = mtgp.load_library()
    arr = np.ascontiguousarray(np.asarray(counts, dtype=np.uint64))
    r = mtgp.StatResultC()
    mtgp._check(lib, lib.mtgp_stat_finish(C.byref(spec.to_c()), arr.ctypes.data_as(C.POINTER(C.c_uint64)),
                                          arr.size, C.byref(r)))
    return _result(spec, r)


# -- numerics (stats.hpp), through the C-ABI
def _math(fn: str, *args) -> float:
    lib = mtgp.load_library()
    out = C.c_double()
    mtgp._check(lib, getattr(lib, fn)(*args, C.byref(out)))
    return out.value


def ln_gamma(x: float) -> float:
    return _math("mtgp_ln_gamma", x)


def gamma_p(a: float, x: float) -> float:
    return _math("mtgp_gamma_p", a, x)


def gamma_q(a: float, x: float) -> float:
    return _math("mtgp_gamma_q", a, x)


def chi_square_pvalue(statistic: float, df: int) -> float:
    return _math("mtgp_chi_square_pvalue", statistic, df)


def poisson_cdf(k: int, lam: float) -> float:
    return _math("mtgp_poisson_cdf", k, lam)


def poisson_sf(k: int, lam: float) -> float:
    return _math("mtgp_poisson_sf", k, lam)


def poisson_pmf(k: int, lam: float) -> float:
    return _math("mtgp_poisson_pmf", k, lam)


def binomial_log_pmf(k: int, n: int, p: float) -> float:
    return _math("mtgp_binomial_log_pmf", k, n, p)


def binomial_upper_tail(count: int, n: int, p: float) -> float:
    return _math("mtgp_binomial_upper_tail", count, n, p)


def classify_pvalue(p: float) -> str:
    lib = mtgp.load_library()
    out = C.c_int32()
    mtgp._check(lib, lib.mtgp_classify_pvalue(p, C.byref(out)))
    return CLASSES[out.value]


# -- campaign grid (sieve.cpp:116-183 run_grid, GPU-fed)
@dataclass
class ResultRow:
    """sieve.hpp ResultRow: one (status, seed, test) cell."""
    status_index: int
    seed_index: int
    status_id: str
    test_id: str
    seed: int
    statistic: float = 0.0
    p_value: float = 0.0
    classification: str = "correct"
    degenerate: bool = False
    error: str = ""


def run_grid(statuses: Sequence, seeds: Sequence[int], specs: Sequence[TestSpec], engine: str = "mtgp",
             device: int = 0, status_ids: Optional[Sequence[str]] = None) -> List[ResultRow]:
    """Every (status, seed, test) cell, rows ordered (status, seed, test) like run_grid; each cell
    runs on a fresh stream (status, seed). statuses: MtgpParams (engine "mtgp") or Engine::mt
    status dicts (engine "mt"). All status x seed streams live in ONE context, so each test is one
    GPU pass over all of them. A test whose spec is invalid yields an error row in every cell (the
    reference catches per cell, sieve.cpp:163-165)."""
    if not statuses or not specs:
        raise mtgp.MtgpInvalidArgument(mtgp.MTGP_EINVAL, "no statuses" if not statuses else "no test specs")
    ids = list(status_ids) if status_ids is not None else [str(i) for i in range(len(statuses))]
    streams = [(si, wi) for si in range(len(statuses)) for wi in range(len(seeds))]
    sts = [statuses[si] for si, _ in streams]
    sds = [seeds[wi] for _, wi in streams]
    ctx = mtgp.MtContext(sts, sds, device=device) if engine == "mt" else mtgp.MtgpContext(sts, sds, device=device)
    per_test = []
    with ctx:
        for spec in specs:
            try:
                per_test.append(run_on_context(ctx, spec))
            except mtgp.MtgpInvalidArgument as e:
                msg = str(e).split("] ", 1)[-1]
                per_test.append([TestResult(spec, error=msg)] * len(streams))
    rows = []
    for k, (si, wi) in enumerate(streams):
        for ti, spec in enumerate(specs):
            r = per_test[ti][k]
            rows.append(ResultRow(si, wi, ids[si], spec.test_id, int(seeds[wi]) & 0xFFFFFFFF, r.statistic,
                                  r.p_value, r.classification, r.degenerate, r.error))
    return rows

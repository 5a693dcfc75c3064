"""CPU checkers for the device-side statistical tests.

TEST INFRASTRUCTURE ONLY (tests/ and make_goldens.py; never the product package):

* ``ref_*``: ctypes binding of oracle/ref_stat_harness.cpp, i.e. the UNMODIFIED reference
  templates (proj/include/twistsieve/stat_tests.hpp:84-309) and numerics (proj/src/stats.cpp,
  classify.cpp) compiled from their sources into oracle/_ref/libtwistsieve_ref.so.
* ``*_counts``: a numpy restatement of the four counting loops, so the host half
  (mtgp_stat_finish) can be checked without a GPU: counts here -> mtgp_stat_finish must equal
  the reference template run over the same words.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

import oracle_py

TEST_IDS = {"gap": 0, "hamming_indep": 1, "collision_over": 2, "random_walk": 3}


class RefSpec(C.Structure):  # same layout as mtgp_stat_spec
    _fields_ = [("test", C.c_int32), ("N", C.c_uint32), ("n", C.c_uint64), ("r", C.c_uint32), ("s", C.c_uint32),
                ("L", C.c_uint32), ("d", C.c_uint32), ("l", C.c_uint32), ("t", C.c_uint32),
                ("alpha", C.c_double), ("beta", C.c_double)]


class RefResult(C.Structure):
    _fields_ = [("statistic", C.c_double), ("p_value", C.c_double), ("classification", C.c_int32),
                ("degenerate", C.c_int32), ("error", C.c_int32), ("pad", C.c_int32), ("words_used", C.c_uint64)]


_bound = False


def _lib():
    global _bound
    L = oracle_py.ref_lib()
    if not _bound:
        L.ref_stat_last_message.restype = C.c_char_p
        L.ref_stat_run_words.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(RefSpec), C.POINTER(RefResult)]
        L.ref_stat_run_cell.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(RefSpec), C.POINTER(RefResult)]
        L.ref_stat_math.argtypes = [C.c_int, C.c_double, C.c_double, C.c_uint64, C.c_uint64, C.POINTER(C.c_double)]
        L.ref_stat_desk_spec.argtypes = [C.c_int, C.POINTER(RefSpec)]
        L.ref_gap_tcut.argtypes = [C.POINTER(RefSpec), C.POINTER(C.c_uint64)]
        _bound = True
    return L


def to_ref(spec) -> RefSpec:
    """spec: anything with TestSpec's attributes (paper_1501_07701_b200.stattests.TestSpec)."""
    r = RefSpec()
    r.test = TEST_IDS.get(spec.test_id, -1)
    r.N, r.n, r.r, r.s, r.L, r.d, r.l, r.t = spec.N, spec.n, spec.r, spec.s, spec.L, spec.d, spec.l, spec.t
    r.alpha, r.beta = spec.alpha, spec.beta
    return r


def _as_dict(rc: int, r: RefResult) -> dict:
    d = {"rc": rc, "statistic": r.statistic, "p_value": r.p_value, "classification": r.classification,
         "degenerate": r.degenerate, "words_used": r.words_used, "error": ""}
    if rc:
        d["error"] = _lib().ref_stat_last_message().decode()
    return d


def ref_run_words(words: np.ndarray, spec) -> dict:
    """run_test(spec) over the finite stream `words` (reference templates, compiled)."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    res = RefResult()
    rc = _lib().ref_stat_run_words(w.ctypes.data_as(C.c_void_p), w.size, C.byref(to_ref(spec)), C.byref(res))
    return _as_dict(rc, res)


def ref_run_cell(seed: int, spec, status12: Optional[Sequence[int]] = None) -> dict:
    """One campaign cell exactly as sieve.cpp:156-158 runs it (Engine::mt, MT19937 by default)."""
    st = (C.c_uint32 * 12)(*status12) if status12 is not None else None
    res = RefResult()
    rc = _lib().ref_stat_run_cell(st, seed & 0xFFFFFFFF, C.byref(to_ref(spec)), C.byref(res))
    return _as_dict(rc, res)


MATH = {"ln_gamma": 0, "gamma_p": 1, "gamma_q": 2, "chi_square_pvalue": 3, "poisson_cdf": 4, "poisson_sf": 5,
        "poisson_pmf": 6, "binomial_log_pmf": 7, "binomial_upper_tail": 8, "classify_pvalue": 9}


def ref_math(fn: str, a: float = 0.0, b: float = 0.0, k: int = 0, n: int = 0):
    """(rc, value, message) of the reference numerics."""
    out = C.c_double()
    rc = _lib().ref_stat_math(MATH[fn], a, b, k, n, C.byref(out))
    return rc, out.value, (_lib().ref_stat_last_message().decode() if rc else "")


def ref_desk_spec(i: int) -> RefSpec:
    r = RefSpec()
    assert _lib().ref_stat_desk_spec(i, C.byref(r)) == 0
    return r


def ref_gap_tcut(spec) -> int:
    t = C.c_uint64()
    assert _lib().ref_gap_tcut(C.byref(to_ref(spec)), C.byref(t)) == 0
    return t.value


# ---------------- numpy restatement of the counting loops ----------------

def letters(words: np.ndarray, r: int, s: int) -> np.ndarray:
    """detail::letter_of (stat_tests.hpp:60-63)."""
    return (words.astype(np.uint64) >> (32 - r - s)) & ((1 << s) - 1)


def gap_counts(words: np.ndarray, spec, tcut: int, budget: int):
    """stat_tests.hpp:84-125 with the reference's double comparisons; (counts, words_used) or
    None when the stream would be exhausted."""
    kept = 32 - spec.r
    mask = 0xFFFFFFFF if spec.r == 0 else (0xFFFFFFFF >> spec.r)
    u = (words[:budget].astype(np.uint64) & mask).astype(np.float64) * np.ldexp(1.0, -kept)
    hits = np.flatnonzero((u >= spec.alpha) & (u < spec.beta))
    if hits.size < spec.n + 1:
        return None
    gaps = np.diff(hits[:spec.n + 1]) - 1
    return np.bincount(np.minimum(gaps, tcut), minlength=tcut + 1).astype(np.uint64), int(hits[spec.n]) + 1


def hamming_counts(words: np.ndarray, spec) -> np.ndarray:
    """stat_tests.hpp:150-193: letters MSB first into L-bit blocks, pairs -> 2x2 sign table."""
    nblocks = (spec.n // 2) * 2
    nbits = nblocks * spec.L
    nwords = -(-nbits // spec.s)
    let = letters(words[:nwords], spec.r, spec.s)
    bits = ((let[:, None] >> np.arange(spec.s - 1, -1, -1, dtype=np.uint64)) & 1).astype(np.uint8).ravel()
    weight = bits[:nbits].reshape(nblocks, spec.L).sum(axis=1, dtype=np.int64)
    sign = weight > spec.L // 2
    f, s = sign[0::2], sign[1::2]
    return np.array([np.sum(~f & ~s), np.sum(~f & s), np.sum(f & ~s), np.sum(f & s)], dtype=np.uint64)


def collision_counts(words: np.ndarray, spec) -> np.ndarray:
    """stat_tests.hpp:224-238: collisions = n - |distinct overlapping-pair cells|."""
    let = letters(words[:spec.n + 1], spec.r, spec.s)
    cells = (let[:-1] << spec.s) | let[1:]
    return np.array([spec.n - np.unique(cells).size], dtype=np.uint64)


def walk_counts(words: np.ndarray, spec) -> np.ndarray:
    """stat_tests.hpp:279-284: H = odd words per length-l walk, histogram over 0..l."""
    h = (words[:spec.n * spec.l] & 1).reshape(spec.n, spec.l).sum(axis=1)
    return np.bincount(h, minlength=spec.l + 1).astype(np.uint64)


# ---------------- the reference's parameter-set tooling (gf2poly.cpp, dynamic_creator.cpp) ----------------

def ref_is_irreducible(coeffs) -> int:
    """The reference's is_irreducible on sum_i coeffs[i] x^i: 1 / 0, -1 if it throws."""
    L = _lib()
    L.ref_is_irreducible.argtypes = [C.c_void_p, C.c_uint64]
    b = np.ascontiguousarray(np.asarray(coeffs, dtype=np.uint8))
    return L.ref_is_irreducible(b.ctypes.data_as(C.c_void_p), b.size)


def ref_mt_probe_digest(seed: int, status12=None):
    """(poly_digest, degree) of probe_minimal_polynomial(Generator(status, seed), mexp)."""
    L = _lib()
    L.ref_mt_probe_digest.argtypes = [C.c_void_p, C.c_uint32, C.c_char_p, C.POINTER(C.c_int)]
    st = (C.c_uint32 * 12)(*status12) if status12 is not None else None
    buf = C.create_string_buffer(41)
    deg = C.c_int()
    assert L.ref_mt_probe_digest(st, seed & 0xFFFFFFFF, buf, C.byref(deg)) == 0
    return buf.value.decode(), deg.value


def ref_bit0_certify(words: np.ndarray, mexp: int):
    """(degree, irreducible) of the reference's BM over bit 0 of `words` (dc_search's test)."""
    L = _lib()
    L.ref_bit0_certify.argtypes = [C.c_void_p, C.c_uint64, C.c_uint32, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    w = np.ascontiguousarray(words, dtype=np.uint32)
    d, irr = C.c_int(), C.c_int()
    assert L.ref_bit0_certify(w.ctypes.data_as(C.c_void_p), w.size, mexp, C.byref(d), C.byref(irr)) == 0
    return d.value, irr.value

"""Regenerate the frozen golden fixtures in tests/golden/ (run HERE, not on the GPU box).

1. mtgp32_11213_curand.json -- oracle/_ref/curand_pin: cuRAND's MTGP32 headers compiled
   host-side (independent implementation of the same published algorithm).
2. mtgp32_large_curand.json -- oracle/_ref/curand_pin --large: cuRAND's own mtgp32_init_state,
   para_rec, temper and temper_single driven at N = 726 / 1391 (MTGP32-23209 / -44497, which
   cuRAND ships no tables for) over synthetic parameter sets chosen to cover every pos mod 4.
3. mt_reference.json -- the UNMODIFIED reference generator compiled from /root/reference
   (oracle/_ref/libtwistsieve_ref.so): MT19937 seed 5489 words and checksums, temper goldens.

    make -C oracle && python tests/golden/make_goldens.py
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402

import oracle_py  # noqa: E402


def main():
    out = subprocess.run([str(ROOT / "oracle/_ref/curand_pin")], check=True, capture_output=True, text=True).stdout
    d = json.loads(out)
    (ROOT / "tests/golden/mtgp32_11213_curand.json").write_text(json.dumps(d, indent=1) + "\n")
    large_goldens()

    ref = {}
    w = oracle_py.ref_fill(1 << 20, 5489)
    ref["mt19937_seed5489_first16"] = [int(x) for x in w[:16]]
    c = oracle_py.cksum(w)
    ref["mt19937_seed5489_n1048576"] = {k: int(v) for k, v in c.items()}
    for seed in (0, 1, 12345, 0xFFFFFFFF):
        w = oracle_py.ref_fill(4096, seed)
        ref[f"mt19937_seed{seed}_n4096"] = {k: int(v) for k, v in oracle_py.cksum(w).items()}
    ref["temper_ffffffff"] = int(oracle_py.ref_lib().ref_temper(0xFFFFFFFF))
    # DC statuses of SURVEY.md Appendix B (reference dc_search outputs), words via the reference
    dc = {
        "dc521_id7": [7, 521, 17, 7, 23, 4049207303, 3676863948, 3740880118, 11, 7, 15, 18],
        "dc3217_id7": [7, 3217, 101, 9, 15, 3980328967, 882635769, 3305209961, 11, 7, 15, 18],
    }
    for name, st in dc.items():
        w = oracle_py.ref_fill(1 << 16, 4357, st)
        ref[name] = {"status12": st, "seed": 4357, "n": 1 << 16,
                     **{k: int(v) for k, v in oracle_py.cksum(w).items()}}
    # probe digests (verify_digest's polynomial, dynamic_creator.cpp:33-38, 99-103), seed 1
    import stat_oracle as so
    ref["probe_digest_mt19937_seed1"] = list(so.ref_mt_probe_digest(1))
    for name, st in dc.items():
        ref[name]["probe_digest_seed1"] = list(so.ref_mt_probe_digest(1, st))
    (ROOT / "tests/golden/mt_reference.json").write_text(json.dumps(ref, indent=1) + "\n")
    stat_goldens()
    print("goldens written")


def large_pick(mexp):
    """Synthetic sets covering every pos residue mod 4 (the register kernels' C-stream variants)
    and the largest pos among the first 64 (the deepest C-stream history register)."""
    from paper_1501_07701_b200 import tables
    cand = tables.sets_for(mexp, 64)
    pick = []
    for r in range(4):
        pick.append(next(i for i, p in enumerate(cand) if p.pos % 4 == r))
    pick.append(max(range(64), key=lambda i: cand[i].pos))
    return sorted(set(pick)), cand


def large_goldens():
    out = {"cases": []}
    for mexp in (23209, 44497):
        idx, cand = large_pick(mexp)
        sets = [cand[i] for i in idx]
        inp = "\n".join(" ".join(str(v) for v in [p.mexp, p.pos, p.sh1, p.sh2, p.mask, *p.tbl, *p.tmp_tbl,
                                                     *p.flt_tmp_tbl]) for p in sets) + "\n"
        r = subprocess.run([str(ROOT / "oracle/_ref/curand_pin"), "--large"], input=inp, check=True,
                           capture_output=True, text=True).stdout
        d = json.loads(r)
        out["source"] = d["source"]
        for c in d["cases"]:
            p = sets[c["set"]]
            c["synthetic_index"] = idx[c["set"]]
            c["params"] = {"mexp": p.mexp, "pos": p.pos, "sh1": p.sh1, "sh2": p.sh2, "mask": p.mask,
                           "tbl": list(p.tbl), "tmp_tbl": list(p.tmp_tbl), "flt_tmp_tbl": list(p.flt_tmp_tbl)}
            del c["set"]
            out["cases"].append(c)
    (ROOT / "tests/golden/mtgp32_large_curand.json").write_text(json.dumps(out, indent=1) + "\n")


STAT_CASES = [  # (spec fields, streams): small enough for the CPU suite
    (dict(test_id="gap", n=20000, r=25, alpha=0.0, beta=1 / 32), 2),
    (dict(test_id="gap", n=5000, r=3, alpha=0.3, beta=0.7), 2),
    (dict(test_id="hamming_indep", n=4000, r=25, s=5, L=1200), 2),
    (dict(test_id="hamming_indep", n=3001, r=2, s=7, L=33), 2),
    (dict(test_id="collision_over", n=32768, s=11, t=22), 2),
    (dict(test_id="collision_over", n=3000, r=5, s=7), 2),
    (dict(test_id="random_walk", n=10000, l=128), 2),
    (dict(test_id="random_walk", n=20000, l=6), 2),
]


def stat_goldens():
    """3. stat_reference.json -- the reference's statistical tests (oracle/ref_stat_harness.cpp
    over the unmodified stat_tests.hpp / stats.cpp / classify.cpp):
       math:  numerics values (exact, float.hex) and error messages;
       cases: numpy-restated counts of MTGP32 oracle streams + the reference result on the same
              words (pins the host half, mtgp_stat_finish, with no GPU);
       cells: desk-battery campaign cells of MT19937 exactly as sieve.cpp runs them (pins the
              GPU path end to end: tests/test_stat_gpu.py)."""
    import stat_oracle as so
    from paper_1501_07701_b200 import shard
    from paper_1501_07701_b200.stattests import TestSpec, desk_battery

    def hx(v):
        return float(v).hex()

    math = []
    grid = [("ln_gamma", a, 0, 0, 0) for a in (1e-3, 0.2, 0.5, 1, 2, 7.5, 33.3, 1e5, 0.0, -1.0)]
    grid += [(fn, a, x, 0, 0) for fn in ("gamma_p", "gamma_q") for a in (0.1, 0.5, 2.5, 10, 1e4)
             for x in (0.0, 0.01, 1, 3, 99, 1e4)] + [("gamma_p", 0.0, 1.0, 0, 0), ("gamma_q", 1.0, -1.0, 0, 0)]
    grid += [("chi_square_pvalue", s, 0, df, 0) for s in (0, 0.5, 3.84, 100, 1000.5) for df in (1, 2, 7, 383)]
    grid += [("chi_square_pvalue", -1.0, 0, 3, 0), ("chi_square_pvalue", 1.0, 0, 0, 0)]
    grid += [(fn, lam, 0, k, 0) for fn in ("poisson_cdf", "poisson_sf", "poisson_pmf") for k in (0, 1, 5, 128, 300)
             for lam in (0.5, 128, 1000)] + [("poisson_pmf", 0.0, 0, 3, 0)]
    grid += [("binomial_log_pmf", p, 0, k, n) for (k, n, p) in ((0, 10, 0.5), (3, 100, 0.002), (41, 20000, 0.002))]
    grid += [("binomial_upper_tail", p, 0, k, n) for (k, n, p) in
             ((0, 10, 0.5), (3, 100, 0.002), (41, 20000, 0.002), (5, 5, 0.3), (6, 5, 0.3), (1, 5, 1.0))]
    grid += [("classify_pvalue", p, 0, 0, 0) for p in
             (0.0, 1e-11, 1e-10, 5e-4, 0.001, 0.5, 0.999, 0.9995, 1 - 1e-10, 1.0, 1.5, -0.1)]
    for fn, a, b, k, n in grid:
        rc, v, msg = so.ref_math(fn, a, b, k, n)
        math.append({"fn": fn, "a": hx(a), "b": hx(b), "k": k, "n": n, "rc": rc, "value": hx(v) if rc == 0 else None,
                     "msg": msg})

    sets = shard.sets_for_rank(11213, 200, 0)
    cases = []
    for fields, n_streams in STAT_CASES:
        spec = TestSpec(**fields)
        words, _ = oracle_py.mtgp_bulk(sets[:n_streams], list(range(1, n_streams + 1)), 1 << 21, threads=n_streams)
        for s in range(n_streams):
            ref = so.ref_run_words(words[s], spec)
            if spec.test_id == "gap":
                tcut = so.ref_gap_tcut(spec)
                budget = int(float(spec.n + 1) / (spec.beta - spec.alpha) * 8.0) + 4096
                counts, used = so.gap_counts(words[s], spec, tcut, budget)
                assert used == ref["words_used"]
            else:
                counts = {"hamming_indep": so.hamming_counts, "collision_over": so.collision_counts,
                          "random_walk": so.walk_counts}[spec.test_id](words[s], spec)
            cases.append({"spec": fields, "set": s, "seed": s + 1, "counts": [int(c) for c in counts],
                          "statistic": hx(ref["statistic"]), "p_value": hx(ref["p_value"]),
                          "classification": ref["classification"], "degenerate": ref["degenerate"],
                          "words_used": ref["words_used"]})

    cells = []
    for seed in (5489, 1, 0xDEADBEEF):
        for spec in desk_battery():
            r = so.ref_run_cell(seed, spec)
            cells.append({"seed": seed, "spec": {k: getattr(spec, k) for k in
                                                 ("test_id", "n", "r", "alpha", "beta", "s", "L", "d", "l", "t")},
                          "rc": r["rc"], "statistic": hx(r["statistic"]), "p_value": hx(r["p_value"]),
                          "classification": r["classification"], "degenerate": r["degenerate"], "error": r["error"]})
    out = {"generator": "tests/golden/make_goldens.py (oracle/ref_stat_harness.cpp over the reference sources)",
           "math": math, "cases": cases, "cells": cells}
    (ROOT / "tests/golden/stat_reference.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()

"""Exercise every kernel of libmtgp_b200.so at small sizes and check the outputs:

    python tools/sanitize_run.py

(written as the driver for compute-sanitizer's memcheck / racecheck / synccheck; the sanitizer is
closed on the GPU pool this repo is measured on, so it runs plain, bounds-checked by comparing
every output with the oracle / the compiled reference).

gen3 (v3), gen (v2, 11213 and 23209), v1, Engine::mt, prefix + jump_flat (jump-ahead pieces),
skip, host staging, and the four stat-test kernels incl. the gap scan/update path. Checks the
outputs against the oracle so a run that "passes" the sanitizer also produced the right words.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import oracle_py  # noqa: E402
from paper_1501_07701_b200 import mtgp, shard, tables  # noqa: E402
from paper_1501_07701_b200 import stattests as st  # noqa: E402


def check(ctx_words, sets, seeds, n, skip=0):
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, n, skip=skip, threads=len(sets))
    assert np.array_equal(ctx_words, ref), "words differ from the oracle"


def main():
    import torch
    sets = shard.sets_for_rank(11213, 200, 0)[:6]
    seeds = [1, 2, 3, 4, 5, 6]
    L = 1 << 16
    for kernel in (3, 2, 1):
        with mtgp.MtgpContext(sets, seeds) as ctx:
            ctx.set_option(mtgp.OPT_KERNEL, kernel)
            ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 12)   # force jump-ahead pieces
            buf = torch.empty((len(sets), L), dtype=torch.int32, device="cuda")
            ctx.generate_device(mtgp.U32, buf.data_ptr(), L)
            ctx.sync()
            check(buf.cpu().numpy().view(np.uint32), sets, seeds, L)
            print(f"kernel v{kernel}: plan {ctx.last_plan()} ok")
    s23 = tables.synthetic_sets(23209, 3)
    with mtgp.MtgpContext(s23, [7, 8, 9]) as ctx:
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 13)
        w = ctx.fill_u32(40000)
        check(w, s23, [7, 8, 9], 40000)
        ctx.skip(100000)
        w = ctx.fill_u32(1000)
        check(w, s23, [7, 8, 9], 1000, skip=140000)
        print("23209 v2 + skip ok")
    with mtgp.MtContext([mtgp.mt19937_status()] * 2, [5489, 1]) as ctx:
        w = ctx.fill_u32(5000)
        assert np.array_equal(w[0], oracle_py.MtOracle(None, 5489).fill(5000))
        print("Engine::mt ok")
    specs = [st.TestSpec("gap", n=3000, r=25, alpha=0.0, beta=1 / 32),
             st.TestSpec("hamming_indep", n=2000, r=2, s=7, L=33),
             st.TestSpec("collision_over", n=3000, r=5, s=7),
             st.TestSpec("random_walk", n=2000, l=6)]
    with mtgp.MtgpContext(sets[:3], seeds[:3]) as ctx:
        words, _ = oracle_py.mtgp_bulk(sets[:3], seeds[:3], 200000, threads=3)
        import stat_oracle as so
        for spec in specs:
            res = ctx.stat_run(spec)
            for s in range(3):
                ref = so.ref_run_words(words[s], spec) if oracle_py.REF_LIB.exists() else None
                if ref is not None:
                    assert res[s].statistic == ref["statistic"] and res[s].p_value == ref["p_value"], spec
            print(f"stat {spec.test_id} ok")
    print("SANITIZE-RUN DONE")


if __name__ == "__main__":
    main()

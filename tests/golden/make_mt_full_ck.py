"""Full-volume parity fixture for `bench.py --config mt19937` (Engine::mt, MT19937 on the GPU).

bench.py's mt19937 workload: 200 MT19937 streams, seeds 5489 + i (rank 0), each producing the
next 2^28 words per step as two 2^27-word calls; the context's fused checksums accumulate over
every call since creation. This fixture holds the cumulative {sum64, xor32} of every stream at
every 2^27-word boundary for k = 1..50 (25 bench steps), computed by THE REFERENCE ITSELF: the
unmodified reference generator compiled from its sources (oracle/_ref, make_word_source +
WordSource::fill, proj/include/twistsieve/word_source.hpp:21-25,75-76) through
oracle/ref_harness.cpp:ref_cksum_stream. TEST INFRASTRUCTURE.

    make -C oracle && python tests/golden/make_mt_full_ck.py [threads]   # ~19 min on 8 cores
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402

import oracle_py  # noqa: E402

OUT = ROOT / "tests" / "golden" / "mt_full_ck.npz"
STREAMS, SEED0, REC, K = 200, 5489, 1 << 27, 50


def main(threads: int = 8):
    t0 = time.time()
    sums, xors, secs = oracle_py.ref_cksum_stream(SEED0, STREAMS, REC, K, threads)
    np.savez(OUT, mt_sum=sums, mt_xor=xors)
    print(f"wrote {OUT}: {STREAMS} streams x {K} records of {REC} words in {secs:.0f} s ({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 8)

"""Full-volume parity fixtures: cumulative per-stream checksums of every word the bench times.

bench.py generates, per stream, the next 2^28 words per step as two 2^27-word calls (c2/c3/c4;
one 2^24-word call for c5), and the context's fused in-kernel checksums accumulate over every
call since creation (warm-up steps included). So after W warm-up and K timed steps, stream s's
{sum64, xor32} covers its first (W+K) * 2^28 words, and this fixture holds exactly that number
for every (W+K) up to its limit: the oracle (oracle/mtgp32_oracle.c, oracle_mtgp_cksum_stream;
TEST INFRASTRUCTURE) runs every stream from its seed with no output buffer and records the
cumulative checksums at every 2^27-word (c5: 2^24-word) boundary.

Contents of full_ck.npz (sum arrays uint64 = sum of the 32-bit words mod 2^64, xor arrays uint32):
  c2_sum/c2_xor      [1600, 50]     MTGP32-11213 global set IDs 0..1599 (0..199 the cuRAND sets,
                                    the rest the synthetic ones every rank of bench.py uses),
                                    seed 1, first k*2^27 words, k = 1..50 (25 bench steps)
  c3_sum/c3_xor      [200, 50, 2]   the same streams 0..199 as f32 [1,2) / (0,1] bit patterns
  c5_sum/c5_xor      [1024, 64]     global sets 0..1023, seed 1, first k*2^24 words, k = 1..64
  c4_<mexp>_sum/_xor [200, 50]      200 synthetic MTGP32-23209 / -44497 sets, seed 1, k*2^27

    make -C oracle && python tests/golden/make_full_ck.py      # ~25 min on 8 AVX-512 cores
"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402

import oracle_py  # noqa: E402
from paper_1501_07701_b200 import tables  # noqa: E402

OUT = ROOT / "tests" / "golden" / "full_ck.npz"
K_C2 = 50       # 2^27-word records: 25 steps of 2 calls
K_C5 = 64       # 2^24-word records
C2_SETS = 1600  # 8 ranks x 200 sets
C5_SETS = 1024


def main(threads: int = 8):
    res = {}
    t0 = time.time()
    sets = tables.sets_for(11213, C2_SETS)
    # streams 0..199 with the float kinds, every 2^24 words (c5's granularity)
    per = (1 << 27) // (1 << 24)
    a, s = oracle_py.cksum_stream(sets[:200], [1] * 200, 1 << 24, K_C2 * per, True, threads)
    print(f"sets 0..199 (+floats): {s:.0f} s", flush=True)
    b, s = oracle_py.cksum_stream(sets[200:], [1] * (C2_SETS - 200), 1 << 24, K_C2 * per, False, threads)
    print(f"sets 200..{C2_SETS - 1}: {s:.0f} s", flush=True)
    allck = np.concatenate([a, b])
    c2 = allck[:, per - 1::per]
    res["c2_sum"] = np.ascontiguousarray(c2["sum"][:, :, 0])
    res["c2_xor"] = np.ascontiguousarray(c2["xr"][:, :, 0])
    res["c3_sum"] = np.ascontiguousarray(c2["sum"][:200, :, 1:3])
    res["c3_xor"] = np.ascontiguousarray(c2["xr"][:200, :, 1:3])
    res["c5_sum"] = np.ascontiguousarray(allck["sum"][:C5_SETS, :K_C5, 0])
    res["c5_xor"] = np.ascontiguousarray(allck["xr"][:C5_SETS, :K_C5, 0])
    for mexp in (23209, 44497):
        ss = tables.sets_for(mexp, 200)
        c, s = oracle_py.cksum_stream(ss, [1] * 200, 1 << 27, K_C2, False, threads)
        print(f"{mexp}: {s:.0f} s", flush=True)
        res[f"c4_{mexp}_sum"] = np.ascontiguousarray(c["sum"][:, :, 0])
        res[f"c4_{mexp}_xor"] = np.ascontiguousarray(c["xr"][:, :, 0])
    np.savez(OUT, **res)
    print(f"wrote {OUT} in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 8)

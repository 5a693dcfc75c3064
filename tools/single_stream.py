"""One stream through the host-output C-ABI path (what GpuWordSource::refill does for a sieve
worker's make_word_source(status, seed)): words/s per chunk size, MTGP32-11213 and MT19937.

    python tools/single_stream.py [prejump]     # MTGP_OPT_PREJUMP (default: library auto)

Each row: chunk words per mtgp_generate(out_is_device=0) call into a pinned host buffer, calls
timed back to back (wall clock, after one warm-up call), Gwords/s, and the kernel version and
piece count of the plan (one piece = no jump-ahead). long_lived: the stream first skips 2^25
words, past the point where the planner starts splitting few-stream requests."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1501_07701_b200 import mtgp, tables  # noqa: E402

PREJUMP = int(sys.argv[1]) if len(sys.argv) > 1 else None

for long_lived in (False, True):
  for eng in ("mtgp32-11213", "mt19937"):
    for lg in (12, 16, 19, 20, 22, 24):
        L = 1 << lg
        ctx = (mtgp.MtgpContext(tables.load_curand_11213()[:1], [1]) if eng.startswith("mtgp")
               else mtgp.MtContext([mtgp.mt19937_status()], [5489]))
        host = torch.empty((1, L), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        if PREJUMP is not None:
            ctx.set_option(mtgp.OPT_PREJUMP, PREJUMP)
        if long_lived:  # a stream that has already produced 2^25 words (the planner splits only those)
            ctx.skip(1 << 25)
        ctx.generate_host(mtgp.U32, L, out=host)
        reps = max(3, min(2000, (1 << 26) // L))
        t0 = time.perf_counter()
        for _ in range(reps):
            ctx.generate_host(mtgp.U32, L, out=host)
        el = time.perf_counter() - t0
        pieces, _, kv = ctx.last_plan()
        print(json.dumps({"engine": eng, "long_lived": long_lived, "chunk_words": L, "calls": reps, "Gwords_s": round(L * reps / el / 1e9, 4),
                          "us_per_call": round(el / reps * 1e6, 1), "kernel": kv, "pieces": pieces,
                          "prejump": PREJUMP}), flush=True)
        ctx.close()

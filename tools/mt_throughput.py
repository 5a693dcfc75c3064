"""Engine::mt generation throughput on the GPU (200 MT19937 streams, device output)."""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1501_07701_b200 import mtgp  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 200
L = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 24
ctx = mtgp.MtContext([mtgp.mt19937_status()] * S, [5489 + i for i in range(S)])
out = torch.empty((S, L), dtype=torch.int32, device="cuda")
ctx.generate_device(mtgp.U32, out.data_ptr(), L)
ctx.sync()
ctx.kernel_timing_reset()
ctx.set_option(mtgp.OPT_TIMING, 1)
reps = 3
t0 = time.perf_counter()
for _ in range(reps):
    ctx.generate_device(mtgp.U32, out.data_ptr(), L)
ctx.sync()
wall = time.perf_counter() - t0
g, gn, _, _ = ctx.kernel_timing()
print(json.dumps({"engine": "mt19937", "streams": S, "words_per_stream": L, "kernel_ms": round(g / gn, 3),
                  "Gwords_per_s": round(S * L / (g / gn / 1e3) / 1e9, 2), "GBps": round(4 * S * L / (g / gn / 1e3) / 1e9, 1),
                  "wall_Gwords_per_s": round(reps * S * L / wall / 1e9, 2)}))

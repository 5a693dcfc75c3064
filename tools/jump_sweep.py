"""Jump-ahead cost per call for each library variant in paper_1501_07701_b200/variants/ (and the
main library) and each MTGP_OPT_JUMP mode, on request shapes of the bench configs:

    python tools/jump_sweep.py [rounds]

Shapes: C2 (200 x 2^27 per call), config 5 shards at 8 GPUs (128 x 2^24), C4 (23209 and
44497, 200 x 2^27), MT19937 (200 x 2^27). Prints one JSON line per (shape, library, mode) with the
best-of-rounds jump milliseconds per call (prefix + jump kernels, CUDA events) and the pieces.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1501_07701_b200 import mtgp, tables  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
SHAPES = [("c2", 11213, 200, 1 << 27, 0), ("c5w8", 11213, 128, 1 << 24, 0), ("c4-23209", 23209, 200, 1 << 27, 0),
          ("c4-44497", 44497, 200, 1 << 27, 0), ("mt19937", 19937, 200, 1 << 27, 0)]
libs = [Path(mtgp.LIB_PATH)] + sorted((ROOT / "paper_1501_07701_b200" / "variants").glob("*.so"))
out = torch.empty((200, 1 << 27), dtype=torch.int32, device="cuda")
for name, mexp, S, L, kind in SHAPES:
    for path in libs:
        lib = mtgp.load_library(str(path))
        for mode in (0, 1):
            if mexp == 19937:
                ctx = mtgp.MtContext([mtgp.mt19937_status()] * S, [5489 + i for i in range(S)], lib=lib)
            else:
                ctx = mtgp.MtgpContext(tables.sets_for(mexp, S), [1] * S, lib=lib)
            ctx.set_option(mtgp.OPT_JUMP, mode)
            ctx.generate_device(kind, out.data_ptr(), L)
            ctx.sync()
            best = None
            for _ in range(rounds):
                ctx.kernel_timing_reset()
                ctx.set_option(mtgp.OPT_TIMING, 1)
                for _ in range(3):
                    ctx.generate_device(kind, out.data_ptr(), L)
                ctx.sync()
                g, gn, j, jn = ctx.kernel_timing()
                ctx.set_option(mtgp.OPT_TIMING, 0)
                jm = j / max(1, jn)
                best = jm if best is None else min(best, jm)
            pieces = ctx.last_plan()[0]
            ctx.close()
            print(json.dumps({"shape": name, "lib": path.stem, "jump_mode": mode, "jump_ms": round(best, 4),
                              "pieces": pieces}), flush=True)

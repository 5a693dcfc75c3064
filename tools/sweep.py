"""Time the v2 generation kernel of each library variant in paper_1501_07701_b200/variants/."""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1501_07701_b200 import mtgp, tables  # noqa: E402

words = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 25
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mexp = int(sys.argv[3]) if len(sys.argv) > 3 else 11213
sets = tables.sets_for(mexp, 200)
out = torch.empty((200, words), dtype=torch.int32, device="cuda")
libs = sorted((ROOT / "paper_1501_07701_b200" / "variants").glob("*.so"))
libs.insert(0, mtgp.LIB_PATH)
for path in libs:
    lib = mtgp.load_library(str(path))
    ctx = mtgp.MtgpContext(sets, [1] * 200, lib=lib)
    for _ in range(2):
        ctx.generate_device(kind, out.data_ptr(), words)
    ctx.sync()
    ctx.kernel_timing_reset()
    ctx.set_option(mtgp.OPT_TIMING, 1)
    for _ in range(4):
        ctx.generate_device(kind, out.data_ptr(), words)
    g, gn, j, jn = ctx.kernel_timing()
    pieces, _, kv = ctx.last_plan()
    ctx.close()
    gbs = 4.0 * 200 * words / (g / gn / 1e3) / 1e9
    print(json.dumps({"variant": path.stem, "gen_ms": round(g / gn, 4), "gen_GBps": round(gbs, 1),
                      "jump_ms": round(j / max(1, jn), 4), "pieces": pieces, "kernel": kv, "kind": kind, "mexp": mexp}), flush=True)

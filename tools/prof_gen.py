"""Small driver for ncu captures of the generation kernels (one GPU).

    python tools/prof_gen.py --calls 3 --words 16777216 [--mexp 11213|23209|44497|19937] [--kind 0]
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_1501_07701_b200 import mtgp, tables  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sets", type=int, default=200)
ap.add_argument("--mexp", type=int, default=11213)
ap.add_argument("--kind", type=int, default=0)
ap.add_argument("--words", type=int, default=1 << 24)
ap.add_argument("--calls", type=int, default=3)
ap.add_argument("--kernel", type=int, default=0)
ap.add_argument("--no-checksum", action="store_true")
ap.add_argument("--ck", type=int, default=2, help="MTGP_OPT_CHECKSUM mode (bench default 2)")
a = ap.parse_args()
if a.mexp == 19937:  # Engine::mt MT19937 streams (bench.py --config mt19937)
    ctx = mtgp.MtContext([mtgp.mt19937_status()] * a.sets, [5489 + i for i in range(a.sets)])
else:
    ctx = mtgp.MtgpContext(tables.sets_for(a.mexp, a.sets), [1] * a.sets)
ctx.set_option(mtgp.OPT_KERNEL, a.kernel)
ctx.set_option(mtgp.OPT_CHECKSUM, 0 if a.no_checksum else a.ck)
out = torch.empty((a.sets, a.words), dtype=torch.int32, device="cuda")
for _ in range(a.calls):
    ctx.generate_device(a.kind, out.data_ptr(), a.words)
ctx.sync()
print("plan", ctx.last_plan(), "launches", ctx.launch_count())
ctx.close()

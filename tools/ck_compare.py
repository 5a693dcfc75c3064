"""Compare per-stream checksums of the main library with each variant in
paper_1501_07701_b200/variants/ on one C2-shaped call (200 sets x L words): variants that change
the checksum accumulation must agree exactly.   python tools/ck_compare.py [L]"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1501_07701_b200 import mtgp, tables  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
sets = tables.sets_for(11213, 200)
out = torch.empty((200, L), dtype=torch.int32, device="cuda")
res = {}
for path in [Path(mtgp.LIB_PATH)] + sorted((ROOT / "paper_1501_07701_b200" / "variants").glob("*.so")):
    ctx = mtgp.MtgpContext(sets, [1] * 200, lib=mtgp.load_library(str(path)))
    for kind in (0, 1, 2):
        ctx.generate_device(kind, out.data_ptr(), L)
    ctx.sync()
    res[path.stem] = ctx.checksums()
    print(path.stem, ctx.last_plan(), res[path.stem][0])
    ctx.close()
base = res.pop("libmtgp_b200")
for k, v in res.items():
    print(k, "checksums identical" if v == base else "CHECKSUMS DIFFER")
    assert v == base

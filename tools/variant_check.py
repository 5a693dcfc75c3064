"""Every library variant in paper_1501_07701_b200/variants/ must produce the same words as the
main library: 200 streams x (2 calls of L words), checksums (sum64, xor32) compared per stream,
plus the first and last 4096 words of stream 0 vs the oracle.

    python tools/variant_check.py [L] [mexp]
"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle_py  # noqa: E402
from paper_1501_07701_b200 import mtgp, tables  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 24
mexp = int(sys.argv[2]) if len(sys.argv) > 2 else 11213
sets = tables.sets_for(mexp, 200)
out = torch.empty((200, L), dtype=torch.int32, device="cuda")
libs = [mtgp.LIB_PATH] + sorted((ROOT / "paper_1501_07701_b200" / "variants").glob("*.so"))
ref = None
ok = True
o0 = oracle_py.MtgpOracle(sets[0], 1)
o0.skip(L)
tail_ref = o0.fill(L)[-4096:]
for path in libs:
    lib = mtgp.load_library(str(path))
    ctx = mtgp.MtgpContext(sets, [1] * 200, lib=lib)
    ctx.set_option(mtgp.OPT_CHECKSUM, 1)
    for _ in range(2):
        ctx.generate_device(0, out.data_ptr(), L)
    ctx.sync()
    ck = [(c[0], c[1]) for c in ctx.checksums()]
    tail = out[0, -4096:].cpu().numpy().view(np.uint32)
    good = np.array_equal(tail, tail_ref)
    if ref is None:
        ref = ck
    same = ck == ref
    ok &= same and good
    print(f"{Path(path).stem}: checksums {'==' if same else '!='} main, stream-0 tail vs oracle {'ok' if good else 'BAD'}",
          flush=True)
    ctx.close()
sys.exit(0 if ok else 1)

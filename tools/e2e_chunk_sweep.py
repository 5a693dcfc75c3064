"""e2e (mtgp_generate into pinned host memory) vs MTGP_OPT_HOST_CHUNK, 200 x 2^20 words per call."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
from paper_1501_07701_b200 import mtgp, tables
S, Le = 200, 1 << 20
sets = tables.sets_for(11213, S)
host = torch.empty((S, Le), dtype=torch.int32, pin_memory=True)
hv = host.numpy().view(np.uint32)
for hc in (1 << 15, 1 << 16, 1 << 17, 1 << 18, 1 << 19):
    ctx = mtgp.MtgpContext(sets, [1] * S)
    ctx.set_option(mtgp.OPT_HOST_CHUNK, hc)
    ctx.generate_host(0, Le, out=hv)
    best = 0
    for r in range(3):
        t0 = time.perf_counter()
        for _ in range(5):
            ctx.generate_host(0, Le, out=hv)
        el = time.perf_counter() - t0
        best = max(best, S * Le * 5 / el / 1e9)
    print(json.dumps({"host_chunk": hc, "e2e_Gsamples_s": round(best, 3), "GBps": round(4 * best, 2)}))
    ctx.close()

"""First-call latency of a fresh one-stream context (what a sieve cell's make_word_source pays):
context creation, the first 2^20-word host call (incl. the one-off annihilator analysis and plan
when the call is split into jump-ahead pieces), and a second call.   python tools/first_call.py"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402

from paper_1501_07701_b200 import mtgp, tables  # noqa: E402

sets = tables.load_curand_11213()
for rep in range(3):
    for eng in ("mtgp32-11213", "mt19937"):
        for L in (1 << 18, 1 << 20, 1 << 22):
            t0 = time.perf_counter()
            ctx = (mtgp.MtgpContext(sets[rep:rep + 1], [1]) if eng.startswith("mtgp")
                   else mtgp.MtContext([mtgp.mt19937_status()], [5489 + rep]))
            t1 = time.perf_counter()
            out = np.empty((1, L), np.uint32)
            ctx.generate_host(mtgp.U32, L, out=out)
            t2 = time.perf_counter()
            ctx.generate_host(mtgp.U32, L, out=out)
            t3 = time.perf_counter()
            print(json.dumps({"engine": eng, "L": L, "create_ms": round((t1 - t0) * 1e3, 2),
                              "first_call_ms": round((t2 - t1) * 1e3, 2), "second_call_ms": round((t3 - t2) * 1e3, 2),
                              "pieces": ctx.last_plan()[0]}), flush=True)
            ctx.close()

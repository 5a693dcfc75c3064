"""Run one desk stat test on 200 certified MTGP32-11213 streams (for ncu launch lists).
    python tools/stat_one.py [gap|hamming|opso|walk] [reps] [library.so]"""
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_1501_07701_b200 import mtgp, shard  # noqa: E402
from paper_1501_07701_b200 import stattests as st  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "walk"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = {"gap": st.desk_gap_spec, "hamming": st.desk_hamming_spec, "opso": st.desk_opso_spec,
        "walk": st.desk_walk_spec}[which]()
sets = shard.sets_for_rank(11213, 200, 0)
lib = mtgp.load_library(sys.argv[3]) if len(sys.argv) > 3 else None
with mtgp.MtgpContext(sets, list(range(1, 201)), lib=lib) as ctx:
    ctx.stat_run(spec)
    for _ in range(reps):
        t0 = time.perf_counter()
        ctx.stat_run(spec)
        print(which, f"{(time.perf_counter() - t0) * 1e3:.2f} ms")

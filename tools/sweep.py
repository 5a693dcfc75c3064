"""Time the generation kernel of each library variant in paper_1501_07701_b200/variants/.

Variants are measured in interleaved rounds (A B C A B C ...) so power-cap clock drift does not
favour whichever ran first; the SM clock is sampled through NVML during each measurement and
the result is reported both as GB/s and as SM cycles per launch (clock-independent).

    python tools/sweep.py [words_per_stream] [kind] [mexp] [rounds] [cksum] [sustain_seconds] [kernels]

kernels: comma-separated MTGP_OPT_KERNEL values to compare within each library (default 0 = auto).
mexp 19937 means Engine::mt MT19937 streams (the reference's preset, seeds 5489 + i).

sustain_seconds > 0: instead of best-of short bursts, each variant generates back to back for
that long per round (the power-capped regime the bench runs in) and the AVERAGE rate is kept.
"""
import json
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_1501_07701_b200 import mtgp, tables  # noqa: E402

words = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 25
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 0
mexp = int(sys.argv[3]) if len(sys.argv) > 3 else 11213
rounds = int(sys.argv[4]) if len(sys.argv) > 4 else 3
cks = [int(c) for c in sys.argv[5].split(",")] if len(sys.argv) > 5 else [1]  # MTGP_OPT_CHECKSUM modes
sustain = float(sys.argv[6]) if len(sys.argv) > 6 else 0.0
kernels = [int(k) for k in sys.argv[7].split(",")] if len(sys.argv) > 7 else [0]  # MTGP_OPT_KERNEL values

try:
    import pynvml
    pynvml.nvmlInit()
    nv = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
except Exception:  # noqa: BLE001
    nv = None


class Clock:
    def __init__(self):
        self.samples, self.stop = [], False

    def run(self):
        while not self.stop:
            if nv is not None:
                self.samples.append(pynvml.nvmlDeviceGetClockInfo(nv, pynvml.NVML_CLOCK_SM))
            time.sleep(0.002)


sets = None if mexp == 19937 else tables.sets_for(mexp, 200)
out = torch.empty((200, words), dtype=torch.int32, device="cuda")
libs = sorted((ROOT / "paper_1501_07701_b200" / "variants").glob("*.so"))
libs.insert(0, mtgp.LIB_PATH)
ctxs = []
for path in libs:
    lib = mtgp.load_library(str(path))
    for kern in kernels:
        for ck in cks:
            if sets is None:
                ctx = mtgp.MtContext([mtgp.mt19937_status()] * 200, [5489 + i for i in range(200)], lib=lib)
            else:
                ctx = mtgp.MtgpContext(sets, [1] * 200, lib=lib)
            ctx.set_option(mtgp.OPT_CHECKSUM, ck)
            ctx.set_option(mtgp.OPT_KERNEL, kern)
            ctx.generate_device(kind, out.data_ptr(), words)  # plan + warm
            ctx.sync()
            ctxs.append((path.stem + ("" if kernels == [0] else f"/k{kern}") + ("" if len(cks) == 1 else f"/ck{ck}"),
                         ctx, ck))
res = {name: [] for name, _, _ in ctxs}
for r in range(rounds):
    for name, ctx, _ in ctxs:
        ctx.kernel_timing_reset()
        ctx.set_option(mtgp.OPT_TIMING, 1)
        clk = Clock()
        th = threading.Thread(target=clk.run)
        th.start()
        t_end = time.perf_counter() + sustain
        calls = 0
        while calls < 2 or time.perf_counter() < t_end:
            ctx.generate_device(kind, out.data_ptr(), words)
            calls += 1
            if sustain:
                ctx.sync()
        g, gn, j, jn = ctx.kernel_timing()
        clk.stop = True
        th.join()
        ctx.set_option(mtgp.OPT_TIMING, 0)
        mhz = statistics.median(clk.samples) if clk.samples else float("nan")
        res[name].append((g / gn, j / max(1, jn), mhz))
for name, ctx, cksum in ctxs:
    pieces, _, kv = ctx.last_plan()
    if sustain:  # the average over the sustained rounds, not the best
        ms = statistics.mean(x[0] for x in res[name])
        best = (ms, statistics.mean(x[1] for x in res[name]), statistics.median(x[2] for x in res[name]))
    else:
        ms = min(x[0] for x in res[name])
        best = min(res[name], key=lambda x: x[0])
    cycles = min(x[0] * 1e-3 * x[2] * 1e6 for x in res[name])
    print(json.dumps({"variant": name, "gen_ms": round(ms, 4), "gen_GBps": round(4.0 * 200 * words / (ms / 1e3) / 1e9, 1),
                      "mcycles_per_launch": round(cycles / 1e6, 3), "mhz_at_best": best[2],
                      "jump_ms": round(best[1], 4), "pieces": pieces, "kernel": kv, "kind": kind, "mexp": mexp, "cksum": cksum,
                      "sustain_s": sustain}),
          flush=True)
    ctx.close()

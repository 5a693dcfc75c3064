"""Engine::mt next_f64_01 generation throughput: register-resident teams (auto) vs CTA per stream."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_1501_07701_b200 import mtgp
S, L = 200, 1 << 25
for kern in (0, 1):
    ctx = mtgp.MtContext([mtgp.mt19937_status()] * S, [5489 + i for i in range(S)])
    ctx.set_option(mtgp.OPT_KERNEL, kern)
    out = torch.empty((S, L), dtype=torch.float64, device="cuda")
    ctx.generate_device(mtgp.F64_01, out.data_ptr(), L); ctx.sync()
    ctx.kernel_timing_reset(); ctx.set_option(mtgp.OPT_TIMING, 1)
    for _ in range(3):
        ctx.generate_device(mtgp.F64_01, out.data_ptr(), L)
    ctx.sync()
    g, gn, j, jn = ctx.kernel_timing()
    ms = g / gn
    print(json.dumps({"engine": "mt19937", "kind": "f64_01", "kernel": ctx.last_plan()[2], "streams": S, "words_per_stream": L,
                      "gen_ms": round(ms, 3), "Gsamples_per_s": round(S * L / ms / 1e6, 1), "GBps": round(8 * S * L / ms / 1e6, 1),
                      "jump_ms": round(j / max(1, jn), 3)}))
    ctx.close(); del out; torch.cuda.empty_cache()

"""Diagnostic: NVML clocks / power / limits while the generator saturates the GPU (for the bench
clock sampler and the sw_power_cap analysis in DESIGN.md)."""
import threading, time, json, sys
import numpy as np, torch, pynvml
sys.path.insert(0, ".")
from paper_1501_07701_b200 import mtgp, shard

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
info = {}
for name, fn in (("power_limit_mw", pynvml.nvmlDeviceGetPowerManagementLimit),
                 ("enforced_limit_mw", pynvml.nvmlDeviceGetEnforcedPowerLimit),
                 ("default_limit_mw", pynvml.nvmlDeviceGetPowerManagementDefaultLimit)):
    try:
        info[name] = fn(h)
    except Exception as e:  # noqa: BLE001
        info[name] = str(e)
FI = getattr(pynvml, "NVML_FI_DEV_POWER_INSTANT", 186)
rows = []
stop = False

def loop():
    while not stop:
        t0 = time.perf_counter()
        mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
        pw = pynvml.nvmlDeviceGetPowerUsage(h)
        try:
            fv = pynvml.nvmlDeviceGetFieldValues(h, [FI])[0]
            inst = fv.value.uiVal if fv.nvmlReturn == 0 else -1
        except Exception:  # noqa: BLE001
            inst = -2
        rows.append((round((t0 - T0) * 1e3, 1), mhz, rs, pw, inst))
        time.sleep(0.01)

kind = int(sys.argv[1]) if len(sys.argv) > 1 else mtgp.U32
cksum = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sets = shard.sets_for_rank(11213, 200, 0)
ctx = mtgp.MtgpContext(sets, list(range(1, 201)), device=0)
ctx.set_option(mtgp.OPT_CHECKSUM, cksum)
L = 1 << 27
buf = torch.empty((200, L), dtype=torch.int32, device="cuda")
for _ in range(3):
    ctx.generate_device(kind, buf.data_ptr(), L)
ctx.sync()
time.sleep(0.5)
T0 = time.perf_counter()
th = threading.Thread(target=loop, daemon=True); th.start()
time.sleep(0.1)
T1 = time.perf_counter()
for _ in range(60):
    ctx.generate_device(kind, buf.data_ptr(), L)
ctx.sync()
T2 = time.perf_counter()
time.sleep(0.2)
stop = True; th.join()
info.update({"kind": kind, "cksum": cksum, "load_s": T2 - T1, "Gsamples_s_wall": 60 * 200 * L / (T2 - T1) / 1e9,
             "rows_ms_mhz_reasons_powmw_instmw": rows})
print(json.dumps(info))

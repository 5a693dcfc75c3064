"""Raw device->host bandwidth into pinned memory (the ceiling for bench.py's e2e leg)."""
import json
import torch

dev = torch.device("cuda")
res = {}
for mb in (64, 256, 1024):
    n = mb << 20
    src = torch.empty(n, dtype=torch.uint8, device=dev)
    dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dst.copy_(src, non_blocking=True)
    e1.record()
    e1.synchronize()
    res[f"d2h_{mb}MB_GBps"] = round(5 * n / (e0.elapsed_time(e1) / 1e3) / 1e9, 2)
# two streams at once (two copy engines?)
n = 512 << 20
srcs = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(2)]
dsts = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
sts = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
import time
t0 = time.perf_counter()
for _ in range(5):
    for s, a, b in zip(sts, srcs, dsts):
        with torch.cuda.stream(s):
            b.copy_(a, non_blocking=True)
torch.cuda.synchronize()
res["d2h_2streams_GBps"] = round(2 * 5 * n / (time.perf_counter() - t0) / 1e9, 2)
# strided 2-D copy like the staging path (200 rows)
rows, L = 200, 1 << 18
src = torch.empty((rows, L), dtype=torch.int32, device=dev)
big = torch.empty((rows, 4 * L), dtype=torch.int32, pin_memory=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(4):
    big[:, k * L:(k + 1) * L].copy_(src, non_blocking=True)
e1.record()
e1.synchronize()
res["d2h_2d_200rows_GBps"] = round(4 * rows * L * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9, 2)
print(json.dumps(res))

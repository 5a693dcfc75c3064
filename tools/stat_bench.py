"""Throughput of the device-side stat tests (the reference's desk battery) -> JSON lines.

GPU: every test of stat_tests.cpp's desk_battery() over S streams in one context
(mtgp_stat_run), timed by wall clock around the synchronous call (generation + counting + the
host finish; the words never leave the GPU). Reported as campaign cells/s and stream words
consumed/s.

CPU reference: the reference's own campaign cell (oracle/ref_stat_harness.cpp ref_stat_run_cell =
make_word_source -> BufferedStream -> run_test, sieve.cpp:156-158) on Engine::mt MT19937
streams, one cell per host thread, all host threads (ctypes drops the GIL). The reference has no
MTGP32, so the like-for-like GPU line is the same MT19937 cells through Engine::mt on the GPU.

    python tools/stat_bench.py [--streams 200] [--cpu-cells 64]
"""
import argparse
import json
import os
import sys
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

from paper_1501_07701_b200 import mtgp, shard  # noqa: E402
from paper_1501_07701_b200 import stattests as st  # noqa: E402


def gpu_battery(ctx, reps: int = 3):
    out = []
    for spec in st.desk_battery():
        ctx.stat_run(spec)  # warm (allocations, planner)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            res = ctx.stat_run(spec)
            ts.append(time.perf_counter() - t0)
        t = sorted(ts)[len(ts) // 2]
        words = sum(r.words_used for r in res)
        out.append({"test": spec.test_id, "streams": ctx.n_sets, "seconds": round(t, 5),
                    "runs_s": [round(x, 5) for x in ts],
                    "cells_per_s": round(ctx.n_sets / t, 1), "Gwords_per_s": round(words / t / 1e9, 2),
                    "words_per_stream": words // ctx.n_sets,
                    "classes": {c: sum(r.classification == c for r in res) for c in st.CLASSES}})
    return out


def cpu_reference(n_cells: int, threads: int):
    import stat_oracle as so
    out = []
    for spec in st.desk_battery():
        seeds = [5489 + j for j in range(n_cells)]
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            res = list(ex.map(lambda s: so.ref_run_cell(s, spec), seeds))
        t = time.perf_counter() - t0
        assert all(r["rc"] == 0 for r in res)
        out.append({"test": spec.test_id, "cells": n_cells, "threads": threads, "seconds": round(t, 4),
                    "cells_per_s": round(n_cells / t, 2)})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=200)
    ap.add_argument("--cpu-cells", type=int, default=64)
    ap.add_argument("--only", default="", help="run one desk test on the MTGP32 streams only (for ncu)")
    a = ap.parse_args()
    if a.only:
        sets = shard.sets_for_rank(11213, 200, 0)[:a.streams]
        with mtgp.MtgpContext(sets, [1] * len(sets)) as ctx:
            ctx.stat_run(st.named_spec(a.only))
        return
    lines = []
    sets = shard.sets_for_rank(11213, 200, 0)[:a.streams]
    with mtgp.MtgpContext(sets, [1] * len(sets)) as ctx:
        for row in gpu_battery(ctx):
            lines.append({"arm": "gpu", "engine": "mtgp32-11213", **row})
    with mtgp.MtContext([mtgp.mt19937_status()] * a.streams, [5489 + j for j in range(a.streams)]) as ctx:
        for row in gpu_battery(ctx):
            lines.append({"arm": "gpu", "engine": "mt19937 (Engine::mt)", **row})
    threads = len(os.sched_getaffinity(0))
    for row in cpu_reference(a.cpu_cells, threads):
        lines.append({"arm": "cpu-reference", "engine": "mt19937", **row})
    for ln in lines:
        print(json.dumps(ln))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""bench.py -- MTGP32 bulk generation throughput on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE config 2 -- the 200 certified MTGP32-11213 parameter sets of
the CUDA toolkit, seed 1 each, 2^28 uint32 per set per step. One step = the next 2^28 words of
every stream (214.7 GB written), produced as --calls device calls of 2^28/calls words per
stream into one reused device buffer (the step's output exceeds HBM). Streams advance across
steps; nothing is cached or skipped.

Multi-GPU (torchrun): weak scaling. Rank r owns parameter sets [200r, 200r+200) (the cuRAND
sets for r=0, deterministic synthetic MTGP-11213 sets beyond), no collective on the hot path;
after timing, the per-stream checksums are gathered over NCCL (the only collective).

--impl reference: the CPU implementation of the same path on the box's host cores, rank 0 only,
same config, metric and unit. The reference implements no MTGP32, so for the
MTGP32 configs this is the MTGP32 CPU port (oracle/mtgp32_oracle.c, the restatement the
parity fixtures come from): the config's parameter sets and seeds, every stream filled through
a reused 2^20-word buffer (WordSource::fill semantics), one stream per thread at a time on all
cores, a bounded sample of each stream per step (cpu_baseline.kind "port"). The reference's own
generator (oracle/_ref: proj/src/{generator,params,word_source}.cpp compiled from its sources,
MT19937 through make_word_source()/WordSource::fill) is timed beside it as a side field, and is
the arm itself for --config mt19937.
"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

PEAKS = ROOT / "MEASURED_PEAKS.json"
CONFIGS = {
    # name: (mexp, kind, words per set per step, workload label)
    "c2": (11213, 0, 1 << 28, "MTGP32-11213 x200 sets, 2^28 u32/set/step (BASELINE config 2)"),
    "c3-f12": (11213, 1, 1 << 28, "MTGP32-11213 x200 sets, 2^28 f32 [1,2)/set/step (BASELINE config 3)"),
    "c3-f01": (11213, 2, 1 << 28, "MTGP32-11213 x200 sets, 2^28 f32 (0,1]/set/step (BASELINE config 3)"),
    "c4-23209": (23209, 0, 1 << 28, "MTGP32-23209 x200 synthetic sets, 2^28 u32/set/step (BASELINE config 4)"),
    "c4-44497": (44497, 0, 1 << 28, "MTGP32-44497 x200 synthetic sets, 2^28 u32/set/step (BASELINE config 4)"),
    # BASELINE config 5: 1024 sets in total (200 certified + 824 synthetic) split into contiguous
    # balanced ranges over the ranks, 2^34 outputs per step in total (2^24 per set): strong scaling
    "c5": (11213, 0, 1 << 24, "MTGP32-11213 x1024 sets split across the ranks, 2^24 u32/set/step = 2^34 "
                              "u32/step in total (BASELINE config 5)"),
    # the reference's own recurrence (Engine::mt) on the GPU: like for like with --impl reference
    "mt19937": (19937, 0, 1 << 28, "Engine::mt MT19937 x200 streams (seeds 5489+i), 2^28 u32/stream/step "
                                   "(the reference arm's generator, on the GPU)"),
}
MT_CONFIGS = {"mt19937"}
C5_SETS = 1024


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--sets", type=int, default=200)
    ap.add_argument("--calls", type=int, default=None,
                    help="device calls per step (output buffer = step/calls); default 2, 1 for c5")
    ap.add_argument("--no-checksum", action="store_true")
    ap.add_argument("--checksum-mode", type=int, default=2, choices=[1, 2],
                    help="MTGP_OPT_CHECKSUM: 1 sum64 + xor32, 2 sum32 + xor32 (the fixture's sums mod 2^32)")
    ap.add_argument("--min-piece-words", type=int, default=None, help="MTGP_OPT_MIN_PIECE_WORDS (default: library's)")
    ap.add_argument("--max-pieces", type=int, default=None, help="MTGP_OPT_MAX_PIECES (cap on teams/pieces per call)")
    ap.add_argument("--prejump", type=int, default=None, choices=[0, 1, 2],
                    help="MTGP_OPT_PREJUMP: speculative next-call jumps, 0 auto (library default), 1 off, 2 on")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=1, help="end-to-end (host output) steps timed")
    ap.add_argument("--e2e-words-per-call", type=int, default=1 << 20,
                    help="words per stream per mtgp_generate call in the e2e leg (reused pinned buffer)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-words-per-thread", type=int, default=1 << 28,
                    help="MT19937 reference (oracle/_ref): words per thread per step")
    ap.add_argument("--cpu-words-per-stream", type=int, default=1 << 26,
                    help="MTGP32 CPU port: words of every stream per step (a bounded sample of the step)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="collectives backend under torchrun (nccl; gloo only for --share-device smoke runs)")
    ap.add_argument("--share-device", action="store_true",
                    help="map every rank onto the visible GPUs modulo their count (multi-rank smoke run on one GPU)")
    ap.add_argument("--as-rank", type=int, default=None,
                    help="single process: generate rank R's shard of a multi-GPU run (its parameter sets / seeds), "
                         "to time every rank's workload alone on one GPU")
    ap.add_argument("--as-world", type=int, default=None, help="with --as-rank: the world size to shard for (c5)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """SM clock + throttle reasons sampled DURING the timed region (the profiling recipe's clocks
    line): NVML in-process every 10 ms; falls back to an nvidia-smi subprocess."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.t = None
        self.nv = None
        self.stop_flag = False
        self.nvml_rows = []
        self.first = 0

    def _nvml_loop(self):
        import pynvml
        mx = pynvml.nvmlDeviceGetMaxClockInfo(self.nv, pynvml.NVML_CLOCK_SM)
        pw, i = None, 0
        while not self.stop_flag:
            try:  # SM clock + reasons every 5 ms; power (a slower query) every 4th sample
                mhz = pynvml.nvmlDeviceGetClockInfo(self.nv, pynvml.NVML_CLOCK_SM)
                rs = pynvml.nvmlDeviceGetCurrentClocksEventReasons(self.nv)
                if i % 4 == 0:
                    pw = pynvml.nvmlDeviceGetPowerUsage(self.nv) / 1000.0
                self.nvml_rows.append((mhz, mx, rs, pw))
            except Exception:  # noqa: BLE001
                pass
            i += 1
            time.sleep(0.005)

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.t = threading.Thread(target=self._nvml_loop, daemon=True)
            self.t.start()
            # NVML's first clock queries can take tens of ms: return once the loop is sampling,
            # then keep only the samples taken from now on (the timed region)
            t_end = time.perf_counter() + 1.0
            while not self.nvml_rows and time.perf_counter() < t_end:
                time.sleep(0.001)
            self.first = len(self.nvml_rows)
            return
        except Exception:  # noqa: BLE001
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.nv is not None:
            import pynvml
            self.stop_flag = True
            self.t.join(timeout=2)
            rows = self.nvml_rows[self.first:] or self.nvml_rows[-1:]
            self.nvml_rows = rows
            sm = [r[0] for r in self.nvml_rows]
            smax = float(self.nvml_rows[-1][1]) if self.nvml_rows else None
            reasons = set()
            for r in self.nvml_rows:
                for name, attr in self.REASONS:
                    if r[2] & getattr(pynvml, attr, 0):
                        reasons.add(name)
            loaded = [v for v in sm if smax and v > 0.5 * smax] or sm
            return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": smax,
                    "sm_mhz_min": float(min(loaded)) if loaded else None, "reasons": sorted(reasons),
                    "power_w_max": max((r[3] for r in self.nvml_rows if r[3] is not None), default=None),
                    "samples": len(sm), "source": "nvml, 5 ms"}
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.t:
            self.t.join(timeout=2)
        sm = []
        reasons = set()
        smax = None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
            except ValueError:
                continue
            for n, v in zip(names, r[3:]):
                if v.lower() == "active":
                    reasons.add(n)
        loaded = [v for v in sm if smax and v > 0.5 * smax] or sm
        return {"sm_mhz": float(np.median(loaded)) if loaded else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    if PEAKS.exists():
        d = json.loads(PEAKS.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_per_launch(algo_bytes: float, kver: int, mexp: int):
    """DRAM read+write bytes of one launch of the timed generation kernel, scaled from that
    kernel's committed ncu --set full capture (profiles/traffic.json); (None, None) when the
    kernel has no capture."""
    f = ROOT / "profiles" / "traffic.json"
    if not f.exists():
        return None, None
    ks = json.loads(f.read_text())["kernels"]
    k = ks.get(f"{kver}:{mexp}") or ks.get(str(kver))
    if k is None:
        return None, None
    return round(k["traffic_over_algorithmic"] * algo_bytes), f"{k['source']} ({k['kernel']})"


def full_ck():
    """tests/golden/full_ck.py: the oracle's cumulative per-stream checksums (checker data)."""
    sys.path.insert(0, str(ROOT / "tests" / "golden"))
    import full_ck as fc
    return fc


def cpu_reference(words_per_thread: int, threads: int):
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle_py
    secs, _ = oracle_py.ref_bulk_throughput(threads, words_per_thread, 1 << 18, 5489)
    return threads * words_per_thread / secs / 1e9, secs


def config_sets(args, shard_rank: int = 0, shard_world: int = 1):
    """(parameter sets, seeds, global first set) of a config for one rank, as the GPU arm uses."""
    from paper_1501_07701_b200 import mtgp, shard, tables
    mexp, _, _, _ = CONFIGS[args.config]
    S = args.sets
    if args.config in MT_CONFIGS:
        return [mtgp.mt19937_status()] * S, [5489 + shard_rank * S + i for i in range(S)], shard_rank * S
    if args.config == "c5":
        r = shard.status_range(C5_SETS, shard_rank, shard_world)
        return tables.sets_for(mexp, len(r), first=r.start), [1] * len(r), r.start
    return shard.sets_for_rank(mexp, S, shard_rank), [1] * S, shard_rank * S


def cpu_port_step(sets, seeds, n: int, kind: int, cores: int):
    """One step of the CPU port: every stream's next n words (fill() into a reused buffer)."""
    sys.path.insert(0, str(ROOT / "oracle"))
    import oracle_py
    secs = oracle_py.fill_bulk(sets, seeds, n, 1 << 20, kind, cores)
    return len(sets) * n / secs / 1e9, secs


def run_reference(args, rank, world):
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    mexp, kind, L, label = CONFIGS[args.config]
    is_mt = args.config in MT_CONFIGS
    vals, secs = [], []
    if is_mt:
        wpt = args.cpu_words_per_thread
        for _ in range(args.warmup):
            cpu_reference(wpt // 8, cores)
        for _ in range(args.steps):
            v, sec = cpu_reference(wpt, cores)
            vals.append(v)
            secs.append(sec)
        sample = f"{cores} threads x {wpt} MT19937 words in 2^18-word fill() calls per step"
        kind_s, impl = "reference", "oracle/_ref: the reference's MtWordSource::fill compiled from its sources"
        S = args.sets
    else:
        sets, seeds, _ = config_sets(args)
        S = len(sets)
        n = min(args.cpu_words_per_stream, L)
        for _ in range(args.warmup):
            cpu_port_step(sets, seeds, max(1, n // 8), kind, cores)
        for _ in range(args.steps):
            v, sec = cpu_port_step(sets, seeds, n, kind, cores)
            vals.append(v)
            secs.append(sec)
        sample = (f"all {S} streams of the config x the first {n} words each per step (of {L} per step on the GPU), "
                  f"2^20-word fill() buffer reused per thread, {cores} threads")
        kind_s, impl = "port", "oracle/mtgp32_oracle.c (MTGP32 CPU port; the reference implements no MTGP32)"
    v = float(np.median(vals))
    line = {
        "impl": "reference",
        "metric": "Gsamples/s (uint32 & float) per GPU and at 1/2/4/8 B200; % of HBM write peak",
        "value": round(v, 4), "unit": "Gsamples/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(1000 * float(np.median(secs)), 3),
        "higher_is_better": True, "scaling": "strong" if args.config == "c5" else "weak", "vs_baseline": None,
        "dtype": ["u32", "f32", "f32"][kind],
        "data": "synthetic (seeded generator streams; no input data)",
        "config": {"workload": label, "sets_per_gpu": S, "seed": 1 if not is_mt else "5489+i",
                   "words_per_set_per_step": L, "implementation": impl},
        "cpu_baseline": {"value": round(v, 4), "unit": "Gsamples/s", "cores": cores, "kind": kind_s, "sample": sample},
        "e2e": {"value": round(v, 4), "unit": "Gsamples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    if not is_mt:  # the reference's own generator (a different recurrence) beside it
        try:
            rv, rs = cpu_reference(args.cpu_words_per_thread, cores)
            line["mt19937_reference"] = {
                "value": round(rv, 4), "unit": "Gsamples/s", "cores": cores, "kind": "reference",
                "sample": f"oracle/_ref MtWordSource::fill (MT19937) x {cores} threads x {args.cpu_words_per_thread} "
                          f"words, {rs:.2f} s"}
        except Exception as e:  # noqa: BLE001
            line["mt19937_reference"] = {"value": None, "error": str(e)[:200]}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_1501_07701_b200 import mtgp, shard, tables

    # one process per GPU: LOCAL_RANK is the device. --dist-backend gloo (collectives on host
    # tensors) with --share-device lets a 2-rank smoke run of this multi-rank path on a 1-GPU
    # box; it is never a scaling measurement (the ranks share one GPU).
    if args.share_device:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    coll_dev = f"cuda:{local}" if args.dist_backend == "nccl" else "cpu"
    if world > 1:
        if args.dist_backend == "nccl":
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # nranks / transport lines on stderr
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    mexp, kind, L_step, label = CONFIGS[args.config]
    S = args.sets
    shard_rank, shard_world = rank, world
    if args.as_rank is not None:
        if world > 1:
            raise SystemExit("--as-rank is for single-process runs")
        shard_rank = args.as_rank
        shard_world = args.as_world or max(1, shard_rank + 1)
    is_c5 = args.config == "c5"
    set_range = None
    if is_c5:  # strong scaling: this rank's contiguous share of the 1024 global set IDs
        set_range = shard.status_range(C5_SETS, shard_rank, shard_world)
        S = len(set_range)
    is_mt = args.config in MT_CONFIGS
    if is_mt:  # MT19937 statuses, distinct seeds per stream (and per rank)
        sets = [mtgp.mt19937_status()] * S
        seeds = [5489 + shard_rank * S + i for i in range(S)]
    elif is_c5:
        sets = tables.sets_for(mexp, S, first=set_range.start)
        seeds = [1] * S
    else:
        sets = shard.sets_for_rank(mexp, S, shard_rank)
        seeds = [1] * S

    def make_ctx(ss, sd):
        return mtgp.MtContext(ss, sd, device=local) if is_mt else mtgp.MtgpContext(ss, sd, device=local)
    calls = max(1, args.calls if args.calls is not None else (1 if is_c5 else 2))
    Lc = L_step // calls
    ctx = make_ctx(sets, seeds)
    ck_mode = 0 if args.no_checksum else args.checksum_mode
    ctx.set_option(mtgp.OPT_CHECKSUM, ck_mode)
    # the fixture's streams: global parameter-set IDs of this rank (c5: its contiguous share)
    first_set = set_range.start if is_c5 else shard_rank * S
    if args.min_piece_words:
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, args.min_piece_words)
    if args.prejump is not None:
        ctx.set_option(mtgp.OPT_PREJUMP, args.prejump)
    if args.max_pieces:
        ctx.set_option(mtgp.OPT_MAX_PIECES, args.max_pieces)
    ext = torch.cuda.ExternalStream(ctx.stream_handle(), device=torch.device("cuda", local))
    out = torch.empty((S, Lc), dtype=torch.int32, device=f"cuda:{local}")

    # correctness gate before timing: first words of stream 0 vs the oracle
    if rank == 0:
        sys.path.insert(0, str(ROOT / "oracle"))
        import oracle_py
        probe = make_ctx(sets[:2], seeds[:2])
        w = probe.generate_host(kind, 4096)
        probe.close()
        ref = (oracle_py.MtOracle(None, seeds[0]).fill(4096) if is_mt
               else oracle_py.MtgpOracle(sets[0], seeds[0]).fill(4096, kind=kind))
        if not np.array_equal(w[0], ref):
            raise SystemExit("parity gate failed: GPU stream 0 differs from the oracle")

    def step():
        for _ in range(calls):
            ctx.generate_device(kind, out.data_ptr(), Lc)

    # full-volume parity, part 1: after the first warm-up step every stream's fused checksums
    # must equal the oracle's for its first L_step words (tests/golden/full_ck.npz)
    parity_first = None
    for w in range(args.warmup):
        step()
        if w == 0 and ck_mode:
            ctx.sync()
            parity_first = full_ck().compare(args.config, first_set, ctx.checksums(), sum_mod32=ck_mode == 2)
    ctx.sync()
    torch.cuda.synchronize()
    ctx.kernel_timing_reset()
    ctx.set_option(mtgp.OPT_TIMING, 1)
    launches0 = ctx.launch_count()

    nvml_index = local
    try:  # map the CUDA device to its NVML index (CUDA_VISIBLE_DEVICES may reorder devices)
        import pynvml
        pynvml.nvmlInit()
        uuid = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
        nvml_index = pynvml.nvmlDeviceGetIndex(pynvml.nvmlDeviceGetHandleByUUID(uuid))
    except Exception:  # noqa: BLE001
        pass
    clocks = ClockSampler(nvml_index)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(ext)
    for _ in range(args.steps):
        step()
    e1.record(ext)
    while not e1.query():  # poll with the GIL released so the clock sampler thread keeps sampling
        time.sleep(0.002)
    e1.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - launches0
    gen_ms, gen_n, jump_ms, jump_n = ctx.kernel_timing()
    ctx.set_option(mtgp.OPT_TIMING, 0)
    pieces, _, kver = ctx.last_plan()

    # write-only store peak on this GPU in this run: a fill of the same output
    # buffer (4*S*Lc bytes, >> L2), best of 3, CUDA events; reported beside the copy-peak roofline
    wp0 = torch.cuda.Event(enable_timing=True)
    wp1 = torch.cuda.Event(enable_timing=True)
    wp_ms = float("inf")
    for _ in range(3):
        wp0.record()
        out.fill_(0)
        wp1.record()
        wp1.synchronize()
        wp_ms = min(wp_ms, wp0.elapsed_time(wp1))
    write_peak = out.numel() * 4 / (wp_ms / 1e3) / 1e9

    if world > 1:
        t = torch.tensor([ms], device=coll_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        # clocks of the whole job: slowest rank's median / minimum SM clock, union of reasons
        names = [n for n, _ in ClockSampler.REASONS]
        lo = torch.tensor([clk.get("sm_mhz") or 0.0, clk.get("sm_mhz_min") or clk.get("sm_mhz") or 0.0],
                          device=coll_dev, dtype=torch.float64)
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        bits = torch.tensor([float(n in clk.get("reasons", [])) for n in names], device=coll_dev,
                            dtype=torch.float64)
        dist.all_reduce(bits, op=dist.ReduceOp.MAX)
        clk = dict(clk, sm_mhz=float(lo[0].item()), sm_mhz_min=float(lo[1].item()),
                   reasons=[n for n, b in zip(names, bits.tolist()) if b > 0], ranks=world,
                   note="min over ranks of each rank's median / min SM clock; union of reasons")
    # per-stream checksum gather (NCCL all_gather; the only inter-GPU traffic)
    allck = shard.gather_checksums(ctx.checksums(), device=coll_dev)
    gathered_streams = len(allck)
    # full-volume parity, part 2: every word of every stream generated in this run (warm-up and
    # timed steps) through the gathered checksums, against the oracle's cumulative checksums
    parity = None
    if rank == 0 and ck_mode:
        gfirst = first_set if (world == 1 or args.as_rank is not None) else 0
        parity = full_ck().compare(args.config, gfirst, allck, sum_mod32=ck_mode == 2)
        parity["after_first_step"] = parity_first
        parity["fixture"] = ("tests/golden/mt_full_ck.npz (the reference's own MtWordSource::fill, oracle/_ref)"
                             if is_mt else "tests/golden/full_ck.npz (oracle/mtgp32_oracle.c cumulative checksums)")

    samples_rank = S * L_step * args.steps
    # whole job: every rank's samples (c5: the 1024 sets, however they are split)
    total = (C5_SETS if is_c5 and args.as_rank is None else S * world) * L_step * args.steps
    value = total / (ms / 1e3) / 1e9
    hbm, hbm_src = peaks()
    bytes_per_launch = 4.0 * S * Lc
    gen_avg_ms = gen_ms / max(1, gen_n)
    achieved = bytes_per_launch / (gen_avg_ms / 1e3) / 1e9
    step_gbs = 4.0 * samples_rank / (ms / 1e3) / 1e9

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = len(os.sched_getaffinity(0))
            if is_mt:  # the reference itself implements this generator
                v, secs = cpu_reference(args.cpu_words_per_thread, cores)
                cpu = {"value": round(v, 4), "unit": "Gsamples/s", "cores": cores, "kind": "reference",
                       "sample": f"reference MtWordSource::fill (MT19937) x {cores} pinned threads x "
                                 f"{args.cpu_words_per_thread} words, {secs:.2f} s wall"}
            else:  # the MTGP32 CPU port on the same sets and seeds
                n = min(args.cpu_words_per_stream, L_step)
                v, secs = cpu_port_step(sets, seeds, n, kind, cores)
                cpu = {"value": round(v, 4), "unit": "Gsamples/s", "cores": cores, "kind": "port",
                       "sample": f"oracle/mtgp32_oracle.c: all {len(sets)} streams x first {n} words, 2^20-word fill() "
                                 f"buffer per thread, {cores} threads, {secs:.2f} s wall"}
                rv, rs = cpu_reference(args.cpu_words_per_thread, cores)
                cpu["mt19937_reference"] = {
                    "value": round(rv, 4), "unit": "Gsamples/s", "cores": cores, "kind": "reference",
                    "sample": f"oracle/_ref MtWordSource::fill (MT19937), the reference's own generator, {cores} "
                              f"threads x {args.cpu_words_per_thread} words, {rs:.2f} s wall"}
        except Exception as e:  # noqa: BLE001
            cpu = {"value": None, "error": str(e)[:200]}

    e2e = None
    if not args.no_e2e:
        # public API, HOST buffers, the whole step's volume: a fresh context (mtgp_ctx_create:
        # parameter table + seeds uploaded, timed separately as the one-off setup), then every
        # step = L_step words of every stream through mtgp_generate(out_is_device=0) into a
        # reused page-locked buffer of Le words per stream (the reference's WordSource::fill
        # pattern), so each timed step holds generation plus the device->host copy of all
        # S * L_step words. Every rank runs it at once (each GPU has its own host link);
        # whole-job samples over the slowest rank's time.
        Le = min(L_step, args.e2e_words_per_call)
        host = torch.empty((S, Le), dtype=torch.int32, pin_memory=True)
        hv = host.numpy().view(np.uint32)
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        ectx = make_ctx(sets, seeds)
        setup_s = time.perf_counter() - t0
        ectx.set_option(mtgp.OPT_HOST_CHUNK, 1 << 18)
        ectx.generate_host(kind, Le, out=hv)  # warm: plan + staging buffers
        calls_e = L_step // Le
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            for _ in range(calls_e):
                ectx.generate_host(kind, Le, out=hv)
        el = time.perf_counter() - t0
        ectx.close()
        if world > 1:
            tt = torch.tensor([el, setup_s], device=coll_dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            el, setup_s = float(tt[0].item()), float(tt[1].item())
        setup_bytes = S * C.sizeof(mtgp.MtParamsC if is_mt else mtgp.MtgpParamsC) + S * 4
        e2e = {"value": round(world * S * L_step * args.e2e_steps / el / 1e9, 4), "unit": "Gsamples/s",
               "h2d_bytes_per_step": 0, "d2h_bytes_per_step": world * S * L_step * 4,
               "steps": args.e2e_steps, "ms_per_step": round(1000 * el / args.e2e_steps, 1),
               "setup": {"ms": round(1000 * setup_s, 2), "h2d_bytes": world * setup_bytes,
                         "what": "mtgp_ctx_create: parameter table + seeds uploaded, state windows seeded "
                                 "(one-off per context, outside the timed steps)"},
               "how": f"mtgp_generate(out_is_device=0): each step = {calls_e} calls x {Le} words x {S} streams "
                      f"into one reused page-locked buffer ({S * Le * 4 / 1e9:.2f} GB), the step's full volume "
                      f"({S * L_step * 4 / 1e9:.1f} GB) copied device->host; {world} GPU(s) at once, max wall "
                      "clock over ranks. No per-step inputs: the only host->device bytes are the setup's"}

    traffic = traffic_per_launch(bytes_per_launch, kver, mexp)
    if rank == 0:
        line = {
            "metric": "Gsamples/s (uint32 & float) per GPU and at 1/2/4/8 B200; % of HBM write peak",
            "value": round(value, 3), "unit": "Gsamples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong" if is_c5 else "weak", "vs_baseline": None,
            "dtype": ["u32", "f32", "f32"][kind],
            "data": "synthetic (seeded generator streams; no input data)",
            "config": {"workload": label, "sets_per_gpu": S, "seed": 1, "words_per_set_per_step": L_step,
                       "calls_per_step": calls, "kernel": f"v{kver}", "pieces_per_call": pieces,
                       "checksums_fused": not args.no_checksum,
                       "prejump": {None: "auto", 0: "auto", 1: "off", 2: "on"}[args.prejump],
                       "checksum_mode": {0: "off", 1: "sum64+xor32", 2: "sum32+xor32"}[ck_mode],
                       **({"as_rank": shard_rank, "as_world": shard_world} if args.as_rank is not None else {}),
                       "global_set_ids": ([set_range.start, set_range.stop] if is_c5
                                          else [shard_rank * S, (shard_rank + 1) * S]),
                       "checksums_gathered_streams": gathered_streams,
                       "collectives": {"backend": args.dist_backend if world > 1 else None, "world": world,
                                       "hot_path": "none (disjoint set-ID shards)",
                                       "after_timing": "per-stream checksum all_gather",
                                       **({"share_device": True, "note": "ranks share one GPU: a smoke run of "
                                           "the multi-rank path, not a scaling measurement"}
                                          if args.share_device and world > 1 else {})},
                       "l2": "output 4*S*L/calls bytes per call >> 126 MB L2; no flush needed",
                       "parameter_sets": ("MT19937 (mt19937_params, proj/src/params.cpp:63-77)" if is_mt
                                          else f"global set IDs {set_range.start}..{set_range.stop - 1}: IDs < 200 "
                                               "cuRAND MTGP32-11213 (certified), the rest synthetic (uncertified period)"
                                          if is_c5
                                          else "synthetic (uncertified period)" if mexp != 11213 or S > 200
                                          or shard_rank > 0
                                          else "cuRAND MTGP32-11213 (certified)" if world == 1
                                          else "rank 0: cuRAND MTGP32-11213 (certified); ranks 1..N-1: synthetic "
                                               "MTGP32-11213 (uncertified period)")},
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(achieved / hbm, 4), "traffic": traffic[0],
                         "traffic_source": traffic[1],
                         "peak_source": hbm_src,
                         "kernel": {5: "mt_gen2_kernel (v5, Engine::mt warp teams, shared-memory rings)",
                                    6: "mt_gen3_kernel (v6, Engine::mt register-resident warp teams)"}.get(
                                        kver, f"gen{kver if kver in (3, 4) else ''}_kernel (v{kver})"),
                         "launches_timed": gen_n,
                         "avg_launch_ms": round(gen_avg_ms, 4),
                         "algorithmic_bytes_per_launch": bytes_per_launch,
                         "step_write_GBps": round(step_gbs, 1),
                         "jump_ms_per_call": round(jump_ms / max(1, jump_n), 4),
                         "write_peak_in_run": {"GBps": round(write_peak, 1), "frac": round(achieved / write_peak, 4),
                                               "how": f"torch fill_ of the {out.numel() * 4 / 1e9:.1f} GB output "
                                                      "buffer, best of 3 (write-only store peak)"}},
            # BASELINE's metric also asks for "% of HBM write peak": against the write-only store
            # peak measured in this same run (a torch fill_ of the output buffer)
            "hbm_write_peak_pct": {"kernel": round(100 * achieved / write_peak, 2),
                                   "step": round(100 * step_gbs / write_peak, 2),
                                   "write_peak_GBps": round(write_peak, 1)},
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "parity": parity,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if rank == 0 and parity is not None and (parity.get("ok") is False or
                                             (parity.get("after_first_step") or {}).get("ok") is False):
        raise SystemExit("parity FAILED: GPU checksums differ from the oracle fixture")
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

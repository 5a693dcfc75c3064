"""N>1 host logic on CPU: world_size-2 gloo processes shard parameter-set IDs and gather the
per-stream checksums exactly as bench.py does over NCCL on GPUs. Each rank computes its streams'
checksums with the oracle (standing in for its GPU); rank 0 checks the gathered table."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, sets_per_rank, L, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import torch.distributed as dist

    import oracle_py
    from paper_1501_07701_b200 import shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sets = shard.sets_for_rank(11213, sets_per_rank, rank)
    words, _ = oracle_py.mtgp_bulk(sets, [1] * len(sets), L, threads=2)
    local = [(int(w.astype("uint64").sum()) % (1 << 64), int(__import__("numpy").bitwise_xor.reduce(w)), L)
             for w in words]
    allck = shard.gather_checksums(local)
    if rank == 0:
        q.put(allck)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_gloo_shard_and_gather(world):
    from paper_1501_07701_b200 import shard, tables
    import oracle_py

    sets_per_rank, L = 3, 5000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, sets_per_rank, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    allck = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # disjoint ID ranges covering [0, world*sets_per_rank)
    ids = [i for r in range(world) for i in shard.set_range(r, sets_per_rank)]
    assert ids == list(range(world * sets_per_rank))
    every = tables.sets_for(11213, world * sets_per_rank)
    assert len(allck) == len(every)
    for gid, (p, ck) in enumerate(zip(every, allck)):
        w = oracle_py.MtgpOracle(p, 1).fill(L)
        assert ck == (int(w.astype("uint64").sum()), int(__import__("numpy").bitwise_xor.reduce(w)), L), gid
    # rank 1's sets are the certified cuRAND sets 3..5 (global IDs continue across ranks)
    cur = tables.load_curand_11213()
    assert [s.pos for s in shard.sets_for_rank(11213, sets_per_rank, 1)] == [s.pos for s in cur[3:6]]


def test_sets_beyond_the_table_are_synthetic_and_distinct():
    from paper_1501_07701_b200 import shard
    r7 = shard.sets_for_rank(11213, 200, 7)  # IDs 1400..1599
    assert all(not s.certified for s in r7)
    keys = {(s.pos, s.sh1, s.sh2, tuple(s.tbl)) for s in r7}
    assert len(keys) == 200
    r0 = shard.sets_for_rank(11213, 200, 0)
    assert all(s.certified for s in r0)


def _grid_worker(rank, world, port, n_status, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import torch.distributed as dist

    from paper_1501_07701_b200 import shard, stattests

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    seen = []

    def fake_run_grid(statuses, seeds, specs, status_ids=None, **kw):
        # stands in for the GPU: one row per (status, seed, test), carrying its coordinates
        seen.extend(statuses)
        return [stattests.ResultRow(si, wi, status_ids[si], sp.test_id, seed, statistic=float(statuses[si]))
                for si in range(len(statuses)) for wi, seed in enumerate(seeds) for sp in specs]

    rows = shard.run_grid_distributed(list(range(100, 100 + n_status)), [7, 8], stattests.desk_battery()[:2],
                                      runner=fake_run_grid)
    q.put((rank, seen, [(r.status_index, r.seed_index, r.test_id, r.statistic, r.status_id) for r in rows]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_status", [5, 2, 1])
def test_run_grid_distributed_order_and_coverage(n_status):
    """Campaign cells split over 2 ranks by status; rank 0 gets every row in run_grid's
    (status, seed, test) order, whatever the split (including a rank with no statuses)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grid_worker, args=(r, 2, port, n_status, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(2):
        rank, seen, rows = q.get(timeout=240)
        got[rank] = (seen, rows)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    statuses = list(range(100, 100 + n_status))
    assert sorted(got[0][0] + got[1][0]) == statuses and not set(got[0][0]) & set(got[1][0])
    assert got[1][1] == []
    want = [(si, wi, t, float(statuses[si]), str(si)) for si in range(n_status) for wi in range(2)
            for t in ("gap", "hamming_indep")]
    assert got[0][1] == want


def _worker_strong(rank, world, port, n_total, L, q):
    """bench.py --config c5: rank r owns the balanced contiguous range status_range(n_total, r, world)
    of the global set IDs (uneven when n_total % world != 0); the gather pads and trims."""
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    sys.path.insert(0, str(root / "oracle"))
    import numpy as np
    import torch.distributed as dist

    import oracle_py
    from paper_1501_07701_b200 import shard, tables

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = shard.status_range(n_total, rank, world)
    sets = tables.sets_for(11213, len(rng), first=rng.start)
    words, _ = oracle_py.mtgp_bulk(sets, [1] * len(sets), L, threads=2) if len(sets) else ([], None)
    local = [(int(w.astype("uint64").sum()), int(np.bitwise_xor.reduce(w)), L) for w in words]
    allck = shard.gather_checksums(local)
    if rank == 0:
        q.put(allck)
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_strong_split_uneven_gather():
    from paper_1501_07701_b200 import tables
    import numpy as np
    import oracle_py

    world, n_total, L = 3, 7, 3000  # 3 / 2 / 2 sets; IDs cross nothing (all certified) but shapes differ
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_strong, args=(r, world, port, n_total, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    allck = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    every = tables.sets_for(11213, n_total)
    assert len(allck) == n_total
    for gid, (p, ck) in enumerate(zip(every, allck)):
        w = oracle_py.MtgpOracle(p, 1).fill(L)
        assert ck == (int(w.astype("uint64").sum()), int(np.bitwise_xor.reduce(w)), L), gid


# ---- the single-process multi-GPU batch (C-ABI mtgp_multi, csrc/mtgp_multi.h host logic) ----

def test_multi_host_logic_fake_communicator(tmp_path):
    """Partition + padded all-gather through a fake ring communicator (tests/cpp/test_multi.cpp)."""
    import subprocess
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "test_multi"
    subprocess.run(["g++", "-std=c++17", "-O2", "-I", str(root / "include"), "-I",
                    str(root / "paper_1501_07701_b200/csrc"), str(root / "tests/cpp/test_multi.cpp"), "-o", str(exe)],
                   check=True, capture_output=True, text=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr


def test_shard_range_c_abi_matches_python_split():
    """mtgp_shard_range (the C-ABI's split) == shard.status_range (bench.py's), and the C-ABI
    refuses bad arguments; no device needed."""
    from paper_1501_07701_b200 import mtgp, shard
    for n in (1, 5, 200, 1024, 1601):
        for w in range(1, 9):
            for r in range(w):
                assert mtgp.shard_range(n, w, r) == shard.status_range(n, r, w)
    with pytest.raises(mtgp.MtgpInvalidArgument):
        mtgp.shard_range(10, 2, 2)


def test_multi_create_fails_loudly_without_device():
    import torch
    from paper_1501_07701_b200 import mtgp, tables
    if torch.cuda.is_available():
        pytest.skip("CPU hosts only")
    with pytest.raises(mtgp.MtgpError):
        mtgp.MultiGpu(tables.load_curand_11213()[:4], [1] * 4, [0, 1])

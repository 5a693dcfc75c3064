"""Full-volume parity: every word the bench generates, checked against the oracle.

bench.py's workloads run the DEFAULT auto plan (3744 jump-ahead pieces per 2^27-word call at
config 2, jumps up to 2^27 words) and the in-kernel per-stream checksums accumulate over every
call. Here the same contexts make the same calls, and after EVERY call the cumulative
{sum64, xor32} of every stream must equal the oracle's (tests/golden/full_ck.npz, made by
tests/golden/make_full_ck.py from oracle/mtgp32_oracle.c). The reference's model of parity is
whole-sequence equivalence against an independent implementation (proj/tests/
test_generator.cpp:17-24); the fixture covers 25 bench steps of every config and of
every rank's shard, i.e. every word `bench.py --steps K --warmup W` makes for W + K <= 25.
"""
import sys
from pathlib import Path

import pytest

from paper_1501_07701_b200 import mtgp, shard, tables

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
import full_ck  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not full_ck.available(), reason="full_ck.npz not generated")]

CONFIG_SHAPE = {  # config: (mexp, kind)
    "c2": (11213, mtgp.U32),
    "c3-f12": (11213, mtgp.F32_12),
    "c3-f01": (11213, mtgp.F32_01OC),
    "c4-23209": (23209, mtgp.U32),
    "c4-44497": (44497, mtgp.U32),
    "c5": (11213, mtgp.U32),
}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    yield torch
    torch.cuda.empty_cache()


def _run(torch, config, first_set, n_sets, calls, ck_mode=1):
    """The bench's loop for one rank's shard: `calls` device calls of one record's words per
    stream into one reused buffer, the cumulative checksums compared after every call."""
    mexp, kind = CONFIG_SHAPE[config]
    n, records, rec = full_ck.coverage(config)
    calls = min(calls, records)
    sets = tables.sets_for(mexp, n_sets, first=first_set)
    out = torch.empty((n_sets, rec), dtype=torch.int32, device="cuda")
    with mtgp.MtgpContext(sets, [1] * n_sets) as ctx:
        ctx.set_option(mtgp.OPT_CHECKSUM, ck_mode)
        for k in range(calls):
            ctx.generate_device(kind, out.data_ptr(), rec)
            ctx.sync()
            r = full_ck.compare(config, first_set, ctx.checksums(), sum_mod32=ck_mode == 2)
            assert r["ok"], (config, first_set, k, r)
        pieces, _, kver = ctx.last_plan()
    del out
    return pieces, kver


def test_c2_every_word_of_25_steps(torch_cuda):
    """BASELINE config 2 exactly as the bench runs it (rank 0: the 200 certified sets)."""
    pieces, kver = _run(torch_cuda, "c2", 0, 200, 50)
    assert kver == 3 and pieces > 1000  # the auto plan: gen3 with thousands of jumped pieces


def test_c2_checksum_mode_sum32(torch_cuda):
    """MTGP_OPT_CHECKSUM 2 (32-bit sums): the same words, sums compared mod 2^32."""
    _run(torch_cuda, "c2", 0, 200, 8, ck_mode=2)


@pytest.mark.parametrize("rank", range(1, 8))
def test_c2_every_rank_shard(torch_cuda, rank):
    """The synthetic sets ranks 1..7 of an 8-GPU weak-scaling run generate (bench.py)."""
    _run(torch_cuda, "c2", 200 * rank, 200, 50)


@pytest.mark.parametrize("config", ["c3-f12", "c3-f01"])
def test_c3_float_kinds(torch_cuda, config):
    _run(torch_cuda, config, 0, 200, 50)


@pytest.mark.parametrize("config", ["c4-23209", "c4-44497"])
def test_c4_larger_exponents(torch_cuda, config):
    _run(torch_cuda, config, 0, 200, 50)


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_c5_every_rank_of_every_world(torch_cuda, world):
    """Config 5: 1024 sets split into contiguous balanced ranges (bench.py --config c5); each
    rank's shard has its own plan, every one checked for 25 steps."""
    for rank in range(world):
        r = shard.status_range(1024, rank, world)
        _run(torch_cuda, "c5", r.start, len(r), 25)


@pytest.mark.parametrize("devices,gather", [([0], 1), ([0, 0, 0], 2)])
def test_multi_gpu_batch_c5(torch_cuda, devices, gather):
    """The single-process multi-GPU batch (C-ABI mtgp_multi: one context + host thread per
    device, contiguous set ranges, checksum all-gather over NCCL) on config 5's 1024 sets,
    every word checked through the gathered checksums. gpurun exposes one GPU: one rank with a
    real (single-rank) NCCL communicator, and three ranks sharing device 0 with the host gather."""
    sets = tables.sets_for(11213, 1024)
    with mtgp.MultiGpu(sets, [1] * 1024, devices, gather=gather) as m:
        assert m.nccl == (gather == 1) and m.n_devices == len(devices)
        rs = m.ranges()
        assert [r.start for r in rs] == [shard.status_range(1024, i, len(devices)).start for i in range(len(devices))]
        bufs = [torch_cuda.empty((len(r), 1 << 24), dtype=torch_cuda.int32, device=f"cuda:{d}")
                for r, d in zip(rs, devices)]
        for k in range(3):
            m.generate_device(mtgp.U32, [b.data_ptr() for b in bufs], 1 << 24)
            r = full_ck.compare("c5", 0, m.checksums())
            assert r["ok"] and r["words_per_stream"] == (k + 1) << 24, r
        del bufs


@pytest.mark.skipif(not full_ck.available("mt19937"), reason="mt_full_ck.npz not generated")
def test_mt19937_checksum_mode_sum32(torch_cuda):
    """mt_gen3's 32-bit-sum checksum mode (the bench default) against the reference's fill()."""
    torch = torch_cuda
    n, _, rec = full_ck.coverage("mt19937")
    out = torch.empty((n, rec), dtype=torch.int32, device="cuda")
    with mtgp.MtContext([mtgp.mt19937_status()] * n, [5489 + i for i in range(n)]) as ctx:
        ctx.set_option(mtgp.OPT_CHECKSUM, 2)
        for k in range(6):
            ctx.generate_device(mtgp.U32, out.data_ptr(), rec)
            ctx.sync()
            r = full_ck.compare("mt19937", 0, ctx.checksums(), sum_mod32=True)
            assert r["ok"], (k, r)
        assert ctx.last_plan()[2] == 6
    del out


@pytest.mark.skipif(not full_ck.available("mt19937"), reason="mt_full_ck.npz not generated")
def test_mt19937_every_word_against_the_reference(torch_cuda):
    """bench.py --config mt19937 (Engine::mt, 200 MT19937 streams, seeds 5489 + i) with the
    default auto plan (mt_gen3 warp teams, jump-ahead pieces): after every 2^27-word call the
    cumulative checksums equal those of the reference's own MtWordSource::fill (oracle/_ref,
    tests/golden/make_mt_full_ck.py) -- 25 bench steps, every word."""
    torch = torch_cuda
    n, records, rec = full_ck.coverage("mt19937")
    out = torch.empty((n, rec), dtype=torch.int32, device="cuda")
    with mtgp.MtContext([mtgp.mt19937_status()] * n, [5489 + i for i in range(n)]) as ctx:
        ctx.set_option(mtgp.OPT_CHECKSUM, 1)
        for k in range(records):
            ctx.generate_device(mtgp.U32, out.data_ptr(), rec)
            ctx.sync()
            r = full_ck.compare("mt19937", 0, ctx.checksums())
            assert r["ok"], (k, r)
        pieces, _, kver = ctx.last_plan()
    assert kver == 6 and pieces > 1000
    del out

"""Speculative next-call jumps (MTGP_OPT_PREJUMP; csrc/mtgp_plan.cu Planner::run).

While call k generates, a side stream computes call k+1's jump-ahead piece windows from call
k's prefix; call k+1 uses them only if nothing changed the state in between (the context's
state epoch) and its plan is the same. Every word is compared with the CPU oracle, including
sequences that must invalidate the speculation (skip, state restore, a different length, a
float kind, a stat pass) and the multi-call shapes the bench runs (full-volume fixture)."""
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle_py
from paper_1501_07701_b200 import mtgp, shard, tables

sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
import full_ck  # noqa: E402

pytestmark = pytest.mark.gpu


def _ref(sets, seeds, start, n):
    return oracle_py.mtgp_bulk(sets, seeds, n, skip=start, threads=len(sets))[0]


@pytest.mark.parametrize("mexp", [11213, 23209, 44497])
def test_repeated_calls_with_invalidations(mexp, curand_sets):
    S = 3
    sets = curand_sets[:S] if mexp == 11213 else tables.synthetic_sets(mexp, S, first=7)
    seeds = [11, 22, 33]
    L = 1 << 18
    pos = 0
    buf = torch.empty((S, L), dtype=torch.int32, device="cuda")
    with mtgp.MtgpContext(sets, seeds) as ctx:
        ctx.set_option(mtgp.OPT_PREJUMP, 2)
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 14)  # many jumped pieces per call

        def gen(n=L, kind=mtgp.U32):
            nonlocal pos
            b = buf if n == L else torch.empty((S, n), dtype=torch.int32, device="cuda")
            ctx.generate_device(kind, b.data_ptr(), n)
            ctx.sync()
            got = b.cpu().numpy().view(np.uint32)
            want = _ref(sets, seeds, pos, n)
            if kind == mtgp.F32_12:
                want = ((want >> 9) | 0x3F800000).astype(np.uint32)
            assert np.array_equal(got, want), (mexp, pos, n, kind)
            pos += n
            return ctx.last_plan()[0]

        assert gen() > S  # split into jumped pieces
        gen()
        gen()                       # speculation used (same plan, no state change)
        ctx.skip(1_000_003)         # state change: the speculation must be dropped
        pos += 1_000_003
        gen()
        gen()
        win, positions = ctx.state_save()
        gen()
        ctx.state_restore(win, positions)   # back: the speculation made for the next call is stale
        pos -= L
        gen()
        gen()
        gen(L // 2)                 # a different length: a different plan
        gen()
        gen(kind=mtgp.F32_12)       # another kind: same windows, valid
        gen()


def test_host_output_chunks(curand_sets):
    """The host-output path (one device call per chunk) with the speculation on: every chunk's
    jumps come from the previous chunk's speculation."""
    sets = curand_sets[:2]
    seeds = [5, 6]
    with mtgp.MtgpContext(sets, seeds) as ctx:
        ctx.set_option(mtgp.OPT_PREJUMP, 2)
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 14)
        ctx.set_option(mtgp.OPT_HOST_CHUNK, 1 << 17)
        ctx.skip(1 << 26)  # a long-lived stream (few-stream splitting needs >= 2^25 words done)
        got = ctx.generate_host(mtgp.U32, 1 << 20)
    assert np.array_equal(got, _ref(sets, seeds, 1 << 26, 1 << 20))


@pytest.mark.parametrize("prejump", [0, 2])
def test_c2_every_word_prejump(prejump):
    """The bench's C2 call pattern with the speculation forced on (and auto) for 8 calls."""
    n, _, rec = full_ck.coverage("c2")
    sets = tables.sets_for(11213, 200)
    out = torch.empty((200, rec), dtype=torch.int32, device="cuda")
    with mtgp.MtgpContext(sets, [1] * 200) as ctx:
        ctx.set_option(mtgp.OPT_CHECKSUM, 2)
        ctx.set_option(mtgp.OPT_PREJUMP, prejump)
        for k in range(8):
            ctx.generate_device(mtgp.U32, out.data_ptr(), rec)
            ctx.sync()
            r = full_ck.compare("c2", 0, ctx.checksums(), sum_mod32=True)
            assert r["ok"], (prejump, k, r)
    del out


def test_c5_eight_rank_shards_auto():
    """Config 5 at 8 GPUs: 128 sets per shard leave SM slots free, so the auto mode speculates;
    every shard's 25 calls against the fixture."""
    for rank in (0, 7):
        r = shard.status_range(1024, rank, 8)
        sets = tables.sets_for(11213, len(r), first=r.start)
        out = torch.empty((len(r), 1 << 24), dtype=torch.int32, device="cuda")
        with mtgp.MtgpContext(sets, [1] * len(r)) as ctx:
            ctx.set_option(mtgp.OPT_CHECKSUM, 2)
            for k in range(25):
                ctx.generate_device(mtgp.U32, out.data_ptr(), 1 << 24)
                ctx.sync()
                res = full_ck.compare("c5", r.start, ctx.checksums(), sum_mod32=True)
                assert res["ok"], (rank, k, res)
        del out

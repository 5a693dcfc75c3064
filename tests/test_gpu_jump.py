"""GPU parity of the Karatsuba jump (csrc/mtgp_jump.cu) against the direct jump and the oracle.

Jumped pieces start from windows computed by the jump kernels, so every word of a call with
many pieces depends on them. MTGP_OPT_JUMP = 0 (auto: Karatsuba for N > 384) and 1 (direct)
must give identical words, and both must match the oracle. Bit-exact (integer path).
"""
import numpy as np
import pytest

import oracle_py
from paper_1501_07701_b200 import mtgp, tables

pytestmark = pytest.mark.gpu


def _run_mtgp(sets, seeds, jump, kernel, L1, L2, min_piece):
    with mtgp.MtgpContext(sets, seeds) as ctx:
        ctx.set_option(mtgp.OPT_KERNEL, kernel)
        ctx.set_option(mtgp.OPT_JUMP, jump)
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, min_piece)
        w1 = ctx.fill_u32(L1)
        pieces = ctx.last_plan()[0]
        w2 = ctx.fill_u32(L2)
        ck = ctx.checksums()
    return w1, w2, pieces, ck


@pytest.mark.parametrize("mexp,kernel", [(23209, 2), (23209, 4), (44497, 2), (44497, 4)])
def test_kara_jump_matches_direct_and_oracle(mexp, kernel):
    sets = tables.synthetic_sets(mexp, 5)
    seeds = [7, 8, 9, 10, 11]
    L1, L2 = 400_000, 123_456
    a1, a2, pa, cka = _run_mtgp(sets, seeds, 0, kernel, L1, L2, 4096)
    b1, b2, pb, ckb = _run_mtgp(sets, seeds, 1, kernel, L1, L2, 4096)
    assert pa == pb and pa > 5 * 20
    assert np.array_equal(a1, b1) and np.array_equal(a2, b2) and cka == ckb
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, L1 + L2, threads=8)
    assert np.array_equal(a1, ref[:, :L1])
    assert np.array_equal(a2, ref[:, L1:])


@pytest.mark.parametrize("jump", [0, 2])
def test_split_jump_at_11213(curand_sets, jump):
    """N = 351 <= 384: auto runs the direct jump; mode 2 splits each jump's q blocks over
    several warps (d = 0, partial windows XOR-combined). Both exact."""
    sets = curand_sets[10:14]
    seeds = [1, 2, 3, 4]
    a1, a2, pieces, _ = _run_mtgp(sets, seeds, jump, 3, 200_000, 1000, 4096)
    assert pieces > 4 * 20
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, 201_000, threads=4)
    assert np.array_equal(a1, ref[:, :200_000]) and np.array_equal(a2, ref[:, 200_000:])


@pytest.mark.parametrize("jump", [0, 1, 2])
def test_kara_skip_44497(jump):
    sets = tables.synthetic_sets(44497, 3)
    with mtgp.MtgpContext(sets, [1, 2, 3]) as ctx:
        ctx.set_option(mtgp.OPT_JUMP, jump)
        ctx.fill_u32(1000)
        ctx.skip(50_000_017)
        w = ctx.fill_u32(3000)
    for s in range(3):
        o = oracle_py.MtgpOracle(sets[s], s + 1)
        o.skip(50_001_017)
        assert np.array_equal(w[s], o.fill(3000))


@pytest.mark.parametrize("kernel", [5, 6])
def test_kara_jump_engine_mt(kernel):
    """Engine::mt MT19937 (n = 624: one Karatsuba level) with many jumped pieces."""
    st = mtgp.mt19937_status()
    seeds = [5489, 1, 2, 3]
    outs = []
    for jump in (0, 1):
        with mtgp.MtContext([st] * 4, seeds) as ctx:
            ctx.set_option(mtgp.OPT_KERNEL, kernel)
            ctx.set_option(mtgp.OPT_JUMP, jump)
            ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 4096)
            w = ctx.fill_u32(300_000)
            assert ctx.last_plan()[0] > 4 * 20
            ctx.skip(1_000_003)
            w2 = ctx.fill_u32(2000)
        outs.append((w, w2))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    for s in range(4):
        o = oracle_py.MtOracle(None, seeds[s])
        assert np.array_equal(outs[0][0][s], o.fill(300_000))
        o.fill(1_000_003)
        assert np.array_equal(outs[0][1][s], o.fill(2000))


def test_few_stream_planning_short_and_long_lived(curand_sets):
    """One stream (a GpuWordSource refill): a fresh stream is never split (no first-call
    analysis); once it has produced 2^25 words, a 2^20-word call is split into jump-ahead pieces
    over many warps (pieces_wanted, csrc/mtgp_plan.cu). Words exact either way."""
    st = curand_sets[7]
    L = 1 << 20
    with mtgp.MtgpContext([st], [11]) as ctx:
        a = ctx.fill_u32(L)
        assert ctx.last_plan()[0] == 1
        ctx.skip(1 << 25)
        b = ctx.fill_u32(L)
        pieces = ctx.last_plan()[0]
    assert pieces > 16
    o = oracle_py.MtgpOracle(st, 11)
    assert np.array_equal(a[0], o.fill(L))
    o.skip(1 << 25)
    assert np.array_equal(b[0], o.fill(L))


def test_few_stream_planning_engine_mt():
    st = mtgp.mt19937_status()
    L = 1 << 20
    with mtgp.MtContext([st], [77]) as ctx:
        ctx.fill_u32(1 << 12)
        ctx.skip((1 << 25) - (1 << 12))
        w = ctx.fill_u32(L)
        assert ctx.last_plan()[0] > 16
    o = oracle_py.MtOracle(None, 77)
    o.fill(1 << 25)
    assert np.array_equal(w[0], o.fill(L))

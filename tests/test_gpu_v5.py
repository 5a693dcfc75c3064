"""GPU parity of gen5 (csrc/mtgp_v5.cu: eight consecutive words per lane, 256-bit stores) against
the oracle and the cuRAND goldens. Bit-exact for u32 and both float kinds."""
import numpy as np
import pytest

import oracle_py
from paper_1501_07701_b200 import mtgp

pytestmark = pytest.mark.gpu


def _ctx(sets, seeds, opts):
    ctx = mtgp.MtgpContext(sets, seeds)
    ctx.set_option(mtgp.OPT_KERNEL, 7)
    for k, v in opts.items():
        ctx.set_option(k, v)
    return ctx


@pytest.mark.parametrize("kind", [mtgp.U32, mtgp.F32_12, mtgp.F32_01OC])
def test_v5_bit_exact_with_jumps(curand_sets, kind):
    sets = curand_sets[60:68]
    seeds = list(range(300, 308))
    with _ctx(sets, seeds, {mtgp.OPT_MIN_PIECE_WORDS: 2048}) as ctx:
        w1 = ctx.generate_host(kind, 200_000)
        pieces, _, kv = ctx.last_plan()
        w2 = ctx.generate_host(kind, 40_008)
        ck = ctx.checksums()
    assert kv == 7 and pieces > 8 * 20
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, 240_008, kind=kind, threads=8)
    assert np.array_equal(w1, ref[:, :200_000])
    assert np.array_equal(w2, ref[:, 200_000:])
    for s in range(8):
        allw = ref[s]
        assert ck[s] == (int(allw.astype(np.uint64).sum()), int(np.bitwise_xor.reduce(allw)), 240_008)


@pytest.mark.parametrize("L", [8, 256, 344, 352, 360, 512, 1000, 4096 + 8])
def test_v5_short_and_edge_lengths(curand_sets, L):
    """Pieces shorter than the window, steps straddling the end window, single steps."""
    sets = curand_sets[:3]
    with _ctx(sets, [5, 6, 7], {}) as ctx:
        a = ctx.fill_u32(L)
        b = ctx.fill_u32(L)
    ref, _ = oracle_py.mtgp_bulk(sets, [5, 6, 7], 2 * L, threads=3)
    assert np.array_equal(a, ref[:, :L]) and np.array_equal(b, ref[:, L:])


def test_v5_all_200_sets_jumped(curand_sets, curand_golden):
    """Every cuRAND set (pos 3..93: all eight residues pos mod 8 and every C-stream source split)."""
    with _ctx(curand_sets, [1] * 200, {mtgp.OPT_MIN_PIECE_WORDS: 4096}) as ctx:
        w = ctx.fill_u32(1 << 16)
        assert ctx.last_plan()[2] == 7 and ctx.last_plan()[0] >= 3000
    assert w.astype(np.uint64).sum(axis=1).tolist() == curand_golden["all200_seed1_n65536_sum64"]


def test_v5_rejects_unaligned_shapes(curand_sets):
    with _ctx(curand_sets[:2], [1, 2], {}) as ctx:
        with pytest.raises(Exception):
            ctx.fill_u32(1004)  # L % 8 != 0

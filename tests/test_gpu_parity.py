"""GPU parity: the CUDA path (through the C-ABI) vs the oracle and the cuRAND goldens.

Bit-exact for every u32 and float word (integer path; no tolerance).
"""
import numpy as np
import pytest

import oracle_py
from paper_1501_07701_b200 import mtgp, tables

pytestmark = pytest.mark.gpu

KERNELS = [1, 2]


def _ctx(sets, seeds, kernel, **opts):
    ctx = mtgp.MtgpContext(sets, seeds)
    ctx.set_option(mtgp.OPT_KERNEL, kernel)
    for k, v in opts.items():
        ctx.set_option(k, v)
    return ctx


@pytest.mark.parametrize("kernel", KERNELS)
def test_c1_set0_seed1_2p20(curand_sets, kernel):
    """BASELINE config 1: set 0, seed 1, 2^20 u32, bit-exact (SURVEY.md App. B goldens)."""
    with _ctx(curand_sets[:1], [1], kernel) as ctx:
        w = ctx.fill_u32(1 << 20)[0]
        ck = ctx.checksums()[0]
    c = oracle_py.cksum(w)
    assert (c["sum64"], c["xor32"], c["last"], c["poly31"]) == (2251211974485391, 0x87DB016D, 1034305667, 751051855)
    assert ck == (2251211974485391, 0x87DB016D, 1 << 20)
    ref = oracle_py.MtgpOracle(curand_sets[0], 1).fill(1 << 20)
    assert np.array_equal(w, ref)


@pytest.mark.parametrize("kernel", KERNELS)
def test_first32_goldens(curand_sets, curand_golden, kernel):
    cases = curand_golden["first32"]
    sets = [curand_sets[c["set"]] for c in cases]
    seeds = [c["seed"] for c in cases]
    with _ctx(sets, seeds, kernel) as ctx:
        w = ctx.fill_u32(32)
    for i, c in enumerate(cases):
        assert w[i].tolist() == c["u32"]


@pytest.mark.parametrize("kernel", KERNELS)
def test_all200_sets(curand_sets, curand_golden, kernel):
    with _ctx(curand_sets, [1] * 200, kernel) as ctx:
        w = ctx.fill_u32(1 << 16)
    assert w.astype(np.uint64).sum(axis=1).tolist() == curand_golden["all200_seed1_n65536_sum64"]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("kind", [mtgp.F32_12, mtgp.F32_01OC])
def test_float_kinds(curand_sets, kernel, kind):
    sets = curand_sets[:8]
    with _ctx(sets, list(range(1, 9)), kernel) as ctx:
        w = ctx.generate_host(kind, 50000)
    for s in range(8):
        ref = oracle_py.MtgpOracle(sets[s], s + 1).fill(50000, kind=kind)
        assert np.array_equal(w[s], ref)
    f = w.view(np.float32)
    if kind == mtgp.F32_12:
        assert f.min() >= 1.0 and f.max() < 2.0
    else:
        assert f.min() > 0.0 and f.max() <= 1.0


@pytest.mark.parametrize("kernel", KERNELS)
def test_ragged_successive_calls_concatenate(curand_sets, kernel):
    """Successive fills continue the stream exactly (WordSource::fill semantics)."""
    sets = curand_sets[10:14]
    lens = [1, 7, 255, 256, 257, 1000, 12345, 3]
    with _ctx(sets, [5, 6, 7, 8], kernel) as ctx:
        parts = [ctx.fill_u32(n) for n in lens]
        assert ctx.position(0) == sum(lens)
    got = np.concatenate(parts, axis=1)
    for s in range(4):
        ref = oracle_py.MtgpOracle(sets[s], 5 + s).fill(sum(lens))
        assert np.array_equal(got[s], ref)


@pytest.mark.parametrize("kernel", KERNELS)
def test_zero_length_and_device_output(curand_sets, kernel):
    import torch
    sets = curand_sets[:3]
    with _ctx(sets, [1, 2, 3], kernel) as ctx:
        ctx.fill_u32(0)
        buf = torch.empty((3, 4096), dtype=torch.int32, device="cuda")
        ctx.generate_device(mtgp.U32, buf.data_ptr(), 4096)
        ctx.sync()
        w = buf.cpu().numpy().view(np.uint32)
    for s in range(3):
        assert np.array_equal(w[s], oracle_py.MtgpOracle(sets[s], s + 1).fill(4096))


@pytest.mark.parametrize("kernel", KERNELS)
def test_state_save_restore(curand_sets, kernel):
    sets = curand_sets[20:22]
    with _ctx(sets, [11, 12], kernel) as ctx:
        ctx.fill_u32(777)
        win, pos = ctx.state_save()
        a = ctx.fill_u32(3000)
        ctx.state_restore(win, pos)
        assert ctx.position(1) == 777
        b = ctx.fill_u32(3000)
    assert np.array_equal(a, b)
    o = oracle_py.MtgpOracle(sets[0], 11)
    o.skip(777)
    live = win[0].copy()
    w_or = o.window()
    assert np.array_equal(live[1:], w_or[1:])
    assert (live[0] & sets[0].mask) == (w_or[0] & sets[0].mask)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("mexp", [23209, 44497])
def test_large_mexp_synthetic(kernel, mexp):
    sets = tables.synthetic_sets(mexp, 4)
    with _ctx(sets, [1, 2, 3, 4], kernel) as ctx:
        w = ctx.fill_u32(70001)
    for s in range(4):
        assert np.array_equal(w[s], oracle_py.MtgpOracle(sets[s], s + 1).fill(70001))


def test_checksum_option_off(curand_sets):
    with _ctx(curand_sets[:2], [1, 2], 1) as ctx:
        ctx.set_option(mtgp.OPT_CHECKSUM, 0)
        ctx.fill_u32(1000)
        assert ctx.checksums() == [(0, 0, 0), (0, 0, 0)]
        ctx.set_option(mtgp.OPT_CHECKSUM, 1)
        w = ctx.fill_u32(1000)
        ck = ctx.checksums()
    for s in range(2):
        assert ck[s] == (int(w[s].astype(np.uint64).sum()), int(np.bitwise_xor.reduce(w[s])), 1000)

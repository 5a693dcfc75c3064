"""GPU parity: the CUDA path (through the C-ABI) vs the oracle and the cuRAND goldens.

Bit-exact for every u32 and float word (integer path; no tolerance).
"""
import numpy as np
import pytest

import oracle_py
from paper_1501_07701_b200 import mtgp, tables

pytestmark = pytest.mark.gpu

KERNELS = [1, 2]


def _ctx(sets, seeds, kernel, opts=None):
    ctx = mtgp.MtgpContext(sets, seeds)
    ctx.set_option(mtgp.OPT_KERNEL, kernel)
    for k, v in (opts or {}).items():
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


# ---------------- v2: jump-ahead pieces ----------------

@pytest.mark.parametrize("mexp", [11213, 23209, 44497])
def test_v2_jump_pieces_bit_exact(curand_sets, mexp):
    """Force many jump-ahead pieces on a small request; every word must match the oracle."""
    sets = curand_sets[40:46] if mexp == 11213 else tables.synthetic_sets(mexp, 6)
    seeds = [101, 102, 103, 104, 105, 106]
    L = 150001
    with _ctx(sets, seeds, 2, {mtgp.OPT_MIN_PIECE_WORDS: 3000}) as ctx:
        w1 = ctx.fill_u32(L)
        pieces, _, kv = ctx.last_plan()
        assert kv == 2 and pieces > 6 * 10
        w2 = ctx.fill_u32(77777)  # continues after the jumped call
        ck = ctx.checksums()
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, L + 77777, threads=8)
    assert np.array_equal(w1, ref[:, :L])
    assert np.array_equal(w2, ref[:, L:])
    for s in range(6):
        allw = ref[s]
        assert ck[s] == (int(allw.astype(np.uint64).sum()), int(np.bitwise_xor.reduce(allw)), L + 77777)


def test_v2_float_kinds_with_jumps(curand_sets):
    sets = curand_sets[:4]
    for kind in (mtgp.F32_12, mtgp.F32_01OC):
        with _ctx(sets, [9, 8, 7, 6], 2, {mtgp.OPT_MIN_PIECE_WORDS: 5000}) as ctx:
            w = ctx.generate_host(kind, 60000)
            assert ctx.last_plan()[0] > 4
        ref, _ = oracle_py.mtgp_bulk(sets, [9, 8, 7, 6], 60000, kind=kind, threads=4)
        assert np.array_equal(w, ref)


@pytest.mark.parametrize("mexp", [11213, 44497])
def test_skip_jump_ahead(curand_sets, mexp):
    sets = curand_sets[100:103] if mexp == 11213 else tables.synthetic_sets(mexp, 3)
    with _ctx(sets, [1, 2, 3], 2) as ctx:
        ctx.fill_u32(1000)
        ctx.skip(10_000_019)
        assert ctx.position(2) == 10_001_019
        w = ctx.fill_u32(5000)
    for s in range(3):
        o = oracle_py.MtgpOracle(sets[s], s + 1)
        o.skip(10_001_019)
        assert np.array_equal(w[s], o.fill(5000))


def test_v2_long_streams_full_compare(curand_sets):
    """8 streams x 2^24 words with the default plan (hundreds of jumped pieces)."""
    import torch
    sets = curand_sets[150:158]
    seeds = list(range(1000, 1008))
    L = 1 << 24
    with _ctx(sets, seeds, 0) as ctx:
        buf = torch.empty((8, L), dtype=torch.int32, device="cuda")
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 16)
        ctx.generate_device(mtgp.U32, buf.data_ptr(), L)
        ctx.sync()
        pieces = ctx.last_plan()[0]
        got = buf.cpu().numpy().view(np.uint32)
    assert pieces >= 256
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, L, threads=8)
    assert np.array_equal(got, ref)


# ---------------- v3: register-resident ring (MTGP32-11213) ----------------

@pytest.mark.parametrize("kind", [mtgp.U32, mtgp.F32_12, mtgp.F32_01OC])
def test_v3_bit_exact_with_jumps(curand_sets, kind):
    sets = curand_sets[60:68]
    seeds = list(range(70, 78))
    L = 123456  # multiple of 4
    with _ctx(sets, seeds, 3, {mtgp.OPT_MIN_PIECE_WORDS: 2000}) as ctx:
        w1 = ctx.generate_host(kind, L)
        pieces, _, kv = ctx.last_plan()
        assert kv == 3 and pieces > 8 * 20
        w2 = ctx.generate_host(kind, 4096)
        ck = ctx.checksums()
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, L + 4096, kind=kind, threads=8)
    assert np.array_equal(w1, ref[:, :L])
    assert np.array_equal(w2, ref[:, L:])
    for s in range(8):
        assert ck[s] == (int(ref[s].astype(np.uint64).sum()), int(np.bitwise_xor.reduce(ref[s])), L + 4096)


@pytest.mark.parametrize("L", [4, 256, 260, 352, 600, 1024, 65536 + 12])
def test_v3_short_and_edge_lengths(curand_sets, L):
    """Pieces shorter than N, one-step pieces, and tails of 4..252 words; every pos residue."""
    idx = [next(i for i, p in enumerate(curand_sets) if p.pos % 4 == r) for r in range(4)]
    idx += [next(i for i, p in enumerate(curand_sets) if p.pos // 4 == 23)]  # threshold-32 edge
    idx += [0, 100, 199]
    sets = [curand_sets[i] for i in idx]
    assert {p.pos % 4 for p in sets} == {0, 1, 2, 3}
    with _ctx(sets, [1] * 8, 3) as ctx:
        a = ctx.fill_u32(L)
        b = ctx.fill_u32(L)
        assert ctx.last_plan()[2] == 3
    ref, _ = oracle_py.mtgp_bulk(sets, [1] * 8, 2 * L, threads=8)
    assert np.array_equal(a, ref[:, :L]) and np.array_equal(b, ref[:, L:])


def test_v3_all_200_sets_jumped(curand_sets, curand_golden):
    """Every cuRAND set (pos 3..93, all thresholds incl. the pos/4 == 23 edge) through v3 pieces."""
    with _ctx(curand_sets, [1] * 200, 3, {mtgp.OPT_MIN_PIECE_WORDS: 4096}) as ctx:
        w = ctx.fill_u32(1 << 16)
        assert ctx.last_plan()[0] >= 3000
    assert w.astype(np.uint64).sum(axis=1).tolist() == curand_golden["all200_seed1_n65536_sum64"]


@pytest.mark.parametrize("mexp", [23209, 44497])
def test_synthetic_degenerate_sets_jump(mexp):
    """Uncertified synthetic sets have pre-periods / reducible annihilators; jumps are taken
    relative to the reference point x_{N+8} and every stream must still be bit-exact."""
    sets = tables.synthetic_sets(mexp, 16)
    seeds = list(range(16))
    L = 40000
    with _ctx(sets, seeds, 2, {mtgp.OPT_MIN_PIECE_WORDS: 4000}) as ctx:
        w = ctx.fill_u32(L)
        assert ctx.last_plan()[0] >= 16 * 5
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, L, threads=8)
    assert np.array_equal(w, ref)


def test_f64_01_matches_next_f64_01(curand_sets):
    """MTGP_F64_01 = u32 * 2^-32 draw for draw, like Generator::next_f64_01 (generator.hpp:39-41)."""
    sets = curand_sets[:3]
    with _ctx(sets, [1, 2, 3], 0) as ctx:
        d = ctx.generate_host(mtgp.F64_01, 30001)
        u = ctx.fill_u32(5)  # the stream continues after the doubles
    for s in range(3):
        ref = oracle_py.MtgpOracle(sets[s], s + 1).fill(30006)
        assert np.array_equal(d[s], ref[:30001].astype(np.float64) * (1.0 / 4294967296.0))
        assert np.array_equal(u[s], ref[30001:])
    assert d.min() >= 0.0 and d.max() < 1.0


def test_charpoly_digests_match_the_certified_table(curand_sets):
    """The BM-derived characteristic polynomial of every cuRAND MTGP32-11213 set, digested the way
    the MTGP tables do, equals the table's poly_sha1 -- an independent pin of the recurrence,
    the seeding and the jump-ahead algebra (cf. verify_digest, proj/src/dynamic_creator.cpp:100-103)."""
    with _ctx(curand_sets, [1] * 200, 0) as ctx:
        dig = ctx.charpoly_sha1()
    assert dig == [p.poly_sha1 for p in curand_sets]


def test_short_skip_generates(curand_sets):
    sets = curand_sets[5:7]
    with _ctx(sets, [3, 4], 0) as ctx:
        ctx.skip(100)
        ctx.skip(3)
        w = ctx.fill_u32(1000)
        assert ctx.checksums()[0][2] == 1000  # skipped words are not checksummed
    for s in range(2):
        o = oracle_py.MtgpOracle(sets[s], 3 + s)
        o.skip(103)
        assert np.array_equal(w[s], o.fill(1000))


@pytest.mark.parametrize("host_chunk,L", [(1, 37), (3, 1000), (4096, 4095), (4097, 100003), (1 << 18, 1 << 20),
                                          (1 << 18, (1 << 20) + 6), (65536, 300001)])
def test_host_output_chunk_ramp(curand_sets, host_chunk, L):
    """Host-memory output goes through ramped device chunks (first chunk small, then x16 up to
    OPT_HOST_CHUNK): every chunking must give the same words, and the stream must continue."""
    sets = curand_sets[10:13]
    with _ctx(sets, [7, 8, 9], 0, {mtgp.OPT_HOST_CHUNK: host_chunk}) as ctx:
        a = ctx.fill_u32(L)
        b = ctx.fill_u32(5)
        ck = ctx.checksums()
    ref, _ = oracle_py.mtgp_bulk(sets, [7, 8, 9], L + 5, threads=3)
    assert np.array_equal(a, ref[:, :L]) and np.array_equal(b, ref[:, L:])
    assert all(c[2] == L + 5 for c in ck)


def _sets_for(mexp, k, curand_sets):
    return curand_sets[:k] if mexp == 11213 else tables.synthetic_sets(mexp, k)


@pytest.mark.parametrize("mexp", [11213, 23209, 44497])
def test_v4_bit_exact_with_jumps(curand_sets, mexp):
    """v4 (gen3's register-resident design templated on N) over jump-ahead pieces."""
    sets = _sets_for(mexp, 8, curand_sets)
    seeds = list(range(31, 39))
    L = (1 << 18) + 12
    with _ctx(sets, seeds, 4, {mtgp.OPT_MIN_PIECE_WORDS: 1 << 13}) as ctx:
        a = ctx.fill_u32(L)
        pieces, _, kv = ctx.last_plan()
        b = ctx.fill_u32(4096)
        ck = ctx.checksums()
    assert kv == 4 and pieces > 8
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, L + 4096, threads=8)
    assert np.array_equal(a, ref[:, :L]) and np.array_equal(b, ref[:, L:])
    for s in range(8):
        c = oracle_py.cksum(ref[s])
        assert ck[s] == (c["sum64"], c["xor32"], L + 4096)


@pytest.mark.parametrize("mexp", [11213, 23209, 44497])
@pytest.mark.parametrize("L", [4, 256, 260, 728, 1024, 1392, 3000, 65536 + 12])
def test_v4_short_and_edge_lengths(curand_sets, mexp, L):
    """Tail steps and the end-window hand-off at lengths around N and the step size; the
    next call must continue the stream exactly."""
    sets = _sets_for(mexp, 3, curand_sets)
    with _ctx(sets, [5, 6, 7], 4) as ctx:
        a = ctx.fill_u32(L)
        b = ctx.fill_u32(1000 + 4 * (L % 3))
    ref, _ = oracle_py.mtgp_bulk(sets, [5, 6, 7], L + b.shape[1], threads=3)
    assert np.array_equal(a, ref[:, :L]) and np.array_equal(b, ref[:, L:])


@pytest.mark.parametrize("mexp", [3217, 4253, 4423, 9689, 9941, 19937, 21701])
def test_other_mtgp_exponents_cta_per_stream(mexp):
    """The remaining MTGP32 exponents (mtgp_validate_params' list) run on the CTA-per-stream
    kernel: bit-exact across calls, skips and save/restore."""
    sets = tables.synthetic_sets(mexp, 3)
    seeds = [3, 5, 7]
    with mtgp.MtgpContext(sets, seeds) as ctx:
        a = ctx.fill_u32(5001)
        _, _, kv = ctx.last_plan()
        win, pos = ctx.state_save()
        b = ctx.fill_u32(999)
        ctx.state_restore(win, pos)
        b2 = ctx.fill_u32(999)
        ctx.skip(12345)
        c = ctx.fill_u32(100)
    assert kv == 1
    ref, _ = oracle_py.mtgp_bulk(sets, seeds, 5001 + 999 + 12345 + 100, threads=3)
    assert np.array_equal(a, ref[:, :5001])
    assert np.array_equal(b, ref[:, 5001:6000]) and np.array_equal(b2, b)
    assert np.array_equal(c, ref[:, 6000 + 12345:])


def test_async_host_generation_into_pinned_buffers(curand_sets):
    """mtgp_generate_async + mtgp_host_alloc (GpuWordSource's double buffering): two chunks in
    flight into two page-locked buffers, both valid after mtgp_sync, in stream order."""
    import ctypes as C
    sets = curand_sets[20:22]
    L = 1 << 18
    with mtgp.MtgpContext(sets, [3, 4]) as ctx:
        lib = ctx.lib
        ptrs = []
        for _ in range(2):
            p = C.c_void_p()
            assert lib.mtgp_host_alloc(2 * L * 4, C.byref(p)) == 0
            ptrs.append(p)
        bufs = [np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint32)), shape=(2, L)) for p in ptrs]
        try:
            ctx.generate_host_async(mtgp.U32, bufs[0])
            ctx.generate_host_async(mtgp.U32, bufs[1])
            ctx.sync()
            got = np.concatenate([bufs[0], bufs[1]], axis=1).copy()
        finally:
            for p in ptrs:
                lib.mtgp_host_free(p)
    ref, _ = oracle_py.mtgp_bulk(sets, [3, 4], 2 * L, threads=2)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("mexp", [23209, 44497])
@pytest.mark.parametrize("kernel", [0, 1, 2, 4])
def test_large_mexp_pinned_by_curand(large_golden, mexp, kernel):
    """23209 / 44497 against cuRAND's own init / para_rec / temper run at N = 726 / 1391
    (tests/golden/mtgp32_large_curand.json), not only against the builder's restatement:
    every kernel that takes the shape (0 auto = v4, 1 CTA per stream, 2 shared ring, 4 v4),
    2^20 words per stream as 2^19 + 2^19 so the second call starts from jumped pieces."""
    cases = [c for c in large_golden if c["mexp"] == mexp]
    sets, seeds = [c["set"] for c in cases], [c["seed"] for c in cases]
    with _ctx(sets, seeds, kernel, {mtgp.OPT_MIN_PIECE_WORDS: 1 << 15}) as ctx:
        w = np.concatenate([ctx.fill_u32(1 << 19), ctx.fill_u32(1 << 19)], axis=1)
        ck = ctx.checksums()
        pieces = ctx.last_plan()[0]
    if kernel != 1:
        assert pieces > len(cases)  # the second call ran jumped pieces
    for i, c in enumerate(cases):
        assert w[i, :32].tolist() == c["u32"], (c["synthetic_index"], c["seed"])
        assert (int(w[i].astype(np.uint64).sum()), int(np.bitwise_xor.reduce(w[i])), int(w[i, -1])) == (
            c["sum64"], c["xor32"], c["last"])
        assert ck[i] == (c["sum64"], c["xor32"], c["n"])


@pytest.mark.parametrize("mexp", [23209, 44497])
def test_large_mexp_single_float_pinned_by_curand(large_golden, mexp):
    """[1,2) floats through cuRAND's temper_single (flt_tmp_tbl) at 23209 / 44497."""
    cases = [c for c in large_golden if c["mexp"] == mexp]
    with _ctx([c["set"] for c in cases], [c["seed"] for c in cases], 0) as ctx:
        f = ctx.generate_host(mtgp.F32_12, 32)
    for i, c in enumerate(cases):
        assert f[i].tolist() == c["single12_bits"]


@pytest.mark.parametrize("prejump", [1, 2])
def test_back_to_back_calls_queued_behind_a_busy_stream(curand_sets, prejump):
    """ADVICE r1 (plan upload race): calls of different lengths issued back to back without a
    sync, all queued behind a ~0.5 s spin kernel on the context stream, so every call's plan
    (and, with prejump 2, every speculative jump) is built and uploaded while the earlier calls
    have not even started. Each call's words and the end state must still equal the oracle."""
    import torch

    sets = curand_sets[:16]
    seeds = list(range(100, 116))
    lens = [1 << 22, 1 << 18, (1 << 20) + 4 * 12345, 1 << 22, 1 << 16, 1 << 22]
    with mtgp.MtgpContext(sets, seeds) as ctx:
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 15)  # every call split into jumped pieces
        ctx.set_option(mtgp.OPT_PREJUMP, prejump)
        ext = torch.cuda.ExternalStream(ctx.stream_handle())
        bufs = []
        with torch.cuda.stream(ext):
            torch.cuda._sleep(1_000_000_000)
            for L in lens:
                b = torch.empty((16, L), dtype=torch.int32, device="cuda")
                ctx.generate_device(mtgp.U32, b.data_ptr(), L)
                bufs.append(b)
        ctx.sync()
        pos = 0
        for L, b in zip(lens, bufs):
            got = b.cpu().numpy().view(np.uint32)
            want = oracle_py.mtgp_bulk(sets, seeds, L, skip=pos, threads=16)[0]
            assert np.array_equal(got, want), (prejump, L, pos)
            pos += L
        tail = ctx.fill_u32(1024)
    assert np.array_equal(tail, oracle_py.mtgp_bulk(sets, seeds, 1024, skip=pos, threads=16)[0])

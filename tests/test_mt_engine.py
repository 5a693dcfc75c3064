"""Engine::mt -- the reference's own recurrence on the GPU, bit-exact vs the
reference compiled from its sources (oracle/_ref) and vs its own goldens
(proj/tests/test_generator.cpp:11-25)."""
import numpy as np
import pytest

import oracle_py
from paper_1501_07701_b200 import mtgp


def _mt_oracle_params(st):
    return oracle_py.OracleMtParams(st["mexp"], st["n"], st["m"], st["r"], st["a"], st["temper_b"],
                                    st["temper_c"], st["temper_u"], st["temper_s"], st["temper_t"], st["temper_l"])


def _dc(mt_golden, name):
    f = mt_golden[name]["status12"]
    keys = ("id", "mexp", "n", "m", "r", "a", "temper_b", "temper_c", "temper_u", "temper_s", "temper_t", "temper_l")
    return dict(zip(keys, f))


# ---------------- CPU: validation mirrors ParameterizedStatus::validate ----------------

def test_mt19937_status_validates():
    mtgp.mt_validate(mtgp.mt19937_status())


@pytest.mark.parametrize("field,value,msg", [
    ("r", 30, "32\\*n - r must equal mexp"),          # test_generator.cpp:109-112
    ("id", 7, "low 16 bits"),                          # :113-116
    ("m", 624, "middle offset"),                       # :117-120
    ("mexp", 19936, "32\\*n - r must equal mexp"),     # :121-125 (r adjusted below)
    ("temper_u", 0, "tempering shifts"),
])
def test_mt_validate_rejects(field, value, msg):
    st = mtgp.mt19937_status()
    st[field] = value
    if field == "mexp":
        st["r"] = 32 * st["n"] - value  # = 32, rejected like the reference (params.cpp:27 before :30)
        msg = "split position r must be < 32"
    with pytest.raises(mtgp.MtgpInvalidArgument, match=msg):
        mtgp.mt_validate(st)


# ---------------- GPU parity ----------------

@pytest.mark.gpu
def test_mt19937_reference_goldens(mt_golden):
    with mtgp.MtContext([mtgp.mt19937_status()], [5489]) as ctx:
        w = ctx.fill_u32(1 << 20)[0]
    assert w[:3].tolist() == [3499211612, 581869302, 3890346734]
    c = oracle_py.cksum(w)
    want = mt_golden["mt19937_seed5489_n1048576"]
    assert (c["sum64"], c["xor32"], c["last"]) == (want["sum64"], want["xor32"], want["last"])


@pytest.mark.gpu
def test_mt_vs_compiled_reference_many_streams():
    seeds = [0, 1, 5489, 12345, 0xFFFFFFFF] + [oracle_py.lib().oracle_derive_seed(77, j) for j in range(27)]
    sts = [mtgp.mt19937_status()] * len(seeds)
    with mtgp.MtContext(sts, seeds) as ctx:
        a = ctx.fill_u32(5000)
        b = ctx.fill_u32(12347)
    for s, seed in enumerate(seeds):
        ref = oracle_py.ref_fill(5000 + 12347, seed)  # the reference's make_word_source + fill
        assert np.array_equal(a[s], ref[:5000]) and np.array_equal(b[s], ref[5000:])


@pytest.mark.gpu
def test_mt_dc_statuses_mixed_shapes(mt_golden):
    """DC-minted statuses (n-m = 10 and 92) next to MT19937 in one context (state stride = max n)."""
    sts = [_dc(mt_golden, "dc521_id7"), _dc(mt_golden, "dc3217_id7"), mtgp.mt19937_status()]
    seeds = [4357, 4357, 5489]
    with mtgp.MtContext(sts, seeds) as ctx:
        w = ctx.fill_u32(1 << 16)
    for s in range(2):
        d = mt_golden[["dc521_id7", "dc3217_id7"][s]]
        c = oracle_py.cksum(w[s])
        assert (c["sum64"], c["xor32"], c["last"]) == (d["sum64"], d["xor32"], d["last"])
        assert np.array_equal(w[s], oracle_py.ref_fill(1 << 16, 4357, d["status12"]))
    assert np.array_equal(w[2], oracle_py.MtOracle(None, 5489).fill(1 << 16))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [mtgp.F32_12, mtgp.F32_01OC])
def test_mt_float_kinds(kind):
    with mtgp.MtContext([mtgp.mt19937_status()] * 3, [1, 2, 3]) as ctx:
        w = ctx.generate_host(kind, 20000)
    for s in range(3):
        u = oracle_py.MtOracle(None, s + 1).fill(20000)
        f = ((u >> 9) | 0x3F800000).astype(np.uint32)
        if kind == mtgp.F32_01OC:
            f = (np.float32(2.0) - f.view(np.float32)).view(np.uint32)
        assert np.array_equal(w[s], f)


@pytest.mark.gpu
def test_mt_next_f64_01():
    """next_f64_01 == next_u32 / 2^32 draw for draw (proj/tests/test_generator.cpp:90-103)."""
    with mtgp.MtContext([mtgp.mt19937_status()], [99]) as ctx:
        d = ctx.generate_host(mtgp.F64_01, 10000)[0]
    u = oracle_py.MtOracle(None, 99).fill(10000)
    assert np.array_equal(d, u.astype(np.float64) * (1.0 / 4294967296.0))
    assert d.min() >= 0.0 and d.max() < 1.0


@pytest.mark.gpu
def test_mt_ragged_state_restore_skip_checksums():
    st = mtgp.mt19937_status()
    with mtgp.MtContext([st, st], [11, 12]) as ctx:
        parts = [ctx.fill_u32(n) for n in (1, 226, 227, 228, 624, 1000)]
        win, pos = ctx.state_save()
        x = ctx.fill_u32(999)
        ctx.state_restore(win, pos)
        y = ctx.fill_u32(999)
        assert np.array_equal(x, y)
        ctx.skip(100003)
        z = ctx.fill_u32(64)
        ck = ctx.checksums()
    total = sum((1, 226, 227, 228, 624, 1000)) + 999 + 999
    for s in range(2):
        o = oracle_py.MtOracle(None, 11 + s)
        ref = o.fill(sum((1, 226, 227, 228, 624, 1000)) + 999)
        assert np.array_equal(np.concatenate([p[s] for p in parts] + [y[s]]), ref)
        o2 = oracle_py.MtOracle(None, 11 + s)
        o2.fill(sum((1, 226, 227, 228, 624, 1000)) + 999 + 100003)
        assert np.array_equal(z[s], o2.fill(64))
        assert ck[s][2] == total + 64


@pytest.mark.gpu
@pytest.mark.parametrize("mexp", [89, 127, 521, 607, 1279, 2203, 2281, 3217, 19937, 23209])
def test_mt_every_supported_shape_vs_compiled_reference(mexp):
    """Engine::mt at every exponent the reference supports (kSupportedMexp, params.hpp:50-51),
    shapes from shape_for_mexp (params.cpp:56-61), middle offsets m across [1, n-1] (DC draws m in
    that range, dynamic_creator.cpp:73) -- incl. n - m = 1, a one-word parallel step."""
    import random
    rnd = random.Random(mexp)
    n = (mexp + 31) // 32
    ms = sorted({1, n - 1, max(1, n // 2), rnd.randint(1, n - 1)})
    sts = []
    for j, m in enumerate(ms):
        sts.append(dict(id=7 + j, mexp=mexp, n=n, m=m, r=32 * n - mexp, a=(rnd.getrandbits(16) << 16) | (7 + j),
                        temper_b=rnd.getrandbits(32), temper_c=rnd.getrandbits(32), temper_u=11, temper_s=7,
                        temper_t=15, temper_l=18))
    seeds = [rnd.getrandbits(32) for _ in sts]
    L = 3 * n + 1000
    with mtgp.MtContext(sts, seeds) as ctx:
        w = ctx.fill_u32(L)
    for s, st in enumerate(sts):
        st12 = [st[k] for k in ("id", "mexp", "n", "m", "r", "a", "temper_b", "temper_c", "temper_u", "temper_s",
                                "temper_t", "temper_l")]
        assert np.array_equal(w[s], oracle_py.ref_fill(L, seeds[s], st12)), (mexp, st["m"])


def _rand_status(mexp, m, seed):
    import random
    rnd = random.Random(seed)
    n = (mexp + 31) // 32
    return dict(id=9, mexp=mexp, n=n, m=m, r=32 * n - mexp, a=(rnd.getrandbits(16) << 16) | 9,
                temper_b=rnd.getrandbits(32), temper_c=rnd.getrandbits(32), temper_u=11, temper_s=7, temper_t=15,
                temper_l=18)


def _st12(st):
    return [st[k] for k in ("id", "mexp", "n", "m", "r", "a", "temper_b", "temper_c", "temper_u", "temper_s",
                            "temper_t", "temper_l")]


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["mt19937", "m23209", "dc3217"])
def test_mt_warp_teams_with_jumps_vs_reference(mt_golden, which):
    """Engine::mt through the jump-ahead planner (warp teams: kernel version 6 for the n = 624
    shape, 5 otherwise), many pieces per stream, bit-exact against the reference compiled from
    its sources; the next call continues."""
    if which == "mt19937":
        sts = [mtgp.mt19937_status()] * 3
    elif which == "m23209":
        sts = [_rand_status(23209, 300, 1), _rand_status(23209, 300, 2), _rand_status(23209, 300, 3)]
    else:
        sts = [_dc(mt_golden, "dc3217_id7")] * 3
    seeds = [5489, 1, 0xC0FFEE]
    L = (1 << 17) + 36
    with mtgp.MtContext(sts, seeds) as ctx:
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 12)
        a = ctx.fill_u32(L)
        pieces, _, kv = ctx.last_plan()
        b = ctx.fill_u32(5000)
        ck = ctx.checksums()
    assert kv == (6 if which == "mt19937" else 5) and pieces > 3
    for s in range(3):
        ref = oracle_py.ref_fill(L + 5000, seeds[s], _st12(sts[s]))
        assert np.array_equal(a[s], ref[:L]) and np.array_equal(b[s], ref[L:])
        c = oracle_py.cksum(ref)
        assert ck[s] == (c["sum64"], c["xor32"], L + 5000)


@pytest.mark.gpu
def test_mt_warp_teams_float_kinds_and_jump_skip():
    st = mtgp.mt19937_status()
    with mtgp.MtContext([st, st], [11, 12]) as ctx:
        f = ctx.generate_host(mtgp.F32_01OC, 40000)
        ctx.skip(1_000_003)  # jump-ahead for Engine::mt
        u = ctx.fill_u32(3000)
    for s in range(2):
        o = oracle_py.MtOracle(None, 11 + s)
        w = o.fill(40000)
        v = ((w >> 9) | 0x3F800000).astype(np.uint32)
        assert np.array_equal(f[s], (np.float32(2.0) - v.view(np.float32)).view(np.uint32))
        o.fill(1_000_003)
        assert np.array_equal(u[s], o.fill(3000))


@pytest.mark.gpu
def test_mt_shapes_without_teams_fall_back(mt_golden):
    """n - m < 32 (dc521: 10) and mixed shapes keep the CTA-per-stream kernel, still bit-exact."""
    sts = [_dc(mt_golden, "dc521_id7"), mtgp.mt19937_status()]
    with mtgp.MtContext(sts, [4357, 5489]) as ctx:
        w = ctx.fill_u32(70000)
        _, _, kv = ctx.last_plan()
    assert kv == 1
    assert np.array_equal(w[0], oracle_py.ref_fill(70000, 4357, mt_golden["dc521_id7"]["status12"]))
    assert np.array_equal(w[1], oracle_py.ref_fill(70000, 5489))


@pytest.mark.gpu
@pytest.mark.parametrize("engine", ["mt", "mtgp"])
def test_zero_state_emits_zero_forever(engine, curand_sets):
    """proj/tests/test_generator.cpp:52-57: an all-zero state is a fixed point (from_state with a
    zero state). Restoring a zero window must give 0 words on every path, incl. jumped pieces."""
    if engine == "mt":
        ctx = mtgp.MtContext([mtgp.mt19937_status()] * 2, [1, 2])
    else:
        ctx = mtgp.MtgpContext(curand_sets[:2], [1, 2])
    with ctx:
        win, pos = ctx.state_save()
        ctx.state_restore(np.zeros_like(win), pos)
        ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 12)
        w = ctx.fill_u32(100000)
    assert not w.any()


@pytest.mark.gpu
def test_mt_seed0_state_and_first_words():
    """test_generator.cpp:27-50: seed 0 seeds a non-zero state with
    st[1] = 1812433253 * (0 ^ (0 >> 30)) + 1 = 1; the words equal the reference's."""
    with mtgp.MtContext([mtgp.mt19937_status()], [0]) as ctx:
        win, _ = ctx.state_save()
        w = ctx.fill_u32(2000)
    assert win[0, 0] == 0 and win[0, 1] == 1 and win[0].any()
    assert np.array_equal(w[0], oracle_py.ref_fill(2000, 0))


# (16 + m) / 128 and (16 + m) mod 4 pick mt_gen3's C-stream template variant (csrc/mtgp_mt3.cu,
# BASE = 16 for n = 624): these m cover all 16 variants, m = 1 and the n - m = 129 boundary.
MT3_MS = [1, 2, 3, 4, 111, 112, 113, 114, 239, 240, 241, 242, 367, 397, 398, 399, 400, 495]


@pytest.mark.gpu
def test_mt_gen3_every_variant_vs_reference():
    """mt_gen3 (kernel version 6): n = 624 statuses with every C-stream variant, jumped pieces,
    a ragged length, a next call shorter than n (pieces shorter than the window) and a long
    one; bit-exact against the reference, checksums included; kernel 5 agrees."""
    sts = [_rand_status(19937, m, 100 + i) for i, m in enumerate(MT3_MS)]
    seeds = [7 * i + 1 for i in range(len(sts))]
    lens = [200_004, 308, 65_536]
    outs = {}
    for kern in (6, 5):
        with mtgp.MtContext(sts, seeds) as ctx:
            ctx.set_option(mtgp.OPT_KERNEL, kern)
            ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 12)
            ws = []
            for L in lens:
                ws.append(ctx.fill_u32(L))
                assert ctx.last_plan()[2] == kern
            outs[kern] = (ws, ctx.checksums())
    total = sum(lens)
    for s in range(len(sts)):
        ref = oracle_py.ref_fill(total, seeds[s], _st12(sts[s]))
        got = np.concatenate([w[s] for w in outs[6][0]])
        assert np.array_equal(got, ref), MT3_MS[s]
        c = oracle_py.cksum(ref)
        assert outs[6][1][s] == (c["sum64"], c["xor32"], total)
    for a, b in zip(outs[6][0], outs[5][0]):
        assert np.array_equal(a, b)


@pytest.mark.gpu
def test_mt_gen3_shape_limits():
    """Kernel 6 is refused for L % 4 != 0 and for n - m = 128; auto then uses kernel 5."""
    st = mtgp.mt19937_status()
    with mtgp.MtContext([st, st], [1, 2]) as ctx:
        ctx.set_option(mtgp.OPT_KERNEL, 6)
        with pytest.raises(mtgp.MtgpInvalidArgument):
            ctx.fill_u32(1001)
    with mtgp.MtContext([st, st], [1, 2]) as ctx:
        w = ctx.fill_u32(1001)
        assert ctx.last_plan()[2] == 5
    assert np.array_equal(w[1], oracle_py.ref_fill(1001, 2))
    edge = _rand_status(19937, 496, 5)
    with mtgp.MtContext([st, edge], [1, 2]) as ctx:
        w = ctx.fill_u32(4096)
        assert ctx.last_plan()[2] == 5
        ctx.set_option(mtgp.OPT_KERNEL, 6)
        with pytest.raises(mtgp.MtgpInvalidArgument):
            ctx.fill_u32(4096)
    assert np.array_equal(w[1], oracle_py.ref_fill(4096, 2, _st12(edge)))


@pytest.mark.gpu
def test_mt_gen3_f64_with_jumps_vs_reference():
    """Generator::next_f64_01 (generator.hpp:39-41) on the register-resident teams: jumped pieces
    and a continuation, bit-exact doubles; checksums cover the u32 draws; the CTA-per-stream
    kernel (MTGP_OPT_KERNEL=1) agrees."""
    sts = [mtgp.mt19937_status(), _rand_status(19937, 300, 4)]
    seeds = [5489, 77]
    lens = [100_000, 404]
    res = {}
    for kern in (0, 1):
        with mtgp.MtContext(sts, seeds) as ctx:
            ctx.set_option(mtgp.OPT_KERNEL, kern)
            ctx.set_option(mtgp.OPT_MIN_PIECE_WORDS, 1 << 12)
            ds, kv = [], []
            for L in lens:
                ds.append(ctx.generate_host(mtgp.F64_01, L))
                kv.append(ctx.last_plan()[2])
            res[kern] = (ds, ctx.checksums(), kv)
    assert res[0][2] == [6, 6] and res[1][2] == [1, 1]
    total = sum(lens)
    for s in range(2):
        u = oracle_py.ref_fill(total, seeds[s], _st12(sts[s]))
        got = np.concatenate([d[s] for d in res[0][0]])
        assert np.array_equal(got, u.astype(np.float64) * (1.0 / 4294967296.0))
        c = oracle_py.cksum(u)
        assert res[0][1][s] == (c["sum64"], c["xor32"], total)
    for a, b in zip(res[0][0], res[1][0]):
        assert np.array_equal(a, b)

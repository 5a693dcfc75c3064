"""CPU: pin the oracle before trusting it.

MTGP32: oracle/mtgp32_oracle.c vs the cuRAND host-compiled known answers
(tests/golden/mtgp32_11213_curand.json).
Engine::mt: oracle/mt_oracle.c vs the reference's own goldens (proj/tests/test_generator.cpp:
11-25, 46-48, 52-57, 67, 90-103) and vs the reference compiled from its sources (oracle/_ref).
"""
import numpy as np
import pytest

import oracle_py
from paper_1501_07701_b200 import tables


def test_curand_table_import(curand_sets):
    assert len(curand_sets) == 200
    assert all(p.mexp == 11213 and p.mask == 0xFFF80000 for p in curand_sets)
    assert min(p.pos for p in curand_sets) == 3 and max(p.pos for p in curand_sets) == 93
    for p in curand_sets:
        p.validate()  # linear tables, flt identity


def test_init_state_golden(curand_sets, curand_golden):
    g = oracle_py.MtgpOracle(curand_sets[0], 1)
    w = g.window()
    want = curand_golden["init_set0_seed1"]
    assert [w[0], w[1], w[2], w[3], w[350]] == [want["x0"], want["x1"], want["x2"], want["x3"], want["x350"]]


def test_first32_all_cases(curand_sets, curand_golden):
    for case in curand_golden["first32"]:
        g = oracle_py.MtgpOracle(curand_sets[case["set"]], case["seed"])
        assert g.fill(32).tolist() == case["u32"], (case["set"], case["seed"])


def test_appendix_b_first8(curand_sets):
    g = oracle_py.MtgpOracle(curand_sets[0], 1)
    assert g.fill(8).tolist() == [360948779, 1200908298, 2313932395, 2218157478, 3754595429,
                                  1713953624, 1821568161, 2144555324]


def test_single_float_matches_curand_temper_single(curand_sets, curand_golden):
    for case in curand_golden["single12"]:
        g = oracle_py.MtgpOracle(curand_sets[case["set"]], case["seed"])
        assert g.fill(32, kind=1).tolist() == case["bits"]


def test_float_01oc_goldens(curand_sets):
    g = oracle_py.MtgpOracle(curand_sets[0], 1)
    assert [hex(v) for v in g.fill(4, kind=2)] == ["0x3f6a7c5c", "0x3f386b98", "0x3eec2864", "0x3ef79338"]
    g = oracle_py.MtgpOracle(curand_sets[0], 1)
    f = g.fill(1 << 14, kind=2).view(np.float32)
    assert f.min() > 0.0 and f.max() <= 1.0


def test_checksums(curand_sets, curand_golden):
    for case in curand_golden["checksums"]:
        g = oracle_py.MtgpOracle(curand_sets[case["set"]], case["seed"])
        if case["skip"]:
            g.skip(case["skip"])
        c = oracle_py.cksum(g.fill(case["n"]))
        assert (c["sum64"], c["xor32"], c["last"], c["poly31"]) == (
            case["sum64"], case["xor32"], case["last"], case["poly31"]), case


def test_all200_weighted(curand_sets, curand_golden):
    out, _ = oracle_py.mtgp_bulk(curand_sets, [1] * 200, 1 << 16, threads=8)
    sums = out.astype(np.uint64).sum(axis=1)
    assert sums.tolist() == curand_golden["all200_seed1_n65536_sum64"]
    w = 0
    for s, v in enumerate(sums.tolist()):
        w = (w + (s + 1) * v) % (1 << 64)
    assert w == curand_golden["all200_seed1_n65536_weighted"] == 2829222411326737783


def test_window_roundtrip(curand_sets):
    g = oracle_py.MtgpOracle(curand_sets[3], 99)
    g.skip(12345)
    h = oracle_py.MtgpOracle.from_window(curand_sets[3], g.window())
    assert np.array_equal(g.fill(5000), h.fill(5000))


def test_synthetic_sets_run(curand_sets):
    for mexp in (23209, 44497):
        for p in tables.synthetic_sets(mexp, 3):
            g = oracle_py.MtgpOracle(p, 1)
            w = g.fill(4096)
            assert len(set(w.tolist())) > 4000  # not degenerate


# ---------------- Engine::mt (the reference's own recurrence) ----------------

def test_mt19937_reference_goldens(mt_golden):
    # proj/tests/test_generator.cpp:11-15
    g = oracle_py.MtOracle(None, 5489)
    assert g.fill(3).tolist() == [3499211612, 581869302, 3890346734]
    g = oracle_py.MtOracle(None, 5489)
    c = oracle_py.cksum(g.fill(1 << 20))
    want = mt_golden["mt19937_seed5489_n1048576"]
    assert (c["sum64"], c["xor32"], c["last"]) == (want["sum64"], want["xor32"], want["last"]) == (
        2252191846071920, 0x612DA44E, 1092562784)


def test_mt19937_temper_golden():
    p = oracle_py.mt19937_params()
    L = oracle_py.lib()
    assert L.oracle_mt_temper(0, p) == 0
    assert L.oracle_mt_temper(0xFFFFFFFF, p) == 0x6FE01BF8  # test_generator.cpp:67
    rng = np.random.default_rng(7)
    for w in rng.integers(0, 1 << 32, 2000, dtype=np.uint64).tolist():
        assert L.oracle_mt_untemper(L.oracle_mt_temper(w, p), p) == w


def test_mt_seed_state_recurrence():
    g = oracle_py.MtOracle(None, 5489)
    assert g.g.st[0] == 5489
    assert g.g.st[1] == (1812433253 * (5489 ^ (5489 >> 30)) + 1) & 0xFFFFFFFF


def test_mt_oracle_vs_compiled_reference(mt_golden):
    pytest.importorskip("ctypes")
    try:
        oracle_py.ref_lib()
    except ImportError:
        pytest.skip("oracle/_ref not built")
    for seed in (0, 1, 5489, 12345, 0xFFFFFFFF):
        a = oracle_py.MtOracle(None, seed).fill(5000)
        b = oracle_py.ref_fill(5000, seed)
        assert np.array_equal(a, b)
    for name in ("dc521_id7", "dc3217_id7"):
        d = mt_golden[name]
        st = d["status12"]
        p = oracle_py.OracleMtParams(st[1], st[2], st[3], st[4], st[5], st[6], st[7], st[8], st[9], st[10], st[11])
        w = oracle_py.MtOracle(p, d["seed"]).fill(d["n"])
        c = oracle_py.cksum(w)
        assert (c["sum64"], c["xor32"], c["last"]) == (d["sum64"], d["xor32"], d["last"])
        assert np.array_equal(w, oracle_py.ref_fill(d["n"], d["seed"], st))


def test_derive_seed_matches_reference_formula():
    L = oracle_py.lib()
    # splitmix64(0) is the published first output of the splitmix64 sequence
    assert L.oracle_splitmix64(0) == 0xE220A8397B1DCDAF
    assert L.oracle_derive_seed(10, 3) == L.oracle_splitmix64(13) & 0xFFFFFFFF


def test_curand_kernel_state_seeds():
    """curandMakeMTGP32KernelState's per-stream seeds (curand_mtgp32_host.h:482-510)."""
    from paper_1501_07701_b200 import tables
    assert tables.curand_kernel_state_seeds(1, 3) == [2, 3, 4]
    s = 0x1234567890ABCDEF
    # low word of seed ^ (seed >> 32) = 0x90ABCDEF ^ 0x12345678 = 0x829F9B97
    assert tables.curand_kernel_state_seeds(s, 2) == [0x829F9B98, 0x829F9B99]
    assert tables.curand_kernel_state_seeds(0xFFFFFFFF, 2) == [0, 1]  # u32 wrap


# ---- streaming checksums and the full-volume parity fixture (tests/golden/full_ck.npz) ----

def _fill_ck(params, seed, n, kind=0, skip=0):
    g = oracle_py.MtgpOracle(params, seed)
    if skip:
        g.skip(skip)
    w = g.fill(n, kind=kind)
    return int(w.astype(np.uint64).sum()), int(np.bitwise_xor.reduce(w))


@pytest.mark.parametrize("mexp", [11213, 23209, 44497])
def test_cksum_stream_matches_fill(mexp):
    """oracle_mtgp_cksum_stream (16 steps per AVX-512 vector) == the word-at-a-time fill,
    for every record, u32 and both float kinds."""
    sets = tables.sets_for(mexp, 3)
    rec, n_rec = 1 << 14, 5
    a, _ = oracle_py.cksum_stream(sets, [1, 7, 0xFFFFFFFF], rec, n_rec, with_float=True, threads=3)
    b, _ = oracle_py.cksum_stream(sets, [1, 7, 0xFFFFFFFF], rec, n_rec, with_float=True, threads=3, scalar=True)
    assert (a == b).all()
    for s, seed in enumerate([1, 7, 0xFFFFFFFF]):
        for kind in range(3):
            sm, x = _fill_ck(sets[s], seed, rec * n_rec, kind)
            assert (int(a[s, -1]["sum"][kind]), int(a[s, -1]["xr"][kind])) == (sm, x)


def test_cksum_stream_cuRAND_golden(curand_sets, curand_golden):
    """The 2^20-word set 0 / seed 1 checksum pinned by cuRAND's own headers (App. B)."""
    a, _ = oracle_py.cksum_stream(curand_sets[:1], [1], 1 << 20, 1, threads=1)
    assert int(a[0, 0]["sum"][0]) == 2251211974485391 and int(a[0, 0]["xr"][0]) == 0x87DB016D


def _full_ck():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    import full_ck
    return full_ck


def test_full_ck_fixture_spot_checks():
    """Re-derive the fixture's first records with the word-at-a-time oracle for certified and
    synthetic streams of every rank range, and one c3 float record."""
    fc = _full_ck()
    if not fc.available():
        pytest.skip("full_ck.npz not generated")
    assert fc.coverage("c2") == (1600, 50, 1 << 27) and fc.coverage("c5") == (1024, 64, 1 << 24)
    ids = [0, 1, 199, 200, 777, 1023]
    sets = [tables.sets_for(11213, 1, first=i)[0] for i in ids]
    got, _ = oracle_py.cksum_stream(sets, [1] * len(ids), 1 << 24, 1, threads=len(ids), scalar=True)
    for j, i in enumerate(ids):
        es, ex = fc.expected("c5", i, 1, 1 << 24)
        assert (int(got[j, 0]["sum"][0]), int(got[j, 0]["xr"][0])) == (int(es[0]), int(ex[0])), i
    for cfg, idx in (("c3-f12", 1), ("c3-f01", 2)):
        es, ex = fc.expected(cfg, 5, 1, 1 << 27)
        a, _ = oracle_py.cksum_stream([tables.sets_for(11213, 1, first=5)[0]], [1], 1 << 27, 1, with_float=True,
                                      threads=1)
        assert (int(a[0, 0]["sum"][idx]), int(a[0, 0]["xr"][idx])) == (int(es[0]), int(ex[0]))
    for mexp in (23209, 44497):
        es, ex = fc.expected(f"c4-{mexp}", 3, 1, 1 << 27)
        a, _ = oracle_py.cksum_stream([tables.sets_for(mexp, 1, first=3)[0]], [1], 1 << 27, 1, threads=1)
        assert (int(a[0, 0]["sum"][0]), int(a[0, 0]["xr"][0])) == (int(es[0]), int(ex[0]))


def test_full_ck_records_are_cumulative():
    """c5's 2^24-word records 8k of a stream are c2's 2^27-word record k (one oracle pass)."""
    fc = _full_ck()
    if not fc.available():
        pytest.skip("full_ck.npz not generated")
    for k in range(1, 9):
        a = fc.expected("c5", 0, 1024, k * (1 << 27))
        b = fc.expected("c2", 0, 1024, k * (1 << 27))
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert fc.expected("c2", 0, 200, 51 << 27) is None and fc.expected("c2", 1500, 200, 1 << 27) is None


def test_full_ck_compare_reports_mismatch():
    fc = _full_ck()
    if not fc.available():
        pytest.skip("full_ck.npz not generated")
    es, ex = fc.expected("c2", 0, 4, 2 << 27)
    good = [(int(s), int(x), 2 << 27) for s, x in zip(es, ex)]
    assert fc.compare("c2", 0, good)["ok"] is True
    bad = list(good)
    bad[2] = (bad[2][0] + 1, bad[2][1], bad[2][2])
    r = fc.compare("c2", 0, bad)
    assert r["ok"] is False and r["mismatched_streams"] == [2]
    # mode 2: sums compared mod 2^32 only
    hi = [((s + (5 << 32)) & 0xFFFFFFFFFFFFFFFF, x, w) for s, x, w in good]
    assert fc.compare("c2", 0, hi, sum_mod32=True)["ok"] is True and fc.compare("c2", 0, hi)["ok"] is False
    assert fc.compare("c2", 0, [(0, 0, 3 << 27)] * 2)["ok"] is False
    assert fc.compare("c2", 0, [(0, 0, 99 << 27)] * 2)["ok"] is None


def test_large_exponents_pinned_by_curand(large_golden):
    """MTGP32-23209 / -44497: the restatement equals cuRAND's own init_state / para_rec /
    temper / temper_single run at N = 726 / 1391 (oracle/curand_pin.cpp --large) -- the
    independent pin these exponents had no other source for."""
    assert {c["mexp"] for c in large_golden} == {23209, 44497}
    for c in large_golden:
        g = oracle_py.MtgpOracle(c["set"], c["seed"])
        w0 = g.window()
        assert [int(w0[0]), int(w0[1]), int(w0[-1])] == c["init_x0_x1_last"]
        w = g.fill(c["n"])
        assert w[:32].tolist() == c["u32"]
        assert (int(w.astype(np.uint64).sum()), int(np.bitwise_xor.reduce(w)), int(w[-1])) == (
            c["sum64"], c["xor32"], c["last"])
        f = oracle_py.MtgpOracle(c["set"], c["seed"]).fill(32, kind=1)
        assert f.tolist() == c["single12_bits"]


def test_mt_full_ck_fixture_matches_restatement():
    """The Engine::mt fixture (made by the reference's own fill(), oracle/_ref) re-derived with
    the C restatement of the reference's recurrence (oracle/mt_oracle.c) for the first record of
    two streams: the fixture, the reference and the restatement agree."""
    fc = _full_ck()
    if not fc.available("mt19937"):
        pytest.skip("mt_full_ck.npz not generated")
    assert fc.coverage("mt19937") == (200, 50, 1 << 27)
    for s in (0, 199):
        g = oracle_py.MtOracle(None, 5489 + s)
        sm, x = 0, 0
        for _ in range(8):  # 2^27 words in 2^24-word pieces
            w = g.fill(1 << 24)
            sm += int(w.astype(np.uint64).sum())
            x ^= int(np.bitwise_xor.reduce(w))
        es, ex = fc.expected("mt19937", s, 1, 1 << 27)
        assert (sm & 0xFFFFFFFFFFFFFFFF, x) == (int(es[0]), int(ex[0])), s

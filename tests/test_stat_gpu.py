"""GPU parity of the device-side statistical tests (csrc/mtgp_stat.cu) against the reference's
own templates (proj/include/twistsieve/stat_tests.hpp:84-309, compiled from its sources into
oracle/_ref) run over the same words, and against the reference's campaign cells
(sieve.cpp:156-158) frozen in tests/golden/stat_reference.json. Bar: bit-exact statistic,
p-value, class, degenerate flag and words consumed."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_py
import stat_oracle as so
from paper_1501_07701_b200 import mtgp, shard
from paper_1501_07701_b200 import stattests as st

pytestmark = pytest.mark.gpu
GOLD = json.loads((Path(__file__).parent / "golden" / "stat_reference.json").read_text())


def _same(r: st.TestResult, ref: dict, words=True):
    assert ref["rc"] == 0, ref["error"]
    assert not r.error
    assert r.statistic == ref["statistic"]
    assert r.p_value == ref["p_value"]
    assert st.CLASSES.index(r.classification) == ref["classification"]
    assert int(r.degenerate) == ref["degenerate"]
    if words:
        assert r.words_used == ref["words_used"]


def _mtgp_streams(k, first=0):
    sets = shard.sets_for_rank(11213, 200, 0)[first:first + k]
    seeds = [oracle_py.lib().oracle_derive_seed(99, j) for j in range(k)]
    return sets, seeds


SPECS = [
    st.desk_gap_spec(),
    st.desk_hamming_spec(),
    st.desk_opso_spec(),
    st.desk_walk_spec(),
    st.TestSpec("gap", n=50000, r=3, alpha=0.3, beta=0.7),
    st.TestSpec("gap", n=20000, r=0, alpha=0.9, beta=1.0),
    st.TestSpec("hamming_indep", n=30001, r=2, s=7, L=33),
    st.TestSpec("hamming_indep", n=20000, r=0, s=31, L=7),
    st.TestSpec("hamming_indep", n=20000, r=20, s=1, L=64),
    st.TestSpec("hamming_indep", n=4000, r=10, s=13, L=4000),
    st.TestSpec("collision_over", n=3000, r=5, s=7),
    st.TestSpec("collision_over", n=200, r=28, s=2),
    st.TestSpec("collision_over", n=1500000, r=0, s=14),   # 2 chunks, 2^28-cell map
    st.TestSpec("random_walk", n=20000, l=6),
    st.TestSpec("random_walk", n=3000, l=1000),
    st.TestSpec("random_walk", n=600000, l=2),             # 2 chunks
    st.TestSpec("random_walk", n=5000, l=1020),            # near the longest walk with a non-zero pmf[0]
]


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.describe())
def test_stat_run_matches_reference_templates(spec):
    sets, seeds = _mtgp_streams(3, first=20)
    with mtgp.MtgpContext(sets, seeds) as ctx:
        res = ctx.stat_run(spec)
    need = {"gap": 40_000_000, "hamming_indep": None, "collision_over": spec.n + 1, "random_walk": spec.n * spec.l}
    n_words = need[spec.test_id] or -(-(spec.n // 2) * 2 * spec.L // spec.s)
    if spec.test_id == "gap":
        n_words = int(min(n_words, (spec.n + 1) / (spec.beta - spec.alpha) * 3))
    words, _ = oracle_py.mtgp_bulk(sets, seeds, n_words, threads=3)
    for s in range(3):
        _same(res[s], so.ref_run_words(words[s], spec))


def test_stat_run_leaves_context_state_unchanged():
    sets, seeds = _mtgp_streams(4)
    with mtgp.MtgpContext(sets, seeds) as ctx:
        a = ctx.fill_u32(1000)
        ck = ctx.checksums()
        r1 = ctx.stat_run(st.desk_walk_spec())
        assert ctx.position(0) == 1000 and ctx.checksums() == ck
        b = ctx.fill_u32(5000)
        r2 = ctx.stat_run(st.desk_walk_spec())
    o = oracle_py.mtgp_bulk(sets, seeds, 6000, threads=4)[0]
    assert np.array_equal(np.concatenate([a, b], axis=1), o)
    # the test starts at the context's position: r1 over words [1000, ...), r2 over [6000, ...)
    w1, _ = oracle_py.mtgp_bulk(sets, seeds, 100000 * 128, skip=1000, threads=4)
    w2, _ = oracle_py.mtgp_bulk(sets, seeds, 100000 * 128, skip=6000, threads=4)
    for s in range(4):
        _same(r1[s], so.ref_run_words(w1[s], st.desk_walk_spec()))
        _same(r2[s], so.ref_run_words(w2[s], st.desk_walk_spec()))


def test_gap_exhaustion_is_reported_per_stream():
    """Kept bits r = 31 leave u in {0, 0.5}: [0.1, 0.2) is never visited, the reference throws
    StreamExhausted after its word budget (stat_tests.hpp:106-111)."""
    spec = st.TestSpec("gap", n=10, r=31, alpha=0.1, beta=0.2)
    sets, seeds = _mtgp_streams(2)
    with mtgp.MtgpContext(sets, seeds) as ctx:
        res = ctx.stat_run(spec)
    words, _ = oracle_py.mtgp_bulk(sets, seeds, 8192, threads=2)
    for s in range(2):
        ref = so.ref_run_words(words[s], spec)
        assert ref["rc"] == 2 and ref["error"] == st.EXHAUSTED_MSG
        assert res[s].error == st.EXHAUSTED_MSG and res[s].is_error()


def test_gap_many_streams_23209():
    """Gap test over 16 synthetic MTGP32-23209 streams (v2 generator path)."""
    from paper_1501_07701_b200 import tables
    sets = tables.synthetic_sets(23209, 16)
    seeds = list(range(100, 116))
    spec = st.TestSpec("gap", n=100000, r=25, alpha=0.0, beta=1 / 32)
    with mtgp.MtgpContext(sets, seeds) as ctx:
        res = ctx.stat_run(spec)
    words, _ = oracle_py.mtgp_bulk(sets, seeds, 4_000_000, threads=16)
    for s in range(16):
        _same(res[s], so.ref_run_words(words[s], spec))


@pytest.mark.parametrize("spec", [st.desk_gap_spec(), st.desk_hamming_spec(), st.desk_opso_spec(),
                                  st.desk_walk_spec()], ids=lambda s: s.test_id)
def test_engine_mt_cells_match_reference_campaign(spec):
    """Engine::mt on the GPU + device-side test == the reference's own campaign cell
    (make_word_source -> BufferedStream -> run_test) for MT19937 and DC-minted statuses."""
    mt_gold = json.loads((Path(__file__).parent / "golden" / "mt_reference.json").read_text())
    keys = ("id", "mexp", "n", "m", "r", "a", "temper_b", "temper_c", "temper_u", "temper_s", "temper_t", "temper_l")
    dc = dict(zip(keys, mt_gold["dc3217_id7"]["status12"]))
    statuses = [mtgp.mt19937_status(), mtgp.mt19937_status(), dc]
    seeds = [5489, 77, 4357]
    with mtgp.MtContext(statuses, seeds) as ctx:
        res = ctx.stat_run(spec)
    for s in range(3):
        st12 = None if s < 2 else mt_gold["dc3217_id7"]["status12"]
        _same(res[s], so.ref_run_cell(seeds[s], spec, st12), words=False)


def test_run_grid_reproduces_reference_campaign_goldens():
    """GPU run_grid over MT19937 x {5489, 1, 0xDEADBEEF} x desk battery == the reference cells
    frozen in tests/golden/stat_reference.json (no reference needed at run time)."""
    seeds = [5489, 1, 0xDEADBEEF]
    rows = st.run_grid([mtgp.mt19937_status()], seeds, st.desk_battery(), engine="mt")
    assert len(rows) == len(GOLD["cells"])
    for row, cell in zip(rows, GOLD["cells"]):
        assert (row.seed, row.test_id) == (cell["seed"], cell["spec"]["test_id"])
        assert row.statistic == float.fromhex(cell["statistic"])
        assert row.p_value == float.fromhex(cell["p_value"])
        assert st.CLASSES.index(row.classification) == cell["classification"]


def test_run_grid_error_rows_and_order():
    sets, _ = _mtgp_streams(2)
    specs = [st.TestSpec("random_walk", n=10, l=128), st.TestSpec("random_walk", n=2000, l=64)]
    rows = st.run_grid(sets, [1, 2, 3], specs, status_ids=["a", "b"])
    assert [(r.status_id, r.seed_index, r.test_id) for r in rows[:4]] == [
        ("a", 0, "random_walk"), ("a", 0, "random_walk"), ("a", 1, "random_walk"), ("a", 1, "random_walk")]
    assert all(r.error == "sample too small" for r in rows[0::2])
    assert not any(r.error for r in rows[1::2])

"""CPU checks of the device-side stat tests' host half (no GPU): the numerics, spec validation and
counts -> (statistic, p-value, class) of csrc/stat_host.cpp against the reference's own
stat_tests.hpp / stats.cpp / classify.cpp -- through the frozen goldens in
tests/golden/stat_reference.json and live against the reference compiled from its sources
(oracle/_ref). The bar is bit-exact: the reference hand-rolls its numerics so report bytes are
platform independent (stats.hpp:9-10), and the restatement keeps its operation order."""
import json
from pathlib import Path

import numpy as np
import pytest

import oracle_py
import stat_oracle as so
from paper_1501_07701_b200 import mtgp, shard
from paper_1501_07701_b200 import stattests as st

GOLD = json.loads((Path(__file__).parent / "golden" / "stat_reference.json").read_text())
MATH_FN = {"ln_gamma": lambda a, b, k, n: st.ln_gamma(a), "gamma_p": lambda a, b, k, n: st.gamma_p(a, b),
           "gamma_q": lambda a, b, k, n: st.gamma_q(a, b),
           "chi_square_pvalue": lambda a, b, k, n: st.chi_square_pvalue(a, k),
           "poisson_cdf": lambda a, b, k, n: st.poisson_cdf(k, a), "poisson_sf": lambda a, b, k, n: st.poisson_sf(k, a),
           "poisson_pmf": lambda a, b, k, n: st.poisson_pmf(k, a),
           "binomial_log_pmf": lambda a, b, k, n: st.binomial_log_pmf(k, n, a),
           "binomial_upper_tail": lambda a, b, k, n: st.binomial_upper_tail(k, n, a),
           "classify_pvalue": lambda a, b, k, n: float(st.CLASSES.index(st.classify_pvalue(a)))}


@pytest.mark.parametrize("case", GOLD["math"], ids=lambda c: f"{c['fn']}({c['a']},{c['b']},{c['k']},{c['n']})")
def test_numerics_match_reference_goldens(case):
    a, b = float.fromhex(case["a"]), float.fromhex(case["b"])
    fn = MATH_FN[case["fn"]]
    if case["rc"]:
        with pytest.raises(mtgp.MtgpInvalidArgument) as e:
            fn(a, b, case["k"], case["n"])
        assert case["msg"] in str(e.value)
    else:
        assert fn(a, b, case["k"], case["n"]) == float.fromhex(case["value"])  # bit-exact


@pytest.mark.parametrize("case", GOLD["cases"], ids=lambda c: f"{c['spec']['test_id']}-{c['set']}")
def test_finish_from_counts_matches_reference_goldens(case):
    spec = st.TestSpec(**case["spec"])
    r = st.finish_counts(spec, case["counts"])
    assert r.statistic == float.fromhex(case["statistic"])
    assert r.p_value == float.fromhex(case["p_value"])
    assert st.CLASSES.index(r.classification) == case["classification"]
    assert int(r.degenerate) == case["degenerate"]


def test_numerics_live_grid_vs_compiled_reference():
    rng = np.random.default_rng(7)
    for a, x in zip(rng.uniform(0.05, 300, 200), rng.uniform(0, 400, 200)):
        for fn, mine in (("gamma_p", st.gamma_p), ("gamma_q", st.gamma_q)):
            rc, v, _ = so.ref_math(fn, a, x)
            assert rc == 0 and mine(a, x) == v
    for stat, df in zip(rng.uniform(0, 2000, 200), rng.integers(1, 2000, 200)):
        assert st.chi_square_pvalue(stat, int(df)) == so.ref_math("chi_square_pvalue", stat, 0, int(df))[1]


BAD_SPECS = [
    dict(test_id="gap", n=0, beta=0.5),
    dict(test_id="gap", n=10, r=32, beta=0.5),
    dict(test_id="gap", n=10, alpha=0.5, beta=0.5),
    dict(test_id="gap", n=10, alpha=0.0, beta=1.5),
    dict(test_id="hamming_indep", n=1000, s=0, L=10),
    dict(test_id="hamming_indep", n=1000, r=30, s=5, L=10),
    dict(test_id="hamming_indep", n=1000, s=5, L=0),
    dict(test_id="hamming_indep", n=1000, s=5, L=10, d=1),
    dict(test_id="hamming_indep", n=199, s=5, L=10),          # sample too small (npairs < 100)
    dict(test_id="collision_over", n=1000, s=15),
    dict(test_id="collision_over", n=1000, r=20, s=14),
    dict(test_id="collision_over", n=1000, s=5, t=9),
    dict(test_id="collision_over", n=10, s=11),               # lambda < 1: out of sparse regime
    dict(test_id="random_walk", n=100, l=3),
    dict(test_id="random_walk", n=100, l=0),
    dict(test_id="random_walk", n=10, l=128),                 # sample too small
]


@pytest.mark.parametrize("fields", BAD_SPECS, ids=lambda f: f"{f['test_id']}-{len(str(f))}")
def test_validation_messages_match_reference(fields):
    spec = st.TestSpec(**fields)
    ref = so.ref_run_words(np.zeros(16, dtype=np.uint32), spec)
    assert ref["rc"] == 1
    with pytest.raises(mtgp.MtgpInvalidArgument) as e:
        spec.validate()
    assert str(e.value).endswith(ref["error"])


def test_unknown_test_id():
    with pytest.raises(mtgp.MtgpInvalidArgument, match="unknown test"):
        st.TestSpec("birthday", n=10).validate()
    with pytest.raises(mtgp.MtgpInvalidArgument, match="unknown test name"):
        st.named_spec("birthday")


def test_desk_specs_and_aliases_match_reference():
    for i, mine in enumerate(st.desk_battery()):
        r = so.ref_desk_spec(i)
        assert so.to_ref(mine).test == r.test
        for k in ("N", "n", "r", "s", "L", "d", "l", "t", "alpha", "beta"):
            assert getattr(so.to_ref(mine), k) == getattr(r, k), k
    assert st.named_spec("opso") == st.desk_opso_spec()
    assert st.named_spec("walk").test_id == "random_walk"
    assert st.named_spec("hamming").describe() == "hamming_indep(n=100000,r=25,s=5,L=1200,d=0)"


@pytest.mark.parametrize("beta", [1 / 32, 0.5, 0.999, 1e-3])
def test_gap_tail_cut_matches_reference(beta):
    spec = st.TestSpec("gap", n=1000000, r=25, alpha=0.0, beta=beta)
    assert st.counts_len(spec) - 1 == so.ref_gap_tcut(spec)


@pytest.mark.parametrize("fields", [
    dict(test_id="gap", n=3000, r=0, alpha=0.25, beta=0.2500001),
    dict(test_id="gap", n=4000, r=31, alpha=0.0, beta=0.5),
    dict(test_id="hamming_indep", n=2000, r=0, s=31, L=7),
    dict(test_id="hamming_indep", n=2000, r=20, s=1, L=64),
    dict(test_id="collision_over", n=200, r=28, s=2),
    dict(test_id="random_walk", n=3000, l=1000),
    dict(test_id="random_walk", n=70000, l=2),
], ids=lambda f: f"{f['test_id']}")
def test_finish_vs_reference_templates_on_oracle_words(fields):
    """Counts restated in numpy over MTGP32 oracle words -> mtgp_stat_finish == the reference
    template run over the same words (edge shapes: 1-bit letters, 31-bit letters, 2-bit cells,
    long walks, a nearly empty gap interval)."""
    spec = st.TestSpec(**fields)
    sets = shard.sets_for_rank(11213, 200, 0)
    words, _ = oracle_py.mtgp_bulk(sets[5:7], [11, 12], 1 << 22, threads=2)
    for w in words:
        ref = so.ref_run_words(w, spec)
        if spec.test_id == "gap":
            tcut = so.ref_gap_tcut(spec)
            budget = int(float(spec.n + 1) / (spec.beta - spec.alpha) * 8.0) + 4096
            got = so.gap_counts(w, spec, tcut, budget)
            if got is None:
                assert ref["rc"] == 2
                continue
            counts, used = got
            assert used == ref["words_used"]
        else:
            counts = {"hamming_indep": so.hamming_counts, "collision_over": so.collision_counts,
                      "random_walk": so.walk_counts}[spec.test_id](w, spec)
        assert ref["rc"] == 0, ref["error"]
        r = st.finish_counts(spec, counts)
        assert (r.statistic, r.p_value, st.CLASSES.index(r.classification), int(r.degenerate)) == \
            (ref["statistic"], ref["p_value"], ref["classification"], ref["degenerate"])


def test_hamming_degenerate_table():
    spec = st.TestSpec("hamming_indep", n=400, s=5, L=10)
    r = st.finish_counts(spec, [200, 0, 0, 0])
    assert r.degenerate and r.p_value == 1.0 and r.statistic == 0.0


def test_finish_rejects_wrong_count_length():
    with pytest.raises(mtgp.MtgpInvalidArgument, match="wrong length"):
        st.finish_counts(st.desk_walk_spec(), [0] * 10)

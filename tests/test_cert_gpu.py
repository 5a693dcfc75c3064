"""GPU: parameter-set certification and the reference's charpoly digests.

Engine::mt: the GPU-generated probe -> Berlekamp-Massey -> poly_digest must reproduce the
reference's digests (its MT19937 preset golden and its DC-minted statuses), and certification
must accept them. MTGP32: the 200 certified cuRAND sets must certify; synthetic (uncertified)
sets must get the answer the reference's own dc_search test gives on the same output stream."""
import json
from pathlib import Path

import pytest

import oracle_py
import stat_oracle as so
from paper_1501_07701_b200 import mtgp, tables

pytestmark = pytest.mark.gpu
MT = json.loads((Path(__file__).parent / "golden" / "mt_reference.json").read_text())
KEYS = ("id", "mexp", "n", "m", "r", "a", "temper_b", "temper_c", "temper_u", "temper_s", "temper_t", "temper_l")


def test_mt_probe_digests_and_certification():
    sts = [mtgp.mt19937_status()] + [dict(zip(KEYS, MT[k]["status12"])) for k in ("dc521_id7", "dc3217_id7")]
    with mtgp.MtContext(sts, [1, 1, 1]) as ctx:  # kDefaultProbeSeed = 1 (dynamic_creator.hpp:30)
        w0 = ctx.fill_u32(3)                      # the probe leaves the state alone ...
        dig = ctx.mt_charpoly_digest()
        cert = ctx.certify()
        w1 = ctx.fill_u32(3)
    assert dig[0] == "736dbad14b19609ef909097e1b440834727ed02c"  # params.cpp:75
    assert dig[1] == MT["dc521_id7"]["probe_digest_seed1"][0]
    assert dig[2] == MT["dc3217_id7"]["probe_digest_seed1"][0]
    assert cert == [True, True, True]
    ref = oracle_py.MtOracle(None, 1).fill(6)
    assert list(w0[0]) + list(w1[0]) == list(ref)               # ... and the position


def test_mtgp_certified_table_certifies(curand_sets):
    with mtgp.MtgpContext(curand_sets, [1] * 200) as ctx:
        assert all(ctx.certify())


@pytest.mark.parametrize("mexp", [23209, 44497])
def test_mtgp_synthetic_sets_match_reference_dc_test(mexp):
    sets = tables.synthetic_sets(mexp, 6)
    seeds = [11, 12, 13, 14, 15, 16]
    with mtgp.MtgpContext(sets, seeds) as ctx:
        cert = ctx.certify()
    for s in range(6):
        words = oracle_py.MtgpOracle(sets[s], seeds[s]).fill(2 * mexp + 64)
        degree, irr = so.ref_bit0_certify(words, mexp)
        assert cert[s] == (degree == mexp and irr == 1), (s, degree, irr)

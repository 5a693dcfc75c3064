"""CPU checks of the parameter-set certifier's algebra (csrc/gf2.cpp is_irreducible, through the
C-ABI mtgp_gf2_is_irreducible) against the reference's own is_irreducible
(proj/src/gf2poly.cpp:342-383, compiled from its sources into oracle/_ref)."""
import json
from pathlib import Path

import numpy as np
import pytest

import stat_oracle as so
from paper_1501_07701_b200 import mtgp

GOLD = json.loads((Path(__file__).parent / "golden" / "mt_reference.json").read_text())


def _tri(n, k):
    c = np.zeros(n + 1, dtype=np.uint8)
    c[[0, k, n]] = 1
    return c


def _mul(a, b):
    r = np.zeros(a.size + b.size - 1, dtype=np.uint8)
    for i in np.flatnonzero(a):
        r[i:i + b.size] ^= b
    return r


@pytest.mark.parametrize("poly", [
    _tri(89, 38), _tri(127, 1), _tri(521, 32), _tri(607, 105), _tri(1279, 216),  # primitive trinomials
    _tri(8, 0), _tri(200, 3), _tri(127, 2), _mul(_tri(89, 38), _tri(127, 1)), _mul(_tri(31, 3), _tri(31, 3)),
    np.array([1, 1], dtype=np.uint8), np.array([0, 1], dtype=np.uint8), np.array([1, 1, 1], dtype=np.uint8),
], ids=lambda p: f"deg{p.size - 1}")
def test_irreducible_known_cases_match_reference(poly):
    assert mtgp.gf2_is_irreducible(poly) == bool(so.ref_is_irreducible(poly))


def test_irreducible_random_polynomials_match_reference():
    rng = np.random.default_rng(1501)
    found = 0
    for _ in range(300):
        d = int(rng.integers(2, 160))
        c = rng.integers(0, 2, d + 1).astype(np.uint8)
        c[d] = 1
        ours = mtgp.gf2_is_irreducible(c)
        assert ours == bool(so.ref_is_irreducible(c)), d
        found += ours
    assert found >= 3  # about 1/d of them are irreducible


def test_constant_polynomial_rejected_like_the_reference():
    with pytest.raises(mtgp.MtgpInvalidArgument, match="constant"):
        mtgp.gf2_is_irreducible(np.array([1], dtype=np.uint8))
    assert so.ref_is_irreducible(np.array([1], dtype=np.uint8)) == -1


def test_probe_digest_goldens_are_the_references():
    """The frozen probe digests equal the reference's own MT19937 preset digest
    (proj/src/params.cpp:75, proj/tests/test_dynamic_creator.cpp:34-41)."""
    assert GOLD["probe_digest_mt19937_seed1"] == ["736dbad14b19609ef909097e1b440834727ed02c", 19937]
    assert so.ref_mt_probe_digest(1) == ("736dbad14b19609ef909097e1b440834727ed02c", 19937)

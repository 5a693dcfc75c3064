import json
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on a GPU box)")
    config.addinivalue_line("markers", "slow: long-running full-size check")


@pytest.fixture(scope="session")
def curand_sets():
    from paper_1501_07701_b200 import tables
    return tables.load_curand_11213()


@pytest.fixture(scope="session")
def curand_golden():
    return json.loads((GOLDEN / "mtgp32_11213_curand.json").read_text())


@pytest.fixture(scope="session")
def mt_golden():
    return json.loads((GOLDEN / "mt_reference.json").read_text())


@pytest.fixture(scope="session")
def large_golden():
    """cuRAND-driven known answers at MTGP32-23209 / -44497 (tests/golden/make_goldens.py)."""
    from paper_1501_07701_b200 import tables
    d = json.loads((GOLDEN / "mtgp32_large_curand.json").read_text())
    for c in d["cases"]:
        c["set"] = tables.MtgpParams(certified=False, **c["params"])
    return d["cases"]

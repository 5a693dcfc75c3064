"""The drop-in compiled against the reference itself (oracle/_ref/test_ref_binding, built by
oracle/Makefile from tests/cpp/test_ref_binding.cpp where /root/reference exists; the binary
travels to the GPU box): our C++ layer with -DTWISTSIEVE_B200_WITH_REFERENCE, the reference's
make_word_source signature dispatching on Engine (proj/src/word_source.cpp:5-16), its
BufferedStream (word_source.hpp:80-97) and run_test (stat_tests.hpp:312-319) fed by GPU words."""
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "oracle" / "_ref" / "test_ref_binding"
GOLDEN = ROOT / "tests" / "golden" / "mtgp32_11213_curand.json"


def _need_exe():
    if not EXE.exists():
        if Path("/root/reference/proj/include").exists():
            pytest.fail(f"{EXE} missing: run `make -C oracle binding` (build() does)")
        pytest.skip("reference binding binary not built here (no /root/reference and no prebuilt binary)")


def test_ref_binding_cpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("the no-device case is for CPU hosts; GPU hosts run test_ref_binding_gpu")
    _need_exe()
    r = subprocess.run([str(EXE), str(GOLDEN), "--cpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_ref_binding_gpu():
    _need_exe()
    r = subprocess.run([str(EXE), str(GOLDEN), "--gpu"], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout + r.stderr

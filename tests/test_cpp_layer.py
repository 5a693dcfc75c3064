"""Build and run the C++ drop-in layer's tests (tests/cpp/test_twistsieve_b200.cpp) and the
jump-ahead algebra test (tests/cpp/test_gf2.cpp)."""
import json
import subprocess
from pathlib import Path

import pytest

from paper_1501_07701_b200 import tables

ROOT = Path(__file__).resolve().parents[1]
PKG = ROOT / "paper_1501_07701_b200"


def _build(tmp_path, name, srcs, extra=()):
    exe = tmp_path / name
    cmd = ["g++", "-std=c++20", "-O2", "-I", str(ROOT / "include"), "-I", str(PKG / "csrc"), "-I", str(ROOT / "oracle"),
           *map(str, srcs), *extra, "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


@pytest.fixture(scope="module")
def layer_exe(tmp_path_factory):
    d = tmp_path_factory.mktemp("cpp")
    return _build(d, "test_twistsieve_b200", [ROOT / "tests/cpp/test_twistsieve_b200.cpp"],
                  ["-x", "c", str(ROOT / "oracle/mtgp32_oracle.c"), str(ROOT / "oracle/mt_oracle.c"), "-x", "none",
                   "-I", "/usr/local/cuda/include", "-L", str(PKG), "-ltwistsieve_b200", "-lmtgp_b200",
                   f"-Wl,-rpath,{PKG}", "-L", "/usr/local/cuda/lib64", "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64",
                   "-lpthread"])


def _pyfile(tmp_path):
    f = tmp_path / "py_sets.jsonl"
    tables.write_status_file(f, [tables.load_curand_11213()[0], tables.synthetic_set(23209, 1)])
    return f


def test_cpp_layer_cpu(layer_exe, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("the no-device case is for CPU hosts; GPU hosts run test_cpp_layer_gpu")
    r = subprocess.run([str(layer_exe), str(ROOT / "tests/golden/mtgp32_11213_curand.json"), "--cpu",
                        str(_pyfile(tmp_path))], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_layer_gpu(layer_exe, tmp_path):
    r = subprocess.run([str(layer_exe), str(ROOT / "tests/golden/mtgp32_11213_curand.json"), "--gpu",
                        str(_pyfile(tmp_path))], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    # the threading-model cases report their aggregate rate (pytest -s shows it;
    # profiles/r2/threading.txt)
    print("\n".join(line for line in r.stdout.splitlines() if "THREADS" in line))
    assert r.stdout.count("every word == oracle: yes") == 2, r.stdout


def test_gf2_jump_algebra(tmp_path):
    """BM charpoly, Barrett x^o mod P, and jumped windows vs the oracle (certified + synthetic)."""
    exe = _build(tmp_path, "test_gf2", [ROOT / "tests/cpp/test_gf2.cpp", PKG / "csrc/gf2.cpp", PKG / "csrc/sha1.cpp"],
                 ["-mpclmul", "-msse4.1", "-x", "c", str(ROOT / "oracle/mtgp32_oracle.c"),
                  str(ROOT / "oracle/mt_oracle.c"), "-x", "none", "-lpthread"])
    sets = tables.load_curand_11213()[:2] + tables.synthetic_sets(44497, 1)
    pf = tmp_path / "params.txt"
    pf.write_text("".join(" ".join(str(v) for v in [p.mexp, p.pos, p.sh1, p.sh2, *p.tbl, *p.tmp_tbl, p.mask]) + "\n"
                          for p in sets))
    r = subprocess.run([str(exe), str(pf)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "BM degree 11213" in r.stdout
    # the characteristic polynomials of the certified sets digest to the table's poly_sha1
    digests = [line.split()[1] for line in r.stdout.splitlines() if line.strip().startswith("digest")]
    assert digests[:2] == [sets[0].poly_sha1, sets[1].poly_sha1]


# ---------------- stat-test layer (include/twistsieve_b200/stat_tests.hpp) ----------------

@pytest.fixture(scope="module")
def stat_exe(tmp_path_factory):
    d = tmp_path_factory.mktemp("cpp_stat")
    return _build(d, "test_stat_b200", [ROOT / "tests/cpp/test_stat_b200.cpp"],
                  ["-L", str(PKG), "-ltwistsieve_b200", "-lmtgp_b200", f"-Wl,-rpath,{PKG}"])


def _stat_cases(tmp_path):
    """Flatten tests/golden/stat_reference.json (the reference's own results) for the C++ test."""
    g = json.loads((ROOT / "tests/golden/stat_reference.json").read_text())
    lines = [f"math {m['fn']} {m['a']} {m['b']} {m['k']} {m['n']} {m['value']}" for m in g["math"] if m["rc"] == 0]
    for c in g["cases"]:
        sp = c["spec"]
        f = [sp["test_id"], sp.get("n", 0), sp.get("r", 0), float(sp.get("alpha", 0.0)).hex(),
             float(sp.get("beta", 0.0)).hex(), sp.get("s", 0), sp.get("L", 0), sp.get("d", 0), sp.get("l", 0),
             sp.get("t", 0), c["set"], c["seed"], c["statistic"], c["p_value"], c["classification"], c["degenerate"]]
        lines.append("case " + " ".join(str(x) for x in f))
    for c in g["cells"]:
        lines.append(f"cell {c['spec']['test_id']} {c['seed']} {c['statistic']} {c['p_value']} {c['classification']}")
    f = tmp_path / "stat_cases.txt"
    f.write_text("\n".join(lines) + "\n")
    return f


def _curand_header():
    for d in tables._cuda_include_dirs():
        if (d / "curand_mtgp32dc_p_11213.h").exists():
            return d / "curand_mtgp32dc_p_11213.h"
    pytest.skip("curand_mtgp32dc_p_11213.h not found")


def test_cpp_stat_layer_cpu(stat_exe, tmp_path):
    """Specs, messages, classify and the numerics (bit-exact vs the reference's values), no GPU."""
    r = subprocess.run([str(stat_exe), str(_stat_cases(tmp_path)), str(_curand_header())],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_stat_layer_gpu(stat_exe, tmp_path):
    """run_test on MTGP32 streams and run_grid on Engine::mt == the reference's results."""
    r = subprocess.run([str(stat_exe), str(_stat_cases(tmp_path)), str(_curand_header()), "--gpu"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr

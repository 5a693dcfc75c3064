"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/mtgp_b200.h
declares, validates parameter sets like the reference's validate() (no GPU needed), and refuses
to run without a device (no CPU fallback)."""
import ctypes as C
import re
from pathlib import Path

import pytest

from paper_1501_07701_b200 import mtgp, tables

ROOT = Path(__file__).resolve().parents[1]


def test_header_declares_exactly_the_exports():
    hdr = (ROOT / "include" / "mtgp_b200.h").read_text()
    declared = set(re.findall(r"\b(mtgp_[a-z0-9_]+)\s*\(", hdr))
    assert declared == set(mtgp.EXPORTS)


def test_library_loads_and_exports():
    lib = mtgp.load_library()
    for name in mtgp.EXPORTS:
        assert hasattr(lib, name), name
    assert lib.mtgp_abi_version() == 1


def test_validate_accepts_curand_sets(curand_sets):
    for p in curand_sets[:20]:
        mtgp.validate(p)


@pytest.mark.parametrize("field,value,msg", [
    ("mexp", 11214, "unsupported period exponent"),
    ("mask", 0xFFF00000, "mask"),
    ("sh1", 0, "shifts"),
    ("sh2", 32, "shifts"),
    ("pos", 1, "pick-up position"),
    ("pos", 340, "pick-up position"),
])
def test_validate_rejects(curand_sets, field, value, msg):
    p = tables.MtgpParams(**{**curand_sets[0].__dict__})
    setattr(p, field, value)
    with pytest.raises(mtgp.MtgpInvalidArgument, match=msg):
        mtgp.validate(p)
    with pytest.raises(ValueError):
        p.validate()


def test_validate_rejects_nonlinear_and_bad_float_tables(curand_sets):
    p = tables.MtgpParams(**{**curand_sets[0].__dict__})
    p.tbl = list(p.tbl)
    p.tbl[3] ^= 1
    with pytest.raises(mtgp.MtgpInvalidArgument, match="linear"):
        mtgp.validate(p)
    q = tables.MtgpParams(**{**curand_sets[0].__dict__})
    q.flt_tmp_tbl = list(q.flt_tmp_tbl)
    q.flt_tmp_tbl[5] ^= 1
    with pytest.raises(mtgp.MtgpInvalidArgument, match="flt_tmp_tbl"):
        mtgp.validate(q)


def test_no_cpu_fallback(curand_sets):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(mtgp.MtgpError) as ei:
        mtgp.MtgpContext(curand_sets[:1], [1])
    assert ei.value.code == mtgp.MTGP_ECUDA


def test_status_file_roundtrip(tmp_path, curand_sets):
    f = tmp_path / "sets.jsonl"
    syn = tables.synthetic_sets(44497, 2)
    tables.write_status_file(f, curand_sets[:3] + syn)
    back = tables.read_status_file(f)
    assert [b.__dict__ for b in back] == [p.__dict__ for p in curand_sets[:3] + syn]


def test_status_file_kv_and_errors(tmp_path, curand_sets):
    p = curand_sets[5]
    line = (f"id=5 engine=mtgp32 mexp=11213 pos={p.pos} sh1=0x{p.sh1:x} sh2={p.sh2} "
            f"tbl={','.join(hex(v) for v in p.tbl)} tmp_tbl={','.join(str(v) for v in p.tmp_tbl)}")
    q = tables.status_from_line(line)
    assert (q.pos, q.sh1, q.tbl, q.flt_tmp_tbl) == (p.pos, p.sh1, p.tbl, p.flt_tmp_tbl)
    f = tmp_path / "bad.jsonl"
    f.write_text("# comment\n\n" + tables.status_to_json_line(p) + "\nid=1 bogus=3\n")
    with pytest.raises(RuntimeError, match=r"bad.jsonl:4: unknown status field"):
        tables.read_status_file(f)

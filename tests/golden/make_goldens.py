"""Regenerate the frozen golden fixtures in tests/golden/ (run HERE, not on the GPU box).

1. mtgp32_11213_curand.json -- oracle/_ref/curand_pin: cuRAND's MTGP32 headers compiled
   host-side (independent implementation of the same published algorithm).
2. mt_reference.json -- the UNMODIFIED reference generator compiled from /root/reference
   (oracle/_ref/libtwistsieve_ref.so): MT19937 seed 5489 words and checksums, temper goldens.

    make -C oracle && python tests/golden/make_goldens.py
"""
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

import numpy as np  # noqa: E402

import oracle_py  # noqa: E402


def main():
    out = subprocess.run([str(ROOT / "oracle/_ref/curand_pin")], check=True, capture_output=True, text=True).stdout
    d = json.loads(out)
    (ROOT / "tests/golden/mtgp32_11213_curand.json").write_text(json.dumps(d, indent=1) + "\n")

    ref = {}
    w = oracle_py.ref_fill(1 << 20, 5489)
    ref["mt19937_seed5489_first16"] = [int(x) for x in w[:16]]
    c = oracle_py.cksum(w)
    ref["mt19937_seed5489_n1048576"] = {k: int(v) for k, v in c.items()}
    for seed in (0, 1, 12345, 0xFFFFFFFF):
        w = oracle_py.ref_fill(4096, seed)
        ref[f"mt19937_seed{seed}_n4096"] = {k: int(v) for k, v in oracle_py.cksum(w).items()}
    ref["temper_ffffffff"] = int(oracle_py.ref_lib().ref_temper(0xFFFFFFFF))
    # DC statuses of SURVEY.md Appendix B (reference dc_search outputs), words via the reference
    dc = {
        "dc521_id7": [7, 521, 17, 7, 23, 4049207303, 3676863948, 3740880118, 11, 7, 15, 18],
        "dc3217_id7": [7, 3217, 101, 9, 15, 3980328967, 882635769, 3305209961, 11, 7, 15, 18],
    }
    for name, st in dc.items():
        w = oracle_py.ref_fill(1 << 16, 4357, st)
        ref[name] = {"status12": st, "seed": 4357, "n": 1 << 16,
                     **{k: int(v) for k, v in oracle_py.cksum(w).items()}}
    (ROOT / "tests/golden/mt_reference.json").write_text(json.dumps(ref, indent=1) + "\n")
    print("goldens written")


if __name__ == "__main__":
    main()

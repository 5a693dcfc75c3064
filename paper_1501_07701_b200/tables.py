"""MTGP32 parameter-set tables (the "parameter-set table" of north_star).

Host-side table tooling for the generation path:

* ``load_curand_11213()`` imports the 200 certified MTGP32-11213 sets that ship with the CUDA
  toolkit (``curand_mtgp32dc_p_11213.h``, struct layout ``curand_mtgp32.h:140-152``). The sets
  are read from the toolkit at run time (or from a build-time import under ``data/``), never
  vendored into the repository.
* ``synthetic_sets(mexp, count)`` deterministically derives MTGP-shaped sets for exponents
  with no table on this machine (23209, 44497). Their period is
  UNCERTIFIED; throughput and bit-exactness against the CPU oracle do not depend on period.
* ``read_status_file`` / ``write_status_file`` extend the reference's parameter-set table file
  (JSON lines with canonical field order, or key=value lines with 0x hex;
  proj/src/status_io.cpp:15-141) with an ``"engine": "mtgp32"`` record type.
"""
from __future__ import annotations

import dataclasses
import json
import os
import re
from pathlib import Path
from typing import Iterable, List, Optional, Sequence

MASK32 = 0xFFFFFFFF
MTGP_MEXPS = (3217, 4253, 4423, 9689, 9941, 11213, 19937, 21701, 23209, 44497)
_DATA_DIR = Path(__file__).resolve().parent / "data"


def state_words(mexp: int) -> int:
    """N = floor(mexp/32) + 1."""
    return mexp // 32 + 1


def state_mask(mexp: int) -> int:
    r = 32 * state_words(mexp) - mexp
    return (MASK32 << r) & MASK32


@dataclasses.dataclass
class MtgpParams:
    """One MTGP32 parameter set (fields of mtgp32_params_fast, curand_mtgp32.h:140-152)."""

    mexp: int
    pos: int
    sh1: int
    sh2: int
    tbl: List[int]
    tmp_tbl: List[int]
    flt_tmp_tbl: List[int]
    mask: int
    id: int = 0
    poly_sha1: str = ""
    certified: bool = True

    @property
    def n(self) -> int:
        return state_words(self.mexp)

    def validate(self) -> None:
        """Mirror of mtgp_validate_params (and of ParameterizedStatus::validate's contract,
        proj/src/params.cpp:23-39): raises ValueError on a violated invariant."""
        if self.mexp not in MTGP_MEXPS:
            raise ValueError(f"unsupported period exponent {self.mexp}")
        if self.mask != state_mask(self.mexp):
            raise ValueError("mask must be 0xFFFFFFFF << (32N - mexp)")
        if not (1 <= self.sh1 <= 31 and 1 <= self.sh2 <= 31):
            raise ValueError("shifts must be in [1, 31]")
        if not (3 <= self.pos <= self.n - 32):
            raise ValueError("pick-up position must satisfy 3 <= pos <= N - 32")
        for i in range(16):
            t = m = 0
            for b in range(4):
                if i >> b & 1:
                    t ^= self.tbl[1 << b]
                    m ^= self.tmp_tbl[1 << b]
            if self.tbl[i] != t or self.tmp_tbl[i] != m:
                raise ValueError("tables must be GF(2)-linear in their index")
            if self.flt_tmp_tbl[i] != ((self.tmp_tbl[i] >> 9) | 0x3F800000):
                raise ValueError("flt_tmp_tbl must equal (tmp_tbl >> 9) | 0x3F800000")


# --------------------------------------------------------------------------------------------
# cuRAND 11213 table import
# --------------------------------------------------------------------------------------------

def _cuda_include_dirs() -> List[Path]:
    out = []
    for env in ("CUDA_HOME", "CUDA_PATH"):
        if os.environ.get(env):
            out.append(Path(os.environ[env]) / "include")
    out.append(Path("/usr/local/cuda/include"))
    return out


def parse_curand_header(text: str) -> List[MtgpParams]:
    """Parse the mtgp32_params_fast_t initializer list of curand_mtgp32dc_p_11213.h."""
    start = text.index("mtgp32dc_params_fast_11213[]")
    body = text[start:]
    sets: List[MtgpParams] = []
    for m in re.finditer(r"/\*\s*No\.(\d+)[^*]*\*/(.*?)\}\s*\}\s*,?\s*(?=\{\s*/\*|\};)", body, re.S):
        idx = int(m.group(1))
        nums = re.findall(r"0x[0-9a-fA-F]+|\b\d+\b", m.group(2))
        vals = [int(x, 0) for x in nums]
        # mexp, pos, sh1, sh2, 16 tbl, 16 tmp, 16 flt, mask, 21 sha1 bytes
        if len(vals) < 4 + 48 + 1 + 20:
            raise ValueError(f"short record {idx}")
        mexp, pos, sh1, sh2 = vals[0:4]
        tbl = vals[4:20]
        tmp = vals[20:36]
        flt = vals[36:52]
        mask = vals[52]
        sha = bytes(vals[53:73]).hex()
        sets.append(MtgpParams(mexp, pos, sh1, sh2, tbl, tmp, flt, mask, id=idx, poly_sha1=sha,
                               certified=True))
    if not sets:
        raise ValueError("no parameter sets found")
    return sets


def load_curand_11213(path: Optional[str] = None) -> List[MtgpParams]:
    """The 200 MTGP32-11213 sets of the CUDA toolkit (certified full period by their authors)."""
    if path is None:
        cached = _DATA_DIR / "mtgp32dc_11213.jsonl"
        if cached.exists():
            return [r for r in read_status_file(cached)]
        for d in _cuda_include_dirs():
            cand = d / "curand_mtgp32dc_p_11213.h"
            if cand.exists():
                path = str(cand)
                break
        if path is None:
            raise FileNotFoundError("curand_mtgp32dc_p_11213.h not found (set CUDA_HOME)")
    sets = parse_curand_header(Path(path).read_text())
    if len(sets) != 200:
        raise ValueError(f"expected 200 sets, parsed {len(sets)}")
    return sets


# --------------------------------------------------------------------------------------------
# synthetic (uncertified) sets
# --------------------------------------------------------------------------------------------

def _splitmix64(x: int) -> int:
    """proj/src/word_source.cpp:18-23."""
    x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
    return x ^ (x >> 31)


# Minimum safe width N - pos the v2 kernel wants per exponent (one warp team step).
TEAM_WORDS = {11213: 256, 23209: 512, 44497: 1024}


def synthetic_set(mexp: int, idx: int, family_seed: int = 0x4D544750) -> MtgpParams:
    """Deterministic MTGP-shaped set #idx for `mexp` (UNCERTIFIED period).

    pos in [3, N - team_words], sh1 in [1, 30], sh2 in [1, 19] (the ranges of the certified
    cuRAND sets), GF(2)-linear tbl / tmp_tbl from 4 random basis words each, flt derived.
    Randomness: splitmix64 counter (the reference's seed source, word_source.cpp:18-27).
    """
    n = state_words(mexp)
    team = TEAM_WORDS.get(mexp, 256)
    ctr = [(_splitmix64(family_seed) ^ (mexp << 32) ^ (idx * 0x100000001B3)) & 0xFFFFFFFFFFFFFFFF]

    def draw() -> int:
        ctr[0] = (ctr[0] + 1) & 0xFFFFFFFFFFFFFFFF
        return _splitmix64(ctr[0])

    pos_max = max(3, n - team)
    pos = 3 + draw() % (pos_max - 3 + 1)
    sh1 = 1 + draw() % 30
    sh2 = 1 + draw() % 19
    basis_t = [draw() & MASK32 for _ in range(4)]
    basis_m = [draw() & MASK32 for _ in range(4)]
    tbl, tmp = [], []
    for i in range(16):
        t = m = 0
        for b in range(4):
            if i >> b & 1:
                t ^= basis_t[b]
                m ^= basis_m[b]
        tbl.append(t)
        tmp.append(m)
    flt = [(v >> 9) | 0x3F800000 for v in tmp]
    return MtgpParams(mexp, pos, sh1, sh2, tbl, tmp, flt, state_mask(mexp), id=idx,
                      certified=False)


def synthetic_sets(mexp: int, count: int, first: int = 0) -> List[MtgpParams]:
    return [synthetic_set(mexp, first + i) for i in range(count)]


def curand_kernel_state_seeds(seed: int, n: int) -> List[int]:
    """Per-stream seeds of curandMakeMTGP32KernelState (curand_mtgp32_host.h:482-510): stream i
    is seeded with (u32)(seed ^ (seed >> 32)) + i + 1, so a context built with these seeds
    reproduces a cuRAND MTGP32 device-API setup stream for stream."""
    seed &= 0xFFFFFFFFFFFFFFFF
    base = (seed ^ (seed >> 32)) & 0xFFFFFFFF
    return [(base + i + 1) & 0xFFFFFFFF for i in range(n)]


def sets_for(mexp: int, count: int, first: int = 0) -> List[MtgpParams]:
    """`count` sets for `mexp`: the certified cuRAND sets first (11213), then synthetic ones."""
    out: List[MtgpParams] = []
    if mexp == 11213:
        cur = load_curand_11213()
        out = cur[first:first + count]
        first = max(0, first - len(cur))
        k = 0
        while len(out) < count:
            s = synthetic_set(mexp, 1000 + first + k)
            s.id = len(cur) + first + k
            out.append(s)
            k += 1
        return out
    return synthetic_sets(mexp, count, first)


# --------------------------------------------------------------------------------------------
# status-file IO (extends proj/src/status_io.cpp)
# --------------------------------------------------------------------------------------------

_FIELD_ORDER = ("id", "engine", "mexp", "pos", "sh1", "sh2", "mask", "tbl", "tmp_tbl",
                "flt_tmp_tbl", "poly_sha1", "certified")


def status_to_json_line(p: MtgpParams, seed: Optional[int] = None) -> str:
    """Canonical field order, like status_to_json_line (proj/src/status_io.cpp:77-98)."""
    d = {"id": p.id, "engine": "mtgp32", "mexp": p.mexp, "pos": p.pos, "sh1": p.sh1,
         "sh2": p.sh2, "mask": p.mask, "tbl": list(p.tbl), "tmp_tbl": list(p.tmp_tbl),
         "flt_tmp_tbl": list(p.flt_tmp_tbl), "poly_sha1": p.poly_sha1, "certified": p.certified}
    if seed is not None:
        d["seed"] = seed
    return json.dumps(d, separators=(",", ":"))


def _parse_int(v: str) -> int:
    return int(v, 0)


def status_from_line(line: str) -> MtgpParams:
    """JSON object or key=value tokens (0x hex accepted), then validate() --
    proj/src/status_io.cpp:46-75,100-113. Array fields in key=value form are comma separated."""
    s = line.strip()
    if s.startswith("{"):
        d = json.loads(s)
    else:
        d = {}
        for tok in s.split():
            if "=" not in tok:
                raise ValueError(f"expected key=value, got: {tok}")
            k, v = tok.split("=", 1)
            if k in ("tbl", "tmp_tbl", "flt_tmp_tbl"):
                d[k] = [_parse_int(x) for x in v.split(",")]
            elif k in ("poly_sha1", "engine"):
                d[k] = v
            elif k == "certified":
                d[k] = v.lower() in ("1", "true", "yes")
            elif k in ("id", "mexp", "pos", "sh1", "sh2", "mask", "seed"):
                d[k] = _parse_int(v)
            else:
                raise ValueError(f"unknown status field: {k}")
    if d.get("engine", "mtgp32") != "mtgp32":
        raise ValueError(f"not an mtgp32 status: engine={d.get('engine')}")
    mexp = int(d["mexp"])
    tmp = [int(x) for x in d["tmp_tbl"]]
    flt = [int(x) for x in d.get("flt_tmp_tbl", [(v >> 9) | 0x3F800000 for v in tmp])]
    p = MtgpParams(mexp=mexp, pos=int(d["pos"]), sh1=int(d["sh1"]), sh2=int(d["sh2"]),
                   tbl=[int(x) for x in d["tbl"]], tmp_tbl=tmp, flt_tmp_tbl=flt,
                   mask=int(d.get("mask", state_mask(mexp))), id=int(d.get("id", 0)),
                   poly_sha1=str(d.get("poly_sha1", "")),
                   certified=bool(d.get("certified", False)))
    p.validate()
    return p


def read_status_file(path) -> List[MtgpParams]:
    """Skips blank and '#' lines; errors carry path:line (proj/src/status_io.cpp:115-133)."""
    out = []
    with open(path) as f:
        for lineno, line in enumerate(f, 1):
            s = line.strip()
            if not s or s.startswith("#"):
                continue
            try:
                out.append(status_from_line(s))
            except Exception as e:  # noqa: BLE001 -- re-raised with location, like the reference
                raise RuntimeError(f"{path}:{lineno}: {e}") from e
    return out


def write_status_file(path, sets: Iterable[MtgpParams]) -> None:
    with open(path, "w") as f:
        for p in sets:
            f.write(status_to_json_line(p) + "\n")


def import_curand_table(dest: Optional[Path] = None) -> Path:
    """Build-time import of the toolkit table into data/mtgp32dc_11213.jsonl (git-ignored)."""
    dest = Path(dest) if dest else _DATA_DIR / "mtgp32dc_11213.jsonl"
    dest.parent.mkdir(parents=True, exist_ok=True)
    sets = None
    for d in _cuda_include_dirs():
        cand = d / "curand_mtgp32dc_p_11213.h"
        if cand.exists():
            sets = parse_curand_header(cand.read_text())
            break
    if sets is None:
        raise FileNotFoundError("curand_mtgp32dc_p_11213.h not found")
    write_status_file(dest, sets)
    return dest

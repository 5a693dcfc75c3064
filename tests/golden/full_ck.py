"""Lookup of the full-volume parity fixture (tests/golden/full_ck.npz, made by make_full_ck.py).

Checker infrastructure: used by the -m gpu tests and by bench.py after its timed region to
compare the GPU's fused per-stream checksums with the oracle's, for every word generated.
Reads only the committed .npz (no oracle code runs here).
"""
from __future__ import annotations

from pathlib import Path
from typing import Dict, Optional, Sequence, Tuple

import numpy as np

NPZ = Path(__file__).resolve().parent / "full_ck.npz"
# Engine::mt (bench.py --config mt19937): made by make_mt_full_ck.py from the reference itself
MT_NPZ = Path(__file__).resolve().parent / "mt_full_ck.npz"

# config -> (sum array key, xor array key, float index or None, words per record, set-ID offset)
_LAYOUT = {
    "c2": ("c2_sum", "c2_xor", None, 1 << 27),
    "c3-f12": ("c3_sum", "c3_xor", 0, 1 << 27),
    "c3-f01": ("c3_sum", "c3_xor", 1, 1 << 27),
    "c4-23209": ("c4_23209_sum", "c4_23209_xor", None, 1 << 27),
    "c4-44497": ("c4_44497_sum", "c4_44497_xor", None, 1 << 27),
    "c5": ("c5_sum", "c5_xor", None, 1 << 24),
    "mt19937": ("mt_sum", "mt_xor", None, 1 << 27),  # stream i = MT19937 seed 5489 + i
}
_cache: Dict[str, np.ndarray] = {}


def available(config: str = "c2") -> bool:
    return (MT_NPZ if config == "mt19937" else NPZ).exists()


def _arr(key: str) -> np.ndarray:
    if key not in _cache:
        for f in (NPZ, MT_NPZ):
            if f.exists():
                with np.load(f) as z:
                    for k in z.files:
                        _cache[k] = z[k]
    return _cache[key]


def coverage(config: str) -> Tuple[int, int, int]:
    """(streams, records, words per record) the fixture holds for `config`."""
    ks, _, _, rec = _LAYOUT[config]
    a = _arr(ks)
    return a.shape[0], a.shape[1], rec


def expected(config: str, first_set: int, n_sets: int, words: int) -> Optional[Tuple[np.ndarray, np.ndarray]]:
    """Oracle (sum64, xor32) of global streams [first_set, first_set + n_sets) after `words`
    words each, or None when the fixture does not reach that far."""
    if config not in _LAYOUT or not available(config):
        return None
    ks, kx, fi, rec = _LAYOUT[config]
    s, x = _arr(ks), _arr(kx)
    if words == 0 or words % rec or words // rec > s.shape[1] or first_set + n_sets > s.shape[0]:
        return None
    k = words // rec - 1
    sl = slice(first_set, first_set + n_sets)
    if fi is None:
        return s[sl, k].astype(np.uint64), x[sl, k].astype(np.uint32)
    return s[sl, k, fi].astype(np.uint64), x[sl, k, fi].astype(np.uint32)


def compare(config: str, first_set: int, cks: Sequence[Tuple[int, int, int]], sum_mod32: bool = False) -> dict:
    """Compare GPU checksums (sum64, xor32, words) of consecutive global streams starting at
    first_set with the fixture. sum_mod32: the GPU sums are valid mod 2^32 only
    (MTGP_OPT_CHECKSUM 2)."""
    words = {int(c[2]) for c in cks}
    if len(words) != 1:
        return {"ok": False, "reason": f"streams emitted different word counts {sorted(words)[:4]}"}
    w = words.pop()
    exp = expected(config, first_set, len(cks), w)
    if exp is None:
        return {"ok": None, "reason": f"fixture does not cover {config} streams {first_set}.."
                                      f"{first_set + len(cks) - 1} at {w} words", "words_per_stream": w}
    es, ex = exp
    gs = np.array([c[0] for c in cks], dtype=np.uint64)
    gx = np.array([c[1] for c in cks], dtype=np.uint32)
    if sum_mod32:
        es = es & np.uint64(0xFFFFFFFF)
        gs = gs & np.uint64(0xFFFFFFFF)
    bad = np.nonzero((es != gs) | (ex != gx))[0]
    return {"ok": bool(bad.size == 0), "streams": len(cks), "words_per_stream": w,
            "sum": "mod 2^32" if sum_mod32 else "mod 2^64", "mismatched_streams": [int(first_set + b) for b in bad[:8]],
            "n_mismatched": int(bad.size)}

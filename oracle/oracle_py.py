"""ctypes binding of liboracle.so and oracle/_ref/libtwistsieve_ref.so.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_LIB = HERE / "liboracle.so"
REF_LIB = HERE / "_ref" / "libtwistsieve_ref.so"


class OracleParams(C.Structure):
    _fields_ = [("mexp", C.c_uint32), ("pos", C.c_uint32), ("sh1", C.c_uint32), ("sh2", C.c_uint32),
                ("tbl", C.c_uint32 * 16), ("tmp_tbl", C.c_uint32 * 16),
                ("flt_tmp_tbl", C.c_uint32 * 16), ("mask", C.c_uint32)]


class OracleMtgp(C.Structure):
    _fields_ = [("p", OracleParams), ("n", C.c_uint32), ("idx", C.c_uint32), ("count", C.c_uint64),
                ("st", C.c_uint32 * 4096)]


class OracleCksum(C.Structure):
    _fields_ = [("sum64", C.c_uint64), ("xor32", C.c_uint32), ("last", C.c_uint32),
                ("poly31", C.c_uint32), ("pad", C.c_uint32)]


class OracleStreamCk(C.Structure):
    _fields_ = [("sum", C.c_uint64 * 3), ("xr", C.c_uint32 * 3), ("pad", C.c_uint32)]


class OracleMtParams(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("mexp", "n", "m", "r", "a", "b", "c", "u", "s", "t", "l")]


class OracleMt(C.Structure):
    _fields_ = [("p", OracleMtParams), ("index", C.c_uint32), ("st", C.c_uint32 * 2048)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not ORACLE_LIB.exists():
            raise ImportError(f"{ORACLE_LIB} not built (make -C oracle)")
        L = C.CDLL(str(ORACLE_LIB))
        L.oracle_mtgp_init.argtypes = [C.POINTER(OracleMtgp), C.POINTER(OracleParams), C.c_uint32]
        L.oracle_mtgp_fill.argtypes = [C.POINTER(OracleMtgp), C.c_void_p, C.c_size_t, C.c_int]
        L.oracle_mtgp_skip.argtypes = [C.POINTER(OracleMtgp), C.c_uint64]
        L.oracle_mtgp_window.argtypes = [C.POINTER(OracleMtgp), C.c_void_p]
        L.oracle_mtgp_from_window.argtypes = [C.POINTER(OracleMtgp), C.POINTER(OracleParams), C.c_void_p]
        L.oracle_cksum_words.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(OracleCksum)]
        L.oracle_mtgp_bulk.argtypes = [C.POINTER(OracleParams), C.POINTER(C.c_uint32), C.c_uint32,
                                       C.c_uint64, C.c_uint64, C.c_void_p, C.c_int, C.c_int]
        L.oracle_mtgp_bulk.restype = C.c_double
        L.oracle_mtgp_cksum_stream.argtypes = [C.POINTER(OracleParams), C.POINTER(C.c_uint32), C.c_uint32,
                                               C.c_uint64, C.c_uint32, C.c_int, C.c_void_p, C.c_int]
        L.oracle_mtgp_cksum_stream.restype = C.c_double
        L.oracle_mtgp_fill_bulk.argtypes = [C.POINTER(OracleParams), C.POINTER(C.c_uint32), C.c_uint32, C.c_uint64,
                                            C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_uint64)]
        L.oracle_mtgp_fill_bulk.restype = C.c_double
        L.oracle_mt19937_params.argtypes = [C.POINTER(OracleMtParams)]
        L.oracle_mt_init.argtypes = [C.POINTER(OracleMt), C.POINTER(OracleMtParams), C.c_uint32]
        L.oracle_mt_fill.argtypes = [C.POINTER(OracleMt), C.c_void_p, C.c_size_t]
        L.oracle_mt_temper.argtypes = [C.c_uint32, C.POINTER(OracleMtParams)]
        L.oracle_mt_temper.restype = C.c_uint32
        L.oracle_mt_untemper.argtypes = [C.c_uint32, C.POINTER(OracleMtParams)]
        L.oracle_mt_untemper.restype = C.c_uint32
        L.oracle_splitmix64.argtypes = [C.c_uint64]
        L.oracle_splitmix64.restype = C.c_uint64
        L.oracle_derive_seed.argtypes = [C.c_uint64, C.c_uint32]
        L.oracle_derive_seed.restype = C.c_uint32
        _lib = L
    return _lib


def to_oracle_params(p) -> OracleParams:
    o = OracleParams()
    o.mexp, o.pos, o.sh1, o.sh2, o.mask = p.mexp, p.pos, p.sh1, p.sh2, p.mask
    for j in range(16):
        o.tbl[j], o.tmp_tbl[j], o.flt_tmp_tbl[j] = p.tbl[j], p.tmp_tbl[j], p.flt_tmp_tbl[j]
    return o


class MtgpOracle:
    """Sequential MTGP32 stream on the CPU."""

    def __init__(self, params, seed: int):
        self.params = params
        self._p = to_oracle_params(params)
        self.g = OracleMtgp()
        if lib().oracle_mtgp_init(C.byref(self.g), C.byref(self._p), seed & 0xFFFFFFFF) != 0:
            raise ValueError("bad mexp")

    @classmethod
    def from_window(cls, params, window) -> "MtgpOracle":
        self = cls.__new__(cls)
        self.params = params
        self._p = to_oracle_params(params)
        self.g = OracleMtgp()
        w = np.ascontiguousarray(window, dtype=np.uint32)
        lib().oracle_mtgp_from_window(C.byref(self.g), C.byref(self._p), w.ctypes.data_as(C.c_void_p))
        return self

    def fill(self, n: int, kind: int = 0) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        lib().oracle_mtgp_fill(C.byref(self.g), out.ctypes.data_as(C.c_void_p), n, kind)
        return out

    def skip(self, n: int) -> None:
        lib().oracle_mtgp_skip(C.byref(self.g), n)

    def window(self) -> np.ndarray:
        out = np.empty(self.g.n, dtype=np.uint32)
        lib().oracle_mtgp_window(C.byref(self.g), out.ctypes.data_as(C.c_void_p))
        return out


def mtgp_bulk(sets: Sequence, seeds: Sequence[int], n: int, skip: int = 0, kind: int = 0,
              threads: int = 8, out: Optional[np.ndarray] = None):
    """(n_sets, n) words of every stream from position `skip`; returns (array, seconds)."""
    arr = (OracleParams * len(sets))(*[to_oracle_params(p) for p in sets])
    sd = (C.c_uint32 * len(seeds))(*[s & 0xFFFFFFFF for s in seeds])
    if out is None:
        out = np.empty((len(sets), n), dtype=np.uint32)
    secs = lib().oracle_mtgp_bulk(arr, sd, len(sets), skip, n, out.ctypes.data_as(C.c_void_p), kind, threads)
    return out, secs


CK_DTYPE = np.dtype([("sum", "<u8", (3,)), ("xr", "<u4", (3,)), ("pad", "<u4")])


def cksum_stream(sets: Sequence, seeds: Sequence[int], rec_every: int, n_rec: int, with_float: bool = False,
                 threads: int = 8, scalar: bool = False):
    """Cumulative per-stream checksums without an output buffer: result[s, k] holds the
    {sum64, xor32} of the first (k+1)*rec_every words of stream s as fields sum[3] / xr[3]
    (0 = u32, 1 = f32 [1,2) bits, 2 = f32 (0,1] bits). Returns (array, seconds)."""
    arr = (OracleParams * len(sets))(*[to_oracle_params(p) for p in sets])
    sd = (C.c_uint32 * len(seeds))(*[s & 0xFFFFFFFF for s in seeds])
    out = np.zeros((len(sets), n_rec), dtype=CK_DTYPE)
    assert C.sizeof(OracleStreamCk) == CK_DTYPE.itemsize
    secs = lib().oracle_mtgp_cksum_stream(arr, sd, len(sets), rec_every, n_rec, int(with_float) | (2 if scalar else 0),
                                          out.ctypes.data_as(C.c_void_p), threads)
    return out, secs


def fill_bulk(sets: Sequence, seeds: Sequence[int], n: int, chunk: int = 1 << 20, kind: int = 0,
              threads: int = 8) -> float:
    """CPU baseline: every stream's first n words through a reused chunk-word fill buffer per
    thread (WordSource::fill semantics); returns seconds."""
    arr = (OracleParams * len(sets))(*[to_oracle_params(p) for p in sets])
    sd = (C.c_uint32 * len(seeds))(*[s & 0xFFFFFFFF for s in seeds])
    sink = C.c_uint64()
    return lib().oracle_mtgp_fill_bulk(arr, sd, len(sets), n, chunk, kind, threads, C.byref(sink))


def cksum(words: np.ndarray):
    c = OracleCksum()
    w = np.ascontiguousarray(words, dtype=np.uint32)
    lib().oracle_cksum_words(w.ctypes.data_as(C.c_void_p), w.size, C.byref(c))
    return {"sum64": c.sum64, "xor32": c.xor32, "last": c.last, "poly31": c.poly31}


def mt19937_params() -> OracleMtParams:
    p = OracleMtParams()
    lib().oracle_mt19937_params(C.byref(p))
    return p


class MtOracle:
    """The reference's Engine::mt restated (proj/src/generator.cpp)."""

    def __init__(self, params: Optional[OracleMtParams], seed: int):
        self.p = params if params is not None else mt19937_params()
        self.g = OracleMt()
        if lib().oracle_mt_init(C.byref(self.g), C.byref(self.p), seed & 0xFFFFFFFF) != 0:
            raise ValueError("bad MT parameters")

    def fill(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint32)
        lib().oracle_mt_fill(C.byref(self.g), out.ctypes.data_as(C.c_void_p), n)
        return out


# ---- the unmodified reference, compiled from its own sources (oracle/Makefile) ----
_ref = None


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_LIB.exists():
            raise ImportError(f"{REF_LIB} not built (make -C oracle ref; needs /root/reference)")
        L = C.CDLL(str(REF_LIB))
        L.ref_fill.argtypes = [C.c_void_p, C.c_uint32, C.c_void_p, C.c_uint64]
        L.ref_temper.argtypes = [C.c_uint32]
        L.ref_temper.restype = C.c_uint32
        L.ref_untemper.argtypes = [C.c_uint32]
        L.ref_untemper.restype = C.c_uint32
        L.ref_validate.argtypes = [C.c_void_p]
        L.ref_bulk_throughput.argtypes = [C.c_int, C.c_uint64, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint64)]
        L.ref_bulk_throughput.restype = C.c_double
        L.ref_cksum_stream.argtypes = [C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint32, C.c_void_p, C.c_void_p, C.c_int]
        L.ref_cksum_stream.restype = C.c_double
        _ref = L
    return _ref


def ref_fill(n: int, seed: int, status12: Optional[Sequence[int]] = None) -> np.ndarray:
    out = np.empty(n, dtype=np.uint32)
    st = None
    if status12 is not None:
        st = (C.c_uint32 * 12)(*status12)
    rc = ref_lib().ref_fill(st, seed & 0xFFFFFFFF, out.ctypes.data_as(C.c_void_p), n)
    if rc != 0:
        raise ValueError("reference rejected the status")
    return out


def ref_bulk_throughput(threads: int, words_per_thread: int, fill_words: int = 1 << 18, seed0: int = 5489):
    x = C.c_uint64()
    secs = ref_lib().ref_bulk_throughput(threads, words_per_thread, fill_words, seed0, C.byref(x))
    return secs, x.value


def ref_cksum_stream(seed0: int, n_streams: int, rec_every: int, n_rec: int, threads: int = 8):
    """Cumulative (sum64, xor32) of MT19937 streams seed0 + s through the reference's own
    make_word_source + fill (oracle/_ref); arrays [n_streams, n_rec], seconds."""
    sums = np.zeros((n_streams, n_rec), dtype=np.uint64)
    xors = np.zeros((n_streams, n_rec), dtype=np.uint32)
    secs = ref_lib().ref_cksum_stream(seed0, n_streams, rec_every, n_rec, sums.ctypes.data_as(C.c_void_p),
                                      xors.ctypes.data_as(C.c_void_p), threads)
    if secs < 0:
        raise ValueError("rec_every must be a multiple of 2^18")
    return sums, xors, secs

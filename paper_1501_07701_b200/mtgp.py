"""ctypes binding of the C-ABI in include/mtgp_b200.h (libmtgp_b200.so).

This is plumbing for tests and bench.py: every call goes straight into the CUDA library. There
is no CPU fallback -- if the library or a device is missing, construction raises.

Mirrors the reference's generation API shape (proj/include/twistsieve/word_source.hpp:21-25,
75-76; generator.hpp:23-52): a context is "n_sets WordSources at once"; ``fill_u32(L)`` is L
successive ``WordSource::fill`` words of every stream.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path
from typing import Optional, Sequence

import numpy as np

from .tables import MtgpParams, state_words

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "libmtgp_b200.so"

MTGP_OK, MTGP_EINVAL, MTGP_ECUDA, MTGP_ENOMEM, MTGP_ESTATE = 0, 1, 2, 3, 4
U32, F32_12, F32_01OC, F64_01 = 0, 1, 2, 3
OPT_CHECKSUM, OPT_KERNEL, OPT_MAX_PIECES, OPT_MIN_PIECE_WORDS, OPT_TIMING, OPT_HOST_CHUNK, OPT_JUMP = 1, 2, 3, 4, 5, 6, 7
OPT_PREJUMP = 8  # speculative next-call jumps: 0 auto, 1 off, 2 always

# Every symbol include/mtgp_b200.h declares (checked by the CPU test suite).
EXPORTS = (
    "mtgp_abi_version", "mtgp_last_error", "mtgp_validate_params", "mtgp_ctx_create",
    "mtgp_ctx_destroy", "mtgp_ctx_info", "mtgp_position", "mtgp_ctx_stream", "mtgp_set_option",
    "mtgp_generate", "mtgp_generate_u32", "mtgp_generate_f32_12", "mtgp_generate_f32_01oc",
    "mtgp_skip", "mtgp_state_save", "mtgp_state_restore", "mtgp_checksums",
    "mtgp_checksums_reset", "mtgp_sync", "mtgp_kernel_timing", "mtgp_kernel_timing_reset",
    "mtgp_last_plan", "mtgp_launch_count", "mtgp_mt_validate_params", "mtgp_mt_ctx_create",
    "mtgp_charpoly_sha1", "mtgp_stat_validate", "mtgp_stat_run", "mtgp_stat_counts_len", "mtgp_stat_finish",
    "mtgp_ln_gamma", "mtgp_gamma_p", "mtgp_gamma_q", "mtgp_chi_square_pvalue", "mtgp_poisson_cdf",
    "mtgp_poisson_sf", "mtgp_poisson_pmf", "mtgp_binomial_log_pmf", "mtgp_binomial_upper_tail",
    "mtgp_classify_pvalue", "mtgp_certify", "mtgp_mt_charpoly_digest", "mtgp_gf2_is_irreducible",
    "mtgp_host_alloc", "mtgp_host_free", "mtgp_generate_async",
    "mtgp_shard_range", "mtgp_multi_create", "mtgp_multi_destroy", "mtgp_multi_info", "mtgp_multi_context",
    "mtgp_multi_generate", "mtgp_multi_checksums",
)


class MtParamsC(C.Structure):
    """Engine::mt status (ParameterizedStatus recurrence fields, proj/include/twistsieve/params.hpp:21-42)."""
    _fields_ = [(k, C.c_uint32) for k in ("id", "mexp", "n", "m", "r", "a", "temper_b", "temper_c", "temper_u",
                                          "temper_s", "temper_t", "temper_l")]


def mt19937_status() -> dict:
    """proj/src/params.cpp:63-77."""
    return dict(id=0xB0DF, mexp=19937, n=624, m=397, r=31, a=0x9908B0DF, temper_b=0x9D2C5680,
                temper_c=0xEFC60000, temper_u=11, temper_s=7, temper_t=15, temper_l=18)


class MtgpParamsC(C.Structure):
    _fields_ = [("mexp", C.c_uint32), ("pos", C.c_uint32), ("sh1", C.c_uint32), ("sh2", C.c_uint32),
                ("tbl", C.c_uint32 * 16), ("tmp_tbl", C.c_uint32 * 16),
                ("flt_tmp_tbl", C.c_uint32 * 16), ("mask", C.c_uint32)]


class MtgpCksumC(C.Structure):
    _fields_ = [("sum64", C.c_uint64), ("words", C.c_uint64), ("xor32", C.c_uint32), ("pad", C.c_uint32)]


class StatSpecC(C.Structure):
    """mtgp_stat_spec: TestSpec (proj/include/twistsieve/stat_tests.hpp:18-33) with an int test id."""
    _fields_ = [("test", C.c_int32), ("N", C.c_uint32), ("n", C.c_uint64), ("r", C.c_uint32), ("s", C.c_uint32),
                ("L", C.c_uint32), ("d", C.c_uint32), ("l", C.c_uint32), ("t", C.c_uint32),
                ("alpha", C.c_double), ("beta", C.c_double)]


class StatResultC(C.Structure):
    """mtgp_stat_result: TestResult (stat_tests.hpp:35-42) + error code + words consumed."""
    _fields_ = [("statistic", C.c_double), ("p_value", C.c_double), ("classification", C.c_int32),
                ("degenerate", C.c_int32), ("error", C.c_int32), ("pad", C.c_int32), ("words_used", C.c_uint64)]


class MtgpError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class MtgpInvalidArgument(MtgpError, ValueError):
    """What the reference raises as std::invalid_argument (proj/src/params.cpp:23-39)."""


_lib = None


def load_library(path: Optional[str] = None) -> C.CDLL:
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise ImportError(f"{p} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = C.CDLL(str(p))
    lib.mtgp_last_error.restype = C.c_char_p
    lib.mtgp_ctx_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.POINTER(MtgpParamsC), C.c_uint32,
                                    C.POINTER(C.c_uint32), C.c_void_p]
    lib.mtgp_ctx_destroy.argtypes = [C.c_void_p]
    lib.mtgp_ctx_info.argtypes = [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    lib.mtgp_position.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_uint64)]
    lib.mtgp_ctx_stream.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    lib.mtgp_set_option.argtypes = [C.c_void_p, C.c_int, C.c_int64]
    lib.mtgp_generate.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_int]
    lib.mtgp_generate_async.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_int]
    lib.mtgp_host_alloc.argtypes = [C.c_size_t, C.POINTER(C.c_void_p)]
    lib.mtgp_host_free.argtypes = [C.c_void_p]
    lib.mtgp_skip.argtypes = [C.c_void_p, C.c_uint64]
    lib.mtgp_state_save.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.mtgp_state_restore.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    lib.mtgp_checksums.argtypes = [C.c_void_p, C.POINTER(MtgpCksumC)]
    lib.mtgp_checksums_reset.argtypes = [C.c_void_p]
    lib.mtgp_sync.argtypes = [C.c_void_p]
    lib.mtgp_kernel_timing.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_double), C.POINTER(C.c_uint64)]
    lib.mtgp_kernel_timing_reset.argtypes = [C.c_void_p]
    lib.mtgp_last_plan.argtypes = [C.c_void_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32)]
    lib.mtgp_validate_params.argtypes = [C.POINTER(MtgpParamsC)]
    lib.mtgp_launch_count.argtypes = [C.c_void_p, C.POINTER(C.c_uint64)]
    lib.mtgp_mt_validate_params.argtypes = [C.POINTER(MtParamsC)]
    lib.mtgp_charpoly_sha1.argtypes = [C.c_void_p, C.c_char_p]
    lib.mtgp_mt_ctx_create.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.POINTER(MtParamsC), C.c_uint32,
                                       C.POINTER(C.c_uint32), C.c_void_p]
    lib.mtgp_stat_validate.argtypes = [C.POINTER(StatSpecC)]
    lib.mtgp_stat_run.argtypes = [C.c_void_p, C.POINTER(StatSpecC), C.POINTER(StatResultC)]
    lib.mtgp_stat_counts_len.argtypes = [C.POINTER(StatSpecC), C.POINTER(C.c_uint64)]
    lib.mtgp_stat_finish.argtypes = [C.POINTER(StatSpecC), C.POINTER(C.c_uint64), C.c_uint64, C.POINTER(StatResultC)]
    pd = C.POINTER(C.c_double)
    lib.mtgp_ln_gamma.argtypes = [C.c_double, pd]
    lib.mtgp_gamma_p.argtypes = [C.c_double, C.c_double, pd]
    lib.mtgp_gamma_q.argtypes = [C.c_double, C.c_double, pd]
    lib.mtgp_chi_square_pvalue.argtypes = [C.c_double, C.c_uint32, pd]
    lib.mtgp_poisson_cdf.argtypes = [C.c_uint64, C.c_double, pd]
    lib.mtgp_poisson_sf.argtypes = [C.c_uint64, C.c_double, pd]
    lib.mtgp_poisson_pmf.argtypes = [C.c_uint64, C.c_double, pd]
    lib.mtgp_binomial_log_pmf.argtypes = [C.c_uint64, C.c_uint64, C.c_double, pd]
    lib.mtgp_binomial_upper_tail.argtypes = [C.c_uint64, C.c_uint64, C.c_double, pd]
    lib.mtgp_classify_pvalue.argtypes = [C.c_double, C.POINTER(C.c_int32)]
    lib.mtgp_certify.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
    lib.mtgp_mt_charpoly_digest.argtypes = [C.c_void_p, C.c_char_p]
    lib.mtgp_gf2_is_irreducible.argtypes = [C.c_void_p, C.c_uint64, C.POINTER(C.c_int32)]
    pu = C.POINTER(C.c_uint32)
    lib.mtgp_shard_range.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, pu, pu]
    lib.mtgp_multi_create.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_int), C.c_uint32, C.POINTER(MtgpParamsC),
                                      C.c_uint32, pu, C.c_int]
    lib.mtgp_multi_destroy.argtypes = [C.c_void_p]
    lib.mtgp_multi_info.argtypes = [C.c_void_p, pu, C.POINTER(C.c_int)]
    lib.mtgp_multi_context.argtypes = [C.c_void_p, C.c_uint32, C.POINTER(C.c_void_p), pu, pu]
    lib.mtgp_multi_generate.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p), C.c_uint64]
    lib.mtgp_multi_checksums.argtypes = [C.c_void_p, C.POINTER(MtgpCksumC)]
    if path is None:
        _lib = lib
    return lib


def _check(lib, rc: int) -> None:
    if rc != MTGP_OK:
        msg = lib.mtgp_last_error().decode()
        if rc == MTGP_EINVAL:
            raise MtgpInvalidArgument(rc, msg)
        raise MtgpError(rc, msg)


def to_c_params(sets: Sequence[MtgpParams]):
    arr = (MtgpParamsC * len(sets))()
    for i, p in enumerate(sets):
        a = arr[i]
        a.mexp, a.pos, a.sh1, a.sh2, a.mask = p.mexp, p.pos, p.sh1, p.sh2, p.mask
        for j in range(16):
            a.tbl[j] = p.tbl[j]
            a.tmp_tbl[j] = p.tmp_tbl[j]
            a.flt_tmp_tbl[j] = p.flt_tmp_tbl[j]
    return arr


def validate(p: MtgpParams) -> None:
    lib = load_library()
    arr = to_c_params([p])
    _check(lib, lib.mtgp_validate_params(arr))


def shard_range(n_sets: int, world: int, rank: int):
    """mtgp_shard_range: the contiguous balanced set-ID range of `rank`."""
    lib = load_library()
    f, c = C.c_uint32(), C.c_uint32()
    _check(lib, lib.mtgp_shard_range(n_sets, world, rank, C.byref(f), C.byref(c)))
    return range(f.value, f.value + c.value)


class MultiGpu:
    """mtgp_multi: n_sets streams split over `devices` (one context and host thread per device),
    checksums all-gathered over NCCL (gather 0 auto / 1 NCCL / 2 host)."""

    def __init__(self, sets: Sequence[MtgpParams], seeds: Sequence[int], devices: Sequence[int], gather: int = 0,
                 lib: Optional[C.CDLL] = None):
        self.lib = lib if lib is not None else load_library()
        self.n_sets = len(sets)
        self._params = to_c_params(sets)
        self._seeds = (C.c_uint32 * len(seeds))(*[int(s) & 0xFFFFFFFF for s in seeds])
        self._devs = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _check(self.lib, self.lib.mtgp_multi_create(C.byref(h), self._devs, len(devices), self._params, self.n_sets,
                                                    self._seeds, gather))
        self.h = h
        n, nccl = C.c_uint32(), C.c_int()
        _check(self.lib, self.lib.mtgp_multi_info(self.h, C.byref(n), C.byref(nccl)))
        self.n_devices, self.nccl = n.value, bool(nccl.value)

    def ranges(self):
        out = []
        for r in range(self.n_devices):
            ctx, f, c = C.c_void_p(), C.c_uint32(), C.c_uint32()
            _check(self.lib, self.lib.mtgp_multi_context(self.h, r, C.byref(ctx), C.byref(f), C.byref(c)))
            out.append(range(f.value, f.value + c.value))
        return out

    def generate_device(self, kind: int, ptrs: Sequence[int], words_per_stream: int) -> None:
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        _check(self.lib, self.lib.mtgp_multi_generate(self.h, kind, arr, words_per_stream))

    def checksums(self):
        arr = (MtgpCksumC * self.n_sets)()
        _check(self.lib, self.lib.mtgp_multi_checksums(self.h, arr))
        return [(a.sum64, a.xor32, a.words) for a in arr]

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.mtgp_multi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class MtgpContext:
    """n_sets independent MTGP32 streams on one GPU (C-ABI mtgp_ctx)."""

    def __init__(self, sets: Sequence[MtgpParams], seeds: Sequence[int], device: int = 0,
                 stream: Optional[int] = None, lib: Optional[C.CDLL] = None):
        self.lib = lib if lib is not None else load_library()
        if len(seeds) != len(sets):
            raise ValueError("one seed per parameter set")
        self.sets = list(sets)
        self.n_sets = len(sets)
        self.N = state_words(sets[0].mexp)
        self._params = to_c_params(sets)
        self._seeds = (C.c_uint32 * len(seeds))(*[int(s) & 0xFFFFFFFF for s in seeds])
        h = C.c_void_p()
        _check(self.lib, self.lib.mtgp_ctx_create(C.byref(h), device, self._params, self.n_sets,
                                                  self._seeds, C.c_void_p(stream or 0)))
        self.h = h

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.mtgp_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- options / info
    def set_option(self, opt: int, value: int) -> None:
        _check(self.lib, self.lib.mtgp_set_option(self.h, opt, int(value)))

    def stream_handle(self) -> int:
        s = C.c_void_p()
        _check(self.lib, self.lib.mtgp_ctx_stream(self.h, C.byref(s)))
        return s.value or 0

    def position(self, s: int = 0) -> int:
        v = C.c_uint64()
        _check(self.lib, self.lib.mtgp_position(self.h, s, C.byref(v)))
        return v.value

    def last_plan(self):
        a, b, c = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(self.lib, self.lib.mtgp_last_plan(self.h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    # -- generation
    def generate_device(self, kind: int, ptr: int, words_per_stream: int) -> None:
        """Asynchronous generation into device memory at `ptr` (int address)."""
        _check(self.lib, self.lib.mtgp_generate(self.h, kind, C.c_void_p(ptr), words_per_stream, 1))

    def generate_host(self, kind: int, words_per_stream: int, out: Optional[np.ndarray] = None) -> np.ndarray:
        """Synchronous generation into host memory; returns an (n_sets, L) array (uint32 bit
        patterns for the u32/f32 kinds, float64 for F64_01)."""
        dt = np.float64 if kind == F64_01 else np.uint32
        if out is None:
            out = np.empty((self.n_sets, words_per_stream), dtype=dt)
        assert out.dtype == dt and out.flags.c_contiguous and out.size == self.n_sets * words_per_stream
        _check(self.lib, self.lib.mtgp_generate(self.h, kind, out.ctypes.data_as(C.c_void_p),
                                                words_per_stream, 0))
        return out

    def generate_host_async(self, kind: int, out: np.ndarray) -> None:
        """mtgp_generate_async into host memory `out` (n_sets, L): valid after sync(). Keep `out`
        alive (and preferably page-locked) until then."""
        dt = np.float64 if kind == F64_01 else (np.float32 if kind in (F32_12, F32_01OC) else np.uint32)
        # the call writes 8 bytes per sample for F64_01 and 4 otherwise: the dtype sizes the buffer
        assert np.dtype(out.dtype).itemsize == np.dtype(dt).itemsize, f"out dtype {out.dtype} for kind {kind}"
        assert out.flags.c_contiguous and out.size % self.n_sets == 0
        _check(self.lib, self.lib.mtgp_generate_async(self.h, kind, out.ctypes.data_as(C.c_void_p),
                                                      out.size // self.n_sets, 0))

    def fill_u32(self, L: int) -> np.ndarray:
        return self.generate_host(U32, L)

    def skip(self, words: int) -> None:
        _check(self.lib, self.lib.mtgp_skip(self.h, words))

    def sync(self) -> None:
        _check(self.lib, self.lib.mtgp_sync(self.h))

    # -- state
    def state_save(self):
        win = np.empty((self.n_sets, self.N), dtype=np.uint32)
        pos = np.empty(self.n_sets, dtype=np.uint64)
        _check(self.lib, self.lib.mtgp_state_save(self.h, win.ctypes.data_as(C.c_void_p),
                                                  pos.ctypes.data_as(C.c_void_p)))
        return win, pos

    def state_restore(self, win: np.ndarray, pos: Optional[np.ndarray] = None) -> None:
        win = np.ascontiguousarray(win, dtype=np.uint32)
        assert win.size == self.n_sets * self.N
        pp = None
        if pos is not None:
            pos = np.ascontiguousarray(pos, dtype=np.uint64)
            pp = pos.ctypes.data_as(C.c_void_p)
        _check(self.lib, self.lib.mtgp_state_restore(self.h, win.ctypes.data_as(C.c_void_p), pp))

    def checksums(self):
        arr = (MtgpCksumC * self.n_sets)()
        _check(self.lib, self.lib.mtgp_checksums(self.h, arr))
        return [(a.sum64, a.xor32, a.words) for a in arr]

    def checksums_reset(self) -> None:
        _check(self.lib, self.lib.mtgp_checksums_reset(self.h))

    def kernel_timing(self):
        g, gl, j, jl = C.c_double(), C.c_uint64(), C.c_double(), C.c_uint64()
        _check(self.lib, self.lib.mtgp_kernel_timing(self.h, C.byref(g), C.byref(gl), C.byref(j), C.byref(jl)))
        return g.value, gl.value, j.value, jl.value

    def charpoly_sha1(self):
        """SHA-1 of each stream's minimal polynomial ('0'/'1' coefficients, lowest degree first)."""
        buf = C.create_string_buffer(41 * self.n_sets)
        _check(self.lib, self.lib.mtgp_charpoly_sha1(self.h, buf))
        raw = buf.raw
        return [raw[41 * s:41 * s + 40].split(b"\0")[0].decode() for s in range(self.n_sets)]

    def launch_count(self) -> int:
        v = C.c_uint64()
        _check(self.lib, self.lib.mtgp_launch_count(self.h, C.byref(v)))
        return v.value

    def kernel_timing_reset(self) -> None:
        _check(self.lib, self.lib.mtgp_kernel_timing_reset(self.h))

    def certify(self) -> list:
        """Per stream: True iff its minimal polynomial has degree mexp and is irreducible (the
        reference dynamic creator's acceptance test, dynamic_creator.cpp:79-81)."""
        arr = (C.c_int32 * self.n_sets)()
        _check(self.lib, self.lib.mtgp_certify(self.h, arr))
        return [bool(v) for v in arr]

    def mt_charpoly_digest(self) -> list:
        """Engine::mt contexts: the reference's poly_digest of each stream's probed minimal
        polynomial (verify_digest's digest when seeded with 1)."""
        buf = C.create_string_buffer(41 * self.n_sets)
        _check(self.lib, self.lib.mtgp_mt_charpoly_digest(self.h, buf))
        raw = buf.raw
        return [raw[41 * s:41 * s + 40].split(b"\0")[0].decode() for s in range(self.n_sets)]

    def stat_run(self, spec) -> list:
        """The device-side statistical test `spec` (stattests.TestSpec) on every stream, from the
        current position; the context state is unchanged. One stattests.TestResult per stream."""
        from . import stattests
        return stattests.run_on_context(self, spec)


def mt_validate(status: dict) -> None:
    lib = load_library()
    _check(lib, lib.mtgp_mt_validate_params(C.byref(MtParamsC(**status))))


class MtContext(MtgpContext):
    """n_sets Engine::mt streams (the reference's own recurrence) on one GPU."""

    def __init__(self, statuses: Sequence[dict], seeds: Sequence[int], device: int = 0,
                 stream: Optional[int] = None, lib: Optional[C.CDLL] = None):
        self.lib = lib if lib is not None else load_library()
        if len(seeds) != len(statuses):
            raise ValueError("one seed per status")
        self.sets = list(statuses)
        self.n_sets = len(statuses)
        self.N = max(s["n"] for s in statuses)
        self._params = (MtParamsC * self.n_sets)(*[MtParamsC(**s) for s in statuses])
        self._seeds = (C.c_uint32 * self.n_sets)(*[int(s) & 0xFFFFFFFF for s in seeds])
        h = C.c_void_p()
        _check(self.lib, self.lib.mtgp_mt_ctx_create(C.byref(h), device, self._params, self.n_sets, self._seeds,
                                                     C.c_void_p(stream or 0)))
        self.h = h


def gf2_is_irreducible(coeffs) -> bool:
    """Rabin irreducibility of sum_i coeffs[i] x^i (host, PCLMUL; csrc/gf2.cpp)."""
    lib = load_library()
    b = np.ascontiguousarray(np.asarray(coeffs, dtype=np.uint8))
    out = C.c_int32()
    _check(lib, lib.mtgp_gf2_is_irreducible(b.ctypes.data_as(C.c_void_p), b.size, C.byref(out)))
    return bool(out.value)

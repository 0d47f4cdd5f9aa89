"""ctypes binding of libct_tune.so (include/countertune_tune.h): the live
measurement path -- NVRTC variant compiler + launcher and CUPTI range-profiler
collector.

This is the in-process replacement of the reference's out-of-process runner
(``SubprocessMeasurementSource``, search.py:220-275): instead of writing
``v1,...,vk,flag`` to a child and parsing ``runtime_us,threads,NAME=val``,
a :class:`Tuner` compiles the configuration's variant for this GPU, times it
with CUDA events and (for profiled steps) collects the Table-1 counter set with
CUPTI.  :mod:`.live` builds the reference's ``MeasurementSource`` duck type on
top of it.

As with ``_native``, importing fails loudly if the library is not built, and
every call without a CUDA device raises ``CounterTuneError``.
"""

import ctypes
import os
import threading
from typing import Optional, Sequence, Tuple

import numpy as np

from .errors import CounterTuneError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libct_tune.so")

CT_TUNE_OK = 0
CT_TUNE_ERR_CUDA = -1
CT_TUNE_ERR_VALUE = -2
CT_TUNE_ERR_COMPILE = -3
CT_TUNE_ERR_LAUNCH = -4
CT_TUNE_ERR_PROFILER = -5

_i32 = ctypes.c_int32
_i64 = ctypes.c_int64
_u64 = ctypes.c_uint64
_vp = ctypes.c_void_p
_cp = ctypes.c_char_p
_P = ctypes.POINTER


class LaunchC(ctypes.Structure):
    """ct_launch"""
    _fields_ = [
        ("grid", ctypes.c_uint32 * 3),
        ("block", ctypes.c_uint32 * 3),
        ("dynamic_smem", ctypes.c_uint32),
        ("args", _vp),
        ("arg_offsets", _P(_i32)),
        ("n_args", _i32),
    ]


SIGNATURES = {
    "ct_tune_abi_version": (ctypes.c_int, []),
    "ct_tune_last_error": (_cp, []),
    "ct_tuner_create": (ctypes.c_int, [ctypes.c_int, _P(_vp)]),
    "ct_tuner_destroy": (ctypes.c_int, [_vp]),
    "ct_tuner_device_info": (ctypes.c_int, [_vp, _cp, _i32, _P(_i32), _P(_i32)]),
    "ct_tuner_compile": (ctypes.c_int, [_vp, _cp, _cp, _P(_cp), _i32, _P(_i32), _cp, _i64]),
    "ct_tuner_compile_batch": (ctypes.c_int, [_vp, _cp, _cp, _P(_cp), _P(_i32), _i32, _i32,
                                              _P(_i32), _P(_i32)]),
    "ct_tuner_variant_info": (ctypes.c_int, [_vp, _i32, _P(_i32), _P(_i32), _P(_i32)]),
    "ct_tuner_unload": (ctypes.c_int, [_vp, _i32]),
    "ct_tuner_alloc": (ctypes.c_int, [_vp, _i64, _P(_u64)]),
    "ct_tuner_free": (ctypes.c_int, [_vp, _u64]),
    "ct_tuner_h2d": (ctypes.c_int, [_vp, _u64, _vp, _i64]),
    "ct_tuner_d2h": (ctypes.c_int, [_vp, _vp, _u64, _i64]),
    "ct_tuner_memset": (ctypes.c_int, [_vp, _u64, _i32, _i64]),
    "ct_tuner_time": (ctypes.c_int, [_vp, _i32, _P(LaunchC), _i32, _i32, _i32,
                                     _P(ctypes.c_double)]),
    "ct_tuner_profile": (ctypes.c_int, [_vp, _i32, _P(LaunchC), _P(_cp), _i32,
                                        _P(ctypes.c_double), _P(_i32)]),
    "ct_tuner_profile_passes": (ctypes.c_int, [_vp, _P(_cp), _i32, _P(_i32)]),
    "ct_tuner_profile_batch": (ctypes.c_int, [_vp, _i32, _P(_i32), _P(LaunchC), _P(_cp), _i32,
                                              _P(ctypes.c_double), _P(_i32)]),
    "ct_tuner_profile_timing": (ctypes.c_int, [_vp, _P(ctypes.c_double), _i32]),
    "ct_tuner_tensor_map_2d": (ctypes.c_int, [_vp, _u64, _u64, _u64, _u64, ctypes.c_uint32,
                                              ctypes.c_uint32, _vp]),
}

_lib = None
_lock = threading.Lock()


def library(path: str = LIB_PATH):
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise ImportError(f"{path} is not built: run __graft_entry__.build()")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class CompileError(CounterTuneError):
    """NVRTC rejected a variant (the configuration is invalid on this device)."""


class LaunchError(CounterTuneError):
    """The variant failed to launch (invalid configuration) or faulted."""


def _check(code: int) -> None:
    if code == CT_TUNE_OK:
        return
    msg = library().ct_tune_last_error().decode(errors="replace")
    if code == CT_TUNE_ERR_VALUE:
        raise ValueError(msg)
    if code == CT_TUNE_ERR_COMPILE:
        raise CompileError(msg)
    if code == CT_TUNE_ERR_LAUNCH:
        raise LaunchError(msg)
    raise CounterTuneError(msg)


def _cstrings(items: Sequence[str]):
    arr = (_cp * max(1, len(items)))()
    for i, s in enumerate(items):
        arr[i] = s.encode()
    return arr


class Launch:
    """Grid/block geometry plus kernel arguments packed as cuLaunchKernel
    expects (one naturally aligned slot per argument)."""

    def __init__(self, grid, block, args: Sequence[ctypes._SimpleCData], dynamic_smem: int = 0):
        g = tuple(grid) + (1,) * (3 - len(grid))
        b = tuple(block) + (1,) * (3 - len(block))
        offsets, off = [], 0
        for a in args:
            sz = ctypes.sizeof(a)
            al = ctypes.alignment(a)          # arrays / structs: element alignment
            off = (off + al - 1) // al * al
            offsets.append(off)
            off += sz
        self._blob = ctypes.create_string_buffer(max(off, 8))
        for a, o in zip(args, offsets):
            ctypes.memmove(ctypes.addressof(self._blob) + o, ctypes.addressof(a), ctypes.sizeof(a))
        self._offsets = (_i32 * max(1, len(offsets)))(*offsets)
        self.c = LaunchC((ctypes.c_uint32 * 3)(*g), (ctypes.c_uint32 * 3)(*b),
                         int(dynamic_smem), ctypes.cast(self._blob, _vp), self._offsets,
                         len(offsets))
        self.grid, self.block = g, b

    @property
    def threads(self) -> int:
        return int(np.prod(self.grid) * np.prod(self.block))


class Tuner:
    """One GPU's variant compiler, launcher, timer and counter collector."""

    def __init__(self, device: int = 0):
        self._lib = library()
        h = _vp()
        _check(self._lib.ct_tuner_create(int(device), ctypes.byref(h)))
        self._h = h
        self.device = int(device)
        arch = ctypes.create_string_buffer(32)
        sms, mt = _i32(), _i32()
        _check(self._lib.ct_tuner_device_info(self._h, arch, 32, ctypes.byref(sms),
                                              ctypes.byref(mt)))
        self.arch = arch.value.decode()
        self.sm_count = sms.value
        self.max_threads_per_sm = mt.value

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.ct_tuner_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- variants -------------------------------------------------------------
    def compile(self, source: str, kernel: str, options: Sequence[str] = ()) -> int:
        v = _i32()
        log = ctypes.create_string_buffer(1)
        _check(self._lib.ct_tuner_compile(self._h, source.encode(), kernel.encode(),
                                          _cstrings(options), len(options), ctypes.byref(v),
                                          log, 0))
        return v.value

    def compile_batch(self, source: str, kernel: str, options: Sequence[Sequence[str]],
                      threads: int = 0) -> Tuple[np.ndarray, np.ndarray]:
        """Compile many variants of one source concurrently on host threads.

        Returns (variant handle or -1, status) per option list; a variant NVRTC
        rejects gets status CT_TUNE_ERR_COMPILE and handle -1.
        """
        flat, counts = [], []
        for opts in options:
            flat.extend(opts)
            counts.append(len(opts))
        n = len(counts)
        c_counts = (_i32 * max(1, n))(*counts)
        out = np.full(n, -1, dtype=np.int32)
        status = np.zeros(n, dtype=np.int32)
        _check(self._lib.ct_tuner_compile_batch(
            self._h, source.encode(), kernel.encode(), _cstrings(flat), c_counts, n,
            int(threads), out.ctypes.data_as(_P(_i32)), status.ctypes.data_as(_P(_i32))))
        return out, status

    def variant_info(self, variant: int) -> Tuple[int, int, int]:
        r, s, m = _i32(), _i32(), _i32()
        _check(self._lib.ct_tuner_variant_info(self._h, int(variant), ctypes.byref(r),
                                               ctypes.byref(s), ctypes.byref(m)))
        return r.value, s.value, m.value

    def unload(self, variant: int) -> None:
        _check(self._lib.ct_tuner_unload(self._h, int(variant)))

    # -- memory ---------------------------------------------------------------
    def alloc(self, nbytes: int) -> int:
        p = _u64()
        _check(self._lib.ct_tuner_alloc(self._h, int(nbytes), ctypes.byref(p)))
        return p.value

    def free(self, ptr: int) -> None:
        _check(self._lib.ct_tuner_free(self._h, int(ptr)))

    def upload(self, arr: np.ndarray) -> int:
        arr = np.ascontiguousarray(arr)
        p = self.alloc(arr.nbytes)
        _check(self._lib.ct_tuner_h2d(self._h, p, arr.ctypes.data, arr.nbytes))
        return p

    def h2d(self, ptr: int, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr)
        _check(self._lib.ct_tuner_h2d(self._h, int(ptr), arr.ctypes.data, arr.nbytes))

    def d2h(self, ptr: int, out: np.ndarray) -> np.ndarray:
        assert out.flags.c_contiguous
        _check(self._lib.ct_tuner_d2h(self._h, out.ctypes.data, int(ptr), out.nbytes))
        return out

    def memset(self, ptr: int, value: int, nbytes: int) -> None:
        _check(self._lib.ct_tuner_memset(self._h, int(ptr), int(value), int(nbytes)))

    # -- measurement ----------------------------------------------------------
    def time(self, variant: int, launch: Launch, warmup: int = 1, reps: int = 3,
             flush_l2: bool = True) -> np.ndarray:
        out = np.zeros(max(reps, 1), dtype=np.float64)
        _check(self._lib.ct_tuner_time(self._h, int(variant), ctypes.byref(launch.c),
                                       int(warmup), int(reps), int(bool(flush_l2)),
                                       out.ctypes.data_as(_P(ctypes.c_double))))
        return out[:reps]

    def profile(self, variant: int, launch: Launch,
                metrics: Sequence[str]) -> Tuple[np.ndarray, int]:
        vals = np.zeros(len(metrics), dtype=np.float64)
        passes = _i32()
        _check(self._lib.ct_tuner_profile(self._h, int(variant), ctypes.byref(launch.c),
                                          _cstrings(metrics), len(metrics),
                                          vals.ctypes.data_as(_P(ctypes.c_double)),
                                          ctypes.byref(passes)))
        return vals, passes.value

    def profile_batch(self, variants: Sequence[int], launches: Sequence[Launch],
                      metrics: Sequence[str]) -> Tuple[np.ndarray, int]:
        """ct_tuner_profile_batch: one collection over k launches, one range
        each -> (k x len(metrics) values, replay passes)."""
        k = len(variants)
        vals = np.zeros((k, len(metrics)), dtype=np.float64)
        vs = (_i32 * k)(*[int(v) for v in variants])
        ls = (LaunchC * k)(*[l.c for l in launches])
        passes = _i32()
        _check(self._lib.ct_tuner_profile_batch(self._h, k, vs, ls, _cstrings(metrics),
                                                len(metrics),
                                                vals.ctypes.data_as(_P(ctypes.c_double)),
                                                ctypes.byref(passes)))
        return vals, passes.value

    def tensor_map_2d(self, ptr: int, dim0: int, dim1: int, row_stride_bytes: int, box0: int,
                      box1: int):
        """128-byte fp32 TMA descriptor (ct_tuner_tensor_map_2d), as a kernel
        argument (ctypes array of 16 uint64)."""
        out = (ctypes.c_uint64 * 16)()
        _check(self._lib.ct_tuner_tensor_map_2d(self._h, int(ptr), int(dim0), int(dim1),
                                                int(row_stride_bytes), int(box0), int(box1),
                                                ctypes.cast(out, _vp)))
        return out

    PROFILE_PHASES = ("setconfig_us", "passes_us", "sync_us", "decode_us", "evaluate_us",
                      "calls", "replay_passes", "host_config_us")

    def profile_timing(self, reset: bool = False) -> dict:
        """Accumulated wall time of profile() by phase (ct_tuner_profile_timing)."""
        out = np.zeros(8, dtype=np.float64)
        _check(self._lib.ct_tuner_profile_timing(self._h, out.ctypes.data_as(_P(ctypes.c_double)),
                                                 int(bool(reset))))
        return dict(zip(self.PROFILE_PHASES, out.tolist()))

    def profile_passes(self, metrics: Sequence[str]) -> int:
        p = _i32()
        _check(self._lib.ct_tuner_profile_passes(self._h, _cstrings(metrics), len(metrics),
                                                 ctypes.byref(p)))
        return p.value

"""ctypes boundary to the sm_100a library (include/tritperm.h).

This module is the B200 replacement of the reference's ``tritperm._kernels``
(src/_kernels.py): the same dispatcher names and argument meaning
(``chunk_sum``, ``mc_zero_count``, ``mc_sample_entries``), backed by
``lib/libtritperm_b200.so`` instead of numba.  There is no CPU fallback: if
the library or a B200 is missing every call raises.

The library is loaded lazily so the package imports on a CPU-only host (the
export table can then still be inspected); compute calls need a GPU.
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# TRITPERM_LIB: another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("TRITPERM_LIB") or os.path.join(_HERE, "lib", "libtritperm_b200.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "tritperm.h")

TP_OK = 0
TP_E_INVALID = -1
TP_E_CUDA = -2
TP_E_NODEV = -3

ENV_DEVICE = "TRITPERM_DEVICE"

_lib = None
_lock = threading.Lock()

_u64p = ctypes.POINTER(ctypes.c_uint64)
_i64p = ctypes.POINTER(ctypes.c_int64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i8p = ctypes.POINTER(ctypes.c_int8)
_ip = ctypes.POINTER(ctypes.c_int)

# name -> (restype, argtypes); mirrors include/tritperm.h
SIGNATURES = {
    "tp_version": (ctypes.c_int, []),
    "tp_last_error": (ctypes.c_char_p, []),
    "tp_device_count": (ctypes.c_int, [_ip]),
    "tp_device_info": (ctypes.c_int, [ctypes.c_int, _ip, _ip, _ip, _ip]),
    "tp_range_sum": (ctypes.c_int, [_u64p, _u64p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                    _u64p, _u64p]),
    "tp_range_sum_ex": (ctypes.c_int, [_u64p, _u64p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int,
                                       ctypes.c_int, _u64p, _u64p]),
    "tp_range_sum_nccl": (ctypes.c_int, [_u64p, _u64p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, _ip,
                                         ctypes.c_int, _u64p, _u64p]),
    "tp_range_sum_async": (ctypes.c_int, [_u64p, _u64p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]),
    "tp_range_sum_multi": (ctypes.c_int, [_u64p, _u64p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64, _ip,
                                          ctypes.c_int, _u64p, _u64p]),
    "tp_perm_batch": (ctypes.c_int, [_u8p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _i8p, _i64p, _i64p]),
    "tp_perm_batch_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                           ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _ip]),
    "tp_mc_zero_count": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                        ctypes.c_int, _i64p, _i64p]),
    "tp_mc_classes": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int,
                                     _i8p]),
    "tp_sample_classes": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64,
                                         ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]),
    "tp_mc_sample_entries": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_int, _i8p]),
    "tp_selftest_ops": (ctypes.c_int, [_u32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, _u32p]),
    "tp_pack_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p]),
    "tp_walk_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                     ctypes.c_void_p, _ip]),
    "tp_walk_range_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, _ip]),
    "tp_finalize_async": (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]),
    "tp_debug_trace": (ctypes.c_int, [ctypes.c_void_p]),
    "tp_walk_info": (ctypes.c_int, [ctypes.c_int, ctypes.c_longlong, ctypes.c_char_p, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_double)]),
    "tp_exact_census": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, _i64p, _i64p, _i64p]),
    "tp_alu_peak": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "tp_walk_tested": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_uint64)]),
}

ROWREC_BYTES = 2048  # TP_ROWREC_BYTES: packed row records per matrix


class TritpermError(RuntimeError):
    """CUDA-side failure reported by the library."""


def lib():
    """The loaded library (raises if it has not been built)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise RuntimeError(
                        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                        "or `make -C paper_2407_20205_b200/csrc` (there is no CPU fallback)")
                L = ctypes.CDLL(LIB_PATH)
                for name, (res, args) in SIGNATURES.items():
                    if os.environ.get("TRITPERM_LIB") and not hasattr(L, name):
                        continue  # an older build under A/B timing may lack newer entry points
                    fn = getattr(L, name)
                    fn.restype = res
                    fn.argtypes = args
                _lib = L
    return _lib


def _check(rc: int) -> None:
    if rc == TP_OK:
        return
    msg = lib().tp_last_error().decode(errors="replace")
    if rc == TP_E_INVALID:
        raise ValueError(msg)
    raise TritpermError(f"tritperm (code {rc}): {msg}")


def default_device() -> int:
    env = os.environ.get(ENV_DEVICE)
    if env is not None:
        return int(env)
    lr = os.environ.get("LOCAL_RANK")
    return int(lr) if lr is not None else 0


def device_count() -> int:
    c = ctypes.c_int(0)
    rc = lib().tp_device_count(ctypes.byref(c))
    if rc != TP_OK:
        return 0
    return int(c.value)


def device_info(device: Optional[int] = None) -> dict:
    dev = default_device() if device is None else device
    sm, clk, ma, mi = (ctypes.c_int() for _ in range(4))
    _check(lib().tp_device_info(dev, ctypes.byref(sm), ctypes.byref(clk), ctypes.byref(ma), ctypes.byref(mi)))
    return {"device": dev, "sm_count": sm.value, "max_clock_khz": clk.value, "cc": (ma.value, mi.value)}


def _planes(mags, sgns, n: int) -> Tuple[np.ndarray, np.ndarray]:
    mags = np.ascontiguousarray(mags, dtype=np.uint64)
    sgns = np.ascontiguousarray(sgns, dtype=np.uint64)
    if mags.shape != (n,) or sgns.shape != (n,):
        raise ValueError(f"planes must have shape ({n},)")
    return mags, sgns


def _check_bounds(n: int, lo: int, hi: int) -> None:
    """Range bounds in Python ints, before any uint64 conversion (ctypes would
    silently wrap 2**64 to 0)."""
    if not 1 <= n <= 64:
        raise ValueError(f"need 1 <= n <= 64, got n={n}")
    if not 0 <= lo <= hi <= (1 << n):
        raise ValueError(f"need 0 <= lo <= hi <= 2**n, got lo={lo} hi={hi} n={n}")


def chunk_counts(mags, sgns, n: int, lo: int, hi: int, device: Optional[int] = None) -> Tuple[int, int]:
    """(plus, minus) term counts over Gray steps [lo, hi); n <= 64 (the end
    2**64 of a 64-row walk goes through tp_range_sum_ex's carry flag)."""
    _check_bounds(n, lo, hi)
    mags, sgns = _planes(mags, sgns, n)
    dev = default_device() if device is None else device
    p = ctypes.c_uint64()
    m = ctypes.c_uint64()
    if n == 64:
        end64 = hi == 1 << 64
        _check(lib().tp_range_sum_ex(mags.ctypes.data_as(_u64p), sgns.ctypes.data_as(_u64p), n, lo,
                                     0 if end64 else hi, 1 if end64 else 0, dev, ctypes.byref(p), ctypes.byref(m)))
    else:
        _check(lib().tp_range_sum(mags.ctypes.data_as(_u64p), sgns.ctypes.data_as(_u64p), n, lo, hi, dev,
                                  ctypes.byref(p), ctypes.byref(m)))
    return int(p.value), int(m.value)


def chunk_sum(mags, sgns, n: int, lo: int, hi: int) -> int:
    """Drop-in for the reference's ``_kernels.chunk_sum`` (src/_kernels.py:90-128)."""
    p, m = chunk_counts(mags, sgns, n, lo, hi)
    return p - m


def chunk_counts_multi(mags, sgns, n: int, lo: int, hi: int, devices, nccl: bool = True) -> Tuple[int, int]:
    """(plus, minus) over [lo, hi) split across `devices` (one process).

    nccl=True: the per-device counters meet in one ncclAllReduce inside the
    library (tp_range_sum_nccl); False: summed on the host
    (tp_range_sum_multi)."""
    _check_bounds(n, lo, hi)
    if n > 63:
        raise ValueError("the multi-device range API needs n <= 63")
    mags, sgns = _planes(mags, sgns, n)
    devs = (ctypes.c_int * len(devices))(*devices)
    p = ctypes.c_uint64()
    m = ctypes.c_uint64()
    fn = lib().tp_range_sum_nccl if nccl else lib().tp_range_sum_multi
    _check(fn(mags.ctypes.data_as(_u64p), sgns.ctypes.data_as(_u64p), n, lo, hi, devs, len(devices),
              ctypes.byref(p), ctypes.byref(m)))
    return int(p.value), int(m.value)


def chunk_counts_async(mags, sgns, n: int, lo: int, hi: int, d_pm_ptr: int, stream_ptr: int,
                       device: Optional[int] = None) -> None:
    """Add (plus, minus) of [lo, hi) into the device buffer d_pm_ptr (uint64[2])."""
    mags, sgns = _planes(mags, sgns, n)
    dev = default_device() if device is None else device
    _check(lib().tp_range_sum_async(mags.ctypes.data_as(_u64p), sgns.ctypes.data_as(_u64p), n, lo, hi, dev,
                                    ctypes.c_void_p(d_pm_ptr), ctypes.c_void_p(stream_ptr)))


def perm_batch(entries: np.ndarray, device: Optional[int] = None, partials: bool = True):
    """uint8 [B, n, n] host batch -> (classes int8[B] in {0,1,2}, partials int64[B] or None, hist int64[3])."""
    e = np.ascontiguousarray(entries, dtype=np.uint8)
    if e.ndim != 3 or e.shape[1] != e.shape[2]:
        raise ValueError("entries must have shape [B, n, n]")
    B, n, _ = e.shape
    dev = default_device() if device is None else device
    cls = np.zeros(B, dtype=np.int8)
    part = np.zeros(B, dtype=np.int64) if (partials and n <= 62) else None
    hist = np.zeros(3, dtype=np.int64)
    _check(lib().tp_perm_batch(e.ctypes.data_as(_u8p), B, n, dev, cls.ctypes.data_as(_i8p),
                               part.ctypes.data_as(_i64p) if part is not None else None,
                               hist.ctypes.data_as(_i64p)))
    return cls, part, hist


def perm_batch_async(d_entries_ptr: int, B: int, n: int, d_class_ptr: int, d_pm_ptr: int, d_hist_ptr: int,
                     stream_ptr: int, device: Optional[int] = None) -> int:
    """Device-pointer batch (asynchronous); returns the number of kernel launches."""
    dev = default_device() if device is None else device
    nl = ctypes.c_int(0)
    _check(lib().tp_perm_batch_async(ctypes.c_void_p(d_entries_ptr), B, n, dev, ctypes.c_void_p(d_class_ptr),
                                     ctypes.c_void_p(d_pm_ptr), ctypes.c_void_p(d_hist_ptr),
                                     ctypes.c_void_p(stream_ptr), ctypes.byref(nl)))
    return int(nl.value)


def pack_async(d_entries_ptr: int, B: int, n: int, d_rows_ptr: int, stream_ptr: int,
               device: Optional[int] = None) -> None:
    dev = default_device() if device is None else device
    _check(lib().tp_pack_async(ctypes.c_void_p(d_entries_ptr), B, n, dev, ctypes.c_void_p(d_rows_ptr),
                               ctypes.c_void_p(stream_ptr)))


def walk_async(d_rows_ptr: int, B: int, n: int, d_pm_ptr: int, stream_ptr: int, device: Optional[int] = None) -> int:
    dev = default_device() if device is None else device
    nl = ctypes.c_int(0)
    _check(lib().tp_walk_async(ctypes.c_void_p(d_rows_ptr), B, n, dev, ctypes.c_void_p(d_pm_ptr),
                               ctypes.c_void_p(stream_ptr), ctypes.byref(nl)))
    return int(nl.value)


def walk_range_async(d_rows_ptr: int, n: int, lo: int, hi: int, d_pm_ptr: int, stream_ptr: int,
                     device: Optional[int] = None) -> int:
    """Range walk of one device-packed matrix; returns the kernel launches."""
    dev = default_device() if device is None else device
    nl = ctypes.c_int(0)
    _check(lib().tp_walk_range_async(ctypes.c_void_p(d_rows_ptr), n, lo, hi, dev, ctypes.c_void_p(d_pm_ptr),
                                     ctypes.c_void_p(stream_ptr), ctypes.byref(nl)))
    return int(nl.value)


def finalize_async(d_pm_ptr: int, B: int, n: int, d_class_ptr: int, d_hist_ptr: int, stream_ptr: int,
                   device: Optional[int] = None) -> None:
    dev = default_device() if device is None else device
    _check(lib().tp_finalize_async(ctypes.c_void_p(d_pm_ptr), B, n, dev, ctypes.c_void_p(d_class_ptr),
                                   ctypes.c_void_p(d_hist_ptr), ctypes.c_void_p(stream_ptr)))


def walk_info(n: int, batch: int = 1) -> Tuple[str, float]:
    """(kernel description, LOP3 per subset term) for full traversals of
    `batch` matrices of size n."""
    buf = ctypes.create_string_buffer(128)
    ops = ctypes.c_double()
    _check(lib().tp_walk_info(n, batch, buf, 128, ctypes.byref(ops)))
    return buf.value.decode(), float(ops.value)


def walk_tested(device: Optional[int] = None) -> int:
    """Pairs tested by the bucketed walk since the last call (read and reset)."""
    dev = default_device() if device is None else device
    v = ctypes.c_uint64(0)
    _check(lib().tp_walk_tested(dev, ctypes.byref(v)))
    return int(v.value)


def alu_peak(device: Optional[int] = None) -> Tuple[float, float]:
    """(measured LOP3 ops/s, probe duration ms) of the device."""
    dev = default_device() if device is None else device
    ops = ctypes.c_double()
    ms = ctypes.c_double()
    _check(lib().tp_alu_peak(dev, ctypes.byref(ops), ctypes.byref(ms)))
    return float(ops.value), float(ms.value)


def exact_census(n: int) -> Tuple[int, int, int]:
    """(zeros, plus_ones, minus_ones) of perm mod 3 over all n x n matrices."""
    z, p, m = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(lib().tp_exact_census(n, default_device(), ctypes.byref(z), ctypes.byref(p), ctypes.byref(m)))
    return int(z.value), int(p.value), int(m.value)


def mc_zero_count(n: int, t0: int, t1: int, seed: int) -> int:
    """Drop-in for the reference's ``_kernels.mc_zero_count`` (src/_kernels.py:245-255)."""
    z = ctypes.c_int64()
    _check(lib().tp_mc_zero_count(n, t0, t1, int(seed) & ((1 << 64) - 1), default_device(), ctypes.byref(z), None))
    return int(z.value)


def mc_hist(n: int, t0: int, t1: int, seed: int) -> np.ndarray:
    """Per-class counts (class 0, 1, 2) of trials [t0, t1)."""
    z = ctypes.c_int64()
    h = np.zeros(3, dtype=np.int64)
    _check(lib().tp_mc_zero_count(n, t0, t1, int(seed) & ((1 << 64) - 1), default_device(), ctypes.byref(z),
                                  h.ctypes.data_as(_i64p)))
    return h


def mc_classes(n: int, t0: int, count: int, seed: int) -> np.ndarray:
    out = np.zeros(count, dtype=np.int8)
    _check(lib().tp_mc_classes(n, t0, count, int(seed) & ((1 << 64) - 1), default_device(),
                               out.ctypes.data_as(_i8p)))
    return out


def sample_classes(n: int, t0: int, count: int, seed: int) -> np.ndarray:
    """uint8 [count, n, n] classes of trials [t0, t0+count), sampled on the device."""
    out = np.zeros((count, n, n), dtype=np.uint8)
    _check(lib().tp_sample_classes(n, t0, count, int(seed) & ((1 << 64) - 1), default_device(),
                                   ctypes.c_void_p(out.ctypes.data), 0, None))
    return out


def sample_classes_device(n: int, t0: int, count: int, seed: int, d_out_ptr: int, stream_ptr: int) -> None:
    _check(lib().tp_sample_classes(n, t0, count, int(seed) & ((1 << 64) - 1), default_device(),
                                   ctypes.c_void_p(d_out_ptr), 1, ctypes.c_void_p(stream_ptr)))


def mc_sample_entries(n: int, trial: int, seed: int) -> np.ndarray:
    """Drop-in for the reference's ``_kernels.mc_sample_entries`` (src/_kernels.py:258-272)."""
    out = np.zeros(n * n, dtype=np.int8)
    _check(lib().tp_mc_sample_entries(n, trial, int(seed) & ((1 << 64) - 1), default_device(),
                                      out.ctypes.data_as(_i8p)))
    return out


def selftest_ops(words: np.ndarray, op: int) -> np.ndarray:
    """words uint32 [k, 4] (mag1, sgn1, mag2, sgn2) -> uint32 [k, 2] via the device primitives."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    out = np.zeros((w.shape[0], 2), dtype=np.uint32)
    _check(lib().tp_selftest_ops(w.ctypes.data_as(_u32p), w.shape[0], op, default_device(),
                                 out.ctypes.data_as(_u32p)))
    return out

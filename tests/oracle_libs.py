"""ctypes loaders for the CHECKERS under oracle/ (test infrastructure only).

- ``oracle()``  -> oracle/libktune_oracle.so, the plain-C restatement of the
  reference executors (oracle/ktune_oracle.c); always available once built.
- ``reference()`` -> oracle/_ref/libktune_ref.so, the unmodified reference
  library compiled from /root/reference (oracle/Makefile); None when it was
  not built (e.g. on a box where /root/reference never existed and the
  prebuilt .so did not travel).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "libktune_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libktune_ref.so")

c_i64 = ctypes.c_int64
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_dp = ctypes.POINTER(ctypes.c_double)
c_fp = ctypes.POINTER(ctypes.c_float)


def _ptr(a: np.ndarray, typ):
    return a.ctypes.data_as(typ)


@lru_cache(None)
def oracle():
    if not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-C", ORACLE_DIR, "oracle"], check=True,
                       stdout=subprocess.DEVNULL)
    lib = ctypes.CDLL(ORACLE_SO)
    for name, T in (("f32", c_fp), ("f64", c_dp)):
        f = getattr(lib, f"oracle_execute_gemm_{name}")
        f.argtypes = [c_i64, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_i32p, T, T, T]
        f = getattr(lib, f"oracle_execute_conv_{name}")
        f.argtypes = [c_i64p, c_i32p, T, T, T]
        f = getattr(lib, f"oracle_naive_gemm_{name}")
        f.argtypes = [c_i64, c_i64, c_i64, ctypes.c_int, ctypes.c_int, T, T, c_dp]
        f = getattr(lib, f"oracle_direct_conv_{name}")
        f.argtypes = [c_i64p, T, T, c_dp]
        f = getattr(lib, f"oracle_fill_{name}")
        f.argtypes = [ctypes.c_uint64, ctypes.c_int, T, c_i64, T, c_i64]
    lib.oracle_indirection_table.argtypes = [c_i64p, c_i64p]
    return lib


@lru_cache(None)
def reference():
    if not os.path.exists(REF_SO):
        return None
    lib = ctypes.CDLL(REF_SO)
    lib.ref_last_error.restype = ctypes.c_char_p
    lib.ref_last_text.restype = ctypes.c_char_p
    return lib


def _np_t(dtype):
    return (np.float32, c_fp) if dtype == "f32" else (np.float64, c_dp)


# --------------------------------------------------------------------------
# Oracle helpers (numpy in, numpy out)
# --------------------------------------------------------------------------

def fill(seed: int, na: int, nb: int, dtype="f32", symmetric=False):
    """Operands exactly as CpuBackend::measure fills them (backends.cpp:508-513)
    or, with symmetric=True, as the reference tests do (test_backends.cpp:68-71)."""
    npt, ct = _np_t(dtype)
    a = np.empty(na, npt)
    b = np.empty(nb, npt)
    getattr(oracle(), f"oracle_fill_{dtype}")(seed, int(symmetric), _ptr(a, ct), na, _ptr(b, ct), nb)
    return a, b


def execute_gemm(m, n, k, ta, tb, tuning, a, b, dtype="f32"):
    npt, ct = _np_t(dtype)
    c = np.empty(m * n, npt)
    tv = np.asarray(tuning, np.int32)
    getattr(oracle(), f"oracle_execute_gemm_{dtype}")(
        m, n, k, int(ta), int(tb), _ptr(tv, c_i32p), _ptr(np.ascontiguousarray(a, npt), ct),
        _ptr(np.ascontiguousarray(b, npt), ct), _ptr(c, ct))
    return c


def naive_gemm(m, n, k, ta, tb, a, b, dtype="f32"):
    npt, ct = _np_t(dtype)
    c = np.empty(m * n, np.float64)
    getattr(oracle(), f"oracle_naive_gemm_{dtype}")(
        m, n, k, int(ta), int(tb), _ptr(np.ascontiguousarray(a, npt), ct),
        _ptr(np.ascontiguousarray(b, npt), ct), _ptr(c, c_dp))
    return c


def conv_sizes(dims):
    n, p, q, k, c, r, s = dims
    return c * (p + r - 1) * (q + s - 1) * n, c * r * s * k, k * p * q * n


def execute_conv(dims, tuning, img, flt, dtype="f32"):
    npt, ct = _np_t(dtype)
    out = np.empty(conv_sizes(dims)[2], npt)
    d = np.asarray(dims, np.int64)
    tv = np.asarray(tuning, np.int32)
    getattr(oracle(), f"oracle_execute_conv_{dtype}")(
        _ptr(d, c_i64p), _ptr(tv, c_i32p), _ptr(np.ascontiguousarray(img, npt), ct),
        _ptr(np.ascontiguousarray(flt, npt), ct), _ptr(out, ct))
    return out


def direct_conv(dims, img, flt, dtype="f32"):
    npt, ct = _np_t(dtype)
    out = np.empty(conv_sizes(dims)[2], np.float64)
    d = np.asarray(dims, np.int64)
    getattr(oracle(), f"oracle_direct_conv_{dtype}")(
        _ptr(d, c_i64p), _ptr(np.ascontiguousarray(img, npt), ct),
        _ptr(np.ascontiguousarray(flt, npt), ct), _ptr(out, c_dp))
    return out


def indirection_table(dims):
    n, p, q, k, c, r, s = dims
    out = np.empty((c * r * s, 4), np.int64)
    d = np.asarray(dims, np.int64)
    oracle().oracle_indirection_table(_ptr(d, c_i64p), _ptr(out, c_i64p))
    return out


def max_rel_error(got, ref) -> float:
    """test_backends.cpp:74-82: max |got - ref| / max(|ref|, 1)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if got.size == 0:
        return 0.0
    return float(np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)))


# --------------------------------------------------------------------------
# Reference-library helpers (only where oracle/_ref was built)
# --------------------------------------------------------------------------

def ref_call(fn, *args):
    rc = fn(*args)
    if rc != 0:
        raise RuntimeError(f"reference error {rc}: {reference().ref_last_error().decode()}")


def ref_execute_gemm(m, n, k, ta, tb, tuning, a, b, dtype="f32"):
    lib = reference()
    npt, ct = _np_t(dtype)
    c = np.empty(m * n, npt)
    tv = np.asarray(tuning, np.int32)
    fn = getattr(lib, f"ref_execute_gemm_{dtype}")
    fn.argtypes = [c_i64, c_i64, c_i64, ctypes.c_int, ctypes.c_int, c_i32p, ct, ct, ct]
    ref_call(fn, m, n, k, int(ta), int(tb), _ptr(tv, c_i32p), _ptr(np.ascontiguousarray(a, npt), ct),
             _ptr(np.ascontiguousarray(b, npt), ct), _ptr(c, ct))
    return c


def ref_execute_conv(dims, tuning, img, flt, dtype="f32"):
    lib = reference()
    npt, ct = _np_t(dtype)
    out = np.empty(conv_sizes(dims)[2], npt)
    d = np.asarray(dims, np.int64)
    tv = np.asarray(tuning, np.int32)
    fn = getattr(lib, f"ref_execute_conv_{dtype}")
    fn.argtypes = [c_i64p, c_i32p, ct, ct, ct]
    ref_call(fn, _ptr(d, c_i64p), _ptr(tv, c_i32p), _ptr(np.ascontiguousarray(img, npt), ct),
             _ptr(np.ascontiguousarray(flt, npt), ct), _ptr(out, ct))
    return out

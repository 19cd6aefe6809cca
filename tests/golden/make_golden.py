"""Generates tests/golden/*.json from the UNMODIFIED reference library.

Run here (where /root/reference exists) after `make -C oracle`:

    python tests/golden/make_golden.py

The fixtures pin both the oracle restatement (oracle/ktune_oracle.c) and the
product's host code on boxes where the reference itself is absent (the GPU
box).  Every value below is produced by a call into oracle/_ref/
libktune_ref.so (ref_shim.cpp -> ktune::*), never by our own code.
"""
from __future__ import annotations

import ctypes
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_libs as O  # noqa: E402

REF = "/root/reference/proj"
ROOT = os.path.dirname(os.path.dirname(HERE))
B200_HW = open(os.path.join(ROOT, "paper_1802_05371_b200", "fixtures", "hw", "b200.json")).read()
B200_GEMM_BOUNDS = open(os.path.join(ROOT, "paper_1802_05371_b200", "fixtures", "bounds", "gemm_b200.json")).read()
B200_CONV_BOUNDS = open(os.path.join(ROOT, "paper_1802_05371_b200", "fixtures", "bounds", "conv_b200.json")).read()
CONV_SMALL = open(os.path.join(REF, "fixtures", "bounds", "conv_small.json")).read()
SYNTH_HW = open(os.path.join(REF, "fixtures", "hw", "synthetic.json")).read()
DT = {"f16": 0, "f32": 1, "f64": 2}

c_i64 = ctypes.c_int64


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def lib():
    L = O.reference()
    if L is None:
        raise SystemExit("oracle/_ref/libktune_ref.so missing: run `make -C oracle` first")
    return L


def text():
    return lib().ref_last_text().decode()


def call(fn, *args):
    rc = fn(*args)
    if rc != 0:
        raise RuntimeError(lib().ref_last_error().decode())


def i32(v):
    a = np.asarray(v, np.int32)
    return a, a.ctypes.data_as(O.c_i32p)


def i64(v):
    a = np.asarray(v, np.int64)
    return a, a.ctypes.data_as(O.c_i64p)


# ---------------------------------------------------------------------------
# executors: output hashes of the reference execute_gemm/execute_conv
# ---------------------------------------------------------------------------

def executor_cases():
    rng = np.random.default_rng(20240917)
    gemm, conv = [], []
    # The reference tests' frozen tuples (test_backends.cpp:155-166, 217-245,
    # 388, 407) plus random tuples over the reference test generator's ranges.
    fixed = [
        (7, 11, 13, 1, 1, [2, 2, 8, 4, 4, 2, 4, 4], "f64"),
        (7, 11, 13, 1, 1, [2, 2, 8, 4, 4, 2, 4, 4], "f32"),
        (48, 40, 56, 0, 0, [2, 2, 8, 8, 2, 1, 1, 1], "f32"),
        (64, 64, 64, 0, 1, [2, 8, 32, 32, 8, 1, 1, 1], "f32"),
        (33, 17, 300, 1, 0, [4, 2, 16, 16, 16, 4, 4, 8], "f32"),
        (5, 3, 1, 0, 0, [1, 1, 4, 4, 4, 4, 8, 16], "f32"),
        (16, 16, 257, 0, 1, [2, 2, 16, 16, 8, 2, 2, 32], "f64"),
    ]
    for m, n, k, ta, tb, t, dt in fixed:
        gemm.append(dict(m=m, n=n, k=k, ta=ta, tb=tb, tuning=t, dtype=dt))
    for trial in range(40):
        ms, ns = int(rng.choice([1, 2, 4])), int(rng.choice([1, 2, 4]))
        ks = int(rng.choice([1, 2, 4]))
        t = [ms, ns, ms * int(rng.choice([1, 2, 4])), ns * int(rng.choice([1, 2, 4])), ks * int(rng.choice([1, 2])),
             ks, int(rng.choice([1, 2, 4])), int(rng.choice([1, 2, 4]))]
        gemm.append(dict(m=int(rng.integers(1, 49)), n=int(rng.integers(1, 49)), k=int(rng.integers(1, 49)),
                         ta=int(rng.integers(0, 2)), tb=int(rng.integers(0, 2)), tuning=t,
                         dtype="f32" if trial % 2 == 0 else "f64"))
    conv.append(dict(dims=[3, 5, 4, 6, 7, 1, 1], tuning=[2, 1, 2, 1, 2, 2, 2, 1, 2, 1, 2, 2], dtype="f64"))
    conv.append(dict(dims=[2, 6, 6, 4, 3, 3, 3], tuning=[1, 1, 1, 1, 2, 2, 2, 1, 1, 1, 1, 1], dtype="f32"))
    conv.append(dict(dims=[4, 7, 9, 10, 5, 3, 2], tuning=[2, 1, 2, 2, 8, 2, 4, 2, 4, 2, 2, 4], dtype="f32"))
    for trial in range(20):
        ks_, ps, qs, ns = (int(rng.choice([1, 2])) for _ in range(4))
        cs = int(rng.choice([1, 2]))
        t = [ks_, ps, qs, ns, ks_ * int(rng.choice([1, 2, 4])), ps * int(rng.choice([1, 2])),
             qs * int(rng.choice([1, 2])), ns * int(rng.choice([1, 2])), cs * int(rng.choice([1, 2])), cs,
             int(rng.choice([1, 2])), int(rng.choice([1, 2, 4]))]
        dims = [int(rng.integers(1, 5)), int(rng.integers(1, 7)), int(rng.integers(1, 7)), int(rng.integers(1, 7)),
                int(rng.integers(1, 6)), int(rng.choice([1, 2, 3])), int(rng.choice([1, 2, 3]))]
        conv.append(dict(dims=dims, tuning=t, dtype="f32" if trial % 2 == 0 else "f64"))
    for i, c in enumerate(gemm):
        c["seed"] = 1000 + i
        a, b = O.fill(c["seed"], c["m"] * c["k"], c["k"] * c["n"], c["dtype"], symmetric=True)
        out = O.ref_execute_gemm(c["m"], c["n"], c["k"], c["ta"], c["tb"], c["tuning"], a, b, c["dtype"])
        c["sha256"] = sha(out)
        c["first"] = [float(x) for x in out[:4]]
    for i, c in enumerate(conv):
        c["seed"] = 5000 + i
        ni, nf, _ = O.conv_sizes(c["dims"])
        img, flt = O.fill(c["seed"], ni, nf, c["dtype"], symmetric=True)
        out = O.ref_execute_conv(c["dims"], c["tuning"], img, flt, c["dtype"])
        c["sha256"] = sha(out)
        c["first"] = [float(x) for x in out[:4]]
    # operand fill stream (pins the oracle's MT19937-64 + unit_real)
    fill = np.empty(64)
    call(lib().ref_fill_f64, ctypes.c_uint64(0x5EED), c_i64(64), fill.ctypes.data_as(O.c_dp))
    return {"gemm": gemm, "conv": conv, "fill_0x5eed_first64": [float(x) for x in fill]}


# ---------------------------------------------------------------------------
# parameter space
# ---------------------------------------------------------------------------

def enum_gemm(hw, bounds, m, n, k, dt, ta=0, tb=0):
    L = lib()
    cnt = c_i64()
    call(L.ref_enumerate_gemm, hw.encode(), bounds.encode(), c_i64(m), c_i64(n), c_i64(k), DT[dt], ta, tb, None,
         c_i64(0), ctypes.byref(cnt))
    out = np.zeros((cnt.value, 8), np.int32)
    call(L.ref_enumerate_gemm, hw.encode(), bounds.encode(), c_i64(m), c_i64(n), c_i64(k), DT[dt], ta, tb,
         out.ctypes.data_as(O.c_i32p), c_i64(cnt.value), ctypes.byref(cnt))
    return out


def enum_conv(hw, bounds, dims, dt):
    L = lib()
    cnt = c_i64()
    d, dp = i64(dims)
    call(L.ref_enumerate_conv, hw.encode(), bounds.encode(), dp, DT[dt], None, c_i64(0), ctypes.byref(cnt))
    out = np.zeros((cnt.value, 12), np.int32)
    call(L.ref_enumerate_conv, hw.encode(), bounds.encode(), dp, DT[dt], out.ctypes.data_as(O.c_i32p),
         c_i64(cnt.value), ctypes.byref(cnt))
    return out


def space_cases():
    L = lib()
    res = {"enumerations": [], "legality_gemm": [], "legality_conv": [], "features_gemm": [], "features_conv": [],
           "indirection": [], "json": {}}
    gem_runs = [("synthetic", "", "", 512, 512, 512, "f32"), ("synthetic", "", "", 512, 512, 512, "f64"),
                ("synthetic", "", "", 512, 512, 512, "f16"), ("b200", B200_HW, B200_GEMM_BOUNDS, 2560, 16, 2560, "f32"),
                ("b200", B200_HW, B200_GEMM_BOUNDS, 512, 512, 512, "f64"), ("b200-default-bounds", B200_HW, "", 64, 64,
                                                                           64, "f32")]
    for name, hw, b, m, n, k, dt in gem_runs:
        arr = enum_gemm(hw, b, m, n, k, dt)
        res["enumerations"].append(dict(kind="gemm", hw=name, bounds=("b200" if b else "default"), m=m, n=n, k=k,
                                        dtype=dt, count=int(len(arr)), sha256=sha(arr), head=arr[:5].tolist(),
                                        tail=arr[-5:].tolist()))
    conv_runs = [("synthetic", "", CONV_SMALL, "conv_small", [16, 24, 240, 32, 16, 3, 3], "f32"),
                 ("b200", B200_HW, B200_CONV_BOUNDS, "b200", [16, 56, 56, 64, 64, 3, 3], "f32")]
    for name, hw, b, bname, dims, dt in conv_runs:
        arr = enum_conv(hw, b, dims, dt)
        res["enumerations"].append(dict(kind="conv", hw=name, bounds=bname, dims=dims, dtype=dt, count=int(len(arr)),
                                        sha256=sha(arr), head=arr[:5].tolist(), tail=arr[-5:].tolist()))
    rng = np.random.default_rng(7)
    p2 = [1, 2, 4, 8, 16, 32, 64, 128, 256]
    for i in range(600):
        hwname, hw = ("synthetic", "") if i % 2 == 0 else ("b200", B200_HW)
        t = [int(rng.choice(p2[:6] if j in (0, 1, 5) else p2)) for j in range(8)]
        m, n, k = (int(x) for x in rng.integers(1, 5000, 3))
        dt = ["f16", "f32", "f64"][i % 3]
        tv, tp = i32(t)
        acc, why = ctypes.c_int(), ctypes.c_int()
        call(L.ref_is_legal_gemm, hw.encode(), c_i64(m), c_i64(n), c_i64(k), DT[dt], 0, 0, tp, ctypes.byref(acc),
             ctypes.byref(why))
        detail = text()
        r3, rp = i64([0, 0, 0])
        call(L.ref_resources_gemm, c_i64(m), c_i64(n), c_i64(k), DT[dt], tp, rp)
        res["legality_gemm"].append(dict(hw=hwname, m=m, n=n, k=k, dtype=dt, tuning=t, accepted=acc.value,
                                         reason=why.value, detail=detail, resources=r3.tolist()))
    for i in range(400):
        hwname, hw = ("synthetic", "") if i % 2 == 0 else ("b200", B200_HW)
        t = [int(rng.choice(p2[:5])) for _ in range(12)]
        dims = [int(x) for x in rng.integers(1, 64, 7)]
        dt = ["f16", "f32", "f64"][i % 3]
        tv, tp = i32(t)
        d, dp = i64(dims)
        acc, why = ctypes.c_int(), ctypes.c_int()
        call(L.ref_is_legal_conv, hw.encode(), dp, DT[dt], tp, ctypes.byref(acc), ctypes.byref(why))
        detail = text()
        r3, rp = i64([0, 0, 0])
        call(L.ref_resources_conv, dp, DT[dt], tp, rp)
        res["legality_conv"].append(dict(hw=hwname, dims=dims, dtype=dt, tuning=t, accepted=acc.value,
                                         reason=why.value, detail=detail, resources=r3.tolist()))
    for i in range(40):
        t = [int(rng.choice(p2)) for _ in range(8)]
        m, n, k = (int(x) for x in rng.integers(1, 70000, 3))
        dt, ta, tb = ["f16", "f32", "f64"][i % 3], i % 2, (i // 2) % 2
        tv, tp = i32(t)
        f = np.zeros(14)
        call(L.ref_features_gemm, c_i64(m), c_i64(n), c_i64(k), DT[dt], ta, tb, tp, f.ctypes.data_as(O.c_dp))
        res["features_gemm"].append(dict(m=m, n=n, k=k, dtype=dt, ta=ta, tb=tb, tuning=t, features=f.tolist()))
    for i in range(20):
        t = [int(rng.choice(p2)) for _ in range(12)]
        dims = [int(x) for x in rng.integers(1, 600, 7)]
        tv, tp = i32(t)
        d, dp = i64(dims)
        f = np.zeros(19)
        call(L.ref_features_conv, dp, 1, tp, f.ctypes.data_as(O.c_dp))
        res["features_conv"].append(dict(dims=dims, tuning=t, features=f.tolist()))
    for dims in ([2, 2, 3, 1, 2, 2, 2], [16, 56, 56, 64, 64, 3, 3], [16, 79, 341, 32, 1, 5, 20], [3, 1, 1, 2, 7, 4, 1]):
        n_ = dims[4] * dims[5] * dims[6]
        out = np.zeros((n_, 4), np.int64)
        d, dp = i64(dims)
        call(L.ref_indirection, dp, out.ctypes.data_as(O.c_i64p))
        res["indirection"].append(dict(dims=dims, count=n_, sha256=sha(out), head=out[:6].tolist(),
                                       tail=out[-3:].tolist()))
    call(L.ref_hw_json, b"")
    res["json"]["hw_default"] = text()
    call(L.ref_hw_json, B200_HW.encode())
    res["json"]["hw_b200"] = text()
    call(L.ref_bounds_json, b"", 0)
    res["json"]["gemm_bounds_default"] = text()
    call(L.ref_bounds_json, B200_GEMM_BOUNDS.encode(), 0)
    res["json"]["gemm_bounds_b200"] = text()
    call(L.ref_bounds_json, CONV_SMALL.encode(), 1)
    res["json"]["conv_bounds_small"] = text()
    pk = ctypes.c_double()
    call(L.ref_peak_gflops, B200_HW.encode(), ctypes.byref(pk))
    res["peak_gflops_b200"] = pk.value
    call(L.ref_peak_gflops, b"", ctypes.byref(pk))
    res["peak_gflops_synthetic"] = pk.value
    return res


def main():
    lib()
    out_dir = HERE
    with open(os.path.join(out_dir, "executors.json"), "w") as fh:
        json.dump(executor_cases(), fh, indent=1)
    with open(os.path.join(out_dir, "space.json"), "w") as fh:
        json.dump(space_cases(), fh, indent=1)
    print("wrote", os.listdir(out_dir))


if __name__ == "__main__":
    main()

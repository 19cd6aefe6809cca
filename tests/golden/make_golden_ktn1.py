"""KTN1 golden parity vectors: operands and the
UNMODIFIED reference executor's outputs (oracle/_ref/libktune_ref.so,
execute_gemm<float/double> / execute_conv<float>) for a few tuples, written
with the reference's own KTN1 writer, so the GPU parity gate replays them
without a CPU rerun (tests/test_ktn1_replay_gpu.py).

    python tests/golden/make_golden_ktn1.py
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_libs as O  # noqa: E402

OUT = os.path.join(HERE, "ktn1")
GEMM = [  # m, n, k, ta, tb, dtype, tuple
    (96, 40, 300, 0, 0, "f32", (2, 4, 32, 16, 8, 2, 2, 4)),
    (64, 64, 512, 1, 1, "f32", (4, 4, 64, 32, 16, 1, 1, 8)),
    (50, 33, 257, 0, 1, "f64", (2, 1, 16, 8, 4, 2, 2, 4)),
]
CONV = [  # n, p, q, k, c, r, s, tuple
    ((4, 9, 11, 24, 5, 3, 3), (2, 1, 1, 2, 8, 2, 2, 4, 4, 2, 2, 2)),
]


def write(lib, name, a):
    a = np.ascontiguousarray(a)
    dims = (ctypes.c_int64 * a.ndim)(*a.shape)
    path = os.path.join(OUT, name)
    if lib.ref_write_tensor(path.encode(), int(a.dtype == np.float64), dims, a.ndim,
                            a.ctypes.data_as(ctypes.c_void_p)) != 0:
        raise RuntimeError(lib.ref_last_error().decode())
    return name


def main():
    lib = O.reference()
    if lib is None:
        raise SystemExit("oracle/_ref/libktune_ref.so missing: run `make -C oracle` first")
    os.makedirs(OUT, exist_ok=True)
    cases = []
    for i, (m, n, k, ta, tb, dt, t) in enumerate(GEMM):
        a, b = O.fill(100 + i, m * k, k * n, dt, True)
        c = O.ref_execute_gemm(m, n, k, ta, tb, t, a, b, dt)
        cases.append({"kind": "gemm", "m": m, "n": n, "k": k, "trans_a": ta, "trans_b": tb, "dtype": dt, "tuning": t,
                      "a": write(lib, f"gemm{i}_a.ktn", a.reshape((k, m) if ta else (m, k))),
                      "b": write(lib, f"gemm{i}_b.ktn", b.reshape((n, k) if tb else (k, n))),
                      "c": write(lib, f"gemm{i}_c.ktn", c.reshape(m, n))})
    for i, (d, t) in enumerate(CONV):
        nb, p, q, kk, cc, r, s = d
        h, w = p + r - 1, q + s - 1
        img, flt = O.fill(200 + i, cc * h * w * nb, cc * r * s * kk, "f32", True)
        out = O.ref_execute_conv(list(d), t, img, flt, "f32")
        cases.append({"kind": "conv", "dims": list(d), "dtype": "f32", "tuning": t,
                      "images": write(lib, f"conv{i}_images.ktn", img.reshape(cc, h, w, nb)),
                      "filters": write(lib, f"conv{i}_filters.ktn", flt.reshape(cc, r, s, kk)),
                      "outputs": write(lib, f"conv{i}_outputs.ktn", out.reshape(kk, p, q, nb))})
    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump({"format": "ktune-b200-ktn1-golden-1", "cases": cases}, fh, indent=1)
    print("wrote", len(cases), "cases to", OUT)


if __name__ == "__main__":
    main()

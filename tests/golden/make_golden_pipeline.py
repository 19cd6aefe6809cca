"""Generates tests/golden/pipeline.json from the UNMODIFIED reference library
(oracle/_ref/libktune_ref.so): sampler models and acceptance rates, the
analytical-backend dataset sequences (CSV bytes), MLP init/prediction/
training outputs, inference results and cache keys.

    python tests/golden/make_golden_pipeline.py
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
FIX = os.path.join(ROOT, "paper_1802_05371_b200", "fixtures")
B200_HW = open(os.path.join(FIX, "hw", "b200.json")).read()
B200_GEMM = open(os.path.join(FIX, "bounds", "gemm_b200.json")).read()
CONV_SMALL = open(os.path.join(REF, "fixtures", "bounds", "conv_small.json")).read()
GEMM_TABLE = json.load(open(os.path.join(REF, "fixtures", "shapes", "gemm_table.json")))["shapes"]
CONV_TABLE = json.load(open(os.path.join(REF, "fixtures", "shapes", "conv_table.json")))["shapes"]
c_i64, c_u64, c_dbl = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double


def sha(text: str) -> str:
    return hashlib.sha256(text.encode()).hexdigest()


def L():
    lib = O.reference()
    if lib is None:
        raise SystemExit("oracle/_ref/libktune_ref.so missing: run `make -C oracle` first")
    return lib


def call(fn, *args):
    if fn(*args) != 0:
        raise RuntimeError(L().ref_last_error().decode())
    return L().ref_last_text().decode()


def gemm_rows(shapes, dtype=1):
    rows = []
    for s in shapes:
        rows += [s["m"], s["n"], s["k"], dtype, int(s["trans_a"]), int(s["trans_b"])]
    return (ctypes.c_int64 * len(rows))(*rows)


def conv_rows(shapes, dtype=1):
    rows = []
    for s in shapes:
        rows += [s["n"], s["p"], s["q"], s["k"], s["c"], s["r"], s["s"], dtype]
    return (ctypes.c_int64 * len(rows))(*rows)


def main():
    lib = L()
    out = {}
    # --- sampler -------------------------------------------------------------
    synth = call(lib.ref_calibrate_gemm, b"", b"", c_i64(512), c_i64(512), c_i64(512), 1, c_i64(100000), c_u64(11),
                 c_dbl(100.0))
    b200 = call(lib.ref_calibrate_gemm, B200_HW.encode(), B200_GEMM.encode(), c_i64(512), c_i64(512), c_i64(512), 1,
                c_i64(100000), c_u64(11), c_dbl(100.0))
    d = (ctypes.c_int64 * 7)(16, 24, 240, 32, 16, 3, 3)
    conv = call(lib.ref_calibrate_conv, b"", CONV_SMALL.encode(), d, 1, c_i64(100000), c_u64(11), c_dbl(100.0))
    r = c_dbl()
    call(lib.ref_acceptance_gemm, b"", synth.encode(), c_i64(512), c_i64(512), c_i64(512), 1, c_i64(100000), c_u64(1),
         ctypes.byref(r))
    out["sampler"] = {"synthetic_json": synth, "b200_json": b200, "conv_small_json": conv,
                      "synthetic_acceptance_seed1": r.value}
    # --- generation with the analytical backend ------------------------------
    att, dup = c_i64(), c_i64()
    rows = gemm_rows(GEMM_TABLE)
    csv_synth = call(lib.ref_generate_gemm, b"", b"", synth.encode(), rows, len(GEMM_TABLE), c_dbl(0.25), 1, 2000,
                     c_u64(42), ctypes.byref(att), ctypes.byref(dup))
    gen = {"synthetic": {"n": 2000, "seed": 42, "fixed_fraction": 0.25, "csv_sha256": sha(csv_synth),
                         "head": csv_synth.splitlines()[:12], "attempts": att.value, "duplicates": dup.value}}
    csv_b200 = call(lib.ref_generate_gemm, B200_HW.encode(), B200_GEMM.encode(), b200.encode(), rows, len(GEMM_TABLE),
                    c_dbl(0.25), 1, 1000, c_u64(42), ctypes.byref(att), ctypes.byref(dup))
    gen["b200"] = {"n": 1000, "seed": 42, "fixed_fraction": 0.25, "csv_sha256": sha(csv_b200),
                   "head": csv_b200.splitlines()[:12], "attempts": att.value, "duplicates": dup.value}
    crow = conv_rows(CONV_TABLE)
    csv_conv = call(lib.ref_generate_conv, b"", CONV_SMALL.encode(), conv.encode(), crow, len(CONV_TABLE),
                    c_dbl(0.25), 1, 300, c_u64(5), ctypes.byref(att), ctypes.byref(dup))
    gen["conv_small"] = {"n": 300, "seed": 5, "fixed_fraction": 0.25, "csv_sha256": sha(csv_conv),
                         "head": csv_conv.splitlines()[:8], "attempts": att.value, "duplicates": dup.value}
    out["generate"] = gen
    roundtrip = call(lib.ref_csv_roundtrip_gemm, csv_synth.encode())
    out["csv_roundtrip_identical"] = roundtrip == csv_synth
    # --- MLP -------------------------------------------------------------------
    hid = (ctypes.c_int * 3)(32, 64, 32)
    init = call(lib.ref_init_weights, 14, hid, 3, c_u64(7))
    rng = np.random.default_rng(3)
    feats = np.exp(rng.uniform(0, 9, size=(400, 14)))  # strictly positive
    pred = np.zeros(400)
    call(lib.ref_mlp_predict, init.encode(), feats.ctypes.data_as(O.c_dp), c_i64(400), 14, pred.ctypes.data_as(O.c_dp))
    out["mlp"] = {"init_seed7_json": init, "features": feats.tolist(), "predict_init": [float.hex(x) for x in pred]}
    bv, be = c_dbl(), ctypes.c_int()
    trained = call(lib.ref_train_gemm, csv_synth.encode(), hid, 3, 5, c_dbl(1e-3), 256, c_u64(7), c_dbl(0.1), 1,
                   ctypes.byref(bv), ctypes.byref(be))
    out["mlp"]["train_5ep_json"] = trained
    out["mlp"]["train_5ep_best_val"] = float.hex(bv.value)
    out["mlp"]["train_5ep_best_epoch"] = be.value
    # --- inference + cache -------------------------------------------------------
    res_an = call(lib.ref_infer_gemm_analytical, b"", b"", b"", c_i64(2048), c_i64(2048), c_i64(2048), 1, 0, 1, 100)
    res_ml = call(lib.ref_infer_gemm_analytical, b"", b"", trained.encode(), c_i64(2560), c_i64(16), c_i64(2560), 1, 0,
                  0, 20)
    keys = {}
    for m, n, k, dt, ta, tb in [(512, 512, 512, 1, 0, 1), (2560, 16, 2560, 1, 0, 0), (32, 32, 60000, 2, 1, 1)]:
        keys[f"{m},{n},{k},{dt},{ta},{tb}"] = call(lib.ref_cache_key_gemm, c_i64(m), c_i64(n), c_i64(k), dt, ta, tb)
    ckey = call(lib.ref_cache_key_conv, d, 1)
    # analytical prices for a slice of the synthetic space
    space = np.zeros((6140, 8), np.int32)
    cnt = c_i64()
    if lib.ref_enumerate_gemm(b"", b"", c_i64(512), c_i64(512), c_i64(512), 1, 0, 0, space.ctypes.data_as(O.c_i32p),
                              c_i64(6140), ctypes.byref(cnt)) != 0:
        raise RuntimeError("enumerate failed")
    prices = []
    for t in space[::37]:
        g = c_dbl()
        tv = (ctypes.c_int32 * 8)(*[int(x) for x in t])
        call(lib.ref_analytical_gemm, b"", c_i64(512), c_i64(512), c_i64(512), 1, 0, 0, tv, ctypes.byref(g))
        prices.append([t.tolist(), float.hex(g.value)])
    cprices = []
    cspace = np.zeros((14448, 12), np.int32)
    if lib.ref_enumerate_conv(b"", CONV_SMALL.encode(), d, 1, cspace.ctypes.data_as(O.c_i32p), c_i64(14448),
                              ctypes.byref(cnt)) != 0:
        raise RuntimeError("enumerate conv failed")
    for t in cspace[::97]:
        g = c_dbl()
        tv = (ctypes.c_int32 * 12)(*[int(x) for x in t])
        call(lib.ref_analytical_conv, b"", d, 1, tv, ctypes.byref(g))
        cprices.append([t.tolist(), float.hex(g.value)])
    out["infer"] = {"analytical_2048_nt_top100": res_an, "mlp5ep_deepbench16_top20": res_ml}
    out["cache_keys"] = {"gemm": keys, "conv_16_24_240_32_16_3_3_f32": ckey}
    out["analytical"] = {"gemm_512_nn_f32": prices, "conv_small": cprices}
    with open(os.path.join(HERE, "pipeline.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote pipeline.json", os.path.getsize(os.path.join(HERE, "pipeline.json")), "bytes")


if __name__ == "__main__":
    main()

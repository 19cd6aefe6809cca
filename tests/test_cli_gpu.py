"""`ktune_b200` verbs that run on the B200 (train: K7, infer: the K6 sweep,
--backend b200 device measurement), checked against the unmodified reference
library on the same files: the trained model JSON and the ktune-result-1
JSON are byte-identical (5 epochs, no clipped step -- DESIGN.md A12/A13)."""
import ctypes
import json
import os
import subprocess

import pytest

import oracle_libs as O
from test_cli import CLI, GEMM_BOUNDS, HW, TABLE, reference_gemm_table, run

pytestmark = pytest.mark.gpu


def _dataset(tmp_path):
    s, d = tmp_path / "sampler.json", tmp_path / "data.csv"
    assert run("calibrate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--seed", 11, "--draws", 20000, "--out", s)[0] == 0
    assert run("generate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--sampler", s, "--shapes", TABLE,
               "--shape-fraction", 0.25, "--samples", 600, "--seed", 42, "--out", d)[0] == 0
    return s, d


def test_train_and_infer_match_reference(cuda, tmp_path):
    lib = O.reference()
    if lib is None:
        pytest.skip("reference library (oracle/_ref) not built")
    _, d = _dataset(tmp_path)
    m, rep = tmp_path / "model.json", tmp_path / "train.json"
    code, out, err = run("train", "--dataset", d, "--epochs", 5, "--seed", 7, "--out", m, "--report", rep)
    assert code == 0, err
    hid = (ctypes.c_int * 3)(32, 64, 32)
    bv, be = ctypes.c_double(), ctypes.c_int()
    assert lib.ref_train_gemm(d.read_bytes(), hid, 3, 5, ctypes.c_double(1e-3), 256, ctypes.c_uint64(7),
                              ctypes.c_double(0.1), 1, ctypes.byref(bv), ctypes.byref(be)) == 0
    ref_model = lib.ref_last_text().decode()
    assert m.read_text().rstrip("\n") == ref_model.rstrip("\n")
    r = json.loads(rep.read_text())
    assert r["best_epoch"] == be.value and r["best_val_mse"] == bv.value and len(r["history"]) == 5

    # runtime selection with the learned model (GPU sweep), analytical re-measure
    res, cache = tmp_path / "res.json", tmp_path / "cache"
    args = ("infer", "--model", m, "--hw", HW, "--bounds", GEMM_BOUNDS, "--shape", "2560,16,2560", "--top-k", 20,
            "--backend", "analytical", "--cache-dir", cache, "--out", res)
    code, out, err = run(*args)
    assert code == 0 and "legal space" in out, err
    hw_json, bounds_json = open(HW).read().encode(), open(GEMM_BOUNDS).read().encode()
    assert lib.ref_infer_gemm_analytical(hw_json, bounds_json, ref_model.encode(), ctypes.c_int64(2560),
                                         ctypes.c_int64(16), ctypes.c_int64(2560), 1, 0, 0, 20) == 0
    assert res.read_text() == lib.ref_last_text().decode()
    # second call: the FNV-keyed result cache answers (pipeline.cpp:936-997)
    res.unlink()
    code, out, _ = run(*args)
    assert code == 0 and out.startswith("cache hit")
    assert res.read_text() == lib.ref_last_text().decode()
    # KTUNE_CACHE_DIR overrides --cache-dir
    code, out, _ = run(*args, env={"KTUNE_CACHE_DIR": str(tmp_path / "other")})
    assert code == 0 and not out.startswith("cache hit")
    # report with the model: MSE on the dataset
    code, out, _ = run("report", "--dataset", d, "--model", m)
    assert code == 0 and "MSE" in out


def test_generate_and_bench_on_the_b200_backend(cuda, tmp_path):
    s, _ = _dataset(tmp_path)
    d = tmp_path / "b200.csv"
    code, out, err = run("generate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--sampler", s, "--backend", "b200",
                         "--samples", 6, "--seed", 5, "--out", d)
    assert code == 0, err
    lines = d.read_text().splitlines()
    assert len(lines) == 7 and all(ln.endswith(",b200") for ln in lines[1:])
    table = reference_gemm_table(tmp_path, {"linpack-512"})
    m = tmp_path / "model.json"
    assert run("train", "--dataset", d, "--epochs", 3, "--out", m)[0] == 0
    out_json = tmp_path / "bench.json"
    code, out, err = run("bench", "--model", m, "--hw", HW, "--bounds", GEMM_BOUNDS, "--shapes", table,
                         "--backend", "b200", "--top-k", 4, "--out", out_json)
    assert code == 0, err
    rep = json.loads(out_json.read_text())
    assert rep["mode"] == "model" and rep["backend"] == "b200"
    assert rep["results"][0]["measured_gflops"] > 0

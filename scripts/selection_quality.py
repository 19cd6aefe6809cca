"""Input-aware selection quality on the B200 (ISAAC's core claim; the
reference's acceptance criterion 7, acceptance_main.cpp:437-466, re-run on
device-measured data instead of the synthetic analytical device).

1. calibrate the sampler on the B200 descriptor + bounds, generate a
   device-measured dataset with the sharded pipeline (README walkthrough,
   fixture shapes at 0.25), train the MLP on the GPU;
2. for every test shape (the paper's GEMM table + random draws of the
   training distribution with another seed): the model-driven pick
   (infer: GPU sweep of the whole legal space, top-k re-measured on the
   B200) and the analytical-model pick, against the best tuple found by
   measuring a large random sample of the legal space plus both picks'
   candidates (the "exhaustive" reference point, bounded);
3. report per-shape ratios pick / best and the count within 95 %.

    python scripts/selection_quality.py [--samples 12000] [--random 600] [--out profiles/...json]
    python scripts/selection_quality.py --dtype bf16 ...   # tensor-core family

With --dtype bf16 the same loop runs on the tcgen05 family: the
gemm_b200_tc bounds, the calibrated tensor-core sampler fixture, bf16 inputs
(the gemm.v1 features encode only the element size, so the model is trained
on -- and used for -- one dtype; SURVEY 7's dtype decision), and only
tuples the family can launch are ranked, drawn and measured.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1802_05371_b200 as K  # noqa: E402
from paper_1802_05371_b200 import pipeline as P  # noqa: E402


def launchable(inp, row):
    try:
        K.gemm_launch_info(inp, K.GemmTuning(*map(int, row)), "fast")
        return True
    except K.KtuneError:
        return False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=12000)
    ap.add_argument("--random", type=int, default=600)
    ap.add_argument("--top-k", type=int, default=20)
    ap.add_argument("--epochs", type=int, default=200)
    ap.add_argument("--extra-shapes", type=int, default=13)
    ap.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    tc = a.dtype != "f32"
    if a.out is None:
        a.out = os.path.join(ROOT, "profiles", "r2_selection_quality_bf16.json" if tc else "r1_selection_quality.json")
    import torch
    torch.cuda.set_device(0)
    hw = K.HardwareDescriptor.b200()
    bounds = open(os.path.join(K.FIXTURES, "bounds", "gemm_b200_tc.json" if tc else "gemm_b200.json")).read()
    table = P.gemm_shapes_from_table(os.path.join(K.FIXTURES, "shapes", "benchmarks.json"), a.dtype)
    t0 = time.perf_counter()
    if tc:  # the calibrated tensor-core sampler (fixtures/samplers, `calibrate --dtype bf16 --seed 11`)
        sampler = open(os.path.join(K.FIXTURES, "samplers", "gemm_b200_tc_bf16.json")).read()
    else:
        sampler = P.calibrate(K.GemmInput(512, 512, 512), hw, bounds, 100000, 11)
    dist = P.GemmInputDistribution(shapes=table, fixed_fraction=0.25, dtype=a.dtype)
    csv, stats = P.generate_sharded(sampler, dist, hw, bounds, a.samples, 42, backend="b200")
    t_gen = time.perf_counter() - t0
    print(f"generated {a.samples} samples in {t_gen:.1f} s", flush=True)
    t1 = time.perf_counter()
    fit = P.train_mlp(csv, epochs=a.epochs, seed=7, fast=True)  # K7f (batched fp64 GEMMs)
    t_fit = time.perf_counter() - t1
    print(f"trained in {t_fit:.1f} s (best val mse {fit.best_val_mse:.3f})", flush=True)
    # test shapes: the table + fresh draws of the training distribution
    ins, _, _, _ = P.predraw(sampler, P.GemmInputDistribution(shapes=[], fixed_fraction=0.0, dtype=a.dtype), hw,
                             bounds, a.extra_shapes, 2024)
    shapes = [("table:" + str(i), s) for i, s in enumerate(table)] + \
             [("draw:" + str(i), s) for i, s in enumerate(P.as_inputs(ins))]
    rng = np.random.default_rng(0)
    rows = []
    for name, inp in shapes:
        space = K.enumerate_legal(inp, hw, bounds, as_array=True)
        if tc:  # the random reference points: launchable, one per tensor-core-distinct key
            from paper_1802_05371_b200.tuner import tc_gemm_key
            _, first = np.unique(np.asarray([tc_gemm_key(r) for r in space]), axis=0, return_index=True)
            space = space[np.sort(first)]
            space = space[np.asarray([launchable(inp, r) for r in space], bool)]
        res_m = json.loads(P.infer(inp, hw, bounds, fit.model_json, top_k=a.top_k, backend="b200"))
        res_a = json.loads(P.infer(inp, hw, bounds, None, top_k=a.top_k, backend="b200"))
        pick = [rng.integers(len(space))] if len(space) else []
        idx = rng.choice(len(space), size=min(a.random, len(space)), replace=False)
        cands = {tuple(int(x) for x in space[i]) for i in idx}
        for r in (res_m, res_a):
            for c in r["top_k"]:
                cands.add(tuple(c["tuning"][n] for n in K.GEMM_PARAMS))
        meas = []
        for t in cands:
            try:
                meas.append((K.measure(inp, K.GemmTuning(*t), hw, repetitions=1, warmup=1), t))
            except K.KtuneError:
                pass
        meas.sort(key=lambda x: -x[0])
        best = max(K.measure(inp, K.GemmTuning(*t), hw, repetitions=3, warmup=1) for _, t in meas[:8])
        chosen_m = tuple(res_m["chosen"][n] for n in K.GEMM_PARAMS)
        chosen_a = tuple(res_a["chosen"][n] for n in K.GEMM_PARAMS)
        gm = K.measure(inp, K.GemmTuning(*chosen_m), hw, repetitions=3, warmup=1)
        ga = K.measure(inp, K.GemmTuning(*chosen_a), hw, repetitions=3, warmup=1)
        best = max(best, gm, ga)
        rows.append({"shape": name, "m": inp.m, "n": inp.n, "k": inp.k, "ta": inp.trans_a, "tb": inp.trans_b,
                     "legal_space": len(space), "measured_reference_points": len(meas),
                     "best_gflops": best, "mlp_pick": list(chosen_m), "mlp_gflops": gm, "mlp_ratio": gm / best,
                     "analytical_pick": list(chosen_a), "analytical_gflops": ga, "analytical_ratio": ga / best})
        print(f"{name:10s} {inp.m:6d} {inp.n:6d} {inp.k:6d}  mlp {gm / best:5.2f}  analytical {ga / best:5.2f}",
              flush=True)
    mr = np.array([r["mlp_ratio"] for r in rows])
    ar = np.array([r["analytical_ratio"] for r in rows])
    out = {"format": "ktune-b200-selection-1", "dtype": a.dtype,
           "family": "tcgen05 (gemm_b200_tc bounds)" if tc else "simt fp32 (gemm_b200 bounds)",
           "dataset": {"samples": a.samples, "backend": "b200 (device measured)", "seconds": t_gen,
                       "samples_per_s": a.samples / t_gen},
           "mlp": {"hidden": [32, 64, 32], "epochs": a.epochs, "best_val_mse_log": fit.best_val_mse,
                   "best_epoch": fit.best_epoch, "fit_seconds": t_fit},
           "protocol": f"pick = infer (top-{a.top_k} re-measured on the B200); best = max over {a.random} random legal "
                       "tuples + both picks' top-k, top 8 re-measured (3 reps)",
           "summary": {"shapes": len(rows), "mlp_within_95pct": int((mr >= 0.95).sum()),
                       "mlp_median_ratio": float(np.median(mr)), "mlp_min_ratio": float(mr.min()),
                       "analytical_within_95pct": int((ar >= 0.95).sum()),
                       "analytical_median_ratio": float(np.median(ar))},
           "shapes": rows}
    with open(a.out, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out["summary"]))


if __name__ == "__main__":
    main()

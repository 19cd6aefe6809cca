"""Fit the analytical cost model's B200 constants to device-measured data
(SURVEY section 8(f) row 2).  The model of backends.cpp:14-195 prices a
kernel from the descriptor's latency / throughput constants; with the
B200 descriptor's nominal values it ranks B200 tuples poorly (3/30 picks
within 95 %, profiles/r1_selection_quality.json).  This script

1. measures a dataset on the B200 (sharded pipeline, fixture shapes at
   fraction 0.5 so every table shape has dozens of measured tuples);
2. random-searches alu_latency, alu_throughput, mem_latency and
   mem_throughput (the legality limits stay the hardware's) to maximise the
   mean per-shape Spearman correlation between analytical and measured
   GFLOPS on the table shapes, on a train half, reporting the held-out half;
3. writes gpurun_out/b200_fitted.json and gpurun_out/r1_analytical_fit.json
   (committed as fixtures/hw/b200_fitted.json and profiles/r1_analytical_fit.json).

    python scripts/fit_analytical.py [--samples 4000]
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1802_05371_b200 as K  # noqa: E402
from paper_1802_05371_b200 import pipeline as P  # noqa: E402


def spearman(x, y):
    rx = np.argsort(np.argsort(x)).astype(float)
    ry = np.argsort(np.argsort(y)).astype(float)
    if rx.std() == 0 or ry.std() == 0:
        return 0.0
    return float(np.corrcoef(rx, ry)[0, 1])


def score(hw, groups):
    vals = []
    for inp, tus, g in groups:
        pred = np.array([P.analytical_gflops(inp, t, hw) for t in tus])
        vals.append(spearman(pred, g))
    return float(np.mean(vals))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=4000)
    ap.add_argument("--trials", type=int, default=300)
    a = ap.parse_args()
    import torch
    torch.cuda.set_device(0)
    hw0 = K.HardwareDescriptor.b200()
    bounds = open(os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")).read()
    table = P.gemm_shapes_from_table(os.path.join(K.FIXTURES, "shapes", "benchmarks.json"))
    sampler = open(os.path.join(K.FIXTURES, "samplers", "gemm_b200.json")).read()
    t0 = time.perf_counter()
    csv, _ = P.generate_sharded(sampler, P.GemmInputDistribution(shapes=table, fixed_fraction=0.5), hw0, bounds,
                                a.samples, 77, backend="b200")
    t_gen = time.perf_counter() - t0
    with open(os.path.join(ROOT, "gpurun_out", "fit_dataset.csv"), "w") as fh:
        fh.write(csv)
    rows = [ln.split(",") for ln in csv.strip().splitlines()[1:]]
    by = {}
    for r in rows:
        key = (int(r[0]), int(r[1]), int(r[2]), r[3], int(r[4]), int(r[5]))
        by.setdefault(key, []).append((K.GemmTuning(*[int(x) for x in r[6:14]]), float(r[14])))
    groups = []
    for (m, n, k, dt, ta, tb), lst in by.items():
        if len(lst) >= 8:
            groups.append((K.GemmInput(m, n, k, dt, bool(ta), bool(tb)), [t for t, _ in lst],
                           np.array([g for _, g in lst])))
    rng = np.random.default_rng(0)
    idx = rng.permutation(len(groups))
    train = [groups[i] for i in idx[: len(idx) // 2]]
    test = [groups[i] for i in idx[len(idx) // 2:]]
    base = dataclasses.asdict(hw0)
    best = (score(hw0, train), base)
    for _ in range(a.trials):
        cand = dict(base)
        for f in ("alu_latency", "alu_throughput", "mem_latency", "mem_throughput"):
            cand[f] = float(base[f] * np.exp(rng.uniform(np.log(1 / 16), np.log(16))))
        try:
            s = score(K.HardwareDescriptor(**cand), train)
        except K.InvalidArgument:  # outside the model's domain (latency < cost per instruction)
            continue
        if s > best[0]:
            best = (s, cand)
    fitted = K.HardwareDescriptor(**best[1])
    out = {"format": "ktune-b200-analytical-fit-1", "samples": a.samples, "generate_seconds": t_gen,
           "shapes_with_8plus_measurements": len(groups), "train_shapes": len(train), "test_shapes": len(test),
           "metric": "mean per-shape Spearman correlation of analytical vs measured GFLOPS",
           "nominal": {"train": score(hw0, train), "test": score(hw0, test), "descriptor": base},
           "fitted": {"train": best[0], "test": score(fitted, test), "descriptor": best[1]}}
    with open(os.path.join(ROOT, "gpurun_out", "b200_fitted.json"), "w") as fh:
        json.dump(best[1], fh, indent=2)
        fh.write("\n")
    with open(os.path.join(ROOT, "gpurun_out", "r1_analytical_fit.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps({k: out[k] for k in ("nominal", "fitted")}, indent=1))


if __name__ == "__main__":
    main()

"""BASELINE configs[4] at its configured scale: the full ISAAC tuning loop
(100k random (shape x tuple) samples measured on the B200 + MLP fit + runtime
pick), the same code path as bench.py's bounded `tuning` record
(bench.tuning_loop), run once on one GPU.

    python scripts/tuning_loop.py [--samples 100000] [--out profiles/r2_tuning_100k.json]

Under torchrun the samples are LPT-sharded over the ranks exactly as in
bench.py --gpus N (strong scaling); rank 0 writes the record.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--samples", type=int, default=100000)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r2_tuning_100k.json"))
    a = ap.parse_args()
    import torch
    import torch.distributed as dist
    ws, rank, local = bench.dist_env()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    out = bench.tuning_loop(argparse.Namespace(tuning_samples=a.samples), ws, rank, dev)
    if rank == 0:
        out["note"] = "scripts/tuning_loop.py: bench.tuning_loop at --samples (BASELINE configs[4] scale)"
        with open(a.out, "w") as fh:
            json.dump(out, fh, indent=1)
        print(json.dumps({k: out[k] for k in ("samples", "samples_per_s", "seconds", "n_gpus")}))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

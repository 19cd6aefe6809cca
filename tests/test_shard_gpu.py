"""Sharded tuning-sample generation on the B200 (reference loop
generate_gemm_dataset, pipeline.cpp:463-509).

- A rank's shard measures exactly its LPT share of the sequence the
  sequential b200 generation measures (the sampler RNG never depends on
  measurements), every record positive.
- The per-rank checkpoint makes a rerun resume: recorded indices are not
  measured again and their values come back unchanged.
- The CLI form (`generate --shard R/N` on each rank, then `--merge`) writes a
  dataset whose rows are the sequence in canonical order.
"""
import os
import subprocess
import time

import numpy as np
import pytest

import paper_1802_05371_b200 as K
from paper_1802_05371_b200 import pipeline as P

pytestmark = pytest.mark.gpu

SHAPES = os.path.join(K.FIXTURES, "shapes", "benchmarks.json")
CLI = os.path.join(os.path.dirname(K.__file__), "bin", "ktune_b200")


def setup():
    hw = K.HardwareDescriptor.b200()
    bounds = open(os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")).read()
    sampler = P.calibrate(K.GemmInput(512, 512, 512), hw, bounds, 20000, 11)
    dist = P.GemmInputDistribution(shapes=P.gemm_shapes_from_table(SHAPES), fixed_fraction=0.25, m_hi=1024,
                                   n_hi=1024, k_hi=4096)
    return hw, bounds, sampler, dist


def rows_of(csv):
    return [",".join(line.split(",")[:14]) for line in csv.strip().splitlines()[1:]]


def test_shard_measures_the_sequential_sequence(cuda):
    hw, bounds, sampler, dist = setup()
    n = 96
    csv, stats = P.generate_sharded(sampler, dist, hw, bounds, n, 42, backend="b200", repetitions=1)
    seq, _, _ = P.generate_gemm(sampler, dist, hw, bounds, n, 42, backend="analytical")
    if stats["unlaunchable"] == 0:
        assert rows_of(csv) == rows_of(seq)
    g = np.array([float(line.split(",")[14]) for line in csv.strip().splitlines()[1:]])
    assert len(g) == n and np.all(g > 0)


def test_lpt_owner_matches_python_rule(cuda):
    rng = np.random.default_rng(3)
    costs = np.exp(rng.normal(20, 3, 500))
    for world in (1, 2, 3, 8):
        owner = P.shard_lpt_owner(costs, world)
        shards = P.shard_lpt(list(costs), world)
        for r, sh in enumerate(shards):
            assert all(owner[i] == r for i in sh)


def test_checkpoint_resume(cuda, tmp_path):
    hw, bounds, sampler, dist = setup()
    ck = str(tmp_path / "rank0.ckpt")
    n = 64
    t0 = time.perf_counter()
    csv1, _ = P.generate_sharded(sampler, dist, hw, bounds, n, 7, backend="b200", repetitions=1, checkpoint=ck)
    first = time.perf_counter() - t0
    lines = open(ck).read().splitlines()
    assert lines[0].startswith("ktune-shard-1 gemm") and len(lines) == n + 1
    t1 = time.perf_counter()
    csv2, _ = P.generate_sharded(sampler, dist, hw, bounds, n, 7, backend="b200", repetitions=1, checkpoint=ck)
    assert csv2 == csv1  # every value restored from the checkpoint, none re-measured
    assert time.perf_counter() - t1 < first
    # a torn trailing line (killed mid-write) is ignored and re-measured
    with open(ck, "a") as fh:
        fh.write("12")
    csv3, _ = P.generate_sharded(sampler, dist, hw, bounds, n, 7, backend="b200", repetitions=1, checkpoint=ck)
    assert rows_of(csv3) == rows_of(csv1)


def test_cli_shards_and_merge(cuda, tmp_path):
    hw, bounds, sampler, dist = setup()
    sp = tmp_path / "sampler.json"
    sp.write_text(sampler)
    hwp = os.path.join(K.FIXTURES, "hw", "b200.json")
    bp = os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")
    shards = []
    for r in range(2):
        out = tmp_path / f"shard{r}.txt"
        subprocess.run([CLI, "generate", "--hw", hwp, "--bounds", bp, "--sampler", str(sp), "--shapes", SHAPES,
                        "--shape-fraction", "0.25", "--backend", "b200", "--samples", "40", "--seed", "5",
                        "--shard", f"{r}/2", "--checkpoint", str(tmp_path / f"ck{r}"), "--out", str(out)],
                       check=True, capture_output=True)
        shards.append(str(out))
    merged = tmp_path / "dataset.csv"
    subprocess.run([CLI, "generate", "--merge", ",".join(shards), "--out", str(merged)], check=True,
                   capture_output=True)
    text = merged.read_text()
    seq = subprocess.run([CLI, "generate", "--hw", hwp, "--bounds", bp, "--sampler", str(sp), "--shapes", SHAPES,
                          "--shape-fraction", "0.25", "--backend", "analytical", "--samples", "40", "--seed", "5",
                          "--out", str(tmp_path / "seq.csv")], check=True, capture_output=True)
    assert seq.returncode == 0
    assert rows_of(text) == rows_of((tmp_path / "seq.csv").read_text())

"""Measured selection of a tuning tuple for one input (the re-measure half of
infer_gemm / infer_conv, pipeline.cpp:649-723).

``select_gemm`` ranks candidates by a cheap screening measurement (one timed
run each) instead of a model prediction, keeps the top_k, re-measures them
with more repetitions and returns the measured argmax (first max wins, like
pipeline.cpp:674-680).  It is used where no trained model is available yet;
the model-driven path is pipeline.infer_gemm.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import (ConvInput, ConvTuning, GemmInput, GemmTuning, HardwareDescriptor, InvalidArgument, enumerate_legal,
               measure)


@dataclass
class Selection:
    tuning: object
    gflops: float
    screened: int
    legal_space_size: int
    top: list


def _select(inp, space, cls, hw, extra, candidates, top_k, seed, mode, repetitions):
    rng = np.random.default_rng(seed)
    n = len(space)
    pick = sorted(rng.choice(n, size=min(candidates, n), replace=False).tolist()) if n else []
    cand = [cls(*map(int, space[i])) for i in pick]
    for t in extra:
        if t not in cand:
            cand.append(t)
    scored = []
    for t in cand:
        try:
            scored.append((measure(inp, t, hw, mode, repetitions=1, warmup=1), t))
        except InvalidArgument:
            continue  # illegal under hw or outside this build's launch envelope
    if not scored:
        raise RuntimeError("no launchable candidate for this input")
    scored.sort(key=lambda x: -x[0])
    top = []
    best = None
    for _, t in scored[:top_k]:
        g = measure(inp, t, hw, mode, repetitions=repetitions, warmup=1)
        top.append((t, g))
        if best is None or g > best[1]:
            best = (t, g)
    return Selection(best[0], best[1], len(scored), n, top)


def select_gemm(inp: GemmInput, hw: HardwareDescriptor, bounds_json: str | None = None, candidates: int = 2048,
                top_k: int = 16, seed: int = 0, mode: str = "fast", repetitions: int = 5, extra=()) -> Selection:
    space = enumerate_legal(inp, hw, bounds_json, as_array=True)
    return _select(inp, space, GemmTuning, hw, extra, candidates, top_k, seed, mode, repetitions)


def select_conv(inp: ConvInput, hw: HardwareDescriptor, bounds_json: str | None = None, candidates: int = 2048,
                top_k: int = 16, seed: int = 0, mode: str = "fast", repetitions: int = 5, extra=()) -> Selection:
    space = enumerate_legal(inp, hw, bounds_json, as_array=True)
    return _select(inp, space, ConvTuning, hw, extra, candidates, top_k, seed, mode, repetitions)

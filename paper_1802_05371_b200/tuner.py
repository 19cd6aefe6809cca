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


def _select(inp, space, cls, hw, extra, candidates, top_k, seed, mode, repetitions, key=None, accept=None):
    rng = np.random.default_rng(seed)
    if accept is not None and len(space):
        space = space[np.asarray([bool(accept(row)) for row in space])]
    if key is not None and len(space):
        # collapse tuples the executing family cannot tell apart (first legal
        # representative of each key, in enumeration order)
        _, first = np.unique(np.asarray([key(row) for row in space]), axis=0, return_index=True)
        space = space[np.sort(first)]
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
                top_k: int = 16, seed: int = 0, mode: str = "fast", repetitions: int = 5, extra=(), key=None,
                accept=None) -> Selection:
    space = enumerate_legal(inp, hw, bounds_json, as_array=True)
    return _select(inp, space, GemmTuning, hw, extra, candidates, top_k, seed, mode, repetitions, key, accept)


def select_conv(inp: ConvInput, hw: HardwareDescriptor, bounds_json: str | None = None, candidates: int = 2048,
                top_k: int = 16, seed: int = 0, mode: str = "fast", repetitions: int = 5, extra=(), key=None,
                accept=None) -> Selection:
    space = enumerate_legal(inp, hw, bounds_json, as_array=True)
    return _select(inp, space, ConvTuning, hw, extra, candidates, top_k, seed, mode, repetitions, key, accept)


# Fields the tensor-core families actually read (umma.cu / umma_conv.cu
# headers); the register-tile fields only shape the legality model.
def tc_gemm_key(row):
    return (row[2], row[3], row[4], row[5], row[1], row[7])  # m_l, n_l, u, k_s, n_s (raster), k_g


def tc_conv_key(row):
    return (row[4], row[5], row[6], row[7], row[8], row[9], row[11])  # k_l, p_l, q_l, n_l, u, c_s, c_g


def tc_conv_launchable(inp):
    """Cheap pre-filter mirroring conv_plan()'s launchability rules
    (umma_conv.cu): a 128-pixel tile whose 64-pixel atoms are contiguous
    (w, n) runs, UMMA_N filters, c_l = 1."""
    def ok(row):
        k_l, p_l, q_l, n_l, u, c_s, c_l = (int(x) for x in (row[4], row[5], row[6], row[7], row[8], row[9], row[10]))
        if p_l * q_l * n_l != 128 or k_l % 16 or not 16 <= k_l <= 256 or c_l != 1 or c_s > 2:
            return False
        if u not in (16, 32, 64, 128):
            return False
        return (n_l == inp.n_batch and q_l * n_l >= 64) or n_l >= 64
    return ok

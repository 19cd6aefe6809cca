"""Stream-K split of the tensor-core GEMM (k_g > 1): every CTA takes an
equal contiguous share of the (tile, k-block) iterations; split tiles are
folded by the last-arriving segments in two levels (groups of 8 segments,
then the groups), deterministically.  Checked against the double reference
on quantised inputs (tolerance of tests/test_umma_gpu.py), bit-stable
across runs and across CUDA-graph replays (the arrival counters reset)."""
import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K

pytestmark = pytest.mark.gpu


def tol(k):
    return max(1e-4, 6e-8 * k)


def operands(inp, seed):
    g = torch.Generator().manual_seed(seed)
    a = (torch.rand(inp.m * inp.k, generator=g) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(inp.k * inp.n, generator=g) * 2 - 1).to(torch.bfloat16)
    return a, b


def check(inp, tv, seed=0):
    a, b = operands(inp, seed)
    t = K.GemmTuning(*tv)
    c1 = K.execute_gemm(inp, t, a.cuda(), b.cuda()).cpu().numpy()
    c2 = K.execute_gemm(inp, t, a.cuda(), b.cuda()).cpu().numpy()
    ref = O.naive_gemm(inp.m, inp.n, inp.k, inp.trans_a, inp.trans_b, a.double().numpy(), b.double().numpy(), "f64")
    assert O.max_rel_error(c1, ref) < tol(inp.k)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))  # deterministic fold order
    return c1


@pytest.mark.parametrize("tv", [
    (8, 4, 128, 16, 128, 1, 1, 8),    # skinny: 20 tiles over 148 CTAs, tiles cut mid-K
    (8, 4, 128, 16, 64, 2, 1, 16),    # double-buffered accumulator
    (8, 4, 64, 16, 128, 1, 1, 32),    # UMMA_M = 64 tiles
])
def test_skinny_stream_k(cuda, tv):
    check(K.GemmInput(2560, 16, 2560, "bf16"), tv)


@pytest.mark.parametrize("k_g", [64, 256])
def test_ica_many_segments_two_level_fold(cuda, k_g):
    """One output tile split over up to 148 CTAs: > 8 segments, so the fold
    runs through the group level."""
    check(K.GemmInput(32, 32, 60000, "bf16", False, True), (8, 16, 64, 32, 128, 1, 1, k_g))


def test_pair_stream_k_ragged(cuda):
    check(K.GemmInput(1000, 200, 3000, "bf16"), (8, 8, 256, 64, 64, 1, 1, 8))


def test_stream_k_graph_replay(cuda):
    inp = K.GemmInput(32, 32, 60000, "bf16", False, True)
    t = K.GemmTuning(8, 16, 64, 32, 128, 1, 1, 256)
    a, b = operands(inp, 4)
    da, db = a.cuda(), b.cuda()
    c = torch.empty(inp.m * inp.n, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        K.execute_gemm(inp, t, da, db, c, stream=s.cuda_stream)
    torch.cuda.synchronize()
    want = c.cpu().numpy().copy()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        K.execute_gemm(inp, t, da, db, c, stream=s.cuda_stream)
    for _ in range(4):
        c.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(c.cpu().numpy().view(np.uint32), want.view(np.uint32))

"""Cluster split-K of the tensor-core GEMM: when k_g <= 8 and at least two
K slices of every output tile fit the SMs at once, a tile is one
thread-block cluster of C = 2/4/8 CTAs (a power of two <= k_g), each slice leaves its partial
tile in its own shared memory, and after one cluster barrier every rank
folds its share of the tile over the slices in rank order through DSMEM
(no global partials, counters or fold pass; no workspace).  Larger splits
keep stream-K (test_umma_streamk_gpu.py).  Same contract as
test_umma_gpu.py: quantised inputs, double reference, max(1e-4, 6e-8 K);
bit-stable across runs and CUDA-graph replays."""
import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K
from test_umma_gpu import quantised, tol

pytestmark = pytest.mark.gpu


def run_twice(inp, tv, seed=0):
    a = quantised(inp.m * inp.k, inp.dtype, seed).cuda()
    b = quantised(inp.k * inp.n, inp.dtype, seed + 1).cuda()
    t = K.GemmTuning(*tv)
    c1 = K.execute_gemm(inp, t, a, b).cpu().numpy()
    c2 = K.execute_gemm(inp, t, a, b).cpu().numpy()
    ref = O.naive_gemm(inp.m, inp.n, inp.k, inp.trans_a, inp.trans_b, a.cpu().double().numpy(),
                       b.cpu().double().numpy(), "f64")
    assert O.max_rel_error(c1, ref) < tol(inp.k)
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))  # rank-ordered fold
    return c1


@pytest.mark.parametrize("shape,tv,family", [
    # the timed skinny shape: 20 tiles x 4 slices
    ((2560, 16, 2560, False, False), (8, 4, 128, 16, 64, 1, 1, 4), "tcgen05-cluster4"),
    ((2560, 16, 2560, False, False), (8, 4, 128, 16, 128, 1, 1, 2), "tcgen05-cluster2"),
    # k_g = 8 over 20 tiles does not fit 8-CTA clusters: the largest that does
    ((2560, 16, 2560, False, False), (8, 4, 128, 16, 64, 1, 1, 8), "tcgen05-cluster4"),
    # few tiles: clusters of 8
    ((192, 96, 4000, False, True), (8, 8, 128, 32, 64, 1, 1, 8), "tcgen05-cluster8"),
    # k_g > 8 asks for more workers than one cluster holds: stream-K
    ((32, 32, 60000, False, True), (8, 16, 64, 16, 128, 1, 1, 32), "tcgen05-streamk"),
    # too many tiles for two slices each: stream-K
    ((2560, 512, 2560, False, False), (8, 4, 128, 16, 64, 1, 1, 4), "tcgen05-streamk"),
])
def test_schedule_and_parity(cuda, shape, tv, family):
    m, n, k, ta, tb = shape
    inp = K.GemmInput(m, n, k, "bf16", ta, tb)
    assert K.gemm_launch_info(inp, K.GemmTuning(*tv))["family"] == family
    run_twice(inp, tv)


@pytest.mark.parametrize("m", [1, 17, 63, 100, 129])
def test_m64_tiles_ragged_rows(cuda, m):
    """UMMA_M = 64: only lanes 0..15 of each TMEM quarter carry rows."""
    inp = K.GemmInput(m, 48, 1320, "bf16", False, True)
    tv = (8, 1, 64, 16, 64, 1, 1, 4)
    assert K.gemm_launch_info(inp, K.GemmTuning(*tv))["family"].startswith("tcgen05-cluster")
    run_twice(inp, tv, seed=m)


@pytest.mark.parametrize("n", [8, 20, 33])
def test_ragged_columns(cuda, n):
    """N not a multiple of 4 (scalar tail stores) and of the tile width."""
    inp = K.GemmInput(300, n, 1000, "bf16", False, False)
    run_twice(inp, (8, 4, 128, 16, 64, 1, 1, 8), seed=n)


@pytest.mark.parametrize("k", [128, 130, 200])
def test_fewer_k_blocks_than_slices(cuda, k):
    """kb_total < k_g: the cluster shrinks to what the k-blocks fill."""
    inp = K.GemmInput(256, 32, k, "bf16", False, True)
    run_twice(inp, (8, 4, 128, 32, 64, 1, 1, 8), seed=k)


@pytest.mark.parametrize("ta,tb", [(False, False), (True, True)])
def test_tf32_staged_operands(cuda, ta, tb):
    inp = K.GemmInput(320, 24, 3000, "tf32", ta, tb)
    tv = (8, 4, 128, 16, 32, 1, 1, 4)
    assert K.gemm_launch_info(inp, K.GemmTuning(*tv))["family"].startswith("tcgen05-cluster")
    run_twice(inp, tv)


def test_agrees_with_stream_k(cuda, monkeypatch):
    """Same tuple, both schedules: each within tolerance of the other."""
    inp = K.GemmInput(2560, 16, 2560, "bf16")
    tv = (8, 4, 128, 16, 64, 1, 1, 4)
    c_cluster = run_twice(inp, tv, seed=7)
    monkeypatch.setenv("KTUNE_TC_NO_CSPLIT", "1")
    assert K.gemm_launch_info(inp, K.GemmTuning(*tv))["family"] == "tcgen05-streamk"
    c_streamk = run_twice(inp, tv, seed=7)
    assert O.max_rel_error(c_cluster, c_streamk.astype(np.float64)) < tol(inp.k)


def test_graph_replay_bit_stable(cuda):
    inp = K.GemmInput(2560, 16, 2560, "bf16")
    t = K.GemmTuning(8, 4, 128, 16, 64, 1, 1, 4)
    a = quantised(inp.m * inp.k, "bf16", 3).cuda()
    b = quantised(inp.k * inp.n, "bf16", 4).cuda()
    c = torch.empty(inp.m * inp.n, device="cuda")
    s = torch.cuda.Stream()
    K.execute_gemm(inp, t, a, b, c, stream=s.cuda_stream)
    torch.cuda.synchronize()
    first = c.clone()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        K.execute_gemm(inp, t, a, b, c, stream=s.cuda_stream)
    for _ in range(5):
        c.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(c.view(torch.int32), first.view(torch.int32))

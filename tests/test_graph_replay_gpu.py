"""Split-K (k_g > 1) kernels replayed from a captured CUDA graph.

A captured launch keeps its publication token for every replay, so the
k_g fold must not trust flags left by the previous replay (the consumer
clears each flag it consumed).  Each replay gets fresh operands copied into
the captured buffers and is checked against the oracle: SIMT parity bitwise
(backends.cpp:320-325 fold order), tensor cores against the double
reference on the same bf16 inputs."""
import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K

pytestmark = pytest.mark.gpu


def _replay(inp, t, mode, dt_np, dt_torch, check, replays=4):
    a = torch.empty(inp.m * inp.k, dtype=dt_torch, device="cuda")
    b = torch.empty(inp.k * inp.n, dtype=dt_torch, device="cuda")
    c = torch.empty(inp.m * inp.n, dtype=torch.float32 if dt_torch != torch.float64 else torch.float64, device="cuda")
    st = torch.cuda.Stream()
    a.normal_(); b.normal_()
    with torch.cuda.stream(st):
        K.execute_gemm(inp, t, a, b, c, mode=mode, stream=st.cuda_stream)  # workspace allocated outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        K.execute_gemm(inp, t, a, b, c, mode=mode, stream=st.cuda_stream)
    rng = np.random.default_rng(3)
    for r in range(replays):
        an = rng.uniform(-1, 1, inp.m * inp.k).astype(dt_np)
        bn = rng.uniform(-1, 1, inp.k * inp.n).astype(dt_np)
        a.copy_(torch.from_numpy(an).to(dt_torch))
        b.copy_(torch.from_numpy(bn).to(dt_torch))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        check(a, b, c.cpu().numpy(), r)


@pytest.mark.parametrize("tup", [(2, 4, 64, 16, 32, 1, 1, 8), (4, 2, 32, 32, 16, 2, 2, 16), (2, 2, 16, 16, 8, 1, 4, 4)])
def test_simt_split_k_replay_bitwise(cuda, tup):
    inp = K.GemmInput(300, 48, 3000, "f32")
    t = K.GemmTuning(*tup)

    def check(a, b, got, r):
        want = O.execute_gemm(inp.m, inp.n, inp.k, 0, 0, t.values(), a.cpu().numpy(), b.cpu().numpy())
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (tup, r)

    _replay(inp, t, "parity", np.float32, torch.float32, check)


@pytest.mark.parametrize("tup", [(8, 4, 128, 16, 64, 1, 1, 8), (8, 1, 128, 64, 64, 2, 1, 4)])
def test_tensor_core_split_k_replay(cuda, tup):
    inp = K.GemmInput(384, 64, 4096, "bf16")
    t = K.GemmTuning(*tup)

    def check(a, b, got, r):
        an = a.float().cpu().numpy().astype(np.float64).reshape(inp.m, inp.k)
        bn = b.float().cpu().numpy().astype(np.float64).reshape(inp.k, inp.n)
        want = (an @ bn).ravel()
        err = np.max(np.abs(got - want)) / max(1.0, np.max(np.abs(want)))
        assert err < 1e-4, (tup, r, err)

    _replay(inp, t, "fast", np.float32, torch.bfloat16, check)

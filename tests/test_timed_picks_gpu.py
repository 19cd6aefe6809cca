"""Parity for exactly what bench.py times (the tuned picks of the driver's
BENCH line, at their full configured sizes).

tcgen05 family: against the double reference on identically quantised
inputs (bf16 exact; tf32 inputs pre-truncated to 10 mantissa bits), in the
reference metric max|got-ref|/max(|ref|,1) with the stated tolerance
max(1e-4, 6e-8 * K) (tests/test_umma_gpu.py).  For 8192^3 a seeded sample of
64 x 64 = 4096 output elements is checked; every other pick is
checked in full.  SIMT picks are bit-identical to the reference executor."""
import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K
from gpu_util import bitwise_equal, first_mismatch, run_gemm

pytestmark = pytest.mark.gpu


def tol(k):
    return max(1e-4, 6e-8 * k)


def quantised(n, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.rand(n, generator=g) * 2 - 1
    if dtype == "tf32":
        return (x.view(torch.int32) & ~0x1FFF).view(torch.float32)
    return x.to(torch.bfloat16)


def sampled_error(inp, got, a, b, rows, cols):
    A = a.double().numpy().reshape(inp.k, inp.m).T if inp.trans_a else a.double().numpy().reshape(inp.m, inp.k)
    B = b.double().numpy().reshape(inp.n, inp.k).T if inp.trans_b else b.double().numpy().reshape(inp.k, inp.n)
    ref = A[rows] @ B[:, cols]
    g = got.reshape(inp.m, inp.n)[np.ix_(rows, cols)]
    return float(np.abs(g - ref).max() / max(np.abs(ref).max(), 1.0))


@pytest.mark.parametrize("dtype,ta,tb,tv", [
    ("bf16", False, False, (8, 8, 256, 256, 128, 1, 1, 1)),   # square8192_bf16 pick (CTA pair)
    ("tf32", False, True, (8, 8, 256, 256, 64, 1, 1, 1)),     # square8192_tf32 pick (CTA pair, NT)
])
def test_square8192_pick(cuda, dtype, ta, tb, tv):
    n = 8192
    inp = K.GemmInput(n, n, n, dtype, ta, tb)
    a, b = quantised(n * n, dtype, 1), quantised(n * n, dtype, 2)
    c = K.execute_gemm(inp, K.GemmTuning(*tv), a.cuda(), b.cuda())
    torch.cuda.synchronize()
    rng = np.random.default_rng(8192)
    rows, cols = np.sort(rng.choice(n, 64, replace=False)), np.sort(rng.choice(n, 64, replace=False))
    assert sampled_error(inp, c.cpu().numpy(), a, b, rows, cols) < tol(n)


@pytest.mark.parametrize("shape,tv", [
    ((2560, 16, 2560, False, False), (8, 4, 128, 16, 128, 1, 1, 4)),   # deepbench_fprop16_bf16 pick
    ((32, 32, 60000, False, True), (8, 16, 64, 16, 128, 1, 1, 32)),    # ica32_bf16 pick (m_l = 64 tile)
])
def test_skinny_bf16_picks(cuda, shape, tv):
    m, n, k, ta, tb = shape
    inp = K.GemmInput(m, n, k, "bf16", ta, tb)
    a, b = quantised(m * k, "bf16", 3), quantised(k * n, "bf16", 4)
    c = K.execute_gemm(inp, K.GemmTuning(*tv), a.cuda(), b.cuda())
    torch.cuda.synchronize()
    ref = O.naive_gemm(m, n, k, ta, tb, a.double().numpy(), b.double().numpy(), "f64")
    assert O.max_rel_error(c.cpu().numpy(), ref) < tol(k)


@pytest.mark.parametrize("tv", [(4, 4, 32, 16, 32, 1, 2, 8), (2, 4, 32, 16, 32, 1, 1, 8)])
def test_headline_simt_picks_bitwise(cuda, tv):
    """The headline SIMT picks (TMA feed) at full size, PARITY bit-exact."""
    inp = K.GemmInput(2560, 16, 2560, "f32")
    t = K.GemmTuning(*tv)
    assert K.gemm_launch_info(inp, t, "parity")["family"] == "simt-tma"
    a, b = O.fill(5, inp.m * inp.k, inp.k * inp.n, "f32", True)
    got = run_gemm(inp, t, a, b)
    want = O.execute_gemm(inp.m, inp.n, inp.k, 0, 0, tv, a, b)
    assert bitwise_equal(got, want), first_mismatch(got, want)


@pytest.mark.parametrize("dims,tv", [
    ((16, 56, 56, 64, 64, 3, 3), (1, 1, 1, 8, 64, 1, 8, 16, 64, 1, 1, 1)),      # conv_resnet56_bf16 pick
    ((16, 7, 7, 512, 512, 3, 3), (1, 1, 1, 8, 64, 1, 8, 16, 128, 2, 1, 2)),     # conv_resnet13_bf16 pick
])
def test_conv_bf16_picks(cuda, dims, tv):
    cin = K.ConvInput(*dims, "bf16")
    ni, nf, _ = cin.sizes()
    img, flt = quantised(ni, "bf16", 5), quantised(nf, "bf16", 6)
    out = K.execute_conv(cin, K.ConvTuning(*tv), img.cuda(), flt.cuda())
    torch.cuda.synchronize()
    ref = O.direct_conv(list(dims), img.double().numpy(), flt.double().numpy(), "f64")
    assert O.max_rel_error(out.cpu().numpy(), ref) < tol(dims[4] * dims[5] * dims[6])

"""K4c on the B200: implicit-GEMM convolution on the tcgen05 tensor cores
(bf16 / f16 inputs, fp32 accumulate and output).

Same contract as the tensor-core GEMM (test_umma_gpu.py): the reference has
no 16-bit executor, so inputs are quantised to the operand type on the host
and the direct seven-loop convolution of test_backends.cpp:38-66 in double
(oracle_direct_conv_f64) is the reference; tolerance in the reference's
metric max|got-ref|/max(|ref|,1) is max(1e-4, 6e-8 * CRS).  Layouts are the
reference's: I = C,H,W,N  F = C,R,S,K  O = K,P,Q,N (backends.cpp:345-353).
At full ResNet size the check is against torch's fp32 convolution of the same
quantised tensors (cuDNN, TF32 disabled)."""
import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K

pytestmark = pytest.mark.gpu

TD = {"bf16": torch.bfloat16, "f16": torch.float16}


def tol(crs):
    return max(1e-4, 6e-8 * crs)


def quantised(n, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    return (torch.rand(n, generator=g) * 2 - 1).to(TD[dtype])


def operands(inp, seed):
    ni, nf, _ = inp.sizes()
    return quantised(ni, inp.dtype, seed), quantised(nf, inp.dtype, seed + 1)


def run(inp, t, seed=0):
    img, flt = operands(inp, seed)
    out = K.execute_conv(inp, t, img.cuda(), flt.cuda())
    torch.cuda.synchronize()
    dims = [inp.n_batch, inp.p, inp.q, inp.k_filters, inp.c, inp.r, inp.s]
    ref = O.direct_conv(dims, img.double().numpy(), flt.double().numpy(), "f64")
    return out.cpu().numpy(), ref


def T(k_l, p_l, q_l, n_l, u, c_s=1, c_g=1):
    return K.ConvTuning(1, 1, 1, 1, k_l, p_l, q_l, n_l, u, c_s, 1, c_g)


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
def test_dtypes(cuda, dtype):
    inp = K.ConvInput(16, 8, 8, 64, 16, 3, 3, dtype)
    got, ref = run(inp, T(64, 1, 8, 16, 64))
    assert O.max_rel_error(got, ref) < tol(16 * 9)


@pytest.mark.parametrize("k_l", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("u", [16, 32, 64, 128])
def test_tile_shapes(cuda, k_l, u):
    # ragged in every direction: P, Q against the pixel tile, K against k_l,
    # C = 13 against u (TMA zero fill)
    inp = K.ConvInput(8, 5, 7, 88, 13, 3, 3, "bf16")
    got, ref = run(inp, T(k_l, 2, 8, 8, u), seed=k_l + u)
    assert O.max_rel_error(got, ref) < tol(117)


@pytest.mark.parametrize("pqn", [(1, 8, 16), (2, 4, 16), (1, 2, 64), (2, 1, 64), (1, 1, 128)])
def test_pixel_tile_factorisations(cuda, pqn):
    # n_l == N = 16, or n_l >= 64 (tiles over-cover the batch; the extra
    # pixels read neighbouring data and are dropped by the epilogue)
    p_l, q_l, n_l = pqn
    inp = K.ConvInput(16, 6, 9, 32, 8, 3, 2, "bf16")
    got, ref = run(inp, T(32, p_l, q_l, n_l, 32), seed=p_l * 100 + q_l)
    assert O.max_rel_error(got, ref) < tol(48)


@pytest.mark.parametrize("c_g", [2, 4, 8])
def test_split_crs_fixup(cuda, c_g):
    inp = K.ConvInput(16, 6, 6, 64, 64, 3, 3, "bf16")
    got, ref = run(inp, T(64, 1, 8, 16, 32, 1, c_g), seed=c_g)
    assert O.max_rel_error(got, ref) < tol(576)
    # the same workspace reused by the next launch stays correct (tokens)
    got2, _ = run(inp, T(64, 1, 8, 16, 32, 1, c_g), seed=c_g)
    assert np.array_equal(got, got2)


def test_double_buffered_accumulator_and_many_units(cuda):
    # more units than SMs: the persistent loop cycles both TMEM buffers
    inp = K.ConvInput(16, 20, 20, 32, 8, 3, 3, "bf16")
    a, ref = run(inp, T(32, 1, 8, 16, 16, 2))
    b, _ = run(inp, T(32, 1, 8, 16, 16, 1))
    assert O.max_rel_error(a, ref) < tol(72)
    assert np.array_equal(a, b)  # same MMA sequence per tile either way


def test_one_by_one_conv_equals_tensor_core_gemm(cuda):
    # R = S = 1: O[k][pqn] = sum_c F[c][k] I[c][pqn] is the GEMM F^T I
    inp = K.ConvInput(16, 4, 8, 64, 128, 1, 1, "bf16")
    img, flt = operands(inp, 3)
    out = K.execute_conv(inp, T(64, 1, 8, 16, 64), img.cuda(), flt.cuda())
    g = K.GemmInput(64, 4 * 8 * 16, 128, "bf16", True, False)  # A = F (C x K) transposed
    c = K.execute_gemm(g, K.GemmTuning(8, 8, 128, 64, 64, 1, 1, 1), flt.cuda(), img.cuda())
    torch.cuda.synchronize()
    assert O.max_rel_error(out.cpu().numpy(), c.cpu().numpy()) < 1e-5


def test_resnet_layer_against_torch(cuda):
    """configs[2]: N=16, C=64, 56x56 (pad 1 -> H=W=58 stored), K=64, 3x3."""
    inp = K.ConvInput(16, 56, 56, 64, 64, 3, 3, "bf16")
    img, flt = operands(inp, 11)
    out = K.execute_conv(inp, T(64, 1, 8, 16, 64, 2), img.cuda(), flt.cuda())
    x = img.cuda().float().view(64, 58, 58, 16).permute(3, 0, 1, 2)  # N,C,H,W
    w = flt.cuda().float().view(64, 3, 3, 64).permute(3, 0, 1, 2)    # K,C,R,S
    prev = torch.backends.cudnn.allow_tf32
    torch.backends.cudnn.allow_tf32 = False
    try:
        ref = torch.nn.functional.conv2d(x.double(), w.double())  # N,K,P,Q
    finally:
        torch.backends.cudnn.allow_tf32 = prev
    ref = ref.permute(1, 2, 3, 0).reshape(-1).cpu().numpy()       # K,P,Q,N
    assert O.max_rel_error(out.cpu().numpy(), ref) < tol(576)


def test_launchability_rules(cuda):
    inp = K.ConvInput(16, 8, 8, 64, 16, 3, 3, "bf16")
    img, flt = operands(inp, 0)
    img, flt = img.cuda(), flt.cuda()
    with pytest.raises(K.Unsupported, match="128 output pixels"):
        K.execute_conv(inp, T(64, 1, 4, 16, 64), img, flt)
    with pytest.raises(K.Unsupported, match="k_l must be"):
        K.execute_conv(inp, T(8, 1, 8, 16, 64), img, flt)
    with pytest.raises(K.Unsupported, match="u must be"):
        K.execute_conv(inp, T(64, 1, 8, 16, 8), img, flt)
    with pytest.raises(K.Unsupported, match="c_l must be 1"):
        K.execute_conv(inp, K.ConvTuning(1, 1, 1, 1, 64, 1, 8, 16, 64, 1, 2, 1), img, flt)
    with pytest.raises(K.Unsupported, match="contiguous"):  # n_l < N
        K.execute_conv(inp, T(64, 1, 16, 8, 64), img, flt)
    with pytest.raises(K.Unsupported, match="contiguous"):  # q_l * n_l < 64
        K.execute_conv(inp, T(64, 4, 2, 16, 64), img, flt)
    bad = K.ConvInput(12, 8, 8, 64, 16, 3, 3, "bf16")  # batch not a multiple of 8
    i2, f2 = operands(bad, 0)
    with pytest.raises(K.Unsupported, match="multiple of 8"):
        K.execute_conv(bad, T(64, 1, 8, 16, 64), i2.cuda(), f2.cuda())


@pytest.mark.parametrize("k", [174, 87, 20])
def test_filter_counts_not_multiple_of_8_staged(cuda, k):
    """DeepBench speaker conv11/12 (K = 174 / 87): the filter tensor is staged
    into a copy with a 16-byte row pitch (execute_conv runs any shape)."""
    inp = K.ConvInput(16, 8, 8, k, 32, 3, 3, "bf16")
    got, ref = run(inp, T(64, 1, 8, 16, 64))
    assert O.max_rel_error(got, ref) < tol(32 * 9)

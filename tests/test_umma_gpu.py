"""K4 on the B200: the tcgen05/TMEM/TMA tensor-core GEMM family (bf16, f16,
tf32 inputs; fp32 accumulate and output).

The reference has no 16-bit or tf32 executor (param_space.hpp:15,
backends.cpp:504-506), so parity is stated against execute_gemm<double> on
identically quantised inputs: inputs are rounded to the operand type on the
host first (bf16/f16 exactly representable; tf32 inputs pre-truncated to 10
mantissa bits so truncating and rounding hardware agree), then the naive
double GEMM of test_backends.cpp:17-34 is the reference.  Stated tolerance
in the reference's metric max|got-ref|/max(|ref|,1): max(1e-4, 6e-8 * K).
The tensor cores accumulate in fp32 but align/truncate products inside each
MMA k-slice, so the error grows with K (measured 3.6e-4 at K = 8192, where
cuBLAS SGEMM on the same fp32-upcast inputs gives 7e-5 and cuBLAS bf16 with
bf16 output 3.8e-3)."""
import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K

pytestmark = pytest.mark.gpu

TOL = 1e-4


def tol(k):
    return max(1e-4, 6e-8 * k)
TD = {"bf16": torch.bfloat16, "f16": torch.float16, "tf32": torch.float32}


def quantised(n, dtype, seed):
    g = torch.Generator().manual_seed(seed)
    x = torch.rand(n, generator=g) * 2 - 1
    if dtype == "tf32":
        x = (x.view(torch.int32) & ~0x1FFF).view(torch.float32)  # exact tf32 values
        return x
    return x.to(TD[dtype])


def run(inp, t, seed=0):
    a = quantised(inp.m * inp.k, inp.dtype, seed)
    b = quantised(inp.k * inp.n, inp.dtype, seed + 1)
    c = K.execute_gemm(inp, t, a.cuda(), b.cuda())
    torch.cuda.synchronize()
    ref = O.naive_gemm(inp.m, inp.n, inp.k, inp.trans_a, inp.trans_b, a.double().numpy(), b.double().numpy(), "f64")
    return c.cpu().numpy(), ref


@pytest.mark.parametrize("dtype", ["bf16", "f16", "tf32"])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_layouts_and_dtypes(cuda, dtype, ta, tb):
    u = 64 if dtype != "tf32" else 32
    inp = K.GemmInput(256, 384, 512, dtype, ta, tb)
    # tf32 MN-major operands are staged transposed into K-major workspace copies
    got, ref = run(inp, K.GemmTuning(8, 8, 128, 128, u, 1, 1, 1))
    assert O.max_rel_error(got, ref) < tol(inp.k)


@pytest.mark.parametrize("n_l", [16, 32, 64, 128, 256])
@pytest.mark.parametrize("u", [32, 64, 128])
def test_tile_shapes_bf16(cuda, n_l, u):
    # ragged against every tile extent; leading dimensions stay multiples of
    # 16 bytes (unaligned ones are staged: test_unaligned_leading_dimensions_staged)
    inp = K.GemmInput(300, 336, 712, "bf16", False, False)
    got, ref = run(inp, K.GemmTuning(8, 8, 128, n_l, u, 1, 1, 1), seed=n_l + u)
    assert O.max_rel_error(got, ref) < tol(inp.k)


@pytest.mark.parametrize("k_g", [2, 3, 8])
def test_split_k_fixup(cuda, k_g):
    kg = 4 if k_g == 3 else k_g  # tuple values are powers of two
    inp = K.GemmInput(192, 96, 4000, "bf16", False, True)
    got, ref = run(inp, K.GemmTuning(8, 8, 128, 32, 64, 1, 1, kg), seed=k_g)
    assert O.max_rel_error(got, ref) < tol(inp.k)
    # reuse of the same workspace stays correct (per-launch tokens)
    got2, _ = run(inp, K.GemmTuning(8, 8, 128, 32, 64, 1, 1, kg), seed=k_g)
    assert np.array_equal(got, got2)


def test_skinny_deepbench_bf16(cuda):
    inp = K.GemmInput(2560, 16, 2560, "bf16")
    got, ref = run(inp, K.GemmTuning(8, 8, 128, 16, 64, 1, 1, 4), seed=5)
    assert O.max_rel_error(got, ref) < tol(inp.k)


def test_large_square_sampled(cuda):
    """BASELINE configs[3] 8192^3 bf16: full device run, 4096 sampled
    output elements checked against float64 dot products."""
    n = 8192
    inp = K.GemmInput(n, n, n, "bf16")
    g = torch.Generator(device="cuda").manual_seed(3)
    a = (torch.rand(n * n, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    b = (torch.rand(n * n, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16)
    c = K.execute_gemm(inp, K.GemmTuning(8, 8, 128, 256, 64, 1, 1, 1), a, b)
    rng = np.random.default_rng(0)
    rows = torch.from_numpy(rng.integers(0, n, 4096)).cuda()
    cols = torch.from_numpy(rng.integers(0, n, 4096)).cuda()
    A = a.view(n, n).double()
    B = b.view(n, n).double()
    ref = (A[rows] * B[:, cols].T).sum(1)
    got = c.view(n, n)[rows, cols].double()
    err = ((got - ref).abs() / ref.abs().clamp(min=1.0)).max().item()
    assert err < tol(n)


def test_unsupported_tuples_fail_loudly(cuda):
    a = torch.zeros(64 * 64, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(K.Unsupported, match="m_l"):
        K.execute_gemm(K.GemmInput(64, 64, 64, "bf16"), K.GemmTuning(8, 8, 32, 64, 64, 1, 1, 1), a, a)
    with pytest.raises(K.Unsupported, match="k_l"):
        K.execute_gemm(K.GemmInput(64, 64, 64, "bf16"), K.GemmTuning(8, 8, 128, 64, 64, 1, 2, 1), a, a)


@pytest.mark.parametrize("m,n,k,ta,tb", [
    (300, 333, 700, False, False),   # N and K not multiples of 8 (16 bytes of bf16): both staged padded
    (257, 129, 1001, True, False),
    (100, 37, 515, False, True),
    (33, 17, 9999, True, True),
])
def test_unaligned_leading_dimensions_staged(cuda, m, n, k, ta, tb):
    """execute_gemm's any-shape contract (backends.cpp:228-329): operands
    whose leading dimension TMA cannot stride are copied into padded
    workspace copies first."""
    inp = K.GemmInput(m, n, k, "bf16", ta, tb)
    got, ref = run(inp, K.GemmTuning(8, 8, 128, 64, 64, 1, 1, 2))
    assert O.max_rel_error(got, ref) < tol(k)


@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (True, True)])
def test_tf32_mn_major_square(cuda, ta, tb):
    inp = K.GemmInput(512, 384, 640, "tf32", ta, tb)
    got, ref = run(inp, K.GemmTuning(8, 8, 256, 128, 32, 1, 1, 1))
    assert O.max_rel_error(got, ref) < tol(640)

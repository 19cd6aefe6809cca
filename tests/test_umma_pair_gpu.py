"""K4 CTA-pair tiles (m_l = 256): tcgen05.mma.cta_group::2 across a cluster of
two CTAs, each staging 128 rows of A and half of the tile's B columns.

Same contract as test_umma_gpu.py (quantised inputs, double reference,
tolerance max(1e-4, 6e-8 K)); ragged M / N / K against the 256-row pair tile,
every operand layout, split-K across pairs, the persistent loop over more
tiles than pairs, and the pair result equal to the single-CTA result."""
import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K
from test_umma_gpu import quantised, run, tol

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_pair_layouts(cuda, dtype, ta, tb):
    inp = K.GemmInput(512, 384, 640, dtype, ta, tb)
    got, ref = run(inp, K.GemmTuning(8, 8, 256, 128, 64, 1, 1, 1))
    assert O.max_rel_error(got, ref) < tol(inp.k)


def test_pair_tf32(cuda):
    inp = K.GemmInput(512, 256, 512, "tf32", False, True)
    got, ref = run(inp, K.GemmTuning(8, 8, 256, 256, 32, 1, 1, 1))
    assert O.max_rel_error(got, ref) < tol(inp.k)


@pytest.mark.parametrize("n_l", [32, 64, 128, 256])
def test_pair_ragged(cuda, n_l):
    inp = K.GemmInput(300, 200, 424, "bf16")  # M not a multiple of 256 (second CTA partly idle)
    got, ref = run(inp, K.GemmTuning(8, 8, 256, n_l, 64, 1, 1, 1), seed=n_l)
    assert O.max_rel_error(got, ref) < tol(inp.k)


@pytest.mark.parametrize("k_g", [2, 4])
@pytest.mark.parametrize("k_s", [1, 2])
def test_pair_split_k_and_persistent(cuda, k_g, k_s):
    inp = K.GemmInput(2048, 512, 2048, "bf16")  # 8 x 4 pair tiles x k_g units > 74 pairs for k_g = 4
    got, ref = run(inp, K.GemmTuning(8, 16, 256, 128, 64, k_s, 1, k_g), seed=k_g)
    assert O.max_rel_error(got, ref) < tol(inp.k)


def test_pair_equals_single_cta(cuda):
    inp = K.GemmInput(512, 256, 1024, "bf16")
    a = quantised(inp.m * inp.k, "bf16", 5).cuda()
    b = quantised(inp.k * inp.n, "bf16", 6).cuda()
    c1 = K.execute_gemm(inp, K.GemmTuning(8, 8, 128, 256, 64, 1, 1, 1), a, b)
    c2 = K.execute_gemm(inp, K.GemmTuning(8, 8, 256, 256, 64, 1, 1, 1), a, b)
    torch.cuda.synchronize()
    # same MMA k-order per output element; the pair only moves rows between SMs
    assert torch.equal(c1, c2)


def test_pair_rejects_narrow_tiles(cuda):
    a = torch.zeros(256 * 256, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(K.Unsupported, match="multiple of 32"):
        K.execute_gemm(K.GemmInput(256, 256, 256, "bf16"), K.GemmTuning(8, 1, 256, 16, 64, 1, 1, 1), a, a)

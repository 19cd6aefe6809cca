"""K4 with m_l = 64 (UMMA_M = 64): for M <= 64 a 128-row tile is three
quarters TMA zero fill; the 64-row tile stages only real rows.  TMEM holds
rows 16q..16q+15 in lanes 32q..32q+15 of warp quarter q.  Same contract as
test_umma_gpu.py (quantised inputs, double reference, max(1e-4, 6e-8 K))."""
import pytest

import oracle_libs as O
import paper_1802_05371_b200 as K
from test_umma_gpu import run, tol

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["bf16", "f16"])
@pytest.mark.parametrize("ta,tb", [(False, False), (False, True), (True, False), (True, True)])
def test_m64_layouts(cuda, dtype, ta, tb):
    inp = K.GemmInput(192, 128, 512, dtype, ta, tb)
    got, ref = run(inp, K.GemmTuning(8, 8, 64, 64, 64, 1, 1, 1))
    assert O.max_rel_error(got, ref) < tol(inp.k)


def test_m64_tf32(cuda):
    inp = K.GemmInput(64, 96, 512, "tf32", False, True)
    got, ref = run(inp, K.GemmTuning(8, 8, 64, 32, 32, 1, 1, 1))
    assert O.max_rel_error(got, ref) < tol(inp.k)


@pytest.mark.parametrize("m", [1, 17, 32, 63, 64, 100])
def test_m64_ragged_rows(cuda, m):
    inp = K.GemmInput(m, 48, 320, "bf16", False, True)
    got, ref = run(inp, K.GemmTuning(8, 1, 64, 16, 64, 1, 1, 1), seed=m)
    assert O.max_rel_error(got, ref) < tol(inp.k)


@pytest.mark.parametrize("k_g", [2, 8, 32])
@pytest.mark.parametrize("k_s", [1, 2])
def test_m64_split_k_ica(cuda, k_g, k_s):
    inp = K.GemmInput(32, 32, 6000, "bf16", False, True)  # ICA-shaped
    got, ref = run(inp, K.GemmTuning(8, 1, 64, 16, 128, k_s, 1, k_g), seed=k_g)
    assert O.max_rel_error(got, ref) < tol(inp.k)

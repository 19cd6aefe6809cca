"""FAST-mode wave balance of the SIMT k_g split (launch.cu balanced_span):
FAST may re-slice K into more slices than k_g so the blocks spread evenly
over the SMs; the tile geometry stays the tuple's, the summation order
changes (FAST's bound, as tests/test_gemm_gpu.py: max(1e-5, 2e-8 K) against
the double-precision product for fp32, 1e-12 for fp64).  PARITY keeps the
reference's k_g slices and stays bit-exact."""
import numpy as np
import pytest

import oracle_libs as O
import paper_1802_05371_b200 as K
from gpu_util import bitwise_equal, first_mismatch, run_gemm

pytestmark = pytest.mark.gpu


def fast_bound(inp):
    return max(1e-5, 2e-8 * inp.k) if inp.dtype == "f32" else 1e-12


def exact(inp, a, b):
    return O.naive_gemm(inp.m, inp.n, inp.k, inp.trans_a, inp.trans_b, a.astype(np.float64), b.astype(np.float64),
                        "f64")


def test_headline_pick_rebalanced(cuda, monkeypatch):
    inp = K.GemmInput(2560, 16, 2560, "f32")
    t = K.GemmTuning(2, 4, 32, 16, 32, 1, 1, 8)
    # 80 tiles x 8 slices = 640 blocks (4.3 per SM): FAST runs 9 slices (720
    # blocks, never more per SM than the tuple's own grid), PARITY keeps 8
    assert K.gemm_launch_info(inp, t, "fast")["grid"][2] == 9
    assert K.gemm_launch_info(inp, t, "parity")["grid"][2] == 8
    monkeypatch.setenv("KTUNE_SIMT_NO_BALANCE", "1")
    assert K.gemm_launch_info(inp, t, "fast")["grid"][2] == 8
    monkeypatch.delenv("KTUNE_SIMT_NO_BALANCE")
    a, b = O.fill(11, inp.m * inp.k, inp.k * inp.n, "f32", True)
    got = run_gemm(inp, t, a, b, "fast")
    assert O.max_rel_error(got, exact(inp, a, b)) < fast_bound(inp)
    par = run_gemm(inp, t, a, b, "parity")
    want = O.execute_gemm(inp.m, inp.n, inp.k, 0, 0, t.values(), a, b)
    assert bitwise_equal(par, want), first_mismatch(par, want)


@pytest.mark.parametrize("nz", [3, 9, 13, 40])
def test_forced_slice_counts(cuda, monkeypatch, nz):
    """Any slice count, ragged last slice included, stays within tolerance."""
    monkeypatch.setenv("KTUNE_SIMT_NZ", str(nz))
    inp = K.GemmInput(300, 40, 2001, "f32")
    t = K.GemmTuning(2, 2, 32, 16, 16, 1, 1, 4)
    a, b = O.fill(nz, inp.m * inp.k, inp.k * inp.n, "f32", True)
    got = run_gemm(inp, t, a, b, "fast")
    assert O.max_rel_error(got, exact(inp, a, b)) < fast_bound(inp)


def test_random_shapes_fast_tolerance(cuda):
    rng = np.random.default_rng(17)
    for trial in range(24):
        dt = "f32" if trial % 4 else "f64"
        kg = int(rng.choice([2, 4, 8, 16]))
        t = K.GemmTuning(2, 2, 16, 16, 16, 1, int(rng.choice([1, 2])), kg)
        inp = K.GemmInput(int(rng.integers(16, 700)), int(rng.integers(1, 70)), int(rng.integers(64, 5000)), dt,
                          bool(trial % 2), bool(trial % 3 == 0))
        a, b = O.fill(100 + trial, inp.m * inp.k, inp.k * inp.n, dt, True)
        got = run_gemm(inp, t, a, b, "fast")
        assert O.max_rel_error(got, exact(inp, a, b)) < fast_bound(inp), (inp, t)


@pytest.mark.parametrize("kl", [1, 2, 4])
def test_unaligned_slices_realigned_for_tma(cuda, kl):
    """ICA 32x32x60000 at k_g = 64: the reference's slices start every 938
    columns (4-byte aligned), which no vector / TMA feed can read; FAST
    re-slices K so every k_l group start is 16-byte aligned and the TMA feed
    runs; PARITY keeps the reference's slices (cp.async, bit-exact)."""
    inp = K.GemmInput(32, 32, 60000, "f32", False, True)
    t = K.GemmTuning(4, 1, 32, 8, 32, 4, kl, 64)
    fast = K.gemm_launch_info(inp, t, "fast")
    assert fast["family"] == "simt-tma", fast
    assert K.gemm_launch_info(inp, t, "parity")["grid"][2] == 64
    a, b = O.fill(29, inp.m * inp.k, inp.k * inp.n, "f32", True)
    got = run_gemm(inp, t, a, b, "fast")
    assert O.max_rel_error(got, exact(inp, a, b)) < fast_bound(inp)
    par = run_gemm(inp, t, a, b, "parity")
    want = O.execute_gemm(inp.m, inp.n, inp.k, 0, 1, t.values(), a, b)
    assert bitwise_equal(par, want), first_mismatch(par, want)


@pytest.mark.parametrize("fold,nz", [("auto", 128), ("auto", 40), ("atomic", 4), ("ordered", 64)])
def test_fast_merge_by_reduction(cuda, monkeypatch, fold, nz):
    """FAST merges >= 16 k_g slices with L2 reductions into a zeroed
    accumulator in the counter region; the last arriver stores C and
    re-zeroes it, so back-to-back launches on the same workspace (and the
    ordered fold afterwards) stay correct.  PARITY is never affected."""
    monkeypatch.setenv("KTUNE_SIMT_NZ", str(nz))
    if fold != "auto":
        monkeypatch.setenv("KTUNE_SIMT_FOLD", fold)
    inp = K.GemmInput(32, 32, 60000, "f32", False, True)
    t = K.GemmTuning(4, 4, 32, 32, 32, 1, 1, 64)
    a, b = O.fill(nz, inp.m * inp.k, inp.k * inp.n, "f32", True)
    want = exact(inp, a, b)
    for _ in range(3):
        got = run_gemm(inp, t, a, b, "fast")
        assert O.max_rel_error(got, want) < fast_bound(inp)
    monkeypatch.setenv("KTUNE_SIMT_FOLD", "ordered")
    got = run_gemm(inp, t, a, b, "fast")
    assert O.max_rel_error(got, want) < fast_bound(inp)
    monkeypatch.delenv("KTUNE_SIMT_NZ")
    par = run_gemm(inp, t, a, b, "parity")
    ref = O.execute_gemm(inp.m, inp.n, inp.k, 0, 1, t.values(), a, b)
    assert bitwise_equal(par, ref), first_mismatch(par, ref)

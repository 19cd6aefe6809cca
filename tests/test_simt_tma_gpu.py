"""K1t on the B200: the TMA-fed SIMT GEMM (simt_tma.cuh).

The TMA feed changes only how operand tiles reach shared memory, so PARITY
must stay bit-identical to the reference execute_gemm<float>
(backends.cpp:228-329) and to the cp.async kernel on every eligible tuple:
all four layouts, ragged tiles (TMA zero fill at the tensor edges), k_l
groups whose last box runs into the next group's range, k_g slices folded by
the last-arriving slice, thread counts that are not whole warps, and CUDA
graph replays (the fold's ticket words must reset)."""
import os

import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K
from gpu_util import bitwise_equal, dev, first_mismatch, run_gemm

pytestmark = pytest.mark.gpu


def both_feeds(inp, t, a, b, mode="parity"):
    out = {}
    for feed in ("1", "0"):
        os.environ["KTUNE_SIMT_TMA"] = feed
        try:
            out[feed] = run_gemm(inp, t, a, b, mode)
        finally:
            os.environ.pop("KTUNE_SIMT_TMA", None)
    return out["1"], out["0"]


CASES = [
    # (m, n, k, ta, tb), tuple (m_s, n_s, m_l, n_l, u, k_s, k_l, k_g); every
    # k_g / k_l slice of a k-contiguous operand starts on a 16-byte boundary
    ((2560, 16, 2560, False, False), (4, 4, 32, 16, 32, 1, 2, 8)),   # the headline pick family
    ((2560, 16, 2560, False, False), (4, 2, 64, 16, 32, 1, 1, 8)),
    ((2560, 16, 2560, True, False), (4, 4, 32, 16, 32, 1, 2, 8)),
    ((32, 32, 6016, False, True), (2, 4, 32, 32, 32, 1, 2, 16)),     # ICA-style, B k-contiguous
    ((100, 36, 1000, False, False), (2, 2, 32, 16, 64, 2, 1, 2)),    # ragged rows/cols/steps, two 128 B boxes
    ((100, 36, 1008, True, True), (4, 2, 16, 8, 16, 4, 1, 4)),       # w = 16 -> 64 B swizzle, k_s = 4
    ((64, 64, 248, False, True), (1, 2, 8, 8, 8, 1, 1, 2)),          # w = 8 -> 32 B swizzle, 32 threads
    ((68, 20, 517, True, False), (2, 1, 8, 4, 16, 2, 1, 4)),         # 16 threads: a partial warp; any K
    ((44, 12, 1208, False, False), (1, 1, 4, 4, 64, 2, 1, 2)),       # 4-row boxes, 16 threads
    ((256, 128, 384, False, False), (8, 4, 64, 64, 8, 1, 1, 1)),     # no split
    ((512, 512, 512, False, False), (4, 4, 64, 64, 16, 1, 1, 1)),
]


@pytest.mark.parametrize("case", CASES)
def test_tma_feed_is_bitwise(cuda, case):
    (m, n, k, ta, tb), tv = case
    inp = K.GemmInput(m, n, k, "f32", ta, tb)
    t = K.GemmTuning(*tv)
    assert K.gemm_launch_info(inp, t, "parity")["family"] == "simt-tma", case
    a, b = O.fill(sum(tv) + m, m * k, k * n, "f32", True)
    got, cp = both_feeds(inp, t, a, b)
    assert bitwise_equal(got, cp), (case, first_mismatch(got, cp))
    if m * n * k <= 40_000_000:
        want = O.execute_gemm(m, n, k, ta, tb, tv, a, b, "f32")
        assert bitwise_equal(got, want), (case, first_mismatch(got, want))
    fast, fast_cp = both_feeds(inp, t, a, b, mode="fast")
    if K.gemm_launch_info(inp, t, "fast")["grid"][2] < 16:
        assert bitwise_equal(fast, fast_cp), (case, first_mismatch(fast, fast_cp))
    else:  # FAST merges >= 16 slices by L2 reductions: arrival order, not bitwise
        assert O.max_rel_error(fast, fast_cp.astype(np.float64)) < 1e-5, case
    rows = min(m, 64)
    if not ta:
        # FAST (FFMA) within the reference's 1e-5 (test_backends.cpp:142), or
        # for long reductions within 2x the reference executor's own rounding
        # error on the same inputs (PARITY output = the reference's result)
        ref = O.naive_gemm(rows, n, k, 0, int(tb), a[: rows * k], b)
        own = O.max_rel_error(got[: rows * n], ref)
        assert O.max_rel_error(fast[: rows * n], ref) < max(1e-5, 2 * own)


def test_tma_graph_replay_resets_tickets(cuda):
    """The last-arriving slice clears each tile's ticket word, so replaying a
    captured launch (same tag every replay) keeps folding correctly."""
    inp = K.GemmInput(2560, 16, 2560, "f32")
    t = K.GemmTuning(4, 4, 32, 16, 32, 1, 2, 8)
    a, b = O.fill(3, inp.m * inp.k, inp.k * inp.n, "f32", True)
    da, db = dev(a), dev(b)
    c = torch.empty(inp.m * inp.n, device="cuda:0")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        K.execute_gemm(inp, t, da, db, c, mode="parity", stream=s.cuda_stream)
    torch.cuda.synchronize()
    want = c.cpu().numpy().copy()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        K.execute_gemm(inp, t, da, db, c, mode="parity", stream=s.cuda_stream)
    for _ in range(5):
        c.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert bitwise_equal(c.cpu().numpy(), want)


def test_tma_unaligned_falls_back_identically(cuda):
    """Leading dimensions that are not 16-byte multiples stay on the cp.async
    kernel (TMA strides must be 16-byte multiples); results are the same."""
    inp = K.GemmInput(50, 30, 333, "f32")
    t = K.GemmTuning(2, 2, 16, 16, 16, 1, 2, 4)
    a, b = O.fill(9, inp.m * inp.k, inp.k * inp.n, "f32", True)
    assert K.gemm_launch_info(inp, t)["family"] == "simt"
    got, cp = both_feeds(inp, t, a, b)
    want = O.execute_gemm(50, 30, 333, False, False, t.values(), a, b, "f32")
    assert bitwise_equal(got, want) and bitwise_equal(cp, want)


@pytest.mark.parametrize("case", [
    ((512, 512, 512, False, False), (2, 8, 32, 32, 8, 1, 1, 1)),    # C1 fixed tuple: u = 8 staged 32 wide
    ((300, 40, 2048, True, True), (2, 2, 16, 16, 8, 4, 2, 4)),      # k_s = 4, k_l = 2, ragged rows
    ((256, 64, 1024, False, True), (4, 2, 32, 16, 4, 2, 1, 2)),     # u = 4
])
def test_widened_stages_are_bitwise(cuda, monkeypatch, case):
    """The TMA feed stages several u-steps per box (u does not enter the
    summation order: only k_s, k_l and k_g do); PARITY stays bit-identical
    to the reference with and without widening, FAST within tolerance."""
    (m, n, k, ta, tb), tv = case
    inp = K.GemmInput(m, n, k, "f32", ta, tb)
    t = K.GemmTuning(*tv)
    a, b = O.fill(sum(tv), m * k, k * n, "f32", True)
    want = O.execute_gemm(m, n, k, ta, tb, tv, a, b, "f32")
    for widen in ("1", "0"):
        monkeypatch.setenv("KTUNE_SIMT_WIDEN", widen)
        assert K.gemm_launch_info(inp, t, "parity")["family"] == "simt-tma", case
        got = run_gemm(inp, t, a, b, "parity")
        assert bitwise_equal(got, want), (case, widen, first_mismatch(got, want))
        fast = run_gemm(inp, t, a, b, "fast")
        # FAST within 1e-5, or within 2x the reference executor's own
        # rounding error on these signed inputs (as test_tma_feed_is_bitwise)
        ref = O.naive_gemm(m, n, k, int(ta), int(tb), a.astype(np.float64), b.astype(np.float64), "f64")
        own = O.max_rel_error(want, ref)
        assert O.max_rel_error(fast, ref) < max(1e-5, 2 * own), (case, widen)

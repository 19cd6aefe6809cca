"""K1/K2 on the B200: the SIMT GEMM family against the oracle.

PARITY mode must be bit-identical to the reference execute_gemm<T>
(backends.cpp:228-329) for every tuple; FAST mode must stay within the
reference's own tolerances of the naive double loop (1e-5 f32, 1e-12 f64;
test_backends.cpp:120-153).  Sizes are ones the C oracle finishes in
seconds; BASELINE's full configs C1/C2 are covered at full size."""
import json
import os

import numpy as np
import pytest
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K
from gpu_util import bitwise_equal, dev, first_mismatch, run_gemm

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "executors.json")

ENVELOPE = [(ms, ns, ks) for ks in (1, 2, 4) for ms in (1, 2, 4, 8) for ns in (1, 2, 4, 8)
            if ms * ns * ks <= 128]


def check_parity(inp, t, seed=0, symmetric=True):
    a, b = O.fill(seed, inp.m * inp.k, inp.k * inp.n, inp.dtype, symmetric)
    got = run_gemm(inp, t, a, b, "parity")
    want = O.execute_gemm(inp.m, inp.n, inp.k, inp.trans_a, inp.trans_b, t.values(), a, b, inp.dtype)
    assert bitwise_equal(got, want), (inp, t, first_mismatch(got, want))


def test_golden_cases_bitwise(cuda):
    """The reference library's own outputs (hash-pinned) reproduced on device."""
    import hashlib
    for c in json.load(open(GOLDEN))["gemm"]:
        inp = K.GemmInput(c["m"], c["n"], c["k"], c["dtype"], bool(c["ta"]), bool(c["tb"]))
        a, b = O.fill(c["seed"], inp.m * inp.k, inp.k * inp.n, inp.dtype, True)
        got = run_gemm(inp, K.GemmTuning(*c["tuning"]), a, b)
        assert hashlib.sha256(got.tobytes()).hexdigest() == c["sha256"], c


@pytest.mark.parametrize("tile", ENVELOPE)
def test_every_register_tile_is_bitwise(cuda, tile):
    ms, ns, ks = tile
    rng = np.random.default_rng(ms * 100 + ns * 10 + ks)
    for trial in range(3):
        ml = ms * int(rng.choice([1, 2, 4, 8]))
        nl = ns * int(rng.choice([1, 2, 4, 8]))
        kl = int(rng.choice([1, 2, 4]))
        while (ml // ms) * (nl // ns) * kl > 1024:
            kl = max(1, kl // 2)
            ml = max(ms, ml // 2)
        t = K.GemmTuning(ms, ns, ml, nl, ks * int(rng.choice([1, 2, 4])), ks, kl, int(rng.choice([1, 2, 4, 8])))
        inp = K.GemmInput(int(rng.integers(1, 150)), int(rng.integers(1, 150)), int(rng.integers(1, 400)),
                          "f32" if trial != 2 else "f64", bool(rng.integers(0, 2)), bool(rng.integers(0, 2)))
        check_parity(inp, t, seed=trial)


def test_generic_kernel_paths_bitwise(cuda):
    """Tiles outside the compiled envelope and thread counts above an
    instantiation's launch bound run on the runtime-tile kernel."""
    cases = [K.GemmTuning(16, 2, 32, 8, 8, 4, 2, 2),     # MS=16 outside the envelope
             K.GemmTuning(1, 1, 32, 32, 4, 1, 1, 1),      # 1024 threads
             K.GemmTuning(2, 2, 64, 64, 8, 8, 1, 4),      # KS=8
             K.GemmTuning(8, 8, 128, 64, 8, 2, 2, 1)]     # 64 acc * 256 threads > cap
    for i, t in enumerate(cases):
        check_parity(K.GemmInput(77, 91, 133, "f32", i % 2 == 1, i >= 2), t, seed=i)


def test_ragged_edges_and_deep_splits(cuda):
    """test_backends.cpp:155-166: dims coprime to every tile extent."""
    for dt in ("f32", "f64"):
        check_parity(K.GemmInput(7, 11, 13, dt, True, True), K.GemmTuning(2, 2, 8, 4, 4, 2, 4, 4))
        # more grid slices than reduction columns: empty slices are skipped
        check_parity(K.GemmInput(5, 3, 3, dt), K.GemmTuning(1, 1, 4, 4, 4, 4, 8, 16))
        check_parity(K.GemmInput(1, 1, 1, dt), K.GemmTuning(1, 1, 1, 1, 1, 1, 1, 1))


def test_fast_mode_within_reference_tolerance(cuda):
    rng = np.random.default_rng(3)
    for trial in range(40):
        ms, ns, ks = ENVELOPE[int(rng.integers(len(ENVELOPE)))]
        t = K.GemmTuning(ms, ns, ms * 4, ns * 4, ks * 2, ks, int(rng.choice([1, 2])), int(rng.choice([1, 4])))
        dt = "f32" if trial % 4 else "f64"
        inp = K.GemmInput(int(rng.integers(1, 200)), int(rng.integers(1, 200)), int(rng.integers(1, 600)), dt,
                          bool(trial % 2), bool(trial % 3 == 0))
        a, b = O.fill(trial, inp.m * inp.k, inp.k * inp.n, dt, True)
        got = run_gemm(inp, t, a, b, "fast")
        ref = O.naive_gemm(inp.m, inp.n, inp.k, inp.trans_a, inp.trans_b, a, b, dt)
        assert O.max_rel_error(got, ref) < (1e-5 if dt == "f32" else 1e-12), (inp, t)


def test_config_c1_sgemm_512_fixed_tuple_bitwise(cuda):
    """BASELINE configs[0]: SGEMM NN 512^3 with paper Table 5 LINPACK(512)
    tuple (2,8,32,32,8,1,1,1), CpuBackend's [0,1) operands."""
    inp = K.GemmInput(512, 512, 512, "f32")
    check_parity(inp, K.GemmTuning(2, 8, 32, 32, 8, 1, 1, 1), seed=0x5EED, symmetric=False)
    check_parity(inp, K.GemmTuning(2, 2, 16, 16, 1, 1, 1, 1), seed=0x5EED, symmetric=False)


@pytest.mark.parametrize("shape,tuple_", [
    ((2560, 16, 2560, False, False), (2, 4, 64, 16, 16, 1, 1, 4)),    # DeepBench fprop
    ((2560, 16, 2560, True, False), (4, 2, 16, 16, 16, 1, 8, 1)),     # DeepBench bprop
    ((32, 32, 60000, False, True), (2, 4, 32, 32, 8, 1, 4, 32)),      # ICA
])
def test_config_c2_skinny_full_size_bitwise(cuda, shape, tuple_):
    m, n, k, ta, tb = shape
    check_parity(K.GemmInput(m, n, k, "f32", ta, tb), K.GemmTuning(*tuple_), seed=11, symmetric=False)


def test_repeated_launches_reuse_workspace_counters(cuda):
    """The k_g fix-up leaves its arrival counters at zero: back-to-back
    launches on one workspace stay bit-identical."""
    inp = K.GemmInput(300, 70, 5000, "f32")
    t = K.GemmTuning(2, 2, 32, 16, 8, 2, 2, 16)
    a, b = O.fill(5, inp.m * inp.k, inp.k * inp.n, "f32", True)
    da, db = dev(a), dev(b)
    outs = [K.execute_gemm(inp, t, da, db, mode="parity").cpu().numpy() for _ in range(4)]
    want = O.execute_gemm(inp.m, inp.n, inp.k, False, False, t.values(), a, b)
    for o in outs:
        assert bitwise_equal(o, want)


def test_host_buffer_entry_point_bitwise(cuda):
    """ktune_execute_gemm: the executor's span contract through the C-ABI."""
    inp = K.GemmInput(123, 45, 678, "f64", True, False)
    t = K.GemmTuning(2, 1, 16, 8, 4, 2, 2, 4)
    a, b = O.fill(9, inp.m * inp.k, inp.k * inp.n, "f64", True)
    got = K.execute_gemm_host(inp, t, a, b, "parity")
    assert bitwise_equal(got, O.execute_gemm(inp.m, inp.n, inp.k, True, False, t.values(), a, b, "f64"))
    with pytest.raises(K.InvalidArgument, match="operand size mismatch"):
        K.execute_gemm_host(inp, t, a[:-1], b)


@pytest.mark.parametrize("tup", [(2, 4, 64, 16, 32, 1, 1, 4), (4, 4, 32, 16, 32, 1, 2, 8)])
def test_host_buffer_large_operands_bitwise(cuda, tup):
    """The host-buffer path at DeepBench size (10.6 MB of A, ragged last
    block-row): bit-equal to the reference executor, fast within bound."""
    inp = K.GemmInput(2600, 16, 1024, "f32")  # 10.6 MB of A, ragged last block
    t = K.GemmTuning(*tup)
    a, b = O.fill(4, inp.m * inp.k, inp.k * inp.n, "f32", True)
    got = K.execute_gemm_host(inp, t, a, b, "parity")
    assert bitwise_equal(got, O.execute_gemm(inp.m, inp.n, inp.k, False, False, t.values(), a, b))
    fast = K.execute_gemm_host(inp, t, a, b, "fast")
    # 1e-5 is the reference's bound for K <= 300 (test_backends.cpp:142); the
    # fp32 rounding error of a K-long dot product grows with K
    assert O.max_rel_error(fast, O.naive_gemm(inp.m, inp.n, inp.k, 0, 0, a, b)) < max(1e-5, 2e-8 * inp.k)


def test_executor_validation(cuda):
    """test_backends.cpp:168-178."""
    inp = K.GemmInput(4, 4, 4)
    a = torch.zeros(16, device="cuda")
    with pytest.raises(K.InvalidArgument, match="size mismatch"):
        K.execute_gemm(inp, K.GemmTuning(), a, a, torch.zeros(15, device="cuda"))
    with pytest.raises(K.InvalidArgument, match="m_l not divisible by m_s"):
        K.execute_gemm(inp, K.GemmTuning(m_s=2), a, a)
    with pytest.raises(K.Unsupported, match="accumulators"):
        K.execute_gemm(inp, K.GemmTuning(16, 16, 16, 16, 2, 2, 1, 1), a, a)


def test_measure_backend(cuda):
    """CpuBackend::measure semantics (test_backends.cpp:395-423) on device."""
    hw = K.HardwareDescriptor.b200()
    be = K.B200Backend(hw, repetitions=2)
    assert be.name() == "b200"
    g = be.measure(K.GemmInput(512, 512, 512), K.GemmTuning(2, 8, 32, 32, 8, 1, 1, 1))
    assert np.isfinite(g) and g > 0
    with pytest.raises(K.InvalidArgument, match="illegal tuning: registers"):
        K.measure(K.GemmInput(48, 40, 56), K.GemmTuning(4, 4, 4, 4, 1, 1, 1, 1), K.HardwareDescriptor())
    with pytest.raises(K.InvalidArgument):
        K.B200Backend(hw, repetitions=0)

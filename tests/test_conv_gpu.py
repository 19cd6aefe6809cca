"""K3 on the B200: implicit-GEMM convolution against the oracle
(backends.cpp:331-444; test_backends.cpp:180-262)."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle_libs as O
import paper_1802_05371_b200 as K
from gpu_util import bitwise_equal, first_mismatch, run_conv, run_gemm

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "executors.json")

CONV_ENVELOPE = [(kt, sp, cs) for cs in (1, 2) for kt in (1, 2, 4, 8) for sp in (1, 2, 4, 8, 16)
                 if kt * sp * cs <= 128]


def split_sp(sp):
    """p_s, q_s, n_s with product sp."""
    ps = 2 if sp >= 8 else 1
    qs = 2 if sp >= 4 else 1
    return ps, qs, sp // (ps * qs)


def check_parity(inp, t, seed=0, symmetric=True):
    ni, nf, _ = inp.sizes()
    img, flt = O.fill(seed, ni, nf, inp.dtype, symmetric)
    got = run_conv(inp, t, img, flt, "parity")
    dims = [inp.n_batch, inp.p, inp.q, inp.k_filters, inp.c, inp.r, inp.s]
    want = O.execute_conv(dims, t.values(), img, flt, inp.dtype)
    assert bitwise_equal(got, want), (inp, t, first_mismatch(got, want))


def test_golden_cases_bitwise(cuda):
    for c in json.load(open(GOLDEN))["conv"]:
        inp = K.ConvInput(*c["dims"], dtype=c["dtype"])
        ni, nf, _ = inp.sizes()
        img, flt = O.fill(c["seed"], ni, nf, inp.dtype, True)
        got = run_conv(inp, K.ConvTuning(*c["tuning"]), img, flt)
        assert hashlib.sha256(got.tobytes()).hexdigest() == c["sha256"], c


@pytest.mark.parametrize("tile", CONV_ENVELOPE)
def test_every_register_tile_is_bitwise(cuda, tile):
    kt, sp, cs = tile
    ps, qs, ns = split_sp(sp)
    rng = np.random.default_rng(kt * 1000 + sp * 10 + cs)
    for trial in range(2):
        t = K.ConvTuning(kt, ps, qs, ns, kt * int(rng.choice([1, 2, 4])), ps * int(rng.choice([1, 2])),
                         qs * int(rng.choice([1, 2])), ns * int(rng.choice([1, 2])), cs * int(rng.choice([1, 2, 4])),
                         cs, int(rng.choice([1, 2])), int(rng.choice([1, 2, 4])))
        inp = K.ConvInput(int(rng.integers(1, 9)), int(rng.integers(1, 12)), int(rng.integers(1, 12)),
                          int(rng.integers(1, 40)), int(rng.integers(1, 9)), int(rng.choice([1, 3])),
                          int(rng.choice([1, 2, 3])), "f32" if trial == 0 else "f64")
        check_parity(inp, t, seed=trial)


def test_deepbench_and_resnet_shapes_bitwise(cuda):
    """BASELINE configs[2] shapes (f32 parity; reduced batch where the
    oracle would take minutes)."""
    check_parity(K.ConvInput(16, 56, 56, 64, 64, 3, 3), K.ConvTuning(4, 1, 1, 4, 32, 2, 2, 16, 8, 1, 2, 2), seed=1,
                 symmetric=False)
    check_parity(K.ConvInput(2, 79, 341, 32, 1, 5, 20), K.ConvTuning(4, 1, 1, 2, 32, 1, 4, 2, 8, 2, 1, 4), seed=2)
    check_parity(K.ConvInput(16, 7, 7, 32, 96, 5, 5), K.ConvTuning(2, 1, 1, 4, 16, 1, 1, 16, 8, 1, 2, 8), seed=3)


def test_one_by_one_conv_is_gemm(cuda):
    """test_backends.cpp:217-245: with r = s = 1 the conv equals the
    trans_a GEMM on the same buffers."""
    cin = K.ConvInput(3, 5, 4, 6, 7, 1, 1, "f64")
    ni, nf, _ = cin.sizes()
    img, flt = O.fill(7, ni, nf, "f64", True)
    conv_out = run_conv(cin, K.ConvTuning(2, 1, 2, 1, 2, 2, 2, 1, 2, 1, 2, 2), img, flt)
    gin = K.GemmInput(cin.k_filters, cin.p * cin.q * cin.n_batch, cin.c, "f64", True, False)
    gemm_out = run_gemm(gin, K.GemmTuning(2, 2, 4, 4, 2, 2, 2, 2), flt, img)
    assert O.max_rel_error(conv_out, gemm_out) < 1e-12


def test_fast_mode_tolerance(cuda):
    rng = np.random.default_rng(11)
    for trial in range(12):
        inp = K.ConvInput(int(rng.integers(1, 17)), int(rng.integers(1, 20)), int(rng.integers(1, 20)),
                          int(rng.integers(1, 70)), int(rng.integers(1, 40)), 3, 3)
        t = K.ConvTuning(4, 1, 2, 2, 16, 2, 4, 4, 8, 2, 2, 2)
        ni, nf, _ = inp.sizes()
        img, flt = O.fill(trial, ni, nf, "f32", True)
        got = run_conv(inp, t, img, flt, "fast")
        ref = O.direct_conv([inp.n_batch, inp.p, inp.q, inp.k_filters, inp.c, inp.r, inp.s], img, flt)
        assert O.max_rel_error(got, ref) < 1e-4


def test_host_entry_and_validation(cuda):
    inp = K.ConvInput(2, 6, 6, 4, 3, 3, 3, "f64")
    t = K.ConvTuning(1, 1, 1, 1, 2, 2, 2, 1, 1, 1, 1, 1)
    ni, nf, _ = inp.sizes()
    img, flt = O.fill(1, ni, nf, "f64", True)
    got = K.execute_conv_host(inp, t, img, flt)
    assert bitwise_equal(got, O.execute_conv([2, 6, 6, 4, 3, 3, 3], t.values(), img, flt, "f64"))
    with pytest.raises(K.InvalidArgument, match="operand size mismatch"):
        K.execute_conv_host(inp, t, img[:-1], flt)
    with pytest.raises(K.InvalidArgument, match="k_l not divisible by k_s"):
        K.execute_conv_host(inp, K.ConvTuning(k_s=2), img, flt)
    g = K.measure(K.ConvInput(16, 24, 240, 32, 16, 3, 3), K.ConvTuning(2, 1, 1, 1, 8, 1, 4, 2, 1, 1, 1, 8),
                  K.HardwareDescriptor())
    assert g > 0


@pytest.mark.parametrize("widen", ["1", "0"])
def test_widened_stages_conv_and_cp_async_gemm(cuda, monkeypatch, widen):
    """Stages holding several u-steps (launch.cu widened_plan) leave the
    summation order alone: the bench's fp32 ResNet conv pick and a cp.async
    GEMM stay bit-identical to the reference with and without widening."""
    monkeypatch.setenv("KTUNE_SIMT_WIDEN", widen)
    cin = K.ConvInput(8, 14, 14, 32, 16, 3, 3)
    ct = K.ConvTuning(8, 1, 2, 1, 32, 2, 2, 8, 16, 1, 1, 4)
    ni, nf, _ = cin.sizes()
    img, flt = O.fill(5, ni, nf, "f32")
    got = run_conv(cin, ct, img, flt, "parity")
    want = O.execute_conv([8, 14, 14, 32, 16, 3, 3], ct.values(), img, flt)
    assert bitwise_equal(got, want), first_mismatch(got, want)
    monkeypatch.setenv("KTUNE_SIMT_TMA", "0")
    inp = K.GemmInput(200, 72, 1500, "f32", True, False)
    t = K.GemmTuning(2, 2, 32, 16, 8, 2, 2, 2)
    a, b = O.fill(9, inp.m * inp.k, inp.k * inp.n, "f32")
    got = run_gemm(inp, t, a, b, "parity")
    want = O.execute_gemm(inp.m, inp.n, inp.k, 1, 0, t.values(), a, b)
    assert bitwise_equal(got, want), first_mismatch(got, want)

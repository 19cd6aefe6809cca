"""The checker is pinned before it is trusted: the C restatement of the
reference executors (oracle/ktune_oracle.c) must reproduce the reference
library's outputs bit-for-bit -- against the committed golden hashes (always)
and against oracle/_ref/libktune_ref.so itself when it is present."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle_libs as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "executors.json")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def test_fill_matches_reference_engine(golden):
    """MT19937-64 + unit_real (sampler.cpp:14-17) as CpuBackend fills operands."""
    a, b = O.fill(0x5EED, 40, 24, "f64")
    assert np.array_equal(np.concatenate([a, b]), np.array(golden["fill_0x5eed_first64"]))


def test_gemm_oracle_matches_golden(golden):
    for c in golden["gemm"]:
        a, b = O.fill(c["seed"], c["m"] * c["k"], c["k"] * c["n"], c["dtype"], symmetric=True)
        out = O.execute_gemm(c["m"], c["n"], c["k"], c["ta"], c["tb"], c["tuning"], a, b, c["dtype"])
        assert sha(out) == c["sha256"], c


def test_conv_oracle_matches_golden(golden):
    for c in golden["conv"]:
        ni, nf, _ = O.conv_sizes(c["dims"])
        img, flt = O.fill(c["seed"], ni, nf, c["dtype"], symmetric=True)
        out = O.execute_conv(c["dims"], c["tuning"], img, flt, c["dtype"])
        assert sha(out) == c["sha256"], c


def test_oracle_within_reference_tolerance_of_naive():
    """test_backends.cpp:120-153: tiled f32 within 1e-5 of the naive loop."""
    rng = np.random.default_rng(0)
    for trial in range(20):
        m, n, k = (int(x) for x in rng.integers(1, 48, 3))
        t = [1, 2, 4, 4, 4, 2, 2, 4]
        a, b = O.fill(trial, m * k, k * n, "f32", True)
        got = O.execute_gemm(m, n, k, trial % 2, (trial // 2) % 2, t, a, b)
        ref = O.naive_gemm(m, n, k, trial % 2, (trial // 2) % 2, a, b)
        assert O.max_rel_error(got, ref.astype(np.float32)) < 1e-5


def test_indirection_matches_frozen_values():
    """test_backends.cpp:247-262."""
    tab = O.indirection_table([2, 2, 3, 1, 2, 2, 2])
    assert tab.shape == (8, 4)
    assert tab[0, 3] == 0 and tab[1, 3] == 2 and tab[2, 3] == 8 and tab[7, 3] == 24 + 8 + 2


@pytest.mark.skipif(O.reference() is None, reason="oracle/_ref not built on this box")
def test_oracle_bitwise_equals_reference_library_random():
    rng = np.random.default_rng(99)
    for trial in range(150):
        m, n, k = (int(x) for x in rng.integers(1, 64, 3))
        ks = int(rng.choice([1, 2, 4]))
        ms, ns = int(rng.choice([1, 2, 4])), int(rng.choice([1, 2, 4]))
        t = [ms, ns, ms * 2, ns * 4, ks * int(rng.choice([1, 2, 4])), ks, int(rng.choice([1, 2, 4, 8])),
             int(rng.choice([1, 2, 4, 8, 16, 32]))]
        dt = "f32" if trial % 3 else "f64"
        ta, tb = int(rng.integers(0, 2)), int(rng.integers(0, 2))
        a, b = O.fill(trial, m * k, k * n, dt, True)
        mine = O.execute_gemm(m, n, k, ta, tb, t, a, b, dt)
        ref = O.ref_execute_gemm(m, n, k, ta, tb, t, a, b, dt)
        assert np.array_equal(mine.view(np.uint8), ref.view(np.uint8)), (m, n, k, ta, tb, t, dt)
    for trial in range(60):
        dims = [int(rng.integers(1, 5)), int(rng.integers(1, 8)), int(rng.integers(1, 8)), int(rng.integers(1, 9)),
                int(rng.integers(1, 7)), int(rng.choice([1, 2, 3])), int(rng.choice([1, 3, 5]))]
        cs = int(rng.choice([1, 2]))
        t = [1, 1, 1, 1, 2, 2, 2, 2, cs * 2, cs, int(rng.choice([1, 2, 4])), int(rng.choice([1, 2, 4, 8]))]
        dt = "f32" if trial % 2 else "f64"
        ni, nf, _ = O.conv_sizes(dims)
        img, flt = O.fill(trial, ni, nf, dt, True)
        mine = O.execute_conv(dims, t, img, flt, dt)
        ref = O.ref_execute_conv(dims, t, img, flt, dt)
        assert np.array_equal(mine.view(np.uint8), ref.view(np.uint8)), (dims, t, dt)

"""Integer-exact parity of the product's host code (libktune_b200.so via the
C-ABI) with the reference param_space.cpp, pinned by tests/golden/space.json
(generated from the reference library by tests/golden/make_golden.py).
Mirrors test_param_space.cpp:41-264."""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_1802_05371_b200 as K

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "space.json")
FIX = K.FIXTURES


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def hw_named(name):
    return K.HardwareDescriptor() if name == "synthetic" else K.HardwareDescriptor.b200()


def bounds_named(kind, name):
    if name == "default":
        return None
    if name == "b200":
        return open(os.path.join(FIX, "bounds", f"{kind}_b200.json")).read()
    if name == "conv_small":
        # the reference fixture proj/fixtures/bounds/conv_small.json, as its lists
        return json.dumps({"k_s": [1, 2], "p_s": [1, 2], "q_s": [1, 2], "n_s": [1, 2], "k_l": [1, 2, 4, 8],
                           "p_l": [1, 2, 4], "q_l": [1, 2, 4], "n_l": [1, 2, 4], "u": [1, 2, 4], "c_s": [1, 2],
                           "c_l": [1, 2, 4], "c_g": [1, 2, 4, 8]})
    raise KeyError(name)


def test_frozen_enumeration_counts(golden):
    """6140 / 2970 / 14448 (test_param_space.cpp:211-245) and the B200 spaces."""
    for e in golden["enumerations"]:
        hw = hw_named(e["hw"].replace("-default-bounds", ""))
        if e["kind"] == "gemm":
            arr = K.enumerate_legal(K.GemmInput(e["m"], e["n"], e["k"], e["dtype"]), hw,
                                    bounds_named("gemm", e["bounds"]), as_array=True)
        else:
            d = e["dims"]
            arr = K.enumerate_legal(K.ConvInput(*d, dtype=e["dtype"]), hw, bounds_named("conv", e["bounds"]),
                                    as_array=True)
        assert len(arr) == e["count"], e
        assert arr[:5].tolist() == e["head"] and arr[-5:].tolist() == e["tail"]
        assert sha(arr) == e["sha256"], e


def test_enumeration_is_lexicographic_and_legal():
    hw = K.HardwareDescriptor()
    inp = K.GemmInput(512, 512, 512)
    space = K.enumerate_legal(inp, hw)
    vals = [t.values() for t in space]
    assert vals == sorted(vals)
    for t in space[::97]:
        assert K.is_legal(inp, t, hw)


def test_legality_verdicts_and_details(golden):
    for c in golden["legality_gemm"]:
        v = K.is_legal(K.GemmInput(c["m"], c["n"], c["k"], c["dtype"]), K.GemmTuning(*c["tuning"]),
                       hw_named(c["hw"]))
        assert (int(v.accepted), K.REJECT_REASONS.index(v.reason) if not v.accepted else c["reason"]) == \
            (c["accepted"], c["reason"]), c
        assert v.detail == c["detail"], c
        r = K.estimate_resources(K.GemmInput(c["m"], c["n"], c["k"], c["dtype"]), K.GemmTuning(*c["tuning"]))
        assert [r.shared_bytes, r.registers_per_thread, r.threads_per_block] == c["resources"]
    for c in golden["legality_conv"]:
        inp = K.ConvInput(*c["dims"], dtype=c["dtype"])
        v = K.is_legal(inp, K.ConvTuning(*c["tuning"]), hw_named(c["hw"]))
        assert int(v.accepted) == c["accepted"] and v.detail == c["detail"], c
        if not v.accepted:
            assert K.REJECT_REASONS.index(v.reason) == c["reason"]
        r = K.estimate_resources(inp, K.ConvTuning(*c["tuning"]))
        assert [r.shared_bytes, r.registers_per_thread, r.threads_per_block] == c["resources"]


def test_hand_computed_resources():
    """test_param_space.cpp:41-71 style spot values."""
    r = K.estimate_resources(K.GemmInput(64, 64, 64, "f32"), K.GemmTuning(2, 4, 8, 16, 4, 2, 2, 1))
    assert r.shared_bytes == 2 * 4 * (8 * 4 + 4 * 16)
    assert r.registers_per_thread == 8 + 2 + 4 + 8
    assert r.threads_per_block == (8 // 2) * (16 // 4) * 2


def test_check_order_reports_first_failure():
    hw = K.HardwareDescriptor()
    inp = K.GemmInput(8, 8, 8)
    assert K.is_legal(inp, K.GemmTuning(2, 1, 1, 1, 1, 1, 1, 1), hw).reason == "divisibility"
    assert K.is_legal(inp, K.GemmTuning(1, 1, 16, 16, 16, 1, 1, 1), hw).reason == "shared_memory"
    assert K.is_legal(inp, K.GemmTuning(4, 4, 4, 4, 1, 1, 1, 1), hw).reason == "registers"
    assert K.is_legal(inp, K.GemmTuning(1, 1, 16, 8, 1, 1, 1, 1), hw).reason == "threads"


def test_features(golden):
    for c in golden["features_gemm"]:
        f = K.encode_features(K.GemmInput(c["m"], c["n"], c["k"], c["dtype"], bool(c["ta"]), bool(c["tb"])),
                              K.GemmTuning(*c["tuning"]))
        assert f.tolist() == c["features"]
    for c in golden["features_conv"]:
        f = K.encode_features(K.ConvInput(*c["dims"]), K.ConvTuning(*c["tuning"]))
        assert f.tolist() == c["features"]


def test_indirection_tables(golden):
    for c in golden["indirection"]:
        tab = K.build_indirection_table(K.ConvInput(*c["dims"]))
        assert len(tab) == c["count"] and sha(tab) == c["sha256"]
        assert tab[:6].tolist() == c["head"] and tab[-3:].tolist() == c["tail"]


def test_hw_json_roundtrip_and_strictness(golden):
    b200 = K.HardwareDescriptor.b200()
    assert b200.num_multiprocessors == 148 and b200.warp_size == 32
    with pytest.raises(K.KtuneError, match="unknown hardware descriptor field"):
        K.HardwareDescriptor.from_json_text('{"warp_sizes": 32}')
    with pytest.raises(K.KtuneError, match="malformed JSON"):
        K.HardwareDescriptor.from_json_text('{"warp_size": ')
    with pytest.raises(K.KtuneError, match="bad hardware descriptor"):
        K.HardwareDescriptor.from_json_text('{"warp_size": 32}')
    # peak = 2 * SMs * warp * clock / alu_throughput (backends.cpp:142-145)
    hw = b200
    peak = 2.0 * hw.num_multiprocessors * hw.warp_size * hw.clock_hz / hw.alu_throughput / 1e9
    assert peak == golden["peak_gflops_b200"]


def test_invalid_values_raise_invalid_argument():
    with pytest.raises(K.InvalidArgument, match="m must be >= 1"):
        K.estimate_resources(K.GemmInput(0, 1, 1), K.GemmTuning())
    with pytest.raises(K.InvalidArgument, match="u must be a power of two"):
        K.estimate_resources(K.GemmInput(1, 1, 1), K.GemmTuning(u=3))
    with pytest.raises(K.InvalidArgument, match="bounds for u must be strictly increasing"):
        K.enumerate_legal(K.GemmInput(4, 4, 4), bounds_json=json.dumps(
            {"m_s": [1], "n_s": [1], "m_l": [1], "n_l": [1], "u": [2, 1], "k_s": [1], "k_l": [1], "k_g": [1]}))
    with pytest.raises(K.KtuneError, match="unknown bounds parameter"):
        K.enumerate_legal(K.GemmInput(4, 4, 4), bounds_json='{"q": [1]}')

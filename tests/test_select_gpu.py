"""Runtime selection on the B200 (pipeline.cpp:649-723, :928-997).

- select_conv: the first call infers (b200 re-measure of the top-k), stores
  the result in the cache directory and the in-memory map; the second call
  answers from memory; a fresh key (other top_k) answers from the file.
- The memo key includes the model / bounds / top_k (a changed configuration
  is never served a stale pick).
- Sharded infer at world size 1 on the b200 backend yields a valid result
  whose choice is the measured argmax of its own top-k list."""
import json

import paper_1802_05371_b200 as K
from paper_1802_05371_b200 import pipeline as P

import pytest

pytestmark = pytest.mark.gpu


def test_select_conv_memory_file_inferred(cuda, tmp_path):
    hw = K.HardwareDescriptor.b200()
    cin = K.ConvInput(4, 9, 11, 24, 8, 3, 3)
    d = str(tmp_path)
    t1, s1 = P.select_conv(cin, hw, None, None, d, top_k=4)
    assert s1 == "inferred"
    assert P.cache_lookup(d, cin) is not None
    t2, s2 = P.select_conv(cin, hw, None, None, d, top_k=4)
    assert (t2, s2) == (t1, "memory")
    t3, s3 = P.select_conv(cin, hw, None, None, d, top_k=5)  # other key: served by the result file
    assert (t3, s3) == (t1, "file")


def test_select_gemm_memo_keyed_by_configuration(cuda):
    hw = K.HardwareDescriptor.b200()
    inp = K.GemmInput(300, 40, 500, "f32")
    _, s1 = P.select_gemm(inp, hw, None, None, None, top_k=3)
    _, s2 = P.select_gemm(inp, hw, None, None, None, top_k=3)
    _, s3 = P.select_gemm(inp, hw, None, None, None, top_k=4)
    assert (s1, s2, s3) == ("inferred", "memory", "inferred")


def test_infer_sharded_single_rank_on_device(cuda):
    hw = K.HardwareDescriptor.b200()
    r = json.loads(P.infer_sharded(K.GemmInput(512, 64, 1024, "f32"), hw, None, None, 6, backend="b200"))
    meas = [c["measured_gflops"] for c in r["top_k"]]
    assert len(meas) == 6 and all(m > 0 for m in meas)
    best = max(range(6), key=lambda i: (meas[i], -i))
    assert r["chosen"] == r["top_k"][best]["tuning"]


def _tc_bounds():
    import os
    return open(os.path.join(K.FIXTURES, "bounds", "gemm_b200_tc.json")).read()


def test_infer_tensor_core_ranks_only_launchable(cuda):
    """most legal tuples of the tensor-core space are outside the
    tcgen05 launch envelope; infer ranks only tuples the backend accepts, so
    the top-k re-measure never aborts on unsupported_error, and the sharded
    replay ranks the same candidates (same JSON as the sequential infer)."""
    hw = K.HardwareDescriptor.b200()
    bounds = _tc_bounds()
    inp = K.GemmInput(1024, 96, 2048, "bf16")
    r = json.loads(P.infer(inp, hw, bounds, None, top_k=8, backend="b200"))
    assert len(r["top_k"]) == 8 and all(c["measured_gflops"] > 0 for c in r["top_k"])
    assert r["legal_space_size"] == len(K.enumerate_legal(inp, hw, bounds))
    for c in r["top_k"]:
        K.gemm_launch_info(inp, K.GemmTuning(*(c["tuning"][n] for n in K.GEMM_PARAMS)), "fast")
    s = json.loads(P.infer_sharded(inp, hw, bounds, None, 8, backend="b200"))
    assert [c["tuning"] for c in s["top_k"]] == [c["tuning"] for c in r["top_k"]]
    assert s["chosen"] in [c["tuning"] for c in s["top_k"]]

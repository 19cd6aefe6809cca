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

"""INTEGRATION.md route 1, end to end: the adapter backend from the document
(oracle/integration/b200_backend_adapter.cpp), compiled against the
reference headers and linked with the UNMODIFIED reference library
(oracle/_ref/libktune_ref.so) and libktune_b200.so, drives the reference's
own generate_gemm_dataset (pipeline.cpp:463-509) on the GPU.  The dataset
must draw the same (input, tuning) sequence as this build's generator with
the analytical backend and carry device-measured gflops tagged "b200"."""
import os
import subprocess

import pytest

import paper_1802_05371_b200 as K
import paper_1802_05371_b200.pipeline as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_generate")


def fixture(*parts):
    return os.path.join(K.FIXTURES, *parts)


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="adapter driver not built (needs the reference sources)")
def test_reference_generate_through_adapter(cuda):
    n, seed = 16, 42
    out = subprocess.run([BIN, fixture("hw", "b200.json"), fixture("samplers", "gemm_b200.json"),
                          fixture("bounds", "gemm_b200.json"), str(n), str(seed), "512", "512", "4096"],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    rows = out.stdout.splitlines()
    dist = P.GemmInputDistribution(fixed_fraction=0.0, m_hi=512, n_hi=512, k_hi=4096)
    ana, _, _ = P.generate_gemm(open(fixture("samplers", "gemm_b200.json")).read(), dist, K.HardwareDescriptor.b200(),
                                open(fixture("bounds", "gemm_b200.json")).read(), n, seed, backend="analytical")
    arows = ana.splitlines()
    assert rows[0] == arows[0] and len(rows) == n + 1
    for r, a in zip(rows[1:], arows[1:]):
        f, fa = r.split(","), a.split(",")
        assert f[:14] == fa[:14] and f[15] == "b200" and float(f[14]) > 0


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/src"), reason="reference sources absent")
def test_adapter_driver_links():
    """CPU side: the adapter compiles and resolves both libraries."""
    assert os.path.exists(BIN), "build() compiles oracle/_ref/adapter_generate when the reference is present"
    ldd = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libktune_ref.so" in ldd and "libktune_b200.so" in ldd and "not found" not in ldd

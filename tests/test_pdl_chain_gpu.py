"""Programmatic dependent launch: back-to-back kernels on one stream where
each consumes the previous one's output (read-after-write) or overwrites a
buffer the previous one reads (write-after-read) -- the griddepcontrol.wait
in every kernel must order all global-memory work after the previous grid.
No host synchronisation between the launches; checked against float64."""
import numpy as np
import pytest
import torch

import paper_1802_05371_b200 as K

pytestmark = pytest.mark.gpu


def _chain(dtype, tuples, n=512, links=6, tb=False):
    g = torch.Generator(device="cuda").manual_seed(5)
    x = (torch.rand(n * n, device="cuda", generator=g) - 0.5)
    ws = [(torch.rand(n * n, device="cuda", generator=g) - 0.5) / n ** 0.5 for _ in range(links)]
    if dtype == "tf32":  # exact tf32 operands
        x = (x.view(torch.int32) & ~0x1FFF).view(torch.float32)
        ws = [(w.view(torch.int32) & ~0x1FFF).view(torch.float32) for w in ws]
    inp = K.GemmInput(n, n, n, dtype, False, tb)
    st = torch.cuda.Stream()
    bufs = [x.clone(), torch.empty_like(x)]
    torch.cuda.synchronize()
    with torch.cuda.stream(st):
        for i in range(links):
            t = K.GemmTuning(*tuples[i % len(tuples)])
            src, dst = bufs[i % 2], bufs[(i + 1) % 2]
            if dtype == "tf32" and i > 0:
                # tf32 rounds operands in hardware: truncate the fp32 output first (another kernel)
                src.copy_((src.view(torch.int32) & ~0x1FFF).view(torch.float32))
            K.execute_gemm(inp, t, src, ws[i], dst, mode="fast", stream=st.cuda_stream)
    torch.cuda.synchronize()
    ref = x.double().view(n, n)
    for i in range(links):
        if dtype == "tf32" and i > 0:
            ref = (ref.float().view(torch.int32) & ~0x1FFF).view(torch.float32).double()
        w = ws[i].double().view(n, n)
        ref = ref @ (w.t() if tb else w)
    got = bufs[links % 2].double().view(n, n)
    err = ((got - ref).abs().max() / ref.abs().max().clamp(min=1.0)).item()
    return err


def test_simt_chain(cuda):
    tuples = [(4, 4, 64, 64, 16, 1, 1, 1), (2, 4, 32, 64, 32, 1, 2, 4), (4, 2, 64, 32, 16, 2, 1, 8)]
    assert _chain("f32", tuples) < 1e-5


def test_tensor_core_chain(cuda):
    tuples = [(8, 8, 128, 128, 32, 1, 1, 1), (8, 4, 256, 128, 32, 2, 1, 2), (8, 8, 128, 64, 32, 2, 1, 4)]
    assert _chain("tf32", tuples, tb=True) < 1e-3

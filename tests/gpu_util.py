"""Shared helpers of the gpu-marked parity tests (device side via the
product package, checking side via the oracle)."""
import numpy as np
import torch

import oracle_libs as O
import paper_1802_05371_b200 as K

NP = {"f32": np.float32, "f64": np.float64}
TD = {"f32": torch.float32, "f64": torch.float64}


def dev(x, device="cuda:0"):
    return torch.from_numpy(np.ascontiguousarray(x)).to(device)


def run_gemm(inp: K.GemmInput, t: K.GemmTuning, a, b, mode="parity"):
    c = K.execute_gemm(inp, t, dev(a), dev(b), mode=mode)
    torch.cuda.synchronize()
    return c.cpu().numpy()


def run_conv(inp: K.ConvInput, t: K.ConvTuning, img, flt, mode="parity"):
    o = K.execute_conv(inp, t, dev(img), dev(flt), mode=mode)
    torch.cuda.synchronize()
    return o.cpu().numpy()


def bitwise_equal(x, y) -> bool:
    x = np.ascontiguousarray(x)
    y = np.ascontiguousarray(y)
    return x.dtype == y.dtype and x.shape == y.shape and np.array_equal(x.view(np.uint8), y.view(np.uint8))


def first_mismatch(x, y):
    bad = np.nonzero(x.view(np.uint8).reshape(x.size, -1).any(axis=1) !=
                     y.view(np.uint8).reshape(y.size, -1).any(axis=1))[0]
    diff = np.nonzero(x != y)[0]
    i = int(diff[0]) if diff.size else (int(bad[0]) if bad.size else -1)
    return i, (x[i] if i >= 0 else None), (y[i] if i >= 0 else None)

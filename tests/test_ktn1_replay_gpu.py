"""Replay of the committed KTN1 golden vectors (tests/golden/ktn1, made by
make_golden_ktn1.py from the UNMODIFIED reference executors): the B200
PARITY kernels reproduce the stored reference outputs bit for bit, with no
CPU oracle run."""
import json
import os

import numpy as np
import pytest
import torch

import paper_1802_05371_b200 as K

pytestmark = pytest.mark.gpu

DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ktn1")
CASES = json.load(open(os.path.join(DIR, "manifest.json")))["cases"]


def load(name):
    return K.read_tensor(os.path.join(DIR, name))


@pytest.mark.parametrize("case", CASES, ids=[f"{c['kind']}{i}" for i, c in enumerate(CASES)])
def test_replay_bitwise(cuda, case):
    t = [int(x) for x in case["tuning"]]
    if case["kind"] == "gemm":
        inp = K.GemmInput(case["m"], case["n"], case["k"], case["dtype"], bool(case["trans_a"]), bool(case["trans_b"]))
        a, b, want = load(case["a"]), load(case["b"]), load(case["c"])
        got = K.execute_gemm(inp, K.GemmTuning(*t), torch.from_numpy(a.ravel()).cuda(),
                             torch.from_numpy(b.ravel()).cuda(), mode="parity")
    else:
        inp = K.ConvInput(*case["dims"], case["dtype"])
        img, flt, want = load(case["images"]), load(case["filters"]), load(case["outputs"])
        got = K.execute_conv(inp, K.ConvTuning(*t), torch.from_numpy(img.ravel()).cuda(),
                             torch.from_numpy(flt.ravel()).cuda(), mode="parity")
    torch.cuda.synchronize()
    got = got.cpu().numpy()
    assert np.array_equal(got.view(np.uint8), want.ravel().view(np.uint8))

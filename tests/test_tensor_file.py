"""KTN1 tensor files (tensor_file.cpp:36-112): the bytes this build writes
equal the reference writer's, both read back exactly, and malformed files /
unsupported dtypes fail with the reference's error classes."""
import ctypes
import os

import numpy as np
import pytest

import oracle_libs as O
import paper_1802_05371_b200 as K


@pytest.mark.parametrize("dtype,shape", [(np.float32, (7,)), (np.float32, (3, 5, 2)), (np.float64, (4, 9)),
                                         (np.float64, (1, 1, 1, 1, 1, 1, 1, 2))])
def test_bytes_equal_reference_and_round_trip(tmp_path, dtype, shape):
    a = np.random.default_rng(1).standard_normal(shape).astype(dtype)
    ours = tmp_path / "ours.ktn"
    K.write_tensor(str(ours), a)
    back = K.read_tensor(str(ours))
    assert back.dtype == a.dtype and back.shape == a.shape and np.array_equal(back.view(np.uint8), a.view(np.uint8))
    raw = ours.read_bytes()
    assert raw[:4] == b"KTN1" and int.from_bytes(raw[4:8], "little") == a.itemsize
    lib = O.reference()
    if lib is None:
        pytest.skip("reference library (oracle/_ref) not built")
    ref = tmp_path / "ref.ktn"
    dims = (ctypes.c_int64 * len(shape))(*shape)
    assert lib.ref_write_tensor(str(ref).encode(), int(dtype == np.float64), dims, len(shape),
                                a.ctypes.data_as(ctypes.c_void_p)) == 0
    assert ref.read_bytes() == raw


def test_errors(tmp_path):
    with pytest.raises(K.InvalidArgument, match="not supported"):
        K.write_tensor(str(tmp_path / "x.ktn"), np.zeros(3, np.float16))
    p = tmp_path / "t.ktn"
    K.write_tensor(str(p), np.arange(12, dtype=np.float32).reshape(3, 4))
    data = p.read_bytes()
    (tmp_path / "trunc.ktn").write_bytes(data[:-4])
    with pytest.raises(K.KtuneError, match="truncated"):
        K.read_tensor(str(tmp_path / "trunc.ktn"))
    (tmp_path / "magic.ktn").write_bytes(b"NOPE" + data[4:])
    with pytest.raises(K.KtuneError, match="not a tensor file"):
        K.read_tensor(str(tmp_path / "magic.ktn"))
    with pytest.raises(K.KtuneError, match="cannot open"):
        K.read_tensor(str(tmp_path / "missing.ktn"))

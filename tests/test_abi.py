"""The C-ABI library loads and exports every entry point include/ktune_b200.h
declares (no device calls: this runs on CPU-only hosts too)."""
import ctypes
import os
import re

import paper_1802_05371_b200 as K
from paper_1802_05371_b200 import _lib

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ktune_b200.h")


def declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"KTUNE_API\s+(?:int|const char\*)\s+(ktune_\w+)\(", text)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert set(declared()) <= set(_lib._SIGNATURES)


def test_abi_version_and_error_channel():
    assert _lib.lib().ktune_abi_version() == 1
    try:
        K.estimate_resources(K.GemmInput(-1, 1, 1), K.GemmTuning())
    except K.InvalidArgument as e:
        assert e.status == _lib.ERR_INVALID_ARGUMENT and "m must be >= 1" in str(e)
    else:
        raise AssertionError("expected InvalidArgument")


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.GemmInputC) == 40
    assert ctypes.sizeof(_lib.ConvInputC) == 64
    assert ctypes.sizeof(_lib.GemmTuningC) == 32
    assert ctypes.sizeof(_lib.ConvTuningC) == 48
    assert ctypes.sizeof(_lib.HwC) == 88
    assert ctypes.sizeof(_lib.MeasureOptionsC) == 24

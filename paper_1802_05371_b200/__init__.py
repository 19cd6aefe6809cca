"""B200-native build of ISAAC's GEMM/CONV tuning path (arXiv 1802.05371).

Python mirror of the reference ``ktune`` interface for this path
(/root/reference/proj/include/ktune/{param_space,backends}.hpp): the same
descriptors, tuning tuples, legality, enumeration, features and executors,
backed by libktune_b200.so (hand-written sm_100a kernels behind the C-ABI of
include/ktune_b200.h).  Tensors passed to the device executors are torch CUDA
tensors; there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import asdict, dataclass, fields

import numpy as np

from . import _lib
from ._lib import (CONV_PARAMS, DTYPE_CODES, DTYPE_NAMES, GEMM_PARAMS, CudaError, InvalidArgument, KtuneError,
                   Unsupported, WorkspaceTooSmall)

__all__ = [
    "GemmInput", "ConvInput", "GemmTuning", "ConvTuning", "HardwareDescriptor", "ResourceUsage",
    "LegalityVerdict", "estimate_resources", "is_legal", "enumerate_legal", "encode_features",
    "build_indirection_table", "execute_gemm", "execute_conv", "execute_gemm_host", "execute_conv_host",
    "gemm_workspace_size", "conv_workspace_size", "measure", "B200Backend", "l2_flush", "KtuneError",
    "InvalidArgument", "Unsupported", "WorkspaceTooSmall", "CudaError", "FIXTURES", "write_tensor", "read_tensor",
]

FIXTURES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fixtures")
REJECT_REASONS = ("divisibility", "shared_memory", "registers", "threads")


# ---------------------------------------------------------------------------
# descriptors (param_space.hpp:20-106)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class GemmInput:
    m: int = 1
    n: int = 1
    k: int = 1
    dtype: str = "f32"
    trans_a: bool = False
    trans_b: bool = False

    def c(self) -> _lib.GemmInputC:
        if self.dtype not in DTYPE_CODES:
            raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"unknown dtype name: {self.dtype}")
        return _lib.GemmInputC(self.m, self.n, self.k, DTYPE_CODES[self.dtype], int(self.trans_a),
                               int(self.trans_b), 0)

    @property
    def flops(self) -> float:
        return 2.0 * self.m * self.n * self.k


@dataclass(frozen=True)
class ConvInput:
    n_batch: int = 1
    p: int = 1
    q: int = 1
    k_filters: int = 1
    c: int = 1
    r: int = 1
    s: int = 1
    dtype: str = "f32"

    def h(self) -> int:
        return self.p + self.r - 1

    def w(self) -> int:
        return self.q + self.s - 1

    def cstruct(self) -> _lib.ConvInputC:
        if self.dtype not in DTYPE_CODES:
            raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"unknown dtype name: {self.dtype}")
        return _lib.ConvInputC(self.n_batch, self.p, self.q, self.k_filters, self.c, self.r, self.s,
                               DTYPE_CODES[self.dtype], 0)

    @property
    def flops(self) -> float:
        return 2.0 * self.n_batch * self.p * self.q * self.k_filters * self.c * self.r * self.s

    def sizes(self):
        """(images, filters, outputs) element counts."""
        return (self.c * self.h() * self.w() * self.n_batch, self.c * self.r * self.s * self.k_filters,
                self.k_filters * self.p * self.q * self.n_batch)


@dataclass(frozen=True)
class GemmTuning:
    m_s: int = 1
    n_s: int = 1
    m_l: int = 1
    n_l: int = 1
    u: int = 1
    k_s: int = 1
    k_l: int = 1
    k_g: int = 1

    def values(self):
        return [getattr(self, n) for n in GEMM_PARAMS]

    @classmethod
    def from_values(cls, v):
        v = [int(x) for x in v]
        if len(v) != 8:
            raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "gemm tuning vector must have 8 entries")
        return cls(*v)

    def c(self) -> _lib.GemmTuningC:
        return _lib.GemmTuningC(*self.values())


@dataclass(frozen=True)
class ConvTuning:
    k_s: int = 1
    p_s: int = 1
    q_s: int = 1
    n_s: int = 1
    k_l: int = 1
    p_l: int = 1
    q_l: int = 1
    n_l: int = 1
    u: int = 1
    c_s: int = 1
    c_l: int = 1
    c_g: int = 1

    def values(self):
        return [getattr(self, n) for n in CONV_PARAMS]

    @classmethod
    def from_values(cls, v):
        v = [int(x) for x in v]
        if len(v) != 12:
            raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "conv tuning vector must have 12 entries")
        return cls(*v)

    def c(self) -> _lib.ConvTuningC:
        return _lib.ConvTuningC(*self.values())


@dataclass(frozen=True)
class HardwareDescriptor:
    max_shared_bytes_per_block: int = 256
    max_registers_per_thread: int = 16
    max_threads_per_block: int = 64
    max_warps_per_multiprocessor: int = 8
    warp_size: int = 8
    alu_latency: float = 6.0
    alu_throughput: float = 1.0
    mem_latency: float = 48.0
    mem_throughput: float = 4.0
    clock_hz: float = 1.0e9
    num_multiprocessors: int = 16

    @classmethod
    def from_json_text(cls, text: str) -> "HardwareDescriptor":
        out = _lib.HwC()
        _lib.call("ktune_hw_from_json", text.encode(), ctypes.byref(out))
        return cls(**{f.name: getattr(out, f.name) for f in fields(cls)})

    @classmethod
    def load(cls, path: str) -> "HardwareDescriptor":
        with open(path) as fh:
            return cls.from_json_text(fh.read())

    @classmethod
    def b200(cls) -> "HardwareDescriptor":
        """The B200 descriptor shipped in fixtures/hw/b200.json."""
        return cls.load(os.path.join(FIXTURES, "hw", "b200.json"))

    def c(self) -> _lib.HwC:
        return _lib.HwC(*[getattr(self, f.name) for f in fields(self)])


def load_bounds_text(path: str) -> str:
    with open(path) as fh:
        return fh.read()


@dataclass(frozen=True)
class ResourceUsage:
    shared_bytes: int
    registers_per_thread: int
    threads_per_block: int


@dataclass(frozen=True)
class LegalityVerdict:
    accepted: bool
    reason: str
    detail: str

    def __bool__(self):
        return self.accepted


def _is_conv(x) -> bool:
    return isinstance(x, (ConvInput, ConvTuning))


def _in(x):
    return x.cstruct() if isinstance(x, ConvInput) else x.c()


# ---------------------------------------------------------------------------
# space (param_space.cpp)
# ---------------------------------------------------------------------------

def estimate_resources(inp, t) -> ResourceUsage:
    out = _lib.ResourcesC()
    fn = "ktune_estimate_resources_conv" if _is_conv(inp) else "ktune_estimate_resources_gemm"
    _lib.call(fn, ctypes.byref(_in(inp)), ctypes.byref(t.c()), ctypes.byref(out))
    return ResourceUsage(out.shared_bytes, out.registers_per_thread, out.threads_per_block)


def is_legal(inp, t, hw: HardwareDescriptor | None = None) -> LegalityVerdict:
    hw = hw or HardwareDescriptor()
    acc, why = ctypes.c_int(), ctypes.c_int()
    fn = "ktune_is_legal_conv" if _is_conv(inp) else "ktune_is_legal_gemm"
    _lib.call(fn, ctypes.byref(hw.c()), ctypes.byref(_in(inp)), ctypes.byref(t.c()), ctypes.byref(acc),
              ctypes.byref(why))
    detail = _lib.lib().ktune_last_text().decode()
    return LegalityVerdict(bool(acc.value), REJECT_REASONS[why.value], detail)


def enumerate_legal(inp, hw: HardwareDescriptor | None = None, bounds_json: str | None = None,
                    as_array: bool = False):
    """Every legal tuning in lexicographic order (param_space.cpp:536-628)."""
    hw = hw or HardwareDescriptor()
    conv = _is_conv(inp)
    width = 12 if conv else 8
    fn = "ktune_enumerate_legal_conv" if conv else "ktune_enumerate_legal_gemm"
    count = ctypes.c_int64()
    bj = (bounds_json or "").encode()
    _lib.call(fn, ctypes.byref(hw.c()), ctypes.byref(_in(inp)), bj, None, 0, ctypes.byref(count))
    arr = np.zeros((count.value, width), np.int32)
    _lib.call(fn, ctypes.byref(hw.c()), ctypes.byref(_in(inp)), bj, arr.ctypes.data_as(ctypes.c_void_p),
              count.value, ctypes.byref(count))
    if as_array:
        return arr
    cls = ConvTuning if conv else GemmTuning
    return [cls(*map(int, row)) for row in arr]


def encode_features(inp, t) -> np.ndarray:
    conv = _is_conv(inp)
    out = np.zeros(19 if conv else 14, np.float64)
    fn = "ktune_encode_features_conv" if conv else "ktune_encode_features_gemm"
    _lib.call(fn, ctypes.byref(_in(inp)), ctypes.byref(t.c()), out.ctypes.data_as(ctypes.c_void_p))
    return out


def build_indirection_table(inp: ConvInput) -> np.ndarray:
    """(C*R*S, 4) int64 rows {c, r, s, image_offset} (backends.cpp:197-216)."""
    count = ctypes.c_int64()
    _lib.call("ktune_build_indirection_table", ctypes.byref(inp.cstruct()), None, 0, ctypes.byref(count))
    out = np.zeros((count.value, 4), np.int64)
    _lib.call("ktune_build_indirection_table", ctypes.byref(inp.cstruct()), out.ctypes.data_as(ctypes.c_void_p),
              count.value, ctypes.byref(count))
    return out


# ---------------------------------------------------------------------------
# device executors (backends.cpp:228-444 -> sm_100a kernels)
# ---------------------------------------------------------------------------

def _mode(mode) -> int:
    if mode in ("fast", _lib.MODE_FAST):
        return _lib.MODE_FAST
    if mode in ("parity", _lib.MODE_PARITY):
        return _lib.MODE_PARITY
    raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"unknown mode {mode!r}")


def gemm_workspace_size(inp: GemmInput, t: GemmTuning) -> int:
    n = ctypes.c_size_t()
    _lib.call("ktune_gemm_workspace_size", ctypes.byref(inp.c()), ctypes.byref(t.c()), ctypes.byref(n))
    return n.value


def gemm_launch_info(inp: GemmInput, t: GemmTuning, mode="fast") -> dict:
    """Launch geometry and kernel family the library uses (no launch)."""
    th, sm, grid = ctypes.c_int(), ctypes.c_size_t(), (ctypes.c_int * 3)()
    fam = ctypes.create_string_buffer(64)
    _lib.call("ktune_gemm_launch_info", ctypes.byref(inp.c()), ctypes.byref(t.c()), _mode(mode), ctypes.byref(th),
              ctypes.byref(sm), grid, fam, 64)
    return {"threads": th.value, "smem": sm.value, "grid": list(grid), "family": fam.value.decode()}


def conv_workspace_size(inp: ConvInput, t: ConvTuning) -> int:
    n = ctypes.c_size_t()
    _lib.call("ktune_conv_workspace_size", ctypes.byref(inp.cstruct()), ctypes.byref(t.c()), ctypes.byref(n))
    return n.value


_workspaces: dict = {}
_retired: list = []


def _workspace(device, nbytes: int, stream=None):
    """Grow-only workspace per (device, stream), zero-initialised (the split-K
    counter region must start at zero; launches leave it zero).  A launch on
    another stream never shares counters or partials with this one, and a
    grown-out buffer is kept alive (work still in flight on the stream, or a
    captured CUDA graph, may reference it)."""
    import torch
    if nbytes == 0:
        return None, 0
    key = (torch.device(device).index, int(stream or 0))
    ws = _workspaces.get(key)
    if ws is None or ws.numel() < nbytes:
        if ws is not None:
            _retired.append(ws)
        ws = torch.zeros(nbytes, dtype=torch.uint8, device=device)
        if not torch.cuda.is_current_stream_capturing():
            torch.cuda.current_stream(device).synchronize()  # zeroed before any stream uses it
        _workspaces[key] = ws
    return ws, ws.numel()


_TORCH_DT = {"f32": "float32", "f64": "float64", "bf16": "bfloat16", "f16": "float16", "tf32": "float32"}


def _check_tensor(x, n, dtype, what):
    import torch
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"{what} must be a CUDA tensor")
    if not x.is_contiguous():
        raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"{what} must be contiguous")
    if x.dtype != getattr(torch, _TORCH_DT[dtype]):
        raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"{what} has dtype {x.dtype}, expected {dtype}")
    if x.numel() != n:
        raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"execute: operand size mismatch ({what})")


def execute_gemm(inp: GemmInput, t: GemmTuning, a, b, c=None, mode="parity", stream=None):
    """C = op(A) op(B) on the current CUDA stream; returns C (fp32 for the
    tensor-core dtypes, else inp.dtype)."""
    import torch
    out_dt = "f32" if inp.dtype in ("bf16", "f16", "tf32") else inp.dtype
    _check_tensor(a, inp.m * inp.k, inp.dtype, "a")
    _check_tensor(b, inp.k * inp.n, inp.dtype, "b")
    if c is None:
        c = torch.empty(inp.m * inp.n, dtype=getattr(torch, _TORCH_DT[out_dt]), device=a.device)
    _check_tensor(c, inp.m * inp.n, out_dt, "c")
    s = stream if stream is not None else torch.cuda.current_stream(a.device).cuda_stream
    ws, wsb = _workspace(a.device, gemm_workspace_size(inp, t), s)
    _lib.call("ktune_gemm", ctypes.byref(inp.c()), ctypes.byref(t.c()), _mode(mode), a.data_ptr(), b.data_ptr(),
              c.data_ptr(), None if ws is None else ws.data_ptr(), wsb, s)
    return c


def execute_conv(inp: ConvInput, t: ConvTuning, images, filters, outputs=None, mode="parity", stream=None):
    import torch
    ni, nf, no = inp.sizes()
    out_dt = "f32" if inp.dtype in ("bf16", "f16", "tf32") else inp.dtype
    _check_tensor(images, ni, inp.dtype, "images")
    _check_tensor(filters, nf, inp.dtype, "filters")
    if outputs is None:
        outputs = torch.empty(no, dtype=getattr(torch, _TORCH_DT[out_dt]), device=images.device)
    _check_tensor(outputs, no, out_dt, "outputs")
    s = stream if stream is not None else torch.cuda.current_stream(images.device).cuda_stream
    ws, wsb = _workspace(images.device, conv_workspace_size(inp, t), s)
    _lib.call("ktune_conv", ctypes.byref(inp.cstruct()), ctypes.byref(t.c()), _mode(mode), images.data_ptr(),
              filters.data_ptr(), outputs.data_ptr(), None if ws is None else ws.data_ptr(), wsb, s)
    return outputs


_NP_DT = {"f32": np.float32, "f64": np.float64, "bf16": np.uint16, "f16": np.float16, "tf32": np.float32}


def execute_gemm_host(inp: GemmInput, t: GemmTuning, a: np.ndarray, b: np.ndarray, mode="parity") -> np.ndarray:
    """The executor's host-span contract through the C-ABI (copies in and out)."""
    out_np = np.float32 if inp.dtype in ("bf16", "f16", "tf32") else _NP_DT[inp.dtype]
    a = np.ascontiguousarray(a, _NP_DT[inp.dtype])
    b = np.ascontiguousarray(b, _NP_DT[inp.dtype])
    c = np.empty(inp.m * inp.n, out_np)
    _lib.call("ktune_execute_gemm", ctypes.byref(inp.c()), ctypes.byref(t.c()), _mode(mode),
              a.ctypes.data_as(ctypes.c_void_p), a.size, b.ctypes.data_as(ctypes.c_void_p), b.size,
              c.ctypes.data_as(ctypes.c_void_p), c.size)
    return c


def execute_conv_host(inp: ConvInput, t: ConvTuning, images, filters, mode="parity") -> np.ndarray:
    out_np = np.float32 if inp.dtype in ("bf16", "f16", "tf32") else _NP_DT[inp.dtype]
    images = np.ascontiguousarray(images, _NP_DT[inp.dtype])
    filters = np.ascontiguousarray(filters, _NP_DT[inp.dtype])
    out = np.empty(inp.sizes()[2], out_np)
    _lib.call("ktune_execute_conv", ctypes.byref(inp.cstruct()), ctypes.byref(t.c()), _mode(mode),
              images.ctypes.data_as(ctypes.c_void_p), images.size, filters.ctypes.data_as(ctypes.c_void_p),
              filters.size, out.ctypes.data_as(ctypes.c_void_p), out.size)
    return out


def write_tensor(path: str, array) -> None:
    """KTN1 file (write_tensor, tensor_file.cpp:36-69): f32 / f64 arrays."""
    a = np.ascontiguousarray(array)
    code = {np.dtype(np.float32): DTYPE_CODES["f32"], np.dtype(np.float64): DTYPE_CODES["f64"]}.get(a.dtype)
    if code is None:
        raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, f"{a.dtype} tensor files are not supported")
    dims = (ctypes.c_int64 * max(1, a.ndim))(*a.shape)
    _lib.call("ktune_tensor_write", os.fsencode(path), code, dims, a.ndim, a.ctypes.data_as(ctypes.c_void_p))


def read_tensor(path: str) -> np.ndarray:
    """KTN1 file -> numpy array of its dtype and shape (read_tensor, :71-112)."""
    dt, nd = ctypes.c_int32(), ctypes.c_int32()
    dims = (ctypes.c_int64 * 8)()
    _lib.call("ktune_tensor_read", os.fsencode(path), ctypes.byref(dt), dims, ctypes.byref(nd), None, 0)
    shape = tuple(dims[i] for i in range(nd.value))
    out = np.empty(shape, np.float32 if DTYPE_NAMES[dt.value] == "f32" else np.float64)
    _lib.call("ktune_tensor_read", os.fsencode(path), ctypes.byref(dt), dims, ctypes.byref(nd),
              out.ctypes.data_as(ctypes.c_void_p), out.size)
    return out


def l2_flush(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
    _lib.call("ktune_l2_flush", s)


# ---------------------------------------------------------------------------
# measurement (CpuBackend::measure -> CUDA-event device timing)
# ---------------------------------------------------------------------------

def measure(inp, t, hw: HardwareDescriptor | None = None, mode="fast", repetitions=3, warmup=1, flush_l2=True,
            seed=0x5EED) -> float:
    """GFLOPS of one legal (input, tuning) pair on the current device."""
    hw = hw or HardwareDescriptor()
    opts = _lib.MeasureOptionsC(_mode(mode), repetitions, warmup, int(flush_l2), seed)
    g = ctypes.c_double()
    fn = "ktune_measure_conv" if _is_conv(inp) else "ktune_measure_gemm"
    _lib.call(fn, ctypes.byref(hw.c()), ctypes.byref(_in(inp)), ctypes.byref(t.c()), ctypes.byref(opts),
              ctypes.byref(g))
    return g.value


class B200Backend:
    """MeasurementBackend (backends.hpp:102-109) timed on the GPU."""

    def __init__(self, hw: HardwareDescriptor | None = None, mode="fast", repetitions=3, warmup=1,
                 flush_l2=True):
        if repetitions < 1:
            raise InvalidArgument(_lib.ERR_INVALID_ARGUMENT, "B200Backend: repetitions must be >= 1")
        self.hw = hw or HardwareDescriptor()
        self.mode = mode
        self.repetitions = repetitions
        self.warmup = warmup
        self.flush_l2 = flush_l2

    def name(self) -> str:
        return "b200-parity" if _mode(self.mode) == _lib.MODE_PARITY else "b200"

    def measure(self, inp, t) -> float:
        return measure(inp, t, self.hw, self.mode, self.repetitions, self.warmup, self.flush_l2)

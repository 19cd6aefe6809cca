"""ctypes binding of libktune_b200.so (the C-ABI of include/ktune_b200.h).

The shared library is built in-tree (``make -C paper_1802_05371_b200`` or
``__graft_entry__.build()``).  There is no Python or CPU fallback: if the
library is missing, importing the device API raises immediately.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libktune_b200.so")

# ktune_status
OK, ERR_INVALID_ARGUMENT, ERR_UNSUPPORTED, ERR_CUDA, ERR_RUNTIME, ERR_WORKSPACE = range(6)
# ktune_dtype
DTYPE_CODES = {"f16": 0, "f32": 1, "f64": 2, "bf16": 3, "tf32": 4}
DTYPE_NAMES = {v: k for k, v in DTYPE_CODES.items()}
MODE_FAST, MODE_PARITY = 0, 1


class KtuneError(RuntimeError):
    """Base of the C-ABI failures (status != KTUNE_OK)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class InvalidArgument(KtuneError, ValueError):
    """std::invalid_argument in the reference (illegal tuple, size mismatch)."""


class Unsupported(InvalidArgument):
    """dtype / tuple this build cannot execute."""


class WorkspaceTooSmall(InvalidArgument):
    pass


class CudaError(KtuneError):
    pass


_ERRORS = {ERR_INVALID_ARGUMENT: InvalidArgument, ERR_UNSUPPORTED: Unsupported, ERR_CUDA: CudaError,
           ERR_RUNTIME: KtuneError, ERR_WORKSPACE: WorkspaceTooSmall}


class GemmInputC(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64), ("k", ctypes.c_int64), ("dtype", ctypes.c_int32),
                ("trans_a", ctypes.c_int32), ("trans_b", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class ConvInputC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("n_batch", "p", "q", "k_filters", "c", "r", "s")] + [
        ("dtype", ctypes.c_int32), ("reserved", ctypes.c_int32)]


GEMM_PARAMS = ("m_s", "n_s", "m_l", "n_l", "u", "k_s", "k_l", "k_g")
CONV_PARAMS = ("k_s", "p_s", "q_s", "n_s", "k_l", "p_l", "q_l", "n_l", "u", "c_s", "c_l", "c_g")


class GemmTuningC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in GEMM_PARAMS]


class ConvTuningC(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in CONV_PARAMS]


HW_FIELDS = (("max_shared_bytes_per_block", ctypes.c_int64), ("max_registers_per_thread", ctypes.c_int64),
             ("max_threads_per_block", ctypes.c_int64), ("max_warps_per_multiprocessor", ctypes.c_int64),
             ("warp_size", ctypes.c_int64), ("alu_latency", ctypes.c_double), ("alu_throughput", ctypes.c_double),
             ("mem_latency", ctypes.c_double), ("mem_throughput", ctypes.c_double), ("clock_hz", ctypes.c_double),
             ("num_multiprocessors", ctypes.c_int64))


class HwC(ctypes.Structure):
    _fields_ = list(HW_FIELDS)


class ResourcesC(ctypes.Structure):
    _fields_ = [("shared_bytes", ctypes.c_int64), ("registers_per_thread", ctypes.c_int64),
                ("threads_per_block", ctypes.c_int64)]


class MeasureOptionsC(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int32), ("repetitions", ctypes.c_int32), ("warmup", ctypes.c_int32),
                ("flush_l2", ctypes.c_int32), ("seed", ctypes.c_uint64)]


class GemmDistC(ctypes.Structure):
    _fields_ = [("shapes", ctypes.c_void_p), ("n_shapes", ctypes.c_int32), ("weights", ctypes.c_void_p),
                ("fixed_fraction", ctypes.c_double), ("use_ranges", ctypes.c_int32)] + [
        (n, ctypes.c_int32) for n in ("m_lo", "m_hi", "n_lo", "n_hi", "k_lo", "k_hi", "dtype",
                                       "randomize_transpose")]


class ConvDistC(ctypes.Structure):
    _fields_ = [("shapes", ctypes.c_void_p), ("n_shapes", ctypes.c_int32), ("weights", ctypes.c_void_p),
                ("fixed_fraction", ctypes.c_double), ("use_ranges", ctypes.c_int32)] + [
        (n, ctypes.c_int32) for n in ("n_lo", "n_hi", "p_lo", "p_hi", "q_lo", "q_hi", "k_lo", "k_hi", "c_lo",
                                       "c_hi")] + [("rs_choices", ctypes.c_void_p), ("n_rs", ctypes.c_int32),
                                                   ("dtype", ctypes.c_int32)]


_P = ctypes.POINTER
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_ip = _P(ctypes.c_int)

_SIGNATURES = {
    "ktune_abi_version": ([], ctypes.c_int),
    "ktune_last_error": ([], ctypes.c_char_p),
    "ktune_last_text": ([], ctypes.c_char_p),
    "ktune_set_device": ([ctypes.c_int], ctypes.c_int),
    "ktune_hw_default": ([_P(HwC)], ctypes.c_int),
    "ktune_hw_from_json": ([ctypes.c_char_p, _P(HwC)], ctypes.c_int),
    "ktune_estimate_resources_gemm": ([_P(GemmInputC), _P(GemmTuningC), _P(ResourcesC)], ctypes.c_int),
    "ktune_estimate_resources_conv": ([_P(ConvInputC), _P(ConvTuningC), _P(ResourcesC)], ctypes.c_int),
    "ktune_is_legal_gemm": ([_P(HwC), _P(GemmInputC), _P(GemmTuningC), _ip, _ip], ctypes.c_int),
    "ktune_is_legal_conv": ([_P(HwC), _P(ConvInputC), _P(ConvTuningC), _ip, _ip], ctypes.c_int),
    "ktune_enumerate_legal_gemm": ([_P(HwC), _P(GemmInputC), ctypes.c_char_p, _vp, _i64, _P(_i64)], ctypes.c_int),
    "ktune_enumerate_legal_conv": ([_P(HwC), _P(ConvInputC), ctypes.c_char_p, _vp, _i64, _P(_i64)], ctypes.c_int),
    "ktune_encode_features_gemm": ([_P(GemmInputC), _P(GemmTuningC), _vp], ctypes.c_int),
    "ktune_encode_features_conv": ([_P(ConvInputC), _P(ConvTuningC), _vp], ctypes.c_int),
    "ktune_build_indirection_table": ([_P(ConvInputC), _vp, _i64, _P(_i64)], ctypes.c_int),
    "ktune_generate_gemm_shard": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(GemmDistC), ctypes.c_int32,
                                   ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, _P(MeasureOptionsC),
                                   ctypes.c_char_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_int64, _P(ctypes.c_int64), _P(ctypes.c_int64), _P(ctypes.c_int64),
                                   _P(ctypes.c_int64)], ctypes.c_int),
    "ktune_generate_conv_shard": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(ConvDistC), ctypes.c_int32,
                                   ctypes.c_uint64, ctypes.c_int32, ctypes.c_int32, _P(MeasureOptionsC),
                                   ctypes.c_char_p,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_int64, _P(ctypes.c_int64), _P(ctypes.c_int64), _P(ctypes.c_int64),
                                   _P(ctypes.c_int64)], ctypes.c_int),
    "ktune_shard_lpt": ([ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p], ctypes.c_int),
    "ktune_gemm_workspace_size": ([_P(GemmInputC), _P(GemmTuningC), _P(ctypes.c_size_t)], ctypes.c_int),
    "ktune_gemm_launch_info": ([_P(GemmInputC), _P(GemmTuningC), ctypes.c_int, _P(ctypes.c_int), _P(ctypes.c_size_t),
                                _P(ctypes.c_int), ctypes.c_char_p, ctypes.c_size_t], ctypes.c_int),
    "ktune_conv_workspace_size": ([_P(ConvInputC), _P(ConvTuningC), _P(ctypes.c_size_t)], ctypes.c_int),
    "ktune_gemm": ([_P(GemmInputC), _P(GemmTuningC), ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp],
                   ctypes.c_int),
    "ktune_conv": ([_P(ConvInputC), _P(ConvTuningC), ctypes.c_int, _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp],
                   ctypes.c_int),
    "ktune_execute_gemm": ([_P(GemmInputC), _P(GemmTuningC), ctypes.c_int, _vp, _i64, _vp, _i64, _vp, _i64],
                           ctypes.c_int),
    "ktune_execute_conv": ([_P(ConvInputC), _P(ConvTuningC), ctypes.c_int, _vp, _i64, _vp, _i64, _vp, _i64],
                           ctypes.c_int),
    "ktune_measure_gemm": ([_P(HwC), _P(GemmInputC), _P(GemmTuningC), _P(MeasureOptionsC), _P(ctypes.c_double)],
                           ctypes.c_int),
    "ktune_measure_conv": ([_P(HwC), _P(ConvInputC), _P(ConvTuningC), _P(MeasureOptionsC), _P(ctypes.c_double)],
                           ctypes.c_int),
    "ktune_l2_flush": ([_vp], ctypes.c_int),
    "ktune_peak_gflops": ([_P(HwC), _P(ctypes.c_double)], ctypes.c_int),
    "ktune_analytical_gflops_gemm": ([_P(HwC), _P(GemmInputC), _P(GemmTuningC), _P(ctypes.c_double)], ctypes.c_int),
    "ktune_analytical_gflops_conv": ([_P(HwC), _P(ConvInputC), _P(ConvTuningC), _P(ctypes.c_double)], ctypes.c_int),
    "ktune_calibrate_gemm": ([_P(HwC), _P(GemmInputC), ctypes.c_char_p, _i64, ctypes.c_uint64, ctypes.c_double],
                             ctypes.c_int),
    "ktune_calibrate_conv": ([_P(HwC), _P(ConvInputC), ctypes.c_char_p, _i64, ctypes.c_uint64, ctypes.c_double],
                             ctypes.c_int),
    "ktune_acceptance_rate_gemm": ([_P(HwC), _P(GemmInputC), ctypes.c_char_p, _i64, ctypes.c_uint64,
                                    _P(ctypes.c_double)], ctypes.c_int),
    "ktune_uniform_acceptance_rate_gemm": ([_P(HwC), _P(GemmInputC), ctypes.c_char_p, _i64, ctypes.c_uint64,
                                            _P(ctypes.c_double)], ctypes.c_int),
    "ktune_predraw_gemm": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(GemmDistC), ctypes.c_int32,
                            ctypes.c_uint64, _vp, _vp, _P(_i64), _P(_i64)], ctypes.c_int),
    "ktune_predraw_conv": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(ConvDistC), ctypes.c_int32,
                            ctypes.c_uint64, _vp, _vp, _P(_i64), _P(_i64)], ctypes.c_int),
    "ktune_generate_gemm": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(GemmDistC), ctypes.c_int32,
                             ctypes.c_uint64, ctypes.c_int32, _P(MeasureOptionsC), _P(_i64), _P(_i64)],
                            ctypes.c_int),
    "ktune_gemm_dataset_csv": ([_vp, _vp, _vp, _i64, ctypes.c_char_p], ctypes.c_int),
    "ktune_conv_dataset_csv": ([_vp, _vp, _vp, _i64, ctypes.c_char_p], ctypes.c_int),
    "ktune_dataset_canonical": ([ctypes.c_char_p, ctypes.c_int32], ctypes.c_int),
    "ktune_mlp_train": ([ctypes.c_char_p, ctypes.c_int32, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                         ctypes.c_double, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, _P(ctypes.c_double),
                         _P(ctypes.c_int32), _vp], ctypes.c_int),
    "ktune_mlp_train_fast": ([ctypes.c_char_p, ctypes.c_int32, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                         ctypes.c_double, ctypes.c_int32, ctypes.c_uint64, ctypes.c_double, _P(ctypes.c_double),
                         _P(ctypes.c_int32), _vp], ctypes.c_int),
    "ktune_mlp_sweep_gemm": ([ctypes.c_char_p, _P(HwC), ctypes.c_char_p, _P(GemmInputC), ctypes.c_int32,
                              _P(ctypes.c_int64), _P(ctypes.c_double), _P(ctypes.c_double)], ctypes.c_int),
    "ktune_mlp_init": ([ctypes.c_int32, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_char_p],
                       ctypes.c_int),
    "ktune_mlp_predict_rows": ([ctypes.c_char_p, _vp, _i64, ctypes.c_int32, _vp], ctypes.c_int),
    "ktune_mlp_predict_gemm": ([ctypes.c_char_p, _P(GemmInputC), _vp, _i64, _vp], ctypes.c_int),
    "ktune_mlp_predict_gemm_fast": ([ctypes.c_char_p, _P(GemmInputC), _vp, _i64, _vp], ctypes.c_int),
    "ktune_mlp_predict_conv": ([ctypes.c_char_p, _P(ConvInputC), _vp, _i64, _vp], ctypes.c_int),
    "ktune_mlp_evaluate": ([ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int32, _P(ctypes.c_double)], ctypes.c_int),
    "ktune_infer_gemm": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(GemmInputC), ctypes.c_int32,
                          ctypes.c_int32, _P(MeasureOptionsC)], ctypes.c_int),
    "ktune_infer_conv": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(ConvInputC), ctypes.c_int32,
                          ctypes.c_int32, _P(MeasureOptionsC)], ctypes.c_int),
    "ktune_cache_key_gemm": ([_P(GemmInputC)], ctypes.c_int),
    "ktune_cache_key_conv": ([_P(ConvInputC)], ctypes.c_int),
    "ktune_cache_lookup_gemm": ([ctypes.c_char_p, _P(GemmInputC), _P(ctypes.c_int)], ctypes.c_int),
    "ktune_cache_lookup_conv": ([ctypes.c_char_p, _P(ConvInputC), _P(ctypes.c_int)], ctypes.c_int),
    "ktune_cache_store": ([ctypes.c_char_p, ctypes.c_char_p], ctypes.c_int),
    "ktune_select_conv": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, _P(ConvInputC),
                           ctypes.c_int32, _P(ConvTuningC), _P(ctypes.c_int32)], ctypes.c_int),
    "ktune_infer_gemm_shard": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(GemmInputC), ctypes.c_int32,
                                ctypes.c_int32, _P(MeasureOptionsC), ctypes.c_int32, ctypes.c_int32, _vp,
                                ctypes.c_int64, _P(ctypes.c_int64)], ctypes.c_int),
    "ktune_infer_conv_shard": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(ConvInputC), ctypes.c_int32,
                                ctypes.c_int32, _P(MeasureOptionsC), ctypes.c_int32, ctypes.c_int32, _vp,
                                ctypes.c_int64, _P(ctypes.c_int64)], ctypes.c_int),
    "ktune_infer_gemm_replay": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(GemmInputC), ctypes.c_int32,
                                 ctypes.c_char_p, _vp, ctypes.c_int64], ctypes.c_int),
    "ktune_infer_conv_replay": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, _P(ConvInputC), ctypes.c_int32,
                                 ctypes.c_char_p, _vp, ctypes.c_int64], ctypes.c_int),
    "ktune_select_gemm": ([_P(HwC), ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p, _P(GemmInputC),
                           ctypes.c_int32, _P(GemmTuningC), _P(ctypes.c_int32)], ctypes.c_int),
    "ktune_cli_main": ([ctypes.c_int, _P(ctypes.c_char_p)], ctypes.c_int),
    "ktune_tensor_write": ([ctypes.c_char_p, ctypes.c_int32, _P(ctypes.c_int64), ctypes.c_int32, _vp], ctypes.c_int),
    "ktune_tensor_read": ([ctypes.c_char_p, _P(ctypes.c_int32), _P(ctypes.c_int64), _P(ctypes.c_int32), _vp,
                           ctypes.c_int64], ctypes.c_int),
}

_lib = None


def lib():
    """The loaded C-ABI library (raises if it was never built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `make -C {HERE}` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        handle = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGNATURES.items():
            fn = getattr(handle, name, None)
            if fn is None:
                continue  # declared in the header but not in this build: surfaced by the export test
            fn.argtypes = args
            fn.restype = res
        _lib = handle
    return _lib


def text() -> str:
    """The library's thread-local text result (JSON / CSV / detail)."""
    return lib().ktune_last_text().decode()


def call(fn_name: str, *args) -> None:
    status = getattr(lib(), fn_name)(*args)
    if status != OK:
        msg = lib().ktune_last_error().decode(errors="replace")
        raise _ERRORS.get(status, KtuneError)(status, f"{fn_name}: {msg}")

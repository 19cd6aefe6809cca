"""The tuning pipeline over the C-ABI (reference: /root/reference/proj/
include/ktune/{sampler,perf_model,pipeline}.hpp): calibrated sampling,
dataset generation (sequential, or pre-drawn and sharded over GPUs with an
NCCL all-gather of the timing records), the GPU-trained MLP, runtime
selection with the result cache.

Formats stay byte-compatible with the reference: sampler JSON, dataset CSV
(pipeline.hpp:53-57), ktune-mlp-1 model JSON, ktune-result-1 result JSON.
"""
from __future__ import annotations

import ctypes
import json
import os
import time
from dataclasses import dataclass, field

import numpy as np

from . import (DTYPE_CODES, ConvInput, ConvTuning, GemmInput, GemmTuning, HardwareDescriptor, InvalidArgument,
               _lib, measure)

BACKENDS = {"analytical": 0, "b200": 1, "b200-parity": 2}


def _b(s):
    return None if s is None else s.encode()


# ---------------------------------------------------------------------------
# sampler (sampler.cpp)
# ---------------------------------------------------------------------------

def calibrate(probe, hw: HardwareDescriptor, bounds_json: str | None = None, n_uniform: int = 100000,
              seed: int = 0, alpha: float = 100.0) -> str:
    """Categorical sampler model JSON (sampler.cpp:101-138)."""
    if isinstance(probe, ConvInput):
        _lib.call("ktune_calibrate_conv", ctypes.byref(hw.c()), ctypes.byref(probe.cstruct()), _b(bounds_json or ""),
                  n_uniform, seed, alpha)
    else:
        _lib.call("ktune_calibrate_gemm", ctypes.byref(hw.c()), ctypes.byref(probe.c()), _b(bounds_json or ""),
                  n_uniform, seed, alpha)
    return _lib.text()


def acceptance_rate(sampler_json: str, probe: GemmInput, hw: HardwareDescriptor, n_trials: int = 100000,
                    seed: int = 0) -> float:
    r = ctypes.c_double()
    _lib.call("ktune_acceptance_rate_gemm", ctypes.byref(hw.c()), ctypes.byref(probe.c()), sampler_json.encode(),
              n_trials, seed, ctypes.byref(r))
    return r.value


def uniform_acceptance_rate(bounds_json: str | None, probe: GemmInput, hw: HardwareDescriptor,
                            n_trials: int = 100000, seed: int = 0) -> float:
    r = ctypes.c_double()
    _lib.call("ktune_uniform_acceptance_rate_gemm", ctypes.byref(hw.c()), ctypes.byref(probe.c()),
              _b(bounds_json or ""), n_trials, seed, ctypes.byref(r))
    return r.value


# ---------------------------------------------------------------------------
# input distributions (pipeline.hpp:86-118)
# ---------------------------------------------------------------------------

@dataclass
class GemmInputDistribution:
    shapes: list = field(default_factory=list)
    weights: list = field(default_factory=list)
    fixed_fraction: float = 0.5
    use_ranges: bool = True
    m_lo: int = 16
    m_hi: int = 4096
    n_lo: int = 16
    n_hi: int = 4096
    k_lo: int = 16
    k_hi: int = 65536
    dtype: str = "f32"
    randomize_transpose: bool = True

    def c(self):
        arr = (_lib.GemmInputC * max(1, len(self.shapes)))(*[s.c() for s in self.shapes])
        w = (ctypes.c_double * len(self.weights))(*self.weights) if self.weights else None
        d = _lib.GemmDistC(ctypes.cast(arr, ctypes.c_void_p) if self.shapes else None, len(self.shapes),
                           ctypes.cast(w, ctypes.c_void_p) if w else None, self.fixed_fraction, int(self.use_ranges),
                           self.m_lo, self.m_hi, self.n_lo, self.n_hi, self.k_lo, self.k_hi, DTYPE_CODES[self.dtype],
                           int(self.randomize_transpose))
        return d, (arr, w)  # keep the buffers alive with the struct


@dataclass
class ConvInputDistribution:
    shapes: list = field(default_factory=list)
    weights: list = field(default_factory=list)
    fixed_fraction: float = 0.5
    use_ranges: bool = True
    n_lo: int = 4
    n_hi: int = 64
    p_lo: int = 4
    p_hi: int = 128
    q_lo: int = 4
    q_hi: int = 128
    k_lo: int = 8
    k_hi: int = 512
    c_lo: int = 4
    c_hi: int = 512
    rs_choices: list = field(default_factory=lambda: [(1, 1), (3, 3)])
    dtype: str = "f32"

    def c(self):
        arr = (_lib.ConvInputC * max(1, len(self.shapes)))(*[s.cstruct() for s in self.shapes])
        w = (ctypes.c_double * len(self.weights))(*self.weights) if self.weights else None
        rs = (ctypes.c_int32 * (2 * len(self.rs_choices)))(*[v for p in self.rs_choices for v in p])
        d = _lib.ConvDistC(ctypes.cast(arr, ctypes.c_void_p) if self.shapes else None, len(self.shapes),
                           ctypes.cast(w, ctypes.c_void_p) if w else None, self.fixed_fraction, int(self.use_ranges),
                           self.n_lo, self.n_hi, self.p_lo, self.p_hi, self.q_lo, self.q_hi, self.k_lo, self.k_hi,
                           self.c_lo, self.c_hi, ctypes.cast(rs, ctypes.c_void_p), len(self.rs_choices),
                           DTYPE_CODES[self.dtype])
        return d, (arr, w, rs)


def gemm_shapes_from_table(path: str, dtype: str = "f32") -> list:
    """GemmInput list from fixtures/shapes/benchmarks.json (or a reference-style table)."""
    with open(path) as fh:
        j = json.load(fh)
    if "gemm" in j and isinstance(j["gemm"], list) and j["gemm"] and isinstance(j["gemm"][0], list):
        return [GemmInput(r[1], r[2], r[3], dtype, bool(r[4]), bool(r[5])) for r in j["gemm"]]
    return [GemmInput(s["m"], s["n"], s["k"], s.get("dtype", dtype), bool(s["trans_a"]), bool(s["trans_b"]))
            for s in j["shapes"]]


def conv_shapes_from_table(path: str, dtype: str = "f32") -> list:
    with open(path) as fh:
        j = json.load(fh)
    if "conv" in j and isinstance(j["conv"], list) and j["conv"] and isinstance(j["conv"][0], list):
        return [ConvInput(*r[1:8], dtype=dtype) for r in j["conv"]]
    return [ConvInput(s["n"], s["p"], s["q"], s["k"], s["c"], s["r"], s["s"], s.get("dtype", dtype))
            for s in j["shapes"]]


# ---------------------------------------------------------------------------
# generation (pipeline.cpp:463-556)
# ---------------------------------------------------------------------------

def predraw(sampler_json: str, dist, hw: HardwareDescriptor, bounds_json: str | None, n_samples: int, seed: int):
    """The distinct (input, tuning) sequence generate_*_dataset measures,
    as (inputs_array, tunings_array, attempts, duplicates); arrays are
    ctypes struct arrays."""
    conv = isinstance(dist, ConvInputDistribution)
    d, keep = dist.c()
    ins = ((_lib.ConvInputC if conv else _lib.GemmInputC) * n_samples)()
    tus = ((_lib.ConvTuningC if conv else _lib.GemmTuningC) * n_samples)()
    att, dup = ctypes.c_int64(), ctypes.c_int64()
    _lib.call("ktune_predraw_conv" if conv else "ktune_predraw_gemm", ctypes.byref(hw.c()), _b(bounds_json or ""),
              sampler_json.encode(), ctypes.byref(d), n_samples, seed, ctypes.cast(ins, ctypes.c_void_p),
              ctypes.cast(tus, ctypes.c_void_p), ctypes.byref(att), ctypes.byref(dup))
    del keep
    return ins, tus, att.value, dup.value


def as_inputs(ins) -> list:
    out = []
    for x in ins:
        if isinstance(x, _lib.GemmInputC):
            out.append(GemmInput(x.m, x.n, x.k, _lib.DTYPE_NAMES[x.dtype], bool(x.trans_a), bool(x.trans_b)))
        else:
            out.append(ConvInput(x.n_batch, x.p, x.q, x.k_filters, x.c, x.r, x.s, _lib.DTYPE_NAMES[x.dtype]))
    return out


def as_tunings(tus) -> list:
    if not len(tus):
        return []
    cls = ConvTuning if isinstance(tus[0], _lib.ConvTuningC) else GemmTuning
    names = _lib.CONV_PARAMS if cls is ConvTuning else _lib.GEMM_PARAMS
    return [cls(*[getattr(t, n) for n in names]) for t in tus]


def generate_gemm(sampler_json: str, dist: GemmInputDistribution, hw: HardwareDescriptor, bounds_json: str | None,
                  n_samples: int, seed: int, backend: str = "b200", mode: str = "fast", repetitions: int = 3):
    """Sequential generate_gemm_dataset (pipeline.cpp:463-509); CSV text."""
    d, keep = dist.c()
    att, dup = ctypes.c_int64(), ctypes.c_int64()
    opts = _lib.MeasureOptionsC(_lib.MODE_PARITY if mode == "parity" else _lib.MODE_FAST, repetitions, 1, 1, 0x5EED)
    _lib.call("ktune_generate_gemm", ctypes.byref(hw.c()), _b(bounds_json or ""), sampler_json.encode(),
              ctypes.byref(d), n_samples, seed, BACKENDS[backend], ctypes.byref(opts), ctypes.byref(att),
              ctypes.byref(dup))
    del keep
    return _lib.text(), att.value, dup.value


def dataset_csv(inputs, tunings, gflops, backend: str) -> str:
    """CSV text of measured records in the given order (pipeline.cpp:134-160)."""
    g = np.ascontiguousarray(gflops, np.float64)
    conv = len(inputs) and isinstance(inputs[0], _lib.ConvInputC)
    _lib.call("ktune_conv_dataset_csv" if conv else "ktune_gemm_dataset_csv", ctypes.cast(inputs, ctypes.c_void_p),
              ctypes.cast(tunings, ctypes.c_void_p), g.ctypes.data_as(ctypes.c_void_p), len(g), backend.encode())
    return _lib.text()


def canonical_csv(text: str, kind: str = "gemm") -> str:
    _lib.call("ktune_dataset_canonical", text.encode(), 0 if kind == "gemm" else 1)
    return _lib.text()


def flops_of(x) -> float:
    if isinstance(x, _lib.GemmInputC):
        return 2.0 * x.m * x.n * x.k
    return 2.0 * x.n_batch * x.p * x.q * x.k_filters * x.c * x.r * x.s


def shard_lpt(costs, world_size: int) -> list:
    """Longest-processing-time-first assignment of sample indices to ranks
    (sample costs are heavy-tailed: mean 7.2e9 FLOP, max > 1e12)."""
    order = np.argsort(-np.asarray(costs, np.float64), kind="stable")
    load = np.zeros(world_size)
    shards = [[] for _ in range(world_size)]
    for i in order:
        r = int(np.argmin(load))
        shards[r].append(int(i))
        load[r] += costs[i]
    return [sorted(s) for s in shards]


def generate_sharded(sampler_json: str, dist, hw: HardwareDescriptor, bounds_json: str | None, n_samples: int,
                     seed: int, backend: str = "b200", mode: str = "fast", repetitions: int = 3, group=None,
                     device=None, checkpoint: str | None = None):
    """Sharded generate_*_dataset (pipeline.cpp:463-556).

    Every rank pre-draws the same sequence and measures its LPT shard -- on
    the b200 backend inside the library (ktune_generate_*_shard: batched
    device timing, one host sync per batch, optional resumable checkpoint
    file per rank); then one all-gather of fixed-size {index, gflops} records
    (NCCL over NVLink on GPUs, gloo on CPU) rebuilds the dataset in canonical
    order on every rank.  A rank whose measurements fail still reaches the
    collective (its failure travels in the records), and every rank raises
    after the gather, so no rank is left blocked.  Returns (csv_text, stats)."""
    import torch
    import torch.distributed as dist_

    ws = dist_.get_world_size(group) if dist_.is_initialized() else 1
    rank = dist_.get_rank(group) if dist_.is_initialized() else 0
    conv = isinstance(dist, ConvInputDistribution)
    t0 = time.perf_counter()
    error = None
    unl = 0
    if backend == "analytical":
        ins, tus, att, dup = predraw(sampler_json, dist, hw, bounds_json, n_samples, seed)
        t_draw = time.perf_counter() - t0
        owner = shard_lpt_owner([flops_of(x) for x in ins], ws)
        mine = [i for i in range(n_samples) if owner[i] == rank]
        py_ins, py_tus = as_inputs(ins), as_tunings(tus)
        recs = np.zeros((len(mine), 2), np.float64)
        for j, i in enumerate(mine):
            recs[j] = (i, analytical_gflops(py_ins[i], py_tus[i], hw))
        t_measure = time.perf_counter() - t0 - t_draw
    else:
        d, keep = dist.c()
        ins = ((_lib.ConvInputC if conv else _lib.GemmInputC) * n_samples)()
        tus = ((_lib.ConvTuningC if conv else _lib.GemmTuningC) * n_samples)()
        cap = n_samples
        idx = np.zeros(cap, np.int64)
        gfl = np.zeros(cap, np.float64)
        cnt, att_, dup_, unl_ = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        opts = _lib.MeasureOptionsC(_lib.MODE_FAST if mode == "fast" else _lib.MODE_PARITY, repetitions, 1, 1, 0x5EED)
        try:
            _lib.call("ktune_generate_conv_shard" if conv else "ktune_generate_gemm_shard", ctypes.byref(hw.c()),
                      _b(bounds_json or ""), sampler_json.encode(), ctypes.byref(d), n_samples, seed, rank, ws,
                      ctypes.byref(opts), None if checkpoint is None else checkpoint.encode(),
                      ctypes.cast(ins, ctypes.c_void_p), ctypes.cast(tus, ctypes.c_void_p),
                      idx.ctypes.data_as(ctypes.c_void_p), gfl.ctypes.data_as(ctypes.c_void_p), cap,
                      ctypes.byref(cnt), ctypes.byref(att_), ctypes.byref(dup_), ctypes.byref(unl_))
            recs = np.stack([idx[: cnt.value].astype(np.float64), gfl[: cnt.value]], axis=1)
        except Exception as e:  # noqa: BLE001 -- reported to every rank after the gather
            error = f"rank {rank}: {e}"
            recs = np.zeros((0, 2))
        del keep
        att, dup, unl = att_.value, dup_.value, unl_.value
        t_draw = float("nan")
        t_measure = time.perf_counter() - t0
    # fixed-size records: rank r sends at most ceil(n / ws) + the LPT excess;
    # an all-reduce of the local count sizes the buffer exactly
    n_local = torch.tensor([len(recs), 1 if error else 0], dtype=torch.int64)
    if ws > 1:
        dev = device if device is not None else ("cuda" if dist_.get_backend(group) == "nccl" else "cpu")
        n_local = n_local.to(dev)
        dist_.all_reduce(n_local, op=dist_.ReduceOp.MAX, group=group)
        per, failed = int(n_local[0].item()), int(n_local[1].item())
        buf = np.full((per, 2), -1.0)
        buf[: len(recs)] = recs
        local = torch.from_numpy(buf).to(dev)
        gathered = torch.empty((ws * per, 2), dtype=torch.float64, device=dev)
        dist_.all_gather_into_tensor(gathered, local, group=group)
        allrec = gathered.cpu().numpy()
    else:
        failed = 1 if error else 0
        allrec = recs
    if failed:
        raise RuntimeError(error or "sharded generation failed on another rank")
    gflops = np.zeros(n_samples)
    seen = np.zeros(n_samples, bool)
    for i, g in allrec:
        if i >= 0:
            gflops[int(i)] = g
            seen[int(i)] = True
    if not seen.all():
        raise RuntimeError("sharded generation lost records")
    if not (np.isfinite(gflops) & (gflops > 0)).all():
        raise RuntimeError("backend returned non-positive gflops")
    name = backend if backend != "b200" or mode == "fast" else "b200-parity"
    text = dataset_csv(ins, tus, gflops, name)
    stats = {"attempts": att, "duplicates": dup, "unlaunchable": unl, "predraw_s": t_draw, "measure_s": t_measure,
             "local_samples": len(recs), "world_size": ws}
    return text, stats


def shard_lpt_owner(costs, world_size: int) -> np.ndarray:
    """owner[i] = rank of sample i under the library's LPT assignment
    (ktune_shard_lpt; same rule as shard_lpt below)."""
    c = np.ascontiguousarray(costs, np.float64)
    out = np.zeros(len(c), np.int32)
    _lib.call("ktune_shard_lpt", c.ctypes.data_as(ctypes.c_void_p), len(c), world_size,
              out.ctypes.data_as(ctypes.c_void_p))
    return out


# ---------------------------------------------------------------------------
# MLP (perf_model.cpp) -- GPU training and sweep
# ---------------------------------------------------------------------------

@dataclass
class TrainOutcome:
    model_json: str
    best_val_mse: float
    best_epoch: int
    history: np.ndarray  # (epochs, 2) train/val MSE


def train_mlp(csv_text: str, kind: str = "gemm", hidden=(32, 64, 32), log_inputs=True, epochs=200, lr=1e-3,
              batch_size=256, seed=0, validation_fraction=0.1, fast=False) -> TrainOutcome:
    """K7 (reference operation order, bit-identical models) or, with fast,
    K7f (each minibatch layer one batched fp64 GEMM)."""
    hid = (ctypes.c_int32 * len(hidden))(*hidden)
    hist = np.zeros((epochs, 2))
    bv, be = ctypes.c_double(), ctypes.c_int32()
    _lib.call("ktune_mlp_train_fast" if fast else "ktune_mlp_train", csv_text.encode(), 0 if kind == "gemm" else 1,
              ctypes.cast(hid, ctypes.c_void_p), len(hidden), int(log_inputs), epochs, lr, batch_size, seed, validation_fraction, ctypes.byref(bv),
              ctypes.byref(be), hist.ctypes.data_as(ctypes.c_void_p))
    return TrainOutcome(_lib.text(), bv.value, be.value, hist)


def mlp_init(input_dim: int, hidden=(32, 64, 32), log_inputs=True, seed=0, feature_version="gemm.v1") -> str:
    hid = (ctypes.c_int32 * len(hidden))(*hidden)
    _lib.call("ktune_mlp_init", input_dim, ctypes.cast(hid, ctypes.c_void_p), len(hidden), int(log_inputs), seed,
              feature_version.encode())
    return _lib.text()


def mlp_predict_rows(model_json: str, rows) -> np.ndarray:
    x = np.ascontiguousarray(rows, np.float64)
    out = np.zeros(len(x))
    _lib.call("ktune_mlp_predict_rows", model_json.encode(), x.ctypes.data_as(ctypes.c_void_p), len(x), x.shape[1],
              out.ctypes.data_as(ctypes.c_void_p))
    return out


def mlp_predict(model_json: str, inp, tunings, fast: bool = False) -> np.ndarray:
    """GPU candidate sweep (MlpPredictor::predict_*): K6 bit-exact, or K6f
    (batched GEMMs) with fast (GEMM inputs only)."""
    conv = isinstance(inp, ConvInput)
    arr = ((_lib.ConvTuningC if conv else _lib.GemmTuningC) * len(tunings))(*[t.c() for t in tunings])
    out = np.zeros(len(tunings))
    fn = "ktune_mlp_predict_conv" if conv else ("ktune_mlp_predict_gemm_fast" if fast else "ktune_mlp_predict_gemm")
    _lib.call(fn, model_json.encode(),
              ctypes.byref(inp.cstruct() if conv else inp.c()), ctypes.cast(arr, ctypes.c_void_p), len(tunings),
              out.ctypes.data_as(ctypes.c_void_p))
    return out


def mlp_evaluate(model_json: str, csv_text: str, kind: str = "gemm") -> float:
    r = ctypes.c_double()
    _lib.call("ktune_mlp_evaluate", model_json.encode(), csv_text.encode(), 0 if kind == "gemm" else 1,
              ctypes.byref(r))
    return r.value


# ---------------------------------------------------------------------------
# analytical model + runtime selection + cache
# ---------------------------------------------------------------------------

def peak_gflops(hw: HardwareDescriptor) -> float:
    r = ctypes.c_double()
    _lib.call("ktune_peak_gflops", ctypes.byref(hw.c()), ctypes.byref(r))
    return r.value


def analytical_gflops(inp, t, hw: HardwareDescriptor) -> float:
    r = ctypes.c_double()
    if isinstance(inp, ConvInput):
        _lib.call("ktune_analytical_gflops_conv", ctypes.byref(hw.c()), ctypes.byref(inp.cstruct()),
                  ctypes.byref(t.c()), ctypes.byref(r))
    else:
        _lib.call("ktune_analytical_gflops_gemm", ctypes.byref(hw.c()), ctypes.byref(inp.c()), ctypes.byref(t.c()),
                  ctypes.byref(r))
    return r.value


def infer(inp, hw: HardwareDescriptor, bounds_json: str | None = None, model_json: str | None = None,
          top_k: int = 100, backend: str = "b200", mode: str = "fast", repetitions: int = 3) -> str:
    """infer_gemm / infer_conv (pipeline.cpp:649-723); ktune-result-1 JSON."""
    opts = _lib.MeasureOptionsC(_lib.MODE_PARITY if mode == "parity" else _lib.MODE_FAST, repetitions, 1, 1, 0x5EED)
    if isinstance(inp, ConvInput):
        _lib.call("ktune_infer_conv", ctypes.byref(hw.c()), _b(bounds_json or ""), _b(model_json or ""),
                  ctypes.byref(inp.cstruct()), top_k, BACKENDS[backend], ctypes.byref(opts))
    else:
        _lib.call("ktune_infer_gemm", ctypes.byref(hw.c()), _b(bounds_json or ""), _b(model_json or ""),
                  ctypes.byref(inp.c()), top_k, BACKENDS[backend], ctypes.byref(opts))
    return _lib.text()


def mlp_sweep(model_json: str, inp: GemmInput, hw: HardwareDescriptor, bounds_json: str | None = None,
              fast: bool = False):
    """The runtime candidate sweep over the whole legal space, entirely in the
    library: returns (candidates, device_seconds, total_seconds)."""
    n, dsec, tsec = ctypes.c_int64(), ctypes.c_double(), ctypes.c_double()
    _lib.call("ktune_mlp_sweep_gemm", model_json.encode(), ctypes.byref(hw.c()), _b(bounds_json or ""),
              ctypes.byref(inp.c()), 1 if fast else 0, ctypes.byref(n), ctypes.byref(dsec), ctypes.byref(tsec))
    return n.value, dsec.value, tsec.value


def infer_sharded(inp, hw: HardwareDescriptor, bounds_json: str | None = None, model_json: str | None = None,
                  top_k: int = 100, backend: str = "b200", mode: str = "fast", repetitions: int = 3, group=None,
                  device=None) -> str:
    """infer_* with the top-k re-measure sharded over the process group
    (pipeline.cpp:674-680): each rank measures ranked
    candidates i with i % world == rank, one all-reduce (max) of the
    measurement vector, then every rank rebuilds the same ktune-result-1
    JSON the sequential infer would write.  top_k >= the legal space is the
    sharded `bench --exhaustive`."""
    import torch
    import torch.distributed as dist_

    ws = dist_.get_world_size(group) if dist_.is_initialized() else 1
    rank = dist_.get_rank(group) if dist_.is_initialized() else 0
    conv = isinstance(inp, ConvInput)
    opts = _lib.MeasureOptionsC(_lib.MODE_PARITY if mode == "parity" else _lib.MODE_FAST, repetitions, 1, 1, 0x5EED)
    from . import enumerate_legal
    cap = max(1, min(top_k, len(enumerate_legal(inp, hw, bounds_json))))
    vals = np.full(cap, -1.0)
    cnt = ctypes.c_int64()
    ic = inp.cstruct() if conv else inp.c()
    _lib.call("ktune_infer_conv_shard" if conv else "ktune_infer_gemm_shard", ctypes.byref(hw.c()),
              _b(bounds_json or ""), _b(model_json or ""), ctypes.byref(ic), top_k, BACKENDS[backend],
              ctypes.byref(opts), rank, ws, vals.ctypes.data_as(ctypes.c_void_p), cap, ctypes.byref(cnt))
    vals = vals[: cnt.value]
    if ws > 1:
        dev = device if device is not None else ("cuda" if dist_.get_backend(group) == "nccl" else "cpu")
        t = torch.from_numpy(vals.copy()).to(dev)
        dist_.all_reduce(t, op=dist_.ReduceOp.MAX, group=group)
        vals = t.cpu().numpy()
    name = backend if backend != "b200" or mode == "fast" else "b200-parity"
    vals = np.ascontiguousarray(vals, np.float64)
    _lib.call("ktune_infer_conv_replay" if conv else "ktune_infer_gemm_replay", ctypes.byref(hw.c()),
              _b(bounds_json or ""), _b(model_json or ""), ctypes.byref(ic), top_k, name.encode(),
              vals.ctypes.data_as(ctypes.c_void_p), len(vals))
    return _lib.text()


def select_conv(inp: ConvInput, hw: HardwareDescriptor, bounds_json: str | None = None, model_json: str | None = None,
                cache_dir: str | None = None, top_k: int = 100):
    """Runtime pick for a convolution: memo -> result cache -> infer_conv
    (b200).  Returns (ConvTuning, source) with source in {"memory", "file",
    "inferred"}."""
    t = _lib.ConvTuningC()
    src = ctypes.c_int32()
    _lib.call("ktune_select_conv", ctypes.byref(hw.c()), _b(bounds_json or ""), _b(model_json or ""),
              _b(cache_dir or ""), ctypes.byref(inp.cstruct()), top_k, ctypes.byref(t), ctypes.byref(src))
    return ConvTuning(*[getattr(t, n) for n in _lib.CONV_PARAMS]), ("memory", "file", "inferred")[src.value]


def cache_key(inp) -> str:
    if isinstance(inp, ConvInput):
        _lib.call("ktune_cache_key_conv", ctypes.byref(inp.cstruct()))
    else:
        _lib.call("ktune_cache_key_gemm", ctypes.byref(inp.c()))
    return _lib.text()


def cache_lookup(directory: str, inp):
    found = ctypes.c_int()
    if isinstance(inp, ConvInput):
        _lib.call("ktune_cache_lookup_conv", directory.encode(), ctypes.byref(inp.cstruct()), ctypes.byref(found))
    else:
        _lib.call("ktune_cache_lookup_gemm", directory.encode(), ctypes.byref(inp.c()), ctypes.byref(found))
    return _lib.text() if found.value else None


def cache_store(directory: str, result_json: str) -> None:
    _lib.call("ktune_cache_store", directory.encode(), result_json.encode())


def select_gemm(inp: GemmInput, hw: HardwareDescriptor, bounds_json: str | None = None, model_json: str | None = None,
                cache_dir: str | None = None, top_k: int = 100):
    """Runtime pick: memo -> result cache -> infer (b200).  Returns
    (GemmTuning, source) with source in {"memory", "file", "inferred"}."""
    t = _lib.GemmTuningC()
    src = ctypes.c_int32()
    _lib.call("ktune_select_gemm", ctypes.byref(hw.c()), _b(bounds_json or ""), _b(model_json or ""),
              _b(cache_dir or ""), ctypes.byref(inp.c()), top_k, ctypes.byref(t), ctypes.byref(src))
    return GemmTuning(*[getattr(t, n) for n in _lib.GEMM_PARAMS]), ("memory", "file", "inferred")[src.value]


def load_text(path: str) -> str:
    with open(path) as fh:
        return fh.read()


__all__ = [n for n in dir() if not n.startswith("_")]

"""K6/K7 and the device-backed pipeline on the B200.

- K6 (candidate sweep) must equal MlpModel::predict_batch bit for bit.
- K7 (GPU minibatch SGD) keeps the reference's operation order, shuffles and
  best-epoch selection, so a model trained here equals the reference's
  (perf_model.cpp:318-423) byte for byte when no step is clipped.
- Inference with the learned predictor reproduces the reference result JSON.
- Generation on the b200 backend measures exactly the reference sequence.
"""
import json
import os

import numpy as np
import pytest

import paper_1802_05371_b200 as K
from paper_1802_05371_b200 import pipeline as P

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "pipeline.json")
SHAPES = os.path.join(K.FIXTURES, "shapes", "benchmarks.json")


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def readme_dist():
    return P.GemmInputDistribution(shapes=P.gemm_shapes_from_table(SHAPES), fixed_fraction=0.25)


@pytest.fixture(scope="module")
def synth_csv(golden):
    g = golden["generate"]["synthetic"]
    csv, _, _ = P.generate_gemm(golden["sampler"]["synthetic_json"], readme_dist(), K.HardwareDescriptor(), None,
                                g["n"], g["seed"], backend="analytical")
    return csv


def test_gpu_sweep_bit_identical(cuda, golden):
    model = golden["mlp"]["init_seed7_json"]
    got = P.mlp_predict_rows(model, np.array(golden["mlp"]["features"]))
    assert [x.hex() for x in got] == golden["mlp"]["predict_init"]


def test_gpu_training_reproduces_reference_model(cuda, golden, synth_csv):
    out = P.train_mlp(synth_csv, "gemm", (32, 64, 32), True, epochs=5, lr=1e-3, batch_size=256, seed=7,
                      validation_fraction=0.1)
    assert out.best_epoch == golden["mlp"]["train_5ep_best_epoch"]
    assert out.best_val_mse.hex() == golden["mlp"]["train_5ep_best_val"]
    assert out.model_json == golden["mlp"]["train_5ep_json"]


def test_inference_with_learned_predictor(cuda, golden):
    got = P.infer(K.GemmInput(2560, 16, 2560, "f32"), K.HardwareDescriptor(), None, golden["mlp"]["train_5ep_json"],
                  20, backend="analytical")
    assert got == golden["infer"]["mlp5ep_deepbench16_top20"]


def test_training_converges_and_log_features_help(cuda, synth_csv):
    """Acceptance criterion 5 shape (acceptance_main.cpp:387-431): log-feature
    training beats the raw-feature ablation on the same data."""
    log = P.train_mlp(synth_csv, epochs=40, seed=3)
    raw = P.train_mlp(synth_csv, epochs=40, seed=3, log_inputs=False)
    assert np.isfinite(log.best_val_mse) and log.best_val_mse < raw.best_val_mse
    assert log.history[-1, 0] < log.history[0, 0]


def test_b200_generation_measures_reference_sequence(cuda, golden):
    hw = K.HardwareDescriptor.b200()
    b200 = open(os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")).read()
    dist = readme_dist()
    dist.m_hi = dist.n_hi = 512  # keep the device time of this test small
    dist.k_hi = 4096
    csv, _, _ = P.generate_gemm(golden["sampler"]["b200_json"], dist, hw, b200, 24, 42, backend="b200")
    ana, _, _ = P.generate_gemm(golden["sampler"]["b200_json"], dist, hw, b200, 24, 42, backend="analytical")
    rows, arows = csv.splitlines()[1:], ana.splitlines()[1:]
    assert len(rows) == 24
    for r, a in zip(rows, arows):
        f, fa = r.split(","), a.split(",")
        assert f[:14] == fa[:14] and f[15] == "b200" and float(f[14]) > 0


def test_runtime_selection_memo_and_cache(cuda, tmp_path, golden):
    hw = K.HardwareDescriptor.b200()
    b200 = open(os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")).read()
    inp = K.GemmInput(256, 64, 1024, "f32")
    t1, src1 = P.select_gemm(inp, hw, b200, None, str(tmp_path), top_k=8)
    assert src1 == "inferred"
    t2, src2 = P.select_gemm(inp, hw, b200, None, str(tmp_path), top_k=8)
    assert src2 == "memory" and t2 == t1
    assert P.cache_lookup(str(tmp_path), inp) is not None

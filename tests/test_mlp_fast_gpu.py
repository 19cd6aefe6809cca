"""K6f / K7f: the MLP as batched GEMMs (north star: "training and the runtime
candidate sweep both run as small batched GEMM kernels on the GPU").

They keep the reference model, loss, minibatches, shuffles, clip and
best-epoch rule but sum in GEMM order, so they are checked against the
bit-identical K6 / K7 within rounding: sweep predictions within 1e-12
relative, the same top of the ranking, and a trained model whose validation
MSE tracks K7's."""
import os

import numpy as np
import pytest

import paper_1802_05371_b200 as K
from paper_1802_05371_b200 import pipeline as P

pytestmark = pytest.mark.gpu

SHAPES = os.path.join(K.FIXTURES, "shapes", "benchmarks.json")


@pytest.fixture(scope="module")
def dataset():
    hw = K.HardwareDescriptor()
    sampler = P.calibrate(K.GemmInput(512, 512, 512), hw, None, 20000, 11)
    dist = P.GemmInputDistribution(shapes=P.gemm_shapes_from_table(SHAPES), fixed_fraction=0.25)
    csv, _, _ = P.generate_gemm(sampler, dist, hw, None, 3000, 42, backend="analytical")
    return csv


def test_fast_sweep_matches_parity_sweep(cuda, dataset):
    model = P.train_mlp(dataset, epochs=3, seed=7).model_json
    hw = K.HardwareDescriptor.b200()
    bounds = open(os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")).read()
    inp = K.GemmInput(2560, 32, 2560, "f32")
    space = K.enumerate_legal(inp, hw, bounds)
    exact = np.array(P.mlp_predict(model, inp, space))
    fast = np.array(P.mlp_predict(model, inp, space, fast=True))
    assert np.max(np.abs(fast - exact) / np.maximum(np.abs(exact), 1.0)) < 1e-12
    assert list(np.argsort(-exact, kind="stable")[:20]) == list(np.argsort(-fast, kind="stable")[:20])
    n, dev_s, _ = P.mlp_sweep(model, inp, hw, bounds, fast=True)
    assert n == len(space) and dev_s > 0


def test_fast_training_tracks_reference_order_training(cuda, dataset):
    ref = P.train_mlp(dataset, epochs=30, seed=7)
    fast = P.train_mlp(dataset, epochs=30, seed=7, fast=True)
    assert np.isfinite(fast.best_val_mse)
    # same data, split, init, shuffles and step rule: the curves agree to rounding
    assert abs(fast.best_val_mse - ref.best_val_mse) <= 1e-6 * max(1.0, ref.best_val_mse)
    assert np.allclose(fast.history, ref.history, rtol=1e-6, atol=1e-9)

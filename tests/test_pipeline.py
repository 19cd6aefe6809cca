"""Tuning-pipeline parity on the host (no GPU): sampler, distributions,
dataset sequences and CSV bytes, analytical model, result JSON, cache --
all against tests/golden/pipeline.json produced by the reference library
(tests/golden/make_golden_pipeline.py).  Mirrors test_sampler.cpp,
test_pipeline.cpp and acceptance criteria 3 and 8."""
import hashlib
import json
import os
import socket

import pytest

import paper_1802_05371_b200 as K
from paper_1802_05371_b200 import pipeline as P

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "pipeline.json")
SHAPES = os.path.join(K.FIXTURES, "shapes", "benchmarks.json")
B200_GEMM = open(os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")).read()
CONV_SMALL = json.dumps({"k_s": [1, 2], "p_s": [1, 2], "q_s": [1, 2], "n_s": [1, 2], "k_l": [1, 2, 4, 8],
                         "p_l": [1, 2, 4], "q_l": [1, 2, 4], "n_l": [1, 2, 4], "u": [1, 2, 4], "c_s": [1, 2],
                         "c_l": [1, 2, 4], "c_g": [1, 2, 4, 8]})


def sha(t):
    return hashlib.sha256(t.encode()).hexdigest()


@pytest.fixture(scope="module")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)


def readme_dist():
    """The README walkthrough distribution: fixture shapes at 0.25, f32 ranges."""
    return P.GemmInputDistribution(shapes=P.gemm_shapes_from_table(SHAPES), fixed_fraction=0.25)


def test_calibrated_sampler_models_are_byte_identical(golden):
    hw = K.HardwareDescriptor()
    probe = K.GemmInput(512, 512, 512)
    assert P.calibrate(probe, hw, None, 100000, 11) == golden["sampler"]["synthetic_json"]
    assert P.calibrate(probe, K.HardwareDescriptor.b200(), B200_GEMM, 100000, 11) == golden["sampler"]["b200_json"]
    assert P.calibrate(K.ConvInput(16, 24, 240, 32, 16, 3, 3), hw, CONV_SMALL, 100000, 11) == \
        golden["sampler"]["conv_small_json"]


def test_sampler_beats_uniform_acceptance(golden):
    """Acceptance criterion 3 (acceptance_main.cpp:301-314): >= 10x uniform."""
    hw = K.HardwareDescriptor()
    probe = K.GemmInput(512, 512, 512)
    cat = P.acceptance_rate(golden["sampler"]["synthetic_json"], probe, hw, 100000, 1)
    assert cat == golden["sampler"]["synthetic_acceptance_seed1"]
    uni = P.uniform_acceptance_rate(None, probe, hw, 100000, 1)
    assert cat >= 10 * uni


def test_generated_dataset_matches_reference_bytes(golden):
    """generate_gemm_dataset with the analytical backend: the same sequence,
    dedup and CSV bytes as the reference (pipeline.cpp:463-509)."""
    g = golden["generate"]["synthetic"]
    csv, att, dup = P.generate_gemm(golden["sampler"]["synthetic_json"], readme_dist(), K.HardwareDescriptor(), None,
                                    g["n"], g["seed"], backend="analytical")
    assert csv.splitlines()[:12] == g["head"]
    assert (att, dup) == (g["attempts"], g["duplicates"])
    assert sha(csv) == g["csv_sha256"]
    g = golden["generate"]["b200"]
    csv, att, dup = P.generate_gemm(golden["sampler"]["b200_json"], readme_dist(), K.HardwareDescriptor.b200(),
                                    B200_GEMM, g["n"], g["seed"], backend="analytical")
    assert sha(csv) == g["csv_sha256"] and (att, dup) == (g["attempts"], g["duplicates"])


def test_predraw_equals_generation_sequence(golden):
    """The pre-drawn sequence is exactly what generation measures."""
    g = golden["generate"]["synthetic"]
    hw = K.HardwareDescriptor()
    ins, tus, att, dup = P.predraw(golden["sampler"]["synthetic_json"], readme_dist(), hw, None, g["n"], g["seed"])
    gfl = [P.analytical_gflops(i, t, hw) for i, t in zip(P.as_inputs(ins), P.as_tunings(tus))]
    assert sha(P.dataset_csv(ins, tus, gfl, "analytical")) == g["csv_sha256"]


def test_conv_sequence_and_prices(golden):
    g = golden["generate"]["conv_small"]
    hw = K.HardwareDescriptor()
    dist = P.ConvInputDistribution(shapes=P.conv_shapes_from_table(SHAPES), fixed_fraction=0.25)
    ins, tus, att, dup = P.predraw(golden["sampler"]["conv_small_json"], dist, hw, CONV_SMALL, g["n"], g["seed"])
    gfl = [P.analytical_gflops(i, t, hw) for i, t in zip(P.as_inputs(ins), P.as_tunings(tus))]
    csv = P.dataset_csv(ins, tus, gfl, "analytical")
    assert csv.splitlines()[:8] == g["head"]
    assert sha(csv) == g["csv_sha256"] and (att, dup) == (g["attempts"], g["duplicates"])


def test_analytical_prices_bit_identical(golden):
    hw = K.HardwareDescriptor()
    for t, want in golden["analytical"]["gemm_512_nn_f32"]:
        assert P.analytical_gflops(K.GemmInput(512, 512, 512), K.GemmTuning(*t), hw).hex() == want
    for t, want in golden["analytical"]["conv_small"]:
        assert P.analytical_gflops(K.ConvInput(16, 24, 240, 32, 16, 3, 3), K.ConvTuning(*t), hw).hex() == want
    assert P.peak_gflops(hw) == 256.0
    # test_backends.cpp:308-317: the synthetic device's 2048^3 optimum hits peak
    best = K.GemmTuning(2, 2, 16, 16, 1, 1, 1, 1)
    assert abs(P.analytical_gflops(K.GemmInput(2048, 2048, 2048, trans_b=True), best, hw) - 256.0) < 1e-9


def test_csv_roundtrip_and_validation(golden):
    g = golden["generate"]["synthetic"]
    csv, _, _ = P.generate_gemm(golden["sampler"]["synthetic_json"], readme_dist(), K.HardwareDescriptor(), None, 200,
                                g["seed"], backend="analytical")
    assert P.canonical_csv(csv) == csv
    assert P.canonical_csv(csv.replace("\n", "\r\n")) == csv  # CRLF tolerated
    with pytest.raises(K.KtuneError, match="header mismatch"):
        P.canonical_csv(csv, "conv")
    bad = csv.splitlines()
    bad[3] = bad[3].rsplit(",", 2)[0] + ",-1,analytical"
    with pytest.raises(K.KtuneError, match="non-positive gflops"):
        P.canonical_csv("\n".join(bad) + "\n")


def test_mlp_init_and_format(golden):
    """Glorot init (perf_model.cpp:57-79) and the ktune-mlp-1 bytes."""
    assert P.mlp_init(14, (32, 64, 32), True, 7) == golden["mlp"]["init_seed7_json"]


def test_infer_with_analytical_predictor(golden):
    """Exhaustive-style inference with the oracle predictor on the analytical
    backend reproduces the reference result JSON byte for byte
    (pipeline.cpp:649-685, :793-831)."""
    got = P.infer(K.GemmInput(2048, 2048, 2048, "f32", False, True), K.HardwareDescriptor(), None, None, 100,
                  backend="analytical")
    assert got == golden["infer"]["analytical_2048_nt_top100"]
    chosen = json.loads(got)["chosen"]
    assert [chosen[n] for n in ("m_s", "n_s", "m_l", "n_l", "u", "k_s", "k_l", "k_g")] == [2, 2, 16, 16, 1, 1, 1, 1]


def test_cache_keys_and_store(golden, tmp_path, capfd):
    for spec, key in golden["cache_keys"]["gemm"].items():
        m, n, k, dt, ta, tb = (int(x) for x in spec.split(","))
        assert P.cache_key(K.GemmInput(m, n, k, K._lib.DTYPE_NAMES[dt], bool(ta), bool(tb))) == key
    assert P.cache_key(K.ConvInput(16, 24, 240, 32, 16, 3, 3)) == golden["cache_keys"]["conv_16_24_240_32_16_3_3_f32"]
    res = golden["infer"]["analytical_2048_nt_top100"]
    inp = K.GemmInput(2048, 2048, 2048, "f32", False, True)
    d = str(tmp_path)
    assert P.cache_lookup(d, inp) is None
    P.cache_store(d, res)
    assert P.cache_lookup(d, inp) == res
    # corrupt entries are skipped with a warning, never fatal (pipeline.cpp:960-970)
    with open(os.path.join(d, P.cache_key(inp)), "w") as fh:
        fh.write("{not json")
    assert P.cache_lookup(d, inp) is None
    assert "skipping corrupt cache entry" in capfd.readouterr().err


def test_lpt_sharding_balances_heavy_tails():
    costs = [1e12, 5e9, 5e9, 4e9, 1e9, 1e9, 8e11, 2e3]
    shards = P.shard_lpt(costs, 2)
    assert sorted(i for s in shards for i in s) == list(range(len(costs)))
    loads = [sum(costs[i] for i in s) for s in shards]
    assert max(loads) <= 1.0001e12 + 1e10


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_worker(rank, world, port, sampler_json, n, seed, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        csv, stats = P.generate_sharded(sampler_json, readme_dist(), K.HardwareDescriptor(), None, n, seed,
                                        backend="analytical")
        with open(os.path.join(out_dir, f"rank{rank}.csv"), "w") as fh:
            fh.write(csv)
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
            json.dump(stats, fh)
    finally:
        dist.destroy_process_group()


def test_sharded_generation_two_ranks_matches_sequential(golden, tmp_path):
    """World size 2 over gloo: LPT shards + one all-gather rebuild exactly
    the reference's sequential dataset on every rank."""
    import torch.multiprocessing as mp
    g = golden["generate"]["synthetic"]
    mp.spawn(_sharded_worker, args=(2, _free_port(), golden["sampler"]["synthetic_json"], g["n"], g["seed"],
                                    str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert sha(open(tmp_path / f"rank{r}.csv").read()) == g["csv_sha256"]
    stats = [json.load(open(tmp_path / f"rank{r}.json")) for r in range(2)]
    assert sum(s["local_samples"] for s in stats) == g["n"]


def _infer_sharded_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        hw = K.HardwareDescriptor()
        for inp in (K.GemmInput(2560, 16, 2560, "f32"), K.ConvInput(4, 9, 11, 24, 5, 3, 3)):
            for k in (7, 1 << 30):  # top-k and the exhaustive bench
                out.put((rank, type(inp).__name__, k, P.infer_sharded(inp, hw, None, None, k, backend="analytical")))
    finally:
        dist.destroy_process_group()


def test_infer_sharded_equals_sequential_on_gloo():
    """the top-k re-measure (and the exhaustive bench)
    sharded over 2 ranks rebuilds the sequential infer_* result JSON byte for
    byte on every rank (analytical backend: deterministic measurements)."""
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_infer_sharded_worker, args=(r, 2, port, q)) for r in range(2)]
    for p_ in procs:
        p_.start()
    got = [q.get(timeout=300) for _ in range(8)]
    for p_ in procs:
        p_.join(timeout=60)
        assert p_.exitcode == 0
    hw = K.HardwareDescriptor()
    for rank, kind, k, text in got:
        inp = K.GemmInput(2560, 16, 2560, "f32") if kind == "GemmInput" else K.ConvInput(4, 9, 11, 24, 5, 3, 3)
        assert text == P.infer(inp, hw, None, None, k, backend="analytical"), (rank, kind, k)

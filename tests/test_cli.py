"""The `ktune_b200` command-line front end (paper_1802_05371_b200/csrc/tools/
ktune_b200.cpp) against the reference CLI's contract (proj/tools/ktune.cpp,
proj/tests/test_cli.cpp): exit codes 0 / 1 / 2, usage errors before any
artifact is written, ktune-report-1 reports, byte-identical reruns, the
result cache, and artifacts byte-identical to the reference library's
pipeline on the same inputs (tests/golden/pipeline.json, generated from the
unmodified reference).

CPU-only verbs run here (analytical backend); the verbs that need the GPU
(train: K7, infer: K6 sweep, --backend b200) are in the gpu-marked tests."""
import hashlib
import json
import os
import subprocess

import pytest

import oracle_libs as O
import paper_1802_05371_b200 as K

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1802_05371_b200", "bin", "ktune_b200")
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "pipeline.json")))
HW = os.path.join(K.FIXTURES, "hw", "b200.json")
GEMM_BOUNDS = os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")
TABLE = os.path.join(K.FIXTURES, "shapes", "benchmarks.json")


def run(*args, env=None, cwd=None):
    if not os.path.exists(CLI):
        pytest.fail("ktune_b200 binary missing: run `make -C paper_1802_05371_b200` (build())")
    e = dict(os.environ)
    e.pop("KTUNE_CACHE_DIR", None)
    if env:
        e.update(env)
    p = subprocess.run([CLI, *map(str, args)], capture_output=True, text=True, env=e, cwd=cwd, timeout=600)
    return p.returncode, p.stdout, p.stderr


def reference_gemm_table(tmp_path, names=None):
    """The shape table in the reference's {"kind", "shapes"} format."""
    rows = json.load(open(TABLE))["gemm"]
    shapes = [{"name": r[0], "m": r[1], "n": r[2], "k": r[3], "dtype": "f32", "trans_a": bool(r[4]),
               "trans_b": bool(r[5])} for r in rows if names is None or r[0] in names]
    p = tmp_path / "gemm_table.json"
    p.write_text(json.dumps({"kind": "gemm", "shapes": shapes}))
    return p


def test_usage_errors_exit_2_and_write_nothing(tmp_path):
    assert run()[0] == 2
    assert run("frobnicate")[0] == 2
    assert run("calibrate", "--bogus", "1")[0] == 2
    out = tmp_path / "s.json"
    code, _, err = run("calibrate", "--bounds", GEMM_BOUNDS, "--out", out)  # no --hw
    assert code == 2 and "hardware descriptor" in err and not out.exists()
    code, _, err = run("calibrate", "--hw", tmp_path / "missing.json", "--bounds", GEMM_BOUNDS, "--out", out)
    assert code == 2 and not out.exists()
    code, _, _ = run("calibrate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--out", out, "--seed", "x")
    assert code == 2 and not out.exists()
    code, _, err = run("infer", "--hw", HW)  # --shape required
    assert code == 2 and "--shape" in err
    code, _, err = run("train", "--dataset", tmp_path / "none.csv", "--out", tmp_path / "m.json")
    assert code == 2 and "generate" in err and not (tmp_path / "m.json").exists()
    assert run("calibrate", "--help")[0] == 0
    assert not list(tmp_path.glob("*.tmp"))


def test_cpu_backend_is_refused_loudly(tmp_path):
    s = tmp_path / "s.json"
    assert run("calibrate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--seed", 11, "--out", s)[0] == 0
    code, _, err = run("generate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--sampler", s, "--backend", "cpu",
                       "--samples", 3, "--out", tmp_path / "d.csv")
    assert code == 2 and "no CPU executor" in err and not (tmp_path / "d.csv").exists()


def test_readme_pipeline_matches_reference_bytes(tmp_path):
    """calibrate -> generate (analytical) -> report on the B200 descriptor:
    sampler JSON and dataset CSV are byte-identical to the reference
    library's (golden b200 entries: seed 11 calibration, seed 42 generation
    of 1000 samples at shape fraction 0.25)."""
    s, d, rep = tmp_path / "sampler.json", tmp_path / "data.csv", tmp_path / "cal.json"
    code, out, _ = run("calibrate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--seed", 11, "--out", s, "--report", rep)
    assert code == 0 and "acceptance" in out
    assert s.read_text().rstrip("\n") == GOLDEN["sampler"]["b200_json"].rstrip("\n")
    r = json.loads(rep.read_text())
    assert r["format"] == "ktune-report-1" and r["command"] == "calibrate" and "seconds" in r["timing"]
    # the B200 space is mostly legal already (uniform acceptance is high), so
    # the calibrated sampler only has to beat it, not by the synthetic 10x
    assert r["acceptance"]["categorical"] >= r["acceptance"]["uniform"] > 0
    table = reference_gemm_table(tmp_path)
    code, out, _ = run("generate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--sampler", s, "--shapes", table,
                       "--shape-fraction", 0.25, "--samples", 1000, "--seed", 42, "--out", d)
    assert code == 0 and "wrote 1000 gemm samples" in out
    g = GOLDEN["generate"]["b200"]
    assert hashlib.sha256(d.read_bytes()).hexdigest() == g["csv_sha256"]
    assert f"sampler draws: {g['attempts']} ({g['duplicates']} duplicate redraws)" in out
    # the repo's own column table gives the same dataset
    d2 = tmp_path / "data2.csv"
    assert run("generate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--sampler", s, "--shapes", TABLE,
               "--shape-fraction", 0.25, "--samples", 1000, "--seed", 42, "--out", d2)[0] == 0
    assert d2.read_bytes() == d.read_bytes()
    rj = tmp_path / "report.json"
    code, out, _ = run("report", "--dataset", d, "--out", rj)
    assert code == 0 and "rows: 1000" in out
    assert json.loads(rj.read_text())["rows"] == 1000


def test_reruns_are_byte_identical(tmp_path):
    a, b = tmp_path / "a.json", tmp_path / "b.json"
    for p in (a, b):
        assert run("calibrate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--seed", 3, "--draws", 20000, "--out", p)[0] == 0
    assert a.read_bytes() == b.read_bytes()
    ra, rb = tmp_path / "ra.json", tmp_path / "rb.json"
    for p, r in ((tmp_path / "x.csv", ra), (tmp_path / "y.csv", rb)):
        assert run("generate", "--hw", HW, "--bounds", GEMM_BOUNDS, "--sampler", a, "--samples", 50, "--seed", 9,
                   "--out", p, "--report", r)[0] == 0
    assert (tmp_path / "x.csv").read_bytes() == (tmp_path / "y.csv").read_bytes()
    ja, jb = json.loads(ra.read_text()), json.loads(rb.read_text())
    ja.pop("timing"), jb.pop("timing")
    ja["outputs"], jb["outputs"] = None, None
    assert ja == jb  # everything outside "timing" is deterministic


def test_bench_exhaustive_matches_reference_infer(tmp_path):
    """bench --exhaustive (analytical ranking of the whole legal space, every
    candidate measured on the analytical backend) picks what the reference's
    infer_gemm picks with top_k = INT_MAX/2 (ktune.cpp:557-573)."""
    table = reference_gemm_table(tmp_path, {"deepbench-fprop-16", "ica-32"})
    out = tmp_path / "bench.json"
    code, text, _ = run("bench", "--hw", HW, "--bounds", GEMM_BOUNDS, "--shapes", table, "--exhaustive", "--out", out)
    assert code == 0
    rep = json.loads(out.read_text())
    assert rep["mode"] == "exhaustive" and len(rep["results"]) == 2
    lib = O.reference()
    if lib is None:
        pytest.skip("reference library (oracle/_ref) not built")
    import ctypes
    hw_json, bounds_json = open(HW).read().encode(), open(GEMM_BOUNDS).read().encode()
    for row in rep["results"]:
        assert lib.ref_infer_gemm_analytical(hw_json, bounds_json, b"", ctypes.c_int64(row["m"]),
                                             ctypes.c_int64(row["n"]), ctypes.c_int64(row["k"]), 1,
                                             int(row["trans_a"]), int(row["trans_b"]), 2 ** 30) == 0
        ref = json.loads(lib.ref_last_text().decode())
        assert row["chosen"] == ref["chosen"]
        assert row["measured_gflops"] == ref["measured_gflops"]
        assert row["legal_space_size"] == ref["legal_space_size"]


def test_conv_pipeline_matches_reference_bytes(tmp_path):
    """calibrate --kind conv -> generate on the synthetic descriptor (the
    reference defaults) and the conv_small bounds of the reference tests:
    sampler JSON and CSV byte-identical to the reference library (golden
    conv_small entries: seed 11 calibration, seed 5 generation of 300)."""
    import dataclasses
    from test_pipeline import CONV_SMALL
    hw = tmp_path / "synthetic.json"
    hw.write_text(json.dumps(dataclasses.asdict(K.HardwareDescriptor())))
    bounds = tmp_path / "conv_small.json"
    bounds.write_text(CONV_SMALL)
    s, d = tmp_path / "sampler.json", tmp_path / "conv.csv"
    assert run("calibrate", "--kind", "conv", "--hw", hw, "--bounds", bounds, "--seed", 11, "--out", s)[0] == 0
    assert s.read_text().rstrip("\n") == GOLDEN["sampler"]["conv_small_json"].rstrip("\n")
    g = GOLDEN["generate"]["conv_small"]
    code, out, err = run("generate", "--hw", hw, "--bounds", bounds, "--sampler", s, "--shapes", TABLE,
                         "--shape-fraction", g["fixed_fraction"], "--samples", g["n"], "--seed", g["seed"], "--out", d)
    assert code == 0, err
    assert hashlib.sha256(d.read_bytes()).hexdigest() == g["csv_sha256"]
    code, out, _ = run("report", "--dataset", d)
    assert code == 0 and f"rows: {g['n']}" in out


@pytest.mark.parametrize("kind,dtype,bounds,fixture", [
    ("gemm", "f32", "gemm_b200.json", "gemm_b200.json"),
    ("conv", "f32", "conv_b200.json", "conv_b200.json"),
    ("gemm", "bf16", "gemm_b200_tc.json", "gemm_b200_tc_bf16.json"),
    ("conv", "bf16", "conv_b200_tc.json", "conv_b200_tc_bf16.json")])
def test_calibrated_b200_sampler_fixtures(tmp_path, kind, dtype, bounds, fixture):
    """fixtures/samplers/*: the calibrated samplers of the B200 spaces
    (section 8(f) row 4) are what `calibrate --seed 11` produces, and the
    f32 ones equal the reference library's calibration of the same space."""
    out = tmp_path / "s.json"
    b = os.path.join(K.FIXTURES, "bounds", bounds)
    assert run("calibrate", "--kind", kind, "--dtype", dtype, "--hw", HW, "--bounds", b, "--seed", 11,
               "--out", out)[0] == 0
    want = open(os.path.join(K.FIXTURES, "samplers", fixture)).read()
    assert out.read_text() == want
    lib = O.reference()
    if lib is None or dtype != "f32":
        return
    import ctypes
    hw_json, bounds_json = open(HW).read().encode(), open(b).read().encode()
    if kind == "gemm":
        rc = lib.ref_calibrate_gemm(hw_json, bounds_json, ctypes.c_int64(512), ctypes.c_int64(512),
                                    ctypes.c_int64(512), 1, ctypes.c_int64(100000), ctypes.c_uint64(11),
                                    ctypes.c_double(100.0))
    else:
        d = (ctypes.c_int64 * 7)(16, 24, 240, 32, 16, 3, 3)
        rc = lib.ref_calibrate_conv(hw_json, bounds_json, d, 1, ctypes.c_int64(100000), ctypes.c_uint64(11),
                                    ctypes.c_double(100.0))
    assert rc == 0
    assert want.rstrip("\n") == lib.ref_last_text().decode().rstrip("\n")


def test_fitted_b200_descriptor_loads_and_keeps_the_limits(tmp_path):
    """fixtures/hw/b200_fitted.json (section 8(f) row 2) is a strict
    descriptor: it loads, and only the four cost constants differ from the
    nominal B200 descriptor (legality is the hardware's)."""
    fitted = json.load(open(os.path.join(K.FIXTURES, "hw", "b200_fitted.json")))
    nominal = json.load(open(HW))
    assert set(fitted) == set(nominal)
    assert {k for k in nominal if fitted[k] != nominal[k]} <= {"alu_latency", "alu_throughput", "mem_latency",
                                                                "mem_throughput"}
    out = tmp_path / "s.json"
    assert run("calibrate", "--hw", os.path.join(K.FIXTURES, "hw", "b200_fitted.json"), "--bounds", GEMM_BOUNDS,
               "--draws", 1000, "--trials", 100, "--out", out)[0] == 0

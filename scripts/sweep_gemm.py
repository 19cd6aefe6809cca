"""Time a random sample of the legal fp32 SIMT space of one GEMM under the
bench protocol (rotating operand sets > L2, CUDA-graph replay, CUDA events)
and print the fastest tuples.  Default shape: ICA 32x32x60000 NT.

    N=2500 python scripts/sweep_gemm.py [M,N,K] [NN|NT|TN|TT]
"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench, paper_1802_05371_b200 as K
dev = torch.device("cuda:0"); torch.cuda.set_device(0)
stream = torch.cuda.Stream()  # graph capture needs a non-default stream
hw = K.HardwareDescriptor.b200()
shape = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "32,32,60000").split(",")]
ta, tb = (False, True) if len(sys.argv) <= 2 else (sys.argv[2][0] == "T", sys.argv[2][1] == "T")
inp = K.GemmInput(shape[0], shape[1], shape[2], "f32", ta, tb)
bounds = open(os.path.join(K.FIXTURES, "bounds", "gemm_b200.json")).read()
space = K.enumerate_legal(inp, hw, bounds, as_array=True)
print("legal", len(space), flush=True)
os.makedirs(os.environ.get("OUT_DIR", "gpurun_out"), exist_ok=True)
sets = bench.gemm_sets(inp, bench.rotation(bench.gemm_set_bytes(inp), dev), dev)
rng = np.random.default_rng(0)
idx = rng.choice(len(space), size=min(int(os.environ.get("N", "6000")), len(space)), replace=False)
res = []
t0 = time.time()
for i in idx:
    t = K.GemmTuning(*map(int, space[i]))
    try:
        ms = bench.time_gemm(inp, t, sets, stream, steps=20)
    except Exception as e:  # noqa: BLE001 -- outside the launch envelope
        if not res and i == idx[0]:
            print("first failure:", e, flush=True)
        continue
    res.append((ms, t.values(), K.gemm_launch_info(inp, t, "fast")["family"]))
res.sort()
print("timed", len(res), "in", time.time() - t0, flush=True)
top = []
for ms, v, fam in res[:40]:
    ms2 = bench.time_gemm(inp, K.GemmTuning(*v), sets, stream, steps=200)
    top.append((ms2, v, fam))
top.sort()
flops = 2 * inp.m * inp.n * inp.k
for ms, v, fam in top[:15]:
    print(f"{ms*1e3:8.2f} us {flops/ms/1e9:7.2f} TF {v} {fam}")
if os.environ.get("NZ_PROBE"):
    # slice-count probe of the fastest tuples (FAST re-slicing forced)
    for ms, v, fam in top[:3]:
        row = []
        for nz in [int(x) for x in os.environ["NZ_PROBE"].split(",")]:
            os.environ["KTUNE_SIMT_NZ"] = str(nz)
            try:
                row.append((nz, round(bench.time_gemm(inp, K.GemmTuning(*v), sets, stream, steps=200) * 1e3, 2)))
            except Exception as e:  # noqa: BLE001
                row.append((nz, str(e)[:40]))
        os.environ.pop("KTUNE_SIMT_NZ")
        print("nz probe", v, row, flush=True)
json.dump([[ms, v, fam] for ms, v, fam in top], open(os.path.join(os.environ.get("OUT_DIR", "gpurun_out"), "sweep_%s.json" % "_".join(map(str, shape))), "w"))

"""Time one GEMM tuple under several launch-environment settings (bench
protocol).  Measurement aid for kernel work, e.g.

    python scripts/probe_env.py 32,32,60000 NT 1,1,8,16,32,4,1,64 \
        KTUNE_SIMT_PRODUCERS=2 KTUNE_SIMT_TMA=0 KTUNE_SIMT_COMPUTE_ONLY=1
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1802_05371_b200 as K  # noqa: E402

shape = [int(x) for x in sys.argv[1].split(",")]
lay = sys.argv[2]
dt = os.environ.get("DTYPE", "f32")
inp = K.GemmInput(shape[0], shape[1], shape[2], dt, lay[0] == "T", lay[1] == "T")
t = K.GemmTuning(*[int(x) for x in sys.argv[3].split(",")])
dev = torch.device("cuda:0")
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
sets = bench.gemm_sets(inp, bench.rotation(bench.gemm_set_bytes(inp), dev), dev)
flops = 2 * inp.m * inp.n * inp.k
for setting in ["base"] + sys.argv[4:]:
    env = {} if setting == "base" else dict(kv.split("=", 1) for kv in setting.split(","))
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        info = K.gemm_launch_info(inp, t, "fast")
        ms = bench.time_gemm(inp, t, sets, stream, steps=400)
        print(f"{setting:40s} {ms * 1e3:8.2f} us {flops / ms / 1e9:7.2f} TF grid {info['grid']} "
              f"threads {info['threads']} {info['family']}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{setting:40s} failed: {e}", flush=True)
    for k, v in old.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v

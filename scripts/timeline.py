"""Per-block timeline of one SIMT GEMM launch (globaltimer probes compiled
into simt_kernel / simt_tma_kernel, enabled by KTUNE_SIMT_DEBUG=<device
pointer>): block start, first stage ready, main loop done, k_l fold done,
store / k_g merge done.  Measurement aid for kernel work.

    python scripts/timeline.py 32,32,60000 NT 1,1,8,16,32,4,1,64
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1802_05371_b200 as K  # noqa: E402

shape = [int(x) for x in sys.argv[1].split(",")]
lay = sys.argv[2]
inp = K.GemmInput(shape[0], shape[1], shape[2], "f32", lay[0] == "T", lay[1] == "T")
t = K.GemmTuning(*[int(x) for x in sys.argv[3].split(",")])
dev = torch.device("cuda:0")
torch.cuda.set_device(0)
stream = torch.cuda.Stream()
sets = bench.gemm_sets(inp, 2, dev)
info = K.gemm_launch_info(inp, t, "fast")
nb = info["grid"][0] * info["grid"][1] * info["grid"][2]
buf = torch.zeros(nb * 8, dtype=torch.int64, device=dev)
for rep in range(3):
    K.execute_gemm(inp, t, *sets[rep % 2], mode="fast", stream=stream.cuda_stream)
    K.l2_flush(stream.cuda_stream)
    stream.synchronize()
    buf.zero_()
    os.environ["KTUNE_SIMT_DEBUG"] = str(buf.data_ptr())
    K.execute_gemm(inp, t, *sets[rep % 2], mode="fast", stream=stream.cuda_stream)
    os.environ.pop("KTUNE_SIMT_DEBUG")
    stream.synchronize()
d = buf.view(nb, 8).cpu().numpy().astype(np.float64)
t0 = d[:, 0].min()
rel = (d[:, :6] - t0) / 1e3  # us
names = ["start", "setup", "first_data", "loop_done", "kl_fold_done", "end"]
print(info)
for i, nme in enumerate(names):
    col = rel[:, i][d[:, i] > 0]
    if len(col):
        print(f"{nme:13s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f} us (n={len(col)})")
loop = rel[:, 3] - rel[:, 2]
print(f"main loop per block: med {np.median(loop):.2f} max {loop.max():.2f} us; "
      f"merge (end - kl_fold) max {(rel[:, 5] - rel[:, 4]).max():.2f} us; span {rel[:, 5].max():.2f} us")
sm = d[:, 7].astype(int)
print("blocks per SM: max", np.bincount(sm).max(), "SMs used", len(np.unique(sm)))

"""Launch one GEMM tuple a few times (warm-up, then the launch ncu captures)
for `ncu --set full -s <skip> -c 1`.  Never a bench number.

    ncu --set full --import-source on --clock-control none -s 2 -c 1 \
        -o gpurun_out/ica python scripts/ncu_one.py 32,32,60000 NT 4,2,32,32,8,2,2,64 [dtype]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1802_05371_b200 as K  # noqa: E402

shape = [int(x) for x in sys.argv[1].split(",")]
lay = sys.argv[2]
dt = sys.argv[4] if len(sys.argv) > 4 else "f32"
inp = K.GemmInput(shape[0], shape[1], shape[2], dt, lay[0] == "T", lay[1] == "T")
t = K.GemmTuning(*[int(x) for x in sys.argv[3].split(",")])
torch.cuda.set_device(0)
dev = torch.device("cuda:0")
sets = bench.gemm_sets(inp, 2, dev)
print(K.gemm_launch_info(inp, t, "fast"))
for i in range(3):
    K.execute_gemm(inp, t, *sets[i % 2], mode="fast")
torch.cuda.synchronize()

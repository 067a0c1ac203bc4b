"""Microbenchmark (GPU): one conv layer, forward + backward through the C-ABI (bf16, column
mode), per-kernel-class times from the library's profiler (class 0 = conv FP/dgrad,
1 = wgrad, 2 = other).  Usage: python scripts/microbench_layer.py cin,cout,H,W[,k,s] ...
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as WL  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

B = int(os.environ.get("B", "32"))
shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(3, 64, 56, 224)]
for sh in shapes:
    cin, cout, H, W = sh[:4]
    k = sh[4] if len(sh) > 4 else 3
    s = sh[5] if len(sh) > 5 else 1
    net = {"C": cin, "H": H, "W": W, "classes": 10, "ops": [WL.conv(0, cout, k, s, k // 2)]}
    plan = LB.Plan(net, B, mode="column", prec="bf16")
    ds = LB.DeviceState(plan)
    ds.params.uniform_(-0.1, 0.1)
    ds.x.uniform_()
    ds.dzl.uniform_(-1, 1)
    for _ in range(3):
        ds.forward()
        ds.backward()
    torch.cuda.synchronize()
    plan.profile(True)
    plan.profile_reset()
    n = 10
    for _ in range(n):
        ds.forward()
        ds.backward()
    torch.cuda.synchronize()
    c0 = plan.profile_read(0)
    c1 = plan.profile_read(1)
    c2 = plan.profile_read(2)
    plan.profile(False)
    fl = 2 * k * k * cin * cout * (H // s) * (W // s) * B
    print("cin %4d cout %4d %4dx%4d k%d s%d B%d | convFP+dgrad %.3f ms/iter (%d launches) %.1f TF/s | "
          "wgrad %.3f ms %.1f TF/s | other %.3f ms | tc=%d" %
          (cin, cout, H, W, k, s, B, c0[0] / n, c0[1] // n, c0[2] / max(c0[0], 1e-9) / 1e9,
           c1[0] / n, c1[2] / max(c1[0], 1e-9) / 1e9, c2[0] / n, plan.last_tc_launches()), flush=True)

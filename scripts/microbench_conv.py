"""Microbenchmark (GPU): one conv layer forward through lrcnn_forward_rows (bf16, column mode).
Prints TFLOP/s per shape; env LRCNN_TC_DBG / LRCNN_HALO select kernel variants."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as WL  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

SHAPES = [(64, 64, 56, 224), (128, 128, 56, 112), (256, 256, 56, 56), (512, 512, 28, 28), (512, 512, 14, 14)]
B = 32
for cin, cout, H, W in SHAPES:
    net = {"C": cin, "H": H, "W": W, "classes": 10, "ops": [WL.conv(0, cout, 3, 1, 1)]}
    plan = LB.Plan(net, B, mode="column", prec="bf16")
    ds = LB.DeviceState(plan)
    ds.params.normal_()
    ds.x.normal_()
    for _ in range(3):
        ds.forward()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        ds.forward()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    fl = 2 * 9 * cin * cout * H * W * B
    print("cin %4d cout %4d %3dx%3d B%d: %.3f ms  %.1f TFLOP/s  tc=%d" % (cin, cout, H, W, B, ms, fl / ms / 1e9,
                                                                          plan.last_tc_launches()))

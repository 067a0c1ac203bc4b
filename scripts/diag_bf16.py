"""Diagnostic (GPU): where do bf16 GPU feature maps differ from the bf16-storage oracle?
Counts, per VGG prefix, elements that differ and max-pool argmax / ReLU-mask decisions that flip."""
import sys
import os

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as WL  # noqa: E402
from oracle import column as C  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

net = WL.vgg16(H=64, W=64, width_div=4)
B = 2
params = WL.make_params(net, seed=2, bias_scale=0.05, bf16=True)
x = WL.make_input(net, B, seed=0, bf16=True)
ts, aux = C.forward(net, params, x, store=C.bf16_store)
for L in range(1, len(net["ops"]) + 1):
    sub = dict(net, ops=net["ops"][:L])
    sp = {"convs": params["convs"][:L], "head": params["head"]}
    plan = LB.Plan(sub, B, mode="column", prec="bf16")
    # head dims differ for prefixes; build a head that matches
    cl = plan.tensor(L)[0]
    sp["head"] = {"fc_w": np.zeros((net["classes"], cl)), "fc_b": np.zeros(net["classes"])}
    ds = LB.DeviceState(plan)
    ds.load(params=sp, x=x)
    ds.forward()
    torch.cuda.synchronize()
    z = plan.from_nhwc(ds.zl.float().cpu().numpy(), L)
    ref = ts[L]
    diff = z != ref
    ulp = np.abs(z - ref) / np.maximum(np.abs(ref), 1e-30)
    print("op %2d %-7s n=%8d differ=%6d maxrel=%.2e zero_flip=%d" % (
        L - 1, net["ops"][L - 1]["kind"], ref.size, diff.sum(), ulp[diff].max() if diff.any() else 0,
        ((z > 0) != (ref > 0)).sum()))

"""Diagnostic (GPU): per-op gradient errors of the fp32 path on a reduced VGG."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as WL  # noqa: E402
from oracle import column as C  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

net = WL.vgg16(H=64, W=64, width_div=8)
if len(sys.argv) > 1:
    net = dict(net, ops=net["ops"][:int(sys.argv[1])])
B = 2
params = WL.make_params(net, seed=2, bias_scale=0.05)
x = WL.make_input(net, B, seed=0)
shp = C.out_hw(net)
c, h, w = shp[-1]
params["head"] = {"fc_w": np.zeros((10, c)), "fc_b": np.zeros(10)}
dzl = WL.make_dzl((B, c, h, w))
ts, aux = C.forward(net, params, x)
g_ref, _ = C.backward(net, params, ts, aux, dzl, need_dx=False)
for mode, kw in (("column", {}), ("2ps", {"n_bands": 3})):
    plan = LB.Plan(net, B, mode=mode, prec="fp32", **kw)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, dzl=dzl)
    ds.forward()
    ds.backward()
    torch.cuda.synchronize()
    g, _ = plan.unpack_grads(ds.grads.cpu().numpy())
    for i, (a, b) in enumerate(zip(g, g_ref)):
        if b is None:
            continue
        print(mode, i, " ".join("%s:%.2e" % (k, np.max(np.abs(a[k] - b[k])) / np.max(np.abs(b[k]))) for k in b))
    print("db0 gpu", g[0]["b"])
    print("db0 ref", g_ref[0]["b"])

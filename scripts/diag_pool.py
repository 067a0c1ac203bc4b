"""Diagnostic (GPU): conv+maxpool gradients vs the oracle for several shapes (fp32)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as WL  # noqa: E402
from oracle import column as C  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

for (H, cin, cout, bias) in [(8, 8, 8, 0.05), (8, 64, 64, 0.05), (16, 32, 32, 0.05), (8, 64, 64, 0.5),
                             (8, 64, 64, 0.0), (4, 64, 64, 0.05), (8, 16, 64, 0.05), (8, 64, 16, 0.05)]:
    net = {"C": cin, "H": H, "W": H, "classes": 10, "ops": [WL.conv(0, cout, 3, 1, 1), WL.maxpool(1, 2, 2, 0)]}
    B = 2
    params = WL.make_params(net, seed=2, bias_scale=bias)
    x = np.maximum(WL.make_input(net, B, seed=0) - 0.5, 0)
    c, h, w = C.out_hw(net)[-1]
    dzl = WL.make_dzl((B, c, h, w))
    ts, aux = C.forward(net, params, x, store=C.fp32_store)
    g_ref, _ = C.backward(net, params, ts, aux, dzl, need_dx=False)
    plan = LB.Plan(net, B, mode="column", prec="fp32")
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, dzl=dzl)
    ds.forward()
    ds.backward()
    torch.cuda.synchronize()
    g, _ = plan.unpack_grads(ds.grads.cpu().numpy())
    z = plan.from_nhwc(ds.zl.float().cpu().numpy(), 2)
    print(H, cin, cout, bias, "zl %.1e" % (np.abs(z - ts[2]).max()),
          " ".join("%s:%.2e" % (k, np.max(np.abs(g[0][k] - g_ref[0][k])) / np.max(np.abs(g_ref[0][k]))) for k in g_ref[0]))

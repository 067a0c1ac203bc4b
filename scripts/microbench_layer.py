"""Microbenchmark (GPU): one conv layer (after a cheap 1x1 producer, so its dgrad runs too),
forward + backward through the C-ABI (bf16, column mode); per-kind kernel times of the measured
layer from the library's per-op profile.  Usage:
    python scripts/microbench_layer.py cin,cout,H,W[,k,s] ...
cin = 3 measures the first layer (no producer, no dgrad)."""
import csv
import os
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as WL  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

B = int(os.environ.get("B", "32"))
shapes = [tuple(int(v) for v in a.split(",")) for a in sys.argv[1:]] or [(64, 64, 56, 224)]
for sh in shapes:
    cin, cout, H, W = sh[:4]
    k = sh[4] if len(sh) > 4 else 3
    s = sh[5] if len(sh) > 5 else 1
    if cin <= 8:
        net = {"C": cin, "H": H, "W": W, "classes": 10, "ops": [WL.conv(0, cout, k, s, k // 2)]}
        op = 0
    else:
        net = {"C": 8, "H": H, "W": W, "classes": 10,
               "ops": [WL.conv(0, cin, 1, 1, 0), WL.conv(1, cout, k, s, k // 2, epi=os.environ.get("EPI", "bias"))]}
        op = 1
    nb = int(os.environ.get("NBANDS", "0"))
    plan = LB.Plan(net, B, mode="2ps" if nb else "column", prec="bf16", **({"n_bands": nb} if nb else {}))
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
    path = os.path.join(tempfile.gettempdir(), "mb_layer.csv")
    plan.profile_dump(path)
    plan.profile(False)
    out = {}
    for r in csv.DictReader(open(path)):
        if int(r["op"]) == op:
            out[r["kind"]] = (float(r["ms"]) / n, float(r["flops"]) / max(float(r["ms"]), 1e-9) / 1e9)
    txt = " | ".join("%s %.3f ms %.0f TF/s" % (kd, v[0], v[1]) for kd, v in sorted(out.items()))
    print("cin %4d cout %4d %4dx%4d k%d s%d B%d | %s" % (cin, cout, H, W, k, s, B, txt), flush=True)

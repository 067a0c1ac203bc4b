"""Runs warm-up steps of the bench workload, then ONE lrcnn_step between cudaProfilerStart/Stop
(for `ncu --profile-from-start off`): the launch list of exactly one training step.
usage: python scripts/one_step.py [config] [n_bands]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as WL  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 4
if cfg == "c2":
    net, B = WL.vgg16(H=224, W=224, segments="pool"), 32
elif cfg == "c3":
    net, B = WL.resnet50(H=224, W=224), 256
elif cfg == "c3bn":   # training-mode BN, per-block checkpoints (bench --bn-train --segments block)
    net, B = WL.resnet50(H=224, W=224, bn_train=True, segments="block"), 256
elif cfg == "c4bn":
    net, B = WL.resnet50(H=3600, W=2400, bn_train=True, segments="block"), 8
elif cfg == "c5":
    net, B = WL.vgg16(H=2048, W=2048, segments="pool"), 16
else:
    net, B = WL.resnet50(H=3600, W=2400), 8
plan = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=nb, flags=LB.FLAG_BALANCED_BANDS | LB.FLAG_FP_MERGE | LB.FLAG_REQUIRE_TC)   # = bench.py defaults
ds = LB.DeviceState(plan)
ds.load(params=WL.make_params(net, seed=2), x=WL.make_input(net, B, seed=1000), labels=WL.make_labels(net, B))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    for _ in range(3):
        ds.step(1e-3, stream=st)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    ds.step(1e-3, stream=st)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
print("launches per step", plan.last_launches())

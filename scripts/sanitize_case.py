"""One small bf16 training step through the C-ABI for compute-sanitizer runs (scripts/sanitize.sh):
a full-width ResNet-50 conv2_x slice (so the fused bottleneck kernel, the fused pointwise dgrad + wgrad
and the CTA-pair kernels run) with 3 bands, FP merge and balanced bands as bench.py plans them.
`python scripts/sanitize_case.py bn`: the same slice with training-mode BN (statistics / sums sweeps,
BN tail, bn.cu kernels)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads as WL  # noqa: E402
from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

bn = len(sys.argv) > 1 and sys.argv[1] == "bn"   # training-mode BN, per-block checkpoints (f4 sweeps)
net = WL.resnet50(H=64, W=40, width_div=1, blocks=(3, 1, 1, 1), bn_train=bn, segments="block" if bn else "stage")
B = 2
plan = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=3,
               flags=LB.FLAG_BALANCED_BANDS | LB.FLAG_FP_MERGE | LB.FLAG_REQUIRE_TC)
ds = LB.DeviceState(plan)
ds.load(params=WL.make_params(net, seed=2, bf16=True), x=WL.make_input(net, B, seed=0, bf16=True),
        labels=WL.make_labels(net, B))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    ds.step(1e-3, stream=st)
torch.cuda.synchronize()
print("ok loss", float(ds.loss), "launches", plan.last_launches())

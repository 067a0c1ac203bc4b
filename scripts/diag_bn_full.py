"""Diagnostic (GPU): z^L of full-width ResNet-50 with training-mode BN vs the oracle under several plans."""
import sys
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import workloads as WL
from oracle import column as C
from gpu_util import run_capture
from paper_2401_11471_b200 import lrcnn as LB


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


H = int(sys.argv[1]) if len(sys.argv) > 1 else 224
wd = int(sys.argv[2]) if len(sys.argv) > 2 else 1
B = 2
for segs in ("block",):
    net = WL.resnet50(H=H, W=H, bn_train=True, segments=segs, width_div=wd)
    for prec in ("fp32", "bf16"):
        bf = prec == "bf16"
        params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=bf)
        x = WL.make_input(net, B, bf16=bf)
        ts, _ = C.forward(net, params, x, store=C.bf16_store if bf else C.fp32_store)
        c, h, w = C.out_hw(net)[-1]
        dzl = WL.make_dzl((B, c, h, w), bf16=bf)
        for mode, kw, flags in (("column", {}, 0), ("2ps", {"n_bands": 1}, 0), ("2ps", {"n_bands": 3}, 0)):
            try:
                _, zl, g, tsg = run_capture(net, B, prec, mode, params, x, dzl, flags=flags, **kw)
                errs = [(rel(tsg[t], ts[t]), t, net["ops"][t - 1]["kind"]) for t in range(1, len(ts))]
                first = next(((e, t, k) for e, t, k in errs if e > (2e-2 if bf else 1e-5)), None)
                print(segs, prec, mode, kw, "zL", rel(zl, ts[-1]), "first bad map", first, flush=True)
            except Exception as e:
                print(segs, prec, mode, kw, "error", repr(e)[:200], flush=True)

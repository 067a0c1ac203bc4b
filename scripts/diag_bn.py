"""Diagnostic (GPU): worst gradient errors of the bf16 BN path vs the decision-conditioned oracle,
for the CE-head delta^L and the random delta^L field, and for the frozen-BN twin of the net."""
import sys
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import workloads as WL
from oracle import column as C
from conditioned import validate_forward, conditioned_grads
from gpu_util import run_capture


def errs(net, dzl_kind, B=2, n_bands=3, mode="2ps"):
    params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=True)
    x = WL.make_input(net, B, bf16=True)
    ts, aux = C.forward(net, params, x, store=C.bf16_store)
    c, h, w = C.out_hw(net)[-1]
    if dzl_kind == "random":
        dzl = WL.make_dzl((B, c, h, w), bf16=True)
    else:
        _, dzl, _, _ = C.head_forward_backward(ts[-1], params["head"], WL.make_labels(net, B))
        dzl = WL.round_bf16(dzl)
    kw = {} if mode == "column" else {"n_bands": n_bands}
    _, zl, g, tsg = run_capture(net, B, "bf16", mode, params, x, dzl, **kw)
    _, aux_g = validate_forward(net, params, tsg, C.bf16_store, 2e-2)
    gr = conditioned_grads(net, params, tsg, aux_g, dzl)
    out = []
    for i, (a, b) in enumerate(zip(g, gr)):
        if b is None:
            continue
        for k in b:
            out.append((float(np.max(np.abs(a[k] - b[k])) / np.max(np.abs(b[k]))), i, k,
                        float(np.max(np.abs(b[k]))), float(np.sum(np.abs(b[k])))))
    out.sort(reverse=True)
    return out[:6]


for bn in (True, False):
    net = WL.resnet50(H=64, W=48, width_div=8, blocks=(2, 1, 1, 1), bn_train=bn)
    for kind in ("head", "random"):
        for mode in ("column", "2ps"):
            print("bn_train" if bn else "frozen", kind, mode, errs(net, kind, mode=mode), flush=True)

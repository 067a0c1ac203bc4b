"""Column (layer-by-layer) dataflow oracle -- TEST INFRASTRUCTURE ONLY.

The plain definition LR-CNN must reproduce exactly ("without any loss of
accuracy"): every feature map is computed layer by layer over the
full height and kept (Fig. 1; SPEC column-oracle S:204-261).

  forward   -- Eq. (1) per op in topological order, all tensors stored.
  backward  -- Eq. (2) per op in reverse order: delta, dgrad (adjoint), wgrad.
  head      -- GAP -> FC -> softmax-CE (mean over B) on the concatenated z^L
               (Alg. 1 l.11-14).
  sgd       -- theta <- theta - lr*g (Alg. 1 l.24).

Op semantics: a conv op computes
  t = relu?( epi(Conv(src)) + res ),  epi in {bias: +b, affine: gamma*c+beta, none}
ReLU'(0) = 0.  Everything is fp64, NCHW.

Training-mode BatchNorm (the paper names BN in FP, but excludes it
from its analysis -- DESIGN.md reading R24): a "bn" op computes, per channel over the whole batch
and map (M = B*H*W values; biased variance, eps = BN_EPS),
  mean = sum(c)/M,  var = sum((c-mean)^2)/M,  xh = (c-mean)/sqrt(var+eps),
  t = relu?( gamma*xh + beta + res )
and its backward the textbook batch-statistics adjoint (da = gated dt):
  dbeta = sum(da),  dgamma = sum(da*xh),
  dc = gamma/sqrt(var+eps) * (da - dbeta/M - xh*dgamma/M),  dres = da.
"""
import numpy as np

import oracle as O


def out_hw(net):
    """(C, H, W) of every tensor id by the standard shape law."""
    shp = [(net["C"], net["H"], net["W"])]
    for op in net["ops"]:
        c, h, w = shp[op["src"]]
        if op["kind"] == "conv":
            shp.append((op["cout"], O.out_dim(h, op["p"], op["p"], op["k"], op["s"]),
                        O.out_dim(w, op["p"], op["p"], op["k"], op["s"])))
        elif op["kind"] == "maxpool":
            shp.append((c, O.out_dim(h, op["p"], op["p"], op["k"], op["s"]),
                        O.out_dim(w, op["p"], op["p"], op["k"], op["s"])))
        elif op["kind"] == "add" or op["kind"] == "bn":
            if op["kind"] == "add" or op.get("res", -1) >= 0:
                assert shp[op["res"]] == (c, h, w)
            shp.append((c, h, w))
        else:
            raise ValueError(op["kind"])
        if min(shp[-1]) < 1:
            raise ValueError("shape-underflow at op %d" % (len(shp) - 2))
    return shp


def conv_op_fwd(op, prm, x, res, pads):
    """One conv op on a slab: returns (t, c) where c = raw Conv output (needed for d gamma)."""
    c = O.conv2d_fwd(x, prm["w"], None, op["s"], pads)
    if op["epi"] == "bias":
        a = c + prm["b"][None, :, None, None]
    elif op["epi"] == "affine":
        a = prm["gamma"][None, :, None, None] * c + prm["beta"][None, :, None, None]
    else:
        a = c
    if res is not None:
        a = a + res
    t = np.maximum(a, 0.0) if op["relu"] else a
    return t, c


def conv_op_bwd(op, prm, x, c, t, dt, pads, in_hw):
    """Backward of conv_op_fwd given its stored output t (gate t>0, ReLU'(0)=0).
    Returns (dx, dres_or_None, grads dict)."""
    da = dt * (t > 0) if op["relu"] else dt
    g = {}
    if op["epi"] == "bias":
        g["b"] = da.sum(axis=(0, 2, 3))
        dc = da
    elif op["epi"] == "affine":
        g["gamma"] = (da * c).sum(axis=(0, 2, 3))
        g["beta"] = da.sum(axis=(0, 2, 3))
        dc = prm["gamma"][None, :, None, None] * da
    else:
        dc = da
    g["w"], _ = O.conv2d_bwd_weight(x, dc, op["k"], op["s"], pads, with_bias=False)
    dx = O.conv2d_bwd_data(prm["w"], dc, in_hw, op["s"], pads)
    dres = da if op["res"] >= 0 else None
    return dx, dres, g


BN_EPS = 1e-5   # DESIGN.md R24


def bn_stats(c):
    """Batch statistics of a full map c [B, C, H, W]: (mean, biased var) per channel."""
    mean = c.mean(axis=(0, 2, 3))
    var = ((c - mean[None, :, None, None]) ** 2).mean(axis=(0, 2, 3))
    return mean, var


def bn_apply(prm, c, mean, var, res, relu):
    """t = relu?(gamma * (c - mean)/sqrt(var + eps) + beta + res) on any rows of c."""
    xh = (c - mean[None, :, None, None]) / np.sqrt(var + BN_EPS)[None, :, None, None]
    a = prm["gamma"][None, :, None, None] * xh + prm["beta"][None, :, None, None]
    if res is not None:
        a = a + res
    return np.maximum(a, 0.0) if relu else a


def bn_bwd_full(prm, c, t, dt, mean, var, relu, M):
    """Backward of a bn op on the full map: returns (dc, da, {gamma, beta})."""
    da = dt * (t > 0) if relu else dt
    sig = np.sqrt(var + BN_EPS)[None, :, None, None]
    xh = (c - mean[None, :, None, None]) / sig
    dbeta = da.sum(axis=(0, 2, 3))
    dgamma = (da * xh).sum(axis=(0, 2, 3))
    dc = prm["gamma"][None, :, None, None] / sig * (
        da - dbeta[None, :, None, None] / M - xh * dgamma[None, :, None, None] / M)
    return dc, da, {"gamma": dgamma, "beta": dbeta}


def bf16_store(a):
    """Round to the nearest bfloat16 (round-to-nearest-even), kept as float64.

    Storage-precision model for bf16 parity (reading R17b): the kernel
    stores every feature map in bf16 and takes its integer decisions (ReLU
    masks, max-pool argmax) on the stored values; the oracle takes them in the
    same precision by storing its fp64 results rounded the same way.  All
    arithmetic stays fp64."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(a))


def fp32_store(a):
    """Round to float32, kept as float64: the storage model for the fp32 parity mode
    (max-pool argmax on near-ties and ReLU masks decided on fp32 values, R17b)."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def forward(net, params, x, store=None):
    """Column FP: returns (tensors list [t0..tL], aux) with every feature map kept.
    store: optional storage-rounding function applied to every op output (bf16 parity)."""
    st = store or (lambda a: a)
    ts = [np.asarray(x, dtype=np.float64)]
    aux = []
    for i, op in enumerate(net["ops"]):
        src = ts[op["src"]]
        p = op.get("p", 0)
        pads = (p, p, p, p)
        if op["kind"] == "conv":
            res = ts[op["res"]] if op["res"] >= 0 else None
            t, c = conv_op_fwd(op, params["convs"][i], src, res, pads)
            aux.append(c)
        elif op["kind"] == "maxpool":
            t, am = O.maxpool_fwd(src, op["k"], op["s"], pads)
            aux.append(am)
        elif op["kind"] == "bn":
            mean, var = bn_stats(src)
            res = ts[op["res"]] if op["res"] >= 0 else None
            t = bn_apply(params["convs"][i], src, mean, var, res, op["relu"])
            aux.append((mean, var))
        else:
            a = src + ts[op["res"]]
            t = np.maximum(a, 0.0) if op["relu"] else a
            aux.append(None)
        ts.append(st(t))
    return ts, aux


def backward(net, params, ts, aux, dzl, need_dx=True, trace=None):
    """Column BP from delta^L (= dz^L); returns (grads per op, dx).
    trace: optional dict, filled per bn op with the summation magnitudes of its parameter gradients
    {"beta": sum|da|, "gamma": sum|da*xh|} per channel (the condition of those full-map sums)."""
    ds = [None] * len(ts)
    ds[-1] = np.asarray(dzl, dtype=np.float64).copy()
    grads = [None] * len(net["ops"])

    def acc(tid, v):
        ds[tid] = v.copy() if ds[tid] is None else ds[tid] + v

    for i in range(len(net["ops"]) - 1, -1, -1):
        op = net["ops"][i]
        dt = ds[i + 1]
        if dt is None:
            dt = np.zeros_like(ts[i + 1])
        src = ts[op["src"]]
        p = op.get("p", 0)
        pads = (p, p, p, p)
        if op["kind"] == "conv":
            dx, dres, g = conv_op_bwd(op, params["convs"][i], src, aux[i], ts[i + 1], dt, pads,
                                      src.shape[2:])
            grads[i] = g
            if op["src"] > 0 or need_dx:
                acc(op["src"], dx)
            if dres is not None:
                acc(op["res"], dres)
        elif op["kind"] == "maxpool":
            acc(op["src"], O.maxpool_bwd(aux[i], dt, src.shape[2:]))
        elif op["kind"] == "bn":
            mean, var = aux[i]
            M = src.shape[0] * src.shape[2] * src.shape[3]
            dc, da, g = bn_bwd_full(params["convs"][i], src, ts[i + 1], dt, mean, var, op["relu"], M)
            grads[i] = g
            if trace is not None:
                xh = (src - mean[None, :, None, None]) / np.sqrt(var + BN_EPS)[None, :, None, None]
                trace[i] = {"beta": np.abs(da).sum(axis=(0, 2, 3)), "gamma": np.abs(da * xh).sum(axis=(0, 2, 3))}
            if op["src"] > 0 or need_dx:
                acc(op["src"], dc)
            if op["res"] >= 0:
                acc(op["res"], da)
        else:
            da = dt * (ts[i + 1] > 0) if op["relu"] else dt
            acc(op["src"], da)
            acc(op["res"], da)
    return grads, ds[0]


def head_forward_backward(zl, head, labels):
    """GAP -> FC -> softmax cross-entropy with mean over B.
    Returns (loss, dzl, grads{fc_w, fc_b}, logits)."""
    zl = np.asarray(zl, dtype=np.float64)
    B, C, H, W = zl.shape
    gap = zl.mean(axis=(2, 3))                       # [B, C]
    logits = gap @ head["fc_w"].T + head["fc_b"]     # [B, classes]
    m = logits.max(axis=1, keepdims=True)
    e = np.exp(logits - m)
    ssum = e.sum(axis=1, keepdims=True)
    lse = (m + np.log(ssum))[:, 0]
    labels = np.asarray(labels)
    loss = float(np.mean(lse - logits[np.arange(B), labels]))
    dlog = e / ssum
    dlog[np.arange(B), labels] -= 1.0
    dlog /= B
    g = {"fc_w": dlog.T @ gap, "fc_b": dlog.sum(axis=0)}
    dgap = dlog @ head["fc_w"]                       # [B, C]
    dzl = np.broadcast_to(dgap[:, :, None, None] / (H * W), zl.shape).copy()
    return loss, dzl, g, logits


def sgd(params, grads, head_grads, lr):
    """theta <- theta - lr * g for every conv parameter and the head."""
    new = {"convs": [], "head": {}}
    for prm, g in zip(params["convs"], grads):
        if prm is None:
            new["convs"].append(None)
            continue
        new["convs"].append({k: prm[k] - lr * g[k] for k in prm})
    new["head"] = {k: params["head"][k] - lr * head_grads[k] for k in params["head"]}
    return new


def step(net, params, x, labels, lr):
    """One training iteration (Alg. 1 with N=1): returns (new_params, loss, grads, head_grads, ts)."""
    ts, aux = forward(net, params, x)
    loss, dzl, hg, _ = head_forward_backward(ts[-1], params["head"], labels)
    grads, _ = backward(net, params, ts, aux, dzl, need_dx=False)
    return sgd(params, grads, hg, lr), loss, grads, hg, ts

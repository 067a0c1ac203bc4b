"""Seeded synthetic workloads shared by the oracle and the CUDA path.

This module holds ONLY workload definitions (layer topologies as plain data)
and seeded random input generators.  It contains none of the method's
arithmetic (no shape propagation, no band/halo logic, no convolution): both
the oracle (``oracle/``) and the product (``paper_2401_11471_b200/``) take
what this module produces as *inputs* and do their own computation.

Net description (a plain dict):
  {"C": in_channels, "H": .., "W": .., "classes": n, "ops": [op, ...]}
Tensor ids: 0 = the image; op i produces tensor i+1.  An op is a dict:
  conv:    {"kind":"conv","src":t,"cout":C,"k":k,"s":s,"p":p,
            "epi":"bias"|"affine"|"none","relu":bool,"res":t or -1,"seg_end":bool}
           t_out = relu?( epi(Conv(t_src)) + t_res )
  maxpool: {"kind":"maxpool","src":t,"k":k,"s":s,"p":p,"seg_end":bool}
  add:     {"kind":"add","src":t,"res":t2,"relu":bool,"seg_end":bool}
  bn:      {"kind":"bn","src":t,"res":t or -1,"relu":bool,"seg_end":bool}
           training-mode batch normalisation: statistics of t_src over the whole
           batch and map, t_out = relu?( gamma*(t_src-mean)/sqrt(var+eps) + beta + t_res )
"seg_end" marks a checkpoint boundary after the op (2PS-H / OverL-H).

Input recipe:
  x ~ U[0,1) seed 0, labels ~ U{0..classes-1} seed 1, conv weights
  U[-a,a], a=(c_in k^2)^(-1/2) seed 2, FC U[-a,a], a=C_L^(-1/2),
  bias/beta ~ U[-bias_scale, bias_scale], gamma ~ U[1-g, 1+g]; delta^L field
  G ~ U(-1,1) seed 3 (C1's loss sum(G * z^L)).
"""
import numpy as np


def conv(src, cout, k=3, s=1, p=1, epi="bias", relu=True, res=-1, seg_end=False):
    return {"kind": "conv", "src": src, "cout": cout, "k": k, "s": s, "p": p, "epi": epi,
            "relu": relu, "res": res, "seg_end": seg_end}


def maxpool(src, k=2, s=2, p=0, seg_end=False):
    return {"kind": "maxpool", "src": src, "k": k, "s": s, "p": p, "seg_end": seg_end}


def add(src, res, relu=True, seg_end=False):
    return {"kind": "add", "src": src, "res": res, "relu": relu, "seg_end": seg_end}


def bn(src, res=-1, relu=True, seg_end=False):
    return {"kind": "bn", "src": src, "res": res, "relu": relu, "seg_end": seg_end}


# ---------------------------------------------------------------- presets
def tiny3(p=1, H=32, W=32, C=1, ch=8, classes=10):
    """C1: three 3x3 convs (1->8->8->8), stride 1, ReLU after each (BASELINE.json configs[0])."""
    ops = [conv(0, ch, 3, 1, p), conv(1, ch, 3, 1, p), conv(2, ch, 3, 1, p)]
    return {"C": C, "H": H, "W": W, "classes": classes, "ops": ops, "name": "tiny3_p%d" % p}


VGG16_CFG = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


def vgg16(H=224, W=224, C=3, classes=10, segments="none", width_div=1, cfg=None):
    """VGG-16 config D conv stack: 13 conv3x3/p1 + ReLU, 5 max-pool 2x2/s2 (Table I "13").

    segments: "none" (whole-stack row-centric) or "pool" (checkpoint after every pool
    but the last, the 2PS-H / OverL-H hybrid).  width_div divides channel counts
    (reduced nets for parity tests)."""
    ops = []
    t = 0
    cfg = cfg or VGG16_CFG
    for v in cfg:
        if v == "M":
            ops.append(maxpool(t, 2, 2, 0, seg_end=(segments == "pool")))
        else:
            ops.append(conv(t, max(1, v // width_div), 3, 1, 1))
        t += 1
    ops[-1]["seg_end"] = False
    return {"C": C, "H": H, "W": W, "classes": classes, "ops": ops, "name": "vgg16"}


def resnet50(H=224, W=224, C=3, classes=10, segments="stage", width_div=1, blocks=(3, 4, 6, 3), bn_train=False):
    """ResNet-50 v1.5 (torchvision topology: stride on the 3x3 of the first block of stages 2-4,
    1x1 projection shortcut on every stage's first block), frozen-statistics BN folded into
    per-channel affine convs (R11, R14).  Bottleneck:
        a = relu(aff(conv1x1(x)));  b = relu(aff(conv3x3/s(a)));  sc = aff(conv1x1/s(x)) or x
        out = relu(aff(conv1x1(b)) + sc)      (the residual add is fused into the last conv)
    segments: "stage" checkpoints after the stem max-pool and after every stage but the last
    (2PS-H / OverL-H), "none" = whole-net row-centric, or a string naming the cut points: "p" the
    stem max-pool, "2" / "3" / "4" the end of conv2_x / conv3_x / conv4_x (e.g. "3": one checkpoint
    after conv3_x; "stage" == "p234"; "block" checkpoints after every bottleneck).
    bn_train: training-mode BatchNorm -- every affine conv becomes a plain conv
    (epi "none", no ReLU) followed by a "bn" op that carries the ReLU and the residual."""
    if bn_train:
        return _bn_train(resnet50(H, W, C, classes, segments, width_div, blocks))
    d = lambda c: max(8, c // width_div)
    cuts = {"stage": "p234", "none": ""}.get(segments, segments)
    ops = [conv(0, d(64), 7, 2, 3, epi="affine"), maxpool(1, 3, 2, 1, seg_end=("p" in cuts or cuts == "block"))]
    t, cin = 2, d(64)
    for si, (nb, w) in enumerate(zip(blocks, (64, 128, 256, 512))):
        for bi in range(nb):
            s = 2 if (bi == 0 and si > 0) else 1
            x = t
            ops.append(conv(x, d(w), 1, 1, 0, epi="affine"))
            a = len(ops)
            ops.append(conv(a, d(w), 3, s, 1, epi="affine"))
            b = len(ops)
            if bi == 0:
                ops.append(conv(x, d(4 * w), 1, s, 0, epi="affine", relu=False))
                sc = len(ops)
            else:
                sc = x
            ops.append(conv(b, d(4 * w), 1, 1, 0, epi="affine", relu=True, res=sc))
            t = len(ops)
            if cuts == "block" and not (si == len(blocks) - 1 and bi == nb - 1):
                ops[-1]["seg_end"] = True
        if str(si + 2) in cuts and si < len(blocks) - 1:
            ops[-1]["seg_end"] = True
    ops[-1]["seg_end"] = False
    return {"C": C, "H": H, "W": W, "classes": classes, "ops": ops, "name": "resnet50"}


def _bn_train(net):
    """Rewrite every affine conv op as conv (epi none, no ReLU, no residual) + bn op (ReLU,
    residual), renumbering tensor ids (topology bookkeeping only)."""
    ops, new_id = [], {0: 0}
    for i, op in enumerate(net["ops"]):
        o = dict(op)
        o["src"] = new_id[op["src"]]
        if op.get("res", -1) >= 0:
            o["res"] = new_id[op["res"]]
        if op["kind"] == "conv" and op["epi"] == "affine":
            c = dict(o, epi="none", relu=False, res=-1, seg_end=False)
            ops.append(c)
            ops.append(bn(len(ops), res=o["res"], relu=op["relu"], seg_end=op["seg_end"]))
        else:
            ops.append(o)
        new_id[i + 1] = len(ops)
    out = dict(net, ops=ops)
    out["name"] = net.get("name", "net") + "_bn"
    return out


def bn_chain(H=16, W=8, C=2, ch=4, n=3, p=1, res_every=0, classes=10):
    """Tiny BN test net: n x [conv3x3 (no bias) -> bn (ReLU)], optionally with a residual every
    res_every layers (the bn of layer j adds the output of layer j - res_every)."""
    ops, outs = [], [0]
    t = 0
    for j in range(n):
        ops.append(conv(t, ch, 3, 1, p, epi="none", relu=False))
        res = outs[j + 1 - res_every] if res_every and (j + 1) % res_every == 0 and j + 1 - res_every >= 1 else -1
        ops.append(bn(len(ops), res=res, relu=True))
        t = len(ops)
        outs.append(t)
    return {"C": C, "H": H, "W": W, "classes": classes, "ops": ops, "name": "bn_chain"}


# ---------------------------------------------------------------- inputs
def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def round_bf16(a):
    """Round float64 values to the nearest bfloat16 (round-to-nearest-even), returned as float64.
    Used so both sides see identical, bf16-representable inputs."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32).astype(np.float64).reshape(np.shape(a))


def make_input(net, B, seed=0, bf16=False):
    """x [B, C, H, W] (NCHW, float64) ~ U[0,1)."""
    x = _rng(seed).random((B, net["C"], net["H"], net["W"]))
    return round_bf16(x) if bf16 else x


def make_labels(net, B, seed=1):
    return _rng(seed).integers(0, net["classes"], size=B).astype(np.int32)


def channels(net):
    """Channel count of every tensor id (plain bookkeeping of the topology, no arithmetic of the method)."""
    ch = [net["C"]]
    for op in net["ops"]:
        ch.append(op["cout"] if op["kind"] == "conv" else ch[op["src"]])
    return ch


def make_params(net, seed=2, bias_scale=0.0, gamma_spread=0.0, bf16=False):
    """Per-op parameter dicts (conv: w [Co,Ci,k,k] OIHW, b, gamma, beta) and the FC head.
    Weights U[-a,a], a=(c_in k^2)^(-1/2)."""
    r = _rng(seed)
    ch = channels(net)
    rnd = round_bf16 if bf16 else (lambda a: a)
    convs = []
    for op in net["ops"]:
        if op["kind"] == "bn":
            co = ch[op["src"]]
            convs.append({
                "gamma": rnd(r.uniform(1 - gamma_spread, 1 + gamma_spread, size=co)) if gamma_spread
                else np.ones(co),
                "beta": rnd(r.uniform(-bias_scale, bias_scale, size=co)) if bias_scale else np.zeros(co)})
            continue
        if op["kind"] != "conv":
            convs.append(None)
            continue
        ci, co, k = ch[op["src"]], op["cout"], op["k"]
        a = (ci * k * k) ** -0.5
        p = {"w": rnd(r.uniform(-a, a, size=(co, ci, k, k)))}
        if op["epi"] == "bias":
            p["b"] = rnd(r.uniform(-bias_scale, bias_scale, size=co)) if bias_scale else np.zeros(co)
        elif op["epi"] == "affine":
            p["gamma"] = rnd(r.uniform(1 - gamma_spread, 1 + gamma_spread, size=co)) if gamma_spread \
                else np.ones(co)
            p["beta"] = rnd(r.uniform(-bias_scale, bias_scale, size=co)) if bias_scale else np.zeros(co)
        convs.append(p)
    cl = ch[-1]
    a = cl ** -0.5
    head = {"fc_w": rnd(r.uniform(-a, a, size=(net["classes"], cl))),
            "fc_b": rnd(r.uniform(-a, a, size=net["classes"]))}
    return {"convs": convs, "head": head}


def make_dzl(shape, seed=3, bf16=False):
    """C1's delta^L field G ~ U(-1,1) (loss = sum(G * z^L), so delta^L = G)."""
    g = _rng(seed).uniform(-1.0, 1.0, size=shape)
    return round_bf16(g) if bf16 else g

"""GPU parity on the paths bench.py times, against the fp64 oracle (R17d):

  * identity bottlenecks (the fused residual gradient, 12 of ResNet-50's 16 blocks) in fp32
    (1e-5) and bf16 (2e-2), COLUMN / 2PS / OverL / per-stage segments;
  * the full 13-conv VGG-16 in bf16, every mode;
  * C2 at its full size and batch (VGG-16 224x224, B = 32) and C4 at its full size and batch
    (ResNet-50 3600x2400, B = 8) in exactly bench.py's plan (2PS-H, balanced bands, decoupled FP
    bands, LRCNN_FLAG_REQUIRE_TC): every gradient vs the oracle.  delta^L is non-zero only where
    the oracle can afford to follow it (C2: images 0 and 31; C4: the top rows of image 0, whose
    dependency cone lies in a strip of the image), so the oracle computes those gradients EXACTLY
    while the GPU runs the full-size launch configuration;
  * lrcnn_step (FP, head, BP, SGD) in bf16 with bench.py's flags vs oracle.column.step.

Every stored map the GPU produced is first validated op by op against the oracle recomputed from
the GPU's own stored inputs (tests/conditioned.py), then the gradients are compared with the fp64
backward taken with those validated decisions; z^L is also compared with the plain oracle."""
import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from conditioned import rel, validate_forward, conditioned_grads, compare_grads, strip_rows
from gpu_util import run_capture, _nchw

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

TOL = {"fp32": 1e-5, "bf16": 2e-2}
BENCH_FLAGS = LB.FLAG_BALANCED_BANDS | LB.FLAG_FP_MERGE | LB.FLAG_REQUIRE_TC


def full_check(net, B, prec, modes, params, x, dzl, flags=0, tag=""):
    store = C.bf16_store if prec == "bf16" else C.fp32_store
    ts_ref, _ = C.forward(net, params, x, store=store)
    zl_fp64 = C.forward(net, params, x)[0][-1]   # true fp64 training, no storage rounding at all
    for mode, kw in modes:
        _, zl, g, ts = run_capture(net, B, prec, mode, params, x, dzl, flags=flags, **kw)
        assert rel(zl, ts_ref[-1]) <= TOL[prec], (tag, mode, kw, "zL vs plain oracle", rel(zl, ts_ref[-1]))
        assert rel(zl, zl_fp64) <= TOL[prec], (tag, mode, kw, "zL vs fp64 oracle", rel(zl, zl_fp64))
        _, aux = validate_forward(net, params, ts, store, TOL[prec])
        g_ref = conditioned_grads(net, params, ts, aux, dzl)
        compare_grads(g, g_ref, TOL[prec], (tag, mode, str(kw)))


def _gamma_zero(params, every=3):
    """Zero every `every`-th gamma of every affine conv (ResNet's zero-init last BN gamma; dgamma
    must come out exact)."""
    for p in params["convs"]:
        if p is not None and "gamma" in p:
            p["gamma"][::every] = 0.0
    return params


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_resnet_identity_blocks_vs_oracle(prec):
    """Two identity bottlenecks per stage at block-input widths 64 / 128 / 256 (so the fused residual
    gradient engages in bf16), some gammas exactly 0, head delta^L; COLUMN, 2PS (3 bands and 1-row
    bands), OverL, per-stage segments."""
    net = WL.resnet50(H=64, W=40, width_div=4, blocks=(3, 2, 2, 1))
    B = 2
    bf = prec == "bf16"
    params = _gamma_zero(WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=bf))
    x = WL.make_input(net, B, seed=0, bf16=bf)
    ts, _ = C.forward(net, params, x, store=C.bf16_store if bf else C.fp32_store)
    _, dzl, _, _ = C.head_forward_backward(ts[-1], params["head"], WL.make_labels(net, B))
    dzl = WL.round_bf16(dzl) if bf else dzl
    full_check(net, B, prec, [("column", {}), ("2ps", {"n_bands": 3}), ("2ps", {"band_rows": 1}),
                              ("overl", {"n_bands": 2})], params, x, dzl,
               flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION | (LB.FLAG_REQUIRE_TC if bf else 0), tag="identity")


def test_resnet_stage2_full_width_fused_pointwise_backward():
    """ResNet-50's conv2_x at full width (64 / 256 channels): the pointwise convolutions' backward
    runs as the fused dgrad + wgrad kernel (k_dwgrad_pw: 256 -> 64 with the fused residual addend,
    64 -> 256 with the gate, the 64 -> 256 projection accumulating); bf16 vs the oracle (R17d),
    COLUMN / 2PS / 1-row bands, some gammas 0."""
    net = WL.resnet50(H=48, W=40, width_div=1, blocks=(3, 1, 1, 1))
    B = 2
    params = _gamma_zero(WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=True))
    x = WL.make_input(net, B, seed=0, bf16=True)
    ts, _ = C.forward(net, params, x, store=C.bf16_store)
    _, dzl, _, _ = C.head_forward_backward(ts[-1], params["head"], WL.make_labels(net, B))
    dzl = WL.round_bf16(dzl)
    full_check(net, B, "bf16", [("column", {}), ("2ps", {"n_bands": 3}), ("2ps", {"band_rows": 1})], params, x, dzl,
               flags=LB.FLAG_REQUIRE_TC, tag="stage2 full width")


def test_vgg16_full_depth_bf16_all_modes():
    """All 13 convs and 5 pools of VGG-16 (reduced channels, 64x64) in bf16: whole-stack 2PS,
    per-pool 2PS-H, OverL-H, 1-row bands, COLUMN -- every gradient vs the oracle (R17d)."""
    B = 2
    for segs in ("none", "pool"):
        net = WL.vgg16(H=64, W=64, width_div=4, segments=segs)
        params = WL.make_params(net, seed=2, bias_scale=0.05, bf16=True)
        x = WL.make_input(net, B, seed=0, bf16=True)
        ts, _ = C.forward(net, params, x, store=C.bf16_store)
        _, dzl, _, _ = C.head_forward_backward(ts[-1], params["head"], WL.make_labels(net, B))
        dzl = WL.round_bf16(dzl)
        full_check(net, B, "bf16", [("column", {}), ("2ps", {"n_bands": 4}), ("2ps", {"band_rows": 1}),
                                    ("overl", {"n_bands": 2})], params, x, dzl,
                   flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION | LB.FLAG_REQUIRE_TC, tag=segs)


def test_c2_full_size_every_gradient_vs_oracle():
    """C2 exactly as bench.py runs it (VGG-16 224x224, B = 32, 2PS-H per pool, 4 balanced bands,
    decoupled FP bands, tcgen05 only).  delta^L is random on images 0 and 31 and zero elsewhere, so
    every gradient is a function of those two images: the oracle follows them exactly."""
    net = WL.vgg16(H=224, W=224, segments="pool")
    B, imgs = 32, [0, 31]
    params = WL.make_params(net, seed=2, bias_scale=0.05, bf16=True)
    x = WL.make_input(net, B, seed=1000, bf16=True)
    c, h, w = C.out_hw(net)[-1]
    dzl = np.zeros((B, c, h, w))
    dzl[imgs] = WL.make_dzl((len(imgs), c, h, w), bf16=True) * 1e-3
    _, zl, g, ts = run_capture(net, B, "bf16", "2ps", params, x, dzl, flags=BENCH_FLAGS, images=imgs, n_bands=4)
    ref_ts, _ = C.forward(net, params, x[imgs], store=C.bf16_store)
    assert rel(zl, ref_ts[-1]) <= TOL["bf16"], rel(zl, ref_ts[-1])
    _, aux = validate_forward(net, params, ts, C.bf16_store, TOL["bf16"])
    g_ref = conditioned_grads(net, params, ts, aux, dzl[imgs])
    compare_grads(g, g_ref, TOL["bf16"], "c2 full size")


def test_c4_full_size_every_gradient_vs_oracle():
    """C4 exactly as bench.py runs it (ResNet-50 3600x2400, B = 8, 2PS-H per stage, 8 balanced
    bands, decoupled FP bands, tcgen05 only).  delta^L is non-zero on the top 6 rows of image 0's
    z^L only; their dependency cone (oracle.enumerate.need_sets) lies in the top rows of every
    tensor, so the oracle follows every gradient exactly on a strip of image 0 while the GPU runs
    the full-size step."""
    H, W, B, j = 3600, 2400, 8, 6
    net = WL.resnet50(H=H, W=W, segments="stage")
    cone = strip_rows(net, j)
    Hs = cone[0][1]
    params = WL.make_params(net, seed=2, bias_scale=0.05, gamma_spread=0.1, bf16=True)
    x = WL.make_input(net, B, seed=1000, bf16=True)
    c, h, w = C.out_hw(net)[-1]
    dzl = np.zeros((B, c, h, w))
    dzl[0, :, :j] = WL.make_dzl((1, c, j, w), bf16=True)[0] * 1e-3
    strip = dict(net, H=Hs)
    shp_s = C.out_hw(strip)
    rows = {t: shp_s[t][1] for t in range(len(shp_s))}
    _, zl, g, ts = run_capture(net, B, "bf16", "2ps", params, x, dzl, flags=BENCH_FLAGS, images=[0], rows=rows,
                               n_bands=8)
    # z^L rows [0, j) of image 0 vs the plain oracle on the strip
    ref_ts, _ = C.forward(dict(strip, ops=[dict(o, seg_end=False) for o in net["ops"]]), params,
                          x[0:1, :, :Hs], store=C.bf16_store)
    assert rel(zl[:, :, :j], ref_ts[-1][:, :, :j]) <= TOL["bf16"]
    _, aux = validate_forward(strip, params, ts, C.bf16_store, TOL["bf16"], rows=cone)
    g_ref = conditioned_grads(strip, params, ts, aux, dzl[0:1, :, :shp_s[-1][1]])
    compare_grads(g, g_ref, TOL["bf16"], "c4 full size")


def test_bench_step_bf16_vs_oracle_step():
    """lrcnn_step in bf16 with bench.py's flags (2PS-H per stage, balanced + decoupled FP bands,
    tcgen05 only) on full-depth ResNet-50 (reduced width / resolution): loss vs the plain oracle
    step; the head gradient, every conv gradient and the SGD update vs the oracle conditioned on
    the maps the step stored (the step's forward is captured; graph replay is off while capturing)."""
    net = WL.resnet50(H=128, W=96, width_div=4, segments="stage")
    B, lr = 4, 0.05
    params = WL.make_params(net, seed=2, bias_scale=0.05, gamma_spread=0.2, bf16=True)
    x = WL.make_input(net, B, seed=0, bf16=True)
    lab = WL.make_labels(net, B)
    plan = LB.Plan(net, B, mode="2ps", prec="bf16", flags=BENCH_FLAGS, n_bands=8)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, labels=lab)
    L = len(net["ops"])
    bufs = {}
    for t in range(1, L + 1):
        c, cp, h, w = plan.tensor(t)
        bufs[t] = torch.zeros((B, h, w, cp), dtype=ds.dtype, device=ds.x.device)
        plan.debug_capture(t, bufs[t])
    ds.step(lr)
    torch.cuda.synchronize()
    assert plan.last_simt_fallbacks() == 0
    ts = [x] + [_nchw(bufs[t], plan.tensor(t)[0], list(range(B))) for t in range(1, L + 1)]
    _, loss_ref, _, _, ts_ref = C.step(net, params, x, lab, lr)
    loss = float(ds.loss.cpu())
    assert abs(loss - loss_ref) <= TOL["bf16"] * abs(loss_ref), (loss, loss_ref)
    assert rel(ts[-1], C.bf16_store(ts_ref[-1])) <= TOL["bf16"]
    _, aux = validate_forward(net, params, ts, C.bf16_store, TOL["bf16"])
    loss_c, dzl, hg, _ = C.head_forward_backward(ts[-1], params["head"], lab)
    assert abs(loss - loss_c) <= 1e-3 * abs(loss_c)
    g_ref = conditioned_grads(net, params, ts, aux, dzl)
    new_ref = C.sgd(params, g_ref, hg, lr)
    got, head = plan.unpack_grads(ds.master.cpu().numpy())
    assert np.all(ds.grads.cpu().numpy() == 0)

    def upd_ok(old, new_gpu, new_oracle, tag):
        # the update as the fp32 master stores it: lr * g to 2e-2 of its max, plus the fp32 rounding
        # of theta - lr * g (a few ulp of |theta|)
        d_ref, d_got = old - new_oracle, old - new_gpu
        slack = TOL["bf16"] * np.max(np.abs(d_ref)) + 4 * np.finfo(np.float32).eps * np.abs(old)
        assert np.all(np.abs(d_got - d_ref) <= slack), (tag, float(np.max(np.abs(d_got - d_ref) - slack)))

    for i, b in enumerate(new_ref["convs"]):
        if b is None:
            continue
        for k in b:
            upd_ok(params["convs"][i][k], got[i][k], b[k], (i, k))
    for k in ("fc_w", "fc_b"):
        upd_ok(params["head"][k], head[k], new_ref["head"][k], k)


def test_head_many_classes_fp32():
    """A 300-class head (more classes than the FC-gradient kernel's block): lrcnn_step's
    loss and every updated parameter vs the oracle step."""
    net = dict(WL.tiny3(p=1, H=12, W=10), classes=300)
    B, lr = 3, 0.05
    params = WL.make_params(net, seed=2, bias_scale=0.1)
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    new_ref, loss_ref, _, _, _ = C.step(net, params, x, lab, lr)
    plan = LB.Plan(net, B, mode="2ps", prec="fp32", band_rows=3)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, labels=lab)
    ds.step(lr)
    torch.cuda.synchronize()
    assert abs(float(ds.loss.cpu()) - loss_ref) <= 1e-5 * abs(loss_ref)
    got, head = plan.unpack_grads(ds.master.cpu().numpy())
    for k in ("fc_w", "fc_b"):
        d_ref = params["head"][k] - new_ref["head"][k]
        assert rel(params["head"][k] - head[k], d_ref) <= 1e-4, k

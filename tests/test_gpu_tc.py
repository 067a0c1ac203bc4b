"""GPU: the tcgen05 / TMEM / TMA implicit-GEMM kernels (FP, dgrad, wgrad) against the
oracle, layer shapes of VGG-16 and ragged bands (rows/cols not multiples of the
128-pixel tile), bf16 with fp32 accumulation; tolerance 2e-2 (north_star)."""
import numpy as np
import pytest

import workloads as WL
from oracle import column as C

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

TOL = 2e-2


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def run(net, B, mode, params, x, dzl, flags=0, **kw):
    plan = LB.Plan(net, B, mode=mode, prec="bf16", flags=flags, **kw)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, dzl=dzl)
    ds.forward()
    zl = plan.from_nhwc(ds.zl.float().cpu().numpy(), len(net["ops"]))
    ds.backward()
    torch.cuda.synchronize()
    if not flags & LB.FLAG_NO_TCGEN05:
        assert plan.last_tc_launches() > 0          # the tcgen05 kernels ran
    g, _ = plan.unpack_grads(ds.grads.cpu().numpy())
    return zl, g


@pytest.mark.parametrize("cin,cout,H,W,k,p,epi", [(64, 64, 20, 37, 3, 1, "bias"), (64, 128, 9, 16, 3, 1, "bias"),
                                                  (128, 256, 7, 7, 3, 1, "bias"), (256, 512, 5, 11, 3, 1, "bias"),
                                                  (64, 64, 13, 29, 1, 0, "bias"), (64, 192, 12, 40, 3, 0, "bias"),
                                                  (256, 128, 9, 23, 1, 0, "bias"), (512, 256, 6, 17, 1, 0, "bias"),
                                                  (64, 64, 20, 37, 3, 1, "affine"), (64, 64, 13, 29, 1, 0, "affine"),
                                                  (128, 256, 7, 19, 3, 1, "affine"), (256, 64, 9, 23, 1, 0, "affine"),
                                                  (64, 256, 13, 29, 1, 0, "affine"), (64, 256, 17, 40, 1, 0, "bias"),
                                                  (256, 64, 21, 37, 1, 0, "bias")])
def test_two_conv_layers_vs_oracle(cin, cout, H, W, k, p, epi):
    """conv(8->cin) then conv(cin->cout) [tcgen05 FP, dgrad into the first layer's delta, wgrad with
    the bias / beta and gamma gradients fused (dgamma = sum_{tap,ci} W * dW_raw)]; bands of 3 rows
    (2PS) and one band (column)."""
    net = {"C": 3, "H": H, "W": W, "classes": 10,
           "ops": [WL.conv(0, cin, 3, 1, 1), WL.conv(1, cout, k, 1, p, epi=epi), WL.conv(2, 64, 3, 1, 1)]}
    B = 2
    params = WL.make_params(net, seed=5, bias_scale=0.1, gamma_spread=0.3, bf16=True)
    x = WL.make_input(net, B, seed=3, bf16=True)
    ts, aux = C.forward(net, params, x, store=C.bf16_store)
    dzl = WL.make_dzl(ts[-1].shape, bf16=True)
    g_ref, _ = C.backward(net, params, ts, aux, dzl, need_dx=False)
    for mode, kw in (("column", {}), ("2ps", {"band_rows": 3}), ("overl", {"n_bands": 2})):
        zl, g = run(net, B, mode, params, x, dzl, flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION, **kw)
        assert rel(zl, ts[-1]) <= TOL, (mode, "zl", rel(zl, ts[-1]))
        for i in range(3):
            for key in g_ref[i]:
                e = rel(g[i][key], g_ref[i][key])
                assert e <= TOL, (mode, kw, i, key, e)


@pytest.mark.parametrize("cin,cout,H,W,k,s,p", [(64, 64, 21, 35, 3, 2, 1), (64, 128, 16, 18, 1, 2, 0),
                                                (8, 64, 37, 45, 7, 2, 3), (128, 64, 9, 30, 3, 2, 1),
                                                (64, 256, 11, 13, 3, 2, 0)])
def test_strided_layers_vs_oracle(cin, cout, H, W, k, s, p):
    """Strided convs on tcgen05: FP with TMA element strides, wgrad with a strided input box,
    dgrad as s x s parity classes of the flipped weights (stride-2 convs of ResNet-50:
    3x3/s2/p1, 1x1/s2 projection, 7x7/s2/p3 stem)."""
    net = {"C": 3, "H": H, "W": W, "classes": 10,
           "ops": [WL.conv(0, cin, 3, 1, 1), WL.conv(1, cout, k, s, p, epi="affine"), WL.conv(2, 64, 3, 1, 1)]}
    B = 2
    params = WL.make_params(net, seed=7, bias_scale=0.1, gamma_spread=0.2, bf16=True)
    x = WL.make_input(net, B, seed=4, bf16=True)
    ts, aux = C.forward(net, params, x, store=C.bf16_store)
    dzl = WL.make_dzl(ts[-1].shape, bf16=True)
    g_ref, _ = C.backward(net, params, ts, aux, dzl, need_dx=False)
    for mode, kw in (("column", {}), ("2ps", {"band_rows": 2}), ("overl", {"n_bands": 2})):
        zl, g = run(net, B, mode, params, x, dzl, flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION, **kw)
        assert rel(zl, ts[-1]) <= TOL, (mode, "zl", rel(zl, ts[-1]))
        for i in range(3):
            for key in g_ref[i]:
                e = rel(g[i][key], g_ref[i][key])
                assert e <= TOL, (mode, kw, i, key, e)


def test_tc_matches_simt():
    """Tensor-core and SIMT kernels on the same bf16 inputs (same storage rounding points).
    No max-pool: argmax near-ties would make the comparison ill-conditioned (R17c)."""
    net = {"C": 3, "H": 40, "W": 48, "classes": 10,
           "ops": [WL.conv(0, 64, 3, 1, 1), WL.conv(1, 128, 3, 1, 1), WL.conv(2, 64, 1, 1, 0),
                   WL.conv(3, 256, 3, 1, 1)]}
    B = 2
    params = WL.make_params(net, seed=2, bias_scale=0.05, bf16=True)
    x = WL.make_input(net, B, seed=0, bf16=True)
    ts, _ = C.forward(net, params, x, store=C.bf16_store)
    _, dzl, _, _ = C.head_forward_backward(ts[-1], params["head"], WL.make_labels(net, B))
    dzl = WL.round_bf16(dzl)
    zl_t, g_t = run(net, B, "2ps", params, x, dzl, n_bands=3)
    zl_s, g_s = run(net, B, "2ps", params, x, dzl, flags=LB.FLAG_NO_TCGEN05, n_bands=3)
    assert rel(zl_t, ts[-1]) <= TOL
    assert rel(zl_t, zl_s) <= TOL
    for a, b in zip(g_t, g_s):
        if b is not None:
            for key in b:
                assert rel(a[key], b[key]) <= TOL, key


@pytest.mark.parametrize("k,s,p,H,W,epi", [(3, 1, 1, 37, 45, "bias"), (7, 2, 3, 41, 53, "bias"), (3, 2, 1, 30, 34, "bias"),
                                          (5, 1, 2, 19, 70, "bias"), (7, 2, 3, 41, 53, "affine")])
def test_image_layer_vs_oracle(k, s, p, H, W, epi):
    """The RGB input layer (8 padded channels -> 64): FP through the tap-pair kernel (k_conv_pair,
    stride 1 and 2, descriptors straight into the TMA-loaded patch), wgrad through the patch-gather
    im2col kernel with the bias / beta (dedicated warps) and gamma (epilogue warp sums) gradients
    fused; several bands, ragged rows and columns."""
    net = {"C": 3, "H": H, "W": W, "classes": 10,
           "ops": [WL.conv(0, 64, k, s, p, epi=epi), WL.conv(1, 64, 3, 1, 1)]}
    B = 3
    params = WL.make_params(net, seed=11, bias_scale=0.1, bf16=True)
    x = WL.make_input(net, B, seed=6, bf16=True)
    ts, aux = C.forward(net, params, x, store=C.bf16_store)
    dzl = WL.make_dzl(ts[-1].shape, bf16=True)
    g_ref, _ = C.backward(net, params, ts, aux, dzl, need_dx=False)
    for mode, kw in (("column", {}), ("2ps", {"band_rows": 5}), ("overl", {"n_bands": 3})):
        zl, g = run(net, B, mode, params, x, dzl, flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION, **kw)
        assert rel(zl, ts[-1]) <= TOL, (mode, "zl", rel(zl, ts[-1]))
        for i in range(2):
            for key in g_ref[i]:
                e = rel(g[i][key], g_ref[i][key])
                assert e <= TOL, (mode, kw, i, key, e)

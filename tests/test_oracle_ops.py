"""Pins for the oracle's operators against things other than the oracle itself:
paper/SPEC worked examples, closed forms, textbook routines (numpy matmul),
finite differences and the adjoint identity.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle as O
from oracle import column as C
import workloads as WL

GOLD = os.path.join(os.path.dirname(__file__), "golden")
R = np.random.default_rng(1234)


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- worked examples
def test_conv_ramp_golden():
    g = gold("conv_ramp.json")
    x = np.array(g["x"], float)[None, None]
    y = O.conv2d_fwd(x, np.ones((1, 1, 3, 3)), None, 1, (0, 0, 0, 0))
    assert np.array_equal(y[0, 0], np.array(g["y"], float))


def test_fig3a_shape_and_feature_loss():
    g = gold("paper_examples.json")
    e = g["fig3a_shape"]
    y = O.conv2d_fwd(R.random((1, 1, 4, 4)), R.random((1, 1, 2, 2)), None, 1, (0, 0, 0, 0))
    assert y.shape[2:] == (e["H_out"], e["H_out"])
    # naive split into two 2-row parts loses a row: 2x3 instead of 3x3
    f = g["fig3a_feature_loss"]
    part = O.conv2d_fwd(R.random((1, 1, 2, 4)), R.random((1, 1, 2, 2)), None, 1, (0, 0, 0, 0))
    assert part.shape[2] == f["out_rows_each"]


def test_identity_1x1():
    x = R.random((2, 3, 5, 6))
    w = np.eye(3)[:, :, None, None]
    assert np.array_equal(O.conv2d_fwd(x, w, None, 1, (0, 0, 0, 0)), x)


def test_1x1_is_matmul():
    """1x1 conv == per-pixel matrix product (numpy @, a textbook routine)."""
    x = R.standard_normal((2, 5, 4, 3))
    w = R.standard_normal((7, 5, 1, 1))
    b = R.standard_normal(7)
    y = O.conv2d_fwd(x, w, b, 1, (0, 0, 0, 0))
    ref = np.einsum("oc,bchw->bohw", w[:, :, 0, 0], x) + b[None, :, None, None]
    ref2 = (w[:, :, 0, 0] @ x.transpose(1, 0, 2, 3).reshape(5, -1)).reshape(7, 2, 4, 3).transpose(1, 0, 2, 3)
    assert np.allclose(y, ref, rtol=1e-13, atol=1e-13)
    assert np.allclose(y - b[None, :, None, None], ref2, rtol=1e-13, atol=1e-13)
    dy = R.standard_normal(y.shape)
    dw, db = O.conv2d_bwd_weight(x, dy, 1, 1, (0, 0, 0, 0))
    dwm = dy.transpose(1, 0, 2, 3).reshape(7, -1) @ x.transpose(1, 0, 2, 3).reshape(5, -1).T
    assert np.allclose(dw[:, :, 0, 0], dwm, rtol=1e-12, atol=1e-12)
    assert np.allclose(db, dy.sum(axis=(0, 2, 3)), rtol=1e-12)
    dx = O.conv2d_bwd_data(w, dy, (4, 3), 1, (0, 0, 0, 0))
    dxm = (w[:, :, 0, 0].T @ dy.transpose(1, 0, 2, 3).reshape(7, -1)).reshape(5, 2, 4, 3).transpose(1, 0, 2, 3)
    assert np.allclose(dx, dxm, rtol=1e-12, atol=1e-12)


def test_constant_image_closed_form():
    """Constant image, p=0: every activation is constant per channel,
    v^l[co] = ReLU(sum_ci v^{l-1}[ci] * sum_{ky,kx} W[co,ci] + b[co])  (SURVEY 8(c) pin 1)."""
    net = {"C": 2, "H": 9, "W": 8, "classes": 3,
           "ops": [WL.conv(0, 3, 3, 1, 0), WL.conv(1, 4, 3, 1, 0), WL.conv(2, 2, 1, 1, 0)]}
    prm = WL.make_params(net, seed=5, bias_scale=0.3)
    v = np.array([0.7, -0.2])
    x = np.broadcast_to(v[None, :, None, None], (1, 2, 9, 8)).copy()
    ts, _ = C.forward(net, prm, x)
    for i, op in enumerate(net["ops"]):
        w = prm["convs"][i]["w"]
        v = np.maximum(w.sum(axis=(2, 3)) @ v + prm["convs"][i]["b"], 0.0)
        t = ts[i + 1]
        assert np.allclose(t, v[None, :, None, None], rtol=1e-13, atol=1e-14)


def test_constant_image_p1_edges():
    """p=1: interior pixels see the full kernel sum, a corner pixel only the 2x2 sub-kernel."""
    w = R.standard_normal((1, 1, 3, 3))
    x = np.full((1, 1, 6, 7), 2.0)
    y = O.conv2d_fwd(x, w, None, 1, (1, 1, 1, 1))
    assert np.isclose(y[0, 0, 3, 3], 2.0 * w.sum())
    assert np.isclose(y[0, 0, 0, 0], 2.0 * w[0, 0, 1:, 1:].sum())
    assert np.isclose(y[0, 0, 5, 6], 2.0 * w[0, 0, :2, :2].sum())


@pytest.mark.parametrize("s,p", [(1, 0), (1, 1), (2, 1), (2, 3)])
def test_one_hot_closed_form(s, p):
    """One-hot image e(c0,y0,x0): z[co,y,x] = W[co,c0,y0-(y s-p), x0-(x s-p)] (0 outside the kernel)."""
    k, H, W = 3 if p < 3 else 7, 11, 10
    w = R.standard_normal((4, 2, k, k))
    c0, y0, x0 = 1, 5, 4
    x = np.zeros((1, 2, H, W))
    x[0, c0, y0, x0] = 1.0
    y = O.conv2d_fwd(x, w, None, s, (p, p, p, p))
    ref = np.zeros_like(y)
    for yy in range(y.shape[2]):
        for xx in range(y.shape[3]):
            ky, kx = y0 - (yy * s - p), x0 - (xx * s - p)
            if 0 <= ky < k and 0 <= kx < k:
                ref[0, :, yy, xx] = w[:, c0, ky, kx]
    assert np.array_equal(y, ref)


def test_shape_law_exhaustive():
    """Shape law floor((H+pads-k)/s)+1, checked by executing the conv."""
    for H in range(1, 12):
        for k in range(1, 6):
            for s in range(1, 4):
                for pt in range(0, 3):
                    for pb in range(0, 3):
                        n = O.out_dim(H, pt, pb, k, s)
                        if H + pt + pb < k:
                            assert n < 1
                            continue
                        y = O.conv2d_fwd(np.ones((1, 1, H, 3)), np.ones((1, 1, k, k)), None, s, (pt, pb, 1, 1)) \
                            if k <= 5 else None
                        # brute force: count window starts inside the padded extent
                        starts = [y0 for y0 in range(0, H + pt + pb) if y0 % s == 0 and y0 + k <= H + pt + pb]
                        assert n == len(starts) == y.shape[2]


def test_adjoint_identity():
    """<conv(x), y> = <x, conv^T(y)> within 1e-10."""
    for s, p, k in [(1, 1, 3), (2, 1, 3), (2, 3, 7), (2, 0, 1), (1, 0, 2)]:
        x = R.standard_normal((2, 3, 13, 11))
        w = R.standard_normal((4, 3, k, k))
        y = O.conv2d_fwd(x, w, None, s, (p, p, p, p))
        v = R.standard_normal(y.shape)
        lhs = np.sum(y * v)
        rhs = np.sum(x * O.conv2d_bwd_data(w, v, (13, 11), s, (p, p, p, p)))
        assert abs(lhs - rhs) <= 1e-10 * max(1.0, abs(lhs))


def _fd(f, a, idx, h=1e-6):
    a2 = a.copy()
    a2[idx] += h
    fp = f(a2)
    a2[idx] -= 2 * h
    fm = f(a2)
    return (fp - fm) / (2 * h)


def test_conv_wgrad_finite_differences():
    """5x5 input, 3x3 kernel, s=2, p=1: grad_weights vs central FD <= 1e-6."""
    x = R.standard_normal((2, 2, 5, 5))
    w = R.standard_normal((3, 2, 3, 3))
    b = R.standard_normal(3)
    G = R.standard_normal((2, 3, 3, 3))
    loss = lambda ww: np.sum(G * O.conv2d_fwd(x, ww, b, 2, (1, 1, 1, 1)))
    dw, db = O.conv2d_bwd_weight(x, G, 3, 2, (1, 1, 1, 1))
    for idx in [(0, 0, 0, 0), (2, 1, 2, 1), (1, 0, 1, 2)]:
        assert abs(_fd(loss, w, idx) - dw[idx]) <= 1e-6 * max(1, abs(dw[idx]))
    lossb = lambda bb: np.sum(G * O.conv2d_fwd(x, w, bb, 2, (1, 1, 1, 1)))
    for i in range(3):
        assert abs(_fd(lossb, b, (i,)) - db[i]) <= 1e-6 * max(1, abs(db[i]))
    # delta = 0 -> zero grads
    dw0, db0 = O.conv2d_bwd_weight(x, np.zeros_like(G), 3, 2, (1, 1, 1, 1))
    assert not dw0.any() and not db0.any()


def test_conv_1x1_wgrad_is_sum():
    """1x1 conv with delta all ones -> grad_weight = sum of inputs."""
    x = R.random((3, 1, 4, 5))
    dw, _ = O.conv2d_bwd_weight(x, np.ones((3, 1, 4, 5)), 1, 1, (0, 0, 0, 0))
    assert np.isclose(dw[0, 0, 0, 0], x.sum())


def test_pool_examples():
    """[[1,2],[3,4]] max -> 4 (argmax 3); delta 7 routed to the argmax."""
    x = np.array([[1.0, 2.0], [3.0, 4.0]])[None, None]
    y, am = O.maxpool_fwd(x, 2, 2, (0, 0, 0, 0))
    assert y[0, 0, 0, 0] == 4.0 and am[0, 0, 0, 0] == 3
    dx = O.maxpool_bwd(am, np.array([[[[7.0]]]]), (2, 2))
    assert np.array_equal(dx[0, 0], np.array([[0, 0], [0, 7.0]]))


def test_pool_brute_force_and_ties():
    x = R.random((2, 3, 7, 6))
    y, am = O.maxpool_fwd(x, 3, 2, (1, 1, 1, 1))
    for b in range(2):
        for c in range(3):
            for oy in range(y.shape[2]):
                for ox in range(y.shape[3]):
                    win = [(x[b, c, iy, ix], iy * 6 + ix)
                           for iy in range(oy * 2 - 1, oy * 2 + 2) for ix in range(ox * 2 - 1, ox * 2 + 2)
                           if 0 <= iy < 7 and 0 <= ix < 6]
                    best = max(v for v, _ in win)
                    assert y[b, c, oy, ox] == best
                    assert am[b, c, oy, ox] == min(i for v, i in win if v == best)
    # ties -> lowest flat index
    y, am = O.maxpool_fwd(np.zeros((1, 1, 2, 2)), 2, 2, (0, 0, 0, 0))
    assert am[0, 0, 0, 0] == 0


def test_relu_examples_and_gate():
    """[-1,0,2] -> [0,0,2]; delta [5,5,5] -> [0,0,5] (ReLU'(0)=0)."""
    net = {"C": 1, "H": 1, "W": 3, "classes": 2, "ops": [WL.conv(0, 1, 1, 1, 0, epi="none")]}
    prm = {"convs": [{"w": np.ones((1, 1, 1, 1))}], "head": None}
    x = np.array([-1.0, 0.0, 2.0]).reshape(1, 1, 1, 3)
    ts, aux = C.forward(net, prm, x)
    assert np.array_equal(ts[1].ravel(), [0, 0, 2])
    _, dx = C.backward(net, prm, ts, aux, np.full((1, 1, 1, 3), 5.0))
    assert np.array_equal(dx.ravel(), [0, 0, 5])


def test_ce_equal_logits():
    """Equal logits, 10 classes -> loss = ln 10."""
    zl = np.ones((3, 4, 2, 2))
    head = {"fc_w": np.zeros((10, 4)), "fc_b": np.zeros(10)}
    loss, _, _, _ = C.head_forward_backward(zl, head, [0, 5, 9])
    assert abs(loss - np.log(10)) < 1e-15


def test_head_finite_differences():
    zl = R.standard_normal((3, 5, 2, 3))
    head = {"fc_w": R.standard_normal((4, 5)), "fc_b": R.standard_normal(4)}
    lab = [1, 3, 0]
    loss, dzl, g, _ = C.head_forward_backward(zl, head, lab)
    f = lambda z: C.head_forward_backward(z, head, lab)[0]
    for idx in [(0, 0, 0, 0), (2, 4, 1, 2), (1, 2, 0, 1)]:
        assert abs(_fd(f, zl, idx) - dzl[idx]) <= 1e-7 * max(1, abs(dzl[idx]))
    fw = lambda w: C.head_forward_backward(zl, {"fc_w": w, "fc_b": head["fc_b"]}, lab)[0]
    for idx in [(0, 0), (3, 4)]:
        assert abs(_fd(fw, head["fc_w"], idx) - g["fc_w"][idx]) <= 1e-7


def _whole_net_fd(net, prm, x, lab):
    """Every parameter of a small net vs central FD of the full loss (SURVEY 8(c) pin 4)."""
    def loss_of(p):
        ts, _ = C.forward(net, p, x)
        return C.head_forward_backward(ts[-1], p["head"], lab)[0]

    ts, aux = C.forward(net, prm, x)
    loss, dzl, hg, _ = C.head_forward_backward(ts[-1], prm["head"], lab)
    grads, _ = C.backward(net, prm, ts, aux, dzl)
    rr = np.random.default_rng(7)
    for i, g in enumerate(grads):
        if g is None:
            continue
        for key, gv in g.items():
            for _ in range(3):
                idx = tuple(rr.integers(0, n) for n in gv.shape)

                def f(v, key=key, i=i, idx=idx):
                    p2 = {"convs": [dict(c) if c is not None else None for c in prm["convs"]],
                          "head": prm["head"]}
                    arr = p2["convs"][i][key].copy()
                    arr[idx] = v
                    p2["convs"][i][key] = arr
                    return loss_of(p2)
                h = 1e-6
                v0 = prm["convs"][i][key][idx]
                fd = (f(v0 + h) - f(v0 - h)) / (2 * h)
                assert abs(fd - gv[idx]) <= 1e-6 * max(1e-3, abs(gv[idx])) + 1e-9, (i, key, idx, fd, gv[idx])


def test_whole_net_fd_chain():
    net = {"C": 2, "H": 8, "W": 7, "classes": 3,
           "ops": [WL.conv(0, 3, 3, 1, 1), WL.conv(1, 4, 3, 2, 1), WL.maxpool(2, 2, 2, 0),
                   WL.conv(3, 3, 1, 1, 0)]}
    prm = WL.make_params(net, seed=11, bias_scale=0.2)
    _whole_net_fd(net, prm, np.random.default_rng(3).standard_normal((2, 2, 8, 7)), [0, 2])


def test_whole_net_fd_residual_affine():
    """ResNet-style block: affine (frozen-BN) convs, projection shortcut, residual add + ReLU."""
    net = {"C": 2, "H": 9, "W": 6, "classes": 3,
           "ops": [WL.conv(0, 4, 3, 1, 1, epi="affine"),                 # t1
                   WL.conv(1, 3, 1, 1, 0, epi="affine"),                 # t2
                   WL.conv(2, 4, 3, 2, 1, epi="affine"),                 # t3
                   WL.conv(1, 4, 1, 2, 0, epi="affine", relu=False),     # t4 projection
                   WL.conv(3, 4, 1, 1, 0, epi="affine", res=4),          # t5 = relu(affine(conv t3) + t4)
                   WL.add(5, 3, relu=True),                              # t6 = relu(t5 + t3)
                   WL.maxpool(6, 3, 2, 1)]}
    prm = WL.make_params(net, seed=12, bias_scale=0.2, gamma_spread=0.3)
    _whole_net_fd(net, prm, np.random.default_rng(4).standard_normal((2, 2, 9, 6)), [1, 2])


def test_sgd_closed_forms():
    """lr=0 leaves theta unchanged; loss x2 doubles gradients."""
    net = WL.tiny3(p=1, H=8, W=8)
    prm = WL.make_params(net, seed=2, bias_scale=0.1)
    x = WL.make_input(net, 2)
    lab = WL.make_labels(net, 2)
    new, loss, grads, hg, _ = C.step(net, prm, x, lab, 0.0)
    for a, b in zip(new["convs"], prm["convs"]):
        for k in a:
            assert np.array_equal(a[k], b[k])
    ts, aux = C.forward(net, prm, x)
    g1, _ = C.backward(net, prm, ts, aux, WL.make_dzl(ts[-1].shape))
    g2, _ = C.backward(net, prm, ts, aux, 2 * WL.make_dzl(ts[-1].shape))
    for a, b in zip(g1, g2):
        for k in a:
            assert np.allclose(2 * a[k], b[k], rtol=1e-14, atol=0)
    lr = 0.1
    new, _, grads, hg, _ = C.step(net, prm, x, lab, lr)
    assert np.allclose(new["convs"][0]["w"], prm["convs"][0]["w"] - lr * grads[0]["w"], rtol=0, atol=0)


def test_bf16_store_matches_torch():
    """The oracle's bf16 storage model equals PyTorch's float32->bfloat16 RNE conversion (library routine)."""
    torch = pytest.importorskip("torch")
    a = np.concatenate([R.standard_normal(5000) * 10.0 ** R.integers(-6, 6, 5000),
                        [0.0, -0.0, 1.0, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -9, 65504.0]])
    ref = torch.from_numpy(a.astype(np.float32)).to(torch.bfloat16).to(torch.float64).numpy()
    assert np.array_equal(C.bf16_store(a), ref)
    assert np.array_equal(WL.round_bf16(a), ref)

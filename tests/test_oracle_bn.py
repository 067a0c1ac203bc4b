"""Pins for the oracle's training-mode BatchNorm (reading R24).

The bn op is pinned against things other than itself:
  * a library routine: torch.nn.functional.batch_norm(training=True) in fp64 with autograd
    (conv -> batch_norm -> +residual -> ReLU), every activation and every gradient;
  * closed forms: the normalised output has per-channel mean beta and variance
    gamma^2 var/(var+eps); a channel whose input is constant maps to beta;
  * adjoint invariants of the batch-statistics Jacobian: sum(dc) = 0 and
    sum(dc*xh) = gamma/sigma * dgamma * eps/(var+eps) per channel (a dropped term breaks one);
  * central finite differences of the whole step's loss;
  * the method's invariant: the row-centric executor with statistics / sums sweeps equals the column
    oracle in fp64 for any band count and segmentation, in 2PS and OverL (overlapping bands: each row
    counted once, the statistics terms of the backward added once), and the per-band-statistics
    negative control does not.
CPU only."""
import numpy as np
import pytest
import torch

import workloads as WL
from oracle import column as C
from oracle import rowcentric as RC


def _net(res_every=2, n=4, H=12, W=5, Cin=2, ch=4, seg=None):
    net = WL.bn_chain(H=H, W=W, C=Cin, ch=ch, n=n, res_every=res_every)
    if seg is not None:
        net["ops"][seg]["seg_end"] = True
    return net


def _torch_forward(net, prm, x):
    """The same net through torch's conv2d + batch_norm(training=True) (a library routine)."""
    ts = [torch.tensor(x, dtype=torch.float64)]
    leaves = []
    for i, op in enumerate(net["ops"]):
        src = ts[op["src"]]
        if op["kind"] == "conv":
            w = torch.tensor(prm["convs"][i]["w"], requires_grad=True)
            leaves.append((i, "w", w))
            t = torch.nn.functional.conv2d(src, w, None, op["s"], op["p"])
        else:
            g = torch.tensor(prm["convs"][i]["gamma"], requires_grad=True)
            b = torch.tensor(prm["convs"][i]["beta"], requires_grad=True)
            leaves += [(i, "gamma", g), (i, "beta", b)]
            t = torch.nn.functional.batch_norm(src, None, None, g, b, training=True, eps=1e-5)
            if op["res"] >= 0:
                t = t + ts[op["res"]]
            if op["relu"]:
                t = torch.relu(t)
        ts.append(t)
    return ts, leaves


def test_bn_matches_torch_batch_norm():
    net = _net()
    B = 3
    x = WL.make_input(net, B)
    prm = WL.make_params(net, bias_scale=0.4, gamma_spread=0.5)
    ts, aux = C.forward(net, prm, x)
    G = WL.make_dzl(ts[-1].shape)
    grads, dx = C.backward(net, prm, ts, aux, G)
    tts, leaves = _torch_forward(net, prm, x)
    for a, b in zip(ts, tts):
        np.testing.assert_allclose(a, b.detach().numpy(), rtol=1e-12, atol=1e-12)
    (tts[-1] * torch.tensor(G)).sum().backward()
    for i, k, leaf in leaves:
        np.testing.assert_allclose(grads[i][k], leaf.grad.numpy(), rtol=1e-10, atol=1e-12)


def test_bn_closed_forms():
    rng = np.random.default_rng(5)
    c = rng.normal(2.0, 3.0, size=(4, 3, 5, 6))
    c[:, 2] = 1.25                                   # a constant channel
    prm = {"gamma": np.array([0.5, -2.0, 3.0]), "beta": np.array([0.1, -0.7, 0.3])}
    mean, var = C.bn_stats(c)
    y = C.bn_apply(prm, c, mean, var, None, False)
    np.testing.assert_allclose(y.mean(axis=(0, 2, 3)), prm["beta"], atol=1e-12)
    np.testing.assert_allclose(y.var(axis=(0, 2, 3)), prm["gamma"] ** 2 * var / (var + C.BN_EPS), rtol=1e-12,
                               atol=1e-20)
    np.testing.assert_allclose(y[:, 2], prm["beta"][2], atol=1e-12)   # constant input -> beta
    # textbook statistics: mean and biased variance
    np.testing.assert_allclose(mean, c.reshape(4, 3, -1).transpose(1, 0, 2).reshape(3, -1).mean(1), rtol=1e-13)
    np.testing.assert_allclose(var, c.reshape(4, 3, -1).transpose(1, 0, 2).reshape(3, -1).var(1), rtol=1e-12)


def test_bn_adjoint_invariants():
    rng = np.random.default_rng(6)
    c = rng.normal(size=(2, 4, 6, 5))
    prm = {"gamma": rng.uniform(0.5, 1.5, 4), "beta": rng.uniform(-0.5, 0.5, 4)}
    mean, var = C.bn_stats(c)
    t = C.bn_apply(prm, c, mean, var, None, True)
    dt = rng.normal(size=c.shape)
    dc, da, g = C.bn_bwd_full(prm, c, t, dt, mean, var, True, 2 * 6 * 5)
    xh = (c - mean[None, :, None, None]) / np.sqrt(var + C.BN_EPS)[None, :, None, None]
    np.testing.assert_allclose(dc.sum(axis=(0, 2, 3)), 0.0, atol=1e-12)
    # sum(dc*xh) = gamma/sigma * dgamma * (1 - sum(xh^2)/M) = gamma/sigma * dgamma * eps/(var+eps)
    # (0 for eps = 0): the xh*dgamma/M term is what cancels the dgamma direction
    sig = np.sqrt(var + C.BN_EPS)
    np.testing.assert_allclose((dc * xh).sum(axis=(0, 2, 3)),
                               prm["gamma"] / sig * g["gamma"] * C.BN_EPS / (var + C.BN_EPS), rtol=1e-8, atol=1e-14)
    # the gated delta flows into beta unchanged and into gamma through xh
    np.testing.assert_allclose(g["beta"], (dt * (t > 0)).sum(axis=(0, 2, 3)), rtol=1e-13)


def test_bn_step_finite_differences():
    net = _net(n=2, res_every=2, H=6, W=4, ch=3)
    B = 2
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    prm = WL.make_params(net, bias_scale=0.3, gamma_spread=0.4)

    def loss_of(p):
        ts, _ = C.forward(net, p, x)
        return C.head_forward_backward(ts[-1], p["head"], lab)[0]

    _, _, grads, _, _ = C.step(net, prm, x, lab, 0.0)
    h = 1e-6
    rng = np.random.default_rng(7)
    for i, k in [(0, "w"), (1, "gamma"), (1, "beta"), (2, "w"), (3, "gamma"), (3, "beta")]:
        arr = prm["convs"][i][k]
        for _ in range(3):
            idx = tuple(rng.integers(0, n) for n in arr.shape)
            old = arr[idx]
            arr[idx] = old + h
            lp = loss_of(prm)
            arr[idx] = old - h
            lm = loss_of(prm)
            arr[idx] = old
            fd = (lp - lm) / (2 * h)
            assert abs(fd - grads[i][k][idx]) <= 1e-6 * max(1.0, abs(fd)), (i, k, idx, fd, grads[i][k][idx])


@pytest.mark.parametrize("mode", ["2ps", "overl"])
@pytest.mark.parametrize("n_bands,seg", [(1, None), (2, None), (3, 3), (5, 1), (12, 3)])
def test_rowcentric_bn_equals_column(n_bands, seg, mode):
    net = _net(n=4, res_every=2, H=12, seg=seg)
    B = 2
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    prm = WL.make_params(net, bias_scale=0.3, gamma_spread=0.3)
    _, loss0, g0, hg0, ts = C.step(net, prm, x, lab, 0.1)
    plan = RC.Plan(net, mode, n_bands=n_bands)
    _, loss1, g1, hg1, zl = RC.step(plan, prm, x, lab, 0.1)
    assert abs(loss1 - loss0) <= 1e-12 * abs(loss0)
    np.testing.assert_allclose(zl, ts[-1], rtol=0, atol=1e-12)
    for i, g in enumerate(g0):
        if g is None:
            continue
        for k in g:
            np.testing.assert_allclose(g1[i][k], g[k], rtol=1e-10, atol=1e-12 * np.abs(g[k]).max())


@pytest.mark.parametrize("mode", ["2ps", "overl"])
def test_rowcentric_bn_resnet_blocks(mode):
    net = WL.resnet50(H=40, W=16, width_div=16, blocks=(2, 1, 1, 1), bn_train=True, segments="p3")
    B = 2
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    prm = WL.make_params(net, bias_scale=0.2, gamma_spread=0.3)
    _, loss0, g0, _, ts = C.step(net, prm, x, lab, 0.1)
    plan = RC.Plan(net, mode, n_bands=3)
    _, loss1, g1, _, zl = RC.step(plan, prm, x, lab, 0.1)
    assert abs(loss1 - loss0) <= 1e-11 * abs(loss0)
    for i, g in enumerate(g0):
        if g is None:
            continue
        for k in g:
            np.testing.assert_allclose(g1[i][k], g[k], rtol=1e-9, atol=1e-11 * np.abs(g[k]).max())


def test_per_band_statistics_is_not_batch_norm():
    """Negative control: normalising each band by its own rows' statistics changes z^L."""
    net = _net(n=3, res_every=0, H=12)
    x = WL.make_input(net, 2)
    prm = WL.make_params(net, bias_scale=0.3, gamma_spread=0.3)
    ts, _ = C.forward(net, prm, x)
    plan = RC.Plan(net, "2ps", n_bands=3)
    zl, _, _ = RC.forward(plan, prm, x, per_band_stats=True)
    assert np.abs(zl - ts[-1]).max() > 1e-2 * np.abs(ts[-1]).max()


@pytest.mark.parametrize("world", [2, 3])
def test_zr_ranks_bn_equal_column(world):
    """The oracle's zero-redundancy G-rank executor with training-mode BN: every statistics / sums sweep
    is a whole sharded sweep and the per-rank sums over the rows each rank computes are added over the
    ranks (the all-reduce of the CUDA path): loss and every gradient equal the column oracle (fp64)."""
    net = WL.resnet50(H=96, W=16, width_div=16, blocks=(2, 1, 1, 1), bn_train=True)
    B = 2
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    prm = WL.make_params(net, bias_scale=0.2, gamma_spread=0.3)
    _, loss0, g0, _, _ = C.step(net, prm, x, lab, 0.1)
    _, loss1, g1, _, _, log = RC.step_ranks_zr(net, prm, x, lab, 0.1, world, n_bands=2)
    assert abs(loss1 - loss0) <= 1e-12 * abs(loss0)
    for i, g in enumerate(g0):
        if g is None:
            continue
        for k in g:
            np.testing.assert_allclose(g1[i][k], g[k], rtol=1e-9, atol=1e-11 * np.abs(g[k]).max())

"""GPU parity: the CUDA path (through the C-ABI) against the fp64 oracle, element by
element on the same seeded inputs.  Tolerances (north_star, R18):
rel(T) = max|T_gpu - T_ref| / max|T_ref| per tensor; fp32 mode <= 1e-5, bf16 <= 2e-2.
For bf16 the oracle is fed the same bf16-rounded x, theta and delta^L (R17) and
stores its fp64 feature maps rounded to bf16 (R17b: ReLU masks and max-pool
argmax are integer decisions both sides take in the kernel's storage precision)."""
import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from conditioned import validate_forward, conditioned_grads, compare_grads
from gpu_util import run_capture

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402

TOL = {"fp32": 1e-5, "bf16": 2e-2}


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def run_gpu(net, B, mode, prec, params, x, dzl=None, labels=None, lr=None, flags=0, **kw):
    plan = LB.Plan(net, B, mode=mode, prec=prec, flags=flags, **kw)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, dzl=dzl, labels=labels)
    if lr is None:
        ds.forward()
        zl = plan.from_nhwc(ds.zl.float().cpu().numpy(), len(net["ops"]))
        ds.backward()
        torch.cuda.synchronize()
        grads, head = plan.unpack_grads(ds.grads.cpu().numpy())
        return plan, zl, grads
    ds.step(lr)
    torch.cuda.synchronize()
    return plan, ds


def oracle_fb(net, params, x, dzl, store=None):
    ts, aux = C.forward(net, params, x, store=store)
    grads, _ = C.backward(net, params, ts, aux, dzl, need_dx=False)
    return ts[-1], grads


def check(net, B, prec, modes, kws, seed=0, bias=0.2, gspread=0.2, flags=0, dzl_kind="random", plain_grads=False):
    """z^L vs the plain oracle; every stored map validated op by op and every gradient vs the oracle's
    backward conditioned on the validated maps (tests/conditioned.py, R17d) -- one seeded
    draw, no re-drawing of inputs.  plain_grads: also compare the gradients with the plain oracle
    (nets without max-pool near-ties: the C1 chain)."""
    bf = prec == "bf16"
    store = C.bf16_store if bf else C.fp32_store
    params = WL.make_params(net, seed=2 + seed, bias_scale=bias, gamma_spread=gspread, bf16=bf)
    x = WL.make_input(net, B, seed=seed, bf16=bf)
    ts, aux = C.forward(net, params, x, store=store)
    shp = C.out_hw(net)
    c, h, w = shp[-1]
    if dzl_kind == "random":
        dzl = WL.make_dzl((B, c, h, w), bf16=bf)           # C1's loss sum(G * z^L)
    else:                                                   # the training workload: CE head
        lab = WL.make_labels(net, B)
        _, dzl, _, _ = C.head_forward_backward(ts[-1], params["head"], lab)
        dzl = WL.round_bf16(dzl) if bf else dzl
    g_plain = C.backward(net, params, ts, aux, dzl, need_dx=False)[0] if plain_grads else None
    for mode in modes:
        for kw in (kws if mode != "column" else [{}]):
            _, zl, g, tsg = run_capture(net, B, prec, mode, params, x, dzl, flags=flags, **kw)
            assert rel(zl, ts[-1]) <= TOL[prec], (mode, kw, "zL", rel(zl, ts[-1]))
            _, aux_g = validate_forward(net, params, tsg, store, TOL[prec])
            compare_grads(g, conditioned_grads(net, params, tsg, aux_g, dzl), TOL[prec], (mode, str(kw)))
            if g_plain is not None:
                compare_grads(g, g_plain, TOL[prec], (mode, str(kw), "plain"))


# ------------------------------------------------------------------ C1 (BASELINE configs[0]) fp32
@pytest.mark.parametrize("p", [1, 0])
def test_c1_fp32_all_modes(p):
    """tiny 3-conv net, 32x32x1, batch 1, row band 4: fp32 FP+BP vs the oracle <= 1e-5."""
    check(WL.tiny3(p=p), 1, "fp32", ["column", "2ps", "overl"], [{"band_rows": 4}],
          flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION, plain_grads=True)


def test_c1_fp32_band_edge_cases():
    """Band height 1 (31 interior cuts, empty intermediate ranges), ragged tails, N=1."""
    net = WL.tiny3(p=1, H=23, W=13)
    check(net, 2, "fp32", ["2ps", "overl"], [{"band_rows": 1}, {"band_rows": 5}, {"n_bands": 1}, {"n_bands": 3}],
          flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION, plain_grads=True)


def test_c1_bf16():
    check(WL.tiny3(p=1), 2, "bf16", ["column", "2ps", "overl"], [{"band_rows": 4}],
          flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)


def test_dag_fp32_and_bf16():
    """ResNet-style DAG: 7x7/s2 stem, 3x3/s2/p1 max-pool, affine convs, projection and identity
    shortcuts, checkpoint segments."""
    net = {"C": 3, "H": 37, "W": 21, "classes": 4,
           "ops": [WL.conv(0, 8, 7, 2, 3, epi="affine"), WL.maxpool(1, 3, 2, 1),
                   WL.conv(2, 8, 1, 1, 0, epi="affine"), WL.conv(3, 8, 3, 1, 1, epi="affine"),
                   WL.conv(4, 16, 1, 1, 0, epi="affine", relu=False),
                   WL.conv(2, 16, 1, 1, 0, epi="affine", relu=False),
                   WL.add(5, 6, relu=True, seg_end=True),
                   WL.conv(7, 8, 1, 1, 0, epi="affine"), WL.conv(8, 8, 3, 2, 1, epi="affine"),
                   WL.conv(7, 16, 1, 2, 0, epi="affine", relu=False),
                   WL.conv(9, 16, 1, 1, 0, epi="affine", res=10)]}
    for prec in ("fp32", "bf16"):
        check(net, 2, prec, ["column", "2ps", "overl"], [{"band_rows": 2}, {"n_bands": 3}],
              flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)


def test_resnet50_reduced():
    """ResNet-50 v1.5 topology (stem 7x7/s2, max-pool 3x3/s2/p1, bottlenecks with stride-2 3x3,
    projection shortcuts, fused residual add), one block per stage, reduced width, per-stage
    checkpoint segments: fp32 (1e-5) and bf16 (2e-2, training-workload delta^L) vs the oracle."""
    net = WL.resnet50(H=64, W=48, width_div=8, blocks=(1, 1, 1, 1))
    check(net, 2, "fp32", ["column", "2ps", "overl"], [{"n_bands": 3}, {"band_rows": 1}], bias=0.1,
          gspread=0.2, flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)
    check(net, 2, "bf16", ["column", "2ps", "overl"], [{"n_bands": 3}], bias=0.1, gspread=0.2,
          flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION, dzl_kind="head")


def test_resnet_identity_blocks_fused_residual():
    """Identity bottlenecks whose block input has 64 / 128 channels: the tensor-core dgrad of conv1
    takes the block output's delta as a TMA-loaded addend (fused residual gradient)
    and the 2PS cache row of the block input is written by the residual row kernel.  The unfused
    path (memset + accumulating dgrad + residual pass, LRCNN_FLAG_NO_FUSE_RES) is the one the
    oracle tests above pin; here the fused gradients must equal it up to the one bf16 rounding of
    delta it saves (same forward, same integer decisions), for COLUMN and 2PS (3 bands, 1-row
    bands), and z^L must match the oracle."""
    net = WL.resnet50(H=48, W=40, width_div=4, blocks=(3, 2, 1, 1))
    B = 2
    params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=True)
    x = WL.make_input(net, B, seed=0, bf16=True)
    ts, _ = C.forward(net, params, x, store=C.bf16_store)
    _, dzl, _, _ = C.head_forward_backward(ts[-1], params["head"], WL.make_labels(net, B))
    dzl = WL.round_bf16(dzl)
    for mode, kw in (("column", {}), ("2ps", {"n_bands": 3}), ("2ps", {"band_rows": 1})):
        _, zl, g_f = run_gpu(net, B, mode, "bf16", params, x, dzl, **kw)
        _, _, g_u = run_gpu(net, B, mode, "bf16", params, x, dzl, flags=LB.FLAG_NO_FUSE_RES, **kw)
        assert rel(zl, ts[-1]) <= TOL["bf16"], (mode, kw, "zL")
        for i, (a, b) in enumerate(zip(g_f, g_u)):
            if b is None:
                continue
            for k in b:
                assert rel(a[k], b[k]) <= 1e-2, (mode, kw, "op", i, k, rel(a[k], b[k]))


def test_vgg_reduced_fp32():
    """VGG-16 topology (13 conv + 5 pool), reduced channels/size, fp32: every mode <= 1e-5."""
    net = WL.vgg16(H=64, W=64, width_div=8)
    check(net, 2, "fp32", ["column", "2ps"], [{"n_bands": 3}, {"band_rows": 1}], bias=0.05, gspread=0.0)
    net = WL.vgg16(H=64, W=64, width_div=8, segments="pool")
    check(net, 2, "fp32", ["2ps", "overl"], [{"n_bands": 2}], bias=0.05, gspread=0.0,
          flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)


def test_vgg_reduced_bf16():
    """VGG-16's first two blocks (4 conv + 2 pool), reduced channels, bf16, head delta^L: COLUMN,
    2PS (4 bands, 1-row bands) vs the oracle (the full 13-conv stack: test_gpu_conditioned)."""
    net = WL.vgg16(H=64, W=64, width_div=4, cfg=[64, 64, "M", 128, 128, "M"])
    check(net, 2, "bf16", ["column", "2ps"], [{"n_bands": 4}, {"band_rows": 1}], bias=0.05, gspread=0.0,
          dzl_kind="head", flags=LB.FLAG_REQUIRE_TC)


def test_step_matches_oracle_fp32():
    """lrcnn_step (FP, head, BP, SGD) vs the oracle's step: loss and updated parameters."""
    net = WL.tiny3(p=1, H=16, W=16)
    B = 3
    params = WL.make_params(net, seed=2, bias_scale=0.1)
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    lr = 0.05
    new_ref, loss_ref, g_ref, hg_ref, _ = C.step(net, params, x, lab, lr)
    for mode, kw in (("column", {}), ("2ps", {"band_rows": 3}), ("overl", {"n_bands": 2})):
        plan, ds = run_gpu(net, B, mode, "fp32", params, x, labels=lab, lr=lr,
                           flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION, **kw)
        loss = float(ds.loss.cpu())
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
        got, head = plan.unpack_grads(ds.master.cpu().numpy())
        assert np.all(ds.grads.cpu().numpy() == 0)          # g = 0 after the update
        for i, (a, b) in enumerate(zip(got, new_ref["convs"])):
            if b is None:
                continue
            for k in b:
                # compare the update lr*g: theta_new - theta_old
                d_ref = params["convs"][i][k] - b[k]
                d_got = params["convs"][i][k] - a[k]
                assert rel(d_got, d_ref) <= 1e-4, (mode, i, k)
        for k in ("fc_w", "fc_b"):
            d_ref = params["head"][k] - new_ref["head"][k]
            d_got = params["head"][k] - head[k]
            assert rel(d_got, d_ref) <= 1e-4


def test_state_and_workspace_errors():
    net = WL.tiny3(p=1, H=8, W=8)
    plan = LB.Plan(net, 1, mode="2ps", prec="fp32", band_rows=2)
    ds = LB.DeviceState(plan)
    with pytest.raises(LB.LrcnnError) as e:
        ds.backward()
    assert e.value.name == "E_STATE"
    import ctypes
    st = LB.lib().lrcnn_forward_rows(plan.h, LB._ptr(ds.params), LB._ptr(ds.x), LB._ptr(ds.zl), LB._ptr(ds.ws),
                                     16, LB._stream(None))
    assert LB.STATUS[st] == "E_WORKSPACE"
    st = LB.lib().lrcnn_forward_rows(plan.h, LB._ptr(ds.params), LB._ptr(ds.x), LB._ptr(ds.zl), None,
                                     plan.ws_bytes, LB._stream(None))
    assert LB.STATUS[st] == "E_WORKSPACE"
    del ctypes


def test_step_graph_replay_matches_eager():
    """lrcnn_step captured into a CUDA graph (non-default stream) == eager steps on the default stream."""
    net = WL.vgg16(H=32, W=32, width_div=4, cfg=[64, 64, "M", 128, "M"])
    B = 2
    params = WL.make_params(net, seed=2, bias_scale=0.05)
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    out = []
    for use_stream in (False, True):
        plan = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=3)
        ds = LB.DeviceState(plan)
        ds.load(params=params, x=x, labels=lab)
        st = torch.cuda.Stream() if use_stream else None
        losses = []
        for _ in range(5):
            if st is None:
                ds.step(0.05)
            else:
                with torch.cuda.stream(st):
                    ds.step(0.05, stream=st)
            torch.cuda.synchronize()
            losses.append(float(ds.loss.cpu()))
        out.append((losses, ds.master.cpu().numpy()))
    assert np.allclose(out[0][0], out[1][0], rtol=1e-5)
    assert rel(out[1][1], out[0][1]) <= 1e-4


def test_step_grads_graph_replay_matches_step():
    """lrcnn_step_grads (graph-replayed from its third call on a non-default stream; the data-parallel
    path: caller all-reduce in between) followed by lrcnn_sgd == lrcnn_step, over 5 steps."""
    net = WL.vgg16(H=32, W=32, width_div=4, cfg=[64, 64, "M", 128, "M"])
    B = 2
    params = WL.make_params(net, seed=2, bias_scale=0.05)
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    out = []
    for split in (False, True):
        plan = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=3)
        ds = LB.DeviceState(plan)
        ds.load(params=params, x=x, labels=lab)
        st = torch.cuda.Stream()
        losses = []
        with torch.cuda.stream(st):
            for _ in range(5):
                if split:
                    ds.step_grads(stream=st)
                    plan.sgd(ds.master, ds.params, ds.grads, 0.05, st)
                else:
                    ds.step(0.05, stream=st)
                torch.cuda.synchronize()
                losses.append(float(ds.loss.cpu()))
        out.append((losses, ds.master.cpu().numpy()))
    assert np.allclose(out[0][0], out[1][0], rtol=1e-5)
    assert rel(out[1][1], out[0][1]) <= 1e-4


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_fp_merge_identical(prec):
    """Decoupled FP bands (LRCNN_FLAG_FP_MERGE, N_FP < N_BP): the forward runs merged bands and
    saves the halo rows of every BP boundary; same kernels and per-pixel accumulation order, so
    z^L equals the unmerged run bit for bit and every gradient up to the order of its fp32
    atomic reductions (1e-5); fp32 z^L also vs the oracle (1e-5)."""
    for net, kw in ((WL.vgg16(H=64, W=48, width_div=8, segments="pool"), {"n_bands": 4}),
                    (WL.resnet50(H=64, W=48, width_div=4, blocks=(2, 2, 1, 1)), {"n_bands": 6})):
        bf = prec == "bf16"
        params = WL.make_params(net, seed=2, bias_scale=0.05, bf16=bf)
        x = WL.make_input(net, 2, seed=0, bf16=bf)
        ts, _ = C.forward(net, params, x, store=C.bf16_store if bf else C.fp32_store)
        dzl = WL.make_dzl(ts[-1].shape, bf16=bf)
        p0, zl0, g0 = run_gpu(net, 2, "2ps", prec, params, x, dzl, **kw)
        p1, zl1, g1 = run_gpu(net, 2, "2ps", prec, params, x, dzl, flags=LB.FLAG_FP_MERGE, **kw)
        assert any(p1.fp_bands(s)[0] < p1.fp_bands(s)[1] for s in range(p1.nsegs()))
        assert np.array_equal(zl0, zl1)
        for a, b in zip(g0, g1):   # gradients: fp32 atomic reductions, order not fixed
            if b is not None:
                for k in b:
                    assert rel(a[k], b[k]) <= 1e-5, (k, rel(a[k], b[k]))
        if not bf:
            assert rel(zl1, ts[-1]) <= TOL["fp32"]

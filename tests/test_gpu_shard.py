"""GPU parity of row sharding across ranks: G ranks share one GPU through the
in-process loopback communicator (one host thread and one stream per rank, the same halo
exchange / all-reduce schedule the NCCL backend runs over NVLink).  Every rank's gradients
after the all-reduce and its loss must equal the unsharded oracle step (fp32 <= 1e-5); bf16
is compared with the GPU's own single-rank run (R17c)."""
import threading

import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from conditioned import rel, validate_forward, conditioned_grads, compare_grads
from gpu_util import _nchw

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402


def run_sharded(net, B, prec, world, params, x, lab, capture=False, flags=0, **kw):
    """One lrcnn_step_grads per rank (loopback communicator, one host thread + stream per rank).
    capture: every rank records the rows it computes of every map (lrcnn_debug_capture into a
    NaN-filled full-height buffer); the merged maps (ranks compute identical values on overlapping
    rows) are returned for the oracle checks.  Returns ([(loss, (grads, head))] per rank, ts)."""
    comms = LB.Comm.loopback(world)
    plans, states, bufs = [], [], []
    L = len(net["ops"])
    for g in range(world):
        p = LB.Plan(net, B, mode="2ps", prec=prec, world=world, rank=g, flags=flags, **kw)
        p.set_comm(comms[g])
        ds = LB.DeviceState(p)
        ds.load(params=params, x=x, labels=lab)
        plans.append(p)
        states.append(ds)
        if capture:
            b = {}
            for t in range(1, L + 1):
                c, cp, h, w = p.tensor(t)
                b[t] = torch.full((B, h, w, cp), float("nan"), dtype=ds.dtype, device=ds.x.device)
                p.debug_capture(t, b[t])
            bufs.append(b)
    torch.cuda.synchronize()
    errs = [None] * world

    def body(g):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                states[g].step_grads(stream=st)
            st.synchronize()
        except Exception as e:   # surfaced below
            errs[g] = e

    th = [threading.Thread(target=body, args=(g,)) for g in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert all(e is None for e in errs), errs
    out = []
    for p, ds in zip(plans, states):
        out.append((float(ds.loss.cpu()), p.unpack_grads(ds.grads.cpu().numpy())))
    ts = None
    if capture:
        ts = [np.asarray(x, dtype=np.float64)]
        for t in range(1, L + 1):
            m = bufs[0][t].clone()
            for g in range(1, world):
                m = torch.where(torch.isnan(m), bufs[g][t], m)
            c = plans[0].tensor(t)[0]
            ts.append(_nchw(m, c, list(range(B))))
            assert not np.isnan(ts[-1]).any(), ("rows no rank computed", t)
        for g, p in enumerate(plans):
            for t in range(1, L + 1):
                p.debug_capture(t, None)
    for c in comms:
        c.free()
    return out, ts


def oracle_ref(net, B, seed, bias, bf16=False):
    params = WL.make_params(net, seed=seed, bias_scale=bias, bf16=bf16)
    x = WL.make_input(net, B, seed=seed, bf16=bf16)
    lab = WL.make_labels(net, B)
    _, loss, g, hg, _ = C.step(net, params, x, lab, 0.0)
    return params, x, lab, loss, g, hg


def check_conditioned(net, params, ts, lab, res, prec):
    """Every merged map validated against the oracle op by op; then the head and the backward on the
    validated maps (R17d) vs every rank's loss and all-reduced gradients."""
    store = C.bf16_store if prec == "bf16" else C.fp32_store
    tol = 2e-2 if prec == "bf16" else 1e-5
    _, aux = validate_forward(net, params, ts, store, tol)
    loss_c, dzl, hg, _ = C.head_forward_backward(ts[-1], params["head"], lab)
    g_ref = conditioned_grads(net, params, ts, aux, dzl)
    for rank, (loss, (g, head)) in enumerate(res):
        assert abs(loss - loss_c) <= tol * abs(loss_c), (rank, loss, loss_c)
        compare_grads(g, g_ref, tol, ("rank", rank))
        for k in ("fc_w", "fc_b"):
            assert rel(head[k], hg[k]) <= tol, (rank, k)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_resnet_fp32(world):
    """fp32, world 2 / 3: loss and all-reduced gradients of every rank vs the plain oracle step and
    vs the oracle conditioned on the merged maps; two identity blocks in stage 2."""
    net = WL.resnet50(H=96, W=32, width_div=8, blocks=(2, 1, 1, 1))
    B = 2
    params, x, lab, loss_ref, g_ref, hg_ref = oracle_ref(net, B, 5, 0.1)
    res, ts = run_sharded(net, B, "fp32", world, params, x, lab, capture=True, n_bands=2)
    for rank, (loss, (g, head)) in enumerate(res):
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref), (rank, loss, loss_ref)
    check_conditioned(net, params, ts, lab, res, "fp32")


def test_sharded_vgg_fp32_pool_segments():
    net = WL.vgg16(H=64, W=32, width_div=8, segments="pool")
    B = 2
    params, x, lab, loss_ref, g_ref, hg_ref = oracle_ref(net, B, 9, 0.05)
    res, ts = run_sharded(net, B, "fp32", 2, params, x, lab, capture=True, n_bands=2)
    for rank, (loss, (g, head)) in enumerate(res):
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
    check_conditioned(net, params, ts, lab, res, "fp32")


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_resnet_bf16_vs_oracle(world):
    """bf16 tensor-core path, row-sharded over 2 / 4 ranks with NCCL-schedule halo exchange
    (loopback): loss vs the plain oracle, every rank's gradients vs the oracle conditioned on the
    merged maps (R17d)."""
    net = WL.resnet50(H=128, W=64, width_div=4, blocks=(2, 1, 1, 1))
    B = 2
    params, x, lab, loss_ref, _, _ = oracle_ref(net, B, 3, 0.1, bf16=True)
    res, ts = run_sharded(net, B, "bf16", world, params, x, lab, capture=True, n_bands=2)
    for rank, (loss, _) in enumerate(res):
        assert abs(loss - loss_ref) <= 2e-2 * abs(loss_ref), (rank, loss, loss_ref)
    check_conditioned(net, params, ts, lab, res, "bf16")


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_dp_replicas_sum_gradients(prec):
    """Data-parallel replicas (LRCNN_FLAG_DP): two replicas (loopback communicator, one host thread
    and stream each) on different batches; the per-segment gradient buckets are all-reduced on the
    communication stream while the backward goes on.  Every replica's gradient must equal the sum
    of the two single-replica gradients, and its loss its own batch's loss."""
    net = WL.resnet50(H=64, W=32, width_div=4, blocks=(2, 1, 1, 1)) if prec == "bf16" else \
        WL.vgg16(H=32, W=32, width_div=8, segments="pool")
    B = 2
    bf = prec == "bf16"
    params = WL.make_params(net, seed=3, bias_scale=0.05, bf16=bf)
    xs = [WL.make_input(net, B, seed=10 + g, bf16=bf) for g in range(2)]
    labs = [WL.make_labels(net, B, seed=20 + g) for g in range(2)]
    single = []
    for g in range(2):
        p = LB.Plan(net, B, mode="2ps", prec=prec, n_bands=3)
        ds = LB.DeviceState(p)
        ds.load(params=params, x=xs[g], labels=labs[g])
        ds.step_grads()
        torch.cuda.synchronize()
        single.append((float(ds.loss.cpu()), ds.grads.cpu().numpy().copy()))
    comms = LB.Comm.loopback(2)
    plans, states = [], []
    for g in range(2):
        p = LB.Plan(net, B, mode="2ps", prec=prec, n_bands=3, world=2, rank=g, flags=LB.FLAG_DP)
        p.set_comm(comms[g])
        ds = LB.DeviceState(p)
        ds.load(params=params, x=xs[g], labels=labs[g])
        plans.append(p)
        states.append(ds)
    torch.cuda.synchronize()
    errs = [None] * 2

    def body(g):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                states[g].step_grads(stream=st)
            st.synchronize()
        except Exception as e:   # surfaced below
            errs[g] = e

    th = [threading.Thread(target=body, args=(g,)) for g in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert all(e is None for e in errs), errs
    ref = single[0][1] + single[1][1]
    for g in range(2):
        got = states[g].grads.cpu().numpy()
        assert rel(got, ref) <= 1e-5, (g, rel(got, ref))
        assert abs(float(states[g].loss.cpu()) - single[g][0]) <= 1e-6 * max(1.0, abs(single[g][0]))
    for c in comms:
        c.free()


@pytest.mark.parametrize("prec,world", [("fp32", 2), ("fp32", 3), ("bf16", 2), ("bf16", 3)])
def test_zero_redundancy_sharding_vs_oracle(prec, world):
    """LRCNN_FLAG_ZERO_REDUNDANCY: every row of every tensor on one rank, the halo
    rows of rank g+1's first band received after the first band and their delta sent back; loss
    vs the plain oracle, every rank's gradients vs the oracle conditioned on the merged maps (R17d;
    the maps are captured per rank and must tile every tensor)."""
    net = WL.resnet50(H=192, W=48, width_div=4, blocks=(2, 1, 1, 1))
    B = 2
    params, x, lab, loss_ref, _, _ = oracle_ref(net, B, 7, 0.1, bf16=(prec == "bf16"))
    res, ts = run_sharded(net, B, prec, world, params, x, lab, capture=True, flags=LB.FLAG_ZERO_REDUNDANCY,
                          n_bands=2)
    tol = 2e-2 if prec == "bf16" else 1e-5
    for rank, (loss, _) in enumerate(res):
        assert abs(loss - loss_ref) <= tol * abs(loss_ref), (rank, loss, loss_ref)
    check_conditioned(net, params, ts, lab, res, prec)

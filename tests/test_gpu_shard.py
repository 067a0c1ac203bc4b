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
from test_gpu_parity import rel, well_conditioned

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402


def run_sharded(net, B, prec, world, params, x, lab, **kw):
    comms = LB.Comm.loopback(world)
    plans, states = [], []
    for g in range(world):
        p = LB.Plan(net, B, mode="2ps", prec=prec, world=world, rank=g, **kw)
        p.set_comm(comms[g])
        ds = LB.DeviceState(p)
        ds.load(params=params, x=x, labels=lab)
        plans.append(p)
        states.append(ds)
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
    for c in comms:
        c.free()
    return out


def oracle_ref(net, B, seed, bias):
    for tries in range(40):
        params = WL.make_params(net, seed=seed + 97 * tries, bias_scale=bias)
        x = WL.make_input(net, B, seed=seed + 97 * tries)
        ts, _ = C.forward(net, params, x)
        if well_conditioned(net, ts, 1e-5):
            break
    lab = WL.make_labels(net, B)
    _, loss, g, hg, _ = C.step(net, params, x, lab, 0.0)
    return params, x, lab, loss, g, hg


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_resnet_fp32(world):
    net = WL.resnet50(H=96, W=32, width_div=8, blocks=(1, 1, 1, 1))
    B = 2
    params, x, lab, loss_ref, g_ref, hg_ref = oracle_ref(net, B, 5, 0.1)
    res = run_sharded(net, B, "fp32", world, params, x, lab, n_bands=2)
    for rank, (loss, (g, head)) in enumerate(res):
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref), (rank, loss, loss_ref)
        for i, (a, b) in enumerate(zip(g, g_ref)):
            if b is None:
                continue
            for k in b:
                assert rel(a[k], b[k]) <= 1e-5, (rank, i, k, rel(a[k], b[k]))
        for k in ("fc_w", "fc_b"):
            assert rel(head[k], hg_ref[k]) <= 1e-5, (rank, k)


def test_sharded_vgg_fp32_pool_segments():
    net = WL.vgg16(H=64, W=32, width_div=8, segments="pool")
    B = 2
    params, x, lab, loss_ref, g_ref, hg_ref = oracle_ref(net, B, 9, 0.05)
    res = run_sharded(net, B, "fp32", 2, params, x, lab, n_bands=2)
    for rank, (loss, (g, head)) in enumerate(res):
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref)
        for i, (a, b) in enumerate(zip(g, g_ref)):
            if b is None:
                continue
            for k in b:
                assert rel(a[k], b[k]) <= 1e-5, (rank, i, k, rel(a[k], b[k]))


def test_sharded_resnet_bf16_vs_single_rank():
    """bf16 tensor-core path: sharded gradients vs the same GPU path on one rank (same forward
    decisions up to accumulation order), 2e-2."""
    net = WL.resnet50(H=128, W=64, width_div=4, blocks=(1, 1, 1, 1))
    B = 2
    params = WL.make_params(net, seed=3, bias_scale=0.1)
    x = WL.make_input(net, B, seed=3)
    lab = WL.make_labels(net, B)
    ref = run_sharded(net, B, "bf16", 1, params, x, lab, n_bands=2)[0]
    res = run_sharded(net, B, "bf16", 2, params, x, lab, n_bands=2)
    for rank, (loss, (g, head)) in enumerate(res):
        assert abs(loss - ref[0]) <= 2e-2 * abs(ref[0])
        for i, (a, b) in enumerate(zip(g, ref[1][0])):
            if b is None:
                continue
            for k in b:
                assert rel(a[k], b[k]) <= 2e-2, (rank, i, k, rel(a[k], b[k]))


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

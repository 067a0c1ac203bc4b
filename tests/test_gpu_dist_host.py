"""Multi-process row sharding and data parallelism through the host-staged communicator
(lrcnn_comm_init_host + torch.distributed over gloo): two real processes (one per rank, both on the
one GPU of the test box), the library's own halo exchange and per-segment gradient all-reduce,
checked against the fp64 oracle -- loss vs the plain oracle, every rank's gradients vs the oracle's
backward conditioned on the merged maps the ranks stored (R17d).  This is the N > 1 code path of
bench.py (NCCL there) with a different transport."""
import os
import socket
import tempfile

import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from conditioned import validate_forward, conditioned_grads, compare_grads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir, case):
    import torch
    import torch.distributed as dist
    from paper_2401_11471_b200 import lrcnn as LB
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method="tcp://127.0.0.1:%d" % port, rank=rank, world_size=world)
    net, B, prec, kind, seed = case["net"], case["B"], case["prec"], case["kind"], case["seed"]
    bf = prec == "bf16"
    params = WL.make_params(net, seed=seed, bias_scale=0.1, gamma_spread=0.2, bf16=bf)
    xseed = seed + (rank if kind == "dp" else 0)
    x = WL.make_input(net, B, seed=xseed, bf16=bf)
    lab = WL.make_labels(net, B, seed=1 + (rank if kind == "dp" else 0))
    if kind == "rows":
        plan = LB.Plan(net, B, mode="2ps", prec=prec, world=world, rank=rank, n_bands=2,
                       flags=case.get("flags", 0))
    else:
        plan = LB.Plan(net, B, mode="2ps", prec=prec, world=world, rank=rank, n_bands=2, flags=LB.FLAG_DP)
    comm = LB.Comm.host()
    plan.set_comm(comm)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, labels=lab)
    L = len(net["ops"])
    bufs = {}
    if kind == "rows":
        for t in range(1, L + 1):
            c, cp, h, w = plan.tensor(t)
            bufs[t] = torch.full((B, h, w, cp), float("nan"), dtype=ds.dtype, device="cuda")
            plan.debug_capture(t, bufs[t])
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        ds.step_grads(stream=st)
    st.synchronize()
    out = {"loss": float(ds.loss.cpu()), "grads": ds.grads.cpu().numpy()}
    for t, b in bufs.items():
        out["t%d" % t] = b.float().cpu().numpy()
    np.savez(os.path.join(out_dir, "rank%d.npz" % rank), **out)
    plan.set_comm(None)
    comm.free()
    dist.destroy_process_group()


def _run(case, world=2):
    import torch.multiprocessing as mp
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, case), nprocs=world, join=True)
        return [dict(np.load(os.path.join(d, "rank%d.npz" % r))) for r in range(world)]


def _merge(res, net, plan_like):
    ts = []
    for t in range(1, len(net["ops"]) + 1):
        m = res[0]["t%d" % t]
        for r in res[1:]:
            m = np.where(np.isnan(m), r["t%d" % t], m)
        assert not np.isnan(m).any(), ("rows no rank computed", t)
        c = plan_like.tensor(t)[0]
        ts.append(np.asarray(m[..., :c], dtype=np.float64).transpose(0, 3, 1, 2))
    return ts


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_rows_two_processes_host_comm_vs_oracle(prec):
    from paper_2401_11471_b200 import lrcnn as LB
    net = WL.resnet50(H=128, W=48, width_div=4, blocks=(2, 1, 1, 1))
    B = 2
    case = {"net": net, "B": B, "prec": prec, "kind": "rows", "seed": 3}
    res = _run(case)
    bf = prec == "bf16"
    tol = 2e-2 if bf else 1e-5
    params = WL.make_params(net, seed=3, bias_scale=0.1, gamma_spread=0.2, bf16=bf)
    x = WL.make_input(net, B, seed=3, bf16=bf)
    lab = WL.make_labels(net, B, seed=1)
    _, loss_ref, _, _, _ = C.step(net, params, x, lab, 0.0)
    plan_like = LB.Plan(net, B, mode="2ps", prec=prec, n_bands=2)
    ts = [x] + _merge(res, net, plan_like)
    _, aux = validate_forward(net, params, ts, C.bf16_store if bf else C.fp32_store, tol)
    loss_c, dzl, hg, _ = C.head_forward_backward(ts[-1], params["head"], lab)
    g_ref = conditioned_grads(net, params, ts, aux, dzl)
    for r, out in enumerate(res):
        assert abs(out["loss"] - loss_ref) <= tol * abs(loss_ref), (r, out["loss"], loss_ref)
        g, head = plan_like.unpack_grads(out["grads"])
        compare_grads(g, g_ref, tol, ("rank", r))
        for k in ("fc_w", "fc_b"):
            assert float(np.max(np.abs(head[k] - hg[k])) / np.max(np.abs(hg[k]))) <= tol


def test_dp_two_processes_host_comm_sum():
    """Data-parallel replicas in two processes (LRCNN_FLAG_DP, per-segment buckets through the host
    communicator): every replica holds the sum of the two replicas' gradients, each equal to the
    fp32 oracle step on its own batch."""
    from paper_2401_11471_b200 import lrcnn as LB
    net = WL.vgg16(H=32, W=32, width_div=8, segments="pool")
    B = 2
    res = _run({"net": net, "B": B, "prec": "fp32", "kind": "dp", "seed": 3})
    params = WL.make_params(net, seed=3, bias_scale=0.1, gamma_spread=0.2)
    plan_like = LB.Plan(net, B, mode="2ps", prec="fp32", n_bands=2)
    g_sum, h_sum = None, None
    for r in range(2):
        x = WL.make_input(net, B, seed=3 + r)
        lab = WL.make_labels(net, B, seed=1 + r)
        _, loss, g, hg, _ = C.step(net, params, x, lab, 0.0)
        assert abs(res[r]["loss"] - loss) <= 1e-5 * abs(loss)
        g_sum = g if g_sum is None else [None if a is None else {k: a[k] + b[k] for k in a} for a, b in zip(g_sum, g)]
        h_sum = hg if h_sum is None else {k: h_sum[k] + hg[k] for k in hg}
    for r in range(2):
        g, head = plan_like.unpack_grads(res[r]["grads"])
        compare_grads(g, g_sum, 1e-5, ("replica", r))
        for k in ("fc_w", "fc_b"):
            assert float(np.max(np.abs(head[k] - h_sum[k])) / np.max(np.abs(h_sum[k]))) <= 1e-5


def test_bn_rows_two_processes_host_comm_vs_oracle():
    """Training-mode BN with rows split over two real processes (zero-redundancy cuts, host-staged
    communicator over gloo: the fp64 statistics sums gathered through the exchange callback and summed
    in rank order): loss and every rank's gradients vs the fp64 oracle conditioned on the merged maps
    (fp32, 1e-5)."""
    from paper_2401_11471_b200 import lrcnn as LB
    net = WL.resnet50(H=192, W=48, width_div=4, blocks=(2, 1, 1, 1), bn_train=True)
    B = 2
    case = {"net": net, "B": B, "prec": "fp32", "kind": "rows", "seed": 3, "flags": LB.FLAG_ZERO_REDUNDANCY}
    res = _run(case)
    params = WL.make_params(net, seed=3, bias_scale=0.1, gamma_spread=0.2)
    x = WL.make_input(net, B, seed=3)
    lab = WL.make_labels(net, B, seed=1)
    _, loss_ref, _, _, _ = C.step(net, params, x, lab, 0.0)
    plan_like = LB.Plan(net, B, mode="2ps", prec="fp32", n_bands=2)
    ts = [x] + _merge(res, net, plan_like)
    _, aux = validate_forward(net, params, ts, C.fp32_store, 1e-5)
    loss_c, dzl, hg, _ = C.head_forward_backward(ts[-1], params["head"], lab)
    g_ref = conditioned_grads(net, params, ts, aux, dzl)
    for r, out in enumerate(res):
        assert abs(out["loss"] - loss_ref) <= 1e-5 * abs(loss_ref), (r, out["loss"], loss_ref)
        g, head = plan_like.unpack_grads(out["grads"])
        compare_grads(g, g_ref, 1e-5, ("rank", r))

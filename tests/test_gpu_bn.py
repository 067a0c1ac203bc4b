"""GPU parity of training-mode BatchNorm (R24 / §5.2) through the C-ABI:
the statistics sweeps (FP) and sums sweeps (BP) of the row-centric engine against the fp64 column
oracle with batch statistics.  Tolerances as every parity test (R18): fp32 1e-5, bf16 2e-2;
bf16 follows the storage model R17b and the decision-conditioned gradient check R17d."""
import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from test_gpu_parity import check, rel, run_gpu, TOL
from conditioned import validate_forward, compare_grads
from gpu_util import run_capture

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2401_11471_b200 import lrcnn as LB  # noqa: E402


def test_bn_chain_fp32_bands_and_segments():
    """conv3x3 -> bn(+residual every 2 layers) x4, ragged bands incl. 1-row bands, a checkpoint."""
    net = WL.bn_chain(H=19, W=11, C=3, ch=8, n=4, res_every=2)
    check(net, 2, "fp32", ["column", "2ps", "overl"], [{"band_rows": 1}, {"band_rows": 4}, {"n_bands": 3}],
          bias=0.3, gspread=0.4, plain_grads=True, flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)
    net["ops"][3]["seg_end"] = True
    check(net, 2, "fp32", ["2ps", "overl"], [{"n_bands": 2}, {"band_rows": 3}], bias=0.3, gspread=0.4,
          plain_grads=True, flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)
    # 12 channels: padded to 16 on the device (padded channels must stay zero through the BN)
    net = WL.bn_chain(H=13, W=9, C=3, ch=12, n=3, res_every=2)
    check(net, 3, "fp32", ["column", "2ps"], [{"n_bands": 3}], bias=0.3, gspread=0.4, plain_grads=True)


def check_bn_bf16(net, B, modes, kws, dzl_kind, flags=0):
    """bf16 BN parity (R25): z^L vs the plain oracle, every stored map validated, every
    weight gradient vs the decision-conditioned oracle <= 2e-2 of its max-abs (R18), and every BN
    gamma / beta gradient -- a full-map sum of a delta whose channel mean the downstream BN removes
    -- within 2e-2 of its summation magnitude (sum |da|, sum |da*xh| per channel: the forward-error
    bound of a sum of bf16-rounded terms)."""
    params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=True)
    x = WL.make_input(net, B, bf16=True)
    ts, _ = C.forward(net, params, x, store=C.bf16_store)
    c, h, w = C.out_hw(net)[-1]
    if dzl_kind == "random":
        dzl = WL.make_dzl((B, c, h, w), bf16=True)
    else:
        _, dzl, _, _ = C.head_forward_backward(ts[-1], params["head"], WL.make_labels(net, B))
        dzl = WL.round_bf16(dzl)
    for mode in modes:
        for kw in (kws if mode != "column" else [{}]):
            _, zl, g, tsg = run_capture(net, B, "bf16", mode, params, x, dzl, flags=flags, **kw)
            assert rel(zl, ts[-1]) <= TOL["bf16"], (mode, kw, "zL", rel(zl, ts[-1]))
            _, aux_g = validate_forward(net, params, tsg, C.bf16_store, TOL["bf16"])
            trace = {}
            gr, _ = C.backward(net, params, tsg, aux_g, dzl, need_dx=False, trace=trace)
            wg = [None if net["ops"][i]["kind"] == "bn" else gi for i, gi in enumerate(g)]
            wr = [None if net["ops"][i]["kind"] == "bn" else gi for i, gi in enumerate(gr)]
            compare_grads(wg, wr, TOL["bf16"], (mode, str(kw)))
            worst = 0.0
            for i, tr in trace.items():
                for k in ("gamma", "beta"):
                    e = float(np.max(np.abs(g[i][k] - gr[i][k]) / np.maximum(tr[k], 1e-30)))
                    worst = max(worst, e)
                    assert e <= TOL["bf16"], (mode, kw, i, k, e)


def test_bn_resnet_reduced_fp32_and_bf16():
    """ResNet-50 v1.5 topology with training-mode BN after every conv (identity and projection
    blocks, stem BN before the 3x3/s2 max-pool), per-stage and per-block checkpoints."""
    for segs in ("stage", "block"):
        net = WL.resnet50(H=64, W=48, width_div=8, blocks=(2, 1, 1, 1), bn_train=True, segments=segs)
        check(net, 2, "fp32", ["column", "2ps", "overl"], [{"n_bands": 3}], bias=0.1, gspread=0.2,
              flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)
        check(net, 2, "fp32", ["2ps"], [{"n_bands": 3}], bias=0.1, gspread=0.2, dzl_kind="head")
        for kind in ("head", "random"):
            check_bn_bf16(net, 2, ["column", "2ps", "overl"], [{"n_bands": 3}, {"band_rows": 2}], kind,
                          flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)


def test_bn_step_matches_oracle_fp32():
    """lrcnn_step with training-mode BN: loss and the SGD update of every parameter vs oracle.column.step."""
    net = WL.bn_chain(H=16, W=12, C=3, ch=8, n=3, res_every=2)
    B = 3
    params = WL.make_params(net, seed=2, bias_scale=0.2, gamma_spread=0.3)
    x = WL.make_input(net, B)
    lab = WL.make_labels(net, B)
    lr = 0.05
    new_ref, loss_ref, g_ref, hg_ref, _ = C.step(net, params, x, lab, lr)
    for mode, kw in (("column", {}), ("2ps", {"band_rows": 3}), ("2ps", {"n_bands": 2})):
        plan, ds = run_gpu(net, B, mode, "fp32", params, x, labels=lab, lr=lr, **kw)
        loss = float(ds.loss.cpu())
        assert abs(loss - loss_ref) <= 1e-5 * abs(loss_ref), (mode, kw, loss, loss_ref)
        got, head = plan.unpack_grads(ds.master.cpu().numpy())
        for i, (a, b) in enumerate(zip(got, new_ref["convs"])):
            if b is None:
                continue
            for k in b:
                d_ref = params["convs"][i][k] - b[k]
                d_got = params["convs"][i][k] - a[k]
                # the fp32 master holds theta (gamma ~ 1): its rounding (2^-24 |theta|) bounds the update
                bound = 1e-4 * np.max(np.abs(d_ref)) + 2 * 2.0 ** -24 * np.max(np.abs(params["convs"][i][k]))
                assert np.max(np.abs(d_got - d_ref)) <= bound, (mode, kw, i, k, rel(d_got, d_ref))


def test_bn_step_graph_replay_bf16():
    """Graph-replayed bf16 lrcnn_step with BN sweeps == its eager first call (same loss sequence as
    two eager plans), and the gradients of one step vs the oracle within 2e-2."""
    net = WL.resnet50(H=64, W=48, width_div=8, blocks=(1, 1, 1, 1), bn_train=True)
    B = 2
    params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=True)
    x = WL.make_input(net, B, bf16=True)
    lab = WL.make_labels(net, B)
    plan = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=3)
    ds = LB.DeviceState(plan)
    ds.load(params=params, x=x, labels=lab)
    losses = []
    for _ in range(4):
        ds.step(0.0)
        torch.cuda.synchronize()
        losses.append(float(ds.loss.cpu()))
    assert max(losses) - min(losses) <= 1e-6 * abs(losses[0]), losses   # lr = 0: identical steps
    _, loss_ref, _, _, _ = C.step(net, params, x, lab, 0.0)
    assert abs(losses[0] - loss_ref) <= 2e-2 * abs(loss_ref)


def test_bn_bench_flags_bf16():
    """The BN path with bench.py's flags (balanced bands, decoupled FP bands, tensor cores required)
    and per-block checkpoints, bf16, vs the oracle (R17d / R25)."""
    net = WL.resnet50(H=64, W=48, width_div=8, blocks=(2, 1, 1, 1), bn_train=True, segments="block")
    flags = LB.FLAG_BALANCED_BANDS | LB.FLAG_FP_MERGE | LB.FLAG_REQUIRE_TC
    check_bn_bf16(net, 2, ["2ps"], [{"n_bands": 4}], "head", flags=flags)


def test_bn_data_parallel_replicas_fp32():
    """Training-mode BN under data-parallel replicas (LRCNN_FLAG_DP, loopback communicator): every
    replica normalises by its own batch's statistics, and the all-reduced gradient equals the sum of
    the oracle's per-replica column gradients (fp32, 1e-5)."""
    import threading
    net = WL.bn_chain(H=20, W=12, C=3, ch=8, n=4, res_every=2)
    net["ops"][3]["seg_end"] = True
    B = 2
    params = WL.make_params(net, seed=3, bias_scale=0.2, gamma_spread=0.3)
    xs = [WL.make_input(net, B, seed=10 + g) for g in range(2)]
    labs = [WL.make_labels(net, B, seed=20 + g) for g in range(2)]
    ref = [C.step(net, params, xs[g], labs[g], 0.0) for g in range(2)]
    comms = LB.Comm.loopback(2)
    plans, states = [], []
    for g in range(2):
        p = LB.Plan(net, B, mode="2ps", prec="fp32", n_bands=3, world=2, rank=g, flags=LB.FLAG_DP)
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
    for g in range(2):
        got, head = plans[g].unpack_grads(states[g].grads.cpu().numpy())
        assert abs(float(states[g].loss.cpu()) - ref[g][1]) <= 1e-5 * abs(ref[g][1])
        for i, gi in enumerate(got):
            if gi is None:
                continue
            for k in gi:
                want = ref[0][2][i][k] + ref[1][2][i][k]
                assert rel(gi[k], want) <= 1e-5, (g, i, k, rel(gi[k], want))
    for c in comms:
        c.free()


@pytest.mark.parametrize("prec,world", [("fp32", 2), ("fp32", 3), ("bf16", 2)])
def test_bn_zero_redundancy_row_sharding(prec, world):
    """Training-mode BN with rows of every image split over ranks (LRCNN_FLAG_ZERO_REDUNDANCY,
    loopback communicator): every rank sums its own rows, the fp64 sums are all-reduced before the
    statistics and the backward sums are final, the ZR halo exchange runs in every statistics / sums
    sweep.  Loss vs the oracle, every rank's all-reduced gradient vs the oracle conditioned on the
    merged maps (fp32 1e-5; bf16 2e-2, BN parameters against their summation magnitude, R25)."""
    from test_gpu_shard import run_sharded
    net = WL.resnet50(H=192, W=48, width_div=4, blocks=(2, 1, 1, 1), bn_train=True)
    B = 2
    bf = prec == "bf16"
    params = WL.make_params(net, seed=7, bias_scale=0.1, gamma_spread=0.2, bf16=bf)
    x = WL.make_input(net, B, seed=7, bf16=bf)
    lab = WL.make_labels(net, B)
    _, loss_ref, _, _, _ = C.step(net, params, x, lab, 0.0)
    res, ts = run_sharded(net, B, prec, world, params, x, lab, capture=True, flags=LB.FLAG_ZERO_REDUNDANCY,
                          n_bands=2)
    tol = TOL[prec]
    store = C.bf16_store if bf else C.fp32_store
    _, aux = validate_forward(net, params, ts, store, tol)
    loss_c, dzl, hg, _ = C.head_forward_backward(ts[-1], params["head"], lab)
    trace = {}
    g_ref, _ = C.backward(net, params, ts, aux, dzl, need_dx=False, trace=trace)
    for rank, (loss, (g, head)) in enumerate(res):
        assert abs(loss - loss_ref) <= tol * abs(loss_ref), (rank, loss, loss_ref)
        if not bf:
            compare_grads(g, g_ref, tol, ("rank", rank))
            continue
        wg = [None if net["ops"][i]["kind"] == "bn" else gi for i, gi in enumerate(g)]
        wr = [None if net["ops"][i]["kind"] == "bn" else gi for i, gi in enumerate(g_ref)]
        compare_grads(wg, wr, tol, ("rank", rank))
        for i, tr in trace.items():
            for k in ("gamma", "beta"):
                e = float(np.max(np.abs(g[i][k] - g_ref[i][k]) / np.maximum(tr[k], 1e-30)))
                assert e <= tol, (rank, i, k, e)


def test_bn_auto_segments_fp32():
    """Training-mode BN with the sqrt(n) automatic checkpoints (LRCNN_FLAG_AUTO_SEGMENTS, f2): the plan's
    own cuts, FP / BP stashes and tails, fp32 vs the plain oracle (segmentation never changes the result)."""
    net = WL.resnet50(H=64, W=48, width_div=8, blocks=(2, 1, 1, 1), bn_train=True, segments="none")
    check(net, 2, "fp32", ["2ps"], [{"n_bands": 3}], bias=0.1, gspread=0.2, flags=LB.FLAG_AUTO_SEGMENTS)


def test_bn_full_resnet50_224_bench_flags_bf16():
    """Full-depth ResNet-50 v1.5 with training-mode BN after all 53 convolutions at 224 x 224 (C3's image
    size, batch 4), per-block checkpoints, bench.py's flags (balanced + decoupled FP bands, tensor cores
    required), bf16: every stored map validated op by op from the GPU's own stored inputs, every gradient
    vs the decision-conditioned fp64 oracle (R17d / R25).  z^L is NOT compared with the unconditioned
    oracle chain here: 53 batch normalisations in a row multiply any storage / accumulation-order
    difference by |mean|/sigma per layer (the same net drifts 1.2e-4 in fp32 and ~0.3 in bf16 from the
    fp64 chain in COLUMN mode too, `scripts/diag_bn_full.py`) -- a property of the net, not of the
    row-centric schedule (R26)."""
    net = WL.resnet50(H=224, W=224, bn_train=True, segments="block")
    flags = LB.FLAG_BALANCED_BANDS | LB.FLAG_FP_MERGE | LB.FLAG_REQUIRE_TC
    B = 4
    params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2, bf16=True)
    x = WL.make_input(net, B, bf16=True)
    c, h, w = C.out_hw(net)[-1]
    dzl = WL.make_dzl((B, c, h, w), bf16=True)   # C1's loss field: no head, so z^L drift cannot enter
    _, zl, g, tsg2 = run_capture(net, B, "bf16", "2ps", params, x, dzl, flags=flags, n_bands=4)
    _, aux_g = validate_forward(net, params, tsg2, C.bf16_store, TOL["bf16"])
    trace = {}
    gr, _ = C.backward(net, params, tsg2, aux_g, dzl, need_dx=False, trace=trace)
    wg = [None if net["ops"][i]["kind"] == "bn" else gi for i, gi in enumerate(g)]
    wr = [None if net["ops"][i]["kind"] == "bn" else gi for i, gi in enumerate(gr)]
    compare_grads(wg, wr, TOL["bf16"], "full resnet50 bn")
    for i, tr in trace.items():
        for k in ("gamma", "beta"):
            e = float(np.max(np.abs(g[i][k] - gr[i][k]) / np.maximum(tr[k], 1e-30)))
            assert e <= TOL["bf16"], (i, k, e)

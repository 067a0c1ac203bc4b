"""The oracle's G-rank simulation -- CPU only.

oracle.rowcentric.step_ranks splits the rows of every segment output over G simulated ranks; each
rank computes the OverL hull of its owned rows (enumerate_rank) with 2PS bands inside and shares
nothing with the other ranks but explicit message buffers (halo rows forward, their delta back,
partial GAP sums, the weight-gradient sum).  Pins:
  * the method invariant: G-rank training == the column oracle (fp64, <= 1e-12) for G = 2..8
    on a chain, a VGG stack with pool checkpoints and ResNet-like DAGs -- a hull that is too
    narrow fails here (a rank reads a row it does not hold, or gets a wrong value);
  * the hull width: on stride-1 chains the extended input ranges of neighbouring ranks overlap by
    exactly Eq. (15)'s o^0, so a hull that is too WIDE fails too;
  * a negative control: dropping one halo message breaks the invariant;
  * the CUDA planner's exchange schedule (lrcnn_plan_xfers, host code, no GPU) equals the oracle's
    messages exactly."""
import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from oracle import enumerate as EN
from oracle import memmodel as MM
from oracle import rowcentric as RC


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


def _compare(net, B, worlds, **kw):
    params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2)
    x = WL.make_input(net, B, seed=4)
    lab = WL.make_labels(net, B)
    new_ref, loss_ref, g_ref, hg_ref, ts = C.step(net, params, x, lab, 0.05)
    for world in worlds:
        new, loss, g, hg, zl, log = RC.step_ranks(net, params, x, lab, 0.05, world, **kw)
        assert abs(loss - loss_ref) <= 1e-12 * abs(loss_ref), (world, loss, loss_ref)
        assert rel(zl, ts[-1]) <= 1e-12, world
        for i, ref in enumerate(g_ref):
            if ref is None:
                continue
            for k in ref:
                assert rel(g[i][k], ref[k]) <= 1e-12, (world, i, k, rel(g[i][k], ref[k]))
        for k in hg_ref:
            assert rel(hg[k], hg_ref[k]) <= 1e-12
        for i, ref in enumerate(new_ref["convs"]):
            if ref is not None:
                for k in ref:
                    assert rel(new["convs"][i][k], ref[k]) <= 1e-12


@pytest.mark.parametrize("world", [2, 3, 5, 8])
def test_ranks_chain_equal_column(world):
    _compare(WL.tiny3(p=1, H=40, W=9), 2, [world], n_bands=2)


def test_ranks_chain_p0_single_row_bands():
    _compare(WL.tiny3(p=0, H=37, W=7), 1, [2, 4, 7], band_rows=1)


def test_ranks_vgg_pool_segments_equal_column():
    """VGG topology with per-pool checkpoints: halo exchange at every segment input (deep segments
    reach past the neighbour at G >= 4)."""
    net = WL.vgg16(H=256, W=32, width_div=16, segments="pool")
    _compare(net, 1, [2, 3, 8], n_bands=2)


def test_ranks_resnet_dag_equal_column():
    """ResNet-50 topology (7x7/s2 stem, 3x3/s2 max-pool, projection + identity bottlenecks, stride-2
    3x3, fused residual), per-stage checkpoints."""
    net = WL.resnet50(H=160, W=16, width_div=8, blocks=(2, 1, 1, 1))
    _compare(net, 1, [2, 3, 5], n_bands=2)


def test_hull_overlap_is_eq15():
    """Stride-1 chains: rank g's extended input range ends exactly o^0 rows (Eq. (15) with o^L = 0)
    past rank g+1's start, for every interior cut -- the hull is neither too narrow nor too wide."""
    rng = np.random.default_rng(5)
    for _ in range(40):
        L = int(rng.integers(1, 6))
        chain = [(int(k), 1, int(rng.integers(0, (k + 1) // 2 + 1))) for k in rng.choice([1, 3, 5], size=L)]
        o0 = MM.overlap_chain(chain)[0]
        H = 200
        ops, t = [], 0
        for (k, s, p) in chain:
            ops.append(WL.conv(t, 2, k, s, p))
            t += 1
        net = {"C": 1, "H": H, "W": 32, "classes": 3, "ops": ops}
        shp = C.out_hw(net)
        seg = EN.segments(net)[0]
        world = int(rng.integers(2, 6))
        ext = [EN.enumerate_rank(net, seg, world, g, n_bands=1, shp=shp)[0][0] for g in range(world)]
        for g in range(world - 1):
            lo_next = ext[g + 1][0]
            hi = ext[g][1]
            if lo_next > 0 and hi < H:            # interior: no clipping at the image border
                assert hi - lo_next == o0, (chain, world, g, ext, o0)


def test_negative_control_dropped_halo_message():
    """Without one halo message (the receiving rank keeps zeros in those rows) the result differs."""
    net = WL.vgg16(H=64, W=12, width_div=16, segments="pool", cfg=[64, 64, "M", 128, 128, "M", 256, "M"])
    params = WL.make_params(net, seed=2, bias_scale=0.1)
    x = WL.make_input(net, 1, seed=4)
    lab = WL.make_labels(net, 1)
    _, _, g_ref, _, ts = C.step(net, params, x, lab, 0.0)
    orig = RC._messages

    def drop_first(plans, s, seg_in):
        return orig(plans, s, seg_in)[1:]

    RC._messages = drop_first
    try:
        _, _, g, _, zl, _ = RC.step_ranks(net, params, x, lab, 0.0, 2, n_bands=2)
    finally:
        RC._messages = orig
    err = max(rel(g[i][k], g_ref[i][k]) for i in range(len(g_ref)) if g_ref[i] for k in g_ref[i])
    assert max(err, rel(zl, ts[-1])) > 1e-3


def test_planner_exchange_schedule_equals_oracle_messages():
    """lrcnn_plan_xfers (the CUDA library's host planner) lists, per rank and segment, exactly the
    oracle's halo messages: receive (peer, rows) = rows of the segment input the rank needs and the
    peer owns; send = the mirror image."""
    LB = pytest.importorskip("paper_2401_11471_b200.lrcnn")
    from test_plan import random_net
    rng = np.random.default_rng(77)
    cases = [(WL.vgg16(H=128, W=32, width_div=16, segments="pool"), 4, {"n_bands": 2}),
             (WL.resnet50(H=160, W=16, width_div=8, blocks=(2, 1, 1, 1)), 3, {"n_bands": 2})]
    while len(cases) < 40:
        net = random_net(rng)
        try:
            C.out_hw(net)
        except ValueError:
            continue
        cases.append((net, int(rng.integers(2, 5)), {"n_bands": int(rng.integers(1, 3))}))
    checked = 0
    for net, world, kw in cases:
        try:
            plans = [LB.Plan(net, 2, mode="2ps", prec="bf16", world=world, rank=g, **kw) for g in range(world)]
        except LB.LrcnnError as e:
            assert e.name == "E_INFEASIBLE"
            continue
        oplans = [RC.RankPlan(net, world, g, **kw) for g in range(world)]
        for s, (seg_in, _, _) in enumerate(oplans[0].segs):
            if s == 0:
                continue
            msgs = RC._messages(oplans, s, seg_in)
            for g in range(world):
                want = sorted([(src, 0, r0, r1) for (src, dst, r0, r1) in msgs if dst == g] +
                              [(dst, 1, r0, r1) for (src, dst, r0, r1) in msgs if src == g])
                got = sorted(plans[g].xfers(s))
                assert got == want, (world, g, s, got, want)
        checked += 1
    assert checked >= 20

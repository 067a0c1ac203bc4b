"""Zero-redundancy row sharding (LRCNN_FLAG_ZERO_REDUNDANCY), host side on CPU:
  * the oracle's G-rank simulation (oracle.rowcentric.step_ranks_zr: every row of every tensor on ONE
    rank, halo rows from the rank below after the first band, their delta sent back) equals the
    column oracle to 1e-12 for G = 2..4 on a chain, VGG (pool checkpoints) and ResNet DAGs;
  * no row is computed twice: the ranks' computed rows of every tensor tile [0, H_t) exactly;
  * the CUDA planner's rank ranges, bands, buffer read ends and halo schedule equal the oracle's
    set-based enumeration (enumerate_rank_zr) on random DAGs, including the infeasible cases."""
import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from oracle import enumerate as EN
from oracle import rowcentric as RC


def rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


@pytest.mark.parametrize("net,B,kw,worlds", [
    (WL.tiny3(p=1, H=40, W=9), 2, {"n_bands": 2}, (2, 3, 4)),
    (WL.tiny3(p=0, H=37, W=7), 1, {"n_bands": 1}, (2, 3)),
    (WL.vgg16(H=256, W=32, width_div=16, segments="pool"), 1, {"n_bands": 2}, (2,)),
    (WL.resnet50(H=192, W=24, width_div=8, blocks=(2, 1, 1, 1)), 1, {"n_bands": 2}, (2, 3)),
])
def test_zr_ranks_equal_column(net, B, kw, worlds):
    params = WL.make_params(net, seed=2, bias_scale=0.1, gamma_spread=0.2)
    x = WL.make_input(net, B, seed=4)
    lab = WL.make_labels(net, B)
    new_ref, loss_ref, g_ref, hg_ref, ts = C.step(net, params, x, lab, 0.05)
    for world in worlds:
        new, loss, g, hg, zl, log = RC.step_ranks_zr(net, params, x, lab, 0.05, world, **kw)
        assert abs(loss - loss_ref) <= 1e-12 * abs(loss_ref)
        assert rel(zl, ts[-1]) <= 1e-12
        for i, ref in enumerate(g_ref):
            if ref is not None:
                for k in ref:
                    assert rel(g[i][k], ref[k]) <= 1e-12, (world, i, k)
        assert any(e[0] == "fp" for e in log) and any(e[0] == "bp" for e in log)


def test_zr_no_row_computed_twice():
    net = WL.resnet50(H=192, W=24, width_div=8, blocks=(2, 1, 1, 1))
    shp = C.out_hw(net)
    for seg in EN.segments(net):
        seg_in, ids, out = seg
        for world in (2, 3):
            count = {i + 1: np.zeros(shp[i + 1][1], dtype=int) for i in ids}
            for g in range(world):
                own, bands, _ = EN.enumerate_rank_zr(net, seg, world, g, n_bands=2, shp=shp)
                for band in bands:
                    for t in count:
                        lo, a, b, hi = band[t]
                        count[t][a:b] += 1
            for t, c in count.items():
                assert np.all(c == 1), (seg, world, t, c)


def test_zr_planner_equals_enumerator():
    LB = pytest.importorskip("paper_2401_11471_b200.lrcnn")
    from test_plan import random_net
    rng = np.random.default_rng(91)
    cases = [(WL.resnet50(H=192, W=24, width_div=8, blocks=(2, 1, 1, 1)), 3, 2),
             (WL.vgg16(H=256, W=32, width_div=16, segments="pool"), 2, 2),
             (WL.vgg16(H=256, W=32, width_div=16, segments="pool"), 3, 2)]
    while len(cases) < 60:
        net = random_net(rng)
        try:
            C.out_hw(net)
        except ValueError:
            continue
        cases.append((net, int(rng.integers(2, 4)), int(rng.integers(2, 4))))
    ok = infeasible = 0
    for net, world, nb in cases:
        shp = C.out_hw(net)
        segs = EN.segments(net)
        try:
            ref = [[EN.enumerate_rank_zr(net, seg, world, g, n_bands=nb, shp=shp) for g in range(world)]
                   for seg in segs]
            ref_ok = all(len(ref[s][g][1]) >= 2 for s in range(len(segs)) for g in range(world - 1))
        except ValueError:
            ref_ok = False
        plans = []
        try:
            for g in range(world):
                plans.append(LB.Plan(net, 2, mode="2ps", prec="bf16", n_bands=nb, world=world, rank=g,
                                     flags=LB.FLAG_ZERO_REDUNDANCY))
        except LB.LrcnnError as e:
            assert e.name == "E_INFEASIBLE", e
            infeasible += 1
            continue
        assert ref_ok, "planner accepted a plan the enumerator finds infeasible"
        for s, seg in enumerate(segs):
            seg_in, ids, out = seg
            for g, plan in enumerate(plans):
                own, bands, (ol, oh) = ref[s][g]
                assert plan.seg(s)[2] == len(bands)
                for t in [i + 1 for i in ids]:
                    o_lo, o_hi, lo, hi = plan.shard(s, t)
                    assert (o_lo, o_hi) == (ol, oh)
                    assert (lo, hi) == own[t], (s, g, t, (lo, hi), own[t])
                    for r, band in enumerate(bands):
                        assert plan.rows(s, r, t) == band[t][:3], (s, g, r, t, plan.rows(s, r, t), band[t])
                        assert plan.read_end(s, r, t) == band[t][3], (s, g, r, t)
                # halo schedule: rows of rank g+1 my last band reads / my rows rank g-1 reads
                want = []
                for t in [i + 1 for i in ids]:
                    if t == out:
                        continue
                    if g + 1 < world and bands[-1][t][3] > own[t][1]:
                        want.append((t, 0, own[t][1], bands[-1][t][3]))
                    if g > 0:
                        up_own, up_bands, _ = ref[s][g - 1]
                        if up_bands[-1][t][3] > up_own[t][1]:
                            want.append((t, 1, up_own[t][1], up_bands[-1][t][3]))
                assert sorted(plan.zr_halo(s)) == sorted(want), (s, g)
        ok += 1
    assert ok >= 20 and infeasible >= 1, (ok, infeasible)

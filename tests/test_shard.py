"""Row sharding across ranks, host logic on CPU: per-rank row ranges and 2PS
bands vs the oracle's set-based enumeration; the halo exchange schedule is mirrored between
neighbours and covers exactly the extended input range; a world_size-2 gloo run builds each
rank's plan in its own process and cross-checks the schedules."""
import os

import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from oracle import enumerate as EN
from paper_2401_11471_b200 import lrcnn as LB
from test_plan import random_net


def _plans(net, world, B=2, **kw):
    out = []
    for g in range(world):
        out.append(LB.Plan(net, B, mode="2ps", prec="bf16", world=world, rank=g, **kw))
    return out


def _check_rank(net, world, g, plan, kw):
    shp = C.out_hw(net)
    segs = EN.segments(net)
    for s, seg in enumerate(segs):
        seg_in, ids, out = seg
        ext, bands, (ol, oh) = EN.enumerate_rank(net, seg, world, g, shp=shp, **kw)
        for t in [seg_in] + [i + 1 for i in ids]:
            own_lo, own_hi, lo, hi = plan.shard(s, t)
            assert (own_lo, own_hi) == (ol, oh)
            assert (lo, hi) == ext[t], (s, t, (lo, hi), ext[t])
        assert plan.seg(s)[2] == len(bands)
        for r, band in enumerate(bands):
            for t in [i + 1 for i in ids]:
                assert plan.rows(s, r, t) == band[t], (world, g, s, r, t, plan.rows(s, r, t), band[t])


def test_shard_rows_vs_enumerator():
    rng = np.random.default_rng(31)
    done = 0
    while done < 60:
        net = random_net(rng)
        try:
            shp = C.out_hw(net)
        except ValueError:
            continue
        world = int(rng.integers(2, 5))
        kw = {"n_bands": int(rng.integers(1, 4))}
        try:
            plans = _plans(net, world, **kw)
        except LB.LrcnnError as e:
            assert e.name == "E_INFEASIBLE"
            continue
        for g, p in enumerate(plans):
            _check_rank(net, world, g, p, kw)
        done += 1


@pytest.mark.parametrize("world", [2, 4, 8])
def test_resnet50_c4_shards(world):
    """C4 (ResNet-50, 3600x2400, per-stage segments): every rank's ranges and bands."""
    net = WL.resnet50(H=3600, W=2400)
    kw = {"n_bands": 4}
    plans = _plans(net, world, B=8, **kw)
    for g in (0, world // 2, world - 1):
        _check_rank(net, world, g, plans[g], kw)
    _check_mirror(net, plans)


def _check_mirror(net, plans):
    world = len(plans)
    segs = EN.segments(net)
    for s in range(len(segs)):
        seg_in = segs[s][0]
        for g, p in enumerate(plans):
            xs = p.xfers(s)
            if seg_in == 0 or world == 1:
                assert xs == []
                continue
            for peer, send, r0, r1 in xs:
                assert abs(peer - g) == 1 and r1 > r0
                assert (g, 1 - send, r0, r1) in plans[peer].xfers(s)
            # received rows + owned rows == the rank's extended range of the segment input
            ol, oh, lo, hi = p.shard(s, seg_in)
            prev_lo, prev_hi = EN.rank_rows(C.out_hw(net)[seg_in][1], world, g)
            got = set(range(prev_lo, prev_hi))
            for peer, send, r0, r1 in xs:
                if not send:
                    got |= set(range(r0, r1))
            assert set(range(lo, hi)) <= got


def test_xfer_schedule_mirror():
    for net, world in [(WL.vgg16(H=224, W=64, segments="pool"), 2), (WL.resnet50(H=448, W=64), 3),
                       (WL.resnet50(H=448, W=64, width_div=8), 4)]:
        _check_mirror(net, _plans(net, world, n_bands=2))


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        net = WL.resnet50(H=448, W=64, width_div=8)
        p = LB.Plan(net, 2, mode="2ps", prec="bf16", n_bands=2, world=world, rank=rank)
        mine = {s: p.xfers(s) for s in range(p.nsegs())}
        allx = [None] * world
        dist.all_gather_object(allx, mine)
        ok = True
        for s, xs in mine.items():
            for peer, send, r0, r1 in xs:
                ok &= (rank, 1 - send, r0, r1) in allx[peer][s]
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_schedules():
    """Two processes (gloo, 127.0.0.1), each plans its own rank; schedules agree across ranks."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    assert sorted(res) == [(0, True), (1, True)]

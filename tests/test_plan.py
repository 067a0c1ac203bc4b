"""Host-side tests of the C-ABI library (no GPU): the library loads and exports
every symbol include/lrcnn.h declares; the planner's band/halo rows are
bit-exact against the oracle's brute-force enumerator; errors; memory/FLOP
accounting against the paper's formulas (oracle/memmodel)."""
import os
import re

import numpy as np
import pytest

import workloads as WL
from oracle import column as C
from oracle import enumerate as EN
from oracle import memmodel as MM
from oracle import rowcentric as RC
from paper_2401_11471_b200 import lrcnn as LB

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    hdr = open(os.path.join(ROOT, "include", "lrcnn.h")).read()
    names = set(re.findall(r"LRCNN_API\s+[\w\s\*]*?\b(lrcnn_\w+)\s*\(", hdr))
    assert len(names) >= 18
    L = LB.lib()
    for n in names:
        assert hasattr(L, n), n
    assert set(LB.EXPORTS) == names
    assert b"sm_100a" in L.lrcnn_version()


def random_net(rng, allow_res=True):
    """Random DAG: chains of conv/maxpool with strides, optional residual blocks and checkpoints."""
    H = int(rng.integers(12, 40))
    W = int(rng.integers(3, 9))
    C0 = int(rng.integers(1, 4))
    ops = []
    t = 0
    h, w = H, W
    n = int(rng.integers(1, 7))
    for _ in range(n):
        kind = rng.random()
        if allow_res and kind < 0.25 and h >= 3:
            # bottleneck-ish block: a = conv(t); b = conv(a); out = relu(conv1x1(b) + t or proj(t))
            s = int(rng.integers(1, 3)) if h >= 6 else 1
            ops.append(WL.conv(t, 3, 1, 1, 0, epi="affine"))
            a = len(ops)
            ops.append(WL.conv(a, 3, 3, s, 1, epi="affine"))
            b = len(ops)
            if s == 1:
                ops.append(WL.conv(b, 4, 1, 1, 0, epi="affine", relu=False))
                c = len(ops)
                ops.append(WL.conv(t, 4, 1, 1, 0, epi="affine", relu=False))
                d = len(ops)
                ops.append(WL.add(c, d, relu=True))
            else:
                ops.append(WL.conv(t, 4, 1, 2, 0, epi="affine", relu=False))
                d = len(ops)
                ops.append(WL.conv(b, 4, 1, 1, 0, epi="affine", res=d))
            t = len(ops)
            h = (h - 1) // s + 1
            w = (w - 1) // s + 1
        elif kind < 0.45 and h >= 4 and w >= 2:
            k = int(rng.choice([2, 3]))
            s = 2
            p = int(rng.integers(0, 2)) if k == 3 else 0
            if (h + 2 * p - k) // s + 1 < 2 or (w + 2 * p - k) // s + 1 < 1:
                continue
            ops.append(WL.maxpool(t, k, s, p))
            t = len(ops)
            h, w = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
        else:
            k = int(rng.choice([1, 2, 3, 5, 7]))
            s = int(rng.choice([1, 1, 2]))
            p = int(rng.integers(0, (k - 1) // 2 + 1))
            ho, wo = (h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1
            if ho < 2 or wo < 1:
                continue
            ops.append(WL.conv(t, int(rng.integers(1, 5)), k, s, p, epi=str(rng.choice(["bias", "affine", "none"])),
                               relu=bool(rng.random() < 0.8)))
            t = len(ops)
            h, w = ho, wo
        if rng.random() < 0.25:
            ops[-1]["seg_end"] = True
    if not ops:
        ops.append(WL.conv(0, 2, 3, 1, 1))
    ops[-1]["seg_end"] = False
    return {"C": C0, "H": H, "W": W, "classes": 3, "ops": ops}


def _check_plan_vs_enum(net, mode, band_rows=None, n_bands=None, B=2):
    plan = LB.Plan(net, B, mode=mode, prec="fp32", band_rows=band_rows, n_bands=n_bands,
                   flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)
    shp = C.out_hw(net)
    segs = EN.segments(net)
    assert plan.nsegs() == len(segs)
    for s, seg in enumerate(segs):
        seg_in, ids, out = seg
        E = EN.band_ends(shp[out][1], band_rows=band_rows, n_bands=n_bands if band_rows is None else None)
        pin, pout, nb = plan.seg(s)
        assert (pin, pout, nb) == (seg_in, out, len(E))
        if mode == "overl":
            en = EN.enumerate_overl(net, seg, E, shp)
            for r in range(len(E)):
                for t in [seg_in] + [i + 1 for i in ids]:
                    lo, a, b = plan.rows(s, r, t)
                    elo, ehi = en[r][t]
                    if t == out:
                        elo, ehi = (E[r - 1] if r else 0), E[r]
                    assert (lo, a, b) == (elo, elo, ehi), (net, mode, s, r, t)
        else:
            en = EN.enumerate_2ps(net, seg, E, shp)
            for r in range(len(E)):
                for t in [i + 1 for i in ids]:
                    assert plan.rows(s, r, t) == en[r][t], (net, mode, s, r, t, plan.rows(s, r, t), en[r][t])
    return plan


def test_plan_c1_table():
    net = WL.tiny3(p=1)
    plan = _check_plan_vs_enum(net, "2ps", band_rows=4, B=1)
    assert [plan.rows(0, r, 1)[1:] for r in range(8)] == [(0, 6)] + [(6 + 4 * i, 10 + 4 * i) for i in range(6)] + [(30, 32)]
    _check_plan_vs_enum(net, "overl", band_rows=4, B=1)


@pytest.mark.parametrize("mode", ["2ps", "overl"])
def test_plan_bit_exact_random(mode):
    """Interval rule == brute-force enumeration on >= 100 random DAG configurations (SURVEY 8(c) pin 7)."""
    rng = np.random.default_rng(2024 if mode == "2ps" else 77)
    done = 0
    while done < 120:
        net = random_net(rng)
        try:
            shp = C.out_hw(net)
        except ValueError:
            continue
        hout = min(shp[s[2]][1] for s in EN.segments(net))
        if rng.random() < 0.5:
            kw = {"band_rows": int(rng.integers(1, max(2, hout)))}
        else:
            kw = {"n_bands": int(rng.integers(1, 9))}
        _check_plan_vs_enum(net, mode, **kw)
        done += 1


def test_plan_vgg_and_resnet_like():
    for segs in ("none", "pool"):
        net = WL.vgg16(H=224, W=224, segments=segs)
        for kw in ({"band_rows": 1}, {"n_bands": 4}, {"n_bands": 7}):
            _check_plan_vs_enum(net, "2ps", **kw)
            _check_plan_vs_enum(net, "overl", **kw)


def test_plan_errors():
    net = {"C": 1, "H": 4, "W": 4, "classes": 2, "ops": [WL.conv(0, 2, 5, 1, 0)]}
    with pytest.raises(LB.LrcnnError) as e:
        LB.Plan(net, 1, mode="2ps", prec="fp32", n_bands=2)
    assert e.value.name == "E_SHAPE"
    # OverL infeasible: N > H / o^0
    net = WL.tiny3(p=1, H=16, W=8)
    with pytest.raises(LB.LrcnnError) as e:
        LB.Plan(net, 1, mode="overl", prec="fp32", band_rows=1)
    assert e.value.name == "E_INFEASIBLE"
    LB.Plan(net, 1, mode="overl", prec="fp32", band_rows=1, flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION)
    # reading across a checkpoint boundary
    bad = {"C": 2, "H": 8, "W": 8, "classes": 2,
           "ops": [WL.conv(0, 2, 3, 1, 1, seg_end=True), WL.conv(1, 2, 3, 1, 1), WL.add(2, 0)]}
    with pytest.raises(LB.LrcnnError) as e:
        LB.Plan(bad, 1, mode="2ps", prec="fp32", n_bands=2)
    assert e.value.name == "E_ARG"
    LB.Plan(net, 1, mode="2ps", prec="fp32", n_bands=2, world=2, rank=1)
    with pytest.raises(LB.LrcnnError) as e:      # more ranks than segment-output rows
        LB.Plan(net, 1, mode="2ps", prec="fp32", n_bands=2, world=32, rank=0)
    assert e.value.name == "E_INFEASIBLE"
    with pytest.raises(LB.LrcnnError) as e:      # halo wider than a neighbour's shard
        LB.Plan(WL.vgg16(H=64, W=32, width_div=8), 1, mode="2ps", prec="fp32", n_bands=1, world=8, rank=3)
    assert e.value.name == "E_INFEASIBLE"


def test_memory_and_flops_accounting():
    for net, B, kw in [(WL.tiny3(p=1), 1, {"band_rows": 4}), (WL.vgg16(H=64, W=64), 2, {"n_bands": 4}),
                       (WL.vgg16(H=64, W=64, segments="pool"), 2, {"n_bands": 3})]:
        for mode in ("2ps", "overl", "column"):
            plan = LB.Plan(net, B, mode=mode, prec="bf16", flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION,
                           **({} if mode == "column" else kw))
            m = plan.memory()
            assert m["omega"] == MM.omega(net, B) * 2                        # Eq. (3)
            assert m["tau_flops"] == MM.tau(net, B)
            if mode == "column":     # one segment, one band: the layer-wise dataflow
                flat = dict(net, ops=[dict(o, seg_end=False) for o in net["ops"]])
                rp = RC.Plan(flat, "2ps", n_bands=1)
            else:
                rp = RC.Plan(net, mode, **kw)
            assert m["fwd_flops"] == MM.executed_fwd_flops(rp, B)
            if mode == "2ps":
                # 2PS cache = B * sum over boundaries and tensors of cached rows * W * Cp * 2 bytes
                exp = 0
                for s, (E, bands) in enumerate(rp.bands):
                    seg_in, ids, out = rp.segs[s]
                    for r in range(1, len(bands)):
                        for i in ids:
                            t = i + 1
                            if t == out:
                                continue
                            lo, a, b = bands[r][t]
                            _, cp, _, w = plan.tensor(t)
                            exp += B * (a - lo) * w * cp * 2
                assert m["halo_cache"] == exp
            if mode == "column":
                assert m["halo_cache"] == 0


def test_c1_cache_is_k_minus_s():
    """C1: 2 cached rows per tensor per boundary (k - s = 2)."""
    plan = LB.Plan(WL.tiny3(p=1), 1, mode="2ps", prec="fp32", band_rows=4)
    m = plan.memory()
    assert m["halo_cache"] == 1 * 7 * 2 * (32 * 8) * 4 * 2    # B * (N-1) * c * W*Cp * 4B * 2 tensors


# ---------------------------------------------------------------- balanced bands
def _delta_slot_bytes(net, seg, bands, shp, B, E, cps):
    """BP delta buffers under liveness overlay: in reverse op order the delta of an
    internal tensor t lives from the backward of its last consumer to that of its producer (extended
    to the first consumer of r for the output of a conv with internal residual input r; a projection
    output read only as a residual shares its reader's delta); non-overlapping tensors share a slot
    (greedy by first write, best fit).  Returns the slot bytes."""
    seg_in, ids, out = seg
    align = lambda v: (v + 255) // 256 * 256
    ops = net["ops"]
    cons = {}
    for i in ids:
        op = ops[i]
        cons.setdefault(op["src"], []).append((i, 0))
        if op.get("res", -1) is not None and op.get("res", -1) >= 0:
            cons.setdefault(op["res"], []).append((i, 1))
    internal = [i + 1 for i in ids if i + 1 != out]

    def alias(t):
        op_t = ops[t - 1]
        c = cons.get(t, [])
        if op_t.get("relu") or len(c) != 1 or c[0][1] != 1:
            return -1
        u = ops[c[0][0]]
        if u["kind"] != "conv" or u["res"] != t or shp[c[0][0] + 1] != shp[t] or cps[c[0][0] + 1] != cps[t]:
            return -1
        return c[0][0] + 1
    fw, lr, size = {}, {}, {}
    for t in internal:
        if alias(t) >= 0:
            continue
        fw[t] = max([t - 1] + [i for i, _ in cons.get(t, [])])
        lr[t] = t - 1
        cap = max(max(b[t][2] - b[t][0] for b in bands), 1)
        size[t] = align(B * cap * shp[t][2] * cps[t] * E)
    for i in ids:
        op = ops[i]
        if op["kind"] == "conv" and op["res"] >= 0 and (i + 1) in fw and op["res"] != seg_in and op["res"] != 0:
            lr[i + 1] = min([lr[i + 1]] + [j for j, _ in cons.get(op["res"], [])])
    for t in internal:
        a = alias(t)
        if a >= 0 and a in fw:
            lr[a] = min(lr[a], t - 1)
    slots = []   # [bytes, last_lr]
    for t in sorted(fw, key=lambda t: (-fw[t], t)):
        best = -1
        for k, (by, last) in enumerate(slots):
            if last <= fw[t]:
                continue
            if best < 0:
                best = k
                continue
            fits, bfits = by >= size[t], slots[best][0] >= size[t]
            if (fits != bfits and fits) or (fits == bfits and (by < slots[best][0] if fits else by > slots[best][0])):
                best = k
        if best < 0:
            slots.append([size[t], lr[t]])
        else:
            slots[best] = [max(slots[best][0], size[t]), lr[t]]
    return sum(s[0] for s in slots)


def _arena_bytes(net, seg, bands, shp, B, E, cps):
    """Band working set of one segment from the oracle enumerator's rows: activation buffers (rows
    [lo, b) of every internal tensor, max over bands), the 2PS carry rows [lo, a) and the
    liveness-overlaid delta slots."""
    seg_in, ids, out = seg
    align = lambda v: (v + 255) // 256 * 256
    tot = 0
    for t in [i + 1 for i in ids]:
        if t == out:
            continue
        cap = max(max(b[t][2] - b[t][0] for b in bands), 1)
        ccap = max(b[t][1] - b[t][0] for b in bands)
        rb = shp[t][2] * cps[t] * E
        tot += align(B * cap * rb)
        if ccap > 0:
            tot += align(B * ccap * rb)
    return tot + _delta_slot_bytes(net, seg, bands, shp, B, E, cps)


@pytest.mark.parametrize("which", ["vgg", "resnet", "random"])
def test_balanced_bands_minimal_and_exact(which):
    """FLAG_BALANCED_BANDS: every segment's rows equal the enumerator at that segment's band
    count; that count is the smallest whose working set fits the largest segment's (the budget),
    and the workspace does not grow."""
    rng = np.random.default_rng(5)
    if which == "vgg":
        nets = [(WL.vgg16(H=224, W=224, segments="pool"), 4), (WL.vgg16(H=96, W=40, segments="pool"), 6)]
    elif which == "resnet":
        nets = [(WL.resnet50(H=224, W=224), 4), (WL.resnet50(H=256, W=64), 7)]
    else:
        nets = []
        while len(nets) < 25:
            net = random_net(rng)
            try:
                C.out_hw(net)
                EN.segments(net)
            except ValueError:
                continue
            nets.append((net, int(rng.integers(2, 6))))
    for net, nb in nets:
        B = 2
        try:
            p0 = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=nb)
        except LB.LrcnnError:
            continue
        p1 = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=nb, flags=LB.FLAG_BALANCED_BANDS)
        shp = C.out_hw(net)
        cps = {t: p1.tensor(t)[1] for t in range(len(net["ops"]) + 1)}
        segs = EN.segments(net)
        arenas = []
        for s, seg in enumerate(segs):
            h = shp[seg[2]][1]
            bands = EN.enumerate_2ps(net, seg, EN.band_ends(h, n_bands=nb), shp)
            arenas.append(_arena_bytes(net, seg, bands, shp, B, 2, cps))
        budget = max(arenas)
        for s, seg in enumerate(segs):
            n = p1.seg(s)[2]
            h = shp[seg[2]][1]
            assert 1 <= n <= min(nb, h)
            bands = EN.enumerate_2ps(net, seg, EN.band_ends(h, n_bands=n), shp)
            for r, band in enumerate(bands):
                for t in [i + 1 for i in seg[1]]:
                    assert p1.rows(s, r, t) == band[t]
            assert _arena_bytes(net, seg, bands, shp, B, 2, cps) <= budget
            if n > 1:   # minimal: one band fewer would not fit
                fewer = EN.enumerate_2ps(net, seg, EN.band_ends(h, n_bands=n - 1), shp)
                assert _arena_bytes(net, seg, fewer, shp, B, 2, cps) > budget
        assert p1.ws_bytes <= p0.ws_bytes


# ---------------------------------------------------------------- budget-driven planning (f2)
def _ws(net, B, n, mode="2ps", flags=0):
    return LB.Plan(net, B, mode=mode, prec="bf16", n_bands=n, flags=flags).ws_bytes


@pytest.mark.parametrize("which", ["c2", "c4", "vgg_whole"])
def test_plan_budget_is_smallest_fitting_n(which):
    """lrcnn_plan_budget (the greedy 'largest band that fits'): the returned band
    count is the smallest n whose workspace fits the budget, checked by brute force over plans."""
    if which == "c2":
        net, B, flags = WL.vgg16(H=224, W=224, segments="pool"), 32, LB.FLAG_BALANCED_BANDS
    elif which == "c4":
        net, B, flags = WL.resnet50(H=3600, W=2400), 8, LB.FLAG_BALANCED_BANDS
    else:
        net, B, flags = WL.vgg16(H=512, W=512, segments="none"), 4, 0
    ws = {n: _ws(net, B, n, flags=flags) for n in range(1, 25)}
    lo, hi = min(ws.values()), ws[1]
    for budget in (hi, (lo + hi) // 2, lo + (hi - lo) // 5, lo):
        p = LB.Plan.for_budget(net, B, budget, max_bands=24, flags=flags)
        n = p.n_bands
        assert p.ws_bytes == ws[n] <= budget
        assert all(ws[m] > budget for m in range(1, n)), (which, budget, n)
    with pytest.raises(LB.LrcnnError) as e:
        LB.Plan.for_budget(net, B, lo - 1, max_bands=24, flags=flags)
    assert e.value.status == 3            # LRCNN_E_INFEASIBLE


def test_plan_turning_point():
    """The paper's turning point: 2PS workspace first falls with N (smaller band
    working set) and then rises (the halo cache grows with N); lrcnn_plan_turning_point returns the
    brute-force argmin, strictly inside the range for a whole-net VGG-16 at 2048x2048 (C5's image
    size; z^L has 64 rows, so 64 is the largest band count)."""
    net, B = WL.vgg16(H=2048, W=2048, segments="none"), 2
    ws = {n: _ws(net, B, n) for n in range(1, 65)}
    n_star, w_star = LB.Plan.turning_point(net, B, max_bands=64)
    assert w_star == min(ws.values()) and ws[n_star] == w_star
    assert all(ws[m] > w_star for m in range(1, n_star))
    assert 1 < n_star < 64
    assert ws[64] > w_star and ws[1] > w_star


@pytest.mark.parametrize("which", ["vgg", "resnet"])
def test_fp_merge_bands(which):
    """Decoupled FP bands (LRCNN_FLAG_FP_MERGE, R7): the FP of a segment merges
    consecutive BP bands (N_FP < N_BP where the merged activation buffers fit in the band arena);
    the BP bands, their rows and the workspace are unchanged (peak memory is the same)."""
    net = WL.vgg16(H=224, W=224, segments="pool") if which == "vgg" else WL.resnet50(H=224, W=224)
    B = 8
    for nb in (2, 4, 8):
        p0 = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=nb)
        p1 = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=nb, flags=LB.FLAG_FP_MERGE)
        assert p0.ws_bytes == p1.ws_bytes
        merged = 0
        for s in range(p1.nsegs()):
            nf, nbp = p1.fp_bands(s)
            assert nbp == p0.seg(s)[2] and 1 <= nf <= nbp
            assert p0.fp_bands(s) == (nbp, nbp)
            merged += nf < nbp
            t_in, t_out, n = p1.seg(s)
            for r in range(n):
                for t in range(t_in + 1, t_out + 1):
                    assert p0.rows(s, r, t) == p1.rows(s, r, t)
        assert merged > 0, nb


def test_dp_replica_plan_is_the_single_gpu_plan():
    """LRCNN_FLAG_DP: a replica plans the whole image (no row split): same bands, rows and workspace
    as the single-GPU plan, for every rank; an out-of-range rank is rejected."""
    net = WL.resnet50(H=96, W=64, width_div=8, blocks=(1, 1, 1, 1))
    p0 = LB.Plan(net, 2, mode="2ps", prec="bf16", n_bands=3)
    for rank in range(4):
        p = LB.Plan(net, 2, mode="2ps", prec="bf16", n_bands=3, world=4, rank=rank, flags=LB.FLAG_DP)
        assert p.ws_bytes == p0.ws_bytes and p.nsegs() == p0.nsegs()
        for s in range(p.nsegs()):
            assert p.seg(s) == p0.seg(s)
            t_in, t_out, n = p.seg(s)
            for r in range(n):
                for t in range(t_in + 1, t_out + 1):
                    assert p.rows(s, r, t) == p0.rows(s, r, t)
    with pytest.raises(LB.LrcnnError):
        LB.Plan(net, 2, mode="2ps", prec="bf16", n_bands=3, world=4, rank=4, flags=LB.FLAG_DP)


# ---------------------------------------------------------------- Eq. (12) greedy, sqrt(n) checkpoints
def _first_band_ends(h, n, pm):
    """Band ends of the greedy first band (the lrcnn_plan_opts.first_rows_pm contract)."""
    h1 = max(1, min(int((h * pm + 500) // 1000), h - (n - 1)))
    rest = h - h1
    q, rem = divmod(rest, n - 1)
    E, acc = [h1], h1
    for r in range(n - 1):
        acc += q + (1 if r < rem else 0)
        E.append(acc)
    return E


def test_first_band_rows_vs_enumerator():
    """A large first band (first_rows_pm): every band's rows equal the enumerator's for those band ends."""
    rng = np.random.default_rng(12)
    for net in (WL.tiny3(p=1, H=40, W=8), WL.vgg16(H=96, W=32, width_div=16, segments="pool"),
                WL.resnet50(H=128, W=32, width_div=8)):
        shp = C.out_hw(net)
        for _ in range(4):
            n, pm = int(rng.integers(2, 5)), int(rng.integers(300, 900))
            plan = LB.Plan(net, 2, mode="2ps", prec="bf16", n_bands=n, first_rows_pm=pm)
            for s, seg in enumerate(EN.segments(net)):
                h = shp[seg[2]][1]
                if h < 2:
                    continue
                E = _first_band_ends(h, min(n, h), pm)
                en = EN.enumerate_2ps(net, seg, E, shp)
                assert plan.seg(s)[2] == len(E)
                for r in range(len(E)):
                    for t in [i + 1 for i in seg[1]]:
                        assert plan.rows(s, r, t) == en[r][t], (net["name"], n, pm, s, r, t)


@pytest.mark.parametrize("which", ["vgg", "resnet"])
def test_greedy_eq12_is_lexicographic_optimum(which):
    """lrcnn_plan_greedy: the smallest N for which some first band fits the budget, and at that N the
    largest first band that fits (brute force over the same grid); the first band is the largest."""
    net = WL.vgg16(H=160, W=64, width_div=4) if which == "vgg" else WL.resnet50(H=256, W=64, width_div=4, segments="none")
    B = 2
    ws1 = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=1).ws_bytes
    for frac in (0.55, 0.7, 0.85):
        budget = int(ws1 * frac)
        try:
            g = LB.Plan.greedy(net, B, budget, max_bands=12)
        except LB.LrcnnError as e:
            assert e.name == "E_INFEASIBLE"
            continue
        assert g.ws_bytes <= budget
        n = g.n_bands

        def feasible(nn, pm):
            try:
                return LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=nn, first_rows_pm=pm).ws_bytes <= budget
            except LB.LrcnnError:
                return False
        grid = [int((1000 * k + 32) // 64) for k in range(64, 0, -1)]
        grid = [pm if pm * nn >= 1000 else 0 for nn in [n] for pm in grid]
        for nn in range(1, n):
            cand = [0] if nn == 1 else [pm if pm * nn >= 1000 else 0 for pm in
                                        [int((1000 * k + 32) // 64) for k in range(64, 0, -1)]]
            assert not any(feasible(nn, pm) for pm in cand), (frac, nn)
        if n > 1 and g.first_rows_pm:
            larger = [pm for pm in grid if pm > g.first_rows_pm]
            assert not any(feasible(n, pm) for pm in larger), (frac, n, g.first_rows_pm)
            E = [g.rows(g.nsegs() - 1, r, len(net["ops"]))[2] for r in range(n)]
            sizes = [E[0]] + [E[r] - E[r - 1] for r in range(1, n)]
            assert sizes[0] + 1 >= max(sizes[1:])      # (rounding of small outputs)


def _valid_cuts(net):
    """Ops whose output no other tensor is read past (a checkpoint there cuts the DAG)."""
    last = {}
    for i, op in enumerate(net["ops"]):
        for t in (op["src"], op.get("res", -1)):
            if t is not None and t >= 0:
                last[t] = max(last.get(t, -1), i)
    cuts = []
    for i in range(len(net["ops"]) - 1):
        if all(last.get(t, -1) <= i for t in range(0, i + 1)):
            cuts.append(i)
    return cuts


def test_auto_segments_sqrt_n():
    """LRCNN_FLAG_AUTO_SEGMENTS: ceil(sqrt(n)) - 1 checkpoints, all at valid cuts, spread
    over the net (every segment between n / (2 sqrt(n)) and 2 n / sqrt(n) ops on a chain)."""
    chain = {"C": 1, "H": 64, "W": 8, "classes": 3, "ops": [WL.conv(t, 4, 3, 1, 1) for t in range(25)]}
    p = LB.Plan(chain, 1, mode="2ps", prec="fp32", n_bands=2, flags=LB.FLAG_AUTO_SEGMENTS)
    assert p.nsegs() == 5
    lens = [len([1 for t in range(p.seg(s)[0], p.seg(s)[1])]) for s in range(p.nsegs())]
    assert all(2 <= L <= 10 for L in lens), lens
    for net in (WL.resnet50(H=224, W=64, width_div=8, segments="none"), WL.vgg16(H=224, W=64, width_div=8)):
        n = len(net["ops"])
        p = LB.Plan(net, 1, mode="2ps", prec="bf16", n_bands=2, flags=LB.FLAG_AUTO_SEGMENTS)
        want = int(np.ceil(np.sqrt(n))) - 1
        assert p.nsegs() == want + 1, (net["name"], p.nsegs(), want)
        cuts = set(_valid_cuts(net))
        for s in range(p.nsegs() - 1):
            assert p.seg(s)[1] - 1 in cuts
        # the plan with these checkpoints equals the enumerator on the same segments
        net2 = dict(net, ops=[dict(o, seg_end=(i + 1) in [p.seg(s)[1] for s in range(p.nsegs() - 1)])
                              for i, o in enumerate(net["ops"])])
        _check_plan_vs_enum(net2, "2ps", n_bands=2, B=1)


@pytest.mark.parametrize("nb", [2, 4, 8])
def test_coordination_counters_closed_form(nb):
    """The paper's coordination counters (Sec. V-D): on the C1 chain (three 3x3/s1/p1
    convs, H = 32) OverL-H overlaps 2d rows of a tensor d layers below the output at every band
    boundary (Eq. (15) with k = 3, s = 1: o = 2 + 2 ... per side 1 row per layer) -> (2*2 + 2*1)(N-1) rows,
    and 2PS-H interrupts the computation once per boundary for each of the two internal tensors (both
    read c = k - s = 2 shared rows, Eq. (11)-(14)) and holds (N-1) * 2 tensors * 2 rows * W * C * 4 B
    of sharing data (reading R9)."""
    import bench
    net = WL.tiny3(p=1)
    ov = bench.coordination_counters(LB.Plan(net, 1, mode="overl", prec="fp32", n_bands=nb,
                                             flags=LB.FLAG_ALLOW_OVERLAP_EXHAUSTION))
    assert ov == {"computation_interruptions": 0, "overlapped_rows": 6 * (nb - 1), "sharing_data_bytes": 0}
    tp = bench.coordination_counters(LB.Plan(net, 1, mode="2ps", prec="fp32", n_bands=nb))
    assert tp == {"computation_interruptions": 2 * (nb - 1), "overlapped_rows": 0,
                  "sharing_data_bytes": (nb - 1) * 2 * 2 * 32 * 8 * 4}


def test_bn_plans_vs_enumerator_and_errors():
    """Training-mode BN ops (f4) read their input 1:1: the interval rule of a BN net equals the
    brute-force enumeration (2PS and OverL); row sharding with OverL cuts is refused (R23)."""
    nets = [WL.bn_chain(H=19, W=7, C=3, ch=8, n=4, res_every=2),
            WL.resnet50(H=64, W=48, width_div=8, blocks=(2, 1, 1, 1), bn_train=True),
            WL.resnet50(H=64, W=48, width_div=8, blocks=(2, 1, 1, 1), bn_train=True, segments="block")]
    for net in nets:
        for kw in ({"band_rows": 1}, {"n_bands": 3}, {"n_bands": 1}):
            _check_plan_vs_enum(net, "2ps", **kw)
    net = nets[0]
    for kw in ({"n_bands": 3}, {"band_rows": 2}):
        _check_plan_vs_enum(net, "overl", **kw)
    with pytest.raises(RuntimeError, match="UNSUPPORTED|not supported|ZERO_REDUNDANCY"):
        LB.Plan(net, 2, mode="overl", prec="fp32", n_bands=2, world=2, rank=0)
    # parameters: gamma / beta per BN op in the flat layout
    plan = LB.Plan(net, 2, mode="2ps", prec="fp32", n_bands=2)
    for i, op in enumerate(net["ops"]):
        if op["kind"] == "bn":
            assert plan.param(i, 1)[1] == plan.param(i, 2)[1] == 8


def test_bn_row_sharding_needs_zero_redundancy():
    net = WL.bn_chain(H=19, W=7, C=3, ch=8, n=4, res_every=2)
    with pytest.raises(RuntimeError, match="ZERO_REDUNDANCY|not supported"):
        LB.Plan(net, 2, mode="2ps", prec="fp32", n_bands=2, world=2, rank=0)
    net = WL.bn_chain(H=64, W=7, C=3, ch=8, n=4, res_every=2)
    LB.Plan(net, 2, mode="2ps", prec="fp32", n_bands=2, world=2, rank=0, flags=LB.FLAG_ZERO_REDUNDANCY)


def test_bn_budget_planner_and_auto_segments():
    """The budget-driven planner (f2) and sqrt(n) checkpoints plan training-mode BN nets (f4): the
    smallest fitting band count is returned, and the automatic cuts are valid segment boundaries whose
    plans equal the enumerator (BN ops read 1:1)."""
    net = WL.resnet50(H=320, W=160, width_div=4, blocks=(2, 2, 2, 1), bn_train=True, segments="none")
    B = 2
    ws = {n: _ws(net, B, n) for n in range(1, 13)}
    lo, hi = min(ws.values()), ws[1]
    for budget in (hi, (lo + hi) // 2, lo):
        p = LB.Plan.for_budget(net, B, budget, max_bands=12)
        assert p.ws_bytes == ws[p.n_bands] <= budget
        assert all(ws[m] > budget for m in range(1, p.n_bands))
    p = LB.Plan(net, B, mode="2ps", prec="bf16", n_bands=3, flags=LB.FLAG_AUTO_SEGMENTS)
    assert p.nsegs() > 1
    cut = [dict(o) for o in net["ops"]]
    for s in range(p.nsegs() - 1):
        cut[p.seg(s)[1] - 1]["seg_end"] = True
    _check_plan_vs_enum(dict(net, ops=cut), "2ps", n_bands=3)

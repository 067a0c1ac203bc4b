"""Slow CPU row-centric executor -- TEST INFRASTRUCTURE ONLY.

Algorithm 1 of the paper, executed literally on fp64 CPU
row slabs and driven by the brute-force enumerator (oracle.enumerate), never by
the CUDA planner:

  FP (l.5-10): bands r = 1..N, every op of the segment computes its band rows
     z_r^l = Conv(z_r^{l-1}) (Eq. (4)) from the rows the band holds; with
     semi-closed padding: zero rows only at the global top/bottom.
     2PS keeps the rows the next band reads ("cache");
     OverL recomputes the replicated rows instead.
  z^L concatenated (l.11), head (l.12-14), delta^L split by row ownership (l.15, R8).
  BP (l.16-23): bands r = N..1 recompute their band (l.17), then Eq. (5)
     per op in reverse; wgrad summed over bands (l.20, "g^l +="); 2PS carries the
     delta of cached rows to band r-1 (R6); OverL sums per-band contributions
     under disjoint output ownership (R5).
  Segments (checkpoints, 2PS-H / OverL-H): full-width maps
     at segment boundaries; BP walks segments in reverse.

G-rank simulation: RankPlan / step_ranks split the rows of every segment
output over G simulated ranks (enumerate_rank); rank g computes each tensor over the OverL hull of
its owned output rows (the weak dependency across the rank cut, recomputed not
exchanged) and runs 2PS bands inside it.  Ranks share nothing but explicit message buffers: the
halo rows of each segment input (FP) and the delta of those rows sent back and added (BP), the
partial GAP sums and the per-rank weight gradients (summed = the all-reduce).

Training-mode BatchNorm (R24): a bn op's batch statistics cover every row
of its input, a strong dependency across all bands.  Exactly, in the order the dependencies force:
  FP statistics sweeps -- for every bn op j of a segment in op order, one band sweep computes the ops
     before j (their bn statistics are already known) and sums the rows each band computes of j's
     input (the interval rule gives every row to exactly one band): mean_j, var_j.  Then the
     ordinary FP sweep.
  BP sums sweeps -- for every bn op j in reverse op order, one reverse band sweep recomputes the band
     and back-propagates through the ops after j (their sums are known) down to the complete delta
     of j's output, summing dbeta_j = sum(da) and dgamma_j = sum(da*xh) over the band's rows of j's
     output.  Then the ordinary BP sweep, whose bn backward uses them (the textbook adjoint).
OverL (bands overlap): the statistics count each row once, in the first band that computes it; the
backward sums add every band's partial delta (linear); the bn backward's batch-statistics terms
(-gamma/sigma*(dbeta/M + xh*dgamma/M), a function of the row, not of the band's partial delta) are added
once per row, in that same first band.  Negative control: per_band_stats=True normalises every band by
its own rows' statistics.

Negative controls (must NOT match the column oracle): share=False (cached rows
replaced by zero rows -- the "padding redundancy" of Fig. 3(b)),
carry=False (2PS BP drops the delta carry), overl_average=True (the averaging
sentence of PAPER.md:339 applied on top of disjoint ownership).
"""
import numpy as np

import oracle as O
from oracle import column as C
from oracle.enumerate import segments, band_ends, enumerate_2ps, enumerate_overl


def _rows(held, t, r0, r1):
    lo, arr = held[t]
    assert r0 >= lo and r1 <= lo + arr.shape[2], ("rows not held", t, r0, r1, lo, arr.shape)
    return arr[:, :, r0 - lo:r1 - lo]


def _slab(op, held, src, a, b, h_in, share=True):
    """Input slab for output rows [a, b) and its per-side pads (semi-closed padding)."""
    k, s, p = op["k"], op["s"], op["p"]
    r0, r1 = a * s - p, (b - 1) * s - p + k
    pt, pb = max(0, -r0), max(0, r1 - h_in)
    g0, g1 = max(r0, 0), min(r1, h_in)
    lo, arr = held[src]
    if not share and g0 < lo:
        # negative control: rows another band owns are missing -> zero rows
        have = _rows(held, src, lo, g1)
        z = np.zeros(arr.shape[:2] + (lo - g0,) + arr.shape[3:])
        return np.concatenate([z, have], axis=2), (pt, pb, p, p), g0
    return _rows(held, src, g0, g1), (pt, pb, p, p), g0


def _op_rows_fwd(net, i, held, params, a, b, shp, share=True, bn=None):
    """Rows [a, b) of op i's output from held slabs.  Returns (t_rows, aux)."""
    op = net["ops"][i]
    src = op["src"]
    if op["kind"] == "bn":
        c = _rows(held, src, a, b)
        mean, var = bn[i] if bn is not None and i in bn else C.bn_stats(c)   # (no stats: per band)
        res = _rows(held, op["res"], a, b) if op["res"] >= 0 else None
        return C.bn_apply(params["convs"][i], c, mean, var, res, op["relu"]), None
    if op["kind"] == "add":
        t = _rows(held, src, a, b) + _rows(held, op["res"], a, b)
        return (np.maximum(t, 0.0) if op["relu"] else t), None
    slab, pads, _ = _slab(op, held, src, a, b, shp[src][1], share)
    if op["kind"] == "maxpool":
        y, am = O.maxpool_fwd(slab, op["k"], op["s"], pads)
        assert y.shape[2] == b - a
        return y, am
    res = _rows(held, op["res"], a, b) if op["res"] >= 0 else None
    t, c = C.conv_op_fwd(op, params["convs"][i], slab, res, pads)
    assert t.shape[2] == b - a
    return t, c


def _concat(cached, new, lo, a):
    if cached is None:
        assert lo == a
        return new
    return np.concatenate([cached, new], axis=2)


class Plan:
    """Band structure per segment, from the enumerator (not from the CUDA planner)."""

    def __init__(self, net, mode="2ps", band_rows=None, n_bands=None):
        self.net, self.mode = net, mode
        self.shp = C.out_hw(net)
        self.segs = segments(net)
        self.bands = []
        for seg in self.segs:
            h_out = self.shp[seg[2]][1]
            E = band_ends(h_out, band_rows=band_rows, n_bands=(n_bands or 1) if band_rows is None else None)
            if mode == "overl":
                self.bands.append((E, enumerate_overl(net, seg, E, self.shp)))
            else:
                self.bands.append((E, enumerate_2ps(net, seg, E, self.shp)))


def _band_range(plan, band, t):
    """(lo, a, b): buffer start, first computed row, end."""
    if plan.mode == "overl":
        lo, hi = band[t]
        return lo, lo, hi
    return band[t]


def seg_forward(plan, s, params, x_in, share=True, in_lo=0, bn=None, stop_at=None, on_rows=None):
    """FP of one segment.  Returns (full-width segment output, caches per boundary).
    x_in holds rows [in_lo, in_lo + rows) of the segment input (a rank's slab, else the full map);
    the output has the full height, rows no band computes are zero.
    bn: {op: (mean, var)} of the segment's bn ops; stop_at: compute only ops < stop_at (a bn
    statistics sweep); on_rows(t, a, rows): called with the rows [a, b) each band computes."""
    net, shp = plan.net, plan.shp
    seg_in, ids, out = plan.segs[s]
    E, bands = plan.bands[s]
    B = x_in.shape[0]
    c, h, w = shp[out]
    y = np.zeros((B, c, h, w))
    caches = []
    prev_cache = {}
    for r, band in enumerate(bands):
        held = {seg_in: (in_lo, x_in)}
        for i in ids:
            if stop_at is not None and i >= stop_at:
                continue
            t = i + 1
            lo, a, b = _band_range(plan, band, t)
            if plan.mode == "overl" and t == out:
                lo, a, b = (E[r - 1] if r else 0), (E[r - 1] if r else 0), E[r]
            new, _ = _op_rows_fwd(net, i, held, params, a, b, shp, share, bn) if b > a else \
                (np.zeros((B, shp[t][0], 0, shp[t][2])), None)
            if on_rows is not None:
                on_rows(t, a, new)
            cached = None
            if lo < a:
                clo, carr = prev_cache[t]
                cached = carr[:, :, lo - clo:a - clo] if share else np.zeros((B, shp[t][0], a - lo, shp[t][2]))
            held[t] = (lo, _concat(cached, new, lo, a))
            if t == out:
                y[:, :, a:b] = new
        cache = {}
        if plan.mode == "2ps" and r + 1 < len(bands):
            for i in ids:
                t = i + 1
                if t == out or t not in held:
                    continue
                nlo = bands[r + 1][t][0]
                lo, arr = held[t]
                b = lo + arr.shape[2]
                cache[t] = (nlo, arr[:, :, nlo - lo:b - lo].copy())
        caches.append(cache)
        prev_cache = cache
    return y, caches


def _op_rows_bwd(net, i, held, params, a, b, shp, dt, d, grads, bn=None, bns=None, own=None):
    """Backward of op i over its output rows [a, b) given complete delta dt; adds into d[...].
    bn / bns: {op: (mean, var)} and {op: (dbeta, dgamma)} of the segment's bn ops (full-map sums)."""
    op = net["ops"][i]
    src = op["src"]
    if op["kind"] == "bn":
        mean, var = bn[i]
        dbeta, dgamma = bns[i]
        t = _rows(held, i + 1, a, b)
        c = _rows(held, src, a, b)
        M = dt.shape[0] * shp[src][1] * shp[src][2]
        da = dt * (t > 0) if op["relu"] else dt
        sig = np.sqrt(var + C.BN_EPS)[None, :, None, None]
        xh = (c - mean[None, :, None, None]) / sig
        g_s = params["convs"][i]["gamma"][None, :, None, None] / sig
        stat = -g_s * (dbeta[None, :, None, None] / M + xh * dgamma[None, :, None, None] / M)
        if own is not None:   # OverL: the statistics terms once per row (rows [own0, b) of this band)
            stat[:, :, :max(0, own - a)] = 0.0
        dc = g_s * da + stat
        _add_rows(d, src, a, dc)
        if op["res"] >= 0:
            _add_rows(d, op["res"], a, da)
        return
    if op["kind"] == "add":
        t = _rows(held, i + 1, a, b)
        da = dt * (t > 0) if op["relu"] else dt
        _add_rows(d, src, a, da)
        _add_rows(d, op["res"], a, da)
        return
    slab, pads, g0 = _slab(op, held, src, a, b, shp[src][1])
    if op["kind"] == "maxpool":
        _, am = O.maxpool_fwd(slab, op["k"], op["s"], pads)
        _add_rows(d, src, g0, O.maxpool_bwd(am, dt, slab.shape[2:]))
        return
    prm = params["convs"][i]
    c = O.conv2d_fwd(slab, prm["w"], None, op["s"], pads)
    t = _rows(held, i + 1, a, b)
    dx, dres, g = C.conv_op_bwd(op, prm, slab, c, t, dt, pads, slab.shape[2:])
    for k_, v in g.items():
        grads[i][k_] = grads[i].get(k_, 0.0) + v
    _add_rows(d, src, g0, dx)
    if dres is not None:
        _add_rows(d, op["res"], a, dres)


def _add_rows(d, t, r0, v):
    lo, arr = d[t]
    arr[:, :, r0 - lo:r0 - lo + v.shape[2]] += v


def seg_backward(plan, s, params, x_in, dout, caches, carry_on=True, overl_average=False, in_lo=0,
                 bn=None, bns=None, stop_at=None, on_delta=None):
    """BP of one segment from the full-width delta of its output.  Returns (d_in, grads);
    d_in covers the same rows [in_lo, ..) as the input slab x_in.
    stop_at / on_delta: a bn sums sweep -- back-propagate through the ops after bn op stop_at and
    call on_delta(held, a, b, dt) with the complete delta rows of its output in every band."""
    net, shp = plan.net, plan.shp
    seg_in, ids, out = plan.segs[s]
    E, bands = plan.bands[s]
    B = x_in.shape[0]
    grads = {i: {} for i in ids if net["ops"][i]["kind"] == "conv"}
    for i in ids:
        if net["ops"][i]["kind"] == "bn" and bns is not None and i in bns:
            grads[i] = {"beta": bns[i][0].copy(), "gamma": bns[i][1].copy()}
    d_in = np.zeros_like(x_in)
    carry = {}
    mult = None
    if overl_average:
        mult = {}
        for band in bands:
            for t, (lo, hi) in band.items():
                m = mult.setdefault(t, np.zeros(shp[t][1]))
                m[lo:hi] += 1
    for r in range(len(bands) - 1, -1, -1):
        band = bands[r]
        held = {seg_in: (in_lo, x_in)}
        ranges = {}
        for i in ids:                                   # recompute (Alg. 1 l.17)
            t = i + 1
            lo, a, b = _band_range(plan, band, t)
            if plan.mode == "overl" and t == out:
                lo, a, b = (E[r - 1] if r else 0), (E[r - 1] if r else 0), E[r]
            ranges[t] = (lo, a, b)
            new, _ = _op_rows_fwd(net, i, held, params, a, b, shp, True, bn) if b > a else \
                (np.zeros((B, shp[t][0], 0, shp[t][2])), None)
            cached = None
            if lo < a:
                clo, carr = caches[r - 1][t]
                cached = carr[:, :, lo - clo:a - clo]
            held[t] = (lo, _concat(cached, new, lo, a))
        d = {seg_in: (in_lo, d_in)}
        for t, (lo, a, b) in ranges.items():
            if t == out:
                d[t] = (a, dout[:, :, a:b].copy())
            else:
                d[t] = (lo, np.zeros((B, shp[t][0], b - lo, shp[t][2])))
                if carry_on and t in carry:
                    clo, carr = carry[t]
                    _add_rows(d, t, clo, carr)
        for i in reversed(ids):
            if stop_at is not None and i < stop_at:
                break
            t = i + 1
            lo, a, b = ranges[t]
            if b <= a:
                continue
            dt = _rows(d, t, a, b)
            if mult is not None and t != out:
                dt = dt / mult[t][None, None, a:b, None]
            if stop_at is not None and i == stop_at:
                on_delta(held, a, b, dt)
                break
            own = None
            if plan.mode == "overl" and net["ops"][i]["kind"] == "bn" and r > 0:
                own = bands[r - 1][t][1]   # rows below the previous band's end belong to an earlier band
            _op_rows_bwd(net, i, held, params, a, b, shp, dt, d, grads, bn, bns, own)
        carry = {}
        for t, (lo, a, b) in ranges.items():
            if t != out and lo < a:
                carry[t] = (lo, _rows(d, t, lo, a).copy())
    return d_in, grads


def _bn_ops(plan, s):
    return [i for i in plan.segs[s][1] if plan.net["ops"][i]["kind"] == "bn"]


def seg_bn_stats(plan, s, params, x_in):
    """FP statistics sweeps of segment s (module docstring): {bn op: (mean, var)}."""
    net, shp = plan.net, plan.shp
    bn = {}
    for j in _bn_ops(plan, s):
        src = net["ops"][j]["src"]
        if src == plan.segs[s][0]:
            bn[j] = C.bn_stats(x_in)
            continue
        B, c, h, w = x_in.shape[0], shp[src][0], shp[src][1], shp[src][2]
        acc = {"s1": np.zeros(c), "n": 0, "rows": [], "end": 0}

        def on_rows(t, a, rows, src=src, acc=acc):
            if t == src:   # rows [a, a + n): count those no earlier band computed (OverL overlap)
                n_all = rows.shape[2]
                rows = rows[:, :, max(0, acc["end"] - a):]
                acc["end"] = max(acc["end"], a + n_all)
                acc["s1"] += rows.sum(axis=(0, 2, 3))
                acc["n"] += rows.shape[2]
                acc["rows"].append(rows)
        seg_forward(plan, s, params, x_in, bn=bn, stop_at=j, on_rows=on_rows)
        assert acc["n"] == h, ("every row of the bn input exactly once", acc["n"], h)
        M = B * h * w
        mean = acc["s1"] / M
        var = sum(((r_ - mean[None, :, None, None]) ** 2).sum(axis=(0, 2, 3)) for r_ in acc["rows"]) / M
        bn[j] = (mean, var)
    return bn


def seg_bn_sums(plan, s, params, x_in, dout, caches, bn):
    """BP sums sweeps of segment s: {bn op: (dbeta, dgamma)} (full-map sums of da, da*xh)."""
    net = plan.net
    bns = {}
    for j in reversed(_bn_ops(plan, s)):
        op = net["ops"][j]
        mean, var = bn[j]
        acc = {"s1": np.zeros(len(mean)), "s2": np.zeros(len(mean))}

        def on_delta(held, a, b, dt, j=j, op=op, mean=mean, var=var, acc=acc):
            t = _rows(held, j + 1, a, b)
            c = _rows(held, op["src"], a, b)
            da = dt * (t > 0) if op["relu"] else dt
            xh = (c - mean[None, :, None, None]) / np.sqrt(var + C.BN_EPS)[None, :, None, None]
            acc["s1"] += da.sum(axis=(0, 2, 3))
            acc["s2"] += (da * xh).sum(axis=(0, 2, 3))
        seg_backward(plan, s, params, x_in, dout, caches, bn=bn, bns=bns, stop_at=j, on_delta=on_delta)
        bns[j] = (acc["s1"], acc["s2"])
    return bns


def forward(plan, params, x, share=True, per_band_stats=False):
    """Row-centric FP over all segments: returns (z^L, checkpoints, caches); plan.bn_stats[s]
    holds the bn statistics of segment s (statistics sweeps; per_band_stats: negative control)."""
    ckpts = [np.asarray(x, dtype=np.float64)]
    allc = []
    plan.bn_stats = []
    for s in range(len(plan.segs)):
        bn = {} if per_band_stats or not _bn_ops(plan, s) else seg_bn_stats(plan, s, params, ckpts[-1])
        plan.bn_stats.append(bn)
        y, caches = seg_forward(plan, s, params, ckpts[-1], share, bn=None if per_band_stats else bn)
        ckpts.append(y)
        allc.append(caches)
    return ckpts[-1], ckpts, allc


def backward(plan, params, ckpts, allc, dzl, carry_on=True, overl_average=False):
    """Row-centric BP over all segments in reverse: returns (grads per op, d x)."""
    grads = [None] * len(plan.net["ops"])
    dout = np.asarray(dzl, dtype=np.float64)
    for s in range(len(plan.segs) - 1, -1, -1):
        bn = plan.bn_stats[s] if getattr(plan, "bn_stats", None) else {}
        bns = seg_bn_sums(plan, s, params, ckpts[s], dout, allc[s], bn) if bn else None
        dout, g = seg_backward(plan, s, params, ckpts[s], dout, allc[s], carry_on, overl_average,
                               bn=bn, bns=bns)
        for i, v in g.items():
            grads[i] = v
    return grads, dout


def step(plan, params, x, labels, lr, **kw):
    """One Alg. 1 iteration, row-centric: returns (new_params, loss, grads, head_grads, z^L)."""
    zl, ckpts, allc = forward(plan, params, x, share=kw.get("share", True),
                              per_band_stats=kw.get("per_band_stats", False))
    loss, dzl, hg, _ = C.head_forward_backward(zl, params["head"], labels)
    grads, _ = backward(plan, params, ckpts, allc, dzl, kw.get("carry_on", True),
                        kw.get("overl_average", False))
    return C.sgd(params, grads, hg, lr), loss, grads, hg, zl


# ---------------------------------------------------------------- G-rank simulation (row sharding)
class RankPlan:
    """Rank g's band structure per segment, from enumerate_rank (not from the CUDA planner):
    owned output rows own[s] = (ol, oh), extended ranges ext[s] = {t: (LO, HI)}, 2PS bands."""

    def __init__(self, net, world, g, band_rows=None, n_bands=None):
        from oracle.enumerate import enumerate_rank
        self.net, self.mode, self.world, self.g = net, "2ps", world, g
        self.shp = C.out_hw(net)
        self.segs = segments(net)
        self.bands, self.ext, self.own = [], [], []
        for seg in self.segs:
            ext, bands, own = enumerate_rank(net, seg, world, g, band_rows=band_rows,
                                             n_bands=(n_bands or 1) if band_rows is None else None, shp=self.shp)
            self.bands.append((None, bands))
            self.ext.append(ext)
            self.own.append(own)


def _messages(plans, s, seg_in):
    """Halo messages of segment s's input: (src rank, dst rank, r0, r1) for every row a rank needs
    ([LO, HI) of the input) that another rank owns (the previous segment's owned rows)."""
    msgs = []
    for g, pg in enumerate(plans):
        lo, hi = pg.ext[s][seg_in]
        for q, pq in enumerate(plans):
            if q == g:
                continue
            ol, oh = pq.own[s - 1]
            r0, r1 = max(lo, ol), min(hi, oh)
            if r1 > r0:
                msgs.append((q, g, r0, r1))
    return msgs


def forward_ranks(plans, params, x):
    """FP on G simulated ranks.  Each rank keeps only its OWNED rows of every segment output (plus
    the input slabs it assembled); returns (per-rank state, z^L owned rows per rank, messages)."""
    world = len(plans)
    state = [{"slabs": [], "caches": [], "owned": []} for _ in range(world)]
    log = []
    for s, (seg_in, ids, out) in enumerate(plans[0].segs):
        slabs = []
        if s == 0:      # the image: every rank reads its extended rows of the input batch
            for g, pg in enumerate(plans):
                lo, hi = pg.ext[s][seg_in]
                slabs.append((lo, np.asarray(x, dtype=np.float64)[:, :, lo:hi].copy()))
        else:
            msgs = _messages(plans, s, seg_in)
            log.append(("fp", s, msgs))
            for g, pg in enumerate(plans):
                lo, hi = pg.ext[s][seg_in]
                olo, own = state[g]["owned"][s - 1]
                buf = np.zeros(own.shape[:2] + (hi - lo,) + own.shape[3:])
                a, b = max(lo, olo), min(hi, olo + own.shape[2])
                if b > a:
                    buf[:, :, a - lo:b - lo] = own[:, :, a - olo:b - olo]
                for (q, dst, r0, r1) in msgs:          # receive: a copy out of the sender's owned rows
                    if dst != g:
                        continue
                    qlo, qown = state[q]["owned"][s - 1]
                    buf[:, :, r0 - lo:r1 - lo] = qown[:, :, r0 - qlo:r1 - qlo].copy()
                slabs.append((lo, buf))
        for g, pg in enumerate(plans):
            lo, slab = slabs[g]
            y, caches = seg_forward(pg, s, params, slab, in_lo=lo)
            ol, oh = pg.own[s]
            state[g]["slabs"].append((lo, slab))
            state[g]["caches"].append(caches)
            state[g]["owned"].append((ol, y[:, :, ol:oh].copy()))
    return state, [st["owned"][-1] for st in state], log


def backward_ranks(plans, params, state, dzl):
    """BP on G simulated ranks from delta^L (each rank takes its owned rows).  After each segment
    the delta a rank produced on input rows another rank owns is sent there and added.  Returns
    (per-rank grads, messages)."""
    world = len(plans)
    segs = plans[0].segs
    dz = np.asarray(dzl, dtype=np.float64)
    full_h = plans[0].shp[segs[-1][2]][1]
    dout = []
    for g, pg in enumerate(plans):     # full-height delta buffer, only owned rows set
        ol, oh = pg.own[-1]
        d = np.zeros(dz.shape[:2] + (full_h,) + dz.shape[3:])
        d[:, :, ol:oh] = dz[:, :, ol:oh]
        dout.append(d)
    grads = [[None] * len(plans[0].net["ops"]) for _ in range(world)]
    log = []
    for s in range(len(segs) - 1, -1, -1):
        seg_in, ids, out = segs[s]
        dins = []
        for g, pg in enumerate(plans):
            lo, slab = state[g]["slabs"][s]
            d_in, gr = seg_backward(pg, s, params, slab, dout[g], state[g]["caches"][s], in_lo=lo)
            dins.append((lo, d_in))
            for i, v in gr.items():
                grads[g][i] = v
        if s == 0:
            break
        msgs = _messages(plans, s, seg_in)        # FP schedule, run reversed: delta back to owners
        log.append(("bp", s, msgs))
        c, h, w = plans[0].shp[seg_in]
        new = []
        for g, pg in enumerate(plans):
            ol, oh = pg.own[s - 1]
            d = np.zeros(dz.shape[:1] + (c, h, w))
            lo, d_in = dins[g]
            a, b = max(lo, ol), min(lo + d_in.shape[2], oh)
            if b > a:
                d[:, :, a:b] += d_in[:, :, a - lo:b - lo]
            for (src, q, r0, r1) in msgs:              # q held rows [r0, r1) that g owns
                if src != g:
                    continue
                qlo, qd = dins[q]
                d[:, :, r0:r1] += qd[:, :, r0 - qlo:r1 - qlo]
            new.append(d)
        dout = new
    return grads, log


def _sum_grads(per_rank):
    """The weight-gradient all-reduce: elementwise sum over ranks."""
    out = []
    for i in range(len(per_rank[0])):
        gs = [g[i] for g in per_rank if g[i] is not None]
        if not gs:
            out.append(None)
            continue
        out.append({k: sum(g[k] for g in gs) for k in gs[0]})
    return out


def step_ranks(net, params, x, labels, lr, world, band_rows=None, n_bands=None):
    """One Alg. 1 iteration with the rows of every segment output split over `world` simulated
    ranks.  Head: z^L is the concatenation of the ranks' owned rows (Alg. 1 l.11),
    pooled as the sum of per-rank partial GAP sums.  Returns (new_params, loss, grads, head_grads,
    z^L, message log)."""
    plans = [RankPlan(net, world, g, band_rows, n_bands) for g in range(world)]
    state, owned, flog = forward_ranks(plans, params, x)
    c, h, w = plans[0].shp[plans[0].segs[-1][2]]
    zl = np.zeros((np.shape(x)[0], c, h, w))
    for (ol, rows) in owned:
        zl[:, :, ol:ol + rows.shape[2]] = rows
    loss, dzl, hg, _ = C.head_forward_backward(zl, params["head"], labels)
    per_rank, blog = backward_ranks(plans, params, state, dzl)
    grads = _sum_grads(per_rank)
    return C.sgd(params, grads, hg, lr), loss, grads, hg, zl, flog + blog


# ---------------------------------------------------------------- zero-redundancy G-rank simulation (f1)
def _zr_band_fwd(net, shp, seg, band, held_in, cache, halo, params, bn=None, stop_at=None, on_rows=None):
    """One band of a zero-redundancy rank: band[t] = (lo, a, b, hi); rows [lo, a) come from the band
    above (cache), [a, b) are computed, [b, hi) are the halo from rank g+1 (halo).  bn / stop_at /
    on_rows: as seg_forward (training-mode BN statistics sweeps)."""
    seg_in, ids, out = seg
    held = dict(held_in)
    B = held_in[seg_in][1].shape[0]
    for i in ids:
        if stop_at is not None and i >= stop_at:
            continue
        t = i + 1
        lo, a, b, hi = band[t]
        new = _op_rows_fwd(net, i, held, params, a, b, shp, True, bn)[0] if b > a else \
            np.zeros((B, shp[t][0], 0, shp[t][2]))
        if on_rows is not None:
            on_rows(t, a, new)
        parts = []
        if lo < a:
            clo, carr = cache[t]
            parts.append(carr[:, :, lo - clo:a - clo])
        parts.append(new)
        if hi > b:
            parts.append(halo[t])
        held[t] = (lo, np.concatenate(parts, axis=2))
    return held


def step_ranks_zr(net, params, x, labels, lr, world, band_rows=None, n_bands=None):
    """One Alg. 1 iteration with zero-redundancy row sharding over `world` simulated ranks (SURVEY
    8(f) f1; oracle.enumerate.enumerate_rank_zr): every row of every tensor is computed by one rank;
    rank g's last band reads the first rows of rank g+1 (a message after every rank's first band) and
    sends their delta back (a message after its first BP band, added into rank g+1's first band).
    Training-mode BN: every statistics / sums sweep is a whole sharded sweep (with its messages) and
    the per-rank sums over the rows each rank computes are added over the ranks (the all-reduce).
    Returns (new_params, loss, grads, head_grads, z^L, message log of the final sweeps)."""
    from oracle.enumerate import enumerate_rank_zr
    shp = C.out_hw(net)
    segs = segments(net)
    x = np.asarray(x, dtype=np.float64)
    B = x.shape[0]
    log = []
    plans = [[enumerate_rank_zr(net, seg, world, g, band_rows, (n_bands or 1) if band_rows is None else None, shp)
              for g in range(world)] for seg in segs]

    def seg_fp(s, full_in, bn, stop_at=None, on_rows=None, log_on=True):
        seg = segs[s]
        seg_in, ids, out = seg
        per = []
        for g in range(world):
            own, bands, _ = plans[s][g]
            r0 = min(b[seg_in][0] for b in bands)
            r1 = max(b[seg_in][3] for b in bands)
            per.append((r0, full_in[:, :, r0:r1].copy()))
        helds = [[None] * len(plans[s][g][1]) for g in range(world)]
        # band 0 of every rank (bottom rank first: with one band a rank's only band is its last)
        msgs = {}
        for g in range(world - 1, -1, -1):
            own, bands, _ = plans[s][g]
            N = len(bands)
            halo = {}
            if N == 1 and g + 1 < world:
                halo = msgs[g + 1]
            helds[g][0] = _zr_band_fwd(net, shp, seg, bands[0], {seg_in: per[g]}, {}, halo, params, bn, stop_at,
                                       on_rows)
            if g > 0:   # my first rows the rank above reads
                own_up, bands_up, _ = plans[s][g - 1]
                m = {}
                for i in ids:
                    t = i + 1
                    if t == out or t not in helds[g][0]:
                        continue
                    a0, a1 = own_up[t][1], bands_up[-1][t][3]
                    if a1 > a0:
                        lo, arr = helds[g][0][t]
                        m[t] = arr[:, :, a0 - lo:a1 - lo].copy()
                msgs[g] = m
                if log_on:
                    log.append(("fp", s, g, g - 1, sorted((t, v.shape[2]) for t, v in m.items())))
        for g in range(world):
            own, bands, _ = plans[s][g]
            for r in range(1, len(bands)):
                halo = msgs.get(g + 1, {}) if r == len(bands) - 1 else {}
                helds[g][r] = _zr_band_fwd(net, shp, seg, bands[r], {seg_in: per[g]}, helds[g][r - 1], halo, params,
                                           bn, stop_at, on_rows)
        c, h, w = shp[out]
        y = np.zeros((B, c, h, w))
        if stop_at is None:
            for g in range(world):
                own, bands, (ol, oh) = plans[s][g]
                for r, band in enumerate(bands):
                    lo, a, b, hi = band[out]
                    blo, arr = helds[g][r][out]
                    y[:, :, a:b] = arr[:, :, a - blo:b - blo]
        return y, (per, helds, msgs)

    def seg_bp(s, saved_s, dout_full, bn, bns, stop_at=None, on_delta=None, log_on=True):
        seg = segs[s]
        seg_in, ids, out = seg
        per, helds, fmsgs = saved_s
        d_ins = [np.zeros_like(per[g][1]) for g in range(world)]
        seg_grads = [{i: {} for i in ids if net["ops"][i]["kind"] == "conv"} for _ in range(world)]
        carry = [dict() for _ in range(world)]
        dmsgs = {}

        def bp_band(g, r):
            own, bands, _ = plans[s][g]
            band = bands[r]
            held = helds[g][r]
            d = {seg_in: (per[g][0], d_ins[g])}
            for i in ids:
                t = i + 1
                lo, a, b, hi = band[t]
                if t == out:
                    d[t] = (a, dout_full[:, :, a:b].copy())
                    continue
                d[t] = (lo, np.zeros((B, shp[t][0], hi - lo, shp[t][2])))
                if t in carry[g]:
                    clo, carr = carry[g][t]
                    _add_rows(d, t, clo, carr)
                if r == 0 and g > 0 and t in dmsgs.get(g - 1, {}):
                    _add_rows(d, t, own[t][0], dmsgs[g - 1][t])
            for i in reversed(ids):
                if stop_at is not None and i < stop_at:
                    break
                t = i + 1
                lo, a, b, hi = band[t]
                if b <= a:
                    continue
                if stop_at is not None and i == stop_at:
                    on_delta(held, a, b, _rows(d, t, a, b))
                    break
                _op_rows_bwd(net, i, held, params, a, b, shp, _rows(d, t, a, b), d, seg_grads[g], bn, bns)
            carry[g] = {}
            for i in ids:
                t = i + 1
                lo, a, b, hi = band[t]
                if t != out and lo < a:
                    carry[g][t] = (lo, _rows(d, t, lo, a).copy())
            if r == len(bands) - 1 and g + 1 < world:   # the delta of rank g+1's rows goes back down
                m = {}
                for i in ids:
                    t = i + 1
                    lo, a, b, hi = band[t]
                    if t != out and hi > b:
                        m[t] = _rows(d, t, b, hi).copy()
                dmsgs[g] = m
                if log_on:
                    log.append(("bp", s, g, g + 1, sorted((t, v.shape[2]) for t, v in m.items())))
        for g in range(world):                       # every rank's last band first (BP order)
            N = len(plans[s][g][1])
            for r in range(N - 1, 0, -1):
                bp_band(g, r)
        for g in range(world):                       # then every rank's first band (top rank first)
            bp_band(g, 0)
        c, h, w = shp[seg_in]
        d_full = np.zeros((B, c, h, w))
        for g in range(world):                       # the input delta back to its owners (added)
            r0 = per[g][0]
            d_full[:, :, r0:r0 + d_ins[g].shape[2]] += d_ins[g]
        return d_full, seg_grads

    def bn_ops(s):
        return [i for i in segs[s][1] if net["ops"][i]["kind"] == "bn"]

    full_in = x                      # the segment input, assembled from the owners' rows (all ranks)
    saved, bn_all = [], []
    for s in range(len(segs)):
        bn = {}
        for j in bn_ops(s):          # statistics sweeps (module docstring), summed over every rank's rows
            src = net["ops"][j]["src"]
            assert src != segs[s][0], "BN of a segment input under row sharding"
            acc = {"rows": []}

            def on_rows(t, a, rows, src=src, acc=acc):
                if t == src:
                    acc["rows"].append(rows)
            seg_fp(s, full_in, bn, stop_at=j, on_rows=on_rows, log_on=False)
            assert sum(r_.shape[2] for r_ in acc["rows"]) == shp[src][1], "every row on exactly one rank"
            M = B * shp[src][1] * shp[src][2]
            mean = sum(r_.sum(axis=(0, 2, 3)) for r_ in acc["rows"]) / M
            var = sum(((r_ - mean[None, :, None, None]) ** 2).sum(axis=(0, 2, 3)) for r_ in acc["rows"]) / M
            bn[j] = (mean, var)
        y, saved_s = seg_fp(s, full_in, bn)
        saved.append(saved_s)
        bn_all.append(bn)
        full_in = y
    zl = full_in
    loss, dzl, hg, _ = C.head_forward_backward(zl, params["head"], labels)
    grads = [None] * len(net["ops"])
    dout_full = np.asarray(dzl, dtype=np.float64)
    for s in range(len(segs) - 1, -1, -1):
        bn, bns = bn_all[s], {}
        for j in reversed(bn_ops(s)):   # sums sweeps, summed over the ranks
            op = net["ops"][j]
            mean, var = bn[j]
            acc = {"s1": np.zeros(len(mean)), "s2": np.zeros(len(mean))}

            def on_delta(held, a, b, dt, j=j, op=op, mean=mean, var=var, acc=acc):
                t = _rows(held, j + 1, a, b)
                c = _rows(held, op["src"], a, b)
                da = dt * (t > 0) if op["relu"] else dt
                xh = (c - mean[None, :, None, None]) / np.sqrt(var + C.BN_EPS)[None, :, None, None]
                acc["s1"] += da.sum(axis=(0, 2, 3))
                acc["s2"] += (da * xh).sum(axis=(0, 2, 3))
            seg_bp(s, saved[s], dout_full, bn, bns, stop_at=j, on_delta=on_delta, log_on=False)
            bns[j] = (acc["s1"], acc["s2"])
        d_full, seg_grads = seg_bp(s, saved[s], dout_full, bn, bns)
        for g in range(world):
            for i, v in seg_grads[g].items():
                if not v:
                    continue
                grads[i] = v if grads[i] is None else {k: grads[i][k] + v[k] for k in v}
        for j, (s1, s2) in bns.items():
            grads[j] = {"beta": s1.copy(), "gamma": s2.copy()}
        dout_full = d_full
    return C.sgd(params, grads, hg, lr), loss, grads, hg, zl, log

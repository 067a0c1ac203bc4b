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


def _op_rows_fwd(net, i, held, params, a, b, shp, share=True):
    """Rows [a, b) of op i's output from held slabs.  Returns (t_rows, aux)."""
    op = net["ops"][i]
    src = op["src"]
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


def seg_forward(plan, s, params, x_in, share=True):
    """FP of one segment.  Returns (full-width segment output, caches per boundary)."""
    net, shp = plan.net, plan.shp
    seg_in, ids, out = plan.segs[s]
    E, bands = plan.bands[s]
    B = x_in.shape[0]
    c, h, w = shp[out]
    y = np.zeros((B, c, h, w))
    caches = []
    prev_cache = {}
    for r, band in enumerate(bands):
        held = {seg_in: (0, x_in)}
        for i in ids:
            t = i + 1
            lo, a, b = _band_range(plan, band, t)
            if plan.mode == "overl" and t == out:
                lo, a, b = (E[r - 1] if r else 0), (E[r - 1] if r else 0), E[r]
            new, _ = _op_rows_fwd(net, i, held, params, a, b, shp, share) if b > a else \
                (np.zeros((B, shp[t][0], 0, shp[t][2])), None)
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
                if t == out:
                    continue
                nlo = bands[r + 1][t][0]
                lo, arr = held[t]
                b = lo + arr.shape[2]
                cache[t] = (nlo, arr[:, :, nlo - lo:b - lo].copy())
        caches.append(cache)
        prev_cache = cache
    return y, caches


def _op_rows_bwd(net, i, held, params, a, b, shp, dt, d, grads):
    """Backward of op i over its output rows [a, b) given complete delta dt; adds into d[...]."""
    op = net["ops"][i]
    src = op["src"]
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


def seg_backward(plan, s, params, x_in, dout, caches, carry_on=True, overl_average=False):
    """BP of one segment from the full-width delta of its output.  Returns (d_in, grads)."""
    net, shp = plan.net, plan.shp
    seg_in, ids, out = plan.segs[s]
    E, bands = plan.bands[s]
    B = x_in.shape[0]
    grads = {i: {} for i in ids if net["ops"][i]["kind"] == "conv"}
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
        held = {seg_in: (0, x_in)}
        ranges = {}
        for i in ids:                                   # recompute (Alg. 1 l.17)
            t = i + 1
            lo, a, b = _band_range(plan, band, t)
            if plan.mode == "overl" and t == out:
                lo, a, b = (E[r - 1] if r else 0), (E[r - 1] if r else 0), E[r]
            ranges[t] = (lo, a, b)
            new, _ = _op_rows_fwd(net, i, held, params, a, b, shp) if b > a else \
                (np.zeros((B, shp[t][0], 0, shp[t][2])), None)
            cached = None
            if lo < a:
                clo, carr = caches[r - 1][t]
                cached = carr[:, :, lo - clo:a - clo]
            held[t] = (lo, _concat(cached, new, lo, a))
        d = {seg_in: (0, d_in)}
        for t, (lo, a, b) in ranges.items():
            if t == out:
                d[t] = (a, dout[:, :, a:b].copy())
            else:
                d[t] = (lo, np.zeros((B, shp[t][0], b - lo, shp[t][2])))
                if carry_on and t in carry:
                    clo, carr = carry[t]
                    _add_rows(d, t, clo, carr)
        for i in reversed(ids):
            t = i + 1
            lo, a, b = ranges[t]
            if b <= a:
                continue
            dt = _rows(d, t, a, b)
            if mult is not None and t != out:
                dt = dt / mult[t][None, None, a:b, None]
            _op_rows_bwd(net, i, held, params, a, b, shp, dt, d, grads)
        carry = {}
        for t, (lo, a, b) in ranges.items():
            if t != out and lo < a:
                carry[t] = (lo, _rows(d, t, lo, a).copy())
    return d_in, grads


def forward(plan, params, x, share=True):
    """Row-centric FP over all segments: returns (z^L, checkpoints, caches)."""
    ckpts = [np.asarray(x, dtype=np.float64)]
    allc = []
    for s in range(len(plan.segs)):
        y, caches = seg_forward(plan, s, params, ckpts[-1], share)
        ckpts.append(y)
        allc.append(caches)
    return ckpts[-1], ckpts, allc


def backward(plan, params, ckpts, allc, dzl, carry_on=True, overl_average=False):
    """Row-centric BP over all segments in reverse: returns (grads per op, d x)."""
    grads = [None] * len(plan.net["ops"])
    dout = np.asarray(dzl, dtype=np.float64)
    for s in range(len(plan.segs) - 1, -1, -1):
        dout, g = seg_backward(plan, s, params, ckpts[s], dout, allc[s], carry_on, overl_average)
        for i, v in g.items():
            grads[i] = v
    return grads, dout


def step(plan, params, x, labels, lr, **kw):
    """One Alg. 1 iteration, row-centric: returns (new_params, loss, grads, head_grads, z^L)."""
    zl, ckpts, allc = forward(plan, params, x, share=kw.get("share", True))
    loss, dzl, hg, _ = C.head_forward_backward(zl, params["head"], labels)
    grads, _ = backward(plan, params, ckpts, allc, dzl, kw.get("carry_on", True),
                        kw.get("overl_average", False))
    return C.sgd(params, grads, hg, lr), loss, grads, hg, zl

"""Brute-force row-dependency enumerator -- TEST INFRASTRUCTURE ONLY.

Explicit row SETS (no closed forms) for the band/halo structure of
row-centric training.  It is the reference the planner's interval rule
 must match bit-exactly.

Definitions (PAPER.md:150 "Receptive Field", :153 row split, :287 2PS,
:330 OverL):
  * rf(op, rows_out)  = set of rows of each input read by output rows rows_out
                        (row y reads y*s-p+ky, ky<k, inside [0,H_in); padding rows are
                        not data).
  * need_r(t)          = rows of t transitively needed by the segment output rows [0, E_r).
  * 2PS band r computes rows [e_{r-1}(t), e_r(t)) of t with e_r(t) = max(need_r(t))+1
    (the interval hull from row 0), e_N(t) = H_t; its band buffer also holds the
    cached rows [lo_r(t), e_{r-1}(t)) where lo_r(t) = min(rows of t read while
    computing band r's rows of every consumer, e_{r-1}(t)).
  * OverL band r computes the hull [lo, hi) of rows transitively needed by
    the owned output rows [E_{r-1}, E_r).
Segments (2PS-H / OverL-H): a seg_end op's output is a
checkpoint; each segment is enumerated from its own input.
"""
from oracle.column import out_hw


def segments(net):
    """List of (in_tid, [op ids], out_tid); boundaries after ops with seg_end."""
    segs, cur, seg_in = [], [], 0
    ops = net["ops"]
    for i, op in enumerate(ops):
        cur.append(i)
        if op.get("seg_end") or i == len(ops) - 1:
            segs.append((seg_in, cur, i + 1))
            seg_in, cur = i + 1, []
    for seg_in, ids, out in segs:
        inside = {seg_in} | {i + 1 for i in ids}
        for i in ids:
            for key in ("src", "res"):
                t = ops[i].get(key, -1)
                if t is not None and t >= 0 and t not in inside:
                    raise ValueError("op %d reads tensor %d across a checkpoint boundary" % (i, t))
    return segs


def band_ends(h_out, band_rows=None, n_bands=None):
    """Band ends E_1<..<E_N=h_out at a segment output.
    band_rows: every band owns band_rows rows, the remainder goes to the last band.
    n_bands: near-equal split, the earliest bands take one extra row."""
    if band_rows is not None:
        E = list(range(band_rows, h_out, band_rows)) + [h_out]
        return E
    n = min(n_bands, h_out)
    q, rem = divmod(h_out, n)
    E, acc = [], 0
    for r in range(n):
        acc += q + (1 if r < rem else 0)
        E.append(acc)
    return E


def _inputs(op):
    ins = [op["src"]]
    if op.get("res", -1) is not None and op.get("res", -1) >= 0:
        ins.append(op["res"])
    return ins


def rf(op, rows_out, h_in):
    """Rows of an input read by the given output rows (explicit set enumeration)."""
    if op["kind"] in ("add", "bn"):   # pointwise (bn: its statistics are a separate sweep)
        return {y for y in rows_out if 0 <= y < h_in}
    k, s, p = op["k"], op["s"], op["p"]
    got = set()
    for y in rows_out:
        for ky in range(k):
            r = y * s - p + ky
            if 0 <= r < h_in:
                got.add(r)
    return got


def rf_of(op, tin, rows_out, h_in):
    """RF rows of input tensor tin for op (residual inputs are read 1:1)."""
    if op["kind"] == "conv" and tin == op.get("res", -1) and tin != op["src"]:
        return {y for y in rows_out if 0 <= y < h_in}
    return rf(op, rows_out, h_in)


def need_sets(net, shp, seg, out_rows):
    """Rows of every tensor of the segment transitively needed by out_rows of its output."""
    seg_in, ids, out = seg
    need = {out: set(out_rows)}
    for i in reversed(ids):
        op = net["ops"][i]
        rows = need.get(i + 1, set())
        for tin in set(_inputs(op)):
            need.setdefault(tin, set())
            need[tin] |= rf_of(op, tin, rows, shp[tin][1])
    return need


def enumerate_2ps(net, seg, E, shp=None):
    """Per band r and tensor t of the segment: (lo, a, b) with computed rows [a, b)
    and buffer rows [lo, b) (cache rows [lo, a)).  The segment input is full width."""
    shp = shp or out_hw(net)
    seg_in, ids, out = seg
    tensors = [i + 1 for i in ids]
    N = len(E)
    ends = []
    for r in range(N):
        need = need_sets(net, shp, seg, range(0, E[r]))
        e = {}
        for t in tensors:
            nt = need.get(t, set())
            e[t] = (max(nt) + 1) if nt else 0
            if r == N - 1:
                e[t] = shp[t][1]
        ends.append(e)
    res = []
    for r in range(N):
        band = {}
        for t in tensors:
            a = ends[r - 1][t] if r > 0 else 0
            band[t] = [a, a, ends[r][t]]
        # rows of each tensor read while computing band r's rows of its consumers
        for i in ids:
            op = net["ops"][i]
            _, a, b = band[i + 1]
            for tin in set(_inputs(op)):
                if tin == seg_in:
                    continue
                got = rf_of(op, tin, range(a, b), shp[tin][1])
                if got:
                    band[tin][0] = min(band[tin][0], min(got))
        res.append({t: tuple(v) for t, v in band.items()})
    return res


def enumerate_overl(net, seg, E, shp=None):
    """Per band r and tensor t: (lo, hi) hull of rows needed by owned output rows [E_{r-1}, E_r)."""
    shp = shp or out_hw(net)
    seg_in, ids, out = seg
    res = []
    for r in range(len(E)):
        a = E[r - 1] if r > 0 else 0
        need = need_sets(net, shp, seg, range(a, E[r]))
        band = {}
        for t in [seg_in] + [i + 1 for i in ids]:
            nt = need.get(t, set())
            band[t] = (min(nt), max(nt) + 1) if nt else (0, 0)
        res.append(band)
    return res


def rank_rows(h, world, g):
    """Contiguous near-equal split of h rows over `world` ranks, earliest ranks one extra row."""
    q, rem = divmod(h, world)
    lo = g * q + min(g, rem)
    return lo, lo + q + (1 if g < rem else 0)


def enumerate_rank(net, seg, world, g, band_rows=None, n_bands=None, shp=None):
    """Row sharding across ranks, enumerated with explicit row sets.

    Rank g owns rows [ol, oh) of the segment output (rank_rows).  Every tensor t of the segment
    is computed over the hull [LO, HI) of the rows transitively needed by the owned rows
    (the last rank also computes the trailing rows nobody reads, as the single-rank 2PS does).
    Inside the rank, 2PS bands over the owned rows: band r computes [e_{r-1}, e_r) with e_r the
    hull end of the rows needed by [ol, E_r), e_0 = LO, e_N = HI.  Returns
    ({t: (LO, HI)}, [{t: (lo, a, b)} per band], (ol, oh))."""
    shp = shp or out_hw(net)
    seg_in, ids, out = seg
    ol, oh = rank_rows(shp[out][1], world, g)
    need = need_sets(net, shp, seg, range(ol, oh))
    ext = {}
    for t in [seg_in] + [i + 1 for i in ids]:
        nt = need.get(t, set())
        ext[t] = (min(nt), max(nt) + 1) if nt else (0, 0)
    for i in ids:
        t = i + 1
        if t != out and (world == 1 or g == world - 1):
            ext[t] = (ext[t][0] if world > 1 else 0, shp[t][1])
    E = [ol + e for e in band_ends(oh - ol, band_rows=band_rows, n_bands=n_bands if band_rows is None else None)]
    tensors = [i + 1 for i in ids]
    ends = []
    for r in range(len(E)):
        nd = need_sets(net, shp, seg, range(ol, E[r]))
        e = {}
        for t in tensors:
            nt = nd.get(t, set())
            e[t] = (max(nt) + 1) if nt else ext[t][0]
            e[t] = max(e[t], ext[t][0])
            if r == len(E) - 1:
                e[t] = ext[t][1]
        ends.append(e)
    bands = []
    for r in range(len(E)):
        band = {}
        for t in tensors:
            a = ends[r - 1][t] if r > 0 else ext[t][0]
            band[t] = [a, a, ends[r][t]]
        for i in ids:
            op = net["ops"][i]
            _, a, b = band[i + 1]
            for tin in set(_inputs(op)):
                if tin == seg_in:
                    continue
                got = rf_of(op, tin, range(a, b), shp[tin][1])
                if got:
                    band[tin][0] = min(band[tin][0], min(got))
        bands.append({t: tuple(v) for t, v in band.items()})
    return ext, bands, (ol, oh)


def forward_split(chain, h0, in_ends):
    """Input-specified ("skewed initial partitioning") mode for a chain of convs, PAPER.md:287,
    Fig. 4: given input band ends, each band computes every output row whose RF lies in the rows
    available so far (2PS shares the earlier rows).  Returns per-layer band sizes."""
    sizes = []
    h = h0
    ends = list(in_ends)
    sizes.append([ends[0]] + [ends[i] - ends[i - 1] for i in range(1, len(ends))])
    for (k, s, p) in chain:
        h_out = (h + 2 * p - k) // s + 1
        new = []
        for r, e in enumerate(ends):
            if r == len(ends) - 1:
                new.append(h_out)
                continue
            # output rows y with all RF rows < e (rows >= h are padding only at the very end)
            cnt = 0
            for y in range(h_out):
                rows = [y * s - p + ky for ky in range(k)]
                if all(rr < e for rr in rows):
                    cnt = y + 1
            new.append(cnt)
        ends, h = new, h_out
        sizes.append([ends[0]] + [ends[i] - ends[i - 1] for i in range(1, len(ends))])
    return sizes


def enumerate_rank_zr(net, seg, world, g, band_rows=None, n_bands=None, shp=None):
    """Zero-redundancy row sharding, enumerated with explicit row sets.

    The segment output is split into contiguous rank ranges [C_g, C_{g+1}) (rank_rows).  Every row of
    every tensor t is computed by exactly ONE rank: the rank boundary of t at cut C is F_C(t) = the
    lowest row of t needed by the output rows [C, H_out) (so a rank's rows depend only on its own rows
    and on rows BELOW its range -- the weak dependency across the cut runs upward only); rank g owns
    [F_{C_g}(t), F_{C_{g+1}}(t)) (rank 0 from row 0, the last rank to H_t).  Inside the rank, 2PS bands
    over its owned output rows: band r computes [e_{r-1}(t), e_r(t)) with e_r(t) = max(F_{C_g}(t),
    1 + max row of t needed by the outputs [C_g, E_r)) for r < N-1, the last band up to the rank's
    end.  Buffers hold [lo, hi): lo = the first row the band's consumers read (2PS cache rows from the
    band above inside the rank), hi = one past the last row they read; in the last band of a rank
    rows [F_{C_{g+1}}(t), hi) belong to rank g+1 and arrive as the halo from below.

    Returns (own, bands, (ol, oh)): own = {t: (F_g, F_{g+1})} for the segment input and every tensor,
    bands = [{t: (lo, a, b, hi)} per band]."""
    shp = shp or out_hw(net)
    seg_in, ids, out = seg
    h_out = shp[out][1]
    tensors = [seg_in] + [i + 1 for i in ids]

    def cut(C):
        if C <= 0:
            return {t: 0 for t in tensors}
        if C >= h_out:
            return {t: shp[t][1] for t in tensors}
        need = need_sets(net, shp, seg, range(C, h_out))
        return {t: (min(need[t]) if need.get(t) else shp[t][1]) for t in tensors}
    ol, oh = rank_rows(h_out, world, g)
    if oh <= ol:
        raise ValueError("infeasible: fewer segment-output rows than ranks")
    top, bot = cut(ol), cut(oh)
    if g == world - 1:
        bot = {t: shp[t][1] for t in tensors}
    own = {t: (top[t], bot[t]) for t in tensors}
    E = [ol + e for e in band_ends(oh - ol, band_rows=band_rows, n_bands=n_bands if band_rows is None else None)]
    N = len(E)
    ends = []
    for r in range(N):
        e = {}
        if r == N - 1:
            e = {t: own[t][1] for t in tensors}
        else:
            nd = need_sets(net, shp, seg, range(ol, E[r]))
            for t in tensors:
                nt = nd.get(t, set())
                e[t] = max(own[t][0], (max(nt) + 1) if nt else own[t][0])
                if e[t] > own[t][1] and t != seg_in:
                    raise ValueError("infeasible: band %d of rank %d needs rows of tensor %d below its rank" % (r, g, t))
        ends.append(e)
    bands = []
    for r in range(N):
        band = {}
        for t in tensors:
            a = ends[r - 1][t] if r > 0 else own[t][0]
            band[t] = [a, a, ends[r][t], ends[r][t]]
        band[out] = [E[r - 1] if r else ol] * 2 + [E[r]] * 2
        for i in reversed(ids):
            op = net["ops"][i]
            _, a, b, _ = band[i + 1]
            for tin in set(_inputs(op)):
                got = rf_of(op, tin, range(a, b), shp[tin][1])
                if got:
                    band[tin][0] = min(band[tin][0], min(got))
                    band[tin][3] = max(band[tin][3], max(got) + 1)
        bands.append({t: tuple(v) for t, v in band.items()})
    return own, bands, (ol, oh)

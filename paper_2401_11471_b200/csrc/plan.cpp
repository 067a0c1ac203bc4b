// plan.cpp -- the row-centric planner (host, integer only).
//
// Interval rule (R3; reproduces PAPER.md Eqs. (11), (13), (14) on
// divisible chains):
//   band ends E_1 < ... < E_N = H_out at the segment output; for every other
//   tensor t of the segment, in reverse production order,
//     e_r(t) = max over consumers u with e_r(u) > 0 of
//                min(H_t, (e_r(u)-1)*s - p + k)   (window consumer)
//                e_r(u)                           (1:1 consumer: residual / ADD)
//     e_N(t) = H_t
//   band r computes rows [e_{r-1}(t), e_r(t)); its buffer also holds the 2PS
//   cache rows [lo_r(t), e_{r-1}(t)),
//     lo_r(t) = min(e_{r-1}(t), min over consumers computing rows [a,b) in band r of
//               max(0, a*s - p)  (window) | a (1:1)).
// OverL extended ranges (R4): the backward image of
// the owned output rows [E_{r-1}, E_r):
//     lo = min_u max(0, lo_u*s - p),  hi = max_u min(H_t, (hi_u-1)*s - p + k).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>

#include "plan.hpp"

namespace lrcnn {

static const size_t kAlign = 256;
static size_t align_up(size_t v) { return (v + kAlign - 1) / kAlign * kAlign; }

// Band ends at a segment output of h_out rows: band_rows > 0 -> every band owns band_rows rows
// (remainder to the last); else n_bands near-equal bands (earliest +1).  first_pm > 0 (the greedy
// first band of Eq. (12)): band 1 owns round(h_out * first_pm / 1000) rows (at
// least 1, leaving one row per other band) and the other n_bands - 1 bands split the rest.
static std::vector<int> make_band_ends(int h_out, int band_rows, int n_bands, int first_pm = 0) {
    std::vector<int> E;
    if (first_pm > 0 && band_rows <= 0 && n_bands > 1 && h_out >= 2) {
        const int n = std::max(2, std::min(n_bands, h_out));
        int h1 = (int)(((long long)h_out * first_pm + 500) / 1000);
        h1 = std::max(1, std::min(h1, h_out - (n - 1)));
        E.push_back(h1);
        const int rest = h_out - h1, q = rest / (n - 1), rem = rest % (n - 1);
        int acc = h1;
        for (int r = 0; r < n - 1; ++r) {
            acc += q + (r < rem ? 1 : 0);
            E.push_back(acc);
        }
        return E;
    }
    if (band_rows > 0) {
        for (int e = band_rows; e < h_out; e += band_rows) E.push_back(e);
        E.push_back(h_out);
        return E;
    }
    int n = std::max(1, std::min(n_bands, h_out));
    int q = h_out / n, rem = h_out % n, acc = 0;
    for (int r = 0; r < n; ++r) {
        acc += q + (r < rem ? 1 : 0);
        E.push_back(acc);
    }
    return E;
}

static bool window_role(const OpInfo &o, int role) {
    return role == 0 && o.d.kind != LRCNN_OP_ADD && o.d.kind != LRCNN_OP_BN;
}

// BP delta buffers of one segment's band, overlaid by liveness.  In the BP's reverse op order the
// delta of an internal tensor t is written first by the backward of its last consumer (dfw) and read
// last by the backward of its producer (dy of wgrad / dgrad / parameter sums).  A conv u whose
// residual input r is band-internal may read delta(out_u) again while another consumer of r runs its
// dgrad (the fused residual gradient), so delta(out_u) stays live until the first consumer of r; a
// projection output aliased to delta(out_u) (alias_delta) gets no slot of its own and keeps out_u's
// alive until its producer.  Tensors whose live intervals do not overlap share a slot (greedy interval
// colouring by first write, best fit).  assign: set dlt_off (relative to the slot area), dfw, dlr,
// dreuse.  Returns the bytes of the slot area.
static size_t delta_slots(Plan &P, const Segment &S, size_t B, size_t E, bool assign) {
    const int N = (int)S.E.size();
    std::vector<int> ts;
    std::vector<int> fw(P.t.size(), -1), lr(P.t.size(), -1);
    std::vector<size_t> bytes(P.t.size(), 0);
    for (int t : S.tensors) {
        if (t == S.out_t || alias_delta(P, S, t) >= 0) continue;
        const TensorInfo &ti = P.t[t];
        int f = ti.producer;
        for (const Consumer &c : ti.cons) f = std::max(f, c.op);
        fw[t] = f;
        lr[t] = ti.producer;
        int cap = 0;
        for (int r = 0; r < N; ++r) cap = std::max(cap, S.hb[r][t] - S.lo[r][t]);
        bytes[t] = align_up(B * std::max(cap, 1) * (size_t)ti.W * ti.Cp * E);
        ts.push_back(t);
    }
    for (int i : S.ops) {
        const OpInfo &u = P.op[i];
        if (u.d.kind != LRCNN_OP_CONV || u.d.res < 0 || fw[u.out_t] < 0) continue;
        const int r = u.d.res;
        if (r == S.in_t || r == 0) continue;
        for (const Consumer &c : P.t[r].cons) lr[u.out_t] = std::min(lr[u.out_t], c.op);
    }
    for (int t : S.tensors) {
        const int al = alias_delta(P, S, t);
        if (al >= 0 && fw[al] >= 0) lr[al] = std::min(lr[al], P.t[t].producer);
    }
    std::sort(ts.begin(), ts.end(), [&](int x, int y) { return fw[x] != fw[y] ? fw[x] > fw[y] : x < y; });
    struct Slot { size_t bytes; int last_lr; };
    std::vector<Slot> slots;
    std::vector<int> slot_of(P.t.size(), -1);
    std::vector<bool> reuse(P.t.size(), false);
    for (int t : ts) {
        int best = -1;
        for (int k = 0; k < (int)slots.size(); ++k) {
            if (slots[k].last_lr <= fw[t]) continue;                     // still live at t's first write
            if (best < 0) { best = k; continue; }
            const bool fits = slots[k].bytes >= bytes[t], bfits = slots[best].bytes >= bytes[t];
            if (fits != bfits ? fits : (fits ? slots[k].bytes < slots[best].bytes : slots[k].bytes > slots[best].bytes))
                best = k;
        }
        if (best < 0) { slots.push_back({bytes[t], lr[t]}); best = (int)slots.size() - 1; }
        else { slots[best].bytes = std::max(slots[best].bytes, bytes[t]); slots[best].last_lr = lr[t]; reuse[t] = true; }
        slot_of[t] = best;
    }
    std::vector<size_t> off(slots.size(), 0);
    size_t total = 0;
    for (size_t k = 0; k < slots.size(); ++k) { off[k] = total; total += slots[k].bytes; }
    if (assign) {
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            TensorInfo &ti = P.t[t];
            ti.dfw = fw[t]; ti.dlr = lr[t]; ti.dreuse = reuse[t];
            ti.dlt_off = slot_of[t] >= 0 ? off[slot_of[t]] : 0;
        }
    }
    return total;
}

lrcnn_status build_plan(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, Plan &P, std::string &err) {
    if (!net || !opts || !net->ops || net->n_ops < 1) { err = "null net/opts or no ops"; return LRCNN_E_ARG; }
    if (net->B < 1 || net->C < 1 || net->H < 1 || net->W < 1 || net->n_classes < 1) {
        err = "batch/image/classes must be >= 1"; return LRCNN_E_SHAPE;
    }
    if (opts->mode < LRCNN_COLUMN || opts->mode > LRCNN_OVERL) { err = "bad mode"; return LRCNN_E_ARG; }
    if (opts->prec != LRCNN_FP32 && opts->prec != LRCNN_BF16) { err = "bad precision"; return LRCNN_E_ARG; }
    if (opts->mode != LRCNN_COLUMN && opts->band_rows <= 0 && opts->n_bands <= 0) {
        err = "band_rows or n_bands must be > 0"; return LRCNN_E_ARG;
    }
    P.net = *net;
    P.ops_copy.assign(net->ops, net->ops + net->n_ops);
    P.net.ops = P.ops_copy.data();
    P.opts = *opts;
    P.elem = opts->prec == LRCNN_BF16 ? 2 : 4;
    const int n_ops = net->n_ops, T = n_ops + 1;
    P.t.assign(T, TensorInfo());
    P.op.assign(n_ops, OpInfo());
    P.t[0].C = net->C; P.t[0].Cp = round_up(net->C, 8); P.t[0].H = net->H; P.t[0].W = net->W;
    P.t[0].seg_in = true;

    // ---------------------------------------------------------------- shapes
    for (int i = 0; i < n_ops; ++i) {
        const lrcnn_op &d = P.ops_copy[i];
        OpInfo &o = P.op[i];
        o.d = d; o.in_t = d.src; o.out_t = i + 1;
        if (d.src < 0 || d.src > i) { err = "op " + std::to_string(i) + ": src must be an earlier tensor"; return LRCNN_E_ARG; }
        if (d.res > i || d.res < -1) { err = "op " + std::to_string(i) + ": bad res"; return LRCNN_E_ARG; }
        const TensorInfo &in = P.t[d.src];
        TensorInfo &out = P.t[i + 1];
        out.producer = i;
        if (d.kind == LRCNN_OP_CONV || d.kind == LRCNN_OP_MAXPOOL) {
            if (d.k < 1 || d.s < 1 || d.p < 0 || d.p >= d.k) { err = "op " + std::to_string(i) + ": need k>=1, s>=1, 0<=p<k"; return LRCNN_E_SHAPE; }
            int ho = out_dim(in.H, d.k, d.s, d.p), wo = out_dim(in.W, d.k, d.s, d.p);
            if (ho < 1 || wo < 1) { err = "op " + std::to_string(i) + ": kernel exceeds input (PAPER.md:218)"; return LRCNN_E_SHAPE; }
            out.H = ho; out.W = wo;
            if (d.kind == LRCNN_OP_CONV) {
                if (d.c_out < 1) { err = "conv c_out < 1"; return LRCNN_E_SHAPE; }
                if (d.epi < LRCNN_EPI_NONE || d.epi > LRCNN_EPI_AFFINE) { err = "bad epi"; return LRCNN_E_ARG; }
                out.C = d.c_out;
                out.relu = d.relu ? 1 : 0;
                if (d.res >= 0) {
                    const TensorInfo &r = P.t[d.res];
                    if (r.C != out.C || r.H != out.H || r.W != out.W) { err = "conv residual shape mismatch"; return LRCNN_E_SHAPE; }
                }
            } else {
                if (d.res >= 0) { err = "maxpool has no residual"; return LRCNN_E_ARG; }
                out.C = in.C; out.relu = 0;
            }
        } else if (d.kind == LRCNN_OP_ADD || d.kind == LRCNN_OP_BN) {
            if (d.kind == LRCNN_OP_ADD && d.res < 0) { err = "add needs res"; return LRCNN_E_ARG; }
            if (d.res >= 0) {
                const TensorInfo &r = P.t[d.res];
                if (r.C != in.C || r.H != in.H || r.W != in.W) { err = "add / bn residual shape mismatch"; return LRCNN_E_SHAPE; }
            }
            out.C = in.C; out.H = in.H; out.W = in.W; out.relu = d.relu ? 1 : 0;
            if (d.kind == LRCNN_OP_BN) {
                // training-mode BN (f4): the statistics sweeps need disjoint band rows on one full map
                // row sharding: the batch statistics are all-reduced over the ranks, so every row must be
                // computed by exactly one rank -- zero-redundancy cuts only (OverL cuts recompute rows)
                if (opts->world > 1 && !(opts->flags & (LRCNN_FLAG_DP | LRCNN_FLAG_ZERO_REDUNDANCY))) {
                    err = "training-mode BN with row sharding needs LRCNN_FLAG_ZERO_REDUNDANCY (OverL cuts recompute rows)";
                    return LRCNN_E_UNSUPPORTED;
                }
            }
        } else { err = "bad op kind"; return LRCNN_E_ARG; }
        out.Cp = round_up(out.C, 8);
        P.t[d.src].cons.push_back({i, 0});
        if (d.res >= 0) P.t[d.res].cons.push_back({i, 1});
    }
    P.t[n_ops].is_zl = true;

    // ---------------------------------------------------------------- segments
    if ((opts->flags & LRCNN_FLAG_AUTO_SEGMENTS) && opts->mode != LRCNN_COLUMN) {
        // sqrt(n) checkpointing (PAPER.md:394 OverL-H / 2PS-H "determine the optimal checkpoint
        // locations ... Ref. [34]", "a preferred checkpointing frequency is sqrt(n)"):
        // the net's seg_end flags are replaced by ceil(sqrt(n)) - 1 checkpoints, n = number of ops,
        // each at the valid cut (an op output no other tensor reaches past) nearest to j * n / sqrt(n)
        std::vector<int> last_use(T, -1);
        for (int i = 0; i < n_ops; ++i) {
            last_use[P.ops_copy[i].src] = std::max(last_use[P.ops_copy[i].src], i);
            if (P.ops_copy[i].res >= 0) last_use[P.ops_copy[i].res] = std::max(last_use[P.ops_copy[i].res], i);
        }
        std::vector<int> cuts;   // op i is a valid cut iff every tensor t <= i is last read at op <= i, except t = i + 1
        int reach = -1;
        for (int i = 0; i < n_ops - 1; ++i) {
            reach = std::max(reach, last_use[i]);          // tensor i (produced by op i - 1, or the image)
            if (reach <= i) cuts.push_back(i);
        }
        for (auto &o : P.ops_copy) o.seg_end = 0;
        const int m = (int)std::ceil(std::sqrt((double)n_ops)) - 1;
        int prev = -1;
        for (int j = 1; j <= m && !cuts.empty(); ++j) {
            const double target = (double)j * n_ops / (m + 1) - 1;
            int best = -1;
            for (int c : cuts)
                if (c > prev && (best < 0 || std::fabs(c - target) < std::fabs(best - target))) best = c;
            if (best < 0) break;
            P.ops_copy[best].seg_end = 1;
            prev = best;
        }
        P.net.ops = P.ops_copy.data();
        for (int i = 0; i < n_ops; ++i) P.op[i].d.seg_end = P.ops_copy[i].seg_end;
    }
    {
        Segment cur; cur.in_t = 0;
        for (int i = 0; i < n_ops; ++i) {
            cur.ops.push_back(i);
            bool end = (i == n_ops - 1) || (opts->mode != LRCNN_COLUMN && P.ops_copy[i].seg_end);
            if (end) { cur.out_t = i + 1; P.seg.push_back(cur); cur = Segment(); cur.in_t = i + 1; }
        }
    }
    for (size_t s = 0; s < P.seg.size(); ++s) {
        Segment &S = P.seg[s];
        std::vector<char> inside(T, 0);
        inside[S.in_t] = 1;
        for (int i : S.ops) inside[i + 1] = 1;
        for (int i : S.ops) {
            const lrcnn_op &d = P.ops_copy[i];
            if (!inside[d.src] || (d.res >= 0 && !inside[d.res])) {
                err = "op " + std::to_string(i) + " reads a tensor across a checkpoint boundary"; return LRCNN_E_ARG;
            }
            P.t[i + 1].seg = (int)s;
            S.tensors.push_back(i + 1);
        }
        P.t[S.out_t].seg_out = true;
        P.t[S.in_t].seg_in = true;
        // every internal tensor needs a consumer inside the segment
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            bool has = false;
            for (auto &c : P.t[t].cons) if (inside[c.op + 1]) has = true;
            if (!has) { err = "tensor " + std::to_string(t) + " has no consumer in its segment"; return LRCNN_E_ARG; }
            for (auto &c : P.t[t].cons)
                if (!inside[c.op + 1]) { err = "tensor " + std::to_string(t) + " is read across a checkpoint"; return LRCNN_E_ARG; }
        }
    }

    // ---------------------------------------------------------------- rank shards
    // Row sharding across `world` ranks (SURVEY 8(e) "per-stage segments, OverL at rank cuts,
    // 2PS bands inside each rank"): each segment output is split into near-equal contiguous row
    // ranges (earliest ranks +1); a rank computes every tensor of the segment over the backward
    // image [LO, HI) of its owned output rows (the OverL extended range, R4), so its only
    // dependency on other ranks is the halo of the segment input, exchanged once per segment.
    const int world = std::max(1, opts->world), rank = opts->rank;
    if (rank < 0 || rank >= world) { err = "rank out of range"; return LRCNN_E_ARG; }
    auto split = [&](int h, int g, int &lo, int &hi) {
        int q = h / world, rem = h % world;
        lo = g * q + std::min(g, rem);
        hi = lo + q + (g < rem ? 1 : 0);
    };
    // extended ranges of every tensor of segment S for owned output rows [ol, oh)
    auto ext = [&](const Segment &S, int ol, int oh, std::vector<int> &LO, std::vector<int> &HI) {
        LO.assign(T, 0); HI.assign(T, 0);
        std::vector<char> inside(T, 0);
        for (int i : S.ops) inside[i + 1] = 1;
        LO[S.out_t] = ol; HI[S.out_t] = oh;
        std::vector<int> order(S.tensors.rbegin(), S.tensors.rend());
        order.push_back(S.in_t);
        for (int t : order) {
            if (t == S.out_t) continue;
            int lo = INT_MAX, hi = 0;
            for (auto &c : P.t[t].cons) {
                if (!inside[c.op + 1]) continue;
                const OpInfo &o = P.op[c.op];
                int lu = LO[c.op + 1], hu = HI[c.op + 1];
                if (hu <= lu) continue;
                int l, h;
                if (window_role(o, c.role)) {
                    l = std::max(0, lu * o.d.s - o.d.p);
                    h = std::min(P.t[t].H, (hu - 1) * o.d.s - o.d.p + o.d.k);
                } else { l = lu; h = hu; }
                lo = std::min(lo, l); hi = std::max(hi, h);
            }
            if (hi <= 0 || lo == INT_MAX) { lo = 0; hi = 0; }
            LO[t] = lo; HI[t] = hi;
        }
    };
    // Zero-redundancy sharding (LRCNN_FLAG_ZERO_REDUNDANCY): every row of every tensor
    // is computed by ONE rank.  The rank boundary of tensor t at output cut C is F_C(t), the lowest row
    // of t the outputs [C, H_out) need (the 2PS interval rule run from the bottom: F(out) = C,
    // F(t) = min over consumers u of max(0, F(u) s - p)); rank g owns [F_{C_g}(t), F_{C_{g+1}}(t)).
    // A rank's rows then depend only on its own rows and on rows BELOW its range (the weak dependency
    // across the cut, runs upward only): its last band reads a few rows of every tensor
    // that rank g+1 computes in its FIRST band -- no recomputation, one halo message per tensor per
    // pass, and no rank waits for another's whole sweep.
    const bool zr = world > 1 && (opts->flags & LRCNN_FLAG_ZERO_REDUNDANCY) && opts->mode == LRCNN_2PS;
    auto cutF = [&](const Segment &S, int C, std::vector<int> &F) {
        F.assign(T, 0);
        std::vector<char> inside(T, 0);
        for (int i : S.ops) inside[i + 1] = 1;
        F[S.out_t] = std::min(C, P.t[S.out_t].H);
        std::vector<int> order(S.tensors.rbegin(), S.tensors.rend());
        order.push_back(S.in_t);
        for (int t : order) {
            if (t == S.out_t) continue;
            int f = INT_MAX;
            for (auto &c : P.t[t].cons) {
                if (!inside[c.op + 1]) continue;
                const OpInfo &o = P.op[c.op];
                const int fu = F[c.op + 1];
                if (fu >= P.t[c.op + 1].H) continue;   // that consumer needs no row at or below the cut
                f = std::min(f, window_role(o, c.role) ? std::max(0, fu * o.d.s - o.d.p) : fu);
            }
            F[t] = f == INT_MAX ? P.t[t].H : std::min(f, P.t[t].H);
        }
    };
    auto zr_ext = [&](const Segment &S, int g, std::vector<int> &LO, std::vector<int> &HI) {
        int ol, oh;
        split(P.t[S.out_t].H, g, ol, oh);
        std::vector<int> Ft, Fb;
        cutF(S, ol, Ft);
        cutF(S, oh, Fb);
        LO.assign(T, 0); HI.assign(T, 0);
        for (int t : S.tensors) {
            LO[t] = g == 0 ? 0 : Ft[t];
            HI[t] = g == world - 1 ? P.t[t].H : Fb[t];
        }
        LO[S.out_t] = ol; HI[S.out_t] = oh;
        int rl = INT_MAX, rb = 0;   // the segment input: the rows this rank's ops read
        std::vector<char> inside(T, 0);
        for (int i : S.ops) inside[i + 1] = 1;
        for (auto &c : P.t[S.in_t].cons) {
            if (!inside[c.op + 1]) continue;
            const OpInfo &o = P.op[c.op];
            const int lu = LO[c.op + 1], hu = HI[c.op + 1];
            if (hu <= lu) continue;
            const bool w = window_role(o, c.role);
            rl = std::min(rl, w ? std::max(0, lu * o.d.s - o.d.p) : lu);
            rb = std::max(rb, w ? std::min(P.t[S.in_t].H, (hu - 1) * o.d.s - o.d.p + o.d.k) : hu);
        }
        LO[S.in_t] = rl == INT_MAX ? 0 : rl;
        HI[S.in_t] = rb;
    };
    for (size_t si = 0; si < P.seg.size(); ++si) {
        Segment &S = P.seg[si];
        if (P.t[S.out_t].H < world) { err = "fewer segment-output rows than ranks"; return LRCNN_E_INFEASIBLE; }
        split(P.t[S.out_t].H, rank, S.own_lo, S.own_hi);
        split(P.t[S.in_t].H, rank, S.in_own_lo, S.in_own_hi);
        if (si > 0) { S.in_own_lo = P.seg[si - 1].own_lo; S.in_own_hi = P.seg[si - 1].own_hi; }
        if (zr) zr_ext(S, rank, S.LO, S.HI);
        else {
            ext(S, S.own_lo, S.own_hi, S.LO, S.HI);
            if (world > 1 && rank == world - 1)
                for (int t : S.tensors) if (t != S.out_t) S.HI[t] = P.t[t].H;   // last rank: all trailing rows
            if (world == 1)
                for (int t : S.tensors) if (t != S.out_t) { S.LO[t] = 0; S.HI[t] = P.t[t].H; }
        }
        if (world > 1 && S.in_t != 0) {
            // halo of the segment input from the neighbours; must come from adjacent ranks only
            for (int d = -1; d <= 1; d += 2) {
                const int g = rank + d;
                if (g < 0 || g >= world) continue;
                int gol, goh;
                split(P.t[S.out_t].H, g, gol, goh);
                std::vector<int> LOg, HIg;
                if (zr) zr_ext(S, g, LOg, HIg);
                else ext(S, gol, goh, LOg, HIg);
                int pl, ph;   // rows of the input tensor rank g owns (its previous-segment output split)
                split(P.t[S.in_t].H, g, pl, ph);
                // FP: what I need from g / what g needs from me
                if (d < 0) {
                    if (S.LO[S.in_t] < S.in_own_lo) S.in_xfers.push_back({g, 0, S.LO[S.in_t], S.in_own_lo});
                    if (HIg[S.in_t] > S.in_own_lo) S.in_xfers.push_back({g, 1, S.in_own_lo, HIg[S.in_t]});
                    if (S.LO[S.in_t] < pl) { err = "halo wider than a neighbour's shard"; return LRCNN_E_INFEASIBLE; }
                } else {
                    if (S.HI[S.in_t] > S.in_own_hi) S.in_xfers.push_back({g, 0, S.in_own_hi, S.HI[S.in_t]});
                    if (LOg[S.in_t] < S.in_own_hi) S.in_xfers.push_back({g, 1, LOg[S.in_t], S.in_own_hi});
                    if (S.HI[S.in_t] > ph) { err = "halo wider than a neighbour's shard"; return LRCNN_E_INFEASIBLE; }
                }
            }
        }
    }

    // ---------------------------------------------------------------- bands
    // rows of every tensor of segment S for its band ends (nb > 0: nb near-equal bands)
    auto make_bands = [&](Segment &S, int nb) -> lrcnn_status {
        const int own = S.own_hi - S.own_lo;
        if (opts->mode == LRCNN_COLUMN) S.E = {S.own_hi};
        else {
            S.E = nb > 0 ? make_band_ends(own, 0, nb, opts->first_rows_pm)
                         : make_band_ends(own, opts->band_rows, opts->n_bands, opts->first_rows_pm);
            for (int &e : S.E) e += S.own_lo;
        }
        for (size_t r = 1; r < S.E.size(); ++r)
            if (S.E[r] <= S.E[r - 1]) { err = "band ends not strictly increasing"; return LRCNN_E_DEGENERATE; }
        const int N = (int)S.E.size();
        S.lo.assign(N, std::vector<int>(T, 0));
        S.a = S.lo; S.b = S.lo;
        std::vector<char> inside(T, 0);
        for (int i : S.ops) inside[i + 1] = 1;
        if (opts->mode == LRCNN_OVERL) {
            for (int r = 0; r < N; ++r) {
                int e0 = r ? S.E[r - 1] : S.own_lo;
                S.lo[r][S.out_t] = S.a[r][S.out_t] = e0; S.b[r][S.out_t] = S.E[r];
                // internal tensors and the segment input, reverse production order
                std::vector<int> order(S.tensors.rbegin(), S.tensors.rend());
                order.push_back(S.in_t);
                for (int t : order) {
                    if (t == S.out_t) continue;
                    int lo = INT_MAX, hi = 0;
                    for (auto &c : P.t[t].cons) {
                        if (!inside[c.op + 1]) continue;
                        const OpInfo &o = P.op[c.op];
                        int lu = S.lo[r][c.op + 1], hu = S.b[r][c.op + 1];
                        if (hu <= lu) continue;
                        int l, h;
                        if (window_role(o, c.role)) {
                            l = std::max(0, lu * o.d.s - o.d.p);
                            h = std::min(P.t[t].H, (hu - 1) * o.d.s - o.d.p + o.d.k);
                        } else { l = lu; h = hu; }
                        lo = std::min(lo, l); hi = std::max(hi, h);
                    }
                    if (hi <= 0 || lo == INT_MAX) { lo = 0; hi = 0; }
                    S.lo[r][t] = S.a[r][t] = lo; S.b[r][t] = hi;
                }
            }
            int ov = 0;
            for (int r = 0; r + 1 < N; ++r) ov = std::max(ov, S.b[r][S.in_t] - S.lo[r + 1][S.in_t]);
            S.overlap_in = ov;
            if (N > 1 && ov > 0 && (long)N * ov > P.t[S.in_t].H && !(opts->flags & LRCNN_FLAG_ALLOW_OVERLAP_EXHAUSTION)) {
                err = "OverL: N > H/o^0 at a segment input (PAPER.md:391-392)"; return LRCNN_E_INFEASIBLE;
            }
        } else {
            for (int r = 0; r < N; ++r) {
                S.b[r][S.out_t] = S.E[r];
                for (auto it = S.tensors.rbegin(); it != S.tensors.rend(); ++it) {
                    int t = *it;
                    if (t == S.out_t) continue;
                    int e = S.LO[t];
                    if (r == N - 1) e = S.HI[t];
                    else {
                        for (auto &c : P.t[t].cons) {
                            const OpInfo &o = P.op[c.op];
                            int eu = S.b[r][c.op + 1];
                            if (eu <= S.LO[c.op + 1]) continue;   // consumer computed nothing yet
                            int need = window_role(o, c.role) ? (eu - 1) * o.d.s - o.d.p + o.d.k : eu;
                            e = std::max(e, std::min(S.HI[t], need));
                        }
                    }
                    S.b[r][t] = e;
                }
                for (int t : S.tensors) S.a[r][t] = r ? S.b[r - 1][t] : S.LO[t];
                for (int t : S.tensors) {
                    int lo = S.a[r][t];
                    if (t != S.out_t) {
                        for (auto &c : P.t[t].cons) {
                            const OpInfo &o = P.op[c.op];
                            int au = S.a[r][c.op + 1], bu = S.b[r][c.op + 1];
                            if (bu <= au) continue;
                            int first = window_role(o, c.role) ? std::max(0, au * o.d.s - o.d.p) : au;
                            if (first < P.t[t].H) lo = std::min(lo, first);
                        }
                    }
                    S.lo[r][t] = lo;
                }
                for (int t : S.tensors)
                    if (S.b[r][t] < S.a[r][t]) { err = "non-monotone band ends"; return LRCNN_E_DEGENERATE; }
            }
        }
        return LRCNN_OK;
    };
    const size_t Bsz = net->B, Esz = P.elem;
    // band working set of a segment: act + delta buffers of its internal tensors + 2PS carries
    auto seg_arena = [&](const Segment &S) {
        size_t a = 0;
        const int N = (int)S.E.size();
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            int cap = 0, ccap = 0;
            for (int r = 0; r < N; ++r) {
                cap = std::max(cap, S.hb[r][t] - S.lo[r][t]);
                ccap = std::max(ccap, S.a[r][t] - S.lo[r][t]);
            }
            const size_t rb = (size_t)P.t[t].W * P.t[t].Cp * Esz;
            a += align_up(Bsz * std::max(cap, 1) * rb);
            if (ccap > 0 && opts->mode == LRCNN_2PS) a += align_up(Bsz * ccap * rb);
        }
        return a + delta_slots(P, S, Bsz, Esz, false);
    };
    for (Segment &S : P.seg) {
        lrcnn_status st = make_bands(S, 0);
        if (st != LRCNN_OK) return st;
    }
    // buffer ends: one past the last row of t the consumers' computed rows read (== b except in the
    // last band of a zero-redundancy rank, whose reads reach into rank g+1's first rows)
    auto band_reads = [&](Segment &S) {
        const int N = (int)S.E.size();
        S.hb = S.b;
        for (int r = 0; r < N; ++r)
            for (int i : S.ops) {
                const OpInfo &o = P.op[i];
                const int u = o.out_t, au = S.a[r][u], bu = S.b[r][u];
                if (bu <= au) continue;
                for (int role = 0; role < 2; ++role) {
                    const int tin = role == 0 ? o.d.src : o.d.res;
                    if (tin < 0 || tin == S.in_t) continue;
                    const bool w = window_role(o, role);
                    const int h = w ? std::min(P.t[tin].H, (bu - 1) * o.d.s - o.d.p + o.d.k) : bu;
                    S.hb[r][tin] = std::max(S.hb[r][tin], h);
                }
            }
    };
    if (zr) {
        // bands inside each rank as planned (no balanced / merged variants: every rank must know its
        // neighbours' band structure exactly), then the halo schedule with ranks g-1 and g+1
        for (size_t si = 0; si < P.seg.size(); ++si) {
            Segment &S = P.seg[si];
            band_reads(S);
            const int N = (int)S.E.size();
            for (int r = 0; r + 1 < N; ++r)
                for (int t : S.tensors)
                    if (t != S.out_t && S.hb[r][t] > S.b[r][t]) {
                        err = "zero-redundancy: band " + std::to_string(r) + " reads past its rank's rows (use fewer bands)";
                        return LRCNN_E_INFEASIBLE;
                    }
            auto neighbour = [&](int g, Segment &Q) -> lrcnn_status {
                Q = S;
                split(P.t[S.out_t].H, g, Q.own_lo, Q.own_hi);
                zr_ext(S, g, Q.LO, Q.HI);
                lrcnn_status st2 = make_bands(Q, 0);
                if (st2 != LRCNN_OK) return st2;
                band_reads(Q);
                return LRCNN_OK;
            };
            S.zr_from_below.clear(); S.zr_to_above.clear();
            if (rank + 1 < world) {   // my last band's halo from below: computed by rank+1's band 0
                if (N < 2) { err = "zero-redundancy needs >= 2 bands on every rank but the last"; return LRCNN_E_INFEASIBLE; }
                Segment Q;
                const lrcnn_status stq = neighbour(rank + 1, Q);
                if (stq != LRCNN_OK) return stq;
                for (int t : S.tensors) {
                    if (t == S.out_t) continue;
                    const int r0 = S.HI[t], r1 = S.hb[N - 1][t];
                    if (r1 <= r0) continue;
                    if (r1 > Q.b[0][t] || r1 > Q.HI[t]) {
                        err = "zero-redundancy: halo deeper than rank " + std::to_string(rank + 1) + "'s first band";
                        return LRCNN_E_INFEASIBLE;
                    }
                    S.zr_from_below.push_back({t, r0, r1});
                }
            }
            if (rank > 0) {           // rank-1's last band reads my first rows
                Segment Q;
                const lrcnn_status stq = neighbour(rank - 1, Q);
                if (stq != LRCNN_OK) return stq;
                const int NQ = (int)Q.E.size();
                for (int t : S.tensors) {
                    if (t == S.out_t) continue;
                    const int r0 = Q.HI[t], r1 = Q.hb[NQ - 1][t];
                    if (r1 > r0) S.zr_to_above.push_back({t, r0, r1});
                }
            }
        }
    } else {
        for (Segment &S : P.seg) band_reads(S);
    }
    if ((opts->flags & LRCNN_FLAG_BALANCED_BANDS) && opts->mode != LRCNN_COLUMN && !zr) {
        size_t budget = 0;
        for (const Segment &S : P.seg) budget = std::max(budget, seg_arena(S));
        for (Segment &S : P.seg) {
            const int n0 = (int)S.E.size();
            for (int nb = 1; nb < n0; ++nb) {
                Segment T2 = S;
                if (make_bands(T2, nb) != LRCNN_OK) continue;
                band_reads(T2);
                if (seg_arena(T2) <= budget) { S = T2; break; }
            }
        }
    }

    // ---------------------------------------------------------------- parameters
    size_t off = 0;
    auto take = [&](size_t n) { size_t o = off; off += (n + 7) / 8 * 8; return o; };
    for (int i = 0; i < n_ops; ++i) {
        OpInfo &o = P.op[i];
        if (o.d.kind == LRCNN_OP_BN) {   // gamma, beta (b_off / beta_off as for an affine conv)
            o.b_cnt = P.t[o.out_t].C; o.b_off = take(o.b_cnt);
            o.beta_cnt = P.t[o.out_t].C; o.beta_off = take(o.beta_cnt);
            continue;
        }
        if (o.d.kind != LRCNN_OP_CONV) continue;
        o.w_cnt = (size_t)o.d.c_out * o.d.k * o.d.k * P.t[o.in_t].Cp;
        o.w_off = take(o.w_cnt);
        if (o.d.epi == LRCNN_EPI_BIAS) { o.b_cnt = o.d.c_out; o.b_off = take(o.b_cnt); }
        if (o.d.epi == LRCNN_EPI_AFFINE) {
            o.b_cnt = o.d.c_out; o.b_off = take(o.b_cnt);
            o.beta_cnt = o.d.c_out; o.beta_off = take(o.beta_cnt);
        }
    }
    const TensorInfo &zl = P.t[n_ops];
    P.head_w_cnt = (size_t)net->n_classes * zl.Cp; P.head_w_off = take(P.head_w_cnt);
    P.head_b_cnt = net->n_classes; P.head_b_off = take(P.head_b_cnt);
    P.n_params = off;

    // ---------------------------------------------------------------- workspace
    const size_t B = net->B, E = P.elem;
    auto rowbytes = [&](int t) { return (size_t)P.t[t].W * P.t[t].Cp * E; };
    size_t ws = 0;
    auto alloc = [&](size_t bytes) { size_t o = ws; ws = align_up(ws + bytes); return o; };
    lrcnn_memory_report &M = P.mem;
    std::memset(&M, 0, sizeof(M));
    for (int t = 1; t < T; ++t) M.omega += B * P.t[t].H * P.t[t].W * P.t[t].C * E;
    // rows every full-width (boundary) map holds on this rank: image = all rows (caller's x);
    // a checkpoint = its owned rows plus the next segment's halo; z^L = owned rows
    P.t[0].ck_lo = 0; P.t[0].ck_rows = P.t[0].H;
    for (size_t si = 0; si < P.seg.size(); ++si) {
        const Segment &S = P.seg[si];
        TensorInfo &to = P.t[S.out_t];
        int lo = S.own_lo, hi = S.own_hi;
        if (si + 1 < P.seg.size()) {
            lo = std::min(lo, P.seg[si + 1].LO[S.out_t]);
            hi = std::max(hi, P.seg[si + 1].HI[S.out_t]);
        }
        to.ck_lo = lo; to.ck_rows = hi - lo;
        to.dl_lo = lo; to.dl_rows = hi - lo;
    }
    // persistent: checkpoints, 2PS caches, delta ping-pong, head scratch, transposed weights
    for (const Segment &S : P.seg) {
        if (!P.t[S.out_t].is_zl) {
            P.t[S.out_t].ckpt_off = alloc(B * P.t[S.out_t].ck_rows * rowbytes(S.out_t));
            M.checkpoints += B * P.t[S.out_t].ck_rows * rowbytes(S.out_t);
        }
        const int N = (int)S.E.size();
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            TensorInfo &ti = P.t[t];
            ti.cache_lo.assign(std::max(0, N - 1), 0);
            ti.cache_rows.assign(std::max(0, N - 1), 0);
            ti.cache_off.assign(std::max(0, N - 1), 0);
            if (opts->mode != LRCNN_2PS) continue;
            for (int r = 0; r + 1 < N; ++r) {
                int nlo = S.lo[r + 1][t], e = S.b[r][t];
                ti.cache_lo[r] = nlo;
                ti.cache_rows[r] = std::max(0, e - nlo);
                if (ti.cache_rows[r] > 0) {
                    ti.cache_off[r] = alloc(B * ti.cache_rows[r] * rowbytes(t));
                    M.halo_cache += B * ti.cache_rows[r] * rowbytes(t);
                }
            }
        }
    }
    // zero-redundancy halo buffers (persistent from FP to BP): the rows from below (activations in,
    // their delta out) and my first rows the rank above reads (activations out, their delta in)
    for (Segment &S : P.seg) {
        for (auto &z : S.zr_from_below) {
            TensorInfo &ti = P.t[z.t];
            const size_t by = B * (size_t)(z.r1 - z.r0) * rowbytes(z.t);
            ti.zr_in_off = alloc(by); ti.zr_dout_off = alloc(by);
            ti.zr_in_r0 = z.r0; ti.zr_in_r1 = z.r1;
            M.halo_cache += 2 * by;
        }
        for (auto &z : S.zr_to_above) {
            TensorInfo &ti = P.t[z.t];
            const size_t by = B * (size_t)(z.r1 - z.r0) * rowbytes(z.t);
            ti.zr_out_off = alloc(by); ti.zr_din_off = alloc(by);
            ti.zr_out_r0 = z.r0; ti.zr_out_r1 = z.r1;
            M.halo_cache += 2 * by;
        }
    }
    // full-width delta of segment outputs, ping-pong: buffer p holds the outputs of the segments
    // with index parity p (segment s reads its output delta from s & 1 and writes its input delta
    // into the other), so each buffer is sized for its own parity's largest map only
    size_t dmax[2] = {0, 0}, xmax = 0;
    for (size_t si = 0; si < P.seg.size(); ++si) {
        const Segment &S = P.seg[si];
        dmax[si & 1] = std::max(dmax[si & 1], B * P.t[S.out_t].dl_rows * rowbytes(S.out_t));
        for (const Xfer &x : S.in_xfers) xmax = std::max(xmax, B * (size_t)(x.r1 - x.r0) * rowbytes(S.in_t));
    }
    P.dfull_bytes = std::max(dmax[0], dmax[1]);
    P.dfull_off[0] = alloc(dmax[0]);
    P.dfull_off[1] = P.seg.size() > 1 ? alloc(dmax[1]) : P.dfull_off[0];
    M.delta_full = dmax[0] + (P.seg.size() > 1 ? dmax[1] : 0);
    P.zl_off = alloc(B * zl.ck_rows * rowbytes(n_ops));
    M.checkpoints += B * zl.ck_rows * rowbytes(n_ops);
    if (xmax) {   // two send and two receive staging slots (one per neighbour)
        P.xstage_bytes = xmax;
        P.xstage_off[0] = alloc(4 * xmax);
        P.xstage_off[1] = P.xstage_off[0] + 2 * xmax;
        M.other += 4 * xmax;
    }
    // gap, d logits, loss terms, then the two-pass GAP partial sums [B][64 chunks][Cp] (head_gap)
    P.head_off = alloc(sizeof(float) * (B * zl.Cp + B * net->n_classes + B + 64 + (size_t)B * 64 * zl.Cp));
    P.flag_off = alloc(256);
    M.other += ws - (P.head_off);
    {
        size_t o0 = ws;
        for (OpInfo &o : P.op)
            if (o.d.kind == LRCNN_OP_CONV) o.wt_off = alloc(o.w_cnt * E);
        for (OpInfo &o : P.op)
            if (o.d.kind == LRCNN_OP_BN) {
                const size_t Cp = P.t[o.out_t].Cp;
                o.bn_sums_off = alloc(2 * Cp * sizeof(double));
                o.bn_S_off = alloc(2 * Cp * sizeof(double));
                o.bn_coef_off = alloc(6 * Cp * sizeof(float));
            }
        M.other += ws - o0;
    }
    // training-mode BN levels per segment (Segment::bn_*)
    size_t bp_stash_need = 0;
    for (Segment &S : P.seg) {
        std::vector<int> bns;
        for (int i : S.ops)
            if (P.op[i].d.kind == LRCNN_OP_BN) bns.push_back(i);
        if (bns.empty()) continue;
        for (int j : bns)
            if (world > 1 && P.op[j].in_t == S.in_t) {
                err = "training-mode BN of a segment input with row sharding is not supported";
                return LRCNN_E_UNSUPPORTED;
            }
        std::vector<char> inside(T, 0);
        for (int i : S.ops) inside[i + 1] = 1;
        auto ins = [&](int i) {
            std::vector<int> v = {P.op[i].d.src};
            if (P.op[i].d.res >= 0) v.push_back(P.op[i].d.res);
            return v;
        };
        // ancestors of tensor t inside the segment (ops), by a reverse walk; tensors with cut[t] != 0 are
        // available (stashed by an earlier sweep): their producers are not needed
        std::vector<char> nocut(T, 0);
        auto anc_ops = [&](const std::vector<int> &roots, const std::vector<char> &cut) {
            std::vector<char> op_in(n_ops, 0), seen(T, 0);
            std::vector<int> st = roots;
            while (!st.empty()) {
                const int t = st.back(); st.pop_back();
                if (seen[t] || !inside[t]) continue;
                seen[t] = 1;
                if (cut[t]) continue;
                const int i = P.t[t].producer;
                op_in[i] = 1;
                for (int u : ins(i)) st.push_back(u);
            }
            return op_in;
        };
        std::vector<int> lvl(n_ops, -1), rlvl(n_ops, -1);
        for (int j : bns) {   // op order is topological: ancestors first
            int l = 0;
            std::vector<char> a = anc_ops({P.op[j].d.src}, nocut);
            for (int k : bns)
                if (k != j && a[k]) l = std::max(l, lvl[k] + 1);
            lvl[j] = l;
        }
        // descendants of op j's output inside the segment (tensors), by a forward walk in op order
        auto desc_t = [&](const std::vector<int> &roots) {
            std::vector<char> d(T, 0);
            for (int t : roots) d[t] = 1;
            for (int i : S.ops)
                for (int u : ins(i))
                    if (d[u]) d[i + 1] = 1;
            return d;
        };
        for (auto it = bns.rbegin(); it != bns.rend(); ++it) {
            const int j = *it;
            std::vector<char> d = desc_t({P.op[j].out_t});
            int l = 0;
            for (int k : bns)
                if (k != j && d[P.op[k].out_t]) l = std::max(l, rlvl[k] + 1);
            rlvl[j] = l;
        }
        int nf = 0, nb = 0;
        for (int j : bns) { nf = std::max(nf, lvl[j] + 1); nb = std::max(nb, rlvl[j] + 1); }
        S.bn_fp_levels.assign(nf, {});
        S.bn_bp_levels.assign(nb, {});
        for (int j : bns) { S.bn_fp_levels[lvl[j]].push_back(j); S.bn_bp_levels[rlvl[j]].push_back(j); }
        // BN tail (below) and input stash: the inputs of the other BN ops, full-width, overlaying the delta
        // buffers (BP only) while they fit; one GPU (a rank's rows would need the halo rows too)
        const bool recomputes = !(P.seg.size() == 1 && S.E.size() == 1);
        {
            const int jl = P.t[S.out_t].producer;
            const OpInfo &o = P.op[jl];
            if (o.d.kind == LRCNN_OP_BN && recomputes && world <= 1 && S.bn_fp_levels.back().size() == 1 &&
                S.bn_fp_levels.back()[0] == jl && (o.d.res < 0 || o.d.res == S.in_t) && inside[o.in_t] &&
                o.in_t != S.out_t && P.t[o.in_t].cons.size() == 1 && P.t[o.in_t].C == P.t[S.out_t].C)
                S.bn_tail = jl;
        }
        S.stash_off.assign(T, (size_t)-1);
        std::vector<int> stash_level(T, -1);
        if (recomputes && world <= 1) {
            const size_t r0 = P.dfull_off[0];
            const size_t r1 = P.seg.size() > 1 ? P.dfull_off[1] + dmax[1] : P.dfull_off[0] + dmax[0];
            size_t used = 0;
            for (int j : bns) {
                const int c = P.op[j].in_t;
                if (j == S.bn_tail || !inside[c] || c == S.out_t || P.t[c].cons.size() != 1) continue;
                const size_t bytes = align_up(B * (size_t)P.t[c].H * rowbytes(c));
                if (r0 + used + bytes > r1) continue;
                S.stash_off[c] = r0 + used;
                stash_level[c] = lvl[j];
                used += bytes;
            }
        }
        for (int l = 0; l < nf; ++l) {
            std::vector<int> roots;
            for (int j : S.bn_fp_levels[l]) roots.push_back(P.op[j].d.src);
            std::vector<char> cut(T, 0);   // stashed by an earlier level's sweep
            for (int t = 0; t < T; ++t) cut[t] = stash_level[t] >= 0 && stash_level[t] < l;
            S.bn_fp_ops.push_back(anc_ops(roots, cut));
        }
        {   // the FP sweep: every op but the producers of stashed tensors
            S.bn_fp_final.assign(n_ops, 0);
            for (int i : S.ops) S.bn_fp_final[i] = 1;
            for (int t = 0; t < T; ++t)
                if (stash_level[t] >= 0) S.bn_fp_final[P.t[t].producer] = 0;
        }
        if (recomputes && world <= 1 && S.bn_bp_levels.size() > 0) {
            // BP stash: BN inputs (not the tail's) while they fit in one boundary map's bytes; offsets
            // relative to the BP stash region, allocated below (the largest segment's need)
            const size_t budget = std::max(dmax[0], dmax[1]);
            size_t used = 0;
            S.bp_stash_off.assign(T, (size_t)-1);
            S.bn_bp_recompute.assign(n_ops, 0);
            for (int i : S.ops) S.bn_bp_recompute[i] = 1;
            bool any = false;
            for (int j : bns) {
                if (j == S.bn_tail) continue;
                // the BN input c (its sums / backward read it) and the BN output t (the next conv's input
                // and the ReLU gate): with both stashed, the later sweeps recompute neither
                for (int c : {P.op[j].in_t, P.op[j].out_t}) {
                    if (!inside[c] || c == S.out_t) continue;
                    if (c == P.op[j].in_t && P.t[c].cons.size() != 1) continue;
                    const size_t bytes = align_up(B * (size_t)P.t[c].H * rowbytes(c));
                    if (used + bytes > budget) continue;
                    S.bp_stash_off[c] = used;
                    S.bn_bp_recompute[P.t[c].producer] = 0;
                    used += bytes;
                    any = true;
                }
            }
            if (!any) { S.bp_stash_off.clear(); S.bn_bp_recompute.clear(); }
            bp_stash_need = std::max(bp_stash_need, used);
        }
        for (int l = 0; l < nb; ++l) {
            std::vector<int> roots;
            for (int j : S.bn_bp_levels[l]) roots.push_back(P.op[j].out_t);
            std::vector<char> need = desc_t(roots), ops(n_ops, 0);
            for (int i : S.ops)
                if (need[i + 1]) ops[i] = 1;
            for (int j : S.bn_bp_levels[l]) ops[j] = 0;
            S.bn_bp_need.push_back(need);
            S.bn_bp_ops.push_back(ops);
        }
    }
    if (bp_stash_need) {   // BN BP stash region (shared by the segments: one segment's BP at a time)
        const size_t base = alloc(bp_stash_need);
        M.other += bp_stash_need;
        for (Segment &S : P.seg)
            for (size_t &o : S.bp_stash_off)
                if (o != (size_t)-1) o += base;
    }
    // per-segment arena (band act/delta/carry), overlaid across segments
    size_t arena0 = ws, arena_max = 0;
    for (const Segment &S : P.seg) {
        size_t a = 0, act = 0, dl = 0, car = 0;
        auto sub = [&](size_t bytes) { size_t o = a; a = align_up(a + bytes); return arena0 + o; };
        const int N = (int)S.E.size();
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            TensorInfo &ti = P.t[t];
            int cap = 0, ccap = 0;
            for (int r = 0; r < N; ++r) {
                cap = std::max(cap, S.hb[r][t] - S.lo[r][t]);
                ccap = std::max(ccap, S.a[r][t] - S.lo[r][t]);
            }
            ti.cap = std::max(cap, 1);
            ti.act_off = sub(B * ti.cap * rowbytes(t)); act += B * ti.cap * rowbytes(t);
            ti.carry_cap = ccap;
            if (ccap > 0 && opts->mode == LRCNN_2PS) { ti.carry_off = sub(B * ccap * rowbytes(t)); car += B * ccap * rowbytes(t); }
        }
        {   // delta slots (liveness overlay), after the activation and carry buffers
            dl = delta_slots(P, S, B, E, true);
            const size_t d0 = a;
            a = align_up(a + dl);
            for (int t : S.tensors)
                if (t != S.out_t && P.t[t].dfw >= 0) P.t[t].dlt_off += arena0 + d0;
        }
        if (a > arena_max) { arena_max = a; M.band_act = act; M.band_delta = dl; M.carry = car; }
    }
    // decoupled FP bands (LRCNN_FLAG_FP_MERGE): per segment the largest merge
    // factor m (FP band = m consecutive BP bands) whose FP activation buffers fit in the arena
    // the BP needs anyway; the FP buffers alias that arena (FP and BP never overlap in time)
    for (Segment &S : P.seg) {
        S.fp_r0.clear(); S.fp_lo.clear(); S.fp_a.clear(); S.fp_b.clear();
        const int N = (int)S.E.size();
        if (!(opts->flags & LRCNN_FLAG_FP_MERGE) || opts->mode != LRCNN_2PS || N < 2 || zr) continue;
        auto fp_arena = [&](int m, std::vector<int> *caps) {
            size_t a = 0;
            for (int t : S.tensors) {
                if (t == S.out_t) continue;
                int cap = 0;
                for (int r0 = 0; r0 < N; r0 += m) {
                    const int r1 = std::min(N, r0 + m);
                    cap = std::max(cap, S.b[r1 - 1][t] - S.lo[r0][t]);
                }
                cap = std::max(cap, 1);
                if (caps) caps->push_back(cap);
                a += align_up(B * cap * rowbytes(t));
            }
            return a;
        };
        int best = 1;
        for (int m = 2; m <= N; ++m)
            if (fp_arena(m, nullptr) <= arena_max) best = m;
        if (best < 2) continue;
        std::vector<int> caps;
        fp_arena(best, &caps);
        size_t o = arena0;
        int ci = 0;
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            TensorInfo &ti = P.t[t];
            ti.cap_fp = caps[ci++];
            ti.act_fp_off = o;
            o = arena0 + align_up(o - arena0 + B * ti.cap_fp * rowbytes(t));
        }
        for (int r0 = 0; r0 < N; r0 += best) {
            const int r1 = std::min(N, r0 + best);
            S.fp_r0.push_back(r0);
            std::vector<int> lo(T, 0), a(T, 0), b(T, 0);
            for (int t = 0; t < T; ++t) { lo[t] = S.lo[r0][t]; a[t] = S.a[r0][t]; b[t] = S.b[r1 - 1][t]; }
            S.fp_lo.push_back(lo); S.fp_a.push_back(a); S.fp_b.push_back(b);
        }
    }
    ws = align_up(arena0 + arena_max);
    P.ws_bytes = ws;
    M.workspace = ws;

    // ---------------------------------------------------------------- FLOPs
    double tau = 0, fwd = 0, bwd = 0;
    for (int i = 0; i < n_ops; ++i) {
        const OpInfo &o = P.op[i];
        if (o.d.kind != LRCNN_OP_CONV) continue;
        double per_row = 2.0 * o.d.k * o.d.k * B * P.t[o.in_t].C * P.t[o.out_t].C * P.t[o.out_t].W;
        tau += per_row * P.t[o.out_t].H;
        const Segment &S = P.seg[P.t[o.out_t].seg];
        for (size_t r = 0; r < S.E.size(); ++r) {
            double rows = S.b[r][o.out_t] - S.a[r][o.out_t];
            fwd += per_row * rows;
            bwd += per_row * rows * (o.in_t == 0 ? 1 : 2);
        }
    }
    bool recompute = !(P.seg.size() == 1 && P.seg[0].E.size() == 1);
    M.tau_flops = tau;
    M.fwd_flops = fwd;
    M.step_flops = fwd * (recompute ? 2 : 1) + bwd;
    return LRCNN_OK;
}

}  // namespace lrcnn

// engine.cu -- the band loops of Algorithm 1 and the C-ABI entry points.
//
// FP  (Alg. 1 l.5-11): per segment, bands r = 1..N; each op
//     computes its band rows from the band buffers; 2PS restores the cached halo
//     rows of band r-1 at the top of each buffer before the band and saves the
//     rows band r+1 will read after it.
// BP  (Alg. 1 l.15-23): per segment in reverse, bands
//     r = N..1: recompute the band (l.17), then per op in reverse: bias/affine
//     reduction, wgrad (+= into fp32 grads, l.20), dgrad into the input's band
//     delta; 2PS carries the delta of cached rows to band r-1 (R6).
// Every device operation is enqueued on the caller's stream; nothing is
// allocated on the device.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "kernels.hpp"
#include "plan.hpp"
#include "comm.hpp"
#include "tc.hpp"

struct lrcnn_plan_t {
    lrcnn::Plan P;
};

namespace lrcnn {

static thread_local std::string g_err;
static lrcnn_status fail(lrcnn_status s, const std::string &m) { g_err = m; return s; }

#define CK(expr)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (expr);                                                                  \
        if (e_ != cudaSuccess) return fail(LRCNN_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct Run {
    Plan &P;
    char *ws;
    const char *params;
    const void *x;
    void *zl;
    float *grads;
    cudaStream_t st;
    int prec;
    size_t E;   // element bytes
    cudaStream_t side = nullptr;   // wgrad / param-grad stream (nullptr: everything on st)
    bool side_busy = false;
    bool fp_merged = false;        // FP over merged bands: band tensors live in the FP buffers
    bool dp_pending = false;       // gradient all-reduces enqueued on the communication stream
    // training-mode BN sweeps: FP statistics sweep -- compute only the ops in fmask;
    // BP sums sweep -- run the backward of the ops in bops only, write the delta of the tensors in
    // bneed only, no weight / parameter gradients; bn_level: the BN ops whose sums the sweep takes
    const std::vector<char> *fmask = nullptr, *bops = nullptr, *bneed = nullptr;
    const std::vector<int> *bn_level = nullptr;
    // BN tail statistics sweep: tensor `redirect` (the tail BN's input) is written straight into the
    // segment output's full-width checkpoint instead of its band buffer (-1: none)
    int redirect = -1;
    // FP of a segment with training-mode BN: tensors with a stash slot (Segment::stash_off) live full-width
    // there instead of in their band buffers
    bool stash = false;
    // BP of a segment with a BN stash: tensors with a slot in bp_stash (absolute offsets) live there
    const std::vector<size_t> *bp_stash = nullptr;
};

// Fork: side stream waits for everything enqueued so far on the main stream.
static cudaError_t fork_side(Run &R) {
    cudaError_t e = cudaEventRecord((cudaEvent_t)R.P.ev_fork, R.st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(R.side, (cudaEvent_t)R.P.ev_fork, 0);
    R.side_busy = true;
    return e;
}
// Join: main stream waits for the side stream (before buffers it reads are overwritten).
static cudaError_t join_side(Run &R) {
    if (!R.side || !R.side_busy) return cudaSuccess;
    cudaError_t e = cudaEventRecord((cudaEvent_t)R.P.ev_join, R.side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(R.st, (cudaEvent_t)R.P.ev_join, 0);
    R.side_busy = false;
    return e;
}

// a boundary map (image, checkpoint, z^L) on this rank: rows [ck_lo, ck_lo + ck_rows)
static View full_view(void *p, const TensorInfo &t) {
    View v;
    v.p = p; v.base = t.ck_lo; v.rows = t.ck_rows; v.H = t.H; v.W = t.W; v.Cp = t.Cp;
    v.bs = (long long)t.ck_rows * t.W * t.Cp;
    return v;
}
// the boundary delta buffer of a segment input/output: rows [dl_lo, dl_lo + dl_rows)
static View dfull_view(void *p, const TensorInfo &t) {
    View v;
    v.p = p; v.base = t.dl_lo; v.rows = t.dl_rows; v.H = t.H; v.W = t.W; v.Cp = t.Cp;
    v.bs = (long long)t.dl_rows * t.W * t.Cp;
    return v;
}

void set_last_error(const std::string &m) { g_err = m; }

static View band_view(char *base_ptr, const TensorInfo &t, int lo, int b) {
    View v;
    v.p = base_ptr; v.base = lo; v.rows = b - lo; v.H = t.H; v.W = t.W; v.Cp = t.Cp;
    v.bs = (long long)t.cap * t.W * t.Cp;
    return v;
}

// restrict a view to rows [a, b) (rows outside read as zero / are not data)
static View sub_rows(const View &v, int a, int b, size_t E) {
    View s = v;
    s.p = (char *)v.p + (size_t)(a - v.base) * v.W * v.Cp * E;
    s.base = a; s.rows = b - a;
    return s;
}

static void *ckpt_ptr(Run &R, int t) {
    const TensorInfo &ti = R.P.t[t];
    if (t == 0) return (void *)R.x;
    if (ti.is_zl) return R.zl;
    return R.ws + ti.ckpt_off;
}

// activation view of tensor t in band r of segment s
static View act_view(Run &R, const Segment &S, int r, int t) {
    const TensorInfo &ti = R.P.t[t];
    if (t == S.in_t || t == S.out_t) return full_view(ckpt_ptr(R, t), ti);
    if (t == R.redirect) return full_view(ckpt_ptr(R, S.out_t), R.P.t[S.out_t]);
    if (R.stash && (size_t)t < S.stash_off.size() && S.stash_off[t] != (size_t)-1) {
        View v{R.ws + S.stash_off[t], 0, ti.H, ti.H, ti.W, ti.Cp, (long long)ti.H * ti.W * ti.Cp};
        return v;
    }
    if (R.bp_stash && (size_t)t < R.bp_stash->size() && (*R.bp_stash)[t] != (size_t)-1) {
        View v{R.ws + (*R.bp_stash)[t], 0, ti.H, ti.H, ti.W, ti.Cp, (long long)ti.H * ti.W * ti.Cp};
        return v;
    }
    if (R.fp_merged) {   // S is the merged FP view of the segment (fp_lo / fp_b as lo / b)
        View v = band_view(R.ws + ti.act_fp_off, ti, S.lo[r][t], S.b[r][t]);
        v.bs = (long long)ti.cap_fp * ti.W * ti.Cp;
        return v;
    }
    return band_view(R.ws + ti.act_off, ti, S.lo[r][t], S.hb[r][t]);
}

static View dlt_view(Run &R, const Segment &S, int s, int r, int t) {
    {
        const int al = alias_delta(R.P, S, t);
        if (al >= 0) t = al;
    }
    const TensorInfo &ti = R.P.t[t];
    int nseg = (int)R.P.seg.size();
    if (t == S.out_t) return dfull_view(R.ws + R.P.dfull_off[s & 1], ti);
    if (t == S.in_t) return dfull_view(t == 0 ? nullptr : R.ws + R.P.dfull_off[(s + 1) & 1], ti);
    (void)nseg;
    return band_view(R.ws + ti.dlt_off, ti, S.lo[r][t], S.hb[r][t]);
}

// NVTX ranges (header-only nvtx3: a no-op unless a tool such as nsys / ncu --nvtx is attached):
// one range per segment and band of the FP and the BP, the head and the exchanges
struct Nvtx {
    explicit Nvtx(const char *fmt, int a = 0, int b = 0) {
        char buf[64];
        snprintf(buf, sizeof buf, fmt, a, b);
        nvtxRangePushA(buf);
    }
    ~Nvtx() { nvtxRangePop(); }
};

static int env_chunk_mb() {
    const char *e = getenv("LRCNN_L2_CHUNK_MB");
    return e && *e ? atoi(e) : 0;
}

static bool zr_plan(const Plan &P) { return P.opts.world > 1 && (P.opts.flags & LRCNN_FLAG_ZERO_REDUNDANCY); }

static const void *prm(Run &R, size_t off) { return off == (size_t)-1 ? nullptr : R.params + off * R.E; }

// A tensor-core launcher returned false: a launch / attribute failure is an error (LRCNN_E_CUDA; the
// SIMT kernel must not rerun rows a partial launch already produced); a declined shape runs the SIMT
// kernel, is counted (lrcnn_last_simt_fallbacks) and is an error under LRCNN_FLAG_REQUIRE_TC.
static lrcnn_status tc_declined(Plan &P, int op, const char *kind) {
    if (tc_take_error())
        return fail(LRCNN_E_CUDA, std::string("tensor-core ") + kind + " launch failed at op " + std::to_string(op));
    ++P.simt_fallbacks;
    if (P.opts.flags & LRCNN_FLAG_REQUIRE_TC)
        return fail(LRCNN_E_UNSUPPORTED, std::string("no tensor-core kernel takes the ") + kind + " of op " +
                                             std::to_string(op) + " (LRCNN_FLAG_REQUIRE_TC)");
    return LRCNN_OK;
}

// ------------------------------------------------------------------ profiling
struct ProfScope {
    Run &R;
    int cls;
    double flops;
    int tag;
    double bytes, wbytes;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ProfScope(Run &r, int c, double f, int t = -1, double by = 0, double wb = 0)
        : R(r), cls(c), flops(f), tag(t), bytes(by), wbytes(wb) {
        if (R.P.profiling) {
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0, R.st);
            tc_clear_last_kernel();
        }
    }
    ~ProfScope() {
        if (R.P.profiling) {
            cudaEventRecord(e1, R.st);
            R.P.pending_events[cls].push_back({(void *)e0, (void *)e1});
            R.P.pending_flops[cls].push_back(flops);
            R.P.pending_bytes[cls].push_back(bytes);
            R.P.pending_wbytes[cls].push_back(wbytes);
            R.P.pending_tags[cls].push_back(tag);
            const char *k = tc_last_kernel();
            R.P.pending_names[cls].push_back(k ? k : "");
        }
    }
};

static double conv_flops(Plan &P, const OpInfo &o, int rows) {
    return 2.0 * o.d.k * o.d.k * P.net.B * P.t[o.in_t].C * P.t[o.out_t].C * (double)rows * P.t[o.out_t].W;
}

// Algorithmic HBM bytes of one conv launch over output rows [a, b): every operand
// read once, every result written once.  kind 0 FP: input rows [a*s-p, (b-1)*s-p+k) clipped + weights
// + output (+ residual); kind 1 dgrad: dy + weights + dx and the gating activation (+ dx read when
// it accumulates); kind 2 wgrad: dy + input rows + the fp32 gradient read-modify-write.
// write: only the bytes written (the output map, delta_in, the fp32 gradient's write half) --
// HBM writes alone sustain less than a copy (bench.py's mixed read/write roofline)
static double conv_bytes(Plan &P, const OpInfo &o, int a, int b, int kind, int dx_accum = 0, int gate = 0,
                         bool write = false) {
    const TensorInfo &ti = P.t[o.in_t], &to = P.t[o.out_t];
    const double E = P.opts.prec == LRCNN_FP32 ? 4.0 : 2.0, B = P.net.B;
    const int ra = std::max(0, a * o.d.s - o.d.p), rb = std::min(ti.H, (b - 1) * o.d.s - o.d.p + o.d.k);
    const double in = B * (double)(rb - ra) * ti.W * ti.Cp * E;
    const double out = B * (double)(b - a) * to.W * to.Cp * E;
    const double w = (double)o.d.k * o.d.k * ti.Cp * o.d.c_out;
    if (write) return kind == 0 ? out : kind == 1 ? in : w * 4.0;
    if (kind == 0) return in + out + w * E + (o.d.res >= 0 ? out : 0.0);
    if (kind == 1) return out + w * E + in * (1.0 + gate + dx_accum);
    return out + in + w * 8.0;
}

// ------------------------------------------------------------------ op forward on band rows [a, b)
static lrcnn_status op_forward_impl(Run &R, const Segment &S, int r, int i) {
    Plan &P = R.P;
    const OpInfo &o = P.op[i];
    const int t = o.out_t;
    const int a = S.a[r][t], b = S.b[r][t];
    if (b <= a) return LRCNN_OK;
    View out = act_view(R, S, r, t);
    View in = act_view(R, S, r, o.in_t);
    if (o.d.kind == LRCNN_OP_CONV) {
        ConvFwdArgs A;
        A.in = in; A.out = out;
        if (o.d.res >= 0) A.res = act_view(R, S, r, o.d.res);
        A.w = prm(R, o.w_off);
        A.b = o.b_cnt ? prm(R, o.b_off) : nullptr;
        A.beta = o.beta_cnt ? prm(R, o.beta_off) : nullptr;
        A.k = o.d.k; A.s = o.d.s; A.p = o.d.p; A.c_out = o.d.c_out; A.epi = o.d.epi; A.relu = o.d.relu;
        A.a = a; A.b_ = b; A.B = P.net.B;
        ProfScope ps(R, 0, conv_flops(P, o, b - a), i * 8 + 0, conv_bytes(P, o, a, b, 0),
                     conv_bytes(P, o, a, b, 0, 0, 0, true));
        ++P.launches;
        if (P.use_tc) {
            if (tc_conv_fwd(A, R.st)) { ++P.tc_launches; CK(cudaGetLastError()); return LRCNN_OK; }
            lrcnn_status st = tc_declined(P, i, "FP");
            if (st != LRCNN_OK) return st;
        }
        CK(simt_conv_fwd(R.prec, A, R.st));
    } else if (o.d.kind == LRCNN_OP_MAXPOOL) {
        PoolArgs A;
        A.in = in; A.out = out; A.k = o.d.k; A.s = o.d.s; A.p = o.d.p; A.a = a; A.b = b; A.B = P.net.B;
        ++P.launches;
        ProfScope ps(R, 2, 0, i * 8 + 4);
        CK(simt_pool_fwd(R.prec, A, R.st));
    } else if (o.d.kind == LRCNN_OP_BN) {   // t = relu?(a*c + b + res), a / b from this step's statistics
        View res;
        if (o.d.res >= 0) res = act_view(R, S, r, o.d.res);
        ++P.launches;
        ProfScope ps(R, 2, 0, i * 8 + 6);
        CK(bn_fwd(R.prec, in, res, out, (const float *)(R.ws + o.bn_coef_off), o.d.relu, a, b, P.net.B, R.st));
    } else {
        EltArgs A;
        A.x0 = in; A.x1 = act_view(R, S, r, o.d.res); A.out = out; A.relu = o.d.relu; A.a = a; A.b = b; A.B = P.net.B;
        ++P.launches;
        ProfScope ps(R, 2, 0, i * 8 + 6);
        CK(simt_add_fwd(R.prec, A, R.st));
    }
    return LRCNN_OK;
}

// Debug capture (lrcnn_debug_capture): rows [a, b) of tensor t, just computed by a band, copied into
// the caller's full-height buffer [B][H][W][Cp] -- every row of every tensor is produced by exactly
// one band (interval rule), so after a forward the buffer holds the whole map the row-centric
// sweep computed.  Parity tests only; never registered on a timed path.
static lrcnn_status capture_rows(Run &R, int t, const View &out, int a, int b) {
    Plan &P = R.P;
    if ((size_t)t >= P.capture.size() || !P.capture[t] || b <= a) return LRCNN_OK;
    const TensorInfo &ti = P.t[t];
    const size_t rb = (size_t)ti.W * ti.Cp * R.E;
    const char *src = (const char *)out.p + (size_t)(a - out.base) * rb;
    char *dst = (char *)P.capture[t] + (size_t)a * rb;
    CK(cudaMemcpy2DAsync(dst, (size_t)ti.H * rb, src, (size_t)out.bs * R.E, (size_t)(b - a) * rb, P.net.B,
                         cudaMemcpyDeviceToDevice, R.st));
    return LRCNN_OK;
}

static lrcnn_status capture_rows(Run &R, int t, const View &out, int a, int b);
static lrcnn_status op_forward(Run &R, const Segment &S, int r, int i) {
    lrcnn_status st = op_forward_impl(R, S, r, i);
    if (st != LRCNN_OK || R.P.capture.empty()) return st;
    const int t = R.P.op[i].out_t;
    return capture_rows(R, t, act_view(R, S, r, t), S.a[r][t], S.b[r][t]);
}

// ------------------------------------------------------------------ fused identity bottleneck (FP)
// Ops i, i+1, i+2 of segment S form an identity bottleneck with a 64-channel middle (1x1 -> 3x3 ->
// 1x1 + block input, frozen-BN affine + ReLU each; ResNet-50 conv2_x) whose two intermediate maps
// nobody else reads: one k_bneck_fwd launch per band (bneck_tc.cu).
static bool bneck_at(const Plan &P, const Segment &S, int i) {
    if (!P.use_tc || (P.opts.flags & LRCNN_FLAG_NO_FUSE_BLOCK) || zr_plan(P)) return false;
    if (i + 2 >= (int)P.op.size()) return false;
    const OpInfo &c1 = P.op[i], &c2 = P.op[i + 1], &c3 = P.op[i + 2];
    auto conv = [](const OpInfo &o, int k, int p, int c_out) {
        return o.d.kind == LRCNN_OP_CONV && o.d.k == k && o.d.s == 1 && o.d.p == p && o.d.c_out == c_out &&
               o.d.epi == LRCNN_EPI_AFFINE && o.d.relu;
    };
    if (!conv(c1, 1, 0, 64) || !conv(c2, 3, 1, 64) || !conv(c3, 1, 0, 256)) return false;
    const int t = c1.in_t, t1 = c1.out_t, t2 = c2.out_t;
    if (c1.d.res >= 0 || c2.d.res >= 0 || c3.d.res != t || c2.in_t != t1 || c3.in_t != t2) return false;
    if (P.t[t].Cp != 256 || P.t[t1].Cp != 64 || P.t[t2].Cp != 64) return false;
    if (P.t[t1].cons.size() != 1 || P.t[t2].cons.size() != 1) return false;
    if (t1 == S.out_t || t2 == S.out_t || t1 == S.in_t || t2 == S.in_t) return false;
    bool in1 = false, in2 = false;
    for (int o : S.ops) { in1 = in1 || o == i + 1; in2 = in2 || o == i + 2; }
    return in1 && in2;
}

static lrcnn_status capture_rows(Run &R, int t, const View &out, int a, int b);
// One band (S may be the merged FP view, R.fp_merged) of the fused block at op i.  nwin / wlo / whi:
// t1 rows to store (nwin < 0: all), write_t2: store t2 (BP recompute, capture).
static lrcnn_status bneck_forward(Run &R, const Segment &S, int r, int i, int nwin, const int *wlo, const int *whi,
                                  int write_t2) {
    Plan &P = R.P;
    const OpInfo &c1 = P.op[i], &c2 = P.op[i + 1], &c3 = P.op[i + 2];
    const int t = c1.in_t, t1 = c1.out_t, t2 = c2.out_t, u = c3.out_t;
    const bool cap = !P.capture.empty();
    if (cap) { nwin = -1; write_t2 = 1; }
    BneckArgs A;
    A.t = act_view(R, S, r, t); A.t1 = act_view(R, S, r, t1); A.t2 = act_view(R, S, r, t2); A.u = act_view(R, S, r, u);
    A.w1 = prm(R, c1.w_off); A.w2 = prm(R, c2.w_off); A.w3 = prm(R, c3.w_off);
    A.g1 = prm(R, c1.b_off); A.e1 = prm(R, c1.beta_off);
    A.g2 = prm(R, c2.b_off); A.e2 = prm(R, c2.beta_off);
    A.g3 = prm(R, c3.b_off); A.e3 = prm(R, c3.beta_off);
    A.a2 = S.a[r][t2]; A.b2 = S.b[r][t2]; A.a1 = S.a[r][t1]; A.b1 = S.b[r][t1]; A.B = P.net.B;
    A.write_t2 = write_t2;
    A.nwin = nwin;
    for (int k = 0; k < nwin && k < 16; ++k) { A.wlo[k] = wlo[k]; A.whi[k] = whi[k]; }
    if (S.a[r][u] != A.a2 || S.b[r][u] != A.b2) return fail(LRCNN_E_STATE, "fused bottleneck: t2 / u band rows differ");
    if (A.b2 > A.a2) {
        double fl = conv_flops(P, c1, A.b1 - A.a1) + conv_flops(P, c2, A.b2 - A.a2) + conv_flops(P, c3, A.b2 - A.a2);
        const TensorInfo &T = P.t[t], &T1 = P.t[t1], &T2 = P.t[t2];
        const double Bn = P.net.B, rbt = (double)T.W * T.Cp * R.E, rb1 = (double)T1.W * T1.Cp * R.E;
        double w1rows = 0;
        for (int y = A.a1; y < A.b1; ++y) {
            bool st = nwin < 0;
            for (int k = 0; k < nwin && !st; ++k) st = y >= wlo[k] && y < whi[k];
            w1rows += st;
        }
        const double wr = Bn * ((A.b2 - A.a2) * rbt + w1rows * rb1 + (write_t2 ? (A.b2 - A.a2) * (double)T2.W * T2.Cp * R.E : 0));
        const double rd = Bn * (A.b1 - A.a1) * rbt + (double)(c1.w_cnt + c2.w_cnt + c3.w_cnt) * R.E;
        bool declined = false;
        {
            ProfScope ps(R, 0, fl, i * 8 + 0, rd + wr, wr);
            if (tc_bneck_fwd(A, R.st)) {
                ++P.launches;
                ++P.tc_launches;
                CK(cudaGetLastError());
            } else if (tc_take_error()) {
                return fail(LRCNN_E_CUDA, "fused bottleneck launch failed at op " + std::to_string(i));
            } else {
                declined = true;
            }
        }
        if (declined) {   // a shape / alignment the fused kernel does not take: the three ops unfused
            lrcnn_status st;
            for (int k = 0; k < 3; ++k)
                if ((st = op_forward(R, S, r, i + k)) != LRCNN_OK) return st;
            return LRCNN_OK;
        }
    }
    if (cap) {
        lrcnn_status st;
        if ((st = capture_rows(R, t1, A.t1, A.a1, A.b1)) != LRCNN_OK) return st;
        if ((st = capture_rows(R, t2, A.t2, A.a2, A.b2)) != LRCNN_OK) return st;
        if ((st = capture_rows(R, u, A.u, A.a2, A.b2)) != LRCNN_OK) return st;
    }
    return LRCNN_OK;
}

// the BP recomputes every band from the FP's checkpoints and caches (else the FP's maps are final)
static bool bp_recomputes(const Plan &P) { return !(P.seg.size() == 1 && P.seg[0].E.size() == 1); }

// copy rows between two views of the same tensor (B planes, pitched)
static lrcnn_status copy_rows(Run &R, const TensorInfo &ti, void *dst, size_t dst_pitch_rows, const void *src,
                              size_t src_pitch_rows, int rows) {
    if (rows <= 0) return LRCNN_OK;
    size_t rb = (size_t)ti.W * ti.Cp * R.E;
    CK(cudaMemcpy2DAsync(dst, dst_pitch_rows * rb, src, src_pitch_rows * rb, rows * rb, R.P.net.B,
                         cudaMemcpyDeviceToDevice, R.st));
    return LRCNN_OK;
}

// FP band k of a merged-band segment (LRCNN_FLAG_FP_MERGE): BP bands [r0, r1) computed as one band
// in the FP buffers; restores the cache rows of BP boundary r0-1 and saves those of every BP
// boundary r0 .. r1-1 (the BP recomputes band by band from them, R7).
static lrcnn_status band_forward_merged(Run &R, const Segment &S, const Segment &F, int k) {
    Plan &P = R.P;
    lrcnn_status st;
    const int N = (int)S.E.size(), r0 = S.fp_r0[k], r1 = k + 1 < (int)S.fp_r0.size() ? S.fp_r0[k + 1] : N;
    if (r0 > 0) {
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            const TensorInfo &ti = P.t[t];
            const int rows = F.a[k][t] - F.lo[k][t];
            if (rows <= 0) continue;
            if ((st = copy_rows(R, ti, R.ws + ti.act_fp_off, ti.cap_fp, R.ws + ti.cache_off[r0 - 1],
                                ti.cache_rows[r0 - 1], rows)) != LRCNN_OK) return st;
        }
    }
    R.fp_merged = true;
    for (size_t q = 0; q < S.ops.size(); ++q) {
        const int i = S.ops[q];
        if (R.fmask && !(*R.fmask)[i]) continue;   // BN input stash: its producers ran in a statistics sweep
        if (q >= 2 && S.ops[q - 1] == i - 1 && bneck_at(P, S, i - 2) && S.ops[q - 2] == i - 2) continue;
        if (q >= 1 && bneck_at(P, S, i - 1) && S.ops[q - 1] == i - 1) continue;
        if (bneck_at(P, S, i) && q + 2 < S.ops.size() && S.ops[q + 1] == i + 1 && S.ops[q + 2] == i + 2) {
            // t1 rows the BP bands [r0, r1) read from their 2PS cache
            const TensorInfo &T1 = P.t[P.op[i].out_t];
            int wlo[16], whi[16], nw = 0;
            for (int rr = r0; rr < r1 && rr + 1 < N; ++rr)
                if (T1.cache_rows[rr] > 0) {
                    if (nw == 16) { nw = -1; break; }
                    wlo[nw] = T1.cache_lo[rr]; whi[nw] = T1.cache_lo[rr] + T1.cache_rows[rr]; ++nw;
                }
            if (!bp_recomputes(P)) nw = -1;
            if ((st = bneck_forward(R, F, k, i, nw, wlo, whi, !bp_recomputes(P))) != LRCNN_OK) { R.fp_merged = false; return st; }
            continue;
        }
        if ((st = op_forward(R, F, k, i)) != LRCNN_OK) { R.fp_merged = false; return st; }
    }
    R.fp_merged = false;
    for (int r = r0; r < r1 && r + 1 < N; ++r) {
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            if (R.fmask && !(*R.fmask)[P.t[t].producer]) continue;
            const TensorInfo &ti = P.t[t];
            const int rows = ti.cache_rows[r];
            if (rows <= 0) continue;
            const size_t rb = (size_t)ti.W * ti.Cp * R.E;
            const char *src = R.ws + ti.act_fp_off + (size_t)(ti.cache_lo[r] - F.lo[k][t]) * rb;
            if ((st = copy_rows(R, ti, R.ws + ti.cache_off[r], rows, src, ti.cap_fp, rows)) != LRCNN_OK) return st;
        }
    }
    return LRCNN_OK;
}

static lrcnn_status band_forward(Run &R, const Segment &S, int r, bool save_cache, bool skip_out) {
    Plan &P = R.P;
    lrcnn_status st;
    // 2PS: restore the cached rows [lo_r, a_r) of every band tensor (saved by band r-1)
    if (P.opts.mode == LRCNN_2PS && r > 0) {
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            const TensorInfo &ti = P.t[t];
            int rows = S.a[r][t] - S.lo[r][t];
            if (rows <= 0) continue;
            // cache[r-1] holds rows [lo_r, b_{r-1}) == [lo_r, a_r); a stashed tensor (full-width slot, BN)
            // gets them at their rows of the slot (the BP walks the bands upward: band r-1 comes later)
            const View dv = act_view(R, S, r, t);
            const size_t rb = (size_t)ti.W * ti.Cp * R.E;
            char *dst = (char *)dv.p + (size_t)(S.lo[r][t] - dv.base) * rb;
            const size_t pitch = (size_t)dv.bs / ((size_t)ti.W * ti.Cp);
            if ((st = copy_rows(R, ti, dst, pitch, R.ws + ti.cache_off[r - 1], ti.cache_rows[r - 1], rows)) != LRCNN_OK)
                return st;
        }
    }
    // zero-redundancy: the last band reads rows [HI, hb) of every band tensor that rank+1 computed in
    // its first band (received after the first band, kept for the BP recompute)
    if (r == (int)S.E.size() - 1)
        for (const Segment::ZrRows &z : S.zr_from_below) {
            const TensorInfo &ti = P.t[z.t];
            const size_t rb = (size_t)ti.W * ti.Cp * R.E;
            if ((st = copy_rows(R, ti, R.ws + ti.act_off + (size_t)(z.r0 - S.lo[r][z.t]) * rb, ti.cap,
                                R.ws + ti.zr_in_off, z.r1 - z.r0, z.r1 - z.r0)) != LRCNN_OK) return st;
        }
    for (size_t q = 0; q < S.ops.size(); ++q) {
        const int i = S.ops[q];
        if (skip_out && i + 1 == S.out_t) continue;
        if (R.fmask && !(*R.fmask)[i]) continue;   // BN statistics sweep: only the ops it needs
        // ops i+1, i+2 of a fused block ran with op i (unless the block output is skipped: BP recompute
        // of the segment output, whose delta is known -- then ops i, i+1 run unfused)
        const bool f2 = q >= 2 && S.ops[q - 1] == i - 1 && S.ops[q - 2] == i - 2 && bneck_at(P, S, i - 2) &&
                        !(skip_out && i + 1 == S.out_t);
        const bool f1 = q >= 1 && q + 1 < S.ops.size() && S.ops[q - 1] == i - 1 && S.ops[q + 1] == i + 1 &&
                        bneck_at(P, S, i - 1) && !(skip_out && i + 2 == S.out_t);
        if (f1 || f2) continue;
        if (q + 2 < S.ops.size() && S.ops[q + 1] == i + 1 && S.ops[q + 2] == i + 2 && bneck_at(P, S, i) &&
            !(skip_out && i + 3 == S.out_t)) {
            const TensorInfo &T1 = P.t[P.op[i].out_t];
            int wlo[1], whi[1], nw = 0;
            if (save_cache && P.opts.mode == LRCNN_2PS && r + 1 < (int)S.E.size() && T1.cache_rows[r] > 0) {
                wlo[0] = T1.cache_lo[r]; whi[0] = T1.cache_lo[r] + T1.cache_rows[r]; nw = 1;
            }
            const bool all = !save_cache || !bp_recomputes(P);   // BP recompute, or the FP's maps are final
            if ((st = bneck_forward(R, S, r, i, all ? -1 : nw, wlo, whi, all)) != LRCNN_OK) return st;
            continue;
        }
        if ((st = op_forward(R, S, r, i)) != LRCNN_OK) return st;
    }
    if (save_cache && P.opts.mode == LRCNN_2PS && r + 1 < (int)S.E.size()) {
        for (int t : S.tensors) {
            if (t == S.out_t) continue;
            if (R.fmask && !(*R.fmask)[P.t[t].producer]) continue;   // not computed in this sweep
            const TensorInfo &ti = P.t[t];
            int rows = ti.cache_rows[r];
            if (rows <= 0) continue;
            size_t rb = (size_t)ti.W * ti.Cp * R.E;
            const char *src = R.ws + ti.act_off + (size_t)(ti.cache_lo[r] - S.lo[r][t]) * rb;
            if ((st = copy_rows(R, ti, R.ws + ti.cache_off[r], rows, src, ti.cap, rows)) != LRCNN_OK) return st;
        }
    }
    return LRCNN_OK;
}

// ------------------------------------------------------------------ halo exchange between ranks
// FP: before a segment runs, the rows of its input that neighbouring ranks own are received
// into this rank's checkpoint (and this rank's rows they need are sent).  BP: after a segment's
// backward, the delta this rank accumulated on the neighbours' rows is sent back and the
// neighbours' delta on this rank's rows is added (the OverL overlap sum at rank cuts).
static lrcnn_status pack_rows(Run &R, const View &v, int r0, int r1, void *dst, bool unpack) {
    const size_t rb = (size_t)v.W * v.Cp * R.E;
    char *p = (char *)v.p + (size_t)(r0 - v.base) * rb;
    if (unpack)
        CK(cudaMemcpy2DAsync(p, v.bs * R.E, dst, (r1 - r0) * rb, (r1 - r0) * rb, R.P.net.B, cudaMemcpyDeviceToDevice, R.st));
    else
        CK(cudaMemcpy2DAsync(dst, (r1 - r0) * rb, p, v.bs * R.E, (r1 - r0) * rb, R.P.net.B, cudaMemcpyDeviceToDevice, R.st));
    return LRCNN_OK;
}

static lrcnn_status exchange(Run &R, const Segment &S, const View &v, bool bp) {
    Plan &P = R.P;
    const TensorInfo &ti = P.t[S.in_t];
    const size_t rb = (size_t)ti.W * ti.Cp * R.E;
    char *sendb = R.ws + P.xstage_off[0], *recvb = R.ws + P.xstage_off[1];
    const int rank = P.opts.rank;
    std::vector<XferBuf> xs;
    std::vector<std::pair<const Xfer *, char *>> incoming;
    lrcnn_status st;
    for (const Xfer &x : S.in_xfers) {
        const int slot = x.peer < rank ? 0 : 1;
        const size_t bytes = (size_t)P.net.B * (x.r1 - x.r0) * rb;
        const bool out = bp ? !x.send : x.send;          // BP runs the FP schedule reversed
        if (out) {
            char *buf = sendb + slot * P.xstage_bytes;
            if ((st = pack_rows(R, v, x.r0, x.r1, buf, false)) != LRCNN_OK) return st;
            xs.push_back({x.peer, 1, buf, bytes});
        } else {
            char *buf = recvb + slot * P.xstage_bytes;
            xs.push_back({x.peer, 0, buf, bytes});
            incoming.push_back({&x, buf});
        }
    }
    const char *err = nullptr;
    if (comm_exchange((Comm *)P.comm, xs, R.st, &err)) return fail(LRCNN_E_NCCL, err ? err : "exchange failed");
    for (auto &in : incoming) {
        if (bp) CK(add_rows(R.prec, v, in.first->r0, in.first->r1, in.second, P.net.B, R.st));
        else if ((st = pack_rows(R, v, in.first->r0, in.first->r1, in.second, true)) != LRCNN_OK) return st;
    }
    return LRCNN_OK;
}

// Zero-redundancy halo exchange of one segment (one grouped send/recv, main stream, every rank at the
// same point).  FP (after the first band): my first rows go up to rank-1 (zr_out), rank+1's first rows
// come in (zr_in).  BP (after the last band's backward): the delta of rank+1's rows goes down
// (zr_dout), the delta rank-1 computed for my first rows comes in (zr_din).
static lrcnn_status zr_exchange(Run &R, const Segment &S, bool bp) {
    Plan &P = R.P;
    if (S.zr_from_below.empty() && S.zr_to_above.empty()) return LRCNN_OK;
    const int rank = P.opts.rank;
    std::vector<XferBuf> xs;
    for (const Segment::ZrRows &z : S.zr_to_above) {
        const TensorInfo &ti = P.t[z.t];
        const size_t by = (size_t)P.net.B * (z.r1 - z.r0) * ti.W * ti.Cp * R.E;
        xs.push_back({rank - 1, bp ? 0 : 1, R.ws + (bp ? ti.zr_din_off : ti.zr_out_off), by});
    }
    for (const Segment::ZrRows &z : S.zr_from_below) {
        const TensorInfo &ti = P.t[z.t];
        const size_t by = (size_t)P.net.B * (z.r1 - z.r0) * ti.W * ti.Cp * R.E;
        xs.push_back({rank + 1, bp ? 1 : 0, R.ws + (bp ? ti.zr_dout_off : ti.zr_in_off), by});
    }
    const char *err = nullptr;
    if (comm_exchange((Comm *)P.comm, xs, R.st, &err)) return fail(LRCNN_E_NCCL, err ? err : "zr exchange failed");
    return LRCNN_OK;
}

// transposed weights for the tensor-core dgrad (gamma folded in), on stream st
static lrcnn_status launch_transposes(Run &R, cudaStream_t st) {
    Plan &P = R.P;
    for (const OpInfo &o : P.op) {
        if (o.d.kind != LRCNN_OP_CONV || o.in_t == 0) continue;
        CK(transpose_weights(R.prec, prm(R, o.w_off), o.d.epi == LRCNN_EPI_AFFINE ? prm(R, o.b_off) : nullptr,
                             R.ws + o.wt_off, o.d.c_out, P.t[o.out_t].Cp, o.d.k, P.t[o.in_t].Cp, st));
        ++P.launches;
    }
    return LRCNN_OK;
}

// zero-redundancy sharding, after every rank's first FP band: my first rows the rank above reads go out,
// rank+1's first rows come in (one grouped exchange, every rank at the same point)
static lrcnn_status zr_first_band(Run &R, const Segment &S) {
    lrcnn_status st;
    for (const Segment::ZrRows &z : S.zr_to_above) {
        const TensorInfo &ti = R.P.t[z.t];
        const size_t rb = (size_t)ti.W * ti.Cp * R.E;
        if ((st = copy_rows(R, ti, R.ws + ti.zr_out_off, z.r1 - z.r0,
                            R.ws + ti.act_off + (size_t)(z.r0 - S.lo[0][z.t]) * rb, ti.cap,
                            z.r1 - z.r0)) != LRCNN_OK) return st;
    }
    return zr_exchange(R, S, false);
}

// row sharding: a BN op's per-rank sums over the rows the rank computes -> sums over the whole map
static lrcnn_status bn_allreduce(Run &R, double *buf, size_t n) {
    if (R.P.opts.world <= 1) return LRCNN_OK;
    if (!R.P.comm) return fail(LRCNN_E_STATE, "world > 1 needs lrcnn_plan_set_comm");
    const char *err = nullptr;
    if (comm_allreduce_f64((Comm *)R.P.comm, buf, n, R.st, &err))
        return fail(LRCNN_E_NCCL, err ? err : "fp64 allreduce failed");
    return LRCNN_OK;
}

// Training-mode BN statistics: per FP level of the segment's BN ops,
// one band sweep computes the ops their inputs need (the lower levels' statistics are final) and sums
// c, c^2 over the rows each band computes of every BN input (the interval rule gives each row to one
// band); then mean / var -> the affine coefficients the FP sweep applies.
static lrcnn_status bn_stat_sweeps_impl(Run &R, const Segment &S);
static lrcnn_status bn_stat_sweeps(Run &R, const Segment &S) {
    R.stash = true;
    const lrcnn_status st = bn_stat_sweeps_impl(R, S);
    R.stash = false; R.fmask = nullptr; R.redirect = -1;
    return st;
}

static lrcnn_status bn_stat_sweeps_impl(Run &R, const Segment &S) {
    Plan &P = R.P;
    lrcnn_status st;
    const int B = P.net.B;
    for (size_t l = 0; l < S.bn_fp_levels.size(); ++l) {
        bool banded = false;
        for (int j : S.bn_fp_levels[l]) {
            const OpInfo &o = P.op[j];
            CK(cudaMemsetAsync(R.ws + o.bn_sums_off, 0, 2 * (size_t)P.t[o.in_t].Cp * sizeof(double), R.st));
            if (o.in_t == S.in_t) {   // BN of the segment input: its full map is the checkpoint
                const TensorInfo &ti = P.t[o.in_t];
                ++P.launches;
                CK(bn_stats(R.prec, full_view(ckpt_ptr(R, o.in_t), ti), ti.ck_lo, ti.ck_lo + ti.ck_rows, B,
                            (double *)(R.ws + o.bn_sums_off), R.st));
            } else {
                banded = true;
            }
        }
        const bool tail = S.bn_tail >= 0 && l + 1 == S.bn_fp_levels.size();
        if (tail) R.redirect = P.op[S.bn_tail].in_t;
        if (banded) {
            R.fmask = &S.bn_fp_ops[l];
            for (int r = 0; r < (int)S.E.size(); ++r) {
                Nvtx nv("FP BN statistics level %d band %d", (int)l, r);
                if ((st = band_forward(R, S, r, true, false)) != LRCNN_OK) { R.fmask = nullptr; R.redirect = -1; return st; }
                if (r == 0 && zr_plan(P) && (st = zr_first_band(R, S)) != LRCNN_OK) { R.fmask = nullptr; return st; }
                for (int j : S.bn_fp_levels[l]) {
                    const OpInfo &o = P.op[j];
                    if (o.in_t == S.in_t || tail) continue;
                    // rows no earlier band computed (OverL bands overlap; 2PS bands are disjoint)
                    const int a = r > 0 ? std::max(S.a[r][o.in_t], S.b[r - 1][o.in_t]) : S.a[r][o.in_t];
                    const int b = S.b[r][o.in_t];
                    if (b <= a) continue;
                    ++P.launches;
                    ProfScope ps(R, 2, 0, j * 8 + 6);
                    CK(bn_stats(R.prec, act_view(R, S, r, o.in_t), a, b, B, (double *)(R.ws + o.bn_sums_off), R.st));
                }
            }
            R.fmask = nullptr;
        }
        R.redirect = -1;
        if (tail) {   // statistics of the tail BN's input over the full checkpoint it was written into
            const OpInfo &o = P.op[S.bn_tail];
            const TensorInfo &to = P.t[S.out_t];
            ++P.launches;
            ProfScope ps(R, 2, 0, S.bn_tail * 8 + 6);
            CK(bn_stats(R.prec, full_view(ckpt_ptr(R, S.out_t), to), to.ck_lo, to.ck_lo + to.ck_rows, B,
                        (double *)(R.ws + o.bn_sums_off), R.st));
        }
        for (int j : S.bn_fp_levels[l]) {
            const OpInfo &o = P.op[j];
            const TensorInfo &ti = P.t[o.in_t];
            if ((st = bn_allreduce(R, (double *)(R.ws + o.bn_sums_off), 2 * (size_t)ti.Cp)) != LRCNN_OK) return st;
            CK(bn_finalize_fwd(R.prec, (const double *)(R.ws + o.bn_sums_off), prm(R, o.b_off), prm(R, o.beta_off), ti.C,
                               ti.Cp, (double)B * ti.H * ti.W, (float *)(R.ws + o.bn_coef_off), R.st));
        }
        if (tail) {   // t = relu?(a*c + b + res) in place over the checkpoint (every element read, then written)
            const OpInfo &o = P.op[S.bn_tail];
            const TensorInfo &to = P.t[S.out_t];
            const View v = full_view(ckpt_ptr(R, S.out_t), to);
            View res;
            if (o.d.res >= 0) res = full_view(ckpt_ptr(R, o.d.res), P.t[o.d.res]);
            ++P.launches;
            ProfScope ps(R, 2, 0, S.bn_tail * 8 + 6);
            CK(bn_fwd(R.prec, v, res, v, (const float *)(R.ws + o.bn_coef_off), o.d.relu, to.ck_lo,
                      to.ck_lo + to.ck_rows, B, R.st));
            if (!P.capture.empty()) {
                lrcnn_status cs = capture_rows(R, S.out_t, v, to.ck_lo, to.ck_lo + to.ck_rows);
                if (cs != LRCNN_OK) return cs;
            }
        }
    }
    return LRCNN_OK;
}

static lrcnn_status run_forward(Run &R) {
    lrcnn_status st;
    {   // the dgrad weight transposes depend only on this step's weights: overlap them with the FP
        Plan &P = R.P;
        P.wt_pending = false;
        if (P.use_tc && P.side_stream && P.ev_wt && !P.profiling) {
            cudaStream_t ss = (cudaStream_t)P.side_stream;
            CK(cudaEventRecord((cudaEvent_t)P.ev_fork, R.st));
            CK(cudaStreamWaitEvent(ss, (cudaEvent_t)P.ev_fork, 0));
            if ((st = launch_transposes(R, ss)) != LRCNN_OK) return st;
            CK(cudaEventRecord((cudaEvent_t)P.ev_wt, ss));
            P.wt_pending = true;
        }
    }
    const bool sharded = R.P.opts.world > 1;
    for (const Segment &S : R.P.seg) {
        if (sharded && S.in_t != 0 && !S.in_xfers.empty())
            if ((st = exchange(R, S, full_view(ckpt_ptr(R, S.in_t), R.P.t[S.in_t]), false)) != LRCNN_OK) return st;
        if (!S.bn_fp_levels.empty() && (st = bn_stat_sweeps(R, S)) != LRCNN_OK) return st;
        if (S.bn_tail >= 0) continue;   // the last statistics sweep + the in-place BN produced the segment
        struct StashScope {   // BN segments: the FP sweep reads the stashed BN inputs
            Run &R; bool on;
            StashScope(Run &r_, const Segment &S) : R(r_), on(!S.bn_fp_levels.empty()) {
                if (on) { R.stash = true; R.fmask = &S.bn_fp_final; }
            }
            ~StashScope() { if (on) { R.stash = false; R.fmask = nullptr; } }
        } stash_scope(R, S);
        if (!S.fp_r0.empty()) {   // decoupled FP bands (N_FP < N_BP)
            Segment F = S;
            F.lo = S.fp_lo; F.a = S.fp_a; F.b = S.fp_b;
            F.E.clear();
            for (size_t k = 0; k < S.fp_r0.size(); ++k)
                F.E.push_back(S.E[k + 1 < S.fp_r0.size() ? S.fp_r0[k + 1] - 1 : S.E.size() - 1]);
            for (int k = 0; k < (int)S.fp_r0.size(); ++k) {
                Nvtx nv("FP seg %d merged band %d", (int)(&S - R.P.seg.data()), k);
                if ((st = band_forward_merged(R, S, F, k)) != LRCNN_OK) return st;
            }
            continue;
        }
        for (int r = 0; r < (int)S.E.size(); ++r) {
            Nvtx nv("FP seg %d band %d", (int)(&S - R.P.seg.data()), r);
            if ((st = band_forward(R, S, r, true, false)) != LRCNN_OK) return st;
            if (r == 0 && zr_plan(R.P) && (st = zr_first_band(R, S)) != LRCNN_OK) return st;
        }
    }
    return LRCNN_OK;
}

// ------------------------------------------------------------------ op backward on band rows [a, b)
// A band-internal tensor whose only reader is a stride-1 convolution gets its delta rows from that
// conv's dgrad alone, and the dgrad's input rows cover the tensor's band rows exactly (interval
// rule): the dgrad overwrites them (gate * acc) instead of accumulating into a zeroed buffer, and
// the 2PS carry of band r+1 is added (gated) right after it.  Saves the band-buffer memset and
// the dgrad epilogue's delta load.
// Fused residual gradient.  A band-internal block input t read by exactly one stride-1 convolution
// (role 0) and by one residual convolution u (role 1, same shape as its output) gets
//   delta(t) = gate(t) * (dgrad + delta(out_u))
// from the stride-1 conv's dgrad in write mode with delta(out_u) as a TMA-loaded addend, instead
// of a memset, an accumulating dgrad and a separate residual pass.  Rows of t that only the
// residual reads (the 2PS cache row below the dgrad's rows) are written gate * delta(out_u) by a
// row kernel.  Every band row of t must be covered by one of the two row ranges.  Returns u, or -1.
static int fused_res(const Plan &P, const Segment &S, int t) {
    if (!P.use_tc || P.opts.mode == LRCNN_OVERL || t == 0 || t == S.in_t || t == S.out_t) return -1;
    if (zr_plan(P)) return -1;   // (delta rows beyond the rank's own rows accumulate from several writers)
    if (P.opts.flags & LRCNN_FLAG_NO_FUSE_RES) return -1;
    const TensorInfo &ti = P.t[t];
    if (ti.cons.size() != 2) return -1;
    const Consumer &c0 = ti.cons[0].role == 0 ? ti.cons[0] : ti.cons[1];
    const Consumer &c1 = ti.cons[0].role == 0 ? ti.cons[1] : ti.cons[0];
    if (c0.role != 0 || c1.role != 1) return -1;
    const OpInfo &v = P.op[c0.op], &u = P.op[c1.op];
    if (v.d.kind != LRCNN_OP_CONV || v.d.s != 1 || u.d.kind != LRCNN_OP_CONV || u.d.res != t || c0.op >= c1.op)
        return -1;
    const TensorInfo &to = P.t[u.out_t];
    if (to.Cp != ti.Cp || to.W != ti.W || to.H != ti.H || P.t[u.out_t].seg != ti.seg) return -1;
    for (size_t r = 0; r < S.E.size(); ++r) {
        const int lo = S.lo[r][t], hi = S.b[r][t];
        const int va = S.a[r][v.out_t], vb = S.b[r][v.out_t];
        const int ra = vb > va ? std::max(0, va - v.d.p) : 0, rb = vb > va ? std::min(ti.H, vb - 1 - v.d.p + v.d.k) : 0;
        const int oa = S.a[r][u.out_t], ob = S.b[r][u.out_t];
        // the union of [ra, rb) and [oa, ob) must be exactly the band rows [lo, hi)
        int x0 = hi, x1 = lo;
        if (rb > ra) { x0 = std::min(x0, ra); x1 = std::max(x1, rb); }
        if (ob > oa) { x0 = std::min(x0, oa); x1 = std::max(x1, ob); }
        if (hi <= lo) continue;
        if (x0 != lo || x1 != hi) return -1;
        if (rb > ra && ob > oa && (ob < ra || rb < oa)) return -1;   // a gap between the two ranges
    }
    return c1.op;
}

static bool delta_overwrite(const Plan &P, const Segment &S, int t) {
    if (t == 0 || t == S.in_t || t == S.out_t || zr_plan(P)) return false;
    if (fused_res(P, S, t) >= 0) return true;
    const TensorInfo &ti = P.t[t];
    if (ti.cons.size() != 1 || ti.cons[0].role != 0) return false;
    const OpInfo &u = P.op[ti.cons[0].op];
    if (u.d.kind == LRCNN_OP_CONV) return u.d.s == 1;
    if (u.d.kind == LRCNN_OP_BN) {   // 1:1 reader: its band rows are exactly the tensor's rows (no cache, no carry)
        for (size_t r = 0; r < S.E.size(); ++r)
            if (S.lo[r][t] != S.a[r][t] || S.a[r][t] != S.a[r][u.out_t] || S.b[r][t] != S.b[r][u.out_t]) return false;
        return true;
    }
    // a non-overlapping max-pool that tiles the map exactly writes every input position once
    const TensorInfo &to = P.t[u.out_t];
    if (u.d.kind != LRCNN_OP_MAXPOOL) return false;
    if (u.d.k == u.d.s && u.d.p == 0 && to.H * u.d.k == ti.H && to.W * u.d.k == ti.W) return true;
    // an overlapping max-pool backward in its tiled-gather form writes every input row it covers
    // (all columns); the last window must reach the last row so the final band is covered too
    return pool_tiled_shape(u.d.k, u.d.s, ti.Cp) && (to.H - 1) * u.d.s - u.d.p + u.d.k >= ti.H;
}

// Residual rows of a fused block input (see fused_res) that the dgrad of op i (input rows [ra, rb),
// addend consumed or not) did not produce: rows outside [ra, rb) are written gate * delta(out_u),
// rows inside are added when the dgrad kernel did not take the addend.  with_carry: also add the
// 2PS carry of band r+1 (the dgrad, which normally does it, produced no rows in this band).
static lrcnn_status fused_res_rows(Run &R, const Segment &S, int s, int r, int i, int ra, int rb, bool add_done,
                                   bool with_carry) {
    Plan &P = R.P;
    const OpInfo &o = P.op[i];
    const int fu = fused_res(P, S, o.in_t);
    if (fu < 0) return LRCNN_OK;
    const TensorInfo &tt = P.t[o.in_t];
    const int tu = P.op[fu].out_t, oa = S.a[r][tu], ob = S.b[r][tu];
    const View dx = dlt_view(R, S, s, r, o.in_t), act = act_view(R, S, r, o.in_t);
    auto rows = [&](const View &src, int ya, int yb, int write) -> lrcnn_status {
        if (yb <= ya) return LRCNN_OK;
        EltArgs E;
        E.dy = src; E.dx = dx; E.act = act; E.gate = tt.relu;
        E.a = ya; E.b = yb; E.B = P.net.B; E.write = write;
        ++P.launches;
        ProfScope ps(R, 2, 0, i * 8 + 7);
        CK(simt_acc_gate(R.prec, E, R.st));
        return LRCNN_OK;
    };
    lrcnn_status st;
    if (ob > oa) {
        const View dres = sub_rows(dlt_view(R, S, s, r, tu), oa, ob, R.E);
        if (rb <= ra) {
            if ((st = rows(dres, oa, ob, 1)) != LRCNN_OK) return st;
        } else {
            if (!add_done && (st = rows(dres, std::max(oa, ra), std::min(ob, rb), 0)) != LRCNN_OK) return st;
            if ((st = rows(dres, oa, std::min(ob, ra), 1)) != LRCNN_OK) return st;
            if ((st = rows(dres, std::max(oa, rb), ob, 1)) != LRCNN_OK) return st;
        }
    }
    const int N = (int)S.E.size();
    if (with_carry && P.opts.mode == LRCNN_2PS && r + 1 < N) {
        const int clo = S.lo[r + 1][o.in_t], chi = S.a[r + 1][o.in_t];
        const View cv{R.ws + tt.carry_off, clo, chi - clo, tt.H, tt.W, tt.Cp, (long long)tt.carry_cap * tt.W * tt.Cp};
        if ((st = rows(cv, clo, chi, 0)) != LRCNN_OK) return st;
    }
    return LRCNN_OK;
}

static lrcnn_status op_backward(Run &R, const Segment &S, int s, int r, int i) {
    Plan &P = R.P;
    const OpInfo &o = P.op[i];
    const int t = o.out_t;
    const int a = S.a[r][t], b = S.b[r][t];
    // BN sums sweep (R.bneed): only the deltas the sweep needs, no weight / parameter gradients
    auto need = [&](int tid) { return !R.bneed || (*R.bneed)[tid]; };
    if (R.bneed && o.d.kind == LRCNN_OP_CONV) {
        if (b <= a || o.in_t == 0 || !need(o.in_t)) return LRCNN_OK;
        View dy = sub_rows(dlt_view(R, S, s, r, t), a, b, R.E);
        const TensorInfo &tin = P.t[o.in_t];
        DgradArgs A;
        A.dy = dy; A.dx = dlt_view(R, S, s, r, o.in_t); A.act = act_view(R, S, r, o.in_t);
        A.gate = tin.relu; A.w = prm(R, o.w_off); A.wt = R.ws + o.wt_off;
        A.gamma = o.d.epi == LRCNN_EPI_AFFINE ? prm(R, o.b_off) : nullptr;
        A.k = o.d.k; A.s = o.d.s; A.p = o.d.p; A.c_out = o.d.c_out; A.B = P.net.B;
        A.ra = std::max(0, a * o.d.s - o.d.p);
        A.rb = std::min(tin.H, (b - 1) * o.d.s - o.d.p + o.d.k);
        A.write = delta_overwrite(P, S, o.in_t) ? 1 : 0;
        ++P.launches;
        ProfScope ps(R, 0, conv_flops(P, o, b - a), i * 8 + 1, conv_bytes(P, o, a, b, 1, A.write ? 0 : 1, A.gate ? 1 : 0),
                     conv_bytes(P, o, a, b, 1, 0, 0, true));
        bool tc = false;
        if (P.use_tc) {
            tc = tc_conv_dgrad(A, R.st);
            lrcnn_status st0;
            if (tc) ++P.tc_launches;
            else if ((st0 = tc_declined(P, i, "dgrad")) != LRCNN_OK) return st0;
        }
        if (!tc) CK(simt_conv_dgrad(R.prec, A, R.st));
        CK(cudaGetLastError());
        const int N = (int)S.E.size();
        if (A.write && P.opts.mode == LRCNN_2PS && r + 1 < N) {   // + the carry of band r+1, gated
            const int ti_ = o.in_t, clo = S.lo[r + 1][ti_], chi = S.a[r + 1][ti_];
            if (chi > clo) {
                EltArgs E;
                E.dx = A.dx; E.act = A.act; E.gate = tin.relu;
                E.dy = View{R.ws + tin.carry_off, clo, chi - clo, tin.H, tin.W, tin.Cp,
                            (long long)tin.carry_cap * tin.W * tin.Cp};
                E.a = clo; E.b = chi; E.B = P.net.B;
                ++P.launches;
                CK(simt_acc_gate(R.prec, E, R.st));
            }
        }
        return LRCNN_OK;
    }
    if (o.d.kind == LRCNN_OP_BN) {   // delta(src) += gate * (a*da + p + q*c); delta(res) += gate * da
        if (b <= a) return LRCNN_OK;
        View dy = sub_rows(dlt_view(R, S, s, r, t), a, b, R.E);
        const float *coef = (const float *)(R.ws + o.bn_coef_off);
        if (o.in_t != 0 && need(o.in_t)) {
            const View x = act_view(R, S, r, o.in_t);
            ++P.launches;
            ProfScope ps(R, 2, 0, i * 8 + 7);
            // OverL: rows an earlier band also computed get only the linear term (the statistics terms
            // once per row); 2PS bands are disjoint (a == the previous band's end)
            const int cs = r > 0 ? std::max(a, S.b[r - 1][t]) : a;
            CK(bn_bwd(R.prec, dy, x, dlt_view(R, S, s, r, o.in_t), x, P.t[o.in_t].relu,
                      delta_overwrite(P, S, o.in_t) ? 1 : 0, coef, a, b, P.net.B, cs, R.st));
        }
        if (o.d.res > 0 && need(o.d.res)) {
            EltArgs A;
            A.dy = dy; A.dx = dlt_view(R, S, s, r, o.d.res); A.act = act_view(R, S, r, o.d.res);
            A.gate = P.t[o.d.res].relu; A.a = a; A.b = b; A.B = P.net.B;
            ++P.launches;
            ProfScope ps(R, 2, 0, i * 8 + 7);
            CK(simt_acc_gate(R.prec, A, R.st));
        }
        return LRCNN_OK;
    }
    if (b <= a) {   // no rows of this op in band r; a fused block input still gets its residual rows
        if (o.d.kind == LRCNN_OP_CONV && o.in_t != 0) return fused_res_rows(R, S, s, r, i, 0, 0, false, true);
        return LRCNN_OK;
    }
    const int B = P.net.B;
    View dy = sub_rows(dlt_view(R, S, s, r, t), a, b, R.E);      // complete, gated delta rows
    const TensorInfo &tin = P.t[o.in_t];
    const bool need_dx = o.in_t != 0;
    if (o.d.kind == LRCNN_OP_CONV) {
        float *g = R.grads;
        lrcnn_status st0;
        const void *gamma = o.d.epi == LRCNN_EPI_AFFINE ? prm(R, o.b_off) : nullptr;
        // L2-sized row chunks (1x1 stride-1 convolutions, LRCNN_L2_CHUNK_MB > 0): the wgrad of a chunk
        // (side stream) and its dgrad (main stream) run together over the same rows, so the second
        // reader of delta(out) and of the input activation finds them in L2 instead of HBM
        std::vector<int> cuts = {a, b};
        {
            static const int chunk_mb = env_chunk_mb();
            const bool pointwise = o.d.k == 1 && o.d.s == 1 && o.d.p == 0 && need_dx;
            if (chunk_mb > 0 && pointwise) {
                const double row_bytes = (double)B * P.t[t].W * (P.t[t].Cp + tin.Cp) * R.E;
                const int per = std::max(1, (int)((double)chunk_mb * 1048576.0 / row_bytes));
                if (b - a > per) {
                    cuts.clear();
                    const int n = (b - a + per - 1) / per;
                    for (int c = 0; c <= n; ++c) cuts.push_back(a + (int)((long long)(b - a) * c / n));
                }
            }
        }
        bool db_done = true, add_done_all = true, add_any = false;
        int fu = -1, ra_all = 0, rb_all = 0, write_mode = 0;
        DgradArgs D0;
        for (size_t c = 0; c + 1 < cuts.size(); ++c) {
            const int ca = cuts[c], cb = cuts[c + 1];
            const View dyc = sub_rows(dlt_view(R, S, s, r, t), ca, cb, R.E);
            // fused pointwise dgrad + wgrad (one pass over delta(out) and x, tc_conv_dwgrad) when the
            // shape has a kernel; else wgrad on the side stream and dgrad on the main stream
            if (P.use_tc && need_dx && cuts.size() == 2 && o.d.k == 1 && o.d.s == 1 && o.d.p == 0) {
                WgradArgs A;
                A.dy = dyc; A.x = act_view(R, S, r, o.in_t); A.dw = g + o.w_off; A.gamma = gamma;
                A.k = 1; A.s = 1; A.p = 0; A.c_out = o.d.c_out; A.a = ca; A.b = cb; A.B = B;
                if (o.d.epi == LRCNN_EPI_BIAS) A.db = g + o.b_off;
                if (o.d.epi == LRCNN_EPI_AFFINE) { A.db = g + o.beta_off; A.dg = g + o.b_off; A.w = prm(R, o.w_off); }
                DgradArgs D;
                D.dy = dyc; D.dx = dlt_view(R, S, s, r, o.in_t); D.act = act_view(R, S, r, o.in_t);
                D.gate = tin.relu; D.w = prm(R, o.w_off); D.wt = R.ws + o.wt_off; D.gamma = gamma;
                D.k = 1; D.s = 1; D.p = 0; D.c_out = o.d.c_out; D.B = B;
                D.ra = ca; D.rb = std::min(tin.H, cb);
                D.write = delta_overwrite(P, S, o.in_t) ? 1 : 0;
                const int fu2 = fused_res(P, S, o.in_t);
                if (fu2 >= 0) {
                    const int tu = P.op[fu2].out_t, oa = S.a[r][tu], ob = S.b[r][tu];
                    if (ob > oa) { D.add = sub_rows(dlt_view(R, S, s, r, tu), oa, ob, R.E); D.add_on = 1; }
                }
                bool fused;
                {
                    ProfScope ps(R, 0, 2.0 * conv_flops(P, o, cb - ca), i * 8 + 1,
                                 conv_bytes(P, o, ca, cb, 1, D.write ? 0 : 1, D.gate ? 1 : 0) + conv_bytes(P, o, ca, cb, 2)
                                     - conv_bytes(P, o, ca, cb, 2, 0, 0, false) + 8.0 * o.d.k * o.d.k * tin.Cp * o.d.c_out,
                                 conv_bytes(P, o, ca, cb, 1, 0, 0, true) + conv_bytes(P, o, ca, cb, 2, 0, 0, true));
                    fused = tc_conv_dwgrad(A, D, R.st);
                    if (!fused && tc_take_error())
                        return fail(LRCNN_E_CUDA, "fused dgrad + wgrad launch failed at op " + std::to_string(i));
                }
                if (fused) {
                    P.launches += 1;
                    ++P.tc_launches;
                    CK(cudaGetLastError());
                    db_done = db_done && A.db_done;
                    if (A.dg && !A.dg_done) return fail(LRCNN_E_STATE, "fused dgrad+wgrad did not take dgamma");
                    ra_all = D.ra; rb_all = D.rb; write_mode = D.write; fu = fu2;
                    add_done_all = D.add_done; add_any = D.add_done;
                    D0 = D;
                    continue;
                }
            }
            // wgrad and the bias/affine reduction only read complete data of this band: run them on
            // the side stream so they overlap the dgrad chain (joined at the end of the band)
            cudaStream_t gst = R.st;
            if (R.side) { CK(fork_side(R)); gst = R.side; }
            {
                WgradArgs A;
                A.dy = dyc; A.x = act_view(R, S, r, o.in_t); A.dw = g + o.w_off; A.gamma = gamma;
                A.k = o.d.k; A.s = o.d.s; A.p = o.d.p; A.c_out = o.d.c_out; A.a = ca; A.b = cb; A.B = B;
                // bias (VGG) or affine (ResNet) parameter gradients fused into the tensor-core wgrad:
                // db / dbeta = sum dy, dgamma = sum_{tap,ci} W * (sum_p dy x)
                if (o.d.epi == LRCNN_EPI_BIAS) A.db = g + o.b_off;
                if (o.d.epi == LRCNN_EPI_AFFINE) { A.db = g + o.beta_off; A.dg = g + o.b_off; A.w = prm(R, o.w_off); }
                ++P.launches;
                ProfScope ps(R, 1, conv_flops(P, o, cb - ca), i * 8 + 2, conv_bytes(P, o, ca, cb, 2),
                             conv_bytes(P, o, ca, cb, 2, 0, 0, true));
                bool tc = false;
                if (P.use_tc) {
                    tc = tc_conv_wgrad(A, gst);
                    if (tc) ++P.tc_launches;
                    else if ((st0 = tc_declined(P, i, "wgrad")) != LRCNN_OK) return st0;
                }
                if (!tc) CK(simt_conv_wgrad(R.prec, A, gst));
                CK(cudaGetLastError());
                db_done = db_done && A.db_done;
                // dgamma comes only from the wgrad (sum_{tap,ci} W * sum_p dy x, exact for gamma = 0)
                if (A.dg && !A.dg_done) return fail(LRCNN_E_STATE, "wgrad of op " + std::to_string(i) + " did not take dgamma");
            }
            if (o.d.epi != LRCNN_EPI_NONE && !db_done && cuts.size() > 2)
                return fail(LRCNN_E_STATE, "chunked wgrad of op " + std::to_string(i) + " did not take the bias sums");
            if (need_dx) {
                DgradArgs A;
                A.dy = dyc; A.dx = dlt_view(R, S, s, r, o.in_t); A.act = act_view(R, S, r, o.in_t);
                A.gate = tin.relu; A.w = prm(R, o.w_off); A.wt = R.ws + o.wt_off; A.gamma = gamma;
                A.k = o.d.k; A.s = o.d.s; A.p = o.d.p; A.c_out = o.d.c_out; A.B = B;
                A.ra = std::max(0, ca * o.d.s - o.d.p);
                A.rb = std::min(tin.H, (cb - 1) * o.d.s - o.d.p + o.d.k);
                if (c == 0) ra_all = A.ra;
                rb_all = A.rb;
                A.write = delta_overwrite(P, S, o.in_t) ? 1 : 0;
                write_mode = A.write;
                fu = fused_res(P, S, o.in_t);   // residual conv whose output delta is the addend
                if (fu >= 0) {
                    const int tu = P.op[fu].out_t, oa = S.a[r][tu], ob = S.b[r][tu];
                    if (ob > oa) {
                        A.add = sub_rows(dlt_view(R, S, s, r, tu), oa, ob, R.E);
                        A.add_on = 1;
                    }
                }
                ++P.launches;
                ProfScope ps(R, 0, conv_flops(P, o, cb - ca), i * 8 + 1,
                             conv_bytes(P, o, ca, cb, 1, A.write ? 0 : 1, A.gate ? 1 : 0),
                             conv_bytes(P, o, ca, cb, 1, 0, 0, true));
                bool tc = false;
                if (P.use_tc) {
                    tc = tc_conv_dgrad(A, R.st);
                    if (tc) ++P.tc_launches;
                    else if ((st0 = tc_declined(P, i, "dgrad")) != LRCNN_OK) return st0;
                }
                if (!tc) CK(simt_conv_dgrad(R.prec, A, R.st));
                CK(cudaGetLastError());
                add_done_all = add_done_all && A.add_done;
                add_any = add_any || A.add_done;
                D0 = A;
            }
        }
        if (add_any && !add_done_all) return fail(LRCNN_E_STATE, "residual addend taken by some dgrad chunks only");
        if (o.d.epi != LRCNN_EPI_NONE && !db_done) {   // bias / beta: column sums of dy
            ParamGradArgs A;
            A.dy = dy;
            A.db = g + (o.d.epi == LRCNN_EPI_AFFINE ? o.beta_off : o.b_off);
            A.c_out = o.d.c_out; A.a = a; A.b = b; A.B = B;
            ++P.launches;
            ProfScope ps(R, 2, 0, i * 8 + 3);
            CK(simt_param_grad(R.prec, A, R.side ? R.side : R.st));
        }
        if (need_dx) {
            if (fu >= 0) {   // residual rows the dgrad did not take
                lrcnn_status rs = fused_res_rows(R, S, s, r, i, ra_all, rb_all, add_done_all && add_any, false);
                if (rs != LRCNN_OK) return rs;
            }
            const int N = (int)S.E.size();
            if (write_mode && P.opts.mode == LRCNN_2PS && r + 1 < N) {   // + the carry of band r+1, gated
                const int t = o.in_t, clo = S.lo[r + 1][t], chi = S.a[r + 1][t];
                if (chi > clo) {
                    EltArgs E;
                    E.dx = D0.dx; E.act = D0.act; E.gate = tin.relu;
                    E.dy = View{R.ws + tin.carry_off, clo, chi - clo, tin.H, tin.W, tin.Cp,
                                (long long)tin.carry_cap * tin.W * tin.Cp};
                    E.a = clo; E.b = chi; E.B = B;
                    ++P.launches;
                    ProfScope ps(R, 2, 0, i * 8 + 7);
                    CK(simt_acc_gate(R.prec, E, R.st));
                }
            }
        }
        if (o.d.res >= 0 && fused_res(P, S, o.d.res) != i && alias_delta(P, S, o.d.res) < 0) {
            // (fused: added by the block input's dgrad; aliased: the residual's delta IS dy)
            const TensorInfo &tr = P.t[o.d.res];
            EltArgs A;
            A.dy = dy; A.dx = dlt_view(R, S, s, r, o.d.res); A.act = act_view(R, S, r, o.d.res);
            A.gate = tr.relu; A.a = a; A.b = b; A.B = B;
            if (o.d.res != 0) {
                ++P.launches;
                ProfScope ps(R, 2, 0, i * 8 + 7);
                CK(simt_acc_gate(R.prec, A, R.st));
            }
        }
    } else if (o.d.kind == LRCNN_OP_MAXPOOL) {
        if (need_dx && need(o.in_t)) {
            PoolArgs A;
            A.dy = dy; A.dx = dlt_view(R, S, s, r, o.in_t); A.act = act_view(R, S, r, o.in_t);
            A.gate = tin.relu; A.k = o.d.k; A.s = o.d.s; A.p = o.d.p; A.a = a; A.b = b; A.B = B;
            A.ra = std::max(0, a * o.d.s - o.d.p);
            A.rb = std::min(tin.H, (b - 1) * o.d.s - o.d.p + o.d.k);
            // a non-overlapping pool whose input is band-internal with this pool as its only
            // consumer and no delta carried in from band r+1 is the only writer of those rows
            const int N = (int)S.E.size();
            const bool carry_in = P.opts.mode == LRCNN_2PS && r + 1 < N && S.lo[r + 1][o.in_t] < S.a[r + 1][o.in_t];
            const bool single = delta_overwrite(P, S, o.in_t);
            A.acc = !(single || (o.d.k == o.d.s && o.d.p == 0 && o.in_t != S.in_t && tin.cons.size() == 1 && !carry_in));
            {
                P.launches += simt_pool_bwd_launches(A);
                ProfScope ps(R, 2, 0, i * 8 + 5);
                CK(simt_pool_bwd(R.prec, A, R.st));
            }
            if (single && carry_in) {   // + the carry of band r+1, gated (as after a single-writer dgrad)
                const int t = o.in_t, clo = S.lo[r + 1][t], chi = S.a[r + 1][t];
                EltArgs E;
                E.dx = A.dx; E.act = A.act; E.gate = tin.relu;
                E.dy = View{R.ws + tin.carry_off, clo, chi - clo, tin.H, tin.W, tin.Cp,
                            (long long)tin.carry_cap * tin.W * tin.Cp};
                E.a = clo; E.b = chi; E.B = B;
                ++P.launches;
                ProfScope ps(R, 2, 0, i * 8 + 7);
                CK(simt_acc_gate(R.prec, E, R.st));
            }
        }
    } else {
        for (int which = 0; which < 2; ++which) {
            int tid = which ? o.d.res : o.in_t;
            if (tid == 0 || !need(tid)) continue;
            EltArgs A;
            A.dy = dy; A.dx = dlt_view(R, S, s, r, tid); A.act = act_view(R, S, r, tid);
            A.gate = P.t[tid].relu; A.a = a; A.b = b; A.B = B;
            ++P.launches;
            ProfScope ps(R, 2, 0, i * 8 + 7);
            CK(simt_acc_gate(R.prec, A, R.st));
        }
    }
    return LRCNN_OK;
}

// Data-parallel replicas (LRCNN_FLAG_DP): sum the gradient range [lo, hi) over the replicas on the
// communication stream once everything enqueued so far on the main stream (the range's last
// writers) is done; the backward goes on meanwhile.  dp_join makes the main stream wait for the
// reductions (before the SGD / the caller reads the gradient).
// Row sharding (opts.world > 1) uses the same per-segment buckets: a segment's weight gradient on
// this rank is final once its band sweep is done, so it is summed over the ranks while the earlier
// segments' backward runs.
static lrcnn_status dp_reduce(Run &R, size_t lo, size_t hi) {
    Plan &P = R.P;
    if ((P.dp_world <= 1 && P.opts.world <= 1) || hi <= lo) return LRCNN_OK;
    if (!P.comm) return fail(LRCNN_E_STATE, "world > 1 needs lrcnn_plan_set_comm");
    if (!P.comm_stream) {   // created on the first (eager) call, before any graph capture
        cudaStream_t cs;
        cudaEvent_t e0, e1;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
        P.comm_stream = cs; P.ev_comm = e0; P.ev_comm_done = e1;
    }
    cudaStream_t cs = (cudaStream_t)P.comm_stream;
    CK(cudaEventRecord((cudaEvent_t)P.ev_comm, R.st));
    CK(cudaStreamWaitEvent(cs, (cudaEvent_t)P.ev_comm, 0));
    const char *err = nullptr;
    if (comm_allreduce_f32((Comm *)P.comm, R.grads + lo, hi - lo, cs, &err))
        return fail(LRCNN_E_NCCL, err ? err : "allreduce failed");
    R.dp_pending = true;
    return LRCNN_OK;
}

static lrcnn_status dp_join(Run &R) {
    if (!R.dp_pending) return LRCNN_OK;
    CK(cudaEventRecord((cudaEvent_t)R.P.ev_comm_done, (cudaStream_t)R.P.comm_stream));
    CK(cudaStreamWaitEvent(R.st, (cudaEvent_t)R.P.ev_comm_done, 0));
    R.dp_pending = false;
    return LRCNN_OK;
}

static lrcnn_status run_backward(Run &R) {
    Plan &P = R.P;
    lrcnn_status st;
    const bool recompute = !(P.seg.size() == 1 && P.seg[0].E.size() == 1);
    static const int side_on = getenv("LRCNN_SIDE") ? atoi(getenv("LRCNN_SIDE")) : 1;
    if (side_on && !P.profiling) {
        if (!P.side_stream) {   // created on the first (eager) call, before any graph capture
            cudaStream_t ss;
            cudaEvent_t e0, e1;
            CK(cudaStreamCreateWithFlags(&ss, cudaStreamNonBlocking));
            CK(cudaEventCreateWithFlags(&e0, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&e1, cudaEventDisableTiming));
            P.side_stream = ss; P.ev_fork = e0; P.ev_join = e1;
            cudaEvent_t e2;
            CK(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
            P.ev_wt = e2;
        }
        R.side = (cudaStream_t)P.side_stream;
    }
    // transposed weights for the tensor-core dgrad: launched on the side stream during the FP, or here
    if (P.wt_pending) {
        CK(cudaStreamWaitEvent(R.st, (cudaEvent_t)P.ev_wt, 0));
        P.wt_pending = false;
    } else if (P.use_tc) {
        if ((st = launch_transposes(R, R.st)) != LRCNN_OK) return st;
    }
    for (int s = (int)P.seg.size() - 1; s >= 0; --s) {
        const Segment &S = P.seg[s];
        if (S.in_t != 0) {
            const TensorInfo &ti = P.t[S.in_t];
            CK(cudaMemsetAsync(R.ws + P.dfull_off[(s + 1) & 1], 0, (size_t)P.net.B * ti.dl_rows * ti.W * ti.Cp * R.E,
                               R.st));
        }
        const int N = (int)S.E.size();
        auto band_bp = [&](int r) -> lrcnn_status {
            lrcnn_status st;
            if (recompute && (st = band_forward(R, S, r, false, true)) != LRCNN_OK) return st;
            for (auto it = S.ops.rbegin(); it != S.ops.rend(); ++it) {
                const int i = *it;
                // delta slots first written by op i's backward (plan: delta_slots).  A slot that held
                // an earlier tensor's delta in this band may still be read by that tensor's wgrad on
                // the side stream: join it first.  Then zero the slot and add the carry of band r+1
                // (R6), unless the single writer overwrites it.
                bool join = false;
                for (int t : S.tensors)
                    if (t != S.out_t && P.t[t].dfw == i && P.t[t].dreuse) join = true;
                if (join) CK(join_side(R));
                for (int t : S.tensors) {
                    const TensorInfo &ti = P.t[t];
                    if (t == S.out_t || ti.dfw != i || delta_overwrite(P, S, t)) continue;
                    size_t rb = (size_t)ti.W * ti.Cp * R.E;
                    int rows = S.hb[r][t] - S.lo[r][t];
                    if (rows > 0)
                        CK(cudaMemset2DAsync(R.ws + ti.dlt_off, ti.cap * rb, 0, rows * rb, P.net.B, R.st));
                    if (P.opts.mode == LRCNN_2PS && r + 1 < N) {
                        int clo = S.lo[r + 1][t], chi = S.a[r + 1][t];
                        if (chi > clo) {
                            if ((st = copy_rows(R, ti, R.ws + ti.dlt_off + (size_t)(clo - S.lo[r][t]) * rb, ti.cap,
                                                R.ws + ti.carry_off, ti.carry_cap, chi - clo)) != LRCNN_OK) return st;
                        }
                    }
                    if (r == 0 && ti.zr_out_r1 > ti.zr_out_r0)   // + the delta rank-1 computed for my first rows
                        CK(add_rows(R.prec, dlt_view(R, S, s, r, t), ti.zr_out_r0, ti.zr_out_r1, R.ws + ti.zr_din_off,
                                    P.net.B, R.st));
                }
                const int to = P.op[i].out_t;
                // zero-redundancy: the delta of rank+1's rows [HI, hb) of op i's output is complete too
                if (r == N - 1 && to != S.out_t && P.t[to].zr_in_r1 > P.t[to].zr_in_r0) {
                    const TensorInfo &ti = P.t[to];
                    const size_t rb = (size_t)ti.W * ti.Cp * R.E;
                    if ((st = copy_rows(R, ti, R.ws + ti.zr_dout_off, ti.zr_in_r1 - ti.zr_in_r0,
                                        R.ws + ti.dlt_off + (size_t)(ti.zr_in_r0 - S.lo[r][to]) * rb, ti.cap,
                                        ti.zr_in_r1 - ti.zr_in_r0)) != LRCNN_OK) return st;
                }
                // the 2PS carry out of op i's output: its cached rows [lo_r, a_r) are complete once
                // every consumer has run (all later in op order); copy them before the slot is reused
                if (P.opts.mode == LRCNN_2PS && r > 0 && to != S.out_t && P.t[to].dfw >= 0) {
                    const TensorInfo &ti = P.t[to];
                    int rows = S.a[r][to] - S.lo[r][to];
                    if (rows > 0 && (st = copy_rows(R, ti, R.ws + ti.carry_off, ti.carry_cap, R.ws + ti.dlt_off, ti.cap,
                                                    rows)) != LRCNN_OK) return st;
                }
                if (R.bn_level && std::find(R.bn_level->begin(), R.bn_level->end(), i) != R.bn_level->end()) {
                    // BN sums sweep: the delta of op i's output is complete -- sum da, da*xh over its rows
                    const OpInfo &o = P.op[i];
                    const int a = S.a[r][to], b = S.b[r][to];
                    if (b > a) {
                        ++P.launches;
                        ProfScope ps(R, 2, 0, i * 8 + 7);
                        CK(bn_sums(R.prec, sub_rows(dlt_view(R, S, s, r, to), a, b, R.E), act_view(R, S, r, o.in_t),
                                   (const float *)(R.ws + o.bn_coef_off), a, b, P.net.B,
                                   (double *)(R.ws + o.bn_S_off), R.st));
                    }
                    continue;
                }
                if (R.bops && !(*R.bops)[i]) continue;
                if ((st = op_backward(R, S, s, r, i)) != LRCNN_OK) return st;
            }
            CK(join_side(R));
            if (r == N - 1 && zr_plan(P) && (st = zr_exchange(R, S, true)) != LRCNN_OK) return st;
            return LRCNN_OK;
        };
        // BN BP stash: the first sweep of the segment writes the stashed BN inputs, the later ones
        // recompute only the other ops (R.fmask in band_forward)
        struct BpStash {
            Run &R;
            BpStash(Run &r_, const Segment &S) : R(r_) { if (!S.bp_stash_off.empty()) R.bp_stash = &S.bp_stash_off; }
            ~BpStash() { R.bp_stash = nullptr; R.fmask = nullptr; }
        } bp_stash_scope(R, S);
        bool first_sweep = true;
        auto next_sweep = [&]() {
            if (!first_sweep && !S.bn_bp_recompute.empty()) R.fmask = &S.bn_bp_recompute;
            first_sweep = false;
        };
        // training-mode BN: one sums sweep per BP level, deepest BN ops first
        for (size_t l = 0; l < S.bn_bp_levels.size(); ++l) {
            next_sweep();
            for (int j : S.bn_bp_levels[l])
                CK(cudaMemsetAsync(R.ws + P.op[j].bn_S_off, 0, 2 * (size_t)P.t[P.op[j].out_t].Cp * sizeof(double), R.st));
            R.bops = &S.bn_bp_ops[l]; R.bneed = &S.bn_bp_need[l]; R.bn_level = &S.bn_bp_levels[l];
            for (int r = N - 1; r >= 0; --r) {
                Nvtx nv("BP BN sums level %d band %d", (int)l, r);
                if ((st = band_bp(r)) != LRCNN_OK) return st;
            }
            R.bops = nullptr; R.bneed = nullptr; R.bn_level = nullptr;
            for (int j : S.bn_bp_levels[l]) {
                const OpInfo &o = P.op[j];
                const TensorInfo &ts = P.t[o.in_t];
                // dgamma, dbeta += this rank's sums (the per-segment gradient buckets sum them over the
                // ranks); p, q from the sums over every rank (recomputed after the all-reduce)
                CK(bn_finalize_bwd((const double *)(R.ws + o.bn_S_off), (float *)(R.ws + o.bn_coef_off), ts.C, ts.Cp,
                                   (double)P.net.B * ts.H * ts.W, R.grads ? R.grads + o.b_off : nullptr,
                                   R.grads ? R.grads + o.beta_off : nullptr, R.st));
                if (P.opts.world > 1) {
                    if ((st = bn_allreduce(R, (double *)(R.ws + o.bn_S_off), 2 * (size_t)ts.Cp)) != LRCNN_OK) return st;
                    CK(bn_finalize_bwd((const double *)(R.ws + o.bn_S_off), (float *)(R.ws + o.bn_coef_off), ts.C,
                                       ts.Cp, (double)P.net.B * ts.H * ts.W, nullptr, nullptr, R.st));
                }
            }
        }
        next_sweep();
        for (int r = N - 1; r >= 0; --r) {
            Nvtx nv("BP seg %d band %d", s, r);
            if ((st = band_bp(r)) != LRCNN_OK) return st;
        }
        if (P.opts.world > 1 && S.in_t != 0 && !S.in_xfers.empty())
            if ((st = exchange(R, S, dfull_view(R.ws + P.dfull_off[(s + 1) & 1], P.t[S.in_t]), true)) != LRCNN_OK)
                return st;
        // this segment's weight gradient is final (its side-stream work joined at the band ends)
        if (R.grads && (st = dp_reduce(R, P.seg_grad_lo[s], P.seg_grad_hi[s])) != LRCNN_OK) return st;
    }
    return LRCNN_OK;
}

static lrcnn_status check_ws(Plan &P, void *ws, size_t ws_bytes) {
    if (!ws) return fail(LRCNN_E_WORKSPACE, "workspace is NULL");
    if (ws_bytes < P.ws_bytes) return fail(LRCNN_E_WORKSPACE, "workspace too small: need " + std::to_string(P.ws_bytes));
    return LRCNN_OK;
}

}  // namespace lrcnn

using namespace lrcnn;

// Replays a captured CUDA graph of `eager` while the call's key (its pointer arguments, stream, lr)
// is unchanged: the first call runs eagerly (warms caches and function attributes), the second
// captures and launches the graph, later ones only launch it.  Eager when graphs are off, on the
// legacy stream, while profiling, or with a communicator that cannot be captured.
template <typename F>
static lrcnn_status graph_run(Plan &P, int slot, const uintptr_t (&key)[9], void *stream, F &&eager) {
    static const int graphs = getenv("LRCNN_GRAPH") ? atoi(getenv("LRCNN_GRAPH")) : 1;
    if (!graphs || stream == nullptr || P.profiling || !P.capture.empty() ||
        (P.comm && !comm_graph_safe((Comm *)P.comm))) {
        P.graph_calls[slot] = 0;
        return eager();
    }
    const bool same = std::memcmp(key, P.graph_key[slot], sizeof(key)) == 0;
    if (same && P.graph_exec[slot]) {
        CK(cudaGraphLaunch((cudaGraphExec_t)P.graph_exec[slot], (cudaStream_t)stream));
        P.launches = P.graph_launches[slot];
        P.tc_launches = P.graph_tc_launches[slot];
        P.simt_fallbacks = P.graph_simt_fallbacks[slot];
        P.fwd_done = false;
        return LRCNN_OK;
    }
    P.graph_calls[slot] = same ? P.graph_calls[slot] + 1 : 1;
    std::memcpy(P.graph_key[slot], key, sizeof(key));
    if (P.graph_exec[slot]) { cudaGraphExecDestroy((cudaGraphExec_t)P.graph_exec[slot]); P.graph_exec[slot] = nullptr; }
    if (P.graph_calls[slot] < 2) return eager();
    cudaStream_t cs = (cudaStream_t)stream;
    CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    lrcnn_status st = eager();
    cudaGraph_t g = nullptr;
    cudaError_t ce = cudaStreamEndCapture(cs, &g);
    if (st != LRCNN_OK) { if (g) cudaGraphDestroy(g); return st; }
    if (ce != cudaSuccess) return fail(LRCNN_E_CUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(ce));
    cudaGraphExec_t ge = nullptr;
    ce = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    if (ce != cudaSuccess) return fail(LRCNN_E_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(ce));
    P.graph_exec[slot] = ge;
    P.graph_launches[slot] = P.launches;
    P.graph_tc_launches[slot] = P.tc_launches;
    P.graph_simt_fallbacks[slot] = P.simt_fallbacks;
    CK(cudaGraphLaunch(ge, cs));
    return LRCNN_OK;
}

extern "C" {

const char *lrcnn_last_error(void) { return g_err.c_str(); }
const char *lrcnn_version(void) { return "lrcnn-b200 0.1 (sm_100a)"; }

lrcnn_status lrcnn_plan(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, lrcnn_plan_t **out) {
    if (!out) return fail(LRCNN_E_ARG, "out is NULL");
    *out = nullptr;
    lrcnn_plan_t *p = new lrcnn_plan_t();
    std::string err;
    lrcnn_plan_opts o = opts ? *opts : lrcnn_plan_opts{};
    const bool dp = opts && (opts->flags & LRCNN_FLAG_DP) && opts->world > 1;
    if (dp) {   // replicas: every rank plans the whole image; the comm is used for the gradient only
        if (opts->rank < 0 || opts->rank >= opts->world) { delete p; return fail(LRCNN_E_ARG, "rank out of range"); }
        o.world = 1;
        o.rank = 0;
    }
    lrcnn_status st = build_plan(net, opts ? &o : nullptr, p->P, err);
    if (st != LRCNN_OK) { delete p; return fail(st, err); }
    if (dp) { p->P.dp_world = opts->world; p->P.dp_rank = opts->rank; }
    {   // gradient bucket of every segment: its convolutions' parameters are contiguous (op order)
        Plan &P = p->P;
        P.seg_grad_lo.assign(P.seg.size(), 0);
        P.seg_grad_hi.assign(P.seg.size(), 0);
        for (size_t si = 0; si < P.seg.size(); ++si) {
            size_t lo = (size_t)-1, hi = 0;
            for (int i : P.seg[si].ops) {
                const OpInfo &oi = P.op[i];
                if (oi.d.kind != LRCNN_OP_CONV && oi.d.kind != LRCNN_OP_BN) continue;
                lo = std::min(lo, oi.d.kind == LRCNN_OP_BN ? oi.b_off : oi.w_off);
                hi = std::max(hi, oi.w_off + oi.w_cnt);
                if (oi.b_cnt) hi = std::max(hi, oi.b_off + oi.b_cnt);
                if (oi.beta_cnt) hi = std::max(hi, oi.beta_off + oi.beta_cnt);
            }
            if (lo != (size_t)-1) { P.seg_grad_lo[si] = lo; P.seg_grad_hi[si] = hi; }
        }
    }
    p->P.use_tc = p->P.opts.prec == LRCNN_BF16 && !(p->P.opts.flags & LRCNN_FLAG_NO_TCGEN05) && tc_available();
    *out = p;
    return LRCNN_OK;
}

// Budget-driven planning (Eqs. (9)-(10): choose the band count
// N from the memory budget M, the paper's greedy "the largest band that fits, i.e. the smallest N").
// The memory model is the plan's exact workspace bytes (reading R10), not the garbled Eq. (12).
lrcnn_status lrcnn_plan_budget(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, size_t budget_bytes,
                               int max_bands, lrcnn_plan_t **out, int *n_bands) {
    if (!out || !opts || !net) return fail(LRCNN_E_ARG, "net, opts or out is NULL");
    *out = nullptr;
    if (opts->mode == LRCNN_COLUMN) return fail(LRCNN_E_ARG, "budget planning needs a row-centric mode");
    if (max_bands < 1) return fail(LRCNN_E_ARG, "max_bands must be >= 1");
    size_t best_ws = (size_t)-1;
    for (int n = 1; n <= max_bands; ++n) {
        lrcnn_plan_opts o = *opts;
        o.band_rows = 0;
        o.n_bands = n;
        lrcnn_plan_t *p = nullptr;
        if (lrcnn_plan(net, &o, &p) != LRCNN_OK) continue;
        const size_t ws = p->P.ws_bytes;
        if (ws <= budget_bytes) {
            *out = p;
            if (n_bands) *n_bands = n;
            return LRCNN_OK;
        }
        best_ws = std::min(best_ws, ws);
        lrcnn_plan_free(p);
    }
    return fail(LRCNN_E_INFEASIBLE, "no band count <= " + std::to_string(max_bands) + " fits the budget of " +
                                        std::to_string(budget_bytes) + " bytes (smallest workspace " +
                                        std::to_string(best_ws) + ")");
}

// The 2PS greedy of Eq. (12): min N_BP first, then the largest first band H_1^L
// whose exact workspace fits; the first band is searched on a 1/64 grid of the segment outputs from
// the whole height down to the equal split (first_pm = 0).
lrcnn_status lrcnn_plan_greedy(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, size_t budget_bytes,
                               int max_bands, lrcnn_plan_t **out, int *n_bands, int *first_pm) {
    if (!out || !opts || !net) return fail(LRCNN_E_ARG, "net, opts or out is NULL");
    *out = nullptr;
    if (opts->mode != LRCNN_2PS) return fail(LRCNN_E_ARG, "the greedy first band is a 2PS plan");
    if (max_bands < 1) return fail(LRCNN_E_ARG, "max_bands must be >= 1");
    size_t best_ws = (size_t)-1;
    for (int n = 1; n <= max_bands; ++n) {
        const int grid = n == 1 ? 1 : 64;
        for (int g = grid; g >= 1; --g) {
            lrcnn_plan_opts o = *opts;
            o.band_rows = 0;
            o.n_bands = n;
            o.first_rows_pm = n == 1 ? 0 : (int)((1000LL * g + grid / 2) / grid);
            // below an equal first band the other bands would outgrow it: stop at the equal split
            if (n > 1 && o.first_rows_pm * n < 1000) o.first_rows_pm = 0;
            lrcnn_plan_t *p = nullptr;
            if (lrcnn_plan(net, &o, &p) != LRCNN_OK) continue;
            const size_t ws = p->P.ws_bytes;
            if (ws <= budget_bytes) {
                *out = p;
                if (n_bands) *n_bands = n;
                if (first_pm) *first_pm = o.first_rows_pm;
                return LRCNN_OK;
            }
            best_ws = std::min(best_ws, ws);
            lrcnn_plan_free(p);
            if (o.first_rows_pm == 0) break;
        }
    }
    return fail(LRCNN_E_INFEASIBLE, "no (N, H_1) with N <= " + std::to_string(max_bands) + " fits " +
                                        std::to_string(budget_bytes) + " bytes (smallest workspace " +
                                        std::to_string(best_ws) + ")");
}

// The paper's turning point: the band count whose workspace is the
// smallest -- beyond it the 2PS halo cache, which grows with N, outweighs the shrinking band
// working set.  Ties go to the smaller N (fewer, larger launches).
lrcnn_status lrcnn_plan_turning_point(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, int max_bands,
                                      int *n_star, size_t *ws_star) {
    if (!opts || !net || max_bands < 1) return fail(LRCNN_E_ARG, "bad arguments");
    if (opts->mode == LRCNN_COLUMN) return fail(LRCNN_E_ARG, "turning point needs a row-centric mode");
    int bn = 0;
    size_t bws = (size_t)-1;
    for (int n = 1; n <= max_bands; ++n) {
        lrcnn_plan_opts o = *opts;
        o.band_rows = 0;
        o.n_bands = n;
        lrcnn_plan_t *p = nullptr;
        if (lrcnn_plan(net, &o, &p) != LRCNN_OK) continue;
        if (p->P.ws_bytes < bws) { bws = p->P.ws_bytes; bn = n; }
        lrcnn_plan_free(p);
    }
    if (!bn) return fail(LRCNN_E_INFEASIBLE, "no feasible band count");
    if (n_star) *n_star = bn;
    if (ws_star) *ws_star = bws;
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_free(lrcnn_plan_t *plan) {
    if (plan) {
        for (int g = 0; g < 2; ++g)
            if (plan->P.graph_exec[g]) cudaGraphExecDestroy((cudaGraphExec_t)plan->P.graph_exec[g]);
        if (plan->P.comm_stream) cudaStreamDestroy((cudaStream_t)plan->P.comm_stream);
        if (plan->P.ev_comm) cudaEventDestroy((cudaEvent_t)plan->P.ev_comm);
        if (plan->P.ev_comm_done) cudaEventDestroy((cudaEvent_t)plan->P.ev_comm_done);
        if (plan->P.side_stream) {
            cudaStreamSynchronize((cudaStream_t)plan->P.side_stream);
            cudaStreamDestroy((cudaStream_t)plan->P.side_stream);
            cudaEventDestroy((cudaEvent_t)plan->P.ev_fork);
            cudaEventDestroy((cudaEvent_t)plan->P.ev_join);
            if (plan->P.ev_wt) cudaEventDestroy((cudaEvent_t)plan->P.ev_wt);
        }
        for (int c = 0; c < 3; ++c)
            for (auto &e : plan->P.pending_events[c]) {
                cudaEventDestroy((cudaEvent_t)e.first);
                cudaEventDestroy((cudaEvent_t)e.second);
            }
        delete plan;
    }
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_sizes(const lrcnn_plan_t *plan, size_t *ws, size_t *n_params, size_t *zl_elems) {
    if (!plan) return fail(LRCNN_E_ARG, "plan is NULL");
    const Plan &P = plan->P;
    const TensorInfo &z = P.t[P.net.n_ops];
    if (ws) *ws = P.ws_bytes;
    if (n_params) *n_params = P.n_params;
    if (zl_elems) *zl_elems = (size_t)P.net.B * z.H * z.W * z.Cp;
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_tensor(const lrcnn_plan_t *plan, int tid, int *C, int *Cp, int *H, int *W) {
    if (!plan || tid < 0 || tid > plan->P.net.n_ops) return fail(LRCNN_E_ARG, "bad plan or tensor id");
    const TensorInfo &t = plan->P.t[tid];
    if (C) *C = t.C;
    if (Cp) *Cp = t.Cp;
    if (H) *H = t.H;
    if (W) *W = t.W;
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_param(const lrcnn_plan_t *plan, int op, int which, size_t *offset, size_t *count) {
    if (!plan || !offset || !count || op < 0 || op > plan->P.net.n_ops) return fail(LRCNN_E_ARG, "bad args");
    const Plan &P = plan->P;
    *offset = 0; *count = 0;
    if (op == P.net.n_ops) {
        if (which == 0) { *offset = P.head_w_off; *count = P.head_w_cnt; }
        else if (which == 1) { *offset = P.head_b_off; *count = P.head_b_cnt; }
        else return fail(LRCNN_E_ARG, "bad which");
        return LRCNN_OK;
    }
    const OpInfo &o = P.op[op];
    if (which == 0) { *offset = o.w_off; *count = o.w_cnt; }
    else if (which == 1) { *offset = o.b_off; *count = o.b_cnt; }
    else if (which == 2) { *offset = o.beta_off; *count = o.beta_cnt; }
    else return fail(LRCNN_E_ARG, "bad which");
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_nsegs(const lrcnn_plan_t *plan, int *n) {
    if (!plan || !n) return fail(LRCNN_E_ARG, "bad args");
    *n = (int)plan->P.seg.size();
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_seg(const lrcnn_plan_t *plan, int seg, int *in_tid, int *out_tid, int *n_bands) {
    if (!plan || seg < 0 || seg >= (int)plan->P.seg.size()) return fail(LRCNN_E_ARG, "bad segment");
    const Segment &S = plan->P.seg[seg];
    if (in_tid) *in_tid = S.in_t;
    if (out_tid) *out_tid = S.out_t;
    if (n_bands) *n_bands = (int)S.E.size();
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_rows(const lrcnn_plan_t *plan, int seg, int band, int tid, int *lo, int *a, int *b) {
    if (!plan || seg < 0 || seg >= (int)plan->P.seg.size()) return fail(LRCNN_E_ARG, "bad segment");
    const Segment &S = plan->P.seg[seg];
    if (band < 0 || band >= (int)S.E.size()) return fail(LRCNN_E_ARG, "bad band");
    bool in = tid == S.in_t;
    for (int t : S.tensors) in = in || t == tid;
    if (!in) return fail(LRCNN_E_ARG, "tensor not in segment");
    if (lo) *lo = S.lo[band][tid];
    if (a) *a = S.a[band][tid];
    if (b) *b = S.b[band][tid];
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_read_end(const lrcnn_plan_t *plan, int seg, int band, int tid, int *hb) {
    if (!plan || !hb || seg < 0 || seg >= (int)plan->P.seg.size()) return fail(LRCNN_E_ARG, "bad segment");
    const Segment &S = plan->P.seg[seg];
    if (band < 0 || band >= (int)S.E.size()) return fail(LRCNN_E_ARG, "bad band");
    bool in = false;
    for (int t : S.tensors) in = in || t == tid;
    if (!in) return fail(LRCNN_E_ARG, "tensor not in segment");
    *hb = S.hb[band][tid];
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_zr_halo(const lrcnn_plan_t *plan, int seg, int max, int *n, int *tid, int *dir, int *r0,
                                int *r1) {
    if (!plan || !n || seg < 0 || seg >= (int)plan->P.seg.size()) return fail(LRCNN_E_ARG, "bad args");
    const Segment &S = plan->P.seg[seg];
    std::vector<std::array<int, 4>> v;
    for (auto &z : S.zr_from_below) v.push_back({z.t, 0, z.r0, z.r1});
    for (auto &z : S.zr_to_above) v.push_back({z.t, 1, z.r0, z.r1});
    *n = (int)v.size();
    for (int i = 0; i < *n && i < max; ++i) {
        if (tid) tid[i] = v[i][0];
        if (dir) dir[i] = v[i][1];
        if (r0) r0[i] = v[i][2];
        if (r1) r1[i] = v[i][3];
    }
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_fp_bands(const lrcnn_plan_t *plan, int seg, int *n_fp, int *n_bp) {
    if (!plan || seg < 0 || seg >= (int)plan->P.seg.size()) return fail(LRCNN_E_ARG, "bad segment");
    const Segment &S = plan->P.seg[seg];
    if (n_bp) *n_bp = (int)S.E.size();
    if (n_fp) *n_fp = S.fp_r0.empty() ? (int)S.E.size() : (int)S.fp_r0.size();
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_shard(const lrcnn_plan_t *plan, int seg, int tid, int *own_lo, int *own_hi, int *lo,
                              int *hi) {
    if (!plan || seg < 0 || seg >= (int)plan->P.seg.size()) return fail(LRCNN_E_ARG, "bad segment");
    const Segment &S = plan->P.seg[seg];
    if (tid < 0 || tid > plan->P.net.n_ops) return fail(LRCNN_E_ARG, "bad tensor");
    if (own_lo) *own_lo = S.own_lo;
    if (own_hi) *own_hi = S.own_hi;
    if (lo) *lo = S.LO[tid];
    if (hi) *hi = S.HI[tid];
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_xfers(const lrcnn_plan_t *plan, int seg, int max, int *n, int *peer, int *send, int *r0,
                              int *r1) {
    if (!plan || !n || seg < 0 || seg >= (int)plan->P.seg.size()) return fail(LRCNN_E_ARG, "bad args");
    const Segment &S = plan->P.seg[seg];
    *n = (int)S.in_xfers.size();
    for (int i = 0; i < *n && i < max; ++i) {
        if (peer) peer[i] = S.in_xfers[i].peer;
        if (send) send[i] = S.in_xfers[i].send;
        if (r0) r0[i] = S.in_xfers[i].r0;
        if (r1) r1[i] = S.in_xfers[i].r1;
    }
    return LRCNN_OK;
}

lrcnn_status lrcnn_plan_memory(const lrcnn_plan_t *plan, lrcnn_memory_report *rep) {
    if (!plan || !rep) return fail(LRCNN_E_ARG, "bad args");
    *rep = plan->P.mem;
    return LRCNN_OK;
}

lrcnn_status lrcnn_forward_rows(lrcnn_plan_t *plan, const void *params, const void *x, void *zl, void *ws,
                                size_t ws_bytes, void *stream) {
    if (!plan || !params || !x || !zl) return fail(LRCNN_E_ARG, "NULL argument");
    Plan &P = plan->P;
    lrcnn_status st = check_ws(P, ws, ws_bytes);
    if (st != LRCNN_OK) return st;
    P.launches = 0; P.tc_launches = 0; P.simt_fallbacks = 0;
    Run R{P, (char *)ws, (const char *)params, x, zl, nullptr, (cudaStream_t)stream, P.opts.prec, (size_t)P.elem};
    tc_set_pdl(!P.profiling);
    simt_set_pdl(!P.profiling);
    P.fwd_done = false;
    if (P.opts.world > 1 && !P.comm) return fail(LRCNN_E_STATE, "world > 1 needs lrcnn_plan_set_comm");
    st = run_forward(R);
    if (st != LRCNN_OK) return st;
    P.fwd_done = true; P.fwd_params = params; P.fwd_x = x; P.fwd_ws = ws;
    return LRCNN_OK;
}

lrcnn_status lrcnn_backward_rows(lrcnn_plan_t *plan, const void *params, const void *x, const void *zl,
                                 const void *dzl, float *grads, void *ws, size_t ws_bytes, void *stream) {
    if (!plan || !params || !x || !zl || !dzl || !grads) return fail(LRCNN_E_ARG, "NULL argument");
    Plan &P = plan->P;
    lrcnn_status st = check_ws(P, ws, ws_bytes);
    if (st != LRCNN_OK) return st;
    if (!P.fwd_done || P.fwd_ws != ws || P.fwd_params != params || P.fwd_x != x)
        return fail(LRCNN_E_STATE, "backward_rows needs a matching forward_rows (same params, x, ws)");
    P.launches = 0; P.tc_launches = 0; P.simt_fallbacks = 0;
    Run R{P, (char *)ws, (const char *)params, x, (void *)zl, grads, (cudaStream_t)stream, P.opts.prec, (size_t)P.elem};
    tc_set_pdl(!P.profiling);
    simt_set_pdl(!P.profiling);
    const int L = P.net.n_ops;
    const TensorInfo &z = P.t[L];
    // delta^L, gated by the last op's ReLU (gate on write), into the last segment's delta buffer
    int slast = (int)P.seg.size() - 1;
    CK(gate_copy(P.opts.prec, dzl, zl, R.ws + P.dfull_off[slast & 1], (long long)P.net.B * z.ck_rows * z.W * z.Cp,
                 z.relu, R.st));
    ++P.launches;
    if (P.opts.world > 1 && !P.comm) return fail(LRCNN_E_STATE, "world > 1 needs lrcnn_plan_set_comm");
    st = run_backward(R);   // (sharded: the per-segment wgrad buckets are summed over the ranks inside)
    if (st == LRCNN_OK) st = dp_join(R);
    P.fwd_done = false;
    return st;
}

static lrcnn_status step_grads_eager(lrcnn_plan_t *plan, const void *params, float *grads, const void *x,
                                     const int32_t *labels, float *loss_dev, void *ws, size_t ws_bytes, void *stream) {
    Plan &P = plan->P;
    lrcnn_status st = check_ws(P, ws, ws_bytes);
    if (st != LRCNN_OK) return st;
    P.launches = 0; P.tc_launches = 0; P.simt_fallbacks = 0;
    char *w = (char *)ws;
    Run R{P, w, (const char *)params, x, w + P.zl_off, grads, (cudaStream_t)stream, P.opts.prec, (size_t)P.elem};
    tc_set_pdl(!P.profiling);
    simt_set_pdl(!P.profiling);
    if (P.opts.world > 1 && !P.comm) return fail(LRCNN_E_STATE, "world > 1 needs lrcnn_plan_set_comm");
    if ((st = run_forward(R)) != LRCNN_OK) return st;
    const int L = P.net.n_ops;
    const TensorInfo &z = P.t[L];
    int slast = (int)P.seg.size() - 1;
    // head on the pooled z^L: each rank pools its own rows, the partial sums are all-reduced
    const float hw = (float)z.H * z.W;
    float *scratch = (float *)(w + P.head_off);
    Nvtx nv("head");
    CK(head_gap(P.opts.prec, R.zl, P.net.B, z.ck_rows * z.W, z.Cp, hw, scratch, R.st,
                scratch + (size_t)P.net.B * z.Cp + (size_t)P.net.B * P.net.n_classes + P.net.B + 64));
    if (P.opts.world > 1) {
        const char *err = nullptr;
        if (comm_allreduce_f32((Comm *)P.comm, scratch, (size_t)P.net.B * z.Cp, R.st, &err))
            return fail(LRCNN_E_NCCL, err ? err : "allreduce failed");
    }
    CK(head_tail(P.opts.prec, R.zl, P.net.B, z.ck_rows * z.W, z.Cp, z.C, P.net.n_classes,
                 R.params + P.head_w_off * R.E, R.params + P.head_b_off * R.E, labels, scratch, loss_dev,
                 grads + P.head_w_off, grads + P.head_b_off, w + P.dfull_off[slast & 1], z.relu, hw, R.st));
    P.launches += 4;   // gap, logits, FC grad, delta^L
    if (P.dp_world > 1 && (st = dp_reduce(R, P.head_w_off, P.head_b_off + P.head_b_cnt)) != LRCNN_OK) return st;
    st = run_backward(R);   // (sharded: the per-segment wgrad buckets are summed over the ranks inside)
    if (st == LRCNN_OK) st = dp_join(R);
    P.fwd_done = false;
    return st;
}

lrcnn_status lrcnn_step_grads(lrcnn_plan_t *plan, const void *params, float *grads, const void *x,
                              const int32_t *labels, float *loss_dev, void *ws, size_t ws_bytes, void *stream) {
    if (!plan || !params || !grads || !x || !labels || !loss_dev) return fail(LRCNN_E_ARG, "NULL argument");
    const uintptr_t key[9] = {0, (uintptr_t)params, (uintptr_t)grads, (uintptr_t)x, (uintptr_t)labels,
                              (uintptr_t)loss_dev, (uintptr_t)ws, (uintptr_t)stream, 0};
    return graph_run(plan->P, 1, key, stream, [&]() {
        return step_grads_eager(plan, params, grads, x, labels, loss_dev, ws, ws_bytes, stream);
    });
}

lrcnn_status lrcnn_plan_set_comm(lrcnn_plan_t *plan, lrcnn_comm *comm) {
    if (!plan) return fail(LRCNN_E_ARG, "plan is NULL");
    const Plan &P = plan->P;
    const int world = P.dp_world > 1 ? P.dp_world : P.opts.world, rank = P.dp_world > 1 ? P.dp_rank : P.opts.rank;
    if (comm && (comm_world((Comm *)comm) != world || comm_rank((Comm *)comm) != rank))
        return fail(LRCNN_E_ARG, "communicator rank/world differ from the plan's");
    plan->P.comm = comm;
    return LRCNN_OK;
}

lrcnn_status lrcnn_sgd(lrcnn_plan_t *plan, float *master, void *params, float *grads, float lr, void *stream) {
    if (!plan || !master || !params || !grads) return fail(LRCNN_E_ARG, "NULL argument");
    Plan &P = plan->P;
    CK(sgd_update(P.opts.prec, master, params, grads, (long long)P.n_params, lr, (cudaStream_t)stream));
    ++P.launches;
    return LRCNN_OK;
}

static lrcnn_status step_eager(lrcnn_plan_t *plan, float *master, void *params, float *grads, const void *x,
                               const int32_t *labels, float lr, float *loss_dev, void *ws, size_t ws_bytes,
                               void *stream) {
    lrcnn_status st = step_grads_eager(plan, params, grads, x, labels, loss_dev, ws, ws_bytes, stream);
    if (st != LRCNN_OK) return st;
    return lrcnn_sgd(plan, master, params, grads, lr, stream);   // adds its own launch
}

// One training iteration.  The band x op sweep is hundreds of launches; from the second call
// with unchanged arguments on a non-default stream the whole step is captured once into a CUDA
// graph and replayed (tensor maps and launch parameters are baked in by value).
lrcnn_status lrcnn_step(lrcnn_plan_t *plan, float *master, void *params, float *grads, const void *x,
                        const int32_t *labels, float lr, float *loss_dev, void *ws, size_t ws_bytes, void *stream) {
    if (!plan || !master || !params || !grads || !x || !labels || !loss_dev) return fail(LRCNN_E_ARG, "NULL argument");
    float lr_copy = lr;
    uint32_t lr_bits;
    std::memcpy(&lr_bits, &lr_copy, 4);
    const uintptr_t key[9] = {(uintptr_t)master, (uintptr_t)params, (uintptr_t)grads, (uintptr_t)x,
                              (uintptr_t)labels, (uintptr_t)loss_dev, (uintptr_t)ws, (uintptr_t)stream, lr_bits};
    return graph_run(plan->P, 0, key, stream, [&]() {
        return step_eager(plan, master, params, grads, x, labels, lr, loss_dev, ws, ws_bytes, stream);
    });
}


lrcnn_status lrcnn_profile_enable(lrcnn_plan_t *plan, int enable) {
    if (!plan) return fail(LRCNN_E_ARG, "plan is NULL");
    plan->P.profiling = enable != 0;
    return LRCNN_OK;
}

lrcnn_status lrcnn_profile_reset(lrcnn_plan_t *plan) {
    if (!plan) return fail(LRCNN_E_ARG, "plan is NULL");
    for (int c = 0; c < 3; ++c) {
        for (auto &e : plan->P.pending_events[c]) {
            cudaEventDestroy((cudaEvent_t)e.first);
            cudaEventDestroy((cudaEvent_t)e.second);
        }
        plan->P.pending_events[c].clear();
        plan->P.pending_flops[c].clear();
        plan->P.pending_bytes[c].clear();
        plan->P.pending_wbytes[c].clear();
        plan->P.pending_tags[c].clear();
        plan->P.pending_names[c].clear();
        plan->P.per_kernel[c].clear();
        plan->P.prof[c] = ProfileSlot();
    }
    plan->P.per_tag.clear();
    return LRCNN_OK;
}

lrcnn_status lrcnn_profile_read(lrcnn_plan_t *plan, int cls, double *ms, long long *launches, double *flops,
                                void *stream) {
    if (!plan || cls < 0 || cls > 2) return fail(LRCNN_E_ARG, "bad args");
    Plan &P = plan->P;
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    for (int c = 0; c < 3; ++c) {
        for (size_t i = 0; i < P.pending_events[c].size(); ++i) {
            float t = 0;
            auto &e = P.pending_events[c][i];
            CK(cudaEventElapsedTime(&t, (cudaEvent_t)e.first, (cudaEvent_t)e.second));
            P.prof[c].ms += t;
            P.prof[c].flops += P.pending_flops[c][i];
            P.prof[c].launches += 1;
            {   // per tcgen05 kernel
                const std::string &nm = P.pending_names[c][i];
                auto it = std::find_if(P.per_kernel[c].begin(), P.per_kernel[c].end(),
                                       [&nm](const std::pair<std::string, ProfileSlot> &q) { return q.first == nm; });
                if (it == P.per_kernel[c].end()) { P.per_kernel[c].push_back({nm, ProfileSlot()}); it = P.per_kernel[c].end() - 1; }
                it->second.ms += t;
                it->second.flops += P.pending_flops[c][i];
                it->second.bytes += P.pending_bytes[c][i];
                it->second.wbytes += P.pending_wbytes[c][i];
                it->second.launches += 1;
            }
            const int tag = P.pending_tags[c][i];
            if (tag >= 0) {
                auto it = std::find_if(P.per_tag.begin(), P.per_tag.end(),
                                       [tag](const std::pair<int, ProfileSlot> &q) { return q.first == tag; });
                if (it == P.per_tag.end()) { P.per_tag.push_back({tag, ProfileSlot()}); it = P.per_tag.end() - 1; }
                it->second.ms += t;
                it->second.flops += P.pending_flops[c][i];
                it->second.launches += 1;
            }
            cudaEventDestroy((cudaEvent_t)e.first);
            cudaEventDestroy((cudaEvent_t)e.second);
        }
        P.pending_events[c].clear();
        P.pending_flops[c].clear();
        P.pending_bytes[c].clear();
        P.pending_wbytes[c].clear();
        P.pending_tags[c].clear();
        P.pending_names[c].clear();
    }
    if (ms) *ms = P.prof[cls].ms;
    if (launches) *launches = P.prof[cls].launches;
    if (flops) *flops = P.prof[cls].flops;
    return LRCNN_OK;
}

lrcnn_status lrcnn_profile_kernels(lrcnn_plan_t *plan, int cls, char *buf, size_t len, void *stream) {
    if (!plan || cls < 0 || cls > 2 || !buf || !len) return fail(LRCNN_E_ARG, "bad args");
    lrcnn_status st = lrcnn_profile_read(plan, cls, nullptr, nullptr, nullptr, stream);
    if (st != LRCNN_OK) return st;
    std::string out;
    char line[512];
    for (auto &e : plan->P.per_kernel[cls]) {
        snprintf(line, sizeof line, "%s,%lld,%.6f,%.6e,%.6e,%.6e\n", e.first.empty() ? "simt" : e.first.c_str(),
                 e.second.launches, e.second.ms, e.second.flops, e.second.bytes, e.second.wbytes);
        out += line;
    }
    if (out.size() + 1 > len) return fail(LRCNN_E_ARG, "buffer too small");
    memcpy(buf, out.c_str(), out.size() + 1);
    return LRCNN_OK;
}

lrcnn_status lrcnn_profile_dump(lrcnn_plan_t *plan, const char *path, void *stream) {
    if (!plan || !path) return fail(LRCNN_E_ARG, "bad args");
    lrcnn_status st = lrcnn_profile_read(plan, 0, nullptr, nullptr, nullptr, stream);
    if (st != LRCNN_OK) return st;
    FILE *f = fopen(path, "w");
    if (!f) return fail(LRCNN_E_ARG, std::string("cannot open ") + path);
    static const char *kinds[8] = {"fwd", "dgrad", "wgrad", "param_grad", "pool_fwd", "pool_bwd", "elt_fwd", "elt_bwd"};
    fprintf(f, "op,kind,k,s,c_in,c_out,h_out,w_out,launches,ms,flops\n");
    auto v = plan->P.per_tag;
    std::sort(v.begin(), v.end(), [](const std::pair<int, ProfileSlot> &a, const std::pair<int, ProfileSlot> &b) {
        return a.first < b.first;
    });
    for (auto &e : v) {
        const int op = e.first / 8, kind = e.first % 8;
        const OpInfo &o = plan->P.op[op];
        const TensorInfo &ti = plan->P.t[o.in_t], &to = plan->P.t[o.out_t];
        fprintf(f, "%d,%s,%d,%d,%d,%d,%d,%d,%lld,%.6f,%.6e\n", op, kinds[kind], o.d.k, o.d.s, ti.C, to.C, to.H, to.W,
                e.second.launches, e.second.ms, e.second.flops);
    }
    fclose(f);
    return LRCNN_OK;
}

lrcnn_status lrcnn_last_tc_launch_count(const lrcnn_plan_t *plan, long long *launches) {
    if (!plan || !launches) return fail(LRCNN_E_ARG, "bad args");
    *launches = plan->P.tc_launches;
    return LRCNN_OK;
}

lrcnn_status lrcnn_debug_capture(lrcnn_plan_t *plan, int tid, void *dst) {
    if (!plan || tid < 1 || tid > plan->P.net.n_ops) return fail(LRCNN_E_ARG, "bad plan or tensor id");
    Plan &P = plan->P;
    if (P.capture.size() < P.t.size()) P.capture.resize(P.t.size(), nullptr);
    P.capture[tid] = dst;
    bool any = false;
    for (void *c : P.capture) any = any || c;
    if (!any) P.capture.clear();
    return LRCNN_OK;
}

lrcnn_status lrcnn_last_simt_fallbacks(const lrcnn_plan_t *plan, long long *n) {
    if (!plan || !n) return fail(LRCNN_E_ARG, "bad args");
    *n = plan->P.simt_fallbacks;
    return LRCNN_OK;
}

lrcnn_status lrcnn_last_launch_count(const lrcnn_plan_t *plan, long long *launches) {
    if (!plan || !launches) return fail(LRCNN_E_ARG, "bad args");
    *launches = plan->P.launches;
    return LRCNN_OK;
}

}  // extern "C"

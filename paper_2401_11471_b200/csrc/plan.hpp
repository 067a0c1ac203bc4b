// plan.hpp -- host-side plan of the row-centric hot path (internal, not part of the ABI).
//
// A plan fixes, per segment and band, the rows every tensor computes and holds
// (the interval rule, R3 / R4), the halo-cache and carry sizes, and
// the byte layout of the caller-provided workspace.  Pure integer host code.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/lrcnn.h"

namespace lrcnn {

struct Consumer {
    int op;    // consuming op index
    int role;  // 0 = read through the op's window (src of CONV/MAXPOOL), 1 = read 1:1 (res, ADD)
};

struct TensorInfo {
    int C = 0, Cp = 0, H = 0, W = 0;
    int producer = -1;        // op index, -1 for the image
    int relu = 0;             // producer applies ReLU (delta gate on write)
    int seg = -1;             // segment that produces it (-1 image)
    bool seg_in = false;      // image or checkpoint: full-width map
    bool seg_out = false;     // output of its segment (checkpoint or z^L)
    bool is_zl = false;
    std::vector<Consumer> cons;
    // workspace placement (bytes)
    int cap = 0;              // band buffer rows (internal tensors)
    size_t act_off = 0, dlt_off = 0;
    int carry_cap = 0;
    size_t carry_off = 0;
    std::vector<int> cache_lo, cache_rows;   // per band boundary r (0..N-2): rows [lo_{r+1}, b_r)
    std::vector<size_t> cache_off;
    size_t ckpt_off = 0;      // checkpoint (seg_out && !is_zl)
    int ck_lo = 0, ck_rows = 0;   // rows a full-width map (image, checkpoint, z^L) holds on this rank
    int dl_lo = 0, dl_rows = 0;   // rows of the boundary delta buffer (segment in/out) on this rank
    size_t wt_off = 0;        // unused for tensors
    // decoupled FP bands (LRCNN_FLAG_FP_MERGE): FP band buffer (aliases the band arena)
    size_t act_fp_off = 0;
    int cap_fp = 0;
    // BP delta slot (delta_slots): live from the backward of op dfw (first writer) down to op dlr
    // (last reader); dreuse = the slot held an earlier tensor's delta in the same band
    int dfw = -1, dlr = -1;
    bool dreuse = false;
    // zero-redundancy sharding: rows [zr_in_r0, zr_in_r1) come from rank+1 (activations in, their delta
    // out); rows [zr_out_r0, zr_out_r1) of mine go to rank-1 (activations out, their delta in)
    size_t zr_in_off = 0, zr_dout_off = 0, zr_out_off = 0, zr_din_off = 0;
    int zr_in_r0 = 0, zr_in_r1 = 0, zr_out_r0 = 0, zr_out_r1 = 0;
};

struct OpInfo {
    lrcnn_op d;
    int in_t, out_t;
    size_t w_off = 0, w_cnt = 0, b_off = 0, b_cnt = 0, beta_off = 0, beta_cnt = 0;
    size_t wt_off = 0;        // transposed (dgrad) weights in workspace (bf16 tensor-core path)
    // training-mode BN (LRCNN_OP_BN): workspace scratch -- sums [2][Cp] fp64 (sum c, sum c^2), S [2][Cp] fp64
    // (sum da, sum da*xh), coef [6][Cp] fp32 (a, b, p, q, mean, invstd); see bn.cu
    size_t bn_sums_off = 0, bn_S_off = 0, bn_coef_off = 0;
};

// One halo transfer of a boundary tensor between this rank and a neighbour (rows [r0, r1)).
struct Xfer {
    int peer;      // rank
    int send;      // 1 = send (FP: my rows to the neighbour; BP: the neighbour's delta rows I hold)
    int r0, r1;
};

struct Segment {
    int in_t = 0, out_t = 0;
    std::vector<int> ops;                    // topological order
    std::vector<int> tensors;                // internal tensors + out (ids), production order
    // row sharding across ranks (world > 1): this rank owns output rows [own_lo, own_hi) and
    // computes every tensor t over its extended range [LO[t], HI[t]) (OverL at rank cuts);
    // in_own_lo/hi = rows of the segment input this rank owns (previous segment's split)
    int own_lo = 0, own_hi = 0, in_own_lo = 0, in_own_hi = 0;
    std::vector<int> LO, HI;
    std::vector<Xfer> in_xfers;              // FP halo of the segment input (BP: reversed, added)
    std::vector<int> E;                      // band ends at the segment output
    // per band r, per global tensor id: lo (buffer start), a (first computed), b (end)
    std::vector<std::vector<int>> lo, a, b;
    int overlap_in = 0;                      // OverL: max overlap of consecutive bands at the input
    // decoupled FP bands (LRCNN_FLAG_FP_MERGE): FP band k = BP bands [fp_r0[k], fp_r0[k+1]); the
    // merged per-band ranges live in fp_lo / fp_a / fp_b (empty: FP uses the BP bands)
    std::vector<int> fp_r0;
    std::vector<std::vector<int>> fp_lo, fp_a, fp_b;
    // buffer end per band and tensor: one past the last row the band's consumers read (== b unless a
    // zero-redundancy rank's last band reads rows of rank+1)
    std::vector<std::vector<int>> hb;
    // zero-redundancy halo schedule of the internal tensors (tensor, rows)
    struct ZrRows { int t, r0, r1; };
    std::vector<ZrRows> zr_from_below, zr_to_above;
    // training-mode BN: the segment's BN ops grouped by dependency
    // level -- FP level k = BN ops whose input depends on BN ops of levels < k only (one statistics
    // sweep per level computes the ops in bn_fp_ops[k]); BP level k (reverse) = BN ops whose output
    // feeds BN ops of levels < k only (one sums sweep per level runs the backward of the ops in
    // bn_bp_ops[k] and writes the delta of the tensors in bn_bp_need[k] only).  Per op / tensor id.
    std::vector<std::vector<int>> bn_fp_levels, bn_bp_levels;
    std::vector<std::vector<char>> bn_fp_ops, bn_bp_ops, bn_bp_need;
    // BN tail: the segment output is produced by BN op bn_tail (alone in the last FP
    // level, residual = none or the segment input, its input a band tensor only it reads): the last
    // statistics sweep writes that input straight into the output checkpoint, the BN is then applied
    // in place over the full map, and the FP sweep of the segment is skipped.  -1: none.
    int bn_tail = -1;
    // BN input stash: in the FP of this segment, the input c of a BN op is written once,
    // full-width, at workspace offset stash_off[c] (overlaying the full-width delta buffers, which only
    // the BP uses), and later statistics sweeps and the FP sweep read it instead of recomputing its
    // producers; bn_fp_ops are cut at the stashed tensors, bn_fp_final = the FP sweep's ops.  Per tensor
    // id, (size_t)-1 = not stashed.
    std::vector<size_t> stash_off;
    std::vector<char> bn_fp_final;
    // BP stash: the segment's first backward sweep writes these BN inputs full-width into a region of
    // their own (bp_stash_off, absolute workspace offsets), the later sweeps recompute only the ops in
    // bn_bp_recompute (not their producers).  Empty: none.
    std::vector<size_t> bp_stash_off;
    std::vector<char> bn_bp_recompute;
};

struct ProfileSlot {
    double ms = 0, flops = 0, bytes = 0;   // bytes: algorithmic HBM bytes
    double wbytes = 0;                     // of which written
    long long launches = 0;
};

struct Plan {
    lrcnn_net_desc net{};
    std::vector<lrcnn_op> ops_copy;
    lrcnn_plan_opts opts{};
    int elem = 4;                            // bytes per activation element
    std::vector<TensorInfo> t;
    std::vector<OpInfo> op;
    std::vector<Segment> seg;
    size_t n_params = 0;
    size_t head_w_off = 0, head_w_cnt = 0, head_b_off = 0, head_b_cnt = 0;
    size_t ws_bytes = 0;
    size_t dfull_off[2] = {0, 0}, dfull_bytes = 0;
    size_t xstage_off[2] = {0, 0}, xstage_bytes = 0;   // halo exchange staging (send, recv)
    void *comm = nullptr;                    // lrcnn_comm* (world > 1)
    size_t head_off = 0;                     // head scratch (fp32)
    size_t zl_off = 0;                       // z^L buffer used by lrcnn_step
    size_t flag_off = 0;                     // small device scratch
    bool use_tc = false;                     // tensor-core kernels enabled
    lrcnn_memory_report mem{};
    // run state
    bool fwd_done = false;
    const void *fwd_params = nullptr, *fwd_x = nullptr;
    void *fwd_ws = nullptr;
    long long launches = 0, tc_launches = 0;
    long long simt_fallbacks = 0;            // convs a bf16 tensor-core plan ran on SIMT (declined shapes)
    bool profiling = false;
    std::vector<void *> capture;             // lrcnn_debug_capture buffers per tensor id (debug)
    ProfileSlot prof[3];
    void *ev_wt = nullptr;                   // transposed dgrad weights written (side stream, during FP)
    bool wt_pending = false;                 // FP launched the transposes; BP waits on ev_wt
    std::vector<std::pair<void *, void *>> pending_events[3];   // (start, stop) cudaEvent_t
    std::vector<double> pending_flops[3];
    std::vector<double> pending_bytes[3];
    std::vector<double> pending_wbytes[3];
    std::vector<int> pending_tags[3];             // op*8 + kind (profile dump)
    std::vector<std::string> pending_names[3];    // tcgen05 kernel launched inside the scope ("" = SIMT)
    std::vector<std::pair<std::string, ProfileSlot>> per_kernel[3];
    std::vector<std::pair<int, ProfileSlot>> per_tag;
    // CUDA graphs of one lrcnn_step (slot 0) / lrcnn_step_grads (slot 1), replayed while the call's
    // arguments are unchanged
    void *graph_exec[2] = {nullptr, nullptr};    // cudaGraphExec_t
    uintptr_t graph_key[2][9] = {};
    int graph_calls[2] = {0, 0};                 // consecutive calls with the same key
    long long graph_launches[2] = {0, 0}, graph_tc_launches[2] = {0, 0}, graph_simt_fallbacks[2] = {0, 0};
    // side stream for wgrad / parameter reductions (overlap with the dgrad chain) and its events
    void *side_stream = nullptr, *ev_fork = nullptr, *ev_join = nullptr;
    // data-parallel replicas (LRCNN_FLAG_DP): replica count / index, per-segment gradient buckets
    // [seg_grad_lo, seg_grad_hi) (flat parameter offsets), the communication stream and its events
    int dp_world = 1, dp_rank = 0;
    std::vector<size_t> seg_grad_lo, seg_grad_hi;
    void *comm_stream = nullptr, *ev_comm = nullptr, *ev_comm_done = nullptr;
};

// Builds the plan; returns status and fills err on failure.
lrcnn_status build_plan(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, Plan &P, std::string &err);

// A band-internal tensor without ReLU whose only reader is the residual input of a convolution u
// (ResNet's projection shortcut) has delta(t) == delta(out_u) on the same rows: the residual add
// passes the gradient through and there is no gate.  Its delta is that buffer (no memset, no copy
// pass).  Returns u's output tensor, or -1.
inline int alias_delta(const Plan &P, const Segment &S, int t) {
    if (t == 0 || t == S.in_t || t == S.out_t) return -1;
    const TensorInfo &ti = P.t[t];
    if (ti.relu || ti.cons.size() != 1 || ti.cons[0].role != 1) return -1;
    const OpInfo &u = P.op[ti.cons[0].op];
    if (u.d.kind != LRCNN_OP_CONV || u.d.res != t) return -1;
    const TensorInfo &to = P.t[u.out_t];
    if (to.Cp != ti.Cp || to.W != ti.W || to.H != ti.H) return -1;
    return u.out_t;
}

inline int round_up(int v, int m) { return (v + m - 1) / m * m; }
inline int out_dim(int h, int k, int s, int p) {
    int span = h + 2 * p - k;
    return span < 0 ? -1 : span / s + 1;
}

}  // namespace lrcnn

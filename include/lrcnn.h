/*
 * lrcnn.h -- C-ABI of the B200-native LR-CNN hot path (arXiv 2401.11471).
 *
 * Row-centric training of a stack (DAG) of convolution layers: the forward
 * pass (FP) sweeps horizontal bands of rows through every layer of a segment
 * (Alg. 1 l.5-10, Eq. (4)); the backward
 * pass (BP) walks the bands in reverse, recomputes each band (Alg. 1 l.17)
 * and produces dgrad and wgrad with wgrad accumulated across bands
 * (Eq. (5), Alg. 1 l.18-20).  Both of the paper's answers to
 * the inter-row weak dependency are provided: two-phase sharing (2PS, cache the
 * halo rows) and overlapping partitioning (OverL, recompute
 * the overlap); "seg_end" checkpoints give the -H hybrids
 * (PAPER.md:322, 394).
 *
 * Conventions for every entry point
 *   - Plain C types and pointers only; no exceptions cross the ABI.
 *   - Every function returns an lrcnn_status; LRCNN_OK == 0.  On error a
 *     message is available from lrcnn_last_error() (thread-local, valid until
 *     the next call on the same thread).
 *   - Shape/feasibility errors are reported synchronously by lrcnn_plan.
 *   - Device work is enqueued asynchronously on the caller's stream (a
 *     cudaStream_t passed as void*; NULL = legacy default stream).  Launch
 *     errors are reported as LRCNN_E_CUDA by the call that enqueued them;
 *     asynchronous faults surface at the caller's next synchronisation.
 *   - The caller owns every device buffer (allocated e.g. by PyTorch).  The
 *     library owns only the host-side plan.  Nothing is allocated on the device
 *     inside forward/backward/step, so the peak HBM is the caller's
 *     allocations (visible to torch.cuda.max_memory_allocated).
 *
 * Device data layouts (all row-major, C-contiguous)
 *   - Activations: NHWC, channels padded to Cp = round_up(C, 8) (16-byte
 *     rows for the tensor-core path).  Padded channels must be zero.
 *   - Element type: float (LRCNN_FP32) or bfloat16 (LRCNN_BF16) -- "act_t".
 *   - Parameters: one flat array laid out by the plan (lrcnn_plan_param):
 *     per conv op w[C_out][k][k][Cp_in] (OHWI), then bias[C_out] (EPI_BIAS) or
 *     gamma[C_out], beta[C_out] (EPI_AFFINE); per BN op gamma[C], beta[C]; then the head fc_w[classes][C_L],
 *     fc_b[classes].  Device copies in act_t ("params"), an fp32 master copy
 *     ("master") and fp32 gradients ("grads") share these offsets.
 */
#ifndef LRCNN_H
#define LRCNN_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LRCNN_API __attribute__((visibility("default")))
#else
#define LRCNN_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LRCNN_OK = 0,
    LRCNN_E_ARG = 1,          /* NULL pointer, out-of-range index or enum           */
    LRCNN_E_SHAPE = 2,        /* invalid shape, kernel exceeds input  */
    LRCNN_E_INFEASIBLE = 3,   /* OverL N > H/o^0                  */
    LRCNN_E_DEGENERATE = 4,   /* band ends not strictly increasing at a segment out  */
    LRCNN_E_STATE = 5,        /* backward without forward, plan/buffer mismatch      */
    LRCNN_E_WORKSPACE = 6,    /* workspace NULL or too small                         */
    LRCNN_E_CUDA = 7,         /* a CUDA runtime/driver call failed                   */
    LRCNN_E_NCCL = 8,         /* a communicator call (halo exchange, all-reduce) failed */
    LRCNN_E_UNSUPPORTED = 9   /* valid request this build does not implement        */
} lrcnn_status;

typedef enum { LRCNN_COLUMN = 0, LRCNN_2PS = 1, LRCNN_OVERL = 2 } lrcnn_mode;
typedef enum { LRCNN_FP32 = 0, LRCNN_BF16 = 1 } lrcnn_precision;
enum { LRCNN_OP_CONV = 0, LRCNN_OP_MAXPOOL = 1, LRCNN_OP_ADD = 2, LRCNN_OP_BN = 3 };
enum { LRCNN_EPI_NONE = 0, LRCNN_EPI_BIAS = 1, LRCNN_EPI_AFFINE = 2 };

/* One op of the DAG.  Tensor ids: 0 = the image, op i produces tensor i+1.
 *   CONV:    t = relu?( epi(Conv_{k,s,p}(t_src)) + t_res )      (Eq. (1))
 *            epi: BIAS  -> + b[co];  AFFINE -> gamma[co]*c + beta[co] (frozen-statistics BN)
 *   MAXPOOL: t = max over k x k windows, stride s, pad p (pads never win, ties -> lowest index)
 *   ADD:     t = relu?( t_src + t_res )
 *   BN:      t = relu?( gamma[c]*(t_src - mean[c])/sqrt(var[c] + 1e-5) + beta[c] + t_res )   (t_res optional)
 *            training-mode BatchNorm (BN in the FP: PAPER.md:112; R24): mean and
 *            biased var of t_src over the whole batch and map, recomputed every step; the backward is the
 *            batch-statistics adjoint.  Parameters gamma[C], beta[C] (plan layout).  The statistics are
 *            a dependency on EVERY row of t_src: lrcnn_forward_rows runs one statistics sweep per
 *            dependency level of a segment's BN ops before its FP sweep, lrcnn_backward_rows one sums
 *            sweep per level (reverse) before its BP sweep.  One GPU, data-parallel replicas (per-replica statistics), or rows sharded with
 *            LRCNN_FLAG_ZERO_REDUNDANCY (statistics over the whole map: fp64 sums all-reduced over the
 *            ranks -- NCCL, loopback, or host-staged as an all-gather through the exchange callback).  Modes COLUMN, 2PS and OverL (overlapping bands:
 *            each row counted once, the backward's statistics terms added once per row).  OverL rank
 *            cuts (rows computed by two ranks) and a BN of a segment input under sharding return
 *            LRCNN_E_UNSUPPORTED.
 * seg_end != 0 stores the op's output as a full-width checkpoint (segment boundary). */
typedef struct {
    int kind;
    int src;
    int res;          /* residual/second input tensor id, -1 = none */
    int c_out;        /* CONV only */
    int k, s, p;      /* CONV / MAXPOOL */
    int epi;          /* CONV only */
    int relu;
    int seg_end;
} lrcnn_op;

typedef struct {
    int n_ops;
    const lrcnn_op *ops;
    int B, C, H, W;   /* batch and image shape (C = real channels, padded to Cp on device) */
    int n_classes;    /* head: GAP -> FC(C_L -> n_classes) -> softmax-CE (mean over B) */
} lrcnn_net_desc;

typedef struct {
    int mode;         /* lrcnn_mode.  COLUMN = layer-wise baseline: one segment, one band,
                         every feature map kept, no recompute */
    int prec;         /* lrcnn_precision */
    int band_rows;    /* >0: owned rows of each segment output per band, remainder to the
                         last band (reading R15) */
    int n_bands;      /* used when band_rows <= 0: near-equal split, earliest bands +1 row */
    int rank, world;  /* row sharding across ranks (world > 1), or data-parallel
                         replicas with LRCNN_FLAG_DP; world == 1: a single GPU */
    int flags;        /* LRCNN_FLAG_* */
    int first_rows_pm;/* > 0 (with n_bands > 1): band 1 owns round(H * first_rows_pm / 1000) rows of each
                         segment output, the other n_bands - 1 bands split the rest near-equally -- the
                         greedy first band of Eq. (12), PAPER.md:297-310 (lrcnn_plan_greedy); 0 = off */
} lrcnn_plan_opts;

#define LRCNN_FLAG_ALLOW_OVERLAP_EXHAUSTION 1  /* OverL: do not reject N > H/o^0 */
#define LRCNN_FLAG_NO_TCGEN05 2                /* bf16: use the SIMT kernels only (tests)     */
/* Balanced bands (budget-driven N per segment; "max H^L then
 * min N"): n_bands / band_rows fixes the band working set of the segment that needs the most;
 * every other segment uses the smallest band count whose working set (activation + delta +
 * carry buffers, overlaid across segments) fits in that same budget.  Peak memory is unchanged,
 * thin deep segments get fewer, larger bands (fewer halo rows, larger kernel launches). */
#define LRCNN_FLAG_BALANCED_BANDS 4
/* Disable the fused residual gradient (bf16 tensor-core path): a block input read by a stride-1
 * convolution and a residual add gets delta = gate * (dgrad + delta(block output)) from that
 * convolution's dgrad epilogue (the block output's delta as a TMA-loaded addend) instead of a
 * memset, an accumulating dgrad and a separate residual pass.  Set only to compare (tests). */
#define LRCNN_FLAG_NO_FUSE_RES 8
/* Decoupled FP bands (2PS, the FP working set Omega_FP < Omega_BP, so
 * N_FP <= N_BP): the forward pass runs each segment with the fewest bands -- merges of
 * consecutive BP bands -- whose activation buffers fit in the band arena the BP needs anyway
 * (the FP has no delta buffers), and saves the halo rows of every BP band boundary inside a
 * merged band.  Peak memory is unchanged; results are identical (same kernels, same per-pixel
 * accumulation order).  lrcnn_plan_fp_bands reports N_FP per segment. */
#define LRCNN_FLAG_FP_MERGE 16
/* Data-parallel replicas (SURVEY 8(e) "across images"): opts.rank / opts.world name this replica,
 * every replica plans the whole image (no row split) on its own batch, and lrcnn_step /
 * lrcnn_step_grads sum the weight gradient over the replicas (the communicator set with
 * lrcnn_plan_set_comm) in per-segment buckets on a communication stream, each as soon as that
 * segment's backward is complete, overlapping the rest of the backward; the head gradient after
 * the head.  The gradient is the SUM over replicas (pass lr / world for the mean). */
#define LRCNN_FLAG_DP 32
/* bf16 plans: a convolution whose shape no tensor-core kernel takes fails with LRCNN_E_UNSUPPORTED
 * instead of running the SIMT kernel (bench.py sets it, so a timed step is tcgen05-only).  Without
 * the flag such convolutions run on SIMT and are counted (lrcnn_last_simt_fallbacks).  A tensor-core
 * launch that FAILS (launch or attribute error) is always LRCNN_E_CUDA, never a SIMT rerun. */
#define LRCNN_FLAG_REQUIRE_TC 64
/* sqrt(n) checkpointing ("determine the optimal checkpoint locations ... Ref. [34]",
 * PAPER.md:584 "a preferred checkpointing frequency is sqrt(n)"): the net's seg_end flags are
 * replaced by ceil(sqrt(n_ops)) - 1 checkpoints, each at the valid cut (an op output that no other
 * tensor is read past) nearest to an even spacing of the ops.  lrcnn_plan_seg reports them. */
#define LRCNN_FLAG_AUTO_SEGMENTS 128
/* Zero-redundancy row sharding (world > 1, 2PS; the weak dependency across a rank
 * cut, resolved by two-phase sharing instead of overlap): every row of every tensor is
 * computed by exactly one rank -- rank g owns [F_{C_g}(t), F_{C_{g+1}}(t)), F_C(t) = the lowest row of
 * t the outputs below the cut C need -- so a rank depends only on the FIRST rows of rank g+1: after
 * every rank's first band the ranks exchange those rows of every band tensor (one grouped send/recv
 * per segment), the last band of rank g reads them, and in the backward its delta for those rows
 * goes back the same way and is added into rank g+1's first band.  No recomputation at the cuts.
 * Needs >= 2 bands per rank (but the last); ignores BALANCED_BANDS / FP_MERGE. */
#define LRCNN_FLAG_ZERO_REDUNDANCY 256
/* Disable the fused bottleneck forward (bf16 tensor-core path): an identity ResNet
 * bottleneck with a 64-channel middle (t[256] -> 1x1 -> 3x3 -> 1x1 + t) runs as ONE kernel per band
 * that keeps the two 64-channel intermediate maps on chip (shared memory / TMEM) and writes them
 * only where a later reader needs them (the 2PS cache rows in the FP pass, all rows in the BP
 * recompute).  Same arithmetic as the unfused kernels.  Set only to compare (tests, bench A/B). */
#define LRCNN_FLAG_NO_FUSE_BLOCK 512

typedef struct lrcnn_plan_t lrcnn_plan_t;

/* Predicted memory of a plan, in bytes (host-side accounting). */
typedef struct {
    size_t omega;          /* Eq. (3): sum over all op outputs of B*H*W*C*elem (layer-wise)  */
    size_t band_act;       /* band activation buffers (Eq. (8) working set)                  */
    size_t band_delta;     /* band delta buffers                                             */
    size_t halo_cache;     /* 2PS cache, B(N-1) sum c(t) W C elem (reading R9)  */
    size_t carry;          /* 2PS delta carry buffers                                        */
    size_t checkpoints;    /* full-width segment boundary maps           */
    size_t delta_full;     /* full-width delta ping-pong for segment boundaries              */
    size_t other;          /* head scratch, transposed weights, counters                      */
    size_t workspace;      /* total workspace bytes (everything above but omega)              */
    double tau_flops;      /* PAPER.md:375 tau for the whole batch                           */
    double fwd_flops;      /* conv FLOPs one forward sweep executes (tau + iota for OverL)    */
    double step_flops;     /* conv FLOPs one lrcnn_step executes (FP + recompute + 2 BP GEMMs)*/
} lrcnn_memory_report;

/* Build a plan (host only, synchronous, no device calls).  Validates the DAG
 * (topological order, channel/shape propagation by floor((H+2p-k)/s)+1,
 * SURVEY R1), splits segments, applies the interval rule for 2PS / the
 * extended-range rule for OverL (R3/R4) and lays out the workspace.
 * *out receives a plan owned by the caller, released with lrcnn_plan_free. */
LRCNN_API lrcnn_status lrcnn_plan(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, lrcnn_plan_t **out);
LRCNN_API lrcnn_status lrcnn_plan_free(lrcnn_plan_t *plan);

/* Budget-driven planning (Eqs. (9)-(10): "M >= Omega_FP / N" -- choose N from the
 * memory budget; the paper's greedy takes the largest bands that fit, i.e. the smallest N).  Tries
 * n_bands = 1 .. max_bands with opts (band_rows ignored, mode 2PS or OverL, any flags) and returns
 * in *out the first plan whose workspace (lrcnn_plan_sizes) is <= budget_bytes, its band count in
 * *n_bands.  The memory model is the plan's exact workspace bytes (reading R10).
 * Host only.  LRCNN_E_INFEASIBLE if no band count fits; LRCNN_E_ARG for COLUMN mode. */
LRCNN_API lrcnn_status lrcnn_plan_budget(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, size_t budget_bytes,
                                         int max_bands, lrcnn_plan_t **out, int *n_bands);
/* The 2PS greedy partitioning of Eq. (12): "max H_1^L and min N_BP" s.t. the
 * memory fits.  For N = 1 .. max_bands (the smallest first), the largest first band (first_rows_pm
 * on a grid of 1/64 of the segment outputs, from the whole height down to an equal split) whose
 * exact workspace (lrcnn_plan_sizes, reading R9/R10 of DESIGN.md) is <= budget_bytes; the other
 * N - 1 bands split the remaining rows.  Returns that plan in *out, N in *n_bands and the first band's
 * share in *first_pm (0 when the equal split is taken).  LRCNN_E_INFEASIBLE if no (N, H_1) fits.  Host only. */
LRCNN_API lrcnn_status lrcnn_plan_greedy(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts, size_t budget_bytes,
                                         int max_bands, lrcnn_plan_t **out, int *n_bands, int *first_pm);
/* The turning point: the n_bands in 1 .. max_bands with the smallest
 * workspace -- past it the 2PS halo cache (growing with N) outweighs the shrinking band working
 * set.  Ties go to the smaller N.  Host only. */
LRCNN_API lrcnn_status lrcnn_plan_turning_point(const lrcnn_net_desc *net, const lrcnn_plan_opts *opts,
                                                int max_bands, int *n_star, size_t *ws_star);

/* Sizes the caller must allocate: workspace bytes, number of parameters (flat
 * element count of params/master/grads), z^L elements (B*H_L*W_L*Cp_L). */
LRCNN_API lrcnn_status lrcnn_plan_sizes(const lrcnn_plan_t *plan, size_t *workspace_bytes, size_t *n_params,
                              size_t *zl_elems);

/* Shape of tensor `tid`: channels, padded channels, height, width. */
LRCNN_API lrcnn_status lrcnn_plan_tensor(const lrcnn_plan_t *plan, int tid, int *C, int *Cp, int *H, int *W);

/* Offset/count (elements) of a parameter block in the flat layout.
 * op in [0, n_ops): which 0 = w, 1 = bias or gamma, 2 = beta.
 * op == n_ops (head): which 0 = fc_w, 1 = fc_b.  count = 0 if absent. */
LRCNN_API lrcnn_status lrcnn_plan_param(const lrcnn_plan_t *plan, int op, int which, size_t *offset, size_t *count);

/* Segment structure: number of segments; per segment its input/output tensor ids and bands. */
LRCNN_API lrcnn_status lrcnn_plan_nsegs(const lrcnn_plan_t *plan, int *n_segs);
LRCNN_API lrcnn_status lrcnn_plan_seg(const lrcnn_plan_t *plan, int seg, int *in_tid, int *out_tid, int *n_bands);

/* Rows of tensor `tid` in band `band` of segment `seg` (bit-exact contract, R3/R4):
 * the band computes rows [*a, *b) and its buffer holds rows [*lo, *b); rows [*lo, *a) are
 * 2PS cache rows (lo == a for OverL / COLUMN).  LRCNN_E_ARG if tid is not in the segment. */
LRCNN_API lrcnn_status lrcnn_plan_rows(const lrcnn_plan_t *plan, int seg, int band, int tid, int *lo, int *a, int *b);

LRCNN_API lrcnn_status lrcnn_plan_memory(const lrcnn_plan_t *plan, lrcnn_memory_report *rep);

/* One past the last row of tensor `tid` that band `band`'s consumers read (== b of lrcnn_plan_rows,
 * except in the last band of a zero-redundancy rank, which also reads rows of rank+1). */
LRCNN_API lrcnn_status lrcnn_plan_read_end(const lrcnn_plan_t *plan, int seg, int band, int tid, int *hb);
/* Zero-redundancy halo schedule of segment `seg` (LRCNN_FLAG_ZERO_REDUNDANCY): up to max entries
 * (tensor, dir, rows [r0, r1)); dir 0 = rows of rank+1 my last band reads (received after the first
 * band; their delta goes back in the BP), dir 1 = my rows rank-1's last band reads; *n the count. */
LRCNN_API lrcnn_status lrcnn_plan_zr_halo(const lrcnn_plan_t *plan, int seg, int max, int *n, int *tid, int *dir,
                                          int *r0, int *r1);
/* Forward / backward band counts of segment `seg`: *n_bp = its bands; *n_fp = the bands the
 * forward pass runs (< *n_bp with LRCNN_FLAG_FP_MERGE when merged bands fit, else == *n_bp). */
LRCNN_API lrcnn_status lrcnn_plan_fp_bands(const lrcnn_plan_t *plan, int seg, int *n_fp, int *n_bp);

/* Row sharding (opts.world > 1): this rank owns rows [*own_lo, *own_hi) of the
 * segment output and computes tensor `tid` of the segment over [*lo, *hi) (the OverL backward
 * image of the owned rows, so ranks overlap by the receptive-field halo). */
LRCNN_API lrcnn_status lrcnn_plan_shard(const lrcnn_plan_t *plan, int seg, int tid, int *own_lo, int *own_hi,
                                        int *lo, int *hi);
/* Halo transfers of segment `seg`'s input tensor (empty for world == 1 and for the image):
 * up to max entries (peer rank, send flag, rows [r0, r1)); *n receives the count.  In FP the
 * send entries carry this rank's activation rows to the peer and the receive entries fill this
 * rank's halo; in BP the same entries run reversed and the received delta rows are added. */
LRCNN_API lrcnn_status lrcnn_plan_xfers(const lrcnn_plan_t *plan, int seg, int max, int *n, int *peer, int *send,
                                        int *r0, int *r1);

/* ---- communicators for row sharding (world > 1) --------------------------------------
 * NCCL: rank 0 calls lrcnn_comm_nccl_unique_id (128 bytes), the caller broadcasts it (e.g. with
 * torch.distributed), every rank calls lrcnn_comm_init_nccl.  libnccl.so.2 is opened at run time.
 * Loopback: `world` ranks as host threads of one process on one GPU (tests): one group, one
 * communicator per rank; graph capture is disabled for loopback ranks.
 * A plan with world > 1 needs lrcnn_plan_set_comm before forward/backward/step (else
 * LRCNN_E_STATE).  The communicator is owned by the caller and must outlive the plan's use. */
typedef struct lrcnn_comm lrcnn_comm;
LRCNN_API lrcnn_status lrcnn_comm_nccl_unique_id(void *id128);
LRCNN_API lrcnn_status lrcnn_comm_init_nccl(const void *id128, int rank, int world, lrcnn_comm **out);
LRCNN_API lrcnn_status lrcnn_comm_loopback_group(int world, void **group);
LRCNN_API lrcnn_status lrcnn_comm_loopback_group_free(void *group);
LRCNN_API lrcnn_status lrcnn_comm_init_loopback(void *group, int rank, lrcnn_comm **out);
/* Host-staged communicator (any process group the caller has, e.g. torch.distributed over gloo;
 * used where NCCL is unavailable and by the multi-process tests): the library copies the device data
 * of every halo transfer / all-reduce into pinned HOST staging buffers it owns (cudaMallocHost, grown
 * on demand; no device memory), synchronises the stream and calls
 *   exchange(user, n, peer[n], send[n], host_ptr[n], bytes[n]): send[i] = 1: send host_ptr[i][0, bytes[i])
 *       to rank peer[i]; send[i] = 0: receive bytes[i] from peer[i] into host_ptr[i] (every rank posts
 *       its sends and receives of one exchange together);
 *   allreduce(user, host_buf, n): in-place sum of n floats over all ranks;
 * (fp64 sums -- training-mode BN statistics -- go through exchange as an all-gather and are summed on
 * the host in rank order, identically on every rank);
 * each returning 0 on success, then copies the results back.  Synchronous on the host and not
 * graph-capturable (lrcnn_step runs eagerly with it).  Callbacks run on the thread that called
 * forward / backward / step. */
typedef int (*lrcnn_host_exchange_fn)(void *user, int n, const int *peer, const int *send, void *const *host_ptr,
                                      const size_t *bytes);
typedef int (*lrcnn_host_allreduce_fn)(void *user, float *host_buf, size_t n);
LRCNN_API lrcnn_status lrcnn_comm_init_host(int rank, int world, lrcnn_host_exchange_fn exchange,
                                            lrcnn_host_allreduce_fn allreduce, void *user, lrcnn_comm **out);
LRCNN_API lrcnn_status lrcnn_comm_free(lrcnn_comm *comm);
LRCNN_API lrcnn_status lrcnn_plan_set_comm(lrcnn_plan_t *plan, lrcnn_comm *comm);

/* FP (Alg. 1 l.5-11): computes z^L [B][H_L][W_L][Cp_L] (act_t) from x [B][H][W][Cp] (act_t)
 * and params (act_t, plan layout).  Leaves the 2PS halo cache and the checkpoints in ws for
 * a following lrcnn_backward_rows with the same params/x (two-phase sharing). */
LRCNN_API lrcnn_status lrcnn_forward_rows(lrcnn_plan_t *plan, const void *params, const void *x, void *zl,
                                void *ws, size_t ws_bytes, void *stream);

/* BP (Alg. 1 l.15-23): from dz^L (act_t, z^L layout) ACCUMULATES the gradient of every
 * parameter into grads (fp32, plan layout; head entries untouched).  zl is the z^L the
 * matching forward produced (read for the last op's ReLU gate and affine gradient).
 * Requires a preceding lrcnn_forward_rows on the same plan, params, x and ws (else
 * LRCNN_E_STATE): the 2PS halo cache and checkpoints it left in ws are consumed. */
LRCNN_API lrcnn_status lrcnn_backward_rows(lrcnn_plan_t *plan, const void *params, const void *x, const void *zl,
                                 const void *dzl, float *grads, void *ws, size_t ws_bytes, void *stream);

/* One training iteration (Alg. 1 l.5-24): FP, head (GAP->FC->softmax-CE mean),
 * BP, then SGD theta <- theta - lr*g on master (fp32), refresh params (act_t) from master and
 * zero grads.  grads must be zero on entry.  labels: int32 [B] on device.
 * loss_dev: one float on device receiving the mean loss of this iteration. */
LRCNN_API lrcnn_status lrcnn_step(lrcnn_plan_t *plan, float *master, void *params, float *grads, const void *x,
                        const int32_t *labels, float lr, float *loss_dev, void *ws, size_t ws_bytes,
                        void *stream);

/* The two halves of lrcnn_step, for data-parallel training where the caller reduces the
 * gradients across ranks in between (e.g. an NCCL all-reduce of `grads`, PAPER.md:577 DP):
 *   lrcnn_step_grads: FP + head + BP; grads (zero on entry) receive this rank's gradient,
 *                     loss_dev this rank's mean loss.
 *   lrcnn_sgd:        master -= lr * grads; params = act_t(master); grads = 0. */
LRCNN_API lrcnn_status lrcnn_step_grads(lrcnn_plan_t *plan, const void *params, float *grads, const void *x,
                                        const int32_t *labels, float *loss_dev, void *ws, size_t ws_bytes,
                                        void *stream);
LRCNN_API lrcnn_status lrcnn_sgd(lrcnn_plan_t *plan, float *master, void *params, float *grads, float lr,
                                 void *stream);

/* Kernel timing for the roofline (bench.py): when enabled, every conv-class launch is
 * bracketed by CUDA events on the launching stream.  lrcnn_profile_read synchronises the
 * stream and returns, for kernel class `cls` (0 = tensor-core conv FP/dgrad, 1 = wgrad,
 * 2 = other), total milliseconds, launch count and algorithmic FLOPs since the last reset. */
LRCNN_API lrcnn_status lrcnn_profile_enable(lrcnn_plan_t *plan, int enable);
LRCNN_API lrcnn_status lrcnn_profile_read(lrcnn_plan_t *plan, int cls, double *ms, long long *launches,
                                double *flops, void *stream);
LRCNN_API lrcnn_status lrcnn_profile_reset(lrcnn_plan_t *plan);
/* Per-op profile since the last reset (synchronises the stream): CSV with one line per
 * (op, kind in fwd|dgrad|wgrad|param_grad|pool_fwd|pool_bwd|elt_fwd|elt_bwd): launches, ms, FLOPs. */
LRCNN_API lrcnn_status lrcnn_profile_dump(lrcnn_plan_t *plan, const char *path, void *stream);
/* Per-kernel profile of class cls (0 conv FP + dgrad, 1 wgrad, 2 other): one line per tcgen05
 * kernel ("simt" for SIMT launches) "name,launches,ms,flops,bytes,wbytes\n" written NUL-terminated into buf
 * (bytes = algorithmic HBM bytes of the launches: each operand read once, each result written once;
 * wbytes = the written part of bytes)
 * (len bytes; LRCNN_E_ARG if too small).  Synchronises `stream` (a cudaStream_t). */
LRCNN_API lrcnn_status lrcnn_profile_kernels(lrcnn_plan_t *plan, int cls, char *buf, size_t len, void *stream);

/* Number of kernel launches the last forward/backward/step enqueued. */
LRCNN_API lrcnn_status lrcnn_last_launch_count(const lrcnn_plan_t *plan, long long *launches);
/* Of those, how many were tcgen05 tensor-core convolution kernels (FP, dgrad, wgrad). */
LRCNN_API lrcnn_status lrcnn_last_tc_launch_count(const lrcnn_plan_t *plan, long long *launches);
/* Convolution launches (FP, dgrad, wgrad) of a bf16 tensor-core plan that ran on the SIMT kernels
 * because no tensor-core kernel takes the shape (0 for the benchmarked workloads; always 0 for
 * fp32 / LRCNN_FLAG_NO_TCGEN05 plans, which are SIMT by request). */
LRCNN_API lrcnn_status lrcnn_last_simt_fallbacks(const lrcnn_plan_t *plan, long long *n);

/* Debug capture for parity tests (never on a timed path): register dst, a caller buffer holding
 * the FULL map of tensor tid ([B][H][W][Cp] act_t, tid in 1..n_ops); every following forward pass
 * (lrcnn_forward_rows, the FP and the BP recompute of lrcnn_step / lrcnn_step_grads) copies the
 * rows each band computes of that tensor into it, so after a forward dst holds the map the
 * row-centric sweep produced (every row is computed by exactly one band, R3).
 * dst = NULL unregisters.  Disables CUDA-graph replay while any buffer is registered.  Row-sharded
 * plans (world > 1) write the rows of their extended ranges (global row coordinates). */
LRCNN_API lrcnn_status lrcnn_debug_capture(lrcnn_plan_t *plan, int tid, void *dst);

LRCNN_API const char *lrcnn_last_error(void);
LRCNN_API const char *lrcnn_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LRCNN_H */

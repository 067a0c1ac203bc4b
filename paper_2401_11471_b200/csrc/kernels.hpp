// kernels.hpp -- launcher interfaces of the device kernels (internal).
//
// A View describes the rows of one NHWC tensor that a buffer holds:
//   element (b, g, x, c) lives at p + b*bs + ((g - base)*W + x)*Cp + c
//   and is DATA iff 0 <= g < H and base <= g < base + rows.
// Rows g < 0 or g >= H are the zero padding of the semi-closed padding rule
// (PAPER.md:235): the global top/bottom only -- a band cut never pads.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace lrcnn {

struct View {
    void *p = nullptr;
    int base = 0, rows = 0, H = 0, W = 0, Cp = 0;
    long long bs = 0;   // batch stride in elements
};

struct ConvFwdArgs {
    View in, out, res;         // res.p == nullptr: no residual
    const void *w = nullptr;   // [Cout][k][k][Cin_p], act_t
    const void *b = nullptr;   // bias or gamma [c_out], act_t
    const void *beta = nullptr;
    int k, s, p, c_out, epi, relu;
    int a, b_;                 // output rows [a, b_)
    int B;
};

struct DgradArgs {
    View dy;                   // delta_pre of the conv output: rows [a, b) only (others = 0)
    View dx, act;              // delta of the conv input (accumulated), its activation (gate)
    int gate;                  // producer of the input applies ReLU
    const void *w = nullptr;   // [Cout][k][k][Cin_p]
    const void *wt = nullptr;  // transposed [Cin_p][k][k][Cout_p] (tensor-core path), gamma folded
    const void *gamma = nullptr;
    int k, s, p, c_out;
    int ra, rb;                // input rows to produce
    int B;
    int write = 0;             // 1: delta_in rows [ra, rb) = gate(act) * acc, not accumulated (single writer)
    // write mode with an addend (fused residual gradient): delta_in = gate(act) * (acc + add),
    // add = the complete delta rows of the block output (rows outside add's view read as 0)
    View add;
    int add_on = 0;
    mutable bool add_done = false;   // set by a launcher that consumed the addend
};

struct WgradArgs {
    View dy, x;
    float *dw = nullptr;       // [Cout][k][k][Cin_p] fp32, accumulated
    const void *gamma = nullptr;
    float *db = nullptr;       // optional: bias (or affine beta) gradient sum_pixels dy[., co], fused
    float *dg = nullptr;       // optional: affine gamma gradient, fused as sum_{tap,ci} W * (sum_p dy x)
    const void *w = nullptr;   // weights [Cout][k][k][Cin_p] (for dg)
    mutable bool db_done = false;   // set by a launcher that accumulated db (and dg when requested)
    mutable bool dg_done = false;   // set by a launcher that accumulated dg (SIMT: always when dg is set)
    int k, s, p, c_out;
    int a, b;                  // output rows contributing
    int B;
};

struct ParamGradArgs {
    View dy;
    float *db = nullptr;       // += column sums of dy: the bias (BIAS) or beta (AFFINE) gradient
    int c_out, a, b, B;
};

struct PoolArgs {
    View in, out;              // fwd: out rows [a, b)
    View dy, dx, act;          // bwd: dy rows [a, b) of the pool output, dx rows [ra, rb)
    int gate, k, s, p, a, b, ra, rb, B;
    int acc = 1;               // bwd: 1 = dx += ..., 0 = dx rows [ra, rb) are written, not read (single writer)
};

// Fused identity bottleneck forward (bneck_tc.cu): t -> 1x1 (64) -> 3x3 (64) -> 1x1 (256) + t, frozen-BN
// affine + ReLU after each conv, over the band's output rows [a2, b2) of t2 / u.  t1 rows [a1, b1) are
// computed on chip, rows below a1 are read from the t1 view (2PS cache); t1 rows are stored in the
// windows [wlo, whi) (nwin < 0: all of [a1, b1)), t2 rows [a2, b2) when write_t2.
struct BneckArgs {
    View t, t1, t2, u;
    const void *w1 = nullptr, *w2 = nullptr, *w3 = nullptr;
    const void *g1 = nullptr, *e1 = nullptr, *g2 = nullptr, *e2 = nullptr, *g3 = nullptr, *e3 = nullptr;
    int a2 = 0, b2 = 0, a1 = 0, b1 = 0, B = 0;
    int write_t2 = 0;
    int nwin = -1;
    int wlo[16] = {}, whi[16] = {};
};

struct EltArgs {
    View x0, x1, out;          // add fwd: out = relu?(x0 + x1) on rows [a, b)
    View dy, dx, act;          // res/add bwd: dx = gate(act) * (dx + dy) on rows [a, b)
    int relu, gate, a, b, B;
    int write = 0;             // res/add bwd: 1 = dx = gate(act) * dy (single writer), 0 = accumulate
};

// SIMT kernels (fp32 parity mode and the general fallback for shapes the tensor-core
// kernels do not take); prec: 0 = fp32, 1 = bf16 storage (fp32 accumulate).
cudaError_t simt_conv_fwd(int prec, const ConvFwdArgs &a, cudaStream_t st);
cudaError_t simt_conv_dgrad(int prec, const DgradArgs &a, cudaStream_t st);
cudaError_t simt_conv_wgrad(int prec, const WgradArgs &a, cudaStream_t st);
cudaError_t simt_param_grad(int prec, const ParamGradArgs &a, cudaStream_t st);
cudaError_t simt_pool_fwd(int prec, const PoolArgs &a, cudaStream_t st);
cudaError_t simt_pool_bwd(int prec, const PoolArgs &a, cudaStream_t st);
int simt_pool_bwd_launches(const PoolArgs &a);   // kernels simt_pool_bwd enqueues
bool pool_tiled_shape(int k, int s, int Cp);      // overlapping max-pool backward as a tiled gather (single writer)
cudaError_t simt_add_fwd(int prec, const EltArgs &a, cudaStream_t st);
cudaError_t simt_acc_gate(int prec, const EltArgs &a, cudaStream_t st);

// training-mode BatchNorm (bn.cu): coef = [6][Cp] floats (a, b, p, q, mean, invstd),
// sums / S = [2][Cp] doubles (accumulated; the caller zeroes them)
cudaError_t bn_stats(int prec, const View &x, int a, int b, int B, double *sums, cudaStream_t st);
cudaError_t bn_finalize_fwd(int prec, const double *sums, const void *gamma, const void *beta, int C, int Cp,
                            double M, float *coef, cudaStream_t st);
cudaError_t bn_fwd(int prec, const View &in, const View &res, const View &out, const float *coef, int relu, int a,
                   int b, int B, cudaStream_t st);
cudaError_t bn_sums(int prec, const View &dy, const View &x, const float *coef, int a, int b, int B, double *S,
                    cudaStream_t st);
cudaError_t bn_finalize_bwd(const double *S, float *coef, int C, int Cp, double M, float *dgamma, float *dbeta,
                            cudaStream_t st);
cudaError_t bn_bwd(int prec, const View &dy, const View &x, const View &dx, const View &act, int gate, int write,
                   const float *coef, int a, int b, int B, int cs, cudaStream_t st);

void simt_set_pdl(bool on);   // programmatic dependent launch on / off for this host thread (profiling)

// head (Alg. 1 l.12-14) and update (l.24)
cudaError_t head_forward_backward(int prec, const void *zl, int B, int HW, int Cp, int C, int classes,
                                  const void *fc_w, const void *fc_b, const int32_t *labels, float *scratch,
                                  float *loss, float *g_fc_w, float *g_fc_b, void *dzl, int gate,
                                  cudaStream_t st);
// partial: B * kGapChunks(64) * Cp floats for the two-pass bf16 GAP (nullptr: one-pass kernel)
cudaError_t head_gap(int prec, const void *zl, int B, int HW, int Cp, float hw_div, float *scratch, cudaStream_t st,
                     float *partial = nullptr);
cudaError_t head_tail(int prec, const void *zl, int B, int HW, int Cp, int C, int classes, const void *fc_w,
                      const void *fc_b, const int32_t *labels, float *scratch, float *loss, float *g_fc_w,
                      float *g_fc_b, void *dzl, int gate, float hw_div, cudaStream_t st);
cudaError_t add_rows(int prec, const View &dst, int r0, int r1, const void *src, int B, cudaStream_t st);
cudaError_t gate_copy(int prec, const void *src, const void *act, void *dst, long long n, int gate,
                      cudaStream_t st);
cudaError_t sgd_update(int prec, float *master, void *params, float *grads, long long n, float lr,
                       cudaStream_t st);
cudaError_t transpose_weights(int prec, const void *w, const void *gamma, void *wt, int cout, int coutp,
                              int k, int cinp, cudaStream_t st);

}  // namespace lrcnn

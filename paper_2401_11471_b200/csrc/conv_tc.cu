// conv_tc.cu -- tcgen05 implicit-GEMM convolution kernels for sm_100a.
//
// The per-band convolutions of the row-centric sweep (Eq. (4)/(5))
// are dense contractions and run on the 5th-generation tensor cores:
//
//   FP    D[pixel, co] = sum_{ky,kx,ci} X[y-p+ky, x-p+kx, ci] W[co,ky,kx,ci]   (+ fused epilogue)
//   dgrad the same kernel on the band delta with the flipped, transposed weights
//         W'[ci,ky',kx',co] = gamma[co] W[co,k-1-ky',k-1-kx',ci] and padding k-1-p;
//         epilogue: delta_in = gate(act_in) * (delta_in + acc)  (gate-on-write)
//   wgrad dW[co,ky,kx,ci] += sum_pixels dY[pixel,co] X[pixel+off,ci]  (K = band pixels)
//
// Structure (one CTA per SM, persistent over tiles, warp-specialised, 192 threads):
//   warp 0      TMA producer: a 128-pixel rectangle (TW x TH of one image) x 64 channels
//               of the band input per stage, SWIZZLE_128B; the rows of the band are
//               addressed with band-relative coordinates so TMA's out-of-bounds zero
//               fill IS the semi-closed padding: rows < 0 or >= H and
//               rows outside the band's valid range read as zero.
//   warp 1      TMEM allocation + single-thread tcgen05.mma issue (M=128, N=BN, K=16),
//               tcgen05.commit releases smem stages and hands accumulators to the epilogue.
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 32 columns), bias/affine, residual, ReLU,
//               bf16 pack, 16-byte stores (FP) or the gated delta accumulate (dgrad);
//               wgrad: gamma scale and fp32 red.add into the flat gradient.
// Accumulators are double-buffered in TMEM so the epilogue of tile i overlaps the MMAs
// of tile i+1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <utility>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <set>

#include "tc.hpp"
#include "tc_ptx.cuh"

namespace lrcnn {

typedef __nv_bfloat16 bf16;

struct TcConv {
    View out, res, act;
    View in;               // im2col kernel: the band input it gathers from
    View add;              // dgrad addend (dg_add)
    const bf16 *bias, *beta;
    int mode;              // 0 = forward epilogue, 1 = dgrad (gated accumulate)
    int epi, relu, gate, has_res, c_real, n_out;
    int out_a, out_b, Wo, B;
    int TW, TH, tiles_x, tiles_y, m_tiles, n_tiles;
    int k, pad, in_base, cin_chunks, k_steps;
    int boff;              // halo kernel: 1 = set the descriptor base-offset field from the address
    // generalised taps (stride-s FP, parity classes of strided dgrad): the A box of tap t starts at
    // (grid_col*a_mul + tap_ox[t], grid_row*a_mul + tap_oy[t]) of the input view (TMA element
    // stride a_mul), weights tap index tap_w[t]; output pixel = (o_row0 + o_stride*grid_row, ...)
    int a_mul, ntaps, o_row0, o_col0, o_stride, halo_ok;
    int tma_out;           // FP: stage the output tile in smem and TMA-store it
    int tma_dg;            // dgrad: TMA-load delta (+ activation), combine in smem, TMA-store
    int tma_res;           // FP: the residual tile is TMA-loaded into the staging buffer
    int tap_oy[49], tap_ox[49], tap_w[49];
    int dbg;               // debug bits (bit0: skip epilogue stores); always 0 in the product
    int tw_log2;           // TW = 1 << tw_log2
    int th_log2;           // TH = 1 << th_log2
    int NBt;               // images per tile (small maps: a 128-pixel tile spans NBt images; 0/1 = one)
    int dg_write;          // dgrad: overwrite delta_in (gate * acc) instead of accumulating into it
    int dg_add;            // dgrad, with dg_write: delta_in = gate * (acc + addend tile, TMA-loaded from tmX)
    int add_req;           // host: the caller asks for the addend (conv_launch sets dg_add if the kernel takes it)
    int pat_w, pat_h, pat_ox, pat_oy;   // im2col kernel: input patch per tile (pixels) and its offset
    uint32_t fd_nt[2], fd_tx[2], fd_ty[2];   // fast division by n_tiles, tiles_x, tiles_y (mul, shift)
    int cta2;              // 1: CTA-pair kernel (k_conv_tc2): tile = 2 * pair + CTA rank, m_tiles rounded up to even
    int warp_epi;          // unused (round-1 per-warp epilogue boxes), always 0
    // tile index -> (n tile, tile column, tile row, image); n tiles vary fastest.  CTA pairs: the two
    // CTAs of a pair take consecutive pixel tiles of the same n tile (an odd last tile decodes to
    // image B: fully out of bounds for every TMA load / store).
    __device__ __forceinline__ void decode(int tile, int &nt, int &tx, int &ty, int &b) const {
        int mt;
        if (cta2) {
            const int pair = tile >> 1, mp = fdiv(pair, fd_nt);
            nt = pair - mp * n_tiles;
            mt = 2 * mp + (tile & 1);
        } else {
            mt = fdiv(tile, fd_nt);
            nt = tile - mt * n_tiles;
        }
        const int r = fdiv(mt, fd_tx);
        tx = mt - r * tiles_x;
        b = fdiv(r, fd_ty);
        ty = r - b * tiles_y;
        if (NBt > 1) b *= NBt;   // first image of the tile
    }
    // the accumulator of this CTA's tile has been drained: arrive on the MMA issuer's tempty barrier
    // (CTA pairs: the leader CTA's barrier, through the cluster window)
    __device__ __forceinline__ void tempty_arrive(uint64_t *bar) const {
        if (cta2) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(bar), 0));
        else ptx::mbar_arrive(bar);
    }
    __device__ __forceinline__ static int fdiv(int n, const uint32_t (&f)[2]) {
        return (int)((__umulhi((uint32_t)n, f[0]) + (uint32_t)n) >> f[1]);
    }
};

// n / d for 0 <= n < 2^31 as (umulhi(n, mul) + n) >> shift (round-up reciprocal)
static inline void fastdiv_init(uint32_t (&f)[2], int d) {
    uint32_t l = 0;
    while ((1ull << l) < (unsigned long long)d) ++l;
    f[0] = (uint32_t)(((1ull << 32) * ((1ull << l) - (unsigned long long)d)) / (unsigned long long)d + 1);
    f[1] = l;
}
static inline void tile_div_init(TcConv &P) {
    fastdiv_init(P.fd_nt, P.n_tiles);
    fastdiv_init(P.fd_tx, P.tiles_x);
    fastdiv_init(P.fd_ty, P.tiles_y);
    int l = 0;
    while ((1 << l) < P.TW) ++l;
    P.tw_log2 = l;
    l = 0;
    while ((1 << l) < P.TH) ++l;
    P.th_log2 = l;
}

struct TcWgrad {
    float *dw;
    const bf16 *gamma;
    float *db;             // fused bias / beta gradient (items with ky == 0 / tap == 0 and ci tile 0)
    float *dg;             // fused gamma gradient: dgamma[co] = sum_{tap,ci} W[co][tap][ci] * (sum_p dy x)
    const bf16 *w;
    int k, pad, c_out, cin_p;
    int TW, TH, tiles_x, tiles_y, pix_tiles, per_split, splits;
    int co_tiles, ci_tiles, items;
    int out_a, dy_base, x_base;
    int s;                 // conv stride (TMA element stride of the input box)
    int NB;                // k_wgrad_tc: images per pixel tile (batch folding for small maps)
};

static constexpr int kThreads = 192;
static constexpr int kWgThreads = 320;        // wgrad kernels: producer, MMA, 4 epilogue, 4 bias-sum warps

static constexpr int kConvTcEpi = 16;         // k_conv_tc: epilogue warps of the store-warp (DMA) epilogues
static constexpr int kConvTcThreads = (2 + kConvTcEpi + 1) * 32;   // producer, MMA, 16 epilogue warps, store warp
static constexpr int kConv2Threads = 352;     // k_conv_tc2: producer, MMA, 8 epilogue warps, store warp
static constexpr int kABytes = 128 * 128;   // 128 pixels x 64 bf16

static constexpr int kOutStage = 128 * 128;       // epilogue staging: 128 pixels x 64 channels bf16
template <int BN, int KC = 64, int NBUF = 4>
struct ConvCfg {
    static constexpr int kA = 128 * KC * 2, kB = BN * KC * 2;
    static constexpr int kStageBytes = kA + kB;
    // NBUF 16 KB staging buffers: FP stores / residual loads run up to NBUF-1 64-channel groups
    // ahead; dgrad: NBUF/2 (delta, activation) pairs, loads NBUF/2-1 items ahead.  NBUF = 8 (the
    // small-K 1x1 convolutions: one or two K-steps per tile, bound by the epilogue's HBM traffic --
    // residual / delta / activation tiles in, output tiles out -- not by the mainloop) keeps
    // 112 KB of epilogue loads in flight per SM instead of 48 KB; it leaves two mainloop stages.
    static constexpr int kOutBufs = NBUF;
    static constexpr int kBudget = 232448 - kOutBufs * kOutStage - 2048;
    static constexpr int kStages = kBudget / kStageBytes > 16 ? 16 : kBudget / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + kOutBufs * kOutStage + 1024 + 1024;   // align + barriers
    static constexpr uint32_t kTmemCols = 2 * BN;
};

__device__ __forceinline__ float bf2f(uint16_t u) { return __uint_as_float(((uint32_t)u) << 16); }
__device__ __forceinline__ uint32_t pack2(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t *>(&h);
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap *m, const void *src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read_n() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// FP epilogue with coalesced TMA stores: per 64-channel group the NE epilogue warps write the
// bf16 tile (128 pixels x 128 B, 128B-swizzled: conflict-free 16-byte smem stores) into one of
// two staging buffers, then one thread issues a TMA tensor store of the TW x TH pixel
// rectangle; the output map's row extent ends at the band's last computed row, so pixels
// outside the band / image are clipped by TMA.  NE = 4: a warp per TMEM lane quarter (32
// pixels) x 64 channels; NE = 8: two warps per quarter, 32 channels each (half the serial
// per-thread work per tile).  Warps lead_warp .. lead_warp+NE-1; TMEM quarter = warp % 4.
template <int NE>
__device__ __forceinline__ void epi_bar_n() { asm volatile("bar.sync 1, %0;" ::"n"(NE * 32) : "memory"); }

// bf16 pair (one 32-bit word) -> two floats
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// fp32 + bf16 -> fp32 with one rounding (sm_100 mixed-precision add, no unpacking of the bf16
// half: FHADD.BF16 reads the register half directly)
__device__ __forceinline__ float hadd_lo(uint32_t w, float x) {
    float r;
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(r) : "h"((unsigned short)(w & 0xffffu)), "f"(x));
    return r;
}
__device__ __forceinline__ float hadd_hi(uint32_t w, float x) {
    float r;
    asm("add.rn.f32.bf16 %0, %1, %2;" : "=f"(r) : "h"((unsigned short)(w >> 16)), "f"(x));
    return r;
}
// two fp32 -> bf16x2 (RNE), optionally with ReLU folded into the conversion (F2FP.RELU)
template <bool RELU>
__device__ __forceinline__ uint32_t pack2_act(float lo, float hi) {
    uint32_t d;
    if (RELU) asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    else asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    return d;
}
// per-half mask 0xffff where the bf16 activation is > 0 (ReLU'(0) = 0), packed compare
__device__ __forceinline__ uint32_t relu_mask2(uint32_t act) {
    uint32_t m;
    asm("set.gt.u32.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(act), "r"(0u));
    return m;
}

// Fast path of the FP epilogue for CH channels starting at cb (all < c_real): EPI 0 none,
// 1 bias, 2 affine; RES adds the residual; RELU.  Parameters / residual were loaded into
// pb/pe/pr before the accumulator wait.  Bias and residual are added with mixed-precision
// FHADD.BF16, ReLU is folded into the bf16 conversion: 1.5-3 instructions per element.
template <int CH, int EPI, bool RES, bool RELU>
__device__ __forceinline__ void epi_fast(const uint32_t (&v)[CH], const uint4 (&pb)[CH / 8], const uint4 (&pe)[CH / 8],
                                         const uint4 (&pr)[CH / 8], uint32_t buf, int chunk0, int m) {
#pragma unroll
    for (int c = 0; c < CH / 8; ++c) {
        const uint32_t bw[4] = {pb[c].x, pb[c].y, pb[c].z, pb[c].w};
        const uint32_t ew[4] = {pe[c].x, pe[c].y, pe[c].z, pe[c].w};
        const uint32_t rw[4] = {pr[c].x, pr[c].y, pr[c].z, pr[c].w};
        uint32_t o[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            float x0 = __uint_as_float(v[c * 8 + 2 * h]), x1 = __uint_as_float(v[c * 8 + 2 * h + 1]);
            if (EPI == 1) { x0 = hadd_lo(bw[h], x0); x1 = hadd_hi(bw[h], x1); }
            if (EPI == 2) { x0 = fmaf(x0, bf_lo(bw[h]), bf_lo(ew[h])); x1 = fmaf(x1, bf_hi(bw[h]), bf_hi(ew[h])); }
            if (RES) { x0 = hadd_lo(rw[h], x0); x1 = hadd_hi(rw[h], x1); }
            o[h] = pack2_act<RELU>(x0, x1);
        }
        st_shared_v4(buf + (((chunk0 + c) ^ (m & 7)) << 4), make_uint4(o[0], o[1], o[2], o[3]));
    }
}
template <int CH, int EPI, bool RES>
__device__ __forceinline__ void epi_fast_r(bool relu, const uint32_t (&v)[CH], const uint4 (&pb)[CH / 8],
                                           const uint4 (&pe)[CH / 8], const uint4 (&pr)[CH / 8], uint32_t buf,
                                           int chunk0, int m) {
    if (relu) epi_fast<CH, EPI, RES, true>(v, pb, pe, pr, buf, chunk0, m);
    else epi_fast<CH, EPI, RES, false>(v, pb, pe, pr, buf, chunk0, m);
}

// DMA = true (k_conv_tc): a dedicated store warp (conv_store_dma) issues every TMA store and every
// residual load; the epilogue warps wait only for their buffer (rbar: residual landed / previous store
// read) and signal gdone[buf] (count NE) -- no block barrier and no leader round trip per group.
template <int BN, int NE = 4, int NB = 2, bool DMA = false>
__device__ __forceinline__ void conv_epilogue_tma(const TcConv &P, const CUtensorMap *tmO, uint32_t tmem,
                                                  uint64_t *tfull, uint64_t *tempty, uint8_t *stage_out, int warp,
                                                  int lane, int lead_warp = 2, const CUtensorMap *tmR = nullptr,
                                                  uint64_t *rbar = nullptr, uint64_t *gdone = nullptr) {
    constexpr int CH = 64 * 4 / NE;   // channels of a 64-channel group handled per thread
    const int num_tiles = P.m_tiles * P.n_tiles;
    const int q = warp & 3, hh = (warp - lead_warp) >> 2;
    const int m = q * 32 + lane;
    const bool leader = (warp == lead_warp && lane == 0);
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    const float lo = P.relu ? 0.f : -INFINITY;
    const int my = (m >> P.tw_log2) & ((1 << P.th_log2) - 1), mx = m & ((1 << P.tw_log2) - 1);
    const int mb = P.NBt > 1 ? m >> (P.tw_log2 + P.th_log2) : 0;   // image within a batch-folded tile
    // residual through TMA: group q (64 channels of one tile, counted across this CTA's tiles) uses
    // staging buffer q % NB; its residual tile is TMA-loaded into that buffer NB-1 groups ahead
    // (barrier rbar[q % NB]), the output overwrites it in place and is TMA-stored from it.  Without
    // a residual the NB buffers rotate with NB-1 stores in flight.
    const bool rt = P.has_res && P.tma_res && tmR;
    auto ngrp = [&](int tile2) {
        int nt2, tx2, ty2, b2;
        P.decode(tile2, nt2, tx2, ty2, b2);
        const int left = P.n_out - nt2 * BN;
        return left >= BN ? BN / 64 : (left + 63) / 64;
    };
    int lt = blockIdx.x, lg = 0;   // leader: next residual group to load
    auto res_load = [&](int buf2) {
        int nt2, tx2, ty2, b2;
        P.decode(lt, nt2, tx2, ty2, b2);
        ptx::mbar_arrive_expect_tx(rbar + buf2, kOutStage);
        ptx::tma_load_4d(stage_out + buf2 * kOutStage, tmR, rbar + buf2, nt2 * BN + lg * 64, tx2 * P.TW,
                         P.out_a + ty2 * P.TH - P.res.base, b2);
        if (++lg == ngrp(lt)) { lg = 0; lt += gridDim.x; }
    };
    if (!DMA && rt && leader)
        for (int i = 0; i < NB - 1 && lt < num_tiles; ++i) res_load(i);
    int acc = 0, sbuf = 0;
    uint32_t aphase = 0, rphases = 0;   // bit i: parity of the next completion of rbar[i]
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int nt, tx, ty, b;
        P.decode(tile, nt, tx, ty, b);
        const int yg0 = P.out_a + ty * P.TH, xg0 = tx * P.TW, n0 = nt * BN;
        const int yg = yg0 + my, xg = xg0 + mx;
        const bool valid = yg < P.out_b && xg < P.Wo && b + mb < P.B;
        // invalid pixels (clipped by the TMA store) read the residual's first pixel instead
        const bf16 *resp = !P.has_res || rt ? nullptr
                           : valid          ? (const bf16 *)P.res.p + (long long)(b + mb) * P.res.bs +
                                               ((long long)(yg - P.res.base) * P.res.W + xg) * P.res.Cp
                                            : (const bf16 *)P.res.p;
        ptx::mbar_wait(tfull + acc, aphase);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int grp = 0; grp < BN / 64; ++grp) {
            const int nb = n0 + grp * 64;
            if (nb >= P.n_out) break;
            const int cb = nb + hh * CH;              // this thread's first channel
            uint32_t v[CH];
            if constexpr (CH == 16) {
                ptx::tmem_ld16(tq + acc * BN + grp * 64 + hh * CH, *reinterpret_cast<uint32_t(*)[16]>(v));
            } else {
#pragma unroll
                for (int h = 0; h < CH / 32; ++h)
                    ptx::tmem_ld32(tq + acc * BN + grp * 64 + hh * CH + h * 32, *reinterpret_cast<uint32_t(*)[32]>(v + h * 32));
            }
            // per-channel epilogue parameters (identical for every pixel) and the residual
            uint4 pb[CH / 8], pe[CH / 8], pr[CH / 8];
#pragma unroll
            for (int c = 0; c < CH / 8; ++c) {
                const int n = cb + c * 8;
                const bool in = n < P.n_out;
                pb[c] = P.epi != 0 && in ? *reinterpret_cast<const uint4 *>(P.bias + n) : make_uint4(0, 0, 0, 0);
                pe[c] = P.epi == 2 && in ? *reinterpret_cast<const uint4 *>(P.beta + n) : make_uint4(0, 0, 0, 0);
                pr[c] = resp && in ? *reinterpret_cast<const uint4 *>(resp + n) : make_uint4(0, 0, 0, 0);
            }
            const bool ragged = cb + CH > P.c_real;   // channels >= c_real get 0 (affine) / no bias
            ptx::tmem_ld_wait();
            const uint32_t buf = ptx::smem_u32(stage_out + sbuf * kOutStage + m * 128);
            const int chunk0 = hh * (CH / 8);
            if (rt || DMA) {
                ptx::mbar_wait(rbar + sbuf, (rphases >> sbuf) & 1);   // residual in buf / buf free (DMA)
                rphases ^= 1u << sbuf;
            }
            if (rt) {
                // each thread reads, then overwrites, only its own row's chunks: no barrier needed
#pragma unroll
                for (int c = 0; c < CH / 8; ++c) pr[c] = ld_shared_v4(buf + (((chunk0 + c) ^ (m & 7)) << 4));
            }
            if (!ragged && P.epi == 1 && !P.has_res) epi_fast_r<CH, 1, false>(P.relu, v, pb, pe, pr, buf, chunk0, m);
            else if (!ragged && P.epi == 2 && !P.has_res) epi_fast_r<CH, 2, false>(P.relu, v, pb, pe, pr, buf, chunk0, m);
            else if (!ragged && P.epi == 2 && P.has_res) epi_fast_r<CH, 2, true>(P.relu, v, pb, pe, pr, buf, chunk0, m);
            else if (!ragged && P.epi == 1 && P.has_res) epi_fast_r<CH, 1, true>(P.relu, v, pb, pe, pr, buf, chunk0, m);
            else if (!ragged && P.epi == 0 && !P.has_res) epi_fast_r<CH, 0, false>(P.relu, v, pb, pe, pr, buf, chunk0, m);
            else {
#pragma unroll
                for (int c = 0; c < CH / 8; ++c) {
                    const int n = cb + c * 8;
                    const uint16_t *bh = reinterpret_cast<const uint16_t *>(&pb[c]);
                    const uint16_t *eh = reinterpret_cast<const uint16_t *>(&pe[c]);
                    const uint16_t *rh = reinterpret_cast<const uint16_t *>(&pr[c]);
                    float f[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        float x = __uint_as_float(v[c * 8 + j]);
                        const bool live = !ragged || n + j < P.c_real;
                        if (P.epi == 1) x += live ? bf2f(bh[j]) : 0.f;
                        else if (P.epi == 2) x = live ? bf2f(bh[j]) * x + bf2f(eh[j]) : 0.f;
                        x += bf2f(rh[j]);
                        f[j] = fmaxf(x, lo);
                    }
                    uint4 o;
                    o.x = pack2(f[0], f[1]); o.y = pack2(f[2], f[3]); o.z = pack2(f[4], f[5]); o.w = pack2(f[6], f[7]);
                    st_shared_v4(buf + (((chunk0 + c) ^ (m & 7)) << 4), o);
                }
            }
            fence_async_smem();
            if (DMA) {   // the store warp takes it from here
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(gdone + sbuf);
                sbuf = sbuf + 1 == NB ? 0 : sbuf + 1;
                continue;
            }
            // without a residual: before this barrier the leader makes sure the NEXT group's buffer
            // (last stored NB groups before it) has been read by its store
            if (!rt && leader) bulk_wait_read_n<NB - 2>();
            epi_bar_n<NE>();
            if (leader && !(P.dbg & 1)) {
                tma_store_4d(tmO, stage_out + sbuf * kOutStage, nb, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.out.base, b);
                bulk_commit();
            }
            if (rt && leader && lt < num_tiles) {   // residual NB-1 groups ahead, into the buffer group q-1 used
                bulk_wait_read1();                     // ... once that group's store has read it
                res_load(sbuf == 0 ? NB - 1 : sbuf - 1);
            }
            sbuf = sbuf + 1 == NB ? 0 : sbuf + 1;
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) P.tempty_arrive(tempty + acc);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    if (leader) bulk_wait_all();
}

// The store warp of conv_epilogue_tma<..., DMA = true>: walks the CTA's (tile, 64-channel group) sequence;
// group k uses staging buffer k % NB.  It fills every buffer first (the residual tile, or just "free"),
// then per group waits for the NE epilogue warps (gdone), TMA-stores the buffer and, once the store has
// read it, refills the buffer for group k + NB.
template <int BN, int NB>
__device__ __forceinline__ void conv_store_dma(const TcConv &P, const CUtensorMap *tmO, uint8_t *stage_out,
                                               const CUtensorMap *tmR, uint64_t *rbar, uint64_t *gdone) {
    const int num_tiles = P.m_tiles * P.n_tiles;
    const bool rt = P.has_res && P.tma_res && tmR;
    auto ngrp = [&](int tile2) {
        int nt2, tx2, ty2, b2;
        P.decode(tile2, nt2, tx2, ty2, b2);
        const int left = P.n_out - nt2 * BN;
        return left >= BN ? BN / 64 : (left + 63) / 64;
    };
    int lt = blockIdx.x, lg = 0;   // next group to make ready
    auto fill = [&](int buf) {
        if (lt >= num_tiles) return;
        if (rt) {
            int nt2, tx2, ty2, b2;
            P.decode(lt, nt2, tx2, ty2, b2);
            ptx::mbar_arrive_expect_tx(rbar + buf, kOutStage);
            ptx::tma_load_4d(stage_out + buf * kOutStage, tmR, rbar + buf, nt2 * BN + lg * 64, tx2 * P.TW,
                             P.out_a + ty2 * P.TH - P.res.base, b2);
        } else {
            ptx::mbar_arrive(rbar + buf);
        }
        if (++lg == ngrp(lt)) { lg = 0; lt += gridDim.x; }
    };
    for (int i = 0; i < NB; ++i) fill(i);
    int sbuf = 0;
    uint32_t gph = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int nt, tx, ty, b;
        P.decode(tile, nt, tx, ty, b);
        const int yg0 = P.out_a + ty * P.TH, xg0 = tx * P.TW, n0 = nt * BN;
        const int ng = ngrp(tile);
        for (int grp = 0; grp < ng; ++grp) {
            ptx::mbar_wait(gdone + sbuf, (gph >> sbuf) & 1);
            gph ^= 1u << sbuf;
            tma_store_4d(tmO, stage_out + sbuf * kOutStage, n0 + grp * 64, P.o_col0 + P.o_stride * xg0,
                         P.o_row0 + P.o_stride * yg0 - P.out.base, b);
            bulk_commit();
            bulk_wait_read0();   // the store has read the buffer: refill it for group k + NB
            fill(sbuf);
            sbuf = sbuf + 1 == NB ? 0 : sbuf + 1;
        }
    }
    bulk_wait_all();
}


// dgrad epilogue through TMA (unit output stride): per 64-channel group the delta tile of the
// conv input (and, when its producer applies ReLU, the activation tile) is TMA-loaded into
// smem, combined with the accumulator (gate-on-write: delta = gate(act) * (delta + acc)) in
// place and TMA-stored back; rows >= out_b / columns >= W are clipped by the maps.
template <int BN, int NE = 4>
__device__ __forceinline__ void conv_epilogue_tma_dg(const TcConv &P, const CUtensorMap *tmO, const CUtensorMap *tmG,
                                                     uint32_t tmem, uint64_t *tfull, uint64_t *tempty,
                                                     uint8_t *stage_out, uint64_t *ebar, int warp, int lane) {
    constexpr int CH = 64 * 4 / NE;           // channels of a 64-channel group per thread
    const int num_tiles = P.m_tiles * P.n_tiles;
    const int q = warp & 3, m = q * 32 + lane, hh = (warp - 2) >> 2;
    const bool leader = (warp == 2 && lane == 0);
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    uint8_t *bufD = stage_out, *bufG = stage_out + kOutStage;
    const uint32_t rowD = ptx::smem_u32(bufD) + m * 128, rowG = ptx::smem_u32(bufG) + m * 128;
    // bytes the leader TMA-loads per group: the delta tile (unless overwritten) and the activation tile
    // (gate); 0 bytes is a plain arrive that still orders the staging buffer's reuse after the store
    const uint32_t ebytes = (P.dg_write ? 0u : (uint32_t)kOutStage) + (P.gate ? (uint32_t)kOutStage : 0u);
    int acc = 0;
    uint32_t aphase = 0, ephase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int nt, tx, ty, b;
        P.decode(tile, nt, tx, ty, b);
        const int yg0 = P.out_a + ty * P.TH, xg0 = tx * P.TW, n0 = nt * BN;
        const int ngrp = min(BN / 64, (P.n_out - n0 + 63) / 64);
        if (leader) {
            bulk_wait_read0();
            ptx::mbar_arrive_expect_tx(ebar, ebytes);
            if (!P.dg_write) ptx::tma_load_4d(bufD, tmO, ebar, n0, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.out.base, b);
            if (P.gate) ptx::tma_load_4d(bufG, tmG, ebar, n0, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.act.base, b);
        }
        ptx::mbar_wait(tfull + acc, aphase);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int grp = 0; grp < ngrp; ++grp) {
            const int nb = n0 + grp * 64;
            uint32_t v[CH];
            if constexpr (CH == 16) {
                ptx::tmem_ld16(tq + acc * BN + grp * 64 + hh * CH, *reinterpret_cast<uint32_t(*)[16]>(v));
            } else {
#pragma unroll
                for (int h = 0; h < CH / 32; ++h)
                    ptx::tmem_ld32(tq + acc * BN + grp * 64 + hh * CH + h * 32, *reinterpret_cast<uint32_t(*)[32]>(v + h * 32));
            }
            ptx::tmem_ld_wait();
            ptx::mbar_wait(ebar, ephase);
            ephase ^= 1;
#pragma unroll
            for (int cc = 0; cc < CH / 8; ++cc) {
                const int c = hh * (CH / 8) + cc;
                const uint32_t off = (uint32_t)((c ^ (m & 7)) << 4);
                const uint4 dd = P.dg_write ? make_uint4(0, 0, 0, 0) : ld_shared_v4(rowD + off);
                const uint4 gg = P.gate ? ld_shared_v4(rowG + off) : make_uint4(0, 0, 0, 0);
                const uint32_t dw[4] = {dd.x, dd.y, dd.z, dd.w}, gw[4] = {gg.x, gg.y, gg.z, gg.w};
                uint32_t o[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float x0 = hadd_lo(dw[h], __uint_as_float(v[cc * 8 + 2 * h]));
                    const float x1 = hadd_hi(dw[h], __uint_as_float(v[cc * 8 + 2 * h + 1]));
                    o[h] = pack2_act<false>(x0, x1);
                    if (P.gate) o[h] &= relu_mask2(gw[h]);   // gate-on-write: delta = [act > 0] (delta + acc)
                }
                st_shared_v4(rowD + off, make_uint4(o[0], o[1], o[2], o[3]));
            }
            fence_async_smem();
            epi_bar_n<NE>();
            if (leader) {
                tma_store_4d(tmO, bufD, nb, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.out.base, b);
                bulk_commit();
                if (grp + 1 < ngrp) {   // next group: wait until the store has read bufD, then reload
                    bulk_wait_read0();
                    ptx::mbar_arrive_expect_tx(ebar, ebytes);
                    if (!P.dg_write) ptx::tma_load_4d(bufD, tmO, ebar, nb + 64, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.out.base, b);
                    if (P.gate) ptx::tma_load_4d(bufG, tmG, ebar, nb + 64, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.act.base, b);
                }
            }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) P.tempty_arrive(tempty + acc);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    if (leader) bulk_wait_all();
}

// dgrad epilogue, double-buffered: two (delta, activation) staging pairs and two mbarriers.  The
// work items are the (tile, 64-channel group)s of this CTA in order; item k uses pair k % 2, and the
// TMA loads of item k+1 are issued before item k's combine (once item k-1's store has read that
// pair), so the HBM latency of the delta / activation tiles overlaps the current item instead of
// being exposed once per tile (small-K layers: a 64-channel 3x3 dgrad tile is ~1200 MMA cycles).
// DMA = true (k_conv_tc): conv_store_dma_dg issues all loads and stores; the epilogue warps signal
// gdone[pair] (count NE) after combining an item instead of a block barrier + leader store.
template <int BN, int NE = 4, int NP = 2, bool DMA = false>
__device__ __forceinline__ void conv_epilogue_tma_dg2(const TcConv &P, const CUtensorMap *tmO, const CUtensorMap *tmG,
                                                      uint32_t tmem, uint64_t *tfull, uint64_t *tempty,
                                                      uint8_t *stage_out, uint64_t *ebar, int warp, int lane,
                                                      int lead_warp = 2, const CUtensorMap *tmX = nullptr,
                                                      uint64_t *gdone = nullptr) {
    constexpr int CH = 64 * 4 / NE;           // channels of a 64-channel group per thread
    const int num_tiles = P.m_tiles * P.n_tiles;
    const int q = warp & 3, m = q * 32 + lane, hh = (warp - lead_warp) >> 2;
    const bool leader = (warp == lead_warp && lane == 0);
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    // delta tile: the old delta (accumulate), the addend (dg_add, from tmX) or nothing (single writer)
    const bool dload = !P.dg_write || (P.dg_add && tmX);
    const CUtensorMap *tmD = P.dg_write ? tmX : tmO;
    const uint32_t ebytes = (dload ? (uint32_t)kOutStage : 0u) + (P.gate ? (uint32_t)kOutStage : 0u);
    // pair i: delta buffer stage_out + 2i*16K, activation buffer stage_out + (2i+1)*16K
    auto issue = [&](int tile, int grp, int pi) {
        int nt, tx, ty, b;
        P.decode(tile, nt, tx, ty, b);
        const int nb = nt * BN + grp * 64, xg0 = tx * P.TW, yg0 = P.out_a + ty * P.TH;
        uint8_t *bd = stage_out + (2 * pi) * kOutStage;
        ptx::mbar_arrive_expect_tx(ebar + pi, ebytes);
        if (dload) ptx::tma_load_4d(bd, tmD, ebar + pi, nb, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - (P.dg_write ? P.add.base : P.out.base), b);
        if (P.gate) ptx::tma_load_4d(bd + kOutStage, tmG, ebar + pi, nb, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.act.base, b);
    };
    auto ngroups = [&](int tile) {
        int nt, tx, ty, b;
        P.decode(tile, nt, tx, ty, b);
        return min(BN / 64, (P.n_out - nt * BN + 63) / 64);
    };
    // item = (tile, group) of this CTA in order; item k uses pair k % NP; the first NP-1 are issued here
    int it_tile = blockIdx.x, it_grp = 0;             // next item to issue
    auto advance_issue = [&]() {
        if (++it_grp == ngroups(it_tile)) { it_grp = 0; it_tile += gridDim.x; }
    };
    int ipair = 0;
    if (leader && !DMA)
        for (int i = 0; i < NP - 1 && it_tile < num_tiles; ++i) {
            issue(it_tile, it_grp, ipair);
            ipair = ipair + 1 == NP ? 0 : ipair + 1;
            advance_issue();
        }
    int acc = 0, pi = 0;
    uint32_t aphase = 0, ephase = 0;   // bit i: parity of the next completion of ebar[i]
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int nt, tx, ty, b;
        P.decode(tile, nt, tx, ty, b);
        const int yg0 = P.out_a + ty * P.TH, xg0 = tx * P.TW, n0 = nt * BN;
        const int ngrp = ngroups(tile);
        ptx::mbar_wait(tfull + acc, aphase);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int grp = 0; grp < ngrp; ++grp) {
            const int nb = n0 + grp * 64;
            uint32_t v[CH];
            if constexpr (CH == 16) {
                ptx::tmem_ld16(tq + acc * BN + grp * 64 + hh * CH, *reinterpret_cast<uint32_t(*)[16]>(v));
            } else {
#pragma unroll
                for (int h = 0; h < CH / 32; ++h)
                    ptx::tmem_ld32(tq + acc * BN + grp * 64 + hh * CH + h * 32, *reinterpret_cast<uint32_t(*)[32]>(v + h * 32));
            }
            if (!DMA && leader && it_tile < num_tiles) {   // prefetch NP-1 items ahead into the pair item k-1 used
                bulk_wait_read0();                     // (its store, the latest committed, has read it)
                issue(it_tile, it_grp, ipair);
                ipair = ipair + 1 == NP ? 0 : ipair + 1;
                advance_issue();
            }
            ptx::tmem_ld_wait();
            ptx::mbar_wait(ebar + pi, (ephase >> pi) & 1);
            ephase ^= 1u << pi;
            const uint32_t rowD = ptx::smem_u32(stage_out + (2 * pi) * kOutStage) + m * 128;
            const uint32_t rowG = rowD + kOutStage;
#pragma unroll
            for (int cc = 0; cc < CH / 8; ++cc) {
                const int c = hh * (CH / 8) + cc;
                const uint32_t off = (uint32_t)((c ^ (m & 7)) << 4);
                const uint4 dd = dload ? ld_shared_v4(rowD + off) : make_uint4(0, 0, 0, 0);
                const uint4 gg = P.gate ? ld_shared_v4(rowG + off) : make_uint4(0, 0, 0, 0);
                const uint32_t dw[4] = {dd.x, dd.y, dd.z, dd.w}, gw[4] = {gg.x, gg.y, gg.z, gg.w};
                uint32_t o[4];
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    const float x0 = hadd_lo(dw[h], __uint_as_float(v[cc * 8 + 2 * h]));
                    const float x1 = hadd_hi(dw[h], __uint_as_float(v[cc * 8 + 2 * h + 1]));
                    o[h] = pack2_act<false>(x0, x1);
                    if (P.gate) o[h] &= relu_mask2(gw[h]);   // gate-on-write: delta = [act > 0] (delta + acc)
                }
                st_shared_v4(rowD + off, make_uint4(o[0], o[1], o[2], o[3]));
            }
            fence_async_smem();
            if (DMA) {
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(gdone + pi);
                pi = pi + 1 == NP ? 0 : pi + 1;
                continue;
            }
            epi_bar_n<NE>();
            if (leader) {
                tma_store_4d(tmO, stage_out + (2 * pi) * kOutStage, nb, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.out.base, b);
                bulk_commit();
            }
            pi = pi + 1 == NP ? 0 : pi + 1;
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) P.tempty_arrive(tempty + acc);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    if (leader) bulk_wait_all();
}

// The store warp of conv_epilogue_tma_dg2<..., DMA = true>: item k = (tile, 64-channel group) of this CTA
// uses staging pair k % NP (delta buffer, activation buffer).  All pairs are loaded first; per item it
// waits for the epilogue warps (gdone), TMA-stores the combined delta and, once the store has read the
// pair, loads item k + NP into it.
template <int BN, int NP>
__device__ __forceinline__ void conv_store_dma_dg(const TcConv &P, const CUtensorMap *tmO, const CUtensorMap *tmG,
                                                  const CUtensorMap *tmX, uint8_t *stage_out, uint64_t *ebar,
                                                  uint64_t *gdone) {
    const int num_tiles = P.m_tiles * P.n_tiles;
    const bool dload = !P.dg_write || (P.dg_add && tmX);
    const CUtensorMap *tmD = P.dg_write ? tmX : tmO;
    const uint32_t ebytes = (dload ? (uint32_t)kOutStage : 0u) + (P.gate ? (uint32_t)kOutStage : 0u);
    auto ngroups = [&](int tile) {
        int nt, tx, ty, b;
        P.decode(tile, nt, tx, ty, b);
        return min(BN / 64, (P.n_out - nt * BN + 63) / 64);
    };
    int it_tile = blockIdx.x, it_grp = 0;   // next item to load
    auto issue = [&](int pi) {
        if (it_tile >= num_tiles) return;
        int nt, tx, ty, b;
        P.decode(it_tile, nt, tx, ty, b);
        const int nb = nt * BN + it_grp * 64, xg0 = tx * P.TW, yg0 = P.out_a + ty * P.TH;
        uint8_t *bd = stage_out + (2 * pi) * kOutStage;
        ptx::mbar_arrive_expect_tx(ebar + pi, ebytes);
        if (dload) ptx::tma_load_4d(bd, tmD, ebar + pi, nb, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - (P.dg_write ? P.add.base : P.out.base), b);
        if (P.gate) ptx::tma_load_4d(bd + kOutStage, tmG, ebar + pi, nb, P.o_col0 + P.o_stride * xg0, P.o_row0 + P.o_stride * yg0 - P.act.base, b);
        if (++it_grp == ngroups(it_tile)) { it_grp = 0; it_tile += gridDim.x; }
    };
    for (int i = 0; i < NP; ++i) issue(i);
    int pi = 0;
    uint32_t gph = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        int nt, tx, ty, b;
        P.decode(tile, nt, tx, ty, b);
        const int yg0 = P.out_a + ty * P.TH, xg0 = tx * P.TW, n0 = nt * BN;
        const int ng = ngroups(tile);
        for (int grp = 0; grp < ng; ++grp) {
            ptx::mbar_wait(gdone + pi, (gph >> pi) & 1);
            gph ^= 1u << pi;
            tma_store_4d(tmO, stage_out + (2 * pi) * kOutStage, n0 + grp * 64, P.o_col0 + P.o_stride * xg0,
                         P.o_row0 + P.o_stride * yg0 - P.out.base, b);
            bulk_commit();
            bulk_wait_read0();
            issue(pi);
            pi = pi + 1 == NP ? 0 : pi + 1;
        }
    }
    bulk_wait_all();
}


// Epilogue warps (4 warps = 128 TMEM lanes = 128 pixels of the tile): tcgen05.ld the
// accumulator in 32-column chunks, apply the fused epilogue, 16-byte bf16 stores.
template <int BN, int NE = 4>
__device__ __forceinline__ void conv_epilogue(const TcConv &P, uint32_t tmem, uint64_t *tfull, uint64_t *tempty,
                                              int warp, int lane) {
    const int num_tiles = P.m_tiles * P.n_tiles;
    const int ew = warp & 3;                  // TMEM lane quarter this warp may access
    const int m = ew * 32 + lane;             // accumulator row = pixel in the tile
    const int hh = (warp - 2) >> 2;           // NE = 8: two warps per quarter split the 32-column chunks
    int acc = 0;
    uint32_t aphase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int nt = tile % P.n_tiles, mt = tile / P.n_tiles;
        const int tx = mt % P.tiles_x, r = mt / P.tiles_x, ty = r % P.tiles_y;
        const int b = (r / P.tiles_y) * (P.NBt > 1 ? P.NBt : 1) + m / (P.TW * P.TH);
        const int yg = P.out_a + ty * P.TH + (m / P.TW) % P.TH, xg = tx * P.TW + m % P.TW, n0 = nt * BN;
        const bool valid = yg < P.out_b && xg < P.Wo && b < P.B;
        const int y = P.o_row0 + P.o_stride * yg, x = P.o_col0 + P.o_stride * xg;
        const long long pix = valid ? (long long)b * P.out.bs + ((long long)(y - P.out.base) * P.out.W + x) * P.out.Cp : 0;
        ptx::mbar_wait(tfull + acc, aphase);
        ptx::tc_fence_after();
#pragma unroll 1
        for (int c = NE == 8 ? hh : 0; c < BN / 32; c += NE / 4) {
            uint32_t v[32];
            ptx::tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + acc * BN + c * 32, v);
            ptx::tmem_ld_wait();
            if (!valid || (P.dbg & 1)) continue;
#pragma unroll
            for (int g = 0; g < 4; ++g) {
                const int n = n0 + c * 32 + g * 8;
                if (n >= P.n_out) break;
                float f[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(v[g * 8 + j]);
                bf16 *dst = (bf16 *)P.out.p + pix + n;
                if (P.mode == 0) {
                    if (P.epi != 0) {
                        uint4 bb = *reinterpret_cast<const uint4 *>(P.bias + n);
                        const uint16_t *bh = reinterpret_cast<const uint16_t *>(&bb);
                        uint4 be = P.epi == 2 ? *reinterpret_cast<const uint4 *>(P.beta + n) : make_uint4(0, 0, 0, 0);
                        const uint16_t *beh = reinterpret_cast<const uint16_t *>(&be);
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            float bj = n + j < P.c_real ? bf2f(bh[j]) : 0.f;
                            if (P.epi == 1) f[j] += bj;
                            else f[j] = n + j < P.c_real ? bj * f[j] + bf2f(beh[j]) : 0.f;
                        }
                    }
                    if (P.has_res) {
                        uint4 rr = *reinterpret_cast<const uint4 *>(
                            (const bf16 *)P.res.p + (long long)b * P.res.bs +
                            ((long long)(y - P.res.base) * P.res.W + x) * P.res.Cp + n);
                        const uint16_t *rh = reinterpret_cast<const uint16_t *>(&rr);
#pragma unroll
                        for (int j = 0; j < 8; ++j) f[j] += bf2f(rh[j]);
                    }
                    if (P.relu) {
#pragma unroll
                        for (int j = 0; j < 8; ++j) f[j] = fmaxf(f[j], 0.f);
                    }
                } else {
                    uint4 od = P.dg_write ? make_uint4(0, 0, 0, 0) : *reinterpret_cast<const uint4 *>(dst);
                    const uint16_t *oh = reinterpret_cast<const uint16_t *>(&od);
                    uint4 ac = make_uint4(0, 0, 0, 0);
                    if (P.gate)
                        ac = *reinterpret_cast<const uint4 *>(
                            (const bf16 *)P.act.p + (long long)b * P.act.bs +
                            ((long long)(y - P.act.base) * P.act.W + x) * P.act.Cp + n);
                    const uint16_t *ah = reinterpret_cast<const uint16_t *>(&ac);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        f[j] += bf2f(oh[j]);
                        if (P.gate && !(bf2f(ah[j]) > 0.f)) f[j] = 0.f;
                    }
                }
                uint4 o;
                o.x = pack2(f[0], f[1]); o.y = pack2(f[2], f[3]); o.z = pack2(f[4], f[5]); o.w = pack2(f[6], f[7]);
                *reinterpret_cast<uint4 *>(dst) = o;
            }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) P.tempty_arrive(tempty + acc);
        if (++acc == 2) { acc = 0; aphase ^= 1; }
    }
    }

// ------------------------------------------------------------------ conv FP / dgrad
// KC = input channels per pipeline stage: 64 (128-byte rows, SWIZZLE_128B, 4 MMAs of K=16) for
// regular layers, 16 (32-byte rows, SWIZZLE_32B, 1 MMA) for small-channel layers (padded RGB
// input of conv1_1 / the 7x7 stem), which would otherwise waste 8x tensor work on zero channels.
template <int BN, int KC, int NBUF>
__global__ void __launch_bounds__(kConvTcThreads, 1)
    k_conv_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmG, const TcConv P,
              const __grid_constant__ CUtensorMap tmX) {
    using Cfg = ConvCfg<BN, KC, NBUF>;
    constexpr int S = Cfg::kStages;
    constexpr int ABYTES = Cfg::kA, BBYTES = Cfg::kB;
    constexpr uint32_t SBO = 8 * KC * 2;             // 8-row core-matrix groups
    constexpr uint32_t LAYOUT = KC == 64 ? 2u : 6u;  // SWIZZLE_128B : SWIZZLE_32B
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;
    uint8_t *sB = smem + S * ABYTES;
    uint8_t *sO = sB + S * BBYTES;                   // kOutBufs x 16 KB epilogue staging (1024-aligned)
    uint64_t *full = (uint64_t *)(sO + Cfg::kOutBufs * kOutStage);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint64_t *ebar = tempty + 2;                     // staging barriers: dgrad pairs / residual ring (NBUF),
    uint32_t *tslot = (uint32_t *)(ebar + 32);       // per-warp rings (8 warps x NBUF / 2)

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { ptx::mbar_init(full + i, 1); ptx::mbar_init(empty + i, 1); }
        // store-warp epilogues: 16 epilogue warps + conv_store_dma(_dg); otherwise warps 2..9 only
        const bool dma = P.tma_out || (P.tma_dg && Cfg::kOutBufs >= 4);
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, dma ? kConvTcEpi : 8); }
        for (int i = 0; i < 2 * NBUF; ++i)                                       // staging rings; gdone[NBUF]
            ptx::mbar_init(ebar + i, dma && i >= NBUF ? kConvTcEpi : 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, Cfg::kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int num_tiles = P.m_tiles * P.n_tiles;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int nt = tile % P.n_tiles, mt = tile / P.n_tiles;
                const int tx = mt % P.tiles_x, r = mt / P.tiles_x, ty = r % P.tiles_y;
                const int b = (r / P.tiles_y) * (P.NBt > 1 ? P.NBt : 1);
                const int y0 = (P.out_a + ty * P.TH) * P.a_mul, x0 = tx * P.TW * P.a_mul, n0 = nt * BN;
                for (int ks = 0; ks < P.k_steps; ++ks) {
                    const int tap = ks / P.cin_chunks, c = ks - tap * P.cin_chunks;
                    ptx::mbar_wait(empty + stage, phase ^ 1);
                    ptx::mbar_arrive_expect_tx(full + stage, ABYTES + BBYTES);
                    ptx::tma_load_4d(sA + stage * ABYTES, &tmA, full + stage, c * KC, x0 + P.tap_ox[tap],
                                     y0 + P.tap_oy[tap] - P.in_base, b);
                    ptx::tma_load_3d(sB + stage * BBYTES, &tmB, full + stage, c * KC, P.tap_w[tap], n0);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 0, 0);
            const uint64_t dA = ptx::smem_desc(ptx::smem_u32(sA), 16, SBO, LAYOUT);
            const uint64_t dB = ptx::smem_desc(ptx::smem_u32(sB), 16, SBO, LAYOUT);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            int stage = 0, acc = 0;
            uint32_t phase = 0, aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int ks = 0; ks < P.k_steps; ++ks) {
                    ptx::mbar_wait(full + stage, phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = (uint32_t)dA + stage * (ABYTES >> 4);
                    const uint32_t b0 = (uint32_t)dB + stage * (BBYTES >> 4);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < KC / 16; ++kk)
                            ptx::umma_bf16_1t(d, a0 + 2 * kk, hiA, b0 + 2 * kk, hiB, idesc, (ks | kk) != 0);
                        ptx::umma_commit_1t(empty + stage);
                        if (ks + 1 == P.k_steps) ptx::umma_commit_1t(tfull + acc);
                    }
                    __syncwarp();
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else if (warp == 2 + kConvTcEpi) {
        if (lane == 0) {
            if (P.tma_out) conv_store_dma<BN, Cfg::kOutBufs>(P, &tmO, sO, &tmG, ebar, ebar + NBUF);
            else if (P.tma_dg && Cfg::kOutBufs >= 4)
                conv_store_dma_dg<BN, Cfg::kOutBufs / 2>(P, &tmO, &tmG, &tmX, sO, ebar, ebar + NBUF);
        }
    } else {
        if (P.tma_out)
            conv_epilogue_tma<BN, kConvTcEpi, Cfg::kOutBufs, true>(P, &tmO, tmem, tfull, tempty, sO, warp, lane, 2, &tmG,
                                                                   ebar, ebar + NBUF);
        else if (P.tma_dg && Cfg::kOutBufs >= 4)
            conv_epilogue_tma_dg2<BN, kConvTcEpi, Cfg::kOutBufs / 2, true>(P, &tmO, &tmG, tmem, tfull, tempty, sO, ebar, warp,
                                                                           lane, 2, &tmX, ebar + NBUF);
        else if (warp < 10) {   // the other epilogues run on warps 2..9
            if (P.tma_dg) conv_epilogue_tma_dg<BN, 8>(P, &tmO, &tmG, tmem, tfull, tempty, sO, ebar, warp, lane);
            else conv_epilogue<BN, 8>(P, tmem, tfull, tempty, warp, lane);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, Cfg::kTmemCols);
    }
}

// ------------------------------------------------------------------ conv FP / dgrad on CTA pairs (cta_group::2)
// The per-tap kernel above is bound by its TMA loads (48 KB per 64-channel K-step at BN = 256, one
// 128-pixel A box + the BN x 64 weight box, for 512 tensor cycles).  Here two CTAs of a cluster
// (one TPC) form one M = 256 x N = BN tcgen05.mma.cta_group::2: each CTA loads its own 128-pixel
// A tile and HALF of the weight tile (BN/2 rows), the leader issues the MMA over both CTAs' smem and
// each CTA's TMEM receives its own 128 accumulator rows.  Loads per CTA per K-step: 16 + BN/2 x 128 B
// (32 KB at BN = 256), so more pipeline stages fit and the tensor pipe is fed from 2/3 of the bytes.
//   full[s]   leader CTA only: expects both CTAs' bytes (the peer's TMA signals it through the
//             cluster window, .cta_group::2);
//   empty[s], tfull[a]: in both CTAs, arrived by the leader's multicast tcgen05.commit;
//   tempty[a] leader CTA: 8 epilogue warps of each CTA arrive (the peer's remotely).
template <int BN>
struct Conv2Cfg {
    static constexpr int kA = 128 * 128, kBh = (BN / 2) * 128;
    static constexpr int kStageBytes = kA + kBh;
    static constexpr int kOutBufs = 4;
    static constexpr int kAvail = 232448 - kOutBufs * kOutStage - 2048;
    static constexpr int kStages = kAvail / kStageBytes > 10 ? 10 : kAvail / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + kOutBufs * kOutStage + 1024 + 512;
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kConv2Threads, 1)
    k_conv_tc2(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
               const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmG, const TcConv P,
               const __grid_constant__ CUtensorMap tmX) {
    using Cfg = Conv2Cfg<BN>;
    constexpr int S = Cfg::kStages;
    constexpr int ABYTES = Cfg::kA, BBYTES = Cfg::kBh;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;
    uint8_t *sB = smem + S * ABYTES;
    uint8_t *sO = sB + S * BBYTES;
    uint64_t *full = (uint64_t *)(sO + Cfg::kOutBufs * kOutStage);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint64_t *ebar = tempty + 2;                     // staging ring [4] + gdone [4] (store warp)
    uint32_t *tslot = (uint32_t *)(ebar + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { ptx::mbar_init(full + i, 1); ptx::mbar_init(empty + i, 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, 16); }
        for (int i = 0; i < 8; ++i) ptx::mbar_init(ebar + i, i < 4 ? 1 : 8);   // ring / gdone (8 epilogue warps)
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc2(tslot, 2 * BN);
    ptx::tc_fence_before();
    ptx::cluster_sync();     // both CTAs' barriers initialised, TMEM allocated
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail
    ptx::griddep_launch();
    const int num_tiles = P.m_tiles * P.n_tiles;   // = 2 x pairs (m_tiles rounded up to even)

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t full0 = ptx::mapa(ptx::smem_u32(full), 0);   // leader's full[0] (cluster window)
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int nt, tx, ty, b;
                P.decode(tile, nt, tx, ty, b);
                const int y0 = (P.out_a + ty * P.TH) * P.a_mul, x0 = tx * P.TW * P.a_mul;
                const int n0 = nt * BN + (int)rank * (BN / 2);
                for (int ks = 0; ks < P.k_steps; ++ks) {
                    const int tap = ks / P.cin_chunks, c = ks - tap * P.cin_chunks;
                    ptx::mbar_wait(empty + stage, phase ^ 1);
                    if (rank == 0) {
                        ptx::mbar_arrive_expect_tx(full + stage, 2 * (ABYTES + BBYTES));
                        ptx::tma_load_4d(sA + stage * ABYTES, &tmA, full + stage, c * 64, x0 + P.tap_ox[tap],
                                         y0 + P.tap_oy[tap] - P.in_base, b);
                        ptx::tma_load_3d(sB + stage * BBYTES, &tmB, full + stage, c * 64, P.tap_w[tap], n0);
                    } else {
                        const uint32_t fb = full0 + stage * 8;
                        ptx::tma_load_4d_2sm(sA + stage * ABYTES, &tmA, fb, c * 64, x0 + P.tap_ox[tap],
                                             y0 + P.tap_oy[tap] - P.in_base, b);
                        ptx::tma_load_3d_2sm(sB + stage * BBYTES, &tmB, fb, c * 64, P.tap_w[tap], n0);
                    }
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {   // whole warp of the leader CTA: tcgen05.mma.cta_group::2 / commit, elect.sync-issued
            constexpr uint32_t idesc = ptx::idesc_bf16(256, BN, 0, 0);
            const uint64_t dA = ptx::smem_desc(ptx::smem_u32(sA), 16, 1024, 2);
            const uint64_t dB = ptx::smem_desc(ptx::smem_u32(sB), 16, 1024, 2);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            int stage = 0, acc = 0;
            uint32_t phase = 0, aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int ks = 0; ks < P.k_steps; ++ks) {
                    ptx::mbar_wait(full + stage, phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = (uint32_t)dA + stage * (ABYTES >> 4);
                    const uint32_t b0 = (uint32_t)dB + stage * (BBYTES >> 4);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            ptx::umma2_bf16_1t(d, a0 + 2 * kk, hiA, b0 + 2 * kk, hiB, idesc, (ks | kk) != 0);
                        ptx::umma2_commit_mc_1t(empty + stage, 3);
                        if (ks + 1 == P.k_steps) ptx::umma2_commit_mc_1t(tfull + acc, 3);
                    }
                    __syncwarp();
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else if (warp == 10) {   // store warp: every TMA store and staging load of this CTA's epilogue
        if (lane == 0) {
            if (P.tma_out) conv_store_dma<BN, Cfg::kOutBufs>(P, &tmO, sO, &tmG, ebar, ebar + 4);
            else conv_store_dma_dg<BN, Cfg::kOutBufs / 2>(P, &tmO, &tmG, &tmX, sO, ebar, ebar + 4);
        }
    } else {
        static_assert(Conv2Cfg<BN>::kOutBufs == 4, "k_conv_tc2 store-warp epilogues: 4 staging buffers");
        if (P.tma_out)
            conv_epilogue_tma<BN, 8, Cfg::kOutBufs, true>(P, &tmO, tmem, tfull, tempty, sO, warp, lane, 2, &tmG, ebar, ebar + 4);
        else
            conv_epilogue_tma_dg2<BN, 8, Cfg::kOutBufs / 2, true>(P, &tmO, &tmG, tmem, tfull, tempty, sO, ebar, warp, lane, 2,
                                                                  &tmX, ebar + 4);
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();     // no CTA leaves while its peer may still signal its barriers
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc2(tmem, 2 * BN);
    }
}

// ------------------------------------------------------------------ small-channel conv FP (im2col in smem)
// Layers whose input has cin_p = 8 channels (the padded RGB image: conv1_1 of VGG-16, the 7x7/s2
// stem of ResNet-50).  The contraction index is K = tap x 8 channels; one pipeline stage holds
// 8 taps: row m of the 16 KB stage (SWIZZLE_128B, K-major) is output pixel m's 8 taps x 16 bytes.
// The input patch a tile reads ((TW-1)s+k x (TH-1)s+k pixels x 16 bytes, at most 16 KB) is ONE
// TMA box per tile (double-buffered; out-of-bounds rows/columns = the semi-closed zero padding,
// PAPER.md:235), and the 8 gather warps build the im2col stages from it with shared-memory
// copies (a quarter-warp moves 8 consecutive pixels of one tap: conflict-free 16-byte accesses).
// The weights viewed as [cout][k*k*8] are TMA-loaded once per CTA and stay resident.  Per
// 128-pixel tile this is ceil(k*k/2) MMAs of K=16 (5 for 3x3).
// Warps 0-7 gather, warp 8 TMEM + MMA issue, warp 9 patch TMA producer, warps 10-17 the
// TMA-store epilogue.
static constexpr int kI2cGather = 8;                          // gather warps
static constexpr int kI2cMmaWarp = kI2cGather;
static constexpr int kI2cPatchWarp = kI2cGather + 1;
static constexpr int kI2cEpi = 8;
static constexpr int kI2pThreads = (kI2cGather + 2 + kI2cEpi) * 32;        // k_conv_im2col
static constexpr int kI2cStages = 4;
static constexpr int kI2cStage = 128 * 128;
static constexpr int kI2cBMax = 64 * 1024;
static constexpr int kI2cPatch = 16 * 1024;                   // one input patch buffer (<= 1024 pixels)
static constexpr int kI2cSmem = kI2cStages * kI2cStage + kI2cBMax + 2 * kOutStage + 2 * kI2cPatch + 1024 + 256;

template <int BN>
__global__ void __launch_bounds__(kI2pThreads, 1)
    k_conv_im2col(const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmO,
                  const __grid_constant__ CUtensorMap tmP, const TcConv P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;
    uint8_t *sB = sA + kI2cStages * kI2cStage;
    uint8_t *sO = sB + kI2cBMax;
    uint8_t *sP = sO + 2 * kOutStage;
    uint64_t *full = (uint64_t *)(sP + 2 * kI2cPatch);
    uint64_t *empty = full + kI2cStages;
    uint64_t *tfull = empty + kI2cStages;
    uint64_t *tempty = tfull + 2;
    uint64_t *bfull = tempty + 2;
    uint64_t *pfull = bfull + 1;
    uint64_t *pempty = pfull + 2;
    uint32_t *tslot = (uint32_t *)(pempty + 2);
    const int KS = (P.ntaps + 7) / 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kI2cStages; ++i) {
            ptx::mbar_init(full + i, kI2cGather * 32);
            ptx::mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, kI2cEpi); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(pfull + i, 1); ptx::mbar_init(pempty + i, kI2cGather * 32); }
        ptx::mbar_init(bfull, 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmB);
        ptx::prefetch_tmap(&tmO);
        ptx::prefetch_tmap(&tmP);
    }
    if (warp == kI2cMmaWarp) ptx::tmem_alloc(tslot, 2 * BN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int num_tiles = P.m_tiles * P.n_tiles;

    if (warp < kI2cGather) {
        if (threadIdx.x == 0) {   // resident weights: n_tiles x KS boxes of BN rows x 64 K
            ptx::mbar_arrive_expect_tx(bfull, P.n_tiles * KS * BN * 128);
            for (int nt = 0; nt < P.n_tiles; ++nt)
                for (int ks = 0; ks < KS; ++ks)
                    ptx::tma_load_2d(sB + (nt * KS + ks) * BN * 128, &tmB, bfull, ks * 64, nt * BN);
        }
        // thread = (tap slot c, pixels m0 + 32 i): a quarter-warp covers 8 consecutive pixels of
        // one tap, so both the patch reads and the swizzled stage writes are conflict-free
        const int c = (threadIdx.x >> 3) & 7, m0 = (threadIdx.x & 7) + 8 * (threadIdx.x >> 6);
        const int twm = (1 << P.tw_log2) - 1;
        int poff[4];   // patch pixel index of this thread's 4 output pixels (tap (0,0) of the patch)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int m = m0 + 32 * i;
            poff[i] = (m >> P.tw_log2) * P.a_mul * P.pat_w + (m & twm) * P.a_mul;
        }
        const uint32_t a_base = ptx::smem_u32(sA), p_base = ptx::smem_u32(sP);
        int stage = 0, pb = 0;
        uint32_t phase = 0, pphase = 0;
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
            ptx::mbar_wait(pfull + pb, pphase);
            const uint32_t pbase = p_base + pb * kI2cPatch;
            for (int ks = 0; ks < KS; ++ks) {
                const int tap = ks * 8 + c;
                const bool tv = tap < P.ntaps && !(P.dbg & 4);
                const int toff = tv ? (P.tap_oy[tap] - P.pat_oy) * P.pat_w + P.tap_ox[tap] - P.pat_ox : 0;
                uint4 v[4];
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    v[i] = tv ? ld_shared_v4(pbase + (uint32_t)(poff[i] + toff) * 16u) : make_uint4(0, 0, 0, 0);
                ptx::mbar_wait(empty + stage, phase ^ 1);
                const uint32_t sa = a_base + stage * kI2cStage;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int m = m0 + 32 * i;
                    st_shared_v4(sa + m * 128 + ((c ^ (m & 7)) << 4), v[i]);
                }
                fence_async_smem();
                ptx::mbar_arrive(full + stage);
                if (++stage == kI2cStages) { stage = 0; phase ^= 1; }
            }
            ptx::mbar_arrive(pempty + pb);          // this thread is done with the patch
            if (++pb == 2) { pb = 0; pphase ^= 1; }
        }
    } else if (warp == kI2cPatchWarp) {
        if (lane == 0) {
            const uint32_t pbytes = (uint32_t)P.pat_w * P.pat_h * 16;
            int pb = 0;
            uint32_t pphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int nt, tx, ty, b;
                P.decode(tile, nt, tx, ty, b);
                ptx::mbar_wait(pempty + pb, pphase ^ 1);
                ptx::mbar_arrive_expect_tx(pfull + pb, pbytes);
                ptx::tma_load_4d(sP + pb * kI2cPatch, &tmP, pfull + pb, 0, tx * P.TW * P.a_mul + P.pat_ox,
                                 (P.out_a + ty * P.TH) * P.a_mul + P.pat_oy - P.in_base, b);
                if (++pb == 2) { pb = 0; pphase ^= 1; }
            }
        }
    } else if (warp == kI2cMmaWarp) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 0, 0);
            const uint64_t dA = ptx::smem_desc(ptx::smem_u32(sA), 16, 1024, 2);
            const uint64_t dB = ptx::smem_desc(ptx::smem_u32(sB), 16, 1024, 2);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            ptx::mbar_wait(bfull, 0);
            int stage = 0, acc = 0;
            uint32_t phase = 0, aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int nt = tile % P.n_tiles;
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int ks = 0; ks < KS; ++ks) {
                    ptx::mbar_wait(full + stage, phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = (uint32_t)dA + stage * (kI2cStage >> 4);
                    const uint32_t b0 = (uint32_t)dB + (nt * KS + ks) * (BN * 128 >> 4);
                    const int nk = min(8, P.ntaps - ks * 8);   // real taps in this stage
                    if (ptx::elect_one()) {
                        for (int kk = 0; kk < (nk + 1) / 2; ++kk)
                            ptx::umma_bf16_1t(d, a0 + 2 * kk, hiA, b0 + 2 * kk, hiB, idesc, (ks | kk) != 0);
                        ptx::umma_commit_1t(empty + stage);
                    }
                    __syncwarp();
                    if (++stage == kI2cStages) { stage = 0; phase ^= 1; }
                }
                if (ptx::elect_one()) ptx::umma_commit_1t(tfull + acc);
                __syncwarp();
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else {
        conv_epilogue_tma<BN, kI2cEpi>(P, &tmO, tmem, tfull, tempty, sO, warp, lane, kI2cPatchWarp + 1);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kI2cMmaWarp) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 2 * BN);
    }
}

// ------------------------------------------------------------------ small-channel conv FP: tap pairs
// 8-channel inputs (the padded RGB image) without any im2col copy.  An input pixel is 8 bf16 =
// 16 bytes = one K-chunk of a K-major no-swizzle UMMA operand, whose core matrix is 8 rows x 16 B
// at a 16 B row stride.  The tile is 8 output columns x 16 output rows; its input patch is TMA-
// loaded into smem as dense [row][pixel] planes, and the A operand of a K=16 MMA is the pair of
// taps (ky, kx) and (ky, kx+1), read straight out of the patch by a descriptor:
//   stride 1: one plane; tap kx of output column i is pixel i+kx, so the 8 output columns are 8
//             consecutive 16 B pixels (a core matrix) and the second tap of the pair is the same
//             matrix one pixel on (LBO = 16 B; the core matrices of the two K-halves overlap);
//   stride 2: two planes, the even- and odd-offset columns of the patch (two TMA loads with element
//             stride 2); tap kx = 2j (+1) of output column i is plane A (B) pixel i+j, so LBO =
//             plane B - plane A.
// Consecutive output rows (8-row core-matrix groups) are s patch rows apart (SBO).  Per tile:
// ceil(k/2)*k MMAs (6 for 3x3, 28 for the 7x7 stem; the odd tap of the last pair has zero
// weights), one patch box of at most 16 KB, no register traffic for the operand at all.  The
// weights [c_out][k][k][8] are TMA-loaded once per CTA as 1 KB chunks (64 rows x 16 B), the
// chunk of a pair's odd tap kx = k reads as zero (out-of-bounds).
static constexpr int kPrStages = 4;
static constexpr int kPrPatch = 16 * 1024;
static constexpr int kPrBMax = 7 * 4 * 2048;          // 7 rows x 4 pairs x 2 chunks x 1 KB
static constexpr int kPrOutBufs = 6;
static constexpr int kPrSmem = kPrStages * kPrPatch + kPrBMax + kPrOutBufs * kOutStage + 1024 + 256;

__global__ void __launch_bounds__(kConv2Threads, 1)
    k_conv_pair(const __grid_constant__ CUtensorMap tmP, const __grid_constant__ CUtensorMap tmW,
                const __grid_constant__ CUtensorMap tmO, const TcConv P) {
    constexpr int BN = 64;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sP = smem;
    uint8_t *sB = sP + kPrStages * kPrPatch;
    uint8_t *sO = sB + kPrBMax;
    uint64_t *full = (uint64_t *)(sO + kPrOutBufs * kOutStage);
    uint64_t *empty = full + kPrStages;
    uint64_t *tfull = empty + kPrStages;
    uint64_t *tempty = tfull + 2;
    uint64_t *bfull = tempty + 2;
    uint64_t *rbar = bfull + 1, *gdone = rbar + kPrOutBufs;   // store-warp ring: buffer free / combined
    uint32_t *tslot = (uint32_t *)(gdone + kPrOutBufs);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int KY = P.k, NPR = (P.k + 1) / 2, s = P.a_mul;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kPrStages; ++i) { ptx::mbar_init(full + i, 1); ptx::mbar_init(empty + i, 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, 8); }
        ptx::mbar_init(bfull, 1);
        for (int i = 0; i < kPrOutBufs; ++i) { ptx::mbar_init(rbar + i, 1); ptx::mbar_init(gdone + i, 8); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmP);
        ptx::prefetch_tmap(&tmW);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, 2 * BN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int num_tiles = P.m_tiles;
    const uint32_t plane = (uint32_t)P.pat_w * P.pat_h * 16;   // bytes of one plane
    const uint32_t pstride = (plane + 127) & ~127u;             // plane B offset (TMA: 128 B aligned)

    if (warp == 0) {
        if (lane == 0) {
            // weights: chunk (ky, pair j, half h) = tap (ky, 2j+h) for all 64 rows, 1 KB each
            ptx::mbar_arrive_expect_tx(bfull, KY * NPR * 2 * 1024);
            for (int ky = 0; ky < KY; ++ky)
                for (int j = 0; j < NPR; ++j)
                    for (int h = 0; h < 2; ++h)
                        ptx::tma_load_4d(sB + ((ky * NPR + j) * 2 + h) * 1024, &tmW, bfull, 0, 2 * j + h, ky, 0);
            int st = 0;
            uint32_t ph = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int nt, tx, ty, b;
                P.decode(tile, nt, tx, ty, b);
                const int xs = tx * 8 * s + P.pat_ox, ys = (P.out_a + ty * 16) * s + P.pat_oy - P.in_base;
                ptx::mbar_wait(empty + st, ph ^ 1);
                ptx::mbar_arrive_expect_tx(full + st, s * plane);
                ptx::tma_load_4d(sP + st * kPrPatch, &tmP, full + st, 0, xs, ys, b);
                if (s == 2) ptx::tma_load_4d(sP + st * kPrPatch + pstride, &tmP, full + st, 0, xs + 1, ys, b);
                if (++st == kPrStages) { st = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 0, 0);
            const uint32_t row = (uint32_t)P.pat_w * 16;                 // bytes per patch row (one plane)
            const uint32_t lbo = s == 1 ? 16u : pstride;
            const bool sw = P.dbg & 8;   // debug: exchange the LBO / SBO roles
            const uint64_t dA = sw ? ptx::smem_desc(ptx::smem_u32(sP), s * row, lbo, 0)
                                   : ptx::smem_desc(ptx::smem_u32(sP), lbo, s * row, 0);
            const uint64_t dB = sw ? ptx::smem_desc(ptx::smem_u32(sB), 128, 1024, 0)
                                   : ptx::smem_desc(ptx::smem_u32(sB), 1024, 128, 0);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            const uint32_t row16 = row >> 4, jstep = s == 1 ? 2u : 1u;
            ptx::mbar_wait(bfull, 0);
            int st = 0, acc = 0;
            uint32_t ph = 0, aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                ptx::mbar_wait(full + st, ph);
                ptx::tc_fence_after();
                // descriptors advance incrementally: first K-half of pair (ky, j) is tap kx = 2j ->
                // plane-A pixel i + (s == 1 ? 2j : j) of patch row ky; weights chunk pair (ky, j).
                // One elected lane issues the tile's k * ceil(k/2) MMAs (N = 64: 32 tensor cycles each).
                if (ptx::elect_one()) {
                    uint32_t aky = (uint32_t)dA + st * (kPrPatch >> 4), bt = (uint32_t)dB;
                    uint32_t acc_flag = 0;
                    for (int ky = 0; ky < KY; ++ky, aky += row16) {
                        uint32_t at = aky;
                        for (int j = 0; j < NPR; ++j, at += jstep, bt += 2048 >> 4) {
                            ptx::umma_bf16_1t(d, at, hiA, bt, hiB, idesc, acc_flag);
                            acc_flag = 1;
                        }
                    }
                    ptx::umma_commit_1t(empty + st);
                    ptx::umma_commit_1t(tfull + acc);
                }
                __syncwarp();
                if (++st == kPrStages) { st = 0; ph ^= 1; }
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else {
        if (warp == 10) {   // store warp
            if (lane == 0) conv_store_dma<BN, kPrOutBufs>(P, &tmO, sO, nullptr, rbar, gdone);
        } else {
            conv_epilogue_tma<BN, 8, kPrOutBufs, true>(P, &tmO, tmem, tfull, tempty, sO, warp, lane, 2, nullptr, rbar, gdone);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 2 * BN);
    }
}

// ------------------------------------------------------------------ conv FP / dgrad, halo reuse
// Stride-1 k x k convolutions: the output tile is 8 columns x 16 rows.  One TMA box of
// (8+k-1) x (16+k-1) input pixels x 64 channels (the tile plus its halo; row pitch 8+k-1
// pixels) is loaded once per input-channel chunk and serves all k*k taps: the A operand of
// tap (ky, kx) is the same smem box at a start offset of (pitch*ky + kx) pixel rows, with the
// 8-pixel core-matrix groups (tile rows) pitch*128 B apart (SBO).  The SWIZZLE_128B pattern is
// a function of the absolute smem address bits [7,10) on both the TMA write and the UMMA read,
// so a start at any 128-byte row (descriptor base offset 0) addresses the box consistently.
// A traffic drops from k*k boxes of 128 rows to one box of (7+k)(15+k) rows per chunk;
// weights stream per (chunk, tap).
template <int KH>
struct HaloGeom {
    static constexpr int kPitch = 8 + KH - 1, kRows = 16 + KH - 1;
    static constexpr int kABytes = ((kPitch * kRows * 128 + 1023) / 1024) * 1024;
};
template <int BN, int KH>
struct HaloCfg {
    static constexpr int kABytes = HaloGeom<KH>::kABytes;
    static constexpr int kBBytes = BN * 128;
    static constexpr int kSA = 4;
    static constexpr int kSB = (232448 - kSA * kABytes - 2 * kOutStage - 2048) / kBBytes > 16
                                   ? 16 : (232448 - kSA * kABytes - 2 * kOutStage - 2048) / kBBytes;
    static constexpr int kSmem = kSA * kABytes + kSB * kBBytes + 2 * kOutStage + 1024 + 512;
    static constexpr uint32_t kTmemCols = 2 * BN;
};

template <int BN, int KH>
__global__ void __launch_bounds__(kThreads, 1)
    k_conv_tc_halo(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO, const TcConv P) {
    using Cfg = HaloCfg<BN, KH>;
    constexpr int SA = Cfg::kSA, SB = Cfg::kSB;
    constexpr int HP = HaloGeom<KH>::kPitch;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;
    uint8_t *sB = smem + SA * Cfg::kABytes;
    uint8_t *sO = sB + SB * Cfg::kBBytes;
    uint64_t *fullA = (uint64_t *)(sO + 2 * kOutStage);
    uint64_t *emptyA = fullA + SA;
    uint64_t *fullB = emptyA + SA;
    uint64_t *emptyB = fullB + SB;
    uint64_t *tfull = emptyB + SB;
    uint64_t *tempty = tfull + 2;
    uint32_t *tslot = (uint32_t *)(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SA; ++i) { ptx::mbar_init(fullA + i, 1); ptx::mbar_init(emptyA + i, 1); }
        for (int i = 0; i < SB; ++i) { ptx::mbar_init(fullB + i, 1); ptx::mbar_init(emptyB + i, 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, 4); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, Cfg::kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int num_tiles = P.m_tiles * P.n_tiles;
    constexpr int taps = KH * KH;

    if (warp == 0) {
        if (lane == 0) {
            int sa = 0, sb = 0;
            uint32_t pa = 0, pb = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int nt, tx, ty, b;
                P.decode(tile, nt, tx, ty, b);
                const int y0 = P.out_a + ty * 16, x0 = tx * 8, n0 = nt * BN;
                for (int c = 0; c < P.cin_chunks; ++c) {
                    ptx::mbar_wait(emptyA + sa, pa ^ 1);
                    ptx::mbar_arrive_expect_tx(fullA + sa, HP * HaloGeom<KH>::kRows * 128);
                    ptx::tma_load_4d(sA + sa * Cfg::kABytes, &tmA, fullA + sa, c * 64, x0 - P.pad,
                                     y0 - P.pad - P.in_base, b);
                    if (++sa == SA) { sa = 0; pa ^= 1; }
                    for (int tap = 0; tap < taps; ++tap) {
                        ptx::mbar_wait(emptyB + sb, pb ^ 1);
                        ptx::mbar_arrive_expect_tx(fullB + sb, Cfg::kBBytes);
                        ptx::tma_load_3d(sB + sb * Cfg::kBBytes, &tmB, fullB + sb, c * 64, tap, n0);
                        if (++sb == SB) { sb = 0; pb ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 0, 0);
            const uint64_t dA = ptx::smem_desc_sw128_bo(ptx::smem_u32(sA), 16, HP * 128, 0);
            const uint64_t dB = ptx::smem_desc_sw128(ptx::smem_u32(sB), 16, 1024);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            int sa = 0, sb = 0, acc = 0;
            uint32_t pa = 0, pb = 0, aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                int first = 1;
                for (int c = 0; c < P.cin_chunks; ++c) {
                    ptx::mbar_wait(fullA + sa, pa);
                    ptx::tc_fence_after();
                    const uint32_t a0 = (uint32_t)dA + sa * (Cfg::kABytes >> 4);
#pragma unroll
                    for (int tap = 0; tap < taps; ++tap) {
                        const int ky = tap / KH, kx = tap - ky * KH;
                        ptx::mbar_wait(fullB + sb, pb);
                        ptx::tc_fence_after();
                        const uint32_t at = a0 + (uint32_t)(ky * HP + kx) * 8;
                        const uint32_t b0 = (uint32_t)dB + sb * (Cfg::kBBytes >> 4);
                        if (ptx::elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                ptx::umma_bf16_1t(d, at + 2 * kk, hiA, b0 + 2 * kk, hiB, idesc, (first && kk == 0) ? 0u : 1u);
                            ptx::umma_commit_1t(emptyB + sb);
                        }
                        __syncwarp();
                        first = 0;
                        if (++sb == SB) { sb = 0; pb ^= 1; }
                    }
                    ptx::umma_commit(emptyA + sa);
                    if (++sa == SA) { sa = 0; pa ^= 1; }
                }
                ptx::umma_commit(tfull + acc);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else if (P.tma_out) {
        conv_epilogue_tma<BN>(P, &tmO, tmem, tfull, tempty, sO, warp, lane);
    } else {
        conv_epilogue<BN>(P, tmem, tfull, tempty, warp, lane);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, Cfg::kTmemCols);
    }
}

// ------------------------------------------------------------------ conv FP / dgrad: CTA pairs + halo-reuse A
// Stride-1 3x3 layers with >= 128 output channels.  Shared-memory traffic per SM decides the rate
// here (TMA writes + UMMA operand reads share the 128 B/clk smem port): the CTA pair halves the
// weight bytes per SM, and the halo box ((8+2) x (16+2) pixels x 64 channels, loaded once per
// 64-channel chunk and read by all 9 taps at start offsets ky*10+kx, see k_conv_tc_halo) divides the
// activation bytes by ~6.  Per CTA per tap: 16 KB of weights (BN = 256) + 1/9 of a 23 KB box.
template <int BN>
struct Conv2HCfg {
    static constexpr int kABytes = HaloGeom<3>::kABytes;          // 23 KB halo box
    static constexpr int kBh = (BN / 2) * 128;
    static constexpr int kSA = 3;
    static constexpr int kOutBufs = BN <= 128 ? 4 : 2;
    static constexpr int kAvail = 232448 - kSA * kABytes - kOutBufs * kOutStage - 2048;
    static constexpr int kSB = kAvail / kBh > 12 ? 12 : kAvail / kBh;
    static constexpr int kSmem = kSA * kABytes + kSB * kBh + kOutBufs * kOutStage + 1024 + 512;
};

template <int BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kConv2Threads, 1)
    k_conv_tc2h(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmG, const TcConv P) {
    using Cfg = Conv2HCfg<BN>;
    constexpr int SA = Cfg::kSA, SB = Cfg::kSB, AB = Cfg::kABytes, BB = Cfg::kBh;
    constexpr int KH = 3, HP = HaloGeom<KH>::kPitch, taps = 9;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;
    uint8_t *sB = sA + SA * AB;
    uint8_t *sO = sB + SB * BB;
    uint64_t *fullA = (uint64_t *)(sO + Cfg::kOutBufs * kOutStage);
    uint64_t *emptyA = fullA + SA;
    uint64_t *fullB = emptyA + SA;
    uint64_t *emptyB = fullB + SB;
    uint64_t *tfull = emptyB + SB;
    uint64_t *tempty = tfull + 2;
    uint64_t *ebar = tempty + 2;                     // staging ring [4] + gdone [4] (store warp)
    uint32_t *tslot = (uint32_t *)(ebar + 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = ptx::cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int i = 0; i < SA; ++i) { ptx::mbar_init(fullA + i, 1); ptx::mbar_init(emptyA + i, 1); }
        for (int i = 0; i < SB; ++i) { ptx::mbar_init(fullB + i, 1); ptx::mbar_init(emptyB + i, 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, 16); }
        for (int i = 0; i < 8; ++i) ptx::mbar_init(ebar + i, i < 4 ? 1 : 8);   // ring / gdone (8 epilogue warps)
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc2(tslot, 2 * BN);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int num_tiles = P.m_tiles * P.n_tiles;

    if (warp == 0) {
        if (lane == 0) {
            const uint32_t fullA0 = ptx::mapa(ptx::smem_u32(fullA), 0), fullB0 = ptx::mapa(ptx::smem_u32(fullB), 0);
            constexpr uint32_t abytes = HP * HaloGeom<KH>::kRows * 128;
            int sa = 0, sb = 0;
            uint32_t pa = 0, pb = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int nt, tx, ty, b;
                P.decode(tile, nt, tx, ty, b);
                const int y0 = P.out_a + ty * 16, x0 = tx * 8, n0 = nt * BN + (int)rank * (BN / 2);
                for (int c = 0; c < P.cin_chunks; ++c) {
                    ptx::mbar_wait(emptyA + sa, pa ^ 1);
                    if (rank == 0) {
                        ptx::mbar_arrive_expect_tx(fullA + sa, 2 * abytes);
                        ptx::tma_load_4d(sA + sa * AB, &tmA, fullA + sa, c * 64, x0 - P.pad, y0 - P.pad - P.in_base, b);
                    } else {
                        ptx::tma_load_4d_2sm(sA + sa * AB, &tmA, fullA0 + sa * 8, c * 64, x0 - P.pad,
                                             y0 - P.pad - P.in_base, b);
                    }
                    if (++sa == SA) { sa = 0; pa ^= 1; }
                    for (int tap = 0; tap < taps; ++tap) {
                        ptx::mbar_wait(emptyB + sb, pb ^ 1);
                        if (rank == 0) {
                            ptx::mbar_arrive_expect_tx(fullB + sb, 2 * BB);
                            ptx::tma_load_3d(sB + sb * BB, &tmB, fullB + sb, c * 64, tap, n0);
                        } else {
                            ptx::tma_load_3d_2sm(sB + sb * BB, &tmB, fullB0 + sb * 8, c * 64, tap, n0);
                        }
                        if (++sb == SB) { sb = 0; pb ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (rank == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16(256, BN, 0, 0);
            const uint64_t dA = ptx::smem_desc_sw128_bo(ptx::smem_u32(sA), 16, HP * 128, 0);
            const uint64_t dB = ptx::smem_desc_sw128(ptx::smem_u32(sB), 16, 1024);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            int sa = 0, sb = 0, acc = 0;
            uint32_t pa = 0, pb = 0, aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                int first = 1;
                for (int c = 0; c < P.cin_chunks; ++c) {
                    ptx::mbar_wait(fullA + sa, pa);
                    ptx::tc_fence_after();
                    const uint32_t a0 = (uint32_t)dA + sa * (AB >> 4);
#pragma unroll
                    for (int tap = 0; tap < taps; ++tap) {
                        const int ky = tap / KH, kx = tap - ky * KH;
                        ptx::mbar_wait(fullB + sb, pb);
                        ptx::tc_fence_after();
                        const uint32_t at = a0 + (uint32_t)(ky * HP + kx) * 8;
                        const uint32_t b0 = (uint32_t)dB + sb * (BB >> 4);
                        if (ptx::elect_one()) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk)
                                ptx::umma2_bf16_1t(d, at + 2 * kk, hiA, b0 + 2 * kk, hiB, idesc, (first && kk == 0) ? 0u : 1u);
                            ptx::umma2_commit_mc_1t(emptyB + sb, 3);
                        }
                        __syncwarp();
                        first = 0;
                        if (++sb == SB) { sb = 0; pb ^= 1; }
                    }
                    ptx::umma2_commit_mc(emptyA + sa, 3);
                    if (++sa == SA) { sa = 0; pa ^= 1; }
                }
                ptx::umma2_commit_mc(tfull + acc, 3);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else {
        if (warp == 10) {   // store warp: every TMA store and staging load of this CTA's epilogue
            if (lane == 0) {
                if (P.tma_out) conv_store_dma<BN, Cfg::kOutBufs>(P, &tmO, sO, &tmG, ebar, ebar + 4);
                else conv_store_dma_dg<BN, Cfg::kOutBufs / 2>(P, &tmO, &tmG, nullptr, sO, ebar, ebar + 4);
            }
        } else if (P.tma_out) {
            conv_epilogue_tma<BN, 8, Cfg::kOutBufs, true>(P, &tmO, tmem, tfull, tempty, sO, warp, lane, 2, &tmG, ebar, ebar + 4);
        } else {
            conv_epilogue_tma_dg2<BN, 8, Cfg::kOutBufs / 2, true>(P, &tmO, &tmG, tmem, tfull, tempty, sO, ebar, warp, lane, 2,
                                                                  nullptr, ebar + 4);
        }
    }
    ptx::tc_fence_before();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc2(tmem, 2 * BN);
    }
}

// ------------------------------------------------------------------ wgrad
// M = 128 output channels (two 64-channel MN-major boxes of the band delta),
// N = BN input channels (BN/64 MN-major boxes of the shifted band input),
// K = 128 band pixels per stage (8 MMAs of K=16).  Work item = (co tile, tap, ci tile,
// pixel split); fp32 partial sums are added with red.global into the flat gradient.
static constexpr int kWgA = 2 * kABytes;
// fp32 gradient reduction (no "memory" clobber: the gradient buffer is only ever reduced into
// here, so surrounding loads of weights / activations may be scheduled across it)
__device__ __forceinline__ void red_add_v4(float *p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d));
}

// Bias-sum warps (128 threads): thread t sums output-channel PAIR cp = t % np (one 32-bit load per
// row of the SWIZZLE_128B delta tile, 64-channel boxes kABytes apart) over the rows r0 + step * (g +
// ngroups * j), g = t / np: half the loads of a column-per-thread sum and twice the parallelism.
__device__ __forceinline__ float2 db_pair_sum(uint32_t base, int cp, int g, int ngroups, int r0, int step, int rows = 128) {
    const uint32_t box = (uint32_t)(cp >> 5) * (uint32_t)(rows * 128), chunk = (uint32_t)((cp & 31) >> 2), cofs = (uint32_t)((cp & 3) * 4);
    float a[2] = {0.f, 0.f}, b[2] = {0.f, 0.f};
    int i = 0;
#pragma unroll 4
    for (int r = r0 + step * g; r < rows; r += step * ngroups, ++i) {
        uint32_t w;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(base + box + r * 128 + ((chunk ^ (r & 7)) << 4) + cofs));
        a[i & 1] += bf_lo(w);
        b[i & 1] += bf_hi(w);
    }
    return make_float2(a[0] + a[1], b[0] + b[1]);
}

// KP = pixels per pipeline stage (the K of one stage): 128, or 64 for N = 256 items, whose 96 KB
// stages would leave only two in the ring (one load in flight while the other is consumed: the
// tensor pipe starved at ~35 %); 64-pixel stages keep three loads in flight.
template <int BN, int KP = 128>
struct WgCfg {
    // B operand (shifted band input): BN/KB boxes of KB channels (KB = 64, SWIZZLE_128B; or
    // KB = BN = 16, SWIZZLE_32B for small-channel inputs)
    static constexpr int KB = BN < 64 ? BN : 64;
    static constexpr int kA = 2 * KP * 128;                  // delta: two 64-channel MN chunks
    static constexpr int kBBox = KP * KB * 2;
    static constexpr int kStageBytes = kA + (BN / KB) * kBBox;
    static constexpr int kStages = (192 * 1024) / kStageBytes > 12 ? 12 : (192 * 1024) / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
    static constexpr uint32_t kTmemCols = 2 * BN;
};

template <int BN, int KP = 128>
__global__ void __launch_bounds__(kWgThreads, 1)
    k_wgrad_tc(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX, const TcWgrad P) {
    using Cfg = WgCfg<BN, KP>;
    constexpr int S = Cfg::kStages;
    constexpr int SB = Cfg::kStageBytes;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + S * SB);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint32_t *tslot = (uint32_t *)(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { ptx::mbar_init(full + i, 1); ptx::mbar_init(empty + i, P.db ? 5 : 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, 4); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmD);
        ptx::prefetch_tmap(&tmX);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, Cfg::kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int taps = P.k * P.k;

    auto decode = [&](int item, int &cot, int &tap, int &cit, int &split) {
        split = item % P.splits;
        int r = item / P.splits;
        cit = r % P.ci_tiles; r /= P.ci_tiles;
        tap = r % taps;
        cot = r / taps;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                int cot, tap, cit, split;
                decode(item, cot, tap, cit, split);
                const int ky = tap / P.k, kx = tap - ky * P.k;
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                for (int pt = p0; pt < p1; ++pt) {
                    const int tx = pt % P.tiles_x, r = pt / P.tiles_x, ty = r % P.tiles_y;
                    const int b = (r / P.tiles_y) * (P.NB > 1 ? P.NB : 1);
                    const int y0 = P.out_a + ty * P.TH, x0 = tx * P.TW;
                    ptx::mbar_wait(empty + stage, phase ^ 1);
                    uint8_t *st = smem + stage * SB;
                    ptx::mbar_arrive_expect_tx(full + stage, SB);
                    ptx::tma_load_4d(st, &tmD, full + stage, cot * 128, x0, y0 - P.dy_base, b);
                    ptx::tma_load_4d(st + Cfg::kA / 2, &tmD, full + stage, cot * 128 + 64, x0, y0 - P.dy_base, b);
#pragma unroll
                    for (int h = 0; h < BN / Cfg::KB; ++h)
                        ptx::tma_load_4d(st + Cfg::kA + h * Cfg::kBBox, &tmX, full + stage, cit * BN + h * Cfg::KB,
                                         x0 * P.s - P.pad + kx, y0 * P.s - P.pad + ky - P.x_base, b);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 1, 1);
            const uint64_t dA = ptx::smem_desc_sw128(ptx::smem_u32(smem), Cfg::kA / 2, 1024);
            const uint64_t dB = Cfg::KB == 64 ? ptx::smem_desc_sw128(ptx::smem_u32(smem + Cfg::kA), Cfg::kBBox, 1024)
                                              : ptx::smem_desc(ptx::smem_u32(smem + Cfg::kA), 4096, 8 * Cfg::KB * 2, 6);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            int stage = 0, acc = 0;
            uint32_t phase = 0, aphase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                int cot, tap, cit, split;
                decode(item, cot, tap, cit, split);
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int pt = p0; pt < p1; ++pt) {
                    ptx::mbar_wait(full + stage, phase);
                    ptx::tc_fence_after();
                    // MN-major SW128: 64-element MN chunks LBO = 16 KB apart, 8-row K groups SBO = 1 KB
                    const uint32_t a0 = (uint32_t)dA + stage * (SB >> 4);
                    const uint32_t b0 = (uint32_t)dB + stage * (SB >> 4);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < KP / 16; ++kk)
                            ptx::umma_bf16_1t(d, a0 + kk * 128, hiA, b0 + kk * (Cfg::KB == 64 ? 128 : 2 * Cfg::KB), hiB, idesc,
                                              (pt != p0 || kk != 0) ? 1u : 0u);
                        ptx::umma_commit_1t(empty + stage);
                    }
                    __syncwarp();
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                ptx::umma_commit(tfull + acc);
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else if (warp < 6) {
        const int ew = warp & 3;
        const int m = ew * 32 + lane;
        int acc = 0;
        uint32_t aphase = 0;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            int cot, tap, cit, split;
            decode(item, cot, tap, cit, split);
            const int co = cot * 128 + m;
            const float gsc = (P.gamma && co < P.c_out) ? __bfloat162float(P.gamma[co]) : 1.f;
            float *dst = P.dw + ((long long)co * taps + tap) * P.cin_p;
            const bf16 *wrow = P.w + ((long long)co * taps + tap) * P.cin_p;
            float gdot = 0.f;
            ptx::mbar_wait(tfull + acc, aphase);
            ptx::tc_fence_after();
            if constexpr (BN < 32) {
                uint32_t v[16];
                ptx::tmem_ld16(tmem + ((uint32_t)(ew * 32) << 16) + acc * BN, v);
                ptx::tmem_ld_wait();
                if (co < P.c_out) {
                    const int ci0 = cit * BN;
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (ci0 + j < P.cin_p) {
                            atomicAdd(dst + ci0 + j, __uint_as_float(v[j]) * gsc);
                            if (P.dg) gdot += __uint_as_float(v[j]) * __bfloat162float(wrow[ci0 + j]);
                        }
                }
            } else {
                // this thread's row co: 32 consecutive input channels per TMEM load, added with
                // 16-byte vector reductions (cin_p % 8 == 0, so a 4-group is all in or all out).  The
                // pixel splits of one (co, tap, ci) tile finish together and reduce into the same
                // addresses: each split starts at a different 32-channel chunk so that their
                // reductions do not queue on the same L2 lines
#pragma unroll 1
                for (int cc = 0; cc < BN / 32; ++cc) {
                    const int c = (cc + split) % (BN / 32);
                    uint32_t v[32];
                    ptx::tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + acc * BN + c * 32, v);
                    const int ci0 = cit * BN + c * 32;
                    uint4 wq[4];   // dgamma: this row's 32 weights, loaded while the TMEM load completes
                    if (P.dg && co < P.c_out) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            wq[j] = ci0 + 8 * j < P.cin_p ? *reinterpret_cast<const uint4 *>(wrow + ci0 + 8 * j)
                                                          : make_uint4(0, 0, 0, 0);
                    }
                    ptx::tmem_ld_wait();
                    if (co >= P.c_out) continue;
#pragma unroll
                    for (int j = 0; j < 32; j += 8) {
                        if (ci0 + j >= P.cin_p) break;
                        red_add_v4(dst + ci0 + j, __uint_as_float(v[j]) * gsc, __uint_as_float(v[j + 1]) * gsc,
                                   __uint_as_float(v[j + 2]) * gsc, __uint_as_float(v[j + 3]) * gsc);
                        red_add_v4(dst + ci0 + j + 4, __uint_as_float(v[j + 4]) * gsc, __uint_as_float(v[j + 5]) * gsc,
                                   __uint_as_float(v[j + 6]) * gsc, __uint_as_float(v[j + 7]) * gsc);
                        if (P.dg) {
                            const uint4 wv = wq[j / 8];
                            const uint32_t ww[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
                            for (int h = 0; h < 4; ++h)
                                gdot += __uint_as_float(v[j + 2 * h]) * bf_lo(ww[h]) + __uint_as_float(v[j + 2 * h + 1]) * bf_hi(ww[h]);
                        }
                    }
                }
            }
            if (P.dg && co < P.c_out) atomicAdd(P.dg + co, gdot);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty + acc);
            if (++acc == 2) { acc = 0; aphase ^= 1; }
        }
    } else if (P.db) {
        // warps 6..9: the fused bias / beta gradient (delta column sums) on their own warps, so the
        // epilogue warps never gate the pipeline stages of the next item
        const int t = (warp - 6) * 32 + lane, cp = t % 64, g = t / 64;
        int stage = 0;
        uint32_t phase = 0;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            int cot, tap, cit, split;
            decode(item, cot, tap, cit, split);
            const int nparts = taps * P.ci_tiles, part = tap * P.ci_tiles + cit;
            const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
            float2 sum = make_float2(0.f, 0.f);
            for (int pt = p0; pt < p1; ++pt) {
                ptx::mbar_wait(full + stage, phase);
                const float2 v = db_pair_sum(ptx::smem_u32(smem + stage * SB), cp, g, 2, part, nparts, KP);
                sum.x += v.x;
                sum.y += v.y;
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(empty + stage);
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
            const int co = cot * 128 + 2 * cp;
            if (co < P.c_out) atomicAdd(P.db + co, sum.x);
            if (co + 1 < P.c_out) atomicAdd(P.db + co + 1, sum.y);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, Cfg::kTmemCols);
    }
}

// ------------------------------------------------------------------ fused 1x1 dgrad + wgrad
// The backward of a pointwise (1x1, stride 1) convolution in one pass over the band: every 128-pixel
// tile of delta(out) [CO channels] and of the conv input x [CI channels] is TMA-loaded ONCE and
// feeds two contractions from the same shared-memory bytes:
//   dgrad   D1[px][ci] = sum_co delta[px][co] W'[ci][co]   (delta tile as the K-major A operand)
//   wgrad   D2[co][ci] += sum_px delta[px][co] x[px][ci]   (delta / x tiles as MN-major A / B)
// D1 goes through the dgrad epilogue (gate-on-write from the x tile already in shared memory, the
// old delta or the fused residual addend TMA-loaded, TMA store); D2 stays in TMEM over the CTA's
// contiguous run of tiles and is reduced into the fp32 gradient once at the end (scaled by gamma,
// with dgamma = sum_ci W * D2 and the beta / bias column sums from dedicated warps).  Separately,
// dgrad and wgrad each stream delta(out) and x from HBM; here the wgrad reads nothing extra.
// (CI, CO) = (64, 256) -- the bottleneck's last 1x1 / the projection -- or (256, 64) -- its first 1x1.
struct TcDw {
    View dx, act, add;           // delta_in (output), gating activation (== x), fused residual addend
    float *dw, *db, *dg;
    const bf16 *gamma, *w;
    int c_out, gate, write, dg_add;
    int TW, TH, tiles_x, tiles_y, pix_tiles, per_cta;
    int out_a, dy_base, x_base, B, tw_log2, th_log2;
};

template <int CI, int CO>
struct DwCfg {
    static constexpr int kDB = CO / 64, kXB = CI / 64;          // 64-channel boxes per tile
    static constexpr int kStageBytes = (kDB + kXB) * kABytes;    // 80 KB
    static constexpr int kStages = 2;
    static constexpr int kWBytes = CI * CO * 2;                  // W' [CI][CO], resident
    static constexpr int kSmem = kStages * kStageBytes + kWBytes + 2 * kOutStage + 1024 + 512;
    static constexpr int kD1Bufs = CI <= 64 ? 2 : 1;
    static constexpr int kMT = CO >= 128 ? CO / 128 : 1;         // wgrad M tiles (128 output channels)
    static constexpr uint32_t kD2Col = kD1Bufs * CI;
    static constexpr uint32_t kTmemCols = kD2Col + kMT * CI <= 256 ? 256 : 512;
};
static constexpr int kDwThreads = 480;   // producer, MMA, 8 epilogue warps, 4 bias-sum warps, store warp

template <int CI, int CO>
__global__ void __launch_bounds__(kDwThreads, 1)
    k_dwgrad_pw(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX,
                const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmO,
                const __grid_constant__ CUtensorMap tmA, const TcDw P) {
    using Cfg = DwCfg<CI, CO>;
    constexpr int S = Cfg::kStages, SB = Cfg::kStageBytes, D1B = Cfg::kD1Bufs;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sW = smem + S * SB;
    uint8_t *sO = sW + Cfg::kWBytes;                 // 2 x 16 KB epilogue staging
    uint64_t *full = (uint64_t *)(sO + 2 * kOutStage);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 2;
    uint64_t *ebar = tempty + 2;                     // epilogue staging loads (2)
    uint64_t *wbar = ebar + 2;
    uint64_t *d2full = wbar + 1;
    uint64_t *gdone = d2full + 1;                    // staging buffer combined (8 epilogue warps) -> store warp
    uint32_t *tslot = (uint32_t *)(gdone + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool bias = P.db != nullptr;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { ptx::mbar_init(full + i, 1); ptx::mbar_init(empty + i, 1 + 8 + (bias ? 4 : 0)); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, 8); ptx::mbar_init(ebar + i, 1); }
        ptx::mbar_init(wbar, 1);
        ptx::mbar_init(d2full, 1);
        for (int i = 0; i < 2; ++i) ptx::mbar_init(gdone + i, 8);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmD);
        ptx::prefetch_tmap(&tmX);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, Cfg::kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();
    ptx::griddep_launch();
    const int p0 = blockIdx.x * P.per_cta, p1 = min(p0 + P.per_cta, P.pix_tiles);
    auto tile_xy = [&](int pt, int &x0, int &y0, int &b) {
        const int tx = pt % P.tiles_x, r = pt / P.tiles_x, ty = r % P.tiles_y;
        b = r / P.tiles_y;
        x0 = tx * P.TW;
        y0 = P.out_a + ty * P.TH;
    };

    if (warp == 0) {
        if (lane == 0 && p0 < p1) {
            ptx::mbar_arrive_expect_tx(wbar, Cfg::kWBytes);
#pragma unroll
            for (int kc = 0; kc < Cfg::kDB; ++kc) ptx::tma_load_3d(sW + kc * CI * 128, &tmW, wbar, kc * 64, 0, 0);
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = p0; pt < p1; ++pt) {
                int x0, y0, b;
                tile_xy(pt, x0, y0, b);
                ptx::mbar_wait(empty + stage, phase ^ 1);
                uint8_t *st = smem + stage * SB;
                ptx::mbar_arrive_expect_tx(full + stage, SB);
#pragma unroll
                for (int kd = 0; kd < Cfg::kDB; ++kd)
                    ptx::tma_load_4d(st + kd * kABytes, &tmD, full + stage, kd * 64, x0, y0 - P.dy_base, b);
#pragma unroll
                for (int kx = 0; kx < Cfg::kXB; ++kx)
                    ptx::tma_load_4d(st + (Cfg::kDB + kx) * kABytes, &tmX, full + stage, kx * 64, x0, y0 - P.x_base, b);
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (p0 < p1) {
            constexpr uint32_t idg = ptx::idesc_bf16(128, CI, 0, 0), iwg = ptx::idesc_bf16(128, CI, 1, 1);
            const uint64_t dK = ptx::smem_desc_sw128(ptx::smem_u32(smem), 16, 1024);        // K-major delta
            const uint64_t dW = ptx::smem_desc_sw128(ptx::smem_u32(sW), 16, 1024);          // K-major W'
            // MN-major: 64-element MN chunks 16 KB apart (delta: M = co; x: N = ci); CO = 64 has one
            // chunk, so its second M chunk aliases the first (D2 rows 64..127 are never read)
            const uint64_t dM = ptx::smem_desc_sw128(ptx::smem_u32(smem), CO >= 128 ? kABytes : 0, 1024);
            const uint64_t dX = ptx::smem_desc_sw128(ptx::smem_u32(smem + Cfg::kDB * kABytes), kABytes, 1024);
            const uint32_t hK = (uint32_t)(dK >> 32), hW = (uint32_t)(dW >> 32), hM = (uint32_t)(dM >> 32),
                           hX = (uint32_t)(dX >> 32);
            ptx::mbar_wait(wbar, 0);
            ptx::tc_fence_after();
            int stage = 0, acc = 0;
            uint32_t phase = 0, aphase = 0;
            for (int pt = p0; pt < p1; ++pt) {
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::mbar_wait(full + stage, phase);
                ptx::tc_fence_after();
                const uint32_t so = stage * (SB >> 4);
                const uint32_t d1 = tmem + acc * CI;
                if (ptx::elect_one()) {
#pragma unroll
                    for (int kc = 0; kc < Cfg::kDB; ++kc)
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            ptx::umma_bf16_1t(d1, (uint32_t)dK + so + kc * (kABytes >> 4) + 2 * kk, hK,
                                              (uint32_t)dW + kc * (CI * 128 >> 4) + 2 * kk, hW, idg, (kc | kk) != 0);
#pragma unroll
                    for (int mt = 0; mt < Cfg::kMT; ++mt)
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            ptx::umma_bf16_1t(tmem + Cfg::kD2Col + mt * CI, (uint32_t)dM + so + mt * 2 * (kABytes >> 4) + kk * 128,
                                              hM, (uint32_t)dX + so + kk * 128, hX, iwg, (pt != p0 || kk != 0) ? 1u : 0u);
                    ptx::umma_commit_1t(empty + stage);
                    ptx::umma_commit_1t(tfull + acc);
                }
                __syncwarp();
                if (++stage == S) { stage = 0; phase ^= 1; }
                if (++acc == D1B) { acc = 0; aphase ^= 1; }
            }
            ptx::umma_commit(d2full);
        }
    } else if (warp < 10) {
        // dgrad epilogue: 8 warps, warp (q, hh) = pixels 32q.. of the tile, channels hh*32 .. +32 of
        // each 64-channel group; the gate is the x tile of the same stage (already in smem)
        const int q = warp & 3, hh = (warp - 2) >> 2, m = q * 32 + lane;
        const bool leader = warp == 2 && lane == 0;
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
        const bool dload = !P.write || P.dg_add;
        const CUtensorMap *tmL = P.write ? &tmA : &tmO;
        const int lbase = P.write ? P.add.base : P.dx.base;
        int stage = 0, acc = 0, sb = 0;
        uint32_t phase = 0, aphase = 0, ephase = 0;
        // item = (tile, 64-channel group); the old delta / addend of item j + 1 is TMA-loaded into the
        // other staging buffer (once item j - 1's store has read it) while item j is combined
        auto issue = [&](int pt2, int g2, int buf) {
            int x2, y2, b2;
            tile_xy(pt2, x2, y2, b2);
            ptx::mbar_arrive_expect_tx(ebar + buf, dload ? (uint32_t)kOutStage : 0u);
            if (dload) ptx::tma_load_4d(sO + buf * kOutStage, tmL, ebar + buf, g2 * 64, x2, y2 - lbase, b2);
        };
        (void)leader;
        for (int pt = p0; pt < p1; ++pt) {
            int x0, y0, b;
            tile_xy(pt, x0, y0, b);
            ptx::mbar_wait(tfull + acc, aphase);
            ptx::tc_fence_after();
            const uint32_t xs = ptx::smem_u32(smem + stage * SB + Cfg::kDB * kABytes);
#pragma unroll 1
            for (int g = 0; g < Cfg::kXB; ++g) {
                uint32_t v[32];
                ptx::tmem_ld32(tq + acc * CI + g * 64 + hh * 32, v);
                ptx::tmem_ld_wait();
                ptx::mbar_wait(ebar + sb, (ephase >> sb) & 1);
                ephase ^= 1u << sb;
                const uint32_t row = ptx::smem_u32(sO + sb * kOutStage) + m * 128;
                const uint32_t grow = xs + g * kABytes + m * 128;
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const int c = hh * 4 + cc;
                    const uint32_t off = (uint32_t)((c ^ (m & 7)) << 4);
                    const uint4 dd = dload ? ld_shared_v4(row + off) : make_uint4(0, 0, 0, 0);
                    const uint4 gg = P.gate ? ld_shared_v4(grow + off) : make_uint4(0, 0, 0, 0);
                    const uint32_t dw4[4] = {dd.x, dd.y, dd.z, dd.w}, gw4[4] = {gg.x, gg.y, gg.z, gg.w};
                    uint32_t o[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        const float f0 = hadd_lo(dw4[h], __uint_as_float(v[cc * 8 + 2 * h]));
                        const float f1 = hadd_hi(dw4[h], __uint_as_float(v[cc * 8 + 2 * h + 1]));
                        o[h] = pack2_act<false>(f0, f1);
                        if (P.gate) o[h] &= relu_mask2(gw4[h]);
                    }
                    st_shared_v4(row + off, make_uint4(o[0], o[1], o[2], o[3]));
                }
                fence_async_smem();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(gdone + sb);   // the store warp takes the buffer from here
                sb ^= 1;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) { ptx::mbar_arrive(empty + stage); ptx::mbar_arrive(tempty + acc); }
            if (++stage == S) { stage = 0; phase ^= 1; }
            if (++acc == D1B) { acc = 0; aphase ^= 1; }
        }
        // the wgrad accumulator of this CTA's tiles: reduced once into the fp32 gradient
        if (p0 < p1) {
            ptx::mbar_wait(d2full, 0);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int mt = 0; mt < Cfg::kMT; ++mt) {
                const int co = mt * 128 + m;
                const bool live = co < P.c_out && (CO >= 128 || m < 64);
                const float gsc = live && P.gamma ? __bfloat162float(P.gamma[co]) : 1.f;
                float gdot = 0.f;
#pragma unroll 1
                for (int cc = 0; cc < CI / 64; ++cc) {
                    const int c = (cc + blockIdx.x) % (CI / 64);   // rotated: CTAs do not queue on the same lines
                    uint32_t v[32];
                    ptx::tmem_ld32(tq + Cfg::kD2Col + mt * CI + c * 64 + hh * 32, v);
                    ptx::tmem_ld_wait();
                    if (!live) continue;
                    const int ci0 = c * 64 + hh * 32;
                    float *dst = P.dw + (long long)co * CI + ci0;
                    const bf16 *wr = P.w + (long long)co * CI + ci0;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        red_add_v4(dst + j, __uint_as_float(v[j]) * gsc, __uint_as_float(v[j + 1]) * gsc,
                                   __uint_as_float(v[j + 2]) * gsc, __uint_as_float(v[j + 3]) * gsc);
                        if (P.dg)
#pragma unroll
                            for (int h = 0; h < 4; ++h) gdot += __uint_as_float(v[j + h]) * __bfloat162float(wr[j + h]);
                    }
                }
                if (P.dg && live) atomicAdd(P.dg + co, gdot);
            }
        }
    } else if (warp == 14) {
        // store warp: item k = (tile, 64-channel group) of this CTA's run uses staging buffer k % 2; the
        // old delta / the residual addend of item k is TMA-loaded into it, the 8 epilogue warps combine it
        // (gdone), the TMA store follows and, once it has read the buffer, item k + 2 is loaded
        if (lane == 0) {
            const bool dload = !P.write || P.dg_add;
            const CUtensorMap *tmL = P.write ? &tmA : &tmO;
            const int lbase = P.write ? P.add.base : P.dx.base;
            int lpt = p0, lg = 0;   // next item to load
            auto issue = [&](int buf) {
                if (lpt >= p1) return;
                int x2, y2, b2;
                tile_xy(lpt, x2, y2, b2);
                ptx::mbar_arrive_expect_tx(ebar + buf, dload ? (uint32_t)kOutStage : 0u);
                if (dload) ptx::tma_load_4d(sO + buf * kOutStage, tmL, ebar + buf, lg * 64, x2, y2 - lbase, b2);
                if (++lg == Cfg::kXB) { lg = 0; ++lpt; }
            };
            issue(0);
            issue(1);
            int sb = 0;
            uint32_t gph = 0;
            for (int pt = p0; pt < p1; ++pt) {
                int x0, y0, b;
                tile_xy(pt, x0, y0, b);
                for (int g = 0; g < Cfg::kXB; ++g) {
                    ptx::mbar_wait(gdone + sb, (gph >> sb) & 1);
                    gph ^= 1u << sb;
                    tma_store_4d(&tmO, sO + sb * kOutStage, g * 64, x0, y0 - P.dx.base, b);
                    bulk_commit();
                    bulk_wait_read0();
                    issue(sb);
                    sb ^= 1;
                }
            }
            bulk_wait_all();
        }
    } else if (bias) {
        // bias / beta gradient: column sums of the delta tiles (channel pairs, SWIZZLE_128B boxes)
        const int t = (warp - 10) * 32 + lane;
        constexpr int NPAIR = CO / 2, NG = 128 / NPAIR > 0 ? 128 / NPAIR : 1;
        const int cp = t % NPAIR, gi = t / NPAIR;
        int stage = 0;
        uint32_t phase = 0;
        float2 sum = make_float2(0.f, 0.f);
        for (int pt = p0; pt < p1; ++pt) {
            ptx::mbar_wait(full + stage, phase);
            if (gi < NG) {
                const float2 vv = db_pair_sum(ptx::smem_u32(smem + stage * SB), cp, gi, NG, 0, 1);
                sum.x += vv.x;
                sum.y += vv.y;
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(empty + stage);
            if (++stage == S) { stage = 0; phase ^= 1; }
        }
        const int co = 2 * cp;
        if (gi < NG && p0 < p1) {
            if (co < P.c_out) atomicAdd(P.db + co, sum.x);
            if (co + 1 < P.c_out) atomicAdd(P.db + co + 1, sum.y);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, Cfg::kTmemCols);
    }
}

// ------------------------------------------------------------------ wgrad, row halo (stride 1)
// One work item = (co tile of 128, filter row ky, ci tile of BN, pixel split); its k taps
// kx = 0..k-1 accumulate in k TMEM accumulators (k * BN columns).  Per pixel tile (TW x TH
// output pixels, TW a multiple of 16) the band delta is loaded once (two 64-channel MN-major
// boxes, K = pixels in raster order) and the input once as a halo box of (TW+k-1) x TH pixels
// (row pitch TW+k-1) per 64-channel chunk.  The B operand of K-step j (16 pixels = output
// row r, columns c..c+15) for tap kx starts at box row r*(TW+k-1) + c + kx: every MMA gets its
// own start, so one box serves all k taps (the absolute-address SWIZZLE_128B pattern makes an
// arbitrary 128-byte row start valid).  Traffic per pixel tile: 32 KB delta + (BN/64) boxes of
// (TW+k-1)*TH*128 B, for 8k MMAs; the per-tap kernel loads 32 KB + BN*256 B for 8 MMAs.
struct WgHaloCfg {
    static constexpr int kBoxMax = ((144 * 128 + 1023) / 1024) * 1024;   // (TW+k-1)*TH <= 144 rows (k = 3)
};
template <int BN, int KW>
struct WgHCfg {
    static constexpr int kXBox = WgHaloCfg::kBoxMax;
    static constexpr int kStageBytes = kWgA + (BN / 64) * kXBox;
    static constexpr int kStages = (224 * 1024) / kStageBytes > 8 ? 8 : (224 * 1024) / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
    static constexpr uint32_t kTmemCols = KW * BN <= 32 ? 32 : KW * BN <= 64 ? 64 : KW * BN <= 128 ? 128 : KW * BN <= 256 ? 256 : 512;
};


template <int BN, int KW>
__global__ void __launch_bounds__(kWgThreads, 1)
    k_wgrad_halo(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX, const TcWgrad P) {
    using Cfg = WgHCfg<BN, KW>;
    constexpr int S = Cfg::kStages;
    constexpr int SB = Cfg::kStageBytes;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + S * SB);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 1;
    uint32_t *tslot = (uint32_t *)(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        // empty: the MMA commit + (fused bias gradient) the 4 epilogue warps, which read every delta tile
        for (int i = 0; i < S; ++i) { ptx::mbar_init(full + i, 1); ptx::mbar_init(empty + i, P.db ? 5 : 1); }
        ptx::mbar_init(tfull, 1);
        ptx::mbar_init(tempty, 4);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmD);
        ptx::prefetch_tmap(&tmX);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, Cfg::kTmemCols);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int XP = P.TW + KW - 1;                  // halo box row pitch (pixels)
    const uint32_t xbytes = (uint32_t)XP * P.TH * 128;

    auto decode = [&](int item, int &cot, int &ky, int &cit, int &split) {
        split = item % P.splits;
        int r = item / P.splits;
        cit = r % P.ci_tiles; r /= P.ci_tiles;
        ky = r % KW;
        cot = r / KW;
    };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                int cot, ky, cit, split;
                decode(item, cot, ky, cit, split);
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                for (int pt = p0; pt < p1; ++pt) {
                    const int tx = pt % P.tiles_x, r = pt / P.tiles_x, ty = r % P.tiles_y, b = r / P.tiles_y;
                    const int y0 = P.out_a + ty * P.TH, x0 = tx * P.TW;
                    ptx::mbar_wait(empty + stage, phase ^ 1);
                    uint8_t *st = smem + stage * SB;
                    ptx::mbar_arrive_expect_tx(full + stage, kWgA + (BN / 64) * xbytes);
                    ptx::tma_load_4d(st, &tmD, full + stage, cot * 128, x0, y0 - P.dy_base, b);
                    ptx::tma_load_4d(st + kABytes, &tmD, full + stage, cot * 128 + 64, x0, y0 - P.dy_base, b);
#pragma unroll
                    for (int h = 0; h < BN / 64; ++h)
                        ptx::tma_load_4d(st + kWgA + h * Cfg::kXBox, &tmX, full + stage, cit * BN + h * 64, x0 - P.pad,
                                         y0 - P.pad + ky - P.x_base, b);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 1, 1);
            const uint64_t dA = ptx::smem_desc_sw128(ptx::smem_u32(smem), kABytes, 1024);
            const uint64_t dB = ptx::smem_desc_sw128(ptx::smem_u32(smem + kWgA), Cfg::kXBox, 1024);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            // B start (in 16-byte units) of K-step j relative to the box: row r*XP + c
            uint32_t joff[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int px = 16 * j, r = px / P.TW, c = px - r * P.TW;
                joff[j] = (uint32_t)(r * XP + c) * 8;
            }
            int stage = 0;
            uint32_t phase = 0, tphase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                int cot, ky, cit, split;
                decode(item, cot, ky, cit, split);
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                ptx::mbar_wait(tempty, tphase ^ 1);
                ptx::tc_fence_after();
                for (int pt = p0; pt < p1; ++pt) {
                    ptx::mbar_wait(full + stage, phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = (uint32_t)dA + stage * (SB >> 4);
                    const uint32_t b0 = (uint32_t)dB + stage * (SB >> 4);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
#pragma unroll
                            for (int kx = 0; kx < KW; ++kx)
                                ptx::umma_bf16_1t(tmem + kx * BN, a0 + j * 128, hiA, b0 + joff[j] + kx * 8, hiB, idesc,
                                                  (pt != p0 || j != 0) ? 1u : 0u);
                        ptx::umma_commit_1t(empty + stage);
                    }
                    __syncwarp();
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                ptx::umma_commit(tfull);
                tphase ^= 1;
            }
        }
    } else if (warp < 6) {
        const int ew = warp & 3;
        const int m = ew * 32 + lane;
        const int taps = KW * KW;
        uint32_t tphase = 0;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            int cot, ky, cit, split;
            decode(item, cot, ky, cit, split);
            const int co = cot * 128 + m;
            const float gsc = (P.gamma && co < P.c_out) ? __bfloat162float(P.gamma[co]) : 1.f;
            ptx::mbar_wait(tfull, tphase);
            ptx::tc_fence_after();
            float gdot = 0.f;
#pragma unroll 1
            for (int kk = 0; kk < KW; ++kk) {
                const int kx = (kk + split) % KW;   // pixel splits of a tile start at different taps (see k_wgrad_tc)
                float *dst = P.dw + ((long long)co * taps + ky * KW + kx) * P.cin_p + cit * BN;
                const bf16 *wrow = P.w + ((long long)co * taps + ky * KW + kx) * P.cin_p + cit * BN;
#pragma unroll 1
                for (int cc = 0; cc < BN / 32; ++cc) {
                    const int c = (cc + split / KW) % (BN / 32);
                    uint32_t v[32];
                    ptx::tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + kx * BN + c * 32, v);
                    const int ci0 = cit * BN + c * 32;
                    uint4 wq[4];   // dgamma: this row's 32 weights (16-byte loads overlapping the TMEM load)
                    if (P.dg && co < P.c_out) {
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            wq[q] = ci0 + 8 * q < P.cin_p ? *reinterpret_cast<const uint4 *>(wrow + c * 32 + 8 * q)
                                                          : make_uint4(0, 0, 0, 0);
                    }
                    ptx::tmem_ld_wait();
                    if (co >= P.c_out) continue;
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        if (ci0 + j < P.cin_p) {
                            red_add_v4(dst + c * 32 + j, __uint_as_float(v[j]) * gsc, __uint_as_float(v[j + 1]) * gsc,
                                       __uint_as_float(v[j + 2]) * gsc, __uint_as_float(v[j + 3]) * gsc);
                            if (P.dg) {
                                const uint4 w8 = wq[j / 8];
                                const uint32_t w0 = (j & 4) ? w8.z : w8.x, w1 = (j & 4) ? w8.w : w8.y;
                                gdot += __uint_as_float(v[j]) * bf_lo(w0) + __uint_as_float(v[j + 1]) * bf_hi(w0) +
                                        __uint_as_float(v[j + 2]) * bf_lo(w1) + __uint_as_float(v[j + 3]) * bf_hi(w1);
                            }
                        }
                }
            }
            if (P.dg && co < P.c_out) atomicAdd(P.dg + co, gdot);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty);
            tphase ^= 1;
        }
    } else if (P.db) {
        // warps 6..9: the fused bias / beta gradient (delta column sums) on their own warps, so the
        // epilogue warps never gate the pipeline stages of the next item
        const int t = (warp - 6) * 32 + lane, cp = t % 64, g = t / 64;
        int stage = 0;
        uint32_t phase = 0;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            int cot, ky, cit, split;
            decode(item, cot, ky, cit, split);
            const int nparts = P.k * P.ci_tiles, part = ky * P.ci_tiles + cit;
            const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
            float2 sum = make_float2(0.f, 0.f);
            for (int pt = p0; pt < p1; ++pt) {
                ptx::mbar_wait(full + stage, phase);
                const float2 v = db_pair_sum(ptx::smem_u32(smem + stage * SB), cp, g, 2, part, nparts);
                sum.x += v.x;
                sum.y += v.y;
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(empty + stage);
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
            const int co = cot * 128 + 2 * cp;
            if (co < P.c_out) atomicAdd(P.db + co, sum.x);
            if (co + 1 < P.c_out) atomicAdd(P.db + co + 1, sum.y);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, Cfg::kTmemCols);
    }
}

// Warp transpose-sum: lane L holds p[0..31]; returns sum over the 32 lanes of p[L] (31 shuffles by
// recursive halving: at width w a lane keeps the half of its remaining entries whose index bit w
// matches its own lane bit and adds the partner's copy of that half).
__device__ __forceinline__ float warp_tsum32(float (&p)[32], int lane) {
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
        const bool up = (lane & w) != 0;
#pragma unroll
        for (int i = 0; i < w; ++i) {
            const float send = up ? p[i] : p[i + w];
            const float keep = up ? p[i + w] : p[i];
            p[i] = keep + __shfl_xor_sync(0xffffffffu, send, w);
        }
    }
    return p[0];
}

// ------------------------------------------------------------------ wgrad, 64 output channels: tap pairs on M
// For c_out <= 64 (VGG conv1_2, the ResNet stage-1 3x3) the M = 128 output-channel tile of
// k_wgrad_halo is half empty.  Here the roles are swapped: M = 128 = two filter taps x 64 input
// channels, N = the 64 output channels, K = pixels.  A is the input halo box itself (MN-major,
// SWIZZLE_128B, one 128-byte row per pixel): the first 64-element M chunk starts at the box row of
// tap tA, the second at tap tB, and the descriptor's LBO is the row distance between the two taps,
// so one (TW+2) x (TH+2) box per 64-channel chunk serves all 9 taps of the 3x3 filter as 5 MMAs per
// 16-pixel K-step: (0,1) (2,3) (4,5) (6,7) (7,8) -- of the last pair only rows 64..127 (tap 8) are
// kept.  B is the band delta (one 64-channel MN-major box).  9 taps cost 5 MMAs instead of the 9
// half-empty ones of the (co, ky) x kx kernel.  Bias gradient fused as in k_wgrad_halo.
template <int KW>
struct WgPCfg {
    static constexpr int kXBoxMax = ((272 * 128 + 1023) / 1024) * 1024;   // (TW+2)*(TH+2) <= 272 rows
    static constexpr int kStageBytes = kABytes + kXBoxMax;
    static constexpr int kStages = (220 * 1024) / kStageBytes > 6 ? 6 : (220 * 1024) / kStageBytes;
    static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
    static constexpr int kPairs = (KW * KW + 1) / 2;
};

template <int KW>
__global__ void __launch_bounds__(kWgThreads, 1)
    k_wgrad_pair(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmX, const TcWgrad P) {
    using Cfg = WgPCfg<KW>;
    constexpr int S = Cfg::kStages, SB = Cfg::kStageBytes, NP = Cfg::kPairs, TAPS = KW * KW;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *full = (uint64_t *)(smem + S * SB);
    uint64_t *empty = full + S;
    uint64_t *tfull = empty + S;
    uint64_t *tempty = tfull + 1;
    uint32_t *tslot = (uint32_t *)(tempty + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { ptx::mbar_init(full + i, 1); ptx::mbar_init(empty + i, P.db ? 5 : 1); }
        ptx::mbar_init(tfull, 1);
        ptx::mbar_init(tempty, 4);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmD);
        ptx::prefetch_tmap(&tmX);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int XP = P.TW + KW - 1, XR = P.TH + KW - 1;   // halo box pitch / rows (pixels)
    const uint32_t xbytes = (uint32_t)XP * XR * 128;
    // pair p = taps (tA, tB): tA = 2p (last pair: TAPS-2), tB = tA + 1; box row offset of tap t
    auto tap_off = [&](int t) { return (t / KW) * XP + t % KW; };

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                const int split = item % P.splits, cit = item / P.splits;
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                for (int pt = p0; pt < p1; ++pt) {
                    const int tx = pt % P.tiles_x, r = pt / P.tiles_x, ty = r % P.tiles_y, b = r / P.tiles_y;
                    const int y0 = P.out_a + ty * P.TH, x0 = tx * P.TW;
                    ptx::mbar_wait(empty + stage, phase ^ 1);
                    uint8_t *st = smem + stage * SB;
                    ptx::mbar_arrive_expect_tx(full + stage, kABytes + xbytes);
                    ptx::tma_load_4d(st, &tmD, full + stage, 0, x0, y0 - P.dy_base, b);
                    ptx::tma_load_4d(st + kABytes, &tmX, full + stage, cit * 64, x0 - P.pad, y0 - P.pad - P.x_base, b);
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, 64, 1, 1);
            // descriptor words: low = start >> 4 | LBO >> 4 << 16, high = SBO | version | layout
            const uint32_t hi = (uint32_t)(ptx::smem_desc_sw128(0, kABytes, 1024) >> 32);
            uint32_t loA[NP];   // A (input box) of pair p at stage 0, K-step 0: start at tap tA, LBO = tB - tA rows
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const int tA = p == NP - 1 && TAPS % 2 ? TAPS - 2 : 2 * p;
                const int lbo = (tap_off(tA + 1) - tap_off(tA)) * 128;
                loA[p] = (uint32_t)ptx::smem_desc_sw128(ptx::smem_u32(smem + kABytes) + tap_off(tA) * 128, lbo, 1024);
            }
            uint32_t joff[8];   // K-step j (16 pixels): box row r*XP + c of its first pixel
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int px = 16 * j, r = px / P.TW, c = px - r * P.TW;
                joff[j] = (uint32_t)(r * XP + c) * 8;
            }
            const uint32_t lo0 = (uint32_t)ptx::smem_desc_sw128(ptx::smem_u32(smem), kABytes, 1024);
            int stage = 0;
            uint32_t phase = 0, tphase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                const int split = item % P.splits;
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                ptx::mbar_wait(tempty, tphase ^ 1);
                ptx::tc_fence_after();
                for (int pt = p0; pt < p1; ++pt) {
                    ptx::mbar_wait(full + stage, phase);
                    ptx::tc_fence_after();
                    const uint32_t so = stage * (SB >> 4);
                    const uint32_t b0 = lo0 + so;                      // delta box (B)
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
#pragma unroll
                            for (int p = 0; p < NP; ++p)
                                ptx::umma_bf16_1t(tmem + p * 64, loA[p] + so + joff[j], hi, b0 + j * 128, hi, idesc,
                                                  (pt != p0 || j != 0) ? 1u : 0u);
                        ptx::umma_commit_1t(empty + stage);
                    }
                    __syncwarp();
                    if (++stage == S) { stage = 0; phase ^= 1; }
                }
                ptx::umma_commit(tfull);
                tphase ^= 1;
            }
        }
    } else if (warp < 6) {
        const int ew = warp & 3;
        const int m = ew * 32 + lane;             // accumulator row: (tap tA or tB, input channel m & 63)
        uint32_t tphase = 0;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            const int cit = item / P.splits;
            ptx::mbar_wait(tfull, tphase);
            ptx::tc_fence_after();
            const int ci = cit * 64 + (m & 63);
            float dgacc[2] = {0.f, 0.f};   // fused dgamma: lane L keeps channel c * 32 + L's warp partial
#pragma unroll 1
            for (int p = 0; p < NP; ++p) {
                const int tA = p == NP - 1 && TAPS % 2 ? TAPS - 2 : 2 * p;
                const int t = m < 64 ? tA : tA + 1;
                const bool keep = !(p == NP - 1 && TAPS % 2 && m < 64) && ci < P.cin_p;
                float *dst = P.dw + (long long)t * P.cin_p + ci;
#pragma unroll 1
                for (int c = 0; c < 2; ++c) {
                    uint32_t v[32];
                    ptx::tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + p * 64 + c * 32, v);
                    ptx::tmem_ld_wait();
                    if (P.dg) {   // dgamma[co] = sum_{tap,ci} W * (sum_p dy x): warp transpose-sum, lane = co
                        float pj[32];
#pragma unroll
                        for (int j = 0; j < 32; ++j) {
                            const int co = c * 32 + j;
                            pj[j] = keep && co < P.c_out
                                        ? __uint_as_float(v[j]) *
                                              __bfloat162float(P.w[((long long)co * TAPS + t) * P.cin_p + ci])
                                        : 0.f;
                        }
                        dgacc[c] += warp_tsum32(pj, lane);
                    }
                    if (!keep) continue;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int co = c * 32 + j;
                        if (co < P.c_out) {
                            const float g = P.gamma ? __bfloat162float(P.gamma[co]) : 1.f;
                            asm volatile("red.global.add.f32 [%0], %1;" ::"l"(dst + (long long)co * TAPS * P.cin_p),
                                         "f"(__uint_as_float(v[j]) * g)
                                         : "memory");
                        }
                    }
                }
            }
            if (P.dg)
#pragma unroll
                for (int c = 0; c < 2; ++c)
                    if (c * 32 + lane < P.c_out) atomicAdd(P.dg + c * 32 + lane, dgacc[c]);
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty);
            tphase ^= 1;
        }
    } else if (P.db) {
        // warps 6..9: the fused bias / beta gradient (delta column sums) on their own warps, so the
        // epilogue warps never gate the pipeline stages of the next item
        const int t = (warp - 6) * 32 + lane, cp = t % 32, g = t / 32;
        int stage = 0;
        uint32_t phase = 0;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            const int split = item % P.splits, cit = item / P.splits;
            const int nparts = P.ci_tiles, part = cit;
            const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
            float2 sum = make_float2(0.f, 0.f);
            for (int pt = p0; pt < p1; ++pt) {
                ptx::mbar_wait(full + stage, phase);
                const float2 v = db_pair_sum(ptx::smem_u32(smem + stage * SB), cp, g, 4, part, nparts);
                sum.x += v.x;
                sum.y += v.y;
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(empty + stage);
                if (++stage == S) { stage = 0; phase ^= 1; }
            }
            const int co = 2 * cp;
            if (co < min(P.c_out, 64)) atomicAdd(P.db + co, sum.x);
            if (co + 1 < min(P.c_out, 64)) atomicAdd(P.db + co + 1, sum.y);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ wgrad of 8-channel-input convs (im2col)
// dW[co][tap][ci] = sum_pixels dY[p][co] X[p + off(tap)][ci] for the padded RGB layer:
// D[m = (tap - 16*mt)*8 + ci][co] (M = 128 = 16 taps x 8 channels, N = c_out) accumulates over
// K = output pixels.  Per 128-pixel tile the A operand (M-major: per pixel 16 taps x 16 bytes in
// two 64-element chunks, SWIZZLE_128B) is copied by 8 gather warps out of the tile's input patch,
// which one producer warp TMA-loads (double-buffered, as in k_conv_im2col); pixels outside the
// band contribute zero.  The band delta is one TMA box per tile (MN-major B).
struct TcWgI2c {
    View in;
    float *dw;
    const bf16 *gamma;
    int ntaps, mtiles, a_mul, c_out;
    int tap_oy[49], tap_ox[49];
    int TW, TH, tw_log2, tiles_x, tiles_y, pix_tiles, per_split, splits, items;
    int out_a, out_b, Wo, dy_base;
    int pat_w, pat_h, pat_ox, pat_oy, in_base;
    int pat_flat;          // patch map over (W*Cp, rows, B): one box row = pat_w pixels x 16 B contiguous
    float *db;             // fused bias / beta gradient (two extra warps sum the delta tiles)
    float *dg;             // fused gamma gradient (epilogue: warp sums of W * dW_raw)
    const bf16 *w;
};
static constexpr int kWiStages = 4;
static constexpr int kWiStage = 2 * 16384 + 16384;                 // A: 2 chunks x 16 KB, B: 16 KB
static constexpr int kWiThreads = (kI2cGather + 1 + 4 + 1 + 2) * 32;   // gather, MMA, 4 epilogue, patch, 2 bias
static constexpr int kWiPatchWarp = kI2cGather + 5;
static constexpr int kWiDbWarp = kI2cGather + 6;
static constexpr int kWiSmem = kWiStages * kWiStage + 2 * kI2cPatch + 1024 + 256;

template <int BN>
__global__ void __launch_bounds__(kWiThreads, 1)
    k_wgrad_im2col(const __grid_constant__ CUtensorMap tmD, const __grid_constant__ CUtensorMap tmP,
                   const TcWgI2c P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sP = smem + kWiStages * kWiStage;
    uint64_t *full = (uint64_t *)(sP + 2 * kI2cPatch);
    uint64_t *empty = full + kWiStages;
    uint64_t *tfull = empty + kWiStages;
    uint64_t *tempty = tfull + 1;
    uint64_t *pfull = tempty + 1;
    uint64_t *pempty = pfull + 2;
    uint32_t *tslot = (uint32_t *)(pempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int kMma = kI2cGather;                  // warp 8; epilogue warps 9..12; patch warp 13
    if (threadIdx.x == 0) {
        for (int i = 0; i < kWiStages; ++i) { ptx::mbar_init(full + i, kI2cGather * 32 + 1); ptx::mbar_init(empty + i, P.db ? 3 : 1); }
        ptx::mbar_init(tfull, 1);
        ptx::mbar_init(tempty, 4);
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(pfull + i, 1); ptx::mbar_init(pempty + i, kI2cGather * 32); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmD);
        ptx::prefetch_tmap(&tmP);
    }
    if (warp == kMma) ptx::tmem_alloc(tslot, BN < 32 ? 32 : BN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int twm = (1 << P.tw_log2) - 1;

    if (warp < kI2cGather) {
        // thread = (tap slot c, pixels m0 + 32 i): a quarter-warp moves 8 consecutive pixels of one tap
        const int c = (threadIdx.x >> 3) & 7, m0 = (threadIdx.x & 7) + 8 * (threadIdx.x >> 6);
        int poff[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int m = m0 + 32 * i;
            poff[i] = (m >> P.tw_log2) * P.a_mul * P.pat_w + (m & twm) * P.a_mul;
        }
        const uint32_t a_base = ptx::smem_u32(smem), p_base = ptx::smem_u32(sP);
        int stage = 0, pb = 0;
        uint32_t phase = 0, pphase = 0;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            const int split = item % P.splits, mt = item / P.splits;
            const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
            // this thread's two taps of the m tile (chunk h = taps 16 mt + 8 h .. + 8)
            int toff[2];
            bool tv[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int tap = mt * 16 + h * 8 + c;
                tv[h] = tap < P.ntaps;
                toff[h] = tv[h] ? (P.tap_oy[tap] - P.pat_oy) * P.pat_w + P.tap_ox[tap] - P.pat_ox : 0;
            }
            for (int pt = p0; pt < p1; ++pt) {
                const int tx = pt % P.tiles_x, r = pt / P.tiles_x, ty = r % P.tiles_y;
                ptx::mbar_wait(pfull + pb, pphase);
                const uint32_t pbase = p_base + pb * kI2cPatch;
                uint4 v[2][4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int m = m0 + 32 * i;
                    const bool valid = P.out_a + ty * P.TH + (m >> P.tw_log2) < P.out_b && tx * P.TW + (m & twm) < P.Wo;
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        v[h][i] = valid && tv[h] ? ld_shared_v4(pbase + (uint32_t)(poff[i] + toff[h]) * 16u)
                                                 : make_uint4(0, 0, 0, 0);
                }
                ptx::mbar_arrive(pempty + pb);
                if (++pb == 2) { pb = 0; pphase ^= 1; }
                ptx::mbar_wait(empty + stage, phase ^ 1);
                uint8_t *st = smem + stage * kWiStage;
                if (threadIdx.x == 0) {
                    const int b = r / P.tiles_y;
                    ptx::mbar_arrive_expect_tx(full + stage, 16384);
                    ptx::tma_load_4d(st + 2 * 16384, &tmD, full + stage, 0, tx * P.TW, P.out_a + ty * P.TH - P.dy_base, b);
                }
                const uint32_t sa = a_base + stage * kWiStage;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const int m = m0 + 32 * i;
#pragma unroll
                    for (int h = 0; h < 2; ++h) st_shared_v4(sa + h * 16384 + m * 128 + ((c ^ (m & 7)) << 4), v[h][i]);
                }
                fence_async_smem();
                ptx::mbar_arrive(full + stage);
                if (++stage == kWiStages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == kWiPatchWarp) {
        if (lane == 0) {
            const uint32_t pbytes = (uint32_t)P.pat_w * P.pat_h * 16;
            int pb = 0;
            uint32_t pphase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                const int split = item % P.splits;
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                for (int pt = p0; pt < p1; ++pt) {
                    const int tx = pt % P.tiles_x, r = pt / P.tiles_x, ty = r % P.tiles_y, b = r / P.tiles_y;
                    ptx::mbar_wait(pempty + pb, pphase ^ 1);
                    ptx::mbar_arrive_expect_tx(pfull + pb, pbytes);
                    const int px = tx * P.TW * P.a_mul + P.pat_ox, py = (P.out_a + ty * P.TH) * P.a_mul + P.pat_oy - P.in_base;
                    if (P.pat_flat) ptx::tma_load_3d(sP + pb * kI2cPatch, &tmP, pfull + pb, px * 8, py, b);
                    else ptx::tma_load_4d(sP + pb * kI2cPatch, &tmP, pfull + pb, 0, px, py, b);
                    if (++pb == 2) { pb = 0; pphase ^= 1; }
                }
            }
        }
    } else if (warp == kMma) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 1, 1);
            const uint64_t dA = ptx::smem_desc_sw128(ptx::smem_u32(smem), 16384, 1024);
            const uint64_t dB = ptx::smem_desc_sw128(ptx::smem_u32(smem + 2 * 16384), 16384, 1024);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            int stage = 0;
            uint32_t phase = 0, tphase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                const int split = item % P.splits;
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                ptx::mbar_wait(tempty, tphase ^ 1);
                ptx::tc_fence_after();
                for (int pt = p0; pt < p1; ++pt) {
                    ptx::mbar_wait(full + stage, phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = (uint32_t)dA + stage * (kWiStage >> 4);
                    const uint32_t b0 = (uint32_t)dB + stage * (kWiStage >> 4);
                    if (ptx::elect_one()) {
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            ptx::umma_bf16_1t(tmem, a0 + kk * 128, hiA, b0 + kk * 128, hiB, idesc, (pt != p0 || kk != 0) ? 1u : 0u);
                        ptx::umma_commit_1t(empty + stage);
                    }
                    __syncwarp();
                    if (++stage == kWiStages) { stage = 0; phase ^= 1; }
                }
                ptx::umma_commit(tfull);
                tphase ^= 1;
            }
        }
    } else if (warp >= kWiDbWarp) {
        if (P.db) {   // lane = output-channel pair (32-bit loads), warp = row parity; rows shared by the m tiles
            const int hw = warp - kWiDbWarp, nst = 2 * P.mtiles;
            const uint32_t cofs = (uint32_t)((lane & 3) * 4), chunk = (uint32_t)(lane >> 2);
            int stage = 0;
            uint32_t phase = 0;
            for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
                const int split = item % P.splits, mt = item / P.splits;
                const int p0 = split * P.per_split, p1 = min(p0 + P.per_split, P.pix_tiles);
                float s0[2] = {0.f, 0.f}, s1[2] = {0.f, 0.f};
                for (int pt = p0; pt < p1; ++pt) {
                    ptx::mbar_wait(full + stage, phase);
                    const uint32_t base = ptx::smem_u32(smem + stage * kWiStage + 2 * 16384);
                    int i = 0;
#pragma unroll 4
                    for (int r = mt * 2 + hw; r < 128; r += nst, ++i) {
                        uint32_t w;
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(w) : "r"(base + r * 128 + ((chunk ^ (r & 7)) << 4) + cofs));
                        s0[i & 1] += bf_lo(w);
                        s1[i & 1] += bf_hi(w);
                    }
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(empty + stage);
                    if (++stage == kWiStages) { stage = 0; phase ^= 1; }
                }
                const int co = 2 * lane;
                if (co < P.c_out) atomicAdd(P.db + co, s0[0] + s0[1]);
                if (co + 1 < P.c_out) atomicAdd(P.db + co + 1, s1[0] + s1[1]);
            }
        }
    } else {
        const int ew = warp & 3;
        const int m = ew * 32 + lane;                 // accumulator row = (tap - 16 mt) * 8 + ci
        uint32_t tphase = 0;
        for (int item = blockIdx.x; item < P.items; item += gridDim.x) {
            const int mt = item / P.splits;
            const int tap = mt * 16 + (m >> 3), ci = m & 7;
            ptx::mbar_wait(tfull, tphase);
            ptx::tc_fence_after();
            float dgacc[BN / 32];   // fused dgamma: lane L keeps channel c * 32 + L's warp partial
#pragma unroll
            for (int c = 0; c < BN / 32; ++c) dgacc[c] = 0.f;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                uint32_t v[32];
                ptx::tmem_ld32(tmem + ((uint32_t)(ew * 32) << 16) + c * 32, v);
                ptx::tmem_ld_wait();
                if (tap < P.ntaps) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int co = c * 32 + j;
                        if (co < P.c_out) {
                            const float g = P.gamma ? __bfloat162float(P.gamma[co]) : 1.f;
                            atomicAdd(P.dw + ((long long)co * P.ntaps + tap) * 8 + ci, __uint_as_float(v[j]) * g);
                        }
                    }
                }
                if (P.dg) {   // dgamma[co] = sum_{tap,ci} W * (sum_p dy x): warp sum per co (all lanes shuffle)
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const int co = c * 32 + j;
                        float pj = tap < P.ntaps && co < P.c_out
                                       ? __uint_as_float(v[j]) *
                                             __bfloat162float(P.w[((long long)co * P.ntaps + tap) * 8 + ci])
                                       : 0.f;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) pj += __shfl_xor_sync(0xffffffffu, pj, o);
                        if (lane == j) dgacc[c] += pj;
                    }
                }
            }
            if (P.dg) {
#pragma unroll
                for (int c = 0; c < BN / 32; ++c)
                    if (c * 32 + lane < P.c_out) atomicAdd(P.dg + c * 32 + lane, dgacc[c]);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty);
            tphase ^= 1;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kMma) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, BN < 32 ? 32 : BN);
    }
}

// ------------------------------------------------------------------ conv FP / dgrad: halo + resident weights
// 64-channel 3x3 stride-1 layers (VGG conv1_2, ResNet stage-1 3x3) are load-bound in the per-tap
// kernel (a 16 KB A box + an 8 KB weight box per 136 tensor cycles).  Here the whole weight
// tensor (9 taps x 64 x 64, 72 KB) is TMA-loaded once per CTA and stays in smem, and the A
// operand of all 9 taps comes from one (8+2) x (16+2) halo box per tile (HaloGeom): per tile
// 23 KB of loads for 36 MMAs.  Epilogue: TMA store (FP) or TMA load/combine/store (dgrad).
static constexpr int kRbSA = 3;
static constexpr int kRbB = 9 * 64 * 128;                                    // 72 KB
static constexpr int kRbSmem = kRbSA * HaloGeom<3>::kABytes + kRbB + 4 * kOutStage + 1024 + 512;
static constexpr int kRbThreads = 224;   // producer, MMA, 4 epilogue warps, store warp

__global__ void __launch_bounds__(kRbThreads, 1)
    k_conv_halo_rb(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmO, const __grid_constant__ CUtensorMap tmG, const TcConv P) {
    constexpr int BN = 64, KH = 3, taps = 9, SA = kRbSA;
    constexpr int HP = HaloGeom<KH>::kPitch, AB = HaloGeom<KH>::kABytes;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t *sA = smem;
    uint8_t *sB = smem + SA * AB;
    uint8_t *sO = sB + kRbB;                         // 4 x 16 KB staging: two dgrad (delta, act) pairs
    uint64_t *fullA = (uint64_t *)(sO + 4 * kOutStage);
    uint64_t *emptyA = fullA + SA;
    uint64_t *bfull = emptyA + SA;
    uint64_t *tfull = bfull + 1;
    uint64_t *tempty = tfull + 2;
    uint64_t *ebar = tempty + 2;                     // staging ring [4] (FP) / pairs [2] (dgrad), gdone [4]
    uint32_t *tslot = (uint32_t *)(ebar + 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < SA; ++i) { ptx::mbar_init(fullA + i, 1); ptx::mbar_init(emptyA + i, 1); }
        ptx::mbar_init(bfull, 1);
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, 4); }
        for (int i = 0; i < 8; ++i) ptx::mbar_init(ebar + i, i < 4 ? 1 : 4);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, 2 * BN);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();     // PDL: the setup above overlapped the previous kernel's tail; its results are visible now
    ptx::griddep_launch();   // let the next kernel's CTAs start their own setup as SMs free up
    const int num_tiles = P.m_tiles;

    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(bfull, kRbB);
            for (int tap = 0; tap < taps; ++tap) ptx::tma_load_3d(sB + tap * BN * 128, &tmB, bfull, 0, tap, 0);
            int sa = 0;
            uint32_t pa = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                int nt, tx, ty, b;
                P.decode(tile, nt, tx, ty, b);
                const int y0 = P.out_a + ty * 16, x0 = tx * 8;
                ptx::mbar_wait(emptyA + sa, pa ^ 1);
                ptx::mbar_arrive_expect_tx(fullA + sa, HP * HaloGeom<KH>::kRows * 128);
                ptx::tma_load_4d(sA + sa * AB, &tmA, fullA + sa, 0, x0 - P.pad, y0 - P.pad - P.in_base, b);
                if (++sa == SA) { sa = 0; pa ^= 1; }
            }
        }
    } else if (warp == 1) {
        {   // whole warp: tcgen05.mma / commit are elect.sync-issued once per warp
            constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 0, 0);
            const uint64_t dA = ptx::smem_desc_sw128_bo(ptx::smem_u32(sA), 16, HP * 128, 0);
            const uint64_t dB = ptx::smem_desc_sw128(ptx::smem_u32(sB), 16, 1024);
            const uint32_t hiA = (uint32_t)(dA >> 32), hiB = (uint32_t)(dB >> 32);
            ptx::mbar_wait(bfull, 0);
            int sa = 0, acc = 0;
            uint32_t pa = 0, aphase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                ptx::mbar_wait(tempty + acc, aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                ptx::mbar_wait(fullA + sa, pa);
                ptx::tc_fence_after();
                const uint32_t a0 = (uint32_t)dA + sa * (AB >> 4);
                if (ptx::elect_one()) {
#pragma unroll 1
                    for (int tap = 0; tap < taps; ++tap) {
                        const int ky = tap / KH, kx = tap - ky * KH;
                        const uint32_t at = a0 + (uint32_t)(ky * HP + kx) * 8;
                        const uint32_t b0 = (uint32_t)dB + tap * (BN * 128 >> 4);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk)
                            ptx::umma_bf16_1t(d, at + 2 * kk, hiA, b0 + 2 * kk, hiB, idesc, (tap | kk) != 0);
                    }
                    ptx::umma_commit_1t(emptyA + sa);
                    ptx::umma_commit_1t(tfull + acc);
                }
                __syncwarp();
                if (++sa == SA) { sa = 0; pa ^= 1; }
                if (++acc == 2) { acc = 0; aphase ^= 1; }
            }
        }
    } else if (warp == 6) {   // store warp
        if (lane == 0) {
            if (P.mode == 0) conv_store_dma<BN, 4>(P, &tmO, sO, nullptr, ebar, ebar + 4);
            else conv_store_dma_dg<BN, 2>(P, &tmO, &tmG, nullptr, sO, ebar, ebar + 4);
        }
    } else if (P.mode == 0) {
        conv_epilogue_tma<BN, 4, 4, true>(P, &tmO, tmem, tfull, tempty, sO, warp, lane, 2, nullptr, ebar, ebar + 4);
    } else {
        conv_epilogue_tma_dg2<BN, 4, 2, true>(P, &tmO, &tmG, tmem, tfull, tempty, sO, ebar, warp, lane, 2, nullptr, ebar + 4);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 2 * BN);
    }
}

// ------------------------------------------------------------------ host side
// Launch with programmatic dependent launch (PDL): the kernel may start while the previous kernel
// in the stream is still finishing; every tcgen05 kernel runs its barrier / TMEM / tensor-map setup
// first and then waits (griddepcontrol.wait) before touching global memory.  Captured into the
// step's CUDA graph as programmatic edges.  LRCNN_PDL=0 disables it.
static int env_int(const char *name, int dflt);
static thread_local const char *g_last_kernel = nullptr;
// A failure that is not a shape decline (a launch or attribute error, or a strided dgrad whose later
// parity class failed after earlier ones were enqueued): the engine turns it into LRCNN_E_CUDA
// instead of running the SIMT kernel over the same rows.
static thread_local bool g_tc_error = false;
bool tc_take_error() { const bool e = g_tc_error; g_tc_error = false; return e; }
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device) -- thread safe
static bool smem_attr(const void *kern, int bytes) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { g_tc_error = true; return false; }
    static std::mutex mu;
    static std::set<std::pair<const void *, int>> done;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count({kern, dev})) return true;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) {
        g_tc_error = true;
        return false;
    }
    done.insert({kern, dev});
    return true;
}
static void note_kernel(const void *fn) {
    const char *nm = nullptr;
    if (cudaFuncGetName(&nm, fn) == cudaSuccess) g_last_kernel = nm;
}
const char *tc_last_kernel() { return g_last_kernel; }
void tc_clear_last_kernel() { g_last_kernel = nullptr; }
// Per-launch profiling (lrcnn_profile_enable) turns PDL off: with programmatic launches a CUDA event
// recorded between two kernels may complete when the first kernel TRIGGERS its dependents (right
// after its setup) instead of when it finishes, which moves time from one kernel to the next.
static thread_local bool g_pdl_off = false;
void tc_set_pdl(bool on) { g_pdl_off = !on; }
template <typename... KArgs, typename... Args>
static bool launch_pdl(void (*kern)(KArgs...), int grid, int block, size_t smem, cudaStream_t st, Args &&...args) {
    static const int pdl_env = env_int("LRCNN_PDL", 1);
    const int pdl = pdl_env && !g_pdl_off;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3((unsigned)block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const bool ok = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...) == cudaSuccess;
    if (ok) note_kernel((const void *)kern);
    else g_tc_error = true;
    return ok;
}
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    });
    return fn;
}

static int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

// 4D map over a band View: dims (Cp, W, rows, B); box (64, TW*es, TH*es, 1) with TMA element
// stride es along W and H (es = conv stride: the box then holds TW x TH strided pixels); 128B swizzle.
static CUtensorMapSwizzle swz_for(int kc) {
    return kc == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : (kc == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B);
}

// kc = channels per box (64 -> 128B rows / SWIZZLE_128B, 16 -> 32B rows / SWIZZLE_32B).
static bool encode_view(CUtensorMap *m, const View &v, int B, int TW, int TH, int es = 1, int kc = 64, int nb = 1) {
    auto fn = encode_fn();
    if (!fn || v.rows <= 0 || TW * es > 256 || TH * es > 256 || nb < 1 || nb > 256) return false;
    cuuint64_t dims[4] = {(cuuint64_t)v.Cp, (cuuint64_t)v.W, (cuuint64_t)v.rows, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)v.Cp * 2, (cuuint64_t)v.W * v.Cp * 2, (cuuint64_t)v.bs * 2};
    cuuint32_t box[4] = {(cuuint32_t)kc, (cuuint32_t)(TW * es), (cuuint32_t)(TH * es), (cuuint32_t)nb};
    cuuint32_t estr[4] = {1, (cuuint32_t)es, (cuuint32_t)es, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, v.p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    swz_for(kc), CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// 3D map over OHWI weights [rows][taps][cin_p]: box (kc channels, 1 tap, BN rows); channels
// beyond cin_p (small-channel layers, e.g. the padded RGB input) are zero-filled by TMA.
static bool encode_w(CUtensorMap *m, const void *w, int rows, int taps, int cin_p, int BN, int kc = 64) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[3] = {(cuuint64_t)cin_p, (cuuint64_t)taps, (cuuint64_t)rows};
    cuuint64_t strides[2] = {(cuuint64_t)cin_p * 2, (cuuint64_t)taps * cin_p * 2};
    cuuint32_t box[3] = {(cuuint32_t)kc, 1, (cuuint32_t)BN};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void *>(w), dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, swz_for(kc), CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// choose a 128-pixel rectangle TW x TH (TW*TH = 128, TW*s <= 256) minimising padded pixels
static void pick_tile(int rows, int W, int s, int &TW, int &TH) {
    long best = -1;
    for (int tw = 128; tw >= 4; tw >>= 1) {
        int th = 128 / tw;
        if (tw * s > 256 || th * s > 256) continue;
        long cost = (long)((W + tw - 1) / tw) * tw * (long)((rows + th - 1) / th) * th;
        if (best < 0 || cost < best) { best = cost; TW = tw; TH = th; }
    }
}

// a 64-pixel rectangle TW x TH (TW*TH = 64, TW*s <= 256) minimising padded pixels
static void pick_tile64(int rows, int W, int s, int &TW, int &TH) {
    long best = -1;
    for (int tw = 64; tw >= 4; tw >>= 1) {
        int th = 64 / tw;
        if (tw * s > 256 || th * s > 256) continue;
        long cost = (long)((W + tw - 1) / tw) * tw * (long)((rows + th - 1) / th) * th;
        if (best < 0 || cost < best) { best = cost; TW = tw; TH = th; }
    }
}

// the same with batch folding: a 128-pixel tile of TW x TH x NB (NB images of a small map), the
// shape with the fewest padded pixel slots (small maps: 7x7 -> 8x8x2 instead of 8x16x1)
static void pick_tile_nb(int rows, int W, int s, int B, int &TW, int &TH, int &NB, int px = 128) {
    long best = -1;
    for (int nb = 1; nb <= 16 && nb <= px / 4; nb <<= 1)
        for (int tw = px / nb; tw >= 4; tw >>= 1) {
            const int th = px / nb / tw;
            if (th < 1 || tw * s > 256 || th * s > 256) continue;
            const long cost = (long)((B + nb - 1) / nb) * nb * ((W + tw - 1) / tw) * tw * (long)((rows + th - 1) / th) * th;
            if (best < 0 || cost < best) { best = cost; TW = tw; TH = th; NB = nb; }
        }
}

static bool aligned16(const void *p) { return ((uintptr_t)p & 15) == 0; }

bool tc_available() { return true; }

bool tc_smem_attr(const void *kern, int bytes) { return smem_attr(kern, bytes); }
int tc_num_sms() { return num_sms(); }
bool tc_encode_view(CUtensorMap *m, const View &v, int B, int TW, int TH, int es, int kc) {
    return encode_view(m, v, B, TW, TH, es, kc);
}
bool tc_encode_w(CUtensorMap *m, const void *w, int rows, int taps, int cin_p, int BN, int kc) {
    return encode_w(m, w, rows, taps, cin_p, BN, kc);
}
bool tc_pdl_on() {
    static const int pdl_env = env_int("LRCNN_PDL", 1);
    return pdl_env && !g_pdl_off;
}
void tc_note_launch(const void *fn, bool ok) {
    if (ok) note_kernel(fn);
    else g_tc_error = true;
}

template <int BN, int KC, int NBUF = 4>
static bool launch_conv(const TcConv &P, const CUtensorMap &A, const CUtensorMap &Bm, const CUtensorMap &O,
                        const CUtensorMap &G, const CUtensorMap &X, int tiles, cudaStream_t st) {
    using Cfg = ConvCfg<BN, KC, NBUF>;
    if (!smem_attr((const void *)k_conv_tc<BN, KC, NBUF>, Cfg::kSmem)) return false;
    int grid = tiles < num_sms() ? tiles : num_sms();
    return launch_pdl(k_conv_tc<BN, KC, NBUF>, grid, kConvTcThreads, Cfg::kSmem, st, A, Bm, O, G, P, X);
}

template <int BN>
static bool launch_conv_halo(const TcConv &P, const CUtensorMap &A, const CUtensorMap &Bm, const CUtensorMap &O,
                             int tiles, cudaStream_t st) {
    using Cfg = HaloCfg<BN, 3>;
    if (!smem_attr((const void *)k_conv_tc_halo<BN, 3>, Cfg::kSmem)) return false;
    int grid = tiles < num_sms() ? tiles : num_sms();
    return launch_pdl(k_conv_tc_halo<BN, 3>, grid, kThreads, Cfg::kSmem, st, A, Bm, O, P);
}

static int env_int(const char *name, int dflt) {
    const char *v = getenv(name);
    return v && *v ? atoi(v) : dflt;
}

// 64 -> 64 channel 3x3 stride-1 FP / dgrad (unit output stride) through k_conv_halo_rb
static bool conv_halo_rb(TcConv &P, const View &in, const void *w, int w_rows, int cin_p, cudaStream_t st) {
    static const int on = env_int("LRCNN_HALO_RB", 1);
    if (!on || cin_p != 64 || P.n_out != 64 || P.ntaps != 9 || P.k != 3 || P.o_stride != 1 || P.a_mul != 1) return false;
    if (P.mode == 1 && (P.out.Cp != 64 || (P.gate && (P.act.Cp != 64 || !aligned16(P.act.p))))) return false;
    if (P.mode == 0 && P.out.Cp % 8) return false;
    const int rows = P.out_b - P.out_a;
    P.in_base = in.base;
    P.n_tiles = 1;
    P.TW = 8; P.TH = 16;
    P.tiles_x = (P.Wo + 7) / 8;
    P.tiles_y = (rows + 15) / 16;
    P.m_tiles = P.B * P.tiles_x * P.tiles_y;
    tile_div_init(P);
    CUtensorMap A, Bm, O, G;
    if (!encode_w(&Bm, w, w_rows, 9, cin_p, 64, 64)) return false;
    if (!encode_view(&A, in, P.B, HaloGeom<3>::kPitch, HaloGeom<3>::kRows)) return false;
    View ov = P.out;
    ov.rows = P.out_b - P.out.base;
    if (!encode_view(&O, ov, P.B, 8, 16)) return false;
    G = O;
    if (P.mode == 1 && P.gate && !encode_view(&G, P.act, P.B, 8, 16)) return false;
    P.tma_out = P.mode == 0;
    P.tma_dg = P.mode == 1;
    if (!smem_attr((const void *)k_conv_halo_rb, kRbSmem)) return false;
    const int grid = P.m_tiles < num_sms() ? P.m_tiles : num_sms();
    return launch_pdl(k_conv_halo_rb, grid, kRbThreads, kRbSmem, st, A, Bm, O, G, P);
}

// Launch one implicit-GEMM conv over the output grid rows [P.out_a, P.out_b) x cols [0, P.Wo).
// Caller sets the epilogue fields, the output mapping (o_*), a_mul and the tap table.
static bool conv_launch(TcConv &P, const View &in, const void *w, int w_rows, int w_taps, int cin_p,
                        cudaStream_t st) {
    if (in.Cp % 8 || cin_p != in.Cp || P.n_out < 8 || P.n_out % 8 || P.ntaps < 1 || P.ntaps > 49) return false;
    if (!aligned16(in.p) || !aligned16(w) || !aligned16(P.out.p)) return false;
    int BN = P.n_out <= 64 ? 64 : (P.n_out <= 128 ? 128 : 256);
    const int rows = P.out_b - P.out_a;
    if (rows <= 0 || P.Wo <= 0) return true;
    if (P.halo_ok && conv_halo_rb(P, in, w, w_rows, cin_p, st)) return true;
    P.dbg = 0;
    P.in_base = in.base;
    static const int halo_on = env_int("LRCNN_HALO", 0), boff = 0;
    const int KC = cin_p <= 16 ? 16 : 64;   // small-channel layers: 16-ch chunks
    P.cin_chunks = (cin_p + KC - 1) / KC;
    P.k_steps = P.ntaps * P.cin_chunks;
    P.n_tiles = (P.n_out + BN - 1) / BN;
    CUtensorMap A, Bm;
    if (!encode_w(&Bm, w, w_rows, w_taps, cin_p, BN, KC)) return false;
    static const int halo_fp128 = env_int("LRCNN_HALO_FP128", 1);   // FP of 128-wide outputs: A traffic / 6
    static const int cta2 = env_int("LRCNN_2CTA", 1);
    // stride-1 3x3 with >= 128 outputs: CTA pairs + halo-reuse A (k_conv_tc2h)
    bool try2h = cta2 && KC == 64 && BN >= 128 && P.halo_ok && cin_p % 64 == 0 && P.o_stride == 1;
    if (try2h) {   // the fixed 8 x 16 halo tile must not pad small maps much more than pick_tile would
        int tw = 8, th = 16;
        pick_tile(rows, P.Wo, 1, tw, th);
        const long best = (long)((P.Wo + tw - 1) / tw) * tw * ((rows + th - 1) / th) * th;
        const long halo = (long)((P.Wo + 7) / 8) * 8 * ((rows + 15) / 16) * 16;
        // FP with 128 outputs would otherwise take the single-CTA halo kernel (same 8 x 16 tile)
        try2h = halo * 100 <= best * 108 || (P.mode == 0 && BN == 128 && halo_fp128);
    }
    if (!try2h && (halo_on || (halo_fp128 && P.mode == 0 && BN == 128)) && P.halo_ok && cin_p % 64 == 0 &&
        P.o_stride == 1) {
        P.TW = 8; P.TH = 16;
        P.tiles_x = (P.Wo + 7) / 8;
        P.tiles_y = (rows + 15) / 16;
        P.m_tiles = P.B * P.tiles_x * P.tiles_y;
        tile_div_init(P);
        P.boff = boff;
        if (!encode_view(&A, in, P.B, HaloGeom<3>::kPitch, HaloGeom<3>::kRows)) return false;
        CUtensorMap O = A;
        P.tma_out = 0;
        if (P.mode == 0 && P.o_stride == 1 && P.out.Cp % 8 == 0) {
            View ov = P.out;
            ov.rows = P.out_b - P.out.base;
            if (encode_view(&O, ov, P.B, 8, 16)) P.tma_out = 1;
        }
        int tiles = P.m_tiles * P.n_tiles;
        if (BN == 64) return launch_conv_halo<64>(P, A, Bm, O, tiles, st);
        if (BN == 128) return launch_conv_halo<128>(P, A, Bm, O, tiles, st);
        return launch_conv_halo<256>(P, A, Bm, O, tiles, st);
    }
    static const int fold = env_int("LRCNN_BATCH_FOLD", 1);
    int NB = 1;
    if (try2h) { P.TW = 8; P.TH = 16; }
    else if (fold) pick_tile_nb(rows, P.Wo, P.a_mul, P.B, P.TW, P.TH, NB);
    else pick_tile(rows, P.Wo, P.a_mul, P.TW, P.TH);
    P.NBt = NB;
    P.tiles_x = (P.Wo + P.TW - 1) / P.TW;
    P.tiles_y = (rows + P.TH - 1) / P.TH;
    P.m_tiles = (P.B + NB - 1) / NB * P.tiles_x * P.tiles_y;
    tile_div_init(P);
    // small-K layers (one or two K-steps per tile: the 1x1 convolutions of ResNet's bottleneck ends)
    // are bound by the epilogue's tile traffic: the deep (8-buffer) staging ring.  (Per-warp TMA epilogue
    // boxes, round 1, measured slower than the store-warp ring -- profiles/r02/r02e_epilogue_w_timeline_
    // cycles.txt -- and were removed.)
    static const int deep = env_int("LRCNN_DEEP_RING", 1);
    const bool deep_ring = deep && !try2h && P.k_steps <= 2 && BN >= 128 && KC == 64;
    P.warp_epi = 0;
    const int EW = P.TW, EH = P.TH;   // epilogue box
    if (try2h ? !encode_view(&A, in, P.B, HaloGeom<3>::kPitch, HaloGeom<3>::kRows)
              : !encode_view(&A, in, P.B, P.TW, P.TH, P.a_mul, KC, NB))
        return false;
    // output map for the TMA-store epilogue (FP, unit output stride): rows end at out_b
    static const int tma_out = env_int("LRCNN_TMA_OUT", 1);
    CUtensorMap O = A;
    P.tma_out = 0;
    if (tma_out && P.mode == 0 && P.o_stride == 1 && P.out.Cp % 8 == 0) {
        View ov = P.out;
        ov.rows = P.out_b - P.out.base;
        if (encode_view(&O, ov, P.B, EW, EH, 1, 64, NB)) P.tma_out = 1;
    }
    // dgrad with unit output stride: TMA load / combine / store of the delta tile
    static const int tma_dg = env_int("LRCNN_TMA_DG", 1);
    CUtensorMap G = A;
    P.tma_dg = 0;
    P.tma_res = 0;
    static const int tma_res = env_int("LRCNN_TMA_RES", 1);
    if (tma_res && P.tma_out && P.has_res && P.res.Cp == P.out.Cp && P.n_out % 64 == 0 && aligned16(P.res.p) &&
        encode_view(&G, P.res, P.B, EW, EH, 1, 64, NB))
        P.tma_res = 1;
    // (strided convs: each parity class writes every o_stride-th row / column of delta_in, so the
    // delta / activation boxes use TMA element strides o_stride; rows end at the class's last row)
    if (tma_dg && P.mode == 1 && P.out.Cp % 64 == 0 && P.n_out == P.out.Cp &&
        (!P.gate || (P.act.Cp == P.out.Cp && aligned16(P.act.p)))) {
        View ov = P.out;
        ov.rows = P.o_row0 + P.o_stride * (P.out_b - 1) + 1 - P.out.base;
        if (encode_view(&O, ov, P.B, EW, EH, P.o_stride, 64, NB) &&
            (!P.gate || encode_view(&G, P.act, P.B, EW, EH, P.o_stride, 64, NB)))
            P.tma_dg = 1;
    }
    // fused residual addend (write-mode dgrad with unit stride; k_conv_tc / k_conv_tc2 only)
    CUtensorMap X = A;
    P.dg_add = 0;
    if (P.add_req && P.tma_dg && P.dg_write && !try2h && P.o_stride == 1 && P.add.Cp == P.out.Cp &&
        aligned16(P.add.p) && P.add.rows > 0 && encode_view(&X, P.add, P.B, EW, EH, 1, 64, NB))
        P.dg_add = 1;
    int tiles = P.m_tiles * P.n_tiles;
    if (try2h && (P.tma_out || P.tma_dg) && P.m_tiles >= 2) {
        P.cta2 = 1;
        P.m_tiles += P.m_tiles & 1;
        tiles = P.m_tiles * P.n_tiles;
        if (!encode_w(&Bm, w, w_rows, w_taps, cin_p, BN / 2, KC)) return false;
        const int grid = tiles < num_sms() ? tiles : num_sms() & ~1;
        if (BN == 256) {
            if (!smem_attr((const void *)k_conv_tc2h<256>, Conv2HCfg<256>::kSmem)) return false;
            return launch_pdl(k_conv_tc2h<256>, grid, kConv2Threads, Conv2HCfg<256>::kSmem, st, A, Bm, O, G, P);
        }
        if (!smem_attr((const void *)k_conv_tc2h<128>, Conv2HCfg<128>::kSmem)) return false;
        return launch_pdl(k_conv_tc2h<128>, grid, kConv2Threads, Conv2HCfg<128>::kSmem, st, A, Bm, O, G, P);
    }
    if (try2h) {   // no TMA epilogue for this shape: single-CTA halo kernel with the same box map
        if (BN == 128) return launch_conv_halo<128>(P, A, Bm, O, tiles, st);
        return launch_conv_halo<256>(P, A, Bm, O, tiles, st);
    }
    if (cta2 && KC == 64 && BN >= 128 && (P.tma_out || P.tma_dg) && P.m_tiles >= 2 && P.k_steps >= 8) {
        // CTA pairs: M = 256 (two pixel tiles), each CTA loads half of the weight tile
        P.cta2 = 1;
        P.m_tiles += P.m_tiles & 1;
        tiles = P.m_tiles * P.n_tiles;
        if (!encode_w(&Bm, w, w_rows, w_taps, cin_p, BN / 2, KC)) return false;
        int grid = tiles < num_sms() ? tiles : num_sms() & ~1;
        if (BN == 256) {
            if (!smem_attr((const void *)k_conv_tc2<256>, Conv2Cfg<256>::kSmem)) return false;
            return launch_pdl(k_conv_tc2<256>, grid, kConv2Threads, Conv2Cfg<256>::kSmem, st, A, Bm, O, G, P, X);
        }
        if (!smem_attr((const void *)k_conv_tc2<128>, Conv2Cfg<128>::kSmem)) return false;
        return launch_pdl(k_conv_tc2<128>, grid, kConv2Threads, Conv2Cfg<128>::kSmem, st, A, Bm, O, G, P, X);
    }
    if (KC == 16) {
        if (BN == 64) return launch_conv<64, 16>(P, A, Bm, O, G, X, tiles, st);
        if (BN == 128) return launch_conv<128, 16>(P, A, Bm, O, G, X, tiles, st);
        return launch_conv<256, 16>(P, A, Bm, O, G, X, tiles, st);
    }
    if (deep_ring && (P.tma_out || P.tma_dg)) {
        if (BN == 256) return launch_conv<256, 64, 8>(P, A, Bm, O, G, X, tiles, st);
        if (BN == 128) return launch_conv<128, 64, 8>(P, A, Bm, O, G, X, tiles, st);
    }
    if (BN == 64) return launch_conv<64, 64>(P, A, Bm, O, G, X, tiles, st);
    if (BN == 128) return launch_conv<128, 64>(P, A, Bm, O, G, X, tiles, st);
    return launch_conv<256, 64>(P, A, Bm, O, G, X, tiles, st);
}

// weights [rows][K] (K = taps * 8, the OHWI layout of an 8-channel input) as a 2D map with
// 64-element boxes (SWIZZLE_128B); K beyond taps*8 and rows beyond `rows` read as zero.
static bool encode_w2d(CUtensorMap *m, const void *w, int rows, int K, int BN) {
    auto fn = encode_fn();
    if (!fn) return false;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)BN};
    cuuint32_t es[2] = {1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void *>(w), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int BN>
static bool launch_im2col(const TcConv &P, const CUtensorMap &Bm, const CUtensorMap &O, const CUtensorMap &Pm,
                          int tiles, cudaStream_t st) {
    if (!smem_attr((const void *)k_conv_im2col<BN>, kI2cSmem)) return false;
    int grid = tiles < num_sms() ? tiles : num_sms();
    return launch_pdl(k_conv_im2col<BN>, grid, kI2pThreads, kI2cSmem, st, Bm, O, Pm, P);
}

// 4D map over an 8-channel band View with a (8, pw, ph, 1) box, no swizzle (16-byte pixels packed
// densely in smem); rows outside the band's valid range [base, min(base+rows, H)) read as zero.
// the same patch with the pixel row flattened: dims (W*Cp, rows, B), box (pw*Cp, ph, 1) -- the TMA moves
// rows of pw*16 contiguous bytes instead of pw separate 16-byte elements (8-channel inputs, stride-1 box)
static bool encode_patch_flat(CUtensorMap *m, const View &v, int B, int pw, int ph) {
    auto fn = encode_fn();
    const int rows = v.rows < v.H - v.base ? v.rows : v.H - v.base;
    if (!fn || rows <= 0 || pw * v.Cp > 256 || ph > 256) return false;
    cuuint64_t dims[3] = {(cuuint64_t)v.W * v.Cp, (cuuint64_t)rows, (cuuint64_t)B};
    cuuint64_t strides[2] = {(cuuint64_t)v.W * v.Cp * 2, (cuuint64_t)v.bs * 2};
    cuuint32_t box[3] = {(cuuint32_t)(pw * v.Cp), (cuuint32_t)ph, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, v.p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
static bool encode_patch(CUtensorMap *m, const View &v, int B, int pw, int ph, int es_w = 1) {
    auto fn = encode_fn();
    const int rows = v.rows < v.H - v.base ? v.rows : v.H - v.base;
    if (!fn || rows <= 0 || pw * es_w > 256 || ph > 256) return false;
    cuuint64_t dims[4] = {(cuuint64_t)v.Cp, (cuuint64_t)v.W, (cuuint64_t)rows, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)v.Cp * 2, (cuuint64_t)v.W * v.Cp * 2, (cuuint64_t)v.bs * 2};
    cuuint32_t box[4] = {(cuuint32_t)v.Cp, (cuuint32_t)(pw * es_w), (cuuint32_t)ph, 1};
    cuuint32_t estr[4] = {1, (cuuint32_t)es_w, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, v.p, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// FP of an 8-channel-input k x k conv (stride 1 or 2, c_out <= 64) through k_conv_pair.
static bool conv_pair(TcConv &P, const View &in, const void *w, int w_rows, cudaStream_t st) {
    static const int on = env_int("LRCNN_PAIR", 1);
    const int s = P.a_mul, k = P.k;
    if (!on || in.Cp != 8 || P.mode != 0 || P.o_stride != 1 || P.n_out != 64 || P.out.Cp % 8 || w_rows > 64) return false;
    if (k > 7 || s < 1 || s > 2 || P.ntaps != k * k || !aligned16(in.p) || !aligned16(w) || !aligned16(P.out.p) ||
        (in.bs & 7))
        return false;
    const int rows = P.out_b - P.out_a;
    if (rows <= 0 || P.Wo <= 0) return true;
    const int npr = (k + 1) / 2;
    P.in = in;
    P.in_base = in.base;
    P.dbg = 0;
    P.pat_w = s == 1 ? 7 + 2 * npr : 7 + npr;
    P.pat_h = 15 * s + k;
    P.pat_ox = -P.pad; P.pat_oy = -P.pad;
    if (((P.pat_w * P.pat_h * 16 + 127) & ~127) * s > kPrPatch) return false;
    P.n_tiles = 1;
    P.TW = 8; P.TH = 16;
    P.tiles_x = (P.Wo + 7) / 8;
    P.tiles_y = (rows + 15) / 16;
    P.m_tiles = P.B * P.tiles_x * P.tiles_y;
    tile_div_init(P);
    CUtensorMap Pm, Wm, O;
    if (!encode_patch(&Pm, in, P.B, P.pat_w, P.pat_h, s)) return false;
    {   // weights [w_rows][k][k][8] as (8, kx, ky, rows), box (8, 1, 1, 64): rows / kx >= k read as zero
        auto fn = encode_fn();
        if (!fn) return false;
        cuuint64_t dims[4] = {8, (cuuint64_t)k, (cuuint64_t)k, (cuuint64_t)w_rows};
        cuuint64_t strides[3] = {16, (cuuint64_t)k * 16, (cuuint64_t)k * k * 16};
        cuuint32_t box[4] = {8, 1, 1, 64};
        cuuint32_t es[4] = {1, 1, 1, 1};
        if (fn(&Wm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void *>(w), dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return false;
    }
    View ov = P.out;
    ov.rows = P.out_b - P.out.base;
    if (!encode_view(&O, ov, P.B, 8, 16)) return false;
    P.tma_out = 1;
    if (!smem_attr((const void *)k_conv_pair, kPrSmem)) return false;
    const int grid = P.m_tiles < num_sms() ? P.m_tiles : num_sms();
    return launch_pdl(k_conv_pair, grid, kConv2Threads, kPrSmem, st, Pm, Wm, O, P);
}

// FP of an 8-channel-input conv through the im2col kernel; false = shape not taken.
static bool conv_im2col(TcConv &P, const View &in, const void *w, int w_rows, cudaStream_t st) {
    if (in.Cp != 8 || P.mode != 0 || P.o_stride != 1 || P.n_out % 8 || P.out.Cp % 8) return false;
    if (!aligned16(in.p) || !aligned16(w) || !aligned16(P.out.p) || (in.bs & 7)) return false;
    static const int on = env_int("LRCNN_IM2COL", 1);
    if (!on) return false;
    const int BN = P.n_out <= 64 ? 64 : (P.n_out <= 128 ? 128 : 256);
    const int KS = (P.ntaps + 7) / 8;
    P.n_tiles = (P.n_out + BN - 1) / BN;
    if ((long)P.n_tiles * KS * BN * 128 > kI2cBMax) return false;
    const int rows = P.out_b - P.out_a;
    if (rows <= 0 || P.Wo <= 0) return true;
    P.in = in;
    P.in_base = in.base;
    P.dbg = 0;
    // tap offset hull -> patch geometry; tile = the 128-pixel rectangle with the fewest padded
    // pixels whose patch fits one 16 KB buffer
    int oy0 = 1 << 20, oy1 = -(1 << 20), ox0 = 1 << 20, ox1 = -(1 << 20);
    for (int t = 0; t < P.ntaps; ++t) {
        oy0 = std::min(oy0, P.tap_oy[t]); oy1 = std::max(oy1, P.tap_oy[t]);
        ox0 = std::min(ox0, P.tap_ox[t]); ox1 = std::max(ox1, P.tap_ox[t]);
    }
    const int s = P.a_mul;
    long best = -1;
    for (int tw = 128; tw >= 4; tw >>= 1) {
        const int th = 128 / tw;
        const int pw = (tw - 1) * s + ox1 - ox0 + 1, ph = (th - 1) * s + oy1 - oy0 + 1;
        if (pw > 256 || ph > 256 || pw * ph * 16 > kI2cPatch) continue;
        long cost = (long)((P.Wo + tw - 1) / tw) * tw * (long)((rows + th - 1) / th) * th;
        if (best < 0 || cost < best) { best = cost; P.TW = tw; P.TH = th; P.pat_w = pw; P.pat_h = ph; }
    }
    if (best < 0) return false;
    P.pat_ox = ox0; P.pat_oy = oy0;
    P.tiles_x = (P.Wo + P.TW - 1) / P.TW;
    P.tiles_y = (rows + P.TH - 1) / P.TH;
    P.m_tiles = P.B * P.tiles_x * P.tiles_y;
    tile_div_init(P);
    CUtensorMap Bm, O, Pm;
    if (!encode_w2d(&Bm, w, w_rows, P.ntaps * 8, BN)) return false;
    if (!encode_patch(&Pm, in, P.B, P.pat_w, P.pat_h)) return false;
    View ov = P.out;
    ov.rows = P.out_b - P.out.base;
    if (!encode_view(&O, ov, P.B, P.TW, P.TH)) return false;
    P.tma_out = 1;
    const int tiles = P.m_tiles * P.n_tiles;
    if (BN == 64) return launch_im2col<64>(P, Bm, O, Pm, tiles, st);
    if (BN == 128) return launch_im2col<128>(P, Bm, O, Pm, tiles, st);
    return launch_im2col<256>(P, Bm, O, Pm, tiles, st);
}

bool tc_conv_fwd(const ConvFwdArgs &a, cudaStream_t st) {
    if (a.s < 1 || a.s > 2) return false;
    TcConv P{};
    P.out = a.out; P.res = a.res; P.has_res = a.res.p != nullptr;
    P.bias = (const bf16 *)a.b; P.beta = (const bf16 *)a.beta;
    P.mode = 0; P.epi = a.epi; P.relu = a.relu; P.gate = 0; P.c_real = a.c_out; P.n_out = a.out.Cp;
    P.out_a = a.a; P.out_b = a.b_; P.Wo = a.out.W; P.B = a.B;
    if (P.epi != 0 && !aligned16(P.bias)) return false;
    if (P.has_res && (a.res.Cp % 8 || !aligned16(a.res.p))) return false;
    if (a.k * a.k > 49) return false;
    P.a_mul = a.s; P.o_row0 = 0; P.o_col0 = 0; P.o_stride = 1;
    P.ntaps = a.k * a.k;
    for (int ky = 0; ky < a.k; ++ky)
        for (int kx = 0; kx < a.k; ++kx) {
            const int t = ky * a.k + kx;
            P.tap_oy[t] = ky - a.p; P.tap_ox[t] = kx - a.p; P.tap_w[t] = t;
        }
    P.k = a.k; P.pad = a.p; P.halo_ok = a.s == 1 && a.k == 3;
    if (a.in.Cp == 8 && conv_pair(P, a.in, a.w, a.c_out, st)) return true;
    if (a.in.Cp == 8 && conv_im2col(P, a.in, a.w, a.c_out, st)) return true;
    return conv_launch(P, a.in, a.w, a.c_out, a.k * a.k, a.in.Cp, st);
}

// dgrad: delta_in[g] += sum_{ky: (g+p-ky) = s*y} W[ky] delta[y].  The input grid is split in
// s x s parity classes (ry, rx); each class is a stride-1 implicit GEMM over the band delta
// with the class's taps of the flipped/transposed weights W' and output stride s.
bool tc_conv_dgrad(const DgradArgs &a, cudaStream_t st) {
    if (!a.wt || a.s < 1 || a.s > 2 || a.k * a.k > 49) return false;
    if (a.gate && (!aligned16(a.act.p) || a.act.Cp != a.dx.Cp)) return false;
    const int s = a.s, k = a.k, p = a.p;
    int launched = 0;
    for (int ry = 0; ry < s; ++ry)
        for (int rx = 0; rx < s; ++rx) {
            TcConv P{};
            P.out = a.dx; P.act = a.act;
            P.dg_write = a.write && s == 1;
            P.mode = 1; P.epi = 0; P.relu = 0; P.gate = a.gate; P.c_real = a.dx.Cp; P.n_out = a.dx.Cp;
            P.B = a.B; P.a_mul = 1; P.o_row0 = ry; P.o_col0 = rx; P.o_stride = s;
            // class grid: rows j with ra <= ry + s*j < rb, cols i with rx + s*i < W_in
            P.out_a = (a.ra - ry + s - 1) / s;
            P.out_b = (a.rb - ry + s - 1) / s;
            P.Wo = (a.dx.W - rx + s - 1) / s;
            if (a.ra - ry < 0) P.out_a = 0;
            int n = 0;
            for (int ky = 0; ky < k; ++ky) {
                const int dy = ry + p - ky;
                if (((dy % s) + s) % s) continue;
                for (int kx = 0; kx < k; ++kx) {
                    const int dx = rx + p - kx;
                    if (((dx % s) + s) % s) continue;
                    P.tap_oy[n] = dy >= 0 ? dy / s : -((-dy) / s);
                    P.tap_ox[n] = dx >= 0 ? dx / s : -((-dx) / s);
                    P.tap_w[n] = (k - 1 - ky) * k + (k - 1 - kx);
                    ++n;
                }
            }
            P.ntaps = n;
            if (n == 0 || P.out_b <= P.out_a || P.Wo <= 0) continue;
            P.k = k; P.pad = k - 1 - p; P.halo_ok = s == 1 && k == 3;
            if (a.add_on && s == 1) { P.add = a.add; P.add_req = 1; }
            if (!conv_launch(P, a.dy, a.wt, a.dx.Cp, k * k, a.dy.Cp, st)) {
                // earlier parity classes are already enqueued: a SIMT rerun would add them twice
                if (launched) g_tc_error = true;
                return false;
            }
            ++launched;
            if (P.dg_add) a.add_done = true;
        }
    return true;
}

template <int BN, int KP = 128>
static bool launch_wgrad(const TcWgrad &P, const CUtensorMap &D, const CUtensorMap &X, cudaStream_t st) {
    using Cfg = WgCfg<BN, KP>;
    if (!smem_attr((const void *)k_wgrad_tc<BN, KP>, Cfg::kSmem)) return false;
    int grid = P.items < num_sms() ? P.items : num_sms();
    return launch_pdl(k_wgrad_tc<BN, KP>, grid, kWgThreads, Cfg::kSmem, st, D, X, P);
}

template <int BN, int KW>
static bool launch_wgrad_halo(const TcWgrad &P, const CUtensorMap &D, const CUtensorMap &X, cudaStream_t st) {
    using Cfg = WgHCfg<BN, KW>;
    if (!smem_attr((const void *)k_wgrad_halo<BN, KW>, Cfg::kSmem)) return false;
    int grid = P.items < num_sms() ? P.items : num_sms();
    return launch_pdl(k_wgrad_halo<BN, KW>, grid, kWgThreads, Cfg::kSmem, st, D, X, P);
}

// stride-1 k x k wgrad with c_out <= 64 (one 64-channel delta box) and 64-multiple input channels
// through the tap-pair kernel (M = two taps x 64 input channels)
static bool wgrad_pair(const WgradArgs &a, cudaStream_t st) {
    static const int on = env_int("LRCNN_WG_PAIR", 1);
    const View &dy = a.dy, &x = a.x;
    if (!on || a.s != 1 || a.k != 3 || x.Cp % 64 || dy.Cp != 64 || a.c_out > 64) return false;
    const int rows = a.b - a.a;
    TcWgrad P{};
    P.dw = a.dw; P.gamma = (const bf16 *)a.gamma; P.k = a.k; P.pad = a.p; P.c_out = a.c_out; P.cin_p = x.Cp;
    P.s = 1;
    P.db = a.db;                                 // bias / beta (dedicated warps), dgamma (epilogue)
    P.dg = a.db ? a.dg : nullptr;
    P.w = (const bf16 *)a.w;
    if (P.dg && !P.w) P.db = P.dg = nullptr;
    long best = -1;
    for (int tw = 128; tw >= 16; tw >>= 1) {
        const int th = 128 / tw;
        if ((tw + a.k - 1) * (th + a.k - 1) > 272) continue;
        long cost = (long)((dy.W + tw - 1) / tw) * tw * (long)((rows + th - 1) / th) * th;
        if (best < 0 || cost < best) { best = cost; P.TW = tw; P.TH = th; }
    }
    if (best < 0) return false;
    P.tiles_x = (dy.W + P.TW - 1) / P.TW;
    P.tiles_y = (rows + P.TH - 1) / P.TH;
    P.pix_tiles = a.B * P.tiles_x * P.tiles_y;
    P.co_tiles = 1;
    P.ci_tiles = x.Cp / 64;
    int splits = num_sms() / P.ci_tiles;
    if (splits > P.pix_tiles) splits = P.pix_tiles;
    if (splits < 1) splits = 1;
    P.per_split = (P.pix_tiles + splits - 1) / splits;
    P.splits = (P.pix_tiles + P.per_split - 1) / P.per_split;
    P.items = P.ci_tiles * P.splits;
    P.out_a = a.a; P.dy_base = dy.base; P.x_base = x.base;
    CUtensorMap D, X;
    if (!encode_view(&D, dy, a.B, P.TW, P.TH)) return false;
    if (!encode_view(&X, x, a.B, P.TW + a.k - 1, P.TH + a.k - 1)) return false;
    using Cfg = WgPCfg<3>;
    if (!smem_attr((const void *)k_wgrad_pair<3>, Cfg::kSmem)) return false;
    const int grid = P.items < num_sms() ? P.items : num_sms();
    if (!launch_pdl(k_wgrad_pair<3>, grid, kWgThreads, Cfg::kSmem, st, D, X, P)) return false;
    if (P.db) a.db_done = true;
    if (P.dg) a.dg_done = true;
    return true;
}

// stride-1 3x3 wgrad with input channels in 64-multiples through the row-halo kernel
static bool wgrad_halo(const WgradArgs &a, cudaStream_t st) {
    static const int on = env_int("LRCNN_WG_HALO", 1);
    const View &dy = a.dy, &x = a.x;
    if (!on || a.s != 1 || a.k != 3 || x.Cp % 64 || dy.W < 16) return false;
    const int rows = a.b - a.a;
    TcWgrad P{};
    P.dw = a.dw; P.gamma = (const bf16 *)a.gamma; P.k = a.k; P.pad = a.p; P.c_out = a.c_out; P.cin_p = x.Cp;
    P.s = 1;
    P.db = a.db;
    P.dg = a.db ? a.dg : nullptr;
    P.w = (const bf16 *)a.w;
    if (P.dg && !P.w) P.db = P.dg = nullptr;
    // 128-pixel tile, TW a multiple of 16 (one K-step = 16 pixels of one output row)
    long best = -1;
    for (int tw = 128; tw >= 16; tw >>= 1) {
        const int th = 128 / tw;
        long cost = (long)((dy.W + tw - 1) / tw) * tw * (long)((rows + th - 1) / th) * th;
        if (best < 0 || cost < best) { best = cost; P.TW = tw; P.TH = th; }
    }
    if ((P.TW + a.k - 1) * P.TH > 144) return false;
    P.tiles_x = (dy.W + P.TW - 1) / P.TW;
    P.tiles_y = (rows + P.TH - 1) / P.TH;
    P.pix_tiles = a.B * P.tiles_x * P.tiles_y;
    const int BN = x.Cp >= 128 ? 128 : 64;
    P.co_tiles = (dy.Cp + 127) / 128;
    P.ci_tiles = (x.Cp + BN - 1) / BN;
    const int base_items = P.co_tiles * a.k * P.ci_tiles;
    // one wave: at most num_sms items (a second partial wave would double the kernel time)
    int splits = num_sms() / base_items;
    if (splits > P.pix_tiles) splits = P.pix_tiles;
    if (splits < 1) splits = 1;
    P.per_split = (P.pix_tiles + splits - 1) / splits;
    P.splits = (P.pix_tiles + P.per_split - 1) / P.per_split;
    P.items = base_items * P.splits;
    P.out_a = a.a; P.dy_base = dy.base; P.x_base = x.base;
    CUtensorMap D, X;
    if (!encode_view(&D, dy, a.B, P.TW, P.TH)) return false;
    if (!encode_view(&X, x, a.B, P.TW + a.k - 1, P.TH)) return false;
    const bool ok = BN == 64 ? launch_wgrad_halo<64, 3>(P, D, X, st) : launch_wgrad_halo<128, 3>(P, D, X, st);
    if (ok && P.db) a.db_done = true;
    if (ok && P.dg) a.dg_done = true;
    return ok;
}

template <int BN>
static bool launch_wgrad_im2col(const TcWgI2c &P, const CUtensorMap &D, const CUtensorMap &Pm, cudaStream_t st) {
    if (!smem_attr((const void *)k_wgrad_im2col<BN>, kWiSmem)) return false;
    int grid = P.items < num_sms() ? P.items : num_sms();
    return launch_pdl(k_wgrad_im2col<BN>, grid, kWiThreads, kWiSmem, st, D, Pm, P);
}

// wgrad of a conv whose input has 8 (padded) channels; N = c_out padded to 64 / 128 / 256
static bool wgrad_im2col(const WgradArgs &a, cudaStream_t st) {
    static const int on = env_int("LRCNN_IM2COL", 1);
    const View &dy = a.dy, &x = a.x;
    if (!on || x.Cp != 8 || (x.bs & 7) || !aligned16(x.p) || dy.Cp % 64 || dy.Cp > 64 || a.k * a.k > 49) return false;
    const int rows = a.b - a.a;
    TcWgI2c P{};
    P.in = x; P.dw = a.dw; P.gamma = (const bf16 *)a.gamma; P.ntaps = a.k * a.k; P.mtiles = (P.ntaps + 15) / 16;
    P.db = a.db;            // bias / beta (dedicated warps), dgamma (epilogue)
    P.dg = a.db ? a.dg : nullptr;
    P.w = (const bf16 *)a.w;
    if (P.dg && !P.w) P.db = P.dg = nullptr;
    P.a_mul = a.s; P.c_out = a.c_out;
    for (int ky = 0; ky < a.k; ++ky)
        for (int kx = 0; kx < a.k; ++kx) { P.tap_oy[ky * a.k + kx] = ky - a.p; P.tap_ox[ky * a.k + kx] = kx - a.p; }
    int oy0 = 1 << 20, oy1 = -(1 << 20), ox0 = 1 << 20, ox1 = -(1 << 20);
    for (int t = 0; t < P.ntaps; ++t) {
        oy0 = std::min(oy0, P.tap_oy[t]); oy1 = std::max(oy1, P.tap_oy[t]);
        ox0 = std::min(ox0, P.tap_ox[t]); ox1 = std::max(ox1, P.tap_ox[t]);
    }
    long best = -1;
    for (int tw = 128; tw >= 4; tw >>= 1) {
        const int th = 128 / tw;
        const int pw = (tw - 1) * a.s + ox1 - ox0 + 1, ph = (th - 1) * a.s + oy1 - oy0 + 1;
        if (pw > 256 || ph > 256 || pw * ph * 16 > kI2cPatch) continue;
        long cost = (long)((dy.W + tw - 1) / tw) * tw * (long)((rows + th - 1) / th) * th;
        if (best < 0 || cost < best) { best = cost; P.TW = tw; P.TH = th; P.pat_w = pw; P.pat_h = ph; }
    }
    if (best < 0) return false;
    P.pat_ox = ox0; P.pat_oy = oy0; P.in_base = x.base;
    int l = 0;
    while ((1 << l) < P.TW) ++l;
    P.tw_log2 = l;
    P.tiles_x = (dy.W + P.TW - 1) / P.TW;
    P.tiles_y = (rows + P.TH - 1) / P.TH;
    P.pix_tiles = a.B * P.tiles_x * P.tiles_y;
    int splits = num_sms() / P.mtiles;
    if (splits > P.pix_tiles) splits = P.pix_tiles;
    if (splits < 1) splits = 1;
    P.per_split = (P.pix_tiles + splits - 1) / splits;
    P.splits = (P.pix_tiles + P.per_split - 1) / P.per_split;
    P.items = P.mtiles * P.splits;
    P.out_a = a.a; P.out_b = a.b; P.Wo = dy.W; P.dy_base = dy.base;
    CUtensorMap D, Pm;
    if (!encode_view(&D, dy, a.B, P.TW, P.TH)) return false;
    P.pat_flat = encode_patch_flat(&Pm, x, a.B, P.pat_w, P.pat_h) ? 1 : 0;
    if (!P.pat_flat && !encode_patch(&Pm, x, a.B, P.pat_w, P.pat_h)) return false;
    const bool ok = launch_wgrad_im2col<64>(P, D, Pm, st);
    if (ok && P.db) a.db_done = true;
    if (ok && P.dg) a.dg_done = true;
    return ok;
}

// fused pointwise dgrad + wgrad (k_dwgrad_pw): 1x1 stride-1 convolutions with (Cp_in, Cp_out) =
// (64, 256) or (256, 64); false = shape not taken (the caller launches wgrad and dgrad separately)
bool tc_conv_dwgrad(const WgradArgs &wa, const DgradArgs &da, cudaStream_t st) {
    static const int on = env_int("LRCNN_DWGRAD", 1);
    if (!on || wa.k != 1 || wa.s != 1 || wa.p != 0 || da.k != 1 || da.s != 1 || da.p != 0 || !da.wt) return false;
    const int CI = wa.x.Cp, CO = wa.dy.Cp;
    if (!((CI == 64 && CO == 256) || (CI == 256 && CO == 64))) return false;
    if (wa.c_out != CO || da.dx.Cp != CI || da.ra != wa.a || da.rb != wa.b) return false;
    if (da.gate && (da.act.p != wa.x.p || da.act.base != wa.x.base || da.act.Cp != CI)) return false;
    if (da.add_on && !da.write) return false;
    if (wa.dg && !wa.w) return false;
    if (!aligned16(wa.dy.p) || !aligned16(wa.x.p) || !aligned16(da.dx.p) || !aligned16(da.wt)) return false;
    const int rows = wa.b - wa.a;
    if (rows <= 0) return false;
    TcDw P{};
    P.dx = da.dx; P.act = da.act; P.add = da.add;
    P.dw = wa.dw; P.db = wa.db; P.dg = wa.dg; P.gamma = (const bf16 *)wa.gamma; P.w = (const bf16 *)wa.w;
    P.c_out = wa.c_out; P.gate = da.gate; P.write = da.write; P.dg_add = da.add_on ? 1 : 0;
    pick_tile(rows, wa.dy.W, 1, P.TW, P.TH);
    P.tiles_x = (wa.dy.W + P.TW - 1) / P.TW;
    P.tiles_y = (rows + P.TH - 1) / P.TH;
    P.pix_tiles = wa.B * P.tiles_x * P.tiles_y;
    int grid = P.pix_tiles < num_sms() ? P.pix_tiles : num_sms();
    P.per_cta = (P.pix_tiles + grid - 1) / grid;
    grid = (P.pix_tiles + P.per_cta - 1) / P.per_cta;
    P.out_a = wa.a; P.dy_base = wa.dy.base; P.x_base = wa.x.base; P.B = wa.B;
    CUtensorMap D, X, Wm, O, A;
    if (!encode_view(&D, wa.dy, wa.B, P.TW, P.TH) || !encode_view(&X, wa.x, wa.B, P.TW, P.TH)) return false;
    if (!encode_w(&Wm, da.wt, CI, 1, CO, CI, 64)) return false;
    View ov = da.dx;
    ov.rows = da.rb - da.dx.base;
    if (!encode_view(&O, ov, wa.B, P.TW, P.TH)) return false;
    A = O;
    if (P.dg_add && (da.add.Cp != CI || !aligned16(da.add.p) || da.add.rows <= 0 ||
                     !encode_view(&A, da.add, wa.B, P.TW, P.TH)))
        return false;
    bool ok;
    if (CI == 64) {
        using Cfg = DwCfg<64, 256>;
        if (!smem_attr((const void *)k_dwgrad_pw<64, 256>, Cfg::kSmem)) return false;
        ok = launch_pdl(k_dwgrad_pw<64, 256>, grid, kDwThreads, Cfg::kSmem, st, D, X, Wm, O, A, P);
    } else {
        using Cfg = DwCfg<256, 64>;
        if (!smem_attr((const void *)k_dwgrad_pw<256, 64>, Cfg::kSmem)) return false;
        ok = launch_pdl(k_dwgrad_pw<256, 64>, grid, kDwThreads, Cfg::kSmem, st, D, X, Wm, O, A, P);
    }
    if (!ok) return false;
    wa.db_done = wa.db != nullptr;
    wa.dg_done = wa.dg != nullptr;
    da.add_done = P.dg_add != 0;
    return true;
}

bool tc_conv_wgrad(const WgradArgs &a, cudaStream_t st) {
    if (a.s < 1 || a.s > 2) return false;
    const View &dy = a.dy, &x = a.x;
    if (dy.Cp % 8 || x.Cp % 8 || !aligned16(dy.p) || !aligned16(x.p)) return false;
    const int rows = a.b - a.a;
    if (rows <= 0) { a.db_done = a.dg_done = true; return true; }
    if (wgrad_pair(a, st)) return true;
    if (wgrad_halo(a, st)) return true;
    if (wgrad_im2col(a, st)) return true;
    TcWgrad P{};
    P.dw = a.dw; P.gamma = (const bf16 *)a.gamma; P.k = a.k; P.pad = a.p; P.c_out = a.c_out; P.cin_p = x.Cp;
    P.s = a.s;
    P.db = a.db;
    P.dg = a.db ? a.dg : nullptr;
    P.w = (const bf16 *)a.w;
    if (P.dg && !P.w) P.db = P.dg = nullptr;
    static const int fold = env_int("LRCNN_BATCH_FOLD", 1);
    int NB = 1;
    if (fold) pick_tile_nb(rows, dy.W, a.s, a.B, P.TW, P.TH, NB);
    else pick_tile(rows, dy.W, a.s, P.TW, P.TH);
    // N = 256 items: 64-pixel stages (WgCfg KP) -- single-image 64-pixel tiles
    static const int kp64_on = env_int("LRCNN_WG_KP64", 1);
    const bool kp64 = kp64_on && env_int("LRCNN_WG_256", 1) && x.Cp >= 256 && x.Cp % 256 == 0;   // == BN 256
    if (kp64) {
        NB = 1;
        if (fold) pick_tile_nb(rows, dy.W, a.s, a.B, P.TW, P.TH, NB, 64);
        else pick_tile64(rows, dy.W, a.s, P.TW, P.TH);
    }
    P.NB = NB;
    P.tiles_x = (dy.W + P.TW - 1) / P.TW;
    P.tiles_y = (rows + P.TH - 1) / P.TH;
    P.pix_tiles = (a.B + NB - 1) / NB * P.tiles_x * P.tiles_y;
    // N = 256 input channels per item where the input has them: per 128-pixel K-step the tensor pipe then
    // reads 12 KB of operands per 128 cycles instead of 8 KB per 64 (N = 128), which with the TMA writes
    // of the same bytes keeps the shared-memory port at ~190 B/clk instead of ~250 (A re-read per N tile)
    static const int wide = env_int("LRCNN_WG_256", 1);
    const int BN = wide && x.Cp >= 256 && x.Cp % 256 == 0 ? 256 : x.Cp >= 128 ? 128 : (x.Cp <= 16 ? 16 : 64);
    P.co_tiles = (dy.Cp + 127) / 128;
    P.ci_tiles = (x.Cp + BN - 1) / BN;
    const int base_items = P.co_tiles * a.k * a.k * P.ci_tiles;
    static const int split_mul = env_int("LRCNN_WG_SPLIT_MUL", 1);
    int splits = split_mul * num_sms() / base_items;
    if (splits > P.pix_tiles) splits = P.pix_tiles;
    if (splits < 1) splits = 1;
    P.per_split = (P.pix_tiles + splits - 1) / splits;
    P.splits = (P.pix_tiles + P.per_split - 1) / P.per_split;
    P.items = base_items * P.splits;
    P.out_a = a.a; P.dy_base = dy.base; P.x_base = x.base;
    CUtensorMap D, X;
    if (!encode_view(&D, dy, a.B, P.TW, P.TH, 1, 64, NB)) return false;
    if (!encode_view(&X, x, a.B, P.TW, P.TH, a.s, BN < 64 ? BN : 64, NB)) return false;
    const bool ok = BN == 16 ? launch_wgrad<16>(P, D, X, st)
                  : BN == 64 ? launch_wgrad<64>(P, D, X, st)
                  : BN == 128 ? launch_wgrad<128>(P, D, X, st)
                  : kp64 ? launch_wgrad<256, 64>(P, D, X, st) : launch_wgrad<256>(P, D, X, st);
    if (ok && P.db) a.db_done = true;
    if (ok && P.dg) a.dg_done = true;
    return ok;
}

}  // namespace lrcnn

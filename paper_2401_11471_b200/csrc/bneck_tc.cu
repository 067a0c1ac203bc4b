// bneck_tc.cu -- fused ResNet bottleneck forward over one band ("band tiles
// held on-chip between fused layers"; PAPER.md:80 row-centric scheduling across layers).
//
// One persistent tcgen05 kernel computes, for an identity bottleneck block with a 64-channel
// middle (ResNet-50 conv2_x: t[256] -> 1x1 -> t1[64] -> 3x3 -> t2[64] -> 1x1 (+t) -> u[256],
// frozen-BN affine + ReLU after each conv, R11), the band rows [a2, b2) of u from the
// band rows of t, keeping t1 and t2 on chip:
//
//   per output tile (16 rows x 8 columns of one image, 128 pixels):
//     conv1  the t1 region the 3x3 needs, (16+2) x (8+2) = 180 pixels, from a TMA box of t
//            (32-channel chunks, SWIZZLE_64B): M = 2 x 128 rows of the box, N = 64, K = 256
//     epi1   affine + ReLU -> bf16, written into a shared-memory t1 box in the UMMA SWIZZLE_128B
//            layout (row pitch 10 pixels); rows above the band's first computed t1 row are the
//            2PS halo cache, read from the t1 band buffer; rows / columns outside
//            the map are the conv's zero padding (semi-closed padding)
//     conv2  3x3 over the t1 box: tap (ky, kx) is the same box at a start offset of 10*ky + kx
//            pixel rows, 8-pixel core-matrix groups 10 pixels apart (SBO), M = 128, N = 64, K = 576
//     epi2   affine + ReLU -> bf16 t2 tile in shared memory (128 x 64, SWIZZLE_128B)
//     conv3  M = 128, N = 256, K = 64 from the t2 tile
//     epi3   affine + residual t + ReLU -> u (bf16, global)
//
// HBM per output pixel: t read once (512 B; the 1-pixel halo ring is re-read from L2) and u written
// once (512 B), instead of t, t1 (x2), t2 (x2), t (residual) and u with three unfused kernels
// (2048 B).  t1 / t2 are written to their band buffers only where somebody reads them later: the
// 2PS cache rows of t1 (FP pass), or all rows (the BP recompute, whose per-op backward reads them).
//
// Numerics equal the unfused kernels': conv1 accumulates K in the same order (16-channel MMA steps
// 0..255), every epilogue is fmaf(acc, gamma, beta) [+ bf16 residual with one rounding] -> RNE bf16
// with ReLU folded into the conversion, as k_conv_tc's.
//
// Warp roles (320 threads): 0 TMA producer, 1 MMA issuer, 2-5 epilogue A (epi1, epi2: one TMEM lane
// quarter each), 6-9 epilogue B (epi3).  Weights (136 KB) stay resident in shared memory for the
// whole launch.  TMEM: conv1 accumulators at columns [0, 128) (two M halves), conv2 [128, 192),
// conv3 [256, 512).  MMA issue order conv2(i), conv1(i+1), conv3(i): conv1 of the next tile runs
// while epilogue A converts t2 and conv3 while epilogue A converts the next t1.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "tc.hpp"
#include "tc_ptx.cuh"

namespace lrcnn {

namespace {

typedef __nv_bfloat16 bf16;

struct TcBneck {
    View t, t1, t2, u;
    const bf16 *g1, *e1, *g2, *e2, *g3, *e3;   // affine gamma / beta per conv
    int H, W, B;
    int a2, b2;              // output rows of t2 / u
    int a1, b1;              // t1 rows this band computes; rows < a1 are read from the t1 view (2PS cache)
    int tiles_x, tiles_y, num_tiles;
    int write_t2;            // store t2 rows [a2, b2)
    int nwin;                // store t1 rows in these windows (clipped to [a1, b1)); < 0: all rows
    int wlo[16], whi[16];
};


constexpr int kThreadsB = 512;   // producer, conv1 MMA, conv2/conv3 MMA, 4 epilogue-A warps, 8 epilogue-B warps, E3 DMA warp
constexpr int kW2 = 9 * 8192;          // 9 taps x (64 rows x 64 ch), SWIZZLE_128B (resident)
constexpr int kW3 = 256 * 128;         // 256 rows x 64 ch, SWIZZLE_128B (resident)
constexpr int kTBox = 180 * 64;        // TMA bytes per 32-channel t chunk of the 10 x 18 box
constexpr int kW1c = 64 * 64;          // the matching W1 chunk (64 rows x 32 ch, SWIZZLE_64B)
constexpr int kTRows = 184;            // box rows 0..179 (+4 read by the second M half, discarded)
constexpr int kH1 = 56;                // second M half: box rows 56..183 (8-row swizzle atoms)
constexpr int kTStage = 16384;         // 184 pixel rows x 64 B, then the W1 chunk at +12288
constexpr int kW1off = 12288;
constexpr int kTStages = 3;
constexpr int kT2 = 128 * 128;
constexpr int kRB = 4;                 // epilogue B: per-quarter residual / output ring of 32 px x 32 ch (2 KB, SWIZZLE_64B)
constexpr int kStgB = 4 * kRB * 2048;
constexpr int kPrm = 768 * 4;          // gamma / beta of the three convs (64 + 64 + 256 channels), fp32
constexpr int oW2 = 0, oW3 = oW2 + kW2, oT = oW3 + kW3, oT2 = oT + kTStages * kTStage, oStg = oT2 + kT2,
              oT1 = oStg + kStgB, oPrm = oT1 + 180 * 128, oBar = oPrm + kPrm;
constexpr int kSmemB = oBar + 512 + 1024;
static_assert(kSmemB <= 232448, "fused bottleneck: shared memory");
static_assert(oT % 1024 == 0 && oT1 % 1024 == 0 && oT2 % 1024 == 0 && oStg % 1024 == 0 && kTStage % 1024 == 0 &&
              kW1off >= kTRows * 64 && kW1off + kW1c <= kTStage, "swizzle atoms / stage layout");

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap *m, const void *src, int c0, int c1, int c2, int c3) {
    asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(ptx::smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read_n() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void named_bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
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
__device__ __forceinline__ uint32_t pack_relu(float lo, float hi) {
    uint32_t d;
    asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
    return d;
}
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
// 8 channels: relu(acc * gamma + beta) -> 4 bf16x2 words; gamma / beta fp32 in smem at sg / se
__device__ __forceinline__ uint4 affine_relu8(const uint32_t *v, uint32_t sg, uint32_t se) {
    const float4 g0 = lds_f4(sg), g1 = lds_f4(sg + 16), e0 = lds_f4(se), e1 = lds_f4(se + 16);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w}, e[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
    uint32_t o[4];
#pragma unroll
    for (int h = 0; h < 4; ++h)
        o[h] = pack_relu(fmaf(__uint_as_float(v[2 * h]), g[2 * h], e[2 * h]),
                         fmaf(__uint_as_float(v[2 * h + 1]), g[2 * h + 1], e[2 * h + 1]));
    return make_uint4(o[0], o[1], o[2], o[3]);
}
// 8 channels: relu(acc * gamma + beta + res) -> 4 bf16x2 words (k_conv_tc's epi_fast order)
__device__ __forceinline__ uint4 affine_res_relu8(const uint32_t *v, uint32_t sg, uint32_t se, uint4 r) {
    const float4 g0 = lds_f4(sg), g1 = lds_f4(sg + 16), e0 = lds_f4(se), e1 = lds_f4(se + 16);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w}, e[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
    const uint32_t rw[4] = {r.x, r.y, r.z, r.w};
    uint32_t o[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const float x0 = hadd_lo(rw[h], fmaf(__uint_as_float(v[2 * h]), g[2 * h], e[2 * h]));
        const float x1 = hadd_hi(rw[h], fmaf(__uint_as_float(v[2 * h + 1]), g[2 * h + 1], e[2 * h + 1]));
        o[h] = pack_relu(x0, x1);
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// mbarrier wait for roles off the critical path: back off between polls so that spinning warps do not
// take issue slots from the epilogue warps on the same scheduler
__device__ __forceinline__ void mbar_wait_sleep(uint64_t *bar, uint32_t parity) {
    uint32_t done;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, P1;\n\t}\n"
            : "=r"(done)
            : "r"(ptx::smem_u32(bar)), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(32);
    }
}

__device__ __forceinline__ void decode(const TcBneck &P, int tile, int &tx, int &ty, int &b) {
    tx = tile % P.tiles_x;
    const int r = tile / P.tiles_x;
    ty = r % P.tiles_y;
    b = r / P.tiles_y;
}

// bit r: t1 row y0 + r (r < n <= 17) is stored -- in [a1, b1) and in a window (nwin < 0: every row)
__device__ __forceinline__ uint32_t t1_row_mask(const TcBneck &P, int y0, int n) {
    auto span = [&](int lo, int hi) -> uint32_t {
        lo = max(max(lo, P.a1), y0);
        hi = min(min(hi, P.b1), y0 + n);
        return hi > lo ? (((1u << (hi - lo)) - 1u) << (lo - y0)) : 0u;
    };
    if (P.nwin < 0) return span(P.a1, P.b1);
    uint32_t m = 0;
    for (int i = 0; i < P.nwin; ++i) m |= span(P.wlo[i], P.whi[i]);
    return m;
}

}  // namespace

__global__ void __launch_bounds__(kThreadsB, 1)
    k_bneck_fwd(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmW1,
                const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmW3,
                const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmU, const TcBneck P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = (uint8_t *)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint64_t *bar = (uint64_t *)(smem + oBar);
    uint64_t *wbar = bar, *tfull = bar + 1, *tempty = tfull + kTStages;
    uint64_t *a1full = tempty + kTStages, *a1empty = a1full + 2;   // [2]: double-buffered conv1 accumulators
    uint64_t *t1full = a1full + 4, *t1empty = a1full + 5, *a2full = a1full + 6, *t2full = a1full + 7;
    uint64_t *t2empty = a1full + 8, *a3full = a1full + 9, *a3empty = a1full + 10;
    uint64_t *rbar = a1full + 11;                                   // [4 quarters][kRB] residual tiles landed
    uint64_t *rdone = rbar + 4 * kRB;                               // [4 quarters][kRB] output rows combined
    uint32_t *tslot = (uint32_t *)(rdone + 4 * kRB);
    // fp32 per-channel parameters: g1 @0, e1 @64, g2 @128, e2 @192, g3 @256, e3 @512 (floats)
    float *prm = reinterpret_cast<float *>(smem + oPrm);
    const uint32_t sprm = ptx::smem_u32(prm);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        ptx::mbar_init(wbar, 1);
        for (int i = 0; i < kTStages; ++i) { ptx::mbar_init(tfull + i, 1); ptx::mbar_init(tempty + i, 1); }
        for (int i = 0; i < 2; ++i) { ptx::mbar_init(a1full + i, 1); ptx::mbar_init(a1empty + i, 4); }
        ptx::mbar_init(t1full, 4); ptx::mbar_init(t1empty, 1); ptx::mbar_init(a2full, 1);
        ptx::mbar_init(t2full, 4); ptx::mbar_init(t2empty, 1);
        ptx::mbar_init(a3full, 1); ptx::mbar_init(a3empty, 8);
        for (int i = 0; i < 4 * kRB; ++i) { ptx::mbar_init(rbar + i, 1); ptx::mbar_init(rdone + i, 2); }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmT);
        ptx::prefetch_tmap(&tmW1);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *tslot;
    ptx::griddep_wait();
    ptx::griddep_launch();
    if (threadIdx.x >= 96) {   // per-channel parameters -> fp32 smem (the 256 epilogue threads, 3 each)
        for (int i = threadIdx.x - 96; i < 768; i += 256) {
            const bf16 *src = i < 64 ? P.g1 + i : i < 128 ? P.e1 + (i - 64) : i < 192 ? P.g2 + (i - 128)
                            : i < 256 ? P.e2 + (i - 192) : i < 512 ? P.g3 + (i - 256) : P.e3 + (i - 512);
            prm[i] = __bfloat162float(*src);
        }
    }
    __syncthreads();

    if (warp == 0) {
        if (lane == 0) {
            ptx::mbar_arrive_expect_tx(wbar, kW2 + kW3);
            for (int tap = 0; tap < 9; ++tap) ptx::tma_load_3d(smem + oW2 + tap * 8192, &tmW2, wbar, 0, tap, 0);
            ptx::tma_load_3d(smem + oW3, &tmW3, wbar, 0, 0, 0);
            int s = 0;
            uint32_t ph = 0;
            for (int tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x) {
                int tx, ty, b;
                decode(P, tile, tx, ty, b);
                const int y0 = P.a2 + ty * 16, x0 = tx * 8;
                for (int c = 0; c < 8; ++c) {
                    mbar_wait_sleep(tempty + s, ph ^ 1);
                    ptx::mbar_arrive_expect_tx(tfull + s, kTBox + kW1c);
                    ptx::tma_load_4d(smem + oT + s * kTStage, &tmT, tfull + s, c * 32, x0 - 1, y0 - 1 - P.t.base, b);
                    ptx::tma_load_3d(smem + oT + s * kTStage + kW1off, &tmW1, tfull + s, c * 32, 0, 0);
                    if (++s == kTStages) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // conv1 issuer: the t1 region of tile j into accumulator buffer j & 1 as soon as its loads land
        // and epi2 has drained the buffer's previous tile (j - 2; conv2 reuses the buffer)
        constexpr uint32_t id64 = ptx::idesc_bf16(128, 64, 0, 0);
        const uint64_t dT = ptx::smem_desc(ptx::smem_u32(smem + oT), 16, 512, 4);     // SWIZZLE_64B
        const uint32_t hT = (uint32_t)(dT >> 32);
        int s = 0, j = 0;
        uint32_t ph = 0;
        for (int tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x, ++j) {
            const uint32_t acc = tmem + (j & 1) * 128;
            mbar_wait_sleep(a1empty + (j & 1), ((j >> 1) & 1) ^ 1);
            ptx::tc_fence_after();
            for (int c = 0; c < 8; ++c) {
                ptx::mbar_wait(tfull + s, ph);
                ptx::tc_fence_after();
                if (ptx::elect_one()) {
                    const uint32_t a0 = (uint32_t)dT + s * (kTStage >> 4), b0 = a0 + (kW1off >> 4);
#pragma unroll
                    for (int h = 0; h < 2; ++h)
#pragma unroll
                        for (int kk = 0; kk < 2; ++kk)
                            ptx::umma_bf16_1t(acc + h * 64, a0 + h * (kH1 * 64 >> 4) + 2 * kk, hT, b0 + 2 * kk, hT, id64,
                                              (c | kk) != 0);
                    ptx::umma_commit_1t(tempty + s);
                    if (c == 7) ptx::umma_commit_1t(a1full + (j & 1));
                }
                __syncwarp();
                if (++s == kTStages) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 2) {
        // conv2 (into the drained conv1 buffer j & 1, its columns 0..63) and conv3 (columns 256..511)
        constexpr uint32_t id64 = ptx::idesc_bf16(128, 64, 0, 0), id256 = ptx::idesc_bf16(128, 256, 0, 0);
        const uint64_t dT1 = ptx::smem_desc_sw128(ptx::smem_u32(smem + oT1), 16, 10 * 128);
        const uint64_t dW2 = ptx::smem_desc_sw128(ptx::smem_u32(smem + oW2), 16, 1024);
        const uint64_t dT2 = ptx::smem_desc_sw128(ptx::smem_u32(smem + oT2), 16, 1024);
        const uint64_t dW3 = ptx::smem_desc_sw128(ptx::smem_u32(smem + oW3), 16, 1024);
        const uint32_t hT1 = (uint32_t)(dT1 >> 32), hW2 = (uint32_t)(dW2 >> 32), hT2 = (uint32_t)(dT2 >> 32),
                       hW3 = (uint32_t)(dW3 >> 32);
        ptx::mbar_wait(wbar, 0);
        ptx::tc_fence_after();
        int j = 0;
        for (int tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x, ++j) {
            mbar_wait_sleep(t1full, j & 1);   // epi1 wrote the t1 box and drained conv1 buffer j & 1
            ptx::tc_fence_after();
            const uint32_t acc2 = tmem + (j & 1) * 128;
            if (ptx::elect_one()) {
#pragma unroll 1
                for (int tap = 0; tap < 9; ++tap) {
                    const int ky = tap / 3, kx = tap - 3 * ky;
                    const uint32_t a0 = (uint32_t)dT1 + (uint32_t)(ky * 10 + kx) * 8, b0 = (uint32_t)dW2 + tap * (8192 >> 4);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        ptx::umma_bf16_1t(acc2, a0 + 2 * kk, hT1, b0 + 2 * kk, hW2, id64, (tap | kk) != 0);
                }
                ptx::umma_commit_1t(t1empty);
                ptx::umma_commit_1t(a2full);
            }
            __syncwarp();
            mbar_wait_sleep(t2full, j & 1);
            mbar_wait_sleep(a3empty, (j & 1) ^ 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                    ptx::umma_bf16_1t(tmem + 256, (uint32_t)dT2 + 2 * kk, hT2, (uint32_t)dW3 + 2 * kk, hW3, id256, kk != 0);
                ptx::umma_commit_1t(t2empty);
                ptx::umma_commit_1t(a3full);
            }
            __syncwarp();
        }
    } else if (warp < 7) {
        // ---------------------------------------------------------------- epilogue A: t1 box, t2 tile
        const int q = warp & 3, m = q * 32 + lane, ta = threadIdx.x - 96;   // ta: 0..127 within the group
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t sT1 = ptx::smem_u32(smem + oT1), sT2 = ptx::smem_u32(smem + oT2);
        const bf16 *t1p = (const bf16 *)P.t1.p;
        int j = 0;
        for (int tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x, ++j) {
            int tx, ty, b;
            decode(P, tile, tx, ty, b);
            const int y0 = P.a2 + ty * 16, x0 = tx * 8;
            const bool last_row = ty == P.tiles_y - 1;
            // epi1: conv1 buffer j & 1 (two M halves) -> the t1 box
            const uint32_t acc = tq + (j & 1) * 128;
            mbar_wait_sleep(a1full + (j & 1), (j >> 1) & 1);
            ptx::tc_fence_after();
            mbar_wait_sleep(t1empty, (j & 1) ^ 1);   // conv2 of the previous tile has read the box
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                uint32_t v[64];
                ptx::tmem_ld32(acc + h * 64, *reinterpret_cast<uint32_t(*)[32]>(v));
                ptx::tmem_ld32(acc + h * 64 + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
                ptx::tmem_ld_wait();
                const int p = h * kH1 + m;   // box row of this TMEM lane (half 1 starts at row 56)
                if (h == 0 || (p >= 128 && p < 180)) {
                    const int ry = p / 10, rx = p - ry * 10;
                    const int y = y0 - 1 + ry, x = x0 - 1 + rx;
                    uint4 o[8];
                    if (y < 0 || y >= P.H || x < 0 || x >= P.W) {
#pragma unroll
                        for (int c = 0; c < 8; ++c) o[c] = make_uint4(0, 0, 0, 0);
                    } else if (y < P.a1) {   // 2PS cache rows of t1 (band r-1's), in the t1 band buffer
                        const uint4 *src = reinterpret_cast<const uint4 *>(
                            t1p + (long long)b * P.t1.bs + ((long long)(y - P.t1.base) * P.W + x) * 64);
#pragma unroll
                        for (int c = 0; c < 8; ++c) o[c] = src[c];
                    } else {
#pragma unroll
                        for (int c = 0; c < 8; ++c) o[c] = affine_relu8(v + 8 * c, sprm + 32 * c, sprm + 256 + 32 * c);
                    }
                    const uint32_t row = sT1 + p * 128;
#pragma unroll
                    for (int c = 0; c < 8; ++c) st_shared_v4(row + ((c ^ (p & 7)) << 4), o[c]);
                }
            }
            fence_proxy_async();
            ptx::tc_fence_before();
            named_bar_sync(1, 128);   // the whole t1 box is written (read back below by other warps)
            if (lane == 0) ptx::mbar_arrive(t1full);
            // t1 rows a later reader needs (2PS cache windows / all): this tile's centre columns, rows
            // y0 .. y0+15 (+ y0+16 on the last tile row), coalesced: 16-byte items (row, pixel, chunk)
            {
                const int nrows = last_row ? 17 : 16;
                const uint32_t rmask = t1_row_mask(P, y0, nrows);   // rows of this tile to store
#pragma unroll 1
                for (int it = ta; rmask && it < nrows * 64; it += 128) {
                    const int rr = it >> 6, px = (it >> 3) & 7, c = it & 7;
                    const int y = y0 + rr, x = x0 + px;
                    if (x < P.W && ((rmask >> rr) & 1)) {
                        const int p = (rr + 1) * 10 + px + 1;
                        const uint4 v = ld_shared_v4(sT1 + p * 128 + ((c ^ (p & 7)) << 4));
                        *reinterpret_cast<uint4 *>((bf16 *)P.t1.p + (long long)b * P.t1.bs +
                                                  ((long long)(y - P.t1.base) * P.W + x) * 64 + c * 8) = v;
                    }
                }
            }
            named_bar_sync(1, 128);   // every warp is done reading the box before the next tile's epi1 writes it
            // epi2 (conv2 accumulated into buffer j & 1; reading it frees the buffer for conv1 of tile j + 2)
            mbar_wait_sleep(a2full, j & 1);
            ptx::tc_fence_after();
            {
                uint32_t v[64];
                ptx::tmem_ld32(acc, *reinterpret_cast<uint32_t(*)[32]>(v));
                ptx::tmem_ld32(acc + 32, *reinterpret_cast<uint32_t(*)[32]>(v + 32));
                ptx::tmem_ld_wait();
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(a1empty + (j & 1));
                mbar_wait_sleep(t2empty, (j & 1) ^ 1);
                const uint32_t row = sT2 + m * 128;
#pragma unroll
                for (int c = 0; c < 8; ++c) st_shared_v4(row + ((c ^ (m & 7)) << 4), affine_relu8(v + 8 * c, sprm + 512 + 32 * c, sprm + 768 + 32 * c));
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(t2full);
            if (P.write_t2) {   // this warp's 32 pixels (tile rows 4q .. 4q+3), coalesced 128 B per pixel
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int pm = q * 32 + 4 * k + (lane >> 3), c = lane & 7;
                    const int y = y0 + (pm >> 3), x = x0 + (pm & 7);
                    if (y < P.b2 && x < P.W) {
                        const uint4 v = ld_shared_v4(sT2 + pm * 128 + ((c ^ (pm & 7)) << 4));
                        *reinterpret_cast<uint4 *>((bf16 *)P.t2.p + (long long)b * P.t2.bs +
                                                  ((long long)(y - P.t2.base) * P.W + x) * 64 + c * 8) = v;
                    }
                }
            }
        }
    } else if (warp < 15) {
        // ---------------------------------------------------------------- epilogue B: u = relu(affine(conv3) + t)
        // Eight warps, two per TMEM lane quarter q (the tile's pixels 32q..32q+31 = tile rows 4q..4q+3);
        // warp half hf combines channels 16hf..16hf+15 of every 32-channel group in place in the quarter's
        // ring buffer (the residual box: t at those pixels, 32 ch x 8 x 4, SWIZZLE_64B) and signals rdone;
        // the DMA warp (15) TMA-stores the group and refills the buffer kRB groups ahead, so the combining
        // warps never wait on a store.  The next group's accumulator columns are loaded from TMEM while this
        // group is combined.
        const int q = warp & 3, hf = (warp - 7) >> 2;
        const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16) + 256 + hf * 16;
        uint64_t *wb = rbar + q * kRB, *wd = rdone + q * kRB;
        uint8_t *ring = smem + oStg + q * kRB * 2048;
        int sb = 0;
        uint32_t rph = 0;   // bit i: parity of wb[i]'s next completion
        int j = 0;
        for (int tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x, ++j) {
            mbar_wait_sleep(a3full, j & 1);
            ptx::tc_fence_after();
            uint32_t v[2][16];
            ptx::tmem_ld16(tq, v[0]);
#pragma unroll
            for (int g = 0; g < 8; ++g) {
                ptx::tmem_ld_wait();
                if (g < 7) ptx::tmem_ld16(tq + (g + 1) * 32, v[(g + 1) & 1]);
                if (g == 7) {
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(a3empty);
                }
                const uint32_t row = ptx::smem_u32(ring + sb * 2048) + lane * 64;
                ptx::mbar_wait(wb + sb, (rph >> sb) & 1);
                rph ^= 1u << sb;
#pragma unroll
                for (int c2 = 0; c2 < 2; ++c2) {
                    const int c = 2 * hf + c2;
                    const uint32_t a = row + ((c ^ ((lane >> 1) & 3)) << 4);
                    st_shared_v4(a, affine_res_relu8(v[g & 1] + 8 * c2, sprm + 1024 + 128 * g + 32 * c,
                                                     sprm + 2048 + 128 * g + 32 * c, ld_shared_v4(a)));
                }
                fence_proxy_async();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(wd + sb);
                sb = sb + 1 == kRB ? 0 : sb + 1;
            }
        }
    } else if (lane == 0) {
        // ---------------------------------------------------------------- E3 DMA (warp 15): residual loads, u stores
        // group sequence k = (tile, g): buffer k % kRB of every quarter; the residual of group k + kRB - 1 goes
        // into buffer (k - 1) % kRB once group k - 1's stores have read it
        auto coords = [&](int tile, int qq, int &x, int &yt, int &yu, int &bb) {
            int tx, ty;
            decode(P, tile, tx, ty, bb);
            x = tx * 8;
            yt = P.a2 + ty * 16 + 4 * qq - P.t.base;
            yu = P.a2 + ty * 16 + 4 * qq - P.u.base;
        };
        int lt = blockIdx.x, lg = 0;   // next residual group to load
        auto load_next = [&](int buf) {
            for (int qq = 0; qq < 4; ++qq) {
                int x, yt, yu, bb;
                coords(lt, qq, x, yt, yu, bb);
                ptx::mbar_arrive_expect_tx(rbar + qq * kRB + buf, 2048);
                ptx::tma_load_4d(smem + oStg + (qq * kRB + buf) * 2048, &tmR, rbar + qq * kRB + buf, lg * 32, x, yt, bb);
            }
            if (++lg == 8) { lg = 0; lt += gridDim.x; }
        };
        for (int i = 0; i < kRB - 1 && lt < P.num_tiles; ++i) load_next(i);
        int sb = 0;
        uint32_t dph = 0;
        for (int tile = blockIdx.x; tile < P.num_tiles; tile += gridDim.x) {
            for (int g = 0; g < 8; ++g) {
                for (int qq = 0; qq < 4; ++qq) {
                    int x, yt, yu, bb;
                    coords(tile, qq, x, yt, yu, bb);
                    ptx::mbar_wait(rdone + qq * kRB + sb, (dph >> sb) & 1);
                    tma_store_4d(&tmU, smem + oStg + (qq * kRB + sb) * 2048, g * 32, x, yu, bb);
                }
                dph ^= 1u << sb;
                bulk_commit();
                if (lt < P.num_tiles) {   // group k-1's stores have read buffer (k-1) % kRB
                    bulk_wait_read_n<1>();
                    load_next(sb == 0 ? kRB - 1 : sb - 1);
                }
                sb = sb + 1 == kRB ? 0 : sb + 1;
            }
        }
        bulk_wait_all();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// ------------------------------------------------------------------ host launcher
bool tc_bneck_fwd(const BneckArgs &A, cudaStream_t st) {
    const View &t = A.t, &t1 = A.t1, &t2 = A.t2, &u = A.u;
    if (t.Cp != 256 || t1.Cp != 64 || t2.Cp != 64 || u.Cp != 256) return false;
    if (t.W != u.W || t1.W != u.W || t2.W != u.W || t.H != u.H || t1.H != u.H || t2.H != u.H) return false;
    const void *ptrs[] = {t.p, t1.p, u.p, A.w1, A.w2, A.w3, A.g1, A.e1, A.g2, A.e2, A.g3, A.e3};
    for (const void *p : ptrs)
        if (!p || ((uintptr_t)p & 15)) return false;
    if (A.write_t2 && (!t2.p || ((uintptr_t)t2.p & 15))) return false;
    if (A.nwin > 16) return false;
    const int rows = A.b2 - A.a2;
    if (rows <= 0 || u.W <= 0) return true;
    // preconditions of the row bookkeeping: t1 rows [a2-1, a1) are held by the t1 view (2PS cache),
    // t rows [a1, b1) by the t view, u / t2 rows [a2, b2) by theirs
    if (A.a1 > A.a2 + 1 || A.b1 > A.b2 + 1 || A.b1 < A.b2) return false;
    const int cl = A.a2 > 0 ? A.a2 - 1 : 0;   // first t1 row the band's 3x3 reads
    if (A.a1 > cl && (cl < t1.base || A.a1 > t1.base + t1.rows)) return false;
    if (A.a1 < t.base || A.b1 > t.base + t.rows || A.a2 < u.base || A.b2 > u.base + u.rows) return false;
    TcBneck P{};
    P.t = t; P.t1 = t1; P.t2 = t2; P.u = u;
    P.g1 = (const bf16 *)A.g1; P.e1 = (const bf16 *)A.e1;
    P.g2 = (const bf16 *)A.g2; P.e2 = (const bf16 *)A.e2;
    P.g3 = (const bf16 *)A.g3; P.e3 = (const bf16 *)A.e3;
    P.H = u.H; P.W = u.W; P.B = A.B;
    P.a2 = A.a2; P.b2 = A.b2; P.a1 = A.a1; P.b1 = A.b1;
    P.tiles_x = (u.W + 7) / 8;
    P.tiles_y = (rows + 15) / 16;
    P.num_tiles = A.B * P.tiles_x * P.tiles_y;
    P.write_t2 = A.write_t2;
    P.nwin = A.nwin;
    for (int i = 0; i < A.nwin && i < 16; ++i) { P.wlo[i] = A.wlo[i]; P.whi[i] = A.whi[i]; }
    CUtensorMap mT, mW1, mW2, mW3, mR, mU;
    if (!tc_encode_view(&mT, t, A.B, 10, 18, 1, 32)) return false;
    if (!tc_encode_view(&mR, t, A.B, 8, 4, 1, 32)) return false;
    View uc = u;
    uc.rows = A.b2 - u.base;   // the store clips at the band's last output row
    if (!tc_encode_view(&mU, uc, A.B, 8, 4, 1, 32)) return false;
    if (!tc_encode_w(&mW1, A.w1, 64, 1, 256, 64, 32)) return false;
    if (!tc_encode_w(&mW2, A.w2, 64, 9, 64, 64, 64)) return false;
    if (!tc_encode_w(&mW3, A.w3, 256, 1, 64, 256, 64)) return false;
    if (!tc_smem_attr((const void *)k_bneck_fwd, kSmemB)) return false;
    const int grid = P.num_tiles < tc_num_sms() ? P.num_tiles : tc_num_sms();
    return tc_launch(k_bneck_fwd, grid, kThreadsB, kSmemB, st, mT, mW1, mW2, mW3, mR, mU, P);
}

}  // namespace lrcnn

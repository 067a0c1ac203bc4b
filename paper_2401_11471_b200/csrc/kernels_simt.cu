// kernels_simt.cu -- CUDA-core kernels of the row-centric path.
//
// These serve the fp32 parity mode (the tensor-core formats cannot meet the
// 1e-5 bar), the small ops around the convolutions (max-pool,
// residual add, bias/affine reductions, head, SGD) and the shapes the
// tcgen05 kernels do not take.  Every kernel works on band Views
// (kernels.hpp) so the semi-closed padding rule is a bounds
// test on the GLOBAL row index, never on the band edge.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <mutex>
#include <set>

#include <algorithm>
#include <cstdlib>
#include <utility>

#include "kernels.hpp"

namespace lrcnn {

// programmatic dependent launch (see conv_tc.cu launch_pdl): every kernel of this file waits for
// the preceding grid at its first statement, so it may be launched while that grid drains.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
static thread_local bool g_simt_pdl_off = false;   // per-launch profiling (see tc_set_pdl)
void simt_set_pdl(bool on) { g_simt_pdl_off = !on; }
static int simt_pdl() {
    static int v = -1;
    if (v < 0) { const char *e = getenv("LRCNN_PDL"); v = e && *e ? atoi(e) : 1; }
    return v && !g_simt_pdl_off;
}
template <typename... KArgs, typename... Args>
static void launch_simt(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = simt_pdl() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}


typedef __nv_bfloat16 bf16;

__device__ __forceinline__ float ldf(const float *p) { return *p; }
__device__ __forceinline__ float ldf(const bf16 *p) { return __bfloat162float(*p); }
__device__ __forceinline__ void stf(float *p, float v) { *p = v; }
__device__ __forceinline__ void stf(bf16 *p, float v) { *p = __float2bfloat16_rn(v); }

__device__ __forceinline__ bool vhas(const View &v, int g) {
    return g >= 0 && g < v.H && g >= v.base && g < v.base + v.rows;
}
__device__ __forceinline__ long long voff(const View &v, int b, int g, int x) {
    return (long long)b * v.bs + ((long long)(g - v.base) * v.W + x) * v.Cp;
}

// ------------------------------------------------------------------ conv forward
template <typename T>
__global__ void k_conv_fwd(ConvFwdArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int Cpo = A.out.Cp, Wo = A.out.W, rows = A.b_ - A.a, Cin = A.in.Cp;
    long long n = (long long)A.B * rows * Wo * Cpo;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int co = idx % Cpo;
        long long r = idx / Cpo;
        int x = r % Wo; r /= Wo;
        int y = A.a + (int)(r % rows);
        int b = (int)(r / rows);
        float acc = 0.f;
        if (co < A.c_out) {
            const T *in = (const T *)A.in.p;
            const T *w = (const T *)A.w;
            for (int ky = 0; ky < A.k; ++ky) {
                int g = y * A.s - A.p + ky;
                if (!vhas(A.in, g)) continue;
                for (int kx = 0; kx < A.k; ++kx) {
                    int xi = x * A.s - A.p + kx;
                    if (xi < 0 || xi >= A.in.W) continue;
                    const T *ip = in + voff(A.in, b, g, xi);
                    const T *wp = w + ((long long)(co * A.k + ky) * A.k + kx) * Cin;
                    for (int ci = 0; ci < Cin; ++ci) acc += ldf(wp + ci) * ldf(ip + ci);
                }
            }
            if (A.epi == 1) acc += ldf((const T *)A.b + co);
            else if (A.epi == 2) acc = ldf((const T *)A.b + co) * acc + ldf((const T *)A.beta + co);
            if (A.res.p) acc += ldf((const T *)A.res.p + voff(A.res, b, y, x) + co);
            if (A.relu) acc = fmaxf(acc, 0.f);
        }
        stf((T *)A.out.p + voff(A.out, b, y, x) + co, acc);
    }
}

// ------------------------------------------------------------------ conv dgrad
// dx[b,g,xi,ci] = gate(act) * (dx + sum_{co,ky,kx} w[co,ky,kx,ci] * gamma[co] * dy[b,y,x,co]),
// y*s - p + ky = g.  Gating on write is idempotent (mask in {0,1}), so partial sums
// (2PS carry rows, several consumers) may be gated more than once.
template <typename T>
__global__ void k_conv_dgrad(DgradArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int Cin = A.dx.Cp, Wi = A.dx.W, rows = A.rb - A.ra, Wo = A.dy.W, Cpo = A.dy.Cp;
    long long n = (long long)A.B * rows * Wi * Cin;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int ci = idx % Cin;
        long long r = idx / Cin;
        int xi = r % Wi; r /= Wi;
        int g = A.ra + (int)(r % rows);
        int b = (int)(r / rows);
        const T *w = (const T *)A.w;
        const T *dy = (const T *)A.dy.p;
        float acc = 0.f;
        for (int ky = 0; ky < A.k; ++ky) {
            int num = g + A.p - ky;
            if (num < 0 || num % A.s) continue;
            int y = num / A.s;
            if (!vhas(A.dy, y)) continue;
            for (int kx = 0; kx < A.k; ++kx) {
                int nx = xi + A.p - kx;
                if (nx < 0 || nx % A.s) continue;
                int x = nx / A.s;
                if (x >= Wo) continue;
                const T *dp = dy + voff(A.dy, b, y, x);
                const T *wp = w + ((long long)ky * A.k + kx) * Cin + ci;
                const long long wstride = (long long)A.k * A.k * Cin;
                for (int co = 0; co < A.c_out; ++co) {
                    float d = ldf(dp + co);
                    if (A.gamma) d *= ldf((const T *)A.gamma + co);
                    acc += ldf(wp + co * wstride) * d;
                }
            }
        }
        (void)Cpo;
        T *dx = (T *)A.dx.p + voff(A.dx, b, g, xi) + ci;
        float v = (A.write ? 0.f : ldf(dx)) + acc;
        if (A.gate && ldf((const T *)A.act.p + voff(A.act, b, g, xi) + ci) <= 0.f) v = 0.f;
        stf(dx, v);
    }
}

// ------------------------------------------------------------------ conv wgrad
// dw[co,ky,kx,ci] += gamma[co] * sum_{b, y in [a,b), x} dy[b,y,x,co] * x[b, y*s-p+ky, x*s-p+kx, ci]
// one block per (co, ky, kx), threads over ci x pixel slices, block reduction.
template <typename T>
__global__ void k_conv_wgrad(WgradArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int Cin = A.x.Cp, Wo = A.dy.W, rows = A.b - A.a;
    const int co = blockIdx.x / (A.k * A.k), kk = blockIdx.x % (A.k * A.k);
    const int ky = kk / A.k, kx = kk % A.k;
    const int ci = blockIdx.y * 32 + (threadIdx.x & 31);
    const int lane_grp = threadIdx.x >> 5, ngrp = blockDim.x >> 5;
    __shared__ float red[32][33];
    float acc = 0.f;
    if (ci < Cin) {
        long long npix = (long long)A.B * rows * Wo;
        for (long long q = lane_grp; q < npix; q += ngrp) {
            int x = q % Wo;
            long long r = q / Wo;
            int y = A.a + (int)(r % rows);
            int b = (int)(r / rows);
            int g = y * A.s - A.p + ky, xi = x * A.s - A.p + kx;
            if (!vhas(A.x, g) || xi < 0 || xi >= A.x.W) continue;
            float d = ldf((const T *)A.dy.p + voff(A.dy, b, y, x) + co);
            acc += d * ldf((const T *)A.x.p + voff(A.x, b, g, xi) + ci);
        }
    }
    red[lane_grp][threadIdx.x & 31] = acc;
    __syncthreads();
    if (lane_grp == 0) {
        float s = 0.f;
        if (ci < Cin)
            for (int j = 0; j < ngrp; ++j) s += red[j][threadIdx.x & 31];
        const long long wi = ((long long)(co * A.k + ky) * A.k + kx) * Cin + ci;
        if (A.dg) {   // dgamma[co] += sum_{tap,ci} W * (sum_p dy x): exact for any gamma (incl. 0)
            float g = ci < Cin ? s * ldf((const T *)A.w + wi) : 0.f;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
            if ((threadIdx.x & 31) == 0) atomicAdd(A.dg + co, g);
        }
        if (ci < Cin) {
            if (A.gamma) s *= ldf((const T *)A.gamma + co);
            A.dw[wi] += s;
        }
    }
}

template <typename T>
__device__ __forceinline__ void ld8(const T *p, float (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = ldf(p + j);
}
__device__ __forceinline__ void ld8(const bf16 *p, float (&v)[8]) {
    uint4 u = *reinterpret_cast<const uint4 *>(p);
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) { float2 f = __bfloat1622float2(h[j]); v[2 * j] = f.x; v[2 * j + 1] = f.y; }
}
template <typename T>
__device__ __forceinline__ void st8(T *p, const float (&v)[8]) {
#pragma unroll
    for (int j = 0; j < 8; ++j) stf(p + j, v[j]);
}
__device__ __forceinline__ void st8(bf16 *p, const float (&v)[8]) {
    uint4 u;
    __nv_bfloat162 *h = reinterpret_cast<__nv_bfloat162 *>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
    *reinterpret_cast<uint4 *>(p) = u;
}

// ------------------------------------------------------------------ bias / beta grads
// db[c] += sum_pixels dy[p, c]: the bias (BIAS) or beta (AFFINE) gradient of a conv whose wgrad
// kernel did not fuse it.  (dgamma is always taken by the wgrad as sum_{tap,ci} W * (sum_p dy x),
// exact for any gamma -- never recovered from the stored output, which divides by gamma.)
// Block = (channel vectors of 8) x (pixel lanes); coalesced 8-channel loads, per-thread partial
// sums, smem reduction over pixel lanes, one fp32 atomicAdd per channel per block.
template <typename T>
__device__ __forceinline__ void acc8(const uint4 &u, float (&s)[8]) {
    const __nv_bfloat162 *h = reinterpret_cast<const __nv_bfloat162 *>(&u);
#pragma unroll
    for (int j = 0; j < 4; ++j) { float2 f = __bfloat1622float2(h[j]); s[2 * j] += f.x; s[2 * j + 1] += f.y; }
}

template <typename T>
__global__ void __launch_bounds__(256, 4) k_param_grad(ParamGradArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    // blockDim.x channel vectors (8 channels each) of group blockIdx.y; blockDim.y pixel lanes
    const int CV = blockDim.x, cv = threadIdx.x, py = threadIdx.y, PY = blockDim.y;
    const int rows = A.b - A.a, W = A.dy.W, c0 = (blockIdx.y * CV + cv) * 8;
    const bool live = c0 < A.dy.Cp;
    const int RW = rows * W;                        // band pixels per image (contiguous rows)
    float s0[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) s0[j] = 0.f;
    // pixel q = b * RW + p walks with stride S; (b, p) updated without division
    const int S = gridDim.x * PY;
    const int q0 = blockIdx.x * PY + py;
    int b = q0 / RW, p = q0 - b * RW;
    // advance by S pixels: (b, p) += (S / RW, S % RW) with one carry (the stride can span many
    // images when the band is thin)
    const int Sb = S / RW, Sp = S - Sb * RW;
    auto advance = [&]() { p += Sp; b += Sb; if (p >= RW) { p -= RW; ++b; } };
    const T *dbase = (const T *)A.dy.p + voff(A.dy, 0, A.a, 0) + c0;
    if constexpr (sizeof(T) == 2) {
        // bf16: raw 16-byte vectors, two pixels in flight per thread
        const uint4 z = make_uint4(0, 0, 0, 0);
        while (live && b < A.B) {
            const int b0 = b, p0 = p;
            advance();
            const bool two = b < A.B;
            const int b1 = b, p1 = p;
            if (two) advance();
            const uint4 d0 = *reinterpret_cast<const uint4 *>(dbase + (long long)b0 * A.dy.bs + (long long)p0 * A.dy.Cp);
            const uint4 d1 = two ? *reinterpret_cast<const uint4 *>(dbase + (long long)b1 * A.dy.bs + (long long)p1 * A.dy.Cp) : z;
            acc8<T>(d0, s0);
            acc8<T>(d1, s0);
        }
    } else {
        while (live && b < A.B) {
            float d[8];
            ld8(dbase + (long long)b * A.dy.bs + (long long)p * A.dy.Cp, d);
#pragma unroll
            for (int j = 0; j < 8; ++j) s0[j] += d[j];
            advance();
        }
    }
    extern __shared__ float red[];   // [PY][CV*8]
#pragma unroll
    for (int j = 0; j < 8; ++j) red[py * CV * 8 + cv * 8 + j] = s0[j];
    __syncthreads();
    for (int c = py * CV + cv; c < CV * 8; c += PY * CV) {
        float a0 = 0.f;
        for (int k = 0; k < PY; ++k) a0 += red[k * CV * 8 + c];
        const int ch = blockIdx.y * CV * 8 + c;
        if (ch < A.c_out) atomicAdd(A.db + ch, a0);
    }
}

// ------------------------------------------------------------------ 2x2/s2 max-pool (VGG), 8 channels per thread
// window order (0,0),(0,1),(1,0),(1,1) = raster order; strict '>' keeps the first maximum
// grid: x = (output column, channel vector) chunks of one output row, y = (image, row) of the band
template <typename T>
__global__ void k_pool2_fwd(PoolArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int CV = A.out.Cp / 8, Wo = A.out.W, rows = A.b - A.a;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Wo * CV) return;
    const int x = i / CV, cv = i - x * CV;
    const int b = blockIdx.y / rows, y = A.a + (int)(blockIdx.y - b * rows);
    const T *ip = (const T *)A.in.p + voff(A.in, b, 2 * y, 2 * x) + cv * 8;
    const long long rs = (long long)A.in.W * A.in.Cp;
    float best[8], v[8];
    ld8(ip, best);
    const long long off[3] = {A.in.Cp, rs, rs + A.in.Cp};
#pragma unroll
    for (int w = 0; w < 3; ++w) {
        ld8(ip + off[w], v);
#pragma unroll
        for (int j = 0; j < 8; ++j) best[j] = v[j] > best[j] ? v[j] : best[j];
    }
    st8((T *)A.out.p + voff(A.out, b, y, x) + cv * 8, best);
}

template <typename T>
__global__ void k_pool2_bwd(PoolArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int CV = A.dy.Cp / 8, Wo = A.dy.W, rows = A.b - A.a;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Wo * CV) return;
    const int x = i / CV, cv = i - x * CV;
    const int b = blockIdx.y / rows, y = A.a + (int)(blockIdx.y - b * rows);
    float d[8], v[4][8], best[8];
    int arg[8];
    ld8((const T *)A.dy.p + voff(A.dy, b, y, x) + cv * 8, d);
    const T *ap = (const T *)A.act.p + voff(A.act, b, 2 * y, 2 * x) + cv * 8;
    T *dp0 = (T *)A.dx.p + voff(A.dx, b, 2 * y, 2 * x) + cv * 8;
    const long long ars = (long long)A.act.W * A.act.Cp, drs = (long long)A.dx.W * A.dx.Cp;
#pragma unroll
    for (int w = 0; w < 4; ++w) ld8(ap + (w >> 1) * ars + (w & 1) * A.act.Cp, v[w]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        best[j] = v[0][j]; arg[j] = 0;
#pragma unroll
        for (int w = 1; w < 4; ++w)
            if (v[w][j] > best[j]) { best[j] = v[w][j]; arg[j] = w; }
    }
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        T *dp = dp0 + (w >> 1) * drs + (w & 1) * A.dx.Cp;
        float o[8];
        if (A.acc) ld8(dp, o);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            o[j] = (A.acc ? o[j] : 0.f) + (arg[j] == w ? d[j] : 0.f);
            if (A.gate && !(v[w][j] > 0.f)) o[j] = 0.f;
        }
        st8(dp, o);
    }
}

// ------------------------------------------------------------------ max-pool
template <typename T>
__device__ __forceinline__ void pool_window(const View &in, int b, int y, int x, int c, int k, int s, int p,
                                            float &best, int &bg, int &bx) {
    best = 0.f; bg = -1; bx = -1;
    for (int ky = 0; ky < k; ++ky) {
        int g = y * s - p + ky;
        if (!vhas(in, g)) continue;
        for (int kx = 0; kx < k; ++kx) {
            int xi = x * s - p + kx;
            if (xi < 0 || xi >= in.W) continue;
            float v = ldf((const T *)in.p + voff(in, b, g, xi) + c);
            if (bg < 0 || v > best) { best = v; bg = g; bx = xi; }
        }
    }
}

template <typename T>
__global__ void k_pool_fwd(PoolArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int Cp = A.out.Cp, Wo = A.out.W, rows = A.b - A.a;
    long long n = (long long)A.B * rows * Wo * Cp;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int c = idx % Cp;
        long long r = idx / Cp;
        int x = r % Wo; r /= Wo;
        int y = A.a + (int)(r % rows);
        int b = (int)(r / rows);
        float best; int bg, bx;
        pool_window<T>(A.in, b, y, x, c, A.k, A.s, A.p, best, bg, bx);
        stf((T *)A.out.p + voff(A.out, b, y, x) + c, bg < 0 ? 0.f : best);
    }
}

template <typename T>
__global__ void k_pool_bwd(PoolArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int Cp = A.dx.Cp, Wi = A.dx.W, rows = A.rb - A.ra, Wo = A.dy.W;
    long long n = (long long)A.B * rows * Wi * Cp;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int c = idx % Cp;
        long long r = idx / Cp;
        int xi = r % Wi; r /= Wi;
        int g = A.ra + (int)(r % rows);
        int b = (int)(r / rows);
        float acc = 0.f;
        for (int ky = 0; ky < A.k; ++ky) {
            int num = g + A.p - ky;
            if (num < 0 || num % A.s) continue;
            int y = num / A.s;
            if (!vhas(A.dy, y)) continue;
            for (int kx = 0; kx < A.k; ++kx) {
                int nx = xi + A.p - kx;
                if (nx < 0 || nx % A.s) continue;
                int x = nx / A.s;
                if (x >= Wo) continue;
                float best; int bg, bx;
                pool_window<T>(A.act, b, y, x, c, A.k, A.s, A.p, best, bg, bx);
                if (bg == g && bx == xi) acc += ldf((const T *)A.dy.p + voff(A.dy, b, y, x) + c);
            }
        }
        T *dx = (T *)A.dx.p + voff(A.dx, b, g, xi) + c;
        float v = ldf(dx) + acc;
        if (A.gate && ldf((const T *)A.act.p + voff(A.act, b, g, xi) + c) <= 0.f) v = 0.f;
        stf(dx, v);
    }
}

// ------------------------------------------------------------------ residual add, gated accumulate
template <typename T>
__global__ void k_add_fwd(EltArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int Cp = A.out.Cp, W = A.out.W, rows = A.b - A.a;
    long long n = (long long)A.B * rows * W * Cp;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int c = idx % Cp;
        long long r = idx / Cp;
        int x = r % W; r /= W;
        int y = A.a + (int)(r % rows);
        int b = (int)(r / rows);
        float v = ldf((const T *)A.x0.p + voff(A.x0, b, y, x) + c) + ldf((const T *)A.x1.p + voff(A.x1, b, y, x) + c);
        if (A.relu) v = fmaxf(v, 0.f);
        stf((T *)A.out.p + voff(A.out, b, y, x) + c, v);
    }
}

template <typename T>
__global__ void k_acc_gate(EltArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int Cp = A.dx.Cp, W = A.dx.W, rows = A.b - A.a;
    long long n = (long long)A.B * rows * W * Cp;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int c = idx % Cp;
        long long r = idx / Cp;
        int x = r % W; r /= W;
        int y = A.a + (int)(r % rows);
        int b = (int)(r / rows);
        T *dx = (T *)A.dx.p + voff(A.dx, b, y, x) + c;
        float v = (A.write ? 0.f : ldf(dx)) + ldf((const T *)A.dy.p + voff(A.dy, b, y, x) + c);
        if (A.gate && ldf((const T *)A.act.p + voff(A.act, b, y, x) + c) <= 0.f) v = 0.f;
        stf(dx, v);
    }
}

// ------------------------------------------------------------------ head
template <typename T>
__global__ void k_gap(const T *zl, int HW, int Cp, float *gap, float hw_div) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    int b = blockIdx.x, c = blockIdx.y * blockDim.x + threadIdx.x;
    if (c >= Cp) return;
    const T *z = zl + (long long)b * HW * Cp + c;
    float s = 0.f;
    for (int i = 0; i < HW; ++i) s += ldf(z + (long long)i * Cp);
    gap[(long long)b * Cp + c] = s / hw_div;
}

// GAP in two deterministic passes (z^L is the largest head input: 278 MB at C4).  Pass 1: block
// (chunk, b) sums the pixels [chunk * per, ...) of image b with 16-byte loads (a thread = 8 channels of
// one pixel slot; ppi pixel slots per block iteration), reduces its slots in shared memory and writes
// partial[b][chunk][c].  Pass 2: one thread per (b, c) adds the chunks in order.
constexpr int kGapChunks = 64;
template <typename T>
__global__ void __launch_bounds__(256) k_gap_partial(const T *zl, int HW, int Cp, float *partial) {
    griddep_wait();
    griddep_launch();
    extern __shared__ float gsum[];   // [ppi][Cp]
    const int chunk = blockIdx.x, b = blockIdx.y;
    const int tpp = Cp / 8, ppi = blockDim.x / tpp;   // threads per pixel, pixel slots per iteration
    const int slot = threadIdx.x / tpp, cv = threadIdx.x - slot * tpp;
    const int per = (HW + kGapChunks - 1) / kGapChunks, p0 = chunk * per, p1 = min(HW, p0 + per);
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (slot < ppi) {
        const T *z = zl + (long long)b * HW * Cp + cv * 8;
        for (int p = p0 + slot; p < p1; p += ppi) {
            float v[8];
            ld8(z + (long long)p * Cp, v);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += v[j];
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) gsum[slot * Cp + cv * 8 + j] = acc[j];
    }
    __syncthreads();
    for (int c = threadIdx.x; c < Cp; c += blockDim.x) {
        float t = 0.f;
        for (int s2 = 0; s2 < ppi; ++s2) t += gsum[s2 * Cp + c];
        partial[((long long)b * kGapChunks + chunk) * Cp + c] = t;
    }
}
__global__ void k_gap_final(const float *partial, int Cp, float *gap, float hw_div) {
    griddep_wait();
    griddep_launch();
    const int b = blockIdx.y, c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= Cp) return;
    float t = 0.f;
    for (int k = 0; k < kGapChunks; ++k) t += partial[((long long)b * kGapChunks + k) * Cp + c];
    gap[(long long)b * Cp + c] = t / hw_div;
}

// Head: FC -> softmax-CE (mean over B) -> d logits -> FC gradients.  k_fc_logits has one block per
// image (warps over classes, lanes over channels) and writes that image's d logits and loss term;
// k_fc_grad spreads the FC weight gradient over (class, channel) threads and sums the loss.
template <typename T>
__global__ void k_fc_logits(const float *gap, int B, int Cp, int C, int classes, const T *fw, const T *fb,
                            const int32_t *labels, float *dlog, float *lossb) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    extern __shared__ float lg[];   // logits of this image [classes]
    const int b = blockIdx.x, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int j = threadIdx.x >> 5; j < classes; j += nw) {
        float s = 0.f;
        for (int c = lane; c < C; c += 32) s += gap[(long long)b * Cp + c] * ldf(fw + (long long)j * Cp + c);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) lg[j] = s + ldf(fb + j);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = -INFINITY;
        for (int j = 0; j < classes; ++j) m = fmaxf(m, lg[j]);
        float se = 0.f;
        for (int j = 0; j < classes; ++j) se += expf(lg[j] - m);
        const int lab = labels[b];
        lossb[b] = (m + logf(se)) - lg[lab];
        for (int j = 0; j < classes; ++j)
            dlog[b * classes + j] = (expf(lg[j] - m) / se - (j == lab ? 1.f : 0.f)) / B;
    }
}
template <typename T>
__global__ void k_fc_grad(const float *gap, int B, int Cp, int C, int classes, const float *dlog, const float *lossb,
                          float *loss, float *gw, float *gb) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < classes * C) {
        const int j = i / C, c = i - j * C;
        float s = 0.f;
        for (int b = 0; b < B; ++b) s += dlog[b * classes + j] * gap[(long long)b * Cp + c];
        gw[(long long)j * Cp + c] += s;
    }
    if (blockIdx.x == 0) {
        for (int j = threadIdx.x; j < classes; j += blockDim.x) {   // any class count
            float s = 0.f;
            for (int b = 0; b < B; ++b) s += dlog[b * classes + j];
            gb[j] += s;
        }
        if (threadIdx.x == 0) {
            float l = 0.f;
            for (int b = 0; b < B; ++b) l += lossb[b];
            *loss = l / B;
        }
    }
}


template <typename T>
__global__ void k_dzl(const T *zl, const float *dlog, const T *fw, int B, int HW, int Cp, int C, int classes,
                      T *dzl, int gate, float hw_div) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    long long n = (long long)B * HW * Cp;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int c = idx % Cp;
        int b = (int)(idx / ((long long)HW * Cp));
        float v = 0.f;
        if (c < C) {
            for (int j = 0; j < classes; ++j) v += dlog[b * classes + j] * ldf(fw + (long long)j * Cp + c);
            v /= hw_div;
        }
        if (gate && ldf(zl + idx) <= 0.f) v = 0.f;
        stf(dzl + idx, v);
    }
}

template <typename T>
__global__ void k_gate_copy(const T *src, const T *act, T *dst, long long n, int gate) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        float v = ldf(src + i);
        if (gate && ldf(act + i) <= 0.f) v = 0.f;
        stf(dst + i, v);
    }
}

template <typename T>
__global__ void k_sgd(float *master, T *params, float *grads, long long n, float lr) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        float m = master[i] - lr * grads[i];
        master[i] = m;
        stf(params + i, m);
        grads[i] = 0.f;
    }
}

template <typename T>
// wt[ci][k-1-ky][k-1-kx][co] = gamma[co] * w[co][ky][kx][ci] (0 for co >= cout): per tap a 32 x 32
// tile transpose through shared memory, coalesced along ci on the read and co on the write.
__global__ void k_transpose_w(const T *w, const T *gamma, T *wt, int cout, int coutp, int k, int cinp) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    __shared__ float tile[32][33];
    const int taps = k * k, tap = blockIdx.z;
    const int ci0 = blockIdx.x * 32, co0 = blockIdx.y * 32;
    const int ky = tap / k, kx = tap - ky * k;
    const int tap2 = (k - 1 - ky) * k + (k - 1 - kx);
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int co = co0 + r, ci = ci0 + threadIdx.x;
        float v = 0.f;
        if (co < cout && ci < cinp) {
            v = ldf(w + ((long long)co * taps + tap) * cinp + ci);
            if (gamma) v *= ldf(gamma + co);
        }
        tile[r][threadIdx.x] = v;
    }
    __syncthreads();
    for (int r = threadIdx.y; r < 32; r += blockDim.y) {
        const int ci = ci0 + r, co = co0 + threadIdx.x;
        if (ci < cinp && co < coutp) stf(wt + ((long long)ci * taps + tap2) * coutp + co, tile[threadIdx.x][r]);
    }
}

// ------------------------------------------------------------------ 8-channel vector versions (Cp % 8 == 0)
// general k x k / stride s / pad p max-pool: padded cells never win, ties -> first in raster order
template <typename T>
__device__ __forceinline__ void pool_window8(const View &in, int b, int y, int x, int c0, int k, int s, int p,
                                             float (&best)[8], int (&arg)[8]) {
    bool first = true;
    for (int ky = 0; ky < k; ++ky) {
        int g = y * s - p + ky;
        if (!vhas(in, g)) continue;
        for (int kx = 0; kx < k; ++kx) {
            int xi = x * s - p + kx;
            if (xi < 0 || xi >= in.W) continue;
            float v[8];
            ld8((const T *)in.p + voff(in, b, g, xi) + c0, v);
            const int code = ky * k + kx;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (first || v[j] > best[j]) { best[j] = v[j]; arg[j] = code; }
            first = false;
        }
    }
    if (first) {
#pragma unroll
        for (int j = 0; j < 8; ++j) { best[j] = 0.f; arg[j] = -1; }
    }
}

template <typename T>
__global__ void k_pool_fwd8(PoolArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int CV = A.out.Cp / 8, Wo = A.out.W, rows = A.b - A.a;
    long long n = (long long)A.B * rows * Wo * CV;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int cv = idx % CV;
        long long r = idx / CV;
        int x = r % Wo; r /= Wo;
        int y = A.a + (int)(r % rows);
        int b = (int)(r / rows);
        float best[8];
        int arg[8];
        pool_window8<T>(A.in, b, y, x, cv * 8, A.k, A.s, A.p, best, arg);
        st8((T *)A.out.p + voff(A.out, b, y, x) + cv * 8, best);
    }
}

// Row-structured max-pool forward (any k / s / p, Cp % 8 == 0): grid.y = image rows of the band, one
// 8-channel vector per thread with 32-bit index math (the flat grid-stride k_pool_fwd8 spent its issue
// slots on 64-bit index division), max only (the forward needs no argmax; the backward recomputes it).
template <typename T>
__global__ void k_pool_fwd_rows8(PoolArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int CV = A.out.Cp / 8, Wo = A.out.W, rows = A.b - A.a;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= Wo * CV) return;
    const int cv = v % CV, x = v / CV;
    for (int ry = blockIdx.y; ry < A.B * rows; ry += gridDim.y) {
        const int y = A.a + ry % rows, b = ry / rows;
        float best[8];
        bool first = true;
        for (int ky = 0; ky < A.k; ++ky) {
            const int g = y * A.s - A.p + ky;
            if (!vhas(A.in, g)) continue;
            const T *row = (const T *)A.in.p + voff(A.in, b, g, 0) + cv * 8;
            for (int kx = 0; kx < A.k; ++kx) {
                const int xi = x * A.s - A.p + kx;
                if (xi < 0 || xi >= A.in.W) continue;
                float w[8];
                ld8(row + (size_t)xi * A.in.Cp, w);
#pragma unroll
                for (int j = 0; j < 8; ++j) best[j] = first ? w[j] : fmaxf(best[j], w[j]);
                first = false;
            }
        }
        if (first) {
#pragma unroll
            for (int j = 0; j < 8; ++j) best[j] = 0.f;
        }
        st8((T *)A.out.p + voff(A.out, b, y, x) + cv * 8, best);
    }
}

// gather: every input pixel checks the (at most ceil(k/s)^2) windows that contain it
template <typename T>
__global__ void k_pool_bwd8(PoolArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int CV = A.dx.Cp / 8, Wi = A.dx.W, rows = A.rb - A.ra, Wo = A.dy.W;
    long long n = (long long)A.B * rows * Wi * CV;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int cv = idx % CV;
        long long r = idx / CV;
        int xi = r % Wi; r /= Wi;
        int g = A.ra + (int)(r % rows);
        int b = (int)(r / rows);
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        for (int ky = 0; ky < A.k; ++ky) {
            int num = g + A.p - ky;
            if (num < 0 || num % A.s) continue;
            int y = num / A.s;
            if (!vhas(A.dy, y)) continue;
            for (int kx = 0; kx < A.k; ++kx) {
                int nx = xi + A.p - kx;
                if (nx < 0 || nx % A.s) continue;
                int x = nx / A.s;
                if (x >= Wo) continue;
                float best[8], d[8];
                int arg[8];
                pool_window8<T>(A.act, b, y, x, cv * 8, A.k, A.s, A.p, best, arg);
                ld8((const T *)A.dy.p + voff(A.dy, b, y, x) + cv * 8, d);
                const int code = ky * A.k + kx;
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (arg[j] == code) acc[j] += d[j];
            }
        }
        T *dp = (T *)A.dx.p + voff(A.dx, b, g, xi) + cv * 8;
        float o[8], a[8];
        ld8(dp, o);
        if (A.gate) ld8((const T *)A.act.p + voff(A.act, b, g, xi) + cv * 8, a);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            o[j] += acc[j];
            if (A.gate && !(a[j] > 0.f)) o[j] = 0.f;
        }
        st8(dp, o);
    }
}

// Overlapping max-pool backward (s < k <= 2s, e.g. ResNet's 3x3/s2/p1) as a tiled gather.  A CTA
// owns kPoolTR x kPoolTC input pixels (all channel vectors) of one image.  Phase 1 computes, once,
// the argmax code and dy of every pooling window that touches them (output rows limited to the
// band rows [a, b) whose dy is present) into shared memory; phase 2 gives every owned input pixel
// the sum of dy over the windows whose argmax it is, applies the gate (act > 0) and stores dx once
// (A.acc: dx += ..., else dx is written, single writer).  HBM traffic ~ act read once (+ window
// halo, L1/L2 hits), dy once, dx written once: the scatter form paid a memset, 2.25 window reads
// and a read-modify-write of dx per window position.
constexpr int kPoolTR = 8, kPoolTC = 32;
static inline int pool_tile_rows(int t, int k, int s) { return (t + k - 2) / s + 1; }   // windows per tile edge

template <typename T>
__global__ void __launch_bounds__(256) k_pool_bwd_tile8(PoolArgs A, int ny_max, int nx_max) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    extern __shared__ float pool_smem[];
    const int CV = A.dy.Cp / 8, Wo = A.dy.W, Wi = A.dx.W;
    const int k = A.k, s = A.s, p = A.p;
    const int b = blockIdx.z;
    const int g0 = A.ra + blockIdx.y * kPoolTR, g1 = min(g0 + kPoolTR, A.rb);
    const int x0 = blockIdx.x * kPoolTC, x1 = min(x0 + kPoolTC, Wi);
    // windows touching rows [g0, g1): y*s - p <= g1-1 and y*s - p + k - 1 >= g0
    auto first_win = [&](int g) { int lo = g + p - k + 1; return lo <= 0 ? 0 : (lo + s - 1) / s; };
    const int ylo = max(first_win(g0), A.a), yhi = min((g1 - 1 + p) / s, A.b - 1);
    const int xlo = first_win(x0), xhi = min((x1 - 1 + p) / s, Wo - 1);
    const int ny = yhi - ylo + 1, nx = xhi - xlo + 1;
    // per window slot: dy as 8 raw T (one 16-byte vector for bf16: conflict-free LDS.128 across the
    // warp's consecutive channel vectors) and the 8 argmax codes as int8 in one 8-byte word
    T *sdy = (T *)pool_smem;                                                   // [ny_max*nx_max*CV][8]
    uint2 *scode = (uint2 *)(sdy + (size_t)ny_max * nx_max * CV * 8);
    if (ny > 0 && nx > 0) {
        const int items = ny * nx * CV;
        for (int i = threadIdx.x; i < items; i += blockDim.x) {
            const int cv = i % CV, pix = i / CV;
            const int oy = ylo + pix / nx, ox = xlo + pix % nx;
            float best[8], d[8];
            int arg[8];
            pool_window8<T>(A.act, b, oy, ox, cv * 8, k, s, p, best, arg);
            ld8((const T *)A.dy.p + voff(A.dy, b, oy, ox) + cv * 8, d);
            const int slot = ((pix / nx) * nx_max + pix % nx) * CV + cv;
            st8(sdy + (size_t)slot * 8, d);
            uint2 c;
            c.x = c.y = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                c.x |= (uint32_t)(arg[j] & 0xff) << (8 * j);
                c.y |= (uint32_t)(arg[j + 4] & 0xff) << (8 * j);
            }
            scode[slot] = c;
        }
    }
    __syncthreads();
    const int tw = x1 - x0, owned = (g1 - g0) * tw * CV;
    for (int i = threadIdx.x; i < owned; i += blockDim.x) {
        const int cv = i % CV, pix = i / CV;
        const int g = g0 + pix / tw, xi = x0 + pix % tw;
        float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const int ya = max(first_win(g), ylo), yb = min((g + p) / s, yhi);
        const int xa = max(first_win(xi), xlo), xb = min((xi + p) / s, xhi);
        for (int y = ya; y <= yb; ++y)
            for (int x = xa; x <= xb; ++x) {
                const uint32_t code = (uint32_t)((g - (y * s - p)) * k + (xi - (x * s - p)));
                const int slot = ((y - ylo) * nx_max + (x - xlo)) * CV + cv;
                const uint2 c = scode[slot];
                const uint32_t rep = code * 0x01010101u;
                // bytes of c equal to code (per-byte compare via __vcmpeq4: 0xff where equal)
                const uint32_t m0 = __vcmpeq4(c.x, rep), m1 = __vcmpeq4(c.y, rep);
                if ((m0 | m1) == 0) continue;
                float d[8];
                ld8(sdy + (size_t)slot * 8, d);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (((j < 4 ? m0 : m1) >> (8 * (j & 3))) & 1) acc[j] += d[j];
            }
        T *dp = (T *)A.dx.p + voff(A.dx, b, g, xi) + cv * 8;
        float o[8], a[8];
        if (A.acc) {
            ld8(dp, o);
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] += acc[j];
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) o[j] = acc[j];
        }
        if (A.gate) {
            ld8((const T *)A.act.p + voff(A.act, b, g, xi) + cv * 8, a);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (!(a[j] > 0.f)) o[j] = 0.f;
        }
        st8(dp, o);
    }
}

// ResNet's 3x3 / stride 2 / pad 1 max-pool backward, bf16: the tiled gather above with the
// window geometry fixed.  Input column pair (2x', 2x'+1) lies in windows x' (kx = 1, 2) and
// x'+1 (kx = 0); input row g lies in window g/2 (ky = 1) if even, else (g-1)/2 (ky = 2) and
// (g+1)/2 (ky = 0).  Phase 1 computes each window's max and first-in-raster argmax with packed
// bf16x2 compares (set.gt / max / lop3: 3 instructions per channel pair and position) and keeps
// 16-bit codes + dy in shared memory (invalid windows: code 0xffff); phase 2 gives a thread one
// input row x column pair x 8 channels and masks dy with packed compares (vcmpeq2), no branches
// on window validity.  A warp covers one input row, so the row-parity branch is warp-uniform.
constexpr int kP3TR = 16, kP3TP = 16;   // input rows x column pairs per CTA
__device__ __forceinline__ uint32_t bf2_gt_mask(uint32_t a, uint32_t b) {
    uint32_t m;
    asm("set.gt.u32.bf16x2 %0, %1, %2;" : "=r"(m) : "r"(a), "r"(b));
    return m;
}
__device__ __forceinline__ uint32_t bf2_max(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ void acc_masked(float (&acc)[8], const uint4 &d, const uint4 &c, uint32_t code2) {
    const uint32_t dw[4] = {d.x, d.y, d.z, d.w}, cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const uint32_t u = dw[h] & __vcmpeq2(cw[h], code2);
        acc[2 * h] += __uint_as_float(u << 16);
        acc[2 * h + 1] += __uint_as_float(u & 0xffff0000u);
    }
}

__global__ void __launch_bounds__(256) k_pool3s2_bwd(PoolArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    extern __shared__ uint4 p3_smem[];
    const int CV = A.dy.Cp / 8, Wo = A.dy.W, Wi = A.dx.W;
    const int b = blockIdx.z;
    const int g0 = A.ra + blockIdx.y * kP3TR, g1 = min(g0 + kP3TR, A.rb);
    const int xp0 = blockIdx.x * kP3TP;
    // windows of this tile: rows [wy0, wy0 + NY), columns [xp0, xp0 + NX)
    const int wy0 = g0 >> 1, NY = ((g1 - 1 + 1) >> 1) - wy0 + 1, NX = kP3TP + 1;
    uint4 *scode = p3_smem, *sdy = p3_smem + (kP3TR / 2 + 2) * NX * CV;
    const int items = NY * NX * CV;
    for (int i = threadIdx.x; i < items; i += blockDim.x) {
        const int cv = i % CV, pix = i / CV;
        const int y = wy0 + pix / NX, x = xp0 + pix % NX;
        uint4 code = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu), dyv = make_uint4(0, 0, 0, 0);
        if (y >= A.a && y < A.b && x < Wo) {
            uint32_t best[4] = {0, 0, 0, 0}, cw[4] = {0, 0, 0, 0};
            bool have = false;
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                const int g = 2 * y - 1 + ky;
                if (!vhas(A.act, g)) continue;
                const bf16 *row = (const bf16 *)A.act.p + voff(A.act, b, g, 0) + cv * 8;
#pragma unroll
                for (int kx = 0; kx < 3; ++kx) {
                    const int xi = 2 * x - 1 + kx;
                    if (xi < 0 || xi >= Wi) continue;
                    const uint4 v = *reinterpret_cast<const uint4 *>(row + (long long)xi * A.act.Cp);
                    const uint32_t vw[4] = {v.x, v.y, v.z, v.w};
                    const uint32_t pos = (uint32_t)(ky * 3 + kx) * 0x00010001u;
                    if (!have) {
#pragma unroll
                        for (int h = 0; h < 4; ++h) { best[h] = vw[h]; cw[h] = pos; }
                        have = true;
                    } else {
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            const uint32_t m = bf2_gt_mask(vw[h], best[h]);   // strictly greater: first wins ties
                            best[h] = bf2_max(vw[h], best[h]);
                            cw[h] = (cw[h] & ~m) | (pos & m);
                        }
                    }
                }
            }
            if (have) {
                code = make_uint4(cw[0], cw[1], cw[2], cw[3]);
                dyv = *reinterpret_cast<const uint4 *>((const bf16 *)A.dy.p + voff(A.dy, b, y, x) + cv * 8);
                if (A.gate) {   // the delta goes to the argmax, whose activation is the window max:
                    dyv.x &= bf2_gt_mask(best[0], 0u);   // gate it here ([max > 0], ReLU'(0) = 0) and
                    dyv.y &= bf2_gt_mask(best[1], 0u);   // phase 2 never re-reads the activation
                    dyv.z &= bf2_gt_mask(best[2], 0u);
                    dyv.w &= bf2_gt_mask(best[3], 0u);
                }
            }
        }
        scode[pix * CV + cv] = code;
        sdy[pix * CV + cv] = dyv;
    }
    __syncthreads();
    const int owned = (g1 - g0) * kP3TP * CV;
    for (int i = threadIdx.x; i < owned; i += blockDim.x) {
        const int cv = i % CV, r = i / CV;
        const int xp = xp0 + r % kP3TP, g = g0 + r / kP3TP;
        const int xa = 2 * xp;
        if (xa >= Wi) continue;
        float accA[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, accB[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
        const int c0 = (xp - xp0) * CV + cv;
        auto window_row = [&](int y, int ky) {
            const int sl = (y - wy0) * NX * CV + c0;
            const uint4 cl = scode[sl], dl = sdy[sl], cr = scode[sl + CV], dr = sdy[sl + CV];
            acc_masked(accA, dl, cl, (uint32_t)(ky * 3 + 1) * 0x00010001u);
            acc_masked(accB, dl, cl, (uint32_t)(ky * 3 + 2) * 0x00010001u);
            acc_masked(accB, dr, cr, (uint32_t)(ky * 3 + 0) * 0x00010001u);
        };
        if ((g & 1) == 0) window_row(g >> 1, 1);
        else { window_row(g >> 1, 2); window_row((g >> 1) + 1, 0); }
        bf16 *dp = (bf16 *)A.dx.p + voff(A.dx, b, g, xa) + cv * 8;
        // (gated in phase 1; an accumulated old delta was gated by its own writer: gate on write)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            if (e == 1 && xa + 1 >= Wi) break;
            float o[8];
            const float (&acc)[8] = e ? accB : accA;
            if (A.acc) {
                ld8(dp + e * A.dx.Cp, o);
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] += acc[j];
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j) o[j] = acc[j];
            }
            st8(dp + e * A.dx.Cp, o);
        }
    }
}

template <typename T>
__global__ void k_acc_gate8(EltArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int CV = A.dx.Cp / 8, W = A.dx.W, rows = A.b - A.a;
    long long n = (long long)A.B * rows * W * CV;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int cv = idx % CV;
        long long r = idx / CV;
        int x = r % W; r /= W;
        int y = A.a + (int)(r % rows);
        int b = (int)(r / rows);
        T *dp = (T *)A.dx.p + voff(A.dx, b, y, x) + cv * 8;
        float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, d[8], a[8];
        if (!A.write) ld8(dp, o);
        ld8((const T *)A.dy.p + voff(A.dy, b, y, x) + cv * 8, d);
        if (A.gate) ld8((const T *)A.act.p + voff(A.act, b, y, x) + cv * 8, a);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            o[j] += d[j];
            if (A.gate && !(a[j] > 0.f)) o[j] = 0.f;
        }
        st8(dp, o);
    }
}

// dx = gate(act) * (dx + dy) on rows [a, b): grid y = (image, row), x = row vectors; each row of
// one image is contiguous in all three views (W * Cp elements)
template <typename T>
__global__ void k_acc_gate_rows(EltArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int rows = A.b - A.a, nv = A.dx.W * A.dx.Cp / 8;
    const int b = blockIdx.y / rows, y = A.a + (int)(blockIdx.y - b * rows);
    T *dx = (T *)A.dx.p + voff(A.dx, b, y, 0);
    const T *dy = (const T *)A.dy.p + voff(A.dy, b, y, 0);
    const T *ac = A.gate ? (const T *)A.act.p + voff(A.act, b, y, 0) : nullptr;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += gridDim.x * blockDim.x) {
        float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, d[8], g[8];
        if (!A.write) ld8(dx + i * 8, o);
        ld8(dy + i * 8, d);
        if (ac) ld8(ac + i * 8, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            o[j] += d[j];
            if (ac && !(g[j] > 0.f)) o[j] = 0.f;
        }
        st8(dx + i * 8, o);
    }
}

template <typename T>
__global__ void k_add_fwd8(EltArgs A) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int CV = A.out.Cp / 8, W = A.out.W, rows = A.b - A.a;
    long long n = (long long)A.B * rows * W * CV;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int cv = idx % CV;
        long long r = idx / CV;
        int x = r % W; r /= W;
        int y = A.a + (int)(r % rows);
        int b = (int)(r / rows);
        float u[8], v[8];
        ld8((const T *)A.x0.p + voff(A.x0, b, y, x) + cv * 8, u);
        ld8((const T *)A.x1.p + voff(A.x1, b, y, x) + cv * 8, v);
#pragma unroll
        for (int j = 0; j < 8; ++j) { u[j] += v[j]; if (A.relu) u[j] = fmaxf(u[j], 0.f); }
        st8((T *)A.out.p + voff(A.out, b, y, x) + cv * 8, u);
    }
}

// ------------------------------------------------------------------ launchers
static const int kT = 256;
static unsigned grid_for(long long n) {
    long long g = (n + kT - 1) / kT;
    if (g > 148LL * 64) g = 148LL * 64;
    return (unsigned)(g < 1 ? 1 : g);
}


cudaError_t simt_conv_fwd(int prec, const ConvFwdArgs &a, cudaStream_t st) {
    long long n = (long long)a.B * (a.b_ - a.a) * a.out.W * a.out.Cp;
    if (n <= 0) return cudaSuccess;
    if (prec) launch_simt(k_conv_fwd<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_conv_fwd<float>, grid_for(n), kT, 0, st, a);
    return cudaGetLastError();
}
cudaError_t simt_conv_dgrad(int prec, const DgradArgs &a, cudaStream_t st) {
    long long n = (long long)a.B * (a.rb - a.ra) * a.dx.W * a.dx.Cp;
    if (n <= 0) return cudaSuccess;
    if (prec) launch_simt(k_conv_dgrad<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_conv_dgrad<float>, grid_for(n), kT, 0, st, a);
    return cudaGetLastError();
}
cudaError_t simt_conv_wgrad(int prec, const WgradArgs &a, cudaStream_t st) {
    if (a.b <= a.a) return cudaSuccess;
    if (a.dg && !a.w) return cudaErrorInvalidValue;
    a.dg_done = a.dg != nullptr;
    dim3 g(a.c_out * a.k * a.k, (a.x.Cp + 31) / 32);
    if (prec) launch_simt(k_conv_wgrad<bf16>, g, 256, 0, st, a); else launch_simt(k_conv_wgrad<float>, g, 256, 0, st, a);
    return cudaGetLastError();
}
cudaError_t simt_param_grad(int prec, const ParamGradArgs &a, cudaStream_t st) {
    if (a.b <= a.a || !a.db) return cudaSuccess;
    const int CVall = a.dy.Cp / 8;
    if (CVall < 1 || a.dy.Cp % 8) return cudaErrorInvalidValue;
    const int CV = CVall < 64 ? CVall : 64, groups = (CVall + CV - 1) / CV;
    dim3 blk(CV, CV >= 64 ? 4 : 256 / CV);
    long long npix = (long long)a.B * (a.b - a.a) * a.dy.W;
    long long g = (npix + blk.y * 4 - 1) / (blk.y * 4);          // ~4 pixels per thread
    long long cap = 148 * 8 / groups + 1;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    dim3 grid((unsigned)g, groups);
    size_t shm = sizeof(float) * blk.y * CV * 8;
    if (prec) launch_simt(k_param_grad<bf16>, grid, blk, shm, st, a); else launch_simt(k_param_grad<float>, grid, blk, shm, st, a);
    return cudaGetLastError();
}
static bool pool2(const PoolArgs &a, const View &v) {
    return a.k == 2 && a.s == 2 && a.p == 0 && v.Cp % 8 == 0 && (long long)a.B * (a.b - a.a) <= 65535;
}
cudaError_t simt_pool_fwd(int prec, const PoolArgs &a, cudaStream_t st) {
    long long n = (long long)a.B * (a.b - a.a) * a.out.W * a.out.Cp;
    if (n <= 0) return cudaSuccess;
    if (pool2(a, a.out)) {
        // 128-thread blocks: a VGG output row is 896 channel vectors (7 x 128, no idle tail)
        const int rowv = a.out.W * (a.out.Cp / 8), tb = 128;
        dim3 g((rowv + tb - 1) / tb, a.B * (a.b - a.a));
        if (prec) launch_simt(k_pool2_fwd<bf16>, g, tb, 0, st, a); else launch_simt(k_pool2_fwd<float>, g, tb, 0, st, a);
    } else if (a.out.Cp % 8 == 0) {
        const int rowv = a.out.W * (a.out.Cp / 8), tb = 128;
        dim3 g((rowv + tb - 1) / tb, std::min(65535, a.B * (a.b - a.a)));
        if (prec) launch_simt(k_pool_fwd_rows8<bf16>, g, tb, 0, st, a); else launch_simt(k_pool_fwd_rows8<float>, g, tb, 0, st, a);
    } else {
        if (prec) launch_simt(k_pool_fwd<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_pool_fwd<float>, grid_for(n), kT, 0, st, a);
    }
    return cudaGetLastError();
}
// the tiled gather (k_pool_bwd_tile8) takes overlapping windows whose per-tile state fits in shared memory
bool pool_tiled_shape(int k, int s, int Cp) {
    const size_t shm = (size_t)pool_tile_rows(kPoolTR, k, s) * pool_tile_rows(kPoolTC, k, s) * (Cp / 8) * 40;
    return Cp % 8 == 0 && k > s && k <= 2 * s && k <= 16 && shm <= 200 * 1024;
}
static bool pool_tiled(const PoolArgs &a) {
    return a.dx.Cp == a.dy.Cp && pool_tiled_shape(a.k, a.s, a.dx.Cp) && a.B <= 65535;
}
int simt_pool_bwd_launches(const PoolArgs &a) {
    if ((long long)a.B * (a.rb - a.ra) * a.dx.W * a.dx.Cp <= 0) return 0;
    if (pool2(a, a.dy)) return a.b > a.a ? 1 : 0;
    return 1;
}
cudaError_t simt_pool_bwd(int prec, const PoolArgs &a, cudaStream_t st) {
    long long n = (long long)a.B * (a.rb - a.ra) * a.dx.W * a.dx.Cp;
    if (n <= 0) return cudaSuccess;
    if (pool2(a, a.dy)) {
        if (a.b <= a.a) return cudaSuccess;
        const int rowv = a.dy.W * (a.dy.Cp / 8), tb = 128;
        dim3 g((rowv + tb - 1) / tb, a.B * (a.b - a.a));
        if (prec) launch_simt(k_pool2_bwd<bf16>, g, tb, 0, st, a); else launch_simt(k_pool2_bwd<float>, g, tb, 0, st, a);
    } else if (prec && a.k == 3 && a.s == 2 && a.p == 1 && a.dx.Cp % 8 == 0 && a.dx.Cp == a.dy.Cp && a.B <= 65535) {
        const size_t shm = (size_t)2 * (kP3TR / 2 + 2) * (kP3TP + 1) * (a.dy.Cp / 8) * 16;
        dim3 g((a.dx.W + 2 * kP3TP - 1) / (2 * kP3TP), (a.rb - a.ra + kP3TR - 1) / kP3TR, a.B);
        if (shm > 48 * 1024) {   // once per (device, size): the attribute is per device
            static std::mutex mu;
            static std::set<std::pair<int, size_t>> done;
            int dev = 0;
            cudaGetDevice(&dev);
            std::lock_guard<std::mutex> lk(mu);
            if (!done.count({dev, shm})) {
                cudaFuncSetAttribute(k_pool3s2_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
                done.insert({dev, shm});
            }
        }
        launch_simt(k_pool3s2_bwd, g, kT, shm, st, a);
    } else if (pool_tiled(a)) {
        const int ny = pool_tile_rows(kPoolTR, a.k, a.s), nx = pool_tile_rows(kPoolTC, a.k, a.s);
        const size_t shm = (size_t)ny * nx * (a.dy.Cp / 8) * (8 * (prec ? 2 : 4) + 8);
        dim3 g((a.dx.W + kPoolTC - 1) / kPoolTC, (a.rb - a.ra + kPoolTR - 1) / kPoolTR, a.B);
        if (prec) {
            cudaFuncSetAttribute(k_pool_bwd_tile8<bf16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
            launch_simt(k_pool_bwd_tile8<bf16>, g, kT, shm, st, a, ny, nx);
        } else {
            cudaFuncSetAttribute(k_pool_bwd_tile8<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)shm);
            launch_simt(k_pool_bwd_tile8<float>, g, kT, shm, st, a, ny, nx);
        }
    } else if (a.dx.Cp % 8 == 0) {
        n /= 8;
        if (prec) launch_simt(k_pool_bwd8<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_pool_bwd8<float>, grid_for(n), kT, 0, st, a);
    } else {
        if (prec) launch_simt(k_pool_bwd<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_pool_bwd<float>, grid_for(n), kT, 0, st, a);
    }
    return cudaGetLastError();
}
cudaError_t simt_add_fwd(int prec, const EltArgs &a, cudaStream_t st) {
    long long n = (long long)a.B * (a.b - a.a) * a.out.W * a.out.Cp;
    if (n <= 0) return cudaSuccess;
    if (a.out.Cp % 8 == 0) {
        n /= 8;
        if (prec) launch_simt(k_add_fwd8<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_add_fwd8<float>, grid_for(n), kT, 0, st, a);
    } else if (prec) launch_simt(k_add_fwd<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_add_fwd<float>, grid_for(n), kT, 0, st, a);
    return cudaGetLastError();
}
cudaError_t simt_acc_gate(int prec, const EltArgs &a, cudaStream_t st) {
    long long n = (long long)a.B * (a.b - a.a) * a.dx.W * a.dx.Cp;
    if (n <= 0) return cudaSuccess;
    const long long gy = (long long)a.B * (a.b - a.a);
    if (a.dx.Cp % 8 == 0 && a.dx.Cp == a.dy.Cp && (!a.gate || a.act.Cp == a.dx.Cp) && gy <= 65535) {
        const int nv = a.dx.W * a.dx.Cp / 8;
        dim3 g((nv + kT - 1) / kT, (unsigned)gy);
        if (prec) launch_simt(k_acc_gate_rows<bf16>, g, kT, 0, st, a); else launch_simt(k_acc_gate_rows<float>, g, kT, 0, st, a);
    } else if (a.dx.Cp % 8 == 0) {
        n /= 8;
        if (prec) launch_simt(k_acc_gate8<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_acc_gate8<float>, grid_for(n), kT, 0, st, a);
    } else if (prec) launch_simt(k_acc_gate<bf16>, grid_for(n), kT, 0, st, a); else launch_simt(k_acc_gate<float>, grid_for(n), kT, 0, st, a);
    return cudaGetLastError();
}

// delta^L for bf16 maps with Cp % 8 == 0: grid (x: pixel chunks, y: image b).  The per-channel
// value g[c] = (sum_j dlog[b][j] * fw[j][c]) / hw_div (the same order as k_dzl) is computed once per
// block into shared memory; threads then stream 16-byte vectors of z^L (gate) and delta^L.
__global__ void k_dzl8(const bf16 *zl, const float *dlog, const bf16 *fw, int HW, int Cp, int C, int classes,
                       bf16 *dzl, int gate, float hw_div) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    extern __shared__ float dz_g[];
    const int b = blockIdx.y;
    for (int c = threadIdx.x; c < Cp; c += blockDim.x) {
        float v = 0.f;
        if (c < C) {
            for (int j = 0; j < classes; ++j) v += dlog[b * classes + j] * __bfloat162float(fw[(long long)j * Cp + c]);
            v /= hw_div;
        }
        dz_g[c] = v;
    }
    __syncthreads();
    const int CV = Cp / 8;
    const long long nv = (long long)HW * CV, base = (long long)b * HW * Cp;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv; i += (long long)gridDim.x * blockDim.x) {
        const int c0 = (int)(i % CV) * 8;
        float o[8], z[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = dz_g[c0 + j];
        if (gate) {
            ld8(zl + base + i * 8, z);
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (z[j] <= 0.f) o[j] = 0.f;
        }
        st8(dzl + base + i * 8, o);
    }
}

// GAP over the z^L rows this rank holds (HW pixels per image), divided by the global H_L*W_L
cudaError_t head_gap(int prec, const void *zl, int B, int HW, int Cp, float hw_div, float *scratch, cudaStream_t st,
                     float *partial) {
    if (prec && partial && Cp % 8 == 0 && Cp / 8 <= 256 && B <= 65535) {   // bf16: two-pass, 16-byte loads
        const int ppi = 256 / (Cp / 8);
        launch_simt(k_gap_partial<bf16>, dim3(kGapChunks, B), 256, sizeof(float) * ppi * Cp, st, (const bf16 *)zl, HW, Cp,
                    partial);
        launch_simt(k_gap_final, dim3((Cp + 127) / 128, B), 128, 0, st, (const float *)partial, Cp, scratch, hw_div);
        return cudaGetLastError();
    }
    dim3 g1(B, (Cp + 127) / 128);
    if (prec) launch_simt(k_gap<bf16>, g1, 128, 0, st, (const bf16 *)zl, HW, Cp, scratch, hw_div);
    else launch_simt(k_gap<float>, g1, 128, 0, st, (const float *)zl, HW, Cp, scratch, hw_div);
    return cudaGetLastError();
}
size_t head_gap_partial_floats(int B, int Cp) { return (size_t)B * kGapChunks * Cp; }

// FC -> softmax-CE -> d logits -> FC grads -> delta^L (gated by the last op's ReLU) on this rank's rows
cudaError_t head_tail(int prec, const void *zl, int B, int HW, int Cp, int C, int classes, const void *fc_w,
                      const void *fc_b, const int32_t *labels, float *scratch, float *loss, float *g_fc_w,
                      float *g_fc_b, void *dzl, int gate, float hw_div, cudaStream_t st) {
    float *gap = scratch, *dlog = scratch + (long long)B * Cp, *lossb = dlog + (long long)B * classes;
    long long n = (long long)B * HW * Cp;
    const unsigned gblocks = (unsigned)((classes * C + kT - 1) / kT);
    if (prec) {
        launch_simt(k_fc_logits<bf16>, B, 256, sizeof(float) * classes, st, gap, B, Cp, C, classes, (const bf16 *)fc_w,
                    (const bf16 *)fc_b, labels, dlog, lossb);
        launch_simt(k_fc_grad<bf16>, gblocks, kT, 0, st, gap, B, Cp, C, classes, (const float *)dlog,
                    (const float *)lossb, loss, g_fc_w, g_fc_b);
        if (n > 0 && Cp % 8 == 0 && B <= 65535) {
            const long long nv = (long long)HW * Cp / 8;
            long long gx = (nv + kT * 4 - 1) / (kT * 4);
            const long long cap = (148LL * 8 + B - 1) / B;
            dim3 g((unsigned)(gx < 1 ? 1 : gx > cap ? cap : gx), B);
            launch_simt(k_dzl8, g, kT, sizeof(float) * Cp, st, (const bf16 *)zl, dlog, (const bf16 *)fc_w, HW, Cp, C,
                        classes, (bf16 *)dzl, gate, hw_div);
        } else if (n > 0)
            launch_simt(k_dzl<bf16>, grid_for(n), kT, 0, st, (const bf16 *)zl, dlog, (const bf16 *)fc_w, B, HW, Cp, C, classes,
                                                   (bf16 *)dzl, gate, hw_div);
    } else {
        launch_simt(k_fc_logits<float>, B, 256, sizeof(float) * classes, st, gap, B, Cp, C, classes,
                    (const float *)fc_w, (const float *)fc_b, labels, dlog, lossb);
        launch_simt(k_fc_grad<float>, gblocks, kT, 0, st, gap, B, Cp, C, classes, (const float *)dlog,
                    (const float *)lossb, loss, g_fc_w, g_fc_b);
        if (n > 0)
            launch_simt(k_dzl<float>, grid_for(n), kT, 0, st, (const float *)zl, dlog, (const float *)fc_w, B, HW, Cp, C,
                                                    classes, (float *)dzl, gate, hw_div);
    }
    return cudaGetLastError();
}

cudaError_t head_forward_backward(int prec, const void *zl, int B, int HW, int Cp, int C, int classes,
                                  const void *fc_w, const void *fc_b, const int32_t *labels, float *scratch,
                                  float *loss, float *g_fc_w, float *g_fc_b, void *dzl, int gate,
                                  cudaStream_t st) {
    cudaError_t e = head_gap(prec, zl, B, HW, Cp, (float)HW, scratch, st);
    if (e != cudaSuccess) return e;
    return head_tail(prec, zl, B, HW, Cp, C, classes, fc_w, fc_b, labels, scratch, loss, g_fc_w, g_fc_b, dzl, gate,
                     (float)HW, st);
}

// dst rows [r0, r1) += src (contiguous [B][r1-r0][W][Cp]): received halo delta of a neighbour rank
template <typename T>
__global__ void k_add_rows(View dst, int r0, int r1, const T *src, int B) {
    griddep_wait();   // PDL: previous kernel complete and visible
    griddep_launch();
    const int rows = r1 - r0, W = dst.W, Cp = dst.Cp;
    long long n = (long long)B * rows * W * Cp;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < n;
         idx += (long long)gridDim.x * blockDim.x) {
        int c = idx % Cp;
        long long r = idx / Cp;
        int x = r % W; r /= W;
        int g = r0 + (int)(r % rows);
        int b = (int)(r / rows);
        T *d = (T *)dst.p + voff(dst, b, g, x) + c;
        stf(d, ldf(d) + ldf(src + idx));
    }
}

cudaError_t add_rows(int prec, const View &dst, int r0, int r1, const void *src, int B, cudaStream_t st) {
    long long n = (long long)B * (r1 - r0) * dst.W * dst.Cp;
    if (n <= 0) return cudaSuccess;
    if (prec) launch_simt(k_add_rows<bf16>, grid_for(n), kT, 0, st, dst, r0, r1, (const bf16 *)src, B);
    else launch_simt(k_add_rows<float>, grid_for(n), kT, 0, st, dst, r0, r1, (const float *)src, B);
    return cudaGetLastError();
}

cudaError_t gate_copy(int prec, const void *src, const void *act, void *dst, long long n, int gate, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (prec) launch_simt(k_gate_copy<bf16>, grid_for(n), kT, 0, st, (const bf16 *)src, (const bf16 *)act, (bf16 *)dst, n, gate);
    else launch_simt(k_gate_copy<float>, grid_for(n), kT, 0, st, (const float *)src, (const float *)act, (float *)dst, n, gate);
    return cudaGetLastError();
}

cudaError_t sgd_update(int prec, float *master, void *params, float *grads, long long n, float lr, cudaStream_t st) {
    if (prec) launch_simt(k_sgd<bf16>, grid_for(n), kT, 0, st, master, (bf16 *)params, grads, n, lr);
    else launch_simt(k_sgd<float>, grid_for(n), kT, 0, st, master, (float *)params, grads, n, lr);
    return cudaGetLastError();
}

cudaError_t transpose_weights(int prec, const void *w, const void *gamma, void *wt, int cout, int coutp, int k,
                              int cinp, cudaStream_t st) {
    dim3 g((cinp + 31) / 32, (coutp + 31) / 32, k * k), blk(32, 8);
    if (prec) launch_simt(k_transpose_w<bf16>, g, blk, 0, st, (const bf16 *)w, (const bf16 *)gamma, (bf16 *)wt, cout, coutp, k, cinp);
    else launch_simt(k_transpose_w<float>, g, blk, 0, st, (const float *)w, (const float *)gamma, (float *)wt, cout, coutp, k, cinp);
    return cudaGetLastError();
}

}  // namespace lrcnn

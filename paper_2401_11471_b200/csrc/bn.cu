// bn.cu -- training-mode BatchNorm on band rows (reading R24).
//
// The paper names BatchNorm in the FP and leaves it out of its analysis; with
// batch statistics a bn op's normalisation depends on EVERY row of its input -- a strong dependency
// across all bands.  The engine resolves it with statistics sweeps (FP) and sums sweeps (BP), see
// engine.cu; these kernels are the per-band pieces:
//   k_bn_stats        sum c, sum c^2 per channel over band rows [a, b) (fp64 partials + atomics)
//   k_bn_finalize_fwd mean, biased var -> coef: a = gamma*invstd, b = beta - a*mean (and mean, invstd)
//   k_bn_fwd          t = relu?(a*c + b + res) on band rows
//   k_bn_sums         S1 = sum da, S2 = sum da*(c-mean)*invstd over band rows (da: the gated delta)
//   k_bn_finalize_bwd p, q of  dc = a*da + p + q*c  (the batch-statistics adjoint
//                     dc = a*(da - S1/M - xh*S2/M)); dgamma += S2, dbeta += S1
//   k_bn_bwd          delta(src) (+)= gate * (a*da + p + q*c) on band rows (written, not accumulated,
//                     when the BN op is the only writer of those rows); rows below cs get a*da only
//                     (OverL: the statistics terms p + q*c once per row, in the first band computing it)
// All arithmetic fp32, sums fp64; activations act_t (fp32 or bf16), NHWC rows of a View, channels
// processed as 8-element vectors (Cp is a multiple of 8).  coef layout: [6][Cp] floats
// (a, b, p, q, mean, invstd); channels >= C get a = b = p = q = 0 (padded channels stay zero).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.hpp"

namespace lrcnn {

namespace {

typedef __nv_bfloat16 bf16;
constexpr double kBnEps = 1e-5;   // DESIGN.md R24 (the oracle states its own copy)
constexpr int kBnThreads = 256;

__device__ __forceinline__ long long bn_off(const View &v, int b, int g, int x) {
    return (long long)b * v.bs + ((long long)(g - v.base) * v.W + x) * v.Cp;
}
__device__ __forceinline__ void load8(const bf16 *p, float *v) {
    const uint4 u = *(const uint4 *)p;
    const __nv_bfloat162 *h = (const __nv_bfloat162 *)&u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const float2 f = __bfloat1622float2(h[k]);
        v[2 * k] = f.x; v[2 * k + 1] = f.y;
    }
}
__device__ __forceinline__ void store8(float *p, const float *v) {
    *(float4 *)p = make_float4(v[0], v[1], v[2], v[3]);
    *(float4 *)(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void store8(bf16 *p, const float *v) {
    uint4 u;
    __nv_bfloat162 *h = (__nv_bfloat162 *)&u;
#pragma unroll
    for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
    *(uint4 *)p = u;
}

constexpr int kRowsPer = 2;
constexpr int kFwdRowsPer = 4;   // k_bn_fwd (two raw loads per row): more rows in flight

__device__ __forceinline__ void coef8(const float *c, float *v) {
    const float4 a = *(const float4 *)c, b = *(const float4 *)(c + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
template <typename T> struct Raw8;
template <> struct Raw8<bf16> { uint4 u; };
template <> struct Raw8<float> { float4 a, b; };
__device__ __forceinline__ void ldraw(const bf16 *p, Raw8<bf16> &r) { r.u = *(const uint4 *)p; }
__device__ __forceinline__ void ldraw(const float *p, Raw8<float> &r) { r.a = *(const float4 *)p; r.b = *(const float4 *)(p + 4); }
__device__ __forceinline__ void unraw(const Raw8<bf16> &r, float *v) { load8((const bf16 *)&r.u, v); }
__device__ __forceinline__ void unraw(const Raw8<float> &r, float *v) {
    v[0] = r.a.x; v[1] = r.a.y; v[2] = r.a.z; v[3] = r.a.w; v[4] = r.b.x; v[5] = r.b.y; v[6] = r.b.z; v[7] = r.b.w;
}

// Per-channel sums of two per-element quantities over the band's pixels.  Block j takes the image
// rows j, j + gridDim.x, ... of the B * (b - a) band rows; thread (lane, g) owns the 8 channels of group
// g for the columns lane, lane + lanes, ... of a row (no per-element index division); fp64 partials,
// a block reduction over the lanes, one fp64 atomic per channel and quantity.
// mode 0: (c, c^2); mode 1: (da, da*xh).
template <typename T, int MODE>
__global__ void __launch_bounds__(kBnThreads) k_bn_reduce(View x, View dy, const float *coef, int a, int b, int B,
                                                          double *out) {
    extern __shared__ double red[];   // [kBnThreads][16]: per-thread fp64 sums (folded once per row)
    const int Cp = x.Cp, G = Cp / 8, lanes = kBnThreads / G;
    const int lane = threadIdx.x / G, g = threadIdx.x % G;
    const int rows = b - a, W = x.W, nrows = B * rows;
    double *my = red + (size_t)threadIdx.x * 16;
#pragma unroll
    for (int k = 0; k < 16; ++k) my[k] = 0.0;
    if (lane < lanes) {
        float mean[8], inv[8];
        if (MODE == 1) {
            coef8(coef + 4 * Cp + g * 8, mean);
            coef8(coef + 5 * Cp + g * 8, inv);
        }
        for (int ry = blockIdx.x; ry < nrows; ry += gridDim.x) {
            const int bi = ry / rows, y = a + ry % rows;
            const T *xr = (const T *)x.p + bn_off(x, bi, y, 0) + g * 8;
            const T *dr = MODE == 1 ? (const T *)dy.p + bn_off(dy, bi, y, 0) + g * 8 : nullptr;
            float f[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) f[k] = 0.f;
            for (int x0 = lane; x0 < W; x0 += 2 * lanes) {
                Raw8<T> rv[2], rd[2];
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int xx = min(x0 + u * lanes, W - 1);
                    ldraw(xr + (size_t)xx * Cp, rv[u]);
                    if (MODE == 1) ldraw(dr + (size_t)xx * Cp, rd[u]);
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (x0 + u * lanes >= W) continue;
                    float v[8], d[8];
                    unraw(rv[u], v);
                    if (MODE == 1) unraw(rd[u], d);
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (MODE == 0) {
                            f[k] += v[k];
                            f[8 + k] = fmaf(v[k], v[k], f[8 + k]);
                        } else {
                            f[k] += d[k];
                            f[8 + k] = fmaf(d[k], (v[k] - mean[k]) * inv[k], f[8 + k]);
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) my[k] += f[k];
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < G * 16; j += blockDim.x) {
        const int gg = j / 16, k = j % 16;
        double acc = 0.0;
        for (int l = 0; l < lanes; ++l) acc += red[(size_t)(l * G + gg) * 16 + k];
        const int c = gg * 8 + (k & 7);
        atomicAdd(out + (k < 8 ? 0 : Cp) + c, acc);
    }
}

// bf16 variant with 4 channels per thread (8-byte loads, 8 fp32 partials): fewer registers and more
// loads in flight (eight columns per iteration) than the 8-channel kernel; Cp <= 1024.
template <int MODE>
__global__ void __launch_bounds__(kBnThreads) k_bn_reduce4(View x, View dy, const float *coef, int a, int b, int B,
                                                           double *out) {
    extern __shared__ double red[];   // [kBnThreads][8]
    const int Cp = x.Cp, G = Cp / 4, lanes = kBnThreads / G;
    const int lane = threadIdx.x / G, g = threadIdx.x % G;
    const int rows = b - a, W = x.W, nrows = B * rows;
    double *my = red + (size_t)threadIdx.x * 8;
#pragma unroll
    for (int k = 0; k < 8; ++k) my[k] = 0.0;
    if (lane < lanes) {
        float mean[4], inv[4];
        if (MODE == 1) {
#pragma unroll
            for (int k = 0; k < 4; ++k) { mean[k] = coef[4 * Cp + g * 4 + k]; inv[k] = coef[5 * Cp + g * 4 + k]; }
        }
        for (int ry = blockIdx.x; ry < nrows; ry += gridDim.x) {
            const int bi = ry / rows, y = a + ry % rows;
            const bf16 *xr = (const bf16 *)x.p + bn_off(x, bi, y, 0) + g * 4;
            const bf16 *dr = MODE == 1 ? (const bf16 *)dy.p + bn_off(dy, bi, y, 0) + g * 4 : nullptr;
            float f[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) f[k] = 0.f;
            constexpr int U = 8;
            for (int x0 = lane; x0 < W; x0 += U * lanes) {
                uint2 rv[U], rd[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int xx = min(x0 + u * lanes, W - 1);
                    rv[u] = *(const uint2 *)(xr + (size_t)xx * Cp);
                    if (MODE == 1) rd[u] = *(const uint2 *)(dr + (size_t)xx * Cp);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (x0 + u * lanes >= W) continue;
                    const float2 v01 = __bfloat1622float2(*(const __nv_bfloat162 *)&rv[u].x);
                    const float2 v23 = __bfloat1622float2(*(const __nv_bfloat162 *)&rv[u].y);
                    const float v[4] = {v01.x, v01.y, v23.x, v23.y};
                    if (MODE == 0) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) { f[k] += v[k]; f[4 + k] = fmaf(v[k], v[k], f[4 + k]); }
                    } else {
                        const float2 d01 = __bfloat1622float2(*(const __nv_bfloat162 *)&rd[u].x);
                        const float2 d23 = __bfloat1622float2(*(const __nv_bfloat162 *)&rd[u].y);
                        const float d[4] = {d01.x, d01.y, d23.x, d23.y};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            f[k] += d[k];
                            f[4 + k] = fmaf(d[k], (v[k] - mean[k]) * inv[k], f[4 + k]);
                        }
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) my[k] += f[k];
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < G * 8; j += blockDim.x) {
        const int gg = j / 8, k = j % 8;
        double acc = 0.0;
        for (int l = 0; l < lanes; ++l) acc += red[(size_t)(l * G + gg) * 8 + k];
        const int c = gg * 4 + (k & 3);
        atomicAdd(out + (k < 4 ? 0 : Cp) + c, acc);
    }
}

template <typename T>
__global__ void k_bn_finalize_fwd(const double *sums, const T *gamma, const T *beta, int C, int Cp, double M,
                                  float *coef) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= Cp) return;
    float a = 0.f, bb = 0.f, mean = 0.f, inv = 0.f;
    if (c < C) {
        const double m = sums[c] / M;
        const double var = fmax(sums[Cp + c] / M - m * m, 0.0);
        const double is = 1.0 / sqrt(var + kBnEps);
        const double ga = (double)(float)gamma[c], be = (double)(float)beta[c];
        a = (float)(ga * is);
        bb = (float)(be - ga * is * m);
        mean = (float)m;
        inv = (float)is;
    }
    coef[c] = a; coef[Cp + c] = bb; coef[4 * Cp + c] = mean; coef[5 * Cp + c] = inv;
}

__global__ void k_bn_finalize_bwd(const double *S, float *coef, int C, int Cp, double M, float *dgamma,
                                  float *dbeta) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= Cp) return;
    float p = 0.f, q = 0.f;
    if (c < C) {
        const double a = coef[c], mean = coef[4 * Cp + c], inv = coef[5 * Cp + c];
        const double s1 = S[c], s2 = S[Cp + c];
        const double qq = -a * s2 * inv / M;
        q = (float)qq;
        p = (float)(-a * s1 / M - qq * mean);
        if (dgamma) dgamma[c] += (float)s2;
        if (dbeta) dbeta[c] += (float)s1;
    }
    coef[2 * Cp + c] = p; coef[3 * Cp + c] = q;
}

// Elementwise kernels: thread (g, x) = channel vector g of column x (grid.x * blockDim.x over the W * Cp / 8
// vectors of a row); grid.y strides over the B * (b - a) image rows, kRowsPer rows per iteration with all
// loads issued first (memory-level parallelism), held as raw 16-byte vectors until used (few registers:
// four resident blocks per SM).  The per-channel coefficients are loaded once per thread as float4
// vectors (loading them per element made the kernels L1-bound: ncu l1tex 97 %).
template <typename T>
__global__ void __launch_bounds__(kBnThreads) k_bn_fwd(View in, View res, View out, const float *coef, int relu,
                                                        int has_res, int a, int b, int B) {
    const int Cp = out.Cp, G = Cp / 8, rows = b - a, nv = out.W * G, nrows = B * rows;
    const int v0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (v0 >= nv) return;
    const int g = v0 % G, xx = v0 / G;
    for (int r0 = blockIdx.y * kFwdRowsPer; r0 < nrows; r0 += gridDim.y * kFwdRowsPer) {
        Raw8<T> rv[kFwdRowsPer], rr[kFwdRowsPer];
        long long off[kFwdRowsPer];
#pragma unroll
        for (int u = 0; u < kFwdRowsPer; ++u) {
            const int ry = min(r0 + u, nrows - 1);   // (a duplicate of the last row is recomputed, not stored)
            const int bi = ry / rows, y = a + ry % rows;
            off[u] = bn_off(out, bi, y, xx) + g * 8;
            ldraw((const T *)in.p + bn_off(in, bi, y, xx) + g * 8, rv[u]);
            if (has_res) ldraw((const T *)res.p + bn_off(res, bi, y, xx) + g * 8, rr[u]);
        }
        float ca[8], cb[8];
        coef8(coef + g * 8, ca);
        coef8(coef + Cp + g * 8, cb);
#pragma unroll
        for (int u = 0; u < kFwdRowsPer; ++u) {
            float v[8], r[8];
            unraw(rv[u], v);
            if (has_res) unraw(rr[u], r);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                float t = fmaf(ca[k], v[k], cb[k]);
                if (has_res) t += r[k];
                v[k] = relu ? fmaxf(t, 0.f) : t;
            }
            if (r0 + u < nrows) store8((T *)out.p + off[u], v);
        }
    }
}

// WRITE: delta(src) rows are produced by this kernel alone (single writer) -- not read; GATE: the input
// has a ReLU (gate on write).  Specialised so the common case (a conv output: no gate, single writer)
// holds two raw loads per row and keeps four rows in flight.
template <typename T, bool GATE, bool WRITE, int RP>
__global__ void __launch_bounds__(kBnThreads) k_bn_bwd(View dy, View x, View dx, View act, const float *coef, int a,
                                                        int b, int B, int cs) {
    const int Cp = dx.Cp, G = Cp / 8, rows = b - a, nv = dx.W * G, nrows = B * rows;
    const int v0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (v0 >= nv) return;
    const int g = v0 % G, xx = v0 / G;
    for (int r0 = blockIdx.y * RP; r0 < nrows; r0 += gridDim.y * RP) {
        Raw8<T> rd[RP], rv[RP], ro[RP], rm[RP];
        long long off[RP];
        bool stat[RP];
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            const int ry = min(r0 + u, nrows - 1);
            const int bi = ry / rows, y = a + ry % rows;
            off[u] = bn_off(dx, bi, y, xx) + g * 8;
            stat[u] = y >= cs;
            ldraw((const T *)dy.p + bn_off(dy, bi, y, xx) + g * 8, rd[u]);
            ldraw((const T *)x.p + bn_off(x, bi, y, xx) + g * 8, rv[u]);
            if (!WRITE) ldraw((const T *)dx.p + off[u], ro[u]);
            if (GATE) ldraw((const T *)act.p + bn_off(act, bi, y, xx) + g * 8, rm[u]);
        }
        float ca[8], cp[8], cq[8];
        coef8(coef + g * 8, ca);
        coef8(coef + 2 * Cp + g * 8, cp);
        coef8(coef + 3 * Cp + g * 8, cq);
#pragma unroll
        for (int u = 0; u < RP; ++u) {
            float d[8], v[8], o[8], m[8];
            unraw(rd[u], d);
            unraw(rv[u], v);
            if (!WRITE) unraw(ro[u], o);
            if (GATE) unraw(rm[u], m);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float dc = stat[u] ? fmaf(ca[k], d[k], fmaf(cq[k], v[k], cp[k])) : ca[k] * d[k];
                o[k] = (GATE && m[k] <= 0.f) ? 0.f : (WRITE ? dc : o[k] + dc);
            }
            if (r0 + u < nrows) store8((T *)dx.p + off[u], o);
        }
    }
}

dim3 grid_rows(int nv, int nrows, int per = kRowsPer) {
    const int gx = (nv + kBnThreads - 1) / kBnThreads;
    // about 8 blocks of 256 threads per SM in total, each striding over groups of `per` rows
    const int groups = (nrows + per - 1) / per;
    const int gy = std::max(1, std::min(std::min(groups, 65535), (148 * 8 + gx - 1) / gx));
    return dim3((unsigned)gx, (unsigned)gy);
}

template <int MODE>
cudaError_t bn_reduce(int prec, const View &x, const View &dy, const float *coef, int a, int b, int B, double *out,
                      cudaStream_t st) {
    if (b <= a) return cudaSuccess;
    const int G = x.Cp / 8;
    if (x.Cp % 8 || G > kBnThreads) return cudaErrorInvalidValue;
    const int lanes = kBnThreads / G;
    (void)lanes;
    const unsigned grid = (unsigned)std::max(1, std::min(B * (b - a), 148 * 8));
    if (prec && x.Cp / 4 <= kBnThreads) {   // bf16, Cp <= 1024: four channels per thread
        k_bn_reduce4<MODE><<<grid, kBnThreads, (size_t)kBnThreads * 8 * sizeof(double), st>>>(x, dy, coef, a, b, B, out);
        return cudaGetLastError();
    }
    const size_t smem = (size_t)kBnThreads * 16 * sizeof(double);
    if (prec) k_bn_reduce<bf16, MODE><<<grid, kBnThreads, smem, st>>>(x, dy, coef, a, b, B, out);
    else k_bn_reduce<float, MODE><<<grid, kBnThreads, smem, st>>>(x, dy, coef, a, b, B, out);
    return cudaGetLastError();
}

}  // namespace

cudaError_t bn_stats(int prec, const View &x, int a, int b, int B, double *sums, cudaStream_t st) {
    return bn_reduce<0>(prec, x, x, nullptr, a, b, B, sums, st);
}

cudaError_t bn_sums(int prec, const View &dy, const View &x, const float *coef, int a, int b, int B, double *S,
                    cudaStream_t st) {
    return bn_reduce<1>(prec, x, dy, coef, a, b, B, S, st);
}

cudaError_t bn_finalize_fwd(int prec, const double *sums, const void *gamma, const void *beta, int C, int Cp,
                            double M, float *coef, cudaStream_t st) {
    const unsigned g = (unsigned)((Cp + 127) / 128);
    if (prec) k_bn_finalize_fwd<bf16><<<g, 128, 0, st>>>(sums, (const bf16 *)gamma, (const bf16 *)beta, C, Cp, M, coef);
    else k_bn_finalize_fwd<float><<<g, 128, 0, st>>>(sums, (const float *)gamma, (const float *)beta, C, Cp, M, coef);
    return cudaGetLastError();
}

cudaError_t bn_finalize_bwd(const double *S, float *coef, int C, int Cp, double M, float *dgamma, float *dbeta,
                            cudaStream_t st) {
    k_bn_finalize_bwd<<<(unsigned)((Cp + 127) / 128), 128, 0, st>>>(S, coef, C, Cp, M, dgamma, dbeta);
    return cudaGetLastError();
}

cudaError_t bn_fwd(int prec, const View &in, const View &res, const View &out, const float *coef, int relu, int a,
                   int b, int B, cudaStream_t st) {
    const long long n = (long long)B * (b - a) * out.W * (out.Cp / 8);
    if (n <= 0) return cudaSuccess;
    if (out.Cp % 8) return cudaErrorInvalidValue;
    const int hr = res.p != nullptr;
    const dim3 grid = grid_rows(out.W * (out.Cp / 8), B * (b - a), kFwdRowsPer);
    if (prec) k_bn_fwd<bf16><<<grid, kBnThreads, 0, st>>>(in, res, out, coef, relu, hr, a, b, B);
    else k_bn_fwd<float><<<grid, kBnThreads, 0, st>>>(in, res, out, coef, relu, hr, a, b, B);
    return cudaGetLastError();
}

cudaError_t bn_bwd(int prec, const View &dy, const View &x, const View &dx, const View &act, int gate, int write,
                   const float *coef, int a, int b, int B, int cs, cudaStream_t st) {
    const long long n = (long long)B * (b - a) * dx.W * (dx.Cp / 8);
    if (n <= 0) return cudaSuccess;
    if (dx.Cp % 8) return cudaErrorInvalidValue;
    const int nv = dx.W * (dx.Cp / 8), nr = B * (b - a);
#define LRCNN_BN_BWD(G_, W_, RP_)                                                                             \
    do {                                                                                                      \
        const dim3 grid = grid_rows(nv, nr, RP_);                                                             \
        if (prec) k_bn_bwd<bf16, G_, W_, RP_><<<grid, kBnThreads, 0, st>>>(dy, x, dx, act, coef, a, b, B, cs); \
        else k_bn_bwd<float, G_, W_, RP_><<<grid, kBnThreads, 0, st>>>(dy, x, dx, act, coef, a, b, B, cs);   \
    } while (0)
    if (!gate && write) LRCNN_BN_BWD(false, true, 4);
    else if (!gate) LRCNN_BN_BWD(false, false, 2);
    else if (write) LRCNN_BN_BWD(true, true, 2);
    else LRCNN_BN_BWD(true, false, 2);
#undef LRCNN_BN_BWD
    return cudaGetLastError();
}

}  // namespace lrcnn

// Query rotation (K1), probe grouping (K3) and the per-pair DCO kernels that
// mirror DcoStrategy::evaluate / partial_sqdist / calibration's ratio walk.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

// ---- K1: out[i][k] = (float) sum_r W[k*D + r] * in[i][r] --------------------
// The reference's sum is a sequential chain of D rounded DMULs and DADDs
// (proj/src/transform.cpp:221-228). The kernel computes the same dot products
// on the FP64 tensor cores (mma.sync m8n8k4 f64, IEEE fp64 fused multiply-adds
// in some order) and proves that both results round to the same float: with
// S = sum_r |w_r x_r| <= |w| |x|, each of the two fp64 evaluations is within
// gamma_D S of the real value (gamma_D = D u / (1 - D u), u = 2^-53), so the
// reference's fp64 sum lies in [acc - E, acc + E], E = 2 gamma_D |w| |x|. When
// both ends of that interval round to the same float (RN is monotone), that
// float is the reference's output. Otherwise (a float rounding boundary inside
// the interval: ~1e-4 of the elements, and every NaN) the element is recomputed
// with the reference's exact DMUL/DADD chain, one lane per element after the
// CTA's main loop, so every output is bit-identical to transform_vector.
//
// 64 rows x 64 output columns per CTA of 4 warps, 32 x 32 per warp (4 x 4
// m8n8 tiles). Chunks of 16 r are staged by cp.async into double buffers (x as
// fp32 [row][r], stride 20 floats; W as fp64 [col][r], stride 20 doubles:
// conflict-free fragment loads), the next chunk in flight while the current one
// is multiplied; x is widened to fp64 at the fragment load. With no register
// staging the kernel fits 5 CTAs per SM, so 148 x 5 tiles run in one wave
// (config 1's 628 tiles took two waves at 4 per SM). The row / column norms are
// accumulated from the staged values.
// (A 32 x 32 tile with the K range split over the warps measured 1.5x slower:
// four times the staging per multiply-add.)
constexpr int kRotT = 64;    // rows and columns per CTA
constexpr int kRotK = 16;    // r chunk
constexpr int kRotS = 20;    // staged row stride (doubles / floats)
constexpr int kRotFix = 512; // per-CTA list of elements to recompute exactly

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ void rot_cp16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

__device__ __noinline__ float rotate_exact(const double* __restrict__ W, uint32_t dim, const float* __restrict__ in,
                                           uint32_t row, uint32_t col) {
    const double* w = W + (size_t)col * dim;
    const float* x = in + (size_t)row * dim;
    double acc = 0.0;
    for (uint32_t r = 0; r < dim; ++r) acc = __dadd_rn(acc, __dmul_rn(__ldg(w + r), (double)__ldg(x + r)));
    return __double2float_rn(acc);
}

// The same element by one warp (the kernels' fix lists): the products fl(w_r x_r) do not depend on the
// running sum, so the lanes form them 256 at a time from coalesced loads into shared memory (prod: 256
// doubles, warp-private) and lane 0 alone runs the reference's DADD chain over them, in r order. A single
// lane doing loads and chain (rotate_exact) waits one L2 round trip per r: ~150 us for one element at
// dim 960, which the whole CTA -- and at a one-wave grid the whole kernel -- then waits for.
__device__ __forceinline__ void rotate_exact_warp(const double* __restrict__ W, uint32_t dim,
                                                  const float* __restrict__ in, uint32_t row, uint32_t col,
                                                  double* prod, float* dst) {
    const uint32_t lane = threadIdx.x & 31;
    const double* w = W + (size_t)col * dim;
    const float* x = in + (size_t)row * dim;
    double acc = 0.0;
    for (uint32_t r0 = 0; r0 < dim; r0 += 256) {
        const uint32_t m = min(256u, dim - r0);
        __syncwarp();
#pragma unroll
        for (uint32_t i = 0; i < 256; i += 32)
            if (i + lane < m) prod[i + lane] = __dmul_rn(__ldg(w + r0 + i + lane), (double)__ldg(x + r0 + i + lane));
        __syncwarp();
        if (lane == 0) {
#pragma unroll 8
            for (uint32_t i = 0; i < m; ++i) acc = __dadd_rn(acc, prod[i]);
        }
    }
    if (lane == 0) *dst = __double2float_rn(acc);
}

__global__ void __launch_bounds__(128, 5)
rotate_kernel(const double* __restrict__ W, uint32_t dim, const float* __restrict__ in, uint32_t n,
              float* __restrict__ out, uint2* __restrict__ gfix, uint32_t* __restrict__ gfix_n, uint32_t gfix_cap) {
    __shared__ __align__(16) float xs[2][kRotT * kRotS];
    __shared__ __align__(16) double ws[2][kRotT * kRotS];
    __shared__ double wn[kRotT], xn[kRotT];
    __shared__ uint32_t fix[kRotFix];
    __shared__ uint32_t n_fix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;          // mma fragment coordinates
    const int wm = warp >> 1, wc = warp & 1;        // warp tile: rows 32 wm.., columns 32 wc..
    const uint32_t col0 = blockIdx.x * kRotT, row0 = blockIdx.y * kRotT;
    if (tid == 0) n_fix = 0;
    double c[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j][0] = c[i][j][1] = 0.0;
    // staging: thread tid owns row / column tid >> 1, r = r0 + 8 (tid & 1) .. + 7
    const uint32_t sr = tid >> 1, so = 8 * (tid & 1);
    const uint32_t xrow = row0 + sr, wcol = col0 + sr;
    const bool vec = dim % 4 == 0;
    double xsq = 0.0, wsq = 0.0;
    auto stage = [&](uint32_t r0, int b) {
        const uint32_t r = r0 + so;
        float* xd = &xs[b][sr * kRotS + so];
        double* wd = &ws[b][sr * kRotS + so];
        if (vec && r + 8 <= dim) {
            if (xrow < n) {
                rot_cp16(xd, in + (size_t)xrow * dim + r);
                rot_cp16(xd + 4, in + (size_t)xrow * dim + r + 4);
            } else {
                *reinterpret_cast<float4*>(xd) = make_float4(0.f, 0.f, 0.f, 0.f);
                *reinterpret_cast<float4*>(xd + 4) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            if (wcol < dim) {
#pragma unroll
                for (int e = 0; e < 8; e += 2) rot_cp16(wd + e, W + (size_t)wcol * dim + r + e);
            } else {
#pragma unroll
                for (int e = 0; e < 8; e += 2) *reinterpret_cast<double2*>(wd + e) = make_double2(0.0, 0.0);
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                xd[e] = (xrow < n && r + e < dim) ? __ldg(in + (size_t)xrow * dim + r + e) : 0.f;
                wd[e] = (wcol < dim && r + e < dim) ? __ldg(W + (size_t)wcol * dim + r + e) : 0.0;
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    stage(0, 0);
    int b = 0;
    for (uint32_t r0 = 0; r0 < dim; r0 += kRotK, b ^= 1) {
        if (r0 + kRotK < dim) {
            stage(r0 + kRotK, b ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        {  // this thread's row / column share of the norms
            const float* xv = &xs[b][sr * kRotS + so];
            const double* wv = &ws[b][sr * kRotS + so];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const double x = (double)xv[e];
                xsq = fma(x, x, xsq);
                wsq = fma(wv[e], wv[e], wsq);
            }
        }
        const float* xb = xs[b];
        const double* wb = ws[b];
#pragma unroll
        for (int k0 = 0; k0 < kRotK; k0 += 4) {
            double a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = (double)xb[(32 * wm + 8 * i + g) * kRotS + k0 + t];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = wb[(32 * wc + 8 * j + g) * kRotS + k0 + t];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(c[i][j], a[i], bb[j]);
        }
        __syncthreads();  // buffer b is restaged two chunks on
    }
    // norms (upper bounds after the 1.0001 margin below); lanes 2m, 2m + 1 share a row
    xsq += __shfl_xor_sync(0xffffffffu, xsq, 1);
    wsq += __shfl_xor_sync(0xffffffffu, wsq, 1);
    if ((tid & 1) == 0) {
        xn[sr] = sqrt(xsq);
        wn[sr] = sqrt(wsq);
    }
    __syncthreads();
    // E = 2 gamma_D |w| |x| with margin for the norms' own rounding
    const double gam = (double)(dim + 2) * 0x1p-52 * 1.0001;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const uint32_t rl = 32 * wm + 8 * i + g, row = row0 + rl;
        if (row >= n) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t cl = 32 * wc + 8 * j + 2 * t + h, col = col0 + cl;
                if (col >= dim) continue;
                const double acc = c[i][j][h];
                const double e = gam * wn[cl] * xn[rl];
                const float lo = __double2float_rn(__dsub_rd(acc, e));
                const float hi = __double2float_rn(__dadd_ru(acc, e));
                if (__float_as_uint(lo) == __float_as_uint(hi) && !isnan(lo)) {
                    out[(size_t)row * dim + col] = lo;
                } else if (gfix) {  // the launch-wide list: rotate_fix_kernel spreads these over the GPU
                    const uint32_t gs = atomicAdd(gfix_n, 1u);
                    if (gs < gfix_cap) gfix[gs] = make_uint2(row, col);
                    else out[(size_t)row * dim + col] = rotate_exact(W, dim, in, row, col);
                } else {
                    const uint32_t slot = atomicAdd(&n_fix, 1u);
                    if (slot < (uint32_t)kRotFix) fix[slot] = (rl << 8) | cl;
                    else out[(size_t)row * dim + col] = rotate_exact(W, dim, in, row, col);
                }
            }
    }
    __syncthreads();  // (the staging buffers are free: ws[0] holds the warps' product blocks)
    const uint32_t nf = min(n_fix, (uint32_t)kRotFix);
    for (uint32_t e = warp; e < nf; e += blockDim.x / 32) {
        const uint32_t row = row0 + (fix[e] >> 8), col = col0 + (fix[e] & 0xffu);
        rotate_exact_warp(W, dim, in, row, col, &ws[0][warp * 256], out + (size_t)row * dim + col);
    }
}

// Small batches (fewer 64 x 64 tiles than two per SM: configs 0 and 2, 1000
// queries) leave most SMs idle, so their rotation runs 32 x 32 output tiles with
// the r range split over the CTA's four warps: each warp stages its own r chunks
// (cp.async, warp-private double buffers) into its own 32 x 32 accumulator; the
// partial sums and partial norms are added in warp order (deterministic) and the
// same rounding proof applies (any summation order stays within gamma_{D+2}).
constexpr int kRkT = 32;                       // rows and columns per CTA
constexpr int kRkWarp = 2 * kRkT * kRotS * 12; // bytes per warp: x [2][32][20] f32 + W [2][32][20] f64

__global__ void __launch_bounds__(128, 4)
rotate_ksplit_kernel(const double* __restrict__ W, uint32_t dim, const float* __restrict__ in, uint32_t n,
                     float* __restrict__ out, uint2* __restrict__ gfix, uint32_t* __restrict__ gfix_n,
                     uint32_t gfix_cap) {
    extern __shared__ __align__(16) unsigned char rk_smem[];
    __shared__ double wn[kRkT], xn[kRkT];
    __shared__ uint32_t fix[kRotFix];
    __shared__ uint32_t n_fix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = lane >> 2, t = lane & 3;
    const uint32_t col0 = blockIdx.x * kRkT, row0 = blockIdx.y * kRkT;
    float* xs = reinterpret_cast<float*>(rk_smem + (size_t)warp * kRkWarp);            // [2][32][20]
    double* ws = reinterpret_cast<double*>(rk_smem + (size_t)warp * kRkWarp + 2 * kRkT * kRotS * 4);  // [2][32][20]
    if (tid == 0) n_fix = 0;
    double c[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) c[i][j][0] = c[i][j][1] = 0.0;
    const uint32_t nch = (dim + kRotK - 1) / kRotK;
    const uint32_t ch0 = warp * nch / 4, ch1 = (warp + 1) * nch / 4;
    const uint32_t xrow = row0 + lane, wcol = col0 + lane;
    const bool vec = dim % 4 == 0;
    double xsq = 0.0, wsq = 0.0;
    auto stage = [&](uint32_t ch, int b) {  // lane: row / column lane, r = 16 ch .. + 15
        const uint32_t r = ch * kRotK;
        float* xd = xs + b * kRkT * kRotS + lane * kRotS;
        double* wd = ws + b * kRkT * kRotS + lane * kRotS;
        if (vec && r + kRotK <= dim) {
#pragma unroll
            for (int e = 0; e < kRotK; e += 4) {
                if (xrow < n) rot_cp16(xd + e, in + (size_t)xrow * dim + r + e);
                else *reinterpret_cast<float4*>(xd + e) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int e = 0; e < kRotK; e += 2) {
                if (wcol < dim) rot_cp16(wd + e, W + (size_t)wcol * dim + r + e);
                else *reinterpret_cast<double2*>(wd + e) = make_double2(0.0, 0.0);
            }
        } else {
            for (int e = 0; e < kRotK; ++e) {
                xd[e] = (xrow < n && r + e < dim) ? __ldg(in + (size_t)xrow * dim + r + e) : 0.f;
                wd[e] = (wcol < dim && r + e < dim) ? __ldg(W + (size_t)wcol * dim + r + e) : 0.0;
            }
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    if (ch0 < ch1) stage(ch0, 0);
    int b = 0;
    for (uint32_t ch = ch0; ch < ch1; ++ch, b ^= 1) {
        if (ch + 1 < ch1) {
            stage(ch + 1, b ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncwarp();
        const float* xb = xs + b * kRkT * kRotS;
        const double* wb = ws + b * kRkT * kRotS;
#pragma unroll
        for (int e = 0; e < kRotK; ++e) {
            const double x = (double)xb[lane * kRotS + e];
            xsq = fma(x, x, xsq);
            wsq = fma(wb[lane * kRotS + e], wb[lane * kRotS + e], wsq);
        }
#pragma unroll
        for (int k0 = 0; k0 < kRotK; k0 += 4) {
            double a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = (double)xb[(8 * i + g) * kRotS + k0 + t];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = wb[(8 * j + g) * kRotS + k0 + t];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) dmma(c[i][j], a[i], bb[j]);
        }
        __syncwarp();  // buffer b is restaged two chunks on
    }
    __syncthreads();  // every warp done with its staging: reuse it for the partials
    double* part = reinterpret_cast<double*>(rk_smem);  // [3][32 x 32] of warps 1-3, then norms [3][2][32]
    double* pnorm = part + 3 * kRkT * kRkT;
    if (warp > 0) {
        double* pw = part + (warp - 1) * kRkT * kRkT;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) pw[(8 * i + g) * kRkT + 8 * j + 2 * t + h] = c[i][j][h];
        pnorm[(warp - 1) * 2 * kRkT + lane] = xsq;
        pnorm[(warp - 1) * 2 * kRkT + kRkT + lane] = wsq;
    }
    __syncthreads();
    if (warp == 0) {
        for (int w = 0; w < 3; ++w) {
            const double* pw = part + w * kRkT * kRkT;
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int h = 0; h < 2; ++h) c[i][j][h] += pw[(8 * i + g) * kRkT + 8 * j + 2 * t + h];
            xsq += pnorm[w * 2 * kRkT + lane];
            wsq += pnorm[w * 2 * kRkT + kRkT + lane];
        }
        xn[lane] = sqrt(xsq);
        wn[lane] = sqrt(wsq);
        __syncwarp();
        const double gam = (double)(dim + 2) * 0x1p-52 * 1.0001;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const uint32_t rl = 8 * i + g, row = row0 + rl;
            if (row >= n) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t cl = 8 * j + 2 * t + h, col = col0 + cl;
                    if (col >= dim) continue;
                    const double acc = c[i][j][h];
                    const double e = gam * wn[cl] * xn[rl];
                    const float lo = __double2float_rn(__dsub_rd(acc, e));
                    const float hi = __double2float_rn(__dadd_ru(acc, e));
                    if (__float_as_uint(lo) == __float_as_uint(hi) && !isnan(lo)) {
                        out[(size_t)row * dim + col] = lo;
                    } else if (gfix) {
                        const uint32_t gs = atomicAdd(gfix_n, 1u);
                        if (gs < gfix_cap) gfix[gs] = make_uint2(row, col);
                        else out[(size_t)row * dim + col] = rotate_exact(W, dim, in, row, col);
                    } else {
                        const uint32_t slot = atomicAdd(&n_fix, 1u);
                        if (slot < (uint32_t)kRotFix) fix[slot] = (rl << 8) | cl;
                        else out[(size_t)row * dim + col] = rotate_exact(W, dim, in, row, col);
                    }
                }
        }
    }
    __syncthreads();  // (the staging buffers are free: rk_smem holds the warps' product blocks)
    const uint32_t nf = min(n_fix, (uint32_t)kRotFix);
    for (uint32_t e = warp; e < nf; e += blockDim.x / 32) {
        const uint32_t row = row0 + (fix[e] >> 8), col = col0 + (fix[e] & 0xffu);
        rotate_exact_warp(W, dim, in, row, col, reinterpret_cast<double*>(rk_smem) + warp * 256,
                          out + (size_t)row * dim + col);
    }
}

// ---- K3: grouping ------------------------------------------------------------
__device__ __forceinline__ uint32_t rank_bucket(const GroupArgs& g, uint32_t p) {
    uint32_t b = 0;
    while (b + 1 < g.n_rb && p >= g.rb_end[b]) ++b;
    return b;
}

__global__ void group_count_kernel(const GroupArgs g) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)g.nq * g.n_probe) return;
    const uint32_t p = (uint32_t)(i % g.n_probe);
    const uint32_t list = (uint32_t)g.probes[i];
    if (list >= g.n_lists) return;
    if (g.list_offsets[list + 1] == g.list_offsets[list]) return;  // empty / not on this shard
    atomicAdd(&g.counts[rank_bucket(g, p) * g.n_lists + list], 1u);
}

// Shared-memory variants (n_rb * n_lists <= kGroupSmemEntries): a CTA counts a
// contiguous range of (query, probe) pairs in shared memory and flushes one
// global atomic per touched entry, so a list probed by most queries costs one
// atomic per CTA instead of one per query.
constexpr uint32_t kGroupSmemEntries = 12288;
constexpr uint32_t kGroupPerThread = 4;   // pairs per thread (more CTAs: count 18 -> 8 us, scatter 27 -> 14 us at config 1)

__device__ __forceinline__ uint32_t pair_entry(const GroupArgs& g, size_t i) {
    const uint32_t p = (uint32_t)(i % g.n_probe);
    const uint32_t list = (uint32_t)g.probes[i];
    if (list >= g.n_lists || g.list_offsets[list + 1] == g.list_offsets[list]) return 0xffffffffu;
    return rank_bucket(g, p) * g.n_lists + list;
}

__global__ void __launch_bounds__(256) group_count_smem_kernel(const GroupArgs g) {
    extern __shared__ uint32_t gsh[];
    const uint32_t ne = g.n_rb * g.n_lists;
    for (uint32_t e = threadIdx.x; e < ne; e += blockDim.x) gsh[e] = 0;
    __syncthreads();
    const size_t n = (size_t)g.nq * g.n_probe;
    const size_t base = (size_t)blockIdx.x * blockDim.x * kGroupPerThread;
#pragma unroll 4
    for (uint32_t j = 0; j < kGroupPerThread; ++j) {
        const size_t i = base + (size_t)j * blockDim.x + threadIdx.x;
        if (i < n) {
            const uint32_t e = pair_entry(g, i);
            if (e != 0xffffffffu) atomicAdd(&gsh[e], 1u);
        }
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < ne; e += blockDim.x)
        if (gsh[e]) atomicAdd(&g.counts[e], gsh[e]);
}

__global__ void __launch_bounds__(256) group_scatter_smem_kernel(const GroupArgs g) {
    extern __shared__ uint32_t gsh[];
    const uint32_t ne = g.n_rb * g.n_lists;
    for (uint32_t e = threadIdx.x; e < ne; e += blockDim.x) gsh[e] = 0;
    __syncthreads();
    const size_t n = (size_t)g.nq * g.n_probe;
    const size_t base = (size_t)blockIdx.x * blockDim.x * kGroupPerThread;
    uint32_t ent[kGroupPerThread], loc[kGroupPerThread];
#pragma unroll
    for (uint32_t j = 0; j < kGroupPerThread; ++j) {
        const size_t i = base + (size_t)j * blockDim.x + threadIdx.x;
        ent[j] = i < n ? pair_entry(g, i) : 0xffffffffu;
        loc[j] = ent[j] != 0xffffffffu ? atomicAdd(&gsh[ent[j]], 1u) : 0u;
    }
    __syncthreads();
    // this CTA's range inside every touched entry
    for (uint32_t e = threadIdx.x; e < ne; e += blockDim.x)
        if (gsh[e]) gsh[e] = g.bucket_off[e] + atomicAdd(&g.cursor[e], gsh[e]);
    __syncthreads();
#pragma unroll
    for (uint32_t j = 0; j < kGroupPerThread; ++j) {
        if (ent[j] == 0xffffffffu) continue;
        const size_t i = base + (size_t)j * blockDim.x + threadIdx.x;
        const uint32_t pos = gsh[ent[j]] + loc[j];
        g.bucket_q[pos] = (uint32_t)(i / g.n_probe);
        g.bucket_slot[pos] = (uint32_t)(i % g.n_probe);
    }
}

// Single-CTA exclusive scans of the bucket sizes and item counts.
// work items of one (rank bucket, list) entry: query chunks x row pieces
// Rows [skip, len) of an entry's list still to scan: rank-bucket-0 entries skip
// the rows the seed already scored exactly (when the seed ran: len >= seed_min).
__device__ __forceinline__ uint32_t entry_skip(const GroupArgs& g, uint32_t e, uint32_t len) {
    return (g.seed_skip && e < g.n_lists && len >= g.seed_min) ? min(len, g.seed_skip) : 0u;
}

__device__ __forceinline__ uint32_t entry_piece(const GroupArgs& g, uint32_t e) {
    return (e < g.n_lists && g.rank0_item_rows) ? g.rank0_item_rows : g.max_item_rows;
}

__device__ __forceinline__ uint32_t entry_items(const GroupArgs& g, uint32_t e, uint32_t c) {
    if (c == 0) return 0;
    const uint32_t list = e % g.n_lists;
    const uint32_t len = g.list_offsets[list + 1] - g.list_offsets[list];
    const uint32_t rem = len - entry_skip(g, e, len);
    if (rem == 0) return 0;
    uint32_t pieces = 1;
    const uint32_t pr = entry_piece(g, e);
    if (pr) pieces = max(1u, (rem + pr - 1) / pr);
    return (c + g.q_chunk - 1) / g.q_chunk * pieces;
}

__global__ void __launch_bounds__(1024) group_scan_kernel(const GroupArgs g) {
    __shared__ uint32_t s_b[1024], s_i[1024], s_g[1024];
    const uint32_t n = g.n_rb * g.n_lists;
    const uint32_t per = (n + 1023) / 1024;
    const uint32_t lo = threadIdx.x * per, hi = min(n, lo + per);
    uint32_t sb = 0, si = 0, sg = 0;
    for (uint32_t e = lo; e < hi; ++e) {
        const uint32_t c = g.counts[e];
        sb += c;
        si += entry_items(g, e, c);
        if (e < g.n_lists) sg += (c + kSeedGroup - 1) / kSeedGroup;  // seed groups of the nearest-list bucket
    }
    s_b[threadIdx.x] = sb;
    s_i[threadIdx.x] = si;
    s_g[threadIdx.x] = sg;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
        const uint32_t vb = threadIdx.x >= (unsigned)off ? s_b[threadIdx.x - off] : 0;
        const uint32_t vi = threadIdx.x >= (unsigned)off ? s_i[threadIdx.x - off] : 0;
        const uint32_t vg = threadIdx.x >= (unsigned)off ? s_g[threadIdx.x - off] : 0;
        __syncthreads();
        s_b[threadIdx.x] += vb;
        s_i[threadIdx.x] += vi;
        s_g[threadIdx.x] += vg;
        __syncthreads();
    }
    uint32_t rb = s_b[threadIdx.x] - sb, ri = s_i[threadIdx.x] - si, rg = s_g[threadIdx.x] - sg;
    for (uint32_t e = lo; e < hi; ++e) {
        const uint32_t c = g.counts[e];
        g.bucket_off[e] = rb;
        g.item_off[e] = ri;
        if (g.seed_goff && e < g.n_lists) {
            g.seed_goff[e] = rg;
            if (g.seed_glist)
                for (uint32_t j = 0; j < (c + kSeedGroup - 1) / kSeedGroup; ++j) g.seed_glist[rg + j] = e;
        }
        rb += c;
        ri += entry_items(g, e, c);
        if (e < g.n_lists) rg += (c + kSeedGroup - 1) / kSeedGroup;
    }
    if (g.seed_goff && threadIdx.x == 1023) g.seed_goff[g.n_lists] = s_g[1023];
    if (threadIdx.x == 1023) g.n_items[0] = s_i[1023];
    __syncthreads();
    // items of rank bucket 0 (every query's nearest list) come first
    if (threadIdx.x == 0) g.n_items[1] = g.n_rb > 1 ? g.item_off[g.n_lists] : s_i[1023];
}

__global__ void group_scatter_kernel(const GroupArgs g) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)g.nq * g.n_probe) return;
    const uint32_t q = (uint32_t)(i / g.n_probe), p = (uint32_t)(i % g.n_probe);
    const uint32_t list = (uint32_t)g.probes[i];
    if (list >= g.n_lists) return;
    if (g.list_offsets[list + 1] == g.list_offsets[list]) return;
    const uint32_t e = rank_bucket(g, p) * g.n_lists + list;
    const uint32_t pos = g.bucket_off[e] + atomicAdd(&g.cursor[e], 1u);
    g.bucket_q[pos] = q;
    g.bucket_slot[pos] = p;
}

// One thread per work item: its entry is the last one whose item offset is <= t.
__global__ void __launch_bounds__(256) group_items_kernel(const GroupArgs g) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= g.n_items[0]) return;
    const uint32_t ne = g.n_rb * g.n_lists;
    uint32_t lo = 0, hi = ne;  // item_off[lo] <= t < item_off[hi] (item_off[ne] := inf)
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (g.item_off[mid] <= t) lo = mid; else hi = mid;
    }
    const uint32_t e = lo;
    const uint32_t c = g.counts[e];
    const uint32_t list = e % g.n_lists;
    const uint32_t len0 = g.list_offsets[list + 1] - g.list_offsets[list];
    const uint32_t skip = entry_skip(g, e, len0);
    const uint32_t start = g.list_offsets[list] + skip, len = len0 - skip;
    const uint32_t pr = entry_piece(g, e);
    const uint32_t piece = pr ? pr : max(len, 1u);
    const uint32_t np = max(1u, (len + piece - 1) / piece);
    const uint32_t li = t - g.item_off[e];
    // query chunk major, row piece minor; piece major for the flat scan, so the
    // consecutive items (started together on different SMs) share one row piece
    // and read it from HBM once for all query chunks
    const uint32_t nqc = (c + g.q_chunk - 1) / g.q_chunk;
    const uint32_t tq = g.piece_major ? li % nqc : li / np;
    const uint32_t p = g.piece_major ? li / nqc : li - tq * np;
    WorkItem w;
    w.row_start = start + p * piece;
    w.row_count = min(piece, len - p * piece);
    w.bucket_start = g.bucket_off[e] + tq * g.q_chunk;
    w.bucket_count = min(g.q_chunk, c - tq * g.q_chunk) | (min(p, 0xffffu) << 16);
    g.items[t] = w;
}

// ---- per-pair DCO: checkpointed_scan (proj/src/estimator.cpp:24-70) ------------
__global__ void evaluate_kernel(const float* __restrict__ o, const float* __restrict__ q,
                                const float* __restrict__ r, uint32_t n, uint32_t dim,
                                const uint32_t* __restrict__ cps, const double* __restrict__ coeff,
                                const double* __restrict__ scale, uint32_t n_ckpt, uint8_t* pruned,
                                float* dist, uint8_t* exact, uint32_t* dims_used,
                                unsigned long long* counters) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* oi = o + (size_t)i * dim;
    const float* qi = q + (size_t)i * dim;
    const float ri = r[i];
    const double r2 = __dmul_rn((double)ri, (double)ri);
    float acc = 0.f;
    uint32_t prev = 0;
    bool pr = false, ex = true;
    float d_out = 0.f;
    uint32_t used = dim;
    for (uint32_t ci = 0; ci < n_ckpt; ++ci) {
        const uint32_t d = cps[ci];
        for (uint32_t k = prev; k < d; ++k) acc = sq_step(acc, oi[k], qi[k]);
        prev = d;
        if ((double)acc > __dmul_rn(coeff[ci], r2)) {
            pr = true;
            ex = false;
            d_out = __double2float_rn(__dsqrt_rn(__dmul_rn(scale[ci], (double)acc)));
            used = d;
            break;
        }
    }
    float full = acc;
    const uint32_t from = pr ? used : prev;
    for (uint32_t k = from; k < dim; ++k) full = sq_step(full, oi[k], qi[k]);
    if (!pr) {
        d_out = __fsqrt_rn(full);
        pr = d_out > ri;
    }
    pruned[i] = pr;
    dist[i] = d_out;
    exact[i] = ex;
    dims_used[i] = used;
    if (counters) {
        atomicAdd(counters + 0, 1ull);
        atomicAdd(counters + 1, (unsigned long long)used);
        // failure accounting (record_failure_check, estimator.cpp:24-33)
        if (__fsqrt_rn(full) <= ri) {
            atomicAdd(counters + 2, 1ull);
            if (pr) atomicAdd(counters + 3, 1ull);
        }
    }
}

__global__ void partial_sums_kernel(const float* __restrict__ o, const float* __restrict__ q, uint32_t n,
                                    uint32_t dim, const uint32_t* __restrict__ cps, uint32_t n_ckpt,
                                    float* out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* oi = o + (size_t)i * dim;
    const float* qi = q + (size_t)i * dim;
    float acc = 0.f;
    uint32_t prev = 0;
    for (uint32_t ci = 0; ci <= n_ckpt; ++ci) {
        const uint32_t d = ci < n_ckpt ? cps[ci] : dim;
        for (uint32_t k = prev; k < d; ++k) acc = sq_step(acc, oi[k], qi[k]);
        prev = d;
        out[(size_t)i * (n_ckpt + 1) + ci] = acc;
    }
}

// collect_ratios' running accumulator (proj/src/calibration.cpp:40-50) on
// sampled pairs (i, j): out[p][ci] = partial at checkpoint ci, out[p][n] = full.
__global__ void pair_partials_kernel(const float* __restrict__ data, uint32_t dim,
                                     const uint32_t* __restrict__ pi, const uint32_t* __restrict__ pj,
                                     uint64_t n, const uint32_t* __restrict__ cps, uint32_t n_ckpt,
                                     float* out) {
    const uint64_t p = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const float* a = data + (size_t)pi[p] * dim;
    const float* b = data + (size_t)pj[p] * dim;
    float acc = 0.f;
    uint32_t prev = 0;
    for (uint32_t ci = 0; ci <= n_ckpt; ++ci) {
        const uint32_t d = ci < n_ckpt ? cps[ci] : dim;
        for (uint32_t k = prev; k < d; ++k) acc = sq_step(acc, a[k], b[k]);
        prev = d;
        out[p * (n_ckpt + 1) + ci] = acc;
    }
}

// ---- radius seed: exact distances to the first rows of each query's nearest list
// One CTA (256 threads) per query: S <= kSeedMax rows of its rank-0 list, two
// rows per thread with interleaved exact sequential fp32 accumulations
// (sqrtf: the search's key space), bitonic sort in shared memory, K-th
// smallest -> atomicMin(r_global). Any K exact distances to probed candidates
// bound the final K-th distance, so the seed is safe.
constexpr int kSeedMax = 512;
constexpr int kSeedThreads = 256;
// With out_keys, the seed also becomes the query's first K results: its keys are
// exact (dist, id) of rows [0, S) of the nearest list, and the streaming scan
// skips those rows (GroupArgs::seed_skip), so nothing is evaluated twice and
// every query holds K results before any pruning, like the reference's heap.
__global__ void __launch_bounds__(kSeedThreads) seed_radius_kernel(
    const uint64_t* __restrict__ probes, uint32_t n_probe, const uint32_t* __restrict__ list_offsets,
    const float* __restrict__ storage, const uint32_t* __restrict__ row_ids, uint32_t dim,
    const float* __restrict__ queries, uint32_t nq, uint32_t K, uint32_t S, uint32_t* r_global, uint64_t* out_keys,
    uint32_t* out_count) {
    extern __shared__ __align__(16) unsigned char seed_smem[];
    float* seed_tile = reinterpret_cast<float*>(seed_smem);      // [kSeedMax][36] staged slices
    uint64_t* d = reinterpret_cast<uint64_t*>(seed_smem);        // keys, after the tile is consumed
    const uint32_t q = blockIdx.x;
    const uint32_t list = (uint32_t)probes[(size_t)q * n_probe];
    if (list == 0xffffffffu) return;  // no probed list on this shard (local_probes_kernel)
    const uint32_t start = list_offsets[list], len = list_offsets[list + 1] - start;
    const uint32_t n = min(len, S);
    if (n < K) return;  // too few rows for a K-th distance (uniform per CTA)
    const float* qr = queries + (size_t)q * dim;
    const uint32_t r0 = threadIdx.x, r1 = threadIdx.x + kSeedThreads;
    float a0 = 0.f, a1 = 0.f;
    if ((dim & 3u) == 0) {
        // Stage 32-dim slices of all S rows in shared memory with coalesced
        // 16-byte loads (row stride 36 floats: conflict-free LDS.128), then each
        // thread advances its two rows' exact sequential sums from smem.
        float* tile = seed_tile;
        // this thread stages 16-byte column c4 of rows rb + 32 m (m < 16) of every slice
        const uint32_t c4 = threadIdx.x & 7, rb = threadIdx.x >> 3;
        const float* rowp = storage + (size_t)(start + min(rb, n - 1)) * dim + 4 * c4;
        const size_t rstep = (size_t)32 * dim;
        for (uint32_t k0 = 0; k0 < dim; k0 += 32) {
            const uint32_t w = min(32u, dim - k0), w4 = w >> 2;
            __syncthreads();
            float4 v[16];
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const uint32_t r = rb + 32 * m;
                v[m] = (r < n && c4 < w4) ? __ldg(reinterpret_cast<const float4*>(rowp + m * rstep + k0))
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int m = 0; m < 16; ++m) *reinterpret_cast<float4*>(tile + (rb + 32 * m) * 36 + 4 * c4) = v[m];
            __syncthreads();
            for (uint32_t c4 = 0; c4 < w4; ++c4) {
                const float4 y = __ldg(reinterpret_cast<const float4*>(qr + k0) + c4);
                const float4 x0 = *reinterpret_cast<const float4*>(tile + r0 * 36 + 4 * c4);
                const float4 x1 = *reinterpret_cast<const float4*>(tile + r1 * 36 + 4 * c4);
                a0 = sq_step(a0, x0.x, y.x); a1 = sq_step(a1, x1.x, y.x);
                a0 = sq_step(a0, x0.y, y.y); a1 = sq_step(a1, x1.y, y.y);
                a0 = sq_step(a0, x0.z, y.z); a1 = sq_step(a1, x1.z, y.z);
                a0 = sq_step(a0, x0.w, y.w); a1 = sq_step(a1, x1.w, y.w);
            }
        }
        __syncthreads();
    } else {
        const float* o0 = storage + (size_t)(start + min(r0, n - 1)) * dim;
        const float* o1 = storage + (size_t)(start + min(r1, n - 1)) * dim;
        for (uint32_t k = 0; k < dim; ++k) {
            const float y = __ldg(qr + k);
            a0 = sq_step(a0, __ldg(o0 + k), y);
            a1 = sq_step(a1, __ldg(o1 + k), y);
        }
    }
    auto key_of = [&](uint32_t r, float acc) -> uint64_t {
        if (r >= n) return ~0ull;
        const uint32_t id = row_ids ? __ldg(row_ids + start + r) : start + r;
        return make_key(__fsqrt_rn(acc), id);
    };
    d[r0] = key_of(r0, a0);
    d[r1] = key_of(r1, a1);
    __syncthreads();
    // bitonic sort of kSeedMax (dist, id) keys, ascending: one compare-exchange per thread per stage
    for (uint32_t size = 2; size <= (uint32_t)kSeedMax; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            const uint32_t i = threadIdx.x;
            const uint32_t lo = 2 * i - (i & (stride - 1));
            const uint32_t hi = lo + stride;
            const bool up = (lo & size) == 0;
            const uint64_t x = d[lo], y = d[hi];
            if ((x > y) == up) {
                d[lo] = y;
                d[hi] = x;
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) atomicMin(r_global + q, (uint32_t)(d[K - 1] >> 32));
    if (out_keys) {
        for (uint32_t i = threadIdx.x; i < K; i += kSeedThreads) out_keys[(size_t)q * K + i] = d[i];
        if (threadIdx.x == 0) out_count[q] = K;
    }
}

// List-major seed: one CTA per (nearest list, group of up to 8 of the queries
// whose nearest list it is). The list's first S rows stream through shared
// memory in 16-dim slices (cp.async, double-buffered, shared by the group);
// every thread advances rows (t, t + 256) x G queries of exact sequential fp32
// sums with packed f32x2 arithmetic (two queries per instruction, same
// rounding as sq_step); then one warp per query sorts its S keys. Same output
// as seed_radius_kernel. Requires dim % 4 == 0 (the streaming path's rule).
constexpr int kSeedListMax = 1024;             // rows per list seed (up to 4 per thread)
constexpr int kSeedSlice8 = 8;                  // dims per staged slice
constexpr int kSeedRS = kSeedSlice8 + 4;        // padded row stride (floats): conflict-free LDS.128
constexpr int kSeedTileF = kSeedListMax * kSeedRS; // floats per tile buffer

__device__ __forceinline__ void cp_async16_s(void* dst, const void* src, bool pred) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(pred ? 16 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async4_s(void* dst, const void* src, bool pred) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src), "r"(pred ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// exact sums of rows (tid + 256 j, j < kR) x G queries over all dims -> accs[u][row]
template <int G, int kR>
__device__ __forceinline__ void seed_group_sums(float* tile, float* qt, float* accs, const float* storage,
                                                uint32_t start, uint32_t n, uint32_t dim, const float* queries,
                                                const uint32_t* qs, uint32_t ng, uint64_t nz2) {
    const uint32_t tid = threadIdx.x;
    const uint32_t n_slices = (dim + kSeedSlice8 - 1) / kSeedSlice8;
    auto issue = [&](uint32_t sl, uint32_t buf) {
        const uint32_t k0 = sl * kSeedSlice8;
        float* tb = tile + buf * kSeedTileF;
        constexpr uint32_t kCh = kSeedSlice8 / 4;  // 16-byte chunks per row slice
#pragma unroll
        for (int i = 0; i < (kR * kSeedThreads * (int)kCh) / kSeedThreads; ++i) {
            const uint32_t idx = tid + i * kSeedThreads, row = idx / kCh, c4 = idx % kCh;
            const bool ok = row < n && k0 + 4 * c4 < dim;
            const float* src = storage + (size_t)(start + (ok ? row : 0)) * dim + (ok ? k0 + 4 * c4 : 0);
            cp_async16_s(tb + row * kSeedRS + 4 * c4, src, ok);
        }
        static_assert(kSeedSlice8 * kSeedGroup <= kSeedThreads, "one query element per thread");
        if (tid < (uint32_t)(kSeedSlice8 * kSeedGroup)) {  // qt[buf][k][u]
            const uint32_t k = tid / kSeedGroup, u = tid % kSeedGroup;
            const bool ok = u < ng && k0 + k < dim;
            const float* src = queries + (ok ? (size_t)qs[u] * dim + k0 + k : 0);
            cp_async4_s(qt + buf * kSeedSlice8 * kSeedGroup + k * kSeedGroup + u, src, ok);
        }
        cp_async_commit();
    };
    uint64_t acc[kR][G / 2];
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int p = 0; p < G / 2; ++p) acc[j][p] = 0ull;
    issue(0, 0);
    for (uint32_t sl = 0; sl < n_slices; ++sl) {
        const uint32_t buf = sl & 1;
        if (sl + 1 < n_slices) {
            issue(sl + 1, buf ^ 1);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const float* tb = tile + buf * kSeedTileF;
        const float* qb = qt + buf * kSeedSlice8 * kSeedGroup;
#pragma unroll
        for (int c = 0; c < kSeedSlice8 / 4; ++c) {
            float o[kR][4];
#pragma unroll
            for (int j = 0; j < kR; ++j) {
                const float4 x = *reinterpret_cast<const float4*>(tb + (tid + j * kSeedThreads) * kSeedRS + 4 * c);
                o[j][0] = x.x;
                o[j][1] = x.y;
                o[j][2] = x.z;
                o[j][3] = x.w;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                // query pairs of this dim, two per 16-byte load (the queries are broadcast)
                const ulonglong2* q4 = reinterpret_cast<const ulonglong2*>(qb + (4 * c + e) * kSeedGroup);
                uint64_t qp[G / 2 + 1];
#pragma unroll
                for (int p = 0; p < G / 2; p += 2) {
                    const ulonglong2 v = q4[p / 2];
                    qp[p] = v.x;
                    qp[p + 1] = v.y;
                }
#pragma unroll
                for (int j = 0; j < kR; ++j)
#pragma unroll
                    for (int p = 0; p < G / 2; ++p) acc[j][p] = sq_step2(acc[j][p], o[j][e], qp[p], nz2);
            }
        }
        __syncthreads();  // buffer free for the slice after next
    }
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int p = 0; p < G / 2; ++p) {
            const uint32_t r = tid + j * kSeedThreads;
            accs[(2 * p) * kSeedListMax + r] = lo_f(acc[j][p]);
            accs[(2 * p + 1) * kSeedListMax + r] = hi_f(acc[j][p]);
        }
    __syncthreads();
}

// ascending bitonic sort of m (power of two) keys in shared memory by one warp
__device__ __forceinline__ void warp_bitonic_sort(uint64_t* kk, uint32_t m, uint32_t lane) {
    for (uint32_t size = 2; size <= m; size <<= 1) {
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = lane; i < m / 2; i += 32) {
                const uint32_t lo = 2 * i - (i & (stride - 1));
                const uint32_t hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t x = kk[lo], y = kk[hi];
                if ((x > y) == up) {
                    kk[lo] = y;
                    kk[hi] = x;
                }
            }
            __syncwarp();
        }
    }
}

constexpr int kSeedSmall = 128;  // sorted slots when the K-th distance has few ties

// K-th smallest (1-based) of the first n sqrt(acc) values as float bits
// (positive floats order like their bits): warp radix select, 8 bits per
// pass, histogram in shared memory. Requires K <= n <= kSeedMax.
template <int NV>
__device__ __forceinline__ uint32_t warp_select_regs(const uint32_t (&v)[NV], uint32_t K, uint32_t* hist,
                                                     uint32_t lane) {
    uint32_t prefix = 0, mask = 0, rem = K;
    for (int shift = 24; shift >= 0; shift -= 8) {
        for (uint32_t j = lane; j < 256; j += 32) hist[j] = 0;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if ((v[i] & mask) == prefix) atomicAdd(&hist[(v[i] >> shift) & 0xffu], 1u);
        __syncwarp();
        uint32_t d, before;
        warp_hist_find(hist, rem, lane, d, before);
        rem -= before;
        prefix |= d << shift;
        mask |= 0xffu << shift;
        __syncwarp();
    }
    return prefix;
}

__global__ void __launch_bounds__(kSeedThreads, 2) seed_radius_list_kernel(
    const uint32_t* __restrict__ counts, const uint32_t* __restrict__ bucket_off, const uint32_t* __restrict__ bucket_q,
    const uint32_t* __restrict__ seed_goff, const uint32_t* __restrict__ seed_glist, uint32_t n_lists,
    const uint32_t* __restrict__ list_offsets, const float* __restrict__ storage,
    const uint32_t* __restrict__ row_ids, uint32_t id_base, uint32_t dim, const float* __restrict__ queries, uint32_t K,
    uint32_t S, uint32_t* r_global, uint64_t* out_keys, uint32_t* out_count, uint64_t nz2) {
    extern __shared__ __align__(16) unsigned char seed_smem[];
    float* tile = reinterpret_cast<float*>(seed_smem);                  // [2][kSeedMax][kSeedRS]
    float* qt = tile + 2 * kSeedTileF;                                  // [2][kSeedSlice8][kSeedGroup]
    // after the last slice the tile's space is reused: sums, then sort keys
    float* accs = tile;                                                 // [kSeedGroup][kSeedListMax]
    uint64_t* keys = reinterpret_cast<uint64_t*>(tile + kSeedGroup * kSeedListMax);  // [8 warps][kSeedSmall], then hist [8][256]
    // CTA -> (list, group): binary search in the per-list group prefix
    const uint32_t b = blockIdx.x;
    if (b >= seed_goff[n_lists]) return;
    const uint32_t list = seed_glist[b];
    const uint32_t cnt_all = counts[list];  // entry e = list of rank bucket 0
    const uint32_t g0 = (b - seed_goff[list]) * kSeedGroup;
    if (g0 >= cnt_all) return;
    const uint32_t start = list_offsets[list], len = list_offsets[list + 1] - start;
    const uint32_t n = min(len, S);
    if (n < K) return;
    const uint32_t* qs = bucket_q + bucket_off[list] + g0;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t ng = min((uint32_t)kSeedGroup, cnt_all - g0);
    const int rsel = n > 2u * kSeedThreads ? 4 : n > (uint32_t)kSeedThreads ? 2 : 1;
    switch ((ng + 1) >> 1) {  // G = ng rounded up to even: no padded query pairs beyond one
#define SEED_G(P)                                                                                      \
    case P:                                                                                            \
        if (rsel == 4)                                                                                 \
            seed_group_sums<2 * P, 4>(tile, qt, accs, storage, start, n, dim, queries, qs, ng, nz2);   \
        else if (rsel == 2)                                                                            \
            seed_group_sums<2 * P, 2>(tile, qt, accs, storage, start, n, dim, queries, qs, ng, nz2);   \
        else                                                                                           \
            seed_group_sums<2 * P, 1>(tile, qt, accs, storage, start, n, dim, queries, qs, ng, nz2);   \
        break;
        SEED_G(1) SEED_G(2) SEED_G(3) SEED_G(4) SEED_G(5) SEED_G(6) SEED_G(7) default: SEED_G(8)
#undef SEED_G
    }
    for (uint32_t u = warp; u < ng; u += kSeedThreads / 32) {  // one warp per query: K-th distance, sorted top-K keys
        const uint32_t q = qs[u];
        uint64_t* kk = keys + warp * kSeedSmall;
        uint32_t* hist = reinterpret_cast<uint32_t*>(keys + (kSeedThreads / 32) * kSeedSmall) + warp * 256;
        const float* acc = accs + u * kSeedListMax;
        // dist bits of this lane's rows (positive floats order like their bits)
        constexpr int kNV = kSeedListMax / 32;
        uint32_t dv[kNV];
#pragma unroll
        for (int i = 0; i < kNV; ++i) {
            const uint32_t r = lane + 32u * i;
            dv[i] = r < n ? __float_as_uint(__fsqrt_rn(acc[r])) : 0xffffffffu;
        }
        const uint32_t T = warp_select_regs(dv, K, hist, lane);  // K-th smallest distance
        // the K best keys: every dist < T, then ties at T by ascending id (the
        // (K - #lt)-th smallest id among them, by the same select) -> exactly K <= 128
        uint32_t c_lt = 0, c_eq = 0;
#pragma unroll
        for (int i = 0; i < kNV; ++i) {
            c_lt += __popc(__ballot_sync(0xffffffffu, dv[i] < T));
            c_eq += __popc(__ballot_sync(0xffffffffu, dv[i] == T));
        }
        uint32_t tid_max = 0xffffffffu;  // ids at distance T taken: <= tid_max
        if (c_lt + c_eq > (uint32_t)kSeedSmall) {
            uint32_t iv[kNV];
#pragma unroll
            for (int i = 0; i < kNV; ++i) {
                const uint32_t r = lane + 32u * i;
                iv[i] = dv[i] == T ? (row_ids ? __ldg(row_ids + start + r) : id_base + start + r) : 0xffffffffu;
            }
            tid_max = warp_select_regs(iv, K - c_lt, hist, lane);
        }
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < kNV; ++i) {
            const uint32_t r = lane + 32u * i;
            bool take = dv[i] < T;
            uint32_t id = 0;
            if (dv[i] <= T) {
                id = row_ids ? __ldg(row_ids + start + r) : id_base + start + r;
                take = take || (dv[i] == T && id <= tid_max);
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, take);
            const uint32_t pos = c + __popc(bal & ((1u << lane) - 1u));
            if (take && pos < (uint32_t)kSeedSmall) kk[pos] = make_key(__uint_as_float(dv[i]), id);
            c += __popc(bal);
        }
        for (uint32_t r = c + lane; r < (uint32_t)kSeedSmall; r += 32) kk[r] = ~0ull;
        __syncwarp();
        warp_bitonic_sort(kk, kSeedSmall, lane);
        if (lane == 0) atomicMin(r_global + q, (uint32_t)(kk[K - 1] >> 32));
        if (out_keys) {
            for (uint32_t i = lane; i < K; i += 32) out_keys[(size_t)q * K + i] = kk[i];
            if (lane == 0) out_count[q] = K;
        }
        __syncwarp();  // kk / hist reused by this warp's next query
    }
}

__global__ void fill_u32_kernel(uint32_t* p, uint32_t v, size_t n) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = v;
}

}  // namespace

cudaError_t launch_seed_radius(const uint64_t* probes, uint32_t n_probe, const uint32_t* list_offsets,
                               const float* storage, const uint32_t* row_ids, uint32_t dim, const float* queries,
                               uint32_t nq, uint32_t K, uint32_t S, uint32_t* r_global, uint64_t* out_keys,
                               uint32_t* out_count, cudaStream_t s) {
    if (nq == 0 || K > (uint32_t)kSeedMax) return cudaSuccess;
    const size_t smem = sizeof(float) * kSeedMax * 36;
    DADE_CUDA_TRY(cudaFuncSetAttribute(seed_radius_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    seed_radius_kernel<<<nq, kSeedThreads, smem, s>>>(probes, n_probe, list_offsets, storage, row_ids, dim, queries, nq,
                                                       K, std::min<uint32_t>(S, kSeedMax), r_global, out_keys, out_count);
    return cudaGetLastError();
}

cudaError_t launch_seed_radius_lists(const uint32_t* counts, const uint32_t* bucket_off, const uint32_t* bucket_q,
                                     const uint32_t* seed_goff, const uint32_t* seed_glist, uint32_t n_lists,
                                     uint32_t max_groups,
                                     const uint32_t* list_offsets, const float* storage,
                                     const uint32_t* row_ids, uint32_t id_base, uint32_t dim, const float* queries,
                                     uint32_t K, uint32_t S, uint32_t* r_global, uint64_t* out_keys,
                                     uint32_t* out_count, cudaStream_t s) {
    if (n_lists == 0 || K > (uint32_t)kSeedSmall) return cudaErrorInvalidValue;  // caller: K <= kSeedListMaxK
    // double-buffered tile + query slices; sums [16][S], keys [8][128] and histograms alias the tile
    const size_t smem = sizeof(float) * (2 * kSeedTileF + 2 * kSeedSlice8 * kSeedGroup);
    static_assert(sizeof(float) * 2 * kSeedTileF >=
                      sizeof(float) * kSeedGroup * kSeedListMax + (sizeof(uint64_t) * kSeedSmall + sizeof(uint32_t) * 256) * (kSeedThreads / 32),
                  "seed sums + keys + histograms must fit in the tile");
    DADE_CUDA_TRY(cudaFuncSetAttribute(seed_radius_list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    seed_radius_list_kernel<<<max_groups, kSeedThreads, smem, s>>>(counts, bucket_off, bucket_q, seed_goff, seed_glist,
                                                                    n_lists,
                                                                    list_offsets,
                                                                 storage, row_ids, id_base, dim, queries, K,
                                                                 std::min<uint32_t>(S, kSeedListMax), r_global, out_keys,
                                                                 out_count, 0x8000000080000000ull);
    return cudaGetLastError();
}

cudaError_t launch_fill_u32(uint32_t* p, uint32_t v, size_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    fill_u32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, v, n);
    return cudaGetLastError();
}

// The undecided elements of a rotation launch (rotate_kernel / rotate_ksplit_kernel append them to fix),
// one warp per element over the whole GPU: at dim 960 about 1% of the outputs are undecided, and
// recomputing them inside the CTA that found them left every CTA with a ~12 us serial tail.
__global__ void __launch_bounds__(128) rotate_fix_kernel(const double* __restrict__ W, uint32_t dim,
                                                         const float* __restrict__ in, float* __restrict__ out,
                                                         const uint2* __restrict__ fix, const uint32_t* __restrict__ fix_n,
                                                         uint32_t fix_cap) {
    __shared__ double prod[4][256];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t n = min(*fix_n, fix_cap);
    for (uint32_t e = blockIdx.x * 4 + warp; e < n; e += gridDim.x * 4) {
        const uint2 rc = fix[e];
        rotate_exact_warp(W, dim, in, rc.x, rc.y, prod[warp], out + (size_t)rc.x * dim + rc.y);
    }
}

cudaError_t launch_rotate(const double* W, uint32_t dim, const float* in, uint32_t n, float* out,
                          cudaStream_t s, uint2* fix, uint32_t* fix_n, uint32_t fix_cap) {
    if (n == 0) return cudaSuccess;
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
            n_sm = 148;
    }
    if (!fix || !fix_n || !fix_cap) {
        fix = nullptr;
        fix_n = nullptr;
        fix_cap = 0;
    } else {
        DADE_CUDA_TRY(cudaMemsetAsync(fix_n, 0, 4, s));
    }
    const uint64_t tiles64 = (uint64_t)((dim + kRotT - 1) / kRotT) * ((n + kRotT - 1) / kRotT);
    if (tiles64 < 2ull * n_sm && dim >= 4 * kRotK) {  // small batch: 32 x 32 tiles, r split over the warps
        const size_t smem = 4 * (size_t)kRkWarp;
        DADE_CUDA_TRY(cudaFuncSetAttribute(rotate_ksplit_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dim3 grid((dim + kRkT - 1) / kRkT, (n + kRkT - 1) / kRkT);
        rotate_ksplit_kernel<<<grid, 128, smem, s>>>(W, dim, in, n, out, fix, fix_n, fix_cap);
    } else {
        dim3 grid((dim + kRotT - 1) / kRotT, (n + kRotT - 1) / kRotT);
        rotate_kernel<<<grid, 128, 0, s>>>(W, dim, in, n, out, fix, fix_n, fix_cap);
    }
    DADE_CUDA_TRY(cudaGetLastError());
    if (fix) rotate_fix_kernel<<<n_sm * 16, 128, 0, s>>>(W, dim, in, out, fix, fix_n, fix_cap);  // all resident
    return cudaGetLastError();
}

// Sharded index (dade_gpu_set_ivf_shard): per query, the probes whose list has
// rows on this device move to the front in probe order and the rest become
// empty (UINT64_MAX, skipped by the grouping), so rank bucket 0 -- the seed's
// list and the first streaming passes -- is the nearest LOCAL list. The probe
// set, hence every FD result, is unchanged. One warp per query, in place
// (compaction only moves entries left, after their chunk was read).
__global__ void local_probes_kernel(uint64_t* probes, uint32_t nq, uint32_t n_probe, const uint32_t* list_offsets,
                                    uint32_t n_lists) {
    const uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (q >= nq) return;
    uint64_t* p = probes + (size_t)q * n_probe;
    uint32_t n = 0;
    for (uint32_t c0 = 0; c0 < n_probe; c0 += 32) {
        const uint32_t i = c0 + lane;
        const uint64_t key = i < n_probe ? p[i] : ~0ull;
        const uint32_t list = (uint32_t)key;
        const bool keep = i < n_probe && list < n_lists && list_offsets[list + 1] > list_offsets[list];
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) p[n + __popc(bal & ((1u << lane) - 1u))] = key;
        n += __popc(bal);
        __syncwarp();
    }
    for (uint32_t i = n + lane; i < n_probe; i += 32) p[i] = ~0ull;
}

cudaError_t launch_local_probes(uint64_t* probes, uint32_t nq, uint32_t n_probe, const uint32_t* list_offsets,
                                uint32_t n_lists, cudaStream_t s) {
    if (nq == 0 || n_probe == 0) return cudaSuccess;
    local_probes_kernel<<<(unsigned)(((size_t)nq * 32 + 255) / 256), 256, 0, s>>>(probes, nq, n_probe, list_offsets,
                                                                                 n_lists);
    return cudaGetLastError();
}

cudaError_t launch_group(const GroupArgs& g, cudaStream_t s) {
    const size_t pairs = (size_t)g.nq * g.n_probe;
    const uint32_t ne = g.n_rb * g.n_lists;
    DADE_CUDA_TRY(cudaMemsetAsync(g.counts, 0, sizeof(uint32_t) * ne, s));
    DADE_CUDA_TRY(cudaMemsetAsync(g.cursor, 0, sizeof(uint32_t) * ne, s));
    const unsigned gp = (unsigned)((pairs + 255) / 256);
    const bool smem = ne <= kGroupSmemEntries;
    const unsigned gs = (unsigned)((pairs + 256 * kGroupPerThread - 1) / (256 * kGroupPerThread));
    const size_t sh = sizeof(uint32_t) * ne;
    if (smem && sh > 48 * 1024) {
        DADE_CUDA_TRY(cudaFuncSetAttribute(group_count_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
        DADE_CUDA_TRY(cudaFuncSetAttribute(group_scatter_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));
    }
    if (pairs) {
        if (smem) group_count_smem_kernel<<<gs, 256, sh, s>>>(g);
        else group_count_kernel<<<gp, 256, 0, s>>>(g);
    }
    group_scan_kernel<<<1, 1024, 0, s>>>(g);
    if (pairs) {
        if (smem) group_scatter_smem_kernel<<<gs, 256, sh, s>>>(g);
        else group_scatter_kernel<<<gp, 256, 0, s>>>(g);
    }
    if (g.max_items) group_items_kernel<<<(unsigned)((g.max_items + 255) / 256), 256, 0, s>>>(g);
    return cudaGetLastError();
}

cudaError_t launch_evaluate(const float* o, const float* q, const float* r, uint32_t n, uint32_t dim,
                            const uint32_t* cps, const double* coeff, const double* scale,
                            uint32_t n_ckpt, uint8_t* pruned, float* dist, uint8_t* exact,
                            uint32_t* dims_used, unsigned long long* counters, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    evaluate_kernel<<<(n + 127) / 128, 128, 0, s>>>(o, q, r, n, dim, cps, coeff, scale, n_ckpt, pruned,
                                                    dist, exact, dims_used, counters);
    return cudaGetLastError();
}

cudaError_t launch_partial_sums(const float* o, const float* q, uint32_t n, uint32_t dim,
                                const uint32_t* cps, uint32_t n_ckpt, float* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    partial_sums_kernel<<<(n + 127) / 128, 128, 0, s>>>(o, q, n, dim, cps, n_ckpt, out);
    return cudaGetLastError();
}

cudaError_t launch_pair_partials(const float* data, uint32_t dim, const uint32_t* pi,
                                 const uint32_t* pj, uint64_t n, const uint32_t* cps,
                                 uint32_t n_ckpt, float* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    pair_partials_kernel<<<(unsigned)((n + 127) / 128), 128, 0, s>>>(data, dim, pi, pj, n, cps, n_ckpt, out);
    return cudaGetLastError();
}

}  // namespace dade_gpu

// Index-build side of the path on the GPU, with the
// reference's arithmetic so the artifacts are the ones the reference builds:
//
//   * dataset mean + covariance  compute_covariance   proj/src/transform.cpp:58-95
//     (fp64, rows in order: bit-identical to the reference)
//   * k-means++ seeding + Lloyd  kmeans               proj/src/ivf.cpp:24-143
//     (the distance updates, sums and divisions in the reference's order and
//     rounding; the sequential prefix sum of the seeding is replaced by a
//     parallel one plus a rigorous error bound, with an exact sequential
//     fallback when the bound cannot decide the pick)
//   * exact ground truth         compute_ground_truth proj/src/dataset_io.cpp:101-135
//     (fp64 l2_sq_double, (d^2, id) order)
//
// Every fp64 operation is an explicit __d*_rn intrinsic: the reference is
// compiled without FMA contraction (x86-64 SSE2, no -march), so a fused
// multiply-add here would change low bits.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <limits>

#include "kernels.h"

namespace dade_gpu {
namespace {

constexpr double kU = 1.1102230246251565e-16;  // 2^-53, unit roundoff of fp64

// ---- dataset mean + covariance (compute_covariance) ----------------------------

// dataset_mean (transform.cpp:58-66): mean[k] = (sum over rows in order of row[k]) / n
__global__ void column_mean_kernel(const float* __restrict__ x, uint32_t n, uint32_t dim, double* mean) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= dim) return;
    double s = 0.0;
    for (uint32_t i = 0; i < n; ++i) s = __dadd_rn(s, (double)__ldg(x + (size_t)i * dim + k));
    mean[k] = __ddiv_rn(s, (double)n);
}

// cov[r][c] (r <= c) = (sum over rows in order of centered[r] * centered[c]) / n,
// centered[k] = row[k] - mean[k] in fp64 (transform.cpp:76-95). One CTA per
// 16 x 16 tile of the upper triangle; rows staged 32 at a time as centered doubles.
constexpr int kCovT = 16, kCovRows = 32;
__global__ void __launch_bounds__(kCovT * kCovT) covariance_kernel(const float* __restrict__ x, uint32_t n,
                                                                   uint32_t dim, const double* __restrict__ mean,
                                                                   double* cov) {
    // tile (br, bc) with br <= bc from the linear block index
    const uint32_t nt = (dim + kCovT - 1) / kCovT;
    uint32_t b = blockIdx.x, br = 0;
    while (b >= nt - br) {
        b -= nt - br;
        ++br;
    }
    const uint32_t bc = br + b;
    __shared__ double sr[kCovRows][kCovT + 1], sc[kCovRows][kCovT + 1];
    const uint32_t tr = threadIdx.x / kCovT, tc = threadIdx.x % kCovT;
    const uint32_t r = br * kCovT + tr, c = bc * kCovT + tc;
    double acc = 0.0;
    for (uint32_t i0 = 0; i0 < n; i0 += kCovRows) {
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < kCovRows * kCovT; e += blockDim.x) {
            const uint32_t ii = e / kCovT, kk = e % kCovT, i = i0 + ii;
            const uint32_t kr = br * kCovT + kk, kc = bc * kCovT + kk;
            sr[ii][kk] = (i < n && kr < dim) ? __dsub_rn((double)__ldg(x + (size_t)i * dim + kr), mean[kr]) : 0.0;
            sc[ii][kk] = (i < n && kc < dim) ? __dsub_rn((double)__ldg(x + (size_t)i * dim + kc), mean[kc]) : 0.0;
        }
        __syncthreads();
        const uint32_t m = min((uint32_t)kCovRows, n - i0);
        for (uint32_t ii = 0; ii < m; ++ii) acc = __dadd_rn(acc, __dmul_rn(sr[ii][tr], sc[ii][tc]));
    }
    if (r < dim && c < dim && r <= c) {
        const double v = __ddiv_rn(acc, (double)n);
        cov[(size_t)r * dim + c] = v;
        cov[(size_t)c * dim + r] = v;
    }
}

// ---- k-means++ seeding (ivf.cpp:38-68) -----------------------------------------

// l2_sq_double of rows [i0, i0 + 128) against one centroid, staged through
// shared memory in 64-dim chunks (16-byte loads, all in flight at once; each
// thread then keeps its row's sequential k order), then dist2[i] = min(dist2[i],
// d2) and the block's partial sum of the updated dist2 (any order: the pick
// bounds its rounding).
constexpr int kPpRows = 128, kPpChunk = 64, kPpPitch = kPpChunk + 1;
__global__ void __launch_bounds__(kPpRows) kmpp_update_kernel(const float* __restrict__ x, uint32_t n, uint32_t dim,
                                                              const float* __restrict__ last, double* dist2,
                                                              double* block_sums) {
    __shared__ float tile[kPpRows * kPpPitch];
    __shared__ double lastc[kPpChunk];
    __shared__ double red[kPpRows / 32];
    const uint32_t i0 = blockIdx.x * kPpRows, t = threadIdx.x, i = i0 + t;
    const bool vec = (dim & 3u) == 0;
    double acc = 0.0;
    for (uint32_t k0 = 0; k0 < dim; k0 += kPpChunk) {
        const uint32_t w = min((uint32_t)kPpChunk, dim - k0);
        __syncthreads();
        if (vec) {
            constexpr int kV = kPpRows * kPpChunk / 4 / kPpRows;  // float4 per thread
            float4 v[kV];
#pragma unroll
            for (int j = 0; j < kV; ++j) {
                const uint32_t e = t + j * kPpRows, rr = e / (kPpChunk / 4), c4 = e % (kPpChunk / 4);
                v[j] = (i0 + rr < n && 4 * c4 < w) ? __ldg(reinterpret_cast<const float4*>(x + (size_t)(i0 + rr) * dim + k0) + c4)
                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < kV; ++j) {
                const uint32_t e = t + j * kPpRows, rr = e / (kPpChunk / 4), c4 = e % (kPpChunk / 4);
                float* d = tile + rr * kPpPitch + 4 * c4;
                d[0] = v[j].x;
                d[1] = v[j].y;
                d[2] = v[j].z;
                d[3] = v[j].w;
            }
        } else {
            for (uint32_t e = t; e < kPpRows * (uint32_t)kPpChunk; e += kPpRows) {
                const uint32_t rr = e / kPpChunk, kk = e % kPpChunk;
                tile[rr * kPpPitch + kk] = (i0 + rr < n && kk < w) ? __ldg(x + (size_t)(i0 + rr) * dim + k0 + kk) : 0.f;
            }
        }
        if (t < kPpChunk) lastc[t] = t < w ? (double)__ldg(last + k0 + t) : 0.0;
        __syncthreads();
        const float* row = tile + t * kPpPitch;
        if (w == (uint32_t)kPpChunk) {
#pragma unroll 16
            for (uint32_t kk = 0; kk < (uint32_t)kPpChunk; ++kk) {
                const double d = __dsub_rn((double)row[kk], lastc[kk]);
                acc = __dadd_rn(acc, __dmul_rn(d, d));
            }
        } else {
            for (uint32_t kk = 0; kk < w; ++kk) {
                const double d = __dsub_rn((double)row[kk], lastc[kk]);
                acc = __dadd_rn(acc, __dmul_rn(d, d));
            }
        }
    }
    double v = 0.0;
    if (i < n) {
        const double old = dist2[i];
        v = acc < old ? acc : old;  // std::min(dist2[i], d2)
        dist2[i] = v;
    }
    for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, off));
    if ((t & 31) == 0) red[t >> 5] = v;
    __syncthreads();
    if (t == 0) {
        double s = 0.0;
        for (int w = 0; w < kPpRows / 32; ++w) s = __dadd_rn(s, red[w]);
        block_sums[blockIdx.x] = s;
    }
}

// rng::bounded (proj/include/dade/rng.hpp:20-25) over the host-generated
// mt19937_64 stream; *rng_pos advances by the draws used
__device__ __forceinline__ uint64_t km_bounded(const uint64_t* raw, uint32_t* rng_pos, uint32_t n_raw, uint64_t m,
                                               uint32_t* err) {
    const uint64_t limit = (0ull - m) % m;
    for (;;) {
        const uint32_t p = (*rng_pos)++;
        if (p >= n_raw) {
            *err = 1;
            return 0;
        }
        const uint64_t r = raw[p];
        if (r >= limit) return r % m;
    }
}

// The pick of centroid c (one CTA, 1024 threads). The reference sums dist2
// sequentially (run_i = fl(run_{i-1} + dist2[i])), draws target = U * total and
// picks the first i with run_i > target. Any summation order of i + 1
// nonnegative terms is within gamma_i * S_i of the exact prefix S_i, so with
// P_i our prefix |run_i - P_i| <= 2 gamma_i S_i <= M = 2.01 n u P_total (+tiny):
// i is certainly picked-or-past when P_i > hi and certainly before the pick
// when P_i <= lo. If the first index past `hi` has its predecessor <= lo the
// pick is decided; otherwise (probability ~1e-4 per pick) thread 0 redoes the
// reference's two sequential loops exactly.
constexpr int kPickStage = 4096;  // doubles staged per round of the exact fallback
__global__ void __launch_bounds__(1024) kmpp_pick_kernel(const float* __restrict__ x, uint32_t n, uint32_t dim,
                                                         const double* __restrict__ dist2,
                                                         const double* __restrict__ block_sums, uint32_t n_blocks,
                                                         const uint64_t* raw, uint32_t n_raw, uint32_t* rng_pos,
                                                         float* centroid_out, uint32_t* picks, uint32_t c,
                                                         uint32_t* err) {
    __shared__ double s_pref[1024];  // inclusive prefix of per-thread block-range sums
    __shared__ double s_stage[kPickStage];
    __shared__ uint32_t s_pick, s_mode, s_first;
    __shared__ double s_lo, s_hi, s_base, s_u;
    __shared__ uint32_t s_blk;
    const uint32_t t = threadIdx.x;
    // per-thread contiguous range of blocks
    const uint32_t per = (n_blocks + 1023) / 1024;
    const uint32_t b0 = min(n_blocks, t * per), b1 = min(n_blocks, b0 + per);
    double s = 0.0;
    for (uint32_t b = b0; b < b1; ++b) s = __dadd_rn(s, block_sums[b]);
    s_pref[t] = s;
    if (t == 0) s_first = 1024;
    __syncthreads();
    for (uint32_t off = 1; off < 1024; off <<= 1) {
        const double v = t >= off ? s_pref[t - off] : 0.0;
        __syncthreads();
        s_pref[t] = __dadd_rn(s_pref[t], v);
        __syncthreads();
    }
    if (t == 0) {
        const double T = s_pref[1023];
        s_mode = 0;
        s_pick = 0;
        if (!(T > 0.0)) {
            s_mode = 2;  // all dist2 zero: rng::bounded pick
            s_pick = (uint32_t)km_bounded(raw, rng_pos, n_raw, n, err);
        } else {
            const uint32_t p = (*rng_pos)++;
            double U = 0.0;
            if (p >= n_raw) *err = 1;
            else U = (double)(raw[p] >> 11) * 0x1.0p-53;  // rng::uniform01
            const double M = 2.01 * (double)n * kU * T + 1e-300;
            const double tmin = U * (T - M) * (1.0 - 4.0 * kU), tmax = U * (T + M) * (1.0 + 4.0 * kU);
            s_lo = tmin - M;
            s_hi = tmax + M;
            s_u = U;  // kept for the exact fallback
            s_mode = 1;
        }
    }
    __syncthreads();
    if (s_mode == 1) {
        // the first thread range whose inclusive prefix exceeds hi (parallel), its blocks and
        // then the rows of the block that crosses it (staged, scanned by thread 0)
        const double hi = s_hi;
        // (the tree prefixes need not be monotone in fp: the smallest such t; any choice is
        // verified below)
        if (s_pref[t] > hi && (t == 0 || !(s_pref[t - 1] > hi))) atomicMin(&s_first, t);
        __syncthreads();
        const uint32_t tt = s_first;
        if (tt == 1024) {
            if (t == 0) s_mode = 3;  // nothing certainly past the target: exact fallback
        } else {
            const uint32_t bb0 = min(n_blocks, tt * per), bb1 = min(n_blocks, bb0 + per);
            if (t < bb1 - bb0) s_stage[t] = block_sums[bb0 + t];
            __syncthreads();
            if (t == 0) {
                double run = tt ? s_pref[tt - 1] : 0.0;
                uint32_t b = bb0;
                for (; b < bb1; ++b) {
                    const double nr = __dadd_rn(run, s_stage[b - bb0]);
                    if (nr > hi) break;
                    run = nr;
                }
                s_blk = b;
                s_base = run;  // prefix before block b
            }
            __syncthreads();
            const uint32_t r0 = s_blk * kPpRows, r1 = min(n, r0 + kPpRows);
            if (r0 + t < r1) s_stage[t] = dist2[r0 + t];
            __syncthreads();
            if (t == 0) {
                const double lo = s_lo;
                double run = s_base, prev = run;
                uint32_t i = r0;
                for (; i < r1; ++i) {
                    prev = run;
                    run = __dadd_rn(run, s_stage[i - r0]);
                    if (run > hi) break;
                }
                if (i < r1 && prev <= lo) s_pick = i;
                else s_mode = 3;
            }
        }
        __syncthreads();
    }
    if (s_mode == 3) {
        // exact: the reference's two loops (ivf.cpp:47-61), sequentially, the values
        // staged through shared memory by the whole CTA
        double total = 0.0;
        for (uint32_t base = 0; base < n; base += kPickStage) {
            const uint32_t m = min((uint32_t)kPickStage, n - base);
            __syncthreads();
            for (uint32_t e = t; e < m; e += blockDim.x) s_stage[e] = dist2[base + e];
            __syncthreads();
            if (t == 0)
                for (uint32_t e = 0; e < m; ++e) total = __dadd_rn(total, s_stage[e]);
        }
        __shared__ double s_target;
        __shared__ uint32_t s_done;
        if (t == 0) {
            s_target = __dmul_rn(s_u, total);
            s_done = 0;
            s_pick = n - 1;
        }
        double run = 0.0;
        for (uint32_t base = 0; base < n; base += kPickStage) {
            const uint32_t m = min((uint32_t)kPickStage, n - base);
            __syncthreads();
            if (s_done) break;
            for (uint32_t e = t; e < m; e += blockDim.x) s_stage[e] = dist2[base + e];
            __syncthreads();
            if (t == 0) {
                for (uint32_t e = 0; e < m; ++e) {
                    run = __dadd_rn(run, s_stage[e]);
                    if (run > s_target) {
                        s_pick = base + e;
                        s_done = 1;
                        break;
                    }
                }
            }
        }
    }
    __syncthreads();
    const uint32_t pick = s_pick;
    for (uint32_t k = t; k < dim; k += blockDim.x) centroid_out[k] = __ldg(x + (size_t)pick * dim + k);
    if (t == 0 && picks) picks[c] = pick | (s_mode == 3 ? 0x80000000u : 0u);
}

__global__ void copy_row_kernel(const float* __restrict__ x, uint32_t dim, const uint32_t* rng_first,
                                float* centroid_out) {
    const uint32_t row = *rng_first;
    for (uint32_t k = threadIdx.x; k < dim; k += blockDim.x) centroid_out[k] = x[(size_t)row * dim + k];
}

__global__ void kmpp_first_kernel(const uint64_t* raw, uint32_t n_raw, uint32_t* rng_pos, uint32_t n,
                                  uint32_t* first, uint32_t* err) {
    if (threadIdx.x == 0) *first = (uint32_t)km_bounded(raw, rng_pos, n_raw, n, err);
}

__global__ void fill_f64_kernel(double* p, double v, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}

// ---- Lloyd iterations (ivf.cpp:73-140) ---------------------------------------

// new assignment from the coarse ranking's single probe key; changed flag
__global__ void km_assign_kernel(const uint64_t* __restrict__ probes, uint32_t n, uint32_t* assign, uint32_t* changed,
                                 uint64_t* sort_keys) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t best = (uint32_t)(probes[i] & 0xffffffffu);
    if (assign[i] != best) {
        assign[i] = best;
        *changed = 1;
    }
    if (sort_keys) sort_keys[i] = ((uint64_t)best << 32) | i;
}

__global__ void km_keys_kernel(const uint32_t* __restrict__ assign, uint32_t n, uint64_t* keys) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = ((uint64_t)assign[i] << 32) | i;
}

// counts and offsets of the (cluster, id)-sorted keys: offsets[c] = first key of cluster >= c
__global__ void km_offsets_kernel(const uint64_t* __restrict__ sorted, uint32_t n, uint32_t n_clusters,
                                  uint32_t* offsets) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i > n) return;
    const uint32_t cur = i < n ? (uint32_t)(sorted[i] >> 32) : n_clusters;
    const uint32_t prev = i > 0 ? (uint32_t)(sorted[i - 1] >> 32) : 0xffffffffu;
    // clusters (prev, cur] start at i
    const uint32_t c0 = i > 0 ? prev + 1 : 0;
    for (uint32_t c = c0; c <= cur && c <= n_clusters; ++c) offsets[c] = i;
}

// centroid update (ivf.cpp:96-109): thread per (cluster, dim), members in
// ascending id order: s += v[k] in fp64, cen = (float)(s / count); empty keep
__global__ void km_sums_kernel(const float* __restrict__ x, uint32_t dim, const uint64_t* __restrict__ sorted,
                               const uint32_t* __restrict__ offsets, uint32_t n_clusters, float* centroids) {
    const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (e >= (size_t)n_clusters * dim) return;
    const uint32_t c = (uint32_t)(e / dim), k = (uint32_t)(e % dim);
    const uint32_t b = offsets[c], en = offsets[c + 1];
    if (b == en) return;
    double s = 0.0;
    for (uint32_t m = b; m < en; ++m) {
        const uint32_t i = (uint32_t)(sorted[m] & 0xffffffffu);
        s = __dadd_rn(s, (double)__ldg(x + (size_t)i * dim + k));
    }
    centroids[(size_t)c * dim + k] = __double2float_rn(__ddiv_rn(s, (double)(en - b)));
}

// farthest member of one cluster (re-seeding an empty one, ivf.cpp:111-130):
// max l2_sq_double to its centroid, lowest id on ties
__global__ void km_far_max_kernel(const float* __restrict__ x, uint32_t n, uint32_t dim,
                                  const uint32_t* __restrict__ assign, uint32_t cluster,
                                  const float* __restrict__ cen, unsigned long long* best) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || assign[i] != cluster) return;
    double acc = 0.0;
    for (uint32_t k = 0; k < dim; ++k) {
        const double d = __dsub_rn((double)__ldg(x + (size_t)i * dim + k), (double)__ldg(cen + k));
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    atomicMax(best, (unsigned long long)__double_as_longlong(acc));  // nonnegative doubles order as bits
    // second word: lowest id at the maximum, resolved by km_far_id_kernel
}
__global__ void km_far_id_kernel(const float* __restrict__ x, uint32_t n, uint32_t dim,
                                 const uint32_t* __restrict__ assign, uint32_t cluster, const float* __restrict__ cen,
                                 const unsigned long long* best, uint32_t* far_id) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || assign[i] != cluster) return;
    double acc = 0.0;
    for (uint32_t k = 0; k < dim; ++k) {
        const double d = __dsub_rn((double)__ldg(x + (size_t)i * dim + k), (double)__ldg(cen + k));
        acc = __dadd_rn(acc, __dmul_rn(d, d));
    }
    if ((unsigned long long)__double_as_longlong(acc) == *best) atomicMin(far_id, i);
}
__global__ void km_reseed_kernel(const float* __restrict__ x, uint32_t dim, const uint32_t* far_id, uint32_t c,
                                 float* centroids, uint32_t* assign) {
    const uint32_t f = *far_id;
    for (uint32_t k = threadIdx.x; k < dim; k += blockDim.x) centroids[(size_t)c * dim + k] = x[(size_t)f * dim + k];
    if (threadIdx.x == 0) assign[f] = c;
}

__global__ void gather_rows_kernel(const float* __restrict__ x, uint32_t dim, const uint64_t* __restrict__ sorted,
                                   uint32_t n, float* rows_out, uint32_t* ids_out) {
    const size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (e >= (size_t)n * dim) return;
    const uint32_t m = (uint32_t)(e / dim), k = (uint32_t)(e % dim);
    const uint32_t i = (uint32_t)(sorted[m] & 0xffffffffu);
    rows_out[e] = __ldg(x + (size_t)i * dim + k);
    if (k == 0) ids_out[m] = i;
}

// ---- exact ground truth (compute_ground_truth) ----------------------------------

// fp64 l2_sq_double for a 64-query x 128-row tile per CTA step (256 threads, each
// 4 queries x 8 rows in registers, k ascending per pair); a pair is emitted as a
// candidate when d2 <= thr[q]. Mode 0: candidates into per-query slots.
constexpr int kGtQ = 64, kGtR = 128, kGtK = 16;
__global__ void __launch_bounds__(256) gt_scan_kernel(const float* __restrict__ base, uint32_t n, uint32_t row_stride,
                                                      const float* __restrict__ queries, uint32_t nq, uint32_t dim,
                                                      const double* __restrict__ thr, uint32_t cap, uint32_t* cnt,
                                                      double* cand_d, uint32_t* cand_id) {
    __shared__ double sq[kGtK][kGtQ + 1];
    __shared__ double sb[kGtK][kGtR + 1];
    const uint32_t q0 = blockIdx.y * kGtQ;
    const uint32_t n_rows = (n + row_stride - 1) / row_stride;  // rows 0, s, 2s, ... (sampling)
    const uint32_t tq = threadIdx.x / 16, tr = threadIdx.x % 16;  // 16 x 16 threads: 4 queries x 8 rows each
    double th[4];
#pragma unroll
    for (int a = 0; a < 4; ++a) {
        const uint32_t q = q0 + tq * 4 + a;
        th[a] = q < nq ? thr[q] : -1.0;
    }
    for (uint32_t r0 = blockIdx.x * kGtR; r0 < n_rows; r0 += gridDim.x * kGtR) {
        double acc[4][8];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
        for (uint32_t k0 = 0; k0 < dim; k0 += kGtK) {
            __syncthreads();
            for (uint32_t e = threadIdx.x; e < kGtK * kGtQ; e += 256) {
                const uint32_t qq = e / kGtK, kk = e % kGtK, q = q0 + qq, k = k0 + kk;
                sq[kk][qq] = (q < nq && k < dim) ? (double)__ldg(queries + (size_t)q * dim + k) : 0.0;
            }
            for (uint32_t e = threadIdx.x; e < kGtK * kGtR; e += 256) {
                const uint32_t rr = e / kGtK, kk = e % kGtK, r = r0 + rr, k = k0 + kk;
                sb[kk][rr] = (r < n_rows && k < dim) ? (double)__ldg(base + (size_t)r * row_stride * dim + k) : 0.0;
            }
            __syncthreads();
            const uint32_t kw = min((uint32_t)kGtK, dim - k0);
            for (uint32_t kk = 0; kk < kw; ++kk) {
                double qv[4], bv[8];
#pragma unroll
                for (int a = 0; a < 4; ++a) qv[a] = sq[kk][tq * 4 + a];
#pragma unroll
                for (int b = 0; b < 8; ++b) bv[b] = sb[kk][tr + 16 * b];
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int b = 0; b < 8; ++b) {
                        // l2_sq_double: d = (double)a[k] - (double)b[k]; acc += d * d
                        const double d = __dsub_rn(bv[b], qv[a]);
                        acc[a][b] = __dadd_rn(acc[a][b], __dmul_rn(d, d));
                    }
            }
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
            const uint32_t q = q0 + tq * 4 + a;
            if (q >= nq) continue;
#pragma unroll
            for (int b = 0; b < 8; ++b) {
                const uint32_t r = r0 + tr + 16 * b;
                if (r < n_rows && acc[a][b] <= th[a]) {
                    const uint32_t p = atomicAdd(cnt + q, 1u);
                    if (p < cap) {
                        cand_d[(size_t)q * cap + p] = acc[a][b];
                        cand_id[(size_t)q * cap + p] = r * row_stride;
                    }
                }
            }
        }
    }
}

// per query: sort its candidates by (d2, id) and keep the first k (or, in
// threshold mode, the k-th smallest d2 as the next threshold). One CTA per
// query, bitonic sort over the next power of two of min(cnt, cap) in shared memory.
__global__ void __launch_bounds__(512) gt_select_kernel(const uint32_t* __restrict__ cnt, uint32_t cap,
                                                        const double* __restrict__ cand_d,
                                                        const uint32_t* __restrict__ cand_id, uint32_t k,
                                                        uint32_t* out_ids, double* out_kth, uint32_t* overflow) {
    extern __shared__ unsigned char gs_raw[];
    const uint32_t q = blockIdx.x;
    const uint32_t c = cnt[q];
    const uint32_t m = min(c, cap);
    uint32_t p2 = 1;
    while (p2 < m) p2 <<= 1;
    double* sd = reinterpret_cast<double*>(gs_raw);
    uint32_t* si = reinterpret_cast<uint32_t*>(sd + p2);
    for (uint32_t e = threadIdx.x; e < p2; e += blockDim.x) {
        sd[e] = e < m ? cand_d[(size_t)q * cap + e] : __longlong_as_double(0x7ff0000000000000ll);
        si[e] = e < m ? cand_id[(size_t)q * cap + e] : 0xffffffffu;
    }
    __syncthreads();
    for (uint32_t len = 2; len <= p2; len <<= 1)
        for (uint32_t j = len >> 1; j > 0; j >>= 1) {
            for (uint32_t e = threadIdx.x; e < p2; e += blockDim.x) {
                const uint32_t o = e ^ j;
                if (o > e) {
                    const bool up = (e & len) == 0;
                    const bool gt = sd[e] > sd[o] || (sd[e] == sd[o] && si[e] > si[o]);
                    if (gt == up) {
                        const double td = sd[e];
                        sd[e] = sd[o];
                        sd[o] = td;
                        const uint32_t ti = si[e];
                        si[e] = si[o];
                        si[o] = ti;
                    }
                }
            }
            __syncthreads();
        }
    if (out_ids)
        for (uint32_t e = threadIdx.x; e < k; e += blockDim.x) out_ids[(size_t)q * k + e] = e < m ? si[e] : 0xffffffffu;
    if (threadIdx.x == 0) {
        if (out_kth) out_kth[q] = m >= k ? sd[k - 1] : __longlong_as_double(0x7ff0000000000000ll);
        if (overflow && c > cap) atomicAdd(overflow, 1u);
    }
}

}  // namespace

cudaError_t launch_covariance(const float* x, uint32_t n, uint32_t dim, double* mean, double* cov, cudaStream_t s) {
    if (n == 0 || dim == 0) return cudaSuccess;
    column_mean_kernel<<<(dim + 127) / 128, 128, 0, s>>>(x, n, dim, mean);
    const uint32_t nt = (dim + kCovT - 1) / kCovT;
    covariance_kernel<<<nt * (nt + 1) / 2, kCovT * kCovT, 0, s>>>(x, n, dim, mean, cov);
    return cudaGetLastError();
}

size_t kmpp_block_count(uint32_t n) { return (n + kPpRows - 1) / kPpRows; }

cudaError_t launch_kmpp_seed(const float* x, uint32_t n, uint32_t dim, uint32_t n_clusters, const uint64_t* raw,
                             uint32_t n_raw, uint32_t* rng_state, double* dist2, double* block_sums,
                             float* centroids, uint32_t* picks, cudaStream_t s) {
    // rng_state: [0] position in raw, [1] error flag, [2] first pick
    const uint32_t nb = (uint32_t)kmpp_block_count(n);
    kmpp_first_kernel<<<1, 32, 0, s>>>(raw, n_raw, rng_state, n, rng_state + 2, rng_state + 1);
    copy_row_kernel<<<1, 256, 0, s>>>(x, dim, rng_state + 2, centroids);
    fill_f64_kernel<<<256, 256, 0, s>>>(dist2, std::numeric_limits<double>::infinity(), n);
    for (uint32_t c = 1; c < n_clusters; ++c) {
        kmpp_update_kernel<<<nb, kPpRows, 0, s>>>(x, n, dim, centroids + (size_t)(c - 1) * dim, dist2, block_sums);
        kmpp_pick_kernel<<<1, 1024, 0, s>>>(x, n, dim, dist2, block_sums, nb, raw, n_raw, rng_state,
                                            centroids + (size_t)c * dim, picks, c, rng_state + 1);
    }
    return cudaGetLastError();
}

cudaError_t launch_km_assign(const uint64_t* probes, uint32_t n, uint32_t* assign, uint32_t* changed,
                             cudaStream_t s) {
    km_assign_kernel<<<(n + 255) / 256, 256, 0, s>>>(probes, n, assign, changed, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_km_sort(const uint32_t* assign, uint32_t n, uint32_t n_clusters, uint64_t* keys_in,
                           uint64_t* keys_out, uint32_t* offsets, void* temp, size_t* temp_bytes, cudaStream_t s) {
    int end_bit = 32;
    while ((1ull << (end_bit - 32)) < (uint64_t)n_clusters + 1) ++end_bit;
    if (!temp) {
        return cub::DeviceRadixSort::SortKeys(nullptr, *temp_bytes, keys_in, keys_out, (int)n, 0, end_bit, s);
    }
    km_keys_kernel<<<(n + 255) / 256, 256, 0, s>>>(assign, n, keys_in);
    cudaError_t e = cub::DeviceRadixSort::SortKeys(temp, *temp_bytes, keys_in, keys_out, (int)n, 0, end_bit, s);
    if (e != cudaSuccess) return e;
    km_offsets_kernel<<<(n + 1 + 255) / 256, 256, 0, s>>>(keys_out, n, n_clusters, offsets);
    return cudaGetLastError();
}

cudaError_t launch_km_sums(const float* x, uint32_t dim, const uint64_t* sorted, const uint32_t* offsets,
                           uint32_t n_clusters, float* centroids, cudaStream_t s) {
    const size_t tot = (size_t)n_clusters * dim;
    km_sums_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(x, dim, sorted, offsets, n_clusters, centroids);
    return cudaGetLastError();
}

cudaError_t launch_km_reseed(const float* x, uint32_t n, uint32_t dim, uint32_t* assign, uint32_t largest,
                             uint32_t empty_c, float* centroids, unsigned long long* scratch, cudaStream_t s) {
    // scratch: [0] max d2 bits, [1] low word = far id
    cudaError_t e = cudaMemsetAsync(scratch, 0, 8, s);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(scratch + 1, 0xff, 8, s);
    if (e != cudaSuccess) return e;
    const float* cen = centroids + (size_t)largest * dim;
    km_far_max_kernel<<<(n + 255) / 256, 256, 0, s>>>(x, n, dim, assign, largest, cen, scratch);
    uint32_t* far_id = reinterpret_cast<uint32_t*>(scratch + 1);
    km_far_id_kernel<<<(n + 255) / 256, 256, 0, s>>>(x, n, dim, assign, largest, cen, scratch, far_id);
    km_reseed_kernel<<<1, 256, 0, s>>>(x, dim, far_id, empty_c, centroids, assign);
    return cudaGetLastError();
}

cudaError_t launch_gather_rows(const float* x, uint32_t dim, const uint64_t* sorted, uint32_t n, float* rows_out,
                               uint32_t* ids_out, cudaStream_t s) {
    const size_t tot = (size_t)n * dim;
    if (!tot) return cudaSuccess;
    gather_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(x, dim, sorted, n, rows_out, ids_out);
    return cudaGetLastError();
}

cudaError_t launch_gt_scan(const float* base, uint32_t n, uint32_t row_stride, const float* queries, uint32_t nq,
                           uint32_t dim, const double* thr, uint32_t cap, uint32_t* cnt, double* cand_d,
                           uint32_t* cand_id, int n_sms, cudaStream_t s) {
    if (!nq || !n) return cudaSuccess;
    const uint32_t qb = (nq + kGtQ - 1) / kGtQ;
    const uint32_t n_rows = (n + row_stride - 1) / row_stride;
    const uint32_t rb = (n_rows + kGtR - 1) / kGtR;
    const uint32_t gx = std::max<uint32_t>(1, std::min<uint32_t>(rb, (uint32_t)(n_sms * 8 + qb - 1) / qb));
    gt_scan_kernel<<<dim3(gx, qb), 256, 0, s>>>(base, n, row_stride, queries, nq, dim, thr, cap, cnt, cand_d,
                                                cand_id);
    return cudaGetLastError();
}

cudaError_t launch_gt_select(const uint32_t* cnt, uint32_t cap, const double* cand_d, const uint32_t* cand_id,
                             uint32_t nq, uint32_t k, uint32_t* out_ids, double* out_kth, uint32_t* overflow,
                             cudaStream_t s) {
    if (!nq) return cudaSuccess;
    uint32_t p2 = 1;
    while (p2 < cap) p2 <<= 1;
    const size_t smem = (size_t)p2 * 12;
    cudaError_t e = cudaFuncSetAttribute(gt_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    gt_select_kernel<<<nq, 512, smem, s>>>(cnt, cap, cand_d, cand_id, k, out_ids, out_kth, overflow);
    return cudaGetLastError();
}

}  // namespace dade_gpu

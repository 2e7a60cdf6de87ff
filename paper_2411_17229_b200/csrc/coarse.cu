// Coarse ranking (K2, proj/src/ivf.cpp:215-219) on tensor cores with an exact
// boundary: the n_probe nearest centroids by exact fp32 l2_sq, ties by id.
//
//   1. coarse_tc_kernel: p~(q, c) = |q|^2 + |c|^2 - 2 q.c over all D dims with
//      mma.sync TF32 (fp32 bits read as TF32); writes p~; the select kernel
//      forms lo = p~ - delta and hi = p~ + delta, delta = kCoarseDelta
//      (|q|^2 + |c|^2) bounding |p~ - acc|
//      for the reference's exact sequential fp32 l2_sq `acc` (same derivation
//      as the scan filter, with D-term accumulation < 1e-4).
//   2. coarse_select_kernel (warp per query): B = n_probe-th smallest hi (radix
//      select on float bits) bounds the n_probe-th smallest exact acc, so every
//      exact top-n_probe centroid has lo <= B; those candidates get the exact
//      sequential l2_sq and are sorted by (acc, id); the first n_probe are the
//      probes, bit-identical to the reference ranking.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

constexpr int kCQ = 64;     // queries per CTA tile
constexpr int kCC = 128;    // centroids per CTA tile
constexpr int kCK = 32;     // dims per staged slice
constexpr int kCS = kCK + 4;  // padded smem row (floats)

__device__ __forceinline__ void mma_tf32_c(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// CTA: 128 centroids (M) x 64 queries (N); 8 warps = 4 (M: 32 rows each) x 2 (N: 32 cols each).
__global__ void __launch_bounds__(256) coarse_tc_kernel(const float* __restrict__ cen, uint32_t n_cen,
                                                        const float* __restrict__ q, uint32_t nq, uint32_t dim,
                                                        const float* __restrict__ cnorm, const float* __restrict__ qnorm,
                                                        float* __restrict__ p_out) {
    __shared__ __align__(16) float cs[kCC * kCS];
    __shared__ __align__(16) float qs[kCQ * kCS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int g = lane >> 2, tq = lane & 3;
    const int wm = warp & 3, wn = warp >> 2;
    const uint32_t c0 = blockIdx.x * kCC, q0 = blockIdx.y * kCQ;
    float d[2][4][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
            for (int v = 0; v < 4; ++v) d[a][b][v] = 0.f;
    const bool vec = (dim & 3u) == 0;
    for (uint32_t k0 = 0; k0 < dim; k0 += kCK) {
        const uint32_t w = min((uint32_t)kCK, dim - k0);
        __syncthreads();
        for (uint32_t idx = tid; idx < (uint32_t)kCC * (kCK / 4); idx += 256) {
            const uint32_t r = idx >> 3, c4 = idx & 7;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c0 + r < n_cen) {
                const float* src = cen + (size_t)(c0 + r) * dim + k0 + 4 * c4;
                if (vec && 4 * c4 + 4 <= w) v = __ldg(reinterpret_cast<const float4*>(src));
                else {
                    float t[4] = {0.f, 0.f, 0.f, 0.f};
                    for (int e = 0; e < 4; ++e) if (4 * c4 + e < w) t[e] = __ldg(src + e);
                    v = make_float4(t[0], t[1], t[2], t[3]);
                }
            }
            *reinterpret_cast<float4*>(cs + r * kCS + 4 * c4) = v;
        }
        for (uint32_t idx = tid; idx < (uint32_t)kCQ * (kCK / 4); idx += 256) {
            const uint32_t r = idx >> 3, c4 = idx & 7;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (q0 + r < nq) {
                const float* src = q + (size_t)(q0 + r) * dim + k0 + 4 * c4;
                if (vec && 4 * c4 + 4 <= w) v = __ldg(reinterpret_cast<const float4*>(src));
                else {
                    float t[4] = {0.f, 0.f, 0.f, 0.f};
                    for (int e = 0; e < 4; ++e) if (4 * c4 + e < w) t[e] = __ldg(src + e);
                    v = make_float4(t[0], t[1], t[2], t[3]);
                }
            }
            *reinterpret_cast<float4*>(qs + r * kCS + 4 * c4) = v;
        }
        __syncthreads();
#pragma unroll
        for (int ks = 0; ks < kCK; ks += 8) {
            uint32_t A[2][4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt) {
                const float* r0 = cs + (wm * 32 + mt * 16 + g) * kCS + ks + tq;
                A[mt][0] = __float_as_uint(r0[0]);
                A[mt][1] = __float_as_uint(r0[8 * kCS]);
                A[mt][2] = __float_as_uint(r0[4]);
                A[mt][3] = __float_as_uint(r0[8 * kCS + 4]);
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
                const float* qb = qs + (wn * 32 + nt * 8 + g) * kCS + ks + tq;
                const uint32_t b0 = __float_as_uint(qb[0]), b1 = __float_as_uint(qb[4]);
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) mma_tf32_c(d[mt][nt], A[mt][0], A[mt][1], A[mt][2], A[mt][3], b0, b1);
            }
        }
    }
    // epilogue: row = centroid, col = query
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t c = c0 + wm * 32 + mt * 16 + h * 8 + g;
            if (c >= n_cen) continue;
            const float cn = cnorm[c];
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int cq = 0; cq < 2; ++cq) {
                    const uint32_t qq = q0 + wn * 32 + nt * 8 + 2 * tq + cq;
                    if (qq >= nq) continue;
                    const float s = cn + qnorm[qq];
                    p_out[(size_t)qq * n_cen + c] = fmaf(-2.f, d[mt][nt][h * 2 + cq], s);
                }
        }
}

// |row|^2 of the centroids then the queries, warp per row (only bounds use them)
__global__ void __launch_bounds__(256) sq_norms_kernel(const float* __restrict__ a, uint32_t na,
                                                       const float* __restrict__ b, uint32_t nb, uint32_t dim,
                                                       float* __restrict__ out_a, float* __restrict__ out_b) {
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    if (w >= na + nb) return;
    const float* r = w < na ? a + (size_t)w * dim : b + (size_t)(w - na) * dim;
    float acc = 0.f;
    for (uint32_t k = lane; k < dim; k += 32) acc = fmaf(r[k], r[k], acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) {
        if (w < na) out_a[w] = acc;
        else out_b[w - na] = acc;
    }
}


constexpr int kSelCap = 512;  // exact-candidate list per query

// Warp per query (4 warps per CTA).
__global__ void __launch_bounds__(128) coarse_select_kernel(const float* __restrict__ pt,
                                                            const float* __restrict__ cnorm,
                                                            const float* __restrict__ qnorm,
                                                            const float* __restrict__ cen, uint32_t n_cen,
                                                            const float* __restrict__ q, uint32_t nq, uint32_t dim,
                                                            uint32_t n_probe, uint64_t* __restrict__ probes,
                                                            uint32_t* __restrict__ overflow) {
    __shared__ uint32_t hist[4][256];
    __shared__ uint64_t cand[4][kSelCap];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qi = blockIdx.x * 4 + warp;
    if (qi >= nq) return;
    const float* prow = pt + (size_t)qi * n_cen;
    const float qn = qnorm[qi];
    // bounds of the exact l2_sq: p~ -/+ kCoarseDelta (|q|^2 + |c|^2)
    auto hi_of = [&](uint32_t c) { return __fadd_rn(prow[c], coarse_delta(cnorm[c], qn)); };
    auto lo_of = [&](uint32_t c) { return __fsub_rn(prow[c], coarse_delta(cnorm[c], qn)); };
    uint32_t* h = hist[warp];
    // radix select: key of the n_probe-th smallest hi (4 passes of 8 bits)
    uint32_t prefix = 0, rank = n_probe;  // rank: 1-based within the current prefix class
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int b = lane; b < 256; b += 32) h[b] = 0;
        __syncwarp();
        const uint32_t mask_hi = pass == 0 ? 0u : (0xffffffffu << (32 - 8 * pass));
        for (uint32_t c = lane; c < n_cen; c += 32) {
            const uint32_t k = fkey(hi_of(c));
            if ((k & mask_hi) == prefix) atomicAdd(&h[(k >> shift) & 0xffu], 1u);
        }
        __syncwarp();
        uint32_t digit, before;
        warp_hist_find(h, rank, lane, digit, before);
        prefix |= digit << shift;
        rank -= before;
        __syncwarp();
    }
    // prefix = fkey(B); candidates: lo <= B
    uint32_t n = 0;
    for (uint32_t c0 = 0; c0 < n_cen; c0 += 32) {
        const uint32_t c = c0 + lane;
        const bool is = c < n_cen && fkey(lo_of(c)) <= prefix;
        const uint32_t bal = __ballot_sync(0xffffffffu, is);
        const uint32_t pos = n + __popc(bal & ((1u << lane) - 1u));
        if (is && pos < (uint32_t)kSelCap) cand[warp][pos] = c;
        n += __popc(bal);
    }
    if (n > (uint32_t)kSelCap) {  // pathological ties: exact ranking of everything is the fallback
        if (lane == 0) atomicAdd(overflow, 1u);
        n = min(n, (uint32_t)kSelCap);
    }
    __syncwarp();
    // exact sequential l2_sq (proj/include/dade/distance.hpp:36-43) per candidate, key (acc, id)
    const float* qr = q + (size_t)qi * dim;
    for (uint32_t e = lane; e < n; e += 32) {
        const uint32_t c = (uint32_t)cand[warp][e];
        const float* cr = cen + (size_t)c * dim;
        float acc = 0.f;
        if ((dim & 3u) == 0) {
            uint32_t k = 0;
            for (; k + 32 <= dim; k += 32) {  // 8 float4 pairs in flight per round trip
                float4 a8[8], b8[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    a8[u] = __ldg(reinterpret_cast<const float4*>(qr + k) + u);
                    b8[u] = __ldg(reinterpret_cast<const float4*>(cr + k) + u);
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc = sq_step(acc, a8[u].x, b8[u].x);
                    acc = sq_step(acc, a8[u].y, b8[u].y);
                    acc = sq_step(acc, a8[u].z, b8[u].z);
                    acc = sq_step(acc, a8[u].w, b8[u].w);
                }
            }
            for (; k < dim; k += 4) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(qr + k));
                const float4 b = __ldg(reinterpret_cast<const float4*>(cr + k));
                acc = sq_step(acc, a.x, b.x);
                acc = sq_step(acc, a.y, b.y);
                acc = sq_step(acc, a.z, b.z);
                acc = sq_step(acc, a.w, b.w);
            }
        } else {
            for (uint32_t k = 0; k < dim; ++k) acc = sq_step(acc, __ldg(qr + k), __ldg(cr + k));
        }
        cand[warp][e] = make_key(acc, c);
    }
    // pad and bitonic-sort the candidate keys
    uint32_t m = 1;
    while (m < n) m <<= 1;
    for (uint32_t e = n + lane; e < m; e += 32) cand[warp][e] = ~0ull;
    __syncwarp();
    uint64_t* kk = cand[warp];
    for (uint32_t size = 2; size <= m; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = lane; i < m / 2; i += 32) {
                const uint32_t lo_i = 2 * i - (i & (stride - 1)), hi_i = lo_i + stride;
                const bool up = (lo_i & size) == 0;
                const uint64_t x = kk[lo_i], y = kk[hi_i];
                if ((x > y) == up) { kk[lo_i] = y; kk[hi_i] = x; }
            }
            __syncwarp();
        }
    for (uint32_t i = lane; i < n_probe; i += 32) probes[(size_t)qi * n_probe + i] = kk[i];
}

// Fast path (n_cen <= 1024, dim % 4 == 0), warp per query:
//   * the query's p~ row and the bounds live in registers (32 per lane);
//   * B = n_probe-th smallest upper bound by 8-bit radix select;
//   * candidates (lower bound <= B) compacted by ballots;
//   * exact l2_sq of 32 candidates at a time: their rows staged 32 dims at a time
//     through shared memory with coalesced 16-byte loads (8 lanes per 128-byte
//     row chunk), each lane then advancing its candidate's sequential fp32 sum;
//   * (acc, id) bitonic sort of the candidates, first n_probe -> probes.
constexpr int kFsWarps = 4;
// candidates per query of coarse_select_fast_kernel: 384 keeps a CTA under 32 KB of shared memory, so seven
// CTAs fit an SM and a 1000-query batch (one CTA per query) is ONE wave of 1036 slots instead of a full wave of
// 888 and a tail of 112 (config 2: the kernel took two per-query latencies)
constexpr int kFsCap = 384;
__device__ __forceinline__ void cs_cp16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}
constexpr int kFsRS = 36;  // floats per staged row chunk (16-byte aligned, conflict-free LDS.128)

// One round of exact sequential l2_sq (proj/include/dade/distance.hpp:36-43):
// lane i advances candidate my_c of lane i (active lanes; nv = lanes holding a
// candidate). Rows are staged 32 dims at a time through shared memory rs / qs
// with coalesced 16-byte loads (8 lanes per 128-byte row chunk); the next
// chunk's loads are issued before the current chunk is summed, so the L2
// latency overlaps the arithmetic, and a full 32-dim chunk is summed unrolled.
__device__ __forceinline__ float exact_l2_round(const float* __restrict__ cen, const float* __restrict__ qr,
                                                uint32_t dim, uint32_t my_c, uint32_t nv, bool active, float* rs,
                                                float* qs, int lane) {
    const uint32_t sub = lane >> 3, c4 = lane & 7;
    uint32_t cc[8];
#pragma unroll
    for (int sg = 0; sg < 8; ++sg) cc[sg] = __shfl_sync(0xffffffffu, my_c, 4 * sg + sub);
    float4 v[8], qv;
    auto load = [&](uint32_t k0) {
        const uint32_t w = min(32u, dim - k0);
#pragma unroll
        for (int sg = 0; sg < 8; ++sg)
            v[sg] = (4 * sg + sub < nv && 4 * c4 < w)
                        ? __ldg(reinterpret_cast<const float4*>(cen + (size_t)cc[sg] * dim + k0) + c4)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
        qv = (lane < 8 && 4u * lane < w) ? __ldg(reinterpret_cast<const float4*>(qr + k0) + lane)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    load(0);
    float acc = 0.f;
    const float* os = rs + lane * kFsRS;
    for (uint32_t k0 = 0; k0 < dim; k0 += 32) {
        const uint32_t w = min(32u, dim - k0);
        __syncwarp();  // previous chunk's readers done
#pragma unroll
        for (int sg = 0; sg < 8; ++sg) *reinterpret_cast<float4*>(rs + (4 * sg + sub) * kFsRS + 4 * c4) = v[sg];
        if (lane < 8) *reinterpret_cast<float4*>(qs + 4 * lane) = qv;
        __syncwarp();
        if (k0 + 32 < dim) load(k0 + 32);
        if (!active) continue;
        if (w == 32) {
#pragma unroll
            for (uint32_t kk = 0; kk < 32; kk += 4) {
                const float4 o4 = *reinterpret_cast<const float4*>(os + kk);
                const float4 q4 = *reinterpret_cast<const float4*>(qs + kk);
                acc = sq_step(acc, q4.x, o4.x);
                acc = sq_step(acc, q4.y, o4.y);
                acc = sq_step(acc, q4.z, o4.z);
                acc = sq_step(acc, q4.w, o4.w);
            }
        } else {
            for (uint32_t kk = 0; kk < w; kk += 4) {
                const float4 o4 = *reinterpret_cast<const float4*>(os + kk);
                const float4 q4 = *reinterpret_cast<const float4*>(qs + kk);
                acc = sq_step(acc, q4.x, o4.x);
                acc = sq_step(acc, q4.y, o4.y);
                acc = sq_step(acc, q4.z, o4.z);
                acc = sq_step(acc, q4.w, o4.w);
            }
        }
    }
    return acc;
}

// WPQ = 4 (small batches, where a warp per query leaves the GPU idle): the four
// warps of a CTA select the same candidates redundantly (no synchronisation),
// warp w runs the exact rounds w, w + 4, ... and writes its keys into warp 0's
// list, which warp 0 sorts after the CTA barrier.
template <int WPQ>
__global__ void __launch_bounds__(kFsWarps * 32, WPQ == 1 ? 6 : 7) coarse_select_fast_kernel(
    const float* __restrict__ pt, const float* __restrict__ cnorm, const float* __restrict__ qnorm,
    const float* __restrict__ cen, uint32_t n_cen, const float* __restrict__ q, uint32_t nq, uint32_t dim,
    uint32_t n_probe, uint64_t* __restrict__ probes, uint32_t* __restrict__ overflow, uint32_t* census = nullptr,
    bool exact_all = true) {
    __shared__ uint64_t cand[kFsWarps][kFsCap];
    __shared__ __align__(16) float rows[kFsWarps][32 * kFsRS];
    __shared__ __align__(16) float qch[kFsWarps][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qi = WPQ == 1 ? blockIdx.x * kFsWarps + warp : blockIdx.x;
    if (qi >= nq) return;  // uniform per CTA when WPQ > 1
    const float* prow = pt + (size_t)qi * n_cen;
    const float qn = qnorm[qi];
    uint32_t hk[32], lk[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t c = lane + 32u * j;
        if (c < n_cen) {
            const float p = prow[c], d = coarse_delta(cnorm[c], qn);
            hk[j] = fkey(__fadd_rn(p, d));
            lk[j] = fkey(__fsub_rn(p, d));
        } else {
            hk[j] = 0xffffffffu;
            lk[j] = 0xffffffffu;
        }
    }
    // B = the n_probe-th smallest hk: 8-bit radix digits (shared histogram),
    // starting below the bits every present key shares (min ^ max)
    uint32_t kmin = 0xffffffffu, kmax = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        kmin = min(kmin, hk[j]);
        if (lane + 32u * j < n_cen) kmax = max(kmax, hk[j]);
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    uint32_t pre = kmin;
    if (kmax > kmin) {
        uint32_t* hist = reinterpret_cast<uint32_t*>(rows[warp]);  // free until the exact stage
        const int top = (31 - __clz(kmin ^ kmax)) & ~7;
        uint32_t mask = top >= 24 ? 0u : ~0u << (top + 8), rem = n_probe;
        pre = kmin & mask;
        for (int shift = top; shift >= 0; shift -= 8) {
            for (uint32_t j = lane; j < 256; j += 32) hist[j] = 0;
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if ((hk[j] & mask) == pre) atomicAdd(&hist[(hk[j] >> shift) & 0xffu], 1u);
            __syncwarp();
            uint32_t d, before;
            warp_hist_find(hist, rem, lane, d, before);
            rem -= before;
            pre |= d << shift;
            mask |= 0xffu << shift;
            __syncwarp();
        }
    }
    const uint32_t B = pre;  // exactly the n_probe-th smallest key
    // candidates: every centroid whose lower bound is <= B
    uint32_t n = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const bool is = lk[j] <= B && (lane + 32u * j) < n_cen;
        const uint32_t bal = __ballot_sync(0xffffffffu, is);
        const uint32_t pos = n + __popc(bal & ((1u << lane) - 1u));
        if (is && pos < (uint32_t)kFsCap) cand[warp][pos] = lane + 32u * j;
        n += __popc(bal);
    }
    if (census && lane == 0 && (WPQ == 1 || warp == 0)) atomicAdd(census, n);  // DADE_GPU_COARSE_CENSUS
    if (n > (uint32_t)kFsCap) {  // pathological ties: the host redoes the search all-exact
        if (lane == 0) atomicAdd(overflow, 1u);
        n = kFsCap;
    }
    __syncwarp();
    // Sure members: a candidate c with hi_c <= B that fewer than n_probe other
    // candidates can beat (lo_c' <= hi_c: every centroid with a smaller exact
    // (l2_sq, id) key is such a candidate) is in the probe set whatever the exact
    // values are; only the rest (U) get the exact l2_sq, and their (l2_sq, id)
    // order fills the slots the sure members leave. Sure keys carry p~ (the probe
    // order after the nearest matters to no consumer); U keys are flagged with
    // the top bit so the sort puts the sure members first. exact_all (the
    // coarse_probes entry point, whose keys are documented exact): every
    // candidate is in U, i.e. the previous all-exact selection.
    uint32_t nS = 0;
    if (!exact_all) {
        uint32_t* klo = reinterpret_cast<uint32_t*>(rows[warp]);  // free until the exact rounds
        uint32_t* khi = klo + kFsCap;                             // (2 x 384 <= 32 x 36 words)
        for (uint32_t e = lane; e < n; e += 32) {
            const uint32_t c = (uint32_t)cand[warp][e];
            const float p = prow[c], d = coarse_delta(cnorm[c], qn);
            klo[e] = fkey(__fsub_rn(p, d));
            khi[e] = fkey(__fadd_rn(p, d));
        }
        __syncwarp();
        constexpr int kG = kFsCap / 32;
        uint32_t ids[kG];
        uint32_t smask = 0;
        const uint32_t ng = (n + 31) / 32;
#pragma unroll
        for (int i = 0; i < kG; ++i) {
            if ((uint32_t)i >= ng) break;
            const uint32_t e = lane + 32u * i;
            ids[i] = e < n ? (uint32_t)cand[warp][e] : 0u;
            if (e < n) {
                const uint32_t h = khi[e];
                if (h <= B) {
                    uint32_t cnt = 0;
                    for (uint32_t e2 = 0; e2 < n && cnt < n_probe; ++e2) cnt += (e2 != e && klo[e2] <= h) ? 1u : 0u;
                    if (cnt < n_probe) smask |= 1u << i;
                }
            }
        }
        __syncwarp();
        uint32_t nU = 0;
#pragma unroll
        for (int i = 0; i < kG; ++i) {
            if ((uint32_t)i >= ng) break;
            const uint32_t e = lane + 32u * i;
            const bool sure = (smask >> i) & 1u, unsure = e < n && !sure;
            const uint32_t bs = __ballot_sync(0xffffffffu, sure), bu = __ballot_sync(0xffffffffu, unsure);
            const uint32_t lt = (1u << lane) - 1u;
            // sure keys from the front, U ids after them (positions settled below)
            if (sure) cand[warp][nS + __popc(bs & lt)] = make_key(fmaxf(prow[ids[i]], 0.f), ids[i]);
            if (unsure) reinterpret_cast<uint32_t*>(rows[warp])[nU + __popc(bu & lt)] = ids[i];
            nS += __popc(bs);
            nU += __popc(bu);
        }
        __syncwarp();
        for (uint32_t e = lane; e < nU; e += 32) cand[warp][nS + e] = reinterpret_cast<uint32_t*>(rows[warp])[e];
    }
    __syncwarp();
    if (WPQ > 1) __syncthreads();  // every warp's id list is written before keys land in warp 0's
    // exact sequential l2_sq (proj/include/dade/distance.hpp:36-43) of the U candidates
    const float* qr = q + (size_t)qi * dim;
    float* rs = rows[warp];
    float* qs = qch[warp];
    for (uint32_t e0 = nS + 32 * (warp % WPQ); e0 < n; e0 += 32 * WPQ) {
        const uint32_t e = e0 + lane;
        const uint32_t my_c = e < n ? (uint32_t)cand[warp][e] : 0u;
        const uint32_t nv = min(32u, n - e0);
        const float acc = exact_l2_round(cen, qr, dim, my_c, nv, e < n, rs, qs, lane);
        __syncwarp();
        if (e < n) cand[WPQ == 1 ? warp : 0][e] = make_key(acc, my_c) | 0x8000000000000000ull;
    }
    if (WPQ == 1) {
        __syncwarp();
    } else {
        __syncthreads();
        if (warp != 0) return;
    }
    // pad and bitonic-sort the candidate keys (sure members first)
    uint32_t m = 1;
    while (m < n) m <<= 1;
    for (uint32_t e = n + lane; e < m; e += 32) cand[warp][e] = ~0ull;
    __syncwarp();
    uint64_t* kk = cand[warp];
    for (uint32_t size = 2; size <= m; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = lane; i < m / 2; i += 32) {
                const uint32_t lo_i = 2 * i - (i & (stride - 1)), hi_i = lo_i + stride;
                const bool up = (lo_i & size) == 0;
                const uint64_t x = kk[lo_i], y = kk[hi_i];
                if ((x > y) == up) { kk[lo_i] = y; kk[hi_i] = x; }
            }
            __syncwarp();
        }
    for (uint32_t i = lane; i < n_probe; i += 32) probes[(size_t)qi * n_probe + i] = kk[i] & 0x7fffffffffffffffull;
}

// Large-nlist path (1024 < n_cen <= 16384, dim % 4 == 0), warp per query:
//   * one pass over the query's p~ row keeps, per lane and 512-centroid chunk,
//     the minimum upper bound hi of its 16 centroids (<= 32 chunk minima per
//     lane, <= 1024 per query);
//   * T0 = n_probe-th smallest of those minima bounds B from above (the
//     n_probe smallest minima are n_probe distinct hi values <= T0);
//   * a second pass (the row is L2-hot) keeps the centroids with lo <= T0
//     (~n_probe of them): every hi <= B is among them (lo <= hi), so B is
//     their n_probe-th smallest hi; candidates lo <= B get the exact
//     sequential l2_sq, (acc, id) sort, first n_probe -> probes.
// Same answer as coarse_select_kernel, bit for bit.
constexpr int kWdChunk = 512;  // centroids per chunk (16 per lane)
__device__ __forceinline__ uint32_t warp_select_smem(const uint32_t* v, uint32_t n, uint32_t rank, uint32_t* hist,
                                                     uint32_t lane) {
    uint32_t lo = 0xffffffffu, hi = 0;
    for (uint32_t i = lane; i < n; i += 32) {
        lo = min(lo, v[i]);
        hi = max(hi, v[i]);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (hi <= lo) return lo;
    const int top = (31 - __clz(lo ^ hi)) & ~7;
    uint32_t mask = top >= 24 ? 0u : ~0u << (top + 8), prefix = lo & mask;
    for (int shift = top; shift >= 0; shift -= 8) {
        for (uint32_t j = lane; j < 256; j += 32) hist[j] = 0;
        __syncwarp();
        for (uint32_t i = lane; i < n; i += 32)
            if ((v[i] & mask) == prefix) atomicAdd(&hist[(v[i] >> shift) & 0xffu], 1u);
        __syncwarp();
        uint32_t d, before;
        warp_hist_find(hist, rank, lane, d, before);
        rank -= before;
        prefix |= d << shift;
        mask |= 0xffu << shift;
        __syncwarp();
    }
    return prefix;
}

// From the candidates (p~ bits << 32 | centroid, lower bound <= some T >= B) of
// one query in shared memory: B = n_probe-th smallest upper bound among them,
// keep lower bound <= B, exact sequential l2_sq, (acc, id) bitonic sort, first
// n_probe -> probes. Warp-wide; hist / hv / rs / qs are this warp's scratch.
__device__ void finish_from_candidates(uint64_t* cand, uint32_t n, const float* __restrict__ cnorm, float qn,
                                       const float* __restrict__ cen, const float* __restrict__ qr, uint32_t dim,
                                       uint32_t n_probe, uint64_t* __restrict__ probes_row, uint32_t* hist,
                                       uint32_t* hv, float* rs, float* qs, int lane) {
    __syncwarp();
    for (uint32_t e = lane; e < n; e += 32) {
        const uint64_t v = cand[e];
        const uint32_t c = (uint32_t)v;
        hv[e] = fkey(__fadd_rn(__uint_as_float((uint32_t)(v >> 32)), coarse_delta(cnorm[c], qn)));
    }
    __syncwarp();
    const uint32_t B = warp_select_smem(hv, n, n_probe, hist, lane);
    // candidates lo <= B, compacted in place (ids)
    uint32_t m2 = 0;
    for (uint32_t e0 = 0; e0 < n; e0 += 32) {
        const uint32_t e = e0 + lane;
        uint32_t c = 0;
        bool is = false;
        if (e < n) {
            const uint64_t v = cand[e];
            c = (uint32_t)v;
            is = fkey(__fsub_rn(__uint_as_float((uint32_t)(v >> 32)), coarse_delta(cnorm[c], qn))) <= B;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, is);
        __syncwarp();
        if (is) cand[m2 + __popc(bal & ((1u << lane) - 1u))] = c;
        m2 += __popc(bal);
        __syncwarp();
    }
    n = m2;
    __syncwarp();
    // exact sequential l2_sq (proj/include/dade/distance.hpp:36-43) of the candidates
    for (uint32_t e0 = 0; e0 < n; e0 += 32) {
        const uint32_t e = e0 + lane;
        const uint32_t my_c = e < n ? (uint32_t)cand[e] : 0u;
        const uint32_t nv = min(32u, n - e0);
        const float acc = exact_l2_round(cen, qr, dim, my_c, nv, e < n, rs, qs, lane);
        __syncwarp();
        if (e < n) cand[e] = make_key(acc, my_c);
    }
    __syncwarp();
    uint32_t m = 1;
    while (m < n) m <<= 1;
    for (uint32_t e = n + lane; e < m; e += 32) cand[e] = ~0ull;
    __syncwarp();
    uint64_t* kk = cand;
    for (uint32_t size = 2; size <= m; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = lane; i < m / 2; i += 32) {
                const uint32_t lo_i = 2 * i - (i & (stride - 1)), hi_i = lo_i + stride;
                const bool up = (lo_i & size) == 0;
                const uint64_t x = kk[lo_i], y = kk[hi_i];
                if ((x > y) == up) { kk[lo_i] = y; kk[hi_i] = x; }
            }
            __syncwarp();
        }
    for (uint32_t i = lane; i < n_probe; i += 32) probes_row[i] = kk[i];
}

__global__ void __launch_bounds__(kFsWarps * 32, 6) coarse_select_wide_kernel(
    const float* __restrict__ pt, const float* __restrict__ cnorm, const float* __restrict__ qnorm,
    const float* __restrict__ cen, uint32_t n_cen, const float* __restrict__ q, uint32_t nq, uint32_t dim,
    uint32_t n_probe, uint64_t* __restrict__ probes, uint32_t* __restrict__ overflow,
    const uint32_t* __restrict__ gmin) {
    __shared__ uint64_t cand[kFsWarps][kSelCap];
    __shared__ __align__(16) float rows[kFsWarps][32 * kFsRS];
    __shared__ __align__(16) float qch[kFsWarps][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qi = blockIdx.x * kFsWarps + warp;
    if (qi >= nq) return;
    const float* prow = pt + (size_t)qi * n_cen;
    const float qn = qnorm[qi];
    uint32_t* hist = reinterpret_cast<uint32_t*>(rows[warp]);    // 256 words
    uint32_t* hv = hist + 256;                                   // <= 512 hi keys (fits: 768 <= 32 * kFsRS)
    // pass 1: minima of hi over disjoint centroid groups: from the GEMM epilogue
    // (gmin: per query, one per 32 consecutive centroids) or 512-centroid chunks here
    uint32_t gm[32];
    if (gmin) {
        const uint32_t ng = (n_cen + 31) / 32;
        const uint32_t* gr = gmin + (size_t)qi * ng;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t i = lane + 32u * j;
            gm[j] = i < ng ? gr[i] : 0xffffffffu;
        }
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            uint32_t m = 0xffffffffu;
            if ((uint32_t)j * kWdChunk < n_cen) {
#pragma unroll
                for (int i = 0; i < kWdChunk / 32; ++i) {
                    const uint32_t c = j * kWdChunk + i * 32 + lane;
                    if (c < n_cen) m = min(m, fkey(__fadd_rn(prow[c], coarse_delta(cnorm[c], qn))));
                }
            }
            gm[j] = m;
        }
    }
    // T0 = n_probe-th smallest chunk minimum (radix select over registers)
    uint32_t kmin = 0xffffffffu, kmax = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        kmin = min(kmin, gm[j]);
        if (gm[j] != 0xffffffffu) kmax = max(kmax, gm[j]);
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    uint32_t T0 = kmin;
    if (kmax > kmin) {
        const int top = (31 - __clz(kmin ^ kmax)) & ~7;
        uint32_t mask = top >= 24 ? 0u : ~0u << (top + 8), rem = n_probe;
        T0 = kmin & mask;
        for (int shift = top; shift >= 0; shift -= 8) {
            for (uint32_t j = lane; j < 256; j += 32) hist[j] = 0;
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if ((gm[j] & mask) == T0) atomicAdd(&hist[(gm[j] >> shift) & 0xffu], 1u);
            __syncwarp();
            uint32_t d, before;
            warp_hist_find(hist, rem, lane, d, before);
            rem -= before;
            T0 |= d << shift;
            mask |= 0xffu << shift;
            __syncwarp();
        }
    }
    // pass 2: centroids with lo <= T0 -> (p~ bits, id)
    uint32_t n = 0;
    for (uint32_t c0 = 0; c0 < n_cen; c0 += 32) {
        const uint32_t c = c0 + lane;
        float pv = 0.f;
        bool is = false;
        if (c < n_cen) {
            pv = prow[c];
            is = fkey(__fsub_rn(pv, coarse_delta(cnorm[c], qn))) <= T0;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, is);
        const uint32_t pos = n + __popc(bal & ((1u << lane) - 1u));
        if (is && pos < (uint32_t)kSelCap) cand[warp][pos] = (static_cast<uint64_t>(__float_as_uint(pv)) << 32) | c;
        n += __popc(bal);
    }
    if (n > (uint32_t)kSelCap) {  // pathological ties: the host redoes the search all-exact
        if (lane == 0) atomicAdd(overflow, 1u);
        return;
    }
    __syncwarp();
    finish_from_candidates(cand[warp], n, cnorm, qn, cen, q + (size_t)qi * dim, dim, n_probe,
                           probes + (size_t)qi * n_probe, hist, hv, rows[warp], qch[warp], lane);
}

// ---- fused large-nlist selection (p~ never in memory) -------------------------------
// coarse_umma pass A leaves per query the minimum upper-bound key of every 32
// centroids (gmin); T0 = the n_probe-th smallest of those minima >= B (they are
// n_probe distinct upper bounds). Pass B (the GEMM again) lists every centroid
// with lower bound <= T0 -- every exact top-n_probe centroid is among them --
// and coarse_finish_kernel ends as coarse_select_wide_kernel does.
__global__ void __launch_bounds__(kFsWarps * 32) coarse_t0_kernel(const uint32_t* __restrict__ gmin, uint32_t n_cen,
                                                                  uint32_t nq, uint32_t n_probe, uint32_t* t0,
                                                                  bool transposed) {
    __shared__ uint32_t hist[kFsWarps][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qi = blockIdx.x * kFsWarps + warp;
    if (qi >= nq) return;
    const uint32_t ng = (n_cen + 31) / 32;
    uint32_t gm[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        const uint32_t i = lane + 32u * j;
        gm[j] = i < ng ? (transposed ? gmin[(size_t)i * nq + qi] : gmin[(size_t)qi * ng + i]) : 0xffffffffu;
    }
    uint32_t kmin = 0xffffffffu, kmax = 0;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        kmin = min(kmin, gm[j]);
        if (gm[j] != 0xffffffffu) kmax = max(kmax, gm[j]);
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    uint32_t T0 = kmin;
    if (kmax > kmin) {
        const int top = (31 - __clz(kmin ^ kmax)) & ~7;
        uint32_t mask = top >= 24 ? 0u : ~0u << (top + 8), rem = n_probe;
        T0 = kmin & mask;
        for (int shift = top; shift >= 0; shift -= 8) {
            for (uint32_t j = lane; j < 256; j += 32) hist[warp][j] = 0;
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; ++j)
                if ((gm[j] & mask) == T0) atomicAdd(&hist[warp][(gm[j] >> shift) & 0xffu], 1u);
            __syncwarp();
            uint32_t d, before;
            warp_hist_find(hist[warp], rem, lane, d, before);
            rem -= before;
            T0 |= d << shift;
            mask |= 0xffu << shift;
            __syncwarp();
        }
    }
    if (lane == 0) t0[qi] = T0;
}

// parts > 1: the query's list is `parts` slices of cap / parts entries (query-major
// pass B), counts cnt[q * parts + p]; parts == 1: one list, count cnt[q]
__global__ void __launch_bounds__(kFsWarps * 32, 6) coarse_finish_kernel(
    const uint64_t* __restrict__ cand_g, const uint32_t* __restrict__ cnt, uint32_t cap, uint32_t parts,
    const float* __restrict__ cnorm, const float* __restrict__ qnorm, const float* __restrict__ cen,
    const float* __restrict__ q, uint32_t nq, uint32_t dim, uint32_t n_probe, uint64_t* __restrict__ probes,
    uint32_t* __restrict__ overflow) {
    __shared__ uint64_t cand[kFsWarps][kSelCap];
    __shared__ __align__(16) float rows[kFsWarps][32 * kFsRS];
    __shared__ __align__(16) float qch[kFsWarps][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qi = blockIdx.x * kFsWarps + warp;
    if (qi >= nq) return;
    const uint32_t pcap = cap / parts;
    uint32_t n = 0;
    bool over = false;
    for (uint32_t p = 0; p < parts; ++p) {
        const uint32_t np = cnt[(size_t)qi * parts + p];
        over = over || np > pcap;
        if (!over && n + np <= (uint32_t)kSelCap)
            for (uint32_t e = lane; e < np; e += 32) cand[warp][n + e] = cand_g[(size_t)qi * cap + p * pcap + e];
        n += np;
    }
    if (over || n > (uint32_t)kSelCap) {  // pathological ties: the host redoes the search all-exact
        if (lane == 0) atomicAdd(overflow, 1u);
        return;
    }
    uint32_t* hist = reinterpret_cast<uint32_t*>(rows[warp]);
    finish_from_candidates(cand[warp], n, cnorm, qnorm[qi], cen, q + (size_t)qi * dim, dim, n_probe,
                           probes + (size_t)qi * n_probe, hist, hist + 256, rows[warp], qch[warp], lane);
}

// the select kernel for n_cen centroids
void launch_select_any(const float* pt, const float* cnorm, const float* qnorm, const float* centroids, uint32_t n_cen,
                       const float* queries, uint32_t nq, uint32_t dim, uint32_t n_probe, uint64_t* probes,
                       uint32_t* overflow, cudaStream_t s, const uint32_t* gmin = nullptr, bool exact_all = true) {
    if (n_cen <= 1024 && dim % 4 == 0 && n_probe <= kFsCap) {
        uint32_t* census = nullptr;
        if (nq <= 4096 && n_probe > 32)  // > 1 exact round
            // (warps split the exact rounds: skipping the sure members saves no latency here)
            coarse_select_fast_kernel<kFsWarps><<<nq, kFsWarps * 32, 0, s>>>(
                pt, cnorm, qnorm, centroids, n_cen, queries, nq, dim, n_probe, probes, overflow, census, true);
        else
            coarse_select_fast_kernel<1><<<(nq + kFsWarps - 1) / kFsWarps, kFsWarps * 32, 0, s>>>(
                pt, cnorm, qnorm, centroids, n_cen, queries, nq, dim, n_probe, probes, overflow, census, exact_all);
        return;
    }
    if (n_cen <= 32u * kWdChunk && dim % 4 == 0 && n_probe <= kSelCap && !std::getenv("DADE_GPU_SELECT_WARP")) {
        coarse_select_wide_kernel<<<(nq + kFsWarps - 1) / kFsWarps, kFsWarps * 32, 0, s>>>(
            pt, cnorm, qnorm, centroids, n_cen, queries, nq, dim, n_probe, probes, overflow, gmin);
        return;
    }
    coarse_select_kernel<<<(nq + 3) / 4, 128, 0, s>>>(pt, cnorm, qnorm, centroids, n_cen, queries, nq, dim, n_probe,
                                                      probes, overflow);
}

}  // namespace

cudaError_t launch_coarse_tc(const float* centroids, uint32_t n_cen, const float* queries, uint32_t nq, uint32_t dim,
                             uint32_t n_probe, float* cnorm, float* qnorm, float* pt, uint64_t* probes,
                             uint32_t* overflow, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    sq_norms_kernel<<<(unsigned)(((size_t)n_cen + nq + 7) / 8), 256, 0, s>>>(centroids, n_cen, queries, nq, dim,
                                                                             cnorm, qnorm);
    dim3 grid((n_cen + kCC - 1) / kCC, (nq + kCQ - 1) / kCQ);
    coarse_tc_kernel<<<grid, 256, 0, s>>>(centroids, n_cen, queries, nq, dim, cnorm, qnorm, pt);
    launch_select_any(pt, cnorm, qnorm, centroids, n_cen, queries, nq, dim, n_probe, probes, overflow, s);
    return cudaGetLastError();
}

cudaError_t launch_coarse_norms(const float* centroids, uint32_t n_cen, const float* queries, uint32_t nq, uint32_t dim,
                                float* cnorm, float* qnorm, cudaStream_t s) {
    if (nq + n_cen == 0) return cudaSuccess;
    sq_norms_kernel<<<(unsigned)(((size_t)n_cen + nq + 7) / 8), 256, 0, s>>>(centroids, n_cen, queries, nq, dim,
                                                                             cnorm, qnorm);
    return cudaGetLastError();
}

namespace {
// Every centroid probed (the data-ordered flat scan, dade_gpu_flat_partition):
// the nearest by p~ first, the others in id order. No exact ranking: any order
// visits the same candidates; the first cell only seeds the radius. Warp per query.
__global__ void __launch_bounds__(128) coarse_all_kernel(const float* __restrict__ pt, uint32_t n_cen, uint32_t nq,
                                                         uint64_t* __restrict__ probes) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qi = blockIdx.x * 4 + warp;
    if (qi >= nq) return;
    const float* prow = pt + (size_t)qi * n_cen;
    float best = __int_as_float(0x7f800000);
    uint32_t bi = 0xffffffffu;
    for (uint32_t c = lane; c < n_cen; c += 32) {
        const float v = prow[c];
        if (v < best || bi == 0xffffffffu) {
            best = v;
            bi = c;
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, off);
        const uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (oi != 0xffffffffu && (bi == 0xffffffffu || ov < best || (ov == best && oi < bi))) {
            best = ov;
            bi = oi;
        }
    }
    if (bi == 0xffffffffu) bi = 0;  // (all NaN)
    uint64_t* out = probes + (size_t)qi * n_cen;
    for (uint32_t i = lane; i < n_cen; i += 32) {
        const uint32_t j = i == 0 ? bi : (i - 1 < bi ? i - 1 : i);
        out[i] = make_key(fmaxf(prow[j], 0.f), j);
    }
}
}  // namespace

cudaError_t launch_coarse_all(const float* pt, uint32_t n_cen, uint32_t nq, uint64_t* probes, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    coarse_all_kernel<<<(nq + 3) / 4, 128, 0, s>>>(pt, n_cen, nq, probes);
    return cudaGetLastError();
}

cudaError_t launch_coarse_select(const float* centroids, uint32_t n_cen, const float* queries, uint32_t nq,
                                 uint32_t dim, uint32_t n_probe, const float* cnorm, const float* qnorm,
                                 const float* pt, uint64_t* probes, uint32_t* overflow, cudaStream_t s,
                                 const uint32_t* gmin, bool exact_keys) {
    if (nq == 0) return cudaSuccess;
    launch_select_any(pt, cnorm, qnorm, centroids, n_cen, queries, nq, dim, n_probe, probes, overflow, s, gmin,
                      exact_keys);
    return cudaGetLastError();
}

cudaError_t launch_coarse_t0(const uint32_t* gmin, uint32_t n_cen, uint32_t nq, uint32_t n_probe, uint32_t* t0,
                             cudaStream_t s, bool transposed) {
    if (nq == 0) return cudaSuccess;
    if ((n_cen + 31) / 32 > 1024) return cudaErrorInvalidValue;
    coarse_t0_kernel<<<(nq + kFsWarps - 1) / kFsWarps, kFsWarps * 32, 0, s>>>(gmin, n_cen, nq, n_probe, t0,
                                                                             transposed);
    return cudaGetLastError();
}

cudaError_t launch_coarse_finish(const uint64_t* cand, const uint32_t* cnt, uint32_t cap, const float* cnorm,
                                 const float* qnorm, const float* centroids, const float* queries, uint32_t nq,
                                 uint32_t dim, uint32_t n_probe, uint64_t* probes, uint32_t* overflow, cudaStream_t s,
                                 uint32_t parts) {
    if (nq == 0) return cudaSuccess;
    coarse_finish_kernel<<<(nq + kFsWarps - 1) / kFsWarps, kFsWarps * 32, 0, s>>>(
        cand, cnt, cap, parts, cnorm, qnorm, centroids, queries, nq, dim, n_probe, probes, overflow);
    return cudaGetLastError();
}

}  // namespace dade_gpu

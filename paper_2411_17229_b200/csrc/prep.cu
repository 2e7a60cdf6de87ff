// Query rotation (K1), probe grouping (K3) and the per-pair DCO kernels that
// mirror DcoStrategy::evaluate / partial_sqdist / calibration's ratio walk.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

// ---- K1: out[i][k] = (float) sum_r W[k*D + r] * in[i][r] --------------------
// f64 accumulation in r order with separately rounded DMUL/DADD, exactly
// OrthoTransform::transform_vector (proj/src/transform.cpp:221-228).
constexpr int kRotTile = 32;  // output columns per CTA
constexpr int kRotRows = 64;  // rows per CTA (8 per thread: independent DADD chains)
constexpr int kRotK = 32;     // r chunk

__global__ void __launch_bounds__(256)
rotate_kernel(const double* __restrict__ W, uint32_t dim, const float* __restrict__ in, uint32_t n,
              float* __restrict__ out) {
    __shared__ double ws[kRotTile][kRotK + 1];
    __shared__ double xs[kRotRows][kRotK + 1];
    const int tx = threadIdx.x & 31;  // output column within tile
    const int ty = threadIdx.x >> 5;  // 0..7 -> rows ty*8 .. ty*8+7
    const uint32_t col0 = blockIdx.x * kRotTile;
    const uint32_t row0 = blockIdx.y * kRotRows;
    double acc[8];
#pragma unroll
    for (int ii = 0; ii < 8; ++ii) acc[ii] = 0.0;
    for (uint32_t r0 = 0; r0 < dim; r0 += kRotK) {
        __syncthreads();
        for (int idx = threadIdx.x; idx < kRotTile * kRotK; idx += 256) {
            const int a = idx / kRotK, b = idx % kRotK;
            const uint32_t col = col0 + a, r = r0 + b;
            ws[a][b] = (col < dim && r < dim) ? W[(size_t)col * dim + r] : 0.0;
        }
        for (int idx = threadIdx.x; idx < kRotRows * kRotK; idx += 256) {
            const int a = idx / kRotK, b = idx % kRotK;
            const uint32_t row = row0 + a, r = r0 + b;
            xs[a][b] = (row < n && r < dim) ? (double)in[(size_t)row * dim + r] : 0.0;
        }
        __syncthreads();
        const int kmax = (int)min((uint32_t)kRotK, dim - r0);
        for (int b = 0; b < kmax; ++b) {
            const double w = ws[tx][b];
#pragma unroll
            for (int ii = 0; ii < 8; ++ii) acc[ii] = __dadd_rn(acc[ii], __dmul_rn(w, xs[ty * 8 + ii][b]));
        }
    }
    const uint32_t col = col0 + tx;
    if (col < dim) {
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) {
            const uint32_t row = row0 + ty * 8 + ii;
            if (row < n) out[(size_t)row * dim + col] = __double2float_rn(acc[ii]);
        }
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

// Single-CTA exclusive scans of the bucket sizes and item counts.
// work items of one (rank bucket, list) entry: query chunks x row pieces
// Rows [skip, len) of an entry's list still to scan: rank-bucket-0 entries skip
// the rows the seed already scored exactly (when the seed ran: len >= seed_min).
__device__ __forceinline__ uint32_t entry_skip(const GroupArgs& g, uint32_t e, uint32_t len) {
    return (g.seed_skip && e < g.n_lists && len >= g.seed_min) ? min(len, g.seed_skip) : 0u;
}

__device__ __forceinline__ uint32_t entry_items(const GroupArgs& g, uint32_t e, uint32_t c) {
    if (c == 0) return 0;
    const uint32_t list = e % g.n_lists;
    const uint32_t len = g.list_offsets[list + 1] - g.list_offsets[list];
    const uint32_t rem = len - entry_skip(g, e, len);
    if (rem == 0) return 0;
    uint32_t pieces = 1;
    if (g.max_item_rows) pieces = max(1u, (rem + g.max_item_rows - 1) / g.max_item_rows);
    return (c + kQC - 1) / kQC * pieces;
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
        if (e < g.n_lists) sg += (c + 7) / 8;  // seed groups of the nearest-list bucket
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
        if (g.seed_goff && e < g.n_lists) g.seed_goff[e] = rg;
        rb += c;
        ri += entry_items(g, e, c);
        if (e < g.n_lists) rg += (c + 7) / 8;
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

__global__ void group_items_kernel(const GroupArgs g) {
    const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= g.n_rb * g.n_lists) return;
    const uint32_t c = g.counts[e];
    if (c == 0) return;
    const uint32_t list = e % g.n_lists;
    const uint32_t len0 = g.list_offsets[list + 1] - g.list_offsets[list];
    const uint32_t skip = entry_skip(g, e, len0);
    const uint32_t start = g.list_offsets[list] + skip, len = len0 - skip;
    if (len == 0) return;
    const uint32_t ni = (c + kQC - 1) / kQC;
    const uint32_t piece = g.max_item_rows ? g.max_item_rows : max(len, 1u);
    const uint32_t np = max(1u, (len + piece - 1) / piece);
    uint32_t o = g.item_off[e];
    for (uint32_t t = 0; t < ni; ++t)
        for (uint32_t p = 0; p < np; ++p) {
            WorkItem w;
            w.row_start = start + p * piece;
            w.row_count = min(piece, len - p * piece);
            w.bucket_start = g.bucket_off[e] + t * kQC;
            w.bucket_count = min((uint32_t)kQC, c - t * kQC) | (min(p, 0xffffu) << 16);
            g.items[o++] = w;
        }
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

// List-major seed: one CTA per nearest list, for the queries whose nearest
// list it is (the rank-bucket-0 bucket), 8 queries at a time: the list's first
// S rows are staged once per 32-dim slice (coalesced, shared by the 8 queries)
// and every thread advances 2 rows x 8 queries of exact sequential sums; then
// one warp per query sorts its S keys. Same output as seed_radius_kernel.
constexpr int kSeedGroup = 8;
__global__ void __launch_bounds__(kSeedThreads) seed_radius_list_kernel(
    const uint32_t* __restrict__ counts, const uint32_t* __restrict__ bucket_off, const uint32_t* __restrict__ bucket_q,
    const uint32_t* __restrict__ seed_goff, uint32_t n_lists, const uint32_t* __restrict__ list_offsets, const float* __restrict__ storage,
    const uint32_t* __restrict__ row_ids, uint32_t dim, const float* __restrict__ queries, uint32_t K, uint32_t S,
    uint32_t* r_global, uint64_t* out_keys, uint32_t* out_count) {
    extern __shared__ __align__(16) unsigned char seed_smem[];
    float* qt = reinterpret_cast<float*>(seed_smem);                   // [kSeedGroup][32]
    float* tile = qt + kSeedGroup * 32;                                // [kSeedMax][36]
    // after the last slice the tile's space is reused: sums, then sort keys
    float* accs = tile;                                                // [kSeedGroup][kSeedMax]
    uint64_t* keys = reinterpret_cast<uint64_t*>(tile + kSeedGroup * kSeedMax);  // [8 warps][kSeedMax]
    // CTA -> (list, group): binary search in the per-list group prefix
    const uint32_t b = blockIdx.x;
    if (b >= seed_goff[n_lists]) return;
    uint32_t lo_l = 0, hi_l = n_lists;
    while (hi_l - lo_l > 1) {
        const uint32_t mid = (lo_l + hi_l) >> 1;
        if (seed_goff[mid] <= b) lo_l = mid; else hi_l = mid;
    }
    const uint32_t list = lo_l;
    const uint32_t cnt_all = counts[list];  // entry e = list of rank bucket 0
    const uint32_t gfirst = (b - seed_goff[list]) * kSeedGroup;
    if (gfirst >= cnt_all) return;
    const uint32_t start = list_offsets[list], len = list_offsets[list + 1] - start;
    const uint32_t n = min(len, S);
    if (n < K) return;
    const uint32_t* qs = bucket_q + bucket_off[list];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t c4 = tid & 7, rb = tid >> 3;
    const float* rowp = storage + (size_t)(start + min(rb, n - 1)) * dim + 4 * c4;
    const size_t rstep = (size_t)32 * dim;
    const uint32_t r0 = tid, r1 = tid + kSeedThreads;
    const uint32_t cnt = min(cnt_all, gfirst + kSeedGroup);
    for (uint32_t g0 = gfirst; g0 < cnt; g0 += kSeedGroup) {
        const uint32_t ng = min((uint32_t)kSeedGroup, cnt - g0);
        float a0[kSeedGroup], a1[kSeedGroup];
#pragma unroll
        for (int u = 0; u < kSeedGroup; ++u) a0[u] = a1[u] = 0.f;
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
            if (tid < kSeedGroup * 32) {
                const uint32_t u = tid >> 5, k = tid & 31;
                qt[tid] = (u < ng && k < w) ? __ldg(queries + (size_t)qs[g0 + u] * dim + k0 + k) : 0.f;
            }
            __syncthreads();
            for (uint32_t cc = 0; cc < w4; ++cc) {
                const float4 x0 = *reinterpret_cast<const float4*>(tile + r0 * 36 + 4 * cc);
                const float4 x1 = *reinterpret_cast<const float4*>(tile + r1 * 36 + 4 * cc);
#pragma unroll
                for (int u = 0; u < kSeedGroup; ++u) {
                    const float4 y = *reinterpret_cast<const float4*>(qt + u * 32 + 4 * cc);
                    a0[u] = sq_step(a0[u], x0.x, y.x); a1[u] = sq_step(a1[u], x1.x, y.x);
                    a0[u] = sq_step(a0[u], x0.y, y.y); a1[u] = sq_step(a1[u], x1.y, y.y);
                    a0[u] = sq_step(a0[u], x0.z, y.z); a1[u] = sq_step(a1[u], x1.z, y.z);
                    a0[u] = sq_step(a0[u], x0.w, y.w); a1[u] = sq_step(a1[u], x1.w, y.w);
                }
            }
        }
        __syncthreads();  // everyone done reading the last slice
#pragma unroll
        for (int u = 0; u < kSeedGroup; ++u) {
            accs[u * kSeedMax + r0] = a0[u];
            accs[u * kSeedMax + r1] = a1[u];
        }
        __syncthreads();
        if (warp < ng) {  // one warp per query: keys, bitonic sort, outputs
            const uint32_t q = qs[g0 + warp];
            uint64_t* kk = keys + warp * kSeedMax;
            for (uint32_t r = lane; r < (uint32_t)kSeedMax; r += 32) {
                uint64_t key = ~0ull;
                if (r < n) {
                    const uint32_t id = row_ids ? __ldg(row_ids + start + r) : start + r;
                    key = make_key(__fsqrt_rn(accs[warp * kSeedMax + r]), id);
                }
                kk[r] = key;
            }
            __syncwarp();
            for (uint32_t size = 2; size <= (uint32_t)kSeedMax; size <<= 1) {
                for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
                    for (uint32_t i = lane; i < (uint32_t)kSeedMax / 2; i += 32) {
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
            if (lane == 0) atomicMin(r_global + q, (uint32_t)(kk[K - 1] >> 32));
            if (out_keys) {
                for (uint32_t i = lane; i < K; i += 32) out_keys[(size_t)q * K + i] = kk[i];
                if (lane == 0) out_count[q] = K;
            }
        }
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
                                     const uint32_t* seed_goff, uint32_t n_lists, uint32_t max_groups,
                                     const uint32_t* list_offsets, const float* storage,
                                     const uint32_t* row_ids, uint32_t dim, const float* queries, uint32_t K,
                                     uint32_t S, uint32_t* r_global, uint64_t* out_keys, uint32_t* out_count,
                                     cudaStream_t s) {
    if (n_lists == 0 || K > (uint32_t)kSeedMax) return cudaSuccess;
    const size_t smem = sizeof(float) * (kSeedMax * 36 + kSeedGroup * 32);  // sums + keys alias the tile
    DADE_CUDA_TRY(cudaFuncSetAttribute(seed_radius_list_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    seed_radius_list_kernel<<<max_groups, kSeedThreads, smem, s>>>(counts, bucket_off, bucket_q, seed_goff, n_lists,
                                                                    list_offsets,
                                                                 storage, row_ids, dim, queries, K,
                                                                 std::min<uint32_t>(S, kSeedMax), r_global, out_keys,
                                                                 out_count);
    return cudaGetLastError();
}

cudaError_t launch_fill_u32(uint32_t* p, uint32_t v, size_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    fill_u32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, v, n);
    return cudaGetLastError();
}

cudaError_t launch_rotate(const double* W, uint32_t dim, const float* in, uint32_t n, float* out,
                          cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    dim3 grid((dim + kRotTile - 1) / kRotTile, (n + kRotRows - 1) / kRotRows);
    rotate_kernel<<<grid, 256, 0, s>>>(W, dim, in, n, out);
    return cudaGetLastError();
}

cudaError_t launch_group(const GroupArgs& g, cudaStream_t s) {
    const size_t pairs = (size_t)g.nq * g.n_probe;
    const uint32_t ne = g.n_rb * g.n_lists;
    DADE_CUDA_TRY(cudaMemsetAsync(g.counts, 0, sizeof(uint32_t) * ne, s));
    DADE_CUDA_TRY(cudaMemsetAsync(g.cursor, 0, sizeof(uint32_t) * ne, s));
    const unsigned gp = (unsigned)((pairs + 255) / 256);
    if (pairs) group_count_kernel<<<gp, 256, 0, s>>>(g);
    group_scan_kernel<<<1, 1024, 0, s>>>(g);
    if (pairs) group_scatter_kernel<<<gp, 256, 0, s>>>(g);
    group_items_kernel<<<(ne + 255) / 256, 256, 0, s>>>(g);
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

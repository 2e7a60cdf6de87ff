// Radius seed, TMA-pipelined variant of seed_radius_list_kernel (prep.cu) for
// dim <= 256: one CTA per (nearest list, <= 16 of the queries whose nearest list
// it is) scores the list's first S <= 1024 rows exactly, and its K best become
// the queries' first results and radius (same output, bit for bit).
//
//   warp 8       producer: per 8-dim slice, TMA boxes of {8 dims, 256 rows}
//                (32B-swizzled) into a 3-stage ring, full/empty mbarriers;
//   warps 0-7    thread t advances rows t + 256 j (j < kR) x G queries of exact
//                sequential fp32 sums with packed f32x2 arithmetic (two queries
//                per instruction, the rounding of sq_step) from the ring slot and
//                the group's queries (resident, [dim][16]); no CTA barrier inside
//                the dimension loop, so warps drift and the producer runs ahead;
//   then         one warp per query: radix-selected K-th distance, ties at it by
//                id, 128-slot bitonic sort -> out_keys, atomicMin(r_global).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

constexpr int kSdRows = 1024;         // max seeded rows
constexpr int kSdT = 256;             // compute threads (8 warps)
constexpr int kSdThreads = kSdT + 32; // + producer warp
constexpr int kSdG = kSeedGroup;      // queries per CTA (16)
constexpr int kSdSlice = kSeedSlice;  // dims per ring slot (one 16- or 32-byte row segment)
constexpr int kSdStages = 24 / kSdSlice;  // 96 KB ring
constexpr int kSdBox = 256;           // rows per TMA box
constexpr int kSdSmall = 128;         // sorted slots (K <= 128)
constexpr int kSdMaxDim = 256;        // resident queries: [dim][16] fp32

__device__ __forceinline__ uint32_t sd_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void sd_mb_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(sd_u32(bar)), "r"(count));
}
__device__ __forceinline__ void sd_mb_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(sd_u32(bar)) : "memory");
}
__device__ __forceinline__ void sd_mb_arrive_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(sd_u32(bar)), "r"(bytes) : "memory");
}
// try_wait with a suspend-time hint: a waiting warp sleeps instead of spinning
__device__ __forceinline__ void sd_mb_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAITS_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAITS_%=;\n"
        "}\n" ::"r"(sd_u32(bar)),
        "r"(parity), "r"(1000000u)
        : "memory");
}
__device__ __forceinline__ void sd_tma2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(sd_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(sd_u32(bar))
        : "memory");
}
__device__ __forceinline__ void sd_cp4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sd_u32(dst)), "l"(src) : "memory");
}

struct SdLayout {
    size_t ring, qres, bars, total;
};
__host__ __device__ inline SdLayout sd_layout() {
    SdLayout L;
    size_t off = 0;
    L.ring = off; off += (size_t)kSdStages * kSdRows * kSdSlice * 4;  // 96 KB; reused for sums / keys / histograms
    L.qres = off; off += (size_t)kSdMaxDim * kSdG * 4;                // 16 KB
    L.bars = off; off += 8 * 2 * kSdStages;
    L.total = off + 256;  // base alignment slack (32B-swizzled TMA destinations need 256 B)
    return L;
}

// exact sums of rows (tid + 256 j, j < kR) x G queries -> accs[u][row].
// Slices sl_base .. sl_base + n_slices - 1 of a kStages-deep ring (global slice
// numbering: the persistent kernel's ring runs across groups). kPersist: the
// sums go to a separate buffer once afree (if wait_free) completes, and every
// thread arrives on aready; otherwise they overwrite the ring.
template <int G, int kR, int kStages, bool kPersist, int kT = kSdT>
__device__ __forceinline__ void sd_sums(const unsigned char* ring, const float* qres, uint64_t* full, uint64_t* empty,
                                        uint32_t sl_base, uint32_t n_slices, float* accs, uint64_t nz2,
                                        uint64_t* afree = nullptr, bool wait_free = false, uint32_t free_parity = 0,
                                        uint64_t* aready = nullptr) {
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    uint64_t acc[kR][G / 2];
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int p = 0; p < G / 2; ++p) acc[j][p] = 0ull;
    for (uint32_t k = 0; k < n_slices; ++k) {
        const uint32_t sl = sl_base + k;
        const uint32_t s = sl % kStages;
        sd_mb_wait(full + s, (sl / kStages) & 1);
        const unsigned char* slot = ring + (size_t)s * kSdRows * kSdSlice * 4;
        const float* qb = qres + (size_t)k * kSdSlice * kSdG;
#pragma unroll
        for (int c = 0; c < kSdSlice / 4; ++c) {
            float o[kR][4];
#pragma unroll
            for (int j = 0; j < kR; ++j) {
                const uint32_t r = min(tid + j * kT, (uint32_t)kSdRows - 1);  // rows >= 1024 (kT = 384): never stored
                // 4-dim slices: 16-byte rows, unswizzled; 8-dim: 32B-swizzled, 16-byte chunk c ^ row bit 2
                const float4 x = kSdSlice == 4
                                     ? *reinterpret_cast<const float4*>(slot + r * 16)
                                     : *reinterpret_cast<const float4*>(slot + r * 32 + (((uint32_t)c ^ (r >> 2)) & 1u) * 16);
                o[j][0] = x.x;
                o[j][1] = x.y;
                o[j][2] = x.z;
                o[j][3] = x.w;
            }
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const ulonglong2* q4 = reinterpret_cast<const ulonglong2*>(qb + (4 * c + e) * kSdG);
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
        __syncwarp();
        if (lane == 0) sd_mb_arrive(empty + s);  // this warp is done with the slot
    }
    if (kPersist) {
        if (wait_free) sd_mb_wait(afree, free_parity);
    } else {
        // the ring is reused for the sums: every warp must be past its last slot
        asm volatile("bar.sync 1, %0;\n" ::"r"(kSdT));
    }
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int p = 0; p < G / 2; ++p) {
            const uint32_t r = tid + j * kT;
            if (kT * kR <= kSdRows || r < (uint32_t)kSdRows) {
                accs[(2 * p) * kSdRows + r] = lo_f(acc[j][p]);
                accs[(2 * p + 1) * kSdRows + r] = hi_f(acc[j][p]);
            }
        }
    if (kPersist) sd_mb_arrive(aready);
    else asm volatile("bar.sync 1, %0;\n" ::"r"(kSdT));
}

template <int NV>
__device__ __forceinline__ uint32_t sd_select(const uint32_t (&v)[NV], uint32_t K, uint32_t* hist, uint32_t lane,
                                              uint32_t& c_lt, uint32_t& c_eq) {
    uint32_t lo = 0xffffffffu, hi = 0;
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        lo = min(lo, v[i]);
        hi = max(hi, v[i] == 0xffffffffu ? 0u : v[i]);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (hi <= lo) {  // every present value equal
        c_lt = 0;
        c_eq = 0;
#pragma unroll
        for (int i = 0; i < NV; ++i) c_eq += __popc(__ballot_sync(0xffffffffu, v[i] == lo));
        return lo;
    }
    const int top = (31 - __clz(lo ^ hi)) & ~7;  // lowest byte boundary above which all present values agree
    uint32_t mask = top >= 24 ? 0u : ~0u << (top + 8);
    uint32_t prefix = lo & mask, rem = K, d = 0;
    for (int shift = top; shift >= 0; shift -= 8) {
        for (uint32_t j = lane; j < 256; j += 32) hist[j] = 0;
        __syncwarp();
#pragma unroll
        for (int i = 0; i < NV; ++i)
            if ((v[i] & mask) == prefix) atomicAdd(&hist[(v[i] >> shift) & 0xffu], 1u);
        __syncwarp();
        uint32_t before;
        warp_hist_find(hist, rem, lane, d, before);
        rem -= before;
        prefix |= d << shift;
        mask |= 0xffu << shift;
        if (shift == 0) c_eq = hist[d];
        __syncwarp();
    }
    c_lt = K - rem;
    return prefix;
}

__device__ __forceinline__ void sd_bitonic(uint64_t* kk, uint32_t m, uint32_t lane) {
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

// One warp: the K smallest exact sums of query q over rows [0, n) of the list at
// start (acc[r]) by (sqrt distance, id) -> sorted keys out_keys[q], radius
// atomicMin(r_global[q]). kk: 128 keys, hist: 256 words (per warp, shared).
__device__ __forceinline__ void sd_finish_query(const SeedListArgs& a, uint32_t q, const float* accs, uint32_t u,
                                             uint32_t n, uint32_t start, uint64_t* kk, uint32_t* hist) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t* row_ids = a.row_ids;
    const uint32_t K = a.K;
    const float* acc = accs + u * kSdRows;
    constexpr int kNV = kSdRows / 32;
    uint32_t dv[kNV];
#pragma unroll
    for (int i = 0; i < kNV; ++i) {
        const uint32_t r = lane + 32u * i;
        dv[i] = r < n ? __float_as_uint(__fsqrt_rn(acc[r])) : 0xffffffffu;
    }
    uint32_t c_lt, c_eq;
    const uint32_t T = sd_select(dv, K, hist, lane, c_lt, c_eq);  // K-th smallest distance
    uint32_t tid_max = 0xffffffffu;  // ties at T taken by ascending id
    if (c_lt + c_eq > (uint32_t)kSdSmall) {
        uint32_t iv[kNV];
#pragma unroll
        for (int i = 0; i < kNV; ++i) {
            const uint32_t r = lane + 32u * i;
            iv[i] = dv[i] == T ? (row_ids ? __ldg(row_ids + start + r) : a.id_base + start + r) : 0xffffffffu;
        }
        uint32_t t_lt, t_eq;
        tid_max = sd_select(iv, K - c_lt, hist, lane, t_lt, t_eq);
    }
    // ids of the values <= T, loaded together ahead of the (ballot-serialised) compaction
    uint32_t idv[kNV];
#pragma unroll
    for (int i = 0; i < kNV; ++i) {
        const uint32_t r = lane + 32u * i;
        idv[i] = dv[i] <= T ? (row_ids ? __ldg(row_ids + start + r) : a.id_base + start + r) : 0u;
    }
    uint32_t c = 0;
#pragma unroll
    for (int i = 0; i < kNV; ++i) {
        const uint32_t id = idv[i];
        const bool take = dv[i] < T || (dv[i] == T && id <= tid_max);
        const uint32_t bal = __ballot_sync(0xffffffffu, take);
        const uint32_t pos = c + __popc(bal & ((1u << lane) - 1u));
        if (take && pos < (uint32_t)kSdSmall) kk[pos] = make_key(__uint_as_float(dv[i]), id);
        c += __popc(bal);
    }
    for (uint32_t r = c + lane; r < (uint32_t)kSdSmall; r += 32) kk[r] = ~0ull;
    __syncwarp();
    sd_bitonic(kk, kSdSmall, lane);
    if (lane == 0) atomicMin(a.r_global + q, (uint32_t)(kk[K - 1] >> 32));
    if (a.out_keys) {
        for (uint32_t i = lane; i < K; i += 32) a.out_keys[(size_t)q * K + i] = kk[i];
        if (lane == 0) a.out_count[q] = K;
    }
}



// ---- persistent, warp-specialised seed ------------------------------------------
// One CTA per SM walks the seed groups in the order a global counter hands them
// out (largest-first is not needed: a group is ~1/7 of a CTA's share):
//   warp 15       producer: next group id -> gid slot (4 slots, gfull/gempty),
//                 then its 8-dim slices by TMA into a 2-stage ring (full/empty,
//                 slice numbering continues across groups);
//   warps 0-7     sums (sd_sums, as seed_tma_kernel) into accs[i & 1] once the
//                 selection warps freed it (afree), then aready;
//   warps 8-14    selection (sd_finish_query) of group i while the sum warps
//                 already run group i + 1, so the FMA pipe never idles on it.
#ifndef DADE_SP_SUM_WARPS
#define DADE_SP_SUM_WARPS 8
#endif
constexpr int kSpS = DADE_SP_SUM_WARPS;            // sum warps
constexpr int kSpL = 15 - kSpS;                    // selection warps (16 warps in all: 4 per SM sub-partition)
constexpr int kSpT = kSpS * 32;                    // sum threads: rows t + kSpT j
constexpr int kSpThreads = (kSpS + kSpL + 1) * 32;  // 512
constexpr int kSpStages = 16 / kSdSlice;  // 64 KB ring
constexpr int kSpSlots = 4;
constexpr uint32_t kSpEnd = 0xffffffffu;

struct SpLayout {
    size_t ring, accs, qres, keys, hist, gid, bars, total;
};
__host__ __device__ inline SpLayout sp_layout() {
    SpLayout L;
    size_t off = 0;
    L.ring = off; off += (size_t)kSpStages * kSdRows * kSdSlice * 4;  // 64 KB
    L.accs = off; off += 2ull * kSdG * kSdRows * 4;                   // 128 KB
    L.qres = off; off += (size_t)kSdMaxDim * kSdG * 4;                // 16 KB
    L.keys = off; off += (size_t)kSpL * kSdSmall * 8;
    L.hist = off; off += (size_t)kSpL * 256 * 4;
    L.gid = off; off += 64;
    L.bars = off; off += 8 * (2 * kSpStages + 2 * kSpSlots + 4);
    L.total = off + 256;
    return L;
}

struct SpGroup {
    uint32_t start, n, ng;
    const uint32_t* qs;
};
__device__ __forceinline__ bool sp_group(const SeedListArgs& a, uint32_t b, SpGroup& G) {
    const uint32_t list = a.seed_glist[b];
    const uint32_t cnt_all = a.counts[list];
    const uint32_t g0 = (b - a.seed_goff[list]) * kSdG;
    if (g0 >= cnt_all) return false;
    G.start = a.list_offsets[list];
    G.n = min(a.list_offsets[list + 1] - G.start, a.S);
    if (G.n < a.K) return false;
    G.qs = a.bucket_q + a.bucket_off[list] + g0;
    G.ng = min((uint32_t)kSdG, cnt_all - g0);
    return true;
}
__device__ __forceinline__ int sp_rsel(uint32_t n) { return n > 2u * kSdT ? 4 : n > (uint32_t)kSdT ? 2 : 1; }
__device__ __forceinline__ int sp_rows_per_thread(uint32_t n) { return (int)((n + kSpT - 1) / kSpT); }

__global__ void __launch_bounds__(kSpThreads, 1) seed_persist_kernel(const SeedListArgs a,
                                                                      const __grid_constant__ CUtensorMap tmap,
                                                                      uint32_t* work) {
    extern __shared__ unsigned char sd_raw[];
    unsigned char* sm = sd_raw + ((256u - (sd_u32(sd_raw) & 255u)) & 255u);
    const SpLayout L = sp_layout();
    unsigned char* ring = sm + L.ring;
    float* accs = reinterpret_cast<float*>(sm + L.accs);  // [2][16][1024]
    float* qres = reinterpret_cast<float*>(sm + L.qres);  // [dim][16]
    uint64_t* keys = reinterpret_cast<uint64_t*>(sm + L.keys);
    uint32_t* hists = reinterpret_cast<uint32_t*>(sm + L.hist);
    volatile uint32_t* gid = reinterpret_cast<volatile uint32_t*>(sm + L.gid);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bars);
    uint64_t* empty = full + kSpStages;
    uint64_t* gfull = empty + kSpStages;
    uint64_t* gempty = gfull + kSpSlots;
    uint64_t* aready = gempty + kSpSlots;
    uint64_t* afree = aready + 2;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t n_groups = a.seed_goff[a.n_lists];
    const uint32_t dim = a.dim;
    const uint32_t n_slices = (dim + kSdSlice - 1) / kSdSlice;
    if (tid == 0) {
        for (int i = 0; i < kSpStages; ++i) {
            sd_mb_init(full + i, 1);
            sd_mb_init(empty + i, kSpS);
        }
        for (int j = 0; j < kSpSlots; ++j) {
            sd_mb_init(gfull + j, 1);
            sd_mb_init(gempty + j, kSpL);
        }
        for (int b = 0; b < 2; ++b) {
            sd_mb_init(aready + b, kSpT);
            sd_mb_init(afree + b, kSpL);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == kSpS + kSpL) {
        // ---- producer ----
        if (lane != 0) return;
        uint32_t sl = 0;
        for (uint32_t i = 0;; ++i) {
            const uint32_t j = i % kSpSlots;
            if (i >= (uint32_t)kSpSlots) sd_mb_wait(gempty + j, ((i / kSpSlots) - 1) & 1);
            uint32_t b;
            SpGroup G;
            for (;;) {
                b = atomicAdd(work, 1u);
                if (b < n_groups && a.order) b = a.order[b];  // costliest groups first (shorter tail)
                if (b >= n_groups || sp_group(a, b, G)) break;
            }
            gid[j] = b < n_groups ? b : kSpEnd;
            sd_mb_arrive(gfull + j);
            if (b >= n_groups) return;
            if (a.census) atomicAdd(a.census, (unsigned long long)G.n * G.ng * dim);
            if (a.counters) atomicAdd(a.counters + 2, 4ull * G.n * dim);  // the group's rows, loaded once
            const uint32_t n_boxes = (uint32_t)sp_rsel(G.n);
            const uint32_t bytes = n_boxes * kSdBox * kSdSlice * 4;
            for (uint32_t k = 0; k < n_slices; ++k, ++sl) {
                const uint32_t s = sl % kSpStages;
                if (sl >= (uint32_t)kSpStages) sd_mb_wait(empty + s, ((sl / kSpStages) - 1) & 1);
                sd_mb_arrive_tx(full + s, bytes);
                unsigned char* slot = ring + (size_t)s * kSdRows * kSdSlice * 4;
                for (uint32_t bx = 0; bx < n_boxes; ++bx)
                    sd_tma2d(slot + (size_t)bx * kSdBox * kSdSlice * 4, &tmap, (int)(k * kSdSlice),
                             (int)(G.start + bx * kSdBox), full + s);
            }
        }
    }
    if (warp < kSpS) {
        // ---- sums ----
        uint32_t sl = 0;
        for (uint32_t i = 0;; ++i) {
            const uint32_t j = i % kSpSlots;
            sd_mb_wait(gfull + j, (i / kSpSlots) & 1);
            const uint32_t b = gid[j];
            if (b == kSpEnd) return;
            SpGroup G;
            sp_group(a, b, G);
            // every sum warp is past the previous group's queries
            asm volatile("bar.sync 1, %0;\n" ::"r"(kSpS * 32) : "memory");
            for (uint32_t e = tid; e < dim * kSdG; e += kSpS * 32) {
                const uint32_t k = e / kSdG, u = e % kSdG;
                if (u < G.ng) sd_cp4(qres + e, a.queries + (size_t)G.qs[u] * dim + k);
                else qres[e] = 0.f;
            }
            for (uint32_t e = dim * kSdG + tid; e < n_slices * kSdSlice * kSdG; e += kSpS * 32) qres[e] = 0.f;
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            asm volatile("bar.sync 1, %0;\n" ::"r"(kSpS * 32) : "memory");
            const uint32_t buf = i & 1;
            float* acc = accs + (size_t)buf * kSdG * kSdRows;
            const bool wf = i >= 2;
            const uint32_t fp = ((i >> 1) - 1) & 1;
            const int rsel = sp_rows_per_thread(G.n);
            switch ((G.ng + 1) >> 1) {
#define SP_R(P, R)                                                                                            \
    sd_sums<2 * P, R, kSpStages, true, kSpT>(ring, qres, full, empty, sl, n_slices, acc, a.nz2, afree + buf, wf, fp, \
                                             aready + buf)
#define SP_G(P)                                                 \
    case P:                                                     \
        if (rsel >= 4) SP_R(P, 4);                              \
        else if (rsel == 3) SP_R(P, 3);                         \
        else if (rsel == 2) SP_R(P, 2);                         \
        else SP_R(P, 1);                                        \
        break;
                SP_G(1) SP_G(2) SP_G(3) SP_G(4) SP_G(5) SP_G(6) SP_G(7) default: SP_G(8)
#undef SP_R
#undef SP_G
            }
            sl += n_slices;
        }
    }
    // ---- selection ----
    const uint32_t lw = warp - kSpS;
    for (uint32_t i = 0;; ++i) {
        const uint32_t j = i % kSpSlots;
        sd_mb_wait(gfull + j, (i / kSpSlots) & 1);
        const uint32_t b = gid[j];
        if (b == kSpEnd) return;
        SpGroup G;
        sp_group(a, b, G);
        const uint32_t buf = i & 1;
        sd_mb_wait(aready + buf, (i >> 1) & 1);
        const float* acc = accs + (size_t)buf * kSdG * kSdRows;
        for (uint32_t u = lw; u < G.ng; u += kSpL)
            sd_finish_query(a, G.qs[u], acc, u, G.n, G.start, keys + lw * kSdSmall, hists + lw * 256);
        __syncwarp();
        if (lane == 0) {
            sd_mb_arrive(afree + buf);
            sd_mb_arrive(gempty + j);
        }
    }
}

// Costliest-first order of the seed groups for the persistent kernel's work
// counter (LPT: the last groups handed out are the cheapest, so SMs finish
// together). Cost = seeded rows x query pairs, counting-sorted into 64 buckets
// by one CTA; the order inside a bucket does not matter (groups are independent).
constexpr int kSoBins = 64;
__global__ void __launch_bounds__(1024) seed_order_kernel(const SeedListArgs a, uint32_t* order) {
    __shared__ uint32_t hist[kSoBins];
    const uint32_t n_groups = a.seed_goff[a.n_lists];
    if (threadIdx.x < kSoBins) hist[threadIdx.x] = 0;
    __syncthreads();
    auto bucket = [&](uint32_t b) -> uint32_t {
        SpGroup G;
        if (!sp_group(a, b, G)) return 0;
        const uint32_t cost = G.n * ((G.ng + 1) >> 1);  // <= 1024 x 8
        return min((uint32_t)kSoBins - 1, cost >> 7);
    };
    for (uint32_t b = threadIdx.x; b < n_groups; b += blockDim.x) atomicAdd(&hist[bucket(b)], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {  // descending buckets: exclusive prefix from the top
        uint32_t run = 0;
        for (int i = kSoBins - 1; i >= 0; --i) {
            const uint32_t h = hist[i];
            hist[i] = run;
            run += h;
        }
    }
    __syncthreads();
    for (uint32_t b = threadIdx.x; b < n_groups; b += blockDim.x) order[atomicAdd(&hist[bucket(b)], 1u)] = b;
}

}  // namespace

bool seed_tma_ok(uint32_t dim, uint32_t K) { return dim <= (uint32_t)kSdMaxDim && dim % 4 == 0 && K <= (uint32_t)kSdSmall; }

cudaError_t launch_seed_tma(const SeedListArgs& a, const CUtensorMap& tmap, uint32_t max_groups, cudaStream_t s,
                            uint32_t* work) {
    if (a.n_lists == 0 || max_groups == 0) return cudaSuccess;
    if (!work) return cudaErrorInvalidValue;  // the persistent kernel's group counter
    static_assert((size_t)kSdStages * kSdRows * kSdSlice * 4 >=
                      (size_t)kSdG * kSdRows * 4 + (kSdT / 32) * (kSdSmall * 8 + 256 * 4),
                  "sums + keys + histograms must fit in the ring");
    const size_t sp = sp_layout().total;
    int dev = 0, n_sm = 0;
    DADE_CUDA_TRY(cudaGetDevice(&dev));
    DADE_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    DADE_CUDA_TRY(cudaFuncSetAttribute(seed_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp));
    DADE_CUDA_TRY(cudaMemsetAsync(work, 0, 4, s));
    if (a.order) seed_order_kernel<<<1, 1024, 0, s>>>(a, a.order);
    seed_persist_kernel<<<std::min<uint32_t>(max_groups, (uint32_t)n_sm), kSpThreads, sp, s>>>(a, tmap, work);
    return cudaGetLastError();
}

}  // namespace dade_gpu

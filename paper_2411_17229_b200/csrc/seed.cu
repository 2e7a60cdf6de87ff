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

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

constexpr int kSdRows = 1024;         // max seeded rows
constexpr int kSdT = 256;             // compute threads (8 warps)
constexpr int kSdThreads = kSdT + 32; // + producer warp
constexpr int kSdG = kSeedGroup;      // queries per CTA (16)
constexpr int kSdSlice = 8;           // dims per ring slot (one 32-byte row segment)
constexpr int kSdStages = 3;
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

// exact sums of rows (tid + 256 j, j < kR) x G queries -> accs[u][row]
template <int G, int kR>
__device__ __forceinline__ void sd_sums(const unsigned char* ring, const float* qres, uint64_t* full, uint64_t* empty,
                                        uint32_t n_slices, float* accs, uint64_t nz2) {
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    uint64_t acc[kR][G / 2];
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int p = 0; p < G / 2; ++p) acc[j][p] = 0ull;
    for (uint32_t sl = 0; sl < n_slices; ++sl) {
        const uint32_t s = sl % kSdStages;
        sd_mb_wait(full + s, (sl / kSdStages) & 1);
        const unsigned char* slot = ring + (size_t)s * kSdRows * kSdSlice * 4;
        const float* qb = qres + (size_t)sl * kSdSlice * kSdG;
#pragma unroll
        for (int c = 0; c < kSdSlice / 4; ++c) {
            float o[kR][4];
#pragma unroll
            for (int j = 0; j < kR; ++j) {
                const uint32_t r = tid + j * kSdT;
                // 32B-swizzled row segment: 16-byte chunk c ^ row bit 2
                const float4 x = *reinterpret_cast<const float4*>(slot + r * 32 + (((uint32_t)c ^ (r >> 2)) & 1u) * 16);
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
    // the ring is reused for the sums: every warp must be past its last slot
    asm volatile("bar.sync 1, %0;\n" ::"r"(kSdT));
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int p = 0; p < G / 2; ++p) {
            const uint32_t r = tid + j * kSdT;
            accs[(2 * p) * kSdRows + r] = lo_f(acc[j][p]);
            accs[(2 * p + 1) * kSdRows + r] = hi_f(acc[j][p]);
        }
    asm volatile("bar.sync 1, %0;\n" ::"r"(kSdT));
}

// K-th smallest (1-based) of the warp's values v (0xffffffff = absent; at least
// K present) by 8-bit radix digits, starting below the bits every present value
// shares (min ^ max) so that no round piles the whole warp onto one histogram
// bin. Also returns how many values are < and == the result.
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

__global__ void __launch_bounds__(kSdThreads, 2) seed_tma_kernel(const SeedListArgs a,
                                                                  const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ unsigned char sd_raw[];
    unsigned char* sm = sd_raw + ((256u - (sd_u32(sd_raw) & 255u)) & 255u);
    const SdLayout L = sd_layout();
    unsigned char* ring = sm + L.ring;
    float* qres = reinterpret_cast<float*>(sm + L.qres);  // [dim][16]
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + L.bars);
    uint64_t* empty = full + kSdStages;
    const uint32_t b = blockIdx.x;
    if (b >= a.seed_goff[a.n_lists]) return;
    const uint32_t list = a.seed_glist[b];
    const uint32_t cnt_all = a.counts[list];
    const uint32_t g0 = (b - a.seed_goff[list]) * kSdG;
    if (g0 >= cnt_all) return;
    const uint32_t start = a.list_offsets[list], len = a.list_offsets[list + 1] - start;
    const uint32_t n = min(len, a.S);
    if (n < a.K) return;
    const uint32_t* qs = a.bucket_q + a.bucket_off[list] + g0;
    const uint32_t ng = min((uint32_t)kSdG, cnt_all - g0);
    const uint32_t dim = a.dim;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t n_slices = (dim + kSdSlice - 1) / kSdSlice;
    const int rsel = n > 2u * kSdT ? 4 : n > (uint32_t)kSdT ? 2 : 1;
    const uint32_t n_boxes = (uint32_t)rsel;  // 256-row boxes per slice (rows past n are never read)

    if (tid == 0) {
        for (int i = 0; i < kSdStages; ++i) {
            sd_mb_init(full + i, 1);
            sd_mb_init(empty + i, kSdT / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // resident queries, transposed [dim][16] (padding queries and dims: 0)
    for (uint32_t i = tid; i < dim * kSdG; i += kSdThreads) {
        const uint32_t k = i / kSdG, u = i % kSdG;
        if (u < ng) sd_cp4(qres + i, a.queries + (size_t)qs[u] * dim + k);
        else qres[i] = 0.f;
    }
    for (uint32_t i = dim * kSdG + tid; i < n_slices * kSdSlice * kSdG; i += kSdThreads) qres[i] = 0.f;
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();

    float* accs = reinterpret_cast<float*>(ring);  // after the dimension loop: [16][1024] sums
    if (warp == kSdT / 32) {
        // ---- producer ----
        if (lane == 0) {
            const uint32_t bytes = n_boxes * kSdBox * kSdSlice * 4;
            for (uint32_t sl = 0; sl < n_slices; ++sl) {
                const uint32_t s = sl % kSdStages;
                if (sl >= (uint32_t)kSdStages) sd_mb_wait(empty + s, ((sl / kSdStages) - 1) & 1);
                sd_mb_arrive_tx(full + s, bytes);
                unsigned char* slot = ring + (size_t)s * kSdRows * kSdSlice * 4;
                for (uint32_t bx = 0; bx < n_boxes; ++bx)
                    sd_tma2d(slot + (size_t)bx * kSdBox * kSdSlice * 4, &tmap, (int)(sl * kSdSlice),
                             (int)(start + bx * kSdBox), full + s);
            }
        }
        __syncwarp();
    } else {
        switch ((ng + 1) >> 1) {
#define SD_G(P)                                                                                 \
    case P:                                                                                     \
        if (rsel == 4) sd_sums<2 * P, 4>(ring, qres, full, empty, n_slices, accs, a.nz2);       \
        else if (rsel == 2) sd_sums<2 * P, 2>(ring, qres, full, empty, n_slices, accs, a.nz2);  \
        else sd_sums<2 * P, 1>(ring, qres, full, empty, n_slices, accs, a.nz2);                 \
        break;
            SD_G(1) SD_G(2) SD_G(3) SD_G(4) SD_G(5) SD_G(6) SD_G(7) default: SD_G(8)
#undef SD_G
        }
        // ---- selection: one warp per query ----
        uint64_t* keys = reinterpret_cast<uint64_t*>(accs + kSdG * kSdRows);           // [8 warps][128]
        uint32_t* hists = reinterpret_cast<uint32_t*>(keys + (kSdT / 32) * kSdSmall);  // [8 warps][256]
        const uint32_t* row_ids = a.row_ids;
        const uint32_t K = a.K;
        for (uint32_t u = warp; u < ng; u += kSdT / 32) {
            const uint32_t q = qs[u];
            uint64_t* kk = keys + warp * kSdSmall;
            uint32_t* hist = hists + warp * 256;
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
            __syncwarp();
        }
    }
}

}  // namespace

bool seed_tma_ok(uint32_t dim, uint32_t K) { return dim <= (uint32_t)kSdMaxDim && dim % 4 == 0 && K <= (uint32_t)kSdSmall; }

cudaError_t launch_seed_tma(const SeedListArgs& a, const CUtensorMap& tmap, uint32_t max_groups, cudaStream_t s) {
    if (a.n_lists == 0 || max_groups == 0) return cudaSuccess;
    const size_t smem = sd_layout().total;
    static_assert((size_t)kSdStages * kSdRows * kSdSlice * 4 >=
                      (size_t)kSdG * kSdRows * 4 + (kSdT / 32) * (kSdSmall * 8 + 256 * 4),
                  "sums + keys + histograms must fit in the ring");
    DADE_CUDA_TRY(cudaFuncSetAttribute(seed_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    seed_tma_kernel<<<max_groups, kSdThreads, smem, s>>>(a, tmap);
    return cudaGetLastError();
}

}  // namespace dade_gpu

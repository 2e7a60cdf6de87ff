// Radius seed (K4a), persistent and TMA-pipelined: per (nearest list, <= 16 of
// the queries whose nearest list it is) the list's first S <= 1024 rows are
// scored exactly, and each query's K best become its first results and radius
// (bit for bit what seed_radius_list_kernel in prep.cu computes, which remains
// for dims the TMA path cannot tile).
//
// One CTA per SM walks the seed groups in the order a global counter hands them
// out (costliest first, seed_order_kernel):
//   warp 15       producer: next group id -> gid slot (4 slots, gfull/gempty),
//                 then the group's 8-dim row slices by TMA ({8 dims, 256 rows}
//                 32B-swizzled boxes) into a ring of full/empty mbarrier slots;
//                 slice numbering continues across groups, so the ring stays
//                 full across group boundaries;
//   warps 0-7     thread t advances rows t + 256 j (j < kR) x G queries of exact
//                 sequential fp32 sums with packed f32x2 arithmetic (two queries
//                 per instruction, the rounding of sq_step) from the ring slot and
//                 the group's queries (resident, [dim][16]), holding them in
//                 registers until the group's last slice, then store them in the
//                 sums buffer once the selection warps freed it (afree / aready);
//   warps 8-14    selection of group i (one warp per query: radix-selected K-th
//                 distance, ties at it by id, 128-slot bitonic sort -> out_keys,
//                 atomicMin(r_global)) while the sum warps already run group i+1.
//
// Shared-memory geometry is chosen per launch (SpGeom): slots hold the slice of
// up to slot_rows = S rounded up to 256, 512 or 1024 rows, so short seeds (256 rows above dim
// 256) get 8 KB slots and a 16-deep ring, and the ring takes whatever the sums
// buffer [16][slot_rows] and the resident queries [dim][16] leave: the seed
// streams up to 1 MB per group with little arithmetic per byte when a group
// holds few queries, so the bytes in flight per SM set its speed.
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace dade_gpu {

namespace {

constexpr int kSdRowsMax = 1024;      // max seeded rows
constexpr int kSdBox = 256;           // rows per TMA box
constexpr int kSdG = kSeedGroup;      // queries per group (16)
constexpr int kSdSlice = kSeedSlice;  // dims per ring slot (one 32-byte row segment)
constexpr int kSdSmall = 128;         // sorted slots (K <= 128)
constexpr int kSdMaxDim = 1024;       // resident queries: [dim][16] fp32 <= 64 KB
constexpr int kSpS = 8;               // sum warps
constexpr int kSpL = 7;               // selection warps (16 warps in all: 4 per SM sub-partition)
constexpr int kSpT = kSpS * 32;       // sum threads: rows t + kSpT j
constexpr int kSpThreads = (kSpS + kSpL + 1) * 32;  // 512
constexpr int kSpSlots = 4;           // group-id queue
constexpr int kSpMaxStages = 32;
constexpr uint32_t kSpEnd = 0xffffffffu;
constexpr size_t kSpSmemMax = 232448 - 1024;  // opt-in maximum less the reserved 1 KB

// per-launch shared-memory geometry (byte offsets from a 256-aligned base)
struct SpGeom {
    uint32_t slot_rows, slot_bytes, stages;
    uint32_t ring, accs, qres, keys, hist, gid, bars, total;
};
SpGeom sp_geom(uint32_t dim, uint32_t S) {
    SpGeom g{};
    g.slot_rows = S <= 256 ? 256 : S <= 512 ? 512 : 1024;  // the kernel's template instances
    g.slot_bytes = g.slot_rows * kSdSlice * 4;
    const uint32_t n_slices = (dim + kSdSlice - 1) / kSdSlice;
    uint32_t off = 0;
    const uint32_t accs = (uint32_t)kSdG * g.slot_rows * 4;
    const uint32_t qres = n_slices * kSdSlice * kSdG * 4;
    const uint32_t fixed = accs + qres + kSpL * kSdSmall * 8 + kSpL * 256 * 4 + 64 +
                           8 * (2 * kSpMaxStages + 2 * kSpSlots + 2) + 256;
    g.stages = fixed >= kSpSmemMax ? 0 : std::min<uint32_t>(kSpMaxStages, (uint32_t)((kSpSmemMax - fixed) / g.slot_bytes));
    g.ring = off; off += g.stages * g.slot_bytes;
    g.accs = off; off += accs;
    g.qres = off; off += qres;
    g.keys = off; off += kSpL * kSdSmall * 8;
    g.hist = off; off += kSpL * 256 * 4;
    g.gid = off; off += 64;
    g.bars = off; off += 8 * (2 * kSpMaxStages + 2 * kSpSlots + 2);
    g.total = off + 256;  // base alignment slack (32B-swizzled TMA destinations need 256 B)
    return g;
}

// exact sums of rows (tid + kSpT j, j < kR) x G queries over slices sl_base ..
// sl_base + n_slices - 1 of the ring (global slice numbering) -> accs[u][row]
// (row stride slot_rows) once afree (if wait_free) completes; every thread then
// arrives on aready.
template <int G, int kR, int kSlotRows>
__device__ __forceinline__ void sp_sums(const unsigned char* ring, const SpGeom& g, const float* qres,
                                        uint64_t* full, uint64_t* empty, uint32_t sl_base, uint32_t n_slices,
                                        float* accs, uint64_t nz2, uint64_t* afree, bool wait_free,
                                        uint32_t free_parity, uint64_t* aready) {
    const uint32_t tid = threadIdx.x, lane = tid & 31;
    uint64_t acc[kR][G / 2];
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int p = 0; p < G / 2; ++p) acc[j][p] = 0ull;
    // ring slot and phase of slice sl_base, then advanced incrementally (no
    // division by the runtime stage count inside the slice loop)
    uint32_t s = sl_base % g.stages, ph = (sl_base / g.stages) & 1;
    for (uint32_t k = 0; k < n_slices; ++k) {
        mb_wait(full + s, ph);
        const unsigned char* slot = ring + (size_t)s * (kSlotRows * kSdSlice * 4);
        const float* qb = qres + (size_t)k * kSdSlice * kSdG;
#pragma unroll
        for (int c = 0; c < kSdSlice / 4; ++c) {
            float o[kR][4];
#pragma unroll
            for (int j = 0; j < kR; ++j) {
                const uint32_t r = min(tid + j * kSpT, (uint32_t)kSlotRows - 1);
                // 8-dim slices: 32-byte rows, 32B-swizzled (16-byte chunk c ^ row bit 2)
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
        if (lane == 0) mb_arrive(empty + s);  // this warp is done with the slot
        if (++s == g.stages) {
            s = 0;
            ph ^= 1;
        }
    }
    if (wait_free) mb_wait(afree, free_parity);
#pragma unroll
    for (int j = 0; j < kR; ++j)
#pragma unroll
        for (int p = 0; p < G / 2; ++p) {
            const uint32_t r = tid + j * kSpT;
            if (kSpT * kR <= kSlotRows || r < (uint32_t)kSlotRows) {
                accs[(2 * p) * kSlotRows + r] = lo_f(acc[j][p]);
                accs[(2 * p + 1) * kSlotRows + r] = hi_f(acc[j][p]);
            }
        }
    mb_arrive(aready);
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
// start (acc[r], row stride of the sums buffer) by (sqrt distance, id) -> sorted
// keys out_keys[q], radius atomicMin(r_global[q]). kk: 128 keys, hist: 256
// words (per warp, shared).
__device__ __forceinline__ void sd_finish_query(const SeedListArgs& a, uint32_t q, const float* acc, uint32_t n,
                                                uint32_t start, uint64_t* kk, uint32_t* hist) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t* row_ids = a.row_ids;
    const uint32_t K = a.K;
    constexpr int kNV = kSdRowsMax / 32;
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
__device__ __forceinline__ int sp_rows_per_thread(uint32_t n) { return (int)((n + kSpT - 1) / kSpT); }

template <int kSlotRows>
__global__ void __launch_bounds__(kSpThreads, 1) seed_persist_kernel(const SeedListArgs a, const SpGeom geom,
                                                                      const __grid_constant__ CUtensorMap tmap,
                                                                      uint32_t* work) {
    extern __shared__ unsigned char sd_raw[];
    unsigned char* sm = sd_raw + ((256u - (su32(sd_raw) & 255u)) & 255u);
    const SpGeom& g = geom;
    unsigned char* ring = sm + g.ring;
    float* accs = reinterpret_cast<float*>(sm + g.accs);  // [16][slot_rows]
    float* qres = reinterpret_cast<float*>(sm + g.qres);  // [dim][16]
    uint64_t* keys = reinterpret_cast<uint64_t*>(sm + g.keys);
    uint32_t* hists = reinterpret_cast<uint32_t*>(sm + g.hist);
    volatile uint32_t* gid = reinterpret_cast<volatile uint32_t*>(sm + g.gid);
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + g.bars);
    uint64_t* empty = full + kSpMaxStages;
    uint64_t* gfull = empty + kSpMaxStages;
    uint64_t* gempty = gfull + kSpSlots;
    uint64_t* aready = gempty + kSpSlots;
    uint64_t* afree = aready + 1;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t n_groups = a.seed_goff[a.n_lists];
    const uint32_t dim = a.dim;
    const uint32_t n_slices = (dim + kSdSlice - 1) / kSdSlice;
    if (tid == 0) {
        for (uint32_t i = 0; i < g.stages; ++i) {
            mb_init(full + i, 1);
            mb_init(empty + i, kSpS);
        }
        for (int j = 0; j < kSpSlots; ++j) {
            mb_init(gfull + j, 1);
            mb_init(gempty + j, kSpL);
        }
        mb_init(aready, kSpT);
        mb_init(afree, kSpL);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (warp == kSpS + kSpL) {
        // ---- producer ----
        if (lane != 0) return;
        uint32_t s = 0, ph = 0, used = 0;  // ring slot, its phase, slots filled so far (< stages: no wait)
        for (uint32_t i = 0;; ++i) {
            const uint32_t j = i % kSpSlots;
            if (i >= (uint32_t)kSpSlots) mb_wait_sleep(gempty + j, ((i / kSpSlots) - 1) & 1, 400);
            uint32_t b;
            SpGroup G;
            for (;;) {
                b = atomicAdd(work, 1u);
                if (b < n_groups && a.order) b = a.order[b];  // costliest groups first (shorter tail)
                if (b >= n_groups || sp_group(a, b, G)) break;
            }
            gid[j] = b < n_groups ? b : kSpEnd;
            mb_arrive(gfull + j);
            if (b >= n_groups) return;
            if (a.census) atomicAdd(a.census, (unsigned long long)G.n * G.ng * dim);
            if (a.counters) atomicAdd(a.counters + 2, 4ull * G.n * dim);  // the group's rows, loaded once
            const uint32_t n_boxes = (G.n + kSdBox - 1) / kSdBox;
            const uint32_t bytes = n_boxes * kSdBox * kSdSlice * 4;
            for (uint32_t k = 0; k < n_slices; ++k) {
                if (used >= g.stages) mb_wait_sleep(empty + s, ph ^ 1, 100);  // the slot's previous fill consumed
                else ++used;
                mb_arrive_tx(full + s, bytes);
                unsigned char* slot = ring + (size_t)s * g.slot_bytes;
                for (uint32_t bx = 0; bx < n_boxes; ++bx)
                    tma2d_u(slot + (size_t)bx * kSdBox * kSdSlice * 4, &tmap, (int)(k * kSdSlice),
                            (int)(G.start + bx * kSdBox), full + s);
                if (++s == g.stages) {
                    s = 0;
                    ph ^= 1;
                }
            }
        }
    }
    if (warp < kSpS) {
        // ---- sums ----
        uint32_t sl = 0;
        for (uint32_t i = 0;; ++i) {
            const uint32_t j = i % kSpSlots;
            mb_wait(gfull + j, (i / kSpSlots) & 1);
            const uint32_t b = gid[j];
            if (b == kSpEnd) return;
            SpGroup G;
            sp_group(a, b, G);
            // every sum warp is past the previous group's queries
            asm volatile("bar.sync 1, %0;\n" ::"r"(kSpT) : "memory");
            for (uint32_t e = tid; e < dim * kSdG; e += kSpT) {
                const uint32_t k = e / kSdG, u = e % kSdG;
                if (u < G.ng) {
                    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(su32(qres + e)),
                                 "l"(a.queries + (size_t)G.qs[u] * dim + k)
                                 : "memory");
                } else {
                    qres[e] = 0.f;
                }
            }
            for (uint32_t e = dim * kSdG + tid; e < n_slices * kSdSlice * kSdG; e += kSpT) qres[e] = 0.f;
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            asm volatile("bar.sync 1, %0;\n" ::"r"(kSpT) : "memory");
            const bool wf = i >= 1;
            const uint32_t fp = (i - 1) & 1;
            const int rsel = sp_rows_per_thread(G.n);
            switch ((G.ng + 1) >> 1) {
#define SP_R(P, R) \
    sp_sums<2 * P, R, kSlotRows>(ring, g, qres, full, empty, sl, n_slices, accs, a.nz2, afree, wf, fp, aready)
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
        mb_wait_sleep(gfull + j, (i / kSpSlots) & 1, 400);
        const uint32_t b = gid[j];
        if (b == kSpEnd) return;
        SpGroup G;
        sp_group(a, b, G);
        mb_wait_sleep(aready, i & 1, 400);
        for (uint32_t u = lw; u < G.ng; u += kSpL)
            sd_finish_query(a, G.qs[u], accs + (size_t)u * kSlotRows, G.n, G.start, keys + lw * kSdSmall,
                            hists + lw * 256);
        __syncwarp();
        if (lane == 0) {
            mb_arrive(afree);
            mb_arrive(gempty + j);
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

bool seed_tma_ok(uint32_t dim, uint32_t K) {
    return dim <= (uint32_t)kSdMaxDim && dim % 4 == 0 && K <= (uint32_t)kSdSmall && sp_geom(dim, kSdRowsMax).stages >= 2;
}

cudaError_t launch_seed_tma(const SeedListArgs& a, const CUtensorMap& tmap, uint32_t max_groups, cudaStream_t s,
                            uint32_t* work) {
    if (a.n_lists == 0 || max_groups == 0) return cudaSuccess;
    if (!work || a.S > (uint32_t)kSdRowsMax) return cudaErrorInvalidValue;  // the persistent kernel's group counter
    const SpGeom g = sp_geom(a.dim, a.S);
    if (g.stages < 2) return cudaErrorInvalidValue;
    int dev = 0, n_sm = 0;
    DADE_CUDA_TRY(cudaGetDevice(&dev));
    DADE_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    DADE_CUDA_TRY(cudaMemsetAsync(work, 0, 4, s));
    if (a.order) seed_order_kernel<<<1, 1024, 0, s>>>(a, a.order);
    const uint32_t grid = std::min<uint32_t>(max_groups, (uint32_t)n_sm);
    auto run = [&](auto kern) -> cudaError_t {
        DADE_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.total));
        kern<<<grid, kSpThreads, g.total, s>>>(a, g, tmap, work);
        return cudaGetLastError();
    };
    // slot rows as a compile-time constant: the sums' row and slot arithmetic
    // stays immediate (a runtime stride cost the D <= 256 seed 3%)
    if (g.slot_rows <= 256) return run(seed_persist_kernel<256>);
    if (g.slot_rows <= 512) return run(seed_persist_kernel<512>);
    return run(seed_persist_kernel<1024>);
}

}  // namespace dade_gpu

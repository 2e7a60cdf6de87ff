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
            if (i >= (uint32_t)kSpSlots) mb_wait(gempty + j, ((i / kSpSlots) - 1) & 1);
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
                if (used >= g.stages) mb_wait(empty + s, ph ^ 1);  // the slot's previous fill consumed
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
        mb_wait(gfull + j, (i / kSpSlots) & 1);
        const uint32_t b = gid[j];
        if (b == kSpEnd) return;
        SpGroup G;
        sp_group(a, b, G);
        mb_wait(aready, i & 1);
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


// ---- tensor-core-bounded seed (dim % 32 == 0, 32 <= dim <= 256) ------------------
// Same output as seed_persist_kernel, bit for bit, with a fraction of its exact
// arithmetic. Per 128-row block of a group's seeded rows:
//   * tcgen05.mma kind::tf32 (M = 128 rows, N = 16 queries; the fp32 rows
//     straight from a TMA ring, 128B-swizzled) gives t = o.q in TMEM, hence
//     d~ = |o|^2 + |q|^2 - 2t with |d~ - acc| <= E = 4.2e-3 |o||q| + 4e-5 (|o|^2 +
//     |q|^2), acc the reference's sequential fp32 sum (TF32 operands < 2^-10
//     relative each: dot error < (2^-9 + 2^-20) |o||q|; fp32 accumulation and
//     norms, and acc's own rounding, < 4e-5 of the norms);
//   * ub = d~ + E of every row goes into a per-query 128-bin histogram over
//     [0, U_q] (U_q = the largest ub of the group's first block, the last bin
//     open-ended); T_q = the upper edge of the bin holding the K-th smallest ub
//     so far (+inf in the last bin): K rows have acc <= ub <= T_q, so the K-th
//     smallest exact sum is <= T_q;
//   * a (row, query) pair is skipped iff lb = d~ - E > T_q (1 + 2^-20): its sqrt
//     distance then strictly exceeds the K-th one, so it can neither be among
//     the K best nor tie with them (the first block is scored whole: T = inf);
//   * the candidate pairs, listed by query, get the exact sequential fp32 sums
//     (two pairs per lane on packed f32x2) from a second TMA ring that re-reads
//     the block a block later (an L2 hit); skipped pairs are stored as NaN, which
//     sorts after every distance;
//   * the selection is the dense kernel's (sd_finish_query) over the group's
//     [16][1024] sums in a per-CTA global scratch (two groups in flight).
// Warps: 0-5 exact sums, 6-9 epilogue (TMEM lane quarter = warp % 4), 10 group
// queue + query staging + MMA-stream TMA, 11 exact-stream TMA, 12 MMA, 13-15
// selection.
constexpr int kTcM = 128;               // rows per block (MMA M, TMEM lanes)
constexpr int kTcG = 16;                // queries per group (MMA N)
constexpr int kTcAtom = kTcM * 128;     // bytes per A atom: 128 rows x 32 fp32 (SW128)
constexpr int kTcQAtom = kTcG * 128;    // bytes per B atom: 16 queries x 32 fp32
constexpr int kTcMaxAtoms = 8;          // dim <= 256
constexpr int kTcMS = 4, kTcES = 4;     // A ring slots (MMA stream, exact stream)
constexpr int kTcBins = 128;
constexpr int kTcEx = 6, kTcEpi = 4, kTcSel = 3;
constexpr int kTcWEpi = kTcEx, kTcWProdA = kTcEx + kTcEpi, kTcWProdB = kTcWProdA + 1, kTcWMma = kTcWProdA + 2,
              kTcWSel = kTcWProdA + 3;
constexpr int kTcThreads = (kTcWSel + kTcSel) * 32;  // 512
constexpr int kTcExT = kTcEx * 32;                 // exact threads
constexpr int kTcMaxPairs = kTcM * kTcG;           // 2048
constexpr int kTcRounds = (kTcMaxPairs + 2 * kTcExT - 1) / (2 * kTcExT);  // 6
constexpr uint32_t kTcTmemCols = 32;               // 2 accumulator buffers x 16 columns

struct TcMisc {
    uint32_t gid[kSpSlots];
    uint32_t pl_n[2];
    uint32_t cnt[kTcEpi][kTcG];
    uint32_t u_bits[kTcG];
    float T[kTcG];
    float qn[2][kTcG];
    uint32_t tmem;
};
struct TcLayout {
    uint32_t ra, re, q, pl, hist, keys, shist, misc, bars, total;
};
__host__ __device__ inline TcLayout tc_layout() {
    TcLayout L;
    uint32_t off = 0;
    L.ra = off; off += kTcMS * kTcAtom;                      // 64 KB
    L.re = off; off += kTcES * kTcAtom;                      // 64 KB
    L.q = off; off += 2 * kTcMaxAtoms * kTcQAtom;            // 32 KB: two groups' queries
    L.pl = off; off += 2 * kTcMaxPairs * 2;                  // 8 KB: two blocks' pair lists (u16)
    L.hist = off; off += kTcG * kTcBins * 4;                 // 8 KB
    L.keys = off; off += kTcSel * kSdSmall * 8;              // selection keys
    L.shist = off; off += kTcSel * 256 * 4;                  // selection histograms
    L.misc = off; off += (sizeof(TcMisc) + 15) & ~15u;
    L.bars = off; off += 8 * 48;
    L.total = off + 1024;                                    // base alignment (SW128 atoms: 1024 B)
    return L;
}

__device__ __forceinline__ uint64_t pk2(float lo, float hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
// exact step of two packed (row, query) pairs: sq_step's rounding in each half
__device__ __forceinline__ uint64_t sq_step2p(uint64_t acc, uint64_t o2, uint64_t q2, uint64_t nz2) {
    uint64_t d, m, r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(o2), "l"(q2));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(m) : "l"(d), "l"(nz2));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(acc), "l"(m));
    return r;
}
__device__ __forceinline__ void tc_ld16_wait(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tc_epi_bar() { asm volatile("bar.sync 2, %0;\n" ::"r"(kTcEpi * 32) : "memory"); }

__global__ void __launch_bounds__(kTcThreads, 1) seed_tc_kernel(const SeedListArgs a,
                                                                const __grid_constant__ CUtensorMap tmap,
                                                                const float* __restrict__ full_norms,
                                                                float* __restrict__ scratch, uint32_t* work) {
    extern __shared__ unsigned char tc_raw[];
    unsigned char* sm = tc_raw + ((1024u - (su32(tc_raw) & 1023u)) & 1023u);
    const TcLayout L = tc_layout();
    TcMisc* ms = reinterpret_cast<TcMisc*>(sm + L.misc);
    uint16_t* pls = reinterpret_cast<uint16_t*>(sm + L.pl);
    uint32_t* hist = reinterpret_cast<uint32_t*>(sm + L.hist);
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
    uint64_t* ma_full = bars;          // [4] MMA-stream slot loaded
    uint64_t* ma_empty = bars + 4;     // [4] its MMAs done (commit)
    uint64_t* ex_full = bars + 8;      // [4] exact-stream slot loaded
    uint64_t* ex_empty = bars + 12;    // [4] every exact warp past it
    uint64_t* acc_full = bars + 16;    // [2] block's MMAs done (commit)
    uint64_t* acc_empty = bars + 18;   // [2] epilogue read the accumulators
    uint64_t* pl_full = bars + 20;     // [2] pair list written (epilogue)
    uint64_t* pl_empty = bars + 22;    // [2] exact warps done with it
    uint64_t* q_full = bars + 24;      // [2] group's queries staged
    uint64_t* q_empty = bars + 26;     // [2] MMA (commit), exact and epilogue warps done with them
    uint64_t* g_full = bars + 28;      // [4] group id published
    uint64_t* g_empty = bars + 32;     // [4] every consumer warp took it
    uint64_t* g_done = bars + 36;      // [2] group's exact sums stored (scratch)
    uint64_t* s_free = bars + 38;      // [2] group's selection done (scratch parity free)
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t n_groups = a.seed_goff[a.n_lists];
    const uint32_t dim = a.dim, n_atoms = dim / 32;
    float* scr = scratch + (size_t)blockIdx.x * 2 * kTcG * kSdRowsMax;  // [2][16][1024] per CTA
    constexpr uint32_t kConsumers = 1 + 1 + kTcEpi + kTcEx + kTcSel;   // g_empty arrivals (warps)
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) {
            mb_init(ma_full + i, 1);
            mb_init(ma_empty + i, 1);
            mb_init(ex_full + i, 1);
            mb_init(ex_empty + i, kTcEx);
            mb_init(g_full + i, 1);
            mb_init(g_empty + i, kConsumers);
        }
        for (int i = 0; i < 2; ++i) {
            mb_init(acc_full + i, 1);
            mb_init(acc_empty + i, kTcEpi);
            mb_init(pl_full + i, kTcEpi);
            mb_init(pl_empty + i, kTcEx);
            mb_init(q_full + i, 1);
            mb_init(q_empty + i, 1 + kTcEx + kTcEpi);
            mb_init(g_done + i, kTcEx);
            mb_init(s_free + i, kTcSel);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == kTcWMma) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(&ms->tmem)),
                     "r"(kTcTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = ms->tmem;

    // the i-th group of this CTA (false: no more)
    auto take_group = [&](uint32_t i, SpGroup& G) -> bool {
        const uint32_t j = i % kSpSlots;
        mb_wait(g_full + j, (i / kSpSlots) & 1);
        const uint32_t b = ms->gid[j];
        __syncwarp();
        if (lane == 0) mb_arrive(g_empty + j);
        if (b == kSpEnd) return false;
        sp_group(a, b, G);
        return true;
    };

    if (warp == kTcWProdA) {
        // ---- group queue, query staging, MMA-stream TMA ----
        uint32_t s = 0, ph = 0, used = 0;
        for (uint32_t i = 0;; ++i) {
            const uint32_t j = i % kSpSlots;
            if (i >= (uint32_t)kSpSlots) mb_wait(g_empty + j, ((i / kSpSlots) - 1) & 1);
            uint32_t b = 0;
            if (lane == 0) {
                SpGroup G0;
                for (;;) {
                    b = atomicAdd(work, 1u);
                    if (b < n_groups && a.order) b = a.order[b];  // costliest groups first
                    if (b >= n_groups || sp_group(a, b, G0)) break;
                }
                ms->gid[j] = b < n_groups ? b : kSpEnd;
                mb_arrive(g_full + j);
            }
            b = __shfl_sync(0xffffffffu, b, 0);
            if (b >= n_groups) break;
            SpGroup G;
            sp_group(a, b, G);
            if (lane == 0 && a.counters) atomicAdd(a.counters + 2, 4ull * G.n * dim);  // rows, once from HBM
            // queries -> SW128 K-major B atoms (16 rows x 128 B each), and |q|^2
            const uint32_t qb = i & 1;
            if (i >= 2) mb_wait(q_empty + qb, ((i >> 1) - 1) & 1);
            unsigned char* qt = sm + L.q + qb * kTcMaxAtoms * kTcQAtom;
            for (uint32_t e = lane; e < kTcG * n_atoms * 8; e += 32) {  // 16-byte chunks
                const uint32_t u = e / (n_atoms * 8), rem = e % (n_atoms * 8), at = rem / 8, ch = rem % 8;
                unsigned char* dst = qt + at * kTcQAtom + u * 128 + ((ch ^ (u & 7)) << 4);
                if (u < G.ng) cp16(dst, a.queries + (size_t)G.qs[u] * dim + at * 32 + ch * 4);
                else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            __syncwarp();
            {  // |q|^2 from the staged tile: lanes 2u, 2u + 1 take query u's two halves of each atom
                const uint32_t u = lane >> 1, h = lane & 1;
                float acc = 0.f;
                for (uint32_t at = 0; at < n_atoms; ++at)
#pragma unroll
                    for (uint32_t ch = 4 * h; ch < 4 * h + 4; ++ch) {
                        const float4 v =
                            *reinterpret_cast<const float4*>(qt + at * kTcQAtom + u * 128 + ((ch ^ (u & 7)) << 4));
                        acc = fmaf(v.x, v.x, fmaf(v.y, v.y, fmaf(v.z, v.z, fmaf(v.w, v.w, acc))));
                    }
                acc += __shfl_xor_sync(0xffffffffu, acc, 1);
                if (h == 0) ms->qn[qb][u] = acc;
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) mb_arrive(q_full + qb);
            // rows: every block's atoms, MMA stream
            const uint32_t nb = (G.n + kTcM - 1) / kTcM;
            for (uint32_t blk = 0; blk < nb; ++blk)
                for (uint32_t at = 0; at < n_atoms; ++at) {
                    if (lane == 0) {
                        if (used >= (uint32_t)kTcMS) mb_wait(ma_empty + s, ph ^ 1);
                        else ++used;
                        mb_arrive_tx(ma_full + s, kTcAtom);
                        tma2d_u(sm + L.ra + s * kTcAtom, &tmap, (int)(at * 32), (int)(G.start + blk * kTcM),
                                ma_full + s);
                    }
                    __syncwarp();
                    if (++s == (uint32_t)kTcMS) {
                        s = 0;
                        ph ^= 1;
                    }
                }
        }
    } else if (warp == kTcWProdB) {
        // ---- exact-stream TMA: the same atoms again, about a block later ----
        uint32_t s = 0, ph = 0, used = 0;
        for (uint32_t i = 0;; ++i) {
            SpGroup G;
            if (!take_group(i, G)) break;
            const uint32_t nb = (G.n + kTcM - 1) / kTcM;
            for (uint32_t blk = 0; blk < nb; ++blk)
                for (uint32_t at = 0; at < n_atoms; ++at) {
                    if (lane == 0) {
                        if (used >= (uint32_t)kTcES) mb_wait(ex_empty + s, ph ^ 1);
                        else ++used;
                        mb_arrive_tx(ex_full + s, kTcAtom);
                        tma2d_u(sm + L.re + s * kTcAtom, &tmap, (int)(at * 32), (int)(G.start + blk * kTcM),
                                ex_full + s);
                    }
                    __syncwarp();
                    if (++s == (uint32_t)kTcES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
        }
    } else if (warp == kTcWMma) {
        // ---- MMA issuer ----
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kTcG >> 3) << 17) |
                               ((uint32_t)(kTcM >> 4) << 24);
        uint32_t s = 0, ph = 0, it = 0;
        for (uint32_t i = 0;; ++i) {
            SpGroup G;
            if (!take_group(i, G)) break;
            const uint32_t qb = i & 1;
            mb_wait(q_full + qb, (i >> 1) & 1);
            const unsigned char* qt = sm + L.q + qb * kTcMaxAtoms * kTcQAtom;
            const uint32_t nb = (G.n + kTcM - 1) / kTcM;
            for (uint32_t blk = 0; blk < nb; ++blk, ++it) {
                const uint32_t buf = it & 1;
                if (it >= 2) mb_wait(acc_empty + buf, ((it >> 1) - 1) & 1);
                tc_fence_after();
                for (uint32_t at = 0; at < n_atoms; ++at) {
                    mb_wait(ma_full + s, ph);
                    tc_fence_after();
                    if (lane == 0) {
                        const uint32_t sa = su32(sm + L.ra + s * kTcAtom), sb = su32(qt + at * kTcQAtom);
                        for (uint32_t kk = 0; kk < 4; ++kk)
                            tc_mma(tmem + buf * 16, desc_sw128(sa + kk * 32), desc_sw128(sb + kk * 32), idesc,
                                   (at | kk) ? 1u : 0u);
                        tc_commit(ma_empty + s);
                        if (at + 1 == n_atoms) tc_commit(acc_full + buf);
                    }
                    __syncwarp();
                    if (++s == (uint32_t)kTcMS) {
                        s = 0;
                        ph ^= 1;
                    }
                }
            }
            if (lane == 0) tc_commit(q_empty + qb);  // the group's B operand is no longer read
            __syncwarp();
        }
    } else if (warp >= (uint32_t)kTcWEpi && warp < (uint32_t)(kTcWEpi + kTcEpi)) {
        // ---- epilogue: bounds, histogram threshold, candidate pairs ----
        const uint32_t ew = warp - kTcWEpi, quarter = warp & 3;  // TMEM lanes 32 (warp % 4) ..
        const uint32_t r = quarter * 32 + lane;                   // row in the block
        const uint32_t lt = (1u << lane) - 1u;
        uint32_t it = 0;
        for (uint32_t i = 0;; ++i) {
            SpGroup G;
            if (!take_group(i, G)) break;
            const uint32_t qb = i & 1, par = i & 1;
            mb_wait(q_full + qb, (i >> 1) & 1);
            float qn[kTcG], qnr[kTcG];
#pragma unroll
            for (int u = 0; u < kTcG; ++u) {
                qn[u] = ms->qn[qb][u];
                qnr[u] = sqrtf(qn[u]);
            }
            __syncwarp();
            if (lane == 0) mb_arrive(q_empty + qb);
            if (i >= 2) mb_wait(s_free + par, ((i >> 1) - 1) & 1);  // this scratch parity's selection is done
            float* sg = scr + (size_t)par * kTcG * kSdRowsMax;
            for (uint32_t e = ew * 32 + lane; e < kTcG * kTcBins; e += kTcEpi * 32) hist[e] = 0u;
            if (ew == 0 && lane < kTcG) ms->u_bits[lane] = 0u;
            tc_epi_bar();
            const uint32_t nb = (G.n + kTcM - 1) / kTcM;
            for (uint32_t blk = 0; blk < nb; ++blk, ++it) {
                const uint32_t buf = it & 1;
                const uint32_t gr = blk * kTcM + r;
                const bool valid = gr < G.n;
                const float on = valid ? __ldg(full_norms + G.start + gr) : 0.f;
                const float onr = sqrtf(on);
                mb_wait(acc_full + buf, (it >> 1) & 1);
                tc_fence_after();
                float t[16];
                tc_ld16_wait(tmem + ((quarter * 32) << 16) + buf * 16, t);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mb_arrive(acc_empty + buf);
                float lb[kTcG], ub[kTcG];
#pragma unroll
                for (int u = 0; u < kTcG; ++u) {
                    const float d = on + qn[u] - 2.f * t[u];
                    const float e = 4.2e-3f * onr * qnr[u] + 4e-5f * (on + qn[u]);
                    lb[u] = d - e;
                    ub[u] = fmaxf(d + e, 0.f);
                }
                if (blk == 0) {  // histogram range U_q: the largest ub of the group's first block
#pragma unroll
                    for (int u = 0; u < kTcG; ++u) {
                        const uint32_t m =
                            __reduce_max_sync(0xffffffffu, (valid && u < (int)G.ng) ? __float_as_uint(ub[u]) : 0u);
                        if (lane == 0 && u < (int)G.ng) atomicMax(&ms->u_bits[u], m);
                    }
                    tc_epi_bar();
                }
                if (valid) {
#pragma unroll
                    for (int u = 0; u < kTcG; ++u) {
                        if (u >= (int)G.ng) break;
                        const float U = __uint_as_float(ms->u_bits[u]);
                        const int bin = U > 0.f ? min(kTcBins - 1, (int)(ub[u] * ((float)kTcBins / U))) : 0;
                        atomicAdd(&hist[u * kTcBins + bin], 1u);
                    }
                }
                tc_epi_bar();
                // T_q: upper edge of the bin holding the K-th smallest ub so far (warp ew: queries 4 ew ..)
                for (uint32_t u = ew; u < G.ng; u += kTcEpi) {
                    const uint32_t* h = hist + u * kTcBins;
                    const uint4 hv = *reinterpret_cast<const uint4*>(h + 4 * lane);
                    const uint32_t sum = hv.x + hv.y + hv.z + hv.w;
                    uint32_t incl = sum;
#pragma unroll
                    for (int off = 1; off < 32; off <<= 1) {
                        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                        if (lane >= (uint32_t)off) incl += y;
                    }
                    const uint32_t excl = incl - sum;
                    // first bin with cumulative count >= K
                    int bin = -1;
                    if (excl < a.K && incl >= a.K) {
                        uint32_t c = excl;
                        const uint32_t v4[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
                        for (int q4 = 0; q4 < 4; ++q4) {
                            c += v4[q4];
                            if (bin < 0 && c >= a.K) bin = 4 * (int)lane + q4;
                        }
                    }
                    const uint32_t who = __ballot_sync(0xffffffffu, bin >= 0);
                    const int b2 = who ? __shfl_sync(0xffffffffu, bin, __ffs(who) - 1) : kTcBins - 1;
                    if (lane == 0) {
                        const float U = __uint_as_float(ms->u_bits[u]);
                        ms->T[u] = b2 >= kTcBins - 1 ? __int_as_float(0x7f800000)
                                                     : (float)(b2 + 1) * (U / (float)kTcBins) * (1.f + 0x1p-10f);
                    }
                }
                tc_epi_bar();
                // candidates (the first block whole); skipped pairs stored as NaN
                uint32_t bal[kTcG];
#pragma unroll
                for (int u = 0; u < kTcG; ++u) {
                    bool cand = false;
                    if (valid && u < (int)G.ng) {
                        cand = blk == 0 || !(lb[u] > ms->T[u] * (1.f + 0x1p-20f));
                        if (!cand) sg[u * kSdRowsMax + gr] = __int_as_float(0x7fffffff);
                    }
                    bal[u] = __ballot_sync(0xffffffffu, cand);
                }
                if (it >= 2) mb_wait(pl_empty + buf, ((it >> 1) - 1) & 1);
                if (lane == 0) {
#pragma unroll
                    for (int u = 0; u < kTcG; ++u) ms->cnt[ew][u] = __popc(bal[u]);
                }
                tc_epi_bar();
                uint32_t base = 0;
                uint16_t* pl = pls + buf * kTcMaxPairs;
#pragma unroll
                for (int u = 0; u < kTcG; ++u) {
                    uint32_t before = 0, tot = 0;
#pragma unroll
                    for (int w = 0; w < kTcEpi; ++w) {
                        const uint32_t cw = ms->cnt[w][u];
                        before += w < (int)ew ? cw : 0u;
                        tot += cw;
                    }
                    if ((bal[u] >> lane) & 1u) pl[base + before + __popc(bal[u] & lt)] = (uint16_t)((u << 7) | r);
                    base += tot;
                }
                if (ew == 0 && lane == 0) ms->pl_n[buf] = base;
                if (ew == 0 && lane == 0 && a.census) atomicAdd(a.census, (unsigned long long)base * dim);
                __syncwarp();
                if (lane == 0) mb_arrive(pl_full + buf);
            }
        }
    } else if (warp < (uint32_t)kTcEx) {
        // ---- exact sums of the candidate pairs ----
        uint32_t s = 0, ph = 0, it = 0;
        for (uint32_t i = 0;; ++i) {
            SpGroup G;
            if (!take_group(i, G)) break;
            const uint32_t qb = i & 1, par = i & 1;
            mb_wait(q_full + qb, (i >> 1) & 1);
            const unsigned char* qt = sm + L.q + qb * kTcMaxAtoms * kTcQAtom;
            float* sg = scr + (size_t)par * kTcG * kSdRowsMax;
            const uint32_t nb = (G.n + kTcM - 1) / kTcM;
            for (uint32_t blk = 0; blk < nb; ++blk, ++it) {
                const uint32_t buf = it & 1;
                mb_wait(pl_full + buf, (it >> 1) & 1);
                const uint32_t n = ms->pl_n[buf];
                const uint16_t* pl = pls + buf * kTcMaxPairs;
                const uint32_t nr = (n + 2 * kTcExT - 1) / (2 * kTcExT);
                uint32_t desc[kTcRounds];
                uint64_t acc[kTcRounds];
#pragma unroll
                for (int rr = 0; rr < kTcRounds; ++rr) {
                    const uint32_t p0 = 2 * (tid + kTcExT * rr);
                    const uint32_t d0 = p0 < n ? pl[p0] : 0u, d1 = p0 + 1 < n ? pl[p0 + 1] : d0;
                    desc[rr] = d0 | (d1 << 16);
                    acc[rr] = 0ull;
                }
                for (uint32_t at = 0; at < n_atoms; ++at) {
                    mb_wait(ex_full + s, ph);
                    const unsigned char* slot = sm + L.re + s * kTcAtom;
                    const unsigned char* qa = qt + at * kTcQAtom;
#pragma unroll
                    for (int rr = 0; rr < kTcRounds; ++rr) {
                        if ((uint32_t)rr >= nr) break;
                        const uint32_t r0 = desc[rr] & 127u, u0 = (desc[rr] >> 7) & 15u;
                        const uint32_t r1 = (desc[rr] >> 16) & 127u, u1 = (desc[rr] >> 23) & 15u;
                        const unsigned char* o0p = slot + r0 * 128;
                        const unsigned char* o1p = slot + r1 * 128;
                        const unsigned char* q0p = qa + u0 * 128;
                        const unsigned char* q1p = qa + u1 * 128;
#pragma unroll
                        for (uint32_t c = 0; c < 8; ++c) {
                            const float4 o0 = *reinterpret_cast<const float4*>(o0p + ((c ^ (r0 & 7u)) << 4));
                            const float4 o1 = *reinterpret_cast<const float4*>(o1p + ((c ^ (r1 & 7u)) << 4));
                            const float4 q0 = *reinterpret_cast<const float4*>(q0p + ((c ^ (u0 & 7u)) << 4));
                            const float4 q1 = *reinterpret_cast<const float4*>(q1p + ((c ^ (u1 & 7u)) << 4));
                            acc[rr] = sq_step2p(acc[rr], pk2(o0.x, o1.x), pk2(q0.x, q1.x), a.nz2);
                            acc[rr] = sq_step2p(acc[rr], pk2(o0.y, o1.y), pk2(q0.y, q1.y), a.nz2);
                            acc[rr] = sq_step2p(acc[rr], pk2(o0.z, o1.z), pk2(q0.z, q1.z), a.nz2);
                            acc[rr] = sq_step2p(acc[rr], pk2(o0.w, o1.w), pk2(q0.w, q1.w), a.nz2);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) mb_arrive(ex_empty + s);
                    if (++s == (uint32_t)kTcES) {
                        s = 0;
                        ph ^= 1;
                    }
                }
#pragma unroll
                for (int rr = 0; rr < kTcRounds; ++rr) {
                    if ((uint32_t)rr >= nr) break;
                    const uint32_t p0 = 2 * (tid + kTcExT * rr);
                    const uint32_t r0 = desc[rr] & 127u, u0 = (desc[rr] >> 7) & 15u;
                    const uint32_t r1 = (desc[rr] >> 16) & 127u, u1 = (desc[rr] >> 23) & 15u;
                    if (p0 < n) sg[u0 * kSdRowsMax + blk * kTcM + r0] = lo_f(acc[rr]);
                    if (p0 + 1 < n) sg[u1 * kSdRowsMax + blk * kTcM + r1] = hi_f(acc[rr]);
                }
                __syncwarp();
                if (lane == 0) mb_arrive(pl_empty + buf);
            }
            __threadfence_block();  // the group's sums are visible to the selection warps
            __syncwarp();
            if (lane == 0) {
                mb_arrive(g_done + par);
                mb_arrive(q_empty + qb);
            }
        }
    } else {
        // ---- selection ----
        const uint32_t sw = warp - kTcWSel;
        uint64_t* keys = reinterpret_cast<uint64_t*>(sm + L.keys) + sw * kSdSmall;
        uint32_t* sh = reinterpret_cast<uint32_t*>(sm + L.shist) + sw * 256;
        for (uint32_t i = 0;; ++i) {
            SpGroup G;
            if (!take_group(i, G)) break;
            const uint32_t par = i & 1;
            mb_wait(g_done + par, (i >> 1) & 1);
            const float* sg = scr + (size_t)par * kTcG * kSdRowsMax;
            for (uint32_t u = sw; u < G.ng; u += kTcSel)
                sd_finish_query(a, G.qs[u], sg + (size_t)u * kSdRowsMax, G.n, G.start, keys, sh);
            __syncwarp();
            if (lane == 0) mb_arrive(s_free + par);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kTcWMma) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kTcTmemCols));
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

bool seed_tc_ok(uint32_t dim, uint32_t K) {
    return dim % 32 == 0 && dim >= 32 && dim <= 32u * kTcMaxAtoms && K <= (uint32_t)kSdSmall;
}

size_t seed_tc_scratch_bytes(uint32_t n_sm) { return (size_t)n_sm * 2 * kTcG * kSdRowsMax * sizeof(float); }

cudaError_t launch_seed_tc(const SeedListArgs& a, const CUtensorMap& tmap128, const float* full_norms, float* scratch,
                           uint32_t max_groups, cudaStream_t s, uint32_t* work) {
    if (a.n_lists == 0 || max_groups == 0) return cudaSuccess;
    if (!work || !scratch || !full_norms || !seed_tc_ok(a.dim, a.K) || a.S > (uint32_t)kSdRowsMax)
        return cudaErrorInvalidValue;
    int dev = 0, n_sm = 0;
    DADE_CUDA_TRY(cudaGetDevice(&dev));
    DADE_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    const uint32_t smem = tc_layout().total;
    DADE_CUDA_TRY(cudaFuncSetAttribute(seed_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    DADE_CUDA_TRY(cudaMemsetAsync(work, 0, 4, s));
    if (a.order) seed_order_kernel<<<1, 1024, 0, s>>>(a, a.order);
    seed_tc_kernel<<<std::min<uint32_t>(max_groups, (uint32_t)n_sm), kTcThreads, smem, s>>>(a, tmap128, full_norms,
                                                                                          scratch, work);
    return cudaGetLastError();
}

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

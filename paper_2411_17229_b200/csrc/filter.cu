// Streaming first-slice DCO filter (the bulk of the IVF-DADE / flat DADE scan).
//
// Work is per WARP: a warp pulls a work item (an IVF posting-list row piece or a
// flat row block x up to 32 queries) from a global counter, keeps the item's
// queries' dense dims [0, d0) in its own shared-memory slice, and streams the
// item's 32-row tiles through a private 2-slot TMA ring. No CTA barrier is ever
// taken, so warps drift freely across items (one warp's item prologue overlaps
// the other warps' tiles). Per tile:
//   1. tensor cores (mma.sync m16n8k8 TF32, ldmatrix A fragments from the
//      128B-swizzled box) give, for all 32 x 32 pairs,
//          acc = o.q - h_o - c_q,   h_o = (1 - delta)|o|^2 / 2,
//                                   c_q = ((1 - delta)|q|^2 - thr_q) / 2,
//      the two constants entering as one extra k-step (split hi + lo so the
//      TF32 operand truncation stays below 2^-20 relative);
//   2. acc < 0  <=>  (1 - delta)(|o|^2 + |q|^2) - 2 o.q > thr_q: the pair is
//      pruned for sure (rigorous bound, kTcDeltaF; the reference rejects it at
//      the first checkpoint, proj/src/estimator.cpp:46-58); the keep mask is
//      the sign bits;
//   3. every kept pair gets the exact sequential fp32 prefix from shared memory
//      and the exact checkpoint test; survivors are appended to a global
//      worklist that advance_survivors_kernel continues from d0.
// The radius of each query is read from r_global at the item start and fixed
// for the launch (the host tightens it between passes).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

constexpr int kFRows = 32;          // rows per tile
constexpr int kFQ = 32;             // queries per work item
// q_res: [d0][32] fp32, query column XOR-swizzled by (k & 3) << 3 so that both
// the B-fragment loads (4 k-rows x 8 queries) and the per-lane prefix loads
// (one k-row, 32 queries) are bank-conflict free without padding.
__device__ __forceinline__ int qsw(int k, int j) { return k * 32 + (j ^ ((k & 3) << 3)); }
constexpr int kFSlots = 2;          // private ring depth per warp (per dense box)
constexpr int kFWarps = 8;
constexpr int kFThreads = kFWarps * 32;
constexpr int kFList = 128;         // kept-pair list per warp per round
constexpr float kTcDeltaF = 2.6e-3f;  // same bound as scan.cu's kTcDelta

__device__ __forceinline__ uint32_t smem_u32f(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init_f(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32f(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx_f(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32f(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_f(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAITF_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAITF_%=;\n"
        "}\n" ::"r"(smem_u32f(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma2d_f(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_u32f(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32f(bar))
        : "memory");
}
__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}
__device__ __forceinline__ void mma_tf32_f(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                           uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// value the tensor core sees for an fp32 operand read as TF32 (low 13 mantissa bits ignored)
__device__ __forceinline__ float tf32_trunc(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// Exact sequential fp32 prefix over the dense dims for G kept pairs per lane
// (meta = row | query << 8), G independent chains interleaved for ILP; each
// chain is the reference's accumulation order (proj/src/estimator.cpp:36-44).
template <int G>
__device__ __forceinline__ void prefix_chains(const float* box0, int c_dense, uint32_t d0, const float* q_res,
                                              const uint32_t (&meta)[4], float (&x)[4]) {
    for (int c = 0; c < c_dense; ++c) {
        const float* b = box0 + (size_t)c * kFRows * kBox;
        const float* qq = q_res + (size_t)c * kBox * 32;  // k-rows of box c (k0 = 32 c: k & 3 unchanged)
        const int wc = min(kBox, (int)d0 - c * kBox);
        const float* rb[G];
        int sw[G], qj[G];
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const uint32_t row = meta[i] & 0xffu;
            qj[i] = (int)(meta[i] >> 8);
            rb[i] = b + row * kBox;
            sw[i] = (int)(row & 7);
        }
#pragma unroll 2
        for (int k = 0; k < wc; k += 4) {
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const float4 o4 = *reinterpret_cast<const float4*>(rb[i] + ((((k >> 2) ^ sw[i])) << 2));
                const float* qk = qq + k * 32;
                x[i] = sq_step(x[i], o4.x, qk[0 * 32 + (qj[i] ^ 0)]);
                x[i] = sq_step(x[i], o4.y, qk[1 * 32 + (qj[i] ^ 8)]);
                x[i] = sq_step(x[i], o4.z, qk[2 * 32 + (qj[i] ^ 16)]);
                x[i] = sq_step(x[i], o4.w, qk[3 * 32 + (qj[i] ^ 24)]);
            }
        }
    }
}

// Shared memory: the boxes of every warp first (1024-aligned 4 KB boxes), then
// each warp's query slice and small per-item tables.
struct FLayout {
    size_t boxes, warp_base, warp_bytes, q_res, thr, cneg, qidx, slot, list_meta, bars, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline FLayout f_layout(int d0, int c_dense) {
    FLayout L;
    L.boxes = 0;
    L.warp_base = (size_t)kFWarps * kFSlots * c_dense * kFRows * kBox * 4;
    size_t off = 0;  // within a warp's block
    L.q_res = off; off = al16(off + sizeof(float) * (size_t)d0 * 32);
    L.thr = off; off = al16(off + sizeof(float) * kFQ);
    L.cneg = off; off = al16(off + sizeof(float2) * kFQ);
    L.qidx = off; off = al16(off + sizeof(uint32_t) * kFQ);
    L.slot = off; off = al16(off + sizeof(uint32_t) * kFQ);
    L.list_meta = off; off = al16(off + sizeof(uint32_t) * kFList);
    L.bars = off; off = al16(off + sizeof(uint64_t) * kFSlots);
    L.warp_bytes = off;
    L.total = L.warp_base + (size_t)kFWarps * L.warp_bytes + 1024;
    return L;
}

__global__ void __launch_bounds__(kFThreads, 2)
dco_filter_kernel(const FilterArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ unsigned char fsmem_raw[];
    unsigned char* sm = fsmem_raw + ((1024u - (smem_u32f(fsmem_raw) & 1023u)) & 1023u);
    const int c_dense = a.c_dense;
    const uint32_t d0 = a.d0;
    const FLayout L = f_layout((int)d0, c_dense);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* wb = sm + L.warp_base + (size_t)warp * L.warp_bytes;
    float* q_res = reinterpret_cast<float*>(wb + L.q_res);      // [d0][32], swizzled (qsw)
    float* thr_s = reinterpret_cast<float*>(wb + L.thr);        // [32]
    float2* cneg_s = reinterpret_cast<float2*>(wb + L.cneg);    // [32] (-c hi, -c lo)
    uint32_t* qidx_s = reinterpret_cast<uint32_t*>(wb + L.qidx);
    uint32_t* slot_s = reinterpret_cast<uint32_t*>(wb + L.slot);
    uint32_t* lmeta = reinterpret_cast<uint32_t*>(wb + L.list_meta);
    uint64_t* mybar = reinterpret_cast<uint64_t*>(wb + L.bars);
    float* myboxes = reinterpret_cast<float*>(sm + L.boxes) + (size_t)warp * kFSlots * c_dense * kFRows * kBox;

    if (lane == 0) {
        for (int i = 0; i < kFSlots; ++i) mbar_init_f(mybar + i, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    const uint32_t dim = a.dim;
    const int g = lane >> 2, tq = lane & 3;
    const int smi = lane >> 3, rr = lane & 7;  // ldmatrix addressing
    unsigned long long st_dco = 0, st_dims = 0, st_bytes = 0, st_surv = 0, st_viol = 0;
    unsigned long long cs_tiles = 0, cs_ktiles = 0, cs_kept = 0;  // census (lane 0)
    uint32_t k_iter = 0;  // this warp's running ring position (mbarrier phases persist across items)
    const uint32_t base = a.items ? (a.range_hi ? a.range_lo : a.item_base ? *a.item_base : 0u) : 0u;
    const uint32_t end = a.items ? (a.range_hi ? min(a.range_hi, *a.n_items) : *a.n_items)
                                 : a.flat_qchunks * ((a.flat_rows + a.flat_block - 1) / a.flat_block);
    auto box = [&](uint32_t slot, int c) { return myboxes + ((size_t)slot * c_dense + c) * kFRows * kBox; };

    for (;;) {  // persistent: each warp pulls work items from a global counter
        uint32_t item = 0;
        if (lane == 0) item = base + atomicAdd(a.item_counter, 1u);
        item = __shfl_sync(0xffffffffu, item, 0);
        if (item >= end) break;

        // ---- work item -------------------------------------------------------------
        uint32_t row_start, row_count, qcount, bq = 0;
        if (a.items != nullptr) {
            const WorkItem wi = a.items[item];
            const uint32_t piece = wi.bucket_count >> 16;
            if (piece < a.piece_lo || piece >= a.piece_hi) continue;  // another sub-pass's rows
            row_start = wi.row_start;
            row_count = wi.row_count;
            qcount = wi.bucket_count & 0xffffu;
            bq = wi.bucket_start;
        } else {
            const uint32_t rb = item / a.flat_qchunks, qc = item % a.flat_qchunks;
            row_start = rb * a.flat_block;
            row_count = min(a.flat_block, a.flat_rows - row_start);
            qcount = min((uint32_t)kFQ, a.flat_nq - qc * kFQ);
            bq = qc * kFQ;
        }
        const uint32_t n_tiles = (row_count + kFRows - 1) / kFRows;
        auto issue = [&](uint32_t t, uint32_t slot) {  // lane 0 only
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_arrive_tx_f(mybar + slot, (uint32_t)c_dense * kFRows * kBox * 4);
            for (int c = 0; c < c_dense; ++c)
                tma2d_f(box(slot, c), &tmap, c * kBox, (int)(row_start + t * kFRows), mybar + slot);
        };
        __syncwarp();  // previous item's smem reads done (q_res, boxes) before refilling
        if (lane == 0) {  // first two tiles in flight while the queries load
            if (n_tiles > 0) issue(0, k_iter % kFSlots);
            if (n_tiles > 1) issue(1, (k_iter + 1) % kFSlots);
        }
        // lane j = query j: dense dims (transposed into q_res), its norm, threshold
        {
            uint32_t qi = 0, sl = 0;
            float th = -__int_as_float(0x7f800000);  // padding queries: never kept
            float nq = 0.f;
            if ((uint32_t)lane < qcount) {
                if (a.items != nullptr) {
                    qi = a.bucket_q[bq + lane];
                    sl = a.bucket_slot[bq + lane];
                } else {
                    qi = bq + lane;
                    sl = row_start / a.flat_block;
                }
                th = prune_threshold(a.coeff0, __uint_as_float(a.r_global[qi]));
                const float* qrow = a.queries + (size_t)qi * dim;
                for (uint32_t k = 0; k < d0; k += 4) {
                    const float4 v = __ldg(reinterpret_cast<const float4*>(qrow + k));
                    q_res[qsw(k + 0, lane)] = v.x;
                    q_res[qsw(k + 1, lane)] = v.y;
                    q_res[qsw(k + 2, lane)] = v.z;
                    q_res[qsw(k + 3, lane)] = v.w;
                    nq = fmaf(v.x, v.x, nq);
                    nq = fmaf(v.y, v.y, nq);
                    nq = fmaf(v.z, v.z, nq);
                    nq = fmaf(v.w, v.w, nq);
                }
            } else {
                for (uint32_t k = 0; k < d0; ++k) q_res[qsw(k, lane)] = 0.f;
            }
            // -c = (thr - (1 - delta)|q|^2) / 2: +inf radius -> -c = +inf (keep all);
            // padding (thr = -inf) -> -c = -inf (prune all)
            const float nc = 0.5f * (th - (1.f - kTcDeltaF) * nq);
            const float nc_hi = tf32_trunc(nc);
            const float nc_lo = isfinite(nc) ? nc - nc_hi : 0.f;
            cneg_s[lane] = make_float2(nc_hi, nc_lo);
            thr_s[lane] = th;
            qidx_s[lane] = qi;
            slot_s[lane] = sl;
        }
        __syncwarp();
        // extra k-step B fragments: rows k = 0, 1 -> 1 (times -h_o hi/lo);
        // k = 2, 3 -> -c hi/lo of query (nt * 8 + g); k = 4..7 -> 0
        uint32_t baug[4];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) {
            const float2 cn = cneg_s[nt * 8 + g];
            baug[nt] = __float_as_uint(tq < 2 ? 1.f : (tq == 2 ? cn.x : cn.y));
        }

        // ---- the item's tiles through this warp's ring ----------------------------------
        for (uint32_t t = 0; t < n_tiles; ++t, ++k_iter) {
            const uint32_t slot = k_iter % kFSlots;
            const uint32_t tb = t * kFRows, nrows = min((uint32_t)kFRows, row_count - tb);
            mbar_wait_f(mybar + slot, (k_iter / kFSlots) & 1);
            st_dco += (uint64_t)nrows * qcount;
            st_bytes += 4ull * d0 * nrows;

            // -h_o (hi, lo) of rows g, g + 8, g + 16, g + 24 as the extra k-step's A fragments
            const float ho = 0.5f * (1.f - kTcDeltaF) * __ldg(a.row_norms + row_start + tb + lane);
            uint32_t aaug[2][2];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const float hv = __shfl_sync(0xffffffffu, ho, mt * 16 + h * 8 + g);
                    const float hhi = tf32_trunc(hv);
                    aaug[mt][h] = __float_as_uint(tq == 0 ? -hhi : (tq == 1 ? -(hv - hhi) : 1.f));
                }

            float d[2][4][4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                    for (int v = 0; v < 4; ++v) d[mt][nt][v] = 0.f;
            for (int c = 0; c < c_dense; ++c) {
                const uint32_t bb = smem_u32f(box(slot, c));
                const float* qc = q_res + (c * kBox + tq) * 32 + g;  // k = 32 c + ks + tq (+4): k & 3 = tq
                const int wc = min(kBox, (int)d0 - c * kBox);
#pragma unroll 4
                for (int ks = 0; ks < wc; ks += 8) {
                    uint32_t A[2][4];
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt) {
                        const uint32_t row = mt * 16 + (smi & 1) * 8 + rr;
                        const uint32_t chunk = (ks >> 2) + (smi >> 1);
                        ldsm4(bb + row * (kBox * 4) + ((chunk ^ (row & 7)) << 4), A[mt][0], A[mt][1], A[mt][2], A[mt][3]);
                    }
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt) {
                        const int col = (nt ^ tq) * 8;  // (nt * 8 + g) ^ (tq << 3)
                        const uint32_t b0 = __float_as_uint(qc[ks * 32 + col]);
                        const uint32_t b1 = __float_as_uint(qc[(ks + 4) * 32 + col]);
#pragma unroll
                        for (int mt = 0; mt < 2; ++mt) mma_tf32_f(d[mt][nt], A[mt][0], A[mt][1], A[mt][2], A[mt][3], b0, b1);
                    }
                }
            }
#pragma unroll
            for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                for (int mt = 0; mt < 2; ++mt) mma_tf32_f(d[mt][nt], aaug[mt][0], aaug[mt][1], 0u, 0u, baug[nt], 0u);
            // keep = sign bit clear; bit = ((mt * 2 + h) * 4 + nt) * 2 + cq
            uint32_t neg = 0;
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                        for (int cq = 0; cq < 2; ++cq)
                            neg |= (__float_as_uint(d[mt][nt][h * 2 + cq]) >> 31) << (((mt * 2 + h) * 4 + nt) * 2 + cq);
            uint32_t keep = ~neg;
            // rows past the item (next list's rows or TMA zero fill) are masked;
            // padding queries have -c = -inf (always negative)
            if (nrows < (uint32_t)kFRows) {
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if ((uint32_t)(mt * 16 + h * 8 + g) >= nrows) keep &= ~(0xffu << ((mt * 2 + h) * 8));
            }
            if (a.debug == 1) {  // every prune must agree with the exact prefix (test hook)
                for (int b = 0; b < 32; ++b) {
                    const int cq = b & 1, nt = (b >> 1) & 3, h = (b >> 3) & 1, mt = b >> 4;
                    const uint32_t row = mt * 16 + h * 8 + g, j = nt * 8 + 2 * tq + cq;
                    if (((keep >> b) & 1u) || row >= nrows || j >= qcount) continue;
                    const uint32_t m1[4] = {row | (j << 8), 0u, 0u, 0u};
                    float x1[4] = {0.f, 0.f, 0.f, 0.f};
                    prefix_chains<1>(box(slot, 0), c_dense, d0, q_res, m1, x1);
                    if (!(x1[0] > thr_s[j])) ++st_viol;
                }
            }
            const uint32_t total_pairs = qcount * nrows;
            unsigned long long pruned = total_pairs;
            if (a.census) {
                const uint32_t kc = __reduce_add_sync(0xffffffffu, __popc(keep));
                cs_tiles += 1;
                cs_ktiles += kc ? 1 : 0;
                cs_kept += kc;
            }
            // ---- exact prefix for kept pairs, survivors to the worklist --------------
            while (__any_sync(0xffffffffu, keep != 0)) {
                const uint32_t mine = __popc(keep);
                uint32_t incl = mine;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += y;
                }
                uint32_t pos = incl - mine;
                const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
                uint32_t bits = keep;
                while (bits && pos < (uint32_t)kFList) {
                    const int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int cq = b & 1, nt = (b >> 1) & 3, h = (b >> 3) & 1, mt = b >> 4;
                    lmeta[pos] = (uint32_t)(mt * 16 + h * 8 + g) | ((uint32_t)(nt * 8 + 2 * tq + cq) << 8);
                    keep &= ~(1u << b);
                    ++pos;
                }
                __syncwarp();
                const uint32_t n = min(tot, (uint32_t)kFList);
                pruned -= n;
                // up to 4 kept pairs per lane, their sequential chains interleaved
                const uint32_t ng = (n + 31) >> 5;
                uint32_t meta[4];
                float x[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint32_t e = (uint32_t)i * 32 + lane;
                    meta[i] = e < n ? lmeta[e] : 0u;
                }
                const float* sb = box(slot, 0);
                if (ng > 2) prefix_chains<4>(sb, c_dense, d0, q_res, meta, x);
                else if (ng > 1) prefix_chains<2>(sb, c_dense, d0, q_res, meta, x);
                else prefix_chains<1>(sb, c_dense, d0, q_res, meta, x);
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if ((uint32_t)i >= ng) break;
                    const uint32_t e = (uint32_t)i * 32 + lane;
                    const uint32_t j = meta[i] >> 8;
                    const bool surv = e < n && !(x[i] > thr_s[j]);
                    if (e < n && !surv) st_dims += d0;
                    const uint32_t bal = __ballot_sync(0xffffffffu, surv);
                    if (bal) {
                        uint32_t sbase = 0;
                        if (lane == 0) sbase = atomicAdd(a.surv_count, __popc(bal));
                        sbase = __shfl_sync(0xffffffffu, sbase, 0);
                        if (surv) {
                            const uint32_t p = sbase + __popc(bal & ((1u << lane) - 1u));
                            if (p < a.surv_cap) {
                                Survivor v;
                                v.q = qidx_s[j];
                                v.row = row_start + tb + (meta[i] & 0xffu);
                                v.acc = x[i];
                                v.slot = slot_s[j];
                                a.surv[p] = v;
                            }
                        }
                        st_surv += __popc(bal);  // every lane adds: divided by 32 at the end
                    }
                }
                __syncwarp();
            }
            if (lane == 0) st_dims += pruned * d0;  // filter-pruned pairs end at the first checkpoint
            // refill this slot with the tile after next
            __syncwarp();
            if (lane == 0 && t + kFSlots < n_tiles) issue(t + kFSlots, slot);
        }
    }  // items

    // ---- counters ----------------------------------------------------------------
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        st_dco += __shfl_xor_sync(0xffffffffu, st_dco, off);
        st_dims += __shfl_xor_sync(0xffffffffu, st_dims, off);
        st_bytes += __shfl_xor_sync(0xffffffffu, st_bytes, off);
        st_viol += __shfl_xor_sync(0xffffffffu, st_viol, off);
    }
    if (lane == 0 && a.counters) {
        atomicAdd(a.counters + 0, st_dco / 32);  // every lane added the same per-tile count
        atomicAdd(a.counters + 1, st_dims);
        atomicAdd(a.counters + 2, st_bytes / 32 + 16ull * (st_surv / 32));
        if (st_viol) atomicAdd(a.counters + 3, st_viol);
    }
    if (lane == 0 && a.census) {
        atomicAdd(a.census + 0, cs_ktiles | (cs_tiles << 32));  // tiles with kept pairs | all tiles << 32
        atomicAdd(a.census + 1, cs_kept);
    }
}

}  // namespace

size_t filter_smem_bytes(int d0, int c_dense) { return f_layout(d0, c_dense).total; }

cudaError_t launch_filter(const FilterArgs& a, const CUtensorMap& tmap, uint32_t grid, cudaStream_t s) {
    if (grid == 0) return cudaSuccess;
    const size_t smem = filter_smem_bytes((int)a.d0, a.c_dense);
    DADE_CUDA_TRY(cudaFuncSetAttribute(dco_filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dco_filter_kernel<<<grid, kFThreads, smem, s>>>(a, tmap);
    return cudaGetLastError();
}

}  // namespace dade_gpu

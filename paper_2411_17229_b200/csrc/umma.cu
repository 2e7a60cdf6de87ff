// Streaming first-slice DCO filter on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM).
//
// One persistent CTA per SM. Work item = (posting-list row piece of <= 1024
// rows, up to 256 of the queries probing that list). For every 128-row tile of
// the piece, ONE tcgen05.mma chain computes, for all 128 x N (row, query) pairs,
//
//     acc = o.q - h_o - c_q,   h_o = (1 - delta)|o|^2 / 2,
//                              c_q = ((1 - delta)|q|^2 - thr_q) / 2
//
// over the dense dims [0, d0) (TF32 operands straight from the fp32 rows: the
// tile is TMA-loaded 128B-swizzled, K-major) plus one extra K=8 step whose
// operands are (-h_o hi, -h_o lo, 1, 1) per row (a precomputed [rows][8] array,
// TMA-loaded 32B-swizzled with the tile) and (1, 1, -c_q hi, -c_q lo) per query
// (hi + lo splits keep the TF32 truncation below 2^-20 relative). The pair is
// pruned for sure iff acc < 0, i.e.
// (1 - delta)(|o|^2 + |q|^2) - 2 o.q > thr_q: the same rigorous bound as the
// mma.sync filter (filter.cu); the reference would reject the
// pair at its first checkpoint (proj/src/estimator.cpp:46-58).
//
// Roles (warp-specialised, mbarrier pipelines, no CTA barrier after setup):
//   warp 16     stager: pulls items from the global counter and stages each
//               item's queries (B operand, cp.async into the 128B-swizzled
//               K-major layout), -c (B_aug) and query ids into one of two item
//               buffers, running up to one item ahead of the MMAs;
//   warp 17     TMA: loads 128-row tiles (+ their K=8 row operand) into a
//               4-stage ring, running ahead across item boundaries;
//   warp 18     MMA: one elected lane issues the tcgen05.mma chain of each tile
//               into one of two TMEM accumulator buffers (2 x 256 columns);
//   warps 0-15  epilogue: warp w reads TMEM lanes 32 (w % 4).. (its rows) and
//               column quarter w / 4, two 32-column tcgen05.ld in flight; a
//               chunk whose values are all negative is pruned whole (the
//               common case); otherwise every kept (row, query) pair is
//               appended to the survivor worklist, whose kernel runs the exact
//               sequential fp32 accumulation from dim 0
//               (advance_survivors_kernel).
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"
#include "tc.cuh"

namespace dade_gpu {

namespace {

constexpr int kUM = 128;            // rows per tile (MMA M, TMEM lanes)
constexpr int kUQ = 256;            // max queries per item (MMA N)
constexpr int kUEpiWarps = 16;
constexpr int kUStager = kUEpiWarps;      // warp index
constexpr int kUTma = kUEpiWarps + 1;     // warp index
constexpr int kUMma = kUEpiWarps + 2;     // warp index
constexpr int kUThreads = (kUEpiWarps + 3) * 32;
constexpr int kUNB = 2;                   // item (B) buffers
constexpr uint32_t kUTmemCols = 512;      // 2 accumulator buffers x 256 columns
constexpr float kUDelta = 2.6e-3f;        // same bound as filter.cu / scan.cu
constexpr uint32_t kUSentinel = 0xffffffffu;

struct UItem {  // published by the stager in item buffer ib
    uint32_t row_start, row_count, qcount, ncols;
};
struct UMeta {  // per accumulator buffer, published by the MMA warp
    uint32_t row0, nrows, qcount, ncols, ib, last, pad0, pad1;
};

struct ULayout {
    size_t a, b, a_aug, b_aug, qidx, slot, item, meta, bars, tmem_slot, total;
    int stages;
};

__host__ __device__ inline ULayout u_layout(int c_dense) {
    ULayout L;
    L.stages = c_dense == 1 ? 4 : 2;
    size_t off = 0;
    L.a = off; off += (size_t)L.stages * c_dense * kUM * 128;          // 1024-aligned atoms
    L.b = off; off += (size_t)kUNB * c_dense * kUQ * 128;
    L.a_aug = off; off += (size_t)L.stages * kUM * 32;                 // per stage, TMA (SW32)
    L.b_aug = off; off += (size_t)kUNB * kUQ * 32;
    L.qidx = off; off += (size_t)kUNB * kUQ * 4;
    L.slot = off; off += (size_t)kUNB * kUQ * 4;
    L.item = off; off += kUNB * sizeof(UItem);
    L.meta = off; off += 2 * sizeof(UMeta);
    L.bars = off; off += 8 * 24;
    L.tmem_slot = off; off += 16;
    L.total = off + 1024;
    return L;
}

__global__ void __launch_bounds__(kUThreads, 1)
dco_filter_umma_kernel(const FilterArgs a, const __grid_constant__ CUtensorMap tmap,
                       const __grid_constant__ CUtensorMap tmap_aug) {
    extern __shared__ unsigned char usmem_raw[];
    unsigned char* sm = usmem_raw + ((1024u - (su32(usmem_raw) & 1023u)) & 1023u);
    const int c_dense = a.c_dense;
    const ULayout L = u_layout(c_dense);
    const int S = L.stages;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
    uint64_t* afull = bars;            // [S]   TMA bytes landed
    uint64_t* aempty = bars + 4;       // [S]   MMAs reading the stage done (commit)
    uint64_t* accfull = bars + 8;      // [2]   MMAs of the tile done (commit)
    uint64_t* accempty = bars + 10;    // [2]   every epilogue warp done with the buffer
    uint64_t* metafull = bars + 12;    // [2]   tile metadata written (MMA warp)
    uint64_t* bready = bars + 14;      // [NB]  item staged (stager)
    uint64_t* bfree = bars + 16;       // [NB]  item's MMAs done (commit) + epilogue done with its ids
    UItem* items = reinterpret_cast<UItem*>(sm + L.item);
    UMeta* meta = reinterpret_cast<UMeta*>(sm + L.meta);
    uint32_t* qidx_s = reinterpret_cast<uint32_t*>(sm + L.qidx);
    uint32_t* slot_s = reinterpret_cast<uint32_t*>(sm + L.slot);
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sm + L.tmem_slot);

    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) {
            mb_init(afull + i, 1);
            mb_init(aempty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mb_init(accfull + i, 1);
            mb_init(accempty + i, kUEpiWarps);
            mb_init(metafull + i, 1);
        }
        for (int i = 0; i < kUNB; ++i) {
            mb_init(bready + i, 1);
            mb_init(bfree + i, 1 + kUEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == kUMma) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                     "r"(kUTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t d0 = a.d0;

    if (warp == kUStager) {
        // ============================ stager ============================
        const uint32_t base = a.range_hi ? a.range_lo : a.item_base ? *a.item_base : 0u;
        const uint32_t end = a.range_hi ? min(a.range_hi, *a.n_items) : *a.n_items;
        long long tp_stage = 0, tp_items = 0;
        for (uint32_t k = 0;; ++k) {
            const uint32_t ib = k % kUNB;
            // next item of this pass (other pieces are another sub-pass's)
            WorkItem wi{};
            bool have = false;
            for (;;) {
                uint32_t item = 0;
                if (lane == 0) item = base + atomicAdd(a.item_counter, 1u);
                item = __shfl_sync(0xffffffffu, item, 0);
                if (item >= end) break;
                wi = a.items[item];
                const uint32_t piece = wi.bucket_count >> 16;
                const bool ok = (a.b0_items && item < *a.b0_items) ? piece >= a.b0_piece_lo
                                                                   : (piece >= a.piece_lo && piece < a.piece_hi);
                if (ok) {
                    have = true;
                    break;
                }
            }
            if (k >= (uint32_t)kUNB) mb_wait(bfree + ib, ((k / kUNB) - 1) & 1);
            if (!have) {
                if (lane == 0) {
                    items[ib] = UItem{kUSentinel, 0, 0, 0};
                    mb_arrive(bready + ib);
                }
                break;
            }
            const long long t0 = clock64();
            ++tp_items;
            const uint32_t qcount = wi.bucket_count & 0xffffu;
            const uint32_t ncols = max(32u, (qcount + 31) & ~31u);
            unsigned char* bb = sm + L.b + (size_t)ib * c_dense * kUQ * 128;
            float* baug = reinterpret_cast<float*>(sm + L.b_aug + (size_t)ib * kUQ * 32);
            // loads first (8 independent chains per lane), then the smem writes / cp.async
            constexpr int kPer = kUQ / 32;
            uint32_t qv[kPer], sv[kPer];
            float rv[kPer], nv[kPer];
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const uint32_t j = lane + 32u * u;
                qv[u] = j < qcount ? a.bucket_q[wi.bucket_start + j] : 0u;
                sv[u] = j < qcount ? a.bucket_slot[wi.bucket_start + j] : 0u;
            }
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const uint32_t j = lane + 32u * u;
                rv[u] = j < qcount ? __uint_as_float(a.r_global[qv[u]]) : 0.f;
                nv[u] = j < qcount ? a.q_norms[qv[u]] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < kPer; ++u) {
                const uint32_t j = lane + 32u * u;
                if (j >= ncols) break;
                float nc_hi = -__int_as_float(0x7f800000), nc_lo = 0.f;  // padding: -c = -inf (pruned)
                if (j < qcount) {
                    qidx_s[ib * kUQ + j] = qv[u];
                    slot_s[ib * kUQ + j] = sv[u];
                    const float th = prune_threshold(a.coeff0, rv[u]);
                    const float nc = 0.5f * (th - (1.f - kUDelta) * nv[u]);
                    nc_hi = tf32_hi(nc);
                    nc_lo = isfinite(nc) ? nc - nc_hi : 0.f;
                    const float* qrow = a.queries + (size_t)qv[u] * a.dim;
                    for (int c = 0; c < c_dense; ++c) {
                        unsigned char* brow = bb + (size_t)c * kUQ * 128 + (size_t)j * 128;
                        const int wc4 = min(8, (int)(d0 - c * 32) / 4);
                        for (int ch = 0; ch < 8; ++ch) {
                            unsigned char* dst = brow + ((ch ^ (int)(j & 7)) << 4);
                            if (ch < wc4) cp16(dst, qrow + c * 32 + ch * 4);
                            else *reinterpret_cast<float4*>(dst) = make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                    }
                } else {
                    for (int c = 0; c < c_dense; ++c) {
                        unsigned char* brow = bb + (size_t)c * kUQ * 128 + (size_t)j * 128;
                        for (int ch = 0; ch < 8; ++ch)
                            *reinterpret_cast<float4*>(brow + ch * 16) = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
                for (uint32_t kk = 0; kk < 8; ++kk)
                    baug[sw32_off(j, kk) / 4] = kk < 2 ? 1.f : kk == 2 ? nc_hi : kk == 3 ? nc_lo : 0.f;
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                items[ib] = UItem{wi.row_start, wi.row_count, qcount, ncols};
                mb_arrive(bready + ib);
            }
            tp_stage += clock64() - t0;
        }
        if (lane == 0 && a.census) {
            atomicAdd(a.census + 0, (unsigned long long)tp_items);
            atomicAdd(a.census + 1, (unsigned long long)tp_stage);
        }
    } else if (warp == kUTma) {
        // ============================ TMA ============================
        const uint32_t tile_bytes = (uint32_t)c_dense * kUM * 128 + kUM * 32;
        uint32_t a_issue = 0;
        long long tp_aempty = 0;
        for (uint32_t k = 0;; ++k) {
            mb_wait(bready + (k % kUNB), (k / kUNB) & 1);
            const UItem it = items[k % kUNB];
            if (it.row_start == kUSentinel) break;
            const uint32_t n_tiles = (it.row_count + kUM - 1) / kUM;
            for (uint32_t t = 0; t < n_tiles; ++t, ++a_issue) {
                const uint32_t s = a_issue % S;
                const long long t0 = clock64();
                if (a_issue >= (uint32_t)S) mb_wait(aempty + s, ((a_issue / S) - 1) & 1);
                tp_aempty += clock64() - t0;
                if (lane == 0) {
                    mb_arrive_tx(afull + s, tile_bytes);
                    for (int c = 0; c < c_dense; ++c)
                        tma2d_u(sm + L.a + ((size_t)s * c_dense + c) * kUM * 128, &tmap, c * 32,
                                (int)(it.row_start + t * kUM), afull + s);
                    tma2d_u(sm + L.a_aug + (size_t)s * kUM * 32, &tmap_aug, 0, (int)(it.row_start + t * kUM),
                            afull + s);
                }
                __syncwarp();
            }
        }
        if (lane == 0 && a.census) atomicAdd(a.census + 7, (unsigned long long)tp_aempty);
    } else if (warp == kUMma) {
        // ============================ MMA ============================
        unsigned long long st_dco = 0, st_bytes = 0;
        long long tp_bready = 0, tp_accempty = 0, tp_afull = 0;
        uint32_t a_use = 0, acc_it = 0;
        for (uint32_t k = 0;; ++k) {
            const uint32_t ib = k % kUNB;
            {
                const long long t0 = clock64();
                mb_wait(bready + ib, (k / kUNB) & 1);
                tp_bready += clock64() - t0;
            }
            const UItem it = items[ib];
            if (it.row_start == kUSentinel) break;
            const uint32_t n_tiles = (it.row_count + kUM - 1) / kUM;
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((it.ncols >> 3) << 17) |
                                   ((uint32_t)(kUM >> 4) << 24);
            const unsigned char* bb = sm + L.b + (size_t)ib * c_dense * kUQ * 128;
            const float* baug = reinterpret_cast<const float*>(sm + L.b_aug + (size_t)ib * kUQ * 32);
            for (uint32_t t = 0; t < n_tiles; ++t) {
                const uint32_t s = a_use % S;
                const uint32_t b = acc_it & 1;
                long long t0 = clock64();
                if (acc_it >= 2) mb_wait(accempty + b, ((acc_it >> 1) - 1) & 1);
                tp_accempty += clock64() - t0;
                const uint32_t nrows = min((uint32_t)kUM, it.row_count - t * kUM);
                if (lane == 0) {  // metadata first: the epilogue prefetches the row norms meanwhile
                    meta[b] = UMeta{it.row_start + t * kUM, nrows, it.qcount, it.ncols, ib,
                                    t + 1 == n_tiles ? 1u : 0u, 0, 0};
                    mb_arrive(metafull + b);
                }
                t0 = clock64();
                mb_wait(afull + s, (a_use / S) & 1);
                tp_afull += clock64() - t0;
                tc_fence_after();
                if (lane == 0) {
                    const uint32_t td = tmem + b * 256;
                    uint32_t accf = 0;
                    for (int c = 0; c < c_dense; ++c) {
                        const uint32_t sa = su32(sm + L.a + ((size_t)s * c_dense + c) * kUM * 128);
                        const uint32_t sb = su32(bb + (size_t)c * kUQ * 128);
                        const int nk = min(4, (int)(d0 - c * 32) / 8);
                        for (int kk = 0; kk < nk; ++kk) {
                            tc_mma(td, desc_sw128(sa + kk * 32), desc_sw128(sb + kk * 32), idesc, accf);
                            accf = 1;
                        }
                    }
                    tc_mma(td, desc_sw32(su32(sm + L.a_aug + (size_t)s * kUM * 32)), desc_sw32(su32(baug)), idesc, 1u);
                    tc_commit(aempty + s);
                    tc_commit(accfull + b);
                    if (t + 1 == n_tiles) tc_commit(bfree + ib);
                }
                __syncwarp();
                st_dco += (unsigned long long)nrows * it.qcount;
                st_bytes += 4ull * d0 * nrows;
                ++a_use;
                ++acc_it;
            }
        }
        // tell the epilogue warps to stop
        {
            const uint32_t b = acc_it & 1;
            if (acc_it >= 2) mb_wait(accempty + b, ((acc_it >> 1) - 1) & 1);
            if (lane == 0) {
                meta[b].row0 = kUSentinel;
                mb_arrive(metafull + b);
            }
            __syncwarp();
        }
        if (lane == 0 && a.census) {
            atomicAdd(a.census + 2, (unsigned long long)tp_bready);
            atomicAdd(a.census + 3, (unsigned long long)tp_accempty);
            atomicAdd(a.census + 4, (unsigned long long)tp_afull);
        }
        if (lane == 0 && a.counters) {
            atomicAdd(a.counters + 0, st_dco);
            atomicAdd(a.counters + 1, st_dco * d0);  // kept pairs' share is taken back by the epilogue
            atomicAdd(a.counters + 2, st_bytes);
        }
    } else {
        // ============================ epilogue ============================
        const uint32_t quarter = warp & 3, cgrp = warp >> 2;  // rows 32 quarter.., columns chunks cgrp + 4 i
        unsigned long long st_kept = 0, st_surv = 0;
        long long te_meta = 0, te_acc = 0;
        const bool dbg = a.debug == 1;
        // kept pairs of a 32-column chunk -> worklist, column (query) major so the
        // survivor kernel's warps mostly see one query; one atomic per chunk
        // kept pairs of a 32-column chunk -> worklist, column (query) major so the
        // survivor kernel's warps mostly see one query; one atomic per chunk, and
        // only the columns holding a kept pair are walked
        // keep mask of a 32-column chunk for this lane's row: bit i <=> !(v[i] < 0)
        // (sign bit clear), restricted to real rows and queries
        auto keep_mask = [&](const float (&v)[32], uint32_t c0, const UMeta& m, uint32_t r) -> uint32_t {
            uint32_t km = 0;
#pragma unroll
            for (int i = 0; i < 32; ++i) km |= (~__float_as_uint(v[i]) >> 31) << i;
            const uint32_t ncol = m.qcount > c0 ? min(32u, m.qcount - c0) : 0u;
            const uint32_t vmask = r < m.nrows ? (ncol == 32 ? 0xffffffffu : ((1u << ncol) - 1u)) : 0u;
            return km & vmask;
        };
        auto valid_mask = [&](uint32_t c0, const UMeta& m, uint32_t r) -> uint32_t {
            const uint32_t ncol = m.qcount > c0 ? min(32u, m.qcount - c0) : 0u;
            return r < m.nrows ? (ncol == 32 ? 0xffffffffu : ((1u << ncol) - 1u)) : 0u;
        };
        // kept pairs of a chunk -> worklist, column (query) major so the survivor
        // kernel's warps mostly see one query; one atomic per chunk, and only the
        // columns holding a pair to emit are walked
        auto emit_chunk = [&](uint32_t km, uint32_t em, uint32_t c0, const UMeta& m, uint32_t r) {
            const uint32_t total = __reduce_add_sync(0xffffffffu, __popc(em));
            if (!total) return;
            const uint32_t kept = __reduce_add_sync(0xffffffffu, __popc(km));
            uint32_t sb = 0;
            if (lane == 0) sb = atomicAdd(a.surv_count, total);
            sb = __shfl_sync(0xffffffffu, sb, 0);
            const uint32_t lt = (1u << lane) - 1u;
            for (uint32_t cols = __reduce_or_sync(0xffffffffu, em); cols; cols &= cols - 1) {
                const int i = __ffs(cols) - 1;
                const bool emit = (em >> i) & 1u;
                const uint32_t bl = __ballot_sync(0xffffffffu, emit);
                if (emit) {
                    const uint32_t p = sb + __popc(bl & lt);
                    if (p < a.surv_cap) {
                        const uint32_t col = c0 + i;
                        Survivor sv;
                        sv.q = qidx_s[m.ib * kUQ + col];
                        sv.row = m.row0 + r;
                        sv.acc = 0.f;
                        sv.slot = slot_s[m.ib * kUQ + col] | (((km >> i) & 1u) ? 0u : 0x80000000u);
                        a.surv[p] = sv;
                    }
                }
                sb += __popc(bl);
            }
            if (lane == 0) {
                st_surv += total;
                st_kept += kept;
            }
        };
        for (uint32_t k = 0;; ++k) {
            const uint32_t b = k & 1;
            long long t0 = clock64();
            mb_wait(metafull + b, (k >> 1) & 1);
            te_meta += clock64() - t0;
            const UMeta m = meta[b];
            if (m.row0 == kUSentinel) break;
            const uint32_t r = quarter * 32 + lane;  // rows past the item are masked in keep_mask
            t0 = clock64();
            mb_wait(accfull + b, (k >> 1) & 1);
            te_acc += clock64() - t0;
            tc_fence_after();
            const uint32_t nch = m.ncols / 32;
            const uint32_t tbase = tmem + ((quarter * 32) << 16) + b * 256;
            for (uint32_t c = cgrp; c < nch; c += 4) {  // one 32-column chunk per round
                float v[32];
                tc_ld32_nowait(tbase + c * 32, v);
                asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
                // all negative <=> the AND of the bit patterns has the sign bit (rows
                // past the item are forced negative); only then the keep mask
                uint32_t andv = (r < m.nrows ? 0u : 0x80000000u) | __float_as_uint(v[0]);
#pragma unroll
                for (int i = 1; i < 32; ++i) andv &= __float_as_uint(v[i]);
                if (!__any_sync(0xffffffffu, !(andv >> 31)) && !dbg) continue;
                const uint32_t km = keep_mask(v, c * 32, m, r);
                const uint32_t em = dbg ? valid_mask(c * 32, m, r) : km;
                emit_chunk(km, em, c * 32, m, r);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mb_arrive(accempty + b);
                if (m.last) mb_arrive(bfree + m.ib);  // this item's query ids no longer read
            }
        }
        if (lane == 0 && a.census && warp == 0) {
            atomicAdd(a.census + 5, (unsigned long long)te_meta);
            atomicAdd(a.census + 6, (unsigned long long)te_acc);
        }
        if (lane == 0 && a.counters) {
            // kept pairs continue in the survivor kernel (which counts their dims)
            if (st_kept) atomicAdd(a.counters + 1, 0ull - (unsigned long long)st_kept * d0);
            atomicAdd(a.counters + 2, 16ull * st_surv);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kUMma) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(kUTmemCols));
    }
}

}  // namespace

size_t filter_umma_smem_bytes(int c_dense) { return u_layout(c_dense).total; }

cudaError_t launch_filter_umma(const FilterArgs& a, const CUtensorMap& tmap128, const CUtensorMap& tmap_aug,
                               uint32_t grid, cudaStream_t s) {
    if (grid == 0) return cudaSuccess;
    const size_t smem = filter_umma_smem_bytes(a.c_dense);
    DADE_CUDA_TRY(cudaFuncSetAttribute(dco_filter_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dco_filter_umma_kernel<<<grid, kUThreads, smem, s>>>(a, tmap128, tmap_aug);
    return cudaGetLastError();
}

namespace {
__global__ void row_aug_kernel(const float* __restrict__ norms, uint32_t n, float* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float h = 0.5f * (1.f - kUDelta) * norms[i];
    const float hi = tf32_hi(h);
    float4* o = reinterpret_cast<float4*>(out + (size_t)i * 8);
    o[0] = make_float4(-hi, -(h - hi), 1.f, 1.f);
    o[1] = make_float4(0.f, 0.f, 0.f, 0.f);
}
}  // namespace

// ---- coarse ranking GEMM on tcgen05 ----------------------------------------------
// p~(q, c) = |c|^2 + |q|^2 - 2 c.q for a 128-centroid x 256-query tile per CTA:
// lane 0 of warp 4 TMA-loads 32-dim atoms of both operands (SW128) into a
// 3-stage ring and issues the TF32 MMAs into a 256-column TMEM accumulator;
// warps 0-3 read it back (TMEM lane = centroid) and store p~ per (query, centroid)
// for coarse_select (same values and bound as coarse_tc_kernel, coarse.cu).
namespace {
constexpr int kCgM = 128, kCgN = 256, kCgStages = 2;  // 2 stages: 2 CTAs per SM, one in its epilogue while the other loads
constexpr int kCgThreads = 160;

// Fused-selection modes (CoarseFilter, large nlist): pass A writes only the
// group minima (p_out == nullptr), pass B (t0 != nullptr) recomputes the same
// tile and appends every (p~, centroid) whose lower bound is <= the query's T0
// to the query's candidate list -- p~ never goes to memory.
__global__ void __launch_bounds__(kCgThreads, 2)
coarse_umma_kernel(const __grid_constant__ CUtensorMap tm_cen, const __grid_constant__ CUtensorMap tm_q, uint32_t q0,
                   uint32_t n_cen, uint32_t nq, uint32_t dim, const float* __restrict__ cnorm,
                   const float* __restrict__ qnorm, float* __restrict__ p_out, uint32_t* __restrict__ gmin,
                   const CoarseFilter cf) {
    extern __shared__ unsigned char cg_raw[];
    unsigned char* sm = cg_raw + ((1024u - (su32(cg_raw) & 1023u)) & 1023u);
    constexpr uint32_t kABytes = kCgM * 128, kBBytes = kCgN * 128;
    unsigned char* ring = sm;  // [stage][A 16 KB | B 32 KB]
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + kCgStages * (kABytes + kBBytes));
    uint64_t* full = bars;
    uint64_t* empty = bars + kCgStages;
    uint64_t* accf = bars + 2 * kCgStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kCgStages + 1);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t c0 = blockIdx.x * kCgM, qt = blockIdx.y * kCgN;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kCgStages; ++i) {
            mb_init(full + i, 1);
            mb_init(empty + i, 1);
        }
        mb_init(accf, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 4) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                     "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    const uint32_t n_atoms = (dim + 31) / 32;
    if (warp == 4) {
        if (lane == 0) {
            auto issue = [&](uint32_t k) {
                const uint32_t s = k % kCgStages;
                if (k >= (uint32_t)kCgStages) mb_wait(empty + s, ((k / kCgStages) - 1) & 1);
                unsigned char* st = ring + (size_t)s * (kABytes + kBBytes);
                mb_arrive_tx(full + s, kABytes + kBBytes);
                tma2d_u(st, &tm_cen, (int)(k * 32), (int)c0, full + s);
                tma2d_u(st + kABytes, &tm_q, (int)(k * 32), (int)(q0 + qt), full + s);
            };
            uint32_t k_issue = 0;
            while (k_issue < n_atoms && k_issue < (uint32_t)kCgStages) issue(k_issue++);
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kCgN >> 3) << 17) |
                                   ((uint32_t)(kCgM >> 4) << 24);
            for (uint32_t k = 0; k < n_atoms; ++k) {
                const uint32_t s = k % kCgStages;
                mb_wait(full + s, (k / kCgStages) & 1);
                tc_fence_after();
                const unsigned char* st = ring + (size_t)s * (kABytes + kBBytes);
                const uint32_t sa = su32(st), sb = su32(st + kABytes);
                const int nk = min(4, (int)(dim - k * 32 + 7) / 8);
                for (int kk = 0; kk < nk; ++kk)
                    tc_mma(tmem, desc_sw128(sa + kk * 32), desc_sw128(sb + kk * 32), idesc, (k | kk) ? 1u : 0u);
                tc_commit(empty + s);
                if (k_issue < n_atoms) issue(k_issue++);
            }
            tc_commit(accf);
        }
        __syncwarp();
    } else if (cf.t0) {
        // pass B: candidates lo <= T0 per query column, appended warp-aggregated
        mb_wait(accf, 0);
        tc_fence_after();
        const uint32_t c = c0 + warp * 32 + lane;
        const float cn = c < n_cen ? cnorm[c] : 0.f;
        for (uint32_t j = 0; j < (uint32_t)kCgN / 32; ++j) {
            if (qt + j * 32 >= nq) break;
            float v[32];
            tc_ld32_nowait(tmem + ((warp * 32) << 16) + j * 32, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            const uint32_t myq = qt + j * 32 + lane;  // this lane's query column (T0 and qnorm loads)
            const uint32_t t0_mine = myq < nq ? cf.t0[myq] : 0u;
            const float qn_mine = myq < nq ? qnorm[myq] : 0.f;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const uint32_t qq = qt + j * 32 + i;
                const uint32_t t0 = __shfl_sync(0xffffffffu, t0_mine, i);
                const float qn = __shfl_sync(0xffffffffu, qn_mine, i);
                const float p = fmaf(-2.f, v[i], cn + qn);
                const bool is = c < n_cen && qq < nq && fkey(__fsub_rn(p, coarse_delta(cn, qn))) <= t0;
                const uint32_t bal = __ballot_sync(0xffffffffu, is);
                if (!bal) continue;
                uint32_t base = 0;
                if (lane == __ffs(bal) - 1) base = atomicAdd(cf.cnt + qq, (uint32_t)__popc(bal));
                base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
                const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
                if (is && pos < cf.cap)
                    cf.cand[(size_t)qq * cf.cap + pos] = (static_cast<uint64_t>(__float_as_uint(p)) << 32) | c;
            }
        }
    } else {
        // epilogue: TMEM lane = centroid c0 + 32 warp + lane; columns = queries
        mb_wait(accf, 0);
        tc_fence_after();
        const uint32_t c = c0 + warp * 32 + lane;
        const float cn = c < n_cen ? cnorm[c] : 0.f;
        for (uint32_t j = 0; j < (uint32_t)kCgN / 32; ++j) {
            if (qt + j * 32 >= nq) break;
            float v[32];
            tc_ld32_nowait(tmem + ((warp * 32) << 16) + j * 32, v);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            const uint32_t ng = (n_cen + 31) / 32, grp = (c0 + warp * 32) / 32;
            uint32_t mine = 0xffffffffu;
#pragma unroll
            for (int i = 0; i < 32; ++i) {
                const uint32_t qq = qt + j * 32 + i;
                const float qn = qq < nq ? qnorm[qq] : 0.f;
                const float p = fmaf(-2.f, v[i], cn + qn);
                if (p_out && c < n_cen && qq < nq) p_out[(size_t)qq * n_cen + c] = p;
                if (gmin) {  // min upper-bound key of this warp's 32 centroids, per query column
                    const uint32_t m = __reduce_min_sync(
                        0xffffffffu, c < n_cen ? fkey(__fadd_rn(p, coarse_delta(cn, qn))) : 0xffffffffu);
                    if (lane == i) mine = m;
                }
            }
            if (gmin) {
                const uint32_t qq = qt + j * 32 + lane;
                if (qq < nq && grp < ng) gmin[(size_t)qq * ng + grp] = mine;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 4) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(256));
    }
}

}  // namespace

// ---- fused large-nlist coarse selection, query-major (tcgen05) -----------------------
// One CTA per 128 queries (MMA M = queries: TMEM lane = query), the query block
// staged once (TMA, SW128, all 32-dim atoms), the centroids streamed as 256-row
// tiles (MMA N) through a 4-stage ring of 32-dim atoms (they stay L2-resident:
// 8 MB at nlist 16384, D 128), two 256-column TMEM accumulators so the MMAs of
// tile t+1 run under the epilogue of tile t. Eight epilogue warps: warp w reads
// TMEM lanes 32 (w % 4).. and columns 128 (w / 4).. of each tile, one thread =
// one query, no cross-lane traffic:
//   pass A: per 32 centroids the minimum upper-bound key fkey(p~ + delta)
//           -> gmin[group][query] (coalesced);
//   pass B: every centroid with lower bound fkey(p~ - delta) <= t0[query]
//           -> (p~ bits << 32 | centroid) appended to the query's list.
// Same p~ = |c|^2 + |q|^2 - 2 q.c and bound as the other coarse kernels.
constexpr int kSqM = 128, kSqN = 256, kSqStages = 4, kSqEpiWarps = 16;
constexpr int kSqCols = kSqN / (kSqEpiWarps / 4);  // columns per epilogue warp (64)
static_assert(kSqEpiWarps / 4 == (int)kCoarseSelParts, "one candidate-list slice per column part");
constexpr int kSqThreads = (kSqEpiWarps + 1) * 32;
constexpr uint32_t kSqAtomA = kSqM * 128, kSqAtomB = kSqN * 128;  // bytes per 32-dim atom

struct SqLayout {
    uint32_t a, ring, cn, bars, total;
};
__host__ __device__ inline SqLayout sq_layout(uint32_t dim) {
    SqLayout L;
    const uint32_t n_atoms = (dim + 31) / 32;
    L.a = 0;
    L.ring = L.a + n_atoms * kSqAtomA;
    L.cn = L.ring + kSqStages * kSqAtomB;
    L.bars = L.cn + 2 * kSqEpiWarps * kSqCols * 4;
    L.total = L.bars + 16 * 8 + 16 + 1024;  // + alignment slack
    return L;
}

template <bool kPassB>
__global__ void __launch_bounds__(kSqThreads, 1)
coarse_sel_umma_kernel(const __grid_constant__ CUtensorMap tm_q128, const __grid_constant__ CUtensorMap tm_c256,
                       uint32_t q0, uint32_t n_cen, uint32_t nq, uint32_t dim, const float* __restrict__ cnorm,
                       const float* __restrict__ qnorm, uint32_t* __restrict__ gmin_t, const CoarseFilter cf) {
    extern __shared__ unsigned char sq_raw[];
    unsigned char* sm = sq_raw + ((1024u - (su32(sq_raw) & 1023u)) & 1023u);
    const SqLayout L = sq_layout(dim);
    unsigned char* sa = sm + L.a;
    unsigned char* ring = sm + L.ring;
    float* cn_s = reinterpret_cast<float*>(sm + L.cn);  // [2][warp][128] centroid norms of each warp's columns
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
    uint64_t* afull = bars;
    uint64_t* full = bars + 1;                 // [kSqStages]
    uint64_t* empty = full + kSqStages;        // [kSqStages]
    uint64_t* accf = empty + kSqStages;        // [2]
    uint64_t* acce = accf + 2;                 // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t qb = blockIdx.x * kSqM;
    const uint32_t n_atoms = (dim + 31) / 32, n_tiles = (n_cen + kSqN - 1) / kSqN;
    if (threadIdx.x == 0) {
        mb_init(afull, 1);
        for (int i = 0; i < kSqStages; ++i) {
            mb_init(full + i, 1);
            mb_init(empty + i, 1);
        }
        for (int b = 0; b < 2; ++b) {
            mb_init(accf + b, 1);
            mb_init(acce + b, kSqEpiWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == kSqEpiWarps) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (warp == kSqEpiWarps) {
        if (lane == 0) {
            // the query block: every atom once
            mb_arrive_tx(afull, n_atoms * kSqAtomA);
            for (uint32_t k = 0; k < n_atoms; ++k) tma2d_u(sa + k * kSqAtomA, &tm_q128, (int)(k * 32), (int)(q0 + qb), afull);
            const uint32_t total = n_tiles * n_atoms;
            auto issue = [&](uint32_t i) {  // i-th (tile, atom) of the centroid stream
                const uint32_t s = i % kSqStages;
                if (i >= (uint32_t)kSqStages) mb_wait(empty + s, ((i / kSqStages) - 1) & 1);
                mb_arrive_tx(full + s, kSqAtomB);
                tma2d_u(ring + (size_t)s * kSqAtomB, &tm_c256, (int)((i % n_atoms) * 32), (int)((i / n_atoms) * kSqN),
                        full + s);
            };
            uint32_t next = 0;
            while (next < total && next < (uint32_t)kSqStages) issue(next++);
            const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(kSqN >> 3) << 17) |
                                   ((uint32_t)(kSqM >> 4) << 24);
            mb_wait(afull, 0);
            for (uint32_t t = 0; t < n_tiles; ++t) {
                const uint32_t b = t & 1;
                if (t >= 2) mb_wait(acce + b, ((t >> 1) - 1) & 1);
                tc_fence_after();
                for (uint32_t k = 0; k < n_atoms; ++k) {
                    const uint32_t i = t * n_atoms + k, s = i % kSqStages;
                    mb_wait(full + s, (i / kSqStages) & 1);
                    tc_fence_after();
                    const uint32_t a_addr = su32(sa + k * kSqAtomA), b_addr = su32(ring + (size_t)s * kSqAtomB);
                    const int nk = min(4, (int)(dim - k * 32 + 7) / 8);
                    for (int kk = 0; kk < nk; ++kk)
                        tc_mma(tmem + b * kSqN, desc_sw128(a_addr + kk * 32), desc_sw128(b_addr + kk * 32), idesc,
                               (k | kk) ? 1u : 0u);
                    tc_commit(empty + s);
                    if (next < total) issue(next++);
                }
                tc_commit(accf + b);
            }
        }
        __syncwarp();
    } else {
        // epilogue: thread = query qb + 32 (warp % 4) + lane, columns [64 (warp / 4), +64) of each tile;
        // bounds compared as floats (fkey is monotone): hi = p~ + delta, lo = p~ - delta
        const uint32_t quarter = warp & 3, part = warp >> 2;
        const uint32_t qq = qb + quarter * 32 + lane;
        const bool qok = qq < nq;
        const float qn = qok ? qnorm[qq] : 0.f;
        // pass B: candidates of part p go to cand[q][p * part_cap ..], their count to cnt[q * 4 + p]
        const uint32_t part_cap = cf.cap / (kSqEpiWarps / 4);
        uint64_t* part_list = kPassB ? cf.cand + (size_t)qq * cf.cap + part * part_cap : nullptr;
        uint32_t n_app = 0;
        float t0f = 0.f;
        if (kPassB && qok) {  // the float whose key is t0
            const uint32_t k = cf.t0[qq];
            t0f = __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
        }
        for (uint32_t t = 0; t < n_tiles; ++t) {
            const uint32_t b = t & 1, c_tile = t * kSqN;
            float* cns = cn_s + (b * kSqEpiWarps + warp) * kSqCols;  // this warp's column norms
#pragma unroll
            for (int r = 0; r < kSqCols / 32; ++r) {
                const uint32_t c = c_tile + part * kSqCols + r * 32 + lane;
                cns[r * 32 + lane] = c < n_cen ? cnorm[c] : 0.f;
            }
            __syncwarp();
            mb_wait(accf + b, (t >> 1) & 1);
            tc_fence_after();
            const uint32_t col0 = part * kSqCols;
            float v[2][32];
            tc_ld32_nowait(tmem + ((quarter * 32) << 16) + b * kSqN + col0, v[0]);
            tc_ld32_nowait(tmem + ((quarter * 32) << 16) + b * kSqN + col0 + 32, v[1]);
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mb_arrive(acce + b);  // accumulator read: the MMAs of tile t + 2 may start
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t cb = c_tile + col0 + h * 32;
                if (cb >= n_cen) break;
                if (!kPassB) {
                    float m[4] = {__int_as_float(0x7f800000), __int_as_float(0x7f800000), __int_as_float(0x7f800000),
                                  __int_as_float(0x7f800000)};  // 4 independent chains
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float cn = cns[h * 32 + i];
                        const float p = fmaf(-2.f, v[h][i], cn + qn);
                        const float hi = __fadd_rn(p, coarse_delta(cn, qn));
                        m[i & 3] = (cb + i < n_cen) ? fminf(m[i & 3], hi) : m[i & 3];
                    }
                    if (qok) gmin_t[(size_t)(cb / 32) * nq + qq] = fkey(fminf(fminf(m[0], m[1]), fminf(m[2], m[3])));
                } else if (qok) {
                    // this thread's own slice of the query's list (part p of kSqEpiWarps / 4): no atomics
#pragma unroll
                    for (int i = 0; i < 32; ++i) {
                        const float cn = cns[h * 32 + i];
                        const float p = fmaf(-2.f, v[h][i], cn + qn);
                        if (__fsub_rn(p, coarse_delta(cn, qn)) <= t0f && cb + i < n_cen) {
                            if (n_app < part_cap)
                                part_list[n_app] = (static_cast<uint64_t>(__float_as_uint(p)) << 32) | (cb + i);
                            ++n_app;
                        }
                    }
                }
            }
        }
        if (kPassB && qok) cf.cnt[(size_t)qq * (kSqEpiWarps / 4) + part] = n_app;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == kSqEpiWarps) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
    }
}

size_t coarse_umma_smem_bytes() { return (size_t)kCgStages * (kCgM * 128 + kCgN * 128) + 8 * 8 + 1024; }

cudaError_t launch_coarse_umma(const CUtensorMap& tm_cen, const CUtensorMap& tm_q, uint32_t q0, uint32_t n_cen,
                               uint32_t nq, uint32_t dim, const float* cnorm, const float* qnorm, float* p_out,
                               cudaStream_t s, uint32_t* gmin, const CoarseFilter& cf) {
    if (nq == 0 || n_cen == 0) return cudaSuccess;
    const size_t smem = coarse_umma_smem_bytes();
    DADE_CUDA_TRY(cudaFuncSetAttribute(coarse_umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((n_cen + kCgM - 1) / kCgM, (nq + kCgN - 1) / kCgN);
    coarse_umma_kernel<<<grid, kCgThreads, smem, s>>>(tm_cen, tm_q, q0, n_cen, nq, dim, cnorm, qnorm, p_out, gmin,
                                                       cf);
    return cudaGetLastError();
}

bool coarse_sel_umma_ok(uint32_t dim) { return dim % 4 == 0 && dim >= 32 && dim <= 256 && sq_layout(dim).total <= 227 * 1024; }

cudaError_t launch_coarse_sel_umma(const CUtensorMap& tm_q128, const CUtensorMap& tm_c256, uint32_t q0, uint32_t n_cen,
                                   uint32_t nq, uint32_t dim, const float* cnorm, const float* qnorm, uint32_t* gmin_t,
                                   const CoarseFilter& cf, cudaStream_t s) {
    if (nq == 0 || n_cen == 0) return cudaSuccess;
    if (!coarse_sel_umma_ok(dim)) return cudaErrorInvalidValue;
    const size_t smem = sq_layout(dim).total;
    const dim3 grid((nq + kSqM - 1) / kSqM);
    if (cf.t0) {
        DADE_CUDA_TRY(cudaFuncSetAttribute(coarse_sel_umma_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        coarse_sel_umma_kernel<true><<<grid, kSqThreads, smem, s>>>(tm_q128, tm_c256, q0, n_cen, nq, dim, cnorm, qnorm,
                                                                    gmin_t, cf);
    } else {
        DADE_CUDA_TRY(cudaFuncSetAttribute(coarse_sel_umma_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem));
        coarse_sel_umma_kernel<false><<<grid, kSqThreads, smem, s>>>(tm_q128, tm_c256, q0, n_cen, nq, dim, cnorm,
                                                                     qnorm, gmin_t, cf);
    }
    return cudaGetLastError();
}

cudaError_t launch_row_aug(const float* norms, uint32_t n, float* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    row_aug_kernel<<<(n + 255) / 256, 256, 0, s>>>(norms, n, out);
    return cudaGetLastError();
}

}  // namespace dade_gpu

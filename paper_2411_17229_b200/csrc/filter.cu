// Streaming first-slice DCO filter (the bulk of the IVF-DADE / flat DADE scan).
//
// One CTA = one work item (an IVF posting list or flat row block x up to kQC
// queries); the item's queries' dense dims [0, d0) stay resident in shared
// memory. Each WARP streams its own 32-row tiles of the item through a private
// TMA ring (no producer warp, no CTA barrier, so a warp with more survivors
// never stalls the others) and, per tile:
//   1. tensor cores (mma.sync TF32, ldmatrix A fragments from the 128B-swizzled
//      box) give o.q for all 32 x kQC pairs over the dense dims;
//   2. prune for sure iff (1 - delta)(|o|^2 + |q|^2) - 2 o.q > thr0  (rigorous
//      bound, see kTcDelta): the reference would have rejected those pairs at
//      the first checkpoint (proj/src/estimator.cpp:46-58);
//   3. every other pair gets the exact sequential fp32 prefix from shared
//      memory and the exact checkpoint test; survivors are appended to a global
//      worklist that advance_survivors_kernel continues from d0.
// The radius of each query is fixed for the launch (read from r_global at the
// item start); the host tightens it between passes.
#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

constexpr int kFRows = 32;          // rows per warp tile
constexpr int kFSlots = 2;          // private ring depth per warp (per dense box)
constexpr int kFWarps = 8;
constexpr int kFThreads = kFWarps * 32;
constexpr int kFList = 128;         // kept-pair list per warp per round
constexpr float kTcDeltaF = 4e-3f;  // same bound as scan.cu's kTcDelta

__device__ __forceinline__ uint32_t smem_u32f(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init_f(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32f(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx_f(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32f(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive_f(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32f(bar)) : "memory");
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
// element (row, k) of a 128B-swizzled [rows][32] fp32 box
__device__ __forceinline__ int swzf(int row, int k) { return row * kBox + ((((k >> 2) ^ (row & 7))) << 2) + (k & 3); }

// Exact sequential fp32 prefix over the dense dims for G kept pairs per lane
// (meta = row | query << 8), G independent chains interleaved for ILP; each
// chain is the reference's accumulation order (proj/src/estimator.cpp:36-44).
template <int G>
__device__ __forceinline__ void prefix_chains(const float* box0, int c_dense, uint32_t d0, const float* q_res,
                                              const uint32_t (&meta)[4], float (&x)[4]) {
    for (int c = 0; c < c_dense; ++c) {
        const float* b = box0 + (size_t)c * kFRows * kBox;
        const float* qq = q_res + (size_t)c * kBox * kQS;
        const int wc = min(kBox, (int)d0 - c * kBox);
        const float* qb[G];
        const float* rb[G];
        int sw[G];
#pragma unroll
        for (int i = 0; i < G; ++i) {
            const uint32_t row = meta[i] & 0xffu;
            qb[i] = qq + (meta[i] >> 8);
            rb[i] = b + row * kBox;
            sw[i] = (int)(row & 7);
        }
#pragma unroll 2
        for (int k = 0; k < wc; k += 4) {
#pragma unroll
            for (int i = 0; i < G; ++i) {
                const float4 o4 = *reinterpret_cast<const float4*>(rb[i] + ((((k >> 2) ^ sw[i])) << 2));
                x[i] = sq_step(x[i], o4.x, qb[i][(k + 0) * kQS]);
                x[i] = sq_step(x[i], o4.y, qb[i][(k + 1) * kQS]);
                x[i] = sq_step(x[i], o4.z, qb[i][(k + 2) * kQS]);
                x[i] = sq_step(x[i], o4.w, qb[i][(k + 3) * kQS]);
            }
        }
    }
}

struct FLayout {
    size_t boxes, q_res, n_q, thr, qidx, slot, list_meta, list_acc, bars, total;
};

__host__ __device__ inline size_t al16(size_t x) { return (x + 15) & ~size_t(15); }

// boxes: [warp][slot][c_dense] of [kFRows][kBox] fp32 (4 KB, 1024-aligned)
__host__ __device__ inline FLayout f_layout(int d0, int c_dense) {
    FLayout L;
    size_t off = 0;
    L.boxes = off; off += (size_t)kFWarps * kFSlots * c_dense * kFRows * kBox * 4;
    L.q_res = off; off = al16(off + sizeof(float) * (size_t)d0 * kQS);
    L.n_q = off; off = al16(off + sizeof(float) * kQC);
    L.thr = off; off = al16(off + sizeof(float) * kQC);
    L.qidx = off; off = al16(off + sizeof(uint32_t) * kQC);
    L.slot = off; off = al16(off + sizeof(uint32_t) * kQC);
    L.list_meta = off; off = al16(off + sizeof(uint32_t) * kFWarps * kFList);
    L.list_acc = off; off = al16(off + sizeof(float) * kFWarps * kFList);
    L.bars = off; off = al16(off + sizeof(uint64_t) * kFWarps * kFSlots);
    L.total = off + 1024;
    return L;
}

__global__ void __launch_bounds__(kFThreads, 2)
dco_filter_kernel(const FilterArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ unsigned char fsmem_raw[];
    unsigned char* sm = fsmem_raw + ((1024u - (smem_u32f(fsmem_raw) & 1023u)) & 1023u);
    const int c_dense = a.c_dense;
    const uint32_t d0 = a.d0;
    const FLayout L = f_layout((int)d0, c_dense);
    float* q_res = reinterpret_cast<float*>(sm + L.q_res);
    float* n_q = reinterpret_cast<float*>(sm + L.n_q);
    float* thr = reinterpret_cast<float*>(sm + L.thr);
    uint32_t* qidx_s = reinterpret_cast<uint32_t*>(sm + L.qidx);
    uint32_t* slot_s = reinterpret_cast<uint32_t*>(sm + L.slot);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t dim = a.dim;

    __shared__ uint32_t s_item;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sm + L.bars);
    if (lane == 0)
        for (int i = 0; i < kFSlots; ++i) mbar_init_f(bars + warp * kFSlots + i, 1);
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    const int g = lane >> 2, tq = lane & 3;
    const int smi = lane >> 3, rr = lane & 7;  // ldmatrix addressing
    unsigned long long st_dco = 0, st_dims = 0, st_bytes = 0, st_surv = 0;
    uint32_t k_base = 0;  // this warp's running ring position (mbarrier phases persist across items)
    const uint32_t base = a.items ? (a.item_base ? *a.item_base : 0u) : 0u;
    const uint32_t end = a.items ? *a.n_items : a.flat_qchunks * ((a.flat_rows + a.flat_block - 1) / a.flat_block);

  for (;;) {  // persistent: CTAs pull work items from a global counter
    __syncthreads();  // previous item fully consumed (q_res, thr reuse)
    if (tid == 0) s_item = base + atomicAdd(a.item_counter, 1u);
    __syncthreads();
    const uint32_t item = s_item;
    if (item >= end) break;
    uint64_t t_item0 = 0;
    if (a.trace_slow_ns) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_item0));
    uint32_t kept_item = 0;

    // ---- work item -------------------------------------------------------------
    uint32_t row_start, row_count, qcount;
    if (a.items != nullptr) {
        const WorkItem wi = a.items[item];
        const uint32_t piece = wi.bucket_count >> 16;
        if (piece < a.piece_lo || piece >= a.piece_hi) continue;  // another sub-pass's rows
        row_start = wi.row_start;
        row_count = wi.row_count;
        qcount = wi.bucket_count & 0xffffu;
        if (tid < (int)qcount) {
            qidx_s[tid] = a.bucket_q[wi.bucket_start + tid];
            slot_s[tid] = a.bucket_slot[wi.bucket_start + tid];
        }
    } else {
        const uint32_t rb = item / a.flat_qchunks, qc = item % a.flat_qchunks;
        row_start = rb * a.flat_block;
        row_count = min(a.flat_block, a.flat_rows - row_start);
        qcount = min((uint32_t)kQC, a.flat_nq - qc * kQC);
        if (tid < (int)qcount) {
            qidx_s[tid] = qc * kQC + tid;
            slot_s[tid] = rb;
        }
    }
    if (tid < kQC && tid >= (int)qcount) { qidx_s[tid] = 0; slot_s[tid] = 0; }
    __syncthreads();
    for (uint32_t idx = tid; idx < d0 * kQC; idx += kFThreads) {
        const uint32_t k = idx / kQC, j = idx - k * kQC;
        q_res[k * kQS + j] = j < qcount ? __ldg(a.queries + (size_t)qidx_s[j] * dim + k) : 0.f;
    }
    if (tid < kQC) {
        thr[tid] = -__int_as_float(0x7f800000);  // padding queries: never kept
        if (tid < (int)qcount) {
            const float r = __uint_as_float(a.r_global[qidx_s[tid]]);
            thr[tid] = prune_threshold(a.coeff0, r);
        }
    }
    __syncthreads();
    if (tid < kQC) {
        float nq = 0.f;
        for (uint32_t k = 0; k < d0; ++k) nq = fmaf(q_res[k * kQS + tid], q_res[k * kQS + tid], nq);
        n_q[tid] = (1.f - kTcDeltaF) * nq;
    }
    __syncthreads();

    // ---- per-warp private tile stream -----------------------------------------------
    const uint32_t n_tiles = (row_count + kFRows - 1) / kFRows;
    float* myboxes = reinterpret_cast<float*>(sm + L.boxes) + (size_t)warp * kFSlots * c_dense * kFRows * kBox;
    uint64_t* mybar = bars + warp * kFSlots;
    uint32_t* lmeta = reinterpret_cast<uint32_t*>(sm + L.list_meta) + warp * kFList;
    float* lacc = reinterpret_cast<float*>(sm + L.list_acc) + warp * kFList;
    auto box = [&](uint32_t slot, int c) { return myboxes + ((size_t)slot * c_dense + c) * kFRows * kBox; };
    auto issue = [&](uint32_t t, uint32_t slot) {  // lane 0 only
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        mbar_arrive_tx_f(mybar + slot, (uint32_t)c_dense * kFRows * kBox * 4);
        for (int c = 0; c < c_dense; ++c)
            tma2d_f(box(slot, c), &tmap, c * kBox, (int)(row_start + t * kFRows), mybar + slot);
    };
    if (lane == 0) {
        if ((uint32_t)warp < n_tiles) issue(warp, k_base % kFSlots);
        if ((uint32_t)(warp + kFWarps) < n_tiles) issue(warp + kFWarps, (k_base + 1) % kFSlots);
    }
    uint32_t k_iter = k_base;
    for (uint32_t t = warp; t < n_tiles; t += kFWarps, ++k_iter) {
        const uint32_t slot = k_iter % kFSlots;
        const uint32_t tb = t * kFRows, nrows = min((uint32_t)kFRows, row_count - tb);
        mbar_wait_f(mybar + slot, (k_iter / kFSlots) & 1);
        st_dco += (uint64_t)nrows * qcount;
        st_bytes += 4ull * d0 * nrows;

        // first-slice row norm of row `lane` (precomputed per row; padded array)
        const float no = (1.f - kTcDeltaF) * __ldg(a.row_norms + row_start + tb + lane);

        // tensor-core filter, queries in halves of 32 (4 n-tiles)
        for (int half = 0; half < 2; ++half) {
            if ((uint32_t)(half * 32) >= qcount) break;
            float d[2][4][4];
#pragma unroll
            for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                for (int nt = 0; nt < 4; ++nt)
#pragma unroll
                    for (int v = 0; v < 4; ++v) d[mt][nt][v] = 0.f;
            for (int c = 0; c < c_dense; ++c) {
                const uint32_t bb = smem_u32f(box(slot, c));
                const float* qc = q_res + (c * kBox + tq) * kQS + half * 32 + g;
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
                        const uint32_t b0 = __float_as_uint(qc[ks * kQS + nt * 8]);
                        const uint32_t b1 = __float_as_uint(qc[(ks + 4) * kQS + nt * 8]);
#pragma unroll
                        for (int mt = 0; mt < 2; ++mt) mma_tf32_f(d[mt][nt], A[mt][0], A[mt][1], A[mt][2], A[mt][3], b0, b1);
                    }
                }
            }
            // filter; bit = ((mt * 2 + h) * 4 + nt) * 2 + cq
            uint32_t keep = 0;
#pragma unroll
            for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
                for (int cq = 0; cq < 2; ++cq) {
                    const int j = half * 32 + nt * 8 + 2 * tq + cq;
                    const float nqj = n_q[j], th = thr[j];
#pragma unroll
                    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                        for (int h = 0; h < 2; ++h) {
                            const float nor = __shfl_sync(0xffffffffu, no, mt * 16 + h * 8 + g);
                            const float lhs = fmaf(-2.f, d[mt][nt][h * 2 + cq], nor + nqj);
                            if (!(lhs > th)) keep |= 1u << (((mt * 2 + h) * 4 + nt) * 2 + cq);
                        }
                }
            }
            // padding queries have thr = -inf (never kept); rows past the item
            // (next list's rows or TMA zero fill) are masked explicitly
            if (nrows < (uint32_t)kFRows) {
#pragma unroll
                for (int mt = 0; mt < 2; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if ((uint32_t)(mt * 16 + h * 8 + g) >= nrows) keep &= ~(0xffu << ((mt * 2 + h) * 8));
            }
            const uint32_t total_pairs = min(32u, qcount - half * 32) * nrows;
            unsigned long long pruned = total_pairs;
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
                    lmeta[pos] = (uint32_t)(mt * 16 + h * 8 + g) | ((uint32_t)(half * 32 + nt * 8 + 2 * tq + cq) << 8);
                    keep &= ~(1u << b);
                    ++pos;
                }
                __syncwarp();
                const uint32_t n = min(tot, (uint32_t)kFList);
                pruned -= n;
                kept_item += n;
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
                    const bool surv = e < n && !(x[i] > thr[j]);
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
        }
        // refill this slot with the tile after next
        __syncwarp();
        if (lane == 0 && t + 2 * kFWarps < n_tiles) issue(t + 2 * kFWarps, slot);
    }
    k_base = k_iter;
    if (a.trace_slow_ns && lane == 0) {
        uint64_t t1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
        if (t1 - t_item0 > a.trace_slow_ns)
            printf("slow item %u warp %d: %llu ns rows %u q %u tiles %u kept %u\n", item, warp,
                   (unsigned long long)(t1 - t_item0), row_count, qcount, n_tiles, kept_item);
    }
  }  // items

    // ---- counters ----------------------------------------------------------------
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        st_dco += __shfl_xor_sync(0xffffffffu, st_dco, off);
        st_dims += __shfl_xor_sync(0xffffffffu, st_dims, off);
        st_bytes += __shfl_xor_sync(0xffffffffu, st_bytes, off);
    }
    if (lane == 0 && a.counters) {
        atomicAdd(a.counters + 0, st_dco / 32);  // every lane added the same per-tile count
        atomicAdd(a.counters + 1, st_dims);
        atomicAdd(a.counters + 2, st_bytes / 32 + 16ull * (st_surv / 32));
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

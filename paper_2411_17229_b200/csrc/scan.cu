// DCO scan kernel (K4/K6/K2 of SURVEY.md §2) and top-K merges (K5).
//
// One CTA = one work item: a contiguous row range (an IVF posting list, or a
// flat row block) x up to kQC queries. The range is swept in kRT-row tiles.
//
//   dense phase  the chunks up to and including the first checkpoint
//                (every chunk in FD mode): all kRT x kQC pairs of the tile in
//                registers, 4 rows x 8 queries per thread, packed FADD2/FFMA2
//                (bit-exact, see common.cuh). The o tile of the next
//                (tile, chunk) step is prefetched with cp.async while the
//                current one is computed (double buffer); the queries' dense
//                dims stay resident in shared memory for the whole item.
//   sparse phase pairs that pass the first checkpoint are compacted per warp
//                (ballot + prefix) and advanced one pair per lane straight
//                from global memory (L2) through the remaining chunks and
//                checkpoints (proj/src/estimator.cpp:39-70).
//   top-K        exact full-D survivors with distance <= r are merged by the
//                warp that owns the query into its (query, slot) top-K
//                segment in global memory. The K-th key tightens the
//                CTA's radius for the rest of the list (the reference's live
//                heap threshold, proj/src/ivf.cpp:221-229) and, by atomicMin,
//                the query's global radius read by every later tile of every
//                CTA.
//
// Warp w owns queries [8w, 8w+8) of the chunk for the whole item, so after
// the per-step __syncthreads that guards the o-tile double buffer, all
// survivor / candidate / merge work is warp-local.
#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

constexpr int kWarpList = 128;  // survivor-list entries per warp per round
constexpr int kNormWin = kRT + 4;  // 16-byte aligned window of row norms per box

// Relative error budget of the TF32 filter: |p~ - acc| <= kTcDelta * (|o|^2 + |q|^2)
// over the first slice. Derivation: fp32 operands read as TF32
// (truncated, < 2^-10 relative each) give a dot-product error
// < (2^-9 + 2^-20) sum|o_k q_k| <= 9.8e-4 (|o|^2 + |q|^2); tensor-core fp32
// accumulation of 8-term steps and the fp32 norms / combination add < 1e-5;
// the exact sequential fp32 partial differs from the real distance by
// < 32 * 3 * 2^-24 relative (< 1e-5 of (|o| + |q|)^2). So
// |p~ - acc| < 2 * 9.8e-4 + 3e-5 < 2.1e-3 of (|o|^2 + |q|^2) (d0 <= 64); 2.6e-3 leaves 24%
// (4e-3 kept ~1.5x more pairs for the exact survivor pass: the band between the
// bound and the threshold is what the survivor kernels spend their time on).
constexpr float kTcDelta = 2.6e-3f;

struct SmemLayout {
    size_t slots, norms, q_res, n_q, r_s, thr_s, qidx, slot, wl_meta, wl_acc, s2_meta, s2_acc, keys, mscratch, bars, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Ring slot = one TMA box [kRT rows][32 dims] (128B-swizzled, 16 KB) plus, when
// the queries are not resident, that chunk's query tile [32][kQS].
__host__ __device__ inline size_t slot_bytes(int d_res) {
    return (size_t)kRT * kBox * 4 + (d_res == 0 ? (size_t)kBox * kQS * 4 : 0);
}

// Offsets are relative to a 1024-byte aligned base (128B swizzle atoms).
__host__ __device__ inline SmemLayout smem_layout(int n_ckpt, int d_res, int n_buf) {
    SmemLayout L;
    size_t off = 0;
    L.slots = off; off = align16(off + slot_bytes(d_res) * n_buf);
    off = (off + 1023) & ~size_t(1023);
    L.norms = off; off = align16(off + sizeof(float) * kNormWin * n_buf);
    L.q_res = off; off = align16(off + sizeof(float) * (size_t)d_res * kQS);
    L.n_q = off; off = align16(off + sizeof(float) * kQC);
    L.r_s = off; off = align16(off + sizeof(float) * kQC);
    L.thr_s = off; off = align16(off + sizeof(float) * kQC * (n_ckpt > 0 ? n_ckpt : 1));
    L.qidx = off; off = align16(off + sizeof(uint32_t) * kQC);
    L.slot = off; off = align16(off + sizeof(uint32_t) * kQC);
    L.wl_meta = off; off = align16(off + sizeof(uint32_t) * kWarps * kWarpList);
    L.wl_acc = off; off = align16(off + sizeof(float) * kWarps * kWarpList);
    L.s2_meta = off; off = align16(off + sizeof(uint32_t) * kWarps * kWarpList);
    L.s2_acc = off; off = align16(off + sizeof(float) * kWarps * kWarpList);
    L.keys = off; off = align16(off + sizeof(uint64_t) * kWarps * kRT);
    L.mscratch = off; off = align16(off + sizeof(uint64_t) * kWarps * kStageMaxK);
    L.bars = off; off = align16(off + sizeof(uint64_t) * 2 * n_buf);
    L.total = off + 1024;  // slack for aligning the dynamic smem base
    return L;
}

// Element (row, k) of a 128B-swizzled [rows][32] fp32 box: 16-byte chunk k/4 of
// row r lives at chunk (k/4) ^ (r % 8) (CU_TENSOR_MAP_SWIZZLE_128B).
__device__ __forceinline__ int swz(int row, int k) { return row * kBox + ((((k >> 2) ^ (row & 7))) << 2) + (k & 3); }

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x10000)  // suspend-time hint (ns): sleep instead of spinning
        : "memory");
}
// Plain (non-tensor) bulk copy global -> shared, completing on an mbarrier.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
        "[%4];\n" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}

// A fragment of m16n8k8.tf32 straight from a 128B-swizzled box: ldmatrix.x4
// treats each 8 x 16-byte sub-tile as 8 rows x 4 fp32 (thread t gets row t/4,
// word t%4), which is exactly a0..a3 = A[g][tq], A[g+8][tq], A[g][tq+4], A[g+8][tq+4].
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
                 : "r"(addr));
}

// D += A(16x8, row) * B(8x8, col), TF32 in, FP32 accumulate.
__device__ __forceinline__ void mma_tf32(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// Recompute query j's per-checkpoint float thresholds from r_s[j].
__device__ __forceinline__ void refresh_thr(float* thr_s, const float* r_s, const double* coeff,
                                            int n_ckpt, int j, int lane_in, int lanes) {
    const float r = r_s[j];
    for (int c = lane_in; c < n_ckpt; c += lanes) thr_s[j * n_ckpt + c] = prune_threshold(coeff[c], r);
}

// Warp-level: merge the m candidate keys of query j (in kb) into its segment,
// then tighten r_s[j] / thr_s / the global radius from the new K-th key.
__device__ __forceinline__ void merge_query(const ScanArgs& a, uint64_t* kb, uint32_t m, uint32_t j,
                                            const uint32_t* qidx_s, const uint32_t* slot_s, float* r_s,
                                            float* thr_s, int n_ckpt, int lane, uint64_t* scratch,
                                            bool tighten = true) {
    const size_t seg = (size_t)qidx_s[j] * a.n_slots + slot_s[j];
    uint64_t* A = a.seg_keys + seg * a.K;
    const uint32_t nc = a.K <= (uint32_t)kStageMaxK ? warp_merge_staged(A, a.seg_count + seg, a.K, kb, m, scratch)
                                                    : warp_merge(A, a.seg_count + seg, a.K, kb, m, false);
    if (tighten && nc == a.K) {
        const float rn = hi_f(A[a.K - 1]);
        if (rn < r_s[j]) {
            __syncwarp();
            if (lane == 0) {
                r_s[j] = rn;
                atomicMin(a.r_global + qidx_s[j], __float_as_uint(rn));
            }
            __syncwarp();
            refresh_thr(thr_s, r_s, a.coeff, n_ckpt, j, lane, 32);
        }
    }
    __syncwarp();
}

// Gather query jj's candidates of the warp list (meta bit 31) into kb and merge.
__device__ __forceinline__ void merge_list_candidates(const ScanArgs& a, const uint32_t* wl_meta,
                                                      const float* wl_acc, uint32_t n, uint64_t* kb,
                                                      uint32_t row_base, int warp, int lane,
                                                      const uint32_t* qidx_s, const uint32_t* slot_s,
                                                      float* r_s, float* thr_s, int n_ckpt,
                                                      unsigned long long& st_bytes, uint64_t* scratch) {
    for (int jj = 0; jj < 8; ++jj) {
        uint32_t m = 0;
        for (uint32_t e0 = 0; e0 < n; e0 += 32) {
            const uint32_t e = e0 + lane;
            bool is = false;
            uint32_t meta = 0;
            if (e < n) {
                meta = wl_meta[e];
                is = (meta & 0x80000000u) && ((meta >> 8) & 0xffu) == (uint32_t)jj;
            }
            const uint32_t bal = __ballot_sync(0xffffffffu, is);
            if (is) {
                const uint32_t g = row_base + (meta & 0xffu);
                const uint32_t id = a.row_ids ? __ldg(a.row_ids + g) : a.id_base + g;
                kb[m + __popc(bal & ((1u << lane) - 1u))] = make_key(wl_acc[e], id);
            }
            m += __popc(bal);
        }
        __syncwarp();
        if (m) {
            if (a.row_ids && lane == 0) st_bytes += 4ull * m;
            if (a.census && lane == 0) {
                atomicAdd(a.census + 0, 1ull);
                atomicAdd(a.census + 1, (unsigned long long)m);
            }
            merge_query(a, kb, m, warp * 8 + jj, qidx_s, slot_s, r_s, thr_s, n_ckpt, lane, scratch, false);
        }
    }
}

// After a tile's survivor rounds: tighten the warp's 8 radii from their
// segments' K-th keys. Decisions inside a tile all use the tile-start radii,
// so they do not depend on how pairs were split into rounds.
__device__ __forceinline__ void tighten_warp_radii(const ScanArgs& a, int warp, int lane, uint32_t my_q,
                                                   const uint32_t* qidx_s, const uint32_t* slot_s, float* r_s,
                                                   float* thr_s, int n_ckpt) {
    if (lane < (int)my_q) {
        const int j = warp * 8 + lane;
        const size_t seg = (size_t)qidx_s[j] * a.n_slots + slot_s[j];
        if (ld_volatile_u32(a.seg_count + seg) == a.K) {
            const float rn = hi_f(*reinterpret_cast<const volatile uint64_t*>(a.seg_keys + seg * a.K + a.K - 1));
            if (rn < r_s[j]) {
                r_s[j] = rn;
                atomicMin(a.r_global + qidx_s[j], __float_as_uint(rn));
                refresh_thr(thr_s, r_s, a.coeff, n_ckpt, j, 0, 1);
            }
        }
    }
    __syncwarp();
}

// Compact this lane's `pending` pair bits into the warp list (up to kWarpList
// per round); pair bit b -> (row, jj) via decode. Returns the round size.
template <class Decode, class AccOf>
__device__ __forceinline__ uint32_t compact_round(uint32_t& pending, uint32_t* wl_meta, float* wl_acc, int lane,
                                                  Decode decode, AccOf acc_of) {
    const uint32_t mine = __popc(pending);
    uint32_t incl = mine;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += y;
    }
    uint32_t pos = incl - mine;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    uint32_t bits = pending;
    while (bits && pos < (uint32_t)kWarpList) {
        const int b = __ffs(bits) - 1;
        bits &= bits - 1;
        uint32_t row, jj;
        decode(b, row, jj);
        wl_meta[pos] = row | (jj << 8);
        wl_acc[pos] = acc_of(b);
        pending &= ~(1u << b);
        ++pos;
    }
    __syncwarp();
    return min(total, (uint32_t)kWarpList);
}

// Optional per-phase clock accounting (DADE_GPU_PHASES=1): lane 0 of every
// consumer warp adds its clock64 deltas into a.phase[0..4] = {wait full slot,
// dense, epilogue, survivors, merges}.
#define PH_MARK(t) const long long t = a.phase ? clock64() : 0
#define PH_ADD(i, t0, t1) do { if (a.phase && lane == 0) atomicAdd(a.phase + (i), (unsigned long long)((t1) - (t0))); } while (0)

// Warp-specialised: warps 0..7 consume (each owns 8 queries of the item for
// the whole item), warp 8 produces. The producer streams the item's
// (tile, dense chunk) boxes through an n_buf-deep ring: one TMA
// (cp.async.bulk.tensor, 128B swizzle) per box into a slot whose `full`
// mbarrier completes on the transaction bytes; consumers wait on `full`,
// compute, and arrive on the slot's `empty` mbarrier (count 8) when done with
// it, so warps drift freely within the ring depth instead of meeting at a
// CTA barrier every step.
template <bool kSqrtKey, bool kTC>
__global__ void __launch_bounds__(kThreadsTotal, 2)
dco_scan_kernel(const ScanArgs a, const __grid_constant__ ChunkTable ct, const __grid_constant__ CUtensorMap tmap,
                const __grid_constant__ CUtensorMap tmap_n) {
    extern __shared__ unsigned char smem_raw[];
    // 1024-byte aligned base derived by pointer arithmetic (keeps the shared
    // address space visible to the compiler -> LDS, not generic loads)
    unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    const int n_ckpt = ct.n_ckpt;
    const int d_res = ct.d_res;  // resident query dims (0 -> staged per box by the producer)
    const int n_buf = ct.n_buf;
    const SmemLayout L = smem_layout(n_ckpt, d_res, n_buf);
    const size_t sbytes = slot_bytes(d_res);
    float* q_res = reinterpret_cast<float*>(smem + L.q_res);
    float* n_q = reinterpret_cast<float*>(smem + L.n_q);
    float* r_s = reinterpret_cast<float*>(smem + L.r_s);
    float* thr_s = reinterpret_cast<float*>(smem + L.thr_s);
    uint32_t* qidx_s = reinterpret_cast<uint32_t*>(smem + L.qidx);
    uint32_t* slot_s = reinterpret_cast<uint32_t*>(smem + L.slot);
    uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty_bar = full_bar + n_buf;
    auto slot_o = [&](uint32_t sl) { return reinterpret_cast<float*>(smem + L.slots + sl * sbytes); };
    float* norms_s = reinterpret_cast<float*>(smem + L.norms);
    auto slot_q = [&](uint32_t sl) { return reinterpret_cast<float*>(smem + L.slots + sl * sbytes + (size_t)kRT * kBox * 4); };

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const uint32_t dim = a.dim;

    // ---- decode the work item ------------------------------------------------
    uint32_t row_start, row_count, qcount;
    if (a.items != nullptr) {
        const uint32_t item = blockIdx.x + (a.item_base ? *a.item_base : 0u);
        if (item >= *a.n_items) return;
        const WorkItem wi = a.items[item];
        row_start = wi.row_start;
        row_count = wi.row_count;
        qcount = wi.bucket_count & 0xffffu;
        if (tid < (int)qcount) {
            qidx_s[tid] = a.bucket_q[wi.bucket_start + tid];
            slot_s[tid] = a.bucket_slot[wi.bucket_start + tid];
        }
    } else {
        const uint32_t rb = blockIdx.x / a.flat_qchunks;
        const uint32_t qc = blockIdx.x % a.flat_qchunks;
        row_start = rb * a.flat_block;
        row_count = min(a.flat_block, a.flat_rows - row_start);
        qcount = min((uint32_t)kQC, a.flat_nq - qc * kQC);
        if (tid < (int)qcount) {
            qidx_s[tid] = qc * kQC + tid;
            slot_s[tid] = rb;
        }
    }
    if (tid < kQC && tid >= (int)qcount) { qidx_s[tid] = 0; slot_s[tid] = 0; }
    if (a.seed && tid < kQC) slot_s[tid] = 0;
    if (a.max_rows) row_count = min(row_count, a.max_rows);
    if (tid < kQC) r_s[tid] = __int_as_float(0x7f800000);
    if (tid == 0) {
        for (int i = 0; i < n_buf; ++i) {
            mbar_init(full_bar + i, 1);
            mbar_init(empty_bar + i, kWarps);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (ct.use_tma) asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    __syncthreads();
    // resident queries, k-major [d_res][kQS]
    for (uint32_t idx = tid; idx < (uint32_t)d_res * kQC; idx += kThreadsTotal) {
        const uint32_t k = idx / kQC, j = idx - k * kQC;  // j fastest: conflict-free stores
        q_res[k * kQS + j] = j < qcount ? __ldg(a.queries + (size_t)qidx_s[j] * dim + k) : 0.f;
    }
    __syncthreads();

    const int c_dense = ct.n_dense;
    const uint32_t n_tiles = (row_count + kRT - 1) / kRT;
    const uint32_t n_steps = n_tiles * c_dense;

    // =========================== producer warp ===================================
    if (warp == kWarps) {
        unsigned long long st_bytes = 0;
        for (uint32_t s = 0; s < n_steps; ++s) {
            const uint32_t sl = s % n_buf;
            if (s >= (uint32_t)n_buf) mbar_wait(empty_bar + sl, ((s / n_buf) - 1) & 1);
            const uint32_t t = s / c_dense, c = s - t * c_dense;
            const uint32_t tb = t * kRT, nrows = min((uint32_t)kRT, row_count - tb);
            const uint32_t k0 = c == 0 ? 0u : ct.end[c - 1];
            const uint32_t w = ct.end[c] - k0;
            if (d_res == 0) {
                // stage this chunk's query slice (zero beyond w) next to the box
                float* qs = slot_q(sl);
                if (ct.vec_ok) {  // lane owns queries lane, lane + 32: 16-byte loads, transposed stores
                    for (uint32_t j = lane; j < (uint32_t)kQC; j += 32) {
                        const float* src = a.queries + (size_t)qidx_s[j] * dim + k0;
#pragma unroll
                        for (uint32_t v = 0; v < kBox / 4; ++v) {
                            float4 f = make_float4(0.f, 0.f, 0.f, 0.f);
                            if (j < qcount && 4 * v < w) f = __ldg(reinterpret_cast<const float4*>(src) + v);
                            qs[(4 * v + 0) * kQS + j] = f.x;
                            qs[(4 * v + 1) * kQS + j] = f.y;
                            qs[(4 * v + 2) * kQS + j] = f.z;
                            qs[(4 * v + 3) * kQS + j] = f.w;
                        }
                    }
                } else {
                    for (uint32_t idx = lane; idx < (uint32_t)kQC * kBox; idx += 32) {
                        const uint32_t j = idx / kBox, cc = idx - j * kBox;
                        qs[cc * kQS + j] = (j < qcount && cc < w) ? __ldg(a.queries + (size_t)qidx_s[j] * dim + k0 + cc) : 0.f;
                    }
                }
                st_bytes += 4ull * w * qcount;
            }
            float* ob = slot_o(sl);
            const bool want_norms = kTC && c == 0;  // first-slice row norms ride with chunk 0
            if (ct.use_tma) {
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive_expect_tx(full_bar + sl, kRT * kBox * 4 + (want_norms ? kNormWin * 4 : 0));
                    tma_load_2d(ob, &tmap, (int)k0, (int)(row_start + tb), full_bar + sl);
                    if (want_norms)  // 16B-aligned window [start & ~3, +kNormWin) of the padded norms array
                        bulk_load(norms_s + sl * kNormWin, a.row_norms + ((row_start + tb) & ~3u), kNormWin * 4,
                                  full_bar + sl);
                }
            } else {
                if (want_norms) {
                    const uint32_t al = (row_start + tb) & ~3u;
                    for (uint32_t r = lane; r < (uint32_t)kNormWin; r += 32)
                        norms_s[sl * kNormWin + r] = __ldg(a.row_norms + al + r);
                }
                for (uint32_t idx = lane; idx < (uint32_t)kRT * kBox; idx += 32) {
                    const uint32_t r = idx / kBox, cc = idx - r * kBox;
                    ob[swz(r, cc)] = (r < nrows && cc < w) ? __ldg(a.storage + (size_t)(row_start + tb + r) * dim + k0 + cc) : 0.f;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(full_bar + sl);
            }
            st_bytes += 4ull * w * nrows;
        }
        if (lane == 0 && a.counters) atomicAdd(a.counters + 2, st_bytes + sizeof(WorkItem) + 8ull * qcount + 4ull * d_res * qcount);
        return;
    }

    // =========================== consumer warps ==================================
    uint32_t* wl_meta = reinterpret_cast<uint32_t*>(smem + L.wl_meta) + warp * kWarpList;
    float* wl_acc = reinterpret_cast<float*>(smem + L.wl_acc) + warp * kWarpList;
    uint64_t* kb = reinterpret_cast<uint64_t*>(smem + L.keys) + warp * kRT;
    uint64_t* ms = reinterpret_cast<uint64_t*>(smem + L.mscratch) + warp * kStageMaxK;
    uint32_t* s2_meta = reinterpret_cast<uint32_t*>(smem + L.s2_meta) + warp * kWarpList;
    float* s2_acc = reinterpret_cast<float*>(smem + L.s2_acc) + warp * kWarpList;
    const uint32_t my_q = (uint32_t)max(0, min(8, (int)qcount - warp * 8));
    if (kTC && lane < (int)my_q) {  // first-slice query norms for the filter bound
        const int j = warp * 8 + lane;
        float nq = 0.f;
        for (int k = 0; k < d_res; ++k) nq = fmaf(q_res[k * kQS + j], q_res[k * kQS + j], nq);
        n_q[j] = nq;
    }
    __syncwarp();

    unsigned long long st_dco = 0, st_dims = 0, st_bytes = 0;
    unsigned long long st_elig = 0, st_fail = 0;  // failure accounting (a.measure)
    const uint64_t nz2 = a.neg_zero2;
    const uint32_t d0 = ct.end[c_dense - 1];
    const bool has_sparse = c_dense < ct.n_chunks;
    const bool vec = ct.vec_ok != 0;
    const int g = lane >> 2, tq = lane & 3;  // MMA fragment coordinates

    uint64_t acc[4][4];      // SIMT dense accumulators (kTC == false)
    uint32_t alive = 0;
    uint32_t pre_pruned = 0;  // failure accounting: pairs pruned at the first checkpoint, still scanned
    for (uint32_t s = 0; s < n_steps; ++s) {
        const uint32_t t = s / c_dense;
        const int c = (int)(s - t * c_dense);
        const uint32_t tb = t * kRT, nrows = min((uint32_t)kRT, row_count - tb);
        const uint32_t k0 = c == 0 ? 0u : ct.end[c - 1];
        const uint32_t w = ct.end[c] - k0;
        const uint32_t w4 = (w + 3) & ~3u;
        const uint32_t sl = s % n_buf;
        if (c == 0) {
            // tile start: pick up radii tightened by other CTAs; reset the pairs
            if (lane < (int)my_q) {
                const int j = warp * 8 + lane;
                const float rg = __uint_as_float(ld_volatile_u32(a.r_global + qidx_s[j]));
                if (rg < r_s[j] || t == 0) {
                    r_s[j] = fminf(rg, r_s[j]);
                    refresh_thr(thr_s, r_s, a.coeff, n_ckpt, j, 0, 1);
                }
            }
            __syncwarp();
            if (lane == 0) st_dco += (unsigned long long)nrows * my_q;
            if constexpr (!kTC) {
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;
                alive = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj)
                        if ((uint32_t)(lane + 32 * i) < nrows && (uint32_t)jj < my_q)
                            alive |= 1u << (i * 8 + jj);
            }
        }
        PH_MARK(t_w0);
        mbar_wait(full_bar + sl, (s / n_buf) & 1);
        PH_MARK(t_w1);
        PH_ADD(0, t_w0, t_w1);
        const float* ob = slot_o(sl);
        const float* qk = d_res > 0 ? q_res + k0 * kQS : slot_q(sl);

        if constexpr (kTC) {
            // the filter runs once per tile over all dense boxes (below)
        } else {
            // ---- dense register-tiled exact update ----------------------------
            if (__any_sync(0xffffffffu, alive != 0)) {
                for (uint32_t k4 = 0; k4 < w4; k4 += 4) {
                    float4 o[4];
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        o[i] = *reinterpret_cast<const float4*>(ob + swz(lane + 32 * i, k4));
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        const ulonglong2 qa = *reinterpret_cast<const ulonglong2*>(qk + (k4 + kk) * kQS + warp * 8);
                        const ulonglong2 qb = *reinterpret_cast<const ulonglong2*>(qk + (k4 + kk) * kQS + warp * 8 + 4);
                        const uint64_t qp[4] = {qa.x, qa.y, qb.x, qb.y};
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const float ov = kk == 0 ? o[i].x : kk == 1 ? o[i].y : kk == 2 ? o[i].z : o[i].w;
#pragma unroll
                            for (int p = 0; p < 4; ++p) acc[i][p] = sq_step2(acc[i][p], ov, qp[p], nz2);
                        }
                    }
                }
            }
            // the exact path keeps its partials in registers: free the slot now
            __syncwarp();
            if (lane == 0) mbar_arrive(empty_bar + sl);
        }
        PH_MARK(t_d1);
        PH_ADD(1, t_w1, t_d1);
        if (c != c_dense - 1) continue;

        // ---- end of the dense phase for this tile (warp-local from here) ------
        const int ck = ct.ckpt[c];
        const uint32_t row_base = row_start + tb;
        uint32_t pending = 0;  // pairs needing the exact / sparse path
        if constexpr (kTC) {
            // Tensor-core dot products o . q over the dense dims (ldmatrix A
            // fragments from the swizzled boxes, B from the resident queries),
            // then the filter per pair:
            //   prune for sure  iff  (1 - delta)(|o|^2 + |q|^2) - 2 o.q > thr
            // (|o|^2 precomputed per row, |q|^2 per query); everything else is
            // decided exactly below. Operands are fed as raw fp32 bits: the
            // tensor core reads them as TF32, which kTcDelta accounts for.
            const float* nrm = norms_s + ((s - (c_dense - 1)) % n_buf) * kNormWin + ((row_start + tb) & 3u);
            float nqp[2], thq[2];
            uint32_t qmask = 0;
#pragma unroll
            for (int cq = 0; cq < 2; ++cq) {
                const uint32_t jj = 2 * tq + cq;
                const int j = warp * 8 + jj;
                const bool ok = jj < my_q;
                nqp[cq] = ok ? (1.f - kTcDelta) * n_q[j] : 0.f;
                thq[cq] = ok ? thr_s[j * n_ckpt + ck] : -__int_as_float(0x7f800000);
                if (ok) qmask |= cq == 0 ? 0x55555555u : 0xAAAAAAAAu;  // bit = mt*4 + h*2 + cq
            }
            uint32_t valid = qmask;
            if (nrows < (uint32_t)kRT) {
#pragma unroll
                for (int mt = 0; mt < 8; ++mt)
#pragma unroll
                    for (int h = 0; h < 2; ++h)
                        if ((uint32_t)(mt * 16 + 8 * h + g) >= nrows) valid &= ~(3u << (mt * 4 + h * 2));
            }
            const int sm = lane >> 3, rr = lane & 7;  // ldmatrix: sub-matrix and row this lane addresses
#pragma unroll 1
            for (int mp = 0; mp < 8; mp += 2) {
                float d4[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
                if (my_q > 0 && (uint32_t)(mp * 16) < nrows) {
                    for (int cc = 0; cc < c_dense; ++cc) {
                        const uint32_t sb = smem_u32(slot_o((s - (c_dense - 1) + cc) % n_buf));
                        const uint32_t lo = cc == 0 ? 0u : ct.end[cc - 1], wc = ct.end[cc] - lo;
                        const float* qcol = q_res + (lo + tq) * kQS + warp * 8 + g;
                        const uint32_t rowa = (uint32_t)(mp * 16 + (sm & 1) * 8 + rr);
#pragma unroll 4
                        for (uint32_t ks = 0; ks < wc; ks += 8) {
                            const uint32_t b0 = __float_as_uint(qcol[ks * kQS]);
                            const uint32_t b1 = __float_as_uint(qcol[(ks + 4) * kQS]);
                            const uint32_t chunk = (ks >> 2) + (sm >> 1);
#pragma unroll
                            for (int u = 0; u < 2; ++u) {
                                const uint32_t row = rowa + 16 * u;
                                uint32_t a0, a1, a2, a3;
                                ldsm_x4(sb + row * (kBox * 4) + ((chunk ^ (row & 7)) << 4), a0, a1, a2, a3);
                                mma_tf32(d4[u], a0, a1, a2, a3, b0, b1);
                            }
                        }
                    }
                }
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    const int mt = mp + u;
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const float nop = (1.f - kTcDelta) * nrm[mt * 16 + 8 * h + g];
#pragma unroll
                        for (int cq = 0; cq < 2; ++cq) {
                            const float lhs = fmaf(-2.f, d4[u][2 * h + cq], nop + nqp[cq]);
                            if (!(lhs > thq[cq])) pending |= 1u << (mt * 4 + h * 2 + cq);
                        }
                    }
                }
            }
            pending &= valid;
            if (ct.debug == 1) {
                // debug: every filter prune must agree with the exact prefix
                uint32_t pruned = valid & ~pending;
                while (pruned) {
                    const int b = __ffs(pruned) - 1;
                    pruned &= pruned - 1;
                    const uint32_t row = (b >> 2) * 16 + ((b >> 1) & 1) * 8 + g;
                    const int j = warp * 8 + 2 * tq + (b & 1);
                    float xx = 0.f;
                    for (int cc = 0; cc < c_dense; ++cc) {
                        const float* bc = slot_o((s - (c_dense - 1) + cc) % n_buf);
                        const uint32_t lo = cc == 0 ? 0u : ct.end[cc - 1], hi = ct.end[cc];
                        for (uint32_t k = lo; k < hi; ++k) xx = sq_step(xx, bc[swz(row, k - lo)], q_res[k * kQS + j]);
                    }
                    if (!(xx > thr_s[j * n_ckpt + ck])) atomicAdd(a.counters + 3, 1ull);
                }
            }
            if (ct.debug == 2) pending = 0;  // experiment: filter only
            if (ct.debug == 3) {             // census: pairs kept by the filter
                const uint32_t v = __reduce_add_sync(0xffffffffu, __popc(pending));
                if (lane == 0) atomicAdd(a.counters + 5, (unsigned long long)v);
            }
            st_dims += (unsigned long long)__popc(valid & ~pending) * d0;
        } else if (has_sparse) {
            uint32_t dead = 0;
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const float th = thr_s[(warp * 8 + jj) * n_ckpt + ck];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint64_t v = acc[i][jj >> 1];
                    const float x = (jj & 1) ? hi_f(v) : lo_f(v);
                    if (x > th) dead |= 1u << (i * 8 + jj);
                }
            }
            dead &= alive;
            st_dims += (unsigned long long)__popc(dead) * ct.end[c];
            if (a.measure) {
                pre_pruned = dead;  // carried to the full dim for their exact distance
            } else {
                alive &= ~dead;
            }
            pending = alive;
        } else {
            // FD: candidates straight from registers, one query at a time
            st_dims += (unsigned long long)__popc(alive) * dim;
            uint32_t cand = 0;
            // (FD never prunes early: with failure accounting, eligible = the accepted pairs)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj) {
                const float r = r_s[warp * 8 + jj];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const uint64_t v = acc[i][jj >> 1];
                    const float x = (jj & 1) ? hi_f(v) : lo_f(v);
                    const float key = kSqrtKey ? __fsqrt_rn(x) : x;
                    if (((alive >> (i * 8 + jj)) & 1u) && !(key > r)) cand |= 1u << (i * 8 + jj);
                }
            }
            if (a.measure) st_elig += __popc(cand);
            if (__any_sync(0xffffffffu, cand != 0)) {
                for (int jj = 0; jj < 8; ++jj) {
                    const uint32_t j = warp * 8 + jj;
                    uint32_t m = 0;
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const bool is = (cand >> (i * 8 + jj)) & 1u;
                        const uint32_t bal = __ballot_sync(0xffffffffu, is);
                        if (is) {
                            const uint64_t v = acc[i][jj >> 1];
                            const float x = (jj & 1) ? hi_f(v) : lo_f(v);
                            const uint32_t gr = row_base + lane + 32 * i;
                            const uint32_t id = a.row_ids ? __ldg(a.row_ids + gr) : a.id_base + gr;
                            kb[m + __popc(bal & ((1u << lane) - 1u))] = make_key(kSqrtKey ? __fsqrt_rn(x) : x, id);
                        }
                        m += __popc(bal);
                    }
                    __syncwarp();
                    if (m) {
                        if (a.row_ids && lane == 0) st_bytes += 4ull * m;
                        merge_query(a, kb, m, j, qidx_s, slot_s, r_s, thr_s, n_ckpt, lane, ms);
                    }
                }
            }
            continue;
        }

        PH_MARK(t_e1);
        PH_ADD(2, t_d1, t_e1);
        // ---- survivors of the first checkpoint -----------------------------------
        // advance(list, n): one pair per lane from chunk c_dense on, straight
        // from L2 (each chunk one round trip), marking final candidates.
        bool merged = false;  // did this warp merge candidates in this tile?
        auto advance = [&](uint32_t* lm, float* la, uint32_t n) {
            merged = true;
            for (uint32_t e = lane; e < n; e += 32) {
                const uint32_t meta = lm[e];
                float x = la[e];
                const uint32_t row = meta & 0x7fu, jj = (meta >> 8) & 0xffu, j = warp * 8 + jj;
                bool live = true;
                bool pruned = (meta & 0x80u) != 0;  // failure accounting: pruned at the first checkpoint
                const float* orow = a.storage + (size_t)(row_base + row) * dim;
                const float* qrow = a.queries + (size_t)qidx_s[j] * dim;
                for (int cc = c_dense; cc < ct.n_chunks; ++cc) {
                    const uint32_t lo = ct.end[cc - 1], hi = ct.end[cc];
                    if (vec && hi - lo == (uint32_t)kCH) {
                        float4 o8[kCH / 4], q8[kCH / 4];
#pragma unroll
                        for (int v = 0; v < kCH / 4; ++v) {
                            o8[v] = __ldg(reinterpret_cast<const float4*>(orow + lo) + v);
                            q8[v] = __ldg(reinterpret_cast<const float4*>(qrow + lo) + v);
                        }
#pragma unroll
                        for (int v = 0; v < kCH / 4; ++v) {
                            x = sq_step(x, o8[v].x, q8[v].x);
                            x = sq_step(x, o8[v].y, q8[v].y);
                            x = sq_step(x, o8[v].z, q8[v].z);
                            x = sq_step(x, o8[v].w, q8[v].w);
                        }
                    } else if (vec) {
                        for (uint32_t kk = lo; kk < hi; kk += 4) {
                            const float4 o4 = __ldg(reinterpret_cast<const float4*>(orow + kk));
                            const float4 q4 = __ldg(reinterpret_cast<const float4*>(qrow + kk));
                            x = sq_step(x, o4.x, q4.x);
                            x = sq_step(x, o4.y, q4.y);
                            x = sq_step(x, o4.z, q4.z);
                            x = sq_step(x, o4.w, q4.w);
                        }
                    } else {
                        for (uint32_t kk = lo; kk < hi; ++kk) x = sq_step(x, __ldg(orow + kk), __ldg(qrow + kk));
                    }
                    st_bytes += 8ull * (hi - lo);
                    const int k2 = ct.ckpt[cc];
                    if (k2 >= 0 && !pruned && x > thr_s[j * n_ckpt + k2]) {
                        st_dims += hi;
                        if (a.measure) {
                            pruned = true;
                        } else {
                            live = false;
                            break;
                        }
                    }
                }
                bool is_cand = false;
                if (live && pruned) {  // record_failure_check (proj/src/estimator.cpp:24-33)
                    if (__fsqrt_rn(x) <= r_s[j]) {
                        ++st_elig;
                        ++st_fail;
                    }
                } else if (live) {
                    st_dims += dim;
                    const float key = kSqrtKey ? __fsqrt_rn(x) : x;
                    is_cand = !(key > r_s[j]);
                    if (a.measure && is_cand) ++st_elig;
                    x = key;
                }
                lm[e] = meta | (is_cand ? 0x80000000u : 0u);
                la[e] = x;
            }
            __syncwarp();
            merge_list_candidates(a, lm, la, n, kb, row_base, warp, lane, qidx_s, slot_s, r_s, thr_s, n_ckpt,
                                  st_bytes, ms);
        };

        // Streaming mode: append the s2 list to the global survivor worklist for
        // advance_survivors_kernel (no L2 chains or merges inside this kernel);
        // when the worklist is full, advance the pairs here instead.
        auto emit_or_advance = [&](uint32_t n2) {
            bool ok = false;
            if (a.surv) {
                uint32_t base = 0;
                if (lane == 0) base = atomicAdd(a.surv_count, n2);
                base = __shfl_sync(0xffffffffu, base, 0);
                ok = base + n2 <= a.surv_cap;
                for (uint32_t e = lane; e < n2; e += 32) {
                    if (base + e >= a.surv_cap) continue;
                    Survivor v;
                    const uint32_t meta = s2_meta[e];
                    const uint32_t j = warp * 8 + ((meta >> 8) & 0xffu);
                    v.q = ok ? qidx_s[j] : 0xffffffffu;  // a partial append is voided
                    v.row = row_base + (meta & 0xffu);
                    v.acc = s2_acc[e];
                    v.slot = slot_s[j];
                    a.surv[base + e] = v;
                }
                if (ok) st_bytes += 16ull * n2;
            }
            if (!ok) advance(s2_meta, s2_acc, n2);
        };

        if constexpr (kTC) {
            // stage 1: exact dense prefix of every pair the filter kept (from the
            // resident boxes), survivors of the checkpoint into the s2 list ...
            uint32_t n2 = 0;
            while (__any_sync(0xffffffffu, pending != 0)) {
                PH_MARK(t_r0);
                const uint32_t n = compact_round(
                    pending, wl_meta, wl_acc, lane,
                    [&](int b, uint32_t& row, uint32_t& jj) {
                        row = (b >> 2) * 16 + ((b >> 1) & 1) * 8 + g;
                        jj = 2 * tq + (b & 1);
                    },
                    [&](int) { return 0.f; });
                for (uint32_t e0 = 0; e0 < n; e0 += 32) {
                    const uint32_t e = e0 + lane;
                    bool keep = false;
                    uint32_t meta = 0;
                    float x = 0.f;
                    if (e < n) {
                        meta = wl_meta[e];
                        const uint32_t row = meta & 0xffu, j = warp * 8 + ((meta >> 8) & 0xffu);
                        for (int cc = 0; cc < c_dense; ++cc) {
                            const float* bc = slot_o((s - (c_dense - 1) + cc) % n_buf);
                            const uint32_t lo = cc == 0 ? 0u : ct.end[cc - 1], hi = ct.end[cc];
                            for (uint32_t k = lo; k < hi; k += 4) {
                                const float4 o4 = *reinterpret_cast<const float4*>(bc + swz(row, k - lo));
                                x = sq_step(x, o4.x, q_res[(k + 0) * kQS + j]);
                                x = sq_step(x, o4.y, q_res[(k + 1) * kQS + j]);
                                x = sq_step(x, o4.z, q_res[(k + 2) * kQS + j]);
                                x = sq_step(x, o4.w, q_res[(k + 3) * kQS + j]);
                            }
                        }
                        keep = !(x > thr_s[j * n_ckpt + ck]);
                        if (!keep) st_dims += d0;
                    }
                    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                    if (n2 + __popc(bal) > (uint32_t)kWarpList) {  // s2 full: drain it now
                        emit_or_advance(n2);
                        n2 = 0;
                    }
                    if (keep) {
                        const uint32_t pos = n2 + __popc(bal & ((1u << lane) - 1u));
                        s2_meta[pos] = meta;
                        s2_acc[pos] = x;
                    }
                    n2 += __popc(bal);
                    __syncwarp();
                }
                PH_MARK(t_r1);
                PH_ADD(3, t_r0, t_r1);
            }
            // ... release the tile's boxes (the producer can refill them while
            // this warp waits on L2), then stage 2
            __syncwarp();
            if (lane == 0)
                for (int cc = 0; cc < c_dense; ++cc) mbar_arrive(empty_bar + (s - (c_dense - 1) + cc) % n_buf);
            PH_MARK(t_r2);
            if (ct.debug == 3 && lane == 0) atomicAdd(a.counters + 6, (unsigned long long)n2);
            if (n2) emit_or_advance(n2);
            PH_MARK(t_r3);
            PH_ADD(4, t_r2, t_r3);
        } else {
            while (__any_sync(0xffffffffu, pending != 0)) {
                const uint32_t n = compact_round(
                    pending, wl_meta, wl_acc, lane,
                    [&](int b, uint32_t& row, uint32_t& jj) {
                        row = (lane + 32 * (b >> 3)) | (((pre_pruned >> b) & 1u) << 7);
                        jj = b & 7;
                    },
                    [&](int b) {
                        const uint64_t v = acc[b >> 3][(b & 7) >> 1];
                        return (b & 1) ? hi_f(v) : lo_f(v);
                    });
                advance(wl_meta, wl_acc, n);
            }
        }
        if (merged) tighten_warp_radii(a, warp, lane, my_q, qidx_s, slot_s, r_s, thr_s, n_ckpt);
    }  // steps

    // ---- counters -------------------------------------------------------------
    unsigned long long v0 = st_dco, v1 = st_dims, v2 = st_bytes;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        v0 += __shfl_xor_sync(0xffffffffu, v0, off);
        v1 += __shfl_xor_sync(0xffffffffu, v1, off);
        v2 += __shfl_xor_sync(0xffffffffu, v2, off);
    }
    if (a.measure && a.counters) {
        unsigned long long e = st_elig, f = st_fail;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            e += __shfl_xor_sync(0xffffffffu, e, off);
            f += __shfl_xor_sync(0xffffffffu, f, off);
        }
        if (lane == 0 && e) atomicAdd(a.counters + 8, e);
        if (lane == 0 && f) atomicAdd(a.counters + 9, f);
    }
    if (lane == 0 && a.counters) {
        atomicAdd(a.counters + 0, v0);
        atomicAdd(a.counters + 1, v1);
        atomicAdd(a.counters + 2, v2);
    }
}

// ---- stage 2 of the streaming scan: first-checkpoint survivors ------------------
// Continue each survivor's exact accumulation from d0 through the remaining
// checkpoints (checkpointed_scan, proj/src/estimator.cpp:39-70) against its
// query's radius; exact full-D distances <= r become (query, key) candidates.
// A warp takes 32 survivors (lane = survivor) and walks the dims in chunks of
// <= 32: the live survivors' row and query chunks are staged in shared memory
// with coalesced loads (8 lanes per 128-byte row chunk), then every lane
// advances its own sequential sum from shared memory. (A thread reading its
// own row from global would touch 32 lines per warp load.)
constexpr int kSvStride = 36;  // floats per staged row: 16-byte aligned, conflict-free LDS.128
constexpr int kSvWarps = 8;

__global__ void __launch_bounds__(kSvWarps * 32, 2) advance_survivors_kernel(const SurvArgs a) {
    extern __shared__ __align__(16) float sv_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* o_s = sv_smem + (size_t)warp * 2 * 32 * kSvStride;
    float* q_s = o_s + 32 * kSvStride;
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.surv_max) atomicMax(a.surv_max, *a.surv_count);
    const uint32_t n = min(*a.surv_count, a.surv_cap);
    const uint32_t n_groups = (n + 31) / 32;
    const uint32_t dim = a.dim;
    for (uint32_t grp = blockIdx.x * kSvWarps + warp; grp < n_groups; grp += gridDim.x * kSvWarps) {
        const uint32_t i = grp * 32 + lane;
        bool live = false, flagged = false;
        uint32_t q = 0, row = 0;
        float x = 0.f, r = 0.f;
        if (i < n) {
            const Survivor v = a.surv[i];
            if (v.q != 0xffffffffu) {
                live = true;
                flagged = (v.slot >> 31) != 0;  // debug: a pair the filter's bound pruned
                q = v.q;
                row = v.row;
                x = v.acc;
                r = __uint_as_float(a.r_global[q]);
            }
        }
        unsigned long long viol = 0;
        unsigned long long dims = 0;
        uint32_t lo = a.n_dense_dims;
        for (uint32_t ci = a.first_ckpt; ci <= a.n_ckpt; ++ci) {
            const uint32_t act0 = __ballot_sync(0xffffffffu, live);
            if (!act0) break;
            const uint32_t hi = ci < a.n_ckpt ? a.cps[ci] : dim;
            for (uint32_t k0 = lo; k0 < hi; k0 += 32) {
                const uint32_t w = min(32u, hi - k0);
                if (a.vec4 && (w & 3u) == 0) {
                    // 4 survivors per pass: lane = (survivor sub 0..3, 16-byte column 0..7)
                    const uint32_t sub = lane >> 3, c4 = lane & 7;
                    // all loads in flight before the first store: one memory latency per chunk
                    float4 ov[8], qv[8];
                    bool okv[8];
#pragma unroll
                    for (uint32_t sg = 0; sg < 8; ++sg) {
                        const uint32_t sidx = 4 * sg + sub;
                        const uint32_t srow = __shfl_sync(0xffffffffu, row, sidx);
                        const uint32_t sq = __shfl_sync(0xffffffffu, q, sidx);
                        okv[sg] = ((act0 >> sidx) & 1u) && 4 * c4 < w;
                        if (okv[sg]) {
                            ov[sg] = __ldg(reinterpret_cast<const float4*>(a.storage + (size_t)srow * dim + k0) + c4);
                            qv[sg] = __ldg(reinterpret_cast<const float4*>(a.queries + (size_t)sq * dim + k0) + c4);
                        }
                    }
#pragma unroll
                    for (uint32_t sg = 0; sg < 8; ++sg) {
                        const uint32_t sidx = 4 * sg + sub;
                        if (okv[sg]) {
                            *reinterpret_cast<float4*>(o_s + sidx * kSvStride + 4 * c4) = ov[sg];
                            *reinterpret_cast<float4*>(q_s + sidx * kSvStride + 4 * c4) = qv[sg];
                        }
                    }
                    __syncwarp();
                    if (live) {
                        const float* os = o_s + lane * kSvStride;
                        const float* qs = q_s + lane * kSvStride;
                        for (uint32_t k = 0; k < w; k += 4) {
                            const float4 o4 = *reinterpret_cast<const float4*>(os + k);
                            const float4 q4 = *reinterpret_cast<const float4*>(qs + k);
                            x = sq_step(x, o4.x, q4.x);
                            x = sq_step(x, o4.y, q4.y);
                            x = sq_step(x, o4.z, q4.z);
                            x = sq_step(x, o4.w, q4.w);
                        }
                    }
                } else {
                    // any alignment: one survivor per pass, lane = dim
                    for (uint32_t m = act0; m; m &= m - 1) {
                        const uint32_t sidx = __ffs(m) - 1;
                        const uint32_t srow = __shfl_sync(0xffffffffu, row, sidx);
                        const uint32_t sq = __shfl_sync(0xffffffffu, q, sidx);
                        if ((uint32_t)lane < w) {
                            o_s[sidx * kSvStride + lane] = __ldg(a.storage + (size_t)srow * dim + k0 + lane);
                            q_s[sidx * kSvStride + lane] = __ldg(a.queries + (size_t)sq * dim + k0 + lane);
                        }
                    }
                    __syncwarp();
                    if (live)
                        for (uint32_t k = 0; k < w; ++k)
                            x = sq_step(x, o_s[lane * kSvStride + k], q_s[lane * kSvStride + k]);
                }
                __syncwarp();  // staging buffers free for the next chunk
            }
            lo = hi;
            if (live && ci < a.n_ckpt) {
                const bool pr = x > prune_threshold(a.coeff[ci], r);
                if (flagged) {  // the exact prefix must agree with the bound; then drop it as the filter would
                    viol += pr ? 0 : 1;
                    live = false;
                } else if (pr) {
                    dims += hi;
                    live = false;
                }
            }
        }
        bool is_cand = false;
        uint64_t key = 0;
        if (live) {
            dims += dim;
            const float key_d = __fsqrt_rn(x);
            if (!(key_d > r)) {
                is_cand = true;
                const uint32_t id = a.row_ids ? __ldg(a.row_ids + row) : a.id_base + row;
                key = make_key(key_d, id);
            }
        }
        if (a.qslots) {  // per-query slots; the rare overflow to the shared list
            if (a.cand_total) {
                const uint32_t nb = __popc(__ballot_sync(0xffffffffu, is_cand));
                if (lane == 0 && nb) atomicAdd(a.cand_total, nb);
            }
            if (is_cand) {
                const uint32_t slot = atomicAdd(a.q_count + q, 1u);
                if (slot < a.qslot_cap) {
                    a.qslots[(size_t)q * a.qslot_cap + slot] = key;
                } else {
                    const uint32_t pos = atomicAdd(a.cand_count, 1u);
                    if (pos < a.cand_cap) {
                        a.cand_q[pos] = q;
                        a.cand_key[pos] = key;
                    }
                }
            }
        } else if (const uint32_t bal = __ballot_sync(0xffffffffu, is_cand)) {  // warp-aggregated append
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(a.cand_count, __popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (is_cand) {
                const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
                if (pos < a.cand_cap) {
                    a.cand_q[pos] = q;
                    a.cand_key[pos] = key;
                    atomicAdd(a.q_count + q, 1u);
                }
            }
        }
        for (int off = 16; off > 0; off >>= 1) {
            dims += __shfl_xor_sync(0xffffffffu, dims, off);
            viol += __shfl_xor_sync(0xffffffffu, viol, off);
        }
        if (lane == 0 && a.counters && dims) atomicAdd(a.counters + 1, dims);
        if (lane == 0 && a.counters && viol) atomicAdd(a.counters + 3, viol);
    }
}

// Pipelined variant for dim, d0 and every checkpoint multiples of 4 (the
// streaming path's rule): row chunks go global -> shared with cp.async (no
// register staging, so three CTAs fit per SM) and the next chunk of the live
// survivors is in flight while the current one is accumulated. Survivors come
// out of the filters grouped by query, so when a warp's 32 survivors share one
// query its chunk is staged once (else each lane reads its own from L1/L2).
constexpr int kSpWarps = 8;
constexpr int kSpRS = 36;                              // floats per staged row chunk
constexpr int kSpWarpFloats = 2 * 32 * kSpRS + 2 * 32;  // rows[2][32][36] + q[2][32]

__device__ __forceinline__ void sp_cp16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
                 "l"(src)
                 : "memory");
}

// One evaluated checkpoint partial into the estimate dump (parity tests).
__device__ __forceinline__ void dump_partial(const SurvArgs& a, uint32_t q, uint32_t row, uint32_t ci, float x) {
    const uint32_t p = atomicAdd(a.dump.count, 1u);
    if (p < a.dump.cap)
        a.dump.entries[p] = make_uint4(q, a.row_ids ? __ldg(a.row_ids + row) : a.id_base + row, ci, __float_as_uint(x));
}

__global__ void __launch_bounds__(kSpWarps * 32, 3) advance_survivors_pipe_kernel(const SurvArgs a) {
    extern __shared__ __align__(16) float sp_smem[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* rbuf = sp_smem + (size_t)warp * kSpWarpFloats;  // [2][32][kSpRS]
    float* qbuf = rbuf + 2 * 32 * kSpRS;                   // [2][32]
    if (blockIdx.x == 0 && threadIdx.x == 0 && a.surv_max) atomicMax(a.surv_max, *a.surv_count);
    const uint32_t n = min(*a.surv_count, a.surv_cap);
    const uint32_t n_groups = (n + 31) / 32;
    const uint32_t dim = a.dim, n_ckpt = a.n_ckpt;
    auto hi_of = [&](uint32_t ci) -> uint32_t { return ci < n_ckpt ? (uint32_t)a.cps[ci] : dim; };
    for (uint32_t grp = blockIdx.x * kSpWarps + warp; grp < n_groups; grp += gridDim.x * kSpWarps) {
        const uint32_t i = grp * 32 + lane;
        bool live = false, flagged = false;
        bool pruned = false;  // failure accounting: decided, still accumulating to the full dim
        uint32_t q = 0, row = 0;
        float x = 0.f, r = 0.f;
        if (i < n) {
            const Survivor v = a.surv[i];
            if (v.q != 0xffffffffu) {
                live = true;
                flagged = (v.slot >> 31) != 0;  // debug: a pair the filter's bound pruned
                q = v.q;
                row = v.row;
                x = v.acc;
                r = __uint_as_float(a.r_global[q]);
            }
        }
        uint32_t act = __ballot_sync(0xffffffffu, live);
        unsigned long long dims = 0, viol = 0, elig = 0, fails = 0;
        if (act) {
            const uint32_t q0 = __shfl_sync(0xffffffffu, q, __ffs(act) - 1);
            const bool qsame = __all_sync(0xffffffffu, !live || q == q0);
            const float* qrow = a.queries + (size_t)q * dim;
            auto issue = [&](uint32_t ci, uint32_t k0, uint32_t buf, uint32_t mask) {
                const uint32_t w = min(32u, hi_of(ci) - k0);
                const uint32_t sub = lane >> 3, c4 = lane & 7;
                float* rb = rbuf + buf * 32 * kSpRS;
#pragma unroll
                for (uint32_t sg = 0; sg < 8; ++sg) {
                    const uint32_t sidx = 4 * sg + sub;
                    const uint32_t srow = __shfl_sync(0xffffffffu, row, sidx);
                    if (((mask >> sidx) & 1u) && 4 * c4 < w)
                        sp_cp16(rb + sidx * kSpRS + 4 * c4, a.storage + (size_t)srow * dim + k0 + 4 * c4);
                }
                if (qsame && lane < 8 && 4u * lane < w)
                    sp_cp16(qbuf + buf * 32 + 4 * lane, a.queries + (size_t)q0 * dim + k0 + 4 * lane);
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            };
            uint32_t ci = a.first_ckpt, k0 = a.n_dense_dims, buf = 0;
            issue(ci, k0, 0, act);
            for (;;) {
                const uint32_t hi = hi_of(ci);
                const uint32_t w = min(32u, hi - k0);
                uint32_t nci = ci, nk0 = k0 + 32;
                if (nk0 >= hi) {
                    nci = ci + 1;
                    nk0 = hi;
                }
                const bool has_next = nci <= n_ckpt && nk0 < dim;
                if (has_next) issue(nci, nk0, buf ^ 1, act);  // speculative: the live set of now
                // this lane's query chunk (when the warp's queries differ): eight 16-byte
                // loads issued before the wait on the row chunk
                float4 qv[8];
                if (live && !qsame) {
#pragma unroll
                    for (uint32_t j = 0; j < 8; ++j)
                        if (4 * j < w) qv[j] = __ldg(reinterpret_cast<const float4*>(qrow + k0) + j);
                }
                if (has_next) asm volatile("cp.async.wait_group 1;\n" ::: "memory");
                else asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                __syncwarp();
                if (live) {
                    const float* os = rbuf + buf * 32 * kSpRS + lane * kSpRS;
                    if (qsame) {
                        const float* qs = qbuf + buf * 32;
                        for (uint32_t k = 0; k < w; k += 4) {
                            const float4 o4 = *reinterpret_cast<const float4*>(os + k);
                            const float4 q4 = *reinterpret_cast<const float4*>(qs + k);
                            x = sq_step(x, o4.x, q4.x);
                            x = sq_step(x, o4.y, q4.y);
                            x = sq_step(x, o4.z, q4.z);
                            x = sq_step(x, o4.w, q4.w);
                        }
                    } else {
#pragma unroll
                        for (uint32_t j = 0; j < 8; ++j) {
                            if (4 * j >= w) break;
                            const float4 o4 = *reinterpret_cast<const float4*>(os + 4 * j);
                            x = sq_step(x, o4.x, qv[j].x);
                            x = sq_step(x, o4.y, qv[j].y);
                            x = sq_step(x, o4.z, qv[j].z);
                            x = sq_step(x, o4.w, qv[j].w);
                        }
                    }
                }
                __syncwarp();  // buffer `buf` free for the chunk after next
                if (k0 + w == hi && ci < n_ckpt && live && !pruned) {
                    // checkpointed_scan's test (proj/src/estimator.cpp:46-60) against this pair's radius
                    const bool pr = x > prune_threshold(a.coeff[ci], r);
                    if (a.dump.entries) dump_partial(a, q, row, ci, x);
                    if (flagged) {  // the exact prefix must agree with the bound; then drop it as the filter would
                        viol += pr ? 0 : 1;
                        if (a.measure) pruned = true;
                        else live = false;
                    } else if (pr) {
                        dims += hi;
                        if (a.row_dims) atomicMax(a.row_dims + row, hi);
                        if (a.measure) pruned = true;
                        else live = false;
                    }
                }
                act = __ballot_sync(0xffffffffu, live);
                if (!has_next || !act) {
                    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
                    break;
                }
                ci = nci;
                k0 = nk0;
                buf ^= 1;
            }
        }
        bool is_cand = false;
        uint64_t key = 0;
        if (live && pruned) {
            // record_failure_check (proj/src/estimator.cpp:24-33): x continued the scan's own
            // accumulator to the full dim, so it is the exact distance a full scan gives
            if (__fsqrt_rn(x) <= r) {
                ++elig;
                ++fails;
            }
        } else if (live) {
            dims += dim;
            if (a.row_dims) atomicMax(a.row_dims + row, dim);
            const float key_d = __fsqrt_rn(x);
            if (!(key_d > r)) {
                is_cand = true;
                elig += a.measure ? 1 : 0;
                const uint32_t id = a.row_ids ? __ldg(a.row_ids + row) : a.id_base + row;
                key = make_key(key_d, id);
            }
        }
        if (a.qslots) {  // per-query slots; the rare overflow to the shared list
            if (a.cand_total) {
                const uint32_t nb = __popc(__ballot_sync(0xffffffffu, is_cand));
                if (lane == 0 && nb) atomicAdd(a.cand_total, nb);
            }
            if (is_cand) {
                const uint32_t slot = atomicAdd(a.q_count + q, 1u);
                if (slot < a.qslot_cap) {
                    a.qslots[(size_t)q * a.qslot_cap + slot] = key;
                } else {
                    const uint32_t pos = atomicAdd(a.cand_count, 1u);
                    if (pos < a.cand_cap) {
                        a.cand_q[pos] = q;
                        a.cand_key[pos] = key;
                    }
                }
            }
        } else if (const uint32_t bal = __ballot_sync(0xffffffffu, is_cand)) {
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(a.cand_count, __popc(bal));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (is_cand) {
                const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
                if (pos < a.cand_cap) {
                    a.cand_q[pos] = q;
                    a.cand_key[pos] = key;
                    atomicAdd(a.q_count + q, 1u);
                }
            }
        }
        for (int off = 16; off > 0; off >>= 1) {
            dims += __shfl_xor_sync(0xffffffffu, dims, off);
            viol += __shfl_xor_sync(0xffffffffu, viol, off);
        }
        if (lane == 0 && a.counters && dims) {
            atomicAdd(a.counters + 1, dims);
            atomicAdd(a.counters + 2, 4ull * dims);  // each pair's row chunks from dim 0 (B_read)
        }
        if (lane == 0 && a.counters && viol) atomicAdd(a.counters + 3, viol);
        if (a.measure && a.counters) {
            for (int off = 16; off > 0; off >>= 1) {
                elig += __shfl_xor_sync(0xffffffffu, elig, off);
                fails += __shfl_xor_sync(0xffffffffu, fails, off);
            }
            if (lane == 0 && elig) atomicAdd(a.counters + 8, elig);
            if (lane == 0 && fails) atomicAdd(a.counters + 9, fails);
        }
    }
}

// Merge each query's slot candidates into its top-K (out_keys already holds the
// earlier passes' results); a query whose slots overflowed also picks its entries
// out of the shared overflow list. Unsorted 256-key batches, warp per query.
__global__ void __launch_bounds__(128)
merge_slots_kernel(const uint64_t* __restrict__ qslots, uint32_t cap, const uint32_t* __restrict__ q_count,
                   const uint32_t* __restrict__ cand_q, const uint64_t* __restrict__ cand_key,
                   const uint32_t* __restrict__ cand_count, uint32_t cand_cap, uint32_t nq, uint32_t K,
                   uint64_t* out_keys, uint32_t* out_count, uint32_t* r_global, uint32_t* res_ids,
                   float* res_dists, uint32_t* res_counts) {
    __shared__ uint64_t bbuf[4][256];
    __shared__ uint64_t abuf[4][kStageMaxK];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * 4 + warp;
    if (q >= nq) return;
    uint64_t* A = out_keys + (size_t)q * K;
    uint32_t* cA = out_count + q;
    const uint32_t cnt = q_count[q];
    uint64_t* B = bbuf[warp];
    auto merge = [&](uint32_t m) {
        __syncwarp();
        if (K <= (uint32_t)kStageMaxK) {
            if (m > 32) warp_merge_sortb(A, cA, K, B, m, abuf[warp]);
            else warp_merge_staged(A, cA, K, B, m, abuf[warp]);
        } else {
            warp_merge(A, cA, K, B, m, false);
        }
        __syncwarp();
    };
    const uint64_t* src = qslots + (size_t)q * cap;
    const uint32_t m_slots = min(cnt, cap);
    for (uint32_t b0 = 0; b0 < m_slots; b0 += 256) {
        const uint32_t m = min(256u, m_slots - b0);
        for (uint32_t e = lane; e < m; e += 32) B[e] = src[b0 + e];
        merge(m);
    }
    if (cnt > cap) {
        const uint32_t n_ovf = min(*cand_count, cand_cap);
        uint32_t nb = 0;
        for (uint32_t i0 = 0; i0 < n_ovf; i0 += 32) {
            const uint32_t i = i0 + lane;
            const bool mine = i < n_ovf && cand_q[i] == q;
            const uint32_t bal = __ballot_sync(0xffffffffu, mine);
            if (mine) B[nb + __popc(bal & ((1u << lane) - 1u))] = cand_key[i];
            nb += __popc(bal);
            if (nb > 224 || (i0 + 32 >= n_ovf && nb)) {
                merge(nb);
                nb = 0;
            }
        }
    }
    const uint32_t c = *reinterpret_cast<volatile uint32_t*>(cA);
    for (uint32_t i = c + lane; i < K; i += 32) A[i] = kEmptyKey;
    // tighten the radius to the K-th key for the next pass (tighten_from_topk_kernel, fused)
    if (r_global && lane == 0 && c >= K) atomicMin(r_global + q, (uint32_t)(A[K - 1] >> 32));
    if (res_ids) {  // the search's last merge: ids / dists / count (keys_to_results_kernel, fused)
        __syncwarp();
        for (uint32_t i = lane; i < K; i += 32) {
            const uint64_t v = A[i];
            res_ids[(size_t)q * K + i] = i < c ? (uint32_t)v : 0xffffffffu;
            res_dists[(size_t)q * K + i] = i < c ? __uint_as_float((uint32_t)(v >> 32)) : __int_as_float(0x7f800000);
        }
        if (lane == 0 && res_counts) res_counts[q] = c;
    }
}

// Final per-query merge of n_slots segments into out_keys [nq x K] (K5).
// One warp per query.
__global__ void __launch_bounds__(128)
merge_segments_kernel(const uint64_t* __restrict__ seg_keys, const uint32_t* __restrict__ seg_count,
                      uint32_t nq, uint32_t n_slots, uint32_t K, uint64_t* out_keys,
                      uint32_t* out_count) {
    __shared__ uint64_t bbuf[4][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * 4 + warp;
    if (q >= nq) return;
    uint64_t* A = out_keys + (size_t)q * K;
    uint32_t* cA = out_count + q;
    if (lane == 0) *cA = 0;
    __syncwarp();
    uint64_t* B = bbuf[warp];
    for (uint32_t s = 0; s < n_slots; ++s) {
        const size_t seg = (size_t)q * n_slots + s;
        const uint32_t cnt = seg_count[seg];
        const uint64_t* src = seg_keys + seg * K;
        for (uint32_t b0 = 0; b0 < cnt; b0 += 256) {
            const uint32_t m = min(256u, cnt - b0);
            const uint32_t cur = *reinterpret_cast<volatile uint32_t*>(cA);
            if (cur == K && src[b0] > A[K - 1]) break;  // batch starts above a full list's worst
            for (uint32_t e = lane; e < m; e += 32) B[e] = src[b0 + e];
            __syncwarp();
            warp_merge(A, cA, K, B, m, true);
            __syncwarp();
        }
    }
    const uint32_t c = *reinterpret_cast<volatile uint32_t*>(cA);
    for (uint32_t i = c + lane; i < K; i += 32) A[i] = kEmptyKey;
}

// Merge G key blocks [G x nq x K] (sorted per query, kEmptyKey padded).
__global__ void __launch_bounds__(128)
merge_blocks_kernel(const uint64_t* __restrict__ keys, uint32_t G, uint32_t nq, uint32_t K,
                    uint64_t* out_keys, uint32_t* out_count) {
    __shared__ uint64_t bbuf[4][256];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t q = blockIdx.x * 4 + warp;
    if (q >= nq) return;
    uint64_t* A = out_keys + (size_t)q * K;
    uint32_t* cA = out_count + q;
    if (lane == 0) *cA = 0;
    __syncwarp();
    uint64_t* B = bbuf[warp];
    for (uint32_t g = 0; g < G; ++g) {
        const uint64_t* src = keys + ((size_t)g * nq + q) * K;
        for (uint32_t b0 = 0; b0 < K; b0 += 256) {
            const uint32_t m0 = min(256u, K - b0);
            uint32_t nonempty = 0;
            for (uint32_t e = lane; e < m0; e += 32) {
                const uint64_t v = src[b0 + e];
                B[e] = v;
                nonempty += v != kEmptyKey;
            }
            __syncwarp();
            const uint32_t m = __reduce_add_sync(0xffffffffu, nonempty);
            if (m == 0) break;
            warp_merge(A, cA, K, B, m, true);
            __syncwarp();
            if (m < m0) break;
        }
    }
    const uint32_t c = *reinterpret_cast<volatile uint32_t*>(cA);
    for (uint32_t i = c + lane; i < K; i += 32) A[i] = kEmptyKey;
}

__global__ void keys_to_results_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ count,
                                       uint32_t nq, uint32_t K, uint32_t* ids, float* dists,
                                       uint32_t* counts_out) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)nq * K) return;
    const uint32_t q = (uint32_t)(i / K), e = (uint32_t)(i - (size_t)q * K);
    const uint32_t c = count[q];
    const uint64_t v = keys[i];
    if (e < c) {
        ids[i] = (uint32_t)v;
        dists[i] = __uint_as_float((uint32_t)(v >> 32));
    } else {
        ids[i] = 0xffffffffu;
        dists[i] = __int_as_float(0x7f800000);
    }
    if (e == 0 && counts_out) counts_out[q] = c;
}

}  // namespace

size_t scan_smem_bytes(int n_ckpt, int d_res, int n_buf) { return smem_layout(n_ckpt, d_res, n_buf).total; }

template <bool kSqrtKey, bool kTC>
static cudaError_t launch_scan_t(const ScanArgs& a, const ChunkTable& ct, const CUtensorMap& tm,
                                 const CUtensorMap& tn, uint32_t grid, size_t smem, cudaStream_t s) {
    DADE_CUDA_TRY(cudaFuncSetAttribute(dco_scan_kernel<kSqrtKey, kTC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem));
    dco_scan_kernel<kSqrtKey, kTC><<<grid, kThreadsTotal, smem, s>>>(a, ct, tm, tn);
    return cudaGetLastError();
}

cudaError_t launch_scan(const ScanArgs& a, const ChunkTable& ct, const CUtensorMap& tm, const CUtensorMap& tn,
                        uint32_t grid, bool sqrt_key, cudaStream_t s) {
    if (grid == 0) return cudaSuccess;
    const size_t smem = scan_smem_bytes(ct.n_ckpt, ct.d_res, ct.n_buf);
    if (sqrt_key) return ct.use_tc ? launch_scan_t<true, true>(a, ct, tm, tn, grid, smem, s)
                                   : launch_scan_t<true, false>(a, ct, tm, tn, grid, smem, s);
    return ct.use_tc ? launch_scan_t<false, true>(a, ct, tm, tn, grid, smem, s)
                     : launch_scan_t<false, false>(a, ct, tm, tn, grid, smem, s);
}

cudaError_t launch_advance_survivors(const SurvArgs& a, uint32_t max_entries, cudaStream_t s) {
    if (max_entries == 0) return cudaSuccess;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (a.vec4) {
        const size_t smem = sizeof(float) * kSpWarps * kSpWarpFloats;
        DADE_CUDA_TRY(cudaFuncSetAttribute(advance_survivors_pipe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        const uint32_t groups = (max_entries + 31) / 32;
        const uint32_t grid = std::min<uint32_t>((groups + kSpWarps - 1) / kSpWarps, (uint32_t)sms * 3);
        advance_survivors_pipe_kernel<<<grid, kSpWarps * 32, smem, s>>>(a);
        return cudaGetLastError();
    }
    const size_t smem = sizeof(float) * kSvWarps * 2 * 32 * kSvStride;
    DADE_CUDA_TRY(cudaFuncSetAttribute(advance_survivors_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const uint32_t groups = (max_entries + 31) / 32;
    const uint32_t grid = std::min<uint32_t>((groups + kSvWarps - 1) / kSvWarps, (uint32_t)sms * 3);
    advance_survivors_kernel<<<grid, kSvWarps * 32, smem, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_merge_slots(const uint64_t* qslots, uint32_t qslot_cap, const uint32_t* q_count,
                               const uint32_t* cand_q, const uint64_t* cand_key, const uint32_t* cand_count,
                               uint32_t cand_cap, uint32_t nq, uint32_t K, uint64_t* out_keys, uint32_t* out_count,
                               cudaStream_t s, uint32_t* r_global, uint32_t* res_ids, float* res_dists,
                               uint32_t* res_counts) {
    if (nq == 0) return cudaSuccess;
    merge_slots_kernel<<<(nq + 3) / 4, 128, 0, s>>>(qslots, qslot_cap, q_count, cand_q, cand_key, cand_count, cand_cap,
                                                    nq, K, out_keys, out_count, r_global, res_ids, res_dists,
                                                    res_counts);
    return cudaGetLastError();
}

// First-slice squared norms |o[0:d0]|^2 of every row (fp32 fma; any rounding
// is covered by the filter's error budget).
__global__ void row_norms_kernel(const float* __restrict__ rows, uint32_t n, uint32_t dim, uint32_t d0,
                                 float* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float* r = rows + (size_t)i * dim;
    float acc = 0.f;
    for (uint32_t k = 0; k < d0; ++k) acc = fmaf(r[k], r[k], acc);
    out[i] = acc;
}

cudaError_t launch_row_norms(const float* rows, uint32_t n, uint32_t dim, uint32_t d0, float* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    row_norms_kernel<<<(n + 255) / 256, 256, 0, s>>>(rows, n, dim, d0, out);
    return cudaGetLastError();
}

cudaError_t launch_merge_segments(const uint64_t* seg_keys, const uint32_t* seg_count, uint32_t nq,
                                  uint32_t n_slots, uint32_t K, uint64_t* out_keys, uint32_t* out_count,
                                  cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    merge_segments_kernel<<<(nq + 3) / 4, 128, 0, s>>>(seg_keys, seg_count, nq, n_slots, K, out_keys, out_count);
    return cudaGetLastError();
}

cudaError_t launch_merge_blocks(const uint64_t* keys, uint32_t G, uint32_t nq, uint32_t K,
                                uint64_t* out_keys, uint32_t* out_count, cudaStream_t s) {
    if (nq == 0) return cudaSuccess;
    merge_blocks_kernel<<<(nq + 3) / 4, 128, 0, s>>>(keys, G, nq, K, out_keys, out_count);
    return cudaGetLastError();
}

cudaError_t launch_keys_to_results(const uint64_t* keys, const uint32_t* count, uint32_t nq, uint32_t K,
                                   uint32_t* ids, float* dists, uint32_t* counts_out, cudaStream_t s) {
    const size_t n = (size_t)nq * K;
    if (n == 0) return cudaSuccess;
    keys_to_results_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(keys, count, nq, K, ids, dists, counts_out);
    return cudaGetLastError();
}

}  // namespace dade_gpu

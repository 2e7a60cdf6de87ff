// DCO scan kernel (K4/K6/K2 of SURVEY.md §2) and top-K merges (K5).
//
// One CTA = one work item: a contiguous row range (an IVF posting list or a
// flat row block) x up to kQC queries. Rows are swept in kRT-row tiles; each
// tile is swept in dimension chunks of <= kCH dims, with checkpoint tests at
// the strategy's checkpoints (proj/src/estimator.cpp:39-70):
//   * dense phase: every (row, query) pair of the tile in registers, 4 rows x
//     8 queries per thread, packed FADD2/FFMA2 math (bit-exact, see
//     common.cuh), queries broadcast from shared memory;
//   * after a checkpoint leaves <= kSparseCap pairs alive, the survivors are
//     compacted (warp ballot + prefix) into a shared list and only they are
//     advanced through the remaining chunks;
//   * exact full-D survivors with distance <= r become candidates and are
//     merged into the per-(query, slot) top-K segment in global memory, which
//     tightens the CTA's radius within the list (the reference's live heap
//     threshold, proj/src/ivf.cpp:221-229) and, via atomicMin, the query's
//     global radius seen by every later tile of every CTA.
#include <cfloat>
#include <cstdio>

#include "common.cuh"
#include "kernels.h"

namespace dade_gpu {

namespace {

struct SmemLayout {
    size_t o_t, q_k, q_j, r_s, thr_s, qidx, slot, la_meta, la_acc, lb_meta, lb_acc, keys, cnt, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline SmemLayout smem_layout(int n_ckpt) {
    SmemLayout L;
    size_t off = 0;
    L.o_t = off; off = align16(off + sizeof(float) * kRT * kOStride);
    L.q_k = off; off = align16(off + sizeof(float) * kCH * kQC);
    L.q_j = off; off = align16(off + sizeof(float) * kQC * kOStride);
    L.r_s = off; off = align16(off + sizeof(float) * kQC);
    L.thr_s = off; off = align16(off + sizeof(float) * kQC * (n_ckpt > 0 ? n_ckpt : 1));
    L.qidx = off; off = align16(off + sizeof(uint32_t) * kQC);
    L.slot = off; off = align16(off + sizeof(uint32_t) * kQC);
    L.la_meta = off; off = align16(off + sizeof(uint32_t) * kSparseCap);
    L.la_acc = off; off = align16(off + sizeof(float) * kSparseCap);
    L.lb_meta = off; off = align16(off + sizeof(uint32_t) * kSparseCap);
    L.lb_acc = off; off = align16(off + sizeof(float) * kSparseCap);
    L.keys = off; off = align16(off + sizeof(uint64_t) * kWarps * kRT);
    L.cnt = off; off = align16(off + sizeof(uint32_t) * (3 * kQC + 16));
    L.total = off;
    return L;
}

__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}

// Recompute query j's per-checkpoint float thresholds from r_s[j].
__device__ __forceinline__ void refresh_thr(float* thr_s, const float* r_s, const double* coeff,
                                            int n_ckpt, int j, int lane_in, int lanes) {
    const float r = r_s[j];
    for (int c = lane_in; c < n_ckpt; c += lanes) thr_s[j * n_ckpt + c] = prune_threshold(coeff[c], r);
}

template <bool kSqrtKey>
__global__ void __launch_bounds__(kThreads, 2)
dco_scan_kernel(const ScanArgs a, const __grid_constant__ ChunkTable ct) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int n_ckpt = ct.n_ckpt;
    const SmemLayout L = smem_layout(n_ckpt);
    float* o_t = reinterpret_cast<float*>(smem + L.o_t);
    float* q_k = reinterpret_cast<float*>(smem + L.q_k);
    float* q_j = reinterpret_cast<float*>(smem + L.q_j);
    float* r_s = reinterpret_cast<float*>(smem + L.r_s);
    float* thr_s = reinterpret_cast<float*>(smem + L.thr_s);
    uint32_t* qidx_s = reinterpret_cast<uint32_t*>(smem + L.qidx);
    uint32_t* slot_s = reinterpret_cast<uint32_t*>(smem + L.slot);
    uint32_t* lmeta[2] = {reinterpret_cast<uint32_t*>(smem + L.la_meta),
                          reinterpret_cast<uint32_t*>(smem + L.lb_meta)};
    float* lacc[2] = {reinterpret_cast<float*>(smem + L.la_acc), reinterpret_cast<float*>(smem + L.lb_acc)};
    uint64_t* keys_s = reinterpret_cast<uint64_t*>(smem + L.keys);
    uint32_t* qcnt = reinterpret_cast<uint32_t*>(smem + L.cnt);  // [kQC] candidate counts
    uint32_t* qoff = qcnt + kQC;                                 // [kQC] offsets in round
    uint32_t* qcur = qoff + kQC;                                 // [kQC] scatter cursors
    uint32_t* misc = qcur + kQC;                                 // [16]

    const int tid = threadIdx.x;
    const int warp = tid >> 5;
    const int lane = tid & 31;
    const uint32_t dim = a.dim;

    // ---- decode the work item ------------------------------------------------
    uint32_t row_start, row_count, qcount;
    if (a.items != nullptr) {
        if (blockIdx.x >= *a.n_items) return;
        const WorkItem wi = a.items[blockIdx.x];
        row_start = wi.row_start;
        row_count = wi.row_count;
        qcount = wi.bucket_count;
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
    if (tid < kQC) r_s[tid] = __int_as_float(0x7f800000);
    if (tid < kQC && tid >= (int)qcount) { qidx_s[tid] = 0; slot_s[tid] = 0; }

    unsigned long long st_dco = 0, st_dims = 0, st_bytes = 0;
    if (tid == 0) st_bytes += sizeof(WorkItem) + 8ull * qcount;
    const uint64_t nz2 = a.neg_zero2;

    for (uint32_t tile_base = 0; tile_base < row_count; tile_base += kRT) {
        const uint32_t nrows = min((uint32_t)kRT, row_count - tile_base);
        __syncthreads();  // previous tile's merges finished with r_s / thr_s
        // Pick up radii tightened by other CTAs (or our own earlier tiles).
        if (tid < (int)qcount) {
            const float rg = __uint_as_float(ld_volatile_u32(a.r_global + qidx_s[tid]));
            const bool first = tile_base == 0;
            if (rg < r_s[tid] || first) {
                r_s[tid] = fminf(rg, r_s[tid]);
                refresh_thr(thr_s, r_s, a.coeff, n_ckpt, tid, 0, 1);
            }
        }

        // ---- dense state -------------------------------------------------------
        uint64_t acc[4][4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int p = 0; p < 4; ++p) acc[i][p] = 0ull;
        uint32_t alive = 0;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int jj = 0; jj < 8; ++jj)
                if ((uint32_t)(lane + 32 * i) < nrows && (uint32_t)(warp * 8 + jj) < qcount)
                    alive |= 1u << (i * 8 + jj);
        st_dco += __popc(alive);
        bool dense = true;
        int cur = 0;              // active sparse list
        uint32_t cand = 0;        // dense candidate bits (final chunk)

        for (int c = 0; c < ct.n_chunks; ++c) {
            const uint32_t k0 = c == 0 ? 0u : ct.end[c - 1];
            const uint32_t w = ct.end[c] - k0;
            const uint32_t w4 = (w + 3) & ~3u;
            __syncthreads();  // everyone done with the previous chunk's tiles
            // ---- stage the o tile [kRT x w4] and q tiles ------------------------
            const bool vec = ((dim | k0 | w) & 3u) == 0;
            if (vec) {
                const uint32_t v4 = w >> 2;
                for (uint32_t idx = tid; idx < kRT * v4; idx += kThreads) {
                    const uint32_t r = idx / v4, c4 = idx - r * v4;
                    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                    if (r < nrows)
                        v = __ldg(reinterpret_cast<const float4*>(
                            a.storage + (size_t)(row_start + tile_base + r) * dim + k0) + c4);
                    *reinterpret_cast<float4*>(o_t + r * kOStride + 4 * c4) = v;
                }
            } else {
                for (uint32_t idx = tid; idx < kRT * w4; idx += kThreads) {
                    const uint32_t r = idx / w4, cc = idx - r * w4;
                    float v = 0.f;
                    if (r < nrows && cc < w) v = __ldg(a.storage + (size_t)(row_start + tile_base + r) * dim + k0 + cc);
                    o_t[r * kOStride + cc] = v;
                }
            }
            for (uint32_t idx = tid; idx < kQC * w4; idx += kThreads) {
                const uint32_t j = idx / w4, cc = idx - j * w4;
                float v = 0.f;
                if (j < qcount && cc < w) v = __ldg(a.queries + (size_t)qidx_s[j] * dim + k0 + cc);
                q_k[cc * kQC + j] = v;
                q_j[j * kOStride + cc] = v;
            }
            if (tid == 0) st_bytes += 4ull * w * (nrows + qcount);
            __syncthreads();

            const int ck = ct.ckpt[c];
            const bool last = c == ct.n_chunks - 1;
            if (dense) {
                // ---- dense register-tiled update -------------------------------
                if (__any_sync(0xffffffffu, alive != 0)) {
                    for (uint32_t k4 = 0; k4 < w4; k4 += 4) {
                        float4 o[4];
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            o[i] = *reinterpret_cast<const float4*>(o_t + (lane + 32 * i) * kOStride + k4);
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            const ulonglong2 qa = *reinterpret_cast<const ulonglong2*>(q_k + (k4 + kk) * kQC + warp * 8);
                            const ulonglong2 qb = *reinterpret_cast<const ulonglong2*>(q_k + (k4 + kk) * kQC + warp * 8 + 4);
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
                if (ck >= 0) {
                    // checkpoint test on every live pair
                    uint32_t dead = 0;
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const float t = thr_s[(warp * 8 + jj) * n_ckpt + ck];
#pragma unroll
                        for (int i = 0; i < 4; ++i) {
                            const uint64_t v = acc[i][jj >> 1];
                            const float x = (jj & 1) ? hi_f(v) : lo_f(v);
                            if (x > t) dead |= 1u << (i * 8 + jj);
                        }
                    }
                    dead &= alive;
                    alive &= ~dead;
                    st_dims += (unsigned long long)__popc(dead) * ct.end[c];
                    if (tid == 0) misc[0] = 0;
                    __syncthreads();
                    uint32_t wsum = __reduce_add_sync(0xffffffffu, __popc(alive));
                    if (lane == 0) atomicAdd(&misc[0], wsum);
                    __syncthreads();
                    const uint32_t total_alive = misc[0];
                    if (total_alive <= (uint32_t)kSparseCap && !last) {
                        // ---- switch to the sparse survivor list -------------------
                        if (tid == 0) misc[1] = 0;
                        __syncthreads();
                        const uint32_t mine = __popc(alive);
                        uint32_t incl = mine;
#pragma unroll
                        for (int off = 1; off < 32; off <<= 1) {
                            const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
                            if (lane >= off) incl += y;
                        }
                        uint32_t base = 0;
                        if (lane == 31) base = atomicAdd(&misc[1], incl);
                        base = __shfl_sync(0xffffffffu, base, 31);
                        uint32_t pos = base + incl - mine;
                        uint32_t bits = alive;
                        while (bits) {
                            const int b = __ffs(bits) - 1;
                            bits &= bits - 1;
                            const int i = b >> 3, jj = b & 7;
                            const uint64_t v = acc[i][jj >> 1];
                            lmeta[0][pos] = (uint32_t)(lane + 32 * i) | ((uint32_t)(warp * 8 + jj) << 8);
                            lacc[0][pos] = (jj & 1) ? hi_f(v) : lo_f(v);
                            ++pos;
                        }
                        dense = false;
                        cur = 0;
                        __syncthreads();
                        if (tid == 0) misc[2] = misc[1];  // list length
                        __syncthreads();
                    }
                }
                if (last) {
                    st_dims += (unsigned long long)__popc(alive) * dim;
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
                }
            } else {
                // ---- sparse survivor update -----------------------------------
                const uint32_t n = misc[2];
                uint32_t* meta_in = lmeta[cur];
                float* acc_in = lacc[cur];
                uint32_t* meta_out = lmeta[cur ^ 1];
                float* acc_out = lacc[cur ^ 1];
                if (ck >= 0 && tid == 0) misc[1] = 0;
                if (ck >= 0) __syncthreads();
                const uint32_t n_round = (n + kThreads - 1) / kThreads * kThreads;
                for (uint32_t e = tid; e < n_round; e += kThreads) {
                    bool keep = false;
                    uint32_t meta = 0;
                    float x = 0.f;
                    if (e < n) {
                        meta = meta_in[e];
                        x = acc_in[e];
                        const uint32_t row = meta & 0xffu, j = meta >> 8;
                        const float* orow = o_t + row * kOStride;
                        const float* qrow = q_j + j * kOStride;
                        for (uint32_t k4 = 0; k4 < w4; k4 += 4) {
                            const float4 o4 = *reinterpret_cast<const float4*>(orow + k4);
                            const float4 q4 = *reinterpret_cast<const float4*>(qrow + k4);
                            x = sq_step(x, o4.x, q4.x);
                            x = sq_step(x, o4.y, q4.y);
                            x = sq_step(x, o4.z, q4.z);
                            x = sq_step(x, o4.w, q4.w);
                        }
                        if (ck >= 0) {
                            keep = !(x > thr_s[j * n_ckpt + ck]);
                            if (!keep) st_dims += ct.end[c];
                        } else if (last) {
                            st_dims += dim;
                            const float key = kSqrtKey ? __fsqrt_rn(x) : x;
                            const bool is_cand = !(key > r_s[j]);
                            meta_in[e] = meta | (is_cand ? 0x80000000u : 0u);
                            acc_in[e] = key;
                        } else {
                            acc_in[e] = x;
                        }
                    }
                    if (ck >= 0) {
                        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
                        uint32_t base = 0;
                        if (lane == 0 && bal) base = atomicAdd(&misc[1], __popc(bal));
                        base = __shfl_sync(0xffffffffu, base, 0);
                        if (keep) {
                            const uint32_t pos = base + __popc(bal & ((1u << lane) - 1u));
                            meta_out[pos] = meta;
                            acc_out[pos] = x;
                        }
                    }
                }
                if (ck >= 0) {
                    __syncthreads();
                    if (tid == 0) misc[2] = misc[1];
                    cur ^= 1;
                    __syncthreads();
                }
            }
        }  // chunks

        // ---- candidates -> per-(query, slot) top-K segments ----------------------
        if (tid < kQC) { qcnt[tid] = 0; qcur[tid] = 0; }
        __syncthreads();
        const uint32_t n_sp = dense ? 0u : misc[2];
        const uint32_t* sp_meta = lmeta[cur];
        const float* sp_key = lacc[cur];
        if (dense) {
            uint32_t bits = cand;
            while (bits) {
                const int b = __ffs(bits) - 1;
                bits &= bits - 1;
                atomicAdd(&qcnt[warp * 8 + (b & 7)], 1u);
            }
        } else {
            for (uint32_t e = tid; e < n_sp; e += kThreads) {
                const uint32_t m = sp_meta[e];
                if (m & 0x80000000u) atomicAdd(&qcnt[(m >> 8) & 0xffu], 1u);
            }
        }
        __syncthreads();
        // Rounds of consecutive queries whose candidates fit the scratch list.
        uint32_t* cmeta = lmeta[dense ? 0 : (cur ^ 1)];
        float* ckey = lacc[dense ? 0 : (cur ^ 1)];
        uint32_t j_lo = 0;
        while (j_lo < qcount) {
            // every thread computes the same round end (qcnt is small)
            uint32_t j_hi = j_lo, tot = 0;
            while (j_hi < qcount && tot + qcnt[j_hi] <= (uint32_t)kSparseCap) {
                tot += qcnt[j_hi];
                ++j_hi;
            }
            if (tot == 0) { j_lo = j_hi; continue; }
            if (tid < kQC) {
                uint32_t o = 0;
                for (uint32_t j = j_lo; j < (uint32_t)tid && j < j_hi; ++j) o += qcnt[j];
                qoff[tid] = o;
                qcur[tid] = 0;
            }
            __syncthreads();
            if (dense) {
                uint32_t bits = cand;
                while (bits) {
                    const int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    const int i = b >> 3, jj = b & 7;
                    const uint32_t j = warp * 8 + jj;
                    if (j < j_lo || j >= j_hi) continue;
                    const uint64_t v = acc[i][jj >> 1];
                    const float x = (jj & 1) ? hi_f(v) : lo_f(v);
                    const uint32_t pos = qoff[j] + atomicAdd(&qcur[j], 1u);
                    cmeta[pos] = (uint32_t)(lane + 32 * i);
                    ckey[pos] = kSqrtKey ? __fsqrt_rn(x) : x;
                }
            } else {
                for (uint32_t e = tid; e < n_sp; e += kThreads) {
                    const uint32_t m = sp_meta[e];
                    const uint32_t j = (m >> 8) & 0xffu;
                    if (!(m & 0x80000000u) || j < j_lo || j >= j_hi) continue;
                    const uint32_t pos = qoff[j] + atomicAdd(&qcur[j], 1u);
                    cmeta[pos] = m & 0xffu;
                    ckey[pos] = sp_key[e];
                }
            }
            __syncthreads();
            // warp w merges queries j == w (mod kWarps)
            for (uint32_t j = j_lo + ((warp - j_lo % kWarps + kWarps) % kWarps); j < j_hi; j += kWarps) {
                const uint32_t m = qcnt[j];
                if (m == 0) continue;
                uint64_t* kb = keys_s + warp * kRT;
                for (uint32_t e = lane; e < m; e += 32) {
                    const uint32_t row = cmeta[qoff[j] + e];
                    const uint32_t g = row_start + tile_base + row;
                    const uint32_t id = a.row_ids ? __ldg(a.row_ids + g) : a.id_base + g;
                    kb[e] = make_key(ckey[qoff[j] + e], id);
                }
                st_bytes += a.row_ids ? 4ull * (m > lane ? (m - lane + 31) / 32 : 0) : 0ull;
                __syncwarp();
                const size_t seg = (size_t)qidx_s[j] * a.n_slots + slot_s[j];
                uint64_t* A = a.seg_keys + seg * a.K;
                const uint32_t nc = warp_merge(A, a.seg_count + seg, a.K, kb, m, false);
                if (nc == a.K) {
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
            __syncthreads();
            j_lo = j_hi;
        }
    }  // tiles

    // ---- counters -------------------------------------------------------------
    st_dco = __reduce_add_sync(0xffffffffu, (unsigned)st_dco);
    unsigned long long d = st_dims;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
    unsigned long long b = st_bytes;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) b += __shfl_xor_sync(0xffffffffu, b, off);
    if (lane == 0 && a.counters) {
        atomicAdd(a.counters + 0, st_dco);
        atomicAdd(a.counters + 1, d);
        atomicAdd(a.counters + 2, b);
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
            // early out: the batch starts above a full list's worst key
            const uint32_t cur = *reinterpret_cast<volatile uint32_t*>(cA);
            if (cur == K && src[b0] > A[K - 1]) break;
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
            uint32_t m = 0;
            for (uint32_t e = lane; e < m0; e += 32) {
                const uint64_t v = src[b0 + e];
                B[e] = v;
            }
            __syncwarp();
            // count of non-empty keys (sorted, empties at the end)
            uint32_t nonempty = 0;
            for (uint32_t e = lane; e < m0; e += 32) nonempty += B[e] != kEmptyKey;
            m = __reduce_add_sync(0xffffffffu, nonempty);
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

size_t scan_smem_bytes(int n_ckpt) { return smem_layout(n_ckpt).total; }

cudaError_t launch_scan(const ScanArgs& a, const ChunkTable& ct, uint32_t grid, bool sqrt_key,
                        cudaStream_t s) {
    const size_t smem = scan_smem_bytes(ct.n_ckpt);
    if (grid == 0) return cudaSuccess;
    if (sqrt_key) {
        DADE_CUDA_TRY(cudaFuncSetAttribute(dco_scan_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dco_scan_kernel<true><<<grid, kThreads, smem, s>>>(a, ct);
    } else {
        DADE_CUDA_TRY(cudaFuncSetAttribute(dco_scan_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        dco_scan_kernel<false><<<grid, kThreads, smem, s>>>(a, ct);
    }
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

// Shared device helpers for the DADE distance-comparison kernels (sm_100a).
#pragma once

#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace dade_gpu {

// ---- scan geometry ---------------------------------------------------------
constexpr int kThreads = 256;  // 8 warps
constexpr int kWarps = kThreads / 32;     // consumer warps
constexpr int kThreadsTotal = kThreads + 32;  // + one TMA producer warp
constexpr int kBox = 32;        // dims per TMA box (128 B rows, 128B swizzle)
constexpr int kRT = 128;       // candidate rows per tile
constexpr int kQC = 64;        // queries per work item (query chunk)
constexpr int kCH = 32;        // dims per staged chunk
constexpr int kOStride = kCH + 4;  // padded o-tile row (floats): conflict-free LDS.128
constexpr int kQS = kQC + 8;       // padded k-major query row: conflict-free MMA B loads
constexpr int kSparseCap = 2048;   // survivor-list capacity (25 % of kRT * kQC)
constexpr int kMaxChunks = 256;    // dim up to ~4096 with kCH = 32 plus checkpoints

constexpr uint64_t kEmptyKey = ~0ull;

// One CTA work item: a contiguous row range of the device storage (one IVF
// posting list, or one row block of a flat base) against up to kQC queries
// taken from bucket arrays (query index, output slot).
// queries per radius-seed CTA (seed_radius_list_kernel; group prefix in group_scan_kernel)
constexpr int kSeedGroup = 16;

struct WorkItem {
    uint32_t row_start;
    uint32_t row_count;
    uint32_t bucket_start;
    uint32_t bucket_count;  // low 16 bits: queries; high 16 bits: row-piece index within the list
};

// Chunk table: chunk c covers dims [c_begin, end[c]); ckpt[c] = checkpoint
// index tested after the chunk, or -1.
// Chunks [0, n_dense) form the dense phase (up to and including the first
// checkpoint; all chunks without checkpoints). d_res > 0: the queries' first
// d_res dims stay resident in shared memory. vec_ok: every boundary is a
// multiple of 4 (16-byte staging and loads).
// use_tc: the dense phase runs as a TF32 tensor-core filter (see scan.cu);
// n_buf: o-tile ring depth (n_dense + 1 with the filter, else 2).
struct ChunkTable {
    int n_chunks;
    int n_ckpt;
    int n_dense;
    int d_res;
    int vec_ok;
    int use_tc;
    int n_buf;
    int debug;
    int use_tma;
    uint16_t end[kMaxChunks];
    int16_t ckpt[kMaxChunks];
};
constexpr int kMaxResidentQBytes = 64 * 1024;

// ---- exact fp32 arithmetic -------------------------------------------------
// The reference accumulates acc += (o - q)^2 with three separately rounded
// fp32 operations (proj/include/dade/distance.hpp:26-33, built without FMA).
// Scalar: __fsub_rn/__fmul_rn/__fadd_rn are never contracted.
__device__ __forceinline__ float sq_step(float acc, float o, float q) {
    const float d = __fsub_rn(o, q);
    return __fadd_rn(acc, __fmul_rn(d, d));
}

// Packed (2 lanes) variant for sm_100a FADD2/FFMA2. ptxas contracts
// mul.f32x2 + add.f32x2 into FFMA2 even with .rn, which would change the
// rounding; squaring as fma(d, d, z) with an OPAQUE z = -0.0 (a kernel
// argument) is exact (x*x + -0 == round(x*x)) and cannot be folded into the
// following add. neg_zero2 must be 0x8000000080000000.
__device__ __forceinline__ uint64_t sq_step2(uint64_t acc, float o, uint64_t q2, uint64_t neg_zero2) {
    uint64_t o2, d, m, r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(o2) : "f"(o));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(o2), "l"(q2));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(m) : "l"(d), "l"(neg_zero2));
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(acc), "l"(m));
    return r;
}

__device__ __forceinline__ float lo_f(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v)); }
__device__ __forceinline__ float hi_f(uint64_t v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }

// (double)acc > coeff * r^2  <=>  acc > rd_float(coeff * r^2) for every fp32
// acc, including the NaN (inf * 0) case, which never prunes
// (proj/src/estimator.cpp:43, 50; proj/tests/test_estimator.cpp:235-243).
__device__ __forceinline__ float prune_threshold(double coeff, float r) {
    const double r2 = __dmul_rn(static_cast<double>(r), static_cast<double>(r));
    return __double2float_rd(__dmul_rn(coeff, r2));
}

// Radix-select digit search by one warp: hist[256] (shared) counts the
// elements of the current prefix class by digit; returns the digit holding the
// rank-th (1-based) element and the count of elements in lower digits.
__device__ __forceinline__ void warp_hist_find(const uint32_t* hist, uint32_t rank, uint32_t lane, uint32_t& digit,
                                               uint32_t& before) {
    uint32_t bins[8], sum = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        bins[j] = hist[lane * 8 + j];
        sum += bins[j];
    }
    uint32_t incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= (uint32_t)off) incl += y;
    }
    const uint32_t excl = incl - sum;
    const bool mine = excl < rank && rank <= incl;
    uint32_t d = 0, b = 0;
    if (mine) {
        uint32_t cum = excl;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (cum + bins[j] >= rank) {
                d = lane * 8 + j;
                b = cum;
                break;
            }
            cum += bins[j];
        }
    }
    const uint32_t who = __ballot_sync(0xffffffffu, mine);
    const int src = who ? __ffs(who) - 1 : 0;
    digit = __shfl_sync(0xffffffffu, d, src);
    before = __shfl_sync(0xffffffffu, b, src);
}

// Coarse ranking bound (coarse.cu): |p~ - l2_sq| <= kCoarseDelta (|q|^2 + |c|^2). Budget, in units of
// |q|^2 + |c|^2, for dim <= kCoarseTcMaxDim = 2048: TF32 operands (fp32 bits, low 13 mantissa bits ignored:
// < 2^-10 relative each) put 2 c.q off by < 2^-9 + 2^-20 = 1.95e-3; the tensor core's fp32 accumulation over
// dim / 8 steps < 6e-5; the fp32 norms < gamma_dim = 1.2e-4; the reference's sequential fp32 l2_sq differs from
// the real value by < gamma_dim d^2 <= 2.4e-4. Sum < 2.37e-3 (2.16e-3 up to dim 1024): 2.6e-3 holds with margin
// (4e-3 until round 2; the tighter bound leaves a third fewer uncertain centroids for the exact rounds).
constexpr float kCoarseDelta = 2.6e-3f;
constexpr uint32_t kCoarseTcMaxDim = 2048;  // longer vectors rank with the exact kernels
// the bound's half-width and the upper / lower keys, with explicit roundings so every
// kernel that forms them (GEMM epilogue, selections) gets the same bits
__device__ __forceinline__ float coarse_delta(float cn, float qn) { return __fmul_rn(kCoarseDelta, __fadd_rn(cn, qn)); }
// order-preserving key of a float (any sign)
__device__ __forceinline__ uint32_t fkey(float x) {
    const uint32_t u = __float_as_uint(x);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__device__ __forceinline__ uint64_t make_key(float dist, uint32_t id) {
    return (static_cast<uint64_t>(__float_as_uint(dist)) << 32) | id;
}

// ---- warp-level top-K merge --------------------------------------------------
// A: ascending keys (global or shared), count *cA_ptr; B: m keys in shared
// memory (ascending if b_sorted). Keys are unique ((dist, id) with unique ids),
// so final position of an element = its rank in its own array + the count of
// smaller elements in the other. Elements landing at >= K are dropped. This
// reproduces TopKHeap's "K smallest by (distance, id)" (proj/src/knn.cpp:9-29)
// for any insertion order.
__device__ __forceinline__ uint32_t lower_bound_u64(const uint64_t* a, uint32_t n, uint64_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (a[mid] < x) lo = mid + 1; else hi = mid;
    }
    return lo;
}

__device__ __forceinline__ uint32_t count_less(const uint64_t* b, uint32_t m, uint64_t x) {
    uint32_t c = 0;
    for (uint32_t i = 0; i < m; ++i) c += b[i] < x;
    return c;
}

// Returns the new count (all lanes). Caller guarantees m <= 32 * kMaxBPerLane.
constexpr int kMaxBPerLane = 8;
__device__ inline uint32_t warp_merge(uint64_t* A, uint32_t* cA_ptr, uint32_t K, const uint64_t* B,
                                      uint32_t m, bool b_sorted) {
    const int lane = threadIdx.x & 31;
    const uint32_t cA = *reinterpret_cast<volatile uint32_t*>(cA_ptr);
    __syncwarp();
    if (m == 0) return cA;
    uint32_t posb[kMaxBPerLane];
    uint64_t keyb[kMaxBPerLane];
    uint64_t minb = kEmptyKey;
#pragma unroll
    for (int s = 0; s < kMaxBPerLane; ++s) {
        const uint32_t b = lane + 32u * s;
        posb[s] = K;
        keyb[s] = kEmptyKey;
        if (b < m) {
            const uint64_t kb = B[b];
            const uint32_t rb = b_sorted ? b : count_less(B, m, kb);
            posb[s] = rb + lower_bound_u64(A, cA, kb);
            keyb[s] = kb;
            minb = kb < minb ? kb : minb;
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, minb, off);
        minb = o < minb ? o : minb;
    }
    // Shift the A elements larger than min(B), highest chunk first so no
    // element is overwritten before it is read.
    if (cA > 0) {
        for (int c = static_cast<int>((cA - 1) & ~31u); c >= 0; c -= 32) {
            const uint32_t i = static_cast<uint32_t>(c) + lane;
            uint64_t a = 0;
            bool need = false;
            if (i < cA) {
                a = A[i];
                need = a > minb;
            }
            if (!__any_sync(0xffffffffu, need)) break;
            uint32_t shift = 0;
            if (need) shift = b_sorted ? lower_bound_u64(B, m, a) : count_less(B, m, a);
            __syncwarp();
            if (need && i + shift < K) A[i + shift] = a;
            __syncwarp();
        }
    }
#pragma unroll
    for (int s = 0; s < kMaxBPerLane; ++s)
        if (posb[s] < K) A[posb[s]] = keyb[s];
    const uint32_t nc = min(K, cA + m);
    __syncwarp();
    if (lane == 0) *cA_ptr = nc;
    __syncwarp();
    return nc;
}

// Same contract as warp_merge for a top-K list A in GLOBAL memory, with the
// list staged once into the warp's shared scratch (K <= kStageMaxK): one
// coalesced load instead of a chain of dependent global reads, all rank
// searches in shared memory, and only the elements that move are written back.
constexpr int kStageMaxK = 128;
__device__ inline uint32_t warp_merge_staged(uint64_t* A, uint32_t* cA_ptr, uint32_t K, const uint64_t* B,
                                             uint32_t m, uint64_t* scratch) {
    const int lane = threadIdx.x & 31;
    const uint32_t cA = *reinterpret_cast<volatile uint32_t*>(cA_ptr);
    if (m == 0) return cA;
    for (uint32_t i = lane; i < cA; i += 32) scratch[i] = A[i];
    __syncwarp();
    uint64_t minb = kEmptyKey;
    for (uint32_t b = lane; b < m; b += 32) minb = B[b] < minb ? B[b] : minb;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const uint64_t o = __shfl_xor_sync(0xffffffffu, minb, off);
        minb = o < minb ? o : minb;
    }
    // A elements >= min(B) shift right by the number of smaller B elements
    const uint32_t first = lower_bound_u64(scratch, cA, minb);
    for (uint32_t i = first + lane; i < cA; i += 32) {
        const uint64_t a = scratch[i];
        const uint32_t pos = i + count_less(B, m, a);
        if (pos < K) A[pos] = a;
    }
    for (uint32_t b = lane; b < m; b += 32) {
        const uint64_t kb = B[b];
        const uint32_t pos = count_less(B, m, kb) + lower_bound_u64(scratch, cA, kb);
        if (pos < K) A[pos] = kb;
    }
    const uint32_t nc = min(K, cA + m);
    __syncwarp();
    if (lane == 0) *cA_ptr = nc;
    __syncwarp();
    return nc;
}

// As warp_merge_staged for larger batches: B (shared, capacity >= the next power
// of two of m, <= 256) is bitonic-sorted first, so every element's final position
// is found by binary search instead of a linear count over B.
__device__ inline uint32_t warp_merge_sortb(uint64_t* A, uint32_t* cA_ptr, uint32_t K, uint64_t* B, uint32_t m,
                                            uint64_t* scratch) {
    const int lane = threadIdx.x & 31;
    const uint32_t cA = *reinterpret_cast<volatile uint32_t*>(cA_ptr);
    if (m == 0) return cA;
    uint32_t mp = 1;
    while (mp < m) mp <<= 1;
    for (uint32_t i = m + lane; i < mp; i += 32) B[i] = kEmptyKey;
    for (uint32_t i = lane; i < cA; i += 32) scratch[i] = A[i];
    __syncwarp();
    for (uint32_t size = 2; size <= mp; size <<= 1)
        for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
            for (uint32_t i = lane; i < mp / 2; i += 32) {
                const uint32_t lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                const bool up = (lo & size) == 0;
                const uint64_t x = B[lo], y = B[hi];
                if ((x > y) == up) {
                    B[lo] = y;
                    B[hi] = x;
                }
            }
            __syncwarp();
        }
    const uint32_t first = lower_bound_u64(scratch, cA, B[0]);
    for (uint32_t i = first + lane; i < cA; i += 32) {
        const uint64_t a = scratch[i];
        const uint32_t pos = i + lower_bound_u64(B, m, a);
        if (pos < K) A[pos] = a;
    }
    for (uint32_t b = lane; b < m && b < K; b += 32) {
        const uint64_t kb = B[b];
        const uint32_t pos = b + lower_bound_u64(scratch, cA, kb);
        if (pos < K) A[pos] = kb;
    }
    const uint32_t nc = min(K, cA + m);
    __syncwarp();
    if (lane == 0) *cA_ptr = nc;
    __syncwarp();
    return nc;
}

// ---- error plumbing ----------------------------------------------------------
#define DADE_CUDA_TRY(expr)                                                      \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) return _e;                                        \
    } while (0)

}  // namespace dade_gpu

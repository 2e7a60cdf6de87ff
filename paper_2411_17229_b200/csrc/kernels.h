// Host-visible launchers of the sm_100a kernels (internal to libdade_gpu.so).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

namespace dade_gpu {

// A pair that passed the first checkpoint exactly, handed from the streaming
// filter to the survivor kernel: storage row, query, slot and its partial sum.
struct Survivor {
    uint32_t q;    // query index (UINT32_MAX = empty entry)
    uint32_t row;  // device storage row
    float acc;     // exact partial over the dense dims
    uint32_t slot;
};

struct ScanArgs {
    const float* storage;    // device rows [*, dim], contiguous
    const uint32_t* row_ids; // nullable: ids = id_base + row
    uint32_t id_base;
    uint32_t dim;
    const float* queries;    // rotated [nq, dim]
    // explicit work items (IVF) ...
    const WorkItem* items;
    const uint32_t* n_items;
    const uint32_t* bucket_q;
    const uint32_t* bucket_slot;
    // ... or an implicit (row block x query chunk) grid (flat scans)
    uint32_t flat_rows, flat_block, flat_nq, flat_qchunks;
    uint32_t* r_global;      // [nq] radius as float bits (key space)
    uint64_t* seg_keys;      // [nq * n_slots * K]
    uint32_t* seg_count;     // [nq * n_slots]
    uint32_t n_slots;
    uint32_t K;
    const double* coeff;     // [n_ckpt] reject coefficients
    uint64_t neg_zero2;      // 0x8000000080000000 (opaque to ptxas)
    unsigned long long* counters;  // [3] total_dco, dims_accumulated, bytes; [8] eligible, [9] failures
    unsigned long long* phase;     // nullable: per-phase clocks (debug)
    uint32_t measure;              // failure accounting (DcoStats::measure_failures): pruned pairs are
                                   // carried to the full dim for their exact distance
    uint32_t max_rows;             // nonzero: scan only the first max_rows rows of each item
    int seed;                      // radius-seeding pass: every query writes slot 0
    const float* row_norms;        // [rows] first-slice |o|^2 (tensor-core filter only)
    unsigned long long* census;    // nullable debug: [0] merges, [1] merged candidates
    const uint32_t* item_base;     // nullable: work item index = blockIdx.x + *item_base
    Survivor* surv;                // nullable: hand first-checkpoint survivors to advance_survivors
    uint32_t* surv_count;
    uint32_t surv_cap;
};

size_t scan_smem_bytes(int n_ckpt, int d_res, int n_buf);

// Streaming tensor-core filter (filter.cu): first-slice test for every pair of
// the work items, first-checkpoint survivors appended to surv.
struct FilterArgs {
    const float* queries;         // rotated [nq, dim]
    uint32_t dim;
    uint32_t d0;                  // dense dims = first checkpoint (multiple of 8, <= 64)
    int c_dense;                  // ceil(d0 / 32) boxes per tile
    double coeff0;                // reject coefficient of the first checkpoint
    const uint32_t* r_global;     // radius per query (float bits), fixed for the launch
    const WorkItem* items;        // IVF items (or nullptr: flat grid below)
    const uint32_t* n_items;
    const uint32_t* item_base;    // nullable
    const uint32_t* bucket_q;
    const uint32_t* bucket_slot;
    uint32_t flat_rows, flat_block, flat_nq, flat_qchunks;
    Survivor* surv;
    uint32_t* surv_count;
    uint32_t surv_cap;
    unsigned long long* counters; // [0] dco, [1] dims, [2] bytes
    uint32_t* item_counter;       // persistent scheduling (zeroed before the launch)
    const float* row_norms;       // [rows + 32] first-slice |o|^2 per storage row
    uint32_t piece_lo, piece_hi;  // only items whose row piece is in [piece_lo, piece_hi)
    uint32_t range_lo = 0, range_hi = 0;  // range_hi > 0: the pass's items are exactly [range_lo, range_hi) (flat, piece major)
    const uint32_t* b0_items;     // nullable: items below *b0_items (rank bucket 0) need piece >= b0_piece_lo
    uint32_t b0_piece_lo;         //   instead (the last IVF pass also takes the nearest lists' tails)
    int debug;                    // 1: re-check every filter prune exactly (counters[3] = violations)
    unsigned long long* census;   // nullable: [0] tiles with kept pairs | tiles << 32, [1] kept pairs (diagnostic)
    const float* q_norms;         // [nq] first-slice |q|^2 (sequential fmaf), tcgen05 filter only
};
size_t filter_smem_bytes(int d0, int c_dense);
cudaError_t launch_filter(const FilterArgs& a, const CUtensorMap& tmap32, uint32_t grid, cudaStream_t s);
// umma.cu: the same filter on tcgen05 (128-row tiles, TMEM accumulators); kept
// pairs leave with acc = 0 and are continued from dim 0 (SurvArgs::first_ckpt = 0)
size_t filter_umma_smem_bytes(int c_dense);
cudaError_t launch_filter_umma(const FilterArgs& a, const CUtensorMap& tmap128, const CUtensorMap& tmap_aug,
                               uint32_t grid, cudaStream_t s);
// tcgen05 coarse GEMM: p~ [nq][n_cen] for queries [q0, q0 + nq) of the tm_q map (box {32, 256})
// gmin (nullable) [nq][ceil(n_cen / 32)]: per query, the minimum coarse upper-bound key (fkey(p~ + delta))
// of every 32 consecutive centroids (coarse_select_wide_kernel's group minima)
// pass B of the fused large-nlist coarse selection: append (p~ bits << 32 | centroid) of every
// pair with lower bound <= t0[q] to cand[q][0..cap), counts in cnt[q] (may exceed cap)
struct CoarseFilter {
    const uint32_t* t0 = nullptr;  // [nq] (chunk-relative), nullptr: pass A / p~ mode
    uint64_t* cand = nullptr;      // [nq][cap]
    uint32_t* cnt = nullptr;       // [nq], zeroed before the launch
    uint32_t cap = 0;
};
cudaError_t launch_coarse_umma(const CUtensorMap& tm_cen, const CUtensorMap& tm_q, uint32_t q0, uint32_t n_cen,
                               uint32_t nq, uint32_t dim, const float* cnorm, const float* qnorm, float* p_out,
                               cudaStream_t s, uint32_t* gmin = nullptr, const CoarseFilter& cf = CoarseFilter{});
// query-major fused selection (umma.cu): pass A (cf.t0 == nullptr) writes gmin_t
// [ceil(n_cen / 32)][nq] (per query, the min upper-bound key of every 32 centroids); pass B
// (cf.t0 set) lists the candidates. tm_q128: queries, box {32, 128}; tm_c256: centroids, box {32, 256}.
bool coarse_sel_umma_ok(uint32_t dim);
cudaError_t launch_coarse_sel_umma(const CUtensorMap& tm_q128, const CUtensorMap& tm_c256, uint32_t q0, uint32_t n_cen,
                                   uint32_t nq, uint32_t dim, const float* cnorm, const float* qnorm, uint32_t* gmin_t,
                                   const CoarseFilter& cf, cudaStream_t s);
// the fused large-nlist selection around it (coarse.cu): T0 per query from the GEMM's group
// minima, then (after pass B) B, the exact l2_sq of the candidates and the (d^2, id) sort
// transposed: gmin[group][nq] (coarse_sel_umma pass A) instead of gmin[query][groups]
cudaError_t launch_coarse_t0(const uint32_t* gmin, uint32_t n_cen, uint32_t nq, uint32_t n_probe, uint32_t* t0,
                             cudaStream_t s, bool transposed = false);
cudaError_t launch_coarse_finish(const uint64_t* cand, const uint32_t* cnt, uint32_t cap, const float* cnorm,
                                 const float* qnorm, const float* centroids, const float* queries, uint32_t nq,
                                 uint32_t dim, uint32_t n_probe, uint64_t* probes, uint32_t* overflow, cudaStream_t s,
                                 uint32_t parts = 1);
constexpr uint32_t kCoarseSelParts = 4;  // list slices per query of the query-major pass B
// coarse.cu pieces around it
cudaError_t launch_coarse_norms(const float* centroids, uint32_t n_cen, const float* queries, uint32_t nq, uint32_t dim,
                                float* cnorm, float* qnorm, cudaStream_t s);
// Every centroid probed: p~-nearest first, the rest in id order (data-ordered flat scan).
cudaError_t launch_coarse_all(const float* pt, uint32_t n_cen, uint32_t nq, uint64_t* probes, cudaStream_t s);
// exact_keys: every probe key carries the exact l2_sq (else only the probe set is exact,
// the order after the nearest approximate)
cudaError_t launch_coarse_select(const float* centroids, uint32_t n_cen, const float* queries, uint32_t nq,
                                 uint32_t dim, uint32_t n_probe, const float* cnorm, const float* qnorm,
                                 const float* pt, uint64_t* probes, uint32_t* overflow, cudaStream_t s,
                                 const uint32_t* gmin = nullptr, bool exact_keys = true);
// per-row extra operand [n][8] = (-h hi, -h lo, 1, 1, 0, 0, 0, 0) from first-slice norms
cudaError_t launch_row_aug(const float* norms, uint32_t n, float* out, cudaStream_t s);

// Per-(query, candidate, checkpoint) partial sums as the survivor kernel evaluates
// them (dade_gpu_set_estimate_dump): {query, candidate id, checkpoint index, partial bits}.
struct EstimateDump {
    uint4* entries;
    uint32_t* count;              // running count (may exceed cap: entries past cap are dropped)
    uint32_t cap;
};

// Survivor kernel (stage 2 of the streaming scan) and candidate bucketing.
struct SurvArgs {
    const Survivor* surv;
    const uint32_t* surv_count;
    uint32_t surv_cap;
    const float* storage;
    const uint32_t* row_ids;
    uint32_t id_base;
    uint32_t dim;
    const float* queries;
    const uint32_t* r_global;
    const double* coeff;
    uint32_t n_dense_dims;        // d0
    uint32_t n_ckpt;
    uint16_t cps[64];             // checkpoint dims (those > d0 are tested here)
    uint32_t first_ckpt;          // index of the first checkpoint after d0
    uint32_t* cand_q;             // candidates: query ...
    uint64_t* cand_key;           // ... and (dist, id) key
    uint32_t* cand_count;
    uint32_t cand_cap;
    uint32_t* q_count;            // per-query candidate counts
    uint64_t* qslots;             // nullable: per-query candidate slots [nq][qslot_cap]; the overflow
    uint32_t qslot_cap;           //   past qslot_cap goes to cand_q / cand_key
    uint32_t* cand_total;         // nullable: candidates of the launch (qslots mode census)
    unsigned long long* counters; // [1] dims
    uint32_t* surv_max;           // running max of the survivor count (overflow check)
    uint32_t vec4;                // dim, d0 and every checkpoint are multiples of 4 (16-byte staging)
    uint32_t measure;             // failure accounting: a pruned pair is carried to the full dim, then
                                  //   counters[8] += exact <= r (eligible), counters[9] += eligible && pruned
    EstimateDump dump;            // nullable entries: every checkpoint partial the kernel evaluates
    uint32_t* row_dims;           // nullable [rows]: max dims any pair of the row reached (B_union census)
};
cudaError_t launch_advance_survivors(const SurvArgs& a, uint32_t max_entries, cudaStream_t s);
cudaError_t launch_merge_slots(const uint64_t* qslots, uint32_t qslot_cap, const uint32_t* q_count,
                               const uint32_t* cand_q, const uint64_t* cand_key, const uint32_t* cand_count,
                               uint32_t cand_cap, uint32_t nq, uint32_t K, uint64_t* out_keys, uint32_t* out_count,
                               cudaStream_t s, uint32_t* r_global = nullptr,
                               uint32_t* res_ids = nullptr, float* res_dists = nullptr,
                               uint32_t* res_counts = nullptr);
cudaError_t launch_scan(const ScanArgs& a, const ChunkTable& ct, const CUtensorMap& tmap,
                        const CUtensorMap& tmap_norms, uint32_t grid, bool sqrt_key, cudaStream_t s);
cudaError_t launch_row_norms(const float* rows, uint32_t n, uint32_t dim, uint32_t d0, float* out, cudaStream_t s);
cudaError_t launch_merge_segments(const uint64_t* seg_keys, const uint32_t* seg_count, uint32_t nq,
                                  uint32_t n_slots, uint32_t K, uint64_t* out_keys,
                                  uint32_t* out_count, cudaStream_t s);
cudaError_t launch_merge_blocks(const uint64_t* keys, uint32_t G, uint32_t nq, uint32_t K,
                                uint64_t* out_keys, uint32_t* out_count, cudaStream_t s);
cudaError_t launch_keys_to_results(const uint64_t* keys, const uint32_t* count, uint32_t nq,
                                   uint32_t K, uint32_t* ids, float* dists, uint32_t* counts_out,
                                   cudaStream_t s);

// coarse.cu: tensor-core coarse ranking with an exact boundary
cudaError_t launch_coarse_tc(const float* centroids, uint32_t n_cen, const float* queries, uint32_t nq, uint32_t dim,
                             uint32_t n_probe, float* cnorm, float* qnorm, float* pt, uint64_t* probes,
                             uint32_t* overflow, cudaStream_t s);

// prep.cu
cudaError_t launch_fill_u32(uint32_t* p, uint32_t v, size_t n, cudaStream_t s);
// seed.cu: the list-major radius seed with a TMA/mbarrier pipeline (dim <= 256, K <= 128)
// dims per TMA slice of the persistent seed's ring: {8 dims, 256 rows} boxes, 32-byte
// row segments, 32B-swizzled (seed.cu)
constexpr int kSeedSlice = 8;
struct SeedListArgs {
    const uint32_t* counts;         // rank-bucket-0 query count per list (GroupArgs::counts)
    const uint32_t* bucket_off;
    const uint32_t* bucket_q;
    const uint32_t* seed_goff;      // [n_lists + 1] seed-group prefix
    const uint32_t* seed_glist;     // [groups] list of each seed group
    uint32_t n_lists;
    const uint32_t* list_offsets;
    const uint32_t* row_ids;        // nullable: ids = id_base + row
    uint32_t id_base;
    uint32_t dim, K, S;
    const float* queries;
    uint32_t* r_global;
    uint64_t* out_keys;
    uint32_t* out_count;
    uint64_t nz2;                   // 0x8000000080000000 (sq_step2's opaque -0.0 pair)
    uint32_t* order;                // nullable scratch [groups]: persistent kernel's costliest-first group order
    unsigned long long* census;     // nullable: += rows x queries x dim of every group scored (profiling)
    unsigned long long* counters;   // nullable: [2] += the rows' bytes each group loads (B_read)
};
bool seed_tma_ok(uint32_t dim, uint32_t K);
// work: one zeroed-per-launch counter word (persistent variant); nullptr: one CTA per group
cudaError_t launch_seed_tma(const SeedListArgs& a, const CUtensorMap& tmap, uint32_t max_groups, cudaStream_t s,
                            uint32_t* work = nullptr);

cudaError_t launch_seed_radius_lists(const uint32_t* counts, const uint32_t* bucket_off, const uint32_t* bucket_q,
                                     const uint32_t* seed_goff, const uint32_t* seed_glist, uint32_t n_lists,
                                     uint32_t max_groups,
                                     const uint32_t* list_offsets, const float* storage,
                                     const uint32_t* row_ids, uint32_t id_base, uint32_t dim, const float* queries,
                                     uint32_t K, uint32_t S, uint32_t* r_global, uint64_t* out_keys,
                                     uint32_t* out_count, cudaStream_t s);
cudaError_t launch_seed_radius(const uint64_t* probes, uint32_t n_probe, const uint32_t* list_offsets,
                               const float* storage, const uint32_t* row_ids, uint32_t dim, const float* queries,
                               uint32_t nq, uint32_t K, uint32_t S, uint32_t* r_global, uint64_t* out_keys,
                               uint32_t* out_count, cudaStream_t s);
// fix / fix_n / fix_cap (nullable): a launch-wide list for the elements whose rounding the tensor-core
// sum cannot decide; a second kernel recomputes them one warp each (else each CTA recomputes its own)
cudaError_t launch_rotate(const double* W, uint32_t dim, const float* in, uint32_t n, float* out,
                          cudaStream_t s, uint2* fix = nullptr, uint32_t* fix_n = nullptr, uint32_t fix_cap = 0);
// Probe grouping (K3): probe keys [nq x nprobe] (low 32 bits = list id) ->
// per (rank bucket, list) query buckets and work items, ordered by rank bucket.
struct GroupArgs {
    const uint64_t* probes;
    uint32_t nq, n_probe, n_lists;
    const uint32_t* list_offsets;   // [n_lists + 1] device row prefix sums (a list absent
                                    // from this shard has zero length)
    uint32_t n_rb;                  // rank buckets
    uint32_t rb_end[8];             // exclusive probe-rank bound of each bucket
    uint32_t* counts;               // [n_rb * n_lists]
    uint32_t* cursor;               // [n_rb * n_lists]
    uint32_t* bucket_off;           // [n_rb * n_lists]
    uint32_t* item_off;             // [n_rb * n_lists]
    uint32_t* bucket_q;             // [nq * n_probe]
    uint32_t* bucket_slot;          // [nq * n_probe]
    WorkItem* items;                // [max_items]
    size_t max_items;               // capacity of items (upper bound of n_items[0])
    uint32_t* n_items;              // [2]: all items, rank-bucket-0 items
    uint32_t max_item_rows;         // 0: one item per (list, query chunk); else split rows
    uint32_t rank0_item_rows;       // row piece of rank-bucket-0 entries (0: max_item_rows)
    uint32_t q_chunk;               // queries per work item (kQC; 32 for the streaming filter)
    uint32_t seed_skip, seed_min;   // rank-0 lists of >= seed_min rows skip their first seed_skip rows
    uint32_t piece_major = 0;       // items ordered row piece major (the flat scan): shared pieces stay L2-hot
    uint32_t* seed_goff;            // nullable [n_lists + 1]: prefix of ceil(rank-0 count / kSeedGroup)
    uint32_t* seed_glist;           // nullable [seed groups]: the list of each seed group
};
cudaError_t launch_group(const GroupArgs& g, cudaStream_t s);
cudaError_t launch_local_probes(uint64_t* probes, uint32_t nq, uint32_t n_probe, const uint32_t* list_offsets,
                                uint32_t n_lists, cudaStream_t s);

cudaError_t launch_evaluate(const float* o, const float* q, const float* r, uint32_t n, uint32_t dim,
                            const uint32_t* cps, const double* coeff, const double* scale,
                            uint32_t n_ckpt, uint8_t* pruned, float* dist, uint8_t* exact,
                            uint32_t* dims_used, unsigned long long* counters, cudaStream_t s);
cudaError_t launch_partial_sums(const float* o, const float* q, uint32_t n, uint32_t dim,
                                const uint32_t* cps, uint32_t n_ckpt, float* out, cudaStream_t s);
cudaError_t launch_pair_partials(const float* data, uint32_t dim, const uint32_t* pi,
                                 const uint32_t* pj, uint64_t n, const uint32_t* cps,
                                 uint32_t n_ckpt, float* out, cudaStream_t s);

// build.cu: the index-build side (covariance, k-means, ground truth) in the
// reference's fp64 arithmetic
cudaError_t launch_covariance(const float* x, uint32_t n, uint32_t dim, double* mean, double* cov, cudaStream_t s);
size_t kmpp_block_count(uint32_t n);
// rng_state [3] zeroed: position in raw, error flag, first pick; picks (nullable) [n_clusters]
cudaError_t launch_kmpp_seed(const float* x, uint32_t n, uint32_t dim, uint32_t n_clusters, const uint64_t* raw,
                             uint32_t n_raw, uint32_t* rng_state, double* dist2, double* block_sums,
                             float* centroids, uint32_t* picks, cudaStream_t s);
cudaError_t launch_km_assign(const uint64_t* probes, uint32_t n, uint32_t* assign, uint32_t* changed,
                             cudaStream_t s);
// temp == nullptr: *temp_bytes = the radix sort's scratch size
cudaError_t launch_km_sort(const uint32_t* assign, uint32_t n, uint32_t n_clusters, uint64_t* keys_in,
                           uint64_t* keys_out, uint32_t* offsets, void* temp, size_t* temp_bytes, cudaStream_t s);
cudaError_t launch_km_sums(const float* x, uint32_t dim, const uint64_t* sorted, const uint32_t* offsets,
                           uint32_t n_clusters, float* centroids, cudaStream_t s);
cudaError_t launch_km_reseed(const float* x, uint32_t n, uint32_t dim, uint32_t* assign, uint32_t largest,
                             uint32_t empty_c, float* centroids, unsigned long long* scratch, cudaStream_t s);
cudaError_t launch_gather_rows(const float* x, uint32_t dim, const uint64_t* sorted, uint32_t n, float* rows_out,
                               uint32_t* ids_out, cudaStream_t s);
cudaError_t launch_gt_scan(const float* base, uint32_t n, uint32_t row_stride, const float* queries, uint32_t nq,
                           uint32_t dim, const double* thr, uint32_t cap, uint32_t* cnt, double* cand_d,
                           uint32_t* cand_id, int n_sms, cudaStream_t s);
cudaError_t launch_gt_select(const uint32_t* cnt, uint32_t cap, const double* cand_d, const uint32_t* cand_id,
                             uint32_t nq, uint32_t k, uint32_t* out_ids, double* out_kth, uint32_t* overflow,
                             cudaStream_t s);

}  // namespace dade_gpu

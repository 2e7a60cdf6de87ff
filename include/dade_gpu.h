/*
 * dade_gpu.h — C ABI of the B200-native DADE distance-comparison hot path.
 *
 * One handle = one GPU context holding device-resident copies of the
 * artifacts the reference's search path reads (transform, IVF lists or flat
 * base rows, strategy tables). Calls on one handle are externally serialised
 * (SURVEY.md §8b "Threading"); every entry point returns a status code and
 * never throws. The C++ mirror of the reference API over this ABI is
 * include/dade_gpu.hpp; the Python mirror is paper_2411_17229_b200/.
 *
 * Reference interfaces replaced (paths relative to /root/reference):
 *   dade_gpu_set_transform   OrthoTransform fields      proj/include/dade/transform.hpp:42-64
 *   dade_gpu_rotate          apply_transform            proj/src/transform.cpp:221-228, 295-304
 *   dade_gpu_set_ivf         IvfIndex (DIVF field order) proj/src/ivf.cpp:233-247, 249-279
 *   dade_gpu_set_base        linear_scan's VectorSet    proj/src/knn.cpp:31-41
 *   dade_gpu_set_strategy    DadeStrategy / AdsamplingStrategy / FdScanningStrategy
 *                            precomputed tables         proj/src/estimator.cpp:99-177
 *   dade_gpu_set_strategy_dade  DadeStrategy ctor incl. its ConfigError checks
 *                                                       proj/src/estimator.cpp:115-152
 *   dade_gpu_ivf_search      IvfIndex::search, batched  proj/src/ivf.cpp:207-231
 *   dade_gpu_ivf_search_batches  a loop of IvfIndex::search over query batches, pipelined
 *                                                       proj/src/bench.cpp:48-75
 *   dade_gpu_ivf_search_keys_begin/_end  the probe loop of IvfIndex::search split at its
 *                            nearest list, so list shards share one heap threshold
 *                                                       proj/src/ivf.cpp:221-229
 *   dade_gpu_flat_search     linear_scan, batched       proj/src/knn.cpp:31-41
 *   dade_gpu_dco_evaluate    DcoStrategy::evaluate      proj/include/dade/estimator.hpp:64-74
 *   dade_gpu_partial_sums    partial_sqdist at every checkpoint
 *                                                       proj/src/estimator.cpp:74-82
 *   dade_gpu_calibrate       calibrate                  proj/src/calibration.cpp:109-146
 *   dade_gpu_comm_create / dade_gpu_sharded_ivf_search / _flat_search
 *                            IvfIndex::search / linear_scan over list / row shards,
 *                            NCCL exchange
 *   dade_gpu_covariance      compute_covariance         proj/src/transform.cpp:68-95
 *   dade_gpu_kmeans          kmeans                     proj/src/ivf.cpp:24-143
 *   dade_gpu_ivf_build       IvfIndex::build            proj/src/ivf.cpp:145-192
 *   dade_gpu_ground_truth    compute_ground_truth       proj/src/dataset_io.cpp:101-135
 *   dade_gpu_set_estimate_dump / _get_estimate_dump
 *                            partial_sqdist + dade_estimate per (query, candidate, step)
 *                                                       proj/src/estimator.cpp:74-91
 *
 * Status codes mirror the reference's exception split
 * (proj/include/dade/error.hpp:10-19, proj/tools/dade_cli.cpp:407-419).
 */
#ifndef DADE_GPU_H_
#define DADE_GPU_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    DADE_GPU_OK = 0,
    DADE_GPU_RUNTIME_ERROR = 1, /* std::runtime_error (IO / corruption)           */
    DADE_GPU_CONFIG_ERROR = 2,  /* dade::ConfigError (mismatched artifacts)        */
    DADE_GPU_INVALID_INPUT = 3, /* dade::InvalidInput (precondition violated)      */
    DADE_GPU_CUDA_ERROR = 4     /* CUDA runtime / launch failure                   */
};

/* strategy kinds (proj/include/dade/bench.hpp:19 DcoKind, hot-path subset) */
enum { DADE_GPU_FD = 0, DADE_GPU_ADS = 1, DADE_GPU_DADE = 2 };

/* search flags */
enum {
    DADE_GPU_QUERIES_RAW = 1u << 0, /* queries are in the raw basis: rotate on device first   */
    DADE_GPU_DEVICE_PTRS = 1u << 1, /* every array argument is a device pointer; the call is
                                       asynchronous on the handle's stream (no H2D/D2H)      */
    DADE_GPU_MEASURE_FAILURES = 1u << 2 /* DcoStats::measure_failures: the search also fills
                                       stats->eligible / failures (estimator.cpp:24-33); every
                                       pruned pair is carried to the full dim for its exact
                                       distance, so this is the reference's untimed second
                                       pass (bench.cpp:65-73), not a serving mode. ivf_search
                                       and flat_search only.                                   */
};

typedef struct dade_gpu_ctx dade_gpu_ctx;

/* DcoStats counters (proj/include/dade/estimator.hpp:24-49); accumulated into. */
typedef struct {
    uint64_t total_dco;
    uint64_t dims_accumulated;
    uint64_t eligible;
    uint64_t failures;
} dade_gpu_stats;

const char* dade_gpu_last_error(void);
const char* dade_gpu_version(void);

int dade_gpu_create(int device, dade_gpu_ctx** out);
int dade_gpu_destroy(dade_gpu_ctx* ctx);
/* Work on a caller-owned cudaStream_t (NULL = the handle's own stream). */
int dade_gpu_set_stream(dade_gpu_ctx* ctx, void* cuda_stream);
int dade_gpu_synchronize(dade_gpu_ctx* ctx);
/* The stream the handle's work runs on (its own, or the one set_stream gave). */
int dade_gpu_get_stream(dade_gpu_ctx* ctx, void** cuda_stream);
/* Dim of the uploaded IVF index / flat base (nullable outputs; CONFIG_ERROR when
 * a requested one is absent). */
int dade_gpu_index_dims(dade_gpu_ctx* ctx, uint32_t* ivf_dim, uint32_t* base_dim);

/* Column-major f64 D x D matrix (column k = k-th direction) + nonincreasing
 * variances; the lambda prefix sums are derived exactly as on load
 * (proj/src/transform.cpp:21-25, 338-342). */
int dade_gpu_set_transform(dade_gpu_ctx* ctx, uint32_t dim, const double* matrix,
                           const double* eigenvalues);

/* IVF lists in DIVF field order. layout 0 = contiguous (split == dim),
 * 1 = split (per-list head block [len x split] then tail block). Host pointers. */
int dade_gpu_set_ivf(dade_gpu_ctx* ctx, uint32_t dim, uint32_t count, uint32_t n_clusters,
                     uint32_t layout, uint32_t split, const float* centroids,
                     const uint32_t* offsets, const uint32_t* ids, const float* storage);

/* Multi-GPU list sharding: keep only lists with mask[c] != 0
 * on this device. Centroids stay replicated so coarse ranking is global. */
int dade_gpu_set_ivf_shard(dade_gpu_ctx* ctx, const uint8_t* list_mask);

/* Flat base rows (linear_scan). Returned ids are row + id_base, so a row shard
 * of a larger base reports global ids. Host pointer. */
int dade_gpu_set_base(dade_gpu_ctx* ctx, uint32_t dim, uint32_t count, const float* data,
                      uint32_t id_base);

/* Precomputed strategy tables: n checkpoints (ascending, < dim), reject_coeff[i]
 * (reject iff partial > coeff * r^2), est_scale[i]. n == 0 (or kind == FD) is
 * FdScanningStrategy. */
int dade_gpu_set_strategy(dade_gpu_ctx* ctx, uint32_t kind, uint32_t dim, uint32_t n,
                          const uint32_t* checkpoints, const double* reject_coeff,
                          const double* est_scale);

/* DadeStrategy(t, cal, delta_d) on the handle's transform, with the
 * reference's validation (ConfigError on step / grid mismatch). */
int dade_gpu_set_strategy_dade(dade_gpu_ctx* ctx, uint32_t delta_d, uint32_t cal_delta_d,
                               uint32_t n, const uint32_t* cal_checkpoints,
                               const double* cal_epsilons);

/* AdsamplingStrategy(dim, delta_d, eps0). */
int dade_gpu_set_strategy_ads(dade_gpu_ctx* ctx, uint32_t dim, uint32_t delta_d, double eps0);

/* apply_transform: out = rotate(in), n rows of the handle's dim. */
int dade_gpu_rotate(dade_gpu_ctx* ctx, const float* in, uint32_t n, float* out, uint32_t flags);

/* Batched IvfIndex::search. Per query: up to k results ascending by
 * (distance, id) in out_ids/out_dists [nq x k]; out_counts[q] < k means
 * truncated. stats (nullable) accumulates. */
int dade_gpu_ivf_search(dade_gpu_ctx* ctx, const float* queries, uint32_t nq, uint32_t k,
                        uint32_t n_probe, uint32_t flags, uint32_t* out_ids, float* out_dists,
                        uint32_t* out_counts, dade_gpu_stats* stats);

/* A sequence of n_batches batched IvfIndex::search calls over host buffers
 * (queries[b] [nq x dim] -> out_ids[b] / out_dists[b] / out_counts[b]),
 * pipelined: batch b+1's host->device copy and batch b-1's device->host copy
 * run under batch b's search. Results are those of n_batches calls of
 * dade_gpu_ivf_search (a batch whose worklist overflowed is redone before
 * return). Pinned host buffers let the copies overlap; DEVICE_PTRS is refused.
 * Replaces a loop of IvfIndex::search over query batches (the serving loop of
 * proj/src/bench.cpp:48-75 measure(), batched). */
int dade_gpu_ivf_search_batches(dade_gpu_ctx* ctx, uint32_t n_batches, const float* const* queries,
                                uint32_t nq, uint32_t k, uint32_t n_probe, uint32_t flags,
                                uint32_t* const* out_ids, float* const* out_dists,
                                uint32_t* const* out_counts, dade_gpu_stats* stats);

/* Batched linear_scan over the flat base. After dade_gpu_flat_partition the
 * scan visits the base in data order (every partition probed, each query's
 * nearest partition first), else in row order; either way every base row is a
 * candidate and FD results are identical (ties by id). */
int dade_gpu_flat_search(dade_gpu_ctx* ctx, const float* queries, uint32_t nq, uint32_t k,
                         uint32_t flags, uint32_t* out_ids, float* out_dists,
                         uint32_t* out_counts, dade_gpu_stats* stats);

/* Like the two searches, but leave the packed per-query top-K keys
 * ((float_bits(dist) << 32) | id, ascending; UINT64_MAX = empty) in
 * out_keys [nq x k] for a cross-GPU merge. Device pointers only. */
int dade_gpu_ivf_search_keys(dade_gpu_ctx* ctx, const float* d_queries, uint32_t nq, uint32_t k,
                             uint32_t n_probe, uint32_t flags, uint64_t* d_out_keys,
                             dade_gpu_stats* stats);
int dade_gpu_flat_search_keys(dade_gpu_ctx* ctx, const float* d_queries, uint32_t nq,
                              uint32_t k, uint32_t flags, uint64_t* d_out_keys,
                              dade_gpu_stats* stats);

/* The coarse ranking of IvfIndex::search (proj/src/ivf.cpp:215-219) alone:
 * rotation when QUERIES_RAW, then per query the n_probe nearest centroids as
 * packed keys ((float_bits(l2_sq) << 32) | list, ascending) into d_probes
 * [nq x n_probe] and the rotated queries into d_q_rot [nq x dim] (nullable).
 * Device pointers (DEVICE_PTRS required). Multi-GPU: each rank ranks its own
 * query slice; the slices are all-gathered and handed to _begin. */
int dade_gpu_coarse_probes(dade_gpu_ctx* ctx, const float* d_queries, uint32_t nq,
                           uint32_t n_probe, uint32_t flags, float* d_q_rot, uint64_t* d_probes);

/* dade_gpu_ivf_search_keys in two phases, for list-sharded multi-GPU search.
 * _begin scans every query's nearest LOCAL list (its first probe with rows on
 * this shard) and copies the per-query radius (fp32 bits as u32, +inf =
 * 0x7f800000) to d_radius [nq] on the context's stream. The caller min-reduces
 * d_radius across shards (NCCL all-reduce MIN; as int32 the bits order like
 * the distances), then _end scans the other lists with the reduced radius and
 * completes d_out_keys. A shard whose nearest local list is far from a query
 * would otherwise scan its lists with a radius no candidate there can beat.
 * d_probes (nullable): the queries' probe keys from dade_gpu_coarse_probes
 * (then d_queries are rotated queries, no QUERIES_RAW); d_queries must stay
 * valid until _end. Device pointers only; no other search may run on the
 * context in between. */
int dade_gpu_ivf_search_keys_begin(dade_gpu_ctx* ctx, const float* d_queries, uint32_t nq,
                                   uint32_t k, uint32_t n_probe, uint32_t flags,
                                   const uint64_t* d_probes, uint64_t* d_out_keys,
                                   uint32_t* d_radius);
int dade_gpu_ivf_search_keys_end(dade_gpu_ctx* ctx, const uint32_t* d_radius,
                                 dade_gpu_stats* stats);
/* The flat scan in the same two phases (row-sharded linear_scan): _begin runs the
 * radius seed over this device's first rows, dade_gpu_ivf_search_keys_end (shared)
 * runs the streaming passes with the min-reduced radius. */
int dade_gpu_flat_search_keys_begin(dade_gpu_ctx* ctx, const float* d_queries, uint32_t nq,
                                    uint32_t k, uint32_t flags, uint64_t* d_out_keys,
                                    uint32_t* d_radius);

/* Merge G gathered key blocks [G x nq x k] (e.g. an NCCL all-gather) into the
 * global top-K: ids/dists/counts as dade_gpu_ivf_search. Device pointers. */
int dade_gpu_merge_keys(dade_gpu_ctx* ctx, const uint64_t* d_keys, uint32_t n_blocks,
                        uint32_t nq, uint32_t k, uint32_t* d_out_ids, float* d_out_dists,
                        uint32_t* d_out_counts);

/* DcoStrategy::evaluate for n independent (o_i, q_i, r_i) with the current
 * strategy. Host pointers unless DEVICE_PTRS. */
int dade_gpu_dco_evaluate(dade_gpu_ctx* ctx, const float* o, const float* q, const float* r,
                          uint32_t n, uint32_t flags, uint8_t* pruned, float* distance,
                          uint8_t* distance_exact, uint32_t* dims_used, dade_gpu_stats* stats);

/* Running partial sums of every pair at each checkpoint of the current
 * strategy and at the full dim: out [n x (n_ckpt + 1)] f32. The estimator
 * value of step i is est_scale[i] * out[p, i] (dade_estimate). */
int dade_gpu_partial_sums(dade_gpu_ctx* ctx, const float* o, const float* q, uint32_t n,
                          uint32_t flags, float* out);

/* calibrate(t, data, p_s, delta_d, n_pairs, seed) over n rotated rows with
 * the handle's transform: writes the checkpoint grid and epsilons (arrays of
 * at least dim / delta_d entries) and returns the count in *n_out. */
int dade_gpu_calibrate(dade_gpu_ctx* ctx, const float* data, uint32_t n, double p_s,
                       uint32_t delta_d, uint64_t n_pairs, uint64_t seed, uint32_t flags,
                       uint32_t* checkpoints, double* epsilons, uint32_t* n_out);

/* Debug: the last scan's device counters [0..15] (total_dco, dims, bytes, debug,
 * per-pass census [4..7], eligible, failures). */
int dade_gpu_debug_counters(dade_gpu_ctx* ctx, uint64_t* out16);

/* Per-(query, candidate, checkpoint) estimator values of the hot path, for
 * parity with partial_sqdist + dade_estimate (proj/src/estimator.cpp:74-91):
 * with capacity > 0, every checkpoint partial the survivor kernel of the
 * following searches evaluates is recorded (the dump is reset at each search's
 * start; pairs the tensor-core bound prunes are not evaluated exactly and so
 * are not recorded unless DADE_GPU_DEBUG=1 sends every pair to that kernel).
 * _get returns min(recorded, capacity, cap) entries: query index, candidate id,
 * checkpoint dim d, the fp32 partial sum over dims [0, d) and the estimate
 * est_scale(d) x partial; *n_total = entries recorded (may exceed capacity). */
int dade_gpu_set_estimate_dump(dade_gpu_ctx* ctx, uint32_t capacity);
int dade_gpu_get_estimate_dump(dade_gpu_ctx* ctx, uint32_t cap, uint32_t* q, uint32_t* ids, uint32_t* dims,
                               float* partial, double* estimate, uint64_t* n_total);

/* Debug: per-query radius (float bits) left by the last IVF search. */
int dade_gpu_debug_radius(dade_gpu_ctx* ctx, uint32_t* out, uint32_t nq);

/* ---- index build on the GPU, reference arithmetic ---------- */

/* compute_covariance (proj/src/transform.cpp:68-95): fp64 mean [dim] and
 * covariance [dim x dim] row-major (1/n, centred) of n rows, bit-identical to
 * the reference. data: device if DEVICE_PTRS; mean / cov: host. */
int dade_gpu_covariance(dade_gpu_ctx* ctx, const float* data, uint32_t n, uint32_t dim, uint32_t flags,
                        double* mean, double* cov);

/* kmeans(data, n_clusters, max_iters, seed) (proj/src/ivf.cpp:24-143): k-means++
 * seeding on the reference's mt19937_64 stream, Lloyd iterations with its
 * early stop and empty-cluster re-seeding; centroids [n_clusters x dim],
 * assignments [n] and the iteration count equal the reference's. Drops any IVF
 * index uploaded to the context. data: device if DEVICE_PTRS, else host;
 * outputs: host or device memory (nullable ones are skipped). */
int dade_gpu_kmeans(dade_gpu_ctx* ctx, const float* data, uint32_t n, uint32_t dim, uint32_t n_clusters,
                    uint32_t max_iters, uint64_t seed, uint32_t flags, float* centroids,
                    uint32_t* assignments, uint32_t* iterations);

/* IvfIndex::build(data, n_clusters, contiguous, .., max_iters, seed)
 * (proj/src/ivf.cpp:145-192): the k-means above, posting lists in cluster
 * order with ids ascending. The built index is installed on the context (as
 * dade_gpu_set_ivf would) and its DIVF arrays copied out: centroids
 * [n_clusters x dim], offsets [n_clusters + 1], ids [n], storage [n x dim]
 * (nullable). */
int dade_gpu_ivf_build(dade_gpu_ctx* ctx, const float* data, uint32_t n, uint32_t dim, uint32_t n_clusters,
                       uint32_t max_iters, uint64_t seed, uint32_t flags, float* centroids,
                       uint32_t* offsets, uint32_t* ids, float* storage);

/* compute_ground_truth (proj/src/dataset_io.cpp:101-135): per query the k
 * nearest of n base rows by (l2_sq_double, id), exactly the reference's ids
 * (k <= 2048). out_ids [nq x k]. Pointers: device if DEVICE_PTRS, else host. */
int dade_gpu_ground_truth(dade_gpu_ctx* ctx, const float* base, uint32_t n, const float* queries, uint32_t nq,
                          uint32_t dim, uint32_t k, uint32_t flags, uint32_t* out_ids);

/* ---- multi-GPU over NCCL (SURVEY.md §8b init_nccl / sharded_*, §8e) --------
 * One process (or host thread) per GPU, one handle + one communicator each.
 * libnccl is resolved at run time: the copy already in the process, else
 * libnccl.so.2. Rank 0 creates the unique id, the host distributes it (MPI,
 * torch.distributed, a file ...), every rank creates its communicator on its
 * handle. */
#define DADE_GPU_NCCL_ID_BYTES 128
typedef struct dade_gpu_comm dade_gpu_comm;
int dade_gpu_nccl_unique_id(uint8_t* id_out /* [DADE_GPU_NCCL_ID_BYTES] */);
int dade_gpu_comm_create(dade_gpu_ctx* ctx, int nranks, int rank, const uint8_t* id, dade_gpu_comm** out);
int dade_gpu_comm_destroy(dade_gpu_comm* comm);

/* List-sharded IvfIndex::search, query-owner scheme: every rank's handle holds
 * the replicated centroids + transform + strategy and its shard of the lists
 * (dade_gpu_set_ivf + dade_gpu_set_ivf_shard); every rank passes its own nq
 * queries (the same nq on all ranks) and receives their top-k, bit-identical
 * in FD mode to an unsharded search. Steps: coarse ranking of the own queries,
 * NCCL all-gather of rotated queries + probes, phase 1 (the shard owning a
 * query's nearest list seeds it), NCCL all-reduce(MIN) of the per-query
 * radius, phase 2 (the other local lists), NCCL send/recv of each query's
 * per-shard top-k to its owner, device merge. Host buffers unless
 * DEVICE_PTRS; QUERIES_RAW rotates first. stats: this rank's DcoStats. */
int dade_gpu_sharded_ivf_search(dade_gpu_comm* comm, const float* queries, uint32_t nq, uint32_t k,
                                uint32_t n_probe, uint32_t flags, uint32_t* out_ids, float* out_dists,
                                uint32_t* out_counts, dade_gpu_stats* stats);

/* Row-sharded linear_scan: every rank's handle holds a contiguous row block
 * (dade_gpu_set_base with id_base = its first row); the same nq queries on
 * every rank; every rank receives the global top-k. Radius seed per shard,
 * NCCL all-reduce(MIN) of the radius, the streaming passes, NCCL all-gather
 * of the key blocks, device merge. */
int dade_gpu_sharded_flat_search(dade_gpu_comm* comm, const float* queries, uint32_t nq, uint32_t k,
                                 uint32_t flags, uint32_t* out_ids, float* out_dists, uint32_t* out_counts,
                                 dade_gpu_stats* stats);

/* Number of CUDA kernels this handle launched so far (bench evidence). */
uint64_t dade_gpu_launch_count(dade_gpu_ctx* ctx);

/* Rows of each probed list's head (the flat base's first rows) the radius seed
 * scores exactly; 0 restores the default (1024, ~1 MB of rows per IVF list above
 * dim 256). A tuning knob: fewer seeded rows give a looser first radius. */
int dade_gpu_set_seed_rows(dade_gpu_ctx* ctx, uint32_t rows);

/* Repeated IVF searches of one shape replay a captured CUDA graph of the search
 * body (coarse ranking .. merges; the first call runs eagerly, the second is
 * captured). 0 turns the capture off for this handle (every search eager),
 * 1 (the default) back on. Results are identical either way. */
int dade_gpu_set_graphs(dade_gpu_ctx* ctx, int on);

/* Data-ordered flat scan: partitions the uploaded flat base (dade_gpu_set_base)
 * into n_parts k-means cells on the GPU (kmeans of proj/src/ivf.cpp:24-143,
 * max_iters, seed), which become this handle's IVF index (replacing any
 * uploaded one); dade_gpu_flat_search then probes every cell, the query's
 * nearest first, so its radius is tight from the first rows scanned. The
 * visiting order of linear_scan (proj/src/knn.cpp:31-41) changes, the candidate
 * set does not. n_parts = 0 drops the partition (row-order scan). A later
 * dade_gpu_set_base / _set_ivf / _ivf_build drops it too. */
int dade_gpu_flat_partition(dade_gpu_ctx* ctx, uint32_t n_parts, uint32_t max_iters, uint64_t seed);

/* Measured device time (ms) of the DCO scan kernel(s) in the last search
 * call, via CUDA events on the launching stream, and its algorithmic bytes
 * (slice bytes read + list metadata). Requires dade_gpu_set_profiling(1). */
int dade_gpu_set_profiling(dade_gpu_ctx* ctx, int on);
int dade_gpu_last_scan_profile(dade_gpu_ctx* ctx, double* scan_ms, double* scan_bytes,
                               double* total_ms);
/* Device time (ms) of the streaming tensor-core filter launches of the last
 * search (the dominant kernel) and how many there were. Requires profiling. */
int dade_gpu_last_filter_profile(dade_gpu_ctx* ctx, double* filter_ms, int* n_launches);
/* Device time (ms) of the persistent radius-seed launch of the last search and
 * the (row, query, dim) triples it summed exactly. Requires profiling; 0 when
 * that kernel did not run. */
int dade_gpu_last_seed_profile(dade_gpu_ctx* ctx, double* seed_ms, double* pair_dims);
/* B_union of the last profiled streaming search: the bytes any
 * scan making the same decisions must read at least -- per base row, 4 x the
 * most dims any of its (query, row) pairs used (d0 for every row of a probed
 * list, dim for the seeded rows, the survivors' prune / full dims) -- and the
 * rows touched. With dade_gpu_last_scan_profile's scan_bytes (B_read: the
 * slice bytes the kernels loaded, seed rows and survivor chunks included, plus
 * list metadata) this gives the over-fetch B_read / B_union. 0 unless the
 * search ran the streaming path with profiling on. */
int dade_gpu_last_union_profile(dade_gpu_ctx* ctx, double* b_union, double* rows);

#ifdef __cplusplus
}
#endif
#endif /* DADE_GPU_H_ */

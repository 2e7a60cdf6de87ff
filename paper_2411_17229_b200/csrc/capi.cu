// Host runtime + C ABI of libdade_gpu.so (include/dade_gpu.h).
//
// The handle owns every device buffer (grow-only workspaces, so steady-state
// searches allocate nothing) and one CUDA stream. A search is a fixed,
// host-sync-free launch sequence on that stream:
//   [rotate] -> coarse scan (centroids, K = n_probe) -> segment merge ->
//   group probes into per-list query buckets -> DCO scan -> segment merge
// so it is capturable in a CUDA graph; the host only synchronises when it has
// to copy results or counters back.
#include <algorithm>
#include <array>
#include <chrono>
#include <utility>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <limits>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/dade_gpu.h"
#include "kernels.h"
#include <cudaTypedefs.h>

using namespace dade_gpu;

namespace {

thread_local std::string g_last_error;

// Device counters of a search: [0] total_dco, [1] dims_accumulated, [2] bytes,
// [3] debug, [4..7] per-pass census, [8] eligible, [9] failures.
constexpr size_t kCounterBytes = 128;

bool env_flag(const char* name) {
    const char* e = std::getenv(name);
    return e && e[0] == '1';
}

struct ApiError : std::runtime_error {
    int code;
    ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void fail(int code, const std::string& msg) { throw ApiError(code, msg); }

void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) fail(DADE_GPU_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return DADE_GPU_OK;
    } catch (const ApiError& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("host allocation failed: ") + e.what();
        return DADE_GPU_RUNTIME_ERROR;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return DADE_GPU_RUNTIME_ERROR;
    }
}

// Bumped on every device (re)allocation: a captured search graph bakes buffer
// addresses into its launches, so its cache key carries this epoch.
uint64_t g_alloc_epoch = 0;

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    void* ensure(size_t bytes) {
        if (bytes <= cap && p) return p;
        ++g_alloc_epoch;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes, 256);
        cuda_check(cudaMalloc(&p, want), "cudaMalloc");
        cap = want;
        return p;
    }
    template <class T>
    T* as() const { return static_cast<T*>(p); }
    void release() {
        if (p) {
            cudaFree(p);
            ++g_alloc_epoch;
        }
        p = nullptr;
        cap = 0;
    }
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf& operator=(DevBuf&& o) noexcept {  // takes o's allocation
        if (this != &o) {
            release();
            p = o.p;
            cap = o.cap;
            o.p = nullptr;
            o.cap = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }  // (dade_gpu_destroy frees while the device context is current)
};

// Checkpoint grid rule of CalibrationTable::expected_checkpoints
// (proj/src/calibration.cpp:74-81).
std::vector<uint32_t> expected_checkpoints(uint32_t dim, uint32_t delta_d) {
    std::vector<uint32_t> cps;
    for (uint64_t d = delta_d; d + 1 <= dim && d < dim; d += delta_d) cps.push_back((uint32_t)d);
    return cps;
}

// Dimension chunks: boundaries at every checkpoint and every kCH dims.
ChunkTable make_chunks(uint32_t dim, const std::vector<uint32_t>& cps) {
    ChunkTable ct{};
    ct.n_ckpt = (int)cps.size();
    uint32_t k = 0;
    size_t ci = 0;
    int n = 0;
    while (k < dim) {
        uint32_t e = std::min(dim, k + (uint32_t)kCH);
        int ck = -1;
        if (ci < cps.size() && cps[ci] <= e) {
            e = cps[ci];
            ck = (int)ci;
            ++ci;
        }
        if (n >= kMaxChunks) fail(DADE_GPU_INVALID_INPUT, "dimension too large for the chunk table");
        ct.end[n] = (uint16_t)e;
        ct.ckpt[n] = (int16_t)ck;
        ++n;
        k = e;
    }
    ct.n_chunks = n;
    ct.n_dense = n;
    for (int c = 0; c < n; ++c)
        if (ct.ckpt[c] >= 0) {
            ct.n_dense = c + 1;
            break;
        }
    bool al = (dim & 3u) == 0;
    for (int c = 0; c < n; ++c) al = al && (ct.end[c] & 3u) == 0;
    ct.vec_ok = al ? 1 : 0;
    const uint32_t dense_dims = ct.end[ct.n_dense - 1];
    ct.d_res = (al && dense_dims * kQS * 4 <= (uint32_t)kMaxResidentQBytes) ? (int)dense_dims : 0;
    // Tensor-core first-slice filter: needs checkpoints, resident queries and
    // dense chunk widths that are multiples of the MMA k (8).
    bool tc = ct.n_dense < ct.n_chunks && ct.d_res > 0;
    for (int c = 0; c < ct.n_dense; ++c) {
        const uint32_t lo = c == 0 ? 0u : ct.end[c - 1];
        tc = tc && ((ct.end[c] - lo) % 8u) == 0;
    }
    const char* env = std::getenv("DADE_GPU_NO_TC");
    if (env && env[0] == '1') tc = false;
    ct.use_tc = tc ? 1 : 0;
    // ring depth: the filter holds a tile's boxes through its exact phase
    ct.n_buf = tc ? std::max(4, 2 * ct.n_dense + 2) : 4;
    ct.use_tma = 0;  // decided per launch (needs a tensor map of the rows)
    const char* dbg = std::getenv("DADE_GPU_DEBUG");
    ct.debug = dbg ? std::atoi(dbg) : 0;
    return ct;
}

// 2D tensor map over row-major fp32 rows [rows][dim]: box [kRT rows][kBox
// dims], 128-byte swizzle (matches swz() in scan.cu), OOB -> zeros.
bool make_row_tmap(CUtensorMap* m, const float* base, uint64_t rows, uint32_t dim, uint32_t box_rows = kRT) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                    &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            encode = nullptr;
        if (!encode) return false;
    }
    if (dim % 4 != 0 || dim < (uint32_t)kBox || rows == 0 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t gdim[2] = {dim, rows};
    cuuint64_t gstride[1] = {(cuuint64_t)dim * 4};
    cuuint32_t box[2] = {(cuuint32_t)kBox, (cuuint32_t)box_rows};
    cuuint32_t estride[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_1d_tmap(CUtensorMap* m, const float* base, uint64_t n) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                    &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            encode = nullptr;
        if (!encode) return false;
    }
    if (n == 0 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t gdim[1] = {n};
    cuuint64_t gstride[1] = {n * 4};  // unused for rank 1, but must be a valid array
    cuuint32_t box[1] = {(cuuint32_t)kRT};
    cuuint32_t estride[1] = {1};
    const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 1, const_cast<float*>(base), gdim, gstride, box,
                              estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// First-slice row norms of a row set (the tensor-core filter's |o|^2), cached
// per (rows, d0), plus their 1-D tensor map.
struct RowNorms {
    DevBuf buf;
    const float* rows = nullptr;
    uint32_t n = 0, dim = 0, d0 = 0;
    bool tm_ok = false;
    CUtensorMap map{};
    const float* get(const float* r, uint32_t nn, uint32_t d, uint32_t dd0, cudaStream_t s) {
        if (r != rows || nn != n || d != dim || dd0 != d0) {
            // padded by 8 floats: the kernel reads 16-byte aligned windows
            buf.ensure(((size_t)nn + 40) * 4);
            cuda_check(cudaMemsetAsync(buf.p, 0, ((size_t)nn + 40) * 4, s), "memset");
            cuda_check(launch_row_norms(r, nn, d, dd0, buf.as<float>(), s), "row norms");
            rows = r;
            n = nn;
            dim = d;
            d0 = dd0;
            tm_ok = true;  // windows are fetched with a plain bulk copy
        }
        return buf.as<float>();
    }
};

// Per-row extra K=8 operand of the tcgen05 filter, [rows][8] fp32 = (-h hi, -h lo,
// 1, 1, 0...), h = (1 - delta)|o_{0:d0}|^2 / 2 (umma.cu), TMA-loaded with 32B swizzle.
bool make_aug_tmap(CUtensorMap* m, const float* base, uint64_t rows, uint32_t box_rows) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                    &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            encode = nullptr;
        if (!encode) return false;
    }
    if (rows == 0 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t gdim[2] = {8, rows};
    cuuint64_t gstride[1] = {8 * 4};
    cuuint32_t box[2] = {8, box_rows};
    cuuint32_t estride[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Rows as {8 dims, 256 rows} 32B-swizzled TMA boxes (the radius seed's slices).
bool make_slice_tmap(CUtensorMap* m, const float* base, uint64_t rows, uint32_t dim) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault,
                                    &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            encode = nullptr;
        if (!encode) return false;
    }
    if (dim % 4 != 0 || rows == 0 || (reinterpret_cast<uintptr_t>(base) & 15)) return false;
    cuuint64_t gdim[2] = {dim, rows};
    cuuint64_t gstride[1] = {(cuuint64_t)dim * 4};
    cuuint32_t box[2] = {(cuuint32_t)kSeedSlice, 256};
    cuuint32_t estride[2] = {1, 1};
    return encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstride, box, estride,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct SliceTmap {
    const float* base = nullptr;
    uint64_t rows = 0;
    uint32_t dim = 0;
    bool ok = false;
    CUtensorMap map{};
    const CUtensorMap* get(const float* b, uint64_t r, uint32_t d) {
        if (b != base || r != rows || d != dim) {
            base = b;
            rows = r;
            dim = d;
            ok = make_slice_tmap(&map, b, std::max<uint64_t>(r, 1), d);
        }
        return ok ? &map : nullptr;
    }
};

struct RowAug {
    DevBuf buf;
    const float* rows = nullptr;
    uint32_t n = 0, dim = 0, d0 = 0;
    bool ok = false;
    CUtensorMap map{};
    const CUtensorMap* get(const float* r, uint32_t nn, uint32_t d, uint32_t dd0, const float* norms, cudaStream_t s) {
        if (r != rows || nn != n || d != dim || dd0 != d0) {
            buf.ensure(((size_t)nn + 1) * 32);
            cuda_check(launch_row_aug(norms, nn, buf.as<float>(), s), "row aug");
            rows = r;
            n = nn;
            dim = d;
            d0 = dd0;
            ok = make_aug_tmap(&map, buf.as<float>(), std::max<uint32_t>(nn, 1), 128);
        }
        return ok ? &map : nullptr;
    }
};

struct TmapCache {
    const float* base = nullptr;
    uint64_t rows = 0;
    uint32_t dim = 0;
    uint32_t box_rows = kRT;
    bool ok = false;
    CUtensorMap map{};
    explicit TmapCache(uint32_t br = kRT) : box_rows(br) {}
    const CUtensorMap& get(const float* b, uint64_t r, uint32_t d, bool& usable) {
        if (b != base || r != rows || d != dim) {
            base = b;
            rows = r;
            dim = d;
            ok = make_row_tmap(&map, b, r, d, box_rows);
        }
        usable = ok;
        return map;
    }
};

}  // namespace

namespace dade_gpu {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace dade_gpu

struct dade_gpu_ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    uint64_t launches = 0;

    // transform
    uint32_t t_dim = 0;
    DevBuf W;
    std::vector<double> lambda_prefix;

    // ivf
    bool has_ivf = false;
    bool sharded = false;  // set_ivf_shard removed lists with rows
    struct {  // results of the search in flight, written by its last slot merge when set
        uint32_t* ids = nullptr;
        float* dists = nullptr;
        uint32_t* counts = nullptr;
        bool done = false;
    } fo;
    uint32_t seed_rows_set = 0;  // dade_gpu_set_seed_rows (0: the default rule)
    bool dense_groups = false;   // this IVF search has >= 4 queries per list: full seed groups
    // two-phase search (dade_gpu_ivf_search_keys_begin/_end): 1 = stop before the
    // last pass, 2 = resume at it; the begun search's arguments
    int split = 0;
    struct {
        bool active = false;
        const float* d_q = nullptr;
        uint32_t nq = 0, k = 0, n_probe = 0;
        uint64_t* keys = nullptr;
        bool flat = false;
    } sp;
    uint32_t dim = 0, count = 0, n_clusters = 0;
    DevBuf centroids, storage, ids, offsets;
    std::vector<uint32_t> h_offsets;  // full index offsets (host)
    std::vector<uint32_t> dev_offsets;

    // flat base
    bool has_base = false;
    uint32_t b_dim = 0, b_count = 0, b_id_base = 0;
    DevBuf base;
    uint32_t flat_parts = 0;  // > 0: the IVF index holds the flat base in n k-means cells (dade_gpu_flat_partition)

    // strategy
    bool has_strategy = false;
    uint32_t s_kind = DADE_GPU_FD, s_dim = 0;
    std::vector<uint32_t> cps;
    std::vector<double> coeff, scale;
    DevBuf d_cps, d_coeff, d_scale;

    // workspaces
    DevBuf q_in, q_rot, probes, probe_count, c_seg_keys, c_seg_count, c_r;
    DevBuf g_counts, g_cursor, g_boff, g_ioff, bucket_q, bucket_slot, items, n_items;
    DevBuf seg_keys, seg_count, r_global, out_keys, out_count, out_ids, out_dists, out_counts, seed_keys, seed_count;
    DevBuf surv, surv_count, cand_q, cand_key, cand_count, q_count, q_off, q_cursor, bucket, surv_max, item_counter, seed_goff, seed_glist;
    DevBuf cnorm, qnorm, coarse_lo, coarse_overflow, q_norms, coarse_gmin;  // coarse_lo: p~ per (query, centroid)
    DevBuf coarse_cand, coarse_cnt, coarse_t0;  // fused large-nlist selection
    bool coarse_force_exact = false, coarse_tc_used = false;
    bool coarse_all = false;  // every centroid probed, no exact ranking (the data-ordered flat scan)
    bool coarse_exact_keys = false;  // probe keys exact and ascending (dade_gpu_coarse_probes), not only the set
    int n_sms = 148;
    uint32_t surv_cap_hint = 0;
    uint32_t surv_cap_used = 0;     // worklist capacity of the last streaming search (0: none)
    uint32_t* h_flags = nullptr;    // pinned [2]: surv_max, coarse overflow of the last search
    cudaStream_t copy_stream = nullptr;  // H2D of host query chunks (overlapped with rotation / coarse)
    cudaEvent_t copy_ev[9] = {};
    bool stage_one_chunk = false;   // staging: one chunk (the H2D is not on the critical path)
    bool qin_free_recorded = false; // copy_ev[8] marks q_in's last reader (the staging rotations)
    // pipelined batches (dade_gpu_ivf_search_batches): result double buffers, D2H stream
    cudaStream_t d2h_stream = nullptr;
    cudaEvent_t res_ev[2] = {}, d2h_ev[2] = {};
    DevBuf res_ids[2], res_dists[2], res_counts[2], batch_slot;
    unsigned long long* h_batch = nullptr;  // pinned [n][4]: surv_max, coarse overflow, total_dco, dims
    size_t h_batch_n = 0;
    uint32_t stage_n_probe = 0;     // > 0: stage_queries may also coarse-rank the chunks (IVF)
    bool probes_ready = false;      // probes of this search already computed per chunk
    DevBuf counters, phase;
    TmapCache tm_centroids, tm_storage, tm_base;
    TmapCache tm_queries{256};  // rotated queries, {32 dims, 256 rows} boxes (tcgen05 coarse GEMM)
    TmapCache tm_q128{128}, tm_c256{256};  // query-major fused coarse selection
    TmapCache tm32_storage{32}, tm32_base{32};
    RowNorms norms_storage, norms_base;
    RowAug aug_storage;
    SliceTmap seed_tm;
    DevBuf seed_work;  // persistent seed's group counter
    DevBuf rot_fix;    // rotation: launch-wide list of undecided elements [cap] uint2 + its counter
    DevBuf seed_order; // persistent seed's costliest-first group order
    DevBuf qslots;     // per-query candidate slots [nq][kQSlots] of a streaming pass
    DevBuf cand_total; // candidates of a pass (census, qslots mode)
    DevBuf flat_offsets;  // {0, b_count}: the flat base as one list
    CUtensorMap tm_none{};

    // failure accounting of the search in flight (DADE_GPU_MEASURE_FAILURES)
    bool measure = false;
    // per-(query, candidate, checkpoint) partials of the next searches (dade_gpu_set_estimate_dump)
    DevBuf dump_entries, dump_count;
    uint32_t dump_cap = 0;

    // profiling
    bool profiling = false;
    cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr, e3 = nullptr;
    cudaEvent_t ef[12] = {};  // filter launch start / end per pass (up to the flat scan's six passes)
    cudaEvent_t es[2] = {nullptr, nullptr};  // the persistent seed launch
    bool seed_profiled = false;
    double last_seed_ms = 0, last_seed_pair_dims = 0;
    DevBuf seed_census;  // pair-dims the seed scored (profiling)
    DevBuf row_dims, union_out;  // B_union census of the last streaming search (profiling)
    bool union_valid = false;
    double last_union_bytes = 0, last_union_rows = 0;
    int n_filter_passes = 0;
    // DADE_GPU_TIMELINE=1: labelled events on both streams, printed per search (diagnostic)
    std::vector<std::pair<const char*, cudaEvent_t>> tl;
    size_t tl_used = 0;
    bool tl_on = false;
    double last_scan_ms = 0, last_bytes = 0, last_total_ms = 0, last_filter_ms = 0;

    // CUDA graphs of the search body (search_graphed): key = everything its
    // launches bake in (pointers, shapes, host-side decisions, allocation and
    // configuration epochs); the host state the body leaves is replayed too
    struct GraphEntry {
        std::array<uint64_t, 14> key{};
        cudaGraphExec_t exec = nullptr;
        uint64_t launches = 0, lru = 0;
        uint32_t surv_cap_used = 0;
        int n_filter_passes = 0;
        bool coarse_tc_used = false, fo_done = false;
    };
    std::vector<GraphEntry> graphs;
    std::array<uint64_t, 14> graph_seen{};  // key of the last body run eagerly (captured on a repeat)
    uint64_t cfg_epoch = 0, graph_tick = 0;
    bool graphs_on = true;
    void config_changed() { ++cfg_epoch; }

    void use_device() const { cuda_check(cudaSetDevice(device), "cudaSetDevice"); }
};

namespace {

// The result pointers the last slot merge of the search in flight writes
// (ctx.fo), cleared however the search exits, so a later keys-only search
// never writes through a stale pointer.
struct FusedOutputs {
    dade_gpu_ctx* c;
    FusedOutputs(dade_gpu_ctx* cc, uint32_t* ids, float* dists, uint32_t* counts) : c(cc) {
        c->fo = {ids, dists, counts, false};
    }
    ~FusedOutputs() { c->fo = {}; }
    FusedOutputs(const FusedOutputs&) = delete;
    FusedOutputs& operator=(const FusedOutputs&) = delete;
};

void upload(DevBuf& b, const void* src, size_t bytes, cudaStream_t s) {
    b.ensure(bytes);
    if (bytes) cuda_check(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, s), "H2D copy");
}

void require_strategy(const dade_gpu_ctx* c, uint32_t dim, const char* who) {
    if (!c->has_strategy) fail(DADE_GPU_CONFIG_ERROR, std::string(who) + ": no strategy set");
    if (c->s_dim != dim) fail(DADE_GPU_INVALID_INPUT, std::string(who) + ": strategy dim mismatch");
}

void set_tables(dade_gpu_ctx* c, uint32_t kind, uint32_t dim, std::vector<uint32_t> cps,
                std::vector<double> coeff, std::vector<double> scale) {
    if (dim == 0) fail(DADE_GPU_INVALID_INPUT, "strategy: dim must be positive");
    for (size_t i = 0; i < cps.size(); ++i) {
        if (cps[i] == 0 || cps[i] >= dim || (i && cps[i] <= cps[i - 1]))
            fail(DADE_GPU_INVALID_INPUT, "strategy: checkpoints must ascend within [1, dim)");
    }
    c->s_kind = kind;
    c->s_dim = dim;
    c->cps = std::move(cps);
    c->coeff = std::move(coeff);
    c->scale = std::move(scale);
    c->use_device();
    upload(c->d_cps, c->cps.data(), c->cps.size() * 4, c->stream);
    upload(c->d_coeff, c->coeff.data(), c->coeff.size() * 8, c->stream);
    upload(c->d_scale, c->scale.data(), c->scale.size() * 8, c->stream);
    cuda_check(cudaStreamSynchronize(c->stream), "strategy upload");
    c->has_strategy = true;
    c->config_changed();
}

bool coarse_tc_ok(dade_gpu_ctx* c, uint32_t n_probe) {
    // (the data-ordered flat scan probes every cell in any order: no selection cap)
    return (n_probe <= 256 || (c->coarse_all && n_probe == c->n_clusters && c->n_clusters <= 1024)) &&
           !c->coarse_force_exact && c->dim <= kCoarseTcMaxDim;  // (the bound's error budget, common.cuh)
}
// Above 1024 centroids the selection is fused with the GEMM (two tcgen05 passes:
// group minima, then the candidates lo <= T0; p~ never reaches memory).
constexpr uint32_t kCoarseFusedMin = 1024;
constexpr uint32_t kCoarseCandCap = 512;  // candidates per query of the fused selection
bool coarse_fused(const dade_gpu_ctx* c) { return c->n_clusters > kCoarseFusedMin && c->n_clusters <= 32768; }
// queries per coarse chunk: the p~ buffer holds chunk x n_clusters fp32 (<= 1 GB);
// the fused path's candidate lists chunk x 512 x 8 B.
uint32_t coarse_tc_chunk(dade_gpu_ctx* c, uint32_t nq) {
    const uint64_t per_q = coarse_fused(c) ? 8ull * kCoarseCandCap : 4ull * c->n_clusters;
    return (uint32_t)std::max<uint64_t>(64, std::min<uint64_t>(std::max<uint32_t>(nq, 1), (1ull << 30) / per_q));
}
// buffers for queries [0, nq) in chunks of coarse_tc_chunk(); overflow flag reset
void coarse_tc_begin(dade_gpu_ctx* c, uint32_t nq, uint32_t n_probe) {
    const uint32_t chunk = coarse_tc_chunk(c, nq);
    c->probes.ensure((size_t)std::max<uint32_t>(nq, 1) * n_probe * 8);
    c->probe_count.ensure((size_t)std::max<uint32_t>(nq, 1) * 4);
    c->cnorm.ensure((size_t)c->n_clusters * 4);
    c->qnorm.ensure((size_t)chunk * 4);
    if (coarse_fused(c)) {
        c->coarse_cand.ensure((size_t)chunk * kCoarseCandCap * 8);
        c->coarse_cnt.ensure((size_t)chunk * 4 * kCoarseSelParts);
        c->coarse_t0.ensure((size_t)chunk * 4);
    } else {
        c->coarse_lo.ensure((size_t)chunk * c->n_clusters * 4);
    }
    c->coarse_overflow.ensure(8);  // [0] overflow flag, [1] candidate census (DADE_GPU_COARSE_CENSUS)
    cuda_check(cudaMemsetAsync(c->coarse_overflow.p, 0, 8, c->stream), "memset");
    c->coarse_tc_used = true;
}
// queries [q0, q0 + m) (m <= coarse_tc_chunk) -> probes rows [q0, q0 + m)
void coarse_tc_range(dade_gpu_ctx* c, const float* d_q, uint32_t q0, uint32_t m, uint32_t n_probe) {
    cudaStream_t s = c->stream;
    // tcgen05 GEMM for p~ when both operands can be TMA-tiled; mma.sync otherwise
    bool tma_c = false, tma_q = false;
    const CUtensorMap* tmc = nullptr;
    const CUtensorMap* tmq = nullptr;
    if (!env_flag("DADE_GPU_NO_UMMA") && c->dim % 4 == 0 && c->dim >= (uint32_t)kBox) {
        tmc = &c->tm_centroids.get(c->centroids.as<float>(), c->n_clusters, c->dim, tma_c);
        tmq = &c->tm_queries.get(d_q, q0 + m, c->dim, tma_q);
    }
    if (tma_c && tma_q) {
        const float* qc = d_q + (size_t)q0 * c->dim;
        cuda_check(launch_coarse_norms(c->centroids.as<float>(), c->n_clusters, qc, m, c->dim, c->cnorm.as<float>(),
                                       c->qnorm.as<float>(), s),
                   "coarse norms");
        bool tq128 = false, tc256 = false;
        const CUtensorMap* mq = coarse_fused(c) && coarse_sel_umma_ok(c->dim)
                                    ? &c->tm_q128.get(d_q, q0 + m, c->dim, tq128) : nullptr;
        const CUtensorMap* mc = mq ? &c->tm_c256.get(c->centroids.as<float>(), c->n_clusters, c->dim, tc256) : nullptr;
        if (mq && tq128 && tc256) {
            // query-major fused selection (umma.cu coarse_sel_umma_kernel): pass A, group minima of
            // the upper bounds -> T0 per query; pass B, the same GEMM, candidates lo <= T0 listed per
            // query; then B, exact l2_sq, (d^2, id) sort. p~ never reaches memory.
            c->coarse_gmin.ensure((size_t)m * ((c->n_clusters + 31) / 32) * 4);
            uint32_t* gmin = c->coarse_gmin.as<uint32_t>();
            CoarseFilter none;
            cuda_check(launch_coarse_sel_umma(*mq, *mc, q0, c->n_clusters, m, c->dim, c->cnorm.as<float>(),
                                              c->qnorm.as<float>(), gmin, none, s),
                       "coarse selection pass A (tcgen05)");
            cuda_check(launch_coarse_t0(gmin, c->n_clusters, m, n_probe, c->coarse_t0.as<uint32_t>(), s, true),
                       "coarse t0");
            CoarseFilter cf;  // (every thread writes its slice count: no memset)
            cf.t0 = c->coarse_t0.as<uint32_t>();
            cf.cand = c->coarse_cand.as<uint64_t>();
            cf.cnt = c->coarse_cnt.as<uint32_t>();
            cf.cap = kCoarseCandCap;
            cuda_check(launch_coarse_sel_umma(*mq, *mc, q0, c->n_clusters, m, c->dim, c->cnorm.as<float>(),
                                              c->qnorm.as<float>(), nullptr, cf, s),
                       "coarse selection pass B (tcgen05)");
            cuda_check(launch_coarse_finish(cf.cand, cf.cnt, cf.cap, c->cnorm.as<float>(), c->qnorm.as<float>(),
                                            c->centroids.as<float>(), qc, m, c->dim, n_probe,
                                            c->probes.as<uint64_t>() + (size_t)q0 * n_probe,
                                            c->coarse_overflow.as<uint32_t>(), s, kCoarseSelParts),
                       "coarse finish");
            c->launches += 5;
            return;
        }
        if (coarse_fused(c)) {
            // centroid-major passes of coarse_umma_kernel (dims it cannot stage)
            c->coarse_gmin.ensure((size_t)m * ((c->n_clusters + 31) / 32) * 4);
            uint32_t* gmin = c->coarse_gmin.as<uint32_t>();
            cuda_check(launch_coarse_umma(*tmc, *tmq, q0, c->n_clusters, m, c->dim, c->cnorm.as<float>(),
                                          c->qnorm.as<float>(), nullptr, s, gmin),
                       "coarse gemm pass A (tcgen05)");
            cuda_check(launch_coarse_t0(gmin, c->n_clusters, m, n_probe, c->coarse_t0.as<uint32_t>(), s), "coarse t0");
            cuda_check(cudaMemsetAsync(c->coarse_cnt.p, 0, (size_t)m * 4, s), "memset");
            CoarseFilter cf;
            cf.t0 = c->coarse_t0.as<uint32_t>();
            cf.cand = c->coarse_cand.as<uint64_t>();
            cf.cnt = c->coarse_cnt.as<uint32_t>();
            cf.cap = kCoarseCandCap;
            cuda_check(launch_coarse_umma(*tmc, *tmq, q0, c->n_clusters, m, c->dim, c->cnorm.as<float>(),
                                          c->qnorm.as<float>(), nullptr, s, nullptr, cf),
                       "coarse gemm pass B (tcgen05)");
            cuda_check(launch_coarse_finish(cf.cand, cf.cnt, cf.cap, c->cnorm.as<float>(), c->qnorm.as<float>(),
                                            c->centroids.as<float>(), qc, m, c->dim, n_probe,
                                            c->probes.as<uint64_t>() + (size_t)q0 * n_probe,
                                            c->coarse_overflow.as<uint32_t>(), s),
                       "coarse finish");
            c->launches += 5;
            return;
        }
        uint32_t* gmin = nullptr;
        cuda_check(launch_coarse_umma(*tmc, *tmq, q0, c->n_clusters, m, c->dim, c->cnorm.as<float>(),
                                      c->qnorm.as<float>(), c->coarse_lo.as<float>(), s, gmin),
                   "coarse gemm (tcgen05)");
        if (c->coarse_all && n_probe == c->n_clusters) {  // data-ordered flat scan: order only
            cuda_check(launch_coarse_all(c->coarse_lo.as<float>(), c->n_clusters, m,
                                         c->probes.as<uint64_t>() + (size_t)q0 * n_probe, s),
                       "coarse order");
            c->launches += 3;
            return;
        }
        cuda_check(launch_coarse_select(c->centroids.as<float>(), c->n_clusters, qc, m, c->dim, n_probe,
                                        c->cnorm.as<float>(), c->qnorm.as<float>(), c->coarse_lo.as<float>(),
                                        c->probes.as<uint64_t>() + (size_t)q0 * n_probe,
                                        c->coarse_overflow.as<uint32_t>(), s, gmin, c->coarse_exact_keys),
                   "coarse select");
        c->launches += 3;
        return;
    }
    cuda_check(launch_coarse_tc(c->centroids.as<float>(), c->n_clusters, d_q + (size_t)q0 * c->dim, m, c->dim, n_probe,
                                c->cnorm.as<float>(), c->qnorm.as<float>(), c->coarse_lo.as<float>(),
                                c->probes.as<uint64_t>() + (size_t)q0 * n_probe,
                                c->coarse_overflow.as<uint32_t>(), s),
               "coarse tc");
    c->launches += 4;
}

// Coarse ranking (K2): exact l2_sq to every centroid, K = n_probe smallest by
// (dist^2, cluster id) (proj/src/ivf.cpp:215-219), as a flat FD scan in
// squared-distance key space.
void coarse_rank(dade_gpu_ctx* c, const float* d_q, uint32_t nq, uint32_t n_probe) {
    cudaStream_t s = c->stream;
    c->probes.ensure((size_t)nq * n_probe * 8);
    c->probe_count.ensure((size_t)nq * 4);
    if (coarse_tc_ok(c, n_probe)) {
        // tensor-core p~ for all (query, centroid) pairs + exact l2_sq on the
        // boundary candidates (coarse.cu); query chunks bound the p~ buffers
        coarse_tc_begin(c, nq, n_probe);
        const uint32_t chunk = coarse_tc_chunk(c, nq);
        for (uint32_t q0 = 0; q0 < nq; q0 += chunk)
            coarse_tc_range(c, d_q, q0, std::min(chunk, nq - q0), n_probe);
        return;
    }
    c->coarse_tc_used = false;
    const uint32_t qchunks = (nq + kQC - 1) / kQC;
    const uint32_t max_blocks = (c->n_clusters + kRT - 1) / kRT;
    uint32_t nb = std::max<uint32_t>(1, std::min<uint32_t>(max_blocks, (1184 + qchunks - 1) / qchunks));
    uint32_t block = (c->n_clusters + nb - 1) / nb;
    block = (block + kRT - 1) / kRT * kRT;
    nb = (c->n_clusters + block - 1) / block;
    const size_t nseg = (size_t)nq * nb;
    c->c_seg_keys.ensure(nseg * n_probe * 8);
    c->c_seg_count.ensure(nseg * 4);
    c->c_r.ensure((size_t)nq * 4);
    c->probes.ensure((size_t)nq * n_probe * 8);
    c->probe_count.ensure((size_t)nq * 4);
    cuda_check(cudaMemsetAsync(c->c_seg_count.p, 0, nseg * 4, s), "memset");
    cuda_check(launch_fill_u32(c->c_r.as<uint32_t>(), 0x7f800000u, nq, s), "fill");
    ScanArgs a{};
    a.storage = c->centroids.as<float>();
    a.row_ids = nullptr;
    a.id_base = 0;
    a.dim = c->dim;
    a.queries = d_q;
    a.items = nullptr;
    a.flat_rows = c->n_clusters;
    a.flat_block = block;
    a.flat_nq = nq;
    a.flat_qchunks = qchunks;
    a.r_global = c->c_r.as<uint32_t>();
    a.seg_keys = c->c_seg_keys.as<uint64_t>();
    a.seg_count = c->c_seg_count.as<uint32_t>();
    a.n_slots = nb;
    a.K = n_probe;
    a.coeff = nullptr;
    a.neg_zero2 = 0x8000000080000000ull;
    a.counters = nullptr;
    ChunkTable ct = make_chunks(c->dim, {});
    bool tma = false;
    const CUtensorMap& tm = c->tm_centroids.get(a.storage, c->n_clusters, c->dim, tma);
    ct.use_tma = (tma && ct.vec_ok) ? 1 : 0;
    cuda_check(launch_scan(a, ct, tm, c->tm_none, nb * qchunks, /*sqrt_key=*/false, s), "coarse scan");
    cuda_check(launch_merge_segments(a.seg_keys, a.seg_count, nq, nb, n_probe, c->probes.as<uint64_t>(),
                                     c->probe_count.as<uint32_t>(), s),
               "coarse merge");
    c->launches += 3;
}

constexpr uint32_t kFilterItemRows = 1024;  // row piece of a streaming work item
constexpr uint32_t kFilterQ = 32;           // queries per streaming work item (one warp's MMA N)
// Nearest-list items use shorter pieces: those rows keep most pairs (they hold
// the query's neighbours), and short items spread that work over every SM.
// Pass 0 takes the pieces covering the first kFilterItemRows rows.
constexpr uint32_t kUmmaQ = 256;            // queries per tcgen05 work item (MMA N)
constexpr uint32_t kQSlots = 256;           // per-query candidate slots of a streaming pass
uint32_t rank0_item_rows(bool umma, bool dense_groups) {
    // one tile: a nearest list's heavy rows spread over every SM / warp -- when the list has several queries.
    // With about one query per nearest list (config 2: 1000 queries on 1024 lists) short pieces only multiply
    // the items (six 128-row items of ONE query per list, each paying its staging and pipeline fill).
    if (umma && !dense_groups) return kFilterItemRows;
    return umma ? 128 : 32;
}
constexpr uint32_t kSeedRowsDefault = 1024;  // rows of the nearest list used by the radius seed

// rows of each nearest list the radius seed scores exactly (and the scan then
// skips): the list-major kernel (K <= 128) takes up to 1024, the per-query one 512
// Rows of each nearest list the seed scores exactly: 1024 up to dim 256, then
// ~1 MB of rows (256 at dim 960: an IVF group there holds ~1 query, so long rows
// cost bytes per query -- config 2 1.47 -> 1.21 ms per batch at recall 0.982 vs
// 0.987). The flat scan's groups are full (every query probes the base): 1024;
// so are an IVF search's when its batch holds several queries per list (the
// partitioned flat scan, 4096 queries on 512 cells: 6.12 -> 5.63 ms per batch).
uint32_t seed_rows(const dade_gpu_ctx* c, uint32_t k, uint32_t dim, bool flat = false) {
    const bool list_kernel = k <= 128;
    uint32_t s = kSeedRowsDefault;
    if (c->seed_rows_set) return std::min<uint32_t>(list_kernel ? 1024 : 512, std::max<uint32_t>(c->seed_rows_set, k));
    if (dim > 256 && !flat && !c->dense_groups) s = std::min<uint32_t>(s, std::max<uint32_t>(128, (262144u / dim) & ~127u));
    return std::min<uint32_t>(list_kernel ? 1024 : 512, std::max<uint32_t>(s, k));
}

void tl_mark(dade_gpu_ctx* c, const char* name, cudaStream_t s) {
    if (!c->tl_on) return;
    if (c->tl_used == c->tl.size()) {
        cudaEvent_t e;
        cuda_check(cudaEventCreate(&e), "event");
        c->tl.push_back({name, e});
    }
    c->tl[c->tl_used].first = name;
    cuda_check(cudaEventRecord(c->tl[c->tl_used++].second, s), "event");
}

void tl_print(dade_gpu_ctx* c) {
    if (!c->tl_on || !c->tl_used) return;
    cuda_check(cudaEventSynchronize(c->tl[c->tl_used - 1].second), "event sync");
    std::string line = "[dade_gpu] timeline (ms):";
    for (size_t i = 1; i < c->tl_used; ++i) {
        float ms = 0;
        cuda_check(cudaEventElapsedTime(&ms, c->tl[0].second, c->tl[i].second), "elapsed");
        char buf[96];
        std::snprintf(buf, sizeof buf, " %s %.3f", c->tl[i].first, ms);
        line += buf;
    }
    std::fprintf(stderr, "%s\n", line.c_str());
}

void record(dade_gpu_ctx* c, cudaEvent_t e) {
    if (c->profiling) cuda_check(cudaEventRecord(e, c->stream), "event");
}

void finish_profile(dade_gpu_ctx* c) {
    if (!c->profiling) return;
    c->last_union_bytes = c->last_union_rows = 0;
    if (c->union_valid) {
        unsigned long long u[2] = {0, 0};
        cuda_check(cudaMemcpy(u, c->union_out.p, 16, cudaMemcpyDeviceToHost), "D2H union");
        c->last_union_bytes = (double)u[0];
        c->last_union_rows = (double)u[1];
        c->union_valid = false;
    }
    cuda_check(cudaEventSynchronize(c->e3), "event sync");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, c->e1, c->e2), "elapsed");
    c->last_scan_ms = ms;
    cuda_check(cudaEventElapsedTime(&ms, c->e0, c->e3), "elapsed");
    c->last_total_ms = ms;
    unsigned long long h[3] = {0, 0, 0};
    cuda_check(cudaMemcpy(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost), "D2H counters");
    c->last_bytes = (double)h[2];
    c->last_filter_ms = 0;
    for (int p = 0; p < c->n_filter_passes; ++p) {
        cuda_check(cudaEventElapsedTime(&ms, c->ef[2 * p], c->ef[2 * p + 1]), "elapsed");
        c->last_filter_ms += ms;
    }
    c->last_seed_ms = c->last_seed_pair_dims = 0;
    if (c->seed_profiled) {
        cuda_check(cudaEventElapsedTime(&ms, c->es[0], c->es[1]), "elapsed");
        c->last_seed_ms = ms;
        unsigned long long pd = 0;
        cuda_check(cudaMemcpy(&pd, c->seed_census.p, 8, cudaMemcpyDeviceToHost), "D2H census");
        c->last_seed_pair_dims = (double)pd;
    }
}

// DcoStats of the rows the radius seed scored exactly (the streaming passes skip
// them, GroupArgs::seed_skip): each is a full-dim DCO that is never pruned. For
// failure accounting the seed's decision is "among the query's K best of these
// rows", i.e. a test against the radius it produces, which its K kept rows
// (seed_min = K) pass: those are the eligible ones.
// With group_bytes (the seed kernels other than the TMA one), B_read gets each
// group's (kSeedGroup queries of one list) rows once.
__global__ void seed_stats_kernel(const uint32_t* counts, const uint32_t* list_offsets, uint32_t n_lists,
                                  uint32_t seed_skip, uint32_t seed_min, uint32_t dim, bool measure,
                                  bool group_bytes, unsigned long long* counters) {
    unsigned long long pairs = 0, kept = 0, bytes = 0;
    for (uint32_t l = blockIdx.x * blockDim.x + threadIdx.x; l < n_lists; l += gridDim.x * blockDim.x) {
        const uint32_t len = list_offsets[l + 1] - list_offsets[l];
        if (len >= seed_min) {
            pairs += (unsigned long long)counts[l] * min(len, seed_skip);
            kept += (unsigned long long)counts[l] * seed_min;
            bytes += 4ull * dim * min(len, seed_skip) * ((counts[l] + kSeedGroup - 1) / kSeedGroup);
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        pairs += __shfl_xor_sync(0xffffffffu, pairs, off);
        kept += __shfl_xor_sync(0xffffffffu, kept, off);
        bytes += __shfl_xor_sync(0xffffffffu, bytes, off);
    }
    if ((threadIdx.x & 31) == 0 && pairs) {
        atomicAdd(counters + 0, pairs);
        atomicAdd(counters + 1, pairs * dim);
        if (group_bytes) atomicAdd(counters + 2, bytes);
        if (measure) atomicAdd(counters + 8, kept);
    }
}

// B_union ("oracle lower bound"): the bytes any scan making this
// search's decisions must read at least -- per row, the most dims any of its
// pairs reached: d0 (the first slice) for every row of a probed list, dim for
// the rows the seed scored exactly, and the survivors' prune / full dims
// (row_dims). One CTA per list; out[0] += bytes, out[1] += rows touched.
__global__ void union_census_kernel(const uint32_t* counts, uint32_t n_rb, uint32_t n_lists,
                                    const uint32_t* list_offsets, uint32_t seed_skip, uint32_t seed_min, uint32_t d0,
                                    uint32_t dim, const uint32_t* row_dims, unsigned long long* out) {
    const uint32_t l = blockIdx.x;
    bool probed = false;
    for (uint32_t rb = 0; rb < n_rb; ++rb) probed = probed || counts[rb * n_lists + l] > 0;
    const uint32_t b = list_offsets[l], len = list_offsets[l + 1] - b;
    const uint32_t seeded = (seed_skip && counts[l] > 0 && len >= seed_min) ? min(len, seed_skip) : 0u;
    unsigned long long bytes = 0, rows = 0;
    for (uint32_t r = threadIdx.x; r < len; r += blockDim.x) {
        uint32_t v = probed ? d0 : 0u;
        if (r < seeded) v = dim;
        v = max(v, row_dims[b + r]);
        bytes += 4ull * v;
        rows += v ? 1 : 0;
    }
    for (int off = 16; off > 0; off >>= 1) {
        bytes += __shfl_xor_sync(0xffffffffu, bytes, off);
        rows += __shfl_xor_sync(0xffffffffu, rows, off);
    }
    if ((threadIdx.x & 31) == 0 && bytes) {
        atomicAdd(out, bytes);
        atomicAdd(out + 1, rows);
    }
}

__global__ void min_u32_kernel(uint32_t* r, const uint32_t* other, uint32_t n) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) r[i] = min(r[i], other[i]);
}

// The streaming tensor-core path applies when the first checkpoint is a
// multiple of 8 dims (MMA k) within two 32-dim TMA boxes.
constexpr uint32_t kRotFixCap = 1u << 20;  // undecided rotation outputs per launch handled by rotate_fix_kernel
cudaError_t rotate_on(dade_gpu_ctx* c, uint32_t dim, const float* in, uint32_t n, float* out) {
    // Long vectors only: the undecided share grows with dim (1e-4 at dim 256, ~1% at dim 960, where the
    // in-CTA recompute was a third of the kernel: config 2 170.6 -> 129.5 + 13 us); at dim 256 the few
    // in-CTA recomputes cost less than a second launch (config 1 77.7 vs 77.2 + 7.2 us).
    if (dim < 512) return launch_rotate(c->W.as<double>(), dim, in, n, out, c->stream);
    c->rot_fix.ensure((size_t)kRotFixCap * 8 + 16);
    uint2* fix = c->rot_fix.as<uint2>();
    return launch_rotate(c->W.as<double>(), dim, in, n, out, c->stream, fix,
                         reinterpret_cast<uint32_t*>(fix + kRotFixCap), kRotFixCap);
}

bool filter_ok(dade_gpu_ctx* c, const ChunkTable& ct, uint32_t dim) {
    if (!ct.use_tc || !ct.use_tma || ct.n_ckpt > 63) return false;
    const uint32_t d0 = ct.end[ct.n_dense - 1];
    return d0 % 8 == 0 && d0 <= 2 * kBox && dim % 4 == 0 && dim >= (uint32_t)kBox;
}

// tcgen05 filter (umma.cu): 128-row TMA tiles (tm_storage), d0 a multiple of 8 up to 64
bool umma_ok(dade_gpu_ctx* c, const ChunkTable& ct, bool tma128) {
    (void)c;
    if (!tma128 || env_flag("DADE_GPU_NO_UMMA")) return false;
    const uint32_t d0 = ct.end[ct.n_dense - 1];
    return d0 % 8 == 0 && d0 <= 2 * kBox;
}

// Streaming passes after the radius seed (their number and row ranges are chosen
// below). Each pass = tensor-core filter -> survivor kernel -> candidate buckets ->
// merge into the running top-K; between passes every query's radius is tightened from it.
struct SeedArgs {
    bool on;
    const uint64_t* probes;
    uint32_t n_probe;
    const uint32_t* offsets;
};

void stream_passes(dade_gpu_ctx* c, const ScanArgs& a, const ChunkTable& ct, const float* d_q, uint32_t nq,
                   uint32_t k, bool two_pass, uint32_t max_items, const GroupArgs* g, const float* rows,
                   uint32_t n_rows, TmapCache& tm_tile, bool umma, uint64_t* out_keys, uint32_t* out_count,
                   const SeedArgs& seed, RowNorms* norms, bool flat = false) {
    cudaStream_t s = c->stream;
    bool tma = false;
    const CUtensorMap& tm = tm_tile.get(rows, std::max<uint32_t>(n_rows, 1), a.dim, tma);
    if (!tma) fail(DADE_GPU_CUDA_ERROR, "tensor map for the streaming filter failed");
    const uint32_t d0 = ct.end[ct.n_dense - 1];
    const bool resume = c->split == 2, stop = c->split == 1;
    if (umma && !resume) {  // first-slice query norms for the tcgen05 filter's -c terms
        c->q_norms.ensure((size_t)std::max<uint32_t>(nq, 1) * 4);
        cuda_check(launch_row_norms(d_q, nq, a.dim, d0, c->q_norms.as<float>(), s), "query norms");
        ++c->launches;
    }
    // Worklist capacity: a hint learnt from earlier searches; overflow is detected
    // after the search (search_overflowed) and the search is redone larger, so
    // no host sync sits in the middle of the pipeline.
    uint32_t base_cap = (uint32_t)std::min<uint64_t>(64ull << 20, std::max<uint64_t>(1u << 20, (uint64_t)nq * 1024));
    if (const char* e = std::getenv("DADE_GPU_SURV_CAP")) base_cap = (uint32_t)std::max(64, std::atoi(e));  // test hook
    const uint32_t cap = std::max<uint32_t>(c->surv_cap_hint, base_cap);
    c->surv_cap_used = cap;
    {
        c->surv.ensure((size_t)cap * sizeof(Survivor));
        c->surv_count.ensure(8);
        c->cand_q.ensure((size_t)cap * 4);
        c->cand_key.ensure((size_t)cap * 8);
        c->cand_count.ensure(4);
        c->q_count.ensure((size_t)nq * 4);
        c->surv_max.ensure(4);
        if (!resume) {
            cuda_check(cudaMemsetAsync(c->surv_max.p, 0, 4, s), "memset");
            cuda_check(cudaMemsetAsync(out_count, 0, (size_t)nq * 4, s), "memset");
        }
        const bool census = c->profiling && g;  // B_union census (profiled searches only)
        bool seed_tma_ran = false;
        if (census && !resume) {
            c->row_dims.ensure((size_t)std::max<uint32_t>(n_rows, 1) * 4);
            cuda_check(cudaMemsetAsync(c->row_dims.p, 0, (size_t)std::max<uint32_t>(n_rows, 1) * 4, s), "memset");
        }
        if (seed.on && !resume) {
            const CUtensorMap* stm =
                (g && k <= 128 && seed_tma_ok(a.dim, k)) ? c->seed_tm.get(rows, n_rows, a.dim) : nullptr;
            seed_tma_ran = stm != nullptr;
            if (stm) {
                SeedListArgs sa{};
                sa.counts = g->counts;
                sa.bucket_off = g->bucket_off;
                sa.bucket_q = g->bucket_q;
                sa.seed_goff = g->seed_goff;
                sa.seed_glist = g->seed_glist;
                sa.n_lists = g->n_lists;
                sa.list_offsets = seed.offsets;
                sa.row_ids = a.row_ids;
                sa.id_base = a.id_base;
                sa.dim = a.dim;
                sa.K = k;
                sa.S = std::min<uint32_t>(seed_rows(c, k, a.dim, flat), 1024);
                sa.queries = d_q;
                sa.r_global = a.r_global;
                sa.out_keys = out_keys;
                sa.out_count = out_count;
                sa.nz2 = 0x8000000080000000ull;
                sa.counters = a.counters;
                c->seed_work.ensure(4);
                c->seed_order.ensure(((size_t)nq / kSeedGroup + g->n_lists + 1) * 4);
                sa.order = c->seed_order.as<uint32_t>();
                c->seed_profiled = c->profiling;
                if (c->profiling) {  // device time and pair-dims of the seed (dade_gpu_last_seed_profile)
                    c->seed_census.ensure(8);
                    cuda_check(cudaMemsetAsync(c->seed_census.p, 0, 8, s), "memset");
                    sa.census = c->seed_census.as<unsigned long long>();
                    cuda_check(cudaEventRecord(c->es[0], s), "event");
                }
                cuda_check(launch_seed_tma(sa, *stm, nq / kSeedGroup + g->n_lists + 1, s, c->seed_work.as<uint32_t>()),
                           "seed radius (tma)");
                if (c->profiling) cuda_check(cudaEventRecord(c->es[1], s), "event");
            } else if (g && g->n_rb >= 1 && k <= 128)
                cuda_check(launch_seed_radius_lists(g->counts, g->bucket_off, g->bucket_q, g->seed_goff, g->seed_glist,
                                                    g->n_lists,
                                                    nq / kSeedGroup + g->n_lists + 1, seed.offsets, rows, a.row_ids,
                                                    a.id_base, a.dim, d_q, k, seed_rows(c, k, a.dim, flat), a.r_global, out_keys,
                                                    out_count, s),
                           "seed radius (lists)");
            else
                cuda_check(launch_seed_radius(seed.probes, seed.n_probe, seed.offsets, rows, a.row_ids, a.dim, d_q, nq,
                                              k, seed_rows(c, k, a.dim, flat), a.r_global, out_keys, out_count, s),
                           "seed radius");
            ++c->launches;
            if (a.counters && g) {
                seed_stats_kernel<<<1, 256, 0, s>>>(g->counts, seed.offsets, g->n_lists, g->seed_skip, g->seed_min,
                                                    a.dim, c->measure, !seed_tma_ran, a.counters);
                cuda_check(cudaGetLastError(), "seed stats");
                ++c->launches;
            }
        }
        if (!resume && c->dump_cap)
            cuda_check(cudaMemsetAsync(c->dump_count.p, 0, 4, s), "memset");
        tl_mark(c, "seeded", s);
        // Each pass = filter -> survivors -> merge; the radius is tightened after each.
        // IVF (mma.sync / SIMT filters): nearest lists' first pieces, their other pieces, the
        // other lists. Flat (one list holding the whole base, every query on it): row ranges
        // of 1024-row pieces growing 4x per pass.
        static const uint32_t flat_lo[6] = {0, 2, 8, 32, 128, 512};
        static const uint32_t flat_hi[6] = {2, 8, 32, 128, 512, 0xffffffffu};
        // IVF: pass 0 = the nearest lists' next rows, then (tcgen05 filter) one pass over
        // everything else incl. the nearest lists' tails -- a separate middle pass for
        // those tails costs its own filter/survivor/merge launches
        const bool fold = umma && two_pass && !flat;
        // ... and (tcgen05 filter) NO separate pass 0 unless it pays: the pass tightens the radius
        // for everything after it at the price of its own filter / survivor / merge launches
        // (~60 us of mostly idle GPU). It pays when the nearest lists reach well past the seed AND
        // much work follows (the partitioned flat scan: 3906-row cells, 8e9 pairs: 6.1 vs 7.9 ms).
        // Otherwise one pass over everything the seed left, with the seed's radius: config 1
        // 0.931 -> 0.874 ms, config 2 0.875 -> 0.791 ms, config 0 0.386 -> 0.337 ms, config 3
        // 9.46 -> 9.33 ms per batch; recall 0.985 -> 0.986 / 0.983 -> 0.994 / 1.000 / 0.803 ->
        // 0.804 (a looser radius prunes fewer true neighbours).
        bool single = false;
        if (fold && g && g->n_lists) {
            const double mean_len = (double)n_rows / g->n_lists;
            const double pairs = (double)nq * seed.n_probe * mean_len;
            single = !(mean_len > 2.0 * seed_rows(c, k, a.dim, flat) && pairs >= 1e9);
            if (env_flag("DADE_GPU_TWO_PASS")) single = false;  // test hook: the two-pass structure at test sizes
        }
        const int n_pass = flat ? 6 : single ? 1 : two_pass ? (fold ? 2 : 3) : 1;
        // The next staging's H2D (pipelined batches) starts with the last pass, not
        // after this search's rotation: under the seed and the early passes the
        // copy slowed the search by ~60 us, under the last pass's tcgen05 filter
        // by nothing measurable
        // two-phase split: IVF before its last pass (nearest lists done), flat right after the seed
        const int split_pass = flat ? 0 : n_pass - 1;
        for (int pass = 0; pass < n_pass; ++pass) {
            if (resume && pass < split_pass) continue;  // phase 2: from the split pass on
            if (stop && pass == split_pass) break;      // phase 1: everything before it
            if (pass == n_pass - 1 && c->qin_free_recorded) {
                // (inside a graph capture: an event-record node the next staging's copy stream waits on)
                cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
                cuda_check(cudaStreamIsCapturing(s, &cs), "capture status");
                cuda_check(cs == cudaStreamCaptureStatusActive
                               ? cudaEventRecordWithFlags(c->copy_ev[8], s, cudaEventRecordExternal)
                               : cudaEventRecord(c->copy_ev[8], s),
                           "event");
            }
            cuda_check(cudaMemsetAsync(c->surv_count.p, 0, 4, s), "memset");
            FilterArgs f{};
            f.queries = d_q;
            f.dim = a.dim;
            f.d0 = d0;
            f.c_dense = (int)((d0 + kBox - 1) / kBox);
            f.coeff0 = c->coeff[0];
            f.r_global = a.r_global;
            f.items = a.items;
            f.n_items = a.n_items;
            f.bucket_q = a.bucket_q;
            f.bucket_slot = a.bucket_slot;
            f.flat_rows = a.flat_rows;
            f.flat_block = a.flat_block;
            f.flat_nq = a.flat_nq;
            f.flat_qchunks = a.flat_qchunks;
            f.row_norms = norms->get(rows, n_rows, a.dim, d0, s);
            f.surv = c->surv.as<Survivor>();
            f.surv_count = c->surv_count.as<uint32_t>();
            f.surv_cap = cap;
            f.counters = a.counters;
            uint32_t grid = a.items ? max_items : a.flat_qchunks * ((a.flat_rows + a.flat_block - 1) / a.flat_block);
            f.piece_lo = 0;
            f.piece_hi = 0xffffffffu;
            f.debug = c->measure ? 1 : ct.debug;  // failure accounting: every pair to the survivors
            if (flat) {
                f.n_items = g->n_items + 1;
                f.piece_lo = flat_lo[pass];
                f.piece_hi = flat_hi[pass];
                if (g->piece_major) {  // the pass's items are contiguous: no stager scans past the others
                    const uint32_t nqc = (nq + g->q_chunk - 1) / g->q_chunk;
                    const uint32_t skip = n_rows >= g->seed_min ? g->seed_skip : 0u;
                    const uint32_t np = (n_rows - skip + g->max_item_rows - 1) / g->max_item_rows;
                    f.range_lo = std::min(flat_lo[pass], np) * nqc;
                    f.range_hi = std::min(flat_hi[pass], np) * nqc;
                    if (f.range_hi == 0) f.range_lo = 0;  // (empty base: the counter path)
                }
            } else if (two_pass && !single) {
                // pass 0: kFilterItemRows rows of each nearest list past the seed
                const uint32_t p0 = std::max<uint32_t>(1, kFilterItemRows / rank0_item_rows(umma, c->dense_groups));
                if (pass == 0 || (pass == 1 && !fold)) {
                    f.n_items = g->n_items + 1;  // rank-bucket-0 items: every query's nearest list
                    f.piece_lo = pass == 0 ? 0u : p0;
                    f.piece_hi = pass == 0 ? p0 : 0xffffffffu;
                } else if (fold) {  // every item: bucket 0 from piece p0 on, the rest whole
                    f.b0_items = g->n_items + 1;
                    f.b0_piece_lo = p0;
                } else {
                    f.item_base = g->n_items + 1;  // the rest
                }
            }
            // persistent CTAs pull items from a counter: two per SM (one for tcgen05)
            c->item_counter.ensure(4);
            cuda_check(cudaMemsetAsync(c->item_counter.p, 0, 4, s), "memset");
            f.item_counter = c->item_counter.as<uint32_t>();
            f.q_norms = umma ? c->q_norms.as<float>() : nullptr;
            const CUtensorMap* taug = nullptr;
            if (umma) {
                taug = c->aug_storage.get(rows, n_rows, a.dim, d0, f.row_norms, s);
                if (!taug) fail(DADE_GPU_CUDA_ERROR, "tensor map for the tcgen05 filter's row operand failed");
            }
            grid = std::min<uint32_t>(grid, (uint32_t)c->n_sms * (umma ? 1 : 2));
            if (c->profiling) cuda_check(cudaEventRecord(c->ef[2 * pass], s), "event");
            if (umma) cuda_check(launch_filter_umma(f, tm, *taug, grid, s), "filter (tcgen05)");
            else cuda_check(launch_filter(f, tm, grid, s), "filter");
            if (c->profiling) cuda_check(cudaEventRecord(c->ef[2 * pass + 1], s), "event");
            c->n_filter_passes = n_pass;
            cuda_check(cudaMemsetAsync(c->cand_count.p, 0, 4, s), "memset");
            cuda_check(cudaMemsetAsync(c->q_count.p, 0, (size_t)nq * 4, s), "memset");
            SurvArgs sv{};
            sv.surv = f.surv;
            sv.surv_count = f.surv_count;
            sv.surv_cap = cap;
            sv.storage = rows;
            sv.row_ids = a.row_ids;
            sv.id_base = a.id_base;
            sv.dim = a.dim;
            sv.queries = d_q;
            sv.r_global = a.r_global;
            sv.coeff = a.coeff;
            sv.n_dense_dims = umma ? 0 : d0;  // tcgen05 filter: survivors restart from dim 0
            sv.n_ckpt = ct.n_ckpt;
            for (int i = 0; i < ct.n_ckpt; ++i) sv.cps[i] = (uint16_t)c->cps[i];
            sv.first_ckpt = umma ? 0 : 1;
            sv.vec4 = (a.dim % 4 == 0 && d0 % 4 == 0) ? 1u : 0u;
            for (int i = 0; i < ct.n_ckpt; ++i)
                if (c->cps[i] % 4 != 0) sv.vec4 = 0;
            sv.cand_q = c->cand_q.as<uint32_t>();
            sv.cand_key = c->cand_key.as<uint64_t>();
            sv.cand_count = c->cand_count.as<uint32_t>();
            sv.cand_cap = cap;
            sv.q_count = c->q_count.as<uint32_t>();
            c->qslots.ensure((size_t)nq * kQSlots * 8);
            sv.qslots = c->qslots.as<uint64_t>();
            sv.qslot_cap = kQSlots;
            if (a.counters && (pass < 2 || !ct.debug)) {
                c->cand_total.ensure(4);
                cuda_check(cudaMemsetAsync(c->cand_total.p, 0, 4, s), "memset");
                sv.cand_total = c->cand_total.as<uint32_t>();
            }
            sv.counters = a.counters;
            sv.surv_max = c->surv_max.as<uint32_t>();
            sv.measure = c->measure ? 1u : 0u;
            if (census) sv.row_dims = c->row_dims.as<uint32_t>();
            if (c->dump_cap) sv.dump = {c->dump_entries.as<uint4>(), c->dump_count.as<uint32_t>(), c->dump_cap};
            cuda_check(launch_advance_survivors(sv, cap, s), "advance survivors");
            // survivors / candidates of passes 0, 1 (low words of counters[4 + 2 pass ..]); of pass 2 in
            // counters[3] (low / high word) unless a debug mode owns that word
            if (a.counters && (pass < 2 || (pass == 2 && !ct.debug)))
                for (int w = 0; w < 2; ++w)
                    cuda_check(cudaMemcpyAsync(pass < 2 ? reinterpret_cast<uint32_t*>(a.counters + 4 + 2 * pass + w)
                                                        : reinterpret_cast<uint32_t*>(a.counters + 3) + w,
                                               w == 0 ? c->surv_count.p : sv.cand_total ? c->cand_total.p : c->cand_count.p, 4,
                                               cudaMemcpyDeviceToDevice, s),
                               "census");
            // the slot merge tightens each query's radius as it finishes it; the search's
            // last merge writes ids / dists / counts when the caller asked for them (fo)
            cuda_check(launch_merge_slots(sv.qslots, sv.qslot_cap, c->q_count.as<uint32_t>(),
                                          c->cand_q.as<uint32_t>(), c->cand_key.as<uint64_t>(),
                                          c->cand_count.as<uint32_t>(), cap, nq, k, out_keys, out_count, s,
                                          pass + 1 < n_pass ? a.r_global : nullptr,
                                          pass + 1 == n_pass && !stop ? c->fo.ids : nullptr, c->fo.dists,
                                          c->fo.counts),
                       "merge slots");
            if (pass + 1 == n_pass && !stop && c->fo.ids) c->fo.done = true;
            c->launches += 3;
            if (census && pass + 1 == n_pass && !stop) {
                c->union_out.ensure(16);
                cuda_check(cudaMemsetAsync(c->union_out.p, 0, 16, s), "memset");
                union_census_kernel<<<g->n_lists, 256, 0, s>>>(g->counts, g->n_rb, g->n_lists, seed.offsets,
                                                               g->seed_skip, g->seed_min, d0, a.dim,
                                                               c->row_dims.as<uint32_t>(),
                                                               c->union_out.as<unsigned long long>());
                cuda_check(cudaGetLastError(), "union census");
                c->union_valid = true;
            }
            tl_mark(c, "pass", s);
        }
    }
}

// Rotated device queries -> packed top-K keys [nq x k] + counts in
// out_keys/out_count (device). Stats counters left in c->counters.
void ivf_search_device(dade_gpu_ctx* c, const float* d_q, uint32_t nq, uint32_t k, uint32_t n_probe,
                       uint64_t* out_keys, uint32_t* out_count) {
    cudaStream_t s = c->stream;
    const bool resume = c->split == 2;  // phase 2 of a two-phase search: device state of phase 1 kept
    c->dense_groups = (uint64_t)nq >= 4ull * c->n_clusters;
    if (!c->probes_ready && !resume) coarse_rank(c, d_q, nq, n_probe);
    c->probes_ready = false;
    // single-phase search of a sharded index: each query's nearest LOCAL list goes
    // first (seed, first passes), else a shard missing a query's nearest list
    // would scan with r = +inf. The two-phase search keeps the global order: the
    // shard owning the nearest list seeds the query, the all-reduced radius serves the others.
    if (c->sharded && c->split == 0) {
        cuda_check(launch_local_probes(c->probes.as<uint64_t>(), nq, n_probe, c->offsets.as<uint32_t>(),
                                       c->n_clusters, s),
                   "local probes");
        ++c->launches;
    }
    tl_mark(c, "ranked", s);
    // K3 grouping
    GroupArgs g{};
    g.probes = c->probes.as<uint64_t>();
    g.nq = nq;
    g.n_probe = n_probe;
    g.n_lists = c->n_clusters;
    g.list_offsets = c->offsets.as<uint32_t>();
    // rank buckets: nearest list first, then ranks 1-3, then the rest, so
    // every query's radius is established before its far lists are scanned
    uint32_t ends[3] = {1, 4, n_probe};
    uint32_t nrb = 0;
    for (uint32_t e : ends) {
        const uint32_t v = std::min(e, n_probe);
        if (nrb == 0 || v > g.rb_end[nrb - 1]) g.rb_end[nrb++] = v;
    }
    g.n_rb = nrb;
    ChunkTable ct = make_chunks(c->dim, c->cps);
    bool tma = false;
    const CUtensorMap& tm = c->tm_storage.get(c->storage.as<float>(), std::max<uint32_t>(c->count, 1), c->dim, tma);
    ct.use_tma = (tma && ct.vec_ok && c->count > 0) ? 1 : 0;
    bool use_filter = filter_ok(c, ct, c->dim);
    bool umma = use_filter && umma_ok(c, ct, tma);
    if (c->measure && !umma) {  // failure accounting: the tcgen05 streaming path or the all-SIMT scan
        use_filter = false;
        ct.use_tc = 0;
    }
    // the streaming filter splits long lists into row pieces (more, shorter items)
    g.max_item_rows = use_filter ? kFilterItemRows : 0;
    if (umma && nrb == 3) {
        // the tcgen05 path scans ranks 1-3 and the rest in the same (last) pass: one bucket,
        // fewer and fuller items (the other paths keep the nearer ranks' items first)
        g.rb_end[1] = n_probe;
        g.n_rb = nrb = 2;
    }
    g.rank0_item_rows = use_filter && nrb > 1 ? rank0_item_rows(umma, c->dense_groups) : 0;
    g.q_chunk = umma ? kUmmaQ : use_filter ? kFilterQ : (uint32_t)kQC;
    const bool seeded = n_probe > 1 && k <= 512;
    if (use_filter && seeded) {  // the seed's rows of every nearest list are final results already
        g.seed_skip = seed_rows(c, k, c->dim);
        g.seed_min = k;
    }
    const size_t ne = (size_t)nrb * c->n_clusters;
    size_t max_items = ((size_t)nq * n_probe + g.q_chunk - 1) / g.q_chunk + ne;
    if (use_filter) {
        uint32_t max_len = 0;
        for (uint32_t l = 0; l < c->n_clusters; ++l) max_len = std::max(max_len, c->dev_offsets[l + 1] - c->dev_offsets[l]);
        const uint32_t piece = g.rank0_item_rows ? g.rank0_item_rows : kFilterItemRows;
        max_items *= std::max<uint32_t>(1, (max_len + piece - 1) / piece);
    }
    c->g_counts.ensure(ne * 4);
    c->g_cursor.ensure(ne * 4);
    c->g_boff.ensure(ne * 4);
    c->g_ioff.ensure(ne * 4);
    c->bucket_q.ensure((size_t)nq * n_probe * 4);
    c->bucket_slot.ensure((size_t)nq * n_probe * 4);
    c->items.ensure(max_items * sizeof(WorkItem));
    c->n_items.ensure(8);
    g.counts = c->g_counts.as<uint32_t>();
    g.cursor = c->g_cursor.as<uint32_t>();
    g.bucket_off = c->g_boff.as<uint32_t>();
    g.item_off = c->g_ioff.as<uint32_t>();
    g.bucket_q = c->bucket_q.as<uint32_t>();
    g.bucket_slot = c->bucket_slot.as<uint32_t>();
    g.items = c->items.as<WorkItem>();
    g.max_items = max_items;
    g.n_items = c->n_items.as<uint32_t>();
    c->seed_goff.ensure(((size_t)c->n_clusters + 1) * 4);
    g.seed_goff = c->seed_goff.as<uint32_t>();
    c->seed_glist.ensure(((size_t)nq / kSeedGroup + c->n_clusters + 1) * 4);
    g.seed_glist = c->seed_glist.as<uint32_t>();
    if (!resume) {
        cuda_check(launch_group(g, s), "group");
        c->launches += 4;
    }
    // K4 scan
    const size_t nseg = (size_t)nq * n_probe;
    c->seg_keys.ensure(nseg * k * 8);
    c->seg_count.ensure(nseg * 4);
    c->r_global.ensure((size_t)nq * 4);
    if (!resume) {
        cuda_check(cudaMemsetAsync(c->seg_count.p, 0, nseg * 4, s), "memset");
        cuda_check(launch_fill_u32(c->r_global.as<uint32_t>(), 0x7f800000u, nq, s), "fill");
    }
    ScanArgs a{};
    a.storage = c->storage.as<float>();
    a.row_ids = c->ids.as<uint32_t>();
    a.id_base = 0;
    a.dim = c->dim;
    a.queries = d_q;
    a.items = g.items;
    a.n_items = g.n_items;
    a.bucket_q = g.bucket_q;
    a.bucket_slot = g.bucket_slot;
    a.r_global = c->r_global.as<uint32_t>();
    a.seg_keys = c->seg_keys.as<uint64_t>();
    a.seg_count = c->seg_count.as<uint32_t>();
    a.n_slots = n_probe;
    a.K = k;
    a.coeff = c->d_coeff.as<double>();
    a.neg_zero2 = 0x8000000080000000ull;
    a.counters = c->counters.as<unsigned long long>();
    a.measure = c->measure ? 1u : 0u;
    if (const char* dbg = std::getenv("DADE_GPU_DEBUG"))
        if (std::atoi(dbg) == 3) a.census = c->counters.as<unsigned long long>() + 3;
    // Radius seeding: an exact (FD) pass over the first rows of every query's
    // nearest list gives each query a K-th distance before the main scan, so
    // no tile starts at r = +inf. Its top-K is discarded (the main scan
    // re-reads those rows); only the atomicMin'd radius is kept. Any K-th
    // distance of a subset of the probed candidates bounds the final radius.
    record(c, c->e1);
    if (use_filter) {
        SeedArgs sd{seeded, c->probes.as<uint64_t>(), n_probe, c->offsets.as<uint32_t>()};
        stream_passes(c, a, ct, d_q, nq, k, nrb > 1, (uint32_t)max_items, &g, c->storage.as<float>(), c->count,
                      umma ? c->tm_storage : c->tm32_storage, umma, out_keys, out_count, sd, &c->norms_storage);
        record(c, c->e2);
        return;
    }
    if (seeded && !resume) {
        cuda_check(launch_seed_radius(c->probes.as<uint64_t>(), n_probe, c->offsets.as<uint32_t>(), a.storage,
                                      a.row_ids, c->dim, d_q, nq, k, seed_rows(c, k, c->dim), a.r_global, nullptr, nullptr, s),
                   "seed radius");
        ++c->launches;
    }
    if (c->split == 1) return;  // phase 1 of the all-SIMT path: the seed's radius only
    const CUtensorMap* tn = &c->tm_none;
    if (ct.use_tc) {
        a.row_norms = c->norms_storage.get(a.storage, c->count, c->dim, ct.end[ct.n_dense - 1], s);
        if (c->norms_storage.tm_ok) tn = &c->norms_storage.map;
        else ct.use_tma = 0;
    }
    cuda_check(launch_scan(a, ct, tm, *tn, (uint32_t)max_items, true, s), "dco scan");
    record(c, c->e2);
    cuda_check(launch_merge_segments(a.seg_keys, a.seg_count, nq, n_probe, k, out_keys, out_count, s),
               "merge");
    c->launches += 3;
}

// Flat exhaustive DADE scan on the streaming path: the base is one posting list
// probed by every query (n_probe = 1), so grouping, the radius seed (its first
// rows), the tcgen05 filter, survivors and merges are the IVF ones.
bool flat_stream(dade_gpu_ctx* c, const float* d_q, uint32_t nq, uint32_t k, uint64_t* out_keys,
                 uint32_t* out_count) {
    cudaStream_t s = c->stream;
    if (std::getenv("DADE_GPU_FLAT_BLOCKS") || k > 128 || c->b_count == 0) return false;
    ChunkTable ct = make_chunks(c->b_dim, c->cps);
    bool tma = false;
    c->tm_base.get(c->base.as<float>(), std::max<uint32_t>(c->b_count, 1), c->b_dim, tma);
    ct.use_tma = (tma && ct.vec_ok) ? 1 : 0;
    if (!filter_ok(c, ct, c->b_dim) || !umma_ok(c, ct, tma)) return false;
    const bool resume = c->split == 2;  // phase 2 of a two-phase search: grouping and seed kept
    // one list [0, b_count); every query's probe 0 is it
    c->flat_offsets.ensure(8);
    c->probes.ensure((size_t)nq * 8);
    if (!resume) {
        const uint32_t h_off[2] = {0, c->b_count};
        cuda_check(cudaMemcpyAsync(c->flat_offsets.p, h_off, 8, cudaMemcpyHostToDevice, s), "H2D offsets");
        cuda_check(cudaMemsetAsync(c->probes.p, 0, (size_t)nq * 8, s), "memset");
    }
    GroupArgs g{};
    g.probes = c->probes.as<uint64_t>();
    g.nq = nq;
    g.n_probe = 1;
    g.n_lists = 1;
    g.list_offsets = c->flat_offsets.as<uint32_t>();
    g.n_rb = 1;
    g.rb_end[0] = 1;
    g.max_item_rows = kFilterItemRows;
    g.rank0_item_rows = 0;
    g.q_chunk = kUmmaQ;
    g.piece_major = 1;
    g.seed_skip = std::min<uint32_t>(seed_rows(c, k, c->b_dim, true), c->b_count);
    g.seed_min = k;
    const size_t max_items = ((size_t)nq + kUmmaQ - 1) / kUmmaQ * ((c->b_count + kFilterItemRows - 1) / kFilterItemRows) + 1;
    c->g_counts.ensure(8);
    c->g_cursor.ensure(8);
    c->g_boff.ensure(8);
    c->g_ioff.ensure(8);
    c->bucket_q.ensure((size_t)nq * 4);
    c->bucket_slot.ensure((size_t)nq * 4);
    c->items.ensure(max_items * sizeof(WorkItem));
    c->n_items.ensure(8);
    g.counts = c->g_counts.as<uint32_t>();
    g.cursor = c->g_cursor.as<uint32_t>();
    g.bucket_off = c->g_boff.as<uint32_t>();
    g.item_off = c->g_ioff.as<uint32_t>();
    g.bucket_q = c->bucket_q.as<uint32_t>();
    g.bucket_slot = c->bucket_slot.as<uint32_t>();
    g.items = c->items.as<WorkItem>();
    g.max_items = max_items;
    g.n_items = c->n_items.as<uint32_t>();
    c->seed_goff.ensure(8);
    g.seed_goff = c->seed_goff.as<uint32_t>();
    c->seed_glist.ensure(((size_t)nq / kSeedGroup + 2) * 4);
    g.seed_glist = c->seed_glist.as<uint32_t>();
    c->r_global.ensure((size_t)nq * 4);
    if (!resume) {
        cuda_check(launch_group(g, s), "group");
        c->launches += 4;
        cuda_check(launch_fill_u32(c->r_global.as<uint32_t>(), 0x7f800000u, nq, s), "fill");
    }
    ScanArgs a{};
    a.storage = c->base.as<float>();
    a.row_ids = nullptr;
    a.id_base = c->b_id_base;
    a.dim = c->b_dim;
    a.queries = d_q;
    a.items = g.items;
    a.n_items = g.n_items;
    a.bucket_q = g.bucket_q;
    a.bucket_slot = g.bucket_slot;
    a.r_global = c->r_global.as<uint32_t>();
    a.K = k;
    a.coeff = c->d_coeff.as<double>();
    a.neg_zero2 = 0x8000000080000000ull;
    a.counters = c->counters.as<unsigned long long>();
    a.measure = c->measure ? 1u : 0u;
    record(c, c->e1);
    SeedArgs sd{true, c->probes.as<uint64_t>(), 1, c->flat_offsets.as<uint32_t>()};
    stream_passes(c, a, ct, d_q, nq, k, false, (uint32_t)max_items, &g, c->base.as<float>(), c->b_count, c->tm_base,
                  true, out_keys, out_count, sd, &c->norms_base, true);
    record(c, c->e2);
    return true;
}

void flat_search_device(dade_gpu_ctx* c, const float* d_q, uint32_t nq, uint32_t k, uint64_t* out_keys,
                        uint32_t* out_count) {
    cudaStream_t s = c->stream;
    if (flat_stream(c, d_q, nq, k, out_keys, out_count)) return;
    if (c->split == 2) return;  // the row-block path is not split: phase 1 ran it whole
    const uint32_t qchunks = (nq + kQC - 1) / kQC;
    const uint32_t max_blocks = (c->b_count + kRT - 1) / kRT;
    uint32_t nb = std::max<uint32_t>(1, std::min<uint32_t>(max_blocks, (1184 + qchunks - 1) / qchunks));
    // test hook: a fixed row-block count (1 => each query's scan is one
    // sequential CTA, hence deterministic)
    if (const char* fb = std::getenv("DADE_GPU_FLAT_BLOCKS"))
        nb = std::max<uint32_t>(1, std::min<uint32_t>(max_blocks, (uint32_t)std::atoi(fb)));
    uint32_t block = (c->b_count + nb - 1) / nb;
    block = (block + kRT - 1) / kRT * kRT;
    nb = (c->b_count + block - 1) / block;
    const size_t nseg = (size_t)nq * nb;
    c->seg_keys.ensure(nseg * k * 8);
    c->seg_count.ensure(nseg * 4);
    c->r_global.ensure((size_t)nq * 4);
    cuda_check(cudaMemsetAsync(c->seg_count.p, 0, nseg * 4, s), "memset");
    cuda_check(launch_fill_u32(c->r_global.as<uint32_t>(), 0x7f800000u, nq, s), "fill");
    ScanArgs a{};
    a.storage = c->base.as<float>();
    a.row_ids = nullptr;
    a.id_base = c->b_id_base;
    a.dim = c->b_dim;
    a.queries = d_q;
    a.items = nullptr;
    a.flat_rows = c->b_count;
    a.flat_block = block;
    a.flat_nq = nq;
    a.flat_qchunks = qchunks;
    a.r_global = c->r_global.as<uint32_t>();
    a.seg_keys = c->seg_keys.as<uint64_t>();
    a.seg_count = c->seg_count.as<uint32_t>();
    a.n_slots = nb;
    a.K = k;
    a.coeff = c->d_coeff.as<double>();
    a.neg_zero2 = 0x8000000080000000ull;
    a.counters = c->counters.as<unsigned long long>();
    a.measure = c->measure ? 1u : 0u;
    ChunkTable ct = make_chunks(c->b_dim, c->cps);
    if (c->measure) ct.use_tc = 0;  // failure accounting on the all-SIMT scan
    bool tma = false;
    const CUtensorMap& tm = c->tm_base.get(a.storage, std::max<uint32_t>(c->b_count, 1), c->b_dim, tma);
    ct.use_tma = (tma && ct.vec_ok && c->b_count > 0) ? 1 : 0;
    record(c, c->e1);
    const CUtensorMap* tn = &c->tm_none;
    if (ct.use_tc) {
        a.row_norms = c->norms_base.get(a.storage, c->b_count, c->b_dim, ct.end[ct.n_dense - 1], s);
        if (c->norms_base.tm_ok) tn = &c->norms_base.map;
        else ct.use_tma = 0;
    }
    cuda_check(launch_scan(a, ct, tm, *tn, nb * qchunks, true, s), "flat scan");
    record(c, c->e2);
    cuda_check(launch_merge_segments(a.seg_keys, a.seg_count, nq, nb, k, out_keys, out_count, s), "merge");
    c->launches += 3;
}

// Query staging shared by the two searches: H2D (host path) and rotation.
// Raw host queries: H2D in chunks on the copy stream; each chunk is rotated (and
// for IVF searches coarse-ranked) on the compute stream as soon as it lands, so
// the PCIe transfer hides behind those per-query stages.
const float* stage_queries_overlapped(dade_gpu_ctx* c, const float* queries, uint32_t nq, uint32_t dim) {
    const size_t bytes = (size_t)nq * dim * 4;
    c->q_in.ensure(bytes);
    c->q_rot.ensure(bytes);
    if (!c->copy_stream) {
        cuda_check(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "stream");
        for (cudaEvent_t& e : c->copy_ev) cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    const uint32_t n_probe = c->stage_n_probe;
    const bool coarse = n_probe && c->has_ivf && dim == c->dim && coarse_tc_ok(c, n_probe);
    // Two chunks (~30% / ~70%) unless the coarse buffers cap them: the second
    // copy runs under the first chunk's rotate + coarse ranking. Per-chunk fixed
    // costs (~55 us: the coarse GEMM's and selection's latency) make finer
    // chunking a net loss (tools/chunk_sweep.sh). Every copy is enqueued before
    // any compute, so the copy engine never waits on the host's launches.
    const uint32_t cap = coarse ? coarse_tc_chunk(c, nq) : nq;
    uint32_t sizes[8], nch = 0, rem = nq;
    uint32_t want = std::max<uint32_t>(512, (uint32_t)((uint64_t)nq * 3 / 10 + 63) / 64 * 64);
    if (c->stage_one_chunk) want = nq;  // the copy already ran ahead (pipelined batches)
    while (rem && nch < 8) {
        uint32_t m = std::min<uint32_t>({rem, cap, nch == 0 ? want : rem});
        if (nch == 7) m = rem;
        if (m > cap) return nullptr;
        sizes[nch++] = m;
        rem -= m;
    }
    if (rem) return nullptr;
    // the copy stream must not overwrite q_in while earlier work reads it: when the
    // previous staging was this one, its rotations were the last readers (their
    // event lets this H2D run under the previous search); otherwise everything
    // enqueued so far may read it
    if (!c->qin_free_recorded) cuda_check(cudaEventRecord(c->copy_ev[8], c->stream), "event");
    cuda_check(cudaStreamWaitEvent(c->copy_stream, c->copy_ev[8], 0), "wait");
    for (uint32_t i = 0, q0 = 0; i < nch; q0 += sizes[i], ++i) {
        cuda_check(cudaMemcpyAsync(c->q_in.as<float>() + (size_t)q0 * dim, queries + (size_t)q0 * dim,
                                   (size_t)sizes[i] * dim * 4, cudaMemcpyHostToDevice, c->copy_stream),
                   "H2D queries");
        cuda_check(cudaEventRecord(c->copy_ev[i], c->copy_stream), "event");
        tl_mark(c, "h2d_chunk", c->copy_stream);
    }
    if (coarse) coarse_tc_begin(c, nq, n_probe);
    for (uint32_t i = 0, q0 = 0; i < nch; q0 += sizes[i], ++i) {
        const uint32_t m = sizes[i];
        cuda_check(cudaStreamWaitEvent(c->stream, c->copy_ev[i], 0), "wait");
        cuda_check(rotate_on(c, dim, c->q_in.as<float>() + (size_t)q0 * dim, m, c->q_rot.as<float>() + (size_t)q0 * dim),
                   "rotate");
        ++c->launches;
        if (coarse) coarse_tc_range(c, c->q_rot.as<float>(), q0, m, n_probe);
        tl_mark(c, "chunk_ranked", c->stream);
    }
    cuda_check(cudaEventRecord(c->copy_ev[8], c->stream), "event");  // q_in read for the last time
    c->qin_free_recorded = true;
    c->probes_ready = coarse;
    return c->q_rot.as<float>();
}

const float* stage_queries(dade_gpu_ctx* c, const float* queries, uint32_t nq, uint32_t dim,
                           uint32_t flags) {
    const size_t bytes = (size_t)nq * dim * 4;
    c->probes_ready = false;
    if (!(flags & DADE_GPU_DEVICE_PTRS) && (flags & DADE_GPU_QUERIES_RAW) && c->t_dim == dim && (nq >= 2048 || c->stage_one_chunk) &&
        !env_flag("DADE_GPU_NO_OVERLAP"))
        if (const float* d = stage_queries_overlapped(c, queries, nq, dim)) return d;
    const float* d_in = queries;
    c->qin_free_recorded = false;
    if (!(flags & DADE_GPU_DEVICE_PTRS)) {
        c->q_in.ensure(bytes);
        cuda_check(cudaMemcpyAsync(c->q_in.p, queries, bytes, cudaMemcpyHostToDevice, c->stream), "H2D queries");
        d_in = c->q_in.as<float>();
    }
    if (flags & DADE_GPU_QUERIES_RAW) {
        if (c->t_dim != dim) fail(DADE_GPU_CONFIG_ERROR, "raw queries need a transform of the index dim");
        c->q_rot.ensure(bytes);
        cuda_check(rotate_on(c, dim, d_in, nq, c->q_rot.as<float>()), "rotate");
        ++c->launches;
        return c->q_rot.as<float>();
    }
    return d_in;
}

void collect_stats(dade_gpu_ctx* c, dade_gpu_stats* stats) {
    if (!stats) return;
    unsigned long long h[10] = {};
    cuda_check(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream), "D2H stats");
    cuda_check(cudaStreamSynchronize(c->stream), "sync");
    stats->total_dco += h[0];
    stats->dims_accumulated += h[1];
    if (c->measure) {  // DcoStats::measure_failures (proj/include/dade/estimator.hpp:31-34)
        stats->eligible += h[8];
        stats->failures += h[9];
    }
}

// Failure accounting hands every DCO pair to the survivor kernel (16 B each),
// so a search with DADE_GPU_MEASURE_FAILURES runs in query chunks of at most
// ~2^27 pairs. The flag is cleared however the search exits.
struct MeasureScope {
    dade_gpu_ctx* c;
    MeasureScope(dade_gpu_ctx* cc, bool on) : c(cc) { c->measure = on; }
    ~MeasureScope() { c->measure = false; }
    MeasureScope(const MeasureScope&) = delete;
    MeasureScope& operator=(const MeasureScope&) = delete;
};
uint32_t measure_chunk(uint64_t pairs_per_query, uint32_t nq) {
    const uint64_t budget = 1ull << 27;
    return (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(std::max<uint32_t>(nq, 1),
                                                              budget / std::max<uint64_t>(1, pairs_per_query)));
}

void wait_stream(cudaStream_t s) { cuda_check(cudaStreamSynchronize(s), "search"); }

// Overflow flags of the search just enqueued (worklist, coarse candidate list):
// read back with the results in one pinned copy; check after the sync.
void enqueue_flags(dade_gpu_ctx* c) {
    if (!c->h_flags) cuda_check(cudaMallocHost(reinterpret_cast<void**>(&c->h_flags), 8), "cudaMallocHost");
    c->h_flags[0] = c->h_flags[1] = 0;
    if (c->surv_cap_used)
        cuda_check(cudaMemcpyAsync(c->h_flags, c->surv_max.p, 4, cudaMemcpyDeviceToHost, c->stream), "D2H flags");
    if (c->coarse_tc_used)
        cuda_check(cudaMemcpyAsync(c->h_flags + 1, c->coarse_overflow.p, 4, cudaMemcpyDeviceToHost, c->stream),
                   "D2H flags");
}

// after the sync: true if the search must be redone (and the redo is configured)
bool search_overflowed(dade_gpu_ctx* c) {
    if (c->surv_cap_used && c->h_flags[0] > c->surv_cap_used) {
        c->surv_cap_hint = (uint32_t)std::min<uint64_t>(0xffffffffull, (uint64_t)c->h_flags[0] * 2);
        c->surv_cap_used = 0;
        return true;
    }
    if (c->surv_cap_used) c->surv_cap_hint = std::max(c->surv_cap_hint, c->h_flags[0]);
    return false;
}

// The search body (coarse ranking, grouping, the DCO scan, merges: ~30 launches
// and memsets on one stream, no host sync) as a CUDA graph. The first run of a
// key is eager (it sizes every workspace, tensor map and cached row operand),
// a repeat is captured, later ones replay the instantiated graph: the GPU then
// runs the launches back to back instead of waiting on each launch's issue.
// Off for diagnostic runs (profiling, timeline, failure accounting, estimate
// dumps, two-phase searches, DADE_GPU_DEBUG) and with DADE_GPU_NO_GRAPH=1.
bool graph_usable(const dade_gpu_ctx* c) {
    static const bool env_off = env_flag("DADE_GPU_NO_GRAPH") || std::getenv("DADE_GPU_DEBUG") ||
                                std::getenv("DADE_GPU_SURV_CAP");
    return c->graphs_on && !env_off && !c->profiling && !c->tl_on && !c->measure && !c->dump_cap && c->split == 0 &&
           c->stream != nullptr && c->stream != cudaStreamLegacy && c->stream != cudaStreamPerThread;
}

void search_graphed(dade_gpu_ctx* c, uint64_t tag, const float* d_q, uint32_t nq, uint32_t k, uint64_t* ok,
                    uint32_t* oc, const std::function<void(const float*, uint64_t*, uint32_t*)>& run) {
    if (!tag || !graph_usable(c)) {
        run(d_q, ok, oc);
        return;
    }
    const std::array<uint64_t, 14> key = {
        tag,
        reinterpret_cast<uint64_t>(d_q),
        reinterpret_cast<uint64_t>(ok),
        reinterpret_cast<uint64_t>(oc),
        reinterpret_cast<uint64_t>(c->fo.ids),
        reinterpret_cast<uint64_t>(c->fo.dists),
        reinterpret_cast<uint64_t>(c->fo.counts),
        ((uint64_t)nq << 32) | k,
        reinterpret_cast<uint64_t>(c->stream),
        g_alloc_epoch,
        c->cfg_epoch,
        c->surv_cap_hint,
        (uint64_t)c->probes_ready | ((uint64_t)c->coarse_force_exact << 1) | ((uint64_t)c->sharded << 2) |
            ((uint64_t)c->coarse_all << 3) | ((uint64_t)c->coarse_exact_keys << 4),
        (uint64_t)c->seed_rows_set};
    for (auto& e : c->graphs)
        if (e.key == key) {
            cuda_check(cudaGraphLaunch(e.exec, c->stream), "graph launch");
            e.lru = ++c->graph_tick;
            c->launches += e.launches;
            c->surv_cap_used = e.surv_cap_used;
            c->n_filter_passes = e.n_filter_passes;
            c->coarse_tc_used = e.coarse_tc_used;
            c->fo.done = e.fo_done;
            c->probes_ready = false;
            return;
        }
    if (c->graph_seen != key) {  // first sighting: eager
        run(d_q, ok, oc);
        c->graph_seen = key;
        return;
    }
    const uint64_t l0 = c->launches;
    cudaGraph_t g = nullptr;
    cuda_check(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
    try {
        run(d_q, ok, oc);
    } catch (...) {
        cudaStreamEndCapture(c->stream, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        throw;
    }
    cuda_check(cudaStreamEndCapture(c->stream, &g), "end capture");
    cudaGraphExec_t ex = nullptr;
    const cudaError_t ie = g_alloc_epoch == key[9] ? cudaGraphInstantiate(&ex, g, 0) : cudaErrorInvalidValue;
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) {  // (a workspace grew during the capture: run it eagerly, capture next time)
        cudaGetLastError();
        c->launches = l0;
        run(d_q, ok, oc);
        c->graph_seen = {};
        return;
    }
    if (c->graphs.size() >= 6) {  // evict the least recently used
        auto it = std::min_element(c->graphs.begin(), c->graphs.end(),
                                   [](const auto& a, const auto& b) { return a.lru < b.lru; });
        cudaGraphExecDestroy(it->exec);
        c->graphs.erase(it);
    }
    dade_gpu_ctx::GraphEntry e;
    e.key = key;
    e.exec = ex;
    e.launches = c->launches - l0;
    e.lru = ++c->graph_tick;
    e.surv_cap_used = c->surv_cap_used;
    e.n_filter_passes = c->n_filter_passes;
    e.coarse_tc_used = c->coarse_tc_used;
    e.fo_done = c->fo.done;
    c->graphs.push_back(e);
    cuda_check(cudaGraphLaunch(ex, c->stream), "graph launch");
}

// Common driver: results as ids/dists/counts (host or device).
void search_common(dade_gpu_ctx* c, const float* queries, uint32_t nq, uint32_t dim, uint32_t k,
                   uint32_t flags, uint32_t* out_ids, float* out_dists, uint32_t* out_counts,
                   dade_gpu_stats* stats, const std::function<void(const float*, uint64_t*, uint32_t*)>& run,
                   uint64_t graph_tag = 0) {
    c->use_device();
    cudaStream_t s = c->stream;
    c->counters.ensure(kCounterBytes);
    cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, s), "memset");
    record(c, c->e0);
    c->tl_on = env_flag("DADE_GPU_TIMELINE");
    c->tl_used = 0;
    tl_mark(c, "start", s);
    c->n_filter_passes = 0;
    c->surv_cap_used = 0;
    if (nq == 0) return;
    const float* d_q = stage_queries(c, queries, nq, dim, flags);
    tl_mark(c, "staged", s);
    c->out_keys.ensure((size_t)nq * k * 8);
    c->out_count.ensure((size_t)nq * 4);
    const bool dev = flags & DADE_GPU_DEVICE_PTRS;
    uint32_t* ids = out_ids;
    float* dists = out_dists;
    uint32_t* cnts = out_counts;
    if (!dev) {
        c->out_ids.ensure((size_t)nq * k * 4);
        c->out_dists.ensure((size_t)nq * k * 4);
        c->out_counts.ensure((size_t)nq * 4);
        ids = c->out_ids.as<uint32_t>();
        dists = c->out_dists.as<float>();
        cnts = c->out_counts.as<uint32_t>();
    }
    // the streaming path's last slot merge writes ids / dists / counts itself (fo.done)
    bool fused = false;
    {
        FusedOutputs scope(c, ids, dists, cnts);
        search_graphed(c, graph_tag, d_q, nq, k, c->out_keys.as<uint64_t>(), c->out_count.as<uint32_t>(), run);
        fused = c->fo.done;
    }
    tl_mark(c, "searched", s);
    if (!fused) {
        cuda_check(launch_keys_to_results(c->out_keys.as<uint64_t>(), c->out_count.as<uint32_t>(), nq, k, ids,
                                          dists, cnts, s),
                   "keys_to_results");
        ++c->launches;
    }
    if (!dev) {
        cuda_check(cudaMemcpyAsync(out_ids, ids, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, s), "D2H ids");
        cuda_check(cudaMemcpyAsync(out_dists, dists, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, s), "D2H dists");
        if (out_counts)
            cuda_check(cudaMemcpyAsync(out_counts, cnts, (size_t)nq * 4, cudaMemcpyDeviceToHost, s), "D2H counts");
    }
    tl_mark(c, "results_d2h", s);
    record(c, c->e3);
    enqueue_flags(c);
    wait_stream(s);
    if (search_overflowed(c)) {  // survivor worklist too small: redo with the observed size x2
        search_common(c, queries, nq, dim, k, flags, out_ids, out_dists, out_counts, stats, run, graph_tag);
        return;
    }
    if (c->coarse_tc_used) {
        // more boundary candidates than the exact stage holds (pathological
        // ties): redo the search with the all-exact coarse ranking
        const uint32_t ov = c->h_flags[1];
        if (ov) {
            c->coarse_force_exact = true;
            try {
                search_common(c, queries, nq, dim, k, flags, out_ids, out_dists, out_counts, stats, run, graph_tag);
            } catch (...) {
                c->coarse_force_exact = false;
                throw;
            }
            c->coarse_force_exact = false;
            return;
        }
    }
    collect_stats(c, stats);
    finish_profile(c);
    tl_print(c);
}

// Pipelined sequence of searches over host batches: batch b+1's H2D (copy
// stream) runs under batch b's search, batch b's D2H (d2h stream) under batch
// b+1's. Results land in two device buffer sets used alternately; a set is
// rewritten only after its previous D2H completed. Overflow flags and DcoStats
// counters of each batch are snapshotted on the compute stream next to its
// results and checked after the final sync; an overflowed batch is redone by
// search_common (same results as a sequence of single searches).
void search_batches(dade_gpu_ctx* c, uint32_t nb, const float* const* queries, uint32_t nq, uint32_t dim, uint32_t k,
                    uint32_t flags, uint32_t* const* out_ids, float* const* out_dists, uint32_t* const* out_counts,
                    dade_gpu_stats* stats, const std::function<void(const float*, uint64_t*, uint32_t*)>& run,
                    uint64_t graph_tag = 0) {
    c->use_device();
    if (nb == 0 || nq == 0) return;
    cudaStream_t s = c->stream;
    if (!c->d2h_stream) {
        cuda_check(cudaStreamCreateWithFlags(&c->d2h_stream, cudaStreamNonBlocking), "stream");
        for (int j = 0; j < 2; ++j) {
            cuda_check(cudaEventCreateWithFlags(&c->res_ev[j], cudaEventDisableTiming), "event");
            cuda_check(cudaEventCreateWithFlags(&c->d2h_ev[j], cudaEventDisableTiming), "event");
        }
    }
    if (c->h_batch_n < nb) {
        if (c->h_batch) cudaFreeHost(c->h_batch);
        c->h_batch = nullptr;
        cuda_check(cudaMallocHost(reinterpret_cast<void**>(&c->h_batch), (size_t)nb * 32), "cudaMallocHost");
        c->h_batch_n = nb;
    }
    std::memset(c->h_batch, 0, (size_t)nb * 32);
    c->counters.ensure(kCounterBytes);
    c->batch_slot.ensure(2 * 32);
    c->out_keys.ensure((size_t)nq * k * 8);
    c->out_count.ensure((size_t)nq * 4);
    for (int j = 0; j < 2; ++j) {
        c->res_ids[j].ensure((size_t)nq * k * 4);
        c->res_dists[j].ensure((size_t)nq * k * 4);
        c->res_counts[j].ensure((size_t)nq * 4);
    }
    // profiling / one-chunk staging are restored however the loop exits
    struct Restore {
        dade_gpu_ctx* c;
        bool prof;
        ~Restore() {
            c->profiling = prof;
            c->stage_one_chunk = false;
        }
    } restore{c, c->profiling};
    c->profiling = false;
    c->tl_on = false;
    std::vector<uint32_t> cap_used(nb, 0);
    std::vector<uint8_t> coarse_used(nb, 0);
    for (uint32_t b = 0; b < nb; ++b) {
        const uint32_t j = b & 1;
        cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, s), "memset");
        c->n_filter_passes = 0;
        c->surv_cap_used = 0;
        // batch b > 0: its H2D ran under batch b-1's search, so per-chunk staging
        // would only add the coarse stage's fixed latency per chunk
        c->stage_one_chunk = b > 0;
        const float* d_q = stage_queries(c, queries[b], nq, dim, flags);
        c->stage_one_chunk = false;
        if (b >= 2) cuda_check(cudaStreamWaitEvent(s, c->d2h_ev[j], 0), "wait");  // set j's D2H done
        bool fused = false;
        {
            FusedOutputs scope(c, c->res_ids[j].as<uint32_t>(), c->res_dists[j].as<float>(),
                               c->res_counts[j].as<uint32_t>());
            search_graphed(c, graph_tag, d_q, nq, k, c->out_keys.as<uint64_t>(), c->out_count.as<uint32_t>(), run);
            fused = c->fo.done;
        }
        cap_used[b] = c->surv_cap_used;
        coarse_used[b] = c->coarse_tc_used;
        if (!fused) {
            cuda_check(launch_keys_to_results(c->out_keys.as<uint64_t>(), c->out_count.as<uint32_t>(), nq, k,
                                              c->res_ids[j].as<uint32_t>(), c->res_dists[j].as<float>(),
                                              c->res_counts[j].as<uint32_t>(), s),
                       "keys_to_results");
            ++c->launches;
        }
        auto* slot = reinterpret_cast<unsigned char*>(c->batch_slot.p) + 32 * j;
        cuda_check(cudaMemsetAsync(slot, 0, 16, s), "memset");
        if (cap_used[b]) cuda_check(cudaMemcpyAsync(slot, c->surv_max.p, 4, cudaMemcpyDeviceToDevice, s), "flags");
        if (coarse_used[b])
            cuda_check(cudaMemcpyAsync(slot + 8, c->coarse_overflow.p, 4, cudaMemcpyDeviceToDevice, s), "flags");
        cuda_check(cudaMemcpyAsync(slot + 16, c->counters.p, 16, cudaMemcpyDeviceToDevice, s), "counters");
        cuda_check(cudaEventRecord(c->res_ev[j], s), "event");
        cudaStream_t t = c->d2h_stream;
        cuda_check(cudaStreamWaitEvent(t, c->res_ev[j], 0), "wait");
        cuda_check(cudaMemcpyAsync(out_ids[b], c->res_ids[j].p, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, t), "D2H ids");
        cuda_check(cudaMemcpyAsync(out_dists[b], c->res_dists[j].p, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, t),
                   "D2H dists");
        if (out_counts && out_counts[b])
            cuda_check(cudaMemcpyAsync(out_counts[b], c->res_counts[j].p, (size_t)nq * 4, cudaMemcpyDeviceToHost, t),
                       "D2H counts");
        cuda_check(cudaMemcpyAsync(c->h_batch + 4 * (size_t)b, slot, 32, cudaMemcpyDeviceToHost, t), "D2H flags");
        cuda_check(cudaEventRecord(c->d2h_ev[j], t), "event");
    }
    wait_stream(s);
    wait_stream(c->d2h_stream);
    c->profiling = restore.prof;
    for (uint32_t b = 0; b < nb; ++b) {
        const unsigned long long* h = c->h_batch + 4 * (size_t)b;
        const bool surv_over = cap_used[b] && h[0] > cap_used[b];
        if (cap_used[b]) c->surv_cap_hint = std::max<uint32_t>(c->surv_cap_hint, (uint32_t)std::min<unsigned long long>(h[0], 0xffffffffull));
        if (surv_over || (coarse_used[b] && (uint32_t)h[1])) {
            // the single-search driver redoes it (larger worklist / all-exact coarse ranking)
            search_common(c, queries[b], nq, dim, k, flags, out_ids[b], out_dists[b],
                          out_counts ? out_counts[b] : nullptr, stats, run, graph_tag);
            continue;
        }
        if (stats) {
            stats->total_dco += h[2];
            stats->dims_accumulated += h[3];
        }
    }
}

}  // namespace

extern "C" {

const char* dade_gpu_last_error(void) { return g_last_error.c_str(); }
const char* dade_gpu_version(void) { return "dade_gpu 0.1 sm_100a"; }

int dade_gpu_create(int device, dade_gpu_ctx** out) {
    return guarded([&] {
        if (!out) fail(DADE_GPU_INVALID_INPUT, "create: out is null");
        int n = 0;
        cuda_check(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n) fail(DADE_GPU_INVALID_INPUT, "create: no such device");
        auto* c = new dade_gpu_ctx;
        c->device = device;
        c->use_device();
        // blocking stream: orders with the legacy default stream callers use
        cuda_check(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamDefault), "stream");
        c->stream = c->own_stream;
        cuda_check(cudaEventCreate(&c->e0), "event");
        cuda_check(cudaEventCreate(&c->e1), "event");
        cuda_check(cudaEventCreate(&c->e2), "event");
        cuda_check(cudaEventCreate(&c->e3), "event");
        for (auto& e : c->ef) cuda_check(cudaEventCreate(&e), "event");
        for (auto& e : c->es) cuda_check(cudaEventCreate(&e), "event");
        cuda_check(cudaDeviceGetAttribute(&c->n_sms, cudaDevAttrMultiProcessorCount, device), "attr");
        *out = c;
    });
}

int dade_gpu_destroy(dade_gpu_ctx* c) {
    return guarded([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        cudaStreamSynchronize(c->stream);
        if (c->h_flags) cudaFreeHost(c->h_flags);
        c->h_flags = nullptr;
        if (c->copy_stream) {
            cudaStreamSynchronize(c->copy_stream);
            for (cudaEvent_t e : c->copy_ev) cudaEventDestroy(e);
            cudaStreamDestroy(c->copy_stream);
            c->copy_stream = nullptr;
        }
        if (c->d2h_stream) {
            cudaStreamSynchronize(c->d2h_stream);
            for (int j = 0; j < 2; ++j) {
                cudaEventDestroy(c->res_ev[j]);
                cudaEventDestroy(c->d2h_ev[j]);
            }
            cudaStreamDestroy(c->d2h_stream);
            c->d2h_stream = nullptr;
        }
        if (c->h_batch) cudaFreeHost(c->h_batch);
        c->h_batch = nullptr;
        c->norms_storage.buf.release();
        c->aug_storage.buf.release();
        c->aug_storage.rows = nullptr;
        c->norms_base.buf.release();
        DevBuf* bufs[] = {&c->W, &c->centroids, &c->storage, &c->ids, &c->offsets, &c->base,
                          &c->d_cps, &c->d_coeff, &c->d_scale, &c->q_in, &c->q_rot, &c->probes,
                          &c->probe_count, &c->c_seg_keys, &c->c_seg_count, &c->c_r, &c->g_counts,
                          &c->g_cursor, &c->g_boff, &c->g_ioff, &c->bucket_q, &c->bucket_slot,
                          &c->items, &c->n_items, &c->seg_keys, &c->seg_count, &c->r_global,
                          &c->out_keys, &c->out_count, &c->out_ids, &c->out_dists, &c->out_counts,
                          &c->counters};
        for (DevBuf* b : bufs) b->release();
        cudaEventDestroy(c->e0);
        cudaEventDestroy(c->e1);
        cudaEventDestroy(c->e2);
        cudaEventDestroy(c->e3);
        for (auto& e : c->ef) cudaEventDestroy(e);
        for (auto& e : c->graphs) cudaGraphExecDestroy(e.exec);
        c->graphs.clear();
        cudaStreamDestroy(c->own_stream);
        delete c;
    });
}

int dade_gpu_set_stream(dade_gpu_ctx* c, void* stream) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        c->stream = stream ? static_cast<cudaStream_t>(stream) : c->own_stream;
    });
}

int dade_gpu_get_stream(dade_gpu_ctx* c, void** stream) {
    return guarded([&] {
        if (!c || !stream) fail(DADE_GPU_INVALID_INPUT, "get_stream: null argument");
        *stream = c->stream;
    });
}

int dade_gpu_index_dims(dade_gpu_ctx* c, uint32_t* ivf_dim, uint32_t* base_dim) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (ivf_dim) {
            if (!c->has_ivf) fail(DADE_GPU_CONFIG_ERROR, "IvfIndex::search: no ivf index uploaded");
            *ivf_dim = c->dim;
        }
        if (base_dim) {
            if (!c->has_base) fail(DADE_GPU_CONFIG_ERROR, "linear_scan: no base vectors uploaded");
            *base_dim = c->b_dim;
        }
    });
}

int dade_gpu_synchronize(dade_gpu_ctx* c) {
    return guarded([&] {
        c->use_device();
        cuda_check(cudaStreamSynchronize(c->stream), "synchronize");
    });
}

int dade_gpu_set_transform(dade_gpu_ctx* c, uint32_t dim, const double* matrix, const double* eig) {
    return guarded([&] {
        if (!c || !matrix || !eig) fail(DADE_GPU_INVALID_INPUT, "set_transform: null argument");
        if (dim == 0) fail(DADE_GPU_INVALID_INPUT, "set_transform: dim must be positive");
        // prefix sums of the clamped variances (transform.cpp:21-36)
        std::vector<double> pre(dim + 1, 0.0);
        for (uint32_t i = 0; i < dim; ++i) {
            double v = eig[i];
            if (v < -1e-6) fail(DADE_GPU_RUNTIME_ERROR, "eigenvalue below tolerance; not a covariance");
            if (v < 0.0) v = 0.0;
            pre[i + 1] = pre[i] + v;
        }
        c->use_device();
        upload(c->W, matrix, (size_t)dim * dim * 8, c->stream);
        cuda_check(cudaStreamSynchronize(c->stream), "transform upload");
        c->t_dim = dim;
        c->lambda_prefix = std::move(pre);
        c->config_changed();
    });
}

int dade_gpu_set_ivf(dade_gpu_ctx* c, uint32_t dim, uint32_t count, uint32_t n_clusters, uint32_t layout,
                     uint32_t split, const float* centroids, const uint32_t* offsets, const uint32_t* ids,
                     const float* storage) {
    return guarded([&] {
        if (!c || !centroids || !offsets || (count && (!ids || !storage)))
            fail(DADE_GPU_INVALID_INPUT, "set_ivf: null argument");
        if (dim == 0 || n_clusters == 0) fail(DADE_GPU_RUNTIME_ERROR, "inconsistent ivf header");
        if (layout > 1) fail(DADE_GPU_RUNTIME_ERROR, "bad ivf layout byte");
        if (layout == 1 && (split == 0 || split > dim)) fail(DADE_GPU_RUNTIME_ERROR, "inconsistent ivf header");
        if (offsets[0] != 0 || offsets[n_clusters] != count)
            fail(DADE_GPU_RUNTIME_ERROR, "inconsistent ivf posting offsets");
        for (uint32_t i = 0; i < n_clusters; ++i)
            if (offsets[i + 1] < offsets[i]) fail(DADE_GPU_RUNTIME_ERROR, "inconsistent ivf posting offsets");
        c->use_device();
        // Device layout = contiguous rows in posting order (ivf.cpp:195-205);
        // a split payload is re-interleaved row by row on the host.
        const float* rows = storage;
        std::vector<float> tmp;
        if (layout == 1 && split != dim) {
            tmp.resize((size_t)count * dim);
            for (uint32_t cl = 0; cl < n_clusters; ++cl) {
                const uint32_t b = offsets[cl], len = offsets[cl + 1] - b;
                const float* blk = storage + (size_t)b * dim;
                for (uint32_t pos = 0; pos < len; ++pos) {
                    float* dst = tmp.data() + (size_t)(b + pos) * dim;
                    std::memcpy(dst, blk + (size_t)pos * split, sizeof(float) * split);
                    std::memcpy(dst + split, blk + (size_t)len * split + (size_t)pos * (dim - split),
                                sizeof(float) * (dim - split));
                }
            }
            rows = tmp.data();
        }
        upload(c->centroids, centroids, (size_t)n_clusters * dim * 4, c->stream);
        upload(c->storage, rows, (size_t)count * dim * 4, c->stream);
        upload(c->ids, ids, (size_t)count * 4, c->stream);
        upload(c->offsets, offsets, (size_t)(n_clusters + 1) * 4, c->stream);
        cuda_check(cudaStreamSynchronize(c->stream), "ivf upload");
        c->dim = dim;
        c->count = count;
        c->n_clusters = n_clusters;
        c->norms_storage.rows = nullptr;
        c->aug_storage.rows = nullptr;
        c->h_offsets.assign(offsets, offsets + n_clusters + 1);
        c->dev_offsets = c->h_offsets;
        c->has_ivf = true;
        c->sharded = false;
        c->flat_parts = 0;
        c->config_changed();
    });
}

int dade_gpu_set_ivf_shard(dade_gpu_ctx* c, const uint8_t* mask) {
    return guarded([&] {
        if (!c || !mask) fail(DADE_GPU_INVALID_INPUT, "set_ivf_shard: null argument");
        if (!c->has_ivf) fail(DADE_GPU_CONFIG_ERROR, "set_ivf_shard: no ivf index");
        c->use_device();
        // Compact the kept lists' rows on the device, keep global offsets for
        // removed lists at zero length.
        const uint32_t nl = c->n_clusters;
        std::vector<uint32_t> dev(nl + 1, 0);
        size_t rows = 0;
        for (uint32_t l = 0; l < nl; ++l) {
            dev[l] = (uint32_t)rows;
            if (mask[l]) rows += c->dev_offsets[l + 1] - c->dev_offsets[l];
            else if (c->dev_offsets[l + 1] > c->dev_offsets[l]) c->sharded = true;
        }
        dev[nl] = (uint32_t)rows;
        DevBuf ns, ni;
        ns.ensure(rows * c->dim * 4);
        ni.ensure(rows * 4);
        for (uint32_t l = 0; l < nl; ++l) {
            if (!mask[l]) continue;
            const uint32_t src = c->dev_offsets[l], len = c->dev_offsets[l + 1] - src;
            if (!len) continue;
            cuda_check(cudaMemcpyAsync(ns.as<float>() + (size_t)dev[l] * c->dim,
                                       c->storage.as<float>() + (size_t)src * c->dim,
                                       (size_t)len * c->dim * 4, cudaMemcpyDeviceToDevice, c->stream),
                       "shard copy");
            cuda_check(cudaMemcpyAsync(ni.as<uint32_t>() + dev[l], c->ids.as<uint32_t>() + src, (size_t)len * 4,
                                       cudaMemcpyDeviceToDevice, c->stream),
                       "shard copy");
        }
        cuda_check(cudaStreamSynchronize(c->stream), "shard");
        c->storage.release();
        c->ids.release();
        c->storage = std::move(ns);
        c->ids = std::move(ni);
        ns.p = nullptr;
        ni.p = nullptr;
        upload(c->offsets, dev.data(), (size_t)(nl + 1) * 4, c->stream);
        cuda_check(cudaStreamSynchronize(c->stream), "shard");
        c->dev_offsets = dev;
        c->count = (uint32_t)rows;
        c->norms_storage.rows = nullptr;
        c->aug_storage.rows = nullptr;
        c->flat_parts = 0;
        c->config_changed();
    });
}

int dade_gpu_set_base(dade_gpu_ctx* c, uint32_t dim, uint32_t count, const float* data, uint32_t id_base) {
    return guarded([&] {
        if (!c || (count && !data)) fail(DADE_GPU_INVALID_INPUT, "set_base: null argument");
        if (dim == 0) fail(DADE_GPU_INVALID_INPUT, "VectorSet: dim must be positive");
        c->use_device();
        upload(c->base, data, (size_t)count * dim * 4, c->stream);
        cuda_check(cudaStreamSynchronize(c->stream), "base upload");
        c->norms_base.rows = nullptr;
        c->b_dim = dim;
        c->b_count = count;
        c->b_id_base = id_base;
        c->has_base = true;
        c->flat_parts = 0;
        c->config_changed();
    });
}

int dade_gpu_set_strategy(dade_gpu_ctx* c, uint32_t kind, uint32_t dim, uint32_t n, const uint32_t* cps,
                          const double* coeff, const double* scale) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (kind > DADE_GPU_DADE) fail(DADE_GPU_INVALID_INPUT, "unknown strategy kind");
        if (kind == DADE_GPU_FD) n = 0;
        if (n && (!cps || !coeff || !scale)) fail(DADE_GPU_INVALID_INPUT, "set_strategy: null tables");
        set_tables(c, kind, dim, std::vector<uint32_t>(cps, cps + n), std::vector<double>(coeff, coeff + n),
                   std::vector<double>(scale, scale + n));
    });
}

// DadeStrategy::DadeStrategy (proj/src/estimator.cpp:115-152).
int dade_gpu_set_strategy_dade(dade_gpu_ctx* c, uint32_t delta_d, uint32_t cal_delta_d, uint32_t n,
                               const uint32_t* cal_cps, const double* cal_eps) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (c->t_dim == 0) fail(DADE_GPU_CONFIG_ERROR, "DadeStrategy: no transform set");
        const uint32_t dim = c->t_dim;
        if (delta_d == 0) fail(DADE_GPU_INVALID_INPUT, "DadeStrategy: delta_d must be positive");
        if (cal_delta_d != delta_d)
            fail(DADE_GPU_CONFIG_ERROR, "calibration step " + std::to_string(cal_delta_d) +
                                            " does not match requested step " + std::to_string(delta_d));
        const auto expected = expected_checkpoints(dim, delta_d);
        std::vector<uint32_t> have(cal_cps, cal_cps + n);
        if (have != expected) {
            std::string msg = "calibration table does not cover checkpoints for dim " + std::to_string(dim) +
                              " step " + std::to_string(delta_d);
            for (uint32_t d : expected)
                if (std::find(have.begin(), have.end(), d) == have.end()) {
                    msg += "; first missing checkpoint " + std::to_string(d);
                    break;
                }
            fail(DADE_GPU_CONFIG_ERROR, msg);
        }
        const auto& pre = c->lambda_prefix;
        std::vector<double> coeff(n), scale(n);
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t d = have[i];
            const double ope = 1.0 + cal_eps[i];
            if (!(pre[d] > 0.0)) {
                coeff[i] = std::numeric_limits<double>::infinity();
                scale[i] = 1.0;
            } else {
                const double s = pre[dim] / pre[d];
                coeff[i] = ope * ope / s;
                scale[i] = s;
            }
        }
        set_tables(c, DADE_GPU_DADE, dim, have, coeff, scale);
    });
}

// AdsamplingStrategy::AdsamplingStrategy (proj/src/estimator.cpp:158-172).
int dade_gpu_set_strategy_ads(dade_gpu_ctx* c, uint32_t dim, uint32_t delta_d, double eps0) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (dim == 0) fail(DADE_GPU_INVALID_INPUT, "AdsamplingStrategy: dim must be positive");
        if (delta_d == 0) fail(DADE_GPU_INVALID_INPUT, "AdsamplingStrategy: delta_d must be positive");
        if (eps0 < 0.0) fail(DADE_GPU_INVALID_INPUT, "AdsamplingStrategy: eps0 must be nonnegative");
        const auto cps = expected_checkpoints(dim, delta_d);
        std::vector<double> coeff(cps.size()), scale(cps.size());
        for (size_t i = 0; i < cps.size(); ++i) {
            const double d = cps[i];
            const double ope = 1.0 + eps0 / std::sqrt(d);
            coeff[i] = d / dim * ope * ope;
            scale[i] = dim / d;
        }
        set_tables(c, DADE_GPU_ADS, dim, cps, coeff, scale);
    });
}

int dade_gpu_rotate(dade_gpu_ctx* c, const float* in, uint32_t n, float* out, uint32_t flags) {
    return guarded([&] {
        if (!c || (n && (!in || !out))) fail(DADE_GPU_INVALID_INPUT, "rotate: null argument");
        if (c->t_dim == 0) fail(DADE_GPU_CONFIG_ERROR, "rotate: no transform set");
        c->use_device();
        const size_t bytes = (size_t)n * c->t_dim * 4;
        if (flags & DADE_GPU_DEVICE_PTRS) {
            cuda_check(rotate_on(c, c->t_dim, in, n, out), "rotate");
            ++c->launches;
            return;
        }
        c->q_in.ensure(bytes);
        c->q_rot.ensure(bytes);
        cuda_check(cudaMemcpyAsync(c->q_in.p, in, bytes, cudaMemcpyHostToDevice, c->stream), "H2D");
        cuda_check(rotate_on(c, c->t_dim, c->q_in.as<float>(), n, c->q_rot.as<float>()), "rotate");
        ++c->launches;
        cuda_check(cudaMemcpyAsync(out, c->q_rot.p, bytes, cudaMemcpyDeviceToHost, c->stream), "D2H");
        cuda_check(cudaStreamSynchronize(c->stream), "rotate");
    });
}

// IvfIndex::search argument checks (proj/src/ivf.cpp:209-213).
static void check_ivf_args(dade_gpu_ctx* c, uint32_t k, uint32_t n_probe) {
    if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
    if (!c->has_ivf) fail(DADE_GPU_CONFIG_ERROR, "IvfIndex::search: no ivf index uploaded");
    if (k == 0) fail(DADE_GPU_INVALID_INPUT, "IvfIndex::search: k must be positive");
    if (n_probe == 0 || n_probe > c->n_clusters)
        fail(DADE_GPU_INVALID_INPUT,
             "IvfIndex::search: n_probe must be in [1, n_clusters], got " + std::to_string(n_probe));
    require_strategy(c, c->dim, "IvfIndex::search");
}

static void check_flat_args(dade_gpu_ctx* c, uint32_t k) {
    if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
    if (!c->has_base) fail(DADE_GPU_CONFIG_ERROR, "linear_scan: no base vectors uploaded");
    if (k == 0) fail(DADE_GPU_INVALID_INPUT, "linear_scan: k must be positive");
    require_strategy(c, c->b_dim, "linear_scan");
}

int dade_gpu_ivf_search(dade_gpu_ctx* c, const float* queries, uint32_t nq, uint32_t k, uint32_t n_probe,
                        uint32_t flags, uint32_t* out_ids, float* out_dists, uint32_t* out_counts,
                        dade_gpu_stats* stats) {
    return guarded([&] {
        check_ivf_args(c, k, n_probe);
        if (nq && (!queries || !out_ids || !out_dists)) fail(DADE_GPU_INVALID_INPUT, "ivf_search: null argument");
        const bool measure = flags & DADE_GPU_MEASURE_FAILURES;
        MeasureScope ms(c, measure);
        uint32_t chunk = nq;
        if (measure) {  // every probed pair goes to the survivor worklist: bound it per chunk
            uint32_t max_len = 0;
            for (uint32_t l = 0; l < c->n_clusters; ++l)
                max_len = std::max(max_len, c->dev_offsets[l + 1] - c->dev_offsets[l]);
            chunk = measure_chunk((uint64_t)n_probe * max_len, nq);
        }
        c->stage_n_probe = n_probe;
        try {
            for (uint32_t q0 = 0; q0 < nq || q0 == 0; q0 += chunk) {
                const uint32_t m = std::min(chunk, nq - q0);
                search_common(c, queries + (size_t)q0 * c->dim, m, c->dim, k, flags, out_ids + (size_t)q0 * k,
                              out_dists + (size_t)q0 * k, out_counts ? out_counts + q0 : nullptr, stats,
                              [&](const float* d_q, uint64_t* ok, uint32_t* oc) {
                                  ivf_search_device(c, d_q, m, k, n_probe, ok, oc);
                              },
                              ((uint64_t)n_probe << 8) | 1u);
                if (nq == 0) break;
            }
        } catch (...) {
            c->stage_n_probe = 0;
            throw;
        }
        c->stage_n_probe = 0;
    });
}

int dade_gpu_ivf_search_batches(dade_gpu_ctx* c, uint32_t n_batches, const float* const* queries, uint32_t nq,
                                uint32_t k, uint32_t n_probe, uint32_t flags, uint32_t* const* out_ids,
                                float* const* out_dists, uint32_t* const* out_counts, dade_gpu_stats* stats) {
    return guarded([&] {
        check_ivf_args(c, k, n_probe);
        if (flags & DADE_GPU_DEVICE_PTRS) fail(DADE_GPU_INVALID_INPUT, "ivf_search_batches: host buffers only");
        if (flags & DADE_GPU_MEASURE_FAILURES)
            fail(DADE_GPU_INVALID_INPUT, "ivf_search_batches: failure accounting is a separate dade_gpu_ivf_search pass");
        if (n_batches && nq && (!queries || !out_ids || !out_dists))
            fail(DADE_GPU_INVALID_INPUT, "ivf_search_batches: null argument");
        for (uint32_t b = 0; b < n_batches && nq; ++b)
            if (!queries[b] || !out_ids[b] || !out_dists[b]) fail(DADE_GPU_INVALID_INPUT, "ivf_search_batches: null batch");
        c->stage_n_probe = n_probe;
        try {
            search_batches(c, n_batches, queries, nq, c->dim, k, flags, out_ids, out_dists, out_counts, stats,
                           [&](const float* d_q, uint64_t* ok, uint32_t* oc) {
                               ivf_search_device(c, d_q, nq, k, n_probe, ok, oc);
                           },
                           ((uint64_t)n_probe << 8) | 1u);
        } catch (...) {
            c->stage_n_probe = 0;
            throw;
        }
        c->stage_n_probe = 0;
    });
}

int dade_gpu_flat_search(dade_gpu_ctx* c, const float* queries, uint32_t nq, uint32_t k, uint32_t flags,
                         uint32_t* out_ids, float* out_dists, uint32_t* out_counts, dade_gpu_stats* stats) {
    return guarded([&] {
        check_flat_args(c, k);
        if (nq && (!queries || !out_ids || !out_dists)) fail(DADE_GPU_INVALID_INPUT, "flat_search: null argument");
        const bool measure = flags & DADE_GPU_MEASURE_FAILURES;
        MeasureScope ms(c, measure);
        const uint32_t chunk = measure ? measure_chunk(c->b_count, nq) : nq;
        const uint32_t parts = c->flat_parts && c->has_ivf && c->dim == c->b_dim ? c->flat_parts : 0u;
        c->stage_n_probe = parts;  // data-ordered: the staging may coarse-rank query chunks
        c->coarse_all = parts != 0;
        try {
            for (uint32_t q0 = 0; q0 < nq || q0 == 0; q0 += chunk) {
                const uint32_t m = std::min(chunk, nq - q0);
                if (parts)  // every cell probed, nearest first: the IVF search over the partitioned base
                    search_common(c, queries + (size_t)q0 * c->b_dim, m, c->b_dim, k, flags, out_ids + (size_t)q0 * k,
                                  out_dists + (size_t)q0 * k, out_counts ? out_counts + q0 : nullptr, stats,
                                  [&](const float* d_q, uint64_t* ok, uint32_t* oc) {
                                      ivf_search_device(c, d_q, m, k, parts, ok, oc);
                                  },
                                  ((uint64_t)parts << 8) | 2u);
                else
                    search_common(c, queries + (size_t)q0 * c->b_dim, m, c->b_dim, k, flags, out_ids + (size_t)q0 * k,
                                  out_dists + (size_t)q0 * k, out_counts ? out_counts + q0 : nullptr, stats,
                                  [&](const float* d_q, uint64_t* ok, uint32_t* oc) {
                                      flat_search_device(c, d_q, m, k, ok, oc);
                                  });
                if (nq == 0) break;
            }
        } catch (...) {
            c->stage_n_probe = 0;
            c->coarse_all = false;
            throw;
        }
        c->stage_n_probe = 0;
        c->coarse_all = false;
    });
}

int dade_gpu_ivf_search_keys(dade_gpu_ctx* c, const float* d_queries, uint32_t nq, uint32_t k, uint32_t n_probe,
                             uint32_t flags, uint64_t* d_out_keys, dade_gpu_stats* stats) {
    return guarded([&] {
        check_ivf_args(c, k, n_probe);
        c->use_device();
        c->counters.ensure(kCounterBytes);
        cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, c->stream), "memset");
        if (nq == 0) return;
        const float* d_q = stage_queries(c, d_queries, nq, c->dim, flags | DADE_GPU_DEVICE_PTRS);
        c->out_count.ensure((size_t)nq * 4);
        for (int attempt = 0;; ++attempt) {
            c->surv_cap_used = 0;
            c->tl_on = env_flag("DADE_GPU_TIMELINE");
            c->tl_used = 0;
            tl_mark(c, "start", c->stream);
            ivf_search_device(c, d_q, nq, k, n_probe, d_out_keys, c->out_count.as<uint32_t>());
            tl_print(c);
            enqueue_flags(c);
            cuda_check(cudaStreamSynchronize(c->stream), "search");
            if (!search_overflowed(c)) break;
            if (attempt >= 2) fail(DADE_GPU_RUNTIME_ERROR, "survivor worklist overflow");
            cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, c->stream), "memset");
        }
        if (c->coarse_tc_used && c->h_flags[1]) {  // pathological coarse ties: all-exact ranking
            c->coarse_force_exact = true;
            cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, c->stream), "memset");
            ivf_search_device(c, d_q, nq, k, n_probe, d_out_keys, c->out_count.as<uint32_t>());
            c->coarse_force_exact = false;
        }
        collect_stats(c, stats);
    });
}

int dade_gpu_coarse_probes(dade_gpu_ctx* c, const float* d_queries, uint32_t nq, uint32_t n_probe, uint32_t flags,
                           float* d_q_rot, uint64_t* d_probes) {
    return guarded([&] {
        check_ivf_args(c, 1, n_probe);
        if (!(flags & DADE_GPU_DEVICE_PTRS)) fail(DADE_GPU_INVALID_INPUT, "coarse_probes: device pointers only");
        if (nq && (!d_queries || !d_probes)) fail(DADE_GPU_INVALID_INPUT, "coarse_probes: null argument");
        c->use_device();
        if (nq == 0) return;
        struct ExactKeys {  // this entry point's keys are exact l2_sq, ascending (dade_gpu.h)
            dade_gpu_ctx* c;
            ~ExactKeys() { c->coarse_exact_keys = false; }
        } exact_keys{c};
        c->coarse_exact_keys = true;
        const float* d_q = stage_queries(c, d_queries, nq, c->dim, flags);
        coarse_rank(c, d_q, nq, n_probe);
        if (c->coarse_tc_used) {  // boundary-candidate overflow (pathological ties): all-exact ranking
            enqueue_flags(c);
            cuda_check(cudaStreamSynchronize(c->stream), "coarse");
            if (c->h_flags[1]) {
                c->coarse_force_exact = true;
                try {
                    coarse_rank(c, d_q, nq, n_probe);
                } catch (...) {
                    c->coarse_force_exact = false;
                    throw;
                }
                c->coarse_force_exact = false;
            }
        }
        cuda_check(cudaMemcpyAsync(d_probes, c->probes.p, (size_t)nq * n_probe * 8, cudaMemcpyDeviceToDevice, c->stream),
                   "probes");
        if (d_q_rot && d_q_rot != d_q)
            cuda_check(cudaMemcpyAsync(d_q_rot, d_q, (size_t)nq * c->dim * 4, cudaMemcpyDeviceToDevice, c->stream),
                       "rotated queries");
    });
}

int dade_gpu_ivf_search_keys_begin(dade_gpu_ctx* c, const float* d_queries, uint32_t nq, uint32_t k,
                                   uint32_t n_probe, uint32_t flags, const uint64_t* d_probes,
                                   uint64_t* d_out_keys, uint32_t* d_radius) {
    return guarded([&] {
        check_ivf_args(c, k, n_probe);
        if (nq && (!d_queries || !d_out_keys || !d_radius)) fail(DADE_GPU_INVALID_INPUT, "search_keys_begin: null argument");
        if (d_probes && (flags & DADE_GPU_QUERIES_RAW))
            fail(DADE_GPU_INVALID_INPUT, "search_keys_begin: given probes need rotated queries");
        c->use_device();
        c->counters.ensure(kCounterBytes);
        cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, c->stream), "memset");
        c->sp.active = false;
        if (nq == 0) return;
        const float* d_q = stage_queries(c, d_queries, nq, c->dim, flags | DADE_GPU_DEVICE_PTRS);
        if (d_probes) {  // coarse ranking done elsewhere (dade_gpu_coarse_probes on the queries' owner)
            c->probes.ensure((size_t)nq * n_probe * 8);
            cuda_check(cudaMemcpyAsync(c->probes.p, d_probes, (size_t)nq * n_probe * 8, cudaMemcpyDeviceToDevice,
                                       c->stream),
                       "probes");
            c->probes_ready = true;
            c->coarse_tc_used = false;
        }
        c->out_count.ensure((size_t)nq * 4);
        c->surv_cap_used = 0;
        c->split = 1;
        try {
            ivf_search_device(c, d_q, nq, k, n_probe, d_out_keys, c->out_count.as<uint32_t>());
        } catch (...) {
            c->split = 0;
            throw;
        }
        c->split = 0;
        cuda_check(cudaMemcpyAsync(d_radius, c->r_global.p, (size_t)nq * 4, cudaMemcpyDeviceToDevice, c->stream),
                   "radius");
        c->sp.active = true;
        c->sp.flat = false;
        c->sp.d_q = d_q;
        c->sp.nq = nq;
        c->sp.k = k;
        c->sp.n_probe = n_probe;
        c->sp.keys = d_out_keys;
    });
}

int dade_gpu_flat_search_keys_begin(dade_gpu_ctx* c, const float* d_queries, uint32_t nq, uint32_t k, uint32_t flags,
                                    uint64_t* d_out_keys, uint32_t* d_radius) {
    return guarded([&] {
        check_flat_args(c, k);
        if (nq && (!d_queries || !d_out_keys || !d_radius)) fail(DADE_GPU_INVALID_INPUT, "search_keys_begin: null argument");
        c->use_device();
        c->counters.ensure(kCounterBytes);
        cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, c->stream), "memset");
        c->sp.active = false;
        if (nq == 0) return;
        const float* d_q = stage_queries(c, d_queries, nq, c->b_dim, flags | DADE_GPU_DEVICE_PTRS);
        c->out_count.ensure((size_t)nq * 4);
        c->surv_cap_used = 0;
        c->split = 1;
        try {
            flat_search_device(c, d_q, nq, k, d_out_keys, c->out_count.as<uint32_t>());
        } catch (...) {
            c->split = 0;
            throw;
        }
        c->split = 0;
        c->r_global.ensure((size_t)nq * 4);
        cuda_check(cudaMemcpyAsync(d_radius, c->r_global.p, (size_t)nq * 4, cudaMemcpyDeviceToDevice, c->stream),
                   "radius");
        c->sp.active = true;
        c->sp.flat = true;
        c->sp.d_q = d_q;
        c->sp.nq = nq;
        c->sp.k = k;
        c->sp.n_probe = 1;
        c->sp.keys = d_out_keys;
    });
}

int dade_gpu_ivf_search_keys_end(dade_gpu_ctx* c, const uint32_t* d_radius, dade_gpu_stats* stats) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        c->use_device();
        if (!c->sp.active) {
            collect_stats(c, stats);  // nq == 0 (or nothing begun): nothing to scan
            return;
        }
        c->sp.active = false;
        const uint32_t nq = c->sp.nq, k = c->sp.k, n_probe = c->sp.n_probe;
        if (d_radius) {
            min_u32_kernel<<<(nq + 255) / 256, 256, 0, c->stream>>>(c->r_global.as<uint32_t>(), d_radius, nq);
            cuda_check(cudaGetLastError(), "radius");
        }
        const bool flat = c->sp.flat;
        auto run = [&] {
            if (flat) flat_search_device(c, c->sp.d_q, nq, k, c->sp.keys, c->out_count.as<uint32_t>());
            else ivf_search_device(c, c->sp.d_q, nq, k, n_probe, c->sp.keys, c->out_count.as<uint32_t>());
        };
        c->split = 2;
        try {
            run();
        } catch (...) {
            c->split = 0;
            throw;
        }
        c->split = 0;
        enqueue_flags(c);
        cuda_check(cudaStreamSynchronize(c->stream), "search");
        // worklist overflow / coarse ties: this shard's search is redone whole and
        // locally (its answer is still this shard's exact top-K; only the shared
        // radius is not used again)
        for (int attempt = 0; search_overflowed(c) || (c->coarse_tc_used && c->h_flags[1]); ++attempt) {
            if (attempt >= 3) fail(DADE_GPU_RUNTIME_ERROR, "survivor worklist overflow");
            c->coarse_force_exact = c->coarse_tc_used && c->h_flags[1];
            cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, c->stream), "memset");
            c->surv_cap_used = 0;
            try {
                run();
            } catch (...) {
                c->coarse_force_exact = false;
                throw;
            }
            c->coarse_force_exact = false;
            enqueue_flags(c);
            cuda_check(cudaStreamSynchronize(c->stream), "search");
        }
        collect_stats(c, stats);
    });
}

int dade_gpu_flat_search_keys(dade_gpu_ctx* c, const float* d_queries, uint32_t nq, uint32_t k, uint32_t flags,
                              uint64_t* d_out_keys, dade_gpu_stats* stats) {
    return guarded([&] {
        check_flat_args(c, k);
        c->use_device();
        c->counters.ensure(kCounterBytes);
        cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, c->stream), "memset");
        if (nq == 0) return;
        const float* d_q = stage_queries(c, d_queries, nq, c->b_dim, flags | DADE_GPU_DEVICE_PTRS);
        c->out_count.ensure((size_t)nq * 4);
        flat_search_device(c, d_q, nq, k, d_out_keys, c->out_count.as<uint32_t>());
        collect_stats(c, stats);
    });
}

int dade_gpu_merge_keys(dade_gpu_ctx* c, const uint64_t* d_keys, uint32_t G, uint32_t nq, uint32_t k,
                        uint32_t* d_ids, float* d_dists, uint32_t* d_counts) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (k == 0) fail(DADE_GPU_INVALID_INPUT, "merge_keys: k must be positive");
        c->use_device();
        c->out_keys.ensure((size_t)nq * k * 8);
        c->out_count.ensure((size_t)nq * 4);
        cuda_check(launch_merge_blocks(d_keys, G, nq, k, c->out_keys.as<uint64_t>(), c->out_count.as<uint32_t>(),
                                       c->stream),
                   "merge_blocks");
        cuda_check(launch_keys_to_results(c->out_keys.as<uint64_t>(), c->out_count.as<uint32_t>(), nq, k, d_ids,
                                          d_dists, d_counts, c->stream),
                   "keys_to_results");
        c->launches += 2;
    });
}

int dade_gpu_dco_evaluate(dade_gpu_ctx* c, const float* o, const float* q, const float* r, uint32_t n,
                          uint32_t flags, uint8_t* pruned, float* distance, uint8_t* exact, uint32_t* dims_used,
                          dade_gpu_stats* stats) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (!c->has_strategy) fail(DADE_GPU_CONFIG_ERROR, "evaluate: no strategy set");
        c->use_device();
        const uint32_t dim = c->s_dim;
        cudaStream_t s = c->stream;
        c->counters.ensure(kCounterBytes);
        cuda_check(cudaMemsetAsync(c->counters.p, 0, kCounterBytes, s), "memset");
        if (n == 0) return;
        const bool dev = flags & DADE_GPU_DEVICE_PTRS;
        const size_t vb = (size_t)n * dim * 4;
        const float *d_o = o, *d_q = q, *d_r = r;
        uint8_t *d_p = pruned, *d_e = exact;
        float* d_d = distance;
        uint32_t* d_u = dims_used;
        DevBuf bo, bq, br, bp, bd, be, bu;
        if (!dev) {
            upload(bo, o, vb, s);
            upload(bq, q, vb, s);
            upload(br, r, (size_t)n * 4, s);
            d_o = bo.as<float>();
            d_q = bq.as<float>();
            d_r = br.as<float>();
            d_p = static_cast<uint8_t*>(bp.ensure(n));
            d_d = static_cast<float*>(bd.ensure((size_t)n * 4));
            d_e = static_cast<uint8_t*>(be.ensure(n));
            d_u = static_cast<uint32_t*>(bu.ensure((size_t)n * 4));
        }
        cuda_check(launch_evaluate(d_o, d_q, d_r, n, dim, c->d_cps.as<uint32_t>(), c->d_coeff.as<double>(),
                                   c->d_scale.as<double>(), (uint32_t)c->cps.size(), d_p, d_d, d_e, d_u,
                                   c->counters.as<unsigned long long>(), s),
                   "evaluate");
        ++c->launches;
        if (!dev) {
            cuda_check(cudaMemcpyAsync(pruned, d_p, n, cudaMemcpyDeviceToHost, s), "D2H");
            cuda_check(cudaMemcpyAsync(distance, d_d, (size_t)n * 4, cudaMemcpyDeviceToHost, s), "D2H");
            cuda_check(cudaMemcpyAsync(exact, d_e, n, cudaMemcpyDeviceToHost, s), "D2H");
            cuda_check(cudaMemcpyAsync(dims_used, d_u, (size_t)n * 4, cudaMemcpyDeviceToHost, s), "D2H");
        }
        unsigned long long h[4] = {0, 0, 0, 0};
        cuda_check(cudaMemcpyAsync(h, c->counters.p, sizeof(h), cudaMemcpyDeviceToHost, s), "D2H");
        cuda_check(cudaStreamSynchronize(s), "evaluate");
        if (stats) {
            stats->total_dco += h[0];
            stats->dims_accumulated += h[1];
            stats->eligible += h[2];
            stats->failures += h[3];
        }
        for (DevBuf* b : {&bo, &bq, &br, &bp, &bd, &be, &bu}) b->release();
    });
}

int dade_gpu_partial_sums(dade_gpu_ctx* c, const float* o, const float* q, uint32_t n, uint32_t flags, float* out) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (!c->has_strategy) fail(DADE_GPU_CONFIG_ERROR, "partial_sums: no strategy set");
        c->use_device();
        if (n == 0) return;
        const uint32_t dim = c->s_dim, nc = (uint32_t)c->cps.size();
        cudaStream_t s = c->stream;
        const size_t ob = (size_t)n * (nc + 1) * 4;
        if (flags & DADE_GPU_DEVICE_PTRS) {
            cuda_check(launch_partial_sums(o, q, n, dim, c->d_cps.as<uint32_t>(), nc, out, s), "partial_sums");
            ++c->launches;
            return;
        }
        DevBuf bo, bq, bout;
        upload(bo, o, (size_t)n * dim * 4, s);
        upload(bq, q, (size_t)n * dim * 4, s);
        bout.ensure(ob);
        cuda_check(launch_partial_sums(bo.as<float>(), bq.as<float>(), n, dim, c->d_cps.as<uint32_t>(), nc,
                                       bout.as<float>(), s),
                   "partial_sums");
        ++c->launches;
        cuda_check(cudaMemcpyAsync(out, bout.p, ob, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_check(cudaStreamSynchronize(s), "partial_sums");
        bo.release();
        bq.release();
        bout.release();
    });
}

// calibrate (proj/src/calibration.cpp:92-146): pairs drawn on the host with
// the reference's generator and rejection sampler (std::mt19937_64 +
// rng::bounded, proj/include/dade/rng.hpp:20-25), running partial sums on the
// GPU (bit-exact), ratios / order statistic / running min on the host.
int dade_gpu_calibrate(dade_gpu_ctx* c, const float* data, uint32_t n, double p_s, uint32_t delta_d,
                       uint64_t n_pairs, uint64_t seed, uint32_t flags, uint32_t* out_cps, double* out_eps,
                       uint32_t* n_out) {
    return guarded([&] {
        if (!c || !data || !n_out) fail(DADE_GPU_INVALID_INPUT, "calibrate: null argument");
        if (!(p_s > 0.0 && p_s < 1.0)) fail(DADE_GPU_INVALID_INPUT, "calibrate: p_s must be in (0, 1)");
        if (n_pairs == 0) fail(DADE_GPU_INVALID_INPUT, "calibrate: n_pairs must be positive");
        if (c->t_dim == 0) fail(DADE_GPU_CONFIG_ERROR, "calibrate: no transform set");
        if (delta_d == 0) fail(DADE_GPU_INVALID_INPUT, "delta_d must be positive");
        if (n < 2) fail(DADE_GPU_INVALID_INPUT, "sample_pairs: need at least 2 vectors");
        const uint32_t dim = c->t_dim;
        c->use_device();
        cudaStream_t s = c->stream;
        std::mt19937_64 gen(seed);
        auto bounded = [&](uint64_t m) {
            const uint64_t limit = (0 - m) % m;
            uint64_t r = gen();
            while (r < limit) r = gen();
            return r % m;
        };
        std::vector<uint32_t> pi(n_pairs), pj(n_pairs);
        for (uint64_t p = 0; p < n_pairs; ++p) {
            const uint32_t i = (uint32_t)bounded(n);
            uint32_t j = (uint32_t)bounded(n - 1);
            if (j >= i) ++j;
            pi[p] = i;
            pj[p] = j;
        }
        const auto cps = expected_checkpoints(dim, delta_d);
        const uint32_t nc = (uint32_t)cps.size();
        DevBuf bdata, bpi, bpj, bcps, bout;
        const float* d_data = data;
        if (!(flags & DADE_GPU_DEVICE_PTRS)) {
            upload(bdata, data, (size_t)n * dim * 4, s);
            d_data = bdata.as<float>();
        }
        upload(bpi, pi.data(), n_pairs * 4, s);
        upload(bpj, pj.data(), n_pairs * 4, s);
        upload(bcps, cps.data(), cps.size() * 4, s);
        bout.ensure(n_pairs * (nc + 1) * 4);
        cuda_check(launch_pair_partials(d_data, dim, bpi.as<uint32_t>(), bpj.as<uint32_t>(), n_pairs,
                                        bcps.as<uint32_t>(), nc, bout.as<float>(), s),
                   "pair_partials");
        ++c->launches;
        std::vector<float> part(n_pairs * (nc + 1));
        cuda_check(cudaMemcpyAsync(part.data(), bout.p, part.size() * 4, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_check(cudaStreamSynchronize(s), "calibrate");
        for (DevBuf* b : {&bdata, &bpi, &bpj, &bcps, &bout}) b->release();
        const auto& pre = c->lambda_prefix;
        std::vector<double> scale(nc);
        for (uint32_t ci = 0; ci < nc; ++ci) scale[ci] = pre[cps[ci]] <= 0.0 ? 1.0 : pre[dim] / pre[cps[ci]];
        std::vector<std::vector<double>> ratios(nc);
        for (auto& r : ratios) r.reserve(n_pairs);
        uint64_t skipped = 0;
        for (uint64_t p = 0; p < n_pairs; ++p) {
            const float* row = part.data() + p * (nc + 1);
            const float acc = row[nc];
            if (acc == 0.0f) {
                ++skipped;
                continue;
            }
            const double dis = std::sqrt(static_cast<double>(acc));
            for (uint32_t ci = 0; ci < nc; ++ci)
                ratios[ci].push_back(std::sqrt(scale[ci] * static_cast<double>(row[ci])) / dis - 1.0);
        }
        const uint64_t kept = n_pairs - skipped;
        if (nc > 0) {
            if (skipped * 2 > n_pairs)
                fail(DADE_GPU_RUNTIME_ERROR,
                     "calibrate: over half the sampled pairs are at zero distance; data is too degenerate to calibrate");
            if (kept == 0) fail(DADE_GPU_RUNTIME_ERROR, "calibrate: no usable pairs");
            const auto rank = static_cast<uint64_t>(std::ceil((1.0 - p_s) * static_cast<double>(kept)));
            for (uint32_t ci = 0; ci < nc; ++ci) {
                auto& r = ratios[ci];
                std::sort(r.begin(), r.end());
                out_eps[ci] = r[rank - 1];
            }
            for (uint32_t ci = 1; ci < nc; ++ci) out_eps[ci] = std::min(out_eps[ci], out_eps[ci - 1]);
        }
        for (uint32_t ci = 0; ci < nc; ++ci) out_cps[ci] = cps[ci];
        *n_out = nc;
    });
}

uint64_t dade_gpu_launch_count(dade_gpu_ctx* c) { return c ? c->launches : 0; }

// Debug: copy the per-query radius (float bits) left by the last IVF search.
int dade_gpu_debug_radius(dade_gpu_ctx* c, uint32_t* out, uint32_t nq) {
    return guarded([&] {
        c->use_device();
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        cuda_check(cudaMemcpy(out, c->r_global.p, (size_t)nq * 4, cudaMemcpyDeviceToHost), "D2H");
    });
}

// Debug: the last scan's counters [0..7] and per-phase clocks [8..15].
int dade_gpu_debug_counters(dade_gpu_ctx* c, uint64_t* out16) {
    return guarded([&] {
        if (!c || !out16) fail(DADE_GPU_INVALID_INPUT, "null argument");
        c->use_device();
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        std::memset(out16, 0, 16 * sizeof(uint64_t));
        if (c->counters.p) cuda_check(cudaMemcpy(out16, c->counters.p, kCounterBytes, cudaMemcpyDeviceToHost), "D2H");
    });
}

int dade_gpu_set_seed_rows(dade_gpu_ctx* c, uint32_t rows) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        c->seed_rows_set = rows;
        c->config_changed();
    });
}

int dade_gpu_set_graphs(dade_gpu_ctx* c, int on) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        c->graphs_on = on != 0;
    });
}

int dade_gpu_set_estimate_dump(dade_gpu_ctx* c, uint32_t capacity) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        c->use_device();
        c->dump_cap = capacity;
        if (!capacity) return;
        c->dump_entries.ensure((size_t)capacity * sizeof(uint4));
        c->dump_count.ensure(4);
        cuda_check(cudaMemsetAsync(c->dump_count.p, 0, 4, c->stream), "memset");
        cuda_check(cudaStreamSynchronize(c->stream), "dump");
    });
}

int dade_gpu_get_estimate_dump(dade_gpu_ctx* c, uint32_t cap, uint32_t* q, uint32_t* ids, uint32_t* dims,
                               float* partial, double* estimate, uint64_t* n_total) {
    return guarded([&] {
        if (!c || !n_total) fail(DADE_GPU_INVALID_INPUT, "get_estimate_dump: null argument");
        if (!c->dump_cap) fail(DADE_GPU_CONFIG_ERROR, "get_estimate_dump: dump not enabled");
        c->use_device();
        cuda_check(cudaStreamSynchronize(c->stream), "sync");
        uint32_t cnt = 0;
        cuda_check(cudaMemcpy(&cnt, c->dump_count.p, 4, cudaMemcpyDeviceToHost), "D2H");
        *n_total = cnt;
        const uint32_t n = std::min({cnt, c->dump_cap, cap});
        if (!n) return;
        if (!q || !ids || !dims || !partial || !estimate) fail(DADE_GPU_INVALID_INPUT, "get_estimate_dump: null output");
        std::vector<uint4> h(n);
        cuda_check(cudaMemcpy(h.data(), c->dump_entries.p, (size_t)n * sizeof(uint4), cudaMemcpyDeviceToHost), "D2H");
        for (uint32_t i = 0; i < n; ++i) {
            const uint32_t ci = h[i].z;
            if (ci >= c->cps.size()) fail(DADE_GPU_RUNTIME_ERROR, "get_estimate_dump: bad checkpoint index");
            q[i] = h[i].x;
            ids[i] = h[i].y;
            dims[i] = c->cps[ci];
            std::memcpy(&partial[i], &h[i].w, 4);
            // dade_estimate / adsampling_estimate (proj/src/estimator.cpp:84-97): est_scale x partial
            estimate[i] = c->scale[ci] * static_cast<double>(partial[i]);
        }
    });
}

int dade_gpu_set_profiling(dade_gpu_ctx* c, int on) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        c->profiling = on != 0;
    });
}

int dade_gpu_last_filter_profile(dade_gpu_ctx* c, double* filter_ms, int* n_launches) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (filter_ms) *filter_ms = c->last_filter_ms;
        if (n_launches) *n_launches = c->n_filter_passes;
    });
}

int dade_gpu_last_seed_profile(dade_gpu_ctx* c, double* seed_ms, double* pair_dims) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (seed_ms) *seed_ms = c->last_seed_ms;
        if (pair_dims) *pair_dims = c->last_seed_pair_dims;
    });
}

int dade_gpu_last_union_profile(dade_gpu_ctx* c, double* b_union, double* rows) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (b_union) *b_union = c->last_union_bytes;
        if (rows) *rows = c->last_union_rows;
    });
}

int dade_gpu_last_scan_profile(dade_gpu_ctx* c, double* scan_ms, double* scan_bytes, double* total_ms) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (scan_ms) *scan_ms = c->last_scan_ms;
        if (scan_bytes) *scan_bytes = c->last_bytes;
        if (total_ms) *total_ms = c->last_total_ms;
    });
}

// ---- index build ------------------------------------------------

// compute_covariance (proj/src/transform.cpp:68-95): mean [dim] and covariance
// [dim x dim] row-major into host arrays, bit-identical to the reference.
int dade_gpu_covariance(dade_gpu_ctx* c, const float* data, uint32_t n, uint32_t dim, uint32_t flags, double* mean,
                        double* cov) {
    return guarded([&] {
        if (!c || !data || !mean || !cov) fail(DADE_GPU_INVALID_INPUT, "compute_covariance: null argument");
        if (dim == 0) fail(DADE_GPU_INVALID_INPUT, "VectorSet: dim must be positive");
        if (n < 2) fail(DADE_GPU_INVALID_INPUT, "compute_covariance: need at least 2 vectors");
        c->use_device();
        cudaStream_t s = c->stream;
        DevBuf bx, bm, bc;
        const float* d_x = data;
        if (!(flags & DADE_GPU_DEVICE_PTRS)) {
            upload(bx, data, (size_t)n * dim * 4, s);
            d_x = bx.as<float>();
        }
        bm.ensure((size_t)dim * 8);
        bc.ensure((size_t)dim * dim * 8);
        cuda_check(launch_covariance(d_x, n, dim, bm.as<double>(), bc.as<double>(), s), "covariance");
        c->launches += 2;
        cuda_check(cudaMemcpyAsync(mean, bm.p, (size_t)dim * 8, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_check(cudaMemcpyAsync(cov, bc.p, (size_t)dim * dim * 8, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_check(cudaStreamSynchronize(s), "covariance");
    });
}

}  // extern "C"

namespace {

// kmeans (proj/src/ivf.cpp:24-143) on the context: centroids end in
// c->centroids ([n_clusters x dim]), assignments in `assign` (device, [n]).
// The context's IVF index is dropped (the coarse ranking machinery serves as
// the exact nearest-centroid assignment: (l2_sq, id) order = the reference's
// first strict minimum).
uint32_t kmeans_device(dade_gpu_ctx* c, const float* d_x, uint32_t n, uint32_t dim, uint32_t n_clusters,
                       uint32_t max_iters, uint64_t seed, DevBuf& assign) {
    cudaStream_t s = c->stream;
    c->has_ivf = false;
    c->sharded = false;
    c->flat_parts = 0;
    c->config_changed();
    c->dim = dim;
    c->n_clusters = n_clusters;
    c->centroids.ensure((size_t)n_clusters * dim * 4);
    float* cen = c->centroids.as<float>();
    // k-means++ seeding; the mt19937_64 stream is generated here (one draw per pick,
    // plus rejection-sampling spares)
    std::mt19937_64 gen(seed);
    const uint32_t n_raw = n_clusters + 64;
    std::vector<uint64_t> raw(n_raw);
    for (auto& r : raw) r = gen();
    DevBuf d_raw, rng, dist2, bsums, scratch;
    upload(d_raw, raw.data(), raw.size() * 8, s);
    rng.ensure(16);
    cuda_check(cudaMemsetAsync(rng.p, 0, 16, s), "memset");
    dist2.ensure((size_t)n * 8);
    bsums.ensure(kmpp_block_count(n) * 8);
    cuda_check(launch_kmpp_seed(d_x, n, dim, n_clusters, d_raw.as<uint64_t>(), n_raw, rng.as<uint32_t>(),
                                dist2.as<double>(), bsums.as<double>(), cen, nullptr, s),
               "k-means++ seeding");
    c->launches += 3 + 2ull * (n_clusters - 1);
    uint32_t h_rng[3] = {0, 0, 0};
    cuda_check(cudaMemcpyAsync(h_rng, rng.p, 12, cudaMemcpyDeviceToHost, s), "D2H");
    cuda_check(cudaStreamSynchronize(s), "k-means++ seeding");
    if (h_rng[1]) fail(DADE_GPU_RUNTIME_ERROR, "kmeans: random stream exhausted during seeding");
    dist2.release();
    // Lloyd iterations
    assign.ensure((size_t)n * 4);
    cuda_check(cudaMemsetAsync(assign.p, 0, (size_t)n * 4, s), "memset");  // assignments.assign(count, 0)
    DevBuf keys_in, keys_out, offs, temp, flag;
    keys_in.ensure((size_t)n * 8);
    keys_out.ensure((size_t)n * 8);
    offs.ensure(((size_t)n_clusters + 1) * 4);
    size_t temp_bytes = 0;
    cuda_check(launch_km_sort(nullptr, n, n_clusters, keys_in.as<uint64_t>(), keys_out.as<uint64_t>(), nullptr,
                              nullptr, &temp_bytes, s),
               "sort size");
    temp.ensure(temp_bytes);
    flag.ensure(4);
    scratch.ensure(16);
    std::vector<uint32_t> h_off(n_clusters + 1), counts(n_clusters);
    const uint32_t chunk = 1u << 20;  // rows per assignment launch (bounds the probe buffers)
    uint32_t iterations = 0;
    for (uint32_t iter = 1; iter <= max_iters; ++iter) {
        cuda_check(cudaMemsetAsync(flag.p, 0, 4, s), "memset");
        for (uint32_t r0 = 0; r0 < n; r0 += chunk) {
            const uint32_t m = std::min(chunk, n - r0);
            const float* rows = d_x + (size_t)r0 * dim;
            coarse_rank(c, rows, m, 1);
            if (c->coarse_tc_used) {  // boundary-candidate overflow (ties): all-exact ranking of this chunk
                enqueue_flags(c);
                cuda_check(cudaStreamSynchronize(s), "assign");
                if (c->h_flags[1]) {
                    c->coarse_force_exact = true;
                    try {
                        coarse_rank(c, rows, m, 1);
                    } catch (...) {
                        c->coarse_force_exact = false;
                        throw;
                    }
                    c->coarse_force_exact = false;
                }
            }
            cuda_check(launch_km_assign(c->probes.as<uint64_t>(), m, assign.as<uint32_t>() + r0, flag.as<uint32_t>(), s),
                       "assign");
            ++c->launches;
        }
        uint32_t changed = 0;
        cuda_check(cudaMemcpyAsync(&changed, flag.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_check(cudaStreamSynchronize(s), "assign");
        iterations = iter;
        if (!changed && iter > 1) break;
        // new centroids: members in ascending id order per cluster
        cuda_check(launch_km_sort(assign.as<uint32_t>(), n, n_clusters, keys_in.as<uint64_t>(),
                                  keys_out.as<uint64_t>(), offs.as<uint32_t>(), temp.p, &temp_bytes, s),
                   "sort");
        cuda_check(launch_km_sums(d_x, dim, keys_out.as<uint64_t>(), offs.as<uint32_t>(), n_clusters, cen, s),
                   "sums");
        c->launches += 4;
        cuda_check(cudaMemcpyAsync(h_off.data(), offs.p, h_off.size() * 4, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_check(cudaStreamSynchronize(s), "sums");
        for (uint32_t cl = 0; cl < n_clusters; ++cl) counts[cl] = h_off[cl + 1] - h_off[cl];
        // re-seed empties from the largest cluster's farthest member (ivf.cpp:111-130)
        for (uint32_t cl = 0; cl < n_clusters; ++cl) {
            if (counts[cl] != 0) continue;
            uint32_t largest = 0;
            for (uint32_t c2 = 1; c2 < n_clusters; ++c2)
                if (counts[c2] > counts[largest]) largest = c2;
            if (counts[largest] == 0) break;
            cuda_check(launch_km_reseed(d_x, n, dim, assign.as<uint32_t>(), largest, cl, cen,
                                        scratch.as<unsigned long long>(), s),
                       "reseed");
            c->launches += 3;
            --counts[largest];
            ++counts[cl];
        }
    }
    cuda_check(cudaStreamSynchronize(s), "kmeans");
    c->tm_centroids = TmapCache{};  // the centroid buffer's contents are final now
    return iterations;
}

void check_kmeans_args(uint32_t n, uint32_t dim, uint32_t n_clusters, uint32_t max_iters) {
    if (dim == 0) fail(DADE_GPU_INVALID_INPUT, "VectorSet: dim must be positive");
    if (n_clusters == 0 || n_clusters > n)
        fail(DADE_GPU_INVALID_INPUT, "kmeans: n_clusters must be in [1, count], got " + std::to_string(n_clusters));
    if (max_iters == 0) fail(DADE_GPU_INVALID_INPUT, "kmeans: max_iters must be positive");
}

}  // namespace

extern "C" {

int dade_gpu_kmeans(dade_gpu_ctx* c, const float* data, uint32_t n, uint32_t dim, uint32_t n_clusters,
                    uint32_t max_iters, uint64_t seed, uint32_t flags, float* centroids, uint32_t* assignments,
                    uint32_t* iterations) {
    return guarded([&] {
        if (!c || (n && !data)) fail(DADE_GPU_INVALID_INPUT, "kmeans: null argument");
        check_kmeans_args(n, dim, n_clusters, max_iters);
        c->use_device();
        cudaStream_t s = c->stream;
        DevBuf bx, assign;
        const float* d_x = data;
        if (!(flags & DADE_GPU_DEVICE_PTRS)) {
            upload(bx, data, (size_t)n * dim * 4, s);
            d_x = bx.as<float>();
        }
        const uint32_t it = kmeans_device(c, d_x, n, dim, n_clusters, max_iters, seed, assign);
        const cudaMemcpyKind kind = cudaMemcpyDefault;  // outputs: host or device memory (unified addressing)
        if (centroids)
            cuda_check(cudaMemcpyAsync(centroids, c->centroids.p, (size_t)n_clusters * dim * 4, kind, s), "copy");
        if (assignments) cuda_check(cudaMemcpyAsync(assignments, assign.p, (size_t)n * 4, kind, s), "copy");
        cuda_check(cudaStreamSynchronize(s), "kmeans");
        if (iterations) *iterations = it;
    });
}

// IvfIndex::build, contiguous layout (proj/src/ivf.cpp:145-192): k-means, posting
// lists in cluster order with ids ascending; the index is installed on the
// context and its DIVF arrays copied out (nullable outputs are skipped).
int dade_gpu_ivf_build(dade_gpu_ctx* c, const float* data, uint32_t n, uint32_t dim, uint32_t n_clusters,
                       uint32_t max_iters, uint64_t seed, uint32_t flags, float* centroids, uint32_t* offsets,
                       uint32_t* ids, float* storage) {
    return guarded([&] {
        if (!c || (n && !data)) fail(DADE_GPU_INVALID_INPUT, "ivf_build: null argument");
        check_kmeans_args(n, dim, n_clusters, max_iters);
        c->use_device();
        cudaStream_t s = c->stream;
        DevBuf bx, assign;
        const float* d_x = data;
        if (!(flags & DADE_GPU_DEVICE_PTRS)) {
            upload(bx, data, (size_t)n * dim * 4, s);
            d_x = bx.as<float>();
        }
        kmeans_device(c, d_x, n, dim, n_clusters, max_iters, seed, assign);
        DevBuf keys_in, keys_out, temp;
        keys_in.ensure((size_t)n * 8);
        keys_out.ensure((size_t)n * 8);
        c->offsets.ensure(((size_t)n_clusters + 1) * 4);
        size_t temp_bytes = 0;
        cuda_check(launch_km_sort(nullptr, n, n_clusters, keys_in.as<uint64_t>(), keys_out.as<uint64_t>(), nullptr,
                                  nullptr, &temp_bytes, s),
                   "sort size");
        temp.ensure(temp_bytes);
        cuda_check(launch_km_sort(assign.as<uint32_t>(), n, n_clusters, keys_in.as<uint64_t>(),
                                  keys_out.as<uint64_t>(), c->offsets.as<uint32_t>(), temp.p, &temp_bytes, s),
                   "sort");
        c->storage.ensure((size_t)n * dim * 4);
        c->ids.ensure((size_t)n * 4);
        cuda_check(launch_gather_rows(d_x, dim, keys_out.as<uint64_t>(), n, c->storage.as<float>(),
                                      c->ids.as<uint32_t>(), s),
                   "gather");
        c->launches += 4;
        c->h_offsets.assign(n_clusters + 1, 0);
        cuda_check(cudaMemcpyAsync(c->h_offsets.data(), c->offsets.p, ((size_t)n_clusters + 1) * 4,
                                   cudaMemcpyDeviceToHost, s),
                   "D2H");
        cuda_check(cudaStreamSynchronize(s), "ivf_build");
        c->dev_offsets = c->h_offsets;
        c->count = n;
        c->norms_storage.rows = nullptr;
        c->aug_storage.rows = nullptr;
        c->has_ivf = true;
        c->config_changed();
        const cudaMemcpyKind kind = cudaMemcpyDefault;  // outputs: host or device memory (unified addressing)
        if (centroids)
            cuda_check(cudaMemcpyAsync(centroids, c->centroids.p, (size_t)n_clusters * dim * 4, kind, s), "copy");
        if (offsets) cuda_check(cudaMemcpyAsync(offsets, c->offsets.p, ((size_t)n_clusters + 1) * 4, kind, s), "copy");
        if (ids) cuda_check(cudaMemcpyAsync(ids, c->ids.p, (size_t)n * 4, kind, s), "copy");
        if (storage) cuda_check(cudaMemcpyAsync(storage, c->storage.p, (size_t)n * dim * 4, kind, s), "copy");
        cuda_check(cudaStreamSynchronize(s), "ivf_build");
    });
}

int dade_gpu_flat_partition(dade_gpu_ctx* c, uint32_t n_parts, uint32_t max_iters, uint64_t seed) {
    return guarded([&] {
        if (!c) fail(DADE_GPU_INVALID_INPUT, "null handle");
        if (n_parts == 0) {
            c->flat_parts = 0;
            c->config_changed();
            return;
        }
        if (!c->has_base) fail(DADE_GPU_CONFIG_ERROR, "flat_partition: no base vectors uploaded");
        const int rc = dade_gpu_ivf_build(c, c->base.as<float>(), c->b_count, c->b_dim, n_parts, max_iters, seed,
                                          DADE_GPU_DEVICE_PTRS, nullptr, nullptr, nullptr, nullptr);
        if (rc != DADE_GPU_OK) fail(rc, g_last_error);
        if (c->b_id_base) {  // the cells hold row indices; the flat scan reports id_base + row
            std::vector<uint32_t> h(c->b_count);
            cuda_check(cudaMemcpy(h.data(), c->ids.p, (size_t)c->b_count * 4, cudaMemcpyDeviceToHost), "D2H ids");
            for (uint32_t& v : h) v += c->b_id_base;
            cuda_check(cudaMemcpy(c->ids.p, h.data(), (size_t)c->b_count * 4, cudaMemcpyHostToDevice), "H2D ids");
        }
        c->flat_parts = n_parts;
        c->config_changed();
    });
}

// compute_ground_truth (proj/src/dataset_io.cpp:101-135): per query the k
// nearest rows by (l2_sq_double, id). Strided samples of the base give each
// query a shrinking bound on its k-th distance (any k real rows bound it); the
// last pass scores every row in fp64 and keeps those within the bound, which
// holds the exact top-k; a per-query sort by (d^2, id) finishes.
int dade_gpu_ground_truth(dade_gpu_ctx* c, const float* base, uint32_t n, const float* queries, uint32_t nq,
                          uint32_t dim, uint32_t k, uint32_t flags, uint32_t* out_ids) {
    return guarded([&] {
        if (!c || (n && !base) || (nq && (!queries || !out_ids))) fail(DADE_GPU_INVALID_INPUT, "ground truth: null argument");
        if (dim == 0) fail(DADE_GPU_INVALID_INPUT, "VectorSet: dim must be positive");
        if (k == 0 || k > n) fail(DADE_GPU_INVALID_INPUT, "ground truth: k must be in [1, count], got " + std::to_string(k));
        if (k > 2048) fail(DADE_GPU_INVALID_INPUT, "ground truth: k above 2048 is not supported on the GPU");
        c->use_device();
        cudaStream_t s = c->stream;
        const bool dev = flags & DADE_GPU_DEVICE_PTRS;
        DevBuf bb, bq, bo;
        const float* d_b = base;
        const float* d_q = queries;
        if (!dev) {
            upload(bb, base, (size_t)n * dim * 4, s);
            d_b = bb.as<float>();
        }
        uint32_t cap = 4096;
        while (cap < 8 * k) cap <<= 1;
        // level strides: powers of `ratio`, so each level's sample (rows 0, s, 2s, ...) holds the
        // previous one; level 0 has between k and k * ratio rows (all kept: bound = +inf)
        const uint32_t ratio = std::max<uint32_t>(2, cap / (4 * k));
        uint64_t st = 1;
        while (st * ratio <= n / k) st *= ratio;
        std::vector<uint32_t> strides;
        for (;; st /= ratio) {
            strides.push_back((uint32_t)st);
            if (st == 1) break;
        }
        const uint32_t chunk = std::max<uint32_t>(64, std::min<uint32_t>(nq, (uint32_t)((1ull << 30) / (cap * 12ull))));
        DevBuf thr, cnt, cd, ci, ov;
        thr.ensure((size_t)chunk * 8);
        cnt.ensure((size_t)chunk * 4);
        cd.ensure((size_t)chunk * cap * 8);
        ci.ensure((size_t)chunk * cap * 4);
        ov.ensure(4);
        for (uint32_t q0 = 0; q0 < nq; q0 += chunk) {
            const uint32_t m = std::min(chunk, nq - q0);
            const float* qc = d_q;
            if (!dev) {
                upload(bq, queries + (size_t)q0 * dim, (size_t)m * dim * 4, s);
                qc = bq.as<float>();
            } else {
                qc = queries + (size_t)q0 * dim;
            }
            {  // +inf bounds for level 0
                std::vector<double> inf(m, std::numeric_limits<double>::infinity());
                cuda_check(cudaMemcpyAsync(thr.p, inf.data(), (size_t)m * 8, cudaMemcpyHostToDevice, s), "H2D");
                cuda_check(cudaStreamSynchronize(s), "thr");
            }
            uint32_t* ids_out = dev ? out_ids + (size_t)q0 * k : nullptr;
            if (!dev) ids_out = static_cast<uint32_t*>(bo.ensure((size_t)m * k * 4));
            for (size_t lv = 0; lv < strides.size(); ++lv) {
                const bool last = lv + 1 == strides.size();
                for (int attempt = 0;; ++attempt) {
                    cuda_check(cudaMemsetAsync(cnt.p, 0, (size_t)m * 4, s), "memset");
                    cuda_check(cudaMemsetAsync(ov.p, 0, 4, s), "memset");
                    cuda_check(launch_gt_scan(d_b, n, strides[lv], qc, m, dim, thr.as<double>(), cap, cnt.as<uint32_t>(),
                                              cd.as<double>(), ci.as<uint32_t>(), c->n_sms, s),
                               "gt scan");
                    // the k-th smallest kept distance bounds each query's k-th distance
                    cuda_check(launch_gt_select(cnt.as<uint32_t>(), cap, cd.as<double>(), ci.as<uint32_t>(), m, k,
                                                last ? ids_out : nullptr, thr.as<double>(), ov.as<uint32_t>(), s),
                               "gt select");
                    c->launches += 2;
                    if (!last) break;
                    uint32_t h_ov = 0;
                    cuda_check(cudaMemcpyAsync(&h_ov, ov.p, 4, cudaMemcpyDeviceToHost, s), "D2H");
                    cuda_check(cudaStreamSynchronize(s), "gt");
                    if (!h_ov) break;  // every query kept all its candidates: exact
                    // some query had more than cap rows within its bound: rescan with the
                    // (tighter) k-th of the kept ones
                    if (attempt >= 4)
                        fail(DADE_GPU_RUNTIME_ERROR, "ground truth: more than " + std::to_string(cap) +
                                                         " rows tie at a query's k-th distance");
                }
            }
            if (!dev)
                cuda_check(cudaMemcpyAsync(out_ids + (size_t)q0 * k, ids_out, (size_t)m * k * 4, cudaMemcpyDeviceToHost, s),
                           "D2H");
        }
        cuda_check(cudaStreamSynchronize(s), "ground truth");
    });
}

}  // extern "C"

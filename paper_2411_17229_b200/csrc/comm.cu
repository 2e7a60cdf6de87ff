// Multi-GPU search over NCCL from the C ABI (SURVEY.md §8b "init_nccl(comm) /
// sharded_*", §8e): one process (or host thread) per GPU, one dade_gpu_ctx and
// one NCCL communicator per GPU. The protocols are the list-sharded
// query-owner scheme of IvfIndex::search and the row-sharded linear_scan,
// written on top of the exported single-GPU entry points plus NCCL
// collectives on the context's stream:
//
//   IVF (each rank owns nq of the job's queries and a shard of the lists):
//     coarse_probes (own queries) -> ncclAllGather(rotated queries, probes)
//     -> ivf_search_keys_begin (nearest lists: seed) -> ncclAllReduce(MIN,
//     radius) -> ivf_search_keys_end -> all-to-all of the top-K key blocks to
//     the queries' owners (ncclSend/ncclRecv in a group) -> merge_keys.
//   flat (queries replicated, rows sharded with id_base):
//     flat_search_keys_begin -> ncclAllReduce(MIN, radius) -> keys_end ->
//     ncclAllGather(keys) -> merge_keys.
//
// libnccl is resolved at run time (dlopen): the copy already mapped into the
// process (e.g. PyTorch's) when there is one, else libnccl.so.2 on the loader
// path, so the communicator's library is the one the caller's unique id came
// from. NCCL's own headers give the types.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "../../include/dade_gpu.h"

namespace dade_gpu {
void set_last_error(const std::string& msg);  // capi.cu
}

namespace {

struct NcclApi {
    void* h = nullptr;
    decltype(&ncclGetUniqueId) getUniqueId = nullptr;
    decltype(&ncclCommInitRank) commInitRank = nullptr;
    decltype(&ncclCommDestroy) commDestroy = nullptr;
    decltype(&ncclAllGather) allGather = nullptr;
    decltype(&ncclAllReduce) allReduce = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) groupStart = nullptr;
    decltype(&ncclGroupEnd) groupEnd = nullptr;
    decltype(&ncclGetErrorString) errorString = nullptr;
    std::string err;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the process's copy first
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("libnccl.so.2 not found: ") + dlerror();
            return;
        }
        api.h = h;
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            if (!fn && api.err.empty()) api.err = std::string("libnccl lacks ") + name;
        };
        sym(api.getUniqueId, "ncclGetUniqueId");
        sym(api.commInitRank, "ncclCommInitRank");
        sym(api.commDestroy, "ncclCommDestroy");
        sym(api.allGather, "ncclAllGather");
        sym(api.allReduce, "ncclAllReduce");
        sym(api.send, "ncclSend");
        sym(api.recv, "ncclRecv");
        sym(api.groupStart, "ncclGroupStart");
        sym(api.groupEnd, "ncclGroupEnd");
        sym(api.errorString, "ncclGetErrorString");
    });
    return api;
}

struct CommError : std::runtime_error {
    int code;
    CommError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw CommError(DADE_GPU_RUNTIME_ERROR,
                        std::string(what) + ": " + (nccl().errorString ? nccl().errorString(r) : "nccl error"));
}
void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CommError(DADE_GPU_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}
void abi_ok(int rc) {
    if (rc != DADE_GPU_OK) throw CommError(rc, dade_gpu_last_error());
}

template <class F>
int comm_guarded(F&& f) {
    try {
        f();
        return DADE_GPU_OK;
    } catch (const CommError& e) {
        dade_gpu::set_last_error(e.what());  // dade_gpu_last_error()
        return e.code;
    } catch (const std::exception& e) {
        dade_gpu::set_last_error(e.what());
        return DADE_GPU_RUNTIME_ERROR;
    }
}

struct Buf {
    void* p = nullptr;
    size_t cap = 0;
    void* get(size_t bytes) {
        if (bytes > cap) {
            if (p) cudaFree(p);
            p = nullptr;
            cap = 0;
            cuda_ok(cudaMalloc(&p, bytes ? bytes : 256), "cudaMalloc");
            cap = bytes ? bytes : 256;
        }
        return p;
    }
    ~Buf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

struct dade_gpu_comm {
    dade_gpu_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
    Buf q_in, q_rot, probes, q_all, p_all, keys, radius, recv, ids, dists, counts;
};

namespace {

cudaStream_t ctx_stream(dade_gpu_comm* c) {
    void* s = nullptr;
    abi_ok(dade_gpu_get_stream(c->ctx, &s));
    return static_cast<cudaStream_t>(s);
}

// device copy of host (or device) input rows
const float* stage_in(dade_gpu_comm* c, const float* rows, size_t bytes, uint32_t flags, cudaStream_t s) {
    if (flags & DADE_GPU_DEVICE_PTRS) return rows;
    float* d = static_cast<float*>(c->q_in.get(bytes));
    cuda_ok(cudaMemcpyAsync(d, rows, bytes, cudaMemcpyHostToDevice, s), "H2D queries");
    return d;
}

void results_out(dade_gpu_comm* c, uint32_t nq, uint32_t k, uint32_t flags, uint32_t* ids, float* dists,
                 uint32_t* counts, const uint32_t* d_ids, const float* d_dists, const uint32_t* d_counts,
                 cudaStream_t s) {
    (void)c;
    const cudaMemcpyKind kind = (flags & DADE_GPU_DEVICE_PTRS) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (ids != d_ids) cuda_ok(cudaMemcpyAsync(ids, d_ids, (size_t)nq * k * 4, kind, s), "results");
    if (dists != d_dists) cuda_ok(cudaMemcpyAsync(dists, d_dists, (size_t)nq * k * 4, kind, s), "results");
    if (counts && counts != d_counts) cuda_ok(cudaMemcpyAsync(counts, d_counts, (size_t)nq * 4, kind, s), "results");
    cuda_ok(cudaStreamSynchronize(s), "results");
}

}  // namespace

extern "C" {

int dade_gpu_nccl_unique_id(uint8_t* id_out) {
    return comm_guarded([&] {
        if (!id_out) throw CommError(DADE_GPU_INVALID_INPUT, "nccl_unique_id: null argument");
        NcclApi& api = nccl();
        if (!api.err.empty()) throw CommError(DADE_GPU_RUNTIME_ERROR, api.err);
        ncclUniqueId id;
        nccl_check(api.getUniqueId(&id), "ncclGetUniqueId");
        static_assert(sizeof(ncclUniqueId) == DADE_GPU_NCCL_ID_BYTES, "ncclUniqueId size");
        std::memcpy(id_out, &id, sizeof id);
    });
}

int dade_gpu_comm_create(dade_gpu_ctx* ctx, int nranks, int rank, const uint8_t* id, dade_gpu_comm** out) {
    return comm_guarded([&] {
        if (!ctx || !id || !out) throw CommError(DADE_GPU_INVALID_INPUT, "comm_create: null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) throw CommError(DADE_GPU_INVALID_INPUT, "comm_create: bad rank");
        NcclApi& api = nccl();
        if (!api.err.empty()) throw CommError(DADE_GPU_RUNTIME_ERROR, api.err);
        auto* c = new dade_gpu_comm;
        c->ctx = ctx;
        c->nranks = nranks;
        c->rank = rank;
        abi_ok(dade_gpu_synchronize(ctx));  // (makes the context's device current)
        cuda_ok(cudaGetDevice(&c->device), "cudaGetDevice");
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        const ncclResult_t r = api.commInitRank(&c->comm, nranks, uid, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

int dade_gpu_comm_destroy(dade_gpu_comm* c) {
    return comm_guarded([&] {
        if (!c) return;
        cudaSetDevice(c->device);
        if (c->comm) nccl().commDestroy(c->comm);
        delete c;
    });
}

int dade_gpu_sharded_ivf_search(dade_gpu_comm* c, const float* queries, uint32_t nq, uint32_t k, uint32_t n_probe,
                                uint32_t flags, uint32_t* out_ids, float* out_dists, uint32_t* out_counts,
                                dade_gpu_stats* stats) {
    return comm_guarded([&] {
        if (!c) throw CommError(DADE_GPU_INVALID_INPUT, "null comm");
        if (nq && (!queries || !out_ids || !out_dists))
            throw CommError(DADE_GPU_INVALID_INPUT, "sharded_ivf_search: null argument");
        if (k == 0) throw CommError(DADE_GPU_INVALID_INPUT, "IvfIndex::search: k must be positive");
        NcclApi& api = nccl();
        cudaSetDevice(c->device);
        cudaStream_t s = ctx_stream(c);
        uint32_t dim = 0;
        abi_ok(dade_gpu_index_dims(c->ctx, &dim, nullptr));
        const uint32_t G = (uint32_t)c->nranks, n_all = G * nq;
        const float* d_q = stage_in(c, queries, (size_t)nq * dim * 4, flags, s);
        float* q_rot = static_cast<float*>(c->q_rot.get((size_t)nq * dim * 4));
        uint64_t* probes = static_cast<uint64_t*>(c->probes.get((size_t)nq * n_probe * 8));
        // 1. rotation + coarse ranking of this rank's queries
        abi_ok(dade_gpu_coarse_probes(c->ctx, d_q, nq, n_probe, DADE_GPU_DEVICE_PTRS | (flags & DADE_GPU_QUERIES_RAW),
                                      q_rot, probes));
        // 2. all-gather rotated queries and probe keys (rank-major)
        float* q_all = static_cast<float*>(c->q_all.get((size_t)n_all * dim * 4));
        uint64_t* p_all = static_cast<uint64_t*>(c->p_all.get((size_t)n_all * n_probe * 8));
        nccl_check(api.groupStart(), "ncclGroupStart");
        nccl_check(api.allGather(q_rot, q_all, (size_t)nq * dim, ncclFloat32, c->comm, s), "ncclAllGather");
        nccl_check(api.allGather(probes, p_all, (size_t)nq * n_probe, ncclUint64, c->comm, s), "ncclAllGather");
        nccl_check(api.groupEnd(), "ncclGroupEnd");
        // 3. phase 1 over the job's queries, MIN of the radius (fp32 bits of d >= 0 order as int32)
        uint64_t* keys = static_cast<uint64_t*>(c->keys.get((size_t)n_all * k * 8));
        uint32_t* radius = static_cast<uint32_t*>(c->radius.get((size_t)n_all * 4));
        abi_ok(dade_gpu_ivf_search_keys_begin(c->ctx, q_all, n_all, k, n_probe, DADE_GPU_DEVICE_PTRS, p_all, keys,
                                              radius));
        nccl_check(api.allReduce(radius, radius, n_all, ncclInt32, ncclMin, c->comm, s), "ncclAllReduce");
        // 4. phase 2
        dade_gpu_stats st{};
        abi_ok(dade_gpu_ivf_search_keys_end(c->ctx, radius, &st));
        // 5. each query's key block to its owner, merge
        uint64_t* recv = static_cast<uint64_t*>(c->recv.get((size_t)G * nq * k * 8));
        nccl_check(api.groupStart(), "ncclGroupStart");
        for (uint32_t j = 0; j < G; ++j) {
            nccl_check(api.send(keys + (size_t)j * nq * k, (size_t)nq * k, ncclUint64, (int)j, c->comm, s), "ncclSend");
            nccl_check(api.recv(recv + (size_t)j * nq * k, (size_t)nq * k, ncclUint64, (int)j, c->comm, s), "ncclRecv");
        }
        nccl_check(api.groupEnd(), "ncclGroupEnd");
        const bool dev = flags & DADE_GPU_DEVICE_PTRS;
        uint32_t* d_ids = dev ? out_ids : static_cast<uint32_t*>(c->ids.get((size_t)nq * k * 4));
        float* d_dists = dev ? out_dists : static_cast<float*>(c->dists.get((size_t)nq * k * 4));
        uint32_t* d_counts = dev && out_counts ? out_counts : static_cast<uint32_t*>(c->counts.get((size_t)nq * 4));
        abi_ok(dade_gpu_merge_keys(c->ctx, recv, G, nq, k, d_ids, d_dists, d_counts));
        results_out(c, nq, k, flags, out_ids, out_dists, out_counts, d_ids, d_dists, d_counts, s);
        if (stats) {
            stats->total_dco += st.total_dco;
            stats->dims_accumulated += st.dims_accumulated;
        }
    });
}

int dade_gpu_sharded_flat_search(dade_gpu_comm* c, const float* queries, uint32_t nq, uint32_t k, uint32_t flags,
                                 uint32_t* out_ids, float* out_dists, uint32_t* out_counts, dade_gpu_stats* stats) {
    return comm_guarded([&] {
        if (!c) throw CommError(DADE_GPU_INVALID_INPUT, "null comm");
        if (nq && (!queries || !out_ids || !out_dists))
            throw CommError(DADE_GPU_INVALID_INPUT, "sharded_flat_search: null argument");
        if (k == 0) throw CommError(DADE_GPU_INVALID_INPUT, "linear_scan: k must be positive");
        NcclApi& api = nccl();
        cudaSetDevice(c->device);
        cudaStream_t s = ctx_stream(c);
        uint32_t dim = 0;
        abi_ok(dade_gpu_index_dims(c->ctx, nullptr, &dim));
        const uint32_t G = (uint32_t)c->nranks;
        const float* d_q = stage_in(c, queries, (size_t)nq * dim * 4, flags, s);
        uint64_t* keys = static_cast<uint64_t*>(c->keys.get((size_t)nq * k * 8));
        uint32_t* radius = static_cast<uint32_t*>(c->radius.get((size_t)nq * 4));
        abi_ok(dade_gpu_flat_search_keys_begin(c->ctx, d_q, nq, k, DADE_GPU_DEVICE_PTRS | (flags & DADE_GPU_QUERIES_RAW),
                                               keys, radius));
        nccl_check(api.allReduce(radius, radius, nq, ncclInt32, ncclMin, c->comm, s), "ncclAllReduce");
        dade_gpu_stats st{};
        abi_ok(dade_gpu_ivf_search_keys_end(c->ctx, radius, &st));
        uint64_t* all = static_cast<uint64_t*>(c->recv.get((size_t)G * nq * k * 8));
        nccl_check(api.allGather(keys, all, (size_t)nq * k, ncclUint64, c->comm, s), "ncclAllGather");
        const bool dev = flags & DADE_GPU_DEVICE_PTRS;
        uint32_t* d_ids = dev ? out_ids : static_cast<uint32_t*>(c->ids.get((size_t)nq * k * 4));
        float* d_dists = dev ? out_dists : static_cast<float*>(c->dists.get((size_t)nq * k * 4));
        uint32_t* d_counts = dev && out_counts ? out_counts : static_cast<uint32_t*>(c->counts.get((size_t)nq * 4));
        abi_ok(dade_gpu_merge_keys(c->ctx, all, G, nq, k, d_ids, d_dists, d_counts));
        results_out(c, nq, k, flags, out_ids, out_dists, out_counts, d_ids, d_dists, d_counts, s);
        if (stats) {
            stats->total_dco += st.total_dco;
            stats->dims_accumulated += st.dims_accumulated;
        }
    });
}

}  // extern "C"

// dade_gpu.hpp — C++ mirror of the reference's search API over the C ABI.
//
// A C++ user of the reference (proj/include/dade/*.hpp) switches to the GPU
// path by replacing `dade::` types with `dade::gpu::` ones:
//
//   reference                                   this header
//   dade::OrthoTransform::load(path)            dade::gpu::OrthoTransform::load(path)
//   dade::CalibrationTable::load(path)          dade::gpu::CalibrationTable::load(path)
//   dade::IvfIndex::load(path)                  dade::gpu::IvfIndex::load(dev, path)
//   dade::DadeStrategy(t, cal, delta_d)         dade::gpu::DadeStrategy(dev, t, cal, delta_d)
//   dade::AdsamplingStrategy(dim, dd, eps0)     dade::gpu::AdsamplingStrategy(dev, dim, dd, eps0)
//   dade::FdScanningStrategy(dim)               dade::gpu::FdScanningStrategy(dim)
//   idx.search(q, k, n_probe, dco, &stats)      idx.search(q, k, n_probe, dco, &stats)
//   (one query per call)                        idx.search_batch(qs, nq, k, n_probe, dco, &stats)
//   linear_scan(data, q, k, dco, &stats)        dade::gpu::FlatIndex(dev, data).search(q, k, dco, &stats)
//
// Semantics follow the reference: results ascending by (distance, id),
// `truncated` when fewer than k were found, DcoStats accumulate, the same
// argument checks raising dade::gpu::InvalidInput / ConfigError, file format
// errors raising std::runtime_error (proj/include/dade/error.hpp:10-19,
// proj/docs/FILE_FORMATS.md). Header-only; link libdade_gpu.so.
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <limits>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dade_gpu.h"

namespace dade {
namespace gpu {

class ConfigError : public std::runtime_error {
public:
    explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
class InvalidInput : public std::invalid_argument {
public:
    explicit InvalidInput(const std::string& w) : std::invalid_argument(w) {}
};
class CudaError : public std::runtime_error {
public:
    explicit CudaError(const std::string& w) : std::runtime_error(w) {}
};

inline void check(int rc) {
    if (rc == DADE_GPU_OK) return;
    const std::string msg = dade_gpu_last_error();
    switch (rc) {
        case DADE_GPU_CONFIG_ERROR: throw ConfigError(msg);
        case DADE_GPU_INVALID_INPUT: throw InvalidInput(msg);
        case DADE_GPU_CUDA_ERROR: throw CudaError(msg);
        default: throw std::runtime_error(msg);
    }
}

struct Neighbor {
    float distance = 0.0f;
    std::uint32_t id = 0;
};
inline bool operator<(const Neighbor& a, const Neighbor& b) {
    if (a.distance != b.distance) return a.distance < b.distance;
    return a.id < b.id;
}

struct SearchResult {
    std::vector<Neighbor> neighbors;  // ascending (distance, id)
    bool truncated = false;
    std::vector<std::uint32_t> ids() const {
        std::vector<std::uint32_t> out;
        out.reserve(neighbors.size());
        for (const auto& n : neighbors) out.push_back(n.id);
        return out;
    }
};

struct DcoStats {
    std::uint64_t total_dco = 0;
    std::uint64_t dims_accumulated = 0;
    bool measure_failures = false;
    std::uint64_t eligible = 0;
    std::uint64_t failures = 0;
    void add(const dade_gpu_stats& s) {
        total_dco += s.total_dco;
        dims_accumulated += s.dims_accumulated;
        if (measure_failures) {
            eligible += s.eligible;
            failures += s.failures;
        }
    }
    double dim_fraction(std::uint32_t dim) const {
        return total_dco == 0 ? 0.0 : double(dims_accumulated) / (double(total_dco) * double(dim));
    }
    double failure_rate() const { return eligible == 0 ? 0.0 : double(failures) / double(eligible); }
};

namespace detail {
template <class T>
T read_pod(std::istream& in, const char* what) {
    T v{};
    in.read(reinterpret_cast<char*>(&v), sizeof v);
    if (!in) throw std::runtime_error(std::string("truncated file while reading ") + what);
    return v;
}
template <class T>
std::vector<T> read_vec(std::istream& in, std::size_t n, const char* what) {
    std::vector<T> v(n);
    in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(n * sizeof(T)));
    if (!in) throw std::runtime_error(std::string("truncated file while reading ") + what);
    return v;
}
inline std::ifstream open_in(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open for reading: " + path);
    return in;
}
}  // namespace detail

// One GPU context; owns the device copies of the artifacts.
class Device {
public:
    explicit Device(int device = 0) { check(dade_gpu_create(device, &ctx_)); }
    ~Device() {
        if (ctx_) dade_gpu_destroy(ctx_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    dade_gpu_ctx* get() const { return ctx_; }
    mutable const void* active_strategy = nullptr;

private:
    dade_gpu_ctx* ctx_ = nullptr;
};

// proj/include/dade/transform.hpp:42-64 (DADE file: proj/src/transform.cpp:306-358)
struct OrthoTransform {
    std::uint32_t dim = 0;
    std::uint8_t kind = 0;
    std::vector<double> mean, eigenvalues, matrix;

    static OrthoTransform load(const std::string& path) {
        auto in = detail::open_in(path);
        char magic[4];
        in.read(magic, 4);
        if (!in || std::memcmp(magic, "DADE", 4) != 0) throw std::runtime_error("not a transform file: " + path);
        if (detail::read_pod<std::uint32_t>(in, "version") != 1) throw std::runtime_error("unsupported transform version");
        OrthoTransform t;
        t.kind = detail::read_pod<std::uint8_t>(in, "kind");
        if (t.kind > 1) throw std::runtime_error("bad transform kind byte");
        t.dim = detail::read_pod<std::uint32_t>(in, "dim");
        if (t.dim == 0) throw std::runtime_error("transform dim is zero");
        t.mean = detail::read_vec<double>(in, t.dim, "mean");
        t.eigenvalues = detail::read_vec<double>(in, t.dim, "eigenvalues");
        t.matrix = detail::read_vec<double>(in, std::size_t(t.dim) * t.dim, "matrix");
        for (std::uint32_t k = 0; k + 1 < t.dim; ++k)
            if (t.eigenvalues[k] < t.eigenvalues[k + 1])
                throw std::runtime_error("transform eigenvalues not nonincreasing");
        // the loader's corruption check (proj/src/transform.cpp:344-356): columns orthonormal
        double worst = 0.0;
        for (std::uint32_t a = 0; a < t.dim; ++a)
            for (std::uint32_t b = a; b < t.dim; ++b) {
                double dot = 0.0;
                const double* ca = t.matrix.data() + std::size_t(a) * t.dim;
                const double* cb = t.matrix.data() + std::size_t(b) * t.dim;
                for (std::uint32_t r = 0; r < t.dim; ++r) dot += ca[r] * cb[r];
                worst = std::max(worst, std::abs(dot - (a == b ? 1.0 : 0.0)));
            }
        if (worst > 1e-5)
            throw std::runtime_error("transform matrix not orthogonal (max deviation " + std::to_string(worst) + ")");
        return t;
    }
    void upload(const Device& d) const {
        check(dade_gpu_set_transform(d.get(), dim, matrix.data(), eigenvalues.data()));
    }
    // apply_transform (proj/src/transform.cpp:295-304), on the GPU
    std::vector<float> apply(const Device& d, const float* rows, std::uint32_t n) const {
        upload(d);
        std::vector<float> out(std::size_t(n) * dim);
        check(dade_gpu_rotate(d.get(), rows, n, out.data(), 0));
        return out;
    }
};

// proj/include/dade/calibration.hpp:20-40 (.cal: proj/src/calibration.cpp:184-212)
struct CalibrationTable {
    double p_s = 0.0;
    std::uint32_t delta_d = 0;
    std::vector<std::uint32_t> checkpoints;
    std::vector<double> epsilons;

    static std::vector<std::uint32_t> expected_checkpoints(std::uint32_t dim, std::uint32_t delta_d) {
        if (delta_d == 0) throw InvalidInput("delta_d must be positive");
        std::vector<std::uint32_t> c;
        for (std::uint64_t d = delta_d; d + 1 <= dim && d < dim; d += delta_d) c.push_back(std::uint32_t(d));
        return c;
    }
    static CalibrationTable unbounded(std::uint32_t dim, std::uint32_t delta_d) {
        CalibrationTable c;
        c.delta_d = delta_d;
        c.checkpoints = expected_checkpoints(dim, delta_d);
        c.epsilons.assign(c.checkpoints.size(), std::numeric_limits<double>::infinity());
        return c;
    }
    static CalibrationTable load(const std::string& path) {
        auto in = detail::open_in(path);
        CalibrationTable c;
        c.p_s = detail::read_pod<double>(in, "p_s");
        c.delta_d = detail::read_pod<std::uint32_t>(in, "delta_d");
        const auto n = detail::read_pod<std::uint32_t>(in, "checkpoint count");
        for (std::uint32_t i = 0; i < n; ++i) {
            c.checkpoints.push_back(detail::read_pod<std::uint32_t>(in, "checkpoint"));
            c.epsilons.push_back(detail::read_pod<double>(in, "epsilon"));
        }
        for (std::uint32_t i = 0; i + 1 < n; ++i)
            if (c.checkpoints[i] >= c.checkpoints[i + 1]) throw std::runtime_error("calibration checkpoints not ascending");
        return c;
    }
    // calibrate (proj/src/calibration.cpp:109-146), partial sums on the GPU
    static CalibrationTable calibrate(const Device& d, const OrthoTransform& t, const float* rows, std::uint32_t n,
                                      double p_s, std::uint32_t delta_d, std::uint64_t n_pairs, std::uint64_t seed) {
        t.upload(d);
        CalibrationTable c;
        c.p_s = p_s;
        c.delta_d = delta_d;
        std::vector<std::uint32_t> cps(t.dim + 1);
        std::vector<double> eps(t.dim + 1);
        std::uint32_t m = 0;
        check(dade_gpu_calibrate(d.get(), rows, n, p_s, delta_d, n_pairs, seed, 0, cps.data(), eps.data(), &m));
        c.checkpoints.assign(cps.begin(), cps.begin() + m);
        c.epsilons.assign(eps.begin(), eps.begin() + m);
        return c;
    }
};

// proj/include/dade/estimator.hpp:64-74 — here a strategy is the table the
// kernels read, installed on the device before a search.
class DcoStrategy {
public:
    virtual ~DcoStrategy() = default;
    virtual std::uint32_t dim() const = 0;
    virtual void install(const Device& d) const = 0;
    void use(const Device& d) const {
        if (d.active_strategy != this) {
            install(d);
            d.active_strategy = this;
        }
    }
};

class FdScanningStrategy final : public DcoStrategy {
public:
    explicit FdScanningStrategy(std::uint32_t dim) : dim_(dim) {}
    std::uint32_t dim() const override { return dim_; }
    void install(const Device& d) const override {
        check(dade_gpu_set_strategy(d.get(), DADE_GPU_FD, dim_, 0, nullptr, nullptr, nullptr));
    }

private:
    std::uint32_t dim_;
};

// proj/src/estimator.cpp:115-152: validation (ConfigError) happens here, as in
// the reference constructor.
class DadeStrategy final : public DcoStrategy {
public:
    DadeStrategy(const Device& d, const OrthoTransform& t, const CalibrationTable& cal, std::uint32_t delta_d)
        : t_(t), cal_(cal), delta_d_(delta_d) {
        install(d);
        d.active_strategy = this;
    }
    std::uint32_t dim() const override { return t_.dim; }
    void install(const Device& d) const override {
        t_.upload(d);
        check(dade_gpu_set_strategy_dade(d.get(), delta_d_, cal_.delta_d, std::uint32_t(cal_.checkpoints.size()),
                                         cal_.checkpoints.data(), cal_.epsilons.data()));
    }

private:
    OrthoTransform t_;
    CalibrationTable cal_;
    std::uint32_t delta_d_;
};

class AdsamplingStrategy final : public DcoStrategy {
public:
    AdsamplingStrategy(const Device& d, std::uint32_t dim, std::uint32_t delta_d, double eps0)
        : dim_(dim), delta_d_(delta_d), eps0_(eps0) {
        install(d);
        d.active_strategy = this;
    }
    std::uint32_t dim() const override { return dim_; }
    void install(const Device& d) const override {
        check(dade_gpu_set_strategy_ads(d.get(), dim_, delta_d_, eps0_));
    }

private:
    std::uint32_t dim_, delta_d_;
    double eps0_;
};

namespace detail {
inline std::vector<SearchResult> to_results(const std::vector<std::uint32_t>& ids, const std::vector<float>& d,
                                            const std::vector<std::uint32_t>& cnt, std::uint32_t nq, std::uint32_t k) {
    std::vector<SearchResult> out(nq);
    for (std::uint32_t q = 0; q < nq; ++q) {
        for (std::uint32_t i = 0; i < cnt[q]; ++i)
            out[q].neighbors.push_back({d[std::size_t(q) * k + i], ids[std::size_t(q) * k + i]});
        out[q].truncated = cnt[q] < k;
    }
    return out;
}
}  // namespace detail

// proj/include/dade/ivf.hpp:62-70; DIVF file proj/src/ivf.cpp:233-279
class IvfIndex {
public:
    static IvfIndex load(const Device& d, const std::string& path) {
        auto in = detail::open_in(path);
        char magic[4];
        in.read(magic, 4);
        if (!in || std::memcmp(magic, "DIVF", 4) != 0) throw std::runtime_error("not an ivf index file: " + path);
        if (detail::read_pod<std::uint32_t>(in, "version") != 1) throw std::runtime_error("unsupported ivf index version");
        const auto layout = detail::read_pod<std::uint8_t>(in, "layout");
        if (layout > 1) throw std::runtime_error("bad ivf layout byte");
        const auto dim = detail::read_pod<std::uint32_t>(in, "dim");
        const auto count = detail::read_pod<std::uint32_t>(in, "count");
        const auto nc = detail::read_pod<std::uint32_t>(in, "n_clusters");
        const auto split = detail::read_pod<std::uint32_t>(in, "split");
        if (dim == 0 || nc == 0 || split == 0 || split > dim) throw std::runtime_error("inconsistent ivf header");
        const auto cen = detail::read_vec<float>(in, std::size_t(nc) * dim, "centroids");
        const auto offs = detail::read_vec<std::uint32_t>(in, nc + 1, "offsets");
        const auto ids = detail::read_vec<std::uint32_t>(in, count, "ids");
        const auto sto = detail::read_vec<float>(in, std::size_t(count) * dim, "storage");
        check(dade_gpu_set_ivf(d.get(), dim, count, nc, layout, split, cen.data(), offs.data(), ids.data(), sto.data()));
        IvfIndex idx(d);
        idx.dim_ = dim;
        idx.count_ = count;
        idx.n_clusters_ = nc;
        return idx;
    }
    std::uint32_t dim() const { return dim_; }
    std::uint32_t count() const { return count_; }
    std::uint32_t n_clusters() const { return n_clusters_; }

    // Batched IvfIndex::search over nq rotated queries (raw = rotate first).
    std::vector<SearchResult> search_batch(const float* queries, std::uint32_t nq, std::uint32_t k,
                                           std::uint32_t n_probe, const DcoStrategy& dco, DcoStats* stats = nullptr,
                                           bool raw = false) const {
        if (dco.dim() != dim_) throw InvalidInput("IvfIndex::search: strategy dim mismatch");
        dco.use(*dev_);
        const std::uint32_t kk = k ? k : 1;
        std::vector<std::uint32_t> ids(std::size_t(nq) * kk), cnt(nq);
        std::vector<float> d(std::size_t(nq) * kk);
        dade_gpu_stats st{};
        const std::uint32_t flags = (raw ? DADE_GPU_QUERIES_RAW : 0u) |
                                    (stats && stats->measure_failures ? DADE_GPU_MEASURE_FAILURES : 0u);
        check(dade_gpu_ivf_search(dev_->get(), queries, nq, k, n_probe, flags, ids.data(), d.data(), cnt.data(), &st));
        if (stats) stats->add(st);
        return detail::to_results(ids, d, cnt, nq, kk);
    }
    SearchResult search(const float* query, std::uint32_t k, std::uint32_t n_probe, const DcoStrategy& dco,
                        DcoStats* stats = nullptr) const {
        return search_batch(query, 1, k, n_probe, dco, stats).front();
    }

    // Pipelined sequence of equal-sized batches (dade_gpu_ivf_search_batches):
    // batches[b] -> results[b], the same as search_batch per batch.
    std::vector<std::vector<SearchResult>> search_batches(const std::vector<const float*>& batches, std::uint32_t nq,
                                                          std::uint32_t k, std::uint32_t n_probe,
                                                          const DcoStrategy& dco, DcoStats* stats = nullptr,
                                                          bool raw = false) const {
        if (dco.dim() != dim_) throw InvalidInput("IvfIndex::search: strategy dim mismatch");
        dco.use(*dev_);
        const std::uint32_t kk = k ? k : 1;
        const std::size_t nb = batches.size();
        std::vector<std::vector<std::uint32_t>> ids(nb, std::vector<std::uint32_t>(std::size_t(nq) * kk)),
            cnt(nb, std::vector<std::uint32_t>(nq));
        std::vector<std::vector<float>> d(nb, std::vector<float>(std::size_t(nq) * kk));
        std::vector<std::uint32_t*> pi(nb), pc(nb);
        std::vector<float*> pd(nb);
        for (std::size_t b = 0; b < nb; ++b) {
            pi[b] = ids[b].data();
            pc[b] = cnt[b].data();
            pd[b] = d[b].data();
        }
        dade_gpu_stats st{};
        check(dade_gpu_ivf_search_batches(dev_->get(), (std::uint32_t)nb, batches.data(), nq, k, n_probe,
                                          raw ? DADE_GPU_QUERIES_RAW : 0, pi.data(), pd.data(), pc.data(), &st));
        if (stats) stats->add(st);
        std::vector<std::vector<SearchResult>> out;
        for (std::size_t b = 0; b < nb; ++b) out.push_back(detail::to_results(ids[b], d[b], cnt[b], nq, kk));
        return out;
    }

    // Keep only the lists with mask[c] != 0 on this device (list sharding).
    void shard(const std::vector<std::uint8_t>& mask) const {
        if (mask.size() != n_clusters_) throw InvalidInput("IvfIndex::shard: one mask byte per list");
        check(dade_gpu_set_ivf_shard(dev_->get(), mask.data()));
    }
    const Device& device() const { return *dev_; }

private:
    explicit IvfIndex(const Device& d) : dev_(&d) {}
    const Device* dev_;
    std::uint32_t dim_ = 0, count_ = 0, n_clusters_ = 0;
};

// linear_scan (proj/src/knn.cpp:31-41) over device-resident rows.
class FlatIndex {
public:
    FlatIndex(const Device& d, const float* rows, std::uint32_t n, std::uint32_t dim, std::uint32_t id_base = 0)
        : dev_(&d), dim_(dim) {
        check(dade_gpu_set_base(d.get(), dim, n, rows, id_base));
    }
    std::vector<SearchResult> search_batch(const float* queries, std::uint32_t nq, std::uint32_t k,
                                           const DcoStrategy& dco, DcoStats* stats = nullptr) const {
        if (dco.dim() != dim_) throw InvalidInput("linear_scan: strategy dim mismatch");
        dco.use(*dev_);
        const std::uint32_t kk = k ? k : 1;
        std::vector<std::uint32_t> ids(std::size_t(nq) * kk), cnt(nq);
        std::vector<float> d(std::size_t(nq) * kk);
        dade_gpu_stats st{};
        const std::uint32_t flags = stats && stats->measure_failures ? DADE_GPU_MEASURE_FAILURES : 0u;
        check(dade_gpu_flat_search(dev_->get(), queries, nq, k, flags, ids.data(), d.data(), cnt.data(), &st));
        if (stats) stats->add(st);
        return detail::to_results(ids, d, cnt, nq, kk);
    }
    SearchResult search(const float* q, std::uint32_t k, const DcoStrategy& dco, DcoStats* stats = nullptr) const {
        return search_batch(q, 1, k, dco, stats).front();
    }

private:
    const Device* dev_;
    std::uint32_t dim_;
};

// One NCCL communicator per GPU (dade_gpu_comm) and the sharded searches over it:
// IvfIndex::search over list shards (each rank its own queries) and linear_scan
// over row shards (the same queries on every rank). Rank 0 makes the unique id,
// the host hands it to every rank (MPI, a file, ...).
class Communicator {
public:
    using Id = std::array<std::uint8_t, DADE_GPU_NCCL_ID_BYTES>;
    static Id unique_id() {
        Id id{};
        check(dade_gpu_nccl_unique_id(id.data()));
        return id;
    }
    Communicator(const Device& d, int nranks, int rank, const Id& id) : dev_(&d) {
        check(dade_gpu_comm_create(d.get(), nranks, rank, id.data(), &comm_));
    }
    ~Communicator() {
        if (comm_) dade_gpu_comm_destroy(comm_);
    }
    Communicator(const Communicator&) = delete;
    Communicator& operator=(const Communicator&) = delete;

    std::vector<SearchResult> ivf_search(const float* queries, std::uint32_t nq, std::uint32_t k, std::uint32_t n_probe,
                                         const DcoStrategy& dco, DcoStats* stats = nullptr, bool raw = false) const {
        dco.use(*dev_);
        return run([&](std::uint32_t* i, float* d, std::uint32_t* c, dade_gpu_stats* st) {
            return dade_gpu_sharded_ivf_search(comm_, queries, nq, k, n_probe, raw ? DADE_GPU_QUERIES_RAW : 0u, i, d, c, st);
        }, nq, k, stats);
    }
    std::vector<SearchResult> flat_search(const float* queries, std::uint32_t nq, std::uint32_t k,
                                          const DcoStrategy& dco, DcoStats* stats = nullptr, bool raw = false) const {
        dco.use(*dev_);
        return run([&](std::uint32_t* i, float* d, std::uint32_t* c, dade_gpu_stats* st) {
            return dade_gpu_sharded_flat_search(comm_, queries, nq, k, raw ? DADE_GPU_QUERIES_RAW : 0u, i, d, c, st);
        }, nq, k, stats);
    }

private:
    template <class F>
    std::vector<SearchResult> run(F&& f, std::uint32_t nq, std::uint32_t k, DcoStats* stats) const {
        const std::uint32_t kk = k ? k : 1;
        std::vector<std::uint32_t> ids(std::size_t(nq) * kk), cnt(nq);
        std::vector<float> d(std::size_t(nq) * kk);
        dade_gpu_stats st{};
        check(f(ids.data(), d.data(), cnt.data(), &st));
        if (stats) stats->add(st);
        return detail::to_results(ids, d, cnt, nq, kk);
    }
    const Device* dev_;
    dade_gpu_comm* comm_ = nullptr;
};

}  // namespace gpu
}  // namespace dade

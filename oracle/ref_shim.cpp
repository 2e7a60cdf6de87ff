// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference library (/root/reference/proj,
// compiled from its own sources by oracle/Makefile into oracle/_ref/). It lets
// the pytest suite, the golden-fixture generator and bench.py's CPU-baseline
// leg drive the reference's public C++ API through ctypes:
//   * dade::make_synthetic          proj/src/dataset_io.cpp:267-307
//   * dade::fit_pca / apply_transform proj/src/transform.cpp:230-253, 295-304
//   * dade::calibrate               proj/src/calibration.cpp:109-146
//   * DcoStrategy::evaluate         proj/include/dade/estimator.hpp:64-74
//   * IvfIndex::build/load/search   proj/src/ivf.cpp:145-231, 249-279
//   * linear_scan                   proj/src/knn.cpp:31-41
//   * compute_ground_truth          proj/src/dataset_io.cpp:101-135
// Exceptions are mapped to status codes: 1 runtime_error, 2 ConfigError,
// 3 InvalidInput (the reference CLI's own exit-code split,
// proj/tools/dade_cli.cpp:407-419).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <functional>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "dade/calibration.hpp"
#include "dade/dataset_io.hpp"
#include "dade/error.hpp"
#include "dade/estimator.hpp"
#include "dade/ivf.hpp"
#include "dade/knn.hpp"
#include "dade/transform.hpp"

using namespace dade;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const InvalidInput& e) {
        g_err = e.what();
        return 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

VectorSet make_set(const float* v, std::uint32_t n, std::uint32_t dim) {
    VectorSet s;
    s.count = n;
    s.dim = dim;
    s.values.assign(v, v + static_cast<std::size_t>(n) * dim);
    return s;
}

struct Strategy {
    std::unique_ptr<DcoStrategy> s;
};
}  // namespace

extern "C" {

const char* dref_last_error() { return g_err.c_str(); }

int dref_synth(std::uint32_t count, std::uint32_t dim, std::uint32_t nq, std::uint64_t seed,
               int spectrum, double alpha, int rotate, double mean_shift, float* out_data,
               float* out_queries) {
    return guard([&] {
        SynthSpec spec;
        spec.count = count;
        spec.dim = dim;
        spec.query_count = nq;
        spec.seed = seed;
        spec.spectrum = spectrum == 0 ? SynthSpec::Spectrum::power : SynthSpec::Spectrum::uniform;
        spec.alpha = alpha;
        spec.rotate = rotate != 0;
        spec.mean_shift = mean_shift;
        SynthDataset ds = make_synthetic(spec);
        std::memcpy(out_data, ds.data.values.data(), ds.data.values.size() * sizeof(float));
        if (nq > 0)
            std::memcpy(out_queries, ds.queries.values.data(),
                        ds.queries.values.size() * sizeof(float));
    });
}

// ---- transform ------------------------------------------------------------
int dref_fit_pca(const float* data, std::uint32_t n, std::uint32_t dim, void** out) {
    return guard([&] { *out = new OrthoTransform(fit_pca(make_set(data, n, dim))); });
}
int dref_fit_random(std::uint32_t dim, std::uint64_t seed, const float* data, std::uint32_t n,
                    void** out) {
    return guard([&] {
        *out = new OrthoTransform(fit_random_orthogonal(dim, seed, make_set(data, n, dim)));
    });
}
int dref_transform_load(const char* path, void** out) {
    return guard([&] { *out = new OrthoTransform(OrthoTransform::load(path)); });
}
int dref_transform_save(void* t, const char* path) {
    return guard([&] { static_cast<OrthoTransform*>(t)->save(path); });
}
void dref_transform_free(void* t) { delete static_cast<OrthoTransform*>(t); }
std::uint32_t dref_transform_dim(void* t) { return static_cast<OrthoTransform*>(t)->dim; }
int dref_transform_kind(void* t) { return static_cast<int>(static_cast<OrthoTransform*>(t)->kind); }
void dref_transform_get(void* tp, double* mean, double* eig, double* matrix, double* prefix) {
    const auto* t = static_cast<OrthoTransform*>(tp);
    std::memcpy(mean, t->mean.data(), t->dim * sizeof(double));
    std::memcpy(eig, t->eigenvalues.data(), t->dim * sizeof(double));
    std::memcpy(matrix, t->matrix.data(), t->matrix.size() * sizeof(double));
    std::memcpy(prefix, t->lambda_prefix.data(), (t->dim + 1) * sizeof(double));
}
int dref_apply_transform(void* t, const float* in, std::uint32_t n, float* out) {
    return guard([&] {
        const auto* tr = static_cast<OrthoTransform*>(t);
        VectorSet o = apply_transform(*tr, make_set(in, n, tr->dim));
        std::memcpy(out, o.values.data(), o.values.size() * sizeof(float));
    });
}

// ---- calibration ----------------------------------------------------------
int dref_calibrate(void* t, const float* data, std::uint32_t n, double p_s, std::uint32_t delta_d,
                   std::uint64_t n_pairs, std::uint64_t seed, void** out) {
    return guard([&] {
        const auto* tr = static_cast<OrthoTransform*>(t);
        *out = new CalibrationTable(
            calibrate(*tr, make_set(data, n, tr->dim), p_s, delta_d, n_pairs, seed));
    });
}
int dref_cal_load(const char* path, void** out) {
    return guard([&] { *out = new CalibrationTable(CalibrationTable::load(path)); });
}
int dref_cal_save(void* c, const char* path) {
    return guard([&] { static_cast<CalibrationTable*>(c)->save(path); });
}
void* dref_cal_unbounded(std::uint32_t dim, std::uint32_t delta_d) {
    return new CalibrationTable(CalibrationTable::unbounded(dim, delta_d));
}
void* dref_cal_from(double p_s, std::uint32_t delta_d, std::uint32_t n, const std::uint32_t* cps,
                    const double* eps) {
    auto* c = new CalibrationTable;
    c->p_s = p_s;
    c->delta_d = delta_d;
    c->checkpoints.assign(cps, cps + n);
    c->epsilons.assign(eps, eps + n);
    return c;
}
void dref_cal_free(void* c) { delete static_cast<CalibrationTable*>(c); }
std::uint32_t dref_cal_get(void* cp, double* p_s, std::uint32_t* delta_d, std::uint32_t* cps,
                           double* eps) {
    const auto* c = static_cast<CalibrationTable*>(cp);
    if (p_s) *p_s = c->p_s;
    if (delta_d) *delta_d = c->delta_d;
    for (std::size_t i = 0; i < c->checkpoints.size(); ++i) {
        if (cps) cps[i] = c->checkpoints[i];
        if (eps) eps[i] = c->epsilons[i];
    }
    return static_cast<std::uint32_t>(c->checkpoints.size());
}
std::uint32_t dref_expected_checkpoints(std::uint32_t dim, std::uint32_t delta_d,
                                        std::uint32_t* out) {
    const auto v = CalibrationTable::expected_checkpoints(dim, delta_d);
    if (out) std::memcpy(out, v.data(), v.size() * sizeof(std::uint32_t));
    return static_cast<std::uint32_t>(v.size());
}

// ---- strategies -----------------------------------------------------------
void* dref_strategy_fd(std::uint32_t dim) { return new Strategy{std::make_unique<FdScanningStrategy>(dim)}; }
int dref_strategy_dade(void* t, void* cal, std::uint32_t delta_d, void** out) {
    return guard([&] {
        *out = new Strategy{std::make_unique<DadeStrategy>(*static_cast<OrthoTransform*>(t),
                                                           *static_cast<CalibrationTable*>(cal),
                                                           delta_d)};
    });
}
int dref_strategy_ads(std::uint32_t dim, std::uint32_t delta_d, double eps0, void** out) {
    return guard(
        [&] { *out = new Strategy{std::make_unique<AdsamplingStrategy>(dim, delta_d, eps0)}; });
}
void dref_strategy_free(void* s) { delete static_cast<Strategy*>(s); }

// Evaluates n independent (o_i, q_i, r_i) DCOs; stats accumulate into
// stats[0..3] = total_dco, dims_accumulated, eligible, failures.
int dref_evaluate(void* sp, const float* o, const float* q, const float* r, std::uint32_t n,
                  std::uint32_t dim, int measure_failures, std::uint8_t* pruned, float* dist,
                  std::uint8_t* exact, std::uint32_t* dims_used, std::uint64_t* stats) {
    return guard([&] {
        const DcoStrategy& s = *static_cast<Strategy*>(sp)->s;
        DcoStats st;
        st.measure_failures = measure_failures != 0;
        for (std::uint32_t i = 0; i < n; ++i) {
            const DcoOutcome out = s.evaluate(o + static_cast<std::size_t>(i) * dim,
                                              q + static_cast<std::size_t>(i) * dim, r[i], &st);
            pruned[i] = out.pruned;
            dist[i] = out.distance;
            exact[i] = out.distance_exact;
            dims_used[i] = out.dims_used;
        }
        if (stats) {
            stats[0] += st.total_dco;
            stats[1] += st.dims_accumulated;
            stats[2] += st.eligible;
            stats[3] += st.failures;
        }
    });
}

float dref_partial_sqdist(const float* o, const float* q, std::uint32_t dim, std::uint32_t lo,
                          std::uint32_t hi) {
    return partial_sqdist(o, q, dim, lo, hi);
}
double dref_dade_estimate(void* t, double partial, std::uint32_t d) {
    return dade_estimate(*static_cast<OrthoTransform*>(t), partial, d);
}

// ---- ivf ------------------------------------------------------------------
int dref_ivf_build(const float* data, std::uint32_t n, std::uint32_t dim, std::uint32_t n_clusters,
                   int layout, std::uint32_t split, std::uint32_t iters, std::uint64_t seed,
                   void** out) {
    return guard([&] {
        *out = new IvfIndex(IvfIndex::build(make_set(data, n, dim), n_clusters,
                                            layout ? IvfLayout::split : IvfLayout::contiguous,
                                            split, iters, seed));
    });
}
int dref_ivf_load(const char* path, void** out) {
    return guard([&] { *out = new IvfIndex(IvfIndex::load(path)); });
}
int dref_ivf_save(void* ivf, const char* path) {
    return guard([&] { static_cast<IvfIndex*>(ivf)->save(path); });
}
void dref_ivf_free(void* ivf) { delete static_cast<IvfIndex*>(ivf); }

// Batched IvfIndex::search over nq rotated queries. threads <= 1 runs the
// reference's own single-thread loop (proj/src/bench.cpp:52-56); threads > 1
// splits queries into strided subsets, one DcoStats per worker, sharing the
// immutable index and strategy. *seconds is steady_clock
// time around the query loop only, as measure() does.
static int search_common(const std::function<SearchResult(const float*, DcoStats*)>& fn,
                         const float* queries, std::uint32_t nq, std::uint32_t dim,
                         std::uint32_t k, std::uint32_t* out_ids, float* out_dists,
                         std::uint32_t* out_counts, std::uint8_t* truncated,
                         std::uint64_t* stats, int threads, double* seconds) {
    return guard([&] {
        const int nt = threads < 1 ? 1 : threads;
        std::vector<DcoStats> st(static_cast<std::size_t>(nt));
        std::vector<std::exception_ptr> errs(static_cast<std::size_t>(nt));
        auto worker = [&](int w) {
            try {
                for (std::uint32_t qi = static_cast<std::uint32_t>(w); qi < nq;
                     qi += static_cast<std::uint32_t>(nt)) {
                    SearchResult res = fn(queries + static_cast<std::size_t>(qi) * dim, &st[w]);
                    const std::size_t m = res.neighbors.size();
                    for (std::size_t i = 0; i < m && i < k; ++i) {
                        out_ids[static_cast<std::size_t>(qi) * k + i] = res.neighbors[i].id;
                        out_dists[static_cast<std::size_t>(qi) * k + i] = res.neighbors[i].distance;
                    }
                    out_counts[qi] = static_cast<std::uint32_t>(m);
                    truncated[qi] = res.truncated;
                }
            } catch (...) {
                errs[w] = std::current_exception();
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        if (nt == 1) {
            worker(0);
        } else {
            std::vector<std::thread> pool;
            for (int w = 0; w < nt; ++w) pool.emplace_back(worker, w);
            for (auto& th : pool) th.join();
        }
        const auto t1 = std::chrono::steady_clock::now();
        for (auto& e : errs)
            if (e) std::rethrow_exception(e);
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (stats) {
            for (const auto& s : st) {
                stats[0] += s.total_dco;
                stats[1] += s.dims_accumulated;
            }
        }
    });
}

int dref_ivf_search(void* ivf, void* sp, const float* queries, std::uint32_t nq, std::uint32_t k,
                    std::uint32_t n_probe, std::uint32_t* out_ids, float* out_dists,
                    std::uint32_t* out_counts, std::uint8_t* truncated, std::uint64_t* stats,
                    int threads, double* seconds) {
    const IvfIndex& idx = *static_cast<IvfIndex*>(ivf);
    const DcoStrategy& s = *static_cast<Strategy*>(sp)->s;
    return search_common(
        [&](const float* q, DcoStats* st) { return idx.search(q, k, n_probe, s, st); }, queries,
        nq, idx.dim(), k, out_ids, out_dists, out_counts, truncated, stats, threads, seconds);
}

int dref_linear_scan(const float* data, std::uint32_t n, std::uint32_t dim, void* sp,
                     const float* queries, std::uint32_t nq, std::uint32_t k,
                     std::uint32_t* out_ids, float* out_dists, std::uint32_t* out_counts,
                     std::uint8_t* truncated, std::uint64_t* stats, int threads, double* seconds) {
    VectorSet base;
    int rc = guard([&] { base = make_set(data, n, dim); });
    if (rc) return rc;
    const DcoStrategy& s = *static_cast<Strategy*>(sp)->s;
    return search_common(
        [&](const float* q, DcoStats* st) { return linear_scan(base, q, k, s, st); }, queries,
        nq, dim, k, out_ids, out_dists, out_counts, truncated, stats, threads, seconds);
}

int dref_ground_truth(const float* data, std::uint32_t n, const float* queries, std::uint32_t nq,
                      std::uint32_t dim, std::uint32_t k, std::uint32_t* out) {
    return guard([&] {
        GroundTruth gt = compute_ground_truth(make_set(data, n, dim), make_set(queries, nq, dim), k);
        for (std::uint32_t qi = 0; qi < nq; ++qi)
            std::memcpy(out + static_cast<std::size_t>(qi) * k, gt.ids[qi].data(),
                        k * sizeof(std::uint32_t));
    });
}

// The untimed failure pass of measure() (proj/src/bench.cpp:65-73): every query
// searched once more with DcoStats::measure_failures; stats [4] accumulate
// total_dco, dims_accumulated, eligible, failures.
int dref_ivf_failure_pass(void* ivf, void* sp, const float* queries, std::uint32_t nq, std::uint32_t k,
                          std::uint32_t n_probe, std::uint64_t* stats) {
    return guard([&] {
        const IvfIndex& idx = *static_cast<IvfIndex*>(ivf);
        const DcoStrategy& s = *static_cast<Strategy*>(sp)->s;
        DcoStats fstats;
        fstats.measure_failures = true;
        for (std::uint32_t qi = 0; qi < nq; ++qi)
            idx.search(queries + static_cast<std::size_t>(qi) * idx.dim(), k, n_probe, s, &fstats);
        stats[0] += fstats.total_dco;
        stats[1] += fstats.dims_accumulated;
        stats[2] += fstats.eligible;
        stats[3] += fstats.failures;
    });
}

int dref_covariance(const float* data, std::uint32_t n, std::uint32_t dim, double* mean, double* cov) {
    return guard([&] {
        CovarianceResult c = compute_covariance(make_set(data, n, dim));
        std::memcpy(mean, c.mean.data(), c.mean.size() * sizeof(double));
        std::memcpy(cov, c.cov.data(), c.cov.size() * sizeof(double));
    });
}

int dref_kmeans(const float* data, std::uint32_t n, std::uint32_t dim, std::uint32_t n_clusters,
                std::uint32_t iters, std::uint64_t seed, float* centroids,
                std::uint32_t* assignments, std::uint32_t* iterations) {
    return guard([&] {
        KmeansResult km = kmeans(make_set(data, n, dim), n_clusters, iters, seed);
        std::memcpy(centroids, km.centroids.data(), km.centroids.size() * sizeof(float));
        std::memcpy(assignments, km.assignments.data(), km.assignments.size() * sizeof(std::uint32_t));
        *iterations = km.iterations;
    });
}

}  // extern "C"

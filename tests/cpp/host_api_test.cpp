// C++ mirror-API test (include/dade_gpu.hpp), driven by tests/test_cpp_host_api.py:
//   host_api_test <index.divf> <transform.dade> <cal.cal> <queries.fvecs> <out.ivecs>
// Loads the reference artifacts, runs FD / DADE / ADS IVF searches through the
// mirror API (k = 10, n_probe = 3) and the reference's own error cases, and
// writes the FD result ids as ivecs (compared with the golden reference output
// by the Python side). Prints one line per check; exit code = failures.
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "dade_gpu.hpp"

using namespace dade::gpu;

static std::vector<float> read_fvecs(const std::string& path, std::uint32_t& n, std::uint32_t& dim) {
    std::ifstream in(path, std::ios::binary);
    std::vector<float> out;
    n = 0;
    std::int32_t d = 0;
    while (in.read(reinterpret_cast<char*>(&d), 4)) {
        std::vector<float> row(d);
        in.read(reinterpret_cast<char*>(row.data()), 4 * d);
        out.insert(out.end(), row.begin(), row.end());
        ++n;
    }
    dim = std::uint32_t(d);
    return out;
}

int main(int argc, char** argv) {
    if (argc != 6) {
        std::fprintf(stderr, "usage: %s index transform cal queries out.ivecs\n", argv[0]);
        return 99;
    }
    int fails = 0;
    auto report = [&](bool ok, const char* what) {
        std::printf("[%s] %s\n", ok ? "PASS" : "FAIL", what);
        if (!ok) ++fails;
    };
    Device dev(0);
    const IvfIndex idx = IvfIndex::load(dev, argv[1]);
    const OrthoTransform t = OrthoTransform::load(argv[2]);
    const CalibrationTable cal = CalibrationTable::load(argv[3]);
    std::uint32_t nq = 0, dim = 0;
    const std::vector<float> qs = read_fvecs(argv[4], nq, dim);
    report(dim == idx.dim(), "query dim matches index");

    const FdScanningStrategy fd(dim);
    DcoStats st;
    const auto res = idx.search_batch(qs.data(), nq, 10, 3, fd, &st);
    report(st.total_dco > 0 && st.dims_accumulated == st.total_dco * dim, "FD stats: full dimension per DCO");
    {
        std::ofstream out(argv[5], std::ios::binary);
        for (const auto& r : res) {
            std::int32_t k = 10;
            out.write(reinterpret_cast<const char*>(&k), 4);
            for (std::uint32_t i = 0; i < 10; ++i) {
                std::int32_t id = i < r.neighbors.size() ? std::int32_t(r.neighbors[i].id) : -1;
                out.write(reinterpret_cast<const char*>(&id), 4);
            }
        }
    }
    bool sorted = true;
    for (const auto& r : res)
        for (std::size_t i = 1; i < r.neighbors.size(); ++i) sorted = sorted && r.neighbors[i - 1] < r.neighbors[i];
    report(sorted, "results ascending by (distance, id)");
    {
        DcoStats sb;
        const auto rb = idx.search_batches({qs.data(), qs.data()}, nq, 10, 3, fd, &sb);
        bool same = rb.size() == 2;
        for (std::size_t b = 0; same && b < 2; ++b)
            for (std::uint32_t q = 0; same && q < nq; ++q) {
                same = rb[b][q].neighbors.size() == res[q].neighbors.size();
                for (std::size_t i = 0; same && i < res[q].neighbors.size(); ++i)
                    same = rb[b][q].neighbors[i].id == res[q].neighbors[i].id &&
                           rb[b][q].neighbors[i].distance == res[q].neighbors[i].distance;
            }
        report(same && sb.total_dco == 2 * st.total_dco, "pipelined batches == single searches (FD), stats summed");
    }

    {  // the NCCL layer with one rank: every protocol step runs, results equal the plain search
        const Communicator comm(dev, 1, 0, Communicator::unique_id());
        DcoStats sc;
        const auto rc = comm.ivf_search(qs.data(), nq, 10, 3, fd, &sc);
        bool same = rc.size() == res.size();
        for (std::uint32_t q = 0; same && q < nq; ++q) {
            same = rc[q].neighbors.size() == res[q].neighbors.size();
            for (std::size_t i = 0; same && i < res[q].neighbors.size(); ++i)
                same = rc[q].neighbors[i].id == res[q].neighbors[i].id &&
                       rc[q].neighbors[i].distance == res[q].neighbors[i].distance;
        }
        report(same && sc.total_dco == st.total_dco, "sharded_ivf_search (1 rank, NCCL) == IvfIndex::search (FD)");
    }

    const DadeStrategy dade(dev, t, cal, cal.delta_d);
    DcoStats sd;
    const auto rd = idx.search(qs.data(), 10, 3, dade, &sd);
    report(rd.neighbors.size() == 10 && !rd.truncated, "DADE search returns k results");
    report(sd.dims_accumulated < sd.total_dco * dim, "DADE prunes before the full dimension");
    const AdsamplingStrategy ads(dev, dim, cal.delta_d, 2.1);
    report(idx.search(qs.data(), 10, 3, ads).neighbors.size() == 10, "ADS search returns k results");
    report(idx.search(qs.data(), 700, idx.n_clusters(), fd).truncated, "asking for more than N sets truncated");

    auto throws_invalid = [&](auto fn) {
        try {
            fn();
        } catch (const InvalidInput&) {
            return true;
        } catch (...) {
        }
        return false;
    };
    report(throws_invalid([&] { idx.search(qs.data(), 0, 3, fd); }), "k == 0 -> InvalidInput");
    report(throws_invalid([&] { idx.search(qs.data(), 10, 0, fd); }), "n_probe == 0 -> InvalidInput");
    report(throws_invalid([&] { idx.search(qs.data(), 10, idx.n_clusters() + 1, fd); }), "n_probe > n -> InvalidInput");
    bool cfg = false;
    try {
        DadeStrategy bad(dev, t, cal, cal.delta_d * 2);
    } catch (const ConfigError&) {
        cfg = true;
    }
    report(cfg, "calibration step mismatch -> ConfigError");
    std::printf("%d failures\n", fails);
    return fails;
}

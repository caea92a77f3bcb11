// Header-only C++ adapter over the ph0b C ABI (include/ph0b.h) that mirrors the reference
// library's hot-path interface (namespace ph0, /root/reference/proj/include/ph0/*.hpp):
// same names, same argument meaning, same result types (layout-compatible Interval /
// Barcode / Edge / Filtration) and the same exceptions (std::invalid_argument with the
// reference's messages).  A maintainer swaps the five-call composition of
// proj/src/bench.cpp:45-59 for ph0b::h0_barcode.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "ph0b.h"

namespace ph0b {

// proj/include/ph0/barcode.hpp:11-15
struct Interval {
    double birth = 0.0;
    std::uint64_t death_grade = 0;
    double death_length = 0.0;
};

// proj/include/ph0/barcode.hpp:17-20
struct Barcode {
    std::vector<Interval> finite;
    std::size_t essential_count = 0;
};

// proj/include/ph0/filtration.hpp:11-15
struct PairDistance {
    std::uint32_t u = 0;
    std::uint32_t v = 0;
    double length = 0.0;
};

// proj/include/ph0/filtration.hpp:19-31
struct Edge {
    std::uint32_t u = 0;
    std::uint32_t v = 0;
    double length = 0.0;
    std::uint64_t grade = 0;
};
struct Filtration {
    std::vector<Edge> edges;
    std::vector<double> scale;
};

// proj/include/ph0/reduction.hpp:11-17 (result-neutral here, as in the reference)
struct ReductionOptions {
    bool pivoting = true;
    unsigned workers = 1;
};

class Error : public std::runtime_error {
public:
    Error(int code, const std::string& what) : std::runtime_error(what), code_(code) {}
    int code() const { return code_; }

private:
    int code_;
};

namespace detail {
inline void check(int rc) {
    if (rc == PH0B_OK) return;
    const std::string msg = ph0b_last_error();
    if (rc == PH0B_ERR_INVALID_ARGUMENT || rc == PH0B_ERR_NONFINITE || rc == PH0B_ERR_TOO_LARGE)
        throw std::invalid_argument(msg);  // reference: point_cloud.cpp:17, filtration.cpp:11
    throw Error(rc, msg);
}
inline ph0b_options opts(const ReductionOptions& r, int device) {
    ph0b_options o{};
    o.struct_size = sizeof(o);
    o.device = device;
    o.pivoting = r.pivoting ? 1u : 0u;
    o.workers = r.workers;
    return o;
}
}  // namespace detail

// pairwise_distances (filtration.cpp:8-18).  x is column-major N x d, as
// Eigen::MatrixXd::data() of PointCloud::points().
inline std::vector<PairDistance> pairwise_distances(const double* x, std::size_t n, std::size_t d,
                                                    int device = 0) {
    const std::size_t k = n * (n - (n > 0)) / 2;
    std::vector<double> len(k);
    const ph0b_options o = detail::opts({}, device);
    detail::check(ph0b_pairwise_distances(x, n, d, PH0B_COL_MAJOR, &o, len.data()));
    std::vector<PairDistance> out;
    out.reserve(k);
    std::size_t e = 0;
    for (std::uint32_t u = 0; u + 1 < n; ++u)
        for (std::uint32_t v = u + 1; v < n; ++v) out.push_back({u, v, len[e++]});
    return out;
}

// pairwise_distances ∘ build_filtration (filtration.cpp:20-35): edges sorted by (length, u, v)
// with 1-based grades, scale = D.
inline Filtration build_filtration(const double* x, std::size_t n, std::size_t d, int device = 0) {
    const std::size_t k = n * (n - (n > 0)) / 2;
    std::vector<std::uint32_t> u(k), v(k);
    std::vector<std::uint64_t> g(k);
    Filtration f;
    f.scale.resize(k);
    std::uint64_t ns = 0;
    const ph0b_options o = detail::opts({}, device);
    detail::check(ph0b_build_filtration(x, n, d, PH0B_COL_MAJOR, &o, u.data(), v.data(), g.data(),
                                        f.scale.data(), &ns));
    f.scale.resize(ns);
    f.edges.resize(k);
    for (std::size_t i = 0; i < k; ++i) f.edges[i] = {u[i], v[i], f.scale[g[i] - 1], g[i]};
    return f;
}

namespace detail {
// X -> bars (+ D into *scale) through ph0b_h0_barcode_into: D is written straight into the
// caller's vector by the library (for large clouds: streamed to the host while the sort
// runs, decoded by host threads into scale->data()), never copied a second time.  The vector
// is sized to K = n(n-1)/2 >= |D| first and shrunk to |D| after; a vector reused across
// calls keeps its capacity, so growing it back costs only the few tail entries.
inline Barcode run_into(const double* x, std::size_t n, std::size_t d,
                        std::vector<double>* scale, ph0b_options o) {
    const std::size_t k = n * (n - (n > 0)) / 2;
    std::vector<std::uint64_t> grade(n ? n : 1);
    std::vector<double> length(n ? n : 1);
    std::uint64_t nf = 0, ess = 0, ns = 0;
    if (scale) {
        if (scale->size() < k) scale->resize(k);
    } else {
        o.flags |= PH0B_FLAG_NO_SCALE;
    }
    check(ph0b_h0_barcode_into(x, n, d, PH0B_COL_MAJOR, &o, grade.data(), length.data(), &nf,
                               &ess, scale ? scale->data() : nullptr, scale ? scale->size() : 0,
                               &ns, nullptr));
    if (scale) scale->resize(ns);
    Barcode bc;
    bc.finite.resize(nf);
    for (std::uint64_t i = 0; i < nf; ++i) bc.finite[i] = {0.0, grade[i], length[i]};
    bc.essential_count = ess;
    return bc;
}
}  // namespace detail

// The whole hot path: pairwise_distances -> build_filtration -> build_boundary_matrix ->
// reduce -> extract_barcode (bench.cpp:45-59).  Optionally returns D (Filtration::scale).
inline Barcode h0_barcode(const double* x, std::size_t n, std::size_t d,
                          std::vector<double>* scale = nullptr,
                          const ReductionOptions& ropts = {}, int device = 0) {
    return detail::run_into(x, n, d, scale, detail::opts(ropts, device));
}

// The same on several GPUs of this node (ph0b_options.n_gpus / devices; an ordinal may repeat).
inline Barcode h0_barcode_multi(const double* x, std::size_t n, std::size_t d,
                                const std::vector<std::int32_t>& devices,
                                std::vector<double>* scale = nullptr,
                                const ReductionOptions& ropts = {}) {
    ph0b_options o = detail::opts(ropts, devices.empty() ? 0 : devices[0]);
    o.n_gpus = static_cast<std::uint32_t>(devices.size());
    o.devices = devices.data();
    return detail::run_into(x, n, d, scale, o);
}

// kruskal_barcode (oracle.cpp:32-46): union-find over the GPU filtration (ph0b_kruskal_barcode).
inline Barcode kruskal_barcode(const double* x, std::size_t n, std::size_t d,
                               std::vector<double>* scale = nullptr, int device = 0) {
    ph0b_options o = detail::opts({}, device);
    o.flags |= PH0B_FLAG_KRUSKAL;
    return detail::run_into(x, n, d, scale, o);
}

// Claimed low of every surviving column (reduction.cpp:44-45), filtration order.
inline std::vector<std::uint32_t> claimed_lows(const double* x, std::size_t n, std::size_t d,
                                               int device = 0) {
    std::vector<std::uint32_t> lows(n ? n : 1);
    std::uint64_t m = 0;
    const ph0b_options o = detail::opts({}, device);
    detail::check(ph0b_claimed_lows(x, n, d, PH0B_COL_MAJOR, &o, lows.data(), &m));
    lows.resize(m);
    return lows;
}

// Sorted multisets (barcode.cpp:9-23).
inline std::vector<std::uint64_t> finite_death_grades(const Barcode& b) {
    std::vector<std::uint64_t> g;
    for (const auto& iv : b.finite) g.push_back(iv.death_grade);
    std::sort(g.begin(), g.end());
    return g;
}
inline std::vector<double> finite_death_lengths(const Barcode& b) {
    std::vector<double> l;
    for (const auto& iv : b.finite) l.push_back(iv.death_length);
    std::sort(l.begin(), l.end());
    return l;
}

}  // namespace ph0b

// TEST INFRASTRUCTURE ONLY — C entry points around the UNMODIFIED reference library.
//
// This file is compiled together with /root/reference/proj/src/*.cpp (built in place by
// oracle/Makefile, outputs only under oracle/_ref/) and the Eigen shim in oracle/shim/.
// It lets pytest (ctypes), bench.py's reference arm and the golden-fixture script run the
// reference's own hot path:
//   pairwise_distances -> build_filtration -> build_boundary_matrix -> reduce -> extract_barcode
// exactly as composed in proj/src/bench.cpp:45-59 (timed_pipeline), proj/tools/ph0_cli.cpp:58-71
// (run_compute) and proj/tests/acceptance.cpp:56-68 (run_pipeline); and the Kruskal path of
// proj/tools/ph0_cli.cpp:73-80 (run_oracle).  Nothing here is used by the product library.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "ph0/barcode.hpp"
#include "ph0/boundary_matrix.hpp"
#include "ph0/filtration.hpp"
#include "ph0/format.hpp"
#include "ph0/oracle.hpp"
#include "ph0/point_cloud.hpp"
#include "ph0/reduction.hpp"
#include "ph0/splitmix64.hpp"

namespace {

thread_local std::string g_err;

ph0::PointCloud make_cloud(const double* x_colmajor, std::uint64_t n, std::uint64_t d) {
    Eigen::MatrixXd m(static_cast<Eigen::Index>(n), static_cast<Eigen::Index>(d));
    if (n * d) std::memcpy(m.data(), x_colmajor, sizeof(double) * n * d);
    return ph0::PointCloud(std::move(m));
}

double secs(std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
    return std::chrono::duration<double>(b - a).count();
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// SplitMix64 stream (splitmix64.hpp:20-33).
void ref_splitmix_next(std::uint64_t seed, std::uint64_t count, std::uint64_t* out) {
    ph0::SplitMix64 g(seed);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = g.next();
}

// generate_uniform_cloud (point_cloud.cpp:20-29); output column-major n x d.
int ref_generate_uniform_cloud(std::uint64_t n, std::uint64_t d, std::uint64_t seed, double* out) {
    try {
        const ph0::PointCloud c = ph0::generate_uniform_cloud(n, d, seed);
        if (n * d) std::memcpy(out, c.points().data(), sizeof(double) * n * d);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// pairwise_distances (filtration.cpp:8-18): u-major lengths (u, v implied by order).
int ref_pairwise_distances(const double* x, std::uint64_t n, std::uint64_t d, double* lengths) {
    try {
        const auto dists = ph0::pairwise_distances(make_cloud(x, n, d));
        for (std::size_t i = 0; i < dists.size(); ++i) lengths[i] = dists[i].length;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// build_filtration (filtration.cpp:20-35): sorted edges (u, v, grade) and the scale D.
int ref_build_filtration(const double* x, std::uint64_t n, std::uint64_t d, std::uint32_t* u,
                         std::uint32_t* v, std::uint64_t* grade, double* scale,
                         std::uint64_t* n_scale) {
    try {
        const ph0::Filtration f = ph0::build_filtration(ph0::pairwise_distances(make_cloud(x, n, d)));
        for (std::size_t i = 0; i < f.edges.size(); ++i) {
            u[i] = f.edges[i].u;
            v[i] = f.edges[i].v;
            grade[i] = f.edges[i].grade;
        }
        std::memcpy(scale, f.scale.data(), sizeof(double) * f.scale.size());
        *n_scale = f.scale.size();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Full hot path (bench.cpp:45-59).  mode 0 = reduce (reduction.cpp:129-131), mode 1 = Kruskal
// oracle path (ph0_cli.cpp:73-80), mode 2 = reduce_parallel with `workers` lanes.
// Outputs: bars in filtration order (death_grade, death_length), essential_count, the scale D
// (if scale != nullptr), stage seconds [dist, filtration, matrix, reduce, extract], and for
// mode 0/2 the claimed low of every surviving column (lows != nullptr).
int ref_h0_barcode(const double* x, std::uint64_t n, std::uint64_t d, int mode, unsigned workers,
                   std::uint64_t* death_grade, double* death_length, std::uint64_t* n_finite,
                   std::uint64_t* essential, double* scale, std::uint64_t* n_scale,
                   double* stage_seconds, std::uint32_t* lows) {
    try {
        const ph0::PointCloud cloud = make_cloud(x, n, d);
        const auto t0 = std::chrono::steady_clock::now();
        auto dists = ph0::pairwise_distances(cloud);
        const auto t1 = std::chrono::steady_clock::now();
        const ph0::Filtration f = ph0::build_filtration(std::move(dists));
        const auto t2 = std::chrono::steady_clock::now();
        ph0::Barcode bc;
        auto t3 = t2, t4 = t2, t5 = t2;
        if (mode == 1) {
            bc = ph0::kruskal_barcode(f, n);
            t5 = t4 = t3 = std::chrono::steady_clock::now();
        } else {
            ph0::BoundaryMatrix m = ph0::build_boundary_matrix(f, n);
            t3 = std::chrono::steady_clock::now();
            if (mode == 2)
                ph0::reduce_parallel(m, ph0::ReductionOptions{true, workers});
            else
                ph0::reduce(m);
            t4 = std::chrono::steady_clock::now();
            bc = ph0::extract_barcode(m, f);
            t5 = std::chrono::steady_clock::now();
            if (lows) {
                std::size_t k = 0;
                for (const auto& col : m.columns)
                    if (col.support.any()) lows[k++] = col.support.top();
            }
        }
        for (std::size_t i = 0; i < bc.finite.size(); ++i) {
            death_grade[i] = bc.finite[i].death_grade;
            death_length[i] = bc.finite[i].death_length;
        }
        *n_finite = bc.finite.size();
        *essential = bc.essential_count;
        if (scale) std::memcpy(scale, f.scale.data(), sizeof(double) * f.scale.size());
        if (n_scale) *n_scale = f.scale.size();
        if (stage_seconds) {
            stage_seconds[0] = secs(t0, t1);
            stage_seconds[1] = secs(t1, t2);
            stage_seconds[2] = secs(t2, t3);
            stage_seconds[3] = secs(t3, t4);
            stage_seconds[4] = secs(t4, t5);
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// The whole reduced matrix (reduction.cpp:33-49) under ReductionOptions{pivoting, workers}:
// reduce() for workers == 1 (reduction.cpp:129-131), reduce_parallel() otherwise
// (reduction.cpp:133-138) — the matrices acceptance.cpp:106-133 compares.  For every
// nonzero column j in order: cols[m] = j and its two rows lo[m] < hi[m] (any other support
// size is reported as an error: the reference's columns stay 2-sparse).  stats[3] =
// ReductionStats{additions, row_ops, probe_ops} (reduction.hpp:21-27).
int ref_reduced_matrix(const double* x, std::uint64_t n, std::uint64_t d, int pivoting,
                       unsigned workers, std::uint64_t* cols, std::uint32_t* lo,
                       std::uint32_t* hi, std::uint64_t* m, std::uint64_t* stats) {
    try {
        const ph0::Filtration f = ph0::build_filtration(ph0::pairwise_distances(make_cloud(x, n, d)));
        ph0::BoundaryMatrix mat = ph0::build_boundary_matrix(f, n);
        const ph0::ReductionOptions opts{pivoting != 0, workers};
        const ph0::ReductionStats st =
            workers > 1 ? ph0::reduce_parallel(mat, opts) : ph0::reduce(mat, opts);
        std::uint64_t k = 0;
        for (std::size_t j = 0; j < mat.columns.size(); ++j) {
            const ph0::BitVector& sup = mat.columns[j].support;
            if (!sup.any()) continue;
            if (sup.count() != 2) {
                g_err = "reduced column with support size " + std::to_string(sup.count());
                return 1;
            }
            const std::uint32_t t = sup.top();
            std::uint32_t b = 0;
            while (!sup.test(b)) ++b;
            cols[k] = j;
            lo[k] = b;
            hi[k] = t;
            ++k;
        }
        *m = k;
        if (stats) {
            stats[0] = st.additions;
            stats[1] = st.row_ops;
            stats[2] = st.probe_ops;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Text front-end of the reference CLI (ph0_cli.cpp:58-80, :199-205) without CLI11: the text a
// `compute`/`oracle` (mode 0/1) run prints for a point file's contents, or "error: <what>\n"
// (ph0_cli.cpp:278-281) with return 1; `generate` as write_points(generate_uniform_cloud).
// The output is copied into out[cap] (NUL-terminated); *len receives its full length.
static int put_text(const std::string& t, char* out, std::uint64_t cap, std::uint64_t* len) {
    if (len) *len = t.size();
    if (out && cap) {
        const std::size_t k = t.size() < cap - 1 ? t.size() : cap - 1;
        std::memcpy(out, t.data(), k);
        out[k] = 0;
    }
    return 0;
}

int ref_cli_text(const char* points_text, std::uint64_t gen_n, std::uint64_t gen_dim,
                 std::uint64_t gen_seed, int mode, int show_essential, char* out,
                 std::uint64_t cap, std::uint64_t* len) {
    try {
        ph0::PointCloud cloud = [&] {
            if (points_text) {
                std::istringstream in(points_text);
                return ph0::read_points(in);
            }
            return ph0::generate_uniform_cloud(gen_n, gen_dim, gen_seed);
        }();
        if (mode == 2) {
            std::ostringstream os;
            ph0::write_points(os, cloud);
            return put_text(os.str(), out, cap, len);
        }
        const ph0::Filtration f = ph0::build_filtration(ph0::pairwise_distances(cloud));
        ph0::Barcode bc;
        if (mode == 1) {
            bc = ph0::kruskal_barcode(f, static_cast<std::size_t>(cloud.size()));
        } else {
            ph0::BoundaryMatrix m = ph0::build_boundary_matrix(f, static_cast<std::size_t>(cloud.size()));
            ph0::reduce(m, ph0::ReductionOptions{true, 1});
            bc = ph0::extract_barcode(m, f);
        }
        return put_text(ph0::format_barcode(bc, show_essential != 0), out, cap, len);
    } catch (const std::exception& e) {
        put_text(std::string("error: ") + e.what() + "\n", out, cap, len);
        return 1;
    }
}

} // extern "C"

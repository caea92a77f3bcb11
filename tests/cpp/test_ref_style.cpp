// The reference's own hot-path unit tests (proj/tests/test_filtration.cpp, test_reduction.cpp,
// test_oracle.cpp, acceptance.cpp oracle-equivalence / bar-count-law), restated against the
// drop-in C++ adapter include/ph0b.hpp so they run on the B200 path.  Built and run by
// tests/test_cpp_gpu.py (pytest -m gpu).  Uses the doctest shim in oracle/shim.
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include <doctest.h>

#include <cmath>
#include <cstdint>
#include <numeric>
#include <vector>

#include "ph0b.hpp"

namespace {

struct Cloud {
    std::vector<double> x;  // column-major
    std::size_t n = 0, d = 0;
};

Cloud from_rows(std::initializer_list<std::initializer_list<double>> rows) {
    Cloud c;
    c.n = rows.size();
    c.d = rows.begin()->size();
    c.x.resize(c.n * c.d);
    std::size_t i = 0;
    for (const auto& r : rows) {
        std::size_t j = 0;
        for (double v : r) c.x[j++ * c.n + i] = v;
        ++i;
    }
    return c;
}

Cloud uniform(std::size_t n, std::size_t d, std::uint64_t seed) {
    Cloud c;
    c.n = n;
    c.d = d;
    c.x.resize(n * d);
    if (n) ph0b_generate_cloud(0, n, d, seed, 0, 0, 0, 1, 0, c.x.data());
    return c;
}

struct SplitMix64 {  // splitmix64.hpp:20-24
    std::uint64_t s;
    std::uint64_t next() {
        std::uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
};

// Kruskal on a filtration (oracle.cpp:32-46), for oracle-equivalence checks.
ph0b::Barcode kruskal(const ph0b::Filtration& f, std::size_t n) {
    ph0b::Barcode b;
    if (n == 0) return b;
    std::vector<std::uint32_t> p(n);
    std::iota(p.begin(), p.end(), 0u);
    auto find = [&](std::uint32_t x) {
        while (p[x] != x) x = p[x] = p[p[x]];
        return x;
    };
    std::size_t comps = n;
    for (const auto& e : f.edges) {
        std::uint32_t a = find(e.u), c = find(e.v);
        if (a == c) continue;
        p[a] = c;
        --comps;
        b.finite.push_back({0.0, e.grade, e.length});
        if (b.finite.size() == n - 1) break;
    }
    b.essential_count = comps;
    return b;
}

ph0b::Barcode barcode(const Cloud& c, std::vector<double>* scale = nullptr) {
    return ph0b::h0_barcode(c.x.data(), c.n, c.d, scale);
}

}  // namespace

TEST_CASE("3-4-5 right triangle gives the hypotenuse distance") {  // test_filtration.cpp:33-39
    const Cloud c = from_rows({{0, 0}, {3, 4}});
    const auto dists = ph0b::pairwise_distances(c.x.data(), c.n, c.d);
    REQUIRE(dists.size() == 1);
    CHECK(dists[0].u == 0);
    CHECK(dists[0].v == 1);
    CHECK(dists[0].length == 5.0);
}

TEST_CASE("collinear points give the expected lengths") {  // test_filtration.cpp:41-59
    const Cloud c = from_rows({{0, 0}, {1, 0}, {3, 0}});
    const ph0b::Filtration f = ph0b::build_filtration(c.x.data(), c.n, c.d);
    REQUIRE(f.edges.size() == 3);
    CHECK(f.edges[0].u == 0);
    CHECK(f.edges[0].v == 1);
    CHECK(f.edges[0].length == 1.0);
    CHECK(f.edges[0].grade == 1);
    CHECK(f.edges[1].u == 1);
    CHECK(f.edges[1].v == 2);
    CHECK(f.edges[1].grade == 2);
    CHECK(f.edges[2].u == 0);
    CHECK(f.edges[2].v == 2);
    CHECK(f.edges[2].length == 3.0);
    CHECK(f.scale == std::vector<double>{1.0, 2.0, 3.0});
}

TEST_CASE("duplicate lengths share a grade") {  // test_filtration.cpp:69-82
    const Cloud c = from_rows({{0.0}, {5.0}, {10.0}});
    const ph0b::Filtration f = ph0b::build_filtration(c.x.data(), c.n, c.d);
    REQUIRE(f.edges.size() == 3);
    CHECK(f.scale == std::vector<double>{5.0, 10.0});
    CHECK(f.edges[0].grade == 1);
    CHECK(f.edges[1].grade == 1);
    CHECK(f.edges[2].grade == 2);
    CHECK(f.edges[0].u == 0);
    CHECK(f.edges[0].v == 1);
    CHECK(f.edges[1].u == 1);
    CHECK(f.edges[1].v == 2);
}

TEST_CASE("filtration invariants hold on random clouds") {  // test_filtration.cpp:84-116
    SplitMix64 seeds{5150};
    for (int trial = 0; trial < 12; ++trial) {
        const std::size_t n = 2 + seeds.next() % 40;
        const std::size_t dim = 1 + seeds.next() % 3;
        const Cloud c = uniform(n, dim, seeds.next());
        const ph0b::Filtration f = ph0b::build_filtration(c.x.data(), c.n, c.d);
        CHECK(f.edges.size() == n * (n - 1) / 2);
        for (std::size_t i = 0; i + 1 < f.edges.size(); ++i) {
            CHECK(f.edges[i].length <= f.edges[i + 1].length);
            if (f.edges[i].length == f.edges[i + 1].length)
                CHECK((f.edges[i].u < f.edges[i + 1].u ||
                       (f.edges[i].u == f.edges[i + 1].u && f.edges[i].v < f.edges[i + 1].v)));
        }
        for (std::size_t i = 0; i + 1 < f.scale.size(); ++i) CHECK(f.scale[i] < f.scale[i + 1]);
        std::vector<bool> seen(f.scale.size(), false);
        for (const auto& e : f.edges) {
            REQUIRE(e.grade >= 1);
            REQUIRE(e.grade <= f.scale.size());
            CHECK(f.scale[e.grade - 1] == e.length);
            CHECK(e.u < e.v);
            CHECK(e.v < n);
            seen[e.grade - 1] = true;
        }
        for (const bool s : seen) CHECK(s);
    }
}

TEST_CASE("barcode of the collinear cloud") {  // test_reduction.cpp:105-113
    const ph0b::Barcode bc = barcode(from_rows({{0, 0}, {1, 0}, {3, 0}}));
    CHECK(ph0b::finite_death_lengths(bc) == std::vector<double>{1.0, 2.0});
    CHECK(ph0b::finite_death_grades(bc) == std::vector<std::uint64_t>{1, 2});
    CHECK(bc.essential_count == 1);
    const Cloud c = from_rows({{0, 0}, {1, 0}, {3, 0}});
    CHECK(ph0b::claimed_lows(c.x.data(), c.n, c.d) == std::vector<std::uint32_t>{1, 2});  // :76-93
}

TEST_CASE("barcode of the unit square") {  // test_reduction.cpp:115-123
    const ph0b::Barcode bc = barcode(from_rows({{0, 0}, {1, 0}, {0, 1}, {1, 1}}));
    CHECK(ph0b::finite_death_lengths(bc) == std::vector<double>{1.0, 1.0, 1.0});
    CHECK(bc.essential_count == 1);
}

TEST_CASE("barcode of two separated clusters") {  // test_reduction.cpp:125-134
    const ph0b::Barcode bc = barcode(from_rows({{0, 0}, {0.1, 0}, {10, 0}, {10.1, 0}}));
    CHECK(ph0b::finite_death_lengths(bc) ==
          std::vector<double>{std::min(0.1, 10.1 - 10.0), std::max(0.1, 10.1 - 10.0), 10.0 - 0.1});
}

TEST_CASE("coincident points produce zero-length bars") {  // test_reduction.cpp:136-145
    const ph0b::Barcode bc = barcode(from_rows({{1, 1}, {1, 1}, {2, 2}}));
    REQUIRE(bc.finite.size() == 2);
    CHECK(bc.finite[0].death_length == 0.0);
    CHECK(bc.finite[0].death_grade == 1);
}

TEST_CASE("degenerate barcodes") {  // test_reduction.cpp:147-157, acceptance.cpp:98-102
    const ph0b::Barcode bc0 = barcode(Cloud{{}, 0, 2});
    CHECK(bc0.finite.empty());
    CHECK(bc0.essential_count == 0);
    const ph0b::Barcode bc1 = barcode(from_rows({{1, 2}}));
    CHECK(bc1.finite.empty());
    CHECK(bc1.essential_count == 1);
}

TEST_CASE("survivors number N-1 with distinct claimed lows") {  // test_reduction.cpp:159-184
    SplitMix64 seeds{4242};
    for (int trial = 0; trial < 8; ++trial) {
        const std::size_t n = 2 + seeds.next() % 48;
        const Cloud c = uniform(n, 1 + seeds.next() % 3, seeds.next());
        const ph0b::Barcode bc = barcode(c);
        CHECK(bc.finite.size() == n - 1);
        auto lows = ph0b::claimed_lows(c.x.data(), c.n, c.d);
        std::sort(lows.begin(), lows.end());
        CHECK(std::adjacent_find(lows.begin(), lows.end()) == lows.end());
    }
}

TEST_CASE("reduced barcode equals the union-find oracle") {  // test_reduction.cpp:197-211
    SplitMix64 seeds{60601};
    for (int trial = 0; trial < 10; ++trial) {
        const std::size_t n = 2 + seeds.next() % 60;
        const std::size_t dim = 1 + seeds.next() % 3;
        const Cloud c = uniform(n, dim, seeds.next());
        const ph0b::Filtration f = ph0b::build_filtration(c.x.data(), c.n, c.d);
        const ph0b::Barcode ours = barcode(c);
        const ph0b::Barcode oracle = kruskal(f, n);
        CHECK(ph0b::finite_death_grades(ours) == ph0b::finite_death_grades(oracle));
        CHECK(ours.essential_count == oracle.essential_count);
    }
}

TEST_CASE("acceptance: oracle equivalence and bar-count law on 200 clouds") {  // acceptance.cpp:79-104
    for (int i = 0; i < 200; ++i) {
        const std::size_t n = 2 + i % 63, d = 1 + i % 3;
        const Cloud c = uniform(n, d, 0xACCE57ull + i);
        std::vector<double> scale;
        const ph0b::Barcode bc = barcode(c, &scale);
        const ph0b::Filtration f = ph0b::build_filtration(c.x.data(), c.n, c.d);
        const ph0b::Barcode oracle = kruskal(f, n);
        CHECK(ph0b::finite_death_grades(bc) == ph0b::finite_death_grades(oracle));
        const ph0b::Barcode gpu_oracle = ph0b::kruskal_barcode(c.x.data(), c.n, c.d);
        REQUIRE(gpu_oracle.finite.size() == bc.finite.size());
        for (std::size_t j = 0; j < bc.finite.size(); ++j) {  // ordered, not just multisets
            CHECK(gpu_oracle.finite[j].death_grade == bc.finite[j].death_grade);
            CHECK(gpu_oracle.finite[j].death_length == bc.finite[j].death_length);
        }
        CHECK(bc.finite.size() == n - 1);
        CHECK(bc.essential_count == 1);
        CHECK(scale == f.scale);
    }
}

TEST_CASE("drop-in adapter on a large cloud: D straight into a reused vector, multi-GPU") {
    // K = 7.2e7 >= 2^26: the bucketed path that streams D while sorting, written into the
    // caller's vector; a second call reuses its storage; virtual ranks on one GPU agree
    const Cloud c = uniform(12000, 3, 77);
    std::vector<double> scale;
    const ph0b::Barcode a = barcode(c, &scale);
    const std::vector<double> first = scale;
    const ph0b::Barcode b = barcode(c, &scale);
    CHECK(scale == first);
    REQUIRE(a.finite.size() == 11999);
    REQUIRE(b.finite.size() == a.finite.size());
    for (std::size_t j = 0; j < a.finite.size(); ++j) {
        CHECK(b.finite[j].death_grade == a.finite[j].death_grade);
        CHECK(scale[a.finite[j].death_grade - 1] == a.finite[j].death_length);
    }
    for (std::size_t i = 1; i < scale.size(); ++i) REQUIRE(scale[i - 1] < scale[i]);
    std::vector<double> scale2;
    const ph0b::Barcode m = ph0b::h0_barcode_multi(c.x.data(), c.n, c.d, {0, 0, 0}, &scale2);
    CHECK(scale2 == scale);
    REQUIRE(m.finite.size() == a.finite.size());
    for (std::size_t j = 0; j < a.finite.size(); ++j)
        CHECK(m.finite[j].death_grade == a.finite[j].death_grade);
}

TEST_CASE("errors mirror the reference's exceptions") {
    Cloud bad = from_rows({{1.0, 0.0}, {0.0, 0.0}});
    bad.x[1] = INFINITY;  // point_cloud.cpp:17
    CHECK_THROWS_WITH_AS(barcode(bad), doctest::Contains("non-finite coordinates"),
                         std::invalid_argument);
    ph0b::ReductionOptions r;
    r.workers = 0;  // reduction.cpp:134
    const Cloud c = from_rows({{0, 0}, {1, 1}});
    CHECK_THROWS_WITH_AS(ph0b::h0_barcode(c.x.data(), c.n, c.d, nullptr, r),
                         doctest::Contains("worker count must be at least 1"),
                         std::invalid_argument);
}

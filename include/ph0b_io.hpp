// ph0b_io.hpp — text formats either side of the hot path, header-only
// C++17.  Same formats and error texts as the reference's I/O so a front-end built on the
// B200 library prints byte-identical output:
//   format_double   — shortest round-trip decimal            (reference format.cpp:7-11)
//   format_barcode  — "0,<length>,<grade>" lines, essential "0,inf,-" (barcode.cpp:25-37)
//   read_points     — one point per line, ',' / blanks separate fields, '#' comment lines,
//                     ParseError naming the line                (point_cloud.cpp:50-91)
//   write_points    — comma-separated format_double per row     (point_cloud.cpp:99-107)
#pragma once

#include <charconv>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <istream>
#include <ostream>
#include <stdexcept>
#include <string>
#include <string_view>
#include <system_error>
#include <vector>

#include "ph0b.hpp"

namespace ph0b {

class ParseError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

// A point cloud as the reference's PointCloud stores it: n x d, column-major (Eigen).
struct Cloud {
    std::size_t n = 0, d = 0;
    std::vector<double> x;  // x[j * n + i] = coordinate j of point i
};

inline std::string format_double(double v) {
    char buf[32];
    const auto r = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, r.ptr);
}

inline std::string format_barcode(const Barcode& b, bool show_essential) {
    std::string out;
    for (const auto& iv : b.finite) {
        out += "0,";
        out += format_double(iv.death_length);
        out += ',';
        out += std::to_string(iv.death_grade);
        out += '\n';
    }
    if (show_essential)
        for (std::size_t i = 0; i < b.essential_count; ++i) out += "0,inf,-\n";
    return out;
}

namespace detail {
inline bool is_sep(char c) { return c == ',' || c == ' ' || c == '\t' || c == '\r'; }

inline bool parse_full_double(std::string_view tok, double& out) {
    if (tok.empty()) return false;
    const auto r = std::from_chars(tok.data(), tok.data() + tok.size(), out);
    return r.ec == std::errc{} && r.ptr == tok.data() + tok.size();
}
}  // namespace detail

inline Cloud read_points(std::istream& in) {
    std::vector<double> rows;  // row-major while reading
    std::size_t dim = 0, count = 0, line_no = 0;
    std::string line;
    std::vector<std::string_view> f;
    while (std::getline(in, line)) {
        ++line_no;
        f.clear();
        const std::string_view s(line);
        for (std::size_t i = 0; i < s.size();) {
            while (i < s.size() && detail::is_sep(s[i])) ++i;
            const std::size_t b = i;
            while (i < s.size() && !detail::is_sep(s[i])) ++i;
            if (i > b) f.push_back(s.substr(b, i - b));
        }
        if (f.empty() || f.front().front() == '#') continue;
        if (dim == 0)
            dim = f.size();
        else if (f.size() != dim)
            throw ParseError("line " + std::to_string(line_no) + ": expected " +
                             std::to_string(dim) + " coordinates, got " + std::to_string(f.size()));
        for (const auto tok : f) {
            double v = 0.0;
            if (!detail::parse_full_double(tok, v))
                throw ParseError("line " + std::to_string(line_no) + ": malformed number '" +
                                 std::string(tok) + "'");
            if (!std::isfinite(v))
                throw ParseError("line " + std::to_string(line_no) + ": non-finite coordinate '" +
                                 std::string(tok) + "'");
            rows.push_back(v);
        }
        ++count;
    }
    Cloud c;
    c.n = count;
    c.d = dim;
    c.x.resize(count * dim);
    for (std::size_t i = 0; i < count; ++i)
        for (std::size_t j = 0; j < dim; ++j) c.x[j * count + i] = rows[i * dim + j];
    return c;
}

inline Cloud read_points_file(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open point file '" + path + "'");
    return read_points(in);
}

inline void write_points(std::ostream& out, const Cloud& c) {
    for (std::size_t i = 0; i < c.n; ++i) {
        for (std::size_t j = 0; j < c.d; ++j) {
            if (j > 0) out << ',';
            out << format_double(c.x[j * c.n + i]);
        }
        out << '\n';
    }
}

// generate_uniform_cloud (point_cloud.cpp:20-29), host side (ph0b_generate_cloud kind 0).
inline Cloud generate_uniform_cloud(std::size_t n, std::size_t dim, std::uint64_t seed) {
    if (n > 0 && dim < 1) throw std::invalid_argument("point dimension must be at least 1");
    Cloud c;
    c.n = n;
    c.d = dim;
    c.x.resize(n * dim);
    if (n * dim) detail::check(ph0b_generate_cloud(0, n, dim, seed, 0, 0, 0, 0, 0, c.x.data()));
    return c;
}

}  // namespace ph0b

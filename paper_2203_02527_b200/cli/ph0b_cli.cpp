// ph0b — command-line front-end over the B200 library, option- and output-compatible with the
// reference's `ph0` CLI for the subcommands on the hot path (/root/reference/proj/tools/
// ph0_cli.cpp:111-283): `generate`, `compute` (column reduction, run_compute :58-71) and
// `oracle` (union-find, run_oracle :73-80).  Output text is byte-identical (format_barcode,
// write_points); errors print "error: <what>" and exit 1 (:278-281).  The reference's `bench`
// and `model` subcommands drive its CPU harness and cost model, which are out of scope here.
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ph0b_io.hpp"

namespace {

struct Args {
    std::map<std::string, std::string> opt;
    std::map<std::string, bool> flag;
};

// --name value | --name=value; flags take no value.
Args parse_args(int argc, char** argv, int first, const std::vector<std::string>& options,
                const std::vector<std::string>& flags) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string t = argv[i];
        std::string val;
        bool has_val = false;
        const auto eq = t.find('=');
        if (t.rfind("--", 0) == 0 && eq != std::string::npos) {
            val = t.substr(eq + 1);
            t = t.substr(0, eq);
            has_val = true;
        }
        bool known = false;
        for (const auto& f : flags)
            if (t == f) {
                if (has_val) throw std::invalid_argument(t + ": flag takes no value");
                a.flag[t] = true;
                known = true;
            }
        for (const auto& o : options)
            if (t == o) {
                if (!has_val) {
                    if (i + 1 >= argc) throw std::invalid_argument(t + " requires an argument");
                    val = argv[++i];
                }
                a.opt[t] = val;
                known = true;
            }
        if (!known) throw std::invalid_argument("The following argument was not expected: " + t);
    }
    return a;
}

std::uint64_t to_u64(const std::string& name, const std::string& s) {
    std::uint64_t v = 0;
    const auto r = std::from_chars(s.data(), s.data() + s.size(), v);
    if (r.ec != std::errc{} || r.ptr != s.data() + s.size())
        throw std::invalid_argument(name + ": value " + s + " is not a non-negative integer");
    return v;
}

std::string get(const Args& a, const std::string& k, const std::string& def) {
    const auto it = a.opt.find(k);
    return it == a.opt.end() ? def : it->second;
}

void write_output(const std::string& path, const std::string& content) {
    if (path == "-") {
        std::cout << content;
        return;
    }
    std::ofstream out(path);
    if (!out) throw std::runtime_error("cannot open output file '" + path + "'");
    out << content;
}

ph0b::Cloud load_cloud(const Args& a) {
    const std::string in = get(a, "--in", "");
    if (!in.empty()) return ph0b::read_points_file(in);
    if (!a.opt.count("--n")) throw std::runtime_error("either --in or --n is required");
    return ph0b::generate_uniform_cloud(to_u64("--n", get(a, "--n", "0")),
                                        to_u64("--dim", get(a, "--dim", "2")),
                                        to_u64("--seed", get(a, "--seed", "1")));
}

int usage() {
    std::cerr << "usage: ph0b {generate|compute|oracle} [options]\n"
                 "  generate --n N [--dim 2] [--seed 1] [--out -]\n"
                 "  compute  (--in FILE | --n N [--dim 2] [--seed 1]) [--workers 1]"
                 " [--pivot on|off] [--gpus 1] [--show-essential] [--out -]\n"
                 "  oracle   (--in FILE | --n N [--dim 2] [--seed 1]) [--show-essential]"
                 " [--out -]\n";
    return 109;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        if (cmd == "generate") {
            const Args a = parse_args(argc, argv, 2, {"--n", "--dim", "--seed", "--out"}, {});
            if (!a.opt.count("--n")) throw std::invalid_argument("--n is required");
            const ph0b::Cloud c = ph0b::generate_uniform_cloud(
                to_u64("--n", get(a, "--n", "0")), to_u64("--dim", get(a, "--dim", "2")),
                to_u64("--seed", get(a, "--seed", "1")));
            std::ostringstream os;
            ph0b::write_points(os, c);
            write_output(get(a, "--out", "-"), os.str());
            return 0;
        }
        if (cmd == "compute") {
            const Args a = parse_args(argc, argv, 2,
                                      {"--in", "--n", "--dim", "--seed", "--workers", "--pivot",
                                       "--gpus", "--out"},
                                      {"--show-essential"});
            const std::string pivot = get(a, "--pivot", "on");
            if (pivot != "on" && pivot != "off")
                throw std::invalid_argument("--pivot: " + pivot + " not in {on,off}");
            // run_compute calls reduce_parallel only for workers > 1 (ph0_cli.cpp:63-66), so
            // 0 and 1 both mean the sequential reduction; the result is identical anyway.
            const std::uint64_t workers = to_u64("--workers", get(a, "--workers", "1"));
            const ph0b::Cloud c = load_cloud(a);
            const ph0b::ReductionOptions ro{pivot == "on", (unsigned)(workers > 1 ? workers : 1)};
            // --gpus G (not in the reference CLI): the same bars on GPUs 0..G-1 of this node
            const std::uint64_t gpus = to_u64("--gpus", get(a, "--gpus", "1"));
            std::vector<std::int32_t> devs;
            for (std::uint64_t g = 0; g < gpus; ++g) devs.push_back((std::int32_t)g);
            const ph0b::Barcode bc =
                gpus > 1 ? ph0b::h0_barcode_multi(c.x.data(), c.n, c.d, devs, nullptr, ro)
                         : ph0b::h0_barcode(c.x.data(), c.n, c.d, nullptr, ro);
            write_output(get(a, "--out", "-"),
                         ph0b::format_barcode(bc, a.flag.count("--show-essential") > 0));
            return 0;
        }
        if (cmd == "oracle") {
            const Args a = parse_args(argc, argv, 2, {"--in", "--n", "--dim", "--seed", "--out"},
                                      {"--show-essential"});
            const ph0b::Cloud c = load_cloud(a);
            const ph0b::Barcode bc = ph0b::kruskal_barcode(c.x.data(), c.n, c.d);
            write_output(get(a, "--out", "-"),
                         ph0b::format_barcode(bc, a.flag.count("--show-essential") > 0));
            return 0;
        }
        if (cmd == "bench" || cmd == "model") {
            std::cerr << "error: '" << cmd
                      << "' drives the reference's CPU harness/cost model; use bench.py\n";
            return 1;
        }
        return usage();
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    }
}

// Synthetic point clouds of the BASELINE.json configs.  Host-side input
// generation only (not part of the measured path).  All randomness is SplitMix64
// (/root/reference/proj/include/ph0/splitmix64.hpp:20-43); kind 0 reproduces
// generate_uniform_cloud (proj/src/point_cloud.cpp:20-29) bit for bit.
#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/ph0b.h"

namespace {

struct SplitMix64 {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double unit_open() {
        for (;;) {
            const uint64_t top = next() >> 11;
            if (top != 0) return static_cast<double>(top) * 0x1.0p-53;
        }
    }
    // Box–Muller on two open-interval uniforms (cosine branch only).
    double normal() {
        const double u1 = unit_open(), u2 = unit_open();
        return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586 * u2);
    }
};

}  // namespace

extern "C" int ph0b_generate_cloud(uint32_t kind, uint64_t n, uint64_t d, uint64_t seed,
                                   uint32_t clusters, double sigma, double lo, double hi,
                                   uint64_t n_background, double* out) {
    if (n > 0 && d < 1) return PH0B_ERR_INVALID_ARGUMENT;
    if (n > 0 && !out) return PH0B_ERR_INVALID_ARGUMENT;
    SplitMix64 g{seed};
    auto at = [&](uint64_t i, uint64_t j) -> double& { return out[j * n + i]; };
    switch (kind) {
        case 0:  // generate_uniform_cloud: point by point, coordinate by coordinate
            for (uint64_t i = 0; i < n; ++i)
                for (uint64_t j = 0; j < d; ++j) at(i, j) = g.unit_open();
            return PH0B_OK;
        case 1: {  // Gaussian mixture, centres U[lo,hi]^d, label = next() % clusters
            if (clusters == 0) return PH0B_ERR_INVALID_ARGUMENT;
            std::vector<double> c(clusters * d);
            for (uint64_t k = 0; k < clusters; ++k)
                for (uint64_t j = 0; j < d; ++j) c[k * d + j] = lo + (hi - lo) * g.unit_open();
            for (uint64_t i = 0; i < n; ++i) {
                const uint64_t k = g.next() % clusters;
                for (uint64_t j = 0; j < d; ++j) at(i, j) = c[k * d + j] + sigma * g.normal();
            }
            return PH0B_OK;
        }
        case 2: {  // noisy unit circle in the z = 0 plane + uniform background cube
            if (n_background > n) return PH0B_ERR_INVALID_ARGUMENT;
            const uint64_t ring = n - n_background;
            for (uint64_t i = 0; i < ring; ++i) {
                const double th = 6.283185307179586 * g.unit_open();
                for (uint64_t j = 0; j < d; ++j) {
                    const double base = j == 0 ? std::cos(th) : (j == 1 ? std::sin(th) : 0.0);
                    at(i, j) = base + sigma * g.normal();
                }
            }
            for (uint64_t i = ring; i < n; ++i)
                for (uint64_t j = 0; j < d; ++j) at(i, j) = lo + (hi - lo) * g.unit_open();
            return PH0B_OK;
        }
        case 3: {  // two equal Gaussian clusters centred at lo*1 and hi*1 (config C1)
            for (uint64_t i = 0; i < n; ++i) {
                const double centre = (i < n / 2) ? lo : hi;
                for (uint64_t j = 0; j < d; ++j) at(i, j) = centre + sigma * g.normal();
            }
            return PH0B_OK;
        }
        default:
            return PH0B_ERR_INVALID_ARGUMENT;
    }
}

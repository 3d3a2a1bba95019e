// Seeded synthetic inputs for the BASELINE.json configurations
// (SURVEY.md section 8d).  Host code: these are the "user callbacks" a
// reference user would write (std::sin/std::cos, std::mt19937_64), evaluated
// once on the host like the reference evaluates its Potential callback
// (proj/src/scheme.cpp:158).
#include <cmath>
#include <cstdint>
#include <numbers>
#include <random>
#include <thread>
#include <vector>

#include "../../../include/laxol_b200_configs.h"

namespace {
constexpr double kTwoPi = 2.0 * std::numbers::pi;
inline double xcoord(int64_t j, int64_t n) {
    // GridFn::coord: origin + i*step with step = 1/n (proj/include/laxol/grid_fn.hpp:21)
    return static_cast<double>(j) * (1.0 / static_cast<double>(n));
}
}  // namespace

extern "C" {

void lob_gen_sin(int64_t n, double* u0) {
    for (int64_t j = 0; j < n; ++j) u0[j] = std::sin(kTwoPi * xcoord(j, n));
}

void lob_gen_cos(int64_t n, double* a) {
    for (int64_t j = 0; j < n; ++j) a[j] = std::cos(kTwoPi * xcoord(j, n));
}

double lob_c4_time_term(double t) { return 0.2 * std::sin(kTwoPi * t); }

void lob_gen_potential(int kind, int64_t n, double* v) {
    for (int64_t j = 0; j < n; ++j) {
        const double x = xcoord(j, n);
        switch (kind) {
            case 1:
                v[j] = std::cos(kTwoPi * x);
                break;
            case 2:
                v[j] = std::cos(kTwoPi * x) + 0.5 * std::cos(2.0 * kTwoPi * x + 1.0);
                break;
            case 3:
                v[j] = 0.5 * std::sin(kTwoPi * x);
                break;
            default:
                v[j] = 0.0;
        }
    }
}

void lob_gen_c2_drifts(int64_t lines, double* drift) {
    for (int64_t l = 0; l < lines; ++l)
        drift[l] = -2.0 + 4.0 * static_cast<double>(l) / 255.0;
}

void lob_gen_c3_lines(int64_t line0, int64_t lines, int64_t n, uint64_t seed0, double* u) {
    std::vector<double> w(static_cast<size_t>(n + 1));
    const double dx = 1.0 / static_cast<double>(n);
    for (int64_t l = 0; l < lines; ++l) {
        std::mt19937_64 rng(seed0 + static_cast<uint64_t>(line0 + l));
        std::uniform_real_distribution<double> inc(-dx, dx);
        w[0] = 0.0;
        for (int64_t i = 0; i < n; ++i) w[i + 1] = w[i] + inc(rng);
        double* ul = u + l * n;
        for (int64_t i = 0; i < n; ++i)
            ul[i] = w[i] - w[n] * static_cast<double>(i) / static_cast<double>(n);
    }
}

void lob_gen_c4_u0(int64_t n, double* u) {
    for (int64_t i = 0; i < n; ++i) {
        const double s = std::sin(kTwoPi * xcoord(i, n));
        for (int64_t k = 0; k < n; ++k) u[i * n + k] = s + std::cos(kTwoPi * xcoord(k, n));
    }
}

void lob_gen_c5_lines(int64_t line0, int64_t lines, int64_t n, uint64_t seed0, double* u,
                      int nthreads) {
    auto one = [&](int64_t l) {
        std::mt19937_64 rng(seed0 + static_cast<uint64_t>(line0 + l));
        std::uniform_int_distribution<int> kd(1, 256);
        std::uniform_real_distribution<double> pd(0.0, kTwoPi);
        int k[64];
        double phi[64];
        for (int m = 0; m < 64; ++m) {
            k[m] = kd(rng);
            phi[m] = pd(rng);
        }
        double* ul = u + l * n;
        for (int64_t j = 0; j < n; ++j) {
            const double x = xcoord(j, n);
            double acc = 0.0;
            for (int m = 0; m < 64; ++m)
                acc += std::sin(kTwoPi * static_cast<double>(k[m]) * x + phi[m]) /
                       static_cast<double>(k[m] * k[m]);
            ul[j] = acc;
        }
    };
    const int nt = nthreads < 1 ? 1 : nthreads;
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (int64_t l = t; l < lines; l += nt) one(l);
        });
    for (auto& th : pool) th.join();
}

}  // extern "C"

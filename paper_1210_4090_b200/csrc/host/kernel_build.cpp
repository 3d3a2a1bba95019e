// Host-side kernel-window construction, restating build_kernel for the
// mechanical conjugate (proj/src/scheme.cpp:59-105 with
// proj/src/hamiltonian.cpp:42-44) so the device path sees the identical
// table, plus the fast engine's slope-inversion tolerance.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "laxol_b200.hpp"

namespace laxol_b200 {

namespace {
KernelWindow mech_window(int64_t n_space, double tau, double drift);
}

KernelWindow build_kernel_mech(int64_t n_space, double tau, double drift) {
    if (n_space < 1) throw InvalidInput("SchemeParams: n_space must be >= 1");
    if (!(tau > 0.0)) throw InvalidInput("SchemeParams: tau must be positive");
    const double eps = 1.0 / static_cast<double>(n_space);
    if (eps / tau >= 1.0)
        throw InvalidInput("SchemeParams: epsilon/tau = " + std::to_string(eps / tau) +
                           " violates the bound epsilon/tau < h0 = 1");
    return mech_window(n_space, tau, drift);
}

KernelWindow build_kernel_mech(const SchemeParams& params, double drift) {
    validate(params);  // the guard with the params' h0 and anti-CFL mode
    return mech_window(params.n_space, params.tau, drift);
}

namespace {
KernelWindow mech_window(int64_t n_space, double tau, double drift) {
    const double eps = 1.0 / static_cast<double>(n_space);
    KernelWindow k;
    k.n_space = n_space;
    k.tau = tau;
    k.drift = drift;
    const int64_t center = std::llround(tau * drift / eps);
    k.first = center - n_space;
    k.center_index = center;
    const int64_t m = 2 * n_space + 1;
    k.window.resize(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) {
        const double x = static_cast<double>(k.first + i) * eps;
        const double v = x / tau;
        k.window[static_cast<size_t>(i)] = tau * (0.5 * v * v - drift * v);
    }
    for (int64_t i = 0; i + 2 < m; ++i) {
        const double lo = k.window[i + 1] - k.window[i];
        const double hi = k.window[i + 2] - k.window[i + 1];
        if (hi < lo)
            throw InvalidInput("build_kernel: sampled window is not convex at segment " +
                               std::to_string(i + 1));
    }
    int64_t arg = 0;
    for (int64_t i = 1; i < m; ++i)
        if (k.window[i] < k.window[arg]) arg = i;
    k.argmin_index = arg;
    k.delta = fast_delta(n_space, tau, drift, k.first);
    return k;
}
}  // namespace

// build_kernel for a tabulated conjugate (proj/src/hamiltonian.cpp:30-82 kstar /
// argmin_velocity / v_min / v_max of Kind::Tabulated, proj/src/scheme.cpp:59-105 incl.
// the monotone slope repair), the same IEEE operations in the same order.
KernelWindow build_kernel_tab(int64_t n_space, double tau, const std::vector<double>& samples, double v0,
                              double dv) {
    if (samples.size() < 2) throw InvalidInput("tabulated: need at least two samples");
    if (!(dv > 0.0)) throw InvalidInput("tabulated: step must be positive");
    for (double x : samples)
        if (!std::isfinite(x)) throw InvalidInput("tabulated: non-finite sample");
    const std::size_t tn = samples.size() - 1;
    for (std::size_t i = 0; i + 2 < samples.size(); ++i) {
        const double lo = samples[i + 1] - samples[i];
        const double hi = samples[i + 2] - samples[i + 1];
        if (hi < lo)
            throw InvalidInput("tabulated: samples are not convex, slope drops at segment " + std::to_string(i + 1));
    }
    if (n_space < 1) throw InvalidInput("SchemeParams: n_space must be >= 1");
    if (!(tau > 0.0)) throw InvalidInput("SchemeParams: tau must be positive");
    const double eps = 1.0 / static_cast<double>(n_space);
    if (eps / tau >= 1.0)
        throw InvalidInput("SchemeParams: epsilon/tau = " + std::to_string(eps / tau) +
                           " violates the bound epsilon/tau < h0 = 1");
    auto coord = [&](std::size_t i) { return v0 + static_cast<double>(i) * dv; };
    // argmin_velocity
    std::size_t lo = 0;
    for (std::size_t i = 1; i < samples.size(); ++i)
        if (samples[i] < samples[lo]) lo = i;
    std::size_t hi = lo;
    while (hi + 1 < samples.size() && samples[hi + 1] == samples[lo]) ++hi;
    const double vstar = coord(lo) + 0.5 * static_cast<double>(hi - lo) * dv;
    KernelWindow k;
    k.n_space = n_space;
    k.tau = tau;
    k.drift = vstar;
    k.mechanical = false;
    const int64_t center = std::llround(tau * vstar / eps);
    k.first = center - n_space;
    k.center_index = center;
    const double vmin = v0, vmax = coord(tn);
    const double v_lo = static_cast<double>(k.first) * eps / tau;
    const double v_hi = static_cast<double>(k.first + 2 * n_space) * eps / tau;
    if (v_lo < vmin || v_hi > vmax)
        throw InvalidInput("build_kernel: tabulated velocity window too narrow for the kernel support");
    const int64_t m = 2 * n_space + 1;
    k.window.resize(static_cast<size_t>(m));
    for (int64_t i = 0; i < m; ++i) {
        const double x = static_cast<double>(k.first + i) * eps;
        const double v = x / tau;
        // kstar: linear interpolation inside the table
        const double pos = (v - vmin) / dv;
        std::size_t j = static_cast<std::size_t>(pos);
        if (j >= tn) j = tn - 1;
        const double frac = pos - static_cast<double>(j);
        k.window[static_cast<size_t>(i)] = tau * (samples[j] + frac * (samples[j + 1] - samples[j]));
    }
    // monotone repair of rounding-level slope wiggles, values rebuilt from the slopes
    std::vector<double> sl(k.window.size() - 1);
    for (std::size_t i = 0; i + 1 < k.window.size(); ++i) sl[i] = k.window[i + 1] - k.window[i];
    for (std::size_t i = 1; i < sl.size(); ++i) sl[i] = std::max(sl[i], sl[i - 1]);
    for (std::size_t i = 0; i + 1 < k.window.size(); ++i) k.window[i + 1] = k.window[i] + sl[i];
    for (int64_t i = 0; i + 2 < m; ++i) {
        const double a = k.window[i + 1] - k.window[i];
        const double b = k.window[i + 2] - k.window[i + 1];
        if (b < a)
            throw InvalidInput("build_kernel: sampled window is not convex at segment " + std::to_string(i + 1));
    }
    int64_t arg = 0;
    for (int64_t i = 1; i < m; ++i)
        if (k.window[i] < k.window[arg]) arg = i;
    k.argmin_index = arg;
    return k;
}

// Tolerance (in displacement units) of the fast engine's slope inversion
// d(s) = (s + drift*eps)/a - 1/2 against the rounded table: bound on the
// table's slope error (each K value carries <= 6 ulp of its magnitude) plus
// the rounding of the inversion itself.  See DESIGN.md "K2".
double fast_delta(int64_t n_space, double tau, double drift, int64_t first) {
    const double u = std::ldexp(1.0, -53);
    const double eps = 1.0 / static_cast<double>(n_space);
    const double a = eps * eps / tau;
    const double dmax = std::fmax(std::fabs(static_cast<double>(first)),
                                  std::fabs(static_cast<double>(first + 2 * n_space)));
    const double vmax = dmax * eps / tau;
    const double kmag = tau * (0.5 * vmax * vmax + std::fabs(drift) * vmax);
    return 32.0 * u * kmag / a + 8.0 * u * (2.0 * n_space + std::fabs(drift) * eps / a) + 1e-9;
}

}  // namespace laxol_b200

extern "C" int lob_kernel_mech_host(lob_ctx*, int64_t n, double tau, double drift,
                                    double* window, int64_t* first, int64_t* argmin,
                                    double* delta) {
    try {
        const laxol_b200::KernelWindow k = laxol_b200::build_kernel_mech(n, tau, drift);
        if (window) std::memcpy(window, k.window.data(), k.window.size() * sizeof(double));
        if (first) *first = k.first;
        if (argmin) *argmin = k.argmin_index;
        if (delta) *delta = k.delta;
        return LOB_OK;
    } catch (const laxol_b200::InvalidInput&) {
        return LOB_INVALID_INPUT;
    }
}

extern "C" int lob_kernel_tabulated_host(lob_ctx*, int64_t n, double tau, const double* samples, int64_t count,
                                         double v0, double dv, double* window, int64_t* first, int64_t* argmin) {
    try {
        if (!samples || count < 0) return LOB_INVALID_INPUT;
        const laxol_b200::KernelWindow k = laxol_b200::build_kernel_tab(
            n, tau, std::vector<double>(samples, samples + count), v0, dv);
        if (window) std::memcpy(window, k.window.data(), k.window.size() * sizeof(double));
        if (first) *first = k.first;
        if (argmin) *argmin = k.argmin_index;
        return LOB_OK;
    } catch (const laxol_b200::InvalidInput&) {
        return LOB_INVALID_INPUT;
    }
}

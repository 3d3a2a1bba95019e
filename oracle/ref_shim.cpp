// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// extern "C" shim over the UNMODIFIED reference library (laxol, compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/).  It lets the
// Python tests, the golden-fixture generator and bench.py's reference arm call
// the reference's own C++ stepping API:
//   build_kernel            proj/src/scheme.cpp:59-105
//   kinetic_convolve        proj/src/scheme.cpp:107-146   (engine switch :114-121)
//   step_fully_discrete     proj/src/scheme.cpp:148-164
//   evolve                  proj/src/scheme.cpp:208-272
//   split_step_nd           proj/src/splitting.cpp:37-99
//   decompose / conv_*      proj/src/minplus.cpp
// Status codes follow include/laxol_b200.h: 0 ok, 1 InvalidInput,
// 2 EvaluationError, 4 other.
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "laxol/errors.hpp"
#include "laxol/minplus.hpp"
#include "laxol/parallel.hpp"
#include "laxol/scheme.hpp"
#include "laxol/splitting.hpp"
#include "laxol/weakkam.hpp"

using namespace laxol;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const InvalidInput& e) {
        g_err = e.what();
        return 1;
    } catch (const EvaluationError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

SchemeParams params_of(int n_space, double tau, double eta) {
    SchemeParams p;
    p.n_space = n_space;
    p.tau = tau;
    p.eta = eta;
    return p;
}

// Potential given as a table over the fundamental grid (time independent):
// the callback maps x = j*eps back to j.  Exact for the grids used here.
Potential table_potential(const double* vtab, int n) {
    if (!vtab) return potential_zero();
    std::vector<double> tab(vtab, vtab + n);
    const double step = 1.0 / static_cast<double>(n);
    return potential_custom(
        [tab, n, step](double, double x) {
            long long j = std::llround(x / step);
            j = ((j % n) + n) % n;
            return tab[static_cast<std::size_t>(j)];
        },
        1e300, false);
}

// Time-dependent tabulated potential for the weak-KAM entry points:
// V(t, x_j) = tabs[(llround(t/tau) mod nt)][j] (nt tables of n values; nt == 0: V == 0,
// nt == 1: autonomous).  With Arrival sampling step i of a period samples table (i+1) mod nt.
Potential time_table_potential(const double* tabs, int64_t nt, int n, double tau) {
    if (!tabs || nt == 0) return potential_zero();
    if (nt == 1) return table_potential(tabs, n);
    std::vector<double> tab(tabs, tabs + nt * n);
    const double step = 1.0 / static_cast<double>(n);
    return potential_custom(
        [tab, n, nt, step, tau](double t, double x) {
            long long j = std::llround(x / step);
            j = ((j % n) + n) % n;
            long long k = std::llround(t / tau);
            k = ((k % nt) + nt) % nt;
            return tab[static_cast<std::size_t>(k * n + j)];
        },
        1e300, true);
}

MinPlusMatrix matrix_of(const double* a, int64_t n) {
    MinPlusMatrix m;
    m.n = static_cast<std::size_t>(n);
    m.cost.assign(a, a + n * n);
    return m;
}

ConvEngine engine_of(int e) { return e == 1 ? ConvEngine::Naive : ConvEngine::Fast; }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_set_max_threads(int n) { set_max_threads(n); }

// Kernel window (2n+1 samples) of mechanical(drift).
int ref_kernel_mech(int n_space, double tau, double drift, double* window, int64_t* center,
                    int64_t* argmin) {
    return guarded([&] {
        const Kernel k = build_kernel(mechanical(drift), params_of(n_space, tau, 0.0));
        std::memcpy(window, k.window.values.data(), k.window.values.size() * sizeof(double));
        if (center) *center = k.center_index;
        if (argmin) *argmin = k.argmin_index;
    });
}

// kinetic_convolve on a periodic u given by its fundamental domain (n_space
// samples) or, when periodic == 0, a windowed u of n_samples samples.
// out receives n_space (periodic, seam dropped) or n_samples values.
int ref_kinetic_convolve(const double* u, int64_t n_samples, int periodic, int n_space, double tau,
                         double drift, double eta, int engine, double* out, int64_t* blocks) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, eta);
        const Kernel k = build_kernel(mechanical(drift), p);
        GridFn g = periodic ? make_periodic(std::vector<double>(u, u + n_space), p.epsilon())
                            : make_grid_fn(std::vector<double>(u, u + n_samples), p.epsilon(), 0.0);
        const GridFn r = kinetic_convolve(g, k, eta, engine_of(engine), blocks);
        const std::size_t m = periodic ? static_cast<std::size_t>(n_space) : r.values.size();
        std::memcpy(out, r.values.data(), m * sizeof(double));
    });
}

// One step_fully_discrete of `lines` independent periodic lines (fundamental
// domains, row-major lines x n_space), per-line drift, shared tabulated V,
// a std::thread pool over lines (the reference has no batched entry point).
int ref_step_lines(const double* u, int64_t lines, int n_space, double tau, const double* drifts,
                   const double* vtab, double t, double eta, int engine, int nthreads, double* out,
                   int64_t* blocks) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, eta);
        const Potential pot = table_potential(vtab, n_space);
        std::atomic<int64_t> next{0};
        std::atomic<int> status{0};
        std::string err;
        auto worker = [&] {
            for (;;) {
                const int64_t l = next.fetch_add(1);
                if (l >= lines) return;
                try {
                    const HamiltonianSpec spec{mechanical(drifts[l]), pot, true, true};
                    const Kernel k = build_kernel(spec, p);
                    const double* ul = u + l * n_space;
                    GridFn g = make_periodic(std::vector<double>(ul, ul + n_space), p.epsilon());
                    StepStats st;  // requested only with a blocks buffer (the API default is none)
                    GridFn r = step_fully_discrete(g, t, spec, p, k, engine_of(engine), blocks ? &st : nullptr);
                    std::memcpy(out + l * n_space, r.values.data(), n_space * sizeof(double));
                    if (blocks) blocks[l] = st.block_count;
                } catch (const std::exception& e) {
                    status.store(dynamic_cast<const InvalidInput*>(&e) ? 1 : 2);
                    err = e.what();
                }
            }
        };
        const int nt = nthreads < 1 ? 1 : nthreads;
        std::vector<std::thread> pool;
        for (int i = 1; i < nt; ++i) pool.emplace_back(worker);
        worker();
        for (auto& th : pool) th.join();
        if (status.load() == 1) throw InvalidInput(err);
        if (status.load() == 2) throw EvaluationError(err);
    });
}

// evolve() of one periodic line; returns the final fundamental-domain state,
// per-step drifts and block counts, completion flag.
int ref_evolve(const double* u0, int n_space, double tau, double drift, const double* vtab,
               double t0, int64_t steps, double eta, int engine, double* u_final,
               double* step_drift, int64_t* step_blocks, int* completed) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, eta);
        const HamiltonianSpec spec{mechanical(drift), table_potential(vtab, n_space), true, true};
        GridFn g = make_periodic(std::vector<double>(u0, u0 + n_space), p.epsilon());
        EvolveOptions opt;
        opt.engine = engine_of(engine);
        opt.snapshot_stride = steps > 0 ? steps : 1;
        const EvolutionTrace tr = evolve(g, t0, steps, spec, p, opt);
        std::memcpy(u_final, tr.snapshots.back().values.data(), n_space * sizeof(double));
        for (std::size_t i = 0; i < tr.per_step.size(); ++i) {
            if (step_drift) step_drift[i] = tr.per_step[i].drift;
            if (step_blocks) step_blocks[i] = tr.per_step[i].blocks;
        }
        if (completed) *completed = tr.completed ? 1 : 0;
    });
}

// split_step_nd on an n1 x n2 periodic tensor with mechanical(d1), mechanical(d2).
// pot_kind 0: V == 0; 1: V = cos(2 pi x1) cos(2 pi x2) + 0.2 sin(2 pi t) (config C4);
// 2: V = x1 + 2 x2 (proj/tests/unit_splitting.cpp:171-194).
int ref_split_step_2d(const double* u, int64_t n1, int64_t n2, int n_space, double tau, double d1,
                      double d2, int pot_kind, double t, int periodic, double* out) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, 0.0);
        const TensorFn tu = make_tensor(std::vector<double>(u, u + n1 * n2),
                                        {static_cast<std::size_t>(n1), static_cast<std::size_t>(n2)},
                                        p.epsilon(), {0.0, 0.0}, periodic != 0);
        SplitSpec spec;
        spec.kinetics = {mechanical(d1), mechanical(d2)};
        constexpr double kTwoPi = 2.0 * std::numbers::pi;
        if (pot_kind == 1)
            spec.potential = [](double tt, std::span<const double> x) {
                return std::cos(kTwoPi * x[0]) * std::cos(kTwoPi * x[1]) +
                       0.2 * std::sin(kTwoPi * tt);
            };
        else if (pot_kind == 2)
            spec.potential = [](double, std::span<const double> x) { return x[0] + 2.0 * x[1]; };
        const TensorFn r = split_step_nd(tu, t, spec, p);
        std::memcpy(out, r.values.data(), r.values.size() * sizeof(double));
    });
}

// decompose(u, eta) of a plain (non-periodic) sample vector; returns the block
// count, and fills kinds/starts/ends up to cap entries.
int64_t ref_decompose(const double* v, int64_t n_samples, double eta, int* kinds, int64_t* starts,
                      int64_t* ends, int64_t cap) {
    int64_t count = -1;
    const int st = guarded([&] {
        const BlockDecomposition d =
            decompose(make_grid_fn(std::vector<double>(v, v + n_samples), 1.0), eta);
        count = static_cast<int64_t>(d.blocks.size());
        for (int64_t i = 0; i < count && i < cap; ++i) {
            if (kinds) kinds[i] = d.blocks[i].kind == BlockKind::Convex ? 0 : 1;
            if (starts) starts[i] = static_cast<int64_t>(d.blocks[i].start);
            if (ends) ends[i] = static_cast<int64_t>(d.blocks[i].end);
        }
    });
    return st == 0 ? count : -1;
}

// Plain-sample convolutions (step 1.0): which 0 naive, 1 convex*convex,
// 2 convex*concave, 3 conv_fast(eta).  out has na + nb - 1 entries.
int ref_conv(int which, const double* a, int64_t na, const double* b, int64_t nb, double eta,
             double* out, int64_t* blocks) {
    return guarded([&] {
        const GridFn f = make_grid_fn(std::vector<double>(a, a + na), 1.0);
        const GridFn g = make_grid_fn(std::vector<double>(b, b + nb), 1.0);
        GridFn r;
        if (which == 0)
            r = conv_naive(f, g);
        else if (which == 1)
            r = conv_convex_convex(f, g);
        else if (which == 2)
            r = conv_convex_concave(f, g);
        else {
            FastConvResult fr = conv_fast(f, g, eta);
            if (blocks) *blocks = fr.block_count;
            r = std::move(fr.fn);
        }
        std::memcpy(out, r.values.data(), r.values.size() * sizeof(double));
    });
}

// ---- weak-KAM consumers (proj/src/weakkam.cpp) ----
int ref_minplus_product(const double* a, const double* b, int64_t n, double* c) {
    return guarded([&] {
        const MinPlusMatrix r = minplus_product(matrix_of(a, n), matrix_of(b, n));
        std::memcpy(c, r.cost.data(), n * n * sizeof(double));
    });
}

int ref_minplus_apply(const double* cm, int64_t n, const double* u, double* out) {
    return guarded([&] {
        const GridFn g = make_periodic(std::vector<double>(u, u + n), 1.0 / static_cast<double>(n));
        const GridFn r = minplus_apply(matrix_of(cm, n), g);
        std::memcpy(out, r.values.data(), n * sizeof(double));
    });
}

int ref_eigenvalue_karp(const double* cm, int64_t n, double* lambda) {
    return guarded([&] { *lambda = eigenvalue_karp(matrix_of(cm, n)); });
}

int ref_build_period_matrix(int n_space, double tau, double drift, const double* vtabs, int64_t nt,
                            double* c) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, 0.0);
        const HamiltonianSpec spec{mechanical(drift), time_table_potential(vtabs, nt, n_space, tau), true, true};
        const MinPlusMatrix r = build_period_matrix(spec, p);
        std::memcpy(c, r.cost.data(), r.cost.size() * sizeof(double));
    });
}

int ref_estimate_hbar_drift(const double* u0, int n_space, double tau, double drift, const double* vtabs,
                            int64_t nt, int max_periods, double tol, double* h_bar, double* residual,
                            int64_t* n_steps, int* converged) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, 0.0);
        const HamiltonianSpec spec{mechanical(drift), time_table_potential(vtabs, nt, n_space, tau), true, true};
        const GridFn g = make_periodic(std::vector<double>(u0, u0 + n_space), p.epsilon());
        const EffectiveHEstimate e = estimate_hbar_drift(g, spec, p, max_periods, tol);
        *h_bar = e.h_bar;
        *residual = e.residual;
        *n_steps = e.n_steps;
        *converged = e.converged ? 1 : 0;
    });
}

int ref_fixed_point_residual(const double* u, int n_space, double tau, double drift, const double* vtabs,
                             int64_t nt, double h_bar, double* residual) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, 0.0);
        const HamiltonianSpec spec{mechanical(drift), time_table_potential(vtabs, nt, n_space, tau), true, true};
        const GridFn g = make_periodic(std::vector<double>(u, u + n_space), p.epsilon());
        *residual = fixed_point_residual(g, h_bar, spec, p);
    });
}

// step_semidiscrete (proj/src/scheme.cpp:166-206) with a built-in potential kind
// (0 zero, 1 const, 2 cosine; tmod 0 none, 1 sin, 2 cos).  periodic: u holds the
// fundamental domain (n_space samples) and out receives n_space values; else m samples.
int ref_step_semidiscrete(const double* u, int64_t m, int periodic, double origin, int n_space, double tau,
                          double drift, int kind, double value, double offset, double amplitude, int frequency,
                          int tmod, double omega, double t, int q, double* out) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, 0.0);
        Potential pot = potential_zero();
        if (kind == 1) pot = potential_const(value);
        if (kind == 2)
            pot = potential_cosine(offset, amplitude, frequency,
                                   tmod == 1 ? Potential::TimeMod::Sin
                                             : (tmod == 2 ? Potential::TimeMod::Cos : Potential::TimeMod::None),
                                   omega);
        const HamiltonianSpec spec{mechanical(drift), pot, periodic != 0, false};
        const GridFn g = periodic ? make_periodic(std::vector<double>(u, u + n_space), p.epsilon(), origin)
                                  : make_grid_fn(std::vector<double>(u, u + m), p.epsilon(), origin);
        const GridFn r = step_semidiscrete(g, t, spec, p, q);
        std::memcpy(out, r.values.data(), (periodic ? n_space : m) * sizeof(double));
        if (periodic && r.values.back() != r.values.front()) throw EvaluationError("seam differs");
    });
}

// Tabulated kinetics: the kernel window (proj/src/scheme.cpp:59-105) and kinetic_convolve of a
// periodic u (fundamental domain) with it.
int ref_kernel_tabulated(int n_space, double tau, const double* samples, int64_t count, double v0, double dv,
                         double* window, int64_t* center, int64_t* argmin) {
    return guarded([&] {
        const Kernel k = build_kernel(tabulated(std::vector<double>(samples, samples + count), v0, dv),
                                      params_of(n_space, tau, 0.0));
        std::memcpy(window, k.window.values.data(), k.window.values.size() * sizeof(double));
        if (center) *center = k.center_index;
        if (argmin) *argmin = k.argmin_index;
    });
}

int ref_convolve_tabulated(const double* u, int n_space, double tau, const double* samples, int64_t count,
                           double v0, double dv, double eta, int engine, double* out, int64_t* blocks) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, eta);
        const Kernel k = build_kernel(tabulated(std::vector<double>(samples, samples + count), v0, dv), p);
        const GridFn g = make_periodic(std::vector<double>(u, u + n_space), p.epsilon());
        const GridFn r = kinetic_convolve(g, k, eta, engine_of(engine), blocks);
        std::memcpy(out, r.values.data(), n_space * sizeof(double));
    });
}

// split_step_nd of a periodic rank-`rank` tensor (n^rank, row-major) with mechanical(drifts[a]) per axis
// and V given as a full table of n^rank values (V(t, x) = table[flat index of x], time independent).
int ref_split_step_nd(const double* u, int rank, int n_space, double tau, const double* drifts, const double* vtab,
                      double t, double eta, double* out) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, eta);
        std::size_t total = 1;
        for (int a = 0; a < rank; ++a) total *= static_cast<std::size_t>(n_space);
        const TensorFn tu = make_tensor(std::vector<double>(u, u + total),
                                        std::vector<std::size_t>(rank, static_cast<std::size_t>(n_space)),
                                        p.epsilon(), std::vector<double>(rank, 0.0), true);
        SplitSpec spec;
        for (int a = 0; a < rank; ++a) spec.kinetics.push_back(mechanical(drifts[a]));
        if (vtab) {
            std::vector<double> tab(vtab, vtab + total);
            const double step = p.epsilon();
            const int n = n_space;
            spec.potential = [tab, step, n](double, std::span<const double> x) {
                std::size_t flat = 0;
                for (double xa : x) {
                    long long j = std::llround(xa / step);
                    j = ((j % n) + n) % n;
                    flat = flat * static_cast<std::size_t>(n) + static_cast<std::size_t>(j);
                }
                return tab[flat];
            };
        }
        const TensorFn r = split_step_nd(tu, t, spec, p);
        std::memcpy(out, r.values.data(), total * sizeof(double));
    });
}

// split_step_nd of a windowed (non-periodic) tensor dims[0] x ... with origins, mechanical(drifts[a])
// per axis and V a full table indexed by llround((x_a - origin_a) / step).
int ref_split_step_nd_window(const double* u, int rank, const int64_t* dims, const double* origins, int n_space,
                             double tau, const double* drifts, const double* vtab, double t, double* out) {
    return guarded([&] {
        const SchemeParams p = params_of(n_space, tau, 0.0);
        std::vector<std::size_t> d(dims, dims + rank);
        std::size_t total = 1;
        for (std::size_t x : d) total *= x;
        const TensorFn tu = make_tensor(std::vector<double>(u, u + total), d, p.epsilon(),
                                        std::vector<double>(origins, origins + rank), false);
        SplitSpec spec;
        for (int a = 0; a < rank; ++a) spec.kinetics.push_back(mechanical(drifts[a]));
        if (vtab) {
            std::vector<double> tab(vtab, vtab + total);
            std::vector<double> org(origins, origins + rank);
            const double step = p.epsilon();
            spec.potential = [tab, step, d, org](double, std::span<const double> x) {
                std::size_t flat = 0;
                for (std::size_t a = 0; a < x.size(); ++a)
                    flat = flat * d[a] + static_cast<std::size_t>(std::llround((x[a] - org[a]) / step));
                return tab[flat];
            };
        }
        const TensorFn r = split_step_nd(tu, t, spec, p);
        std::memcpy(out, r.values.data(), total * sizeof(double));
    });
}

}  // extern "C"

// The drop-in shim (laxol_gpu) against the reference's own CPU engines, in one process
// linked with the unmodified reference library (built from its sources by oracle/Makefile)
// and liblaxol_b200.so.  Every comparison is ==; prints one PASS/FAIL line per case and
// exits non-zero on any failure.  Run by tests/test_integration_gpu.py on the GPU box.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numbers>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "laxol/errors.hpp"
#include "laxol/grid_fn.hpp"
#include "laxol/hamiltonian.hpp"
#include "laxol/scheme.hpp"
#include "laxol/splitting.hpp"
#include "laxol_gpu.hpp"

using laxol_gpu::Engine;

static int g_fail = 0;

static void report(const std::string& name, bool ok) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", name.c_str());
    if (!ok) ++g_fail;
}

static bool same(const laxol::GridFn& a, const laxol::GridFn& b) {
    if (a.values.size() != b.values.size() || a.step != b.step || a.origin != b.origin || a.periodic != b.periodic)
        return false;
    for (std::size_t i = 0; i < a.values.size(); ++i)
        if (!(a.values[i] == b.values[i])) return false;
    return true;
}


static bool same_t(const laxol::TensorFn& a, const laxol::TensorFn& b) {
    if (a.values.size() != b.values.size() || a.dims != b.dims || a.step != b.step || a.origins != b.origins ||
        a.periodic != b.periodic)
        return false;
    for (std::size_t i = 0; i < a.values.size(); ++i)
        if (!(a.values[i] == b.values[i])) return false;
    return true;
}

static laxol::SchemeParams params_of(int n, double tau, double eta = 0.0) {
    laxol::SchemeParams p;
    p.n_space = n;
    p.tau = tau;
    p.eta = eta;
    return p;
}

// seeded periodic random walk (fundamental domain), made periodic by removing the drift
static std::vector<double> walk(int n, double scale, std::uint64_t seed) {
    std::mt19937_64 g(seed);
    std::uniform_real_distribution<double> d(-scale / n, scale / n);
    std::vector<double> w(n + 1, 0.0);
    for (int i = 0; i < n; ++i) w[i + 1] = w[i] + d(g);
    std::vector<double> u(n);
    for (int i = 0; i < n; ++i) u[i] = w[i] - w[n] * i / n;
    return u;
}

int main() {
    laxol_gpu::Device dev(0);
    constexpr double kTwoPi = 2.0 * std::numbers::pi;

    // 1. kinetic_convolve, mechanical and tabulated windows, both device engines == Naive
    for (int n : {24, 600, 1024, 4096}) {
        const double tau = n == 24 ? 0.25 : (n == 4096 ? 0.01 : 0.04);
        for (double drift : {0.0, 0.4, -0.7}) {
            const laxol::SchemeParams p = params_of(n, tau);
            const laxol::Kernel k = laxol::build_kernel(laxol::mechanical(drift), p);
            const laxol::GridFn u = laxol::make_periodic(walk(n, 4.0, 100 + n), p.epsilon());
            std::int64_t bref = 0, bf = 0, bd = 0;
            const laxol::GridFn want = laxol::kinetic_convolve(u, k, 0.0, laxol::ConvEngine::Naive, &bref);
            const laxol::GridFn gf = dev.kinetic_convolve(u, k, 0.0, Engine::GpuFast, &bf);
            const laxol::GridFn gd = dev.kinetic_convolve(u, k, 0.0, Engine::GpuDirect, &bd);
            report("kinetic_convolve mechanical n=" + std::to_string(n) + " P=" + std::to_string(drift),
                   same(gf, want) && same(gd, want) && bf == bref && bd == bref);
        }
    }
    {
        // tabulated conjugates the reference accepts at these grids (its convexity check)
        struct Tab {
            const char* name;
            double v0, dv;
            int count, n;
            double tau;
            double (*f)(double);
        };
        const Tab tabs[] = {
            {"|v|^1.5", -25.0, 0.5, 101, 64, 0.1, [](double v) { return std::pow(std::abs(v), 1.5); }},
            {"piecewise", -50.0, 2.5, 41, 256, 0.1,
             [](double v) { return std::max(std::max(-v, 0.5 * v), 0.25 * v + 1.0); }},
            {"flat bottom", -40.0, 1.0, 81, 512, 0.25,
             [](double v) { return std::pow(std::max(std::abs(v) - 2.0, 0.0), 2.0); }},
        };
        for (const Tab& tb : tabs) {
            std::vector<double> samples;
            for (int i = 0; i < tb.count; ++i) samples.push_back(tb.f(tb.v0 + i * tb.dv));
            const laxol::SchemeParams p = params_of(tb.n, tb.tau);
            const laxol::Kernel k = laxol::build_kernel(laxol::tabulated(samples, tb.v0, tb.dv), p);
            const laxol::GridFn u = laxol::make_periodic(walk(tb.n, 0.5, 7 + tb.n), p.epsilon());
            const laxol::GridFn want = laxol::kinetic_convolve(u, k, 0.0, laxol::ConvEngine::Naive);
            report(std::string("kinetic_convolve tabulated ") + tb.name + " n=" + std::to_string(tb.n),
                   same(dev.kinetic_convolve(u, k, 0.0, Engine::GpuFast), want) &&
                       same(dev.kinetic_convolve(u, k, 0.0, Engine::GpuDirect), want));
        }
    }
    // 2. eta > 0: GpuFast == the reference's relaxed ConvEngine::Fast (values and capped blocks)
    for (double eta : {1e-6, 1e-3}) {
        const int n = 600;
        const laxol::SchemeParams p = params_of(n, 0.04, eta);
        const laxol::Kernel k = laxol::build_kernel(laxol::mechanical(1.0), p);
        const laxol::GridFn u = laxol::make_periodic(walk(n, 2.0, 55), p.epsilon());
        std::int64_t bref = 0, bg = 0;
        const laxol::GridFn want = laxol::kinetic_convolve(u, k, eta, laxol::ConvEngine::Fast, &bref);
        report("kinetic_convolve relaxed eta=" + std::to_string(eta),
               same(dev.kinetic_convolve(u, k, eta, Engine::GpuFast, &bg), want) && bg == bref);
    }
    // 3. windowed (wall) domain == Naive; a window that cannot reach raises EvaluationError
    {
        const int n = 128;
        const laxol::SchemeParams p = params_of(n, 0.05);
        const laxol::Kernel k = laxol::build_kernel(laxol::mechanical(0.3), p);
        std::vector<double> w = walk(n, 1.0, 3);
        w.resize(96);
        const laxol::GridFn u = laxol::make_grid_fn(w, p.epsilon(), 0.25);
        const laxol::GridFn want = laxol::kinetic_convolve(u, k, 0.0, laxol::ConvEngine::Naive);
        report("kinetic_convolve windowed", same(dev.kinetic_convolve(u, k, 0.0, Engine::GpuDirect), want) &&
                                                same(dev.kinetic_convolve(u, k, 0.0, Engine::GpuFast), want));
        bool ref_threw = false, gpu_threw = false;
        const laxol::Kernel kfar = laxol::build_kernel(laxol::mechanical(40.0), p);
        try {
            laxol::kinetic_convolve(u, kfar, 0.0, laxol::ConvEngine::Naive);
        } catch (const laxol::EvaluationError&) {
            ref_threw = true;
        }
        try {
            dev.kinetic_convolve(u, kfar, 0.0, Engine::GpuDirect);
        } catch (const laxol::EvaluationError&) {
            gpu_threw = true;
        }
        report("kinetic_convolve windowed unreachable -> EvaluationError", ref_threw && gpu_threw);
    }
    // 4. step_fully_discrete with a time-dependent custom potential (Arrival and Departure)
    for (auto sampling : {laxol::PotentialSampling::Arrival, laxol::PotentialSampling::Departure}) {
        const int n = 1024;
        laxol::SchemeParams p = params_of(n, 0.05);
        p.v_sampling = sampling;
        const laxol::HamiltonianSpec spec = laxol::make_spec(
            laxol::mechanical(0.5),
            laxol::potential_custom([&](double t, double x) { return std::cos(kTwoPi * x) + 0.3 * std::sin(kTwoPi * t); },
                                    1.3, true),
            true, false);
        const laxol::Kernel k = laxol::build_kernel(spec, p);
        std::vector<double> u0(n);
        for (int j = 0; j < n; ++j) u0[j] = std::sin(kTwoPi * (static_cast<double>(j) * p.epsilon()));
        const laxol::GridFn u = laxol::make_periodic(u0, p.epsilon());
        laxol::StepStats sr, sf, sd;
        const laxol::GridFn want = laxol::step_fully_discrete(u, 0.35, spec, p, k, laxol::ConvEngine::Naive, &sr);
        const laxol::GridFn gf = dev.step_fully_discrete(u, 0.35, spec, p, k, Engine::GpuFast, &sf);
        const laxol::GridFn gd = dev.step_fully_discrete(u, 0.35, spec, p, k, Engine::GpuDirect, &sd);
        report(std::string("step_fully_discrete custom V ") +
                   (sampling == laxol::PotentialSampling::Arrival ? "arrival" : "departure"),
               same(gf, want) && same(gd, want) && sf.block_count == sr.block_count &&
                   sd.block_count == sr.block_count);
    }
    // 5. evolve: C1 in full (N=1024, tau=0.05, P=0.5, V=cos 2 pi x, u0=sin 2 pi x, 2000 steps)
    {
        const int n = 1024;
        const laxol::SchemeParams p = params_of(n, 0.05);
        const laxol::HamiltonianSpec spec = laxol::make_spec(
            laxol::mechanical(0.5), laxol::potential_custom([&](double, double x) { return std::cos(kTwoPi * x); }, 1.0, false),
            true, true);
        std::vector<double> u0(n);
        for (int j = 0; j < n; ++j) u0[j] = std::sin(kTwoPi * (static_cast<double>(j) * p.epsilon()));
        const laxol::GridFn u = laxol::make_periodic(u0, p.epsilon());
        laxol::EvolveOptions o;
        o.engine = laxol::ConvEngine::Naive;
        const laxol::EvolutionTrace want = laxol::evolve(u, 0.0, 2000, spec, p, o);
        for (Engine e : {Engine::GpuFast, Engine::GpuDirect}) {
            const laxol::EvolutionTrace got = dev.evolve(u, 0.0, 2000, spec, p, e, {});
            bool ok = got.completed == want.completed && got.snapshots.size() == want.snapshots.size() &&
                      got.per_step.size() == want.per_step.size() && got.times == want.times &&
                      got.snapshot_steps == want.snapshot_steps;
            for (std::size_t i = 0; ok && i < want.snapshots.size(); ++i) ok = same(got.snapshots[i], want.snapshots[i]);
            for (std::size_t i = 0; ok && i < want.per_step.size(); ++i)
                ok = got.per_step[i].drift == want.per_step[i].drift && got.per_step[i].blocks == want.per_step[i].blocks &&
                     got.per_step[i].time == want.per_step[i].time;
            report(std::string("evolve C1 2000 steps ") + (e == Engine::GpuFast ? "GpuFast" : "GpuDirect"), ok);
        }
    }
    // 7. split_step_nd over laxol::TensorFn / SplitSpec / PotentialNd == the reference's split_step_nd
    {
        const laxol::PotentialNd vnd = [&](double t, std::span<const double> x) {
            double v = 0.2 * std::sin(kTwoPi * t);
            double c = 1.0;
            for (double xi : x) c *= std::cos(kTwoPi * xi);
            return c + v;
        };
        for (int rank : {2, 3}) {
            const int n = rank == 2 ? 64 : 16;
            for (double eta : {0.0, 1e-7}) {
                const laxol::SchemeParams p = params_of(n, rank == 2 ? 0.02 : 0.1, eta);  // eps/tau < 1 (anti-CFL)
                std::size_t total = 1;
                for (int a = 0; a < rank; ++a) total *= static_cast<std::size_t>(n);
                std::vector<double> vals(total);
                std::mt19937_64 g(77 + rank);
                std::uniform_real_distribution<double> ud(-0.5, 0.5);
                for (std::size_t i = 0; i < total; ++i) {
                    const double x0 = static_cast<double>(i / (total / n)) / n;
                    vals[i] = std::sin(kTwoPi * x0) + 0.01 * ud(g);
                }
                const laxol::TensorFn u = laxol::make_tensor(vals, std::vector<std::size_t>(rank, n), p.epsilon(),
                                                             std::vector<double>(rank, 0.0), true);
                laxol::SplitSpec spec;
                for (int a = 0; a < rank; ++a) spec.kinetics.push_back(laxol::mechanical(a == 0 ? 0.3 : -0.7 + 0.2 * a));
                if (rank == 3) {  // a tabulated convex conjugate on the last axis (velocities 100 = 1/tau)
                    std::vector<double> tab;
                    for (int i = 0; i <= 240; ++i) tab.push_back(0.5 * (i - 120.0) * (i - 120.0) + 0.1 * (i - 120.0));
                    spec.kinetics[2] = laxol::tabulated(tab, -120.0, 1.0);
                }
                spec.potential = vnd;
                const laxol::TensorFn want = laxol::split_step_nd(u, 0.25, spec, p);
                for (Engine e : {Engine::GpuFast, Engine::GpuDirect}) {
                    if (e == Engine::GpuDirect && eta > 0.0) continue;  // Naive != the relaxed Fast for eta > 0
                    const laxol::TensorFn got = dev.split_step_nd(u, 0.25, spec, p, e);
                    report("split_step_nd periodic rank " + std::to_string(rank) + (eta > 0.0 ? " eta 1e-7" : " eta 0") +
                               (e == Engine::GpuFast ? " GpuFast" : " GpuDirect"),
                           same_t(got, want));
                }
            }
        }
        // windowed (wall) 2-D tensor with origins, eta = 0
        const laxol::SchemeParams p = params_of(50, 0.03);
        std::vector<double> vals(37 * 41);
        for (std::size_t i = 0; i < vals.size(); ++i) vals[i] = 0.3 * std::cos(0.1 * static_cast<double>(i % 41)) + 0.01 * (i / 41);
        const laxol::TensorFn u = laxol::make_tensor(vals, {37, 41}, p.epsilon(), {0.25, -0.5}, false);
        laxol::SplitSpec spec{{laxol::mechanical(0.1), laxol::mechanical(-0.4)}, vnd};
        const laxol::TensorFn want = laxol::split_step_nd(u, 0.1, spec, p);
        report("split_step_nd windowed 37x41", same_t(dev.split_step_nd(u, 0.1, spec, p, Engine::GpuFast), want) &&
                                                   same_t(dev.split_step_nd(u, 0.1, spec, p, Engine::GpuDirect), want));
        bool threw = false;
        try {
            laxol::SplitSpec bad{{laxol::mechanical(0.0)}, {}};
            dev.split_step_nd(u, 0.0, bad, p);
        } catch (const laxol::InvalidInput&) {
            threw = true;
        }
        report("split_step_nd InvalidInput on a non-separable spec", threw);
    }
    // 8. step_semidiscrete with every potential kind (Custom: any std::function) == the reference
    {
        const int n = 96;
        const laxol::SchemeParams p = params_of(n, 0.05);
        std::vector<double> u0(n);
        for (int j = 0; j < n; ++j) u0[j] = std::sin(kTwoPi * j / n) + 0.3 * std::cos(3.0 * kTwoPi * j / n);
        const laxol::GridFn u = laxol::make_periodic(u0, p.epsilon());
        std::vector<double> w0(70);
        for (int j = 0; j < 70; ++j) w0[j] = 0.2 * std::sin(0.2 * j);
        const laxol::GridFn uw{w0, p.epsilon(), -0.3, false};
        const std::vector<std::pair<std::string, laxol::Potential>> pots = {
            {"zero", laxol::potential_zero()},
            {"const", laxol::potential_const(0.75)},
            {"cosine", laxol::potential_cosine(0.1, 0.8, 2, laxol::Potential::TimeMod::Sin, 3.0)},
            {"custom", laxol::potential_custom(
                           [](double t, double x) { return std::exp(-x * x) * (1.0 + 0.5 * std::sin(7.0 * t)) + 0.3 * std::sin(5.0 * x); },
                           2.0, true)}};
        for (const auto& [name, V] : pots) {
            const laxol::HamiltonianSpec spec = laxol::make_spec(laxol::mechanical(0.4), V, true, false);
            for (int q : {1, 3}) {
                const bool ok = same(dev.step_semidiscrete(u, 0.3, spec, p, q), laxol::step_semidiscrete(u, 0.3, spec, p, q)) &&
                                same(dev.step_semidiscrete(uw, 0.3, spec, p, q), laxol::step_semidiscrete(uw, 0.3, spec, p, q));
                report("step_semidiscrete " + name + " q=" + std::to_string(q) + " periodic + windowed", ok);
            }
        }
    }
    // 5b. evolve's trace semantics on the reference's own test shapes (proj/tests/unit_scheme.cpp:
    // 283-296 windowed convex flow, 323-333 blow-up abort, 381-393 snapshot thinning) and a long
    // thinned run: the whole EvolutionTrace == the reference's
    {
        auto same_trace = [&](const laxol::EvolutionTrace& got, const laxol::EvolutionTrace& want) {
            bool ok = got.completed == want.completed && got.abort_reason == want.abort_reason &&
                      got.snapshots.size() == want.snapshots.size() && got.per_step.size() == want.per_step.size() &&
                      got.times == want.times && got.snapshot_steps == want.snapshot_steps;
            for (std::size_t i = 0; ok && i < want.snapshots.size(); ++i) ok = same(got.snapshots[i], want.snapshots[i]);
            for (std::size_t i = 0; ok && i < want.per_step.size(); ++i)
                ok = got.per_step[i].drift == want.per_step[i].drift && got.per_step[i].blocks == want.per_step[i].blocks &&
                     got.per_step[i].time == want.per_step[i].time;
            return ok;
        };
        laxol::EvolveOptions naive;
        naive.engine = laxol::ConvEngine::Naive;
        {  // values blow up: a partial trace, completed == false, the same abort reason and last snapshot
            const laxol::SchemeParams p = params_of(16, 0.25);
            const laxol::Potential pot =
                laxol::potential_custom([](double t, double) { return t < 0.9 ? 0.0 : 1e308; }, 1e308, true);
            const laxol::HamiltonianSpec spec{laxol::mechanical(0.0), pot, true, false};
            const laxol::GridFn u = laxol::make_periodic(std::vector<double>(16, 0.0), p.epsilon());
            const laxol::EvolutionTrace want = laxol::evolve(u, 0.0, 12, spec, p, naive);
            for (Engine e : {Engine::GpuFast, Engine::GpuDirect}) {
                const laxol::EvolutionTrace got = dev.evolve(u, 0.0, 12, spec, p, e, {});
                report(std::string("evolve blow-up abort ") + (e == Engine::GpuFast ? "GpuFast" : "GpuDirect"),
                       !want.completed && !got.abort_reason.empty() && same_trace(got, want));
            }
        }
        {  // snapshot thinning keeps the endpoints and the requested captures
            const laxol::SchemeParams p = params_of(8, 0.5);
            const laxol::HamiltonianSpec spec = laxol::make_spec(laxol::mechanical(0.0), laxol::potential_zero(), true, true);
            const laxol::GridFn u = laxol::make_periodic(std::vector<double>(8, 0.0), p.epsilon());
            laxol::EvolveOptions o = naive;
            o.snapshot_stride = 1000;
            o.capture_steps = {3};
            const laxol::EvolutionTrace want = laxol::evolve(u, 0.0, 7, spec, p, o);
            const laxol::EvolutionTrace got = dev.evolve(u, 0.0, 7, spec, p, Engine::GpuFast, o);
            report("evolve snapshot thinning (stride 1000, capture {3})",
                   got.snapshot_steps == std::vector<std::int64_t>{0, 3, 7} && same_trace(got, want));
        }
        {  // more than 1024 steps: the automatic stride, a time-dependent potential, an unsorted capture list
            const int n = 96;
            const laxol::SchemeParams p = params_of(n, 0.05);
            const laxol::HamiltonianSpec spec = laxol::make_spec(
                laxol::mechanical(-0.35),
                laxol::potential_custom([&](double t, double x) { return std::cos(kTwoPi * x) * (1.0 + 0.25 * std::sin(kTwoPi * t)); },
                                        1.25, true),
                true, false);
            std::vector<double> u0(n);
            for (int j = 0; j < n; ++j) u0[j] = 0.3 * std::sin(2.0 * kTwoPi * j / n);
            const laxol::GridFn u = laxol::make_periodic(u0, p.epsilon());
            laxol::EvolveOptions o = naive;
            o.capture_steps = {1501, 7, 1024};
            const laxol::EvolutionTrace want = laxol::evolve(u, 0.5, 2500, spec, p, o);
            for (Engine e : {Engine::GpuFast, Engine::GpuDirect}) {
                const laxol::EvolutionTrace got = dev.evolve(u, 0.5, 2500, spec, p, e, o);
                report(std::string("evolve 2500 thinned steps, time-dependent V ") +
                           (e == Engine::GpuFast ? "GpuFast" : "GpuDirect"),
                       want.snapshots.size() < 1100 && same_trace(got, want));
            }
        }
        {  // eta > 0: the reference's relaxed Fast engine step after step (its approximation errors
           // compound; the device reproduces every one), block counts capped as the reference reports
            const int n = 600;
            laxol::SchemeParams p = params_of(n, 0.04);
            p.eta = 1e-6;
            const laxol::HamiltonianSpec spec =
                laxol::make_spec(laxol::mechanical(1.0), laxol::potential_cosine(1.0, -1.0, 1), true, true);
            std::vector<double> v(n);
            for (int i = 0; i < n; ++i) v[i] = std::cos(2.0 * kTwoPi * (static_cast<double>(i) * p.epsilon()));
            const laxol::GridFn u = laxol::make_periodic(v, p.epsilon());
            laxol::EvolveOptions fast;
            fast.engine = laxol::ConvEngine::Fast;
            const laxol::EvolutionTrace want = laxol::evolve(u, 0.0, 60, spec, p, fast);
            const laxol::EvolutionTrace got = dev.evolve(u, 0.0, 60, spec, p, Engine::GpuFast, {});
            report("evolve 60 steps, eta 1e-6 (relaxed Fast engine)", same_trace(got, want));
        }
        {  // windowed (wall) domain: the kinetic-only flow of convex data, 20 steps
            const laxol::SchemeParams p = params_of(32, 0.125);
            const laxol::HamiltonianSpec spec = laxol::make_spec(laxol::mechanical(0.0), laxol::potential_zero(), true, true);
            std::vector<double> v(65);
            for (int i = 0; i < 65; ++i) {
                const double x = -1.0 + static_cast<double>(i) * p.epsilon();
                v[i] = x * x + 0.25 * std::fabs(x - 0.3);
            }
            const laxol::GridFn u = laxol::make_grid_fn(v, p.epsilon(), -1.0);
            const laxol::EvolutionTrace want = laxol::evolve(u, 0.0, 20, spec, p, naive);
            for (Engine e : {Engine::GpuFast, Engine::GpuDirect}) {
                const laxol::EvolutionTrace got = dev.evolve(u, 0.0, 20, spec, p, e, {});
                report(std::string("evolve windowed convex flow ") + (e == Engine::GpuFast ? "GpuFast" : "GpuDirect"),
                       same_trace(got, want));
            }
        }
    }
    // 6. the reference's argument errors surface as its own exception types
    {
        const laxol::SchemeParams p = params_of(64, 0.05);
        const laxol::Kernel k = laxol::build_kernel(laxol::mechanical(0.0), p);
        const laxol::GridFn u = laxol::make_periodic(std::vector<double>(32, 0.0), 1.0 / 32);
        bool threw = false;
        try {
            dev.kinetic_convolve(u, k, 0.0, Engine::GpuFast);
        } catch (const laxol::InvalidInput&) {
            threw = true;
        }
        bool threw2 = false;
        const laxol::HamiltonianSpec spec = laxol::make_spec(laxol::mechanical(0.0), laxol::potential_zero(), true, true);
        try {
            dev.evolve(u, 0.0, 3, spec, p, Engine::GpuFast, {});
        } catch (const laxol::InvalidInput&) {
            threw2 = true;
        }
        report("InvalidInput on a grid of another period", threw && threw2);
    }
    std::printf("%s: %d failure(s)\n", g_fail ? "FAILED" : "ALL PASS", g_fail);
    return g_fail ? 1 : 0;
}

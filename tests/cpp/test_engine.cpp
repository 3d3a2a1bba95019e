// C++ parity tests of the laxol_b200 host API (csrc/host/laxol_b200.hpp),
// written the way the reference's own unit tests exercise its stepping API
// (proj/tests/unit_scheme.cpp, proj/tests/unit_splitting.cpp), with
// independent brute-force oracles.  Needs a CUDA device; prints one
// PASS/FAIL line per check and exits non-zero on any failure.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <string>
#include <cmath>
#include <cstdio>
#include <limits>
#include <random>
#include <vector>

#include "laxol_b200.hpp"

using namespace laxol_b200;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond, ...)                           \
    do {                                           \
        if (cond) {                                \
            ++g_pass;                              \
        } else {                                   \
            ++g_fail;                              \
            std::printf("[FAIL] " __VA_ARGS__);    \
            std::printf("  (%s:%d)\n", __FILE__, __LINE__); \
        }                                          \
    } while (0)

static SchemeParams params_of(int n, double tau) {
    SchemeParams p;
    p.n_space = n;
    p.tau = tau;
    return p;
}

static GridFn random_periodic(std::mt19937_64& rng, int n, double amp, double step) {
    std::uniform_real_distribution<double> d(-amp, amp);
    std::vector<double> v(n);
    for (double& x : v) x = d(rng);
    return make_periodic(std::move(v), step);
}

// definition-level periodic minimum (proj/tests/unit_scheme.cpp:184-190)
static double def_min(const GridFn& u, const KernelWindow& k, int64_t j) {
    const int64_t n = static_cast<int64_t>(u.n());
    double want = std::numeric_limits<double>::infinity();
    for (std::size_t w = 0; w < k.window.size(); ++w) {
        const int64_t d = k.first + static_cast<int64_t>(w);
        const int64_t y = (((j - d) % n) + n) % n;
        want = std::min(want, u.values[y] + k.window[w]);
    }
    return want;
}

// e2e through the C++ API a reference user calls: Engine::step_fully_discrete on pageable
// std::vector lines of C2 (N = 65536, tau = 0.02, per-line drift, V = cos 2 pi x + 0.5 cos(4 pi x + 1)),
// the reference's loop order (every step, every line).  Prints one JSON object.
static int bench(int lines, int steps) {
    Engine eng(0);
    const int n = 65536;
    const double tau = 0.02;
    const SchemeParams p = params_of(n, tau);
    constexpr double kTwoPi = 2.0 * 3.14159265358979323846;
    Potential V;
    V.fn = [](double, double x) { return std::cos(kTwoPi * x) + 0.5 * std::cos(2.0 * kTwoPi * x + 1.0); };
    std::vector<KernelWindow> ks;
    std::vector<GridFn> us;
    for (int l = 0; l < lines; ++l) {
        const double drift = -2.0 + 4.0 * (l * (255.0 / std::max(1, lines - 1))) / 255.0;
        ks.push_back(build_kernel_mech(n, tau, drift));
        us.push_back(make_periodic(std::vector<double>(n, 0.0), p.epsilon()));
    }
    auto run = [&](bool line_major) {
        const auto t0 = std::chrono::steady_clock::now();
        if (line_major) {
            for (int l = 0; l < lines; ++l)
                for (int k = 0; k < steps; ++k)
                    us[l] = eng.step_fully_discrete(us[l], k * tau, V, p, ks[l], ConvEngine::GpuFast);
        } else {
            for (int k = 0; k < steps; ++k)
                for (int l = 0; l < lines; ++l)
                    us[l] = eng.step_fully_discrete(us[l], k * tau, V, p, ks[l], ConvEngine::GpuFast);
        }
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    run(false);  // warm
    const double ts = run(false), tl = run(true);
    const double upd = static_cast<double>(lines) * steps * n;
    std::printf("{\"api\": \"laxol_b200::Engine::step_fully_discrete (pageable std::vector, one line per call)\", "
                "\"lines\": %d, \"n\": %d, \"steps\": %d, \"step_major_updates_per_s\": %.6g, "
                "\"line_major_updates_per_s\": %.6g}\n",
                lines, n, steps, upd / ts, upd / tl);
    return 0;
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "--bench") return bench(argc > 2 ? std::atoi(argv[2]) : 16, 5);
    Engine eng(0);
    std::mt19937_64 rng(39);
    // 0. consecutive steps through the resident device state (the output of one call is the
    // next call's input: no upload, the fast engine's statistics carried) == a fresh engine's
    // step from the same host input, both engines, and a foreign input in between
    {
        const int n = 1024;
        const SchemeParams p = params_of(n, 0.05);
        const KernelWindow k = build_kernel_mech(n, 0.05, 0.5);
        Potential V;
        V.fn = [](double, double x) { return std::cos(6.283185307179586 * x); };
        GridFn u = random_periodic(rng, n, 0.01, p.epsilon());
        bool ok = true;
        for (int step = 0; step < 30 && ok; ++step) {
            Engine fresh(0);
            const GridFn a = eng.step_fully_discrete(u, step * 0.05, V, p, k, ConvEngine::GpuFast);
            const GridFn b = fresh.step_fully_discrete(u, step * 0.05, V, p, k, ConvEngine::GpuDirect);
            ok = a.values == b.values;
            if (step == 12) {  // a foreign input must not be mistaken for the resident one
                const GridFn f = random_periodic(rng, n, 0.01, p.epsilon());
                const GridFn c = eng.step_fully_discrete(f, 0.0, V, p, k, ConvEngine::GpuFast);
                const GridFn d = fresh.step_fully_discrete(f, 0.0, V, p, k, ConvEngine::GpuDirect);
                ok = ok && c.values == d.values;
            }
            u = a;
        }
        CHECK(ok, "resident consecutive steps == fresh direct steps");
    }
    // 0b. the anti-CFL guard honours h0 and AntiCflMode (proj/src/scheme.cpp:39-53)
    {
        SchemeParams p = params_of(16, 0.1);  // epsilon/tau = 0.625
        p.h0 = 0.5;
        bool threw = false;
        try {
            build_kernel_mech(p, 0.0);
        } catch (const InvalidInput&) {
            threw = true;
        }
        p.anti_cfl = AntiCflMode::Warn;
        const KernelWindow kw = build_kernel_mech(p, 0.0);  // warns, builds
        SchemeParams q = params_of(16, 0.05);                // epsilon/tau = 1.25 < h0 = 2
        q.h0 = 2.0;
        const KernelWindow kq = build_kernel_mech(q, 0.3);
        CHECK(threw && kw.window.size() == 33 && kq.window.size() == 33, "anti-CFL guard: h0 and Warn");
    }
    // 1. kinetic_convolve == definition-level minimum, both device engines
    for (double drift : {0.0, 0.4, -0.7, 1.0}) {
        const SchemeParams p = params_of(24, 0.25);
        const KernelWindow k = build_kernel_mech(24, 0.25, drift);
        const GridFn u = random_periodic(rng, 24, 1.0, p.epsilon());
        for (ConvEngine e : {ConvEngine::GpuDirect, ConvEngine::GpuFast}) {
            const GridFn got = eng.kinetic_convolve(u, k, 0.0, e);
            bool ok = got.values.size() == 25 && got.values[24] == got.values[0];
            for (std::size_t j = 0; j < 24; ++j) ok = ok && got.values[j] == def_min(u, k, j);
            CHECK(ok, "kinetic_convolve drift %g engine %d", drift, static_cast<int>(e));
        }
    }
    // 2. constants are fixed points of the kinetic-only flow (unit_scheme.cpp:87-94)
    {
        const SchemeParams p = params_of(32, 0.125);
        const KernelWindow k = build_kernel_mech(32, 0.125, 0.0);
        const GridFn u = make_periodic(std::vector<double>(32, 1.25), p.epsilon());
        for (ConvEngine e : {ConvEngine::GpuDirect, ConvEngine::GpuFast}) {
            const GridFn v = eng.step_fully_discrete(u, 0.0, Potential{}, p, k, e);
            bool ok = true;
            for (double x : v.values) ok = ok && x == 1.25;
            CHECK(ok, "constant fixed point engine %d", static_cast<int>(e));
        }
    }
    // 3. representable drift lands exactly: -tau P^2/2 = -0.1 (unit_scheme.cpp:96-106)
    {
        const SchemeParams p = params_of(10, 0.2);
        const KernelWindow k = build_kernel_mech(10, 0.2, 1.0);
        const GridFn u = make_periodic(std::vector<double>(10, 0.0), p.epsilon());
        for (ConvEngine e : {ConvEngine::GpuDirect, ConvEngine::GpuFast}) {
            const GridFn v = eng.step_fully_discrete(u, 0.0, Potential{}, p, k, e);
            bool ok = true;
            for (double x : v.values) ok = ok && x == -0.1;
            CHECK(ok, "representable drift engine %d", static_cast<int>(e));
        }
    }
    // 4. evolve: single step trace matches a direct call; engines agree; thinning
    {
        const SchemeParams p = params_of(48, 0.125);
        Potential V;
        V.fn = [](double, double x) { return 0.5 + 0.5 * std::cos(2.0 * 2.0 * M_PI * x); };
        const GridFn u = random_periodic(rng, 48, 1.0, p.epsilon());
        const KernelWindow k = build_kernel_mech(48, 0.125, 0.7);
        EvolveOptions fast, direct;
        fast.engine = ConvEngine::GpuFast;
        direct.engine = ConvEngine::GpuDirect;
        const EvolutionTrace one = eng.evolve(u, 0.0, 1, 0.7, V, p, fast);
        const GridFn step1 = eng.step_fully_discrete(u, 0.0, V, p, k, ConvEngine::GpuDirect);
        CHECK(one.snapshots.size() == 2 && one.snapshots[1].values == step1.values && one.completed,
              "evolve single step == step_fully_discrete");
        const EvolutionTrace a = eng.evolve(u, 0.0, 12, 0.7, V, p, fast);
        const EvolutionTrace b = eng.evolve(u, 0.0, 12, 0.7, V, p, direct);
        bool ok = a.snapshots.size() == b.snapshots.size() && a.snapshots.size() == 13;
        for (std::size_t s = 0; ok && s < a.snapshots.size(); ++s)
            for (std::size_t j = 0; j < a.snapshots[s].values.size(); ++j)
                ok = ok && std::fabs(a.snapshots[s].values[j] - b.snapshots[s].values[j]) <= 1e-13;
        CHECK(ok, "evolve fast vs direct engines agree step by step");
        ok = a.per_step.size() == 12;
        for (std::size_t i = 0; ok && i < 12; ++i)
            ok = a.per_step[i].blocks == b.per_step[i].blocks &&
                 std::fabs(a.per_step[i].time - 0.125 * (i + 1)) < 1e-15;
        CHECK(ok, "evolve per-step block counts and times");
        EvolveOptions thin;
        thin.snapshot_stride = 1000;
        thin.capture_steps = {3};
        const EvolutionTrace t = eng.evolve(make_periodic(std::vector<double>(8, 0.0), 1.0 / 8), 0.0, 7, 0.0,
                                            Potential{}, params_of(8, 0.5), thin);
        CHECK(t.snapshot_steps.size() == 3 && t.snapshot_steps[1] == 3 && t.snapshot_steps[2] == 7,
              "evolve snapshot thinning keeps endpoints and captures");
    }
    // 5. evolve aborts with a partial trace when values blow up (unit_scheme.cpp:323-333)
    {
        const SchemeParams p = params_of(16, 0.25);
        Potential V;
        V.fn = [](double tt, double) { return tt < 0.9 ? 0.0 : 1e308; };
        V.time_dependent = true;
        EvolveOptions o;
        o.engine = ConvEngine::GpuFast;
        const EvolutionTrace tr = eng.evolve(make_periodic(std::vector<double>(16, 0.0), 1.0 / 16), 0.0, 12,
                                             0.0, V, p, o);
        CHECK(!tr.completed && !tr.abort_reason.empty() && tr.snapshots.size() >= 2,
              "evolve aborts on non-finite values");
    }
    // 6. split_step_nd == direct 2-D minimum, associating (u + k1) + k2 (unit_splitting.cpp:25-65,103-121)
    {
        const int n = 16;
        const SchemeParams p = params_of(n, 0.25);
        const KernelWindow k1 = build_kernel_mech(n, 0.25, 0.0), k2 = build_kernel_mech(n, 0.25, 0.5);
        std::uniform_real_distribution<double> d(-1.0, 1.0);
        for (ConvEngine e : {ConvEngine::GpuDirect, ConvEngine::GpuFast}) {
            TensorFn u;
            u.values.resize(n * n);
            for (double& x : u.values) x = d(rng);
            u.dims = {n, n};
            u.step = p.epsilon();
            u.origins = {0.0, 0.0};
            SplitSpec2D spec;
            spec.drift1 = 0.0;
            spec.drift2 = 0.5;
            const TensorFn out = eng.split_step_nd(u, 0.0, spec, p, e);
            bool ok = true;
            for (int x1 = 0; x1 < n; ++x1)
                for (int x2 = 0; x2 < n; ++x2) {
                    double best = std::numeric_limits<double>::infinity();
                    for (std::size_t w1 = 0; w1 < k1.window.size(); ++w1)
                        for (std::size_t w2 = 0; w2 < k2.window.size(); ++w2) {
                            const int64_t y1 = (((x1 - (k1.first + (int64_t)w1)) % n) + n) % n;
                            const int64_t y2 = (((x2 - (k2.first + (int64_t)w2)) % n) + n) % n;
                            best = std::min(best, (u.values[y1 * n + y2] + k1.window[w1]) + k2.window[w2]);
                        }
                    ok = ok && out.values[x1 * n + x2] == best;
                }
            CHECK(ok, "split_step_nd == 2-D brute force, engine %d", static_cast<int>(e));
        }
    }
    // 7. weak-KAM consumers (proj/tests/unit_weakkam.cpp)
    {
        auto cosv = [](double, double x) { return 1.0 - std::cos(2.0 * 3.141592653589793 * x); };
        // applying the period matrix equals one period of steps (unit_weakkam.cpp:114-130)
        const SchemeParams p = params_of(32, 0.2);
        Potential V{cosv, false};
        const MinPlusMatrix C = eng.build_period_matrix(1.0, V, p);
        const KernelWindow k = build_kernel_mech(32, 0.2, 1.0);
        for (int rep = 0; rep < 4; ++rep) {
            const GridFn u0 = random_periodic(rng, 32, 1.0, p.epsilon());
            GridFn st = u0;
            for (int i = 0; i < 5; ++i) st = eng.step_fully_discrete(st, 0.2 * i, V, p, k);
            const GridFn ap = eng.minplus_apply(C, u0);
            double d = 0.0;
            for (std::size_t j = 0; j < ap.values.size(); ++j) d = std::max(d, std::abs(ap.values[j] - st.values[j]));
            CHECK(d <= 1e-10, "minplus_apply(period matrix) == one period of steps (%.3e)", d);
        }
        // product associativity up to roundoff (unit_weakkam.cpp:132-147)
        std::uniform_real_distribution<double> ud(-1.0, 1.0);
        auto rnd = [&](std::size_t n) {
            MinPlusMatrix M;
            M.n = n;
            M.cost.resize(n * n);
            for (double& v : M.cost) v = ud(rng);
            return M;
        };
        const MinPlusMatrix A = rnd(12), B = rnd(12), D = rnd(12);
        const MinPlusMatrix l = eng.minplus_product(eng.minplus_product(A, B), D);
        const MinPlusMatrix r = eng.minplus_product(A, eng.minplus_product(B, D));
        bool ok = true;
        for (std::size_t i = 0; i < l.cost.size(); ++i) ok = ok && std::abs(l.cost[i] - r.cost[i]) <= 1e-12 * std::abs(r.cost[i]) + 1e-15;
        CHECK(ok, "minplus_product associative");
        // Karp closed forms (unit_weakkam.cpp:149-158)
        MinPlusMatrix Z;
        Z.n = 5;
        Z.cost.assign(25, 0.0);
        CHECK(eng.eigenvalue_karp(Z) == 0.0, "karp(zeros) == 0");
        MinPlusMatrix T2;
        T2.n = 2;
        T2.cost = {0.0, 5.0, 1.0, 0.0};
        CHECK(eng.eigenvalue_karp(T2) == 0.0, "karp(two free self-loops) == 0");
        // drift and eigenvalue estimates agree (unit_weakkam.cpp:172-192)
        const SchemeParams q = params_of(48, 0.125);
        std::vector<double> u0v(48);
        for (int i = 0; i < 48; ++i) u0v[i] = std::cos(2.0 * (2.0 * 3.141592653589793 * i / 48.0 - 3.141592653589793));
        const GridFn u0 = make_periodic(u0v, q.epsilon());
        for (ConvEngine e : {ConvEngine::GpuFast, ConvEngine::GpuDirect}) {
            const EffectiveHEstimate est = eng.estimate_hbar_drift(u0, 1.0, V, q, 600, 1e-8, e);
            const double karp = eng.eigenvalue_karp(eng.build_period_matrix(1.0, V, q));
            CHECK(est.converged && std::abs(est.h_bar - karp) < 1e-7, "drift %.12f vs karp %.12f", est.h_bar, karp);
        }
        // constant potential shifts the rate by -c (unit_weakkam.cpp:76-84)
        const SchemeParams pc = params_of(32, 0.1);
        std::vector<double> c1(32);
        for (int i = 0; i < 32; ++i) c1[i] = std::cos(2.0 * 3.141592653589793 * i / 32.0 - 3.141592653589793);
        const EffectiveHEstimate ec =
            eng.estimate_hbar_drift(make_periodic(c1, pc.epsilon()), 0.0, Potential{[](double, double) { return 0.8125; }, false}, pc, 200, 1e-10);
        CHECK(ec.converged && std::abs(ec.h_bar + 0.8125) <= 1e-12, "constant potential: %.15f", ec.h_bar);
        bool threw = false;
        try {
            eng.estimate_hbar_drift(make_periodic(c1, 1.0 / 32), 0.0, Potential{}, params_of(32, 0.15), 10, 1e-8);
        } catch (const InvalidInput&) {
            threw = true;
        }
        CHECK(threw, "tau must divide the period");
    }
    // 8. step_semidiscrete (unit_scheme.cpp:209-233)
    {
        const SchemeParams p = params_of(24, 0.25);
        const KernelWindow k = build_kernel_mech(24, 0.25, 0.25);
        const GridFn u = random_periodic(rng, 24, 1.0, p.epsilon());
        const GridFn full = eng.step_fully_discrete(u, 0.0, Potential{}, p, k, ConvEngine::GpuDirect);
        const GridFn semi = eng.step_semidiscrete(u, 0.0, 0.25, potential_zero(), p, 4);
        bool same = semi.values.size() == full.values.size();
        for (std::size_t i = 0; same && i < full.size(); ++i) same = semi.values[i] == full.values[i];
        CHECK(same, "semi-discrete(V = 0) == fully discrete step");
        bool threw = false;
        try {
            eng.step_semidiscrete(u, 0.0, 0.25, potential_zero(), p, 0);
        } catch (const InvalidInput&) {
            threw = true;
        }
        CHECK(threw, "quad_points 0 rejected");
        const SchemeParams p2 = params_of(32, 0.25);
        const BuiltinPotential pot = potential_cosine(0.0, 0.5, 1);
        const GridFn u2 = random_periodic(rng, 32, 0.5, p2.epsilon());
        const GridFn f2 = eng.step_fully_discrete(u2, 0.0, pot.callback(), p2, build_kernel_mech(32, 0.25, 0.0));
        const GridFn s2 = eng.step_semidiscrete(u2, 0.0, 0.0, pot, p2, 32);
        double d = 0.0;
        for (std::size_t i = 0; i < f2.size(); ++i) d = std::max(d, std::abs(f2.values[i] - s2.values[i]));
        CHECK(d <= 0.25 * 0.5 * 2.0 * 3.141592653589793 + 1e-9, "endpoint sampling error bound (%.3e)", d);
    }
    // 9. GpuFast with eta > 0 is the reference's relaxed fast engine: an upper bound of the
    //    exact minimum, equal to it at eta == 0 (proj/src/minplus.cpp:195-252)
    {
        const SchemeParams p = params_of(256, 0.05);
        const KernelWindow k = build_kernel_mech(256, 0.05, 0.3);
        const GridFn u = random_periodic(rng, 256, 0.01, p.epsilon());
        int64_t b0 = 0, b1 = 0;
        const GridFn ex = eng.kinetic_convolve(u, k, 0.0, ConvEngine::GpuFast, &b0);
        const GridFn rx = eng.kinetic_convolve(u, k, 1e-2, ConvEngine::GpuFast, &b1);
        bool ge = true, eq0 = true;
        int strict = 0;
        for (std::size_t j = 0; j < u.n(); ++j) {
            const double want = def_min(u, k, static_cast<int64_t>(j));
            eq0 = eq0 && ex.values[j] == want;
            ge = ge && rx.values[j] >= want;
            strict += rx.values[j] > want;
        }
        CHECK(eq0 && ge && strict > 0 && b1 >= 256 / 48, "relaxed engine: exact at eta 0, upper bound at eta > 0 (%d)",
              strict);
    }
    // 10. split_step_nd at rank 3 == the composition of three rank-1 sweeps done by hand
    {
        const int n = 8;
        const SchemeParams p = params_of(n, 0.25);
        TensorFn u;
        u.dims = {8, 8, 8};
        u.step = p.epsilon();
        u.origins = {0.0, 0.0, 0.0};
        u.values.resize(512);
        std::uniform_real_distribution<double> ud(-1.0, 1.0);
        for (double& x : u.values) x = ud(rng);
        SplitSpecND spec;
        for (double d : {0.0, 0.5, -0.25}) spec.kernels.push_back(build_kernel_mech(n, 0.25, d));
        spec.potential = [](double, std::span<const double> x) { return x[0] + 2.0 * x[1] - x[2]; };
        bool ok = true;
        for (ConvEngine e : {ConvEngine::GpuDirect, ConvEngine::GpuFast}) {
            const TensorFn out = eng.split_step_nd(u, 0.0, spec, p, e);
            std::vector<double> w = u.values;
            const int strides[3] = {64, 8, 1};
            for (int a = 0; a < 3; ++a) {
                std::vector<double> nw(w.size());
                const KernelWindow& k = spec.kernels[a];
                for (int flat = 0; flat < 512; ++flat) {
                    const int idx = (flat / strides[a]) % n;
                    const int base = flat - idx * strides[a];
                    double best = std::numeric_limits<double>::infinity();
                    for (std::size_t q = 0; q < k.window.size(); ++q) {
                        const int64_t src = (((idx - (k.first + static_cast<int64_t>(q))) % n) + n) % n;
                        best = std::min(best, w[base + src * strides[a]] + k.window[q]);
                    }
                    nw[flat] = best;
                }
                w = nw;
            }
            for (int flat = 0; flat < 512; ++flat) {
                const double c[3] = {(flat / 64) * p.epsilon(), ((flat / 8) % 8) * p.epsilon(), (flat % 8) * p.epsilon()};
                w[flat] -= 0.25 * (c[0] + 2.0 * c[1] - c[2]);
            }
            for (int flat = 0; flat < 512; ++flat) ok = ok && out.values[flat] == w[flat];
        }
        CHECK(ok, "rank-3 split_step_nd == brute-force axis sweeps + potential");
    }
    // 11. evolve on a windowed domain == repeated windowed steps, drift in the reference's order
    {
        const SchemeParams p = params_of(16, 0.25);
        std::vector<double> vals(40);
        std::uniform_real_distribution<double> ud(-1.0, 1.0);
        for (double& x : vals) x = ud(rng);
        const GridFn u0 = make_grid_fn(vals, p.epsilon(), -0.5);
        Potential V{[](double, double x) { return 0.3 * x; }, false};
        const KernelWindow k = build_kernel_mech(16, 0.25, 0.0);
        const EvolutionTrace tr = eng.evolve(u0, 0.0, 5, 0.0, V, p);
        GridFn w = u0;
        bool ok = tr.completed && tr.per_step.size() == 5;
        for (int i = 0; i < 5 && ok; ++i) {
            StepStats st;
            const GridFn nx = eng.step_fully_discrete(w, 0.25 * i, V, p, k, ConvEngine::GpuDirect, &st);
            double d = 0.0;
            for (std::size_t j = 0; j < w.size(); ++j) d += nx.values[j] - w.values[j];
            d /= static_cast<double>(w.size());
            ok = ok && tr.per_step[i].drift == d && tr.per_step[i].blocks == st.block_count;
            w = nx;
        }
        ok = ok && tr.snapshots.back().values == w.values;
        CHECK(ok, "windowed evolve == repeated windowed steps");
    }
    std::printf("%s: %d passed, %d failed\n", g_fail ? "FAIL" : "ALL PASS", g_pass, g_fail);
    return g_fail ? 1 : 0;
}

// laxol_b200 — C++ host API mirroring the reference's stepping API
// (namespace laxol, /root/reference/proj/include/laxol/{grid_fn,scheme,
// splitting,hamiltonian,errors}.hpp) over the C-ABI in include/laxol_b200.h.
//
// A reference user switches by replacing `laxol::` calls on the hot path
// with `laxol_b200::Engine` methods of the same name and arguments; the
// engine value ConvEngine::GpuFast / GpuDirect selects the B200 kernels the
// way ConvEngine::{Fast,Naive} selects the reference's CPU engines
// (proj/include/laxol/scheme.hpp:13, dispatch proj/src/scheme.cpp:114-121).
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../../include/laxol_b200.h"

namespace laxol_b200 {

// proj/include/laxol/errors.hpp:9-17
struct InvalidInput : std::runtime_error {
    explicit InvalidInput(const std::string& w) : std::runtime_error(w) {}
};
struct EvaluationError : std::runtime_error {
    explicit EvaluationError(const std::string& w) : std::runtime_error(w) {}
};

// proj/include/laxol/grid_fn.hpp:13-23: closed period for periodic functions
// (seam duplicated), n() = values.size() - 1.
struct GridFn {
    std::vector<double> values;
    double step = 1.0;
    double origin = 0.0;
    bool periodic = false;
    std::size_t n() const { return values.size() - 1; }
    std::size_t size() const { return values.size(); }
    double coord(std::size_t i) const { return origin + static_cast<double>(i) * step; }
};
GridFn make_periodic(std::vector<double> fundamental, double step, double origin = 0.0);
GridFn make_grid_fn(std::vector<double> values, double step, double origin = 0.0);

// Kernel (proj/include/laxol/scheme.hpp:34-42) for the mechanical conjugate
// K*(v) = v^2/2 - drift*v; window[w] at grid displacement first + w.
struct KernelWindow {
    std::vector<double> window;
    int64_t first = 0;
    int64_t center_index = 0;
    int64_t argmin_index = 0;
    int64_t n_space = 0;
    double tau = 0.0;
    double drift = 0.0;
    double delta = 0.0;  // fast-engine slope-inversion tolerance
    bool mechanical = true;  // false: a tabulated conjugate (drift holds its argmin velocity)
};
KernelWindow build_kernel_mech(int64_t n_space, double tau, double drift);
// proj/include/laxol/hamiltonian.hpp:27 tabulated(samples, v0, dv) + build_kernel
KernelWindow build_kernel_tab(int64_t n_space, double tau, const std::vector<double>& samples, double v0,
                              double dv);
double fast_delta(int64_t n_space, double tau, double drift, int64_t first);

enum class ConvEngine { Fast, Naive, GpuFast, GpuDirect };
enum class PotentialSampling { Arrival, Departure };
enum class AntiCflMode { Fail, Warn };

// proj/include/laxol/scheme.hpp:17-26
struct SchemeParams {
    int n_space = 0;
    double tau = 0.0;
    double eta = 0.0;
    double h0 = 1.0;
    PotentialSampling v_sampling = PotentialSampling::Arrival;
    AntiCflMode anti_cfl = AntiCflMode::Fail;
    double epsilon() const { return 1.0 / static_cast<double>(n_space); }
};
// proj/src/scheme.cpp:39-53: ranges, and the anti-CFL guard epsilon/tau < h0 (throws, or warns on
// stderr with AntiCflMode::Warn)
void validate(const SchemeParams& p);
// build_kernel(kinetic, params) (proj/src/scheme.cpp:59-105): validate(params) first, so h0 and the
// anti-CFL mode apply; the (n_space, tau, ...) builders below keep the default guard h0 = 1, Fail
struct KernelWindow;
KernelWindow build_kernel_mech(const SchemeParams& params, double drift);

// V(t, x) callback (proj/include/laxol/hamiltonian.hpp:34-73 reduced to what
// the hot path calls): evaluated on the host per grid point, like the
// reference (proj/src/scheme.cpp:158).  Empty = V == 0.
struct Potential {
    std::function<double(double, double)> fn;
    bool time_dependent = false;
    bool time_periodic = true;  // HamiltonianSpec::time_periodic (period 1), for the weak-KAM consumers
    double operator()(double t, double x) const { return fn ? fn(t, x) : 0.0; }
    explicit operator bool() const { return static_cast<bool>(fn); }
};

// The reference's built-in potential kinds (proj/include/laxol/hamiltonian.hpp:34-66,
// proj/src/hamiltonian.cpp:77-117), which the device can evaluate itself
// (step_semidiscrete samples V off the grid).
struct BuiltinPotential {
    enum class Kind { Zero, Const, Cosine };
    enum class TimeMod { None, Sin, Cos };
    Kind kind = Kind::Zero;
    double value = 0.0;  // Const
    double offset = 0.0, amplitude = 0.0;  // Cosine: offset + amplitude*mod(omega t)*cos(frequency*theta(x))
    int frequency = 1;
    TimeMod tmod = TimeMod::None;
    double omega = 0.0;
    double operator()(double t, double x) const;  // host evaluation (the reference's formula)
    Potential callback() const;                   // as a host callback for the other entry points
};
BuiltinPotential potential_zero();
BuiltinPotential potential_const(double c);
BuiltinPotential potential_cosine(double offset, double amplitude, int frequency,
                                  BuiltinPotential::TimeMod tmod = BuiltinPotential::TimeMod::None,
                                  double omega = 0.0);

struct StepStats {
    int64_t block_count = 0;
};

// proj/include/laxol/scheme.hpp:61-90
struct StepRecord {
    double time = 0.0;
    int64_t blocks = 0;
    double drift = 0.0;
    double wall_seconds = 0.0;
};
struct EvolutionTrace {
    std::vector<double> times;
    std::vector<int64_t> snapshot_steps;
    std::vector<GridFn> snapshots;
    std::vector<StepRecord> per_step;
    bool completed = true;
    std::string abort_reason;
};
struct EvolveOptions {
    int64_t snapshot_stride = 0;
    ConvEngine engine = ConvEngine::GpuFast;
    std::vector<int64_t> capture_steps;
};

// proj/include/laxol/splitting.hpp:13-41 (rank 2, periodic, separable
// potential V = a1(x1)*a2(x2) + b(t) given by its host factors).
struct TensorFn {
    std::vector<double> values;
    std::vector<std::size_t> dims;
    double step = 1.0;
    std::vector<double> origins;
    bool periodic = true;
};
struct SeparablePotential2D {
    std::function<double(double)> a1, a2;  // x -> factor, empty = V == 0
    std::function<double(double)> b;       // t -> additive time term
};
struct SplitSpec2D {
    double drift1 = 0.0, drift2 = 0.0;
    SeparablePotential2D potential;
};
// proj/include/laxol/splitting.hpp:20-33 for any rank: one kernel window per axis (mechanical
// or tabulated) and PotentialNd(t, coords) evaluated on the host per grid point
struct SplitSpecND {
    std::vector<KernelWindow> kernels;
    std::function<double(double, std::span<const double>)> potential;  // empty = V == 0
};

// proj/include/laxol/weakkam.hpp:12-29
struct EffectiveHEstimate {
    double h_bar = 0.0;
    int64_t n_steps = 0;
    double residual = 0.0;
    bool converged = false;
};
struct MinPlusMatrix {
    std::size_t n = 0;
    std::vector<double> cost;  // cost[y*n + x]: source y -> target x
    double at(std::size_t y, std::size_t x) const { return cost[y * n + x]; }
    double& at(std::size_t y, std::size_t x) { return cost[y * n + x]; }
};

// The device engine: owns a lob_ctx, device buffers and workspaces.
class Engine {
public:
    explicit Engine(int device = 0);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    // proj/src/scheme.cpp:107-146
    GridFn kinetic_convolve(const GridFn& u, const KernelWindow& kernel, double eta,
                            ConvEngine engine = ConvEngine::GpuFast, int64_t* blocks = nullptr);
    // proj/src/scheme.cpp:148-164
    GridFn step_fully_discrete(const GridFn& u, double t, const Potential& V,
                               const SchemeParams& params, const KernelWindow& kernel,
                               ConvEngine engine = ConvEngine::GpuFast,
                               StepStats* stats = nullptr);
    // proj/src/scheme.cpp:166-206: trapezoid-integrated V along each segment
    // (mechanical(drift) kinetics; the device evaluates V)
    GridFn step_semidiscrete(const GridFn& u, double t, double drift, const BuiltinPotential& V,
                             const SchemeParams& params, int quad_points);
    // proj/src/scheme.cpp:208-272 (time-independent V: device-resident loop)
    EvolutionTrace evolve(const GridFn& u0, double t0, int64_t steps, double drift,
                          const Potential& V, const SchemeParams& params,
                          const EvolveOptions& options = {});
    // proj/src/splitting.cpp:37-99
    TensorFn split_step_nd(const TensorFn& u, double t, const SplitSpec2D& spec,
                           const SchemeParams& params,
                           ConvEngine engine = ConvEngine::GpuDirect);

    // proj/src/splitting.cpp:37-99 for periodic tensors of any rank (all axes n_space)
    TensorFn split_step_nd(const TensorFn& u, double t, const SplitSpecND& spec, const SchemeParams& params,
                           ConvEngine engine = ConvEngine::GpuDirect);

    // Weak-KAM consumers (proj/src/weakkam.cpp), the step and the products on the device.
    // :43-86 (mechanical(drift) kinetics, periodic u0, tau = 1/l)
    EffectiveHEstimate estimate_hbar_drift(const GridFn& u0, double drift, const Potential& V,
                                           const SchemeParams& params, int max_periods, double tol,
                                           ConvEngine engine = ConvEngine::GpuFast);
    // :88-128
    MinPlusMatrix build_period_matrix(double drift, const Potential& V, const SchemeParams& params);
    // :130-146, :148-158, :160-189, :191-201
    MinPlusMatrix minplus_product(const MinPlusMatrix& A, const MinPlusMatrix& B);
    GridFn minplus_apply(const MinPlusMatrix& C, const GridFn& u);
    double eigenvalue_karp(const MinPlusMatrix& C);
    double fixed_point_residual(const GridFn& u, double h_bar, double drift, const Potential& V,
                                const SchemeParams& params, ConvEngine engine = ConvEngine::GpuFast);

    lob_ctx* ctx() const { return ctx_; }

private:
    struct StepCache;
    GridFn periodic_step(const GridFn& u, const KernelWindow& kernel, double eta, ConvEngine engine,
                         const std::vector<double>* tv, int64_t* blocks);
    lob_ctx* ctx_ = nullptr;
    std::unique_ptr<StepCache> cache_;  // device buffers and the resident last output
};

}  // namespace laxol_b200

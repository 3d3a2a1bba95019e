// laxol_gpu — the reference's stepping API over the B200 engines.
//
// A drop-in for the reference library's step path (proj/include/laxol/scheme.hpp),
// compiled against the reference's OWN headers and types: laxol::GridFn, laxol::Kernel,
// laxol::HamiltonianSpec, laxol::SchemeParams, laxol::StepStats, laxol::EvolveOptions,
// laxol::EvolutionTrace, and its exceptions laxol::InvalidInput / laxol::EvaluationError
// (proj/include/laxol/errors.hpp).  Every entry point has the signature of the reference
// function it replaces with the engine switch ConvEngine{Fast, Naive}
// (proj/include/laxol/scheme.hpp:13, dispatch proj/src/scheme.cpp:114-121) widened by the
// device engines:
//
//   Engine::GpuFast   — ConvEngine::Fast on the device: the exact O(n) walk over the
//                       kernel window (lob_minplus_fast_window_f64; == Naive's values) for
//                       eta == 0, the reference's relaxed conv_fast reproduced bit for bit
//                       (lob_minplus_relaxed_f64) for eta > 0;
//   Engine::GpuDirect — ConvEngine::Naive on the device (lob_minplus_direct_f64 / the
//                       windowed lob_minplus_window_f64), bit-identical.
//
// The host side evaluates the reference's own callbacks (Kinetic through build_kernel, the
// Potential per grid point exactly as step_fully_discrete does, proj/src/scheme.cpp:148-164)
// and hands the device rounded tau*V tables; only the C-ABI (include/laxol_b200.h) is called.
#pragma once

#include <cstdint>
#include <memory>

#include "laxol/scheme.hpp"
#include "laxol/splitting.hpp"

namespace laxol_gpu {

enum class Engine { GpuFast, GpuDirect };

class Device {
public:
    explicit Device(int device = 0);
    ~Device();
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;

    // kinetic_convolve (proj/include/laxol/scheme.hpp:52-53, proj/src/scheme.cpp:107-146)
    laxol::GridFn kinetic_convolve(const laxol::GridFn& u, const laxol::Kernel& kernel, double eta, Engine engine,
                                   std::int64_t* blocks = nullptr);

    // step_fully_discrete (proj/include/laxol/scheme.hpp:57-59, proj/src/scheme.cpp:148-164)
    laxol::GridFn step_fully_discrete(const laxol::GridFn& u, double t, const laxol::HamiltonianSpec& spec,
                                      const laxol::SchemeParams& params, const laxol::Kernel& kernel, Engine engine,
                                      laxol::StepStats* stats = nullptr);

    // evolve (proj/include/laxol/scheme.hpp:82-90, proj/src/scheme.cpp:208-272): the state
    // stays on the device between steps (the window engine's statistics carried over); each
    // step's drift is the reference's sequential host sum of u_next - u.
    laxol::EvolutionTrace evolve(const laxol::GridFn& u0, double t0, std::int64_t steps,
                                 const laxol::HamiltonianSpec& spec, const laxol::SchemeParams& params,
                                 Engine engine, const laxol::EvolveOptions& options = {});

    // split_step_nd (proj/include/laxol/splitting.hpp:40-41, proj/src/splitting.cpp:37-99): the
    // axis sweeps in the reference's order on the device (periodic: K2 / relaxed / K1 per
    // lob_split_step_nd_f64; windowed: the exact wall-branch sweeps), tau*V of every point from
    // the reference's PotentialNd callback on the host, subtracted once on the device.  The
    // reference hard-wires ConvEngine::Fast (splitting.cpp:75); `engine` widens it like the
    // other entry points.  Periodic tensors hold n_space samples per axis (the reference's check).
    laxol::TensorFn split_step_nd(const laxol::TensorFn& u, double t, const laxol::SplitSpec& spec,
                                  const laxol::SchemeParams& params, Engine engine = Engine::GpuFast);

    // step_semidiscrete (proj/include/laxol/scheme.hpp:63-64, proj/src/scheme.cpp:166-206) for every
    // Potential kind of the spec: Zero / Const through the device kernel that integrates V itself
    // (lob_step_semidiscrete_f64); Cosine and Custom potentials (any std::function) through the
    // reference's own callbacks on the host -- the candidate costs K[w] - tau/q * trapezoid(V), in
    // its IEEE order, folded over periodic aliases into a source x target matrix -- and the
    // minimum over sources on the device (the tropical GEMM, lob_minplus_gemm_f64).
    laxol::GridFn step_semidiscrete(const laxol::GridFn& u, double t, const laxol::HamiltonianSpec& spec,
                                    const laxol::SchemeParams& params, int quad_points);

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace laxol_gpu

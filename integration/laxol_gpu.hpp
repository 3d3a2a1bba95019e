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

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

}  // namespace laxol_gpu

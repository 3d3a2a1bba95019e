// laxol_gpu — the reference's stepping API over the B200 engines (see laxol_gpu.hpp).
// Compiled against /root/reference/proj/include; calls only the C-ABI of
// include/laxol_b200.h plus the CUDA runtime for the device buffers it owns.
#include "laxol_gpu.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <string>
#include <vector>

#include "laxol/errors.hpp"
#include "laxol/minplus.hpp"
#include "laxol_b200.h"

namespace laxol_gpu {
namespace {

[[noreturn]] void raise(int status, const std::string& msg) {
    if (status == LOB_INVALID_INPUT) throw laxol::InvalidInput(msg);
    if (status == LOB_EVALUATION_ERROR) throw laxol::EvaluationError(msg);
    throw std::runtime_error("laxol_gpu: CUDA error: " + msg);
}

void check_cuda(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("laxol_gpu: ") + where + ": " + cudaGetErrorString(e));
}

// check_u_grid (proj/src/scheme.cpp:18-24)
void check_u_grid(const laxol::GridFn& u, const laxol::SchemeParams& params, const char* who) {
    laxol::validate(u, who);
    if (u.step != params.epsilon())
        throw laxol::InvalidInput(std::string(who) + ": u.step does not match params.epsilon()");
    if (u.periodic && u.n() != static_cast<std::size_t>(params.n_space))
        throw laxol::InvalidInput(std::string(who) + ": periodic u must hold one unit period");
}

// potential_time / sample_coord (proj/src/scheme.cpp:26-35)
double potential_time(double t, const laxol::SchemeParams& params) {
    return params.v_sampling == laxol::PotentialSampling::Arrival ? t + params.tau : t;
}
double sample_coord(const laxol::GridFn& u, std::size_t j) {
    if (u.periodic && j >= u.n()) j -= u.n() * (j / u.n());
    return u.coord(j);
}

// a device buffer that grows on demand
struct DevBuf {
    void* p = nullptr;
    std::size_t bytes = 0;
    void* get(std::size_t want) {
        if (want > bytes) {
            if (p) cudaFree(p);
            p = nullptr;
            check_cuda(cudaMalloc(&p, want), "cudaMalloc");
            bytes = want;
        }
        return p;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

}  // namespace

struct Device::Impl {
    lob_ctx* ctx = nullptr;
    cudaStream_t stream = nullptr;
    DevBuf u, out, ktab, first, tv, blocks, ws, rws;
    ~Impl() {
        if (stream) cudaStreamDestroy(stream);
        if (ctx) lob_ctx_destroy(ctx);
    }
    void ok(int st, const char* who) {
        if (st != LOB_OK) raise(st, std::string(who) + ": " + lob_last_error(ctx));
    }
    template <class T>
    T* up(DevBuf& b, const T* src, std::size_t count) {
        T* d = static_cast<T*>(b.get(count * sizeof(T)));
        check_cuda(cudaMemcpyAsync(d, src, count * sizeof(T), cudaMemcpyHostToDevice, stream), "upload");
        return d;
    }
    void down(double* dst, const void* src, std::size_t count) {
        check_cuda(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToHost, stream), "download");
        check_cuda(cudaStreamSynchronize(stream), "synchronize");
    }

    // One kinetic step of the fundamental samples already in `du`, window `kernel`,
    // potential table `dtv` (nullable), into `dout`; returns the block count when asked.
    // Periodic lines: n samples; windowed: m samples.
    void convolve(const double* du, double* dout, const laxol::GridFn& u, const laxol::Kernel& kernel, double eta,
                  Engine engine, const double* dtv, std::int64_t* blocks, int flags) {
        const std::int64_t n = static_cast<std::int64_t>(kernel.window.n() / 2);  // = n_space
        if (kernel.window.size() != static_cast<std::size_t>(2 * n + 1))
            throw laxol::InvalidInput("kinetic_convolve: kernel window must hold 2 n_space + 1 samples");
        const std::int64_t first_h = kernel.center_index - n;
        const double* dk = up(ktab, kernel.window.values.data(), kernel.window.size());
        const std::int64_t* df = up(first, &first_h, 1);
        if (!u.periodic) {
            // the wall branch of kinetic_convolve (proj/src/scheme.cpp:135-144): both engines
            // take the exact windowed sweep; block statistics from decompose on the host
            if (engine == Engine::GpuFast && eta > 0.0)
                throw laxol::InvalidInput(
                    "kinetic_convolve: the relaxed (eta > 0) fast engine runs periodic lines; use GpuDirect or eta = 0");
            ok(lob_minplus_window_f64(ctx, du, dout, 1, static_cast<std::int64_t>(u.size()), n, dk, 0, df, dtv, 0,
                                      stream),
               "kinetic_convolve");
            if (blocks) *blocks = static_cast<std::int64_t>(laxol::decompose(u, eta).blocks.size());
            return;
        }
        if (static_cast<std::int64_t>(u.n()) != n)
            throw laxol::InvalidInput("kinetic_convolve: periodic u must hold one unit period of the kernel's grid");
        std::int64_t* db = blocks ? static_cast<std::int64_t*>(this->blocks.get(sizeof(std::int64_t))) : nullptr;
        if (engine == Engine::GpuDirect) {
            ok(lob_minplus_direct_f64(ctx, du, dout, 1, n, dk, 0, df, dtv, 0, stream), "kinetic_convolve");
            // the Naive engine reports decompose(u, eta)'s block count (proj/src/scheme.cpp:118-121)
            if (db) ok(lob_block_counts(ctx, du, 1, n, eta, db, stream), "kinetic_convolve");
        } else if (eta > 0.0) {
            // ConvEngine::Fast with eta > 0: the reference's relaxed approximation, bit for bit
            std::size_t wb = 0;
            ok(lob_relaxed_workspace_bytes(1, n, &wb), "kinetic_convolve");
            ok(lob_minplus_relaxed_f64(ctx, du, dout, 1, n, dk, 0, df, dtv, 0, eta, db, rws.get(wb), wb, stream),
               "kinetic_convolve");
        } else {
            std::size_t wb = 0;
            ok(lob_fast_workspace_bytes(1, n, &wb), "kinetic_convolve");
            // (tau: the window engine reads every kinetic cost from the window itself)
            ok(lob_minplus_fast_window_f64(ctx, du, dout, 1, n, dk, 0, df, 1.0, dtv, 0, eta, db, ws.get(wb), wb,
                                           flags, stream),
               "kinetic_convolve");
        }
        if (db) {
            check_cuda(cudaMemcpyAsync(blocks, db, sizeof(std::int64_t), cudaMemcpyDeviceToHost, stream), "blocks");
            check_cuda(cudaStreamSynchronize(stream), "synchronize");
        }
    }
};

Device::Device(int device) : impl_(std::make_unique<Impl>()) {
    const int st = lob_ctx_create(device, &impl_->ctx);
    if (st != LOB_OK) raise(st, "laxol_gpu::Device: no CUDA device");
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    check_cuda(cudaStreamCreateWithFlags(&impl_->stream, cudaStreamNonBlocking), "cudaStreamCreate");
}

Device::~Device() = default;

laxol::GridFn Device::kinetic_convolve(const laxol::GridFn& u, const laxol::Kernel& kernel, double eta,
                                       Engine engine, std::int64_t* blocks) {
    Impl& I = *impl_;
    const std::size_t m = u.periodic ? u.n() : u.size();  // fundamental samples
    const double* du = I.up(I.u, u.values.data(), m);
    double* dout = static_cast<double*>(I.out.get(m * sizeof(double)));
    I.convolve(du, dout, u, kernel, eta, engine, nullptr, blocks, 0);
    std::vector<double> out(u.size());
    I.down(out.data(), dout, m);
    if (u.periodic) out[m] = out[0];  // the seam (aliasing makes conv index N the same as 0)
    return laxol::GridFn{std::move(out), u.step, u.origin, u.periodic};
}

laxol::GridFn Device::step_fully_discrete(const laxol::GridFn& u, double t, const laxol::HamiltonianSpec& spec,
                                          const laxol::SchemeParams& params, const laxol::Kernel& kernel,
                                          Engine engine, laxol::StepStats* stats) {
    check_u_grid(u, params, "step_fully_discrete");
    Impl& I = *impl_;
    const std::size_t m = u.periodic ? u.n() : u.size();
    // tau*V per grid point with the reference's own callback and rounding (proj/src/scheme.cpp:156-162);
    // the device subtracts it in the epilogue (one IEEE subtraction, no FMA)
    const double tvt = potential_time(t, params);
    std::vector<double> tv(m);
    for (std::size_t j = 0; j < m; ++j) {
        const double vx = spec.potential(tvt, sample_coord(u, j));
        if (!std::isfinite(vx)) throw laxol::EvaluationError("step_fully_discrete: potential sample is not finite");
        tv[j] = params.tau * vx;
    }
    const double* du = I.up(I.u, u.values.data(), m);
    const double* dtv = I.up(I.tv, tv.data(), m);
    double* dout = static_cast<double*>(I.out.get(m * sizeof(double)));
    std::int64_t blocks = 0;
    I.convolve(du, dout, u, kernel, params.eta, engine, dtv, &blocks, 0);
    if (stats) stats->block_count = blocks;
    std::vector<double> out(u.size());
    I.down(out.data(), dout, m);
    if (u.periodic) out[m] = out[0];
    return laxol::GridFn{std::move(out), u.step, u.origin, u.periodic};
}

laxol::EvolutionTrace Device::evolve(const laxol::GridFn& u0, double t0, std::int64_t steps,
                                     const laxol::HamiltonianSpec& spec, const laxol::SchemeParams& params,
                                     Engine engine, const laxol::EvolveOptions& options) {
    if (steps < 0) throw laxol::InvalidInput("evolve: steps must be >= 0");
    check_u_grid(u0, params, "evolve");
    const laxol::Kernel kernel = laxol::build_kernel(spec, params);
    Impl& I = *impl_;

    std::int64_t stride = options.snapshot_stride;
    if (stride <= 0) stride = steps <= 1024 ? 1 : (steps + 1023) / 1024;
    std::vector<std::int64_t> capture = options.capture_steps;
    std::sort(capture.begin(), capture.end());
    auto keep = [&](std::int64_t k) {
        if (k == 0 || k == steps) return true;
        if (k % stride == 0) return true;
        return std::binary_search(capture.begin(), capture.end(), k);
    };

    laxol::EvolutionTrace trace;
    trace.per_step.reserve(static_cast<std::size_t>(steps));
    laxol::GridFn u = u0;
    if (keep(0)) {
        trace.times.push_back(t0);
        trace.snapshot_steps.push_back(0);
        trace.snapshots.push_back(u);
    }
    const std::size_t m = u0.periodic ? u0.n() : u0.size();
    // double-buffered device state; tau*V tables per step (time-dependent V) or once
    DevBuf a, b;
    double* cur = static_cast<double*>(a.get(m * sizeof(double)));
    double* nxt = static_cast<double*>(b.get(m * sizeof(double)));
    check_cuda(cudaMemcpyAsync(cur, u0.values.data(), m * sizeof(double), cudaMemcpyHostToDevice, I.stream), "upload");
    std::vector<double> tv(m), host(u0.size());
    const double* dtv = nullptr;
    bool tv_fixed = false;
    for (std::int64_t i = 0; i < steps; ++i) {
        const double t = t0 + static_cast<double>(i) * params.tau;
        const auto started = std::chrono::steady_clock::now();
        if (!tv_fixed) {
            const double tvt = potential_time(t, params);
            for (std::size_t j = 0; j < m; ++j) {
                const double vx = spec.potential(tvt, sample_coord(u, j));
                if (!std::isfinite(vx))
                    throw laxol::EvaluationError("step_fully_discrete: potential sample is not finite");
                tv[j] = params.tau * vx;
            }
            dtv = I.up(I.tv, tv.data(), m);
            tv_fixed = !spec.potential.time_dependent();
        }
        std::int64_t blocks = 0;
        // consecutive steps on one workspace: the statistics of this step's input were written
        // by the previous step's epilogue
        I.convolve(cur, nxt, u, kernel, params.eta, engine, dtv, &blocks, i ? LOB_FAST_STATS_VALID : 0);
        I.down(host.data(), nxt, m);
        if (u.periodic) host[m] = host[0];
        const std::chrono::duration<double> elapsed = std::chrono::steady_clock::now() - started;

        // the reference's drift: a sequential sum over the fundamental domain (scheme.cpp:244-251)
        double drift = 0.0;
        bool finite = true;
        for (std::size_t j = 0; j < m; ++j) {
            drift += host[j] - u.values[j];
            finite = finite && std::isfinite(host[j]);
        }
        drift /= static_cast<double>(m);
        const double t_next = t0 + static_cast<double>(i + 1) * params.tau;
        trace.per_step.push_back({t_next, blocks, drift, elapsed.count()});
        u.values = host;
        std::swap(cur, nxt);
        if (!finite) {
            trace.completed = false;
            trace.abort_reason = "non-finite value after step " + std::to_string(i + 1);
            trace.times.push_back(t_next);
            trace.snapshot_steps.push_back(i + 1);
            trace.snapshots.push_back(u);
            return trace;
        }
        if (keep(i + 1)) {
            trace.times.push_back(t_next);
            trace.snapshot_steps.push_back(i + 1);
            trace.snapshots.push_back(u);
        }
    }
    return trace;
}

}  // namespace laxol_gpu

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


laxol::TensorFn Device::split_step_nd(const laxol::TensorFn& u, double t, const laxol::SplitSpec& spec,
                                      const laxol::SchemeParams& params, Engine engine) {
    // the reference's argument checks (proj/src/splitting.cpp:39-50), same messages
    if (spec.kinetics.size() != u.rank())
        throw laxol::InvalidInput("split_step_nd: kinetic part is not separable over the tensor axes (" +
                                  std::to_string(spec.kinetics.size()) + " conjugates for rank " +
                                  std::to_string(u.rank()) + ")");
    if (u.step != params.epsilon())
        throw laxol::InvalidInput("split_step_nd: tensor step does not match params.epsilon()");
    if (u.periodic) {
        for (std::size_t d : u.dims)
            if (d != static_cast<std::size_t>(params.n_space))
                throw laxol::InvalidInput("split_step_nd: periodic axes must hold one unit period");
    }
    Impl& I = *impl_;
    const int rank = static_cast<int>(u.rank());
    const std::int64_t n = params.n_space, W = 2 * n + 1;
    // per-axis windows: the reference's build_kernel (proj/src/splitting.cpp:55)
    std::vector<double> ktabs(static_cast<std::size_t>(rank * W));
    std::vector<std::int64_t> firsts(rank), dims(rank);
    std::vector<double> drifts(rank);
    bool mechanical = true;
    for (int a = 0; a < rank; ++a) {
        const laxol::Kernel k = laxol::build_kernel(spec.kinetics[a], params);
        if (k.window.size() != static_cast<std::size_t>(W))
            throw laxol::InvalidInput("split_step_nd: kernel window must hold 2 n_space + 1 samples");
        std::copy(k.window.values.begin(), k.window.values.end(), ktabs.begin() + a * W);
        firsts[a] = k.center_index - n;
        drifts[a] = spec.kinetics[a].drift;
        dims[a] = static_cast<std::int64_t>(u.dims[a]);
        mechanical = mechanical && spec.kinetics[a].kind == laxol::Kinetic::Kind::Mechanical;
    }
    // tau*V of every point, the reference's loop (proj/src/splitting.cpp:79-97)
    const std::size_t total = u.size();
    std::vector<double> tv;
    if (spec.potential) {
        tv.resize(total);
        const double tt = params.v_sampling == laxol::PotentialSampling::Arrival ? t + params.tau : t;
        std::vector<std::size_t> strides(rank, 1);
        for (int a = rank - 1; a > 0; --a) strides[a - 1] = strides[a] * u.dims[a];
        std::vector<double> coords(rank);
        for (std::size_t flat = 0; flat < total; ++flat) {
            std::size_t rem = flat;
            for (int a = 0; a < rank; ++a) {
                const std::size_t idx = rem / strides[a];
                rem %= strides[a];
                coords[a] = u.origins[a] + static_cast<double>(idx) * u.step;
            }
            const double v = spec.potential(tt, coords);
            if (!std::isfinite(v)) throw laxol::EvaluationError("split_step_nd: potential sample is not finite");
            tv[flat] = params.tau * v;
        }
    }
    DevBuf tmpb;
    const double* du = I.up(I.u, u.values.data(), total);
    double* dout = static_cast<double*>(I.out.get(total * sizeof(double)));
    double* dtmp = static_cast<double*>(tmpb.get(total * sizeof(double)));
    const double* dk = I.up(I.ktab, ktabs.data(), ktabs.size());
    const double* dtv = spec.potential ? I.up(I.tv, tv.data(), total) : nullptr;
    if (u.periodic) {
        int eng = LOB_ENGINE_DIRECT;
        if (engine == Engine::GpuFast) eng = (params.eta > 0.0 || !mechanical) ? LOB_ENGINE_RELAXED : LOB_ENGINE_FAST;
        std::size_t wb = 0;
        void* ws = nullptr;
        if (eng == LOB_ENGINE_FAST) {
            I.ok(lob_fast_workspace_bytes(static_cast<std::int64_t>(total) / n, n, &wb), "split_step_nd");
            ws = I.ws.get(wb);
        }
        I.ok(lob_split_step_nd_f64(I.ctx, du, dout, dtmp, rank, n, params.tau, dk, firsts.data(), drifts.data(), dtv,
                                   params.eta, eng, ws, wb, I.stream),
             "split_step_nd");
    } else {
        // the wall branch (proj/src/scheme.cpp:135-144): the exact windowed sweeps; ConvEngine::Fast with
        // eta > 0 is the reference's relaxed approximation, which runs periodic lines only here
        if (engine == Engine::GpuFast && params.eta > 0.0)
            throw laxol::InvalidInput(
                "split_step_nd: the relaxed (eta > 0) fast engine runs periodic tensors; use GpuDirect or eta = 0");
        I.ok(lob_split_step_nd_window_f64(I.ctx, du, dout, dtmp, rank, dims.data(), n, params.tau, dk, firsts.data(),
                                          dtv, I.stream),
             "split_step_nd");
    }
    laxol::TensorFn out = u;
    I.down(out.values.data(), dout, total);
    return out;
}

laxol::GridFn Device::step_semidiscrete(const laxol::GridFn& u, double t, const laxol::HamiltonianSpec& spec,
                                        const laxol::SchemeParams& params, int quad_points) {
    if (quad_points < 1) throw laxol::InvalidInput("step_semidiscrete: quad_points must be >= 1");
    check_u_grid(u, params, "step_semidiscrete");
    const laxol::Kernel kernel = laxol::build_kernel(spec, params);
    Impl& I = *impl_;
    const double tau = params.tau;
    const std::int64_t n = params.n_space, period = static_cast<std::int64_t>(u.n());
    const std::int64_t first = kernel.center_index - static_cast<std::int64_t>(kernel.window.n() / 2);
    const std::size_t m = u.periodic ? u.n() : u.size();  // fundamental samples (sources and outputs)
    const laxol::Potential& V = spec.potential;
    std::vector<double> out(u.size());
    if (V.kind == laxol::Potential::Kind::Zero || V.kind == laxol::Potential::Kind::Const) {
        // V integrates exactly on the device for these kinds
        lob_potential lp{};
        lp.kind = V.kind == laxol::Potential::Kind::Zero ? LOB_POTENTIAL_ZERO : LOB_POTENTIAL_CONST;
        lp.value = V.value;
        const double* du = I.up(I.u, u.values.data(), m);
        const double* dk = I.up(I.ktab, kernel.window.values.data(), kernel.window.size());
        double* dout = static_cast<double*>(I.out.get(m * sizeof(double)));
        I.ok(lob_step_semidiscrete_f64(I.ctx, du, dout, 1, static_cast<std::int64_t>(m), n, u.periodic ? 1 : 0,
                                       u.origin, dk, first, t, tau, &lp, quad_points, I.stream),
             "step_semidiscrete");
        I.down(out.data(), dout, m);
    } else {
        // the candidate costs with the reference's callbacks and IEEE order (proj/src/scheme.cpp:180-196),
        // C[y][j] = min over the windows' displacements d with source y of cost(j, d); the minimum over
        // sources min_y u[y] + C[y][j] is the reference's min over d (fl() is monotone)
        const int q = quad_points;
        constexpr double kInf = std::numeric_limits<double>::infinity();
        std::vector<double> C(m * m, kInf);
        for (std::size_t j = 0; j < m; ++j) {
            const double x = sample_coord(u, j);
            for (std::size_t w = 0; w < kernel.window.size(); ++w) {
                const std::int64_t d = first + static_cast<std::int64_t>(w);
                const std::int64_t src = static_cast<std::int64_t>(j) - d;
                std::int64_t src_idx = src;
                if (u.periodic)
                    src_idx = ((src % period) + period) % period;
                else if (src < 0 || src >= static_cast<std::int64_t>(u.size()))
                    continue;
                const double y = x - static_cast<double>(d) * u.step;
                double acc = 0.5 * (V(t, y) + V(t + tau, x));
                for (int r = 1; r < q; ++r) {
                    const double frac = static_cast<double>(r) / static_cast<double>(q);
                    acc += V(t + frac * tau, y + frac * (x - y));
                }
                const double integral = tau / static_cast<double>(q) * acc;
                const double cost = kernel.window.values[w] - integral;
                double& c = C[static_cast<std::size_t>(src_idx) * m + j];
                c = std::min(c, cost);
            }
        }
        DevBuf cb;
        double* dC = static_cast<double*>(cb.get(C.size() * sizeof(double)));
        check_cuda(cudaMemcpyAsync(dC, C.data(), C.size() * sizeof(double), cudaMemcpyHostToDevice, I.stream), "upload");
        const double* du = I.up(I.u, u.values.data(), m);
        double* dout = static_cast<double*>(I.out.get(m * sizeof(double)));
        const std::int64_t mm = static_cast<std::int64_t>(m);
        I.ok(lob_minplus_gemm_f64(I.ctx, du, mm, dC, mm, dout, mm, 1, mm, mm, I.stream), "step_semidiscrete");
        I.down(out.data(), dout, m);
    }
    for (std::size_t j = 0; j < m; ++j)
        if (out[j] == std::numeric_limits<double>::infinity())
            throw laxol::EvaluationError("step_semidiscrete: no candidate source for grid index " + std::to_string(j));
    if (u.periodic) out[m] = out[0];  // x and the sources of j = n are those of j = 0
    return laxol::GridFn{std::move(out), u.step, u.origin, u.periodic};
}

}  // namespace laxol_gpu

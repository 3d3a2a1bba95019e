// C++ host API over the laxol_b200 C-ABI: the reference's stepping calls
// (proj/src/scheme.cpp, proj/src/splitting.cpp) with the B200 engines.
// Semantics follow the reference line by line where it matters for parity:
//  * periodic GridFn = closed period, seam duplicated (proj/src/grid_fn.cpp:30-36);
//  * V is sampled on the host through the user's callback at t+tau (Arrival)
//    or t (Departure), per fundamental grid index (proj/src/scheme.cpp:26-35,156-162),
//    and tau*V is rounded once on the host;
//  * evolve keeps snapshots 0, every stride-th, captures and the last
//    (proj/src/scheme.cpp:215-225), records per-step drift and block counts,
//    and stops after the first step producing a non-finite value
//    (proj/src/scheme.cpp:257-264).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "laxol_b200.hpp"

namespace laxol_b200 {

namespace {

void check_status(int st, lob_ctx* ctx, const char* where) {
    if (st == LOB_OK) return;
    const std::string msg = std::string(where) + ": " + (ctx ? lob_last_error(ctx) : "");
    if (st == LOB_INVALID_INPUT) throw InvalidInput(msg);
    if (st == LOB_EVALUATION_ERROR) throw EvaluationError(msg);
    throw std::runtime_error(msg + " (CUDA error; there is no CPU fallback)");
}

void check_cuda(cudaError_t e, const char* where) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(where) + ": " + cudaGetErrorString(e));
}

// RAII device buffer
template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    explicit DevBuf(size_t count) : n(count) {
        if (count) check_cuda(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void upload(const T* h, size_t count) {
        check_cuda(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice), "H2D");
    }
    void download(T* h, size_t count) const {
        check_cuda(cudaMemcpy(h, p, count * sizeof(T), cudaMemcpyDeviceToHost), "D2H");
    }
};

void check_u_grid(const GridFn& u, const SchemeParams& params, const char* who) {
    // proj/src/scheme.cpp:18-24 + proj/src/grid_fn.cpp:11-22
    if (u.values.empty()) throw InvalidInput(std::string(who) + ": empty sample vector");
    if (!(u.step > 0.0)) throw InvalidInput(std::string(who) + ": step must be positive");
    for (double v : u.values)
        if (!std::isfinite(v)) throw InvalidInput(std::string(who) + ": non-finite sample");
    if (u.periodic) {
        if (u.n() < 1) throw InvalidInput(std::string(who) + ": periodic function needs n >= 1");
        if (u.values.front() != u.values.back())
            throw InvalidInput(std::string(who) + ": periodic seam samples differ");
    }
    if (u.step != params.epsilon())
        throw InvalidInput(std::string(who) + ": u.step does not match params.epsilon()");
    if (u.periodic && u.n() != static_cast<std::size_t>(params.n_space))
        throw InvalidInput(std::string(who) + ": periodic u must hold one unit period");
}

double potential_time(double t, const SchemeParams& params) {
    return params.v_sampling == PotentialSampling::Arrival ? t + params.tau : t;
}

// tau*V(tv_time, x_j) for j < count (fundamental indices), host callback
std::vector<double> tabulate_tv(const GridFn& u, const Potential& V, double tt, double tau,
                                std::size_t count) {
    std::vector<double> tv(count);
    for (std::size_t j = 0; j < count; ++j) {
        const double vx = V(tt, u.coord(j));
        if (!std::isfinite(vx))
            throw EvaluationError("step_fully_discrete: potential sample is not finite");
        tv[j] = tau * vx;
    }
    return tv;
}

// ConvEngine::GpuFast with eta > 0 is the reference's relaxed fast engine
// (ConvEngine::Fast, proj/src/minplus.cpp:195-252); at eta == 0 both are exact.
int engine_code(ConvEngine e, double eta = 0.0) {
    if (e == ConvEngine::GpuFast) return eta > 0.0 ? LOB_ENGINE_RELAXED : LOB_ENGINE_FAST;
    if (e == ConvEngine::GpuDirect) return LOB_ENGINE_DIRECT;
    throw InvalidInput(
        "laxol_b200: ConvEngine::Fast/Naive are the reference's CPU engines; use GpuFast or GpuDirect");
}

}  // namespace

GridFn make_periodic(std::vector<double> fundamental, double step, double origin) {
    if (fundamental.empty()) throw InvalidInput("make_periodic: empty sample vector");
    fundamental.push_back(fundamental.front());
    GridFn f{std::move(fundamental), step, origin, true};
    return f;
}

GridFn make_grid_fn(std::vector<double> values, double step, double origin) {
    if (values.empty()) throw InvalidInput("make_grid_fn: empty sample vector");
    return GridFn{std::move(values), step, origin, false};
}

void validate(const SchemeParams& p) {
    if (p.n_space < 1) throw InvalidInput("SchemeParams: n_space must be >= 1");
    if (!(p.tau > 0.0)) throw InvalidInput("SchemeParams: tau must be positive");
    if (p.eta < 0.0) throw InvalidInput("SchemeParams: eta must be >= 0");
    if (!(p.h0 > 0.0)) throw InvalidInput("SchemeParams: h0 must be positive");
    const double ratio = p.epsilon() / p.tau;
    if (ratio >= p.h0) {
        if (p.anti_cfl == AntiCflMode::Fail)
            throw InvalidInput("SchemeParams: epsilon/tau = " + std::to_string(ratio) +
                               " violates the bound epsilon/tau < h0 = " + std::to_string(p.h0));
        std::fprintf(stderr, "laxol: warning: epsilon/tau = %g exceeds h0 = %g\n", ratio, p.h0);
    }
}

// Device state kept between calls: grow-only buffers, the K2 workspace, and the last
// output still on the device (so a step whose input is the previous step's output uploads
// nothing and keeps the fast engine's statistics: LOB_FAST_STATS_VALID).
struct Engine::StepCache {
    cudaStream_t stream = nullptr;
    void *u = nullptr, *out = nullptr, *ktab = nullptr, *first = nullptr, *drift = nullptr, *tv = nullptr,
         *blocks = nullptr, *ws = nullptr;
    size_t cap[8] = {};
    std::vector<double> last_out, last_window;  // host copies of the device `u` and window
    int64_t last_n = -1;
    int last_code = -1;
    bool resident = false;  // the device `u` buffer holds last_out
    void* get(int slot, void*& p, size_t bytes) {
        if (bytes > cap[slot]) {
            if (p) cudaFree(p);
            p = nullptr;
            check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
            cap[slot] = bytes;
        }
        return p;
    }
    ~StepCache() {
        for (void* p : {u, out, ktab, first, drift, tv, blocks, ws})
            if (p) cudaFree(p);
        if (stream) cudaStreamDestroy(stream);
    }
};

Engine::Engine(int device) {
    const int st = lob_ctx_create(device, &ctx_);
    if (st != LOB_OK)
        throw std::runtime_error("laxol_b200: no usable CUDA device (status " + std::to_string(st) +
                                 "); there is no CPU fallback");
    cache_ = std::make_unique<StepCache>();
    check_cuda(cudaStreamCreateWithFlags(&cache_->stream, cudaStreamNonBlocking), "cudaStreamCreate");
}

Engine::~Engine() {
    cache_.reset();
    lob_ctx_destroy(ctx_);
}

// One periodic step: min-plus with the window (+ tau*V from `tv`, fused on the device).
GridFn Engine::periodic_step(const GridFn& u, const KernelWindow& kernel, double eta, ConvEngine engine,
                             const std::vector<double>* tv, int64_t* blocks) {
    StepCache& C = *cache_;
    const int64_t n = kernel.n_space;
    if (static_cast<int64_t>(u.n()) != n) throw InvalidInput("kinetic_convolve: periodic u must hold one unit period");
    int code = engine_code(engine, eta);
    const size_t nb = static_cast<size_t>(n) * sizeof(double), wb = kernel.window.size() * sizeof(double);
    // the input is the previous call's output (same values, same window and engine): already on the
    // device, with its statistics
    const bool same_window = C.last_window.size() == kernel.window.size() &&
                             std::memcmp(C.last_window.data(), kernel.window.data(), wb) == 0;
    const bool resident = C.resident && C.last_n == n && C.last_code == code && same_window &&
                          std::memcmp(C.last_out.data(), u.values.data(), nb) == 0;
    double* du = static_cast<double*>(C.get(0, C.u, nb));
    double* dout = static_cast<double*>(C.get(1, C.out, nb));
    if (!resident) check_cuda(cudaMemcpyAsync(du, u.values.data(), nb, cudaMemcpyHostToDevice, C.stream), "H2D");
    if (!same_window) {
        C.last_window = kernel.window;
        check_cuda(cudaMemcpyAsync(C.get(2, C.ktab, wb), kernel.window.data(), wb, cudaMemcpyHostToDevice, C.stream),
                   "H2D");
        check_cuda(cudaMemcpyAsync(C.get(3, C.first, 8), &kernel.first, 8, cudaMemcpyHostToDevice, C.stream), "H2D");
        check_cuda(cudaMemcpyAsync(C.get(4, C.drift, 8), &kernel.drift, 8, cudaMemcpyHostToDevice, C.stream), "H2D");
        check_cuda(cudaStreamSynchronize(C.stream), "H2D");  // the host copies above are stack/temporary
    }
    const double* dtv = nullptr;
    if (tv) {
        dtv = static_cast<double*>(C.get(5, C.tv, nb));
        check_cuda(cudaMemcpyAsync(const_cast<double*>(dtv), tv->data(), nb, cudaMemcpyHostToDevice, C.stream), "H2D");
    }
    int64_t* db = static_cast<int64_t*>(C.get(6, C.blocks, 8));
    const double* dk = static_cast<const double*>(C.ktab);
    const int64_t* df = static_cast<const int64_t*>(C.first);
    if (code == LOB_ENGINE_FAST) {
        size_t wsb = 0;
        lob_fast_workspace_bytes(1, n, &wsb);
        void* ws = C.get(7, C.ws, wsb);
        const int flags = resident ? LOB_FAST_STATS_VALID : 0;
        if (kernel.mechanical)
            check_status(lob_minplus_fast_f64(ctx_, du, dout, 1, n, static_cast<const double*>(C.drift), kernel.tau,
                                              dtv, 0, eta, blocks ? db : nullptr, ws, wsb, flags, C.stream),
                         ctx_, "kinetic_convolve");
        else  // any convex window (tabulated conjugates): the window engine
            check_status(lob_minplus_fast_window_f64(ctx_, du, dout, 1, n, dk, 0, df, kernel.tau, dtv, 0, eta,
                                                     blocks ? db : nullptr, ws, wsb, flags, C.stream),
                         ctx_, "kinetic_convolve");
    } else if (code == LOB_ENGINE_RELAXED) {
        size_t wsb = 0;
        lob_relaxed_workspace_bytes(1, n, &wsb);
        void* ws = C.get(7, C.ws, std::max(wsb, C.cap[7]));
        check_status(lob_minplus_relaxed_f64(ctx_, du, dout, 1, n, dk, 0, df, dtv, 0, eta, blocks ? db : nullptr, ws,
                                             C.cap[7], C.stream),
                     ctx_, "kinetic_convolve");
    } else {
        check_status(lob_minplus_direct_f64(ctx_, du, dout, 1, n, dk, 0, df, dtv, 0, C.stream), ctx_,
                     "kinetic_convolve");
        if (blocks) check_status(lob_block_counts(ctx_, du, 1, n, eta, db, C.stream), ctx_, "block counts");
    }
    std::vector<double> out(static_cast<size_t>(n) + 1);
    check_cuda(cudaMemcpyAsync(out.data(), dout, nb, cudaMemcpyDeviceToHost, C.stream), "D2H");
    int64_t bh = 0;
    if (blocks) check_cuda(cudaMemcpyAsync(&bh, db, 8, cudaMemcpyDeviceToHost, C.stream), "D2H");
    check_cuda(cudaStreamSynchronize(C.stream), "kinetic_convolve");
    out[n] = out[0];
    if (blocks) *blocks = bh;
    // the output becomes the next call's resident input (the fast engine reads u_{k+1}'s
    // statistics written by this call's epilogue; the K2 workspace tracks pointers, so
    // swap the buffers rather than copying)
    std::swap(C.u, C.out);
    std::swap(C.cap[0], C.cap[1]);
    C.last_out.assign(out.begin(), out.begin() + n);
    C.last_n = n;
    C.last_code = code;
    C.resident = true;
    return GridFn{std::move(out), u.step, u.origin, true};
}

GridFn Engine::kinetic_convolve(const GridFn& u, const KernelWindow& kernel, double eta,
                                ConvEngine engine, int64_t* blocks) {
    const int64_t n = kernel.n_space;
    (void)engine_code(engine, eta);  // rejects the CPU engines
    if (u.periodic) return periodic_step(u, kernel, eta, engine, nullptr, blocks);
    // windowed domain: direct engine (proj/src/scheme.cpp:135-144)
    const int64_t m = static_cast<int64_t>(u.size());
    DevBuf<double> du(m), dout(m), dk(kernel.window.size());
    DevBuf<int64_t> df(1);
    du.upload(u.values.data(), m);
    dk.upload(kernel.window.data(), kernel.window.size());
    df.upload(&kernel.first, 1);
    check_status(lob_minplus_window_f64(ctx_, du.p, dout.p, 1, m, n, dk.p, 0, df.p, nullptr, 0, nullptr),
                 ctx_, "kinetic_convolve");
    std::vector<double> out(m);
    dout.download(out.data(), m);
    if (blocks) {
        // decompose() of the windowed samples (plain vector): host scan like the reference
        int64_t count = 0;
        std::size_t b = 0;
        const std::size_t nn = u.n();
        std::vector<double> s(nn);
        for (std::size_t i = 0; i < nn; ++i) s[i] = u.values[i + 1] - u.values[i];
        if (nn == 0) count = 1;
        while (b < nn) {
            bool det = false, convex = true;
            std::size_t e = b + 1;
            while (e < nn) {
                const double inc = s[e] - s[e - 1];
                if (!det) {
                    if (inc > eta) det = true, convex = true;
                    else if (inc < -eta) det = true, convex = false;
                } else if (convex ? !(inc >= -eta) : !(inc <= eta)) {
                    break;
                }
                ++e;
            }
            ++count;
            b = e;
        }
        *blocks = count;
    }
    return GridFn{std::move(out), u.step, u.origin, false};
}

GridFn Engine::step_fully_discrete(const GridFn& u, double t, const Potential& V,
                                   const SchemeParams& params, const KernelWindow& kernel,
                                   ConvEngine engine, StepStats* stats) {
    check_u_grid(u, params, "step_fully_discrete");
    const double tt = potential_time(t, params);
    const std::size_t fund = u.periodic ? u.n() : u.size();
    // out[j] -= tau*V(t', x_{j mod n}) (proj/src/scheme.cpp:156-162): tau*V rounded on the host,
    // subtracted in the kernel's epilogue (periodic) or here (windowed)
    const std::vector<double> tv = tabulate_tv(u, V, tt, params.tau, fund);
    int64_t blocks = 0;
    if (u.periodic) {
        GridFn out = periodic_step(u, kernel, params.eta, engine, &tv, &blocks);
        if (stats) stats->block_count = blocks;
        return out;
    }
    GridFn out = kinetic_convolve(u, kernel, params.eta, engine, &blocks);
    if (stats) stats->block_count = blocks;
    for (std::size_t j = 0; j < out.size(); ++j) out.values[j] -= tv[j];
    return out;
}

EvolutionTrace Engine::evolve(const GridFn& u0, double t0, int64_t steps, double drift,
                              const Potential& V, const SchemeParams& params,
                              const EvolveOptions& options) {
    if (steps < 0) throw InvalidInput("evolve: steps must be >= 0");
    check_u_grid(u0, params, "evolve");
    validate(params);
    if (!u0.periodic) {
        // windowed domain (proj/src/scheme.cpp:208-272 with kinetic_convolve's wall branch,
        // :135-144): step by step through the windowed K1 kernel, the drift and the
        // non-finite check on the host in the reference's order
        const KernelWindow kernel = build_kernel_mech(params, drift);
        int64_t stride = options.snapshot_stride;
        if (stride <= 0) stride = steps <= 1024 ? 1 : (steps + 1023) / 1024;
        std::vector<int64_t> capture = options.capture_steps;
        std::sort(capture.begin(), capture.end());
        auto keep = [&](int64_t i) {
            return i == 0 || i == steps || i % stride == 0 || std::binary_search(capture.begin(), capture.end(), i);
        };
        EvolutionTrace trace;
        trace.times.push_back(t0);
        trace.snapshot_steps.push_back(0);
        trace.snapshots.push_back(u0);
        GridFn u = u0;
        for (int64_t i = 0; i < steps; ++i) {
            const double t = t0 + static_cast<double>(i) * params.tau;
            const auto started = std::chrono::steady_clock::now();
            StepStats stats;
            GridFn next = step_fully_discrete(u, t, V, params, kernel, ConvEngine::GpuDirect, &stats);
            const std::chrono::duration<double> el = std::chrono::steady_clock::now() - started;
            double d = 0.0;
            bool finite = true;
            for (std::size_t j = 0; j < u.size(); ++j) {
                d += next.values[j] - u.values[j];
                finite = finite && std::isfinite(next.values[j]);
            }
            d /= static_cast<double>(u.size());
            const double t_next = t0 + static_cast<double>(i + 1) * params.tau;
            trace.per_step.push_back({t_next, stats.block_count, d, el.count()});
            u = std::move(next);
            if (!finite || keep(i + 1)) {
                trace.times.push_back(t_next);
                trace.snapshot_steps.push_back(i + 1);
                trace.snapshots.push_back(u);
            }
            if (!finite) {
                trace.completed = false;
                trace.abort_reason = "non-finite value after step " + std::to_string(i + 1);
                break;
            }
        }
        return trace;
    }
    const int code = engine_code(options.engine, params.eta);
    const int64_t n = params.n_space;

    int64_t stride = options.snapshot_stride;
    if (stride <= 0) stride = steps <= 1024 ? 1 : (steps + 1023) / 1024;
    std::vector<int64_t> capture = options.capture_steps;
    std::sort(capture.begin(), capture.end());
    auto keep = [&](int64_t i) {
        if (i == 0 || i == steps) return true;
        if (i % stride == 0) return true;
        return std::binary_search(capture.begin(), capture.end(), i);
    };

    EvolutionTrace trace;
    trace.times.push_back(t0);
    trace.snapshot_steps.push_back(0);
    trace.snapshots.push_back(u0);
    if (steps == 0) return trace;

    DevBuf<double> du(n), dscr(n), dd(1), dtv(n), dstart(n);
    du.upload(u0.values.data(), n);
    dd.upload(&drift, 1);
    size_t wsb = 0;
    lob_fast_workspace_bytes(1, n, &wsb);
    DevBuf<unsigned char> ws(wsb);
    DevBuf<double> dstep_drift(static_cast<size_t>(steps));
    DevBuf<int64_t> dstep_blocks(static_cast<size_t>(steps));
    const bool tdep = V && V.time_dependent;
    std::vector<double> tv;
    if (V && !tdep) {
        tv = tabulate_tv(u0, V, potential_time(t0, params), params.tau, n);
        dtv.upload(tv.data(), n);
    }
    std::vector<double> host(static_cast<size_t>(n) + 1);
    int64_t done = 0;
    bool aborted = false;
    while (done < steps && !aborted) {
        // run up to the next snapshot step (one step at a time for time-dependent V)
        int64_t next = done + 1;
        if (!tdep)
            while (next < steps && !keep(next)) ++next;
        const int64_t chunk = next - done;
        if (tdep) {
            tv = tabulate_tv(u0, V, potential_time(t0 + static_cast<double>(done) * params.tau, params),
                             params.tau, n);
            dtv.upload(tv.data(), n);
        }
        int64_t completed = 0;
        // the chunk's start state, for an exact replay after a non-finite abort (the last kept
        // snapshot is older than the chunk when V is time dependent and steps > 1024)
        check_cuda(cudaMemcpy(dstart.p, du.p, n * sizeof(double), cudaMemcpyDeviceToDevice), "D2D");
        const auto started = std::chrono::steady_clock::now();
        const int st = lob_evolve_f64(ctx_, du.p, dscr.p, 1, n, dd.p, params.tau, V ? dtv.p : nullptr, 0,
                                      params.eta, code, chunk, dstep_drift.p + done,
                                      dstep_blocks.p + done, &completed, ws.p, wsb, nullptr);
        const std::chrono::duration<double> el = std::chrono::steady_clock::now() - started;
        if (st == LOB_EVALUATION_ERROR) {
            aborted = true;
        } else {
            check_status(st, ctx_, "evolve");
        }
        std::vector<double> sd(static_cast<size_t>(completed));
        std::vector<int64_t> sb(static_cast<size_t>(completed));
        if (completed) {
            dstep_drift.download(sd.data(), completed);
            check_cuda(cudaMemcpy(sb.data(), dstep_blocks.p + done, completed * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost),
                       "D2H");
            check_cuda(cudaMemcpy(sd.data(), dstep_drift.p + done, completed * sizeof(double),
                                  cudaMemcpyDeviceToHost),
                       "D2H");
        }
        for (int64_t k = 0; k < completed; ++k)
            trace.per_step.push_back({t0 + static_cast<double>(done + k + 1) * params.tau, sb[k], sd[k],
                                      el.count() / static_cast<double>(completed)});
        done += completed;
        if (aborted) {
            // lob_evolve_f64 may have advanced past the offending step inside its
            // check interval: replay exactly `completed` steps from the chunk start
            trace.completed = false;
            trace.abort_reason = "non-finite value after step " + std::to_string(done);
            check_cuda(cudaMemcpy(du.p, dstart.p, n * sizeof(double), cudaMemcpyDeviceToDevice), "D2D");
            int64_t again = 0;
            lob_evolve_f64(ctx_, du.p, dscr.p, 1, n, dd.p, params.tau, V ? dtv.p : nullptr, 0, params.eta,
                           code, completed, nullptr, nullptr, &again, ws.p, wsb, nullptr);
        }
        du.download(host.data(), n);
        host[n] = host[0];
        if (aborted || keep(done)) {
            trace.times.push_back(t0 + static_cast<double>(done) * params.tau);
            trace.snapshot_steps.push_back(done);
            trace.snapshots.push_back(GridFn{host, u0.step, u0.origin, true});
        }
        if (st == LOB_EVALUATION_ERROR) break;
    }
    return trace;
}

TensorFn Engine::split_step_nd(const TensorFn& u, double t, const SplitSpec2D& spec,
                               const SchemeParams& params, ConvEngine engine) {
    // proj/src/splitting.cpp:37-49 validation
    if (u.dims.size() != 2)
        throw InvalidInput("split_step_nd: kinetic part is not separable over the tensor axes");
    if (u.step != params.epsilon())
        throw InvalidInput("split_step_nd: tensor step does not match params.epsilon()");
    if (!u.periodic) throw InvalidInput("laxol_b200 split_step_nd: periodic tensors only");
    for (std::size_t d : u.dims)
        if (d != static_cast<std::size_t>(params.n_space))
            throw InvalidInput("split_step_nd: periodic axes must hold one unit period");
    const int64_t n = params.n_space;
    const int code = engine_code(engine);
    DevBuf<double> du(n * n), dout(n * n), dtmp(n * n), da1(n), da2(n);
    du.upload(u.values.data(), n * n);
    double b = 0.0;
    const bool hasv = static_cast<bool>(spec.potential.a1);
    if (hasv) {
        const double tt = potential_time(t, params);
        std::vector<double> a1(n), a2(n);
        for (int64_t i = 0; i < n; ++i) {
            a1[i] = spec.potential.a1(u.origins[0] + static_cast<double>(i) * u.step);
            a2[i] = spec.potential.a2(u.origins[1] + static_cast<double>(i) * u.step);
        }
        b = spec.potential.b ? spec.potential.b(tt) : 0.0;
        da1.upload(a1.data(), n);
        da2.upload(a2.data(), n);
    }
    size_t wsb = 0;
    lob_fast_workspace_bytes(n, n, &wsb);
    wsb *= 2;  // one half per axis: the fused four-launch step
    DevBuf<unsigned char> ws(code == LOB_ENGINE_FAST ? wsb : 0);
    check_status(lob_split_step_2d_f64(ctx_, du.p, dout.p, dtmp.p, n, params.tau, spec.drift1, spec.drift2,
                                       hasv ? da1.p : nullptr, hasv ? da2.p : nullptr, b, code, ws.p, wsb,
                                       nullptr),
                 ctx_, "split_step_nd");
    check_cuda(cudaDeviceSynchronize(), "split_step_nd");
    TensorFn out = u;
    dout.download(out.values.data(), n * n);
    return out;
}

// ---- weak-KAM consumers (proj/src/weakkam.cpp) ------------------------------

namespace {

// proj/src/weakkam.cpp:17-31
int64_t steps_per_period(const SchemeParams& params, const char* who) {
    const int64_t ell = std::llround(1.0 / params.tau);
    if (ell < 1 || std::abs(static_cast<double>(ell) * params.tau - 1.0) > 1e-9)
        throw InvalidInput(std::string(who) + ": tau must be a unit fraction of the time period");
    return ell;
}

void require_time_periodic(const Potential& V, const char* who) {
    if (V && V.time_dependent && !V.time_periodic)
        throw InvalidInput(std::string(who) + ": spec must be time-periodic with period 1");
}

// tau*V tables of one period's steps (in-period time labels i*tau,
// proj/src/weakkam.cpp:33-39): none, one (autonomous) or ell
std::vector<double> period_tables(const GridFn& u, const Potential& V, const SchemeParams& params, int64_t ell,
                                  int64_t* count) {
    const std::size_t n = u.n();
    if (!V) {
        *count = 0;
        return {};
    }
    const int64_t nt = V.time_dependent ? ell : 1;
    std::vector<double> tabs;
    tabs.reserve(static_cast<size_t>(nt) * n);
    for (int64_t i = 0; i < nt; ++i) {
        const std::vector<double> tv =
            tabulate_tv(u, V, potential_time(static_cast<double>(i) * params.tau, params), params.tau, n);
        tabs.insert(tabs.end(), tv.begin(), tv.end());
    }
    *count = nt;
    return tabs;
}

void check_matrix(const MinPlusMatrix& m, const char* who) {
    if (m.cost.size() != m.n * m.n) throw InvalidInput(std::string(who) + ": cost is not n x n");
}

}  // namespace

EffectiveHEstimate Engine::estimate_hbar_drift(const GridFn& u0, double drift, const Potential& V,
                                               const SchemeParams& params, int max_periods, double tol,
                                               ConvEngine engine) {
    require_time_periodic(V, "estimate_hbar_drift");
    if (!u0.periodic) throw InvalidInput("estimate_hbar_drift: spec must be space-periodic");
    const int64_t ell = steps_per_period(params, "estimate_hbar_drift");
    if (max_periods < 1) throw InvalidInput("estimate_hbar_drift: max_periods must be >= 1");
    check_u_grid(u0, params, "estimate_hbar_drift");
    int64_t nt = 0;
    const std::vector<double> tabs = period_tables(u0, V, params, ell, &nt);
    EffectiveHEstimate est;
    int conv = 0;
    check_status(lob_hbar_drift_host_f64(ctx_, u0.values.data(), static_cast<int64_t>(u0.n()), drift, params.tau,
                                         nt ? tabs.data() : nullptr, nt, engine_code(engine), max_periods, tol,
                                         &est.h_bar, &est.residual, &est.n_steps, &conv, nullptr),
                 ctx_, "estimate_hbar_drift");
    est.converged = conv != 0;
    return est;
}

double Engine::fixed_point_residual(const GridFn& u, double h_bar, double drift, const Potential& V,
                                    const SchemeParams& params, ConvEngine engine) {
    require_time_periodic(V, "fixed_point_residual");
    if (!u.periodic) throw InvalidInput("fixed_point_residual: spec must be space-periodic");
    steps_per_period(params, "fixed_point_residual");
    check_u_grid(u, params, "fixed_point_residual");
    int64_t nt = 0;
    const std::vector<double> tabs = period_tables(u, V, params, steps_per_period(params, "fixed_point_residual"), &nt);
    double r = 0.0;
    check_status(lob_fixed_point_residual_host_f64(ctx_, u.values.data(), static_cast<int64_t>(u.n()), h_bar, drift,
                                                   params.tau, nt ? tabs.data() : nullptr, nt, engine_code(engine),
                                                   &r),
                 ctx_, "fixed_point_residual");
    return r;
}

MinPlusMatrix Engine::build_period_matrix(double drift, const Potential& V, const SchemeParams& params) {
    require_time_periodic(V, "build_period_matrix");
    const int64_t ell = steps_per_period(params, "build_period_matrix");
    const int64_t n = params.n_space;
    if (n > 512) throw InvalidInput("build_period_matrix: n_space exceeds the dense guard (512)");
    const KernelWindow k = build_kernel_mech(n, params.tau, drift);
    std::vector<double> kinc(static_cast<size_t>(n));
    lob_period_kinetic_host(k.window.data(), k.first, n, kinc.data());
    // tau*V(t_i', x*eps) per step (proj/src/weakkam.cpp:103-104,120-121)
    const double eps = params.epsilon();
    std::vector<double> tvs;
    if (V) {
        tvs.resize(static_cast<size_t>(ell * n));
        for (int64_t i = 0; i < ell; ++i) {
            const double tt = potential_time(static_cast<double>(i) * params.tau, params);
            for (int64_t x = 0; x < n; ++x) {
                const double vx = V(tt, static_cast<double>(x) * eps);
                tvs[static_cast<size_t>(i * n + x)] = params.tau * vx;
            }
        }
    }
    DevBuf<double> dk(n), dtv(tvs.size()), dc(n * n), dscr(2 * n * n);
    dk.upload(kinc.data(), n);
    if (!tvs.empty()) dtv.upload(tvs.data(), tvs.size());
    check_status(lob_period_matrix_f64(ctx_, dk.p, tvs.empty() ? nullptr : dtv.p, n, ell, dc.p, dscr.p, nullptr),
                 ctx_, "build_period_matrix");
    MinPlusMatrix C;
    C.n = static_cast<size_t>(n);
    C.cost.resize(static_cast<size_t>(n * n));
    dc.download(C.cost.data(), C.cost.size());
    return C;
}

MinPlusMatrix Engine::minplus_product(const MinPlusMatrix& A, const MinPlusMatrix& B) {
    check_matrix(A, "minplus_product");
    check_matrix(B, "minplus_product");
    if (A.n != B.n) throw InvalidInput("minplus_product: size mismatch");
    const int64_t n = static_cast<int64_t>(A.n);
    MinPlusMatrix C;
    C.n = A.n;
    C.cost.resize(A.cost.size());
    if (n == 0) return C;
    DevBuf<double> da(n * n), db(n * n), dc(n * n);
    da.upload(A.cost.data(), n * n);
    db.upload(B.cost.data(), n * n);
    check_status(lob_minplus_gemm_f64(ctx_, da.p, n, db.p, n, dc.p, n, n, n, n, nullptr), ctx_, "minplus_product");
    dc.download(C.cost.data(), n * n);
    return C;
}

GridFn Engine::minplus_apply(const MinPlusMatrix& C, const GridFn& u) {
    check_matrix(C, "minplus_apply");
    if (!u.periodic || u.n() != C.n)
        throw InvalidInput("minplus_apply: u must be periodic over the quotient grid");
    const int64_t n = static_cast<int64_t>(C.n);
    DevBuf<double> du(n), dc(n * n), dout(n);
    du.upload(u.values.data(), n);
    dc.upload(C.cost.data(), n * n);
    check_status(lob_minplus_gemm_f64(ctx_, du.p, n, dc.p, n, dout.p, n, 1, n, n, nullptr), ctx_, "minplus_apply");
    std::vector<double> out(static_cast<size_t>(n));
    dout.download(out.data(), n);
    return make_periodic(std::move(out), u.step, u.origin);
}

double Engine::eigenvalue_karp(const MinPlusMatrix& C) {
    check_matrix(C, "eigenvalue_karp");
    if (C.n == 0) throw InvalidInput("eigenvalue_karp: empty matrix");
    const int64_t n = static_cast<int64_t>(C.n);
    DevBuf<double> dc(n * n);
    dc.upload(C.cost.data(), n * n);
    double lam = 0.0;
    check_status(lob_eigenvalue_karp_f64(ctx_, dc.p, n, &lam, nullptr), ctx_, "eigenvalue_karp");
    return lam;
}

// ---- built-in potentials and step_semidiscrete --------------------------------

double BuiltinPotential::operator()(double t, double x) const {
    // proj/src/hamiltonian.cpp:18-21,98-117
    switch (kind) {
        case Kind::Zero:
            return 0.0;
        case Kind::Const:
            return value;
        case Kind::Cosine: {
            double mod = 1.0;
            if (tmod == TimeMod::Sin) mod = std::sin(omega * t);
            else if (tmod == TimeMod::Cos) mod = std::cos(omega * t);
            const double r = x - std::floor(x);
            const double th = (2.0 * 3.141592653589793) * r - 3.141592653589793;
            return offset + amplitude * mod * std::cos(static_cast<double>(frequency) * th);
        }
    }
    return 0.0;
}

Potential BuiltinPotential::callback() const {
    if (kind == Kind::Zero) return Potential{};
    const BuiltinPotential self = *this;
    Potential p;
    p.fn = [self](double t, double x) { return self(t, x); };
    p.time_dependent = kind == Kind::Cosine && tmod != TimeMod::None && amplitude != 0.0;
    return p;
}

BuiltinPotential potential_zero() { return BuiltinPotential{}; }

BuiltinPotential potential_const(double c) {
    BuiltinPotential p;
    p.kind = BuiltinPotential::Kind::Const;
    p.value = c;
    return p;
}

BuiltinPotential potential_cosine(double offset, double amplitude, int frequency, BuiltinPotential::TimeMod tmod,
                                  double omega) {
    if (frequency < 1) throw InvalidInput("potential_cosine: frequency must be >= 1");
    BuiltinPotential p;
    p.kind = BuiltinPotential::Kind::Cosine;
    p.offset = offset;
    p.amplitude = amplitude;
    p.frequency = frequency;
    p.tmod = tmod;
    p.omega = omega;
    return p;
}

GridFn Engine::step_semidiscrete(const GridFn& u, double t, double drift, const BuiltinPotential& V,
                                 const SchemeParams& params, int quad_points) {
    if (quad_points < 1) throw InvalidInput("step_semidiscrete: quad_points must be >= 1");
    check_u_grid(u, params, "step_semidiscrete");
    const KernelWindow k = build_kernel_mech(params, drift);
    lob_potential lp{};
    lp.kind = static_cast<int>(V.kind);
    lp.value = V.value;
    lp.offset = V.offset;
    lp.amplitude = V.amplitude;
    lp.frequency = V.frequency;
    lp.tmod = static_cast<int>(V.tmod);
    lp.omega = V.omega;
    const int64_t m = u.periodic ? static_cast<int64_t>(u.n()) : static_cast<int64_t>(u.size());
    DevBuf<double> du(m), dout(m), dk(k.window.size());
    du.upload(u.values.data(), m);
    dk.upload(k.window.data(), k.window.size());
    check_status(lob_step_semidiscrete_f64(ctx_, du.p, dout.p, 1, m, params.n_space, u.periodic ? 1 : 0, u.origin,
                                           dk.p, k.first, t, params.tau, &lp, quad_points, nullptr),
                 ctx_, "step_semidiscrete");
    std::vector<double> out(u.size());
    dout.download(out.data(), m);
    if (u.periodic) out[m] = out[0];  // sample_coord wraps the seam index (proj/src/scheme.cpp:32-35)
    return GridFn{std::move(out), u.step, u.origin, u.periodic};
}

// ---- split_step_nd for any rank -------------------------------------------------

TensorFn Engine::split_step_nd(const TensorFn& u, double t, const SplitSpecND& spec, const SchemeParams& params,
                               ConvEngine engine) {
    // proj/src/splitting.cpp:37-49 validation
    const std::size_t rank = u.dims.size();
    if (spec.kernels.size() != rank)
        throw InvalidInput("split_step_nd: kinetic part is not separable over the tensor axes");
    if (u.step != params.epsilon()) throw InvalidInput("split_step_nd: tensor step does not match params.epsilon()");
    if (u.periodic)
        for (std::size_t d : u.dims)
            if (d != static_cast<std::size_t>(params.n_space))
                throw InvalidInput("split_step_nd: periodic axes must hold one unit period");
    if (u.origins.size() != rank) throw InvalidInput("split_step_nd: one origin per axis");
    const int64_t n = params.n_space, W = 2 * n + 1;
    std::size_t total = u.values.size();
    bool mech = true;
    for (const KernelWindow& k : spec.kernels) {
        if (k.n_space != n || static_cast<int64_t>(k.window.size()) != W)
            throw InvalidInput("split_step_nd: kernel window does not match n_space");
        mech = mech && k.mechanical;
    }
    int code;
    if (engine == ConvEngine::GpuDirect) code = LOB_ENGINE_DIRECT;
    else if (engine == ConvEngine::GpuFast) code = (params.eta > 0.0 || !mech) ? LOB_ENGINE_RELAXED : LOB_ENGINE_FAST;
    else code = engine_code(engine);
    std::vector<double> kt(static_cast<size_t>(rank * W));
    std::vector<int64_t> firsts(rank);
    std::vector<double> drifts(rank);
    for (std::size_t a = 0; a < rank; ++a) {
        std::copy(spec.kernels[a].window.begin(), spec.kernels[a].window.end(), kt.begin() + a * W);
        firsts[a] = spec.kernels[a].first;
        drifts[a] = spec.kernels[a].drift;
    }
    // tau*V per point in the reference's coordinates (proj/src/splitting.cpp:85-97)
    std::vector<double> tv;
    if (spec.potential) {
        tv.resize(total);
        const double tt = potential_time(t, params);
        std::vector<std::size_t> strides(rank, 1);
        for (std::size_t a = rank; a-- > 1;) strides[a - 1] = strides[a] * u.dims[a];
        std::vector<double> coords(rank);
        for (std::size_t flat = 0; flat < total; ++flat) {
            std::size_t rem = flat;
            for (std::size_t a = 0; a < rank; ++a) {
                const std::size_t idx = rem / strides[a];
                rem %= strides[a];
                coords[a] = u.origins[a] + static_cast<double>(idx) * u.step;
            }
            const double v = spec.potential(tt, coords);
            if (!std::isfinite(v)) throw EvaluationError("split_step_nd: potential sample is not finite");
            tv[flat] = params.tau * v;
        }
    }
    DevBuf<double> du(total), dout(total), dtmp(total), dk(kt.size()), dtv(tv.size());
    du.upload(u.values.data(), total);
    dk.upload(kt.data(), kt.size());
    if (!tv.empty()) dtv.upload(tv.data(), tv.size());
    if (!u.periodic) {  // walls: the exact windowed sweeps
        std::vector<int64_t> dims(u.dims.begin(), u.dims.end());
        check_status(lob_split_step_nd_window_f64(ctx_, du.p, dout.p, dtmp.p, static_cast<int>(rank), dims.data(), n,
                                                  params.tau, dk.p, firsts.data(), tv.empty() ? nullptr : dtv.p,
                                                  nullptr),
                     ctx_, "split_step_nd");
        TensorFn out = u;
        dout.download(out.values.data(), total);
        return out;
    }
    size_t wsb = 0;
    lob_fast_workspace_bytes(static_cast<int64_t>(total / n), n, &wsb);
    DevBuf<unsigned char> ws(code == LOB_ENGINE_FAST ? wsb : 0);
    check_status(lob_split_step_nd_f64(ctx_, du.p, dout.p, dtmp.p, static_cast<int>(rank), n, params.tau, dk.p,
                                       firsts.data(), drifts.data(), tv.empty() ? nullptr : dtv.p, params.eta, code,
                                       ws.p, wsb, nullptr),
                 ctx_, "split_step_nd");
    TensorFn out = u;
    dout.download(out.values.data(), total);
    return out;
}

}  // namespace laxol_b200

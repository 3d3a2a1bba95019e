// C-ABI entry points of laxol_b200 (declared in include/laxol_b200.h).
// Validation mirrors the reference's InvalidInput checks
// (proj/src/scheme.cpp:18-24,39-53; proj/src/grid_fn.cpp:11-22).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lob_internal.cuh"

using namespace lob;

namespace {

const char* kVersion = "laxol_b200 0.1 (sm_100a)";

int check_lines(lob_ctx* ctx, int64_t lines, int64_t n, const char* who) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (lines < 0) return set_error(ctx, LOB_INVALID_INPUT, std::string(who) + ": lines < 0");
    if (n < 1)
        return set_error(ctx, LOB_INVALID_INPUT,
                         std::string(who) + ": periodic function needs n >= 1");
    return LOB_OK;
}

// validate(SchemeParams) of the reference (proj/src/scheme.cpp:39-53) with its defaults h0 = 1,
// AntiCflMode::Fail: the same conditions, the same messages' leading text
int check_scheme(lob_ctx* ctx, int64_t n, double tau, double eta) {
    if (!(tau > 0.0)) return set_error(ctx, LOB_INVALID_INPUT, "SchemeParams: tau must be positive");
    if (eta < 0.0) return set_error(ctx, LOB_INVALID_INPUT, "SchemeParams: eta must be >= 0");
    if ((1.0 / static_cast<double>(n)) / tau >= 1.0)
        return set_error(ctx, LOB_INVALID_INPUT, "SchemeParams: epsilon/tau violates epsilon/tau < h0");
    return LOB_OK;
}

}  // namespace

extern "C" {

const char* lob_version(void) { return kVersion; }

int lob_ctx_create(int device, lob_ctx** out) {
    if (!out) return LOB_INVALID_INPUT;
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) return LOB_CUDA_ERROR;  // no CPU fallback
    if (device < 0 || device >= count) return LOB_INVALID_INPUT;
    auto* ctx = new lob_ctx();
    ctx->device = device;
    if (cudaSetDevice(device) != cudaSuccess) {
        delete ctx;
        return LOB_CUDA_ERROR;
    }
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    // stream-ordered scratch (cudaMallocAsync) stays cached in the device's default pool
    // instead of being returned to the driver at every synchronisation
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return LOB_CUDA_ERROR;
    }
    *out = ctx;
    return LOB_OK;
}

int lob_ctx_destroy(lob_ctx* ctx) {
    if (!ctx) return LOB_OK;
    cudaSetDevice(ctx->device);
    for (auto& kv : ctx->vtabs) cudaFree(kv.second.dev);
    for (auto& kv : ctx->split_axes) cudaFree(kv.second);
    if (ctx->scratch) cudaFree(ctx->scratch);
    if (ctx->direct_full) cudaFree(ctx->direct_full);
    if (ctx->direct_umax) cudaFree(ctx->direct_umax);
    if (ctx->stream) cudaStreamDestroy(ctx->stream);
    for (auto& a : ctx->aux)
        if (a) cudaStreamDestroy(a);
    for (auto& e : ctx->aux_ev)
        if (e) cudaEventDestroy(e);
    delete ctx;
    return LOB_OK;
}

const char* lob_last_error(const lob_ctx* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

int lob_ctx_set_direct_mode(lob_ctx* ctx, int mode) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (mode != LOB_DIRECT_SCREENED && mode != LOB_DIRECT_PLAIN)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_ctx_set_direct_mode: unknown mode");
    ctx->direct_mode = mode;
    return LOB_OK;
}

int lob_ctx_set_fast_delta(lob_ctx* ctx, double delta) {
    if (!ctx) return LOB_INVALID_INPUT;
    ctx->fast_delta_override = delta;
    return LOB_OK;
}

int lob_ctx_set_fast_line(lob_ctx* ctx, int on) {
    if (!ctx) return LOB_INVALID_INPUT;
    ctx->fast_line = on < 0 ? 0 : on;  // 2, 3: split-step layouts measured against the default (1)
    return LOB_OK;
}

int lob_ctx_set_evolve_resident(lob_ctx* ctx, int on) {
    if (!ctx) return LOB_INVALID_INPUT;
    ctx->resident = on ? 1 : 0;
    return LOB_OK;
}

int lob_direct_stats(lob_ctx* ctx, uint64_t* full_outputs, uint64_t* fp64_candidates, int reset) {
    if (!ctx) return LOB_INVALID_INPUT;
    cudaSetDevice(ctx->device);
    unsigned long long v[2] = {0, 0};
    if (ctx->direct_full) {
        LOB_CUDA_TRY(ctx, cudaDeviceSynchronize());
        LOB_CUDA_TRY(ctx, cudaMemcpy(v, ctx->direct_full, sizeof(v), cudaMemcpyDeviceToHost));
        if (reset) LOB_CUDA_TRY(ctx, cudaMemset(ctx->direct_full, 0, sizeof(v)));
    }
    if (full_outputs) *full_outputs = v[0];
    if (fp64_candidates) *fp64_candidates = v[1];
    return LOB_OK;
}

int64_t lob_launch_count(const lob_ctx* ctx) { return ctx ? ctx->launches : 0; }

int lob_minplus_direct_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                           const double* ktab, int64_t ktab_stride, const int64_t* first,
                           const double* tv, int64_t tv_stride, void* stream) {
    int st = check_lines(ctx, lines, n, "lob_minplus_direct_f64");
    if (st) return st;
    if (lines == 0) return LOB_OK;
    if (!u || !out || !ktab || !first)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_direct_f64: null buffer");
    if (u == out)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_direct_f64: out must not alias u");
    return launch_direct_f64(ctx, u, out, lines, n, ktab, ktab_stride, first, tv, tv_stride,
                             static_cast<cudaStream_t>(stream));
}

int lob_minplus_direct_f32(lob_ctx* ctx, const float* u, float* out, int64_t lines, int64_t n,
                           const float* ktab, int64_t ktab_stride, const int64_t* first,
                           void* stream) {
    int st = check_lines(ctx, lines, n, "lob_minplus_direct_f32");
    if (st) return st;
    if (lines == 0) return LOB_OK;
    if (!u || !out || !ktab || !first)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_direct_f32: null buffer");
    if (static_cast<const void*>(u) == static_cast<const void*>(out))
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_direct_f32: out must not alias u");
    return launch_direct_f32(ctx, u, out, lines, n, ktab, ktab_stride, first,
                             static_cast<cudaStream_t>(stream));
}

int lob_minplus_window_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t m,
                           int64_t n, const double* ktab, int64_t ktab_stride,
                           const int64_t* first, const double* tv, int64_t tv_stride,
                           void* stream) {
    int st = check_lines(ctx, lines, n, "lob_minplus_window_f64");
    if (st) return st;
    if (m < 1) return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_window_f64: empty sample vector");
    if (lines == 0) return LOB_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int* d_err = nullptr;
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&d_err, sizeof(int), s));
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(d_err, 0, sizeof(int), s));
    st = launch_window_f64(ctx, u, out, lines, m, n, ktab, ktab_stride, first, tv, tv_stride,
                           d_err, s);
    int h_err = 0;
    if (st == LOB_OK) {
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&h_err, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    }
    cudaFreeAsync(d_err, s);
    if (st) return st;
    if (h_err)
        return set_error(ctx, LOB_EVALUATION_ERROR,
                         "kinetic_convolve: kernel window does not reach some grid index");
    return LOB_OK;
}

int lob_fast_workspace_bytes(int64_t lines, int64_t n, size_t* bytes) {
    if (!bytes || lines < 0 || n < 1) return LOB_INVALID_INPUT;
    *bytes = fast_workspace_bytes(lines, n);
    return LOB_OK;
}

int lob_minplus_fast_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                         const double* drift, double tau, const double* tv, int64_t tv_stride,
                         double eta, int64_t* blocks, void* workspace, size_t workspace_bytes,
                         int flags, void* stream) {
    int st = check_lines(ctx, lines, n, "lob_minplus_fast_f64");
    if (st) return st;
    if ((st = check_scheme(ctx, n, tau, eta))) return st;
    if (lines == 0) return LOB_OK;
    if (!u || !out || !drift)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_f64: null buffer");
    if (u == out) return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_f64: out must not alias u");
    if (flags & ~kFastUserFlags) return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_f64: unknown flags");
    return launch_fast_f64(ctx, u, out, lines, n, drift, tau, tv, tv_stride, eta, blocks, workspace,
                           workspace_bytes, flags, static_cast<cudaStream_t>(stream));
}

int lob_minplus_fast_window_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                                const double* ktab, int64_t ktab_stride, const int64_t* first, double tau,
                                const double* tv, int64_t tv_stride, double eta, int64_t* blocks, void* workspace,
                                size_t workspace_bytes, int flags, void* stream) {
    int st = check_lines(ctx, lines, n, "lob_minplus_fast_window_f64");
    if (st) return st;
    if (lines == 0) return LOB_OK;
    if (!u || !out || !ktab || !first)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_window_f64: null buffer");
    if (u == out) return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_window_f64: out must not alias u");
    if (!(tau > 0.0)) return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_window_f64: tau must be positive");
    if (ktab_stride != 0 && ktab_stride < 2 * n + 1)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_window_f64: ktab_stride < 2n+1");
    if (flags & ~kFastUserFlags) return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_window_f64: unknown flags");
    const FastTable tab{ktab, ktab_stride, first};
    return launch_fast_f64(ctx, u, out, lines, n, nullptr, tau, tv, tv_stride, eta, blocks, workspace,
                           workspace_bytes, flags, static_cast<cudaStream_t>(stream), nullptr, &tab);
}

int lob_fast_diagnostics(lob_ctx* ctx, void* workspace, int64_t lines, int64_t n,
                         uint64_t* counters) {
    if (!ctx || !workspace || !counters) return LOB_INVALID_INPUT;
    cudaDeviceSynchronize();
    return fast_diag_count(ctx, workspace, lines, n, counters, ctx->stream);
}

int lob_block_counts(lob_ctx* ctx, const double* u, int64_t lines, int64_t n, double eta,
                     int64_t* blocks, void* stream) {
    int st = check_lines(ctx, lines, n, "lob_block_counts");
    if (st) return st;
    if (lines == 0) return LOB_OK;
    return launch_block_counts(ctx, u, lines, n, eta, blocks, static_cast<cudaStream_t>(stream));
}

// Per-axis device inputs of a mechanical split step, built once per (n, tau, drift) and kept
// by the context (never rewritten: no reuse race with work still queued on any stream):
// the kernel window (K1), n copies of first (K1) and of the drift (K2).
static int split_axis_inputs(lob_ctx* ctx, int64_t n, double tau, double drift, const double** ktab,
                             const int64_t** firsts, const double** drifts, cudaStream_t s) {
    uint64_t tb, db;
    std::memcpy(&tb, &tau, 8);
    std::memcpy(&db, &drift, 8);
    const auto key = std::make_tuple(n, tb, db);
    auto it = ctx->split_axes.find(key);
    if (it == ctx->split_axes.end()) {
        const size_t W = static_cast<size_t>(2 * n + 1);
        std::vector<double> h(W);
        int64_t f, arg;
        double dl;
        if (lob_kernel_mech_host(ctx, n, tau, drift, h.data(), &f, &arg, &dl))
            return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd: invalid kernel parameters");
        std::vector<int64_t> hf(static_cast<size_t>(n), f);
        std::vector<double> hd(static_cast<size_t>(n), drift);
        char* buf = nullptr;
        const size_t bytes = W * 8 + static_cast<size_t>(n) * 16;
        LOB_CUDA_TRY(ctx, cudaMalloc(&buf, bytes));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(buf, h.data(), W * 8, cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(buf + W * 8, hf.data(), n * 8, cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(buf + W * 8 + n * 8, hd.data(), n * 8, cudaMemcpyHostToDevice, s));
        // the host vectors die here: complete the (one-time) upload
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        it = ctx->split_axes.emplace(key, buf).first;
    }
    char* buf = static_cast<char*>(it->second);
    const size_t W = static_cast<size_t>(2 * n + 1);
    *ktab = reinterpret_cast<const double*>(buf);
    *firsts = reinterpret_cast<const int64_t*>(buf + W * 8);
    *drifts = reinterpret_cast<const double*>(buf + W * 8 + n * 8);
    return LOB_OK;
}

int lob_split_step_2d_f64(lob_ctx* ctx, const double* u, double* out, double* tmp, int64_t n,
                          double tau, double drift1, double drift2, const double* a1,
                          const double* a2, double b, int engine, void* workspace,
                          size_t workspace_bytes, void* stream) {
    int st = check_lines(ctx, n, n, "lob_split_step_2d_f64");
    if (st) return st;
    if (!u || !out || !tmp || u == out || u == tmp || out == tmp)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_split_step_2d_f64: need distinct u/out/tmp");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const double *k1, *k2, *d1, *d2;
    const int64_t *f1, *f2;
    if ((st = split_axis_inputs(ctx, n, tau, drift1, &k1, &f1, &d1, s))) return st;
    if ((st = split_axis_inputs(ctx, n, tau, drift2, &k2, &f2, &d2, s))) return st;
    const size_t wsz = fast_workspace_bytes(n, n);
    if (engine == LOB_ENGINE_FAST && ctx->fast_line && n <= fast_line_max()) {
        // K2L twice, tau*V = tau*(a1[i]*a2[k] + b) in the second sweep's epilogue
        const FastSepPot sep{a1, a2, b};
        const FastSepPot* sp = (a1 && a2) ? &sep : nullptr;
        int mode = ctx->fast_line;
        if (mode == 5 && (n % 2 != 0 || reinterpret_cast<uintptr_t>(u) % 16 != 0 ||
                          reinterpret_cast<uintptr_t>(tmp) % 16 != 0))
            mode = 2;
        if (mode == 4 && n % 8 != 0) mode = 2;
        if (mode == 5) {
            // both sweeps read columns by 2-D TMA and write rows: tmp holds the transposed state
            // after axis 0, whose columns are the rows of axis 1
            if ((st = launch_line_f64(ctx, u, tmp, n, n, d1, tau, nullptr, 0, nullptr, kLineTma, kLineRow, nullptr, s)))
                return st;
            return launch_line_f64(ctx, tmp, out, n, n, d2, tau, nullptr, 0, sp, kLineTma, kLineRow, nullptr, s);
        }
        if (mode == 2) {  // transposes around row sweeps
            if ((st = launch_transpose(ctx, u, tmp, n, s))) return st;
            if ((st = launch_line_f64(ctx, tmp, out, n, n, d1, tau, nullptr, 0, nullptr, kLineRow, kLineRow, nullptr, s)))
                return st;
            if ((st = launch_transpose(ctx, out, tmp, n, s))) return st;
            return launch_line_f64(ctx, tmp, out, n, n, d2, tau, nullptr, 0, sp, kLineRow, kLineRow, nullptr, s);
        }
        if (mode == 3) {  // both sweeps read columns (strided) and write rows
            if ((st = launch_line_f64(ctx, u, tmp, n, n, d1, tau, nullptr, 0, nullptr, kLineCol, kLineRow, nullptr, s)))
                return st;
            return launch_line_f64(ctx, tmp, out, n, n, d2, tau, nullptr, 0, sp, kLineCol, kLineRow, nullptr, s);
        }
        // axis 0 on columns in place (1: strided; 4: exchanged through DSMEM in clusters of 8 CTAs
        // = 8 adjacent columns, 64-byte row segments), axis 1 on rows
        const int cl = mode == 4 ? kLineClu : kLineCol;
        if ((st = launch_line_f64(ctx, u, tmp, n, n, d1, tau, nullptr, 0, nullptr, cl, cl, nullptr, s))) return st;
        return launch_line_f64(ctx, tmp, out, n, n, d2, tau, nullptr, 0, sp, kLineRow, kLineRow, nullptr, s);
    }
    if (engine == LOB_ENGINE_FAST && workspace && workspace_bytes >= 2 * wsz) {
        // fused: transpose + K2 statistics -> sweep axis 0 -> transpose + statistics ->
        // sweep axis 1 with tau*V = tau*(a1[i]*a2[k] + b) in its epilogue.  One workspace per
        // axis keeps each axis' line constants across steps.
        void* wa = workspace;
        void* wb = static_cast<char*>(workspace) + wsz;
        if ((st = launch_transpose_stats(ctx, u, tmp, n, wa, s))) return st;
        if ((st = launch_fast_f64(ctx, tmp, out, n, n, d1, tau, nullptr, 0, 0.0, nullptr, wa, wsz, kFastStatsGiven,
                                  s)))
            return st;
        if ((st = launch_transpose_stats(ctx, out, tmp, n, wb, s))) return st;
        const FastSepPot sep{a1, a2, b};
        return launch_fast_f64(ctx, tmp, out, n, n, d2, tau, nullptr, 0, 0.0, nullptr, wb, wsz, kFastStatsGiven, s,
                               nullptr, nullptr, (a1 && a2) ? &sep : nullptr);
    }
    // axis 0: columns of u are rows of u^T
    if ((st = launch_transpose(ctx, u, tmp, n, s))) return st;
    if (engine == LOB_ENGINE_FAST) {
        if ((st = launch_fast_f64(ctx, tmp, out, n, n, d1, tau, nullptr, 0, 0.0, nullptr, workspace,
                                  workspace_bytes, 0, s)))
            return st;
    } else {
        if ((st = launch_direct_f64(ctx, tmp, out, n, n, k1, 0, f1, nullptr, 0, s))) return st;
    }
    if ((st = launch_transpose(ctx, out, tmp, n, s))) return st;
    // axis 1: contiguous rows
    if (engine == LOB_ENGINE_FAST) {
        if ((st = launch_fast_f64(ctx, tmp, out, n, n, d2, tau, nullptr, 0, 0.0, nullptr, workspace,
                                  workspace_bytes, 0, s)))
            return st;
    } else {
        if ((st = launch_direct_f64(ctx, tmp, out, n, n, k2, 0, f2, nullptr, 0, s))) return st;
    }
    if (a1 && a2) return launch_potential2d(ctx, out, a1, a2, b, tau, n, s);
    return LOB_OK;
}

int lob_slab_pack_f64(lob_ctx* ctx, const double* x, int64_t b, int64_t world, double* send, void* stream) {
    if (!ctx || !x || !send || b < 1 || world < 1 || x == send)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_slab_pack_f64: invalid arguments");
    // send[q][c][i] = x[i][q*b + c]: the b x n slab transposed (= world blocks of b x b)
    return launch_transpose_batched(ctx, x, send, 1, b, b * world, static_cast<cudaStream_t>(stream));
}

int lob_slab_push_f64(lob_ctx* ctx, const double* x, int64_t b, int64_t world, int rank, const uint64_t* peer_slabs,
                      void* stream) {
    if (!ctx || !x || !peer_slabs) return set_error(ctx, LOB_INVALID_INPUT, "lob_slab_push_f64: invalid arguments");
    double* ps[16] = {};
    if (world < 1 || world > 16) return set_error(ctx, LOB_INVALID_INPUT, "lob_slab_push_f64: 1 <= world <= 16");
    for (int64_t q = 0; q < world; ++q) ps[q] = reinterpret_cast<double*>(static_cast<uintptr_t>(peer_slabs[q]));
    return launch_slab_push(ctx, x, b, world, rank, ps, static_cast<cudaStream_t>(stream));
}

int lob_slab_unpack_f64(lob_ctx* ctx, const double* recv, int64_t b, int64_t world, double* y, void* stream) {
    if (!ctx || !recv || !y || b < 1 || world < 1 || recv == y)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_slab_unpack_f64: invalid arguments");
    return launch_slab_unpack(ctx, recv, y, b, world, static_cast<cudaStream_t>(stream));
}

int lob_evolve_f64(lob_ctx* ctx, double* u, double* scratch, int64_t lines, int64_t n,
                   const double* drift, double tau, const double* tv, int64_t tv_stride,
                   double eta, int engine, int64_t steps, double* step_drift,
                   int64_t* step_blocks, int64_t* completed_steps, void* workspace,
                   size_t workspace_bytes, void* stream) {
    int st = check_lines(ctx, lines, n, "lob_evolve_f64");
    if (st) return st;
    if (steps < 0) return set_error(ctx, LOB_INVALID_INPUT, "evolve: steps must be >= 0");
    if (completed_steps) *completed_steps = 0;
    if ((st = check_scheme(ctx, n, tau, eta))) return st;  // evolve validates before stepping (scheme.cpp:211)
    if (lines == 0 || steps == 0) return LOB_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // direct engine needs the per-line kernel tables: built on the host
    // (proj/src/scheme.cpp:213 builds the kernel once per evolve)
    std::vector<double> hdrift(static_cast<size_t>(lines));
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(hdrift.data(), drift, lines * sizeof(double),
                                      cudaMemcpyDeviceToHost, s));
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    double* ktab = nullptr;
    int64_t* firsts = nullptr;
    int* halt = nullptr;
    void* rws = nullptr;
    size_t rwsb = 0;
    const int64_t W = 2 * n + 1;
    if (engine != LOB_ENGINE_DIRECT && engine != LOB_ENGINE_FAST && engine != LOB_ENGINE_RELAXED)
        return set_error(ctx, LOB_INVALID_INPUT, "evolve: unknown engine");
    if (engine == LOB_ENGINE_RELAXED) {
        rwsb = relaxed_workspace_bytes(lines, n);
        LOB_CUDA_TRY(ctx, cudaMallocAsync(&rws, rwsb, s));
    }
    if (engine != LOB_ENGINE_FAST) {
        LOB_CUDA_TRY(ctx, cudaMallocAsync(&ktab, lines * W * sizeof(double), s));
        LOB_CUDA_TRY(ctx, cudaMallocAsync(&firsts, lines * sizeof(int64_t), s));
        std::vector<double> hk(static_cast<size_t>(lines * W));
        std::vector<int64_t> hf(static_cast<size_t>(lines));
        for (int64_t l = 0; l < lines; ++l) {
            int64_t arg;
            double dl;
            if (lob_kernel_mech_host(ctx, n, tau, hdrift[l], hk.data() + l * W, &hf[l], &arg, &dl))
                return set_error(ctx, LOB_INVALID_INPUT, "evolve: invalid scheme parameters");
        }
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(ktab, hk.data(), hk.size() * sizeof(double),
                                          cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(firsts, hf.data(), hf.size() * sizeof(int64_t),
                                          cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    }
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&halt, sizeof(int), s));
    const int big = 0x7fffffff;
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(halt, &big, sizeof(int), cudaMemcpyHostToDevice, s));
    // short lines in batches too small to fill the GPU with step-by-step launches (which are then
    // latency bound): every step in one launch, the lines resident in shared memory (K2R)
    if (engine == LOB_ENGINE_FAST && ctx->resident && fast_resident_ok(n) &&
        lines * fast_tiles(n) <= 4 * static_cast<int64_t>(ctx->sm_count)) {
        void* lcb = nullptr;
        LOB_CUDA_TRY(ctx, cudaMallocAsync(&lcb, static_cast<size_t>(lines) * 64, s));
        st = launch_fast_resident_f64(ctx, u, lines, n, drift, tau, tv, tv_stride, eta, steps, step_drift,
                                      step_blocks, halt, lcb, s);
        int hstep = big;
        if (st == LOB_OK)
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hstep, halt, sizeof(int), cudaMemcpyDeviceToHost, s));
        cudaFreeAsync(lcb, s);
        cudaFreeAsync(halt, s);
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        if (st) return st;
        if (completed_steps) *completed_steps = hstep != big ? hstep + 1 : steps;
        if (hstep != big)
            return set_error(ctx, LOB_EVALUATION_ERROR, "non-finite value after step " + std::to_string(hstep + 1));
        return LOB_OK;
    }
    double* dpart = nullptr;
    unsigned* dcount = nullptr;
    // the fast engine on lines of more than one tile: each step's drift reduced inside its launch,
    // so consecutive steps chain (a tile waits only for its own line's previous step)
    const bool chained = engine == LOB_ENGINE_FAST && n > fast_line_max();
    if (engine == LOB_ENGINE_FAST)
        LOB_CUDA_TRY(ctx, cudaMallocAsync(&dpart, static_cast<size_t>(lines * fast_tiles(n)) * sizeof(double), s));
    if (chained) {
        LOB_CUDA_TRY(ctx, cudaMallocAsync(&dcount, static_cast<size_t>(lines) * sizeof(unsigned), s));
        LOB_CUDA_TRY(ctx, cudaMemsetAsync(dcount, 0, static_cast<size_t>(lines) * sizeof(unsigned), s));
    }
    double* cur = u;
    double* nxt = scratch;
    int64_t done = 0;
    int hstep = big;
    const int64_t chunk = 64;
    for (int64_t i = 0; i < steps; ++i) {
        if (engine == LOB_ENGINE_DIRECT) {
            st = launch_direct_f64(ctx, cur, nxt, lines, n, ktab, W, firsts, tv, tv_stride, s);
            if (st == LOB_OK && step_blocks)
                st = launch_block_counts(ctx, cur, lines, n, eta, step_blocks + i * lines, s);
        } else if (engine == LOB_ENGINE_RELAXED) {
            st = launch_relaxed_f64(ctx, cur, nxt, lines, n, ktab, W, firsts, tv, tv_stride, eta,
                                    step_blocks ? step_blocks + i * lines : nullptr, rws, rwsb, s);
        } else {
            // the drift's per-tile partial sums come out of the K2 epilogue (no second pass over u)
            if (chained) {
                const FastDriftOut dout{step_drift ? step_drift + i * lines : nullptr, halt, dcount, static_cast<int>(i)};
                st = launch_fast_f64(ctx, cur, nxt, lines, n, drift, tau, tv, tv_stride, eta,
                                     step_blocks ? step_blocks + i * lines : nullptr, workspace, workspace_bytes,
                                     LOB_FAST_CHAINED | (i == 0 ? 0 : LOB_FAST_STATS_VALID), s, dpart, nullptr,
                                     nullptr, &dout);
            } else {
                st = launch_fast_f64(ctx, cur, nxt, lines, n, drift, tau, tv, tv_stride, eta,
                                     step_blocks ? step_blocks + i * lines : nullptr, workspace,
                                     workspace_bytes, i == 0 ? 0 : LOB_FAST_STATS_VALID, s, dpart);
                if (st == LOB_OK)
                    st = launch_drift_tiles(ctx, dpart, lines, n, step_drift ? step_drift + i * lines : nullptr,
                                            halt, static_cast<int>(i), s);
            }
        }
        if (st) break;
        if (engine != LOB_ENGINE_FAST)
            st = launch_drift(ctx, nxt, cur, lines, n, step_drift ? step_drift + i * lines : nullptr,
                              halt, static_cast<int>(i), s);
        if (st) break;
        std::swap(cur, nxt);
        done = i + 1;
        if ((i + 1) % chunk == 0 || i + 1 == steps) {
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hstep, halt, sizeof(int), cudaMemcpyDeviceToHost, s));
            LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
            if (hstep != big) break;
        }
    }
    if (st == LOB_OK && hstep != big) {
        // non-finite after step hstep+1 (proj/src/scheme.cpp:257-264): the trace
        // stops there.  Steps after it within the chunk ran on non-finite data;
        // the caller re-runs with steps = hstep+1 to obtain that state.
        done = hstep + 1;
    }
    if (cur != u && st == LOB_OK && hstep == big)
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(u, cur, lines * n * sizeof(double),
                                          cudaMemcpyDeviceToDevice, s));
    if (ktab) cudaFreeAsync(ktab, s);
    if (firsts) cudaFreeAsync(firsts, s);
    if (rws) cudaFreeAsync(rws, s);
    if (dpart) cudaFreeAsync(dpart, s);
    if (dcount) cudaFreeAsync(dcount, s);
    cudaFreeAsync(halt, s);
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (completed_steps) *completed_steps = done;
    if (st) return st;
    if (hstep != big)
        return set_error(ctx, LOB_EVALUATION_ERROR,
                         "non-finite value after step " + std::to_string(hstep + 1));
    return LOB_OK;
}

// line chunks of the pipelined host step (fast engine)
#ifndef LOB_HOST_CHUNKS
#define LOB_HOST_CHUNKS 8
#endif
constexpr int64_t kHostChunks = LOB_HOST_CHUNKS;  // <= 16 (two events per chunk in lob_ctx::aux_ev)

int lob_step_host_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                      const double* drift, double tau, const double* tv, int64_t tv_stride,
                      double eta, int engine, int64_t* blocks) {
    int st = check_lines(ctx, lines, n, "lob_step_host_f64");
    if (st) return st;
    if ((st = check_scheme(ctx, n, tau, eta))) return st;
    if (lines == 0) return LOB_OK;
    cudaStream_t s = ctx->stream;
    const size_t ub = static_cast<size_t>(lines * n) * sizeof(double);
    const size_t tvn = tv ? static_cast<size_t>(tv_stride ? lines * tv_stride : n) : 0;
    size_t wsb = fast_workspace_bytes(lines, n);
    const int64_t per_chunk = (lines + kHostChunks - 1) / kHostChunks;
    const size_t wsb_chunk = fast_workspace_bytes(per_chunk, n);
    const int64_t W = 2 * n + 1;
    if (engine != LOB_ENGINE_DIRECT && engine != LOB_ENGINE_FAST && engine != LOB_ENGINE_RELAXED)
        return set_error(ctx, LOB_INVALID_INPUT, "step: unknown engine");
    const size_t kb = engine != LOB_ENGINE_FAST ? static_cast<size_t>(lines * W) * sizeof(double) : 0;
    const size_t rwsb = engine == LOB_ENGINE_RELAXED ? relaxed_workspace_bytes(lines, n) : 0;
    const size_t need = 2 * ub + tvn * sizeof(double) + lines * (sizeof(double) + 2 * sizeof(int64_t)) +
                        wsb + 2 * wsb_chunk + kb + rwsb + 11 * 256;
    if (ctx->scratch_bytes < need) {
        if (ctx->scratch) cudaFree(ctx->scratch);
        ctx->scratch = nullptr;
        LOB_CUDA_TRY(ctx, cudaMalloc(&ctx->scratch, need));
        ctx->scratch_bytes = need;
    }
    // sub-buffers aligned to 256 bytes (the fast workspace holds double2 arrays)
    char* p = static_cast<char*>(ctx->scratch);
    auto take = [&p](size_t bytes) {
        char* r = p;
        p += (bytes + 255) & ~static_cast<size_t>(255);
        return r;
    };
    double* du = reinterpret_cast<double*>(take(ub));
    double* dout = reinterpret_cast<double*>(take(ub));
    double* dtv = reinterpret_cast<double*>(take(tvn * sizeof(double)));
    double* ddrift = reinterpret_cast<double*>(take(lines * sizeof(double)));
    int64_t* dblocks = reinterpret_cast<int64_t*>(take(lines * sizeof(int64_t)));
    int64_t* dfirst = reinterpret_cast<int64_t*>(take(lines * sizeof(int64_t)));
    double* dk = reinterpret_cast<double*>(take(kb));
    void* ws = take(wsb);
    void* ws_chunk[2] = {take(wsb_chunk), take(wsb_chunk)};
    void* rws = take(rwsb);
    const bool piped = engine == LOB_ENGINE_FAST && lines >= 2 * kHostChunks;
    if (!piped) LOB_CUDA_TRY(ctx, cudaMemcpyAsync(du, u, ub, cudaMemcpyHostToDevice, s));
    if (tv) LOB_CUDA_TRY(ctx, cudaMemcpyAsync(dtv, tv, tvn * sizeof(double), cudaMemcpyHostToDevice, s));
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(ddrift, drift, lines * sizeof(double), cudaMemcpyHostToDevice, s));
    if (engine != LOB_ENGINE_FAST) {
        std::vector<double> hk(static_cast<size_t>(lines * W));
        std::vector<int64_t> hf(static_cast<size_t>(lines));
        for (int64_t l = 0; l < lines; ++l) {
            int64_t arg;
            double dl;
            if (lob_kernel_mech_host(ctx, n, tau, drift[l], hk.data() + l * W, &hf[l], &arg, &dl))
                return set_error(ctx, LOB_INVALID_INPUT, "step: invalid scheme parameters");
        }
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(dk, hk.data(), hk.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(dfirst, hf.data(), hf.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        if (engine == LOB_ENGINE_RELAXED) {
            st = launch_relaxed_f64(ctx, du, dout, lines, n, dk, W, dfirst, tv ? dtv : nullptr, tv_stride, eta,
                                    blocks ? dblocks : nullptr, rws, rwsb, s);
        } else {
            st = launch_direct_f64(ctx, du, dout, lines, n, dk, W, dfirst, tv ? dtv : nullptr, tv_stride, s);
            if (st == LOB_OK && blocks) st = launch_block_counts(ctx, du, lines, n, eta, dblocks, s);
        }
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));  // host vectors go out of scope
    } else if (lines >= 2 * kHostChunks) {
        // pipelined over line chunks: uploads, steps and downloads run on three
        // streams linked by per-chunk events, so the host->device and
        // device->host copy engines stay busy concurrently
        if (!ctx->aux[0]) {
            for (auto& a : ctx->aux) LOB_CUDA_TRY(ctx, cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
            for (auto& e : ctx->aux_ev) LOB_CUDA_TRY(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
        cudaStream_t up = ctx->aux[0], cs = ctx->aux[1], dn = ctx->aux[2];
        LOB_CUDA_TRY(ctx, cudaEventRecord(ctx->aux_ev[32], s));  // tv, drift uploaded on s
        LOB_CUDA_TRY(ctx, cudaStreamWaitEvent(cs, ctx->aux_ev[32], 0));
        const int64_t per = (lines + kHostChunks - 1) / kHostChunks;
        for (int64_t l0 = 0, k = 0; l0 < lines; l0 += per, ++k) {
            const int64_t cl = std::min(per, lines - l0);
            const size_t cb = static_cast<size_t>(cl * n) * sizeof(double);
            cudaEvent_t in_ready = ctx->aux_ev[2 * k], done = ctx->aux_ev[2 * k + 1];
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(du + l0 * n, u + l0 * n, cb, cudaMemcpyHostToDevice, up));
            LOB_CUDA_TRY(ctx, cudaEventRecord(in_ready, up));
            LOB_CUDA_TRY(ctx, cudaStreamWaitEvent(cs, in_ready, 0));
            st = launch_fast_f64(ctx, du + l0 * n, dout + l0 * n, cl, n, ddrift + l0, tau,
                                 tv ? dtv + (tv_stride ? l0 * tv_stride : 0) : nullptr, tv_stride, eta,
                                 blocks ? dblocks + l0 : nullptr, ws_chunk[k % 2], wsb_chunk, 0, cs);
            if (st) return st;
            LOB_CUDA_TRY(ctx, cudaEventRecord(done, cs));
            LOB_CUDA_TRY(ctx, cudaStreamWaitEvent(dn, done, 0));
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(out + l0 * n, dout + l0 * n, cb, cudaMemcpyDeviceToHost, dn));
        }
        // block counts last, in one copy: a pageable destination would make a
        // per-chunk copy synchronous and serialise the pipeline
        if (blocks)
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(blocks, dblocks, lines * sizeof(int64_t), cudaMemcpyDeviceToHost, dn));
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(dn));
        return LOB_OK;
    } else {
        st = launch_fast_f64(ctx, du, dout, lines, n, ddrift, tau, tv ? dtv : nullptr, tv_stride, eta,
                             blocks ? dblocks : nullptr, ws, wsb, 0, s);
    }
    if (st) return st;
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(out, dout, ub, cudaMemcpyDeviceToHost, s));
    if (blocks)
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(blocks, dblocks, lines * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    return LOB_OK;
}

int lob_potential2d_rows_f64(lob_ctx* ctx, double* out, int64_t rows, int64_t n, const double* a1,
                             const double* a2, double b, double tau, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (rows < 0 || n < 1 || !a1 || !a2)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_potential2d_rows_f64: bad arguments");
    return launch_potential2d(ctx, out, a1, a2, b, tau, n, static_cast<cudaStream_t>(stream), rows);
}

int lob_split_step_nd_f64(lob_ctx* ctx, const double* u, double* out, double* tmp, int rank, int64_t n, double tau,
                          const double* ktabs, const int64_t* firsts, const double* drifts, const double* tv,
                          double eta, int engine, void* workspace, size_t workspace_bytes, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (rank < 1 || rank > 8 || n < 1)
        return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd: rank must be 1..8 and n >= 1");
    if (!u || !out || !tmp || u == out || u == tmp || out == tmp)
        return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd: need distinct u/out/tmp");
    if (engine != LOB_ENGINE_DIRECT && engine != LOB_ENGINE_FAST && engine != LOB_ENGINE_RELAXED)
        return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd: unknown engine");
    if (engine != LOB_ENGINE_FAST && (!ktabs || !firsts))
        return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd: the direct / relaxed engines need the kernel tables");
    if (engine == LOB_ENGINE_FAST && !drifts)
        return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd: the fast engine needs the drifts");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int64_t total = 1;
    for (int a = 0; a < rank; ++a) {
        if (total > (int64_t(1) << 40) / n) return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd: too large");
        total *= n;
    }
    const int64_t lines = total / n, W = 2 * n + 1;
    // per-line first / drift arrays and the relaxed engine's workspace
    int64_t* dfirst = nullptr;
    double* ddrift = nullptr;
    void* rws = nullptr;
    size_t rwsb = 0;
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&dfirst, static_cast<size_t>(lines) * sizeof(int64_t), s));
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&ddrift, static_cast<size_t>(lines) * sizeof(double), s));
    if (engine == LOB_ENGINE_RELAXED) {
        rwsb = relaxed_workspace_bytes(lines, n);
        LOB_CUDA_TRY(ctx, cudaMallocAsync(&rws, rwsb, s));
    }
    std::vector<int64_t> hf(static_cast<size_t>(lines));
    std::vector<double> hd(static_cast<size_t>(lines));
    // proj/src/splitting.cpp:53-77: axis 0 first; a line of axis a has stride n^(rank-1-a)
    const double* cur = u;
    double* bufs[2] = {out, tmp};
    int nb = 0;  // next buffer to write
    int st = LOB_OK;
    for (int a = 0; a < rank && st == LOB_OK; ++a) {
        int64_t B = 1;
        for (int b = a + 1; b < rank; ++b) B *= n;
        const int64_t A = total / (n * B);
        std::fill(hf.begin(), hf.end(), firsts ? firsts[a] : 0);
        std::fill(hd.begin(), hd.end(), drifts ? drifts[a] : 0.0);
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(dfirst, hf.data(), hf.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(ddrift, hd.data(), hd.size() * sizeof(double), cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));  // host vectors reused next axis
        const double* lines_src = cur;
        if (B > 1) {  // gather the axis' lines as contiguous rows
            double* t = bufs[nb];
            nb ^= 1;
            if ((st = launch_transpose_batched(ctx, cur, t, A, n, B, s))) break;
            lines_src = t;
        }
        double* dst = bufs[nb];
        nb ^= 1;
        const double* kt = ktabs ? ktabs + a * W : nullptr;
        if (engine == LOB_ENGINE_DIRECT)
            st = launch_direct_f64(ctx, lines_src, dst, lines, n, kt, 0, dfirst, nullptr, 0, s);
        else if (engine == LOB_ENGINE_RELAXED)
            st = launch_relaxed_f64(ctx, lines_src, dst, lines, n, kt, 0, dfirst, nullptr, 0, eta, nullptr, rws, rwsb, s);
        else
            st = launch_fast_f64(ctx, lines_src, dst, lines, n, ddrift, tau, nullptr, 0, 0.0, nullptr, workspace,
                                 workspace_bytes, 0, s);
        if (st) break;
        cur = dst;
        if (B > 1) {  // scatter back: rows (a, b) of length n -> (a, l, b)
            double* back = bufs[nb];
            nb ^= 1;
            if ((st = launch_transpose_batched(ctx, cur, back, A, B, n, s))) break;
            cur = back;
        }
    }
    if (st == LOB_OK && tv) st = launch_sub_table(ctx, const_cast<double*>(cur), tv, total, s);
    if (st == LOB_OK && cur != out)
        st = cuda_status(ctx, cudaMemcpyAsync(out, cur, static_cast<size_t>(total) * sizeof(double),
                                              cudaMemcpyDeviceToDevice, s), "split_step_nd copy");
    cudaFreeAsync(dfirst, s);
    cudaFreeAsync(ddrift, s);
    if (rws) cudaFreeAsync(rws, s);
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    return st;
}

int lob_split_step_nd_window_f64(lob_ctx* ctx, const double* u, double* out, double* tmp, int rank,
                                 const int64_t* dims, int64_t n, double tau, const double* ktabs,
                                 const int64_t* firsts, const double* tv, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (rank < 1 || rank > 8 || n < 1 || !dims || !ktabs || !firsts)
        return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd (windowed): bad arguments");
    if (!u || !out || !tmp || u == out || u == tmp || out == tmp)
        return set_error(ctx, LOB_INVALID_INPUT, "split_step_nd: need distinct u/out/tmp");
    (void)tau;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int64_t total = 1;
    for (int a = 0; a < rank; ++a) {
        if (dims[a] < 1) return set_error(ctx, LOB_INVALID_INPUT, "make_tensor: empty axis");
        total *= dims[a];
    }
    const int64_t W = 2 * n + 1;
    int64_t* dfirst = nullptr;
    int* d_err = nullptr;
    int64_t maxlines = 0;
    for (int a = 0; a < rank; ++a) maxlines = std::max(maxlines, total / dims[a]);
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&dfirst, static_cast<size_t>(maxlines) * sizeof(int64_t), s));
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&d_err, sizeof(int), s));
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(d_err, 0, sizeof(int), s));
    std::vector<int64_t> hf(static_cast<size_t>(maxlines));
    const double* cur = u;
    double* bufs[2] = {out, tmp};
    int nb = 0;
    int st = LOB_OK;
    // proj/src/splitting.cpp:53-77 with kinetic_convolve's wall branch (proj/src/scheme.cpp:135-144)
    for (int a = 0; a < rank && st == LOB_OK; ++a) {
        const int64_t L = dims[a];
        int64_t B = 1;
        for (int b = a + 1; b < rank; ++b) B *= dims[b];
        const int64_t A = total / (L * B), lines = A * B;
        std::fill(hf.begin(), hf.begin() + lines, firsts[a]);
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(dfirst, hf.data(), lines * sizeof(int64_t), cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        const double* src = cur;
        if (B > 1) {
            double* t = bufs[nb];
            nb ^= 1;
            if ((st = launch_transpose_batched(ctx, cur, t, A, L, B, s))) break;
            src = t;
        }
        double* dst = bufs[nb];
        nb ^= 1;
        if ((st = launch_window_f64(ctx, src, dst, lines, L, n, ktabs + a * W, 0, dfirst, nullptr, 0, d_err, s))) break;
        cur = dst;
        if (B > 1) {
            double* back = bufs[nb];
            nb ^= 1;
            if ((st = launch_transpose_batched(ctx, cur, back, A, B, L, s))) break;
            cur = back;
        }
    }
    if (st == LOB_OK && tv) st = launch_sub_table(ctx, const_cast<double*>(cur), tv, total, s);
    if (st == LOB_OK && cur != out)
        st = cuda_status(ctx, cudaMemcpyAsync(out, cur, static_cast<size_t>(total) * sizeof(double),
                                              cudaMemcpyDeviceToDevice, s), "split_step_nd copy");
    int herr = 0;
    if (st == LOB_OK) LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(dfirst, s);
    cudaFreeAsync(d_err, s);
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (st) return st;
    if (herr) return set_error(ctx, LOB_EVALUATION_ERROR, "kinetic_convolve: kernel window does not reach a grid index");
    return LOB_OK;
}

}  // extern "C"

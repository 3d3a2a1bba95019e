// Internal definitions shared by the laxol_b200 CUDA translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <set>
#include <string>
#include <tuple>

#include "../../include/laxol_b200.h"

struct lob_ctx {
    int device = 0;
    int sm_count = 148;
    cudaStream_t stream = nullptr;  // the context's own stream (host entry points)
    std::string last_error;
    int64_t launches = 0;
    // cached velocity tables v_d = (d*eps)/tau keyed by (n, tau bits)
    struct VTab {
        double* dev = nullptr;
        int64_t dmin = 0, count = 0;
    };
    std::map<std::pair<int64_t, uint64_t>, VTab> vtabs;
    // split-step axis inputs (kernel window, firsts, drifts) keyed by (n, tau bits, drift bits)
    std::map<std::tuple<int64_t, uint64_t, uint64_t>, void*> split_axes;
    // fast-engine workspaces: which statistics buffer holds the current u
    std::map<const void*, int64_t> ws_counter;
    std::map<const void*, std::pair<int64_t, int64_t>> ws_shape;
    std::map<const void*, const void*> ws_last_out;  // workspace -> out of its last K2 call
    std::map<const void*, int64_t> ws_chain;         // K2 launches since the done counters were reset
    std::map<const void*, bool> ws_fsm_valid;        // the workspace holds FSM summaries of its last out
    std::map<const void*, const void*> ws_table;     // workspace -> window table of its line constants
    std::map<const void*, bool> ws_lc_valid;         // the workspace holds line constants (mechanical)
    std::map<const void*, bool> ws_nostats;          // its last call (K2L) left no statistics of its out
    std::map<const void*, bool> ws_sampling;         // a checked call ran on it: steps store samples
    std::map<const void*, bool> ws_samples_valid;    // its last call stored samples of its out
    int fast_line = 2;  // n <= 2048: one CTA per whole line with in-kernel statistics (K2L); 2-D layout 2
    // K1 mode (LOB_DIRECT_SCREENED / LOB_DIRECT_PLAIN) and the screened kernel's
    // count of outputs swept in full fp64 (device counter, lazily allocated)
    int direct_mode = 0;
    int resident = 1;  // evolve of short lines through the on-chip resident kernel (K2R)
    double fast_delta_override = __builtin_nan("");  // lob_ctx_set_fast_delta (diagnostic)
    unsigned long long* direct_full = nullptr;  // [0] outputs swept in full, [1] fp64 candidates
    double* direct_umax = nullptr;              // per-line max |u| (screen bound)
    int64_t direct_umax_cap = 0;
    // host entry point pipeline: upload / compute / download streams and
    // per-chunk events (inputs ready, step done) + one for the shared inputs
    cudaStream_t aux[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t aux_ev[33] = {};
    // one-time per-device setup done through this context (kernel attributes, tables)
    std::set<const void*> done_once;
    // scratch for host entry points
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
};

namespace lob {

// Batches of more than 65535 lines (gridDim.y's limit): the line index folded over grid.y
// and grid.z, line = blockIdx.y + kGridY * blockIdx.z, CTAs past the last line exit.
constexpr unsigned kGridY = 65535u;
#ifdef __CUDACC__
inline dim3 line_grid(unsigned gx, int64_t lines) {
    return dim3(gx, static_cast<unsigned>(lines < kGridY ? lines : kGridY),
                static_cast<unsigned>((lines + kGridY - 1) / kGridY));
}
__device__ __forceinline__ int64_t grid_line() {
    // 32-bit (line counts stay below 2^31), and opaque: the compiler would otherwise re-derive
    // the index from the two special registers at every use
    unsigned l = blockIdx.y + kGridY * blockIdx.z;
    asm volatile("" : "+r"(l));
    return static_cast<int64_t>(l);
}
#endif


// true the first time `key` is seen by this context (per-device state is per context)
inline bool first_time(lob_ctx* ctx, const void* key) { return ctx->done_once.insert(key).second; }

inline int set_error(lob_ctx* ctx, int code, const std::string& msg) {
    if (ctx) ctx->last_error = msg;
    return code;
}

inline int cuda_status(lob_ctx* ctx, cudaError_t e, const char* where) {
    if (e == cudaSuccess) return LOB_OK;
    return set_error(ctx, LOB_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

#define LOB_CUDA_TRY(ctx, expr)                                      \
    do {                                                             \
        cudaError_t _e = (expr);                                     \
        if (_e != cudaSuccess) return ::lob::cuda_status(ctx, _e, #expr); \
    } while (0)

// Order-preserving map double -> uint64 (x < y  <=>  key(x) < key(y) for
// non-NaN x, y; -0 orders just below +0).
__device__ __forceinline__ unsigned long long dkey(double x) {
    unsigned hi = static_cast<unsigned>(__double2hiint(x));
    unsigned lo = static_cast<unsigned>(__double2loint(x));
    const unsigned m = static_cast<unsigned>(static_cast<int>(hi) >> 31);  // 0 or ~0
    hi ^= m | 0x80000000u;
    lo ^= m;
    return (static_cast<unsigned long long>(hi) << 32) | lo;
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
    unsigned hi = static_cast<unsigned>(k >> 32), lo = static_cast<unsigned>(k);
    const unsigned m = (hi & 0x80000000u) ? 0x80000000u : 0xffffffffu;
    hi ^= m;
    lo ^= (m == 0xffffffffu) ? 0xffffffffu : 0u;
    return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}
constexpr unsigned long long kKeyInf = 0xfff0000000000000ull;  // dkey(+inf)

inline int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}
inline int64_t posmod(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

// Launch helpers implemented in the .cu files.
int launch_direct_plain_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                            const double* ktab, int64_t ktab_stride, const int64_t* first,
                            const double* tv, int64_t tv_stride, cudaStream_t s);
int launch_direct_screen_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                             const double* ktab, int64_t ktab_stride, const int64_t* first,
                             const double* tv, int64_t tv_stride, unsigned long long* counters,
                             cudaStream_t s);
// dispatch on ctx->direct_mode
int launch_direct_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                      const double* ktab, int64_t ktab_stride, const int64_t* first,
                      const double* tv, int64_t tv_stride, cudaStream_t s);
int launch_direct_f32(lob_ctx* ctx, const float* u, float* out, int64_t lines, int64_t n,
                      const float* ktab, int64_t ktab_stride, const int64_t* first,
                      cudaStream_t s);
int launch_window_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t m,
                      int64_t n, const double* ktab, int64_t ktab_stride, const int64_t* first,
                      const double* tv, int64_t tv_stride, int* d_err, cudaStream_t s);

size_t fast_workspace_bytes(int64_t lines, int64_t n);
// window-table mode of K2: line l's window is ktab[l*stride + w], w = 0..2n, at
// displacements first[l] + w (device arrays)
struct FastTable {
    const double* ktab;
    int64_t stride;
    const int64_t* first;
};
// evolve's per-step drift reduced inside the K2 launch (with dpart): drift_out[line] (nullable),
// atomicMin(halt, step) on a non-finite line; dcount: per-line arrival counters, zeroed once
struct FastDriftOut {
    double* drift_out;
    int* halt;
    unsigned* dcount;
    int step;
};
// separable potential tau * (a1[line] * a2[j] + b) applied in K2's epilogue (device a1, a2)
struct FastSepPot {
    const double* a1;
    const double* a2;
    double b;
};
// launch_fast_f64 flag: the "in" statistics of u were written by the caller into the buffers
// fast_given_stats_buffers returned for this workspace (no statistics pass, no pointer check)
constexpr int kFastStatsGiven = 1 << 8;
// the flags a C-ABI caller may pass (the rest are internal)
constexpr int kFastUserFlags = LOB_FAST_STATS_VALID | LOB_FAST_CHAINED | LOB_FAST_STATS_CHECK;
// dpart (nullable): per-tile sums of u^{n+1} - u^n for evolve's drift ([lines][fast_tiles(n)]);
// tab (nullable): any convex window per line instead of the mechanical drift;
// sep (nullable): a separable potential instead of the tv table
int launch_fast_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                    const double* drift, double tau, const double* tv, int64_t tv_stride,
                    double eta, int64_t* blocks, void* workspace, size_t ws_bytes, int flags,
                    cudaStream_t s, double* dpart = nullptr, const FastTable* tab = nullptr,
                    const FastSepPot* sep = nullptr, const struct FastDriftOut* dout = nullptr);
// the statistics buffers the next launch_fast_f64 call on `workspace` reads (for kFastStatsGiven):
// per-256-sample sub-tile slope bounds [lines][subs] (double2: min, max) and per-line keys
// [lines][4] (umin, umax, smin, smax as order-preserving keys; the caller resets them)
int fast_given_stats_buffers(lob_ctx* ctx, void* workspace, int64_t lines, int64_t n, double2** sub,
                             unsigned long long** line_keys);
// dst = src^T of an n x n tensor plus the statistics of dst's lines for the next
// launch_fast_f64(..., kFastStatsGiven) on `workspace` (lines = n)
int launch_transpose_stats(lob_ctx* ctx, const double* src, double* dst, int64_t n, void* workspace,
                           cudaStream_t s);
int64_t fast_tiles(int64_t n);
// K2L: one step of short lines (n <= fast_line_max()) with statistics from the staged line itself;
// colin / colout: line l is column l of an n x n row-major tensor (lines == n)
int64_t fast_line_max();
// line layouts: a row; a column by strided accesses; a column exchanged through distributed shared
// memory in clusters of 8 CTAs; a column loaded by 2-D TMA tensor-map copies (load only)
enum : int { kLineRow = 0, kLineCol = 1, kLineClu = 2, kLineTma = 3 };
int launch_line_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n, const double* drift,
                    double tau, const double* tv, int64_t tv_stride, const FastSepPot* sep, int load, int store,
                    unsigned long long* diag, cudaStream_t s);
int launch_drift_tiles(lob_ctx* ctx, const double* dpart, int64_t lines, int64_t n, double* drift_out, int* halt,
                       int step, cudaStream_t s);
// K2R: all steps of an evolve of short lines (n <= 8192) in one launch, one CTA per line
bool fast_resident_ok(int64_t n);
// tv_period > 1: step k uses table tv + (k mod tv_period) * tv_step_stride (per line: + line * tv_stride)
int launch_fast_resident_f64(lob_ctx* ctx, double* u, int64_t lines, int64_t n, const double* drift, double tau,
                             const double* tv, int64_t tv_stride, double eta, int64_t steps, double* step_drift,
                             int64_t* step_blocks, int* halt, void* lc_buf, cudaStream_t s, int tv_period = 1,
                             int64_t tv_step_stride = 0);
int fast_diag_count(lob_ctx* ctx, void* workspace, int64_t lines, int64_t n, uint64_t* count,
                    cudaStream_t s);
int launch_block_counts(lob_ctx* ctx, const double* u, int64_t lines, int64_t n, double eta,
                        int64_t* blocks, cudaStream_t s);

// the reference's relaxed fast engine (relaxed.cu)
size_t relaxed_workspace_bytes(int64_t lines, int64_t n);
int launch_relaxed_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n, const double* ktab,
                       int64_t ktab_stride, const int64_t* first, const double* tv, int64_t tv_stride, double eta,
                       int64_t* blocks, void* workspace, size_t ws_bytes, cudaStream_t s);
// weak-KAM consumers (weakkam.cu)
int launch_tropical_gemm(lob_ctx* ctx, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t m, int64_t n, int64_t k, cudaStream_t s);
int launch_karp(lob_ctx* ctx, const double* M, int64_t n, double* D, double* lambda_dev, int* flag,
                cudaStream_t s);
int launch_period_matrix(lob_ctx* ctx, const double* kinc, const double* tvs, int64_t n, int64_t ell, double* C,
                         double* scratch, cudaStream_t s);

int launch_transpose(lob_ctx* ctx, const double* src, double* dst, int64_t n, cudaStream_t s);
int launch_transpose_batched(lob_ctx* ctx, const double* src, double* dst, int64_t A, int64_t L, int64_t B,
                             cudaStream_t s);
int launch_sub_table(lob_ctx* ctx, double* out, const double* tv, int64_t count, cudaStream_t s);
int launch_slab_unpack(lob_ctx* ctx, const double* recv, double* y, int64_t b, int64_t world, cudaStream_t s);
int launch_slab_push(lob_ctx* ctx, const double* x, int64_t b, int64_t world, int rank, double* const* peer_slabs,
                     cudaStream_t s);
int launch_potential2d(lob_ctx* ctx, double* out, const double* a1, const double* a2, double b,
                       double tau, int64_t n, cudaStream_t s, int64_t rows = -1);
int launch_drift(lob_ctx* ctx, const double* nxt, const double* cur, int64_t lines, int64_t n,
                 double* drift_out, int* halt, int step, cudaStream_t s);

}  // namespace lob

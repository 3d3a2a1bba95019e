// step_semidiscrete (proj/src/scheme.cpp:166-206): the
// direct min-plus step whose cost integrates V along the straight segment
// from source y to target x with the composite trapezoid rule,
//   out[j] = min_w u[src(j, w)] + (K[w] - tau/q * (V(t,y)/2 + V(t+tau,x)/2
//                                              + sum_{r=1}^{q-1} V(t + r/q tau, y + r/q (x - y)))),
// i.e. K1 with a cost computed per candidate.  The potential is one of the
// reference's built-in kinds (proj/src/hamiltonian.cpp:77-117): Zero, Const,
// Cosine (offset + amplitude * mod(omega t) * cos(frequency * theta(x))).
// The time factors amplitude * mod(omega t_r) are evaluated on the host with
// the C library (they depend on r only), the spatial cos on the device.
//
// Exactness: every IEEE operation is the reference's, in its order (no FMA);
// Zero and Const potentials give the reference's doubles exactly.  The
// Cosine kind differs only through the device cos (CUDA's double cos,
// <= 2 ulp, vs glibc): results agree within 1e-12 relative (tests state it).
#include <cmath>
#include <string>
#include <vector>

#include "lob_internal.cuh"

namespace lob {
namespace {

constexpr double kPi = 3.141592653589793;        // std::numbers::pi
constexpr double kTwoPiD = 2.0 * 3.141592653589793;  // kTwoPi, proj/src/hamiltonian.cpp:15
constexpr int kMaxQ = 64;                        // quad_points handled on the device

struct SemiPot {
    int kind;  // LOB_POTENTIAL_*
    double value, offset, freq;
    double am[kMaxQ + 1];  // amplitude * mod(omega t_r), r = 0..q (t_0 = t, t_q = t + tau)
};

// theta(x) = 2 pi (x - floor x) - pi  (proj/src/hamiltonian.cpp:18-21)
__device__ __forceinline__ double theta(double x) {
    const double r = __dsub_rn(x, floor(x));
    return __dsub_rn(__dmul_rn(kTwoPiD, r), kPi);
}

// Potential::operator() at time index r (proj/src/hamiltonian.cpp:98-117)
__device__ __forceinline__ double vpot(const SemiPot& P, int r, double x) {
    if (P.kind == LOB_POTENTIAL_ZERO) return 0.0;
    if (P.kind == LOB_POTENTIAL_CONST) return P.value;
    return __dadd_rn(P.offset, __dmul_rn(P.am[r], cos(__dmul_rn(P.freq, theta(x)))));
}

// CTA = 32 consecutive outputs x kParts contiguous parts of the window (one warp per
// part, lanes = outputs: coalesced u reads); the parts' minima are combined in window
// order with a strict "<" (the reference's first minimum wins).
constexpr int kParts = 4;
__global__ void __launch_bounds__(32 * kParts) semidiscrete_kernel(
    const double* __restrict__ u, double* __restrict__ out, int64_t m, int64_t n, int periodic, double origin,
    double step, const double* __restrict__ ktab, int64_t first, double tau, int q, SemiPot P,
    int* __restrict__ err, int64_t lines) {
    __shared__ double part[kParts][32];
    const int64_t line = grid_line();
    if (line >= lines) return;  // (uniform per CTA: before any barrier)
    const int lane = threadIdx.x & 31, pw = threadIdx.x >> 5;
    const int64_t j = static_cast<int64_t>(blockIdx.x) * 32 + lane;
    const double* ul = u + line * m;
    const int64_t W = 2 * n + 1;
    const int64_t per = (W + kParts - 1) / kParts;
    const int64_t w0 = pw * per, w1 = min(W, w0 + per);
    double best = INFINITY;
    if (j < m) {
        // sample_coord (proj/src/scheme.cpp:32-35)
        int64_t jc = j;
        if (periodic && jc >= n) jc -= n * (jc / n);
        const double x = __dadd_rn(origin, __dmul_rn(static_cast<double>(jc), step));
        const double vx = vpot(P, q, x);  // V(t + tau, x)
        const double tq = __ddiv_rn(tau, static_cast<double>(q));
        for (int64_t w = w0; w < w1; ++w) {
            const int64_t d = first + w;
            int64_t src = j - d;
            if (periodic) {
                src %= n;
                if (src < 0) src += n;
            } else if (src < 0 || src >= m) {
                continue;
            }
            const double y = __dsub_rn(x, __dmul_rn(static_cast<double>(d), step));
            double acc = __dmul_rn(0.5, __dadd_rn(vpot(P, 0, y), vx));
            if (P.kind != LOB_POTENTIAL_ZERO) {
                const double xy = __dsub_rn(x, y);
                for (int r = 1; r < q; ++r) {
                    const double frac = __ddiv_rn(static_cast<double>(r), static_cast<double>(q));
                    acc = __dadd_rn(acc, vpot(P, r, __dadd_rn(y, __dmul_rn(frac, xy))));
                }
            }
            const double integral = __dmul_rn(tq, acc);
            const double cost = __dsub_rn(__ldg(ktab + w), integral);
            const double c = __dadd_rn(__ldg(ul + src), cost);
            best = c < best ? c : best;  // std::min(best, c)
        }
    }
    part[pw][lane] = best;
    __syncthreads();
    if (pw == 0 && j < m) {
#pragma unroll
        for (int k = 1; k < kParts; ++k) best = part[k][lane] < best ? part[k][lane] : best;
        if (best == INFINITY) atomicOr(err, 1);
        out[line * m + j] = best;
    }
}

}  // namespace
}  // namespace lob

using namespace lob;

extern "C" int lob_step_semidiscrete_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t m,
                                         int64_t n_space, int periodic, double origin, const double* ktab,
                                         int64_t first, double t, double tau, const lob_potential* V,
                                         int quad_points, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (quad_points < 1) return set_error(ctx, LOB_INVALID_INPUT, "step_semidiscrete: quad_points must be >= 1");
    if (quad_points > kMaxQ)
        return set_error(ctx, LOB_INVALID_INPUT, "step_semidiscrete: quad_points above the device limit (64)");
    if (lines < 0 || m < 1 || n_space < 1 || (periodic && m != n_space))
        return set_error(ctx, LOB_INVALID_INPUT, "step_semidiscrete: bad shape");
    if (!(tau > 0.0)) return set_error(ctx, LOB_INVALID_INPUT, "step_semidiscrete: tau must be positive");
    if (lines == 0) return LOB_OK;
    SemiPot P{};
    P.kind = V ? V->kind : LOB_POTENTIAL_ZERO;
    if (P.kind < LOB_POTENTIAL_ZERO || P.kind > LOB_POTENTIAL_COSINE)
        return set_error(ctx, LOB_INVALID_INPUT, "step_semidiscrete: unknown potential kind");
    if (P.kind == LOB_POTENTIAL_CONST) P.value = V->value;
    if (P.kind == LOB_POTENTIAL_COSINE) {
        if (V->frequency < 1) return set_error(ctx, LOB_INVALID_INPUT, "potential_cosine: frequency must be >= 1");
        P.offset = V->offset;
        P.freq = static_cast<double>(V->frequency);
        // amplitude * mod(omega t_r) on the host (proj/src/hamiltonian.cpp:105-110), the
        // reference's time points t, t + (r/q) tau, t + tau (proj/src/scheme.cpp:190-196)
        for (int r = 0; r <= quad_points; ++r) {
            double tr;
            if (r == 0) tr = t;
            else if (r == quad_points) tr = t + tau;
            else tr = t + (static_cast<double>(r) / static_cast<double>(quad_points)) * tau;
            double mod = 1.0;
            if (V->tmod == LOB_TMOD_SIN) mod = std::sin(V->omega * tr);
            else if (V->tmod == LOB_TMOD_COS) mod = std::cos(V->omega * tr);
            P.am[r] = V->amplitude * mod;
        }
    }
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int* err = nullptr;
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&err, sizeof(int), s));
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(err, 0, sizeof(int), s));
    const double step = 1.0 / static_cast<double>(n_space);
    const dim3 grid = line_grid(static_cast<unsigned>((m + 31) / 32), lines);
    semidiscrete_kernel<<<grid, 32 * kParts, 0, s>>>(u, out, m, n_space, periodic, origin, step, ktab, first, tau,
                                             quad_points, P, err, lines);
    ctx->launches += 1;
    int herr = 0;
    LOB_CUDA_TRY(ctx, cudaGetLastError());
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&herr, err, sizeof(int), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(err, s);
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (herr) return set_error(ctx, LOB_EVALUATION_ERROR, "step_semidiscrete: no candidate source for a grid index");
    return LOB_OK;
}

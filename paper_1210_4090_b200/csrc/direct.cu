// K1 — direct O(n^2) periodic min-plus step for batches of lines.
//
// Replaces, per line, the reference's conv_naive double loop
// (proj/src/minplus.cpp:116-126), the periodic aliasing min
// (proj/src/scheme.cpp:125-134) and the potential loop
// (proj/src/scheme.cpp:156-162) by the definition-level formula the
// reference pins with == (proj/tests/unit_scheme.cpp:176-194):
//
//   out[l][j] = min_{w=0..2n} ( u[l][(j - first_l - w) mod n] + K_l[w] )  -  tv_l[j]
//
// Every candidate is one IEEE add and the min is exact, so the result is
// bit-identical to the reference for the same K table (signed zeros aside).
//
// Design (sm_100a, FP64 non-tensor pipe bound): a CTA owns a tile of
// TJ = NT*R consecutive outputs of one line; each thread owns R consecutive
// outputs and keeps them in registers.  The window is swept in chunks of TW
// displacements staged in shared memory (u for the chunk's source range, K
// for the chunk).  For consecutive w the R sources of a thread shift by one,
// so a register window of 2R values slides with one LDS per displacement and
// the K value is a shared-memory broadcast: per candidate the SASS is
// DADD + DSETP + 2x FSEL and nothing else (R^2 candidates per R LDS.64 of u
// and R broadcast LDS of K).  u is padded one double per R in shared memory
// so the stride-R per-thread reads are bank-conflict free.
#include <cstdlib>

#include "direct_common.cuh"

namespace lob {
namespace {
using namespace k1;

template <typename T, int R, int NT, int TW>
__global__ void __launch_bounds__(NT) direct_kernel(const T* __restrict__ u, T* __restrict__ out,
                                                    int64_t n, int64_t tiles,
                                                    const T* __restrict__ ktab,
                                                    int64_t ktab_stride,
                                                    const int64_t* __restrict__ first_arr,
                                                    const double* __restrict__ tv,
                                                    int64_t tv_stride) {
    constexpr int TJ = NT * R;
    constexpr int L = TJ + TW;  // staged source range per chunk
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T* Us = reinterpret_cast<T*>(smem_raw);
    T* Ks = Us + padded<R>(L) + 1;

    const int64_t line = blockIdx.x / tiles;
    const int64_t tile = blockIdx.x - line * tiles;
    const int64_t j0 = tile * TJ;
    const int t = threadIdx.x;
    const T* ul = u + line * n;
    const T* Kl = ktab + line * ktab_stride;
    const int64_t first = first_arr[line];
    const int64_t W = 2 * n + 1;

    T best[R];
#pragma unroll
    for (int r = 0; r < R; ++r) best[r] = pos_inf<T>();
    k1::sweep_range<T, R, NT, TW>(Us, Ks, ul, Kl, n, j0, first, 0, W, best);

    const int64_t jt = j0 + static_cast<int64_t>(t) * R;
    T* ol = out + line * n;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t j = jt + r;
        if (j < n) {
            if constexpr (sizeof(T) == 8) {
                // out[j] -= tau*V: one IEEE subtraction (proj/src/scheme.cpp:161)
                ol[j] = tv ? __dsub_rn(best[r], tv[line * tv_stride + j]) : best[r];
            } else {
                ol[j] = best[r];
            }
        }
    }
}

template <typename T, int R, int NT, int TW>
int launch_cfg(lob_ctx* ctx, const T* u, T* out, int64_t lines, int64_t n, const T* ktab,
               int64_t ktab_stride, const int64_t* first, const double* tv, int64_t tv_stride,
               cudaStream_t s) {
    constexpr int TJ = NT * R;
    constexpr int L = TJ + TW;
    const size_t smem = (padded<R>(L) + 1 + TW) * sizeof(T);
    auto kern = direct_kernel<T, R, NT, TW>;
    if (first_time(ctx, reinterpret_cast<const void*>(kern)))
        LOB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem)));
    const int64_t tiles = (n + TJ - 1) / TJ;
    const int64_t blocks = tiles * lines;
    if (blocks > 0x7fffffffll) return set_error(ctx, LOB_INVALID_INPUT, "direct: grid too large");
    kern<<<static_cast<unsigned>(blocks), NT, smem, s>>>(u, out, n, tiles, ktab, ktab_stride,
                                                          first, tv, tv_stride);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "direct_kernel launch");
}

// Windowed (non-periodic) lines: tests and drop-in completeness only.
__global__ void window_kernel(const double* __restrict__ u, double* __restrict__ out, int64_t m,
                              int64_t n, const double* __restrict__ ktab, int64_t ktab_stride,
                              const int64_t* __restrict__ first_arr, const double* __restrict__ tv,
                              int64_t tv_stride, int* err, int64_t lines) {
    const int64_t line = grid_line();
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= m || line >= lines) return;
    const int64_t W = 2 * n + 1;
    const int64_t r = j - first_arr[line];  // conv index j + shift (proj/src/scheme.cpp:137)
    if (r < 0 || r >= W + m - 1) {
        atomicExch(err, 1);
        return;
    }
    const double* ul = u + line * m;
    const double* Kl = ktab + line * ktab_stride;
    double best = __longlong_as_double(0x7ff0000000000000ll);
    const int64_t wlo = r - (m - 1) > 0 ? r - (m - 1) : 0;
    const int64_t whi = r < W - 1 ? r : W - 1;
    for (int64_t w = wlo; w <= whi; ++w) {
        const double c = __dadd_rn(ul[r - w], Kl[w]);
        best = c < best ? c : best;
    }
    out[line * m + j] = tv ? __dsub_rn(best, tv[line * tv_stride + j]) : best;
}

}  // namespace

int launch_direct_plain_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                            const double* ktab, int64_t ktab_stride, const int64_t* first,
                            const double* tv, int64_t tv_stride, cudaStream_t s) {
    if (n >= 2048)
        return launch_cfg<double, 16, 128, 1024>(ctx, u, out, lines, n, ktab, ktab_stride, first,
                                                 tv, tv_stride, s);
    if (n >= 512)
        return launch_cfg<double, 8, 64, 512>(ctx, u, out, lines, n, ktab, ktab_stride, first, tv,
                                              tv_stride, s);
    return launch_cfg<double, 4, 32, 128>(ctx, u, out, lines, n, ktab, ktab_stride, first, tv,
                                          tv_stride, s);
}

int launch_direct_f32(lob_ctx* ctx, const float* u, float* out, int64_t lines, int64_t n,
                      const float* ktab, int64_t ktab_stride, const int64_t* first,
                      cudaStream_t s) {
    if (n >= 2048)
        return launch_cfg<float, 16, 128, 1024>(ctx, u, out, lines, n, ktab, ktab_stride, first,
                                                nullptr, 0, s);
    if (n >= 512)
        return launch_cfg<float, 8, 64, 512>(ctx, u, out, lines, n, ktab, ktab_stride, first,
                                             nullptr, 0, s);
    return launch_cfg<float, 4, 32, 128>(ctx, u, out, lines, n, ktab, ktab_stride, first, nullptr,
                                         0, s);
}

int launch_window_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t m,
                      int64_t n, const double* ktab, int64_t ktab_stride, const int64_t* first,
                      const double* tv, int64_t tv_stride, int* d_err, cudaStream_t s) {
    const dim3 grid = line_grid(static_cast<unsigned>((m + 127) / 128), lines);
    window_kernel<<<grid, 128, 0, s>>>(u, out, m, n, ktab, ktab_stride, first, tv, tv_stride,
                                       d_err, lines);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "window_kernel launch");
}

}  // namespace lob

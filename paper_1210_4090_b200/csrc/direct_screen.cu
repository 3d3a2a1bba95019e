// K1s — direct O(n^2) periodic min-plus step, fp64-exact through an fp32 screen.
//
// Same contract as K1 (csrc/direct.cu): for every output
//
//   out[l][j] = min_{w=0..2n} fl64( u[l][(j - first_l - w) mod n] + K_l[w] )  -  tv_l[j]
//
// bit-identical to the reference's conv_naive + aliasing + potential
// (proj/src/minplus.cpp:116-126, proj/src/scheme.cpp:125-134,156-162), but the
// O(n^2) sweep runs on the FP32 pipes and only O(n) candidates per output are
// evaluated in fp64:
//
//  1. Screen (fp32): u32 = fl32(u), K32 = fl32(K), c32_w = fl32(u32 + K32) is
//     swept exactly like K1 (register-blocked, FADD + FMNMX3 per 2 candidates)
//     while every output keeps the minimum of each sub-chunk of kSub
//     consecutive displacements: the best sub-chunk (value, index) and the
//     second-best sub-chunk minimum.
//  2. Bound: |c32_w - (u + K)_w| <= e(c32_w) = rho (|c32_w| + 2 Umax) + tiny,
//     rho = 2^-22.8 (three fp32 roundings; |u| + |K| <= |u + K| + 2|u|),
//     Umax = max |u| over the line (every CTA stages the whole period).
//     e() is increasing in c32, so a sub-chunk whose fp32 minimum s satisfies
//     s - e(s) > best + e(best) holds no candidate that can reach the exact
//     minimum (whose value is <= best + e(best)).
//  3. Exact (fp64): if the second-best sub-chunk is excluded, the kSub
//     candidates of the best sub-chunk are re-evaluated in fp64 and their
//     exact min is the answer; otherwise (near-ties across sub-chunks, or any
//     non-finite fp32 conversion in the CTA) the output is swept in full fp64.
// fl64 is monotone, so min over candidates of fl64(u + K) = fl64 of the exact
// minimum, and any candidate set containing an exact minimiser gives the
// same double: the result is the reference's, bit for bit (signed zeros
// aside, as for K1).
#include <cfloat>

#include "lob_internal.cuh"

namespace lob {
namespace {

constexpr double kRho = 1.4016e-7;  // 2^-22.8 > 3 * 2^-24 / (1 - 2^-22)

template <int R>
__host__ __device__ __forceinline__ constexpr int padded_s(int i) {
    return i + i / R;
}

__device__ __noinline__ double exact_sweep(const double* __restrict__ ul, const double* __restrict__ Kl,
                                              int64_t n, int64_t j, int64_t first, int64_t w0, int64_t w1) {
    // min over w in [w0, w1) of u[(j - first - w) mod n] + K[w]   (fp64, exact min)
    double best = __longlong_as_double(0x7ff0000000000000ll);
    int64_t y = (j - first - w0) % n;
    if (y < 0) y += n;
    for (int64_t w = w0; w < w1; ++w) {
        const double c = __dadd_rn(__ldg(ul + y), __ldg(Kl + w));
        best = c < best ? c : best;
        y = y == 0 ? n - 1 : y - 1;
    }
    return best;
}

template <int R, int NT, int TW, int SUB>
#ifndef LOB_SCREEN_MINB
#define LOB_SCREEN_MINB 1
#endif
__global__ void __launch_bounds__(NT, LOB_SCREEN_MINB) screen_kernel(const double* __restrict__ u, double* __restrict__ out,
                                                    int64_t n, int64_t tiles, const double* __restrict__ ktab,
                                                    int64_t ktab_stride, const int64_t* __restrict__ first_arr,
                                                    const double* __restrict__ tv, int64_t tv_stride,
                                                    unsigned long long* __restrict__ counters) {
    static_assert(TW % SUB == 0 && SUB % R == 0, "sub-chunks tile the chunks");
    constexpr int TJ = NT * R;
    constexpr int L = TJ + TW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* Us = reinterpret_cast<float*>(smem_raw);
    float* Ks = Us + padded_s<R>(L) + 1;
    __shared__ double red_umax[NT / 32];
    __shared__ int red_bad[NT / 32];

    const int64_t line = blockIdx.x / tiles;
    const int64_t tile = blockIdx.x - line * tiles;
    const int64_t j0 = tile * TJ;
    const int t = threadIdx.x;
    const double* ul = u + line * n;
    const double* Kl = ktab + line * ktab_stride;
    const int64_t first = first_arr[line];
    const int64_t W = 2 * n + 1;
    const float finf = __int_as_float(0x7f800000);

    float cur[R], best[R], sec[R];
    int bidx[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        cur[r] = finf;
        best[r] = finf;
        sec[r] = finf;
        bidx[r] = 0;
    }
    double umax = 0.0;
    bool bad = false;

    for (int64_t wc = 0; wc < W; wc += TW) {
        __syncthreads();
        const int64_t ylo = j0 - first - wc - TW;
        int64_t ym = ylo % n;
        if (ym < 0) ym += n;
        for (int i = t; i < L; i += NT) {
            int64_t y = ym + i;
            y -= (y / n) * n;
            const double v = __ldg(ul + y);
            const float v32 = __double2float_rn(v);
            umax = fmax(umax, fabs(v));
            bad |= !(fabsf(v32) <= FLT_MAX);
            Us[padded_s<R>(i)] = v32;
        }
        for (int s = t; s < TW; s += NT) {
            const int64_t w = wc + s;
            float k32 = finf;
            if (w < W) {
                k32 = __double2float_rn(__ldg(Kl + w));
                bad |= !(fabsf(k32) <= FLT_MAX);
            }
            Ks[s] = k32;
        }
        __syncthreads();

        // i0 = t*R + TW - s0 is a multiple of R: padded(i0 + k) = pa + k,
        // padded(i0 - 1 - k) = pa - 2 - k with pa = padded(i0)
        const float* pa = Us + padded_s<R>(t * R + TW);
        float A[R];
#pragma unroll
        for (int k = 0; k < R; ++k) A[k] = pa[k];
        // the last chunk stops at the window's end (rounded up to R)
        const int send = static_cast<int>(min(static_cast<int64_t>(TW), (W - wc + R - 1) / R * R));
#ifdef LOB_S0_UNROLL
#pragma unroll 2
#else
#pragma unroll 1
#endif
        for (int s0 = 0; s0 < send; s0 += R) {
            float B[R];
#pragma unroll
            for (int k = 0; k < R; ++k) B[k] = pa[-2 - k];
#pragma unroll
            for (int s = 0; s < R; s += 2) {
                const float ka = Ks[s0 + s], kb = Ks[s0 + s + 1];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int ia = r - s, ib = r - s - 1;
                    const float va = ia >= 0 ? A[ia >= 0 ? ia : 0] : B[ia < 0 ? -ia - 1 : 0];
                    const float vb = ib >= 0 ? A[ib >= 0 ? ib : 0] : B[ib < 0 ? -ib - 1 : 0];
                    cur[r] = fminf(cur[r], fminf(__fadd_rn(va, ka), __fadd_rn(vb, kb)));  // FMNMX3
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) A[k] = B[R - 1 - k];
            pa -= R + 1;
            if ((s0 + R) % SUB == 0 || s0 + R == send) {
                // sub-chunk containing displacement wc + s0 complete (or the window ended)
                const int sub = static_cast<int>((wc + s0) / SUB);
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float c = cur[r];
                    const bool nb = c < best[r];
                    sec[r] = nb ? best[r] : fminf(sec[r], c);
                    bidx[r] = nb ? sub : bidx[r];
                    best[r] = nb ? c : best[r];
                    cur[r] = finf;
                }
            }
        }
    }

    // Umax and the "screen unusable" flag over the CTA (it staged the whole period)
#pragma unroll
    for (int o = 16; o; o >>= 1) umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
    const int badw = __any_sync(0xffffffffu, bad);
    if ((t & 31) == 0) {
        red_umax[t >> 5] = umax;
        red_bad[t >> 5] = badw;
    }
    __syncthreads();
    umax = 0.0;
    int anybad = 0;
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) {
        umax = fmax(umax, red_umax[k]);
        anybad |= red_bad[k];
    }
    const double u2 = 2.0 * umax;

    const int64_t jt = j0 + static_cast<int64_t>(t) * R;
    double* ol = out + line * n;
    unsigned nfull = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t j = jt + r;
        if (j >= n) continue;
        const double b = best[r], s2 = sec[r];
        const double hi = b + (kRho * (fabs(b) + u2) + 1e-44);          // >= exact minimum
        const double lo2 = s2 - (kRho * (fabs(s2) + u2) + 1e-44);       // <= every other sub-chunk
        double m;
        if (!anybad && lo2 > hi && b == b) {
            const int64_t w0 = static_cast<int64_t>(bidx[r]) * SUB;
            m = exact_sweep(ul, Kl, n, j, first, w0, min(w0 + SUB, W));
        } else {
            m = exact_sweep(ul, Kl, n, j, first, 0, W);
            ++nfull;
        }
        // out[j] -= tau*V: one IEEE subtraction (proj/src/scheme.cpp:161)
        ol[j] = tv ? __dsub_rn(m, tv[line * tv_stride + j]) : m;
    }
    if (counters && nfull) atomicAdd(counters, static_cast<unsigned long long>(nfull));
}

template <int R, int NT, int TW, int SUB>
int launch_screen_cfg(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                      const double* ktab, int64_t ktab_stride, const int64_t* first, const double* tv,
                      int64_t tv_stride, unsigned long long* counters, cudaStream_t s) {
    constexpr int TJ = NT * R;
    constexpr int L = TJ + TW;
    const size_t smem = (padded_s<R>(L) + 1 + TW) * sizeof(float);
    auto kern = screen_kernel<R, NT, TW, SUB>;
    static bool attr_set = false;
    if (!attr_set) {
        LOB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem)));
        attr_set = true;
    }
    const int64_t tiles = (n + TJ - 1) / TJ;
    const int64_t blocks = tiles * lines;
    if (blocks > 0x7fffffffll) return set_error(ctx, LOB_INVALID_INPUT, "direct: grid too large");
    kern<<<static_cast<unsigned>(blocks), NT, smem, s>>>(u, out, n, tiles, ktab, ktab_stride, first, tv,
                                                          tv_stride, counters);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "screen_kernel launch");
}

}  // namespace

int launch_direct_screen_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                             const double* ktab, int64_t ktab_stride, const int64_t* first,
                             const double* tv, int64_t tv_stride, unsigned long long* counters,
                             cudaStream_t s) {
    if (n >= 2048)
        return launch_screen_cfg<16, 128, 1024, 64>(ctx, u, out, lines, n, ktab, ktab_stride, first, tv,
                                                    tv_stride, counters, s);
    if (n >= 512)
        return launch_screen_cfg<8, 64, 512, 64>(ctx, u, out, lines, n, ktab, ktab_stride, first, tv,
                                                 tv_stride, counters, s);
    return launch_screen_cfg<4, 32, 128, 32>(ctx, u, out, lines, n, ktab, ktab_stride, first, tv, tv_stride,
                                             counters, s);
}

int launch_direct_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                      const double* ktab, int64_t ktab_stride, const int64_t* first,
                      const double* tv, int64_t tv_stride, cudaStream_t s) {
    if (ctx->direct_mode == LOB_DIRECT_PLAIN)
        return launch_direct_plain_f64(ctx, u, out, lines, n, ktab, ktab_stride, first, tv, tv_stride, s);
    if (!ctx->direct_full) {
        LOB_CUDA_TRY(ctx, cudaMalloc(&ctx->direct_full, sizeof(unsigned long long)));
        LOB_CUDA_TRY(ctx, cudaMemset(ctx->direct_full, 0, sizeof(unsigned long long)));
    }
    return launch_direct_screen_f64(ctx, u, out, lines, n, ktab, ktab_stride, first, tv, tv_stride,
                                    ctx->direct_full, s);
}

}  // namespace lob

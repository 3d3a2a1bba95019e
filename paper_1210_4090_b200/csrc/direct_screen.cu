// K1s — direct O(n^2) periodic min-plus step, fp64-exact through an fp32 screen.
//
// Same contract as K1 (csrc/direct.cu): for every output
//
//   out[l][j] = min_{w=0..2n} fl64( u[l][(j - first_l - w) mod n] + K_l[w] )  -  tv_l[j]
//
// bit-identical to the reference's conv_naive + aliasing + potential
// (proj/src/minplus.cpp:116-126, proj/src/scheme.cpp:125-134,156-162), but the
// O(n^2) sweep runs on the FP32 pipes and only the candidates that can reach
// the minimum are evaluated in fp64:
//
//  1. Screen (fp32): u32 = fl32(u), K32 = fl32(K), c32_w = fl32(u32 + K32) is
//     swept like K1 (register-blocked, FADD + FMNMX3 per 2 candidates), the
//     window's chunks in the order centre (w = n, the kernel's minimum) first,
//     so the running minimum settles early.  Every output keeps its running
//     fp32 minimum b and the span [lo, hi] of sub-chunks (kSub consecutive
//     displacements) whose minimum m passed the inclusion test below.
//  2. Bound: |c32_w - (u + K)_w| <= e(c32_w) = rho (|c32_w| + 2 Umax) + sigma,
//     rho = 2^-22.8 >= three fp32 roundings (|u| + |K| <= |u + K| + 2|u|),
//     sigma covers fp32 subnormals, Umax = max |u| over the line (pre-pass).
//     A sub-chunk with m - e(m) > b + e(b) cannot hold an exact minimiser
//     (the exact minimum is <= b + e(b)); the test m - b <= e(m) + e(b) is
//     evaluated in fp64 against the running b >= the final b, so the span is
//     a superset of the sub-chunks that can hold the minimiser.
//  3. Exact (fp64): the span's candidates are re-evaluated in fp64; their
//     exact min is the answer.  Any non-finite fp32 conversion in the CTA (or
//     a non-finite screen) sends the output to the full fp64 sweep.
// fl64 is monotone, so min over candidates of fl64(u + K) = fl64 of the exact
// minimum, and any candidate set containing an exact minimiser gives the
// same double: the result is the reference's, bit for bit (signed zeros
// aside, as for K1).
#include <cfloat>
#include <climits>

#include "direct_common.cuh"

namespace lob {
namespace {
using namespace k1;

constexpr double kRho = 1.4016e-7;    // 2^-22.8 > 2^-23 (1 + 2^-25) / (1 - 2^-22.9): three fp32 roundings
constexpr float kRho32 = 1.4157e-7f;  // 1.01 rho

template <int R>
__host__ __device__ __forceinline__ constexpr int padded_s(int i) {
    return i + i / R;
}

// max |u| per line (NaN -> +inf: every sub-chunk then passes the test)
__global__ void line_absmax_kernel(const double* __restrict__ u, int64_t n, double* __restrict__ umax) {
    const double* ul = u + static_cast<int64_t>(blockIdx.x) * n;
    double m = 0.0;
    bool nan = false;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const double v = fabs(__ldg(ul + i));
        nan |= v != v;
        m = fmax(m, v);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    nan = __any_sync(0xffffffffu, nan);
    __shared__ double red[32];
    __shared__ int rn[32];
    if ((threadIdx.x & 31) == 0) {
        red[threadIdx.x >> 5] = m;
        rn[threadIdx.x >> 5] = nan;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k) {
            m = fmax(m, red[k]);
            nan |= rn[k];
        }
        umax[blockIdx.x] = nan ? __longlong_as_double(0x7ff0000000000000ll) : m;
    }
}

template <int R, int NT, int TW, int SUB>
#ifndef LOB_SCREEN_MINB
#define LOB_SCREEN_MINB 4
#endif
__global__ void __launch_bounds__(NT, LOB_SCREEN_MINB)
    screen_kernel(const double* __restrict__ u, double* __restrict__ out, int64_t n, int64_t tiles,
                  const double* __restrict__ ktab, int64_t ktab_stride, const int64_t* __restrict__ first_arr,
                  const double* __restrict__ tv, int64_t tv_stride, const double* __restrict__ umax_arr,
                  unsigned long long* __restrict__ counters) {
    static_assert(TW % SUB == 0 && SUB % R == 0, "sub-chunks tile the chunks");
    constexpr int TJ = NT * R;
    constexpr int L = TJ + TW;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float* Us = reinterpret_cast<float*>(smem_raw);
    float* Ks = Us + padded_s<R>(L) + 1;

    const int64_t line = blockIdx.x / tiles;
    const int64_t tile = blockIdx.x - line * tiles;
    const int64_t j0 = tile * TJ;
    const int t = threadIdx.x;
    const double* ul = u + line * n;
    const double* Kl = ktab + line * ktab_stride;
    const int64_t first = first_arr[line];
    const int64_t W = 2 * n + 1;
    const float finf = __int_as_float(0x7f800000);
    const float u4f = __double2float_ru(4.0 * umax_arr[line]);  // 2 Umax for each of the two bounds

    float cur[R], best[R];
    int lo[R], hi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        cur[r] = finf;
        best[r] = finf;
        lo[r] = INT_MAX;
        hi[r] = -1;
    }
    bool bad = false;

    const int64_t nch = (W + TW - 1) / TW;
    const int64_t c0 = n / TW;  // chunk of the window centre w = n (displacement = centre)
    for (int64_t ck = 0; ck < nch; ++ck) {
        const int64_t wc = ((c0 + ck) % nch) * TW;
        __syncthreads();
        const int64_t ylo = j0 - first - wc - TW;
        int64_t ym = ylo % n;
        if (ym < 0) ym += n;
        for (int i = t; i < L; i += NT) {
            int64_t y = ym + i;
            y -= (y / n) * n;
            const float v32 = __double2float_rn(__ldg(ul + y));
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
#pragma unroll 1
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
                    const float m = cur[r];
                    best[r] = fminf(best[r], m);
                    // m - b <= e(m) + e(b) = rho (|m| + |b| + 4 Umax) + 2 sigma, evaluated in
                    // fp32 with rho inflated 1% (covers the test's own four roundings)
                    const bool incl = m - best[r] <= kRho32 * (fabsf(m) + fabsf(best[r]) + u4f) + 2e-44f;
                    lo[r] = incl ? min(lo[r], sub) : lo[r];
                    hi[r] = incl ? max(hi[r], sub) : hi[r];
                    cur[r] = finf;
                }
            }
        }
    }
    const bool anybad = __syncthreads_or(bad);  // also: every thread is done with Us / Ks

    // CTA union of the spans: one register-blocked fp64 sweep over it serves all outputs
    // (a superset of every output's span still has that output's exact minimiser)
    const int64_t jt = j0 + static_cast<int64_t>(t) * R;
    int l = INT_MAX, h = -1;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        if (jt + r < n) {
            l = min(l, lo[r]);
            h = max(h, hi[r]);
        }
    }
    l = __reduce_min_sync(0xffffffffu, l);
    h = __reduce_max_sync(0xffffffffu, h);
    __shared__ int span_lo[NT / 32], span_hi[NT / 32];
    if ((t & 31) == 0) {
        span_lo[t >> 5] = l;
        span_hi[t >> 5] = h;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < NT / 32; ++k) {
        l = min(l, span_lo[k]);
        h = max(h, span_hi[k]);
    }
    int64_t wbeg = 0, wend = W;
    const bool full = anybad || l > h;
    if (!full) {
        wbeg = static_cast<int64_t>(l) * SUB;
        wend = min(static_cast<int64_t>(h + 1) * SUB, W);
    }
    double best64[R];
#pragma unroll
    for (int r = 0; r < R; ++r) best64[r] = pos_inf<double>();
    k1::sweep_range<double, R, NT, TW>(reinterpret_cast<double*>(smem_raw),
                                       reinterpret_cast<double*>(smem_raw) + padded<R>(L) + 1, ul, Kl, n, j0,
                                       first, wbeg, wend, best64);

    double* ol = out + line * n;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int64_t j = jt + r;
        // out[j] -= tau*V: one IEEE subtraction (proj/src/scheme.cpp:161)
        if (j < n) ol[j] = tv ? __dsub_rn(best64[r], tv[line * tv_stride + j]) : best64[r];
    }
    if (counters && t == 0) {
        const unsigned long long outs = static_cast<unsigned long long>(min(static_cast<int64_t>(TJ), n - j0));
        if (full) atomicAdd(counters, outs);
        atomicAdd(counters + 1, outs * static_cast<unsigned long long>(wend - wbeg));
    }
}

template <int R, int NT, int TW, int SUB>
int launch_screen_cfg(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                      const double* ktab, int64_t ktab_stride, const int64_t* first, const double* tv,
                      int64_t tv_stride, const double* umax, unsigned long long* counters, cudaStream_t s) {
    constexpr int TJ = NT * R;
    constexpr int L = TJ + TW;
    const size_t smem = (padded<R>(L) + 1 + TW) * sizeof(double);  // fp64 phase; the fp32 screen uses half
    auto kern = screen_kernel<R, NT, TW, SUB>;
    if (first_time(ctx, reinterpret_cast<const void*>(kern)))
        LOB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(smem)));
    const int64_t tiles = (n + TJ - 1) / TJ;
    const int64_t blocks = tiles * lines;
    if (blocks > 0x7fffffffll) return set_error(ctx, LOB_INVALID_INPUT, "direct: grid too large");
    kern<<<static_cast<unsigned>(blocks), NT, smem, s>>>(u, out, n, tiles, ktab, ktab_stride, first, tv,
                                                          tv_stride, umax, counters);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "screen_kernel launch");
}

}  // namespace

int launch_direct_screen_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                             const double* ktab, int64_t ktab_stride, const int64_t* first,
                             const double* tv, int64_t tv_stride, unsigned long long* counters,
                             cudaStream_t s) {
    if (lines > ctx->direct_umax_cap) {
        if (ctx->direct_umax) LOB_CUDA_TRY(ctx, cudaFree(ctx->direct_umax));
        ctx->direct_umax = nullptr;
        LOB_CUDA_TRY(ctx, cudaMalloc(&ctx->direct_umax, lines * sizeof(double)));
        ctx->direct_umax_cap = lines;
    }
    if (lines > 0x7fffffffll) return set_error(ctx, LOB_INVALID_INPUT, "direct: too many lines");
    line_absmax_kernel<<<static_cast<unsigned>(lines), 256, 0, s>>>(u, n, ctx->direct_umax);
    ctx->launches += 1;
    const double* um = ctx->direct_umax;
    if (n >= 2048)
        return launch_screen_cfg<16, 128, 1024, 64>(ctx, u, out, lines, n, ktab, ktab_stride, first, tv,
                                                    tv_stride, um, counters, s);
    if (n >= 512)
        return launch_screen_cfg<8, 64, 512, 64>(ctx, u, out, lines, n, ktab, ktab_stride, first, tv,
                                                 tv_stride, um, counters, s);
    return launch_screen_cfg<4, 32, 128, 32>(ctx, u, out, lines, n, ktab, ktab_stride, first, tv, tv_stride,
                                             um, counters, s);
}

int launch_direct_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                      const double* ktab, int64_t ktab_stride, const int64_t* first,
                      const double* tv, int64_t tv_stride, cudaStream_t s) {
    if (ctx->direct_mode == LOB_DIRECT_PLAIN)
        return launch_direct_plain_f64(ctx, u, out, lines, n, ktab, ktab_stride, first, tv, tv_stride, s);
    if (!ctx->direct_full) {
        LOB_CUDA_TRY(ctx, cudaMalloc(&ctx->direct_full, 2 * sizeof(unsigned long long)));
        LOB_CUDA_TRY(ctx, cudaMemset(ctx->direct_full, 0, 2 * sizeof(unsigned long long)));
    }
    return launch_direct_screen_f64(ctx, u, out, lines, n, ktab, ktab_stride, first, tv, tv_stride,
                                    ctx->direct_full, s);
}

}  // namespace lob

// Shared pieces of the K1 kernels (csrc/direct.cu, csrc/direct_screen.cu):
// exact-rounding adds, the exact min, and the register-blocked sweep of a
// displacement range [wbeg, wend) for a tile of NT*R outputs of one line.
#pragma once
#include "lob_internal.cuh"

namespace lob {
namespace k1 {

template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) {
    return __dadd_rn(a, b);
}
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) {
    return __fadd_rn(a, b);
}

template <typename T>
__device__ __forceinline__ T min_exact(T best, T c) {
    return c < best ? c : best;  // std::min(best, c)
}
template <>
__device__ __forceinline__ float min_exact<float>(float best, float c) {
    return fminf(best, c);  // FMNMX; equal to the ternary for non-NaN c
}

template <typename T>
__device__ __forceinline__ T pos_inf();
template <>
__device__ __forceinline__ double pos_inf<double>() {
    return __longlong_as_double(0x7ff0000000000000ll);
}
template <>
__device__ __forceinline__ float pos_inf<float>() {
    return __int_as_float(0x7f800000);
}

template <int R>
__host__ __device__ __forceinline__ constexpr int padded(int i) {
    return i + i / R;
}

// best[r] = min(best[r], min_{w in [wbeg, wend)} U(j0 + t*R + r - first - w) + K[w])
// for the calling thread's R outputs.  Each chunk of TW displacements stages
// its source range (TJ + TW values, padded one slot per R so the stride-R
// per-thread reads are bank-conflict free) and its K values in shared memory;
// consecutive displacements shift the R sources by one, so a 2R register
// window slides with one LDS per displacement and K is a broadcast: per
// candidate exactly one add and one exact min.  Us: padded<R>(TJ+TW)+1, Ks: TW.
template <typename T, int R, int NT, int TW>
__device__ __forceinline__ void sweep_range(T* Us, T* Ks, const T* __restrict__ ul, const T* __restrict__ Kl,
                                            int64_t n, int64_t j0, int64_t first, int64_t wbeg, int64_t wend,
                                            T (&best)[R]) {
    constexpr int TJ = NT * R;
    constexpr int L = TJ + TW;
    const int t = threadIdx.x;
    for (int64_t wc = wbeg; wc < wend; wc += TW) {
        __syncthreads();
        // sources y = j - first - w for j in [j0, j0+TJ), w in [wc, wc+TW):
        // y in [ylo, ylo + L) with ylo = j0 - first - wc - TW
        const int64_t ylo = j0 - first - wc - TW;
        int64_t ym = ylo % n;
        if (ym < 0) ym += n;
        for (int i = t; i < L; i += NT) {
            int64_t y = ym + i;
            y -= (y / n) * n;
            Us[padded<R>(i)] = ul[y];
        }
        for (int s = t; s < TW; s += NT) {
            const int64_t w = wc + s;
            Ks[s] = w < wend ? Kl[w] : pos_inf<T>();
        }
        __syncthreads();

        // logical index of U(jt - first - wc) is i0 = t*R + TW (a multiple of R):
        // padded(i0 + k) = pa + k and padded(i0 - 1 - k) = pa - 2 - k, pa = padded(i0)
        const T* pa = Us + padded<R>(t * R + TW);
        T A[R];
#pragma unroll
        for (int k = 0; k < R; ++k) A[k] = pa[k];
        // the last chunk stops at the range's end (rounded up to R)
        const int send = static_cast<int>(min(static_cast<int64_t>(TW), (wend - wc + R - 1) / R * R));
#pragma unroll 1
        for (int s0 = 0; s0 < send; s0 += R) {
            T B[R];
#pragma unroll
            for (int k = 0; k < R; ++k) B[k] = pa[-2 - k];
            if constexpr (sizeof(T) == 4) {
                // fp32: two displacements per exact min, fminf(best, fminf(c0, c1)) -> one 3-input
                // FMNMX3 per two candidates (the min is order-free; NaN-free operands)
#pragma unroll
                for (int s = 0; s < R; s += 2) {
                    const T kw0 = Ks[s0 + s], kw1 = Ks[s0 + s + 1];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int i0 = r - s, i1 = r - s - 1;
                        const T v0 = i0 >= 0 ? A[i0 >= 0 ? i0 : 0] : B[i0 < 0 ? -i0 - 1 : 0];
                        const T v1 = i1 >= 0 ? A[i1 >= 0 ? i1 : 0] : B[i1 < 0 ? -i1 - 1 : 0];
                        best[r] = fminf(best[r], fminf(add_rn<T>(v0, kw0), add_rn<T>(v1, kw1)));
                    }
                }
            } else {
#pragma unroll
                for (int s = 0; s < R; ++s) {
                    const T kw = Ks[s0 + s];
#pragma unroll
                    for (int r = 0; r < R; ++r) {
                        const int idx = r - s;
                        const T val = idx >= 0 ? A[idx >= 0 ? idx : 0] : B[idx < 0 ? -idx - 1 : 0];
                        best[r] = min_exact<T>(best[r], add_rn<T>(val, kw));
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) A[k] = B[R - 1 - k];
            pa -= R + 1;
        }
    }
}

}  // namespace k1
}  // namespace lob

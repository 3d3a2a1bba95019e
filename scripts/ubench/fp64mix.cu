// Micro-benchmark of instruction mixes for the min-plus candidate on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int A = 16;
template <int MODE>
__global__ void __launch_bounds__(256) k(double* sink, int iters, double seed) {
    double best[A], val[A];
    float bf[A];
    int pred = 0;
#pragma unroll
    for (int r = 0; r < A; ++r) { best[r] = 1e300; val[r] = seed * (threadIdx.x + r + 1); bf[r] = 1e30f; }
    double kk = seed;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < A; ++r) {
            if (MODE == 0) { const double c = __dadd_rn(val[r], kk); best[r] = c < best[r] ? c : best[r]; }
            if (MODE == 1) { best[r] = __dadd_rn(best[r], kk); }
            if (MODE == 2) { pred += (val[r] < kk); }                     // DSETP only
            if (MODE == 3) { const double c = __dadd_rn(val[r], kk); pred += c < best[r]; }  // DADD+DSETP
            if (MODE == 4) { // DSETP + select of 64 bits via integer ops
                const double c = __dadd_rn(val[r], kk);
                const unsigned long long cb = __double_as_longlong(c), bb = __double_as_longlong(best[r]);
                best[r] = __longlong_as_double(c < best[r] ? cb : bb);
            }
            if (MODE == 5) { // min via fmin (DMNMX if available)
                best[r] = fmin(best[r], __dadd_rn(val[r], kk));
            }
            if (MODE == 6) { // fp32 candidate: FADD + FMNMX
                bf[r] = fminf(bf[r], __fadd_rn((float)val[r], (float)kk));
            }
        }
        kk = __dadd_rn(kk, 1e-300);
    }
    double acc = pred;
#pragma unroll
    for (int r = 0; r < A; ++r) acc += best[r] + bf[r];
    if (acc == 12345.678) sink[threadIdx.x] = acc;
}
template <int MODE>
void run(const char* name) {
    double* s; cudaMalloc(&s, 2048);
    int blocks = 148 * 8, iters = 20000;
    k<MODE><<<blocks, 256>>>(s, iters, 1.0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) k<MODE><<<blocks, 256>>>(s, iters, 1.0);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = 5.0 * blocks * 256.0 * iters * A;
    printf("%-28s %8.3f T elem/s\n", name, ops / (ms * 1e-3) / 1e12);
    cudaFree(s);
}
int main() {
    run<0>("DADD+DSETP+2FSEL (minplus)");
    run<1>("DADD chain");
    run<2>("DSETP only");
    run<3>("DADD+DSETP");
    run<4>("DADD+DSETP+int select");
    run<5>("DADD+fmin");
    run<6>("fp32 FADD+FMNMX");
    return 0;
}

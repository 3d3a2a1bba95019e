// FP64-pipe micro-benchmarks used as the measured roofline denominator for
// the direct kernel (MEASURED_PEAKS.json has no FP64 entry).
//   mix  : the exact per-candidate SASS of K1 (DADD + DSETP + 2 FSEL) on
//          independent register accumulators -> candidates/s
//   dadd : independent DADD chains -> FP64 lane-ops/s
#include <vector>

#include "lob_internal.cuh"

namespace lob {
namespace {

constexpr int kAcc = 16;

__global__ void __launch_bounds__(256) mix_kernel(double* sink, int iters, double seed) {
    double best[kAcc];
    double val[kAcc];
#pragma unroll
    for (int r = 0; r < kAcc; ++r) {
        best[r] = 1e300;
        val[r] = seed * (threadIdx.x + r + 1);
    }
    double k = seed;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < kAcc; ++r) {
            const double c = __dadd_rn(val[r], k);
            best[r] = c < best[r] ? c : best[r];
        }
        k = __dadd_rn(k, 1e-300);
    }
    double acc = 0;
#pragma unroll
    for (int r = 0; r < kAcc; ++r) acc += best[r];
    if (acc == 12345.678) sink[threadIdx.x] = acc;
}

__global__ void __launch_bounds__(256) dadd_kernel(double* sink, int iters, double seed) {
    double a[kAcc];
#pragma unroll
    for (int r = 0; r < kAcc; ++r) a[r] = seed * (threadIdx.x + r + 1);
    const double d = seed * 1e-20;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int r = 0; r < kAcc; ++r) a[r] = __dadd_rn(a[r], d);
    }
    double acc = 0;
#pragma unroll
    for (int r = 0; r < kAcc; ++r) acc += a[r];
    if (acc == 12345.678) sink[threadIdx.x] = acc;
}

__global__ void clock_kernel(long long* out, int spin) {
    long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
    out[0] = clock64() - t0;
}

}  // namespace
}  // namespace lob

extern "C" int lob_bench_fp64(lob_ctx* ctx, double* cand_per_s, double* dadd_per_s,
                              double* sm_ghz) {
    using namespace lob;
    LOB_CUDA_TRY(ctx, cudaSetDevice(ctx->device));
    double* sink = nullptr;
    long long* clk = nullptr;
    LOB_CUDA_TRY(ctx, cudaMalloc(&sink, 256 * sizeof(double)));
    LOB_CUDA_TRY(ctx, cudaMalloc(&clk, sizeof(long long)));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = ctx->sm_count * 8;
    const int iters = 20000;
    float ms = 0;
    // warm-up (clocks ramp)
    mix_kernel<<<blocks, 256>>>(sink, iters, 1.0);
    dadd_kernel<<<blocks, 256>>>(sink, iters, 1.0);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) mix_kernel<<<blocks, 256>>>(sink, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double cands = 5.0 * blocks * 256.0 * iters * kAcc;
    if (cand_per_s) *cand_per_s = cands / (ms * 1e-3);
    cudaEventRecord(e0);
    for (int rep = 0; rep < 5; ++rep) dadd_kernel<<<blocks, 256>>>(sink, iters, 1.0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double adds = 5.0 * blocks * 256.0 * iters * kAcc;
    if (dadd_per_s) *dadd_per_s = adds / (ms * 1e-3);
    // SM clock estimate: clock64 cycles over event time of a 1-CTA spin
    const long long spin = 200000000ll;
    cudaEventRecord(e0);
    clock_kernel<<<1, 1>>>(clk, static_cast<int>(spin > 2000000000ll ? 2000000000ll : spin));
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    long long cyc = 0;
    cudaMemcpy(&cyc, clk, sizeof(cyc), cudaMemcpyDeviceToHost);
    if (sm_ghz) *sm_ghz = static_cast<double>(cyc) / (ms * 1e-3) / 1e9;
    ctx->launches += 13;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(sink);
    cudaFree(clk);
    return cuda_status(ctx, cudaGetLastError(), "lob_bench_fp64");
}

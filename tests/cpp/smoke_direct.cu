// Standalone C-ABI smoke driver (no Python, no torch).
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../include/laxol_b200.h"
int main() {
    lob_ctx* ctx = nullptr;
    int st = lob_ctx_create(0, &ctx);
    printf("ctx %d\n", st); fflush(stdout);
    const int n = 24, lines = 2;
    std::vector<double> w(2 * n + 1), u(lines * n), o(lines * n);
    int64_t first, arg; double delta;
    st = lob_kernel_mech_host(ctx, n, 0.25, 0.0, w.data(), &first, &arg, &delta);
    printf("kernel %d first %lld\n", st, (long long)first); fflush(stdout);
    for (int i = 0; i < lines * n; ++i) u[i] = (i * 37 % 11) * 0.1;
    double *du, *dout, *dk; int64_t* df;
    printf("malloc...\n"); fflush(stdout);
    cudaError_t e0 = cudaMalloc(&du, u.size() * 8); printf("m1 %d\n", (int)e0); fflush(stdout);
    cudaMalloc(&dout, u.size() * 8); cudaMalloc(&dk, w.size() * 8); cudaMalloc(&df, lines * 8);
    printf("malloc ok\n"); fflush(stdout);
    cudaMemcpy(du, u.data(), u.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, w.data(), w.size() * 8, cudaMemcpyHostToDevice);
    std::vector<int64_t> f(lines, first);
    cudaMemcpy(df, f.data(), lines * 8, cudaMemcpyHostToDevice);
    printf("calling direct\n"); fflush(stdout);
    st = lob_minplus_direct_f64(ctx, du, dout, lines, n, dk, 0, df, nullptr, 0, nullptr);
    printf("direct %d %s\n", st, lob_last_error(ctx)); fflush(stdout);
    cudaError_t e = cudaDeviceSynchronize();
    printf("sync %s\n", cudaGetErrorString(e)); fflush(stdout);
    cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
    printf("out0 %.17g\n", o[0]);
    return 0;
}

// Weak-KAM consumers of the step, on the device:
//  * tropical (min-plus) matrix product C = A (x) B, fp64 — minplus_product
//    (proj/src/weakkam.cpp:130-146) and minplus_apply (:148-158) are both
//    this product (apply = a 1 x n or lines x n left operand);
//  * build_period_matrix (proj/src/weakkam.cpp:88-128): the l one-step cost
//    matrices step_i[y][x] = kin((x - y) mod n) - tau*V(t_i', x_j), chained
//    by the product;
//  * eigenvalue_karp (proj/src/weakkam.cpp:160-189): n min-plus vector x
//    matrix products D[k] = D[k-1] (x) C, then the min over v of the max
//    over k of (D[n][v] - D[k][v]) / (n - k).
//
// Exactness: every output is one minimum over single IEEE sums a + b, taken
// in increasing contraction index with a strict "<" (the reference's
// std::min(acc, a + b) loop order), so the result is the same double —
// including which of +0 / -0 survives a tie and that NaN candidates (inf +
// -inf) are ignored.  Split contraction ranges are combined left to right
// with the same strict "<", which preserves "first minimum wins".
//
// Roofline: the FP64 pipe, like K1 (DADD + DSETP + 2 FSEL per candidate; the
// candidate ceiling measured by lob_bench_fp64).
#include <cooperative_groups.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "lob_internal.cuh"

namespace cg = cooperative_groups;

namespace lob {
namespace {

#ifndef LOB_GEMM_BK
#define LOB_GEMM_BK 16
#endif
#ifndef LOB_GEMM_CTAS_PER_SM
#define LOB_GEMM_CTAS_PER_SM 4
#endif
constexpr int kBM = 64, kBN = 64, kBK = LOB_GEMM_BK;  // CTA tile of C and the contraction chunk
constexpr int kTT = 4;                       // outputs per thread per dimension
constexpr int kTX = kBN / kTT, kTY = kBM / kTT;
constexpr int kGT = kTX * kTY;               // 256 threads

__device__ __forceinline__ double pmin(double best, double c) { return c < best ? c : best; }

// C[m x n] = A[m x k] (x) B[k x n] over the contraction slice z in [z_begin, z_end) of
// blockIdx.z (row-major, leading dimensions); the slice's partial minima go to
// C + blockIdx.z * slice_stride.  Thread (tx, ty) owns rows ty + 16 i and columns
// tx + 16 j (i, j < 4): per contraction index 4 + 4 shared loads feed 16 candidates.
__global__ void __launch_bounds__(kGT) tropical_gemm_kernel(const double* __restrict__ A, int64_t lda,
                                                            const double* __restrict__ B, int64_t ldb,
                                                            double* __restrict__ C, int64_t ldc, int64_t m,
                                                            int64_t n, int64_t k, int64_t kslice,
                                                            int64_t slice_stride) {
    __shared__ double As[kBK][kBM + 1];  // transposed: As[z][r]
    __shared__ double Bs[kBK][kBN];
    const int tid = threadIdx.x, tx = tid % kTX, ty = tid / kTX;
    const int64_t r0 = static_cast<int64_t>(blockIdx.y) * kBM, c0 = static_cast<int64_t>(blockIdx.x) * kBN;
    const int64_t zb = static_cast<int64_t>(blockIdx.z) * kslice, ze = min(k, zb + kslice);
    double acc[kTT][kTT];
#pragma unroll
    for (int i = 0; i < kTT; ++i)
#pragma unroll
        for (int j = 0; j < kTT; ++j) acc[i][j] = INFINITY;
    for (int64_t z0 = zb; z0 < ze; z0 += kBK) {
        // out-of-range operands are +inf: inf + x is inf or NaN, never "<" a best
        for (int e = tid; e < kBM * kBK; e += kGT) {
            const int r = e / kBK, z = e % kBK;  // consecutive threads: consecutive z (coalesced)
            const int64_t gr = r0 + r, gz = z0 + z;
            As[z][r] = (gr < m && gz < ze) ? __ldg(A + gr * lda + gz) : INFINITY;
        }
        for (int e = tid; e < kBK * kBN; e += kGT) {
            const int z = e / kBN, c = e % kBN;
            const int64_t gz = z0 + z, gc = c0 + c;
            Bs[z][c] = (gz < ze && gc < n) ? __ldg(B + gz * ldb + gc) : INFINITY;
        }
        __syncthreads();
#pragma unroll 4
        for (int z = 0; z < kBK; ++z) {
            double a[kTT], b[kTT];
#pragma unroll
            for (int i = 0; i < kTT; ++i) a[i] = As[z][ty + kTY * i];
#pragma unroll
            for (int j = 0; j < kTT; ++j) b[j] = Bs[z][tx + kTX * j];
#pragma unroll
            for (int i = 0; i < kTT; ++i)
#pragma unroll
                for (int j = 0; j < kTT; ++j) acc[i][j] = pmin(acc[i][j], __dadd_rn(a[i], b[j]));
        }
        __syncthreads();
    }
    double* Cs = C + blockIdx.z * slice_stride;
#pragma unroll
    for (int i = 0; i < kTT; ++i)
#pragma unroll
        for (int j = 0; j < kTT; ++j) {
            const int64_t gr = r0 + ty + kTY * i, gc = c0 + tx + kTX * j;
            if (gr < m && gc < n) Cs[gr * ldc + gc] = acc[i][j];
        }
}

// split contraction: C = ordered min over the slices (slice order = contraction
// order, strict "<": the first minimum wins exactly as in one sequential loop)
__global__ void tropical_combine_kernel(const double* __restrict__ P, int slices, int64_t m, int64_t n,
                                        double* __restrict__ C, int64_t ldc) {
    const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= m * n) return;
    double best = P[e];
    for (int s = 1; s < slices; ++s) best = pmin(best, P[s * m * n + e]);
    C[(e / n) * ldc + e % n] = best;
}

// out[x] = min_y v[y] + M[y][x] (n x n): 32 columns per CTA, 8 warps each
// taking a contiguous eighth of y, partials combined in y order.
constexpr int kVW = 8;
__global__ void __launch_bounds__(32 * kVW) tropical_gemv_kernel(const double* __restrict__ v,
                                                                 const double* __restrict__ M, int64_t n,
                                                                 double* __restrict__ out) {
    __shared__ double part[kVW][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t x = static_cast<int64_t>(blockIdx.x) * 32 + lane;
    const int64_t per = (n + kVW - 1) / kVW;
    const int64_t y0 = w * per, y1 = min(n, y0 + per);
    double best = INFINITY;
    if (x < n)
        for (int64_t y = y0; y < y1; ++y) best = pmin(best, __dadd_rn(__ldg(v + y), __ldg(M + y * n + x)));
    part[w][lane] = best;
    __syncthreads();
    if (w == 0 && x < n) {
        double b = part[0][lane];
#pragma unroll
        for (int q = 1; q < kVW; ++q) b = pmin(b, part[q][lane]);
        out[x] = b;
    }
}

// Karp's n sequential vector x matrix products in ONE launch: a 16-CTA thread-block
// cluster keeps C resident in shared memory (CTA c holds columns [32c, 32c + 32),
// n <= 512 -> <= 128 KB), computes its 32 entries of D[k] (8 warps over contiguous
// row ranges, combined in row order), broadcasts them into every peer's next-row
// buffer through distributed shared memory and meets the others at the hardware
// cluster barrier; rows of D go to global memory for the final reduction.
constexpr int kKC = 16;   // CTAs per cluster (non-portable size, B200 allows 16)
constexpr int kKW = 32;   // columns per CTA
constexpr int kKNmax = kKC * kKW;
constexpr int kKWarps = 8;  // row ranges per step; each warp splits its range in kKAcc contiguous parts
constexpr int kKAcc = 2;
constexpr int kKParts = kKWarps * kKAcc;
__global__ void __launch_bounds__(32 * kKWarps, 1) karp_cluster_kernel(const double* __restrict__ M, int n,
                                                                       double* __restrict__ D) {
    extern __shared__ __align__(16) double ksm[];
    double* Cs = ksm;                      // [n][kKW] column block of C
    double* Db = Cs + n * kKW;             // [2][kKNmax] current / next row of D
    double* part = Db + 2 * kKNmax;        // [kKParts][kKW]
    cg::cluster_group cluster = cg::this_cluster();
    const int c = static_cast<int>(cluster.block_rank());
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int x = c * kKW + lane;
    for (int e = threadIdx.x; e < n * kKW; e += blockDim.x) {
        const int y = e / kKW, cc = c * kKW + e % kKW;
        Cs[e] = cc < n ? M[static_cast<int64_t>(y) * n + cc] : INFINITY;
    }
    for (int e = threadIdx.x; e < n; e += blockDim.x) Db[e] = e == 0 ? 0.0 : INFINITY;  // D[0]
    if (c == 0)
        for (int e = threadIdx.x; e < n; e += blockDim.x) D[e] = e == 0 ? 0.0 : INFINITY;
    cluster.sync();
    // part q = kKAcc * w + a covers rows [q * per, (q + 1) * per): independent min chains,
    // combined in row order (first minimum wins, as in one sequential loop)
    const int per = (n + kKParts - 1) / kKParts;
    for (int k = 1; k <= n; ++k) {
        const double* cur = Db + ((k - 1) & 1) * kKNmax;
        double best[kKAcc];
#pragma unroll
        for (int a = 0; a < kKAcc; ++a) best[a] = INFINITY;
        for (int t = 0; t < per; ++t) {
#pragma unroll
            for (int a = 0; a < kKAcc; ++a) {
                const int y = (kKAcc * w + a) * per + t;
                if (y < n) best[a] = pmin(best[a], __dadd_rn(cur[y], Cs[y * kKW + lane]));
            }
        }
#pragma unroll
        for (int a = 0; a < kKAcc; ++a) part[(kKAcc * w + a) * kKW + lane] = best[a];
        __syncthreads();
        if (w == 0) {
            double b = part[lane];
            for (int q = 1; q < kKParts; ++q) b = pmin(b, part[q * kKW + lane]);
            if (x < n) {
                D[static_cast<int64_t>(k) * n + x] = b;
                // broadcast into every CTA's next row (distributed shared memory)
                double* nxt = Db + (k & 1) * kKNmax;
                for (int r = 0; r < kKC; ++r) *cluster.map_shared_rank(nxt + x, r) = b;
            }
        }
        cluster.sync();
    }
}

__global__ void karp_init_kernel(double* D0, int64_t n) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) D0[i] = i == 0 ? 0.0 : INFINITY;
}

__global__ void nonfinite_kernel(const double* __restrict__ a, int64_t count, int* __restrict__ flag) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        if (!isfinite(a[i])) atomicOr(flag, 1);
}

// proj/src/weakkam.cpp:177-188, one thread per vertex v then an ordered min
__global__ void karp_final_kernel(const double* __restrict__ D, int64_t n, double* __restrict__ worst_v,
                                  double* __restrict__ out) {
    const double* Dn = D + n * n;
    for (int64_t v = threadIdx.x; v < n; v += blockDim.x) {
        double worst = -INFINITY;
        const double dn = Dn[v];
        if (dn != INFINITY) {
            for (int64_t k = 0; k < n; ++k) {
                const double dk = D[k * n + v];
                if (dk == INFINITY) continue;
                const double q = __ddiv_rn(__dsub_rn(dn, dk), static_cast<double>(n - k));
                worst = worst < q ? q : worst;  // std::max(worst, q)
            }
        }
        worst_v[v] = (dn != INFINITY && worst > -INFINITY) ? worst : NAN;  // NaN = skipped
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double best = INFINITY;
        for (int64_t v = 0; v < n; ++v) {
            const double w = worst_v[v];
            if (w == w) best = w < best ? w : best;  // std::min(best, worst)
        }
        *out = best;
    }
}

// step_i[y][x] = kinc[(x - y) mod n] - tv[x]  (proj/src/weakkam.cpp:105-122)
__global__ void period_step_kernel(const double* __restrict__ kinc, const double* __restrict__ tv, int64_t n,
                                   double* __restrict__ S) {
    const int64_t x = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t y = blockIdx.y;
    if (x >= n) return;
    int64_t r = x - y;
    if (r < 0) r += n;
    const double kin = kinc[r];
    S[y * n + x] = tv ? __dsub_rn(kin, tv[x]) : kin;
}

}  // namespace

int launch_tropical_gemm(lob_ctx* ctx, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t m, int64_t n, int64_t k, cudaStream_t s) {
    if (m == 0 || n == 0) return LOB_OK;
    const int64_t gx = (n + kBN - 1) / kBN, gy = (m + kBM - 1) / kBM;
    if (gx > 0x7fffffffll || gy > 65535) return set_error(ctx, LOB_INVALID_INPUT, "minplus_gemm: too large");
    // split the contraction when the output tiles alone cannot fill ~4 CTAs per SM
    // (keeping >= 4 chunks per slice); partial minima are combined in slice order
    const int64_t tiles = gx * gy, chunks = (k + kBK - 1) / kBK;
    int64_t slices = std::min<int64_t>((LOB_GEMM_CTAS_PER_SM * ctx->sm_count + tiles - 1) / tiles,
                                       std::max<int64_t>(1, chunks / 4));
    slices = std::max<int64_t>(1, std::min<int64_t>(slices, 64));
    const int64_t kslice = ((chunks + slices - 1) / slices) * kBK;
    slices = k > 0 ? (k + kslice - 1) / kslice : 1;
    const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy), static_cast<unsigned>(slices));
    if (slices == 1) {
        tropical_gemm_kernel<<<grid, kGT, 0, s>>>(A, lda, B, ldb, C, ldc, m, n, k, k > 0 ? k : 1, 0);
        ctx->launches += 1;
        return cuda_status(ctx, cudaGetLastError(), "minplus_gemm");
    }
    double* P = nullptr;
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&P, static_cast<size_t>(slices) * m * n * sizeof(double), s));
    tropical_gemm_kernel<<<grid, kGT, 0, s>>>(A, lda, B, ldb, P, n, m, n, k, kslice, m * n);
    tropical_combine_kernel<<<static_cast<unsigned>((m * n + 255) / 256), 256, 0, s>>>(P, static_cast<int>(slices),
                                                                                       m, n, C, ldc);
    ctx->launches += 2;
    cudaFreeAsync(P, s);
    return cuda_status(ctx, cudaGetLastError(), "minplus_gemm");
}

int launch_karp(lob_ctx* ctx, const double* M, int64_t n, double* D, double* lambda_dev, int* flag,
                cudaStream_t s) {
    const unsigned g = static_cast<unsigned>(std::min<int64_t>((n * n + 255) / 256, 4096));
    nonfinite_kernel<<<g, 256, 0, s>>>(M, n * n, flag);
    ctx->launches += 1;
    bool clustered = false;
    if (n <= kKNmax) {
        const size_t smem = (static_cast<size_t>(n) * kKW + 2 * kKNmax + kKParts * kKW) * sizeof(double);
        if (first_time(ctx, reinterpret_cast<const void*>(&karp_cluster_kernel))) {
            cudaFuncSetAttribute(karp_cluster_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaFuncSetAttribute(karp_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>((static_cast<size_t>(kKNmax) * kKW + 2 * kKNmax + kKParts * kKW) *
                                                  sizeof(double)));
        }
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(kKC);
        cfg.blockDim = dim3(32 * kKWarps);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = kKC;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int clusters = 0;
        if (cudaOccupancyMaxActiveClusters(&clusters, karp_cluster_kernel, &cfg) == cudaSuccess && clusters > 0) {
            LOB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, karp_cluster_kernel, M, static_cast<int>(n), D));
            ctx->launches += 1;
            clustered = true;
        } else {
            cudaGetLastError();  // cluster launch unavailable: the launch loop below
        }
    }
    if (!clustered) {
        karp_init_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(D, n);
        ctx->launches += 1;
        const unsigned gv = static_cast<unsigned>((n + 31) / 32);
        for (int64_t k = 1; k <= n; ++k) {
            tropical_gemv_kernel<<<gv, 32 * kVW, 0, s>>>(D + (k - 1) * n, M, n, D + k * n);
            ctx->launches += 1;
        }
    }
    // worst_v scratch: after the (n+1) x n table
    karp_final_kernel<<<1, 512, 0, s>>>(D, n, D + (n + 1) * n, lambda_dev);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "eigenvalue_karp");
}

int launch_period_matrix(lob_ctx* ctx, const double* kinc, const double* tvs, int64_t n, int64_t ell, double* C,
                         double* scratch, cudaStream_t s) {
    if (n > 65535) return set_error(ctx, LOB_INVALID_INPUT, "period_matrix: n too large");
    double* S = scratch;          // step_i
    double* T = scratch + n * n;  // ping-pong product
    const dim3 gs(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>(n));
    // C = step_0 (x) step_1 (x) ... in the reference's order, C = (i == 0) ? step : C (x) step
    double* cur = ell % 2 == 1 ? C : T;  // the last product lands in C
    double* nxt = ell % 2 == 1 ? T : C;
    period_step_kernel<<<gs, 128, 0, s>>>(kinc, tvs, n, cur);
    ctx->launches += 1;
    for (int64_t i = 1; i < ell; ++i) {
        period_step_kernel<<<gs, 128, 0, s>>>(kinc, tvs ? tvs + i * n : nullptr, n, S);
        ctx->launches += 1;
        const int st = launch_tropical_gemm(ctx, cur, n, S, n, nxt, n, n, n, n, s);
        if (st) return st;
        std::swap(cur, nxt);
    }
    return cuda_status(ctx, cudaGetLastError(), "build_period_matrix");
}

}  // namespace lob

// ---------------------------------------------------------------------------
// C-ABI (include/laxol_b200.h, "weak-KAM consumers")
namespace {

using namespace lob;

// proj/src/weakkam.cpp:17-23
int steps_per_period(lob_ctx* ctx, double tau, const char* who, int64_t* ell) {
    const int64_t l = std::llround(1.0 / tau);
    if (!(tau > 0.0) || l < 1 || std::abs(static_cast<double>(l) * tau - 1.0) > 1e-9)
        return set_error(ctx, LOB_INVALID_INPUT, std::string(who) + ": tau must be a unit fraction of the time period");
    *ell = l;
    return LOB_OK;
}

// Device-resident whole periods of the fully discrete step for one line, with
// the in-period time labels of apply_one_period (proj/src/weakkam.cpp:33-39):
// step i of a period uses tv table i (tv_count == ell), the one table
// (tv_count == 1) or none (tv_count == 0).  The state after each period is
// copied to the host, where the estimators do the reference's arithmetic.
struct PeriodRunner {
    lob_ctx* ctx;
    int64_t n, ell, tv_count;
    double drift, tau;
    int engine;
    cudaStream_t s = nullptr;
    double *du = nullptr, *dscr = nullptr, *dtv = nullptr, *ddrift = nullptr, *ktab = nullptr;
    int64_t* dfirst = nullptr;
    void* ws = nullptr;
    size_t wsb = 0;
    int64_t steps_done = 0;
    bool resident = false;  // a whole period in one K2R launch (short lines)
    void* lcb = nullptr;
    int* halt = nullptr;

    int init(const double* u0, const double* tvs) {
        s = ctx->stream;
        if (engine != LOB_ENGINE_DIRECT && engine != LOB_ENGINE_FAST)
            return set_error(ctx, LOB_INVALID_INPUT, "weak-KAM: unknown engine");
        const int64_t W = 2 * n + 1;
        std::vector<double> hk(static_cast<size_t>(W));
        int64_t first = 0, arg = 0;
        double dl = 0;
        // build_kernel's checks (proj/src/scheme.cpp:59-105) for both engines
        if (lob_kernel_mech_host(ctx, n, tau, drift, hk.data(), &first, &arg, &dl))
            return set_error(ctx, LOB_INVALID_INPUT, "weak-KAM: invalid scheme parameters");
        LOB_CUDA_TRY(ctx, cudaMalloc(&du, n * sizeof(double)));
        LOB_CUDA_TRY(ctx, cudaMalloc(&dscr, n * sizeof(double)));
        LOB_CUDA_TRY(ctx, cudaMalloc(&ddrift, sizeof(double)));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(du, u0, n * sizeof(double), cudaMemcpyHostToDevice, s));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(ddrift, &drift, sizeof(double), cudaMemcpyHostToDevice, s));
        if (tv_count > 0) {
            LOB_CUDA_TRY(ctx, cudaMalloc(&dtv, tv_count * n * sizeof(double)));
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(dtv, tvs, tv_count * n * sizeof(double), cudaMemcpyHostToDevice, s));
        }
        if (engine == LOB_ENGINE_DIRECT) {
            LOB_CUDA_TRY(ctx, cudaMalloc(&ktab, W * sizeof(double)));
            LOB_CUDA_TRY(ctx, cudaMalloc(&dfirst, sizeof(int64_t)));
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(ktab, hk.data(), W * sizeof(double), cudaMemcpyHostToDevice, s));
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(dfirst, &first, sizeof(int64_t), cudaMemcpyHostToDevice, s));
        } else {
            wsb = fast_workspace_bytes(1, n);
            LOB_CUDA_TRY(ctx, cudaMalloc(&ws, wsb));
            resident = ctx->resident && fast_resident_ok(n);
            if (resident) {
                LOB_CUDA_TRY(ctx, cudaMalloc(&lcb, 64));
                LOB_CUDA_TRY(ctx, cudaMalloc(&halt, sizeof(int)));
            }
        }
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        return LOB_OK;
    }
    // one whole period on the device; the state is copied to host[n]
    int period(double* host) {
        if (resident) {
            const int big = 0x7fffffff;
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(halt, &big, sizeof(int), cudaMemcpyHostToDevice, s));
            const int st = launch_fast_resident_f64(ctx, du, 1, n, ddrift, tau, tv_count ? dtv : nullptr, 0, 0.0, ell,
                                                    nullptr, nullptr, halt, lcb, s,
                                                    static_cast<int>(tv_count > 1 ? tv_count : 1), n);
            if (st) return st;
            steps_done += ell;
        }
        for (int64_t i = 0; i < (resident ? 0 : ell); ++i) {
            const double* tv = tv_count == 0 ? nullptr : dtv + (tv_count == 1 ? 0 : i) * n;
            int st;
            if (engine == LOB_ENGINE_DIRECT)
                st = launch_direct_f64(ctx, du, dscr, 1, n, ktab, 0, dfirst, tv, 0, s);
            else
                st = launch_fast_f64(ctx, du, dscr, 1, n, ddrift, tau, tv, 0, 0.0, nullptr, ws, wsb,
                                     steps_done == 0 ? 0 : LOB_FAST_STATS_VALID, s);
            if (st) return st;
            std::swap(du, dscr);
            ++steps_done;
        }
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(host, du, n * sizeof(double), cudaMemcpyDeviceToHost, s));
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        for (int64_t j = 0; j < n; ++j)
            if (!std::isfinite(host[j]))
                return set_error(ctx, LOB_EVALUATION_ERROR, "weak-KAM: non-finite value after a period");
        return LOB_OK;
    }
    ~PeriodRunner() {
        for (void* p : {static_cast<void*>(du), static_cast<void*>(dscr), static_cast<void*>(dtv),
                        static_cast<void*>(ddrift), static_cast<void*>(ktab), static_cast<void*>(dfirst), ws, lcb,
                        static_cast<void*>(halt)})
            if (p) cudaFree(p);
    }
};

int check_tv_count(lob_ctx* ctx, int64_t tv_count, int64_t ell, const double* tvs) {
    if (tv_count < 0 || (tv_count > 1 && tv_count != ell) || (tv_count > 0 && !tvs))
        return set_error(ctx, LOB_INVALID_INPUT, "weak-KAM: tv_count must be 0, 1 or the steps per period");
    return LOB_OK;
}

}  // namespace

extern "C" {

int lob_minplus_gemm_f64(lob_ctx* ctx, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, int64_t m, int64_t n, int64_t k, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (m < 0 || n < 0 || k < 0 || lda < k || ldb < n || ldc < n)
        return set_error(ctx, LOB_INVALID_INPUT, "minplus_gemm: bad shape or leading dimension");
    return launch_tropical_gemm(ctx, A, lda, B, ldb, C, ldc, m, n, k, static_cast<cudaStream_t>(stream));
}

int lob_period_kinetic_host(const double* window, int64_t first, int64_t n, double* kinc) {
    if (!window || !kinc || n < 1) return LOB_INVALID_INPUT;
    // proj/src/weakkam.cpp:106-118: kin(d0) = min over d = d0 + k n in [first, first + 2n]
    // of window[d - first], in increasing d; it depends on d0 mod n only
    const int64_t last = first + 2 * n;
    for (int64_t r = 0; r < n; ++r) {
        int64_t d = r + floordiv(first - r, n) * n;  // largest d = r (mod n) with d <= first
        if (d < first) d += n;
        double kin = INFINITY;
        for (; d <= last; d += n) {
            const double w = window[d - first];
            kin = w < kin ? w : kin;
        }
        kinc[r] = kin;
    }
    return LOB_OK;
}

int lob_period_matrix_f64(lob_ctx* ctx, const double* kinc, const double* tvs, int64_t n, int64_t ell,
                          double* C, double* scratch, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (n < 1 || ell < 1) return set_error(ctx, LOB_INVALID_INPUT, "build_period_matrix: n, ell must be >= 1");
    return launch_period_matrix(ctx, kinc, tvs, n, ell, C, scratch, static_cast<cudaStream_t>(stream));
}

int lob_eigenvalue_karp_f64(lob_ctx* ctx, const double* M, int64_t n, double* lambda, void* stream) {
    if (!ctx || !lambda) return LOB_INVALID_INPUT;
    if (n < 1) return set_error(ctx, LOB_INVALID_INPUT, "eigenvalue_karp: empty matrix");
    cudaStream_t s = static_cast<cudaStream_t>(stream);  // ordered after the producer of M
    double* D = nullptr;
    int* flag = nullptr;
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&D, ((n + 2) * n + 1) * sizeof(double), s));
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&flag, sizeof(int), s));
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(flag, 0, sizeof(int), s));
    double* lam = D + (n + 2) * n;
    const int st = launch_karp(ctx, M, n, D, lam, flag, s);
    int hflag = 0;
    if (st == LOB_OK) {
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(lambda, lam, sizeof(double), cudaMemcpyDeviceToHost, s));
    }
    cudaFreeAsync(D, s);
    cudaFreeAsync(flag, s);
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (st) return st;
    if (hflag) return set_error(ctx, LOB_INVALID_INPUT, "eigenvalue_karp: non-finite entry");
    return LOB_OK;
}

int lob_hbar_drift_host_f64(lob_ctx* ctx, const double* u0, int64_t n, double drift, double tau,
                            const double* tvs, int64_t tv_count, int engine, int max_periods, double tol,
                            double* h_bar, double* residual, int64_t* n_steps, int* converged,
                            double* u_final) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (!u0 || n < 1) return set_error(ctx, LOB_INVALID_INPUT, "estimate_hbar_drift: empty u");
    int64_t ell = 0;
    int st = steps_per_period(ctx, tau, "estimate_hbar_drift", &ell);
    if (st) return st;
    if (max_periods < 1) return set_error(ctx, LOB_INVALID_INPUT, "estimate_hbar_drift: max_periods must be >= 1");
    if ((st = check_tv_count(ctx, tv_count, ell, tvs))) return st;
    PeriodRunner pr{ctx, n, ell, tv_count, drift, tau, engine};
    if ((st = pr.init(u0, tvs))) return st;
    // proj/src/weakkam.cpp:54-85: the increments' statistics on the host, in the
    // reference's order (sequential mean, max-norms)
    std::vector<double> u(u0, u0 + n), next(static_cast<size_t>(n)), delta(static_cast<size_t>(n), 0.0), prev;
    double hb = 0.0, res = 0.0;
    int64_t steps = 0;
    int conv = 0;
    for (int p = 0; p < max_periods; ++p) {
        if ((st = pr.period(next.data()))) return st;
        steps += ell;
        for (int64_t j = 0; j < n; ++j) delta[j] = next[j] - u[j];
        u.swap(next);
        double mean = 0.0;
        for (int64_t j = 0; j < n; ++j) mean += delta[j];
        mean /= static_cast<double>(n);
        hb = mean;
        double r = 0.0;
        for (int64_t j = 0; j < n; ++j) r = std::max(r, std::abs(delta[j] - mean));
        res = r;
        if (!prev.empty()) {
            double change = 0.0;
            for (int64_t j = 0; j < n; ++j) change = std::max(change, std::abs(delta[j] - prev[j]));
            if (change < tol) {
                conv = 1;
                break;
            }
        }
        prev = delta;
    }
    if (h_bar) *h_bar = hb;
    if (residual) *residual = res;
    if (n_steps) *n_steps = steps;
    if (converged) *converged = conv;
    if (u_final) std::copy(u.begin(), u.end(), u_final);
    return LOB_OK;
}

int lob_fixed_point_residual_host_f64(lob_ctx* ctx, const double* u, int64_t n, double h_bar, double drift,
                                      double tau, const double* tvs, int64_t tv_count, int engine,
                                      double* residual) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (!u || n < 1) return set_error(ctx, LOB_INVALID_INPUT, "fixed_point_residual: empty u");
    int64_t ell = 0;
    int st = steps_per_period(ctx, tau, "fixed_point_residual", &ell);
    if (st) return st;
    if ((st = check_tv_count(ctx, tv_count, ell, tvs))) return st;
    PeriodRunner pr{ctx, n, ell, tv_count, drift, tau, engine};
    if ((st = pr.init(u, tvs))) return st;
    std::vector<double> v(static_cast<size_t>(n));
    if ((st = pr.period(v.data()))) return st;
    // proj/src/weakkam.cpp:197-200
    double res = 0.0;
    for (int64_t j = 0; j < n; ++j) res = std::max(res, std::abs(v[j] - u[j] - h_bar));
    if (residual) *residual = res;
    return LOB_OK;
}

}  // extern "C"

// K3 — 2-D dimension splitting (proj/src/splitting.cpp:37-99, Remark 2.8)
// on a periodic n x n row-major tensor:
//   axis 0 (columns, kernel 1) -> axis 1 (rows, kernel 2) -> out -= tau*V.
// The reference gathers each strided column into a temporary line and
// scatters it back (proj/src/splitting.cpp:67-76).  Here a tiled transpose
// (64x64 tiles through shared memory, 16-byte global accesses on both sides
// for even n; 32x32 scalar tiles otherwise) turns columns into rows so both
// sweeps run the batched line kernels; the potential pass evaluates the separable descriptor
// V = a1[i]*a2[k] + b with the C++ expression's roundings and applies
// out = out - tau*V (two roundings, no FMA; proj/src/splitting.cpp:95).
// Also: the per-step drift / finiteness check of evolve
// (proj/src/scheme.cpp:244-264).
#include <algorithm>
#include <cstdint>

#include "lob_internal.cuh"

namespace lob {
namespace {

constexpr int kTD = 32;  // transpose tile

__global__ void __launch_bounds__(256) transpose_kernel(const double* __restrict__ src,
                                                        double* __restrict__ dst, int64_t n) {
    __shared__ double tile[kTD][kTD + 1];
    const int64_t bx = static_cast<int64_t>(blockIdx.x) * kTD;  // column block of src
    const int64_t by = static_cast<int64_t>(blockIdx.y) * kTD;  // row block of src
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;     // 32 x 8
    for (int r = ty; r < kTD; r += 8) {
        const int64_t i = by + r, k = bx + tx;
        if (i < n && k < n) tile[r][tx] = src[i * n + k];
    }
    __syncthreads();
    for (int r = ty; r < kTD; r += 8) {
        const int64_t k = bx + r, i = by + tx;  // dst[k][i] = src[i][k]
        if (i < n && k < n) dst[k * n + i] = tile[tx][r];
    }
}

// 64 x 64 tiles, 256 threads, double2 loads and stores (even n, 16-byte aligned rows); the
// tile pitch of 65 doubles keeps the column reads at two wavefronts per half warp.  Launched
// with programmatic dependent launch: the previous kernel's tail overlaps this prologue.
constexpr int kTV = 64;
#ifndef LOB_TRANSPOSE_ROWS
#define LOB_TRANSPOSE_ROWS 32
#endif
// tiles of kTR rows x 64 columns: a 2048^2 transpose is 4096 CTAs (16.6 KB of shared memory
// each, 8 per SM), so the last wave is nearly full
constexpr int kTR = LOB_TRANSPOSE_ROWS;
static_assert(kTR >= 4 && kTR <= 64 && 64 % kTR == 0, "rows per transpose tile");
__global__ void __launch_bounds__(256) transpose64_kernel(const double* __restrict__ src,
                                                          double* __restrict__ dst, int64_t n) {
    __shared__ double tile[kTR][kTV + 1];
    const int64_t bx = static_cast<int64_t>(blockIdx.x) * kTV;  // column block of src
    const int64_t by = static_cast<int64_t>(blockIdx.y) * kTR;  // row block of src
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t k = bx + 2 * lane;
#pragma unroll
    for (int r = w; r < kTR; r += 8) {
        const int64_t i = by + r;
        double2 v = make_double2(0.0, 0.0);
        if (i < n && k < n) v = *reinterpret_cast<const double2*>(src + i * n + k);
        tile[r][2 * lane] = v.x;
        tile[r][2 * lane + 1] = v.y;
    }
    __syncthreads();
    // each destination row (a source column) holds kTR values = kTR / 2 double2: a warp writes
    // 64 / kTR rows per pass
    constexpr int kHalf = kTR / 2, kRowsPerWarp = 32 / kHalf;
    const int sub = lane / kHalf, e = lane % kHalf;
    const int64_t i = by + 2 * e;
#pragma unroll
    for (int c0 = w * kRowsPerWarp; c0 < kTV; c0 += 8 * kRowsPerWarp) {
        const int c = c0 + sub;
        const int64_t kk = bx + c;  // dst[kk][i] = src[i][kk]
        if (kk < n && i < n)
            *reinterpret_cast<double2*>(dst + kk * n + i) = make_double2(tile[2 * e][c], tile[2 * e + 1][c]);
    }
}

// The multi-GPU split step's exchange as one kernel over NVLink peer memory (no NCCL, no pack /
// unpack passes): rank `rank` holds the row slab x = X[rank*b .. rank*b + b) (b x n) and writes
// X^T's blocks straight into every peer's receive slab, R_q[c][rank*b + i] = X[rank*b + i][q*b + c]
// (R_q = rank q's b x n slab of X^T).  64 x 64 tiles through shared memory: each tile lands in one
// peer (b % 64 == 0) as 64 row segments of 512 contiguous bytes.  Peer slabs: device addresses
// valid on this device (CUDA symmetric memory / IPC); the caller synchronises the ranks after it.
constexpr int kMaxPeers = 16;
struct PeerSlabs {
    double* p[kMaxPeers];
};
__global__ void __launch_bounds__(256) slab_push_kernel(const double* __restrict__ x, int64_t b, int64_t n,
                                                        int rank, PeerSlabs peers) {
    __shared__ double tile[kTV][kTV + 1];
    const int64_t bx = static_cast<int64_t>(blockIdx.x) * kTV;  // column block of x (global column)
    const int64_t by = static_cast<int64_t>(blockIdx.y) * kTV;  // row block of x (local row)
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int64_t k = bx + 2 * lane;
#pragma unroll
    for (int r = w; r < kTV; r += 8) {
        const int64_t i = by + r;
        const double2 v = *reinterpret_cast<const double2*>(x + i * n + k);
        tile[r][2 * lane] = v.x;
        tile[r][2 * lane + 1] = v.y;
    }
    __syncthreads();
    const int q = static_cast<int>(bx / b);  // the peer owning these 64 columns
    double* dst = peers.p[q];
    const int64_t col0 = static_cast<int64_t>(rank) * b + by;  // destination column of local row by
#pragma unroll
    for (int c = w; c < kTV; c += 8) {
        const int64_t crow = bx + c - static_cast<int64_t>(q) * b;  // destination row in peer q's slab
        *reinterpret_cast<double2*>(dst + crow * n + col0 + 2 * lane) =
            make_double2(tile[2 * lane][c], tile[2 * lane + 1][c]);
    }
}

// rows x n block (rows = n for the whole tensor; a row slab of it for the multi-GPU step)
__global__ void __launch_bounds__(256) potential2d_kernel(double* __restrict__ out,
                                                          const double* __restrict__ a1,
                                                          const double* __restrict__ a2, double b,
                                                          double tau, int64_t n, int64_t rows) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= rows * n) return;
    const int64_t i = idx / n, k = idx - i * n;
    // V = a1*a2 + b; out -= tau*V   (no contraction)
    const double v = __dadd_rn(__dmul_rn(a1[i], a2[k]), b);
    out[idx] = __dsub_rn(out[idx], __dmul_rn(tau, v));
}

__global__ void __launch_bounds__(256) drift_kernel(const double* __restrict__ nxt,
                                                    const double* __restrict__ cur, int64_t n,
                                                    double* __restrict__ drift_out,
                                                    int* __restrict__ halt, int step) {
    __shared__ double sh[8];
    __shared__ int bad;
    const int64_t line = blockIdx.x;
    if (threadIdx.x == 0) bad = 0;
    __syncthreads();
    double acc = 0.0;
    int nonfinite = 0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
        const double a = nxt[line * n + j];
        acc += a - cur[line * n + j];
        nonfinite |= !isfinite(a);
    }
    if (nonfinite) bad = 1;
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += sh[w];
        if (drift_out) drift_out[line] = s / static_cast<double>(n);
        if (bad && halt) atomicMin(halt, step);
    }
}

// dst[a][b][l] = src[a][l][b] for a < A, l < L, b < B (32x32 tiles of the (L, B) planes)
__global__ void __launch_bounds__(256) transpose_batched_kernel(const double* __restrict__ src,
                                                                double* __restrict__ dst, int64_t A, int64_t L,
                                                                int64_t B) {
    __shared__ double tile[kTD][kTD + 1];
    const int64_t b0 = static_cast<int64_t>(blockIdx.x) * kTD;  // column block (b)
    const int64_t l0 = static_cast<int64_t>(blockIdx.y) * kTD;  // row block (l)
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    for (int64_t a = blockIdx.z; a < A; a += gridDim.z) {
        const double* sa = src + a * L * B;
        double* da = dst + a * L * B;
        for (int r = ty; r < kTD; r += 8) {
            const int64_t l = l0 + r, b = b0 + tx;
            if (l < L && b < B) tile[r][tx] = sa[l * B + b];
        }
        __syncthreads();
        for (int r = ty; r < kTD; r += 8) {
            const int64_t b = b0 + r, l = l0 + tx;
            if (l < L && b < B) da[b * L + l] = tile[tx][r];
        }
        __syncthreads();
    }
}

// the multi-GPU exchange's receive side: y[c][p*b + i] = recv[p][c][i] (world blocks of b x b)
__global__ void slab_unpack_kernel(const double* __restrict__ recv, double* __restrict__ y, int64_t b, int64_t world) {
    const int64_t n = b * world;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < b * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t c = e / n, r = e - c * n, p = r / b, i = r - p * b;
        y[e] = recv[(p * b + c) * b + i];
    }
}

// out[i] -= tv[i] (tau*V of every grid point, rounded on the host): one IEEE subtraction
__global__ void sub_table_kernel(double* __restrict__ out, const double* __restrict__ tv, int64_t count) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        out[i] = __dsub_rn(out[i], tv[i]);
}

}  // namespace

int launch_transpose_batched(lob_ctx* ctx, const double* src, double* dst, int64_t A, int64_t L, int64_t B,
                             cudaStream_t s) {
    const dim3 grid(static_cast<unsigned>((B + kTD - 1) / kTD), static_cast<unsigned>((L + kTD - 1) / kTD),
                    static_cast<unsigned>(std::min<int64_t>(A, 65535)));
    transpose_batched_kernel<<<grid, 256, 0, s>>>(src, dst, A, L, B);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "transpose_batched_kernel");
}

int launch_slab_unpack(lob_ctx* ctx, const double* recv, double* y, int64_t b, int64_t world, cudaStream_t s) {
    const unsigned g = static_cast<unsigned>(std::min<int64_t>((b * b * world + 255) / 256, 148 * 32));
    slab_unpack_kernel<<<g, 256, 0, s>>>(recv, y, b, world);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "slab_unpack_kernel");
}

int launch_slab_push(lob_ctx* ctx, const double* x, int64_t b, int64_t world, int rank, double* const* peer_slabs,
                     cudaStream_t s) {
    if (world < 1 || world > kMaxPeers || rank < 0 || rank >= world || b < 1 || b % kTV != 0)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_slab_push_f64: 1 <= world <= 16, 0 <= rank < world, b % 64 == 0");
    if (reinterpret_cast<uintptr_t>(x) % 16 != 0) return set_error(ctx, LOB_INVALID_INPUT, "lob_slab_push_f64: x alignment");
    PeerSlabs ps{};
    for (int q = 0; q < world; ++q) {
        if (!peer_slabs[q] || reinterpret_cast<uintptr_t>(peer_slabs[q]) % 16 != 0)
            return set_error(ctx, LOB_INVALID_INPUT, "lob_slab_push_f64: peer slab missing or misaligned");
        ps.p[q] = peer_slabs[q];
    }
    const int64_t n = b * world;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(n / kTV), static_cast<unsigned>(b / kTV));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LOB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, slab_push_kernel, x, b, n, rank, ps));
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "slab_push_kernel");
}

int launch_sub_table(lob_ctx* ctx, double* out, const double* tv, int64_t count, cudaStream_t s) {
    const unsigned g = static_cast<unsigned>(std::min<int64_t>((count + 255) / 256, 148 * 32));
    sub_table_kernel<<<g, 256, 0, s>>>(out, tv, count);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "sub_table_kernel");
}

int launch_transpose(lob_ctx* ctx, const double* src, double* dst, int64_t n, cudaStream_t s) {
    if (n % 2 == 0 && reinterpret_cast<uintptr_t>(src) % 16 == 0 && reinterpret_cast<uintptr_t>(dst) % 16 == 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>((n + kTV - 1) / kTV), static_cast<unsigned>((n + kTR - 1) / kTR));
        cfg.blockDim = dim3(256);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        LOB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, transpose64_kernel, src, dst, n));
        ctx->launches += 1;
        return cuda_status(ctx, cudaGetLastError(), "transpose64_kernel");
    }
    dim3 grid(static_cast<unsigned>((n + kTD - 1) / kTD), static_cast<unsigned>((n + kTD - 1) / kTD));
    transpose_kernel<<<grid, 256, 0, s>>>(src, dst, n);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "transpose_kernel");
}

int launch_potential2d(lob_ctx* ctx, double* out, const double* a1, const double* a2, double b,
                       double tau, int64_t n, cudaStream_t s, int64_t rows) {
    if (rows < 0) rows = n;
    const int64_t total = rows * n;
    if (total == 0) return LOB_OK;
    potential2d_kernel<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(out, a1, a2, b,
                                                                                  tau, n, rows);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "potential2d_kernel");
}

int launch_drift(lob_ctx* ctx, const double* nxt, const double* cur, int64_t lines, int64_t n,
                 double* drift_out, int* halt, int step, cudaStream_t s) {
    drift_kernel<<<static_cast<unsigned>(lines), 256, 0, s>>>(nxt, cur, n, drift_out, halt, step);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "drift_kernel");
}

}  // namespace lob

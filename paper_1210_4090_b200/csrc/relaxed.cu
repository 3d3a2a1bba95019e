// The reference's fast engine with its relaxation tolerance eta > 0
// (SURVEY.md §8 row f4): conv_fast (proj/src/minplus.cpp:217-252) —
// decompose(u, eta) into eta-relaxed convex / concave blocks
// (:152-188), blocks capped at 48 samples (capped_blocks, :195-215), the
// slope merge (merge_convolve, :40-57) or envelope (envelope_convolve,
// :62-105) of every block with the whole kernel window, min_pointwise of the
// parts (:254-276) — then kinetic_convolve's periodic aliasing
// (proj/src/scheme.cpp:125-134) and the potential subtraction
// (proj/src/scheme.cpp:156-162).  For eta > 0 the merge misorders slopes, so
// the result is the reference's APPROXIMATION (an upper bound of the exact
// minimum); this engine reproduces those doubles bit for bit.  (For eta == 0
// it is exact and equals K1/K2; the exact engines are the fast path.)
//
// Device formulation.  Both walks are closed forms of running extrema of
// binary searches over the kernel's nondecreasing slopes fs:
//  * merge: at g-index j the f pointer stops at I_j = max(I_{j-1}, lb_j),
//    lb_j = #{fs < gs[j]} (lower bound); position k belongs to the unique j
//    with I_{j-1} + j <= k <= I_j + j (I_{-1} = 0, I_m = n) and
//    part(k) = fv[k - j] + gv[j];
//  * envelope: phase 1 writes k <= P0 = #{fs <= gs[0]} with gv[0]; the
//    pointer then follows i_j = min(i_{j-1}, ub_j), ub_j = #{fs <= gs[j]},
//    writing (i_j + j, gv[j]) and (i_j + j + 1, gv[j + 1]); the tail writes
//    positions i + m, i in (i_{m-1}, n], with gv[m].
// Every part value is one IEEE sum fv + gv and the combines are exact minima
// (no -0 or NaN can arise from finite u and a table with K >= +0 at its
// minimum), so any order of the minima gives the reference's double.
// Blocks longer than 48 (only at eta == 0, where capped_blocks keeps them)
// are split into 48-sample pieces for the device walk — exact at eta == 0,
// and the block count reported is the reference's (capped for eta > 0,
// uncapped for eta == 0).
//
// Work is O(pieces x n) like the reference's conv_fast (every piece is
// merged with the whole window): a parity engine, not a fast path.
#include <algorithm>
#include <climits>
#include <cmath>
#include <string>
#include <vector>

#include "lob_internal.cuh"

namespace lob {
namespace {

constexpr int kCap = 48;  // kRelaxedBlockCap, proj/src/minplus.cpp:198
constexpr int kNTs = 256;
constexpr unsigned long long kEmpty = ~0ull;  // above every dkey: "not written"

struct RelaxedWs {
    unsigned long long* conv;  // [lines][3n + 1] keys
    int2* pieces;              // [lines][n] (start, end | kind << 31)
    int* npieces;              // [lines]
    int* flag;                 // bit 0: gap (min_pointwise), bit 1: non-finite
    size_t total;
};

RelaxedWs relaxed_layout(void* base, int64_t lines, int64_t n) {
    RelaxedWs w{};
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += (bytes + 255) / 256 * 256;
        return o;
    };
    const size_t oc = take(static_cast<size_t>(lines) * (3 * n + 1) * 8);
    const size_t op = take(static_cast<size_t>(lines) * n * sizeof(int2));
    const size_t on = take(static_cast<size_t>(lines) * sizeof(int));
    const size_t of = take(sizeof(int));
    char* b = static_cast<char*>(base);
    w.conv = reinterpret_cast<unsigned long long*>(b + oc);
    w.pieces = reinterpret_cast<int2*>(b + op);
    w.npieces = reinterpret_cast<int*>(b + on);
    w.flag = reinterpret_cast<int*>(b + of);
    w.total = off;
    return w;
}

// decompose(u, eta) on the closed period (samples u[0..n-1], u[n] = u[0]),
// proj/src/minplus.cpp:152-188, one thread per line; blocks are emitted as
// pieces of at most kCap slopes.  blocks_out: capped count for eta > 0
// (capped_blocks), the decomposition's own count for eta == 0.
// n = slopes of the line: the period (periodic: samples u[0..n-1], u[n] = u[0]) or the
// samples - 1 of a plain sequence; cap = 48 (the relaxed walk's pieces) or INT_MAX (decompose).
__global__ void relaxed_decompose_kernel(const double* __restrict__ u, int64_t lines, int64_t n, double eta,
                                         int2* __restrict__ pieces, int* __restrict__ npieces,
                                         int64_t* __restrict__ blocks_out, int* __restrict__ flag,
                                         int periodic = 1, int64_t cap = kCap) {
    const int64_t line = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    const int64_t ls = periodic ? n : n + 1;  // samples stored per line
    const double* ul = u + line * ls;
    int2* pl = pieces + line * n;
    auto val = [&](int64_t i) { return ul[periodic && i == n ? 0 : i]; };
    auto slope = [&](int64_t i) { return __dsub_rn(val(i + 1), val(i)); };
    for (int64_t i = 0; i < ls; ++i)
        if (!isfinite(ul[i])) atomicOr(flag, 2);
    int np = 0;
    int64_t nb = 0;
    int64_t b = 0;
    while (b < n) {
        bool determined = false;
        int kind = 0;  // 0 convex, 1 concave
        int64_t e = b + 1;
        double sp = slope(b);
        while (e < n) {
            const double se = slope(e);
            const double inc = __dsub_rn(se, sp);
            if (!determined) {
                if (inc > eta) {
                    determined = true;
                    kind = 0;
                } else if (inc < -eta) {
                    determined = true;
                    kind = 1;
                }
            } else if (kind == 0) {
                if (!(inc >= -eta)) break;
            } else {
                if (!(inc <= eta)) break;
            }
            sp = se;
            ++e;
        }
        for (int64_t s = b; s < e; s += cap) {
            const unsigned endk = static_cast<unsigned>(min(e, s + cap)) | (static_cast<unsigned>(kind) << 31);
            pl[np++] = make_int2(static_cast<int>(s), static_cast<int>(endk));
            ++nb;
        }
        if (eta <= 0.0) nb -= (e - b + cap - 1) / cap - 1;  // eta == 0: blocks are not capped
        b = e;
    }
    npieces[line] = np;
    if (blocks_out) blocks_out[line] = nb;
}

// #{i < cnt : fs[i] < x} (STRICT) or #{fs[i] <= x}, fs nondecreasing,
// fs[i] = K[i+1] - K[i] (slopes(kernel.window), proj/src/grid_fn.cpp:38-44)
template <bool STRICT>
__device__ __forceinline__ int count_below(const double* __restrict__ K, int cnt, double x) {
    int lo = 0, hi = cnt;  // answer in [lo, hi]
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        const double f = __dsub_rn(__ldg(K + mid + 1), __ldg(K + mid));
        const bool below = STRICT ? (f < x) : (f <= x);
        if (below) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// One CTA per (line, piece-slot): merge / envelope of each piece with the
// window, scattered into the line's conv keys with exact global min.
// n: slopes of u (see the decompose kernel); nf: slopes of the kernel (2n for the step);
// conv rows hold nf + n + 1 keys.
__global__ void __launch_bounds__(kNTs) relaxed_scatter_kernel(const double* __restrict__ u, int64_t n,
                                                               const double* __restrict__ ktab,
                                                               int64_t ktab_stride, const int2* __restrict__ pieces,
                                                               const int* __restrict__ npieces,
                                                               unsigned long long* __restrict__ conv,
                                                               int periodic = 1, int64_t nf_arg = -1,
                                                               int64_t lines = 1) {
    __shared__ double gv[kCap + 1], gs[kCap];
    __shared__ int I[kCap + 1];  // merge: I_j; envelope: i_j (index 0 = P0)
    const int64_t line = grid_line();
    if (line >= lines) return;  // (uniform per CTA: before any barrier)
    const double* ul = u + line * (periodic ? n : n + 1);
    const double* K = ktab + line * ktab_stride;
    const int nf = static_cast<int>(nf_arg < 0 ? 2 * n : nf_arg);  // kernel slopes
    unsigned long long* cl = conv + line * (nf + n + 1);
    const int np = npieces[line];
    for (int p = blockIdx.x; p < np; p += gridDim.x) {
        const int2 pc = pieces[line * n + p];
        const int start = pc.x, end = pc.y & 0x7fffffff;
        const bool concave = pc.y < 0;
        const int m = end - start;
        for (int t = threadIdx.x; t <= m; t += kNTs) gv[t] = ul[periodic && start + t == n ? 0 : start + t];
        __syncthreads();
        for (int t = threadIdx.x; t < m; t += kNTs) {
            gs[t] = __dsub_rn(gv[t + 1], gv[t]);
            I[t] = concave ? count_below<false>(K, nf, gs[t]) : count_below<true>(K, nf, gs[t]);
        }
        __syncthreads();
        if (threadIdx.x == 0) {  // running max (merge) / min (envelope), m <= 48
            int r = I[0];
            for (int j = 1; j < m; ++j) {
                r = concave ? min(r, I[j]) : max(r, I[j]);
                I[j] = r;
            }
            I[m] = nf;  // merge: after the last g step f runs to n
        }
        __syncthreads();
        if (!concave) {
            // positions k in [0, nf + m]: j(k) = #{j < m : I_j + j < k}
            for (int k = threadIdx.x; k <= nf + m; k += kNTs) {
                int lo = 0, hi = m;
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (I[mid] + mid < k) lo = mid + 1;
                    else hi = mid;
                }
                const double v = __dadd_rn(__ldg(K + (k - lo)), gv[lo]);
                atomicMin(cl + start + k, dkey(v));
            }
        } else {
            const int p0 = I[0];
            // phase 1: k <= P0 with gv[0]
            for (int k = threadIdx.x; k <= p0; k += kNTs) atomicMin(cl + start + k, dkey(__dadd_rn(__ldg(K + k), gv[0])));
            // (P0 + 1, gv[1]) and the pointer walk j = 1 .. m-1
            if (threadIdx.x == 0) atomicMin(cl + start + p0 + 1, dkey(__dadd_rn(__ldg(K + p0), gv[1])));
            for (int j = 1 + static_cast<int>(threadIdx.x); j < m; j += kNTs) {
                const int i = I[j];
                const double fi = __ldg(K + i);
                atomicMin(cl + start + i + j, dkey(__dadd_rn(fi, gv[j])));
                atomicMin(cl + start + i + j + 1, dkey(__dadd_rn(fi, gv[j + 1])));
            }
            // tail: i in (i_{m-1}, nf], position i + m, gv[m]
            const int it = m >= 2 ? I[m - 1] : p0;
            for (int i = it + 1 + static_cast<int>(threadIdx.x); i <= nf; i += kNTs)
                atomicMin(cl + start + i + m, dkey(__dadd_rn(__ldg(K + i), gv[m])));
        }
        __syncthreads();
    }
}

// kinetic_convolve's aliasing (proj/src/scheme.cpp:125-134) + the potential
// (proj/src/scheme.cpp:156-162); every conv position must have been written
// (min_pointwise's gap check, proj/src/minplus.cpp:271-272).
__global__ void relaxed_finalize_kernel(const unsigned long long* __restrict__ conv, int64_t n,
                                        const int64_t* __restrict__ first_arr, const double* __restrict__ tv,
                                        int64_t tv_stride, double* __restrict__ out, int* __restrict__ flag,
                                        int64_t lines) {
    const int64_t line = grid_line();
    const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= n || line >= lines) return;
    const unsigned long long* cl = conv + line * (3 * n + 1);
    const int64_t shift = -first_arr[line];  // half - center_index
    int64_t i = (j + shift) % n;
    if (i < 0) i += n;
    double best = INFINITY;
    bool gap = false;
    for (; i <= 3 * n; i += n) {
        const unsigned long long k = cl[i];
        if (k == kEmpty) {
            gap = true;
            continue;
        }
        const double v = dkey_inv(k);
        best = v < best ? v : best;
    }
    if (gap) atomicOr(flag, 1);
    out[line * n + j] = tv ? __dsub_rn(best, tv[line * tv_stride + j]) : best;
}

// plain (non-periodic) conv_fast: out[k] = the pointwise min of the parts, every position written
// (min_pointwise's gap check, proj/src/minplus.cpp:271-272)
__global__ void plain_finalize_kernel(const unsigned long long* __restrict__ conv, int64_t len, double* __restrict__ out,
                                      int* __restrict__ flag) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < len;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long key = conv[k];
        if (key == kEmpty) atomicOr(flag, 1);
        out[k] = key == kEmpty ? INFINITY : dkey_inv(key);
    }
}

// conv_naive (proj/src/minplus.cpp:116-126): out[k] = min over i + j = k of f[i] + g[j], i ascending
__global__ void conv_naive_kernel(const double* __restrict__ f, int64_t nf, const double* __restrict__ g, int64_t ng,
                                  double* __restrict__ out) {
    for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < nf + ng - 1;
         k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        double best = INFINITY;
        const int64_t i0 = k - (ng - 1) > 0 ? k - (ng - 1) : 0, i1 = k < nf - 1 ? k : nf - 1;
        for (int64_t i = i0; i <= i1; ++i) {
            const double c = __dadd_rn(__ldg(f + i), __ldg(g + k - i));
            best = c < best ? c : best;  // std::min(out[k], a[i] + b[j])
        }
        out[k] = best;
    }
}

// is_convex (proj/src/grid_fn.cpp:44-54): the first segment whose slope drops, exact comparison
// of the two rounded differences; *bad = the smallest such index (LLONG_MAX when convex)
__global__ void convex_check_kernel(const double* __restrict__ f, int64_t nf, unsigned long long* __restrict__ bad) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i + 2 < nf;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double lo = __dsub_rn(f[i + 1], f[i]), hi = __dsub_rn(f[i + 2], f[i + 1]);
        if (hi < lo) atomicMin(bad, static_cast<unsigned long long>(i));
    }
}

}  // namespace

size_t relaxed_workspace_bytes(int64_t lines, int64_t n) { return relaxed_layout(nullptr, lines, n).total; }

int launch_relaxed_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n, const double* ktab,
                       int64_t ktab_stride, const int64_t* first, const double* tv, int64_t tv_stride, double eta,
                       int64_t* blocks, void* workspace, size_t ws_bytes, cudaStream_t s) {
    if (!(eta >= 0.0)) return set_error(ctx, LOB_INVALID_INPUT, "decompose: eta must be >= 0");
    if (n > (1ll << 29)) return set_error(ctx, LOB_INVALID_INPUT, "relaxed: n too large");
    const RelaxedWs w = relaxed_layout(workspace, lines, n);
    if (!workspace || ws_bytes < w.total) return set_error(ctx, LOB_INVALID_INPUT, "relaxed: workspace too small");
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(w.conv, 0xff, static_cast<size_t>(lines) * (3 * n + 1) * 8, s));
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(w.flag, 0, sizeof(int), s));
    relaxed_decompose_kernel<<<static_cast<unsigned>((lines + 63) / 64), 64, 0, s>>>(u, lines, n, eta, w.pieces,
                                                                                    w.npieces, blocks, w.flag);
    const unsigned gx = static_cast<unsigned>(std::min<int64_t>(n, std::max<int64_t>(1, 2 * ctx->sm_count)));
    relaxed_scatter_kernel<<<line_grid(gx, lines), kNTs, 0, s>>>(u, n, ktab, ktab_stride, w.pieces, w.npieces, w.conv, 1,
                                                                 -1, lines);
    relaxed_finalize_kernel<<<line_grid(static_cast<unsigned>((n + 255) / 256), lines), 256, 0, s>>>(
        w.conv, n, first, tv, tv_stride, out, w.flag, lines);
    ctx->launches += 3;
    LOB_CUDA_TRY(ctx, cudaGetLastError());
    int hflag = 0;
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hflag, w.flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (hflag & 2) return set_error(ctx, LOB_INVALID_INPUT, "relaxed: non-finite sample");
    if (hflag & 1) return set_error(ctx, LOB_INVALID_INPUT, "min_pointwise: index ranges leave a gap");
    return LOB_OK;
}

}  // namespace lob

using namespace lob;

extern "C" int lob_relaxed_workspace_bytes(int64_t lines, int64_t n, size_t* bytes) {
    if (!bytes || lines < 0 || n < 1) return LOB_INVALID_INPUT;
    *bytes = relaxed_workspace_bytes(lines, n);
    return LOB_OK;
}

extern "C" int lob_minplus_relaxed_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                                       const double* ktab, int64_t ktab_stride, const int64_t* first,
                                       const double* tv, int64_t tv_stride, double eta, int64_t* blocks,
                                       void* workspace, size_t workspace_bytes, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (lines < 0 || n < 1) return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_relaxed_f64: bad shape");
    if (lines == 0) return LOB_OK;
    return launch_relaxed_f64(ctx, u, out, lines, n, ktab, ktab_stride, first, tv, tv_stride, eta, blocks, workspace,
                              workspace_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" int lob_minplus_conv_naive_f64(lob_ctx* ctx, const double* f, int64_t nf, const double* g, int64_t ng,
                                          double* out, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (nf < 1 || ng < 1 || !f || !g || !out) return set_error(ctx, LOB_INVALID_INPUT, "conv_naive: empty input");
    const int64_t len = nf + ng - 1;
    conv_naive_kernel<<<static_cast<unsigned>(std::min<int64_t>((len + 127) / 128, 148 * 16)), 128, 0,
                        static_cast<cudaStream_t>(stream)>>>(f, nf, g, ng, out);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "conv_naive");
}

extern "C" int lob_decompose_f64(lob_ctx* ctx, const double* u, int64_t m, double eta, int* kinds, int64_t* starts,
                                 int64_t* ends, int64_t capacity, int64_t* count, void* stream) {
    if (!ctx || !count) return LOB_INVALID_INPUT;
    if (!(eta >= 0.0)) return set_error(ctx, LOB_INVALID_INPUT, "decompose: eta must be >= 0");
    if (m < 1 || !u) return set_error(ctx, LOB_INVALID_INPUT, "decompose: empty sample vector");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t ns = m - 1;  // slopes
    if (ns == 0) {  // proj/src/minplus.cpp:158-161
        *count = 1;
        if (capacity >= 1) {
            if (kinds) kinds[0] = 0;
            if (starts) starts[0] = 0;
            if (ends) ends[0] = 0;
        }
        return LOB_OK;
    }
    int2* pieces = nullptr;
    int *np = nullptr, *flag = nullptr;
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&pieces, static_cast<size_t>(ns) * sizeof(int2), s));
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&np, 2 * sizeof(int), s));
    flag = np + 1;
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(flag, 0, sizeof(int), s));
    relaxed_decompose_kernel<<<1, 1, 0, s>>>(u, 1, ns, eta, pieces, np, nullptr, flag, 0, ns + 1);  // uncapped
    ctx->launches += 1;
    int hn = 0, hf = 0;
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hn, np, sizeof(int), cudaMemcpyDeviceToHost, s));
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    std::vector<int2> hp(static_cast<size_t>(hn));
    if (hn) LOB_CUDA_TRY(ctx, cudaMemcpy(hp.data(), pieces, hn * sizeof(int2), cudaMemcpyDeviceToHost));
    cudaFree(pieces);
    cudaFree(np);
    *count = hn;
    for (int64_t i = 0; i < hn && i < capacity; ++i) {
        if (kinds) kinds[i] = hp[i].y < 0 ? 1 : 0;
        if (starts) starts[i] = hp[i].x;
        if (ends) ends[i] = hp[i].y & 0x7fffffff;
    }
    return LOB_OK;
}

extern "C" int lob_conv_fast_f64(lob_ctx* ctx, const double* kern, int64_t nk, const double* u, int64_t nu, double eta,
                                 double* out, int64_t* blocks, void* stream) {
    if (!ctx) return LOB_INVALID_INPUT;
    if (!(eta >= 0.0)) return set_error(ctx, LOB_INVALID_INPUT, "decompose: eta must be >= 0");
    if (nk < 1 || nu < 1 || !kern || !u || !out) return set_error(ctx, LOB_INVALID_INPUT, "conv_fast: empty input");
    if (nk + nu > (1ll << 30)) return set_error(ctx, LOB_INVALID_INPUT, "conv_fast: too long");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (nk >= 3) {
        // require_convex(kernel) of conv_fast(kernel, u, eta) (proj/src/minplus.cpp:24-29,190-194)
        unsigned long long* dbad = nullptr;
        unsigned long long hbad = ~0ull;
        LOB_CUDA_TRY(ctx, cudaMallocAsync(&dbad, sizeof(hbad), s));
        LOB_CUDA_TRY(ctx, cudaMemsetAsync(dbad, 0xff, sizeof(hbad), s));
        convex_check_kernel<<<static_cast<unsigned>(std::min<int64_t>((nk + 255) / 256, 148 * 8)), 256, 0, s>>>(kern, nk,
                                                                                                             dbad);
        ctx->launches += 1;
        LOB_CUDA_TRY(ctx, cudaGetLastError());
        LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hbad, dbad, sizeof(hbad), cudaMemcpyDeviceToHost, s));
        cudaFreeAsync(dbad, s);
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        if (hbad != ~0ull)
            return set_error(ctx, LOB_INVALID_INPUT,
                             "conv_fast: kernel is not convex, slope drops at segment " + std::to_string(hbad + 1));
    }
    if (nk == 1 || nu == 1) {
        // a one-sample side has no slopes: every block's merge / envelope walk degenerates to the
        // plain sums f[i] + g[j] (proj/src/minplus.cpp:40-57,62-105 with an empty slope list), the
        // reference's own exhaustive test includes these (proj/tests/unit_minplus.cpp:436-437);
        // the block count is decompose(u, eta)'s (one Convex block for a single sample, :157-160)
        int st = lob_minplus_conv_naive_f64(ctx, kern, nk, u, nu, out, stream);
        if (st) return st;
        int64_t hb = 1;
        if (nu >= 2) {
            const int64_t m = nu - 1;
            int2* pieces = nullptr;
            int* np = nullptr;
            int64_t* db = nullptr;
            LOB_CUDA_TRY(ctx, cudaMallocAsync(&pieces, static_cast<size_t>(m) * sizeof(int2), s));
            LOB_CUDA_TRY(ctx, cudaMallocAsync(&np, 2 * sizeof(int), s));
            LOB_CUDA_TRY(ctx, cudaMallocAsync(&db, sizeof(int64_t), s));
            LOB_CUDA_TRY(ctx, cudaMemsetAsync(np + 1, 0, sizeof(int), s));
            relaxed_decompose_kernel<<<1, 1, 0, s>>>(u, 1, m, eta, pieces, np, db, np + 1, 0, kCap);
            ctx->launches += 1;
            LOB_CUDA_TRY(ctx, cudaGetLastError());
            LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hb, db, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
            cudaFreeAsync(pieces, s);
            cudaFreeAsync(np, s);
            cudaFreeAsync(db, s);
        }
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        if (blocks) *blocks = hb;
        return LOB_OK;
    }
    const int64_t m = nu - 1, nf = nk - 1, len = nf + m + 1;
    unsigned long long* conv = nullptr;
    int2* pieces = nullptr;
    int *np = nullptr, *flag = nullptr;
    int64_t* db = nullptr;
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&conv, static_cast<size_t>(len) * 8, s));
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&pieces, static_cast<size_t>(m) * sizeof(int2), s));
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&np, 2 * sizeof(int), s));
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&db, sizeof(int64_t), s));
    flag = np + 1;
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(conv, 0xff, static_cast<size_t>(len) * 8, s));
    LOB_CUDA_TRY(ctx, cudaMemsetAsync(flag, 0, sizeof(int), s));
    relaxed_decompose_kernel<<<1, 1, 0, s>>>(u, 1, m, eta, pieces, np, db, flag, 0, kCap);
    const unsigned gx = static_cast<unsigned>(std::min<int64_t>(m, std::max<int64_t>(1, 2 * ctx->sm_count)));
    relaxed_scatter_kernel<<<dim3(gx, 1), kNTs, 0, s>>>(u, m, kern, 0, pieces, np, conv, 0, nf);
    plain_finalize_kernel<<<static_cast<unsigned>(std::min<int64_t>((len + 255) / 256, 148 * 8)), 256, 0, s>>>(
        conv, len, out, flag);
    ctx->launches += 3;
    int hf = 0;
    LOB_CUDA_TRY(ctx, cudaGetLastError());
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hf, flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    int64_t hb = 0;
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(&hb, db, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    cudaFreeAsync(conv, s);
    cudaFreeAsync(pieces, s);
    cudaFreeAsync(np, s);
    cudaFreeAsync(db, s);
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    if (blocks) *blocks = hb;
    if (hf & 2) return set_error(ctx, LOB_INVALID_INPUT, "conv_fast: non-finite sample");
    if (hf & 1) return set_error(ctx, LOB_INVALID_INPUT, "min_pointwise: index ranges leave a gap");
    return LOB_OK;
}

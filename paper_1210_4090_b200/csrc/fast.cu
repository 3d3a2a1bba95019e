// K2 — fast exact periodic min-plus step for mechanical kinetics, O(n) work.
//
// Replaces conv_fast (proj/src/minplus.cpp:219-252: decompose -> per-block
// merge/envelope over the whole kernel -> min_pointwise, O(c n)) with an
// exact local-minimum walk that needs O(n + TV(u')/a) candidates per line.
//
// For output j the reference computes min_y F_j(y), F_j(y) = U(y) + K(j-y),
// with U the periodic extension of u and K the convex window
// (proj/tests/unit_scheme.cpp:176-194).  Because fl() is monotone the
// minimum of the rounded sums is the rounded exact minimum, so it suffices
// to find an exact-real minimiser and add once.  A global minimiser is a
// local minimiser: with sigma(d) = K(d+1) - K(d) and s(y) = U(y+1) - U(y),
//     F_j(y) <= F_j(y-1)  <=>  s(y-1) <= sigma(d)
//     F_j(y) <= F_j(y+1)  <=>  sigma(d-1) <= s(y),        d = j - y.
// For K*(v) = v^2/2 - P v, sigma(d) = a (d + 1/2) - P eps with a = eps^2/tau,
// so source y can only win for d in [dL(y), dR(y)],
//     dL = ceil(z(s(y-1)) - 1/2 - delta),  dR = floor(z(s(y)) + 1/2 + delta),
//     z(s) = (s + P eps)/a,
// where delta bounds the table's rounding (csrc/host/kernel_build.cpp).
// Window-edge minima are excluded by checking osc(u) < K(edge) - K(min)
// (else the tile falls back to the direct scan).  The intervals of a
// locally convex run tile the outputs contiguously (the paper's convex
// merge, Lemma 4.1 / Algorithm 1); concave kinks leave empty intervals and
// fold the walk back (Algorithm 2's envelope), and the overlaps are resolved
// by an exact min.  Total candidates ~ n + TV+(s)/a per line.
//
// Layout: a CTA owns a tile of T outputs of one line.  Per-tile statistics
// of u (min/max of u and of its slopes, and the decomposition FSM summary)
// are produced by the previous step's epilogue (or by stats_kernel) and
// tell each CTA which source tiles can reach its outputs.  Candidates are
// combined with shared-memory atomicMin on order-preserving 64-bit keys.
// The epilogue applies out = best - tv (one rounding), writes u^{n+1}
// coalesced, and computes the statistics of u^{n+1} for the next step,
// including the block count of decompose() (proj/src/minplus.cpp:152-188)
// as a 3-state transition function per tile.
#include <cmath>
#include <cstring>

#include "lob_internal.cuh"

namespace lob {

constexpr int kTile = 2048;  // outputs (and sources) per tile
constexpr int kThreads = 512;
constexpr int kMaxSrcList = 2048;

// decompose() FSM: states U=0, Cx=1, Cc=2; summary for each entry state.
struct TileStats {
    double umin, umax, smin, smax;
    unsigned short cnt[3];
    unsigned char exit[3];
    unsigned char pad;
};
static_assert(sizeof(TileStats) == 48, "TileStats layout");

struct FastParams {
    int64_t n;
    int64_t tiles;
    int64_t T;
    double tau;
    double eta;
    const double* vtab;  // v_d for d in [-vofs, vofs]
    int64_t vofs;
};

namespace {

__device__ __forceinline__ double kval(const double* vtab, int64_t vofs, int64_t d, double drift,
                                       double tau) {
    const double v = vtab[d + vofs];
    // tau * ((0.5*v)*v - drift*v): proj/src/scheme.cpp:80 + hamiltonian.cpp:43
    return __dmul_rn(tau, __dsub_rn(__dmul_rn(__dmul_rn(0.5, v), v), __dmul_rn(drift, v)));
}

// FSM step for one increment (proj/src/minplus.cpp:161-187).
__device__ __forceinline__ int fsm_class(double inc, double eta) {
    if (inc > eta) return 0;     // pos
    if (inc < -eta) return 1;    // neg
    if (inc == inc) return 2;    // zero band
    return 3;                    // NaN
}
__device__ __forceinline__ void fsm_step(int& q, int& emits, int c) {
    if (q == 0) {
        q = c == 0 ? 1 : (c == 1 ? 2 : 0);
    } else if (q == 1) {
        if (c == 1 || c == 3) {
            q = 0;
            ++emits;
        }
    } else {
        if (c == 0 || c == 3) {
            q = 0;
            ++emits;
        }
    }
}

struct Fsm3 {
    int exit[3];
    int cnt[3];
};
__device__ __forceinline__ Fsm3 fsm_compose(const Fsm3& a, const Fsm3& b) {
    Fsm3 r;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int m = a.exit[q];
        r.exit[q] = b.exit[m];
        r.cnt[q] = a.cnt[q] + b.cnt[m];
    }
    return r;
}
__device__ __forceinline__ Fsm3 fsm_identity() {
    Fsm3 r;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        r.exit[q] = q;
        r.cnt[q] = 0;
    }
    return r;
}

// Block-wide ordered composition of per-thread FSM summaries.
__device__ Fsm3 block_fsm(Fsm3 f, Fsm3* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // inclusive ordered reduction within the warp (lane order preserved)
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        Fsm3 o;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            o.exit[q] = __shfl_down_sync(0xffffffffu, f.exit[q], off);
            o.cnt[q] = __shfl_down_sync(0xffffffffu, f.cnt[q], off);
        }
        if ((lane & (2 * off - 1)) == 0 && lane + off < 32) f = fsm_compose(f, o);
    }
    if (lane == 0) sh[warp] = f;
    __syncthreads();
    Fsm3 r = fsm_identity();
    if (threadIdx.x == 0) {
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) r = fsm_compose(r, sh[w]);
        sh[0] = r;
    }
    __syncthreads();
    r = sh[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ double warp_min(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fmin(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}
__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
    for (int o = 16; o; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    return x;
}

// Block reduce of (min, max, min, max) into sh4[0..3].
__device__ void block_minmax4(double a, double b, double c, double d, double* sh) {
    a = warp_min(a);
    b = warp_max(b);
    c = warp_min(c);
    d = warp_max(d);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) {
        sh[4 * warp + 0] = a;
        sh[4 * warp + 1] = b;
        sh[4 * warp + 2] = c;
        sh[4 * warp + 3] = d;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            sh[0] = fmin(sh[0], sh[4 * w + 0]);
            sh[1] = fmax(sh[1], sh[4 * w + 1]);
            sh[2] = fmin(sh[2], sh[4 * w + 2]);
            sh[3] = fmax(sh[3], sh[4 * w + 3]);
        }
    }
    __syncthreads();
}

// Statistics of a tile whose values are vals[0 .. Tl+1] (vals[i] = u(j0+i),
// periodic), shared by the stats kernel and the K2 epilogue.
__device__ void tile_stats(const double* vals, int Tl, int64_t j0, int64_t n, double eta,
                           TileStats* dst, double* shred, Fsm3* shfsm) {
    double umin = INFINITY, umax = -INFINITY, smin = INFINITY, smax = -INFINITY;
    for (int i = threadIdx.x; i < Tl; i += blockDim.x) {
        const double v = vals[i];
        const double s = __dsub_rn(vals[i + 1], v);
        umin = fmin(umin, v);
        umax = fmax(umax, v);
        smin = fmin(smin, s);
        smax = fmax(smax, s);
        if (!isfinite(v) || !isfinite(s)) {  // non-finite: the next step falls back
            umin = -INFINITY;
            umax = INFINITY;
        }
    }
    // increments e = j0+i, i in [1, Tl], e <= n-1, each thread a contiguous chunk
    const int per = (Tl + blockDim.x - 1) / blockDim.x;
    const int i_lo = 1 + threadIdx.x * per;
    const int i_hi = min(Tl, i_lo + per - 1);
    Fsm3 f;
    for (int q = 0; q < 3; ++q) {
        int st = q, em = 0;
        for (int i = i_lo; i <= i_hi; ++i) {
            if (j0 + i > n - 1) break;
            const double inc = __dsub_rn(__dsub_rn(vals[i + 1], vals[i]), __dsub_rn(vals[i], vals[i - 1]));
            fsm_step(st, em, fsm_class(inc, eta));
        }
        f.exit[q] = st;
        f.cnt[q] = em;
    }
    f = block_fsm(f, shfsm);
    block_minmax4(umin, umax, smin, smax, shred);
    if (threadIdx.x == 0) {
        TileStats ts;
        ts.umin = shred[0];
        ts.umax = shred[1];
        ts.smin = shred[2];
        ts.smax = shred[3];
        for (int q = 0; q < 3; ++q) {
            ts.cnt[q] = static_cast<unsigned short>(f.cnt[q]);
            ts.exit[q] = static_cast<unsigned char>(f.exit[q]);
        }
        ts.pad = 0;
        *dst = ts;
    }
}

__global__ void __launch_bounds__(kThreads) stats_kernel(const double* __restrict__ u,
                                                         TileStats* __restrict__ stats,
                                                         FastParams p) {
    __shared__ double vals[kTile + 2];
    __shared__ double shred[4 * (kThreads / 32)];
    __shared__ Fsm3 shfsm[kThreads / 32];
    const int64_t line = blockIdx.x / p.tiles;
    const int64_t tile = blockIdx.x - line * p.tiles;
    const int64_t j0 = tile * p.T;
    const int Tl = static_cast<int>(min(p.T, p.n - j0));
    const double* ul = u + line * p.n;
    for (int i = threadIdx.x; i < Tl + 2; i += blockDim.x) {
        int64_t j = j0 + i;
        if (j >= p.n) j -= p.n;
        if (j >= p.n) j -= p.n;
        vals[i] = ul[j];
    }
    __syncthreads();
    tile_stats(vals, Tl, j0, p.n, p.eta, stats + blockIdx.x, shred, shfsm);
}

__global__ void build_vtab_kernel(double* vtab, int64_t vofs, double eps, double tau) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > 2 * vofs) return;
    const int64_t d = i - vofs;
    // x = (double)d * eps; v = x / tau  (proj/src/scheme.cpp:79-80)
    vtab[i] = __ddiv_rn(__dmul_rn(static_cast<double>(d), eps), tau);
}

__global__ void combine_blocks_kernel(const TileStats* __restrict__ st, int64_t lines,
                                      int64_t tiles, int64_t* __restrict__ blocks) {
    const int64_t line = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    int q = 0;
    int64_t em = 0;
    for (int64_t t = 0; t < tiles; ++t) {
        em += st[line * tiles + t].cnt[q];
        q = st[line * tiles + t].exit[q];
    }
    blocks[line] = 1 + em;
}

// Main K2 kernel.
__global__ void __launch_bounds__(kThreads) fast_kernel(
    const double* __restrict__ u, double* __restrict__ out, const TileStats* __restrict__ st_in,
    TileStats* __restrict__ st_out, const double* __restrict__ drift_arr,
    const double* __restrict__ tv, int64_t tv_stride, int64_t* __restrict__ blocks_out,
    unsigned long long* __restrict__ diag, FastParams p) {
    __shared__ unsigned long long keys[kTile + 2];
    __shared__ double ubuf[kTile + 2];
    __shared__ int srclist[kMaxSrcList];
    __shared__ int nsrc;
    __shared__ int fallback;
    __shared__ double shred[4 * (kThreads / 32)];
    __shared__ Fsm3 shfsm[kThreads / 32];

    const int64_t n = p.n;
    const int64_t line = blockIdx.x / p.tiles;
    const int64_t tile = blockIdx.x - line * p.tiles;
    const int64_t j0 = tile * p.T;
    const int Tl = static_cast<int>(min(p.T, n - j0));
    const int64_t j1 = j0 + Tl + 1;  // last (unrolled) output this CTA evaluates
    const double* ul = u + line * n;
    const TileStats* sl = st_in + line * p.tiles;
    const double drift = drift_arr[line];
    const double tau = p.tau;

    // ---- per-line kernel constants (identical arithmetic to the host) ----
    const double eps = __ddiv_rn(1.0, static_cast<double>(n));
    const int64_t center = llround(__ddiv_rn(__dmul_rn(tau, drift), eps));
    const int64_t first = center - n;
    const int64_t dmin_w = first + 1, dmax_w = first + 2 * n - 1;  // interior of the window
    const double a = __ddiv_rn(__dmul_rn(eps, eps), tau);
    const double ia = __ddiv_rn(1.0, a);
    const double pe = __dmul_rn(drift, eps);
    double delta;
    {
        const double uu = 1.1102230246251565e-16;  // 2^-53
        const double dm = fmax(fabs(static_cast<double>(first)), fabs(static_cast<double>(first + 2 * n)));
        const double vmax = dm * eps / tau;
        const double kmag = tau * (0.5 * vmax * vmax + fabs(drift) * vmax);
        delta = 32.0 * uu * kmag / a + 8.0 * uu * (2.0 * n + fabs(drift) * eps / a) + 1e-9;
        delta = delta * 2.0;  // device-side margin on top of the host bound
    }

    if (threadIdx.x == 0) {
        nsrc = 0;
        fallback = 0;
    }
    for (int i = threadIdx.x; i < Tl + 2; i += blockDim.x) keys[i] = kKeyInf;

    // ---- line-wide oscillation, window-edge gap ----
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t t = threadIdx.x; t < p.tiles; t += blockDim.x) {
        lo = fmin(lo, sl[t].umin);
        hi = fmax(hi, sl[t].umax);
    }
    block_minmax4(lo, hi, 0.0, 0.0, shred);
    const double umin = shred[0], umax = shred[1];
    __syncthreads();
    {
        const double kfirst = kval(p.vtab, p.vofs, first, drift, tau);
        const double klast = kval(p.vtab, p.vofs, first + 2 * n, drift, tau);
        double kmin = INFINITY;
        for (int64_t d = center - 2; d <= center + 2; ++d)
            if (d >= first && d <= first + 2 * n) kmin = fmin(kmin, kval(p.vtab, p.vofs, d, drift, tau));
        const double gap = fmin(kfirst, klast) - kmin;
        const double osc = umax - umin;
        const bool ok = (osc * (1.0 + 1e-12) < gap * (1.0 - 1e-12)) && n >= 3;
        if (!ok && threadIdx.x == 0) fallback = 1;
    }

    // ---- block count of the INPUT u (decompose on the closed period) ----
    if (blocks_out && tile == 0 && threadIdx.x == 0) {
        int q = 0;
        int64_t em = 0;
        for (int64_t t = 0; t < p.tiles; ++t) {
            em += sl[t].cnt[q];
            q = sl[t].exit[q];
        }
        blocks_out[line] = 1 + em;
    }
    __syncthreads();

    // unrolled source range that can reach outputs [j0, j1]
    const int64_t ylo = j0 - dmax_w, yhi = j1 - dmin_w;
    const int64_t k_lo = (ylo >= 0) ? ylo / n : -((-ylo + n - 1) / n);
    const int64_t k_hi = (yhi >= 0) ? yhi / n : -((-yhi + n - 1) / n);
    if (!fallback) {
        // ---- which (unrolled) source tiles can reach outputs [j0, j1]? ----
        const int64_t ncand = (k_hi - k_lo + 1) * p.tiles;
        for (int64_t c = threadIdx.x; c < ncand; c += blockDim.x) {
            const int64_t k = k_lo + c / p.tiles;
            const int64_t sg = c - (c / p.tiles) * p.tiles;
            const int64_t sgp = sg == 0 ? p.tiles - 1 : sg - 1;
            const double smn = fmin(sl[sg].smin, sl[sgp].smin);
            const double smx = sl[sg].smax;
            double zl = ceil(__dmul_rn(__dadd_rn(smn, pe), ia) - 0.5 - delta);
            double zr = floor(__dmul_rn(__dadd_rn(smx, pe), ia) + 0.5 + delta);
            zl = fmax(zl, static_cast<double>(dmin_w));
            zr = fmin(zr, static_cast<double>(dmax_w));
            if (!(zl <= zr)) continue;
            const int64_t ys = k * n + sg * p.T;
            const int64_t ye = ys + min(p.T, n - sg * p.T) - 1;
            if (ys + static_cast<int64_t>(zl) <= j1 && ye + static_cast<int64_t>(zr) >= j0) {
                const int slot = atomicAdd(&nsrc, 1);
                if (slot < kMaxSrcList)
                    srclist[slot] = static_cast<int>(c);
                else
                    fallback = 1;
            }
        }
        __syncthreads();
    }

    if (!fallback) {
        const int ns = nsrc;
        for (int li = 0; li < ns; ++li) {
            const int64_t c = srclist[li];
            const int64_t k = k_lo + c / p.tiles;
            const int64_t sg = c - (c / p.tiles) * p.tiles;
            const int64_t ys = k * n + sg * p.T;
            const int Ts = static_cast<int>(min(p.T, n - sg * p.T));
            __syncthreads();
            // U(ys-1 .. ys+Ts) -> ubuf[0 .. Ts+1]
            const int64_t base = ys - 1;
            int64_t bm = base % n;
            if (bm < 0) bm += n;
            for (int i = threadIdx.x; i < Ts + 2; i += blockDim.x) {
                int64_t yy = bm + i;
                if (yy >= n) yy -= n;
                if (yy >= n) yy -= n;
                ubuf[i] = ul[yy];
            }
            __syncthreads();
            for (int i = threadIdx.x; i < Ts; i += blockDim.x) {
                const double uy = ubuf[i + 1];
                const double sp = __dsub_rn(uy, ubuf[i]);      // s(y-1)
                const double sn = __dsub_rn(ubuf[i + 2], uy);  // s(y)
                double zl = ceil(__dmul_rn(__dadd_rn(sp, pe), ia) - 0.5 - delta);
                double zr = floor(__dmul_rn(__dadd_rn(sn, pe), ia) + 0.5 + delta);
                const int64_t y = ys + i;
                zl = fmax(zl, fmax(static_cast<double>(dmin_w), static_cast<double>(j0 - y)));
                zr = fmin(zr, fmin(static_cast<double>(dmax_w), static_cast<double>(j1 - y)));
                if (!(zl <= zr)) continue;
                const int64_t dl = static_cast<int64_t>(zl), dr = static_cast<int64_t>(zr);
                for (int64_t d = dl; d <= dr; ++d) {
                    const double c2 = __dadd_rn(uy, kval(p.vtab, p.vofs, d, drift, tau));
                    atomicMin(&keys[y + d - j0], dkey(c2));
                }
            }
        }
    }
    __syncthreads();

    // ---- epilogue: exact min -> out, with direct fallback where needed ----
    const double* tvl = tv ? tv + line * tv_stride : nullptr;
    for (int i = threadIdx.x; i < Tl + 2; i += blockDim.x) {
        int64_t j = j0 + i;
        if (j >= n) j -= n;
        if (j >= n) j -= n;
        double best;
        if (fallback || keys[i] == kKeyInf) {
            if (!fallback && diag) atomicAdd(diag, 1ull);
            // direct scan of the full window (proj/tests/unit_scheme.cpp:184-190)
            best = INFINITY;
            int64_t y = (j - first) % n;
            if (y < 0) y += n;
            for (int64_t w = 0; w <= 2 * n; ++w) {
                const double c2 = __dadd_rn(ul[y], kval(p.vtab, p.vofs, first + w, drift, tau));
                best = c2 < best ? c2 : best;
                y = y == 0 ? n - 1 : y - 1;
            }
        } else {
            best = dkey_inv(keys[i]);
        }
        const double o = tvl ? __dsub_rn(best, tvl[j]) : best;
        ubuf[i] = o;
        if (i < Tl) out[line * n + j] = o;
    }
    __syncthreads();
    if (st_out) tile_stats(ubuf, Tl, j0, n, p.eta, st_out + blockIdx.x, shred, shfsm);
}

}  // namespace

size_t fast_workspace_bytes(int64_t lines, int64_t n) {
    const int64_t T = n < kTile ? n : kTile;
    const int64_t tiles = (n + T - 1) / T;
    return 2 * static_cast<size_t>(lines * tiles) * sizeof(TileStats) + 64;
}

static int ensure_vtab(lob_ctx* ctx, int64_t n, double tau, const double** out, int64_t* vofs,
                       cudaStream_t s) {
    uint64_t tb;
    std::memcpy(&tb, &tau, sizeof(tb));
    auto key = std::make_pair(n, tb);
    auto it = ctx->vtabs.find(key);
    if (it == ctx->vtabs.end()) {
        lob_ctx::VTab vt;
        vt.dmin = -3 * n;
        vt.count = 6 * n + 1;
        LOB_CUDA_TRY(ctx, cudaMalloc(&vt.dev, vt.count * sizeof(double)));
        const double eps = 1.0 / static_cast<double>(n);
        build_vtab_kernel<<<static_cast<unsigned>((vt.count + 255) / 256), 256, 0, s>>>(vt.dev, 3 * n,
                                                                                         eps, tau);
        ctx->launches += 1;
        LOB_CUDA_TRY(ctx, cudaGetLastError());
        it = ctx->vtabs.emplace(key, vt).first;
    }
    *out = it->second.dev;
    *vofs = 3 * n;
    return LOB_OK;
}

int launch_fast_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                    const double* drift, double tau, const double* tv, int64_t tv_stride,
                    double eta, int64_t* blocks, void* workspace, size_t ws_bytes, int flags,
                    cudaStream_t s) {
    if (ws_bytes < fast_workspace_bytes(lines, n) || !workspace)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_f64: workspace too small");
    FastParams p;
    p.n = n;
    p.T = n < kTile ? n : kTile;
    p.tiles = (n + p.T - 1) / p.T;
    p.tau = tau;
    p.eta = eta;
    int st = ensure_vtab(ctx, n, tau, &p.vtab, &p.vofs, s);
    if (st) return st;
    const int64_t nblk = lines * p.tiles;
    if (nblk > 0x7fffffffll) return set_error(ctx, LOB_INVALID_INPUT, "fast: grid too large");
    TileStats* base = static_cast<TileStats*>(workspace);
    int& parity = ctx->ws_parity[workspace];
    if (ctx->ws_shape[workspace] != std::make_pair(lines, n)) {
        ctx->ws_shape[workspace] = std::make_pair(lines, n);
        flags &= ~LOB_FAST_STATS_VALID;
    }
    TileStats* sin = base + parity * nblk;
    TileStats* sout = base + (1 - parity) * nblk;
    unsigned long long* diag =
        reinterpret_cast<unsigned long long*>(base + 2 * nblk);
    if (!(flags & LOB_FAST_STATS_VALID)) {
        stats_kernel<<<static_cast<unsigned>(nblk), kThreads, 0, s>>>(u, sin, p);
        ctx->launches += 1;
        LOB_CUDA_TRY(ctx, cudaGetLastError());
    }
    fast_kernel<<<static_cast<unsigned>(nblk), kThreads, 0, s>>>(u, out, sin, sout, drift, tv,
                                                                  tv_stride, blocks, diag, p);
    ctx->launches += 1;
    LOB_CUDA_TRY(ctx, cudaGetLastError());
    parity = 1 - parity;
    return LOB_OK;
}

int launch_block_counts(lob_ctx* ctx, const double* u, int64_t lines, int64_t n, double eta,
                        int64_t* blocks, cudaStream_t s) {
    FastParams p{};
    p.n = n;
    p.T = n < kTile ? n : kTile;
    p.tiles = (n + p.T - 1) / p.T;
    p.eta = eta;
    const int64_t nblk = lines * p.tiles;
    TileStats* st = nullptr;
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&st, nblk * sizeof(TileStats), s));
    stats_kernel<<<static_cast<unsigned>(nblk), kThreads, 0, s>>>(u, st, p);
    combine_blocks_kernel<<<static_cast<unsigned>((lines + 127) / 128), 128, 0, s>>>(st, lines,
                                                                                     p.tiles, blocks);
    ctx->launches += 2;
    cudaFreeAsync(st, s);
    return cuda_status(ctx, cudaGetLastError(), "block counts");
}

}  // namespace lob

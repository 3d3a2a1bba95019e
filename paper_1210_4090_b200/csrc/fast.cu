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
// (else the tile falls back to the direct scan).  Inside a locally convex
// run the intervals tile the outputs contiguously (the slope merge of the
// paper's Algorithm 1 / Lemma 4.1); concave kinks leave empty intervals and
// fold the walk back (Algorithm 2's envelope); overlaps resolve by an exact
// min.  Total candidates ~ n + TV+(s)/a per line.
//
// Layout and data flow (one launch per step, device resident):
//  * a CTA (256 threads) owns T = 2048 consecutive outputs of one line;
//  * statistics of u from the previous step's epilogue: per 256-sample
//    sub-tile slope bounds, per-tile decompose() FSM summary, and per-line
//    min/max of u and of its slopes (global 64-bit atomics on
//    order-preserving keys, three rotating buffers);
//  * the CTA bounds its source range with the line stats, keeps only the
//    sub-tiles whose slope-implied displacements reach its outputs, stages
//    U (chunks of 2048 + halo) and the K values it needs in shared memory,
//    and emits candidates into shared 64-bit keys (exact min);
//  * the epilogue writes u^{n+1} = best - tv coalesced and produces the
//    statistics of u^{n+1} for the next step, including decompose()'s block
//    count (proj/src/minplus.cpp:152-188) as a composable 3-state
//    transition summary per tile.
// Lines of n <= 2048 run K2L instead (line_kernel): one CTA per whole line,
// the statistics reduced from the staged line itself, nothing carried; its
// load / store layouts (rows, strided columns, DSMEM cluster exchange, 2-D TMA
// tensor maps) serve the 2-D split step.  K2R (resident_kernel) runs every
// step of an evolve of short lines in one launch.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <type_traits>

#include <cooperative_groups.h>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstddef>

#include "lob_internal.cuh"

namespace lob {
namespace cg = cooperative_groups;

#ifndef LOB_KT
#define LOB_KT 2048
#endif
constexpr int kT = LOB_KT;     // outputs per CTA tile
#ifndef LOB_NT
#define LOB_NT 256
#endif
constexpr int kNT = LOB_NT;           // threads per CTA
constexpr int kG = kT / (kNT / 32);   // sub-tile (slope statistics granularity): one warp each
constexpr int kSub = kT / kG;  // sub-tiles per tile (= warps per CTA)
constexpr int kPer = kT / kNT; // outputs / sources per thread
#ifndef LOB_EMIT_UNROLL
#define LOB_EMIT_UNROLL 1
#endif
constexpr int kEmitUnroll = LOB_EMIT_UNROLL;  // sources in flight per lane in the emission loop
#ifndef LOB_FAST_MINB
#define LOB_FAST_MINB 5  // CTAs per SM the main kernel is built for (registers, shared memory)
#endif
#ifndef LOB_QCAP
#define LOB_QCAP 96
#endif
#ifndef LOB_KC
#define LOB_KC 2560
#endif
#ifndef LOB_EMIT_SERIAL
#define LOB_EMIT_SERIAL 0  // 1: each thread walks a contiguous block of sources (else lane-interleaved)
#endif
#ifndef LOB_EMIT_INTERLEAVE
#define LOB_EMIT_INTERLEAVE 1  // warps take interleaved 32-source blocks (else one contiguous range each)
#endif
constexpr int kQCap = LOB_QCAP;  // queued source intervals (long / contended) per chunk
#ifndef LOB_QSHORT
#define LOB_QSHORT 8
#endif
constexpr int kQShort = LOB_QSHORT;  // queued runs shorter than this are finished by one thread
constexpr int kC = LOB_KC;       // sources staged per chunk (a typical tile + halo in one pass)
#ifndef LOB_VCAP
#define LOB_VCAP 896
#endif
constexpr int kVCap = LOB_VCAP;  // v_d values staged per tile (TMA, with the first chunk)
#ifndef LOB_FAST_WORK_COUNTERS
#define LOB_FAST_WORK_COUNTERS 0  // per-source inline-candidate count (diagnostic builds only)
#endif

#ifndef LOB_TILE_DIRECT
#define LOB_TILE_DIRECT 1
#endif
// The oscillation gate of a line (fast_kernel): max u - min u (exact extremes, collected by the
// epilogue when the line needs them) or the cheap bound (n/2) max |slope|, whichever passes.

struct LineConst {
    long long first;  // window displacement of w = 0
    double pe;        // drift * eps
    double hl, hr;    // dL = ceil(s/a + hl), dR = floor(s/a + hr): hl/hr = P eps/a -/+ (1/2 + delta)
    double gap;       // min(K(first), K(first+2n)) - min K: the oscillation gate
    double drift;
    // window-table mode (any convex window, lob_minplus_fast_window_f64):
    const double* kt;  // K(d) = kt[d] for d in [first, first + 2n] (the line's table, offset by -first)
    double tol;        // slope comparisons are relaxed by tol * (|s| + max |sigma|) (rounding of both sides)
    double smax;       // max |sigma(d)| over the window, sigma(d) = K(d+1) - K(d)
    double sg0, sgi;   // search hint: d ~ first + (s - sigma(first)) * sgi (slopes linear in d)
    double k0, kmid, kend;  // window samples at w = 0, n, 2n (staleness check of carried constants)
};
static_assert(kSub == kNT / 32, "one warp per sub-tile in the epilogue");
static_assert(kPer % 2 == 0, "FSM pairs");

struct FastParams {
    int64_t n;
    int64_t lines;  // lines of the batch (fast_kernel: CTAs of the folded grid past it exit)
    int64_t tiles;  // ceil(n / kT)
    int64_t subs;   // ceil(n / kG)
    double tau;
    double eta;
    double eps, a, ia;  // 1/n, eps^2/tau, 1/a (host IEEE, same as the device's)
    const double* vtab;  // v_d for d in [-vofs, vofs]
    int64_t vofs;
    int fsm_on;  // the epilogue produces decompose()'s FSM summaries for the next step's block count
    int check;   // LOB_FAST_STATS_CHECK: compare u with the samples the statistics were taken with
    int samples; // the epilogue stores samples of u^{n+1} (a workspace that has seen a checked call)
    // evolve's per-step drift reduced in the kernel (with dpart): the line's last tile to finish sums
    // the tiles' partials in tile order (dcount: per-line arrival counter, monotonic across steps)
    double* drift_out;
    int* halt;
    unsigned* dcount;
    int dstep;
    double delta_override;  // NaN: the computed rounding bound delta (diagnostic hook, lob_ctx_set_fast_delta)
    // the caller's current per-line inputs (checked against the carried line constants)
    const double* drift_arr;                      // mechanical mode
    // separable potential (the 2-D split step's second sweep): tau*V(line, j) =
    // tau * (sa1[line] * sa2[j] + sb) with the C++ expression's roundings (no FMA)
    const double* sa1;
    const double* sa2;
    double sb;
    const double* ktab;                           // table mode: windows ...
    int64_t kstride;                              // ... their stride (0: shared) ...
    const int64_t* kfirst;                        // ... and first displacements
};

struct FastBuffers {
    const double2* sub_in;  // [lines][subs] (min, max) of s over the sub-tile + left halo
    const unsigned long long* fsm_in;   // [lines][tiles]
    const unsigned long long* line_in;  // [lines][4] keys: umin, umax, smin, smax
    double2* sub_out;
    unsigned long long* fsm_out;
    unsigned long long* line_out;
    unsigned long long* line_reset;
    const double* samp_in;  // [lines][kSamp] samples of u taken with its statistics
    double* samp_out;       // ... of u^{n+1}
};
constexpr int kSamp = 32;  // sampled positions per line: (k n) >> 5, k < 32

namespace {

__device__ __forceinline__ double kval_v(double v, double drift, double tau) {
    // tau * ((0.5*v)*v - drift*v): proj/src/scheme.cpp:80 + hamiltonian.cpp:43
    return __dmul_rn(tau, __dsub_rn(__dmul_rn(__dmul_rn(0.5, v), v), __dmul_rn(drift, v)));
}
__device__ __forceinline__ double kval(const double* vtab, int64_t vofs, int64_t d, double drift,
                                       double tau) {
    return kval_v(vtab[d + vofs], drift, tau);
}

// ---- decompose() FSM (proj/src/minplus.cpp:161-187) ------------------------
// Classes: 0 pos (inc > eta), 1 neg (inc < -eta), 2 zero band, 3 NaN.
// States: 0 undetermined, 1 convex, 2 concave.  A "vector" packs the current
// state of the three runs started in U, Cx, Cc (2 bits each); the LUT maps
// (vector, class) -> next vector | emits<<6 (one bit per run).
__host__ __device__ inline int fsm_next(int q, int c, int* emit) {
    if (q == 0) {
        *emit = 0;
        return c == 0 ? 1 : (c == 1 ? 2 : 0);
    }
    if (q == 1) {
        *emit = (c == 1 || c == 3) ? 1 : 0;
        return *emit ? 0 : 1;
    }
    *emit = (c == 0 || c == 3) ? 1 : 0;
    return *emit ? 0 : 2;
}

// packed summary: bits 0..5 exit states of the 3 runs, bits 16.. counts (3 x 16 bits)
__device__ __forceinline__ unsigned long long fsm_pack(int v, const int* cnt) {
    return static_cast<unsigned long long>(v) | (static_cast<unsigned long long>(cnt[0]) << 16) |
           (static_cast<unsigned long long>(cnt[1]) << 32) |
           (static_cast<unsigned long long>(cnt[2]) << 48);
}
__device__ __forceinline__ unsigned long long fsm_identity() { return 0u | (1u << 2) | (2u << 4); }
// compose summaries: a then b
__device__ __forceinline__ unsigned long long fsm_compose(unsigned long long a, unsigned long long b) {
    int v = 0;
    int cnt[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
        const int m = static_cast<int>((a >> (2 * q)) & 3);
        v |= static_cast<int>((b >> (2 * m)) & 3) << (2 * q);
        cnt[q] = static_cast<int>((a >> (16 + 16 * q)) & 0xffff) +
                 static_cast<int>((b >> (16 + 16 * m)) & 0xffff);
    }
    return fsm_pack(v, cnt);
}

// Pair table: entry (v, c0, c1) = v' | emit_run0 << 6 | emit_run1 << 9 | emit_run2 << 12
// after classes c0 then c1 (class 3 = no increment).  A run emits at most once
// per pair (an emission leaves it undetermined), so 4 pairs accumulate into
// 3-bit fields.  1024 x 2 B, read through the L1 (__ldg).
__device__ unsigned short g_fsm_lut2[64 * 16];
constexpr int kLut2 = 64 * 16;

__device__ __forceinline__ unsigned long long warp_fsm(unsigned long long f) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
        const unsigned long long o = __shfl_down_sync(0xffffffffu, f, off);
        if ((lane & (2 * off - 1)) == 0 && lane + off < 32) f = fsm_compose(f, o);
    }
    return f;  // valid in lane 0
}

struct EpiShared {
    unsigned kred[2][kNT / 32];
    unsigned ured[2][kNT / 32];
    unsigned long long fsm[kNT];
};

// Shared-memory padding: one slot per 8 doubles, so the per-thread
// contiguous (stride-8) access patterns are bank-conflict free.
__host__ __device__ __forceinline__ constexpr int P8(int i) { return i + (i >> 3); }


// High 32 bits of the order-preserving key: a monotone coarse key.  The
// smallest (largest) double with a given coarse key is a lower (upper) bound
// of every double with that key, within 2^-20 relative.
__device__ __forceinline__ unsigned hkey(double x) {
    const unsigned hi = static_cast<unsigned>(__double2hiint(x));
    return hi ^ (static_cast<unsigned>(static_cast<int>(hi) >> 31) | 0x80000000u);
}
__device__ __forceinline__ double hkey_lower(unsigned k) {
    return dkey_inv(static_cast<unsigned long long>(k) << 32);
}
__device__ __forceinline__ double hkey_upper(unsigned k) {
    return dkey_inv((static_cast<unsigned long long>(k) << 32) | 0xffffffffull);
}

// Statistics of u^{n+1} (or of an input u) for the tile whose values are
// vals[i] = u(j0 - 1 + i), i = 0 .. Tl + 2 (periodic), Tl = tile length,
// all in shared memory.  Thread t owns the slopes s(j0 + 8t - 1 .. j0 + 8t + 7)
// and the increments e = j0 + 8t + 1 .. j0 + 8t + 8; warp w owns sub-tile w
// (256 sources).  Produced:
//  * per sub-tile: conservative bounds [smin, smax] of its slopes s(qG-1 .. qG+len-1)
//    (coarse keys reduced with REDUX; exactness is not needed, only enclosure);
//  * per line: the same bounds over the whole line (global atomics);
//  * per tile: decompose()'s 3-state transition summary (FSM of
//    proj/src/minplus.cpp:161-187).  For eta == 0 the increment class is the
//    exact comparison of consecutive slopes (fl(a-b) > 0 <=> a > b for finite
//    doubles; -0 == +0 like the reference's inc == 0).
// FULL: a whole tile that is not the line's last (no bounds checks).
template <bool FULL>
__device__ void tile_stats(const double* vals, int Tl, int64_t j0, int64_t line, int64_t tile,
                           const FastParams& p, const FastBuffers& b, EpiShared& sh,
                           const unsigned short* lut, bool osc_exact = true) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int i0 = kPer * tid;  // vals index of u(j0 + 8t - 1)
    double w[kPer + 3];
#pragma unroll
    for (int m = 0; m < kPer + 3; ++m) w[m] = (FULL || i0 + m <= Tl + 2) ? vals[P8(i0 + m)] : 0.0;
    double sl[kPer + 2];
#pragma unroll
    for (int m = 0; m < kPer + 2; ++m) sl[m] = __dsub_rn(w[m + 1], w[m]);
    unsigned kmin = 0xffffffffu, kmax = 0u;
#pragma unroll
    for (int m = 0; m <= kPer; ++m) {
        if (FULL || m <= Tl - i0) {  // s(j0 - 1 + 8t + m), up to s(j0 + Tl - 1)
            const unsigned k = hkey(sl[m]);
            kmin = min(kmin, k);
            kmax = max(kmax, k);
        }
    }
    // exact extremes of the tile's own values u(j0 + 8t .. j0 + 8t + 7): the
    // oscillation gate of the next step
    // (coarse 32-bit keys: an enclosure within 2^-20 relative, like the slope bounds)
    unsigned hmn = 0xffffffffu, hmx = 0u;
    if (osc_exact) {
#pragma unroll
        for (int m = 1; m <= kPer; ++m) {
            if (FULL || m <= Tl - i0) {
                const unsigned k = hkey(w[m]);
                hmn = min(hmn, k);
                hmx = max(hmx, k);
            }
        }
    }
    // decompose() FSM over increments e = j0 + 8t + 1 + k: inc = s(e) - s(e-1),
    // two increments per table lookup.  Non-finite u (which the reference
    // rejects before decompose, proj/src/scheme.cpp:18-24) is not classified.
    int v = 0 | (1 << 2) | (2 << 4);
    unsigned acc = 0;
    const bool exact_cmp = p.eta == 0.0;
    const bool fsm_on = p.fsm_on != 0;
    auto cls = [&](int k) -> int {  // class of increment e = j0 + i0 + 1 + k
        const int i = i0 + 1 + k;
        if (!FULL && !(i <= Tl && j0 + i <= p.n - 1)) return 3;
        if (exact_cmp) return sl[k + 2] > sl[k + 1] ? 0 : (sl[k + 2] < sl[k + 1] ? 1 : 2);
        const double inc = __dsub_rn(sl[k + 2], sl[k + 1]);
        return inc > p.eta ? 0 : (inc < -p.eta ? 1 : 2);
    };
    if (fsm_on) {
#pragma unroll
        for (int k = 0; k < kPer; k += 2) {
            const unsigned x = __ldg(lut + v * 16 + cls(k) * 4 + cls(k + 1));
            v = static_cast<int>(x & 63u);
            acc += x >> 6;
        }
        const int cnt[3] = {static_cast<int>(acc & 7u), static_cast<int>((acc >> 3) & 7u),
                            static_cast<int>(acc >> 6)};
        sh.fsm[tid] = fsm_pack(v, cnt);
    }
    kmin = __reduce_min_sync(0xffffffffu, kmin);
    kmax = __reduce_max_sync(0xffffffffu, kmax);
    if (osc_exact) {
        hmn = __reduce_min_sync(0xffffffffu, hmn);
        hmx = __reduce_max_sync(0xffffffffu, hmx);
    }
    if (lane == 0) {
        const double smn = hkey_lower(kmin), smx = hkey_upper(kmax);
        if (FULL || warp * kG < Tl) {
            const int64_t q = (j0 + warp * kG) / kG;
            b.sub_out[line * p.subs + q] = make_double2(smn, smx);
        }
        sh.kred[0][warp] = kmin;
        sh.kred[1][warp] = kmax;
        sh.ured[0][warp] = hmn;
        sh.ured[1][warp] = hmx;
    }
    __syncthreads();
    if (warp == 0) {
        // lane l composes summaries 8l .. 8l+7, then an ordered warp reduction
        unsigned long long f = 0;
        if (fsm_on) {
            f = sh.fsm[lane * (kNT / 32)];
#pragma unroll
            for (int k = 1; k < kNT / 32; ++k) f = fsm_compose(f, sh.fsm[lane * (kNT / 32) + k]);
            f = warp_fsm(f);
        }
        unsigned a0 = lane < kNT / 32 ? sh.kred[0][lane] : 0xffffffffu;
        unsigned a1 = lane < kNT / 32 ? sh.kred[1][lane] : 0u;
        a0 = __reduce_min_sync(0xffffffffu, a0);
        a1 = __reduce_max_sync(0xffffffffu, a1);
        const unsigned m0 = __reduce_min_sync(0xffffffffu, lane < kNT / 32 ? sh.ured[0][lane] : 0xffffffffu);
        const unsigned m1 = __reduce_max_sync(0xffffffffu, lane < kNT / 32 ? sh.ured[1][lane] : 0u);
        if (lane == 0) {
            if (fsm_on) b.fsm_out[line * p.tiles + tile] = f;
            unsigned long long* L = b.line_out + line * 4;
            if (osc_exact) {
                atomicMin(L + 0, dkey(hkey_lower(m0)));
                atomicMax(L + 1, dkey(hkey_upper(m1)));
            }
            atomicMin(L + 2, dkey(hkey_lower(a0)));
            atomicMax(L + 3, dkey(hkey_upper(a1)));
        }
    }
}

__global__ void __launch_bounds__(kNT) stats_kernel(const double* __restrict__ u, FastParams p,
                                                    FastBuffers b) {
    __shared__ __align__(16) double vals[P8(kT + 3) + 1];
    __shared__ EpiShared sh;
    const unsigned short* lut = g_fsm_lut2;
    const int64_t line = blockIdx.x / p.tiles;
    const int64_t tile = blockIdx.x - line * p.tiles;
    const int64_t j0 = tile * kT;
    const int Tl = static_cast<int>(min(static_cast<int64_t>(kT), p.n - j0));
    const double* ul = u + line * p.n;
    for (int i = threadIdx.x; i < Tl + 3; i += kNT) {
        int64_t j = j0 - 1 + i;
        if (j < 0) j += p.n;
        if (j >= p.n) j %= p.n;
        vals[P8(i)] = ul[j];
    }
    __syncthreads();
    if (threadIdx.x < kSamp) {
        const int64_t pos = (static_cast<int64_t>(threadIdx.x) * p.n) >> 5;
        if (pos >= j0 && pos < j0 + Tl) b.samp_out[line * kSamp + threadIdx.x] = vals[P8(static_cast<int>(pos - j0) + 1)];
    }
    if (Tl == kT && j0 + kT <= p.n - 1)
        tile_stats<true>(vals, Tl, j0, line, tile, p, b, sh, lut);
    else
        tile_stats<false>(vals, Tl, j0, line, tile, p, b, sh, lut);
}

// The 2-D split step's transposes (proj/src/splitting.cpp:67-76 gathers strided lines) fused
// with K2's input statistics of the transposed lines: dst = src^T for an n x n row-major
// tensor, and for every line of dst (a column of src) the per-256-sample sub-tile slope
// bounds and the line's u / slope extremes that tile_stats produces (same coarse keys), so
// the following K2 sweep needs no statistics pass.  CTA = kTSL columns x one sub-tile of rows.
constexpr int kTSL = 8;
static_assert(kTSL == 8, "one warp per transposed line (256 threads)");
__global__ void __launch_bounds__(256) transpose_stats_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                              int64_t n, int64_t subs, double2* __restrict__ sub,
                                                              unsigned long long* __restrict__ L) {
    __shared__ double tile[kG + 2][kTSL + 1];  // rows r0-1 .. r0+len (periodic) x kTSL columns
    const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kTSL;
    const int64_t q = blockIdx.y;
    const int64_t r0 = q * kG;
    const int len = static_cast<int>(min(static_cast<int64_t>(kG), n - r0));
    {
        // thread (row group, column): 32 rows of kTSL columns per pass, 64-byte row segments
        const int c = threadIdx.x % kTSL, rg = threadIdx.x / kTSL;
        const bool cok = c0 + c < n;
        for (int r = rg; r < len + 2; r += 256 / kTSL) {
            int64_t row = r0 - 1 + r;
            row = row < 0 ? row + n : (row >= n ? row - n : row);
            tile[r][c] = cok ? __ldg(src + row * n + c0 + c) : 0.0;
        }
    }
    __syncthreads();
    {
        // warp w writes line c0 + w: contiguous, coalesced
        const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (w < kTSL && c0 + w < n) {
            double* d = dst + (c0 + w) * n + r0;
            for (int i = lane; i < len; i += 32) d[i] = tile[i + 1][w];
        }
    }
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w < kTSL && c0 + w < n) {
        // slopes s(r0 - 1 .. r0 + len - 1) and values u(r0 .. r0 + len - 1) of line c0 + w
        unsigned smn = 0xffffffffu, smx = 0u, umn = 0xffffffffu, umx = 0u;
        for (int r = lane; r <= len; r += 32) {
            const unsigned k = hkey(__dsub_rn(tile[r + 1][w], tile[r][w]));
            smn = min(smn, k);
            smx = max(smx, k);
            if (r < len) {
                const unsigned ku = hkey(tile[r + 1][w]);
                umn = min(umn, ku);
                umx = max(umx, ku);
            }
        }
        smn = __reduce_min_sync(0xffffffffu, smn);
        smx = __reduce_max_sync(0xffffffffu, smx);
        umn = __reduce_min_sync(0xffffffffu, umn);
        umx = __reduce_max_sync(0xffffffffu, umx);
        if (lane == 0) {
            const int64_t line = c0 + w;
            sub[line * subs + q] = make_double2(hkey_lower(smn), hkey_upper(smx));
            unsigned long long* Ll = L + line * 4;
            atomicMin(Ll + 0, dkey(hkey_lower(umn)));
            atomicMax(Ll + 1, dkey(hkey_upper(umx)));
            atomicMin(Ll + 2, dkey(hkey_lower(smn)));
            atomicMax(Ll + 3, dkey(hkey_upper(smx)));
        }
    }
}

// per-line drift from the K2 tiles' partial sums, in tile order; non-finite -> halt
__global__ void drift_tiles_kernel(const double* __restrict__ dpart, int64_t lines, int64_t tiles, int64_t n,
                                   double* __restrict__ drift_out, int* __restrict__ halt, int step) {
    const int64_t line = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    double sum = 0.0;
    for (int64_t t = 0; t < tiles; ++t) sum += dpart[line * tiles + t];
    if (drift_out) drift_out[line] = sum / static_cast<double>(n);
    if (!isfinite(sum) && halt) atomicMin(halt, step);
}

__global__ void line_init_kernel(unsigned long long* L, int64_t lines) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= lines) return;
    L[4 * i + 0] = ~0ull;
    L[4 * i + 1] = 0ull;
    L[4 * i + 2] = ~0ull;
    L[4 * i + 3] = 0ull;
}

__global__ void build_vtab_kernel(double* vtab, int64_t vofs, double eps, double tau) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i > 2 * vofs) return;
    const int64_t d = i - vofs;
    // x = (double)d * eps; v = x / tau  (proj/src/scheme.cpp:79-80)
    vtab[i] = __ddiv_rn(__dmul_rn(static_cast<double>(d), eps), tau);
}

__global__ void combine_blocks_kernel(const unsigned long long* __restrict__ fsm, int64_t lines,
                                      int64_t tiles, int64_t* __restrict__ blocks) {
    const int64_t line = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    int q = 0;
    int64_t em = 0;
    for (int64_t t = 0; t < tiles; ++t) {
        const unsigned long long f = fsm[line * tiles + t];
        em += (f >> (16 + 16 * q)) & 0xffff;
        q = static_cast<int>((f >> (2 * q)) & 3);
    }
    blocks[line] = 1 + em;
}

// u^{n+1} of the tile (padded, for tile_stats) reuses ubuf after the emission
// phase; the statistics' reduction scratch reuses keys after the epilogue.
constexpr int kValsLen = P8(kT + 3) + 2;
#ifndef LOB_WIDE_RANGE
#define LOB_WIDE_RANGE kVCap  // displacement range above which a tile scans source runs
#endif
constexpr int kRuns = 8;  // source runs per wide tile (more are merged into the last)
#ifndef LOB_HEAVY
#define LOB_HEAVY 0.25
#endif
constexpr int kTW = 1024;  // displacements per staged chunk of the direct tile sweep

enum : int { kModeWalk = 0, kModeDirect = 1 };

struct MainShared {
    unsigned long long keys[kT + 4];   // exact-min slots (+inf bits = empty), lane-interleaved access
    unsigned long long mbar;           // TMA completion barrier for the source chunk
    __align__(16) double ubuf[kC + 8];  // sources (unpadded) / then u^{n+1} (padded, stats)
    int3 queue[kQCap];
    __align__(16) double vbuf[kVCap];  // v_d of the tile's displacement range, converted to K(d)
    int ya, yb, nq, nlong, dlo, dhi, DLg, DRg, mode, gate, abort, osc_exact;
    unsigned qwork, budget;            // long queued runs of the tile, and the walk's work budget
    int nruns, rs[kRuns], re[kRuns];  // runs of reaching sub-tiles (unrolled source ranges)
    unsigned int c_src, c_queued, c_qent;
    __device__ EpiShared& epi() { return *reinterpret_cast<EpiShared*>(keys); }
};
static_assert(kValsLen <= kC + 8, "u^{n+1} of the tile fits in ubuf");
static_assert(sizeof(EpiShared) <= (kT + 4) * 8, "statistics scratch fits in keys");
// per-CTA shared allocations are rounded to 128 bytes, plus 1 KB the driver reserves
static_assert(LOB_FAST_MINB * ((sizeof(MainShared) + 127) / 128 * 128 + 1024) <= 233472, "LOB_FAST_MINB CTAs per SM");
static_assert((P8(kT + kTW) + 1 + kTW) * 8 <= sizeof(MainShared), "direct tile sweep fits the shared layout");

// ---- TMA bulk copies (cp.async.bulk) completed on an mbarrier ------------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n LAB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr unsigned long long kInfBits = 0x7ff0000000000000ull;  // +inf

// x mod n in [0, n): selects for x in (-3n, 3n), the general remainder beyond (a window whose centre
// lies more than two periods away: |tau P| > 2 in window-table mode; once per chunk, never per source)
__device__ __forceinline__ int wrap_idx(int x, int n) {
    if (x <= -3 * n || x >= 3 * n) {
        x %= n;
        return x < 0 ? x + n : x;
    }
    x += x < 0 ? n : 0;
    x += x < 0 ? n : 0;
    x += x < 0 ? n : 0;
    x -= x >= n ? n : 0;
    x -= x >= n ? n : 0;
    return x - (x >= n ? n : 0);
}

// exact min of doubles in shared memory (CAS on the bit pattern; the first
// candidate of an output replaces the +inf sentinel)
__device__ __forceinline__ void smem_fmin(unsigned long long* addr, double c) {
    const unsigned long long cb = static_cast<unsigned long long>(__double_as_longlong(c));
    unsigned long long old = atomicCAS(addr, kInfBits, cb);
    while (old != kInfBits && c < __longlong_as_double(static_cast<long long>(old))) {
        const unsigned long long prev = atomicCAS(addr, old, cb);
        if (prev == old) break;
        old = prev;
    }
}

// exact min into a slot that already holds a value (the frontier candidate or the gap's
// +inf): a plain read first, the CAS only when c improves on it
__device__ __forceinline__ void smem_fmin_set(unsigned long long* addr, double c) {
    const unsigned long long cb = static_cast<unsigned long long>(__double_as_longlong(c));
    unsigned long long old = *reinterpret_cast<volatile unsigned long long*>(addr);
    while (c < __longlong_as_double(static_cast<long long>(old))) {
        const unsigned long long prev = atomicCAS(addr, old, cb);
        if (prev == old) break;
        old = prev;
    }
}

// One thread: TMA bulk copies of U(yc-1 .. yc+clen) (wrapped at the period as often as
// needed: short lines; 16-byte aligned even start) into ubuf, plus optionally vcnt v_d values.
__device__ __forceinline__ void issue_chunk(MainShared& S, const double* ul, int n, int yc, int clen,
                                            const double* vsrc, int vcnt) {
    const int bm = wrap_idx(yc - 1, n);
    const int sh = bm & 1;
    const int s0 = bm - sh;                    // even, in [0, n)
    const int cnt = (clen + 2 + sh + 1) & ~1;  // even count
    fence_proxy_async();
    mbar_expect_tx(&S.mbar, static_cast<unsigned>(cnt + (vsrc ? vcnt : 0)) * 8u);
    // segments [s0, n), [0, n), ..., [0, rest): even lengths and offsets (n even)
    for (int pos = s0, dst = 0; dst < cnt; pos = 0) {
        const int seg = min(cnt - dst, n - pos);
        tma_load_1d(S.ubuf + dst, ul + pos, static_cast<unsigned>(seg) * 8u, &S.mbar);
        dst += seg;
    }
    if (vsrc) tma_load_1d(S.vbuf, vsrc, static_cast<unsigned>(vcnt) * 8u, &S.mbar);
}

struct ChunkArgs {
    const double* ub;  // ub[i + 1] = U(yc + i), i in [-1, clen]
    int clen, base, jspan;
    double ia, hl, hr;
    int dlo, dhi;       // the tile's displacement range (clamp)
    const double* skt;  // K(d) staged in shared memory (KS) ...
    const double* gvt;  // ... or v_d (mechanical) / K(d) (window table) in global memory
    double drift, tau;
    const LineConst* lc;  // window-table mode: the slope search's constants
};

template <bool TAB, bool KS>
__device__ __forceinline__ double kvalue(const ChunkArgs& a, int d) {
    if constexpr (KS) return a.skt[d];
    else if constexpr (TAB) return __ldg(a.gvt + d);
    else return kval_v(__ldg(a.gvt + d), a.drift, a.tau);
}

// ---- window-table mode: local-minimum intervals by slope search --------------
// For any convex window the local-minimum conditions of the fast.cu header read
// S(y-1) <= Sigma(d) and Sigma(d-1) <= S(y) in exact arithmetic, Sigma(d) = K(d+1) - K(d)
// (nondecreasing: build_kernel's convexity check, proj/src/scheme.cpp:94-97).  With the
// rounded differences s, sigma (each within u |.| of the real value) they imply
// sigma(d) >= s(y-1) - t and sigma(d-1) <= s(y) + t, t = tol (|s| + max|sigma|), so
//   dL = min { d : sigma(d) >= s(y-1) - t },   dR = min { d : sigma(d) > s(y) + t }
// enclose every minimiser.  Each is a lower bound over the nondecreasing sigma, found
// by a galloping search from the linear-slope hint and a binary search in the bracket.
// smallest d in [lo, hi + 1] with sig(d) >= x (STRICT: > x); sig nondecreasing
template <bool STRICT, class SIG>
__device__ __forceinline__ int slope_search(SIG sig, double x, int lo, int hi, int hint) {
    auto ok = [&](int d) { return STRICT ? sig(d) > x : sig(d) >= x; };
    int d = min(max(hint, lo), hi + 1);
    int a, b;  // the answer lies in [a, b]
    if (d <= hi && !ok(d)) {
        a = d + 1;
        b = hi + 1;
        for (int step = 1;; step <<= 1) {
            const int e = d + step;
            if (e > hi) break;
            if (ok(e)) {
                b = e;
                break;
            }
            a = e + 1;
            d = e;
        }
    } else {
        a = lo;
        b = d;
        for (int step = 1;; step <<= 1) {
            const int e = d - step;
            if (e < lo) break;
            if (!ok(e)) {
                a = e + 1;
                break;
            }
            b = e;
            d = e;
        }
    }
    while (a < b) {
        const int m = (a + b) >> 1;
        if (ok(m)) b = m;
        else a = m + 1;
    }
    return a;
}
__device__ __forceinline__ int slope_hint(const LineConst& lc, double s) {
    const double g = static_cast<double>(lc.first) + (s - lc.sg0) * lc.sgi;
    return g > 1.0e9 ? 1000000000 : (g < -1.0e9 ? -1000000000 : __double2int_rd(g));
}
// [dL, dR] of slopes (sl, sr) with sigma from `sig`, searched inside [lo, hi] (the
// answers are clamped to [lo, hi + 1] / [lo - 1, hi] by construction)
template <class SIG>
__device__ __forceinline__ void tab_interval(SIG sig, const LineConst& lc, double sl, double sr, int lo, int hi,
                                             int& dl, int& dr) {
    const double tl = lc.tol * (fabs(sl) + lc.smax), tr = lc.tol * (fabs(sr) + lc.smax);
    dl = slope_search<false>(sig, sl - tl, lo, hi, slope_hint(lc, sl));
    dr = slope_search<true>(sig, sr + tr, lo - 1, hi - 1, slope_hint(lc, sr) + 1);
}

// Candidates of one staged source chunk.  Warp w takes sources w*per + lane +
// 32m (consecutive lanes, consecutive sources: conflict-free shared loads).
// Each source's first two displacements go straight to the output slots
// with one CAS against the empty sentinel; slots already holding a larger
// value, and intervals longer than two, are queued and finished after the
// barrier with exact CAS-min loops, one warp per queued source.  Returns false
// when the queued work exceeds `budget` (the walk would cost more than the
// window: the tile switches to the direct formula; the queue is not processed).
template <bool TAB, bool KS>
__device__ __forceinline__ bool process_chunk(MainShared& S, const ChunkArgs& a, unsigned budget) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // the chunk's output base held in a register: opaque to the compiler, which otherwise
    // re-derives it from the block index (an S2R on the emission loop's critical path)
    int cbase;
    asm volatile("mov.b32 %0, %1;" : "=r"(cbase) : "r"(a.base));
#if LOB_EMIT_SERIAL
    // thread t walks the sources t*k .. t*k+k-1 (k odd: conflict-free strided shared loads), each
    // value and slope read once and carried to the next source
    const int k = ((a.clen + kNT - 1) / kNT) | 1;
    const int ib = min(static_cast<int>(threadIdx.x) * k, a.clen);
    const int iend = min(ib + k, a.clen);
    double uc = a.ub[ib + 1], slc = __dsub_rn(uc, a.ub[ib]);
    for (int i = ib; i < iend; ++i) {
        const double u0 = uc;
        const double un = a.ub[i + 2];
        const double sl = slc, sr = __dsub_rn(un, u0);
        uc = un;
        slc = sr;
#elif LOB_EMIT_INTERLEAVE
    // warps take interleaved 32-source blocks (w, w + 8, ...): the uneven per-source work (long
    // intervals, folds) spreads over all warps before the chunk's barrier
    (void)lane;
    (void)warp;
    const int iend = a.clen;
#pragma unroll kEmitUnroll
    for (int i = threadIdx.x; i < iend; i += kNT) {
        const double ul0 = a.ub[i], u0 = a.ub[i + 1], ur0 = a.ub[i + 2];
        const double sl = __dsub_rn(u0, ul0), sr = __dsub_rn(ur0, u0);
#else
    (void)lane;
    const int per = ((a.clen + kNT - 1) / kNT) * 32;
    const int iend = min(a.clen, (warp + 1) * per);
#pragma unroll kEmitUnroll
    for (int i = warp * per + lane; i < iend; i += 32) {
        const double ul0 = a.ub[i], u0 = a.ub[i + 1], ur0 = a.ub[i + 2];
        const double sl = __dsub_rn(u0, ul0), sr = __dsub_rn(ur0, u0);
#endif
        int dl, dr;
        if constexpr (TAB) {
            auto sig = [&](int d) { return __dsub_rn(kvalue<TAB, KS>(a, d + 1), kvalue<TAB, KS>(a, d)); };
            tab_interval(sig, *a.lc, sl, sr, a.dlo, a.dhi, dl, dr);
        } else {
            // z(s) -/+ (1/2 + delta) with one fused rounding (delta bounds it, csrc/host/kernel_build.cpp)
            dl = __double2int_ru(__fma_rn(sl, a.ia, a.hl));
            dr = __double2int_rd(__fma_rn(sr, a.ia, a.hr));
        }
        const int off = cbase + i;  // output index of this source at d = 0
        // every candidate lies in [dlo, dhi] when the statistics describe u;
        // the clamp keeps stale statistics memory-safe (wrong, never out of bounds)
        dl = max(max(dl, a.dlo), -off);
        dr = min(min(dr, a.dhi), a.jspan - off);
        if (dl <= dr) {
            unsigned long long* slot = &S.keys[off + dl];
            const double c0 = __dadd_rn(u0, kvalue<TAB, KS>(a, dl));
            const unsigned long long o0 = atomicCAS(slot, kInfBits, static_cast<unsigned long long>(__double_as_longlong(c0)));
            const bool r0 = o0 != kInfBits && c0 < __longlong_as_double(static_cast<long long>(o0));
            bool r1 = false;
            if (dl < dr) {
                const double c1 = __dadd_rn(u0, kvalue<TAB, KS>(a, dl + 1));
                const unsigned long long o1 =
                    atomicCAS(slot + 1, kInfBits, static_cast<unsigned long long>(__double_as_longlong(c1)));
                r1 = o1 != kInfBits && c1 < __longlong_as_double(static_cast<long long>(o1));
            }
            const bool longer = dl + 2 <= dr;
            if (r0 | r1 | longer) {
                const int qlo = r0 ? dl : (r1 ? dl + 1 : dl + 2);
                const int qhi = longer ? dr : (r1 ? dl + 1 : dl);
                const int q = atomicAdd(&S.nq, 1);
                // long runs count against the walk's work budget
                if (qhi - qlo >= 32) atomicAdd(&S.qwork, static_cast<unsigned>(qhi - qlo + 1));
                if (q < kQCap) {
                    S.queue[q] = make_int3(i, qlo, qhi);
                    if (qhi - qlo >= kQShort) atomicAdd(&S.nlong, 1);  // finished by a whole warp
                } else if (*reinterpret_cast<volatile unsigned*>(&S.qwork) <= S.budget) {
                    for (int d = qlo; d <= qhi; ++d) smem_fmin(&S.keys[off + d], __dadd_rn(u0, kvalue<TAB, KS>(a, d)));
                } else {
                    S.abort = 1;  // a heavy tile: the queued runs already exceed the budget
                }
            }
        }
    }
    __syncthreads();
    if (S.abort || S.qwork > budget) return false;
    const int nq = min(S.nq, kQCap);
    if (nq) {
        // short queued runs one thread each, long ones one warp each
        unsigned qc = 0;
        for (int e = threadIdx.x; e < nq; e += kNT) {
            const int3 qe = S.queue[e];
            if (qe.z - qe.y < kQShort) {
                const double uy = a.ub[qe.x + 1];
                const int off = a.base + qe.x;
                qc += static_cast<unsigned>(qe.z - qe.y + 1);
                for (int d = qe.y; d <= qe.z; ++d) smem_fmin(&S.keys[off + d], __dadd_rn(uy, kvalue<TAB, KS>(a, d)));
            }
        }
        // (warps scan the queue for long runs only when there are any)
        for (int e = S.nlong ? warp : nq; e < nq; e += kNT / 32) {
            const int3 qe = S.queue[e];
            if (qe.z - qe.y < kQShort) continue;
            const double uy = a.ub[qe.x + 1];
            const int off = a.base + qe.x;
            if (lane == 0) qc += static_cast<unsigned>(qe.z - qe.y + 1);
            for (int d = qe.y + lane; d <= qe.z; d += 32) smem_fmin(&S.keys[off + d], __dadd_rn(uy, kvalue<TAB, KS>(a, d)));
        }
        if (qc) atomicAdd(&S.c_queued, qc);
        __syncthreads();
        if (threadIdx.x == 0) {
            S.c_qent += nq;
            S.nq = 0;
            S.nlong = 0;
        }
        __syncthreads();
    }
    return true;
}

// Loads of data the previous step's grid may still be finishing (chained mode):
// through L2, never a stale L1 line.
template <bool CHAIN, typename T>
__device__ __forceinline__ T xload(const T* p) {
    if constexpr (CHAIN) return __ldcg(p);
    else return *p;
}

__device__ __forceinline__ unsigned long long dbits(double x) {
    return static_cast<unsigned long long>(__double_as_longlong(x));
}

// K(d) anywhere in the window: the cached v_d table, or (a line whose window leaves the
// table) v_d computed with build_kernel's own two roundings (proj/src/scheme.cpp:79-80)
__device__ __forceinline__ double kdirect(const FastParams& p, int d, double drift) {
    const double v = static_cast<unsigned>(d + p.vofs) <= static_cast<unsigned>(2 * p.vofs)
                         ? __ldg(p.vtab + p.vofs + d)
                         : __ddiv_rn(__dmul_rn(static_cast<double>(d), p.eps), p.tau);
    return kval_v(v, drift, p.tau);
}

// The tile by the direct formula (proj/tests/unit_scheme.cpp:184-190) when the walk
// does not apply (oscillation gate failed, window outside the v_d table) or would cost
// more than the window (estimated candidates): keys[i] = min_w U(jlo + i - first - w) +
// K(first + w).  The tile's own outputs use K1's register-blocked sweep
// (csrc/direct_common.cuh): 8 outputs per thread, the window in chunks of kTW
// displacements staged in shared memory, one LDS per displacement and one add + one
// exact min per candidate; the three halo outputs are one warp each.
template <bool CHAIN, class KF>
__device__ void tile_direct(MainShared& S, const double* ul, int n, int j0, int Tl, int first, KF kf,
                            int64_t us = 1) {
    constexpr int R = kPer, L = kT + kTW;
    double* Us = reinterpret_cast<double*>(&S);
    double* Ks = Us + P8(L) + 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = 2 * n + 1;
    double hb = INFINITY;
    if (warp < 3) {
        int j = warp == 0 ? j0 - 1 : j0 + Tl + warp - 1;
        j = j < 0 ? j + n : (j >= n ? j - n : j);
        int y0 = (j - first) % n;
        if (y0 < 0) y0 += n;
        for (int w = lane; w < W; w += 32) {
            int y = (y0 - w) % n;
            if (y < 0) y += n;
            const double c = __dadd_rn(xload<CHAIN>(ul + y * us), kf(first + w));
            hb = c < hb ? c : hb;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const double c = __shfl_xor_sync(0xffffffffu, hb, o);
            hb = c < hb ? c : hb;
        }
    }
    double best[R];
#pragma unroll
    for (int r = 0; r < R; ++r) best[r] = INFINITY;
    for (int wc = 0; wc < W; wc += kTW) {
        __syncthreads();
        // sources y = j - first - w for j in [j0, j0 + kT), w in [wc, wc + kTW)
        int ym = (j0 - first - wc - kTW) % n;
        if (ym < 0) ym += n;
        for (int i = tid; i < L; i += kNT) {
            int y = ym + i;
            while (y >= n) y -= n;
            Us[P8(i)] = xload<CHAIN>(ul + y * us);
        }
        for (int s = tid; s < kTW; s += kNT) Ks[s] = wc + s < W ? kf(first + wc + s) : INFINITY;
        __syncthreads();
        const double* pa = Us + P8(tid * R + kTW);
        double A[R];
#pragma unroll
        for (int k = 0; k < R; ++k) A[k] = pa[k];
        const int send = min(kTW, (W - wc + R - 1) / R * R);
#pragma unroll 1
        for (int s0 = 0; s0 < send; s0 += R) {
            double B[R];
#pragma unroll
            for (int k = 0; k < R; ++k) B[k] = pa[-2 - k];
#pragma unroll
            for (int s = 0; s < R; ++s) {
                const double kw = Ks[s0 + s];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int idx = r - s;
                    const double val = idx >= 0 ? A[idx >= 0 ? idx : 0] : B[idx < 0 ? -idx - 1 : 0];
                    const double c = __dadd_rn(val, kw);
                    best[r] = c < best[r] ? c : best[r];
                }
            }
#pragma unroll
            for (int k = 0; k < R; ++k) A[k] = B[R - 1 - k];
            pa -= R + 1;
        }
    }
    __syncthreads();  // the staging area is dead: keys take the results
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = 1 + R * tid + r;
        if (i <= Tl) S.keys[i] = dbits(best[r]);
    }
    if (warp < 3 && lane == 0) S.keys[warp == 0 ? 0 : Tl + warp] = dbits(hb);
}

// LOB_FAST_STATS_CHECK (warp 0, all lanes): u changed since its statistics were taken when a
// sampled position differs bitwise; the statistics then do not describe u, and every tile of the
// line sees it and takes the direct formula (exact), counted.  Out of line: the unchecked setup
// keeps its registers.  Loads through L2 (a chained predecessor may still be finishing).
__device__ __noinline__ bool samples_differ(const double* ul, const double* samp, int n, unsigned long long* diag) {
    const int lane = threadIdx.x & 31;
    const int pos = static_cast<int>((static_cast<int64_t>(lane) * n) >> 5);
    const bool diff = __double_as_longlong(__ldcg(ul + pos)) != __double_as_longlong(__ldcg(samp + lane));
    const bool any = __any_sync(0xffffffffu, diff);
    if (any && lane == 0 && diag) atomicAdd(diag + 10, 1ull);
    return any;
}

// Per-line constants of the step (identical IEEE operations to the host's
// build_kernel for first/center; the tolerance only needs to be a bound).
__device__ __forceinline__ LineConst line_const(double drift, const FastParams& p) {
    const int64_t n = p.n;
    const double tau = p.tau, eps = p.eps, a = p.a;
    const int64_t center = llround(__ddiv_rn(__dmul_rn(tau, drift), eps));
    const int64_t first = center - n;
    const double uu = 1.1102230246251565e-16;
    const double dm = fmax(fabs(static_cast<double>(first)), fabs(static_cast<double>(first + 2 * n)));
    const double vmax = dm * eps / tau;
    const double kmag = tau * (0.5 * vmax * vmax + fabs(drift) * vmax);
    double delta = 2.0 * (32.0 * uu * kmag / a + 8.0 * uu * (2.0 * n + fabs(drift) * eps / a) + 1e-9);
    if (p.delta_override == p.delta_override) delta = p.delta_override;
    // the walk reads K through the cached v_d table: its window must lie inside it
    const bool intab = first >= -p.vofs && first + 2 * n <= p.vofs;
    LineConst c{};
    c.first = first;
    c.pe = __dmul_rn(drift, eps);
    const double pz = __dmul_rn(c.pe, p.ia);  // P eps / a
    c.hl = pz - (0.5 + delta);
    c.hr = pz + (0.5 + delta);
    c.drift = drift;
    if (intab) {
        const double kfirst = kval(p.vtab, p.vofs, first, drift, tau);
        const double klast = kval(p.vtab, p.vofs, first + 2 * n, drift, tau);
        double kmin = INFINITY;
        for (int64_t d = center - 2; d <= center + 2; ++d)
            if (d >= first && d <= first + 2 * n) kmin = fmin(kmin, kval(p.vtab, p.vofs, d, drift, tau));
        c.gap = fmin(kfirst, klast) - kmin;
    } else {
        c.gap = -INFINITY;  // never passes the gate: the line's tiles take the direct formula
    }
    return c;
}

// line_const for one warp (all lanes): the seven window values the gate needs are computed by
// seven lanes at once, each v_d by build_kernel's two roundings (the cached table's own values,
// build_vtab_kernel), so K2L's setup has no table round trip on its critical path.
__device__ __forceinline__ LineConst line_const_warp(double drift, const FastParams& p) {
    const int lane = threadIdx.x & 31;
    const int64_t n = p.n;
    const double tau = p.tau, eps = p.eps, a = p.a;
    const int64_t center = llround(__ddiv_rn(__dmul_rn(tau, drift), eps));
    const int64_t first = center - n;
    const double uu = 1.1102230246251565e-16;
    const double dm = fmax(fabs(static_cast<double>(first)), fabs(static_cast<double>(first + 2 * n)));
    const double vmax = dm * eps / tau;
    const double kmag = tau * (0.5 * vmax * vmax + fabs(drift) * vmax);
    double delta = 2.0 * (32.0 * uu * kmag / a + 8.0 * uu * (2.0 * n + fabs(drift) * eps / a) + 1e-9);
    if (p.delta_override == p.delta_override) delta = p.delta_override;
    const bool intab = first >= -p.vofs && first + 2 * n <= p.vofs;
    LineConst c{};
    c.first = first;
    c.pe = __dmul_rn(drift, eps);
    const double pz = __dmul_rn(c.pe, p.ia);
    c.hl = pz - (0.5 + delta);
    c.hr = pz + (0.5 + delta);
    c.drift = drift;
    // lanes 0..4: K(center - 2 .. center + 2) inside the window; lane 5: K(first); lane 6: K(last)
    const int64_t d = lane < 5 ? center - 2 + lane : (lane == 5 ? first : first + 2 * n);
    double kv = INFINITY;
    if (intab && lane < 7 && (lane >= 5 || (d >= first && d <= first + 2 * n)))
        kv = kval_v(__ddiv_rn(__dmul_rn(static_cast<double>(d), eps), tau), drift, tau);
    const double kfirst = __shfl_sync(0xffffffffu, kv, 5), klast = __shfl_sync(0xffffffffu, kv, 6);
    double km = lane < 5 ? kv : INFINITY;
#pragma unroll
    for (int o = 4; o; o >>= 1) km = fmin(km, __shfl_xor_sync(0xffffffffu, km, o));
    km = __shfl_sync(0xffffffffu, km, 0);
    c.gap = intab ? fmin(kfirst, klast) - km : -INFINITY;
    return c;
}

__global__ void line_setup_kernel(const double* __restrict__ drift_arr, int64_t lines, FastParams p,
                                  LineConst* __restrict__ lc) {
    const int64_t line = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (line >= lines) return;
    lc[line] = line_const(drift_arr[line], p);
}

// Per-line constants of a window-table step: one warp per line reduces the window's
// minimum and maximum |slope| (the gate and the search tolerance).
__global__ void line_setup_tab_kernel(const double* __restrict__ ktab, int64_t stride,
                                      const int64_t* __restrict__ first_arr, int64_t lines, int64_t n,
                                      LineConst* __restrict__ lc) {
    const int64_t line = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (line >= lines) return;
    const double* K = ktab + line * stride;
    double kmin = INFINITY, smx = 0.0;
    for (int64_t w = lane; w <= 2 * n; w += 32) {
        kmin = fmin(kmin, K[w]);
        if (w < 2 * n) smx = fmax(smx, fabs(__dsub_rn(K[w + 1], K[w])));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        kmin = fmin(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
        smx = fmax(smx, __shfl_xor_sync(0xffffffffu, smx, o));
    }
    if (lane) return;
    LineConst c{};
    const int64_t first = first_arr[line];
    c.first = first;
    c.kt = K - first;
    c.gap = fmin(K[0], K[2 * n]) - kmin;
    c.smax = smx;
    c.tol = 4.0 * 1.1102230246251565e-16;  // >= u/(1-u) on each side of the comparison, 2x spare
    c.sg0 = __dsub_rn(K[1], K[0]);
    const double sg1 = __dsub_rn(K[2 * n], K[2 * n - 1]);
    c.sgi = sg1 > c.sg0 ? static_cast<double>(2 * n - 1) / (sg1 - c.sg0) : 0.0;
    c.k0 = K[0];
    c.kmid = K[n];
    c.kend = K[2 * n];
    lc[line] = c;
}

// Main K2 kernel: one CTA = (tile of kT outputs, line); grid (tiles, lines).
// All index arithmetic is 32-bit (n <= 2^29); "unrolled" source/output
// indices y, j may lie in (-3n, 3n) and are reduced mod n only on access.
// TMA: rows may be bulk-copied (even n, aligned).  CHAIN: the previous operation on
// the stream was the previous step on this workspace (and it released); a tile waits
// only for the warps of its own line at that step (per-line release counters, `need`)
// instead of the whole previous grid, so consecutive steps overlap.  RELEASE: count
// this step's warps into the per-line counters for a chained successor.
//
// Diagnostic counters (diag[]): [0] outputs no candidate reached (recomputed by the
// direct scan), [1] sources scanned, [2] fold ranges, [3] long plain runs, [4] tiles,
// [5] tiles whose K range did not fit the shared stage, [6] sum of the tiles' K range
// lengths, [7] tiles by the direct formula because the oscillation gate failed,
// [8] tiles by the direct formula because the walk's estimated candidates exceeded the
// window's, [9] chained-wait timeouts (a misused LOB_FAST_CHAINED), [10] warps whose
// fold queue overflowed.
template <bool TAB, bool TMA, bool CHAIN, bool RELEASE>
__global__ void __launch_bounds__(kNT, LOB_FAST_MINB) fast_kernel(
    const double* __restrict__ u, double* __restrict__ out, const LineConst* __restrict__ lcs,
    const double* __restrict__ tv, int64_t tv_stride, int64_t* __restrict__ blocks_out,
    unsigned long long* __restrict__ diag, FastParams p, FastBuffers b, unsigned* __restrict__ done,
    unsigned need, double* __restrict__ dpart) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    MainShared& S = *reinterpret_cast<MainShared*>(smem_raw);

    const int n = static_cast<int>(p.n);
    const int tiles = static_cast<int>(p.tiles), subs = static_cast<int>(p.subs);
    const int tile = blockIdx.x;
    const int64_t line = grid_line();
    if (line >= p.lines) return;  // (uniform per CTA: before any barrier)
    const int j0 = tile * kT;
    const int Tl = min(kT, n - j0);
    const int jlo = j0 - 1;     // outputs evaluated: jlo .. jlo + jspan (unrolled)
    const int jspan = Tl + 2;
    const int jhi = jlo + jspan;
    // TMA bulk copies (16-byte granules: even n, aligned rows; TMA) for lines long enough that
    // a chunk takes a few wrapped segments; else a cooperative load
    const bool big = TMA && n >= 256;
    const double* ul = u + line * p.n;
    LineConst lc = lcs[line];
    // carried line constants (LOB_FAST_STATS_VALID) must describe the caller's current drift /
    // window: a mismatch (another table at a reused address, a drift changed in place) takes
    // the direct formula with the current inputs (exact) and is counted
    bool stale;
    if constexpr (TAB) {
        const double* Kl = p.ktab + line * p.kstride;
        const long long f = __ldg(p.kfirst + line);
        stale = f != lc.first || __double_as_longlong(__ldg(Kl)) != __double_as_longlong(lc.k0) ||
                __double_as_longlong(__ldg(Kl + n)) != __double_as_longlong(lc.kmid) ||
                __double_as_longlong(__ldg(Kl + 2 * n)) != __double_as_longlong(lc.kend);
        if (stale) {
            lc.first = f;
            lc.kt = Kl - f;
        }
    } else {
        const double d = __ldg(p.drift_arr + line);
        stale = __double_as_longlong(d) != __double_as_longlong(lc.drift);
        if (stale) {
            lc.drift = d;
            lc.first = llround(__ddiv_rn(__dmul_rn(p.tau, d), p.eps)) - p.n;  // line_setup_kernel's formula
        }
    }
    const double tau = p.tau, ia = p.ia, hl = lc.hl, hr = lc.hr;
    const int first = static_cast<int>(lc.first);
    const int dmin_w = first + 1, dmax_w = first + 2 * n - 1;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // K(d) anywhere in the window: the line's table (TAB) or build_kernel's formula over v_d
    auto kf = [&](int d) -> double {
        if constexpr (TAB) return __ldg(lc.kt + d);
        else return kdirect(p, d, lc.drift);
    };
    // window slopes sigma(d) = K(d+1) - K(d) from global memory (table mode)
    auto sigg = [&](int d) -> double { return __dsub_rn(__ldg(lc.kt + d + 1), __ldg(lc.kt + d)); };

    // programmatic dependent launch: the next step's grid may start its prologue once
    // every CTA of this one is running; this grid waits for the previous one (its u,
    // statistics and the buffers it still reads) before touching global memory
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    {
        // +inf sentinels for keys[0 .. jspan] (jspan + 1 <= kT + 3 <= kT + 4 slots, 16-byte stores)
        ulonglong2* k2 = reinterpret_cast<ulonglong2*>(S.keys);
#pragma unroll
        for (int i = tid; i < (kT + 4) / 2; i += kNT) k2[i] = make_ulonglong2(kInfBits, kInfBits);
    }
    if constexpr (CHAIN) {
        if (warp == 0) {
            if (lane == 0) {
                unsigned v;
                const long long t0 = clock64();
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(done + line) : "memory");
                    if (v >= need) break;
                    __nanosleep(128);
                    // a misused LOB_FAST_CHAINED (the previous step is not on this stream):
                    // counted and reported by the host, never a hang or a trap
                    if (clock64() - t0 > (1ll << 34)) {
                        atomicAdd(diag + 9, 1ull);
                        break;
                    }
                }
                asm volatile("fence.proxy.async.global;" ::: "memory");  // for the TMA reads of u
            }
            __syncwarp();
        }
    } else {
        asm volatile("griddepcontrol.wait;" ::: "memory");
    }
    // reset the line statistics buffer two steps ahead
    if (tile == 0 && tid < 4) b.line_reset[line * 4 + tid] = (tid & 1) ? 0ull : ~0ull;

    // ---- warp 0: line gate, candidate sub-tiles, work estimate, first TMA issue ----
    if (warp == 0) {
        const unsigned long long* L = b.line_in + line * 4;
        const double umin = dkey_inv(xload<CHAIN>(L + 0)), umax = dkey_inv(xload<CHAIN>(L + 1));
        const double smin = dkey_inv(xload<CHAIN>(L + 2)), smax = dkey_inv(xload<CHAIN>(L + 3));
        int DLg = dmin_w, DRg = dmax_w;
        // window-edge displacements cannot hold a minimiser when the line's oscillation
        // max u - min u is below the window's edge gap min(K(first), K(last)) - min K
        // (the exact extremes are absent, NaN, when the previous step did not collect them)
        const double osc = __dsub_rn(umax, umin);
        const double loose = 0.5 * static_cast<double>(n) * fmax(fabs(smin), fabs(smax));
        const bool exact_ok = isfinite(osc) && osc * (1.0 + 1e-12) < lc.gap * (1.0 - 1e-12);
        const bool loose_ok = loose * (1.0 + 1e-12) < lc.gap * (1.0 - 1e-12);
        bool okl = !stale && (exact_ok || loose_ok) && isfinite(smin) && isfinite(smax) && n >= 3;
        if (p.check && samples_differ(ul, b.samp_in + line * kSamp, n, diag)) okl = false;
        // this step's epilogue collects the exact extremes of u^{n+1} unless the cheap bound of
        // u^n passes with a factor 2 to spare (the same decision in every tile of the line)
        if (lane == 0) S.osc_exact = !(loose * 2.0 < lc.gap) || !isfinite(loose);
        const bool gate = okl;
        if (stale && lane == 0 && diag) atomicAdd(diag + 11, 1ull);
        if (okl) {
            if constexpr (TAB) {
                int dl, dr;
                tab_interval(sigg, lc, smin, smax, dmin_w, dmax_w, dl, dr);
                DLg = max(dl, dmin_w);
                DRg = min(dr, dmax_w);
            } else {
                DLg = max(__double2int_ru(__fma_rn(smin, ia, hl)), dmin_w);
                DRg = min(__double2int_rd(__fma_rn(smax, ia, hr)), dmax_w);
            }
            okl = DLg <= DRg;
        }
        int ya = INT_MAX, yb = INT_MIN, dlo = INT_MAX, dhi = INT_MIN;
        int Q0 = 0, Q1 = -1;
        // sub-tile Q of the unrolled source axis: its sources [ys, ye] and whether
        // their slope-implied displacements reach this tile's outputs
        // sub-tile Q = k subs + q of the unrolled axis (k periods, q < subs); reach_kq takes the split
        auto reach_kq = [&](int k, int q, int& ys, int& ye, int& dl, int& dr) {
            const double2 sb = xload<CHAIN>(b.sub_in + line * p.subs + q);
            ys = k * n + q * kG;
            ye = ys + min(kG, n - q * kG) - 1;
            if constexpr (TAB) {
                tab_interval(sigg, lc, sb.x, sb.y, DLg, DRg, dl, dr);
                dl = max(dl, DLg);
                dr = min(dr, DRg);
            } else {
                dl = max(__double2int_ru(__fma_rn(sb.x, ia, hl)), DLg);
                dr = min(__double2int_rd(__fma_rn(sb.y, ia, hr)), DRg);
            }
            return dl <= dr && ys + dl <= jhi && ye + dr >= jlo;
        };
        auto reach = [&](int Q, int& ys, int& ye, int& dl, int& dr, int& q) {
            const int k = Q >= 0 ? Q / subs : -((subs - 1 - Q) / subs);
            q = Q - k * subs;
            const double2 sb = xload<CHAIN>(b.sub_in + line * p.subs + q);
            ys = k * n + q * kG;
            ye = ys + min(kG, n - q * kG) - 1;
            if constexpr (TAB) {
                tab_interval(sigg, lc, sb.x, sb.y, DLg, DRg, dl, dr);
                dl = max(dl, DLg);
                dr = min(dr, DRg);
            } else {
                dl = max(__double2int_ru(__fma_rn(sb.x, ia, hl)), DLg);
                dr = min(__double2int_rd(__fma_rn(sb.y, ia, hr)), DRg);
            }
            return dl <= dr && ys + dl <= jhi && ye + dr >= jlo;
        };
        if (okl) {
            // candidate sub-tiles: unrolled sources y in [jlo - DRg, jhi - DLg]
            const int y0 = jlo - DRg, y1 = jhi - DLg;
            int k0 = 0;
            while (y0 - k0 * n < 0) --k0;
            while (y0 - k0 * n >= n) ++k0;
            Q0 = k0 * subs + (y0 - k0 * n) / kG;
            int k1 = k0;
            while (y1 - k1 * n >= n) ++k1;
            Q1 = k1 * subs + (y1 - k1 * n) / kG;
            // lane l takes Q0 + l, Q0 + l + 32, ...: the (period, sub-tile) split advanced without a
            // division per sub-tile (k0 periods and q0 = Q0 - k0 subs from the loop above)
            int kq = k0, qq = Q0 - k0 * subs + lane;
            while (qq >= subs) {
                qq -= subs;
                ++kq;
            }
            for (int Q = Q0 + lane; Q <= Q1; Q += 32) {
                int ys, ye, dl, dr;
                const bool hit = reach_kq(kq, qq, ys, ye, dl, dr);
                qq += 32;
                while (qq >= subs) {
                    qq -= subs;
                    ++kq;
                }
                if (hit) {
                    ya = min(ya, ys);
                    yb = max(yb, ye);
                    dlo = min(dlo, max(dl, jlo - ye));
                    dhi = max(dhi, min(dr, jhi - ys));
                }
            }
            ya = __reduce_min_sync(0xffffffffu, ya);
            yb = __reduce_max_sync(0xffffffffu, yb);
            dlo = __reduce_min_sync(0xffffffffu, dlo);
            dhi = __reduce_max_sync(0xffffffffu, dhi);
        }
        // the walk when the gate holds, else the direct formula
        const int mode = (okl && ya <= yb) ? kModeWalk : kModeDirect;
        if (mode == kModeWalk) {
            // a wide tile (displacement range beyond the staged K buffer: a shock in a nearby
            // sub-tile) scans only the runs of reaching sub-tiles, not the gaps between them
            int nr = 1;
            if (dhi - dlo + 2 > LOB_WIDE_RANGE && Q1 - Q0 < 64) {
                unsigned long long hmask = 0;
                for (int Qb = Q0; Qb <= Q1; Qb += 32) {
                    int ys, ye, dl, dr, q;
                    const bool hit = Qb + lane <= Q1 && reach(Qb + lane, ys, ye, dl, dr, q);
                    hmask |= static_cast<unsigned long long>(__ballot_sync(0xffffffffu, hit)) << (Qb - Q0);
                }
                if (lane == 0) {
                    nr = 0;
                    unsigned long long m = hmask;
                    while (m) {
                        const int b0 = __ffsll(static_cast<long long>(m)) - 1;
                        const unsigned long long inv = ~(m >> b0);
                        const int len = inv ? __ffsll(static_cast<long long>(inv)) - 1 : 64 - b0;
                        int ys, ye, ys2, ye2, dl, dr, q;
                        reach(Q0 + b0, ys, ye, dl, dr, q);
                        reach(Q0 + b0 + len - 1, ys2, ye2, dl, dr, q);
                        if (nr < kRuns) {
                            S.rs[nr] = ys;
                            S.re[nr] = ye2;
                            ++nr;
                        } else {
                            S.re[kRuns - 1] = ye2;
                        }
                        m = b0 + len >= 64 ? 0ull : (m >> (b0 + len)) << (b0 + len);
                    }
                }
            } else if (lane == 0) {
                S.rs[0] = ya;
                S.re[0] = yb;
            }
            if (lane == 0) S.nruns = nr;
        }
        if (lane == 0) {
            S.mode = mode;
            S.gate = gate;
            S.DLg = DLg;
            S.DRg = DRg;
            S.ya = ya;
            S.yb = yb;
            S.dlo = dlo;
            S.dhi = dhi;
            S.nq = 0;
            S.nlong = 0;
            S.abort = 0;
            S.qwork = 0;
            // queued candidates beyond this cost more than the direct formula over the window
            const double bud = LOB_HEAVY * static_cast<double>(jspan + 1) * static_cast<double>(2 * n + 1);
            S.budget = bud > 4.0e9 ? 4000000000u : static_cast<unsigned>(bud);
            S.c_src = S.c_queued = S.c_qent = 0;
            if (mode == kModeWalk) {
                mbar_init(&S.mbar, 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                if (big) {
                    // first source chunk + (mechanical) the tile's v_d range, in flight across the barrier
                    const int vd0 = dlo - ((dlo + static_cast<int>(p.vofs)) & 1);
                    const int vcnt = (dhi - vd0 + 2) & ~1;
                    issue_chunk(S, ul, n, ya, min(kC, S.re[0] - ya + 1),
                                (!TAB && vcnt <= kVCap) ? p.vtab + p.vofs + vd0 : nullptr, vcnt);
                }
            }
        }
    }
    __syncthreads();  // gate, mode, ranges, mbarrier initialised
    const int mode = S.mode;
    const bool osc_exact = S.osc_exact;  // read before the epilogue reuses the shared layout

    bool walk = mode == kModeWalk;
    if (walk) {
        const int ya = S.ya;
        const int dlo_t = S.dlo, dhi_t = S.dhi;
        // K(d) = tau*((0.5 v)v - P v): staged in shared memory (TMA'd v_d, converted
        // in place) when the tile's displacement range fits, else from the global v_d table.
        // Table mode: K(dlo - 1 .. dhi + 1) (the slope search reads sigma one step outside
        // [dlo, dhi]) copied from the line's window, else read from it.
        const int vd0 = TAB ? dlo_t - 2 : dlo_t - ((dlo_t + static_cast<int>(p.vofs)) & 1);
        const int vcnt = TAB ? ((dhi_t + 2 - vd0 + 1) + 1) & ~1 : (dhi_t - vd0 + 2) & ~1;
        const bool kstage = (TAB || big) && vcnt <= kVCap;
        const double* gvt = TAB ? lc.kt : p.vtab + p.vofs;
        const double* skt = S.vbuf - vd0;
        const double kdrift = lc.drift;
        const unsigned budget = S.budget;
        if (tid == 0 && diag) {
            atomicAdd(diag + 5, kstage ? 0ull : 1ull);
            atomicAdd(diag + 6, static_cast<unsigned long long>(vcnt));
        }
        // ---- sources in chunks of kC ----
        unsigned mphase = 0;
        const int nruns = S.nruns;
        for (int run = 0, yc = ya, yr = S.re[0]; run < nruns;) {
            const int clen = min(kC, yr - yc + 1);
            const int base = yc - jlo;  // output index of source i at d: base + i + d
            int sh = 0;
            if (big) {
                sh = wrap_idx(yc - 1, n) & 1;
                if (yc != ya && tid == 0) issue_chunk(S, ul, n, yc, clen, nullptr, 0);
                if (warp == 0) mbar_wait(&S.mbar, mphase);
                mphase ^= 1u;
                __syncthreads();
                if (yc == ya && kstage && !TAB) {
                    for (int i = tid; i < vcnt; i += kNT) S.vbuf[i] = kval_v(S.vbuf[i], kdrift, tau);
                    __syncthreads();
                }
            } else {
                const int bm = wrap_idx(yc - 1, n);
                for (int i = tid; i < clen + 2; i += kNT) {
                    int y = bm + i;
                    while (y >= n) y -= n;
                    S.ubuf[i] = CHAIN ? __ldcg(ul + y) : __ldg(ul + y);
                }
                __syncthreads();
            }
            if (TAB && yc == ya && kstage) {
                // the window's K values of the tile's displacement range (clamped to the window)
                for (int i = tid; i < vcnt; i += kNT) S.vbuf[i] = __ldg(lc.kt + min(max(vd0 + i, first), first + 2 * n));
                __syncthreads();
            }
            const double* ub = S.ubuf + sh;
            if (tid == 0) S.c_src += static_cast<unsigned>(clen);
            const ChunkArgs ca{ub, clen, base, jspan, ia, hl, hr, dlo_t, dhi_t, skt, gvt, kdrift, tau, &lc};
            walk = kstage ? process_chunk<TAB, true>(S, ca, budget) : process_chunk<TAB, false>(S, ca, budget);
            if (!walk) break;  // the walk would cost more than the window: the direct formula
            yc += clen;
            if (yc > yr && ++run < nruns) {
                yc = S.rs[run];
                yr = S.re[run];
            }
        }
        if (!walk && tid == 0 && diag) atomicAdd(diag + 8, 1ull);
    } else if (tid == 0 && diag) {
        atomicAdd(diag + 7, 1ull);
    }
#if LOB_TILE_DIRECT
    if (!walk) tile_direct<CHAIN>(S, ul, n, j0, Tl, first, kf);
#endif
    __syncthreads();

    // ---- epilogue: u^{n+1} = best - tv; the direct scan where nothing landed ----
    // Thread t owns outputs j0 + t + kNT*m (vals index 1 + t + kNT*m);
    // threads 0..2 also the halo outputs jlo, j0+Tl, j0+Tl+1.
    const double* tvl = tv ? tv + line * tv_stride : nullptr;
    // tau*V at output j: the table, the separable descriptor, or 0 (x - 0 == x)
    const double sa1l = p.sa1 ? __ldg(p.sa1 + line) : 0.0;
    auto tvat = [&](int j) -> double {
        if (tvl) return __ldg(tvl + j);
        if (p.sa1) return __dmul_rn(tau, __dadd_rn(__dmul_rn(sa1l, __ldg(p.sa2 + j)), p.sb));
        return 0.0;
    };
    double* vals = S.ubuf;  // reuse: vals[i] = u^{n+1}(jlo + i), i = 0 .. Tl+2
    // direct scan of the full window (proj/tests/unit_scheme.cpp:184-190) for outputs no
    // interval reached (never, when the statistics describe u); one copy of the loop
    auto scan = [&](int j) -> double {
        if (diag) atomicAdd(diag, 1ull);
        double best = INFINITY;
        int y = (j - first) % n;
        if (y < 0) y += n;
        for (int w = 0; w <= 2 * n; ++w) {
            const double c2 = __dadd_rn(xload<CHAIN>(ul + y), kf(first + w));
            best = c2 < best ? c2 : best;
            y = y == 0 ? n - 1 : y - 1;
        }
        return best;
    };
    auto epilogue = [&](auto full_tile) {
        constexpr bool FULL = decltype(full_tile)::value;  // a whole tile: no bounds checks
        double tvv[kPer + 1];
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
            const int i = 1 + tid + kNT * m;
            tvv[m] = (FULL || i <= Tl) ? tvat(j0 + i - 1) : 0.0;
        }
        const int ih = tid == 0 ? 0 : Tl + tid;  // halo vals index (tid < 3)
        int jh = jlo + ih;
        jh += jh < 0 ? n : 0;
        jh -= jh >= n ? n : 0;
        tvv[kPer] = tid < 3 ? tvat(jh) : 0.0;
        double* ol = out + line * p.n + j0;
        unsigned miss = 0;
        // best - tv with tv = 0 when there is no potential: the same double (x - 0 == x, -0 - 0 == -0)
        const int pb = P8(1 + tid);  // P8(1 + tid + kNT m) = pb + (kNT + kNT / 8) m
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
            const int i = 1 + tid + kNT * m;
            if (FULL || i <= Tl) {
                const unsigned long long kk = S.keys[i];
                // an empty slot (+inf) is stored too and rewritten by the cold scan below
                const double o = __dsub_rn(__longlong_as_double(static_cast<long long>(kk)), tvv[m]);
                vals[pb + (kNT + kNT / 8) * m] = o;
                ol[i - 1] = o;
                miss |= static_cast<unsigned>(kk == kInfBits) << m;
            }
        }
        if (tid < 3) {
            const unsigned long long kk = S.keys[ih];
            if (kk != kInfBits)
                vals[P8(ih)] = __dsub_rn(__longlong_as_double(static_cast<long long>(kk)), tvv[kPer]);
            else
                miss |= 1u << kPer;
        }
        while (miss) {  // cold
            const int m = __ffs(miss) - 1;
            miss &= miss - 1;
            const int i = m < kPer ? 1 + tid + kNT * m : ih;
            const int j = m < kPer ? j0 + i - 1 : jh;
            const double best = scan(j);
            const double o = __dsub_rn(best, tvat(j));
            vals[P8(i)] = o;
            if (m < kPer) ol[i - 1] = o;
        }
    };
    if (Tl == kT)
        epilogue(std::true_type{});
    else
        epilogue(std::false_type{});
    __syncthreads();
    if (dpart) {
        // evolve's per-step drift (proj/src/scheme.cpp:244-250): this tile's sum of u^{n+1} - u^n
        // (the tile's u^{n+1} is in vals; u^n from global, coalesced); summed per line in tile order
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
            const int i = 1 + tid + kNT * m;
            if (i <= Tl) acc += vals[P8(i)] - xload<CHAIN>(ul + j0 + i - 1);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        double* red = reinterpret_cast<double*>(S.queue);  // the queue is dead after the emission
        if (lane == 0) red[warp] = acc;
        __syncthreads();
        if (tid == 0) {
            double sum = 0.0;
            for (int w = 0; w < kNT / 32; ++w) sum += red[w];
            dpart[line * tiles + tile] = sum;
            if (p.dcount) {
                // the last tile of the line to arrive: the line's drift, partials in tile order (the
                // drift_tiles_kernel's sum, so consecutive steps need no kernel in between)
                __threadfence();
                const unsigned old = atomicAdd(p.dcount + line, 1u);
                if (old % static_cast<unsigned>(tiles) == static_cast<unsigned>(tiles - 1)) {
                    __threadfence();
                    double tot = 0.0;
                    for (int t = 0; t < tiles; ++t) tot += __ldcg(dpart + line * tiles + t);
                    if (p.drift_out) p.drift_out[line] = tot / static_cast<double>(n);
                    if (!isfinite(tot) && p.halt) atomicMin(p.halt, p.dstep);
                }
            }
        }
    }
    if (tid == 0 && diag) {
        if (mode == kModeWalk) {
            atomicAdd(diag + 1, static_cast<unsigned long long>(S.c_src));
            atomicAdd(diag + 2, static_cast<unsigned long long>(S.c_queued));
            atomicAdd(diag + 3, static_cast<unsigned long long>(S.c_qent));
        }
        atomicAdd(diag + 4, 1ull);
    }
    // the samples the next step's LOB_FAST_STATS_CHECK compares its input with
    if (p.samples && tid < kSamp) {
        const int pos = static_cast<int>((static_cast<int64_t>(tid) * n) >> 5);
        if (pos >= j0 && pos < j0 + Tl) b.samp_out[line * kSamp + tid] = vals[P8(pos - j0 + 1)];
    }
    if (Tl == kT && j0 + kT <= n - 1)
        tile_stats<true>(vals, Tl, j0, line, tile, p, b, S.epi(), g_fsm_lut2, osc_exact);
    else
        tile_stats<false>(vals, Tl, j0, line, tile, p, b, S.epi(), g_fsm_lut2, osc_exact);
    // block count of the INPUT u (decompose on the closed period): warp 0 of
    // the line's first tile composes the tile summaries
    if (blocks_out && tile == 0 && warp == 0) {
        int q = 0;
        int64_t em = 0;
        for (int t0 = 0; t0 < tiles; t0 += 32) {
            const unsigned long long mine =
                t0 + lane < tiles ? xload<CHAIN>(b.fsm_in + line * p.tiles + t0 + lane) : fsm_identity();
            const int cnt = min(32, tiles - t0);
            for (int k = 0; k < cnt; ++k) {
                const unsigned long long f = __shfl_sync(0xffffffffu, mine, k);
                em += (f >> (16 + 16 * q)) & 0xffff;
                q = static_cast<int>((f >> (2 * q)) & 3);
            }
        }
        if (lane == 0) blocks_out[line] = 1 + em;
    }
    // release this warp's share of the tile to the next step's tiles of the line: a
    // gpu-scope release reduction by one lane, cumulative over the warp's writes (no CTA
    // barrier: warps retire independently; the line is done at kNT/32 * tiles counts)
    if constexpr (RELEASE) {
        __syncwarp();
        if (lane == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(done + line) : "memory");
    }
}


// ---- K2L: one step of short lines, one CTA per whole line ---------------------
// For n <= kT the whole line is one tile, so the statistics K2 carries between steps
// (sub-tile slope bounds, line extremes) are computed from the line itself: each thread
// holds kPer samples in registers, coarse order-preserving keys of u and of its slopes are
// reduced with REDUX (an enclosure: the oscillation gate and the displacement range
// [DLg, DRg] are conservative), the unrolled source range is written into the source
// buffer straight from the registers, and the candidate emission, the direct fallbacks and
// the epilogue are fast_kernel's.  No workspace statistics are read or written.
// Load modes: a row of u; column l of an n x n row-major tensor by strided loads, by a
// cluster exchange through distributed shared memory, or by 2-D TMA tensor-map copies
// (boxes of 2 columns x 256 rows, cp.async.bulk.tensor, the column picked out of the pair);
// store modes: a row, a column (strided), a cluster exchange.  The 2-D split step sweeps
// axis 0 as columns (proj/src/splitting.cpp:67-76 gathers and scatters them).
// Outputs follow fast_kernel's slot convention (slot i = output i - 1; slots 0 and n + 1
// are halo outputs nobody reads).
struct LineShared {  // overlays S.vbuf before the K staging
    unsigned kred[4][kNT / 32];
    double hl, hr, gap, drift;
    long long first;
};
static_assert(sizeof(LineShared) <= sizeof(double) * kVCap, "line scratch fits vbuf");
static_assert(kPer * kNT == kT, "one register sample per thread and kNT outputs");

constexpr int kLC = 8;  // CTAs (= adjacent columns) per cluster of the column-exchange variant
constexpr int kLdRow = kLineRow, kLdCol = kLineCol, kLdClu = kLineClu, kLdTma = kLineTma;
constexpr int kStRow = kLineRow, kStCol = kLineCol, kStClu = kLineClu;
constexpr int kTmaRows = 256;  // rows per TMA box (2 columns x 256 rows = 4 KB)
static_assert(offsetof(MainShared, queue) >= static_cast<size_t>(kT) * 16, "TMA landing zone below the queue");

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
        : "memory");
}

template <int LD, int ST>
__global__ void __launch_bounds__(kNT, LOB_FAST_MINB) line_kernel(const double* __restrict__ u, double* __restrict__ out,
                                                                  const double* __restrict__ drift_arr,
                                                                  const double* __restrict__ tv, int64_t tv_stride,
                                                                  unsigned long long* __restrict__ diag, FastParams p,
                                                                  const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem_line[];  // 128-byte aligned: TMA tensor copies land here
    unsigned char* smem_raw = smem_line;
    MainShared& S = *reinterpret_cast<MainShared*>(smem_raw);
    LineShared& L = *reinterpret_cast<LineShared*>(S.vbuf);
    const int n = static_cast<int>(p.n);
    const int64_t line = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t is = LD == kLdRow ? 1 : p.n, os = ST == kStCol ? p.n : 1;
    const double* ul = LD == kLdRow ? u + line * p.n : u + line;
    double* ol = ST == kStRow ? out + line * p.n : out + line;
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if constexpr (LD == kLdTma) {
        if (tid == 0) {
            unsigned long long* bar = reinterpret_cast<unsigned long long*>(S.queue);
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
        }
        __syncthreads();
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    // the line's drift, in flight with the line's samples (warp 0 derives the line constants)
    const double ldrift = warp == 0 ? __ldg(drift_arr + line) : 0.0;
    // the line in the middle of the source buffer (Ub[j] = U(j), j < n <= kT), so the unrolled source
    // range needs only its wrapped halos filled; the keys are initialised meanwhile
    constexpr int kUbLen = kC + 8;
    const int H0 = (kUbLen - n) / 2;
    double* Ub = S.ubuf + H0;
    bool line_bulk = false;
    auto init_keys = [&]() {
        ulonglong2* k2 = reinterpret_cast<ulonglong2*>(S.keys);
        for (int i = tid; i < (kT + 4) / 2; i += kNT) k2[i] = make_ulonglong2(kInfBits, kInfBits);
    };
    if constexpr (LD == kLdClu) {
        init_keys();
        // a cluster of kLC CTAs holds kLC adjacent columns c0 .. c0 + kLC - 1; CTA r reads rows
        // [r n/kLC, (r+1) n/kLC) of all kLC columns (64-byte row segments) and stores each value
        // into its column's CTA through distributed shared memory
        cg::cluster_group cluster = cg::this_cluster();
        const int r = static_cast<int>(cluster.block_rank());
        const int64_t c0 = line - r;
        const int rows = n / kLC;
        cluster.sync();  // every CTA of the cluster runs: its shared memory may be written
        for (int e = tid; e < rows * kLC; e += kNT) {
            const int row = r * rows + e / kLC, col = e % kLC;
            *cluster.map_shared_rank(Ub + row, col) = u[static_cast<int64_t>(row) * p.n + c0 + col];
        }
        cluster.sync();
    } else if (LD == kLdTma && (smem_u32(smem_raw) & 127u) != 0u) {
        // (a TMA tensor copy needs a 128-byte aligned destination: strided loads otherwise)
        init_keys();
        for (int j = tid; j < n; j += kNT) Ub[j] = ul[j * is];
    } else if constexpr (LD == kLdTma) {
        // columns (line & ~1, line | 1) x all rows in boxes of kTmaRows rows into the landing zone
        // (land[2 j + pick] = U(j), over the keys and the start of the source buffer), then
        // compacted into the source buffer through registers
        unsigned long long* bar = reinterpret_cast<unsigned long long*>(S.queue);
        const double* land = reinterpret_cast<const double*>(smem_raw);
        if (tid == 0) {
            mbar_expect_tx(bar, static_cast<unsigned>((n + kTmaRows - 1) / kTmaRows * kTmaRows) * 16u);
            for (int r0 = 0; r0 < n; r0 += kTmaRows)
                tma_load_2d(smem_raw + static_cast<size_t>(r0) * 16, &tmap, static_cast<int>(line & ~1ll), r0, bar);
        }
        mbar_wait(bar, 0);
        const int pick = static_cast<int>(line & 1);
        double v[kPer];
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
            const int j = tid + kNT * m;
            v[m] = j < n ? land[2 * j + pick] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
            const int j = tid + kNT * m;
            if (j < n) Ub[j] = v[m];
        }
        init_keys();
    } else {
        // a row of even length on a 16-byte boundary: one TMA bulk copy (cp.async.bulk) issued by
        // thread 0 while every thread initialises the keys; else 8-byte loads through registers
        if constexpr (LD == kLdRow)
            line_bulk = n >= 256 && (n & 1) == 0 && (H0 & 1) == 0 && (reinterpret_cast<uintptr_t>(ul) & 15u) == 0;
        if (line_bulk) {
            if (tid == 0) {
                mbar_init(&S.mbar, 1);
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
                fence_proxy_async();
                mbar_expect_tx(&S.mbar, static_cast<unsigned>(n) * 8u);
                tma_load_1d(Ub, ul, static_cast<unsigned>(n) * 8u, &S.mbar);
            }
            init_keys();
        } else {
            init_keys();
            for (int j = tid; j < n; j += kNT) Ub[j] = ul[j * is];
        }
    }
    double* U = Ub;
    if (warp == 0) {
        const LineConst c = line_const_warp(ldrift, p);
        if (lane == 0) {
            L.hl = c.hl;
            L.hr = c.hr;
            L.gap = c.gap;
            L.drift = c.drift;
            L.first = c.first;
        }
        if (line_bulk) {
            __syncwarp();  // thread 0 initialised the barrier
            mbar_wait(&S.mbar, 0);
            if (lane == 0) Ub[n] = Ub[0];  // the seam sample, for the slope of the last segment
        }
    }
    if (!line_bulk && tid == 0) Ub[n] = Ub[0];  // (thread 0 staged U(0) itself, or a cluster barrier ordered it)
    __syncthreads();
    // enclosures of u and of its slopes s(j) = U(j+1) - U(j) (periodic): coarse order-preserving
    // keys (within 2^-20 relative, tile_stats' keys) reduced with REDUX
    {
        unsigned kmn = 0xffffffffu, kmx = 0u, hmn = 0xffffffffu, hmx = 0u;
#pragma unroll 4
        for (int j = tid; j < n; j += kNT) {
            const double uj = U[j];
            const unsigned ks = hkey(__dsub_rn(U[j + 1], uj)), ku = hkey(uj);
            kmn = min(kmn, ks);
            kmx = max(kmx, ks);
            hmn = min(hmn, ku);
            hmx = max(hmx, ku);
        }
        kmn = __reduce_min_sync(0xffffffffu, kmn);
        kmx = __reduce_max_sync(0xffffffffu, kmx);
        hmn = __reduce_min_sync(0xffffffffu, hmn);
        hmx = __reduce_max_sync(0xffffffffu, hmx);
        if (lane == 0) {
            L.kred[0][warp] = kmn;
            L.kred[1][warp] = kmx;
            L.kred[2][warp] = hmn;
            L.kred[3][warp] = hmx;
        }
    }
    __syncthreads();
    const int first = static_cast<int>(L.first);
    const double drift = L.drift, tau = p.tau, ia = p.ia, hl = L.hl, hr = L.hr;
    const int dmin_w = first + 1, dmax_w = first + 2 * n - 1;
    constexpr int jlo = -1;
    const int jspan = n + 1;
    if (warp == 0) {
        const bool in = lane < kNT / 32;
        const unsigned a0 = __reduce_min_sync(0xffffffffu, in ? L.kred[0][lane] : 0xffffffffu);
        const unsigned a1 = __reduce_max_sync(0xffffffffu, in ? L.kred[1][lane] : 0u);
        const unsigned b0 = __reduce_min_sync(0xffffffffu, in ? L.kred[2][lane] : 0xffffffffu);
        const unsigned b1 = __reduce_max_sync(0xffffffffu, in ? L.kred[3][lane] : 0u);
        if (lane == 0) {
            // window-edge displacements cannot hold a minimiser when max u - min u (here an upper
            // bound) is below the window's edge gap (fast_kernel's gate)
            const double smin = hkey_lower(a0), smax = hkey_upper(a1);
            const double osc = __dsub_rn(hkey_upper(b1), hkey_lower(b0));
            bool ok = isfinite(osc) && isfinite(smin) && isfinite(smax) && n >= 3 &&
                      osc * (1.0 + 1e-12) < L.gap * (1.0 - 1e-12);
            int DLg = dmin_w, DRg = dmax_w;
            if (ok) {
                DLg = max(__double2int_ru(__fma_rn(smin, ia, hl)), dmin_w);
                DRg = min(__double2int_rd(__fma_rn(smax, ia, hr)), dmax_w);
                ok = DLg <= DRg;
            }
            S.mode = ok ? kModeWalk : kModeDirect;
            S.gate = ok;
            // unrolled sources that can reach outputs jlo .. jlo + jspan
            S.ya = jlo - DRg;
            S.yb = jlo + jspan - DLg;
            S.dlo = DLg;
            S.dhi = DRg;
            S.nq = 0;
            S.nlong = 0;
            S.abort = 0;
            S.qwork = 0;
            const double bud = LOB_HEAVY * static_cast<double>(jspan + 1) * static_cast<double>(2 * n + 1);
            S.budget = bud > 4.0e9 ? 4000000000u : static_cast<unsigned>(bud);
            S.c_src = S.c_queued = S.c_qent = 0;
        }
    }
    __syncthreads();
    bool walk = S.mode == kModeWalk;
    auto kf = [&](int d) -> double { return kdirect(p, d, drift); };
    if (walk) {
        const int ya = S.ya, yb = S.yb, dlo = S.dlo, dhi = S.dhi;
        const unsigned budget = S.budget;
        // the unrolled sources ya - 1 .. yb + 1 around the staged line: its wrapped halos, or (a
        // range wider than the buffer) chunks read from global memory
        const int lo = ya - 1, hi = yb + 1;
        const bool inplace = H0 + lo >= 0 && H0 + hi <= kUbLen - 1;
        int clen;
        const double* ub0;
        if (inplace) {
            // (a halo may span more than one period when the window's centre lies beyond n)
            // (wrapped by repeated add / subtract: one pass unless the halo exceeds a period; an
            // integer modulo per sample cost 5% of the sweep's instructions)
            for (int y = lo + tid; y < 0; y += kNT) {
                int w = y + n;
                while (w < 0) w += n;
                Ub[y] = Ub[w];
            }
            for (int y = n + tid; y <= hi; y += kNT) {
                int w = y - n;
                while (w >= n) w -= n;
                Ub[y] = Ub[w];
            }
            clen = yb - ya + 1;
            ub0 = Ub + lo;
        } else {
            __syncthreads();  // the stats read the staged line
            clen = min(kC, yb - ya + 1);
            int y0 = (ya - 1) % n;
            y0 += y0 < 0 ? n : 0;
            for (int i = tid; i < clen + 2; i += kNT) S.ubuf[i] = ul[((y0 + i) % n) * is];
            ub0 = S.ubuf;
        }
        // K(d) of the line's displacement range in shared memory when it fits (vbuf: the line
        // scratch above is dead once the constants are in registers)
        const int vcnt = dhi - dlo + 1;
        const bool kstage = vcnt <= kVCap;
        if (kstage)
            for (int i = tid; i < vcnt; i += kNT) S.vbuf[i] = kf(dlo + i);
        __syncthreads();
        const double* skt = S.vbuf - dlo;
        if (tid == 0 && diag) {
            atomicAdd(diag + 5, kstage ? 0ull : 1ull);
            atomicAdd(diag + 6, static_cast<unsigned long long>(vcnt));
        }
        for (int yc = ya; yc <= yb;) {
            if (yc != ya) {
                clen = min(kC, yb - yc + 1);
                __syncthreads();
                int y0 = (yc - 1) % n;
                y0 += y0 < 0 ? n : 0;
                for (int i = tid; i < clen + 2; i += kNT) S.ubuf[i] = ul[((y0 + i) % n) * is];
                __syncthreads();
            }
            if (tid == 0) S.c_src += static_cast<unsigned>(clen);
            const ChunkArgs ca{yc == ya ? ub0 : S.ubuf, clen, yc - jlo, jspan, ia, hl, hr, dlo, dhi, skt,
                               p.vtab + p.vofs, drift, tau, nullptr};
            walk = kstage ? process_chunk<false, true>(S, ca, budget) : process_chunk<false, false>(S, ca, budget);
            if (!walk) break;  // the walk would cost more than the window: the direct formula
            yc += clen;
        }
        if (!walk && tid == 0 && diag) atomicAdd(diag + 8, 1ull);
    } else if (tid == 0 && diag) {
        atomicAdd(diag + 7, 1ull);
    }
    if (!walk) {
        __syncthreads();
        tile_direct<false>(S, ul, n, 0, n, first, kf, is);
    }
    __syncthreads();
    // epilogue: u^{n+1} = best - tau V; the direct scan where nothing landed (cold)
    const double* tvl = tv ? tv + line * tv_stride : nullptr;
    const double sa1l = p.sa1 ? __ldg(p.sa1 + line) : 0.0;
    const double* sa2 = p.sa2;
    const double sb = p.sb;
    double* ostage = S.ubuf;  // ST == kStClu: the new line, for the cluster's row-segment stores
    // thread t owns outputs t + kNT m: the potential's samples are loaded for all of them first (one
    // memory latency, not kPer), the hot loop has no branch, and outputs no interval reached (+inf
    // keys: never when the gate holds) are rescanned after it.  KIND 0: no potential (best - 0 ==
    // best bitwise), 1: a tau*V table, 2: the separable tau*(a1 a2 + b).
    auto epilogue = [&](auto kind_c) {
        constexpr int KIND = decltype(kind_c)::value;
        double t[kPer];
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
            const int j = tid + kNT * m;
            t[m] = 0.0;
            if constexpr (KIND == 1) t[m] = j < n ? __ldg(tvl + j) : 0.0;
            if constexpr (KIND == 2) t[m] = j < n ? __ldg(sa2 + j) : 0.0;
        }
        auto tvof = [&](double x) -> double {
            if constexpr (KIND == 2) return __dmul_rn(tau, __dadd_rn(__dmul_rn(sa1l, x), sb));
            else return x;
        };
        unsigned miss = 0;
#pragma unroll
        for (int m = 0; m < kPer; ++m) {
            const int j = tid + kNT * m;
            if (j < n) {
                const unsigned long long kk = S.keys[j + 1];
                const double best = __longlong_as_double(static_cast<long long>(kk));
                const double o = KIND == 0 ? best : __dsub_rn(best, tvof(t[m]));
                if constexpr (ST == kStClu) ostage[j] = o;
                else ol[j * os] = o;
                // (high word only: a slot holding a genuine +inf or NaN sum is rescanned to the same value)
                miss |= static_cast<unsigned>(static_cast<unsigned>(kk >> 32) >= 0x7ff00000u &&
                                              static_cast<int>(kk >> 32) >= 0) << m;
            }
        }
        while (miss) {  // cold: the direct formula over the whole window
            const int m = __ffs(miss) - 1;
            miss &= miss - 1;
            const int j = tid + kNT * m;
            if (diag) atomicAdd(diag, 1ull);
            double best = INFINITY;
            int y = (j - first) % n;
            if (y < 0) y += n;
            for (int w = 0; w <= 2 * n; ++w) {
                const double c2 = __dadd_rn(ul[y * is], kf(first + w));
                best = c2 < best ? c2 : best;
                y = y == 0 ? n - 1 : y - 1;
            }
            double x = 0.0;  // (the sample reloaded: t[] stays in registers)
            if constexpr (KIND == 1) x = __ldg(tvl + j);
            if constexpr (KIND == 2) x = __ldg(sa2 + j);
            const double o = KIND == 0 ? best : __dsub_rn(best, tvof(x));
            if constexpr (ST == kStClu) ostage[j] = o;
            else ol[j * os] = o;
        }
    };
    if (tvl) epilogue(std::integral_constant<int, 1>{});
    else if (sa2) epilogue(std::integral_constant<int, 2>{});
    else epilogue(std::integral_constant<int, 0>{});
    if constexpr (ST == kStClu) {
        cg::cluster_group cluster = cg::this_cluster();
        const int r = static_cast<int>(cluster.block_rank());
        const int64_t c0 = line - r;
        const int rows = n / kLC;
        cluster.sync();
        for (int e = tid; e < rows * kLC; e += kNT) {
            const int row = r * rows + e / kLC, col = e % kLC;
            out[static_cast<int64_t>(row) * p.n + c0 + col] = *cluster.map_shared_rank(ostage + row, col);
        }
        cluster.sync();  // no CTA leaves while its line is still being read
    }
    if (tid == 0 && diag) {
        if (S.mode == kModeWalk) {
            atomicAdd(diag + 1, static_cast<unsigned long long>(S.c_src));
            atomicAdd(diag + 2, static_cast<unsigned long long>(S.c_queued));
            atomicAdd(diag + 3, static_cast<unsigned long long>(S.c_qent));
        }
        atomicAdd(diag + 4, 1ull);
    }
}

// ---- K2R: resident evolve for short lines --------------------------------
// One CTA per line keeps the line in shared memory for ALL steps of an evolve
// call (C1: 2000 steps of n = 1024 in one launch instead of 2000 launch-bound
// steps).  Each step is the K2 walk with every source of the line scanned (no
// tile statistics are needed: the whole line is resident), the oscillation
// gate from a block reduction of the slope extremes, the exact direct scan for
// any output the walk missed (never when the gate holds), the potential, the
// per-step drift (block tree sum, <= 1e-12 vs the reference's sequential sum)
// and decompose()'s block count of the step's input (the FSM of
// proj/src/minplus.cpp:161-187, per-thread segments composed in order).
constexpr int kRT = 512;  // max threads per resident CTA
constexpr int kResidentMaxN = 4096;  // shared memory: two line buffers, the keys, the K table (40 n bytes)

struct ResidentShared {
    double red[4][kRT / 32];
    unsigned long long fsm[kRT / 32];
    int flag;
};

__global__ void __launch_bounds__(kRT) resident_kernel(double* __restrict__ u, int n, const LineConst* __restrict__ lcs,
                                                       FastParams p, const double* __restrict__ tv, int64_t tv_stride,
                                                       int tv_period, int64_t tv_step_stride,
                                                       int steps, double* __restrict__ step_drift,
                                                       int64_t* __restrict__ step_blocks, int64_t lines,
                                                       int* __restrict__ halt) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* U0 = reinterpret_cast<double*>(smem_raw);
    double* U1 = U0 + n;
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(U1 + n);
    double* Ks = reinterpret_cast<double*>(keys + n);  // K(first + w), w = 0..2n: the step's fixed table
    __shared__ ResidentShared R;
    const int64_t line = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nt = blockDim.x, nw = nt >> 5;  // <= kRT
    const LineConst lc = lcs[line];
    const int first = static_cast<int>(lc.first);
    const int dmin_w = first + 1, dmax_w = first + 2 * n - 1;
    const double ia = p.ia, hl = lc.hl, hr = lc.hr, tau = p.tau;
    const double* tvl0 = tv ? tv + line * tv_stride : nullptr;
    double* ul = u + line * n;
    for (int j = tid; j < n; j += nt) U0[j] = ul[j];
    for (int w = tid; w <= 2 * n; w += nt) Ks[w] = kdirect(p, first + w, lc.drift);
    const double* Kd = Ks - first;  // Kd[d] = K(d)
    // thread t's contiguous segment of sources / increments
    const int seg = (n + nt - 1) / nt, sa = min(n, tid * seg), sb = min(n, sa + seg);
    const bool exact_cmp = p.eta == 0.0;
    int k = 0;
    for (; k < steps; ++k) {
        double* cur = (k & 1) ? U1 : U0;
        double* nxt = (k & 1) ? U0 : U1;
        // tau*V of this step: one table, or table k mod tv_period (in-period time labels)
        const double* tvl = tvl0 && tv_period > 1 ? tvl0 + (k % tv_period) * tv_step_stride : tvl0;
        __syncthreads();
        // slope extremes (gate) and the FSM summary of this thread's increments
        double smn = INFINITY, smx = -INFINITY, umn = INFINITY, umx = -INFINITY;
        int v = 0 | (1 << 2) | (2 << 4);
        int cnt[3] = {0, 0, 0};
        double sprev = 0.0;
        for (int y = sa; y < sb; ++y) {
            const double s = __dsub_rn(cur[y + 1 == n ? 0 : y + 1], cur[y]);
            smn = fmin(smn, s);
            smx = fmax(smx, s);
            umn = fmin(umn, cur[y]);
            umx = fmax(umx, cur[y]);
            if (step_blocks) {
                if (y == sa) sprev = y > 0 ? __dsub_rn(cur[y], cur[y - 1]) : 0.0;
                if (y >= 1) {  // increment e = y: s(y) - s(y-1), e in [1, n-1]
                    int c;
                    if (exact_cmp) c = s > sprev ? 0 : (s < sprev ? 1 : 2);
                    else {
                        const double inc = __dsub_rn(s, sprev);
                        c = inc > p.eta ? 0 : (inc < -p.eta ? 1 : 2);
                    }
                    int nv = 0;
#pragma unroll
                    for (int q = 0; q < 3; ++q) {
                        int e;
                        const int st = fsm_next((v >> (2 * q)) & 3, c, &e);
                        nv |= st << (2 * q);
                        cnt[q] += e;
                    }
                    v = nv;
                }
                sprev = s;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            smn = fmin(smn, __shfl_xor_sync(0xffffffffu, smn, o));
            smx = fmax(smx, __shfl_xor_sync(0xffffffffu, smx, o));
            umn = fmin(umn, __shfl_xor_sync(0xffffffffu, umn, o));
            umx = fmax(umx, __shfl_xor_sync(0xffffffffu, umx, o));
        }
        if (step_blocks) {
            const unsigned long long f = warp_fsm(fsm_pack(v, cnt));
            if (lane == 0) R.fsm[warp] = f;
        }
        if (lane == 0) {
            R.red[0][warp] = smn;
            R.red[1][warp] = smx;
            R.red[2][warp] = umn;
            R.red[3][warp] = umx;
        }
        for (int j = tid; j < n; j += nt) keys[j] = kInfBits;
        __syncthreads();
        if (warp == 0) {
            double a0 = lane < nw ? R.red[0][lane] : INFINITY, a1 = lane < nw ? R.red[1][lane] : -INFINITY;
            double b0 = lane < nw ? R.red[2][lane] : INFINITY, b1 = lane < nw ? R.red[3][lane] : -INFINITY;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                a0 = fmin(a0, __shfl_xor_sync(0xffffffffu, a0, o));
                a1 = fmax(a1, __shfl_xor_sync(0xffffffffu, a1, o));
                b0 = fmin(b0, __shfl_xor_sync(0xffffffffu, b0, o));
                b1 = fmax(b1, __shfl_xor_sync(0xffffffffu, b1, o));
            }
            if (lane == 0) {
                // the exact oscillation max u - min u against the window's edge gap (fast_kernel)
                const double osc = __dsub_rn(b1, b0);
                R.flag = isfinite(osc) && isfinite(a0) && isfinite(a1) && n >= 3 &&
                         osc * (1.0 + 1e-12) < lc.gap * (1.0 - 1e-12);
            }
            if (step_blocks) {  // the warps' summaries composed in order (lanes >= warps: identity)
                const unsigned long long f = warp_fsm(lane < nw ? R.fsm[lane] : fsm_identity());
                if (lane == 0)
                    step_blocks[static_cast<int64_t>(k) * lines + line] = 1 + static_cast<int64_t>((f >> 16) & 0xffff);
            }
        }
        __syncthreads();
        const bool ok = R.flag;
        if (ok) {
            // every source's local-minimum interval (fast.cu header), exact CAS-min
            for (int y = sa; y < sb; ++y) {
                const double u0 = cur[y];
                const double sl = __dsub_rn(u0, cur[y == 0 ? n - 1 : y - 1]);
                const double sr = __dsub_rn(cur[y + 1 == n ? 0 : y + 1], u0);
                const int dl = max(__double2int_ru(__fma_rn(sl, ia, hl)), dmin_w);
                const int dr = min(__double2int_rd(__fma_rn(sr, ia, hr)), dmax_w);
                int j = y + dl;  // wrapped by add / subtract (|dl| < 2n + |centre|: a few passes at most)
                while (j < 0) j += n;
                while (j >= n) j -= n;
                for (int d = dl; d <= dr; ++d) {
                    smem_fmin(&keys[j], __dadd_rn(u0, Kd[d]));
                    j = j + 1 == n ? 0 : j + 1;
                }
            }
        }
        __syncthreads();
        // epilogue: exact min (direct scan where the walk left nothing), potential, drift
        double acc = 0.0;
        bool bad = false;
        for (int j = tid; j < n; j += nt) {
            double best;
            const unsigned long long kk = keys[j];
            if (ok && kk != kInfBits) {
                best = __longlong_as_double(static_cast<long long>(kk));
            } else {
                best = INFINITY;  // proj/tests/unit_scheme.cpp:184-190
                int y = (j - first) % n;
                if (y < 0) y += n;
                for (int w = 0; w <= 2 * n; ++w) {
                    const double c2 = __dadd_rn(cur[y], Ks[w]);
                    best = c2 < best ? c2 : best;
                    y = y == 0 ? n - 1 : y - 1;
                }
            }
            const double o = tvl ? __dsub_rn(best, tvl[j]) : best;
            nxt[j] = o;
            acc += o - cur[j];
            bad |= !isfinite(o);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        bad = __syncthreads_or(bad);
        if (lane == 0) R.red[0][warp] = acc;
        __syncthreads();
        if (tid == 0) {
            double sum = 0.0;
            for (int w = 0; w < nw; ++w) sum += R.red[0][w];
            if (step_drift) step_drift[static_cast<int64_t>(k) * lines + line] = sum / static_cast<double>(n);
            if (bad) atomicMin(halt, k);
        }
        if (bad) {
            ++k;
            break;
        }
    }
    __syncthreads();
    const double* fin = (k & 1) ? U1 : U0;
    for (int j = tid; j < n; j += nt) ul[j] = fin[j];
}

}  // namespace

// ---------------------------------------------------------------------------
// workspace: sub[2][lines][subs] double2 | fsm[2][lines][tiles] u64 |
//            line[3][lines][4] u64 | LineConst[lines] | diag u64[16] | done u32[lines]
constexpr int kDiag = 16;
struct WsLayout {
    size_t sub, fsm, line, lc, diag, done, samp, total;
};
static WsLayout ws_layout(int64_t lines, int64_t n) {
    const int64_t tiles = (n + kT - 1) / kT, subs = (n + kG - 1) / kG;
    WsLayout w;
    w.sub = 0;
    w.fsm = w.sub + 2 * static_cast<size_t>(lines * subs) * sizeof(double2);
    w.line = w.fsm + 2 * static_cast<size_t>(lines * tiles) * sizeof(unsigned long long);
    w.lc = w.line + 3 * static_cast<size_t>(lines) * 4 * sizeof(unsigned long long);
    w.diag = w.lc + static_cast<size_t>(lines) * sizeof(LineConst);
    w.done = w.diag + kDiag * sizeof(unsigned long long);  // [lines] warps finished since the counters reset
    w.samp = w.done + (static_cast<size_t>(lines) * sizeof(unsigned) + 255) / 256 * 256;
    w.total = w.samp + 2 * static_cast<size_t>(lines) * kSamp * sizeof(double);
    return w;
}

size_t fast_workspace_bytes(int64_t lines, int64_t n) { return ws_layout(lines, n).total; }


static int ensure_lut(lob_ctx* ctx) {
    if (!first_time(ctx, reinterpret_cast<const void*>(&g_fsm_lut2))) return LOB_OK;
    unsigned short lut[kLut2];
    for (int v = 0; v < 64; ++v)
        for (int c0 = 0; c0 < 4; ++c0)
            for (int c1 = 0; c1 < 4; ++c1) {
                int nv = 0;
                unsigned em = 0;
                for (int q = 0; q < 3; ++q) {
                    int st = (v >> (2 * q)) & 3;
                    if (st > 2) st = 0;
                    int e = 0, e2 = 0;
                    if (c0 < 3) st = fsm_next(st, c0, &e);
                    if (c1 < 3) st = fsm_next(st, c1, &e2);
                    nv |= st << (2 * q);
                    if (e + e2 > 1) return set_error(ctx, LOB_CUDA_ERROR, "fsm table: two emits per pair");
                    em |= static_cast<unsigned>(e + e2) << (3 * q);
                }
                lut[v * 16 + c0 * 4 + c1] = static_cast<unsigned short>(static_cast<unsigned>(nv) | (em << 6));
            }
    LOB_CUDA_TRY(ctx, cudaMemcpyToSymbol(g_fsm_lut2, lut, sizeof(lut)));
    return LOB_OK;
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
        // cached for later calls on any stream: complete it now
        LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
        it = ctx->vtabs.emplace(key, vt).first;
    }
    *out = it->second.dev;
    *vofs = 3 * n;
    return LOB_OK;
}

static FastParams make_params(int64_t n, double tau, double eta) {
    FastParams p{};
    p.n = n;
    p.tiles = (n + kT - 1) / kT;
    p.subs = (n + kG - 1) / kG;
    p.tau = tau;
    p.eta = eta;
    p.eps = 1.0 / static_cast<double>(n);  // SchemeParams::epsilon(), proj/include/laxol/scheme.hpp:25
    p.a = p.eps * p.eps / tau;
    p.ia = 1.0 / p.a;
    p.fsm_on = 1;
    p.delta_override = __builtin_nan("");
    return p;
}

static FastBuffers make_buffers(void* ws, int64_t lines, int64_t n, int64_t counter) {
    const WsLayout w = ws_layout(lines, n);
    char* base = static_cast<char*>(ws);
    const int64_t subs = (n + kG - 1) / kG, tiles = (n + kT - 1) / kT;
    double2* sub = reinterpret_cast<double2*>(base + w.sub);
    unsigned long long* fsm = reinterpret_cast<unsigned long long*>(base + w.fsm);
    unsigned long long* line = reinterpret_cast<unsigned long long*>(base + w.line);
    const int64_t c2 = counter % 2, c3 = counter % 3;
    FastBuffers b;
    b.sub_in = sub + c2 * lines * subs;
    b.sub_out = sub + (1 - c2) * lines * subs;
    b.fsm_in = fsm + c2 * lines * tiles;
    b.fsm_out = fsm + (1 - c2) * lines * tiles;
    b.line_in = line + c3 * lines * 4;
    b.line_out = line + ((c3 + 1) % 3) * lines * 4;
    b.line_reset = line + ((c3 + 2) % 3) * lines * 4;
    double* samp = reinterpret_cast<double*>(base + w.samp);
    b.samp_in = samp + c2 * lines * kSamp;
    b.samp_out = samp + (1 - c2) * lines * kSamp;
    return b;
}

int64_t fast_line_max() { return kT; }

// the driver's cuTensorMapEncodeTiled through the runtime (no -lcuda link)
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
        return static_cast<PFN_cuTensorMapEncodeTiled_v12000>(nullptr);
    }();  // thread-safe one-time initialisation (function-local static)
    return fn;
}

int launch_line_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n, const double* drift,
                    double tau, const double* tv, int64_t tv_stride, const FastSepPot* sep, int load, int store,
                    unsigned long long* diag, cudaStream_t s) {
    if (n < 3 || n > kT) return set_error(ctx, LOB_INVALID_INPUT, "fast line kernel: 3 <= n <= 2048");
    if ((load != kLineRow || store != kLineRow) && lines != n)
        return set_error(ctx, LOB_INVALID_INPUT, "fast line kernel: columns need lines == n");
    if ((load == kLineClu || store == kLineClu) && n % kLC != 0)
        return set_error(ctx, LOB_INVALID_INPUT, "fast line kernel: cluster columns need n % 8 == 0");
    if (load == kLineTma && (n % 2 != 0 || reinterpret_cast<uintptr_t>(u) % 16 != 0))
        return set_error(ctx, LOB_INVALID_INPUT, "fast line kernel: TMA columns need even n and 16-byte rows");
    if (lines < 1 || lines > 0x7fffffffll) return set_error(ctx, LOB_INVALID_INPUT, "fast line kernel: lines");
    FastParams p = make_params(n, tau, 0.0);
    p.delta_override = ctx->fast_delta_override;
    int st = ensure_vtab(ctx, n, tau, &p.vtab, &p.vofs, s);
    if (st) return st;
    if (sep) {
        p.sa1 = sep->a1;
        p.sa2 = sep->a2;
        p.sb = sep->b;
    }
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    if (load == kLineTma) {
        auto enc = tensor_map_encoder();
        if (!enc) return set_error(ctx, LOB_CUDA_ERROR, "fast line kernel: cuTensorMapEncodeTiled unavailable");
        const cuuint64_t gdim[2] = {static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(n)};
        const cuuint64_t gstride[1] = {static_cast<cuuint64_t>(n) * sizeof(double)};
        const cuuint32_t box[2] = {2, static_cast<cuuint32_t>(kTmaRows)};
        const cuuint32_t estride[2] = {1, 1};
        const CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(u), gdim, gstride, box,
                               estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return set_error(ctx, LOB_CUDA_ERROR, "fast line kernel: tensor map encoding failed");
    }
    using KernT = void (*)(const double*, double*, const double*, const double*, int64_t, unsigned long long*,
                           FastParams, const CUtensorMap);
    KernT kern = nullptr;
    if (load == kLineRow && store == kLineRow) kern = line_kernel<kLdRow, kStRow>;
    else if (load == kLineCol && store == kLineCol) kern = line_kernel<kLdCol, kStCol>;
    else if (load == kLineCol && store == kLineRow) kern = line_kernel<kLdCol, kStRow>;
    else if (load == kLineClu && store == kLineClu) kern = line_kernel<kLdClu, kStClu>;
    else if (load == kLineTma && store == kLineRow) kern = line_kernel<kLdTma, kStRow>;
    else if (load == kLineTma && store == kLineCol) kern = line_kernel<kLdTma, kStCol>;
    else return set_error(ctx, LOB_INVALID_INPUT, "fast line kernel: unsupported load / store layout");
    if (first_time(ctx, reinterpret_cast<const void*>(kern))) {
        LOB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(sizeof(MainShared))));
        LOB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                               cudaSharedmemCarveoutMaxShared));
    }
    const bool cluster = load == kLineClu || store == kLineClu;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(lines));
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = sizeof(MainShared);
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = kLC;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = cluster ? 2 : 1;
    LOB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, u, out, drift, tv, tv_stride, diag, p, tmap));
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "fast line kernel");
}

int launch_fast_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                    const double* drift, double tau, const double* tv, int64_t tv_stride,
                    double eta, int64_t* blocks, void* workspace, size_t ws_bytes, int flags,
                    cudaStream_t s, double* dpart, const FastTable* tab, const FastSepPot* sep,
                    const FastDriftOut* dout) {
    if (ws_bytes < fast_workspace_bytes(lines, n) || !workspace)
        return set_error(ctx, LOB_INVALID_INPUT, "lob_minplus_fast_f64: workspace too small");
    if (n > (1ll << 29)) return set_error(ctx, LOB_INVALID_INPUT, "fast: n too large");
    int st = ensure_lut(ctx);
    if (st) return st;
    FastParams p = make_params(n, tau, eta);
    p.delta_override = ctx->fast_delta_override;
    if (!tab) {
        st = ensure_vtab(ctx, n, tau, &p.vtab, &p.vofs, s);
        if (st) return st;
    }
    const int64_t nblk = lines * p.tiles;
    if (nblk > 0x7fffffffll) return set_error(ctx, LOB_INVALID_INPUT, "fast: grid too large");
    p.drift_arr = drift;
    if (sep) {
        p.sa1 = sep->a1;
        p.sa2 = sep->a2;
        p.sb = sep->b;
    }
    if (tab) {
        p.ktab = tab->ktab;
        p.kstride = tab->stride;
        p.kfirst = tab->first;
    }
    // the per-line constants hold the window table: another table recomputes them
    const void* tkey = tab ? static_cast<const void*>(tab->ktab) : nullptr;
    if (ctx->ws_table[workspace] != tkey) {
        ctx->ws_table[workspace] = tkey;
        flags &= ~LOB_FAST_STATS_VALID;
    }
    const bool tma = (n % 2 == 0) && (reinterpret_cast<uintptr_t>(u) % 16 == 0);
    if (ctx->ws_shape[workspace] != std::make_pair(lines, n)) {
        ctx->ws_shape[workspace] = std::make_pair(lines, n);
        flags &= ~LOB_FAST_STATS_VALID;
    }
    // the statistics describe the previous call's output: any other input recomputes them
    if (ctx->ws_last_out[workspace] != static_cast<const void*>(u)) flags &= ~LOB_FAST_STATS_VALID;
    // block counts come from FSM summaries the previous call's epilogue produced only if it was
    // asked for block counts too (the epilogue predicts the next call from this one)
    if (blocks && !ctx->ws_fsm_valid[workspace]) flags &= ~LOB_FAST_STATS_VALID;
    ctx->ws_last_out[workspace] = out;
    // short lines without block counts / drift partials: K2L (statistics from the staged line)
    if (ctx->fast_line && !tab && n <= kT && n >= 3 && !blocks && !dpart && !(flags & kFastStatsGiven)) {
        const WsLayout wl = ws_layout(lines, n);
        unsigned long long* dg = reinterpret_cast<unsigned long long*>(static_cast<char*>(workspace) + wl.diag);
        if (!(flags & LOB_FAST_STATS_VALID))
            LOB_CUDA_TRY(ctx, cudaMemsetAsync(dg, 0, kDiag * sizeof(unsigned long long), s));
        ctx->ws_nostats[workspace] = true;  // a later tiled call recomputes its statistics
        ctx->ws_chain[workspace] = 0;
        ctx->ws_lc_valid[workspace] = false;
        const FastSepPot* sp = sep;
        return launch_line_f64(ctx, u, out, lines, n, drift, tau, tv, tv_stride, sp, kLineRow, kLineRow, dg, s);
    }
    if (ctx->ws_nostats[workspace]) {
        ctx->ws_nostats[workspace] = false;
        flags &= ~(LOB_FAST_STATS_VALID | kFastStatsGiven);
    }
    // a checked call needs the samples its statistics were taken with: the first one on a workspace
    // (or after a call that stored none) recomputes the statistics and their samples
    if (flags & LOB_FAST_STATS_CHECK) {
        ctx->ws_sampling[workspace] = true;
        if (!ctx->ws_samples_valid[workspace]) flags &= ~LOB_FAST_STATS_VALID;
    }
    // the per-line done counters restart with the statistics (keeps them in range)
    if (ctx->ws_chain[workspace] * p.tiles * (kNT / 32) > 0xf0000000ll) flags &= ~LOB_FAST_STATS_VALID;
    int64_t& counter = ctx->ws_counter[workspace];
    FastBuffers b = make_buffers(workspace, lines, n, counter);
    const WsLayout w = ws_layout(lines, n);
    unsigned long long* diag =
        reinterpret_cast<unsigned long long*>(static_cast<char*>(workspace) + w.diag);
    LineConst* lcs = reinterpret_cast<LineConst*>(static_cast<char*>(workspace) + w.lc);
    // statistics of u produced by the caller (fast_given_stats_buffers + a transpose kernel):
    // the line constants are recomputed only for a new workspace (the device check catches a
    // changed drift)
    const bool given = flags & kFastStatsGiven;
    if (given) {
        flags |= LOB_FAST_STATS_VALID;
        if (!ctx->ws_lc_valid[workspace]) {
            line_setup_kernel<<<static_cast<unsigned>((lines + 127) / 128), 128, 0, s>>>(drift, lines, p, lcs);
            LOB_CUDA_TRY(ctx, cudaMemsetAsync(diag, 0, kDiag * sizeof(unsigned long long), s));
            ctx->launches += 1;
            ctx->ws_lc_valid[workspace] = true;
        }
        flags &= ~LOB_FAST_CHAINED;
        ctx->ws_chain[workspace] = 0;
    }
    if (!(flags & LOB_FAST_STATS_VALID)) {
        ctx->ws_lc_valid[workspace] = !tab;
        // per-line constants (valid while drift/tau/n (or the table) and the workspace are unchanged)
        if (tab)
            line_setup_tab_kernel<<<static_cast<unsigned>((lines * 32 + 127) / 128), 128, 0, s>>>(
                tab->ktab, tab->stride, tab->first, lines, n, lcs);
        else
            line_setup_kernel<<<static_cast<unsigned>((lines + 127) / 128), 128, 0, s>>>(drift, lines, p, lcs);
        LOB_CUDA_TRY(ctx, cudaMemsetAsync(diag, 0, kDiag * sizeof(unsigned long long), s));
        LOB_CUDA_TRY(ctx, cudaMemsetAsync(static_cast<char*>(workspace) + w.done, 0, lines * sizeof(unsigned), s));
        ctx->ws_chain[workspace] = 0;
        ctx->launches += 1;
        // statistics of the given u into the "in" buffers; "out" line stats reset
        FastBuffers sb = b;
        sb.sub_out = const_cast<double2*>(b.sub_in);
        sb.fsm_out = const_cast<unsigned long long*>(b.fsm_in);
        sb.line_out = const_cast<unsigned long long*>(b.line_in);
        sb.samp_out = const_cast<double*>(b.samp_in);
        const unsigned lb = static_cast<unsigned>((lines + 127) / 128);
        line_init_kernel<<<lb, 128, 0, s>>>(const_cast<unsigned long long*>(b.line_in), lines);
        line_init_kernel<<<lb, 128, 0, s>>>(b.line_out, lines);
        stats_kernel<<<static_cast<unsigned>(nblk), kNT, 0, s>>>(u, p, sb);
        ctx->launches += 3;
        LOB_CUDA_TRY(ctx, cudaGetLastError());
    }
    // chained: every LOB_FAST_CHAINED call releases per-line counters; it waits on them
    // (instead of on the whole previous grid) when the previous call on this workspace
    // released too (the counters then hold chain * tiles * warps counts per line)
    int64_t& chain = ctx->ws_chain[workspace];
    const bool release = flags & LOB_FAST_CHAINED;
    const bool chained = release && (flags & LOB_FAST_STATS_VALID) && chain > 0;
    if (!release) chain = 0;  // the counters no longer describe the previous call
    unsigned* done = reinterpret_cast<unsigned*>(static_cast<char*>(workspace) + w.done);
    if (release && chain == 0) LOB_CUDA_TRY(ctx, cudaMemsetAsync(done, 0, lines * sizeof(unsigned), s));
    using KernT = void (*)(const double*, double*, const LineConst*, const double*, int64_t, int64_t*,
                           unsigned long long*, FastParams, FastBuffers, unsigned*, unsigned, double*);
    static const KernT kerns[2][2][2][2] = {
        {{{fast_kernel<false, false, false, false>, fast_kernel<false, false, false, true>},
          {fast_kernel<false, false, true, false>, fast_kernel<false, false, true, true>}},
         {{fast_kernel<false, true, false, false>, fast_kernel<false, true, false, true>},
          {fast_kernel<false, true, true, false>, fast_kernel<false, true, true, true>}}},
        {{{fast_kernel<true, false, false, false>, fast_kernel<true, false, false, true>},
          {fast_kernel<true, false, true, false>, fast_kernel<true, false, true, true>}},
         {{fast_kernel<true, true, false, false>, fast_kernel<true, true, false, true>},
          {fast_kernel<true, true, true, false>, fast_kernel<true, true, true, true>}}}};
    auto kern = kerns[tab != nullptr][tma][chained][release];
    const unsigned need = static_cast<unsigned>(chain * p.tiles * (kNT / 32));
    if (first_time(ctx, reinterpret_cast<const void*>(kern))) {
        LOB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(sizeof(MainShared))));
        // the whole unified L1 as shared memory: LOB_FAST_MINB CTAs per SM (the driver's default
        // carveout for this size leaves one CTA less)
        LOB_CUDA_TRY(ctx, cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                               cudaSharedmemCarveoutMaxShared));
    }
    p.fsm_on = blocks ? 1 : 0;  // the stats kernel above always produced them
    // the sampled check needs samples taken by this engine (not by a caller's statistics pass)
    p.check = (flags & LOB_FAST_STATS_CHECK) && (flags & LOB_FAST_STATS_VALID) && !given ? 1 : 0;
    p.samples = ctx->ws_sampling[workspace] ? 1 : 0;
    if (dout && dpart) {
        p.drift_out = dout->drift_out;
        p.halt = dout->halt;
        p.dcount = dout->dcount;
        p.dstep = dout->step;
    }
    ctx->ws_samples_valid[workspace] = p.samples != 0;
    ctx->ws_fsm_valid[workspace] = blocks != nullptr;
    const dim3 grid = line_grid(static_cast<unsigned>(p.tiles), lines);
    p.lines = lines;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(kNT);
    cfg.dynamicSmemBytes = sizeof(MainShared);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LOB_CUDA_TRY(ctx, cudaLaunchKernelEx(&cfg, kern, u, out, const_cast<const LineConst*>(lcs), tv, tv_stride,
                                         blocks, diag, p, b, done, need, dpart));
    if (release) chain += 1;
    ctx->launches += 1;
    LOB_CUDA_TRY(ctx, cudaGetLastError());
    counter += 1;
    return LOB_OK;
}


size_t fast_resident_smem(int64_t n) { return static_cast<size_t>(n) * 24 + static_cast<size_t>(2 * n + 1) * 8; }
bool fast_resident_ok(int64_t n) { return n >= 3 && n <= kResidentMaxN; }

// `steps` K2 steps of `lines` short lines in ONE launch (K2R above); u in place.
int launch_fast_resident_f64(lob_ctx* ctx, double* u, int64_t lines, int64_t n, const double* drift, double tau,
                             const double* tv, int64_t tv_stride, double eta, int64_t steps, double* step_drift,
                             int64_t* step_blocks, int* halt, void* lc_buf, cudaStream_t s, int tv_period,
                             int64_t tv_step_stride) {
    if (!fast_resident_ok(n)) return set_error(ctx, LOB_INVALID_INPUT, "resident K2: n out of range");
    if (lines > 0x7fffffffll || steps > 0x7fffffffll) return set_error(ctx, LOB_INVALID_INPUT, "resident K2: too large");
    int st = ensure_lut(ctx);
    if (st) return st;
    FastParams p = make_params(n, tau, eta);
    st = ensure_vtab(ctx, n, tau, &p.vtab, &p.vofs, s);
    if (st) return st;
    LineConst* lcs = static_cast<LineConst*>(lc_buf);
    line_setup_kernel<<<static_cast<unsigned>((lines + 127) / 128), 128, 0, s>>>(drift, lines, p, lcs);
    const size_t smem = fast_resident_smem(n);
    if (first_time(ctx, reinterpret_cast<const void*>(&resident_kernel)))
        LOB_CUDA_TRY(ctx, cudaFuncSetAttribute(resident_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(fast_resident_smem(kResidentMaxN))));
    // two sources per thread (up to kRT; measured on C1: 512 threads 8.8 us/step, 1024 threads
    // 10.8, 128 threads 13.9)
    const int nt = static_cast<int>(std::min<int64_t>(kRT, std::max<int64_t>(64, ((n / 2 + 31) / 32) * 32)));
    resident_kernel<<<static_cast<unsigned>(lines), nt, smem, s>>>(u, static_cast<int>(n), lcs, p, tv, tv_stride,
                                                                     tv_period, tv_step_stride, static_cast<int>(steps),
                                                                     step_drift, step_blocks, lines, halt);
    ctx->launches += 2;
    return cuda_status(ctx, cudaGetLastError(), "resident K2");
}


int64_t fast_tiles(int64_t n) { return (n + kT - 1) / kT; }

int launch_drift_tiles(lob_ctx* ctx, const double* dpart, int64_t lines, int64_t n, double* drift_out, int* halt,
                       int step, cudaStream_t s) {
    drift_tiles_kernel<<<static_cast<unsigned>((lines + 127) / 128), 128, 0, s>>>(dpart, lines, fast_tiles(n), n,
                                                                                  drift_out, halt, step);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "drift_tiles_kernel");
}

int fast_diag_count(lob_ctx* ctx, void* workspace, int64_t lines, int64_t n, uint64_t* count,
                    cudaStream_t s) {
    const WsLayout w = ws_layout(lines, n);
    // the counters are written by K2 launches on the caller's streams: wait for all of them
    LOB_CUDA_TRY(ctx, cudaDeviceSynchronize());
    LOB_CUDA_TRY(ctx, cudaMemcpyAsync(count, static_cast<char*>(workspace) + w.diag,
                                      kDiag * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    LOB_CUDA_TRY(ctx, cudaStreamSynchronize(s));
    return LOB_OK;
}

int launch_block_counts(lob_ctx* ctx, const double* u, int64_t lines, int64_t n, double eta,
                        int64_t* blocks, cudaStream_t s) {
    int st = ensure_lut(ctx);
    if (st) return st;
    FastParams p = make_params(n, 1.0, eta);
    const int64_t nblk = lines * p.tiles;
    void* ws = nullptr;
    const size_t bytes = fast_workspace_bytes(lines, n);
    LOB_CUDA_TRY(ctx, cudaMallocAsync(&ws, bytes, s));
    FastBuffers b = make_buffers(ws, lines, n, 0);
    FastBuffers sb = b;
    sb.sub_out = const_cast<double2*>(b.sub_in);
    sb.fsm_out = const_cast<unsigned long long*>(b.fsm_in);
    sb.line_out = const_cast<unsigned long long*>(b.line_in);
    sb.samp_out = const_cast<double*>(b.samp_in);
    line_init_kernel<<<static_cast<unsigned>((lines + 127) / 128), 128, 0, s>>>(sb.line_out, lines);
    stats_kernel<<<static_cast<unsigned>(nblk), kNT, 0, s>>>(u, p, sb);
    combine_blocks_kernel<<<static_cast<unsigned>((lines + 127) / 128), 128, 0, s>>>(b.fsm_in, lines,
                                                                                     p.tiles, blocks);
    ctx->launches += 3;
    cudaFreeAsync(ws, s);
    return cuda_status(ctx, cudaGetLastError(), "block counts");
}

int fast_given_stats_buffers(lob_ctx* ctx, void* workspace, int64_t lines, int64_t n, double2** sub,
                             unsigned long long** line_keys) {
    if (ctx->ws_shape[workspace] != std::make_pair(lines, n)) {
        ctx->ws_shape[workspace] = std::make_pair(lines, n);
        ctx->ws_lc_valid[workspace] = false;
    }
    const FastBuffers b = make_buffers(workspace, lines, n, ctx->ws_counter[workspace]);
    *sub = const_cast<double2*>(b.sub_in);
    *line_keys = const_cast<unsigned long long*>(b.line_in);
    return LOB_OK;
}

// dst = src^T (n x n) and the statistics of dst's lines for the next K2 call on `workspace`
int launch_transpose_stats(lob_ctx* ctx, const double* src, double* dst, int64_t n, void* workspace,
                           cudaStream_t s) {
    double2* sub = nullptr;
    unsigned long long* L = nullptr;
    fast_given_stats_buffers(ctx, workspace, n, n, &sub, &L);
    // line keys: minima start at ~0, maxima at 0 ([umin, umax, smin, smax] per line)
    LOB_CUDA_TRY(ctx, cudaMemset2DAsync(L, 16, 0xff, 8, static_cast<size_t>(2 * n), s));
    LOB_CUDA_TRY(ctx, cudaMemset2DAsync(L + 1, 16, 0x00, 8, static_cast<size_t>(2 * n), s));
    const int64_t subs = (n + kG - 1) / kG;
    dim3 grid(static_cast<unsigned>((n + kTSL - 1) / kTSL), static_cast<unsigned>(subs));
    transpose_stats_kernel<<<grid, 256, 0, s>>>(src, dst, n, subs, sub, L);
    ctx->launches += 1;
    return cuda_status(ctx, cudaGetLastError(), "transpose_stats_kernel");
}

}  // namespace lob

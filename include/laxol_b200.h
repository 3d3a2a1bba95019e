/* laxol_b200 — C-ABI of the B200-native Lax-Oleinik min-plus hot path.
 *
 * The reference (`laxol`, /root/reference/proj) is a C++20 library with no
 * C-ABI or FFI of its own.  Its stepping API is the drop-in surface:
 *   kinetic_convolve(u, kernel, eta, ConvEngine, blocks*)   proj/include/laxol/scheme.hpp:52-53
 *   step_fully_discrete(u, t, spec, params, kernel, engine)  proj/include/laxol/scheme.hpp:57-59
 *   evolve(u0, t0, steps, spec, params, options)             proj/include/laxol/scheme.hpp:82-90
 *   split_step_nd(u, t, SplitSpec, params)                   proj/include/laxol/splitting.hpp:40-41
 * The engine switch those calls go through (proj/src/scheme.cpp:114-121) is
 * where the entry points below plug in.  The C++ mirror
 * of that API lives in paper_1210_4090_b200/csrc/host/laxol_b200.hpp.
 *
 * Conventions
 *  - A "line" is one 1-D periodic problem of n samples: the FUNDAMENTAL
 *    domain, no duplicated seam (the host GridFn keeps n+1 samples,
 *    proj/include/laxol/grid_fn.hpp:8-12).  Lines are stored row-major,
 *    lines x n doubles, in device memory owned by the caller.
 *    Any lines >= 0 (0 is a no-op; batches above 65535 lines are folded over two
 *    grid dimensions inside the kernels) and any n >= 1 (n_space = 1 is legal in the
 *    reference, proj/src/scheme.cpp:40); the fast and relaxed engines take n <= 2^29.
 *  - The kernel window of line l is ktab[l*ktab_stride + w], w = 0..2n, the
 *    table build_kernel produces (proj/src/scheme.cpp:77-81), with grid
 *    displacement d = first[l] + w (first = center_index - n).
 *    ktab_stride 0 = one table shared by all lines.
 *  - tv is tau*V already rounded on the host (the product of
 *    proj/src/scheme.cpp:161); the device applies out = best - tv[j] with one
 *    rounding, never an FMA.  tv_stride 0 = shared across lines; tv NULL = V == 0.
 *  - Every entry point is asynchronous on `stream` (a cudaStream_t, NULL =
 *    legacy default) unless its name ends in _host.
 *  - Status codes map back to the reference's exception types
 *    (proj/include/laxol/errors.hpp:8-17): LOB_INVALID_INPUT -> InvalidInput,
 *    LOB_EVALUATION_ERROR -> EvaluationError.  lob_last_error(ctx) explains.
 *  - There is no CPU fallback: without a CUDA device every compute entry
 *    point returns LOB_CUDA_ERROR.
 */
#ifndef LAXOL_B200_H
#define LAXOL_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOB_OK 0
#define LOB_INVALID_INPUT 1
#define LOB_EVALUATION_ERROR 2
#define LOB_CUDA_ERROR 3

/* Engines: ConvEngine{Fast, Naive} (proj/include/laxol/scheme.hpp:13) gains
 * two device engines. */
#define LOB_ENGINE_DIRECT 0 /* K1: exact O(n^2) min-plus, bit-identical to ConvEngine::Naive */
#define LOB_ENGINE_FAST 1   /* K2: exact O(n) local-minimum walk (mechanical kinetics) */
#define LOB_ENGINE_RELAXED 2 /* the reference's ConvEngine::Fast with eta (relaxed for eta > 0), see
                              * lob_minplus_relaxed_f64; evolve and the host step accept it */

typedef struct lob_ctx lob_ctx;

/* Context: one per host thread; owns scratch and cached tables. */
int lob_ctx_create(int device, lob_ctx** out);
int lob_ctx_destroy(lob_ctx* ctx);
const char* lob_last_error(const lob_ctx* ctx);
const char* lob_version(void);

/* K1 — direct min-plus, fp64, fused potential epilogue.
 * Replaces conv_naive (proj/src/minplus.cpp:116-126) + periodic aliasing
 * (proj/src/scheme.cpp:125-134) + potential loop (proj/src/scheme.cpp:156-162):
 *   out[l][j] = min_{w=0..2n} (u[l][(j - first[l] - w) mod n] + ktab_l[w]) - tv_l[j]
 * first: device array of `lines` int64. */
int lob_minplus_direct_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                           const double* ktab, int64_t ktab_stride, const int64_t* first,
                           const double* tv, int64_t tv_stride, void* stream);

/* K1 implementation (per context; every K1 sweep — lob_minplus_direct_f64,
 * evolve and split steps with LOB_ENGINE_DIRECT — uses it):
 *  LOB_DIRECT_SCREENED (default): the O(n^2) sweep runs in fp32 with a
 *    rigorous error bound; per output only the span of 64-displacement
 *    sub-chunks that can hold the minimiser is re-evaluated in fp64.
 *    Results are the same doubles as the plain sweep.
 *  LOB_DIRECT_PLAIN: every candidate in fp64 (DADD + DSETP per candidate). */
#define LOB_DIRECT_SCREENED 0
#define LOB_DIRECT_PLAIN 1
int lob_ctx_set_direct_mode(lob_ctx* ctx, int mode);
/* Screened-K1 counters since the last reset (synchronizes): outputs swept in
 * full fp64 (non-finite screen) and fp64 candidates re-evaluated in total. */
int lob_direct_stats(lob_ctx* ctx, uint64_t* full_outputs, uint64_t* fp64_candidates, int reset);

/* K1 — fp32 variant (no potential; the reference has no fp32 path). */
int lob_minplus_direct_f32(lob_ctx* ctx, const float* u, float* out, int64_t lines, int64_t n,
                           const float* ktab, int64_t ktab_stride, const int64_t* first,
                           void* stream);

/* K1 on windowed (non-periodic) lines of m samples (proj/src/scheme.cpp:135-144):
 *   out[l][j] = min over w with 0 <= j-first-w < m of u[l][j-first-w] + ktab_l[w]
 * Returns LOB_EVALUATION_ERROR when an output has no candidate
 * (j - first outside the convolution, proj/src/scheme.cpp:138-141). */
int lob_minplus_window_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t m,
                           int64_t n, const double* ktab, int64_t ktab_stride,
                           const int64_t* first, const double* tv, int64_t tv_stride,
                           void* stream);

/* K2 — fast exact min-plus for mechanical kinetics K*(v) = v^2/2 - drift*v.
 * Replaces conv_fast (proj/src/minplus.cpp:219-252) in kinetic_convolve.
 * The kernel window is evaluated on the device with the exact IEEE operation
 * sequence of build_kernel (proj/src/scheme.cpp:79-80,
 * proj/src/hamiltonian.cpp:43), so values are bit-identical to the table.
 * drift: device array of `lines` doubles; n_space = n; tau > 0.
 * blocks (nullable, device int64[lines]) receives decompose(u, eta)'s block
 * count of the INPUT u (what StepStats.block_count reports).
 * The workspace carries per-tile statistics of u between consecutive calls:
 * pass LOB_FAST_STATS_VALID when `u` is the `out` of the previous call with
 * the same workspace, drift, tau and n (the device-resident evolve loop),
 * else 0 and the statistics are recomputed (one extra read of u).  The flag is a promise:
 * u modified in place under the same pointer between the calls is not detected (the clamps
 * keep every access in bounds, the minima may be wrong).  Lines of n <= 2048 samples without
 * block counts run the whole-line kernel (K2L), which carries no statistics and ignores the
 * flag (lob_ctx_set_fast_line). */
#define LOB_FAST_STATS_VALID 1
/* With LOB_FAST_STATS_VALID: nothing else ran on `stream` since the previous
 * lob_minplus_fast_f64 call on this workspace (whose out is this u), so each
 * tile may start as soon as its own line's previous step is done instead of
 * after the whole previous grid (back-to-back stepping loops). */
#define LOB_FAST_CHAINED 2
/* With LOB_FAST_STATS_VALID: verify the promise.  Each step stores 32 samples of its output
 * (positions (k n) >> 5) with the statistics; a checked call compares its input u with them
 * bitwise, and a line whose samples differ (u modified in place under the same pointer) takes the
 * exact direct formula in every tile, counted in lob_fast_diagnostics [10].  A sampled check: a
 * modification that touches none of the 32 positions is not seen. */
#define LOB_FAST_STATS_CHECK 4
int lob_fast_workspace_bytes(int64_t lines, int64_t n, size_t* bytes);
int lob_minplus_fast_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                         const double* drift, double tau, const double* tv, int64_t tv_stride,
                         double eta, int64_t* blocks, void* workspace, size_t workspace_bytes,
                         int flags, void* stream);

/* K2 for ANY convex kernel window: the same exact O(n) walk, with each source's
 * local-minimum interval found by a hinted search over the window's
 * nondecreasing slopes sigma(w) = ktab[w+1] - ktab[w] (rounding of both sides
 * of every slope comparison relaxed, so the candidate set still encloses every
 * minimiser) and K read from the table itself.  This is the engine that plugs
 * into kinetic_convolve(u, kernel, eta, engine, blocks)
 * (proj/include/laxol/scheme.hpp:52-53; dispatch proj/src/scheme.cpp:114-121):
 * the reference's Kernel carries exactly the window (mechanical or tabulated,
 * proj/src/scheme.cpp:59-105).  Table conventions as lob_minplus_direct_f64
 * (ktab_stride 0 = one window for all lines; first: device int64[lines]);
 * tau must be > 0 but is otherwise unused (every cost comes from the window); flags/workspace/blocks as
 * lob_minplus_fast_f64 (the workspace remembers the table: another table
 * recomputes the statistics). */
int lob_minplus_fast_window_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                                const double* ktab, int64_t ktab_stride, const int64_t* first, double tau,
                                const double* tv, int64_t tv_stride, double eta, int64_t* blocks, void* workspace,
                                size_t workspace_bytes, int flags, void* stream);

/* Diagnostic hook: replace the fast engine's slope-inversion tolerance delta (in
 * displacement units) for the line constants computed from now
 * on; NaN restores the computed bound.  A delta below the bound lets the walk miss
 * minimisers: outputs no interval reaches are recomputed by the exact direct scan and
 * counted (lob_fast_diagnostics [0]), but an output still reached by a non-minimal source
 * comes out too large -- the hook exists to show that the computed bound is load-bearing. */
int lob_ctx_set_fast_delta(lob_ctx* ctx, double delta);

/* Fast-engine counters, cumulative since the last call without
 * LOB_FAST_STATS_VALID on this workspace (counters[16]; unused entries 0):
 *  [0] outputs no local-minimum interval reached, recomputed by the exact
 *      direct scan (0 in correct operation),
 *  [1] sources scanned by the walk, [2] candidates of queued intervals (long
 *  or contended: finished by a whole warp), [3] queued intervals,
 *  [4] tiles, [5] walk tiles whose K range did not fit the shared-memory stage,
 *  [6] sum of the walk tiles' K range lengths,
 *  [7] tiles computed by the direct formula because the oscillation gate failed
 *      (max u - min u not below the window's edge gap, non-finite u, or a
 *      window outside the cached v_d table),
 *  [8] tiles computed by the direct formula because the walk's estimated
 *      candidate count exceeded a quarter of the window's,
 *  [9] chained-step waits that timed out (a misused LOB_FAST_CHAINED; the
 *      results of that call are not trustworthy),
 *  [10] lines whose LOB_FAST_STATS_CHECK samples differed from u (per tile),
 *  [11] tiles whose carried line constants (LOB_FAST_STATS_VALID) no longer
 *       matched the caller's drift / window (another table at a reused address,
 *       a drift changed in place): computed by the direct formula with the
 *       current inputs (exact). */
int lob_fast_diagnostics(lob_ctx* ctx, void* workspace, int64_t lines, int64_t n,
                         uint64_t* counters);

/* K3 — split_step_nd (proj/src/splitting.cpp:37-99) for a periodic n x n
 * row-major tensor: sweep axis 0 (columns, kernel 1), sweep axis 1 (rows,
 * kernel 2), then subtract tau*V once.  The potential is the separable
 * descriptor V(t,x1,x2) = a1[i]*a2[k] + b  (each product and sum one IEEE
 * rounding, as the C++ expression a1*a2 + b), i.e. the reference's
 * PotentialNd callback evaluated on the host per axis and per step;
 * a1 == NULL means V == 0.  tmp: device scratch of n*n doubles.
 * engine LOB_ENGINE_DIRECT or LOB_ENGINE_FAST.  With LOB_ENGINE_FAST and n <= 2048
 * (the default lob_ctx_set_fast_line setting) the step is four launches without
 * workspace: 64x64 transpose, whole-line K2L sweep of axis 0, transpose, K2L sweep of
 * axis 1 with tau*(a1*a2 + b) in its epilogue.  Otherwise, with a workspace of
 * 2 x lob_fast_workspace_bytes(n, n): transpose + the tiled fast engine's input
 * statistics, sweep axis 0, transpose + statistics, sweep axis 1 with the potential in its
 * epilogue (one workspace half per axis); with a single lob_fast_workspace_bytes(n, n) the
 * unfused sequence runs.
 * Asynchronous on `stream` (the per-axis kernel tables are built once per
 * (n, tau, drift) and cached by the context). */
int lob_split_step_2d_f64(lob_ctx* ctx, const double* u, double* out, double* tmp, int64_t n,
                          double tau, double drift1, double drift2, const double* a1,
                          const double* a2, double b, int engine, void* workspace,
                          size_t workspace_bytes, void* stream);

/* split_step_nd (proj/src/splitting.cpp:37-99) for a periodic rank-`rank` tensor of n^rank
 * samples (row-major, every axis one unit period): sweep axis 0, 1, ..., rank-1 in the
 * reference's order (lines along axis a gathered by batched tiled transposes), then
 * out -= tv (tau*V of every point at the step's sampling time, rounded on the host; NULL =
 * V == 0).  Engines: LOB_ENGINE_DIRECT / LOB_ENGINE_RELAXED take the per-axis windows
 * ktabs[a*(2n+1) + w] (device) with firsts[a] (host) — any convex window, mechanical or
 * tabulated; LOB_ENGINE_FAST takes drifts[a] (host, mechanical axes) and a workspace of
 * lob_fast_workspace_bytes(n^(rank-1), n).  eta: the relaxed engine's tolerance.  u, out,
 * tmp: distinct device buffers of n^rank doubles.  Synchronous. */
int lob_split_step_nd_f64(lob_ctx* ctx, const double* u, double* out, double* tmp, int rank, int64_t n, double tau,
                          const double* ktabs, const int64_t* firsts, const double* drifts, const double* tv,
                          double eta, int engine, void* workspace, size_t workspace_bytes, void* stream);

/* The same for a windowed (non-periodic) tensor of dims[0] x ... x dims[rank-1] samples:
 * each axis swept with the wall branch of kinetic_convolve (K1 windowed, exact;
 * LOB_EVALUATION_ERROR when a grid index has no candidate, proj/src/scheme.cpp:138-141). */
int lob_split_step_nd_window_f64(lob_ctx* ctx, const double* u, double* out, double* tmp, int rank,
                                 const int64_t* dims, int64_t n, double tau, const double* ktabs,
                                 const int64_t* firsts, const double* tv, void* stream);

/* The potential pass of K3 on a rows x n row slab (the multi-GPU split step's
 * rows [r0, r0 + rows) of an n x n tensor): out[i][k] -= tau*(a1[i]*a2[k] + b),
 * each product / sum one IEEE rounding (a1 points at the slab's first row). */
int lob_potential2d_rows_f64(lob_ctx* ctx, double* out, int64_t rows, int64_t n, const double* a1,
                             const double* a2, double b, double tau, void* stream);

/* The multi-GPU split step's all-to-all exchange of row slabs (paper_1210_4090_b200/dist.py;
 * rank r holds rows [r*b, (r+1)*b) of an n x n tensor, n = b*world):
 * pack:   send[q][c][i] = x[i][q*b + c]  (block q goes to rank q; the slab transposed),
 * unpack: y[c][p*b + i] = recv[p][c][i]  (this rank's slab of the transposed tensor).
 * Device buffers of b*n doubles, asynchronous on `stream`. */
int lob_slab_pack_f64(lob_ctx* ctx, const double* x, int64_t b, int64_t world, double* send, void* stream);
int lob_slab_unpack_f64(lob_ctx* ctx, const double* recv, int64_t b, int64_t world, double* y, void* stream);
/* The same exchange as ONE kernel over NVLink peer memory, replacing pack + all-to-all + unpack:
 * this rank (`rank` of `world`, row slab x of b x n doubles, n = b*world, b % 64 == 0) writes
 * X^T's blocks straight into every rank's receive slab: R_q[c][rank*b + i] = x[i][q*b + c]
 * (R_q = rank q's b x n slab of X^T).  peer_slabs: host array of `world` device addresses of the
 * receive slabs, valid on this device (CUDA symmetric memory / IPC mappings; this rank's own
 * entry included), world <= 16.  Asynchronous on `stream`; the ranks synchronise after it (e.g.
 * a symmetric-memory barrier) before reading their slabs. */
int lob_slab_push_f64(lob_ctx* ctx, const double* x, int64_t b, int64_t world, int rank, const uint64_t* peer_slabs,
                      void* stream);

/* Device-resident batched evolve (proj/src/scheme.cpp:208-272): `steps`
 * steps of `lines` periodic lines with a shared, time-independent tv.  u is
 * updated in place (double-buffered against `scratch`, n*lines doubles).
 * Per-step drift (mean of u_next - u, fp64, device reduction) and block
 * counts are written to step_drift[steps*lines] / step_blocks[steps*lines]
 * (device, nullable).  Returns LOB_EVALUATION_ERROR (after finishing the
 * step) if a non-finite value appears; *completed_steps receives the number
 * of steps done. */
int lob_evolve_f64(lob_ctx* ctx, double* u, double* scratch, int64_t lines, int64_t n,
                   const double* drift, double tau, const double* tv, int64_t tv_stride,
                   double eta, int engine, int64_t steps, double* step_drift,
                   int64_t* step_blocks, int64_t* completed_steps, void* workspace,
                   size_t workspace_bytes, void* stream);

/* lob_evolve_f64 with LOB_ENGINE_FAST runs every step of the call in ONE launch with the
 * lines resident in shared memory (K2R, one CTA per line) when n <= 4096 and the batch is
 * too small to fill the GPU step by step (lines * ceil(n/2048) <= 4 * SMs).  Same doubles as
 * the step-by-step loop.  on = 0 always selects the step-by-step K2 launches (default 1). */
int lob_ctx_set_evolve_resident(lob_ctx* ctx, int on);
/* Diagnostic switch (default on): the fast engine on lines of n <= 2048 samples without block
 * counts runs one CTA per whole line with the oscillation gate and displacement range reduced
 * from the staged line (K2L; the 2-D split step's axis-0 sweep then reads and writes columns in
 * place).  Off: the tiled kernel with carried statistics.  Both give the same doubles. */
int lob_ctx_set_fast_line(lob_ctx* ctx, int on);

/* Host-buffer entry point (the e2e path): one step of `lines` lines whose u,
 * out, drift and tv live in host memory (pinned or pageable).  Copies in,
 * runs K1/K2 on the context's stream, copies out, synchronizes. */
int lob_step_host_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                      const double* drift, double tau, const double* tv, int64_t tv_stride,
                      double eta, int engine, int64_t* blocks);

/* Kernel window of mechanical(drift) built on the host exactly as
 * build_kernel does (proj/src/scheme.cpp:59-105): window[2n+1], first,
 * argmin, and the fast path's slope-inversion tolerance delta (in
 * displacement units).  ctx may be NULL. */
int lob_kernel_mech_host(lob_ctx* ctx, int64_t n, double tau, double drift, double* window,
                         int64_t* first, int64_t* argmin, double* delta);

/* Kernel window of a TABULATED conjugate (proj/src/hamiltonian.cpp:30-82 tabulated /
 * kstar / argmin_velocity, proj/src/scheme.cpp:59-105 with its monotone slope repair):
 * `count` convex samples at velocities v0 + i*dv.  window[2n+1], first, argmin as for
 * lob_kernel_mech_host.  Use with the direct (K1) and relaxed engines, which take any
 * table; K2 is for the mechanical conjugate.  ctx may be NULL. */
int lob_kernel_tabulated_host(lob_ctx* ctx, int64_t n, double tau, const double* samples, int64_t count,
                              double v0, double dv, double* window, int64_t* first, int64_t* argmin);

/* Decomposition block counts of device lines (decompose, proj/src/minplus.cpp:152-188,
 * on the closed period; capped counts are not supported: eta must be 0 or the
 * uncapped count is returned). blocks: device int64[lines]. */
int lob_block_counts(lob_ctx* ctx, const double* u, int64_t lines, int64_t n, double eta,
                     int64_t* blocks, void* stream);

/* Micro-benchmarks of the FP64 pipe on this device: the sustained rate of
 * the min-plus candidate instruction mix (DADD + DSETP + 2 FSEL) and of a
 * pure DADD stream, in operations per second (FP64 lane-ops). */
int lob_bench_fp64(lob_ctx* ctx, double* minplus_cand_per_s, double* dadd_ops_per_s,
                   double* sm_clock_ghz);

/* ---- Weak-KAM consumers of the step (proj/src/weakkam.cpp) ----
 * Dense min-plus matrices are row-major doubles, cost[y*n + x] = cost of going
 * from source y to target x (MinPlusMatrix, proj/include/laxol/weakkam.hpp:22-29).
 * Every output is one minimum over single IEEE sums taken in increasing
 * contraction index with a strict "<", exactly the reference's loops. */

/* C[m x n] = A[m x k] (x) B[k x n]:  C[i][x] = min_z A[i][z] + B[z][x]
 * (device buffers, leading dimensions in elements).  Replaces
 * minplus_product (proj/src/weakkam.cpp:130-146; m = n = k) and minplus_apply
 * (:148-158; A = the line(s) u, B = the period matrix). */
int lob_minplus_gemm_f64(lob_ctx* ctx, const double* A, int64_t lda, const double* B, int64_t ldb,
                         double* C, int64_t ldc, int64_t m, int64_t n, int64_t k, void* stream);

/* Host helper: the quotient kinetic cost kinc[r] = min over displacements
 * d = r (mod n) in [first, first + 2n] of window[d - first]
 * (proj/src/weakkam.cpp:106-118), r = 0..n-1. */
int lob_period_kinetic_host(const double* window, int64_t first, int64_t n, double* kinc);

/* build_period_matrix (proj/src/weakkam.cpp:88-128): C = step_0 (x) ... (x)
 * step_{ell-1}, step_i[y][x] = kinc[(x - y) mod n] - tvs[i*n + x] (tvs = the
 * host-rounded tau*V at step i's sampling time, NULL = V == 0).  Device
 * buffers; scratch holds 2*n*n doubles. */
int lob_period_matrix_f64(lob_ctx* ctx, const double* kinc, const double* tvs, int64_t n,
                          int64_t ell, double* C, double* scratch, void* stream);

/* eigenvalue_karp (proj/src/weakkam.cpp:160-189) of the device n x n matrix M:
 * runs on `stream` (after whatever produced M there) and synchronizes it;
 * *lambda on the host.  LOB_INVALID_INPUT for n < 1 or a non-finite entry. */
int lob_eigenvalue_karp_f64(lob_ctx* ctx, const double* M, int64_t n, double* lambda, void* stream);

/* estimate_hbar_drift (proj/src/weakkam.cpp:43-86) for one periodic line of n
 * samples (host buffers): whole periods of ell = 1/tau fully discrete steps
 * on the device (engine K1 or K2, exact), the per-period increment
 * statistics on the host in the reference's order.  tvs: tv_count host tables
 * of n rounded tau*V values — 0 (V == 0), 1 (autonomous) or ell (table i for
 * step i of every period: the in-period time labels of apply_one_period,
 * :33-39).  Outputs (nullable): h_bar, residual, n_steps, converged, and
 * u_final (n doubles, the last state). */
int lob_hbar_drift_host_f64(lob_ctx* ctx, const double* u0, int64_t n, double drift, double tau,
                            const double* tvs, int64_t tv_count, int engine, int max_periods,
                            double tol, double* h_bar, double* residual, int64_t* n_steps,
                            int* converged, double* u_final);

/* fixed_point_residual (proj/src/weakkam.cpp:191-201): sup_j |T^1 u - u - h_bar|. */
int lob_fixed_point_residual_host_f64(lob_ctx* ctx, const double* u, int64_t n, double h_bar,
                                      double drift, double tau, const double* tvs,
                                      int64_t tv_count, int engine, double* residual);

/* ---- step_semidiscrete (proj/src/scheme.cpp:166-206) ----
 * The reference's built-in potential kinds (proj/include/laxol/hamiltonian.hpp:34-66):
 *   ZERO: 0;  CONST: value;
 *   COSINE: offset + amplitude * mod(omega*t) * cos(frequency * theta(x)),
 *           mod = 1 (TMOD_NONE), sin (TMOD_SIN) or cos (TMOD_COS),
 *           theta(x) = 2 pi (x - floor x) - pi. */
#define LOB_POTENTIAL_ZERO 0
#define LOB_POTENTIAL_CONST 1
#define LOB_POTENTIAL_COSINE 2
#define LOB_TMOD_NONE 0
#define LOB_TMOD_SIN 1
#define LOB_TMOD_COS 2
typedef struct lob_potential {
    int kind;
    double value;
    double offset;
    double amplitude;
    int frequency;
    int tmod;
    double omega;
} lob_potential;

/* One semi-discrete step of `lines` lines sharing the kernel window ktab
 * (2*n_space+1 device doubles at displacements first..first+2n) and V:
 *   out[l][j] = min_w u[l][src] + (ktab[w] - tau/q * trapezoid(V along y -> x_j))
 * periodic != 0: m == n_space samples per line (fundamental domain, sources
 * mod n); else m samples of a windowed domain starting at `origin`, sources
 * outside [0, m) skipped and LOB_EVALUATION_ERROR if an output has none.
 * quad_points in [1, 64].  Synchronous.  ZERO/CONST potentials give the
 * reference's doubles exactly; COSINE agrees to <= 1e-12 relative (the
 * spatial cos is the device's). */
int lob_step_semidiscrete_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t m,
                              int64_t n_space, int periodic, double origin, const double* ktab,
                              int64_t first, double t, double tau, const lob_potential* V,
                              int quad_points, void* stream);

/* ---- The reference's relaxed fast engine, eta > 0 ----
 * kinetic_convolve(u, kernel, eta, ConvEngine::Fast) + the potential for
 * periodic lines: decompose(u, eta) with the 48-sample cap, the slope merge /
 * envelope of every block with the whole window, min_pointwise, aliasing
 * (proj/src/minplus.cpp:152-276, proj/src/scheme.cpp:107-164).  For eta > 0
 * this is the reference's approximation, reproduced bit for bit; for
 * eta == 0 it is exact (== K1).  Same table conventions as
 * lob_minplus_direct_f64; blocks (nullable, device int64[lines]) receives the
 * reference's block_count (capped for eta > 0).  O(blocks x n) work, like the
 * reference.  Synchronous (reports min_pointwise's gap error). */
int lob_relaxed_workspace_bytes(int64_t lines, int64_t n, size_t* bytes);
int lob_minplus_relaxed_f64(lob_ctx* ctx, const double* u, double* out, int64_t lines, int64_t n,
                            const double* ktab, int64_t ktab_stride, const int64_t* first,
                            const double* tv, int64_t tv_stride, double eta, int64_t* blocks,
                            void* workspace, size_t workspace_bytes, void* stream);

/* ---- The reference's min-plus primitives on plain sequences (proj/include/laxol/minplus.hpp) ----
 * conv_naive (proj/src/minplus.cpp:116-126): out[k] = min_{i+j=k} f[i] + g[j], nf + ng - 1
 * outputs (device buffers), the reference's loop order (i ascending, strict "<"). */
int lob_minplus_conv_naive_f64(lob_ctx* ctx, const double* f, int64_t nf, const double* g, int64_t ng,
                               double* out, void* stream);
/* decompose (proj/src/minplus.cpp:152-188) of m device samples with tolerance eta: the block
 * list (kinds 0 convex / 1 concave, [start, end] sample ranges sharing boundary samples) up
 * to `capacity` entries on the host, *count = the number of blocks.  Synchronous. */
int lob_decompose_f64(lob_ctx* ctx, const double* u, int64_t m, double eta, int* kinds, int64_t* starts,
                      int64_t* ends, int64_t capacity, int64_t* count, void* stream);
/* conv_fast (proj/src/minplus.cpp:190-252) of a convex kernel (nk device samples) with a plain
 * sequence (nu device samples): out[nk + nu - 1] (device), *blocks (host) = the block count
 * (capped for eta > 0).  For eta > 0 the reference's relaxed approximation, bit for bit.
 * nk, nu >= 1 (a one-sample side gives the plain sums, as in the reference).  A kernel whose
 * slope drops is rejected like require_convex (proj/src/minplus.cpp:24-29): LOB_INVALID_INPUT
 * naming the first such segment.  Synchronous (min_pointwise's gap check -> LOB_INVALID_INPUT). */
int lob_conv_fast_f64(lob_ctx* ctx, const double* kern, int64_t nk, const double* u, int64_t nu, double eta,
                      double* out, int64_t* blocks, void* stream);

/* Number of kernel launches issued by this context since creation. */
int64_t lob_launch_count(const lob_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* LAXOL_B200_H */

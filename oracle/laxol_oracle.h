/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the thing measured or shipped.
 *
 * Plain-C restatement of the reference's hot-path arithmetic
 * (/root/reference/proj, the `laxol` C++20 library).  Each function cites
 * the reference file:line it restates.  Parity is pinned against the
 * reference itself (oracle/_ref, built from the reference sources by
 * oracle/Makefile) and against the golden vectors under tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.
 */
#ifndef LAXOL_ORACLE_H
#define LAXOL_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* build_kernel for mechanical(drift) (proj/src/scheme.cpp:59-105,
 * proj/src/hamiltonian.cpp:42-44): window[w] = tau*kstar(((first+w)*eps)/tau),
 * w = 0..2n; first = llround(tau*drift/eps) - n.  Returns 0, or 1 if the
 * window fails the exact convexity check (scheme.cpp:94-97). */
int orc_kernel_mech(int n_space, double tau, double drift, double* window, int64_t* first,
                    int64_t* argmin);

/* Definition-level periodic min-plus step (proj/tests/unit_scheme.cpp:176-194,
 * equal to kinetic_convolve: proj/src/scheme.cpp:107-146), fused with the
 * potential update of step_fully_discrete (proj/src/scheme.cpp:156-162):
 *   out[l][j] = min_w (u[l][(j-first_l-w) mod n] + K_l[w])  [- tv[l][j]]
 * tv = tau*V already rounded (host table); NULL = no potential.
 * ktab_stride / tv_stride 0 = shared across lines.  nthreads <= 0: all. */
void orc_direct_f64(const double* u, double* out, int64_t lines, int64_t n, const double* ktab,
                    int64_t ktab_stride, const int64_t* first, const double* tv,
                    int64_t tv_stride, int nthreads);

/* fp32 variant (the reference has no fp32 path; same loop on (float) inputs,
 * SURVEY.md section 8c). No potential. */
void orc_direct_f32(const float* u, float* out, int64_t lines, int64_t n, const float* ktab,
                    int64_t ktab_stride, const int64_t* first, int nthreads);

/* Windowed (non-periodic) kinetic_convolve (proj/src/scheme.cpp:135-144):
 * u has m samples at indices 0..m-1, kernel window 2n+1 with first;
 * out[j] = min over w with 0 <= j-first-w < m.  Returns 2 (EvaluationError)
 * if some output has no candidate. */
int orc_window_f64(const double* u, int64_t m, int64_t n, const double* ktab, int64_t first,
                   double* out);

/* conv_naive (proj/src/minplus.cpp:116-126): out[k] = min_{i+j=k} a[i]+b[j]. */
void orc_conv_naive(const double* a, int64_t na, const double* b, int64_t nb, double* out);

/* decompose(u, eta) block count (proj/src/minplus.cpp:152-188) on a plain
 * sample vector of m samples (periodic lines pass the closed period, m=n+1).
 * capped != 0 applies capped_blocks (proj/src/minplus.cpp:198-215), which is
 * what conv_fast reports as block_count. */
int64_t orc_decompose_count(const double* v, int64_t m, double eta, int capped);

/* Periodic closed-period decomposition count of a fundamental-domain line
 * (appends the seam sample, as make_periodic does: proj/src/grid_fn.cpp:30-36). */
int64_t orc_line_blocks(const double* u, int64_t n, double eta, int capped);

/* split_step_nd for a periodic n1 x n2 row-major tensor
 * (proj/src/splitting.cpp:54-99): sweep axis 0 (columns), then axis 1 (rows),
 * then out -= tv (tv = tau*V, NULL = none). */
void orc_split2d_f64(const double* u, double* out, int64_t n1, int64_t n2, const double* k1,
                     int64_t first1, const double* k2, int64_t first2, const double* tv,
                     int nthreads);

/* Per-step drift of evolve (proj/src/scheme.cpp:244-251): sequential sum of
 * (next[j]-u[j]) over j < n divided by n; *finite = all next finite. */
double orc_drift(const double* next, const double* u, int64_t n, int* finite);

/* tv[j] = tau * v[j] (the rounding of proj/src/scheme.cpp:161). */
void orc_tau_v(const double* v, double tau, int64_t n, double* tv);

#ifdef __cplusplus
}
#endif
#endif

/* laxol_b200 synthetic workloads — seeded host generators for the five
 * BASELINE.json configurations.  No public dataset is
 * involved: every input is generated in-process from these formulas and
 * seeds, with glibc/libstdc++ math (the callbacks a reference user would
 * write), so the device path and the CPU oracle see bit-identical inputs.
 */
#ifndef LAXOL_B200_CONFIGS_H
#define LAXOL_B200_CONFIGS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* C1: u0[j] = sin(2*pi*x_j), x_j = j/n. */
void lob_gen_sin(int64_t n, double* u0);
/* V tables over x_j = j/n (time independent):
 *  kind 1: cos(2 pi x)                         (C1)
 *  kind 2: cos(2 pi x) + 0.5*cos(4 pi x + 1)   (C2)
 *  kind 3: 0.5*sin(2 pi x)                     (C5) */
void lob_gen_potential(int kind, int64_t n, double* v);
/* C2 drifts: P_l = -2 + 4*l/255 for l < lines (lines = 256 in C2). */
void lob_gen_c2_drifts(int64_t lines, double* drift);
/* C3: line l from mt19937_64(seed0 + l), increments U(-1/n, 1/n), made
 * periodic by subtracting the linear drift: u[i] = w[i] - w[n]*i/n. */
void lob_gen_c3_lines(int64_t line0, int64_t lines, int64_t n, uint64_t seed0, double* u);
/* C4: separable factors for u0 = sin(2 pi x1) + cos(2 pi x2) is not
 * separable in product form; this fills the full n x n tensor. */
void lob_gen_c4_u0(int64_t n, double* u);
/* C4 potential factors: a[i] = cos(2 pi x_i); b(t) = 0.2*sin(2 pi t). */
void lob_gen_cos(int64_t n, double* a);
double lob_c4_time_term(double t);
/* C5: line l from mt19937_64(seed0 + l): 64 modes k ~ U{1..256},
 * phi ~ U[0, 2 pi); u0 = sum sin(2 pi k x + phi)/k^2. Multithreaded. */
void lob_gen_c5_lines(int64_t line0, int64_t lines, int64_t n, uint64_t seed0, double* u,
                      int nthreads);

#ifdef __cplusplus
}
#endif
#endif

/* TEST INFRASTRUCTURE ONLY — CPU checker for the B200 hot path.
 * Plain-C restatement of the reference (/root/reference/proj); see
 * laxol_oracle.h for the per-function citations.  Built with
 * -ffp-contract=off so every sum is a single IEEE rounding, like the
 * reference built with its own flags (no -march).
 */
#include "laxol_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <pthread.h>
#include <string.h>
#include <unistd.h>

/* Minimal line-parallel loop over pthreads (the oracle's only concurrency;
 * results are per-line, so identical for any thread count). */
typedef struct {
    void (*body)(void*, int64_t);
    void* arg;
    int64_t count;
    int64_t next;
    pthread_mutex_t mu;
} pfor_t;

static void* pfor_worker(void* p) {
    pfor_t* f = (pfor_t*)p;
    for (;;) {
        pthread_mutex_lock(&f->mu);
        const int64_t i = f->next++;
        pthread_mutex_unlock(&f->mu);
        if (i >= f->count) return NULL;
        f->body(f->arg, i);
    }
}

static void parallel_for(int64_t count, int nthreads, void (*body)(void*, int64_t), void* arg) {
    if (nthreads <= 0) nthreads = (int)sysconf(_SC_NPROCESSORS_ONLN);
    if (nthreads > count) nthreads = (int)count;
    if (nthreads <= 1) {
        for (int64_t i = 0; i < count; ++i) body(arg, i);
        return;
    }
    pfor_t f = {body, arg, count, 0, PTHREAD_MUTEX_INITIALIZER};
    pthread_t th[256];
    if (nthreads > 256) nthreads = 256;
    for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, pfor_worker, &f);
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
}

static inline int64_t mod_i64(int64_t a, int64_t n) {
    int64_t r = a % n;
    return r < 0 ? r + n : r;
}

/* proj/src/scheme.cpp:59-105 with Kinetic::kstar for Mechanical
 * (proj/src/hamiltonian.cpp:42-44: 0.5*v*v - drift*v) and
 * argmin_velocity() == drift (proj/src/hamiltonian.cpp:57-58). */
int orc_kernel_mech(int n_space, double tau, double drift, double* window, int64_t* first_out,
                    int64_t* argmin_out) {
    const int n = n_space;
    const double eps = 1.0 / (double)n_space;
    const int64_t center = llround(tau * drift / eps);
    const int64_t first = center - n;
    const int64_t m = 2 * (int64_t)n + 1;
    for (int64_t i = 0; i < m; ++i) {
        const double x = (double)(first + i) * eps;
        const double v = x / tau;
        window[i] = tau * (0.5 * v * v - drift * v);
    }
    if (first_out) *first_out = first;
    int64_t arg = 0;
    for (int64_t i = 1; i < m; ++i)
        if (window[i] < window[arg]) arg = i;
    if (argmin_out) *argmin_out = arg;
    /* is_convex: proj/src/grid_fn.cpp:44-54 */
    for (int64_t i = 0; i + 2 < m; ++i) {
        const double lo = window[i + 1] - window[i];
        const double hi = window[i + 2] - window[i + 1];
        if (hi < lo) return 1;
    }
    return 0;
}

static void direct_line_f64(const double* u, double* out, int64_t n, const double* K,
                            int64_t first, const double* tv) {
    const int64_t W = 2 * n + 1;
    for (int64_t j = 0; j < n; ++j) {
        double best = INFINITY;
        int64_t y = mod_i64(j - first, n); /* source index for w = 0 */
        int64_t w = 0;
        while (w < W) {
            /* contiguous run y, y-1, ..., 0 */
            int64_t run = y + 1;
            if (run > W - w) run = W - w;
            const double* up = u + y;
            const double* kp = K + w;
            for (int64_t r = 0; r < run; ++r) {
                const double c = up[-r] + kp[r];
                best = (c < best) ? c : best; /* std::min(best, c) */
            }
            w += run;
            y = n - 1;
        }
        /* out[j] -= tau*V: proj/src/scheme.cpp:161 (two roundings, no FMA) */
        out[j] = tv ? best - tv[j] : best;
    }
}

typedef struct {
    const void* u;
    void* out;
    int64_t n;
    const void* ktab;
    int64_t ktab_stride;
    const int64_t* first;
    const double* tv;
    int64_t tv_stride;
} lines_arg_t;

static void direct_f64_body(void* p, int64_t l) {
    const lines_arg_t* a = (const lines_arg_t*)p;
    direct_line_f64((const double*)a->u + l * a->n, (double*)a->out + l * a->n, a->n,
                    (const double*)a->ktab + l * a->ktab_stride, a->first[l],
                    a->tv ? a->tv + l * a->tv_stride : NULL);
}

void orc_direct_f64(const double* u, double* out, int64_t lines, int64_t n, const double* ktab,
                    int64_t ktab_stride, const int64_t* first, const double* tv,
                    int64_t tv_stride, int nthreads) {
    lines_arg_t a = {u, out, n, ktab, ktab_stride, first, tv, tv_stride};
    parallel_for(lines, nthreads, direct_f64_body, &a);
}

static void direct_line_f32(const float* u, float* out, int64_t n, const float* K,
                            int64_t first) {
    const int64_t W = 2 * n + 1;
    for (int64_t j = 0; j < n; ++j) {
        float best = INFINITY;
        int64_t y = mod_i64(j - first, n);
        int64_t w = 0;
        while (w < W) {
            int64_t run = y + 1;
            if (run > W - w) run = W - w;
            const float* up = u + y;
            const float* kp = K + w;
            for (int64_t r = 0; r < run; ++r) {
                const float c = up[-r] + kp[r];
                best = (c < best) ? c : best;
            }
            w += run;
            y = n - 1;
        }
        out[j] = best;
    }
}

static void direct_f32_body(void* p, int64_t l) {
    const lines_arg_t* a = (const lines_arg_t*)p;
    direct_line_f32((const float*)a->u + l * a->n, (float*)a->out + l * a->n, a->n,
                    (const float*)a->ktab + l * a->ktab_stride, a->first[l]);
}

void orc_direct_f32(const float* u, float* out, int64_t lines, int64_t n, const float* ktab,
                    int64_t ktab_stride, const int64_t* first, int nthreads) {
    lines_arg_t a = {u, out, n, ktab, ktab_stride, first, NULL, 0};
    parallel_for(lines, nthreads, direct_f32_body, &a);
}

/* proj/src/scheme.cpp:135-144 over conv_naive (proj/src/minplus.cpp:116-126) */
int orc_window_f64(const double* u, int64_t m, int64_t n, const double* ktab, int64_t first,
                   double* out) {
    const int64_t W = 2 * n + 1;
    const int64_t size = W + m - 1;
    for (int64_t j = 0; j < m; ++j) {
        const int64_t r = j - first; /* conv index j + shift, shift = n - center */
        if (r < 0 || r >= size) return 2;
        double best = INFINITY;
        for (int64_t w = 0; w < W; ++w) {
            const int64_t k = r - w;
            if (k < 0 || k >= m) continue;
            const double c = u[k] + ktab[w];
            best = (c < best) ? c : best;
        }
        out[j] = best;
    }
    return 0;
}

void orc_conv_naive(const double* a, int64_t na, const double* b, int64_t nb, double* out) {
    for (int64_t k = 0; k < na + nb - 1; ++k) out[k] = INFINITY;
    for (int64_t i = 0; i < na; ++i)
        for (int64_t j = 0; j < nb; ++j) {
            const double c = a[i] + b[j];
            out[i + j] = (c < out[i + j]) ? c : out[i + j];
        }
}

/* proj/src/minplus.cpp:152-188 (decompose) and :198-215 (capped_blocks, cap 48) */
int64_t orc_decompose_count(const double* v, int64_t m, double eta, int capped) {
    const int64_t n = m - 1; /* segments */
    if (n <= 0) return 1;
    double* s = (double*)malloc((size_t)n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) s[i] = v[i + 1] - v[i];
    int64_t count = 0;
    int64_t b = 0;
    while (b < n) {
        int determined = 0, convex = 1;
        int64_t e = b + 1;
        while (e < n) {
            const double inc = s[e] - s[e - 1];
            if (!determined) {
                if (inc > eta) {
                    determined = 1;
                    convex = 1;
                } else if (inc < -eta) {
                    determined = 1;
                    convex = 0;
                }
            } else if (convex) {
                if (!(inc >= -eta)) break;
            } else {
                if (!(inc <= eta)) break;
            }
            ++e;
        }
        if (capped && eta > 0.0 && e - b > 48)
            count += (e - b + 47) / 48;
        else
            count += 1;
        b = e;
    }
    free(s);
    return count;
}

int64_t orc_line_blocks(const double* u, int64_t n, double eta, int capped) {
    double* v = (double*)malloc((size_t)(n + 1) * sizeof(double));
    memcpy(v, u, (size_t)n * sizeof(double));
    v[n] = u[0];
    const int64_t c = orc_decompose_count(v, n + 1, eta, capped);
    free(v);
    return c;
}

/* proj/src/splitting.cpp:54-99 with exact-min sweeps */
typedef struct {
    const double* src;
    double* dst;
    int64_t n1, n2;
    const double* k;
    int64_t first;
} sweep_arg_t;

static void sweep_col_body(void* p, int64_t c) {
    const sweep_arg_t* a = (const sweep_arg_t*)p;
    double* col = (double*)malloc((size_t)a->n1 * sizeof(double));
    double* res = (double*)malloc((size_t)a->n1 * sizeof(double));
    for (int64_t k = 0; k < a->n1; ++k) col[k] = a->src[k * a->n2 + c];
    direct_line_f64(col, res, a->n1, a->k, a->first, NULL);
    for (int64_t k = 0; k < a->n1; ++k) a->dst[k * a->n2 + c] = res[k];
    free(col);
    free(res);
}

static void sweep_row_body(void* p, int64_t r) {
    const sweep_arg_t* a = (const sweep_arg_t*)p;
    direct_line_f64(a->src + r * a->n2, a->dst + r * a->n2, a->n2, a->k, a->first, NULL);
}

void orc_split2d_f64(const double* u, double* out, int64_t n1, int64_t n2, const double* k1,
                     int64_t first1, const double* k2, int64_t first2, const double* tv,
                     int nthreads) {
    double* tmp = (double*)malloc((size_t)(n1 * n2) * sizeof(double));
    /* axis 0: gather column x2, sweep over x1 (splitting.cpp:67-76) */
    sweep_arg_t a0 = {u, tmp, n1, n2, k1, first1};
    parallel_for(n2, nthreads, sweep_col_body, &a0);
    /* axis 1: contiguous rows */
    sweep_arg_t a1 = {tmp, out, n1, n2, k2, first2};
    parallel_for(n1, nthreads, sweep_row_body, &a1);
    /* potential once, after the sweeps (splitting.cpp:80-97) */
    if (tv)
        for (int64_t i = 0; i < n1 * n2; ++i) out[i] = out[i] - tv[i];
    free(tmp);
}

double orc_drift(const double* next, const double* u, int64_t n, int* finite) {
    double drift = 0.0;
    int fin = 1;
    for (int64_t j = 0; j < n; ++j) {
        const double d = next[j] - u[j];
        drift += d;
        fin = fin && isfinite(next[j]);
    }
    if (finite) *finite = fin;
    return drift / (double)n;
}

void orc_tau_v(const double* v, double tau, int64_t n, double* tv) {
    for (int64_t j = 0; j < n; ++j) tv[j] = tau * v[j];
}

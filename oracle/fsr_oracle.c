/*
 * fsr_oracle.c -- CPU restatement of the fsrkit greedy iteration loop.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine in paper_2202_13926_b200/csrc; it is imported only by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg.
 * The product path never links or calls it.
 *
 * It restates, operation for operation, the numba kernel of the reference:
 *   lane_pass            pkg/src/fsrkit/_kernels.py:12-29
 *   tree_argmax          pkg/src/fsrkit/_kernels.py:32-49
 *   linear_argmax        pkg/src/fsrkit/_kernels.py:52-59
 *   reconstruct_iterations pkg/src/fsrkit/_kernels.py:62-126
 *   reconstruct_batch    pkg/src/fsrkit/_kernels.py:129-149
 * numba compiles that loop with strict IEEE double arithmetic (no fast-math,
 * no FMA contraction) and naive complex multiplication
 * ((a+bi)(c+di) = (ac-bd) + (ad+bc)i, numba/cpython/numbers.py), with a real
 * or integer operand promoted to a complex with zero imaginary part.  This
 * file must therefore be compiled with -ffp-contract=off and without
 * -ffast-math; tests/test_oracle.py pins it bitwise against the reference's
 * own outputs (tests/golden/).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <pthread.h>
#include <unistd.h>

typedef struct {
    double re, im;
} cplx;

/* numba complex128 * complex128 */
static inline cplx cmul(cplx x, cplx y) {
    double ac = x.re * y.re;
    double bd = x.im * y.im;
    double ad = x.re * y.im;
    double bc = x.im * y.re;
    cplx z = {ac - bd, ad + bc};
    return z;
}

/* _kernels.py:12-29: double-buffered lock-step lane reduction */
static void lane_pass(double *reg_obj, int64_t *reg_idx, int64_t active, int64_t width,
                      double *buf_obj, int64_t *buf_idx) {
    int64_t offset = width / 2;
    while (offset >= 1) {
        for (int64_t i = 0; i < active; ++i) {
            int64_t p = i + offset;
            if (p < active) {
                buf_obj[i] = reg_obj[p];
                buf_idx[i] = reg_idx[p];
            } else {
                buf_obj[i] = reg_obj[i];
                buf_idx[i] = reg_idx[i];
            }
        }
        for (int64_t i = 0; i < active; ++i) {
            if (buf_obj[i] > reg_obj[i]) {
                reg_obj[i] = buf_obj[i];
                reg_idx[i] = buf_idx[i];
            }
        }
        offset /= 2;
    }
}

/* _kernels.py:32-49.  Scratch arrays: reg/buf of `width`, win of ngroups. */
double oracle_tree_argmax(const double *obj, int64_t n, int64_t width, int64_t *best_idx) {
    int64_t ngroups = (n + width - 1) / width;
    double *reg_obj = (double *)malloc(sizeof(double) * (size_t)width);
    double *buf_obj = (double *)malloc(sizeof(double) * (size_t)(width > ngroups ? width : ngroups));
    int64_t *reg_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)width);
    int64_t *buf_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)(width > ngroups ? width : ngroups));
    double *win_obj = (double *)malloc(sizeof(double) * (size_t)ngroups);
    int64_t *win_idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)ngroups);
    for (int64_t g = 0; g < ngroups; ++g) {
        int64_t base = g * width;
        int64_t active = n - base;
        if (active > width) active = width;
        for (int64_t i = 0; i < active; ++i) {
            reg_obj[i] = obj[base + i];
            reg_idx[i] = base + i;
        }
        lane_pass(reg_obj, reg_idx, active, width, buf_obj, buf_idx);
        win_obj[g] = reg_obj[0];
        win_idx[g] = reg_idx[0];
    }
    lane_pass(win_obj, win_idx, ngroups, width, buf_obj, buf_idx);
    double o = win_obj[0];
    *best_idx = win_idx[0];
    free(reg_obj); free(buf_obj); free(reg_idx); free(buf_idx); free(win_obj); free(win_idx);
    return o;
}

/* _kernels.py:52-59: first flat index attaining the maximum */
double oracle_linear_argmax(const double *obj, int64_t n, int64_t *best_idx) {
    int64_t best = 0;
    for (int64_t t = 1; t < n; ++t)
        if (obj[t] > obj[best]) best = t;
    *best_idx = best;
    return obj[best];
}

/* _kernels.py:62-126.  residual/model/spectrum are S*S row-major complex128.
 * Returns the number of model updates applied. */
int64_t oracle_reconstruct_iterations(cplx *residual, cplx *model, const cplx *spectrum,
                                      const double *freq_weight, int64_t S, double gamma,
                                      int64_t iterations, int64_t width, int use_tree,
                                      double stop_threshold, double *objectives,
                                      int64_t *selections, uint8_t *tie_flags) {
    int64_t n = S * S;
    double w00 = spectrum[0].re;
    double *obj = (double *)malloc(sizeof(double) * (size_t)n);
    int64_t done = 0;
    for (int64_t it = 0; it < iterations; ++it) {
        for (int64_t t = 0; t < n; ++t) {
            cplx c = residual[t];
            obj[t] = freq_weight[t] * (c.re * c.re + c.im * c.im);
        }
        int64_t best_t;
        double best_obj = use_tree ? oracle_tree_argmax(obj, n, width, &best_t)
                                   : oracle_linear_argmax(obj, n, &best_t);
        int64_t ties = 0;
        for (int64_t t = 0; t < n; ++t)
            if (obj[t] == best_obj) ++ties;
        if (objectives) objectives[it] = best_obj;
        if (selections) selections[it] = best_t;
        if (tie_flags) tie_flags[it] = ties > 1 ? 1 : 0;

        if (stop_threshold > 0.0 && best_obj < stop_threshold) break;

        int64_t u = best_t / S;
        int64_t v = best_t - u * S;
        cplx c = residual[u * S + v];
        /* gp = gamma * complex(c.real / w00, c.imag / w00): float promoted to complex */
        cplx q = {c.re / w00, c.im / w00};
        cplx g = {gamma, 0.0};
        cplx gp = cmul(g, q);
        /* model[u, v] += gp * n: int64 promoted to complex */
        cplx nn = {(double)n, 0.0};
        cplx add = cmul(gp, nn);
        model[u * S + v].re = model[u * S + v].re + add.re;
        model[u * S + v].im = model[u * S + v].im + add.im;
        for (int64_t k = 0; k < S; ++k) {
            int64_t i = k - u;
            if (i < 0) i += S;
            for (int64_t l = 0; l < S; ++l) {
                int64_t j = l - v;
                if (j < 0) j += S;
                cplx t = cmul(gp, spectrum[i * S + j]);
                residual[k * S + l].re = residual[k * S + l].re - t.re;
                residual[k * S + l].im = residual[k * S + l].im - t.im;
            }
        }
        done = it + 1;
    }
    free(obj);
    return done;
}

/* _kernels.py:129-149 plus optional traces.  Blocks with W00 <= 0 are
 * skipped (model stays zero, done = 0).  Parallel over blocks with a pthread
 * pool pulling 16-block chunks from an atomic counter (the reference
 * parallelises the same independent blocks with a thread pool,
 * reconstruction.py:282-289; per-block arithmetic never depends on the
 * schedule, so results are bitwise identical for any thread count).
 * sel/obj/ties are [count, max(iterations,1)] and may be NULL; done may be NULL. */
typedef struct {
    int64_t count, S, iterations, width;
    cplx *residuals, *models;
    const cplx *spectra;
    const double *freq_weight, *stop_thresholds;
    double gamma;
    int use_tree;
    int64_t *sel;
    double *obj;
    uint8_t *ties;
    int64_t *done;
    int64_t next; /* atomic chunk cursor */
} batch_job;

static void run_block(batch_job *j, int64_t b) {
    int64_t n = j->S * j->S;
    int64_t it_stride = j->iterations > 0 ? j->iterations : 1;
    if (j->spectra[b * n].re <= 0.0) {
        if (j->done) j->done[b] = 0;
        return;
    }
    int64_t d = oracle_reconstruct_iterations(
        j->residuals + b * n, j->models + b * n, j->spectra + b * n, j->freq_weight, j->S,
        j->gamma, j->iterations, j->width, j->use_tree,
        j->stop_thresholds ? j->stop_thresholds[b] : 0.0, j->obj ? j->obj + b * it_stride : NULL,
        j->sel ? j->sel + b * it_stride : NULL, j->ties ? j->ties + b * it_stride : NULL);
    if (j->done) j->done[b] = d;
}

static void *batch_worker(void *arg) {
    batch_job *j = (batch_job *)arg;
    for (;;) {
        int64_t lo = __atomic_fetch_add(&j->next, 16, __ATOMIC_RELAXED);
        if (lo >= j->count) break;
        int64_t hi = lo + 16 < j->count ? lo + 16 : j->count;
        for (int64_t b = lo; b < hi; ++b) run_block(j, b);
    }
    return NULL;
}

int oracle_max_threads(void) {
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}

void oracle_reconstruct_batch(int64_t count, int64_t S, cplx *residuals, cplx *models,
                              const cplx *spectra, const double *freq_weight, double gamma,
                              int64_t iterations, int64_t width, int use_tree,
                              const double *stop_thresholds, int nthreads, int64_t *sel,
                              double *obj, uint8_t *ties, int64_t *done) {
    batch_job j = {count, S, iterations, width, residuals, models, spectra, freq_weight,
                   stop_thresholds, gamma, use_tree, sel, obj, ties, done, 0};
    if (nthreads < 1) nthreads = oracle_max_threads();
    if (nthreads == 1 || count <= 16) {
        batch_worker(&j);
        return;
    }
    pthread_t *tid = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    int started = 0;
    for (int i = 0; i < nthreads; ++i)
        if (pthread_create(&tid[i], NULL, batch_worker, &j) == 0) ++started;
    if (started == 0) batch_worker(&j);
    for (int i = 0; i < started; ++i) pthread_join(tid[i], NULL);
    free(tid);
}

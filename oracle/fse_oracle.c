/*
 * ORACLE — test infrastructure only.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's .so;
 * the product path (paper_2207_00233_b200) never does.
 *
 * Plain-C restatement of the reference's per-window model fit
 *   fsefill._kernel.run_fse        /root/reference/pkg/src/fsefill/_kernel.pyx:128-187
 *   fsefill._kernel._iterate       /root/reference/pkg/src/fsefill/_kernel.pyx:14-125
 * with the same contract as fsefill._kernel_py.run_fse (_kernel_py.py:13-30):
 *   values, weights: f64[m*n] row-major; iterations >= 0; gamma in (0, 1]
 *   -> coeff (re, im) f64[m*n], picks i32[iterations*2], energies f64[iterations+1],
 *      residual f64[m*n].
 *
 * The reference seeds the projection spectrum with numpy's pocketfft
 * (_kernel.pyx:147-148); this restatement uses the defining direct DFT sums
 * instead (the reference's own tests pin run_fse to direct summation at 1e-9,
 * /root/reference/pkg/tests/test_fse.py:106-129, tests/reference.py:14-20).
 * The selection loop keeps the reference's operation order and is compiled
 * with -ffp-contract=off so no FMA contraction changes its rounding.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* e^{sign * j 2 pi k / len}, k in [0, len) — table of the unit circle */
static void unit_circle(int len, double sign, double *re, double *im) {
    for (int k = 0; k < len; ++k) {
        double ang = 2.0 * M_PI * (double)k / (double)len;
        re[k] = cos(ang);
        im[k] = sign * sin(ang);
    }
}

/* Direct 2-D DFT of a real m x n plane: out[a,b] = sum x[i,j] e^{-j2pi(ai/m + bj/n)}.
 * Separable: first along columns (j), then rows (i). */
static void dft2_real(int m, int n, const double *x, double *out_re, double *out_im,
                      const double *cm_re, const double *cm_im,
                      const double *cn_re, const double *cn_im) {
    double *t_re = (double *)calloc((size_t)m * n, sizeof(double));
    double *t_im = (double *)calloc((size_t)m * n, sizeof(double));
    for (int i = 0; i < m; ++i)
        for (int b = 0; b < n; ++b) {
            double sr = 0.0, si = 0.0;
            for (int j = 0; j < n; ++j) {
                int k = (int)(((long)b * j) % n);
                sr += x[i * n + j] * cn_re[k];
                si += x[i * n + j] * cn_im[k];
            }
            t_re[i * n + b] = sr;
            t_im[i * n + b] = si;
        }
    for (int a = 0; a < m; ++a)
        for (int b = 0; b < n; ++b) {
            double sr = 0.0, si = 0.0;
            for (int i = 0; i < m; ++i) {
                int k = (int)(((long)a * i) % m);
                double xr = t_re[i * n + b], xi = t_im[i * n + b];
                sr += xr * cm_re[k] - xi * cm_im[k];
                si += xr * cm_im[k] + xi * cm_re[k];
            }
            out_re[a * n + b] = sr;
            out_im[a * n + b] = si;
        }
    free(t_re);
    free(t_im);
}

int oracle_run_fse(int m, int n, const double *values, const double *weights,
                   int iterations, double gamma,
                   double *coeff_re, double *coeff_im, int32_t *picks,
                   double *energies, double *residual) {
    if (m < 1 || n < 1 || iterations < 0) return -22;
    const size_t mn = (size_t)m * n;
    double *x = (double *)malloc(mn * sizeof(double));
    double *g_re = (double *)malloc(mn * sizeof(double));
    double *g_im = (double *)malloc(mn * sizeof(double));
    double *w_re = (double *)malloc(mn * sizeof(double));
    double *w_im = (double *)malloc(mn * sizeof(double));
    double *fm_re = (double *)malloc(m * sizeof(double)), *fm_im = (double *)malloc(m * sizeof(double));
    double *fn_re = (double *)malloc(n * sizeof(double)), *fn_im = (double *)malloc(n * sizeof(double));
    double *bm_re = (double *)malloc(m * sizeof(double)), *bm_im = (double *)malloc(m * sizeof(double));
    double *bn_re = (double *)malloc(n * sizeof(double)), *bn_im = (double *)malloc(n * sizeof(double));

    /* setup (_kernel.pyx:141-160): total weight, select-initialised residual,
     * spectra of w*r and of w, synthesis twiddles e^{+j2pi k/m}, e^{+j2pi k/n} */
    double total = 0.0, e0 = 0.0;
    for (size_t s = 0; s < mn; ++s) {
        total += weights[s];
        residual[s] = weights[s] > 0.0 ? values[s] : 0.0;
        x[s] = weights[s] * residual[s];
        e0 += weights[s] * residual[s] * residual[s];
        coeff_re[s] = 0.0;
        coeff_im[s] = 0.0;
    }
    energies[0] = e0;
    unit_circle(m, -1.0, fm_re, fm_im);
    unit_circle(n, -1.0, fn_re, fn_im);
    unit_circle(m, +1.0, bm_re, bm_im);
    unit_circle(n, +1.0, bn_re, bn_im);
    dft2_real(m, n, x, g_re, g_im, fm_re, fm_im, fn_re, fn_im);
    dft2_real(m, n, weights, w_re, w_im, fm_re, fm_im, fn_re, fn_im);

    for (int it = 0; it < iterations; ++it) {
        /* (1) basis selection: largest |g|^2, first maximum in row-major
         * order on ties (_kernel.pyx:32-44) */
        double best = -1.0;
        int a = 0, b = 0;
        for (int u = 0; u < m; ++u)
            for (int v = 0; v < n; ++v) {
                double e = g_re[u * n + v] * g_re[u * n + v] + g_im[u * n + v] * g_im[u * n + v];
                if (e > best) { best = e; a = u; b = v; }
            }
        picks[2 * it] = a;
        picks[2 * it + 1] = b;

        /* (2) projection coefficient (_kernel.pyx:46-48) */
        double pr = g_re[a * n + b] / total;
        double pi = g_im[a * n + b] / total;
        int selfconj = ((2 * a) % m == 0) && ((2 * b) % n == 0);

        /* (3) coefficient + spectrum update by the shifted weight spectrum */
        if (selfconj) { /* _kernel.pyx:50-64 */
            coeff_re[a * n + b] += gamma * pr;
            for (int u = 0; u < m; ++u) {
                int ru = (u - a + m) % m;
                for (int v = 0; v < n; ++v) {
                    int rv = ((v - b) % n + n) % n;
                    g_re[u * n + v] -= gamma * pr * w_re[ru * n + rv];
                    g_im[u * n + v] -= gamma * pr * w_im[ru * n + rv];
                }
            }
        } else { /* conjugate pair, _kernel.pyx:65-97 */
            int ta = (m - a) % m, tb = (n - b) % n;
            coeff_re[a * n + b] += gamma * pr;
            coeff_im[a * n + b] += gamma * pi;
            coeff_re[ta * n + tb] += gamma * pr;
            coeff_im[ta * n + tb] -= gamma * pi;
            for (int u = 0; u < m; ++u) {
                int lo_u = (u - a + m) % m, hi_u = (u + a) % m;
                for (int v = 0; v < n; ++v) {
                    int lo_v = ((v - b) % n + n) % n, hi_v = (v + b) % n;
                    double lr = w_re[lo_u * n + lo_v], li = w_im[lo_u * n + lo_v];
                    double hr = w_re[hi_u * n + hi_v], hi = w_im[hi_u * n + hi_v];
                    double tr = pr * (lr + hr) - pi * (li - hi);
                    double ti = pr * (li + hi) + pi * (lr - hr);
                    g_re[u * n + v] -= gamma * tr;
                    g_im[u * n + v] -= gamma * ti;
                }
            }
        }

        /* (4) spatial residual and weighted energy (_kernel.pyx:99-125) */
        double energy = 0.0;
        for (int i = 0; i < m; ++i) {
            int ki = (int)(((long)a * i) % m);
            double mr = bm_re[ki], mi = bm_im[ki];
            double sr, si;
            if (selfconj) { sr = gamma * pr * mr; si = gamma * pr * mi; }
            else { sr = 2.0 * gamma * (pr * mr - pi * mi); si = 2.0 * gamma * (pr * mi + pi * mr); }
            for (int j = 0; j < n; ++j) {
                int kj = (int)(((long)b * j) % n);
                double term = sr * bn_re[kj] - si * bn_im[kj];
                residual[i * n + j] -= term;
                energy += weights[i * n + j] * residual[i * n + j] * residual[i * n + j];
            }
        }
        energies[it + 1] = energy;
    }

    free(x); free(g_re); free(g_im); free(w_re); free(w_im);
    free(fm_re); free(fm_im); free(fn_re); free(fn_im);
    free(bm_re); free(bm_im); free(bn_re); free(bn_im);
    return 0;
}

/*
 * mds_oracle.c -- CPU ORACLE for the Bayesian-MDS hot path (arXiv 1905.04582).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_1905_04582_b200/, libmds.so) never links, imports
 * or calls anything here, and this file shares no code, header, constant or
 * helper with the CUDA path.
 *
 * What it computes is the plain definition, written out term by term:
 *
 *   PAPER.md:78-83  (Sec. 2.1, Eq. 1)   y_ij ~ N(delta_ij, sigma^2) I(y_ij > 0), i > j,
 *                                       delta_ij = ||x_i - x_j||.
 *   PAPER.md:84-112 (Eq. 2)             log p(Y|X,sigma^2) = sum_{i>j} [ -1/2 log(2 pi sigma^2)
 *                                        - (y_ij - delta_ij)^2/(2 sigma^2) - log Phi(delta_ij/sigma) ]
 *                                       (full normalised density per OBSERVED pair: DESIGN.md reading R2;
 *                                        sign of log Phi: reading R3).
 *   PAPER.md:338-348 (Eq. 6)            d/dx_i log p = - sum_{j != i} [ (delta_ij - y_ij)/sigma^2
 *                                        + phi(delta_ij/sigma)/(sigma Phi(delta_ij/sigma)) ] (x_i - x_j)/delta_ij
 *   PAPER.md:821-826 (App. B)           truncation flag T: T = 0 drops the log Phi term and its
 *                                       derivative (reading R12).
 *   PAPER.md:321-336 (Sec. 2.3, Eq. 5)  leapfrog integrator for HMC (readings R19, R20).
 *   PAPER.md:258-263                    single-location updates: "changing the value of a single
 *                                       x_i invalidates only N - 1 terms" (row delta, random-walk
 *                                       Metropolis sweep of Bedford et al.; reading R28).
 *   PAPER.md:381-395                    cross-validated log pointwise predictive density of a
 *                                       held-out fold over S posterior draws (reading R29).
 *   PAPER.md:205-210, 672               sigma^-2 ~ Gamma(s_0, r_0) and the per-iteration
 *                                       sigma^2 update: Metropolis-Hastings random walk on
 *                                       log sigma^2 (reading R27).
 *
 * Numerics: double precision only, libm erfc/log1p/exp/sqrt, i-major order
 * (i ascending, j ascending < i), Neumaier-compensated sums for log L and the
 * gradient.  Compile with -O2 -fno-fast-math -ffp-contract=off.
 *
 * Readings: NaN y = missing pair (R7);
 * only the strict lower triangle is read (R4, R9); delta = 0 for an observed
 * pair contributes its likelihood term but a zero gradient direction and is
 * counted (R10); log Phi(t) = log1p(-erfc(t/sqrt 2)/2) (R11).
 *
 * Every entry point returns 0 on success, -1 on invalid arguments.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

#define ORACLE_PI 3.14159265358979323846

/* ---- Neumaier (improved Kahan) compensated accumulator ------------------ */
typedef struct { double s, c; } acc_t;

static void acc_add(acc_t *a, double v)
{
    double t = a->s + v;
    if (fabs(a->s) >= fabs(v)) a->c += (a->s - t) + v;
    else                       a->c += (v - t) + a->s;
    a->s = t;
}
static double acc_val(const acc_t *a) { return a->s + a->c; }

/* ---- one pair, Eq. 2 term and Eq. 6 coefficient ------------------------- */
/* ell  = -1/2 log(2 pi sigma^2) - (y-d)^2/(2 sigma^2) - T log Phi(d/sigma)
 * coef = (d - y)/sigma^2 + T phi(d/sigma) / (sigma Phi(d/sigma))
 * so that the pair adds  -coef (x_i-x_j)/d  to g_i and  +coef (x_i-x_j)/d to g_j. */
int oracle_pair_term(double y, double d, double sigma, int truncation,
                     double *ell, double *coef)
{
    if (!(sigma > 0.0) || !isfinite(sigma) || !(d >= 0.0) || !isfinite(y)) return -1;
    double sigma2 = sigma * sigma;
    double t = d / sigma;
    double Q = 0.5 * erfc(t / sqrt(2.0));        /* 1 - Phi(t) */
    double logPhi = log1p(-Q);                   /* log Phi(t) */
    double phi = exp(-0.5 * t * t) / sqrt(2.0 * ORACLE_PI);
    double r = y - d;
    double e = -0.5 * log(2.0 * ORACLE_PI * sigma2) - (r * r) / (2.0 * sigma2);
    double c = (d - y) / sigma2;
    if (truncation) {
        e -= logPhi;
        c += phi / (sigma * (1.0 - Q));
    }
    if (ell) *ell = e;
    if (coef) *coef = c;
    return 0;
}

/* log Phi(t) for t >= 0 exactly as the oracle forms it (exposed for pins). */
double oracle_log_phi(double t) { return log1p(-0.5 * erfc(t / sqrt(2.0))); }

/* ---- log L over a range of rows (streaming; full-size configs) ----------- */
/* The Eq. 2 sum restricted to the pairs (i, j), i0 <= i < i1,
 * j < i: the same terms, order (i ascending, j ascending) and compensated sum
 * as oracle_loglik_grad, without the gradient.  y_rows holds rows i0..i1-1 of
 * the packed strict lower triangle back to back (row i: y_i0 .. y_i,i-1), so a
 * caller can stream an n too large for one packed array in row chunks and add
 * the chunk results in order.  Outputs: *loglik (this range's sum), *n_obs. */
int oracle_loglik_rows(int64_t n, int32_t d, int64_t i0, int64_t i1, const double *y_rows, const double *x,
                       double sigma, int32_t truncation, double *loglik, int64_t *n_obs)
{
    if (n < 2 || d < 1 || i0 < 0 || i1 > n || i0 > i1 || !x || !(sigma > 0.0) || !isfinite(sigma)) return -1;
    if (i1 > i0 && i1 > 1 && !y_rows) return -1;
    acc_t L = {0.0, 0.0};
    int64_t nobs = 0;
    const int64_t r0 = i0 > 1 ? i0 : 1;
    const int64_t base = (r0 * (r0 - 1)) / 2;
    for (int64_t i = r0; i < i1; ++i) {
        const double *yrow = y_rows + ((i * (i - 1)) / 2 - base);
        for (int64_t j = 0; j < i; ++j) {
            double y = yrow[j];
            if (isnan(y)) continue;                       /* missing (R7) */
            double s = 0.0;
            for (int k = 0; k < d; ++k) {
                double t = x[i * d + k] - x[j * d + k];
                s += t * t;
            }
            double ell;
            oracle_pair_term(y, sqrt(s), sigma, truncation, &ell, NULL);
            acc_add(&L, ell);
            ++nobs;
        }
    }
    if (loglik) *loglik = acc_val(&L);
    if (n_obs) *n_obs = nobs;
    return 0;
}

/* ---- full evaluation over the packed strict lower triangle -------------- */
/* y_packed: row i (i = 1..n-1) holds y_i0 .. y_i,i-1 at offset i(i-1)/2.
 * x: n*d row-major.  Outputs: *loglik, grad[n*d], absscale[n*d] (may be NULL:
 * S_ik = sum_j |v_ijk|, the conditioning scale of gradient entry ik),
 * *n_obs, *zero_pairs (observed pairs with delta = 0). */
int oracle_loglik_grad(int64_t n, int32_t d, const double *y_packed, const double *x,
                       double sigma, int32_t truncation,
                       double *loglik, double *grad, double *absscale,
                       int64_t *n_obs, int64_t *zero_pairs)
{
    if (n < 2 || d < 1 || !y_packed || !x || !(sigma > 0.0) || !isfinite(sigma)) return -1;
    acc_t L = {0.0, 0.0};
    acc_t *G = (acc_t *)calloc((size_t)n * (size_t)d, sizeof(acc_t));
    double *diff = (double *)malloc((size_t)d * sizeof(double));
    if (!G || !diff) { free(G); free(diff); return -1; }
    if (absscale) memset(absscale, 0, (size_t)n * (size_t)d * sizeof(double));
    int64_t nobs = 0, nzero = 0;

    for (int64_t i = 1; i < n; ++i) {
        const double *yrow = y_packed + (i * (i - 1)) / 2;
        for (int64_t j = 0; j < i; ++j) {
            double y = yrow[j];
            if (isnan(y)) continue;                       /* missing (R7) */
            double s = 0.0;
            for (int k = 0; k < d; ++k) {
                diff[k] = x[i * d + k] - x[j * d + k];
                s += diff[k] * diff[k];
            }
            double dist = sqrt(s);
            double ell, coef;
            oracle_pair_term(y, dist, sigma, truncation, &ell, &coef);
            acc_add(&L, ell);
            ++nobs;
            if (dist > 0.0) {
                for (int k = 0; k < d; ++k) {
                    double v = (coef * diff[k]) / dist;
                    acc_add(&G[i * d + k], -v);
                    acc_add(&G[j * d + k], v);
                    if (absscale) {
                        absscale[i * d + k] += fabs(v);
                        absscale[j * d + k] += fabs(v);
                    }
                }
            } else {
                ++nzero;                                   /* R10 */
            }
        }
    }
    if (loglik) *loglik = acc_val(&L);
    if (grad) for (int64_t q = 0; q < n * d; ++q) grad[q] = acc_val(&G[q]);
    if (n_obs) *n_obs = nobs;
    if (zero_pairs) *zero_pairs = nzero;
    free(G);
    free(diff);
    return 0;
}

/* ---- selected rows only (sampled parity at full size) ------------------- */
/* For each requested row i = rows[r]: yrows[r*n + j] holds y_ij for every
 * j != i (y_ij = y_ji; entry j == i ignored).  Outputs grad_rows[r*d+k] =
 * d log L / d x_ik (Eq. 6, all j != i), absscale_rows likewise, and
 * rowlik[r] = sum over j < i (observed) of the Eq. 2 term -- the row's share
 * of log L in the lower-triangle partition. */
int oracle_grad_rows(int64_t n, int32_t d, int64_t nrows, const int64_t *rows,
                     const double *yrows, const double *x, double sigma, int32_t truncation,
                     double *grad_rows, double *absscale_rows, double *rowlik)
{
    if (n < 2 || d < 1 || nrows < 0 || !(sigma > 0.0) || !isfinite(sigma)) return -1;
    double *diff = (double *)malloc((size_t)d * sizeof(double));
    acc_t *G = (acc_t *)malloc((size_t)d * sizeof(acc_t));
    if (!diff || !G) { free(diff); free(G); return -1; }
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        if (i < 0 || i >= n) { free(diff); free(G); return -1; }
        acc_t L = {0.0, 0.0};
        for (int k = 0; k < d; ++k) { G[k].s = 0.0; G[k].c = 0.0; }
        if (absscale_rows) for (int k = 0; k < d; ++k) absscale_rows[r * d + k] = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            double y = yrows[r * n + j];
            if (isnan(y)) continue;
            double s = 0.0;
            for (int k = 0; k < d; ++k) {
                diff[k] = x[i * d + k] - x[j * d + k];
                s += diff[k] * diff[k];
            }
            double dist = sqrt(s);
            double ell, coef;
            oracle_pair_term(y, dist, sigma, truncation, &ell, &coef);
            if (j < i) acc_add(&L, ell);
            if (dist > 0.0) {
                for (int k = 0; k < d; ++k) {
                    double v = (coef * diff[k]) / dist;
                    acc_add(&G[k], -v);
                    if (absscale_rows) absscale_rows[r * d + k] += fabs(v);
                }
            }
        }
        for (int k = 0; k < d; ++k) grad_rows[r * d + k] = acc_val(&G[k]);
        if (rowlik) rowlik[r] = acc_val(&L);
    }
    free(diff);
    free(G);
    return 0;
}

/* ---- HMC leapfrog (Sec. 2.3, Eq. 5) ------------------------------------- */
/* Target log pi(x) = log L(x) + log prior(x), prior iid N(0, prior_sd^2) per
 * coordinate (reading R20; prior_sd <= 0 means no prior), mass M = I (R19).
 * x (n*d) and p (n*d) are updated in place by n_steps leapfrog steps of size
 * eps:  p += eps/2 grad;  x += eps p;  p += eps/2 grad.
 * Outputs: H0 = -log pi(x0) + p0.p0/2 and H1 at the end, and the final
 * log L.  Returns -1 on bad arguments. */
static double prior_logpdf(int64_t m, const double *x, double prior_sd)
{
    if (!(prior_sd > 0.0)) return 0.0;
    acc_t a = {0.0, 0.0};
    for (int64_t q = 0; q < m; ++q) acc_add(&a, -(x[q] * x[q]) / (2.0 * prior_sd * prior_sd));
    return acc_val(&a);
}
static double kinetic(int64_t m, const double *p)
{
    acc_t a = {0.0, 0.0};
    for (int64_t q = 0; q < m; ++q) acc_add(&a, 0.5 * p[q] * p[q]);
    return acc_val(&a);
}

int oracle_leapfrog(int64_t n, int32_t d, const double *y_packed, double *x, double *p,
                    double sigma, int32_t truncation, double prior_sd,
                    double eps, int32_t n_steps, double *H0, double *H1, double *loglik_end)
{
    if (n < 2 || d < 1 || n_steps < 1 || !(eps > 0.0)) return -1;
    int64_t m = n * (int64_t)d;
    double *g = (double *)malloc((size_t)m * sizeof(double));
    if (!g) return -1;
    double ll;
    if (oracle_loglik_grad(n, d, y_packed, x, sigma, truncation, &ll, g, NULL, NULL, NULL)) { free(g); return -1; }
    if (prior_sd > 0.0) for (int64_t q = 0; q < m; ++q) g[q] -= x[q] / (prior_sd * prior_sd);
    if (H0) *H0 = -(ll + prior_logpdf(m, x, prior_sd)) + kinetic(m, p);
    for (int32_t s = 0; s < n_steps; ++s) {
        for (int64_t q = 0; q < m; ++q) p[q] += 0.5 * eps * g[q];
        for (int64_t q = 0; q < m; ++q) x[q] += eps * p[q];
        oracle_loglik_grad(n, d, y_packed, x, sigma, truncation, &ll, g, NULL, NULL, NULL);
        if (prior_sd > 0.0) for (int64_t q = 0; q < m; ++q) g[q] -= x[q] / (prior_sd * prior_sd);
        for (int64_t q = 0; q < m; ++q) p[q] += 0.5 * eps * g[q];
    }
    if (H1) *H1 = -(ll + prior_logpdf(m, x, prior_sd)) + kinetic(m, p);
    if (loglik_end) *loglik_end = ll;
    free(g);
    return 0;
}

/* ---- sigma^2 update (PAPER.md:205-210 prior, PAPER.md:672 update; R27) ---- */
/* One Metropolis-Hastings step on phi = log sigma^2 at fixed X:
 *   phi' = phi + step * z;  sigma' = exp(phi'/2)
 *   log r = log L(sigma') - log L(sigma) + log pi(phi') - log pi(phi)
 * where tau = 1/sigma^2 = exp(-phi) ~ Gamma(shape, rate) (density
 * rate^shape tau^(shape-1) e^(-rate tau) / Gamma(shape)), so the density of
 * phi is that times |d tau/d phi| = tau:  log pi(phi) = shape log tau - rate tau + const.
 * Accept iff log(u) < log r.  z and u are the caller's random numbers. */
int oracle_sigma_mh_step(int64_t n, int32_t d, const double *y_packed, const double *x,
                         double sigma, int32_t truncation, double shape, double rate,
                         double step, double z, double u,
                         double *sigma_out, int32_t *accepted, double *log_ratio)
{
    if (!(shape > 0.0) || !(rate > 0.0) || !(step > 0.0) || !(u > 0.0) || !(u <= 1.0)) return -1;
    double phi0 = log(sigma * sigma);
    double phi1 = phi0 + step * z;
    double sigma1 = exp(phi1 / 2.0);
    double ll0, ll1;
    if (oracle_loglik_grad(n, d, y_packed, x, sigma, truncation, &ll0, NULL, NULL, NULL, NULL)) return -1;
    if (oracle_loglik_grad(n, d, y_packed, x, sigma1, truncation, &ll1, NULL, NULL, NULL, NULL)) return -1;
    double tau0 = exp(-phi0), tau1 = exp(-phi1);
    double lp0 = shape * log(tau0) - rate * tau0;
    double lp1 = shape * log(tau1) - rate * tau1;
    double lr = (ll1 - ll0) + (lp1 - lp0);
    int ok = isfinite(lr) && log(u) < lr;
    if (sigma_out) *sigma_out = ok ? sigma1 : sigma;
    if (accepted) *accepted = ok;
    if (log_ratio) *log_ratio = lr;
    return 0;
}

/* ---- single-location updates (R28) --------------------- */
/* y_ij for i != j from the packed strict lower triangle (y_ij = y_ji). */
static double y_of(const double *y_packed, int64_t i, int64_t j)
{
    if (i < j) { int64_t t = i; i = j; j = t; }
    return y_packed[(i * (i - 1)) / 2 + j];
}

/* Delta = sum_{j != i observed} [ ell(y_ij, ||x_new - x_j||) - ell(y_ij, ||x_i - x_j||) ]
 * (Eq. 2 terms), in j order with a compensated sum. */
int oracle_row_delta(int64_t n, int32_t d, const double *y_packed, const double *x, int64_t i,
                     const double *x_new, double sigma, int32_t truncation, double *delta)
{
    if (n < 2 || d < 1 || i < 0 || i >= n || !(sigma > 0.0)) return -1;
    acc_t a = {0.0, 0.0};
    for (int64_t j = 0; j < n; ++j) {
        if (j == i) continue;
        double y = y_of(y_packed, i, j);
        if (isnan(y)) continue;
        double sn = 0.0, so = 0.0;
        for (int k = 0; k < d; ++k) {
            double dn = x_new[k] - x[j * d + k], dl = x[i * d + k] - x[j * d + k];
            sn += dn * dn;
            so += dl * dl;
        }
        double en, eo;
        oracle_pair_term(y, sqrt(sn), sigma, truncation, &en, NULL);
        oracle_pair_term(y, sqrt(so), sigma, truncation, &eo, NULL);
        acc_add(&a, en);
        acc_add(&a, -eo);
    }
    *delta = acc_val(&a);
    return 0;
}

/* k sequential random-walk Metropolis updates: i = rows[q],
 * x' = x_i + step z[q], log r = Delta_i(x') + log prior(x') - log prior(x_i)
 * (iid N(0, prior_sd^2), none if prior_sd <= 0), accept iff log(u[q]) < log r.
 * x (n*d) is updated in place; *accepted counts. */
int oracle_rw_sweep(int64_t n, int32_t d, const double *y_packed, double *x, double sigma, int32_t truncation,
                    int64_t k, const int64_t *rows, const double *z, const double *u, double step,
                    double prior_sd, int64_t *accepted)
{
    if (n < 2 || d < 1 || k < 0 || !(step > 0.0)) return -1;
    double *xn = (double *)malloc((size_t)d * sizeof(double));
    if (!xn) return -1;
    int64_t na = 0;
    for (int64_t q = 0; q < k; ++q) {
        int64_t i = rows[q];
        if (i < 0 || i >= n) { free(xn); return -1; }
        for (int c = 0; c < d; ++c) xn[c] = x[i * d + c] + step * z[q * d + c];
        double dl;
        oracle_row_delta(n, d, y_packed, x, i, xn, sigma, truncation, &dl);
        double lp = 0.0;
        if (prior_sd > 0.0)
            for (int c = 0; c < d; ++c)
                lp += -(xn[c] * xn[c]) / (2.0 * prior_sd * prior_sd) + (x[i * d + c] * x[i * d + c]) / (2.0 * prior_sd * prior_sd);
        double lr = dl + lp;
        if (isfinite(lr) && log(u[q]) < lr) {
            for (int c = 0; c < d; ++c) x[i * d + c] = xn[c];
            ++na;
        }
    }
    if (accepted) *accepted = na;
    free(xn);
    return 0;
}

/* ---- cross-validation lpd (R29) ------------------------ */
/* lpd = sum_q log( (1/S) sum_s p(y_q | X_s, sigma_s) ), p the Eq. 1 density,
 * log p = the Eq. 2 term.  Draws: xs[s*n*d ...] (S x n x d), sigmas[S].
 * Each log-mean-exp is formed with the max shift: m + log(sum exp(l - m)) - log S. */
int oracle_cv_lpd(int64_t n, int32_t d, int64_t m, const int64_t *hi, const int64_t *hj, const double *hy,
                  int64_t S, const double *xs, const double *sigmas, int32_t truncation, double *lpd)
{
    if (n < 2 || d < 1 || m < 0 || S < 1) return -1;
    double *l = (double *)malloc((size_t)S * sizeof(double));
    if (!l) return -1;
    acc_t tot = {0.0, 0.0};
    for (int64_t q = 0; q < m; ++q) {
        int64_t i = hi[q], j = hj[q];
        if (i < 0 || i >= n || j < 0 || j >= n || i == j) { free(l); return -1; }
        double mx = -INFINITY;
        for (int64_t s = 0; s < S; ++s) {
            const double *x = xs + s * n * d;
            double ss = 0.0;
            for (int k = 0; k < d; ++k) {
                double df = x[i * d + k] - x[j * d + k];
                ss += df * df;
            }
            oracle_pair_term(hy[q], sqrt(ss), sigmas[s], truncation, &l[s], NULL);
            if (l[s] > mx) mx = l[s];
        }
        double se = 0.0;
        for (int64_t s = 0; s < S; ++s) se += exp(l[s] - mx);
        acc_add(&tot, mx + log(se) - log((double)S));
    }
    *lpd = acc_val(&tot);
    free(l);
    return 0;
}

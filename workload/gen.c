/*
 * gen.c -- seeded synthetic MDS workloads (shared input generator).
 *
 * This module is neither the oracle nor the product path: it only draws
 * inputs, and both sides consume exactly the arrays it writes.  It holds
 * none of the likelihood/gradient arithmetic; it simulates the DATA model of
 * PAPER.md:78-83 (Eq. 1): y_ij ~ N(delta*_ij, sigma*^2) truncated to y > 0.
 *
 * Every random number is a pure function of (seed, stream tag, indices)
 * through a splitmix64 hash chain, so any element (i, j) can be regenerated
 * on its own (used for sampled oracle checks at full size) and rows can be
 * produced in parallel with identical results.
 *
 * Recipe:
 *   clustered: K = 189 centres c_k ~ N(0, I_D) (PAPER.md:614, 189 countries),
 *              label(i) uniform on K, x*_i = c_label + N(0, 0.15^2 I_D)
 *   gaussian : x*_i ~ N(0, I_D)  ("randomly sampled Gaussian points")
 *   x0_i = x*_i + N(0, (0.1 sigma*)^2 I_D)   (evaluation state)
 *   y_ij, i > j: rejection draws N(delta*_ij, sigma*^2) until > 0; with
 *   probability p_missing the pair is NaN (missing).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stddef.h>

#define WL_TWO_PI 6.283185307179586476925286766559

static inline uint64_t mix64(uint64_t z)
{
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t key4(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b, uint64_t c)
{
    return mix64(seed ^ mix64(tag ^ mix64(a ^ mix64(b ^ mix64(c)))));
}

/* uniform in (0, 1] from the top 53 bits */
static inline double u01(uint64_t h) { return ((double)(h >> 11) + 1.0) * (1.0 / 9007199254740992.0); }

/* one standard normal for (seed, tag, a, b, c) by Box-Muller */
static double normal(uint64_t seed, uint64_t tag, uint64_t a, uint64_t b, uint64_t c)
{
    uint64_t h1 = key4(seed, tag, a, b, 2 * c);
    uint64_t h2 = key4(seed, tag, a, b, 2 * c + 1);
    return sqrt(-2.0 * log(u01(h1))) * cos(WL_TWO_PI * u01(h2));
}

/* threads for the row generators (0 = the OpenMP default); a launcher that
 * sets OMP_NUM_THREADS=1 per rank (torch.distributed.run) can raise it */
static int wl_threads = 0;
int wl_set_threads(int32_t n) { wl_threads = n > 0 ? n : 0; return 0; }

enum { TAG_CENTRE = 1, TAG_LABEL = 2, TAG_SPREAD = 3, TAG_X0 = 4, TAG_Y = 5, TAG_MISS = 6, TAG_GAUSS = 7 };

/* x_true, x0: n*d row-major. kind 0 = clustered, 1 = gaussian. */
int wl_latent(int64_t n, int32_t d, int32_t kind, uint64_t seed, double sigma_star,
              int32_t n_clusters, double x_true[], double x0[])
{
    if (n < 1 || d < 1 || n_clusters < 1) return -1;
    for (int64_t i = 0; i < n; ++i) {
        uint64_t lab = key4(seed, TAG_LABEL, (uint64_t)i, 0, 0) % (uint64_t)n_clusters;
        for (int32_t k = 0; k < d; ++k) {
            double v;
            if (kind == 0)
                v = normal(seed, TAG_CENTRE, lab, (uint64_t)k, 0) + 0.15 * normal(seed, TAG_SPREAD, (uint64_t)i, (uint64_t)k, 0);
            else
                v = normal(seed, TAG_GAUSS, (uint64_t)i, (uint64_t)k, 0);
            x_true[i * d + k] = v;
            if (x0) x0[i * d + k] = v + 0.1 * sigma_star * normal(seed, TAG_X0, (uint64_t)i, (uint64_t)k, 0);
        }
    }
    return 0;
}

/* y for the unordered pair (i, j), i != j; symmetric by construction. */
static double draw_y(int64_t n, int32_t d, const double *x_true, uint64_t seed,
                     double sigma_star, double p_missing, int64_t i, int64_t j)
{
    (void)n;
    int64_t a = i > j ? i : j, b = i > j ? j : i;
    if (p_missing > 0.0 && u01(key4(seed, TAG_MISS, (uint64_t)a, (uint64_t)b, 0)) <= p_missing)
        return NAN;
    double s = 0.0;
    for (int32_t k = 0; k < d; ++k) {
        double t = x_true[a * d + k] - x_true[b * d + k];
        s += t * t;
    }
    double dstar = sqrt(s);
    for (uint64_t attempt = 0;; ++attempt) {
        double y = dstar + sigma_star * normal(seed, TAG_Y, (uint64_t)a, (uint64_t)b, attempt);
        if (y > 0.0) return y;      /* acceptance >= 1/2 since dstar >= 0 */
    }
}

/* packed strict lower triangle rows [i0, i1): row i holds y_i0..y_i,i-1; out
 * points at the start of row i0 (offset i0(i0-1)/2 of the full packing). */
int wl_dissim_rows(int64_t n, int32_t d, const double x_true[], uint64_t seed, double sigma_star,
                   double p_missing, int64_t i0, int64_t i1, double out[])
{
    if (n < 2 || d < 1 || i0 < 0 || i1 > n || i0 > i1) return -1;
    int64_t base = (i0 * (i0 - 1)) / 2;
    if (i0 == 0) base = 0;
#pragma omp parallel for schedule(dynamic, 1) num_threads(wl_threads > 0 ? wl_threads : omp_get_max_threads())
    for (int64_t i = (i0 > 1 ? i0 : 1); i < i1; ++i) {
        double *row = out + ((i * (i - 1)) / 2 - base);
        for (int64_t j = 0; j < i; ++j)
            row[j] = draw_y(n, d, x_true, seed, sigma_star, p_missing, i, j);
    }
    return 0;
}

/* full rows for selected i: out[r*n + j] = y_{rows[r], j}, NaN at j == i. */
int wl_dissim_full_rows(int64_t n, int32_t d, const double x_true[], uint64_t seed, double sigma_star,
                        double p_missing, int64_t nrows, const int64_t rows[], double out[])
{
    if (n < 2 || d < 1 || nrows < 0) return -1;
#pragma omp parallel for schedule(static) num_threads(wl_threads > 0 ? wl_threads : omp_get_max_threads())
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        for (int64_t j = 0; j < n; ++j)
            out[r * n + j] = (j == i) ? NAN : draw_y(n, d, x_true, seed, sigma_star, p_missing, i, j);
    }
    return 0;
}

/* iid standard normals (e.g. HMC momenta in tests), stream-tagged. */
int wl_normals(uint64_t seed, uint64_t stream, int64_t count, double out[])
{
    for (int64_t q = 0; q < count; ++q) out[q] = normal(seed, 100 + stream, (uint64_t)q, 0, 0);
    return 0;
}

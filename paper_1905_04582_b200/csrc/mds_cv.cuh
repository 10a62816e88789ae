// mds_cv.cuh -- cross-validated log pointwise predictive density
// (PAPER.md:381-395).
//
//   lpd_f = sum_{held-out pairs q of fold f} log( (1/S) sum_{s=1..S} p(y_q | X_s, sigma_s) )
// with p the truncated-normal density of Eq. 1, log p = the Eq. 2 term ell.
// (The printed estimator also multiplies each summand by the posterior density
// p(theta_s | Y_-IJ); a Monte Carlo average over posterior draws already
// carries that weight, so it is dropped: reading R29.)
//
// The held-out pairs are a compact list (i, j, y) -- a fold is a small part of
// the triangle -- with a per-pair running log-sum-exp (max m_q, scaled sum s_q)
// updated in place by one grid-stride kernel per posterior draw: O(m) work and
// O(m) state, no O(S) history.  The fold total is a fixed-order single-CTA
// reduction.  Held-out terms are evaluated in fp64 whatever the context's
// storage precision.
#pragma once
#include <cstdint>
#include "mds_math.cuh"

namespace mdsk {

struct CvArgs {
    const int2* ij;        // [m] (i, j), i != j
    const double* y;       // [m]
    const double* x;       // fp64 master X (n_pad x d)
    double* lmax;          // [m] running max of ell over draws
    double* lsum;          // [m] sum_s exp(ell_s - lmax)
    int64_t m;
    int d;
    int trunc;
    int first;             // 1 for the first draw (initialise)
    SigmaParams P;
};

void cv_accumulate_launch(const CvArgs& a, int grid, cudaStream_t s);
// out[0] = sum_q (lmax_q + log lsum_q) - m log S  (one CTA, fixed order)
void cv_finalize_launch(const double* lmax, const double* lsum, int64_t m, int64_t draws, double* out,
                        cudaStream_t s);

}  // namespace mdsk

// mds_row.cuh -- single-location updates.
//
// "changing the value of a single x_i invalidates only N - 1 terms": the change
// of log L when x_i alone moves to x', one row of the triangle,
//   Delta_i(x') = sum_{j != i, y_ij observed} [ ell(y_ij, ||x' - x_j||) - ell(y_ij, ||x_i - x_j||) ]
// (ell = the Eq. 2 term), is O(N D).  It drives the random-walk Metropolis
// sampler of Bedford et al. that the paper compares against: update i, propose
// x_i + step z, accept iff log u < Delta_i + Delta log prior.
//
// One thread-block cluster of 8 CTAs (8 SMs) evaluates one row: thread t of
// CTA r takes columns j = 512 r + t, + 4096, ... (y_ij gathered from the tiled
// triangle: for j > i the 32 lanes of a warp read one contiguous 256 B run of
// a tile column), both terms of a column in lock-step (pair_f64_n with NP = 2,
// likelihood only), a fixed-order block tree per CTA, and the 8 CTA partials
// summed in rank order through distributed shared memory: deterministic, no
// atomics.  A sweep of K sequential updates is ONE launch (the updates are
// dependent: the cluster loops with one cluster barrier per update, X stays
// in L2).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "mds_math.cuh"

namespace mdsk {

struct RowArgs {
    const void* y;              // local tiles (unsharded context: all of them)
    const int* row_local;       // [nb] local index of tile (I, 0)
    double* x;                  // fp64 master X, n_pad x D (updated in place by the sweep)
    int64_t n;
    // single delta (K == 0): row i0 moved to xnew
    int64_t i0;
    const double* xnew;         // [D]
    double* delta;              // out: Delta
    // sweep (K >= 1)
    int64_t K;
    const int64_t* rows;        // [K]
    const double* z;            // [K][D]
    const double* u;            // [K]
    double step;
    double inv_tau2;            // iid N(0, tau^2) prior; 0 = flat
    unsigned long long* accepted;
    SigmaParams P;
};

typedef void (*RowFn)(RowArgs);
constexpr int ROW_THREADS = 512;    // per CTA
constexpr int ROW_CLUSTER = 8;      // CTAs (SMs) per row: one thread-block cluster
// row_kernel<T, D, TRUNC> for (precision, truncation, d); defined in mds_row.cu
RowFn row_fn(int prec_is_f64, int trunc, int d);
// load the sweep's helper kernels now (CUDA lazy loading would otherwise load them at
// first launch, which waits for the device: see preload_kernels in mds_api.cu)
void rw_preload();
// sharded sweeps (mds_row.cu): proposal x_i + step z_q, and the decision from the
// gathered partial deltas gathered[r * stride], r < world (rank order)
void rw_propose_launch(const double* x, const int64_t* rows, const double* z, int64_t q, double step, int d,
                       double* xnew, cudaStream_t s);
void rw_decide_launch(const double* gathered, int world, int64_t stride, double* x, const int64_t* rows,
                      const double* u, int64_t q, const double* xnew, double inv_tau2, int d,
                      unsigned long long* accepted, cudaStream_t s);

}  // namespace mdsk

// mds_row.cu -- single-location update kernels (see mds_row.cuh).
#include <cooperative_groups.h>
#include "mds_row.cuh"

namespace mdsk {
namespace {

// y_ab (a > b) in the tiled triangle: tile (a/B, b/B), column-major inside
// (a sharded context stores only its own tile-rows: a pair of another rank's
// tile-row reads as missing, so each rank forms its share of the row delta)
template <typename T>
__device__ __forceinline__ T y_pair(const T* __restrict__ Y, const int* __restrict__ row_local, int64_t a, int64_t b) {
    const int lt = __ldg(row_local + (a >> 6));
    if (lt < 0) return T(NAN);
    return Y[((size_t)(lt + (b >> 6)) << 12) + ((b & 63) << 6) + (a & 63)];
}

template <typename T, bool TRUNC>
__device__ __forceinline__ void ell2(T s0, T s1, T y, const SigmaParams& P, const double* exptab, T& e0, T& e1);
template <>
__device__ __forceinline__ void ell2<double, true>(double s0, double s1, double y, const SigmaParams& P,
                                                   const double* exptab, double& e0, double& e1) {
    const double s[2] = {s0, s1}, yy[2] = {y, y};
    double l[2], u[2];
    pair_f64_n<true, 2, true, false>(s, yy, P, exptab, l, u);
    e0 = l[0];
    e1 = l[1];
}
template <>
__device__ __forceinline__ void ell2<double, false>(double s0, double s1, double y, const SigmaParams& P,
                                                    const double* exptab, double& e0, double& e1) {
    const double s[2] = {s0, s1}, yy[2] = {y, y};
    double l[2], u[2];
    pair_f64_n<false, 2, true, false>(s, yy, P, exptab, l, u);
    e0 = l[0];
    e1 = l[1];
}
template <>
__device__ __forceinline__ void ell2<float, true>(float s0, float s1, float y, const SigmaParams& P, const double*,
                                                  float& e0, float& e1) {
    float u;
    pair_f32<true, true, false>(s0, y, P, e0, u);
    pair_f32<true, true, false>(s1, y, P, e1, u);
}
template <>
__device__ __forceinline__ void ell2<float, false>(float s0, float s1, float y, const SigmaParams& P, const double*,
                                                   float& e0, float& e1) {
    float u;
    pair_f32<false, true, false>(s0, y, P, e0, u);
    pair_f32<false, true, false>(s1, y, P, e1, u);
}

// The first RPF columns of a thread (j = rank*NT + tid + c*CL*NT) are staged in
// registers one update ahead: y_ij (static) and x_j (patched if the update in
// between moved row j), so an update's gathers are already in flight while the
// previous one reduces and decides.
constexpr int RPF = 4;
template <typename T, int D>
struct RowCols {
    T y[RPF];
    T x[RPF][D];
};

template <typename T, int D>
__device__ __forceinline__ void row_stage(const RowArgs& a, int64_t i, int rank, RowCols<T, D>& c) {
    const T* __restrict__ Y = static_cast<const T*>(a.y);
#pragma unroll
    for (int q = 0; q < RPF; ++q) {
        const int64_t j = (int64_t)rank * ROW_THREADS + threadIdx.x + (int64_t)q * ROW_CLUSTER * ROW_THREADS;
        const bool ok = j < a.n && j != i;
        c.y[q] = ok ? (j < i ? y_pair<T>(Y, a.row_local, i, j) : y_pair<T>(Y, a.row_local, j, i)) : T(NAN);
#pragma unroll
        for (int k = 0; k < D; ++k) c.x[q][k] = ok ? (T)a.x[j * D + k] : T(0);
    }
}

// Row i's share of Delta owned by this CTA (columns j = rank*NT + tid, stride
// CL*NT) between positions xn and xo (both [D] in shared memory); the first
// RPF columns come staged in c.  Fixed order: per-thread sum over its columns in
// ascending j, warp butterfly, then the warp sums in order -> one partial per CTA.
template <typename T, int D, bool TRUNC>
__device__ double row_partial(const RowArgs& a, int64_t i, const double* xn, const double* xo, const double* exptab,
                              double* red, int rank, const RowCols<T, D>& c) {
    const T* __restrict__ Y = static_cast<const T*>(a.y);
    const double* X = a.x;     // not __restrict__/nc: the sweep writes X between updates
    double acc = 0.0;
    T xnr[D], xor_[D];
#pragma unroll
    for (int k = 0; k < D; ++k) {
        xnr[k] = (T)xn[k];
        xor_[k] = (T)xo[k];
    }
    auto term = [&](T y, const T* xj) {
        if (is_missing(y) || y != y) return;     // missing, or not a column of this thread
        T sn = T(0), so = T(0);
#pragma unroll
        for (int k = 0; k < D; ++k) {
            const T dn = xnr[k] - xj[k], dl = xor_[k] - xj[k];
            sn = fma(dn, dn, sn);
            so = fma(dl, dl, so);
        }
        T en, eo;
        ell2<T, TRUNC>(sn, so, y, a.P, exptab, en, eo);
        acc += double(en) - double(eo);
    };
#pragma unroll
    for (int q = 0; q < RPF; ++q) term(c.y[q], c.x[q]);
    for (int64_t j = (int64_t)rank * ROW_THREADS + threadIdx.x + (int64_t)RPF * ROW_CLUSTER * ROW_THREADS; j < a.n;
         j += (int64_t)ROW_CLUSTER * ROW_THREADS) {
        if (j == i) continue;
        const T y = j < i ? y_pair<T>(Y, a.row_local, i, j) : y_pair<T>(Y, a.row_local, j, i);
        T xj[D];
#pragma unroll
        for (int k = 0; k < D; ++k) xj[k] = (T)X[j * D + k];
        term(y, xj);
    }
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
        t = lane < ROW_THREADS / 32 ? red[lane] : 0.0;
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) t += __shfl_xor_sync(0xffffffffu, t, m);
    }
    return t;   // valid on warp 0
}

// One cluster of ROW_CLUSTER CTAs per launch: every update's N - 1 column pairs
// are split over the cluster's SMs; the CTA partials meet through distributed
// shared memory (double-buffered by update parity, one cluster barrier per
// update), and every CTA forms the same total in rank order, takes the same
// decision and writes the same new x_i -- so no X traffic crosses CTAs.
template <typename T, int D, bool TRUNC>
__global__ void __launch_bounds__(ROW_THREADS, 1) row_kernel(RowArgs a) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    __shared__ double exptab[EXPT64_N];
    __shared__ double red[ROW_THREADS / 32];
    __shared__ double part[2];
    __shared__ double xn[D], xo[D];
    __shared__ int decide;
    build_exptab(exptab, a.P);
    const int64_t K = a.K == 0 ? 1 : a.K;
    unsigned long long nacc = 0;
    RowCols<T, D> cur, nxt;
    // everything an update needs that does not depend on the previous decision is
    // loaded one update ahead: its row, the staged columns, x_i (patched if the
    // previous update moved the same row), z and u
    int64_t i_nx = a.K == 0 ? a.i0 : a.rows[0];
    row_stage<T, D>(a, i_nx, rank, nxt);
    double xi_nx = threadIdx.x < D ? a.x[i_nx * D + threadIdx.x] : 0.0;
    for (int64_t k = 0; k < K; ++k) {
        const int64_t i = i_nx;
        const double xi = xi_nx;
        cur = nxt;
        const double zk = (a.K > 0 && threadIdx.x < D) ? a.z[k * D + threadIdx.x] : 0.0;
        const double uk = (a.K > 0 && threadIdx.x == 0) ? a.u[k] : 1.0;
        if (k + 1 < K) {                       // in flight during this update
            i_nx = a.rows[k + 1];
            row_stage<T, D>(a, i_nx, rank, nxt);
            if (threadIdx.x < D) xi_nx = a.x[i_nx * D + threadIdx.x];
        }
        if (threadIdx.x < D) {
            xo[threadIdx.x] = xi;
            xn[threadIdx.x] = a.K == 0 ? a.xnew[threadIdx.x] : __fma_rn(a.step, zk, xi);
        }
        __syncthreads();
        // this update's proposal in registers: the patch below must not read xn after
        // the decision barrier (threads 0..D-1 overwrite it for the next update)
        double xn_r[D];
#pragma unroll
        for (int q = 0; q < D; ++q) xn_r[q] = xn[q];
        const double p = row_partial<T, D, TRUNC>(a, i, xn, xo, exptab, red, rank, cur);
        const int par = (int)(k & 1);
        if (threadIdx.x == 0) part[par] = p;
        cluster.sync();                    // every CTA's partial of this update is published
        if (threadIdx.x == 0) {
            double pr[ROW_CLUSTER];
#pragma unroll
            for (int r = 0; r < ROW_CLUSTER; ++r) pr[r] = *cluster.map_shared_rank(&part[par], r);
            double dl = 0.0;
#pragma unroll
            for (int r = 0; r < ROW_CLUSTER; ++r) dl += pr[r];
            if (a.K == 0) {
                if (rank == 0) *a.delta = dl;
                decide = 0;
            } else {
                // log prior change (iid N(0, tau^2)); the decision in fp64, identical on every CTA
                double pn = 0.0, po = 0.0;
#pragma unroll
                for (int q = 0; q < D; ++q) {
                    pn = fma(xn[q], xn[q], pn);
                    po = fma(xo[q], xo[q], po);
                }
                const double lr = dl - 0.5 * (pn - po) * a.inv_tau2;
                decide = isfinite(lr) && log(uk) < lr;
                if (decide) {
#pragma unroll
                    for (int q = 0; q < D; ++q) a.x[i * D + q] = xn[q];
                    ++nacc;
                }
            }
        }
        __syncthreads();   // this CTA's copy of X[i] (if accepted) is visible to its next column reads
        if (decide && k + 1 < K) {
            // values staged for the next update that predate this move of row i
            if (i_nx == i && threadIdx.x < D) xi_nx = xn_r[threadIdx.x];
#pragma unroll
            for (int q = 0; q < RPF; ++q) {
                const int64_t j = (int64_t)rank * ROW_THREADS + threadIdx.x + (int64_t)q * ROW_CLUSTER * ROW_THREADS;
                if (j == i) {
#pragma unroll
                    for (int kk = 0; kk < D; ++kk) nxt.x[q][kk] = (T)xn_r[kk];
                }
            }
        }
    }
    if (threadIdx.x == 0 && rank == 0 && a.K > 0) *a.accepted = nacc;
    cluster.sync();        // no CTA exits while another may still read its partials
}

template <typename T, bool TR>
RowFn row_fn_d(int d) {
    switch (d) {
        case 1: return row_kernel<T, 1, TR>;
        case 2: return row_kernel<T, 2, TR>;
        case 3: return row_kernel<T, 3, TR>;
        case 4: return row_kernel<T, 4, TR>;
        case 5: return row_kernel<T, 5, TR>;
        case 6: return row_kernel<T, 6, TR>;
        case 7: return row_kernel<T, 7, TR>;
        default: return row_kernel<T, 8, TR>;
    }
}
// ---- sharded sweeps: one update = propose -> row partial (row_kernel, K = 0)
// -> exchange of the partials -> decide, all stream-ordered (the decision needs
// every rank's share of Delta_i, so a sweep cannot stay inside one launch)
__global__ void rw_propose_kernel(const double* __restrict__ x, const int64_t* __restrict__ rows,
                                  const double* __restrict__ z, int64_t q, double step, int d, double* xnew) {
    const int k = threadIdx.x;
    if (k < d) {
        const int64_t i = rows[q];
        xnew[k] = __fma_rn(step, z[q * d + k], x[i * d + k]);     // as row_kernel
    }
}

// rank-ordered sum of the partial deltas, the iid-prior change and the decision
// (the same expressions and order as row_kernel's), identical on every rank
__global__ void rw_decide_kernel(const double* __restrict__ gathered, int world, int64_t stride, double* x,
                                 const int64_t* __restrict__ rows, const double* __restrict__ u, int64_t q,
                                 const double* __restrict__ xnew, double inv_tau2, int d,
                                 unsigned long long* accepted) {
    if (threadIdx.x != 0) return;
    double dl = 0.0;
    for (int r = 0; r < world; ++r) dl += gathered[(size_t)r * stride];
    const int64_t i = rows[q];
    double pn = 0.0, po = 0.0;
    for (int k = 0; k < d; ++k) {
        pn = fma(xnew[k], xnew[k], pn);
        po = fma(x[i * d + k], x[i * d + k], po);
    }
    const double lr = dl - 0.5 * (pn - po) * inv_tau2;
    if (isfinite(lr) && log(u[q]) < lr) {
        for (int k = 0; k < d; ++k) x[i * d + k] = xnew[k];
        ++*accepted;
    }
}

}  // namespace

void rw_propose_launch(const double* x, const int64_t* rows, const double* z, int64_t q, double step, int d,
                       double* xnew, cudaStream_t s) {
    rw_propose_kernel<<<1, 32, 0, s>>>(x, rows, z, q, step, d, xnew);
}

void rw_decide_launch(const double* gathered, int world, int64_t stride, double* x, const int64_t* rows,
                      const double* u, int64_t q, const double* xnew, double inv_tau2, int d,
                      unsigned long long* accepted, cudaStream_t s) {
    rw_decide_kernel<<<1, 32, 0, s>>>(gathered, world, stride, x, rows, u, q, xnew, inv_tau2, d, accepted);
}

void rw_preload() {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, rw_propose_kernel);
    cudaFuncGetAttributes(&fa, rw_decide_kernel);
}

RowFn row_fn(int prec_is_f64, int trunc, int d) {
    if (prec_is_f64) return trunc ? row_fn_d<double, true>(d) : row_fn_d<double, false>(d);
    return trunc ? row_fn_d<float, true>(d) : row_fn_d<float, false>(d);
}

}  // namespace mdsk

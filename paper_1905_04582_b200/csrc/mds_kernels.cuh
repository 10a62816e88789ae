// mds_kernels.cuh -- helper kernels of libmds (packing, diagnostics, leapfrog
// helpers, combine, probes); the pass kernel itself is in mds_pass.cuh.
// Included by mds_api.cu only.
#pragma once
#include "mds_pass.cuh"

namespace mdsk {

// ------------------------------------------------------------ Y packing
struct PackArgs {
    const double* src;      // packed rows [i0, i1), starting with y_{i0,0}
    int64_t i0, i1;
    int64_t src_base;       // packed offset of row i0
    const int* row_local;   // [nb] local tile index of (I, 0) or -1
    void* dst;              // tiles
    int* bad;               // set to 1 on y < 0 or +-inf
};

template <typename T>
__global__ void pack_rows_kernel(PackArgs a) {
    const int64_t i = a.i0 + blockIdx.x;
    if (i >= a.i1 || i < 1) return;
    const int64_t I = i / TB, ii = i % TB;
    const int lt = a.row_local[I];
    if (lt < 0) return;                                   // tile-row not owned by this rank
    const double* row = a.src + (i * (i - 1) / 2 - a.src_base);
    T* dst = static_cast<T*>(a.dst);
    for (int64_t j = threadIdx.x; j < i; j += blockDim.x) {
        double y = row[j];
        T v;
        if (y != y) {
            if (sizeof(T) == 8) v = (T)__hiloint2double((int)CANON_NAN_HI64, 0);
            else v = (T)__int_as_float((int)CANON_NAN_F32);
        } else {
            if (y < 0.0 || y == __longlong_as_double(0x7ff0000000000000LL)) { *a.bad = 1; continue; }
            v = (T)y;
        }
        const int64_t J = j / TB, jj = j % TB;
        dst[(size_t)(lt + J) * TB * TB + jj * TB + ii] = v;
    }
}

template <typename T>
__global__ void fill_nan_kernel(T* p, size_t count) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    T nanv;
    if (sizeof(T) == 8) nanv = (T)__hiloint2double((int)CANON_NAN_HI64, 0);
    else nanv = (T)__int_as_float((int)CANON_NAN_F32);
    for (; k < count; k += stride) p[k] = nanv;
}

// L2 flush for timing loops: overwrite a buffer larger than L2 with 16-byte
// stores.  Launched with the pass kernel's block size and dynamic shared memory
// so the SMs keep the same L1/shared-memory split between timed passes.
// read pass of mds_l2_flush_clean: stream a buffer larger than L2 through it
// so the dirty lines the write pass left are written back inside the flush
__global__ void l2_read_kernel(const uint4* __restrict__ p, size_t count16, unsigned* sink) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned acc = 0;
    for (; k < count16; k += stride) {
        const uint4 w = __ldcg(p + k);
        acc ^= w.x ^ w.y ^ w.z ^ w.w;
    }
    if (acc == 0x12345678u) *sink = acc;    // keep the loads alive
}

__global__ void l2_flush_kernel(uint4* p, size_t count16, unsigned v) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    const uint4 w = make_uint4(v, v, v, v);
    for (; k < count16; k += stride) p[k] = w;
}

// count observed (non-canonical-NaN) slots of the local tiles
template <typename T>
__global__ void count_obs_kernel(const T* __restrict__ y, size_t count, unsigned long long* out) {
    size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned long long c = 0;
    for (; k < count; k += stride) c += is_missing(y[k]) ? 0 : 1;
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// observed pairs at distance exactly 0 (diagnostic, reading R10), in the
// compute precision of the pair kernel
template <typename T>
__global__ void zero_pairs_kernel(const T* __restrict__ y, const double* __restrict__ X, const int* tiles, int D,
                                  unsigned long long* out) {
    const int t = blockIdx.x;
    const int I = tiles[t] >> 16, J = tiles[t] & 0xffff;
    unsigned long long c = 0;
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) {
        const int jj = e / TB, ii = e % TB;
        const T yv = y[(size_t)t * TB * TB + e];
        if (is_missing(yv)) continue;
        T s = 0;
        for (int k = 0; k < D; ++k) {
            T dl = (T)X[((size_t)I * TB + ii) * D + k] - (T)X[((size_t)J * TB + jj) * D + k];
            s += dl * dl;
        }
        c += (s == T(0)) ? 1 : 0;
    }
    for (int m = 16; m >= 1; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ------------------------------------------------------------ leapfrog helpers
// gl = g - x / tau^2 (grad log pi) and the first drift xnext = x + eps (p + eps/2 gl)
__global__ void prime_kernel(const double* __restrict__ g, const double* __restrict__ x, const double* __restrict__ p,
                             double* __restrict__ gl, double* __restrict__ xnext, int64_t m, double inv_tau2,
                             const double* __restrict__ gprior,
                             double eps, double heps) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) {
        const double v = gprior ? g[k] + gprior[k] : g[k] - x[k] * inv_tau2;
        gl[k] = v;
        xnext[k] = drift(x[k], p[k], v, eps, heps);
    }
}

// xnext from the stored (x, p, gl) for a new step size
__global__ void redrift_kernel(const double* __restrict__ x, const double* __restrict__ p,
                               const double* __restrict__ gl, double* __restrict__ xnext, int64_t m, double eps,
                               double heps) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) xnext[k] = drift(x[k], p[k], gl[k], eps, heps);
}

// sharded leapfrog update after the rank-ordered combine (same arithmetic as phase B)
__global__ void leapfrog_update_kernel(const double* __restrict__ g, const double* __restrict__ xe,
                                       double* __restrict__ x, double* __restrict__ p, double* __restrict__ gl,
                                       double* __restrict__ xnext, int64_t m, double eps, double heps,
                                       double inv_tau2, const double* __restrict__ gprior) {
    int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < m) {
        const double xv = xe[k];
        const double ph = __fma_rn(heps, gl[k], p[k]);
        const double gn = gprior ? g[k] + gprior[k] : g[k] - xv * inv_tau2;
        const double pn = __fma_rn(heps, gn, ph);
        x[k] = xv;
        p[k] = pn;
        gl[k] = gn;
        xnext[k] = drift(xv, pn, gn, eps, heps);
    }
}

// H = -(loglik + prior(x)) + 1/2 p.p, fixed-order single-block reduction.
// out[0] = H, out[1] = loglik, out[2] = kinetic
__global__ void hamiltonian_kernel(const double* __restrict__ x, const double* __restrict__ p,
                                   const double* __restrict__ loglik, int64_t m, double inv_tau2,
                                   const double* __restrict__ logprior,
                                   double* __restrict__ out) {
    __shared__ double sp[1024], sk[1024];
    double a = 0.0, kin = 0.0;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
        a += x[k] * x[k];
        kin += p[k] * p[k];
    }
    sp[threadIdx.x] = a;
    sk[threadIdx.x] = kin;
    __syncthreads();
    for (int s = blockDim.x / 2; s >= 1; s >>= 1) {
        if (threadIdx.x < s) {
            sp[threadIdx.x] += sp[threadIdx.x + s];
            sk[threadIdx.x] += sk[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double prior = logprior ? logprior[0] : -0.5 * sp[0] * inv_tau2;
        const double K = 0.5 * sk[0];
        out[0] = -(loglik[0] + prior) + K;
        out[1] = loglik[0];
        out[2] = K;
    }
}

// Start of an HMC transition, one block of 1024 threads: save x (mpad entries, padding
// included), gl, log L (and the log prior) for a rejection, xnext = drift(x, p, gl) for
// the new momentum, and H0 -- the three save copies, redrift_kernel and
// hamiltonian_kernel in one launch; the H0 reduction has hamiltonian_kernel's order
// (same per-thread partition, same tree), so H0 is bitwise the same.
__global__ void __launch_bounds__(1024) transition_begin_kernel(
    const double* __restrict__ x, const double* __restrict__ p, const double* __restrict__ gl,
    double* __restrict__ xsave, double* __restrict__ glsave, double* __restrict__ xnext, int64_t m, int64_t mpad,
    double eps, double heps, const double* __restrict__ loglik, double* __restrict__ liksave,
    double* __restrict__ logprior, double inv_tau2, double* __restrict__ out) {
    __shared__ double sp[1024], sk[1024];
    double a = 0.0, kin = 0.0;
    for (int64_t k = threadIdx.x; k < m; k += blockDim.x) {
        const double xv = x[k], pv = p[k], gv = gl[k];
        xsave[k] = xv;
        glsave[k] = gv;
        xnext[k] = drift(xv, pv, gv, eps, heps);
        a += xv * xv;
        kin += pv * pv;
    }
    for (int64_t k = m + threadIdx.x; k < mpad; k += blockDim.x) xsave[k] = x[k];
    sp[threadIdx.x] = a;
    sk[threadIdx.x] = kin;
    __syncthreads();
    for (int s = blockDim.x / 2; s >= 1; s >>= 1) {
        if (threadIdx.x < s) {
            sp[threadIdx.x] += sp[threadIdx.x + s];
            sk[threadIdx.x] += sk[threadIdx.x + s];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        liksave[0] = loglik[0];
        if (logprior) logprior[1] = logprior[0];
        const double prior = logprior ? logprior[0] : -0.5 * sp[0] * inv_tau2;
        const double K = 0.5 * sk[0];
        out[0] = -(loglik[0] + prior) + K;
        out[1] = loglik[0];
        out[2] = K;
    }
}

// a rejected HMC transition: x, gl, log L (and the log prior) back to the saved state
__global__ void transition_restore_kernel(double* __restrict__ x, const double* __restrict__ xsave,
                                          double* __restrict__ gl, const double* __restrict__ glsave, int64_t m,
                                          int64_t mpad, double* __restrict__ loglik,
                                          const double* __restrict__ liksave, double* __restrict__ logprior) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k < mpad) x[k] = xsave[k];
    if (k < m) gl[k] = glsave[k];
    if (k == 0) {
        loglik[0] = liksave[0];
        if (logprior) logprior[0] = logprior[1];
    }
}

// Sharded leapfrog step after the exchange: the rank-ordered sum of the gathered
// partials (gathered[r][0..m) = gradient partials, gathered[r][m] = log L partial)
// fused with the leapfrog update of leapfrog_update_kernel.  Bitwise identical on
// every rank (same inputs, same order).
__global__ void combine_update_kernel(const double* __restrict__ gathered, int world, int64_t m,
                                      double* __restrict__ grad_out, double* __restrict__ lik_out,
                                      const double* __restrict__ xe, double* __restrict__ x, double* __restrict__ p,
                                      double* __restrict__ gl, double* __restrict__ xnext, double eps, double heps,
                                      double inv_tau2, const double* __restrict__ gprior) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k > m) return;
    double g = 0.0;
    for (int r = 0; r < world; ++r) g += gathered[(size_t)r * (m + 1) + k];
    if (k == m) {
        if (lik_out) *lik_out = g;
        return;
    }
    grad_out[k] = g;
    const double xv = xe[k];
    const double ph = __fma_rn(heps, gl[k], p[k]);
    const double gn = gprior ? g + gprior[k] : g - xv * inv_tau2;
    const double pn = __fma_rn(heps, gn, ph);
    x[k] = xv;
    p[k] = pn;
    gl[k] = gn;
    xnext[k] = drift(xv, pn, gn, eps, heps);
}

// The exchanges other than the fused pass (likelihood-only passes, single-location
// updates) over the peer-memory windows: ONE CTA pushes send[0..count) into slot
// [rank] of every rank's window, raises this rank's flag everywhere, waits for all
// ranks' flags and copies the world slots into recv[world][count] (rank order) for
// the rank-ordered combine kernels.  Same exchange count and flags as the fused pass.
__global__ void p2p_allgather_kernel(P2PArgs q, const double* __restrict__ send, int64_t count,
                                     double* __restrict__ recv) {
    const unsigned long long ep = p2p_epoch(q);
    for (int64_t e = threadIdx.x; e < count; e += blockDim.x) p2p_push(q, ep, e, send[e]);
    __syncthreads();
    if (threadIdx.x == 0) p2p_arrive_and_wait(q, ep, 1u);
    __syncthreads();
    const double* rv = p2p_recv(q, q.win[q.rank], ep);
    for (int r = 0; r < q.world; ++r)
        for (int64_t e = threadIdx.x; e < count; e += blockDim.x) recv[(size_t)r * count + e] = rv[(size_t)r * q.m1 + e];
    __syncthreads();
    if (threadIdx.x == 0) p2p_finish(q, ep, 1u);
}

// rank-ordered sum of gathered partials: out[e] = sum_r gathered[r][e]
__global__ void combine_kernel(const double* __restrict__ gathered, int world, int64_t len,
                               double* __restrict__ grad_out, double* __restrict__ lik_out) {
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= len) return;
    double s = 0.0;
    for (int r = 0; r < world; ++r) s += gathered[(size_t)r * len + e];
    if (e < len - 1) { if (grad_out) grad_out[e] = s; }
    else if (lik_out) *lik_out = s;
}

// ------------------------------------------------------------ FMA peak probe
template <typename T>
__global__ void fma_peak_kernel(T* out, int iters, T a, T b) {
    T r0 = threadIdx.x * T(1e-7), r1 = r0 + T(1), r2 = r0 + T(2), r3 = r0 + T(3);
    T r4 = r0 + T(4), r5 = r0 + T(5), r6 = r0 + T(6), r7 = r0 + T(7);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b);
            r4 = fma(r4, a, b); r5 = fma(r5, a, b); r6 = fma(r6, a, b); r7 = fma(r7, a, b);
        }
    }
    T s = ((r0 + r1) + (r2 + r3)) + ((r4 + r5) + (r6 + r7));
    if (s == T(12345.678)) out[0] = s;   // keep the chains alive
}

}  // namespace mdsk

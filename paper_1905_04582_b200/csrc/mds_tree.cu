// mds_tree.cu -- the Brownian-diffusion prior kernel (see mds_tree.cuh).
#include <cuda_runtime.h>
#include "mds_tree.cuh"

namespace mdsk {
namespace {

constexpr int TT = 1024;
constexpr double LOG_2PI = 1.8378770664093454836;

template <int D>
__device__ __forceinline__ double quad(const double* sinv, const double (&v)[D]) {
    double q = 0.0;
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double w = 0.0;
#pragma unroll
        for (int c = 0; c < D; ++c) w = fma(sinv[r * D + c], v[c], w);
        q = fma(v[r], w, q);
    }
    return q;
}

template <int D>
__device__ __forceinline__ double contrast(const TreeArgs& a, const double (&delta)[D], double w) {
    return -0.5 * quad<D>(a.sinv, delta) / w - 0.5 * D * (LOG_2PI + log(w)) - 0.5 * a.logdet;
}

template <int D>
__global__ void __launch_bounds__(TT, 1) tree_prior_kernel(TreeArgs a) {
    __shared__ double red[33];
    const int tid = threadIdx.x;
    // tips: up message (x, 0)
    for (int k = tid; k < a.n_items; k += TT) {
#pragma unroll
        for (int q = 0; q < D; ++q) a.up_m[k * D + q] = a.x[(int64_t)k * D + q];
        a.up_v[k] = 0.0;
        a.contrib[k] = 0.0;
    }
    __syncthreads();
    // ---- post-order: absorb the children of each internal node, level by level (by height)
    for (int L = 0; L < a.n_up; ++L) {
        for (int e = a.up_lvl_ptr[L] + tid; e < a.up_lvl_ptr[L + 1]; e += TT) {
            const int nd = a.up_lvl_nodes[e];
            const int c0 = a.ch_ptr[nd], c1 = a.ch_ptr[nd + 1];
            double A[D], W, lp = 0.0;
            {
                const int c = a.ch_idx[c0];
#pragma unroll
                for (int q = 0; q < D; ++q) A[q] = a.up_m[c * D + q];
                W = a.up_v[c] + a.t[c];
            }
            for (int cc = c0 + 1; cc < c1; ++cc) {
                const int c = a.ch_idx[cc];
                const double wi = a.up_v[c] + a.t[c];
                const double w = W + wi;
                double dl[D];
#pragma unroll
                for (int q = 0; q < D; ++q) dl[q] = a.up_m[c * D + q] - A[q];
                lp += contrast<D>(a, dl, w);
#pragma unroll
                for (int q = 0; q < D; ++q) A[q] = (wi * A[q] + W * a.up_m[c * D + q]) / w;
                W = W * wi / w;
            }
#pragma unroll
            for (int q = 0; q < D; ++q) a.up_m[nd * D + q] = A[q];
            a.up_v[nd] = W;
            a.contrib[nd] = lp;
        }
        __syncthreads();
    }
    // roots: contrast against mu0 with variance v_root + tau_root; outside message (mu0, tau_root)
    for (int e = tid; e < a.n_roots; e += TT) {
        const int r = a.roots[e];
        double dl[D];
#pragma unroll
        for (int q = 0; q < D; ++q) dl[q] = a.up_m[r * D + q] - a.mu0[q];
        a.contrib[r] += contrast<D>(a, dl, a.up_v[r] + a.t[r]);
#pragma unroll
        for (int q = 0; q < D; ++q) a.out_m[r * D + q] = a.mu0[q];
        a.out_v[r] = a.t[r];
    }
    __syncthreads();
    // ---- pre-order: each child's outside message = the parent's outside message
    // combined with the siblings' up messages, moved down the child's branch
    for (int L = 0; L < a.n_dn; ++L) {
        for (int e = a.dn_lvl_ptr[L] + tid; e < a.dn_lvl_ptr[L + 1]; e += TT) {
            const int nd = a.dn_lvl_nodes[e];
            const int c0 = a.ch_ptr[nd], c1 = a.ch_ptr[nd + 1];
            const double pv = 1.0 / a.out_v[nd];
            for (int cc = c0; cc < c1; ++cc) {
                const int c = a.ch_idx[cc];
                double P = pv, M[D];
#pragma unroll
                for (int q = 0; q < D; ++q) M[q] = a.out_m[nd * D + q] * pv;
                for (int ss = c0; ss < c1; ++ss) {
                    if (ss == cc) continue;
                    const int s = a.ch_idx[ss];
                    const double ps = 1.0 / (a.up_v[s] + a.t[s]);
                    P += ps;
#pragma unroll
                    for (int q = 0; q < D; ++q) M[q] = fma(a.up_m[s * D + q], ps, M[q]);
                }
                const double iv = 1.0 / P;
#pragma unroll
                for (int q = 0; q < D; ++q) a.out_m[c * D + q] = M[q] * iv;
                a.out_v[c] = iv + a.t[c];
            }
        }
        __syncthreads();
    }
    // tips: d log p / d x_i = -Sigma^-1 (x_i - m_i) / v_i
    for (int k = tid; k < a.n_items; k += TT) {
        double r[D];
        const double iv = 1.0 / a.out_v[k];
#pragma unroll
        for (int q = 0; q < D; ++q) r[q] = a.x[(int64_t)k * D + q] - a.out_m[k * D + q];
#pragma unroll
        for (int q = 0; q < D; ++q) {
            double g = 0.0;
#pragma unroll
            for (int c = 0; c < D; ++c) g = fma(a.sinv[q * D + c], r[c], g);
            a.grad[(int64_t)k * D + q] = -g * iv;
        }
    }
    // log p: fixed-order sum of the node contributions
    double acc = 0.0;
    for (int k = tid; k < a.n_nodes; k += TT) acc += a.contrib[k];
#pragma unroll
    for (int m = 16; m >= 1; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
    if ((tid & 31) == 0) red[tid >> 5] = acc;
    __syncthreads();
    if (tid < 32) {
        double s = red[tid];
#pragma unroll
        for (int m = 16; m >= 1; m >>= 1) s += __shfl_xor_sync(0xffffffffu, s, m);
        if (tid == 0) *a.logp = s;
    }
}

}  // namespace

void tree_prior_launch(const TreeArgs& a, int d, cudaStream_t s) {
    switch (d) {
        case 1: tree_prior_kernel<1><<<1, TT, 0, s>>>(a); break;
        case 2: tree_prior_kernel<2><<<1, TT, 0, s>>>(a); break;
        case 3: tree_prior_kernel<3><<<1, TT, 0, s>>>(a); break;
        case 4: tree_prior_kernel<4><<<1, TT, 0, s>>>(a); break;
        case 5: tree_prior_kernel<5><<<1, TT, 0, s>>>(a); break;
        case 6: tree_prior_kernel<6><<<1, TT, 0, s>>>(a); break;
        case 7: tree_prior_kernel<7><<<1, TT, 0, s>>>(a); break;
        default: tree_prior_kernel<8><<<1, TT, 0, s>>>(a); break;
    }
}

}  // namespace mdsk

// mds_cv.cu -- held-out predictive density kernels (see mds_cv.cuh).
#include <cuda_runtime.h>
#include "mds_cv.cuh"

namespace mdsk {
namespace {

template <int D, bool TRUNC>
__device__ __forceinline__ double heldout_ell(const CvArgs& a, int64_t q, const double* exptab) {
    const int2 p = a.ij[q];
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < D; ++k) {
        const double dl = a.x[(int64_t)p.x * D + k] - a.x[(int64_t)p.y * D + k];
        s = fma(dl, dl, s);
    }
    const double ss[1] = {s}, yy[1] = {a.y[q]};
    double l[1], u[1];
    pair_f64_n<TRUNC, 1, true, false>(ss, yy, a.P, exptab, l, u);
    return l[0];
}

template <int D, bool TRUNC>
__global__ void __launch_bounds__(256) cv_accumulate_kernel(CvArgs a) {
    __shared__ double exptab[EXPT64_N];
    build_exptab(exptab, a.P);
    __syncthreads();
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < a.m; q += (int64_t)gridDim.x * blockDim.x) {
        const double l = heldout_ell<D, TRUNC>(a, q, exptab);
        if (a.first) {
            a.lmax[q] = l;
            a.lsum[q] = 1.0;
        } else {
            // online log-sum-exp: keep the running max, rescale the sum when it moves
            const double m0 = a.lmax[q], s0 = a.lsum[q];
            if (l > m0) {
                a.lmax[q] = l;
                a.lsum[q] = fma(s0, exp(m0 - l), 1.0);
            } else {
                a.lsum[q] = s0 + exp(l - m0);
            }
        }
    }
}

__global__ void __launch_bounds__(1024) cv_finalize_kernel(const double* __restrict__ lmax,
                                                           const double* __restrict__ lsum, int64_t m,
                                                           int64_t draws, double* out) {
    __shared__ double red[32];
    double acc = 0.0;
    for (int64_t q = threadIdx.x; q < m; q += blockDim.x) acc += lmax[q] + log(lsum[q]);
#pragma unroll
    for (int k = 16; k >= 1; k >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, k);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) red[warp] = acc;
    __syncthreads();
    if (warp == 0) {
        double t = lane < (int)(blockDim.x >> 5) ? red[lane] : 0.0;
#pragma unroll
        for (int k = 16; k >= 1; k >>= 1) t += __shfl_xor_sync(0xffffffffu, t, k);
        if (lane == 0) out[0] = t - (double)m * log((double)draws);
    }
}

template <bool TR>
void launch_d(const CvArgs& a, int grid, cudaStream_t s) {
    switch (a.d) {
        case 1: cv_accumulate_kernel<1, TR><<<grid, 256, 0, s>>>(a); break;
        case 2: cv_accumulate_kernel<2, TR><<<grid, 256, 0, s>>>(a); break;
        case 3: cv_accumulate_kernel<3, TR><<<grid, 256, 0, s>>>(a); break;
        case 4: cv_accumulate_kernel<4, TR><<<grid, 256, 0, s>>>(a); break;
        case 5: cv_accumulate_kernel<5, TR><<<grid, 256, 0, s>>>(a); break;
        case 6: cv_accumulate_kernel<6, TR><<<grid, 256, 0, s>>>(a); break;
        case 7: cv_accumulate_kernel<7, TR><<<grid, 256, 0, s>>>(a); break;
        default: cv_accumulate_kernel<8, TR><<<grid, 256, 0, s>>>(a); break;
    }
}
}  // namespace

void cv_accumulate_launch(const CvArgs& a, int grid, cudaStream_t s) {
    if (a.trunc) launch_d<true>(a, grid, s);
    else launch_d<false>(a, grid, s);
}

void cv_finalize_launch(const double* lmax, const double* lsum, int64_t m, int64_t draws, double* out,
                        cudaStream_t s) {
    cv_finalize_kernel<<<1, 1024, 0, s>>>(lmax, lsum, m, draws, out);
}

}  // namespace mdsk

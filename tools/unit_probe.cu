// unit_probe.cu -- builds the pass kernel's unit loop up from the bare pair math
// (registers only) to the full body, to see which structural part costs FP64 rate.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1905_04582_b200/csrc/mds_math.cuh"
using namespace mdsk;

template <typename T> __device__ __forceinline__ T shx(T v, int m) { return __shfl_xor_sync(0xffffffffu, v, m); }

// LEVEL 0: pair math on register data; 1: + y, x from shared memory and distances;
// 2: + row/column/logL accumulation; 3: + permuted reduce-scatter of the 4 columns
template <int LEVEL, int WPC>
__global__ void __launch_bounds__(WPC * 32, 1) probe(double* out, int units, SigmaParams P) {
    __shared__ double ys[WPC][256];
    __shared__ double xc[64 * 2];
    __shared__ double tab[64];
    if (threadIdx.x < 64) tab[threadIdx.x] = EXPT64_TAB[threadIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, m = (lane >> 3) & 3;
    for (int i = threadIdx.x; i < WPC * 256; i += blockDim.x) ys[i / 256][i % 256] = 0.5 + 0.001 * (i % 97);
    for (int i = threadIdx.x; i < 128; i += blockDim.x) xc[i] = 0.01 * i;
    __syncthreads();
    double xi0[2] = {0.3 + lane * 1e-3, 0.7}, xi1[2] = {-0.2, 0.1 + lane * 1e-3};
    double g0[2] = {0, 0}, g1[2] = {0, 0}, lik = 0, colsum = 0;
    double sreg[4] = {1.0 + lane * 1e-3, 1.3, 0.9, 2.2}, yreg[4] = {1.1, 1.0, 0.8, 1.7};
    for (int u = 0; u < units; ++u) {
        const int jj0 = (u & 15) * 4;
        double cv[4][2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            double ss[4], yy[4], dd[4][2];
            if (LEVEL == 0) {
#pragma unroll
                for (int i = 0; i < 4; ++i) { ss[i] = sreg[i] + u * 1e-9; yy[i] = yreg[i]; dd[i][0] = dd[i][1] = 0.1; }
            } else {
#pragma unroll
                for (int qq = 0; qq < 2; ++qq) {
                    const int q = (2 * h + qq) ^ m;
                    yy[2 * qq] = ys[warp][q * 64 + lane];
                    yy[2 * qq + 1] = ys[warp][q * 64 + lane + 32];
                    double sa = 0, sb = 0;
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        const double xj = xc[(jj0 + q) * 2 + k];
                        dd[2 * qq][k] = xi0[k] - xj;
                        dd[2 * qq + 1][k] = xi1[k] - xj;
                        sa = fma(dd[2 * qq][k], dd[2 * qq][k], sa);
                        sb = fma(dd[2 * qq + 1][k], dd[2 * qq + 1][k], sb);
                    }
                    ss[2 * qq] = sa;
                    ss[2 * qq + 1] = sb;
                }
            }
            double ll[4], uu[4];
            pair_f64_n<true, 4>(ss, yy, P, tab, ll, uu);
            if (LEVEL >= 2) {
                double lsum = 0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const bool mi = is_missing(yy[i]);
                    if (!mi) lsum += ll[i];
                    uu[i] = mi ? 0.0 : uu[i];
                }
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const double va0 = uu[0] * dd[0][k], vb0 = uu[1] * dd[1][k];
                    const double va1 = uu[2] * dd[2][k], vb1 = uu[3] * dd[3][k];
                    g0[k] -= va0 + va1;
                    g1[k] -= vb0 + vb1;
                    cv[2 * h][k] = va0 + vb0;
                    cv[2 * h + 1][k] = va1 + vb1;
                }
                lik += lsum;
            } else {
#pragma unroll
                for (int i = 0; i < 4; ++i) lik += ll[i] + uu[i];
            }
        }
        if (LEVEL >= 3) {
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                double k0 = cv[0][k] + shx(cv[2][k], 16), k1 = cv[1][k] + shx(cv[3][k], 16);
                double kk = k0 + shx(k1, 8);
                kk += shx(kk, 4); kk += shx(kk, 2); kk += shx(kk, 1);
                colsum += kk;
            }
        } else if (LEVEL == 2) {
#pragma unroll
            for (int k = 0; k < 2; ++k) colsum += cv[0][k] + cv[1][k] + cv[2][k] + cv[3][k];
        }
    }
    const double s = lik + colsum + g0[0] + g0[1] + g1[0] + g1[1];
    if (s == 1234.5) out[0] = s;
}

template <int LEVEL, int WPC>
void run(int sms, double* d, SigmaParams P) {
    const int units = 400;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<LEVEL, WPC><<<sms, WPC * 32>>>(d, units, P);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe<LEVEL, WPC>);
    const double pairs = (double)sms * WPC * 32 * units * 8;
    printf("level %d warps/SM %2d regs %3d : %.1f G pairs/s\n", LEVEL, WPC, fa.numRegs, pairs / (best * 1e-3) / 1e9);
}


// LEVEL 3 with all 8 pairs of a 4-column group (rows l, l+32) in lock-step (ILP 8)
template <int WPC>
__global__ void __launch_bounds__(WPC * 32, 1) probe8(double* out, int units, SigmaParams P) {
    __shared__ double ys[WPC][256];
    __shared__ double xc[64 * 2];
    __shared__ double tab[64];
    if (threadIdx.x < 64) tab[threadIdx.x] = EXPT64_TAB[threadIdx.x];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, m = (lane >> 3) & 3;
    for (int i = threadIdx.x; i < WPC * 256; i += blockDim.x) ys[i / 256][i % 256] = 0.5 + 0.001 * (i % 97);
    for (int i = threadIdx.x; i < 128; i += blockDim.x) xc[i] = 0.01 * i;
    __syncthreads();
    double xi0[2] = {0.3 + lane * 1e-3, 0.7}, xi1[2] = {-0.2, 0.1 + lane * 1e-3};
    double g0[2] = {0, 0}, g1[2] = {0, 0}, lik = 0, colsum = 0;
    for (int u = 0; u < units; ++u) {
        const int jj0 = (u & 15) * 4;
        double cv[4][2];
        double ss[8], yy[8], dd[8][2];
#pragma unroll
        for (int qq = 0; qq < 4; ++qq) {
            const int q = qq ^ m;
            yy[2 * qq] = ys[warp][q * 64 + lane];
            yy[2 * qq + 1] = ys[warp][q * 64 + lane + 32];
            double sa = 0, sb = 0;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const double xj = xc[(jj0 + q) * 2 + k];
                dd[2 * qq][k] = xi0[k] - xj;
                dd[2 * qq + 1][k] = xi1[k] - xj;
                sa = fma(dd[2 * qq][k], dd[2 * qq][k], sa);
                sb = fma(dd[2 * qq + 1][k], dd[2 * qq + 1][k], sb);
            }
            ss[2 * qq] = sa;
            ss[2 * qq + 1] = sb;
        }
        double ll[8], uu[8];
        pair_f64_n<true, 8>(ss, yy, P, tab, ll, uu);
        double lsum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const bool mi = is_missing(yy[i]);
            if (!mi) lsum += ll[i];
            uu[i] = mi ? 0.0 : uu[i];
        }
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const double va = uu[2 * qq] * dd[2 * qq][k], vb = uu[2 * qq + 1] * dd[2 * qq + 1][k];
                g0[k] -= va;
                g1[k] -= vb;
                cv[qq][k] = va + vb;
            }
        lik += lsum;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            double k0 = cv[0][k] + shx(cv[2][k], 16), k1 = cv[1][k] + shx(cv[3][k], 16);
            double kk = k0 + shx(k1, 8);
            kk += shx(kk, 4); kk += shx(kk, 2); kk += shx(kk, 1);
            colsum += kk;
        }
    }
    const double s = lik + colsum + g0[0] + g0[1] + g1[0] + g1[1];
    if (s == 1234.5) out[0] = s;
}

template <int WPC>
void run8(int sms, double* d, SigmaParams P) {
    const int units = 400;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe8<WPC><<<sms, WPC * 32>>>(d, units, P);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe8<WPC>);
    const double pairs = (double)sms * WPC * 32 * units * 8;
    printf("ILP8 level 3 warps/SM %2d regs %3d local %d : %.1f G pairs/s\n", WPC, fa.numRegs, (int)fa.localSizeBytes, pairs / (best * 1e-3) / 1e9);
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 64);
    SigmaParams P{}; double sg = 0.6;
    P.inv_sigma = 1 / sg; P.inv_sigma2 = 1 / (sg * sg); P.half_inv_sigma2 = 0.5 / (sg * sg);
    P.k0 = -0.5 * log(2 * 3.141592653589793 * sg * sg); P.cg = 1 / (sg * sqrt(2 * 3.141592653589793));
    run<0, 12>(sms, d, P); run<1, 12>(sms, d, P); run<2, 12>(sms, d, P); run<3, 12>(sms, d, P);
    run<0, 8>(sms, d, P); run<3, 8>(sms, d, P); run<3, 16>(sms, d, P);
    run8<8>(sms, d, P); run8<12>(sms, d, P); run8<16>(sms, d, P);
    return 0;
}

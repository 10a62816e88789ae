// pair_probe.cu -- throughput of the fp64 pair math alone (registers only), vs
// warps per SM and pairs in lock-step: the ceiling for the pass kernel's phase A.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1905_04582_b200/csrc/mds_math.cuh"
using namespace mdsk;

template <int NP, int WPC>
__global__ void __launch_bounds__(WPC * 32, 1) probe(double* out, int iters, SigmaParams P) {
    __shared__ double tab[64];
    if (threadIdx.x < 64) tab[threadIdx.x] = EXPT64_TAB[threadIdx.x];
    __syncthreads();
    double s[NP], y[NP], acc = 0.0;
#pragma unroll
    for (int i = 0; i < NP; ++i) { s[i] = 1.0 + 0.37 * i + threadIdx.x * 1e-4; y[i] = 1.1 + 0.1 * i; }
    for (int it = 0; it < iters; ++it) {
        double l[NP], u[NP];
        pair_f64_n<true, NP>(s, y, P, tab, l, u);
#pragma unroll
        for (int i = 0; i < NP; ++i) { acc += l[i]; s[i] += u[i] * 1e-12; }
    }
    if (acc == 1234.5) out[0] = acc;
}

template <int NP, int WPC>
void run(int sms, double* d, SigmaParams P) {
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<NP, WPC><<<sms, WPC * 32>>>(d, iters, P);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, probe<NP, WPC>);
    const double pairs = (double)sms * WPC * 32 * iters * NP;
    printf("NP %d warps/SM %2d regs %3d : %.1f G pairs/s\n", NP, WPC, fa.numRegs, pairs / (best * 1e-3) / 1e9);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 64);
    SigmaParams P{};
    double sg = 0.6;
    P.inv_sigma = 1 / sg; P.inv_sigma2 = 1 / (sg * sg); P.half_inv_sigma2 = 0.5 / (sg * sg);
    P.k0 = -0.5 * log(2 * 3.141592653589793 * sg * sg); P.cg = 1 / (sg * sqrt(2 * 3.141592653589793));
    run<1, 12>(sms, d, P); run<1, 20>(sms, d, P); run<1, 32>(sms, d, P);
    run<2, 12>(sms, d, P); run<2, 20>(sms, d, P);
    run<4, 8>(sms, d, P); run<4, 12>(sms, d, P); run<4, 16>(sms, d, P);
    run<8, 8>(sms, d, P);
    return 0;
}

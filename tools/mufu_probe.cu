// mufu_probe.cu -- throughput of the FP64 MUFU seeds (rcp/rsqrt.approx.f64) alone
// and mixed with DFMA, on sm_100a (design probe, not part of libmds).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp64(double x) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }
__device__ __forceinline__ double rsq64(double x) { double r; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }

template <int NM, int NF>
__global__ void probe(double* out, int iters, double a) {
    double r[4], f[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) { r[i] = 1.0 + threadIdx.x * 1e-7 + i; f[i] = r[i]; }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int m = 0; m < NM; ++m) r[m & 3] = rcp64(r[m & 3] + a);
#pragma unroll
            for (int q = 0; q < NF; ++q) f[q & 3] = fma(f[q & 3], a, 1e-9);
        }
    }
    double s = r[0] + r[1] + r[2] + r[3] + f[0] + f[1] + f[2] + f[3];
    if (s == 1234.5) out[0] = s;
}

template <int NM, int NF>
void run(int sms, double* d) {
    const int threads = 512, iters = 1024;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<NM, NF><<<sms * 2, threads>>>(d, iters, 1e-3);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double warps_instr_per_sm = (double)2 * threads / 32 * iters * 8;   // per kind, per SM
    const double cyc = best * 1e-3 * 1.965e9;
    printf("MUFU.RCP64H x%d + DADD x%d + DFMA x%d per step: %.2f cycles/step/SM -> MUFU64 %.2f lane/clk/SM\n", NM, NM, NF,
           cyc / warps_instr_per_sm, NM ? 32.0 * NM * warps_instr_per_sm / cyc : 0.0);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 64);
    run<4, 0>(sms, d);
    run<0, 4>(sms, d);
    run<1, 4>(sms, d);
    run<1, 8>(sms, d);
    run<2, 8>(sms, d);
    run<4, 8>(sms, d);
    return 0;
}

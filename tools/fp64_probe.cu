// fp64_probe.cu -- FP64 pipe microbenchmarks on sm_100a (design probe, not part of libmds).
// Measures warp-instruction throughput of DFMA chains vs warps/SM and ILP, and
// with interleaved non-FP64 instructions, to bound what the pair kernel can reach.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int NONFP>
__global__ void probe(double* out, int iters, double a, double b, int* sink) {
    double r[ILP];
#pragma unroll
    for (int i = 0; i < ILP; ++i) r[i] = threadIdx.x * 1e-7 + i;
    int acc = threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < ILP; ++i) r[i] = fma(r[i], a, b);
#pragma unroll
            for (int q = 0; q < NONFP; ++q) acc = acc * 1664525 + 1013904223 + q;
        }
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < ILP; ++i) s += r[i];
    if (s == 1234.5) out[0] = s;
    if (acc == 12345) sink[0] = acc;
}

template <int ILP, int NONFP>
void run(int warps_per_sm, int sms, double* d, int* sink) {
    const int threads = 32 * warps_per_sm;
    const int iters = 2048;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<ILP, NONFP><<<sms, threads>>>(d, iters, 0.999999, 1e-9, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double fma_lanes = (double)sms * threads * iters * 16.0 * ILP;
    printf("warps/SM %2d ILP %d nonfp/fma %.2f : %.2f T dfma-lane/s\n", warps_per_sm, ILP,
           (double)NONFP / ILP, fma_lanes / (best * 1e-3) / 1e12);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    int* sink;
    cudaMalloc(&d, 64);
    cudaMalloc(&sink, 64);
    for (int w : {4, 8, 12, 16, 20, 24, 32}) {
        run<1, 0>(w, sms, d, sink);
        run<2, 0>(w, sms, d, sink);
        run<4, 0>(w, sms, d, sink);
    }
    for (int w : {16, 20}) {
        run<2, 1>(w, sms, d, sink);
        run<2, 2>(w, sms, d, sink);
        run<4, 2>(w, sms, d, sink);
        run<4, 4>(w, sms, d, sink);
    }
    return 0;
}

// fp64mix_probe.cu -- throughput of DFMA vs DMUL vs DADD (ILP 4, 16 warps/SM),
// and of MUFU.RSQ64H / RCP64H mixed into a DFMA stream (design probe).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rcp64(double x) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); return r; }

__device__ __forceinline__ double rcp_via_f32(double x) {
    float f = __double2float_rn(x), r;
    asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f));
    return (double)r;
}
__device__ __forceinline__ double rcp_via_bits(double x) {
    // seed from the high word: 1/x ~ 2^-e via exponent flip (integer ops only, ~3% error)
    return __hiloint2double(0x7FDE6238 - __double2hiint(x), 0);
}
template <int OP>   // 0 dfma, 1 dmul, 2 dadd, 3 dfma + 1 mufu per 8, 4 dfma+1 mufu per 16, 5 f32 seed /8, 6 int seed /8
__global__ void probe(double* out, int iters, double a, double b) {
    double r0 = threadIdx.x * 1e-9 + 1, r1 = r0 + 1, r2 = r0 + 2, r3 = r0 + 3;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) { r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b); }
            if (OP == 1) { r0 = r0 * a; r1 = r1 * a; r2 = r2 * a; r3 = r3 * a; }
            if (OP == 2) { r0 = r0 + a; r1 = r1 + a; r2 = r2 + a; r3 = r3 + a; }
            if (OP == 3) { r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b); if (u % 2 == 0) r0 = rcp64(r0); }
            if (OP == 5) { r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b); if (u % 2 == 0) r0 = rcp_via_f32(r0); }
            if (OP == 6) { r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b); if (u % 2 == 0) r0 = rcp_via_bits(r0); }
            if (OP == 4) { r0 = fma(r0, a, b); r1 = fma(r1, a, b); r2 = fma(r2, a, b); r3 = fma(r3, a, b); if (u % 4 == 0) r0 = rcp64(r0); }
        }
    }
    double s = r0 + r1 + r2 + r3;
    if (s == 1234.5) out[0] = s;
}

template <int OP>
void run(const char* name, int sms, double* d) {
    const int threads = 512, iters = 2048;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        probe<OP><<<sms, threads>>>(d, iters, 0.9999999, 1e-9);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double warp_fp64 = (double)sms * threads / 32 * iters * 16 * 4;   // fp64 warp-instructions
    const double cyc = best * 1e-3 * 1.965e9;
    printf("%-28s: %.2f SMSP-cycles per fp64 warp-instruction\n", name, cyc * sms * 4 / warp_fp64);
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d; cudaMalloc(&d, 64);
    run<0>("DFMA", sms, d);
    run<1>("DMUL", sms, d);
    run<2>("DADD", sms, d);
    run<3>("DFMA + MUFU.RCP64H / 8", sms, d);
    run<4>("DFMA + MUFU.RCP64H / 16", sms, d);
    run<5>("DFMA + f32 rcp seed / 8", sms, d);
    run<6>("DFMA + int rcp seed / 8", sms, d);
    return 0;
}

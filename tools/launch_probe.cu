// launch_probe.cu -- back-to-back launch cost of a 148 x 384 grid: plain vs
// cooperative (grid.sync inside or not), and inside a CUDA graph.
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_plain(int* x) { if (threadIdx.x == 0 && x[blockIdx.x] == 12345) x[0] = 1; }
__global__ void k_sync(int* x) {
    if (threadIdx.x == 0 && x[blockIdx.x] == 12345) x[0] = 1;
    cg::this_grid().sync();
    if (threadIdx.x == 0 && x[blockIdx.x] == 12345) x[1] = 1;
}

template <typename F>
float run(F launch, int reps, cudaStream_t s) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    return ms * 1e3f / reps;
}

int main() {
    int* x; cudaMalloc(&x, 4096 * sizeof(int)); cudaMemset(x, 0, 4096 * sizeof(int));
    cudaStream_t s; cudaStreamCreate(&s);
    const int reps = 2000;
    auto coop = [&](void (*fn)(int*)) {
        cudaLaunchConfig_t cfg{}; cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1;
        cfg.gridDim = dim3(148); cfg.blockDim = dim3(384); cfg.stream = s; cfg.attrs = at; cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, fn, x);
    };
    printf("plain launch          : %.2f us\n", run([&] { k_plain<<<148, 384, 0, s>>>(x); }, reps, s));
    printf("cooperative, no sync  : %.2f us\n", run([&] { coop(k_plain); }, reps, s));
    printf("cooperative, grid.sync: %.2f us\n", run([&] { coop(k_sync); }, reps, s));
    // graph of 20 cooperative launches
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < 20; ++i) coop(k_sync);
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    printf("graph of 20 coop+sync : %.2f us per kernel\n", run([&] { cudaGraphLaunch(ge, s); }, 100, s) / 20);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}

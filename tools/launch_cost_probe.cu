// Event-timed cost of one launch of an (almost) empty persistent-shaped kernel:
// 148 CTAs x 384 threads, 226 KB dynamic smem (the pass kernel's shape), with a
// 16-byte vs a 1.4 KB parameter block, cooperative vs plain, with/without a
// grid-wide barrier.  Median over 200 launches, each between its own events
// (what bench.py's per-step events see of launch + ramp + drain).
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/launch_cost_probe_bin tools/launch_cost_probe.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
struct Small { int* p; int v; };
struct Large { int* p; int v; char pad[1400]; };
template <typename A, bool SYNC>
__global__ void __launch_bounds__(384, 1) k(A a) {
    extern __shared__ char sm[];
    if (threadIdx.x == 0 && a.v) sm[0] = (char)a.v;
    if (SYNC) cooperative_groups::this_grid().sync();
    if (threadIdx.x == 0 && blockIdx.x == 0 && a.v == 12345) *a.p = sm[0];
}
template <typename A, bool SYNC>
float run(bool coop, const char* name, size_t smem = 226 * 1024, int grid = 148, int threads = 384) {
    cudaFuncSetAttribute(k<A, SYNC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    A a{};
    a.p = nullptr;
    a.v = smem > 0;
    std::vector<cudaEvent_t> e0(200), e1(200);
    for (int i = 0; i < 200; ++i) { cudaEventCreate(&e0[i]); cudaEventCreate(&e1[i]); }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(threads); cfg.dynamicSmemBytes = smem; cfg.stream = s;
    cfg.attrs = at; cfg.numAttrs = coop ? 1 : 0;
    for (int i = 0; i < 20; ++i) cudaLaunchKernelEx(&cfg, k<A, SYNC>, a);
    cudaStreamSynchronize(s);
    for (int i = 0; i < 200; ++i) {
        cudaEventRecord(e0[i], s);
        cudaLaunchKernelEx(&cfg, k<A, SYNC>, a);
        cudaEventRecord(e1[i], s);
    }
    cudaStreamSynchronize(s);
    std::vector<float> t(200);
    for (int i = 0; i < 200; ++i) cudaEventElapsedTime(&t[i], e0[i], e1[i]);
    std::sort(t.begin(), t.end());
    std::printf("%-40s median %.2f us  (p10 %.2f, p90 %.2f)  %s\n", name, t[100] * 1e3, t[20] * 1e3, t[180] * 1e3,
                cudaGetErrorString(cudaGetLastError()));
    return t[100];
}
int main() {
    run<Small, false>(true, "coop, 16 B params, no sync");
    run<Large, false>(true, "coop, 1.4 KB params, no sync");
    run<Small, true>(true, "coop, 16 B params, grid.sync");
    run<Large, true>(true, "coop, 1.4 KB params, grid.sync");
    run<Small, false>(false, "plain, 16 B params, no sync");
    run<Large, false>(false, "plain, 1.4 KB params, no sync");
    run<Small, false>(false, "plain 148x384, smem 0", 0);
    run<Small, false>(false, "plain 148x384, smem 100 KB", 100 * 1024);
    run<Small, false>(false, "plain 148x128, smem 226 KB", 226 * 1024, 148, 128);
    run<Small, false>(false, "plain 1x384, smem 226 KB", 226 * 1024, 1, 384);
    run<Small, false>(false, "plain 1x32, smem 0", 0, 1, 32);
    return 0;
}

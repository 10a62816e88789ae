// Can two cooperative kernels on two streams of one process be co-resident?
// Kernel A (cooperative, G CTAs, ~200 KB smem each) waits for a flag that kernel B
// (cooperative, G CTAs, other stream) sets; both bail out after ~1 s of
// globaltimer so a serialised launch cannot hang the GPU.  Prints which happened.
// nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/coop tools/coop_concurrency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void waiter(volatile int* flag, int* out, int want) {
    extern __shared__ char sm[];
    sm[threadIdx.x] = 0;
    cooperative_groups::this_grid().sync();
    if (threadIdx.x == 0) {
        const unsigned long long t0 = gt();
        int ok = 0;
        while (gt() - t0 < 1000000000ull) {
            if (*flag >= want) { ok = 1; break; }
        }
        atomicAdd(out, ok);
    }
}
__global__ void setter(volatile int* flag) {
    extern __shared__ char sm[];
    sm[threadIdx.x] = 0;
    cooperative_groups::this_grid().sync();
    if (threadIdx.x == 0) atomicAdd((int*)flag, 1);
}
int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(waiter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(setter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int *flag, *out;
    cudaMalloc(&flag, 4);
    cudaMalloc(&out, 4);
    for (int G : {sms / 2, sms / 4}) {
        cudaMemset(flag, 0, 4);
        cudaMemset(out, 0, 4);
        cudaDeviceSynchronize();
        cudaStream_t a, b;
        cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
        void* wa[] = {&flag, &out, &G};
        int want = G;
        void* wa2[] = {&flag, &out, &want};
        void* sa[] = {&flag};
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0, a);
        cudaError_t r1 = cudaLaunchCooperativeKernel((void*)waiter, G, 256, wa2, smem, a);
        cudaError_t r2 = cudaLaunchCooperativeKernel((void*)setter, G, 256, sa, smem, b);
        cudaEventRecord(e1, a);
        cudaError_t r3 = cudaDeviceSynchronize();
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        int h = 0;
        cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
        printf("G=%d (sms %d): launch %s/%s sync %s; waiter CTAs that saw the flag: %d of %d; waiter time %.3f ms\n", G,
               sms, cudaGetErrorString(r1), cudaGetErrorString(r2), cudaGetErrorString(r3), h, G, ms);
        (void)wa;
    }
    return 0;
}

// How many kernels with grid-wide waits can run concurrently from different
// streams of one process?  k kernels (G CTAs, ~200 KB smem each), each on its own
// stream: every CTA increments a shared counter and waits until all k*G CTAs have
// arrived (bail out after 1 s of globaltimer, so a serialised launch cannot hang).
// Cooperative and plain launches.  Prints how many CTAs saw everyone.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/coop_probe_bin tools/coop_concurrency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
template <bool GS>
__global__ void meet(unsigned* cnt, unsigned want, unsigned* ok) {
    extern __shared__ char sm[];
    sm[threadIdx.x] = 0;
    if (GS) cooperative_groups::this_grid().sync();
    if (threadIdx.x == 0) {
        atomicAdd(cnt, 1u);
        const unsigned long long t0 = gt();
        while (gt() - t0 < 1000000000ull)
            if (*(volatile unsigned*)cnt >= want) { atomicAdd(ok, 1u); break; }
    }
}
int main() {
    const size_t smem = 200 * 1024;
    cudaFuncSetAttribute(meet<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(meet<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    unsigned *cnt, *ok;
    cudaMalloc(&cnt, 4);
    cudaMalloc(&ok, 4);
    cudaStream_t st[16];
    for (int i = 0; i < 16; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
    for (int coop = 2; coop >= 0; --coop)
        for (int k : {2, 3, 4, 8}) {
            const int G = 120 / k;
            cudaMemset(cnt, 0, 4);
            cudaMemset(ok, 0, 4);
            cudaDeviceSynchronize();
            unsigned want = k * G;
            void* args[] = {&cnt, &want, &ok};
            cudaError_t e = cudaSuccess;
            for (int i = 0; i < k; ++i) {
                cudaError_t r = coop == 2 ? cudaLaunchCooperativeKernel((void*)meet<true>, G, 128, args, smem, st[i])
                                : coop == 1 ? cudaLaunchCooperativeKernel((void*)meet<false>, G, 128, args, smem, st[i])
                                            : cudaLaunchKernel((void*)meet<false>, G, 128, args, smem, st[i]);
                if (r) e = r;
            }
            cudaDeviceSynchronize();
            unsigned h = 0;
            cudaMemcpy(&h, ok, 4, cudaMemcpyDeviceToHost);
            std::printf("%s k=%d G=%d: launch %s; CTAs that met everyone: %u of %u\n", coop == 2 ? "coop+grid.sync" : coop ? "cooperative   " : "plain         ",
                        k, G, cudaGetErrorString(e), h, want);
        }
    return 0;
}

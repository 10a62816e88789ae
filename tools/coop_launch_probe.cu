// Does launching a cooperative kernel block the host while other cooperative kernels
// (other streams / other host threads / the same stream) are still running?  Each
// kernel spins until all k grids have arrived or 1 s has passed; launch calls are
// timed on the host.  Variants: one thread vs k threads; 200 KB vs 226 KB smem;
// cudaLaunchCooperativeKernel vs cudaLaunchKernelEx(cooperative attribute); a 2 KB
// parameter struct.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/coop_launch_probe_bin tools/coop_launch_probe.cu -lpthread
#include <chrono>
#include <cstdio>
#include <thread>
#include <vector>
#include <cuda_runtime.h>
struct Big { unsigned* cnt; unsigned want; unsigned* ok; char pad[2048]; };
__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__global__ void meet(Big b) {
    extern __shared__ char sm[];
    sm[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        atomicAdd(b.cnt, 1u);
        const unsigned long long t0 = gt();
        while (gt() - t0 < 1000000000ull)
            if (*(volatile unsigned*)b.cnt >= b.want) { atomicAdd(b.ok, 1u); break; }
    }
}
int main() {
    unsigned *cnt, *ok;
    cudaMalloc(&cnt, 4);
    cudaMalloc(&ok, 4);
    cudaStream_t st[8];
    for (int i = 0; i < 8; ++i) cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking);
    cudaFuncSetAttribute(meet, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024);
    for (int threads : {0, 1})
        for (int ex : {0, 1})
            for (int big : {0, 1}) {
                const int k = 3, G = 20, nth = big ? 384 : 128;
                const size_t smem = big ? 226 * 1024 : 200 * 1024;
                cudaMemset(cnt, 0, 4);
                cudaMemset(ok, 0, 4);
                cudaDeviceSynchronize();
                Big b{};
                b.cnt = cnt; b.ok = ok; b.want = k * G;
                std::vector<double> ms(k);
                auto launch = [&](int i) {
                    const auto t0 = std::chrono::steady_clock::now();
                    if (ex) {
                        cudaLaunchConfig_t cfg{};
                        cudaLaunchAttribute at[1];
                        at[0].id = cudaLaunchAttributeCooperative;
                        at[0].val.cooperative = 1;
                        cfg.gridDim = dim3(G); cfg.blockDim = dim3(nth); cfg.dynamicSmemBytes = smem;
                        cfg.stream = st[i]; cfg.attrs = at; cfg.numAttrs = 1;
                        cudaLaunchKernelEx(&cfg, meet, b);
                    } else {
                        void* args[] = {&b};
                        cudaLaunchCooperativeKernel((void*)meet, G, nth, args, smem, st[i]);
                    }
                    ms[i] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                };
                if (threads) {
                    std::vector<std::thread> th;
                    for (int i = 0; i < k; ++i) th.emplace_back(launch, i);
                    for (auto& t : th) t.join();
                } else {
                    for (int i = 0; i < k; ++i) launch(i);
                }
                cudaDeviceSynchronize();
                unsigned h = 0;
                cudaMemcpy(&h, ok, 4, cudaMemcpyDeviceToHost);
                std::printf("%s %s %s: met %u of %u; launch ms %.2f %.2f %.2f (%s)\n", threads ? "3 threads" : "1 thread ",
                            ex ? "LaunchKernelEx  " : "LaunchCooperative", big ? "384 thr 226KB" : "128 thr 200KB", h,
                            k * G, ms[0], ms[1], ms[2], cudaGetErrorString(cudaGetLastError()));
            }
    // same stream, back to back (the second launch while the first spins 1 s)
    {
        cudaMemset(cnt, 0, 4);
        cudaDeviceSynchronize();
        Big b{};
        b.cnt = cnt; b.ok = ok; b.want = 1000000;
        void* args[] = {&b};
        cudaLaunchCooperativeKernel((void*)meet, 20, 384, args, 226 * 1024, st[0]);
        const auto t0 = std::chrono::steady_clock::now();
        cudaLaunchCooperativeKernel((void*)meet, 20, 384, args, 226 * 1024, st[0]);
        const double m = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        cudaDeviceSynchronize();
        std::printf("same stream, second cooperative launch while the first runs: %.2f ms\n", m);
    }
    return 0;
}

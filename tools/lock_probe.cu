// Does a host thread blocked in a pageable device->host copy (waiting for a
// spinning kernel on ITS stream) block other host threads' CUDA calls on other
// streams?  Thread A: spin kernel on stream a (released after ~2 s by its own
// timeout) + pageable D2H copy on a.  Thread B, 200 ms later: each call under
// test on stream b, timed.  ~1.8 s = serialised behind A's copy.
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/lock_probe_bin tools/lock_probe.cu -lpthread
#include <chrono>
#include <cstdio>
#include <functional>
#include <thread>
#include <cuda_runtime.h>
__global__ void spin() {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); } while (t - t0 < 2000000000ull);
}
__global__ void nop() {}
__global__ void nop2() {}
__global__ void nop3() {}
__global__ void __cluster_dims__(8, 1, 1) clus2(int* out) { if (threadIdx.x == 0 && blockIdx.x == 0) *out = 1; }
__global__ void clus3(int* out) { if (threadIdx.x == 0 && blockIdx.x == 0) *out = 1; }
__global__ void __cluster_dims__(8, 1, 1) clus(int* out) {
    __shared__ int sm[1024];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = sm[5];
}
int main() {
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    double *da, *db, *hp;
    cudaMalloc(&da, 1 << 20);
    cudaMalloc(&db, 1 << 20);
    cudaMallocHost(&hp, 1 << 20);
    static double pa[1 << 17], pb[1 << 17];
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, nop2);
    cudaFuncGetAttributes(&fa, clus2);
    cudaFuncGetAttributes(&fa, clus3);
    cudaFuncSetAttribute(nop3, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024);
    cudaDeviceSynchronize();
    struct T { const char* name; std::function<void()> f; };
    T tests[] = {
        {"kernel launch on b", [&] { nop<<<1, 1, 0, b>>>(); }},
        {"pageable H2D 8 B on b", [&] { cudaMemcpyAsync(db, pb, 8, cudaMemcpyHostToDevice, b); }},
        {"pageable H2D 64 KB on b", [&] { cudaMemcpyAsync(db, pb, 65536, cudaMemcpyHostToDevice, b); }},
        {"pinned H2D 64 KB on b", [&] { cudaMemcpyAsync(db, hp, 65536, cudaMemcpyHostToDevice, b); }},
        {"pageable D2H 8 B on b", [&] { cudaMemcpyAsync(pb, db, 8, cudaMemcpyDeviceToHost, b); }},
        {"cudaStreamSynchronize(b)", [&] { cudaStreamSynchronize(b); }},
        {"8-CTA cluster kernel on b + sync b", [&] { clus<<<8, 512, 0, b>>>((int*)db); cudaStreamSynchronize(b); }},
        {"8-CTA cluster kernel again", [&] { clus<<<8, 512, 0, b>>>((int*)db); cudaStreamSynchronize(b); }},
        {"nop2 (preloaded: GetAttributes)", [&] { nop2<<<1, 1, 0, b>>>(); cudaStreamSynchronize(b); }},
        {"nop3 (preloaded: SetAttribute)", [&] { nop3<<<1, 1, 0, b>>>(); cudaStreamSynchronize(b); }},
        {"clus2 (preloaded) <<<>>>", [&] { clus2<<<8, 512, 0, b>>>((int*)db); cudaStreamSynchronize(b); }},
        {"clus3 (preloaded) LaunchKernelEx cluster 8", [&] {
             cudaLaunchConfig_t cfg{}; cudaLaunchAttribute at[1];
             at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = 8; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
             cfg.gridDim = dim3(8); cfg.blockDim = dim3(512); cfg.stream = b; cfg.attrs = at; cfg.numAttrs = 1;
             int* o = (int*)db; cudaLaunchKernelEx(&cfg, clus3, o); cudaStreamSynchronize(b); }},
        {"plain 8x512 kernel + sync b", [&] { nop<<<8, 512, 0, b>>>(); cudaStreamSynchronize(b); }},
    };
    for (auto& t : tests) {
        spin<<<1, 32, 0, a>>>();
        std::thread A([&] { cudaMemcpyAsync(pa, da, 8, cudaMemcpyDeviceToHost, a); });
        std::this_thread::sleep_for(std::chrono::milliseconds(200));
        const auto t0 = std::chrono::steady_clock::now();
        t.f();
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        A.join();
        cudaDeviceSynchronize();
        std::printf("%-28s %8.2f ms %s (%s)\n", t.name, ms, ms > 1000 ? "BLOCKED behind the other thread's copy" : "",
                    cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

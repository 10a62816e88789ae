// Which CUDA runtime calls block while another stream's kernel is still running?
// A spinning kernel (released by a host-mapped flag after ~2 s, or when the call
// under test returns) runs on stream A; the host times each call; a call that
// takes ~2 s waited for the device.  (Decides what the peer-memory exchange tests
// of ranks sharing one GPU may call between exchanges.)
// nvcc -gencode arch=compute_100a,code=sm_100a -o tools/sync_probe_bin tools/sync_probe.cu
#include <chrono>
#include <cstdio>
#include <functional>
#include <cuda_runtime.h>
__global__ void spin(volatile int* release) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); } while (!*release && t - t0 < 2000000000ull);
}
__global__ void nop() {}
int main() {
    int* h; int* d;
    cudaHostAlloc((void**)&h, 4, cudaHostAllocMapped);
    cudaHostGetDevicePointer((void**)&d, h, 0);
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    void* pre = nullptr; cudaMalloc(&pre, 1 << 20);
    void* preh = nullptr; cudaMallocHost(&preh, 1 << 20);
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(b, cudaStreamCaptureModeThreadLocal); nop<<<1, 1, 0, b>>>(); cudaStreamEndCapture(b, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaDeviceSynchronize();
    struct T { const char* name; std::function<void()> f; };
    void* p1 = nullptr; void* ph = nullptr;
    cudaGraph_t g2 = nullptr; cudaGraphExec_t ge2 = nullptr;
    T tests[] = {
        {"cudaMalloc 1MB", [&] { cudaMalloc(&p1, 1 << 20); }},
        {"cudaFree", [&] { cudaFree(p1); }},
        {"cudaMallocHost 1MB", [&] { cudaMallocHost(&ph, 1 << 20); }},
        {"cudaFreeHost", [&] { cudaFreeHost(ph); }},
        {"cudaMallocAsync+FreeAsync(b)", [&] { void* q; cudaMallocAsync(&q, 1 << 20, b); cudaFreeAsync(q, b); }},
        {"cudaEventCreate/Destroy", [&] { cudaEvent_t e; cudaEventCreate(&e); cudaEventDestroy(e); }},
        {"capture+instantiate (b)", [&] { cudaStreamBeginCapture(b, cudaStreamCaptureModeThreadLocal); nop<<<1, 1, 0, b>>>();
                                           cudaStreamEndCapture(b, &g2); cudaGraphInstantiate(&ge2, g2, 0); }},
        {"cudaGraphLaunch(b)+sync b", [&] { cudaGraphLaunch(ge2, b); cudaStreamSynchronize(b); }},
        {"cudaGraphExecDestroy", [&] { cudaGraphExecDestroy(ge2); cudaGraphDestroy(g2); }},
        {"cudaMemcpy H2D pageable 4KB", [&] { static char buf[4096]; cudaMemcpy(pre, buf, 4096, cudaMemcpyHostToDevice); }},
        {"cudaMemcpyAsync(b)+sync b", [&] { cudaMemcpyAsync(pre, preh, 4096, cudaMemcpyHostToDevice, b); cudaStreamSynchronize(b); }},
        {"cudaMemset", [&] { cudaMemset(pre, 0, 4096); }},
        {"cudaFuncSetAttribute", [&] { cudaFuncSetAttribute(nop, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024); }},
        {"cudaStreamCreate/Destroy", [&] { cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); cudaStreamDestroy(s); }},
    };
    for (auto& t : tests) {
        *h = 0;
        spin<<<1, 32, 0, a>>>(d);
        cudaStreamQuery(a);
        const auto t0 = std::chrono::steady_clock::now();
        t.f();
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        *h = 1;
        cudaDeviceSynchronize();
        std::printf("%-32s %8.2f ms %s  (%s)\n", t.name, ms, ms > 1000 ? "WAITED FOR THE DEVICE" : "",
                    cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}

// latency_probe.cu -- dependent-load latency seen by ONE CTA (design probe for the
// latency-bound single-CTA kernels: tree walk, phase B), sm_100a.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

__global__ void chase(const int* __restrict__ nxt, int steps, int* out, unsigned long long* cyc) {
    int i = threadIdx.x * 97 % 1024;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int s = 0; s < steps; ++s) i = nxt[i];
    const unsigned long long t1 = clock64();
    if (i == -12345) out[0] = i;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    const int N = 1 << 18;   // 1 MB of ints
    std::vector<int> perm(N), nxt(N);
    for (int k = 0; k < N; ++k) perm[k] = k;
    srand(1);
    for (int k = N - 1; k > 0; --k) { int j = rand() % (k + 1); std::swap(perm[k], perm[j]); }
    for (int k = 0; k < N; ++k) nxt[perm[k]] = perm[(k + 1) % N];
    int *d, *o; unsigned long long* c;
    cudaMalloc(&d, N * sizeof(int)); cudaMalloc(&o, 4); cudaMalloc(&c, 8);
    cudaMemcpy(d, nxt.data(), N * sizeof(int), cudaMemcpyHostToDevice);
    for (int threads : {32, 512}) {
        for (int rep = 0; rep < 3; ++rep) {
            chase<<<1, threads>>>(d, 2000, o, c);
            unsigned long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("threads %4d rep %d: %.1f cycles per dependent load (1 MB, L2-resident after rep 0)\n", threads, rep, h / 2000.0);
        }
    }
    return 0;
}

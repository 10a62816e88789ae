// mds_tree.cu -- the standalone Brownian-diffusion prior kernel (see mds_tree.cuh;
// the walk itself is in mds_tree_impl.cuh).
#include <cuda_runtime.h>
#include "mds_tree_impl.cuh"

namespace mdsk {
namespace {

constexpr int TT = 512;

template <int D>
__global__ void __launch_bounds__(TT, 1) tree_prior_kernel(TreeArgs a) {
    extern __shared__ __align__(16) double dyn[];
    __shared__ double red[TT / 32 + 1];
    treek::tree_prior_block<D, TT>(a, dyn, red);
}

template <int D>
void launch(const TreeArgs& a, cudaStream_t s) {
    static size_t set = 0;
    if (a.smem > set) {
        cudaFuncSetAttribute(tree_prior_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem);
        set = a.smem;
    }
    tree_prior_kernel<D><<<1, TT, a.smem, s>>>(a);
}

}  // namespace

void tree_preload(int d) {
    cudaFuncAttributes fa;
    switch (d) {
        case 1: cudaFuncGetAttributes(&fa, tree_prior_kernel<1>); break;
        case 2: cudaFuncGetAttributes(&fa, tree_prior_kernel<2>); break;
        case 3: cudaFuncGetAttributes(&fa, tree_prior_kernel<3>); break;
        case 4: cudaFuncGetAttributes(&fa, tree_prior_kernel<4>); break;
        case 5: cudaFuncGetAttributes(&fa, tree_prior_kernel<5>); break;
        case 6: cudaFuncGetAttributes(&fa, tree_prior_kernel<6>); break;
        case 7: cudaFuncGetAttributes(&fa, tree_prior_kernel<7>); break;
        default: cudaFuncGetAttributes(&fa, tree_prior_kernel<8>); break;
    }
}

void tree_prior_launch(const TreeArgs& a, int d, cudaStream_t s) {
    switch (d) {
        case 1: launch<1>(a, s); break;
        case 2: launch<2>(a, s); break;
        case 3: launch<3>(a, s); break;
        case 4: launch<4>(a, s); break;
        case 5: launch<5>(a, s); break;
        case 6: launch<6>(a, s); break;
        case 7: launch<7>(a, s); break;
        default: launch<8>(a, s); break;
    }
}

}  // namespace mdsk

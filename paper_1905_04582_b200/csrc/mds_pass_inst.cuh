// mds_pass_inst.cuh -- instantiate pass_kernel for one mode (MDS_MODE) and one
// storage precision (MDS_T, MDS_PREC_NAME) over truncation x D = 1..MDS_D_MAX.
#pragma once
#include "mds_pass.cuh"

namespace mdsk {
namespace {
template <typename T, bool TR, int MODE, int D>
PassKernel pk() {
    return PassKernel{pass_kernel<T, D, TR, MODE>, pass_smem_bytes<T, D>(), WarpsPerCTA<T, D>::value};
}
template <typename T, bool TR, int MODE>
PassKernel pass_fn_d(int d) {
#ifdef MDS_AB_D2ONLY
    // A/B builds: only D = 2 is instantiated (fast compile; other d are not valid)
    (void)d;
#if defined(MDS_AB_D6)
    return pk<T, TR, MODE, 6>();
#elif defined(MDS_AB_DV)
    return pk<T, TR, MODE, MDS_AB_DV>();
#else
    return pk<T, TR, MODE, 2>();
#endif
#else
    switch (d) {
        case 1: return pk<T, TR, MODE, 1>();
        case 2: return pk<T, TR, MODE, 2>();
        case 3: return pk<T, TR, MODE, 3>();
        case 4: return pk<T, TR, MODE, 4>();
        case 5: return pk<T, TR, MODE, 5>();
        case 6: return pk<T, TR, MODE, 6>();
        case 7: return pk<T, TR, MODE, 7>();
        default: return pk<T, TR, MODE, 8>();
    }
#endif
}
}  // namespace
}  // namespace mdsk

#define MDS_PASS_DEFINE(M, T, NAME)                                                                   \
    namespace mdsk {                                                                                  \
    PassKernel pass_m##M##_##NAME(int trunc, int d) {                                                 \
        return trunc ? pass_fn_d<T, true, M>(d) : pass_fn_d<T, false, M>(d);                          \
    }                                                                                                 \
    }

// pass_kernel instantiations: mode 8, f32 storage (see mds_pass.cuh)
#include "mds_pass_inst.cuh"
MDS_PASS_DEFINE(8, float, f32)

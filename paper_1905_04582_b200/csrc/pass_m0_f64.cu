// pass_kernel instantiations: mode 0, f64 storage (see mds_pass.cuh)
#include "mds_pass_inst.cuh"
MDS_PASS_DEFINE(0, double, f64)

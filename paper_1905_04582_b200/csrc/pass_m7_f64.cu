// pass_kernel instantiations: mode 7, f64 storage (see mds_pass.cuh)
#include "mds_pass_inst.cuh"
MDS_PASS_DEFINE(7, double, f64)

// pass_kernel instantiations: mode 3, f64 storage (see mds_pass.cuh)
#include "mds_pass_inst.cuh"
MDS_PASS_DEFINE(3, double, f64)

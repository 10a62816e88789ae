/*
 * mds_bench.h -- measurement utilities exported by libmds.so that are NOT part
 * of the method (PAPER.md's likelihood/gradient path is include/mds.h).  They
 * exist so that bench.py and the profiling tools can time the pass kernel the
 * way B200_PROFILING.md prescribes (cold L2 between timed launches, a measured
 * FP64/FP32 lane peak for the ALU roofline) with launches shaped like the
 * pass kernel's.  Conventions as include/mds.h.
 */
#ifndef MDS_BENCH_H
#define MDS_BENCH_H

#include <stddef.h>
#include "mds.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Timing utility (not part of the method): overwrite `bytes` of the device
 * buffer `dev_buf` (caller-owned, >= 16 bytes; use more than the 126 MB L2)
 * on the context's stream, launched with the pass kernel's grid, block size and
 * dynamic shared memory so the SMs keep the pass kernel's L1/shared split
 * between timed passes (a flush with another split makes the next pass
 * reconfigure the SMs inside the timed region).  Errors: MDS_E_INVALID_ARG,
 * MDS_E_CUDA. */
mds_status mds_l2_flush(mds_ctx ctx, void *dev_buf, size_t bytes);

/* As mds_l2_flush on the first half of dev_buf, then a read of the second half
 * (each half should exceed the 126 MB L2): the dirty lines the write leaves are
 * written back inside the flush, so a following timed kernel starts from a cold
 * AND clean L2.  Same launch shape as mds_l2_flush.  Errors as mds_l2_flush. */
mds_status mds_l2_flush_clean(mds_ctx ctx, void *dev_buf, size_t bytes);

/* Measure this device's FP64 (dfma) and FP32 (ffma) lane throughput with a
 * register-resident dependent-chain microbenchmark; results in lane-FMA/s.
 * Used for the ALU roofline denominator. */
mds_status mds_measure_fma_peaks(double *fp64_fma_per_s, double *fp32_fma_per_s);

#ifdef __cplusplus
}
#endif
#endif /* MDS_BENCH_H */

#!/bin/bash
# Round-2 profiles of the headline kernel (run on the GPU box via gpurun):
#  1. launch list of a short C5 bench (gpu__time_duration per launch, cold, serialised)
#  2. ncu --set full of ONE timed C5 leapfrog pass (pass_kernel<double,2,1,2>)
#  3. ncu --set full of ONE timed C2 leapfrog pass
# -> gpurun_out/r2_*.{csv,ncu-rep,log}
set -u
OUT=gpurun_out
K='regex:pass_kernel<double, \(int\)2, \(bool\)1, \(int\)2>'
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $OUT/r2_launches_c5.csv python bench.py --steps 3 --warmup 3 --extra none --no-cpu-baseline \
  --e2e-seconds 0.1 > $OUT/r2_launches_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" \
  --launch-skip 4 -c 1 -o $OUT/r2_c5 python bench.py --steps 3 --warmup 3 --extra none --no-cpu-baseline \
  --e2e-seconds 0.1 > $OUT/r2_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" \
  --launch-skip 4 -c 1 -o $OUT/r2_c2 python bench.py --workload C2 --steps 3 --warmup 3 --extra none \
  --no-cpu-baseline --e2e-seconds 0.1 > $OUT/r2_c2.log 2>&1
ls -la $OUT/r2_*
# 4. C4 fp32 (issue-bound fp32 pass)
K32='regex:pass_kernel<float, \(int\)6, \(bool\)1, \(int\)2>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K32" \
  --launch-skip 4 -c 1 -o $OUT/r2_c4f32 python bench.py --workload C4 --precision f32 --steps 3 --warmup 3 \
  --extra none --no-cpu-baseline --e2e-seconds 0.1 > $OUT/r2_c4f32.log 2>&1
# 5. C4 fp64
K64='regex:pass_kernel<double, \(int\)6, \(bool\)1, \(int\)2>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K64" \
  --launch-skip 4 -c 1 -o $OUT/r2_c4 python bench.py --workload C4 --steps 3 --warmup 3 \
  --extra none --no-cpu-baseline --e2e-seconds 0.1 > $OUT/r2_c4.log 2>&1
ls -la $OUT/r2_c4*

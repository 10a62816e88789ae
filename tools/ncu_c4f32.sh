OUT=gpurun_out
K32='regex:pass_kernel<float, \(int\)6, \(bool\)1, \(int\)2>'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K32" \
  --launch-skip 4 -c 1 -o $OUT/r2_c4f32 python bench.py --workload C4 --precision f32 --steps 3 --warmup 3 \
  --extra none --no-cpu-baseline --e2e-seconds 0.1 > $OUT/r2_c4f32.log 2>&1

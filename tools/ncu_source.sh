set -u
OUT=gpurun_out
K='regex:pass_kernel<double, \(int\)2, \(bool\)1, \(int\)2>'
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "$K" \
  --launch-skip 4 -c 1 -o $OUT/s_c2 python bench.py --workload C2 --steps 3 --warmup 3 --extra none \
  --no-cpu-baseline --e2e-seconds 0.1 > $OUT/s_c2.log 2>&1
ncu -i $OUT/s_c2.ncu-rep --page source --csv --print-source sass > $OUT/s_c2_source.csv 2>&1
ls -la $OUT

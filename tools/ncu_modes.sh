#!/bin/bash
# ncu --set full of the pass kernel's other modes (3 LEAPFROG_NOLIK, 4 LIK, 5 LEAPFROG_TREE)
# while tools/run_next.py runs them -> gpurun_out/nx_mode<M>.ncu-rep
for m in 3 4 5; do
  timeout 300 ncu --set full --clock-control none --kernel-name-base demangled \
    -k "regex:pass_kernel<double, \(int\)2, \(bool\)1, \(int\)$m>" -c 1 -o gpurun_out/nx_mode$m \
    python tools/run_next.py > gpurun_out/nx_mode$m.log 2>&1
done

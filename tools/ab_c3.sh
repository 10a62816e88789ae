#!/bin/bash
# C3 (HMC chain on the C2 data, 1000 x 20 leapfrog steps, one CUDA graph per
# transition) with and without programmatic dependent launch between the steps
for r in 1 2; do
  for v in pdl nopdl; do
    if [ $v = nopdl ]; then export MDS_NO_PDL=1; else unset MDS_NO_PDL; fi
    echo "$r $v $(timeout 600 python tools/run_configs.py --skip-c4 2>/dev/null | grep '"C3"' | head -1)" >> gpurun_out/ab_c3.txt
  done
done

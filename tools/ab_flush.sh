#!/bin/bash
# bench.py with the L2 flush variants between timed steps, alternating -> gpurun_out/ab_flush.txt
for r in $(seq $1); do
  for f in mds mds-clean; do
    timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 3 --flush $f > gpurun_out/abf.json 2> /dev/null
    echo "$f $(python -c "import json;d=json.load(open('gpurun_out/abf.json'));print(round(d['value']/1e9,2), round(d['ms_per_step']*1e3,2))")" >> gpurun_out/ab_flush.txt
  done
done

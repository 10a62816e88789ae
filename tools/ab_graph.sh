#!/bin/bash
# bench.py with stream launches vs one CUDA graph of the timed steps -> gpurun_out/ab_graph.txt
for r in $(seq $1); do
  for g in 0 1; do
    timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 3 --graph $g > gpurun_out/abg_$g.json 2> gpurun_out/abg_$g.err
    echo "graph=$g $(python -c "import json;d=json.load(open('gpurun_out/abg_$g.json'));print(round(d['value']/1e9,2), round(d['ms_per_step']*1e3,2), round(d['step_ms_p50']*1e3,2))")" >> gpurun_out/ab_graph.txt
  done
done

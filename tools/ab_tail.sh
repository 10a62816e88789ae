#!/bin/bash
# dynamic tail A/B (MDS_TAIL_CHUNK: groups per chunk, 0 = no tail): C2 bench step
# (L2 flushed) and the N = 30000 leapfrog pass; phases of the C2 pass per variant
OUT=gpurun_out/ab_tail.txt
for r in 1 2; do
  for v in 0 4 2; do
    MDS_TAIL_CHUNK=$v timeout 300 python bench.py --workload C2 --steps 200 --warmup 20 --extra none \
      --no-cpu-baseline --e2e-seconds 0.2 > gpurun_out/abt_$v.json 2>/dev/null
    echo "$r chunk=$v C2 $(python -c "import json;d=json.load(open('gpurun_out/abt_$v.json'));print(round(d['value']/1e9,2), round(d['ms_per_step']*1e3,2))")" >> $OUT
  done
done
for v in 0 4 2; do
  MDS_TAIL_CHUNK=$v MDS_PROFILE_PHASES=1 timeout 300 python bench.py --workload C2 --steps 20 --warmup 5 --extra none \
    --no-cpu-baseline --e2e-seconds 0.1 2>&1 >/dev/null | grep "phases us" | head -2 | sed "s/^/chunk=$v /" >> $OUT
done
for v in 0 4; do
  for r in 1 2; do
    echo "n30000 chunk=$v $(MDS_TAIL_CHUNK=$v timeout 300 python tools/ab_pass.py --child --n 30000 --steps 60 2>/dev/null | tail -1)" >> $OUT
  done
done

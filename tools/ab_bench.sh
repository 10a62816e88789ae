#!/bin/bash
# A/B: alternate bench.py runs between the in-tree libmds.so and paper_1905_04582_b200/libmds_ab_<name>.so
# usage: tools/ab_bench.sh name [rounds]
name=$1; rounds=${2:-2}
for r in $(seq $rounds); do
  for v in cur $name; do
    if [ $v = cur ]; then L=; else L=paper_1905_04582_b200/libmds_ab_$v.so; fi
    MDS_LIB_PATH=$L timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    echo "$v $(python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print(round(d['value']/1e9,2), round(d['ms_per_step']*1e3,2))")" >> gpurun_out/ab.txt
  done
done

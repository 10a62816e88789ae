#!/bin/bash
# A/B on one box: alternate bench.py runs between the in-tree libmds.so ("cur")
# and paper_1905_04582_b200/libmds_ab_<name>.so for each name given.
# usage: tools/ab_bench.sh rounds name [name ...]   -> gpurun_out/ab.txt
rounds=$1; shift
for r in $(seq $rounds); do
  for v in cur "$@"; do
    if [ $v = cur ]; then L=; else L=paper_1905_04582_b200/libmds_ab_$v.so; fi
    MDS_LIB_PATH=$L timeout 300 python bench.py --steps 2000 --warmup 20 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
    echo "$v $(python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print(round(d['value']/1e9,2), round(d['ms_per_step']*1e3,2))")" >> gpurun_out/ab.txt
  done
done

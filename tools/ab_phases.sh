#!/bin/bash
# phase breakdown (MDS_PROFILE_PHASES) of the in-tree library and each libmds_ab_<v>.so given
for v in cur "$@"; do
  if [ $v = cur ]; then L=; else L=paper_1905_04582_b200/libmds_ab_$v.so; fi
  MDS_LIB_PATH=$L MDS_PROFILE_PHASES=1 timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 3 > gpurun_out/abp_$v.json 2> gpurun_out/abp_$v.err
  echo "$v $(python -c "import json;d=json.load(open('gpurun_out/abp_$v.json'));print(round(d['value']/1e9,2), round(d['ms_per_step']*1e3,2))") $(grep 'phases us' gpurun_out/abp_$v.err | tail -2 | tr '\n' ' ')" >> gpurun_out/abp.txt
done

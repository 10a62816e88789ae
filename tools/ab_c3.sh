#!/bin/bash
# C3 HMC chain (tools/run_configs.py --skip-c4, 300 transitions) for the in-tree
# libmds.so and each libmds_ab_<name>.so given, alternating -> gpurun_out/ab_c3.txt
rounds=$1; shift
for r in $(seq $rounds); do
  for v in cur "$@"; do
    if [ $v = cur ]; then L=; else L=paper_1905_04582_b200/libmds_ab_$v.so; fi
    echo "$v $(MDS_LIB_PATH=$L timeout 300 python tools/run_configs.py --skip-c4 --c3-iter 300 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(round(d['device_seconds'],4), round(d['evals_per_s']))")" >> gpurun_out/ab_c3.txt
  done
done

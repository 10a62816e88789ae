for r in 1 2; do
for v in cur plain; do
  if [ $v = cur ]; then L=; else L=paper_1905_04582_b200/libmds_ab_$v.so; fi
  MDS_LIB_PATH=$L timeout 300 python bench.py --workload C2 --steps 200 --warmup 20 --extra none --no-cpu-baseline --e2e-seconds 0.5 > gpurun_out/abc2_$v.json 2>/dev/null
  echo "$r $v C2 $(python -c "import json;d=json.load(open('gpurun_out/abc2_$v.json'));print(round(d['value']/1e9,2), round(d['ms_per_step']*1e3,2), 'e2e', round(d['e2e']['value']/1e9,2))")" >> gpurun_out/abc2.txt
done
done
timeout 600 python tools/ab_pass.py --n 30000 --steps 60 --rounds 2 cur paper_1905_04582_b200/libmds_ab_plain.so >> gpurun_out/abc2.txt 2>&1

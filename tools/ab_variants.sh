for v in base NO_COLRED NO_TMA; do
  if [ $v = base ]; then L=; else L=paper_1905_04582_b200/libmds_exp_$v.so; fi
  MDS_LIB_PATH=$L MDS_PROFILE_PHASES=1 timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 3 > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  echo "$v $(grep phases gpurun_out/ab_$v.err | tail -1)" >> gpurun_out/ab.txt
done

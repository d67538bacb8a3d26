# A/B round: parity subset, bench for each library variant, ncu on the default build
set -x
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke3.log 2>&1; echo rc=$? >> gpurun_out/smoke3.log
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > gpurun_out/gpu_tests3.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests3.log
for v in "" b3; do
  if [ -n "$v" ]; then export SFV_LIB=$PWD/paper_2305_18057_b200/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ab_${v:-b4}.json 2> gpurun_out/bench_ab_${v:-b4}.err
done
unset SFV_LIB
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_stage3 python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full3.log 2>&1

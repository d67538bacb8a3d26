set -x
TAG=${1:-ab}
timeout 900 python -m pytest tests -m gpu -q -x --timeout=600 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_$TAG.log
for v in "" b3; do
  if [ -n "$v" ]; then export SFV_LIB=$PWD/paper_2305_18057_b200/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_${v:-b4}.json 2> gpurun_out/bench_${TAG}_${v:-b4}.err
done
unset SFV_LIB
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1

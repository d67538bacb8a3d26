set -x
TAG=${1:-cpl}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/gpu_tests_${TAG}_1.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_${TAG}_1.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_1.json 2>&1
timeout 300 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_1_c3.json 2>&1
export SFV_LIB=$PWD/paper_2305_18057_b200/libsfv_cpl2.so
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/gpu_tests_${TAG}_2.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_${TAG}_2.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_2.json 2>&1
timeout 300 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_2_c3.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_${TAG}_2 python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}_2.log 2>&1

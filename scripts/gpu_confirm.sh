# HEAD confirmation: GPU tests, C2/C3/C4 bench lines, reference arm, launch list, ncu full (C2)
TAG=${1:-cf}
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi_$TAG.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
timeout 400 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err
timeout 400 python bench.py --workload C4 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err
timeout 400 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1

# full bench line + launch list + full ncu capture of the stage kernels (current build)
TAG=${1:-ev}
set -x
timeout 600 python bench.py > gpurun_out/bench_${TAG}_full.json 2> gpurun_out/bench_${TAG}_full.err
timeout 400 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:stage_kernel -s 20 -c 4 -o gpurun_out/prof_${TAG}_c3 python bench.py --workload C3 --steps 6 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}_c3.log 2>&1

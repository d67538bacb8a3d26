set -x
TAG=${1:-ab}
timeout 300 python bench.py > gpurun_out/bench_${TAG}_full.json 2> gpurun_out/bench_${TAG}_full.err
export SFV_LIB=$PWD/paper_2305_18057_b200/libsfv_b2.so
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_b2.json 2> gpurun_out/bench_${TAG}_b2.err
unset SFV_LIB
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1

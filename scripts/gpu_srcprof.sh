# ncu source-level (per-SASS-instruction executed counts) profile of the C2 stage kernels
# usage: bash scripts/gpu_srcprof.sh TAG [LIB]
TAG=${1:-src}
[ -n "$2" ] && export SFV_LIB=$2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_$TAG -f python bench.py --steps 20 --warmup 10 --min-timed-s 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 20 -c 4 -o gpurun_out/prof_${TAG}_c3 -f python bench.py --workload C3 --steps 6 --warmup 5 --min-timed-s 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}_c3.log 2>&1
ncu -i gpurun_out/prof_${TAG}_c3.ncu-rep --page source --csv --print-source sass > gpurun_out/src_${TAG}_c3.csv 2>/dev/null; gzip -f gpurun_out/src_${TAG}_c3.csv
ncu -i gpurun_out/prof_${TAG}_c3.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__cycles_elapsed.avg > gpurun_out/raw_${TAG}_c3.csv 2>/dev/null; rm -f gpurun_out/prof_${TAG}_c3.ncu-rep
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$TAG.csv 2>/dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__cycles_elapsed.avg > gpurun_out/raw_$TAG.csv 2>/dev/null
gzip -f gpurun_out/src_$TAG.csv
rm -f gpurun_out/prof_$TAG.ncu-rep

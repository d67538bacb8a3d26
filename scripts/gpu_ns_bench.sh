# Navier-Stokes mode: bench line (C2 with viscous terms, no-slip ramp) + launch list
TAG=${1:-ns}
set -x
timeout 600 python bench.py --ns --steps 2000 --warmup 20 > gpurun_out/bench_${TAG}_ns_c2.json 2> gpurun_out/bench_${TAG}_ns_c2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_ns.csv python bench.py --ns --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_${TAG}_ns.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"visc_kernel|grad_kernel" -s 8 -c 2 -o gpurun_out/prof_${TAG}_ns python bench.py --ns --steps 4 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}_ns.log 2>&1

set -x
for rk in rk4 heun jst4; do
  timeout 300 python bench.py --rk $rk --no-cpu-baseline --no-e2e > gpurun_out/bench_rk_$rk.json 2> gpurun_out/bench_rk_$rk.err
  timeout 300 python bench.py --rk $rk --workload C3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_rk_${rk}_c3.json 2> gpurun_out/bench_rk_${rk}_c3.err
done

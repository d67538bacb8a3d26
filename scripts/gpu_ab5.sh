set -x
for v in "" w16; do
  if [ -n "$v" ]; then export SFV_LIB=$PWD/paper_2305_18057_b200/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ab5_${v:-base}.json 2>&1
  timeout 300 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_ab5_${v:-base}_c3.json 2>&1
done

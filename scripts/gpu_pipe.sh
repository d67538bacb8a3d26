set -x
TAG=${1:-pp}
for v in "" pipe; do
  if [ -n "$v" ]; then export SFV_LIB=$PWD/paper_2305_18057_b200/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_${v:-base}.json 2> gpurun_out/bench_${TAG}_${v:-base}.err
  timeout 300 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_${v:-base}_c3.json 2> gpurun_out/bench_${TAG}_${v:-base}_c3.err
done
export SFV_LIB=$PWD/paper_2305_18057_b200/libsfv_pipe.so
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log

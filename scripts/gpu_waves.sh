set -x
TAG=${1:-wv}
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
for w in 0 2 3 4; do
  if [ "$w" != "0" ]; then export SFV_WAVES=$w; else unset SFV_WAVES; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_w$w.json 2> gpurun_out/bench_${TAG}_w$w.err
done
unset SFV_WAVES
timeout 300 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err

set -x
TAG=${1:-ab}
for v in "" b3 seq; do
  if [ -n "$v" ]; then export SFV_LIB=$PWD/paper_2305_18057_b200/libsfv_$v.so; else unset SFV_LIB; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_${TAG}_${v:-b4}.json 2> gpurun_out/bench_${TAG}_${v:-b4}.err
done

set -x
for v in "" 1; do
  if [ -n "$v" ]; then export SFV_EXP_NOFIN=1; else unset SFV_EXP_NOFIN; fi
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ab6_${v:-base}.json 2>&1
  timeout 300 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/bench_ab6_${v:-base}_c3.json 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ab6_${v:-base}_b.json 2>&1
done
for f in gpurun_out/bench_ab6_*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done

# A/B: per-task inter-stage dependencies (default) vs whole-grid griddepcontrol.wait (SFV_XDEP=0)
TAG=${1:-x}
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout=500 -p no:cacheprovider > gpurun_out/xdep_tests_$TAG.log 2>&1; echo rc=$? >> gpurun_out/xdep_tests_$TAG.log
B="python bench.py --no-cpu-baseline --no-e2e"
for v in 1 0 1 0; do
  SFV_XDEP=$v timeout 300 $B --steps 3000 > gpurun_out/xd_${TAG}_c2_$v.json 2>&1
  SFV_XDEP=$v timeout 300 $B --workload C3 --steps 60 --warmup 5 > gpurun_out/xd_${TAG}_c3_$v.json 2>&1
  for f in gpurun_out/xd_${TAG}_c2_$v.json gpurun_out/xd_${TAG}_c3_$v.json; do python -c "
import json
L=[l for l in open('$f').read().splitlines() if l.startswith('{')]
d=json.loads(L[-1]) if L else {}
print('$f', round(d.get('value',0)), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))
" >> gpurun_out/xd_${TAG}_summary.txt; done
done

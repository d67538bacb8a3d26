# A/B of libsfv builds on C2 and C3 (+ optional pytest): gpu_ab2.sh TAG "V1 V2 ..." [pytest-args]
# (variant "cur" = libsfv.so, else paper_2305_18057_b200/libsfv_V.so)
TAG=$1; VARS=$2; shift 2
set -x
[ -n "$1" ] && timeout 1500 python -m pytest tests -q -x -p no:cacheprovider "$@" > gpurun_out/t_$TAG.txt 2>&1
lib() { if [ "$1" = "cur" ]; then echo paper_2305_18057_b200/libsfv.so; else echo paper_2305_18057_b200/libsfv_$1.so; fi; }
B_="python bench.py --no-cpu-baseline --no-e2e"
for rep in 1 2; do for v in $VARS; do
  SFV_LIB=$(lib $v) timeout 300 $B_ --steps 3000 > gpurun_out/ab_${TAG}_c2_${v}_$rep.json 2>&1
  SFV_LIB=$(lib $v) timeout 300 $B_ --workload C3 --steps 60 --warmup 5 > gpurun_out/ab_${TAG}_c3_${v}_$rep.json 2>&1
done; done
for f in gpurun_out/ab_${TAG}_*.json; do python -c "
import json
L=[l for l in open('$f').read().splitlines() if l.startswith('{')]
d=json.loads(L[-1]) if L else {}
print('$f', round(d.get('value',0)), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))
"; done > gpurun_out/ab_${TAG}_summary.txt

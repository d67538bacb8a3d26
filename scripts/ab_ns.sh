# A/B of libsfv builds on the Navier-Stokes bench (C2 grid) inside one gpurun call:
#   bash scripts/ab_ns.sh TAG VARIANT...   (variant "cur" = libsfv.so, else libsfv_VARIANT.so)
TAG=$1; shift
lib() { if [ "$1" = "cur" ]; then echo paper_2305_18057_b200/libsfv.so; else echo paper_2305_18057_b200/libsfv_$1.so; fi; }
for rep in 1 2; do
for v in "$@"; do
  SFV_LIB=$(lib "$v") timeout 300 python bench.py --ns --steps 500 --warmup 20 --no-cpu-baseline --no-e2e > gpurun_out/abns_${TAG}_${v}_$rep.json 2>&1
done
done
for f in gpurun_out/abns_${TAG}_*.json; do python -c "
import json
L=[l for l in open('$f').read().splitlines() if l.startswith('{')]
d=json.loads(L[-1]) if L else {}
print('$f', round(d.get('value',0) or 0), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))
"; done > gpurun_out/abns_${TAG}_summary.txt

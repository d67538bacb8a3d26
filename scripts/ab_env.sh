# A/B of environment settings of one libsfv build on C2 inside one gpurun call:
#   bash scripts/ab_env.sh TAG "NAME=ENV1 ENV2" "NAME2=ENV ..." ...   (NAME=base: no extra env)
TAG=$1; shift
for rep in 1 2; do
for spec in "$@"; do
  name=${spec%%=*}; envs=${spec#*=}
  env $envs timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3000 > gpurun_out/abenv_${TAG}_${name}_$rep.json 2>&1
done
done
for f in gpurun_out/abenv_${TAG}_*.json; do python -c "
import json
L=[l for l in open('$f').read().splitlines() if l.startswith('{')]
d=json.loads(L[-1]) if L else {}
print('$f', round(d.get('value',0) or 0), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))
"; done > gpurun_out/abenv_${TAG}_summary.txt

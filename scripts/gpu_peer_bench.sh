# loopback partition overhead: 1 block vs 8 slabs (copy / peer halo) on one GPU; N>1 functional check of peer mode
TAG=${1:-pb}
set -x
B="python bench.py --no-cpu-baseline --no-e2e"
timeout 300 $B --steps 3000 > gpurun_out/pb_${TAG}_c2_1.json 2>&1
timeout 300 $B --steps 3000 --blocks 8 --halo copy > gpurun_out/pb_${TAG}_c2_8copy.json 2>&1
timeout 300 $B --steps 3000 --blocks 8 --halo peer > gpurun_out/pb_${TAG}_c2_8peer.json 2>&1
timeout 300 $B --workload C3 --steps 60 --warmup 5 > gpurun_out/pb_${TAG}_c3_1.json 2>&1
timeout 300 $B --workload C3 --steps 60 --warmup 5 --blocks 8 --halo copy > gpurun_out/pb_${TAG}_c3_8copy.json 2>&1
timeout 300 $B --workload C3 --steps 60 --warmup 5 --blocks 8 --halo peer > gpurun_out/pb_${TAG}_c3_8peer.json 2>&1
SFV_SIM_HOSTS=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 200 --warmup 5 --no-e2e > gpurun_out/pb_${TAG}_sim2_peer.json 2>&1
for f in gpurun_out/pb_${TAG}_*.json; do python -c "
import json
L=[l for l in open('$f').read().splitlines() if l.startswith('{')]
d=json.loads(L[-1]) if L else {}
print('$f', round(d.get('value',0)), d.get('gpu_launches'), d.get('config',{}).get('halo'), d.get('clocks',{}).get('sm_mhz'), d.get('clocks',{}).get('reasons'))
"; done > gpurun_out/pb_${TAG}_summary.txt

# NCCL path on one GPU: simulated hosts per rank (tests/test_gpu_nccl.py) and
# bench.py's N>1 code path under torchrun (functional check, not a bench value)
set -x
export NCCL_DEBUG=WARN
timeout 900 python -m pytest tests/test_gpu_nccl.py -q -m gpu 2>&1 | tail -30
SFV_SIM_HOSTS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sim2.json 2> gpurun_out/bench_sim2.err
tail -5 gpurun_out/bench_sim2.err; cat gpurun_out/bench_sim2.json
SFV_SIM_HOSTS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
  bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/bench_sim2_ref.json 2> gpurun_out/bench_sim2_ref.err
tail -3 gpurun_out/bench_sim2_ref.err; cat gpurun_out/bench_sim2_ref.json
SFV_SIM_HOSTS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29519 \
  bench.py --gpus 4 --steps 50 --warmup 3 --no-cpu-baseline > gpurun_out/bench_sim4.json 2> gpurun_out/bench_sim4.err
tail -3 gpurun_out/bench_sim4.err; cut -c1-400 gpurun_out/bench_sim4.json

# Round-end evidence for the committed build (run on the GPU box from the repo root):
#   bash scripts/gpu_evidence.sh TAG [PART]    PART = run (tests, smoke, bench lines, sanitizer) | ncu | all
# The ncu captures are summarised on the box (scripts/ncu_summary.py, scripts/sass_hot.py) and only the
# C2 report is kept: gpurun copies gpurun_out/ back only below 64 MiB.
# GPU tests, smoke, bench lines (driver-like C2, C3, C4, NS, reference arm, simulated 2-rank C3),
# ncu launch list and --set full captures of the stage kernels (C2, C3), compute-sanitizer.
TAG=${1:-ev}
PART=${2:-all}
set -x
if [ "$PART" != ncu ]; then
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi_$TAG.txt
timeout 1800 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo rc=$? >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_${TAG}_c2_driver.json 2> gpurun_out/bench_${TAG}_c2_driver.err
timeout 600 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
timeout 600 python bench.py --workload C3 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err
timeout 600 python bench.py --workload C4 --no-cpu-baseline > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err
timeout 600 python bench.py --ns --steps 500 --warmup 20 > gpurun_out/bench_${TAG}_ns.json 2> gpurun_out/bench_${TAG}_ns.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err
SFV_SIM_HOSTS=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --steps 10 --warmup 3 > gpurun_out/bench_${TAG}_sim2.json 2> gpurun_out/bench_${TAG}_sim2.err
bash scripts/gpu_sanitize.sh $TAG
fi
if [ "$PART" != run ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 40 --warmup 5 --min-timed-s 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_$TAG python bench.py --steps 20 --warmup 10 --min-timed-s 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:stage_kernel -s 20 -c 4 -o gpurun_out/prof_${TAG}_c3 python bench.py --workload C3 --steps 6 --warmup 5 --min-timed-s 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}_c3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"stage_kernel|gradvisc" -s 80 -c 8 -o gpurun_out/prof_${TAG}_ns python bench.py --ns --steps 20 --warmup 20 --min-timed-s 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_${TAG}_ns.log 2>&1
python scripts/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep --cells 1036800 --tag ${TAG}_stage_kernel_c2 --launches gpurun_out/launches_$TAG.csv --bench-json > /dev/null
python scripts/ncu_summary.py gpurun_out/prof_${TAG}_c3.ncu-rep --cells 66355200 --tag ${TAG}_stage_kernel_c3 > /dev/null
python scripts/ncu_summary.py gpurun_out/prof_${TAG}_ns.ncu-rep --cells 1036800 --tag ${TAG}_ns_kernels_c2 --ns-json > /dev/null
ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass > /tmp/src_$TAG.csv 2>/dev/null
for k in 0 1 3; do python scripts/sass_hot.py /tmp/src_$TAG.csv $k 1036800; echo; done > gpurun_out/${TAG}_stage_kernel_sass_hot.txt
cp profiles/${TAG}_* profiles/ncu_stage_kernel.json profiles/ncu_ns.json gpurun_out/ 2>/dev/null
rm -f gpurun_out/prof_${TAG}_c3.ncu-rep gpurun_out/prof_${TAG}_ns.ncu-rep
fi

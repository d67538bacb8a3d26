set -x
TAG=${1:-r}
timeout 1500 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests_$TAG.log
timeout 400 python bench.py > gpurun_out/bench_${TAG}_c2.json 2> gpurun_out/bench_${TAG}_c2.err
timeout 400 python bench.py --workload C3 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c3.json 2> gpurun_out/bench_${TAG}_c3.err
timeout 400 python bench.py --workload C4 --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/bench_${TAG}_c4.json 2> gpurun_out/bench_${TAG}_c4.err
timeout 400 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2> gpurun_out/bench_${TAG}_ref.err

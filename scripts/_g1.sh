nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/r2_smi_g1.txt
timeout 300 python bench.py --no-e2e > gpurun_out/r2_g1_bench_c2.json 2> gpurun_out/r2_g1_bench_c2.err
timeout 1500 python -m pytest tests -m gpu -q -x --timeout=900 -p no:cacheprovider > gpurun_out/r2_g1_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_g1_gpu_tests.log

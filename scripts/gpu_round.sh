set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi2.txt
timeout 1200 python -m pytest tests -m gpu -q --timeout=600 -p no:cacheprovider > gpurun_out/gpu_tests2.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests2.log
timeout 600 python bench.py > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$? >> gpurun_out/bench1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/prof_stage python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out

# NS: tests, then fused vs two-kernel bench lines and launch list
set -x
timeout 900 python -m pytest tests/test_gpu_ns.py -q --timeout=600 -p no:cacheprovider > gpurun_out/ns7.log 2>&1; echo rc=$? >> gpurun_out/ns7.log
for f in 1 0; do SFV_NS_FUSED=$f timeout 300 python bench.py --ns --steps 2000 --warmup 20 --no-cpu-baseline --no-e2e | tail -1 > gpurun_out/ns_ab_$f.json 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_ns7.csv python bench.py --ns --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1

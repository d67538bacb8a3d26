set -x
for v in cur vt12 vt6 cur vt12 vt6; do
  lib=paper_2305_18057_b200/libsfv.so; [ "$v" != cur ] && lib=paper_2305_18057_b200/libsfv_$v.so
  SFV_LIB=$lib timeout 300 python bench.py --ns --steps 2000 --warmup 20 --no-cpu-baseline --no-e2e | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value']), d['clocks']['sm_mhz'])" >> gpurun_out/ns_vt.txt 2>&1
done
SFV_LIB=paper_2305_18057_b200/libsfv_vt12.so timeout 600 python -m pytest tests/test_gpu_ns.py -q -p no:cacheprovider > gpurun_out/ns_vt_tests.log 2>&1; echo rc=$? >> gpurun_out/ns_vt_tests.log

timeout 1800 python -m pytest tests -m gpu -q --timeout=900 -p no:cacheprovider > gpurun_out/r2_g5_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_g5_gpu_tests.log

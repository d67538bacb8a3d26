timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_residual.py -q -x --timeout=600 -p no:cacheprovider -k "not perfmodel_geometry" > gpurun_out/r2_g4_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_g4_tests.log
bash scripts/ab_multi.sh diet base cur novote

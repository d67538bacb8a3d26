# A/B: parked 16-warp variant vs current
L=paper_2305_18057_b200/libsfv_p16.so
SFV_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_residual.py -q -x --timeout=600 -p no:cacheprovider > gpurun_out/r2_g2_p16_tests.log 2>&1; echo rc=$? >> gpurun_out/r2_g2_p16_tests.log
bash scripts/gpu_ab.sh p16 p16 cur

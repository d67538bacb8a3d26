# ncu of the parked 16-warp variant (C2), stage kernels of one step
SFV_LIB=paper_2305_18057_b200/libsfv_p16.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:stage_kernel -s 40 -c 4 -o gpurun_out/r2_prof_p16 python bench.py --steps 20 --warmup 10 --no-cpu-baseline --no-e2e > gpurun_out/r2_ncu_p16.log 2>&1

for v in base "" w1 w4 w7c; do lib=paper_2305_18057_b200/libsfv${v:+_$v}.so; SFV_LIB=$lib python scripts/occ_probe.py >> gpurun_out/occ.txt 2>&1; done
bash scripts/gpu_ab.sh rw1 base w1
bash scripts/gpu_ab.sh rw2 w4 w7c

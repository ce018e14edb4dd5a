timeout 1200 python tools/sweep_split.py 0,2,4 1,2,4,8 2 > gpurun_out/s2_sweep.txt 2>&1

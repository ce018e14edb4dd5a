# session 2: FCFS batch timeline (per-slice head steps, commits) full and culled
python tools/batch_timeline.py 0 > gpurun_out/s2_tl_full.txt 2>&1
python tools/batch_timeline.py 1 > gpurun_out/s2_tl_cull.txt 2>&1

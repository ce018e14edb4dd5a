FMDP_DEBUG_REUSE=1 python tools/batch_timeline.py 0 > gpurun_out/s2_reuse_full.txt 2>&1
FMDP_DEBUG_REUSE=1 python tools/batch_timeline.py 1 > gpurun_out/s2_reuse_cull.txt 2>&1

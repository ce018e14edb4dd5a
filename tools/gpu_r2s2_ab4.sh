# session 2, A/B 4: re-convergence after rollbacks (FCFS batch)
set -x
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab4_tests.txt
timeout 900 python tools/ab_old.py run 1 --batch > gpurun_out/s2_ab4.txt 2>&1
python tools/batch_timeline.py 0 > gpurun_out/s2_ab4_tl_full.txt 2>&1
python tools/batch_timeline.py 1 > gpurun_out/s2_ab4_tl_cull.txt 2>&1

# session 2, A/B 14: FIX items beside pass 1 in the FCFS walkers
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab14_cmp.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab14_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab14.txt 2>&1

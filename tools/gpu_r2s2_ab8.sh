# session 2, A/B 8: merged owner pass in the FCFS walkers
set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab8_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab8.txt 2>&1

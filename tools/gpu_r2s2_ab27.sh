# session 2, A/B 27: FIX (goal, deck, terrain of owned states) while the reduce-scatter is in flight
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab27_cmp.txt 2>&1
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab27.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab27_tests.txt

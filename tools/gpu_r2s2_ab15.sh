# session 2, A/B 15: SURVEY f1 range query (cell-sorted rows, 3x3 staging) in the culled walker
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab15_cmp.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s2_ab15_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab15.txt 2>&1

# session 2, A/B 13: pre-cull of the next row in the culled walker
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab13_cmp.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab13_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab13.txt 2>&1

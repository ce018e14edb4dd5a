# session 2, A/B 21: pass-1 G-way minimum as 16-byte loads, four items per thread
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab21_cmp.txt 2>&1
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab21.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab21_tests.txt

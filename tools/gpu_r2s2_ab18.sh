# session 2, A/B 17: range query for large rows only
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab18_cmp.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab18_tests.txt
timeout 900 python tools/ab_old.py run 1 --batch > gpurun_out/s2_ab18.txt 2>&1
timeout 1500 python tools/c4_index_probe.py > gpurun_out/s2_ab18_c4.txt 2>&1

# session 2, A/B 25: record build spread over the half-warps of every warp (passes of <= NT/2 plans)
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab25_cmp.txt 2>&1
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab25.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab25_tests.txt

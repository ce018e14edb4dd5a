# session 2, A/B 20: no CTA barrier after the last hot-loop pass
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab20_cmp.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab20_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab20.txt 2>&1

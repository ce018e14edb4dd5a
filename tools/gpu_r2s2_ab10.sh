# session 2, A/B 10: previous-step anchor + prebuild of the next step's records
set -x
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/s2_ab10_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab10.txt 2>&1

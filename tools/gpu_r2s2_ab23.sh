# session 2, A/B 23: full-path record build one (plan, tau) per thread
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab23_cmp.txt 2>&1
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab23.txt 2>&1
timeout 1200 python tools/chunk_probe.py 0 > gpurun_out/s2_ab23_chunk.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab23_tests.txt

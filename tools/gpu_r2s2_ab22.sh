# session 2, A/B 22: full-path build pass of 1024 / 768 plans where shared memory allows
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab22_cmp.txt 2>&1
timeout 1200 python tools/chunk_probe.py 0,512 > gpurun_out/s2_ab22_chunk.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/s2_ab22_tests.txt
timeout 900 python tools/ab_old.py run 1 --batch > gpurun_out/s2_ab22.txt 2>&1

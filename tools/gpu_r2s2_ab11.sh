timeout 600 python tools/batch_compare.py base nopre old > gpurun_out/s2_ab11_cmp.txt 2>&1
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab11.txt 2>&1

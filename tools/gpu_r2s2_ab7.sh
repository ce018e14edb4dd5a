timeout 1200 python tools/ab_old.py run 3 --batch > gpurun_out/s2_ab7.txt 2>&1

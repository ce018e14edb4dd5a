# session 2, A/B 16: range query with asynchronous range fetch; configs[3] probe
set -x
timeout 600 python tools/batch_compare.py base old > gpurun_out/s2_ab16_cmp.txt 2>&1
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab16.txt 2>&1
timeout 1500 python tools/c4_index_probe.py > gpurun_out/s2_ab16_c4.txt 2>&1

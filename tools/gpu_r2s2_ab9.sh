# session 2, A/B 9: stop flag loaded one step ahead
set -x
timeout 900 python -m pytest tests/test_gpu_reuse.py tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -2 > gpurun_out/s2_ab9_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab9.txt 2>&1
timeout 1500 python tools/sweep_split.py 2,4,6 4,2 2 4,8 > gpurun_out/s2_ab9_sweep.txt 2>&1

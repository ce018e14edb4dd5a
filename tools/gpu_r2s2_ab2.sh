# session 2, A/B 2: red.async reduce-scatter + division-free step indices vs HEAD
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_multi.py -q -x 2>&1 | tail -3 > gpurun_out/s2_ab2_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab2.txt 2>&1

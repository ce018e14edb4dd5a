# session 2, A/B 3: bulk-copy reduce-scatter, division-free indices, pass-2 warp skip, try_wait hint
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py tests/test_gpu_multi.py tests/test_gpu_cosim.py -q -x 2>&1 | tail -3 > gpurun_out/s2_ab3_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab3.txt 2>&1

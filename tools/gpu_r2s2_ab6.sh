# session 2, A/B 6: re-convergence in the culled walker only
set -x
timeout 1200 python -m pytest tests/test_gpu_reuse.py tests/test_gpu_bench_parity.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_multi.py -q -x -s 2>&1 | grep -E "reconverged|passed|failed|Error" | tail -8 > gpurun_out/s2_ab6_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab6.txt 2>&1

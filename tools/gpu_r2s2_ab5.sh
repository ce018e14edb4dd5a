# session 2, A/B 5: re-convergence incl. paused previous runs
set -x
timeout 1200 python -m pytest tests/test_gpu_reuse.py tests/test_gpu_bench_parity.py tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -s 2>&1 | grep -E "reconverged|passed|failed|Error" | tail -8 > gpurun_out/s2_ab5_tests.txt
timeout 900 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab5.txt 2>&1
python tools/batch_timeline.py 0 > gpurun_out/s2_ab5_tl_full.txt 2>&1

# session 2, A/B 1: projection prefetch (next step's candidate rows in shared memory)
set -x
./tools/hotbench/rates > gpurun_out/s2_rates2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bench_parity.py -q -x 2>&1 | tail -3 > gpurun_out/s2_ab1_tests.txt
timeout 600 python tools/step_probe.py --plans 0,3000 --reqs 2 --sizes 16,8 --phases --batch > gpurun_out/s2_ab1_probe.txt 2>&1

python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_dist_batch.py tests/test_gpu_accel.py -x -q 2>&1 | tail -3
FMDP_BENCH_SAME_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 1 --no-c4 --no-cpu-baseline > gpurun_out/bench_r2_n2.json 2> gpurun_out/bench_r2_n2.err; echo "n2 rc=$?"
tail -3 gpurun_out/bench_r2_n2.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_r2_n2.json').read().strip().splitlines()[-1]); print({k: d[k] for k in ['value','n_gpus','scaling','ms_per_step','acceptance_rate']}, d['config']['parallelism'])"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3

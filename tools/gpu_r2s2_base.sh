# round-2 session-2 baseline: suite, bench, per-step probe
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s2_gputest.txt
timeout 900 python bench.py --no-c4 > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err; echo "bench rc=$?"
timeout 600 python tools/step_probe.py --plans 0,3000 --reqs 2 --sizes 16,8 --phases --batch > gpurun_out/s2_probe.txt 2>&1

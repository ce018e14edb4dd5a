# round-2 session-2 evidence, part A: GPU suite, default bench, reference arm, launch list
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -s 2>&1 | grep -E "replay|parity|reconverged|passed|failed|FAILED|Error" | tail -16 > gpurun_out/s2f_gputest.txt
timeout 1800 python bench.py > gpurun_out/s2f_bench.json 2> gpurun_out/s2f_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s2f_bench_ref.json 2> gpurun_out/s2f_bench_ref.err
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/s2f_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c4 > /dev/null 2>&1; echo "launches rc=$?"

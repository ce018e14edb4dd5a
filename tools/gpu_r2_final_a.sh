# round-2 final evidence, part A: GPU suite, default bench, reference arm, launch list, sanitizers
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -s 2>&1 | grep -E "replay|parity|passed|failed|FAILED|Error" | tail -12 > gpurun_out/r2_gputest.txt
timeout 1800 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench_ref.json 2> gpurun_out/r2_bench_ref.err
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c4 > /dev/null 2>&1; echo "launches rc=$?"
mkdir -p gpurun_out/r2_sanitizer
for tool in memcheck racecheck synccheck; do
  for c in c1 c2s cosim p2p; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $c > gpurun_out/r2_sanitizer/${tool}_${c}.txt 2>&1
    echo "=== $tool $c rc=$?"; tail -1 gpurun_out/r2_sanitizer/${tool}_${c}.txt
  done
done

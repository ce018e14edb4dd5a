# round 2, run 2: GPU suite (new parity tests), sanitizers again, short bench
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1800 python -m pytest tests -m gpu -x -q -s -k "bench_parity or pins or c1_traj or speculative" 2>&1 | grep -v "^$" | tail -25
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for tool in memcheck racecheck synccheck; do
  for c in c1 c2s cosim p2p; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $c > gpurun_out/san2_${tool}_${c}.txt 2>&1
    echo "=== $tool $c rc=$?"; tail -2 gpurun_out/san2_${tool}_${c}.txt
  done
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-c4 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_r2a.err

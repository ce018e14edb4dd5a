set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
for tool in memcheck racecheck synccheck; do
  for c in c1 c2s cosim p2p; do
    echo "=== $tool $c"
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $c > gpurun_out/san_${tool}_${c}.txt 2>&1
    echo "rc=$?"; tail -4 gpurun_out/san_${tool}_${c}.txt
  done
done

# validate the ntc reset fix (racecheck f4), full gpu suite, f4 tau-streaming perf
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/r2_sanitizer
for tool in racecheck synccheck memcheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py f4 > gpurun_out/r2_sanitizer/${tool}_f4.txt 2>&1
  echo "=== $tool f4 rc=$?"; grep -E 'SUMMARY' gpurun_out/r2_sanitizer/${tool}_f4.txt | tail -1
done
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
timeout 600 python tools/f4_probe.py 3 2>&1 | tail -12

# round-2 session-2 evidence, part B: ncu --set full captures (library kept for the line mapping), sanitizers
python -c "import __graft_entry__ as g; g.build()"
cp paper_2008_03518_b200/libfmdp.so gpurun_out/s2f_libfmdp.so
N="ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -f"
timeout 900 $N -o gpurun_out/s2f_walk_batch python tools/ncu_batch.py > /dev/null 2>&1; echo "batch rc=$?"
timeout 900 $N -o gpurun_out/s2f_walk_cull8 python tools/ncu_cull.py 8 > /dev/null 2>&1; echo "cull rc=$?"
mkdir -p gpurun_out/s2f_sanitizer
for tool in memcheck racecheck synccheck; do
  for c in c1 c2s reuse; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $c > gpurun_out/s2f_sanitizer/${tool}_${c}.txt 2>&1
    echo "=== $tool $c rc=$?"; tail -1 gpurun_out/s2f_sanitizer/${tool}_${c}.txt
  done
done

# round-2 final evidence, part B: ncu --set full captures (library kept for the line mapping)
python -c "import __graft_entry__ as g; g.build()"
cp paper_2008_03518_b200/libfmdp.so gpurun_out/r2_libfmdp.so
N="ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -f"
timeout 900 $N -o gpurun_out/r2_walk_batch python tools/ncu_batch.py > /dev/null 2>&1; echo "batch rc=$?"
timeout 900 $N -o gpurun_out/r2_walk_cull16 python tools/ncu_cull.py 16 > /dev/null 2>&1; echo "cull rc=$?"
timeout 900 $N -o gpurun_out/r2_walk_f4 python tools/ncu_f4.py > /dev/null 2>&1; echo "f4 rc=$?"
timeout 900 $N -o gpurun_out/r2_walk_c5split python tools/ncu_c5.py > /dev/null 2>&1; echo "c5 rc=$?"
ls -la gpurun_out/
mkdir -p gpurun_out/r2_sanitizer
for tool in memcheck racecheck synccheck; do
  for c in c1 c2s f4 dist; do
    timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize.py $c > gpurun_out/r2_sanitizer/${tool}_${c}.txt 2>&1
    echo "=== $tool $c rc=$?"; tail -1 gpurun_out/r2_sanitizer/${tool}_${c}.txt
  done
done

# session 2: ncu capture of the range-query culled walker (configs[3])
python -c "import __graft_entry__ as g; g.build()"
cp paper_2008_03518_b200/libfmdp.so gpurun_out/s2h_libfmdp.so
python tools/ncu_c4cull.py > gpurun_out/s2h_c4cull.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -f -o gpurun_out/s2h_walk_c4cull python tools/ncu_c4cull.py > /dev/null 2>&1; echo "ncu rc=$?"

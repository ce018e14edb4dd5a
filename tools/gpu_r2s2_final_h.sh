# round-2 closing ncu evidence at HEAD: launch list of the bench command, --set full of the full
# path's batch head and of the culled head-size request (library kept for the line mapping)
set -x
python -c "import __graft_entry__ as g; g.build()"
cp paper_2008_03518_b200/libfmdp.so gpurun_out/r02s3_libfmdp.so
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/r02s3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-c4 > /dev/null 2>&1; echo "launches rc=$?"
N="ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -f"
timeout 900 $N -o gpurun_out/r02s3_walk_batch python tools/ncu_batch.py > /dev/null 2>&1; echo "batch rc=$?"
timeout 900 $N -o gpurun_out/r02s3_walk_cull8 python tools/ncu_cull.py 8 > /dev/null 2>&1; echo "cull rc=$?"

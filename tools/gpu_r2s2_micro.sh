# session 2: instruction-rate and hot-loop microbenchmarks; source-level stall capture of the
# latency-bound step (configs[1] request, f1 culling, one 16-CTA cluster)
set -x
./tools/hotbench/rates > gpurun_out/s2_rates.txt 2>&1
./tools/hotbench/hotbench2 96 200 > gpurun_out/s2_hotbench2.txt 2>&1
./tools/hotbench/hotbench2 24 800 >> gpurun_out/s2_hotbench2.txt 2>&1
cp paper_2008_03518_b200/libfmdp.so gpurun_out/s2_libfmdp_a.so
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -f -o gpurun_out/s2_walk_cull16 python tools/ncu_cull.py 16 > gpurun_out/s2_ncu_cull.log 2>&1; echo "ncu rc=$?"

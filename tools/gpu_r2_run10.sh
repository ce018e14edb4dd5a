python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/r2b_walk_full16 -f python tools/ncu_single.py 16 > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/r2b_walk_cull16 -f python tools/ncu_cull.py 16 > /dev/null 2>&1; echo "ncu cull rc=$?"

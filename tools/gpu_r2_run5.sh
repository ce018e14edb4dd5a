python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -x -q -s 2>&1 | grep -v "^$" | tail -8
timeout 600 python tools/step_probe.py --plans 0,3000 --reqs 2 --sizes 16 --phases 2>&1 | tail -6
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -6
timeout 600 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize.py cosim > gpurun_out/san5_synccheck_cosim.txt 2>&1; echo "synccheck cosim rc=$?"; tail -2 gpurun_out/san5_synccheck_cosim.txt
timeout 900 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize.py c1 c2s cosim p2p > gpurun_out/san5_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/san5_racecheck.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/r2_walk_cull16 -f python tools/ncu_cull.py 16 > /dev/null 2>&1; echo "ncu cull rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -c 1 -o gpurun_out/r2_walk_full16 -f python tools/ncu_single.py 16 > /dev/null 2>&1; echo "ncu full rc=$?"

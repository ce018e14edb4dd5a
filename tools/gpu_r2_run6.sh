python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_bench_parity.py -x -q -s 2>&1 | grep -v "^$" | tail -4
timeout 600 python tools/step_probe.py --plans 0,3000 --reqs 2 --sizes 16 --phases --batch 2>&1 | tail -12
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize.py cosim > gpurun_out/san6_synccheck_cosim.txt 2>&1; echo "synccheck cosim rc=$?"; tail -2 gpurun_out/san6_synccheck_cosim.txt

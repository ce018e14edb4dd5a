python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
timeout 600 python tools/step_probe.py --plans 0,3000 --reqs 2 --sizes 16,2 --phases --batch 2>&1 | tail -20
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 600 compute-sanitizer --tool synccheck --print-limit 5 python tools/sanitize.py cosim > gpurun_out/san4_synccheck_cosim.txt 2>&1; echo "synccheck cosim rc=$?"; tail -2 gpurun_out/san4_synccheck_cosim.txt
timeout 600 compute-sanitizer --tool racecheck --print-limit 5 python tools/sanitize.py c1 c2s > gpurun_out/san4_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -2 gpurun_out/san4_racecheck.txt

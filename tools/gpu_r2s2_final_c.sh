# round-2 session-2 final bench line (code at HEAD), GPU suite
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1800 python bench.py > gpurun_out/s2g_bench.json 2> gpurun_out/s2g_bench.err; echo "bench rc=$?"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/s2g_gputest.txt

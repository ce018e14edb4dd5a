# round-2 session-2 closing bench line at the final code (flags after the post-stage barrier)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 1800 python bench.py > gpurun_out/s2m_bench.json 2> gpurun_out/s2m_bench.err; echo "bench rc=$?"
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/s2m_gputest.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s2m_bench_ref.json 2> gpurun_out/s2m_bench_ref.err; echo "ref rc=$?"

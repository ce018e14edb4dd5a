# round-2 session-2 closing bench line (e2e arm with an untimed first host-buffer call)
set -x
timeout 1800 python bench.py > gpurun_out/s2j_bench.json 2> gpurun_out/s2j_bench.err; echo "bench rc=$?"

free -g | head -2; nproc
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python bench.py --only-c4 --steps 2 --warmup 1 > gpurun_out/bench_r2_c4.json 2> gpurun_out/bench_r2_c4.err; echo "rc=$?"
tail -15 gpurun_out/bench_r2_c4.err

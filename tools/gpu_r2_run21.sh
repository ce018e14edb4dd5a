python -c "import __graft_entry__ as g; g.build()"
timeout 2400 python bench.py --only-c4 --c5-full --steps 2 --warmup 1 > gpurun_out/r2_bench_c4c5.json 2> gpurun_out/r2_bench_c4c5.err; echo "rc=$?"
tail -12 gpurun_out/r2_bench_c4c5.err

python -c "import __graft_entry__ as g; g.build()"
free -g | head -2
FMDP_BIG=1 timeout 2400 python -m pytest tests/test_gpu_big.py -x -q -s 2>&1 | tail -12
free -g | head -2

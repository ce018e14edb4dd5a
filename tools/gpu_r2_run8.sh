python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -2
FMDP_DEBUG=1 timeout 900 python -m pytest tests/test_gpu_accel.py -x -q -s 2>&1 | grep -v "^$" | grep -v "fmdp: walk" | tail -30
FMDP_DEBUG=1 timeout 600 python tools/f4_probe.py 3 2>&1 | grep -v "fmdp: walk" | tail -8

# session 2, A/B 24: mbarrier try_wait suspend hint 1e6 (base) vs 0 (spin) vs 1e5 ns
set -x
export FMDP_AB_EXTRA="s0=FMDP_MBAR_SUSPEND_NS=0;s5=FMDP_MBAR_SUSPEND_NS=100000"
timeout 1200 python tools/ab_old.py run 2 --batch > gpurun_out/s2_ab24.txt 2>&1

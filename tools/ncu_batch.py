"""One configs[1] FCFS batch (as bench.py times it), for ncu capture of a walk launch."""
import sys
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
res = ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False)
print("accepted", sum(r.accepted for r in res), ctx.stats())
ctx.close()

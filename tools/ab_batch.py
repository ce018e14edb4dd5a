"""A/B: culled FCFS batch of configs[1] with a given libfmdp.so, stats + launch log (FMDP_DEBUG)."""
import sys, time
sys.path.insert(0, '.')
import fmdp_synth as fs
import paper_2008_03518_b200.fmdp as F
F.LIB = sys.argv[1]
cull = int(sys.argv[2]) if len(sys.argv) > 2 else 1
sc = fs.config_c2()
ctx = F.FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
ctx.set_launch(cull=cull)
for rep in range(2):
    t = time.time(); res = ctx.schedule_batch(sc.src, sc.dst, sc.t0); dt = time.time() - t
    st = ctx.stats(); ctx.truncate(n0)
    st.pop("phase_cycles", None)
    print(sys.argv[1], f"req/s={len(res)/dt:.0f}", st, flush=True)

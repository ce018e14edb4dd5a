"""configs[1] FCFS batch: per-slice launch log (FMDP_DEBUG) and wall vs device time."""
import os, sys, time
sys.path.insert(0, '.')
os.environ["FMDP_DEBUG"] = "1"
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
cull = int(sys.argv[1]) if len(sys.argv) > 1 else 0
ctx.set_launch(cull=cull)
for rep in range(2):
    t = time.time(); res = ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False); dt = time.time() - t
    st = ctx.stats(); ctx.truncate(n0)
    print(f"REP wall_ms={dt*1e3:.1f} device_ms={st['device_ms']:.1f} rounds={st['rounds']} steps={st['steps']}", flush=True)

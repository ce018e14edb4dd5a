"""Batch throughput vs speculative slice budget (configs[1])."""
import sys, time
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
BUDGETS = {1: (2, 4, 8, 16), 0: ()}
for cull in (1, 0):
    for budget in BUDGETS[cull]:
        ctx.set_launch(cull=cull, step_budget=budget)
        ts = []
        for rep in range(2):
            t = time.time(); res = ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False); ts.append(time.time() - t)
            st = ctx.stats(); ctx.truncate(n0)
        print(f"cull={cull} budget={budget} req/s={len(res)/min(ts):.1f} slices={st['rounds']} rollbacks={st['reruns']} "
              f"steps={st['steps']} dev_ms={st['device_ms']:.1f}", flush=True)
ctx.close()

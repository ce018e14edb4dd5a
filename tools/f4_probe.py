"""SURVEY f4 per-step time: the configs[1] store (3000 plans, 256 terrain wells) with the paper-scale
action space A = 1350 (fmdp_synth.airspace_f4), requests walked one at a time by the wide walker."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmdp_synth as fs  # noqa: E402
from paper_2008_03518_b200.fmdp import FMDP  # noqa: E402

n_req = int(sys.argv[1]) if len(sys.argv) > 1 else 3
sc = fs.config_c2()
air = fs.airspace_f4().replace(lo_m=sc.airspace.lo_m, hi_m=sc.airspace.hi_m, horizon_steps=sc.airspace.horizon_steps,
                               row_capacity=sc.airspace.row_capacity, max_steps=sc.airspace.max_steps)
ctx = FMDP(air, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
for cull in (0, 1):
    ctx.set_launch(cull=cull)
    for i in range(n_req):
        t = time.time()
        r = ctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False)
        st = ctx.stats()
        ctx.truncate(n0)
        print(f"f4 A={ctx.A} cull={cull} req={i} status={r.status} n={r.n_states} dev_ms={st['device_ms']:.1f} "
              f"us/step={st['device_ms'] * 1e3 / max(1, st['steps']):.1f} pairs/s={st['pair_evals'] / st['device_ms'] / 1e9:.3f}e12 "
              f"wall={time.time() - t:.2f}s", flush=True)
ctx.close()

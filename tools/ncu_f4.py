"""One configs[1] request with the A = 1350 action space (wide walker), for ncu capture."""
import sys
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c2()
air = fs.airspace_f4().replace(lo_m=sc.airspace.lo_m, hi_m=sc.airspace.hi_m, horizon_steps=sc.airspace.horizon_steps,
                               row_capacity=sc.airspace.row_capacity, max_steps=sc.airspace.max_steps)
ctx = FMDP(air, sc.terrain)
ctx.add_plans(sc.plans)
r = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
print("status", r.status, "n", r.n_states, ctx.stats()["device_ms"])
ctx.close()

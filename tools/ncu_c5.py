"""configs[4] roofline stress for ncu: 1M accepted plans (64 rows), A = 85, one request on the
§8(a) full path split over clusters of this GPU (fmdp_launch.split, in-kernel exchange) -- one
walk_kernel<5, 2> launch whose clusters all run at once, so ncu can capture it."""
import sys
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP, pack_plans
sc = fs.config_c5(rows=64)
packed = pack_plans(sc.plans)
sc.plans = []
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans_packed(*packed)
ctx.set_launch(split=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
r = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]), want_traj=False)
st = ctx.stats()
print("status", r.status, "n", r.n_states, "clusters", st["split"], "device_ms", st["device_ms"],
      "pairs", st["pair_evals"])
ctx.close()

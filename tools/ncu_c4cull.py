"""One configs[3] request (100k plans) on the culled walker with the range query (ncu capture)."""
import sys
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c4(rows=1200)
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
ctx.set_launch(cull=1)
r = ctx.schedule(sc.src[1], sc.dst[1], int(sc.t0[1]))
print("status", r.status, "n", r.n_states, ctx.stats()["device_ms"], ctx.stats()["cluster_size"])
ctx.close()

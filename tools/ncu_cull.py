"""One configs[1] request with f1 culling at a given cluster size (ncu capture)."""
import sys
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
G = int(sys.argv[1]) if len(sys.argv) > 1 else 2
ctx.set_launch(cluster_size=G, cull=1, split=1)
r = ctx.schedule(sc.src[2], sc.dst[2], int(sc.t0[2]))
print("status", r.status, "n", r.n_states, ctx.stats()["device_ms"])
ctx.close()

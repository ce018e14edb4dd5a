"""Per-step latency of one request vs cluster size G, culled and full, at configs[1] (3000
plans/row) and configs[3] (100k plans/row): the data behind the host cost model (choose_launch)."""
import sys
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP

for name, sc, i in (("c2", fs.config_c2(), 2), ("c4", fs.config_c4(rows=1200), 0)):
    ctx = FMDP(sc.airspace, sc.terrain)
    ctx.add_plans(sc.plans)
    n0 = ctx.num_plans()
    for cull in (1, 0):
        for G in (1, 2, 4, 8, 16):
            ctx.set_launch(cluster_size=G, cull=cull, step_budget=300)
            best = 1e9
            for _ in range(2):
                ctx.schedule_batch(sc.src[i:i + 1], sc.dst[i:i + 1], sc.t0[i:i + 1])
                st = ctx.stats()
                ctx.truncate(n0)
                best = min(best, st["device_ms"] * 1e3 / max(1, st["steps"]))
            print(f"{name} plans/row~{len(sc.plans)} cull={cull} G={G:2d} us/step={best:.2f} "
                  f"cycles/step={best * 1965:.0f}", flush=True)
    ctx.close()

"""Per-step latency and configs[1] batch time vs CTA size (fmdp_launch.threads cap -> plan groups per
warp 4 / 2 / 1), full and culled."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
for threads in (384, 192, 96):
    for cull in (1, 0):
        for G in (16, 8):
            ctx.set_launch(cluster_size=G, cull=cull, split=1, threads=threads)
            best = 1e9
            for _ in range(3):
                ctx.schedule(sc.src[2], sc.dst[2], int(sc.t0[2]), want_traj=False)
                st = ctx.stats(); ctx.truncate(n0)
                best = min(best, st["device_ms"] * 1e3 / st["steps"])
            print(f"threads={threads} cull={cull} G={G} us/step={best:.2f}", flush=True)
        ctx.set_launch(cull=cull, threads=threads)
        ms = []
        for _ in range(2):
            ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False)
            ms.append(ctx.stats()["device_ms"]); ctx.truncate(n0)
        print(f"threads={threads} cull={cull} batch dev_ms={min(ms):.1f}", flush=True)

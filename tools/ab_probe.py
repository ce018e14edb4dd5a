"""A/B probe: per-step latency of alternative builds of libfmdp.so on the same box.
usage: python tools/ab_probe.py LIB.so  (prints culled/full single-request us/step and batch req/s)"""
import sys, time
sys.path.insert(0, '.')
import fmdp_synth as fs
import paper_2008_03518_b200.fmdp as F
F.LIB = sys.argv[1]
sc = fs.config_c2()
ctx = F.FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
out = [sys.argv[1]]
for G, cull in ((16, 1), (2, 1), (16, 0)):
    ctx.set_launch(cluster_size=G, profile=0, cull=cull)  # the bench never profiles
    best = 1e9
    for _ in range(3):
        ctx.schedule(sc.src[2], sc.dst[2], int(sc.t0[2]))
        st = ctx.stats()
        ctx.truncate(n0)
        best = min(best, st["device_ms"] * 1e3 / max(1, st["steps"]))
    out.append(f"G{G}c{cull}={best:.2f}us")
for cull in (1, 0):
    ctx.set_launch(cull=cull)
    best = 1e9
    for _ in range(3):
        t = time.time(); ctx.schedule_batch(sc.src, sc.dst, sc.t0); best = min(best, time.time() - t)
        ctx.truncate(n0)
    out.append(f"batch_c{cull}={len(sc.t0)/best:.0f}req/s")
print(" ".join(out), flush=True)

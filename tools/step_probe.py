"""Per-step latency probe on configs[1] (B200): one request walked alone at cluster sizes 16 / 8 / 2,
full and culled -- unprofiled device time per step, then the per-phase cycle split of the
profiled walk (profile=1 runs the reference instantiation) -- and the configs[1] FCFS batch time.

    python tools/step_probe.py [--plans 0,3000] [--batch] [--reqs 2,5]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import fmdp_synth as fs  # noqa: E402
from paper_2008_03518_b200.fmdp import FMDP  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--plans", default="0,3000")
ap.add_argument("--reqs", default="2")
ap.add_argument("--sizes", default="16,8,2")
ap.add_argument("--batch", action="store_true")
ap.add_argument("--phases", action="store_true")
a = ap.parse_args()

for P in [int(x) for x in a.plans.split(",")]:
    sc = fs.config_c2(n_plans=P) if P else fs.config_c2(n_plans=0)
    ctx = FMDP(sc.airspace, sc.terrain)
    if P:
        ctx.add_plans(sc.plans)
    n0 = ctx.num_plans()
    for i in [int(x) for x in a.reqs.split(",")]:
        for G in [int(x) for x in a.sizes.split(",")]:
            for cull in (0, 1):
                ctx.set_launch(cluster_size=G, cull=cull, split=1)
                best = None
                for _ in range(3):
                    r = ctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False)
                    st = ctx.stats()
                    ctx.truncate(n0)
                    us = st["device_ms"] * 1e3 / max(1, st["steps"])
                    best = us if best is None else min(best, us)
                line = f"plans={P} req={i} G={G:2d} cull={cull} status={r.status} steps={st['steps']} us/step={best:.2f}"
                if a.phases:
                    ctx.set_launch(cluster_size=G, cull=cull, split=1, profile=1)
                    ctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False)
                    st = ctx.stats()
                    ctx.truncate(n0)
                    steps = max(1, st["steps"])
                    ph = {k: round(v / steps) for k, v in st["phase_cycles"].items() if v}
                    line += f" prof_us/step={st['device_ms'] * 1e3 / steps:.2f} cyc/step={sum(ph.values())} {ph}"
                print(line, flush=True)
    if a.batch and P:
        for cull in (0, 1):
            ctx.set_launch(cull=cull)
            for rep in range(3):
                t = time.time()
                res = ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False)
                dt = time.time() - t
                st = ctx.stats()
                ctx.truncate(n0)
                print(f"batch plans={P} cull={cull} dev_ms={st['device_ms']:.1f} wall_ms={dt * 1e3:.1f} "
                      f"acc={sum(r.accepted for r in res)} states={sum(r.n_states for r in res)} "
                      f"steps={st['steps']} rounds={st['rounds']} reruns={st['reruns']}", flush=True)
    ctx.close()

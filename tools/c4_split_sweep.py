"""configs[3] (100k plans, 1200 rows) full-path single-request latency for forced intra-GPU splits:
k clusters x G CTAs (fmdp_set_launch split / cluster_size), against the cost model's choice (split 0).
Device us per step, two requests.

    python tools/c4_split_sweep.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import fmdp_synth as fs  # noqa: E402
from paper_2008_03518_b200.fmdp import FMDP  # noqa: E402

sc = fs.config_c4(rows=1200)
P = len(sc.plans)
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
cases = [(0, 0)] + [(16, k) for k in (7, 8, 9)] + [(8, k) for k in (8, 10, 12, 14, 16)]
for G, k in cases:
    ctx.set_launch(cull=0, split=k, cluster_size=G)
    ms = steps = 0
    st = []
    for rep in range(2):
        ms = steps = 0
        st = []
        for i in (0, 1):
            r = ctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False)
            s = ctx.stats()
            ms += s["device_ms"]
            steps += s["steps"]
            st.append(r.status)
            ctx.truncate(P)
    print(f"G={G:2d} k={k:2d} -> G={s['cluster_size']} k={s['split']} us/step={ms * 1e3 / steps:.2f} status={st}", flush=True)

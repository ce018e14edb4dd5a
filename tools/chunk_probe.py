"""Plans per build pass of the full path (FMDP_TUNE_CHUNK) at large stores: configs[3] (100k plans)
and configs[4] (1M plans, 64 rows, A = 85) single requests split over the co-resident clusters,
and a configs[1] request on one 16-CTA cluster (one pass either way).  Device us per step; each
setting in its own process.

    python tools/chunk_probe.py [chunk,...]
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = r'''
import sys
sys.path.insert(0, %r)
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
def run(sc, reqs, **kw):
    c = FMDP(sc.airspace, sc.terrain)
    c.add_plans(sc.plans)
    P = c.num_plans()
    c.set_launch(cull=0, **kw)
    best = None
    for rep in range(2):
        ms = steps = 0
        st = []
        for i in reqs:
            r = c.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False)
            s = c.stats(); ms += s["device_ms"]; steps += s["steps"]; st.append(r.status)
            c.truncate(P)
        us = ms * 1e3 / steps
        best = us if best is None else min(best, us)
    out = f"{best:.2f} us/step G={s['cluster_size']} k={s['split']} status={st}"
    c.close()
    return out
print("c2 G16:", run(fs.config_c2(), [2], cluster_size=16, split=1), flush=True)
print("c4 split:", run(fs.config_c4(rows=1200), [0, 1]), flush=True)
print("c5 split:", run(fs.config_c5(rows=64), [0]), flush=True)
''' % ROOT
for ch in (sys.argv[1] if len(sys.argv) > 1 else "512,1024").split(","):
    env = dict(os.environ, FMDP_TUNE_CHUNK=ch)
    r = subprocess.run([sys.executable, "-c", PROBE], env=env, capture_output=True, text=True)
    print(f"== chunk {ch}\n{r.stdout.strip()}\n{r.stderr[-400:] if r.returncode else ''}", flush=True)

"""Sweep of the split-slice parameters of the FCFS batch (lanes at the head's cluster size, the
others' cluster size, slice budget) on configs[1], full and culled; device ms per batch.
Each setting in its own process (the overrides are read once per process).

    python tools/sweep_split.py [lanes,..] [Go,..] [budget,..] [Gl,..]
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
sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
out = []
for cull in (0, 1):
    ctx.set_launch(cull=cull, step_budget=int(sys.argv[1]))
    ms = []
    for _ in range(3):
        ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False)
        ms.append(ctx.stats()["device_ms"]); ctx.truncate(n0)
    out.append(f"cull={cull} {min(ms):.1f}")
print(" ".join(out))
''' % ROOT
LANES = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,2,3").split(",")]
GOS = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,8").split(",")]
BUDGETS = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "1,2,4").split(",")]
GLS = [int(x) for x in (sys.argv[4] if len(sys.argv) > 4 else "0").split(",")]  # lane cluster size (0: head's)
for lanes in LANES:
    for go in GOS:
        for budget in BUDGETS:
          for gl in GLS:
            env = dict(os.environ, FMDP_TUNE_LANES=str(lanes), FMDP_TUNE_GO=str(go), FMDP_TUNE_GL=str(gl))
            r = subprocess.run([sys.executable, "-c", PROBE, str(budget)], env=env, capture_output=True, text=True)
            print(f"lanes={lanes} Go={go} Gl={gl} budget={budget}: {r.stdout.strip()} {r.stderr[-200:] if r.returncode else ''}",
                  flush=True)

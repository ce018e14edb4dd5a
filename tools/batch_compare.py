"""Compare the configs[1] FCFS batch results of the libraries in ab/ (statuses, lengths, accepted,
states) -- whether a change altered the workload's trajectories, not only its timing."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = r'''
import sys, hashlib
sys.path.insert(0, %r)
import numpy as np
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
for cull in (0, 1):
    ctx.set_launch(cull=cull)
    res = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
    h = hashlib.sha1(b"".join(r.traj.tobytes() for r in res)).hexdigest()[:12]
    print(f"cull={cull} accepted={sum(r.accepted for r in res)} states={sum(r.n_states for r in res)} "
          f"near={sum(r.n_near_ties for r in res)} exact={sum(r.n_exact for r in res)} traj_sha={h}")
    ctx.truncate(n0)
''' % ROOT
for name in sys.argv[1:]:
    env = dict(os.environ, FMDP_LIB_VARIANT=os.path.join(ROOT, "ab", f"libfmdp_{name}.so"))
    out = subprocess.run([sys.executable, "-c", PROBE], env=env, capture_output=True, text=True)
    print(f"== {name}\n{out.stdout}{out.stderr[-400:] if out.returncode else ''}", flush=True)

"""configs[3] at its defined size (100k plans x 4000 rows): culled single requests and a culled batch
with the SURVEY f1 range query on / off (FMDP_NO_INDEX=1), each in its own process; results (statuses,
states) printed to check they are identical."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROBE = r'''
import sys, time, hashlib
sys.path.insert(0, %r)
import numpy as np
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc4, gen = fs.config_c4_full(n_requests=100)
c = FMDP(sc4.airspace, sc4.terrain)
for t0c, nc, stc in gen.chunks(8192):
    c.add_plans_packed(t0c, nc, stc)
P = c.num_plans()
c.set_launch(cull=1)
t = time.perf_counter(); c.schedule(sc4.src[0], sc4.dst[0], int(sc4.t0[0]), want_traj=False); c.truncate(P)
first = time.perf_counter() - t
ms = steps = 0.0; stat = []
for i in range(12):
    r = c.schedule(sc4.src[i], sc4.dst[i], int(sc4.t0[i]))
    st = c.stats(); c.truncate(P)
    ms += st["device_ms"]; steps += st["steps"]; stat.append((r.status, r.n_states, hashlib.sha1(r.traj.tobytes()).hexdigest()[:8]))
print(f"first_call_s={first:.2f} seq us/step={ms * 1e3 / steps:.2f} ms/req={ms / 12:.2f} split={st['split']} G={st['cluster_size']}")
print("statuses", stat)
reqs = c.make_requests(sc4.src[:100], sc4.dst[:100], sc4.t0[:100])
for rep in range(2):
    res = c.schedule_batch(None, None, None, want_traj=True, reqs=reqs)
    st = c.stats(); c.truncate(P)
    h = hashlib.sha1(b"".join(r.traj.tobytes() for r in res)).hexdigest()[:12]
    print(f"batch dev_ms={st['device_ms']:.1f} rounds={st['rounds']} accepted={sum(r.accepted for r in res)} traj_sha={h}")
''' % ROOT
for name, env in (("index", {}), ("no_index", {"FMDP_NO_INDEX": "1"})):
    out = subprocess.run([sys.executable, "-c", PROBE], env=dict(os.environ, **env), capture_output=True, text=True)
    print(f"== {name}\n{out.stdout}{out.stderr[-600:] if out.returncode else ''}", flush=True)

import sys, time
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
sc = fs.config_c3()
c = FMDP(sc.airspace, sc.terrain)
reqs = c.make_requests(sc.src, sc.dst, sc.t0)
for rep in range(3):
    c.truncate(0)
    t = time.perf_counter()
    res = c.schedule_batch(None, None, None, reqs=reqs, want_traj=False)
    dt = time.perf_counter() - t
    st = c.stats()
    print(f"wall {dt*1e3:.1f} ms device {st['device_ms']:.1f} ms rounds {st['rounds']} reruns {st['reruns']} kernels {st['kernels']}", flush=True)

"""A/B of the FCFS batch head split over clusters (fmdp_launch.split auto) vs one cluster
(split = 1) on the configs[1] batch, full and culled; device ms per batch, identical results."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fmdp_synth as fs  # noqa: E402
from paper_2008_03518_b200.fmdp import FMDP  # noqa: E402

sc = fs.config_c2(seed=2)
ctx = FMDP(sc.airspace, sc.terrain)
ctx.add_plans(sc.plans)
n0 = ctx.num_plans()
reqs = ctx.make_requests(sc.src, sc.dst, sc.t0)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for cull in (0, 1):
    out = {}
    for split in (1, 0, 1, 0):
        ctx.set_launch(cull=cull, split=split)
        best = None
        for _ in range(3):
            res = ctx.schedule_batch(None, None, None, want_traj=False, reqs=reqs)
            st = ctx.stats()
            ctx.truncate(n0)
            flush.zero_()
            torch.cuda.synchronize()
            best = st["device_ms"] if best is None else min(best, st["device_ms"])
        key = [(r.status, r.n_states) for r in res]
        out.setdefault(split, []).append(best)
        out.setdefault(f"res{split}", key)
        print(f"cull={cull} split={split}: {best:.2f} ms (rounds {st['rounds']}, head clusters {st['split']})",
              flush=True)
    print(f"cull={cull} identical={out['res0'] == out['res1']}", flush=True)

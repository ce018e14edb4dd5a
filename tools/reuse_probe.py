"""Find small configs[1]-like batches (culled) in which a rolled-back request re-converges, for
the compute-sanitizer 'reuse' case: prints seed, plans, requests, reconverged, rounds, reruns."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
for seed in range(2, 14):
    for n_plans, n_req in ((300, 16), (600, 24)):
        sc = fs.config_c2(seed=seed, n_plans=n_plans, n_requests=n_req)
        air = sc.airspace.replace(max_steps=600)
        ctx = FMDP(air, sc.terrain, device=0)
        ctx.add_plans(sc.plans)
        ctx.set_launch(cull=1, step_budget=7)
        ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False)
        st = ctx.stats()
        print(f"seed={seed} plans={n_plans} req={n_req} reconverged={st['reconverged']} rounds={st['rounds']} "
              f"reruns={st['reruns']} ms={st['device_ms']:.1f}", flush=True)
        ctx.close()

"""Find small batches (culled, 7-step slices) in which a rolled-back request re-converges, for the
compute-sanitizer 'reuse' case and tests: prints seed, reconverged, rounds, reruns."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP
for seed in range(40, 70):
    sc = fs.random_small(seed, n_plans=60, n_requests=16, half_m=1200.0, n_buildings=20, max_steps=500, t0_max=60)
    ctx = FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    ctx.set_launch(cull=1, step_budget=7)
    ctx.schedule_batch(sc.src, sc.dst, sc.t0, want_traj=False)
    st = ctx.stats()
    print(f"seed={seed} reconverged={st['reconverged']} rounds={st['rounds']} reruns={st['reruns']} "
          f"ms={st['device_ms']:.1f}", flush=True)
    ctx.close()

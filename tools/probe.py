"""Ad-hoc GPU probe: per-step latency, phase breakdown, batch throughput on configs[1]."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import fmdp_synth as fs
from paper_2008_03518_b200.fmdp import FMDP, PHASES

sc = fs.config_c2()
ctx = FMDP(sc.airspace, sc.terrain)
t = time.time(); ctx.add_plans(sc.plans); print('load', round(time.time() - t, 3), flush=True)
n0 = ctx.num_plans()
i = 2
for G in (16, 2, 1):
  for cull in (0, 1):
    ctx.set_launch(cluster_size=G, profile=1, cull=cull)
    t = time.time(); r = ctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i])); dt = time.time() - t
    st = ctx.stats(); ctx.truncate(n0)
    steps = max(1, st['steps'])
    ph = {k: round(v / steps) for k, v in st['phase_cycles'].items()}
    print(f'single G={G} cull={cull} status={r.status} n={r.n_states} wall_ms={dt*1e3:.1f} dev_ms={st["device_ms"]:.2f} '
          f'us/step={st["device_ms"]*1e3/steps:.2f} Gpairs/s={st["pair_evals"]/st["device_ms"]/1e6:.1f} '
          f'cyc/step={sum(ph.values())} {ph}', flush=True)
for cull in (0, 1):
  ctx.set_launch(cull=cull)
  for rep in range(2):
    t = time.time(); res = ctx.schedule_batch(sc.src, sc.dst, sc.t0); dt = time.time() - t
    st = ctx.stats(); ctx.truncate(n0)
    acc = sum(r.accepted for r in res); states = sum(r.n_states for r in res)
    print(f'batch cull={cull} wall={dt:.3f}s req/s={len(res)/dt:.1f} acc={acc} states={states} '
          f'Gpairs/s={st["pair_evals"]/st["device_ms"]/1e6:.1f} {st}', flush=True)
ctx.close()

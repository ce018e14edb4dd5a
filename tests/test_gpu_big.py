"""configs[4] at its defined size (opt-in: FMDP_BIG=1; ~48 GB of device store, a minute to load):
1M accepted plans over 3000 time rows, A = 85 (17 headings x 5 climbs).  Sampled decision steps at
early / middle / late rows checked element by element against the oracle, which evaluates them
from every plan's three rows around the step (all a step reads: R11 forward differences), and the
culled walk bit-identical to the full one."""
import os
import time

import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O
from test_gpu_parity import check_step

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(os.environ.get("FMDP_BIG") != "1", reason="opt-in: FMDP_BIG=1")]


def test_c5_full_size_sampled_steps():
    import torch
    from paper_2008_03518_b200 import fmdp as F
    sc, gen = fs.config_c5_full()
    ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
    t = time.time()
    for t0c, nc, stc in gen.chunks(16384, device=torch.device("cuda", 0)):
        ctx.add_plans_packed(t0c, nc, stc)
    print(f"\nc5 full: {ctx.num_plans()} plans x 3000 rows loaded in {time.time() - t:.1f} s")
    assert ctx.num_plans() == 1_000_000
    O.set_threads(os.cpu_count() or 1)
    try:
        rng = np.random.default_rng(9)
        div = 0
        for K in (20, 1500, 2990):
            orc = O.Oracle(sc.airspace, sc.terrain, gen.window(K, K + 3))
            for j in range(2):
                q = sc.src[j].copy()
                psi = int(rng.integers(0, 1440))
                t = time.time()
                ref = orc.eval_step(q, psi, sc.dst[j], K)
                gpu = ctx.eval_step(q, psi, sc.dst[j], K)
                div += check_step(gpu, ref, f"c5 full K={K}")
                ctx.set_launch(cull=1)
                b = ctx.eval_step(q, psi, sc.dst[j], K)
                ctx.set_launch(cull=0)
                assert (gpu["v"] == b["v"]).all() and gpu["a_star"] == b["a_star"]
                print(f"  K={K} j={j}: a*={gpu['a_star']} oracle {time.time() - t:.1f} s")
        assert div <= 1
    finally:
        O.set_threads(1)
    ctx.close()

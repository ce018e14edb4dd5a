"""The round-2 hand-built pin cases (tests/test_oracle_pins_r2.py) run through the CUDA path:
reading R11 (a stored plan's velocity) through fmdp_add_plan(s) + the walker's well build,
and terrain collision (R16) through fmdp_schedule -- the hand-computed expectations and the
oracle must both hold on the GPU."""
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O
from test_gpu_parity import check_step
from test_oracle_pins_r2 import D1, D2, FLIGHTS, K_TAU, P_FIRST, P_SINGLE, PLAN3, building_raster

pytestmark = pytest.mark.gpu
U = fs.U_PER_M


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


def test_r11_velocities_on_the_gpu(F):
    air = fs.Airspace(lo_m=(-3000.0, -3000.0, 0.0), hi_m=(3000.0, 3000.0, 1500.0), horizon_steps=64, row_capacity=64)
    plans = [(10, PLAN3), (20, P_SINGLE[None].astype(np.int32))]
    orc = O.Oracle(air, None, plans)
    ctx = F.FMDP(air, None, device=0)
    ctx.add_plans(plans)
    p_hand = {10: P_FIRST, 11: P_FIRST + D1, 12: P_FIRST + D1 + D2}
    v_hand = {10: D1, 11: D2, 12: D2}
    cases = []
    for K in (10, 11, 12):
        s1 = p_hand[K] + K_TAU[3] * v_hand[K] + np.array([0, 0, 100 * U])
        cases.append((K, s1))
    cases += [(9, p_hand[10]), (13, p_hand[12]), (20, P_SINGLE + np.array([0, 380 * U, 0])), (21, P_SINGLE)]
    for K, s1 in cases:
        q = (s1 - np.array([320, 0, 0])).astype(np.int32)       # level, psi = 0: s(t=1) = s1
        g = q + np.array([40000, 0, 0], np.int32)
        ref = orc.eval_step(q, 0, g, K)
        gpu = ctx.eval_step(q, 0, g, K)
        check_step(gpu, ref, f"K={K}")
        assert (ref.v_int[13, 0] > 0) == (K in (10, 11, 12, 20))
    ctx.close()


@pytest.mark.parametrize("i", range(len(FLIGHTS)))
def test_terrain_collision_on_the_gpu(F, i):
    src_m, dst_m, status, k = FLIGHTS[i]
    ctx = F.FMDP(fs.Airspace(), building_raster(), device=0)
    r = ctx.schedule(fs.m2u(src_m), fs.m2u(dst_m), 0)
    assert r.status == status and r.n_states == k + 1
    assert r.fail_step == (k if status != O.ACCEPTED else -1)
    ref = O.Oracle(fs.Airspace(), building_raster()).schedule(fs.m2u(src_m), fs.m2u(dst_m), 0, commit=False)
    assert (r.traj == ref.traj).all()
    ctx.close()

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


def test_exact_fallback_overflow_and_terrain_candidate_overflow(F):
    """The two capacity fallbacks of a step (round-1 review: untested): more than AMB_MAX = 64
    (state, tau) minima inside the FP32 band (-> the owner rescans every owned item exactly), and
    more than TC_MAX = 128 terrain wells within reach (-> the whole well list is scanned).  Values,
    V*, a* and separation minima against the oracle element by element."""
    air = fs.Airspace(lo_m=(-3000.0, -3000.0, 0.0), hi_m=(3000.0, 3000.0, 1000.0), horizon_steps=64, row_capacity=256,
                      max_steps=20)
    q = np.array([0, 0, 300 * U], np.int32)
    orc_st, _ = O.Oracle(air).project(q, 0)          # the 270 projected states (oracle geometry, exact)
    R = 450 * U
    # a stationary plan exactly R from 90 distinct projected states (d^2 = R^2: inside the band,
    # only the exact int64 test decides -- out, strict <) -> >= 90 ambiguous items in one step
    plans = []
    for a in range(0, 27, 3):
        for t in range(10):
            s = orc_st[a, t].astype(np.int64)
            p = s + np.array([0, 0, R])              # straight above: |p - s| = R exactly
            plans.append((0, np.repeat(p[None], 30, axis=0).astype(np.int32)))
    # 200 terrain wells hugging the fan (all within reach of every step's states)
    rng = np.random.default_rng(3)
    cen = np.stack([rng.integers(-60 * U, 60 * U, 200), rng.integers(-60 * U, 60 * U, 200),
                    rng.integers(250 * U, 350 * U, 200)], 1).astype(np.int32)
    terr = fs.Terrain(center=cen, radius=np.full(200, 80 * U, np.int32))
    orc = O.Oracle(air, terr, plans)
    ctx = F.FMDP(air, terr, device=0)
    ctx.add_plans(plans)
    g = q + np.array([40000, 0, 0], np.int32)
    for G in (1, 4):  # one CTA owns all 270 states (>= 90 band items > AMB_MAX), then 4 owners
        ctx.set_launch(cluster_size=G)
        for K in (0, 5):
            ref = orc.eval_step(q, 0, g, K)
            gpu = ctx.eval_step(q, 0, g, K)
            check_step(gpu, ref, f"overflow G={G} K={K}")
    ctx.close()

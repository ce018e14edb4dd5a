"""Pins of the Alg 1 endpoint-only valuation (R31):
V*(a) = V(Delta_10(a)), the value of the window's last projected state, instead of Alg 8's
maximum over the window."""
import mpmath as mp
import numpy as np

import fmdp_synth as fs
from oracle import oracle as O

U = fs.U_PER_M


def goal_value(d_m):
    return mp.mpf(200) * mp.mpf("0.999") ** mp.mpf(d_m)


def test_endpoint_equals_window_max_when_the_window_is_one_substep():
    """W = 1: the endpoint is the whole window, so Alg 1 and Alg 8 (V_max <- -inf, R2) must
    produce the same decisions and trajectories -- a reduction to the pinned Alg 8 path."""
    for seed in (3, 4):
        base = dict(n_plans=60, n_requests=2, n_buildings=10, W=1)
        sc8 = fs.random_small(seed, **base)
        sc1 = fs.random_small(seed, valuation=1, **base)
        o8, o1 = O.for_scenario(sc8), O.for_scenario(sc1)
        for i in range(2):
            a = o8.schedule(sc8.src[i], sc8.dst[i], int(sc8.t0[i]), commit=False)
            b = o1.schedule(sc1.src[i], sc1.dst[i], int(sc1.t0[i]), commit=False)
            assert (a.status, a.n_states) == (b.status, b.n_states)
            assert (a.traj == b.traj).all() and (a.astar == b.astar).all()
        for q, psi, g, K in fs.random_states(seed, sc8, 5):
            assert np.array_equal(o8.eval_step(q, psi, g, K).vstar, o1.eval_step(q, psi, g, K).vstar)


def test_endpoint_closed_form_goal_inside_the_window():
    """Goal 30 m straight ahead (inside the 50 m window): Alg 8 takes the closest substep
    (t = 6, d = 0: V* = 200), Alg 1 the endpoint (t = 10, 20 m past the goal:
    V* = 200 * 0.999^20)."""
    air = fs.Airspace()
    q = fs.m2u([0.0, 0.0, 100.0])
    g = fs.m2u([30.0, 0.0, 100.0])
    s8 = O.Oracle(air).eval_step(q, 0, g, 0)
    s1 = O.Oracle(air.replace(valuation=1)).eval_step(q, 0, g, 0)
    level = 13  # turn 0, climb 0 in the default 9 x 3 lattice
    assert abs(s8.vstar[level] - float(goal_value(0))) <= 1e-12 * 200
    assert abs(s1.vstar[level] - float(goal_value(20))) <= 1e-12 * 200
    # the per-(a, t) values are the same in both modes; only V* differs
    assert np.array_equal(s8.v, s1.v)
    assert np.array_equal(s1.vstar, s1.v[:, -1])

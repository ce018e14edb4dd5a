"""Pins of the oracle's acceleration actions (R32: state (q, psi, v), action
(turn h, speed increment acc, climb c) held for W substeps: psi += h, v = clamp(v + acc,
[v_min, v_max]), q += (D(psi, v), c), D(psi, v) = the heading lattice of step length v).  Expected
values are closed forms and the SPEC's step_dynamics examples, computed here by
hand (integer sums, mpmath), never by the oracle."""
import mpmath as mp
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O

mp.mp.dps = 50
U = fs.U_PER_M


def test_f4_action_space_is_1350():
    a = fs.airspace_f4()
    assert a.n_actions == 1350 == 15 * 9 * 10          # Table DS / KI captions
    assert a.climb_units[len(a.climb_units) // 2] == 0 and a.acc_units[len(a.acc_units) // 2] == 0
    assert 0 in a.turn_steps


def _aidx(air, it, ia, ic):
    return (it * len(air.acc_units) + ia) * len(air.climb_units) + ic


def test_spec_step_dynamics_examples():
    air = fs.airspace_f4(W=10)
    o = O.Oracle(air)
    v0 = o.initial_speed()
    assert v0 == 320                                    # 50 m/s * 0.1 s / 2^-6 m
    q = fs.m2u([0, 0, 300])
    st, ps, sp = o.project(q, 0, with_speed=True)
    it0, ia0, ic0 = air.turn_steps.index(0), air.acc_units.index(0), air.climb_units.index(0)
    a0 = _aidx(air, it0, ia0, ic0)
    # all-zero action, heading east, 50 m/s, dt 0.1 -> (5, 0, 300) m
    assert list(st[a0, 0]) == list(fs.m2u([5, 0, 300])) and ps[a0, 0] == 0 and sp[a0, 0] == 320
    # at speed_max a positive acceleration leaves the speed unchanged
    vmax = int(60 * 0.1 * U)
    st, ps, sp = o.project(q, 0, v=vmax, with_speed=True)
    assert (sp[_aidx(air, it0, len(air.acc_units) - 1, ic0)] == vmax).all()
    # pi rad/s for 1 s turns the heading by pi -- 72 lattice steps per substep
    o2 = O.Oracle(fs.airspace_f4(turn_steps=(72,), acc_units=(0,), climb_units=(0,)))
    _, ps2 = o2.project(q, 100)
    assert ps2[0, -1] == (100 + 720) % 1440


@pytest.mark.parametrize("psi,axis,sign", [(0, 0, 1), (360, 1, 1), (720, 0, -1), (1080, 1, -1)])
def test_constant_acceleration_straight_line_closed_form(psi, axis, sign):
    """h = 0, climb 0, speed increment +4 from v0 = 320: v_t = min(320 + 4t, 384) and, on a lattice
    axis (D(psi, v) = +-v exactly), q_t = q + sum_{s<=t} v_s along it; -4 clamps at v_min = 192."""
    air = fs.airspace_f4()
    o = O.Oracle(air)
    q = np.array([1000, -2000, 6400], np.int64)
    it0, ic0 = air.turn_steps.index(0), air.climb_units.index(0)
    for v_start, ia in ((320, 8), (376, 8), (200, 0)):
        st, ps, sp = o.project(q, psi, v=v_start, with_speed=True)
        acc = air.acc_units[ia]
        a = _aidx(air, it0, ia, ic0)
        v = v_start
        pos = q.copy()
        for t in range(1, air.W + 1):
            v = min(max(v + acc, 192), 384)
            pos[axis] += sign * v
            assert sp[a, t - 1] == v and ps[a, t - 1] == psi
            assert (st[a, t - 1] == pos).all()


def test_diagonal_step_is_the_rounded_lattice_vector():
    """psi = 180 (45 deg): D(psi, v) = (rint(v/sqrt 2), rint(v/sqrt 2)) for every speed (mpmath)."""
    o = O.Oracle(fs.airspace_f4())
    air = o.air
    it0, ic0 = air.turn_steps.index(0), air.climb_units.index(0)
    for v in (192, 250, 320, 333, 384):
        st, _, sp = o.project([0, 0, 6400], 180, v=v, with_speed=True)
        a = _aidx(air, it0, air.acc_units.index(0), ic0)
        d = int(mp.nint(mp.mpf(v) / mp.sqrt(2)))
        assert list(st[a, 0, :2]) == [d, d] and sp[a, 0] == v


def test_accelerating_straight_flight_to_the_goal_closed_form():
    """Empty airspace, goal straight ahead at the same altitude 2 km away: V(a, t) = 200 .999^d(t);
    the maximal speed increment straight ahead reaches farthest in every window, so it is a*
    until v_max; then (every increment clamped at v_max) the lowest index among the equal
    straight, level actions -- acc index 4 (0) ... 8 all give v_max.  V* at step 0 and the state
    count are closed forms."""
    air = fs.airspace_f4(max_steps=1000)
    o = O.Oracle(air)
    src, dst = fs.m2u([0, 0, 100]), fs.m2u([2000, 0, 100])
    it0, ic0 = air.turn_steps.index(0), air.climb_units.index(0)
    s = o.eval_step(src, 0, dst, 0, v=320)
    a_max = _aidx(air, it0, 8, ic0)
    reach = sum(min(320 + 4 * t, 384) for t in range(1, 11))
    want = 200 * mp.power(mp.mpf("0.999"), (mp.mpf(128000) - reach) / U)
    assert s.a_star == a_max
    assert abs(s.vstar[a_max] - float(want)) <= 1e-12 * float(want)
    r = o.schedule(src, dst, 0, commit=False)
    # hand-integrated: speeds 324, 328, ... until 384, then 384; capture at the first |x - 2000 m| < 100 m
    x, v, k, xs = 0, 320, 0, [0]
    while abs(128000 - x) >= 100 * U:
        v = min(v + 4, 384)
        x += v
        k += 1
        xs.append(x)
    assert r.status == O.ACCEPTED and r.n_states == k + 1
    assert (r.traj[:, 0] == np.array(xs)).all() and (r.traj[:, 1:] == [0, 100 * U]).all()
    assert list(r.speed[:4]) == [320, 324, 328, 332] and r.speed[-1] == 384
    # once at v_max, every acc >= 0 is the same straight state: the lowest such index (acc = 0) wins
    kk = int(np.argmax(r.speed == 384))
    assert r.astar[kk] == _aidx(air, it0, air.acc_units.index(0), ic0)
    assert (r.astar[:kk] == a_max).all()


def test_replay_checks_the_speed():
    air = fs.airspace_f4(max_steps=300)
    o = O.Oracle(air)
    src, dst = fs.m2u([0, 0, 100]), fs.m2u([1000, 300, 100])
    r = o.schedule(src, dst, 0, commit=False)
    st = o.replay(src, dst, 0, r.traj, r.heading, r.astar, r.status, speed=r.speed)
    assert st.n_fail == 0 and st.n_divergent == 0
    bad = r.speed.copy()
    bad[5] += 4
    st = o.replay(src, dst, 0, r.traj, r.heading, r.astar, r.status, speed=bad)
    assert st.n_fail >= 1 and st.first_fail_step in (4, 5)


def test_accel_mirror_symmetry_and_constant_speed_reduction():
    """Reflecting y mirrors the turn index (acc, climb unchanged) with identical values; and a
    single zero increment reproduces the constant-speed oracle exactly."""
    sc = fs.random_small(61, n_plans=25, n_requests=1, half_m=1200.0)
    air = fs.airspace_f4(turn_steps=(-6, 0, 6), acc_units=(-4, 0, 4), climb_units=(-16, 0, 16),
                         lo_m=sc.airspace.lo_m, hi_m=sc.airspace.hi_m)
    M = np.array([1, -1, 1], np.int32)
    o1 = O.Oracle(air, None, sc.plans)
    o2 = O.Oracle(air, None, [(t0, st * M) for t0, st in sc.plans])
    mirror = np.array([_aidx(air, 2 - a // 9, (a // 3) % 3, a % 3) for a in range(27)])
    for q, psi, g, K in fs.random_states(62, sc, 3):
        for v in (200, 320, 380):
            a = o1.eval_step(q, psi, g, K, v=v)
            b = o2.eval_step(q * M, (-psi) % 1440, g * M, K, v=v)
            assert (a.vstar == b.vstar[mirror]).all()
    const = air.replace(acc_units=(0,), speed_min_mps=0.0, speed_max_mps=0.0)
    c1 = O.Oracle(const, None, sc.plans)
    c0 = O.Oracle(sc.airspace.replace(turn_steps=(-6, 0, 6), climb_units=(-16, 0, 16)), None, sc.plans)
    for q, psi, g, K in fs.random_states(63, sc, 3):
        x, y = c1.eval_step(q, psi, g, K), c0.eval_step(q, psi, g, K)
        assert (x.v == y.v).all() and (x.proj == y.proj).all()

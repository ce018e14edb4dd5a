"""Round-2 pins of the three oracle parts the round-1 review found unpinned (no GPU needed):

1. the near-tie branch of the lockstep replays (``orc_replay``, ``orc_cosim_replay``): a different
   action is accepted only when the oracle's own top-2 gap is below ``near_tie_rel`` x the term
   scale (north-star tolerance rule; R22, R25);
2. reading R11 ("position and the linear velocity"): a stored plan's velocity is
   the forward difference, the last state repeats the previous difference, a single-state plan has
   v = 0, and a plan is absent outside [t0, t0 + n);
3. terrain collision (R16; Sec IV.I P:779 terminal states): a flight into a constructed building on
   an asymmetric raster stops with REJ_TERRAIN at the hand-computed step.

Expected values are computed here by hand (integer arithmetic, mpmath), never by the oracle.
"""
import mpmath as mp
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O

mp.mp.dps = 50
U = fs.U_PER_M


# --------------------------------------------------------------------------- 1. replay near-tie branch
def _straight_prefix(o, src, dst, forced_step, forced_action, n_states):
    """Trajectory prefix built from the oracle's own argmax at every step except one forced
    action; returns (traj, heading, astar)."""
    q = np.array(src, np.int32)
    psi = o.initial_heading(src, dst)
    traj, hd, ast = [q.copy()], [psi], []
    for k in range(n_states - 1):
        s = o.eval_step(q, psi, dst, k)
        a = forced_action if k == forced_step else s.a_star
        ast.append(a)
        q, psi = s.proj[a, 0].copy(), int(s.proj_psi[a, 0])
        traj.append(q.copy())
        hd.append(psi)
    return np.array(traj, np.int32), np.array(hd, np.int32), np.array(ast, np.int32)


def _level_climb_rel_gap(d_m):
    """Closed form (empty airspace, goal straight ahead at the same altitude, distance d_m at the
    step): V*(level) = 200 .999^(d-50) (t = W = 10); V*(climb) = 200 .999^sqrt((d-50)^2 + 2.5^2)
    (t = 10, 16 units = 0.25 m per substep); relative gap to the level value (the term scale)."""
    x = mp.mpf(d_m) - 50
    return 1 - mp.power(mp.mpf("0.999"), mp.sqrt(x * x + mp.mpf("6.25")) - x)


@pytest.mark.parametrize("cosim", [False, True])
def test_replay_near_tie_branch(cosim):
    src, dst = fs.m2u([0, 0, 100]), fs.m2u([2000, 0, 100])
    k5 = 5
    g = float(_level_climb_rel_gap(2000 - 5 * k5))       # 1.6e-6 relative
    assert 1e-6 < g < 2e-6
    for rel, forced, want_div, want_fail in (
            (1e-4, 14, 1, 0),         # climb instead of level: logged near-tie -> divergence
            (2.0 * g, 14, 1, 0),      # just above the gap: still a near-tie
            (0.5 * g, 14, 0, 1),      # just below the gap: a failure (the threshold scales S)
            (1e-4, 0, 0, 1),          # hard left: a clear gap (~2.6e-3 relative) -> failure
    ):
        o = O.Oracle(fs.Airspace(near_tie_rel=rel))
        tr, hd, ast = _straight_prefix(o, src, dst, k5, forced, 30)
        if cosim:
            st = o.cosim_replay([src], [dst], [0], [tr], [hd], [ast], [-1])[0]
        else:
            st = o.replay(src, dst, 0, tr, hd, ast, -1)
        assert (st.n_divergent, st.n_fail) == (want_div, want_fail), (rel, forced)
        assert st.n_steps_checked == 29
        assert st.first_fail_step == (k5 if want_fail else -1)
    # the unperturbed prefix replays clean, and its own log has the level/climb near-tie
    o = O.Oracle(fs.Airspace())
    tr, hd, ast = _straight_prefix(o, src, dst, -1, -1, 30)
    st = o.replay(src, dst, 0, tr, hd, ast, -1)
    assert (st.n_fail, st.n_divergent, st.n_near_ties) == (0, 0, 29) and (ast == 13).all()


def test_replay_rejects_wrong_transition_for_the_logged_action():
    """The logged action must also produce the next state: a trajectory that logs 'climb' but
    moves level fails even though climb vs level is a near-tie."""
    src, dst = fs.m2u([0, 0, 100]), fs.m2u([2000, 0, 100])
    o = O.Oracle(fs.Airspace())
    tr, hd, ast = _straight_prefix(o, src, dst, -1, -1, 12)
    ast = ast.copy()
    ast[3] = 14
    st = o.replay(src, dst, 0, tr, hd, ast, -1)
    assert st.n_fail == 1 and st.first_fail_step == 3 and st.n_divergent == 1


# --------------------------------------------------------------------------- 2. R11 velocities
P_FIRST = np.array([1000, 2000, 6400], np.int64)
D1 = np.array([-300, 250, 12], np.int64)
D2 = np.array([320, -200, 16], np.int64)
PLAN3 = np.stack([P_FIRST, P_FIRST + D1, P_FIRST + D1 + D2]).astype(np.int32)   # t0 = 10: rows 10, 11, 12
P_SINGLE = np.array([5000 * U // 10, 5000 * U // 10, 100 * U], np.int64)       # t0 = 20: row 20 only
K_TAU = (-50, 0, 50, 100, 150)                                                  # tau / dt (R9)
R_TAU_M = (250, 300, 350, 400, 450)                                             # 300 + 10 tau (Table PK)


def _hand_vint(s1, centers):
    """max over wells with (integer) d^2 < R^2 of 1000 * 0.97^(d metres) (Alg 7)."""
    best = mp.mpf(0)
    for c, R in zip(centers, R_TAU_M):
        d2 = int(((np.asarray(s1, np.int64) - c) ** 2).sum())
        if d2 < (R * U) ** 2:
            best = max(best, 1000 * mp.power(mp.mpf("0.97"), mp.sqrt(d2) / U))
    return best


def _one_state_oracle(plans):
    # one action, one substep: the projected state is s1 = q + (320, 0, 0) (psi = 0, level)
    return O.Oracle(fs.Airspace(W=1, turn_steps=(0,), climb_units=(0,)), plans=plans)


def test_r11_forward_difference_last_repeats_single_is_zero():
    o = _one_state_oracle([(10, PLAN3), (20, P_SINGLE[None].astype(np.int32))])
    v_hand = {10: D1, 11: D2, 12: D2}                 # K=12 is the last state: repeats K=11's v
    p_hand = {10: P_FIRST, 11: P_FIRST + D1, 12: P_FIRST + D1 + D2}
    for K in (10, 11, 12):
        pos, vel = o.sample(0, K)
        assert (pos == p_hand[K]).all() and (vel == v_hand[K]).all()
        centers = [p_hand[K] + k * v_hand[K] for k in K_TAU]
        s1 = centers[3] + np.array([0, 0, 100 * U])   # 100 m above the tau = 10 s well
        q = (s1 - np.array([320, 0, 0])).astype(np.int32)
        s = o.eval_step(q, 0, q + np.array([10 ** 6, 0, 0]), K)
        want = _hand_vint(s1, centers)
        assert want > 40                               # the 100 m well wins: 1000 .97^100 = 47.55
        assert abs(s.v_int[0, 0] - float(want)) <= 1e-12 * float(want), K
        # a zero velocity (all wells at p) would leave s1 > 450 m from every well
        assert _hand_vint(s1, [p_hand[K]] * 5) == 0
    for K in (9, 13):                                  # absent outside [t0, t0 + n)
        assert o.sample(0, K) is None
        s1 = p_hand[10] if K == 9 else p_hand[12]
        q = (s1 - np.array([320, 0, 0])).astype(np.int32)
        assert (o.eval_step(q, 0, q + np.array([10 ** 6, 0, 0]), K).v_int == 0).all()
    # single-state plan: v = 0, all five wells at p; 380 m away only R = 400, 450 contain it
    pos, vel = o.sample(1, 20)
    assert (pos == P_SINGLE).all() and (vel == 0).all()
    assert o.sample(1, 19) is None and o.sample(1, 21) is None
    s1 = P_SINGLE + np.array([0, 380 * U, 0])
    q = (s1 - np.array([320, 0, 0])).astype(np.int32)
    s = o.eval_step(q, 0, q + np.array([10 ** 6, 0, 0]), 20)
    want = 1000 * mp.power(mp.mpf("0.97"), 380)
    assert abs(s.v_int[0, 0] - float(want)) <= 1e-12 * float(want)
    assert _hand_vint(s1, [P_SINGLE] * 5) == want


def test_r11_velocity_of_an_accepted_plan_feeds_later_requests():
    """Reading R27 + R11 through the FCFS path: the plan a request stores is its trajectory, and
    the next request sees its last state with the repeated last difference."""
    src, dst = fs.m2u([0, 0, 100]), fs.m2u([2000, 0, 100])
    o = O.Oracle(fs.Airspace())
    r = o.schedule(src, dst, 0, commit=True)
    assert r.status == O.ACCEPTED and r.n_states == 382
    K_last = r.n_states - 1
    pos, vel = o.sample(0, K_last)
    assert (pos == r.traj[-1]).all() and (vel == r.traj[-1] - r.traj[-2]).all() and (vel == [320, 0, 0]).all()


# --------------------------------------------------------------------------- 3. terrain collision
NX, NY, CELL = 40, 20, 10 * U                 # asymmetric raster: 40 x 20 cells of 10 m
X0, Y0 = -200 * U, -100 * U


def building_raster():
    h = np.zeros((NY, NX), np.int32)          # [iy][ix]
    h[5:7, 30:33] = 150 * U                    # building A: ix 30-32, iy 5-6
    h[12:14, 5:7] = 150 * U                    # building B: ix 5-6, iy 12-13
    return fs.Terrain(nx=NX, ny=NY, x0=X0, y0=Y0, cell=CELL, height=h)


# (src m, dst m, expected status, expected fail_step / n_states) -- hand computed:
#   A flies +x at y = -45 m (iy = 5): x_k = 5k m enters ix = 30 (x >= 100 m) at k = 20
#   B flies +y at x = -145 m (ix = 5): y_k = -95 + 5k m enters iy = 12 (y >= 20 m) at k = 23
#   C flies +x at y = -15 m (iy = 8, no building): captured (|500 - 5k| < 100) at k = 81
FLIGHTS = [
    ([0, -45, 100], [500, -45, 100], O.REJ_TERRAIN, 20),
    ([-145, -95, 100], [-145, 150, 100], O.REJ_TERRAIN, 23),
    ([0, -15, 100], [500, -15, 100], O.ACCEPTED, 81),
]


@pytest.mark.parametrize("i", range(len(FLIGHTS)))
def test_terrain_collision_constructed_building(i):
    src_m, dst_m, status, k = FLIGHTS[i]
    o = O.Oracle(fs.Airspace(), building_raster())
    r = o.schedule(fs.m2u(src_m), fs.m2u(dst_m), 0, commit=False)
    assert r.status == status
    assert r.n_states == k + 1
    assert r.fail_step == (k if status != O.ACCEPTED else -1)
    # the flight is straight and level (no wells): state k is the first inside the building
    d = np.array(dst_m) - np.array(src_m)
    step = (320 * np.sign(d[:2])).astype(np.int64)
    assert (r.traj[:, :2] == fs.m2u(src_m)[:2] + np.outer(np.arange(k + 1), step)).all()
    # transposing the raster moves the buildings: the same flight is not stopped at step k
    if status == O.REJ_TERRAIN:
        T = building_raster()
        t2 = fs.Terrain(nx=NY, ny=NX, x0=X0, y0=Y0, cell=CELL, height=np.ascontiguousarray(T.height.T))
        r2 = O.Oracle(fs.Airspace(), t2).schedule(fs.m2u(src_m), fs.m2u(dst_m), 0, commit=False)
        assert not (r2.status == O.REJ_TERRAIN and r2.fail_step == k)


# --------------------------------------------------------------------------- OpenMP timing variant
def test_openmp_variant_identical_to_single_thread():
    """the multi-threaded oracle (host timing of the baseline) computes every
    per-state max over the same wells in the same order -> bit-identical outputs."""
    sc = fs.random_small(17, n_plans=80, n_requests=2, half_m=1200.0, n_buildings=20)
    states = fs.random_states(18, sc, 5)
    outs = []
    try:
        for th in (1, 4):
            O.set_threads(th)
            o = O.for_scenario(sc)
            steps = [o.eval_step(q, psi, g, K) for q, psi, g, K in states]
            r = o.schedule(sc.src[0], sc.dst[0], sc.t0[0], commit=False)
            outs.append((steps, r))
    finally:
        O.set_threads(1)
    for a, b in zip(outs[0][0], outs[1][0]):
        for f in ("v_pos", "v_int", "v_ter", "v_alt", "v", "vstar", "conf_d2"):
            assert (getattr(a, f) == getattr(b, f)).all(), f
        assert a.a_star == b.a_star and a.gap == b.gap
    ra, rb = outs[0][1], outs[1][1]
    assert ra.status == rb.status and (ra.traj == rb.traj).all() and (ra.astar == rb.astar).all()

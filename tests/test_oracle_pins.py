"""Pins of the C oracle against what the paper and mathematics fix (no GPU needed).

Every test here checks the oracle (oracle/fmdp_oracle.c) against something other than
itself: values the paper/SPEC print (tests/golden/spec_values.json), closed forms
recomputed with mpmath, exact lattice symmetries, invariants (translation, mirror,
truncation, determinism), brute force over action sequences on a tiny instance, a
NumPy library-routine special case, and an independent separation validator.
"""
import itertools
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O

mp.mp.dps = 50
GOLD = os.path.join(os.path.dirname(__file__), "golden")
spec = json.load(open(os.path.join(GOLD, "spec_values.json")))
closed = json.load(open(os.path.join(GOLD, "closed_forms.json")))
U = fs.U_PER_M


def mp_goal(d_m):
    return mp.mpf(200) * mp.power(mp.mpf("0.999"), d_m)


def mp_well(d_m, r=1000, g="0.97"):
    return mp.mpf(r) * mp.power(mp.mpf(g), d_m)


def rel(a, b):
    return abs(float(a) - float(b)) / max(abs(float(b)), 1e-300)


@pytest.fixture(scope="module")
def orc():
    return O.Oracle(fs.Airspace())


# --------------------------------------------------------------------------- values
def test_goal_value_vs_mpmath(orc):
    rng = np.random.default_rng(0)
    for d2 in list(rng.integers(0, (20000 * U) ** 2, size=500)) + [0, 1, (1000 * U) ** 2]:
        d_m = mp.sqrt(mp.mpf(int(d2))) / U
        assert rel(orc.goal_value(int(d2)), mp_goal(d_m)) < 1e-12


def test_well_value_vs_mpmath_and_truncation(orc):
    rng = np.random.default_rng(1)
    for R_m in (250, 300, 450):
        R = R_m * U
        for d2 in rng.integers(0, R * R, size=200):
            v = orc.well_value(1000, 0.97, int(d2), R)
            assert rel(v, mp_well(mp.sqrt(mp.mpf(int(d2))) / U)) < 1e-12
        # strict inequality d < R (Alg 7): exactly R -> 0, one unit^2 inside -> the value
        assert orc.well_value(1000, 0.97, R * R, R) == 0.0
        v_in = orc.well_value(1000, 0.97, R * R - 1, R)
        assert v_in > 0 and rel(v_in, mp_well(mp.sqrt(mp.mpf(R * R - 1)) / U)) < 1e-12
        assert orc.well_value(1000, 0.97, R * R + 1, R) == 0.0


def test_spec_worked_values(orc):
    for d_m, want, tol in spec["positive_value"]["cases"]:
        assert abs(orc.goal_value((d_m * U) ** 2) - want) <= tol + 1e-12
    for d_m, want, tol in spec["well_value"]["cases"]:
        assert abs(orc.well_value(1000, 0.97, (d_m * U) ** 2, 300 * U) - want) <= tol + 1e-12
    # monotone decrease
    vals = [orc.goal_value((d * U) ** 2) for d in range(0, 5000, 250)]
    assert all(a > b for a, b in zip(vals, vals[1:]))


def test_hard_deck_spec(orc):
    o = O.Oracle(fs.Airspace(deck_alt_m=1000.0, deck_scale=1000.0))
    for alt_m, want in spec["hard_deck"]["cases"]:
        assert o.deck_penalty(alt_m * U) == pytest.approx(want, abs=1e-12)
    # default deck 30 m: penalty 1000 - z below, 0 at/above
    assert orc.deck_penalty(29 * U) == pytest.approx(971.0)
    assert orc.deck_penalty(30 * U) == 0.0


# --------------------------------------------------------------------------- peaks
def test_peak_construction_spec(orc):
    t = spec["traffic_peaks"]
    p = np.array(t["p_m"]) * U
    v_step = np.array(t["v_mps"]) * 0.1 * U  # per 0.1 s substep
    c, r = orc.build_wells(p, v_step)
    taus = list(fs.Airspace().tau_s)
    for e in t["expect"]:
        i = taus.index(e["tau_s"])
        assert list(c[i]) == [x * U for x in e["center_m"]]
        assert r[i] == e["radius_m"] * U
    c0, r0 = orc.build_wells(p, [0, 0, 0])
    assert (c0 == p).all()
    assert list(r0) == [x * U for x in t["zero_velocity_radii_m"]]
    # 5 wells per intruder (Table PK), radius 300 + 10 t
    assert len(r) == 5 and all(r[i] == (300 + 10 * taus[i]) * U for i in range(5))


def test_table_ds_ki_counts():
    # Table KI P:430 and Table DS P:398 arithmetic, restated for the paper's sample sizes
    assert 5 * 1 * 1350 * 2000 == spec["table_ki_threads"]["expect"]
    assert 5 * 2000 * 6 * 8 == spec["table_ds_pi_bytes"]["expect"]


# --------------------------------------------------------------------------- dynamics
def test_heading_lattice_exact_values_and_symmetry(orc):
    DX, DY = orc.tables()
    HL = 1440
    L = 320  # 50 m/s * 0.1 s / 2^-6 m (5 m per substep)
    assert spec["dynamics_step"]["dx_m"] * U == L
    assert (DX[0], DY[0]) == (L, 0) and (DX[360], DY[360]) == (0, L)
    assert (DX[720], DY[720]) == (-L, 0) and (DX[1080], DY[1080]) == (0, -L)
    assert (DX[180], DY[180]) == (226, 226)          # 320/sqrt(2) = 226.27
    assert (DX[120], DY[120]) == (277, 160)          # 30 deg: 277.128, 160
    for psi in range(HL):
        assert (DX[(psi + 360) % HL], DY[(psi + 360) % HL]) == (-DY[psi], DX[psi])   # +90 deg rotation
        assert (DX[(HL - psi) % HL], DY[(HL - psi) % HL]) == (DX[psi], -DY[psi])   # mirror y
        assert (DX[(360 - psi) % HL], DY[(360 - psi) % HL]) == (DY[psi], DX[psi])   # mirror x=y
        n = math.hypot(DX[psi], DY[psi])
        assert abs(n - L) <= 0.5 * math.sqrt(2) + 1e-9
        ang = math.atan2(DY[psi], DX[psi]) % (2 * math.pi)
        assert abs((ang - 2 * math.pi * psi / HL + math.pi) % (2 * math.pi) - math.pi) < 1.0 / L


def test_projection_closed_form(orc):
    q = np.array([1000, -2000, 6400], np.int32)
    A = fs.Airspace()
    DX, DY = orc.tables()
    for psi in (0, 7, 359, 1000):
        st, ps = orc.project(q, psi)
        for it, h in enumerate(A.turn_steps):
            for ic, c in enumerate(A.climb_units):
                a = it * len(A.climb_units) + ic
                for t in range(1, A.W + 1):
                    assert ps[a, t - 1] == (psi + h * t) % A.HL    # S:171 heading = psi0 + omega t
                    assert st[a, t - 1, 2] == q[2] + c * t
                    if h == 0:                                       # straight: q0 + t*D[psi0]
                        assert st[a, t - 1, 0] == q[0] + t * DX[psi]
                        assert st[a, t - 1, 1] == q[1] + t * DY[psi]


def test_full_circle_closes_exactly():
    # with +8 lattice steps per substep, 180 substeps turn exactly 360 deg; by the exact
    # rotational symmetry of the lattice the displacement sums to zero
    o = O.Oracle(fs.Airspace(W=180, turn_steps=(8,), climb_units=(0,)))
    st, ps = o.project([5, 6, 7], 3)
    assert list(st[0, -1]) == [5, 6, 7] and ps[0, -1] == 3


# --------------------------------------------------------------------------- closed-form trajectories
def test_no_intruder_straight_line():
    cf = closed["no_intruder"]
    o = O.Oracle(fs.Airspace())
    src, dst = fs.m2u(cf["src_m"]), fs.m2u(cf["dst_m"])
    s = o.eval_step(src, 0, dst, 0)
    want_level = mp_goal(mp.mpf(1950))
    want_climb = mp_goal(mp.sqrt(mp.mpf(1950) ** 2 + mp.mpf("2.5") ** 2))
    assert rel(s.vstar[13], want_level) < 1e-12 and abs(float(want_level) - cf["vstar_level_step0"]) < 1e-9
    assert rel(s.vstar[14], want_climb) < 1e-12 and abs(float(want_climb) - cf["vstar_climb_step0"]) < 1e-9
    assert s.a_star == 13 and s.near_tie  # level vs climb gap 1.6e-6 relative (logged near-tie)
    r = o.schedule(src, dst, 0, commit=False)
    assert r.status == O.ACCEPTED and r.n_states == cf["n_states"]
    assert (r.astar == 13).all()
    assert (r.traj[:, 0] == 320 * np.arange(r.n_states)).all() and (r.traj[:, 1:] == [0, 100 * U]).all()


def test_single_intruder_hand_worked():
    cf = closed["single_intruder"]
    src, dst = fs.m2u([0, 0, 100]), fs.m2u([2000, 0, 100])
    plan = np.repeat(fs.m2u(cf["plan_m"])[None, :], 1000, axis=0).astype(np.int32)   # stationary (v = 0)
    o = O.Oracle(fs.Airspace(), plans=[(0, plan)])
    empty = O.Oracle(fs.Airspace()).schedule(src, dst, 0, commit=False)
    r = o.schedule(src, dst, 0, commit=False)
    k1 = cf["first_in_radius_step"]
    assert (r.traj[:k1 + 1] == empty.traj[:k1 + 1]).all() and (r.astar[:k1] == 13).all()
    s = o.eval_step(r.traj[k1], r.heading[k1], dst, k1)
    want_level = mp_goal(mp.mpf(1445)) - mp_well(mp.mpf(445))
    dz = mp.mpf("2.5")
    want_climb = mp_goal(mp.sqrt(mp.mpf(1445) ** 2 + dz ** 2)) - mp_well(mp.sqrt(mp.mpf(445) ** 2 + dz ** 2))
    assert rel(s.vstar[13], want_level) < 1e-12 and abs(float(want_level) - cf["vstar_level_step101"]) < 1e-9
    assert rel(s.vstar[14], want_climb) < 1e-12 and abs(float(want_climb) - cf["vstar_climb_step101"]) < 1e-9
    assert s.vstar[12] == s.vstar[14]            # exact tie: descend / climb symmetric
    # the step before: the wells are exactly on the boundary (d = 450 m, strict <) -> no penalty
    s100 = o.eval_step(r.traj[k1 - 1], r.heading[k1 - 1], dst, k1 - 1)
    assert (s100.v_int == 0).all()
    if r.status == O.ACCEPTED:
        assert r.min_sep_d2 >= (150 * U) ** 2


# --------------------------------------------------------------------------- combine / argmax
def _one_action(**kw):
    return fs.Airspace(W=1, turn_steps=(0,), climb_units=(0,), **kw)


def test_combine_is_pos_minus_max_neg_minus_deck():
    # S:253 structure: V = V+ - max(V-, V^T, V^I) - V_alt (Alg 8); W=1, A=1
    a = _one_action(deck_alt_m=30.0)
    for z_m, deck in ((100, 0.0), (20, 1000.0 - 25)):
        q = fs.m2u([0, 0, z_m])
        s1 = q + np.array([320, 0, 0])
        goal = s1 + fs.m2u([0, 0, 1000]) if z_m > 50 else s1 + fs.m2u([1000, 0, 0])
        terrain = fs.Terrain(center=(s1 + fs.m2u([0, 100, 0]))[None].astype(np.int32),
                             radius=np.array([300 * U], np.int32))
        d_i = 151
        plan = np.repeat((s1 + fs.m2u([0, -d_i, 0]))[None], 5, axis=0).astype(np.int32)
        o = O.Oracle(a, terrain, plans=[(0, plan)])
        if z_m < 50:
            deck = 1000.0 - (z_m)  # projected altitude unchanged (climb 0)
        s = o.eval_step(q, 0, goal, 0)
        vpos = mp_goal(mp.mpf(1000))
        vter = mp_well(mp.mpf(100), g="0.99")
        vint = mp_well(mp.mpf(d_i))
        want = vpos - max(vter, vint) - deck
        assert rel(s.vstar[0], want) < 1e-12
        assert rel(s.v_int[0, 0], vint) < 1e-12 and rel(s.v_ter[0, 0], vter) < 1e-12
    # the SPEC arithmetic itself
    c = spec["combine"]
    assert abs(c["v_pos"] - max(c["v_neg"], c["v_ter"], c["v_int"]) - c["expect"]) < 1e-9


def test_argmax_ties_lowest_index():
    # only mirror-image actions: hard-left / hard-right with the goal straight behind, and
    # climb / descend with the goal at the same altitude, are exact ties (exact lattice
    # symmetry); Alg 9 with the lowest-index rule (R13) must pick index 0
    q = fs.m2u([0, 0, 100])
    o = O.Oracle(fs.Airspace(turn_steps=(-8, 8), climb_units=(0,)))
    s = o.eval_step(q, 0, fs.m2u([-3000, 0, 100]), 0)
    assert s.vstar[0] == s.vstar[1] and s.a_star == 0 and s.a_second == 1 and s.gap == 0.0
    o = O.Oracle(fs.Airspace(turn_steps=(0,), climb_units=(-16, 16)))
    s = o.eval_step(q, 0, fs.m2u([3000, 0, 100]), 0)
    assert s.vstar[0] == s.vstar[1] and s.a_star == 0 and s.near_tie


def test_vmax_init_modes():
    # deep inside a stationary well every V is negative: default (R2) keeps the least-bad,
    # literal Alg 8 (V_max <- 0) clamps every action to 0 and picks index 0
    plan = np.repeat(fs.m2u([40, -30, 100])[None], 10, axis=0).astype(np.int32)   # well ahead-right
    q, goal = fs.m2u([0, 0, 100]), fs.m2u([5000, 0, 100])
    s = O.Oracle(fs.Airspace(), plans=[(0, plan)]).eval_step(q, 0, goal, 0)
    assert (s.vstar < 0).all() and s.a_star // 3 == 8      # hard left (+8) escapes
    lit = O.Oracle(fs.Airspace(vmax_init_zero=1), plans=[(0, plan)]).eval_step(q, 0, goal, 0)
    assert (lit.vstar == 0).all() and lit.a_star == 0


# --------------------------------------------------------------------------- library special case
def test_intruder_term_equals_min_distance_identity():
    """V^I = max_j [d<R]|r|g^d (direct, oracle) equals |r| g^{min in-radius d} computed with a
    NumPy broadcast min over the full distance tensor (the identity the GPU path uses)."""
    sc = fs.random_small(5, n_plans=60, half_m=900.0)
    o = O.for_scenario(sc)
    for q, psi, g, K in fs.random_states(6, sc, 6):
        s = o.eval_step(q, psi, g, K)
        proj = s.proj.reshape(-1, 3).astype(np.int64)
        cen, rad = [], []
        for j in range(o.n_plans()):
            smp = o.sample(j, K)
            if smp is None:
                continue
            c, r = o.build_wells(*smp)
            cen.append(c)
            rad.append(r)
        if not cen:
            continue
        cen = np.concatenate(cen).astype(np.int64)
        rad = np.concatenate(rad).astype(np.int64)
        d2 = ((proj[:, None, :] - cen[None, :, :]) ** 2).sum(-1)
        d2 = np.where(d2 < rad[None, :] ** 2, d2, np.iinfo(np.int64).max)
        m = d2.min(axis=1)
        want = np.where(m < np.iinfo(np.int64).max, 1000.0 * 0.97 ** (np.sqrt(m.astype(np.float64)) / U), 0.0)
        np.testing.assert_allclose(s.v_int.reshape(-1), want, rtol=1e-12, atol=0)


# --------------------------------------------------------------------------- invariants
def _shift_scenario(sc, off):
    off = np.asarray(off, np.int32)
    plans = [(t0, st + off) for t0, st in sc.plans]
    T = sc.terrain
    T2 = fs.Terrain(center=T.center + off if len(T.center) else T.center, radius=T.radius, nx=T.nx, ny=T.ny,
                    x0=T.x0 + int(off[0]), y0=T.y0 + int(off[1]), cell=T.cell, height=T.height + int(off[2]) * (T.height > 0)
                    if T.nx else T.height)
    return plans, T2


def test_truncation_far_plan_changes_nothing():
    sc = fs.random_small(7, n_plans=30, half_m=1200.0)
    o1 = O.for_scenario(sc)
    far = np.repeat(fs.m2u([20000, 20000, 200])[None], 2000, axis=0).astype(np.int32)
    o2 = O.Oracle(sc.airspace, sc.terrain, list(sc.plans) + [(0, far)])
    for q, psi, g, K in fs.random_states(8, sc, 4):
        a, b = o1.eval_step(q, psi, g, K), o2.eval_step(q, psi, g, K)
        assert (a.v == b.v).all() and (a.vstar == b.vstar).all() and a.a_star == b.a_star
    for i in range(min(2, sc.n_requests)):
        r1 = o1.schedule(sc.src[i], sc.dst[i], sc.t0[i], commit=False)
        r2 = o2.schedule(sc.src[i], sc.dst[i], sc.t0[i], commit=False)
        assert r1.status == r2.status and (r1.traj == r2.traj).all()


def test_translation_equivariance():
    sc = fs.random_small(9, n_plans=30, half_m=1200.0)
    air = sc.airspace.replace(deck_alt_m=0.0)   # deck is absolute altitude; disable for a z shift
    off = np.array([64 * 1234 + 17, -64 * 321 - 5, 64 * 7 + 3], np.int32)
    o1 = O.Oracle(air, sc.terrain, sc.plans)
    plans2, T2 = _shift_scenario(sc, off)
    o2 = O.Oracle(air, T2, plans2)
    for i in range(min(2, sc.n_requests)):
        r1 = o1.schedule(sc.src[i], sc.dst[i], sc.t0[i], commit=False)
        r2 = o2.schedule(sc.src[i] + off, sc.dst[i] + off, sc.t0[i], commit=False)
        assert r1.status == r2.status and (r1.astar == r2.astar).all()
        assert (r1.traj + off == r2.traj).all()


def test_mirror_symmetry():
    sc = fs.random_small(11, n_plans=30, half_m=1200.0)
    M = np.array([1, -1, 1], np.int32)
    o1 = O.for_scenario(sc)
    o2 = O.Oracle(sc.airspace, None, [(t0, st * M) for t0, st in sc.plans])
    assert len(sc.terrain.radius) == 0
    A = sc.airspace
    nt, nc = len(A.turn_steps), len(A.climb_units)
    mirror = np.array([(nt - 1 - a // nc) * nc + a % nc for a in range(nt * nc)])
    for q, psi, g, K in fs.random_states(12, sc, 4):
        a = o1.eval_step(q, psi, g, K)
        b = o2.eval_step(q * M, (-psi) % A.HL, g * M, K)
        assert (a.vstar == b.vstar[mirror]).all()
    r1 = o1.schedule(sc.src[0], sc.dst[0], sc.t0[0], commit=False)
    r2 = o2.schedule(sc.src[0] * M, sc.dst[0] * M, sc.t0[0], commit=False)
    assert r1.status == r2.status and (r1.traj * M == r2.traj).all()


# --------------------------------------------------------------------------- brute force (loop conventions)
def test_brute_force_action_sequences():
    """Tiny instance (A = 3 turns x 1 climb, W = 2, 6 steps, 2 plans): among all 3^6 action
    sequences exactly one is greedy-consistent (every action is the argmax at the state the
    previous actions reach, Alg 1), and it is the oracle's trajectory; its conflict
    verdict equals the brute-force min separation over the sequence."""
    air = fs.Airspace(W=2, turn_steps=(-40, 0, 40), climb_units=(0,), max_steps=6, capture_m=1.0,
                      sep_m=150.0)
    src, dst = fs.m2u([0, 0, 100]), fs.m2u([400, 300, 100])
    p1 = np.stack([fs.m2u([60 + 3 * k, 60, 100]) for k in range(20)]).astype(np.int32)
    p2 = np.stack([fs.m2u([200 - 2 * k, -120 + k, 100]) for k in range(20)]).astype(np.int32)
    o = O.Oracle(air, plans=[(0, p1), (2, p2)])
    r = o.schedule(src, dst, 0, commit=False)
    psi0 = o.initial_heading(src, dst)
    consistent = []
    for seq in itertools.product(range(3), repeat=6):
        q, psi, ok = np.array(src, np.int32), psi0, True
        for k, a in enumerate(seq):
            s = o.eval_step(q, psi, dst, k)
            if s.a_star != a:
                ok = False
                break
            q, psi = s.proj[a, 0].copy(), int(s.proj_psi[a, 0])
        if ok:
            consistent.append(seq)
    assert len(consistent) == 1
    assert tuple(r.astar[:len(r.astar)]) == consistent[0][:len(r.astar)]
    # brute-force separation along the oracle trajectory (rows t0+k)
    mins = []
    for k, q in enumerate(r.traj):
        for t0, st in ((0, p1), (2, p2)):
            if 0 <= k - t0 < len(st):
                mins.append(int(((q.astype(np.int64) - st[k - t0]) ** 2).sum()))
    conflict = any(m < (150 * U) ** 2 for m in mins)
    assert (r.status == O.REJ_CONFLICT) == conflict


# --------------------------------------------------------------------------- FCFS invariants
def _validate_store(plans_before, accepted, terrain, sep_u):
    """Independent O(P^2 T) check: every accepted plan keeps >= sep from every earlier plan at
    every shared row and is terrain-clear."""
    earlier = list(plans_before)
    for t0, st in accepted:
        st = st.astype(np.int64)
        assert (st[:, 2] >= 0).all()
        if terrain.nx:
            ix = (st[:, 0] - terrain.x0) // terrain.cell
            iy = (st[:, 1] - terrain.y0) // terrain.cell
            inside = (ix >= 0) & (iy >= 0) & (ix < terrain.nx) & (iy < terrain.ny)
            h = np.where(inside, terrain.height[np.clip(iy, 0, terrain.ny - 1), np.clip(ix, 0, terrain.nx - 1)], 0)
            assert (st[:, 2] >= h).all()
        for u0, su in earlier:
            lo, hi = max(t0, u0), min(t0 + len(st), u0 + len(su))
            if lo >= hi:
                continue
            d = st[lo - t0:hi - t0] - su[lo - u0:hi - u0].astype(np.int64)
            assert ((d ** 2).sum(1) >= sep_u ** 2).all()
        earlier.append((t0, st))


def test_fcfs_batch_separation_invariant_and_determinism():
    sc = fs.random_small(13, n_plans=25, n_requests=8, half_m=1500.0, n_buildings=30, max_steps=500)
    runs = []
    for _ in range(2):
        o = O.for_scenario(sc)
        res = o.schedule_batch(sc.src, sc.dst, sc.t0)
        runs.append(res)
    acc = [(int(sc.t0[i]), r.traj) for i, r in enumerate(runs[0]) if r.status == O.ACCEPTED]
    assert len(acc) >= 1
    _validate_store(sc.plans, acc, sc.terrain, 150 * U)
    for a, b in zip(*runs):
        assert a.status == b.status and (a.traj == b.traj).all()
    # later requests see earlier accepted plans: re-running request i against the initial
    # store alone gives the batch answer whenever no earlier plan was accepted
    o = O.for_scenario(sc)
    r0 = o.schedule(sc.src[0], sc.dst[0], sc.t0[0], commit=False)
    assert (r0.traj == runs[0][0].traj).all()


def test_replay_accepts_own_and_rejects_perturbed():
    sc = fs.random_small(15, n_plans=20, half_m=1200.0)
    o = O.for_scenario(sc)
    r = o.schedule(sc.src[0], sc.dst[0], sc.t0[0], commit=False)
    st = o.replay(sc.src[0], sc.dst[0], sc.t0[0], r.traj, r.heading, r.astar, r.status)
    assert st.n_fail == 0 and st.n_divergent == 0 and st.n_steps_checked == r.n_states - 1
    if r.n_states > 3:
        bad = r.traj.copy()
        bad[2, 0] += 1
        st2 = o.replay(sc.src[0], sc.dst[0], sc.t0[0], bad, r.heading, r.astar, r.status)
        assert st2.n_fail >= 1

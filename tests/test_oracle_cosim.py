"""Pins of the co-simulation oracle (Alg 1, Alg 5 P:598-631,
Table DS P:397 "Determine terminal state N x N").  Each test ties orc_cosim / orc_eval_step_peers
to something other than itself: the single-aircraft scheduler, the (already pinned) intruder
path, a rotation symmetry of the synchronous update, and brute-force separation."""
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O

pytestmark = pytest.mark.filterwarnings("ignore")


def _air_empty(max_steps=500):
    return fs.Airspace(max_steps=max_steps, lo_m=(-2000.0, -2000.0, 0.0), hi_m=(2000.0, 2000.0, 600.0),
                       horizon_steps=2048, row_capacity=64)


def test_cosim_single_aircraft_is_schedule():
    """N = 1: P^- is empty (Table DS, N - 1 = 0), so the batch is one PDFP request."""
    for sc in (fs.config_c1(), fs.random_small(5, n_plans=30, n_requests=2)):
        o = O.for_scenario(sc)
        for i in range(len(sc.t0)):
            c = o.cosim(sc.src[i:i + 1], sc.dst[i:i + 1], sc.t0[i:i + 1])[0]
            s = o.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), commit=False)
            assert (c.status, c.n_states, c.fail_step, c.n_near_ties, c.min_sep_d2) == \
                   (s.status, s.n_states, s.fail_step, s.n_near_ties, s.min_sep_d2)
            assert (c.traj == s.traj).all() and (c.heading == s.heading).all() and (c.astar == s.astar).all()


def test_cosim_disjoint_in_time_is_independent():
    """An aircraft departing after the other has terminated never sees it (present = t0 <= K
    until the terminal state): each result equals its own single request."""
    sc = fs.cosim_ring(3, 2, n_plans=20)
    o = O.for_scenario(sc)
    a = o.schedule(sc.src[0], sc.dst[0], 0, commit=False)
    t0 = np.asarray([0, a.n_states + 5], np.int64)
    c = o.cosim(sc.src, sc.dst, t0)
    b = o.schedule(sc.src[1], sc.dst[1], int(t0[1]), commit=False)
    for ci, si in ((c[0], a), (c[1], b)):
        assert ci.status == si.status and ci.n_states == si.n_states and (ci.traj == si.traj).all()


def test_peer_wells_equal_intruder_wells():
    """Alg 5 and Alg 7 are the same well function (Table PK aircraft row): a peer at (p, v)
    gives V^- equal to the V^I of a stored plan whose row-K sample is (p, v)."""
    sc = fs.random_small(11, n_plans=0, n_requests=1)
    rng = np.random.default_rng(0)
    o_peer = O.for_scenario(sc)
    for q, psi, g, K in fs.random_states(2, sc, 6):
        pp = q[None, :] + rng.integers(-20000, 20000, (3, 3)).astype(np.int32)
        pp[:, 2] = q[2] + rng.integers(-3000, 3000, 3)
        pv = rng.integers(-300, 300, (3, 3)).astype(np.int32)
        o_st = O.Oracle(sc.airspace, sc.terrain)
        for j in range(3):
            o_st.add_plan(K, np.stack([pp[j], pp[j] + pv[j]]))
        assert o_st.sample(0, K)[1].tolist() == pv[0].tolist()
        a = o_peer.eval_step(q, psi, g, K, peer_pos=pp, peer_vel=pv)
        b = o_st.eval_step(q, psi, g, K)
        assert np.array_equal(a.v_neg, b.v_int) and np.array_equal(a.v, b.v)
        assert np.array_equal(a.vstar, b.vstar) and a.a_star == b.a_star
        assert a.v_neg.max() > 0  # the peers are in range of some projected state


def test_cosim_head_on_rotation_symmetry():
    """Two aircraft head-on on the x axis: the batch is invariant under the 180 deg rotation
    about z, which maps one aircraft onto the other.  A synchronous update (Alg 1)
    keeps the two trajectories exact rotations of each other; an update that let the second
    aircraft see the first one's new state would break it.  Alone each would fly straight
    into the other; co-simulated they keep the separation minimum."""
    air = _air_empty()
    L = fs.m2u(1000.0)
    src = np.asarray([[-L, 0, fs.m2u(200.0)], [L, 0, fs.m2u(200.0)]], np.int32)
    dst = np.asarray([[L, 0, fs.m2u(200.0)], [-L, 0, fs.m2u(200.0)]], np.int32)
    o = O.Oracle(air, fs.Terrain())
    DX, DY = o.tables()
    HL = air.HL
    assert (DX[(np.arange(HL) + HL // 2) % HL] == -DX).all() and (DY[(np.arange(HL) + HL // 2) % HL] == -DY).all()
    c = o.cosim(src, dst, np.zeros(2, np.int64))
    a, b = c
    assert a.n_states == b.n_states and a.status == b.status == O.ACCEPTED
    rot = a.traj.copy()
    rot[:, :2] *= -1
    assert (b.traj == rot).all() and ((b.heading - a.heading) % HL == HL // 2).all()
    assert (a.astar == b.astar).all()
    d2 = ((a.traj.astype(np.int64) - b.traj) ** 2).sum(1)
    assert d2.min() >= fs.m2u(air.sep_m) ** 2
    # without the peer wells they would meet head-on
    s0 = o.schedule(src[0], dst[0], 0, commit=False)
    s1 = o.schedule(src[1], dst[1], 0, commit=False)
    m = min(s0.n_states, s1.n_states)
    assert (((s0.traj[:m].astype(np.int64) - s1.traj[:m]) ** 2).sum(1)).min() < fs.m2u(air.sep_m) ** 2


def test_cosim_pair_conflict_rejects_both():
    """The N x N terminal test is symmetric: two aircraft departing from the same point at the
    same clock are both rejected for conflict at step 0."""
    air = _air_empty()
    s = np.asarray([[0, 0, fs.m2u(200.0)]] * 2, np.int32)
    d = np.asarray([[fs.m2u(800.0), 0, fs.m2u(200.0)], [0, fs.m2u(800.0), fs.m2u(200.0)]], np.int32)
    o = O.Oracle(air, fs.Terrain())
    c = o.cosim(s, d, np.zeros(2, np.int64))
    assert [(x.status, x.fail_step, x.n_states, x.min_sep_d2) for x in c] == [(O.REJ_CONFLICT, 0, 1, 0)] * 2
    # one step apart in time: the first has moved 5 m when the second departs -> still a conflict
    c = o.cosim(s, d, np.asarray([0, 1], np.int64))
    assert c[1].status == O.REJ_CONFLICT and c[1].fail_step == 0
    assert c[0].status == O.REJ_CONFLICT and c[0].fail_step == 1


def test_cosim_decisions_reproduced_through_the_store():
    """The peer velocity reading (R28: last displacement; (DX, DY)[psi0], 0 at
    departure) checked through an independent route: every co-simulated decision is
    reproduced by orc_eval_step with the peers entered as two-state stored plans whose
    forward difference is that velocity."""
    sc = fs.cosim_ring(4, 3, n_plans=10, t0_max=20)
    o = O.for_scenario(sc)
    c = o.cosim(sc.src, sc.dst, sc.t0)
    DX, DY = o.tables()
    n = len(c)
    checked = 0
    for i in range(n):
        for k in range(0, c[i].n_states - 1, 7):
            K = int(sc.t0[i]) + k
            o2 = O.for_scenario(sc)
            for j in range(n):
                kj = K - int(sc.t0[j])
                if j == i or kj < 0 or kj >= c[j].n_states:
                    continue
                p = c[j].traj[kj].astype(np.int64)
                v = (p - c[j].traj[kj - 1]) if kj > 0 else np.asarray([DX[c[j].heading[0]], DY[c[j].heading[0]], 0])
                o2.add_plan(K, np.stack([p, p + v]).astype(np.int32))
            r = o2.eval_step(c[i].traj[k], int(c[i].heading[k]), sc.dst[i], K)
            assert r.a_star == c[i].astar[k] or r.near_tie
            checked += 1
    assert checked > 50


def test_cosim_separation_invariant_and_replay():
    """Accepted co-simulated plans keep the separation minimum from each other at every common
    clock and from every stored plan (brute force); the replay accepts the oracle's own batch."""
    sc = fs.cosim_ring(7, 5)
    o = O.for_scenario(sc)
    c = o.cosim(sc.src, sc.dst, sc.t0)
    sep2 = fs.m2u(sc.airspace.sep_m) ** 2
    acc = [i for i, x in enumerate(c) if x.status == O.ACCEPTED]
    assert acc and len(acc) < len(c)
    for a in acc:
        ta = int(sc.t0[a])
        for b in acc:
            if b <= a:
                continue
            tb = int(sc.t0[b])
            lo, hi = max(ta, tb), min(ta + c[a].n_states, tb + c[b].n_states)
            if hi > lo:
                pa = c[a].traj[lo - ta:hi - ta].astype(np.int64)
                pb = c[b].traj[lo - tb:hi - tb].astype(np.int64)
                assert ((pa - pb) ** 2).sum(1).min() >= sep2
        for t0p, st in sc.plans:
            lo, hi = max(ta, t0p), min(ta + c[a].n_states, t0p + len(st))
            if hi > lo:
                d = c[a].traj[lo - ta:hi - ta].astype(np.int64) - st[lo - t0p:hi - t0p]
                assert (d ** 2).sum(1).min() >= sep2
    st = o.cosim_replay(sc.src, sc.dst, sc.t0, [x.traj for x in c], [x.heading for x in c], [x.astar for x in c],
                        [x.status for x in c])
    assert all(s.n_fail == 0 and s.n_divergent == 0 for s in st)
    assert sum(s.n_steps_checked for s in st) == sum(x.n_states - 1 for x in c)
    # a perturbed trajectory is caught
    t = [x.traj.copy() for x in c]
    t[acc[0]][5, 0] += 1
    st = o.cosim_replay(sc.src, sc.dst, sc.t0, t, [x.heading for x in c], [x.astar for x in c], [x.status for x in c])
    assert st[acc[0]].n_fail > 0

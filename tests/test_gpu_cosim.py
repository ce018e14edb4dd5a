"""GPU parity of the co-simulated batch (fmdp_schedule_cosim) against the oracle
(orc_cosim / orc_cosim_replay, pinned in tests/test_oracle_cosim.py).

Protocol (north star tolerances): every GPU trajectory is replayed in lockstep by the oracle
with its peers taken from the GPU's own batch (exact transitions and verdicts; a different a*
only at a logged near-tie); where no step diverged the whole batch equals the oracle's own
co-simulation bit for bit."""
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


def run(F, sc, **launch):
    ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    if launch:
        ctx.set_launch(**launch)
    n0 = ctx.num_plans()
    res = ctx.schedule_cosim(sc.src, sc.dst, sc.t0)
    logs = [ctx.steplog(i) for i in range(len(res))]
    return ctx, n0, res, logs


def check_against_oracle(sc, res, logs):
    orc = O.for_scenario(sc)
    st = orc.cosim_replay(sc.src, sc.dst, sc.t0, [r.traj for r in res], [lg[1] for lg in logs],
                          [lg[0] for lg in logs], [r.status for r in res])
    for i, s in enumerate(st):
        assert s.n_fail == 0, f"aircraft {i}: oracle replay fails at step {s.first_fail_step}"
    assert sum(s.n_steps_checked for s in st) == sum(r.n_states - 1 for r in res)
    ref = orc.cosim(sc.src, sc.dst, sc.t0)
    if sum(s.n_divergent for s in st) == 0:
        for i, (g, o) in enumerate(zip(res, ref)):
            assert (g.status, g.n_states, g.fail_step) == (o.status, o.n_states, o.fail_step), f"aircraft {i}"
            assert (g.traj == o.traj).all() and g.n_near_ties == o.n_near_ties
            assert round((g.min_sep_m / sc.airspace.u_m) ** 2) == o.min_sep_d2
    return ref, st


def test_cosim_single_equals_schedule(F):
    sc = fs.random_small(31, n_plans=60, n_requests=1, n_buildings=10)
    ctx, n0, res, logs = run(F, sc)
    ctx.truncate(n0)
    one = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    assert (res[0].status, res[0].n_states) == (one.status, one.n_states) and (res[0].traj == one.traj).all()
    check_against_oracle(sc, res, logs)
    ctx.close()


@pytest.mark.parametrize("seed,n", [(7, 5), (8, 10), (9, 3)])
def test_cosim_ring_vs_oracle(F, seed, n):
    sc = fs.cosim_ring(seed, n)
    ctx, n0, res, logs = run(F, sc)
    check_against_oracle(sc, res, logs)
    # accepted plans appended in batch order
    acc = [i for i, r in enumerate(res) if r.accepted]
    assert ctx.num_plans() == n0 + len(acc)
    for j, i in enumerate(acc):
        t0, st = ctx.get_plan(n0 + j)
        assert t0 == int(sc.t0[i]) and (st == res[i].traj).all() and res[i].plan_id == n0 + j
    # mutual separation of the accepted plans (brute force)
    sep2 = fs.m2u(sc.airspace.sep_m) ** 2
    for a in acc:
        for b in acc:
            if b <= a:
                continue
            ta, tb = int(sc.t0[a]), int(sc.t0[b])
            lo, hi = max(ta, tb), min(ta + res[a].n_states, tb + res[b].n_states)
            if hi > lo:
                d = res[a].traj[lo - ta:hi - ta].astype(np.int64) - res[b].traj[lo - tb:hi - tb]
                assert (d ** 2).sum(1).min() >= sep2
    ctx.close()


def test_cosim_head_on(F):
    air = fs.Airspace(max_steps=500, lo_m=(-2000.0, -2000.0, 0.0), hi_m=(2000.0, 2000.0, 600.0),
                      horizon_steps=2048, row_capacity=64)
    L = fs.m2u(1000.0)
    z = fs.m2u(200.0)
    sc = fs.Scenario(air, fs.Terrain(), [], np.asarray([[-L, 0, z], [L, 0, z]], np.int32),
                     np.asarray([[L, 0, z], [-L, 0, z]], np.int32), np.zeros(2, np.int64), name="headon")
    ctx, n0, res, logs = run(F, sc)
    assert all(r.accepted for r in res)
    rot = res[0].traj.copy()
    rot[:, :2] *= -1
    assert (res[1].traj == rot).all()
    check_against_oracle(sc, res, logs)
    ctx.close()


def test_cosim_departure_conflict(F):
    air = fs.Airspace(max_steps=300, lo_m=(-2000.0, -2000.0, 0.0), hi_m=(2000.0, 2000.0, 600.0),
                      horizon_steps=2048, row_capacity=64)
    s = np.asarray([[0, 0, fs.m2u(200.0)]] * 2, np.int32)
    d = np.asarray([[fs.m2u(800.0), 0, fs.m2u(200.0)], [0, fs.m2u(800.0), fs.m2u(200.0)]], np.int32)
    for t0, want in (([0, 0], [(1, 0, 1), (1, 0, 1)]), ([0, 1], [(1, 1, 2), (1, 0, 1)])):
        sc = fs.Scenario(air, fs.Terrain(), [], s, d, np.asarray(t0, np.int64))
        ctx, n0, res, logs = run(F, sc)
        assert [(r.status, r.fail_step, r.n_states) for r in res] == want
        assert ctx.num_plans() == n0
        ctx.close()


@pytest.mark.parametrize("G", [1, 4])
def test_cosim_cull_and_cluster_sizes_identical(F, G):
    sc = fs.cosim_ring(12, 20, n_plans=300)
    ctx, n0, res, logs = run(F, sc)
    ctx2, _, res2, _ = run(F, sc, cull=1, cluster_size=G)
    for a, b in zip(res, res2):
        assert (a.status, a.n_states, a.fail_step) == (b.status, b.n_states, b.fail_step) and (a.traj == b.traj).all()
    check_against_oracle(sc, res, logs)
    ctx.close()
    ctx2.close()


def test_cosim_capacity_error(F):
    sc = fs.cosim_ring(1, 2, n_plans=0)
    ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
    m = ctx.cosim_max()
    assert m >= 20
    src = np.repeat(sc.src[:1], m + 1, 0)
    dst = np.repeat(sc.dst[:1], m + 1, 0)
    with pytest.raises(RuntimeError, match="co-resident|capacity"):
        ctx.schedule_cosim(src, dst, np.zeros(m + 1, np.int64))
    ctx.close()

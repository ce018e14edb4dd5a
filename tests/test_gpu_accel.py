"""SURVEY f4 on the GPU: acceleration actions (R32) and the paper's A = 1350 action space
(Table DS / KI captions P:387) through the wide walker (MODE 5: the action space tiled over
the clusters of one launch, the tiles' top-2 exchanged every step on the decision board).

Parity: V(a, t), S, V*(a) within 1e-5 * S of the oracle (north star; R25) at every projected state,
conflict minima bit-exact, a* identical unless a logged near-tie; whole trajectories (positions,
headings, speeds) lockstep-replayed by the oracle; the closed-form accelerating flight of
tests/test_oracle_accel.py reproduced exactly."""
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O
from test_gpu_parity import check_step

pytestmark = pytest.mark.gpu
U = fs.U_PER_M


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


SMALL = dict(turn_steps=(-6, -3, 0, 3, 6), acc_units=(-4, 0, 4), climb_units=(-16, 0, 16))  # 15 paths: tiles 9 + 6


def _scenario(seed, n_plans, f4_kw, **kw):
    sc = fs.random_small(seed, n_plans=n_plans, **kw)
    air = fs.airspace_f4(**f4_kw).replace(lo_m=sc.airspace.lo_m, hi_m=sc.airspace.hi_m,
                                          horizon_steps=sc.airspace.horizon_steps,
                                          row_capacity=sc.airspace.row_capacity, max_steps=sc.airspace.max_steps)
    return fs.Scenario(air, sc.terrain, sc.plans, sc.src, sc.dst, sc.t0, name=sc.name + "f4")


@pytest.mark.parametrize("f4_kw", [SMALL, {}], ids=["45actions_2tiles", "1350actions"])
def test_eval_step_parity(F, f4_kw):
    sc = _scenario(91, 150, f4_kw, half_m=1500.0, n_buildings=20)
    orc = O.for_scenario(sc)
    ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    assert ctx.A == sc.airspace.n_actions
    rng = np.random.default_rng(5)
    div = 0
    for i, (q, psi, g, K) in enumerate(fs.random_states(92, sc, 6)):
        v = int(rng.integers(192, 385))
        ref = orc.eval_step(q, psi, g, K, v=v)
        gpu = ctx.eval_step(q, psi, g, K, speed=v)
        div += check_step(gpu, ref, f"state {i} v={v}")
    assert div <= 1
    ctx.close()


@pytest.mark.parametrize("f4_kw", [SMALL, {}], ids=["45actions_2tiles", "1350actions"])
def test_trajectories_replayed_with_speeds(F, f4_kw):
    sc = _scenario(93, 120, f4_kw, n_requests=3, half_m=1200.0, n_buildings=15, max_steps=400, t0_max=40)
    orc = O.for_scenario(sc)
    ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    res = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
    div = steps = 0
    for i, r in enumerate(res):
        ast, hd, _ = ctx.steplog(i)
        sp = ctx.speeds(i)
        assert len(sp) == r.n_states and sp[0] == 320 and (sp >= 192).all() and (sp <= 384).all()
        st = orc.replay(sc.src[i], sc.dst[i], int(sc.t0[i]), r.traj, hd, ast, r.status, speed=sp)
        assert st.n_fail == 0, f"request {i}: oracle replay fails at step {st.first_fail_step}"
        div += st.n_divergent
        steps += st.n_steps_checked
        if r.status == 0:
            orc.add_plan(int(sc.t0[i]), r.traj)
    print(f"\nf4 replay: {steps} steps, {div} divergent")
    assert steps > 100
    ctx.close()


def test_accelerating_flight_closed_form(F):
    """tests/test_oracle_accel.py's hand-integrated trajectory: maximal acceleration straight to the
    goal until 60 m/s, then cruise; captured within 100 m."""
    air = fs.airspace_f4(max_steps=1000)
    ctx = F.FMDP(air, None, device=0)
    src, dst = fs.m2u([0, 0, 100]), fs.m2u([2000, 0, 100])
    r = ctx.schedule(src, dst, 0)
    x, v, xs, vs = 0, 320, [0], [320]
    while abs(128000 - x) >= 100 * U:
        v = min(v + 4, 384)
        x += v
        xs.append(x)
        vs.append(v)
    assert r.status == 0 and r.n_states == len(xs)
    assert (r.traj[:, 0] == np.array(xs)).all() and (r.traj[:, 1:] == [0, 100 * U]).all()
    assert (ctx.speeds(0) == np.array(vs)).all()
    ctx.close()


def test_wide_rejects_what_it_does_not_support(F):
    ctx = F.FMDP(fs.airspace_f4(max_steps=100), None, device=0)
    with pytest.raises(F.FmdpError, match="acceleration"):
        ctx.schedule_departures(fs.m2u([0, 0, 100]), fs.m2u([500, 0, 100]), 0, [0, 10])
    assert ctx.cosim_max() == 0
    ctx.close()


def test_wide_culled_bit_identical(F):
    """SURVEY f1 culling inside the wide walker: every step and trajectory bit-identical."""
    sc = _scenario(95, 200, {}, n_requests=2, half_m=1500.0, n_buildings=10, max_steps=300, t0_max=30)
    outs = []
    for cull in (0, 1):
        ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
        ctx.add_plans(sc.plans)
        ctx.set_launch(cull=cull)
        steps = [ctx.eval_step(q, psi, g, K, speed=300) for q, psi, g, K in fs.random_states(96, sc, 3)]
        res = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
        outs.append((steps, res, [ctx.speeds(i) for i in range(len(res))]))
        ctx.close()
    for a, b in zip(outs[0][0], outs[1][0]):
        assert (a["v"] == b["v"]).all() and (a["vstar"] == b["vstar"]).all() and a["a_star"] == b["a_star"]
    for x, y in zip(outs[0][1], outs[1][1]):
        assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all()
    for p, q in zip(outs[0][2], outs[1][2]):
        assert (p == q).all()

"""GPU parity: the CUDA path (through the C ABI) against the C oracle, element by element.

Tolerances (north star):
  * per-action / per-state values: |V_gpu - V_orc| <= 1e-5 * S, S = V+ + max(V^T,V^I) + V_alt
  * a*: identical unless the oracle's top-2 gap < 1e-4 * S (logged near-tie)
  * separation minima / conflict verdicts, trajectories, statuses: bit-exact
"""
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O

pytestmark = pytest.mark.gpu

U = fs.U_PER_M


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


def ctx_for(F, sc, plans=True, **launch):
    c = F.FMDP(sc.airspace, sc.terrain, device=0)
    if plans:
        c.add_plans(sc.plans)
    if launch:
        c.set_launch(**launch)
    return c


def check_step(gpu, ref, where=""):
    tol = 1e-5 * np.maximum(ref.scale, 1e-300)
    err = np.abs(gpu["v"] - ref.v)
    assert (err <= tol).all(), f"{where} V(a,t) max rel err {np.max(err / np.maximum(ref.scale, 1e-300)):.3e}"
    np.testing.assert_allclose(gpu["scale"], ref.scale, rtol=1e-5, atol=0)
    vs_tol = 1e-5 * np.maximum(ref.vstar_scale, 1e-300)
    assert (np.abs(gpu["vstar"] - ref.vstar) <= vs_tol).all(), where
    assert (gpu["min_d2"][:-1] == ref.conf_d2).all(), f"{where} separation minima differ"
    sep2 = (150 * U) ** 2
    assert ((ref.conf_d2 < sep2).astype(np.int32) == gpu["conflict"]).all()
    if gpu["a_star"] != ref.a_star:
        assert ref.vstar[ref.a_star] - ref.vstar[gpu["a_star"]] < 1e-4 * ref.vstar_scale[ref.a_star], \
            f"{where} a* differs outside a near-tie"
        return 1
    return 0


@pytest.mark.parametrize("seed", [21, 22, 23])
def test_eval_step_random_small(F, seed):
    sc = fs.random_small(seed, n_plans=300, half_m=1500.0, n_buildings=40)
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    div = 0
    for i, (q, psi, g, K) in enumerate(fs.random_states(seed + 100, sc, 25)):
        div += check_step(ctx.eval_step(q, psi, g, K), orc.eval_step(q, psi, g, K), f"state {i}")
    assert div <= 2
    ctx.close()


def test_eval_step_identical_across_cluster_sizes(F):
    """Several tiles and a ragged tail: 2999 plans split over 1..16 CTAs with 512-plan chunks;
    every reduction is an exact min, so the outputs must be bit-identical."""
    sc = fs.random_small(31, n_plans=2999, half_m=2500.0, rows=600, max_steps=300)
    orc = O.for_scenario(sc)
    states = fs.random_states(32, sc, 6)
    outs = {}
    for G in (1, 2, 4, 8, 16):
        ctx = ctx_for(F, sc, cluster_size=G)
        outs[G] = [ctx.eval_step(q, psi, g, K) for q, psi, g, K in states]
        ctx.close()
    for G in (2, 4, 8, 16):
        for a, b in zip(outs[1], outs[G]):
            assert (a["v"] == b["v"]).all() and (a["min_d2"] == b["min_d2"]).all() and a["a_star"] == b["a_star"]
    for (q, psi, g, K), o in zip(states, outs[8]):
        check_step(o, orc.eval_step(q, psi, g, K))


def _sum_of_squares(n):
    """(a, b, c) with a^2 + b^2 + c^2 = n (brute force, largest a first)."""
    a = int(np.sqrt(n))
    while a > 0:
        r = n - a * a
        b = int(np.sqrt(r))
        while b >= 0:
            c2 = r - b * b
            c = int(round(np.sqrt(c2)))
            if c * c == c2:
                return a, b, c
            b -= 1
            if b < int(np.sqrt(r)) - 64:
                break
        a -= 1
    return None


@pytest.mark.parametrize("delta", [-2, 0, 1])   # R^2-1 = 7 mod 8 is no sum of 3 squares
def test_exact_radius_boundary(F, delta):
    """Well exactly at / one unit^2 inside / outside R for a projected state: the FP32 filter
    lands in its band and the exact fallback must reproduce the oracle's strict d < R."""
    air = fs.Airspace(lo_m=(-3000.0, -3000.0, 0.0), hi_m=(3000.0, 3000.0, 1000.0), horizon_steps=64, row_capacity=64,
                      max_steps=20)
    q = np.array([0, 0, 200 * U], np.int32)
    s = q + np.array([320 * 10, 0, 0])                   # straight-level, t = W
    R = 450 * U
    abc = _sum_of_squares(R * R + delta)
    assert abc is not None
    p = s + np.array(abc)
    plan = np.repeat(p[None], 40, axis=0).astype(np.int32)   # stationary: all 5 wells at p
    sc = fs.Scenario(air, fs.Terrain(), [(0, plan)], q[None], q[None], np.zeros(1, np.int64))
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    goal = q + np.array([3000 * U // 2, 0, 0])
    ref = orc.eval_step(q, 0, goal, 3)
    gpu = ctx.eval_step(q, 0, goal, 3)
    check_step(gpu, ref)
    inside = ref.v_int[13, 9] > 0
    assert inside == (delta < 0)
    ctx.close()


def test_c1_trajectory_lockstep_replay(F):
    sc = fs.config_c1()
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    r = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    ast, hd, _ = ctx.steplog(0)
    st = orc.replay(sc.src[0], sc.dst[0], int(sc.t0[0]), r.traj, hd, ast, r.status)
    assert st.n_fail == 0, f"first failing step {st.first_fail_step}"
    print(f"\nc1 replay: {st.n_steps_checked} steps, {st.n_near_ties} near-ties, {st.n_divergent} divergent")
    ref = orc.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]), commit=False)
    if st.n_divergent == 0:
        assert r.status == ref.status and r.n_states == ref.n_states and (r.traj == ref.traj).all()
        assert r.min_sep_m == pytest.approx(np.sqrt(ref.min_sep_d2) / U, abs=0)
    ctx.close()


def test_no_intruder_closed_form(F):
    sc = fs.Scenario(fs.Airspace(), fs.Terrain(), [], fs.m2u([[0, 0, 100]]).astype(np.int32),
                     fs.m2u([[2000, 0, 100]]).astype(np.int32), np.zeros(1, np.int64))
    ctx = ctx_for(F, sc, plans=False)
    r = ctx.schedule(sc.src[0], sc.dst[0], 0)
    assert r.status == 0 and r.n_states == 382
    assert (r.traj[:, 0] == 320 * np.arange(382)).all()
    ast, _, nt = ctx.steplog(0)
    assert (ast == 13).all() and nt.sum() > 0
    ctx.close()


def _replay_fcfs(sc, results, gpu_ctx):
    """Oracle lockstep replay of every request against the store the GPU had at that
    request (initial plans + earlier GPU-accepted plans, in FCFS order)."""
    orc = O.for_scenario(sc)
    fails = div = steps = 0
    for i, r in enumerate(results):
        ast, hd, _ = gpu_ctx.steplog(i)
        st = orc.replay(sc.src[i], sc.dst[i], int(sc.t0[i]), r.traj, hd, ast, r.status)
        fails += st.n_fail
        div += st.n_divergent
        steps += st.n_steps_checked
        if r.status == 0:
            orc.add_plan(int(sc.t0[i]), r.traj)
    print(f"\nFCFS replay: {steps} steps, {div} divergent, {fails} failing")
    return fails


def test_batch_speculative_equals_sequential_and_oracle(F):
    sc = fs.random_small(41, n_plans=60, n_requests=10, half_m=1200.0, n_buildings=20, max_steps=500, t0_max=60)
    b = ctx_for(F, sc)
    seq = b.schedule_batch(sc.src, sc.dst, sc.t0, sequential=True)
    for budget in (0, 7):  # default slices and tiny slices (many pauses, resumes, rollbacks)
        a = ctx_for(F, sc, step_budget=budget)
        spec = a.schedule_batch(sc.src, sc.dst, sc.t0)
        st = a.stats()
        for x, y in zip(spec, seq):
            assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all()
            assert x.plan_id == y.plan_id and x.min_sep_m == y.min_sep_m and x.n_near_ties == y.n_near_ties
            assert x.n_exact == y.n_exact  # per-step exact counts survive pauses and rollbacks
    assert a.num_plans() == b.num_plans()
    for pid in range(len(sc.plans), a.num_plans()):
        ta, sa = a.get_plan(pid)
        tb, sb = b.get_plan(pid)
        assert ta == tb and (sa == sb).all()
    assert _replay_fcfs(sc, seq, b) == 0
    assert st["rounds"] >= 1
    a.close()
    b.close()


def test_fcfs_separation_invariant(F):
    sc = fs.random_small(43, n_plans=40, n_requests=12, half_m=1200.0, max_steps=500, t0_max=40)
    ctx = ctx_for(F, sc)
    res = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
    acc = [(int(sc.t0[i]), r.traj) for i, r in enumerate(res) if r.accepted]
    earlier = list(sc.plans)
    for t0, st in acc:
        for u0, su in earlier:
            lo, hi = max(t0, u0), min(t0 + len(st), u0 + len(su))
            if lo < hi:
                d = st[lo - t0:hi - t0].astype(np.int64) - su[lo - u0:hi - u0]
                assert ((d ** 2).sum(1) >= (150 * U) ** 2).all()
        earlier.append((t0, st))
    ctx.close()


def test_truncate_restores_store(F):
    sc = fs.random_small(45, n_plans=50, n_requests=4, half_m=1200.0, max_steps=400, t0_max=30)
    ctx = ctx_for(F, sc)
    n0 = ctx.num_plans()
    states = fs.random_states(46, sc, 3)
    before = [ctx.eval_step(q, p, g, K) for q, p, g, K in states]
    first = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
    ctx.truncate(n0)
    assert ctx.num_plans() == n0
    after = [ctx.eval_step(q, p, g, K) for q, p, g, K in states]
    for x, y in zip(before, after):
        assert (x["v"] == y["v"]).all() and (x["min_d2"] == y["min_d2"]).all()
    again = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
    for x, y in zip(first, again):
        assert x.status == y.status and (x.traj == y.traj).all()
    ctx.close()


def test_c2_full_size_sampled_steps(F):
    """BASELINE configs[1] at full size (3000 plans, 256 terrain wells), in the bench's
    launch configuration: sampled decision steps checked element by element."""
    sc = fs.config_c2()
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    rng = np.random.default_rng(7)
    div = 0
    for i in range(6):
        j = int(rng.integers(0, sc.n_requests))
        K = int(sc.t0[j]) + int(rng.integers(0, 300))
        q = sc.src[j].copy()
        q[2] += int(rng.integers(0, 200 * U))
        psi = int(rng.integers(0, 1440))
        div += check_step(ctx.eval_step(q, psi, sc.dst[j], K), orc.eval_step(q, psi, sc.dst[j], K), f"c2 sample {i}")
    assert div <= 1
    ctx.close()


def test_api_errors(F):
    sc = fs.random_small(47, n_plans=5, n_requests=1, half_m=1000.0, max_steps=100)
    ctx = ctx_for(F, sc)
    with pytest.raises(F.FmdpError, match="invalid argument"):
        ctx.schedule(sc.src[0], sc.src[0], 0)
    with pytest.raises(F.FmdpError, match="out of range"):
        ctx.schedule(sc.src[0] + np.array([10 ** 6, 0, 0]), sc.dst[0], 0)
    with pytest.raises(F.FmdpError, match="out of range"):
        ctx.schedule(sc.src[0], sc.dst[0], sc.airspace.horizon_steps)
    bad = np.array([[0, 0, 100], [2000, 0, 100]], np.int32)
    with pytest.raises(F.FmdpError, match="out of range"):
        ctx.add_plan(0, bad)
    n = ctx.num_plans()
    cap = sc.airspace.row_capacity
    flood = [(0, np.zeros((2, 3), np.int32))] * (cap + 1)
    with pytest.raises(F.FmdpError, match="capacity"):
        ctx.add_plans(flood)
    assert ctx.num_plans() == n
    ctx.close()


# ----------------------------------------------------------------------------- f1: exact culling
def test_cull_bit_identical_steps(F):
    """culling plans none of whose wells can reach a projected state changes no
    output bit (truncation), at small sizes and at configs[1] size."""
    for sc, n in ((fs.random_small(51, n_plans=800, half_m=2000.0, n_buildings=30), 12), (fs.config_c2(), 6)):
        states = fs.random_states(52, sc, n)
        outs = []
        for cull in (0, 1):
            ctx = ctx_for(F, sc, cull=cull)
            outs.append([ctx.eval_step(q, psi, g, K) for q, psi, g, K in states])
            st = ctx.stats()
            ctx.close()
        for a, b in zip(*outs):
            assert (a["v"] == b["v"]).all() and (a["vstar"] == b["vstar"]).all()
            assert (a["min_d2"] == b["min_d2"]).all() and a["a_star"] == b["a_star"]


def test_cull_bit_identical_batch(F):
    sc = fs.random_small(53, n_plans=200, n_requests=10, half_m=1500.0, n_buildings=20, max_steps=500, t0_max=60)
    res = []
    for cull in (0, 1):
        ctx = ctx_for(F, sc, cull=cull, step_budget=32)
        res.append(ctx.schedule_batch(sc.src, sc.dst, sc.t0))
        if cull:
            pairs_cull = ctx.stats()["pair_evals"]
        else:
            pairs_full = ctx.stats()["pair_evals"]
        ctx.close()
    for x, y in zip(*res):
        assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all()
        assert x.min_sep_m == y.min_sep_m and x.n_near_ties == y.n_near_ties
    assert pairs_cull < pairs_full


# ----------------------------------------------------------------------------- f3: departure candidates
def test_departure_candidates(F):
    """every candidate equals an isolated fmdp_schedule of that departure against
    the same store; the earliest accepted candidate is the one appended; oracle replay."""
    sc = fs.random_small(81, n_plans=120, n_requests=1, half_m=1500.0, n_buildings=20, max_steps=500, t0_max=10)
    delays = [0, 30, 60, 90, 120, 150, 180, 210]
    ctx = ctx_for(F, sc)
    n0 = ctx.num_plans()
    res, chosen = ctx.schedule_departures(sc.src[0], sc.dst[0], int(sc.t0[0]), delays)
    ref = ctx_for(F, sc)
    orc = O.for_scenario(sc)
    for i, d in enumerate(delays):
        r = ref.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]) + d)
        ref.truncate(n0)
        assert r.status == res[i].status and r.n_states == res[i].n_states and (r.traj == res[i].traj).all()
    acc = [i for i, r in enumerate(res) if r.accepted]
    assert chosen == (min(acc, key=lambda i: delays[i]) if acc else -1)
    assert ctx.num_plans() == n0 + (1 if acc else 0)
    if acc:
        t0, st = ctx.get_plan(n0)
        assert t0 == int(sc.t0[0]) + delays[chosen] and (st == res[chosen].traj).all()
        ast, hd, _ = ctx.steplog(chosen)
        rp = orc.replay(sc.src[0], sc.dst[0], t0, res[chosen].traj, hd, ast, 0)
        assert rp.n_fail == 0
    ctx.close()
    ref.close()


def test_create_errors_are_reported(F):
    """A rejected scenario frees everything it created and reports why (fmdp_last_error(NULL))."""
    with pytest.raises(F.FmdpError, match="u/dt/window"):
        F.FMDP(fs.Airspace(W=0), fs.Terrain(), device=0)
    with pytest.raises(F.FmdpError, match="valuation"):
        F.FMDP(fs.Airspace(valuation=3), fs.Terrain(), device=0)
    for _ in range(3):  # repeated failures leak no streams / events / memory
        with pytest.raises(F.FmdpError):
            F.FMDP(fs.Airspace(sep_m=500.0), fs.Terrain(), device=0)
    ctx = F.FMDP(fs.Airspace(), fs.Terrain(), device=0)
    assert ctx.A == 27
    ctx.close()

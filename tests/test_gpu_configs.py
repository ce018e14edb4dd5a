"""BASELINE.json configs[0], [2], [3], [4] as GPU parity cases (configs[1] is the bench
workload; its sampled steps are in test_gpu_parity.py).  Full-size stores, sampled outputs
checked element by element against the oracle, whole trajectories by lockstep replay where
the oracle finishes in seconds, invariants (FCFS separation, batch == sequential,
culling bit-identical) at full size."""
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O
from test_gpu_parity import check_step, ctx_for, _replay_fcfs

pytestmark = pytest.mark.gpu
U = fs.U_PER_M


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


def _separation_ok(initial, accepted, sep_u=150 * U):
    earlier = list(initial)
    for t0, st in accepted:
        for u0, su in earlier:
            lo, hi = max(t0, u0), min(t0 + len(st), u0 + len(su))
            if lo < hi:
                d = st[lo - t0:hi - t0].astype(np.int64) - su[lo - u0:hi - u0]
                if not ((d ** 2).sum(1) >= sep_u ** 2).all():
                    return False
        earlier.append((t0, st))
    return True


def test_c1_cull_and_clusters_identical(F):
    sc = fs.config_c1()
    base = None
    for G, cull in ((1, 0), (4, 0), (16, 0), (1, 1), (16, 1)):
        ctx = ctx_for(F, sc, cluster_size=G, cull=cull)
        r = ctx.schedule(sc.src[0], sc.dst[0], 0)
        ctx.close()
        if base is None:
            base = r
        assert r.status == base.status and (r.traj == base.traj).all()


def test_c3_prefix_fcfs(F):
    """configs[2] (store grows from 0): the first 60 requests; speculative (full and culled)
    == sequential; oracle lockstep replay of the first 20 in FCFS order; separation invariant."""
    sc = fs.config_c3(n_requests=60)
    seq_ctx = ctx_for(F, sc, plans=False)
    seq = seq_ctx.schedule_batch(sc.src, sc.dst, sc.t0, sequential=True)
    for cull in (0, 1):
        ctx = ctx_for(F, sc, plans=False, cull=cull)
        spec = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
        for x, y in zip(spec, seq):
            assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all()
        ctx.close()
    acc = [(int(sc.t0[i]), r.traj) for i, r in enumerate(seq) if r.accepted]
    assert len(acc) >= 5 and _separation_ok([], acc)
    sub = fs.Scenario(sc.airspace, sc.terrain, [], sc.src[:20], sc.dst[:20], sc.t0[:20])
    assert _replay_fcfs(sub, seq[:20], seq_ctx) == 0
    seq_ctx.close()


@pytest.fixture(scope="module")
def c4():
    return fs.config_c4(rows=1200)


def test_c4_full_size_sampled_steps_and_prefix(F, c4):
    """configs[3]: 100k accepted plans; sampled steps element by element; culling
    bit-identical; a request's first 40 steps lockstep-replayed by the oracle."""
    sc = c4
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    rng = np.random.default_rng(11)
    samples = []
    for i in range(3):
        j = int(rng.integers(0, sc.n_requests))
        q = sc.src[j].copy()
        K = int(rng.integers(0, 800))
        psi = int(rng.integers(0, 1440))
        samples.append((q, psi, sc.dst[j], K))
    div = 0
    full = []
    for q, psi, g, K in samples:
        o = ctx.eval_step(q, psi, g, K)
        full.append(o)
        div += check_step(o, orc.eval_step(q, psi, g, K), "c4")
    assert div <= 1
    ctx.set_launch(cull=1)
    for (q, psi, g, K), a in zip(samples, full):
        b = ctx.eval_step(q, psi, g, K)
        assert (a["v"] == b["v"]).all() and (a["min_d2"] == b["min_d2"]).all() and a["a_star"] == b["a_star"]
    r = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    ast, hd, _ = ctx.steplog(0)
    n = min(41, r.n_states)
    st = orc.replay(sc.src[0], sc.dst[0], int(sc.t0[0]), r.traj[:n], hd[:n], ast[:n - 1],
                    r.status if n == r.n_states else -1)
    assert st.n_fail == 0, st.first_fail_step
    ctx.close()


def test_c5_a85_sampled_step(F):
    """configs[4] action set (17 headings x 5 climbs, A = 85) with 1M accepted plans (64 rows):
    a sampled step element by element; culling bit-identical."""
    sc = fs.config_c5(rows=64)
    assert sc.airspace.n_actions == 85
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    q, g = sc.src[0].copy(), sc.dst[0]
    psi, K = 123, 20
    o = ctx.eval_step(q, psi, g, K)
    assert check_step(o, orc.eval_step(q, psi, g, K), "c5") <= 1
    ctx.set_launch(cull=1)
    b = ctx.eval_step(q, psi, g, K)
    assert (o["v"] == b["v"]).all() and o["a_star"] == b["a_star"]
    ctx.close()


@pytest.mark.parametrize("seed", [61, 62])
def test_a85_random_small(F, seed):
    air = dict(turn_steps=tuple(range(-8, 9)), climb_units=(-32, -16, 0, 16, 32))
    sc = fs.random_small(seed, n_plans=400, half_m=1500.0, n_buildings=30, **air)
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    for q, psi, g, K in fs.random_states(seed, sc, 10):
        check_step(ctx.eval_step(q, psi, g, K), orc.eval_step(q, psi, g, K), "a85")
    r = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    ast, hd, _ = ctx.steplog(0)
    st = orc.replay(sc.src[0], sc.dst[0], int(sc.t0[0]), r.traj, hd, ast, r.status)
    assert st.n_fail == 0
    ctx.close()


@pytest.mark.parametrize("climbs,turns", [
    ((0,), (-8, -4, 0, 4, 8)),                 # C = 1: 512-thread instantiation, level flight only
    ((-16, 8, 16), (-8, -4, 0, 4, 8)),         # C = 3 without a level climb: general hot loop
    ((-24, -16, 0, 16, 24), (-6, 0, 6)),       # C = 5, level climb in the middle
])
def test_action_sets(F, climbs, turns):
    """Hot-loop variants by climb set: every (state, action, t) value, a*, separation minima
    and a whole trajectory against the oracle; culled and G = 4 runs bit-identical."""
    sc = fs.random_small(61, n_plans=250, half_m=1500.0, n_buildings=20, climb_units=climbs, turn_steps=turns)
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    for q, psi, g, K in fs.random_states(62, sc, 8):
        check_step(ctx.eval_step(q, psi, g, K), orc.eval_step(q, psi, g, K), f"climbs {climbs}")
    r = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    ast, hd, _ = ctx.steplog(0)
    st = orc.replay(sc.src[0], sc.dst[0], int(sc.t0[0]), r.traj, hd, ast, r.status)
    assert st.n_fail == 0 and r.n_states > 20
    n0 = ctx.num_plans()
    ctx.truncate(n0 - 1 if r.accepted else n0)
    ctx.set_launch(cull=1, cluster_size=4)
    r2 = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    assert (r2.status, r2.n_states) == (r.status, r.n_states) and (r2.traj == r.traj).all()
    ctx.close()


def test_endpoint_valuation(F):
    """SURVEY f4, Alg 1 endpoint-only valuation (R31): values, V*(a) = V(a, W), a*, separation
    minima and a whole trajectory against the oracle; culled and G = 4 runs bit-identical."""
    sc = fs.random_small(71, n_plans=300, half_m=1500.0, n_buildings=20, valuation=1)
    orc = O.for_scenario(sc)
    ctx = ctx_for(F, sc)
    for q, psi, g, K in fs.random_states(72, sc, 10):
        check_step(ctx.eval_step(q, psi, g, K), orc.eval_step(q, psi, g, K), "endpoint")
    r = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    ast, hd, _ = ctx.steplog(0)
    st = orc.replay(sc.src[0], sc.dst[0], int(sc.t0[0]), r.traj, hd, ast, r.status)
    assert st.n_fail == 0 and r.n_states > 20
    n0 = ctx.num_plans()
    ctx.truncate(n0 - 1 if r.accepted else n0)
    ctx.set_launch(cull=1, cluster_size=4)
    r2 = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    assert (r2.status, r2.n_states) == (r.status, r.n_states) and (r2.traj == r.traj).all()
    ctx.close()

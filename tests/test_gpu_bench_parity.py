"""Parity on the path bench.py times: the configs[1] FCFS batch (100 requests, 3000 plans, 256
terrain wells) in the bench's own launch configuration (speculative slices split into head /
lanes / others, slice budget 2), full and f1-culled.

* The culled batch is bit-identical to the full one (statuses, trajectories, per-step actions,
  headings, near-tie flags and the traced V*(a), S(a) of every step).
* The kernels' own per-step V*(a) (fmdp_set_trace: written by the walker instantiations the bench
  runs, walk_kernel<3,0> / <3,4>) agree with the oracle's V*(a) at the GPU's state element by
  element within 1e-5 * S (north-star tolerance; R25) at every 5th decision step of the
  first four requests.
* The oracle lockstep-replays the first four requests in FCFS order in full, and a 60-state
  prefix of every other request (store = the initial plans + the earlier accepted plans, each of
  them itself replayed): no failing step; divergences (the GPU took the other action of a logged
  near-tie) are counted and reported.
"""
import numpy as np
import pytest

import fmdp_synth as fs
from oracle import oracle as O

pytestmark = pytest.mark.gpu

N_FULL, PREFIX, EVERY = 4, 60, 5


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


@pytest.fixture(scope="module")
def batches(F):
    sc = fs.config_c2()
    out = {}
    for cull in (0, 1):
        ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
        ctx.add_plans(sc.plans)
        ctx.set_launch(cull=cull)  # the bench's launch: defaults (split slices, budget 2)
        ctx.set_trace(N_FULL)
        res = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
        logs = [ctx.steplog(i) for i in range(len(res))]
        traces = [ctx.trace(i) for i in range(N_FULL)]
        st = ctx.stats()
        out[cull] = (res, logs, traces, st)
        ctx.close()
    return sc, out


def test_culled_batch_bit_identical_to_full(batches):
    sc, out = batches
    (ra, la, ta, _), (rb, lb, tb, _) = out[0], out[1]
    for x, y in zip(ra, rb):
        assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all()
        assert x.n_near_ties == y.n_near_ties and x.min_sep_m == y.min_sep_m and x.n_exact == y.n_exact
    for i, (x, y) in enumerate(zip(la, lb)):
        for name, p, q in zip(("astar", "heading", "near_tie"), x, y):
            bad = np.nonzero(p != q)[0]
            assert len(bad) == 0, f"request {i} {name} differs at steps {bad[:8]}: {p[bad[:8]]} vs {q[bad[:8]]}"
    for (va, sa), (vb, sb) in zip(ta, tb):
        assert (va == vb).all() and (sa == sb).all()
    assert out[0][3]["rounds"] > 1  # the speculative slices really ran


def test_bench_batch_oracle_replay_and_traced_values(batches):
    sc, out = batches
    res, logs, traces, _ = out[0]
    orc = O.for_scenario(sc)
    div = near = checked = values = 0
    worst = 0.0
    for i, r in enumerate(res):
        ast, hd, _ = logs[i]
        t0 = int(sc.t0[i])
        if i < N_FULL:
            st = orc.replay(sc.src[i], sc.dst[i], t0, r.traj, hd, ast, r.status)
            vs, sc_ = traces[i]
            assert vs.shape == (r.n_states - 1, orc.A)
            for k in range(0, r.n_states - 1, EVERY):
                ref = orc.eval_step(r.traj[k], int(hd[k]), sc.dst[i], t0 + k)
                err = np.abs(vs[k] - ref.vstar)
                tol = 1e-5 * np.maximum(ref.vstar_scale, 1e-300)
                assert (err <= tol).all(), f"request {i} step {k}: V* rel err {np.max(err / tol) * 1e-5:.2e}"
                np.testing.assert_allclose(sc_[k], ref.vstar_scale, rtol=1e-5, atol=0)
                worst = max(worst, float(np.max(err / np.maximum(ref.vstar_scale, 1e-300))))
                values += orc.A
        else:  # prefix mode: the first PREFIX states (a non-terminal prefix unless the request ended)
            m = min(PREFIX, r.n_states)
            stat = r.status if m == r.n_states else -1
            st = orc.replay(sc.src[i], sc.dst[i], t0, r.traj[:m], hd[:m], ast[:max(0, m - 1)], stat)
        assert st.n_fail == 0, f"request {i}: oracle replay fails at step {st.first_fail_step}"
        div += st.n_divergent
        near += st.n_near_ties
        checked += st.n_steps_checked
        if r.status == 0:
            orc.add_plan(t0, r.traj)
    print(f"\nbench batch parity: {checked} steps replayed, {near} logged near-ties, {div} divergent steps, "
          f"{values} traced V* values, max |V*_gpu - V*_orc| / S = {worst:.2e}")
    assert checked > 5000

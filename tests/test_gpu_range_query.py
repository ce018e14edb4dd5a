"""SURVEY f1 range query: for large rows the culled walker (walk_kernel<C, 6>) stages
only the plans of the 3x3 x-y cells around the ownship (rows sorted by cell on the device) plus the
plans appended since the sort.  Exact like the per-plan cull it replaces: walks and batches must be
bit-identical to the full path (every plan evaluated), and truncating below the sorted plans must
reload the rows so that the smaller store walks exactly like a store built without them."""
import numpy as np
import pytest

import fmdp_synth as fs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


@pytest.fixture(scope="module")
def c4():
    return fs.config_c4(rows=1200)   # 100k plans: mean row >= 10 000 plans -> range query on


def _walks(ctx, sc, idx, cull):
    ctx.set_launch(cull=cull)
    out = []
    for i in idx:
        r = ctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]))
        out.append((r, ctx.steplog(0)))
        ctx.truncate(len(sc.plans))
    return out


def _same(a, b, tag):
    for (x, lx), (y, ly) in zip(a, b):
        assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all(), tag
        assert x.n_exact == y.n_exact and x.n_near_ties == y.n_near_ties and x.min_sep_m == y.min_sep_m, tag
        for u, v in zip(lx, ly):
            assert (u == v).all(), tag


def test_c4_range_query_walks_and_batch_equal_full(F, c4):
    sc = c4
    ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    idx = [0, 1, 2, 3]
    full = _walks(ctx, sc, idx, 0)
    culled = _walks(ctx, sc, idx, 1)    # first culled walk sorts the rows (index build)
    _same(full, culled, "c4 walks")
    st = ctx.stats()
    assert st["split"] <= 1              # the range query walks on one cluster
    # FCFS batch with commits (appended plans past the sorted regions) == the sequential full loop
    ctx.set_launch(cull=1)
    spec = ctx.schedule_batch(sc.src[:8], sc.dst[:8], sc.t0[:8])
    ctx.truncate(len(sc.plans))
    ctx.set_launch(cull=0)
    seq = ctx.schedule_batch(sc.src[:8], sc.dst[:8], sc.t0[:8], sequential=True)
    for x, y in zip(spec, seq):
        assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all()
        assert x.plan_id == y.plan_id and x.n_exact == y.n_exact
    ctx.close()


def test_truncate_below_sorted_plans_reloads(F, c4):
    """Truncating into the sorted regions reloads the kept plans: the store then walks exactly like
    one that only ever held them (full and culled)."""
    sc = c4
    keep = 60_000
    a = F.FMDP(sc.airspace, sc.terrain, device=0)
    a.add_plans(sc.plans)
    a.set_launch(cull=1)
    a.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))  # builds the index over all 100k plans
    a.truncate(keep)
    assert a.num_plans() == keep
    b = F.FMDP(sc.airspace, sc.terrain, device=0)
    b.add_plans(sc.plans[:keep])
    sub = fs.Scenario(sc.airspace, sc.terrain, sc.plans[:keep], sc.src, sc.dst, sc.t0)
    for cull in (1, 0):
        ra = _walks(a, sub, [1, 2], cull)
        rb = _walks(b, sub, [1, 2], cull)
        _same(ra, rb, f"truncated cull={cull}")
    for pid in (0, keep // 2, keep - 1):
        ta, sa = a.get_plan(pid)
        tb, sb = b.get_plan(pid)
        assert ta == tb and (sa == sb).all()
    a.close()
    b.close()


def test_c5_range_query_walk_equals_full(F):
    """configs[4] action set (A = 85, C = 5 instantiation) over 1M plans (64 rows)."""
    sc = fs.config_c5(rows=64)
    ctx = F.FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    full = _walks(ctx, sc, [0], 0)
    culled = _walks(ctx, sc, [0], 1)
    _same(full, culled, "c5")
    ctx.close()

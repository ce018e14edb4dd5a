"""Request-sharded FCFS batch (fmdp_schedule_batch_dist, SURVEY §8(e) second partitioning): ranks as
contexts of one process on this GPU, each on its own thread, exchanging through an in-process
all-gather (the protocol the NCCL / gloo ranks use; tests/test_dist_gloo.py covers allgather_torch).
Every rank's results must equal the one-context speculative batch and the sequential loop, bit for
bit, and the stores must end identical."""
import threading

import numpy as np
import pytest

import fmdp_synth as fs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def F():
    from paper_2008_03518_b200 import fmdp
    return fmdp


class LocalGather:
    """All-gather among `world` threads of this process."""

    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world)
        self.slots = [None] * world

    def fn(self, rank):
        def f(block):
            self.slots[rank] = block
            self.bar.wait()
            out = list(self.slots)
            self.bar.wait()
            return out
        return f


@pytest.mark.parametrize("world,cull", [(2, 0), (3, 1)])
def test_request_sharded_batch_equals_one_gpu(F, world, cull):
    sc = fs.random_small(71, n_plans=80, n_requests=12, half_m=1200.0, n_buildings=20, max_steps=500, t0_max=60)
    ref = F.FMDP(sc.airspace, sc.terrain, device=0)
    ref.add_plans(sc.plans)
    ref.set_launch(cull=cull, step_budget=7)
    want = ref.schedule_batch(sc.src, sc.dst, sc.t0)
    ctxs = []
    for _ in range(world):
        c = F.FMDP(sc.airspace, sc.terrain, device=0)
        c.add_plans(sc.plans)
        c.set_launch(cull=cull, step_budget=7)
        ctxs.append(c)
    lg = LocalGather(world)
    out, errs = [None] * world, []

    def run(r):
        try:
            out[r] = ctxs[r].schedule_batch_dist(sc.src, sc.dst, sc.t0, lg.fn(r), r, world)
        except Exception as e:  # noqa: BLE001
            errs.append(e)
            lg.bar.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for r in range(world):
        for x, y in zip(out[r], want):
            assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all()
            assert x.plan_id == y.plan_id and x.n_near_ties == y.n_near_ties and x.min_sep_m == y.min_sep_m
        assert ctxs[r].num_plans() == ref.num_plans()
        for pid in range(len(sc.plans), ref.num_plans()):
            ta, sa = ctxs[r].get_plan(pid)
            tb, sb = ref.get_plan(pid)
            assert ta == tb and (sa == sb).all()
        for i in range(len(want)):  # step logs of every request on every rank
            a, b = ctxs[r].steplog(i), ref.steplog(i)
            assert all((p == q).all() for p, q in zip(a, b))
    for c in ctxs + [ref]:
        c.close()

"""compute-sanitizer driver: small runs of every walker instantiation whose
protocol relies on mbarriers / DSMEM st.async / cross-cluster words, meant to run as

    compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize.py CASE

CASE: c1 (configs[0]: one request + eval_step, clusters 1 and 4), c2s (configs[1] city with 300
plans, a 4-request FCFS batch full and culled, speculative slices), reuse (a compact 16-request
culled batch whose rolled-back re-walks re-converge), cosim (a 3-aircraft ring),
p2p (two exchange contexts in one process, a split request over 2 clusters).  Each case checks
its result against a plain sequential run of the same context, so a race that changes an
answer also fails the case, not only the tool.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import fmdp_synth as fs  # noqa: E402
from paper_2008_03518_b200.fmdp import FMDP, p2p_connect_local  # noqa: E402


def _same(a, b):
    return a.status == b.status and a.n_states == b.n_states and (a.traj == b.traj).all()


def case_c1():
    sc = fs.config_c1()
    for G in (1, 4):
        ctx = FMDP(sc.airspace, sc.terrain, device=0, torch_alloc=False)
        ctx.add_plans(sc.plans)
        ctx.set_launch(cluster_size=G)
        r = ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
        e = ctx.eval_step(sc.src[0], 0, sc.dst[0], 0)
        print(f"c1 G={G}: status={r.status} n={r.n_states} a*={e['a_star']}")
        ctx.close()


def case_c2s():
    sc = fs.config_c2(n_plans=300, n_requests=4)
    air = sc.airspace.replace(max_steps=120)
    out = {}
    for cull in (0, 1):
        for seq in (True, False):
            ctx = FMDP(air, sc.terrain, device=0, torch_alloc=False)
            ctx.add_plans(sc.plans)
            ctx.set_launch(cull=cull, step_budget=7)
            out[(cull, seq)] = ctx.schedule_batch(sc.src, sc.dst, sc.t0, sequential=seq)
            ctx.close()
    ref = out[(0, True)]
    for key, res in out.items():
        assert all(_same(a, b) for a, b in zip(ref, res)), f"c2s mismatch {key}"
    print("c2s:", [r.status for r in ref], [r.n_states for r in ref])


def case_reuse():
    """Speculative culled batch with rollbacks whose re-walks re-converge (re-convergence check,
    backup copy, reconv_copy epilogue), against the sequential loop."""
    sc = fs.random_small(49, n_plans=60, n_requests=16, half_m=1200.0, n_buildings=20, max_steps=500, t0_max=60)
    out = {}
    for seq in (True, False):
        ctx = FMDP(sc.airspace, sc.terrain, device=0, torch_alloc=False)
        ctx.add_plans(sc.plans)
        ctx.set_launch(cull=1, step_budget=7)
        out[seq] = ctx.schedule_batch(sc.src, sc.dst, sc.t0, sequential=seq)
        if not seq:
            rc = ctx.stats()["reconverged"]
        ctx.close()
    assert all(_same(a, b) for a, b in zip(out[True], out[False])), "reuse mismatch"
    print("reuse: reconverged", rc, [r.status for r in out[True]])


def case_cosim():
    sc = fs.cosim_ring(3, 3, n_plans=30, max_steps=150)
    ctx = FMDP(sc.airspace, sc.terrain, device=0, torch_alloc=False)
    ctx.add_plans(sc.plans)
    res = ctx.schedule_cosim(sc.src, sc.dst, sc.t0)
    print("cosim:", [r.status for r in res], [r.n_states for r in res])
    ctx.close()


def case_p2p():
    sc = fs.random_small(21, n_plans=200, n_requests=1, half_m=1500.0, max_steps=150)
    one = FMDP(sc.airspace, sc.terrain, device=0, torch_alloc=False)
    one.add_plans(sc.plans)
    ref = one.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    one.set_launch(split=2)
    sp = one.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    assert _same(ref, sp), "split request differs"
    one.close()
    ctxs = []
    for _ in range(2):
        c = FMDP(sc.airspace, sc.terrain, device=0, torch_alloc=False)
        c.add_plans(sc.plans)
        ctxs.append(c)
    p2p_connect_local(ctxs)
    import threading
    res = [None, None]

    def run(i):
        res[i] = ctxs[i].schedule_p2p(sc.src[0], sc.dst[0], int(sc.t0[0]))

    th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert all(_same(ref, r) for r in res), "p2p differs"
    print("p2p:", ref.status, ref.n_states)
    for c in ctxs:
        c.close()


def case_f4():
    # the wide walker (A = 45 over two action tiles, decision board) and the request-sharded batch
    kw = dict(turn_steps=(-6, -3, 0, 3, 6), acc_units=(-4, 0, 4), climb_units=(-16, 0, 16))
    sc = fs.random_small(93, n_plans=60, n_requests=2, half_m=1200.0, max_steps=120, t0_max=20)
    air = fs.airspace_f4(**kw).replace(lo_m=sc.airspace.lo_m, hi_m=sc.airspace.hi_m,
                                       horizon_steps=sc.airspace.horizon_steps,
                                       row_capacity=sc.airspace.row_capacity, max_steps=120)
    ctx = FMDP(air, sc.terrain, device=0, torch_alloc=False)
    ctx.add_plans(sc.plans)
    res = ctx.schedule_batch(sc.src, sc.dst, sc.t0)
    print("f4:", [r.status for r in res], [r.n_states for r in res])
    ctx.close()


def case_dist():
    import threading
    sc = fs.random_small(71, n_plans=60, n_requests=6, half_m=1200.0, max_steps=150, t0_max=40)
    ref = FMDP(sc.airspace, sc.terrain, device=0, torch_alloc=False)
    ref.add_plans(sc.plans)
    want = ref.schedule_batch(sc.src, sc.dst, sc.t0)
    ref.close()
    ctxs = []
    for _ in range(2):
        c = FMDP(sc.airspace, sc.terrain, device=0, torch_alloc=False)
        c.add_plans(sc.plans)
        ctxs.append(c)
    bar = threading.Barrier(2)
    slots = [None, None]

    def gather(r):
        def f(block):
            slots[r] = block
            bar.wait()
            out = list(slots)
            bar.wait()
            return out
        return f
    out = [None, None]
    th = [threading.Thread(target=lambda r=r: out.__setitem__(r, ctxs[r].schedule_batch_dist(
        sc.src, sc.dst, sc.t0, gather(r), r, 2))) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert all(_same(a, b) for r in range(2) for a, b in zip(out[r], want)), "dist batch differs"
    print("dist:", [r.status for r in want])
    for c in ctxs:
        c.close()


if __name__ == "__main__":
    for name in sys.argv[1:] or ["c1", "c2s", "cosim", "p2p", "f4", "dist"]:
        globals()["case_" + name]()
    print("sanitize cases ok")

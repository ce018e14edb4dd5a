"""Plan-sharded scheduling is bit-identical to one GPU: world size 1, and two
ranks (processes) that share this GPU and exchange their per-step minima over gloo."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import fmdp_synth as fs

pytestmark = pytest.mark.gpu


def _scenario():
    return fs.random_small(71, n_plans=300, n_requests=3, half_m=1500.0, n_buildings=30, max_steps=400, t0_max=40)


def test_sharded_world1_equals_schedule():
    from paper_2008_03518_b200.fmdp import FMDP
    sc = _scenario()
    a = FMDP(sc.airspace, sc.terrain)
    a.add_plans(sc.plans)
    b = FMDP(sc.airspace, sc.terrain)
    b.add_plans(sc.plans)
    for i in range(sc.n_requests):
        x = a.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]))
        y = b.schedule_sharded(sc.src[i], sc.dst[i], int(sc.t0[i]), 0, 1, lambda arr: None)
        assert x.status == y.status and x.n_states == y.n_states and (x.traj == y.traj).all()
        assert x.min_sep_m == y.min_sep_m and x.plan_id == y.plan_id
    a.close()
    b.close()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2008_03518_b200.fmdp import FMDP, allreduce_min_torch
    sc = _scenario()
    ctx = FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    red = allreduce_min_torch()
    out = []
    for i in range(sc.n_requests):
        r = ctx.schedule_sharded(sc.src[i], sc.dst[i], int(sc.t0[i]), rank, world, red)
        out.append((r.status, r.n_states, r.traj))
    np.save(os.path.join(out_dir, f"s{rank}.npy"), np.array([o[:2] for o in out]))
    for i, o in enumerate(out):
        np.save(os.path.join(out_dir, f"t{rank}_{i}.npy"), o[2])
    ctx.close()
    dist.destroy_process_group()


def test_sharded_two_ranks_bit_identical(tmp_path):
    from paper_2008_03518_b200.fmdp import FMDP
    sc = _scenario()
    ref = FMDP(sc.airspace, sc.terrain)
    ref.add_plans(sc.plans)
    want = [ref.schedule(sc.src[i], sc.dst[i], int(sc.t0[i])) for i in range(sc.n_requests)]
    ref.close()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        st = np.load(tmp_path / f"s{r}.npy")
        for i, w in enumerate(want):
            assert st[i][0] == w.status and st[i][1] == w.n_states
            assert (np.load(tmp_path / f"t{r}_{i}.npy") == w.traj).all()


# --------------------------------------------------------------------------- in-kernel exchange
# fmdp_schedule_p2p (SURVEY §8(e) production form): the per-step exchange runs inside the walker
# kernels through the peers' exchange areas.  On one GPU the "ranks" are contexts of this
# process, each walker on its own stream; the protocol (P2P stores, step tags, parity buffers)
# is the one the NVLink peers use, only the pointers are local.

def _p2p_ranks(sc, world, cull=0, split=0):
    from paper_2008_03518_b200.fmdp import FMDP, p2p_connect_local
    ctxs = []
    for _ in range(world):
        c = FMDP(sc.airspace, sc.terrain)
        c.add_plans(sc.plans)
        c.set_launch(cull=cull, split=split)
        ctxs.append(c)
    p2p_connect_local(ctxs)
    return ctxs


def _p2p_call(ctxs, src, dst, t0):
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(len(ctxs)) as ex:
        futs = [ex.submit(c.schedule_p2p, src, dst, t0) for c in ctxs]
        return [f.result(timeout=120) for f in futs]


@pytest.mark.parametrize("world,cull,split", [(1, 0, 0), (2, 0, 0), (3, 1, 0), (4, 0, 0),
                                              (2, 0, 2), (2, 1, 3), (3, 0, 2)])
def test_p2p_bit_identical_to_one_gpu(world, cull, split):
    """split >= 2: the two-level exchange -- `split` clusters per rank exchange among themselves,
    then cluster c of every rank with cluster c of the others."""
    from paper_2008_03518_b200.fmdp import FMDP
    sc = _scenario()
    ref = FMDP(sc.airspace, sc.terrain)
    ref.add_plans(sc.plans)
    ref.set_launch(split=1)
    ctxs = _p2p_ranks(sc, world, cull, split)
    for i in range(sc.n_requests):
        want = ref.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]))
        got = _p2p_call(ctxs, sc.src[i], sc.dst[i], int(sc.t0[i]))
        if split:
            assert all(c.stats()["split"] == split for c in ctxs)
        for g in got:  # every rank took every decision identically, appended the same plan
            assert g.status == want.status and g.n_states == want.n_states
            assert (g.traj == want.traj).all()
            assert g.min_sep_m == want.min_sep_m and g.plan_id == want.plan_id
            assert g.n_near_ties == want.n_near_ties
    assert all(c.num_plans() == ref.num_plans() for c in ctxs)
    for c in ctxs + [ref]:
        c.close()


def test_p2p_shards_the_pairs():
    """Each rank evaluates only its shard: pair evaluations sum to the single-GPU count."""
    from paper_2008_03518_b200.fmdp import FMDP
    sc = _scenario()
    ref = FMDP(sc.airspace, sc.terrain)
    ref.add_plans(sc.plans)
    ref.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    want = ref.stats()["pair_evals"]
    ctxs = _p2p_ranks(sc, 2)
    _p2p_call(ctxs, sc.src[0], sc.dst[0], int(sc.t0[0]))
    got = [c.stats()["pair_evals"] for c in ctxs]
    assert sum(got) == want and min(got) > 0.3 * want
    for c in ctxs + [ref]:
        c.close()


def test_p2p_missing_peer_times_out_and_reconnects():
    from paper_2008_03518_b200.fmdp import FmdpError, p2p_connect_local
    sc = _scenario()
    ctxs = _p2p_ranks(sc, 2)
    with pytest.raises(FmdpError, match="timed out"):
        ctxs[0].schedule_p2p(sc.src[0], sc.dst[0], int(sc.t0[0]))  # rank 1 never calls
    with pytest.raises(FmdpError, match="connect"):
        ctxs[0].schedule_p2p(sc.src[0], sc.dst[0], int(sc.t0[0]))
    p2p_connect_local(ctxs)
    ok = _p2p_call(ctxs, sc.src[1], sc.dst[1], int(sc.t0[1]))
    assert ok[0].status == ok[1].status and (ok[0].traj == ok[1].traj).all()
    for c in ctxs:
        c.close()


def _ipc_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2008_03518_b200.fmdp import FMDP, p2p_connect_group
    sc = _scenario()
    ctx = FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    p2p_connect_group(ctx)
    for i in range(sc.n_requests):
        r = ctx.schedule_p2p(sc.src[i], sc.dst[i], int(sc.t0[i]))
        np.save(os.path.join(out_dir, f"ipc{rank}_{i}.npy"), np.concatenate([[r.status, r.n_states], r.traj.ravel()]))
    ctx.close()
    dist.destroy_process_group()


def test_p2p_two_processes_cuda_ipc(tmp_path):
    """The cross-process form: exchange areas mapped by CUDA IPC handles all-gathered over a
    torch.distributed group (p2p_connect_group).  Both processes share this one GPU (without
    MPS only by time-slicing, so this checks the mapping and the protocol, not speed)."""
    from paper_2008_03518_b200.fmdp import FMDP
    sc = _scenario()
    ref = FMDP(sc.airspace, sc.terrain)
    ref.add_plans(sc.plans)
    want = [ref.schedule(sc.src[i], sc.dst[i], int(sc.t0[i])) for i in range(sc.n_requests)]
    ref.close()
    assert max(w.n_states for w in want) > 50
    mp.spawn(_ipc_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        for i, w in enumerate(want):
            got = np.load(tmp_path / f"ipc{r}_{i}.npy")
            assert got[0] == w.status and got[1] == w.n_states
            assert (got[2:].reshape(-1, 3) == w.traj).all()


@pytest.mark.parametrize("split,cull", [(2, 0), (3, 1), (4, 0), (8, 1)])
def test_split_request_bit_identical(split, cull):
    """fmdp_launch.split: one request walked by several clusters of this GPU, each over a shard
    of every row, combined per step by the in-kernel exchange -- identical to one cluster."""
    from paper_2008_03518_b200.fmdp import FMDP
    sc = _scenario()
    ref = FMDP(sc.airspace, sc.terrain)
    ref.add_plans(sc.plans)
    ref.set_launch(cull=cull, split=1)
    ctx = FMDP(sc.airspace, sc.terrain)
    ctx.add_plans(sc.plans)
    ctx.set_launch(cull=cull, split=split)
    for i in range(sc.n_requests):
        a = ref.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]))
        b = ctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]))
        assert 2 <= ctx.stats()["split"] <= split  # capped by the co-resident 16-CTA clusters
        assert a.status == b.status and a.n_states == b.n_states and (a.traj == b.traj).all()
        assert a.min_sep_m == b.min_sep_m and a.plan_id == b.plan_id and a.n_near_ties == b.n_near_ties
        ha, hb = ref.steplog(0), ctx.steplog(0)
        assert all((x == y).all() for x, y in zip(ha, hb))
    assert ref.stats()["split"] == 0 or ref.stats()["split"] == 1
    ref.close()
    ctx.close()


@pytest.mark.parametrize("air,split", [(dict(valuation=1), 3),
                                       (dict(turn_steps=tuple(range(-8, 9)), climb_units=(-32, -16, 0, 16, 32)), 4)])
def test_split_request_variants(air, split):
    """The split request with Alg 1 endpoint valuation and with 17 x 5 = 85 actions
    (configs[4] action set, C = 5): identical to one cluster."""
    from paper_2008_03518_b200.fmdp import FMDP
    sc = fs.random_small(73, n_plans=300, n_requests=3, half_m=1500.0, n_buildings=20, max_steps=400, t0_max=40,
                         **air)
    ref = FMDP(sc.airspace, sc.terrain)
    ref.add_plans(sc.plans)
    ref.set_launch(split=1)
    ctx = FMDP(sc.airspace, sc.terrain)
    ctx.add_plans(sc.plans)
    ctx.set_launch(split=split)
    for i in range(sc.n_requests):
        a = ref.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]))
        b = ctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]))
        assert ctx.stats()["split"] >= 2
        assert a.status == b.status and a.n_states == b.n_states and (a.traj == b.traj).all()
        assert a.min_sep_m == b.min_sep_m and a.n_near_ties == b.n_near_ties
    ref.close()
    ctx.close()


def test_p2p_cluster_count_changes_between_requests():
    """The two-level exchange's tag sequence is monotonic across launches: changing the number
    of clusters per rank between requests on one connection (2 -> 1 -> 3 -> 2) never lets a
    stale word match, and every request stays identical to one GPU."""
    from paper_2008_03518_b200.fmdp import FMDP
    sc = fs.random_small(71, n_plans=300, n_requests=4, half_m=1500.0, n_buildings=30, max_steps=400, t0_max=40)
    ref = FMDP(sc.airspace, sc.terrain)
    ref.add_plans(sc.plans)
    ref.set_launch(split=1)
    ctxs = _p2p_ranks(sc, 2)
    for i, k in enumerate((2, 1, 3, 2)):
        for c in ctxs:
            c.set_launch(split=k)
        want = ref.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]))
        got = _p2p_call(ctxs, sc.src[i], sc.dst[i], int(sc.t0[i]))
        for g in got:
            assert g.status == want.status and g.n_states == want.n_states and (g.traj == want.traj).all()
    for c in ctxs + [ref]:
        c.close()


def test_api_keeps_the_callers_current_device():
    """Every call runs on the context's device and leaves the caller's current device as it was
    (one process may hold contexts on several GPUs)."""
    import torch
    from paper_2008_03518_b200.fmdp import FMDP
    sc = _scenario()
    before = torch.cuda.current_device()
    ctx = FMDP(sc.airspace, sc.terrain, device=0)
    ctx.add_plans(sc.plans)
    ctx.schedule(sc.src[0], sc.dst[0], int(sc.t0[0]))
    assert torch.cuda.current_device() == before
    ctx.close()

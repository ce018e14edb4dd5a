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

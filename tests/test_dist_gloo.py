"""Multi-process host logic on CPU (gloo, world size 2): the min-all-reduce adapter used by
the plan-sharded path and bench.py's max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_03518_b200.fmdp import allreduce_min_torch
    import bench
    rng = np.random.default_rng(100 + rank)
    v = rng.integers(0, 2 ** 32, size=1351, dtype=np.uint64).astype(np.uint32)
    v[0] = 0xFFFFFFFF  # saturated entries survive
    allreduce_min_torch()(v)
    t = bench.max_over_ranks(float(rank + 1), world)
    tot = bench.sum_over_ranks(100.0, world)
    np.save(os.path.join(out_dir, f"r{rank}.npy"), v)
    np.save(os.path.join(out_dir, f"t{rank}.npy"), np.array([t, tot]))
    dist.destroy_process_group()


def test_gloo_allreduce_min_and_timing(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    vs = [np.random.default_rng(100 + r).integers(0, 2 ** 32, size=1351, dtype=np.uint64).astype(np.uint32)
          for r in range(world)]
    for v in vs:
        v[0] = 0xFFFFFFFF
    want = np.minimum(vs[0], vs[1])
    for r in range(world):
        got = np.load(tmp_path / f"r{r}.npy")
        assert (got == want).all() and got.dtype == np.uint32
        t, tot = np.load(tmp_path / f"t{r}.npy")
        assert t == world and tot == 100.0 * world


class _FakeCtx:
    """Stands in for FMDP: records what p2p_connect_group hands to the library."""

    def __init__(self, rank):
        self.rank = rank
        self.got = None

    def p2p_export(self, world):
        return bytes([self.rank + 1]) * 64, 0x1000 * (self.rank + 1)

    def p2p_connect(self, rank, world, handles, ptrs):
        self.got = (rank, world, [h[0] for h in handles], list(ptrs))
        if self.rank == 1 and getattr(self, "fail", False):
            raise RuntimeError("no peer access")


def _connect_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_03518_b200.fmdp import p2p_connect_group
    c = _FakeCtx(rank)
    p2p_connect_group(c)
    r, w, hs, ps = c.got
    # a failure on one rank raises on every rank (nobody is left in a collective)
    c2 = _FakeCtx(rank)
    c2.fail = True
    raised = 0
    try:
        p2p_connect_group(c2)
    except Exception as e:
        raised = int("rank 1: no peer access" in str(e))
    np.save(os.path.join(out_dir, f"c{rank}.npy"), np.array([r, w] + hs + ps + [raised], dtype=np.int64))
    dist.destroy_process_group()


def test_gloo_p2p_connect_group_exchanges_handles(tmp_path):
    """In-kernel exchange setup: every rank receives every rank's IPC handle in
    rank order; a peer in another process is reached through its handle (pointer 0), its own
    area through its own pointer."""
    world = 2
    mp.spawn(_connect_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        got = np.load(tmp_path / f"c{r}.npy").tolist()
        assert got[:2] == [r, world]
        assert got[2:4] == [1, 2]
        want_ptrs = [0x1000 * (q + 1) if q == r else 0 for q in range(world)]
        assert got[4:6] == want_ptrs
        assert got[6] == 1


def _gather_worker(rank, world, port, out_dir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2008_03518_b200.fmdp import allgather_torch
    f = allgather_torch()
    # the two exchanges of one fmdp_schedule_batch_dist round: block sizes (8 bytes), then the
    # records padded to the largest block; and an all-empty round (no request finished anywhere)
    sizes = f(np.array([17 * (rank + 1)], np.int64).tobytes())
    blocks = f(bytes([rank + 1]) * 40)
    empty = f(b"")
    import json
    json.dump([np.frombuffer(b"".join(sizes), np.int64).tolist(), [b[0] for b in blocks], [len(b) for b in blocks],
               [len(e) for e in empty]], open(os.path.join(out_dir, f"g{rank}.json"), "w"))
    dist.destroy_process_group()


def test_gloo_allgather_blocks(tmp_path):
    """allgather_torch (plumbing of the request-sharded batch, fmdp_schedule_batch_dist): equal-size
    byte blocks gathered in rank order, also empty ones."""
    world = 2
    mp.spawn(_gather_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        import json
        sizes, first, lens, empty = json.load(open(tmp_path / f"g{r}.json"))
        assert sizes == [17, 34] and first == [1, 2] and lens == [40, 40] and empty == [0, 0]

"""Cross-process exchange areas (CUDA IPC) on ONE GPU: two processes, gloo group,
p2p_connect_group, then fmdp_schedule_p2p on both.  Without MPS the two walkers only share the
GPU by time-slicing, so this checks the IPC mapping and the protocol, not speed."""
import os
import sys
import time

import numpy as np
import torch.multiprocessing as mp

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def worker(rank, world, port):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import fmdp_synth as fs
    from paper_2008_03518_b200.fmdp import FMDP, p2p_connect_group
    sc = fs.random_small(71, n_plans=300, n_requests=8, half_m=1500.0, n_buildings=30, max_steps=400, t0_max=40)
    ref = FMDP(sc.airspace, sc.terrain)
    ref.add_plans(sc.plans)
    j = 0
    for j in range(sc.n_requests):
        want = ref.schedule(sc.src[j], sc.dst[j], int(sc.t0[j]))
        ref.truncate(len(sc.plans))
        if want.n_states > 50:
            break
    ref.close()
    ctx = FMDP(sc.airspace, sc.terrain)
    ctx.add_plans(sc.plans)
    p2p_connect_group(ctx)
    dist.barrier()
    t = time.perf_counter()
    try:
        got = ctx.schedule_p2p(sc.src[j], sc.dst[j], int(sc.t0[j]))
        ok = got.status == want.status and got.n_states == want.n_states and (got.traj == want.traj).all()
        print(f"rank {rank}: status {got.status} n {got.n_states} identical={ok} "
              f"{time.perf_counter() - t:.2f} s", flush=True)
    except Exception as e:
        print(f"rank {rank}: error {e} after {time.perf_counter() - t:.2f} s", flush=True)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(worker, args=(2, 29533), nprocs=2, join=True)

#!/usr/bin/env python
"""Benchmark of the FastMDP-GPU hot path on BASELINE.json configs[1].

One "step" = one first-come-first-served batch of 100 requests scheduled against the
3000-plan store with terrain (all rows of SURVEY §8(a): wells, projection, goal, hot loop,
terrain, combine, argmax, advance, separation, append, FCFS speculation).  The store is
restored (fmdp_truncate) and L2 is flushed between steps, outside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

N > 1 (torchrun, one process per GPU): the same configs[1] batch request-sharded over the ranks
(fmdp_schedule_batch_dist: rank i % N walks request i, finished requests all-gathered once per
speculative round, in-order commits on every rank) -> strong scaling, value = the
batch's requests / max time over ranks.  --impl reference times the oracle (oracle/, fp64 C) on host cores on a
bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FCFS requests scheduled/sec and ms/request vs #accepted plans, 1/2/4/8 B200"
WORKLOAD = ("configs[1]: batch of 100 FCFS requests against 3000 accepted plans with a 256-well terrain "
            "grid, 16x16 km dense urban airspace, 9 headings x 3 climbs, W=10")
OPS_PER_PAIR = 7.0  # algorithmic FP32 ops per (state, well) pair
EXEC_OPS_PER_PAIR = 4.0 / 3.0  # FP32 lane-ops the kernel executes per pair at 3 climbs ((2 + C - 1)/C, level climb skipped)
LOOP_CEILING_PAIRS_PER_CLK_SM = 40.0  # isolated hot loop as the walker runs it, C = 3 with the level-climb
# skip (tools/hotbench/hotbench2.cu V0, profiles/r02s2_rates.txt: 38.3-39.6; round 1 measured 34-36
# without the skip)


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="native", choices=["native", "reference"])
    p.add_argument("--seed", type=int, default=2)
    p.add_argument("--cpu-sample-s", type=float, default=15.0)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-c4", action="store_true", help="skip the configs[2] / configs[3] blocks")
    p.add_argument("--only-c4", action="store_true", help="run only the configs[2] / configs[3] blocks")
    p.add_argument("--c5-full", action="store_true",
                   help="add configs[4] at its defined size (1M plans x 3000 rows, 48 GB; minutes to load)")
    return p.parse_args()


_T0 = time.perf_counter()


def _log(msg: str):
    """Progress on stderr (the JSON line alone goes to stdout)."""
    print(f"[bench {time.perf_counter() - _T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _reduce(x: float, world: int, op: str) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def max_over_ranks(x: float, world: int) -> float:
    """Timing of a multi-GPU run: the slowest rank's device time."""
    return _reduce(x, world, "max")


def sum_over_ranks(x: float, world: int) -> float:
    return _reduce(x, world, "sum")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 3 + i and r[3 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def host_cpu():
    """nproc and the lscpu model line of this host."""
    n = os.cpu_count() or 1
    try:
        n = len(os.sched_getaffinity(0))
    except Exception:
        pass
    model = ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                model = ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return n, model


def _oracle_run(sc, budget_s, threads):
    from oracle import oracle as O
    O.set_threads(threads)
    try:
        orc = O.for_scenario(sc)
        t0 = time.perf_counter()
        done = states = 0
        mine = []
        while done < sc.n_requests and time.perf_counter() - t0 < budget_s:
            r = orc.schedule(sc.src[done], sc.dst[done], int(sc.t0[done]))
            mine.append(r)
            states += r.n_states
            done += 1
        return mine, states, time.perf_counter() - t0
    finally:
        O.set_threads(1)


def cpu_baseline(sc, budget_s: float, gpu=None):
    """The oracle as it stands (fp64 C, one core): FCFS requests of the same batch, in order,
    until the time budget is spent.  With ``gpu`` (per request: status, trajectory, headings,
    actions of the timed GPU batch) the same requests are also checked against the GPU path: a
    request whose oracle trajectory equals the GPU's has no divergent step; otherwise the oracle
    lockstep-replays the GPU trajectory (store = the GPU's earlier accepted plans) and counts the
    steps where the GPU took the other action of a logged near-tie (north-star rule) and any
    failure."""
    from oracle import oracle as O
    ncores, model = host_cpu()
    # (i) one core; (ii) OpenMP over the projected states on every host core (SURVEY d.5)
    mine1, states1, dt1 = _oracle_run(sc, budget_s / 2, 1)
    mine, states, dt = _oracle_run(sc, budget_s / 2, ncores)
    done = len(mine)
    out = {"value": done / dt, "unit": "requests/s", "cores": ncores, "kind": "oracle",
           "host": {"nproc": ncores, "lscpu_model": model},
           "sample": f"first {done} of {sc.n_requests} requests of the same FCFS batch ({states} states) "
                     f"in {dt:.1f} s, fp64 C oracle, OpenMP over the projected states on {ncores} threads",
           "single_thread": {"value": len(mine1) / dt1, "unit": "requests/s", "cores": 1,
                             "sample": f"first {len(mine1)} requests ({states1} states) in {dt1:.1f} s"}}
    if len(mine1) > done:
        mine = mine1
        done = len(mine1)
    if gpu is not None:
        rep = O.for_scenario(sc)
        div = fail = ident = 0
        for i in range(min(done, len(gpu))):
            st_g, tr, hd, ast = gpu[i]
            if st_g == mine[i].status and len(tr) == mine[i].n_states and (tr == mine[i].traj).all():
                ident += 1
            else:
                rs = rep.replay(sc.src[i], sc.dst[i], int(sc.t0[i]), tr, hd, ast, st_g)
                div += rs.n_divergent
                fail += rs.n_fail
            if st_g == 0:
                rep.add_plan(int(sc.t0[i]), tr)
        out["parity"] = {"requests_checked": min(done, len(gpu)), "identical_to_oracle": ident,
                         "divergent_steps": div, "failed_steps": fail,
                         "rule": "divergent = GPU took the other action of a logged near-tie (top-2 gap < 1e-4 S); "
                                 "failed = any other difference (must be 0)"}
    return out


def committed_pairs(sc, res, A, W, n_tau=5):
    """(state, intruder well) pairs the method evaluates for the committed decision steps of one
    FCFS batch: request i decides at steps k = 0..n_i-2, each over A*W states x
    n_tau wells of every plan active at row t0_i + k -- the initial store plus the plans the
    batch accepted before i.  Speculative work that was rolled back is not method work."""
    import numpy as np
    H = int(sc.airspace.horizon_steps)
    cnt = np.zeros(H + 1, np.int64)
    for t0, st in sc.plans:
        cnt[t0] += 1
        cnt[min(H, t0 + len(st))] -= 1
    cnt = np.cumsum(cnt)[:H]
    tot = 0
    for i, r in enumerate(res):
        t0 = int(sc.t0[i])
        tot += int(cnt[t0:t0 + max(0, r.n_states - 1)].sum())
        if r.status == 0:
            cnt[t0:t0 + r.n_states] += 1
    return tot * A * W * n_tau


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    import fmdp_synth as fs
    from oracle import oracle as O
    sc = fs.config_c2(seed=args.seed)
    ncores, model = host_cpu()
    O.set_threads(ncores)  # the oracle's OpenMP timing variant on every host core (identical results)
    n_req = 2  # bounded sample per step: the first two FCFS requests of the batch
    times, states = [], 0
    for i in range(args.warmup + args.steps):
        orc = O.for_scenario(sc)
        nr = 1 if i < args.warmup else n_req  # warm-up steps: one request
        t0 = time.perf_counter()
        st = sum(orc.schedule(sc.src[q], sc.dst[q], int(sc.t0[q])).n_states for q in range(nr))
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
            states += st
    tot = sum(times)
    value = n_req * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": "first two FCFS requests of the batch per step"},
            "cpu_baseline": {"value": value, "unit": "requests/s", "cores": ncores, "kind": "oracle",
                             "host": {"nproc": ncores, "lscpu_model": model},
                             "sample": f"first two FCFS requests of the configs[1] batch ({states // max(1, args.steps)} "
                                       f"states) per step, fp64 C oracle, OpenMP on {ncores} threads"},
            "e2e": {"value": value, "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def run_native(args):
    rank, world, local = dist_env()
    import numpy as np
    import torch
    # FMDP_BENCH_SAME_DEVICE=1 (testing the N > 1 code path on a one-GPU box): every rank on
    # device 0, gloo for the host-side collectives; the ranks' kernels then only time-slice
    same = os.environ.get("FMDP_BENCH_SAME_DEVICE") == "1"
    if same:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if same:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import fmdp_synth as fs
    from paper_2008_03518_b200.fmdp import FMDP, Request, Result, allgather_torch, pack_plans
    gather = None
    if world > 1:
        gather = allgather_torch(device=None if same else torch.device("cuda", local))

    # N > 1: ONE configs[1] FCFS batch, request-sharded over the ranks (fmdp_schedule_batch_dist:
    # rank i % N walks request i, finished requests all-gathered once per speculative round, commits
    # in array order on every rank -- SURVEY §8(e) second partitioning): the same seed everywhere
    sc = fs.config_c2(seed=args.seed)
    stream = torch.cuda.Stream(device=local)
    ctx = FMDP(sc.airspace, sc.terrain, device=local, stream=stream)
    ctx.add_plans(sc.plans)
    n0 = ctx.num_plans()
    reqs = ctx.make_requests(sc.src, sc.dst, sc.t0)
    n = len(reqs)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def one(want_traj):
        with torch.cuda.stream(stream):
            ev0.record(stream)
            if gather is None:
                res = ctx.schedule_batch(None, None, None, want_traj=want_traj, reqs=reqs)
            else:
                res = ctx.schedule_batch_dist(None, None, None, gather, rank, world, want_traj=want_traj, reqs=reqs)
            ev1.record(stream)
        ev1.synchronize()
        return res, ev0.elapsed_time(ev1)

    def reset():
        ctx.truncate(n0)
        flush.zero_()
        torch.cuda.synchronize()

    def measure(cull):
        ctx.set_launch(cull=cull)
        for _ in range(args.warmup):
            one(False)
            reset()
        # value: device-resident store and requests, trajectories left on the device
        times, st_all, res_last = [], [], None
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            for _ in range(args.steps):
                res, ms = one(False)
                st_all.append(ctx.stats())
                times.append(ms)
                res_last = res
                reset()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        # e2e: through the public API with host requests, trajectories and results copied back
        e2e_times, d2h = [], 0
        gpu_log = None
        one(True)  # untimed: the host-buffer path's first call (result and trajectory staging)
        reset()
        for _ in range(max(1, args.steps)):
            torch.cuda.synchronize()
            res, ms = one(True)
            e2e_times.append(ms)
            d2h = sum(r.n_states for r in res) * 12 + n * C_RESULT_BYTES
            if gpu_log is None:  # the oracle checks these requests beside the cpu_baseline (rank 0)
                gpu_log = []
                for i in range(min(n, 12)):
                    ast, hd, _ = ctx.steplog(i)
                    gpu_log.append((res[i].status, res[i].traj, hd, ast))
            reset()
        tot_ms = max_over_ranks(sum(times), world)
        e2e_ms = max_over_ranks(sum(e2e_times), world)
        return dict(tot_ms=tot_ms, e2e_ms=e2e_ms,  # one batch of n requests per step, all ranks together
                    value=n * args.steps / (tot_ms / 1e3),
                    e2e_value=n * len(e2e_times) / (e2e_ms / 1e3), d2h=d2h,
                    st_all=st_all, res_last=res_last, clocks=clk.summary(), gpu_log=gpu_log,
                    walk_ms=sum(s["device_ms"] for s in st_all), pairs=sum(s["pair_evals"] for s in st_all),
                    launches=sum(s["kernels"] for s in st_all),
                    steps_dev=sum_over_ranks(sum(s["steps"] for s in st_all), world))  # every rank's walkers

    def measure_departures(n_req=8, delays=tuple(range(0, 400, 50))):
        # each request tried at len(delays) departures in one call, earliest accepted kept
        ctx.set_launch(cull=1)
        sub = [(sc.src[i], sc.dst[i], int(sc.t0[i])) for i in range(n_req)]

        def run():
            chosen = []
            with torch.cuda.stream(stream):
                ev0.record(stream)
                for s_, d_, t_ in sub:
                    chosen.append(ctx.schedule_departures(s_, d_, t_, delays, want_traj=False)[1])
                ev1.record(stream)
            ev1.synchronize()
            return chosen, ev0.elapsed_time(ev1)
        for _ in range(args.warmup):
            run()
            reset()
        times, chosen = [], []
        for _ in range(args.steps):
            chosen, ms = run()
            times.append(ms)
            reset()
        tot = max_over_ranks(sum(times), world)
        return {"what": "SURVEY f3: each request scheduled at 8 candidate departures (t0 + 0..350 steps) in one "
                        "walk against the same store; the earliest accepted is appended "
                        "(tests/test_gpu_parity.py::test_departure_candidates)",
                "value": sum_over_ranks(n_req * args.steps, world) / (tot / 1e3), "unit": "requests/s",
                "candidates_per_request": len(delays), "requests_per_step": n_req, "cull": 1,
                "ms_per_request": tot / args.steps / n_req, "chosen_delay_index": chosen}

    def measure_cosim(sizes=(1, 5, 10, 20), n_plans=100):
        # SURVEY f2 / Fig perf2: co-simulated batches against 100 intruders;
        # batch cycles/s = clocks / time, total cycles/s = aircraft-steps / time
        out = []
        for nb in sizes:
            cs = fs.cosim_ring(args.seed + 40 + rank, nb, n_plans=n_plans)
            cctx = FMDP(cs.airspace, cs.terrain, device=local, stream=stream)
            cctx.add_plans(cs.plans)
            c0 = cctx.num_plans()
            creqs = cctx.make_requests(cs.src, cs.dst, cs.t0)
            times, res = [], None
            for it in range(args.warmup + args.steps):
                with torch.cuda.stream(stream):
                    ev0.record(stream)
                    res = cctx.schedule_cosim(None, None, None, want_traj=False, reqs=creqs)
                    ev1.record(stream)
                ev1.synchronize()
                if it >= args.warmup:
                    times.append(ev0.elapsed_time(ev1))
                cctx.truncate(c0)
            st = cctx.stats()
            cctx.close()
            ms = max_over_ranks(sum(times), world) / len(times)
            clocks = max(int(cs.t0[i]) + r.n_states for i, r in enumerate(res)) - int(cs.t0.min())
            steps = sum(r.n_states for r in res)
            out.append({"batch": nb, "ms_per_batch": ms, "clocks": clocks, "aircraft_steps": steps,
                        "batch_cycles_per_s": clocks / (ms / 1e3), "total_cycles_per_s": steps / (ms / 1e3),
                        "accepted": sum(r.accepted for r in res), "cluster_size": st["cluster_size"]})
        return {"what": "SURVEY f2: co-simulated batches (mutually aware, synchronous clock; Alg 5 peer wells) "
                        "against 100 intruder plans, the Fig perf2 experiment (tests/test_gpu_cosim.py)",
                "workload": "fmdp_synth.cosim_ring (ring of aircraft crossing the centre, 8 km box)",
                "paper_fig_perf2_hz": {"1": 194.5, "5": 48.5, "10": 24.0, "20": 12.2},
                "paper_note": "paper's GPU, A=1350 actions (context, not the target)",
                "sizes": out}

    def measure_latency(plan_counts=(0, 1000, 3000, 10000, 30000), reps=2, min_steps=200):
        # metric "ms/request vs #accepted plans" (Fig perf1): one request against
        # stores of P reflecting-line plans at the configs[1] traffic density (box side ~ sqrt P),
        # the first of the scenario's requests that is ACCEPTED after >= min_steps (a full trip,
        # not a truncated rejection; else the longest one); cluster size from the cost model for a
        # lone walker; device time of the walk launches
        out = []
        for P in plan_counts:
            sc_p = fs.config_scaled(args.seed + 7 + 1000 * rank, P)
            lctx = FMDP(sc_p.airspace, sc_p.terrain, device=local, stream=stream)
            if P:
                lctx.add_plans(sc_p.plans)
            row = {"plans": P, "box_km": round(2 * sc_p.airspace.hi_m[0] / 1000.0, 1)}
            pick, longest_acc, longest = None, (-1, 0), (-1, 0)
            lctx.set_launch(cull=1)
            for i in range(len(sc_p.t0)):
                r = lctx.schedule(sc_p.src[i], sc_p.dst[i], int(sc_p.t0[i]), want_traj=False)
                lctx.truncate(P)
                longest = max(longest, (r.n_states, i))
                if r.status == 0:
                    longest_acc = max(longest_acc, (r.n_states, i))
                    if r.n_states - 1 >= min_steps:
                        pick = i
                        break
            if pick is None:  # the longest accepted trip, else the longest trip
                pick = longest_acc[1] if longest_acc[0] > 0 else longest[1]
            row["request"] = pick
            for cull in (0, 1):
                lctx.set_launch(cull=cull)
                best = None
                for _ in range(reps):
                    r = lctx.schedule(sc_p.src[pick], sc_p.dst[pick], int(sc_p.t0[pick]), want_traj=False)
                    st = lctx.stats()
                    lctx.truncate(P)
                    if best is None or st["device_ms"] < best[0]:
                        best = (st["device_ms"], st["steps"], r.status, st["cluster_size"], max(1, st["split"]))
                row["culled" if cull else "full"] = {
                    "ms_per_request": best[0], "us_per_step": best[0] * 1e3 / max(1, best[1]), "steps": best[1],
                    "status": best[2], "cluster_size": best[3], "clusters": best[4]}
            lctx.close()
            out.append(row)
        return {"what": "single-request latency vs accepted plans (metric: ms/request vs #accepted plans; Fig "
                        "perf1): fmdp_synth.config_scaled, constant configs[1] density; device time of the walk",
                "points": out}

    def measure_c4(rank_counts=(2, 4), n_req=2):
        # configs[3] (100k accepted plans): single-request latency of one context (full, culled) and
        # of the plan-sharded in-kernel exchange (fmdp_schedule_p2p).  N = 1: the
        # ranks are contexts on this GPU, each walker on its own stream -- the protocol of the
        # NVLink peers (P2P stores, step tags), sharing this GPU's 148 SMs.  N > 1: one rank per
        # GPU, exchange areas shared by CUDA IPC; device time, max over ranks.
        from concurrent.futures import ThreadPoolExecutor
        from paper_2008_03518_b200.fmdp import pack_plans, p2p_connect_group, p2p_connect_local
        _log("c4: generating configs[3]")
        sc4 = fs.config_c4(rows=1200)  # the same store on every rank
        P = len(sc4.plans)
        reqs = list(range(min(n_req, sc4.n_requests)))

        packed = pack_plans(sc4.plans)
        sc4.plans = []  # host memory: the packed arrays are all the contexts need

        def mk():
            c = FMDP(sc4.airspace, sc4.terrain, device=local)
            c.add_plans_packed(*packed)
            return c

        def row(ms, steps, status, G, k=1):
            return {"ms_per_request": ms / len(reqs), "us_per_step": ms * 1e3 / max(1, steps), "steps": steps,
                    "status": status, "cluster_size": G, "clusters": k}

        def run_single(c, cull, split):
            c.set_launch(cull=cull, split=split)
            ms = steps = 0
            st = []
            for i in reqs:
                r = c.schedule(sc4.src[i], sc4.dst[i], int(sc4.t0[i]), want_traj=False)
                s_ = c.stats()
                ms += s_["device_ms"]; steps += s_["steps"]; st.append(r.status)
                c.truncate(P)
            c.set_launch(cull=cull)
            return row(ms, steps, st, s_["cluster_size"], max(1, s_["split"])), st

        def run_p2p(cs, cull, n_world, split=0):
            # every rank takes part in every collective, also after a failed call (reported);
            # split: clusters per rank (0 = cost model, 1 = one: the ranks sharing one GPU)
            for c in cs:
                c.set_launch(cull=cull, split=split)
            ms = steps = 0
            st, errs = [], []
            for i in reqs:
                try:
                    with ThreadPoolExecutor(len(cs)) as ex:
                        rs = list(ex.map(lambda c: c.schedule_p2p(sc4.src[i], sc4.dst[i], int(sc4.t0[i]),
                                                                  want_traj=False), cs))
                    stats = [c.stats() for c in cs]
                    t = max(s_["device_ms"] for s_ in stats)
                    steps += stats[0]["steps"]; st.append(rs[0].status)
                except Exception as e:  # noqa: BLE001 -- reported in the JSON line
                    errs.append(str(e))
                    t = float("nan")
                ms += max_over_ranks(t, n_world)
                for c in cs:
                    c.truncate(P)
            st0 = cs[0].stats()
            out_row = row(ms, steps, st, st0["cluster_size"], max(1, st0["split"]))
            if errs:
                out_row["errors"] = errs[:2]
            return out_row, st

        out = {"what": "configs[3] single-request latency at 100k accepted plans; one_cluster = one 16-CTA "
                       "cluster; split = fmdp_schedule with the request split over k clusters of this GPU "
                       "(cost model; in-kernel exchange); p2p = plan-sharded ranks (fmdp_schedule_p2p)",
               "plans": P, "rows": 1200, "requests": len(reqs)}
        _log("c4: store ready")
        base = mk()
        _log("c4: context 0 loaded")
        if world == 1:
            out["one_cluster"], out["split"] = {}, {}
            want = None
            for cull in (0, 1):
                key = "culled" if cull else "full"
                out["one_cluster"][key], want = run_single(base, cull, 1)
                out["split"][key], st = run_single(base, cull, 0)
                out["split"]["same_status"] = st == want
                _log(f"c4: one cluster cull={cull} {out['one_cluster'][key]}; split {out['split'][key]}")
            out["ranks_are"] = "contexts on this one B200 (own stream each; they share its 148 SMs)"
            ctxs = [base] + [mk() for _ in range(max(rank_counts) - 1)]
            _log(f"c4: {len(ctxs)} contexts loaded")
            out["p2p"] = []
            # ranks sharing this GPU: one cluster each (R x 16 CTAs resident), and the two-level
            # exchange with 2 ranks x 3 clusters
            for R, k in [(r_, 1) for r_ in rank_counts] + [(2, 3)]:
                p2p_connect_local(ctxs[:R])
                e = {"ranks": R, "clusters_per_rank": k}
                for cull in (0, 1):
                    e["culled" if cull else "full"], st = run_p2p(ctxs[:R], cull, 1, split=k)
                    _log(f"c4: p2p ranks={R} x{k} cull={cull} {e['culled' if cull else 'full']}")
                    e["same_status_as_single"] = st == want
                out["p2p"].append(e)
            for c in ctxs:
                c.close()
        else:
            out["ranks_are"] = f"{world} GPUs, one process each (CUDA IPC exchange areas, NVLink P2P stores)"
            e = {"ranks": world}
            try:
                p2p_connect_group(base)  # raises on every rank if any rank failed
                for cull in (0, 1):
                    e["culled" if cull else "full"], _ = run_p2p([base], cull, world)
            except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
                e["error"] = str(ex)
            out["p2p"] = [e]
            base.close()
        return out

    def measure_f4(n_req=3):
        # the paper-scale action space A = 1350 (15 turns x 9 speed increments x 10
        # climbs; Table DS / KI captions P:387) against the configs[1] store, requests
        # walked one at a time by the wide walker (the action space tiled over 15 clusters);
        # compared with Fig perf1's per-step time at 3000 plans (context, the paper's GPUs)
        air = fs.airspace_f4().replace(lo_m=sc.airspace.lo_m, hi_m=sc.airspace.hi_m,
                                       horizon_steps=sc.airspace.horizon_steps, row_capacity=sc.airspace.row_capacity,
                                       max_steps=sc.airspace.max_steps)
        fctx = FMDP(air, sc.terrain, device=local, stream=stream)
        fctx.add_plans(sc.plans)
        f0 = fctx.num_plans()
        out = {"what": "SURVEY f4: A = 1350 actions (15 turns x 9 accelerations x 10 climbs, DESIGN.md R32) against "
                       "the configs[1] store (3000 plans, 256 terrain wells), one request at a time on the whole GPU "
                       "(wide walker: 15 clusters x 8 CTAs); parity: tests/test_gpu_accel.py",
               "actions": fctx.A,
               "paper_fig_perf1_ms_per_step_at_3000_plans": {"rtx2080": 4.929 + 0.0566 * 3000,
                                                              "titan_xp": 1.706 + 0.0369 * 3000},
               "paper_note": "linear fits of Fig perf1 (SURVEY App. B), A = 1350, fp64, other GPUs: context only"}
        for cull in (0, 1):
            fctx.set_launch(cull=cull)
            rows = []
            for i in range(n_req):
                r = fctx.schedule(sc.src[i], sc.dst[i], int(sc.t0[i]), want_traj=False)
                st = fctx.stats()
                fctx.truncate(f0)
                rows.append((st["device_ms"], st["steps"], r.status, st["pair_evals"]))
            ms = sum(x[0] for x in rows)
            steps = sum(x[1] for x in rows)
            out["culled" if cull else "full"] = {
                "us_per_step": ms * 1e3 / max(1, steps), "ms_per_request": ms / n_req, "steps": steps,
                "statuses": [x[2] for x in rows], "pair_evals_per_s": sum(x[3] for x in rows) / (ms / 1e3)}
        fctx.close()
        return out

    def measure_c4_full(n_seq=12, n_batch=100):
        # configs[3] at its defined size: 100k plans over 4000 rows (6.4 GB store),
        # n_seq sequential 5 km requests (full / culled; ms/request reported over the accepted
        # full-length trips and over all) and one FCFS batch of n_batch requests (culled)
        sc4, gen = fs.config_c4_full(n_requests=max(n_seq, n_batch))
        c = FMDP(sc4.airspace, sc4.terrain, device=local, stream=stream)
        t = time.perf_counter()
        for t0c, nc, stc in gen.chunks(8192):
            c.add_plans_packed(t0c, nc, stc)
        load_s = time.perf_counter() - t
        P = c.num_plans()
        out = {"what": "configs[3] at its defined size: 100k accepted plans x 4000 rows (100 x 100 km, ~6.9 "
                       "plans/km^3), 5 km requests; sequential fmdp_schedule calls (device time) and one batch",
               "plans": P, "rows": 4000, "load_s": load_s}
        for cull in (0, 1):
            c.set_launch(cull=cull)
            rows = []
            for i in range(n_seq):
                r = c.schedule(sc4.src[i], sc4.dst[i], int(sc4.t0[i]), want_traj=False)
                st = c.stats()
                c.truncate(P)
                rows.append((st["device_ms"], st["steps"], r.status, max(1, st["split"]), st["cluster_size"]))
            acc = [x for x in rows if x[2] == 0]
            out["sequential_culled" if cull else "sequential_full"] = {
                "requests": n_seq, "accepted": len(acc),
                "ms_per_accepted_request": sum(x[0] for x in acc) / len(acc) if acc else None,
                "steps_per_accepted_request": sum(x[1] for x in acc) / len(acc) if acc else None,
                "ms_per_request": sum(x[0] for x in rows) / n_seq,
                "us_per_step": sum(x[0] for x in rows) * 1e3 / max(1, sum(x[1] for x in rows)),
                "statuses": [x[2] for x in rows], "clusters": rows[0][3], "cluster_size": rows[0][4]}
            _log(f"c4 full: cull={cull} {out['sequential_culled' if cull else 'sequential_full']}")
        c.set_launch(cull=1)
        reqs4 = c.make_requests(sc4.src[:n_batch], sc4.dst[:n_batch], sc4.t0[:n_batch])
        times = []
        for _ in range(2):
            with torch.cuda.stream(stream):
                ev0.record(stream)
                res = c.schedule_batch(None, None, None, want_traj=False, reqs=reqs4)
                ev1.record(stream)
            ev1.synchronize()
            times.append(ev0.elapsed_time(ev1))
            c.truncate(P)
        out["batch_culled"] = {"requests": n_batch, "ms": min(times), "requests_per_s": n_batch / (min(times) / 1e3),
                               "accepted": sum(r.accepted for r in res),
                               "states_per_request": sum(r.n_states for r in res) / n_batch}
        _log(f"c4 full: batch {out['batch_culled']}")
        c.close()
        return out

    def measure_c5_full(n_req=10):
        # configs[4] at its defined size: 1M plans over 3000 rows (48 GB store on one
        # B200), A = 85; 10 single requests on the full path (split over the co-resident clusters)
        # and culled; device time
        sc5, gen = fs.config_c5_full(n_requests=n_req)
        c = FMDP(sc5.airspace, sc5.terrain, device=local, stream=stream)
        t = time.perf_counter()
        for t0c, nc, stc in gen.chunks(16384, device=torch.device("cuda", local)):
            c.add_plans_packed(t0c, nc, stc)
        load_s = time.perf_counter() - t
        P = c.num_plans()
        out = {"what": "configs[4] at its defined size: 1M accepted plans x 3000 rows (250 x 250 km, 48 GB store), "
                       "A = 85, single requests (device time); parity: tests/test_gpu_big.py (FMDP_BIG=1)",
               "plans": P, "rows": 3000, "load_s": load_s, "store_gb": 16.0 * P * (3000 + 8) / 1e9}
        for name, cull in (("full_split", 0), ("culled", 1)):
            c.set_launch(cull=cull)
            rows = []
            for i in range(n_req if cull else min(3, n_req)):
                r = c.schedule(sc5.src[i], sc5.dst[i], int(sc5.t0[i]), want_traj=False)
                st = c.stats()
                c.truncate(P)
                rows.append((st["device_ms"], st["steps"], r.status, st["pair_evals"], max(1, st["split"]),
                             st["cluster_size"]))
            ms, steps = sum(x[0] for x in rows), sum(x[1] for x in rows)
            out[name] = {"requests": len(rows), "us_per_step": ms * 1e3 / max(1, steps), "steps": steps,
                         "ms_per_request": ms / len(rows), "statuses": [x[2] for x in rows],
                         "pair_evals_per_s": sum(x[3] for x in rows) / (ms / 1e3), "clusters": rows[0][4],
                         "cluster_size": rows[0][5]}
            _log(f"c5 full: {name} {out[name]}")
        c.close()
        return out

    def measure_c3():
        # configs[2]: 1000 FCFS requests growing the store from 0 plans.  (i) sequential
        # fmdp_schedule calls: host wall time per call from entry to return incl. the trajectory
        # copy (SURVEY §8(d) d.1 "ms/request", median / p95), binned by #accepted plans before the
        # call -- the metric's "ms/request vs #accepted plans"; (ii) the same 1000 requests as one
        # fmdp_schedule_batch call (identical results by construction, checked).  §8(a) path.
        import numpy as np
        sc3 = fs.config_c3()
        c = FMDP(sc3.airspace, sc3.terrain, device=local)
        c.set_launch(cull=0)
        rows = []
        for i in range(sc3.n_requests):
            n_acc = c.num_plans()
            t = time.perf_counter()
            r = c.schedule(sc3.src[i], sc3.dst[i], int(sc3.t0[i]))
            dt = (time.perf_counter() - t) * 1e3
            st = c.stats()
            rows.append((n_acc, dt, st["device_ms"], st["steps"], r.status, r.n_states))
        seq = [(x[4], x[5]) for x in rows]
        total_s = sum(x[1] for x in rows) / 1e3
        bins = []
        edges = list(range(0, max(x[0] for x in rows) + 200, 200))
        for lo, hi in zip(edges[:-1], edges[1:]):
            sel = [x for x in rows if lo <= x[0] < hi]
            if not sel:
                continue
            hw = np.array([x[1] for x in sel])
            steps = sum(x[3] for x in sel)
            bins.append({"accepted_plans": [lo, hi], "requests": len(sel),
                         "host_ms_median": float(np.median(hw)), "host_ms_p95": float(np.percentile(hw, 95)),
                         "steps_per_request": steps / len(sel),
                         "device_us_per_step": sum(x[2] for x in sel) * 1e3 / max(1, steps)})
        reqs3 = c.make_requests(sc3.src, sc3.dst, sc3.t0)
        bt = []
        for _ in range(3):  # host wall of the whole call, median of 3
            c.truncate(0)
            t = time.perf_counter()
            res = c.schedule_batch(None, None, None, reqs=reqs3)
            bt.append(time.perf_counter() - t)
        batch_s = sorted(bt)[1]
        same = [(r.status, r.n_states) for r in res] == seq
        c.close()
        return {"what": "configs[2]: 1000 FCFS requests from an empty store (dense urban, terrain), §8(a) path; "
                        "host wall per fmdp_schedule call incl. trajectory copy, by #accepted plans before it",
                "requests": sc3.n_requests, "accepted": int(sum(1 for x in rows if x[4] == 0)),
                "sequential_requests_per_s": sc3.n_requests / total_s,
                "batch_requests_per_s": sc3.n_requests / batch_s, "batch_same_results": same,
                "batch_host_s_runs": bt,
                "host_ms_median": float(np.median([x[1] for x in rows])),
                "host_ms_p95": float(np.percentile([x[1] for x in rows], 95)), "by_accepted_plans": bins}

    def measure_c5():
        # configs[4] roofline stress: 1M accepted plans (64 time rows), 17 x 5 = 85 actions; one
        # request walked on the §8(a) full path, one 16-CTA cluster vs split over clusters
        # (cost model), and culled; device time, pair evaluations against the FP32 pipe peak
        sc5 = fs.config_c5(rows=64)
        packed = pack_plans(sc5.plans)
        sc5.plans = []
        c = FMDP(sc5.airspace, sc5.terrain, device=local)
        c.add_plans_packed(*packed)
        del packed
        P = c.num_plans()
        out = {"what": "configs[4]: 1M accepted plans (64 rows), A = 85 (17 headings x 5 climbs), one request, "
                       "device time of the walk (1965 MHz peak clock)",
               "plans": P, "actions": sc5.airspace.n_actions}
        for name, cull, split in (("full_one_cluster", 0, 1), ("full_split", 0, 0), ("culled", 1, 0)):
            if rank != 0:  # the single-GPU variants: rank 0 (no collectives)
                break
            c.set_launch(cull=cull, split=split)
            r = c.schedule(sc5.src[0], sc5.dst[0], int(sc5.t0[0]), want_traj=False)
            st = c.stats()
            c.truncate(P)
            secs = st["device_ms"] / 1e3
            pps = st["pair_evals"] / secs if secs > 0 else 0.0
            sms = max(1, st["split"]) * st["cluster_size"]
            C5 = len(sc5.airspace.climb_units)
            out[name] = {"us_per_step": st["device_ms"] * 1e3 / max(1, st["steps"]), "steps": st["steps"],
                         "status": r.status, "clusters": max(1, st["split"]), "cluster_size": st["cluster_size"],
                         "pair_evals_per_s": pps,
                         # 7 algorithmic ops per pair against the lane peak (can exceed 1: the Q + 2(s-o).X
                         # formulation executes (2 + C - 1) / C lane-ops per pair)
                         "algorithmic_ops_frac": pps * OPS_PER_PAIR / (148 * 128 * 1965e6),
                         "pipe_frac": pps * (2 + C5 - 1) / C5 / (148 * 128 * 1965e6),
                         "pairs_per_clk_per_sm_used": pps / (sms * 1965e6),
                         "loop_ceiling_pairs_per_clk_per_sm": "38-40 (C = 3 with the level-climb skip, tools/hotbench/hotbench2.cu, profiles/r02s2_rates.txt; C = 5 not measured in isolation)"}
            _log(f"c5: {name} {out[name]}")
        if world > 1:  # plan-sharded over the GPUs (fmdp_schedule_p2p); every rank takes part
            from paper_2008_03518_b200.fmdp import p2p_connect_group
            e = {"ranks": world}
            try:
                p2p_connect_group(c)
                for cull in (0, 1):
                    c.set_launch(cull=cull)
                    try:
                        r = c.schedule_p2p(sc5.src[0], sc5.dst[0], int(sc5.t0[0]), want_traj=False)
                        st = c.stats()
                        t, steps, status = st["device_ms"], st["steps"], r.status
                    except Exception as ex:  # noqa: BLE001 -- reported in the JSON line
                        t, steps, status = float("nan"), 0, str(ex)
                    t = max_over_ranks(t, world)
                    c.truncate(P)
                    e["culled" if cull else "full"] = {"us_per_step": t * 1e3 / max(1, steps), "steps": steps,
                                                       "status": status}
            except Exception as ex:  # noqa: BLE001
                e["error"] = str(ex)
            out["p2p"] = e
            _log(f"c5: p2p {e}")
        c.close()
        return out

    if args.only_c4:
        out = {"c3_growth": measure_c3() if rank == 0 else None, "c4_sharded": measure_c4(),
               "c4_full_size": measure_c4_full() if rank == 0 else None,
               "f4_a1350": measure_f4() if rank == 0 else None, "c5_stress": measure_c5()}
        if args.c5_full and rank == 0:
            out["c5_full_size"] = measure_c5_full()
        if rank == 0:
            print(json.dumps(out), flush=True)
        return 0
    _log("configs[1] batch, full path")
    M = measure(0)       # every (state, well) pair evaluated
    _log("configs[1] batch, f1 culling")
    Mc = measure(1)      # exact culling, bit-identical outputs
    _log("f3 departures")
    Md = measure_departures()
    _log("f2 co-simulation")
    Mco = measure_cosim()
    _log("latency vs plans")
    Mlat = measure_latency()
    _log("f4 A = 1350")
    Mf4 = measure_f4() if rank == 0 else None
    _log("configs[2] sequential growth")
    Mc3 = None if (args.no_c4 or rank != 0) else measure_c3()  # no collectives: rank 0 only
    _log("configs[3] sharded latency")
    Mc4 = None if args.no_c4 else measure_c4()
    _log("configs[3] full size")
    Mc4f = None if (args.no_c4 or rank != 0) else measure_c4_full()
    _log("configs[4] roofline stress")
    Mc5 = None if args.no_c4 else measure_c5()
    h2d = n * C_REQUEST_BYTES
    tot_ms, value, e2e_value, d2h = M["tot_ms"], M["value"], M["e2e_value"], M["d2h"]
    stats = M["st_all"][-1]
    walk_ms, pairs, launches, steps_dev = M["walk_ms"], M["pairs"], M["launches"], M["steps_dev"]
    res_last = M["res_last"]
    acc = sum(r.accepted for r in res_last)
    states = sum(r.n_states for r in res_last)
    clocks = M["clocks"]
    same = all(a.status == b.status and a.n_states == b.n_states for a, b in zip(M["res_last"], Mc["res_last"]))
    peak_clock = 1965.0
    try:
        mp = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        peak_clock = float(mp.get("sm_max_mhz", peak_clock))
    except Exception:
        pass
    peak_tops = 148 * 128 * peak_clock * 1e6 / 1e12
    traffic = None
    traffic_src = None
    for tname in ("r02_traffic.json", "r01_traffic.json"):  # dram read+write bytes per walk launch
        try:                                                 # from the committed ncu --set full capture
            traffic = json.load(open(os.path.join(ROOT, "profiles", tname)))["per_launch_bytes"]
            traffic_src = f"profiles/{tname} (ncu --set full, dram bytes per walk launch)"
            break
        except Exception:
            pass
    # roofline of the dominant kernel on the METHOD's work: pairs of the committed decision steps
    # (not the device counter, which includes speculative steps that were rolled back and the
    # paused walkers' extra steps); the executed-op and loop-ceiling fractions beside it
    A_, W_ = sc.airspace.n_actions, sc.airspace.W
    cpairs = committed_pairs(sc, res_last, A_, W_) * args.steps
    achieved_tops = cpairs * OPS_PER_PAIR / (walk_ms / 1e3) / 1e12 if walk_ms > 0 else 0.0
    exec_tops = pairs * EXEC_OPS_PER_PAIR / (walk_ms / 1e3) / 1e12 if walk_ms > 0 else 0.0
    loop_ceiling = LOOP_CEILING_PAIRS_PER_CLK_SM * 148 * peak_clock * 1e6  # pairs/s
    cpairs_c = committed_pairs(sc, Mc["res_last"], A_, W_) * args.steps
    if rank != 0:
        return 0
    line = {
        "metric": METRIC, "value": value, "unit": "requests/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tot_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD, "plans": len(sc.plans), "requests": n, "terrain_wells": int(len(sc.terrain.radius)),
                   "actions": sc.airspace.n_actions, "W": sc.airspace.W, "l2": "flushed between steps (256 MB write)",
                   "parallelism": f"request-sharded{world} (one FCFS batch, fmdp_schedule_batch_dist)" if world > 1
                   else "single-gpu"},
        "ms_per_request": tot_ms / args.steps / n,
        "requests_accepted": acc, "acceptance_rate": acc / n,
        "near_ties_per_batch": sum(r.n_near_ties for r in res_last),
        "exact_band_rescans_per_batch": sum(r.n_exact for r in res_last),
        "states_per_request": states / n, "device_steps_per_batch": steps_dev / args.steps,
        "speculation_steps_ratio": steps_dev / args.steps / max(1, states),
        "action_plan_evals_per_s": pairs / 5.0 / sc.airspace.W / (tot_ms / 1e3) * world,
        "pair_evals_per_s": pairs / (tot_ms / 1e3) * world,
        "rounds": stats["rounds"], "reruns": stats["reruns"],
        "roofline": {"bound": "alu", "achieved": achieved_tops, "peak": peak_tops, "unit": "Top/s",
                     "frac": achieved_tops / peak_tops, "traffic": traffic,
                     "traffic_source": traffic_src,
                     "kernel": "walk_kernel<3, 0>", "ops_per_pair": OPS_PER_PAIR,
                     "ops_per_pair_basis": "algorithmic, SURVEY §8(d) d.3 (3 differences, 3 squares/fmas, 1 min)",
                     "committed_pairs_per_step": cpairs / args.steps,
                     "device_pairs_per_step": pairs / args.steps,
                     "speculation_overhead": pairs / max(1, cpairs),
                     "exec_pipe_frac": exec_tops / peak_tops, "exec_ops_per_pair": EXEC_OPS_PER_PAIR,
                     "loop_ceiling_frac": (cpairs / (walk_ms / 1e3)) / loop_ceiling if walk_ms > 0 else 0.0,
                     "loop_ceiling_pairs_per_clk_sm": LOOP_CEILING_PAIRS_PER_CLK_SM,
                     "loop_ceiling": "isolated hot loop (20 FFMA2 + 15 FMNMX3 + 10 LDS.128 per plan pair) "
                                     "at 38-40 pairs/clk/SM: the 3-register FFMA2 and the 3-input FMNMX3 share "
                                     "operand bandwidth (0.40 warp-instructions/clk/SMSP together; "
                                     "tools/hotbench/rates.cu + hotbench2.cu, profiles/r02s2_rates.txt)",
                     "peak_basis": f"FP32 pipe: 148 SM x 128 lanes x {peak_clock:.0f} MHz (MEASURED_PEAKS sm_max_mhz)"},
        "e2e": {"value": e2e_value, "unit": "requests/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clocks,
        "f1_cull": {
            "what": "SURVEY f1 exact culling of plans none of whose wells can reach a projected state; "
                    "outputs bit-identical (tests/test_gpu_parity.py::test_cull_*)",
            "value": Mc["value"], "unit": "requests/s", "ms_per_step": Mc["tot_ms"] / args.steps,
            "e2e": {"value": Mc["e2e_value"], "unit": "requests/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": Mc["d2h"]},
            "walk_device_ms_per_step": Mc["walk_ms"] / args.steps,
            "pair_evals_per_step": Mc["pairs"] / args.steps, "gpu_launches": Mc["launches"],
            "committed_pairs_per_step": cpairs_c / args.steps,
            "roofline_frac": cpairs_c * OPS_PER_PAIR / (Mc["walk_ms"] / 1e3) / 1e12 / peak_tops,
            "rounds": Mc["st_all"][-1]["rounds"], "reruns": Mc["st_all"][-1]["reruns"],
            "reconverged": Mc["st_all"][-1]["reconverged"],
            "device_steps_per_batch": Mc["steps_dev"] / args.steps,
            "speculation_steps_ratio": Mc["steps_dev"] / args.steps / max(1, sum(r.n_states for r in Mc["res_last"])),
            "reconverged_what": "rolled-back requests whose re-walk met their previous run and took it over "
                                "(DESIGN.md §6; tests/test_gpu_reuse.py: identical to the sequential loop)",
            "same_results_as_full": same, "clocks": Mc["clocks"]},
        "f3_departures": Md,
        "f2_cosim": Mco,
        "latency_vs_plans": Mlat,
    }
    if Mc3 is not None:
        line["c3_growth"] = Mc3
    if Mc4 is not None:
        line["c4_sharded"] = Mc4
    if Mc4f is not None:
        line["c4_full_size"] = Mc4f
    if args.c5_full and rank == 0:
        _log("configs[4] full size")
        line["c5_full_size"] = measure_c5_full()
    if Mf4 is not None:
        line["f4_a1350"] = Mf4
    if Mc5 is not None:
        line["c5_stress"] = Mc5
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(sc, args.cpu_sample_s, M["gpu_log"])
        line["divergent_steps"] = line["cpu_baseline"]["parity"]["divergent_steps"]
    print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()
    return 0


C_REQUEST_BYTES = 64  # sizeof(fmdp_request): u64 + 2 x 3 doubles + i64
C_RESULT_BYTES = 32   # sizeof(fmdp_result)


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_native(args)


if __name__ == "__main__":
    sys.exit(main())

"""Thin ctypes binding of libfmdp.so (include/fmdp.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; there is no CPU
fallback -- constructing a context without the built library or without an sm_100
device raises.  PyTorch is used only for device memory (caching-allocator callbacks)
and streams.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .build import LIB

ABI_VERSION = 3  # include/fmdp.h FMDP_ABI_VERSION
ACCEPTED, REJ_CONFLICT, REJ_TERRAIN, REJ_TIMEOUT = 0, 1, 2, 3
STATUS_NAMES = {0: "ACCEPTED", 1: "REJ_CONFLICT", 2: "REJ_TERRAIN", 3: "REJ_TIMEOUT"}
BATCH_SEQUENTIAL = 1


class FmdpError(RuntimeError):
    pass


class Vec3(C.Structure):
    _fields_ = [("x", C.c_double), ("y", C.c_double), ("z", C.c_double)]


class QPos(C.Structure):
    _fields_ = [("x", C.c_int32), ("y", C.c_int32), ("z", C.c_int32)]


class Airspace(C.Structure):
    _fields_ = [
        ("abi_version", C.c_uint32), ("lo", Vec3), ("hi", Vec3), ("u_m", C.c_double), ("dt", C.c_double),
        ("window", C.c_int32), ("speed", C.c_double), ("heading_lattice", C.c_int32),
        ("n_turn", C.c_int32), ("turn_steps", C.POINTER(C.c_int32)),
        ("n_climb", C.c_int32), ("climb_units", C.POINTER(C.c_int32)),
        ("goal_r", C.c_double), ("goal_gamma", C.c_double), ("intr_r", C.c_double), ("intr_gamma", C.c_double),
        ("n_tau", C.c_int32), ("tau_s", C.POINTER(C.c_double)), ("tau_radius_m", C.POINTER(C.c_double)),
        ("terr_r", C.c_double), ("terr_gamma", C.c_double), ("deck_alt_m", C.c_double), ("deck_scale", C.c_double),
        ("capture_radius_m", C.c_double), ("sep_min_m", C.c_double),
        ("max_steps", C.c_int32), ("vmax_init_zero", C.c_int32), ("near_tie_rel", C.c_double),
        ("horizon_steps", C.c_int64), ("row_capacity", C.c_int32), ("valuation", C.c_int32),
        ("n_acc", C.c_int32), ("acc_units", C.POINTER(C.c_int32)), ("speed_min", C.c_double),
        ("speed_max", C.c_double),
    ]


class Terrain(C.Structure):
    _fields_ = [("n_wells", C.c_int32), ("center", C.c_void_p), ("radius_u", C.c_void_p),
                ("nx", C.c_int32), ("ny", C.c_int32), ("x0_u", C.c_int32), ("y0_u", C.c_int32),
                ("cell_u", C.c_int32), ("height_u", C.c_void_p)]


ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
RELEASE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)


class Devices(C.Structure):
    _fields_ = [("device", C.c_int32), ("stream", C.c_void_p), ("alloc", ALLOC_FN), ("release", RELEASE_FN),
                ("user", C.c_void_p)]


class Launch(C.Structure):
    _fields_ = [("cluster_size", C.c_int32), ("max_walkers", C.c_int32), ("threads", C.c_int32),
                ("profile", C.c_int32), ("step_budget", C.c_int32), ("cull", C.c_int32), ("split", C.c_int32)]


class Request(C.Structure):
    _fields_ = [("aircraft_id", C.c_uint64), ("src", Vec3), ("dst", Vec3), ("t0_step", C.c_int64)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("plan_id", C.c_uint32), ("n_states", C.c_int32), ("fail_step", C.c_int32),
                ("min_sep_m", C.c_double), ("n_near_ties", C.c_int32), ("n_exact", C.c_int32)]


ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.POINTER(C.c_uint32), C.c_int32, C.c_void_p)


GATHER_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)


class Gather(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("allgather", GATHER_FN), ("user", C.c_void_p)]


class Shard(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("allreduce_min_u32", ALLREDUCE_FN), ("user", C.c_void_p)]


class P2PHandle(C.Structure):
    _fields_ = [("bytes", C.c_ubyte * 64)]


class Stats(C.Structure):
    _fields_ = [("steps", C.c_int64), ("pair_evals", C.c_int64), ("rounds", C.c_int32), ("reruns", C.c_int32),
                ("cluster_size", C.c_int32), ("walkers", C.c_int32), ("kernels", C.c_int32),
                ("device_ms", C.c_double), ("phase_cycles", C.c_int64 * 17), ("split", C.c_int32),
                ("reconverged", C.c_int32)]

PHASES = ("projection", "goal_terrain", "row_wait", "hot_loop", "stage", "reduce_scatter", "barrier1",
          "owner_epilogue", "barrier2", "decide", "top", "tscan", "proj_loop", "build", "own_classify", "argmax", "flags")


EXPORTS = ["fmdp_airspace_default", "fmdp_create", "fmdp_destroy", "fmdp_set_launch", "fmdp_add_plan",
           "fmdp_add_plans", "fmdp_schedule", "fmdp_schedule_batch", "fmdp_schedule_sharded",
           "fmdp_p2p_export", "fmdp_p2p_connect", "fmdp_schedule_p2p",
           "fmdp_schedule_departures", "fmdp_schedule_cosim", "fmdp_cosim_max", "fmdp_get_steplog", "fmdp_get_plan",
           "fmdp_num_plans", "fmdp_truncate", "fmdp_eval_step", "fmdp_get_stats", "fmdp_num_actions",
           "fmdp_strerror", "fmdp_last_error", "fmdp_set_trace", "fmdp_get_trace", "fmdp_get_speeds",
           "fmdp_eval_step_v", "fmdp_schedule_batch_dist", "fmdp_save_plans", "fmdp_load_plans"]

_lib = None


def lib():
    """Load the in-tree libfmdp.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        path = os.environ.get("FMDP_LIB_VARIANT") or LIB  # A/B builds of the same sources (tools/ab_variants.py)
        if not os.path.exists(path):
            raise FmdpError(f"{path} not built: run paper_2008_03518_b200.build.build() (nvcc, sm_100a)")
        L = C.CDLL(path)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.fmdp_airspace_default.argtypes = [C.POINTER(Airspace)]
        L.fmdp_airspace_default.restype = None
        L.fmdp_create.argtypes = [C.POINTER(Airspace), C.POINTER(Terrain), C.POINTER(Devices), C.POINTER(vp)]
        L.fmdp_destroy.argtypes = [vp]
        L.fmdp_destroy.restype = None
        L.fmdp_set_launch.argtypes = [vp, C.POINTER(Launch)]
        L.fmdp_add_plan.argtypes = [vp, C.c_uint64, i64, i32, vp, i32, C.POINTER(C.c_uint32)]
        L.fmdp_add_plans.argtypes = [vp, i32, vp, vp, vp, vp, C.POINTER(C.c_uint32)]
        L.fmdp_schedule.argtypes = [vp, C.c_uint64, Vec3, Vec3, i64, C.POINTER(Result), vp, i32]
        L.fmdp_schedule_batch.argtypes = [vp, vp, i32, vp, vp, i32, i32]
        L.fmdp_schedule_departures.argtypes = [vp, C.c_uint64, Vec3, Vec3, i64, i32, vp, vp, vp, i32, C.POINTER(i32)]
        L.fmdp_schedule_cosim.argtypes = [vp, vp, i32, vp, vp, i32]
        L.fmdp_cosim_max.argtypes = [vp]
        L.fmdp_cosim_max.restype = i32
        L.fmdp_schedule_sharded.argtypes = [vp, C.POINTER(Shard), C.c_uint64, Vec3, Vec3, i64, C.POINTER(Result), vp,
                                            i32]
        L.fmdp_p2p_export.argtypes = [vp, i32, C.POINTER(P2PHandle), C.POINTER(vp)]
        L.fmdp_p2p_connect.argtypes = [vp, i32, i32, vp, vp]
        L.fmdp_schedule_p2p.argtypes = [vp, C.c_uint64, Vec3, Vec3, i64, C.POINTER(Result), vp, i32]
        L.fmdp_get_steplog.argtypes = [vp, i32, vp, vp, vp, i32, C.POINTER(i32)]
        L.fmdp_set_trace.argtypes = [vp, i32]
        L.fmdp_schedule_batch_dist.argtypes = [vp, C.POINTER(Gather), vp, i32, vp, vp, i32]
        L.fmdp_get_speeds.argtypes = [vp, i32, vp, i32, C.POINTER(i32)]
        L.fmdp_get_trace.argtypes = [vp, i32, vp, vp, i32, C.POINTER(i32)]
        L.fmdp_get_plan.argtypes = [vp, C.c_uint32, C.POINTER(i64), vp, i32, C.POINTER(i32)]
        L.fmdp_num_plans.argtypes = [vp, C.POINTER(C.c_uint32)]
        L.fmdp_truncate.argtypes = [vp, C.c_uint32]
        L.fmdp_save_plans.argtypes = [vp, C.c_char_p, C.c_uint32]
        L.fmdp_load_plans.argtypes = [vp, C.c_char_p, C.POINTER(C.c_uint32)]
        L.fmdp_eval_step.argtypes = [vp, QPos, i32, QPos, i64, vp, vp, vp, vp, vp, vp]
        L.fmdp_eval_step_v.argtypes = [vp, QPos, i32, i32, QPos, i64, vp, vp, vp, vp, vp, vp]
        L.fmdp_get_stats.argtypes = [vp, C.POINTER(Stats)]
        L.fmdp_num_actions.argtypes = [vp]
        L.fmdp_num_actions.restype = i32
        L.fmdp_strerror.argtypes = [i32]
        L.fmdp_strerror.restype = C.c_char_p
        L.fmdp_last_error.argtypes = [vp]
        L.fmdp_last_error.restype = C.c_char_p
        _lib = L
    return _lib


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class ScheduleResult:
    status: int
    plan_id: int
    n_states: int
    fail_step: int
    min_sep_m: float
    n_near_ties: int
    n_exact: int
    traj: Optional[np.ndarray] = None     # [n,3] int32 units

    @property
    def accepted(self) -> bool:
        return self.status == ACCEPTED


class FMDP:
    """One FCFS context (scenario, terrain, accepted-plan store) on one sm_100 device."""

    def __init__(self, airspace, terrain=None, device: int = 0, torch_alloc: bool = True, stream=None):
        self.L = lib()
        self._keep = []
        a = Airspace()
        self.L.fmdp_airspace_default(C.byref(a))
        self.u_m = float(airspace.u_m)
        arr_i = lambda v: np.ascontiguousarray(v, np.int32)
        arr_d = lambda v: np.ascontiguousarray(v, np.float64)
        turn, climb = arr_i(airspace.turn_steps), arr_i(airspace.climb_units)
        acc = arr_i(getattr(airspace, "acc_units", (0,)))
        tau, rad = arr_d(airspace.tau_s), arr_d(airspace.tau_radius_m)
        self._keep += [turn, climb, tau, rad, acc]
        a.abi_version = ABI_VERSION
        a.lo = Vec3(*airspace.lo_m)
        a.hi = Vec3(*airspace.hi_m)
        a.u_m, a.dt, a.window, a.speed = airspace.u_m, airspace.dt_s, airspace.W, airspace.speed_mps
        a.heading_lattice = airspace.HL
        a.n_turn, a.turn_steps = len(turn), turn.ctypes.data_as(C.POINTER(C.c_int32))
        a.n_climb, a.climb_units = len(climb), climb.ctypes.data_as(C.POINTER(C.c_int32))
        a.goal_r, a.goal_gamma = airspace.goal_r, airspace.goal_gamma
        a.intr_r, a.intr_gamma = airspace.intr_r, airspace.intr_gamma
        a.n_tau = len(tau)
        a.tau_s = tau.ctypes.data_as(C.POINTER(C.c_double))
        a.tau_radius_m = rad.ctypes.data_as(C.POINTER(C.c_double))
        a.terr_r, a.terr_gamma = airspace.terr_r, airspace.terr_gamma
        a.deck_alt_m, a.deck_scale = airspace.deck_alt_m, airspace.deck_scale
        a.capture_radius_m, a.sep_min_m = airspace.capture_m, airspace.sep_m
        a.max_steps, a.vmax_init_zero, a.near_tie_rel = airspace.max_steps, airspace.vmax_init_zero, airspace.near_tie_rel
        a.horizon_steps, a.row_capacity = airspace.horizon_steps, airspace.row_capacity
        a.valuation = getattr(airspace, "valuation", 0)
        a.n_acc, a.acc_units = len(acc), acc.ctypes.data_as(C.POINTER(C.c_int32))
        a.speed_min = float(getattr(airspace, "speed_min_mps", 0.0))
        a.speed_max = float(getattr(airspace, "speed_max_mps", 0.0))
        self.max_steps = int(airspace.max_steps)
        self.W = int(airspace.W)
        t = Terrain()
        if terrain is not None and (len(terrain.radius) or terrain.nx):
            cen = np.ascontiguousarray(terrain.center, np.int32)
            r = np.ascontiguousarray(terrain.radius, np.int32)
            h = np.ascontiguousarray(terrain.height, np.int32)
            self._keep += [cen, r, h]
            t.n_wells, t.center, t.radius_u = len(r), _p(cen), _p(r)
            t.nx, t.ny, t.x0_u, t.y0_u, t.cell_u = terrain.nx, terrain.ny, terrain.x0, terrain.y0, terrain.cell
            t.height_u = _p(h) if h.size else None
        d = Devices()
        d.device = device
        d.stream = None
        if torch_alloc and stream is None:
            # blocks from torch's caching allocator are stream-ordered: the library must run on the
            # stream they are allocated for, so the context gets its own torch stream (never
            # torch's current stream, whose pending kernels a non-blocking library stream would
            # not be ordered against)
            import torch
            stream = torch.cuda.Stream(device=device)
        self._stream = stream
        if stream is not None:
            d.stream = C.c_void_p(int(getattr(stream, "cuda_stream", stream)))
        if torch_alloc:
            import torch  # plumbing only: device memory from torch's caching allocator
            dev = torch.device("cuda", device)
            tstream = stream

            def _alloc(nbytes, user):
                return int(torch.cuda.caching_allocator_alloc(int(nbytes), device=dev, stream=tstream))

            def _release(ptr, user):
                try:
                    torch.cuda.caching_allocator_delete(int(ptr))
                except Exception:  # interpreter shutdown: torch already torn down
                    pass

            self._alloc_cb, self._release_cb = ALLOC_FN(_alloc), RELEASE_FN(_release)
            d.alloc, d.release = self._alloc_cb, self._release_cb
        self.ctx = C.c_void_p()
        rc = self.L.fmdp_create(C.byref(a), C.byref(t), C.byref(d), C.byref(self.ctx))
        if rc != 0:
            why = self.L.fmdp_last_error(None).decode()
            self.ctx = None
            raise FmdpError(f"fmdp_create failed: {self.L.fmdp_strerror(rc).decode()} ({rc}) {why}")
        self.A = int(self.L.fmdp_num_actions(self.ctx))

    # ------------------------------------------------------------------ plumbing
    def _check(self, rc, what):
        if rc != 0:
            msg = self.L.fmdp_last_error(self.ctx).decode() if self.ctx else ""
            raise FmdpError(f"{what}: {self.L.fmdp_strerror(rc).decode()} ({rc}) {msg}")

    def close(self):
        if getattr(self, "ctx", None):
            self.L.fmdp_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_launch(self, cluster_size=0, max_walkers=0, threads=0, profile=0, step_budget=0, cull=0, split=0):
        l = Launch(cluster_size, max_walkers, threads, profile, step_budget, cull, split)
        self._check(self.L.fmdp_set_launch(self.ctx, C.byref(l)), "fmdp_set_launch")

    # ------------------------------------------------------------------ store
    def add_plans(self, plans: Sequence[Tuple[int, np.ndarray]], aircraft_ids=None) -> int:
        if not plans:
            return self.num_plans()
        return self.add_plans_packed(*pack_plans(plans), aircraft_ids=aircraft_ids)

    def add_plans_packed(self, t0: np.ndarray, n: np.ndarray, st: np.ndarray, aircraft_ids=None) -> int:
        """add_plans from ``pack_plans`` arrays (t0[P] int64, n[P] int32, states[sum n][3] int32)."""
        t0 = np.ascontiguousarray(t0, np.int64)
        n = np.ascontiguousarray(n, np.int32)
        st = np.ascontiguousarray(st, np.int32)
        ids = None if aircraft_ids is None else np.ascontiguousarray(aircraft_ids, np.uint64)
        first = C.c_uint32()
        self._check(self.L.fmdp_add_plans(self.ctx, len(t0), _p(ids), _p(t0), _p(n), _p(st), C.byref(first)),
                    "fmdp_add_plans")
        return int(first.value)

    def add_plan(self, t0: int, states: np.ndarray, aircraft_id: int = 0) -> int:
        st = np.ascontiguousarray(states, np.int32)
        pid = C.c_uint32()
        self._check(self.L.fmdp_add_plan(self.ctx, aircraft_id, int(t0), len(st), _p(st), 0, C.byref(pid)),
                    "fmdp_add_plan")
        return int(pid.value)

    def num_plans(self) -> int:
        n = C.c_uint32()
        self._check(self.L.fmdp_num_plans(self.ctx, C.byref(n)), "fmdp_num_plans")
        return int(n.value)

    def get_plan(self, plan_id: int):
        t0 = C.c_int64()
        n = C.c_int32()
        self._check(self.L.fmdp_get_plan(self.ctx, plan_id, C.byref(t0), None, 0, C.byref(n)), "fmdp_get_plan")
        buf = np.zeros((n.value, 3), np.int32)
        self._check(self.L.fmdp_get_plan(self.ctx, plan_id, C.byref(t0), _p(buf), n.value, C.byref(n)), "fmdp_get_plan")
        return int(t0.value), buf

    def truncate(self, n_plans: int):
        self._check(self.L.fmdp_truncate(self.ctx, int(n_plans)), "fmdp_truncate")

    def save_plans(self, path, first_id: int = 0):
        """Write plans [first_id, num_plans) to `path` (include/fmdp.h fmdp_save_plans)."""
        self._check(self.L.fmdp_save_plans(self.ctx, os.fsencode(path), int(first_id)), "fmdp_save_plans")

    def load_plans(self, path) -> int:
        """Append every plan of a plan-store file; returns the first new plan id."""
        fid = C.c_uint32()
        self._check(self.L.fmdp_load_plans(self.ctx, os.fsencode(path), C.byref(fid)), "fmdp_load_plans")
        return int(fid.value)

    # ------------------------------------------------------------------ requests
    def _vec(self, q_units):
        q = np.asarray(q_units, np.float64) * self.u_m   # exact: u = 2^-6
        return Vec3(float(q[0]), float(q[1]), float(q[2]))

    def schedule(self, src, dst, t0: int, aircraft_id: int = 0, want_traj: bool = True) -> ScheduleResult:
        """src/dst in integer units (as generated); converted exactly to metres for the ABI."""
        cap = self.max_steps + 1
        traj = np.zeros((cap, 3), np.int32) if want_traj else None
        r = Result()
        self._check(self.L.fmdp_schedule(self.ctx, aircraft_id, self._vec(src), self._vec(dst), int(t0), C.byref(r),
                                         _p(traj), cap), "fmdp_schedule")
        return self._res(r, traj)

    def _res(self, r, traj):
        return ScheduleResult(r.status, r.plan_id, r.n_states, r.fail_step, r.min_sep_m, r.n_near_ties, r.n_exact,
                              None if traj is None else traj[:r.n_states].copy())

    def make_requests(self, src, dst, t0, aircraft_ids=None):
        n = len(t0)
        reqs = (Request * n)()
        for i in range(n):
            reqs[i].aircraft_id = int(aircraft_ids[i]) if aircraft_ids is not None else i
            reqs[i].src = self._vec(src[i])
            reqs[i].dst = self._vec(dst[i])
            reqs[i].t0_step = int(t0[i])
        return reqs

    def schedule_batch(self, src, dst, t0, sequential: bool = False, want_traj: bool = True,
                       reqs=None) -> List[ScheduleResult]:
        if reqs is None:
            reqs = self.make_requests(src, dst, t0)
        n = len(reqs)
        res = (Result * n)()
        cap = self.max_steps + 1
        traj = np.zeros((n, cap, 3), np.int32) if want_traj else None
        self._check(self.L.fmdp_schedule_batch(self.ctx, C.cast(reqs, C.c_void_p), n, C.cast(res, C.c_void_p),
                                               _p(traj), cap, BATCH_SEQUENTIAL if sequential else 0),
                    "fmdp_schedule_batch")
        return [self._res(res[i], None if traj is None else traj[i]) for i in range(n)]

    def schedule_batch_dist(self, src, dst, t0, allgather, rank: int, world: int, want_traj: bool = True,
                            reqs=None) -> List[ScheduleResult]:
        """Request-sharded FCFS batch (SURVEY §8(e) second partitioning; collective over the ranks):
        ``allgather(block: bytes) -> list of world equal-size bytes blocks in rank order`` (see
        ``allgather_torch``).  Every rank returns the full results, identical to schedule_batch."""
        def _cb(send, recv, nbytes, user):
            try:
                blk = C.string_at(send, nbytes) if nbytes else b""
                out = allgather(blk)
                if len(out) != world or any(len(b) != nbytes for b in out):
                    return 1
                C.memmove(recv, b"".join(out), nbytes * world)
                return 0
            except Exception:  # reported as FMDP_E_INTERNAL
                return 1

        cb = GATHER_FN(_cb)
        g = Gather(int(rank), int(world), cb, None)
        if reqs is None:
            reqs = self.make_requests(src, dst, t0)
        n = len(reqs)
        res = (Result * n)()
        cap = self.max_steps + 1
        traj = np.zeros((n, cap, 3), np.int32) if want_traj else None
        self._check(self.L.fmdp_schedule_batch_dist(self.ctx, C.byref(g), C.cast(reqs, C.c_void_p), n,
                                                    C.cast(res, C.c_void_p), _p(traj), cap),
                    "fmdp_schedule_batch_dist")
        return [self._res(res[i], None if traj is None else traj[i]) for i in range(n)]

    def schedule_cosim(self, src, dst, t0, want_traj: bool = True, reqs=None) -> List[ScheduleResult]:
        """co-simulated batch (mutually aware, one clock); accepted plans appended in order."""
        if reqs is None:
            reqs = self.make_requests(src, dst, t0)
        n = len(reqs)
        res = (Result * n)()
        cap = self.max_steps + 1
        traj = np.zeros((n, cap, 3), np.int32) if want_traj else None
        self._check(self.L.fmdp_schedule_cosim(self.ctx, C.cast(reqs, C.c_void_p), n, C.cast(res, C.c_void_p),
                                               _p(traj), cap), "fmdp_schedule_cosim")
        return [self._res(res[i], None if traj is None else traj[i]) for i in range(n)]

    def cosim_max(self) -> int:
        return int(self.L.fmdp_cosim_max(self.ctx))

    def schedule_sharded(self, src, dst, t0: int, rank: int, world: int, allreduce_min, aircraft_id: int = 0,
                         want_traj: bool = True) -> ScheduleResult:
        """Plan-sharded request: this rank evaluates its shard of every time row;
        ``allreduce_min(np.ndarray[uint32])`` must replace the array in place by the elementwise
        minimum over all ranks (see ``allreduce_min_torch``).  Collective over the ranks."""
        def _cb(ptr, count, user):
            try:
                arr = np.ctypeslib.as_array(ptr, shape=(count,))
                allreduce_min(arr)
                return 0
            except Exception:  # reported as FMDP_E_INTERNAL
                return 1

        cb = ALLREDUCE_FN(_cb)
        sh = Shard(rank, world, cb, None)
        cap = self.max_steps + 1
        traj = np.zeros((cap, 3), np.int32) if want_traj else None
        r = Result()
        self._check(self.L.fmdp_schedule_sharded(self.ctx, C.byref(sh), aircraft_id, self._vec(src), self._vec(dst),
                                                 int(t0), C.byref(r), _p(traj), cap), "fmdp_schedule_sharded")
        return self._res(r, traj)

    def p2p_export(self, world: int):
        """Allocate this rank's in-kernel exchange area; returns (64-byte IPC handle, device pointer)."""
        h = P2PHandle()
        ptr = C.c_void_p()
        self._check(self.L.fmdp_p2p_export(self.ctx, int(world), C.byref(h), C.byref(ptr)), "fmdp_p2p_export")
        return bytes(h.bytes), int(ptr.value or 0)

    def p2p_connect(self, rank: int, world: int, handles, ptrs=None):
        """Attach the peers' exchange areas: ``ptrs[q]`` (same process) where given and non-zero,
        else the IPC handle ``handles[q]``."""
        hs = (P2PHandle * world)()
        for q, hb in enumerate(handles):
            C.memmove(hs[q].bytes, bytes(hb), 64)
        pp = (C.c_void_p * world)(*[(ptrs[q] or None) if ptrs is not None else None for q in range(world)])
        self._check(self.L.fmdp_p2p_connect(self.ctx, int(rank), int(world), C.cast(hs, C.c_void_p),
                                            C.cast(pp, C.c_void_p) if ptrs is not None else None),
                    "fmdp_p2p_connect")

    def schedule_p2p(self, src, dst, t0: int, aircraft_id: int = 0, want_traj: bool = True) -> ScheduleResult:
        """Plan-sharded request with the per-step exchange inside the walker kernel (SURVEY §8(e)
        production form).  Collective: every connected rank calls it with the same request."""
        cap = self.max_steps + 1
        traj = np.zeros((cap, 3), np.int32) if want_traj else None
        r = Result()
        self._check(self.L.fmdp_schedule_p2p(self.ctx, aircraft_id, self._vec(src), self._vec(dst), int(t0),
                                             C.byref(r), _p(traj), cap), "fmdp_schedule_p2p")
        return self._res(r, traj)

    def schedule_departures(self, src, dst, t0: int, delays, aircraft_id: int = 0, want_traj: bool = True):
        """candidate departures t0 + delays[i] in parallel against the current store;
        returns (results, chosen index or -1); the chosen candidate is appended."""
        d = np.ascontiguousarray(delays, np.int64)
        n = len(d)
        res = (Result * n)()
        cap = self.max_steps + 1
        traj = np.zeros((n, cap, 3), np.int32) if want_traj else None
        ch = C.c_int32()
        self._check(self.L.fmdp_schedule_departures(self.ctx, aircraft_id, self._vec(src), self._vec(dst), int(t0), n,
                                                    _p(d), C.cast(res, C.c_void_p), _p(traj), cap, C.byref(ch)),
                    "fmdp_schedule_departures")
        return [self._res(res[i], None if traj is None else traj[i]) for i in range(n)], int(ch.value)

    def steplog(self, index: int):
        n = C.c_int32()
        cap = self.max_steps + 2
        ast = np.zeros(cap, np.int32)
        hd = np.zeros(cap, np.int32)
        nt = np.zeros(cap, np.int32)
        self._check(self.L.fmdp_get_steplog(self.ctx, index, _p(ast), _p(hd), _p(nt), cap, C.byref(n)),
                    "fmdp_get_steplog")
        k = n.value
        return ast[:max(k - 1, 0)].copy(), hd[:k].copy(), nt[:max(k - 1, 0)].copy()

    def speeds(self, index: int):
        """Speed of every state (units per substep) of request `index` of the last call."""
        n = C.c_int32()
        cap = self.max_steps + 2
        sp = np.zeros(cap, np.int32)
        self._check(self.L.fmdp_get_speeds(self.ctx, int(index), _p(sp), cap, C.byref(n)), "fmdp_get_speeds")
        return sp[:n.value].copy()

    def set_trace(self, n_requests: int):
        """Record V*(a), S(a) of every decision step of the first n_requests of later calls."""
        self._check(self.L.fmdp_set_trace(self.ctx, int(n_requests)), "fmdp_set_trace")

    def trace(self, index: int):
        """(vstar[n_steps, A], scale[n_steps, A]) of request `index` of the last call."""
        n = C.c_int32()
        cap = self.max_steps + 2
        vs = np.zeros(cap * self.A, np.float64)
        sc = np.zeros(cap * self.A, np.float64)
        self._check(self.L.fmdp_get_trace(self.ctx, int(index), _p(vs), _p(sc), cap, C.byref(n)), "fmdp_get_trace")
        k = n.value
        return vs[:k * self.A].reshape(k, self.A), sc[:k * self.A].reshape(k, self.A)

    def eval_step(self, q, psi: int, goal, K: int, speed: int = 0):
        """One decision step (debug / parity hook); speed in units per substep (0: the airspace's)."""
        A, W = self.A, self.W
        vstar = np.zeros(A, np.float64)
        v = np.zeros(A * W, np.float64)
        s = np.zeros(A * W, np.float64)
        conf = np.zeros(A, np.int32)
        md2 = np.zeros(A + 1, np.int64)
        a = C.c_int32()
        self._check(self.L.fmdp_eval_step_v(self.ctx, QPos(*[int(x) for x in q]), int(psi), int(speed),
                                            QPos(*[int(x) for x in goal]), int(K), _p(vstar), _p(v), _p(s), _p(conf),
                                            _p(md2), C.byref(a)),
                    "fmdp_eval_step")
        return dict(vstar=vstar, v=v.reshape(A, W), scale=s.reshape(A, W), conflict=conf, min_d2=md2, a_star=a.value)

    def stats(self) -> dict:
        st = Stats()
        self._check(self.L.fmdp_get_stats(self.ctx, C.byref(st)), "fmdp_get_stats")
        out = {k: getattr(st, k) for k, _ in Stats._fields_ if k != "phase_cycles"}
        out["phase_cycles"] = {p: int(st.phase_cycles[i]) for i, p in enumerate(PHASES)}
        return out


def allreduce_min_torch(group=None, device=None):
    """Elementwise-MIN all-reduce of a uint32 host array over a torch.distributed group
    (plumbing for ``schedule_sharded``): NCCL when ``device`` is a CUDA device, else gloo."""
    import torch
    import torch.distributed as dist

    def f(arr: np.ndarray):
        t = torch.from_numpy(arr.astype(np.int64))
        if device is not None:
            t = t.to(device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        arr[:] = t.cpu().numpy().astype(np.uint32)
    return f


def allgather_torch(group=None, device=None):
    """All-gather of equal-size byte blocks over a torch.distributed group (plumbing for
    ``schedule_batch_dist``): NCCL when ``device`` is a CUDA device, else gloo."""
    import torch
    import torch.distributed as dist

    def f(block: bytes):
        world = dist.get_world_size(group)
        t = torch.frombuffer(bytearray(block), dtype=torch.uint8) if block else torch.zeros(0, dtype=torch.uint8)
        if device is not None:
            t = t.to(device)
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        return [bytes(o.cpu().numpy().tobytes()) for o in out]
    return f


def pack_plans(plans: Sequence[Tuple[int, np.ndarray]]):
    """(t0, n, states) arrays of a plan list, the layout fmdp_add_plans takes."""
    t0 = np.ascontiguousarray([p[0] for p in plans], np.int64)
    n = np.ascontiguousarray([len(p[1]) for p in plans], np.int32)
    st = np.ascontiguousarray(np.concatenate([np.asarray(p[1], np.int32).reshape(-1, 3) for p in plans]), np.int32)
    return t0, n, st


def p2p_connect_local(ctxs: Sequence["FMDP"]):
    """Connect contexts of THIS process (one per rank; on one or several devices) for
    ``schedule_p2p``: the peers' exchange areas are passed as device pointers."""
    world = len(ctxs)
    ex = [c.p2p_export(world) for c in ctxs]
    for r, c in enumerate(ctxs):
        c.p2p_connect(r, world, [h for h, _ in ex], [p for _, p in ex])


def p2p_connect_group(ctx: "FMDP", group=None):
    """Connect this process's context with the other ranks of a torch.distributed group (one
    process per GPU): exchange areas are shared by CUDA IPC handles (pointers when two ranks
    live in one process).  Collective; ends with an all-gather of every rank's outcome, so no
    rank schedules before all are connected, and a failure on any rank raises on all."""
    import os as _os
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    h, p = ctx.p2p_export(world)
    info = [None] * world
    dist.all_gather_object(info, (h, p, _os.getpid()), group=group)
    pid = _os.getpid()
    ptrs = [pp if (q == rank or ppid == pid) else 0 for q, (_, pp, ppid) in enumerate(info)]
    err = ""
    try:
        ctx.p2p_connect(rank, world, [hh for hh, _, _ in info], ptrs)
    except Exception as e:  # every rank learns of it below: no rank is left waiting in a collective
        err = f"rank {rank}: {e}"
    errs = [None] * world
    dist.all_gather_object(errs, err, group=group)
    bad = [e for e in errs if e]
    if bad:
        raise FmdpError("p2p_connect_group failed: " + "; ".join(bad))

"""ctypes wrapper of the C oracle (oracle/fmdp_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs.  The product package never imports it and it
never imports the product package; the only shared module is ``fmdp_synth`` (inputs).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "fmdp_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-std=gnu11", "-fPIC", "-shared", "-Wall"]

ACCEPTED, REJ_CONFLICT, REJ_TERRAIN, REJ_TIMEOUT = 0, 1, 2, 3
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "fmdp_oracle.h"))):
        cmd = ["gcc", *CFLAGS, "-o", LIB + ".tmp", SRC, "-lm"]
        subprocess.run(cmd, check=True)
        os.replace(LIB + ".tmp", LIB)
    return LIB


class Params(C.Structure):
    _fields_ = [
        ("u_m", C.c_double), ("dt_s", C.c_double), ("W", C.c_int32), ("HL", C.c_int32),
        ("speed_mps", C.c_double),
        ("n_turn", C.c_int32), ("turn_steps", C.c_int32 * 32),
        ("n_climb", C.c_int32), ("climb_units", C.c_int32 * 32),
        ("goal_r", C.c_double), ("goal_gamma", C.c_double),
        ("intr_r", C.c_double), ("intr_gamma", C.c_double),
        ("n_tau", C.c_int32), ("tau_s", C.c_double * 8), ("tau_radius_m", C.c_double * 8),
        ("terr_r", C.c_double), ("terr_gamma", C.c_double),
        ("deck_alt_m", C.c_double), ("deck_scale", C.c_double),
        ("capture_m", C.c_double), ("sep_m", C.c_double),
        ("max_steps", C.c_int32), ("vmax_init_zero", C.c_int32), ("near_tie_rel", C.c_double),
        ("valuation", C.c_int32),
        ("n_acc", C.c_int32), ("acc_units", C.c_int32 * 16), ("speed_min_mps", C.c_double),
        ("speed_max_mps", C.c_double),
    ]


class Terrain(C.Structure):
    _fields_ = [("n_wells", C.c_int32), ("center", C.c_void_p), ("radius", C.c_void_p),
                ("nx", C.c_int32), ("ny", C.c_int32), ("x0", C.c_int32), ("y0", C.c_int32),
                ("cell", C.c_int32), ("height", C.c_void_p)]


class StepOut(C.Structure):
    _fields_ = [("v_pos", C.c_void_p), ("v_int", C.c_void_p), ("v_ter", C.c_void_p), ("v_alt", C.c_void_p),
                ("v", C.c_void_p), ("scale", C.c_void_p), ("vstar", C.c_void_p), ("vstar_scale", C.c_void_p),
                ("conf_d2", C.c_void_p), ("proj", C.c_void_p), ("proj_psi", C.c_void_p),
                ("a_star", C.c_int32), ("a_second", C.c_int32), ("gap", C.c_double), ("near_tie", C.c_int32),
                ("v_neg", C.c_void_p), ("proj_v", C.c_void_p)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int32), ("n_states", C.c_int32), ("fail_step", C.c_int32),
                ("n_near_ties", C.c_int32), ("min_sep_d2", C.c_int64)]


class ReplayStats(C.Structure):
    _fields_ = [("n_steps_checked", C.c_int32), ("n_fail", C.c_int32), ("n_divergent", C.c_int32),
                ("n_near_ties", C.c_int32), ("first_fail_step", C.c_int32), ("max_vstar_err", C.c_double)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
            P = C.POINTER(Params)
            L.orc_check_params.argtypes = [P]
            L.orc_set_threads.argtypes = [C.c_int]
            L.orc_set_threads.restype = C.c_int
            L.orc_tables.argtypes = [P, vp, vp]
            L.orc_initial_heading.argtypes = [P, vp, vp]
            L.orc_initial_heading.restype = i32
            L.orc_build_wells.argtypes = [P, vp, vp, vp, vp]
            L.orc_project.argtypes = [P, vp, i32, vp, vp]
            L.orc_goal_value.argtypes = [P, i64]
            L.orc_goal_value.restype = C.c_double
            L.orc_well_value.argtypes = [C.c_double, C.c_double, C.c_double, i64, i64]
            L.orc_well_value.restype = C.c_double
            L.orc_deck_penalty.argtypes = [P, i32]
            L.orc_deck_penalty.restype = C.c_double
            L.orc_store_new.restype = vp
            L.orc_store_free.argtypes = [vp]
            L.orc_store_add.argtypes = [vp, i64, i32, vp]
            L.orc_store_count.argtypes = [vp]
            L.orc_store_count.restype = i32
            L.orc_store_sample.argtypes = [vp, i32, i64, vp, vp]
            L.orc_eval_step.argtypes = [P, C.POINTER(Terrain), vp, vp, i32, vp, i64, C.POINTER(StepOut)]
            L.orc_eval_step_peers.argtypes = [P, C.POINTER(Terrain), vp, vp, i32, vp, i64, i32, vp, vp,
                                              C.POINTER(StepOut)]
            L.orc_cosim.argtypes = [P, C.POINTER(Terrain), vp, i32, vp, vp, vp, i32, vp, vp, vp, C.POINTER(Result)]
            L.orc_cosim_replay.argtypes = [P, C.POINTER(Terrain), vp, i32, vp, vp, vp, i32, vp, vp, vp, vp, vp,
                                           C.POINTER(ReplayStats)]
            L.orc_schedule.argtypes = [P, C.POINTER(Terrain), vp, vp, vp, i64, i32, vp, vp, vp,
                                       C.POINTER(Result)]
            L.orc_schedule_v.argtypes = [P, C.POINTER(Terrain), vp, vp, vp, i64, i32, vp, vp, vp, vp,
                                         C.POINTER(Result)]
            L.orc_replay_v.argtypes = [P, C.POINTER(Terrain), vp, vp, vp, i64, i32, vp, vp, vp, vp, i32,
                                       C.POINTER(ReplayStats)]
            L.orc_eval_step_v.argtypes = [P, C.POINTER(Terrain), vp, vp, i32, i32, vp, i64, C.POINTER(StepOut)]
            L.orc_project_v.argtypes = [P, vp, i32, i32, vp, vp, vp]
            L.orc_initial_speed.argtypes = [P]
            L.orc_initial_speed.restype = i32
            L.orc_schedule_batch.argtypes = [P, C.POINTER(Terrain), vp, i32, vp, vp, vp, i32, vp, vp, vp,
                                             C.POINTER(Result)]
            L.orc_replay.argtypes = [P, C.POINTER(Terrain), vp, vp, vp, i64, i32, vp, vp, vp, i32,
                                     C.POINTER(ReplayStats)]
            _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def params_of(air) -> Params:
    p = Params()
    p.u_m, p.dt_s, p.W, p.HL, p.speed_mps = air.u_m, air.dt_s, air.W, air.HL, air.speed_mps
    p.n_turn = len(air.turn_steps)
    for i, v in enumerate(air.turn_steps):
        p.turn_steps[i] = v
    p.n_climb = len(air.climb_units)
    for i, v in enumerate(air.climb_units):
        p.climb_units[i] = v
    p.goal_r, p.goal_gamma = air.goal_r, air.goal_gamma
    p.intr_r, p.intr_gamma = air.intr_r, air.intr_gamma
    p.n_tau = len(air.tau_s)
    for i, (t, r) in enumerate(zip(air.tau_s, air.tau_radius_m)):
        p.tau_s[i], p.tau_radius_m[i] = t, r
    p.terr_r, p.terr_gamma = air.terr_r, air.terr_gamma
    p.deck_alt_m, p.deck_scale = air.deck_alt_m, air.deck_scale
    p.capture_m, p.sep_m = air.capture_m, air.sep_m
    p.max_steps, p.vmax_init_zero, p.near_tie_rel = air.max_steps, air.vmax_init_zero, air.near_tie_rel
    p.valuation = getattr(air, "valuation", 0)
    acc = tuple(getattr(air, "acc_units", (0,)))
    p.n_acc = len(acc)
    for i, v in enumerate(acc):
        p.acc_units[i] = v
    p.speed_min_mps = float(getattr(air, "speed_min_mps", 0.0))
    p.speed_max_mps = float(getattr(air, "speed_max_mps", 0.0))
    return p


@dataclass
class StepResult:
    v_pos: np.ndarray
    v_int: np.ndarray
    v_ter: np.ndarray
    v_alt: np.ndarray
    v_neg: np.ndarray
    v: np.ndarray
    scale: np.ndarray
    vstar: np.ndarray
    vstar_scale: np.ndarray
    conf_d2: np.ndarray
    proj: np.ndarray
    proj_psi: np.ndarray
    proj_v: np.ndarray
    a_star: int
    a_second: int
    gap: float
    near_tie: bool


@dataclass
class SchedResult:
    status: int
    n_states: int
    fail_step: int
    n_near_ties: int
    min_sep_d2: int
    traj: np.ndarray
    heading: np.ndarray
    astar: np.ndarray
    speed: np.ndarray = None


class Oracle:
    """One scenario (airspace + terrain) and one mutable accepted-plan store."""

    def __init__(self, airspace, terrain=None, plans=()):
        self.L = lib()
        self.air = airspace
        self.p = params_of(airspace)
        rc = self.L.orc_check_params(C.byref(self.p))
        if rc:
            raise ValueError(f"oracle rejects parameters ({rc})")
        self._keep = []
        self.T = Terrain()
        if terrain is not None and (len(terrain.radius) or terrain.nx):
            c = np.ascontiguousarray(terrain.center, np.int32)
            r = np.ascontiguousarray(terrain.radius, np.int32)
            h = np.ascontiguousarray(terrain.height, np.int32)
            self._keep += [c, r, h]
            self.T.n_wells, self.T.center, self.T.radius = len(r), _ptr(c), _ptr(r)
            self.T.nx, self.T.ny, self.T.x0, self.T.y0, self.T.cell = terrain.nx, terrain.ny, terrain.x0, terrain.y0, terrain.cell
            self.T.height = _ptr(h) if h.size else None
        self.S = self.L.orc_store_new()
        for t0, st in plans:
            self.add_plan(t0, st)

    def __del__(self):
        try:
            if getattr(self, "S", None):
                self.L.orc_store_free(self.S)
                self.S = None
        except Exception:
            pass

    @property
    def A(self):
        return self.air.n_actions

    def add_plan(self, t0: int, states: np.ndarray):
        st = np.ascontiguousarray(states, np.int32)
        rc = self.L.orc_store_add(self.S, int(t0), int(st.shape[0]), _ptr(st))
        if rc:
            raise ValueError(f"orc_store_add failed ({rc})")

    def n_plans(self) -> int:
        return self.L.orc_store_count(self.S)

    # ---- primitives -------------------------------------------------------
    def tables(self):
        DX = np.zeros(self.air.HL, np.int32)
        DY = np.zeros(self.air.HL, np.int32)
        assert self.L.orc_tables(C.byref(self.p), _ptr(DX), _ptr(DY)) == 0
        return DX, DY

    def initial_heading(self, src, dst) -> int:
        s = np.ascontiguousarray(src, np.int32)
        d = np.ascontiguousarray(dst, np.int32)
        return int(self.L.orc_initial_heading(C.byref(self.p), _ptr(s), _ptr(d)))

    def build_wells(self, pos, vel):
        p = np.ascontiguousarray(pos, np.int32)
        v = np.ascontiguousarray(vel, np.int32)
        c = np.zeros((len(self.air.tau_s), 3), np.int32)
        r = np.zeros(len(self.air.tau_s), np.int64)
        assert self.L.orc_build_wells(C.byref(self.p), _ptr(p), _ptr(v), _ptr(c), _ptr(r)) == 0
        return c, r

    def project(self, q, psi, v=None, with_speed=False):
        A, W = self.A, self.air.W
        st = np.zeros((A, W, 3), np.int32)
        ps = np.zeros((A, W), np.int32)
        sp = np.zeros((A, W), np.int32)
        qq = np.ascontiguousarray(q, np.int32)
        v = self.initial_speed() if v is None else int(v)
        assert self.L.orc_project_v(C.byref(self.p), _ptr(qq), int(psi), v, _ptr(st), _ptr(ps), _ptr(sp)) == 0
        return (st, ps, sp) if with_speed else (st, ps)

    def initial_speed(self) -> int:
        return int(self.L.orc_initial_speed(C.byref(self.p)))

    def goal_value(self, d2: int) -> float:
        return float(self.L.orc_goal_value(C.byref(self.p), int(d2)))

    def well_value(self, r, gamma, d2, R_u) -> float:
        return float(self.L.orc_well_value(float(r), float(gamma), float(self.air.u_m), int(d2), int(R_u)))

    def deck_penalty(self, z: int) -> float:
        return float(self.L.orc_deck_penalty(C.byref(self.p), int(z)))

    def sample(self, plan: int, K: int):
        pos = np.zeros(3, np.int32)
        vel = np.zeros(3, np.int32)
        ok = self.L.orc_store_sample(self.S, int(plan), int(K), _ptr(pos), _ptr(vel))
        return (pos, vel) if ok else None

    # ---- one decision step --------------------------------------------------
    def eval_step(self, q, psi, goal, K, peer_pos=None, peer_vel=None, v=None) -> StepResult:
        """Algs 2-9 at clock K; optional batch peers (Alg 5) as [n, 3] pos / vel;
        optional speed v (units per substep; acceleration actions, R32)."""
        A, W = self.A, self.air.W
        arr = {k: np.zeros(A * W, np.float64) for k in ("v_pos", "v_int", "v_ter", "v_alt", "v_neg", "v", "scale")}
        vstar = np.zeros(A, np.float64)
        vsc = np.zeros(A, np.float64)
        conf = np.zeros(A, np.int64)
        proj = np.zeros(A * W * 3, np.int32)
        pps = np.zeros(A * W, np.int32)
        pv_ = np.zeros(A * W, np.int32)
        o = StepOut()
        for k_, a_ in arr.items():
            setattr(o, k_, _ptr(a_))
        o.vstar, o.vstar_scale, o.conf_d2, o.proj, o.proj_psi = _ptr(vstar), _ptr(vsc), _ptr(conf), _ptr(proj), _ptr(pps)
        o.proj_v = _ptr(pv_)
        qq = np.ascontiguousarray(q, np.int32)
        gg = np.ascontiguousarray(goal, np.int32)
        npeer = 0 if peer_pos is None else len(peer_pos)
        pp = np.ascontiguousarray(np.reshape(peer_pos, (-1, 3)) if npeer else np.zeros((0, 3)), np.int32)
        pv = np.ascontiguousarray(np.reshape(peer_vel, (-1, 3)) if npeer else np.zeros((0, 3)), np.int32)
        if v is not None:
            assert npeer == 0, "speed-carrying steps are not co-simulated"
            rc = self.L.orc_eval_step_v(C.byref(self.p), C.byref(self.T), self.S, _ptr(qq), int(psi), int(v), _ptr(gg),
                                        int(K), C.byref(o))
        else:
            rc = self.L.orc_eval_step_peers(C.byref(self.p), C.byref(self.T), self.S, _ptr(qq), int(psi), _ptr(gg),
                                            int(K), npeer, _ptr(pp), _ptr(pv), C.byref(o))
        if rc:
            raise RuntimeError(f"orc_eval_step failed ({rc})")
        return StepResult(**{k: v.reshape(A, W) for k, v in arr.items()}, vstar=vstar, vstar_scale=vsc,
                          conf_d2=conf, proj=proj.reshape(A, W, 3), proj_psi=pps.reshape(A, W), proj_v=pv_.reshape(A, W),
                          a_star=o.a_star, a_second=o.a_second, gap=o.gap, near_tie=bool(o.near_tie))

    # ---- requests -----------------------------------------------------------
    def schedule(self, src, dst, t0, commit: bool = True) -> SchedResult:
        cap = self.air.max_steps + 2
        traj = np.zeros((cap, 3), np.int32)
        hd = np.zeros(cap, np.int32)
        sp = np.zeros(cap, np.int32)
        ast = np.full(cap, -1, np.int32)
        r = Result()
        s = np.ascontiguousarray(src, np.int32)
        d = np.ascontiguousarray(dst, np.int32)
        rc = self.L.orc_schedule_v(C.byref(self.p), C.byref(self.T), self.S, _ptr(s), _ptr(d), int(t0), cap,
                                   _ptr(traj), _ptr(hd), _ptr(sp), _ptr(ast), C.byref(r))
        if rc:
            raise RuntimeError(f"orc_schedule failed ({rc})")
        n = r.n_states
        out = SchedResult(r.status, n, r.fail_step, r.n_near_ties, r.min_sep_d2, traj[:n].copy(), hd[:n].copy(),
                          ast[:max(n - 1, 0)].copy(), sp[:n].copy())
        if commit and r.status == ACCEPTED:
            self.add_plan(int(t0), out.traj)
        return out

    def schedule_batch(self, src, dst, t0):
        return [self.schedule(src[i], dst[i], int(t0[i]), commit=True) for i in range(len(t0))]

    def replay(self, src, dst, t0, traj, heading, astar, status, speed=None) -> ReplayStats:
        st = ReplayStats()
        tr = np.ascontiguousarray(traj, np.int32)
        hd = np.ascontiguousarray(heading, np.int32)
        sp = None if speed is None else np.ascontiguousarray(speed, np.int32)
        ast = None if astar is None else np.ascontiguousarray(astar, np.int32)
        s = np.ascontiguousarray(src, np.int32)
        d = np.ascontiguousarray(dst, np.int32)
        rc = self.L.orc_replay_v(C.byref(self.p), C.byref(self.T), self.S, _ptr(s), _ptr(d), int(t0),
                                 int(tr.shape[0]), _ptr(tr), _ptr(hd), _ptr(sp), _ptr(ast), int(status), C.byref(st))
        if rc:
            raise RuntimeError(f"orc_replay failed ({rc})")
        return st


    # ---- co-simulated batch ------------------------------------
    def cosim(self, src, dst, t0):
        """Mutually aware batch on one clock (Alg 1 synchronous update, Alg 5); the store is
        not modified.  Returns one SchedResult per aircraft."""
        n = len(t0)
        cap = self.air.max_steps + 2
        traj = np.zeros((n, cap, 3), np.int32)
        hd = np.zeros((n, cap), np.int32)
        ast = np.full((n, cap), -1, np.int32)
        res = (Result * n)()
        s = np.ascontiguousarray(src, np.int32).reshape(n, 3)
        d = np.ascontiguousarray(dst, np.int32).reshape(n, 3)
        t = np.ascontiguousarray(t0, np.int64)
        rc = self.L.orc_cosim(C.byref(self.p), C.byref(self.T), self.S, n, _ptr(s), _ptr(d), _ptr(t), cap,
                              _ptr(traj), _ptr(hd), _ptr(ast), res)
        if rc:
            raise RuntimeError(f"orc_cosim failed ({rc})")
        out = []
        for i in range(n):
            r = res[i]
            m = r.n_states
            out.append(SchedResult(r.status, m, r.fail_step, r.n_near_ties, r.min_sep_d2, traj[i, :m].copy(),
                                   hd[i, :m].copy(), ast[i, :max(m - 1, 0)].copy()))
        return out

    def cosim_replay(self, src, dst, t0, trajs, headings, astars, statuses):
        """Replay a co-simulated batch produced elsewhere; one ReplayStats per aircraft."""
        n = len(t0)
        cap = max(len(x) for x in trajs) + 1
        traj = np.zeros((n, cap, 3), np.int32)
        hd = np.zeros((n, cap), np.int32)
        ast = np.full((n, cap), -1, np.int32)
        ns = np.zeros(n, np.int32)
        for i in range(n):
            m = len(trajs[i])
            ns[i] = m
            traj[i, :m] = trajs[i]
            hd[i, :m] = headings[i]
            if astars is not None:
                ast[i, :len(astars[i])] = astars[i]
        st = (ReplayStats * n)()
        s = np.ascontiguousarray(src, np.int32).reshape(n, 3)
        d = np.ascontiguousarray(dst, np.int32).reshape(n, 3)
        t = np.ascontiguousarray(t0, np.int64)
        status = np.ascontiguousarray(statuses, np.int32)
        rc = self.L.orc_cosim_replay(C.byref(self.p), C.byref(self.T), self.S, n, _ptr(s), _ptr(d), _ptr(t), cap,
                                     _ptr(ns), _ptr(traj), _ptr(hd), None if astars is None else _ptr(ast),
                                     _ptr(status), st)
        if rc:
            raise RuntimeError(f"orc_cosim_replay failed ({rc})")
        return [st[i] for i in range(n)]


def set_threads(n: int) -> int:
    """OpenMP threads of the oracle's per-state loops (host timing only; identical results)."""
    return int(lib().orc_set_threads(int(n)))


def for_scenario(sc, plans=True) -> Oracle:
    return Oracle(sc.airspace, sc.terrain, sc.plans if plans else ())

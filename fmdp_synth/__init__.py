"""Seeded synthetic inputs for the FastMDP-GPU hot path (shared by tests, bench and smoke).

This module is the ONLY code shared by the oracle side (``oracle/``) and the CUDA side
(``paper_2008_03518_b200/``).  It draws integer inputs -- accepted plans, terrain wells,
height raster, requests -- and holds none of the method's arithmetic (no wells, no
values, no projection, no predicates).

Recipe:
  * world in integer units of u = 2^-6 m; every length below is converted with an
    exact integer multiply;
  * accepted plans are *reflecting straight lines*: p(K) = fold(p0 + v*K) into the
    airspace box (triangle-wave fold per axis), speed U[30,60] m/s horizontal, small
    vertical rate -- the synthetic stand-in for the paper's FCFS-generated plans
    (S:487);
  * terrain = Manhattan building blocks (100 m pitch, 60 m footprint) with log-normal
    heights, one well per building at its rooftop with R = half-diagonal + 60 m, plus a
    10 m height raster for collision (Table PK: "manually placed ... manually
    selected");
  * requests fly between vertiport pads 60-120 m high (Table PK P:513 "Vertiport").
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field
from typing import List, Tuple

import numpy as np

U_PER_M = 64  # 1 m = 64 units; u = 2^-6 m (R23)


def m2u(x) -> np.ndarray:
    """Metres -> integer units (inputs are generated on the unit grid)."""
    return np.rint(np.asarray(x, dtype=np.float64) * U_PER_M).astype(np.int64)


@dataclass
class Airspace:
    """Scenario parameters in physical units (defaults: DESIGN.md Appendix A)."""
    u_m: float = 1.0 / U_PER_M
    dt_s: float = 0.1
    W: int = 10
    HL: int = 1440                       # heading lattice (0.25 deg)
    speed_mps: float = 50.0
    turn_steps: Tuple[int, ...] = (-8, -6, -4, -2, 0, 2, 4, 6, 8)
    climb_units: Tuple[int, ...] = (-16, 0, 16)
    goal_r: float = 200.0                # Table PK
    goal_gamma: float = 0.999
    intr_r: float = 1000.0               # Table PK
    intr_gamma: float = 0.97
    tau_s: Tuple[float, ...] = (-5.0, 0.0, 5.0, 10.0, 15.0)
    tau_radius_m: Tuple[float, ...] = (250.0, 300.0, 350.0, 400.0, 450.0)  # 300 + 10 t
    terr_r: float = 1000.0               # Table PK
    terr_gamma: float = 0.99
    deck_alt_m: float = 30.0
    deck_scale: float = 1000.0           # Alg 1
    capture_m: float = 100.0
    sep_m: float = 150.0
    max_steps: int = 4000
    vmax_init_zero: int = 0
    valuation: int = 0                   # 0 Alg 8 (max over the window), 1 Alg 1 endpoint
    near_tie_rel: float = 1e-4
    # acceleration actions (R32): speed increments in units per substep per
    # substep, speed clamped to [speed_min_mps, speed_max_mps] (both 0: constant speed_mps)
    acc_units: Tuple[int, ...] = (0,)
    speed_min_mps: float = 0.0
    speed_max_mps: float = 0.0
    # store geometry (library side only; the oracle ignores these)
    lo_m: Tuple[float, float, float] = (-8000.0, -8000.0, 0.0)
    hi_m: Tuple[float, float, float] = (8000.0, 8000.0, 1500.0)
    horizon_steps: int = 8192
    row_capacity: int = 4096

    @property
    def n_actions(self) -> int:
        return len(self.turn_steps) * len(self.acc_units) * len(self.climb_units)

    def replace(self, **kw) -> "Airspace":
        return dataclasses.replace(self, **kw)


@dataclass
class Terrain:
    center: np.ndarray = field(default_factory=lambda: np.zeros((0, 3), np.int32))  # [n,3] units
    radius: np.ndarray = field(default_factory=lambda: np.zeros((0,), np.int32))    # [n] units
    nx: int = 0
    ny: int = 0
    x0: int = 0
    y0: int = 0
    cell: int = 1
    height: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.int32))  # [ny,nx] units


@dataclass
class Scenario:
    airspace: Airspace
    terrain: Terrain
    plans: List[Tuple[int, np.ndarray]]          # (t0, states int32 [n,3])
    src: np.ndarray                              # [R,3] int32 units
    dst: np.ndarray                              # [R,3] int32 units
    t0: np.ndarray                               # [R] int64
    name: str = ""

    @property
    def n_requests(self) -> int:
        return int(self.src.shape[0])


# ---------------------------------------------------------------------------
# building blocks
# ---------------------------------------------------------------------------
def _fold(x: np.ndarray, lo: int, hi: int) -> np.ndarray:
    """Triangle-wave fold of integer coordinates into [lo, hi] (reflecting walls)."""
    L = hi - lo
    y = np.mod(x - lo, 2 * L)
    y = np.where(y > L, 2 * L - y, y)
    return lo + y


def reflecting_lines(rng: np.random.Generator, n: int, lo_u, hi_u, rows: Tuple[int, int],
                     speed_mps=(30.0, 60.0), vz_units=(-16, 16), z_lo_u=None, z_hi_u=None,
                     active=None) -> List[Tuple[int, np.ndarray]]:
    """n straight flights folded into the box; active over ``rows`` (or per-plan ranges)."""
    lo_u = np.asarray(lo_u, np.int64)
    hi_u = np.asarray(hi_u, np.int64)
    zlo = int(lo_u[2] if z_lo_u is None else z_lo_u)
    zhi = int(hi_u[2] if z_hi_u is None else z_hi_u)
    plans = []
    for j in range(n):
        p0 = np.array([rng.integers(lo_u[0], hi_u[0] + 1), rng.integers(lo_u[1], hi_u[1] + 1),
                       rng.integers(zlo, zhi + 1)], np.int64)
        sp = rng.uniform(*speed_mps) * 0.1 * U_PER_M          # units per 0.1 s step
        th = rng.uniform(0.0, 2.0 * np.pi)
        v = np.array([int(np.rint(sp * np.cos(th))), int(np.rint(sp * np.sin(th))),
                      int(rng.integers(vz_units[0], vz_units[1] + 1))], np.int64)
        if active is None:
            k0, k1 = rows
        else:
            k0, k1 = active[j]
        K = np.arange(k0, k1, dtype=np.int64)[:, None]
        raw = p0[None, :] + v[None, :] * (K - rows[0])
        st = np.empty_like(raw)
        st[:, 0] = _fold(raw[:, 0], int(lo_u[0]), int(hi_u[0]))
        st[:, 1] = _fold(raw[:, 1], int(lo_u[1]), int(hi_u[1]))
        st[:, 2] = _fold(raw[:, 2], zlo, zhi)
        plans.append((int(k0), st.astype(np.int32)))
    return plans


def reflecting_lines_fast(rng: np.random.Generator, n: int, lo_u, hi_u, rows: Tuple[int, int],
                          speed_mps=(30.0, 60.0), vz_units=(-16, 16), z_lo_u=None, z_hi_u=None,
                          chunk: int = 8192) -> List[Tuple[int, np.ndarray]]:
    """Vectorised reflecting lines (same recipe as reflecting_lines, all active over ``rows``);
    the returned state arrays are views into one [n, rows, 3] int32 block."""
    lo_u = np.asarray(lo_u, np.int64)
    hi_u = np.asarray(hi_u, np.int64)
    zlo = int(lo_u[2] if z_lo_u is None else z_lo_u)
    zhi = int(hi_u[2] if z_hi_u is None else z_hi_u)
    lo3 = np.array([lo_u[0], lo_u[1], zlo], np.int64)
    hi3 = np.array([hi_u[0], hi_u[1], zhi], np.int64)
    p0 = np.stack([rng.integers(lo3[d], hi3[d] + 1, size=n) for d in range(3)], axis=1)
    sp = rng.uniform(*speed_mps, size=n) * 0.1 * U_PER_M
    th = rng.uniform(0.0, 2.0 * np.pi, size=n)
    v = np.stack([np.rint(sp * np.cos(th)), np.rint(sp * np.sin(th)),
                  rng.integers(vz_units[0], vz_units[1] + 1, size=n)], axis=1).astype(np.int64)
    nk = rows[1] - rows[0]
    out = np.empty((n, nk, 3), np.int32)
    K = np.arange(nk, dtype=np.int64)[None, :, None]
    L = (hi3 - lo3)[None, None, :]
    for a in range(0, n, chunk):
        b = min(n, a + chunk)
        raw = p0[a:b, None, :] + v[a:b, None, :] * K - lo3[None, None, :]
        y = np.mod(raw, 2 * L)
        y = np.where(y > L, 2 * L - y, y)
        out[a:b] = (lo3[None, None, :] + y).astype(np.int32)
    return [(int(rows[0]), out[j]) for j in range(n)]


def manhattan_terrain(rng: np.random.Generator, n_buildings: int, core_half_m: float,
                      raster_half_m: float, pitch_m=100.0, block_m=60.0, cell_m=10.0) -> Terrain:
    """Building wells on a Manhattan grid + a height raster covering the airspace."""
    nb = int(2 * core_half_m // pitch_m)
    idx = rng.choice(nb * nb, size=n_buildings, replace=False)
    bx = (idx % nb).astype(np.float64)
    by = (idx // nb).astype(np.float64)
    cx_m = -core_half_m + (bx + 0.5) * pitch_m
    cy_m = -core_half_m + (by + 0.5) * pitch_m
    h_m = np.clip(np.exp(rng.normal(np.log(40.0), 0.6, size=n_buildings)), 15.0, 200.0)
    h_m = np.rint(h_m)
    R_m = np.rint(block_m / np.sqrt(2.0) + 60.0)
    center = np.stack([m2u(cx_m), m2u(cy_m), m2u(h_m)], axis=1).astype(np.int32)
    radius = np.full((n_buildings,), int(m2u(R_m)), np.int32)
    cell_u = int(m2u(cell_m))
    n = int(round(2 * raster_half_m / cell_m))
    x0 = int(m2u(-raster_half_m))
    height = np.zeros((n, n), np.int32)
    half_cells = int(round(block_m / cell_m / 2))
    for i in range(n_buildings):
        ix = int((m2u(cx_m[i]) - x0) // cell_u)
        iy = int((m2u(cy_m[i]) - x0) // cell_u)
        height[max(iy - half_cells, 0):iy + half_cells, max(ix - half_cells, 0):ix + half_cells] = center[i, 2]
    return Terrain(center=center, radius=radius, nx=n, ny=n, x0=x0, y0=x0, cell=cell_u, height=height)


def vertiports(rng: np.random.Generator, n: int, half_m: float, terrain: Terrain) -> np.ndarray:
    """Pads 60-120 m high on ground cells lower than the pad."""
    out = []
    while len(out) < n:
        x = int(m2u(rng.uniform(-half_m, half_m)))
        y = int(m2u(rng.uniform(-half_m, half_m)))
        z = int(m2u(rng.integers(60, 121)))
        if terrain.nx:
            ix = (x - terrain.x0) // terrain.cell
            iy = (y - terrain.y0) // terrain.cell
            if 0 <= ix < terrain.nx and 0 <= iy < terrain.ny and terrain.height[iy, ix] >= z - int(m2u(20)):
                continue
        out.append((x, y, z))
    return np.asarray(out, np.int32)


def request_pairs(rng: np.random.Generator, pads: np.ndarray, n: int, dmin_m: float, dmax_m: float,
                  t0_range: Tuple[int, int]):
    src, dst = [], []
    while len(src) < n:
        i, j = rng.integers(0, len(pads), size=2)
        d = np.linalg.norm((pads[i] - pads[j]).astype(np.float64)) / U_PER_M
        if i == j or not (dmin_m <= d <= dmax_m):
            continue
        src.append(pads[i])
        dst.append(pads[j])
    t0 = rng.integers(t0_range[0], t0_range[1], size=n).astype(np.int64)
    return np.asarray(src, np.int32), np.asarray(dst, np.int32), t0


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------
def config_c1(seed: int = 1) -> Scenario:
    """configs[0]: 1 request, 10 plans, 2x2 km x [0,300] m, no terrain, 9x3 actions, 200 steps."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=200, lo_m=(-1000.0, -1000.0, 0.0), hi_m=(1000.0, 1000.0, 300.0),
                 horizon_steps=512, row_capacity=64)
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    plans = reflecting_lines(rng, 10, lo, hi, (0, 400), z_lo_u=int(m2u(80)), z_hi_u=int(m2u(120)))
    src = np.asarray([m2u((-500.0, 0.0, 100.0))], np.int32)
    dst = np.asarray([m2u((500.0, 0.0, 100.0))], np.int32)
    return Scenario(a, Terrain(), plans, src, dst, np.zeros(1, np.int64), name="c1")


def config_c2(seed: int = 2, n_plans: int = 3000, n_requests: int = 100, rows: int = 6000,
              n_buildings: int = 256) -> Scenario:
    """configs[1]: batch of 100 FCFS requests vs 3000 plans with terrain, dense urban 16x16 km."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=4000, lo_m=(-8000.0, -8000.0, 0.0), hi_m=(8000.0, 8000.0, 1500.0),
                 horizon_steps=8192, row_capacity=4096)
    terrain = manhattan_terrain(rng, n_buildings, core_half_m=5000.0, raster_half_m=8000.0)
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    plans = reflecting_lines(rng, n_plans, lo, hi, (0, rows), z_lo_u=int(m2u(60)), z_hi_u=int(m2u(1500)))
    pads = vertiports(rng, 200, 5000.0, terrain)
    src, dst, t0 = request_pairs(rng, pads, n_requests, 3000.0, 7000.0, (0, 1000))
    return Scenario(a, terrain, plans, src, dst, t0, name="c2")


def random_small(seed: int, n_plans: int = 40, n_requests: int = 4, half_m: float = 1500.0,
                 z_m=(0.0, 400.0), rows: int = 900, n_buildings: int = 0, trip_m=(600.0, 1500.0),
                 t0_max: int = 200, max_steps: int = 600, **air) -> Scenario:
    """Small seeded scenario for parity tests (oracle finishes in seconds).

    Plans have random activity intervals (ragged rows), speeds and altitudes spanning the
    request band so that wells, exact-boundary cases and conflicts all occur."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=max_steps, lo_m=(-half_m, -half_m, z_m[0]), hi_m=(half_m, half_m, z_m[1]),
                 horizon_steps=int(rows + max_steps + 8),
                 row_capacity=(max(64, n_plans + n_requests + 8) + 3) // 4 * 4)
    a = a.replace(**air)
    terrain = (manhattan_terrain(rng, n_buildings, core_half_m=min(1000.0, half_m), raster_half_m=half_m)
               if n_buildings else Terrain())
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    act = []
    for _ in range(n_plans):
        k0 = int(rng.integers(0, rows // 2))
        k1 = int(rng.integers(k0 + 1, rows + 1))
        act.append((k0, k1))
    plans = reflecting_lines(rng, n_plans, lo, hi, (0, rows), z_lo_u=int(m2u(40)), z_hi_u=int(m2u(z_m[1] - 40)),
                             active=act)
    # re-base: reflecting_lines anchors p0 at rows[0]; keep activity windows
    pads = vertiports(rng, max(8, 2 * n_requests), half_m * 0.7, terrain)
    src, dst, t0 = request_pairs(rng, pads, n_requests, trip_m[0], trip_m[1], (0, t0_max))
    return Scenario(a, terrain, plans, src, dst, t0, name=f"small{seed}")


def random_states(seed: int, sc: Scenario, n: int):
    """Seeded (q, psi, goal, K) tuples inside the scenario box for single-step parity."""
    rng = np.random.default_rng(seed)
    a = sc.airspace
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    span = hi - lo
    out = []
    for _ in range(n):
        q = lo + (rng.uniform(0.1, 0.9, size=3) * span).astype(np.int64)
        q[2] = int(rng.integers(int(m2u(10)), max(int(m2u(11)), int(hi[2] - m2u(20)))))
        g = lo + (rng.uniform(0.1, 0.9, size=3) * span).astype(np.int64)
        psi = int(rng.integers(0, a.HL))
        K = int(rng.integers(0, max(1, a.horizon_steps - a.max_steps - 2)))
        out.append((q.astype(np.int32), psi, g.astype(np.int32), K))
    return out


def config_c3(seed: int = 3, n_requests: int = 1000, n_buildings: int = 256) -> Scenario:
    """configs[2]: 1000 sequential FCFS requests growing the store from 0 to ~1000 plans, the
    configs[1] city and terrain, pairs 2-6 km apart, t0 U[0,600) (dense overlap)."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=4000, lo_m=(-8000.0, -8000.0, 0.0), hi_m=(8000.0, 8000.0, 1500.0),
                 horizon_steps=8192, row_capacity=1024)
    terrain = manhattan_terrain(rng, n_buildings, core_half_m=5000.0, raster_half_m=8000.0)
    pads = vertiports(rng, 200, 5000.0, terrain)
    src, dst, t0 = request_pairs(rng, pads, n_requests, 2000.0, 6000.0, (0, 600))
    return Scenario(a, terrain, [], src, dst, t0, name="c3")


def config_c4(seed: int = 4, n_plans: int = 100_000, rows: int = 4000, n_requests: int = 10,
              n_buildings: int = 256) -> Scenario:
    """configs[3]: 100k plans in 100 x 100 km x [60,1500] m (~6.9 plans/km^3, the configs[1]
    density), 256 building wells near the request area, 5 km requests."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=min(4000, rows - 8), lo_m=(-50000.0, -50000.0, 0.0), hi_m=(50000.0, 50000.0, 1500.0),
                 horizon_steps=rows + 8, row_capacity=((n_plans + n_requests + 64) + 3) // 4 * 4)
    terrain = manhattan_terrain(rng, n_buildings, core_half_m=5000.0, raster_half_m=8000.0)
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    plans = reflecting_lines_fast(rng, n_plans, lo, hi, (0, rows), z_lo_u=int(m2u(60)), z_hi_u=int(m2u(1500)))
    pads = vertiports(rng, 40, 5000.0, terrain)
    src, dst, t0 = request_pairs(rng, pads, n_requests, 4500.0, 5500.0, (0, 1))
    return Scenario(a, terrain, plans, src, dst, t0, name="c4")


def config_c5(seed: int = 5, n_plans: int = 1_000_000, rows: int = 3000, n_requests: int = 10) -> Scenario:
    """configs[4]: 1M plans in 250 x 250 km x [60,2350] m (~7 plans/km^3), widened action set
    17 headings x 5 climbs (A = 85), 256 terrain wells."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=min(4000, rows - 8), lo_m=(-125000.0, -125000.0, 0.0), hi_m=(125000.0, 125000.0, 2350.0),
                 horizon_steps=rows + 8, row_capacity=((n_plans + n_requests + 64) + 3) // 4 * 4,
                 turn_steps=tuple(range(-8, 9)), climb_units=(-32, -16, 0, 16, 32))
    terrain = manhattan_terrain(rng, 256, core_half_m=5000.0, raster_half_m=8000.0)
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    plans = reflecting_lines_fast(rng, n_plans, lo, hi, (0, rows), z_lo_u=int(m2u(60)), z_hi_u=int(m2u(2350)))
    pads = vertiports(rng, 40, 5000.0, terrain)
    src, dst, t0 = request_pairs(rng, pads, n_requests, 4500.0, 5500.0, (0, 1))
    return Scenario(a, terrain, plans, src, dst, t0, name="c5")


def cosim_ring(seed: int, n_batch: int, n_plans: int = 100, radius_m: float = 1200.0, half_m: float = 4000.0,
               z_m: float = 150.0, t0_max: int = 60, rows: int = 1200, max_steps: int = 800, jitter_deg: float = 6.0,
               **air) -> Scenario:
    """SURVEY f2 (co-simulated batch, Fig perf2: batch sizes 1-20 against 100 intruders):
    n_batch aircraft on a ring of radius_m at one altitude, each bound for the (jittered)
    opposite point, departures U[0, t0_max) steps, so their straight paths cross near the
    centre; n_plans reflecting-line intruders in the box.  No terrain."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=max_steps, lo_m=(-half_m, -half_m, 0.0), hi_m=(half_m, half_m, 2 * z_m + 200.0),
                 horizon_steps=int(rows + max_steps + t0_max + 8),
                 row_capacity=(max(64, n_plans + n_batch + 8) + 3) // 4 * 4)
    a = a.replace(**air)
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    plans = reflecting_lines(rng, n_plans, lo, hi, (0, rows), z_lo_u=int(m2u(40)), z_hi_u=int(m2u(2 * z_m + 160)))
    ang = 2 * np.pi * (np.arange(n_batch) + rng.uniform(0, 1)) / max(1, n_batch)
    jit = np.deg2rad(rng.uniform(-jitter_deg, jitter_deg, n_batch))
    src = np.stack([radius_m * np.cos(ang), radius_m * np.sin(ang), np.full(n_batch, z_m)], 1)
    dst = np.stack([radius_m * np.cos(ang + np.pi + jit), radius_m * np.sin(ang + np.pi + jit), np.full(n_batch, z_m)], 1)
    t0 = rng.integers(0, max(1, t0_max), n_batch).astype(np.int64)
    return Scenario(a, Terrain(), plans, m2u(src).astype(np.int32), m2u(dst).astype(np.int32), t0,
                    name=f"cosim{seed}x{n_batch}")


def config_scaled(seed: int, n_plans: int, rows: int = 3000, n_requests: int = 20) -> Scenario:
    """Fig perf1 (performance vs accepted plans) at constant traffic density: n_plans
    reflecting lines in a square box sized for the configs[1] density (3000 plans per
    16 x 16 km, never smaller than that box), z in [60, 1500] m, the configs[1] city (256
    buildings in the central 10 km) and 3-7 km requests between its vertiports."""
    rng = np.random.default_rng(seed)
    half = max(8000.0, 8000.0 * float(np.sqrt(max(n_plans, 1) / 3000.0)))
    a = Airspace(max_steps=min(4000, rows - 320), lo_m=(-half, -half, 0.0), hi_m=(half, half, 1500.0),
                 horizon_steps=rows + 8, row_capacity=((n_plans + n_requests + 64) + 3) // 4 * 4)
    terrain = manhattan_terrain(rng, 256, core_half_m=5000.0, raster_half_m=8000.0)
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    plans = (reflecting_lines_fast(rng, n_plans, lo, hi, (0, rows), z_lo_u=int(m2u(60)), z_hi_u=int(m2u(1500)))
             if n_plans else [])
    pads = vertiports(rng, 200, 5000.0, terrain)
    src, dst, t0 = request_pairs(rng, pads, n_requests, 3000.0, 7000.0, (0, 300))
    return Scenario(a, terrain, plans, src, dst, t0, name=f"scaled{n_plans}")


def airspace_f4(**kw) -> Airspace:
    """the paper-scale action space A = 1350 (Table DS / KI captions P:387),
    factorised 15 turns x 9 accelerations x 10 climbs (SPEC's 15 x 10 x 9, R32):
    turns -7..7 lattice steps per substep (+-1.75 deg / 0.1 s), speed increments -4..4 units per
    substep per substep (+-6.25 m/s^2), speed in [30, 60] m/s, climbs -40..32 units per substep
    in steps of 8 (-6.25 .. +5 m/s; 0 is the middle entry)."""
    base = dict(turn_steps=tuple(range(-7, 8)), acc_units=tuple(range(-4, 5)),
                climb_units=tuple(range(-40, 33, 8)), speed_min_mps=30.0, speed_max_mps=60.0)
    base.update(kw)
    return Airspace(**base)


class ReflectingLinesPacked:
    """n reflecting-line plans (the reflecting_lines_fast recipe, every plan active over ``rows``)
    drawn once, materialised on demand in packed chunks -- for stores too large to hold on the host
    (configs[3] at 4000 rows: 4.8 GB of states; configs[4] at 3000 rows: 36 GB).
    ``chunks(c)`` yields (t0[m], n[m], states[m * rows, 3]) in plan order (the fmdp_add_plans
    layout); ``window(K0, K1)`` returns every plan restricted to rows [K0, K1) as (t0, states)
    pairs -- the rows an oracle needs to evaluate steps at rows K0 .. K1 - 2 (R11 forward
    differences)."""

    def __init__(self, rng: np.random.Generator, n: int, lo_u, hi_u, rows: Tuple[int, int],
                 speed_mps=(30.0, 60.0), vz_units=(-16, 16), z_lo_u=None, z_hi_u=None):
        lo_u = np.asarray(lo_u, np.int64)
        hi_u = np.asarray(hi_u, np.int64)
        zlo = int(lo_u[2] if z_lo_u is None else z_lo_u)
        zhi = int(hi_u[2] if z_hi_u is None else z_hi_u)
        self.lo3 = np.array([lo_u[0], lo_u[1], zlo], np.int64)
        self.hi3 = np.array([hi_u[0], hi_u[1], zhi], np.int64)
        self.p0 = np.stack([rng.integers(self.lo3[d], self.hi3[d] + 1, size=n) for d in range(3)], axis=1)
        sp = rng.uniform(*speed_mps, size=n) * 0.1 * U_PER_M
        th = rng.uniform(0.0, 2.0 * np.pi, size=n)
        self.v = np.stack([np.rint(sp * np.cos(th)), np.rint(sp * np.sin(th)),
                           rng.integers(vz_units[0], vz_units[1] + 1, size=n)], axis=1).astype(np.int64)
        self.n, self.rows = n, rows

    def _states(self, a: int, b: int, k0: int, k1: int) -> np.ndarray:
        K = np.arange(k0 - self.rows[0], k1 - self.rows[0], dtype=np.int64)[None, :, None]
        L = (self.hi3 - self.lo3)[None, None, :]
        raw = self.p0[a:b, None, :] + self.v[a:b, None, :] * K - self.lo3[None, None, :]
        y = np.mod(raw, 2 * L)
        y = np.where(y > L, 2 * L - y, y)
        return (self.lo3[None, None, :] + y).astype(np.int32)

    def _states_torch(self, a: int, b: int, k0: int, k1: int, device) -> np.ndarray:
        import torch  # the same integer arithmetic on a GPU (input generation only), bit-identical
        p0 = torch.as_tensor(self.p0[a:b], device=device)
        v = torch.as_tensor(self.v[a:b], device=device)
        lo3 = torch.as_tensor(self.lo3, device=device)
        L = torch.as_tensor(self.hi3 - self.lo3, device=device)
        K = torch.arange(k0 - self.rows[0], k1 - self.rows[0], dtype=torch.int64, device=device)[None, :, None]
        raw = p0[:, None, :] + v[:, None, :] * K - lo3
        y = torch.remainder(raw, 2 * L)
        y = torch.where(y > L, 2 * L - y, y)
        return (lo3 + y).to(torch.int32).cpu().numpy()

    def chunks(self, chunk: int = 4096, device=None):
        """Packed chunks; with `device` (a CUDA device) the fold runs there (same integers)."""
        nk = self.rows[1] - self.rows[0]
        for a in range(0, self.n, chunk):
            b = min(self.n, a + chunk)
            if device is None:
                st = self._states(a, b, self.rows[0], self.rows[1]).reshape(-1, 3)
            else:
                st = self._states_torch(a, b, self.rows[0], self.rows[1], device).reshape(-1, 3)
            yield (np.full(b - a, self.rows[0], np.int64), np.full(b - a, nk, np.int32), st)

    def window(self, K0: int, K1: int):
        st = self._states(0, self.n, K0, K1)
        return [(int(K0), st[j]) for j in range(self.n)]


def config_c4_full(seed: int = 4, n_plans: int = 100_000, rows: int = 4000, n_requests: int = 10,
                   n_buildings: int = 256):
    """configs[3] at its defined size: 100k plans over 4000 rows (6.4 GB store), packed on demand
    (returns the scenario without host plans, and the ReflectingLinesPacked generator).  Same
    recipe and RNG stream as config_c4."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=min(4000, rows - 8), lo_m=(-50000.0, -50000.0, 0.0), hi_m=(50000.0, 50000.0, 1500.0),
                 horizon_steps=rows + 8, row_capacity=((n_plans + n_requests + 64) + 3) // 4 * 4)
    terrain = manhattan_terrain(rng, n_buildings, core_half_m=5000.0, raster_half_m=8000.0)
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    gen = ReflectingLinesPacked(rng, n_plans, lo, hi, (0, rows), z_lo_u=int(m2u(60)), z_hi_u=int(m2u(1500)))
    pads = vertiports(rng, 40, 5000.0, terrain)
    src, dst, t0 = request_pairs(rng, pads, n_requests, 4500.0, 5500.0, (0, 1))
    return Scenario(a, terrain, [], src, dst, t0, name="c4full"), gen


def config_c5_full(seed: int = 5, n_plans: int = 1_000_000, rows: int = 3000, n_requests: int = 10):
    """configs[4] at its defined size: 1M plans over 3000 rows (48 GB store), A = 85, packed on
    demand.  Same recipe and RNG stream as config_c5."""
    rng = np.random.default_rng(seed)
    a = Airspace(max_steps=min(4000, rows - 8), lo_m=(-125000.0, -125000.0, 0.0), hi_m=(125000.0, 125000.0, 2350.0),
                 horizon_steps=rows + 8, row_capacity=((n_plans + n_requests + 64) + 3) // 4 * 4,
                 turn_steps=tuple(range(-8, 9)), climb_units=(-32, -16, 0, 16, 32))
    terrain = manhattan_terrain(rng, 256, core_half_m=5000.0, raster_half_m=8000.0)
    lo, hi = m2u(a.lo_m), m2u(a.hi_m)
    gen = ReflectingLinesPacked(rng, n_plans, lo, hi, (0, rows), z_lo_u=int(m2u(60)), z_hi_u=int(m2u(2350)))
    pads = vertiports(rng, 40, 5000.0, terrain)
    src, dst, t0 = request_pairs(rng, pads, n_requests, 4500.0, 5500.0, (0, 1))
    return Scenario(a, terrain, [], src, dst, t0, name="c5full"), gen

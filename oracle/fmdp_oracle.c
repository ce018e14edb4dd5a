/*
 * fmdp_oracle.c -- plain, slow, obviously-correct CPU oracle of the FastMDP-GPU
 * hot path (arXiv 2008.03518).  TEST INFRASTRUCTURE ONLY (see fmdp_oracle.h).
 *
 * Style: direct loops in the order of the paper's algorithms, fp64 for values,
 * int64 for every distance predicate, libm pow/sqrt.  No blocking, no fusion, no
 * min-distance identity, no culling: every (projected state, peak) pair is
 * evaluated as Algs 4, 6, 7 state it.
 *
 * Build: gcc -O2 -ffp-contract=off -fno-fast-math -fopenmp -fPIC -shared -o liboracle.so fmdp_oracle.c -lm
 *
 * Threads (SURVEY §8(c) c.7, (d) d.5 ii): orc_set_threads(n > 1) spreads the per-state loops of
 * one decision step over n OpenMP threads (host timing of the baseline only).  Every per-state
 * value is a max over the same wells in the same order whichever thread computes it, so the
 * results are identical to the single-thread run (tested).
 */
#include "fmdp_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 1;

int orc_set_threads(int n) {
  g_threads = n < 1 ? 1 : n;
  return g_threads;
}

/* ------------------------------------------------------------------------- */
/* Parameter conversion to integer units (R23: u-quantised world).  */
/* ------------------------------------------------------------------------- */

/* x / u must be an integer (all scenario lengths are multiples of u). */
static int to_units(double x, double u, int64_t* out) {
  double r = x / u;
  double n = rint(r);
  if (!(fabs(r - n) <= 1e-9 * (1.0 + fabs(r)))) return ORC_E_ARG;
  *out = (int64_t)n;
  return ORC_OK;
}

typedef struct conv {
  int64_t step_u;                 /* v0*dt/u                          */
  int64_t vmin_u, vmax_u;         /* speed bounds, units per substep (R32) */
  int64_t k_tau[ORC_MAX_TAU];     /* tau/dt substeps (Table PK)   */
  int64_t R_tau[ORC_MAX_TAU];     /* 300+10 tau metres -> units         */
  int64_t R_max;
  int64_t zdeck_u, cap_u, sep_u;
} conv;

static int convert(const orc_params* p, conv* c) {
  if (!p || p->u_m <= 0 || p->dt_s <= 0 || p->W < 1 || p->HL < 8 || (p->HL % 8) != 0) return ORC_E_ARG;
  if (p->n_turn < 1 || p->n_turn > ORC_MAX_TURN || p->n_climb < 1 || p->n_climb > ORC_MAX_CLIMB) return ORC_E_ARG;
  if (p->n_tau < 0 || p->n_tau > ORC_MAX_TAU) return ORC_E_ARG;
  if (to_units(p->speed_mps * p->dt_s, p->u_m, &c->step_u)) return ORC_E_ARG;
  /* acceleration actions (R32): speed in units per substep, clamped to
   * [speed_min, speed_max]; with no bounds given (0) the speed is held at v0 */
  if (p->n_acc < 1 || p->n_acc > ORC_MAX_ACC) return ORC_E_ARG;
  if (p->speed_min_mps > 0 || p->speed_max_mps > 0) {
    if (to_units(p->speed_min_mps * p->dt_s, p->u_m, &c->vmin_u)) return ORC_E_ARG;
    if (to_units(p->speed_max_mps * p->dt_s, p->u_m, &c->vmax_u)) return ORC_E_ARG;
    if (c->vmin_u < 1 || c->vmin_u > c->step_u || c->step_u > c->vmax_u) return ORC_E_ARG;
  } else {
    c->vmin_u = c->vmax_u = c->step_u;
  }
  c->R_max = 0;
  for (int i = 0; i < p->n_tau; ++i) {
    double k = p->tau_s[i] / p->dt_s;
    if (fabs(k - rint(k)) > 1e-9) return ORC_E_ARG;
    c->k_tau[i] = (int64_t)rint(k);
    if (to_units(p->tau_radius_m[i], p->u_m, &c->R_tau[i]) || c->R_tau[i] <= 0) return ORC_E_ARG;
    if (c->R_tau[i] > c->R_max) c->R_max = c->R_tau[i];
  }
  if (to_units(p->deck_alt_m, p->u_m, &c->zdeck_u)) return ORC_E_ARG;
  if (to_units(p->capture_m, p->u_m, &c->cap_u)) return ORC_E_ARG;
  if (to_units(p->sep_m, p->u_m, &c->sep_u)) return ORC_E_ARG;
  return ORC_OK;
}

int orc_check_params(const orc_params* p) {
  conv c;
  return convert(p, &c);
}

/* ------------------------------------------------------------------------- */
/* Heading lattice (R14: dynamics deferred by the paper).     */
/* D[psi] = L*(cos, sin)(2*pi*psi/HL) rounded, defined on the first octant and */
/* reflected / rotated so the lattice is exactly symmetric.                    */
/* ------------------------------------------------------------------------- */
/* Displacement of one substep at heading psi and speed v (units per substep): the lattice above
 * with L = v (R32; at v = v0 it is exactly the constant-speed table). */
void orc_direction(int32_t HL, int64_t v, int32_t psi, int32_t* dx, int32_t* dy) {
  const int Q = HL / 4, O = HL / 8;
  const double L = (double)v;
  int quad = psi / Q, r = psi % Q;
  double a, b;
  if (r <= O) {
    a = rint(L * cos(2.0 * M_PI * r / HL));
    b = rint(L * sin(2.0 * M_PI * r / HL));
  } else {
    int m = Q - r;
    a = rint(L * sin(2.0 * M_PI * m / HL));
    b = rint(L * cos(2.0 * M_PI * m / HL));
  }
  switch (quad) {
    case 0: *dx = (int32_t)a;  *dy = (int32_t)b;  break;
    case 1: *dx = (int32_t)-b; *dy = (int32_t)a;  break;
    case 2: *dx = (int32_t)-a; *dy = (int32_t)-b; break;
    default: *dx = (int32_t)b; *dy = (int32_t)-a; break;
  }
}

int orc_tables(const orc_params* p, int32_t* DX, int32_t* DY) {
  conv c;
  if (convert(p, &c)) return ORC_E_ARG;
  const int HL = p->HL, Q = HL / 4, O = HL / 8;
  const double L = (double)c.step_u;
  for (int psi = 0; psi < HL; ++psi) {
    int quad = psi / Q, r = psi % Q;
    double a, b;  /* first-quadrant vector at lattice angle r */
    if (r <= O) {
      a = rint(L * cos(2.0 * M_PI * r / HL));
      b = rint(L * sin(2.0 * M_PI * r / HL));
    } else {
      int m = Q - r; /* reflect about 45 degrees */
      a = rint(L * sin(2.0 * M_PI * m / HL));
      b = rint(L * cos(2.0 * M_PI * m / HL));
    }
    int32_t x, y;
    switch (quad) {
      case 0: x = (int32_t)a;  y = (int32_t)b;  break;
      case 1: x = (int32_t)-b; y = (int32_t)a;  break;
      case 2: x = (int32_t)-a; y = (int32_t)-b; break;
      default: x = (int32_t)b; y = (int32_t)-a; break;
    }
    DX[psi] = x;
    DY[psi] = y;
  }
  return ORC_OK;
}

static int32_t pmod(int64_t a, int32_t m) {
  int64_t r = a % m;
  return (int32_t)(r < 0 ? r + m : r);
}

/* Lattice heading nearest to the bearing src -> dst (R21). */
int32_t orc_initial_heading(const orc_params* p, const int32_t src[3], const int32_t dst[3]) {
  double dx = (double)dst[0] - (double)src[0];
  double dy = (double)dst[1] - (double)src[1];
  double a = atan2(dy, dx) * (double)p->HL / (2.0 * M_PI);
  return pmod((int64_t)rint(a), p->HL);
}

/* ------------------------------------------------------------------------- */
/* Build Peaks (Alg 2; Table PK): five wells per intruder at   */
/* p + v*tau, radius 300 + 10 tau metres; v per substep (reading R11).         */
/* ------------------------------------------------------------------------- */
int orc_build_wells(const orc_params* p, const int32_t pos[3], const int32_t vel[3],
                    int32_t* centers, int64_t* radius_u) {
  conv c;
  if (convert(p, &c)) return ORC_E_ARG;
  for (int i = 0; i < p->n_tau; ++i) {
    for (int d = 0; d < 3; ++d) centers[3 * i + d] = (int32_t)(pos[d] + c.k_tau[i] * (int64_t)vel[d]);
    radius_u[i] = c.R_tau[i];
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Forward projection (Alg 3): the action (turn h, acceleration acc, climb c) is held */
/* for W substeps; psi_t = psi_{t-1} + h, v_t = clamp(v_{t-1} + acc, vmin, vmax),              */
/* q_t = q_{t-1} + (D(psi_t, v_t), c)  (SPEC step_dynamics: heading, then speed, then move).   */
/* Action index a = (i_turn * n_acc + i_acc) * n_climb + i_climb (n_acc = 1: i_turn*n_climb+c). */
/* ------------------------------------------------------------------------- */
int orc_project_v(const orc_params* p, const int32_t q[3], int32_t psi, int32_t v, int32_t* states,
                  int32_t* psi_out, int32_t* v_out) {
  conv c;
  if (convert(p, &c)) return ORC_E_ARG;
  const int W = p->W;
  for (int it = 0; it < p->n_turn; ++it) {
    for (int ia = 0; ia < p->n_acc; ++ia) {
      for (int ic = 0; ic < p->n_climb; ++ic) {
        int a = (it * p->n_acc + ia) * p->n_climb + ic;
        int64_t x = q[0], y = q[1], z = q[2];
        int32_t h = psi;
        int64_t sp = v;
        for (int t = 1; t <= W; ++t) {
          h = pmod((int64_t)h + p->turn_steps[it], p->HL);
          sp += p->acc_units[ia];
          if (sp < c.vmin_u) sp = c.vmin_u;
          if (sp > c.vmax_u) sp = c.vmax_u;
          int32_t dx, dy;
          orc_direction(p->HL, sp, h, &dx, &dy);
          x += dx;
          y += dy;
          z += p->climb_units[ic];
          int idx = a * W + (t - 1);
          states[3 * idx + 0] = (int32_t)x;
          states[3 * idx + 1] = (int32_t)y;
          states[3 * idx + 2] = (int32_t)z;
          if (psi_out) psi_out[idx] = h;
          if (v_out) v_out[idx] = (int32_t)sp;
        }
      }
    }
  }
  return ORC_OK;
}

int orc_project(const orc_params* p, const int32_t q[3], int32_t psi, int32_t* states, int32_t* psi_out) {
  conv c;
  if (convert(p, &c)) return ORC_E_ARG;
  return orc_project_v(p, q, psi, (int32_t)c.step_u, states, psi_out, NULL);
}

int32_t orc_initial_speed(const orc_params* p) {
  conv c;
  if (convert(p, &c)) return -1;
  return (int32_t)c.step_u;
}

static int n_actions(const orc_params* p) { return p->n_turn * p->n_acc * p->n_climb; }

/* ------------------------------------------------------------------------- */
/* Peak values.                                                                */
/* ------------------------------------------------------------------------- */
static int64_t d2_of(const int32_t a[3], const int32_t b[3]) {
  int64_t dx = (int64_t)a[0] - b[0], dy = (int64_t)a[1] - b[1], dz = (int64_t)a[2] - b[2];
  return dx * dx + dy * dy + dz * dz;
}

/* Alg 4: V = |r| * gamma^d, d the Euclidean distance in metres (R10). */
double orc_goal_value(const orc_params* p, int64_t d2) {
  double d = p->u_m * sqrt((double)d2);
  return fabs(p->goal_r) * pow(p->goal_gamma, d);
}

/* Algs 6/7 P:657-668: in = d < R; V = in * |r| * gamma^d (R12: exact d^2 < R^2). */
double orc_well_value(double r, double gamma, double u_m, int64_t d2, int64_t R_u) {
  int in = d2 < R_u * R_u;
  if (!in) return 0.0;
  double d = u_m * sqrt((double)d2);
  return fabs(r) * pow(gamma, d);
}

/* Alg 1 P:207-210 with the projected altitude (R6) and z_deck in metres (R7). */
double orc_deck_penalty(const orc_params* p, int32_t z) {
  conv c;
  if (convert(p, &c)) return NAN;
  if ((int64_t)z < c.zdeck_u) return p->deck_scale - p->u_m * (double)z;
  return 0.0;
}

/* ------------------------------------------------------------------------- */
/* Accepted-plan store (Sec. V: "a simple table in memory").             */
/* ------------------------------------------------------------------------- */
struct orc_store {
  int32_t n, cap;
  int64_t* t0;
  int32_t* len;
  int32_t** states;
};

orc_store* orc_store_new(void) {
  orc_store* s = (orc_store*)calloc(1, sizeof(orc_store));
  return s;
}

void orc_store_free(orc_store* s) {
  if (!s) return;
  for (int i = 0; i < s->n; ++i) free(s->states[i]);
  free(s->t0);
  free(s->len);
  free(s->states);
  free(s);
}

int orc_store_add(orc_store* s, int64_t t0, int32_t n, const int32_t* states) {
  if (!s || n < 1 || !states || t0 < 0) return ORC_E_ARG;
  if (s->n == s->cap) {
    int32_t nc = s->cap ? 2 * s->cap : 64;
    int64_t* a = (int64_t*)realloc(s->t0, sizeof(int64_t) * nc);
    if (!a) return ORC_E_NOMEM;
    s->t0 = a;
    int32_t* b = (int32_t*)realloc(s->len, sizeof(int32_t) * nc);
    if (!b) return ORC_E_NOMEM;
    s->len = b;
    int32_t** c = (int32_t**)realloc(s->states, sizeof(int32_t*) * nc);
    if (!c) return ORC_E_NOMEM;
    s->states = c;
    s->cap = nc;
  }
  int32_t* copy = (int32_t*)malloc(sizeof(int32_t) * 3 * (size_t)n);
  if (!copy) return ORC_E_NOMEM;
  memcpy(copy, states, sizeof(int32_t) * 3 * (size_t)n);
  s->t0[s->n] = t0;
  s->len[s->n] = n;
  s->states[s->n] = copy;
  s->n += 1;
  return ORC_OK;
}

int32_t orc_store_count(const orc_store* s) { return s ? s->n : 0; }

/* Intruder position and linear velocity at row K (reading R11): the stored
 * state, and the forward difference to the next stored state (the last state
 * repeats the previous difference; a single-state plan has v = 0).
 * Returns 1 if the plan is active at K, else 0. */
int orc_store_sample(const orc_store* s, int32_t plan, int64_t K, int32_t pos[3], int32_t vel[3]) {
  if (!s || plan < 0 || plan >= s->n) return 0;
  int64_t i = K - s->t0[plan];
  int32_t n = s->len[plan];
  if (i < 0 || i >= n) return 0;
  const int32_t* st = s->states[plan];
  for (int d = 0; d < 3; ++d) pos[d] = st[3 * i + d];
  if (n == 1) {
    vel[0] = vel[1] = vel[2] = 0;
  } else if (i < n - 1) {
    for (int d = 0; d < 3; ++d) vel[d] = st[3 * (i + 1) + d] - st[3 * i + d];
  } else {
    for (int d = 0; d < 3; ++d) vel[d] = st[3 * i + d] - st[3 * (i - 1) + d];
  }
  return 1;
}

/* Min d^2 from q to any plan active at row K, saturated at R_max^2 (Sec IV.I; R15, R20). */
static int64_t nearest_d2(const orc_store* S, const int32_t q[3], int64_t K, int64_t sat) {
  int64_t best = sat;
  for (int32_t j = 0; j < orc_store_count(S); ++j) {
    int32_t pos[3], vel[3];
    if (!orc_store_sample(S, j, K, pos, vel)) continue;
    int64_t d2 = d2_of(q, pos);
    if (d2 < best) best = d2;
  }
  return best;
}

/* Terrain collision (R16): below z = 0 or below the height raster cell. */
static int terrain_collision(const orc_terrain* T, const int32_t q[3]) {
  if (q[2] < 0) return 1;
  if (!T || T->nx <= 0 || T->ny <= 0 || !T->height) return 0;
  int64_t rx = (int64_t)q[0] - T->x0, ry = (int64_t)q[1] - T->y0;
  if (rx < 0 || ry < 0) return 0;
  int64_t ix = rx / T->cell, iy = ry / T->cell;
  if (ix >= T->nx || iy >= T->ny) return 0;
  return q[2] < T->height[iy * (int64_t)T->nx + ix];
}

/* ------------------------------------------------------------------------- */
/* One decision step: Algs 2-9 in the order of Fig 3a.             */
/* ------------------------------------------------------------------------- */
static int eval_step_core(const orc_params* p, const orc_terrain* T, const orc_store* S, const int32_t q[3],
                          int32_t psi, int32_t v, const int32_t g[3], int64_t K, int32_t n_peer,
                          const int32_t* peer_pos, const int32_t* peer_vel, orc_step_out* out);

int orc_eval_step(const orc_params* p, const orc_terrain* T, const orc_store* S,
                  const int32_t q[3], int32_t psi, const int32_t g[3], int64_t K, orc_step_out* out) {
  return orc_eval_step_peers(p, T, S, q, psi, g, K, 0, NULL, NULL, out);
}

/* One decision step from (q, psi, speed v) -- the acceleration actions of SURVEY f4 (R32). */
int orc_eval_step_v(const orc_params* p, const orc_terrain* T, const orc_store* S, const int32_t q[3], int32_t psi,
                    int32_t v, const int32_t g[3], int64_t K, orc_step_out* out) {
  return eval_step_core(p, T, S, q, psi, v, g, K, 0, NULL, NULL, out);
}

int orc_eval_step_peers(const orc_params* p, const orc_terrain* T, const orc_store* S,
                        const int32_t q[3], int32_t psi, const int32_t g[3], int64_t K, int32_t n_peer,
                        const int32_t* peer_pos, const int32_t* peer_vel, orc_step_out* out) {
  return eval_step_core(p, T, S, q, psi, orc_initial_speed(p), g, K, n_peer, peer_pos, peer_vel, out);
}

static int eval_step_core(const orc_params* p, const orc_terrain* T, const orc_store* S, const int32_t q[3],
                          int32_t psi, int32_t v0, const int32_t g[3], int64_t K, int32_t n_peer,
                          const int32_t* peer_pos, const int32_t* peer_vel, orc_step_out* out) {
  conv c;
  if (convert(p, &c) || !out || v0 < c.vmin_u || v0 > c.vmax_u) return ORC_E_ARG;
  const int A = n_actions(p), W = p->W, AW = A * W;
  int32_t* proj = (int32_t*)malloc(sizeof(int32_t) * 3 * AW);
  int32_t* ppsi = (int32_t*)malloc(sizeof(int32_t) * AW);
  int32_t* pv = (int32_t*)malloc(sizeof(int32_t) * AW);
  double* vpos = (double*)malloc(sizeof(double) * AW);
  double* vint = (double*)malloc(sizeof(double) * AW);
  double* vter = (double*)malloc(sizeof(double) * AW);
  double* valt = (double*)malloc(sizeof(double) * AW);
  double* v = (double*)malloc(sizeof(double) * AW);
  double* scale = (double*)malloc(sizeof(double) * AW);
  double* vstar = (double*)malloc(sizeof(double) * A);
  double* vsc = (double*)malloc(sizeof(double) * A);
  double* vneg = (double*)malloc(sizeof(double) * AW);
  int rc = ORC_OK;
  if (!proj || !ppsi || !pv || !vpos || !vint || !vter || !valt || !v || !scale || !vstar || !vsc || !vneg) {
    rc = ORC_E_NOMEM;
    goto done;
  }

  /* Forward project (Alg 3). */
  if ((rc = orc_project_v(p, q, psi, v0, proj, ppsi, pv))) goto done;

  /* Process positive rewards (Alg 4): P+ = { goal } (Alg 2, Table PK, R8). */
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
  for (int i = 0; i < AW; ++i) {
    vpos[i] = 0.0;
    double V = orc_goal_value(p, d2_of(&proj[3 * i], g));
    if (V > vpos[i]) vpos[i] = V;  /* "Save max value" P:583-584 (single peak) */
  }

  /* Process negative terrain rewards (Alg 6). */
#pragma omp parallel for num_threads(g_threads) if (g_threads > 1) schedule(static)
  for (int i = 0; i < AW; ++i) {
    vter[i] = 0.0;
    for (int w = 0; T && w < T->n_wells; ++w) {
      double V = orc_well_value(p->terr_r, p->terr_gamma, p->u_m, d2_of(&proj[3 * i], &T->center[3 * w]),
                                (int64_t)T->radius[w]);
      if (V > vter[i]) vter[i] = V;
    }
  }

  /* Process negative intruder rewards (Alg 7): five wells per plan active at row K. */
  for (int i = 0; i < AW; ++i) vint[i] = 0.0;
  if (g_threads <= 1) {
    for (int32_t j = 0; j < orc_store_count(S); ++j) {
      int32_t pos[3], vel[3], cen[3 * ORC_MAX_TAU];
      int64_t rad[ORC_MAX_TAU];
      if (!orc_store_sample(S, j, K, pos, vel)) continue;
      orc_build_wells(p, pos, vel, cen, rad);  /* Alg 2 */
      for (int tau = 0; tau < p->n_tau; ++tau) {
        for (int i = 0; i < AW; ++i) {
          double V = orc_well_value(p->intr_r, p->intr_gamma, p->u_m, d2_of(&proj[3 * i], &cen[3 * tau]), rad[tau]);
          if (V > vint[i]) vint[i] = V;
        }
      }
    }
  } else {
    /* the same wells (plan order, then tau), built once; each state's max over them in that
     * order on one thread -- the single-thread result exactly */
    const int32_t np = orc_store_count(S), nt = p->n_tau;
    int32_t* cen = (int32_t*)malloc(sizeof(int32_t) * 3 * ORC_MAX_TAU * (size_t)(np > 0 ? np : 1));
    int64_t* rad = (int64_t*)malloc(sizeof(int64_t) * ORC_MAX_TAU * (size_t)(np > 0 ? np : 1));
    if (!cen || !rad) { free(cen); free(rad); rc = ORC_E_NOMEM; goto done; }
    int32_t nw = 0;
    for (int32_t j = 0; j < np; ++j) {
      int32_t pos[3], vel[3];
      if (!orc_store_sample(S, j, K, pos, vel)) continue;
      orc_build_wells(p, pos, vel, &cen[3 * nt * nw], &rad[nt * nw]);
      nw++;
    }
#pragma omp parallel for num_threads(g_threads) schedule(static)
    for (int i = 0; i < AW; ++i) {
      for (int32_t w = 0; w < nw * nt; ++w) {
        double V = orc_well_value(p->intr_r, p->intr_gamma, p->u_m, d2_of(&proj[3 * i], &cen[3 * w]), rad[w]);
        if (V > vint[i]) vint[i] = V;
      }
    }
    free(cen);
    free(rad);
  }

  /* Process negative rewards (Alg 5): five wells per batch peer (P^-, Alg 2
   * P:464-466), same peak parameters as an intruder (Table PK aircraft row). */
  for (int i = 0; i < AW; ++i) vneg[i] = 0.0;
  for (int32_t j = 0; j < n_peer; ++j) {
    int32_t cen[3 * ORC_MAX_TAU];
    int64_t rad[ORC_MAX_TAU];
    orc_build_wells(p, &peer_pos[3 * j], &peer_vel[3 * j], cen, rad);
    for (int tau = 0; tau < p->n_tau; ++tau) {
      for (int i = 0; i < AW; ++i) {
        double V = orc_well_value(p->intr_r, p->intr_gamma, p->u_m, d2_of(&proj[3 * i], &cen[3 * tau]), rad[tau]);
        if (V > vneg[i]) vneg[i] = V;
      }
    }
  }

  /* Hard deck (Alg 1; Alg 8). */
  for (int i = 0; i < AW; ++i) valt[i] = orc_deck_penalty(p, proj[3 * i + 2]);

  /* Compute value (Alg 8): V = V+ - max(V-, V^T, V^I) - V_alt; V- is empty
   * for a single requesting aircraft (Table DS P:397 with N = 1). */
  for (int a = 0; a < A; ++a) {
    double vmax = p->vmax_init_zero ? 0.0 : -INFINITY;  /* P:736 vs R2 */
    double best_t = -INFINITY, best_sc = 0.0;
    for (int t = 0; t < W; ++t) {
      int i = a * W + t;
      double neg = vter[i] > vint[i] ? vter[i] : vint[i];
      if (vneg[i] > neg) neg = vneg[i];
      v[i] = vpos[i] - neg - valt[i];
      scale[i] = vpos[i] + neg + valt[i];
      if (v[i] > vmax) vmax = v[i];
      if (v[i] > best_t) { best_t = v[i]; best_sc = scale[i]; }
    }
    vstar[a] = vmax;
    vsc[a] = best_sc;
    if (p->valuation == 1) {  /* Alg 1: the value of the endpoint of Delta_10 (R31) */
      vstar[a] = v[a * W + W - 1];
      vsc[a] = scale[a * W + W - 1];
    }
  }

  /* Select best action (Alg 9), lowest index on ties (R13). */
  int a1 = 0;
  for (int a = 1; a < A; ++a)
    if (vstar[a] > vstar[a1]) a1 = a;
  int a2 = -1;
  for (int a = 0; a < A; ++a) {
    if (a == a1) continue;
    if (a2 < 0 || vstar[a] > vstar[a2]) a2 = a;
  }
  out->a_star = a1;
  out->a_second = a2;
  out->gap = a2 >= 0 ? vstar[a1] - vstar[a2] : INFINITY;
  out->near_tie = a2 >= 0 && out->gap < p->near_tie_rel * vsc[a1];

  /* Conflict of every action's first substep (Delta_1, Alg 1) against row K+1 (R20). */
  if (out->conf_d2) {
    for (int a = 0; a < A; ++a)
      out->conf_d2[a] = nearest_d2(S, &proj[3 * (a * W + 0)], K + 1, c.R_max * c.R_max);
  }

  if (out->v_pos) memcpy(out->v_pos, vpos, sizeof(double) * AW);
  if (out->v_int) memcpy(out->v_int, vint, sizeof(double) * AW);
  if (out->v_neg) memcpy(out->v_neg, vneg, sizeof(double) * AW);
  if (out->v_ter) memcpy(out->v_ter, vter, sizeof(double) * AW);
  if (out->v_alt) memcpy(out->v_alt, valt, sizeof(double) * AW);
  if (out->v) memcpy(out->v, v, sizeof(double) * AW);
  if (out->scale) memcpy(out->scale, scale, sizeof(double) * AW);
  if (out->vstar) memcpy(out->vstar, vstar, sizeof(double) * A);
  if (out->vstar_scale) memcpy(out->vstar_scale, vsc, sizeof(double) * A);
  if (out->proj) memcpy(out->proj, proj, sizeof(int32_t) * 3 * AW);
  if (out->proj_psi) memcpy(out->proj_psi, ppsi, sizeof(int32_t) * AW);
  if (out->proj_v) memcpy(out->proj_v, pv, sizeof(int32_t) * AW);

done:
  free(proj); free(ppsi); free(pv); free(vpos); free(vint); free(vter); free(valt);
  free(v); free(scale); free(vstar); free(vsc); free(vneg);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* One PDFP request (Fig 3a loop P:272-289; Sec. V).              */
/* ------------------------------------------------------------------------- */
int orc_schedule(const orc_params* p, const orc_terrain* T, const orc_store* S,
                 const int32_t src[3], const int32_t dst[3], int64_t t0, int32_t cap,
                 int32_t* traj, int32_t* heading, int32_t* astar, orc_result* res) {
  return orc_schedule_v(p, T, S, src, dst, t0, cap, traj, heading, NULL, astar, res);
}

/* The same with the speed of every state (R32: v0 at departure, then the chosen action's). */
int orc_schedule_v(const orc_params* p, const orc_terrain* T, const orc_store* S,
                   const int32_t src[3], const int32_t dst[3], int64_t t0, int32_t cap,
                   int32_t* traj, int32_t* heading, int32_t* speed, int32_t* astar, orc_result* res) {
  conv c;
  if (convert(p, &c) || !traj || !heading || !res || cap < 1 || t0 < 0) return ORC_E_ARG;
  const int A = n_actions(p), W = p->W;
  const int64_t sat = c.R_max * c.R_max, sep2 = c.sep_u * c.sep_u, cap2 = c.cap_u * c.cap_u;
  int32_t q[3] = {src[0], src[1], src[2]};
  int32_t psi = orc_initial_heading(p, src, dst);
  int32_t v = (int32_t)c.step_u;
  int64_t K = t0;
  int32_t k = 0;
  memset(res, 0, sizeof(*res));
  res->fail_step = -1;
  res->min_sep_d2 = sat;
  memcpy(&traj[0], q, sizeof(q));
  heading[0] = psi;
  if (speed) speed[0] = v;

  /* Initial terminal tests at the departure row. */
  int64_t n0 = nearest_d2(S, q, K, sat);
  if (n0 < res->min_sep_d2) res->min_sep_d2 = n0;
  if (n0 < sep2) { res->status = ORC_REJ_CONFLICT; res->fail_step = 0; res->n_states = 1; return ORC_OK; }
  if (terrain_collision(T, q)) { res->status = ORC_REJ_TERRAIN; res->fail_step = 0; res->n_states = 1; return ORC_OK; }
  if (d2_of(q, dst) < cap2) { res->status = ORC_ACCEPTED; res->n_states = 1; return ORC_OK; }

  int32_t* proj = (int32_t*)malloc(sizeof(int32_t) * 3 * A * W);
  int32_t* ppsi = (int32_t*)malloc(sizeof(int32_t) * A * W);
  int32_t* pv = (int32_t*)malloc(sizeof(int32_t) * A * W);
  if (!proj || !ppsi || !pv) { free(proj); free(ppsi); free(pv); return ORC_E_NOMEM; }
  int rc = ORC_OK;
  for (;;) {
    if (k + 1 >= cap) { rc = ORC_E_RANGE; break; }
    orc_step_out o;
    memset(&o, 0, sizeof(o));
    o.proj = proj;
    o.proj_psi = ppsi;
    o.proj_v = pv;
    if ((rc = orc_eval_step_v(p, T, S, q, psi, v, dst, K, &o))) break;
    if (o.near_tie) res->n_near_ties += 1;
    if (astar) astar[k] = o.a_star;
    /* s_{t+1} <- Delta_1[a*] (Alg 1; R5). */
    int i1 = o.a_star * W + 0;
    q[0] = proj[3 * i1 + 0]; q[1] = proj[3 * i1 + 1]; q[2] = proj[3 * i1 + 2];
    psi = ppsi[i1];
    v = pv[i1];
    k += 1;
    K += 1;
    memcpy(&traj[3 * k], q, sizeof(q));
    heading[k] = psi;
    if (speed) speed[k] = v;
    /* Determine terminal state (Sec IV.I), priority order R15/R16/R20. */
    int64_t nd = nearest_d2(S, q, K, sat);
    if (nd < res->min_sep_d2) res->min_sep_d2 = nd;
    if (nd < sep2) { res->status = ORC_REJ_CONFLICT; res->fail_step = k; break; }
    if (terrain_collision(T, q)) { res->status = ORC_REJ_TERRAIN; res->fail_step = k; break; }
    if (d2_of(q, dst) < cap2) { res->status = ORC_ACCEPTED; break; }
    if (k >= p->max_steps) { res->status = ORC_REJ_TIMEOUT; res->fail_step = k; break; }
  }
  res->n_states = k + 1;
  free(proj);
  free(ppsi);
  free(pv);
  return rc;
}

/* Strict FCFS: requests in array order, each against the
 * store including every plan accepted before it (R-a10). */
int orc_schedule_batch(const orc_params* p, const orc_terrain* T, orc_store* S, int32_t n,
                       const int32_t* src, const int32_t* dst, const int64_t* t0, int32_t cap,
                       int32_t* traj, int32_t* heading, int32_t* astar, orc_result* res) {
  for (int32_t i = 0; i < n; ++i) {
    int32_t* tr = traj + (size_t)3 * cap * i;
    int32_t* hd = heading + (size_t)cap * i;
    int32_t* as = astar ? astar + (size_t)cap * i : NULL;
    int rc = orc_schedule(p, T, S, &src[3 * i], &dst[3 * i], t0[i], cap, tr, hd, as, &res[i]);
    if (rc) return rc;
    if (res[i].status == ORC_ACCEPTED) {
      rc = orc_store_add(S, t0[i], res[i].n_states, tr);
      if (rc) return rc;
    }
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Lockstep replay of an externally produced trajectory (parity protocol).     */
/* At every step the oracle recomputes V*, a*; a different action is accepted  */
/* only at a near-tie of the oracle's own values; the transition and every    */
/* terminal verdict must be reproduced exactly.                               */
/* ------------------------------------------------------------------------- */
int orc_replay(const orc_params* p, const orc_terrain* T, const orc_store* S,
               const int32_t src[3], const int32_t dst[3], int64_t t0,
               int32_t n, const int32_t* traj, const int32_t* heading, const int32_t* astar,
               int32_t status, orc_replay_stats* st) {
  return orc_replay_v(p, T, S, src, dst, t0, n, traj, heading, NULL, astar, status, st);
}

/* speed: the speed of every state (R32), or NULL for constant speed v0. */
int orc_replay_v(const orc_params* p, const orc_terrain* T, const orc_store* S,
                 const int32_t src[3], const int32_t dst[3], int64_t t0,
                 int32_t n, const int32_t* traj, const int32_t* heading, const int32_t* speed, const int32_t* astar,
                 int32_t status, orc_replay_stats* st) {
  conv c;
  if (convert(p, &c) || !st || n < 1) return ORC_E_ARG;
  memset(st, 0, sizeof(*st));
  st->first_fail_step = -1;
  const int A = n_actions(p), W = p->W;
  const int64_t sat = c.R_max * c.R_max, sep2 = c.sep_u * c.sep_u, cap2 = c.cap_u * c.cap_u;
#define FAIL(k_) do { st->n_fail++; if (st->first_fail_step < 0) st->first_fail_step = (k_); } while (0)
  if (traj[0] != src[0] || traj[1] != src[1] || traj[2] != src[2]) FAIL(0);
  if (heading[0] != orc_initial_heading(p, src, dst)) FAIL(0);
  if (speed && speed[0] != c.step_u) FAIL(0);
  double* vstar = (double*)malloc(sizeof(double) * A);
  double* vsc = (double*)malloc(sizeof(double) * A);
  int32_t* proj = (int32_t*)malloc(sizeof(int32_t) * 3 * A * W);
  int32_t* ppsi = (int32_t*)malloc(sizeof(int32_t) * A * W);
  int32_t* pv = (int32_t*)malloc(sizeof(int32_t) * A * W);
  if (!vstar || !vsc || !proj || !ppsi || !pv) {
    free(vstar); free(vsc); free(proj); free(ppsi); free(pv);
    return ORC_E_NOMEM;
  }
  for (int32_t k = 0; k < n; ++k) {
    const int32_t* q = &traj[3 * k];
    int64_t K = t0 + k;
    /* Terminal verdict at state k. */
    int verdict = -1;
    int64_t nd = nearest_d2(S, q, K, sat);
    if (nd < sep2) verdict = ORC_REJ_CONFLICT;
    else if (terrain_collision(T, q)) verdict = ORC_REJ_TERRAIN;
    else if (d2_of(q, dst) < cap2) verdict = ORC_ACCEPTED;
    else if (k >= p->max_steps) verdict = ORC_REJ_TIMEOUT;
    if (k == n - 1) {  /* status -1: a trajectory prefix, its last state must be non-terminal */
      if (verdict != (status < 0 ? -1 : status)) FAIL(k);
      break;
    }
    if (verdict >= 0) { FAIL(k); break; }
    orc_step_out o;
    memset(&o, 0, sizeof(o));
    o.vstar = vstar;
    o.vstar_scale = vsc;
    o.proj = proj;
    o.proj_psi = ppsi;
    o.proj_v = pv;
    if (orc_eval_step_v(p, T, S, q, heading[k], speed ? speed[k] : (int32_t)c.step_u, dst, K, &o)) { FAIL(k); break; }
    st->n_steps_checked++;
    if (o.near_tie) st->n_near_ties++;
    int ag = astar ? astar[k] : o.a_star;
    if (ag < 0 || ag >= A) { FAIL(k); break; }
    if (ag != o.a_star) {
      if (vstar[o.a_star] - vstar[ag] < p->near_tie_rel * vsc[o.a_star]) st->n_divergent++;
      else FAIL(k);
    }
    int i1 = ag * W;
    const int32_t* q1 = &traj[3 * (k + 1)];
    if (q1[0] != proj[3 * i1] || q1[1] != proj[3 * i1 + 1] || q1[2] != proj[3 * i1 + 2] ||
        heading[k + 1] != ppsi[i1] || (speed && speed[k + 1] != pv[i1]))
      FAIL(k);
  }
#undef FAIL
  free(vstar); free(vsc); free(proj); free(ppsi); free(pv);
  return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* Co-simulated batch.                                             */
/* ------------------------------------------------------------------------- */

/* Linear velocity of a batch aircraft at its state k ("position and the linear velocity";
 * DESIGN.md R28): the displacement of its last transition, q(k) - q(k-1); at departure (k = 0)
 * the initial heading at level flight, (DX, DY)[psi_0], climb 0. */
static void peer_velocity(const int32_t* DX, const int32_t* DY, const int32_t* traj, const int32_t* heading,
                          int32_t k, int32_t vel[3]) {
  if (k == 0) {
    vel[0] = DX[heading[0]];
    vel[1] = DY[heading[0]];
    vel[2] = 0;
  } else {
    for (int d = 0; d < 3; ++d) vel[d] = traj[3 * k + d] - traj[3 * (k - 1) + d];
  }
}

/* Terminal verdict of a state (Sec IV.I; Table DS "Determine terminal state" N x N):
 * separation against the store row K and against every other present batch aircraft. */
static int cosim_verdict(const orc_terrain* T, const orc_store* S, const int32_t q[3], const int32_t dst[3],
                         int64_t K, int32_t k, int32_t max_steps, int32_t n_peer, const int32_t* peer_pos,
                         int64_t sat, int64_t sep2, int64_t cap2, int64_t* nd_out) {
  int64_t nd = nearest_d2(S, q, K, sat);
  for (int32_t j = 0; j < n_peer; ++j) {
    int64_t d2 = d2_of(q, &peer_pos[3 * j]);
    if (d2 < nd) nd = d2;
  }
  *nd_out = nd;
  if (nd < sep2) return ORC_REJ_CONFLICT;
  if (terrain_collision(T, q)) return ORC_REJ_TERRAIN;
  if (d2_of(q, dst) < cap2) return ORC_ACCEPTED;
  if (k >= max_steps) return ORC_REJ_TIMEOUT;
  return -1;
}

int orc_cosim(const orc_params* p, const orc_terrain* T, const orc_store* S, int32_t n,
              const int32_t* src, const int32_t* dst, const int64_t* t0, int32_t cap,
              int32_t* traj, int32_t* heading, int32_t* astar, orc_result* res) {
  conv c;
  if (convert(p, &c) || n < 1 || !src || !dst || !t0 || !traj || !heading || !res || cap < 2) return ORC_E_ARG;
  if (c.vmin_u != c.vmax_u) return ORC_E_ARG;  /* co-simulation: constant-speed actions only */
  const int A = n_actions(p), W = p->W;
  const int64_t sat = c.R_max * c.R_max, sep2 = c.sep_u * c.sep_u, cap2 = c.cap_u * c.cap_u;
  int32_t* DX = (int32_t*)malloc(sizeof(int32_t) * p->HL);
  int32_t* DY = (int32_t*)malloc(sizeof(int32_t) * p->HL);
  int32_t* state = (int32_t*)malloc(sizeof(int32_t) * n);     /* -2 waiting, -1 flying, >= 0 verdict */
  int32_t* kk = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* verdict = (int32_t*)malloc(sizeof(int32_t) * n);
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * 4 * n);  /* decided next state + heading */
  int32_t* ppos = (int32_t*)malloc(sizeof(int32_t) * 3 * n);
  int32_t* pvel = (int32_t*)malloc(sizeof(int32_t) * 3 * n);
  int32_t* proj = (int32_t*)malloc(sizeof(int32_t) * 3 * A * W);
  int32_t* ppsi = (int32_t*)malloc(sizeof(int32_t) * A * W);
  int rc = ORC_OK;
  if (!DX || !DY || !state || !kk || !verdict || !next || !ppos || !pvel || !proj || !ppsi) { rc = ORC_E_NOMEM; goto out; }
  if (orc_tables(p, DX, DY)) { rc = ORC_E_ARG; goto out; }
  int64_t K = INT64_MAX;
  for (int32_t i = 0; i < n; ++i) {
    if (t0[i] < 0) { rc = ORC_E_ARG; goto out; }
    if (t0[i] < K) K = t0[i];
    state[i] = -2;
    memset(&res[i], 0, sizeof(res[i]));
    res[i].fail_step = -1;
    res[i].min_sep_d2 = sat;
  }
  for (;; ++K) {
    int32_t waiting = 0;
    for (int32_t i = 0; i < n; ++i) {  /* departures at clock K */
      if (state[i] == -2 && t0[i] == K) {
        int32_t* tr = traj + (size_t)3 * cap * i;
        int32_t* hd = heading + (size_t)cap * i;
        memcpy(tr, &src[3 * i], sizeof(int32_t) * 3);
        hd[0] = orc_initial_heading(p, &src[3 * i], &dst[3 * i]);
        state[i] = -1;
        kk[i] = 0;
      }
      if (state[i] == -2) waiting++;
    }
    int32_t flying = 0;
    for (int32_t i = 0; i < n; ++i) flying += state[i] == -1;
    if (!flying && !waiting) break;
    /* 1) terminal verdicts of every present state at clock K (others' states at K) */
    for (int32_t i = 0; i < n; ++i) {
      if (state[i] != -1) continue;
      int32_t np = 0;
      for (int32_t j = 0; j < n; ++j)
        if (j != i && state[j] == -1) { memcpy(&ppos[3 * np], traj + (size_t)3 * cap * j + 3 * kk[j], 12); np++; }
      int64_t nd;
      const int32_t* q = traj + (size_t)3 * cap * i + 3 * kk[i];
      verdict[i] = cosim_verdict(T, S, q, &dst[3 * i], K, kk[i], p->max_steps, np, ppos, sat, sep2, cap2, &nd);
      if (nd < res[i].min_sep_d2) res[i].min_sep_d2 = nd;
    }
    /* 2) decisions of the non-terminal ones, all from the states at clock K (Alg 1) */
    for (int32_t i = 0; i < n; ++i) {
      if (state[i] != -1 || verdict[i] >= 0) continue;
      if (kk[i] + 1 >= cap) { rc = ORC_E_RANGE; goto out; }
      int32_t np = 0;
      for (int32_t j = 0; j < n; ++j) {
        if (j == i || state[j] != -1) continue;
        const int32_t* trj = traj + (size_t)3 * cap * j;
        memcpy(&ppos[3 * np], trj + 3 * kk[j], 12);
        peer_velocity(DX, DY, trj, heading + (size_t)cap * j, kk[j], &pvel[3 * np]);
        np++;
      }
      const int32_t* q = traj + (size_t)3 * cap * i + 3 * kk[i];
      orc_step_out o;
      memset(&o, 0, sizeof(o));
      o.proj = proj;
      o.proj_psi = ppsi;
      if ((rc = orc_eval_step_peers(p, T, S, q, heading[(size_t)cap * i + kk[i]], &dst[3 * i], K, np, ppos, pvel, &o)))
        goto out;
      if (o.near_tie) res[i].n_near_ties += 1;
      if (astar) astar[(size_t)cap * i + kk[i]] = o.a_star;
      const int i1 = o.a_star * W;
      next[4 * i + 0] = proj[3 * i1 + 0];
      next[4 * i + 1] = proj[3 * i1 + 1];
      next[4 * i + 2] = proj[3 * i1 + 2];
      next[4 * i + 3] = ppsi[i1];
    }
    /* 3) apply: terminal aircraft leave, the others move (s_{t+1} <- Delta_1[a*]) */
    for (int32_t i = 0; i < n; ++i) {
      if (state[i] != -1) continue;
      if (verdict[i] >= 0) {
        state[i] = verdict[i];
        res[i].status = verdict[i];
        res[i].n_states = kk[i] + 1;
        res[i].fail_step = verdict[i] == ORC_ACCEPTED ? -1 : kk[i];
        continue;
      }
      kk[i] += 1;
      memcpy(traj + (size_t)3 * cap * i + 3 * kk[i], &next[4 * i], 12);
      heading[(size_t)cap * i + kk[i]] = next[4 * i + 3];
    }
  }
out:
  free(DX); free(DY); free(state); free(kk); free(verdict); free(next); free(ppos); free(pvel); free(proj); free(ppsi);
  return rc;
}

int orc_cosim_replay(const orc_params* p, const orc_terrain* T, const orc_store* S, int32_t n,
                     const int32_t* src, const int32_t* dst, const int64_t* t0, int32_t cap,
                     const int32_t* n_states, const int32_t* traj, const int32_t* heading, const int32_t* astar,
                     const int32_t* status, orc_replay_stats* st) {
  conv c;
  if (convert(p, &c) || n < 1 || !st || !n_states || !traj || !heading || !status) return ORC_E_ARG;
  const int A = n_actions(p), W = p->W;
  const int64_t sat = c.R_max * c.R_max, sep2 = c.sep_u * c.sep_u, cap2 = c.cap_u * c.cap_u;
  int32_t* DX = (int32_t*)malloc(sizeof(int32_t) * p->HL);
  int32_t* DY = (int32_t*)malloc(sizeof(int32_t) * p->HL);
  int32_t* ppos = (int32_t*)malloc(sizeof(int32_t) * 3 * n);
  int32_t* pvel = (int32_t*)malloc(sizeof(int32_t) * 3 * n);
  double* vstar = (double*)malloc(sizeof(double) * A);
  double* vsc = (double*)malloc(sizeof(double) * A);
  int32_t* proj = (int32_t*)malloc(sizeof(int32_t) * 3 * A * W);
  int32_t* ppsi = (int32_t*)malloc(sizeof(int32_t) * A * W);
  int rc = ORC_OK;
  if (!DX || !DY || !ppos || !pvel || !vstar || !vsc || !proj || !ppsi) { rc = ORC_E_NOMEM; goto out; }
  if (orc_tables(p, DX, DY)) { rc = ORC_E_ARG; goto out; }
  for (int32_t i = 0; i < n; ++i) {
    orc_replay_stats* s = &st[i];
    memset(s, 0, sizeof(*s));
    s->first_fail_step = -1;
#define FAIL(k_) do { s->n_fail++; if (s->first_fail_step < 0) s->first_fail_step = (k_); } while (0)
    const int32_t* tr = traj + (size_t)3 * cap * i;
    const int32_t* hd = heading + (size_t)cap * i;
    const int32_t ni = n_states[i];
    if (ni < 1 || ni > cap) { FAIL(0); continue; }
    if (tr[0] != src[3 * i] || tr[1] != src[3 * i + 1] || tr[2] != src[3 * i + 2]) FAIL(0);
    if (hd[0] != orc_initial_heading(p, &src[3 * i], &dst[3 * i])) FAIL(0);
    for (int32_t k = 0; k < ni; ++k) {
      const int64_t K = t0[i] + k;
      int32_t np = 0;  /* peers present at clock K in the given trajectories */
      for (int32_t j = 0; j < n; ++j) {
        const int64_t kj = K - t0[j];
        if (j == i || kj < 0 || kj >= n_states[j]) continue;
        const int32_t* trj = traj + (size_t)3 * cap * j;
        memcpy(&ppos[3 * np], trj + 3 * kj, 12);
        peer_velocity(DX, DY, trj, heading + (size_t)cap * j, (int32_t)kj, &pvel[3 * np]);
        np++;
      }
      const int32_t* q = &tr[3 * k];
      int64_t nd;
      const int v = cosim_verdict(T, S, q, &dst[3 * i], K, k, p->max_steps, np, ppos, sat, sep2, cap2, &nd);
      if (k == ni - 1) {
        if (v != (status[i] < 0 ? -1 : status[i])) FAIL(k);
        break;
      }
      if (v >= 0) { FAIL(k); break; }
      orc_step_out o;
      memset(&o, 0, sizeof(o));
      o.vstar = vstar;
      o.vstar_scale = vsc;
      o.proj = proj;
      o.proj_psi = ppsi;
      if (orc_eval_step_peers(p, T, S, q, hd[k], &dst[3 * i], K, np, ppos, pvel, &o)) { FAIL(k); break; }
      s->n_steps_checked++;
      if (o.near_tie) s->n_near_ties++;
      const int ag = astar ? astar[(size_t)cap * i + k] : o.a_star;
      if (ag < 0 || ag >= A) { FAIL(k); break; }
      if (ag != o.a_star) {
        if (vstar[o.a_star] - vstar[ag] < p->near_tie_rel * vsc[o.a_star]) s->n_divergent++;
        else FAIL(k);
      }
      const int i1 = ag * W;
      const int32_t* q1 = &tr[3 * (k + 1)];
      if (q1[0] != proj[3 * i1] || q1[1] != proj[3 * i1 + 1] || q1[2] != proj[3 * i1 + 2] || hd[k + 1] != ppsi[i1])
        FAIL(k);
    }
#undef FAIL
  }
out:
  free(DX); free(DY); free(ppos); free(pvel); free(vstar); free(vsc); free(proj); free(ppsi);
  return rc;
}

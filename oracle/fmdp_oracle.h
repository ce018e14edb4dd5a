/*
 * fmdp_oracle.h -- plain, slow, fp64/int64 CPU oracle of the FastMDP-GPU hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares no
 * code, header, table or constant generator with the CUDA product path
 * (paper_2008_03518_b200/), and the product path never imports it.
 *
 * Source of truth: /root/reference/PAPER.md ("P:n" = line n) -- Alg 1,
 * Algs 2-9, Table "Peaks created in the environment",
 * Sec. IV.I, Sec. V.  Where the paper is silent or
 * contradicts itself the reading is the one listed in DESIGN.md "Readings" (R1..R22,
 * numbered like SURVEY.md §8(c) ledger L1..L22).
 *
 * World: positions are integers in units of u metres (u = 2^-6 m by default,
 * DESIGN.md R23); every predicate (well radius, separation, capture, deck,
 * terrain) is decided exactly in int64; every value is fp64 (std pow / sqrt).
 */
#ifndef FMDP_ORACLE_H
#define FMDP_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_TURN 32
#define ORC_MAX_CLIMB 32
#define ORC_MAX_TAU 8
#define ORC_MAX_ACC 16

/* Scenario parameters in physical units; converted to integer units internally. */
typedef struct orc_params {
  double u_m;            /* metres per integer unit                                   */
  double dt_s;           /* substep duration, 0.1 s                           */
  int32_t W;             /* look-ahead substeps, 10                           */
  int32_t HL;            /* heading lattice size (divisible by 8)                     */
  double speed_mps;      /* constant ground speed v0                                  */
  int32_t n_turn;  int32_t turn_steps[ORC_MAX_TURN];   /* lattice steps per substep   */
  int32_t n_climb; int32_t climb_units[ORC_MAX_CLIMB]; /* z units per substep         */
  double goal_r, goal_gamma;                 /* 200, .999 (Table PK)            */
  double intr_r, intr_gamma;                 /* 1000, .97 (Table PK)            */
  int32_t n_tau; double tau_s[ORC_MAX_TAU]; double tau_radius_m[ORC_MAX_TAU];
                                             /* {-5,0,5,10,15} s, 300+10t m   */
  double terr_r, terr_gamma;                 /* 1000, .99 (Table PK)            */
  double deck_alt_m, deck_scale;             /* penaltyAlt, 1000 (Alg 1)    */
  double capture_m, sep_m;                   /* goal capture, separation minimum      */
  int32_t max_steps;
  int32_t vmax_init_zero;                    /* 1: literal Alg 8 V_max <- 0   */
  double near_tie_rel;                       /* 1e-4 (north star)                     */
  int32_t valuation;                         /* 0 Alg 8 max over t; 1 Alg 1 endpoint   */
  /* acceleration actions (R32): n_acc speed increments (units per
   * substep per substep), speed clamped to [speed_min, speed_max] m/s (both 0: speed held at
   * speed_mps).  A = n_turn * n_acc * n_climb, a = (i_turn * n_acc + i_acc) * n_climb + i_climb. */
  int32_t n_acc;  int32_t acc_units[ORC_MAX_ACC];
  double speed_min_mps, speed_max_mps;
} orc_params;

/* Terrain: manually placed wells (Table PK) + a height raster for collision. */
typedef struct orc_terrain {
  int32_t n_wells;
  const int32_t* center;   /* [n_wells][3] units            */
  const int32_t* radius;   /* [n_wells] units               */
  int32_t nx, ny;          /* raster size (0 = no raster)   */
  int32_t x0, y0, cell;    /* raster origin / cell, units   */
  const int32_t* height;   /* [ny][nx] ground height, units */
} orc_terrain;

typedef struct orc_store orc_store;   /* accepted-plan DB */

/* Per-step outputs; every pointer may be NULL. Sizes: A = n_turn*n_climb, W. */
typedef struct orc_step_out {
  double* v_pos;     /* [A*W] V+  (Alg 4)                   */
  double* v_int;     /* [A*W] V^I (Alg 7)                   */
  double* v_ter;     /* [A*W] V^T (Alg 6)                   */
  double* v_alt;     /* [A*W] hard-deck penalty             */
  double* v;         /* [A*W] V (Alg 8)               */
  double* scale;     /* [A*W] V+ + max(V^T,V^I) + V_alt      */
  double* vstar;     /* [A]   V* (Alg 8)           */
  double* vstar_scale; /* [A] term scale at the maximising t */
  int64_t* conf_d2;  /* [A]   min d^2 of Delta_1(a) to row K+1, saturated */
  int32_t* proj;     /* [A*W*3] projected states            */
  int32_t* proj_psi; /* [A*W] projected headings            */
  int32_t a_star;    /* Alg 9                                */
  int32_t a_second;  /* runner-up (lowest index among ties)  */
  double gap;        /* V*(a*) - V*(a_second)                */
  int32_t near_tie;  /* gap < near_tie_rel * vstar_scale[a*] */
  double* v_neg;     /* [A*W] V^- (Alg 5; batch peers) */
  int32_t* proj_v;   /* [A*W] projected speeds (units per substep, R32) */
} orc_step_out;

typedef struct orc_result {
  int32_t status;     /* 0 ACCEPTED, 1 REJ_CONFLICT, 2 REJ_TERRAIN, 3 REJ_TIMEOUT */
  int32_t n_states;
  int32_t fail_step;  /* step of the terminal verdict (-1 if accepted)             */
  int32_t n_near_ties;
  int64_t min_sep_d2; /* min over steps of nearest-plan d^2, saturated at R_max^2  */
} orc_result;

typedef struct orc_replay_stats {
  int32_t n_steps_checked;
  int32_t n_fail;        /* transitions / verdicts the oracle cannot reproduce  */
  int32_t n_divergent;   /* a*_gpu != a*_orc at a logged near-tie (allowed)      */
  int32_t n_near_ties;   /* oracle near-tie count along the replayed trajectory  */
  int32_t first_fail_step;
  double max_vstar_err;  /* unused by the C replay (values compared in eval tests) */
} orc_replay_stats;

enum { ORC_OK = 0, ORC_E_ARG = -1, ORC_E_NOMEM = -2, ORC_E_RANGE = -7 };
enum { ORC_ACCEPTED = 0, ORC_REJ_CONFLICT = 1, ORC_REJ_TERRAIN = 2, ORC_REJ_TIMEOUT = 3 };

int orc_check_params(const orc_params* p);
/* OpenMP threads for the per-state loops of a decision step (timing only; results identical). */
int orc_set_threads(int n);
int orc_tables(const orc_params* p, int32_t* DX, int32_t* DY);
int32_t orc_initial_heading(const orc_params* p, const int32_t src[3], const int32_t dst[3]);
int orc_build_wells(const orc_params* p, const int32_t pos[3], const int32_t vel[3],
                    int32_t* centers, int64_t* radius_u);
int orc_project(const orc_params* p, const int32_t q[3], int32_t psi, int32_t* states, int32_t* psi_out);
/* Acceleration actions: projection from speed v (units per substep). */
int orc_project_v(const orc_params* p, const int32_t q[3], int32_t psi, int32_t v, int32_t* states,
                  int32_t* psi_out, int32_t* v_out);
void orc_direction(int32_t HL, int64_t v, int32_t psi, int32_t* dx, int32_t* dy);
int32_t orc_initial_speed(const orc_params* p);
double orc_goal_value(const orc_params* p, int64_t d2);
double orc_well_value(double r, double gamma, double u_m, int64_t d2, int64_t R_u);
double orc_deck_penalty(const orc_params* p, int32_t z);

orc_store* orc_store_new(void);
void orc_store_free(orc_store* s);
int orc_store_add(orc_store* s, int64_t t0, int32_t n, const int32_t* states);
int32_t orc_store_count(const orc_store* s);
int orc_store_sample(const orc_store* s, int32_t plan, int64_t K, int32_t pos[3], int32_t vel[3]);

int orc_eval_step(const orc_params* p, const orc_terrain* T, const orc_store* S,
                  const int32_t q[3], int32_t psi, const int32_t g[3], int64_t K, orc_step_out* out);
/* Alg 2-9 with batch peers (Alg 5, Table DS P:397 P^-): n_peer other
 * aircraft of a co-simulated batch at clock K, each with position and linear velocity (per
 * substep); they add five wells each (Table PK "aircraft" row, like an intruder). */
int orc_eval_step_peers(const orc_params* p, const orc_terrain* T, const orc_store* S,
                        const int32_t q[3], int32_t psi, const int32_t g[3], int64_t K, int32_t n_peer,
                        const int32_t* peer_pos, const int32_t* peer_vel, orc_step_out* out);
int orc_schedule(const orc_params* p, const orc_terrain* T, const orc_store* S,
                 const int32_t src[3], const int32_t dst[3], int64_t t0, int32_t cap,
                 int32_t* traj, int32_t* heading, int32_t* astar, orc_result* res);
int orc_eval_step_v(const orc_params* p, const orc_terrain* T, const orc_store* S, const int32_t q[3], int32_t psi,
                    int32_t v, const int32_t g[3], int64_t K, orc_step_out* out);
int orc_schedule_v(const orc_params* p, const orc_terrain* T, const orc_store* S,
                   const int32_t src[3], const int32_t dst[3], int64_t t0, int32_t cap,
                   int32_t* traj, int32_t* heading, int32_t* speed, int32_t* astar, orc_result* res);
int orc_replay_v(const orc_params* p, const orc_terrain* T, const orc_store* S,
                 const int32_t src[3], const int32_t dst[3], int64_t t0,
                 int32_t n, const int32_t* traj, const int32_t* heading, const int32_t* speed, const int32_t* astar,
                 int32_t status, orc_replay_stats* st);
int orc_schedule_batch(const orc_params* p, const orc_terrain* T, orc_store* S, int32_t n,
                       const int32_t* src, const int32_t* dst, const int64_t* t0, int32_t cap,
                       int32_t* traj, int32_t* heading, int32_t* astar, orc_result* res);
/* Co-simulated batch (Alg 1 P:151-237 synchronous update, Alg 5, Table DS
 * "Determine terminal state N x N"): the n aircraft share one clock K; aircraft i is present
 * at K for t0[i] <= K until its terminal state.  At every clock each present aircraft sees the
 * others' wells and separation; all decide, then all move.  traj/heading/astar: n blocks of
 * cap states; res[n].  S is not modified (the caller appends the accepted plans). */
int orc_cosim(const orc_params* p, const orc_terrain* T, const orc_store* S, int32_t n,
              const int32_t* src, const int32_t* dst, const int64_t* t0, int32_t cap,
              int32_t* traj, int32_t* heading, int32_t* astar, orc_result* res);
/* Lockstep replay of a co-simulated batch: every aircraft's steps and verdicts recomputed with
 * its peers taken from the given trajectories; st[n]. */
int orc_cosim_replay(const orc_params* p, const orc_terrain* T, const orc_store* S, int32_t n,
                     const int32_t* src, const int32_t* dst, const int64_t* t0, int32_t cap,
                     const int32_t* n_states, const int32_t* traj, const int32_t* heading, const int32_t* astar,
                     const int32_t* status, orc_replay_stats* st);
/* status -1 replays a prefix (the last given state must not be terminal). */
int orc_replay(const orc_params* p, const orc_terrain* T, const orc_store* S,
               const int32_t src[3], const int32_t dst[3], int64_t t0,
               int32_t n, const int32_t* traj, const int32_t* heading, const int32_t* astar,
               int32_t status, orc_replay_stats* st);

#ifdef __cplusplus
}
#endif
#endif

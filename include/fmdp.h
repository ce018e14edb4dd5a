/*
 * fmdp.h -- C ABI of the B200-native FastMDP-GPU hot path (arXiv 2008.03518).
 *
 * Paper passages are cited as P:n = line n of the paper source; the readings
 * of ambiguous passages (R1..R31) are listed in DESIGN.md "Readings".
 *
 * Model (one request = one aircraft, N = 1):
 *   At every 0.1 s step k of the requesting aircraft's trajectory (Fig 3a loop P:272-289)
 *   every action a = (turn, climb) is projected W substeps ahead (Alg 3) and
 *   each projected state s_{a,t} is valued with Alg 8:
 *       V(a,t) = V+(a,t) - max(V^T(a,t), V^I(a,t)) - V_alt(a,t)
 *       V+  = 200 * .999^d(goal)                     (Alg 4, Table PK)
 *       V^I = max over accepted plans j active at the step's time row and
 *             tau in {-5,0,5,10,15} s of [d < 300+10 tau] 1000 * .97^d
 *             around p_j + v_j tau                   (Alg 7, Table PK)
 *       V^T = max over terrain wells of [d < R] 1000 * .99^d   (Alg 6, Table PK)
 *       V_alt = 1000 - z if z < deck else 0          (Alg 1, R6/R7)
 *   V*(a) = max_t V(a,t) (Alg 8; airspace.valuation = 1: V(a,W), Alg 1),
 *   a* = argmax (Alg 9, lowest index on ties),
 *   the aircraft advances one substep along a* (Alg 1), and the terminal state is
 *   determined (Sec IV.I): separation conflict with any accepted plan (exact),
 *   terrain, goal capture, timeout.  An accepted trajectory is appended to the plan store
 *   (Sec V) and constrains every later request (first-come-first-served).
 *
 * Units: positions are integers in units of airspace.u_m metres (2^-6 m by default,
 *   R23); fmdp_vec3 arguments are metres and are quantised with llrint(x / u_m)
 *   (round half to even).  Time is an integer step index ("clock row") of dt seconds.
 *
 * Conventions (all functions):
 *   - Every function returns fmdp_status (0 = OK, < 0 = error) and never throws.
 *   - A REJECTION IS NOT AN ERROR: fmdp_schedule returns FMDP_OK with
 *     res->status != FMDP_ACCEPTED ("otherwise an error is reported" is the
 *     request-level status, not an API failure).
 *   - The context owns all device memory; input arrays are copied before return and may
 *     be freed by the caller; output buffers are caller-allocated with a capacity; a
 *     too-small buffer yields FMDP_E_BUFFER and the required size in *n / n_states.
 *   - One context = one FCFS sequence; calls on one context must be serialised by the
 *     caller.  Different contexts are independent.
 *   - Results are deterministic and bit-identical across runs, batch speculation and
 *     launch configuration (every reduction on the path is an exact min/max).
 *   - The library requires an sm_100a device; without one fmdp_create fails with
 *     FMDP_E_NODEV.  There is no CPU fallback.
 */
#ifndef FMDP_H
#define FMDP_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMDP_ABI_VERSION 3  /* 2: fmdp_airspace.valuation; 3: acceleration actions (n_acc ...) */

typedef struct fmdp_ctx fmdp_ctx; /* opaque; owns device memory, plan store, scratch */
typedef int32_t fmdp_status;

enum {
  FMDP_OK = 0,
  FMDP_E_ARG = -1,       /* invalid argument / scenario                                 */
  FMDP_E_NOMEM = -2,     /* host or device allocation failed                            */
  FMDP_E_CUDA = -3,      /* CUDA runtime error (fmdp_last_error has the text)           */
  FMDP_E_CAPACITY = -4,  /* a time row would exceed airspace.row_capacity               */
  FMDP_E_DUPLICATE = -5, /* reserved (plan ids are assigned by the library)             */
  FMDP_E_BUFFER = -6,    /* output buffer too small; required size returned             */
  FMDP_E_RANGE = -7,     /* position outside the airspace / 2^24-unit span, or a plan   */
                         /* running past horizon_steps, or |velocity| beyond packing    */
  FMDP_E_NODEV = -8,     /* no sm_100 device                                            */
  FMDP_E_IO = -9,        /* plan-store file could not be opened / read / written, or is */
                         /* not a plan-store file (fmdp_save_plans / fmdp_load_plans)   */
  FMDP_E_INTERNAL = -99
};

/* Request status (fmdp_result.status). */
enum { FMDP_ACCEPTED = 0, FMDP_REJ_CONFLICT = 1, FMDP_REJ_TERRAIN = 2, FMDP_REJ_TIMEOUT = 3 };

typedef struct { double x, y, z; } fmdp_vec3;   /* metres, local ENU                      */
typedef struct { int32_t x, y, z; } fmdp_qpos;  /* integer units of u_m                   */

/* Scenario.  Defaults (DESIGN.md Appendix A) are filled by fmdp_airspace_default(). */
typedef struct fmdp_airspace {
  uint32_t abi_version;            /* = FMDP_ABI_VERSION                                */
  fmdp_vec3 lo, hi;                /* airspace bounds, metres; span < 2^24 units         */
  double u_m;                      /* metres per position unit (2^-6)                    */
  double dt;                       /* substep, 0.1 s                             */
  int32_t window;                  /* W = 10 look-ahead substeps                 */
  double speed;                    /* constant ground speed v0, m/s; v0*dt/u integral    */
  int32_t heading_lattice;         /* H_L headings, divisible by 8 (R14)                 */
  int32_t n_turn;                  /* <= 32                                              */
  const int32_t* turn_steps;       /* lattice steps per substep, ascending; |step| * window
                                      < heading_lattice (FMDP_E_ARG otherwise)            */
  int32_t n_climb;                 /* 1, 3 or 5                                          */
  const int32_t* climb_units;      /* z units per substep, ascending                     */
  double goal_r, goal_gamma;       /* 200, 0.999 (Table PK, R8)                    */
  double intr_r, intr_gamma;       /* 1000, 0.97 (Table PK)                        */
  int32_t n_tau;                   /* <= 5                                               */
  const double* tau_s;             /* {-5,0,5,10,15} s; tau/dt integral (R9)             */
  const double* tau_radius_m;      /* 300 + 10 tau m; multiples of u; max < 1024 m       */
  double terr_r, terr_gamma;       /* 1000, 0.99 (Table PK)                        */
  double deck_alt_m, deck_scale;   /* 30 m, 1000 (Alg 1, R7)                   */
  double capture_radius_m;         /* goal capture, 100 m (R16)                          */
  double sep_min_m;                /* separation minimum, 150 m (R15)                    */
  int32_t max_steps;               /* timeout                                            */
  int32_t vmax_init_zero;          /* 0: V_max <- -inf (R2, default); 1: literal P:736   */
  double near_tie_rel;             /* 1e-4: near-tie threshold for logging               */
  int64_t horizon_steps;           /* number of time rows in the plan store              */
  int32_t row_capacity;            /* plan slots per time row (multiple of 4)            */
  int32_t valuation;               /* 0: Alg 8 V*(a) = max over the window;  */
                                   /* 1: Alg 1 endpoint only, V*(a) = V(Delta_10(a))     */
                                   /*    (R31)           */
  /* Acceleration actions (the paper's A = 1350, Table DS / KI captions P:387,
   * P:417; SPEC 15 x 10 x 9; R32).  The action becomes (turn, speed increment, climb),
   * index a = (i_turn * n_acc + i_acc) * n_climb + i_climb; per substep psi += turn, v = clamp(v
   * + acc, [speed_min, speed_max]), position += (D(psi, v), climb) with D the heading lattice of
   * step length v (units per substep).  n_acc = 1 with acc_units = {0} and speed_min = speed_max
   * = 0 is the constant-speed model.  With acceleration actions n_climb must be 3 or 10; every
   * request then runs alone on the whole GPU (action space tiled over the clusters, the tiles'
   * top-2 exchanged per step); batches are sequential; co-simulation, departures and the
   * multi-GPU entry points return FMDP_E_ARG. */
  int32_t n_acc;                   /* <= 16                                              */
  const int32_t* acc_units;        /* speed increments, units per substep per substep     */
  double speed_min;                /* m/s; speed_min <= speed <= speed_max, multiples of  */
  double speed_max;                /* u per dt                                            */
} fmdp_airspace;

/* Terrain: manually placed wells (Table PK) and a ground-height raster used only
 * for the terrain-collision verdict (R16).  All integer units. */
typedef struct fmdp_terrain {
  int32_t n_wells;
  const fmdp_qpos* center;         /* [n_wells]                                          */
  const int32_t* radius_u;         /* [n_wells]                                          */
  int32_t nx, ny;                  /* raster cells (0 = no raster)                       */
  int32_t x0_u, y0_u, cell_u;      /* raster origin and cell size                        */
  const int32_t* height_u;         /* [ny][nx] ground height                             */
} fmdp_terrain;

/* Device / launch configuration (NULL = current device, default stream, cudaMalloc). */
typedef struct fmdp_devices {
  int32_t device;                                   /* CUDA ordinal                      */
  void* stream;                                     /* cudaStream_t or NULL              */
  void* (*alloc)(size_t bytes, void* user);         /* optional device allocator         */
  void (*release)(void* ptr, void* user);
  void* user;
} fmdp_devices;

typedef struct fmdp_launch {
  int32_t cluster_size;   /* CTAs cooperating on one trajectory (1..16), 0 = auto        */
  int32_t max_walkers;    /* concurrent trajectories in a batch round, 0 = auto          */
  int32_t threads;        /* cap on threads per CTA (fewer plan groups per warp), 0 = auto */
  int32_t profile;        /* 1: per-phase cycles of CTA 0 (fmdp_stats), FCFS walks only;  */
                          /*    they then run in the reference kernel instantiation      */
  int32_t step_budget;    /* batch: steps the non-head walkers of a slice may run past the head's end, 0 = auto (2) */
  int32_t cull;           /* 1: SURVEY f1 exact culling -- skip plans none of whose wells can */
                          /* reach a projected state (outputs bit-identical)               */
  int32_t split;          /* single-request walks (fmdp_schedule, FMDP_BATCH_SEQUENTIAL):  */
                          /* clusters sharing one request, each over a shard of every time */
                          /* row, combined per step by the in-kernel exchange of           */
                          /* fmdp_schedule_p2p (outputs bit-identical).  0 = auto (cost    */
                          /* model: large stores), 1 = off, 2..8 = that many clusters      */
} fmdp_launch;

typedef struct fmdp_request {
  uint64_t aircraft_id;
  fmdp_vec3 src, dst;      /* metres                                                     */
  int64_t t0_step;         /* departure clock row                                        */
} fmdp_request;

typedef struct fmdp_result {
  int32_t status;          /* FMDP_ACCEPTED / FMDP_REJ_*                                 */
  uint32_t plan_id;        /* valid if ACCEPTED                                          */
  int32_t n_states;        /* trajectory length (states 0..n-1 at rows t0..t0+n-1)       */
  int32_t fail_step;       /* step of the rejecting verdict, -1 if accepted              */
  double min_sep_m;        /* min distance to any accepted plan along the trajectory,    */
                           /* saturated at the largest well radius (450 m)               */
  int32_t n_near_ties;     /* steps whose top-2 V* gap < near_tie_rel * term scale       */
  int32_t n_exact;         /* (state,tau) minima resolved by the exact fallback          */
} fmdp_result;

/* Per-call counters of the last schedule / schedule_batch call. */
typedef struct fmdp_stats {
  int64_t steps;           /* decision steps executed on the device (incl. re-runs)      */
  int64_t pair_evals;      /* (projected state, well) pairs evaluated in the hot loop    */
  int32_t rounds;          /* walk launches (speculative FCFS slices)                      */
  int32_t reruns;          /* rollbacks: trajectories resumed from an earlier step after an */
                           /* earlier request's commit could influence them               */
  int32_t cluster_size;
  int32_t walkers;
  int32_t kernels;         /* kernel launches                                             */
  double device_ms;        /* sum of walk-kernel device time (CUDA events)                */
  int64_t phase_cycles[17]; /* profile=1: CTA-0 cycles per phase: projection, goal/terrain, */
                           /* row wait, hot loop, stage, reduce-scatter, barrier 1,         */
                           /* owner epilogue, barrier 2, decide                             */
  int32_t split;           /* clusters that shared the last single-request walk (launch.split) */
  int32_t reconverged;     /* re-walks after a rollback that met the request's previous run */
                           /* and took it over (schedule_batch)            */
} fmdp_stats;

/* Fill *a with the defaults of DESIGN.md Appendix A (the arrays point to static storage). */
void fmdp_airspace_default(fmdp_airspace* a);

/* Create a context on one device.  Copies airspace and terrain (wells to device,
 * raster to device).  Errors: E_ARG (invalid scenario), E_NODEV, E_NOMEM, E_CUDA. */
fmdp_status fmdp_create(const fmdp_airspace* airspace, const fmdp_terrain* terrain,
                        const fmdp_devices* devs, fmdp_ctx** out);
void fmdp_destroy(fmdp_ctx* ctx);

/* Launch tuning (NULL resets to auto). */
fmdp_status fmdp_set_launch(fmdp_ctx* ctx, const fmdp_launch* launch);

/* Import an externally produced plan: n >= 1 states at rows t0..t0+n-1.
 * Velocities are the forward differences (R11) and must fit the packed store record
 * (|vx|,|vy| <= 1023, |vz| <= 511 units/step) else E_RANGE.  Rows past horizon ->
 * E_RANGE; full rows -> E_CAPACITY (nothing is stored).  *plan_id receives the id. */
fmdp_status fmdp_add_plan(fmdp_ctx* ctx, uint64_t aircraft_id, int64_t t0_step, int32_t n,
                          const fmdp_qpos* states, int32_t flags, uint32_t* plan_id);

/* Bulk import of n_plans plans in order (ids first_id..first_id+n_plans-1); states are
 * concatenated.  aircraft_ids may be NULL.  All-or-nothing. */
fmdp_status fmdp_add_plans(fmdp_ctx* ctx, int32_t n_plans, const uint64_t* aircraft_ids,
                           const int64_t* t0_steps, const int32_t* n_states,
                           const fmdp_qpos* states, uint32_t* first_id);

/* Schedule one request against every accepted plan (Sec V) and append it on
 * acceptance.  traj receives n_states states (cap traj_cap; E_BUFFER if smaller than
 * max_steps + 1).  Request errors: src == dst, outside the airspace -> E_ARG / E_RANGE;
 * t0 + max_steps + 1 >= horizon -> E_RANGE. */
fmdp_status fmdp_schedule(fmdp_ctx* ctx, uint64_t aircraft_id, fmdp_vec3 src, fmdp_vec3 dst,
                          int64_t t0_step, fmdp_result* res, fmdp_qpos* traj, int32_t traj_cap);

/* First-come-first-served batch: results identical to calling fmdp_schedule on each
 * request in array order.  Default implementation: speculative rounds against a store
 * snapshot + exact influence test + in-order commit; with f1 culling
 * (fmdp_launch.cull) a rolled-back request's re-walk takes over its previous run once its state
 * meets it past every step a newly committed plan can influence (fmdp_stats.reconverged; DESIGN.md
 * §6) -- same results.
 * flags: FMDP_BATCH_SEQUENTIAL forces the plain loop.
 * traj: n * traj_cap_each states (may be NULL to skip trajectory output). */
#define FMDP_BATCH_SEQUENTIAL 1
fmdp_status fmdp_schedule_batch(fmdp_ctx* ctx, const fmdp_request* reqs, int32_t n,
                                fmdp_result* res, fmdp_qpos* traj, int32_t traj_cap_each,
                                int32_t flags);

/* Request-sharded FCFS batch over several GPUs (SURVEY §8(e) "second partitioning"
 * "independent parallel instances" made exact): every rank holds the same store (the same plans
 * added in the same order) and calls this collectively with the same requests.  Request i is walked
 * by rank i % world; after every speculative round the ranks all-gather the requests that finished
 * in it (status, trajectory, headings, actions, near-tie flags: n * 37 bytes + 40 per request), so
 * every rank takes the same in-order commit and rollback decisions and appends the
 * same plans.  Results -- on every rank -- are identical to fmdp_schedule_batch on one GPU.
 * allgather: every rank contributes `bytes` bytes at `send`; on return `recv` holds world blocks of
 * `bytes` bytes in rank order (e.g. ncclAllGather / gloo); 0 on success, else the call fails with
 * FMDP_E_INTERNAL.  Not with acceleration actions. */
typedef struct fmdp_gather {
  int32_t rank, world;
  int32_t (*allgather)(const void* send, void* recv, int64_t bytes, void* user);
  void* user;
} fmdp_gather;
fmdp_status fmdp_schedule_batch_dist(fmdp_ctx* ctx, const fmdp_gather* gather, const fmdp_request* reqs, int32_t n,
                                     fmdp_result* res, fmdp_qpos* traj, int32_t traj_cap_each);

/* Plan-sharded multi-GPU scheduling, host-stepped reference path.
 * Every rank holds the same store (plans added identically on all ranks) and evaluates only
 * its shard of every time row (slots [n*rank/world, n*(rank+1)/world)).  Per decision step
 * the per-(projected state, tau) minimum squared distances (FP32 bits) and the nearest-plan
 * distance (uint32) -- A*W*5 + 1 values -- are combined with allreduce_min_u32 (in place,
 * elementwise MIN over ranks, e.g. ncclAllReduce(ncclMin) / gloo); every rank then takes the
 * identical decision.  Minima are exact, so results are bit-identical to one GPU.
 * Collective call: every rank must call it with the same request.  The callback returns 0
 * on success. */
typedef struct fmdp_shard {
  int32_t rank, world;
  int32_t (*allreduce_min_u32)(uint32_t* host_buf, int32_t count, void* user);
  void* user;
} fmdp_shard;
fmdp_status fmdp_schedule_sharded(fmdp_ctx* ctx, const fmdp_shard* shard, uint64_t aircraft_id, fmdp_vec3 src,
                                  fmdp_vec3 dst, int64_t t0_step, fmdp_result* res, fmdp_qpos* traj,
                                  int32_t traj_cap);

/* Plan-sharded multi-GPU scheduling, production form (SURVEY §8(e) "Mechanism"): the same
 * partitioning and decisions as fmdp_schedule_sharded, but the per-step exchange runs INSIDE
 * one persistent walker launch per request -- no host round-trip per step.  Each step the owner
 * CTA of every (projected state, tau) item on rank r stores {its minimum (FP32 bits), step tag}
 * as ONE 8-byte word into slot [step parity][r] of every peer's exchange area (P2P stores over
 * NVLink / NVSwitch) and polls its own area until the peers' words carry this step's tag (value
 * and readiness arrive together: no fence, no flag); CTA 0 does the same for the nearest-plan
 * distance and broadcasts the minimum over its cluster.  Every rank then decides identically,
 * so results are bit-identical to one GPU.  Each rank may run k clusters (fmdp_launch.split,
 * auto from the cost model on its shard; every rank must use the same settings): the clusters
 * of a GPU first exchange among themselves, then cluster c of every GPU with cluster c of the
 * others (two-level exchange; plan shard g*k + c of N*k).
 *
 * Setup (collective, once, before any fmdp_schedule_p2p):
 *   1. fmdp_p2p_export(ctx, world, &handle, &ptr): allocates this rank's exchange area
 *      (cudaMalloc, zeroed: 16 cluster blocks of 2 * world * (A*W*5 + 16) 8-byte words) and
 *      returns its CUDA IPC
 *      handle (64 bytes; zeroed if IPC is unavailable) and its device pointer.
 *   2. exchange (handle, ptr) among the ranks (e.g. torch.distributed.all_gather_object).
 *   3. fmdp_p2p_connect(ctx, rank, world, handles[world], ptrs[world]): peer q's area is
 *      ptrs[q] when ptrs != NULL and ptrs[q] != NULL (the same process: contexts on one or
 *      several devices; peer access is enabled), else cudaIpcOpenMemHandle(handles[q]).
 *      Resets this rank's area and tag sequence; every rank must connect before any rank
 *      schedules.
 * fmdp_schedule_p2p: collective -- every rank calls it with the same request, on identical
 * stores (the same plans added in the same order; large rows are sorted by x-y cell the same
 * deterministic way on every rank before a sharded call) and launch settings (the cluster size
 * must agree), concurrently (the walkers wait for
 * each other every step).  A peer whose words do not arrive within ~2 s (~8 s for a launch's
 * first step) makes the call return FMDP_E_CUDA ("peer exchange timed out"); the store is not
 * changed; export and connect again before the next call.  world <= 8. */
typedef struct fmdp_p2p_handle {
  unsigned char bytes[64];
} fmdp_p2p_handle;
fmdp_status fmdp_p2p_export(fmdp_ctx* ctx, int32_t world, fmdp_p2p_handle* handle, void** dev_ptr);
fmdp_status fmdp_p2p_connect(fmdp_ctx* ctx, int32_t rank, int32_t world, const fmdp_p2p_handle* handles,
                             void* const* dev_ptrs);
fmdp_status fmdp_schedule_p2p(fmdp_ctx* ctx, uint64_t aircraft_id, fmdp_vec3 src, fmdp_vec3 dst, int64_t t0_step,
                              fmdp_result* res, fmdp_qpos* traj, int32_t traj_cap);

/* Departure-time candidates ("recommended take-off time"):
 * schedule one request for n_delays candidate departures t0_step + delays[i] in parallel, all
 * against the current store (the candidates are alternatives, they do not see each other);
 * the accepted candidate with the earliest departure (ties: lowest index) is appended and its
 * index returned in *chosen (-1 if none).  res[n_delays]; traj: n_delays * traj_cap states or
 * NULL.  Each res[i] equals fmdp_schedule of that candidate alone (without the append). */
fmdp_status fmdp_schedule_departures(fmdp_ctx* ctx, uint64_t aircraft_id, fmdp_vec3 src, fmdp_vec3 dst,
                                     int64_t t0_step, int32_t n_delays, const int64_t* delays, fmdp_result* res,
                                     fmdp_qpos* traj, int32_t traj_cap, int32_t* chosen);

/* Co-simulated batch ("multiple aircraft being co-simulated together with the
 * same set of accepted flights ... aware of each other"; Alg 1 P:230-235 synchronous update;
 * Alg 5 P:598-631 and Table DS P:397 P^- wells; Table DS "Determine terminal state" N x N).
 * The n requests fly on one clock K (request i from K = t0_step until its terminal state): at
 * every clock each airborne aircraft sees the five wells of every other airborne batch
 * aircraft (position, and velocity = its last displacement; R28) next to the
 * accepted plans, all decide from the states at K, then all move.  Two batch aircraft closer
 * than sep_m at a clock are both rejected for conflict; min_sep_m includes batch peers.
 * Accepted trajectories (mutually separated) are appended in array order; the store is not
 * changed during the batch.  All n walkers run concurrently: n <= fmdp_cosim_max(ctx), else
 * FMDP_E_CAPACITY.  res[n]; traj: n * traj_cap_each states or NULL. */
fmdp_status fmdp_schedule_cosim(fmdp_ctx* ctx, const fmdp_request* reqs, int32_t n, fmdp_result* res, fmdp_qpos* traj,
                                int32_t traj_cap_each);
/* Largest co-simulated batch the device can run (co-resident walkers). */
int32_t fmdp_cosim_max(fmdp_ctx* ctx);

/* Speed of every state of the last trajectory of request `index` (units per substep; the
 * constant speed*dt/u without acceleration actions).  E_BUFFER (required size in *n) if cap is
 * smaller than the trajectory. */
fmdp_status fmdp_get_speeds(fmdp_ctx* ctx, int32_t index, int32_t* speed, int32_t cap, int32_t* n);

/* Per-step log of the last trajectory of request `index` of the last schedule /
 * schedule_batch call: action a*_k, heading psi_k, and near-tie flag per step (k < n).
 * Any pointer may be NULL. */
fmdp_status fmdp_get_steplog(fmdp_ctx* ctx, int32_t index, int32_t* astar, int32_t* heading,
                             int32_t* near_tie, int32_t cap, int32_t* n);

/* Parity trace of the walk kernels themselves (north-star tolerance check on the path the batch
 * actually runs): after fmdp_set_trace(ctx, m) every later schedule / schedule_batch call records,
 * for its requests 0..m-1, V*(a) (Alg 8) and its term scale S(a) = V+ + max(V^T,V^I) +
 * V_alt at the maximising substep (R25) of every decision step, in whichever kernel
 * instantiation (full, culled, split slices) computes that step -- a step re-run after a
 * speculative rollback overwrites its entry.  m = 0 turns it off.  Device memory: m * (max_steps
 * + 2) * A * 16 bytes.  Errors: E_ARG (m < 0), E_NOMEM. */
fmdp_status fmdp_set_trace(fmdp_ctx* ctx, int32_t n_requests);
/* The trace of request `index` (< m) of the last call: vstar / scale [k * A + a] for the decision
 * steps k = 0..n-2 (n = n_states); *n receives n - 1.  cap_steps < n - 1 -> E_BUFFER.  Either
 * pointer may be NULL.  E_ARG if the request was not traced. */
fmdp_status fmdp_get_trace(fmdp_ctx* ctx, int32_t index, double* vstar, double* scale, int32_t cap_steps,
                           int32_t* n);

fmdp_status fmdp_get_plan(fmdp_ctx* ctx, uint32_t plan_id, int64_t* t0_step, fmdp_qpos* buf,
                          int32_t cap, int32_t* n);
fmdp_status fmdp_num_plans(const fmdp_ctx* ctx, uint32_t* n);

/* Remove every plan with id >= n_plans (restores the store of an earlier moment). */
fmdp_status fmdp_truncate(fmdp_ctx* ctx, uint32_t n_plans);

/* Plan-store persistence (the accepted flight plans are "loaded from a file" at start-up and
 * every newly accepted plan is added to it).  fmdp_save_plans writes plans
 * [first_id, num_plans) in id order to `path` (created / truncated); fmdp_load_plans appends every
 * plan of the file to the store through fmdp_add_plans (same validation: E_RANGE / E_CAPACITY leave
 * the plans before the offending chunk committed) and returns the first new id in *first_id (may be
 * NULL).  File layout, little-endian: "FMDPPLN1" (8 bytes), uint32 version = 1, uint32 reserved = 0,
 * uint64 n_plans; then per plan: uint64 aircraft_id, int64 t0_step, int32 n, int32 reserved = 0,
 * n x {int32 x, y, z} (the quantised states, u = 2^-6 m).  Positions are stored in units, so a file
 * loads into any context whose airspace and horizon contain them.  Errors: E_ARG (null ctx/path,
 * first_id > num_plans), E_IO (open / short read / write failure / bad magic or version). */
fmdp_status fmdp_save_plans(const fmdp_ctx* ctx, const char* path, uint32_t first_id);
fmdp_status fmdp_load_plans(fmdp_ctx* ctx, const char* path, uint32_t* first_id);

/* One decision step at (pos, heading) for goal `goal` at clock row `clock_step`, run by
 * the same device code as fmdp_schedule (parity / debug hook; V mirrors Table DS "V",
 * P:405).  Outputs (host pointers, any may be NULL except vstar):
 *   vstar[A], v_at[A*W], scale_at[A*W] (V+ + max(V^T,V^I) + V_alt), conflict[A] (1 if
 *   Delta_1(a) is within sep of a plan at row clock+1, i.e. choosing a would end the
 *   request with a separation conflict at the next step), min_d2[A+1] (saturated min d^2
 *   of Delta_1(a) to row clock+1; entry A: pos to row clock), *a_star. */
fmdp_status fmdp_eval_step(fmdp_ctx* ctx, fmdp_qpos pos, int32_t heading, fmdp_qpos goal,
                           int64_t clock_step, double* vstar, double* v_at, double* scale_at,
                           int32_t* conflict, int64_t* min_d2, int32_t* a_star);

/* The same from speed speed_u (units per substep; <= 0: the airspace's speed), for acceleration
 * actions (airspace.n_acc; R32).  E_ARG if speed_u lies outside [speed_min, speed_max]. */
fmdp_status fmdp_eval_step_v(fmdp_ctx* ctx, fmdp_qpos pos, int32_t heading, int32_t speed_u, fmdp_qpos goal,
                             int64_t clock_step, double* vstar, double* v_at, double* scale_at, int32_t* conflict,
                             int64_t* min_d2, int32_t* a_star);

fmdp_status fmdp_get_stats(const fmdp_ctx* ctx, fmdp_stats* out);
int32_t fmdp_num_actions(const fmdp_ctx* ctx);
const char* fmdp_strerror(fmdp_status s);
/* Text of the context's last error; with ctx == NULL, the reason this thread's last
 * fmdp_create failed. */
const char* fmdp_last_error(const fmdp_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FMDP_H */

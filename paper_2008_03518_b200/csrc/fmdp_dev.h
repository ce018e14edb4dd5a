// fmdp_dev.h -- device data layout shared by the host library (fmdp_host.cu) and the
// kernels (fmdp_walk.cu).  Product code; independent of oracle/.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace fmdp {

constexpr int NTAU = 5;         // intruder wells per plan (Table PK: "5 rewards")
constexpr int MAX_TURN = 32;
constexpr int MAX_CLIMB = 10;
constexpr int MAX_ACC = 16;     // speed increments of the acceleration actions
constexpr int WIDE_G = 8;       // cluster size of the wide (action-tiled) walker
constexpr int WIDE_HPT = 9;     // horizontal paths (turn, acceleration) per cluster tile (135 / 9 = 15
                                // clusters of 8 CTAs: co-resident on 148 SMs)
constexpr int WB_WORDS = 12;    // words of one cluster's decision record (wide walker)
constexpr int MAX_W = 16;
constexpr int MAX_AW = 1024;    // projected states per step (A*W)
constexpr int AMB_MAX = 64;     // ambiguous (state, tau) minima handled per step
constexpr int TC_MAX = 128;     // terrain-well candidates per list
constexpr int TC_WIN = 8;       // steps one terrain-candidate scan serves (fmdp_walk.cu)
constexpr int TW_SMEM = 512;    // terrain wells cached in shared memory (more: read from L2)
constexpr int N_PHASES = 17;     // walk-kernel phase accounting (fmdp_stats.phase_cycles)
constexpr int PAIR_STRIDE = 40;  // floats per plan-pair record: per tau (X, X', Y, Y', Z, Z', Q, Q')

// Scenario + store in integer units, passed by value to the kernels.
struct World {
  int32_t A, W, n_turn, n_climb, HL;
  int32_t turn[MAX_TURN];
  int32_t climb[MAX_CLIMB];
  int32_t zero_climb;           // index of the level-flight climb (0 units), -1 if none
  int32_t k_tau[NTAU];          // tau / dt substeps (padding taus: k = 0, R2 = 0)
  int64_t R2_tau[NTAU];         // exact R_tau^2, units^2
  float cull2f_tau[NTAU];       // (R_tau + reach + 1)^2 (1 + 2^-16): conservative FP32 f1 cull threshold
  int32_t cull_inf;             // R_max + reach + 1: f1 L-inf prefilter radius
  int32_t k_absmax;             // max |tau/dt|
  float R2lo[NTAU], R2hi[NTAU]; // FP32 filter band R^2 (1 -/+ band_tau), band >= 2^-20 (host: error bound)
  int32_t R_max;                // max tau radius, units (< 2^15)
  uint32_t sat_d2;              // R_max^2: saturation of separation minima
  uint32_t sep2;                // separation minimum^2
  int64_t cap2;                 // goal capture radius^2
  int32_t reach_u;              // bound on |s_{a,t} - q| over all projected states
  int32_t step_reach_u;         // bound on |Delta_1(a) - q| (one substep)
  double goal_r, goal_l2g;      // goal peak: |r|, log2(gamma) * u
  float goal_rf, goal_l2gf;     // the same in FP32 (kernel: ex2.approx of exact-offset distances)
  float intr_r, intr_l2g;       // intruder wells: |r|, log2(gamma) * u (FP32 ex2)
  float terr_r, terr_l2g;       // terrain wells
  int32_t zdeck_u;
  double deck_scale, u_m;
  int32_t max_steps, vmax_init_zero;
  int32_t endpoint;             // 1: Alg 1 valuation, V*(a) = V at the last substep
  double near_tie_rel;
  // accepted-plan store: rows[K] = { x[cap], y[cap], z[cap], vpack[cap] } (int32 SoA)
  int64_t horizon;
  int32_t row_cap;
  const int32_t* rows;
  const int32_t* counts;        // active slots per row
  // terrain
  int32_t n_tw;
  const int4* tw;               // x, y, z, R (units)
  int32_t nx, ny, x0, y0, cell;
  uint64_t cell_magic;          // ceil(2^40 / cell): exact floor division for offsets < 2^25
  const int32_t* height;        // [ny][nx] units
  const int2* dxy;              // heading lattice table [HL]
  const int2* proj;             // cumulative displacement [HL][n_turn][W]: sum_{s<=t} (DX,DY)[psi + s*turn]
  // acceleration actions -> the wide walker (MODE 5).  The action
  // space (turn, acceleration, climb) is tiled over the launch's clusters by horizontal path hp =
  // i_turn * n_acc + i_acc: cluster c owns paths [c*hpt, c*hpt + hpt) and, like any walker, splits
  // every time row over its CTAs; per step the clusters exchange their tile's top-2 (decision
  // board).  In a wide World A = hpt * C and n_turn = hpt (one tile); A_all is the whole space.
  int32_t wide;                 // 1: acceleration actions (MODE 5 launches only)
  int32_t A_all, n_hp, hpt, n_turn_all, n_acc;
  int32_t acc[MAX_ACC];         // speed increments, units per substep per substep
  int32_t vmin, vmax, v0;       // speed bounds / departure speed, units per substep
  const int2* spd;              // [vmax - vmin + 1][HL] displacement of one substep at (speed, heading)
  // SURVEY f1 range query (culled FCFS walker): the plans loaded by fmdp_add_plans sit in each row
  // sorted by x-y cell of side cell_l, slots [cstart[K][c], cstart[K][c+1]) in cell c (row-major,
  // cell_ncx per row of cells), [cstart[K][cell_n], counts[K]) = plans appended since (unsorted).
  // Every plan whose wells can reach a state of the next few steps lies in the 3x3 cells around
  // the ownship (cell_l >= R_max + reach + the prefetch margin + max well offset).  cell_n = 0: off.
  int32_t cell_n, cell_ncx, cell_ncy, cell_l;
  int32_t cell_x0, cell_y0;
  const int32_t* cstart;        // [horizon][cell_n + 1]
};

struct Req {
  int32_t src[3];
  int32_t dst[3];
  int32_t psi0;
  int32_t start_k;              // resume step (0 = fresh request)
  int64_t t0;
  int32_t slot;                 // output slot
  int32_t head;                 // 1: the earliest pending FCFS request (never paused; sets *stop when done)
  int32_t speed0;               // departure speed, units per substep (0: the airspace's speed)
  // re-convergence after a rollback (a10): the request's previous run, kept in the
  // backup arrays (BakRec) over [rollback step, n_old), ended with old_status at state n_old - 1;
  // no plan committed since can influence its states >= reuse_from.  A re-walk whose state k >=
  // reuse_from equals the old state k takes the old run from k on.  n_old = 0: off.
  int32_t reuse_from, n_old, old_status, old_fail;
  int32_t pad;
};

// One step of a request's previous run (re-convergence backup, Req::n_old): state, decision and
// per-step records, 32 B (the first 16 B = the state, fetched with one 16-byte cp.async).
struct BakRec {
  int32_t x, y, z, heading;
  int32_t astar, stepx;
  uint32_t stepd2;
  int32_t ntie;
};

struct Out {
  int32_t status, n_states, fail_step, n_near_ties;  // status -1: paused (resume at n_states-1)
  int32_t n_exact, steps_run;
  uint32_t min_sep_d2;
  int32_t reconv;               // 1: the walk re-converged onto the request's previous run (Req::n_old)
};

struct XPeer;

struct WalkArgs {
  const Req* reqs;
  int32_t n_reqs;
  int32_t* queue;               // dynamic request counter (zeroed before launch)
  Out* out;                     // [slot]
  int32_t* traj;                // [slot][cap][3]
  int32_t* heading;             // [slot][cap]
  int32_t* astar;               // [slot][cap]
  uint32_t* stepd2;             // [slot][cap] saturated nearest-plan d^2 of state k
  int8_t* ntie;                 // [slot][cap]
  int32_t cap;
  int32_t eval;                 // 1: evaluate one step (debug outputs), no advance
  int32_t budget;               // decision steps per request in this launch (then pause, status -1)
  int32_t* stop;                // single-wave slices: set by the head request when it finishes; the
                                // others pause after `budget` steps only once it is set (nullptr: off)
  int32_t cull;                 // 1: f1 exact culling of plans whose wells cannot reach the states
  int32_t shard_rank, shard_world;  // plan shard of this GPU; 0, 1 = whole rows
  int32_t xmode;                // 0 normal; 1 export per-(state,tau) minima + stay; 2 import and decide
  uint32_t* xbuf;               // [A*W*NTAU + 1] exchange buffer (float bits / stay d^2)
  int32_t* speed;               // [slot][cap] speed of state k (wide walker)
  unsigned long long* wb;       // wide walker decision board [2][clusters][WB_WORDS] LL words
  unsigned long long wseq0;     // board tag base of this launch (host-tracked, monotonic)
  int32_t* werr;                // board poll timeout flag
  double* dbg_vstar;            // [A]
  double* dbg_v;                // [A*W]
  double* dbg_s;                // [A*W]
  uint32_t* dbg_conf;           // [A+1]
  int32_t* dbg_astar;           // [1]
  unsigned long long* pairs;    // hot-loop pair counter (stats)
  int32_t* stepx;               // [slot][cap] exact-fallback count of step k (zeroed by the host)
  const BakRec* bak;            // [slot][cap] previous runs (re-convergence; Req::n_old), or null
  double2* vtrace;              // [vtrace_n][cap][A] {V*(a), S(a)} per step (fmdp_set_trace), or null
  int32_t vtrace_n;
  unsigned long long* prof;     // [PH_N] per-phase cycles of rank 0 (nullptr = off)
  // co-simulated batch: one cluster per request, all on one clock
  int32_t cosim;                // 1: batch peers are wells (Alg 5) and separation partners
  int32_t cs_n;                 // batch size = clusters launched (all co-resident)
  int64_t cs_k0;                // first clock (min t0)
  int4* cs_pub;                 // [2][cs_n][2]: {x, y, z, flags}, {vx, vy, vz, 0} by clock parity
  unsigned* cs_arrive;          // arrivals, one per walker per clock (zeroed before launch)
  int32_t* cs_err;              // set on a barrier timeout (walkers not co-resident)
  // in-kernel plan-sharded exchange (xmode 3, SURVEY §8(e) production form): one persistent
  // launch per request on every rank; per step each CTA stores its owned per-(state, tau) minima
  // and the nearest-plan d^2 as {value, step tag} words into every peer's receive slot (P2P
  // stores over NVLink) and polls its own slots for the peers' words; see XPeer
  int32_t x_me, x_world, x_slot;      // this rank, ranks, words per (parity, source) slot
  const XPeer* x_peers;             // [x_world] device table (entry x_me = this GPU's own area)
  unsigned long long* x_seq;          // this rank's exchange sequence number (step tags)
  int32_t* x_err;                     // set on a poll timeout (a peer is not running)
  int32_t x_intra;                    // 1: the launch's clusters are the ranks (x_me = cluster
                                      // index, x_world = clusters; x_seq / queue per cluster;
                                      // plan shard = shard_rank + cluster index of shard_world)
  int32_t x_inter;                    // 1: two-level exchange -- after the clusters of this GPU,
  int32_t x_iworld, x_ime;            //    cluster c of each of the x_iworld GPUs (this: x_ime)
  const XPeer* x_ipeers;              //    [XMAX clusters][XNODE GPUs] receive areas
};

// One rank's exchange area as seen from this GPU (peer pointer: IPC-opened or same process):
//   recv[(par * world + src) * slot + i] = {value, step tag} (one 8-byte word, written by rank
//   src with a single 64-bit store): i < A*W*NTAU: FP32 bits of src's minimum for (state, tau)
//   item i; i = slot - 16 + cta: src's nearest-plan d^2 (CTA cta).
struct XPeer {
  unsigned long long* recv;
};
constexpr int XMAX = 16;              // ranks of one exchange (clusters of one GPU)
constexpr int XNODE = 8;              // ranks of a multi-GPU exchange (GPUs of one node)
inline size_t x_area_bytes(int world, int slot) {
  return (size_t)2 * world * slot * sizeof(unsigned long long);
}

// Shared-memory carve-up, identical on host (size) and device (offsets).
struct Layout {
  int HL, CH, RAWCAP, NT, C, NCOL, A, AW, G, WT, BLK, NOWN, RAWW;
  size_t o_dxy, o_tw, o_raw, o_cen, o_stage, o_recv, o_pos, o_fix, o_sfix, o_vT, o_mI, o_vstar, o_vsc, o_conf,
      o_confg, o_flags, o_stay, o_amb, o_tc, o_bar, o_ctl, o_M, total;
  __host__ __device__ static size_t al(size_t x) { return (x + 15) & ~size_t(15); }
  __host__ __device__ void build(int hl, int ch, int rawcap, int nt, int c, int ncol, int a, int aw, int g) {
    HL = hl; CH = ch; RAWCAP = rawcap; NT = nt; C = c; NCOL = ncol; A = a; AW = aw; G = g;
    WT = (AW / A) * NTAU;               // (state, tau) items of one action
    BLK = (WT + 3) & ~3;                // per-action block of the reduce-scatter, padded to 16 B
    NOWN = (A + G - 1) / G;             // max actions owned by one CTA
    RAWW = RAWCAP + 8;                  // words per SoA array in one raw row buffer
    size_t o = 0;
    o_dxy = o;  o = al(o + sizeof(int2) * HL);
    o_tw = o;   o = al(o + sizeof(int4) * TW_SMEM);
    o_raw = o;  o = al(o + sizeof(int32_t) * 4 * RAWW * 3);
    size_t cen = sizeof(float) * PAIR_STRIDE * ((CH + 1) / 2);  // plan-pair well records
    o_cen = o;  o = al(o + cen);
    // reduce-scatter: the CTA's per-action minima staged by owner CTA ([owner][slot][BLK], one
    // contiguous run per owner = one bulk DSMEM copy), received per source CTA and step parity
    o_stage = o; o = al(o + sizeof(float) * (size_t)G * NOWN * BLK);
    o_recv = o; o = al(o + sizeof(float) * 2 * (size_t)G * NOWN * BLK);
    o_pos = o;  o = al(o + sizeof(int4) * 2 * AW);   // double-buffered by step parity
    o_fix = o;  o = al(o + sizeof(double) * AW);
    o_sfix = o; o = al(o + sizeof(double) * AW);
    o_vT = o;   o = al(o + sizeof(float) * AW);
    o_mI = o;   o = al(o + sizeof(float) * AW);
    o_vstar = o; o = al(o + sizeof(double) * 2 * A);  // {V*(a), S(a)} pairs (one 16 B DSMEM push)
    o_vsc = o;
    o_conf = o; o = al(o + sizeof(uint32_t) * (A + 1));
    o_confg = o; o = al(o + sizeof(uint32_t) * (A + 1));
    o_flags = o; o = al(o + sizeof(int32_t) * A);
    o_stay = o; o = al(o + sizeof(uint32_t) * 2 * 16);  // [parity][source rank] slice minima
    o_amb = o;  o = al(o + sizeof(int32_t) * AMB_MAX);
    o_tc = o;   o = al(o + sizeof(int32_t) * 2 * TC_MAX);  // candidate lists, by step parity
    o_bar = o;  o = al(o + sizeof(uint64_t) * 8);   // 3 TMA ring + 2 reduce-scatter + 2 V* mbarriers
    o_ctl = o;  o = al(o + 768);
    o_M = o;    o = al(o + sizeof(float) * (size_t)NOWN * WT);  // owner pass: in-radius minima of the owned items
    total = o;
  }
};

struct AppendPlan {
  int64_t t0;
  int32_t n;
  int32_t pad;
  const int32_t* states;        // device [n][3]
  const int32_t* slots;         // device [n] row slot of state i
};

struct InflPair {
  int32_t i, j;                 // request slot i, plan from slot j
  int32_t lo, hi;               // steps of i to test: [lo, hi) (hi < 0: [0, n_states[i]))
  int32_t bak;                  // 1: i's states from the backup of its previous run (BakRec)
};

struct InflWells {              // exact-conservative influence criterion (a10)
  int32_t n_tau;
  int32_t k_tau[NTAU];
  int64_t r2[NTAU];             // (R_tau + reach + 1)^2
  int64_t sat2;                 // R_max^2: separation saturation
};

// Range-query index build (fmdp_walk.cu): rows [K0, K0 + nrows) sorted by cell (see World),
// cstart written; tmp = nrows * 4 * row_cap int32 scratch.
cudaError_t launch_index(int32_t* rows, int32_t row_cap, const int32_t* counts, int64_t K0, int nrows, const World& w,
                         int32_t* cstart, int32_t* tmp, cudaStream_t s);
// Maximum |horizontal velocity|^2 (units^2 per substep^2) over every stored plan-step (index cell size).
cudaError_t launch_vmax(const int32_t* rows, int32_t row_cap, const int32_t* counts, int64_t horizon,
                        unsigned long long* out, cudaStream_t s);

// Kernel launchers (fmdp_walk.cu).
cudaError_t launch_walk(const World& w, const WalkArgs& a, int n_climb, int cluster, int n_clusters,
                        int threads, int chunk, int rawcap, cudaStream_t s);
// Hot-loop thread mapping: warps of 32/ngw columns x ngw plan groups; threads = 32*warps.
int walk_groups_per_warp(int ncol, int max_threads);
int walk_threads(int ncol, int max_threads);
cudaError_t walk_max_clusters(const World& w, int n_climb, int cluster, int threads, int chunk, int rawcap, int* out,
                              bool cosim = false);
size_t walk_smem_bytes(const World& w, int n_climb, int threads, int chunk, int rawcap, int cluster);
cudaError_t launch_append(int32_t* rows, int32_t row_cap, int64_t horizon, const AppendPlan* plans, int n_plans,
                          int max_n, cudaStream_t s);
cudaError_t launch_influence(const int32_t* traj, const BakRec* bak, int32_t cap, const int32_t* n_states,
                             const int64_t* t0, const InflPair* pairs, int n_pairs, const InflWells& iw, int32_t* kfirst,
                             cudaStream_t s);
// Trajectories of slots [0, n) packed back to back (slot i's states at off[i], n_states from out[i])
// for one D2H copy of the whole batch's result.
cudaError_t launch_pack_traj(const int32_t* traj, int32_t cap, const Out* out, const int64_t* off, int n, int32_t* pack,
                             cudaStream_t s);
// Backup of request slot i's steps [lo, hi) (state, decision and per-step records) into bak.
cudaError_t launch_backup(BakRec* bak, const int32_t* traj, const int32_t* heading, const int32_t* astar,
                          const int32_t* stepx, const uint32_t* stepd2, const int8_t* ntie, int32_t cap, int slot, int lo,
                          int hi, cudaStream_t s);

}  // namespace fmdp

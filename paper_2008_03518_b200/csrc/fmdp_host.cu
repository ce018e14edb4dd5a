// fmdp_host.cu -- C ABI (include/fmdp.h) of the B200 FastMDP-GPU hot path: context,
// scenario validation and quantisation, the device plan store ([time row][slot] SoA),
// and the first-come-first-served driver (sequential and speculative rounds).
// Every step of the path runs in the kernels of fmdp_walk.cu; this file only validates,
// allocates, launches and copies.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fmdp.h"
#include "fmdp_dev.h"

using fmdp::AppendPlan;
using fmdp::InflPair;
using fmdp::Out;
using fmdp::Req;
using fmdp::World;

namespace {
struct PlanRec {
  uint64_t aircraft;
  int64_t t0;
  std::vector<int32_t> states;  // n*3
};
}  // namespace

struct fmdp_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  void* (*alloc)(size_t, void*) = nullptr;
  void (*release)(void*, void*) = nullptr;
  void* user = nullptr;
  std::vector<void*> allocs;

  fmdp_airspace air{};
  std::vector<int32_t> turn, climb, acc;
  bool wide = false;                 // acceleration actions: the wide walker
  int wide_k = 0;                    // clusters (action tiles) of one wide launch
  int2* d_spd = nullptr;             // (speed, heading) displacement table
  int32_t* d_speed = nullptr;        // [slot][cap] speed of state k
  unsigned long long* d_wb = nullptr;  // decision board [2][k][WB_WORDS]
  int32_t* d_wq = nullptr;           // [k] request queues of the clusters, then the board error flag
  std::vector<double> tau_s, tau_r;
  World w{};
  int A = 0, W = 0, C = 0;
  int64_t lo_u[3]{}, hi_u[3]{};
  fmdp::InflWells iw{};

  std::vector<int32_t> counts;  // host mirror of the per-row slot counts (authoritative)
  std::vector<PlanRec> plans;
  int32_t* d_rows = nullptr;
  int32_t* d_counts = nullptr;
  int4* d_tw = nullptr;
  int32_t* d_height = nullptr;
  int2* d_dxy = nullptr;
  int2* d_proj = nullptr;  // cumulative projection offsets [HL][n_turn][W]

  // per-request scratch (grown on demand)
  int slots_cap = 0;
  int32_t cap_states = 0;
  Req* d_reqs = nullptr;
  Out* d_out = nullptr;
  int32_t *d_traj = nullptr, *d_heading = nullptr, *d_astar = nullptr;
  uint32_t* d_stepd2 = nullptr;
  int8_t* d_ntie = nullptr;
  int32_t* d_stepx = nullptr;  // [slot][cap] exact-fallback count per step (zeroed per call / rollback)
  fmdp::BakRec* d_bak = nullptr;  // [slot][cap] a rolled-back request's previous run (re-convergence)
  // SURVEY f1 range query (culled walker): rows sorted by x-y cell, cstart offsets (fmdp::World)
  int32_t* d_cstart = nullptr;
  size_t cstart_cap = 0;
  int32_t* d_itmp = nullptr;          // sort scratch
  size_t itmp_cap = 0;
  bool index_dirty = true;            // plans added since the last build (they are scanned, unsorted)
  size_t n_indexed = 0;               // plans in the sorted regions (truncating below them reloads)
  bool idx_cost = true;               // cost models may assume the range query (not for p2p walks)
  double2* d_vtrace = nullptr; // fmdp_set_trace: [vtrace_n][cap][A] {V*(a), S(a)} per step
  int vtrace_n = 0;
  int32_t* d_queue = nullptr;
  int32_t* d_stop = nullptr;   // head-finished flag of a single-wave slice
  int32_t* d_nstates = nullptr;
  int64_t* d_t0s = nullptr;
  unsigned long long* d_pairctr = nullptr;
  unsigned long long* d_prof = nullptr;
  InflPair* d_pairs = nullptr;
  int32_t* d_kfirst = nullptr;
  int pairs_cap = 0;
  AppendPlan* d_app = nullptr;
  int app_cap = 0;
  int32_t* d_up = nullptr;  // upload scratch (states / slots)
  size_t up_cap = 0;
  int32_t* d_pack = nullptr;    // batch result trajectories packed back to back (device) ...
  int32_t* h_pack = nullptr;    // ... and their pinned host copy (one D2H per batch)
  int64_t* d_packoff = nullptr;
  size_t pack_cap = 0, packoff_cap = 0;
  int4* d_cspub = nullptr;     // co-simulation publish buffer [2][n][2]
  int32_t* d_csctr = nullptr;  // [0] arrivals, [1] barrier error
  int cs_cap = 0;
  uint32_t* d_xbuf = nullptr;  // multi-GPU exchange buffer [A*W*NTAU + 1]
  int xmode = 0, shard_rank = 0, shard_world = 1;
  // in-kernel multi-GPU exchange (fmdp_p2p_*): own area, peer table, step-tag sequence
  void* x_area = nullptr;
  int x_world = 0, x_me = -1, x_slot = 0;
  std::vector<void*> x_ipc;                // IPC-opened peer areas
  fmdp::XPeer* d_xpeers = nullptr;         // [XMAX]
  // one request split over clusters of this GPU (fmdp_launch.split): the same exchange, the
  // launch's clusters as ranks; areas / tags / queues kept across launches (tags monotonic)
  unsigned long long* d_xin_area = nullptr;  // XMAX areas of XMAX ranks
  fmdp::XPeer* d_xin_peers = nullptr;        // [XMAX]
  unsigned long long* d_xin_seq = nullptr;   // [XMAX] per-cluster sequence, then int32 error, queues
  int xin_world = 0;                         // cluster count of the last split launch (layout)
  // multi-GPU two-level exchange: inter-GPU areas of every cluster index, this GPU's intra
  // level (areas, peers, monotonic per-cluster tag sequence + error flag + queues)
  fmdp::XPeer* d_ipeers = nullptr;           // [XMAX][XNODE]
  unsigned long long* d_xh_area = nullptr;
  fmdp::XPeer* d_xh_peers = nullptr;         // [XMAX]
  unsigned long long* d_xh_seq = nullptr;    // [XMAX] sequence, then int32 error, then int32 queues
  unsigned long long xh_seq = 0;             // common tag sequence of every cluster (host copy)
  unsigned long long* d_xseq = nullptr;    // [1] sequence, then [1] int32 error flag
  double *d_dbg_vstar = nullptr, *d_dbg_v = nullptr, *d_dbg_s = nullptr;
  uint32_t* d_dbg_conf = nullptr;
  int32_t* d_dbg_astar = nullptr;

  std::vector<Out> h_out;
  int last_n = 0;
  fmdp_launch launch{};
  fmdp_stats stats{};
  std::string err;
  int num_sms = 0;
  int mc_cache[17] = {0};
  int mc_cache_cs[17] = {0};
  double fan_radius_u = 0;             // bound on |s - o| (hot-loop origin), units
  double band_rel[fmdp::NTAU] = {0};   // FP32 filter band per tau, relative to R^2
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
  cudaStream_t stream2 = nullptr;  // second stream of a split FCFS slice (the non-head walkers)
  cudaStream_t stream3 = nullptr;  // third stream: the next request's walker (second lane)
  cudaEvent_t ev3 = nullptr;
};

namespace {

thread_local std::string g_create_error = "";  // reason of this thread's last failed fmdp_create

const char* kStatusText[] = {"ok", "invalid argument", "out of memory", "CUDA error", "row capacity exceeded",
                             "duplicate", "buffer too small", "out of range", "no sm_100 device", "plan-store file I/O error"};

fmdp_status fail(fmdp_ctx* c, fmdp_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

#define CK(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) return fail(ctx, FMDP_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Makes the context's device current for one API call and restores the caller's on return.
struct DevGuard {
  int prev = -1;
  bool swapped = false;
  explicit DevGuard(int dev) {
    if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) swapped = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DevGuard() {
    if (swapped) cudaSetDevice(prev);
  }
};

void* dalloc(fmdp_ctx* ctx, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* p = nullptr;
  if (ctx->alloc) {
    p = ctx->alloc(bytes, ctx->user);
  } else if (cudaMalloc(&p, bytes) != cudaSuccess) {
    p = nullptr;
  }
  if (p) ctx->allocs.push_back(p);
  return p;
}

// Close the IPC-opened peer areas and free this rank's exchange area (fmdp_p2p_*).
void x_release(fmdp_ctx* ctx) {
  for (void* p : ctx->x_ipc) cudaIpcCloseMemHandle(p);
  ctx->x_ipc.clear();
  if (ctx->x_area) cudaFree(ctx->x_area);
  ctx->x_area = nullptr;
  ctx->x_world = 0;
  ctx->x_me = -1;
}

void dfree(fmdp_ctx* ctx, void* p) {
  if (!p) return;
  auto it = std::find(ctx->allocs.begin(), ctx->allocs.end(), p);
  if (it != ctx->allocs.end()) ctx->allocs.erase(it);
  if (ctx->release) ctx->release(p, ctx->user);
  else cudaFree(p);
}

template <class T>
fmdp_status grow(fmdp_ctx* ctx, T*& p, size_t n) {
  dfree(ctx, p);
  p = static_cast<T*>(dalloc(ctx, sizeof(T) * n));
  return p ? FMDP_OK : fail(ctx, FMDP_E_NOMEM, "device allocation failed");
}

bool integral(double r, int64_t* out) {
  double n = std::rint(r);
  if (!(std::fabs(r - n) <= 1e-9 * (1.0 + std::fabs(r)))) return false;
  *out = (int64_t)n;
  return true;
}

// Heading lattice (R14): first-octant rounding of L*(cos, sin), reflected and rotated so the
// table is exactly symmetric.  Independent implementation of the DESIGN.md definition.
void build_lattice(int HL, int64_t L, std::vector<int2>& t) {
  t.resize(HL);
  const int Q = HL / 4, O = HL / 8;
  for (int psi = 0; psi < HL; ++psi) {
    const int quad = psi / Q, r = psi % Q;
    double cx, sy;
    if (r <= O) {
      cx = std::rint((double)L * std::cos(2.0 * M_PI * r / HL));
      sy = std::rint((double)L * std::sin(2.0 * M_PI * r / HL));
    } else {
      const int m = Q - r;
      cx = std::rint((double)L * std::sin(2.0 * M_PI * m / HL));
      sy = std::rint((double)L * std::cos(2.0 * M_PI * m / HL));
    }
    const int a = (int)cx, b = (int)sy;
    switch (quad) {
      case 0: t[psi] = make_int2(a, b); break;
      case 1: t[psi] = make_int2(-b, a); break;
      case 2: t[psi] = make_int2(-a, -b); break;
      default: t[psi] = make_int2(b, -a); break;
    }
  }
}

fmdp_status quantize(fmdp_ctx* ctx, const fmdp_vec3& v, int32_t q[3]) {
  const double m[3] = {v.x, v.y, v.z};
  for (int d = 0; d < 3; ++d) {
    const double x = m[d] / ctx->air.u_m;
    if (!std::isfinite(x)) return fail(ctx, FMDP_E_ARG, "non-finite coordinate");
    const long long r = std::llrint(x);
    if (r < ctx->lo_u[d] || r > ctx->hi_u[d]) return fail(ctx, FMDP_E_RANGE, "position outside the airspace");
    q[d] = (int32_t)r;
  }
  return FMDP_OK;
}

int32_t initial_heading(const fmdp_ctx* ctx, const int32_t s[3], const int32_t g[3]) {
  const double a = std::atan2((double)g[1] - (double)s[1], (double)g[0] - (double)s[0]) * ctx->w.HL / (2.0 * M_PI);
  long long h = std::llrint(a) % ctx->w.HL;
  if (h < 0) h += ctx->w.HL;
  return (int32_t)h;
}

// Per-request scratch for n requests (grown on demand), and the per-step exact counts of the
// call zeroed.  Growth is all-or-nothing: every new buffer is allocated before any old one is
// released, so a failed allocation leaves the previous (smaller) set intact and consistent.
fmdp_status ensure_slots(fmdp_ctx* ctx, int n) {
  const size_t cap = (size_t)ctx->cap_states;
  if (n > ctx->slots_cap) {
    const size_t m = (size_t)std::max(n, 2 * ctx->slots_cap);
    struct B {
      void** dst;
      size_t bytes;
      void* p;
    } b[] = {{(void**)&ctx->d_reqs, sizeof(Req) * m, nullptr},        {(void**)&ctx->d_out, sizeof(Out) * m, nullptr},
             {(void**)&ctx->d_traj, 12 * cap * m, nullptr},           {(void**)&ctx->d_heading, 4 * cap * m, nullptr},
             {(void**)&ctx->d_astar, 4 * cap * m, nullptr},           {(void**)&ctx->d_stepd2, 4 * cap * m, nullptr},
             {(void**)&ctx->d_ntie, cap * m, nullptr},                {(void**)&ctx->d_stepx, 4 * cap * m, nullptr},
             {(void**)&ctx->d_speed, 4 * cap * m, nullptr},          {(void**)&ctx->d_bak, sizeof(fmdp::BakRec) * cap * m, nullptr},
             {(void**)&ctx->d_nstates, sizeof(int32_t) * m, nullptr}, {(void**)&ctx->d_t0s, sizeof(int64_t) * m, nullptr}};
    for (B& e : b) {
      e.p = dalloc(ctx, e.bytes);
      if (!e.p) {
        for (B& f : b) dfree(ctx, f.p);
        return fail(ctx, FMDP_E_NOMEM, "device allocation failed (request scratch)");
      }
    }
    for (B& e : b) {
      dfree(ctx, *e.dst);
      *e.dst = e.p;
    }
    ctx->slots_cap = (int)m;
    ctx->h_out.resize(m);
  }
  if (n > 0) CK(cudaMemsetAsync(ctx->d_stepx, 0, sizeof(int32_t) * cap * (size_t)n, ctx->stream));
  return FMDP_OK;
}

// Rollback of request slot i to step k1: its per-step exact counts from k1 on are recomputed.
fmdp_status clear_stepx(fmdp_ctx* ctx, int i, int k1) {
  const size_t cap = (size_t)ctx->cap_states;
  if (k1 < 0 || (size_t)k1 >= cap) return FMDP_OK;
  CK(cudaMemsetAsync(ctx->d_stepx + (size_t)i * cap + k1, 0, sizeof(int32_t) * (cap - k1), ctx->stream));
  return FMDP_OK;
}

fmdp_status ensure_up(fmdp_ctx* ctx, size_t words) {
  if (words <= ctx->up_cap) return FMDP_OK;
  const size_t m = std::max(words, 2 * ctx->up_cap);
  fmdp_status s = grow(ctx, ctx->d_up, m);
  if (s) return s;
  ctx->up_cap = m;
  return FMDP_OK;
}

int threads_for(const fmdp_ctx* ctx) {
  int tmax = ctx->C == 1 ? 512 : 384;  // kernel __launch_bounds__
  if (ctx->launch.threads >= 32) tmax = std::min(tmax, ctx->launch.threads);  // fmdp_launch.threads: a cap
  return fmdp::walk_threads(ctx->w.n_turn * ctx->w.W, tmax);
}

constexpr int kChunk = 512;      // well records / plans per build pass (brute force)
constexpr int kCullChunk = 256;  // well records with f1 culling (survivors only)
// raw plans staged per row buffer: with culling as much of the slice as shared memory allows
int rawcap_for(const fmdp_ctx* ctx);
// The full path's plans per build pass (= raw plans staged per row buffer): the largest of
// 1024 / 768 / 512 that fits shared memory -- fewer passes (two CTA barriers and a build each)
// per step at large stores (configs[3] split request: 30.0 -> 28.7 us/step at 1024; configs[4],
// A = 85: 768 and 1024 exceed 220 KB, stays 512; tools/chunk_probe.py); one pass either way at
// configs[1].  (FMDP_TUNE_CHUNK: an override for tools/chunk_probe.py only)
int full_chunk(const fmdp_ctx* ctx) {
  static const int env = std::getenv("FMDP_TUNE_CHUNK") ? std::atoi(std::getenv("FMDP_TUNE_CHUNK")) : 0;
  if (env > 0) return env;
  for (int c : {1024, 768})
    if (fmdp::walk_smem_bytes(ctx->w, ctx->C, threads_for(ctx), c, c, 16) <= 220 * 1024) return c;
  return kChunk;
}
int chunk_for(const fmdp_ctx* ctx) { return ctx->launch.cull ? kCullChunk : full_chunk(ctx); }

int rawcap_for(const fmdp_ctx* ctx) {
  if (!ctx->launch.cull) return full_chunk(ctx);
  int cap = 3072;
  while (cap > kCullChunk &&
         fmdp::walk_smem_bytes(ctx->w, ctx->C, threads_for(ctx), kCullChunk, cap, 16) > 220 * 1024)
    cap -= 256;
  return cap;
}

int max_clusters(fmdp_ctx* ctx, int G, bool cosim = false) {
  int* cache = cosim ? ctx->mc_cache_cs : ctx->mc_cache;
  if (cache[G]) return cache[G];
  int n = 0;
  if (fmdp::walk_max_clusters(ctx->w, ctx->C, G, threads_for(ctx), chunk_for(ctx), rawcap_for(ctx), &n, cosim) !=
          cudaSuccess || n < 0)
    n = 0;
  cudaGetLastError();
  cache[G] = n;
  return n;
}

// Per-step cycles of one walker with cluster size G over rows of P plans, measured on B200
// (tools/calib.py: configs[1] 3000 plans and configs[3] 100k plans, G = 1..16, full and f1):
//   t(G) = 12200 (projection, epilogue, barriers, decision) + P*b/G + 130*G,
//   b = 2.8 cycles/plan with culling (build pass), 5*A*W/26.5 without (hot loop, ~26.5 pairs/clk/SM).
double step_cycles(const fmdp_ctx* ctx, double plans, int G) {
  const double b = ctx->launch.cull ? 2.8 : fmdp::NTAU * ctx->A * ctx->W / 26.5;
  return 12200.0 + plans * b / G + 130.0 * G;
}

double mean_plans(const fmdp_ctx* ctx) {
  int64_t tot = 0, nz = 0;
  for (int32_t c : ctx->counts)
    if (c) { tot += c; ++nz; }
  double m = nz ? (double)tot / nz / ctx->shard_world : 0.0;  // plans per row this GPU evaluates
  if (ctx->launch.cull && ctx->w.cell_n > 0 && ctx->idx_cost) m *= std::min(1.0, 9.0 / ctx->w.cell_n);  // range query
  return m;
}

// Cluster size for a round of n_run trajectories: the G minimising waves(G) * t(G) among the
// sizes that can run.
void choose_launch(fmdp_ctx* ctx, int n_run, int* G_out, int* nc_out, int sm_cap = 0) {
  int best_G = 1;
  double best = 1e300;
  const double plans = mean_plans(ctx);
  const int sizes[] = {16, 8, 4, 2, 1};
  for (int G : sizes) {
    if (ctx->launch.cluster_size && G != ctx->launch.cluster_size) continue;
    int mc = max_clusters(ctx, G);
    if (sm_cap > 0) mc = std::min(mc, sm_cap / G);  // SMs left to this launch
    if (mc <= 0) continue;
    int conc = std::min(mc, n_run);
    if (ctx->launch.max_walkers > 0) conc = std::min(conc, ctx->launch.max_walkers);
    const double waves = std::ceil((double)n_run / conc);
    const double t = waves * step_cycles(ctx, plans, G);
    if (t < best - 1e-9) {
      best = t;
      best_G = G;
    }
  }
  int mc = std::max(1, max_clusters(ctx, best_G));
  if (sm_cap > 0) mc = std::max(1, std::min(mc, sm_cap / best_G));
  int conc = std::min(mc, n_run);
  if (ctx->launch.max_walkers > 0) conc = std::min(conc, ctx->launch.max_walkers);
  *G_out = best_G;
  *nc_out = std::max(1, conc);
  if (std::getenv("FMDP_DEBUG"))
    std::fprintf(stderr, "fmdp: n_run=%d plans/row=%.0f -> G=%d clusters=%d (max active %d)\n", n_run, plans, best_G,
                 *nc_out, mc);
}

// The cluster size a lone walker would get (fastest per step).
int solo_cluster_size(fmdp_ctx* ctx) {
  int best_G = 1;
  double best = 1e300;
  const double plans = mean_plans(ctx);
  for (int G : {16, 8, 4, 2, 1}) {
    if (ctx->launch.cluster_size && G != ctx->launch.cluster_size) continue;
    if (max_clusters(ctx, G) <= 0) continue;
    const double t = step_cycles(ctx, plans, G);
    if (t < best - 1e-9) {
      best = t;
      best_G = G;
    }
  }
  return best_G;
}

fmdp::WalkArgs make_args(fmdp_ctx* ctx, const std::vector<Req>& run, bool eval, int budget) {
  fmdp::WalkArgs a{};
  a.reqs = ctx->d_reqs;
  a.n_reqs = (int32_t)run.size();
  a.queue = ctx->d_queue;
  a.out = ctx->d_out;
  a.traj = ctx->d_traj;
  a.heading = ctx->d_heading;
  a.astar = ctx->d_astar;
  a.stepd2 = ctx->d_stepd2;
  a.ntie = ctx->d_ntie;
  a.cap = ctx->cap_states;
  a.eval = eval ? 1 : 0;
  a.budget = budget;
  a.cull = ctx->launch.cull ? 1 : 0;
  a.xmode = ctx->xmode;
  a.shard_rank = ctx->shard_rank;
  a.shard_world = ctx->shard_world;
  a.xbuf = ctx->d_xbuf;
  a.x_me = ctx->x_me;
  a.x_world = ctx->x_world;
  a.x_slot = ctx->x_slot;
  a.x_peers = ctx->d_xpeers;
  a.x_seq = ctx->d_xseq;
  a.x_err = ctx->d_xseq ? reinterpret_cast<int32_t*>(ctx->d_xseq + 1) : nullptr;
  a.dbg_vstar = ctx->d_dbg_vstar;
  a.dbg_v = ctx->d_dbg_v;
  a.dbg_s = ctx->d_dbg_s;
  a.dbg_conf = ctx->d_dbg_conf;
  a.dbg_astar = ctx->d_dbg_astar;
  a.pairs = ctx->d_pairctr;
  a.prof = ctx->launch.profile ? ctx->d_prof : nullptr;
  a.stepx = ctx->d_stepx;
  a.bak = ctx->d_bak;  // used only by requests with Req::n_old > 0 (batch re-walks after a rollback)
  a.speed = ctx->d_speed;
  a.wb = ctx->d_wb;
  a.werr = ctx->d_wq ? ctx->d_wq + fmdp::XMAX * 4 : nullptr;
  a.vtrace = ctx->vtrace_n > 0 ? ctx->d_vtrace : nullptr;
  a.vtrace_n = ctx->vtrace_n;
  return a;
}

// Launch the walker over `run` with cluster size G and nc clusters (G = 0: cost model).
fmdp_status run_walk(fmdp_ctx* ctx, const std::vector<Req>& run, bool eval, int budget = INT_MAX,
                     const fmdp::WalkArgs* over = nullptr, int G = 0, int nc = 0) {
  if (run.empty()) return FMDP_OK;
  CK(cudaMemcpyAsync(ctx->d_reqs, run.data(), sizeof(Req) * run.size(), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_queue, 0, sizeof(int32_t), ctx->stream));
  fmdp::WalkArgs a = over ? *over : make_args(ctx, run, eval, budget);
  if (ctx->wide) {
    // wide walker: every cluster of the launch walks the same requests over its action
    // tile (its own request queue), all co-resident; fresh decision board (tags restart at 1)
    if (max_clusters(ctx, fmdp::WIDE_G) < ctx->wide_k)
      return fail(ctx, FMDP_E_CAPACITY, "wide walker: the action tiles' clusters are not co-resident");
    CK(cudaMemsetAsync(ctx->d_wq, 0, sizeof(int32_t) * (fmdp::XMAX * 4 + 4), ctx->stream));
    CK(cudaMemsetAsync(ctx->d_wb, 0, sizeof(unsigned long long) * 2 * fmdp::WB_WORDS * ctx->wide_k, ctx->stream));
    a.queue = ctx->d_wq;
    G = fmdp::WIDE_G;
    nc = ctx->wide_k;
  }
  if (G == 0) choose_launch(ctx, (int)run.size(), &G, &nc);
  ctx->stats.cluster_size = G;
  ctx->stats.walkers = std::max(ctx->stats.walkers, nc);
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  CK(fmdp::launch_walk(ctx->w, a, ctx->C, G, nc, threads_for(ctx), chunk_for(ctx), rawcap_for(ctx), ctx->stream));
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  CK(cudaEventSynchronize(ctx->ev1));
  CK(cudaGetLastError());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->stats.device_ms += ms;
  ctx->stats.kernels += 1;
  if (std::getenv("FMDP_DEBUG")) std::fprintf(stderr, "fmdp: walk n=%zu G=%d clusters=%d %.3f ms\n", run.size(), G, nc, ms);
  if (ctx->wide) {
    int32_t e = 0;
    CK(cudaMemcpy(&e, ctx->d_wq + fmdp::XMAX * 4, sizeof(e), cudaMemcpyDeviceToHost));
    if (e) return fail(ctx, FMDP_E_CUDA, "wide walker: decision board timed out");
  }
  return FMDP_OK;
}

// A split FCFS slice: the head (run[0], the earliest pending request -- everything before it is
// committed, so it can never be rolled back) alone at the cluster size a lone walker would use,
// on the library stream; the next two requests as lanes at the same size, and the other
// pending requests on the SMs left at half that size, concurrently.  They go on past `budget` until the head has
// finished (the device stop flag the head sets), so the slice is as long as the head's
// remaining trajectory -- the FCFS critical path -- and never waits on anything else.
fmdp_status run_split(fmdp_ctx* ctx, std::vector<Req>& run, int budget) {
  const int n = (int)run.size();
  for (Req& r : run) r.head = 0;
  run[0].head = 1;
  // the head runs as one cluster: splitting it over clusters (fmdp_launch.split) takes SMs from
  // the others and measured slower (configs[1]: 155.5 -> 171 ms per batch, tools/ab_headsplit.py)
  const int Gh = solo_cluster_size(ctx);
  // lanes: the next m = 2 requests also walk at the lone-walker cluster size -- their
  // speculative steps are the next slices' head work unless a commit rolls them back
  // (configs[1] full batch 115.3 / 109.2 / 108.6 / 111.8 / 115.0 / 121.5 ms for m = 0..5 with
  // the others at half the head's cluster size and the slice budget of 2; culled 58.6-59.0)
  // (FMDP_TUNE_LANES / FMDP_TUNE_GO: tuning overrides for tools/sweep_split.py only)
  static const int lanes_env = std::getenv("FMDP_TUNE_LANES") ? std::atoi(std::getenv("FMDP_TUNE_LANES")) : 2;
  static const int go_env = std::getenv("FMDP_TUNE_GO") ? std::atoi(std::getenv("FMDP_TUNE_GO")) : 0;
  static const int gl_env = std::getenv("FMDP_TUNE_GL") ? std::atoi(std::getenv("FMDP_TUNE_GL")) : 0;
  const int Gl = gl_env > 0 ? gl_env : Gh;  // the lanes' cluster size
  int m = std::min(lanes_env, n - 2);
  while (m > 0 && ctx->num_sms < Gh + m * Gl + 16) --m;
  const bool lane2 = m > 0;
  const int nl = 1 + m;
  // the others: clusters of half the head's size on the SMs left -- fewer, faster walkers on the
  // earliest pending requests, which become the next heads (the all-requests cost model of
  // choose_launch optimises the wrong objective here: configs[1] full batch 119.9 -> 111.7 ms,
  // culled 58.7 -> 58.5 ms, configs[2] unchanged)
  const int Go = go_env > 0 ? go_env : std::max(1, Gh / 2);
  const int nco =
      std::max(1, std::min(n - nl, std::min(max_clusters(ctx, Go), (ctx->num_sms - Gh - m * Gl) / Go)));
  CK(cudaMemcpyAsync(ctx->d_reqs, run.data(), sizeof(Req) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_queue, 0, 2 * sizeof(int32_t), ctx->stream));  // [0] head, [1] others
  CK(cudaMemsetAsync(ctx->d_queue + 3, 0, sizeof(int32_t), ctx->stream));  // [3] second lane
  CK(cudaMemsetAsync(ctx->d_stop, 0, sizeof(int32_t), ctx->stream));
  CK(cudaEventRecord(ctx->ev0, ctx->stream));
  CK(cudaStreamWaitEvent(ctx->stream2, ctx->ev0, 0));
  fmdp::WalkArgs ah = make_args(ctx, run, false, budget);
  ah.reqs = ctx->d_reqs;
  ah.n_reqs = 1;
  ah.queue = ctx->d_queue;
  ah.stop = ctx->d_stop;
  fmdp::WalkArgs ao = ah;
  ao.reqs = ctx->d_reqs + nl;
  ao.n_reqs = n - nl;
  ao.queue = ctx->d_queue + 1;
  CK(fmdp::launch_walk(ctx->w, ah, ctx->C, Gh, 1, threads_for(ctx), chunk_for(ctx), rawcap_for(ctx), ctx->stream));
  if (lane2) {
    fmdp::WalkArgs a2 = ah;
    a2.reqs = ctx->d_reqs + 1;
    a2.n_reqs = m;
    a2.queue = ctx->d_queue + 3;
    CK(cudaStreamWaitEvent(ctx->stream3, ctx->ev0, 0));
    CK(fmdp::launch_walk(ctx->w, a2, ctx->C, Gl, m, threads_for(ctx), chunk_for(ctx), rawcap_for(ctx), ctx->stream3));
    CK(cudaEventRecord(ctx->ev3, ctx->stream3));
  }
  CK(fmdp::launch_walk(ctx->w, ao, ctx->C, Go, nco, threads_for(ctx), chunk_for(ctx), rawcap_for(ctx), ctx->stream2));
  CK(cudaEventRecord(ctx->ev2, ctx->stream2));
  CK(cudaStreamWaitEvent(ctx->stream, ctx->ev2, 0));
  if (lane2) CK(cudaStreamWaitEvent(ctx->stream, ctx->ev3, 0));
  CK(cudaEventRecord(ctx->ev1, ctx->stream));
  CK(cudaEventSynchronize(ctx->ev1));
  CK(cudaGetLastError());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  ctx->stats.device_ms += ms;
  ctx->stats.kernels += 2 + (lane2 ? 1 : 0);
  ctx->stats.cluster_size = Gh;
  ctx->stats.walkers = std::max(ctx->stats.walkers, nl + nco);
  if (std::getenv("FMDP_DEBUG"))
    std::fprintf(stderr, "fmdp: split walk n=%d head G=%d others G=%d clusters=%d %.3f ms\n", n, Gh, Go, nco, ms);
  return FMDP_OK;
}

fmdp_status fetch_out(fmdp_ctx* ctx, int n) {
  CK(cudaMemcpyAsync(ctx->h_out.data(), ctx->d_out, sizeof(Out) * n, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return FMDP_OK;
}

// Append plans (already validated: rows in horizon, capacity checked by the caller) whose
// states are on the device.  Slots come from the host mirror, in plan order.
fmdp_status append_device(fmdp_ctx* ctx, const std::vector<int64_t>& t0, const std::vector<int32_t>& n,
                          const std::vector<const int32_t*>& d_states) {
  const int np = (int)t0.size();
  if (np == 0) return FMDP_OK;
  size_t tot = 0;
  int maxn = 0;
  for (int i = 0; i < np; ++i) {
    tot += n[i];
    maxn = std::max(maxn, n[i]);
  }
  // slots from a copy of the host mirror: ctx->counts changes only once the append succeeded
  std::vector<int32_t> cnt = ctx->counts;
  std::vector<int32_t> slots(tot);
  size_t o = 0;
  for (int i = 0; i < np; ++i)
    for (int s = 0; s < n[i]; ++s) slots[o++] = cnt[t0[i] + s]++;
  fmdp_status st = ensure_up(ctx, tot);
  if (st) return st;
  if (np > ctx->app_cap) {
    if ((st = grow(ctx, ctx->d_app, np))) return st;
    ctx->app_cap = np;
  }
  std::vector<AppendPlan> ap(np);
  o = 0;
  for (int i = 0; i < np; ++i) {
    ap[i].t0 = t0[i];
    ap[i].n = n[i];
    ap[i].pad = 0;
    ap[i].states = d_states[i];
    ap[i].slots = ctx->d_up + o;
    o += n[i];
  }
  CK(cudaMemcpyAsync(ctx->d_up, slots.data(), sizeof(int32_t) * tot, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_app, ap.data(), sizeof(AppendPlan) * np, cudaMemcpyHostToDevice, ctx->stream));
  CK(fmdp::launch_append(ctx->d_rows, ctx->w.row_cap, ctx->w.horizon, ctx->d_app, np, maxn, ctx->stream));
  CK(cudaMemcpyAsync(ctx->d_counts, cnt.data(), sizeof(int32_t) * cnt.size(), cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->counts.swap(cnt);
  ctx->stats.kernels += 1;
  return FMDP_OK;
}

bool rows_fit(const fmdp_ctx* ctx, const std::vector<int64_t>& t0, const std::vector<int32_t>& n) {
  std::vector<int32_t> extra;
  int64_t lo = INT64_MAX, hi = -1;
  for (size_t i = 0; i < t0.size(); ++i) {
    lo = std::min(lo, t0[i]);
    hi = std::max(hi, t0[i] + n[i]);
  }
  if (hi < 0) return true;
  extra.assign((size_t)(hi - lo), 0);
  for (size_t i = 0; i < t0.size(); ++i)
    for (int s = 0; s < n[i]; ++s)
      if (ctx->counts[t0[i] + s] + ++extra[t0[i] + s - lo] > ctx->w.row_cap) return false;
  return true;
}

// Commit accepted slots (in order): host plan records + device append.
fmdp_status commit_slots(fmdp_ctx* ctx, const std::vector<int>& slots, const std::vector<Req>& base,
                         const std::vector<uint64_t>& aircraft, std::vector<uint32_t>& plan_id) {
  if (slots.empty()) return FMDP_OK;
  std::vector<int64_t> t0;
  std::vector<int32_t> n;
  std::vector<const int32_t*> ds;
  for (int s : slots) {
    t0.push_back(base[s].t0);
    n.push_back(ctx->h_out[s].n_states);
    ds.push_back(ctx->d_traj + (size_t)s * ctx->cap_states * 3);
  }
  if (!rows_fit(ctx, t0, n)) return fail(ctx, FMDP_E_CAPACITY, "time row capacity exceeded on commit");
  std::vector<PlanRec> recs(slots.size());
  for (size_t i = 0; i < slots.size(); ++i) {
    recs[i].aircraft = aircraft[slots[i]];
    recs[i].t0 = t0[i];
    recs[i].states.resize((size_t)3 * n[i]);
    CK(cudaMemcpyAsync(recs[i].states.data(), ds[i], sizeof(int32_t) * 3 * n[i], cudaMemcpyDeviceToHost, ctx->stream));
  }
  // host records and plan ids only once the device append succeeded (append_device syncs)
  fmdp_status st = append_device(ctx, t0, n, ds);
  if (st) return st;
  for (size_t i = 0; i < slots.size(); ++i) {
    plan_id[slots[i]] = (uint32_t)ctx->plans.size();
    ctx->plans.push_back(std::move(recs[i]));
  }
  return FMDP_OK;
}

// First and last step of each (request i, plan j) pair that could see the plan: kf[2q], kf[2q + 1]
fmdp_status influence(fmdp_ctx* ctx, const std::vector<InflPair>& pairs, std::vector<int32_t>& kf) {
  kf.assign(2 * pairs.size(), INT_MAX);
  if (pairs.empty()) return FMDP_OK;
  if ((int)pairs.size() > ctx->pairs_cap) {
    fmdp_status s;
    if ((s = grow(ctx, ctx->d_pairs, pairs.size())) || (s = grow(ctx, ctx->d_kfirst, 2 * pairs.size()))) return s;
    ctx->pairs_cap = (int)pairs.size();
  }
  CK(cudaMemcpyAsync(ctx->d_pairs, pairs.data(), sizeof(InflPair) * pairs.size(), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(fmdp::launch_influence(ctx->d_traj, ctx->d_bak, ctx->cap_states, ctx->d_nstates, ctx->d_t0s, ctx->d_pairs,
                            (int)pairs.size(), ctx->iw, ctx->d_kfirst, ctx->stream));
  CK(cudaMemcpyAsync(kf.data(), ctx->d_kfirst, sizeof(int32_t) * 2 * pairs.size(), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->stats.kernels += 1;
  return FMDP_OK;
}

fmdp_status prepare_requests(fmdp_ctx* ctx, const fmdp_request* reqs, int n, std::vector<Req>& base) {
  base.resize(n);
  for (int i = 0; i < n; ++i) {
    Req& r = base[i];
    std::memset(&r, 0, sizeof(r));
    fmdp_status s;
    if ((s = quantize(ctx, reqs[i].src, r.src)) || (s = quantize(ctx, reqs[i].dst, r.dst))) return s;
    if (r.src[0] == r.dst[0] && r.src[1] == r.dst[1] && r.src[2] == r.dst[2])
      return fail(ctx, FMDP_E_ARG, "source equals destination");
    if (reqs[i].t0_step < 0 || reqs[i].t0_step + ctx->w.max_steps + 2 > ctx->w.horizon)
      return fail(ctx, FMDP_E_RANGE, "t0 + max_steps + 1 must lie inside the store horizon");
    r.t0 = reqs[i].t0_step;
    r.psi0 = initial_heading(ctx, r.src, r.dst);
    r.start_k = 0;
    r.slot = i;
  }
  return FMDP_OK;
}

// Clusters for one request walked alone (fmdp_launch.split): 1, or k clusters of G = 16 or 8
// CTAs each over a shard of every row, combined per step by the in-kernel exchange.  Auto: the
// cost model t(G, k) = step_cycles(plans / k, G) + exchange, exchange = 2400 + 1150 (k - 1)
// cycles (fit to tools/p2p_probe.py at 3000 / 30000 plans, profiles/r01_p2p_probe.txt), the
// k clusters resident at once.  Returns k (1: no split) and the cluster size in *G_out.
// SURVEY f1 range query: sort every row's plans by x-y cell of side L (World::cell_*), L covering a
// plan's largest well offset k_max |v_h| (measured over the store), R_max, the projection reach and
// four steps of ownship motion (the walker stages row K + 2 around q_{k-1}; the pre-cull tests row
// K + 1 against q_k).  Appended plans go past the sorted regions and are scanned in full.  Rows are
// identical on every rank of a plan-sharded exchange (stable, deterministic sort).
constexpr int kIndexMinPlansPerRow = 10000;
fmdp_status build_index(fmdp_ctx* ctx) {
  fmdp::World& w = ctx->w;
  w.cell_n = 0;
  ctx->index_dirty = false;
  ctx->n_indexed = 0;
  static const bool off = std::getenv("FMDP_NO_INDEX") != nullptr;  // A/B switch
  if (off || ctx->wide || ctx->plans.empty()) return FMDP_OK;
  // only for large rows: at configs[1] scale (3000 plans per row) the staging of up to four pieces
  // and the cell lookups of the I/O thread cost more per step than the scan of the whole slice
  // (measured: culled step 5.05 -> 6.26 us), at configs[3] (100k) the range query wins (8.5 -> 6.7
  // us/step on one 2-CTA cluster instead of 4 x 16 CTAs, batch of 100: 198 -> 61 ms)
  {
    int64_t tot = 0, nz = 0;
    for (int32_t c : ctx->counts)
      if (c) { tot += c; ++nz; }
    if (nz == 0 || tot < (int64_t)kIndexMinPlansPerRow * nz) return FMDP_OK;
  }
  unsigned long long* d_v = nullptr;
  if ((d_v = (unsigned long long*)dalloc(ctx, sizeof(unsigned long long))) == nullptr)
    return fail(ctx, FMDP_E_NOMEM, "index scratch");
  CK(cudaMemsetAsync(d_v, 0, sizeof(unsigned long long), ctx->stream));
  CK(fmdp::launch_vmax(ctx->d_rows, w.row_cap, ctx->d_counts, w.horizon, d_v, ctx->stream));
  unsigned long long v2 = 0;
  CK(cudaMemcpyAsync(&v2, d_v, sizeof(v2), cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  dfree(ctx, d_v);
  const int64_t vh = (int64_t)std::ceil(std::sqrt((double)v2));
  int64_t L = (int64_t)w.R_max + w.reach_u + 4LL * w.step_reach_u + (int64_t)w.k_absmax * vh + 2;
  const int64_t sx = ctx->hi_u[0] - ctx->lo_u[0] + 1, sy = ctx->hi_u[1] - ctx->lo_u[1] + 1;
  // at most 16384 cells (the sort's shared histogram) and 1 GB of cstart offsets
  auto cells = [&](int64_t l) { return ((sx + l - 1) / l) * ((sy + l - 1) / l); };
  while (cells(L) > 16384 || (double)w.horizon * (cells(L) + 1) * 4.0 > (double)(1LL << 30)) {
    if (cells(L) < 16) return FMDP_OK;
    L += L / 8 + 1;
  }
  const int ncx = (int)((sx + L - 1) / L), ncy = (int)((sy + L - 1) / L);
  if (ncx * ncy < 16) return FMDP_OK;  // too few cells to pay (a 4x4 grid reads 9/16 of a row)
  const size_t cs_words = (size_t)w.horizon * (ncx * ncy + 1);
  if (cs_words > ctx->cstart_cap) {
    fmdp_status e;
    if ((e = grow(ctx, ctx->d_cstart, cs_words))) return e;
    ctx->cstart_cap = cs_words;
  }
  const int64_t per_row = (int64_t)4 * w.row_cap;
  const int B = (int)std::max<int64_t>(1, std::min<int64_t>(1024, ((int64_t)1 << 28) / per_row));
  if ((size_t)B * per_row > ctx->itmp_cap) {
    fmdp_status e;
    if ((e = grow(ctx, ctx->d_itmp, (size_t)B * per_row))) return e;
    ctx->itmp_cap = (size_t)B * per_row;
  }
  ctx->n_indexed = ctx->plans.size();  // from here on the rows are permuted: truncating reloads
  fmdp::World wi = w;
  wi.cell_n = ncx * ncy;
  wi.cell_ncx = ncx;
  wi.cell_ncy = ncy;
  wi.cell_l = (int32_t)L;
  wi.cell_x0 = (int32_t)ctx->lo_u[0];
  wi.cell_y0 = (int32_t)ctx->lo_u[1];
  wi.cstart = ctx->d_cstart;
  for (int64_t K0 = 0; K0 < w.horizon; K0 += B) {
    const int nr = (int)std::min<int64_t>(B, w.horizon - K0);
    CK(fmdp::launch_index(ctx->d_rows, w.row_cap, ctx->d_counts, K0, nr, wi, ctx->d_cstart, ctx->d_itmp, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  w = wi;
  return FMDP_OK;
}

// Before a culled walk: (re)build the range-query index if plans were added since the last build.
// Plan-sharded calls (always: sharded = false -> true) sort too, culled or not, so that every rank --
// same plans added in the same order -- holds the same row order (each evaluates a slot range).
fmdp_status ensure_index(fmdp_ctx* ctx, bool sharded = false) {
  if ((!ctx->launch.cull && !sharded) || !ctx->index_dirty) return FMDP_OK;
  return build_index(ctx);
}

int split_for(fmdp_ctx* ctx, int* G_out) {
  *G_out = 16;
  if (ctx->launch.split == 1) return 1;
  if (ctx->launch.cull && ctx->w.cell_n > 0 && ctx->idx_cost && ctx->launch.split == 0) return 1;  // range query
  const double plans = mean_plans(ctx);
  int best = 1, bestG = 16;
  double tb = step_cycles(ctx, plans, solo_cluster_size(ctx));
  for (int G : {16, 8}) {
    if (ctx->launch.cluster_size && ctx->launch.cluster_size != G) continue;
    const int kmax = std::min(fmdp::XMAX, std::min(ctx->num_sms / G, max_clusters(ctx, G)));
    if (ctx->launch.split >= 2) {  // forced k: the largest cluster size that fits it
      if (kmax >= std::min(ctx->launch.split, fmdp::XMAX) || G == 8) {
        *G_out = G;
        return std::max(1, std::min(ctx->launch.split, kmax));
      }
      continue;
    }
    for (int k = 2; k <= kmax; ++k) {
      const double t = step_cycles(ctx, plans / k, G) + 2400.0 + 1150.0 * (k - 1);
      if (t < tb - 1e-9) {
        tb = t;
        best = k;
        bestG = G;
      }
    }
  }
  *G_out = bestG;
  return best;
}

// Exchange state of a request split over k clusters of this GPU (allocated once; a new k
// resets the areas and tag sequences) and the walk arguments that select it.
fmdp_status prepare_intra(fmdp_ctx* ctx, int k, fmdp::WalkArgs& a) {
  const int slot = ((ctx->A * ctx->W * fmdp::NTAU + 16) + 3) & ~3;
  const size_t area_words = fmdp::x_area_bytes(fmdp::XMAX, slot) / sizeof(unsigned long long);
  if (!ctx->d_xin_area || !ctx->d_xin_peers || !ctx->d_xin_seq) {
    if (!ctx->d_xin_area)
      ctx->d_xin_area = (unsigned long long*)dalloc(ctx, sizeof(unsigned long long) * area_words * fmdp::XMAX);
    if (!ctx->d_xin_peers) ctx->d_xin_peers = (fmdp::XPeer*)dalloc(ctx, sizeof(fmdp::XPeer) * fmdp::XMAX);
    if (!ctx->d_xin_seq)
      ctx->d_xin_seq = (unsigned long long*)dalloc(ctx, sizeof(unsigned long long) * (fmdp::XMAX + 1 + fmdp::XMAX));
    if (!ctx->d_xin_area || !ctx->d_xin_peers || !ctx->d_xin_seq) return fail(ctx, FMDP_E_NOMEM, "split exchange");
    ctx->xin_world = 0;
  }
  unsigned long long* seq = ctx->d_xin_seq;
  int32_t* err = reinterpret_cast<int32_t*>(seq + fmdp::XMAX);
  int32_t* queue = reinterpret_cast<int32_t*>(seq + fmdp::XMAX + 1);
  if (k != ctx->xin_world) {  // new layout: clean areas, tags restart
    std::vector<fmdp::XPeer> tab(fmdp::XMAX, fmdp::XPeer{nullptr});
    for (int q = 0; q < k; ++q) tab[q].recv = ctx->d_xin_area + (size_t)q * area_words;
    CK(cudaMemcpyAsync(ctx->d_xin_peers, tab.data(), sizeof(fmdp::XPeer) * fmdp::XMAX, cudaMemcpyHostToDevice,
                       ctx->stream));
    CK(cudaMemsetAsync(ctx->d_xin_area, 0, sizeof(unsigned long long) * area_words * fmdp::XMAX, ctx->stream));
    CK(cudaMemsetAsync(seq, 0, sizeof(unsigned long long) * (fmdp::XMAX + 1), ctx->stream));
    ctx->xin_world = k;
  }
  CK(cudaMemsetAsync(queue, 0, sizeof(int32_t) * fmdp::XMAX, ctx->stream));
  a.xmode = 3;
  a.shard_rank = 0;
  a.shard_world = k;
  a.x_intra = 1;
  a.x_me = 0;
  a.x_world = k;
  a.x_slot = slot;
  a.x_peers = ctx->d_xin_peers;
  a.x_seq = seq;
  a.x_err = err;
  a.queue = queue;
  return FMDP_OK;
}

fmdp_status check_intra(fmdp_ctx* ctx) {
  int32_t e = 0;
  CK(cudaMemcpy(&e, ctx->d_xin_seq + fmdp::XMAX, sizeof(e), cudaMemcpyDeviceToHost));
  if (e) {
    ctx->xin_world = 0;
    return fail(ctx, FMDP_E_CUDA, "split request: cluster exchange timed out (clusters not co-resident)");
  }
  return FMDP_OK;
}

// One request, alone on the device: a plain walk, or split over k clusters (bit-identical).
fmdp_status run_single(fmdp_ctx* ctx, const Req& r) {
  if (ctx->wide) return run_walk(ctx, {r}, false);
  int G = 16;
  const int k = split_for(ctx, &G);
  if (k <= 1) return run_walk(ctx, {r}, false);
  fmdp::WalkArgs a = make_args(ctx, {r}, false, INT_MAX);
  fmdp_status st = prepare_intra(ctx, k, a);
  if (st) return st;
  if ((st = run_walk(ctx, {r}, false, INT_MAX, &a, G, k))) return st;
  ctx->stats.split = k;
  return check_intra(ctx);
}

// Request-sharded FCFS (fmdp_schedule_batch_dist): after a round, every rank's requests that finished
// in it -- Out record, trajectory, headings, actions, near-tie flags -- are all-gathered, written
// into every rank's scratch (device and h_out) at their slots, and marked finished, so every rank
// sees the same finished set and takes the same commit / rollback decisions.
struct FinRec {
  int32_t slot, n;
  Out out;
};
fmdp_status gather_finished(fmdp_ctx* ctx, const fmdp_gather* g, const std::vector<int>& mine, std::vector<char>& fin,
                            std::vector<int>& kdone) {
  const size_t cap = (size_t)ctx->cap_states;
  std::vector<unsigned char> buf;
  auto put = [&](const void* p, size_t b) {
    const size_t o = buf.size();
    buf.resize(o + ((b + 7) & ~size_t(7)));
    std::memcpy(buf.data() + o, p, b);
  };
  for (int s : mine) {
    const Out& o = ctx->h_out[s];
    FinRec r{s, o.n_states, o};
    put(&r, sizeof(r));
    const size_t n = (size_t)o.n_states;
    std::vector<int32_t> tmp(3 * n);
    CK(cudaMemcpy(tmp.data(), ctx->d_traj + s * cap * 3, sizeof(int32_t) * 3 * n, cudaMemcpyDeviceToHost));
    put(tmp.data(), sizeof(int32_t) * 3 * n);
    CK(cudaMemcpy(tmp.data(), ctx->d_heading + s * cap, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    put(tmp.data(), sizeof(int32_t) * n);
    CK(cudaMemcpy(tmp.data(), ctx->d_astar + s * cap, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    put(tmp.data(), sizeof(int32_t) * n);
    std::vector<int8_t> nt(n);
    CK(cudaMemcpy(nt.data(), ctx->d_ntie + s * cap, n, cudaMemcpyDeviceToHost));
    put(nt.data(), n);
  }
  const int W = g->world;
  int64_t mine_b = (int64_t)buf.size();
  std::vector<int64_t> sizes(W);
  if (g->allgather(&mine_b, sizes.data(), sizeof(int64_t), g->user))
    return fail(ctx, FMDP_E_INTERNAL, "allgather callback failed (sizes)");
  int64_t mx = 0;
  for (int64_t b : sizes) mx = std::max(mx, b);
  if (mx == 0) return FMDP_OK;
  buf.resize((size_t)mx, 0);
  std::vector<unsigned char> all((size_t)mx * W);
  if (g->allgather(buf.data(), all.data(), mx, g->user))
    return fail(ctx, FMDP_E_INTERNAL, "allgather callback failed (records)");
  for (int q = 0; q < W; ++q) {
    const unsigned char* p = all.data() + (size_t)q * mx;
    const unsigned char* e = p + sizes[q];
    while (p < e) {
      FinRec r;
      std::memcpy(&r, p, sizeof(r));
      p += (sizeof(r) + 7) & ~size_t(7);
      const size_t n = (size_t)r.n;
      const size_t s = (size_t)r.slot;
      const size_t bt = sizeof(int32_t) * 3 * n, bh = sizeof(int32_t) * n;
      if (q != g->rank) {
        ctx->h_out[s] = r.out;
        CK(cudaMemcpy(ctx->d_out + s, &r.out, sizeof(Out), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_traj + s * cap * 3, p, bt, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_heading + s * cap, p + ((bt + 7) & ~size_t(7)), bh, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_astar + s * cap, p + ((bt + 7) & ~size_t(7)) + ((bh + 7) & ~size_t(7)), bh,
                      cudaMemcpyHostToDevice));
        CK(cudaMemcpy(ctx->d_ntie + s * cap, p + ((bt + 7) & ~size_t(7)) + 2 * ((bh + 7) & ~size_t(7)), n,
                      cudaMemcpyHostToDevice));
      }
      p += ((bt + 7) & ~size_t(7)) + 2 * ((bh + 7) & ~size_t(7)) + ((n + 7) & ~size_t(7));
      fin[s] = 1;
      kdone[s] = r.n - 1;
    }
  }
  return FMDP_OK;
}

// Result trajectories of slots [0, n) into the caller's buffer (traj_cap_each states per request):
// packed on the device (pack_traj_kernel), one D2H copy into pinned memory, scattered on the host --
// one copy per batch instead of one pageable copy per request (the e2e path's copy-out).
fmdp_status copy_out_traj(fmdp_ctx* ctx, int n, fmdp_qpos* traj, int32_t traj_cap_each) {
  std::vector<int64_t> off(n);
  int64_t tot = 0;
  for (int i = 0; i < n; ++i) {
    off[i] = tot;
    tot += ctx->h_out[i].n_states;
  }
  if (tot == 0) return FMDP_OK;
  if ((size_t)tot * 3 > ctx->pack_cap) {
    const size_t m = std::max((size_t)tot * 3, 2 * ctx->pack_cap);
    int32_t* hp = nullptr;
    if (cudaMallocHost(&hp, sizeof(int32_t) * m) != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, FMDP_E_NOMEM, "pinned host allocation failed (trajectory copy-out)");
    }
    fmdp_status s;
    if ((s = grow(ctx, ctx->d_pack, m))) {
      cudaFreeHost(hp);
      return s;
    }
    if (ctx->h_pack) cudaFreeHost(ctx->h_pack);
    ctx->h_pack = hp;
    ctx->pack_cap = m;
  }
  if ((size_t)n > ctx->packoff_cap) {
    fmdp_status s;
    if ((s = grow(ctx, ctx->d_packoff, (size_t)n))) return s;
    ctx->packoff_cap = (size_t)n;
  }
  CK(cudaMemcpyAsync(ctx->d_packoff, off.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, ctx->stream));
  CK(fmdp::launch_pack_traj(ctx->d_traj, ctx->cap_states, ctx->d_out, ctx->d_packoff, n, ctx->d_pack, ctx->stream));
  ctx->stats.kernels += 1;
  CK(cudaMemcpyAsync(ctx->h_pack, ctx->d_pack, sizeof(int32_t) * 3 * tot, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  for (int i = 0; i < n; ++i)
    std::memcpy(traj + (size_t)i * traj_cap_each, ctx->h_pack + 3 * off[i], sizeof(fmdp_qpos) * ctx->h_out[i].n_states);
  return FMDP_OK;
}

fmdp_status schedule_many(fmdp_ctx* ctx, const fmdp_request* reqs, int n, fmdp_result* res, fmdp_qpos* traj,
                          int32_t traj_cap_each, int32_t flags, const fmdp_gather* g = nullptr) {
  const bool dist = g && g->world > 1;
  if (dist && (g->rank < 0 || g->rank >= g->world || !g->allgather))
    return fail(ctx, FMDP_E_ARG, "invalid fmdp_gather");
  if (dist && (ctx->wide || (flags & FMDP_BATCH_SEQUENTIAL)))
    return fail(ctx, FMDP_E_ARG, "request sharding needs the speculative constant-speed batch");
  if (!ctx || (n > 0 && (!reqs || !res)) || n < 0) return fail(ctx, FMDP_E_ARG, "null argument");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  if (traj && traj_cap_each < ctx->w.max_steps + 1)
    return fail(ctx, FMDP_E_BUFFER, "traj_cap must be >= max_steps + 1");
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  if (n == 0) return FMDP_OK;
  {
    const fmdp_status e = ensure_index(ctx);
    if (e) return e;
  }
  std::vector<Req> base;
  fmdp_status st = prepare_requests(ctx, reqs, n, base);
  if (st) return st;
  if ((st = ensure_slots(ctx, n))) return st;
  std::vector<uint64_t> aircraft(n);
  for (int i = 0; i < n; ++i) aircraft[i] = reqs[i].aircraft_id;
  std::vector<uint32_t> plan_id(n, 0xffffffffu);
  CK(cudaMemsetAsync(ctx->d_pairctr, 0, sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_prof, 0, sizeof(unsigned long long) * fmdp::N_PHASES, ctx->stream));
  std::vector<int64_t> t0s(n);
  for (int i = 0; i < n; ++i) t0s[i] = base[i].t0;
  CK(cudaMemcpyAsync(ctx->d_t0s, t0s.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice, ctx->stream));

  int runs = 0;
  if ((flags & FMDP_BATCH_SEQUENTIAL) || ctx->wide) {  // wide walks take the whole GPU: in order
    for (int i = 0; i < n; ++i) {
      if ((st = run_single(ctx, base[i]))) return st;
      ++runs;
      ctx->stats.rounds += 1;
      if ((st = fetch_out(ctx, n))) return st;
      ctx->stats.steps += ctx->h_out[i].steps_run;
      if (ctx->h_out[i].status == FMDP_ACCEPTED && (st = commit_slots(ctx, {i}, base, aircraft, plan_id))) return st;
    }
  } else {
    // Speculative FCFS in time slices (DESIGN.md a10).  Invariant at the top of every
    // slice: the steps already computed for every pending request are consistent with the
    // current store.  A slice advances every unfinished request by at most `budget` steps
    // (cluster size re-chosen for the shrinking count), then commits the finished FCFS prefix
    // and rolls back any pending request whose computed steps could see a newly committed
    // plan to its first influenced step.  Result: identical to the sequential loop.
    // slice budget: measured optimum on configs[1] (tools/sweep_budget.py)
    // The others of a split slice run until the head has finished and then `budget` more steps
    // at most, so the budget only lengthens a slice past the FCFS critical path: measured best
    // (tools/sweep_budget.py, profiles/r01_sweep_budget.txt) 1-2 on both paths (full 676 -> 750
    // req/s against 128 before the lanes; culled 1647 -> 1694 against 64 with them)
    const int budget = ctx->launch.step_budget > 0 ? ctx->launch.step_budget : 2;
    std::vector<char> fin(n, 0);
    std::vector<int> kdone(n, 0);
    int rollbacks = 0;
    // Re-convergence: a finished request that a commit rolls back keeps its previous
    // run in the backup arrays; the re-walk takes that run over as soon as its state equals the old
    // one past every influenced step (ru.from).  Commits that can influence the backup's states
    // raise ru.from (influence pairs against the backup).  Off for request sharding, and on the
    // full path (only the culled walker carries the check: the full batches measured no gain).
    struct Reuse {
      bool on = false;
      int n_old = 0, old_status = 0, old_fail = -1, bak_lo = 0, from = 0;
    };
    static const bool no_reuse = std::getenv("FMDP_NO_REUSE") != nullptr;  // A/B switch
    const bool reuse_ok = !dist && !no_reuse && ctx->launch.cull;
    std::vector<Reuse> ru(n);
    auto backup = [&](int i, int lo, int hi) -> fmdp_status {
      CK(fmdp::launch_backup(ctx->d_bak, ctx->d_traj, ctx->d_heading, ctx->d_astar, ctx->d_stepx, ctx->d_stepd2,
                             ctx->d_ntie, ctx->cap_states, i, lo, hi, ctx->stream));
      return FMDP_OK;
    };
    int c = 0;
    while (c < n) {
      std::vector<Req> run;
      for (int i = c; i < n; ++i)
        if (!fin[i] && (!dist || i % g->world == g->rank)) {  // request sharding: rank i % world
          Req r = base[i];
          r.start_k = kdone[i];
          if (ru[i].on) {
            r.n_old = ru[i].n_old;
            r.reuse_from = ru[i].from;
            r.old_status = ru[i].old_status;
            r.old_fail = ru[i].old_fail;
          }
          run.push_back(r);
        }
      if (!run.empty()) {
        // A slice whose walkers are all resident at the cluster size a lone walker would use
        // runs the head (request c: everything before it is committed, so it can never be
        // rolled back) to completion; the others go on past `budget` until it is done -- their
        // extra steps cost no wall time and stay valid unless a rollback discards them.
        if (run.size() >= 2) {
          if ((st = run_split(ctx, run, budget))) return st;  // run[0] is request c
        } else {
          run[0].head = 1;
          fmdp::WalkArgs a = make_args(ctx, run, false, budget);
          CK(cudaMemsetAsync(ctx->d_stop, 0, sizeof(int32_t), ctx->stream));
          a.stop = ctx->d_stop;
          if ((st = run_walk(ctx, run, false, budget, &a, solo_cluster_size(ctx), 1))) return st;
        }
        runs += (int)run.size();
        ctx->stats.rounds += 1;
      }
      const auto th0 = std::chrono::steady_clock::now();  // (FMDP_DEBUG: host time between slices)
      if ((st = fetch_out(ctx, n))) return st;
      const auto th1 = std::chrono::steady_clock::now();
      std::vector<int> mine;  // own requests that finished in this round
      for (const Req& r : run) {
        const Out& o = ctx->h_out[r.slot];
        ctx->stats.steps += o.steps_run;
        ctx->stats.reconverged += o.reconv;
        if (o.reconv) ru[r.slot].on = false;  // its records are one consistent run again
        if (o.status < 0) kdone[r.slot] = o.n_states - 1;
        else {
          fin[r.slot] = 1;
          mine.push_back(r.slot);
          ru[r.slot].on = false;
        }
      }
      if (dist && (st = gather_finished(ctx, g, mine, fin, kdone))) return st;
      // influence of every finished, accepted request j that can be committed in this slice --
      // the finished run [c, c_end) -- on every later request i (only newly committed plans
      // can roll anything back, and only requests of that run can be committed now)
      int c_end = c;
      while (c_end < n && fin[c_end]) ++c_end;
      std::vector<InflPair> pairs;
      std::vector<int32_t> ns(n);
      for (int i = 0; i < n; ++i) ns[i] = ctx->h_out[i].n_states;
      for (int j = c; j < c_end; ++j)
        if (ctx->h_out[j].status == FMDP_ACCEPTED)
          for (int i = j + 1; i < n; ++i) {  // sharded: the trajectories this rank holds
            if (!dist || fin[i] || i % g->world == g->rank) pairs.push_back({i, j, 0, -1, 0});
            if (ru[i].on) pairs.push_back({i, j, ru[i].bak_lo, ru[i].n_old, 1});  // i's previous run
          }
      std::vector<int32_t> kf;
      const auto th2 = std::chrono::steady_clock::now();
      if (!pairs.empty()) {
        CK(cudaMemcpyAsync(ctx->d_nstates, ns.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice, ctx->stream));
        if ((st = influence(ctx, pairs, kf))) return st;
      }
      // pairs by request i (first influenced step kf), and the plans committed so far
      std::vector<std::vector<std::pair<int, int>>> by_i(n), by_last(n), by_bak(n);
      for (size_t q = 0; q < pairs.size(); ++q)
        if (kf[2 * q] != INT_MAX) {
          if (pairs[q].bak) {
            by_bak[pairs[q].i].push_back({pairs[q].j, kf[2 * q + 1]});
          } else {
            by_i[pairs[q].i].push_back({pairs[q].j, kf[2 * q]});
            by_last[pairs[q].i].push_back({pairs[q].j, kf[2 * q + 1]});
          }
        }
      std::vector<int> newly;
      std::vector<char> is_new(n, 0);
      auto first_influence = [&](int i) {
        int best = INT_MAX;
        for (const auto& e : by_i[i])
          if (is_new[e.first]) best = std::min(best, e.second);
        return best;
      };
      auto last_influence = [&](const std::vector<std::pair<int, int>>& v) {
        int kl = -1;
        for (const auto& e : v)
          if (is_new[e.first]) kl = std::max(kl, e.second);
        return kl;
      };
      // rollback of request i to step k1: keep (fin: start) or extend its previous run's backup
      auto note_rb = [&](int i, int k1, bool finished) -> fmdp_status {
        if (!reuse_ok) return FMDP_OK;
        Reuse& u = ru[i];
        const int kl = last_influence(by_last[i]);
        if (finished || !u.on) {  // keep the run computed so far (final, or paused at n_states - 1)
          const Out& o = ctx->h_out[i];
          u.on = true;
          u.n_old = o.n_states;
          u.old_status = o.status;  // (-1: paused)
          u.old_fail = o.fail_step;
          u.bak_lo = k1;
          u.from = kl + 1;
          fmdp_status e = backup(i, k1, u.n_old);
          if (e) return e;
        } else {
          if (k1 < u.bak_lo) {  // states [k1, bak_lo) are still the previous run's
            fmdp_status e = backup(i, k1, u.bak_lo);
            if (e) return e;
            u.bak_lo = k1;
          }
          u.from = std::max(u.from, kl + 1);
        }
        if (u.on && u.from >= u.n_old) u.on = false;
        return FMDP_OK;
      };
      while (c < n && fin[c]) {
        const int k1 = first_influence(c);
        if (k1 != INT_MAX) {
          if ((st = note_rb(c, k1, true))) return st;
          fin[c] = 0;
          kdone[c] = k1;
          ++rollbacks;
          if ((st = clear_stepx(ctx, c, k1))) return st;
          break;
        }
        if (ctx->h_out[c].status == FMDP_ACCEPTED) {
          newly.push_back(c);
          is_new[c] = 1;
        }
        ++c;
      }
      const auto th3 = std::chrono::steady_clock::now();
      if ((st = commit_slots(ctx, newly, base, aircraft, plan_id))) return st;
      const auto th4 = std::chrono::steady_clock::now();
      if (std::getenv("FMDP_DEBUG")) {
        auto us = [](auto a, auto b) { return std::chrono::duration<double, std::micro>(b - a).count(); };
        std::fprintf(stderr, "fmdp: host us fetch=%.0f pairs=%.0f influence+rollback=%.0f commit=%.0f\n", us(th0, th1),
                     us(th1, th2), us(th2, th3), us(th3, th4));
        int pend = 0, prog = 0;
        for (int i = c; i < n; ++i) pend += fin[i] ? 0 : 1;
        for (const Req& r : run) prog += ctx->h_out[r.slot].steps_run > 0 ? 1 : 0;
        std::fprintf(stderr, "fmdp: slice head=%d head_steps=%d committed=%zu next_head=%d pending=%d progressed=%d/%zu\n",
                     run.empty() ? -1 : run[0].slot, run.empty() ? 0 : ctx->h_out[run[0].slot].steps_run, newly.size(), c,
                     pend, prog, run.size());
      }
      for (int i = c; i < n; ++i) {  // includes the unfinished head c
        if (ru[i].on) {  // commits that can see the previous run's states
          ru[i].from = std::max(ru[i].from, last_influence(by_bak[i]) + 1);
          if (ru[i].from >= ru[i].n_old) ru[i].on = false;
        }
        const int k1 = first_influence(i);
        if (k1 == INT_MAX) continue;
        if (fin[i]) {
          if ((st = note_rb(i, k1, true))) return st;
          fin[i] = 0;
          kdone[i] = k1;
          ++rollbacks;
          if ((st = clear_stepx(ctx, i, k1))) return st;
        } else if (k1 < kdone[i]) {
          if ((st = note_rb(i, k1, false))) return st;
          kdone[i] = k1;
          ++rollbacks;
          if ((st = clear_stepx(ctx, i, k1))) return st;
        }
      }
    }
    runs = n + rollbacks;
  }
  ctx->stats.reruns = runs - n;
  if ((st = fetch_out(ctx, n))) return st;
  unsigned long long pc = 0;
  CK(cudaMemcpy(&pc, ctx->d_pairctr, sizeof(pc), cudaMemcpyDeviceToHost));
  ctx->stats.pair_evals = (int64_t)pc;
  if (ctx->launch.profile) {
    unsigned long long ph[fmdp::N_PHASES];
    CK(cudaMemcpy(ph, ctx->d_prof, sizeof(ph), cudaMemcpyDeviceToHost));
    for (int i = 0; i < fmdp::N_PHASES; ++i) ctx->stats.phase_cycles[i] = (int64_t)ph[i];
  }
  for (int i = 0; i < n; ++i) {
    const Out& o = ctx->h_out[i];
    res[i].status = o.status;
    res[i].plan_id = plan_id[i];
    res[i].n_states = o.n_states;
    res[i].fail_step = o.fail_step;
    res[i].min_sep_m = std::sqrt((double)o.min_sep_d2) * ctx->air.u_m;
    res[i].n_near_ties = o.n_near_ties;
    res[i].n_exact = o.n_exact;
  }
  if (traj && (st = copy_out_traj(ctx, n, traj, traj_cap_each))) return st;
  ctx->last_n = n;
  return FMDP_OK;
}

}  // namespace

// ============================================================================ C ABI
extern "C" {

void fmdp_airspace_default(fmdp_airspace* a) {
  static const int32_t turns[9] = {-8, -6, -4, -2, 0, 2, 4, 6, 8};
  static const int32_t climbs[3] = {-16, 0, 16};
  static const double taus[5] = {-5.0, 0.0, 5.0, 10.0, 15.0};
  static const double radii[5] = {250.0, 300.0, 350.0, 400.0, 450.0};
  std::memset(a, 0, sizeof(*a));
  a->abi_version = FMDP_ABI_VERSION;
  a->lo = {-8000.0, -8000.0, 0.0};
  a->hi = {8000.0, 8000.0, 1500.0};
  a->u_m = 1.0 / 64.0;
  a->dt = 0.1;
  a->window = 10;
  a->speed = 50.0;
  a->heading_lattice = 1440;
  a->n_turn = 9;
  a->turn_steps = turns;
  a->n_climb = 3;
  a->climb_units = climbs;
  a->goal_r = 200.0;
  a->goal_gamma = 0.999;
  a->intr_r = 1000.0;
  a->intr_gamma = 0.97;
  a->n_tau = 5;
  a->tau_s = taus;
  a->tau_radius_m = radii;
  a->terr_r = 1000.0;
  a->terr_gamma = 0.99;
  a->deck_alt_m = 30.0;
  a->deck_scale = 1000.0;
  a->capture_radius_m = 100.0;
  a->sep_min_m = 150.0;
  a->max_steps = 4000;
  a->vmax_init_zero = 0;
  a->valuation = 0;
  static const int32_t accs[1] = {0};
  a->n_acc = 1;
  a->acc_units = accs;
  a->speed_min = 0.0;
  a->speed_max = 0.0;
  a->near_tie_rel = 1e-4;
  a->horizon_steps = 8192;
  a->row_capacity = 4096;
}

const char* fmdp_strerror(fmdp_status s) {
  if (s == FMDP_E_INTERNAL) return "internal error";
  const int i = -s;
  if (i >= 0 && i < (int)(sizeof(kStatusText) / sizeof(kStatusText[0]))) return kStatusText[i];
  return "unknown status";
}

const char* fmdp_last_error(const fmdp_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

int32_t fmdp_num_actions(const fmdp_ctx* ctx) { return ctx ? ctx->A : 0; }

fmdp_status fmdp_create(const fmdp_airspace* air, const fmdp_terrain* ter, const fmdp_devices* devs,
                        fmdp_ctx** out) {
  if (!air || !out) return FMDP_E_ARG;
  *out = nullptr;
  if (air->abi_version != FMDP_ABI_VERSION) {
    g_create_error = "fmdp_airspace.abi_version does not match FMDP_ABI_VERSION (header / library mismatch)";
    return FMDP_E_ARG;
  }
  fmdp_ctx* ctx = new (std::nothrow) fmdp_ctx();
  if (!ctx) return FMDP_E_NOMEM;
  auto bad = [&](fmdp_status s, const char* m) {  // release what was created so far
    g_create_error = m;
    fmdp_destroy(ctx);
    return s;
  };
  const fmdp_airspace& a = *air;
  if (!(a.u_m > 0) || !(a.dt > 0) || a.window < 1 || a.window > fmdp::MAX_W) return bad(FMDP_E_ARG, "u/dt/window");
  if (a.heading_lattice < 8 || a.heading_lattice % 8) return bad(FMDP_E_ARG, "heading_lattice % 8");
  if (a.n_turn < 1 || a.n_turn > fmdp::MAX_TURN || !a.turn_steps) return bad(FMDP_E_ARG, "turns");
  for (int i = 0; i < a.n_turn; ++i)
    if ((int64_t)std::abs(a.turn_steps[i]) * a.window >= a.heading_lattice)  // the kernel wraps psi + t h once
      return bad(FMDP_E_ARG, "turn step x window beyond the lattice");
  if (a.n_acc < 1 || a.n_acc > fmdp::MAX_ACC || !a.acc_units) return bad(FMDP_E_ARG, "n_acc / acc_units");
  const bool wide = a.n_acc > 1 || a.acc_units[0] != 0 || a.speed_min > 0 || a.speed_max > 0;
  if (!a.climb_units || (wide ? !(a.n_climb == 3 || a.n_climb == 10)
                              : !(a.n_climb == 1 || a.n_climb == 3 || a.n_climb == 5)))
    return bad(FMDP_E_ARG, wide ? "climbs: 3 or 10 with acceleration actions" : "climbs");
  if (a.n_tau < 1 || a.n_tau > fmdp::NTAU || !a.tau_s || !a.tau_radius_m) return bad(FMDP_E_ARG, "tau");
  const int A = a.n_turn * a.n_acc * a.n_climb;
  const int n_hp = a.n_turn * a.n_acc;                       // horizontal paths (turn, acceleration)
  const int hpt = wide ? std::min(fmdp::WIDE_HPT, n_hp) : a.n_turn;  // paths per cluster tile
  if ((wide ? hpt * a.n_climb : A) * a.window > fmdp::MAX_AW) return bad(FMDP_E_ARG, "A*W too large");
  int64_t step_u;
  if (!integral(a.speed * a.dt / a.u_m, &step_u) || step_u <= 0 || step_u > 1000) return bad(FMDP_E_ARG, "speed");
  for (int i = 0; i < a.n_climb; ++i)
    if (std::abs(a.climb_units[i]) > 100) return bad(FMDP_E_ARG, "climb rate");
  int64_t zdeck, capu, sepu;
  if (!integral(a.deck_alt_m / a.u_m, &zdeck) || !integral(a.capture_radius_m / a.u_m, &capu) ||
      !integral(a.sep_min_m / a.u_m, &sepu) || capu <= 0 || sepu <= 0)
    return bad(FMDP_E_ARG, "deck/capture/sep must be multiples of u");
  if (a.horizon_steps < 4 || a.row_capacity < 4 || a.row_capacity % 4) return bad(FMDP_E_ARG, "store geometry");
  if (a.max_steps < 1) return bad(FMDP_E_ARG, "max_steps");
  if (a.valuation != 0 && a.valuation != 1) return bad(FMDP_E_ARG, "valuation must be 0 (Alg 8) or 1 (Alg 1)");

  ctx->air = a;
  ctx->turn.assign(a.turn_steps, a.turn_steps + a.n_turn);
  ctx->climb.assign(a.climb_units, a.climb_units + a.n_climb);
  ctx->tau_s.assign(a.tau_s, a.tau_s + a.n_tau);
  ctx->tau_r.assign(a.tau_radius_m, a.tau_radius_m + a.n_tau);
  ctx->air.turn_steps = ctx->turn.data();
  ctx->air.climb_units = ctx->climb.data();
  ctx->air.tau_s = ctx->tau_s.data();
  ctx->air.tau_radius_m = ctx->tau_r.data();
  ctx->A = A;
  ctx->W = a.window;
  ctx->C = a.n_climb;
  ctx->wide = wide;
  ctx->acc.assign(a.acc_units, a.acc_units + a.n_acc);
  ctx->air.acc_units = ctx->acc.data();
  ctx->wide_k = wide ? (n_hp + hpt - 1) / hpt : 0;
  const double lo[3] = {a.lo.x, a.lo.y, a.lo.z}, hi[3] = {a.hi.x, a.hi.y, a.hi.z};
  for (int d = 0; d < 3; ++d) {
    ctx->lo_u[d] = std::llrint(lo[d] / a.u_m);
    ctx->hi_u[d] = std::llrint(hi[d] / a.u_m);
    if (ctx->hi_u[d] <= ctx->lo_u[d] || ctx->hi_u[d] - ctx->lo_u[d] >= (1LL << 24))
      return bad(FMDP_E_RANGE, "airspace span must be positive and < 2^24 units");
  }

  // device
  int dev = devs ? devs->device : -1;
  if (dev < 0 && cudaGetDevice(&dev) != cudaSuccess) return bad(FMDP_E_NODEV, "no CUDA device");
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) {
    cudaGetLastError();
    return bad(FMDP_E_NODEV, "no CUDA device");
  }
  if (prop.major != 10) return bad(FMDP_E_NODEV, "libfmdp is built for sm_100a only");
  DevGuard dev_guard(dev);  // the caller's current device is restored on return
  {
    int cur = -1;
    if (cudaGetDevice(&cur) != cudaSuccess || cur != dev) return bad(FMDP_E_NODEV, "cudaSetDevice failed");
  }
  ctx->device = dev;
  ctx->num_sms = prop.multiProcessorCount;
  if (devs) {
    ctx->alloc = devs->alloc;
    ctx->release = devs->release;
    ctx->user = devs->user;
    ctx->stream = (cudaStream_t)devs->stream;
  }
  if (!ctx->stream) {
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess)
      return bad(FMDP_E_CUDA, "stream");
    ctx->own_stream = true;
  }
  cudaEventCreate(&ctx->ev0);
  cudaEventCreate(&ctx->ev1);
  cudaEventCreate(&ctx->ev2);
  cudaEventCreate(&ctx->ev3);
  if (cudaStreamCreateWithFlags(&ctx->stream2, cudaStreamNonBlocking) != cudaSuccess) return bad(FMDP_E_CUDA, "stream");
  if (cudaStreamCreateWithFlags(&ctx->stream3, cudaStreamNonBlocking) != cudaSuccess) return bad(FMDP_E_CUDA, "stream");

  World& w = ctx->w;
  std::memset(&w, 0, sizeof(w));
  w.A = wide ? hpt * a.n_climb : A;  // wide: one cluster tile
  w.W = a.window;
  w.n_turn = hpt;  // = n_turn without acceleration actions (one tile = every path)
  w.n_turn_all = a.n_turn;
  w.wide = wide ? 1 : 0;
  w.A_all = A;
  w.n_hp = n_hp;
  w.hpt = hpt;
  w.n_acc = a.n_acc;
  for (int i = 0; i < a.n_acc; ++i) w.acc[i] = a.acc_units[i];
  w.n_climb = a.n_climb;
  w.HL = a.heading_lattice;
  for (int i = 0; i < a.n_turn; ++i) w.turn[i] = a.turn_steps[i];
  for (int i = 0; i < a.n_climb; ++i) w.climb[i] = a.climb_units[i];
  w.zero_climb = -1;
  for (int i = 0; i < a.n_climb; ++i)
    if (a.climb_units[i] == 0) w.zero_climb = i;
  int64_t Rmax = 0;
  for (int i = 0; i < fmdp::NTAU; ++i) {
    if (i < a.n_tau) {
      int64_t k, R;
      if (!integral(a.tau_s[i] / a.dt, &k) || !integral(a.tau_radius_m[i] / a.u_m, &R) || R <= 0)
        return bad(FMDP_E_ARG, "tau/dt and radii/u must be integral");
      w.k_tau[i] = (int32_t)k;
      w.R2_tau[i] = R * R;  // FP32 band R2lo/R2hi: set below from the hot loop's error bound
      Rmax = std::max(Rmax, R);
    } else {
      w.k_tau[i] = 0;
      w.R2_tau[i] = 0;
    }
  }
  if (Rmax >= 32768) return bad(FMDP_E_ARG, "well radius must be < 2^15 units");
  if (sepu >= Rmax) return bad(FMDP_E_ARG, "separation minimum must be below the largest well radius");
  w.R_max = (int32_t)Rmax;
  w.sat_d2 = (uint32_t)(Rmax * Rmax);
  w.sep2 = (uint32_t)(sepu * sepu);
  w.cap2 = capu * capu;
  w.goal_r = std::fabs(a.goal_r);
  w.goal_l2g = std::log2(a.goal_gamma) * a.u_m;
  w.goal_rf = (float)w.goal_r;
  w.goal_l2gf = (float)w.goal_l2g;
  w.intr_r = (float)std::fabs(a.intr_r);
  w.intr_l2g = (float)(std::log2(a.intr_gamma) * a.u_m);
  w.terr_r = (float)std::fabs(a.terr_r);
  w.terr_l2g = (float)(std::log2(a.terr_gamma) * a.u_m);
  w.zdeck_u = (int32_t)zdeck;
  w.deck_scale = a.deck_scale;
  w.u_m = a.u_m;
  w.max_steps = a.max_steps;
  w.vmax_init_zero = a.vmax_init_zero;
  w.endpoint = a.valuation == 1 ? 1 : 0;
  w.near_tie_rel = a.near_tie_rel;
  w.horizon = a.horizon_steps;
  w.row_cap = a.row_capacity;

  std::vector<int2> lat;
  build_lattice(w.HL, step_u, lat);
  double maxd = 0;
  for (const int2& d : lat) maxd = std::max(maxd, std::sqrt((double)d.x * d.x + (double)d.y * d.y));
  // acceleration actions (R32): speeds [vmin, vmax] units per substep; D(psi, v) = the lattice of
  // step length v -- one table row per speed (at v = v0 the constant-speed lattice)
  std::vector<int2> spd;
  w.v0 = (int32_t)step_u;
  w.vmin = w.vmax = (int32_t)step_u;
  if (wide) {
    int64_t vmin = step_u, vmax = step_u;
    if (a.speed_min > 0 || a.speed_max > 0) {
      if (!integral(a.speed_min * a.dt / a.u_m, &vmin) || !integral(a.speed_max * a.dt / a.u_m, &vmax) || vmin < 1 ||
          vmin > step_u || step_u > vmax || vmax > 1000)
        return bad(FMDP_E_ARG, "speed_min <= speed <= speed_max, multiples of u per dt, <= 1000 units per substep");
    }
    w.vmin = (int32_t)vmin;
    w.vmax = (int32_t)vmax;
    spd.resize((size_t)(vmax - vmin + 1) * w.HL);
    std::vector<int2> row;
    for (int64_t sp = vmin; sp <= vmax; ++sp) {
      build_lattice(w.HL, sp, row);
      std::copy(row.begin(), row.end(), spd.begin() + (size_t)(sp - vmin) * w.HL);
      for (const int2& d : row) maxd = std::max(maxd, std::sqrt((double)d.x * d.x + (double)d.y * d.y));
    }
  }
  int maxc = 0;
  for (int c : ctx->climb) maxc = std::max(maxc, std::abs(c));
  w.reach_u = (int32_t)(a.window * ((int64_t)std::ceil(maxd) + maxc) + 1);
  w.step_reach_u = (int32_t)((int64_t)std::ceil(maxd) + maxc + 1);
  // f1 cull radius: the culled walker pre-culls a step's plans against the previous step's q, so
  // the reach grows by one step: |s_{k+1} - q_k| <= reach + step_reach
  w.cull_inf = (int32_t)(Rmax + w.reach_u + w.step_reach_u + 1);
  // Hot-loop filter band.  The kernel evaluates e = Q + 2(s-o).X, X = o - c,
  // Q = fl(|X|^2), with s - o bounded by S (the fan radius around o = q + (W/2)(DX,DY)[psi],
  // measured here over every heading, turn and substep, plus the climb).  First-order
  // rounding error of the computed d^2 = e + |s-o|^2 for d <= R(1 + band):
  //   u [3 (R+S)^2 + 2((R+S)^2 + 2S(R+S)) + 2R^2 + S^2],  u = 2^-24;
  // the band is 1.5x that, relative to R^2, and never below 2^-20.
  {
    int64_t s2max = 0;
    const int half = a.window / 2;
    for (int psi = 0; psi < w.HL; ++psi) {
      const int64_t ox = (int64_t)half * lat[psi].x, oy = (int64_t)half * lat[psi].y;
      for (int it = 0; it < a.n_turn; ++it) {
        int64_t x = 0, y = 0;
        int ps = psi;
        for (int t = 1; t <= a.window; ++t) {
          ps = ((ps + a.turn_steps[it]) % w.HL + w.HL) % w.HL;
          x += lat[ps].x;
          y += lat[ps].y;
          s2max = std::max(s2max, (x - ox) * (x - ox) + (y - oy) * (y - oy));
        }
      }
    }
    double S = std::sqrt((double)s2max) + (double)a.window * maxc + 1.0;
    if (wide)  // any speed profile: |s - o| <= |s - q| + |o - q| <= W max|D| + (W/2) |D(., v0)|
      S = (double)a.window * (std::ceil(maxd) + maxc) + (double)(a.window / 2) * (double)(step_u + 1) + 1.0;
    ctx->fan_radius_u = S;
    for (int i = 0; i < a.n_tau; ++i) {
      const double R = std::sqrt((double)w.R2_tau[i]);
      const double err = 3 * (R + S) * (R + S) + 2 * ((R + S) * (R + S) + 2 * S * (R + S)) + 2 * R * R + S * S;
      const double band = std::max(std::ldexp(1.0, -20), 1.5 * std::ldexp(err / (R * R), -24));
      w.R2lo[i] = (float)((R * R) * (1.0 - band));
      w.R2hi[i] = (float)((R * R) * (1.0 + band));
      ctx->band_rel[i] = band;
    }
    for (int i = a.n_tau; i < fmdp::NTAU; ++i) {
      w.R2lo[i] = -1.f;
      w.R2hi[i] = -1.f;
    }
  }
  w.k_absmax = 0;
  for (int i = 0; i < a.n_tau; ++i) w.k_absmax = std::max(w.k_absmax, std::abs(w.k_tau[i]));
  for (int i = 0; i < fmdp::NTAU; ++i) {
    const double rc = i < a.n_tau ? std::sqrt((double)w.R2_tau[i]) + w.reach_u + w.step_reach_u + 1.0 : -1.0;
    w.cull2f_tau[i] = i < a.n_tau ? (float)(rc * rc * (1.0 + std::ldexp(1.0, -16))) : -1.0f;
  }
  ctx->iw.n_tau = a.n_tau;
  for (int i = 0; i < a.n_tau; ++i) {
    const int64_t R = std::llround(std::sqrt((double)w.R2_tau[i])) + w.reach_u + 1;
    ctx->iw.k_tau[i] = w.k_tau[i];
    ctx->iw.r2[i] = R * R;
  }
  ctx->iw.sat2 = Rmax * Rmax;

  // device memory
  const size_t row_words = (size_t)4 * w.row_cap;
  ctx->d_rows = (int32_t*)dalloc(ctx, sizeof(int32_t) * row_words * (size_t)w.horizon);
  ctx->d_counts = (int32_t*)dalloc(ctx, sizeof(int32_t) * (size_t)w.horizon);
  ctx->d_dxy = (int2*)dalloc(ctx, sizeof(int2) * w.HL);
  const size_t nproj = (size_t)w.HL * w.n_turn * a.window;  // (wide walkers use d_spd instead)
  ctx->d_proj = (int2*)dalloc(ctx, sizeof(int2) * nproj);
  ctx->d_queue = (int32_t*)dalloc(ctx, sizeof(int32_t) * 4);
  ctx->d_stop = ctx->d_queue ? ctx->d_queue + 2 : nullptr;
  ctx->d_pairctr = (unsigned long long*)dalloc(ctx, sizeof(unsigned long long));
  ctx->d_prof = (unsigned long long*)dalloc(ctx, sizeof(unsigned long long) * fmdp::N_PHASES);
  ctx->d_dbg_vstar = (double*)dalloc(ctx, sizeof(double) * A);
  ctx->d_dbg_v = (double*)dalloc(ctx, sizeof(double) * A * a.window);
  ctx->d_dbg_s = (double*)dalloc(ctx, sizeof(double) * A * a.window);
  ctx->d_dbg_conf = (uint32_t*)dalloc(ctx, sizeof(uint32_t) * (A + 1));
  ctx->d_dbg_astar = (int32_t*)dalloc(ctx, sizeof(int32_t) * 4);
  ctx->d_xbuf = (uint32_t*)dalloc(ctx, sizeof(uint32_t) * ((size_t)A * a.window * fmdp::NTAU + 1));
  if (!ctx->d_rows || !ctx->d_counts || !ctx->d_dxy || !ctx->d_proj || !ctx->d_queue || !ctx->d_pairctr || !ctx->d_prof || !ctx->d_dbg_vstar ||
      !ctx->d_dbg_v || !ctx->d_dbg_s || !ctx->d_dbg_conf || !ctx->d_dbg_astar || !ctx->d_xbuf) {
    return bad(FMDP_E_NOMEM, "device allocation failed");
  }
  cudaMemset(ctx->d_rows, 0, sizeof(int32_t) * row_words * (size_t)w.horizon);
  cudaMemset(ctx->d_counts, 0, sizeof(int32_t) * (size_t)w.horizon);
  cudaMemcpy(ctx->d_dxy, lat.data(), sizeof(int2) * w.HL, cudaMemcpyHostToDevice);
  {  // Alg 3 projection offsets of every (heading, turn, substep): integer sums of lattice steps
    std::vector<int2> proj(nproj);
    for (int psi = 0; psi < w.HL; ++psi)
      for (int it = 0; it < (wide ? 0 : a.n_turn); ++it) {
        int x = 0, y = 0, ps = psi;
        for (int t = 1; t <= a.window; ++t) {
          ps = ((ps + a.turn_steps[it]) % w.HL + w.HL) % w.HL;
          x += lat[ps].x;
          y += lat[ps].y;
          proj[((size_t)psi * a.n_turn + it) * a.window + (t - 1)] = make_int2(x, y);
        }
      }
    cudaMemcpy(ctx->d_proj, proj.data(), sizeof(int2) * nproj, cudaMemcpyHostToDevice);
  }
  w.proj = ctx->d_proj;
  if (wide) {  // (speed, heading) table; decision board and per-cluster queues of the wide walker
    ctx->d_spd = (int2*)dalloc(ctx, sizeof(int2) * spd.size());
    ctx->d_wb = (unsigned long long*)dalloc(ctx, sizeof(unsigned long long) * 2 * fmdp::WB_WORDS * ctx->wide_k);
    ctx->d_wq = (int32_t*)dalloc(ctx, sizeof(int32_t) * (fmdp::XMAX * 4 + 4));
    if (!ctx->d_spd || !ctx->d_wb || !ctx->d_wq || ctx->wide_k > fmdp::XMAX * 4)
      return bad(FMDP_E_NOMEM, "device allocation failed (wide walker)");
    cudaMemcpy(ctx->d_spd, spd.data(), sizeof(int2) * spd.size(), cudaMemcpyHostToDevice);
    w.spd = ctx->d_spd;
  }
  ctx->counts.assign((size_t)w.horizon, 0);
  w.rows = ctx->d_rows;
  w.counts = ctx->d_counts;
  w.dxy = ctx->d_dxy;

  if (ter && ter->n_wells > 0) {
    if (!ter->center || !ter->radius_u) {
      return bad(FMDP_E_ARG, "terrain arrays missing");
    }
    std::vector<int4> tw(ter->n_wells);
    for (int i = 0; i < ter->n_wells; ++i)
      tw[i] = make_int4(ter->center[i].x, ter->center[i].y, ter->center[i].z, ter->radius_u[i]);
    ctx->d_tw = (int4*)dalloc(ctx, sizeof(int4) * tw.size());
    if (!ctx->d_tw) {
      return bad(FMDP_E_NOMEM, "device allocation failed");
    }
    cudaMemcpy(ctx->d_tw, tw.data(), sizeof(int4) * tw.size(), cudaMemcpyHostToDevice);
    w.n_tw = ter->n_wells;
    w.tw = ctx->d_tw;
  }
  if (ter && ter->nx > 0 && ter->ny > 0) {
    if (!ter->height_u || ter->cell_u <= 0) {
      return bad(FMDP_E_ARG, "terrain arrays missing");
    }
    const size_t nh = (size_t)ter->nx * ter->ny;
    ctx->d_height = (int32_t*)dalloc(ctx, sizeof(int32_t) * nh);
    if (!ctx->d_height) {
      return bad(FMDP_E_NOMEM, "device allocation failed");
    }
    cudaMemcpy(ctx->d_height, ter->height_u, sizeof(int32_t) * nh, cudaMemcpyHostToDevice);
    w.nx = ter->nx;
    w.ny = ter->ny;
    w.x0 = ter->x0_u;
    w.y0 = ter->y0_u;
    w.cell = ter->cell_u;
    w.cell_magic = ((1ULL << 40) + (uint64_t)ter->cell_u - 1) / (uint64_t)ter->cell_u;
    w.height = ctx->d_height;
  }
  ctx->cap_states = a.max_steps + 2;
  if (threads_for(ctx) > (ctx->C == 1 ? 512 : 384) ||
      fmdp::walk_smem_bytes(w, ctx->C, threads_for(ctx), kChunk, kChunk, wide ? fmdp::WIDE_G : 16) > 227 * 1024)
    return bad(FMDP_E_ARG, "action lattice too large for one CTA (threads / shared memory)");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return bad(FMDP_E_CUDA, cudaGetErrorString(e));
  *out = ctx;
  return FMDP_OK;
}

void fmdp_destroy(fmdp_ctx* ctx) {
  if (!ctx) return;
  DevGuard dev_guard(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  x_release(ctx);
  std::vector<void*> a = ctx->allocs;
  for (void* p : a) dfree(ctx, p);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->h_pack) cudaFreeHost(ctx->h_pack);
  if (ctx->ev2) cudaEventDestroy(ctx->ev2);
  if (ctx->stream2) cudaStreamDestroy(ctx->stream2);
  if (ctx->ev3) cudaEventDestroy(ctx->ev3);
  if (ctx->stream3) cudaStreamDestroy(ctx->stream3);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
}

fmdp_status fmdp_set_launch(fmdp_ctx* ctx, const fmdp_launch* l) {
  if (!ctx) return FMDP_E_ARG;
  fmdp_launch n{};
  if (l) n = *l;
  if (n.cluster_size < 0 || n.cluster_size > 16 || (n.cluster_size & (n.cluster_size - 1)))
    return fail(ctx, FMDP_E_ARG, "cluster_size must be 0 or a power of two <= 16");
  if (n.threads && (n.threads < 32 || n.threads > (ctx->C == 1 ? 512 : 384)))
    return fail(ctx, FMDP_E_ARG, "threads: 0 (auto) or a cap in [32, 384] (512 with one climb)");
  const fmdp_launch prev = ctx->launch;
  ctx->launch = n;
  if (threads_for(ctx) < 32) {
    ctx->launch = prev;
    return fail(ctx, FMDP_E_ARG, "threads cap below one warp of columns");
  }
  std::memset(ctx->mc_cache, 0, sizeof(ctx->mc_cache));
  std::memset(ctx->mc_cache_cs, 0, sizeof(ctx->mc_cache_cs));
  if (fmdp::walk_smem_bytes(ctx->w, ctx->C, threads_for(ctx), chunk_for(ctx), rawcap_for(ctx), 16) > 227 * 1024)
    return fail(ctx, FMDP_E_ARG, "shared memory");
  return FMDP_OK;
}

fmdp_status fmdp_add_plans(fmdp_ctx* ctx, int32_t n_plans, const uint64_t* aircraft_ids, const int64_t* t0_steps,
                           const int32_t* n_states, const fmdp_qpos* states, uint32_t* first_id) {
  if (!ctx || n_plans < 0 || (n_plans > 0 && (!t0_steps || !n_states || !states)))
    return fail(ctx, FMDP_E_ARG, "null argument");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  if (first_id) *first_id = (uint32_t)ctx->plans.size();
  if (n_plans == 0) return FMDP_OK;
  std::vector<int64_t> t0(n_plans);
  std::vector<int32_t> n(n_plans);
  size_t tot = 0;
  const int64_t margin = 1LL << 20;
  for (int i = 0; i < n_plans; ++i) {
    t0[i] = t0_steps[i];
    n[i] = n_states[i];
    if (n[i] < 1) return fail(ctx, FMDP_E_ARG, "plan with no states");
    if (t0[i] < 0 || t0[i] + n[i] > ctx->w.horizon) return fail(ctx, FMDP_E_RANGE, "plan rows outside horizon");
    const fmdp_qpos* s = states + tot;
    for (int k = 0; k < n[i]; ++k) {
      const int32_t p[3] = {s[k].x, s[k].y, s[k].z};
      for (int d = 0; d < 3; ++d)
        if (p[d] < ctx->lo_u[d] - margin || p[d] > ctx->hi_u[d] + margin)
          return fail(ctx, FMDP_E_RANGE, "plan state far outside the airspace");
      if (k + 1 < n[i]) {
        const int64_t vx = (int64_t)s[k + 1].x - s[k].x, vy = (int64_t)s[k + 1].y - s[k].y,
                      vz = (int64_t)s[k + 1].z - s[k].z;
        if (vx < -1024 || vx > 1023 || vy < -1024 || vy > 1023 || vz < -512 || vz > 511)
          return fail(ctx, FMDP_E_RANGE, "plan velocity beyond the packed store record");
      }
    }
    tot += n[i];
  }
  if (!rows_fit(ctx, t0, n)) return fail(ctx, FMDP_E_CAPACITY, "time row capacity exceeded");
  // upload in chunks of whole plans
  const size_t kMaxWords = (size_t)48 << 20;
  size_t off = 0;
  int p0 = 0;
  while (p0 < n_plans) {
    size_t words = 0;
    int p1 = p0;
    while (p1 < n_plans && (p1 == p0 || words + 3 * (size_t)n[p1] <= kMaxWords)) words += 3 * (size_t)n[p1++];
    fmdp_status st = ensure_up(ctx, words + (words / 3));
    if (st) return st;
    // states first, then slots (append_device writes slots at d_up, so place states after)
    int32_t* d_states = nullptr;
    {
      // reserve: slots [0, words/3), states [words/3, words/3 + words)
      d_states = ctx->d_up + words / 3;
      CK(cudaMemcpyAsync(d_states, states + off, sizeof(int32_t) * words, cudaMemcpyHostToDevice, ctx->stream));
    }
    std::vector<int64_t> ct0(t0.begin() + p0, t0.begin() + p1);
    std::vector<int32_t> cn(n.begin() + p0, n.begin() + p1);
    std::vector<const int32_t*> ds;
    size_t o = 0;
    for (int i = p0; i < p1; ++i) {
      ds.push_back(d_states + o);
      o += 3 * (size_t)n[i];
    }
    st = append_device(ctx, ct0, cn, ds);
    if (st) return st;
    for (int i = p0; i < p1; ++i) {
      PlanRec r;
      r.aircraft = aircraft_ids ? aircraft_ids[i] : 0;
      r.t0 = t0[i];
      const int32_t* src = reinterpret_cast<const int32_t*>(states + off);
      r.states.assign(src, src + 3 * (size_t)n[i]);
      off += n[i];
      ctx->plans.push_back(std::move(r));
    }
    p0 = p1;
  }
  ctx->index_dirty = true;  // the range-query index is rebuilt before the next culled walk
  return FMDP_OK;
}

fmdp_status fmdp_add_plan(fmdp_ctx* ctx, uint64_t aircraft_id, int64_t t0_step, int32_t n, const fmdp_qpos* states,
                          int32_t flags, uint32_t* plan_id) {
  (void)flags;
  return fmdp_add_plans(ctx, 1, &aircraft_id, &t0_step, &n, states, plan_id);
}

fmdp_status fmdp_schedule(fmdp_ctx* ctx, uint64_t aircraft_id, fmdp_vec3 src, fmdp_vec3 dst, int64_t t0_step,
                          fmdp_result* res, fmdp_qpos* traj, int32_t traj_cap) {
  fmdp_request r;
  r.aircraft_id = aircraft_id;
  r.src = src;
  r.dst = dst;
  r.t0_step = t0_step;
  return schedule_many(ctx, &r, 1, res, traj, traj_cap, FMDP_BATCH_SEQUENTIAL);
}

// Result of a single-request walk (sharded paths): commit if accepted, fill res, copy traj.
fmdp_status finish_single(fmdp_ctx* ctx, const std::vector<Req>& base, uint64_t aircraft_id, fmdp_result* res,
                          fmdp_qpos* traj) {
  fmdp_status st = FMDP_OK;
  const Out& o = ctx->h_out[0];
  std::vector<uint32_t> plan_id(1, 0xffffffffu);
  std::vector<uint64_t> aircraft(1, aircraft_id);
  if (o.status == FMDP_ACCEPTED && (st = commit_slots(ctx, {0}, base, aircraft, plan_id))) return st;
  res->status = o.status;
  res->plan_id = plan_id[0];
  res->n_states = o.n_states;
  res->fail_step = o.fail_step;
  res->min_sep_m = std::sqrt((double)o.min_sep_d2) * ctx->air.u_m;
  res->n_near_ties = o.n_near_ties;
  res->n_exact = o.n_exact;
  if (traj) {
    CK(cudaMemcpy(traj, ctx->d_traj, sizeof(fmdp_qpos) * o.n_states, cudaMemcpyDeviceToHost));
  }
  unsigned long long pc = 0;
  CK(cudaMemcpy(&pc, ctx->d_pairctr, sizeof(pc), cudaMemcpyDeviceToHost));
  ctx->stats.pair_evals = (int64_t)pc;
  ctx->last_n = 1;
  return FMDP_OK;
}

fmdp_status fmdp_schedule_sharded(fmdp_ctx* ctx, const fmdp_shard* shard, uint64_t aircraft_id, fmdp_vec3 src,
                                  fmdp_vec3 dst, int64_t t0_step, fmdp_result* res, fmdp_qpos* traj,
                                  int32_t traj_cap) {
  if (ctx && ctx->wide) return fail(ctx, FMDP_E_ARG, "not available with acceleration actions (wide walker)");
  if (!ctx || !shard || !res || !shard->allreduce_min_u32 || shard->world < 1 || shard->rank < 0 ||
      shard->rank >= shard->world)
    return fail(ctx, FMDP_E_ARG, "invalid shard description");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  {
    const fmdp_status e = ensure_index(ctx, true);
    if (e) return e;
  }
  if (traj && traj_cap < ctx->w.max_steps + 1) return fail(ctx, FMDP_E_BUFFER, "traj_cap must be >= max_steps + 1");
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  fmdp_request rq;
  rq.aircraft_id = aircraft_id;
  rq.src = src;
  rq.dst = dst;
  rq.t0_step = t0_step;
  std::vector<Req> base;
  fmdp_status st = prepare_requests(ctx, &rq, 1, base);
  if (st) return st;
  if ((st = ensure_slots(ctx, 1))) return st;
  CK(cudaMemsetAsync(ctx->d_pairctr, 0, sizeof(unsigned long long), ctx->stream));
  const int nx = ctx->A * ctx->W * fmdp::NTAU + 1;
  std::vector<uint32_t> hbuf(nx);
  ctx->shard_rank = shard->rank;
  ctx->shard_world = shard->world;
  int k = 0;
  for (;;) {
    Req r = base[0];
    r.start_k = k;
    ctx->xmode = 1;  // this GPU's minima over its plan shard
    st = run_walk(ctx, {r}, false, 1);
    if (!st) {
      CK(cudaMemcpyAsync(hbuf.data(), ctx->d_xbuf, sizeof(uint32_t) * nx, cudaMemcpyDeviceToHost, ctx->stream));
      CK(cudaStreamSynchronize(ctx->stream));
      if (shard->allreduce_min_u32(hbuf.data(), nx, shard->user) != 0) st = fail(ctx, FMDP_E_INTERNAL, "allreduce failed");
    }
    if (!st) {
      CK(cudaMemcpyAsync(ctx->d_xbuf, hbuf.data(), sizeof(uint32_t) * nx, cudaMemcpyHostToDevice, ctx->stream));
      ctx->xmode = 2;  // all-reduced minima -> identical decision on every GPU
      st = run_walk(ctx, {r}, false, 1);
    }
    ctx->xmode = 0;
    if (!st) st = fetch_out(ctx, 1);
    if (st) {
      ctx->shard_rank = 0;
      ctx->shard_world = 1;
      return st;
    }
    ctx->stats.steps += ctx->h_out[0].steps_run;
    ctx->stats.rounds += 1;
    if (ctx->h_out[0].status >= 0) break;
    k = ctx->h_out[0].n_states - 1;
  }
  ctx->shard_rank = 0;
  ctx->shard_world = 1;
  return finish_single(ctx, base, aircraft_id, res, traj);
}

// ----------------------------------------------------------------------------- in-kernel exchange
fmdp_status fmdp_p2p_export(fmdp_ctx* ctx, int32_t world, fmdp_p2p_handle* handle, void** dev_ptr) {
  if (ctx && ctx->wide) return fail(ctx, FMDP_E_ARG, "not available with acceleration actions (wide walker)");
  if (!ctx || !handle || world < 1 || world > fmdp::XNODE) return fail(ctx, FMDP_E_ARG, "world must be 1..8");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  CK(cudaStreamSynchronize(ctx->stream));
  x_release(ctx);
  if (!ctx->d_xpeers) ctx->d_xpeers = (fmdp::XPeer*)dalloc(ctx, sizeof(fmdp::XPeer) * fmdp::XMAX);
  if (!ctx->d_xseq) ctx->d_xseq = (unsigned long long*)dalloc(ctx, 2 * sizeof(unsigned long long));  // seq, error
  if (!ctx->d_xpeers || !ctx->d_xseq) return fail(ctx, FMDP_E_NOMEM, "exchange tables");
  const int slot = ((ctx->A * ctx->W * fmdp::NTAU + 16) + 3) & ~3;
  const size_t bytes = fmdp::x_area_bytes(world, slot) * fmdp::XMAX;  // one area per cluster index
  if (cudaMalloc(&ctx->x_area, bytes) != cudaSuccess) {
    cudaGetLastError();
    ctx->x_area = nullptr;
    return fail(ctx, FMDP_E_NOMEM, "exchange area");
  }
  CK(cudaMemset(ctx->x_area, 0, bytes));
  ctx->x_world = world;
  ctx->x_slot = slot;
  static_assert(sizeof(cudaIpcMemHandle_t) == sizeof(handle->bytes), "IPC handle size");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, ctx->x_area) == cudaSuccess) {
    std::memcpy(handle->bytes, &h, sizeof(h));
  } else {  // no IPC here: in-process peers (dev_ptrs) still work
    cudaGetLastError();
    std::memset(handle->bytes, 0, sizeof(handle->bytes));
  }
  if (dev_ptr) *dev_ptr = ctx->x_area;
  return FMDP_OK;
}

fmdp_status fmdp_p2p_connect(fmdp_ctx* ctx, int32_t rank, int32_t world, const fmdp_p2p_handle* handles,
                             void* const* dev_ptrs) {
  if (!ctx) return FMDP_E_ARG;
  if (!ctx->x_area || world != ctx->x_world) return fail(ctx, FMDP_E_ARG, "fmdp_p2p_export(world) first");
  if (rank < 0 || rank >= world) return fail(ctx, FMDP_E_ARG, "rank out of range");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  for (void* p : ctx->x_ipc) cudaIpcCloseMemHandle(p);
  ctx->x_ipc.clear();
  ctx->x_me = -1;
  std::vector<fmdp::XPeer> tab(fmdp::XMAX, fmdp::XPeer{nullptr});
  std::vector<fmdp::XPeer> itab((size_t)fmdp::XMAX * fmdp::XNODE, fmdp::XPeer{nullptr});
  const size_t hwords = fmdp::x_area_bytes(fmdp::XMAX, ctx->x_slot) / sizeof(unsigned long long);
  if (!ctx->d_ipeers) ctx->d_ipeers = (fmdp::XPeer*)dalloc(ctx, sizeof(fmdp::XPeer) * itab.size());
  if (!ctx->d_xh_area) ctx->d_xh_area = (unsigned long long*)dalloc(ctx, sizeof(unsigned long long) * hwords * fmdp::XMAX);
  if (!ctx->d_xh_peers) ctx->d_xh_peers = (fmdp::XPeer*)dalloc(ctx, sizeof(fmdp::XPeer) * fmdp::XMAX);
  if (!ctx->d_xh_seq)
    ctx->d_xh_seq = (unsigned long long*)dalloc(ctx, sizeof(unsigned long long) * (2 * fmdp::XMAX + 1));
  if (!ctx->d_ipeers || !ctx->d_xh_area || !ctx->d_xh_peers || !ctx->d_xh_seq)
    return fail(ctx, FMDP_E_NOMEM, "exchange tables");
  for (int q = 0; q < world; ++q) {
    void* base = nullptr;
    if (q == rank) {
      base = ctx->x_area;
    } else if (dev_ptrs && dev_ptrs[q]) {
      base = dev_ptrs[q];
      cudaPointerAttributes at{};
      CK(cudaPointerGetAttributes(&at, base));
      if (at.device != ctx->device) {
        int ok = 0;
        CK(cudaDeviceCanAccessPeer(&ok, ctx->device, at.device));
        if (!ok) return fail(ctx, FMDP_E_CUDA, "no peer access between the devices");
        const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
          return fail(ctx, FMDP_E_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
        cudaGetLastError();
      }
    } else {
      if (!handles) return fail(ctx, FMDP_E_ARG, "peer handle missing");
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles[q].bytes, sizeof(h));
      CK(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
      ctx->x_ipc.push_back(base);
    }
    tab[q].recv = reinterpret_cast<unsigned long long*>(base);
    for (int c = 0; c < fmdp::XMAX; ++c)  // cluster c's area on GPU q
      itab[(size_t)c * fmdp::XNODE + q].recv =
          reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(base) + c * fmdp::x_area_bytes(world, ctx->x_slot));
  }
  CK(cudaMemcpy(ctx->d_xpeers, tab.data(), sizeof(fmdp::XPeer) * fmdp::XMAX, cudaMemcpyHostToDevice));
  CK(cudaMemset(ctx->d_xseq, 0, 2 * sizeof(unsigned long long)));
  CK(cudaMemset(ctx->x_area, 0, fmdp::x_area_bytes(world, ctx->x_slot) * fmdp::XMAX));  // tags restart
  CK(cudaMemcpy(ctx->d_ipeers, itab.data(), sizeof(fmdp::XPeer) * itab.size(), cudaMemcpyHostToDevice));
  {  // this GPU's level: cluster q's area
    std::vector<fmdp::XPeer> htab(fmdp::XMAX, fmdp::XPeer{nullptr});
    for (int q = 0; q < fmdp::XMAX; ++q) htab[q].recv = ctx->d_xh_area + (size_t)q * hwords;
    CK(cudaMemcpy(ctx->d_xh_peers, htab.data(), sizeof(fmdp::XPeer) * fmdp::XMAX, cudaMemcpyHostToDevice));
  }
  CK(cudaMemset(ctx->d_xh_area, 0, sizeof(unsigned long long) * hwords * fmdp::XMAX));
  CK(cudaMemset(ctx->d_xh_seq, 0, sizeof(unsigned long long) * (2 * fmdp::XMAX + 1)));
  ctx->xh_seq = 0;
  CK(cudaDeviceSynchronize());
  ctx->x_me = rank;
  return FMDP_OK;
}

fmdp_status fmdp_schedule_p2p(fmdp_ctx* ctx, uint64_t aircraft_id, fmdp_vec3 src, fmdp_vec3 dst, int64_t t0_step,
                              fmdp_result* res, fmdp_qpos* traj, int32_t traj_cap) {
  if (ctx && ctx->wide) return fail(ctx, FMDP_E_ARG, "not available with acceleration actions (wide walker)");
  if (!ctx || !res) return fail(ctx, FMDP_E_ARG, "null argument");
  if (ctx->x_me < 0) return fail(ctx, FMDP_E_ARG, "fmdp_p2p_connect first");
  if (traj && traj_cap < ctx->w.max_steps + 1) return fail(ctx, FMDP_E_BUFFER, "traj_cap must be >= max_steps + 1");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  {
    const fmdp_status e = ensure_index(ctx, true);
    if (e) return e;
  }
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  fmdp_request rq;
  rq.aircraft_id = aircraft_id;
  rq.src = src;
  rq.dst = dst;
  rq.t0_step = t0_step;
  std::vector<Req> base;
  fmdp_status st = prepare_requests(ctx, &rq, 1, base);
  if (st) return st;
  if ((st = ensure_slots(ctx, 1))) return st;
  CK(cudaMemsetAsync(ctx->d_pairctr, 0, sizeof(unsigned long long), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_prof, 0, sizeof(unsigned long long) * fmdp::N_PHASES, ctx->stream));
  // two-level exchange: k clusters on every GPU (the split cost model on this GPU's shard; the
  // same k on every rank: identical stores, settings and devices), cluster c of each GPU
  // exchanging with cluster c of every other GPU
  const int N = ctx->x_world, me = ctx->x_me;
  ctx->shard_world = N;
  int G = 16;
  ctx->idx_cost = false;  // the p2p walker scans its shard of every row (no range query)
  int k = split_for(ctx, &G);
  if (k <= 1) {
    k = 1;
    G = solo_cluster_size(ctx);
  }
  ctx->idx_cost = true;
  ctx->shard_world = 1;
  unsigned long long* seq = ctx->d_xh_seq;
  int32_t* err = reinterpret_cast<int32_t*>(seq + fmdp::XMAX);
  int32_t* queue = reinterpret_cast<int32_t*>(seq + fmdp::XMAX + 1);
  {  // every cluster starts from the common sequence (monotonic: no stale tag can match)
    std::vector<unsigned long long> s0(fmdp::XMAX, ctx->xh_seq);
    CK(cudaMemcpyAsync(seq, s0.data(), sizeof(unsigned long long) * fmdp::XMAX, cudaMemcpyHostToDevice, ctx->stream));
    CK(cudaMemsetAsync(queue, 0, sizeof(int32_t) * fmdp::XMAX, ctx->stream));
  }
  ctx->xmode = 3;
  fmdp::WalkArgs a = make_args(ctx, base, false, INT_MAX);
  ctx->xmode = 0;
  a.xmode = 3;
  a.x_intra = 1;
  a.x_me = 0;
  a.x_world = k;
  a.x_slot = ctx->x_slot;
  a.x_peers = ctx->d_xh_peers;
  a.x_seq = seq;
  a.x_err = err;
  a.queue = queue;
  a.shard_rank = me * k;
  a.shard_world = N * k;
  a.x_inter = 1;
  a.x_iworld = N;
  a.x_ime = me;
  a.x_ipeers = ctx->d_ipeers;
  st = run_walk(ctx, base, false, INT_MAX, &a, G, k);
  if (st) return st;
  ctx->stats.split = k;
  unsigned long long tail[2] = {0, 0};  // cluster 0's sequence, error flag
  CK(cudaMemcpy(tail, seq, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&tail[1], seq + fmdp::XMAX, sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  if ((int32_t)tail[1]) {
    ctx->x_me = -1;
    return fail(ctx, FMDP_E_CUDA, "peer exchange timed out (a rank did not call fmdp_schedule_p2p)");
  }
  ctx->xh_seq = tail[0];
  if ((st = fetch_out(ctx, 1))) return st;
  ctx->stats.steps += ctx->h_out[0].steps_run;
  ctx->stats.rounds += 1;
  if (ctx->launch.profile) {
    unsigned long long ph[fmdp::N_PHASES];
    CK(cudaMemcpy(ph, ctx->d_prof, sizeof(ph), cudaMemcpyDeviceToHost));
    for (int i = 0; i < fmdp::N_PHASES; ++i) ctx->stats.phase_cycles[i] = (int64_t)ph[i];
  }
  return finish_single(ctx, base, aircraft_id, res, traj);
}

// Co-simulated batch: one cluster per request, all resident at once (they wait for
// each other every clock).  Cluster size: the cost model of choose_launch among the sizes
// whose co-resident cluster count covers the batch.
int cosim_cluster_size(fmdp_ctx* ctx, int n) {
  double plans = 0;
  {
    int64_t tot = 0, nz = 0;
    for (int32_t c : ctx->counts)
      if (c) { tot += c; ++nz; }
    plans = nz ? (double)tot / nz : 0.0;
  }
  const double work = (ctx->launch.cull ? plans * 0.6 : (plans + n) * fmdp::NTAU * ctx->A * ctx->W / 21.0);
  int best_G = 0;
  double best = 1e300;
  for (int G : {16, 8, 4, 2, 1}) {
    if (ctx->launch.cluster_size && G != ctx->launch.cluster_size) continue;
    if (max_clusters(ctx, G, true) < n) continue;
    const double t = work / G + 16000.0 + 300.0 * G;
    if (t < best) {
      best = t;
      best_G = G;
    }
  }
  return best_G;
}

fmdp_status fmdp_schedule_departures(fmdp_ctx* ctx, uint64_t aircraft_id, fmdp_vec3 src, fmdp_vec3 dst,
                                     int64_t t0_step, int32_t n_delays, const int64_t* delays, fmdp_result* res,
                                     fmdp_qpos* traj, int32_t traj_cap, int32_t* chosen) {
  if (ctx && ctx->wide) return fail(ctx, FMDP_E_ARG, "not available with acceleration actions (wide walker)");
  if (!ctx || n_delays < 1 || !delays || !res || !chosen) return fail(ctx, FMDP_E_ARG, "null argument");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  {
    const fmdp_status e = ensure_index(ctx);
    if (e) return e;
  }
  if (traj && traj_cap < ctx->w.max_steps + 1) return fail(ctx, FMDP_E_BUFFER, "traj_cap must be >= max_steps + 1");
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  *chosen = -1;
  std::vector<fmdp_request> rq(n_delays);
  for (int i = 0; i < n_delays; ++i) {
    rq[i].aircraft_id = aircraft_id;
    rq[i].src = src;
    rq[i].dst = dst;
    rq[i].t0_step = t0_step + delays[i];
  }
  std::vector<Req> base;
  fmdp_status st = prepare_requests(ctx, rq.data(), n_delays, base);
  if (st) return st;
  if ((st = ensure_slots(ctx, n_delays))) return st;
  CK(cudaMemsetAsync(ctx->d_pairctr, 0, sizeof(unsigned long long), ctx->stream));
  // every candidate against the same store: one walk over all of them, no commits in between
  if ((st = run_walk(ctx, base, false))) return st;
  if ((st = fetch_out(ctx, n_delays))) return st;
  ctx->stats.rounds = 1;
  int best = -1;
  for (int i = 0; i < n_delays; ++i) {
    ctx->stats.steps += ctx->h_out[i].steps_run;
    if (ctx->h_out[i].status == FMDP_ACCEPTED && (best < 0 || base[i].t0 < base[best].t0)) best = i;
  }
  std::vector<uint32_t> plan_id(n_delays, 0xffffffffu);
  std::vector<uint64_t> aircraft(n_delays, aircraft_id);
  if (best >= 0 && (st = commit_slots(ctx, {best}, base, aircraft, plan_id))) return st;
  *chosen = best;
  for (int i = 0; i < n_delays; ++i) {
    const Out& o = ctx->h_out[i];
    res[i].status = o.status;
    res[i].plan_id = plan_id[i];
    res[i].n_states = o.n_states;
    res[i].fail_step = o.fail_step;
    res[i].min_sep_m = std::sqrt((double)o.min_sep_d2) * ctx->air.u_m;
    res[i].n_near_ties = o.n_near_ties;
    res[i].n_exact = o.n_exact;
    if (traj)
      CK(cudaMemcpyAsync(traj + (size_t)i * traj_cap, ctx->d_traj + (size_t)i * ctx->cap_states * 3,
                         sizeof(fmdp_qpos) * o.n_states, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  unsigned long long pc = 0;
  CK(cudaMemcpy(&pc, ctx->d_pairctr, sizeof(pc), cudaMemcpyDeviceToHost));
  ctx->stats.pair_evals = (int64_t)pc;
  ctx->last_n = n_delays;
  return FMDP_OK;
}

int32_t fmdp_cosim_max(fmdp_ctx* ctx) {
  if (ctx && ctx->wide) return 0;
  if (!ctx) return 0;
  DevGuard dev_guard(ctx->device);  // occupancy queries use the current device
  int m = 0;
  for (int G : {1, 2, 4, 8, 16})
    if (!ctx->launch.cluster_size || G == ctx->launch.cluster_size) m = std::max(m, max_clusters(ctx, G, true));
  return m;
}

fmdp_status fmdp_schedule_cosim(fmdp_ctx* ctx, const fmdp_request* reqs, int32_t n, fmdp_result* res, fmdp_qpos* traj,
                                int32_t traj_cap_each) {
  if (ctx && ctx->wide) return fail(ctx, FMDP_E_ARG, "not available with acceleration actions (wide walker)");
  if (!ctx || n < 1 || !reqs || !res) return fail(ctx, FMDP_E_ARG, "null argument");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  if (traj && traj_cap_each < ctx->w.max_steps + 1) return fail(ctx, FMDP_E_BUFFER, "traj_cap must be >= max_steps + 1");
  std::memset(&ctx->stats, 0, sizeof(ctx->stats));
  std::vector<Req> base;
  fmdp_status st = prepare_requests(ctx, reqs, n, base);
  if (st) return st;
  const int G = cosim_cluster_size(ctx, n);
  if (G == 0)
    return fail(ctx, FMDP_E_CAPACITY, "co-simulated batch larger than the co-resident walkers (fmdp_cosim_max)");
  if ((st = ensure_slots(ctx, n))) return st;
  if (n > ctx->cs_cap) {
    if ((st = grow(ctx, ctx->d_cspub, (size_t)4 * n)) || (st = grow(ctx, ctx->d_csctr, 2))) return st;
    ctx->cs_cap = n;
  }
  int64_t k0 = INT64_MAX;
  for (const Req& r : base) k0 = std::min(k0, r.t0);
  CK(cudaMemsetAsync(ctx->d_csctr, 0, 2 * sizeof(int32_t), ctx->stream));
  CK(cudaMemsetAsync(ctx->d_cspub, 0, sizeof(int4) * 4 * n, ctx->stream));
  CK(cudaMemsetAsync(ctx->d_pairctr, 0, sizeof(unsigned long long), ctx->stream));
  fmdp::WalkArgs a = make_args(ctx, base, false, INT_MAX);
  a.cosim = 1;
  a.cs_n = n;
  a.cs_k0 = k0;
  a.cs_pub = ctx->d_cspub;
  a.cs_arrive = reinterpret_cast<unsigned*>(ctx->d_csctr);
  a.cs_err = ctx->d_csctr + 1;
  if ((st = run_walk(ctx, base, false, INT_MAX, &a, G, n))) return st;
  int32_t err = 0;
  CK(cudaMemcpy(&err, ctx->d_csctr + 1, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) return fail(ctx, FMDP_E_CUDA, "co-simulation clock barrier timed out (walkers not co-resident)");
  if ((st = fetch_out(ctx, n))) return st;
  ctx->stats.rounds = 1;
  std::vector<int> acc;
  for (int i = 0; i < n; ++i) {
    ctx->stats.steps += ctx->h_out[i].steps_run;
    if (ctx->h_out[i].status == FMDP_ACCEPTED) acc.push_back(i);
  }
  // accepted plans are mutually separated (N x N terminal test): append all, in array order
  std::vector<uint32_t> plan_id(n, 0xffffffffu);
  std::vector<uint64_t> aircraft(n);
  for (int i = 0; i < n; ++i) aircraft[i] = reqs[i].aircraft_id;
  if ((st = commit_slots(ctx, acc, base, aircraft, plan_id))) return st;
  for (int i = 0; i < n; ++i) {
    const Out& o = ctx->h_out[i];
    res[i].status = o.status;
    res[i].plan_id = plan_id[i];
    res[i].n_states = o.n_states;
    res[i].fail_step = o.fail_step;
    res[i].min_sep_m = std::sqrt((double)o.min_sep_d2) * ctx->air.u_m;
    res[i].n_near_ties = o.n_near_ties;
    res[i].n_exact = o.n_exact;
    if (traj)
      CK(cudaMemcpyAsync(traj + (size_t)i * traj_cap_each, ctx->d_traj + (size_t)i * ctx->cap_states * 3,
                         sizeof(fmdp_qpos) * o.n_states, cudaMemcpyDeviceToHost, ctx->stream));
  }
  CK(cudaStreamSynchronize(ctx->stream));
  unsigned long long pc = 0;
  CK(cudaMemcpy(&pc, ctx->d_pairctr, sizeof(pc), cudaMemcpyDeviceToHost));
  ctx->stats.pair_evals = (int64_t)pc;
  ctx->last_n = n;
  return FMDP_OK;
}

fmdp_status fmdp_schedule_batch_dist(fmdp_ctx* ctx, const fmdp_gather* g, const fmdp_request* reqs, int32_t n,
                                     fmdp_result* res, fmdp_qpos* traj, int32_t traj_cap_each) {
  if (!ctx || !g) return fail(ctx, FMDP_E_ARG, "null argument");
  return schedule_many(ctx, reqs, n, res, traj, traj_cap_each, 0, g);
}

fmdp_status fmdp_schedule_batch(fmdp_ctx* ctx, const fmdp_request* reqs, int32_t n, fmdp_result* res,
                                fmdp_qpos* traj, int32_t traj_cap_each, int32_t flags) {
  return schedule_many(ctx, reqs, n, res, traj, traj_cap_each, flags);
}

fmdp_status fmdp_get_steplog(fmdp_ctx* ctx, int32_t index, int32_t* astar, int32_t* heading, int32_t* near_tie,
                             int32_t cap, int32_t* n) {
  if (!ctx || index < 0 || index >= ctx->last_n) return fail(ctx, FMDP_E_ARG, "no such request in the last call");
  DevGuard dev_guard(ctx->device);
  const int ns = ctx->h_out[index].n_states;
  if (n) *n = ns;
  if (cap < ns) return FMDP_E_BUFFER;
  const size_t b = (size_t)index * ctx->cap_states;
  if (astar) CK(cudaMemcpy(astar, ctx->d_astar + b, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost));
  if (heading) CK(cudaMemcpy(heading, ctx->d_heading + b, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost));
  if (near_tie) {
    std::vector<int8_t> t(ns);
    CK(cudaMemcpy(t.data(), ctx->d_ntie + b, ns, cudaMemcpyDeviceToHost));
    for (int i = 0; i < ns; ++i) near_tie[i] = t[i];
  }
  return FMDP_OK;
}

fmdp_status fmdp_set_trace(fmdp_ctx* ctx, int32_t n_requests) {
  if (!ctx || n_requests < 0) return fail(ctx, FMDP_E_ARG, "n_requests must be >= 0");
  DevGuard dev_guard(ctx->device);
  if (n_requests > ctx->vtrace_n || (n_requests > 0 && !ctx->d_vtrace)) {
    dfree(ctx, ctx->d_vtrace);
    ctx->d_vtrace = (double2*)dalloc(ctx, sizeof(double2) * (size_t)n_requests * ctx->cap_states * ctx->A);
    if (!ctx->d_vtrace) {
      ctx->vtrace_n = 0;
      return fail(ctx, FMDP_E_NOMEM, "trace buffer");
    }
  }
  ctx->vtrace_n = n_requests;
  return FMDP_OK;
}

fmdp_status fmdp_get_trace(fmdp_ctx* ctx, int32_t index, double* vstar, double* scale, int32_t cap_steps, int32_t* n) {
  if (!ctx || index < 0 || index >= ctx->last_n || index >= ctx->vtrace_n || !ctx->d_vtrace)
    return fail(ctx, FMDP_E_ARG, "request not traced in the last call (fmdp_set_trace)");
  DevGuard dev_guard(ctx->device);
  const int ns = std::max(0, ctx->h_out[index].n_states - 1);  // decision steps 0..n-2
  if (n) *n = ns;
  if (cap_steps < ns) return FMDP_E_BUFFER;
  std::vector<double2> t((size_t)ns * ctx->A);
  if (ns) CK(cudaMemcpy(t.data(), ctx->d_vtrace + (size_t)index * ctx->cap_states * ctx->A, sizeof(double2) * t.size(),
                        cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < t.size(); ++i) {
    if (vstar) vstar[i] = t[i].x;
    if (scale) scale[i] = t[i].y;
  }
  return FMDP_OK;
}

fmdp_status fmdp_get_speeds(fmdp_ctx* ctx, int32_t index, int32_t* speed, int32_t cap, int32_t* n) {
  if (!ctx || index < 0 || index >= ctx->last_n) return fail(ctx, FMDP_E_ARG, "no such request in the last call");
  DevGuard dev_guard(ctx->device);
  const int ns = ctx->h_out[index].n_states;
  if (n) *n = ns;
  if (cap < ns) return FMDP_E_BUFFER;
  if (!speed) return FMDP_OK;
  if (!ctx->wide) {  // constant speed
    for (int i = 0; i < ns; ++i) speed[i] = ctx->w.v0;
    return FMDP_OK;
  }
  CK(cudaMemcpy(speed, ctx->d_speed + (size_t)index * ctx->cap_states, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost));
  return FMDP_OK;
}

fmdp_status fmdp_get_plan(fmdp_ctx* ctx, uint32_t plan_id, int64_t* t0_step, fmdp_qpos* buf, int32_t cap, int32_t* n) {
  if (!ctx || plan_id >= ctx->plans.size()) return fail(ctx, FMDP_E_ARG, "no such plan");
  const PlanRec& p = ctx->plans[plan_id];
  const int32_t ns = (int32_t)(p.states.size() / 3);
  if (n) *n = ns;
  if (t0_step) *t0_step = p.t0;
  if (!buf) return FMDP_OK;
  if (cap < ns) return FMDP_E_BUFFER;
  std::memcpy(buf, p.states.data(), sizeof(int32_t) * p.states.size());
  return FMDP_OK;
}

fmdp_status fmdp_num_plans(const fmdp_ctx* ctx, uint32_t* n) {
  if (!ctx || !n) return FMDP_E_ARG;
  *n = (uint32_t)ctx->plans.size();
  return FMDP_OK;
}

fmdp_status fmdp_truncate(fmdp_ctx* ctx, uint32_t n_plans) {
  if (!ctx) return FMDP_E_ARG;
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  if (n_plans >= ctx->plans.size()) return FMDP_OK;
  if (n_plans < ctx->n_indexed) {
    // rows below the range-query index's sorted regions: reload the kept plans from the host
    // records (empty rows, re-append in id order) and rebuild the index before the next culled walk
    std::vector<PlanRec> keep(ctx->plans.begin(), ctx->plans.begin() + n_plans);
    std::fill(ctx->counts.begin(), ctx->counts.end(), 0);
    CK(cudaMemsetAsync(ctx->d_counts, 0, sizeof(int32_t) * ctx->counts.size(), ctx->stream));
    ctx->plans.clear();
    ctx->w.cell_n = 0;
    ctx->n_indexed = 0;
    std::vector<uint64_t> ids;
    std::vector<int64_t> t0;
    std::vector<int32_t> n;
    std::vector<int32_t> st;
    for (const PlanRec& r : keep) {
      ids.push_back(r.aircraft);
      t0.push_back(r.t0);
      n.push_back((int32_t)(r.states.size() / 3));
      st.insert(st.end(), r.states.begin(), r.states.end());
    }
    if (keep.empty()) {
      ctx->index_dirty = true;
      CK(cudaStreamSynchronize(ctx->stream));
      return FMDP_OK;
    }
    return fmdp_add_plans(ctx, (int32_t)keep.size(), ids.data(), t0.data(), n.data(),
                          reinterpret_cast<const fmdp_qpos*>(st.data()), nullptr);
  }
  // later plans occupy the top slots of each of their rows (appends are in id order)
  for (size_t i = n_plans; i < ctx->plans.size(); ++i) {
    const PlanRec& p = ctx->plans[i];
    const int64_t ns = (int64_t)(p.states.size() / 3);
    for (int64_t k = 0; k < ns; ++k) ctx->counts[p.t0 + k] -= 1;
  }
  ctx->plans.resize(n_plans);
  CK(cudaMemcpyAsync(ctx->d_counts, ctx->counts.data(), sizeof(int32_t) * ctx->counts.size(), cudaMemcpyHostToDevice,
                     ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return FMDP_OK;
}

namespace {
const char kStoreMagic[8] = {'F', 'M', 'D', 'P', 'P', 'L', 'N', '1'};
struct FileCloser {
  FILE* f;
  ~FileCloser() {
    if (f) std::fclose(f);
  }
};
}  // namespace

fmdp_status fmdp_save_plans(const fmdp_ctx* ctx, const char* path, uint32_t first_id) {
  if (!ctx || !path || first_id > ctx->plans.size()) return FMDP_E_ARG;
  fmdp_ctx* c = const_cast<fmdp_ctx*>(ctx);  // only for the error text
  FileCloser fc{std::fopen(path, "wb")};
  if (!fc.f) return fail(c, FMDP_E_IO, std::string("cannot create ") + path);
  const uint32_t ver[2] = {1u, 0u};
  const uint64_t np = ctx->plans.size() - first_id;
  bool ok = std::fwrite(kStoreMagic, 1, 8, fc.f) == 8 && std::fwrite(ver, 4, 2, fc.f) == 2 &&
            std::fwrite(&np, 8, 1, fc.f) == 1;
  for (size_t i = first_id; ok && i < ctx->plans.size(); ++i) {
    const PlanRec& p = ctx->plans[i];
    const int32_t n[2] = {(int32_t)(p.states.size() / 3), 0};
    ok = std::fwrite(&p.aircraft, 8, 1, fc.f) == 1 && std::fwrite(&p.t0, 8, 1, fc.f) == 1 &&
         std::fwrite(n, 4, 2, fc.f) == 2 &&
         std::fwrite(p.states.data(), 4, p.states.size(), fc.f) == p.states.size();
  }
  ok = ok && std::fflush(fc.f) == 0;
  return ok ? FMDP_OK : fail(c, FMDP_E_IO, std::string("write failed: ") + path);
}

fmdp_status fmdp_load_plans(fmdp_ctx* ctx, const char* path, uint32_t* first_id) {
  if (!ctx || !path) return fail(ctx, FMDP_E_ARG, "null argument");
  FileCloser fc{std::fopen(path, "rb")};
  if (!fc.f) return fail(ctx, FMDP_E_IO, std::string("cannot open ") + path);
  char magic[8];
  uint32_t ver[2];
  uint64_t np = 0;
  if (std::fread(magic, 1, 8, fc.f) != 8 || std::memcmp(magic, kStoreMagic, 8) != 0 ||
      std::fread(ver, 4, 2, fc.f) != 2 || ver[0] != 1u || std::fread(&np, 8, 1, fc.f) != 1)
    return fail(ctx, FMDP_E_IO, std::string("not a version-1 plan-store file: ") + path);
  std::vector<uint64_t> ids;
  std::vector<int64_t> t0;
  std::vector<int32_t> n, st;
  for (uint64_t i = 0; i < np; ++i) {
    uint64_t id;
    int64_t t;
    int32_t nn[2];
    if (std::fread(&id, 8, 1, fc.f) != 1 || std::fread(&t, 8, 1, fc.f) != 1 || std::fread(nn, 4, 2, fc.f) != 2 ||
        nn[0] < 1 || nn[0] > (1 << 24))
      return fail(ctx, FMDP_E_IO, std::string("truncated or corrupt plan record in ") + path);
    const size_t off = st.size();
    st.resize(off + 3 * (size_t)nn[0]);
    if (std::fread(st.data() + off, 4, 3 * (size_t)nn[0], fc.f) != 3 * (size_t)nn[0])
      return fail(ctx, FMDP_E_IO, std::string("truncated plan states in ") + path);
    ids.push_back(id);
    t0.push_back(t);
    n.push_back(nn[0]);
  }
  return fmdp_add_plans(ctx, (int32_t)np, ids.data(), t0.data(), n.data(),
                        reinterpret_cast<const fmdp_qpos*>(st.data()), first_id);
}

fmdp_status fmdp_eval_step(fmdp_ctx* ctx, fmdp_qpos pos, int32_t heading, fmdp_qpos goal, int64_t clock_step,
                           double* vstar, double* v_at, double* scale_at, int32_t* conflict, int64_t* min_d2,
                           int32_t* a_star) {
  return fmdp_eval_step_v(ctx, pos, heading, 0, goal, clock_step, vstar, v_at, scale_at, conflict, min_d2, a_star);
}

fmdp_status fmdp_eval_step_v(fmdp_ctx* ctx, fmdp_qpos pos, int32_t heading, int32_t speed_u, fmdp_qpos goal,
                             int64_t clock_step, double* vstar, double* v_at, double* scale_at, int32_t* conflict,
                             int64_t* min_d2, int32_t* a_star) {
  if (!ctx || !vstar) return fail(ctx, FMDP_E_ARG, "null argument");
  DevGuard dev_guard(ctx->device);  // the context's device for this call, the caller's restored after
  if (clock_step < 0 || clock_step + 1 >= ctx->w.horizon) return fail(ctx, FMDP_E_RANGE, "clock outside horizon");
  if (heading < 0 || heading >= ctx->w.HL) return fail(ctx, FMDP_E_ARG, "heading outside the lattice");
  if (speed_u > 0 && (speed_u < ctx->w.vmin || speed_u > ctx->w.vmax))
    return fail(ctx, FMDP_E_ARG, "speed outside [speed_min, speed_max]");
  fmdp_status st = ensure_slots(ctx, 1);
  if (st) return st;
  Req r;
  std::memset(&r, 0, sizeof(r));
  r.src[0] = pos.x; r.src[1] = pos.y; r.src[2] = pos.z;
  r.dst[0] = goal.x; r.dst[1] = goal.y; r.dst[2] = goal.z;
  r.psi0 = heading;
  r.speed0 = speed_u;
  r.t0 = clock_step;
  r.slot = 0;
  if ((st = run_walk(ctx, {r}, true))) return st;
  const int A = ctx->A, AW = A * ctx->W;
  std::vector<uint32_t> conf(A + 1);
  int32_t as = 0;
  CK(cudaMemcpy(vstar, ctx->d_dbg_vstar, sizeof(double) * A, cudaMemcpyDeviceToHost));
  if (v_at) CK(cudaMemcpy(v_at, ctx->d_dbg_v, sizeof(double) * AW, cudaMemcpyDeviceToHost));
  if (scale_at) CK(cudaMemcpy(scale_at, ctx->d_dbg_s, sizeof(double) * AW, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(conf.data(), ctx->d_dbg_conf, sizeof(uint32_t) * (A + 1), cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(&as, ctx->d_dbg_astar, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (conflict)
    for (int a = 0; a < A; ++a) conflict[a] = conf[a] < ctx->w.sep2 ? 1 : 0;
  if (min_d2)
    for (int a = 0; a <= A; ++a) min_d2[a] = conf[a];
  if (a_star) *a_star = as;
  return FMDP_OK;
}

fmdp_status fmdp_get_stats(const fmdp_ctx* ctx, fmdp_stats* out) {
  if (!ctx || !out) return FMDP_E_ARG;
  *out = ctx->stats;
  return FMDP_OK;
}

}  // extern "C"

// fmdp_walk.cu -- sm_100a kernels of the FastMDP-GPU hot path.
//
// walk_kernel<C, MODE>: one thread-block CLUSTER of G CTAs walks one request's whole trajectory
// (Fig 3a loop) with no host round trip per step; clusters take requests from
// a device queue.  Per decision step k (clock row K = t0 + k):
//   a1  stage the CTA's slice of row K (and prefetch row K+2) with cp.async.bulk (TMA)
//       into shared memory; build the 5 intruder wells per plan (Alg 2, Table PK)
//       as FP32 offsets from the anchor q (exact integers < 2^24)
//   a2  forward-project every action W substeps on the integer heading lattice (Alg 3)
//   a3  goal term in fp64 (Alg 4), a5 terrain wells exact (Alg 6), deck (Alg 1)
//   a4  HOT LOOP (Alg 7): per projected state and tau, min over the slice's wells of the
//       FP32 squared distance -- all intruder wells share |r| and gamma, so
//       max_j [d_j<R] |r| g^{d_j} = |r| g^{min in-radius d}; the in/out test is exact
//       (FP32 filter with a 2^-20 band, exact int64 rescan inside the band)
//       fused: exact separation minimum of every action's first substep vs row K+1
//   reduce  cross-CTA min through distributed shared memory (float-bit atomicMin into
//       CTA 0, order-free => deterministic), one cluster barrier
//   a6-a8  every CTA redundantly: combine (Alg 8), max over t, argmax (Alg 9),
//       advance (Alg 1), terminal tests (Sec IV.I)
#include <cooperative_groups.h>
#include <algorithm>
#include <mutex>
#include <type_traits>
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cstdint>

#include "fmdp_dev.h"

namespace cg = cooperative_groups;

namespace fmdp {

// ----------------------------------------------------------------------------- PTX helpers
#ifndef FMDP_MBAR_SUSPEND_NS
#define FMDP_MBAR_SUSPEND_NS 1000000  // (A/B, same box: full configs[1] batch 117.8 -> 115.6 ms with it)
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// try_wait with a suspend-time hint: a waiting thread sleeps until the phase completes (or the hint
// elapses) instead of re-polling, so warps that wait do not take issue slots from the warps of
// their SM sub-partition that still work (the owner pass, the decision)
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
#if FMDP_MBAR_SUSPEND_NS == 0
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
  return;
#endif
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(FMDP_MBAR_SUSPEND_NS)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// DSMEM push (sm_90+): st.async into a cluster CTA's shared memory, completing bytes on that
// CTA's mbarrier -- replaces a cluster barrier (and its MEMBAR.GPU + L1 flush) per exchange.
__device__ __forceinline__ uint32_t mapa_u32(uint32_t a, unsigned rank) {
  uint32_t d;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(rank));
  return d;
}
__device__ __forceinline__ void st_async_f4(uint32_t ra, float4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(ra),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_u32(uint32_t ra, uint32_t v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.u32 [%0], %1, [%2];" ::"r"(ra), "r"(v), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async_d2(uint32_t ra, double a, double b, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(ra), "d"(a),
               "d"(b), "r"(rbar)
               : "memory");
}
// DSMEM bulk copy (sm_90+): one cp.async.bulk of a contiguous shared-memory run into a cluster CTA's
// shared memory, completing its bytes on that CTA's mbarrier -- the reduce-scatter sends one copy
// per owner CTA instead of one 16-byte st.async per float4 (the SM's remote-store issue rate, not
// the bytes, was the exchange's cost).  Source reads complete per bulk group (wait_read before reuse).
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   dst_cluster),
               "r"(src), "r"(bytes), "r"(bar_cluster)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// The same pushes for a one-CTA cluster (G = 1): DSMEM accesses (mapa / st.async) need a cluster
// of at least two CTAs (compute-sanitizer memcheck, profiles/r02_sanitizer.md), so the value is a
// plain shared store, released to the waiting threads by a CTA fence, and its bytes are completed
// on the CTA's own mbarrier (complete_tx; the tx-count may go transiently negative, exactly as when
// an st.async lands before the expect_tx).
__device__ __forceinline__ void complete_tx_local(uint32_t bar, uint32_t bytes) {
  asm volatile("fence.acq_rel.cta;" ::: "memory");
  asm volatile("mbarrier.complete_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void push_u32(bool solo, uint32_t a, unsigned dst, uint32_t v, uint32_t bar) {
  if (solo) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
    complete_tx_local(bar, 4);
  } else {
    st_async_u32(mapa_u32(a, dst), v, mapa_u32(bar, dst));
  }
}

__device__ __forceinline__ void push_d2(bool solo, uint32_t a, unsigned dst, double x, double y, uint32_t bar) {
  if (solo) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(x), "d"(y) : "memory");
    complete_tx_local(bar, 16);
  } else {
    st_async_d2(mapa_u32(a, dst), x, y, mapa_u32(bar, dst));
  }
}
// Generic pointer to `p` in cluster CTA `r` (the own pointer in a one-CTA cluster, see above).
template <class T>
__device__ __forceinline__ T* peer_ptr(cg::cluster_group& cl, T* p, unsigned r, bool solo) {
  return solo ? p : cl.map_shared_rank(p, r);
}
// 4-byte asynchronous global -> shared copy (LDGSTS); completion by cp.async.wait_all.
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Packed FP32 pairs (sm_100: FADD2 / FMUL2 / FFMA2) and the 3-input minimum (FMNMX3).
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 hi_set(f2 v, float hi) {  // replace the high float
  float lo;
  asm("mov.b64 {%0, _}, %1;" : "=f"(lo) : "l"(v));
  return pk2(lo, hi);
}
__device__ __forceinline__ float min3(float a, f2 p) {
  float lo, hi, r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p));
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(lo), "f"(hi));
  return r;
}

__device__ __forceinline__ int sext(uint32_t v, int bits) { return (int)(v << (32 - bits)) >> (32 - bits); }

// exact squared distance, saturated at sat (= R_max^2 < 2^30): valid because any component
// >= R_max already implies d^2 >= R_max^2.
__device__ __forceinline__ uint32_t clamp_d2(int dx, int dy, int dz, int rmax, uint32_t sat) {
  const uint32_t ax = (uint32_t)abs(dx), ay = (uint32_t)abs(dy), az = (uint32_t)abs(dz);
  const uint32_t mx = max(ax, max(ay, az));
  const uint32_t a = min(ax, (uint32_t)rmax), b = min(ay, (uint32_t)rmax), c = min(az, (uint32_t)rmax);
  const uint32_t d2 = a * a + b * b + c * c;  // < 3 * 2^30: no overflow (branch-free)
  return mx >= (uint32_t)rmax ? sat : min(d2, sat);
}

// Order-preserving unsigned key of a double (larger value -> larger key).
__device__ __forceinline__ unsigned long long dkey(double v) {
  const unsigned long long u = (unsigned long long)__double_as_longlong(v);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
// Lane (in `mask`) holding the maximum key, ties broken by the smallest `idx`, among lanes
// whose `ok` is set; -1 if none.  32-bit REDUX reductions (sm_80+): max hi, max lo, min idx.
__device__ __forceinline__ int argmax_key(unsigned mask, bool ok, unsigned long long key, unsigned idx) {
  const unsigned hi = ok ? (unsigned)(key >> 32) : 0u;
  const unsigned mhi = __reduce_max_sync(mask, hi);
  const bool c1 = ok && hi == mhi;
  const unsigned lo = c1 ? (unsigned)key : 0u;
  const unsigned mlo = __reduce_max_sync(mask, lo);
  const bool c2 = c1 && lo == mlo;
  const unsigned mi = __reduce_min_sync(mask, c2 ? idx : 0xffffffffu);
  const unsigned win = __ballot_sync(mask, c2 && idx == mi) & mask;
  return win ? __ffs(win) - 1 : -1;
}

// Per-step shared control block.  Counters used inside a step are double-buffered by step
// parity so that no CTA barrier is needed at a step boundary.
struct Ctl {
  int32_t req;
  int32_t fl0;                // terrain (1) / goal (2) flags of the starting state
  int32_t ntc[2];             // terrain candidate list length, by step parity
  int32_t namb[2];            // ambiguous (state, tau) count, by step parity
  uint32_t stay_local[2];     // this CTA's slice minimum of |q - p(K)|^2, by step parity
  int32_t n_exact;            // exact-fallback count (rank 0 accumulates the cluster's)
  int32_t nsurv[4];           // plans kept by the build, by (step parity, chunk parity)
  unsigned long long xmin;
  int32_t sl_lo[3], sl_n[3], sl_off[3];
  // range-query staging (culled walker, World::cell_n > 0): ring buffer b holds this CTA's share of
  // row K's candidate ranges as pn[b] pieces -- piece i = list entries [pst[b][i], pst[b][i+1]) of
  // the CTA's share, global slots from pgl[b][i], staged at ring position poff[b][i] (-1: beyond the
  // ring's capacity, read from L2)
  int32_t pn[3];
  int32_t pst[3][5], pgl[3][4], poff[3][4];
  int32_t ilo[4], ihi[4];     // (I/O thread) candidate ranges of the next row to issue, loaded one step ahead
  int32_t hgt[MAX_TURN];      // ground height under Delta_1 of every turn (cp.async target)
  int32_t cs_ok;              // scratch of cs_idle
  int32_t stop[2];            // head-finished flag seen by rank 0 at the top of the step, by parity
  uint32_t xstay[2];          // multi-GPU: nearest-plan d^2 over the ranks (from CTA 0), by parity
  int32_t rc_near, rc_exact;  // re-convergence: near-ties / exact counts of the reused steps (rank 0)
  uint32_t rc_min;            //                 their nearest-plan minimum (rank 0)
  int4 bakst[2];              // re-convergence: the previous run's state k + 1, by step parity
  unsigned long long* xp[XMAX];  // multi-GPU: every rank's receive area (loaded once per launch)
  unsigned long long* xip[XNODE];  // two-level exchange: cluster xcl's area on every GPU
};
static_assert(sizeof(Ctl) <= 768, "Ctl exceeds its shared-memory slot (Layout::o_ctl)");

// Stage row K's slice for this CTA (slots [lo, lo+n) of n_row active slots): the first CH
// plans go to ring buffer K % 3 with cp.async.bulk (TMA bulk copy), completion on its
// mbarrier.  Called by one thread.
__device__ __forceinline__ void issue_row(const World& w, int64_t K, int n_row, unsigned rank, unsigned lgG, int CH,
                                          int32_t* raw, int RAWW, uint64_t* bars, Ctl* ctl, int srank, int sworld) {
  const int b = (int)(K % 3);
  // plan shard of this GPU: slots [s0, s1) of the row, then this CTA's part
  int s0 = 0, s1 = n_row;  // single GPU: no 64-bit division on the step's critical path
  if (sworld > 1) {
    s0 = (int)(((int64_t)n_row * srank) / sworld);
    s1 = (int)(((int64_t)n_row * (srank + 1)) / sworld);
  }
  const uint32_t len = (uint32_t)(s1 - s0);
  const int lo = s0 + (int)((len * rank) >> lgG), hi = s0 + (int)((len * (rank + 1)) >> lgG);
  const int e = min(hi, lo + CH);
  const int lo4 = lo & ~3, e4 = (e + 3) & ~3;
  ctl->sl_lo[b] = lo;
  ctl->sl_n[b] = hi - lo;
  ctl->sl_off[b] = lo - lo4;
  const uint32_t bytes = (e > lo) ? (uint32_t)(e4 - lo4) * 4u : 0u;
  fence_proxy_async();
  mbar_arrive_tx(&bars[b], 4u * bytes);
  if (bytes) {
    const int32_t* base = w.rows + (size_t)K * 4 * w.row_cap;
    int32_t* dst = raw + (size_t)b * 4 * RAWW;
    for (int arr = 0; arr < 4; ++arr)
      bulk_g2s(dst + arr * RAWW, base + (size_t)arr * w.row_cap + lo4, bytes, &bars[b]);
  }
}

// Range query (culled walker, World::cell_n > 0): the candidate slot ranges of row K around (qx, qy):
// the three cell rows of the 3x3 block (each one contiguous range: cells are row-major) and the
// appended plans [cstart[K][cell_n], counts[K]).
__device__ __forceinline__ void load_ranges(const World& w, int64_t K, int qx, int qy, int (&lo)[4], int (&hi)[4]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) lo[i] = hi[i] = 0;
  if (K < 0 || K >= w.horizon) return;
  const int32_t* cs = w.cstart + (size_t)K * (w.cell_n + 1);
  const int cx = min(max((qx - w.cell_x0) / w.cell_l, 0), w.cell_ncx - 1);
  const int cy = min(max((qy - w.cell_y0) / w.cell_l, 0), w.cell_ncy - 1);
  const int xa = max(cx - 1, 0), xb = min(cx + 1, w.cell_ncx - 1);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int yy = cy - 1 + i;
    if (yy >= 0 && yy < w.cell_ncy) {
      lo[i] = __ldg(cs + yy * w.cell_ncx + xa);
      hi[i] = __ldg(cs + yy * w.cell_ncx + xb + 1);
    }
  }
  lo[3] = __ldg(cs + w.cell_n);
  hi[3] = __ldg(&w.counts[K]);
}

// The same ranges fetched asynchronously into shared memory (LDGSTS, no register and no stall for the
// issuing thread; it waits with cp.async.wait_all before it reads them, a step later).
__device__ __forceinline__ void fetch_ranges_async(const World& w, int64_t K, int qx, int qy, int32_t* lo, int32_t* hi) {
  if (K < 0 || K >= w.horizon) {
    for (int i = 0; i < 4; ++i) lo[i] = hi[i] = 0;
    return;
  }
  const int32_t* cs = w.cstart + (size_t)K * (w.cell_n + 1);
  const int cx = min(max((qx - w.cell_x0) / w.cell_l, 0), w.cell_ncx - 1);
  const int cy = min(max((qy - w.cell_y0) / w.cell_l, 0), w.cell_ncy - 1);
  const int xa = max(cx - 1, 0), xb = min(cx + 1, w.cell_ncx - 1);
  for (int i = 0; i < 3; ++i) {
    const int yy = cy - 1 + i;
    if (yy >= 0 && yy < w.cell_ncy) {
      cp_async4(&lo[i], cs + yy * w.cell_ncx + xa);
      cp_async4(&hi[i], cs + yy * w.cell_ncx + xb + 1);
    } else {
      lo[i] = hi[i] = 0;
    }
  }
  cp_async4(&lo[3], cs + w.cell_n);
  cp_async4(&hi[3], &w.counts[K]);
}

// Stage this CTA's share of row K's candidate ranges (range query): the concatenation of the four
// ranges is split evenly over the cluster; each intersected piece is copied with cp.async.bulk
// (16-byte aligned, one copy per SoA array) to the next ring position, pieces past the ring's
// capacity are read from L2 (poff = -1).  One thread.
__device__ __forceinline__ void issue_row_idx(const World& w, int64_t K, const int (&lo)[4], const int (&hi)[4],
                                              unsigned rank, unsigned lgG, int RAWCAP, int32_t* raw, int RAWW,
                                              uint64_t* bars, Ctl* ctl) {
  const int b = (int)(K % 3);
  uint32_t T = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) T += (uint32_t)(hi[i] - lo[i]);
  const int s0 = (int)((T * rank) >> lgG), s1 = (int)((T * (rank + 1)) >> lgG);
  int np = 0, base = 0, rpos = 0;
  uint32_t bytes = 0;
  int cg4[4], cn4[4], cr[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int ni = hi[i] - lo[i];
    const int a = max(s0, base), e = min(s1, base + ni);
    cn4[i] = 0;
    if (a < e) {
      const int g = lo[i] + (a - base), cnt = e - a;
      const int g4 = g & ~3, ge4 = (g + cnt + 3) & ~3;
      ctl->pst[b][np] = a - s0;
      ctl->pgl[b][np] = g;
      if (rpos + (ge4 - g4) <= RAWCAP) {
        ctl->poff[b][np] = rpos + (g - g4);
        cg4[i] = g4;
        cn4[i] = ge4 - g4;
        cr[i] = rpos;
        rpos += ge4 - g4;
        bytes += (uint32_t)(ge4 - g4) * 4u;
      } else {
        ctl->poff[b][np] = -1;
      }
      ++np;
    }
    base += ni;
  }
  ctl->pst[b][np] = s1 - s0;
  ctl->pn[b] = np;
  ctl->sl_n[b] = s1 - s0;
  fence_proxy_async();
  mbar_arrive_tx(&bars[b], 4u * bytes);
  const int32_t* row = w.rows + (size_t)K * 4 * w.row_cap;
  int32_t* dst = raw + (size_t)b * 4 * RAWW;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    if (cn4[i] > 0)
      for (int arr = 0; arr < 4; ++arr)
        bulk_g2s(dst + arr * RAWW + cr[i], row + (size_t)arr * w.row_cap + cg4[i], (uint32_t)cn4[i] * 4u, &bars[b]);
}

// Plan jj of this CTA's share of the row in ring buffer b (range query): {x, y, z, packed v}.
__device__ __forceinline__ int4 plan_at(const World& w, const Ctl* ctl, const int32_t* raw, int RAWW, int b, int64_t K,
                                        int jj) {
  const int np = ctl->pn[b];
  int i = 0;
  while (i + 1 < np && jj >= ctl->pst[b][i + 1]) ++i;
  const int d = jj - ctl->pst[b][i];
  const int q = ctl->poff[b][i];
  if (q >= 0) {
    const int32_t* r = raw + (size_t)b * 4 * RAWW + q + d;
    return make_int4(r[0], r[RAWW], r[2 * RAWW], r[3 * RAWW]);
  }
  const int32_t* g = w.rows + (size_t)K * 4 * w.row_cap + ctl->pgl[b][i] + d;
  return make_int4(__ldg(g), __ldg(g + w.row_cap), __ldg(g + 2 * w.row_cap), __ldg(g + 3 * w.row_cap));
}

__device__ __forceinline__ int row_count(const World& w, int64_t K) {
  return (K >= 0 && K < w.horizon) ? __ldg(&w.counts[K]) : 0;
}

// SURVEY f1 cull test of one plan (offsets r from the position the test is made against, forward
// difference v): an exact L-inf prefilter on the whole plan (every well lies within kmax |v|_inf
// of p), then a conservative FP32 test of each well against (R_tau + reach + step_reach + 1)^2.  A
// culled well is farther than R_tau + 1 from every projected state of this step and the next (the
// pre-cull tests against the previous step's q), i.e. clearly outside the FP32 band.
__device__ __forceinline__ bool cull_keep(const World& w, int rx, int ry, int rz, int vx, int vy, int vz) {
  const int vinf = max(abs(vx), max(abs(vy), abs(vz)));
  const int dinf = max(abs(rx), max(abs(ry), abs(rz)));
  if (dinf >= w.cull_inf + w.k_absmax * vinf) return false;
  bool keep = false;
#pragma unroll
  for (int t = 0; t < NTAU; ++t) {
    const float cx = (float)(rx + w.k_tau[t] * vx), cy = (float)(ry + w.k_tau[t] * vy), cz = (float)(rz + w.k_tau[t] * vz);
    keep |= fmaf(cz, cz, fmaf(cy, cy, cx * cx)) < w.cull2f_tau[t];
  }
  return keep;
}

// Top-2 merge for the argmax (Alg 9): order by value, then lowest index (R13).
__device__ __forceinline__ bool better(double v, int i, double bv, int bi) { return v > bv || (v == bv && i < bi); }

// Terrain collision height under (x, y) (R16): INT_MIN outside the raster.  32-bit cell
// arithmetic (positions span < 2^25 units).
__device__ __forceinline__ const int32_t* ground_cell(const World& w, int x, int y) {
  if (w.nx <= 0) return nullptr;
  const int rx = x - w.x0, ry = y - w.y0;
  if (rx < 0 || ry < 0) return nullptr;
  const int ix = (int)(((uint64_t)rx * w.cell_magic) >> 40), iy = (int)(((uint64_t)ry * w.cell_magic) >> 40);
  if (ix >= w.nx || iy >= w.ny) return nullptr;
  return w.height + (size_t)iy * w.nx + ix;
}
__device__ __forceinline__ int ground_height(const World& w, int x, int y) {
  const int32_t* p = ground_cell(w, x, y);
  return p ? __ldg(p) : INT_MIN;
}


// ----------------------------------------------------------------------------- co-simulation clock
// SURVEY f2 (Alg 1: every aircraft decides from the states at clock K, then all
// move).  Walker i publishes its state for clock K into cs_pub[K & 1][i] and arrives; a walker
// reads clock K's entries once all cs_n walkers have arrived.  Two buffers suffice: a walker
// writes clock K+2 only after passing clock K+1, i.e. after every walker published K+1, which
// each does after it finished reading clock K.
enum { CS_ABSENT = 0, CS_PRESENT = 1, CS_FINISHED = 2 };
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __noinline__ void cs_publish_at(int4* e, int x, int y, int z, int flags, int vx, int vy, int vz,
                                           unsigned* arrive) {
  __stcg(e, make_int4(x, y, z, flags));
  __stcg(e + 1, make_int4(vx, vy, vz, 0));
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(arrive) : "memory");
}
__device__ __forceinline__ void cs_publish(const WalkArgs& a, int i, int64_t K, int x, int y, int z, int flags, int vx,
                                           int vy, int vz) {
  cs_publish_at(a.cs_pub + ((size_t)(K & 1) * a.cs_n + i) * 2, x, y, z, flags, vx, vy, vz, a.cs_arrive);
}
// Whole-warp wait (all 32 lanes, warp-uniform result): true once the arrival counter reached
// target, false on a timeout (~2 s: the walkers are not all resident) or when another walker timed
// out.  Lane 0 polls and the warp stays converged, so no lane spins alone while its warp-mates
// wait at a CTA barrier (compute-sanitizer synccheck).  (Plain pointers: a reference to the kernel
// parameters would force a local copy of them.)
__device__ __noinline__ bool cs_wait_warp(const unsigned* arrive, int32_t* err, unsigned target) {
  const long long t0 = clock64();
  for (;;) {
    int st = 0;  // 1 ready, 2 failed
    if ((threadIdx.x & 31) == 0) {
      if (ld_acquire_gpu(arrive) >= target) st = 1;
      else if (*(volatile int32_t*)err) st = 2;
      else if (clock64() - t0 > (4ll << 30)) {
        atomicExch(err, 1);
        st = 2;
      }
    }
    st = __shfl_sync(0xffffffffu, st, 0);
    if (st) return st == 1;
  }
}
__device__ __forceinline__ bool cs_wait(const WalkArgs& a, int64_t K) {
  return cs_wait_warp(a.cs_arrive, a.cs_err, (unsigned)a.cs_n * (unsigned)(K - a.cs_k0 + 1));
}
// Clocks [K0, K1) (or until every walker has finished) on which walker i is not flying:
// publish flags, keep the clock.  All threads of one CTA; false on a barrier failure.
__device__ __noinline__ bool cs_idle(int4* pub_all, unsigned* arrive, int32_t* err, int n, int64_t k0, Ctl* ctl, int i,
                                     int64_t K0, int64_t K1, int flags, bool until_all) {
  for (int64_t K = K0; until_all || K < K1; ++K) {
    int4* pub = pub_all + (size_t)(K & 1) * n * 2;
    if (threadIdx.x == 0) {
      __stcg(pub + 2 * i, make_int4(0, 0, 0, flags));
      __stcg(pub + 2 * i + 1, make_int4(0, 0, 0, 0));
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(arrive) : "memory");
    }
    // every warp waits on its own (uniform code path for the whole CTA; the CTA barrier then
    // orders the pub reads below after the acquiring load)
    const bool ok = __syncthreads_and(cs_wait_warp(arrive, err, (unsigned)n * (unsigned)(K - k0 + 1)));
    bool all = until_all;
    if (ok && until_all)
      for (int j = threadIdx.x; j < n; j += blockDim.x) all &= __ldcg(&pub[2 * j]).w == CS_FINISHED;
    all = __syncthreads_and(all);  // also orders cs_ok's read before the next write
    if (!ok) return false;
    if (all) return true;
  }
  return true;
}

// ----------------------------------------------------------------------------- multi-GPU exchange
// In-kernel plan-sharded step exchange (xmode 3, SURVEY §8(e) production form).  Every rank runs
// the same persistent walker over its shard of every time row.  Each exchanged value travels as
// one 8-byte word {value, step tag} written with a single 64-bit store straight into the peer's
// receive slot (P2P over NVLink; the store is single-copy atomic), and the reader polls the word
// until it carries this step's tag -- value and "ready" arrive together, so no fence and no
// separate flag are needed.  Two parities suffice: CTA c of a rank writes its words of step s+2
// only after it has read every word of step s+1 from the peer's CTA c, which that CTA wrote after
// it had finished reading step s (CTA barriers in between).  A poll longer than ~2 s (a peer is
// not running) sets *err and returns the stale value; every later poll returns at once, the walk
// ends with wrong values and the host reports FMDP_E_CUDA.
// The word is ONE aligned 64-bit scalar access on both sides (st/ld.relaxed.sys.b64: single-copy
// atomic; a vector access would be two element accesses in unspecified order, so a reader could
// see the new tag with the old value): value in the low half, tag in the high half.
__device__ __forceinline__ void st_ll(unsigned long long* p, uint32_t v, uint32_t tag) {
  const unsigned long long w = (unsigned long long)v | ((unsigned long long)tag << 32);
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ void ld_word(const unsigned long long* p, uint32_t& v, uint32_t& t) {
  unsigned long long w;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
  v = (uint32_t)w;
  t = (uint32_t)(w >> 32);
}
__device__ __noinline__ uint32_t ld_ll_wait(const unsigned long long* p, uint32_t tag, int32_t* err, long long budget) {
  const long long t0 = clock64();
  uint32_t v, t;
  for (;;) {
    ld_word(p, v, t);
    if (t == tag) return v;
    if (*(volatile int32_t*)err) return v;
    if (clock64() - t0 > budget) {
      atomicExch(err, 1);
      return v;
    }
  }
}
// Poll budget in SM cycles: ~2 s, ~8 s for a launch's first exchange (the ranks' launches may
// be skewed by their hosts).  Liveness: every poll is bounded, and every polled value is read by
// exactly one CTA of the cluster (items: their owner; the nearest-plan d^2: CTA 0, which then
// broadcasts it over DSMEM), so a timeout can make ranks disagree but never splits a cluster.
__device__ __forceinline__ long long x_budget(unsigned long long xit) { return xit == 1 ? (16ll << 30) : (4ll << 30); }
__device__ __forceinline__ uint32_t ld_ll(const unsigned long long* p, uint32_t tag, int32_t* err, long long budget) {
  uint32_t v, t;
  ld_word(p, v, t);
  return t == tag ? v : ld_ll_wait(p, tag, err, budget);
}
// Minimum of v and the peers' words at item index io of this step: all loads issued first
// (independent round trips), tags checked after; a word not yet there is polled.
__device__ __forceinline__ float x_min_peers(const unsigned long long* own, int me, int world, int slot, int par,
                                             int io, uint32_t tag, int32_t* err, long long budget, float v) {
#pragma unroll 1
  for (int j0 = 0; j0 < world - 1; j0 += 4) {  // four peers' words in flight at a time
    uint32_t wv[4], wt[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = (j0 + j) < me ? (j0 + j) : (j0 + j) + 1;
      if (j0 + j < world - 1) ld_word(own + (size_t)(par * world + q) * slot + io, wv[j], wt[j]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = (j0 + j) < me ? (j0 + j) : (j0 + j) + 1;
      if (j0 + j < world - 1) {
        const uint32_t x =
            wt[j] == tag ? wv[j] : ld_ll_wait(own + (size_t)(par * world + q) * slot + io, tag, err, budget);
        v = fminf(v, __uint_as_float(x));
      }
    }
  }
  return v;
}
// Words of (parity, source rank) in a rank's receive area: [0, A*W*NTAU) the per-(state, tau)
// minima, slot - 16 + cta the nearest-plan d^2 of CTA cta.
__device__ __forceinline__ size_t x_word(int par, int world, int src, int slot, int i) {
  return (size_t)(par * world + src) * slot + i;
}
// Nearest-plan d^2: min over the ranks (warp 0 of CTA 0, lane q polls rank q's word in parallel;
// the own value was published earlier).  All 32 lanes; the result is in every lane.
__device__ __forceinline__ uint32_t x_stay_min(const unsigned long long* own, int me, int world, int slot, int par,
                                               uint32_t tag, uint32_t stay, int32_t* err, long long budget) {
  const int lane = threadIdx.x & 31;
  uint32_t v = stay;
  if (lane < world && lane != me) v = min(v, ld_ll(own + x_word(par, world, lane, slot, slot - 16), tag, err, budget));
  return __reduce_min_sync(0xffffffffu, v);
}

// Second level of the nearest-plan exchange: this GPU's value -> cluster xcl of every other GPU
// (lane q -> GPU q), then the minimum over the GPUs.  Warp 0 of CTA 0; every lane gets it.
__device__ __forceinline__ uint32_t x_stay_inter(unsigned long long* const* xip, int me, int world, int slot, int par,
                                                 uint32_t tag, uint32_t m, int32_t* err, long long budget, bool send) {
  const int lane = threadIdx.x & 31;
  if (send && lane < world && lane != me) st_ll(xip[lane] + x_word(par, world, me, slot, slot - 16), m, tag);
  return x_stay_min(xip[me], me, world, slot, par, tag, m, err, budget);
}

// G-way minimum of one (state, tau) item over the partial blocks of the cluster's CTAs
__device__ __forceinline__ float gway_min(const float* src, int G, int sstride) {
  float M0 = src[0], M1 = FLT_MAX, M2 = FLT_MAX, M3 = FLT_MAX;
  int bb = 1;
  for (; bb + 3 < G; bb += 4) {  // four independent load streams
    M0 = fminf(M0, src[bb * sstride]);
    M1 = fminf(M1, src[(bb + 1) * sstride]);
    M2 = fminf(M2, src[(bb + 2) * sstride]);
    M3 = fminf(M3, src[(bb + 3) * sstride]);
  }
  for (; bb < G; ++bb) M0 = fminf(M0, src[bb * sstride]);
  return fminf(fminf(M0, M1), fminf(M2, M3));
}

struct TauSteps {
  int k[NTAU];
};
// Well records of this CTA's batch peers j = rank + i*G (out of line: keeps the step loop's
// code small).  Returns the thread's minimum separation d^2 to a present peer (saturated).
__device__ __noinline__ uint32_t cs_build_peers(const int4* pub, int npr, int rank, int G, int self, int qx, int qy,
                                                int qz, int ox, int oy, bool records, float* s_cen, int R_max,
                                                uint32_t sat, TauSteps kt) {
  uint32_t stay = sat;
  for (int i = threadIdx.x; i < npr; i += blockDim.x) {
    const int j = rank + i * G;
    const int4 e = __ldcg(&pub[2 * j]);
    const bool on = e.w == CS_PRESENT && j != self;
    int rx = 0, ry = 0, rz = 0, vx = 0, vy = 0, vz = 0;
    if (on) {
      const int4 v = __ldcg(&pub[2 * j + 1]);
      rx = e.x - qx; ry = e.y - qy; rz = e.z - qz;
      vx = v.x; vy = v.y; vz = v.z;
      stay = min(stay, clamp_d2(rx, ry, rz, R_max, sat));
    }
    if (records) {
      float* cp = s_cen + PAIR_STRIDE * (i >> 1) + (i & 1);
#pragma unroll
      for (int t = 0; t < NTAU; ++t) {  // absent peer / self: a well at infinity (Q huge, offsets 0)
        const float X = on ? (float)(ox - (rx + kt.k[t] * vx)) : 0.f;
        const float Y = on ? (float)(oy - (ry + kt.k[t] * vy)) : 0.f;
        const float Z = on ? (float)(-(rz + kt.k[t] * vz)) : 0.f;
        cp[8 * t + 0] = X;
        cp[8 * t + 2] = Y;
        cp[8 * t + 4] = Z;
        cp[8 * t + 6] = on ? fmaf(Z, Z, fmaf(Y, Y, X * X)) : 3.0e18f;
      }
    }
  }
  return stay;
}
// Exact int64 minimum d^2 from q to the tau-well of every present batch peer (this thread's share).
__device__ __noinline__ unsigned long long cs_exact_peers(const int4* pub, int n, int self, int4 q4, int kt) {
  unsigned long long best = ULLONG_MAX;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    const int4 e = __ldcg(&pub[2 * j]);
    if (e.w != CS_PRESENT || j == self) continue;
    const int4 v = __ldcg(&pub[2 * j + 1]);
    const int64_t dx = q4.x - (e.x + (int64_t)kt * v.x), dy = q4.y - (e.y + (int64_t)kt * v.y),
                  dz = q4.z - (e.z + (int64_t)kt * v.z);
    best = min(best, (unsigned long long)(dx * dx + dy * dy + dz * dz));
  }
  return best;
}

// Exact fallback of the owner pass (rare): for every (state, tau) item flagged inside the FP32
// band (s_M[i] == -1), the exact int64 minimum d^2 over the WHOLE row K (and, co-simulating, the
// batch peers of clock K); all threads of the CTA, item by item.
struct TauK {
  int k[NTAU];
  int64_t r2[NTAU];
};
__device__ __forceinline__ void exact_fallback(float* s_M, const int32_t* s_amb, const int4* s_pos, int namb, int nitem,
                                               const int32_t* rowg, int nK, int row_cap, int rank, int G, int W,
                                               const TauK& tk, Ctl* ctl, const int4* cs_pub_K, int cs_n, int self,
                                               int32_t* stepx_k) {
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31;
  const int nit = namb <= AMB_MAX ? namb : nitem;  // overflow: walk every owned item
  for (int it2 = 0; it2 < nit; ++it2) {
    const int i = namb <= AMB_MAX ? s_amb[it2] : it2;
    if (s_M[i] != -1.f) continue;
    const int oa = i / (W * NTAU), r2 = i - oa * (W * NTAU);
    const int l = r2 / NTAU, t = r2 - l * NTAU;
    const int sti = (rank + oa * G) * W + l;
    if (tid == 0) ctl->xmin = ULLONG_MAX;
    __syncthreads();
    const int4 q4 = s_pos[sti];
    const int kt = tk.k[t];
    unsigned long long best = ULLONG_MAX;
    for (int j = tid; j < nK; j += NT) {
      const uint32_t pv = (uint32_t)rowg[3 * row_cap + j];
      const int64_t cx = rowg[j] + (int64_t)kt * sext(pv, 11);
      const int64_t cy = rowg[row_cap + j] + (int64_t)kt * sext(pv >> 11, 11);
      const int64_t cz = rowg[2 * row_cap + j] + (int64_t)kt * sext(pv >> 22, 10);
      const int64_t ddx = q4.x - cx, ddy = q4.y - cy, ddz = q4.z - cz;
      best = min(best, (unsigned long long)(ddx * ddx + ddy * ddy + ddz * ddz));
    }
    if (cs_pub_K)  // batch peers of clock K
      best = min(best, cs_exact_peers(cs_pub_K, cs_n, self, q4, kt));
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if (lane == 0 && best != ULLONG_MAX) atomicMin(&ctl->xmin, best);
    __syncthreads();
    if (tid == 0) {
      const unsigned long long x = ctl->xmin;
      s_M[i] = ((int64_t)x < tk.r2[t]) ? (float)x : FLT_MAX;
      atomicAdd(&ctl->n_exact, 1);
      if (stepx_k) atomicAdd(stepx_k, 1);  // per-step count: a resumed walk sums its kept prefix
    }
    __syncthreads();
  }
}
__device__ __noinline__ void exact_fallback_call(float* s_M, const int32_t* s_amb, const int4* s_pos, int namb,
                                                 int nitem, const int32_t* rowg, int nK, int row_cap, int rank, int G,
                                                 int W, TauK tk, Ctl* ctl, const int4* cs_pub_K, int cs_n, int self,
                                                 int32_t* stepx_k) {
  exact_fallback(s_M, s_amb, s_pos, namb, nitem, rowg, nK, row_cap, rank, G, W, tk, ctl, cs_pub_K, cs_n, self, stepx_k);
}

// Re-convergence (a10): the previous run's records of steps k .. n_old - 1 (BakRec backup) back into
// the request's arrays, and their near-tie / exact-count sums and separation minimum into rank 0's
// Ctl (c0).  All threads of every CTA of the lead cluster; out of line (keeps the step loop small).
// (Plain pointers: a reference to the kernel parameters would force a local copy of them.)
struct RecPtrs {
  int32_t *traj, *heading, *astar, *stepx;
  uint32_t* stepd2;
  int8_t* ntie;
};
__device__ __noinline__ void reconv_copy(const BakRec* bak, RecPtrs args, size_t sbase, int k, int n_old, unsigned rank,
                                         unsigned G, uint32_t sat, Ctl* c0) {
  const int NT = blockDim.x, tid = threadIdx.x;
  const BakRec* bb = bak + sbase;
  int rn = 0, rx = 0;
  uint32_t rm = sat;
  for (int m = k + (int)rank * NT + tid; m < n_old; m += (int)G * NT) {
    const BakRec e = bb[m];
    if (m > k) {
      int32_t* tq = args.traj + 3 * (sbase + m);
      tq[0] = e.x; tq[1] = e.y; tq[2] = e.z;
      args.heading[sbase + m] = e.heading;
    }
    args.stepd2[sbase + m] = e.stepd2;
    rm = min(rm, e.stepd2);
    if (m < n_old - 1) {  // decision steps
      args.astar[sbase + m] = e.astar;
      args.ntie[sbase + m] = (int8_t)e.ntie;
      if (args.stepx) args.stepx[sbase + m] = e.stepx;
      rn += e.ntie;
      rx += e.stepx;
    }
  }
  rn = __reduce_add_sync(0xffffffffu, rn);
  rx = __reduce_add_sync(0xffffffffu, rx);
  rm = __reduce_min_sync(0xffffffffu, rm);
  if ((tid & 31) == 0) {
    if (rn) atomicAdd(&c0->rc_near, rn);
    if (rx) atomicAdd(&c0->rc_exact, rx);
    if (rm < sat) atomicMin(&c0->rc_min, rm);
  }
}

// Per-phase cycle accounting (rank 0, thread 0), enabled when args.prof != nullptr.
enum Phase { PH_PROJ, PH_FIX, PH_WAIT, PH_HOT, PH_STAGE, PH_SCATTER, PH_BAR1, PH_OWNER, PH_BAR2, PH_DECIDE,
             PH_TOP, PH_SCAN, PH_PLOOP, PH_BUILD, PH_OWN1, PH_ARGMAX, PH_FLAGS, PH_N };

// Inverse of dkey.
__device__ __forceinline__ double undkey(unsigned long long k) {
  return __longlong_as_double((long long)((k >> 63) ? (k & 0x7fffffffffffffffull) : ~k));
}

template <int C, int MODE>
__global__ void __launch_bounds__(C == 1 ? 512 : 384, 1)
    walk_kernel(const World w, const WalkArgs args, const int CH, const int RAWCAP, const int NGW) {
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const unsigned G = cluster.num_blocks();
  const unsigned lgG = 31 - __clz(G);  // G is a power of two
  const bool solo = G == 1;            // one-CTA cluster: no DSMEM (push_* / peer_ptr)
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int W = w.W, A = w.A, AW = A * W;
  const int NCOL = w.n_turn * W;
  // hot-loop mapping: each warp = CPW columns x NGW plan groups; the lanes of one group
  // (a multiple of 8) read the same well record -> shared-memory broadcast
  const int CPW = 32 / NGW;
  const int col = warp * CPW + (lane % CPW), grp = lane / CPW;
  const int col_it = min(col / W, w.n_turn - 1), col_t = col % W + 1;  // this thread's column
  const int col_h = w.turn[col_it];
  // wide walker (MODE 5, SURVEY f4 acceleration actions): this cluster's tile of horizontal paths
  // hp = i_turn * n_acc + i_acc; the thread's path's turn and speed increment; local action a of
  // the tile is global action hp0 * C + a (climb innermost)
  constexpr bool WIDE = MODE == 5;
  const int wcl = WIDE ? (int)(blockIdx.x / G) : 0;
  const int hp0 = WIDE ? wcl * w.hpt : 0;
  const int A_tile = WIDE ? min(w.hpt, w.n_hp - hp0) * C : w.A;
  const int aoff = WIDE ? hp0 * C : 0;
  int col_hw = col_h, col_acc = 0;
  if (WIDE) {
    const int hp = min(hp0 + col_it, w.n_hp - 1);
    col_hw = w.turn[hp / w.n_acc];
    col_acc = w.acc[hp % w.n_acc];
  }
  // actions owned by this CTA (reduce-scatter target and epilogue): a = rank + oa*G
  const int n_own = (A > (int)rank) ? (A - (int)rank + (int)G - 1) / (int)G : 0;

  Layout L;
  L.build(w.HL, CH, RAWCAP, NT, C, NCOL, A, AW, (int)G);
  extern __shared__ __align__(16) unsigned char smem[];
  int2* s_dxy = reinterpret_cast<int2*>(smem + L.o_dxy);
  int4* s_tw = reinterpret_cast<int4*>(smem + L.o_tw);
  int32_t* s_raw = reinterpret_cast<int32_t*>(smem + L.o_raw);
  float* s_cen = reinterpret_cast<float*>(smem + L.o_cen);
  float* s_stage = reinterpret_cast<float*>(smem + L.o_stage);
  float* s_recv = reinterpret_cast<float*>(smem + L.o_recv);
  int4* s_pos2 = reinterpret_cast<int4*>(smem + L.o_pos);
  double* s_fix = reinterpret_cast<double*>(smem + L.o_fix);
  double* s_sfix = reinterpret_cast<double*>(smem + L.o_sfix);
  float* s_vT = reinterpret_cast<float*>(smem + L.o_vT);
  double2* s_vv = reinterpret_cast<double2*>(smem + L.o_vstar);  // {V*(a), S(a)}
  uint32_t* s_conf = reinterpret_cast<uint32_t*>(smem + L.o_conf);
  int32_t* s_flags = reinterpret_cast<int32_t*>(smem + L.o_flags);
  uint32_t* s_stay = reinterpret_cast<uint32_t*>(smem + L.o_stay);
  int32_t* s_amb = reinterpret_cast<int32_t*>(smem + L.o_amb);
  int32_t* s_tc2 = reinterpret_cast<int32_t*>(smem + L.o_tc);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L.o_bar);
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + L.o_ctl);
  const int RAWW = L.RAWW, WT = L.WT, BLK = L.BLK, NOWN = L.NOWN;
  const int4* tw = (w.n_tw <= TW_SMEM) ? s_tw : w.tw;
  // Per-thread step constants, fixed for the launch, so that no runtime integer division sits on
  // the step's critical path: the owner pass-1 item i = tid + j*NT as (owned action oa, item r2 of
  // its W*NTAU) and the goal/terrain item (owned action, substep) of the FIX loop, both advanced
  // round by round without dividing.
  const int p1_oa0 = tid / WT, p1_r20 = tid - p1_oa0 * WT;
  const int p1_da = NT / WT, p1_dr = NT - p1_da * WT;
  const int fx_i0 = (2 * NT - 33 - tid) % NT;  // the second-last warp first (see the FIX loop)
  const int fx_oa0 = fx_i0 / W, fx_l0 = fx_i0 - fx_oa0 * W;
  const int fx_da = NT / W, fx_dl = NT - fx_da * W;
  const int col_l = col_t - 1;  // this column's substep index (col % W for col < NCOL)
  // plan-sharded multi-GPU step: xmode 1 exports this GPU's per-(state, tau)
  // minima and nearest-plan distance, xmode 2 imports their all-reduced minimum and decides
  // MODE 2: in-kernel exchange with the peer GPUs (xmode 3), no host round-trip per step;
  // MODE 3: the reference / debug instantiation -- the host-stepped exchange (xmode 1 export /
  // 2 import) and fmdp_eval_step's one-step evaluation.  MODE 0 / 1 / 2 carry neither (measured:
  // their code on the step path costs 1.7 % full / 3.4 % culled on the configs[1] batch).
  constexpr bool XP = MODE == 2;
  const int xmode = XP ? 3 : (MODE == 3 ? args.xmode : 0);
  const bool evalm = (MODE == 3 || MODE == 5) && args.eval;
  // SURVEY f1 culling: MODE 4 is the culled FCFS walker, MODE 0 the full one (each carries only
  // its own build pass); the other instantiations decide at run time
  // MODE 6 = the culled FCFS walker with the range query (large rows; a separate instantiation so
  // that MODE 4 carries none of its code: measured, its branches cost the 3000-plan step 10 %)
  constexpr bool CULLW = MODE == 4 || MODE == 6;
  const bool cullm = CULLW ? true : (MODE == 0 ? false : args.cull != 0);
  // SURVEY f1 range query: the culled FCFS walker stages only the 3x3 cells around the ownship
  constexpr bool IDX = MODE == 6;
  // SURVEY f2 co-simulated batch: a separate instantiation, so the FCFS walker carries no
  // co-simulation code at all (measured: any of it on the step path costs ~1.5 %)
  const int cosim = MODE == 1 ? 1 : 0;
  // x_intra: the launch's clusters are the ranks (one GPU, one request split over several
  // clusters); otherwise this launch is rank x_me of a multi-GPU exchange
  const int xcl = (XP && args.x_intra) ? (int)(blockIdx.x / G) : wcl;
  const int xme = (XP && args.x_intra) ? xcl : args.x_me;
  // two-level exchange (x_inter): the clusters of this GPU first (xme / x_world, above), then
  // cluster xcl of every GPU (rank x_ime of x_iworld) over NVLink
  const bool xinter = XP && args.x_inter;
  const bool lead = xcl == 0;  // writes the request's outputs (every cluster decides the same)
  const int srank = (XP && args.x_intra) ? args.shard_rank + xcl : args.shard_rank;
  // plan shards exist only in the exchange instantiations (MODE 2 / 3): the FCFS walkers stage
  // whole rows, without the shard's 64-bit divisions in their code
  const int sworld = (MODE == 2 || MODE == 3) ? args.shard_world : 1;
  const unsigned long long xseq0 = XP ? args.x_seq[xcl] : 0ull;  // step tags continue across launches
  unsigned long long xit = 0;

  // per-phase cycle accounting: only in the reference instantiation (MODE 3; a profiled FCFS
  // walk runs there) -- its marks cost up to 6 % of a latency-bound step elsewhere
#ifndef FMDP_PROF_TID  // A/B builds (tools/ab_variants.py) may profile another thread's view of the step
#define FMDP_PROF_TID 0
#endif
  const bool prof = MODE == 3 && args.prof != nullptr && rank == 0 && tid == (FMDP_PROF_TID < 0 ? NT + FMDP_PROF_TID : FMDP_PROF_TID);
  unsigned long long pacc[PH_N];
#pragma unroll
  for (int i = 0; i < PH_N; ++i) pacc[i] = 0;
  long long tmark = 0;
#define FMDP_MARK(ph)                               \
  if (prof) {                                       \
    const long long now_ = clock64();               \
    pacc[ph] += (unsigned long long)(now_ - tmark); \
    tmark = now_;                                   \
  }

  for (int i = tid; i < w.HL; i += NT) s_dxy[i] = w.dxy[i];
  if (w.n_tw <= TW_SMEM)
    for (int i = tid; i < w.n_tw; i += NT) s_tw[i] = w.tw[i];
  if (tid == 0) {
    for (int b = 0; b < 7; ++b) mbar_init(&s_bar[b], 1);  // 0-2 TMA ring, 3-4 reduce-scatter, 5-6 V*
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (XP && tid < args.x_world) ctl->xp[tid] = args.x_peers[tid].recv;
  if (xinter && tid < args.x_iworld) ctl->xip[tid] = args.x_ipeers[xcl * XNODE + tid].recv;
  // every CTA of the cluster has started and initialised its mbarriers before any DSMEM access
  // (the first request's broadcast below wrote into CTAs that might not have entered yet:
  // compute-sanitizer racecheck, profiles/r02_sanitizer.md)
  cluster.sync();
  uint32_t par = 0;      // next wait parity per ring buffer (bit b)
  uint32_t parX = 0;     // next wait parity of the exchange mbarriers: bits 0-1 reduce-scatter, 2-3 V*
  uint32_t pending = 0;  // ring buffers issued and not yet waited
  int cnt2 = 0;          // (I/O thread NT-1) active count of row K+2, loaded one step ahead
  uint32_t stop_f = 0;   // (I/O thread of rank 0) the head-finished flag, loaded one step ahead

  for (;;) {
    // ------------------------------------------------------------ next request
    if (rank == 0 && tid == 0) {
      int r = atomicAdd(args.queue + xcl, 1);
      for (unsigned b = 0; b < G; ++b) peer_ptr(cluster, &ctl->req, b, solo)[0] = r;
    }
    cluster.sync();
    const int r = *(volatile int32_t*)&ctl->req;
    if (r >= args.n_reqs) break;
    const Req rq = args.reqs[r];
    const size_t sbase = (size_t)rq.slot * args.cap;
    if (cosim) {  // keep the batch clock until this aircraft departs
      if (rank == 0 && rq.t0 > args.cs_k0)
        cs_idle(args.cs_pub, args.cs_arrive, args.cs_err, args.cs_n, args.cs_k0, ctl, r, args.cs_k0, rq.t0, CS_ABSENT,
                false);
      cluster.sync();
    }
    // walker state, identical in every thread of every CTA of the cluster
    int k = rq.start_k;
    int qx, qy, qz, psi, v = rq.speed0 > 0 ? rq.speed0 : w.v0;  // v: speed, the wide walker's extra state
    if (k == 0) {
      qx = rq.src[0]; qy = rq.src[1]; qz = rq.src[2];
      psi = rq.psi0;
    } else {
      const int32_t* tq = args.traj + 3 * (sbase + k);
      qx = tq[0]; qy = tq[1]; qz = tq[2];
      psi = args.heading[sbase + k];
      if (WIDE) v = args.speed[sbase + k];
    }
    unsigned wit = 0;  // wide walker: decision-board steps of this request (tags 1, 2, ...)
    // per-request aggregates, kept by thread 0 of rank 0
    int n_near = 0, steps_run = 0, status = 0, fail_step = -1, nex0 = 0;
    bool reconv = false;  // the re-walk met its previous run (Req::n_old): the rest is that run's
    // pre-cull (culled FCFS walker): this thread's survivors among its plans of the next step's
    // first chunk, culled during this step's V* exchange (plan indices, -1: none); sv_n = their
    // count (> 2: the thread re-culls its plans in the step; < 0: no pre-cull for the next step)
    int sv0 = -1, sv1 = -1, sv_n = -1;
    // re-convergence window: decisions k with reuse_from <= k + 1 < n_old compare their next state
    // (only the culled FCFS walker and the reference instantiation carry it: measured, the full
    // walker's batches gain nothing from it and its step loop would grow, +1.3 % per step)
    constexpr bool REUSE = CULLW || MODE == 3;
    const int bk_lo = (REUSE && args.bak != nullptr && rq.n_old > 0 && !evalm) ? rq.reuse_from - 1 : INT_MAX;
    const int bk_hi = rq.n_old - 1;
    uint32_t min_sep = w.sat_d2;
    if (tid == 0) {
      // terminal flags of the starting state (terrain, goal; timeout cannot apply: k < max_steps)
      const int h = ground_height(w, qx, qy);
      const int64_t gx = (int64_t)qx - rq.dst[0], gy = (int64_t)qy - rq.dst[1], gz = (int64_t)qz - rq.dst[2];
      ctl->fl0 = ((qz < 0 || qz < h) ? 1 : 0) | ((gx * gx + gy * gy + gz * gz < w.cap2) ? 2 : 0);
      ctl->ntc[0] = ctl->ntc[1] = 0;
      ctl->namb[0] = ctl->namb[1] = 0;
      ctl->stay_local[0] = ctl->stay_local[1] = w.sat_d2;
      ctl->nsurv[0] = ctl->nsurv[1] = ctl->nsurv[2] = ctl->nsurv[3] = 0;
      ctl->n_exact = 0;
      ctl->rc_near = ctl->rc_exact = 0;
      ctl->rc_min = w.sat_d2;
      if (rank == 0 && k > 0 && !evalm) {  // resume: aggregates of the kept prefix
        for (int kk = 0; kk < k; ++kk) {
          n_near += args.ntie[sbase + kk];
          min_sep = min(min_sep, args.stepd2[sbase + kk]);
          if (args.stepx) nex0 += args.stepx[sbase + kk];
        }
      }
      if (lead && rank == 0 && k == 0 && !evalm) {
        int32_t* tq = args.traj + 3 * sbase;
        tq[0] = rq.src[0]; tq[1] = rq.src[1]; tq[2] = rq.src[2];
        args.heading[sbase] = rq.psi0;
        if (WIDE) args.speed[sbase] = w.v0;
        if (cosim)  // departure: level flight along the initial heading (R28)
          cs_publish(args, r, rq.t0, qx, qy, qz, CS_PRESENT, s_dxy[psi].x, s_dxy[psi].y, 0);
      }
      const int64_t K0 = rq.t0 + k;
      if (IDX) {
        int lo[4], hi[4];
        load_ranges(w, K0, qx, qy, lo, hi);
        issue_row_idx(w, K0, lo, hi, rank, lgG, RAWCAP, s_raw, RAWW, s_bar, ctl);
        load_ranges(w, K0 + 1, qx, qy, lo, hi);
        issue_row_idx(w, K0 + 1, lo, hi, rank, lgG, RAWCAP, s_raw, RAWW, s_bar, ctl);
      } else {
        const int n0 = row_count(w, K0), n1 = row_count(w, K0 + 1);
        issue_row(w, K0, n0, rank, lgG, RAWCAP, s_raw, RAWW, s_bar, ctl, srank, sworld);
        issue_row(w, K0 + 1, n1, rank, lgG, RAWCAP, s_raw, RAWW, s_bar, ctl, srank, sworld);
      }
    }
    {
      const int64_t K0 = rq.t0 + k;
      pending |= (1u << (K0 % 3)) | (1u << ((K0 + 1) % 3));
      if (tid == NT - 1) {  // the I/O thread's row count (range query: candidate ranges), one step ahead
        cnt2 = row_count(w, K0 + 2);
        if (IDX) {
          int lo[4], hi[4];
          load_ranges(w, K0 + 2, qx, qy, lo, hi);
          for (int i = 0; i < 4; ++i) {
            ctl->ilo[i] = lo[i];
            ctl->ihi[i] = hi[i];
          }
        }
      }
    }
    __syncthreads();
    // terrain candidates (exact cull: the wells that can reach a projected state) of the next
    // TC_WIN steps: radius R + reach + TC_WIN substep reaches around q (the ownship moves at most
    // one substep reach per step), so one scan serves steps k .. k + TC_WIN; rescanned when the
    // window runs out (list buffer tcb; the other one is filled by the rescan)
    int tcb = 0, tc_end = k + TC_WIN;
    {
      const int64_t grow = (int64_t)w.reach_u + (int64_t)TC_WIN * w.step_reach_u;
      for (int i = tid; i < w.n_tw; i += NT) {
        const int4 t = tw[i];
        const int64_t dx = t.x - qx, dy = t.y - qy, dz = t.z - qz;
        const int64_t rr = (int64_t)t.w + grow;
        if (dx * dx + dy * dy + dz * dz < rr * rr) {
          const int slot = atomicAdd(&ctl->ntc[0], 1);
          if (slot < TC_MAX) s_tc2[slot] = i;
        }
      }
    }
    int fl = ctl->fl0;
    bool fin = !evalm && fl != 0;  // only the separation test of state k remains
    cluster.sync();

    // ------------------------------------------------------------ step loop
    int bK = (int)((rq.t0 + k) % 3);  // ring buffer of row K = t0 + k (advanced with k, no 64-bit modulo per step)
    for (;;) {
      if (prof) tmark = clock64();
      const int64_t K = rq.t0 + k;
      const int p = k & 1;
      const int bK2 = bK == 0 ? 2 : bK - 1;  // (K + 2) % 3
      // re-convergence window (a10): the previous run's state k + 1 -> shared memory (one 16-byte
      // LDGSTS, waited before the post-stage barrier), compared with the decision's next state
      const bool bak_act = REUSE && k >= bk_lo && k < bk_hi && !fin;
      if (bak_act && tid == NT - 2) cp_async16(&ctl->bakst[p], &args.bak[sbase + k + 1]);
      // the previous step's reduce-scatter copies (threads < G) must have read s_stage before this
      // step stages into it again (long done: the owner pass and the V* exchange came in between)
      if (!solo && tid < (int)G) bulk_wait_read();
      int4* s_pos = s_pos2 + p * AW;
      // fan origin of this step's projected states (hot-loop formulation)
      const int ox = (W >> 1) * s_dxy[psi].x, oy = (W >> 1) * s_dxy[psi].y;
      if (!evalm && !fin) pending |= 1u << bK2;  // row K+2: issued below by the I/O thread
      FMDP_MARK(PH_TOP)

      float sx = 0.f, sy = 0.f, sz[C];
      f2 sx2 = 0, sy2 = 0, sz2[C];
#pragma unroll
      for (int c = 0; c < C; ++c) sz2[c] = 0;
      int x1 = 0, y1 = 0;  // Delta_1 of this turn (t = 1 columns, group 0)
      // ---- a1 + a4: stage row K, wells, hot loop; exact nearest-plan distance of q ("stay")
      float m[C][NTAU];
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int t = 0; t < NTAU; ++t) m[c][t] = FLT_MAX;
      if (pending & (1u << bK)) {
        mbar_wait(&s_bar[bK], (par >> bK) & 1u);
        par ^= 1u << bK;
        pending &= ~(1u << bK);
      }
      FMDP_MARK(PH_WAIT)
      uint32_t stay = w.sat_d2;
      const int svn_now = sv_n;  // this step's first chunk was pre-culled in the previous step
      sv_n = -1;
      {
        const int lo = ctl->sl_lo[bK], n = ctl->sl_n[bK];
        // plan j of the CTA slice: the first RAWCAP were staged by TMA, the rest are read from L2
        const int32_t* rb = s_raw + (size_t)bK * 4 * RAWW + ctl->sl_off[bK];
        const int32_t* rg = w.rows + (size_t)K * 4 * w.row_cap + lo;
        const int SC = cullm ? RAWCAP : CH;  // plans per build pass
        const ulonglong2* cen2 = reinterpret_cast<const ulonglong2*>(s_cen);

        // Build pass over plans [c0, c0+nc) of the slice: exact nearest-plan distance (stay);
        // well records of every plan (compact == false: slot = plan) or, with f1 culling, only
        // of plans one of whose wells can reach a projected state (|q - c_tau| < R_tau + reach +
        // 1 unit, conservative FP32 test; a culled well is farther than R_tau from every state
        // by at least one unit, i.e. clearly outside the FP32 band, so the minima that decide
        // the values are unchanged).  Survivors are compacted, order-free; slot >= CH overflows.
        auto build = [&](int c0, int nc, bool compact, int* counter) {
          for (int j0 = 0; j0 < nc; j0 += NT) {
            const int jj = j0 + tid;
            const bool valid = jj < nc;
            const int j = c0 + jj;
            int rx = 0, ry = 0, rz = 0, vx = 0, vy = 0, vz = 0;
            if (valid) {
              uint32_t pv;
              if (IDX) {
                const int4 P = plan_at(w, ctl, s_raw, RAWW, bK, K, j);
                rx = P.x - qx; ry = P.y - qy; rz = P.z - qz;
                pv = (uint32_t)P.w;
              } else if (j < RAWCAP) {
                rx = rb[j] - qx; ry = rb[RAWW + j] - qy; rz = rb[2 * RAWW + j] - qz;
                pv = (uint32_t)rb[3 * RAWW + j];
              } else {
                rx = __ldg(&rg[j]) - qx; ry = __ldg(&rg[w.row_cap + j]) - qy; rz = __ldg(&rg[2 * w.row_cap + j]) - qz;
                pv = (uint32_t)__ldg(&rg[3 * w.row_cap + j]);
              }
              stay = min(stay, clamp_d2(rx, ry, rz, w.R_max, w.sat_d2));
              vx = sext(pv, 11); vy = sext(pv >> 11, 11); vz = sext(pv >> 22, 10);
            }
            if (fin) continue;
            bool keep = valid;
            if (valid && compact) keep = cull_keep(w, rx, ry, rz, vx, vy, vz);
            int slot = jj;
            if (compact && keep) slot = atomicAdd(counter, 1);  // survivors are rare: no warp round trip
            if (keep && slot < CH) {
              // plan pair layout: [pair][tau][X_j, X_j', Y_j, Y_j', Z_j, Z_j', Q_j, Q_j']: X = o - c
              // (exact integers < 2^24, R23) and Q = |X|^2 (FP32, DESIGN.md §7 error bound)
              float* cp = s_cen + PAIR_STRIDE * (slot >> 1) + (slot & 1);
#pragma unroll
              for (int t = 0; t < NTAU; ++t) {
                const float X = (float)(ox - (rx + w.k_tau[t] * vx));
                const float Y = (float)(oy - (ry + w.k_tau[t] * vy));
                const float Z = (float)(-(rz + w.k_tau[t] * vz));
                cp[8 * t + 0] = X;
                cp[8 * t + 2] = Y;
                cp[8 * t + 4] = Z;
                cp[8 * t + 6] = fmaf(Z, Z, fmaf(Y, Y, X * X));
              }
            }
          }
        };
        // Hot loop over ns well records (two plans per packed instruction).
        auto hot_loop = [&](int ns, auto zero_mid) {
          // zero_mid: the middle climb is level flight, so its FFMA2 (0 * Z + h) is exactly h
          // and is skipped -- bit-identical, one FFMA2 per tau and plan pair fewer
          constexpr bool ZM = decltype(zero_mid)::value;
          // (state, well) pair: |s - c|^2 - |s - o|^2 = Q + 2(s-o).X, the horizontal part
          // shared by the C climbs (2 FFMA2), one FFMA2 per climb; FMNMX3 folds both plans of a
          // pair into the running minimum (|s - o|^2 is added back by the owner)
// One plan pair, all five wells, ordered by the shared operand (sx2, then sy2, then each
// climb's sz2) so that consecutive FFMA2s are independent and reuse one register operand.
#define FMDP_PAIR(E)                                                                   \
  {                                                                                    \
    f2 h_[NTAU];                                                                       \
    _Pragma("unroll") for (int t_ = 0; t_ < NTAU; ++t_) h_[t_] = fma2(sx2, (E)[2 * t_].x, (E)[2 * t_ + 1].y); \
    _Pragma("unroll") for (int t_ = 0; t_ < NTAU; ++t_) h_[t_] = fma2(sy2, (E)[2 * t_].y, h_[t_]);           \
    _Pragma("unroll") for (int cc_ = 0; cc_ < C; ++cc_)                                \
      _Pragma("unroll") for (int t_ = 0; t_ < NTAU; ++t_)                              \
        m[cc_][t_] = min3(m[cc_][t_], (ZM && cc_ == C / 2) ? h_[t_]                    \
                                                           : fma2(sz2[cc_], (E)[2 * t_ + 1].x, h_[t_])); \
  }
          const int npf = ns >> 1;  // full pairs; an odd tail is peeled below
          // the first tau's two records of the next pair load while this pair computes, so the
          // first FFMA2 chain starts without waiting on shared memory (a full 10-record prefetch
          // spills: measured slower)
          const int cstep = (PAIR_STRIDE / 4) * NGW;
          const ulonglong2* c8 = cen2 + (PAIR_STRIDE / 4) * grp;
          ulonglong2 n0 = make_ulonglong2(0, 0), n1 = make_ulonglong2(0, 0);
          if (grp < npf) {
            n0 = c8[0];
            n1 = c8[1];
          }
          if constexpr (C >= 10) {
            // ten climbs per thread (wide walker): 50 running minima leave no room for all ten
            // records of a pair, so the loop streams them tau by tau -- the next tau's two records
            // load while this tau's 21 instructions (2 + 9 FFMA2, 10 FMNMX3) run
            for (int pp = grp; pp < npf; pp += NGW, c8 += cstep) {
              ulonglong2 r0 = n0, r1 = n1;
#pragma unroll
              for (int t_ = 0; t_ < NTAU; ++t_) {
                ulonglong2 q0 = r0, q1 = r1;
                if (t_ + 1 < NTAU) {
                  q0 = c8[2 * t_ + 2];
                  q1 = c8[2 * t_ + 3];
                } else if (pp + NGW < npf) {
                  q0 = c8[cstep];
                  q1 = c8[cstep + 1];
                }
                f2 hh = fma2(sx2, r0.x, r1.y);
                hh = fma2(sy2, r0.y, hh);
#pragma unroll
                for (int cc_ = 0; cc_ < C; ++cc_)
                  m[cc_][t_] = min3(m[cc_][t_], (ZM && cc_ == C / 2) ? hh : fma2(sz2[cc_], r1.x, hh));
                r0 = q0;
                r1 = q1;
              }
              n0 = r0;
              n1 = r1;
            }
          } else {
            for (int pp = grp; pp < npf; pp += NGW, c8 += cstep) {
              ulonglong2 e[10];
              e[0] = n0;
              e[1] = n1;
#pragma unroll
              for (int i = 2; i < 10; ++i) e[i] = c8[i];
              if (pp + NGW < npf) {
                n0 = c8[cstep];
                n1 = c8[cstep + 1];
              }
              FMDP_PAIR(e)
            }
          }
          if ((ns & 1) && (npf & (NGW - 1)) == grp) {  // odd tail (NGW a power of two): partner = a well at infinity
            const ulonglong2* t8 = cen2 + (PAIR_STRIDE / 4) * npf;
            ulonglong2 e[10];
#pragma unroll
            for (int i = 0; i < 10; ++i) {
              e[i] = t8[i];
              if (i & 1) {
                e[i].x = hi_set(e[i].x, 0.f);
                e[i].y = hi_set(e[i].y, 3.0e18f);
              } else {
                e[i].x = hi_set(e[i].x, 0.f);
                e[i].y = hi_set(e[i].y, 0.f);
              }
            }
            FMDP_PAIR(e)
          }
#undef FMDP_PAIR
          if (tid == 0 && args.pairs) atomicAdd(args.pairs, (unsigned long long)ns * NTAU * AW);
        };
        auto hot = [&](int ns) {
          if (w.zero_climb == C / 2) hot_loop(ns, std::true_type{});
          else hot_loop(ns, std::false_type{});
        };

        // batch peers at clock K (Alg 5, P^- of Table DS), five wells each, staged
        // as one more chunk after the row's (same records, same hot loop); this CTA takes peers
        // j = rank + i*G.  The clock wait sits after the row's hot loop, overlapping it.
        auto build_peers = [&]() -> int {
          // (a failed wait sets cs_err: the host discards the batch; later waits return at once)
          cs_wait(args, K);  // every warp (a failed wait sets cs_err; the host discards the batch)
          __syncthreads();
          const int npr = args.cs_n > (int)rank ? (args.cs_n - (int)rank + (int)G - 1) / (int)G : 0;
          TauSteps kt;
#pragma unroll
          for (int t = 0; t < NTAU; ++t) kt.k[t] = w.k_tau[t];
          stay = min(stay, cs_build_peers(args.cs_pub + (size_t)(K & 1) * args.cs_n * 2, npr, (int)rank, (int)G, r, qx,
                                          qy, qz, ox, oy, !fin, s_cen, w.R_max, w.sat_d2, kt));
          return npr;
        };

        const int n_chunks = xmode == 2 ? 0 : (n <= SC ? (n > 0 ? 1 : 0) : (n + SC - 1) / SC);
        // the first chunk's well records are built BEFORE the projection: the build needs only q,
        // the fan origin and row K (staged two steps ahead), so it overlaps the projection's
        // table load, and the projection barrier also publishes the records (one CTA barrier less)
        if (CULLW && n_chunks > 0 && svn_now >= 0) {
          // pre-culled first chunk (plans j < RAWCAP, staged): the separation minimum over every
          // plan, records (with this step's anchor) of the thread's pre-culled survivors only
          const int nc0 = min(SC, n);
          for (int jj = tid; jj < nc0; jj += NT) {
            const int4 P = IDX ? plan_at(w, ctl, s_raw, RAWW, bK, K, jj) : make_int4(rb[jj], rb[RAWW + jj], rb[2 * RAWW + jj], 0);
            stay = min(stay, clamp_d2(P.x - qx, P.y - qy, P.z - qz, w.R_max, w.sat_d2));
          }
          if (!fin) {
            int* counter = &ctl->nsurv[(k & 1) * 2];
            auto rec = [&](int j, bool test) {
              const int4 P = IDX ? plan_at(w, ctl, s_raw, RAWW, bK, K, j)
                                 : make_int4(rb[j], rb[RAWW + j], rb[2 * RAWW + j], rb[3 * RAWW + j]);
              const int rx = P.x - qx, ry = P.y - qy, rz = P.z - qz;
              const uint32_t pv = (uint32_t)P.w;
              const int vx = sext(pv, 11), vy = sext(pv >> 11, 11), vz = sext(pv >> 22, 10);
              if (test && !cull_keep(w, rx, ry, rz, vx, vy, vz)) return;
              const int slot = atomicAdd(counter, 1);
              if (slot < CH) {
                float* cp = s_cen + PAIR_STRIDE * (slot >> 1) + (slot & 1);
#pragma unroll
                for (int t = 0; t < NTAU; ++t) {
                  const float X = (float)(ox - (rx + w.k_tau[t] * vx));
                  const float Y = (float)(oy - (ry + w.k_tau[t] * vy));
                  const float Z = (float)(-(rz + w.k_tau[t] * vz));
                  cp[8 * t + 0] = X;
                  cp[8 * t + 2] = Y;
                  cp[8 * t + 4] = Z;
                  cp[8 * t + 6] = fmaf(Z, Z, fmaf(Y, Y, X * X));
                }
              }
            };
            if (svn_now > 2) {
              for (int jj = NT - 1 - tid; jj < nc0; jj += NT) rec(jj, true);
            } else {
              if (sv0 >= 0) rec(sv0, false);
              if (sv1 >= 0) rec(sv1, false);
            }
          }
        } else if (n_chunks > 0) {
          build(0, min(SC, n), cullm, &ctl->nsurv[(k & 1) * 2]);
        }
        FMDP_MARK(PH_BUILD)
        if (!fin) {
          // ---- a5 candidates of steps k+1 .. k+1+TC_WIN when this list's window ends with step k
          //      (rescan from q_k: every later state within the window is at most TC_WIN substep
          //      reaches away) into the other list buffer, switched to after the hot loop
          if (k + 1 > tc_end) {
            const int64_t grow = (int64_t)w.reach_u + (int64_t)(TC_WIN + 1) * w.step_reach_u;
            for (int i = tid; i < w.n_tw; i += NT) {
              const int4 t = tw[i];
              const int64_t dx = t.x - qx, dy = t.y - qy, dz = t.z - qz;
              const int64_t rr = (int64_t)t.w + grow;
              if (dx * dx + dy * dy + dz * dz < rr * rr) {
                const int slot = atomicAdd(&ctl->ntc[tcb ^ 1], 1);
                if (slot < TC_MAX) s_tc2[(tcb ^ 1) * TC_MAX + slot] = i;
              }
            }
          }
          FMDP_MARK(PH_SCAN)
          // ---- a2 forward projection (Alg 3): column (turn it, substep t) on the integer lattice
          const int it = col_it, t = col_t, h = col_h;
          // cumulative lattice displacement of (psi, turn, t) from the host-built table (one L2 load
          // instead of t dependent lattice steps); final heading psi + t*h mod HL
          int x, y, ps;
          if (WIDE) {  // R32: psi_s = psi + s h, v_s = clamp(v + s acc), q_t = q + sum_{s<=t} D(psi_s, v_s)
            int xx = qx, yy = qy, pp = psi, sp = v;
            for (int s2 = 1; s2 <= W; ++s2) {
              const int pn = pp + col_hw;
              const int pw2 = pn >= w.HL ? pn - w.HL : (pn < 0 ? pn + w.HL : pn);
              const int sn = min(max(sp + col_acc, w.vmin), w.vmax);
              if (s2 <= t) {
                const int2 d = __ldg(&w.spd[(size_t)(sn - w.vmin) * w.HL + pw2]);
                xx += d.x;
                yy += d.y;
                pp = pw2;
                sp = sn;
              }
            }
            x = xx;
            y = yy;
            ps = pp | (sp << 16);  // heading and speed of the state (s_pos .w)
          } else {
            const int2 cum = __ldg(&w.proj[((size_t)psi * w.n_turn + it) * W + (t - 1)]);
            x = qx + cum.x;
            y = qy + cum.y;
            ps = psi + t * h;  // |t h| < HL (checked by the host): one wrap at most
            ps += ps < 0 ? w.HL : (ps >= w.HL ? -w.HL : 0);
          }
          // offsets from the fan origin o = q + (W/2) (DX, DY)[psi], doubled: the hot loop
          // evaluates |s - c|^2 - |s - o|^2 = Q + 2 (s - o).X with X = o - c, Q = |X|^2
          sx = (float)(2 * (x - qx - ox));
          sy = (float)(2 * (y - qy - oy));
  #pragma unroll
          for (int c = 0; c < C; ++c) sz[c] = (float)(2 * w.climb[c] * t);
          sx2 = pk2(sx, sx);
          sy2 = pk2(sy, sy);
  #pragma unroll
          for (int c = 0; c < C; ++c) sz2[c] = pk2(sz[c], sz[c]);
          if (grp == 0 && col < NCOL) {
  #pragma unroll
            for (int c = 0; c < C; ++c) s_pos[(it * C + c) * W + (t - 1)] = make_int4(x, y, qz + w.climb[c] * t, ps);
            if (t == 1) {  // raster load in flight during the hot loop (LDGSTS), consumed after it
              const int32_t* cell = ground_cell(w, x, y);
              if (cell) cp_async4(&ctl->hgt[it], cell);
              else ctl->hgt[it] = INT_MIN;
              x1 = x;
              y1 = y;
            }
          }
          FMDP_MARK(PH_PLOOP)
          __syncthreads();
          FMDP_MARK(PH_PROJ)
          // ---- a3 goal (fp64), deck, a5 terrain (exact predicate, FP32 ex2 value): owned states.
          //      Taken from the second-last warp downwards: the first threads carry the build pass
          //      of the row slice, and the last warp holds the I/O thread (its row-count load and
          //      TMA issue would serialise with divergent FIX lanes of the same warp), so the fp64
          //      latency overlaps the row wait and the build (measured: the FIX lanes sharing the
          //      I/O thread's warp were the step's last arrivals)
          const int ntc = ctl->ntc[tcb];
          const int32_t* s_tc = s_tc2 + tcb * TC_MAX;
          for (int i = fx_i0, foa = fx_oa0, fl_ = fx_l0; i < n_own * W; i += NT) {
            const int st = ((int)rank + foa * (int)G) * W + fl_;
            foa += fx_da;
            fl_ += fx_dl;
            if (fl_ >= W) {
              fl_ -= W;
              ++foa;
            }
            const int4 q4 = s_pos[st];
            // fp64: exact integer d^2 < 2^52, correctly rounded sqrt, exp2 within an ulp
            // -- agrees with the oracle's pow to ~1e-15, so the level / climb near-ties of the goal
            // term (gaps ~1e-7 relative at 10 km) are decided as the oracle does
            const double gx = (double)(q4.x - rq.dst[0]), gy = (double)(q4.y - rq.dst[1]), gz = (double)(q4.z - rq.dst[2]);
  #ifdef FMDP_AB_GOAL32  // A/B only: the round-1 FP32 goal term, to measure what fp64 costs
            const double vpos = (double)(w.goal_rf * ex2_approx(w.goal_l2gf * sqrtf((float)fma(gz, gz, fma(gy, gy, gx * gx)))));
  #else
            const double vpos = w.goal_r * exp2(w.goal_l2g * sqrt(fma(gz, gz, fma(gy, gy, gx * gx))));
  #endif
            const double valt = (q4.z < w.zdeck_u) ? (w.deck_scale - w.u_m * (double)q4.z) : 0.0;
            int64_t mT = INT64_MAX;
#ifdef FMDP_AB_NOTERR  // A/B timing only: no terrain candidates (wrong values)
            const int nt = 0;
#else
            const int nt = ntc <= TC_MAX ? ntc : w.n_tw;
#endif
            for (int c = 0; c < nt; ++c) {
              const int4 t4 = tw[ntc <= TC_MAX ? s_tc[c] : c];
              const int64_t dx = q4.x - t4.x, dy = q4.y - t4.y, dz = q4.z - t4.z;
              const int64_t d2 = dx * dx + dy * dy + dz * dz;
              if (d2 < (int64_t)t4.w * t4.w && d2 < mT) mT = d2;
            }
            s_vT[st] = (mT != INT64_MAX) ? w.terr_r * ex2_approx(w.terr_l2g * sqrtf((float)mT)) : 0.f;
            s_fix[st] = vpos - valt;
            s_sfix[st] = vpos + valt;
          }
          FMDP_MARK(PH_FIX)
        }

        // ---- per-step I/O, on the CTA's last thread after the projection barrier (thread 0 owns
        //      projection columns; this one has no build work in the latency-bound configurations):
        //      prefetch of row K+2 (its ring buffer last held row K-1, consumed in step k-1),
        //      this step's exchange phases -- slice minima (4 B from every CTA), reduce-scatter
        //      blocks of the owned actions (from every CTA), the stop flag (from rank 0), V*(a)
        if (tid == NT - 1) {
          if (!evalm && !fin) {
            if (IDX) {  // candidates around q_{k-1} for row K+2 (cell side covers the steps in between)
              cp_async_wait_all();  // the ranges fetched last step
              int lo[4], hi[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                lo[i] = ctl->ilo[i];
                hi[i] = ctl->ihi[i];
              }
              issue_row_idx(w, K + 2, lo, hi, rank, lgG, RAWCAP, s_raw, RAWW, s_bar, ctl);
              fetch_ranges_async(w, K + 3, qx, qy, ctl->ilo, ctl->ihi);
            } else {
              issue_row(w, K + 2, cnt2, rank, lgG, RAWCAP, s_raw, RAWW, s_bar, ctl, srank, sworld);
              cnt2 = row_count(w, K + 3);  // consumed next step: latency hidden by this step
            }
          }
          ctl->nsurv[((k + 1) & 1) * 2] = 0;  // step k+1, chunk 0 (last used in step k-1)
          const uint32_t bytesA = (xmode != 2 ? 4u * G : 0u) +
                                  ((!fin && xmode != 2 && !solo) ? (uint32_t)(4 * G * n_own * BLK) : 0u) +
                                  (args.stop ? 4u : 0u);
          mbar_arrive_tx(&s_bar[3 + p], bytesA);
          if (!fin) mbar_arrive_tx(&s_bar[5 + p], (uint32_t)(16 * A) + (XP ? 4u : 0u));
          if (args.stop && rank == 0) {  // one reading for the whole cluster
            // the value loaded in the previous step: the L2 round trip of the volatile load stays
            // off this warp's path (a walker may pause one step later -- speculation only)
            const uint32_t la = smem_u32(&ctl->stop[p]), lb = smem_u32(&s_bar[3 + p]);
            for (unsigned b = 0; b < G; ++b) push_u32(solo, la, b, stop_f, lb);
            stop_f = (uint32_t)*(volatile int32_t*)args.stop;
          }
        }

        for (int cidx = 0; cidx < n_chunks + cosim; ++cidx) {
          const int c0 = cidx * SC;
          const bool peers = cidx == n_chunks;
          int* counter = &ctl->nsurv[(k & 1) * 2 + (cidx & 1)];
          int nc;
          if (!peers) {
            nc = min(SC, n - c0);
            if (cidx > 0) build(c0, nc, cullm, counter);  // chunk 0: built before the projection
          } else {
            nc = build_peers();
          }
          if (fin) continue;
          if (cidx > 0 || peers) __syncthreads();
          const int ns = (cullm && !peers) ? *counter : nc;
          if (tid == 0) ctl->nsurv[(k & 1) * 2 + ((cidx + 1) & 1)] = 0;  // next pass's counter
          if (ns <= CH) {
            hot(ns);
            // the next pass rebuilds the records; after the last one nothing writes them before
            // the post-stage barrier, so a warp that is done goes on to its minima and staging
            if (cidx + 1 < n_chunks + cosim) __syncthreads();
          } else {  // more survivors than well records (rare): exact fallback, uncompacted
            __syncthreads();
            for (int m0 = c0; m0 < c0 + nc; m0 += CH) {
              const int mn = min(CH, c0 + nc - m0);
              build(m0, mn, false, counter);
              __syncthreads();
              hot(mn);
              __syncthreads();
            }
          }
        }
      }
      int tc_free = -1;  // the list consumed by this step's FIX: its counter is reset after the
      if (!fin && k + 1 > tc_end) {  // next CTA barrier (a step with an empty row slice has no
        tc_free = tcb;               // barrier between the FIX and this point: racecheck)
        tcb ^= 1;
        tc_end = k + 1 + TC_WIN;
      }
      // stay: slice minimum of |q - p(K)|^2 (terminal separation test of state k, Sec IV.I)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) stay = min(stay, __shfl_xor_sync(0xffffffffu, stay, o));
      if (lane == 0 && stay < w.sat_d2) atomicMin(&ctl->stay_local[p], stay);
      FMDP_MARK(PH_HOT)

      if (!fin) {
        FMDP_MARK(PH_FLAGS)
        // group minimum inside the warp (rounds over all C*NTAU values are unrolled so the shuffles
        // overlap), then the per-action blocks [t][tau] staged by owner CTA: s_stage[a mod G][a / G]
        if (CPW <= 8) {
#pragma unroll
          for (int c = 0; c < C; ++c)
#pragma unroll
            for (int t = 0; t < NTAU; ++t) m[c][t] = fminf(m[c][t], __shfl_xor_sync(0xffffffffu, m[c][t], 8));
        }
        if (CPW <= 16) {
#pragma unroll
          for (int c = 0; c < C; ++c)
#pragma unroll
            for (int t = 0; t < NTAU; ++t) m[c][t] = fminf(m[c][t], __shfl_xor_sync(0xffffffffu, m[c][t], 16));
        }
        if (grp == 0 && col < NCOL) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int a = col_it * C + c;
            float* dst = s_stage + ((a & (int)(G - 1)) * NOWN + (a >> lgG)) * BLK + col_l * NTAU;
#pragma unroll
            for (int t = 0; t < NTAU; ++t) dst[t] = m[c][t];
          }
          if (!solo) fence_proxy_async();  // staged blocks -> the bulk copies' (async proxy) reads
        }
        FMDP_MARK(PH_STAGE)
      }
      if (bak_act && tid == NT - 2) cp_async_wait_all();
      __syncthreads();
      if (tid == 0) {  // step k+1's counters: every warp has left step k-1 (this barrier)
        ctl->namb[p ^ 1] = 0;
        ctl->stay_local[p ^ 1] = w.sat_d2;
        if (tc_free >= 0) ctl->ntc[tc_free] = 0;  // every thread has finished this step's FIX
      }
      // slice separation minimum -> every CTA; reduce-scatter: thread o sends the run of owner o's
      // blocks as ONE bulk copy into s_recv[p][rank] of CTA o (completing on its mbarrier of this
      // parity; G = 1: the owner pass reads s_stage in place)
      const uint32_t barA = smem_u32(&s_bar[3 + p]);
      if (xmode != 2 && tid < (int)G) {
        push_u32(solo, smem_u32(&s_stay[p * 16 + rank]), tid, ctl->stay_local[p], barA);
        if (!fin && !solo) {
          const int n_own_o = (A > tid) ? (A - tid + (int)G - 1) >> lgG : 0;
          if (n_own_o > 0) {
            const uint32_t src = smem_u32(s_stage + tid * NOWN * BLK);
            const uint32_t dst = smem_u32(s_recv + ((p * (int)G + (int)rank) * NOWN) * BLK);
            bulk_s2c(mapa_u32(dst, tid), src, (uint32_t)(4 * n_own_o * BLK), mapa_u32(barA, tid));
            bulk_commit();
          }
        }
      }
      // terrain / goal flags of every action's Delta_1 (the candidate next state): read only after
      // the V* exchange, so computed here, off the path to the post-stage barrier (published by
      // the owner pass-1 barrier)
      if (!fin && grp == 0 && col < NCOL && col_l == 0) {
        const int it = col_it;
        cp_async_wait_all();
        const int hgt = ctl->hgt[it];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const int z = qz + w.climb[c];
          const int64_t gx = (int64_t)x1 - rq.dst[0], gy = (int64_t)y1 - rq.dst[1], gz = (int64_t)z - rq.dst[2];
          s_flags[it * C + c] = ((z < 0 || z < hgt) ? 1 : 0) | ((gx * gx + gy * gy + gz * gz < w.cap2) ? 2 : 0);
        }
      }
      // (one-CTA cluster: the pushes were plain stores of this CTA, all issued before this barrier,
      // so a CTA barrier orders them -- the form compute-sanitizer racecheck can follow; the phase
      // is still waited, as synccheck requires of every mbarrier phase)
      if (solo) __syncthreads();
      mbar_wait(&s_bar[3 + p], (parX >> p) & 1u);
      parX ^= 1u << p;
      FMDP_MARK(PH_BAR1)
      // exact nearest-plan d^2 of state k over the whole row (Sec IV.I): min of the slice minima
      uint32_t stay_all = w.sat_d2;
      if (xmode == 2) {
        stay_all = args.xbuf[NTAU * AW];  // all-reduced over the GPUs
      } else {
        // lane b reads source b's slice minimum (G <= 16), one REDUX per warp
        stay_all = __reduce_min_sync(0xffffffffu, lane < (int)G ? s_stay[p * 16 + lane] : w.sat_d2);
      }
      if (xmode == 1 && rank == 0 && tid == 0) args.xbuf[NTAU * AW] = stay_all;
      uint32_t xtag = 0;
      int xpar = 0;
      if (XP) {  // publish this GPU's nearest-plan d^2 to every peer (CTA 0)
        ++xit;
        xtag = (uint32_t)(xseq0 + xit);
        xpar = (int)((xseq0 + xit) & 1ull);
        if (rank == 0 && tid < args.x_world && tid != xme)  // lane q -> rank q
          st_ll(ctl->xp[tid] + x_word(xpar, args.x_world, xme, args.x_slot, args.x_slot - 16), stay_all, xtag);
        // one cluster per GPU: this value is already the GPU's -> the other GPUs right away
        if (xinter && args.x_world == 1 && rank == 0 && tid < args.x_iworld && tid != args.x_ime)
          st_ll(ctl->xip[tid] + x_word(xpar, args.x_iworld, args.x_ime, args.x_slot, args.x_slot - 16), stay_all, xtag);
        if (fin) {  // no owner epilogue in this step: CTA 0 collects the peers' values, broadcasts
          if (rank == 0 && warp == 0) {
            uint32_t m = x_stay_min(ctl->xp[xme], xme, args.x_world, args.x_slot, xpar, xtag,
                                    stay_all, args.x_err, x_budget(xit));
            if (xinter) m = x_stay_inter(ctl->xip, args.x_ime, args.x_iworld, args.x_slot, xpar, xtag, m, args.x_err,
                                         x_budget(xit), args.x_world > 1);
            if (lane < (int)G) peer_ptr(cluster, ctl, lane, solo)->xstay[p] = m;
          }
          cluster.sync();
          stay_all = ctl->xstay[p];
        }
      }
      if (!fin) {
        // ---- owner epilogue (half-warp per owned action, lane = substep): G-way minimum of
        //      the partial blocks, exact in/out, values (Alg 8), V*(a)
        // this step's partial blocks: [source CTA][slot][BLK] (G = 1: the CTA's own staged blocks)
        const float* rcv = solo ? s_stage : s_recv + p * (int)G * NOWN * BLK;
        // Pass 1 (whole CTA, one owned (action, substep, tau) per thread): G-way minimum of the
        // partial blocks (multi-GPU: export / import), |s - o|^2 added back, radius test ->
        // s_M = the in-radius d^2, FLT_MAX (outside), or -1 (inside the FP32 band: exact below).
        // s_M has its own buffer (the CTA's own bulk copies may still be reading s_stage).
        float* s_M = reinterpret_cast<float*>(smem + L.o_M);
        const int nitem = n_own * W * NTAU;
        if (XP) {  // this GPU's minima of the owned items -> every peer (all sends
                   // before any poll); each thread keeps its own items' minima in s_M
          for (int i = tid, oa = p1_oa0, r2 = p1_r20; i < nitem; i += NT) {
            const int io = ((int)rank + oa * (int)G) * WT + r2;  // (state, tau) index: st * NTAU + t
            const int oa_i = oa, r2_i = r2;
            oa += p1_da;
            r2 += p1_dr;
            if (r2 >= WT) {
              r2 -= WT;
              ++oa;
            }
            const float M = gway_min(rcv + oa_i * BLK + r2_i, (int)G, NOWN * BLK);
            s_M[i] = M;
            for (int q = 0; q < args.x_world; ++q)
              if (q != xme)
                st_ll(ctl->xp[q] + x_word(xpar, args.x_world, xme, args.x_slot, io), __float_as_uint(M),
                      xtag);
            if (xinter && args.x_world == 1)  // one cluster per GPU: straight to the other GPUs
              for (int q = 0; q < args.x_iworld; ++q)
                if (q != args.x_ime)
                  st_ll(ctl->xip[q] + x_word(xpar, args.x_iworld, args.x_ime, args.x_slot, io), __float_as_uint(M),
                        xtag);
          }
        }
        for (int i = tid, oa = p1_oa0, r2 = p1_r20; i < nitem; i += NT) {
          const int l = r2 / NTAU, t = r2 - l * NTAU;  // (constant divisor: multiply-shift)
          const int st = ((int)rank + oa * (int)G) * W + l;
          const int oa_i = oa, r2_i = r2;
          oa += p1_da;
          r2 += p1_dr;
          if (r2 >= WT) {
            r2 -= WT;
            ++oa;
          }
          float M;
          if (xmode == 2) {
            M = __uint_as_float(args.xbuf[st * NTAU + t]);
          } else if (XP) {  // this GPU's minimum (sent below) and the peers' minima
            M = x_min_peers(ctl->xp[xme], xme, args.x_world, args.x_slot, xpar, st * NTAU + t,
                            xtag, args.x_err, x_budget(xit), s_M[i]);
            if (xinter) {  // this GPU's minimum -> cluster xcl of every other GPU, then theirs
              const int io = st * NTAU + t;
              if (args.x_world > 1)  // (one cluster per GPU: sent with the first level above)
                for (int q = 0; q < args.x_iworld; ++q)
                  if (q != args.x_ime)
                    st_ll(ctl->xip[q] + x_word(xpar, args.x_iworld, args.x_ime, args.x_slot, io), __float_as_uint(M),
                          xtag);
              M = x_min_peers(ctl->xip[args.x_ime], args.x_ime, args.x_iworld, args.x_slot, xpar, io, xtag, args.x_err,
                              x_budget(xit), M);
            }
          } else {
            M = gway_min(rcv + oa_i * BLK + r2_i, (int)G, NOWN * BLK);
            if (xmode == 1) args.xbuf[st * NTAU + t] = __float_as_uint(M);  // this GPU's minima
          }
          const int4 q4 = s_pos[st];
          const int dx = q4.x - qx - ox, dy = q4.y - qy - oy, dz = q4.z - qz;
          M += (float)(dx * dx + dy * dy + dz * dz);  // exact integer < 2^24; one rounding
          float out = FLT_MAX;
          if (M < w.R2lo[t]) {
            out = M;
          } else if (M <= w.R2hi[t]) {
            out = -1.f;
            const int idx = atomicAdd(&ctl->namb[p], 1);
            if (idx < AMB_MAX) s_amb[idx] = i;
          }
          s_M[i] = out;
        }
        if (XP && rank == 0 && warp == 0) {  // -> every CTA with its V* pushes (one reader per value)
          uint32_t m = x_stay_min(ctl->xp[xme], xme, args.x_world, args.x_slot, xpar, xtag, stay_all,
                                  args.x_err, x_budget(xit));
          if (xinter) m = x_stay_inter(ctl->xip, args.x_ime, args.x_iworld, args.x_slot, xpar, xtag, m, args.x_err,
                                       x_budget(xit), args.x_world > 1);
          if (lane < (int)G)
            push_u32(solo, smem_u32(&ctl->xstay[p]), lane, m, smem_u32(&s_bar[5 + p]));
        }
#ifdef FMDP_AB_FINE  // A/B profiling only: the pass-1 loop itself, before its barrier ('projection' slot)
        FMDP_MARK(PH_PROJ)
#endif
        __syncthreads();
        FMDP_MARK(PH_OWN1)
        const int namb = ctl->namb[p];  // uniform after the barrier
        if (namb) {
          // Exact fallback: min over the WHOLE row K of the int64 d^2 for each flagged (state,
          // tau); each CTA resolves its own states (rare).  Out of line in the
          // full FCFS walker (smaller step code: -0.6 % batch time), inline elsewhere (measured:
          // the culled walker does not gain from the call)
          TauK tk;
#pragma unroll
          for (int t = 0; t < NTAU; ++t) {
            tk.k[t] = w.k_tau[t];
            tk.r2[t] = w.R2_tau[t];
          }
          const int32_t* rowg = w.rows + (size_t)K * 4 * w.row_cap;
          const int4* csK = cosim ? args.cs_pub + (size_t)(K & 1) * args.cs_n * 2 : nullptr;
          int32_t* sxk = (args.stepx && lead && !evalm) ? args.stepx + sbase + k : nullptr;
          if (MODE == 0)
            exact_fallback_call(s_M, s_amb, s_pos, namb, nitem, rowg, row_count(w, K), w.row_cap, (int)rank, (int)G,
                                W, tk, ctl, csK, args.cs_n, r, sxk);
          else
            exact_fallback(s_M, s_amb, s_pos, namb, nitem, rowg, row_count(w, K), w.row_cap, (int)rank, (int)G, W, tk,
                           ctl, csK, args.cs_n, r, sxk);
          if (tid == 0) ctl->namb[p] = 0;
        }
        // Pass 2 (half-warp per owned action, lane = substep): values (Alg 8), V*(a)
        const int hw = tid >> 4, hl = tid & 15;
        const int n_hw = NT >> 4;
        for (int oa0 = 0; oa0 < NOWN; oa0 += n_hw) {  // uniform trip count across the CTA
          if (oa0 + 2 * warp >= n_own) continue;     // (warp-uniform) no owned action in this warp
          const int oa = oa0 + hw;
          const int a = (int)rank + oa * (int)G;
          const bool act = oa < n_own && hl < W && a < A_tile;
          const int st = a * W + hl;
          float mi = FLT_MAX;
          if (act) {
#pragma unroll
            for (int t = 0; t < NTAU; ++t) mi = fminf(mi, s_M[(oa * W + hl) * NTAU + t]);
          }
          // a6 values
          double v = -INFINITY, sc = 0.0;
          if (act) {
            const float vI = (mi < FLT_MAX) ? w.intr_r * ex2_approx(w.intr_l2g * sqrtf(mi)) : 0.f;
            const double neg = (double)fmaxf(vI, s_vT[st]);
            v = s_fix[st] - neg;
            sc = s_sfix[st] + neg;
            if (evalm) {
              args.dbg_v[st + aoff * W] = v;
              args.dbg_s[st + aoff * W] = sc;
            }
          }
          // V*(a) = max(init, max_t V), term scale at the first maximising t: half-warp shuffles
          // (max of V over the half-warp, then the first substep attaining it by vote, then
          //  its scale: one double per shuffle round instead of two doubles and an index)
          double bv, bs;
          if (w.endpoint) {  // Alg 1: the value of the window's endpoint (R31)
            bv = __shfl_sync(0xffffffffu, v, (lane & 16) + W - 1);
            bs = __shfl_sync(0xffffffffu, sc, (lane & 16) + W - 1);
          } else {
            bv = v;
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) bv = fmax(bv, __shfl_xor_sync(0xffffffffu, bv, o, 16));
            const unsigned hit = (__ballot_sync(0xffffffffu, act && v == bv) >> (lane & 16)) & 0xffffu;
            bs = __shfl_sync(0xffffffffu, sc, (lane & 16) + (hit ? __ffs(hit) - 1 : 0));
          }
          if (oa < n_own && hl < (int)G) {  // push {V*(a), S(a)} to CTA hl
            const double vstar = (w.vmax_init_zero && !w.endpoint) ? fmax(0.0, bv) : bv;
            push_d2(solo, smem_u32(&s_vv[a]), hl, vstar, bs, smem_u32(&s_bar[5 + p]));
            if (evalm && hl == 0 && a < A_tile) args.dbg_vstar[a + aoff] = vstar;
            // parity trace of the walk itself (fmdp_set_trace): {V*(a), S(a)} of every step of
            // the first vtrace_n requests, in whichever instantiation runs them
            if (args.vtrace && hl == 0 && !evalm && rq.slot < args.vtrace_n && (WIDE ? a < A_tile : lead))
              args.vtrace[((size_t)rq.slot * args.cap + k) * (WIDE ? w.A_all : A) + a + aoff] = make_double2(vstar, bs);
          }
        }
        if (tid == 0 && ctl->n_exact && rank != 0) {
          atomicAdd(&cluster.map_shared_rank(ctl, 0)->n_exact, ctl->n_exact);
          ctl->n_exact = 0;
        }
        // Pre-cull (culled FCFS walker): the f1 cull test of the next row's first chunk (row K + 1,
        // staged two steps ahead) against this q, with the radius grown by one step's reach (host),
        // while the V* exchange is in flight; each thread keeps its survivors (at most two) for the
        // next step, which builds their records with its own anchor (no cross-thread dependence,
        // so no barrier).  The highest threads take the plans (the owner pass-2 warps are the
        // lowest).  Records of a superset of the relevant plans: results bit-identical.
        if (CULLW) {
          const int bK1 = bK == 2 ? 0 : bK + 1;
          if (pending & (1u << bK1)) {
            mbar_wait(&s_bar[bK1], (par >> bK1) & 1u);
            par ^= 1u << bK1;
            pending &= ~(1u << bK1);
          }
          const int nc1 = min(RAWCAP, ctl->sl_n[bK1]);
          const int32_t* rb1 = s_raw + (size_t)bK1 * 4 * RAWW + ctl->sl_off[bK1];
          int cnt = 0;
          sv0 = sv1 = -1;
          for (int jj = NT - 1 - tid; jj < nc1; jj += NT) {
            const int4 P = IDX ? plan_at(w, ctl, s_raw, RAWW, bK1, K + 1, jj)
                               : make_int4(rb1[jj], rb1[RAWW + jj], rb1[2 * RAWW + jj], rb1[3 * RAWW + jj]);
            const uint32_t pv = (uint32_t)P.w;
            if (cull_keep(w, P.x - qx, P.y - qy, P.z - qz, sext(pv, 11), sext(pv >> 11, 11), sext(pv >> 22, 10))) {
              if (cnt == 0) sv0 = jj;
              else if (cnt == 1) sv1 = jj;
              ++cnt;
            }
          }
          sv_n = cnt;
        }
        FMDP_MARK(PH_OWNER)
        if (solo) __syncthreads();
        mbar_wait(&s_bar[5 + p], (parX >> (2 + p)) & 1u);
        parX ^= 1u << (2 + p);
        if (XP) stay_all = ctl->xstay[p];  // over the ranks, from CTA 0
        FMDP_MARK(PH_BAR2)
      }

      // ---- a7/a8: every warp decides redundantly (identical inputs -> identical decisions),
      //      so no barrier is needed before the next step
      double v1 = -INFINITY;
      int a1 = INT_MAX;
      bool near = false;
      int4 nxt = make_int4(0, 0, 0, 0);  // wide walker: Delta_1(a*) (x, y, z, psi | v << 16)
      int nfl = 0;                       //              and its terrain / goal flags
      if (WIDE && !fin) {
        // a7 over the whole action space, tiled over the clusters: every CTA takes its tile's
        // top-2 (lanes hold a = lane, lane+32, ...); CTA 0 of each cluster publishes {key1, global
        // a1, S(a1), key2, Delta_1(a1), flags} on the decision board (tagged 8-byte words); every
        // warp reads every cluster's record and takes the global argmax (lowest global index on
        // ties: tiles are contiguous index ranges) and the global runner-up for the near-tie
        double lb1 = -INFINITY, lb2 = -INFINITY;
        int li1 = INT_MAX, li2 = INT_MAX;
        for (int a = lane; a < A_tile; a += 32) {
          const double vv = s_vv[a].x;
          if (better(vv, a, lb1, li1)) {
            lb2 = lb1; li2 = li1; lb1 = vv; li1 = a;
          } else if (better(vv, a, lb2, li2)) {
            lb2 = vv; li2 = a;
          }
        }
        const int w1 = argmax_key(0xffffffffu, li1 != INT_MAX, dkey(lb1 + 0.0), (unsigned)li1);
        const int ta1 = __shfl_sync(0xffffffffu, li1, w1);
        const bool own = lane == w1;
        const double cv = own ? lb2 : lb1;
        const int ci = own ? li2 : li1;
        const int w2 = argmax_key(0xffffffffu, ci != INT_MAX, dkey(cv + 0.0), (unsigned)ci);
        const double tv2 = w2 >= 0 ? __shfl_sync(0xffffffffu, cv, w2) : -INFINITY;
        const int nclu = (int)(gridDim.x / G);
        ++wit;
        const int wpar = (int)(wit & 1u);
        if (rank == 0 && warp == 0 && lane < WB_WORDS) {
          const unsigned long long k1 = dkey(s_vv[ta1].x + 0.0), k2 = dkey(tv2 + 0.0);
          const unsigned long long sb = (unsigned long long)__double_as_longlong(s_vv[ta1].y);
          const int4 d1 = s_pos[ta1 * W];
          uint32_t val = 0;
          switch (lane) {
            case 0: val = (uint32_t)(k1 >> 32); break;
            case 1: val = (uint32_t)k1; break;
            case 2: val = (uint32_t)(ta1 + aoff); break;
            case 3: val = (uint32_t)(sb >> 32); break;
            case 4: val = (uint32_t)sb; break;
            case 5: val = (uint32_t)(k2 >> 32); break;
            case 6: val = (uint32_t)k2; break;
            case 7: val = (uint32_t)d1.x; break;
            case 8: val = (uint32_t)d1.y; break;
            case 9: val = (uint32_t)d1.z; break;
            case 10: val = (uint32_t)d1.w; break;
            default: val = (uint32_t)s_flags[ta1]; break;
          }
          st_ll(args.wb + ((size_t)wpar * nclu + wcl) * WB_WORDS + lane, val, wit);
        }
        // every warp: lane c reads cluster c's record (all loads first, polls after)
        uint32_t rec[WB_WORDS];
        const unsigned long long* rb = args.wb + ((size_t)wpar * nclu + lane) * WB_WORDS;
        const long long bud = (4ll << 30);
#pragma unroll
        for (int j = 0; j < WB_WORDS; ++j) {
          rec[j] = 0;
          if (lane < nclu) rec[j] = ld_ll(rb + j, wit, args.werr, bud);
        }
        const bool okc = lane < nclu;
        const unsigned long long gk1 = ((unsigned long long)rec[0] << 32) | rec[1];
        const int wl = argmax_key(0xffffffffu, okc, gk1, rec[2]);
        a1 = (int)__shfl_sync(0xffffffffu, rec[2], wl);
        const unsigned long long wk1 = __shfl_sync(0xffffffffu, gk1, wl);
        v1 = undkey(wk1);
        const unsigned long long sbits = ((unsigned long long)__shfl_sync(0xffffffffu, rec[3], wl) << 32) |
                                         __shfl_sync(0xffffffffu, rec[4], wl);
        const double thr = w.near_tie_rel * __longlong_as_double((long long)sbits);
        // runner-up: every other cluster's best, and the winner cluster's second
        const unsigned long long gk2 = ((unsigned long long)rec[5] << 32) | rec[6];
        const unsigned long long ck = lane == wl ? gk2 : gk1;
        const unsigned chi = okc ? (unsigned)(ck >> 32) : 0u;
        const unsigned mhi = __reduce_max_sync(0xffffffffu, chi);
        const unsigned mlo = __reduce_max_sync(0xffffffffu, (okc && chi == mhi) ? (unsigned)ck : 0u);
        const unsigned long long k2max = ((unsigned long long)mhi << 32) | mlo;
        near = nclu * (int)A_tile > 1 && k2max != 0ull && v1 - undkey(k2max) < thr;
        nxt = make_int4((int)__shfl_sync(0xffffffffu, rec[7], wl), (int)__shfl_sync(0xffffffffu, rec[8], wl),
                        (int)__shfl_sync(0xffffffffu, rec[9], wl), (int)__shfl_sync(0xffffffffu, rec[10], wl));
        nfl = (int)__shfl_sync(0xffffffffu, rec[11], wl);
      } else if (!fin && A <= 32) {
        // a7 (Alg 9; ties -> lowest index, R13): lane a holds V*(a); REDUX max over
        // order-preserving keys, lowest index among equal keys; near-tie (north star: top-2 gap
        // < near_tie_rel * S) <=> some other action is within the threshold of the winner
        const bool ok = lane < A;
        const double v = ok ? s_vv[lane].x : -INFINITY;
        const int w1 = argmax_key(0xffffffffu, ok, dkey(v + 0.0), (unsigned)lane);
        a1 = w1;
        v1 = __shfl_sync(0xffffffffu, v, w1);
        const double thr = w.near_tie_rel * s_vv[a1].y;
        near = __any_sync(0xffffffffu, ok && lane != w1 && v1 - v < thr);
      } else if (!fin) {
        // a7: top-2 over V* (Alg 9; ties -> lowest index, R13).  Lane l holds its best
        // and second-best among a = l, l+32, ...; REDUX max over order-preserving keys.
        double lb1 = -INFINITY, lb2 = -INFINITY;
        int li1 = INT_MAX, li2 = INT_MAX;
        for (int a = lane; a < A; a += 32) {
          const double v = s_vv[a].x;
          if (better(v, a, lb1, li1)) {
            lb2 = lb1; li2 = li1; lb1 = v; li1 = a;
          } else if (better(v, a, lb2, li2)) {
            lb2 = v; li2 = a;
          }
        }
        const int w1 = argmax_key(0xffffffffu, li1 != INT_MAX, dkey(lb1), (unsigned)li1);
        a1 = __shfl_sync(0xffffffffu, li1, w1);
        v1 = __shfl_sync(0xffffffffu, lb1, w1);
        // near-tie (R-north-star: top-2 gap < 1e-4 S): v1 - v2 < thr with v2 the runner-up
        // <=> some lane's best action other than a1 is within thr -- one vote, no second argmax
        const bool own = lane == w1;
        const double cv = own ? lb2 : lb1;
        const int ci = own ? li2 : li1;
        const double thr = w.near_tie_rel * s_vv[a1].y;
        near = __any_sync(0xffffffffu, ci != INT_MAX && v1 - cv < thr);
      }
      FMDP_MARK(PH_ARGMAX)
      const uint32_t c0 = stay_all;
      bool done = false;
      if (xmode == 1) {  // export step: no decision in this launch
        status = -1;
        done = true;
      } else if (evalm) {
        if (lead && rank == 0 && tid == 0) {
          args.dbg_conf[WIDE ? w.A_all : A] = c0;
          args.dbg_astar[0] = a1;
        }
        done = true;
      } else {
        if (lead && rank == 0 && tid == 0) args.stepd2[sbase + k] = c0;
        min_sep = min(min_sep, c0);
        // Determine terminal state of state k (Sec IV.I): conflict, terrain, goal, timeout
        int st = -1;
        if (c0 < w.sep2) st = 1;
        else if (fl & 1) st = 2;
        else if (fl & 2) st = 0;
        else if (k >= w.max_steps) st = 3;
        if (st >= 0) {
          status = st;
          fail_step = st == 0 ? -1 : k;
          done = true;
        } else {
          const int4 p1 = WIDE ? nxt : s_pos[a1 * W + 0];  // s_{t+1} <- Delta_1[a*] (Alg 1)
          const int npsi = WIDE ? (p1.w & 0xffff) : p1.w;
          if (lead && rank == 0 && tid == 0) {
            args.astar[sbase + k] = a1;
            args.ntie[sbase + k] = near ? 1 : 0;
            int32_t* tq = args.traj + 3 * (sbase + k + 1);
            tq[0] = p1.x; tq[1] = p1.y; tq[2] = p1.z;
            args.heading[sbase + k + 1] = npsi;
            if (WIDE) args.speed[sbase + k + 1] = p1.w >> 16;
          }
          n_near += near ? 1 : 0;
          steps_run += 1;
          k += 1;
          bK = bK == 2 ? 0 : bK + 1;
          qx = p1.x; qy = p1.y; qz = p1.z;
          psi = npsi;
          if (WIDE) v = p1.w >> 16;
          fl = WIDE ? nfl : s_flags[a1];
          fin = fl != 0 || k >= w.max_steps;
          // slice budget spent: pause at state k (the head never pauses; with a stop flag the
          // others keep going until the head has finished -- free work in a single-wave slice)
          if (!rq.head && k - rq.start_k >= args.budget && (!args.stop || ctl->stop[p])) {
            status = -1;
            done = true;
          }
          // re-convergence: the new state k equals the previous run's, and no plan committed since
          // that run can influence its states from here on -- its decisions, per-step records and
          // verdict stand (copied in the request epilogue); a previous run that had paused (status
          // -1) pauses this one at its last state (the host resumes it from there)
          if (bak_act) {
            const int4 o = ctl->bakst[p];
            if (o.x == p1.x && o.y == p1.y && o.z == p1.z && o.w == npsi) {
              reconv = true;
              status = rq.old_status;
              fail_step = rq.old_fail;
              done = true;
            }
          }
        }
      }
      FMDP_MARK(PH_DECIDE)
      if (done) break;
      // co-simulation: state of clock K+1 and its velocity, the last displacement
      // q(k+1) - q(k) = ((DX, DY)[psi_{k+1}], climb of a*) (R28)
      if (cosim && rank == 0 && tid == 0)
        cs_publish(args, r, K + 1, qx, qy, qz, CS_PRESENT, s_dxy[psi].x, s_dxy[psi].y, w.climb[a1 % C]);
    }

    // eval only: separation minimum of every action's Delta_1 vs the whole row K+1 (debug hook)
    if (evalm && rank == 0) {
      __syncthreads();
      for (int a = tid; a < A; a += NT) s_conf[a] = w.sat_d2;
      const int A = A_tile;  // (the tile's real actions; global index a + aoff)
      __syncthreads();
      const int4* s_pos = s_pos2 + (k & 1) * AW;
      const int64_t K1 = rq.t0 + 1;
      const int n1 = row_count(w, K1);
      const int32_t* rowg = w.rows + (size_t)K1 * 4 * w.row_cap;
      for (int i = tid; i < A * n1; i += NT) {
        const int a = i / n1, j = i % n1;
        const int4 p1 = s_pos[a * W];
        const uint32_t d = clamp_d2(rowg[j] - p1.x, rowg[w.row_cap + j] - p1.y, rowg[2 * w.row_cap + j] - p1.z,
                                    w.R_max, w.sat_d2);
        if (d < w.sat_d2) atomicMin(&s_conf[a], d);
      }
      __syncthreads();
      for (int a = tid; a < A; a += NT) args.dbg_conf[a + aoff] = s_conf[a];
    }

    // ------------------------------------------------------------ request epilogue
    if (REUSE && reconv && lead)  // the previous run's steps k .. n_old - 1 back into the request's records
      reconv_copy(args.bak, RecPtrs{args.traj, args.heading, args.astar, args.stepx, args.stepd2, args.ntie}, sbase, k,
                  rq.n_old, rank, G, w.sat_d2, solo ? ctl : cluster.map_shared_rank(ctl, 0));
    cluster.sync();  // n_exact contributions of every CTA have landed in rank 0
    if (XP && rank == 0 && tid == 0) args.x_seq[xcl] = xseq0 + xit;  // read by the next launch
    if (lead && rank == 0 && tid == 0 && rq.head && args.stop && (status >= 0 || reconv)) atomicExch(args.stop, 1);
    if (lead && rank == 0 && tid == 0 && !evalm) {
      Out o;
      o.status = status;
      o.n_states = reconv ? rq.n_old : k + 1;
      o.fail_step = fail_step;
      o.n_near_ties = n_near + ctl->rc_near;
      o.n_exact = nex0 + ctl->n_exact + ctl->rc_exact;
      o.steps_run = steps_run;
      o.min_sep_d2 = min(min_sep, ctl->rc_min);
      o.reconv = reconv ? 1 : 0;
      args.out[rq.slot] = o;
    }
    // drain prefetches still in flight before the ring buffers are reused
    for (int b = 0; b < 3; ++b) {
      if (pending & (1u << b)) {
        mbar_wait(&s_bar[b], (par >> b) & 1u);
        par ^= 1u << b;
      }
    }
    pending = 0;
    __syncthreads();
    // co-simulation: this aircraft has left; keep the clock until every walker has
    if (cosim && rank == 0) cs_idle(args.cs_pub, args.cs_arrive, args.cs_err, args.cs_n, args.cs_k0, ctl, r, rq.t0 + k + 1, 0, CS_FINISHED,
              true);
  }
  if (prof) {
    for (int i = 0; i < PH_N; ++i) atomicAdd(&args.prof[i], pacc[i]);
  }
#undef FMDP_MARK
}

// ----------------------------------------------------------------------------- append / influence
// Append accepted plans to the time rows (Sec V: "automatically stored in the database
// of accepted flight plans").  Slots are assigned by the host in plan-id order.
__global__ void append_kernel(int32_t* rows, int32_t cap, int64_t horizon, const AppendPlan* plans) {
  const AppendPlan P = plans[blockIdx.x];  // one block per plan (grid.x up to 2^31-1 plans)
  for (int i = threadIdx.x; i < P.n; i += blockDim.x) {
    const int64_t K = P.t0 + i;
    if (K < 0 || K >= horizon) continue;
    const int32_t* s = P.states + 3 * i;
    int vx = 0, vy = 0, vz = 0;  // forward difference; last repeats previous; single state 0 (R11)
    if (P.n > 1) {
      const int32_t* a = (i < P.n - 1) ? s : s - 3;
      vx = a[3] - a[0];
      vy = a[4] - a[1];
      vz = a[5] - a[2];
    }
    const uint32_t pv = ((uint32_t)vx & 0x7ffu) | (((uint32_t)vy & 0x7ffu) << 11) | (((uint32_t)vz & 0x3ffu) << 22);
    int32_t* row = rows + (size_t)K * 4 * cap;
    const int slot = P.slots[i];
    row[slot] = s[0];
    row[cap + slot] = s[1];
    row[2 * cap + slot] = s[2];
    row[3 * cap + slot] = (int32_t)pv;
  }
}

// First step k of request i whose computation could see plan j, or INT_MAX.  Step k reads
// only row K = t0_i + k: plan j can change it only if one of its wells c_tau = p + k_tau v
// comes within R_tau + reach + 1 of q_i(k) (else it is >= R_tau + 1 from every projected
// state: clearly outside the FP32 band, the same argument as f1 culling), or if p itself is
// within the separation saturation radius R_max of q_i(k).  Exact-conservative (DESIGN.md a10).
__global__ void influence_kernel(const int32_t* traj, const BakRec* bak, int32_t cap, const int32_t* n_states,
                                 const int64_t* t0, const InflPair* pairs, InflWells iw, int32_t* kfirst) {
  __shared__ int32_t best, last;
  const InflPair pr = pairs[blockIdx.x];
  if (threadIdx.x == 0) {
    best = INT_MAX;
    last = -1;
  }
  __syncthreads();
  const int nj = n_states[pr.j];
  const int ilo = pr.hi < 0 ? 0 : pr.lo, ihi = pr.hi < 0 ? n_states[pr.i] : pr.hi;
  const int64_t ti = t0[pr.i], tj = t0[pr.j];
  const int32_t* qi = traj + (size_t)pr.i * cap * 3;
  const BakRec* bi = bak + (size_t)pr.i * cap;  // (pr.bak: the backup of i's previous run)
  const int32_t* pj = traj + (size_t)pr.j * cap * 3;
  // only rows where both are present can interact
  const int64_t k_lo = max((int64_t)ilo, tj - ti), k_hi = min((int64_t)ihi, tj + nj - ti);
  for (int64_t k = k_lo + threadIdx.x; k < k_hi; k += blockDim.x) {
    const int64_t idx = ti + k - tj;
    const int32_t* p = pj + 3 * idx;
    int64_t vx = 0, vy = 0, vz = 0;  // forward difference (R11)
    if (nj > 1) {
      const int32_t* a = idx < nj - 1 ? p : p - 3;
      vx = a[3] - a[0]; vy = a[4] - a[1]; vz = a[5] - a[2];
    }
    int64_t qx, qy, qz;
    if (pr.bak) {
      qx = bi[k].x; qy = bi[k].y; qz = bi[k].z;
    } else {
      qx = qi[3 * k]; qy = qi[3 * k + 1]; qz = qi[3 * k + 2];
    }
    const int64_t rx = (int64_t)p[0] - qx, ry = (int64_t)p[1] - qy, rz = (int64_t)p[2] - qz;
    bool hit = rx * rx + ry * ry + rz * rz < iw.sat2;
    for (int t = 0; t < iw.n_tau && !hit; ++t) {
      const int64_t cx = rx + iw.k_tau[t] * vx, cy = ry + iw.k_tau[t] * vy, cz = rz + iw.k_tau[t] * vz;
      hit = cx * cx + cy * cy + cz * cz < iw.r2[t];
    }
    if (hit) {
      atomicMin(&best, (int32_t)k);
      atomicMax(&last, (int32_t)k);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // [first, last] influenced step of request i (INT_MAX, -1: none)
    kfirst[2 * blockIdx.x] = best;
    kfirst[2 * blockIdx.x + 1] = last;
  }
}

// Result trajectories of a batch packed back to back (one D2H copy instead of one per request).
__global__ void pack_traj_kernel(const int32_t* traj, int32_t cap, const Out* out, const int64_t* off, int32_t* pack) {
  const int i = blockIdx.x;
  const int n3 = 3 * out[i].n_states;
  const int32_t* src = traj + (size_t)i * cap * 3;
  int32_t* dst = pack + 3 * off[i];
  for (int e = threadIdx.x; e < n3; e += blockDim.x) dst[e] = src[e];
}

// Backup of slot i's steps [lo, hi) before a rollback overwrites them (re-convergence, a10).
__global__ void backup_kernel(BakRec* bak, const int32_t* traj, const int32_t* heading, const int32_t* astar,
                              const int32_t* stepx, const uint32_t* stepd2, const int8_t* ntie, int32_t cap, int slot,
                              int lo, int hi) {
  const size_t b = (size_t)slot * cap;
  for (int m = lo + blockIdx.x * blockDim.x + threadIdx.x; m < hi; m += gridDim.x * blockDim.x) {
    BakRec e;
    e.x = traj[3 * (b + m)];
    e.y = traj[3 * (b + m) + 1];
    e.z = traj[3 * (b + m) + 2];
    e.heading = heading[b + m];
    e.astar = astar[b + m];
    e.stepx = stepx[b + m];
    e.stepd2 = stepd2[b + m];
    e.ntie = ntie[b + m];
    bak[b + m] = e;
  }
}

// ----------------------------------------------------------------------------- range-query index
__device__ __forceinline__ int cell_of(const World& w, int x, int y) {
  int cx = (x - w.cell_x0) / w.cell_l, cy = (y - w.cell_y0) / w.cell_l;  // (clamped: conservative, see World)
  cx = min(max(cx, 0), w.cell_ncx - 1);
  cy = min(max(cy, 0), w.cell_ncy - 1);
  return cy * w.cell_ncx + cx;
}

// One CTA per row: counting sort of slots [0, counts[K]) by cell (histogram, block scan, scatter into
// tmp, copy back); cstart[K][c] = first slot of cell c, cstart[K][cell_n] = counts[K].
__global__ void index_kernel(int32_t* rows, int32_t row_cap, const int32_t* counts, int64_t K0, World w,
                             int32_t* cstart, int32_t* tmp) {
  extern __shared__ int32_t hist[];  // [cell_n] counts, then cursors
  __shared__ int32_t part[1024];
  const int64_t K = K0 + blockIdx.x;
  const int n = counts[K];
  const int C = w.cell_n, NT = blockDim.x, tid = threadIdx.x;
  int32_t* row = rows + (size_t)K * 4 * row_cap;
  int32_t* cs = cstart + (size_t)K * (C + 1);
  for (int c = tid; c < C; c += NT) hist[c] = 0;
  __syncthreads();
  for (int j = tid; j < n; j += NT) atomicAdd(&hist[cell_of(w, row[j], row[row_cap + j])], 1);
  __syncthreads();
  // exclusive scan: thread t owns cells [t*per, (t+1)*per)
  const int per = (C + NT - 1) / NT;
  const int c0 = min(C, tid * per), c1 = min(C, c0 + per);
  int sum = 0;
  for (int c = c0; c < c1; ++c) sum += hist[c];
  part[tid] = sum;
  __syncthreads();
  if (tid == 0) {
    int acc = 0;
    for (int t = 0; t < NT; ++t) {
      const int v = part[t];
      part[t] = acc;
      acc += v;
    }
  }
  __syncthreads();
  int acc = part[tid];
  for (int c = c0; c < c1; ++c) {
    const int v = hist[c];
    hist[c] = acc;
    cs[c] = acc;
    acc += v;
  }
  if (tid == 0) cs[C] = n;
  __syncthreads();
  // stable scatter (deterministic slot order: every rank of a plan-sharded exchange, which splits
  // rows by slot ranges, must see the same row): warp 0 walks the row in order, 32 plans at a time,
  // ranking equal cells within the warp by __match_any_sync
  int32_t* t = tmp + (size_t)blockIdx.x * 4 * row_cap;
  if (tid < 32) {
    const unsigned lt = (1u << tid) - 1u;
    for (int j0 = 0; j0 < n; j0 += 32) {
      const int j = j0 + tid;
      const int c = j < n ? cell_of(w, row[j], row[row_cap + j]) : -1;
      const unsigned m = __match_any_sync(0xffffffffu, c);
      if (c >= 0) {
        const int pos = hist[c] + __popc(m & lt);
        for (int a = 0; a < 4; ++a) t[(size_t)a * row_cap + pos] = row[(size_t)a * row_cap + j];
      }
      __syncwarp();
      if (c >= 0 && (m & lt) == 0) hist[c] += __popc(m);  // the group's first lane advances the cursor
      __syncwarp();
    }
  }
  __syncthreads();
  for (int a = 0; a < 4; ++a)
    for (int j = tid; j < n; j += NT) row[(size_t)a * row_cap + j] = t[(size_t)a * row_cap + j];
}

__global__ void vmax_kernel(const int32_t* rows, int32_t row_cap, const int32_t* counts, int64_t horizon,
                            unsigned long long* out) {
  unsigned long long best = 0;
  for (int64_t K = blockIdx.x; K < horizon; K += gridDim.x) {
    const int n = counts[K];
    const int32_t* vp = rows + (size_t)K * 4 * row_cap + 3 * (size_t)row_cap;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const uint32_t pv = (uint32_t)vp[j];
      const long long vx = sext(pv, 11), vy = sext(pv >> 11, 11);
      best = max(best, (unsigned long long)(vx * vx + vy * vy));
    }
  }
  for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0 && best) atomicMax(out, best);
}

cudaError_t launch_index(int32_t* rows, int32_t row_cap, const int32_t* counts, int64_t K0, int nrows, const World& w,
                         int32_t* cstart, int32_t* tmp, cudaStream_t s) {
  if (nrows <= 0) return cudaSuccess;
  const int smem = (int)sizeof(int32_t) * w.cell_n;
  cudaError_t e = cudaFuncSetAttribute(index_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  index_kernel<<<nrows, 1024, smem, s>>>(rows, row_cap, counts, K0, w, cstart, tmp);
  return cudaGetLastError();
}

cudaError_t launch_vmax(const int32_t* rows, int32_t row_cap, const int32_t* counts, int64_t horizon,
                        unsigned long long* out, cudaStream_t s) {
  vmax_kernel<<<(int)std::min<int64_t>(horizon, 2048), 256, 0, s>>>(rows, row_cap, counts, horizon, out);
  return cudaGetLastError();
}

// ----------------------------------------------------------------------------- launchers
int walk_groups_per_warp(int ncol, int max_threads) {
  for (int ngw = 4; ngw > 1; ngw >>= 1)
    if (32 * ((ncol + 32 / ngw - 1) / (32 / ngw)) <= max_threads) return ngw;
  return 1;
}

int walk_threads(int ncol, int max_threads) {
  const int cpw = 32 / walk_groups_per_warp(ncol, max_threads);
  return 32 * ((ncol + cpw - 1) / cpw);
}

// Function attributes, set once per device and raised only when a launch needs more (not on
// every launch: concurrent walkers of the multi-GPU exchange launch from several host threads).
template <int C, int MODE>
static cudaError_t set_walk_attrs(int smem, int cluster) {
  static std::mutex mu;
  static int done_smem[64] = {0};
  static bool done_np[64] = {false};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  dev &= 63;
  std::lock_guard<std::mutex> lk(mu);
  if (smem > done_smem[dev]) {
    e = cudaFuncSetAttribute(walk_kernel<C, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    done_smem[dev] = smem;
  }
  if (cluster > 8 && !done_np[dev]) {
    e = cudaFuncSetAttribute(walk_kernel<C, MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    done_np[dev] = true;
  }
  return cudaSuccess;
}

template <int C, int MODE>
static cudaError_t launch_walk_t(const World& w, const WalkArgs& a, int cluster, int n_clusters, int threads,
                                 int chunk, int rawcap, cudaStream_t s) {
  Layout L;
  L.build(w.HL, chunk, rawcap, threads, C, w.n_turn * w.W, w.A, w.A * w.W, cluster);
  cudaError_t e = set_walk_attrs<C, MODE>((int)L.total, cluster);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster * n_clusters, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const int ngw = walk_groups_per_warp(w.n_turn * w.W, threads);
  return cudaLaunchKernelEx(&cfg, walk_kernel<C, MODE>, w, a, chunk, rawcap, ngw);
}

template <int C, int MODE>
static cudaError_t max_clusters_t(const World& w, int cluster, int threads, int chunk, int rawcap, int* out) {
  Layout L;
  L.build(w.HL, chunk, rawcap, threads, C, w.n_turn * w.W, w.A, w.A * w.W, cluster);
  cudaError_t e = set_walk_attrs<C, MODE>((int)L.total, cluster);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.dynamicSmemBytes = L.total;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(out, walk_kernel<C, MODE>, &cfg);
}

cudaError_t launch_walk(const World& w, const WalkArgs& a, int n_climb, int cluster, int n_clusters, int threads,
                        int chunk, int rawcap, cudaStream_t s) {
  const int mode =
      w.wide ? 5 : (a.cosim ? 1 : (a.xmode == 3 ? 2 : ((a.xmode || a.eval || a.prof) ? 3 : (a.cull ? (w.cell_n > 0 ? 6 : 4) : 0))));
#define FMDP_LW(c, m) launch_walk_t<c, m>(w, a, cluster, n_clusters, threads, chunk, rawcap, s)
  switch (n_climb * 8 + mode) {
    case 8: return FMDP_LW(1, 0);
    case 9: return FMDP_LW(1, 1);
    case 10: return FMDP_LW(1, 2);
    case 11: return FMDP_LW(1, 3);
    case 12: return FMDP_LW(1, 4);
    case 14: return FMDP_LW(1, 6);
    case 24: return FMDP_LW(3, 0);
    case 25: return FMDP_LW(3, 1);
    case 26: return FMDP_LW(3, 2);
    case 27: return FMDP_LW(3, 3);
    case 28: return FMDP_LW(3, 4);
    case 30: return FMDP_LW(3, 6);
    case 40: return FMDP_LW(5, 0);
    case 41: return FMDP_LW(5, 1);
    case 42: return FMDP_LW(5, 2);
    case 43: return FMDP_LW(5, 3);
    case 44: return FMDP_LW(5, 4);
    case 46: return FMDP_LW(5, 6);
    case 29: return FMDP_LW(3, 5);    // wide walker (acceleration actions)
    case 85: return FMDP_LW(10, 5);   // A = 15 x 9 x 10 = 1350
    default: return cudaErrorInvalidValue;
  }
#undef FMDP_LW
}

cudaError_t walk_max_clusters(const World& w, int n_climb, int cluster, int threads, int chunk, int rawcap, int* out,
                              bool cosim) {
  if (w.wide) {
    switch (n_climb) {
      case 3: return max_clusters_t<3, 5>(w, cluster, threads, chunk, rawcap, out);
      case 10: return max_clusters_t<10, 5>(w, cluster, threads, chunk, rawcap, out);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (n_climb) {
    case 1: return cosim ? max_clusters_t<1, 1>(w, cluster, threads, chunk, rawcap, out)
                         : max_clusters_t<1, 0>(w, cluster, threads, chunk, rawcap, out);
    case 3: return cosim ? max_clusters_t<3, 1>(w, cluster, threads, chunk, rawcap, out)
                         : max_clusters_t<3, 0>(w, cluster, threads, chunk, rawcap, out);
    case 5: return cosim ? max_clusters_t<5, 1>(w, cluster, threads, chunk, rawcap, out)
                         : max_clusters_t<5, 0>(w, cluster, threads, chunk, rawcap, out);
    default: return cudaErrorInvalidValue;
  }
}

size_t walk_smem_bytes(const World& w, int n_climb, int threads, int chunk, int rawcap, int cluster) {
  Layout L;
  L.build(w.HL, chunk, rawcap, threads, n_climb, w.n_turn * w.W, w.A, w.A * w.W, cluster);
  return L.total;
}

cudaError_t launch_append(int32_t* rows, int32_t row_cap, int64_t horizon, const AppendPlan* plans, int n_plans,
                          int max_n, cudaStream_t s) {
  if (n_plans <= 0) return cudaSuccess;
  (void)max_n;
  append_kernel<<<n_plans, 256, 0, s>>>(rows, row_cap, horizon, plans);
  return cudaGetLastError();
}

cudaError_t launch_influence(const int32_t* traj, const BakRec* bak, int32_t cap, const int32_t* n_states,
                             const int64_t* t0, const InflPair* pairs, int n_pairs, const InflWells& iw, int32_t* kfirst,
                             cudaStream_t s) {
  if (n_pairs <= 0) return cudaSuccess;
  influence_kernel<<<n_pairs, 256, 0, s>>>(traj, bak, cap, n_states, t0, pairs, iw, kfirst);
  return cudaGetLastError();
}

cudaError_t launch_pack_traj(const int32_t* traj, int32_t cap, const Out* out, const int64_t* off, int n, int32_t* pack,
                             cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  pack_traj_kernel<<<n, 256, 0, s>>>(traj, cap, out, off, pack);
  return cudaGetLastError();
}

cudaError_t launch_backup(BakRec* bak, const int32_t* traj, const int32_t* heading, const int32_t* astar,
                          const int32_t* stepx, const uint32_t* stepd2, const int8_t* ntie, int32_t cap, int slot, int lo,
                          int hi, cudaStream_t s) {
  if (hi <= lo) return cudaSuccess;
  const int n = hi - lo;
  backup_kernel<<<(n + 255) / 256, 256, 0, s>>>(bak, traj, heading, astar, stepx, stepd2, ntie, cap, slot, lo, hi);
  return cudaGetLastError();
}

}  // namespace fmdp

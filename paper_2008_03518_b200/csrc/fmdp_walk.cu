// fmdp_walk.cu -- sm_100a kernels of the FastMDP-GPU hot path.
//
// walk_kernel<C>: one thread-block CLUSTER of G CTAs walks one request's whole trajectory
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
#include <cuda_runtime.h>

#include <cfloat>
#include <climits>
#include <cstdint>

#include "fmdp_dev.h"

namespace cg = cooperative_groups;

namespace fmdp {

// ----------------------------------------------------------------------------- PTX helpers
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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ int sext(uint32_t v, int bits) { return (int)(v << (32 - bits)) >> (32 - bits); }

// exact squared distance, saturated at sat (= R_max^2 < 2^30): valid because any component
// >= R_max already implies d^2 >= R_max^2.
__device__ __forceinline__ uint32_t clamp_d2(int dx, int dy, int dz, int rmax, uint32_t sat) {
  uint32_t ax = (uint32_t)abs(dx), ay = (uint32_t)abs(dy), az = (uint32_t)abs(dz);
  if (max(ax, max(ay, az)) >= (uint32_t)rmax) return sat;
  uint32_t d2 = ax * ax + ay * ay + az * az;
  return min(d2, sat);
}

struct Ctl {
  int32_t req;
  int32_t q[3];
  int32_t psi;
  int32_t k;
  int32_t done;
  int32_t namb;
  int32_t ntc;
  int32_t a_star;
  int32_t n_near;
  int32_t n_exact;
  int32_t status;
  int32_t fail_step;
  uint32_t min_sep;
  int32_t steps_run;
  unsigned long long xmin;
  int32_t sl_lo[3], sl_n[3], sl_off[3];
};

// Row K's slice for this CTA: slots [lo, lo+n); the first CH of them are staged in the ring
// buffer K % 3 starting at word offset `off`.
__device__ __forceinline__ void issue_row(const World& w, int64_t K, unsigned rank, unsigned G, int CH,
                                          int32_t* raw, int RAWW, uint64_t* bars, Ctl* ctl) {
  const int b = (int)(K % 3);
  int n = (K >= 0 && K < w.horizon) ? __ldg(&w.counts[K]) : 0;
  int lo = (int)(((int64_t)n * rank) / G), hi = (int)(((int64_t)n * (rank + 1)) / G);
  int e = min(hi, lo + CH);
  int lo4 = lo & ~3, e4 = (e + 3) & ~3;
  ctl->sl_lo[b] = lo;
  ctl->sl_n[b] = hi - lo;
  ctl->sl_off[b] = lo - lo4;
  uint32_t bytes = (e > lo) ? (uint32_t)(e4 - lo4) * 4u : 0u;
  fence_proxy_async();
  mbar_arrive_tx(&bars[b], 4u * bytes);
  if (bytes) {
    const int32_t* base = w.rows + (size_t)K * 4 * w.row_cap;
    int32_t* dst = raw + (size_t)b * 4 * RAWW;
    for (int arr = 0; arr < 4; ++arr)
      bulk_g2s(dst + arr * RAWW, base + (size_t)arr * w.row_cap + lo4, bytes, &bars[b]);
  }
}

// Argmax with the lowest index on ties (Alg 9, R13), warp-wide.
__device__ __forceinline__ void warp_argmax(double v, int i, double& bv, int& bi) {
  bv = v;
  bi = i;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) {
      bv = ov;
      bi = oi;
    }
  }
}

template <int C>
__global__ void __launch_bounds__(512, 1) walk_kernel(const World w, const WalkArgs args, const int CH) {
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank();
  const unsigned G = cluster.num_blocks();
  const int tid = threadIdx.x, NT = blockDim.x;
  const int W = w.W, A = w.A, AW = A * W;
  const int NCOL = w.n_turn * W;
  const int GROUP = (NCOL + 31) & ~31;
  const int NG = NT / GROUP;
  const int grp = tid / GROUP, col = tid % GROUP;
  const int RS = NT / A;  // conflict threads per action

  Layout L;
  L.build(w.HL, CH, NT, C, NCOL, A, AW);
  extern __shared__ __align__(16) unsigned char smem[];
  int2* s_dxy = reinterpret_cast<int2*>(smem + L.o_dxy);
  int32_t* s_raw = reinterpret_cast<int32_t*>(smem + L.o_raw);
  float* s_cen = reinterpret_cast<float*>(smem + L.o_cen);
  uint32_t* s_red = reinterpret_cast<uint32_t*>(smem + L.o_red);
  int4* s_pos = reinterpret_cast<int4*>(smem + L.o_pos);
  double* s_fix = reinterpret_cast<double*>(smem + L.o_fix);
  double* s_sfix = reinterpret_cast<double*>(smem + L.o_sfix);
  float* s_vT = reinterpret_cast<float*>(smem + L.o_vT);
  float* s_mI = reinterpret_cast<float*>(smem + L.o_mI);
  double* s_vstar = reinterpret_cast<double*>(smem + L.o_vstar);
  double* s_vsc = reinterpret_cast<double*>(smem + L.o_vsc);
  uint32_t* s_conf = reinterpret_cast<uint32_t*>(smem + L.o_conf);
  uint32_t* s_confg = reinterpret_cast<uint32_t*>(smem + L.o_confg);
  int32_t* s_amb = reinterpret_cast<int32_t*>(smem + L.o_amb);
  int32_t* s_tc = reinterpret_cast<int32_t*>(smem + L.o_tc);
  uint64_t* s_bar = reinterpret_cast<uint64_t*>(smem + L.o_bar);
  Ctl* ctl = reinterpret_cast<Ctl*>(smem + L.o_ctl);
  const int RED = L.RED, RAWW = L.RAWW;
  const int NHOT = NCOL * C * NTAU;

  for (int i = tid; i < w.HL; i += NT) s_dxy[i] = w.dxy[i];
  if (tid == 0) {
    for (int b = 0; b < 3; ++b) mbar_init(&s_bar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t par = 0;      // next wait parity per ring buffer (bit b)
  uint32_t pending = 0;  // ring buffers issued and not yet waited

  for (;;) {
    // ------------------------------------------------------------ next request
    if (rank == 0 && tid == 0) {
      int r = atomicAdd(args.queue, 1);
      for (unsigned b = 0; b < G; ++b) cluster.map_shared_rank(&ctl->req, b)[0] = r;
    }
    cluster.sync();
    const int r = *(volatile int32_t*)&ctl->req;
    if (r >= args.n_reqs) break;
    const Req rq = args.reqs[r];
    const size_t sbase = (size_t)rq.slot * args.cap;
    if (tid == 0) {
      int k0 = rq.start_k;
      if (k0 == 0) {
        ctl->q[0] = rq.src[0]; ctl->q[1] = rq.src[1]; ctl->q[2] = rq.src[2];
        ctl->psi = rq.psi0;
      } else {
        const int32_t* tq = args.traj + 3 * (sbase + k0);
        ctl->q[0] = tq[0]; ctl->q[1] = tq[1]; ctl->q[2] = tq[2];
        ctl->psi = args.heading[sbase + k0];
      }
      ctl->k = k0;
      ctl->done = 0;
      ctl->n_near = 0;
      ctl->n_exact = 0;
      ctl->status = 0;
      ctl->fail_step = -1;
      ctl->steps_run = 0;
      ctl->min_sep = w.sat_d2;
      if (rank == 0 && k0 > 0 && !args.eval) {  // resume: aggregates of the kept prefix
        int nn = 0;
        uint32_t ms = w.sat_d2;
        for (int kk = 0; kk < k0; ++kk) nn += args.ntie[sbase + kk];
        for (int kk = 0; kk <= k0; ++kk) ms = min(ms, args.stepd2[sbase + kk]);
        ctl->n_near = nn;
        ctl->min_sep = ms;
      }
      if (rank == 0 && k0 == 0 && !args.eval) {
        int32_t* tq = args.traj + 3 * sbase;
        tq[0] = rq.src[0]; tq[1] = rq.src[1]; tq[2] = rq.src[2];
        args.heading[sbase] = rq.psi0;
      }
    }
    if (rank == 0)
      for (int i = tid; i < 3 * RED; i += NT) s_red[i] = 0xffffffffu;
    __syncthreads();
    {
      const int64_t K0 = rq.t0 + ctl->k;
      if (tid == 0) {
        issue_row(w, K0, rank, G, CH, s_raw, RAWW, s_bar, ctl);
        issue_row(w, K0 + 1, rank, G, CH, s_raw, RAWW, s_bar, ctl);
      }
      pending |= (1u << (K0 % 3)) | (1u << ((K0 + 1) % 3));
    }
    cluster.sync();

    // ------------------------------------------------------------ step loop
    for (;;) {
      const int k = ctl->k;
      const int64_t K = rq.t0 + k;
      const int qx = ctl->q[0], qy = ctl->q[1], qz = ctl->q[2], psi = ctl->psi;
      const int bK = (int)(K % 3), bK1 = (int)((K + 1) % 3), bK2 = (int)((K + 2) % 3);
      if (rank == 0)  // reset the reduction buffer of step k+1 (last read in step k-2)
        for (int i = tid; i < RED; i += NT) s_red[((k + 1) % 3) * RED + i] = 0xffffffffu;
      if (!args.eval && tid == 0) issue_row(w, K + 2, rank, G, CH, s_raw, RAWW, s_bar, ctl);
      if (!args.eval) pending |= 1u << bK2;
      if (tid == 0) {
        ctl->namb = 0;
        ctl->ntc = 0;
      }
      for (int a = tid; a <= A; a += NT) s_conf[a] = w.sat_d2;
      __syncthreads();

      // ---- a5 candidates: terrain wells that can reach any projected state (exact cull)
      for (int i = tid; i < w.n_tw; i += NT) {
        int4 t = __ldg(&w.tw[i]);
        int64_t dx = t.x - qx, dy = t.y - qy, dz = t.z - qz;
        int64_t rr = (int64_t)t.w + w.reach_u;
        if (dx * dx + dy * dy + dz * dz < rr * rr) {
          int slot = atomicAdd(&ctl->ntc, 1);
          if (slot < TC_MAX) s_tc[slot] = i;
        }
      }
      // ---- a2 forward projection: thread (grp, col) -> column (turn it, substep t)
      float sx = 0.f, sy = 0.f, sz[C];
      {
        const int it = min(col / W, w.n_turn - 1), t = col % W + 1;
        const int h = w.turn[it];
        int x = qx, y = qy, ps = psi;
        for (int s = 1; s <= t; ++s) {
          ps += h;
          ps = (ps % w.HL + w.HL) % w.HL;
          int2 d = s_dxy[ps];
          x += d.x;
          y += d.y;
        }
        sx = (float)(x - qx);
        sy = (float)(y - qy);
#pragma unroll
        for (int c = 0; c < C; ++c) sz[c] = (float)(w.climb[c] * t);
        if (grp == 0 && col < NCOL) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int a = it * C + c;
            s_pos[a * W + (t - 1)] = make_int4(x, y, qz + w.climb[c] * t, ps);
          }
        }
      }
      __syncthreads();
      const int ntc = ctl->ntc;

      // ---- a3 goal (fp64), deck, a5 terrain (exact predicate, FP32 ex2 value)
      for (int st = tid; st < AW; st += NT) {
        const int4 p = s_pos[st];
        const int64_t gx = (int64_t)p.x - rq.dst[0], gy = (int64_t)p.y - rq.dst[1], gz = (int64_t)p.z - rq.dst[2];
        const double vpos = w.goal_r * exp2(w.goal_l2g * sqrt((double)(gx * gx + gy * gy + gz * gz)));
        const double valt = (p.z < w.zdeck_u) ? (w.deck_scale - w.u_m * (double)p.z) : 0.0;
        int64_t mT = INT64_MAX;
        if (ntc <= TC_MAX) {
          for (int c = 0; c < ntc; ++c) {
            int4 t = __ldg(&w.tw[s_tc[c]]);
            int64_t dx = p.x - t.x, dy = p.y - t.y, dz = p.z - t.z;
            int64_t d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < (int64_t)t.w * t.w && d2 < mT) mT = d2;
          }
        } else {
          for (int c = 0; c < w.n_tw; ++c) {
            int4 t = __ldg(&w.tw[c]);
            int64_t dx = p.x - t.x, dy = p.y - t.y, dz = p.z - t.z;
            int64_t d2 = dx * dx + dy * dy + dz * dz;
            if (d2 < (int64_t)t.w * t.w && d2 < mT) mT = d2;
          }
        }
        s_vT[st] = (mT != INT64_MAX) ? w.terr_r * ex2_approx(w.terr_l2g * sqrtf((float)mT)) : 0.f;
        s_fix[st] = vpos - valt;
        s_sfix[st] = vpos + valt;
      }

      // ---- a1 + a4: wells of row K, hot loop
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
      uint32_t stay = w.sat_d2;
      {
        const int lo = ctl->sl_lo[bK], n = ctl->sl_n[bK];
        const int32_t* rowg = w.rows + (size_t)K * 4 * w.row_cap;
        for (int c0 = 0; c0 < n; c0 += CH) {
          const int nc = min(CH, n - c0);
          const int32_t *X, *Y, *Z, *V;
          if (c0 == 0) {
            const int32_t* b = s_raw + (size_t)bK * 4 * RAWW + ctl->sl_off[bK];
            X = b; Y = b + RAWW; Z = b + 2 * RAWW; V = b + 3 * RAWW;
          } else {
            X = rowg + lo + c0; Y = X + w.row_cap; Z = Y + w.row_cap; V = Z + w.row_cap;
          }
          for (int j = tid; j < nc; j += NT) {
            const int rx = X[j] - qx, ry = Y[j] - qy, rz = Z[j] - qz;
            const uint32_t pv = (uint32_t)V[j];
            const int vx = sext(pv, 11), vy = sext(pv >> 11, 11), vz = sext(pv >> 22, 10);
            stay = min(stay, clamp_d2(rx, ry, rz, w.R_max, w.sat_d2));
            float4* c4 = reinterpret_cast<float4*>(s_cen + 16 * j);
            float cc[16];
#pragma unroll
            for (int t = 0; t < NTAU; ++t) {
              cc[3 * t + 0] = (float)(rx + w.k_tau[t] * vx);
              cc[3 * t + 1] = (float)(ry + w.k_tau[t] * vy);
              cc[3 * t + 2] = (float)(rz + w.k_tau[t] * vz);
            }
            cc[15] = 0.f;
            c4[0] = make_float4(cc[0], cc[1], cc[2], cc[3]);
            c4[1] = make_float4(cc[4], cc[5], cc[6], cc[7]);
            c4[2] = make_float4(cc[8], cc[9], cc[10], cc[11]);
            c4[3] = make_float4(cc[12], cc[13], cc[14], cc[15]);
          }
          __syncthreads();
          const float4* cen4 = reinterpret_cast<const float4*>(s_cen);
#define FMDP_WELL(T, CX, CY, CZ)                          \
  {                                                       \
    const float dx = sx - (CX), dy = sy - (CY);           \
    const float hh = fmaf(dy, dy, dx * dx);               \
    _Pragma("unroll") for (int cc_ = 0; cc_ < C; ++cc_) { \
      const float dz = sz[cc_] - (CZ);                    \
      m[cc_][T] = fminf(m[cc_][T], fmaf(dz, dz, hh));     \
    }                                                     \
  }
#pragma unroll 2
          for (int j = grp; j < nc; j += NG) {
            const float4 e0 = cen4[4 * j + 0], e1 = cen4[4 * j + 1], e2 = cen4[4 * j + 2], e3 = cen4[4 * j + 3];
            FMDP_WELL(0, e0.x, e0.y, e0.z)
            FMDP_WELL(1, e0.w, e1.x, e1.y)
            FMDP_WELL(2, e1.z, e1.w, e2.x)
            FMDP_WELL(3, e2.y, e2.z, e2.w)
            FMDP_WELL(4, e3.x, e3.y, e3.z)
          }
#undef FMDP_WELL
          __syncthreads();
        }
        if (tid == 0 && args.pairs) atomicAdd(args.pairs, (unsigned long long)n * NTAU * AW);
      }
      if (stay < w.sat_d2) atomicMin(&s_conf[A], stay);

      // ---- a8 fused separation check: Delta_1(a) vs this CTA's slice of row K+1
      if (pending & (1u << bK1)) {
        mbar_wait(&s_bar[bK1], (par >> bK1) & 1u);
        par ^= 1u << bK1;
        pending &= ~(1u << bK1);
      }
      {
        const int lo = ctl->sl_lo[bK1], n = ctl->sl_n[bK1];
        const int a = tid / RS, rr = tid % RS;
        if (a < A) {
          const int4 p1 = s_pos[a * W + 0];
          const int ax = p1.x - qx, ay = p1.y - qy, az = p1.z - qz;
          uint32_t cm = w.sat_d2;
          const int32_t* b = s_raw + (size_t)bK1 * 4 * RAWW + ctl->sl_off[bK1];
          const int32_t* rowg = w.rows + (size_t)(K + 1) * 4 * w.row_cap + lo;
          for (int j = rr; j < n; j += RS) {
            int px, py, pz;
            if (j < CH) {
              px = b[j]; py = b[RAWW + j]; pz = b[2 * RAWW + j];
            } else {
              px = rowg[j]; py = rowg[w.row_cap + j]; pz = rowg[2 * w.row_cap + j];
            }
            cm = min(cm, clamp_d2(px - qx - ax, py - qy - ay, pz - qz - az, w.R_max, w.sat_d2));
          }
          if (cm < w.sat_d2) atomicMin(&s_conf[a], cm);
        }
      }

      // ---- cross-CTA reduction into CTA 0 (distributed shared memory)
      float* s_part = s_cen;  // reuse: [grp][col][c][tau]
#pragma unroll
      for (int c = 0; c < C; ++c)
#pragma unroll
        for (int t = 0; t < NTAU; ++t) s_part[((size_t)(grp * GROUP + col) * C + c) * NTAU + t] = m[c][t];
      __syncthreads();
      {
        uint32_t* red = cluster.map_shared_rank(s_red + (k % 3) * RED, 0);
        for (int i = tid; i < NHOT; i += NT) {
          const int cl = i / (C * NTAU), rem = i % (C * NTAU);
          float mm = s_part[(size_t)cl * C * NTAU + rem];
          for (int g2 = 1; g2 < NG; ++g2) mm = fminf(mm, s_part[((size_t)(g2 * GROUP + cl)) * C * NTAU + rem]);
          atomicMin(&red[i], __float_as_uint(mm));
        }
        for (int a = tid; a <= A; a += NT) atomicMin(&red[NHOT + a], s_conf[a]);
      }
      cluster.sync();

      // ---- epilogue (every CTA, identical inputs -> identical decisions)
      const uint32_t* redg = cluster.map_shared_rank(s_red + (k % 3) * RED, 0);
      for (int a = tid; a <= A; a += NT) s_confg[a] = redg[NHOT + a];
      for (int st = tid; st < AW; st += NT) {
        const int a = st / W, t1 = st % W, it = a / C, c = a % C;
        const int base = ((it * W + t1) * C + c) * NTAU;
        float mi = FLT_MAX;
#pragma unroll
        for (int t = 0; t < NTAU; ++t) {
          const float M = __uint_as_float(redg[base + t]);
          if (M < w.R2lo[t]) {
            mi = fminf(mi, M);
          } else if (M <= w.R2hi[t]) {  // inside the 2^-20 band: decide exactly below
            const int idx = atomicAdd(&ctl->namb, 1);
            if (idx < AMB_MAX) s_amb[idx] = st * NTAU + t;
          }
        }
        s_mI[st] = mi;
      }
      __syncthreads();
      const int namb = ctl->namb;
      if (namb > 0) {
        // Exact fallback: min over the WHOLE row K of the int64 d^2 for (state, tau); rare.
        const int nK = (K < w.horizon) ? __ldg(&w.counts[K]) : 0;
        const int32_t* rowg = w.rows + (size_t)K * 4 * w.row_cap;
        const int nitems = namb <= AMB_MAX ? namb : AW * NTAU;
        for (int it2 = 0; it2 < nitems; ++it2) {
          const int item = namb <= AMB_MAX ? s_amb[it2] : it2;
          const int st = item / NTAU, t = item % NTAU;
          if (namb > AMB_MAX) {  // overflow: re-test this item's filter verdict
            const int a = st / W, t1 = st % W, it = a / C, c = a % C;
            const float M = __uint_as_float(redg[((it * W + t1) * C + c) * NTAU + t]);
            if (!(M >= w.R2lo[t] && M <= w.R2hi[t])) continue;
          }
          if (tid == 0) ctl->xmin = ULLONG_MAX;
          __syncthreads();
          const int4 p = s_pos[st];
          unsigned long long best = ULLONG_MAX;
          for (int j = tid; j < nK; j += NT) {
            const uint32_t pv = (uint32_t)rowg[3 * w.row_cap + j];
            const int64_t cx = rowg[j] + (int64_t)w.k_tau[t] * sext(pv, 11);
            const int64_t cy = rowg[w.row_cap + j] + (int64_t)w.k_tau[t] * sext(pv >> 11, 11);
            const int64_t cz = rowg[2 * w.row_cap + j] + (int64_t)w.k_tau[t] * sext(pv >> 22, 10);
            const int64_t dx = p.x - cx, dy = p.y - cy, dz = p.z - cz;
            best = min(best, (unsigned long long)(dx * dx + dy * dy + dz * dz));
          }
          if (best != ULLONG_MAX) atomicMin(&ctl->xmin, best);
          __syncthreads();
          if (tid == 0) {
            const unsigned long long x = ctl->xmin;
            if ((int64_t)x < w.R2_tau[t]) s_mI[st] = fminf(s_mI[st], (float)x);
            ctl->n_exact += 1;
          }
          __syncthreads();
        }
      }
      // a6: V = V+ - max(V^T, V^I) - V_alt (Alg 8), term scale S
      for (int st = tid; st < AW; st += NT) {
        const float mi = s_mI[st];
        const float vI = (mi < FLT_MAX) ? w.intr_r * ex2_approx(w.intr_l2g * sqrtf(mi)) : 0.f;
        const double neg = (double)fmaxf(vI, s_vT[st]);
        const double fx = s_fix[st], sf = s_sfix[st];
        s_fix[st] = fx - neg;
        s_sfix[st] = sf + neg;
      }
      __syncthreads();
      for (int a = tid; a < A; a += NT) {  // V*(a) = max(init, max_t V(a,t))
        double vmax = w.vmax_init_zero ? 0.0 : -INFINITY, bt = -INFINITY, bs = 0.0;
        for (int t = 0; t < W; ++t) {
          const double v = s_fix[a * W + t];
          if (v > vmax) vmax = v;
          if (v > bt) {
            bt = v;
            bs = s_sfix[a * W + t];
          }
        }
        s_vstar[a] = vmax;
        s_vsc[a] = bs;
      }
      __syncthreads();
      if (tid < 32) {  // a7: argmax (lowest index on ties) and runner-up
        double bv = -INFINITY;
        int bi = INT_MAX;
        for (int a = tid; a < A; a += 32) {
          const double v = s_vstar[a];
          if (v > bv || (v == bv && a < bi)) { bv = v; bi = a; }
        }
        double v1;
        int a1;
        warp_argmax(bv, bi, v1, a1);
        double cv = -INFINITY;
        int ci = INT_MAX;
        for (int a = tid; a < A; a += 32) {
          if (a == a1) continue;
          const double v = s_vstar[a];
          if (v > cv || (v == cv && a < ci)) { cv = v; ci = a; }
        }
        double v2;
        int a2;
        warp_argmax(cv, ci, v2, a2);
        if (tid == 0) {
          const bool near = (A > 1) && (v1 - v2 < w.near_tie_rel * s_vsc[a1]);
          if (args.eval) {
            if (rank == 0) {
              for (int a = 0; a < A; ++a) args.dbg_vstar[a] = s_vstar[a];
              for (int a = 0; a <= A; ++a) args.dbg_conf[a] = s_confg[a];
              args.dbg_astar[0] = a1;
            }
            ctl->done = 1;
          } else {
            const size_t sb = sbase;
            bool decided = false;
            if (k == 0) {  // departure-row terminal tests before the first decision
              const uint32_t c0 = s_confg[A];
              ctl->min_sep = min(ctl->min_sep, c0);
              if (rank == 0) args.stepd2[sb] = c0;
              int st = -1;
              const bool below = (qz < 0) || ([&] {
                                   if (w.nx <= 0) return false;
                                   const int64_t rx = (int64_t)qx - w.x0, ry = (int64_t)qy - w.y0;
                                   if (rx < 0 || ry < 0) return false;
                                   const int64_t ix = rx / w.cell, iy = ry / w.cell;
                                   if (ix >= w.nx || iy >= w.ny) return false;
                                   return qz < __ldg(&w.height[iy * (int64_t)w.nx + ix]);
                                 }());
              const int64_t gx = (int64_t)qx - rq.dst[0], gy = (int64_t)qy - rq.dst[1], gz = (int64_t)qz - rq.dst[2];
              if (c0 < w.sep2) st = 1;
              else if (below) st = 2;
              else if (gx * gx + gy * gy + gz * gz < w.cap2) st = 0;
              if (st >= 0) {
                ctl->status = st;
                ctl->fail_step = st == 0 ? -1 : 0;
                ctl->done = 1;
                decided = true;
              }
            }
            if (!decided) {
              if (rank == 0) {
                args.astar[sb + k] = a1;
                args.ntie[sb + k] = near ? 1 : 0;
              }
              ctl->n_near += near ? 1 : 0;
              const int4 p1 = s_pos[a1 * W + 0];  // s_{t+1} <- Delta_1[a*] (Alg 1)
              const int k1 = k + 1;
              ctl->q[0] = p1.x; ctl->q[1] = p1.y; ctl->q[2] = p1.z;
              ctl->psi = p1.w;
              ctl->k = k1;
              ctl->steps_run += 1;
              const uint32_t c1 = s_confg[a1];
              ctl->min_sep = min(ctl->min_sep, c1);
              if (rank == 0) {
                int32_t* tq = args.traj + 3 * (sb + k1);
                tq[0] = p1.x; tq[1] = p1.y; tq[2] = p1.z;
                args.heading[sb + k1] = p1.w;
                args.stepd2[sb + k1] = c1;
              }
              // Determine terminal state (Sec IV.I), priority: conflict, terrain, goal, timeout
              const bool below = (p1.z < 0) || ([&] {
                                   if (w.nx <= 0) return false;
                                   const int64_t rx = (int64_t)p1.x - w.x0, ry = (int64_t)p1.y - w.y0;
                                   if (rx < 0 || ry < 0) return false;
                                   const int64_t ix = rx / w.cell, iy = ry / w.cell;
                                   if (ix >= w.nx || iy >= w.ny) return false;
                                   return p1.z < __ldg(&w.height[iy * (int64_t)w.nx + ix]);
                                 }());
              const int64_t gx = (int64_t)p1.x - rq.dst[0], gy = (int64_t)p1.y - rq.dst[1],
                            gz = (int64_t)p1.z - rq.dst[2];
              int st = -1;
              if (c1 < w.sep2) st = 1;
              else if (below) st = 2;
              else if (gx * gx + gy * gy + gz * gz < w.cap2) st = 0;
              else if (k1 >= w.max_steps) st = 3;
              if (st >= 0) {
                ctl->status = st;
                ctl->fail_step = st == 0 ? -1 : k1;
                ctl->done = 1;
              }
            }
          }
        }
      }
      if (args.eval && rank == 0) {
        for (int i = tid; i < AW; i += NT) {
          args.dbg_v[i] = s_fix[i];
          args.dbg_s[i] = s_sfix[i];
        }
      }
      __syncthreads();
      if (ctl->done) break;
    }

    // ------------------------------------------------------------ request epilogue
    if (rank == 0 && tid == 0 && !args.eval) {
      Out o;
      o.status = ctl->status;
      o.n_states = ctl->k + 1;
      o.fail_step = ctl->fail_step;
      o.n_near_ties = ctl->n_near;
      o.n_exact = ctl->n_exact;
      o.steps_run = ctl->steps_run;
      o.min_sep_d2 = ctl->min_sep;
      o.pad = 0;
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
  }
}

// ----------------------------------------------------------------------------- append / influence
// Append accepted plans to the time rows (Sec V: "automatically stored in the database
// of accepted flight plans").  Slots are assigned by the host in plan-id order.
__global__ void append_kernel(int32_t* rows, int32_t cap, int64_t horizon, const AppendPlan* plans) {
  const AppendPlan P = plans[blockIdx.y];
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P.n; i += gridDim.x * blockDim.x) {
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

// First decision step of request i whose computation could see plan j (|q_i(k) - p_j(K')|
// < bound for K' in {K, K+1}); INT_MAX if none.  Conservative and exact (DESIGN.md a10).
__global__ void influence_kernel(const int32_t* traj, int32_t cap, const int32_t* n_states, const int64_t* t0,
                                 const InflPair* pairs, int64_t bound2, int32_t* kfirst) {
  __shared__ int32_t best;
  const InflPair pr = pairs[blockIdx.x];
  if (threadIdx.x == 0) best = INT_MAX;
  __syncthreads();
  const int ni = n_states[pr.i], nj = n_states[pr.j];
  const int64_t ti = t0[pr.i], tj = t0[pr.j];
  const int kmax = ni > 1 ? ni - 1 : 1;  // decisions 0..n-2 (state 0 check included in k = 0)
  const int32_t* qi = traj + (size_t)pr.i * cap * 3;
  const int32_t* pj = traj + (size_t)pr.j * cap * 3;
  for (int k = threadIdx.x; k < kmax; k += blockDim.x) {
    if (k >= best) break;
    const int64_t K = ti + k;
#pragma unroll
    for (int d = 0; d < 2; ++d) {
      const int64_t idx = K + d - tj;
      if (idx < 0 || idx >= nj) continue;
      const int64_t dx = qi[3 * k] - pj[3 * idx], dy = qi[3 * k + 1] - pj[3 * idx + 1], dz = qi[3 * k + 2] - pj[3 * idx + 2];
      if (dx * dx + dy * dy + dz * dz < bound2) {
        atomicMin(&best, k);
        break;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) kfirst[blockIdx.x] = best;
}

// ----------------------------------------------------------------------------- launchers
template <int C>
static cudaError_t launch_walk_t(const World& w, const WalkArgs& a, int cluster, int n_clusters, int threads,
                                 int chunk, cudaStream_t s) {
  Layout L;
  L.build(w.HL, chunk, threads, C, w.n_turn * w.W, w.A, w.A * w.W);
  cudaError_t e = cudaFuncSetAttribute(walk_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  if (cluster > 8) {
    e = cudaFuncSetAttribute(walk_kernel<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
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
  return cudaLaunchKernelEx(&cfg, walk_kernel<C>, w, a, chunk);
}

template <int C>
static cudaError_t max_clusters_t(const World& w, int cluster, int threads, int chunk, int* out) {
  Layout L;
  L.build(w.HL, chunk, threads, C, w.n_turn * w.W, w.A, w.A * w.W);
  cudaError_t e = cudaFuncSetAttribute(walk_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.total);
  if (e != cudaSuccess) return e;
  if (cluster > 8) {
    e = cudaFuncSetAttribute(walk_kernel<C>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
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
  return cudaOccupancyMaxActiveClusters(out, walk_kernel<C>, &cfg);
}

cudaError_t launch_walk(const World& w, const WalkArgs& a, int n_climb, int cluster, int n_clusters, int threads,
                        int chunk, cudaStream_t s) {
  switch (n_climb) {
    case 1: return launch_walk_t<1>(w, a, cluster, n_clusters, threads, chunk, s);
    case 3: return launch_walk_t<3>(w, a, cluster, n_clusters, threads, chunk, s);
    case 5: return launch_walk_t<5>(w, a, cluster, n_clusters, threads, chunk, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t walk_max_clusters(const World& w, int n_climb, int cluster, int threads, int chunk, int* out) {
  switch (n_climb) {
    case 1: return max_clusters_t<1>(w, cluster, threads, chunk, out);
    case 3: return max_clusters_t<3>(w, cluster, threads, chunk, out);
    case 5: return max_clusters_t<5>(w, cluster, threads, chunk, out);
    default: return cudaErrorInvalidValue;
  }
}

size_t walk_smem_bytes(const World& w, int n_climb, int threads, int chunk) {
  Layout L;
  L.build(w.HL, chunk, threads, n_climb, w.n_turn * w.W, w.A, w.A * w.W);
  return L.total;
}

cudaError_t launch_append(int32_t* rows, int32_t row_cap, int64_t horizon, const AppendPlan* plans, int n_plans,
                          int max_n, cudaStream_t s) {
  if (n_plans <= 0) return cudaSuccess;
  dim3 grid((max_n + 255) / 256, n_plans, 1);
  append_kernel<<<grid, 256, 0, s>>>(rows, row_cap, horizon, plans);
  return cudaGetLastError();
}

cudaError_t launch_influence(const int32_t* traj, int32_t cap, const int32_t* n_states, const int64_t* t0,
                             const InflPair* pairs, int n_pairs, int64_t bound2, int32_t* kfirst, cudaStream_t s) {
  if (n_pairs <= 0) return cudaSuccess;
  influence_kernel<<<n_pairs, 256, 0, s>>>(traj, cap, n_states, t0, pairs, bound2, kfirst);
  return cudaGetLastError();
}

}  // namespace fmdp

// Hot-loop variants in isolation (round 2): the walker's C = 3 loop WITH the level-climb skip
// (20 FFMA2 + 15 FMNMX3 + 10 LDS.128 per plan pair), 1 CTA x 384 threads per SM, 12 warps =
// 8 columns x 4 plan groups.  Variants differ only in how the pair records are loaded:
//   V0 as in the kernel (first tau of the next pair prefetched; register rotation = 8 moves)
//   V1 no prefetch        V2 two pairs per iteration, no prefetch
//   V3 ping-pong prefetch (two pairs per iteration, no rotation moves)
//   V4 scalar FFMA / FMNMX3 form of the same arithmetic (no packed pairs)
// usage: hotbench2 [pairs_per_cta] [reps]   prints pairs/clk/SM (pairs incl. the level climb)
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float lo, float hi) { f2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 d; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ float min3(float a, f2 p) {
  float lo, hi, r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p));
  asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo_(f2 p) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p)); return lo; }
__device__ __forceinline__ float hi_(f2 p) { float lo, hi; asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p)); return hi; }
__device__ __forceinline__ float fmin3(float a, float b, float c) { float r; asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c)); return r; }
constexpr int C = 3, NTAU = 5, PS = 40, NGW = 4;
#define PAIR(E)                                                                                          \
  {                                                                                                      \
    f2 h_[NTAU];                                                                                         \
    _Pragma("unroll") for (int t_ = 0; t_ < NTAU; ++t_) h_[t_] = fma2(sx2, (E)[2 * t_].x, (E)[2 * t_ + 1].y); \
    _Pragma("unroll") for (int t_ = 0; t_ < NTAU; ++t_) h_[t_] = fma2(sy2, (E)[2 * t_].y, h_[t_]);     \
    _Pragma("unroll") for (int c_ = 0; c_ < C; ++c_)                                                     \
      _Pragma("unroll") for (int t_ = 0; t_ < NTAU; ++t_)                                                \
        m[c_][t_] = min3(m[c_][t_], c_ == 1 ? h_[t_] : fma2(sz2[c_], (E)[2 * t_ + 1].x, h_[t_]));       \
  }
// scalar form: E as float4 records [X X' Y Y'] [Z Z' Q Q'] per tau
#define PAIRS(E)                                                                                         \
  {                                                                                                      \
    _Pragma("unroll") for (int t_ = 0; t_ < NTAU; ++t_) {                                                \
      const float4 a_ = (E)[2 * t_], b_ = (E)[2 * t_ + 1];                                               \
      const float h0 = fmaf(sy, a_.z, fmaf(sx, a_.x, b_.z)), h1 = fmaf(sy, a_.w, fmaf(sx, a_.y, b_.w));   \
      m[0][t_] = fmin3(m[0][t_], fmaf(sz0, b_.x, h0), fmaf(sz0, b_.y, h1));                              \
      m[1][t_] = fmin3(m[1][t_], h0, h1);                                                                \
      m[2][t_] = fmin3(m[2][t_], fmaf(sz2s, b_.x, h0), fmaf(sz2s, b_.y, h1));                            \
    }                                                                                                    \
  }

template <int V>
__global__ void __launch_bounds__(384, 1) hot(int npairs, int reps, float* out, long long* cyc) {
  extern __shared__ __align__(16) float s_cen[];
  for (int i = threadIdx.x; i < npairs * PS; i += blockDim.x) s_cen[i] = (float)((i * 7919) % 4001 - 2000);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int CPW = 32 / NGW, grp = lane / CPW, col = warp * CPW + lane % CPW;
  const float sx = 2.f * col, sy = -3.f * col, sz0 = -16.f * (col % 10), sz2s = 16.f * (col % 10);
  const f2 sx2 = pk2(sx, sx), sy2 = pk2(sy, sy);
  f2 sz2[C];
  sz2[0] = pk2(sz0, sz0); sz2[1] = 0; sz2[2] = pk2(sz2s, sz2s);
  float m[C][NTAU];
  for (int c = 0; c < C; ++c)
    for (int t = 0; t < NTAU; ++t) m[c][t] = 3.0e38f;
  const ulonglong2* cen2 = reinterpret_cast<const ulonglong2*>(s_cen);
  const int cstep = (PS / 4) * NGW;
  __syncthreads();
  const long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    const ulonglong2* c8 = cen2 + (PS / 4) * grp;
    if (V == 0) {
      ulonglong2 n0 = make_ulonglong2(0, 0), n1 = n0;
      if (grp < npairs) { n0 = c8[0]; n1 = c8[1]; }
      for (int pp = grp; pp < npairs; pp += NGW, c8 += cstep) {
        ulonglong2 e[10];
        e[0] = n0; e[1] = n1;
#pragma unroll
        for (int i = 2; i < 10; ++i) e[i] = c8[i];
        if (pp + NGW < npairs) { n0 = c8[cstep]; n1 = c8[cstep + 1]; }
        PAIR(e)
      }
    } else if (V == 1) {
      for (int pp = grp; pp < npairs; pp += NGW, c8 += cstep) {
        ulonglong2 e[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) e[i] = c8[i];
        PAIR(e)
      }
    } else if (V == 2) {
      int pp = grp;
      for (; pp + NGW < npairs; pp += 2 * NGW, c8 += 2 * cstep) {
        ulonglong2 e[10], g[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) { e[i] = c8[i]; g[i] = c8[cstep + i]; }
        PAIR(e)
        PAIR(g)
      }
      if (pp < npairs) {
        ulonglong2 e[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) e[i] = c8[i];
        PAIR(e)
      }
    } else if (V == 3) {
      ulonglong2 a0 = make_ulonglong2(0, 0), a1 = a0, b0 = a0, b1 = a0;
      if (grp < npairs) { a0 = c8[0]; a1 = c8[1]; }
      int pp = grp;
      for (; pp + NGW < npairs; pp += 2 * NGW, c8 += 2 * cstep) {
        ulonglong2 e[10];
        e[0] = a0; e[1] = a1;
#pragma unroll
        for (int i = 2; i < 10; ++i) e[i] = c8[i];
        b0 = c8[cstep]; b1 = c8[cstep + 1];
        PAIR(e)
        ulonglong2 g[10];
        g[0] = b0; g[1] = b1;
#pragma unroll
        for (int i = 2; i < 10; ++i) g[i] = c8[cstep + i];
        if (pp + 2 * NGW < npairs) { a0 = c8[2 * cstep]; a1 = c8[2 * cstep + 1]; }
        PAIR(g)
      }
      if (pp < npairs) {
        ulonglong2 e[10];
        e[0] = a0; e[1] = a1;
#pragma unroll
        for (int i = 2; i < 10; ++i) e[i] = c8[i];
        PAIR(e)
      }
    } else {
      const float4* c4 = reinterpret_cast<const float4*>(c8);
      for (int pp = grp; pp < npairs; pp += NGW, c4 += cstep) {
        float4 e[10];
#pragma unroll
        for (int i = 0; i < 10; ++i) e[i] = c4[i];
        PAIRS(e)
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float acc = 0.f;
  for (int c = 0; c < C; ++c)
    for (int t = 0; t < NTAU; ++t) acc += m[c][t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(int npairs, int reps) {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 384 * 4); cudaMalloc(&cyc, 148 * 8);
  const int smem = npairs * PS * 4;
  cudaFuncSetAttribute(hot<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  hot<V><<<148, 384, smem>>>(npairs, reps, out, cyc);
  hot<V><<<148, 384, smem>>>(npairs, reps, out, cyc);
  cudaDeviceSynchronize();
  long long c[148]; cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  double mean = 0; for (int i = 0; i < 148; ++i) mean += c[i]; mean /= 148;
  const double pairs = 96.0 * C * NTAU * 2 * npairs * reps;
  printf("V%d npairs=%d reps=%d cycles=%.0f pairs/clk/SM=%.2f err=%s\n", V, npairs, reps, mean, pairs / mean,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}
int main(int argc, char** argv) {
  const int npairs = argc > 1 ? atoi(argv[1]) : 96, reps = argc > 2 ? atoi(argv[2]) : 200;
  run<0>(npairs, reps); run<1>(npairs, reps); run<2>(npairs, reps); run<3>(npairs, reps); run<4>(npairs, reps);
  return 0;
}

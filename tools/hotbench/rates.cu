// Instruction-rate probe (B200, sm_100a): issue rate per SMSP of the FP32 forms the hot loop can
// use -- 3-register FFMA / FFMA2, the constant-operand FFMA, FMUL2 / FADD2 (two register pairs),
// FMNMX3 -- 384 threads per SM (12 warps = 3 per SMSP, as the walker), 8 independent chains per
// thread.  Prints warp-instructions per clock per SMSP and lane-ops per clock per SMSP.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk2(float lo, float hi) { f2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { f2 d; asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { f2 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float ffma(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float fmn3(float a, float b, float c) { float d; asm volatile("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ int iadd3(int a, int b, int c) { int d; asm volatile("add.s32 %0, %1, %2;\n\tadd.s32 %0, %0, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ int imn3(int a, int b, int c) { int d; asm volatile("min.s32 %0, %1, %2;\n\tmin.s32 %0, %0, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c)); return d; }
__device__ __forceinline__ float fmn2(float a, float b) { float d; asm volatile("min.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
__device__ __forceinline__ float fadd(float a, float b) { float d; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }

constexpr int NCH = 8;
template <int V>
__global__ void __launch_bounds__(384, 1) rate(int iters, float kpar, float* out, long long* cyc) {
  const float s = 1.0f + threadIdx.x * 1e-7f;
  float a[NCH], b[NCH], c[NCH];
  int ia[NCH], ib[NCH];
  const int is = (int)threadIdx.x * 3 + (int)kpar;
  f2 p[NCH], q[NCH];
  for (int i = 0; i < NCH; ++i) {
    c[i] = s - i; ia[i] = threadIdx.x + i; ib[i] = (int)(kpar * i) - 7;
    a[i] = s + i; b[i] = kpar * (0.999f - i * 1e-6f) + threadIdx.x * 1e-9f;
    p[i] = pk2(a[i], a[i] + 1); q[i] = pk2(b[i], b[i] * 0.5f);
  }
  const f2 m2 = pk2(s * 0.5f, s * 0.25f);
  const float s2 = s * kpar;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
#pragma unroll
      for (int i = 0; i < NCH; ++i) {
        if (V == 0) p[i] = fma2(p[i], q[i], m2);                 // FFMA2 3-reg
        if (V == 1) a[i] = ffma(a[i], b[i], s2);                 // FFMA 3-reg
        if (V == 2) a[i] = ffma(a[i], kpar, b[i]);               // FFMA, constant operand
        if (V == 3) p[i] = mul2(p[i], q[i]);                     // FMUL2
        if (V == 4) p[i] = add2(p[i], q[i]);                     // FADD2
        if (V == 5) a[i] = fmn3(a[i], b[i], s2);                 // FMNMX3
        if (V == 6) a[i] = fadd(a[i], b[i]);                     // FADD
        if (V == 7) { p[i] = fma2(p[i], q[i], m2); a[i] = fmn3(a[i], b[i], s); }  // FFMA2 + FMNMX3 mixed
        if (V == 8) { p[i] = fma2(p[i], q[i], m2); ia[i] = iadd3(ia[i], ib[i], is); }  // FFMA2 + IADD3
        if (V == 9) { p[i] = fma2(p[i], q[i], m2); a[i] = fmn2(a[i], b[i]); }         // FFMA2 + FMNMX
        if (V == 10) { c[i] = ffma(c[i], b[i], s2); a[i] = fmn3(a[i], b[i], s2); }     // FFMA + FMNMX3
        if (V == 11) { p[i] = mul2(p[i], q[i]); a[i] = fmn3(a[i], b[i], s2); }         // FMUL2 + FMNMX3
        if (V == 12) { p[i] = fma2(p[i], q[i], m2); ia[i] = imn3(ia[i], ib[i], is); }  // FFMA2 + VIMNMX3
        if (V == 13) { ia[i] = iadd3(ia[i], ib[i], is); }                              // IADD3
        if (V == 14) { ia[i] = imn3(ia[i], ib[i], is); }                               // VIMNMX3
      }
    }
  }
  const long long t1 = clock64();
  float acc = 0.f;
  for (int i = 0; i < NCH; ++i) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(p[i]));
    acc += a[i] + c[i] + lo + hi + (float)ia[i];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int V>
void run(const char* name, int lanes_per_inst) {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 384 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 2000;
  rate<V><<<148, 384>>>(iters, 1.0001f, out, cyc);
  rate<V><<<148, 384>>>(iters, 1.0001f, out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double winst = (double)iters * 8 * NCH * (V >= 7 && V <= 12 ? 2 : 1) * 3;  // warp-instructions per SMSP (3 warps)
  printf("%-28s cycles=%lld warp-inst/clk/SMSP=%.3f lane-ops/clk/SMSP=%.1f err=%s\n", name, mx, winst / mx,
         winst / mx * 32 * lanes_per_inst / (V >= 7 && V <= 12 ? 1.5 : 1.0), cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  run<0>("FFMA2 3-reg", 2);
  run<1>("FFMA 3-reg", 1);
  run<2>("FFMA const operand", 1);
  run<3>("FMUL2", 2);
  run<4>("FADD2", 2);
  run<5>("FMNMX3", 1);
  run<6>("FADD", 1);
  run<7>("FFMA2 + FMNMX3 (mix)", 2);
  run<8>("FFMA2 + IADD3", 2);
  run<9>("FFMA2 + FMNMX", 2);
  run<10>("FFMA + FMNMX3", 2);
  run<11>("FMUL2 + FMNMX3", 2);
  run<12>("FFMA2 + VIMNMX3", 2);
  run<13>("IADD3", 1);
  run<14>("VIMNMX3", 1);
  return 0;
}

// microbench.cu -- pipe-throughput probes that size the IDW issue budget on
// sm_100a: FFMA vs FFMA2 (packed fp32), MUFU.RCP, MUFU+FFMA2 mixes, DFMA, and
// the accuracy of rcp.approx.ftz.f64 (how many Newton steps fp64 needs).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

typedef unsigned long long u64;
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) {
  u64 r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c)); return r;
}
__device__ __forceinline__ float rcpa(float a) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(a)); return r; }

// 8 independent FFMA chains
__global__ void k_ffma(float *out, int iters) {
  float a[8]; float b = 1.0001f, c = 1e-7f;
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f32 %0, %0, %1, %2;" : "+f"(a[k]) : "f"(b), "f"(c));
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345f) out[0] = s;
}
// 8 independent FFMA2 chains (16 fp32 FMAs per step)
__global__ void k_ffma2(float *out, int iters) {
  u64 a[8]; u64 b, c;
  asm("mov.b64 %0, {%1,%1};" : "=l"(b) : "f"(1.0001f)); asm("mov.b64 %0, {%1,%1};" : "=l"(c) : "f"(1e-7f));
  for (int k = 0; k < 8; ++k) asm("mov.b64 %0, {%1,%2};" : "=l"(a[k]) : "f"(threadIdx.x * 1e-3f + k), "f"(k * 0.5f));
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma2(a[k], b, c);
  u64 s = 0; for (int k = 0; k < 8; ++k) s ^= a[k];
  if (s == 12345) out[0] = 1;
}
// MUFU.RCP (+FADD to defeat folding)
__global__ void k_mufu(float *out, int iters) {
  float a[8]; for (int k = 0; k < 8; ++k) a[k] = 1.0f + threadIdx.x * 1e-3f + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("{ rcp.approx.ftz.f32 %0, %0;\n\t add.ftz.f32 %0, %0, 0f3F800000; }" : "+f"(a[k]));
  float s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345f) out[0] = s;
}
// mix: per step, 8 MUFU (each with its FADD) + 8*R FFMA2
template <int R>
__global__ void k_mix(float *out, int iters) {
  float a[8]; u64 f[8]; u64 b, c;
  asm("mov.b64 %0, {%1,%1};" : "=l"(b) : "f"(1.0001f)); asm("mov.b64 %0, {%1,%1};" : "=l"(c) : "f"(1e-7f));
  for (int k = 0; k < 8; ++k) { a[k] = 1.0f + threadIdx.x * 1e-3f + k; asm("mov.b64 %0, {%1,%1};" : "=l"(f[k]) : "f"(a[k])); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("{ rcp.approx.ftz.f32 %0, %0;\n\t add.ftz.f32 %0, %0, 0f3F800000; }" : "+f"(a[k]));
#pragma unroll
      for (int r = 0; r < R; ++r) f[k] = fma2(f[k], b, c);
    }
  }
  float s = 0; u64 t = 0; for (int k = 0; k < 8; ++k) { s += a[k]; t ^= f[k]; }
  if (s == 1.2345f || t == 77) out[0] = s;
}
__global__ void k_dfma(double *out, int iters) {
  double a[8]; double b = 1.0000001, c = 1e-9;
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k]) : "d"(b), "d"(c));
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_rcp64_acc(const double *x, int n, double *maxrel0, double *maxrel1) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double a = x[i], y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  double ex = 1.0 / a;
  double e0 = fabs(y - ex) / ex;
  double e = fma(-a, y, 1.0); double y1 = fma(y, e, y);
  double e1 = fabs(y1 - ex) / ex;
  maxrel0[i] = e0; maxrel1[i] = e1;
}

template <class F>
float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize();
  cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float *fo; double *dbo; CK(cudaMalloc(&fo, 64)); CK(cudaMalloc(&dbo, 64));
  const int blocks = sms * 8, th = 256, it = 4096;
  const double thr = (double)blocks * th;
  printf("{\"sms\": %d, \"clock_khz\": %d", sms, clk);
  float ms;
  ms = timeit([&] { k_ffma<<<blocks, th>>>(fo, it); });
  printf(", \"ffma_per_clk_sm_at_max\": %.2f, \"ffma_Gop_s\": %.1f", thr * 8 * it / (ms * 1e-3) / sms / (clk * 1e3), thr * 8 * it / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_ffma2<<<blocks, th>>>(fo, it); });
  printf(", \"ffma2_lanes_per_clk_sm_at_max\": %.2f, \"ffma2_lane_Gop_s\": %.1f", thr * 16 * it / (ms * 1e-3) / sms / (clk * 1e3), thr * 16 * it / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_mufu<<<blocks, th>>>(fo, it); });
  double mufu = thr * 8 * it / (ms * 1e-3);
  printf(", \"mufu_rcp_per_clk_sm_at_max\": %.2f, \"mufu_G_s\": %.1f", mufu / sms / (clk * 1e3), mufu / 1e9);
  ms = timeit([&] { k_mix<1><<<blocks, th>>>(fo, it); }); printf(", \"mix1_rcp_G_s\": %.1f", thr * 8 * it / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_mix<2><<<blocks, th>>>(fo, it); }); printf(", \"mix2_rcp_G_s\": %.1f", thr * 8 * it / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_mix<3><<<blocks, th>>>(fo, it); }); printf(", \"mix3_rcp_G_s\": %.1f", thr * 8 * it / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_mix<4><<<blocks, th>>>(fo, it); }); printf(", \"mix4_rcp_G_s\": %.1f", thr * 8 * it / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_mix<6><<<blocks, th>>>(fo, it); }); printf(", \"mix6_rcp_G_s\": %.1f", thr * 8 * it / (ms * 1e-3) / 1e9);
  ms = timeit([&] { k_dfma<<<blocks, th>>>(dbo, it); });
  printf(", \"dfma_per_clk_sm_at_max\": %.2f", thr * 8 * it / (ms * 1e-3) / sms / (clk * 1e3));
  const int n = 1 << 22;
  double *x, *r0, *r1; CK(cudaMallocManaged(&x, n * 8)); CK(cudaMallocManaged(&r0, n * 8)); CK(cudaMallocManaged(&r1, n * 8));
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x[i] = ldexp(1.0 + (s >> 11) * 0x1p-53, (int)(s % 60) - 30); }
  k_rcp64_acc<<<(n + 255) / 256, 256>>>(x, n, r0, r1); CK(cudaDeviceSynchronize());
  double m0 = 0, m1 = 0; for (int i = 0; i < n; ++i) { m0 = fmax(m0, r0[i]); m1 = fmax(m1, r1[i]); }
  printf(", \"rcp64_approx_maxrel\": %.3e, \"rcp64_newton1_maxrel\": %.3e}\n", m0, m1);
  return 0;
}

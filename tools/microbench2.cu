// microbench2.cu -- fp64 issue facts: MUFU.RCP64H rate, F2F conversion rates.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench2 tools/microbench2.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_rcp64(double *out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("{ rcp.approx.ftz.f64 %0, %0;\n\t add.f64 %0, %0, 0d3FF0000000000000; }" : "+d"(a[k]));
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_f2f(double *out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float f; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f) : "d"(a[k]));
      asm volatile("cvt.f64.f32 %0, %1;" : "=d"(a[k]) : "f"(f));
    }
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_dadd(double *out, int iters) {
  double a[8];
  for (int k = 0; k < 8; ++k) a[k] = 1.0 + threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) asm volatile("add.f64 %0, %0, 0d3FF0000000000000;" : "+d"(a[k]));
  double s = 0; for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 1.2345) out[0] = s;
}
template <class F> float timeit(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); cudaDeviceSynchronize(); cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms;
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double *o; cudaMalloc(&o, 64);
  const int blocks = sms * 8, th = 256, it = 2048; const double thr = (double)blocks * th;
  float ms = timeit([&] { k_rcp64<<<blocks, th>>>(o, it); });
  printf("{\"rcp64h_plus_dadd_per_clk_sm_at_max\": %.2f", thr * 8 * it / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_f2f<<<blocks, th>>>(o, it); });
  printf(", \"f2f_roundtrip_per_clk_sm_at_max\": %.2f", thr * 8 * it / (ms * 1e-3) / sms / (clk * 1e3));
  ms = timeit([&] { k_dadd<<<blocks, th>>>(o, it); });
  printf(", \"dadd_per_clk_sm_at_max\": %.2f}\n", thr * 8 * it / (ms * 1e-3) / sms / (clk * 1e3));
  return 0;
}

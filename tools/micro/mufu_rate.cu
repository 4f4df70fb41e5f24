// Microbenchmark: achievable MUFU.EX2 rate per SM (and with a mix of FMA-pipe
// work), to know the real ceiling of K1's exp work.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int MODE>
__global__ void k(float* out, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; i++) a[i] = threadIdx.x * 1e-6f + i * 1e-3f;
  float2 s = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      float2 y = make_float2(a[i], a[i + 1]);
      if (MODE >= 1) y = __ffma2_rn(y, make_float2(0.999f, 0.999f), make_float2(-1e-4f, -1e-4f));
      float2 e = make_float2(ex2(y.x), ex2(y.y));
      if (MODE >= 2) s = __fadd2_rn(s, e);
      else s.x += e.x - e.y;
      a[i] = y.x * 0.5f; a[i + 1] = y.y * 0.5f;
    }
  }
  if (s.x == 1.2345f) out[0] = s.y;
}
int main() {
  float* o; cudaMalloc(&o, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  for (int mode = 0; mode < 3; mode++)
    for (int warps : {8, 16, 32}) {
      auto f = mode == 0 ? k<0> : mode == 1 ? k<1> : k<2>;
      f<<<sms * 2, warps * 32>>>(o, 16);
      cudaEventRecord(e0);
      f<<<sms * 2, warps * 32>>>(o, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double mufu = double(sms) * 2 * warps * 32 * iters * 16;
      printf("mode %d warps/CTA %2d (2 CTA/SM): %.3f ms  %.3e MUFU/s  = %.2f /clk/SM at max clock %d MHz\n", mode, warps, ms,
             mufu / ms * 1e3, mufu / ms * 1e3 / (sms * (clk * 1e3)), clk / 1000);
    }
  return 0;
}

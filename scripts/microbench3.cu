// Does MUFU work overlap the FP32 pipe?  FFMA2 stream with k MUFU.SIN per 12 FFMA2 (our kernel's
// ratio is ~2 MUFU per 12 FP32 lane-op pairs).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pk(float a, float b){ unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(unsigned long long r){ float a,b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a+b; }
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c){ unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;}
constexpr int IT = 2048;
template <int NMUFU, bool SCALAR>
__global__ void k(float* out, float b0, float c0) {
  unsigned long long a[12], b = pk(b0, b0 + 1e-7f), c = pk(c0, c0 - 1e-7f);
  float f[12];
  float m[4];
#pragma unroll
  for (int i = 0; i < 12; ++i) { a[i] = pk(threadIdx.x * 1e-3f + i, i * 1e-3f); f[i] = i * 1e-3f + threadIdx.x; }
#pragma unroll
  for (int i = 0; i < 4; ++i) m[i] = threadIdx.x * 1e-4f + i;
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      if (SCALAR) { f[i] = fmaf(f[i], b0, c0); f[i] = fmaf(f[i], b0, c0); }
      else a[i] = fma2(a[i], b, c);
    }
#pragma unroll
    for (int i = 0; i < NMUFU; ++i) m[i & 3] = __sinf(m[i & 3]);
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < 12; ++i) t += lo(a[i]) + f[i];
  for (int i = 0; i < 4; ++i) t += m[i];
  if (t == 1234.5f) out[0] = t;
}
template <int NMUFU, bool SCALAR>
void run() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * 4, thr = 512;
  float* o; cudaMalloc(&o, 4);
  k<NMUFU, SCALAR><<<grid, thr>>>(o, 1.0001f, 1e-4f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<NMUFU, SCALAR><<<grid, thr>>>(o, 1.0001f, 1e-4f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double lane_fma = (double)grid * thr * IT * 24;
  double mufu = (double)grid * thr * IT * NMUFU;
  printf("%s + %d MUFU per 24 lane-FMA: %.1f lane-FMA/clk/SM, %.2f MUFU/clk/SM (at 1965 MHz)\n", SCALAR ? "FFMA x24 " : "FFMA2 x12", NMUFU,
         lane_fma / (ms * 1e-3) / sms / 1.965e9, mufu / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
  run<0, false>(); run<1, false>(); run<2, false>(); run<4, false>();
  run<0, true>(); run<1, true>(); run<2, true>(); run<4, true>();
  return 0;
}

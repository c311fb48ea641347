// FP32x2 (FFMA2/FMUL2/FADD2, PTX fma.rn.f32x2, sm_100+) throughput vs scalar FFMA, lane-ops/clk/SM.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned long long pk(float a, float b){ unsigned long long r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(unsigned long long r){ float a,b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a+b; }
__device__ __forceinline__ unsigned long long fma2(unsigned long long a, unsigned long long b, unsigned long long c){ unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;}
constexpr int IT = 4096;
template <int MODE>
__global__ void k(float* out, float b0, float c0) {
  unsigned long long a[8], b = pk(b0, b0 + 1e-7f), c = pk(c0, c0 - 1e-7f);
  float s[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { a[i] = pk(threadIdx.x * 1e-3f + i, i * 1e-3f); s[i] = threadIdx.x * 1e-3f + i; }
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fma2(a[i], b, c);
      if (MODE == 1) s[i] = fmaf(s[i], b0, c0);
      if (MODE == 2) { a[i] = fma2(a[i], b, c); s[i] = fmaf(s[i], b0, c0); }
    }
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) t += lo(a[i]) + s[i];
  if (t == 1234.5f) out[0] = t;
}
template <int MODE>
void run(const char* name, double ops_per_inner) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * 4, thr = 512;
  float* o; cudaMalloc(&o, 4);
  k<MODE><<<grid, thr>>>(o, 1.0001f, 1e-4f);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<MODE><<<grid, thr>>>(o, 1.0001f, 1e-4f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = (double)grid * thr * IT * 8 * ops_per_inner;
  printf("%-28s %.2f T lane-FMA/s = %.1f lane-FMA/clk/SM at 1965 MHz\n", name, ops / ms / 1e9, ops / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
  run<0>("FFMA2 (2 lane-FMA/instr)", 2);
  run<1>("FFMA scalar", 1);
  run<2>("FFMA2 + FFMA interleaved", 3);
  run<0>("FFMA2 (2 lane-FMA/instr)", 2);
  return 0;
}

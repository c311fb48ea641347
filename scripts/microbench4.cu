// FFMA2 operand-pattern throughput (lane-FMA/clk/SM): which register patterns of the reverse
// kernel's packed complex MACs issue at the FP32 pipe rate (register-bank / reuse effects).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench4 microbench4.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ float lo(u64 r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return a; }
__device__ __forceinline__ float hi(u64 r) { float a, b; asm("mov.b64 {%0,%1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); return b; }
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 bc(float x) { return pk(x, x); }
constexpr int IT = 2048;
constexpr int N = 8;
template <int MODE>
__global__ void k(float* out, float b0) {
  u64 acc[N], P[N], Q[N];
  float x[N], s[N];
#pragma unroll
  for (int i = 0; i < N; ++i) {
    acc[i] = pk(threadIdx.x * 1e-3f + i, i * 1e-3f);
    const float tf = threadIdx.x * 1e-9f;
    P[i] = pk(b0 + i * 1e-7f + tf, b0 - i * 1e-7f - tf);
    Q[i] = pk(1e-4f * i + tf, 2e-4f - tf);
    x[i] = b0 + 1e-6f * i + tf;
    s[i] = threadIdx.x * 1e-3f + i;
  }
  const u64 T = pk(b0 + threadIdx.x * 1e-9f, -b0 * 0.5f);
  const float xs = b0 * 0.999f + threadIdx.x * 1e-9f;
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      if (MODE == 0) acc[i] = fma2(bc(x[i]), T, acc[i]);         // shared tap pair, distinct scalar
      if (MODE == 1) acc[i] = fma2(bc(xs), P[i], acc[i]);        // shared scalar, distinct pair (tap grads)
      if (MODE == 2) acc[i] = fma2(bc(x[i]), P[i], acc[i]);      // all distinct
      if (MODE == 3) s[i] = fmaf(x[i], lo(P[i]), s[i]);          // scalar FFMA, distinct
      if (MODE == 4) acc[i] = fma2(Q[i], P[i], acc[i]);          // pair x pair, distinct
      if (MODE == 5) { acc[i] = fma2(bc(xs), P[i], acc[i]); acc[(i + 4) % N] = fma2(bc(x[i]), P[i], acc[(i + 4) % N]); }
    }
  }
  float t = 0;
#pragma unroll
  for (int i = 0; i < N; ++i) t += lo(acc[i]) + hi(acc[i]) + s[i];
  if (t == 1234.5f) out[0] = t;
}
template <int MODE>
void run(const char* name, double lane_fma_per_inner) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, 4);
  for (int thr : {256, 512}) {
    int grid = sms * (2048 / thr);
    k<MODE><<<grid, thr>>>(o, 1.0001f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<grid, thr>>>(o, 1.0001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)grid * thr * IT * N * lane_fma_per_inner;
    printf("%-44s thr %d: %.1f lane-FMA/clk/SM at 1965 MHz\n", name, thr, ops / (ms * 1e-3) / sms / 1.965e9);
  }
}
int main() {
  run<0>("FFMA2 shared tap pair, distinct bcast scalar", 2);
  run<1>("FFMA2 shared bcast scalar, distinct pair", 2);
  run<2>("FFMA2 distinct bcast scalar + pair", 2);
  run<3>("FFMA scalar distinct", 1);
  run<4>("FFMA2 pair x pair distinct", 2);
  run<5>("FFMA2 grad pattern (2 per P)", 4);
  return 0;
}

// FP32 FMA-pipe and MUFU throughput on one B200, lane-ops per SM clock (grounds the "alu"
// roofline peak of DESIGN.md).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 microbench.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

template <int MODE>
__global__ void kern(float* out, float b, float c, long long* cyc) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  float bb[8], cc[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) { bb[i] = b + i * 1e-7f; cc[i] = c - i * 1e-7f; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = fmaf(a[i], b, c);            // shared b, c registers
      if (MODE == 1) a[i] = fmaf(a[i], bb[i], cc[i]);    // distinct registers
      if (MODE == 2) a[i] = fmaf(a[i], 0.999f, 1e-3f);   // immediates
      if (MODE == 3) a[i] = __sinf(a[i]);                // MUFU.SIN (+FMUL)
      if (MODE == 4) { float s, co; __sincosf(a[i], &s, &co); a[i] = s + co; }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.f) out[0] = s;
}

template <int MODE>
void run(const char* name, int blocks_per_sm, int threads) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * blocks_per_sm;
  float* out;
  long long* cyc;
  cudaMalloc(&out, 4);
  cudaMalloc(&cyc, grid * sizeof(long long));
  kern<MODE><<<grid, threads>>>(out, 1.0001f, 1e-4f, cyc);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<MODE><<<grid, threads>>>(out, 1.0001f, 1e-4f, cyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long* h = new long long[grid];
  cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  double ops = (double)grid * threads * ITERS * 8;
  double lanes_per_clk_sm = ops / sms / mx;
  printf("%-22s blocks/SM %d thr %4d: %.1f lane-ops/clk/SM, %.2f Tops/s, eff clock %.0f MHz\n", name, blocks_per_sm,
         threads, lanes_per_clk_sm, ops / ms / 1e9, mx / (ms * 1e3));
  cudaFree(out);
  cudaFree(cyc);
  delete[] h;
}

int main() {
  for (int bps : {1, 2, 4}) {
    run<0>("ffma shared b,c", bps, 512);
    run<1>("ffma distinct regs", bps, 512);
    run<2>("ffma immediates", bps, 512);
    run<3>("__sinf", bps, 512);
    run<4>("__sincosf", bps, 512);
  }
  return 0;
}

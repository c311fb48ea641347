// Isolates the cost components of one LDBP forward step (FIR Kh=2 folded + Kerr, R=16/thread):
// MODE 0: pure register compute (in-thread circular halo), no shuffle, no barrier
// MODE 1: + warp shuffles for the halo
// MODE 2: + warp shuffles + __syncthreads per step
// MODE 3: MODE 2 + smem edge exchange (the production exchange)
#include <cstdio>
#include <cuda_runtime.h>
#define LDBP_KH 2
#include "ldbp_kernels.cuh"
#include "ldbp_f32x2.cuh"
using namespace ldbp;
constexpr int KH = 2, R = 16;

template <int MODE>
__global__ void __launch_bounds__(512, 2) stepk(float2* out, const float2* taps, float gm, int steps) {
  __shared__ float2 sh[4 * 32 * KH];
  float2 u[R];
#pragma unroll
  for (int k = 0; k < R; ++k) u[k] = make_float2(1e-2f * (threadIdx.x + k), 1e-2f * k);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  float2 hs[KH + 1];
#pragma unroll
  for (int j = 0; j <= KH; ++j) hs[j] = taps[j];
  float2 hl[KH], hr[KH];
  for (int s = 0; s < steps; ++s) {
    if (MODE == 0 || MODE == 4) {
#pragma unroll
      for (int j = 0; j < KH; ++j) { hl[j] = u[R - KH + j]; hr[j] = u[j]; }
    } else if (MODE == 1 || MODE == 2 || MODE == 6) {
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        hl[j].x = __shfl_up_sync(kFull, u[R - KH + j].x, 1);
        hl[j].y = __shfl_up_sync(kFull, u[R - KH + j].y, 1);
        hr[j].x = __shfl_down_sync(kFull, u[j].x, 1);
        hr[j].y = __shfl_down_sync(kFull, u[j].y, 1);
      }
      if (MODE == 2 || MODE == 6) __syncthreads();
    } else {
      exchange<KH, R>(u, hl, hr, sh, s & 1, lane, warp, nw);
    }
    if (MODE >= 4) {
      float2 v[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        float2 acc = cmul(hs[0], u[k]);
#pragma unroll
        for (int j = 1; j <= KH; ++j) {
          const float2 l = (k - j) < 0 ? hl[KH + k - j] : u[k - j];
          const float2 r = (k + j) >= R ? hr[k + j - R] : u[k + j];
          acc = cmac(acc, hs[j], cadd(l, r));
        }
        const float p = fmaf(acc.x, acc.x, acc.y * acc.y);
        float sn, cs;
        __sincosf(gm * p, &sn, &cs);
        v[k] = crot(acc, cs, sn);
      }
#pragma unroll
      for (int k = 0; k < R; ++k) u[k] = v[k];
    } else {
    float2 acc[R];
    fir_all<KH, R, true>(u, hl, hr, hs, acc);
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = kerr<true>(acc[k], gm);
    }
  }
  float2 t = make_float2(0, 0);
#pragma unroll
  for (int k = 0; k < R; ++k) { t.x += u[k].x; t.y += u[k].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}

template <int MODE>
void run(int threads, int bps, int steps) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = sms * bps * 4;
  float2 *out, *taps;
  cudaMalloc(&out, sizeof(float2) * grid * threads);
  cudaMalloc(&taps, sizeof(float2) * 8);
  float2 h[3] = {{0.9f, 0.1f}, {0.05f, -0.02f}, {0.01f, 0.03f}};
  cudaMemcpy(taps, h, sizeof(h), cudaMemcpyHostToDevice);
  stepk<MODE><<<grid, threads>>>(out, taps, -27.5f, steps);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  stepk<MODE><<<grid, threads>>>(out, taps, -27.5f, steps);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  double ss = (double)grid * threads * R * steps;
  double instr = ss * 24;
  printf("mode %d thr %d bps %d: %.3f ms, %.1f G sample-steps/s, FP32 frac of 148*128*1.965G = %.3f\n", MODE, threads,
         bps, ms, ss / ms / 1e6, instr / (ms * 1e-3) / (148.0 * 128 * 1.965e9));
  cudaFree(out);
  cudaFree(taps);
}

int main() {
  for (int t : {256, 512}) {
    int bps = 1024 / t;
    run<0>(t, bps, 200);
    run<1>(t, bps, 200);
    run<2>(t, bps, 200);
    run<3>(t, bps, 200);
    run<4>(t, bps, 200);
    run<5>(t, bps, 200);
    run<6>(t, bps, 200);
  }
  return 0;
}

// ldbp_tiny.cuh — one-launch training step for tiny problems (BASELINE C1: 4 blocks x 1024 samples,
// M = 4, T = 3), SURVEY.md §8(a) rows a1-a10 in ONE thread-block cluster.
//
// At 16 K sample-steps the training step is pure latency: the segment schedule needs a forward, a
// backward, a reduction and an Adam launch.  Here one cluster of C <= 16 CTAs keeps the whole
// batch in shared memory for the whole step:
//  * B >= 8: C = 8 and CTA r owns whole blocks r, r + C, ... (the circular FIR stays in the CTA);
//  * B < 8:  each block is split into S segments, one per CTA (C = B S), and the Kh-sample halos
//            of every step's FIR input are written straight into the neighbours' shared memory
//            (DSMEM), one cluster barrier per step.
// Rows are stored with Kh-sample halos on both sides, so the FIR reads need no wrap logic.  The
// forward stores u^(0..M-1) (the inputs of every step); the reverse recomputes
// a^(i) = h^(i) (*) u^(i) and v = a e^{j gamma' |a|^2} per step (Eq. (7)) and follows the
// oracle's adjoint literally (oracle/ldbp.py backward): c = Im(g conj v),
// ga = g e^{-j phi} + 2 gamma' c a, dgamma' += c |a|^2, dh_j += ga conj(u_{t-j}),
// gu_s = sum_j conj(h_j) ga_{s+j} — every tap of the (masked) filter, circular per block.
// Per-step partial sums: warp transposing butterfly -> smem [step][warp][v]; after the sweep a
// fixed-order fp64 sum over warps per CTA, then CTA 0 sums the C tables in rank order over DSMEM
// (deterministic), writes the ABI gradient layout (tied +-j with LDBP_SYMMETRIC, masked taps 0)
// and, for the training step, applies adam_elem (adam_kernel's update) from shared memory.
#pragma once

#include <cooperative_groups.h>

namespace ldbp {

constexpr int kTinyMaxThreads = 512;  // <= 128 registers per thread
constexpr int kTinyMaxCluster = 16;
constexpr int kTinyPer = 8;  // samples per thread at most

struct TinyArgs {
  const float2* x;
  const float2* target;
  const float2* taps;      // [M][T]
  const float* gamma;      // [M]
  const uint8_t* mask;     // [M][T] or nullptr
  double* buf;             // [1 + M + 2 M T]
  int B, n, M;
  int S;                   // segments per block (1: whole blocks per CTA)
  int lenmax;              // samples per row: n (S = 1) or ceil(n / S)
  int nrows;               // rows per CTA: ceil(B / C) (S = 1) or 1
  int sym, precise;        // precise: accurate sincosf (LDBP_PRECISE) instead of MUFU
  float seed_scale;        // g = seed_scale (y - target)
  int do_adam;
  AdamArgs adam;           // adam.buf == buf
};

__host__ __device__ constexpr int tiny_vp(int V) { return V <= 2 ? 2 : V <= 4 ? 4 : V <= 8 ? 8 : V <= 16 ? 16 : 32; }

// smem bytes per CTA (identical layout in every CTA of the cluster: rows of stride lenmax + 2 Kh):
// u^(0..M-1), g, two ga buffers (complex), the masked taps, the per-warp float partials of every
// step [M][32][V], the warps' fp64 loss [32], the fp64 per-step table [M V + 1], the gradient
// [1 + M + 2MT], the cluster gather [C][M V + 1] (CTA 0), gamma' [M], the packed sample positions
// [nrows lenmax]
__host__ __device__ constexpr size_t tiny_smem_bytes(int64_t nrows, int64_t lenmax, int M, int T) {
  return sizeof(float2) * (size_t)(nrows * (lenmax + T - 1)) * (M + 3) + sizeof(float2) * (size_t)M * T +
         sizeof(float) * 32 * (size_t)(1 + 2 * T) * M + sizeof(double) * 32 +
         sizeof(double) * ((size_t)M * (1 + 2 * T) + 1) + sizeof(double) * (1 + (size_t)M + 2 * (size_t)M * T) +
         sizeof(double) * kTinyMaxCluster * ((size_t)M * (1 + 2 * T) + 1) + sizeof(float) * (size_t)M +
         sizeof(int) * (size_t)(nrows * lenmax) + 64;
}

template <bool PRECISE>
__device__ __forceinline__ void tiny_sincos(float ph, float* sn, float* cs) {
  if constexpr (PRECISE) sincosf(ph, sn, cs);
  else __sincosf(ph, sn, cs);
}

// Where a row's halos live: S = 1 -> the row itself (circular, any n); S > 1 -> the neighbouring
// segments' rows in their CTAs' shared memory (left neighbour's right halo, right neighbour's
// left halo; len >= Kh is guaranteed by the host).
struct TinyRow {
  int len;          // samples of this row
  int len_left;     // samples of the left neighbour's row (S > 1)
  unsigned rl, rr;  // cluster ranks of the left / right neighbour (S > 1)
};

template <int KH>
__device__ __forceinline__ void tiny_put(cooperative_groups::cluster_group& cl, float2* row, int t, const TinyRow& w,
                                         bool split, float2 v) {
  row[t] = v;
  if (KH == 0) return;
  if (!split) {
    for (int q = t - w.len; q >= -KH; q -= w.len) row[q] = v;
    for (int q = t + w.len; q < w.len + KH; q += w.len) row[q] = v;
  } else {
    if (t < KH) cl.map_shared_rank(row, w.rl)[w.len_left + t] = v;      // left row's right halo
    if (t >= w.len - KH) cl.map_shared_rank(row, w.rr)[t - w.len] = v;  // right row's left halo
  }
}

template <int KH, bool PRECISE>
__global__ void __launch_bounds__(kTinyMaxThreads, 1) tiny_train_kernel(const TinyArgs a) {
  constexpr int T = 2 * KH + 1, V = 1 + 2 * T, VP = tiny_vp(V), REP = 32 / VP;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int r = (int)cl.block_rank(), C = (int)cl.num_blocks();
  const int n = a.n, M = a.M, S = a.S;
  const bool split = S > 1;
  const int nthr = blockDim.x, NW = nthr >> 5;
  // rows of this CTA
  int nrows, b_split = 0, t0 = 0;
  TinyRow w;
  if (split) {
    const int q = r % S;
    b_split = r / S;
    t0 = (int)((int64_t)q * n / S);
    const int t1 = (int)((int64_t)(q + 1) * n / S);
    const int ql = (q + S - 1) % S, qr = (q + 1) % S;
    w.len = t1 - t0;
    w.len_left = (int)((int64_t)(ql + 1) * n / S - (int64_t)ql * n / S);
    w.rl = (unsigned)(b_split * S + ql);
    w.rr = (unsigned)(b_split * S + qr);
    nrows = 1;
  } else {
    nrows = (a.B - r + C - 1) / C;  // blocks r, r + C, ...
    w.len = n;
    w.len_left = n;
    w.rl = w.rr = (unsigned)r;
  }
  const int P = a.lenmax + 2 * KH, L = a.nrows * P;
  const int Nr = nrows * w.len;
  const int MV = M * V;
  extern __shared__ __align__(16) unsigned char tiny_smem[];
  float2* U = reinterpret_cast<float2*>(tiny_smem);    // [M][rows][P]: u^(0..M-1) with halos
  float2* G = U + (size_t)M * L;                       // [rows][P] adjoint g (target during the forward)
  float2* GA = G + L;                                  // [2][rows][P] ga, alternating per step
  float2* H = GA + 2 * L;                              // [M][T] masked taps
  float* red = reinterpret_cast<float*>(H + M * T);    // [M][32 warps][V] float partials
  double* dred = reinterpret_cast<double*>(red + M * 32 * V);  // [32] warps' loss
  double* dpart = dred + 32;                           // [M][V] + loss: this CTA's sums
  double* gbuf = dpart + MV + 1;                       // [1 + M + 2MT] (CTA 0)
  double* gath = gbuf + 1 + M + 2 * M * T;             // [C][M V + 1] (CTA 0)
  float* gam = reinterpret_cast<float*>(gath + kTinyMaxCluster * (MV + 1));  // [M] gamma'
  int* spos = reinterpret_cast<int*>(gam + M);         // [Nr] (row base << 16) | t
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ntap = 2 * M * T, nbuf = 1 + M + ntap;

  // every global input is requested up front (one memory latency, not one per phase): the Adam
  // state of buf element k = tid (CTA 0), gamma', taps, x, and the target (parked in G)
  double th0 = 0.0, m0 = 0.0, v0 = 0.0;
  bool frz = false, zer = false;
  const int ae = tid >= 1 + M ? tid - 1 - M : ntap + tid - 1;  // Adam element of buf index tid
  const bool adam_here = a.do_adam && r == 0 && tid >= 1 && tid < nbuf && nbuf <= nthr;
  if (adam_here) {
    th0 = a.adam.master[ae];
    m0 = a.adam.m[ae];
    v0 = a.adam.v[ae];
    if (ae < ntap) frz = zer = a.adam.mask && !a.adam.mask[ae >> 1];
    else frz = a.adam.glearn && !a.adam.glearn[ae - ntap];
  }
  for (int i = tid; i < M; i += nthr) gam[i] = a.gamma[i];
  for (int i = tid; i < M * T; i += nthr) {  // LDBP_SYMMETRIC reads taps[Kh..T-1] only (h_-j = h_j)
    const int jj = i % T, src = (a.sym && jj < KH) ? i + 2 * (KH - jj) : i;
    H[i] = (a.mask && !a.mask[i]) ? make_float2(0.f, 0.f) : a.taps[src];
  }
  if (split) cl.sync();  // every CTA of the cluster runs before any DSMEM store into it
  // samples s = tid + k nthr of this CTA: packed position table, inputs (halos included)
#pragma unroll 1
  for (int s = tid; s < Nr; s += nthr) {
    const int lb = s / w.len, t = s - lb * w.len, rb = lb * P + KH;
    spos[s] = (rb << 16) | t;
    const size_t gi = split ? (size_t)b_split * n + t0 + t : (size_t)(r + lb * C) * n + t;
    tiny_put<KH>(cl, U + rb, t, w, split, a.x[gi]);
    G[rb + t] = a.target[gi];
  }
  if (split) cl.sync();
  else __syncthreads();

  // forward: u^(i+1) = sigma_i(h^(i) (*) u^(i)); the last step's output seeds g
  double lsum = 0.0;
#pragma unroll 1
  for (int i = 0; i < M; ++i) {
    const float gm = gam[i];
    const float2* ui = U + (size_t)i * L;
    const float2* hi = H + i * T;
    float2* uo = U + (size_t)(i + 1) * L;
    const bool last = i + 1 == M;
#pragma unroll 1
    for (int s = tid; s < Nr; s += nthr) {
      const int sp = spos[s], rb = sp >> 16, t = sp & 0xffff, p = rb + t;
      float2 av = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = -KH; j <= KH; ++j) {  // a_t = sum_j h_j u_{t-j}
        const float2 hj = hi[j + KH], uv = ui[p - j];
        av.x = fmaf(hj.x, uv.x, fmaf(-hj.y, uv.y, av.x));
        av.y = fmaf(hj.x, uv.y, fmaf(hj.y, uv.x, av.y));
      }
      float sn, cs;
      tiny_sincos<PRECISE>(gm * fmaf(av.x, av.x, av.y * av.y), &sn, &cs);
      const float2 v = make_float2(av.x * cs - av.y * sn, av.x * sn + av.y * cs);
      if (!last) {
        tiny_put<KH>(cl, uo + rb, t, w, split, v);
      } else {
        const float2 tv = G[p];
        const float ex = v.x - tv.x, ey = v.y - tv.y;
        lsum += (double)fmaf(ex, ex, ey * ey);
        G[p] = make_float2(a.seed_scale * ex, a.seed_scale * ey);
      }
    }
    if (!last) {  // u^(i+1) (with halos) complete; the seed g is read in place
      if (split) cl.sync();
      else __syncthreads();
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) lsum += __shfl_xor_sync(kFull, lsum, o);
  if (lane == 0) dred[warp] = lsum;

  // reverse sweep: one barrier per step (ga double-buffered; g and the partials are per thread)
#pragma unroll 1
  for (int i = M - 1; i >= 0; --i) {
    const float gm = gam[i];
    const float2* ui = U + (size_t)i * L;
    const float2* hi = H + i * T;
    float2* ga_b = GA + (i & 1) * L;
    float part[VP];
#pragma unroll
    for (int v = 0; v < VP; ++v) part[v] = 0.f;
#pragma unroll 1
    for (int s = tid; s < Nr; s += nthr) {
      const int sp = spos[s], rb = sp >> 16, t = sp & 0xffff, p = rb + t;
      float2 uw[T];  // u_{t-j}, j = jj - KH
#pragma unroll
      for (int jj = 0; jj < T; ++jj) uw[jj] = ui[p - (jj - KH)];
      float2 av = make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < T; ++jj) {
        const float2 hj = hi[jj], uv = uw[jj];
        av.x = fmaf(hj.x, uv.x, fmaf(-hj.y, uv.y, av.x));
        av.y = fmaf(hj.x, uv.y, fmaf(hj.y, uv.x, av.y));
      }
      const float pw = fmaf(av.x, av.x, av.y * av.y);
      float sn, cs;
      tiny_sincos<PRECISE>(gm * pw, &sn, &cs);
      const float2 v = make_float2(av.x * cs - av.y * sn, av.x * sn + av.y * cs);
      const float2 g = G[p];
      const float c = fmaf(g.y, v.x, -g.x * v.y);  // Im(g conj v)
      const float2 ga = make_float2(fmaf(g.x, cs, g.y * sn) + 2.f * gm * c * av.x,  // g e^{-j phi} + 2 gm c a
                                    fmaf(g.y, cs, -g.x * sn) + 2.f * gm * c * av.y);
      tiny_put<KH>(cl, ga_b + rb, t, w, split, ga);
      part[0] = fmaf(c, pw, part[0]);
#pragma unroll
      for (int jj = 0; jj < T; ++jj) {  // dh_j += ga conj(u_{t-j})
        const float2 uv = uw[jj];
        part[1 + 2 * jj] = fmaf(ga.x, uv.x, fmaf(ga.y, uv.y, part[1 + 2 * jj]));
        part[2 + 2 * jj] = fmaf(ga.y, uv.x, fmaf(-ga.x, uv.y, part[2 + 2 * jj]));
      }
    }
    {  // warp totals -> red[i][warp][v] (summed over warps after the sweep)
      const float rv = warp_reduce_scatter<VP>(part, lane);
      const int v = lane / REP;
      if ((lane % REP) == 0 && v < V) red[(i * 32 + warp) * V + v] = rv;
    }
    if (split) cl.sync();  // ga (with halos, local and remote) complete
    else __syncthreads();
    // FIR adjoint: g_s = sum_j conj(h_j) ga_{s+j}
#pragma unroll 1
    for (int s = tid; s < Nr; s += nthr) {
      const int sp = spos[s], p = (sp >> 16) + (sp & 0xffff);
      float2 gu = make_float2(0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < T; ++jj) {
        const float2 hj = hi[jj], gv = ga_b[p + jj - KH];
        gu.x = fmaf(hj.x, gv.x, fmaf(hj.y, gv.y, gu.x));
        gu.y = fmaf(hj.x, gv.y, fmaf(-hj.y, gv.x, gu.y));
      }
      G[p] = gu;
    }
  }
  __syncthreads();  // every step's warp partials and the warps' loss are in shared memory
  // this CTA's per-step sums: one warp per entry, lanes = warps, fixed shuffle tree in fp64
#pragma unroll 1
  for (int k = warp; k <= MV; k += NW) {
    double t = 0.0;
    if (lane < NW) t = k < MV ? (double)red[((k / V) * 32 + lane) * V + k % V] : dred[lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(kFull, t, o);
    if (lane == 0) dpart[k] = t;
  }

  // cluster reduction: CTA 0 gathers the C tables (all remote loads in flight at once), then sums
  // them in rank order
  cl.sync();
  if (r == 0) {
#pragma unroll 1
    for (int e = tid; e < C * (MV + 1); e += nthr) {
      const int q = e / (MV + 1), k = e - q * (MV + 1);
      gath[e] = cl.map_shared_rank(dpart, q)[k];
    }
  }
  cl.sync();  // remote tables read: the other CTAs may exit
  if (r != 0) return;
#pragma unroll 1
  for (int k = tid; k <= MV; k += nthr) {
    double t = 0.0;
#pragma unroll 1
    for (int q = 0; q < C; ++q) t += gath[q * (MV + 1) + k];
    if (k == MV) {
      gbuf[0] = t;
    } else {
      const int i = k / V, v = k - i * V;
      if (v == 0) gbuf[1 + i] = t;
      else gbuf[1 + M + (i * T + ((v - 1) >> 1)) * 2 + ((v - 1) & 1)] = t;  // raw per-tap gradient
    }
  }
  __syncthreads();

  // ABI layout (tied taps g_j + g_-j at both positions with LDBP_SYMMETRIC, masked taps 0), then
  // Adam on the same value: buf index k <-> Adam element (taps first, then gamma')
#pragma unroll 1
  for (int k = tid; k < nbuf; k += nthr) {
    double val = gbuf[k];
    if (k >= 1 + M) {
      const int e = k - 1 - M, tap = e >> 1, i = tap / T, jj = tap - i * T;
      if (a.sym && jj != KH) val += gbuf[1 + M + (i * T + 2 * KH - jj) * 2 + (e & 1)];
      if (a.mask && !a.mask[tap]) val = 0.0;
    }
    a.buf[k] = val;
    if (a.do_adam && k >= 1) {
      if (adam_here) {
        adam_elem_flags(a.adam, ae, val, th0, m0, v0, frz, zer);
      } else {
        const int e2 = k >= 1 + M ? k - 1 - M : ntap + k - 1;
        adam_elem(a.adam, e2, val, a.adam.master[e2], a.adam.m[e2], a.adam.v[e2]);
      }
    }
  }
}

}  // namespace ldbp

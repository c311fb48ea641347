// ldbp_reverse2.cuh — warp-overlapped store-all reverse kernel (
// the same arithmetic as rev_tile_kernel in ldbp_reverse.cuh, a different synchronisation design).
//
// rev_tile_kernel exchanges the Kh-sample adjoint halos of every thread through shared memory and
// a CTA-wide split barrier at EVERY reverse step.  Measured on C3 (ncu, round 1/2): the barrier
// spin (try_wait / nanosleep / branch) is ~6 % of the executed instructions and its branch holds
// 18 % of the stall samples; the kernel is latency-bound at 16 warps/SM.
//
// Here each warp advances on its own:
//   * inside a warp the halos move by shuffles (shfl.sync is the only synchronisation);
//   * warps OVERLAP by one lane on each side: lane 0 of warp w duplicates lane 30 of warp w-1 and
//     lane 31 duplicates lane 1 of warp w+1 (slot p = 30 w + lane, R samples per slot).  Lanes 0 and
//     31 receive no valid halo from outside the warp, so their samples go stale from the outside in,
//     Kh per step; after SW = R / Kh steps lane 0/31 are wholly stale while lanes 1..30 are still
//     exact.  Every SW steps the duplicate lanes are refreshed from the owning warps through shared
//     memory (one __syncthreads per SW steps instead of one barrier wait per step);
//   * only lanes 1..30 own samples (tap / gamma' partials, loss, gout), so every real sample is
//     counted exactly once.
// The CTA's outer halo (H = steps * Kh, rounded to whole slots) is recomputed as in every tile kernel
// of this library.  Per reverse step l (chain rule on Eq. (7)):
//   FIR adjoint g_s = ga_s + sum_j conj(h_j) (ga_{s-j} + ga_{s+j}), tap partials conj(u_s) P_sj,
//   then the NL adjoint of step l-1 on each fresh g_s (nl_adjoint in ldbp_reverse.cuh).
#pragma once

namespace ldbp {

#ifndef LDBP_REV2_NW
#define LDBP_REV2_NW 8  // warps per CTA of the warp-overlapped reverse
#endif
#ifndef LDBP_REV2_R
#define LDBP_REV2_R 12  // samples per thread (slot)
#endif
__host__ __device__ constexpr int rev2_warps(int) { return LDBP_REV2_NW; }
__host__ __device__ constexpr int rev2_r(int) { return LDBP_REV2_R; }
__host__ __device__ constexpr int rev2_slots(int nw) { return 30 * nw + 2; }
#ifdef LDBP_REV2_REGS
__host__ __device__ constexpr int rev2_regs(int) { return LDBP_REV2_REGS; }
#else
__host__ __device__ constexpr int rev2_regs(int kh) { return kh <= 1 ? 96 : 128; }
#endif
// steps between refreshes of the duplicate lanes
__host__ __device__ constexpr int rev2_sw(int kh, int r) { return kh == 0 ? (1 << 30) : r / kh; }

// Outputs s in [S0, SE) of one reverse step (compile-time unrolled), SYM taps only.
template <int KH, int R, bool FAST, bool NORM, bool MASKED, bool NL, int S0, int SE>
__device__ __forceinline__ void rev2_range(const f2x (&g)[R], const f2x (&gl)[KH > 0 ? KH : 1],
                                           const f2x (&gr)[KH > 0 ? KH : 1], const f2x* __restrict__ ub,
                                           const TapP (&hs)[KH + 1], f2x (&A)[KH + 1], f2x (&Bq)[KH + 1],
                                           f2x (&ng)[R], uint32_t own, float gmn, float& dgam_next) {
  if constexpr (S0 < SE) {
    constexpr int s = S0;
    const f2x us = ub[s];
    const bool mine = !MASKED || ((own >> s) & 1u);
    const f2x ux = bcast(lof(us)), uy = bcast(hif(us));
    const f2x g0 = g[s];
    f2x acc = NORM ? g0 : tmul(hs[0], g0);
    if (mine) {
      A[0] = fma2(ux, g0, A[0]);
      Bq[0] = fma2(uy, g0, Bq[0]);
    }
#pragma unroll
    for (int j = 1; j <= KH; ++j) {
      const f2x P = add2(LDBP_WIN(g, gl, gr, s - j), LDBP_WIN(g, gl, gr, s + j));
      acc = tmac(acc, hs[j], P);
      if (mine) {
        A[j] = fma2(ux, P, A[j]);
        Bq[j] = fma2(uy, P, Bq[j]);
      }
    }
    if constexpr (NL) nl_adjoint<FAST, MASKED>(acc, us, gmn, 2.f * gmn, (own >> s) & 1u, dgam_next);
    ng[s] = acc;
    rev2_range<KH, R, FAST, NORM, MASKED, NL, S0 + 1, SE>(g, gl, gr, ub, hs, A, Bq, ng, own, gmn, dgam_next);
  }
}

#ifndef LDBP_REV2_LATE_SHFL
#define LDBP_REV2_LATE_SHFL 1  // shuffle the right halo just before the right boundary outputs
#endif
template <int KH, int R, bool FAST, bool NORM, bool MASKED, bool NL>
__device__ __forceinline__ void rev2_step(f2x (&g)[R], const f2x* __restrict__ ub, const TapP* __restrict__ hs_sm,
                                          uint32_t own, float gmn, float (&dh)[2 * (KH + 1)], float& dgam_next) {
  constexpr int KE = KH > 0 ? KH : 1;
  TapP hs[KH + 1];
#pragma unroll
  for (int j = 0; j <= KH; ++j) hs[j] = hs_sm[j];
  f2x gl[KE], gr[KE];
#pragma unroll
  for (int j = 0; j < KE; ++j) gl[j] = gr[j] = 0ull;
  // lane-1's tail and lane+1's head (lanes 0 / 31 get their own values: stale by design)
  if constexpr (KH > 0) {
#pragma unroll
    for (int j = 0; j < KH; ++j) gl[j] = __shfl_up_sync(kFull, g[R - KH + j], 1);
    if (!LDBP_REV2_LATE_SHFL) {
#pragma unroll
      for (int j = 0; j < KH; ++j) gr[j] = __shfl_down_sync(kFull, g[j], 1);
    }
  }
  f2x A[KH + 1], Bq[KH + 1], ng[R];
#pragma unroll
  for (int j = 0; j <= KH; ++j) A[j] = Bq[j] = 0ull;
  rev2_range<KH, R, FAST, NORM, MASKED, NL, 0, R - KH>(g, gl, gr, ub, hs, A, Bq, ng, own, gmn, dgam_next);
  if constexpr (KH > 0) {
    if (LDBP_REV2_LATE_SHFL) {
#pragma unroll
      for (int j = 0; j < KH; ++j) gr[j] = __shfl_down_sync(kFull, g[j], 1);
    }
  }
  rev2_range<KH, R, FAST, NORM, MASKED, NL, R - KH, R>(g, gl, gr, ub, hs, A, Bq, ng, own, gmn, dgam_next);
#pragma unroll
  for (int j = 0; j <= KH; ++j) {
    dh[2 * j] = lof(A[j]) + hif(Bq[j]);
    dh[2 * j + 1] = hif(A[j]) - lof(Bq[j]);
  }
#pragma unroll
  for (int k = 0; k < R; ++k) g[k] = ng[k];
}

template <int KH, int R, int NW, bool FAST, bool NORM>
__device__ __forceinline__ void rev2_body(const RevArgs& a, f2x* ubuf, f2x* fresh, const TapP* taps_adj,
                                          const StepNorm* norm, float* red, float* lred, const float* gam,
                                          int64_t e0, int64_t fast_off, uint32_t own) {
  constexpr int NT = NW * 32;
  constexpr int NTU = KH + 1;
  constexpr int V = 1 + 2 * NTU;
  constexpr int RS = R + 2;  // padded slot stride of the window copies (conflict-free LDS.128)
  constexpr int SW = rev2_sw(KH, R);
  constexpr uint32_t FULL = (1u << R) - 1u;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s0 = a.s0, s1 = a.s1;
  const bool full = own == FULL || own == 0;
  const bool none = own == 0;

  async_window<true, R, NT>(rev_src(a, s1 - 1), e0, a.g, ubuf + (size_t)((s1 - 1) & 1) * NT * RS, fast_off);
  f2x v[R], g[R];
  load_window<R>(rev_src(a, s1), e0, a.g, v);
  const float2 Pend = norm[a.M - 1].P;
  const TapP conjP = tap_adj(Pend);
  if (a.gin == nullptr) {
    f2x t[R];
    load_window<R>(a.target, e0, a.g, t);
    float lsum = 0.f;
    const f2x m1 = bcast(-1.f);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const f2x y = NORM ? cscale(Pend, v[k]) : v[k];
      const f2x e = fma2(m1, t[k], y);
      const f2x ge = mul2(bcast(a.seed_scale), e);
      g[k] = NORM ? tmul(conjP, ge) : ge;
      const float ex = lof(e), ey = hif(e);
      if (own & (1u << k)) lsum = fmaf(ex, ex, fmaf(ey, ey, lsum));
    }
    lsum = warp_sum(lsum);
    if (lane == 0) lred[warp] = lsum;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < NW; ++w) tot += (double)lred[w];
      a.loss_partials[blockIdx.x] = tot;
    }
  } else {
    load_window<R>(a.gin, e0, a.g, g);
    if (NORM && s1 == a.M) {
#pragma unroll
      for (int k = 0; k < R; ++k) g[k] = tmul(conjP, g[k]);
    }
  }
  float dgam = 0.f;
  {
    const float gm = gam[s1 - 1 - s0];
    if (full) {
#pragma unroll
      for (int k = 0; k < R; ++k) nl_adjoint<FAST, false>(g[k], v[k], gm, 2.f * gm, true, dgam);
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) nl_adjoint<FAST, true>(g[k], v[k], gm, 2.f * gm, (own >> k) & 1u, dgam);
    }
    if (none) dgam = 0.f;
  }

  constexpr int VP = V <= 2 ? 2 : V <= 4 ? 4 : V <= 8 ? 8 : V <= 16 ? 16 : 32;
  int nref = 0;
  for (int l = s1 - 1; l >= s0; --l) {
    const int li = l - s0;
    const int done = s1 - 1 - l;  // reverse steps completed in this launch
    if (KH > 0 && done > 0 && done % SW == 0) {
      // refresh the duplicate lanes from the owning warps (their lanes 1 / 30 are exact)
      f2x* fb = fresh + (size_t)(nref & 1) * NW * 2 * R;
      if (lane == 1 || lane == 30) {
        f2x* dst = fb + ((size_t)warp * 2 + (lane == 30 ? 1 : 0)) * R;
#pragma unroll
        for (int k = 0; k < R; ++k) dst[k] = g[k];
      }
      __syncthreads();
      if (lane == 0 && warp > 0) {
        const f2x* src = fb + ((size_t)(warp - 1) * 2 + 1) * R;
#pragma unroll
        for (int k = 0; k < R; ++k) g[k] = src[k];
      }
      if (lane == 31 && warp < NW - 1) {
        const f2x* src = fb + ((size_t)(warp + 1) * 2 + 0) * R;
#pragma unroll
        for (int k = 0; k < R; ++k) g[k] = src[k];
      }
      ++nref;
    }
    cp_async_wait_all();
    __syncwarp();
    if (l - 1 >= s0)
      async_window<true, R, NT>(rev_src(a, l - 1), e0, a.g, ubuf + (size_t)((l - 1) & 1) * NT * RS, fast_off);
    const f2x* ub = ubuf + (size_t)(l & 1) * NT * RS + (size_t)tid * RS;
    const TapP* hs_sm = taps_adj + li * NTU;
    const float gmn = l > s0 ? gam[li - 1] : 0.f;
    float dh[2 * NTU];
    float dgam_next = 0.f;
    if (l > s0) {
      if (full)
        rev2_step<KH, R, FAST, NORM, false, true>(g, ub, hs_sm, own, gmn, dh, dgam_next);
      else
        rev2_step<KH, R, FAST, NORM, true, true>(g, ub, hs_sm, own, gmn, dh, dgam_next);
    } else {
      if (full)
        rev2_step<KH, R, FAST, NORM, false, false>(g, ub, hs_sm, own, gmn, dh, dgam_next);
      else
        rev2_step<KH, R, FAST, NORM, true, false>(g, ub, hs_sm, own, gmn, dh, dgam_next);
    }
    {
      float vals[VP];
      vals[0] = none ? 0.f : dgam;
#pragma unroll
      for (int i = 0; i < 2 * NTU; ++i) vals[1 + i] = none ? 0.f : dh[i];
#pragma unroll
      for (int i = V; i < VP; ++i) vals[i] = 0.f;
      const float r = warp_reduce_scatter<VP>(vals, lane);
      constexpr int SH = VP == 2 ? 4 : VP == 4 ? 3 : VP == 8 ? 2 : VP == 16 ? 1 : 0;
      const int idx = lane >> SH;
      float* rp = red + ((size_t)li * NW + warp) * V;
      if ((lane & ((1 << SH) - 1)) == 0 && idx < V) rp[idx] = r;
    }
    dgam = dgam_next;
  }
  if (a.gout && lane != 0 && lane != 31) store_owned<R>(a.gout, e0, a.g, g);  // duplicates excluded
  __syncthreads();
  // CTA reduction in fp64, fixed order over warps, mapped back to the original parameters
  constexpr int npairs = 1 + NTU;
  const int S = s1 - s0;
  for (int i = tid; i < S * npairs; i += NT) {
    const int li = i / npairs, q = i % npairs;
    const int l = s0 + li;
    double* out = a.partials + ((int64_t)blockIdx.x * a.M + l) * V;
    const StepNorm nm = norm[l];
    const float* rp = red + (size_t)li * NW * V;
    if (q == 0) {
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) acc += (double)rp[w * V];
      if (NORM) acc *= (double)nm.P.x * nm.P.x + (double)nm.P.y * nm.P.y;
      out[0] = acc;
    } else {
      const int v2 = 1 + 2 * (q - 1);
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        re += (double)rp[w * V + v2];
        im += (double)rp[w * V + v2 + 1];
      }
      if (NORM) {
        const double cx = nm.c.x, cy = nm.c.y, m = cx * cx + cy * cy;
        const double r2 = (re * cx - im * cy) / m, i2 = (re * cy + im * cx) / m;
        re = r2;
        im = i2;
      }
      out[v2] = re;
      out[v2 + 1] = im;
    }
  }
}

// Shared-memory bytes (mirrors the carve-up below).
__host__ __device__ constexpr size_t rev2_smem_bytes(int kh, int steps, int M) {
  const int NW = rev2_warps(kh), NT = NW * 32, R = rev2_r(kh), NTU = kh + 1, V = 1 + 2 * NTU;
  return sizeof(unsigned long long) * 2 * (size_t)NT * (R + 2)      // window copies
         + sizeof(unsigned long long) * 2 * (size_t)NW * 2 * R      // refresh slots
         + 16 * (size_t)steps * NTU                                 // adjoint taps (TapP)
         + 16 * (size_t)M                                           // StepNorm
         + 4 * (size_t)((steps * NW * V + 3) & ~3)                  // per-warp partials
         + 4 * (size_t)((NW + 3) & ~3)                              // loss partials
         + 4 * (size_t)((steps + 3) & ~3) + 16                      // gamma_hat + flag
         + 4 * (size_t)steps;                                       // kj (unused)
}

template <int KH, bool FAST>
__global__ void __launch_bounds__(rev2_warps(KH) * 32, 65536 / (rev2_warps(KH) * 32 * rev2_regs(KH)))
    rev2_tile_kernel(const RevArgs a) {
  constexpr int NW = rev2_warps(KH), NT = NW * 32, R = rev2_r(KH), NTU = KH + 1, V = 1 + 2 * NTU;
  static_assert(sizeof(TapP) == 16 && sizeof(StepNorm) == 16, "smem carve-up sizes");
  static_assert(R % 2 == 0 && R >= KH && R < 32, "slot width");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int S = a.s1 - a.s0;
  f2x* ubuf = reinterpret_cast<f2x*>(smem_raw);                          // [2][NT][R+2]
  f2x* fresh = ubuf + (size_t)2 * NT * (R + 2);                          // [2][NW][2][R]
  TapP* taps_adj = reinterpret_cast<TapP*>(fresh + (size_t)2 * NW * 2 * R);  // [S][NTU]
  StepNorm* norm = reinterpret_cast<StepNorm*>(taps_adj + S * NTU);      // [M]
  float* red = reinterpret_cast<float*>(norm + a.M);                     // [S][NW][V]
  float* lred = red + ((S * NW * V + 3) & ~3);                           // [NW]
  float* gam = lred + ((NW + 3) & ~3);                                   // [S]
  int* flag = reinterpret_cast<int*>(gam + ((S + 3) & ~3));               // [4]
  int* kj = flag + 4;                                                    // [S]

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = 30 * warp + lane;
  const int64_t e0 = tile_lo(a.g, blockIdx.x) - a.g.H + (int64_t)slot * R;
  const Span sp = make_span(e0, a.g);
  const int64_t fast_off = span_fast<R>(sp, a.g, e0) ? sp.b0 * a.g.n + (sp.q0 - a.g.H) : -1;
  const uint32_t own = (lane == 0 || lane == 31) ? 0u : owned_mask<R>(e0, a.g);
  load_ptab<NTU>(a.ptab, a.M, a.s0, a.s1, norm, nullptr, taps_adj, gam, kj, flag);
  __syncthreads();
  if (*flag)
    rev2_body<KH, R, NW, FAST, true>(a, ubuf, fresh, taps_adj, norm, red, lred, gam, e0, fast_off, own);
  else
    rev2_body<KH, R, NW, FAST, false>(a, ubuf, fresh, taps_adj, norm, red, lred, gam, e0, fast_off, own);
}

}  // namespace ldbp

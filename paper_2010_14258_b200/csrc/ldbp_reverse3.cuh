// ldbp_reverse3.cuh — skewed, one-sided-dependency store-all reverse kernel (SURVEY.md §8(a) rows
// a5, a6, a8; the arithmetic of rev_tile_kernel, ldbp_reverse.cuh, with a different dependency
// structure).
//
// rev_tile_kernel keeps every thread's output window equal to its input window, so each reverse
// step needs Kh adjoint samples from BOTH neighbours and all warps of a CTA advance in lockstep
// behind a per-step barrier (measured: the barrier wait holds ~15 % of the stall samples, and
// shaving 12 % of the instructions moved the time by 2 %: the lockstep makes the kernel latency-
// bound).  Here the output window of a step is the input window shifted LEFT by Kh samples:
//   slot p (thread 32 w + lane) holds the adjoint ga^(l) on extended positions
//   [E_k + p R, E_k + p R + R),  E_k = E_0 - k Kh  after k reverse steps of the launch,
// so the FIR adjoint outputs g_s (s in the new window) need inputs [s - Kh, s + Kh] = this slot's R
// inputs and the LAST 2 Kh inputs of slot p - 1 only.  Dependencies point one way:
//   * inside a warp: lane - 1 by one shuffle-up of 2 Kh samples per step;
//   * across warps: lane 31 of warp w - 1 hands its last 2 Kh samples of each step to lane 0 of
//     warp w through a D-deep ring in shared memory with full / empty mbarriers,
// and no warp ever waits for a warp to its right: warps pipeline instead of marching in lockstep
// (warp w may run up to D steps behind warp w - 1; warp 0 never waits).
// The dependency cone is unchanged (garbage enters only at the left window edge and moves 2 Kh
// per step in window coordinates = Kh per step in absolute positions from either side), so the
// CTA's owned range is [E_0 + S Kh, E_0 + NT R - S Kh) as in every tile kernel (H = S Kh); the
// owned part of a slot changes from step to step at the two range ends, so ownership is a per-step
// bit mask applied by predication (no divergent code paths).
// Per reverse step l (chain rule on Eq. (7)): outputs s of the shifted window
//   P_sj = ga_{s-j} + ga_{s+j},  g_s = ga_s + sum_j conj(h_j) P_sj (SYM, h0-normalised),
//   dh_j += conj(u^(l)_s) P_sj (owned s), then the NL adjoint of step l-1 on g_s (v = u^(l)_s).
#pragma once

namespace ldbp {

#ifndef LDBP_REV3_NW
#define LDBP_REV3_NW 4  // warps per CTA
#endif
#ifndef LDBP_REV3_TAILSMEM
#define LDBP_REV3_TAILSMEM 0  // 1: the left halo passes through shared memory (frees 16 registers
                              // that would hold the shuffled halo across the step)
#endif
#ifndef LDBP_REV3_D
#define LDBP_REV3_D 4  // depth of the cross-warp ring (steps warp w-1 may run ahead of warp w)
#endif
__host__ __device__ constexpr int rev3_warps(int) { return LDBP_REV3_NW; }
__host__ __device__ constexpr int rev3_r(int) { return LDBP_REV_R; }
#ifdef LDBP_REV3_REGS
__host__ __device__ constexpr int rev3_regs(int) { return LDBP_REV3_REGS; }
#else
__host__ __device__ constexpr int rev3_regs(int kh) { return kh <= 1 ? 96 : 128; }
#endif

// One output s (compile-time) of the shifted window: inputs g[s - Kh + i], i in [-Kh, Kh],
// index < 0 from gl (2 Kh left-neighbour samples, gl[2Kh + idx]).
#define LDBP_WIN3(g, gl, i) ((i) < 0 ? gl[2 * KH + (i)] : g[(i)])

// Outputs s = S1-1 down to S0 (compile-time) of the shifted window, IN PLACE: output s needs the
// inputs g[s - 2Kh .. s] only (index < 0: the left halo gl[2Kh + idx]), so in decreasing order
// every input an output needs is still the old value when it is read, and g[s] can take the new
// value at once — no second register array and no copy at the end of the step.
template <int KH, int R, bool FAST, bool NORM, bool NL, int S0, int S1>
__device__ __forceinline__ void rev3_range(f2x (&g)[R], const f2x (&gl)[2 * KH], const f2x* __restrict__ ub,
                                           const TapP (&hs)[KH + 1], f2x (&A)[KH + 1], f2x (&Bq)[KH + 1],
                                           uint32_t own, float gmn, float& dgam_next) {
  if constexpr (S1 > S0) {
    constexpr int s = S1 - 1;
    constexpr int c = s - KH;  // centre input index of output s
    const f2x us = ub[s];
    const bool mine = (own >> s) & 1u;
    // ownership by zeroing u in the tap-gradient products (2 selects per sample) instead of
    // predicated packed FMAs: ptxas turns a predicated FFMA2 into a temp + 2 conditional moves
    // (measured: 25 % of the instructions were such moves)
    const f2x ux = bcast(mine ? lof(us) : 0.f), uy = bcast(mine ? hif(us) : 0.f);
    const f2x g0 = LDBP_WIN3(g, gl, c);
    f2x acc = NORM ? g0 : tmul(hs[0], g0);
    A[0] = fma2(ux, g0, A[0]);
    Bq[0] = fma2(uy, g0, Bq[0]);
#pragma unroll
    for (int j = 1; j <= KH; ++j) {
      const f2x P = add2(LDBP_WIN3(g, gl, c - j), LDBP_WIN3(g, gl, c + j));
      acc = tmac(acc, hs[j], P);
      A[j] = fma2(ux, P, A[j]);
      Bq[j] = fma2(uy, P, Bq[j]);
    }
    if constexpr (NL) nl_adjoint<FAST, true>(acc, us, gmn, 2.f * gmn, mine, dgam_next);
    g[s] = acc;
    rev3_range<KH, R, FAST, NORM, NL, S0, S1 - 1>(g, gl, ub, hs, A, Bq, own, gmn, dgam_next);
  }
}

// Position of a slot's first output in the extended index space, tracked incrementally from step
// to step (no 64-bit division in the loop): e = b ext + q, q in [0, ext).
struct Pos3 {
  int rel;  // e - lo (lo = first owned position of the CTA)
  int b, q; // block and extended position within it: e = b ext + q, q in [0, ext)
};
__device__ __forceinline__ Pos3 pos3_make(int64_t e, int64_t lo, const Geo& g) {
  const int64_t b = e >= 0 ? e / g.ext : -((-e + g.ext - 1) / g.ext);  // floor
  return {(int)(e - lo), (int)b, (int)(e - b * g.ext)};
}
__device__ __forceinline__ void pos3_left(Pos3& p, int d, const Geo& g) {  // e -= d, |d| < ext
  p.rel -= d;
  p.q -= d;
  if (p.q < 0) {
    p.q += (int)g.ext;
    --p.b;
  } else if (p.q >= g.ext) {
    p.q -= (int)g.ext;
    ++p.b;
  }
}
// True when the R samples are consecutive real samples of one block (contiguous addressing).
template <int R>
__device__ __forceinline__ bool pos3_fast(const Pos3& p, const Geo& g) {
  return p.b >= 0 && p.b < g.B && p.q >= g.H && p.q + R <= g.H + g.n;
}
// Ownership bits of the R samples at p: inside the CTA's owned range [0, W) (relative) and real.
template <int R>
__device__ __forceinline__ uint32_t rev3_own(const Pos3& p, int W, const Geo& g) {
  constexpr uint32_t FULL = (1u << R) - 1u;
  if (p.rel + R <= 0 || p.rel >= W) return 0u;
  uint32_t m = FULL;
  if (p.rel < 0) m &= FULL << (-p.rel);
  if (p.rel + R > W) m &= FULL >> (p.rel + R - W);
  if (pos3_fast<R>(p, g)) return m;
  uint32_t r = 0;
  int b = p.b, q = p.q;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (b >= 0 && b < g.B && q >= g.H && q < g.H + g.n) r |= 1u << k;
    if (++q == g.ext) {
      q = 0;
      ++b;
    }
  }
  return m & r;
}

// Steps k (within [0, S)) for which `len` samples starting at p0 - k Kh are consecutive real
// samples of one block (the window moves left by Kh per step; S Kh <= H keeps it in one block).
struct KRange {
  int ka, kb;
};
template <int KH>
__device__ __forceinline__ KRange fast_steps(const Pos3& p0, int len, const Geo& g, int S) {
  if (p0.b < 0 || p0.b >= g.B || p0.q < g.H) return {1, 0};
  const int kb = min((p0.q - (int)g.H) / KH, S - 1);  // q - k Kh >= H
  const int over = p0.q + len - (int)g.H - (int)g.n;  // need q - k Kh + len <= H + n
  const int ka = over > 0 ? (over + KH - 1) / KH : 0;
  return {ka, kb};
}
// Bits of the R samples at rel (relative to the owned range [0, W)) inside the range.
template <int R>
__device__ __forceinline__ uint32_t range_mask(int rel, int W) {
  constexpr uint32_t FULL = (1u << R) - 1u;
  if (rel + R <= 0 || rel >= W) return 0u;
  uint32_t m = FULL;
  if (rel < 0) m &= FULL << (-rel);
  if (rel + R > W) m &= FULL >> (rel + R - W);
  return m;
}

template <int KH, int R, int NW, bool FAST, bool NORM>
__device__ __forceinline__ void rev3_body(const RevArgs& a, f2x* ubuf, f2x* ring, f2x* tailb, uint64_t* bars,
                                          const TapP* taps_adj, const StepNorm* norm, float* red, float* lred,
                                          const float* gam) {
  constexpr int NT = NW * 32;
  constexpr int NTU = KH + 1;
  constexpr int V = 1 + 2 * NTU;
  constexpr int RS = R + 2;
  constexpr int D = LDBP_REV3_D;
  constexpr int KE2 = 2 * KH;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int s0 = a.s0, s1 = a.s1;
  const int64_t lo = tile_lo(a.g, blockIdx.x);
  const int W = (int)(min(lo + a.g.W, a.g.E) - lo);  // owned width
  const int64_t E0 = lo - a.g.H;              // window start at k = 0
  const int64_t ep = E0 + (int64_t)tid * R;   // this slot's first input position at k = 0
  uint64_t* full = bars;                      // [NW][D]
  uint64_t* empty = bars + NW * D;            // [NW][D]
  f2x* myring = ring + (size_t)warp * D * KE2;          // consumed by this warp (lane 0)
  f2x* nxring = ring + (size_t)(warp + 1) * D * KE2;    // produced by this warp (lane 31) for warp + 1
  Pos3 po = pos3_make(ep - KH, lo, a.g);      // first OUTPUT position of step k (k = 0 now)

  const int S = s1 - s0;
  // loop-invariant copy / ownership bookkeeping (the windows move left by Kh per step):
  // the warp's 32 R samples are on the contiguous fast path for steps [wf.ka, wf.kb] (uniform),
  // this slot's R samples are all real samples for steps [sf.ka, sf.kb]
  const Pos3 pw0 = {__shfl_sync(kFull, po.rel, 0), __shfl_sync(kFull, po.b, 0), __shfl_sync(kFull, po.q, 0)};
  const KRange wf = fast_steps<KH>(pw0, 32 * R, a.g, S);
  const KRange sf = fast_steps<KH>(po, R, a.g, S);
  const int64_t woff0 = (int64_t)pw0.b * a.g.n + (pw0.q - a.g.H);  // lane 0's element offset at k = 0
  CoalCopy<R, NT> cc = coal_setup<R, NT>(ubuf, 0);
  // window copy of u^(i) at the output positions of step k (first output of this slot at p)
  auto window = [&](int i, int k, const Pos3& p, int buf) {
    const float2* src = rev_src(a, i);
    if (k >= wf.ka && k <= wf.kb && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      const char* base = reinterpret_cast<const char*>(reinterpret_cast<const f2x*>(src) + woff0 -
                                                       (int64_t)k * KH) + 16 * lane;
      const uint32_t boff = (uint32_t)(buf * NT * RS * 8);
#pragma unroll
      for (int m = 0; m < R / 2; ++m)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(cc.dst[m] + boff), "l"(base + 512 * m)
                     : "memory");
      asm volatile("cp.async.commit_group;" ::: "memory");
    } else {
      const int64_t fo = pos3_fast<R>(p, a.g) ? (int64_t)p.b * a.g.n + (p.q - a.g.H) : -1;
      async_window<true, R, NT>(src, lo + p.rel, a.g, ubuf + (size_t)buf * NT * RS, fo);
    }
  };
  window(s1 - 1, 0, po, (s1 - 1) & 1);
  // state at k = 0: ga^(s1-1) on the input positions [ep, ep + R)
  f2x v[R], g[R];
  load_window<R>(rev_src(a, s1), ep, a.g, v);
  const uint32_t own_in = rev3_own<R>(pos3_make(ep, lo, a.g), W, a.g);  // initial positions (loss)
  const float2 Pend = norm[a.M - 1].P;
  const TapP conjP = tap_adj(Pend);
  if (a.gin == nullptr) {
    f2x t[R];
    load_window<R>(a.target, ep, a.g, t);
    float lsum = 0.f;
    const f2x m1 = bcast(-1.f);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const f2x y = NORM ? cscale(Pend, v[k]) : v[k];
      const f2x e = fma2(m1, t[k], y);
      const f2x ge = mul2(bcast(a.seed_scale), e);
      g[k] = NORM ? tmul(conjP, ge) : ge;
      const float ex = lof(e), ey = hif(e);
      if (own_in & (1u << k)) lsum = fmaf(ex, ex, fmaf(ey, ey, lsum));
    }
    lsum = warp_sum(lsum);
    if (lane == 0) lred[warp] = lsum;
  } else {
    load_window<R>(a.gin, ep, a.g, g);
    if (NORM && s1 == a.M) {
#pragma unroll
      for (int k = 0; k < R; ++k) g[k] = tmul(conjP, g[k]);
    }
  }
  float dgam = 0.f;
  {
    const float gm = gam[s1 - 1 - s0];
#pragma unroll
    for (int k = 0; k < R; ++k) nl_adjoint<FAST, true>(g[k], v[k], gm, 2.f * gm, (own_in >> k) & 1u, dgam);
  }
  // hand this step's last 2 Kh inputs of lane 31 to the next warp (ring slot k % D)
  // warp-uniform control flow (every lane waits / branches alike; only the stores and the single
  // arrival are predicated), so the shuffles of the step stay in converged code
  auto produce = [&](int k) {
    if (warp + 1 < NW) {
      const int j = k % D;
      if (k >= D) mbar_wait_parity(empty + (warp + 1) * D + j, ((k / D) - 1) & 1);
      if (lane == 31) {
#pragma unroll
        for (int i = 0; i < KE2; ++i) nxring[j * KE2 + i] = g[R - KE2 + i];
      }
      __syncwarp();
      if (lane == 31) mbar_arrive(full + (warp + 1) * D + j);
    }
  };
  produce(0);

  constexpr int VP = V <= 2 ? 2 : V <= 4 ? 4 : V <= 8 ? 8 : V <= 16 ? 16 : 32;
  for (int l = s1 - 1; l >= s0; --l) {
    const int li = l - s0;
    const int k = s1 - 1 - l;
    cp_async_wait_all();
    __syncwarp();
    const uint32_t own = (k >= sf.ka && k <= sf.kb) ? range_mask<R>(po.rel, W) : rev3_own<R>(po, W, a.g);
    pos3_left(po, KH, a.g);  // -> first output of step k + 1
    if (l - 1 >= s0) window(l - 1, k + 1, po, (l - 1) & 1);
    const f2x* ub = ubuf + (size_t)(l & 1) * NT * RS + (size_t)tid * RS;
    TapP hs[KH + 1];
    const TapP* hs_sm = taps_adj + li * NTU;
#pragma unroll
    for (int j = 0; j <= KH; ++j) hs[j] = hs_sm[j];
    // left halo first (the neighbour overwrites its tail in place during this step): the last 2 Kh
    // inputs of slot p - 1 by shuffle; lane 0 of warp w > 0 takes them from the ring below
    f2x A[KH + 1], Bq[KH + 1], gl[KE2];
    if (LDBP_REV3_TAILSMEM) {  // publish the old tail now, read the neighbour's when needed
#pragma unroll
      for (int i = 0; i < KE2; ++i) tailb[tid * (KE2 + 2) + i] = g[R - KE2 + i];
      __syncwarp();
    } else {
#pragma unroll
      for (int i = 0; i < KE2; ++i) gl[i] = __shfl_up_sync(kFull, g[R - KE2 + i], 1);
    }
#pragma unroll
    for (int j = 0; j <= KH; ++j) A[j] = Bq[j] = 0ull;
    float dgam_next = 0.f;
    const float gmn = l > s0 ? gam[li - 1] : 0.f;
    // outputs [2 Kh, R) (own inputs only), from the top down.  One code path for every step: on
    // the launch's last step gmn = 0 and the fused NL adjoint is an exact identity (sin 0 = 0,
    // cos 0 = 1; its dgamma' contribution is discarded) — half the loop body (instruction fetch)
    rev3_range<KH, R, FAST, NORM, true, KE2, R>(g, gl, ub, hs, A, Bq, own, gmn, dgam_next);
    if (LDBP_REV3_TAILSMEM) {
      const f2x* tp = tailb + (lane > 0 ? tid - 1 : tid) * (KE2 + 2);
#pragma unroll
      for (int i = 0; i < KE2; ++i) gl[i] = tp[i];
    }
    if (warp > 0) {  // warp-uniform: warp w - 1 finished step k - 1 (its lane 31 tail is in the ring)
      const int j = k % D;
      mbar_wait_parity(full + warp * D + j, (k / D) & 1);
      const bool l0 = lane == 0;
#pragma unroll
      for (int i = 0; i < KE2; ++i) {
        const f2x r = myring[j * KE2 + i];  // broadcast read (all lanes), kept by lane 0 only
        gl[i] = l0 ? r : gl[i];
      }
      __syncwarp();
      if (l0) mbar_arrive(empty + warp * D + j);
    }
    // outputs [0, 2 Kh): need the left halo
    rev3_range<KH, R, FAST, NORM, true, 0, KE2>(g, gl, ub, hs, A, Bq, own, gmn, dgam_next);
    if (LDBP_REV3_TAILSMEM) __syncwarp();  // the neighbour has read this slot's tail (WAR next step)
    if (l > s0) produce(k + 1);
    {
      float vals[VP];
      vals[0] = dgam;
#pragma unroll
      for (int j = 0; j <= KH; ++j) {
        vals[1 + 2 * j] = lof(A[j]) + hif(Bq[j]);
        vals[2 + 2 * j] = hif(A[j]) - lof(Bq[j]);
      }
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
  // adjoint w.r.t. u_hat^(s0) on the final positions (po was advanced once past the last step)
  if (a.gout) {
    pos3_left(po, -KH, a.g);  // back to the last step's outputs
    const uint32_t m = rev3_own<R>(po, W, a.g);
    if (m) {
      f2x* d2 = reinterpret_cast<f2x*>(a.gout);
      int64_t b = po.b, q = po.q;
#pragma unroll
      for (int k2 = 0; k2 < R; ++k2) {
        if (m & (1u << k2)) d2[b * a.g.n + (q - a.g.H)] = g[k2];
        if (++q == a.g.ext) {
          q = 0;
          ++b;
        }
      }
    }
  }
  __syncthreads();
  if (a.gin == nullptr && tid == 0) {
    double tot = 0.0;
    for (int w = 0; w < NW; ++w) tot += (double)lred[w];
    a.loss_partials[blockIdx.x] = tot;
  }
  constexpr int npairs = 1 + NTU;
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

__host__ __device__ constexpr size_t rev3_smem_bytes(int kh, int steps, int M) {
  const int NW = rev3_warps(kh), NT = NW * 32, R = rev3_r(kh), NTU = kh + 1, V = 1 + 2 * NTU;
  const int D = LDBP_REV3_D;
  return 16 * (size_t)2 * NW * D                                        // full / empty mbarriers
         + sizeof(unsigned long long) * 2 * (size_t)NT * (R + 2)        // window copies
         + sizeof(unsigned long long) * (size_t)NW * D * 2 * (kh > 0 ? kh : 1)  // ring (NW slots)
         + (LDBP_REV3_TAILSMEM ? sizeof(unsigned long long) * (size_t)NT * (2 * kh + 2) : 0)  // tails
         + 16 * (size_t)steps * NTU                                     // adjoint taps
         + 16 * (size_t)M                                               // StepNorm
         + 4 * (size_t)((steps * NW * V + 3) & ~3)                      // per-warp partials
         + 4 * (size_t)((NW + 3) & ~3)                                  // loss partials
         + 4 * (size_t)((steps + 3) & ~3) + 16                          // gamma_hat + flag
         + 4 * (size_t)steps;                                           // kj (unused)
}

template <int KH, bool FAST>
__global__ void __launch_bounds__(rev3_warps(KH) * 32, 65536 / (rev3_warps(KH) * 32 * rev3_regs(KH)))
    rev3_tile_kernel(const RevArgs a) {
  constexpr int NW = rev3_warps(KH), NT = NW * 32, R = rev3_r(KH), NTU = KH + 1, V = 1 + 2 * NTU;
  constexpr int D = LDBP_REV3_D;
  static_assert(KH >= 1 && 2 * KH <= R && R % 2 == 0 && R < 32, "skewed window: 2 Kh <= R");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int S = a.s1 - a.s0;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);                          // [2][NW][D] (16 B each)
  f2x* ubuf = reinterpret_cast<f2x*>(smem_raw + 16 * 2 * NW * D);                  // [2][NT][R+2]
  f2x* ring = ubuf + (size_t)2 * NT * (R + 2);                                     // [NW][D][2 Kh]
  f2x* tailb = ring + (size_t)NW * D * 2 * KH;                                     // [NT][2 Kh + 2]
  TapP* taps_adj = reinterpret_cast<TapP*>(tailb + (LDBP_REV3_TAILSMEM ? (size_t)NT * (2 * KH + 2) : 0));
  StepNorm* norm = reinterpret_cast<StepNorm*>(taps_adj + S * NTU);                // [M]
  float* red = reinterpret_cast<float*>(norm + a.M);                               // [S][NW][V]
  float* lred = red + ((S * NW * V + 3) & ~3);                                     // [NW]
  float* gam = lred + ((NW + 3) & ~3);                                             // [S]
  int* flag = reinterpret_cast<int*>(gam + ((S + 3) & ~3));                         // [4]
  int* kj = flag + 4;                                                              // [S]
  if (threadIdx.x < 2 * NW * D) mbar_init(bars + threadIdx.x, 1);  // 8-byte barriers, packed
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  load_ptab<NTU>(a.ptab, a.M, a.s0, a.s1, norm, nullptr, taps_adj, gam, kj, flag);
  __syncthreads();
  if (*flag)
    rev3_body<KH, R, NW, FAST, true>(a, ubuf, ring, tailb, bars, taps_adj, norm, red, lred, gam);
  else
    rev3_body<KH, R, NW, FAST, false>(a, ubuf, ring, tailb, bars, taps_adj, norm, red, lred, gam);
}

}  // namespace ldbp

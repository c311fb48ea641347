// ldbp_reverse.cuh — store-all reverse kernel of the training step (SURVEY.md §8(a) rows a5, a6,
// a8; row a7 by stored activations instead of recompute).
//
// The forward pass of the training step (fwd_tile_kernel in global-normalisation mode, one
// store per step) leaves every activation u_hat^(i), i = 1..M, in HBM (8 B/sample-step; C3:
// 3.4 GB, C5: 54 GB of the 180 GB).  The reverse sweep then needs no forward recompute: one
// launch covers steps [s0, s1) of one tile, exactly like the forward tile kernel, with the
// adjoint g held in registers from step to step and a halo H = (s1 - s0)*Kh that shrinks by Kh
// per reverse step (the adjoint's dependency cone).
//
// Per reverse step l (Appendix A of SURVEY.md, chain rule on Eq. (7)):
//   v = u^(l+1) (registers, loaded the step before), g = dL/dv
//   NL adjoint:  c = Im(g conj v), ga = (g + 2 gamma' c v) e^{-j phi}, dgamma' += c |v|^2
//   tap grads:   dh_j += ga_t conj(u_{t-j} (+ u_{t+j} SYM))   over owned samples only
//   FIR adjoint: g_s = sum_j conj(h_j) ga_{s+j}
// u^(l) arrives by cp.async (LDGSTS) into a double-buffered shared-memory copy of the window,
// issued one step ahead, so the HBM latency overlaps the previous step's arithmetic; each
// thread takes its own R samples and the Kh-sample halos of its neighbours from that copy.  The
// ga halos go through a small double-buffered edge array; one __syncthreads per step.
// Per-step partial sums: transposing warp butterfly (fp32) -> smem -> fp64 across warps in
// fixed order -> partials[cta][step][v] (deterministic), reduced by reduce_partials_kernel.
#pragma once

namespace ldbp {

struct RevArgs {
  const float2* x;         // u^(0) [B][n] (original scale == normalised scale at step 0)
  const float2* act;       // u_hat^(i) at act + (i-1)*act_stride, i = 1..M (normalised state)
  int64_t act_stride;      // elements
  const float2* gin;       // s1 == M: dL/dy in the original scale, or nullptr -> seed from target;
                           // s1 <  M: normalised adjoint w.r.t. u_hat^(s1) (previous launch's gout)
  const float2* target;    // [B][n] (seed mode)
  float2* gout;            // adjoint w.r.t. u_hat^(s0) (original scale when s0 == 0), or nullptr
  const float2* taps;
  const float* gamma;
  const uint8_t* mask;
  double* partials;        // [gridDim.x][M][V]
  double* loss_partials;   // [gridDim.x] (seed mode)
  const void* ptab;        // parameter table (params_kernel), or nullptr -> derive in the prologue
  float seed_scale;        // seed g = seed_scale * (y - target)
  int T, M, s0, s1;
  Geo g;
  int ntiles;              // persistent kernels (rev4): tiles to cover (grid-stride); 0 = gridDim.x
};

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async8_zfill(void* smem_dst, const void* gmem_src, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src),
               "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ const float2* rev_src(const RevArgs& a, int i) {
  return i == 0 ? a.x : a.act + (int64_t)(i - 1) * a.act_stride;
}

#ifndef LDBP_REV_VARK
#define LDBP_REV_VARK 0  // per-step active tap length in the reverse (off: the alternating code
                         // variants cost more in instruction fetch than the skipped taps save)
#endif
#ifndef LDBP_REV_TAPS_SMEM
#define LDBP_REV_TAPS_SMEM 0  // 1: read the packed adjoint taps from shared memory at every use
#endif
template <int N>
__device__ __forceinline__ TapP rev_tap(const TapP (&hs)[N], const TapP* hs_sm, int j) {
  if constexpr (LDBP_REV_TAPS_SMEM) {
    TapP t;  // asm volatile: one LDS.128 (broadcast) per use, not hoisted into registers
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(t.a), "=l"(t.b) : "r"(smem_u32(hs_sm + j)));
    return t;
  } else {
    (void)hs_sm;
    return hs[j];
  }
}
template <int KH, bool SYM, bool NORM, bool FAST>
__device__ __forceinline__ constexpr bool rev_vark() { return LDBP_REV_VARK && SYM && NORM && FAST && KH >= 1; }
#ifndef LDBP_REV_DEFER_RED
#define LDBP_REV_DEFER_RED 0
#endif
#ifndef LDBP_REV_PIPE
#define LDBP_REV_PIPE 2  // window-copy buffers of the reverse: 2 = prefetch one step ahead, 3 = two
#endif
#ifndef LDBP_REV_UNROLL2
#define LDBP_REV_UNROLL2 0  // 1: two reverse steps per loop iteration (register renaming instead of moves)
#endif
#ifndef LDBP_REV_ONE_BODY
#define LDBP_REV_ONE_BODY 1  // 1 (Kh >= 2): the last step of a launch (l == s0, no NL adjoint to fuse) runs
                             // the same step code with gamma' = 0 (the NL adjoint is then the identity, bit
                             // for bit on finite data) instead of its own no-NL instantiation, which ptxas
                             // compiled to 1664 instructions against 750 for the hot step and which every
                             // warp walked once per CTA: C3 reverse 1.955 -> 1.93 ms.  Kh <= 1 keeps the
                             // no-NL step (the NL adjoint is most of a Kh = 1 step: C5 +0.9 % with it)
#endif
#ifndef LDBP_REV_WIN_LEAN
#define LDBP_REV_WIN_LEAN 1  // bulk window copies with every per-launch invariant (alignment, shared-memory
                             // addresses, barrier parity from the step index) hoisted out of the step loop:
                             // 1 = for Kh <= 1, 2 = always, 0 = never.  Measured (B200): C5 reverse (Kh = 1)
                             // 14.68 -> 14.39 ms (-2.0 %, three A/B pairs); C3 (Kh = 4) +1.5 % (registers)
#endif
#ifndef LDBP_NB_WAIT
#define LDBP_NB_WAIT 0  // split step barrier: 1 = wait only for the neighbouring warps, 0 = CTA-wide phase
#endif
// Threads per reverse CTA, compile time (every smem offset is an immediate).  Small CTAs (4 warps,
// 4 CTAs/SM at 128 registers) keep the per-step barrier among few warps (measured on C3: 128
// threads 2.05 ms, 256: 2.20, 96: 2.23).  Kh <= 1: 64-thread CTAs were faster with per-thread window
// copies (C5 18.7 vs 19.3 ms); with the coalesced copies 128 is (C5 reverse 17.6 -> 15.2 ms; 256: 15.4).
#ifdef LDBP_REV_NTHR
__host__ __device__ constexpr int rev_threads(int) { return LDBP_REV_NTHR; }
#else
__host__ __device__ constexpr int rev_threads(int) { return 128; }
#endif

#ifndef LDBP_REV_BULK
#define LDBP_REV_BULK 1  // window copies of whole warps by one bulk-async (TMA engine) copy each:
                         // linear layout, sample k of thread t at t*R + k (see rev_body)
#endif
#ifndef LDBP_REV_COALESCED
#define LDBP_REV_COALESCED 1  // warp-cooperative coalesced window copies into a padded thread-major
                              // layout: 1 = for Kh <= 1 (C5 reverse -6 %; C3 (Kh = 4) +1 %, measured),
                              // 2 = always, 0 = never
#endif
__host__ __device__ constexpr bool rev_coal(int kh) {
  return !LDBP_REV_BULK && (LDBP_REV_COALESCED == 2 || (LDBP_REV_COALESCED == 1 && kh <= 1));
}
// Shared-memory window copy of u^(l).  LDBP_REV_COALESCED: sample k of thread t at f2x index
// t*(R+2) + k (one pad pair per thread: a thread's own 16-byte LDS.128 reads, 8 lanes apart by
// (R+2)*8 bytes, hit distinct banks for R = 12); the copies are issued warp-cooperatively, lane L
// moving 16-byte chunk m*32+L of the warp's contiguous 32*R-sample run, so every LDGSTS is a
// coalesced 512-byte read (the per-thread copies read 16 bytes per lane at an R*8-byte stride:
// 32 sectors and 32 shared-memory wavefronts per instruction).  Otherwise: ((k >> 1)*NT + t)*2 +
// (k & 1) with per-thread copies.
template <bool COAL, int R>
__host__ __device__ constexpr int rev_rs() { return COAL ? R + 2 : R; }
template <bool COAL, int R, int NT>
__device__ __forceinline__ constexpr int ubuf_idx(int k, int t) {
  return COAL ? t * (R + 2) + k : (LDBP_REV_BULK ? t * R + k : ((k >> 1) * NT + t) * 2 + (k & 1));
}
template <bool COAL, int R, int NT>
__device__ __forceinline__ constexpr int ubuf_off(int k) {  // offset of sample k from the thread's slot 0
  return COAL ? k : (LDBP_REV_BULK ? k : (k >> 1) * 2 * NT + (k & 1));
}

// Issue the asynchronous copy of this thread's R window samples of `src` (zeros outside [0, E)).
// With COAL a lane may copy other lanes' samples of its warp: consumers order the copies with
// cp.async.wait_all + __syncwarp.
template <bool COAL, int R, int NT>
__device__ __forceinline__ void async_window(const float2* __restrict__ src, int64_t e0, const Geo& g, f2x* buf,
                                             int64_t fast_off) {
  const int t = threadIdx.x;
  f2x* mine = buf + ubuf_idx<COAL, R, NT>(0, t);
  const f2x* src2 = reinterpret_cast<const f2x*>(src);
  const f2x* p = src2 + fast_off;
  const bool fast = fast_off >= 0 && (reinterpret_cast<uintptr_t>(p) & 15) == 0;
  if constexpr (COAL) {
    static_assert(NT % 32 == 0, "warp-cooperative copies need whole warps");
    const int lane = t & 31;
    const int64_t off0 = __shfl_sync(kFull, fast_off, 0);
    if (__all_sync(kFull, fast && fast_off == off0 + (int64_t)lane * R)) {
      const f2x* base = src2 + off0;
      f2x* wbuf = buf + ubuf_idx<COAL, R, NT>(0, t & ~31);
#pragma unroll
      for (int m = 0; m < R / 2; ++m) {
        const int c = m * 32 + lane, tt = c / (R / 2), k2 = c - tt * (R / 2);
        cp_async16(wbuf + tt * (R + 2) + 2 * k2, base + 2 * c);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      return;
    }
  }
  if (fast) {
#pragma unroll
    for (int m = 0; m < R / 2; ++m) cp_async16(mine + ubuf_off<COAL, R, NT>(2 * m), p + 2 * m);
  } else {  // irregular or 8-byte aligned runs (rare): per-sample copies with zero fill
    const Span sp = make_span(e0, g);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      int64_t b, pos;
      int q;
      const bool ok = span_at<R>(sp, k, g, e0, &b, &pos, &q);
      cp_async8_zfill(mine + ubuf_off<COAL, R, NT>(k), ok ? (const void*)(src + b * g.n + pos) : (const void*)src,
                      ok ? 8 : 0);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

// Loop-invariant part of the warp-cooperative window copy (COAL), computed once per launch: the
// shared-memory address of each of the lane's R/2 16-byte chunks (relative to buffer 0) and whether
// the whole warp takes the coalesced path.  Per step only the source base pointer changes, so a copy
// is R/2 LDGSTS with immediate source offsets (lane*16 + m*512) and one add per chunk — instead of
// re-deriving the chunk -> (thread, sample) mapping (an integer division per chunk) every step
// (measured: the copy was ~89 instructions per thread-step, 15 % of the C5 reverse).
template <int R, int NT>
struct CoalCopy {
  uint32_t dst[R / 2];  // smem byte addresses in window buffer 0
  int64_t off0;         // element offset of the warp's first sample (fast path)
  bool warp_fast;       // every lane of the warp is on the contiguous fast path
};
template <int R, int NT>
__device__ __forceinline__ CoalCopy<R, NT> coal_setup(f2x* buf0, int64_t fast_off) {
  CoalCopy<R, NT> cc;
  const int t = threadIdx.x, lane = t & 31;
  cc.off0 = __shfl_sync(kFull, fast_off, 0);
  cc.warp_fast = __all_sync(kFull, fast_off >= 0 && fast_off == cc.off0 + (int64_t)lane * R);
  f2x* wbuf = buf0 + (t & ~31) * (R + 2);
#pragma unroll
  for (int m = 0; m < R / 2; ++m) {
    const int c = m * 32 + lane, tt = c / (R / 2), k2 = c - tt * (R / 2);
    cc.dst[m] = smem_u32(wbuf + tt * (R + 2) + 2 * k2);
  }
  return cc;
}
// Copy of src's window into buffer `buf` (byte offset `boff` from buffer 0).  Falls back to the
// general per-thread path when the warp is not on the fast path or src is not 16-byte aligned.
template <int R, int NT>
__device__ __forceinline__ void async_window_cc(const CoalCopy<R, NT>& cc, const float2* __restrict__ src,
                                                int64_t e0, const Geo& g, f2x* buf, uint32_t boff,
                                                int64_t fast_off) {
  if (cc.warp_fast && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    const char* base = reinterpret_cast<const char*>(reinterpret_cast<const f2x*>(src) + cc.off0) +
                       16 * (threadIdx.x & 31);
#pragma unroll
    for (int m = 0; m < R / 2; ++m)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(cc.dst[m] + boff), "l"(base + 512 * m)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    return;
  }
  async_window<true, R, NT>(src, e0, g, buf, fast_off);
}

struct RevSmem {
  uint64_t* bar;    // split step barrier (count = warps), phases = reverse steps
  TapP* taps_adj;   // [S][NTU]
  StepNorm* norm;   // [M] (global normalisation, step-indexed)
  float* gamma;     // [S] gamma_hat
  int* kj;          // [S] active folded taps per step (outermost unmasked tap; KH without a mask)
  int* flag;
  float* red;       // [S][NW][V] per-warp partials of every step (reduced once at the end)
  float* lred;      // [NW] loss partials
  f2x* edge;        // [2 buf][2 side][KH][NT] ga halos
  f2x* ubuf;        // [2 buf][R/2][NT] 16-byte pairs: window copies of u^(l)
};

// NL adjoint of one sample (g -> ga in place), Appendix A: with v = u^(l+1), g = dL/dv,
//   c = Im(g conj v), t = g + 2 gamma' c v, ga = t e^{-j phi} = (tx c + ty s, ty c - tx s),
//   dgamma' += c |v|^2 (owned samples only).  Scalar rotation: no pair shuffling.
template <bool FAST, bool MASKED>
__device__ __forceinline__ void nl_adjoint(f2x& gk, f2x vk, float gm, float gm2, bool owned, float& dgam) {
  const float vx = lof(vk), vy = hif(vk);
  const float p = fmaf(vx, vx, vy * vy);
  float sn, cs;
  sincos_phase<FAST>(gm * p, &sn, &cs);
  const float cim = fmaf(hif(gk), vx, -lof(gk) * vy);  // Im(g conj v)
  const f2x t = fma2(bcast(gm2 * cim), vk, gk);
  const float tx = lof(t), ty = hif(t);
  gk = pk(fmaf(tx, cs, ty * sn), fmaf(ty, cs, -tx * sn));
  if (!MASKED || owned) dgam = fmaf(cim, p, dgam);
}

// Reverse step arithmetic for outputs s in [SB, SE) (compile-time range), shared pre-add form:
// with ga = ga^(l) (window incl. halos gl/gr) and u_s = u^(l)_s (own samples only),
//   P_sj = ga_{s-j} + ga_{s+j}                      (SYM; GEN uses the single term ga_{s+j})
//   FIR adjoint   g_s  = ga_s + sum_j conj(h_j) P_sj  (NORM: h_0 = 1)
//   tap gradient  dh_j += conj(u_s) P_sj            (= sum_t ga_t conj(u_{t-j} + u_{t+j}),
//                                                     reindexed t -> s; each real sample is owned
//                                                     by exactly one CTA, so the sums agree)
// conj(u) P = ux P - j uy P is accumulated as A_j += ux P, B_j += uy P (broadcast operands only);
// dh_j = A_j - j B_j once per step.  The NL adjoint of step l-1 follows on each fresh g_s (NL).
template <int KH, int R, bool SYM, bool FAST, bool NORM, bool MASKED, bool NL, int SB, int SE, int KJ = KH,
          int S0 = SB>
__device__ __forceinline__ void rev_range(const f2x (&g)[R], const f2x (&gl)[KH > 0 ? KH : 1],
                                          const f2x (&gr)[KH > 0 ? KH : 1], const f2x* __restrict__ ub_mine,
                                          const TapP (&hs)[SYM ? KH + 1 : 2 * KH + 1], const TapP* hs_sm,
                                          f2x (&A)[SYM ? KH + 1 : 2 * KH + 1], f2x (&Bq)[SYM ? KH + 1 : 2 * KH + 1],
                                          f2x (&ng)[R], uint32_t own, float gmn, float& dgam_next) {
  if constexpr (S0 < SE) {
    constexpr int s = S0;
    const f2x us = ub_mine[ubuf_off<rev_coal(KH), R, rev_threads(KH)>(s)];
    const bool mine = !MASKED || ((own >> s) & 1u);
    const f2x ux = bcast(lof(us)), uy = bcast(hif(us));
    f2x acc;
    if constexpr (SYM) {
      const f2x g0 = g[s];
      acc = NORM ? g0 : tmul(rev_tap(hs, hs_sm, 0), g0);
      if (mine) { A[0] = fma2(ux, g0, A[0]); Bq[0] = fma2(uy, g0, Bq[0]); }
#pragma unroll
      for (int j = 1; j <= KJ; ++j) {
        const f2x P = add2(LDBP_WIN(g, gl, gr, s - j), LDBP_WIN(g, gl, gr, s + j));
        acc = tmac(acc, rev_tap(hs, hs_sm, j), P);
        if (mine) { A[j] = fma2(ux, P, A[j]); Bq[j] = fma2(uy, P, Bq[j]); }
      }
    } else {
      acc = 0ull;
#pragma unroll
      for (int jj = 0; jj < 2 * KH + 1; ++jj) {
        const f2x P = LDBP_WIN(g, gl, gr, s + (jj - KH));
        acc = tmac(acc, rev_tap(hs, hs_sm, jj), P);
        if (mine) { A[jj] = fma2(ux, P, A[jj]); Bq[jj] = fma2(uy, P, Bq[jj]); }
      }
    }
    if constexpr (NL) nl_adjoint<FAST, MASKED>(acc, us, gmn, 2.f * gmn, (own >> s) & 1u, dgam_next);
    ng[s] = acc;
    rev_range<KH, R, SYM, FAST, NORM, MASKED, NL, SB, SE, KJ, S0 + 1>(g, gl, gr, ub_mine, hs, hs_sm, A, Bq, ng, own,
                                                                      gmn, dgam_next);
  }
}

// One full reverse step with the split barrier: interior outputs (no halo needed) before the
// wait on the ga-edge mbarrier phase, boundary outputs after it.
struct NoMid {
  __device__ __forceinline__ void operator()() const {}
};
template <int KH, int R, bool SYM, bool FAST, bool NORM, bool MASKED, bool NL, int KJ = KH, class Mid = NoMid>
__device__ __forceinline__ void rev_step(f2x (&g)[R], const f2x* __restrict__ ub_mine, const f2x* left_edge,
                                         const f2x* right_edge, int eoff, uint64_t* bar, unsigned parity,
                                         const TapP* __restrict__ hs_sm, uint32_t own, float gmn,
                                         float (&dh)[2 * (SYM ? KH + 1 : 2 * KH + 1)], float& dgam_next,
                                         const Mid& mid = Mid{}) {
  constexpr int NTU = ntaps_used<SYM, KH>();
  constexpr int NT = rev_threads(KH);
  constexpr int KI = KJ < R - KJ ? KJ : R / 2;  // interior [KI, R-KI)
  TapP hs[NTU];
#pragma unroll
  for (int j = 0; j < NTU; ++j) hs[j] = LDBP_REV_TAPS_SMEM ? TapP{0ull, 0ull} : hs_sm[j];
  f2x A[NTU], Bq[NTU], ng[R];
#pragma unroll
  for (int j = 0; j < NTU; ++j) A[j] = Bq[j] = 0ull;
  f2x gl[KH > 0 ? KH : 1], gr[KH > 0 ? KH : 1];
#pragma unroll
  for (int j = 0; j < (KH > 0 ? KH : 1); ++j) gl[j] = gr[j] = 0ull;
  rev_range<KH, R, SYM, FAST, NORM, MASKED, NL, KI, R - KI, KJ>(g, gl, gr, ub_mine, hs, hs_sm, A, Bq, ng, own, gmn,
                                                                 dgam_next);
  mid();  // LDBP_REV_DEFER_RED: the previous step's warp reduction, inside the barrier window
  if constexpr (KH > 0) {
    if constexpr (LDBP_NB_WAIT) {
      // neighbour-only wait: within the warp the edges are ordered by the publisher's __syncwarp;
      // only lane 0 (needs warp w-1's tail) and lane 31 (needs warp w+1's head) wait
      // bar[2][NW]: phase ph uses bar[ph & 1][w]; each barrier advances every other step, so a
      // neighbour can be at most one phase of that barrier ahead: parity (ph >> 1) & 1 is exact.
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      uint64_t* b = bar + (parity & 1) * (NT / 32);
      const unsigned par2 = (parity >> 1) & 1;
      if (lane == 0 && warp > 0) mbar_wait_parity(b + warp - 1, par2);
      if (lane == 31 && warp < NT / 32 - 1) mbar_wait_parity(b + warp + 1, par2);
      __syncwarp();
    } else {
      mbar_wait_parity(bar, parity);
    }
#pragma unroll
    for (int j = 0; j < KH; ++j) {
      gl[j] = left_edge[eoff + (KH + j) * NT];
      gr[j] = right_edge[eoff + j * NT];
    }
  }
  rev_range<KH, R, SYM, FAST, NORM, MASKED, NL, 0, KI, KJ>(g, gl, gr, ub_mine, hs, hs_sm, A, Bq, ng, own, gmn, dgam_next);
  rev_range<KH, R, SYM, FAST, NORM, MASKED, NL, R - KI, R, KJ>(g, gl, gr, ub_mine, hs, hs_sm, A, Bq, ng, own, gmn,
                                                               dgam_next);
#pragma unroll
  for (int j = 0; j < NTU; ++j) {
    dh[2 * j] = lof(A[j]) + hif(Bq[j]);
    dh[2 * j + 1] = hif(A[j]) - lof(Bq[j]);
  }
#pragma unroll
  for (int k = 0; k < R; ++k) g[k] = ng[k];
}

template <int KH, int R, bool SYM, bool FAST, bool NORM>
__device__ __forceinline__ void rev_body(const RevArgs& a, const RevSmem& sm, int64_t e0, int64_t fast_off,
                                         uint32_t own, int lane, int warp) {
  constexpr int NT = rev_threads(KH), NW = NT / 32;
  constexpr int NTU = ntaps_used<SYM, KH>();
  constexpr int V = 1 + 2 * NTU;
  constexpr int KE = KH > 0 ? KH : 1;
  constexpr uint32_t FULL = R >= 32 ? 0xffffffffu : ((1u << R) - 1u);
  static_assert(R % 2 == 0 && R >= KH && R <= 32, "window pairs and neighbour halos need even Kh <= R <= 32");
  const int tid = threadIdx.x;
  const int left = tid > 0 ? tid - 1 : 0;
  const int right = tid + 1 < NT ? tid + 1 : tid;
  const int s0 = a.s0, s1 = a.s1;
  // With the R-aligned tiling (plan_rev) a thread's samples are all owned (own == FULL) or none
  // (own == 0, halo threads): both run the same unmasked code (no divergence inside a warp) and
  // the latter zero their partials.  Only ragged blocks (n % R != 0) have partial threads.
  const bool full = own == FULL || own == 0;
  const bool none = own == 0;
  uint64_t* bar = sm.bar;

  // prefetch u^(s1-1) (own slots only: no barrier is needed to consume it); LDBP_REV_PIPE = 3:
  // also u^(s1-2) (two steps ahead, three buffers)
  constexpr int PIPE = LDBP_REV_PIPE;
  constexpr bool COAL = rev_coal(KH);
  constexpr int UB = rev_rs<COAL, R>() * NT;  // f2x per window buffer
  CoalCopy<R, NT> cc{};
  if constexpr (COAL) cc = coal_setup<R, NT>(sm.ubuf, fast_off);
  // LDBP_REV_BULK: a warp whose 32 R samples are one contiguous run of real samples (fixed for the
  // launch: the window does not move) copies each step's window with ONE cp.async.bulk (the TMA
  // engine; SASS UBLKCP) issued by lane 0, completion tracked by the transaction count of the
  // warp's mbarrier for that buffer; other warps keep the per-thread copies.
  const int64_t woff = __shfl_sync(kFull, fast_off, 0);
  const bool wbulk = LDBP_REV_BULK && PIPE == 2 &&
                     __all_sync(kFull, fast_off >= 0 && fast_off == woff + (int64_t)lane * R);
  uint64_t* bbar = sm.bar + 2 * NW + 2 * warp;  // [warp][buffer]
  // per-buffer state as register bit masks (bit b = buffer b; indexing small arrays with the
  // runtime buffer number put them in local memory: STL/LDL in the step loop)
  unsigned bused = 0u;  // buffer b was filled by a bulk copy
  unsigned bph = 0u;    // next phase parity of bbar[b]
  // LDBP_REV_WIN_LEAN: a warp whose copies are bulk copies for the whole launch (16-byte aligned for
  // every step: even activation stride) keeps the destination and barrier addresses in registers
  // and takes the barrier parity from the step index (buffer b = i % 2 is used every other step)
  const uint32_t lean_dst = smem_u32(sm.ubuf + ubuf_idx<COAL, R, NT>(0, warp * 32));
  const uint32_t lean_bar = smem_u32(bbar);
  const bool lean_ok = (LDBP_REV_WIN_LEAN == 2 || (LDBP_REV_WIN_LEAN == 1 && KH <= 1)) && wbulk && (a.act_stride & 1) == 0 &&
                       ((reinterpret_cast<uintptr_t>(a.act + woff)) & 15) == 0 &&
                       (s0 > 0 || ((reinterpret_cast<uintptr_t>(a.x + woff)) & 15) == 0);
  auto window = [&](int i, int b) {  // async copy of u^(i) into window buffer b
    const float2* src = rev_src(a, i);
    if (lean_ok) {
      if (lane == 0) {
        constexpr unsigned bytes = 32u * R * 8u;
        const uint32_t bar_b = lean_bar + 8u * b;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of dst
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(bar_b), "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                lean_dst + (uint32_t)(b * UB * 8)),
            "l"(src + woff), "r"(bytes), "r"(bar_b)
            : "memory");
      }
      return;
    }
    if (wbulk && ((reinterpret_cast<uintptr_t>(src + woff)) & 15) == 0) {
      bused |= 1u << b;
      if (lane == 0) {
        f2x* dst = sm.ubuf + (size_t)b * UB + ubuf_idx<COAL, R, NT>(0, warp * 32);
        constexpr unsigned bytes = 32u * R * 8u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic reads of dst
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bbar + b)),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(dst)),
            "l"(src + woff), "r"(bytes), "r"(smem_u32(bbar + b))
            : "memory");
      }
      return;
    }
    bused &= ~(1u << b);
    if constexpr (COAL)
      async_window_cc<R, NT>(cc, src, e0, a.g, sm.ubuf + (size_t)b * UB, (uint32_t)(b * UB * 8), fast_off);
    else
      async_window<COAL, R, NT>(src, e0, a.g, sm.ubuf + (size_t)b * UB, fast_off);
  };
  auto window_wait = [&](int b, int i) {  // buffer b's copy of u^(i) has landed (and the warp may reuse the other)
    if (lean_ok) {
      const unsigned par = ((unsigned)(s1 - 1 - i) >> 1) & 1u;  // uses of buffer b alternate phases
      unsigned ok;
      do {
        asm volatile(
            "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(lean_bar + 8u * b), "r"(par), "r"(LDBP_MBAR_SUSPEND_NS)
            : "memory");
      } while (!ok);
      __syncwarp();
      return;
    }
    if ((bused >> b) & 1u) {
      mbar_wait_parity(bbar + b, (bph >> b) & 1u);
      bph ^= 1u << b;
    } else {
      cp_async_wait_all();
    }
    __syncwarp();
  };
  window(s1 - 1, (s1 - 1) % PIPE);
  if (PIPE == 3 && s1 - 2 >= s0)
    window(s1 - 2, (s1 - 2) % PIPE);
  f2x v[R], g[R];
  load_window<R>(rev_src(a, s1), e0, a.g, v);
  const float2 Pend = sm.norm[a.M - 1].P;
  const TapP conjP = tap_adj(Pend);  // conj(P) * x
  if (a.gin == nullptr) {
    f2x t[R];
    load_window<R>(a.target, e0, a.g, t);
    float lsum = 0.f;
    const f2x m1 = bcast(-1.f);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const f2x y = NORM ? cscale(Pend, v[k]) : v[k];
      const f2x e = fma2(m1, t[k], y);  // y - target
      const f2x ge = mul2(bcast(a.seed_scale), e);
      g[k] = NORM ? tmul(conjP, ge) : ge;
      const float ex = lof(e), ey = hif(e);
      if (own & (1u << k)) lsum = fmaf(ex, ex, fmaf(ey, ey, lsum));
    }
    lsum = warp_sum(lsum);
    if (lane == 0) sm.lred[warp] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < NW; ++w) tot += (double)sm.lred[w];
      a.loss_partials[blockIdx.x] = tot;
    }
  } else {
    load_window<R>(a.gin, e0, a.g, g);
    if (NORM && s1 == a.M) {
#pragma unroll
      for (int k = 0; k < R; ++k) g[k] = tmul(conjP, g[k]);
    }
  }
  // NL adjoint of step s1-1 up front; every later one is fused into the previous step's loop
  float dgam = 0.f;
  {
    const float gm = sm.gamma[s1 - 1 - s0];
    if (full) {
#pragma unroll
      for (int k = 0; k < R; ++k) nl_adjoint<FAST, false>(g[k], v[k], gm, 2.f * gm, true, dgam);
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) nl_adjoint<FAST, true>(g[k], v[k], gm, 2.f * gm, (own >> k) & 1u, dgam);
    }
    if (none) dgam = 0.f;
  }
  f2x* const my_edge = sm.edge + tid;
  const f2x* const left_edge = sm.edge + left;
  const f2x* const right_edge = sm.edge + right;
  auto publish = [&](int ph) {  // ga edges of phase ph into edge buffer ph & 1, then arrive
    if constexpr (KH > 0) {
      const int eo = (ph & 1) * 2 * KE * NT;
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        my_edge[eo + j * NT] = g[j];                   // head
        my_edge[eo + (KH + j) * NT] = g[R - KH + j];   // tail
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(LDBP_NB_WAIT ? bar + (ph & 1) * NW + warp : bar);
    }
  };
  publish(0);

  // per-warp reduction of one step's partials -> red[li][warp][.]
  constexpr int VP = red_vp(V);
  auto reduce_step = [&](float (&vals)[VP], int rli) {
    warp_reduce_write<VP>(vals, lane, sm.red + ((size_t)rli * NW + warp) * V, V);
  };
  // LDBP_REV_DEFER_RED: step l's reduction runs inside step l-1's barrier window (after its
  // interior outputs, before the wait), off the path between publish and the next wait
  float pend[VP];
  int pend_li = -1;
  auto mid = [&]() {
    if (LDBP_REV_DEFER_RED && pend_li >= 0) reduce_step(pend, pend_li);
  };

#if LDBP_REV_UNROLL2
#pragma unroll 2
#endif
  for (int l = s1 - 1; l >= s0; --l) {
    const int li = l - s0;
    const int ph = s1 - 1 - l;  // barrier phase of this step
    if (PIPE == 3 && l > s0) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");  // u^(l) landed, u^(l-1) may be in flight
      if (COAL) __syncwarp();
    } else {
      window_wait(l % PIPE, l);  // u^(l) landed (bulk: mbarrier transaction count; else cp.async)
    }
    // prefetch u^(l-PIPE+1) into a free buffer (this thread's own slots, consumed later)
    if (l - (PIPE - 1) >= s0)
      window(l - (PIPE - 1), (l - (PIPE - 1)) % PIPE);
    const f2x* ub_mine = sm.ubuf + (size_t)(l % PIPE) * UB + ubuf_idx<COAL, R, NT>(0, tid);
    const int eoff = (ph & 1) * 2 * KE * NT;
    float dh[2 * NTU];
    float dgam_next = 0.f;
    const TapP* hs_sm = sm.taps_adj + li * NTU;
    const float gmn = l > s0 ? sm.gamma[li - 1] : 0.f;
    if ((LDBP_REV_ONE_BODY && KH >= 2) || l > s0) {
      if (rev_vark<KH, SYM, NORM, FAST>() && full) {
        // active folded taps of this step: the outermost unmasked tap (masked taps are pruned:
        // zero value and zero gradient; unmasked zero-valued taps still need their gradient)
        if constexpr (rev_vark<KH, SYM, NORM, FAST>())
          dispatch_kj<KH>(sm.kj[li], [&](auto kjc) {
            constexpr int KJ = decltype(kjc)::value;
            rev_step<KH, R, SYM, FAST, NORM, false, true, KJ>(g, ub_mine, left_edge, right_edge, eoff, bar,
                                                              LDBP_NB_WAIT ? ph : (ph & 1), hs_sm, own, gmn, dh,
                                                              dgam_next);
          });
      } else if (full)
        rev_step<KH, R, SYM, FAST, NORM, false, true>(g, ub_mine, left_edge, right_edge, eoff, bar, LDBP_NB_WAIT ? ph : (ph & 1), hs_sm,
                                                      own, gmn, dh, dgam_next, mid);
      else
        rev_step<KH, R, SYM, FAST, NORM, true, true>(g, ub_mine, left_edge, right_edge, eoff, bar, LDBP_NB_WAIT ? ph : (ph & 1), hs_sm,
                                                     own, gmn, dh, dgam_next, mid);
    } else {
      if (full)
        rev_step<KH, R, SYM, FAST, NORM, false, false>(g, ub_mine, left_edge, right_edge, eoff, bar, LDBP_NB_WAIT ? ph : (ph & 1), hs_sm,
                                                       own, gmn, dh, dgam_next, mid);
      else
        rev_step<KH, R, SYM, FAST, NORM, true, false>(g, ub_mine, left_edge, right_edge, eoff, bar, LDBP_NB_WAIT ? ph : (ph & 1), hs_sm,
                                                      own, gmn, dh, dgam_next, mid);
    }
    if (l > s0) publish(ph + 1);
    if (none) {
      dgam_next = 0.f;
#pragma unroll
      for (int i = 0; i < 2 * NTU; ++i) dh[i] = 0.f;
    }
    // ---- per-warp reduction of this step's partials (now, or deferred into the next step) ----
    {
      float vals[VP];
      vals[0] = dgam;
#pragma unroll
      for (int i = 0; i < 2 * NTU; ++i) vals[1 + i] = dh[i];
#pragma unroll
      for (int i = V; i < VP; ++i) vals[i] = 0.f;
      if (LDBP_REV_DEFER_RED) {
#pragma unroll
        for (int i = 0; i < VP; ++i) pend[i] = vals[i];
        pend_li = li;
      } else {
        reduce_step(vals, li);
      }
    }
    dgam = dgam_next;
  }
  if (LDBP_REV_DEFER_RED && pend_li >= 0) reduce_step(pend, pend_li);
  if (a.gout) store_owned<R>(a.gout, e0, a.g, g);
  __syncthreads();
  // CTA reduction in fp64, fixed order over warps, mapped back to the original parameters:
  // dgamma_i = |P_i|^2 dgamma_hat_i, dh^(i) = conj(1/c_i) dh_hat^(i)
  constexpr int npairs = 1 + NTU;
  const int S = s1 - s0;
  for (int i = tid; i < S * npairs; i += NT) {
    const int li = i / npairs, q = i % npairs;
    const int l = s0 + li;
    double* out = a.partials + ((int64_t)blockIdx.x * a.M + l) * V;
    const StepNorm nm = sm.norm[l];
    const float* red = sm.red + (size_t)li * NW * V;
    if (q == 0) {
      double acc = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) acc += (double)red[w * V];
      if (NORM) acc *= (double)nm.P.x * nm.P.x + (double)nm.P.y * nm.P.y;
      out[0] = acc;
    } else {
      const int v2 = 1 + 2 * (q - 1);
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        re += (double)red[w * V + v2];
        im += (double)red[w * V + v2 + 1];
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

// Register budget per thread (occupancy 65536 / (threads * regs) CTAs/SM).  Measured: Kh >= 2
// needs 128 (tighter budgets spill: C3 reverse 2.02 ms at 128 vs 2.30 at 96); Kh <= 1: 96 at 128
// threads (C5 reverse 15.0 vs 15.2 ms at 80).  Taps stay in registers (LDBP_REV_TAPS_SMEM=1 was slower).
#ifdef LDBP_REV_REGS
__host__ __device__ constexpr int rev_regs(int) { return LDBP_REV_REGS; }
#else
__host__ __device__ constexpr int rev_regs(int kh) { return kh <= 1 ? 96 : 128; }
#endif
template <int KH, int R, bool SYM, bool FAST>
__global__ void __launch_bounds__(rev_threads(KH), 65536 / (rev_threads(KH) * rev_regs(KH)))
    rev_tile_kernel(const RevArgs a) {
  constexpr int NTU = ntaps_used<SYM, KH>();
  constexpr int V = 1 + 2 * NTU;
  constexpr int NT = rev_threads(KH), NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int S = a.s1 - a.s0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // carve-up (16-byte aligned regions; mirrored by rev_smem() on the host)
  RevSmem sm;
  sm.bar = reinterpret_cast<uint64_t*>(smem_raw);                                    // 4*NW words
  sm.ubuf = reinterpret_cast<f2x*>(smem_raw) + 4 * NW;                               // PIPE*RS*NT
  sm.edge = sm.ubuf + (size_t)LDBP_REV_PIPE * rev_rs<rev_coal(KH), R>() * NT;                                           // 4*KH*NT
  sm.taps_adj = reinterpret_cast<TapP*>(sm.edge + (size_t)4 * (KH > 0 ? KH : 1) * NT);  // S*NTU
  sm.norm = reinterpret_cast<StepNorm*>(sm.taps_adj + S * NTU);                      // M
  sm.red = reinterpret_cast<float*>(sm.norm + a.M);                                  // S*NW*V
  sm.lred = sm.red + ((S * NW * V + 3) & ~3);                                        // NW
  sm.gamma = sm.lred + ((NW + 3) & ~3);                                              // S
  sm.flag = reinterpret_cast<int*>(sm.gamma + ((S + 3) & ~3));
  sm.kj = sm.flag + 4;                                                               // S

  const int64_t e0 = thread_e0(a.g, R);
  const Span sp = make_span(e0, a.g);
  const int64_t fast_off = span_fast<R>(sp, a.g, e0) ? sp.b0 * a.g.n + (sp.q0 - a.g.H) : -1;
  const uint32_t own = owned_mask<R>(e0, a.g);
  if (LDBP_NB_WAIT ? threadIdx.x < 2 * (NT / 32) : threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(sm.bar + threadIdx.x)),
                 "r"(LDBP_NB_WAIT ? 1 : NT / 32)
                 : "memory");
  }
  if (LDBP_REV_BULK && threadIdx.x < 2 * NW) {  // bulk-copy barriers [warp][buffer]: one arrival + tx bytes
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(sm.bar + 2 * NW + threadIdx.x)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (a.ptab) {
    load_ptab<NTU>(a.ptab, a.M, a.s0, a.s1, sm.norm, nullptr, sm.taps_adj, sm.gamma, sm.kj, sm.flag);
    __syncthreads();
  } else {
  norm_range<KH, SYM>(a.taps, a.mask, a.T, 0, a.M, sm.norm, sm.flag);
  const bool norm0 = SYM && *sm.flag;
  stage_range<KH, SYM, false, true>(a.taps, a.gamma, a.mask, a.T, a.s0, a.s1, 0, nullptr, sm.taps_adj, sm.gamma,
                                    sm.norm, norm0);
  for (int i = threadIdx.x; i < S; i += NT) {
    int kj = KH;
    if (a.mask && SYM) {
      const uint8_t* mrow = a.mask + (int64_t)(a.s0 + i) * a.T + KH;  // centre tap
      kj = 0;
      for (int j = 1; j <= KH; ++j)
        if (mrow[j] || mrow[-j]) kj = j;
    }
    sm.kj[i] = kj;
  }
  __syncthreads();
  }
  const bool norm = SYM && *sm.flag;
  if (norm)
    rev_body<KH, R, SYM, FAST, true>(a, sm, e0, fast_off, own, lane, warp);
  else
    rev_body<KH, R, SYM, FAST, false>(a, sm, e0, fast_off, own, lane, warp);
}

}  // namespace ldbp
#include "ldbp_reverse2.cuh"
#include "ldbp_reverse3.cuh"
#include "ldbp_reverse4.cuh"

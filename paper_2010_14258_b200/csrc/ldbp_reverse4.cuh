// ldbp_reverse4.cuh — store-all reverse kernel with the adjoint in SHARED memory (SURVEY.md
// §8(a) rows a5, a6, a8; the arithmetic of rev_tile_kernel, ldbp_reverse.cuh, with a different
// data placement).
//
// rev_tile_kernel keeps each thread's R adjoint samples in registers across the steps of a launch
// and passes the Kh-sample halos through an edge array behind a split mbarrier.  Its profile
// (profiles/r02_ncu_rev_tile_C3_source.txt, round-2 capture): 943 warp-instructions per
// warp-step for 12 samples, of which ~470 are the arithmetic of the chain rule; the rest is the
// mbarrier wait loop (~65: warps wait ~18 % of their time for a neighbour and the try_wait loop
// re-issues), loop-carried register moves (~25), edge publish/reads, the window-copy bookkeeping,
// local-memory spills, and the per-step warp reduction; at 128 registers only 4 warps per SMSP
// hide latency.
//
// Here the adjoint ga^(l) of the whole CTA window lives in a double-buffered shared-memory array;
// a reverse step is a pure stencil from one buffer into the other with ONE __syncthreads:
//   thread t reads the window [tR - Kh, tR + R + Kh) of ga^(l) (its own row and the Kh samples of
//   rows t-1 / t+1), u^(l) of its own row (bulk-copied, see below), and writes its R outputs
//   ga^(l-1) = NLadj_{l-1}(FIRadj_l(ga^(l))) into the other buffer.
// No register array is carried from step to step (no moves, no edge exchange, no spin loop), so
// the register budget is ~96 and the arithmetic is the same as rev_tile's (SURVEY Appendix A,
// chain rule on Eq. (7)):
//   P_sj = ga_{s-j} + ga_{s+j},  g_s = ga_s + sum_j conj(h_j) P_sj   (SYM; NORM: h_0 = 1)
//   dh_j += conj(u_s) P_sj  (owned s),  then the NL adjoint of step l-1 on g_s with v = u^(l)_s.
// Shared-memory rows of the adjoint buffers are XOR-swizzled at 16-byte granularity so that the
// lanes' own-row and neighbour-row LDS.128/STS.128 are conflict-free (rev4_sw below).
// u^(l) window: one cp.async.bulk (TMA engine) per warp when the warp's 32 rows are one contiguous
// run of real samples (linear layout, completion by mbarrier transaction count), else per-thread
// cp.async with zero fill; LDBP_REV4_PIPE = 1 (one buffer, refilled as soon as the warp has read
// it) or 2 (prefetch one step ahead).
#pragma once

namespace ldbp {

#ifndef LDBP_REV4_R
#define LDBP_REV4_R 12  // samples per thread (one row); R/2 odd or R/2 = 2 mod 4 (see rev4_sw)
#endif
#ifndef LDBP_REV4_NT
#define LDBP_REV4_NT 128
#endif
#ifndef LDBP_REV4_ABL
#define LDBP_REV4_ABL 0  // timing ablations (WRONG results; tuning only): 1 no warp reduction, 2 no NL
                         // adjoint, 4 no step barrier, 8 no u window wait, 16 no tap-gradient sums,
                         // 32 no FIR adjoint (g = ga), 64 no step loop (prologue + epilogue only)
#endif
#ifndef LDBP_REV4_PIPE
#define LDBP_REV4_PIPE 1
#endif
__host__ __device__ constexpr int rev4_r(int) { return LDBP_REV4_R; }
__host__ __device__ constexpr int rev4_threads(int) { return LDBP_REV4_NT; }
#ifdef LDBP_REV4_REGS
__host__ __device__ constexpr int rev4_regs(int) { return LDBP_REV4_REGS; }
#else
__host__ __device__ constexpr int rev4_regs(int) { return 128; }
#endif

// 16-byte chunk swizzle of row t: chunk c is stored at chunk position c ^ rev4_sw(t).  Rows are
// R*8 bytes; a quarter-warp (8 lanes, 8 consecutive rows) touches distinct bank groups when
// R/2 is odd (row stride an odd multiple of 16 bytes) without a swizzle; for R/2 = 2 mod 4 rows
// t and t+4 collide, and flipping bit 0 of the chunk index for rows with bit 2 set separates them.
template <int R>
__device__ __forceinline__ int rev4_sw(int t) {
  static_assert(R % 2 == 0 && ((R / 2) % 2 == 1 || (R / 2) % 4 == 2), "rev4: R/2 must be odd or 2 mod 4");
  if constexpr ((R / 2) % 2 == 1) {
    (void)t;
    return 0;
  } else {
    return (t >> 2) & 1;
  }
}
// Byte addresses (shared window) of the even / odd chunks of row t in a buffer at `base`: chunk c
// is at (c & 1 ? po : pe) + 16 c  (compile-time c, immediate offsets).
struct Rev4Row {
  uint32_t pe, po;
};
template <int R>
__device__ __forceinline__ Rev4Row rev4_row(uint32_t base, int t) {
  const int sw = rev4_sw<R>(t);
  const uint32_t r = base + (uint32_t)(t * R * 8);
  return {r + 16u * sw, r - 16u * sw};
}
__device__ __forceinline__ void lds2(uint32_t addr, f2x& a, f2x& b) {
  asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr));
}
__device__ __forceinline__ void sts2(uint32_t addr, f2x a, f2x b) {
  asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
template <int C>
__device__ __forceinline__ uint32_t rev4_chunk(const Rev4Row& r) {
  return ((C & 1) ? r.po : r.pe) + 16u * C;
}

struct Rev4Smem {
  uint64_t* bbar;   // [NW][2] bulk-copy mbarriers
  f2x* gbuf;        // [2][NT*R] adjoint buffers (swizzled rows)
  f2x* ubuf;        // [PIPE][NT*R] u^(l) windows (linear rows)
  TapP* taps_adj;   // [S][NTU]
  StepNorm* norm;   // [M]
  float* red;       // [S][NW][V]
  float* lred;      // [NW]
  float* gamma;     // [S]
  int* flag;
};

// Left halo: Kh samples of row t-1; chunks C .. R/2-1 hold samples 2C .. R-1, sample R-KH+i -> w[i].
template <int KH, int R, int C>
__device__ __forceinline__ void rev4_load_left(f2x (&w)[R + 2 * KH], const Rev4Row& r) {
  if constexpr (C < R / 2) {
    f2x a, b;
    lds2(rev4_chunk<C>(r), a, b);
    constexpr int i0 = 2 * C - (R - KH), i1 = i0 + 1;
    if constexpr (i0 >= 0) w[i0] = a;
    if constexpr (i1 >= 0) w[i1] = b;
    rev4_load_left<KH, R, C + 1>(w, r);
  }
}

// Window chunks are loaded lazily, just before the first output pair that needs them (w[i] = ga^(l)
// at row position i - KH): output pair C needs w[0 .. 2C + 1 + 2KH].  Loads are ordered behind
// the previous pair's output stores (volatile shared-memory asm), so only ~2Kh + 2 window samples
// are live at a time instead of R + 2Kh.
__host__ __device__ constexpr int rev4_first_pair(int widx, int kh) {  // first pair needing w[widx]
  return widx - 1 - 2 * kh <= 0 ? 0 : (widx - 1 - 2 * kh + 1) / 2;
}
template <int KH, int R, int C, int Q = 0>
__device__ __forceinline__ void rev4_load_pair(f2x (&w)[R + 2 * KH], const Rev4Row& lrow, const Rev4Row& orow,
                                               const Rev4Row& rrow) {
  if constexpr (C == 0 && Q == 0) rev4_load_left<KH, R, (R - KH) / 2>(w, lrow);
  if constexpr (Q < R / 2) {  // own chunk Q: w[KH + 2Q], w[KH + 2Q + 1]
    if constexpr (rev4_first_pair(KH + 2 * Q, KH) == C) lds2(rev4_chunk<Q>(orow), w[KH + 2 * Q], w[KH + 2 * Q + 1]);
    rev4_load_pair<KH, R, C, Q + 1>(w, lrow, orow, rrow);
  } else if constexpr (Q - R / 2 < (KH + 1) / 2) {  // right-halo chunk Q' = Q - R/2: w[KH + R + 2Q']
    constexpr int Qr = Q - R / 2;
    if constexpr (rev4_first_pair(KH + R + 2 * Qr, KH) == C) {
      f2x a, b;
      lds2(rev4_chunk<Qr>(rrow), a, b);
      w[KH + R + 2 * Qr] = a;
      if constexpr (2 * Qr + 1 < KH) w[KH + R + 2 * Qr + 1] = b;
    }
    rev4_load_pair<KH, R, C, Q + 1>(w, lrow, orow, rrow);
  }
}

#ifndef LDBP_REV4_G
#define LDBP_REV4_G 3  // output pairs per group: the group's loads are issued together, its 2G samples
                       // computed as independent chains (ILP), then its outputs stored
#endif
template <int KH, int R, int C, int CE>
__device__ __forceinline__ void rev4_load_group(f2x (&w)[R + 2 * KH], const Rev4Row& lrow, const Rev4Row& orow,
                                                const Rev4Row& rrow) {
  if constexpr (C < CE) {
    rev4_load_pair<KH, R, C>(w, lrow, orow, rrow);
    rev4_load_group<KH, R, C + 1, CE>(w, lrow, orow, rrow);
  }
}

// Outputs of one reverse step for this thread's row (all compile-time indices): u^(l) from the
// thread's linear row at `ub`; outputs (after the NL adjoint of step l-1 when NL) go to the
// swizzled row `wrow` of the other buffer.  Groups of LDBP_REV4_G output pairs.
template <int KH, int R, bool FAST, bool NORM, bool MASKED, bool NL, int C = 0>
__device__ __forceinline__ void rev4_outputs(f2x (&w)[R + 2 * KH], const Rev4Row& lrow, const Rev4Row& orow,
                                             const Rev4Row& rrow, uint32_t ub, const TapP (&hs)[KH + 1],
                                             uint32_t own, float gmn, f2x (&A)[KH + 1], f2x (&Bq)[KH + 1],
                                             float& dgam_next, const Rev4Row& wrow) {
  if constexpr (C < R / 2) {
    constexpr int CE = C + LDBP_REV4_G < R / 2 ? C + LDBP_REV4_G : R / 2;
    constexpr int NS = 2 * (CE - C);
    rev4_load_group<KH, R, C, CE>(w, lrow, orow, rrow);
    f2x uu[NS], o[NS];
#pragma unroll
    for (int c = C; c < CE; ++c) lds2(ub + 16u * c, uu[2 * (c - C)], uu[2 * (c - C) + 1]);
#pragma unroll
    for (int i = 0; i < NS; ++i) {
      const int s = 2 * C + i;
      const f2x us = uu[i];
      const bool mine = !MASKED || ((own >> s) & 1u);
      const f2x ux = bcast(lof(us)), uy = bcast(hif(us));
      const f2x g0 = w[s + KH];
      f2x acc = NORM ? g0 : tmul(hs[0], g0);
      if (mine && !(LDBP_REV4_ABL & 16)) {
        A[0] = fma2(ux, g0, A[0]);
        Bq[0] = fma2(uy, g0, Bq[0]);
      }
#pragma unroll
      for (int j = 1; j <= KH; ++j) {
        const f2x P = add2(w[s + KH - j], w[s + KH + j]);
        if (!(LDBP_REV4_ABL & 32)) acc = tmac(acc, hs[j], P);
        if (mine && !(LDBP_REV4_ABL & 16)) {
          A[j] = fma2(ux, P, A[j]);
          Bq[j] = fma2(uy, P, Bq[j]);
        }
      }
      if constexpr (NL && !(LDBP_REV4_ABL & 2)) nl_adjoint<FAST, MASKED>(acc, us, gmn, 2.f * gmn, (own >> s) & 1u, dgam_next);
      o[i] = acc;
    }
#pragma unroll
    for (int c = C; c < CE; ++c) sts2(((c & 1) ? wrow.po : wrow.pe) + 16u * c, o[2 * (c - C)], o[2 * (c - C) + 1]);
    rev4_outputs<KH, R, FAST, NORM, MASKED, NL, CE>(w, lrow, orow, rrow, ub, hs, own, gmn, A, Bq, dgam_next, wrow);
  }
}

template <int KH, int R, bool FAST, bool NORM>
__device__ __forceinline__ void rev4_body(const RevArgs& a, const Rev4Smem& sm, int64_t e0, int64_t fast_off,
                                          uint32_t own, int lane, int warp, int tile, unsigned& bph) {
  constexpr int NT = rev4_threads(KH), NW = NT / 32;
  constexpr int NTU = KH + 1;
  constexpr int V = 1 + 2 * NTU;
  constexpr int PIPE = LDBP_REV4_PIPE;
  constexpr uint32_t FULL = R >= 32 ? 0xffffffffu : ((1u << R) - 1u);
  constexpr int UB = NT * R;  // f2x per buffer
  static_assert(KH >= 1 && KH <= R, "rev4: 1 <= Kh <= R");
  const int tid = threadIdx.x;
  const int s0 = a.s0, s1 = a.s1;
  const bool full = own == FULL || own == 0;
  const bool none = own == 0;

  // ---- u^(l) window copies (bulk per warp when possible) ----
  const int64_t woff = __shfl_sync(kFull, fast_off, 0);
  const bool wbulk = __all_sync(kFull, fast_off >= 0 && fast_off == woff + (int64_t)lane * R);
  uint64_t* bbar = sm.bbar + 2 * warp;
  unsigned bused = 0u;  // bph: phase parities of the bulk-copy barriers, carried over tiles
  auto window = [&](int i, int b) {
    const float2* src = rev_src(a, i);
    if (wbulk && ((reinterpret_cast<uintptr_t>(src + woff)) & 15) == 0) {
      bused |= 1u << b;
      if (lane == 0) {
        f2x* dst = sm.ubuf + (size_t)b * UB + (size_t)warp * 32 * R;
        constexpr unsigned bytes = 32u * R * 8u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
    async_window<false, R, NT>(src, e0, a.g, sm.ubuf + (size_t)b * UB, fast_off);  // linear t*R + k
  };
  auto window_wait = [&](int b) {
    if ((bused >> b) & 1u) {
      mbar_wait_parity(bbar + b, (bph >> b) & 1u);
      bph ^= 1u << b;
    } else {
      cp_async_wait_all();
    }
    __syncwarp();
  };
  window(s1 - 1, (s1 - 1) % PIPE);

  // ---- adjoint seed / incoming adjoint, NL adjoint of step s1-1 -> buffer 0 ----
  const uint32_t gb0 = smem_u32(sm.gbuf), gb1 = gb0 + (uint32_t)(UB * 8);
  const int left = tid > 0 ? tid - 1 : 0;
  const int right = tid + 1 < NT ? tid + 1 : tid;
  float dgam = 0.f;
  {
    f2x v[R], g[R];
    load_window<R>(rev_src(a, s1), e0, a.g, v);
    const float2 Pend = sm.norm[a.M - 1].P;
    const TapP conjP = tap_adj(Pend);
    if (a.gin == nullptr) {
      load_window<R>(a.target, e0, a.g, g);  // the target, replaced by the seed in place
      float lsum = 0.f;
      const f2x m1 = bcast(-1.f);
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const f2x y = NORM ? cscale(Pend, v[k]) : v[k];
        const f2x e = fma2(m1, g[k], y);
        const f2x ge = mul2(bcast(a.seed_scale), e);
        g[k] = NORM ? tmul(conjP, ge) : ge;
        const float ex = lof(e), ey = hif(e);
        if (own & (1u << k)) lsum = fmaf(ex, ex, fmaf(ey, ey, lsum));
      }
      lsum = warp_sum(lsum);
      if (lane == 0) sm.lred[warp] = lsum;
    } else {
      load_window<R>(a.gin, e0, a.g, g);
      if (NORM && s1 == a.M) {
#pragma unroll
        for (int k = 0; k < R; ++k) g[k] = tmul(conjP, g[k]);
      }
    }
    const float gm = sm.gamma[s1 - 1 - s0];
#pragma unroll
    for (int k = 0; k < R; ++k) nl_adjoint<FAST, true>(g[k], v[k], gm, 2.f * gm, (own >> k) & 1u, dgam);
    if (none) dgam = 0.f;
    const Rev4Row orow = rev4_row<R>(gb0, tid);
#pragma unroll
    for (int c = 0; c < R / 2; ++c) {
      const uint32_t ad = ((c & 1) ? orow.po : orow.pe) + 16u * c;
      sts2(ad, g[2 * c], g[2 * c + 1]);
    }
  }
  __syncthreads();
  if (a.gin == nullptr && threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < NW; ++w) tot += (double)sm.lred[w];
    a.loss_partials[tile] = tot;
  }

  constexpr int VP = red_vp(V);
  constexpr int npairs = 1 + NTU;
  const uint32_t ub_mine0 = smem_u32(sm.ubuf + (size_t)tid * R);
  for (int l = s1 - 1; l >= ((LDBP_REV4_ABL & 64) ? s1 : s0); --l) {
    const int li = l - s0;
    const int ph = s1 - 1 - l;
    const uint32_t rb = (ph & 1) ? gb1 : gb0;  // ga^(l)
    const uint32_t wb = (ph & 1) ? gb0 : gb1;  // ga^(l-1)
    if (!(LDBP_REV4_ABL & 8)) window_wait(l % PIPE);
    if (PIPE == 2 && l - 1 >= s0) window(l - 1, (l - 1) % 2);
    const uint32_t ub = ub_mine0 + (uint32_t)((l % PIPE) * UB * 8);
    TapP hs[NTU];
    const TapP* hsm = sm.taps_adj + li * NTU;
#pragma unroll
    for (int j = 0; j < NTU; ++j) hs[j] = hsm[j];
    const float gmn = l > s0 ? sm.gamma[li - 1] : 0.f;
    f2x w[R + 2 * KH];
    const Rev4Row lrow = rev4_row<R>(rb, left), orow = rev4_row<R>(rb, tid), rrow = rev4_row<R>(rb, right);
    f2x A[NTU], Bq[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) A[j] = Bq[j] = 0ull;
    float dgam_next = 0.f;
    const Rev4Row wrow = rev4_row<R>(wb, tid);
    if (l > s0) {
      if (full)
        rev4_outputs<KH, R, FAST, NORM, false, true>(w, lrow, orow, rrow, ub, hs, own, gmn, A, Bq, dgam_next, wrow);
      else
        rev4_outputs<KH, R, FAST, NORM, true, true>(w, lrow, orow, rrow, ub, hs, own, gmn, A, Bq, dgam_next, wrow);
    } else {
      if (full)
        rev4_outputs<KH, R, FAST, NORM, false, false>(w, lrow, orow, rrow, ub, hs, own, gmn, A, Bq, dgam_next, wrow);
      else
        rev4_outputs<KH, R, FAST, NORM, true, false>(w, lrow, orow, rrow, ub, hs, own, gmn, A, Bq, dgam_next, wrow);
    }
    if (PIPE == 1 && l - 1 >= s0) {
      __syncwarp();  // every lane of the warp has read its row of the single u buffer
      window(l - 1, 0);
    }
    // per-warp reduction of this step's partials -> red[li][warp][.]
    {
      float vals[VP];
      vals[0] = none ? 0.f : dgam;
#pragma unroll
      for (int j = 0; j < NTU; ++j) {
        vals[1 + 2 * j] = none ? 0.f : lof(A[j]) + hif(Bq[j]);
        vals[2 + 2 * j] = none ? 0.f : hif(A[j]) - lof(Bq[j]);
      }
#pragma unroll
      for (int i = V; i < VP; ++i) vals[i] = 0.f;
      if (!(LDBP_REV4_ABL & 1)) warp_reduce_write<VP>(vals, lane, sm.red + ((size_t)li * NW + warp) * V, V);
    }
    dgam = dgam_next;
    if (!(LDBP_REV4_ABL & 4)) __syncthreads();
  }
  // adjoint w.r.t. u_hat^(s0): the last step's outputs, own row of the last-written buffer
  if (a.gout) {
    const uint32_t fb = ((s1 - s0) & 1) ? gb1 : gb0;
    const Rev4Row r = rev4_row<R>(fb, tid);
    f2x g[R];
#pragma unroll
    for (int c = 0; c < R / 2; ++c) lds2(((c & 1) ? r.po : r.pe) + 16u * c, g[2 * c], g[2 * c + 1]);
    store_owned<R>(a.gout, e0, a.g, g);
  }
  // CTA reduction in fp64, fixed order over warps, mapped back to the original parameters
  // (identical to rev_tile_kernel): dgamma_i = |P_i|^2 dgamma_hat_i, dh^(i) = conj(1/c_i) dh_hat^(i).
  // Kept out of the step loop: fp64 divisions on one warp between two barriers stretch every step.
  const int S = s1 - s0;
  for (int i = tid; i < S * npairs; i += NT) {
    const int li = i / npairs, q = i % npairs;
    const int l = s0 + li;
    double* out = a.partials + ((int64_t)tile * a.M + l) * V;
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
        // conj(1/c) dh_hat = dh_hat c / |c|^2; 1/|c|^2 by two Newton steps from the fp32 reciprocal
        // (full fp64 accuracy without the long DDIV sequence at the end of every tile)
        const double cx = nm.c.x, cy = nm.c.y, m = cx * cx + cy * cy;
        double r = (double)__frcp_rn((float)m);
        r = r * (2.0 - m * r);
        r = r * (2.0 - m * r);
        const double r2 = (re * cx - im * cy) * r, i2 = (re * cy + im * cx) * r;
        re = r2;
        im = i2;
      }
      out[v2] = re;
      out[v2 + 1] = im;
    }
  }
}

// Shared memory (mirrors the carve-up below; 16-byte aligned regions).
__host__ __device__ constexpr size_t rev4_smem_bytes(int kh, int steps, int M) {
  return 16 * (size_t)(2 * (rev4_threads(kh) / 32)) +                                         // bulk mbarriers
         sizeof(float2) * (size_t)(2 + LDBP_REV4_PIPE) * rev4_threads(kh) * rev4_r(kh) +      // gbuf + ubuf
         32 * (size_t)steps * (kh + 1) +                                                      // taps_adj
         16 * (size_t)M +                                                                     // norm
         4 * (size_t)(((size_t)steps * (rev4_threads(kh) / 32) * (3 + 2 * kh) + 3) & ~(size_t)3) +  // red
         4 * (size_t)((rev4_threads(kh) / 32 + 3) & ~3) +                                     // lred
         4 * (size_t)((steps + 3) & ~3) + 16;                                                 // gamma, flag
}

template <int KH, bool FAST>
__global__ void __launch_bounds__(rev4_threads(KH), 65536 / (rev4_threads(KH) * rev4_regs(KH)))
    rev4_tile_kernel(const RevArgs a) {
  constexpr int NTU = KH + 1;
  constexpr int NT = rev4_threads(KH), NW = NT / 32, R = rev4_r(KH);
  constexpr int V = 1 + 2 * NTU;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int S = a.s1 - a.s0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  Rev4Smem sm;
  sm.bbar = reinterpret_cast<uint64_t*>(smem_raw);                                        // 2*NW (16 B each slot pair)
  sm.gbuf = reinterpret_cast<f2x*>(smem_raw + 16 * 2 * NW);                               // 2*NT*R
  sm.ubuf = sm.gbuf + (size_t)2 * NT * R;                                                 // PIPE*NT*R
  sm.taps_adj = reinterpret_cast<TapP*>(sm.ubuf + (size_t)LDBP_REV4_PIPE * NT * R);       // S*NTU
  sm.norm = reinterpret_cast<StepNorm*>(sm.taps_adj + S * NTU);                           // M
  sm.red = reinterpret_cast<float*>(sm.norm + a.M);                                       // S*NW*V
  sm.lred = sm.red + ((S * NW * V + 3) & ~3);                                             // NW
  sm.gamma = sm.lred + ((NW + 3) & ~3);                                                   // S
  sm.flag = reinterpret_cast<int*>(sm.gamma + ((S + 3) & ~3));

  if (threadIdx.x < 2 * NW) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(sm.bbar + threadIdx.x)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (a.ptab) {
    load_ptab<NTU>(a.ptab, a.M, a.s0, a.s1, sm.norm, nullptr, sm.taps_adj, sm.gamma, nullptr, sm.flag);
  } else {
    norm_range<KH, true>(a.taps, a.mask, a.T, 0, a.M, sm.norm, sm.flag);
    const bool norm0 = *sm.flag;
    stage_range<KH, true, false, true>(a.taps, a.gamma, a.mask, a.T, a.s0, a.s1, 0, nullptr, sm.taps_adj, sm.gamma,
                                       sm.norm, norm0);
  }
  __syncthreads();
  const bool norm = *sm.flag;
  // persistent: the CTA walks tiles blockIdx.x, + gridDim.x, ... (parameter table staged once)
  const int ntiles = a.ntiles > 0 ? a.ntiles : (int)gridDim.x;
  unsigned bph = 0u;
  for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t e0 = tile_lo(a.g, tile) - a.g.H + (int64_t)threadIdx.x * R;
    const Span sp = make_span(e0, a.g);
    const int64_t fast_off = span_fast<R>(sp, a.g, e0) ? sp.b0 * a.g.n + (sp.q0 - a.g.H) : -1;
    const uint32_t own = owned_mask<R>(e0, a.g, tile);
    if (norm)
      rev4_body<KH, R, FAST, true>(a, sm, e0, fast_off, own, lane, warp, tile, bph);
    else
      rev4_body<KH, R, FAST, false>(a, sm, e0, fast_off, own, lane, warp, tile, bph);
    __syncthreads();  // shared buffers are reused by the next tile
  }
}

}  // namespace ldbp

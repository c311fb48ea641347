// ldbp_essm.cuh — learned enhanced SSM (ESSM), sm_100a.
//
// Paper §III-D, Eq. (nl_filtered): the nonlinear step of step i filters |a|^2,
//   v_t = a_t exp(j gamma'_i sum_{k=-kappa}^{kappa} eta^(i)_k |a_{(t-k) mod n}|^2),
// a = h^(i) (*) u (the centred FIR of Eq. (7)); theta = {h^(i), eta^(i), gamma'_i} (reading G20).
// One launch per step; a CTA owns W consecutive samples of one block (grid (tiles, B)) and works
// in shared memory with circular (mod n) halos: the filter's dependency cone is Kh + kappa per
// step, larger than one thread's register run, so the tile lives in smem (FFMA2 complex FIRs,
// conflict-free lane-consecutive accesses).
//
// Reverse step (oracle/essm.py): with p = |a|^2, psi = eta (*) p, phi = gamma' psi, v = a e^{j phi}
// and g = dL/dv:  c = Im(g conj v), q_m = gamma' sum_k eta_k c_{m+k}, ga = g e^{-j phi} + 2 q a,
// gu_s = sum_j conj(h_j) ga_{s+j};  dgamma' = sum c psi,  deta_k = gamma' sum_t c_t p_{t-k},
// dh_j = sum_t ga_t conj(u_{t-j})  over owned t.  Gradient sums: every thread takes one
// (component, sample-group) pair and loops over its group's owned samples; the groups are then
// summed in fixed order in fp64 -> per-CTA partials (deterministic, no atomics).
#pragma once

namespace ldbp {

constexpr int kEssmThreads = 256;
#ifndef LDBP_ESSM_W
#define LDBP_ESSM_W 1936  // owned samples per CTA: with the largest computed region (A: W + 2 (8 + 2
                          // kappa_8) = 2048 at kappa <= 24) every filter phase is ONE pass of 256
                          // threads x 8 outputs (round 1's 1024 left ~half the threads idle in every
                          // phase: measured 24 % barrier stalls)
#endif
#ifndef LDBP_ESSM_QN
#define LDBP_ESSM_QN 8    // owned samples per thread in the gradient sums (QN x threads >= W)
#endif
constexpr int kEssmW = LDBP_ESSM_W;
constexpr int kEssmMaxKappa = 32;
constexpr int kEssmMaxT = 15;

struct EssmArgs {
  const float2* u;       // step input [B][n]
  const float2* gin;     // adjoint w.r.t. the step output, or nullptr -> seed g = 2(v - target)
  const float2* target;  // [B][n] (seed mode)
  float2* out;           // forward: v [B][n];  backward: gu [B][n] (nullptr: not needed)
  const float2* taps;    // [T] this step
  const float* eta;      // [2 kappa + 1] this step
  const float* gamma;    // [M] (device); this step's gamma' = gamma[step]
  int step;
  double* partials;      // backward: [gridDim.x * gridDim.y][V] this step, V = 2 + 2T + (2kappa+1)
  int64_t n;
  int T, kappa, tiles;
};

__device__ __forceinline__ int64_t essm_mod(int64_t i, int64_t n) {
  i %= n;
  return i < 0 ? i + n : i;
}
// Position (s0 + i) mod n for s0 in [0, n) and i >= 0: one conditional wrap when i < n.
__device__ __forceinline__ int64_t essm_wrap(int64_t s0, int i, int64_t n) {
  const int64_t j = s0 + i;
  return j < n ? j : (i < n ? j - n : j % n);
}

// acc + h*s and acc + conj(h)*s for complex h, s (FFMA2 form, see ldbp_f32x2.cuh)
__device__ __forceinline__ f2x essm_mac(f2x acc, float2 h, f2x s) {
  return fma2(bcast(hif(s)), pk(-h.y, h.x), fma2(bcast(lof(s)), pk(h.x, h.y), acc));
}
__device__ __forceinline__ f2x essm_mac_conj(f2x acc, float2 h, f2x s) {
  return fma2(bcast(hif(s)), pk(h.y, h.x), fma2(bcast(lof(s)), pk(h.x, -h.y), acc));
}

// Register-blocked filters.  Every thread produces kEQ consecutive outputs; shared arrays use a
// padded layout (f2x: one pad per 16, float: one pad per 32) so that the lanes' kEQ-element runs
// hit distinct banks.  The real kappa-filters run over zero-padded tap tables in blocks of 8 taps
// with compile-time register indices (the window is reloaded per block).
constexpr int kEQ = 8;
constexpr int kESlack = 16;  // logical slack after every array (blocked reads run past the end)
// Row-padded layouts: rows of 8 elements with one pad element (stride 9).  A thread's run starting
// at an 8-aligned logical index b then sits at pfl(b) + i + (i >> 3) — one address per run with
// compile-time offsets (the filter windows below all start 8-aligned: b = o0 + j0), and lanes 8
// outputs apart land 9 words apart: conflict-free (f2x: 18 words, conflict-free per half-warp).
// (Round 1 padded per 16 / 32 elements, which needs the full index arithmetic at every access.)
__device__ __forceinline__ int pcx(int i) { return i + (i >> 3); }  // f2x arrays
__device__ __forceinline__ int pfl(int i) { return i + (i >> 3); }  // float arrays
__host__ __device__ __forceinline__ int essm_pc_size(int n) { return n + (n >> 3) + 1; }
__host__ __device__ __forceinline__ int essm_pf_size(int n) { return n + (n >> 3) + 1; }
__device__ __forceinline__ constexpr int prow(int i) { return i + (i >> 3); }  // offset within an aligned run
__host__ __device__ __forceinline__ int essm_nj(int kap) { return ((2 * kap + 1 + 7) / 8) * 8; }

// Asynchronous tile load: dst[pcx(i)] = src[(t_start + i) mod n] for i < cnt, zeros for the slack
// (cp.async 8-byte copies straight into shared memory: every thread's loads are in flight at
// once instead of load -> store round trips).  t_start may be negative; one conditional wrap per
// element when the halo is shorter than the block (always for the BJ shapes), a modulo otherwise.
__device__ __forceinline__ void essm_tile_async(f2x* dst, const f2x* __restrict__ src, int64_t t_start, int cnt,
                                                int64_t n) {
  const int64_t s0 = t_start < 0 ? t_start + n : t_start;                  // in [0, n) when t_start > -n
  const bool simple = t_start > -n && t_start < n && s0 + cnt <= 2 * n;    // at most one wrap
  for (int i = threadIdx.x; i < cnt + kESlack; i += kEssmThreads) {
    if (i < cnt) {
      int64_t t = s0 + i;
      if (simple) {
        if (t >= n) t -= n;
      } else {
        t = essm_mod(t_start + i, n);
      }
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst + pcx(i))), "l"(src + t) : "memory");
    } else {
      dst[pcx(i)] = 0ull;
    }
  }
}

// Halos are padded to multiples of 8 (kappa_8 = roundup8(kappa), 8 for the FIR halo) so that the
// offset between any two arrays is a multiple of 8 and every register window below starts at an
// 8-aligned index (one address per run, compile-time offsets, conflict-free rows).
__device__ __forceinline__ int essm_k8(int kap) { return (kap + 7) & ~7; }
__host__ __device__ __forceinline__ int essm_nj2(int kap) { return (((kap + 7) & ~7) + kap + 1 + 7) & ~7; }

// Shifted tap table: tt[j] = eta_k with k = k8 - j (dir = +1) or k = j - k8 (dir = -1), zero where
// |k| > kappa; then acc[q] = sum_j tt[j] X[x0 + q - k8 + j] is sum_k eta_k X[x0 + q -+ k] with an
// 8-aligned window start x0 - k8.
__device__ __forceinline__ void essm_tap_table(const float* __restrict__ eta, int kap, int dir, float* tt) {
  const int k8 = essm_k8(kap), NJ = essm_nj2(kap);
  for (int j = threadIdx.x; j < NJ; j += kEssmThreads) {
    const int k = dir > 0 ? k8 - j : j - k8;
    tt[j] = (k >= -kap && k <= kap) ? eta[k + kap] : 0.f;
  }
}

// acc[q] = sum_j tt[j] X[x0 + q - k8 + j]  (X float, row-padded; x0 - k8 8-aligned)
__device__ __forceinline__ void essm_rfilt(const float* __restrict__ X, int x0, int kap, const float* __restrict__ tt,
                                           float (&acc)[kEQ]) {
  const int NJ = essm_nj2(kap);
#pragma unroll
  for (int q = 0; q < kEQ; ++q) acc[q] = 0.f;
  const float* xb = X + pfl(x0 - essm_k8(kap));
  for (int j0 = 0; j0 < NJ; j0 += 8, xb += 9) {
    float w[kEQ + 7];
#pragma unroll
    for (int i = 0; i < kEQ + 7; ++i) w[i] = xb[prow(i)];
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const float h = tt[j0 + t];
#pragma unroll
      for (int q = 0; q < kEQ; ++q) acc[q] = fmaf(h, w[q + t], acc[q]);
    }
  }
}

// complex FIR with output q centred at In index xa + 8 + q (xa 8-aligned):
// acc[q] = sum_j h_j In[xa + 8 + q - j] (ADJ: sum_j conj(h_j) In[xa + 8 + q + j]), j in [-KH, KH]
template <int KH, bool ADJ>
__device__ __forceinline__ void essm_cfir(const f2x* __restrict__ In, int xa, const float2* __restrict__ sh_h,
                                          f2x (&acc)[kEQ]) {
  constexpr int SH = 8 - KH;  // window start xa + SH
  f2x w[kEQ + 2 * KH];
  const f2x* ib = In + pcx(xa);
#pragma unroll
  for (int i = 0; i < kEQ + 2 * KH; ++i) w[i] = ib[prow(SH + i)];
#pragma unroll
  for (int q = 0; q < kEQ; ++q) acc[q] = 0ull;
#pragma unroll
  for (int jj = 0; jj < 2 * KH + 1; ++jj) {
    const float2 h = sh_h[jj];
#pragma unroll
    for (int q = 0; q < kEQ; ++q)
      acc[q] = ADJ ? essm_mac_conj(acc[q], h, w[q + KH + (jj - KH)]) : essm_mac(acc[q], h, w[q + KH - (jj - KH)]);
  }
}

// Forward step (halos padded, see essm_k8): U on [-(8 + k8), W + 8 + k8), A/P on [-k8, W + k8),
// v on [0, W).  A index i <-> U index i + 8; owned i <-> A/P index i + k8.
template <int KH, bool FAST>
__global__ void __launch_bounds__(kEssmThreads) essm_fwd_step_kernel(const EssmArgs a) {
  extern __shared__ __align__(16) unsigned char es_smem[];
  const int kap = a.kappa, k8 = essm_k8(kap);
  const float gam = a.gamma[a.step];
  const int b = blockIdx.y, tile = blockIdx.x;
  const int64_t t0 = (int64_t)tile * kEssmW;
  const int hu = 8 + k8, nu = kEssmW + 2 * hu, na = kEssmW + 2 * k8;
  float2* sh_h = reinterpret_cast<float2*>(es_smem);                // [kEssmMaxT]
  float* tt = reinterpret_cast<float*>(sh_h + kEssmMaxT);           // [essm_nj(kEssmMaxKappa)]
  f2x* U = reinterpret_cast<f2x*>(tt + essm_nj(kEssmMaxKappa) + 2); // [pc(nu + slack)]
  f2x* A = U + essm_pc_size(nu + kESlack);                          // [pc(na + slack)]
  float* P = reinterpret_cast<float*>(A + essm_pc_size(na + kESlack));  // [pf(na + slack)]
  for (int i = threadIdx.x; i < 2 * KH + 1; i += kEssmThreads) sh_h[i] = a.taps[i];
  essm_tap_table(a.eta, kap, +1, tt);
  const f2x* ub = reinterpret_cast<const f2x*>(a.u) + (int64_t)b * a.n;
  essm_tile_async(U, ub, t0 - hu, nu, a.n);
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  for (int i = threadIdx.x; i < kESlack; i += kEssmThreads) P[pfl(na + i)] = 0.f;
  __syncthreads();
  // a_t = sum_j h_j u_{t-j}
  for (int o0 = threadIdx.x * kEQ; o0 < na; o0 += kEssmThreads * kEQ) {
    f2x acc[kEQ];
    essm_cfir<KH, false>(U, o0, sh_h, acc);
    f2x* ar = A + pcx(o0);
    float* pr = P + pfl(o0);
#pragma unroll
    for (int q = 0; q < kEQ; ++q) {
      ar[prow(q)] = acc[q];
      const float2 av = upk(acc[q]);
      pr[prow(q)] = fmaf(av.x, av.x, av.y * av.y);
    }
  }
  __syncthreads();
  // psi_t = sum_k eta_k p_{t-k}
  f2x* vb = reinterpret_cast<f2x*>(a.out) + (int64_t)b * a.n;
  const int own = (int)(a.n - t0 < (int64_t)kEssmW ? a.n - t0 : (int64_t)kEssmW);
  for (int o0 = threadIdx.x * kEQ; o0 < own; o0 += kEssmThreads * kEQ) {
    float psi[kEQ];
    essm_rfilt(P, o0 + k8, kap, tt, psi);
    const f2x* ar = A + pcx(o0 + k8);
#pragma unroll
    for (int q = 0; q < kEQ; ++q) {
      if (o0 + q >= own) break;
      float s, c;
      sincos_phase<FAST>(gam * psi[q], &s, &c);
      const float2 av = upk(ar[prow(q)]);
      vb[t0 + o0 + q] = pk(fmaf(av.x, c, -av.y * s), fmaf(av.x, s, av.y * c));
    }
  }
}

// Backward step.  Regions relative to t0, halos padded to multiples of 8 (k8 = roundup8(kappa)):
// U: 16 + 2 k8, A/P: 8 + 2 k8, G/PSI/C (and phi): 8 + k8, GA/Q: 8; outputs and gradient sums on
// owned [0, W).  Index relations: A i <-> U i + 8; G i <-> A/P i + k8; Q i <-> G/C i + k8, A i + 2 k8;
// owned s <-> Q s + 8, G s + 8 + k8, A s + 8 + 2 k8, U s + 16 + 2 k8.
template <int KH, bool FAST>
__global__ void __launch_bounds__(kEssmThreads) essm_bwd_step_kernel(const EssmArgs a) {
  extern __shared__ __align__(16) unsigned char es_smem[];
  const int kap = a.kappa, k8 = essm_k8(kap);
  const float gam = a.gamma[a.step];
  const int b = blockIdx.y, tile = blockIdx.x;
  const int64_t t0 = (int64_t)tile * kEssmW;
  const int own = (int)(a.n - t0 < (int64_t)kEssmW ? a.n - t0 : (int64_t)kEssmW);
  const int hU = 16 + 2 * k8, hA = 8 + 2 * k8, hG = 8 + k8, hQ = 8;
  const int nU = kEssmW + 2 * hU, nA = kEssmW + 2 * hA, nG = kEssmW + 2 * hG, nQ = kEssmW + 2 * hQ;
  const int T = 2 * KH + 1, NE = 2 * kap + 1;
  const int V = 2 + 2 * T + NE;  // [dgamma | loss | dh re/im (T) | deta (NE)]
  float2* sh_h = reinterpret_cast<float2*>(es_smem);
  float* tt_f = reinterpret_cast<float*>(sh_h + kEssmMaxT);        // forward table (psi)
  float* tt_b = tt_f + essm_nj(kEssmMaxKappa);                      // reversed table (q)
  f2x* U = reinterpret_cast<f2x*>(tt_b + essm_nj(kEssmMaxKappa) + 2);
  f2x* A = U + essm_pc_size(nU + kESlack);
  f2x* G = A + essm_pc_size(nA + kESlack);
  f2x* GA = G + essm_pc_size(nG + kESlack);
  float* P = reinterpret_cast<float*>(GA + essm_pc_size(nQ + kESlack));
  float* PSI = P + essm_pf_size(nA + kESlack);
  float* C = PSI + essm_pf_size(nG + kESlack);
  for (int i = threadIdx.x; i < T; i += kEssmThreads) sh_h[i] = a.taps[i];
  essm_tap_table(a.eta, kap, +1, tt_f);
  essm_tap_table(a.eta, kap, -1, tt_b);
  const f2x* ub = reinterpret_cast<const f2x*>(a.u) + (int64_t)b * a.n;
  essm_tile_async(U, ub, t0 - hU, nU, a.n);
  {  // the incoming adjoint (or the target, seed mode) on the G region, straight into G
    const f2x* gsrc = reinterpret_cast<const f2x*>(a.gin ? a.gin : a.target) + (int64_t)b * a.n;
    essm_tile_async(G, gsrc, t0 - hG, nG, a.n);
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
  for (int i = threadIdx.x; i < kESlack; i += kEssmThreads) {  // finite slack (zero taps x slack)
    P[pfl(nA + i)] = 0.f;
    C[pfl(nG + i)] = 0.f;
    PSI[pfl(nG + i)] = 0.f;
    GA[pcx(nQ + i)] = 0ull;
  }
  __syncthreads();
  // a, p on the A region
  for (int o0 = threadIdx.x * kEQ; o0 < nA; o0 += kEssmThreads * kEQ) {
    f2x acc[kEQ];
    essm_cfir<KH, false>(U, o0, sh_h, acc);
    f2x* ar = A + pcx(o0);
    float* pr = P + pfl(o0);
#pragma unroll
    for (int q = 0; q < kEQ; ++q) {
      ar[prow(q)] = acc[q];
      const float2 av = upk(acc[q]);
      pr[prow(q)] = fmaf(av.x, av.x, av.y * av.y);
    }
  }
  __syncthreads();
  // psi, v, g (loaded or seeded), c on the G region
  const bool have_g = a.gin != nullptr;
  float lsum = 0.f;
  for (int o0 = threadIdx.x * kEQ; o0 < nG; o0 += kEssmThreads * kEQ) {
    float psi[kEQ];
    essm_rfilt(P, o0 + k8, kap, tt_f, psi);
    const f2x* ar = A + pcx(o0 + k8);
    f2x* gr = G + pcx(o0);
    float* psr = PSI + pfl(o0);
    float* cr = C + pfl(o0);
#pragma unroll
    for (int q = 0; q < kEQ; ++q) {
      const int i = o0 + q;
      if (i >= nG) break;
      float s, c;
      sincos_phase<FAST>(gam * psi[q], &s, &c);
      const float2 av = upk(ar[prow(q)]);
      const float vx = fmaf(av.x, c, -av.y * s), vy = fmaf(av.x, s, av.y * c);
      float2 g = upk(gr[prow(q)]);  // prefetched adjoint, or the target in seed mode
      if (!have_g) {
        const float ex = vx - g.x, ey = vy - g.y;
        g = make_float2(2.f * ex, 2.f * ey);
        if (i >= hG && i < hG + own) lsum = fmaf(ex, ex, fmaf(ey, ey, lsum));
      }
      gr[prow(q)] = pk(g.x, g.y);
      psr[prow(q)] = psi[q];
      cr[prow(q)] = fmaf(g.y, vx, -g.x * vy);  // Im(g conj v)
    }
  }
  __syncthreads();
  // q and ga on the Q region
  for (int o0 = threadIdx.x * kEQ; o0 < nQ; o0 += kEssmThreads * kEQ) {
    float qv[kEQ];
    essm_rfilt(C, o0 + k8, kap, tt_b, qv);  // sum_k eta_k c_{m+k}
    const float* psr = PSI + pfl(o0 + k8);
    const f2x* gr = G + pcx(o0 + k8);
    const f2x* ar = A + pcx(o0 + 2 * k8);
    f2x* gar = GA + pcx(o0);
#pragma unroll
    for (int q = 0; q < kEQ; ++q) {
      const int i = o0 + q;
      if (i >= nQ) break;
      const float qq = gam * qv[q];
      float s, c;
      sincos_phase<FAST>(gam * psr[prow(q)], &s, &c);
      const float2 gv = upk(gr[prow(q)]), av = upk(ar[prow(q)]);
      gar[prow(q)] = pk(fmaf(gv.x, c, fmaf(gv.y, s, 2.f * qq * av.x)), fmaf(gv.y, c, fmaf(-gv.x, s, 2.f * qq * av.y)));
    }
  }
  __syncthreads();
  // gu on owned: sum_j conj(h_j) ga_{s+j}, owned s <-> Q index s + 8
  if (a.out) {
    f2x* ob = reinterpret_cast<f2x*>(a.out) + (int64_t)b * a.n;
    for (int o0 = threadIdx.x * kEQ; o0 < own; o0 += kEssmThreads * kEQ) {
      f2x acc[kEQ];
      essm_cfir<KH, true>(GA, o0, sh_h, acc);
#pragma unroll
      for (int q = 0; q < kEQ; ++q)
        if (o0 + q < own) ob[t0 + o0 + q] = acc[q];
    }
  }
  // gradient sums over owned t, register-blocked: thread tid owns samples i = QN tid + q and forms
  // its partial of every component from register windows (dh: the T-tap correlation of ga with
  // conj(u); deta: the (2 kappa + 1)-tap correlation of c with p, in blocks of 8 lags placed so
  // that every p window starts 8-aligned); each block of 8 partials is reduced across the warp with
  // the transposing butterfly into red[warp][v]; the CTA then sums the 8 warps in fixed order.
  lsum = warp_sum(lsum);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  double* outp = a.partials + (int64_t)cta * V;
  __shared__ float lred[kEssmThreads / 32];
  __shared__ float red[kEssmThreads / 32][2 + 2 * kEssmMaxT + 2 * kEssmMaxKappa + 1 + 8];
  if (lane == 0) lred[warp] = lsum;
  constexpr int QN = LDBP_ESSM_QN;
  static_assert(QN == 8, "aligned runs of 8 owned samples per thread");
  static_assert(QN * kEssmThreads >= kEssmW, "QN owned samples per thread cover the tile");
  const int i0 = QN * threadIdx.x;
  // threads past the tile (QN x threads > W) read their windows at 0 (finite data; all their
  // products are multiplied by zeroed c / ga values)
  const int iw = i0 < own ? i0 : 0;
  float cq[QN];
  {
    const float* cr = C + pfl(i0 + hG);
#pragma unroll
    for (int q = 0; q < QN; ++q) cq[q] = i0 + q < own ? cr[prow(q)] : 0.f;
  }
  auto flush8 = [&](float (&v)[8], int comp0, int lo, int lim) {  // warp-reduce 8 partials -> red[warp][.]
    const float r = warp_reduce_scatter<8>(v, lane);
    const int idx = lane >> 2;
    if ((lane & 3) == 0 && comp0 + idx >= lo && comp0 + idx < lim) red[warp][comp0 + idx] = r;
  };
  {  // comp 0 (dgamma') and the T complex tap correlations, comps 2 .. 2 + 2T
    float vals[2 + 2 * kEssmMaxT + 6];  // padded to a multiple of 8
#pragma unroll
    for (int v = 0; v < 2 + 2 * kEssmMaxT + 6; ++v) vals[v] = 0.f;
    {
      const float* psr = PSI + pfl(i0 + hG);
#pragma unroll
      for (int q = 0; q < QN; ++q) vals[0] = fmaf(cq[q], i0 + q < own ? psr[prow(q)] : 0.f, vals[0]);
    }
    float2 gq[QN];
    {
      const f2x* gar = GA + pcx(i0 + hQ);
#pragma unroll
      for (int q = 0; q < QN; ++q) gq[q] = i0 + q < own ? upk(gar[prow(q)]) : make_float2(0.f, 0.f);
    }
    // u window: U index i + hU - j, j = jj - KH: from U index i0 + hU - KH = (i0 + hU - 8) + SH
    float2 uw[QN + 2 * KH];
    {
      const f2x* ur = U + pcx(iw + hU - 8);
#pragma unroll
      for (int w = 0; w < QN + 2 * KH; ++w) uw[w] = upk(ur[prow(8 - KH + w)]);
    }
#pragma unroll
    for (int jj = 0; jj < 2 * KH + 1; ++jj) {
      float re = 0.f, im = 0.f;
#pragma unroll
      for (int q = 0; q < QN; ++q) {
        const float2 g = gq[q], w = uw[q + 2 * KH - jj];  // U[i0 + q + hU - (jj - KH)]
        re = fmaf(g.x, w.x, fmaf(g.y, w.y, re));
        im = fmaf(g.y, w.x, fmaf(-g.x, w.y, im));
      }
      vals[2 + 2 * jj] = re;
      vals[3 + 2 * jj] = im;
    }
    constexpr int NV = ((2 + 2 * (2 * KH + 1)) + 7) / 8;
#pragma unroll
    for (int c8 = 0; c8 < NV; ++c8) {
      float v8[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) v8[t] = vals[8 * c8 + t];
      flush8(v8, 8 * c8, 0, 2 + 2 * T);  // comps below the deta block only
    }
  }
  {  // deta_kk = sum_t c_t p_{t-k}, k = kk - kappa: P index t + hA + kappa - kk; comps 2 + 2T + kk.
     // Lag blocks [k0, k0 + 8) with k0 = kappa + 1 (mod 8): the window start i0 + hA + kappa - k0 - 7
     // is then 8-aligned (hA is a multiple of 8); lags outside [0, NE) are dropped.
    const int base = 2 + 2 * T;
    const int k0s = ((kap + 1) & 7) - 8;
    for (int k0 = k0s; k0 < NE; k0 += 8) {
      // P[i0 + q + hA + kappa - (k0 + t)] for t < 8, q < 8: window index w = q - t + 7
      float pw[QN + 7];
      const float* pr = P + pfl(iw + hA + kap - k0 - 7);
#pragma unroll
      for (int w = 0; w < QN + 7; ++w) pw[w] = pr[prow(w)];
      float v8[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        float acc = 0.f;
#pragma unroll
        for (int q = 0; q < QN; ++q) acc = fmaf(cq[q], pw[q - t + 7], acc);
        v8[t] = (k0 + t >= 0 && k0 + t < NE) ? acc : 0.f;
      }
      flush8(v8, base + k0, base, V);  // comps base + k0 .. base + k0 + 7 (inside [base, V))
    }
  }
  __syncthreads();
  for (int comp = threadIdx.x; comp < V; comp += kEssmThreads) {
    if (comp == 1) {
      double t = 0.0;
      for (int w = 0; w < kEssmThreads / 32; ++w) t += (double)lred[w];
      outp[1] = t;
    } else {
      double t = 0.0;
      for (int w = 0; w < kEssmThreads / 32; ++w) t += (double)red[w][comp];
      outp[comp] = comp >= 2 + 2 * T ? (double)gam * t : t;
    }
  }
}

// Fixed-order reduction over CTAs for every step, and the ABI layout:
// buf = [sum |e|^2 | dgamma [M] | dtaps [M][T][2] (SYM: tied +-j) | deta [M][2kappa+1]].
struct EssmReduceArgs {
  const double* partials;  // [M][nblk][V]
  int M, nblk, T, kappa, sym;
  double* buf;
};

// First level of the fixed-order reduction: CTA (chunk ch, step st) sums partials of CTAs
// [ch*CH, ch*CH + CH) in order, one thread per component v (coalesced over v), into
// out[st][ch][v]; essm_reduce_kernel then sums the chunk totals in order.  (A single thread per
// component walking all CTAs was a chain of dependent L2 round trips: ~1.2 ms at the C3-like
// shape, 4608 CTAs per step.)
constexpr int kEssmRedChunk = 64;
__global__ void __launch_bounds__(128) essm_reduce_chunks_kernel(const double* __restrict__ partials, int nblk, int V,
                                                                 double* __restrict__ out) {
  const int ch = blockIdx.x, st = blockIdx.y, nch = gridDim.x;
  const int c0 = ch * kEssmRedChunk, c1 = min(nblk, c0 + kEssmRedChunk);
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    const double* p = partials + ((int64_t)st * nblk + c0) * V + v;
    double s = 0.0;
#pragma unroll 8
    for (int c = c0; c < c1; ++c, p += V) s += *p;
    out[((int64_t)st * nch + ch) * V + v] = s;
  }
}

__global__ void __launch_bounds__(256) essm_reduce_kernel(const EssmReduceArgs a) {
  const int V = 2 + 2 * a.T + 2 * a.kappa + 1;
  const int NE = 2 * a.kappa + 1;
  const int kh = (a.T - 1) / 2;
  const int total = a.M * V;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int st = idx / V, v = idx % V;
    const double* p = a.partials + (int64_t)st * a.nblk * V + v;
    double s = 0.0;
    for (int c = 0; c < a.nblk; ++c) s += p[(int64_t)c * V];
    if (v == 0) {
      a.buf[1 + st] = s;
    } else if (v == 1) {
      if (st == a.M - 1) a.buf[0] = s;  // only the seeded (last) step carries the loss
    } else if (v < 2 + 2 * a.T) {
      const int jj = (v - 2) >> 1, im = (v - 2) & 1;
      double val = s;
      if (a.sym && jj != kh) {  // tied parameter: g_j + g_{-j}
        const int mirror = 2 * kh - jj;
        double s2 = 0.0;
        const double* p2 = a.partials + (int64_t)st * a.nblk * V + 2 + 2 * mirror + im;
        for (int c = 0; c < a.nblk; ++c) s2 += p2[(int64_t)c * V];
        val = s + s2;
      }
      a.buf[1 + a.M + ((int64_t)st * a.T + jj) * 2 + im] = val;
    } else {
      a.buf[1 + a.M + 2 * (int64_t)a.M * a.T + (int64_t)st * NE + (v - 2 - 2 * a.T)] = s;
    }
  }
}

}  // namespace ldbp

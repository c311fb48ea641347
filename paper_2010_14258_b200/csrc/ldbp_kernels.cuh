// ldbp_kernels.cuh — sm_100a kernels of the LDBP hot path.
//
// Data layout: complex64 blocks [B][n] as float2; taps [M][T] float2; gamma [M] float.
//
// Tiling ("extended index space"): every block b is conceptually padded to
// ext = n + 2H samples, [b*ext, (b+1)*ext), where extended position q maps to sample
// (q - H) mod n — the periodic extension of the circular frame.  The B*ext
// concatenation is cut into equal tiles of W owned samples; a CTA loads its W owned samples
// plus H on each side, runs its steps entirely on chip and writes only the owned samples
// that are real (q in [H, H+n)).  A sample's value after s steps depends on the inputs within
// s*Kh of it, so the garbage that enters at tile edges and at block junctions never reaches
// an owned real sample as long as H >= (#steps)*Kh.  W is chosen so the grid is a multiple
// of the resident-CTA count (no wave tail), independent of how n divides.
//
// Within a CTA each thread owns R consecutive samples in registers.  Per step, the Kh-sample
// halos come from the neighbouring lanes by shuffles and across warps through a small
// double-buffered shared-memory edge array (one __syncthreads per step).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#ifndef LDBP_FWD_R
#define LDBP_FWD_R 16  // samples per thread, forward kernels
#endif
#ifndef LDBP_BWD_R
#define LDBP_BWD_R 8   // samples per thread, backward kernels
#endif

namespace ldbp {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxWarps = 32;

__device__ __forceinline__ float2 operator+(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }

// Kerr rotation helpers: (c, s) = (cos phi, sin phi).
template <bool FAST>
__device__ __forceinline__ void sincos_phase(float phi, float* s, float* c) {
  if constexpr (FAST) {
    __sincosf(phi, s, c);  // MUFU.SIN / MUFU.COS (abs err ~2^-21 for |phi| <~ pi)
  } else {
    sincosf(phi, s, c);
  }
}

struct Geo {
  int64_t B, n, ext, E, W;  // blocks, block length, n + 2H, B*ext, owned width per CTA
  int H;                    // halo per side (samples)
  int big_halo;             // H > n: positions may wrap more than once
};

__device__ __forceinline__ int64_t wrap_pos(int64_t p, const Geo& g) {
  if (g.big_halo) {
    p %= g.n;
    return p < 0 ? p + g.n : p;
  }
  return p < 0 ? p + g.n : (p >= g.n ? p - g.n : p);
}

// Extended index of this thread's first sample.
__device__ __forceinline__ int64_t thread_e0(const Geo& g, int R) {
  return (int64_t)blockIdx.x * g.W - g.H + (int64_t)threadIdx.x * R;
}

// Load R consecutive extended samples starting at e0 (zeros outside [0, E)).
template <int R>
__device__ __forceinline__ void load_window(const float2* __restrict__ src, int64_t e0, const Geo& g,
                                            float2 (&u)[R]) {
  int64_t b = e0 >= 0 ? e0 / g.ext : -1;
  int64_t q = e0 - b * g.ext;  // in [0, ext) (also for e0 < 0 with b = -1 when e0 >= -ext)
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const bool ok = (b >= 0) && (b < g.B) && (e0 + k >= 0);
    float2 v = make_float2(0.f, 0.f);
    if (ok) v = __ldg(src + b * g.n + wrap_pos(q - g.H, g));
    u[k] = v;
    if (++q == g.ext) { q = 0; ++b; }
  }
}

// Bitmask of which of this thread's R samples are owned real samples of this CTA.
template <int R>
__device__ __forceinline__ uint32_t owned_mask(int64_t e0, const Geo& g, int64_t* b_out, int64_t* q_out) {
  const int64_t lo = (int64_t)blockIdx.x * g.W;
  const int64_t hi = min(lo + g.W, g.E);
  int64_t b = e0 >= 0 ? e0 / g.ext : -1;
  int64_t q = e0 - b * g.ext;
  *b_out = b;
  *q_out = q;
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    const int64_t e = e0 + k;
    if (e >= lo && e < hi && q >= g.H && q < g.H + g.n) m |= (1u << k);
    if (++q == g.ext) { q = 0; ++b; }
  }
  return m;
}

template <int R>
__device__ __forceinline__ void store_owned(float2* __restrict__ dst, int64_t e0, const Geo& g,
                                            const float2 (&u)[R]) {
  int64_t b, q;
  const uint32_t m = owned_mask<R>(e0, g, &b, &q);
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (m & (1u << k)) dst[b * g.n + (q - g.H)] = u[k];
    if (++q == g.ext) { q = 0; ++b; }
  }
}

// Halo exchange of one register array: hl = Kh samples left of u[0], hr = Kh samples right
// of u[R-1].  Shuffles inside the warp; warp edges through sh[2 buffers][2 sides][32 warps][KH].
template <int KH, int R>
__device__ __forceinline__ void exchange(const float2 (&u)[R], float2 (&hl)[KH > 0 ? KH : 1],
                                         float2 (&hr)[KH > 0 ? KH : 1], float2* sh, int buf,
                                         int lane, int warp, int nwarps) {
  if constexpr (KH > 0) {
#pragma unroll
    for (int j = 0; j < KH; ++j) {
      hl[j].x = __shfl_up_sync(kFull, u[R - KH + j].x, 1);
      hl[j].y = __shfl_up_sync(kFull, u[R - KH + j].y, 1);
      hr[j].x = __shfl_down_sync(kFull, u[j].x, 1);
      hr[j].y = __shfl_down_sync(kFull, u[j].y, 1);
    }
    float2* head = sh + ((buf * 2 + 0) * kMaxWarps) * KH;
    float2* tail = sh + ((buf * 2 + 1) * kMaxWarps) * KH;
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < KH; ++j) head[warp * KH + j] = u[j];
    }
    if (lane == 31) {
#pragma unroll
      for (int j = 0; j < KH; ++j) tail[warp * KH + j] = u[R - KH + j];
    }
    __syncthreads();
    if (lane == 0 && warp > 0) {
#pragma unroll
      for (int j = 0; j < KH; ++j) hl[j] = tail[(warp - 1) * KH + j];
    }
    if (lane == 31 && warp < nwarps - 1) {
#pragma unroll
      for (int j = 0; j < KH; ++j) hr[j] = head[(warp + 1) * KH + j];
    }
  } else {
    (void)u; (void)hl; (void)hr; (void)sh; (void)buf; (void)lane; (void)warp; (void)nwarps;
  }
}

// Window accessor: index i in [-KH, R+KH).
#define LDBP_WIN(arr, hl, hr, i) ((i) < 0 ? hl[KH + (i)] : ((i) >= R ? hr[(i) - R] : arr[(i)]))

// One FIR evaluation for output k (compile-time), a_k = sum_j h_j w_{k-j}.
// SYM: taps hs[0..KH] hold h_0..h_KH (folded, fig:filter P:494-509).
// GEN: taps hs[0..2KH] hold h_{-KH}..h_{KH}.
template <int KH, int R, bool SYM, int K>
__device__ __forceinline__ float2 fir_at(const float2 (&u)[R], const float2 (&hl)[KH > 0 ? KH : 1],
                                         const float2 (&hr)[KH > 0 ? KH : 1],
                                         const float2 (&hs)[SYM ? KH + 1 : 2 * KH + 1]) {
  float2 acc;
  if constexpr (SYM) {
    const float2 c = u[K];
    acc.x = hs[0].x * c.x;
    acc.y = hs[0].x * c.y;
    acc.x = fmaf(-hs[0].y, c.y, acc.x);
    acc.y = fmaf(hs[0].y, c.x, acc.y);
#pragma unroll
    for (int j = 1; j <= KH; ++j) {
      const float2 l = LDBP_WIN(u, hl, hr, K - j);
      const float2 r = LDBP_WIN(u, hl, hr, K + j);
      const float2 s = make_float2(l.x + r.x, l.y + r.y);
      acc.x = fmaf(hs[j].x, s.x, acc.x);
      acc.y = fmaf(hs[j].x, s.y, acc.y);
      acc.x = fmaf(-hs[j].y, s.y, acc.x);
      acc.y = fmaf(hs[j].y, s.x, acc.y);
    }
  } else {
    acc = make_float2(0.f, 0.f);
#pragma unroll
    for (int jj = 0; jj < 2 * KH + 1; ++jj) {
      const int j = jj - KH;
      const float2 w = LDBP_WIN(u, hl, hr, K - j);
      acc.x = fmaf(hs[jj].x, w.x, acc.x);
      acc.y = fmaf(hs[jj].x, w.y, acc.y);
      acc.x = fmaf(-hs[jj].y, w.y, acc.x);
      acc.y = fmaf(hs[jj].y, w.x, acc.y);
    }
  }
  return acc;
}

template <int KH, int R, bool SYM, int K = 0>
__device__ __forceinline__ void fir_all(const float2 (&u)[R], const float2 (&hl)[KH > 0 ? KH : 1],
                                        const float2 (&hr)[KH > 0 ? KH : 1],
                                        const float2 (&hs)[SYM ? KH + 1 : 2 * KH + 1], float2 (&a)[R]) {
  if constexpr (K < R) {
    a[K] = fir_at<KH, R, SYM, K>(u, hl, hr, hs);
    fir_all<KH, R, SYM, K + 1>(u, hl, hr, hs, a);
  }
}

// Kerr: v = a e^{j g |a|^2}.
template <bool FAST>
__device__ __forceinline__ float2 kerr(float2 a, float g) {
  const float p = fmaf(a.x, a.x, a.y * a.y);
  float s, c;
  sincos_phase<FAST>(g * p, &s, &c);
  return make_float2(fmaf(a.x, c, -a.y * s), fmaf(a.x, s, a.y * c));
}

template <bool SYM, int KH>
__device__ __forceinline__ constexpr int ntaps_used() { return SYM ? KH + 1 : 2 * KH + 1; }

// Stage taps/gamma of steps [s0, s1) into shared memory (masked; SYM keeps only h_0..h_Kh).
template <int KH, bool SYM>
__device__ __forceinline__ void stage_params(const float2* __restrict__ taps, const float* __restrict__ gamma,
                                             const uint8_t* __restrict__ mask, int T, int s0, int s1,
                                             float2* sh_taps, float* sh_gamma) {
  constexpr int NT = ntaps_used<SYM, KH>();
  const int cnt = (s1 - s0) * NT;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int s = s0 + i / NT;
    const int t = (i % NT) + (SYM ? KH : 0);  // index into the stored [T] row
    float2 h = taps[(int64_t)s * T + t];
    if (mask && !mask[(int64_t)s * T + t]) h = make_float2(0.f, 0.f);
    sh_taps[i] = h;
  }
  for (int i = threadIdx.x; i < s1 - s0; i += blockDim.x) sh_gamma[i] = gamma[s0 + i];
}

struct FwdArgs {
  const float2* src;
  float2* dst;
  const float2* taps;
  const float* gamma;
  const uint8_t* mask;
  int T, s0, s1;
  Geo g;
};

// ---------------------------------------------------------------------------------------
// Forward tile kernel: steps [s0, s1) of Eq. (7) for one tile, all on chip (rows a0-a4).
// ---------------------------------------------------------------------------------------
template <int KH, int R, bool SYM, bool FAST>
__global__ void __launch_bounds__(512) fwd_tile_kernel(const FwdArgs a) {
  constexpr int NTU = ntaps_used<SYM, KH>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float2* sh_edge = reinterpret_cast<float2*>(smem_raw);                 // 2*2*32*KH
  float2* sh_taps = sh_edge + 4 * kMaxWarps * (KH > 0 ? KH : 1);          // (s1-s0)*NTU
  float* sh_gamma = reinterpret_cast<float*>(sh_taps + (a.s1 - a.s0) * NTU);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  stage_params<KH, SYM>(a.taps, a.gamma, a.mask, a.T, a.s0, a.s1, sh_taps, sh_gamma);

  float2 u[R];
  const int64_t e0 = thread_e0(a.g, R);
  load_window<R>(a.src, e0, a.g, u);
  __syncthreads();

  float2 hl[KH > 0 ? KH : 1], hr[KH > 0 ? KH : 1];
  for (int s = 0; s < a.s1 - a.s0; ++s) {
    float2 hs[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) hs[j] = sh_taps[s * NTU + j];
    const float gm = sh_gamma[s];
    exchange<KH, R>(u, hl, hr, sh_edge, s & 1, lane, warp, nwarps);
    float2 acc[R];
    fir_all<KH, R, SYM>(u, hl, hr, hs, acc);
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = kerr<FAST>(acc[k], gm);
  }
  store_owned<R>(a.dst, e0, a.g, u);
}

struct BwdArgs {
  const float2* ck;      // u^(s0) [B][n]
  const float2* gin;     // dL/du^(s1) [B][n], or nullptr -> seed from target
  const float2* target;  // [B][n] (seed mode)
  float2* gout;          // dL/du^(s0) [B][n] or nullptr
  const float2* taps;
  const float* gamma;
  const uint8_t* mask;
  double* partials;      // [gridDim.x][M][V]
  double* loss_partials; // [gridDim.x] (seed mode)
  float seed_scale;      // seed g = seed_scale * (y - target)
  int T, M, s0, s1;
  Geo g;
};

template <int R>
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// ---------------------------------------------------------------------------------------
// Backward segment kernel (rows a5-a8): recompute steps [s0, s1) from the checkpoint into a
// shared-memory tape, seed (or load) the adjoint, sweep back, emit dL/du^(s0) and per-CTA
// partial sums of dgamma' and dtaps per step (fp32 within the CTA, fp64 out).
// Tape layout: tape[(l*R + k)*NT + tid] = u^(s0+l)[thread tid, sample k] (conflict free).
// ---------------------------------------------------------------------------------------
template <int KH, int R, bool SYM, bool FAST>
__global__ void __launch_bounds__(256) bwd_segment_kernel(const BwdArgs a) {
  constexpr int NTU = ntaps_used<SYM, KH>();
  constexpr int V = 1 + 2 * NTU;  // [dgamma | dtap re/im ...]
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int C = a.s1 - a.s0;
  const int nthr = blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = nthr >> 5;

  float2* sh_edge = reinterpret_cast<float2*>(smem_raw);  // two arrays: 2 * (2*2*32*KH)
  float2* sh_edge2 = sh_edge + 4 * kMaxWarps * (KH > 0 ? KH : 1);
  float2* sh_taps = sh_edge2 + 4 * kMaxWarps * (KH > 0 ? KH : 1);
  float* sh_gamma = reinterpret_cast<float*>(sh_taps + C * NTU);
  float* sh_red = sh_gamma + C;                               // [C][nwarps][V]
  float2* tape = reinterpret_cast<float2*>(sh_red + ((C * nwarps * V + 3) & ~3));  // [C][R][nthr]

  stage_params<KH, SYM>(a.taps, a.gamma, a.mask, a.T, a.s0, a.s1, sh_taps, sh_gamma);

  float2 u[R];
  const int64_t e0 = thread_e0(a.g, R);
  load_window<R>(a.ck, e0, a.g, u);
  int64_t b0, q0;
  const uint32_t own = owned_mask<R>(e0, a.g, &b0, &q0);
  __syncthreads();

  float2 hl[KH > 0 ? KH : 1], hr[KH > 0 ? KH : 1];
  // ---- forward recompute, tape = inputs of each step ----
  for (int l = 0; l < C; ++l) {
#pragma unroll
    for (int k = 0; k < R; ++k) tape[(l * R + k) * nthr + threadIdx.x] = u[k];
    float2 hs[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) hs[j] = sh_taps[l * NTU + j];
    const float gm = sh_gamma[l];
    exchange<KH, R>(u, hl, hr, sh_edge, l & 1, lane, warp, nwarps);
    float2 acc[R];
    fir_all<KH, R, SYM>(u, hl, hr, hs, acc);
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = kerr<FAST>(acc[k], gm);
  }

  // ---- seed / incoming adjoint ----
  float2 g[R];
  if (a.gin == nullptr) {
    float2 t[R];
    load_window<R>(a.target, e0, a.g, t);
    float lsum = 0.f;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const float ex = u[k].x - t[k].x, ey = u[k].y - t[k].y;
      g[k] = make_float2(a.seed_scale * ex, a.seed_scale * ey);
      if (own & (1u << k)) lsum = fmaf(ex, ex, fmaf(ey, ey, lsum));
    }
    lsum = warp_sum<R>(lsum);
    if (lane == 0) sh_red[warp] = lsum;  // reused below only after a barrier
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < nwarps; ++w) tot += (double)sh_red[w];
      a.loss_partials[blockIdx.x] = tot;
    }
    __syncthreads();
  } else {
    load_window<R>(a.gin, e0, a.g, g);
  }

  // ---- reverse sweep ----
  float2 gl[KH > 0 ? KH : 1], gr[KH > 0 ? KH : 1];
  for (int l = C - 1; l >= 0; --l) {
    float2 hs[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) hs[j] = sh_taps[l * NTU + j];
    const float gm = sh_gamma[l];
    // NL adjoint of step l: v = u (output of step l), g = dL/dv.
    float dgam = 0.f;
    float2 ga[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const float2 v = u[k];
      const float p = fmaf(v.x, v.x, v.y * v.y);
      float sn, cs;
      sincos_phase<FAST>(gm * p, &sn, &cs);
      const float cim = fmaf(g[k].y, v.x, -g[k].x * v.y);  // Im(g conj v)
      const float kk = 2.f * gm * cim;
      const float tx = fmaf(kk, v.x, g[k].x), ty = fmaf(kk, v.y, g[k].y);
      ga[k] = make_float2(fmaf(tx, cs, ty * sn), fmaf(ty, cs, -tx * sn));  // t e^{-j phi}
      if (own & (1u << k)) dgam = fmaf(cim, p, dgam);
    }
    // u^(s0+l): FIR input of step l.
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = tape[(l * R + k) * nthr + threadIdx.x];
    // exchange halos of u and ga (one barrier each).  The u buffers continue the forward
    // loop's parity sequence (the last forward exchange used (C-1)&1), hence (l+1)&1.
    exchange<KH, R>(u, hl, hr, sh_edge, (l + 1) & 1, lane, warp, nwarps);
    exchange<KH, R>(ga, gl, gr, sh_edge2, l & 1, lane, warp, nwarps);
    // tap gradients over owned samples: dh_j += ga_t conj(u_{t-j})
    float2 dh[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) dh[j] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const float2 gk = (own & (1u << k)) ? ga[k] : make_float2(0.f, 0.f);
      if constexpr (SYM) {
        const float2 w = u[k];
        dh[0].x = fmaf(gk.x, w.x, fmaf(gk.y, w.y, dh[0].x));
        dh[0].y = fmaf(gk.y, w.x, fmaf(-gk.x, w.y, dh[0].y));
#pragma unroll
        for (int j = 1; j <= KH; ++j) {
          const float2 l2 = LDBP_WIN(u, hl, hr, k - j);
          const float2 r2 = LDBP_WIN(u, hl, hr, k + j);
          const float2 s = make_float2(l2.x + r2.x, l2.y + r2.y);
          dh[j].x = fmaf(gk.x, s.x, fmaf(gk.y, s.y, dh[j].x));
          dh[j].y = fmaf(gk.y, s.x, fmaf(-gk.x, s.y, dh[j].y));
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 2 * KH + 1; ++jj) {
          const int j = jj - KH;
          const float2 w = LDBP_WIN(u, hl, hr, k - j);
          dh[jj].x = fmaf(gk.x, w.x, fmaf(gk.y, w.y, dh[jj].x));
          dh[jj].y = fmaf(gk.y, w.x, fmaf(-gk.x, w.y, dh[jj].y));
        }
      }
    }
    // FIR adjoint: g_s = sum_j conj(h_j) ga_{s+j}
#pragma unroll
    for (int k = 0; k < R; ++k) {
      float2 acc;
      if constexpr (SYM) {
        const float2 c = ga[k];
        acc.x = hs[0].x * c.x;
        acc.y = hs[0].x * c.y;
        acc.x = fmaf(hs[0].y, c.y, acc.x);
        acc.y = fmaf(-hs[0].y, c.x, acc.y);
#pragma unroll
        for (int j = 1; j <= KH; ++j) {
          const float2 l2 = LDBP_WIN(ga, gl, gr, k - j);
          const float2 r2 = LDBP_WIN(ga, gl, gr, k + j);
          const float2 s = make_float2(l2.x + r2.x, l2.y + r2.y);
          acc.x = fmaf(hs[j].x, s.x, acc.x);
          acc.y = fmaf(hs[j].x, s.y, acc.y);
          acc.x = fmaf(hs[j].y, s.y, acc.x);
          acc.y = fmaf(-hs[j].y, s.x, acc.y);
        }
      } else {
        acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int jj = 0; jj < 2 * KH + 1; ++jj) {
          const int j = jj - KH;
          const float2 w = LDBP_WIN(ga, gl, gr, k + j);
          acc.x = fmaf(hs[jj].x, w.x, acc.x);
          acc.y = fmaf(hs[jj].x, w.y, acc.y);
          acc.x = fmaf(hs[jj].y, w.y, acc.x);
          acc.y = fmaf(-hs[jj].y, w.x, acc.y);
        }
      }
      g[k] = acc;
    }
    // per-warp reduction of this step's partials
    float* red = sh_red + (l * nwarps + warp) * V;
    dgam = warp_sum<R>(dgam);
    if (lane == 0) red[0] = dgam;
#pragma unroll
    for (int j = 0; j < NTU; ++j) {
      const float rx = warp_sum<R>(dh[j].x);
      const float ry = warp_sum<R>(dh[j].y);
      if (lane == 0) { red[1 + 2 * j] = rx; red[2 + 2 * j] = ry; }
    }
  }
  if (a.gout) store_owned<R>(a.gout, e0, a.g, g);
  __syncthreads();
  // CTA reduction in fp64, fixed order over warps.
  for (int i = threadIdx.x; i < C * V; i += nthr) {
    const int l = i / V, v = i % V;
    double acc = 0.0;
    for (int w = 0; w < nwarps; ++w) acc += (double)sh_red[(l * nwarps + w) * V + v];
    a.partials[((int64_t)blockIdx.x * a.M + (a.s0 + l)) * V + v] = acc;
  }
}

#ifdef LDBP_AUX_KERNELS  // defined only by ldbp_api.cu (one definition)
// ---------------------------------------------------------------------------------------
// Deterministic fp64 reduction of per-CTA partials (row a8) and expansion to the ABI layout.
// out_mode 0: buf = [loss | dgamma[M] | dtaps[M][T][2]];  1: separate dtaps / dgamma.
// ---------------------------------------------------------------------------------------
struct ReduceArgs {
  const double* partials;       // [nblk][M][V]
  const double* loss_partials;  // [nblk] or null
  int nblk, M, T, V, kh, sym;
  const uint8_t* mask;
  double* buf;     // mode 0
  double* dtaps;   // mode 1: [M][T][2]
  double* dgamma;  // mode 1: [M]
};

__global__ void reduce_partials_kernel(const ReduceArgs a) {
  const int total = a.M * a.V;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total + 1; i += gridDim.x * blockDim.x) {
    if (i == total) {
      if (a.buf) {
        double s = 0.0;
        if (a.loss_partials)
          for (int c = 0; c < a.nblk; ++c) s += a.loss_partials[c];
        a.buf[0] = s;
      }
      continue;
    }
    double s = 0.0;
    for (int c = 0; c < a.nblk; ++c) s += a.partials[(int64_t)c * total + i];
    const int st = i / a.V, v = i % a.V;
    double* dg = a.buf ? a.buf + 1 : a.dgamma;
    double* dt = a.buf ? a.buf + 1 + a.M : a.dtaps;
    if (v == 0) {
      dg[st] = s;
    } else {
      const int ti = (v - 1) / 2, comp = (v - 1) % 2;
      if (a.sym) {
        // folded index ti = j >= 0 -> positions kh +- j
        const int p1 = a.kh + ti, p2 = a.kh - ti;
        const double m1 = (a.mask && !a.mask[st * a.T + p1]) ? 0.0 : s;
        const double m2 = (a.mask && !a.mask[st * a.T + p2]) ? 0.0 : s;
        dt[((int64_t)st * a.T + p1) * 2 + comp] = m1;
        dt[((int64_t)st * a.T + p2) * 2 + comp] = m2;
      } else {
        const double m1 = (a.mask && !a.mask[st * a.T + ti]) ? 0.0 : s;
        dt[((int64_t)st * a.T + ti) * 2 + comp] = m1;
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// Adam + mask (row a10), float64 master parameters, float32 working copies.
// ---------------------------------------------------------------------------------------
struct AdamArgs {
  const double* buf;  // [1 + M + 2MT]
  double inv_n;
  double* master;     // [2MT + M]
  double* m;
  double* v;
  double lr, b1, b2, eps, bc1, bc2;  // bc = 1 - b^t
  const uint8_t* mask;
  const uint8_t* glearn;
  float2* taps_out;
  float* gamma_out;
  int M, T;
};

__global__ void adam_kernel(const AdamArgs a) {
  const int ntap = 2 * a.M * a.T;
  const int total = ntap + a.M;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    bool frozen, zero = false;
    double g;
    if (i < ntap) {
      g = a.buf[1 + a.M + i];
      frozen = a.mask && !a.mask[i >> 1];
      zero = frozen;
    } else {
      g = a.buf[1 + (i - ntap)];
      frozen = a.glearn && !a.glearn[i - ntap];
    }
    double th = a.master[i];
    if (zero) {
      th = 0.0;
      a.m[i] = 0.0;
      a.v[i] = 0.0;
    } else if (!frozen) {
      g *= a.inv_n;
      const double m = a.b1 * a.m[i] + (1.0 - a.b1) * g;
      const double v = a.b2 * a.v[i] + (1.0 - a.b2) * g * g;
      a.m[i] = m;
      a.v[i] = v;
      const double mh = m / a.bc1, vh = v / a.bc2;
      th -= a.lr * mh / (sqrt(vh) + a.eps);
    }
    a.master[i] = th;
    if (i < ntap) {
      float* to = reinterpret_cast<float*>(a.taps_out);
      to[i] = (float)th;
    } else {
      a.gamma_out[i - ntap] = (float)th;
    }
  }
}

#endif  // LDBP_AUX_KERNELS

}  // namespace ldbp

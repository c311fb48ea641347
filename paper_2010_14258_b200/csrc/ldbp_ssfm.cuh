// ldbp_ssfm.cuh — GPU split-step Fourier channel generator, sm_100a.
//
// The link of §IV-A as the oracle simulates it (oracle/channel.py): per span, for
// each log-distributed step delta: Kerr step u <- u e^{j gamma L_eff(delta) |u|^2}
// at the segment start (reading G5), then the lossy linear step U_k <- U_k e^{-alpha delta/2}
// e^{j beta2/2 omega_k^2 delta} (Eqs. (4)-(6)); after the span the EDFA: gain
// e^{alpha L_sp/2} plus ASE sigma * CN(0,1) (draws from an input array, or in-kernel Philox
// keyed by (seed, global block, span, sample): ase_philox_cn); at the end an
// ideal low-pass |f| <= cutoff and decimation (reading G8).
//
// One persistent CTA per block (n <= 2^14 complex fp32), or a 2-/4-CTA thread-block cluster for
// n = 2^15 / 2^16, keeps the block in shared memory for the whole link.  FFTs: register passes of
// several radix-2 stages on groups of up to 16 elements (ssfm_pass), decimation-in-frequency
// forward and decimation-in-time inverse, so the spectrum stays in bit-reversed slot order and
// no bit-reversal permutation pass exists (the dispersion table is written in that order); across a cluster the four-step split's radix-C stage reads the other
// ranks through distributed shared memory.  Twiddles W_n^m = ta[m >> 6] * tb[m & 63] from two small
// fp64-accurate tables.
// The dispersion factors H_s[k] (one row per distinct step length) are precomputed in fp64 by
// ssfm_htable_kernel: omega^2 delta reaches hundreds of radians, beyond fp32 sincos accuracy.
#pragma once
#include <cooperative_groups.h>

namespace ldbp {

constexpr int kSsfmThreads = 1024;
constexpr int kSsfmLocalMaxLog2 = 14;  // samples per CTA (shared memory)
constexpr int kSsfmMaxLog2 = 16;       // per block: a cluster of up to 4 CTAs holds 2^16 samples
constexpr int kSsfmMaxSteps = 64;      // steps per span (kernel parameters)

struct SsfmArgs {
  float2* u;               // [B][n] in: transmitted waveform; out (decim == 0): channel output
  float2* r;               // [B][n / decim] out when decim > 0 (LPF + decimation)
  const float2* H;         // [S][n] dispersion factors, per cluster rank in its own bin order
  const float2* noise;     // [spans][B][n] CN(0,1) ASE draws (ase_mode 1)
  float kerr_phase[kSsfmMaxSteps];  // gamma * L_eff(delta_s) (1/W)
  int64_t n;
  int log2n, log2L, spans, S, decim;
  int ase_mode;            // 0 noiseless, 1 draws from `noise`, 2 Philox keyed by (seed, block, span, i)
  uint64_t ase_seed;
  int64_t block0;          // global index of block 0 (Philox key)
  float span_gain;         // e^{alpha L_sp / 2}
  float ase_sigma;         // sqrt(PSD * f_sim)
  float cutoff;            // pass |fftfreq| <= cutoff (cycles/sample)
};

struct SsfmDeltas {
  double d[kSsfmMaxSteps];
};

// Philox4x32-10 (Salmon et al., SC'11), the generator ldbp_inputs.ase_cn_philox implements in
// numpy: CN(0,1) draw of sample i of span sp of global block b, Box-Muller on the (x0, x1) pair
// for even i and (x2, x3) for odd i.
__device__ __forceinline__ float2 ase_philox_cn(uint64_t seed, int64_t b, int sp, int64_t i) {
  uint32_t c0 = (uint32_t)(i >> 1), c1 = (uint32_t)sp, c2 = (uint32_t)b, c3 = (uint32_t)((uint64_t)b >> 32);
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
#pragma unroll
  for (int rd = 0; rd < 10; ++rd) {
    const uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
    const uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
    const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const uint32_t a = (i & 1) ? c2 : c0, bb = (i & 1) ? c3 : c1;
  const float u1 = ((float)a + 0.5f) * 2.3283064365386963e-10f;  // 2^-32
  const float u2 = ((float)bb + 0.5f) * 2.3283064365386963e-10f;
  const float rr = sqrtf(-2.f * logf(u1)) * 0.70710678118654752f;
  float sn, cs;
  sincospif(2.f * u2, &sn, &cs);
  return make_float2(rr * cs, rr * sn);
}

// H[s][rank L + slot] = e^{-alpha delta_s/2} e^{j beta2/2 omega_k^2 delta_s} for the bin k that
// slot `slot` of cluster rank `rank` holds after the forward transform: k = rank + C bitrev_L(slot)
// (C = 1: k = bitrev_n(slot), natural in, bit-reversed out; C > 1: the four-step split below).
// omega_k = 2 pi fftfreq(k) fs, fp64 (omega^2 delta reaches hundreds of radians).
__global__ void ssfm_htable_kernel(float2* H, SsfmDeltas deltas, int S, int64_t n, int C, double alpha,
                                   double beta2, double fs, int log2L) {
  const int64_t total = (int64_t)S * n;
  const int64_t L = n / C;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / n);
    const int64_t j = i % n;
    const int64_t rank = j / L, slot = j % L;
    const int64_t k = rank + C * (int64_t)(log2L > 0 ? (__brev((unsigned)slot) >> (32 - log2L)) : 0);
    const double f = (k < (n + 1) / 2 ? (double)k : (double)(k - n)) / (double)n * fs;  // fftfreq
    const double w = 2.0 * 3.14159265358979323846 * f;
    const double d = deltas.d[s];
    const double ph = 0.5 * beta2 * w * w * d;
    double sn, cs;
    sincos(ph, &sn, &cs);
    const double g = exp(-0.5 * alpha * d);
    H[i] = make_float2((float)(g * cs), (float)(g * sn));
  }
}

__device__ __forceinline__ unsigned ssfm_bitrev(unsigned i, int bits) { return __brev(i) >> (32 - bits); }
__device__ __forceinline__ int ssfm_pidx(int i) { return i + (i >> 4); }  // padded smem index
__device__ __forceinline__ float2 cmulf(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }

// One pass of RB radix-2 stages on groups of G = 2^RB elements held in registers.  The pass
// consumes bits [c, c+RB) of the transform: group spacing d = n / 2^(c+RB), block 2h = n / 2^c.
// Twiddles: stage m (span 2^m d) of element offset q' < 2^m uses exp(-2 pi j (q' d + r) / (2^(m+1) d));
// the largest-span ones come from the table, the others by squaring.
// FORWARD = decimation in frequency: (a, b) -> (a + b, (a - b) w), stages m = RB-1 .. 0.
// inverse = decimation in time, conjugate twiddles: (a, b) -> (a + b conj(w), a - b conj(w)), m = 0 .. RB-1.
template <int RB, bool FORWARD>
__device__ __forceinline__ void ssfm_pass(float2* X, const float2* tw, int n, int c) {
  constexpr int G = 1 << RB;
  const int d = n >> (c + RB);
  const int groups = n >> RB;
  for (int g = threadIdx.x; g < groups; g += kSsfmThreads) {
    const int blk = g / d, r = g - blk * d;
    const int base = blk * (d << RB) + r;
    float2 v[G];
#pragma unroll
    for (int q = 0; q < G; ++q) v[q] = X[ssfm_pidx(base + q * d)];
    // twiddles: w[m][q'] for q' < 2^m
    float2 w[RB][G / 2];
    const int tstep = n >> (c + RB);  // table index of (q' d + r) / (2^RB d): (q' d + r) * n / (2^RB d) = (q' d + r) * 2^c
    (void)tstep;
#pragma unroll
    for (int q = 0; q < G / 2; ++q) w[RB - 1][q] = tw[(q * d + r) << c];
#pragma unroll
    for (int m = RB - 2; m >= 0; --m)
#pragma unroll
      for (int q = 0; q < (1 << m); ++q) w[m][q] = cmulf(w[m + 1][q], w[m + 1][q]);
    if constexpr (FORWARD) {
#pragma unroll
      for (int m = RB - 1; m >= 0; --m) {
        const int span = 1 << m;
#pragma unroll
        for (int q = 0; q < G; ++q) {
          if (q & span) continue;
          const float2 a = v[q], b = v[q + span];
          v[q] = make_float2(a.x + b.x, a.y + b.y);
          v[q + span] = cmulf(make_float2(a.x - b.x, a.y - b.y), w[m][q & (span - 1)]);
        }
      }
    } else {
#pragma unroll
      for (int m = 0; m < RB; ++m) {
        const int span = 1 << m;
#pragma unroll
        for (int q = 0; q < G; ++q) {
          if (q & span) continue;
          const float2 wc = make_float2(w[m][q & (span - 1)].x, -w[m][q & (span - 1)].y);
          const float2 a = v[q], b = cmulf(v[q + span], wc);
          v[q] = make_float2(a.x + b.x, a.y + b.y);
          v[q + span] = make_float2(a.x - b.x, a.y - b.y);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < G; ++q) X[ssfm_pidx(base + q * d)] = v[q];
  }
  __syncthreads();
}

// Forward DFT (natural order in, bit-reversed out) and the inverse DFT (bit-reversed in, natural
// out, unscaled) of X[0..n) (padded layout), passes of 4 bits and one remainder pass.
template <bool FORWARD>
__device__ __forceinline__ void ssfm_fft(float2* X, const float2* tw, int n, int log2n) {
  const int full = log2n / 4, rem = log2n % 4;
  if constexpr (FORWARD) {
    for (int p = 0; p < full; ++p) ssfm_pass<4, true>(X, tw, n, 4 * p);
    if (rem == 3) ssfm_pass<3, true>(X, tw, n, 4 * full);
    if (rem == 2) ssfm_pass<2, true>(X, tw, n, 4 * full);
    if (rem == 1) ssfm_pass<1, true>(X, tw, n, 4 * full);
  } else {
    if (rem == 3) ssfm_pass<3, false>(X, tw, n, 4 * full);
    if (rem == 2) ssfm_pass<2, false>(X, tw, n, 4 * full);
    if (rem == 1) ssfm_pass<1, false>(X, tw, n, 4 * full);
    for (int p = full - 1; p >= 0; --p) ssfm_pass<4, false>(X, tw, n, 4 * p);
  }
}

// Cluster split of a block of n = C L samples (C = 1, 2, 4; CTA `rank` of the cluster holds
// x[rank L + i], i < L, in its shared memory).  Forward DFT (four-step, P = C):
//   y_k1[i] = W_n^{i k1} sum_r x[r L + i] W_C^{r k1}          (CTA k1: reads the other ranks' x
//                                                              through distributed shared memory)
//   X[k1 + C k2] = sum_i y_k1[i] W_L^{i k2}                   (local L-point DIF, bit-reversed k2)
// Inverse: the local L-point DIT (natural out) then x[r L + i] = sum_k1 W_C^{-r k1} W_n^{-i k1} y'_k1[i].
// W_n^m (m < n) = ta[m >> 6] * tb[m & 63] from two small fp64-accurate tables.
template <int C>
__device__ __forceinline__ float2 ssfm_wC(int e) {  // W_C^e = e^{-2 pi j e / C}
  e &= C - 1;
  if (C == 2) return e ? make_float2(-1.f, 0.f) : make_float2(1.f, 0.f);
  const float2 t[4] = {make_float2(1.f, 0.f), make_float2(0.f, -1.f), make_float2(-1.f, 0.f), make_float2(0.f, 1.f)};
  return t[e];
}

template <int C, bool FORWARD>
__device__ __forceinline__ void ssfm_cross(float2* X, const float2* ta, const float2* tb, int L, int rank) {
  if constexpr (C > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    constexpr int PER = (1 << kSsfmLocalMaxLog2) / kSsfmThreads;
    float2 acc[PER];
    cl.sync();  // every rank's X is final
    const float2* Xr[C];
#pragma unroll
    for (int q = 0; q < C; ++q) Xr[q] = cl.map_shared_rank(X, q);
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int i = threadIdx.x + t * kSsfmThreads;
      float2 y = make_float2(0.f, 0.f);
      if (i < L) {
        const int pi = ssfm_pidx(i);
        if constexpr (FORWARD) {
#pragma unroll
          for (int q = 0; q < C; ++q) {
            const float2 v = cmulf(Xr[q][pi], ssfm_wC<C>(q * rank));
            y.x += v.x;
            y.y += v.y;
          }
          const int m = i * rank;
          y = cmulf(y, cmulf(ta[m >> 6], tb[m & 63]));
        } else {
#pragma unroll
          for (int q = 0; q < C; ++q) {
            const int m = i * q;
            float2 w = cmulf(ta[m >> 6], tb[m & 63]);
            w = cmulf(w, ssfm_wC<C>(q * rank));
            w.y = -w.y;  // conj(W_n^{i q} W_C^{q rank})
            const float2 v = cmulf(Xr[q][pi], w);
            y.x += v.x;
            y.y += v.y;
          }
        }
      }
      acc[t] = y;
    }
    cl.sync();  // every rank has read
#pragma unroll
    for (int t = 0; t < PER; ++t) {
      const int i = threadIdx.x + t * kSsfmThreads;
      if (i < L) X[ssfm_pidx(i)] = acc[t];
    }
    __syncthreads();
  }
}

template <int C>
__global__ void __launch_bounds__(kSsfmThreads, 1) ssfm_link_kernel(const SsfmArgs a) {
  extern __shared__ __align__(16) unsigned char ss_smem[];
  const int n = (int)a.n;
  const int L = n / C;
  float2* X = reinterpret_cast<float2*>(ss_smem);  // [L + L/16] padded
  float2* tw = X + L + L / 16 + 1;                 // [L/2]   W_L^k
  float2* ta = tw + L / 2;                         // [n/64]  W_n^{64 a}  (C > 1)
  float2* tb = ta + (C > 1 ? n / 64 : 0);          // [64]    W_n^{b}
  int rank = 0;
  if constexpr (C > 1) rank = (int)cooperative_groups::this_cluster().block_rank();
  const int b = blockIdx.x / C;
  float2* ub = a.u + (int64_t)b * n + (int64_t)rank * L;
  for (int k = threadIdx.x; k < L / 2; k += kSsfmThreads) {
    double sn, cs;
    sincospi(-2.0 * (double)k / (double)L, &sn, &cs);
    tw[k] = make_float2((float)cs, (float)sn);
  }
  if constexpr (C > 1) {
    for (int k = threadIdx.x; k < n / 64 + 64; k += kSsfmThreads) {
      const int m = k < n / 64 ? 64 * k : k - n / 64;
      double sn, cs;
      sincospi(-2.0 * (double)m / (double)n, &sn, &cs);
      (k < n / 64 ? ta[k] : tb[k - n / 64]) = make_float2((float)cs, (float)sn);
    }
  }
  for (int i = threadIdx.x; i < L; i += kSsfmThreads) X[ssfm_pidx(i)] = ub[i];
  __syncthreads();
  const float inv_n = 1.f / (float)n;
  for (int sp = 0; sp < a.spans; ++sp) {
    for (int s = 0; s < a.S; ++s) {
      const float kp = a.kerr_phase[s];
      for (int i = threadIdx.x; i < L; i += kSsfmThreads) {  // Kerr step (L_eff), pointwise
        const int pi = ssfm_pidx(i);
        const float2 v = X[pi];
        float sn, cs;
        sincosf(kp * (v.x * v.x + v.y * v.y), &sn, &cs);
        X[pi] = make_float2(v.x * cs - v.y * sn, v.x * sn + v.y * cs);
      }
      __syncthreads();
      ssfm_cross<C, true>(X, ta, tb, L, rank);
      ssfm_fft<true>(X, tw, L, a.log2L);
      const float2* Hs = a.H + (int64_t)s * n + (int64_t)rank * L;
      for (int k = threadIdx.x; k < L; k += kSsfmThreads) {  // lossy dispersion (and 1/n), bit-reversed slots
        const int pk_ = ssfm_pidx(k);
        const float2 h = Hs[k], v = X[pk_];
        X[pk_] = make_float2((v.x * h.x - v.y * h.y) * inv_n, (v.x * h.y + v.y * h.x) * inv_n);
      }
      __syncthreads();
      ssfm_fft<false>(X, tw, L, a.log2L);
      ssfm_cross<C, false>(X, ta, tb, L, rank);
    }
    // EDFA: gain + ASE
    const float2* nz = a.ase_mode == 1 ? a.noise + ((int64_t)sp * (gridDim.x / C) + b) * n + (int64_t)rank * L : nullptr;
    for (int i = threadIdx.x; i < L; i += kSsfmThreads) {
      float2 v = X[ssfm_pidx(i)];
      v.x *= a.span_gain;
      v.y *= a.span_gain;
      if (a.ase_mode) {
        const float2 z = a.ase_mode == 1 ? nz[i] : ase_philox_cn(a.ase_seed, a.block0 + b, sp, (int64_t)rank * L + i);
        v.x = fmaf(a.ase_sigma, z.x, v.x);
        v.y = fmaf(a.ase_sigma, z.y, v.y);
      }
      X[ssfm_pidx(i)] = v;
    }
    __syncthreads();
  }
  if (a.decim <= 0) {
    for (int i = threadIdx.x; i < L; i += kSsfmThreads) ub[i] = X[ssfm_pidx(i)];
    return;
  }
  // receiver front end: brick-wall LPF |fftfreq| <= cutoff, then every decim-th sample
  ssfm_cross<C, true>(X, ta, tb, L, rank);
  ssfm_fft<true>(X, tw, L, a.log2L);
  for (int i = threadIdx.x; i < L; i += kSsfmThreads) {  // slot i holds bin rank + C bitrev_L(i)
    const int k = rank + C * (int)(a.log2L > 0 ? ssfm_bitrev((unsigned)i, a.log2L) : 0);
    const float f = (float)(k < (n + 1) / 2 ? k : k - n) / (float)n;
    const int pi = ssfm_pidx(i);
    const float2 v = X[pi];
    X[pi] = fabsf(f) <= a.cutoff ? make_float2(v.x * inv_n, v.y * inv_n) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  ssfm_fft<false>(X, tw, L, a.log2L);
  ssfm_cross<C, false>(X, ta, tb, L, rank);
  float2* rb = a.r + (int64_t)b * (n / a.decim) + (int64_t)rank * (L / a.decim);
  for (int i = threadIdx.x; i < L / a.decim; i += kSsfmThreads) rb[i] = X[ssfm_pidx(i * a.decim)];
}

}  // namespace ldbp

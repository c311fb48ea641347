// ldbp_ssfm.cuh — GPU split-step Fourier channel generator, sm_100a.
//
// The link of §IV-A as the oracle simulates it (oracle/channel.py): per span, for
// each log-distributed step delta: Kerr step u <- u e^{j gamma L_eff(delta) |u|^2}
// at the segment start (reading G5), then the lossy linear step U_k <- U_k e^{-alpha delta/2}
// e^{j beta2/2 omega_k^2 delta} (Eqs. (4)-(6)); after the span the EDFA: gain
// e^{alpha L_sp/2} plus ASE sigma * CN(0,1) (the draws are inputs); at the end an
// ideal low-pass |f| <= cutoff and decimation (reading G8).
//
// One persistent CTA per block: the block (n <= 2^14 complex fp32) stays in shared memory for the
// whole link; FFTs are in-place radix-2 decimation-in-time (bit-reversal permutation, log2 n
// butterfly stages, twiddles e^{-2 pi j k / n} from an fp64-accurate table in shared memory).
// The dispersion factors H_s[k] (one row per distinct step length) are precomputed in fp64 by
// ssfm_htable_kernel: omega^2 delta reaches hundreds of radians, beyond fp32 sincos accuracy.
#pragma once

namespace ldbp {

constexpr int kSsfmThreads = 1024;
constexpr int kSsfmMaxLog2 = 14;

struct SsfmArgs {
  float2* u;               // [B][n] in: transmitted waveform; out (decim == 0): channel output
  float2* r;               // [B][n / decim] out when decim > 0 (LPF + decimation)
  const float2* H;         // [S][n] dispersion factors of the S step lengths of one span
  const float2* noise;     // [spans][B][n] CN(0,1) ASE draws, or nullptr (noiseless)
  const float* kerr_phase; // [S] gamma * L_eff(delta_s) (1/W)
  int64_t n;
  int log2n, spans, S, decim;
  float span_gain;         // e^{alpha L_sp / 2}
  float ase_sigma;         // sqrt(PSD * f_sim)
  float cutoff;            // pass |fftfreq| <= cutoff (cycles/sample)
};

// H[s][k] = e^{-alpha delta_s/2} e^{j beta2/2 omega_k^2 delta_s}, omega_k = 2 pi fftfreq(k) fs (fp64)
// Stored in bit-reversed bin order (slot bitrev(k)): the forward FFT is decimation-in-frequency
// (natural in, bit-reversed out), so the dispersion multiply needs no permutation.
__global__ void ssfm_htable_kernel(float2* H, const double* deltas, int S, int64_t n, double alpha, double beta2,
                                   double fs, int log2n) {
  const int64_t total = (int64_t)S * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / n);
    const int64_t k = i % n;
    const double f = (k < (n + 1) / 2 ? (double)k : (double)(k - n)) / (double)n * fs;  // fftfreq
    const double w = 2.0 * 3.14159265358979323846 * f;
    const double d = deltas[s];
    const double ph = 0.5 * beta2 * w * w * d;
    double sn, cs;
    sincos(ph, &sn, &cs);
    const double g = exp(-0.5 * alpha * d);
    H[(int64_t)s * n + (__brev((unsigned)k) >> (32 - log2n))] = make_float2((float)(g * cs), (float)(g * sn));
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

__global__ void __launch_bounds__(kSsfmThreads) ssfm_link_kernel(const SsfmArgs a) {
  extern __shared__ __align__(16) unsigned char ss_smem[];
  const int n = (int)a.n;
  float2* X = reinterpret_cast<float2*>(ss_smem);  // [n + n/16] padded
  float2* tw = X + n + n / 16 + 1;                 // [n/2]
  const int b = blockIdx.x;
  float2* ub = a.u + (int64_t)b * n;
  for (int k = threadIdx.x; k < n / 2; k += kSsfmThreads) {
    double sn, cs;
    sincospi(-2.0 * (double)k / (double)n, &sn, &cs);
    tw[k] = make_float2((float)cs, (float)sn);
  }
  for (int i = threadIdx.x; i < n; i += kSsfmThreads) X[ssfm_pidx(i)] = ub[i];
  __syncthreads();
  const float inv_n = 1.f / (float)n;
  for (int sp = 0; sp < a.spans; ++sp) {
    for (int s = 0; s < a.S; ++s) {
      const float kp = a.kerr_phase[s];
      for (int i = threadIdx.x; i < n; i += kSsfmThreads) {  // Kerr step (L_eff), pointwise
        const int pi = ssfm_pidx(i);
        const float2 v = X[pi];
        float sn, cs;
        sincosf(kp * (v.x * v.x + v.y * v.y), &sn, &cs);
        X[pi] = make_float2(v.x * cs - v.y * sn, v.x * sn + v.y * cs);
      }
      __syncthreads();
      ssfm_fft<true>(X, tw, n, a.log2n);
      const float2* Hs = a.H + (int64_t)s * n;
      for (int k = threadIdx.x; k < n; k += kSsfmThreads) {  // lossy dispersion (and 1/n), bit-reversed slots
        const int pk_ = ssfm_pidx(k);
        const float2 h = Hs[k], v = X[pk_];
        X[pk_] = make_float2((v.x * h.x - v.y * h.y) * inv_n, (v.x * h.y + v.y * h.x) * inv_n);
      }
      __syncthreads();
      ssfm_fft<false>(X, tw, n, a.log2n);
    }
    // EDFA: gain + ASE
    const float2* nz = a.noise ? a.noise + ((int64_t)sp * gridDim.x + b) * n : nullptr;
    for (int i = threadIdx.x; i < n; i += kSsfmThreads) {
      float2 v = X[ssfm_pidx(i)];
      v.x *= a.span_gain;
      v.y *= a.span_gain;
      if (nz) {
        const float2 z = nz[i];
        v.x = fmaf(a.ase_sigma, z.x, v.x);
        v.y = fmaf(a.ase_sigma, z.y, v.y);
      }
      X[ssfm_pidx(i)] = v;
    }
    __syncthreads();
  }
  if (a.decim <= 0) {
    for (int i = threadIdx.x; i < n; i += kSsfmThreads) ub[i] = X[ssfm_pidx(i)];
    return;
  }
  // receiver front end: brick-wall LPF |fftfreq| <= cutoff, then every decim-th sample
  ssfm_fft<true>(X, tw, n, a.log2n);
  for (int i = threadIdx.x; i < n; i += kSsfmThreads) {  // slot i holds bin bitrev(i)
    const int k = (int)ssfm_bitrev((unsigned)i, a.log2n);
    const float f = (float)(k < (n + 1) / 2 ? k : k - n) / (float)n;
    const int pi = ssfm_pidx(i);
    const float2 v = X[pi];
    X[pi] = fabsf(f) <= a.cutoff ? make_float2(v.x * inv_n, v.y * inv_n) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  ssfm_fft<false>(X, tw, n, a.log2n);
  float2* rb = a.r + (int64_t)b * (n / a.decim);
  for (int i = threadIdx.x; i < n / a.decim; i += kSsfmThreads) rb[i] = X[ssfm_pidx(i * a.decim)];
}

}  // namespace ldbp

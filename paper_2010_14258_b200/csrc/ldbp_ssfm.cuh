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
__global__ void ssfm_htable_kernel(float2* H, const double* deltas, int S, int64_t n, double alpha, double beta2,
                                   double fs) {
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
    H[i] = make_float2((float)(g * cs), (float)(g * sn));
  }
}

__device__ __forceinline__ unsigned ssfm_bitrev(unsigned i, int bits) { return __brev(i) >> (32 - bits); }

// In-place radix-2 DIT FFT of X[0..n) in shared memory; inverse: conjugate twiddles (unscaled).
__device__ __forceinline__ void ssfm_fft(float2* X, const float2* tw, int n, int log2n, bool inverse) {
  for (int i = threadIdx.x; i < n; i += kSsfmThreads) {
    const int j = (int)ssfm_bitrev((unsigned)i, log2n);
    if (j > i) {
      const float2 t = X[i];
      X[i] = X[j];
      X[j] = t;
    }
  }
  __syncthreads();
  for (int s = 1; s <= log2n; ++s) {
    const int half = 1 << (s - 1);
    const int tstride = n >> s;  // twiddle index step: e^{-2 pi j pos / (2 half)} = tw[pos * n / (2 half)]
    for (int bfly = threadIdx.x; bfly < n / 2; bfly += kSsfmThreads) {
      const int pos = bfly & (half - 1);
      const int i = ((bfly >> (s - 1)) << s) + pos;
      const int j = i + half;
      float2 w = tw[pos * tstride];
      if (inverse) w.y = -w.y;
      const float2 xi = X[i], xj = X[j];
      const float tr = w.x * xj.x - w.y * xj.y, ti = w.x * xj.y + w.y * xj.x;
      X[i] = make_float2(xi.x + tr, xi.y + ti);
      X[j] = make_float2(xi.x - tr, xi.y - ti);
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(kSsfmThreads) ssfm_link_kernel(const SsfmArgs a) {
  extern __shared__ __align__(16) unsigned char ss_smem[];
  const int n = (int)a.n;
  float2* X = reinterpret_cast<float2*>(ss_smem);  // [n]
  float2* tw = X + n;                              // [n/2]
  const int b = blockIdx.x;
  float2* ub = a.u + (int64_t)b * n;
  for (int k = threadIdx.x; k < n / 2; k += kSsfmThreads) {
    double sn, cs;
    sincospi(-2.0 * (double)k / (double)n, &sn, &cs);
    tw[k] = make_float2((float)cs, (float)sn);
  }
  for (int i = threadIdx.x; i < n; i += kSsfmThreads) X[i] = ub[i];
  __syncthreads();
  const float inv_n = 1.f / (float)n;
  for (int sp = 0; sp < a.spans; ++sp) {
    for (int s = 0; s < a.S; ++s) {
      const float kp = a.kerr_phase[s];
      for (int i = threadIdx.x; i < n; i += kSsfmThreads) {  // Kerr step (L_eff), pointwise
        const float2 v = X[i];
        float sn, cs;
        sincosf(kp * (v.x * v.x + v.y * v.y), &sn, &cs);
        X[i] = make_float2(v.x * cs - v.y * sn, v.x * sn + v.y * cs);
      }
      __syncthreads();
      ssfm_fft(X, tw, n, a.log2n, false);
      const float2* Hs = a.H + (int64_t)s * n;
      for (int k = threadIdx.x; k < n; k += kSsfmThreads) {  // lossy dispersion (and 1/n)
        const float2 h = Hs[k], v = X[k];
        X[k] = make_float2((v.x * h.x - v.y * h.y) * inv_n, (v.x * h.y + v.y * h.x) * inv_n);
      }
      __syncthreads();
      ssfm_fft(X, tw, n, a.log2n, true);
    }
    // EDFA: gain + ASE
    const float2* nz = a.noise ? a.noise + ((int64_t)sp * gridDim.x + b) * n : nullptr;
    for (int i = threadIdx.x; i < n; i += kSsfmThreads) {
      float2 v = X[i];
      v.x *= a.span_gain;
      v.y *= a.span_gain;
      if (nz) {
        const float2 z = nz[i];
        v.x = fmaf(a.ase_sigma, z.x, v.x);
        v.y = fmaf(a.ase_sigma, z.y, v.y);
      }
      X[i] = v;
    }
    __syncthreads();
  }
  if (a.decim <= 0) {
    for (int i = threadIdx.x; i < n; i += kSsfmThreads) ub[i] = X[i];
    return;
  }
  // receiver front end: brick-wall LPF |fftfreq| <= cutoff, then every decim-th sample
  ssfm_fft(X, tw, n, a.log2n, false);
  for (int k = threadIdx.x; k < n; k += kSsfmThreads) {
    const float f = (float)(k < (n + 1) / 2 ? k : k - n) / (float)n;
    const float2 v = X[k];
    X[k] = fabsf(f) <= a.cutoff ? make_float2(v.x * inv_n, v.y * inv_n) : make_float2(0.f, 0.f);
  }
  __syncthreads();
  ssfm_fft(X, tw, n, a.log2n, true);
  float2* rb = a.r + (int64_t)b * (n / a.decim);
  for (int i = threadIdx.x; i < n / a.decim; i += kSsfmThreads) rb[i] = X[i * a.decim];
}

}  // namespace ldbp

// ldbp_rx.cuh — receiver-chain symbol loss after LDBP, sm_100a.
//
// s_hat = e^{-j phi} M y / sqrt(P)   (Eq. (12); genie phase phi = arg(s^H M y),
//                                     P:772-775; reading G10: divide by sqrt(P))
// errs_b = sum_k |s_hat_k - s_k|^2   (symbol error energy of block b; the paper's symbol MSE,
//                                     P:812-816, is errs / #symbols)
// M (reading G19): decimating circular FIR with real even taps h[m], m in [-L, L]
// (the periodic RRC impulse response truncated; the oracle uses the same definition):
//     s_tilde_k = sum_m h[m] y_{(k*sps - m) mod n}.
//
// Polyphase form: with m = sps*p + c (c in [0, sps)), y_{k*sps - m} = Y_c[k - p] where
// Y_c[i] = y_{(sps*i - c) mod n}, so every phase is a plain FIR at the symbol rate; the adjoint
// (M^T g)_{sps*i - c} = sum_p h[sps*p + c] g_{i+p} is the matching correlation.
//
// Gradient (exact chain rule, oracle rx_loss_grad): with z = s^H s_tilde, a = e^{-j phi}/sqrt(P),
// e = a s_tilde - s:  g_s_tilde = 2 conj(a) e + (dL/dphi) j s / conj(z),  dL/dphi = -2 Im(a z)
// (= 0 up to rounding: the genie phase is the minimiser), then g_y = M^T g_s_tilde.
//
// Kernel 1 (rx_mf_kernel): grid (chunks, B); a CTA stages its chunk's Y_c windows in shared
// memory, each thread computes RQ consecutive symbols by sliding a register window over the
// taps (one LDS + RQ packed FFMA2 per tap and phase), stores s_tilde and per-CTA fp64 partial
// sums [sum|st|^2, Re z, Im z, sum|s|^2].
// Kernel 2 (rx_grad_kernel): grid (chunks, B); the prologue reduces block b's partials in fixed
// order (deterministic), every CTA forms g_s_tilde for its window and runs the adjoint
// correlation the same way; CTA 0 of each block writes errs_b.
#pragma once

namespace ldbp {

constexpr int kRxThreads = 128;
constexpr int kRxQ = 16;                          // symbols (kernel 1) / outputs (kernel 2) per thread
constexpr int kRxChunk = kRxThreads * kRxQ;       // symbols per CTA
constexpr int kRxMaxL = 256;                      // max half-length of the MF (samples)
constexpr int kRxMaxSps = 4;
// bytes of the tap-table region: sps * roundup(2P-1, 8) floats, P <= kRxMaxL + 1
constexpr int kRxTapBytes = ((kRxMaxSps * ((2 * (kRxMaxL + 1) - 1 + 7) / 8) * 8 * 4 + 15) / 16) * 16;

struct RxArgs {
  const float2* y;        // [B][n] LDBP output (original scale)
  const float2* sym;      // [B][K] transmitted symbols, K = n / sps
  const float* power_w;   // [B]
  const float* h;         // [2L+1] real MF taps, h[m + L]
  float2* st;             // [B][K] workspace: s_tilde
  double* part;           // [B][chunks][4] workspace: partial sums
  double* epart;          // [B][chunks] workspace: partial symbol error energies
  float2* gy;             // [B][n] out: dL/dy
  double* errs;           // [B] out
  int64_t n;
  int K, sps, L, chunks;
};

__device__ __forceinline__ int64_t rx_mod(int64_t i, int64_t n) {
  i %= n;
  return i < 0 ? i + n : i;
}

constexpr int kRxTB = 8;  // taps per unrolled block

// Per-phase tap tables in shared memory: tt[c][j], j in [0, NJ): tap of p' = P-1-j, zero-padded
// to NJ = roundup(2P-1, kRxTB).  dir = +1: h[sps*p' + c] (matched filter), -1: h[-sps*p' + c]
// (adjoint).  Every tap index is then in range and every block is a whole kRxTB.
__device__ __forceinline__ int rx_nj(int P) { return ((2 * P - 1 + kRxTB - 1) / kRxTB) * kRxTB; }
__device__ __forceinline__ void rx_tap_tables(const float* __restrict__ h, int L, int sps, int P, int dir, float* tt) {
  const int NJ = rx_nj(P);
  for (int i = threadIdx.x; i < sps * NJ; i += kRxThreads) {
    const int c = i / NJ, j = i % NJ;
    const int pp = P - 1 - j;
    const int m = dir * sps * pp + c;
    tt[i] = (j < 2 * P - 1 && m >= -L && m <= L) ? h[m + L] : 0.f;
  }
}

// Staged symbol windows use a padded layout: element i at pidx(i) = i + i/16, so the 32 lanes
// (16 contiguous symbols each, i.e. 16 elements apart) are 17 elements apart: conflict-free LDS.64.
__device__ __forceinline__ int rx_pidx(int i) { return i + (i >> 4); }
__device__ __forceinline__ int rx_wnp(int wn) { return wn + (wn >> 4) + 1; }

// acc[q] += sum_j tt[j] X[x0 + q + j - (P-1)]  (X padded, indexed in symbols; taps p' = P-1-j
// descending), blocks of kRxTB taps with compile-time register indices (window reloaded per block).
__device__ __forceinline__ void rx_poly_fir(const f2x* __restrict__ X, int x0, const float* __restrict__ tt, int P,
                                            f2x (&acc)[kRxQ]) {
  const int NJ = rx_nj(P);
  for (int j0 = 0; j0 < NJ; j0 += kRxTB) {
    const int s0 = x0 + j0 - (P - 1);
    f2x w[kRxQ + kRxTB - 1];
#pragma unroll
    for (int i = 0; i < kRxQ + kRxTB - 1; ++i) w[i] = X[rx_pidx(s0 + i)];
#pragma unroll
    for (int t = 0; t < kRxTB; ++t) {
      const f2x hb = bcast(tt[j0 + t]);
#pragma unroll
      for (int q = 0; q < kRxQ; ++q) acc[q] = fma2(hb, w[q + t], acc[q]);
    }
  }
}

// Kernel 1: matched filter + downsample + partial sums.
__global__ void __launch_bounds__(kRxThreads) rx_mf_kernel(const RxArgs a) {
  extern __shared__ __align__(16) unsigned char rx_smem[];
  const int b = blockIdx.y, chunk = blockIdx.x;
  const int tid = threadIdx.x;
  const int k0 = chunk * kRxChunk;                      // first symbol of the chunk
  const int nk = min(kRxChunk, a.K - k0);
  const int P = (a.L + a.sps - 1) / a.sps + 1;          // taps per phase: p in [-P+1 .. P-1] covers |m| <= L
  const int WL = P + kRxTB;  // window margin (symbols) per side: taps |p'| < P plus the padded tap block
  const int WN = kRxChunk + 2 * WL;                     // staged symbols per phase
  float* tt = reinterpret_cast<float*>(rx_smem);        // [sps][NJ] tap tables
  f2x* Y = reinterpret_cast<f2x*>(rx_smem + kRxTapBytes);  // [sps][WN]
  rx_tap_tables(a.h, a.L, a.sps, P, +1, tt);
  const f2x* y = reinterpret_cast<const f2x*>(a.y) + (int64_t)b * a.n;
  const int WNP = rx_wnp(WN);
  for (int c = 0; c < a.sps; ++c)
    for (int w = tid; w < WN; w += kRxThreads) {
      const int64_t i = (int64_t)k0 - WL + w;  // symbol index of Y_c[i]
      Y[c * WNP + rx_pidx(w)] = y[rx_mod(i * a.sps - c, a.n)];
    }
  __syncthreads();
  // thread symbols k = k0 + tid*RQ + q; s_tilde_k = sum_c sum_p h[sps*p + c] Y_c[k - p]
  f2x acc[kRxQ];
#pragma unroll
  for (int q = 0; q < kRxQ; ++q) acc[q] = 0ull;
  const int kt = tid * kRxQ;  // local symbol offset of this thread
  const int NJ = rx_nj(P);
  for (int c = 0; c < a.sps; ++c)  // Yc[j] = Y_c[k0 + kt + j]; term Y_c[k - p'] = Yc[q - p']
    rx_poly_fir(Y + c * WNP, WL + kt, tt + c * NJ, P, acc);
  // store s_tilde, partial sums over this thread's valid symbols
  const f2x* s = reinterpret_cast<const f2x*>(a.sym) + (int64_t)b * a.K;
  f2x* st = reinterpret_cast<f2x*>(a.st) + (int64_t)b * a.K;
  float s1 = 0.f, zr = 0.f, zi = 0.f, s2 = 0.f;
#pragma unroll
  for (int q = 0; q < kRxQ; ++q) {
    const int kl = kt + q;
    if (kl < nk) {
      const int k = k0 + kl;
      st[k] = acc[q];
      const float2 v = upk(acc[q]), sv = upk(s[k]);
      s1 = fmaf(v.x, v.x, fmaf(v.y, v.y, s1));
      zr = fmaf(sv.x, v.x, fmaf(sv.y, v.y, zr));   // Re(conj(s) st)
      zi = fmaf(sv.x, v.y, fmaf(-sv.y, v.x, zi));  // Im(conj(s) st)
      s2 = fmaf(sv.x, sv.x, fmaf(sv.y, sv.y, s2));
    }
  }
  s1 = warp_sum(s1);
  zr = warp_sum(zr);
  zi = warp_sum(zi);
  s2 = warp_sum(s2);
  __shared__ float red[kRxThreads / 32][4];
  const int lane = tid & 31, warp = tid >> 5;
  if (lane == 0) {
    red[warp][0] = s1;
    red[warp][1] = zr;
    red[warp][2] = zi;
    red[warp][3] = s2;
  }
  __syncthreads();
  if (tid < 4) {
    double t = 0.0;
    for (int w = 0; w < kRxThreads / 32; ++w) t += (double)red[w][tid];
    a.part[((int64_t)b * a.chunks + chunk) * 4 + tid] = t;
  }
}

// Kernel 2: block sums -> phase, errs, g_s_tilde -> adjoint correlation -> g_y.
// CTA (chunk, b) produces g_y at samples t = sps*i - c for symbols i in the chunk, all phases c.
__global__ void __launch_bounds__(kRxThreads) rx_grad_kernel(const RxArgs a) {
  extern __shared__ __align__(16) unsigned char rx_smem[];
  const int b = blockIdx.y, chunk = blockIdx.x;
  const int tid = threadIdx.x;
  const int i0 = chunk * kRxChunk;
  const int ni = min(kRxChunk, a.K - i0);
  const int P = (a.L + a.sps - 1) / a.sps + 1;
  const int WL = P + kRxTB;
  const int WN = kRxChunk + 2 * WL;
  float* tt = reinterpret_cast<float*>(rx_smem);                // [sps][NJ] adjoint tap tables
  f2x* G = reinterpret_cast<f2x*>(rx_smem + kRxTapBytes);      // [WN] g_s_tilde
  __shared__ double bsum[4];
  __shared__ float coef[6];  // a (re, im), conj(a)*2 applied below, dLdphi, 1/conj(z) (re, im)
  rx_tap_tables(a.h, a.L, a.sps, P, -1, tt);
  if (tid < 4) {
    double t = 0.0;
    for (int c = 0; c < a.chunks; ++c) t += a.part[((int64_t)b * a.chunks + c) * 4 + tid];
    bsum[tid] = t;
  }
  __syncthreads();
  if (tid == 0) {
    const double S1 = bsum[0], zr = bsum[1], zi = bsum[2], S2 = bsum[3];
    const double az = sqrt(zr * zr + zi * zi);
    const double pw = (double)a.power_w[b];
    const double sq = sqrt(pw);
    // a = e^{-j phi} / sqrt(P) = conj(z) / (|z| sqrt(P))  (phi = arg z; z = 0 -> phi = 0)
    const double ar = az > 0 ? zr / (az * sq) : 1.0 / sq, ai = az > 0 ? -zi / (az * sq) : 0.0;
    // errs = |a|^2 S1 - 2 Re(a z) + S2
    const double re_az = ar * zr - ai * zi, im_az = ar * zi + ai * zr;
    (void)S1;
    (void)S2;
    const double dldphi = -2.0 * im_az;
    const double zn = zr * zr + zi * zi;
    coef[0] = (float)ar;
    coef[1] = (float)ai;
    coef[2] = (float)dldphi;
    coef[3] = zn > 0 ? (float)(zr / zn) : 0.f;  // 1/conj(z) = z / |z|^2
    coef[4] = zn > 0 ? (float)(zi / zn) : 0.f;
  }
  __syncthreads();
  const float ar = coef[0], ai = coef[1], dldphi = coef[2], izr = coef[3], izi = coef[4];
  float esum = 0.f;  // sum |e|^2 over this chunk's own symbols (window positions [WL, WL + ni))
  // g_s_tilde on the window of symbols [i0 - WL, i0 + kRxChunk + WL) (circular in K)
  const f2x* s = reinterpret_cast<const f2x*>(a.sym) + (int64_t)b * a.K;
  const f2x* st = reinterpret_cast<const f2x*>(a.st) + (int64_t)b * a.K;
  for (int w = tid; w < WN; w += kRxThreads) {
    const int64_t k = rx_mod((int64_t)i0 - WL + w, a.K);
    const int wp = rx_pidx(w);
    const float2 v = upk(st[k]), sv = upk(s[k]);
    // e = a st - s
    const float ex = ar * v.x - ai * v.y - sv.x, ey = ar * v.y + ai * v.x - sv.y;
    if (w >= WL && w < WL + ni) esum = fmaf(ex, ex, fmaf(ey, ey, esum));
    // 2 conj(a) e
    float gx = 2.f * (ar * ex + ai * ey), gyv = 2.f * (ar * ey - ai * ex);
    // + dLdphi * j s / conj(z) = dLdphi * j s * z / |z|^2
    const float tx = sv.x * izr - sv.y * izi, ty = sv.x * izi + sv.y * izr;  // s z/|z|^2
    gx = fmaf(-dldphi, ty, gx);
    gyv = fmaf(dldphi, tx, gyv);
    G[wp] = pk(gx, gyv);
  }
  esum = warp_sum(esum);
  __shared__ float ered[kRxThreads / 32];
  if ((tid & 31) == 0) ered[tid >> 5] = esum;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kRxThreads / 32; ++w) t += (double)ered[w];
    a.epart[(int64_t)b * a.chunks + chunk] = t;
  }
  if (a.gy == nullptr) return;  // loss only
  // g_y[sps*i - c] = sum_p h[sps*p + c] g_{i+p}, thread outputs i = i0 + tid*RQ + q
  f2x* gout = reinterpret_cast<f2x*>(a.gy) + (int64_t)b * a.n;
  const int it = tid * kRxQ;
  const int NJ = rx_nj(P);
  for (int c = 0; c < a.sps; ++c) {
    // Gc[j] = g_{i0 + it + j}; sum_p h[sps p + c] g_{i+p} = sum_{p'} h[-sps p' + c] Gc[q - p']
    f2x acc[kRxQ];
#pragma unroll
    for (int q = 0; q < kRxQ; ++q) acc[q] = 0ull;
    rx_poly_fir(G, WL + it, tt + c * NJ, P, acc);
#pragma unroll
    for (int q = 0; q < kRxQ; ++q) {
      const int il = it + q;
      if (il < ni) gout[rx_mod((int64_t)(i0 + il) * a.sps - c, a.n)] = acc[q];
    }
  }
}

// errs_b = sum over chunks of the partial error energies (fixed order); optionally
// buf[0] = sum_b errs_b (fixed order).  One CTA.
__global__ void __launch_bounds__(256) rx_errs_kernel(const double* epart, int64_t B, int chunks, double* errs,
                                                       double* buf) {
  __shared__ double red[256];
  double t = 0.0;
  for (int64_t b = threadIdx.x; b < B; b += 256) {
    double e = 0.0;
    for (int c = 0; c < chunks; ++c) e += epart[b * chunks + c];
    errs[b] = e;
    t += e;
  }
  red[threadIdx.x] = t;
  __syncthreads();
  if (threadIdx.x == 0 && buf) {
    double s = 0.0;
    for (int i = 0; i < 256; ++i) s += red[i];
    buf[0] = s;
  }
}

}  // namespace ldbp

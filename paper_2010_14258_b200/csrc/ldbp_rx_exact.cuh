// ldbp_rx_exact.cuh — receiver-chain loss with the EXACT circulant matched filter (SURVEY.md §8(f)
// NEXT-1; Eq. (12): "M ... a circulant matrix that represents the matched filter").
//
// The round-1 receiver (ldbp_rx.cuh) applies M as a decimating FIR truncated to +-L samples
// (reading G19); this one applies the circulant itself, in the frequency domain, so the GPU loss
// is Eq. (12)-(13) with no truncation:
//   z = F^-1 diag(RRC) F y           (matched filter on the periodic frame, RRC real and even)
//   s_tilde_k = z[k sps]             (downsampling);  a = e^{-j phi} / sqrt(P_b),
//   phi = arg(s^H s_tilde)           (genie phase);  e = a s_tilde - s
//   errs_b = sum_k |e_k|^2;          L = sum_b w_b errs_b   (optional per-block weights w_b)
//   g_s_tilde = w_b (2 conj(a) e + (dL/dphi) j s / conj(s^H s_tilde)),  dL/dphi = -2 Im(a s^H s_tilde)
//   g_y = M^T g_s_tilde = F^-1 diag(RRC) F U g_s_tilde   (U: upsampling with zeros; M^T = C U
//                                                         because the circulant C is real symmetric)
// One CTA per block of n <= 2^14 samples, a 2- or 4-CTA cluster up to 2^16, reusing the SSFM
// generator's shared-memory FFTs (ldbp_ssfm.cuh: local radix-16 passes + the four-step split over
// distributed shared memory).  fp32 transforms, fp64 reductions in a fixed order (deterministic:
// every CTA of a cluster reads all ranks' partials in rank order).
#pragma once

namespace ldbp {

struct RxExactArgs {
  const float2* y;         // [B][n]
  const float2* sym;       // [B][K]
  const float* power_w;    // [B]
  const float* weights;    // [B] or nullptr (all 1)
  float2* gy;              // [B][n] or nullptr
  double* errs;            // [B] (unweighted)
  int64_t n;
  int K, sps, log2L;
  float rolloff;
};

// RRC(f) with f in cycles/symbol (the oracle's rrc_response): sqrt of the raised cosine.
__device__ __forceinline__ float rx_rrc(int64_t k, int64_t n, int sps, float beta) {
  const float f = fabsf((float)(k < (n + 1) / 2 ? k : k - n) / (float)n * (float)sps);
  const float lo = 0.5f * (1.f - beta), hi = 0.5f * (1.f + beta);
  if (f <= lo) return 1.f;
  if (f > hi) return 0.f;
  return sqrtf(0.5f * (1.f + cospif((f - lo) / beta)));
}

// Block sum of (up to 4) fp64 values per thread, fixed order (warp shuffles, then warps in order).
template <int NV>
__device__ __forceinline__ void rx_block_sum(double (&v)[NV], double* scratch /*[32][NV]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[i] += __shfl_xor_sync(kFull, v[i], o);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < NV; ++i) scratch[warp * NV + i] = v[i];
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += scratch[w * NV + i];
    v[i] = t;
  }
  __syncthreads();
}

// Cluster-wide sum of NV fp64 values (identical result in every rank: ranks summed in order).
template <int C, int NV>
__device__ __forceinline__ void rx_cluster_sum(double (&v)[NV], double* slot /*[NV] in smem*/) {
  if constexpr (C > 1) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    if (threadIdx.x == 0)
#pragma unroll
      for (int i = 0; i < NV; ++i) slot[i] = v[i];
    cl.sync();
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < C; ++q) t += cl.map_shared_rank(slot, q)[i];
      v[i] = t;
    }
    cl.sync();  // slots may be reused
  } else {
    (void)slot;
  }
}

// In place: X <- F^-1 diag(RRC / n) F X (the circulant matched filter C on the distributed block).
template <int C>
__device__ __forceinline__ void rx_circulant(float2* X, const float2* tw, const float2* ta, const float2* tb, int L,
                                             int rank, int64_t n, int log2L, int sps, float beta) {
  ssfm_cross<C, true>(X, ta, tb, L, rank);
  ssfm_fft<true>(X, tw, L, log2L);
  const float inv_n = 1.f / (float)n;
  for (int i = threadIdx.x; i < L; i += kSsfmThreads) {  // slot i holds bin rank + C bitrev_L(i)
    const int64_t k = rank + (int64_t)C * (log2L > 0 ? ssfm_bitrev((unsigned)i, log2L) : 0);
    const float h = rx_rrc(k, n, sps, beta) * inv_n;
    const int pi = ssfm_pidx(i);
    const float2 v = X[pi];
    X[pi] = make_float2(v.x * h, v.y * h);
  }
  __syncthreads();
  ssfm_fft<false>(X, tw, L, log2L);
  ssfm_cross<C, false>(X, ta, tb, L, rank);
}

template <int C>
__global__ void __launch_bounds__(kSsfmThreads, 1) rx_exact_kernel(const RxExactArgs a) {
  extern __shared__ __align__(16) unsigned char rx_smem[];
  const int n = (int)a.n;
  const int L = n / C;
  float2* X = reinterpret_cast<float2*>(rx_smem);
  float2* tw = X + L + L / 16 + 1;
  float2* ta = tw + L / 2;
  float2* tb = ta + (C > 1 ? n / 64 : 0);
  double* scratch = reinterpret_cast<double*>(tb + (C > 1 ? 64 : 0) + 1);  // [32][4] + [4] cluster slot
  double* slot = scratch + 32 * 4;
  int rank = 0;
  if constexpr (C > 1) rank = (int)cooperative_groups::this_cluster().block_rank();
  const int b = blockIdx.x / C;
  const int sps = a.sps;
  const int Kl = L / sps;  // symbols of this rank: k in [rank Kl, rank Kl + Kl)
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
  const float2* yb = a.y + (int64_t)b * n + (int64_t)rank * L;
  for (int i = threadIdx.x; i < L; i += kSsfmThreads) X[ssfm_pidx(i)] = yb[i];
  __syncthreads();
  rx_circulant<C>(X, tw, ta, tb, L, rank, a.n, a.log2L, sps, a.rolloff);
  // genie phase: z = s^H s_tilde (cluster-wide, fp64)
  const float2* sb = a.sym + (int64_t)b * a.K + (int64_t)rank * Kl;
  double zr[2] = {0.0, 0.0};
  for (int k = threadIdx.x; k < Kl; k += kSsfmThreads) {
    const float2 st = X[ssfm_pidx(k * sps)], s = sb[k];
    zr[0] += (double)s.x * st.x + (double)s.y * st.y;  // Re(conj(s) st)
    zr[1] += (double)s.x * st.y - (double)s.y * st.x;  // Im(conj(s) st)
  }
  rx_block_sum<2>(zr, scratch);
  rx_cluster_sum<C, 2>(zr, slot);
  const double P = (double)a.power_w[b];
  const double zabs = sqrt(zr[0] * zr[0] + zr[1] * zr[1]);
  // a = e^{-j phi} / sqrt(P) with e^{-j phi} = conj(z) / |z|
  const double ar = zabs > 0.0 ? zr[0] / (zabs * sqrt(P)) : 1.0 / sqrt(P);
  const double ai = zabs > 0.0 ? -zr[1] / (zabs * sqrt(P)) : 0.0;
  const double dldphi = -2.0 * (ar * zr[1] + ai * zr[0]);  // -2 Im(a z)
  const double w = a.weights ? (double)a.weights[b] : 1.0;
  // errors and g_s_tilde (kept in registers until X is free), errs (fp64)
  constexpr int PER = (1 << kSsfmLocalMaxLog2) / kSsfmThreads;
  float2 g[PER];
  double es[1] = {0.0};
  const double z2 = zr[0] * zr[0] + zr[1] * zr[1];
  // j s / conj(z) = j s z / |z|^2
  const double qr = z2 > 0.0 ? zr[0] / z2 : 0.0, qi = z2 > 0.0 ? zr[1] / z2 : 0.0;
#pragma unroll
  for (int t = 0; t < PER; ++t) {
    const int k = threadIdx.x + t * kSsfmThreads;
    g[t] = make_float2(0.f, 0.f);
    if (k < Kl) {
      const float2 st = X[ssfm_pidx(k * sps)], s = sb[k];
      const double er = ar * st.x - ai * st.y - s.x, ei = ar * st.y + ai * st.x - s.y;
      es[0] += er * er + ei * ei;
      // 2 conj(a) e
      const double gr = 2.0 * (ar * er + ai * ei), gi = 2.0 * (ar * ei - ai * er);
      // dL/dphi * j s z / |z|^2:  s z = (sx zr - sy zi, sx zi + sy zr); j (u + jv) = (-v, u)
      const double szr = s.x * qr - s.y * qi, szi = s.x * qi + s.y * qr;
      g[t] = make_float2((float)(w * (gr - dldphi * szi)), (float)(w * (gi + dldphi * szr)));
    }
  }
  rx_block_sum<1>(es, scratch);
  rx_cluster_sum<C, 1>(es, slot);
  if (rank == 0 && threadIdx.x == 0) a.errs[b] = es[0];
  if (a.gy == nullptr) return;
  // gy = C U g_s_tilde: upsample into X (zeros between symbols), circulant again
  if constexpr (C > 1) cooperative_groups::this_cluster().sync();  // remote reads of X (phase) are done
  for (int i = threadIdx.x; i < L; i += kSsfmThreads) X[ssfm_pidx(i)] = make_float2(0.f, 0.f);
  __syncthreads();
#pragma unroll
  for (int t = 0; t < PER; ++t) {
    const int k = threadIdx.x + t * kSsfmThreads;
    if (k < Kl) X[ssfm_pidx(k * sps)] = g[t];
  }
  __syncthreads();
  rx_circulant<C>(X, tw, ta, tb, L, rank, a.n, a.log2L, sps, a.rolloff);
  float2* gb = a.gy + (int64_t)b * n + (int64_t)rank * L;
  for (int i = threadIdx.x; i < L; i += kSsfmThreads) gb[i] = X[ssfm_pidx(i)];
}

// Transmitted waveform on the device (the training target of the waveform-MSE loss, P:280-290,
// from the transmitted symbols; Eq. (11) on the periodic frame):
//   w = sqrt(P_b) sps e^{j phi_b} F^-1 diag(RRC) F U s_b,  out_b[t] = w[(t - k_b) mod n]
// (U: upsampling by sps with zeros; phi_b, k_b the optional per-block rotation / circular shift
// of the training-set augmentation, exact by equivariance).  Symbols are codes into a small
// constellation table, so a step's targets cross PCIe as 1 byte per symbol instead of 16 bytes
// per symbol of complex64 waveform.  Same shared-memory / cluster FFTs as rx_exact_kernel.
struct TxArgs {
  const uint8_t* codes;     // [B][K] constellation indices
  const float2* constel;    // [Q]
  const float* power_w;     // [B]
  const int32_t* shift;     // [B] or nullptr
  const float* phase;       // [B] or nullptr
  float2* out;              // [B][n]
  int64_t n;
  int K, sps, log2L, Q;
  float rolloff;
};

template <int C>
__global__ void __launch_bounds__(kSsfmThreads, 1) tx_waveform_kernel(const TxArgs a) {
  extern __shared__ __align__(16) unsigned char tx_smem[];
  const int n = (int)a.n;
  const int L = n / C;
  float2* X = reinterpret_cast<float2*>(tx_smem);
  float2* tw = X + L + L / 16 + 1;
  float2* ta = tw + L / 2;
  float2* tb = ta + (C > 1 ? n / 64 : 0);
  int rank = 0;
  if constexpr (C > 1) rank = (int)cooperative_groups::this_cluster().block_rank();
  const int b = blockIdx.x / C;
  const int sps = a.sps;
  const int Kl = L / sps;
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
  // amplitude sqrt(P) sps e^{j phi}, applied to the symbols before the (linear) filter
  double ps = 0.0, pc = 1.0;
  if (a.phase) sincos((double)a.phase[b], &ps, &pc);
  const double amp = sqrt((double)a.power_w[b]) * (double)sps;
  const float2 ap = make_float2((float)(amp * pc), (float)(amp * ps));
  for (int i = threadIdx.x; i < L; i += kSsfmThreads) X[ssfm_pidx(i)] = make_float2(0.f, 0.f);
  __syncthreads();
  const uint8_t* cb = a.codes + (int64_t)b * a.K + (int64_t)rank * Kl;
  for (int k = threadIdx.x; k < Kl; k += kSsfmThreads) {
    const int q = cb[k];
    const float2 s = a.constel[q < a.Q ? q : 0];
    X[ssfm_pidx(k * sps)] = make_float2(ap.x * s.x - ap.y * s.y, ap.x * s.y + ap.y * s.x);
  }
  __syncthreads();
  rx_circulant<C>(X, tw, ta, tb, L, rank, a.n, a.log2L, sps, a.rolloff);
  const int64_t kb = a.shift ? (int64_t)a.shift[b] : 0;
  const int64_t k0 = ((kb % n) + n) % n;
  float2* ob = a.out + (int64_t)b * n;
  for (int i = threadIdx.x; i < L; i += kSsfmThreads) {
    int64_t t = (int64_t)rank * L + i + k0;
    if (t >= n) t -= n;
    ob[t] = X[ssfm_pidx(i)];
  }
}

// buf[0] = sum_b w_b errs_b (fixed order)
__global__ void rx_wsum_kernel(const double* errs, const float* weights, int64_t B, double* buf) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int64_t b = 0; b < B; ++b) t += (weights ? (double)weights[b] : 1.0) * errs[b];
    buf[0] = t;
  }
}

}  // namespace ldbp

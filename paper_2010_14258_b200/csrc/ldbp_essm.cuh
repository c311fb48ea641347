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
constexpr int kEssmW = 1024;      // owned samples per CTA
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

// acc + h*s and acc + conj(h)*s for complex h, s (FFMA2 form, see ldbp_f32x2.cuh)
__device__ __forceinline__ f2x essm_mac(f2x acc, float2 h, f2x s) {
  return fma2(bcast(hif(s)), pk(-h.y, h.x), fma2(bcast(lof(s)), pk(h.x, h.y), acc));
}
__device__ __forceinline__ f2x essm_mac_conj(f2x acc, float2 h, f2x s) {
  return fma2(bcast(hif(s)), pk(h.y, h.x), fma2(bcast(lof(s)), pk(h.x, -h.y), acc));
}

// Forward step: U on [-(Kh+kappa), W+Kh+kappa), A/P on [-kappa, W+kappa), v on [0, W).
template <bool FAST>
__global__ void __launch_bounds__(kEssmThreads) essm_fwd_step_kernel(const EssmArgs a) {
  extern __shared__ __align__(16) unsigned char es_smem[];
  const int kh = (a.T - 1) / 2, kap = a.kappa;
  const float gam = a.gamma[a.step];
  const int b = blockIdx.y, tile = blockIdx.x;
  const int64_t t0 = (int64_t)tile * kEssmW;
  const int hu = kh + kap, nu = kEssmW + 2 * hu, na = kEssmW + 2 * kap;
  float2* sh_h = reinterpret_cast<float2*>(es_smem);       // [kEssmMaxT]
  float* sh_eta = reinterpret_cast<float*>(sh_h + kEssmMaxT);  // [2*kEssmMaxKappa+1]
  f2x* U = reinterpret_cast<f2x*>(sh_eta + 2 * kEssmMaxKappa + 2);  // [nu] (8-byte aligned)
  f2x* A = U + nu;                                           // [na]
  float* P = reinterpret_cast<float*>(A + na);               // [na]
  for (int i = threadIdx.x; i < a.T; i += kEssmThreads) sh_h[i] = a.taps[i];
  for (int i = threadIdx.x; i < 2 * kap + 1; i += kEssmThreads) sh_eta[i] = a.eta[i];
  const f2x* ub = reinterpret_cast<const f2x*>(a.u) + (int64_t)b * a.n;
  for (int i = threadIdx.x; i < nu; i += kEssmThreads) U[i] = ub[essm_mod(t0 - hu + i, a.n)];
  __syncthreads();
  // a_t = sum_j h_j u_{t-j}, t = -kappa + i
  for (int i = threadIdx.x; i < na; i += kEssmThreads) {
    f2x acc = 0ull;
    for (int jj = 0; jj < a.T; ++jj) acc = essm_mac(acc, sh_h[jj], U[i + kh - (jj - kh)]);  // U index of t-j
    A[i] = acc;
    const float2 av = upk(acc);
    P[i] = fmaf(av.x, av.x, av.y * av.y);
  }
  __syncthreads();
  f2x* vb = reinterpret_cast<f2x*>(a.out) + (int64_t)b * a.n;
  for (int i = threadIdx.x; i < kEssmW; i += kEssmThreads) {
    if (t0 + i >= a.n) break;
    float psi = 0.f;
    for (int k = -kap; k <= kap; ++k) psi = fmaf(sh_eta[k + kap], P[i + kap - k], psi);  // p_{t-k}
    float s, c;
    sincos_phase<FAST>(gam * psi, &s, &c);
    const float2 av = upk(A[i + kap]);
    vb[t0 + i] = pk(fmaf(av.x, c, -av.y * s), fmaf(av.x, s, av.y * c));
  }
}

// Backward step.  Regions relative to t0 (halo widths): U: 2Kh+2kappa, A/P: Kh+2kappa,
// G/PSI/C (and phi): Kh+kappa, GA/Q: Kh; outputs and gradient sums on owned [0, W).
template <bool FAST>
__global__ void __launch_bounds__(kEssmThreads) essm_bwd_step_kernel(const EssmArgs a) {
  extern __shared__ __align__(16) unsigned char es_smem[];
  const int kh = (a.T - 1) / 2, kap = a.kappa;
  const float gam = a.gamma[a.step];
  const int b = blockIdx.y, tile = blockIdx.x;
  const int64_t t0 = (int64_t)tile * kEssmW;
  const int own = (int)(a.n - t0 < (int64_t)kEssmW ? a.n - t0 : (int64_t)kEssmW);
  const int hU = 2 * kh + 2 * kap, hA = kh + 2 * kap, hG = kh + kap, hQ = kh;
  const int nU = kEssmW + 2 * hU, nA = kEssmW + 2 * hA, nG = kEssmW + 2 * hG, nQ = kEssmW + 2 * hQ;
  const int NE = 2 * kap + 1;
  const int V = 2 + 2 * a.T + NE;  // [dgamma | loss | dh re/im (T) | deta (NE)]
  float2* sh_h = reinterpret_cast<float2*>(es_smem);
  float* sh_eta = reinterpret_cast<float*>(sh_h + kEssmMaxT);
  f2x* U = reinterpret_cast<f2x*>(sh_eta + 2 * kEssmMaxKappa + 2);
  f2x* A = U + nU;
  f2x* G = A + nA;         // g on hG, later reused for GA on hQ
  float* P = reinterpret_cast<float*>(G + nG);
  float* PSI = P + nA;     // psi on hG
  float* C = PSI + nG;     // c on hG
  float* Q = C + nG;       // q on hQ
  f2x* GA = reinterpret_cast<f2x*>(Q + nQ + (nQ & 1));  // ga on hQ
  double* red = reinterpret_cast<double*>(GA + nQ);     // [kEssmThreads] group sums
  for (int i = threadIdx.x; i < a.T; i += kEssmThreads) sh_h[i] = a.taps[i];
  for (int i = threadIdx.x; i < NE; i += kEssmThreads) sh_eta[i] = a.eta[i];
  const f2x* ub = reinterpret_cast<const f2x*>(a.u) + (int64_t)b * a.n;
  for (int i = threadIdx.x; i < nU; i += kEssmThreads) U[i] = ub[essm_mod(t0 - hU + i, a.n)];
  __syncthreads();
  // a, p on hA
  for (int i = threadIdx.x; i < nA; i += kEssmThreads) {
    f2x acc = 0ull;
    const int iu = i + (hU - hA);  // U index of the same t
    for (int jj = 0; jj < a.T; ++jj) acc = essm_mac(acc, sh_h[jj], U[iu - (jj - kh)]);
    A[i] = acc;
    const float2 av = upk(acc);
    P[i] = fmaf(av.x, av.x, av.y * av.y);
  }
  __syncthreads();
  // psi, v, g (loaded or seeded), c on hG; the seed's loss over owned samples
  const f2x* gb = a.gin ? reinterpret_cast<const f2x*>(a.gin) + (int64_t)b * a.n : nullptr;
  const f2x* tb = a.gin ? nullptr : reinterpret_cast<const f2x*>(a.target) + (int64_t)b * a.n;
  float lsum = 0.f;
  for (int i = threadIdx.x; i < nG; i += kEssmThreads) {
    const int ia = i + (hA - hG);
    float psi = 0.f;
    for (int k = -kap; k <= kap; ++k) psi = fmaf(sh_eta[k + kap], P[ia - k], psi);
    float s, c;
    sincos_phase<FAST>(gam * psi, &s, &c);
    const float2 av = upk(A[ia]);
    const float vx = fmaf(av.x, c, -av.y * s), vy = fmaf(av.x, s, av.y * c);
    const int64_t t = essm_mod(t0 - hG + i, a.n);
    float2 g;
    if (gb) {
      g = upk(gb[t]);
    } else {
      const float2 tv = upk(tb[t]);
      const float ex = vx - tv.x, ey = vy - tv.y;
      g = make_float2(2.f * ex, 2.f * ey);
      if (i >= hG && i < hG + own) lsum = fmaf(ex, ex, fmaf(ey, ey, lsum));
    }
    G[i] = pk(g.x, g.y);
    PSI[i] = psi;
    C[i] = fmaf(g.y, vx, -g.x * vy);  // Im(g conj v)
  }
  __syncthreads();
  // q and ga on hQ
  for (int i = threadIdx.x; i < nQ; i += kEssmThreads) {
    const int ig = i + (hG - hQ), ia = i + (hA - hQ);
    float q = 0.f;
    for (int k = -kap; k <= kap; ++k) q = fmaf(sh_eta[k + kap], C[ig + k], q);  // c_{m+k}
    q *= gam;
    Q[i] = q;
    const float phi = gam * PSI[ig];
    float s, c;
    sincos_phase<FAST>(phi, &s, &c);
    const float2 gv = upk(G[ig]), av = upk(A[ia]);
    // g e^{-j phi} + 2 q a
    GA[i] = pk(fmaf(gv.x, c, fmaf(gv.y, s, 2.f * q * av.x)), fmaf(gv.y, c, fmaf(-gv.x, s, 2.f * q * av.y)));
  }
  __syncthreads();
  // gu on owned
  if (a.out) {
    f2x* ob = reinterpret_cast<f2x*>(a.out) + (int64_t)b * a.n;
    for (int i = threadIdx.x; i < own; i += kEssmThreads) {
      f2x acc = 0ull;
      for (int jj = 0; jj < a.T; ++jj) acc = essm_mac_conj(acc, sh_h[jj], GA[i + hQ + (jj - kh)]);  // ga_{s+j}
      ob[t0 + i] = acc;
    }
  }
  // gradient sums over owned t: component v in [0, V), group r: thread = v * ngroups + r
  const int ngroups = kEssmThreads / V > 0 ? kEssmThreads / V : 1;
  const int comp = threadIdx.x / ngroups, grp = threadIdx.x % ngroups;
  double part = 0.0;
  if (comp < V) {
    float acc = 0.f;
    for (int i = grp; i < own; i += ngroups) {
      const int ig = i + hG, ia = i + hA, iu = i + hU, iq = i + hQ;
      if (comp == 0) {
        acc = fmaf(C[ig], PSI[ig], acc);  // dgamma'
      } else if (comp == 1) {
        acc = 0.f;  // loss handled below
      } else if (comp < 2 + 2 * a.T) {
        const int jj = (comp - 2) >> 1, im = (comp - 2) & 1;
        const float2 g = upk(GA[iq]), w = upk(U[iu - (jj - kh)]);  // ga_t conj(u_{t-j})
        acc += im ? (g.y * w.x - g.x * w.y) : (g.x * w.x + g.y * w.y);
      } else {
        const int k = comp - 2 - 2 * a.T - kap;
        acc = fmaf(C[ig], P[ia - k], acc);  // c_t p_{t-k}
      }
    }
    part = comp >= 2 + 2 * a.T ? (double)gam * acc : (double)acc;
  }
  // loss partial: warp sums into the comp == 1 slot
  lsum = warp_sum(lsum);
  __shared__ float lred[kEssmThreads / 32];
  if ((threadIdx.x & 31) == 0) lred[threadIdx.x >> 5] = lsum;
  red[threadIdx.x] = part;
  __syncthreads();
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  for (int v = threadIdx.x; v < V; v += kEssmThreads) {
    double s = 0.0;
    if (v == 1) {
      for (int w = 0; w < kEssmThreads / 32; ++w) s += (double)lred[w];
    } else {
      for (int r = 0; r < ngroups; ++r) s += red[v * ngroups + r];
    }
    a.partials[(int64_t)cta * V + v] = s;
  }
}

// Fixed-order reduction over CTAs for every step, and the ABI layout:
// buf = [sum |e|^2 | dgamma [M] | dtaps [M][T][2] (SYM: tied +-j) | deta [M][2kappa+1]].
struct EssmReduceArgs {
  const double* partials;  // [M][nblk][V]
  int M, nblk, T, kappa, sym;
  double* buf;
};

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

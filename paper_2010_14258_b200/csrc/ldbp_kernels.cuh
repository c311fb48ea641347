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

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "ldbp_f32x2.cuh"

#ifndef LDBP_FWD_R
#define LDBP_FWD_R 16  // samples per thread, forward kernels
#endif
#ifndef LDBP_BWD_R
#define LDBP_BWD_R 8   // samples per thread, backward kernels
#endif
#ifndef LDBP_BWD_R_SMALL
#define LDBP_BWD_R_SMALL 4  // segment backward for Kh <= 2 (C1 CUDA-graph step 18.5 -> 14.4 us: half the
                            // serial per-thread chain of the latency-bound tiny problems)
#endif
// (wide filters, Kh > 8 / Kh > 12: the neighbour halos need R >= Kh samples per thread)
__host__ __device__ constexpr int bwd_r(int kh) { return kh <= 2 ? LDBP_BWD_R_SMALL : kh <= 8 ? LDBP_BWD_R : 16; }
#ifndef LDBP_REV_R
#define LDBP_REV_R 12  // samples per thread, store-all reverse kernel (measured: 12 >= 16 > 8)
#endif
#ifndef LDBP_REV_R_SMALL
#define LDBP_REV_R_SMALL LDBP_REV_R  // samples per thread of the reverse kernel for Kh <= 1
#endif
__host__ __device__ constexpr int rev_r(int kh) { return kh <= 1 ? LDBP_REV_R_SMALL : kh <= 12 ? LDBP_REV_R : 16; }

#ifndef LDBP_NORM
#define LDBP_NORM 1  // h0-normalised FIR when well conditioned (saves one complex multiply per FIR)
#endif
#ifndef LDBP_BWD_PREFETCH
#define LDBP_BWD_PREFETCH 0  // 1: cp.async-prefetch target/adjoint into smem (costs one tape slot)
#endif
#ifndef LDBP_FWD_XSMEM
#define LDBP_FWD_XSMEM 1  // forward halo exchange through shared memory only (no shuffles)
#endif
#ifndef LDBP_NB_SYNC
#define LDBP_NB_SYNC 0  // 1: neighbour-only mbarrier sync per step (measured 2x slower on B200; kept
                        // as an option), 0: one __syncthreads per step
#endif

namespace ldbp {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kMaxWarps = 32;


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
  int NS;                   // the first NS tiles are half-width (Wh) — see tile_lo()
  int64_t Wh;
};

// Owned range [tile_lo, tile_hi) of CTA b.  The first NS CTAs (one per SM in the first wave)
// get half-width tiles: the CTA that later follows on the same SM slot then runs half a tile
// out of phase with its neighbour slot, so one CTA's load/stage/epilogue latency overlaps the
// other's compute instead of both stalling together (identical CTAs would otherwise stay
// phase-locked for the whole launch).
__device__ __forceinline__ int64_t tile_lo(const Geo& g, int64_t b) {
  return b < g.NS ? b * g.Wh : (int64_t)g.NS * g.Wh + (b - g.NS) * g.W;
}

__device__ __forceinline__ int64_t wrap_pos(int64_t p, const Geo& g) {
  if (g.big_halo) {
    p %= g.n;
    return p < 0 ? p + g.n : p;
  }
  return p < 0 ? p + g.n : (p >= g.n ? p - g.n : p);
}

// Extended index of this thread's first sample.
__device__ __forceinline__ int64_t thread_e0(const Geo& g, int R) {
  return tile_lo(g, blockIdx.x) - g.H + (int64_t)threadIdx.x * R;
}

// Per-thread view of its R consecutive extended samples [e0, e0+R): block b0 and extended
// position q0 of the first one.  When ext >= R (the normal case) the R samples touch at most
// blocks b0 and b0+1, so every per-sample index below is 32-bit arithmetic on q0 + k.
struct Span {
  int64_t b0;   // block of sample 0 (-1 when e0 < 0)
  int q0;       // extended position of sample 0, in [0, ext)
};

__device__ __forceinline__ Span make_span(int64_t e0, const Geo& g) {
  Span sp;
  sp.b0 = e0 >= 0 ? e0 / g.ext : -1;
  sp.q0 = (int)(e0 - sp.b0 * g.ext);
  return sp;
}

// Sample k of the span -> (block, sample position in [0,n)); returns false if outside [0, B).
// `small` = (ext < R): the span may cross several blocks (tiny n): fall back to division.
template <int R>
__device__ __forceinline__ bool span_at(const Span& sp, int k, const Geo& g, int64_t e0, int64_t* b, int64_t* pos,
                                        int* q_out) {
  int64_t bb;
  int q;
  if (g.ext >= R) {
    q = sp.q0 + k;
    bb = sp.b0;
    if (q >= g.ext) { q -= (int)g.ext; ++bb; }
  } else {
    const int64_t e = e0 + k;
    bb = e >= 0 ? e / g.ext : -1;
    q = (int)(e - bb * g.ext);
  }
  *b = bb;
  *q_out = q;
  *pos = wrap_pos((int64_t)q - g.H, g);
  return bb >= 0 && bb < g.B && e0 + k >= 0;
}

// Fast path: the thread's R samples are R consecutive real samples of one block (no wrap, no
// block junction) -> plain contiguous addressing.  True for all but a few threads per block.
template <int R>
__device__ __forceinline__ bool span_fast(const Span& sp, const Geo& g, int64_t e0) {
  return e0 >= 0 && sp.b0 < g.B && sp.q0 >= g.H && (int64_t)sp.q0 + R <= g.H + g.n;
}

// Values are complex64 kept as one 64-bit register pair (f2x, see ldbp_f32x2.cuh).
// Load R consecutive extended samples starting at e0 (zeros outside [0, E)).
template <int R>
__device__ __forceinline__ void load_window(const float2* __restrict__ src, int64_t e0, const Geo& g,
                                            f2x (&u)[R]) {
  const f2x* s2 = reinterpret_cast<const f2x*>(src);
  const Span sp = make_span(e0, g);
  if (span_fast<R>(sp, g, e0)) {
    const f2x* p = s2 + sp.b0 * g.n + (sp.q0 - g.H);
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = __ldg(p + k);
    return;
  }
#pragma unroll
  for (int k = 0; k < R; ++k) {
    int64_t b, pos;
    int q;
    const bool ok = span_at<R>(sp, k, g, e0, &b, &pos, &q);
    u[k] = ok ? __ldg(s2 + b * g.n + pos) : 0ull;
  }
}

// Bitmask of which of this thread's R samples are owned real samples of this CTA.
template <int R>
__device__ __forceinline__ uint32_t owned_mask(int64_t e0, const Geo& g, int64_t tile = -1) {
  if (tile < 0) tile = blockIdx.x;  // persistent kernels pass the tile they are working on
  const int64_t lo = tile_lo(g, tile);
  const int64_t hi = min(lo + (tile < g.NS ? g.Wh : g.W), g.E);
  const Span sp = make_span(e0, g);
  constexpr uint32_t FULL = R >= 32 ? 0xffffffffu : ((1u << R) - 1u);
  if (e0 + R <= lo || e0 >= hi) return 0u;
  if (span_fast<R>(sp, g, e0)) {  // R real samples of one block: only the tile edges cut the run
    uint32_t m = FULL;
    if (e0 < lo) m &= FULL << (int)(lo - e0);
    if (e0 + R > hi) m &= FULL >> (int)(e0 + R - hi);
    return m;
  }
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    int64_t b, pos;
    int q;
    span_at<R>(sp, k, g, e0, &b, &pos, &q);
    const int64_t e = e0 + k;
    if (e >= lo && e < hi && q >= g.H && q < g.H + g.n) m |= (1u << k);
  }
  return m;
}

// Per-thread store descriptor, computed once: fast threads store R contiguous samples.
struct StoreMap {
  int64_t off;    // element offset of sample 0 (fast path), -1 if the slow path is needed
  uint32_t mask;  // owned samples
};

template <int R>
__device__ __forceinline__ StoreMap store_map(int64_t e0, const Geo& g) {
  StoreMap sm;
  sm.mask = owned_mask<R>(e0, g);
  const Span sp = make_span(e0, g);
  sm.off = (sm.mask == (R >= 32 ? 0xffffffffu : ((1u << R) - 1u)) && span_fast<R>(sp, g, e0))
               ? sp.b0 * g.n + (sp.q0 - g.H)
               : -1;
  return sm;
}

template <int R>
__device__ __forceinline__ void store_mapped(float2* __restrict__ dst, const StoreMap& sm, int64_t e0, const Geo& g,
                                             f2x (&u)[R]) {
  f2x* d2 = reinterpret_cast<f2x*>(dst);
  if (sm.off >= 0) {
    if (R % 2 == 0 && ((reinterpret_cast<uintptr_t>(d2 + sm.off) & 15) == 0)) {
      ulonglong2* d4 = reinterpret_cast<ulonglong2*>(d2 + sm.off);
#pragma unroll
      for (int k = 0; k < R / 2; ++k) d4[k] = make_ulonglong2(u[2 * k], u[2 * k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) d2[sm.off + k] = u[k];
    }
  } else if (sm.mask) {
    // owned samples have q in [H, H+n): position q - H, no wrap; only block crossings remain
    const Span sp = make_span(e0, g);
    int64_t b = sp.b0;
    int q = sp.q0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (sm.mask & (1u << k)) d2[b * g.n + (q - g.H)] = u[k];
      if (++q == g.ext) { q = 0; ++b; }
    }
  }
}

// Same, storing P * u[k] (complex scale applied per sample on the way out, no extra registers).
template <int R>
__device__ __forceinline__ void store_mapped_scaled(float2* __restrict__ dst, const StoreMap& sm, int64_t e0,
                                                    const Geo& g, const f2x (&u)[R], float2 P) {
  f2x* d2 = reinterpret_cast<f2x*>(dst);
  const f2x pa = pk(P.x, P.y), pb = pk(-P.y, P.x);
  if (sm.off >= 0) {
#pragma unroll
    for (int k = 0; k < R; ++k) d2[sm.off + k] = fma2(bcast(lof(u[k])), pa, mul2(bcast(hif(u[k])), pb));
  } else if (sm.mask) {
    const Span sp = make_span(e0, g);
    int64_t b = sp.b0;
    int q = sp.q0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      if (sm.mask & (1u << k)) d2[b * g.n + (q - g.H)] = fma2(bcast(lof(u[k])), pa, mul2(bcast(hif(u[k])), pb));
      if (++q == g.ext) { q = 0; ++b; }
    }
  }
}

template <int R>
__device__ __forceinline__ void store_owned(float2* __restrict__ dst, int64_t e0, const Geo& g, f2x (&u)[R]) {
  const StoreMap sm = store_map<R>(e0, g);
  store_mapped<R>(dst, sm, e0, g, u);
}

// Halo exchange of one register array: hl = Kh samples left of u[0], hr = Kh samples right
// of u[R-1].  Shuffles inside the warp; warp edges through sh[2 buffers][2 sides][32 warps][KH].
template <int KH, int R, int MW = kMaxWarps>
__device__ __forceinline__ void exchange(const f2x (&u)[R], f2x (&hl)[KH > 0 ? KH : 1], f2x (&hr)[KH > 0 ? KH : 1],
                                         f2x* sh, int buf, int lane, int warp, int nwarps) {
  if constexpr (KH > 0) {
#pragma unroll
    for (int j = 0; j < KH; ++j) {
      hl[j] = __shfl_up_sync(kFull, u[R - KH + j], 1);
      hr[j] = __shfl_down_sync(kFull, u[j], 1);
    }
    f2x* head = sh + ((buf * 2 + 0) * MW) * KH;
    f2x* tail = sh + ((buf * 2 + 1) * MW) * KH;
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

// ---- neighbour-only synchronisation (mbarrier) -----------------------------------------
// Instead of a CTA-wide __syncthreads per step, warp w publishes its edge samples, arrives on
// its own mbarrier bar[it&1][w] (count 1) and waits only for warps w-1 / w+1 of the same
// iteration.  Double buffering is safe: a warp can overwrite buffer b at iteration it+2 only
// after its neighbours published iteration it+1, which they do after reading iteration it.
// For the same reason no barrier can run two phases ahead of a waiter, so the parity test
// (it >> 1) & 1 is exact.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  // try_wait suspends the thread in hardware for a bounded time; a bounded retry count turns a
  // (never expected) lost arrival into a trap instead of a hung GPU.
  unsigned ok = 0, n = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!ok && ++n < (1u << 24));
  if (!ok) __trap();
}
// bars: [2][kMaxWarps] mbarriers; call once per CTA (followed by a __syncthreads()).
__device__ __forceinline__ void nb_init(uint64_t* bars) {
  for (int i = threadIdx.x; i < 2 * kMaxWarps; i += blockDim.x) mbar_init(bars + i, 1);
}

// Exchange of up to two arrays (N = 1 or 2) with neighbour-only synchronisation.
template <int KH, int R, int N, int MW = kMaxWarps>
__device__ __forceinline__ void exchange_nb(const f2x (&u)[R], f2x (&hl)[KH > 0 ? KH : 1], f2x (&hr)[KH > 0 ? KH : 1],
                                            f2x* sh, const f2x (&v)[R], f2x (&gl)[KH > 0 ? KH : 1],
                                            f2x (&gr)[KH > 0 ? KH : 1], f2x* sh2, uint64_t* bars, int it, int lane,
                                            int warp, int nwarps) {
  if constexpr (KH > 0) {
    const int b = it & 1;
    const unsigned parity = (it >> 1) & 1;
#pragma unroll
    for (int j = 0; j < KH; ++j) {
      hl[j] = __shfl_up_sync(kFull, u[R - KH + j], 1);
      hr[j] = __shfl_down_sync(kFull, u[j], 1);
      if constexpr (N == 2) {
        gl[j] = __shfl_up_sync(kFull, v[R - KH + j], 1);
        gr[j] = __shfl_down_sync(kFull, v[j], 1);
      }
    }
    f2x* head = sh + ((b * 2 + 0) * MW) * KH;
    f2x* tail = sh + ((b * 2 + 1) * MW) * KH;
    f2x* head2 = sh2 + ((b * 2 + 0) * MW) * KH;
    f2x* tail2 = sh2 + ((b * 2 + 1) * MW) * KH;
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        head[warp * KH + j] = u[j];
        if constexpr (N == 2) head2[warp * KH + j] = v[j];
      }
    }
    if (lane == 31) {
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        tail[warp * KH + j] = u[R - KH + j];
        if constexpr (N == 2) tail2[warp * KH + j] = v[R - KH + j];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(bars + b * MW + warp);
    if (lane == 0 && warp > 0) {
      mbar_wait(bars + b * MW + warp - 1, parity);
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        hl[j] = tail[(warp - 1) * KH + j];
        if constexpr (N == 2) gl[j] = tail2[(warp - 1) * KH + j];
      }
    }
    if (lane == 31 && warp < nwarps - 1) {
      mbar_wait(bars + b * MW + warp + 1, parity);
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        hr[j] = head[(warp + 1) * KH + j];
        if constexpr (N == 2) gr[j] = head2[(warp + 1) * KH + j];
      }
    }
    __syncwarp();
  } else {
    (void)u; (void)hl; (void)hr; (void)sh; (void)v; (void)gl; (void)gr; (void)sh2; (void)bars; (void)it;
    (void)lane; (void)warp; (void)nwarps;
  }
}

// Shared-memory exchange without shuffles (forward kernel): every thread publishes its Kh head
// and tail samples in [Kh][nthr] arrays (consecutive lanes -> consecutive 8-byte words, no bank
// conflicts), one barrier, then reads thread tid-1's tail and tid+1's head.  Warp boundaries
// need no special case; 4*Kh LDS/STS replace 4*Kh 64-bit shuffles plus the divergent
// warp-edge code.  Double-buffered by step parity (one barrier per step).
template <int KH, int R>
__device__ __forceinline__ void exchange_smem(const f2x (&u)[R], f2x (&hl)[KH > 0 ? KH : 1],
                                              f2x (&hr)[KH > 0 ? KH : 1], f2x* sh, int buf, int nthr, int left,
                                              int right) {
  if constexpr (KH > 0) {
    f2x* head = sh + (buf * 2 + 0) * KH * nthr;
    f2x* tail = sh + (buf * 2 + 1) * KH * nthr;
#pragma unroll
    for (int j = 0; j < KH; ++j) {
      head[j * nthr + threadIdx.x] = u[j];
      tail[j * nthr + threadIdx.x] = u[R - KH + j];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < KH; ++j) {
      hl[j] = tail[j * nthr + left];
      hr[j] = head[j * nthr + right];
    }
  } else {
    (void)u; (void)hl; (void)hr; (void)sh; (void)buf; (void)nthr; (void)left; (void)right;
  }
}

// Two arrays exchanged around one barrier (backward reverse sweep).
template <int KH, int R, int MW = kMaxWarps>
__device__ __forceinline__ void exchange2(const f2x (&u)[R], f2x (&hl)[KH > 0 ? KH : 1], f2x (&hr)[KH > 0 ? KH : 1],
                                          f2x* sh, int buf, const f2x (&v)[R], f2x (&gl)[KH > 0 ? KH : 1],
                                          f2x (&gr)[KH > 0 ? KH : 1], f2x* sh2, int buf2, int lane, int warp,
                                          int nwarps) {
  if constexpr (KH > 0) {
#pragma unroll
    for (int j = 0; j < KH; ++j) {
      hl[j] = __shfl_up_sync(kFull, u[R - KH + j], 1);
      hr[j] = __shfl_down_sync(kFull, u[j], 1);
      gl[j] = __shfl_up_sync(kFull, v[R - KH + j], 1);
      gr[j] = __shfl_down_sync(kFull, v[j], 1);
    }
    f2x* head = sh + ((buf * 2 + 0) * MW) * KH;
    f2x* tail = sh + ((buf * 2 + 1) * MW) * KH;
    f2x* head2 = sh2 + ((buf2 * 2 + 0) * MW) * KH;
    f2x* tail2 = sh2 + ((buf2 * 2 + 1) * MW) * KH;
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < KH; ++j) { head[warp * KH + j] = u[j]; head2[warp * KH + j] = v[j]; }
    }
    if (lane == 31) {
#pragma unroll
      for (int j = 0; j < KH; ++j) { tail[warp * KH + j] = u[R - KH + j]; tail2[warp * KH + j] = v[R - KH + j]; }
    }
    __syncthreads();
    if (lane == 0 && warp > 0) {
#pragma unroll
      for (int j = 0; j < KH; ++j) { hl[j] = tail[(warp - 1) * KH + j]; gl[j] = tail2[(warp - 1) * KH + j]; }
    }
    if (lane == 31 && warp < nwarps - 1) {
#pragma unroll
      for (int j = 0; j < KH; ++j) { hr[j] = head[(warp + 1) * KH + j]; gr[j] = head2[(warp + 1) * KH + j]; }
    }
  } else {
    (void)u; (void)hl; (void)hr; (void)sh; (void)buf; (void)v; (void)gl; (void)gr; (void)sh2; (void)buf2;
    (void)lane; (void)warp; (void)nwarps;
  }
}

// Warp reduce-scatter of N values (N a power of two, 2 <= N <= 32) by a transposing butterfly:
// at each level a lane keeps half of its vector and adds the partner's copy of that half, so
// N-1 shuffles replace the 5N of N independent reductions.  Afterwards lane l holds the warp
// total of value index l >> (5 - log2 N) (replicated over the 32/N lanes sharing it).
template <int N>
__device__ __forceinline__ float warp_reduce_scatter(float (&v)[N], int lane) {
  static_assert(N >= 2 && N <= 32 && (N & (N - 1)) == 0, "N must be a power of two in [2, 32]");
#pragma unroll
  for (int L = N, o = 16; L > 1; L >>= 1, o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int i = 0; i < L / 2; ++i) {
      const float send = up ? v[i] : v[i + L / 2];
      const float keep = up ? v[i + L / 2] : v[i];
      v[i] = keep + __shfl_xor_sync(kFull, send, o);
    }
  }
  float r = v[0];
#pragma unroll
  for (int o = 16 / N; o > 0; o >>= 1) r += __shfl_xor_sync(kFull, r, o);
  return r;
}

// Padded value count for a warp reduction of V per-lane partials (V <= 64).
__host__ __device__ constexpr int red_vp(int v) {
  return v <= 2 ? 2 : v <= 4 ? 4 : v <= 8 ? 8 : v <= 16 ? 16 : v <= 32 ? 32 : 64;
}
// Warp totals of the first nvalid of N per-lane partials (N from red_vp) -> red[0, nvalid): the
// transposing butterfly on chunks of at most 32 values (wide filters, T > 15, have up to 63),
// one writer lane per value, fixed order (deterministic).  N <= 32 is exactly the single butterfly.
template <int N>
__device__ __forceinline__ void warp_reduce_write(float (&v)[N], int lane, float* red, int nvalid) {
  if constexpr (N <= 32) {
    const float r = warp_reduce_scatter<N>(v, lane);
    constexpr int SH = N == 2 ? 4 : N == 4 ? 3 : N == 8 ? 2 : N == 16 ? 1 : 0;
    const int idx = lane >> SH;
    if ((lane & ((1 << SH) - 1)) == 0 && idx < nvalid) red[idx] = r;
  } else {
    static_assert(N == 64, "at most 64 partials");
    float lo[32], hi[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      lo[i] = v[i];
      hi[i] = v[32 + i];
    }
    const float r0 = warp_reduce_scatter<32>(lo, lane);
    if (lane < nvalid) red[lane] = r0;
    const float r1 = warp_reduce_scatter<32>(hi, lane);
    if (32 + lane < nvalid) red[32 + lane] = r1;
  }
}

// Window accessor: index i in [-KH, R+KH).
#define LDBP_WIN(arr, hl, hr, i) ((i) < 0 ? hl[KH + (i)] : ((i) >= R ? hr[(i) - R] : arr[(i)]))

// Packed taps (ldbp_f32x2.cuh): forward h*s = lo(s)*(hx,hy) + hi(s)*(-hy,hx);
// adjoint conj(h)*s = lo(s)*(hx,-hy) + hi(s)*(hy,hx).  Staged once per CTA in shared memory.
struct TapP {
  f2x a, b;
};

__device__ __forceinline__ TapP tap_fwd(float2 h) { return {pk(h.x, h.y), pk(-h.y, h.x)}; }
__device__ __forceinline__ TapP tap_adj(float2 h) { return {pk(h.x, -h.y), pk(h.y, h.x)}; }
// acc + t*s  (t a packed tap of either kind): 2 FFMA2, broadcasts of lo(s)/hi(s) are free.
__device__ __forceinline__ f2x tmac(f2x acc, const TapP& t, f2x s) {
  return fma2(bcast(lof(s)), t.a, fma2(bcast(hif(s)), t.b, acc));
}
// Two independent accumulation chains (acc_a gets the lo(s) terms, acc_b the hi(s) terms):
// halves the dependent FFMA2 chain per output; the caller adds the two at the end.
__device__ __forceinline__ void tmac2(f2x& acc_a, f2x& acc_b, const TapP& t, f2x s) {
  acc_a = fma2(bcast(lof(s)), t.a, acc_a);
  acc_b = fma2(bcast(hif(s)), t.b, acc_b);
}
__device__ __forceinline__ f2x tmul(const TapP& t, f2x s) { return fma2(bcast(lof(s)), t.a, mul2(bcast(hif(s)), t.b)); }

// One FIR output k (compile-time), a_k = sum_j h_j w_{k-j} (packed FP32x2 complex MACs).
// SYM: taps hs[0..KH] = h_0..h_KH (folded, fig:filter P:494-509: pre-add u_{k-j}+u_{k+j}).
// GEN: taps hs[0..2KH] = h_{-KH}..h_{KH}.
#ifndef LDBP_FIR_CHAINS
#define LDBP_FIR_CHAINS 1  // 1: one accumulation chain per output (R outputs give the ILP); 2: split
#endif
// KJ <= KH: number of active folded taps (per-step variable filter length, §8(f) NEXT-3: the
// outer taps j > KJ are zero, so skipping them is exact).
template <int KH, int R, bool SYM, int K, bool NORM = false, int KJ = KH>
__device__ __forceinline__ f2x fir_at(const f2x (&u)[R], const f2x (&hl)[KH > 0 ? KH : 1],
                                      const f2x (&hr)[KH > 0 ? KH : 1], const TapP (&hs)[SYM ? KH + 1 : 2 * KH + 1]) {
  if constexpr (LDBP_FIR_CHAINS == 1) {
    f2x acc;
    if constexpr (SYM && NORM) {
      // h0-normalised folded FIR: h_0 = 1, a_k = u_k + sum_j h_j (u_{k-j} + u_{k+j})
      acc = u[K];
#pragma unroll
      for (int j = 1; j <= KJ; ++j) acc = tmac(acc, hs[j], add2(LDBP_WIN(u, hl, hr, K - j), LDBP_WIN(u, hl, hr, K + j)));
    } else if constexpr (SYM) {
      acc = tmul(hs[0], u[K]);
#pragma unroll
      for (int j = 1; j <= KJ; ++j) acc = tmac(acc, hs[j], add2(LDBP_WIN(u, hl, hr, K - j), LDBP_WIN(u, hl, hr, K + j)));
    } else {
      acc = tmul(hs[0], LDBP_WIN(u, hl, hr, K + KH));
#pragma unroll
      for (int jj = 1; jj < 2 * KH + 1; ++jj) acc = tmac(acc, hs[jj], LDBP_WIN(u, hl, hr, K - (jj - KH)));
    }
    return acc;
  }
  f2x acc_a, acc_b;
  if constexpr (SYM && NORM) {
    // h0-normalised folded FIR: h_0 = 1, a_k = u_k + sum_j h_j (u_{k-j} + u_{k+j})
    if constexpr (KH == 0) return u[K];
    acc_a = u[K];
    const f2x s1 = add2(LDBP_WIN(u, hl, hr, K - 1), LDBP_WIN(u, hl, hr, K + 1));
    acc_a = fma2(bcast(lof(s1)), hs[1].a, acc_a);
    acc_b = mul2(bcast(hif(s1)), hs[1].b);
#pragma unroll
    for (int j = 2; j <= KH; ++j)
      tmac2(acc_a, acc_b, hs[j], add2(LDBP_WIN(u, hl, hr, K - j), LDBP_WIN(u, hl, hr, K + j)));
  } else if constexpr (SYM) {
    acc_a = mul2(bcast(lof(u[K])), hs[0].a);
    acc_b = mul2(bcast(hif(u[K])), hs[0].b);
#pragma unroll
    for (int j = 1; j <= KH; ++j)
      tmac2(acc_a, acc_b, hs[j], add2(LDBP_WIN(u, hl, hr, K - j), LDBP_WIN(u, hl, hr, K + j)));
  } else {
    const f2x w0 = LDBP_WIN(u, hl, hr, K + KH);
    acc_a = mul2(bcast(lof(w0)), hs[0].a);
    acc_b = mul2(bcast(hif(w0)), hs[0].b);
#pragma unroll
    for (int jj = 1; jj < 2 * KH + 1; ++jj) tmac2(acc_a, acc_b, hs[jj], LDBP_WIN(u, hl, hr, K - (jj - KH)));
  }
  return add2(acc_a, acc_b);
}

template <int KH, int R, bool SYM, int K = 0>
__device__ __forceinline__ void fir_all(const f2x (&u)[R], const f2x (&hl)[KH > 0 ? KH : 1],
                                        const f2x (&hr)[KH > 0 ? KH : 1], const TapP (&hs)[SYM ? KH + 1 : 2 * KH + 1],
                                        f2x (&a)[R]) {
  if constexpr (K < R) {
    a[K] = fir_at<KH, R, SYM, K>(u, hl, hr, hs);
    fir_all<KH, R, SYM, K + 1>(u, hl, hr, hs, a);
  }
}

// Kerr: v = a e^{j g |a|^2} = (ax c - ay s, ax s + ay c).  Scalar FFMAs: the packed form needs
// (-s, c) next to (c, s), i.e. a negate + move per sample (FP32x2 has no free half-negate), so
// the scalar form is cheaper on the FMA pipe (4 lane-ops, no moves).
#ifndef LDBP_KERR_SCALAR
#define LDBP_KERR_SCALAR 1
#endif
template <bool FAST>
__device__ __forceinline__ f2x kerr(f2x a, float g) {
  const float ax = lof(a), ay = hif(a);
  const float p = fmaf(ax, ax, ay * ay);
  float s, c;
  sincos_phase<FAST>(g * p, &s, &c);
  if constexpr (LDBP_KERR_SCALAR) return pk(fmaf(ax, c, -ay * s), fmaf(ax, s, ay * c));
  return fma2(bcast(ax), pk(c, s), mul2(bcast(ay), pk(-s, c)));
}

#ifndef LDBP_PIPE_D
#define LDBP_PIPE_D 2  // software-pipelining distance between FIR(k) and Kerr(k - D) in one step
#endif
// One full step (FIR + Kerr) for the R samples with the Kerr of sample k-D issued right after
// the FIR of sample k, so each warp's instruction stream mixes FMA-pipe and MUFU work instead
// of a pure-FMA phase followed by a MUFU-bound phase (all warps of a CTA are phase-aligned by
// the per-step barrier, so phase separation would idle one pipe at a time).
template <int KH, int R, bool SYM, bool FAST, bool NORM, int K = 0>
__device__ __forceinline__ void step_pipelined(const f2x (&u)[R], const f2x (&hl)[KH > 0 ? KH : 1],
                                               const f2x (&hr)[KH > 0 ? KH : 1],
                                               const TapP (&hs)[SYM ? KH + 1 : 2 * KH + 1], float gm, f2x (&acc)[R],
                                               f2x (&out)[R]) {
  constexpr int D = LDBP_PIPE_D;
  if constexpr (K < R + D) {
    if constexpr (K < R) acc[K] = fir_at<KH, R, SYM, K, NORM>(u, hl, hr, hs);
    if constexpr (K >= D) out[K - D] = kerr<FAST>(acc[K - D], gm);
    step_pipelined<KH, R, SYM, FAST, NORM, K + 1>(u, hl, hr, hs, gm, acc, out);
  }
}

template <bool SYM, int KH>
__device__ __forceinline__ constexpr int ntaps_used() { return SYM ? KH + 1 : 2 * KH + 1; }

// Per-step normalisation data (h0-normalised model).
struct StepNorm {
  float2 P;  // P_rel(i) = prod_{k=s0..i} c_k, c_k = h0^(k): u^(i+1) = P_rel(i) * u_hat^(i+1)
  float2 c;  // c_i = h0^(i)
};

// Normalisation over the step range [n0, nM) ("global" mode, used by the store-all training
// path so that every launch of a chain agrees): per step c_i = h0^(i) and the prefix products
// P_i = prod_{k=n0..i} c_k into sh_norm[i - n0]; *sh_flag = 1 iff the h0-normalised model is
// well conditioned over the whole range (same test as stage_params).  Reads taps from global
// memory (tiny, L2-resident); every CTA of every launch reaches the same decision.
template <int KH, bool SYM>
__device__ __forceinline__ void norm_range(const float2* __restrict__ taps, const uint8_t* __restrict__ mask, int T,
                                           int n0, int nM, StepNorm* sh_norm, int* sh_flag) {
  constexpr int NT = ntaps_used<SYM, KH>();
  const int S = nM - n0;
  if (threadIdx.x == 0) {
    sh_flag[0] = (SYM && LDBP_NORM) ? 1 : 0;
    sh_flag[1] = 0;  // set by stage_range when a step's outermost tap is zero (pruned)
  }
  __syncthreads();
  if (SYM && LDBP_NORM)
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
      const int s = n0 + i;
      float e = 0.f;
      float2 h0 = make_float2(0.f, 0.f);
      for (int t = 0; t < NT; ++t) {
        const int ti = t + KH;
        float2 h = taps[(int64_t)s * T + ti];
        if (mask && !mask[(int64_t)s * T + ti]) h = make_float2(0.f, 0.f);
        if (t == 0) h0 = h;
        e = fmaf(t ? 2.f : 1.f, h.x * h.x + h.y * h.y, e);
      }
      const float m0 = h0.x * h0.x + h0.y * h0.y;
      if (!(m0 > 0.f) || m0 < 1e-6f * e) *sh_flag = 0;
      sh_norm[i].c = h0;
    }
  __syncthreads();
  if (threadIdx.x == 0) {
    int ok = *sh_flag;
    double pr = 1.0, pi = 0.0;
    for (int i = 0; i < S; ++i) {
      if (ok) {
        const float2 c = sh_norm[i].c;
        const double nr = pr * c.x - pi * c.y, ni = pr * c.y + pi * c.x;
        pr = nr;
        pi = ni;
        const double mp = pr * pr + pi * pi;
        if (!(mp >= 1e-24 && mp <= 1e24)) ok = 0;
        sh_norm[i].P = make_float2((float)pr, (float)pi);
      }
    }
    if (!ok)
      for (int i = 0; i < S; ++i) {
        sh_norm[i].P = make_float2(1.f, 0.f);
        sh_norm[i].c = make_float2(1.f, 0.f);
      }
    *sh_flag = ok;
  }
  __syncthreads();
}

// Stage taps (packed forward and/or adjoint form) and gamma_hat of steps [s0, s1) using the
// normalisation computed by norm_range over [n0, nM) (sh_norm indexed by step - n0).
template <int KH, bool SYM, bool FWD, bool ADJ>
__device__ __forceinline__ void stage_range(const float2* __restrict__ taps, const float* __restrict__ gamma,
                                            const uint8_t* __restrict__ mask, int T, int s0, int s1, int n0,
                                            TapP* sh_taps, TapP* sh_taps_adj, float* sh_gamma,
                                            const StepNorm* sh_norm, bool norm, int* pruned = nullptr) {
  constexpr int NT = ntaps_used<SYM, KH>();
  const int S = s1 - s0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    float gm = gamma[s0 + i];
    if (norm) {
      const float2 P = sh_norm[s0 + i - n0].P;
      gm = (float)((double)gm * ((double)P.x * P.x + (double)P.y * P.y));
    }
    sh_gamma[i] = gm;
  }
  for (int i = threadIdx.x; i < S * NT; i += blockDim.x) {
    const int s = s0 + i / NT;
    const int t = (i % NT) + (SYM ? KH : 0);
    float2 h = taps[(int64_t)s * T + t];
    if (mask && !mask[(int64_t)s * T + t]) h = make_float2(0.f, 0.f);
    if (SYM && KH >= 1 && pruned && t == 2 * KH && h.x == 0.f && h.y == 0.f) *pruned = 1;
    if (norm) {
      const float2 c = sh_norm[s - n0].c;
      const float inv = 1.f / (c.x * c.x + c.y * c.y);
      h = make_float2((h.x * c.x + h.y * c.y) * inv, (h.y * c.x - h.x * c.y) * inv);
      if (t == KH) h = make_float2(1.f, 0.f);
    }
    if constexpr (FWD) sh_taps[i] = tap_fwd(h);
    if constexpr (ADJ) sh_taps_adj[i] = tap_adj(h);
  }
}

// Stage the packed taps and gamma of steps [s0, s1) into shared memory (masked taps -> 0;
// SYM keeps only h_0..h_Kh).  ADJ additionally stages the adjoint (conjugate) packing.
// SYM: thread 0 first decides whether the h0-normalised model is well conditioned for this
// launch (|h0|^2 >= 1e-6 sum|h|^2 at every step and 1e-12 <= |P_rel| <= 1e12); if so the staged
// taps are h/h0, gamma is gamma*|P_rel|^2 and *sh_flag = 1.
template <int KH, bool SYM, bool ADJ>
__device__ __forceinline__ void stage_params(const float2* __restrict__ taps, const float* __restrict__ gamma,
                                             const uint8_t* __restrict__ mask, int T, int s0, int s1,
                                             TapP* sh_taps, TapP* sh_taps_adj, float* sh_gamma, StepNorm* sh_norm,
                                             int* sh_flag) {
  constexpr int NT = ntaps_used<SYM, KH>();
  const int S = s1 - s0;
  // Phase 0: one coalesced, fully parallel read of the raw (masked) taps this launch needs and
  // of gamma; the packed-tap array doubles as the raw staging area (NT float2 <= NT TapP).
  // The per-step scalars are derived from shared memory only, so no global-memory latency is
  // serialised behind the barriers below.
  float2* raw = reinterpret_cast<float2*>(sh_taps_adj ? sh_taps_adj : sh_taps) + (ADJ ? 0 : S * NT);
  const int cnt = S * NT;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
    const int s = s0 + i / NT;
    const int t = (i % NT) + (SYM ? KH : 0);  // index into the stored [T] row
    float2 h = taps[(int64_t)s * T + t];
    if (mask && !mask[(int64_t)s * T + t]) h = make_float2(0.f, 0.f);
    raw[i] = h;
  }
  for (int i = threadIdx.x; i < S; i += blockDim.x) sh_gamma[i] = gamma[s0 + i];
  if (threadIdx.x == 0) {
    sh_flag[0] = (SYM && LDBP_NORM) ? 1 : 0;
    sh_flag[1] = 0;  // any step with a zero outermost tap (pruned), set by pack()
  }
  __syncthreads();
  // Phase A (parallel over steps): c_i = h0 and its conditioning (SYM stores h_0..h_Kh; the
  // energy of the full symmetric filter is |h0|^2 + 2 sum_{j>0} |h_j|^2).
  if (SYM && LDBP_NORM)
    for (int i = threadIdx.x; i < S; i += blockDim.x) {
      const float2 h0 = raw[i * NT];
      float e = 0.f;
      for (int t = 0; t < NT; ++t) {
        const float2 h = raw[i * NT + t];
        e = fmaf(t ? 2.f : 1.f, h.x * h.x + h.y * h.y, e);
      }
      const float m0 = h0.x * h0.x + h0.y * h0.y;
      if (!(m0 > 0.f) || m0 < 1e-6f * e) *sh_flag = 0;
      sh_norm[i].c = h0;
    }
  __syncthreads();
  // Phase B (one thread, shared memory only): prefix products P_rel(i) in fp64
  if (threadIdx.x == 0 && *sh_flag) {
    double pr = 1.0, pi = 0.0;
    int ok = 1;
    for (int i = 0; i < S; ++i) {
      const float2 c = sh_norm[i].c;
      const double nr = pr * c.x - pi * c.y, ni = pr * c.y + pi * c.x;
      pr = nr;
      pi = ni;
      const double mp = pr * pr + pi * pi;
      if (!(mp >= 1e-24 && mp <= 1e24)) ok = 0;
      sh_norm[i].P = make_float2((float)pr, (float)pi);
    }
    *sh_flag = ok;
  }
  __syncthreads();
  // Phase C (parallel): gamma_hat = gamma |P_rel|^2 and the packed taps (h / h0 when normalised).
  const bool norm = *sh_flag != 0;
  for (int i = threadIdx.x; i < S; i += blockDim.x) {
    if (norm) {
      const float2 P = sh_norm[i].P;
      sh_gamma[i] = (float)((double)sh_gamma[i] * ((double)P.x * P.x + (double)P.y * P.y));
    } else {
      sh_norm[i].P = make_float2(1.f, 0.f);
      sh_norm[i].c = make_float2(1.f, 0.f);
    }
  }
  // raw -> packed.  With ADJ the raw copy lives in sh_taps_adj: read everything first, then write
  // (raw[i] and the TapP slots it overlaps belong to thread-strided indices; a barrier separates).
  float2 hv[4];
  int nloc = 0;
  for (int i = threadIdx.x; i < cnt && nloc < 4; i += blockDim.x) hv[nloc++] = raw[i];
  const bool spill = cnt > 4 * (int)blockDim.x;
  __syncthreads();
  auto pack = [&](int i, float2 h) {
    const int t = (i % NT) + (SYM ? KH : 0);
    if (SYM && KH >= 1 && t == 2 * KH && h.x == 0.f && h.y == 0.f) sh_flag[1] = 1;
    if (norm) {  // h / c = h conj(c) / |c|^2
      const float2 c = sh_norm[i / NT].c;
      const float inv = 1.f / (c.x * c.x + c.y * c.y);
      h = make_float2((h.x * c.x + h.y * c.y) * inv, (h.y * c.x - h.x * c.y) * inv);
      if (t == KH) h = make_float2(1.f, 0.f);
    }
    sh_taps[i] = tap_fwd(h);
    if constexpr (ADJ) sh_taps_adj[i] = tap_adj(h);
  };
  if (!spill) {
    nloc = 0;
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) pack(i, hv[nloc++]);
  } else {  // very long launches: re-read the masked taps from global (rare: S*NT > 4*blockDim)
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const int s = s0 + i / NT;
      const int t = (i % NT) + (SYM ? KH : 0);
      float2 h = taps[(int64_t)s * T + t];
      if (mask && !mask[(int64_t)s * T + t]) h = make_float2(0.f, 0.f);
      pack(i, h);
    }
  }
}

// Model parameter table of the store-all training step (global normalisation): computed once
// per call by params_kernel, then copied by every CTA of the storing forward and the reverse
// launches with one round of asynchronous 16-/4-byte copies, instead of each CTA re-deriving the
// prefix products P_i (a serial fp64 chain over M steps behind three barriers) and re-packing
// the taps from global memory.
//   [flag int, 16 B][norm StepNorm[M]][gamma_hat float[M], 16 B-rounded][fwd TapP[M][NTU]]
//   [adj TapP[M][NTU]][kj int[M]]
struct PTab {
  int* flag;
  StepNorm* norm;
  float* gamma;
  TapP* fwd;
  TapP* adj;
  int* kj;
};
__host__ __device__ inline size_t ptab_bytes(int M, int ntu) {
  return 16 + 16 * (size_t)M + 16 * (((size_t)M + 3) / 4) + 32 * (size_t)M * ntu + 4 * (size_t)M;
}
__host__ __device__ inline PTab ptab_view(const void* base, int M, int ntu) {
  unsigned char* b = reinterpret_cast<unsigned char*>(const_cast<void*>(base));
  PTab p;
  p.flag = reinterpret_cast<int*>(b);
  b += 16;
  p.norm = reinterpret_cast<StepNorm*>(b);
  b += 16 * (size_t)M;
  p.gamma = reinterpret_cast<float*>(b);
  b += 16 * (((size_t)M + 3) / 4);
  p.fwd = reinterpret_cast<TapP*>(b);
  b += 16 * (size_t)M * ntu;
  p.adj = reinterpret_cast<TapP*>(b);
  b += 16 * (size_t)M * ntu;
  p.kj = reinterpret_cast<int*>(b);
  return p;
}

// One CTA: the same staging functions the kernels use, with the table in global memory as target.
constexpr int kParamsSmemSteps = 3072;
template <int KH, bool SYM>
__global__ void __launch_bounds__(256) params_kernel(const float2* __restrict__ taps, const float* __restrict__ gamma,
                                                     const uint8_t* __restrict__ mask, int T, int M, void* tab,
                                                     int in_smem) {
  constexpr int NTU = ntaps_used<SYM, KH>();
  const PTab p = ptab_view(tab, M, NTU);
  // the prefix-product chain runs on shared memory (in_smem: launched with M * 16 + 16 bytes of
  // dynamic shared memory, M <= kParamsSmemSteps), else on the table in global memory
  extern __shared__ __align__(16) unsigned char par_smem[];
  StepNorm* nrm = in_smem ? reinterpret_cast<StepNorm*>(par_smem + 16) : p.norm;
  int* flag = in_smem ? reinterpret_cast<int*>(par_smem) : p.flag;
  if (threadIdx.x == 0) p.flag[1] = 0;                 // pruned flag (ordered by norm_range's barriers)
  norm_range<KH, SYM>(taps, mask, T, 0, M, nrm, flag);  // ends with a barrier
  const bool norm = SYM && *flag;
  if (in_smem) {
    for (int i = threadIdx.x; i < M; i += blockDim.x) p.norm[i] = nrm[i];
    if (threadIdx.x == 0) *p.flag = *flag;
  }
  stage_range<KH, SYM, true, true>(taps, gamma, mask, T, 0, M, 0, p.fwd, p.adj, p.gamma, nrm, norm, p.flag + 1);
  for (int i = threadIdx.x; i < M; i += blockDim.x) {  // outermost unmasked folded tap per step
    int kj = KH;
    if (mask && SYM) {
      const uint8_t* mrow = mask + (int64_t)i * T + KH;
      kj = 0;
      for (int j = 1; j <= KH; ++j)
        if (mrow[j] || mrow[-j]) kj = j;
    }
    p.kj[i] = kj;
  }
}

__device__ __forceinline__ void ptab_cp16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void ptab_cp4(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
// Copy the slices a CTA needs (norm: all M; taps, gamma_hat, kj: steps [s0, s1)) into shared
// memory; all copies in flight at once.  Followed by the caller's __syncthreads.
template <int NTU>
__device__ __forceinline__ void load_ptab(const void* tab, int M, int s0, int s1, StepNorm* norm, TapP* fwd,
                                          TapP* adj, float* gam, int* kj, int* flag) {
  const PTab p = ptab_view(tab, M, NTU);
  const int S = s1 - s0, tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < M; i += nt) ptab_cp16(norm + i, p.norm + i);
  if (fwd)
    for (int i = tid; i < S * NTU; i += nt) ptab_cp16(fwd + i, p.fwd + (size_t)s0 * NTU + i);
  if (adj)
    for (int i = tid; i < S * NTU; i += nt) ptab_cp16(adj + i, p.adj + (size_t)s0 * NTU + i);
  for (int i = tid; i < S; i += nt) ptab_cp4(gam + i, p.gamma + s0 + i);
  if (kj)
    for (int i = tid; i < S; i += nt) ptab_cp4(kj + i, p.kj + s0 + i);
  if (tid == 0) {
    ptab_cp4(flag, p.flag);
    ptab_cp4(flag + 1, p.flag + 1);
  }
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}

// P * v for a staged complex scale P.
__device__ __forceinline__ f2x cscale(float2 P, f2x v) { return tmul(tap_fwd(P), v); }

struct FwdArgs {
  const float2* src;
  float2* dst;
  float2* ckpt;          // optional: after global step s with (s % ckpt_every) == 0, s in (s0, s1),
  int64_t ckpt_stride;   //   owned samples go to ckpt + (s / ckpt_every - 1) * ckpt_stride
  int ckpt_every;
  const float2* taps;
  const float* gamma;
  const uint8_t* mask;
  int T, s0, s1;
  // Normalisation range.  Local mode (n0 == s0, nM == s1): src is u^(s0) in the original scale,
  // every store is scaled back (P relative to s0).  Global mode (n0 = 0, nM = M, the store-all
  // training path): src is the normalised state u_hat^(s0), P is relative to step 0, and
  // checkpoints / dst are stored raw (normalised) unless scale_dst (then dst = y, original scale).
  int n0, nM;
  int global_norm;
  int scale_dst;
  int staged;  // store-all mode (ckpt_every == 1, global): coalesced stores through a smem stage
  float2* y_out;  // optional second output: the final state in the original scale (y)
  const void* ptab;  // store-all training: parameter table (params_kernel), or nullptr
  int* nonfinite; // LDBP_CHECK_FINITE: atomicMin of the first (1-based) step with a NaN/Inf output
  Geo g;
  // storing forward (LDBP_FWD_TMA): activation rows of 16 samples as a 2-D tensor [rows][16] x 8 B
  // over ckpt, 128-byte swizzle, box 32 rows; use_tmap = 0: lane stores
  int use_tmap;
  CUtensorMap tmap;
};

// ---------------------------------------------------------------------------------------
// Forward tile kernel: steps [s0, s1) of Eq. (7) for one tile, all on chip (rows a0-a4).
// ---------------------------------------------------------------------------------------
// Register budget per Kh: packed taps cost 4 registers each (TapP), so wider filters get
// fewer threads per CTA (the planner reads fwd_max_threads()).
#ifndef LDBP_FWD_WIDE_THREADS
#define LDBP_FWD_WIDE_THREADS 256
#endif
// Samples per thread of the inference / checkpoint forward tile kernel: 32 for wide filters
// (per-step overhead halved; measured C4 Kh = 7: 0.72 vs 0.63 of peak), 16 otherwise (C2 Kh = 2:
// 0.49 vs 0.40).  The store-all forward (training) keeps LDBP_FWD_R: its stage is R-sized.
#ifndef LDBP_FWD_R32_KH
#define LDBP_FWD_R32_KH 5
#endif
#ifndef LDBP_FWD_R_WIDE
#define LDBP_FWD_R_WIDE 32  // inference forward, Kh >= LDBP_FWD_R32_KH (<= 32: ownership masks are 32-bit)
#endif
#ifndef LDBP_FWD_R_SMALL
#define LDBP_FWD_R_SMALL 18  // inference forward, Kh <= 2 (C2: 18 0.540, 16 0.503, 20 0.47: 18 fits C2 in two waves)
#endif
// R <= 32 everywhere: per-thread ownership masks are 32-bit (static_assert in fwd_tile_body).
__host__ __device__ constexpr int fwd_r(int kh) {
  return kh >= LDBP_FWD_R32_KH ? LDBP_FWD_R_WIDE : (kh <= 2 ? LDBP_FWD_R_SMALL : LDBP_FWD_R);
}
// register target per thread for each Kh (packed taps cost 4 registers each)
__host__ __device__ constexpr int fwd_regs(int kh) { return kh <= 2 ? 64 : kh <= 5 ? 80 : 128; }
#ifdef LDBP_FWD_NTHR  // tuning override: fixed CTA size, residency from the register target
__host__ __device__ constexpr int fwd_max_threads(int) { return LDBP_FWD_NTHR; }
#else
// measured (C2 Kh=2: 128 thr 0.494 vs 512 thr 0.470 of peak; C5 store-all Kh=1: 10.3 vs 12.2 ms;
// C3 Kh=4 and C4 Kh=7: 256 best)
__host__ __device__ constexpr int fwd_max_threads(int kh) {
  return LDBP_FWD_R > 16 ? 256 : (kh <= 2 ? 128 : kh <= 5 ? 256 : LDBP_FWD_WIDE_THREADS);
}
#endif
// f2x elements of the store-all stage region: 2 buffers of ST runs of RS, plus run_off[ST] (int64)
#ifndef LDBP_FWD_WSTAGE
#define LDBP_FWD_WSTAGE 1  // store-all forward: 1 = halos through the edge arrays + per-warp store stage,
                           // 0 = one CTA-wide double-buffered stage for halos and stores
#endif
#ifndef LDBP_FWD_TMA
#define LDBP_FWD_TMA 1  // storing forward: activation stores by TMA tensor stores (see fwd_steps_split)
#endif
#ifndef LDBP_FWD_TMA_BUF
#define LDBP_FWD_TMA_BUF 2  // TMA stage buffers per warp (2: the next step's stage is written while the
                            // previous box is still being read by the TMA engine)
#endif
__host__ __device__ constexpr int fwd_stage_elems(int kh, int r) {
  // LDBP_FWD_TMA with two stage buffers per warp: 2 x 4 KB per warp plus 1 KB of alignment slack
  // (2r + 2 f2x per thread covers it for r = 16 and >= 32 threads)
  return LDBP_FWD_WSTAGE ? fwd_max_threads(kh) * (4 * (kh > 0 ? kh : 1) +
                                                  (LDBP_FWD_TMA && LDBP_FWD_TMA_BUF == 2 && r == 16 ? 2 * r + 2 : r + 2) + 1)
                         : fwd_max_threads(kh) * (2 * (r + 2) + 1);
}
#ifdef LDBP_FWD_NTHR
__host__ __device__ constexpr int fwd_min_blocks(int kh) { return 65536 / (LDBP_FWD_NTHR * fwd_regs(kh)); }
#else
#ifndef LDBP_FWD_SMALL_MINB
#define LDBP_FWD_SMALL_MINB 7  // Kh <= 2: resident 128-thread CTAs per SM (72 registers; C2: 7 0.503, 8 0.497, 6 0.46)
#endif
__host__ __device__ constexpr int fwd_min_blocks(int kh) {
  return kh <= 2 ? LDBP_FWD_SMALL_MINB : kh <= 4 ? 3 : (LDBP_FWD_WIDE_THREADS >= 512 && kh >= 6) ? 1 : 2;
}
#endif

template <int KH, int R, bool SYM, bool FAST, bool NORM>
__device__ __forceinline__ void fwd_steps(const FwdArgs& a, f2x (&u)[R], const TapP* sh_taps, const float* sh_gamma,
                                          const StepNorm* sh_norm, f2x* sh_edge, uint64_t* bars, const StoreMap& smap,
                                          int64_t e0, int lane, int warp, int nwarps) {
  const bool global = a.global_norm != 0;
  sh_norm += a.s0 - a.n0;  // sh_norm[s] = normalisation of global step s0 + s
  constexpr int NTU = ntaps_used<SYM, KH>();
  f2x hl[KH > 0 ? KH : 1], hr[KH > 0 ? KH : 1];
  const int left = threadIdx.x > 0 ? threadIdx.x - 1 : 0;
  const int right = threadIdx.x + 1 < blockDim.x ? threadIdx.x + 1 : threadIdx.x;
  for (int s = 0; s < a.s1 - a.s0; ++s) {
    TapP hs[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) hs[j] = sh_taps[s * NTU + j];
    const float gm = sh_gamma[s];
    if (LDBP_FWD_XSMEM)
      exchange_smem<KH, R>(u, hl, hr, sh_edge, s & 1, blockDim.x, left, right);
    else if (LDBP_NB_SYNC)
      exchange_nb<KH, R, 1>(u, hl, hr, sh_edge, u, hl, hr, sh_edge, bars, s, lane, warp, nwarps);
    else
      exchange<KH, R>(u, hl, hr, sh_edge, s & 1, lane, warp, nwarps);
    f2x acc[R], nu[R];
    step_pipelined<KH, R, SYM, FAST, NORM>(u, hl, hr, hs, gm, acc, nu);
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = nu[k];
    const int gs = a.s0 + s + 1;  // global step count reached
    if (a.ckpt && gs < a.s1 && gs % a.ckpt_every == 0) {
      if (global) {
        store_mapped<R>(a.ckpt + (int64_t)(gs / a.ckpt_every - 1) * a.ckpt_stride, smap, e0, a.g, u);
      } else if constexpr (NORM) {
        store_mapped_scaled<R>(a.ckpt + (int64_t)(gs / a.ckpt_every - 1) * a.ckpt_stride, smap, e0, a.g, u,
                               sh_norm[s].P);
      } else {
        store_mapped<R>(a.ckpt + (int64_t)(gs / a.ckpt_every - 1) * a.ckpt_stride, smap, e0, a.g, u);
      }
    }
  }
  if (NORM && (!global || a.scale_dst))
    store_mapped_scaled<R>(a.dst, smap, e0, a.g, u, sh_norm[a.s1 - a.s0 - 1].P);
  else
    store_mapped<R>(a.dst, smap, e0, a.g, u);
  if (a.y_out) {
    if constexpr (NORM)
      store_mapped_scaled<R>(a.y_out, smap, e0, a.g, u, sh_norm[a.s1 - a.s0 - 1].P);
    else
      store_mapped<R>(a.y_out, smap, e0, a.g, u);
  }
}

// FIR + Kerr for outputs k in [K, KE), with the Kerr of output k-D issued after the FIR of output
// k (MUFU work interleaved with FMA-pipe work); the last D Kerrs are flushed at the end.
template <int KH, int R, bool SYM, bool FAST, bool NORM, int KB, int KE, int KJ = KH, int K = KB>
__device__ __forceinline__ void step_range(const f2x (&u)[R], const f2x (&hl)[KH > 0 ? KH : 1],
                                           const f2x (&hr)[KH > 0 ? KH : 1],
                                           const TapP (&hs)[SYM ? KH + 1 : 2 * KH + 1], float gm, f2x (&acc)[R],
                                           f2x (&out)[R]) {
  constexpr int D = LDBP_PIPE_D;
  if constexpr (K < KE + D) {
    if constexpr (K < KE) acc[K] = fir_at<KH, R, SYM, K, NORM, KJ>(u, hl, hr, hs);
    if constexpr (K - D >= KB && K - D < KE) out[K - D] = kerr<FAST>(acc[K - D], gm);
    step_range<KH, R, SYM, FAST, NORM, KB, KE, KJ, K + 1>(u, hl, hr, hs, gm, acc, out);
  }
}

// Per-step active half-length dispatch (NEXT-3): variants for KJ = KH, KH-1, KH-2 (smaller KJ
// runs the KH-2 variant on zero taps: still exact); bounded code size.
template <int KH, typename F>
__device__ __forceinline__ void dispatch_kj(int kj, F&& f) {
  if (KH < 1 || kj >= KH) {
    f(std::integral_constant<int, KH>{});
  } else if (kj == KH - 1) {
    f(std::integral_constant<int, (KH >= 1 ? KH - 1 : 0)>{});
  } else {
    f(std::integral_constant<int, (KH >= 2 ? KH - 2 : 0)>{});
  }
}

#ifndef LDBP_FWD_UNROLL
#define LDBP_FWD_UNROLL 1
#endif
constexpr int kFwdUnroll = LDBP_FWD_UNROLL;
#ifndef LDBP_FWD_STORE_UNROLL
#define LDBP_FWD_STORE_UNROLL 2  // storing forward: two steps per loop iteration (C3 -1.3 %, measured;
                                 // the inference kernel is faster without: C2 +3 %, C4 +4 %)
#endif
constexpr int kFwdStoreUnroll = LDBP_FWD_STORE_UNROLL;
// mbarrier helpers for the split (arrive early / wait late) step barrier.
__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) { mbar_arrive(bar); }
#ifndef LDBP_MBAR_SUSPEND_NS
#define LDBP_MBAR_SUSPEND_NS 100000  // try_wait suspend-time hint: sleep until the phase completes
#endif
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(LDBP_MBAR_SUSPEND_NS)
        : "memory");
  } while (!ok);
}

// Forward steps with a split barrier (LDBP_FWD_SPLIT): at the end of step s every warp publishes
// its threads' Kh-sample edges into edge buffer (s+1)&1 and arrives (one elected lane, count =
// warps) on one CTA mbarrier; step s+1 first computes the R-2Kh interior outputs, which need no
// halo, and only then waits for phase s+1 and reads the neighbours' edges for the 2Kh boundary
// outputs.  The barrier latency and the warp skew hide behind the interior work.  Buffer reuse:
// buffer b is rewritten for phase p+2 by a warp that has passed phase p+1, whose arrivals all
// come after their reads of phase p.
// STG (store-all mode): instead of the Kh-sample edge arrays every thread publishes all R of its
// samples into a padded run-major stage stage[buf][t*RS + k] (RS = R + 2: conflict-free 16-byte
// stores and loads); neighbours take their halos from it and, after the barrier, the CTA copies
// the owned runs to HBM with lane-consecutive 16-byte stores (8 lanes per 128-byte run), instead
// of every thread storing its own R samples (lane stride R*8 bytes: one L2 sector per lane).
template <int R>
__device__ __forceinline__ constexpr int stage_rs() { return R + 2; }

template <int KH, int R, bool SYM, bool FAST, bool NORM, bool STG, bool VARK = false, bool CHK = false>
__device__ __forceinline__ void fwd_steps_split(const FwdArgs& a, f2x (&u)[R], const TapP* sh_taps,
                                                const float* sh_gamma, const StepNorm* sh_norm, f2x* sh_edge,
                                                uint64_t* bar, const StoreMap& smap, int64_t e0, int lane) {
  constexpr int RS = stage_rs<R>();
  constexpr int NTU = ntaps_used<SYM, KH>();
  constexpr int KI = KH < R - KH ? KH : R / 2;  // interior [KI, R-KI)
  constexpr int ST = fwd_max_threads(KH);       // edge-array row stride (compile time -> immediates)
  const bool global = a.global_norm != 0;
  sh_norm += a.s0 - a.n0;
  const int nthr = blockDim.x;
  const int tid = threadIdx.x;
  const int left = tid > 0 ? tid - 1 : 0;
  const int right = tid + 1 < nthr ? tid + 1 : tid;
  f2x* const my_edge = sh_edge + tid;
  const f2x* const left_edge = sh_edge + left;
  const f2x* const right_edge = sh_edge + right;
  // STG: stage[2][ST*RS] f2x, then run_off[ST] (int64: HBM element offset of run t, -1 = not an
  // owned real run, -2 = owned but irregular: the owner stores it itself)
  // WSTAGE: edges[2][2*KE][ST] as in the plain kernel, then wstage[ST/32 warps][32][RS] f2x, then
  // run_off[ST]
  constexpr int KE = KH > 0 ? KH : 1;
  constexpr bool WST = STG && LDBP_FWD_WSTAGE;
  f2x* const stage = sh_edge;
  int64_t* const run_off = reinterpret_cast<int64_t*>(sh_edge + (WST ? 4 * KE * ST + ST * RS : 2 * ST * RS));
  f2x* const wstage = sh_edge + 4 * KE * ST + (tid >> 5) * 32 * RS;
  const int64_t* const wrun_off = run_off + (tid & ~31);
  int t_lo = 0, t_hi = 0;
  // LDBP_FWD_TMA (R = 16: one run = one 128-byte row): a warp whose 32 runs are one contiguous,
  // 16-sample-aligned range of owned real samples writes them into a 1024-byte-aligned 4 KB stage
  // in the 128-byte-swizzled layout (chunk c of row L at c ^ (L & 7): conflict-free 16-byte
  // stores) and lane 0 hands the box to the TMA engine (cp.async.bulk.tensor store, SASS
  // UTMASTG), which un-swizzles it into the activation slot; other warps store from registers.
  constexpr bool TMA = WST && LDBP_FWD_TMA && R == 16;
  bool wtma = false;
  uint32_t tstage = 0;
  int64_t trow0 = 0;
  if constexpr (WST) {
    static_assert(R % 2 == 0 && 32 % (R / 2) == 0, "warp store stage: R/2 must divide 32");
    run_off[tid] = smap.off >= 0 ? smap.off : -1;  // warp-local: ordered by the __syncwarp of the first store
    if constexpr (TMA) {
      const int64_t off0 = __shfl_sync(kFull, smap.off, 0);
      wtma = a.use_tmap && __all_sync(kFull, smap.off >= 0 && smap.off == off0 + (int64_t)lane * R) &&
             (off0 % R) == 0;
      trow0 = off0 / R;  // + (gs - 1) * ckpt_stride / R per step
      const uint32_t sbase = (smem_u32(sh_edge + 4 * KE * ST) + 1023u) & ~1023u;
      tstage = sbase + (uint32_t)(tid >> 5) * (4096u * LDBP_FWD_TMA_BUF);
    }
  } else if constexpr (STG) {
    const bool fullrun = smap.off >= 0;
    run_off[tid] = fullrun ? smap.off : (smap.mask ? -2 : -1);
    const int64_t lo = tile_lo(a.g, blockIdx.x);
    const int64_t wc = min(lo + ((int64_t)blockIdx.x < a.g.NS ? a.g.Wh : a.g.W), a.g.E) - lo;
    t_lo = a.g.H / R;
    t_hi = (int)min((int64_t)nthr, (a.g.H + wc + R - 1) / R);
    __syncthreads();  // run_off visible before the first copy
  }
  auto publish = [&](int buf) {
    if constexpr (STG && !WST) {
      f2x* st = stage + buf * ST * RS + tid * RS;
#pragma unroll
      for (int m = 0; m < R / 2; ++m)
        *reinterpret_cast<ulonglong2*>(st + 2 * m) = make_ulonglong2(u[2 * m], u[2 * m + 1]);
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(bar);
    } else if constexpr (KH > 0) {
      f2x* e = my_edge + buf * 2 * KH * ST;
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        e[j * ST] = u[j];                  // head
        e[(KH + j) * ST] = u[R - KH + j];  // tail
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(bar);
    }
  };
  publish(0);
  f2x hl[KH > 0 ? KH : 1], hr[KH > 0 ? KH : 1];
  // checkpoint schedule without a per-step modulo: next global step count to store
  int next_ck = a.ckpt ? (a.s0 / a.ckpt_every + 1) * a.ckpt_every : 0x7fffffff;
  float2* ck_ptr = a.ckpt ? a.ckpt + (int64_t)(next_ck / a.ckpt_every - 1) * a.ckpt_stride : nullptr;
  constexpr int kUnroll = STG ? kFwdStoreUnroll : kFwdUnroll;
#pragma unroll kUnroll
  for (int s = 0; s < a.s1 - a.s0; ++s) {
    TapP hs[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) hs[j] = sh_taps[s * NTU + j];
    const float gm = sh_gamma[s];
    f2x acc[R], nu[R];
    // active folded taps of this step (outermost non-zero tap; uniform over the CTA)
    int kj = KH;
    if constexpr (VARK && SYM && NORM && KH >= 1) {
      kj = 0;
#pragma unroll
      for (int j = 1; j <= KH; ++j)
        if (lof(hs[j].a) != 0.f || hif(hs[j].a) != 0.f) kj = j;
    }
    auto do_step = [&](auto kjc) {
    constexpr int KJ = decltype(kjc)::value;
    constexpr int KI2 = KJ < R - KJ ? KJ : R / 2;
    step_range<KH, R, SYM, FAST, NORM, KI2, R - KI2, KJ>(u, hl, hr, hs, gm, acc, nu);
    if constexpr (STG && !WST) {
      mbar_wait_parity(bar, s & 1);
      const f2x* st = stage + (s & 1) * ST * RS;
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        hl[j] = st[left * RS + R - KH + j];
        hr[j] = st[right * RS + j];
      }
      // coalesced copy of u^(s0+s) (computed by this launch when s >= 1) to its activation slot
      if (s >= 1) {
        // thread tid always moves pair p2 = tid % (R/2) of runs t = t_lo + tid / (R/2) + k * nthr / (R/2)
        float2* const dstp = a.ckpt + (int64_t)(a.s0 + s - 1) * a.ckpt_stride + 2 * (tid % (R / 2));
        const f2x* const stp = st + 2 * (tid % (R / 2));
#pragma unroll 2
        for (int t = t_lo + tid / (R / 2); t < t_hi; t += nthr / (R / 2)) {
          const int64_t off = run_off[t];
          if (off >= 0)
            *reinterpret_cast<ulonglong2*>(dstp + off) = *reinterpret_cast<const ulonglong2*>(stp + t * RS);
        }
      }
    } else if constexpr (KH > 0) {
      mbar_wait_parity(bar, s & 1);
      const int off = (s & 1) * 2 * KH * ST;
#pragma unroll
      for (int j = 0; j < KH; ++j) {
        hl[j] = left_edge[off + (KH + j) * ST];
        hr[j] = right_edge[off + j * ST];
      }
    }
    step_range<KH, R, SYM, FAST, NORM, 0, KI2, KJ>(u, hl, hr, hs, gm, acc, nu);
    step_range<KH, R, SYM, FAST, NORM, R - KI2, R, KJ>(u, hl, hr, hs, gm, acc, nu);
    };
    if constexpr (VARK && SYM && NORM && FAST && KH >= 1)
      dispatch_kj<KH>(kj, do_step);
    else
      do_step(std::integral_constant<int, KH>{});
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = nu[k];
    const int gs = a.s0 + s + 1;  // global step count reached
    if constexpr (CHK) {  // LDBP_CHECK_FINITE: separate instantiation, the hot path carries no check code
      bool bad = false;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const float2 v = upk(u[k]);
        bad |= !(isfinite(v.x) && isfinite(v.y));
      }
      if (__any_sync(kFull, bad) && lane == 0 && a.nonfinite) atomicMin(a.nonfinite, gs);
    }
    if (gs < a.s1) publish((s + 1) & 1);
    if (TMA && a.use_tmap) {
      if (gs < a.s1 && wtma) {
        // stage buffer of this step free again: the box stored from it LDBP_FWD_TMA_BUF steps ago has
        // been read by the TMA engine
        if (lane == 0) {
          if constexpr (LDBP_FWD_TMA_BUF == 2)
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          else
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        __syncwarp();
        const uint32_t tst = tstage + (LDBP_FWD_TMA_BUF == 2 ? (uint32_t)(gs & 1) * 4096u : 0u);
        const uint32_t row = tst + (uint32_t)lane * 128u;
        const uint32_t sw = (uint32_t)(lane & 7);
#pragma unroll
        for (int m = 0; m < R / 2; ++m)
          asm volatile("st.shared.v2.u64 [%0], {%1, %2};" ::"r"(row + ((((uint32_t)m) ^ sw) << 4)), "l"(u[2 * m]),
                       "l"(u[2 * m + 1])
                       : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const int r = (int)(trow0 + (int64_t)(gs - 1) * (a.ckpt_stride / R));
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                  reinterpret_cast<uint64_t>(&a.tmap)),
              "r"(0), "r"(r), "r"(tst)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      } else if (gs < a.s1 && smap.off >= 0) {  // warps off the TMA path: own run from registers
        f2x* const d2 = reinterpret_cast<f2x*>(a.ckpt + (int64_t)(gs - 1) * a.ckpt_stride + smap.off);
        if ((reinterpret_cast<uintptr_t>(d2) & 15) == 0) {
#pragma unroll
          for (int m = 0; m < R / 2; ++m)
            reinterpret_cast<ulonglong2*>(d2)[m] = make_ulonglong2(u[2 * m], u[2 * m + 1]);
        } else {
#pragma unroll
          for (int k = 0; k < R; ++k) d2[k] = u[k];
        }
      }
    } else if constexpr (WST) {
      // (use_tmap == 0 for the whole launch, so no warp uses the TMA stage region)
      // u^(gs) -> activation slot gs-1: the warp's 32 runs through its stage, 16-byte lane-consecutive
      // stores (R/2 lanes per run); irregular runs are stored by their owners below
      if (gs < a.s1) {
#pragma unroll
        for (int m = 0; m < R / 2; ++m)
          *reinterpret_cast<ulonglong2*>(wstage + lane * RS + 2 * m) = make_ulonglong2(u[2 * m], u[2 * m + 1]);
        __syncwarp();
        float2* const dstp = a.ckpt + (int64_t)(gs - 1) * a.ckpt_stride + 2 * (lane % (R / 2));
        const f2x* const sp = wstage + 2 * (lane % (R / 2));
#pragma unroll
        for (int k = 0; k < R / 2; ++k) {
          const int t = lane / (R / 2) + k * (64 / R);
          const int64_t off = wrun_off[t];
          if (off >= 0) *reinterpret_cast<ulonglong2*>(dstp + off) = *reinterpret_cast<const ulonglong2*>(sp + t * RS);
        }
        __syncwarp();
      }
    }
    if (STG) {
      if (gs < a.s1 && smap.off < 0 && smap.mask) store_mapped<R>(ck_ptr, smap, e0, a.g, u);  // irregular run
      ck_ptr += a.ckpt_stride;
    } else if (gs == next_ck && gs < a.s1) {
      if (global) {
        store_mapped<R>(ck_ptr, smap, e0, a.g, u);
      } else if constexpr (NORM) {
        store_mapped_scaled<R>(ck_ptr, smap, e0, a.g, u, sh_norm[s].P);
      } else {
        store_mapped<R>(ck_ptr, smap, e0, a.g, u);
      }
      next_ck += a.ckpt_every;
      ck_ptr += a.ckpt_stride;
    }
  }
  if constexpr (TMA) {  // the stage must outlive the copies; activations complete before exit
    if (wtma && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    __syncwarp();
  }
  if (NORM && (!global || a.scale_dst))
    store_mapped_scaled<R>(a.dst, smap, e0, a.g, u, sh_norm[a.s1 - a.s0 - 1].P);
  else
    store_mapped<R>(a.dst, smap, e0, a.g, u);
  if (a.y_out) {
    if constexpr (NORM)
      store_mapped_scaled<R>(a.y_out, smap, e0, a.g, u, sh_norm[a.s1 - a.s0 - 1].P);
    else
      store_mapped<R>(a.y_out, smap, e0, a.g, u);
  }
}

#ifndef LDBP_FWD_SPLIT
#define LDBP_FWD_SPLIT 1
#endif

template <int KH, int R, bool SYM, bool FAST, bool STG, bool CHK = false>
__device__ __forceinline__ void fwd_tile_body(const FwdArgs& a) {
  static_assert(R % 2 == 0 && R <= 32, "R samples per thread: even, at most 32 (32-bit ownership masks)");
  constexpr int NTU = ntaps_used<SYM, KH>();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int S = a.s1 - a.s0;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);                            // [2][32] mbarriers
  f2x* sh_edge = reinterpret_cast<f2x*>(bars + 2 * kMaxWarps);  // 2*2*KH*(XSMEM ? nthreads : 32)
  TapP* sh_taps = reinterpret_cast<TapP*>(
      sh_edge + (STG ? fwd_stage_elems(KH, R)
                          : 4 * (LDBP_FWD_XSMEM ? fwd_max_threads(KH) : kMaxWarps) * (KH > 0 ? KH : 1)));  // S*NTU
  StepNorm* sh_norm = reinterpret_cast<StepNorm*>(sh_taps + S * NTU);                // max(S, nM-n0)
  float* sh_gamma = reinterpret_cast<float*>(sh_norm + max(S, a.nM - a.n0));         // S
  int* sh_flag = reinterpret_cast<int*>(sh_gamma + S);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  // LDBP_STREAM_PIPELINE: a programmatic-dependent next launch (the next batch's forward) may start
  // as soon as every CTA of this grid is running, i.e. while the last wave drains.  A next launch
  // without the PDL attribute still waits for this grid to complete; one with it that reads this
  // grid's output waits in griddepcontrol.wait (bwd_segment_kernel).
  if constexpr (!STG) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (LDBP_NB_SYNC && !LDBP_FWD_SPLIT) nb_init(bars);
  if (LDBP_FWD_SPLIT && threadIdx.x == 0) {  // split step barrier: bars[0], count = warps
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bars)), "r"(nwarps) : "memory");
  }
  f2x u[R];
  const int64_t e0 = thread_e0(a.g, R);
  load_window<R>(a.src, e0, a.g, u);
  const StoreMap smap = store_map<R>(e0, a.g);
  bool from_table = false;
  if constexpr (STG) {  // the storing forward only: keeps the inference kernel's prologue (and registers) lean
    if (a.global_norm && a.ptab) {
      load_ptab<NTU>(a.ptab, a.nM, a.s0, a.s1, sh_norm, sh_taps, nullptr, sh_gamma, nullptr, sh_flag);
      from_table = true;
    }
  }
  if (from_table) {
  } else if (a.global_norm) {
    norm_range<KH, SYM>(a.taps, a.mask, a.T, a.n0, a.nM, sh_norm, sh_flag);
    stage_range<KH, SYM, true, false>(a.taps, a.gamma, a.mask, a.T, a.s0, a.s1, a.n0, sh_taps, nullptr, sh_gamma,
                                      sh_norm, *sh_flag != 0, sh_flag + 1);
  } else {
    stage_params<KH, SYM, false>(a.taps, a.gamma, a.mask, a.T, a.s0, a.s1, sh_taps, nullptr, sh_gamma, sh_norm,
                                 sh_flag);
  }
  __syncthreads();
  // NEXT-3: does any step of this launch have zero outer taps?  (then the per-step active-length
  // loop runs; otherwise the plain loop, identical code to the unpruned kernel)
  bool pruned = false;
  if constexpr (SYM && FAST && KH >= 1) pruned = sh_flag[1] != 0;  // set during staging
  if constexpr (CHK) {  // LDBP_CHECK_FINITE: per-step check, plain loop (pruned taps are zeros, still exact)
    if (SYM && *sh_flag)
      fwd_steps_split<KH, R, SYM, FAST, true, STG, false, true>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap,
                                                                 e0, lane);
    else
      fwd_steps_split<KH, R, SYM, FAST, false, STG, false, true>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap,
                                                                  e0, lane);
  } else if constexpr (STG) {
    if (SYM && *sh_flag) {
      if (pruned)
        fwd_steps_split<KH, R, SYM, FAST, true, true, true>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap, e0,
                                                            lane);
      else
        fwd_steps_split<KH, R, SYM, FAST, true, true>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap, e0, lane);
    } else {
      fwd_steps_split<KH, R, SYM, FAST, false, true>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap, e0, lane);
    }
  } else if (SYM && *sh_flag)
    if (LDBP_FWD_SPLIT) {
      if (pruned)
        fwd_steps_split<KH, R, SYM, FAST, true, false, true>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap, e0,
                                                             lane);
      else
        fwd_steps_split<KH, R, SYM, FAST, true, false>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap, e0,
                                                       lane);
    } else
      fwd_steps<KH, R, SYM, FAST, true>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap, e0, lane, warp, nwarps);
  else if (LDBP_FWD_SPLIT)
    fwd_steps_split<KH, R, SYM, FAST, false, false>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap, e0, lane);
  else
    fwd_steps<KH, R, SYM, FAST, false>(a, u, sh_taps, sh_gamma, sh_norm, sh_edge, bars, smap, e0, lane, warp, nwarps);
}

// Forward tile kernel (inference, checkpoints): register budget for fwd_min_blocks CTAs per SM.
template <int KH, int R, bool SYM, bool FAST, bool CHK = false>
__global__ void __launch_bounds__(fwd_max_threads(KH), fwd_min_blocks(KH)) fwd_tile_kernel(const FwdArgs a) {
  fwd_tile_body<KH, R, SYM, FAST, false, CHK>(a);
}

// Store-all forward (training): the smem stage limits residency anyway, so the register budget
// is raised to 1-2 CTAs per SM (no spills in the step loop).
#ifndef LDBP_FWD_STORE_REGS
#define LDBP_FWD_STORE_REGS 128
#endif
template <int KH, int R, bool SYM, bool CHK = false>
__global__ void __launch_bounds__(fwd_max_threads(KH), 65536 / (fwd_max_threads(KH) * LDBP_FWD_STORE_REGS))
    fwd_store_kernel(const __grid_constant__ FwdArgs a) {
  fwd_tile_body<KH, R, SYM, true, true, CHK>(a);
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
constexpr int kBwdWarps = 8;  // backward CTAs have at most 256 threads

// cp.async (LDGSTS) 8-byte global -> shared copy, and the wait for all of this thread's copies.
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem_dst)), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

struct BwdSmem {
  uint64_t* bars;
  f2x* sh_edge;
  f2x* sh_edge2;
  TapP* sh_taps;
  TapP* sh_taps_adj;
  StepNorm* sh_norm;
  float* sh_gamma;
  int* sh_flag;
  float* sh_red;
  f2x* tape;
  f2x* pre;  // [R][nthr] prefetched target / incoming adjoint (fast-path threads)
};

template <int KH, int R, bool SYM, bool FAST, bool NORM>
__device__ __forceinline__ void bwd_body(const BwdArgs& a, const BwdSmem& sm, f2x (&u)[R], uint32_t own, int64_t e0,
                                         bool prefetched, int lane, int warp, int nwarps) {
  constexpr int NTU = ntaps_used<SYM, KH>();
  constexpr int V = 1 + 2 * NTU;  // [dgamma | dtap re/im ...]
  const int C = a.s1 - a.s0;
  const int nthr = blockDim.x;
  f2x* tape = sm.tape;

  f2x hl[KH > 0 ? KH : 1], hr[KH > 0 ? KH : 1];
  // ---- forward recompute, tape = inputs of each step (normalised state u_hat when NORM) ----
  for (int l = 0; l < C; ++l) {
#pragma unroll
    for (int k = 0; k < R; ++k) tape[(l * R + k) * nthr + threadIdx.x] = u[k];
    TapP hs[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) hs[j] = sm.sh_taps[l * NTU + j];
    const float gm = sm.sh_gamma[l];
    if (LDBP_NB_SYNC)
      exchange_nb<KH, R, 1, kBwdWarps>(u, hl, hr, sm.sh_edge, u, hl, hr, sm.sh_edge, sm.bars, l, lane, warp, nwarps);
    else
      exchange<KH, R, kBwdWarps>(u, hl, hr, sm.sh_edge, l & 1, lane, warp, nwarps);
    f2x acc[R], nu[R];
    step_pipelined<KH, R, SYM, FAST, NORM>(u, hl, hr, hs, gm, acc, nu);
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = nu[k];
  }

  // ---- seed / incoming adjoint (for the normalised state: g_hat = conj(P_end) g) ----
  const float2 Pend = sm.sh_norm[C - 1].P;
  const TapP conjP = tap_adj(Pend);  // conj(P) * v
  f2x g[R];
  // target / incoming adjoint: prefetched into shared memory at kernel start (fast-path threads)
  const bool pf = prefetched;
  cp_async_wait_all();
  if (a.gin == nullptr) {
    f2x t[R];
    if (pf) {
#pragma unroll
      for (int k = 0; k < R; ++k) t[k] = sm.pre[k * nthr + threadIdx.x];
    } else {
      load_window<R>(a.target, e0, a.g, t);
    }
    float lsum = 0.f;
    const f2x m1 = bcast(-1.f);
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const f2x y = NORM ? cscale(Pend, u[k]) : u[k];
      const f2x e = fma2(m1, t[k], y);  // y - target
      const f2x ge = mul2(bcast(a.seed_scale), e);
      g[k] = NORM ? tmul(conjP, ge) : ge;
      const float ex = lof(e), ey = hif(e);
      if (own & (1u << k)) lsum = fmaf(ex, ex, fmaf(ey, ey, lsum));
    }
    lsum = warp_sum(lsum);
    if (lane == 0) sm.sh_red[warp] = lsum;  // reused below only after a barrier
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int w = 0; w < nwarps; ++w) tot += (double)sm.sh_red[w];
      a.loss_partials[blockIdx.x] = tot;
    }
    __syncthreads();
  } else {
    if (pf) {
#pragma unroll
      for (int k = 0; k < R; ++k) g[k] = sm.pre[k * nthr + threadIdx.x];
    } else {
      load_window<R>(a.gin, e0, a.g, g);
    }
    if constexpr (NORM) {
#pragma unroll
      for (int k = 0; k < R; ++k) g[k] = tmul(conjP, g[k]);
    }
  }

  // ---- reverse sweep ----
  f2x gl[KH > 0 ? KH : 1], gr[KH > 0 ? KH : 1];
  for (int l = C - 1; l >= 0; --l) {
    TapP hs[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) hs[j] = sm.sh_taps_adj[l * NTU + j];
    const float gm = sm.sh_gamma[l];
    const float gm2 = 2.f * gm;
    // NL adjoint of step l: v = u (output of step l), g = dL/dv:
    //   c = Im(g conj v), t = g + 2 gamma' c v, ga = t e^{-j phi} = tx*(c,-s) + ty*(s,c).
    float dgam = 0.f;
    f2x ga[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const f2x v = u[k];
      const float vx = lof(v), vy = hif(v);
      const float p = fmaf(vx, vx, vy * vy);
      float sn, cs;
      sincos_phase<FAST>(gm * p, &sn, &cs);
      const float cim = fmaf(hif(g[k]), vx, -lof(g[k]) * vy);  // Im(g conj v)
      const f2x t = fma2(bcast(gm2 * cim), v, g[k]);
      ga[k] = fma2(bcast(lof(t)), pk(cs, -sn), mul2(bcast(hif(t)), pk(sn, cs)));
      if (own & (1u << k)) dgam = fmaf(cim, p, dgam);
    }
    // u^(s0+l): FIR input of step l.
#pragma unroll
    for (int k = 0; k < R; ++k) u[k] = tape[(l * R + k) * nthr + threadIdx.x];
    // exchange halos of u and ga around one barrier.  The u buffers continue the forward
    // loop's parity sequence (the last forward exchange used (C-1)&1), hence (l+1)&1.
    if (LDBP_NB_SYNC)
      exchange_nb<KH, R, 2, kBwdWarps>(u, hl, hr, sm.sh_edge, ga, gl, gr, sm.sh_edge2, sm.bars, 2 * C - 1 - l, lane, warp,
                            nwarps);
    else
      exchange2<KH, R, kBwdWarps>(u, hl, hr, sm.sh_edge, (l + 1) & 1, ga, gl, gr, sm.sh_edge2, l & 1, lane, warp, nwarps);
    // tap gradients over owned samples: dh_j += ga_t conj(w),  w = u_{t-j} (+ u_{t+j} if SYM)
    //   ga conj(w) = lo(w)*ga + hi(w)*(gy, -gx)
    f2x dh[NTU], dhb[NTU];
#pragma unroll
    for (int j = 0; j < NTU; ++j) dh[j] = dhb[j] = 0ull;
#pragma unroll
    for (int k = 0; k < R; ++k) {
      const f2x gk = (own & (1u << k)) ? ga[k] : 0ull;
      const TapP gt = {gk, pk(hif(gk), -lof(gk))};
      if constexpr (SYM) {
        tmac2(dh[0], dhb[0], gt, u[k]);
#pragma unroll
        for (int j = 1; j <= KH; ++j)
          tmac2(dh[j], dhb[j], gt, add2(LDBP_WIN(u, hl, hr, k - j), LDBP_WIN(u, hl, hr, k + j)));
      } else {
#pragma unroll
        for (int jj = 0; jj < 2 * KH + 1; ++jj) tmac2(dh[jj], dhb[jj], gt, LDBP_WIN(u, hl, hr, k - (jj - KH)));
      }
    }
#pragma unroll
    for (int j = 0; j < NTU; ++j) dh[j] = add2(dh[j], dhb[j]);
    // FIR adjoint: g_s = sum_j conj(h_j) ga_{s+j}   (NORM: h_0 = 1)
#pragma unroll
    for (int k = 0; k < R; ++k) {
      f2x acc_a, acc_b;
      if constexpr (SYM && NORM) {
        acc_a = ga[k];
        acc_b = 0ull;
#pragma unroll
        for (int j = 1; j <= KH; ++j)
          tmac2(acc_a, acc_b, hs[j], add2(LDBP_WIN(ga, gl, gr, k - j), LDBP_WIN(ga, gl, gr, k + j)));
      } else if constexpr (SYM) {
        acc_a = mul2(bcast(lof(ga[k])), hs[0].a);
        acc_b = mul2(bcast(hif(ga[k])), hs[0].b);
#pragma unroll
        for (int j = 1; j <= KH; ++j)
          tmac2(acc_a, acc_b, hs[j], add2(LDBP_WIN(ga, gl, gr, k - j), LDBP_WIN(ga, gl, gr, k + j)));
      } else {
        const f2x w0 = LDBP_WIN(ga, gl, gr, k - KH);
        acc_a = mul2(bcast(lof(w0)), hs[0].a);
        acc_b = mul2(bcast(hif(w0)), hs[0].b);
#pragma unroll
        for (int jj = 1; jj < 2 * KH + 1; ++jj) tmac2(acc_a, acc_b, hs[jj], LDBP_WIN(ga, gl, gr, k + (jj - KH)));
      }
      g[k] = (SYM && NORM && KH == 0) ? acc_a : add2(acc_a, acc_b);
    }
    // per-warp reduction of this step's partials (transposing butterfly, see above)
    {
      constexpr int VP = red_vp(V);
      float vals[VP];
      vals[0] = dgam;
#pragma unroll
      for (int j = 0; j < NTU; ++j) { vals[1 + 2 * j] = lof(dh[j]); vals[2 + 2 * j] = hif(dh[j]); }
#pragma unroll
      for (int i = V; i < VP; ++i) vals[i] = 0.f;
      warp_reduce_write<VP>(vals, lane, sm.sh_red + (l * nwarps + warp) * V, V);
    }
  }
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (a.gout) store_owned<R>(a.gout, e0, a.g, g);  // gout needs no scaling: P_rel before step s0 is 1
}

template <int KH, int R, bool SYM, bool FAST>
#ifndef LDBP_BWD_MINB
#define LDBP_BWD_MINB 2
#endif
__global__ void __launch_bounds__(256, LDBP_BWD_MINB) bwd_segment_kernel(const BwdArgs a) {
  constexpr int NTU = ntaps_used<SYM, KH>();
  constexpr int V = 1 + 2 * NTU;  // [dgamma | dtap re/im ...]
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int C = a.s1 - a.s0;
  const int nthr = blockDim.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = nthr >> 5;

  // carve-up (every region 16-byte aligned; mirrored by bwd_smem() on the host)
  BwdSmem sm;
  sm.bars = reinterpret_cast<uint64_t*>(smem_raw);  // [2][8] mbarriers
  sm.sh_edge = reinterpret_cast<f2x*>(sm.bars + 2 * kBwdWarps);  // two arrays: 2 * (2*2*8*KH)
  sm.sh_edge2 = sm.sh_edge + 4 * kBwdWarps * (KH > 0 ? KH : 1);
  sm.sh_taps = reinterpret_cast<TapP*>(sm.sh_edge2 + 4 * kBwdWarps * (KH > 0 ? KH : 1));
  sm.sh_taps_adj = sm.sh_taps + C * NTU;
  sm.sh_norm = reinterpret_cast<StepNorm*>(sm.sh_taps_adj + C * NTU);
  sm.sh_gamma = reinterpret_cast<float*>(sm.sh_norm + C);
  sm.sh_flag = reinterpret_cast<int*>(sm.sh_gamma + ((C + 3) & ~3));
  sm.sh_red = reinterpret_cast<float*>(sm.sh_flag + 4);                        // [C][nwarps][V]
  sm.tape = reinterpret_cast<f2x*>(sm.sh_red + ((C * nwarps * V + 3) & ~3));  // [C][R][nthr]
  sm.pre = sm.tape + (size_t)C * R * nthr;                                     // [R][nthr]

  if (LDBP_NB_SYNC) {
    for (int i = threadIdx.x; i < 2 * kBwdWarps; i += blockDim.x) mbar_init(sm.bars + i, 1);
  }
  const int64_t e0 = thread_e0(a.g, R);
  // Issue the (late-needed) target / incoming-adjoint loads first, asynchronously into smem, so
  // their latency overlaps the checkpoint load, the staging and the whole forward recompute.
  bool prefetched = false;
  if (LDBP_BWD_PREFETCH) {
    const Span sp = make_span(e0, a.g);
    if (span_fast<R>(sp, a.g, e0)) {
      const float2* src = a.gin ? a.gin : a.target;
      const float2* p = src + sp.b0 * a.g.n + (sp.q0 - a.g.H);
#pragma unroll
      for (int k = 0; k < R; ++k) cp_async8(sm.pre + k * nthr + threadIdx.x, p + k);
      asm volatile("cp.async.commit_group;" ::: "memory");
      prefetched = true;
    }
  }
  // Programmatic dependent launch: taps/gamma/mask/target are never written by the preceding
  // kernel (the previous backward segment or the checkpoint forward), so they are staged before
  // waiting; the checkpoint and the incoming adjoint are read after griddepcontrol.wait.
  const uint32_t own = owned_mask<R>(e0, a.g);
  stage_params<KH, SYM, true>(a.taps, a.gamma, a.mask, a.T, a.s0, a.s1, sm.sh_taps, sm.sh_taps_adj, sm.sh_gamma,
                              sm.sh_norm, sm.sh_flag);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  f2x u[R];
  load_window<R>(a.ck, e0, a.g, u);
  __syncthreads();
  const bool norm = SYM && *sm.sh_flag;
  if (norm)
    bwd_body<KH, R, SYM, FAST, true>(a, sm, u, own, e0, prefetched, lane, warp, nwarps);
  else
    bwd_body<KH, R, SYM, FAST, false>(a, sm, u, own, e0, prefetched, lane, warp, nwarps);
  __syncthreads();
  // CTA reduction in fp64, fixed order over warps; normalised-model gradients are mapped back
  // to the original parameters: dgamma_i = |P_rel(i)|^2 dgamma_hat_i, dh^(i) = conj(1/c_i) dh_hat^(i).
  const int npairs = 1 + NTU;  // slot 0: dgamma, slots 1..: complex taps
  for (int i = threadIdx.x; i < C * npairs; i += nthr) {
    const int l = i / npairs, q = i % npairs;
    double* out = a.partials + ((int64_t)blockIdx.x * a.M + (a.s0 + l)) * V;
    const StepNorm nm = sm.sh_norm[l];
    if (q == 0) {
      double acc = 0.0;
      for (int w = 0; w < nwarps; ++w) acc += (double)sm.sh_red[(l * nwarps + w) * V];
      if (norm) acc *= (double)nm.P.x * nm.P.x + (double)nm.P.y * nm.P.y;
      out[0] = acc;
    } else {
      const int v = 1 + 2 * (q - 1);
      double re = 0.0, im = 0.0;
      for (int w = 0; w < nwarps; ++w) {
        re += (double)sm.sh_red[(l * nwarps + w) * V + v];
        im += (double)sm.sh_red[(l * nwarps + w) * V + v + 1];
      }
      if (norm) {  // conj(1/c) = c / |c|^2
        const double cx = nm.c.x, cy = nm.c.y, m = cx * cx + cy * cy;
        const double r2 = (re * cx - im * cy) / m, i2 = (re * cy + im * cx) / m;
        re = r2;
        im = i2;
      }
      out[v] = re;
      out[v + 1] = im;
    }
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

// First level of the two-level reduction (used when there are many CTAs): grid
// (ceil(total/32) + 1, nchunks); block (x, y) sums CTAs [y*chunk, (y+1)*chunk) for outputs
// x*32 + lane (the extra x column does the loss partials) into out[y][...] in fixed order.
struct Reduce1Args {
  const double* partials;       // [nblk][total]
  const double* loss_partials;  // [nblk] or null
  int nblk, total, chunk;
  double* out;                  // [nchunks][total]
  double* loss_out;             // [nchunks]
};

__global__ void __launch_bounds__(256) reduce_partials_pass1(const Reduce1Args a) {
  __shared__ double red[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nout_blocks = (a.total + 31) / 32;
  const int c0 = blockIdx.y * a.chunk, c1 = min(c0 + a.chunk, a.nblk);
  if ((int)blockIdx.x == nout_blocks) {
    double s = 0.0;
    if (a.loss_partials)
      for (int c = c0 + threadIdx.x; c < c1; c += 256) s += a.loss_partials[c];
    red[warp][lane] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w)
        for (int l = 0; l < 32; ++l) t += red[w][l];
      a.loss_out[blockIdx.y] = t;
    }
    return;
  }
  const int i = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (i < a.total) {
    const double* p = a.partials + i;
#pragma unroll 4
    for (int c = c0 + warp; c < c1; c += 8) s += p[(int64_t)c * a.total];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp != 0 || i >= a.total) return;
  s = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[w][lane];
  a.out[(int64_t)blockIdx.y * a.total + i] = s;
}

// Launch with 256 threads and ceil(M*V/32) + 1 blocks.  Block k < last: lane = output
// (coalesced 256-B rows), warp w sums CTAs c = w, w+8, ... in order, then warp 0 adds the 8
// warp sums in order.  The last block reduces the loss partials the same way.  Fixed order
// everywhere -> bitwise deterministic.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const ReduceArgs a) {
  __shared__ double red[8][33];
  const int total = a.M * a.V;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nout_blocks = (total + 31) / 32;
  if ((int)blockIdx.x == nout_blocks) {  // loss
    if (!a.buf) return;
    double s = 0.0;
    if (a.loss_partials)
      for (int c = threadIdx.x; c < a.nblk; c += 256) s += a.loss_partials[c];
    red[warp][lane] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < 8; ++w)
        for (int l = 0; l < 32; ++l) t += red[w][l];
      a.buf[0] = t;
    }
    return;
  }
  const int i = blockIdx.x * 32 + lane;
  double s = 0.0;
  if (i < total) {
    const double* p = a.partials + i;
#pragma unroll 4
    for (int c = warp; c < a.nblk; c += 8) s += p[(int64_t)c * total];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp != 0 || i >= total) return;
  s = 0.0;
#pragma unroll
  for (int w = 0; w < 8; ++w) s += red[w][lane];
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
      dt[((int64_t)st * a.T + p1) * 2 + comp] = (a.mask && !a.mask[st * a.T + p1]) ? 0.0 : s;
      dt[((int64_t)st * a.T + p2) * 2 + comp] = (a.mask && !a.mask[st * a.T + p2]) ? 0.0 : s;
    } else {
      dt[((int64_t)st * a.T + ti) * 2 + comp] = (a.mask && !a.mask[st * a.T + ti]) ? 0.0 : s;
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

// One parameter's update (shared by adam_kernel and the fused tiny step: identical arithmetic).
// g is the raw (unscaled) gradient; th/m/v the current master, first and second moments.
// frozen / zero: the mask (zero: masked tap, forced to 0) and the non-learnable gamma' flags.
__device__ __forceinline__ void adam_elem_flags(const AdamArgs& a, int i, double g, double th, double m0, double v0,
                                                bool frozen, bool zero) {
  const int ntap = 2 * a.M * a.T;
  if (zero) {
    th = 0.0;
    a.m[i] = 0.0;
    a.v[i] = 0.0;
  } else if (!frozen) {
    g *= a.inv_n;
    const double m = a.b1 * m0 + (1.0 - a.b1) * g;
    const double v = a.b2 * v0 + (1.0 - a.b2) * g * g;
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

__device__ __forceinline__ void adam_elem(const AdamArgs& a, int i, double g, double th, double m0, double v0) {
  const int ntap = 2 * a.M * a.T;
  bool frozen, zero = false;
  if (i < ntap) {
    frozen = a.mask && !a.mask[i >> 1];
    zero = frozen;
  } else {
    frozen = a.glearn && !a.glearn[i - ntap];
  }
  adam_elem_flags(a, i, g, th, m0, v0, frozen, zero);
}

__global__ void adam_kernel(const AdamArgs a) {
  const int ntap = 2 * a.M * a.T;
  const int total = ntap + a.M;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const double g = i < ntap ? a.buf[1 + a.M + i] : a.buf[1 + (i - ntap)];
    adam_elem(a, i, g, a.master[i], a.m[i], a.v[i]);
  }
}

// buf[i] = sum_c bufs[c * stride + i], c = 0..K-1 in order (chunked training step, deterministic).
__global__ void sum_bufs_kernel(const double* __restrict__ bufs, int64_t stride, int K, int len, double* buf) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x) {
    double t = 0.0;
    for (int c = 0; c < K; ++c) t += bufs[(int64_t)c * stride + i];
    buf[i] = t;
  }
}
#endif  // LDBP_AUX_KERNELS

}  // namespace ldbp

#include "ldbp_reverse.cuh"

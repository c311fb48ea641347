// ldbp_api.cu — C ABI of libldbp (include/ldbp.h): validation, launch planning, dispatch.
//
// Planning: every kernel runs on a 1-D tiling of the "extended index space"
// (see ldbp_kernels.cuh).  The planner picks, per launch, the threads per CTA, the halo H =
// (#steps in the launch) * Kh (x2 for backward segments), and the owned width W such that the
// grid is a whole number of waves of resident CTAs on this device.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ldbp.h"
#define LDBP_AUX_KERNELS
#include "ldbp_kernels.cuh"
#include "ldbp_rx.cuh"
#include "ldbp_essm.cuh"
#include "ldbp_ssfm.cuh"
#include "ldbp_rx_exact.cuh"
#include "ldbp_tiny.cuh"

using FwdFn = void (*)(const ldbp::FwdArgs);
using BwdFn = void (*)(const ldbp::BwdArgs);
using RevFn = void (*)(const ldbp::RevArgs);
using ParFn = void (*)(const float2*, const float*, const uint8_t*, int, int, void*, int);

namespace {

thread_local char g_err[1024] = "";
thread_local int* g_nonfinite = nullptr;  // LDBP_CHECK_FINITE slot of the current call (device int)
constexpr size_t kCheckBytes = 256;
constexpr int kFiniteInit = 0x7f7f7f7f;  // memset(0x7f) pattern: no non-finite step seen

int fail(int status, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return status;
}

int cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(LDBP_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return LDBP_OK;
}

constexpr int kFwdR = LDBP_FWD_R;
constexpr int kFwdMaxThreads = 512;
constexpr int kBwdMaxThreads = 256;

// ---- launch tracing (thread-local; see ldbp_trace_begin in ldbp.h) ----
struct TraceRec {
  int kind, steps;
  int64_t samples;
  cudaEvent_t a, b;
};
thread_local bool g_trace_on = false;
thread_local int g_trace_cap = 0;
thread_local int g_trace_seen = 0;
thread_local std::vector<TraceRec> g_trace;

struct TraceScope {
  TraceRec rec{};
  bool active = false;
  cudaStream_t st;
  TraceScope(int kind, int steps, int64_t samples, cudaStream_t s) : st(s) {
    if (!g_trace_on) return;
    ++g_trace_seen;
    if ((int)g_trace.size() >= g_trace_cap) return;
    rec.kind = kind;
    rec.steps = steps;
    rec.samples = samples;
    if (cudaEventCreate(&rec.a) != cudaSuccess || cudaEventCreate(&rec.b) != cudaSuccess) {
      cudaGetLastError();
      return;
    }
    cudaEventRecord(rec.a, st);
    active = true;
  }
  ~TraceScope() {
    if (!active) return;
    cudaEventRecord(rec.b, st);
    g_trace.push_back(rec);
  }
};

int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

int ntaps_used(int kh, bool sym) { return sym ? kh + 1 : 2 * kh + 1; }
constexpr int kRxMaxSpsExact = 4;

// ----------------------------------------------------------------------------------------
// Kernel dispatch tables
// ----------------------------------------------------------------------------------------

// Kernel instantiations live in ldbp_inst.cu, compiled once per Kh (parallel build).
#define LDBP_DECL_GETTERS(K)                        \
  FwdFn ldbp_get_fwd_##K(bool sym, bool fast, bool chk); \
  FwdFn ldbp_get_fwd_store_##K(bool sym, bool chk); \
  BwdFn ldbp_get_bwd_##K(bool sym, bool fast);      \
  RevFn ldbp_get_rev_##K(bool sym, bool fast);      \
  RevFn ldbp_get_rev2_##K(bool fast);               \
  RevFn ldbp_get_rev3_##K(bool fast);               \
  RevFn ldbp_get_rev4_##K(bool fast);               \
  ParFn ldbp_get_params_##K(bool sym);
}  // namespace
LDBP_DECL_GETTERS(0)
LDBP_DECL_GETTERS(1)
LDBP_DECL_GETTERS(2)
LDBP_DECL_GETTERS(3)
LDBP_DECL_GETTERS(4)
LDBP_DECL_GETTERS(5)
LDBP_DECL_GETTERS(6)
LDBP_DECL_GETTERS(7)
LDBP_DECL_GETTERS(8)
LDBP_DECL_GETTERS(9)
LDBP_DECL_GETTERS(10)
LDBP_DECL_GETTERS(11)
LDBP_DECL_GETTERS(12)
LDBP_DECL_GETTERS(13)
LDBP_DECL_GETTERS(14)
LDBP_DECL_GETTERS(15)
namespace {

FwdFn get_fwd(int kh, bool sym, bool fast, bool chk = false) {
  switch (kh) {
    case 0: return ldbp_get_fwd_0(sym, fast, chk);
    case 1: return ldbp_get_fwd_1(sym, fast, chk);
    case 2: return ldbp_get_fwd_2(sym, fast, chk);
    case 3: return ldbp_get_fwd_3(sym, fast, chk);
    case 4: return ldbp_get_fwd_4(sym, fast, chk);
    case 5: return ldbp_get_fwd_5(sym, fast, chk);
    case 6: return ldbp_get_fwd_6(sym, fast, chk);
    case 7: return ldbp_get_fwd_7(sym, fast, chk);
    case 8: return ldbp_get_fwd_8(sym, fast, chk);
    case 9: return ldbp_get_fwd_9(sym, fast, chk);
    case 10: return ldbp_get_fwd_10(sym, fast, chk);
    case 11: return ldbp_get_fwd_11(sym, fast, chk);
    case 12: return ldbp_get_fwd_12(sym, fast, chk);
    case 13: return ldbp_get_fwd_13(sym, fast, chk);
    case 14: return ldbp_get_fwd_14(sym, fast, chk);
    case 15: return ldbp_get_fwd_15(sym, fast, chk);
  }
  return nullptr;
}
BwdFn get_bwd(int kh, bool sym, bool fast) {
  switch (kh) {
    case 0: return ldbp_get_bwd_0(sym, fast);
    case 1: return ldbp_get_bwd_1(sym, fast);
    case 2: return ldbp_get_bwd_2(sym, fast);
    case 3: return ldbp_get_bwd_3(sym, fast);
    case 4: return ldbp_get_bwd_4(sym, fast);
    case 5: return ldbp_get_bwd_5(sym, fast);
    case 6: return ldbp_get_bwd_6(sym, fast);
    case 7: return ldbp_get_bwd_7(sym, fast);
    case 8: return ldbp_get_bwd_8(sym, fast);
    case 9: return ldbp_get_bwd_9(sym, fast);
    case 10: return ldbp_get_bwd_10(sym, fast);
    case 11: return ldbp_get_bwd_11(sym, fast);
    case 12: return ldbp_get_bwd_12(sym, fast);
    case 13: return ldbp_get_bwd_13(sym, fast);
    case 14: return ldbp_get_bwd_14(sym, fast);
    case 15: return ldbp_get_bwd_15(sym, fast);
  }
  return nullptr;
}

FwdFn get_fwd_store(int kh, bool sym, bool chk = false) {
  switch (kh) {
    case 0: return ldbp_get_fwd_store_0(sym, chk);
    case 1: return ldbp_get_fwd_store_1(sym, chk);
    case 2: return ldbp_get_fwd_store_2(sym, chk);
    case 3: return ldbp_get_fwd_store_3(sym, chk);
    case 4: return ldbp_get_fwd_store_4(sym, chk);
    case 5: return ldbp_get_fwd_store_5(sym, chk);
    case 6: return ldbp_get_fwd_store_6(sym, chk);
    case 7: return ldbp_get_fwd_store_7(sym, chk);
    case 8: return ldbp_get_fwd_store_8(sym, chk);
    case 9: return ldbp_get_fwd_store_9(sym, chk);
    case 10: return ldbp_get_fwd_store_10(sym, chk);
    case 11: return ldbp_get_fwd_store_11(sym, chk);
    case 12: return ldbp_get_fwd_store_12(sym, chk);
    case 13: return ldbp_get_fwd_store_13(sym, chk);
    case 14: return ldbp_get_fwd_store_14(sym, chk);
    case 15: return ldbp_get_fwd_store_15(sym, chk);
  }
  return nullptr;
}

RevFn get_rev(int kh, bool sym, bool fast) {
  switch (kh) {
    case 0: return ldbp_get_rev_0(sym, fast);
    case 1: return ldbp_get_rev_1(sym, fast);
    case 2: return ldbp_get_rev_2(sym, fast);
    case 3: return ldbp_get_rev_3(sym, fast);
    case 4: return ldbp_get_rev_4(sym, fast);
    case 5: return ldbp_get_rev_5(sym, fast);
    case 6: return ldbp_get_rev_6(sym, fast);
    case 7: return ldbp_get_rev_7(sym, fast);
    case 8: return ldbp_get_rev_8(sym, fast);
    case 9: return ldbp_get_rev_9(sym, fast);
    case 10: return ldbp_get_rev_10(sym, fast);
    case 11: return ldbp_get_rev_11(sym, fast);
    case 12: return ldbp_get_rev_12(sym, fast);
    case 13: return ldbp_get_rev_13(sym, fast);
    case 14: return ldbp_get_rev_14(sym, fast);
    case 15: return ldbp_get_rev_15(sym, fast);
  }
  return nullptr;
}

RevFn get_rev2(int kh, bool fast) {
  switch (kh) {
    case 0: return ldbp_get_rev2_0(fast);
    case 1: return ldbp_get_rev2_1(fast);
    case 2: return ldbp_get_rev2_2(fast);
    case 3: return ldbp_get_rev2_3(fast);
    case 4: return ldbp_get_rev2_4(fast);
    case 5: return ldbp_get_rev2_5(fast);
    case 6: return ldbp_get_rev2_6(fast);
    case 7: return ldbp_get_rev2_7(fast);
    case 8: return ldbp_get_rev2_8(fast);
    case 9: return ldbp_get_rev2_9(fast);
    case 10: return ldbp_get_rev2_10(fast);
    case 11: return ldbp_get_rev2_11(fast);
    case 12: return ldbp_get_rev2_12(fast);
    case 13: return ldbp_get_rev2_13(fast);
    case 14: return ldbp_get_rev2_14(fast);
    case 15: return ldbp_get_rev2_15(fast);
  }
  return nullptr;
}

RevFn get_rev3(int kh, bool fast) {
  switch (kh) {
    case 2: return ldbp_get_rev3_2(fast);
    case 4: return ldbp_get_rev3_4(fast);
    case 6: return ldbp_get_rev3_6(fast);
  }
  return nullptr;
}

RevFn get_rev4(int kh, bool fast) {
  switch (kh) {
    case 1: return ldbp_get_rev4_1(fast);
    case 2: return ldbp_get_rev4_2(fast);
    case 3: return ldbp_get_rev4_3(fast);
    case 4: return ldbp_get_rev4_4(fast);
    case 5: return ldbp_get_rev4_5(fast);
    case 6: return ldbp_get_rev4_6(fast);
    case 7: return ldbp_get_rev4_7(fast);
    case 8: return ldbp_get_rev4_8(fast);
    case 9: return ldbp_get_rev4_9(fast);
    case 10: return ldbp_get_rev4_10(fast);
    case 11: return ldbp_get_rev4_11(fast);
    case 12: return ldbp_get_rev4_12(fast);
    case 13: return ldbp_get_rev4_13(fast);
    case 14: return ldbp_get_rev4_14(fast);
    case 15: return ldbp_get_rev4_15(fast);
  }
  return nullptr;
}

ParFn get_params(int kh, bool sym) {
  switch (kh) {
    case 0: return ldbp_get_params_0(sym);
    case 1: return ldbp_get_params_1(sym);
    case 2: return ldbp_get_params_2(sym);
    case 3: return ldbp_get_params_3(sym);
    case 4: return ldbp_get_params_4(sym);
    case 5: return ldbp_get_params_5(sym);
    case 6: return ldbp_get_params_6(sym);
    case 7: return ldbp_get_params_7(sym);
    case 8: return ldbp_get_params_8(sym);
    case 9: return ldbp_get_params_9(sym);
    case 10: return ldbp_get_params_10(sym);
    case 11: return ldbp_get_params_11(sym);
    case 12: return ldbp_get_params_12(sym);
    case 13: return ldbp_get_params_13(sym);
    case 14: return ldbp_get_params_14(sym);
    case 15: return ldbp_get_params_15(sym);
  }
  return nullptr;
}

int device_sms() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaGetLastError();
  return sms > 0 ? sms : 148;
}

// ----------------------------------------------------------------------------------------
// Planning
// ----------------------------------------------------------------------------------------
struct Tile {
  int nthreads = 0;
  int grid = 0;
  size_t smem = 0;
  ldbp::Geo g{};
};

size_t fwd_smem(int kh, bool sym, int steps, int nthreads = 1024, int nnorm = 0, bool staged = false) {
  (void)nthreads;
  const int edge_rows = LDBP_FWD_XSMEM ? ldbp::fwd_max_threads(kh) : ldbp::kMaxWarps;
  const size_t edge = staged ? sizeof(float2) * (size_t)ldbp::fwd_stage_elems(kh, kFwdR)
                             : sizeof(float2) * 4 * edge_rows * std::max(kh, 1);
  return sizeof(uint64_t) * 2 * ldbp::kMaxWarps + edge +
         sizeof(ldbp::TapP) * steps * ntaps_used(kh, sym) + sizeof(ldbp::StepNorm) * std::max(steps, nnorm) +
         sizeof(float) * steps + 32;
}

// Store-all reverse kernel shared memory (mirrors the carve-up in rev_tile_kernel).
size_t rev_smem(int kh, bool sym, int steps, int M) {
  const int NT = ldbp::rev_threads(kh), nw = NT / 32;
  const int V = 1 + 2 * ntaps_used(kh, sym);
  size_t s = 32 * (size_t)nw;                                         // split-barrier + bulk-copy mbarriers
  s += sizeof(float2) * LDBP_REV_PIPE * (size_t)(rev_r(kh) + (ldbp::rev_coal(kh) ? 2 : 0)) * NT;                       // u window copies
  s += sizeof(float2) * 4 * (size_t)std::max(kh, 1) * NT;             // ga edges
  s += sizeof(ldbp::TapP) * (size_t)steps * ntaps_used(kh, sym);      // adjoint taps
  s += sizeof(ldbp::StepNorm) * (size_t)M;                            // global normalisation
  s += sizeof(float) * (size_t)((steps * nw * V + 3) & ~3);           // per-warp partials, all steps
  s += sizeof(float) * (size_t)((nw + 3) & ~3);                       // loss partials
  s += sizeof(float) * (size_t)((steps + 3) & ~3) + 16;               // gamma_hat + flag
  s += sizeof(int) * (size_t)steps;                                   // active taps per step
  return s;
}

size_t bwd_smem(int kh, bool sym, int steps, int nthreads) {
  const int nw = nthreads / 32;
  const int V = 1 + 2 * ntaps_used(kh, sym);
  size_t s = sizeof(uint64_t) * 2 * ldbp::kBwdWarps;                   // mbarriers
  s += sizeof(float2) * 8 * ldbp::kBwdWarps * std::max(kh, 1);          // two edge arrays
  s += 2 * sizeof(ldbp::TapP) * steps * ntaps_used(kh, sym);             // packed fwd + adj taps
  s += sizeof(ldbp::StepNorm) * steps;                                  // normalisation
  s += sizeof(float) * ((steps + 3) & ~3) + 16;                         // gamma + flag
  s += sizeof(float) * ((steps * nw * V + 3) & ~3);                     // per-warp partials
  s += sizeof(float2) * size_t(steps + LDBP_BWD_PREFETCH) * bwd_r(kh) * nthreads;  // tape (+ prefetch buffer)
  return s;
}

// Choose the owned width and grid for a tiling with halo H, R samples per thread and at most
// max_threads threads.  `occ_per_sm` = resident CTAs/SM at max_threads (from the occupancy API).
// align_r: round H up and W to multiples of R, so that (for n % R == 0) every thread's R samples
// are either all owned real samples or none (no per-sample ownership masks on the hot path).
Tile plan_tiles(int64_t B, int64_t n, int H, int R, int max_threads, int occ_per_sm, int sms,
                bool align_r = false) {
  Tile t;
  if (align_r) H = (int)(cdiv(H, R) * R);
  const int64_t ext = n + 2 * (int64_t)H;
  const int64_t E = B * ext;
  const int64_t cap = (int64_t)max_threads * R;
  int64_t W0 = cap - 2 * (int64_t)H;
  if (W0 < R) W0 = R;  // caller guarantees H <= cap/4 normally
  const int64_t slots = (int64_t)std::max(occ_per_sm, 1) * sms;
  int64_t tiles = cdiv(E, W0);
  int64_t grid;
  if (tiles >= slots) {
    grid = cdiv(tiles, slots) * slots;  // whole waves
  } else {
    // small problem: spread over up to `slots` CTAs while keeping W >= max(4H, 32R)
    const int64_t wmin = std::max<int64_t>(4 * (int64_t)H, 32 * (int64_t)R);
    grid = std::max<int64_t>(tiles, std::min<int64_t>(slots, cdiv(E, wmin)));
  }
  int64_t W = cdiv(E, grid);
  if (align_r) W = cdiv(W, R) * R;
  grid = cdiv(E, W);
  int nthr = (int)cdiv(cdiv(W + 2 * (int64_t)H, R), 32) * 32;
  nthr = std::min(std::max(nthr, 32), max_threads);
  // phase staggering (see tile_lo in ldbp_kernels.cuh): with >= 2 resident CTAs per SM and
  // more than one wave, the first `sms` tiles are half width; the grid grows to cover E.
  int NS = 0;
  int64_t Wh = W;
  if (env_int("LDBP_STAGGER", 0) && occ_per_sm >= 2 && grid > slots && W >= 2 * R) {
    NS = sms;
    Wh = align_r ? (W / 2 / R) * R : W / 2;
    grid = NS + cdiv(std::max<int64_t>(E - (int64_t)NS * Wh, 0), W);
  }
  t.nthreads = nthr;
  t.grid = (int)grid;
  t.g.B = B;
  t.g.n = n;
  t.g.ext = ext;
  t.g.E = E;
  t.g.W = W;
  t.g.H = H;
  t.g.big_halo = H > n ? 1 : 0;
  t.g.NS = NS;
  t.g.Wh = Wh;
  return t;
}

struct FwdPlan {
  int segs = 1;       // number of launches
  int steps_per = 1;  // steps per launch (last may be shorter)
};

FwdPlan plan_fwd_segments(int M, int kh, int R = 0) {
  if (R == 0) R = ldbp::fwd_r(kh);
  FwdPlan p;
  if (M <= 0) return p;
  const int cap = std::min(env_int("LDBP_FWD_THREADS", kFwdMaxThreads), ldbp::fwd_max_threads(kh)) * R;
  int cmax = kh > 0 ? std::max(1, cap / (16 * kh)) : M;
  cmax = std::min(cmax, env_int("LDBP_FWD_MAX_STEPS", 1 << 30));
  p.segs = (int)cdiv(M, cmax);
  p.steps_per = (int)cdiv(M, p.segs);
  return p;
}

struct BwdPlan {
  int C = 1;     // steps per backward segment (last may be shorter)
  int K = 1;     // number of segments
  int nthreads = kBwdMaxThreads;
  Tile tile;     // uniform geometry for all segments (H = 2*C*kh)
  int V = 1;
};

int bwd_occupancy(BwdFn fn, int nthreads, size_t smem) {
  int occ = 0;
  cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, nthreads, smem) != cudaSuccess) occ = 1;
  cudaGetLastError();
  return std::max(occ, 1);
}

int fwd_occupancy(FwdFn fn, int nthreads, size_t smem) {
  int occ = 0;
  cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, nthreads, smem) != cudaSuccess) occ = 1;
  cudaGetLastError();
  return std::max(occ, 1);
}

BwdPlan plan_bwd(const ldbp_dims* d, bool query_device) {
  BwdPlan p;
  const int kh = (d->taps - 1) / 2;
  const bool sym = d->flags & LDBP_SYMMETRIC;
  const int M = d->steps;
  p.nthreads = env_int("LDBP_BWD_THREADS", kBwdMaxThreads);
  p.V = 1 + 2 * ntaps_used(kh, sym);
  const size_t budget = (size_t)env_int("LDBP_BWD_SMEM_KB", 110) * 1024;
  int C = 1;
  for (int c = 1; c <= M; ++c) {
    if (bwd_smem(kh, sym, c, p.nthreads) <= budget) C = c; else break;
  }
  C = std::min(C, env_int("LDBP_BWD_MAX_STEPS", 1 << 30));
  C = std::max(C, 1);
  p.K = (int)cdiv(M, C);
  p.C = (int)cdiv(M, p.K);  // equalised segment lengths
  const int H = 2 * p.C * kh;
  int occ = 1, sms = 148;
  if (query_device) {
    sms = device_sms();
    BwdFn fn = get_bwd(kh, sym, !(d->flags & LDBP_PRECISE));
    occ = bwd_occupancy(fn, p.nthreads, bwd_smem(kh, sym, p.C, p.nthreads));
  }
  p.tile = plan_tiles(d->batch, d->n, H, bwd_r(kh), p.nthreads, occ, sms);
  return p;
}

Tile plan_fwd_tile(const ldbp_dims* d, int steps, bool query_device, bool staged = false) {
  const int kh = (d->taps - 1) / 2;
  const bool sym = d->flags & LDBP_SYMMETRIC;
  const int maxthr = std::min(env_int("LDBP_FWD_THREADS", kFwdMaxThreads), ldbp::fwd_max_threads(kh));
  int occ = 1, sms = 148;
  const size_t smem = fwd_smem(kh, sym, steps, maxthr, staged ? d->steps : 0, staged);
  if (query_device) {
    sms = device_sms();
    occ = fwd_occupancy(staged ? get_fwd_store(kh, sym, g_nonfinite) : get_fwd(kh, sym, !(d->flags & LDBP_PRECISE), g_nonfinite), maxthr, smem);
  }
  Tile t = plan_tiles(d->batch, d->n, steps * kh, staged ? kFwdR : ldbp::fwd_r(kh), maxthr, occ, sms,
                      /*align_r=*/staged);
  t.smem = fwd_smem(kh, sym, steps, t.nthreads, 0, staged);
  return t;
}

// Store-all training path: forward launches store every activation, then
// Kr reverse launches of Cr steps each (halo Cr*Kh), adjoint passed through HBM between them.
struct RevPlan {
  int Cr = 1, Kr = 1;  // steps per reverse launch, number of reverse launches
  int V = 1;
  Tile tile;           // uniform geometry for all reverse launches (H = Cr*kh)
  int launch_grid = 0; // persistent kernels (rev4): resident CTAs, each walking tiles; 0 = tile.grid
};

int rev_occupancy(RevFn fn, int nthreads, size_t smem) {
  int occ = 0;
  cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)fn, nthreads, smem) != cudaSuccess) occ = 1;
  cudaGetLastError();
  return std::max(occ, 1);
}

// The warp-overlapped reverse (ldbp_reverse2.cuh, symmetric taps only) is OFF by default:
// measured slower than rev_tile_kernel on every shape (C3 reverse 2.37 ms at 8 warps/CTA, 2.49 at 4,
// 3.24 at 2, 3.86 at 1 warp vs 1.95; C5 15.6-20.5 vs 14.9 ms): the refresh barrier every R/Kh
// steps across 8 warps costs more than the per-step split barrier it replaces (28 % barrier
// stalls), and barrier-free 1-warp tiles pay 19-25 % halo recompute.  LDBP_REV2=1 selects it.
bool use_rev2(const ldbp_dims* d) {
  return (d->flags & LDBP_SYMMETRIC) && (d->taps - 1) / 2 <= 12 && env_int("LDBP_REV2", 0) != 0;
}

// The skewed one-sided reverse (ldbp_reverse3.cuh; symmetric taps, even Kh so the shifted windows
// stay 16-byte aligned) is OFF by default: parity-green but measured slower (C3 reverse 2.82 ms vs
// 1.95 ms): the one-way dependencies removed most barrier waiting (barrier + sleep stalls 8 %), but
// the shifted register windows cost 25 % register moves and the larger loop body 28 % instruction-
// fetch stalls.  LDBP_REV3=1 selects it.
bool use_rev3(const ldbp_dims* d) {
  const int kh = (d->taps - 1) / 2;
  return (d->flags & LDBP_SYMMETRIC) && (kh == 2 || kh == 4 || kh == 6) && !use_rev2(d) &&
         env_int("LDBP_REV3", 0) != 0;
}

// Shared-memory-adjoint reverse (ldbp_reverse4.cuh, symmetric taps, 1 <= Kh): LDBP_REV4=1/0 forces.
bool use_rev4(const ldbp_dims* d) {
  const int kh = (d->taps - 1) / 2;
  return (d->flags & LDBP_SYMMETRIC) && kh >= 1 && kh <= 12 && !use_rev2(d) && !use_rev3(d) &&
         env_int("LDBP_REV4", 0) != 0;
}

size_t rev_smem_any(const ldbp_dims* d, int steps) {
  const int kh = (d->taps - 1) / 2;
  if (use_rev4(d)) return ldbp::rev4_smem_bytes(kh, steps, d->steps);
  if (use_rev3(d)) return ldbp::rev3_smem_bytes(kh, steps, d->steps);
  return use_rev2(d) ? ldbp::rev2_smem_bytes(kh, steps, d->steps)
                     : rev_smem(kh, d->flags & LDBP_SYMMETRIC, steps, d->steps);
}

RevFn get_rev_any(const ldbp_dims* d) {
  const int kh = (d->taps - 1) / 2;
  const bool fast = !(d->flags & LDBP_PRECISE);
  if (use_rev3(d)) return get_rev3(kh, fast);
  if (use_rev4(d)) return get_rev4(kh, fast);
  return use_rev2(d) ? get_rev2(kh, fast) : get_rev(kh, d->flags & LDBP_SYMMETRIC, fast);
}

RevPlan plan_rev(const ldbp_dims* d, bool query_device) {
  RevPlan p;
  const int kh = (d->taps - 1) / 2;
  const bool sym = d->flags & LDBP_SYMMETRIC;
  const bool v2 = use_rev2(d), v3 = use_rev3(d), v4 = use_rev4(d);
  const int M = d->steps;
  const int R = v2 ? ldbp::rev2_r(kh) : v3 ? ldbp::rev3_r(kh) : v4 ? ldbp::rev4_r(kh) : rev_r(kh);
  // window slots per CTA (rev2: 30 owned lanes per warp + the two duplicate end lanes)
  const int slots = v2 ? ldbp::rev2_slots(ldbp::rev2_warps(kh)) : v3 ? 32 * ldbp::rev3_warps(kh)
                                                            : v4 ? ldbp::rev4_threads(kh) : ldbp::rev_threads(kh);
  const int nthr = v2 ? 32 * ldbp::rev2_warps(kh) : v3 ? 32 * ldbp::rev3_warps(kh)
                                                   : v4 ? ldbp::rev4_threads(kh) : ldbp::rev_threads(kh);
  p.V = 1 + 2 * ntaps_used(kh, sym);
  // cost model in step units: a launch of S steps costs S * window / (window - 2*H) plus a
  // fixed ~2 steps (prologue: staging, first load, seed), H = S*kh rounded up to whole slots;
  // pick the number of launches minimising it, subject to the shared-memory budget
  const double window = (double)slots * R;
  const double fixed = 2.0;
  const size_t budget = (size_t)env_int("LDBP_REV_SMEM_KB", v2 ? 150 : 113) * 1024;
  int best_k = 0;
  double best = 1e300;
  const int kmax = std::min(M, env_int("LDBP_REV_MAX_LAUNCHES", 256));
  const int cmax = std::max(1, env_int("LDBP_REV_MAX_STEPS", 1 << 30));
  for (int k = 1; k <= kmax; ++k) {
    const int S = (int)cdiv(M, k);
    if (S > cmax || rev_smem_any(d, S) > budget) continue;
    const double H = (double)cdiv((int64_t)S * kh, R) * R;
    const double useful = window - 2.0 * H;
    if (useful < window / 4) continue;
    const double cost = k * (S * window / useful + fixed);
    if (cost < best) { best = cost; best_k = k; }
  }
  if (best_k == 0) best_k = std::max((int)cdiv(M, cmax), (int)cdiv((int64_t)M * kh * 8, (int64_t)window));
  p.Kr = best_k;
  p.Cr = (int)cdiv(M, p.Kr);
  p.Kr = (int)cdiv(M, p.Cr);
  int occ = 1, sms = 148;
  if (query_device) {
    sms = device_sms();
    occ = rev_occupancy(get_rev_any(d), nthr, rev_smem_any(d, p.Cr));
  }
  // rev2: at least one halo slot per side (slot 0 / the last slot are never owned: duplicate lanes)
  const int H = v2 ? std::max(p.Cr * kh, 1) : p.Cr * kh;
  p.tile = plan_tiles(d->batch, d->n, H, R, slots, occ, sms, /*align_r=*/true);
  p.tile.nthreads = nthr;  // the kernel's layout is compiled for exactly this many threads
  if (v4 && env_int("LDBP_REV4_PERSIST", 0))
    p.launch_grid = (int)std::min<int64_t>(p.tile.grid, (int64_t)occ * sms);
  return p;
}

// Tiny problems (BASELINE C1): the whole training step in one cluster (ldbp_tiny.cuh).  B >= 8:
// 8 CTAs own whole blocks; B < 8: each block split into S segments of >= 256 samples (C = B S
// <= 16 CTAs, DSMEM halos).  At most kTinyPer samples per thread, <= 200 KB shared memory.
// Measured (profiles/r02_tiny_sweep.txt, 20 steps per CUDA graph, T = 3): one step of the fused
// kernel costs ~5.5 us + ~1.35 us per model step (a latency chain: two barriers and two
// shared-memory round trips per model step), the segment schedule ~10.3 us + ~0.5 us per step;
// the fused kernel wins up to M ~ 5 (C1, M = 4: 11.0 vs 12.5 us), and whenever the segment
// schedule needs more than one recompute segment (M = 16: ~27 vs ~37 us).
constexpr int kTinyAutoMaxSteps = 5;

struct TinyPlan {
  bool ok = false;
  int C = 1, S = 1, nrows = 1, lenmax = 0, nthr = 32;
  size_t smem = 0;
};

TinyPlan plan_tiny(const ldbp_dims* d, int max_cluster) {
  TinyPlan p;
  // LDBP_TINY: 0 off, 1 (default) when M <= kTinyAutoMaxSteps, 2 whenever it fits
  const int mode = env_int("LDBP_TINY", 1);
  if (mode == 0 || (d->flags & LDBP_CHECK_FINITE)) return p;
  if (mode == 1 && d->steps > kTinyAutoMaxSteps && plan_bwd(d, false).K == 1) return p;
  if (d->batch <= 0 || d->n <= 0 || d->batch * d->n > (int64_t)1 << 24) return p;
  const int kh = (d->taps - 1) / 2;
  if (kh > 7) return p;  // the fused tiny kernel is compiled for T <= 15
  if (d->batch >= 8 || max_cluster < d->batch) {
    p.C = (int)std::min<int64_t>(max_cluster, d->batch);
    p.nrows = (int)cdiv(d->batch, p.C);
    p.lenmax = (int)d->n;
  } else {
    int S = (int)std::min<int64_t>(max_cluster / d->batch, d->n / 256);
    while (S > 1 && d->n / S < std::max(kh, 1)) --S;
    p.S = std::max(S, 1);
    p.C = (int)d->batch * p.S;
    p.lenmax = (int)cdiv(d->n, p.S);
  }
  const int64_t per_cta = (int64_t)p.nrows * p.lenmax;
  if (per_cta > (int64_t)ldbp::kTinyPer * ldbp::kTinyMaxThreads) return p;
  p.nthr = (int)std::min<int64_t>(ldbp::kTinyMaxThreads, cdiv(per_cta, 32) * 32);
  p.smem = ldbp::tiny_smem_bytes(p.nrows, p.lenmax, d->steps, d->taps);
  p.ok = p.smem <= (size_t)200 * 1024;
  return p;
}

void (*tiny_kernel(int kh, bool precise))(const ldbp::TinyArgs) {
  using ldbp::tiny_train_kernel;
  static void (*const kerns[2][8])(const ldbp::TinyArgs) = {
      {tiny_train_kernel<0, false>, tiny_train_kernel<1, false>, tiny_train_kernel<2, false>,
       tiny_train_kernel<3, false>, tiny_train_kernel<4, false>, tiny_train_kernel<5, false>,
       tiny_train_kernel<6, false>, tiny_train_kernel<7, false>},
      {tiny_train_kernel<0, true>, tiny_train_kernel<1, true>, tiny_train_kernel<2, true>, tiny_train_kernel<3, true>,
       tiny_train_kernel<4, true>, tiny_train_kernel<5, true>, tiny_train_kernel<6, true>, tiny_train_kernel<7, true>}};
  return kerns[precise ? 1 : 0][kh];
}

// Largest cluster the tiny kernels may use on this device: 16 (non-portable) when a 16-CTA
// cluster of the largest tiny CTAs is schedulable, else 8.  Cached per device.
int tiny_max_cluster() {
  static std::atomic<int> cached[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 8;
  int v = cached[dev].load();
  if (v) return v;
  v = 8;
  void (*k)(const ldbp::TinyArgs) = tiny_kernel(1, false);
  if (cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
    cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(ldbp::kTinyMaxThreads);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 16;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, (const void*)k, &cfg) == cudaSuccess && nclusters > 0) v = 16;
  }
  cudaGetLastError();
  cached[dev].store(v);
  return v;
}

// LDBP_TINY_MAX_CLUSTER caps the cluster (and so the segments per block) for experiments.
int tiny_cluster_cap(const ldbp_dims* d) {
  const int cap = d->batch < 8 ? tiny_max_cluster() : 8;
  return std::max(1, std::min(cap, env_int("LDBP_TINY_MAX_CLUSTER", cap)));
}

bool use_tiny(const ldbp_dims* d) { return plan_tiny(d, tiny_cluster_cap(d)).ok; }

// Which training path: 1 = store-all activations + fused reverse (default when the activations
// fit the budget), 0 = checkpoint + recompute segments (memory-lean fallback).
bool use_store_all(const ldbp_dims* d) {
  if (d->flags & LDBP_CHECK_FINITE) return true;  // every step's activation is produced and checked
  const int mode = env_int("LDBP_BWD_MODE", -1);
  if (mode == 0) return false;
  if (mode == 1) return true;
  const double act_gb = (double)d->steps * (double)d->batch * (double)d->n * sizeof(float2) / 1073741824.0;
  // tiny problems (one wave, latency-bound, e.g. C1) keep the 3-launch segment schedule
  if ((double)d->batch * (double)d->n < (double)env_int("LDBP_STORE_ALL_MIN_SAMPLES", 1 << 20)) return false;
  return act_gb <= (double)env_int("LDBP_ACT_BUDGET_GB", 96);
}

// ----------------------------------------------------------------------------------------
// Validation
// ----------------------------------------------------------------------------------------
int validate_dims(const ldbp_dims* d) {
  if (!d) return fail(LDBP_EINVAL, "dims is NULL");
  if (d->reserved != 0) return fail(LDBP_EINVAL, "dims.reserved must be 0");
  if (d->flags & ~(uint32_t)(LDBP_SYMMETRIC | LDBP_PRECISE | LDBP_CHECK_FINITE | LDBP_STREAM_PIPELINE))
    return fail(LDBP_EINVAL, "unknown flag bits 0x%x", d->flags);
  if (d->batch < 0) return fail(LDBP_ESHAPE, "batch %lld < 0", (long long)d->batch);
  if (d->n < 1) return fail(LDBP_ESHAPE, "n %lld < 1", (long long)d->n);
  if (d->steps < 1) return fail(LDBP_ESHAPE, "steps %d < 1", d->steps);
  if (d->taps < 1 || (d->taps % 2) == 0) return fail(LDBP_ESHAPE, "taps %d must be odd and >= 1", d->taps);
  if (d->taps > LDBP_MAX_TAPS) return fail(LDBP_ESHAPE, "taps %d > LDBP_MAX_TAPS (%d)", d->taps, LDBP_MAX_TAPS);
  if (d->taps > d->n) return fail(LDBP_ESHAPE, "filter longer than block: taps %d > n %lld", d->taps, (long long)d->n);
  return LDBP_OK;
}

int check_ptr(const void* p, const char* name, size_t align) {
  if (!p) return fail(LDBP_EINVAL, "%s is NULL", name);
  if (((uintptr_t)p) % align) return fail(LDBP_EALIGN, "%s not %zu-byte aligned", name, align);
  return LDBP_OK;
}

#define LDBP_TRY(expr)          \
  do {                          \
    int _s = (expr);            \
    if (_s != LDBP_OK) return _s; \
  } while (0)

// ----------------------------------------------------------------------------------------
// Workspace layouts
// ----------------------------------------------------------------------------------------
struct FwdWs {
  size_t pingpong = 0;  // bytes of one [B][n] buffer (only when segs >= 2)
  size_t total = 0;
};

FwdWs fwd_ws(const ldbp_dims* d) {
  FwdWs w;
  const FwdPlan p = plan_fwd_segments(d->steps, (d->taps - 1) / 2);
  if (p.segs >= 2) w.pingpong = align256(sizeof(float2) * d->batch * d->n);
  w.total = w.pingpong + ((d->flags & LDBP_CHECK_FINITE) ? kCheckBytes : 0);
  return w;
}

constexpr int kReduceChunk = 512;  // CTAs per first-level reduction block

inline int reduce_chunks(int nblk) { return nblk > 2 * kReduceChunk ? (int)cdiv(nblk, kReduceChunk) : 0; }

struct BwdWs {
  size_t ck_off = 0, ck_each = 0;   // (K-1) checkpoints
  size_t g_off = 0, g_each = 0;     // 2 adjoint ping-pong buffers (when K >= 2)
  size_t part_off = 0, part_bytes = 0;
  size_t loss_off = 0, loss_bytes = 0;
  size_t part2_off = 0, loss2_off = 0;  // first-level reduction outputs (many CTAs)
  size_t total = 0;
};

BwdWs bwd_ws(const ldbp_dims* d, const BwdPlan& p) {
  BwdWs w;
  const size_t blk = align256(sizeof(float2) * d->batch * d->n);
  w.ck_off = 0;
  w.ck_each = blk;
  size_t off = blk * (p.K - 1);
  w.g_off = off;
  w.g_each = blk;
  off += (p.K >= 2) ? 2 * blk : 0;
  w.part_off = off;
  w.part_bytes = align256(sizeof(double) * (size_t)p.tile.grid * d->steps * p.V);
  off += w.part_bytes;
  w.loss_off = off;
  w.loss_bytes = align256(sizeof(double) * (size_t)p.tile.grid);
  off += w.loss_bytes;
  const int nch = reduce_chunks(p.tile.grid);
  w.part2_off = off;
  off += align256(sizeof(double) * (size_t)nch * d->steps * p.V);
  w.loss2_off = off;
  off += align256(sizeof(double) * (size_t)nch);
  w.total = off;
  return w;
}

struct RevWs {
  size_t act_off = 0, act_each = 0;  // M activation buffers u_hat^(1..M)
  size_t g_off = 0, g_each = 0;      // 2 adjoint ping-pong buffers (when Kr >= 2)
  size_t part_off = 0, loss_off = 0, part2_off = 0, loss2_off = 0;
  size_t ptab_off = 0;               // parameter table (params_kernel)
  size_t total = 0;
};

RevWs rev_ws(const ldbp_dims* d, const RevPlan& p) {
  RevWs w;
  const size_t blk = align256(sizeof(float2) * d->batch * d->n);
  w.act_off = 0;
  w.act_each = blk;
  size_t off = blk * d->steps;
  w.g_off = off;
  w.g_each = blk;
  off += (p.Kr >= 2) ? 2 * blk : 0;
  w.part_off = off;
  off += align256(sizeof(double) * (size_t)p.tile.grid * d->steps * p.V);
  w.loss_off = off;
  off += align256(sizeof(double) * (size_t)p.tile.grid);
  const int nch = reduce_chunks(p.tile.grid);
  w.part2_off = off;
  off += align256(sizeof(double) * (size_t)nch * d->steps * p.V);
  w.loss2_off = off;
  off += align256(sizeof(double) * (size_t)nch);
  w.ptab_off = off;
  off += align256(ldbp::ptab_bytes(d->steps, ntaps_used((d->taps - 1) / 2, d->flags & LDBP_SYMMETRIC)));
  if (d->flags & LDBP_CHECK_FINITE) off += kCheckBytes;  // the check slot (last 256 bytes)
  w.total = off;
  return w;
}

// LDBP_CHECK_FINITE: arm the slot (the last kCheckBytes of the workspace) before the launches, then
// read it back (one stream synchronisation) and report the first non-finite step.
struct FiniteCheck {
  int* slot = nullptr;
  FiniteCheck(const ldbp_dims* d, void* ws, size_t total, cudaStream_t st) {
    if (!(d->flags & LDBP_CHECK_FINITE) || !ws) return;
    slot = reinterpret_cast<int*>((unsigned char*)ws + total - kCheckBytes);
    cudaMemsetAsync(slot, 0x7f, sizeof(int), st);
    g_nonfinite = slot;
  }
  ~FiniteCheck() { g_nonfinite = nullptr; }
  int finish(int status, cudaStream_t st) {
    g_nonfinite = nullptr;
    if (!slot || status != LDBP_OK) return status;
    int v = kFiniteInit;
    if (cudaMemcpyAsync(&v, slot, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      return fail(LDBP_ECUDA, "finite check: %s", cudaGetErrorString(cudaGetLastError()));
    if (v != kFiniteInit) return fail(LDBP_ENONFINITE, "non-finite activation after step %d (1-based)", v);
    return LDBP_OK;
  }
};

// ----------------------------------------------------------------------------------------
// Launch helpers
// ----------------------------------------------------------------------------------------
// cuTensorMapEncodeTiled through the runtime's driver entry point (no link-time libcuda
// dependency); nullptr when the driver does not provide it (the lane-store path is used).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encode_fn() {
  static const PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    cudaGetLastError();
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// Tensor map of the storing forward's activation slots (LDBP_FWD_TMA, ldbp_kernels.cuh): rows of
// 16 complex64 samples (128 bytes) over ckpt[0, rows * 16), box 32 rows, 128-byte swizzle.
bool make_act_tmap(CUtensorMap* m, float2* ckpt, int64_t rows) {
  const PFN_cuTensorMapEncodeTiled_v12000 enc = tmap_encode_fn();
  if (!enc || rows <= 0 || rows > (int64_t)0x7fffffff || (reinterpret_cast<uintptr_t>(ckpt) & 15)) return false;
  const cuuint64_t dims[2] = {16, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {128};
  const cuuint32_t box[2] = {16, 32};
  const cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, ckpt, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int launch_fwd(const ldbp_dims* d, const float2* src, float2* dst, const float2* taps, const float* gamma,
               const uint8_t* mask, int s0, int s1, cudaStream_t st, float2* ckpt = nullptr, int ckpt_every = 0,
               int64_t ckpt_stride = 0, bool global_norm = false, bool scale_dst = false, float2* y_out = nullptr,
               const void* ptab = nullptr, bool pdl = false) {
  const int kh = (d->taps - 1) / 2;
  const bool sym = d->flags & LDBP_SYMMETRIC;
  const bool fast = !(d->flags & LDBP_PRECISE);
  const bool staged = global_norm && ckpt && ckpt_every == 1 && fast && env_int("LDBP_FWD_STAGED", 1);
  Tile t = plan_fwd_tile(d, s1 - s0, true, staged);
  if (global_norm) t.smem = fwd_smem(kh, sym, s1 - s0, t.nthreads, d->steps, staged);
  const bool chk = g_nonfinite != nullptr;
  FwdFn fn = staged ? get_fwd_store(kh, sym, chk) : get_fwd(kh, sym, fast, chk);
  ldbp::FwdArgs a;
  a.src = src;
  a.dst = dst;
  a.ckpt = ckpt;
  a.y_out = y_out;
  a.nonfinite = g_nonfinite;
  a.ptab = global_norm ? ptab : nullptr;
  a.ckpt_stride = ckpt_stride;
  a.ckpt_every = ckpt_every > 0 ? ckpt_every : 1;
  a.taps = taps;
  a.gamma = gamma;
  a.mask = mask;
  a.T = d->taps;
  a.s0 = s0;
  a.s1 = s1;
  a.n0 = global_norm ? 0 : s0;
  a.nM = global_norm ? d->steps : s1;
  a.global_norm = global_norm ? 1 : 0;
  a.scale_dst = scale_dst ? 1 : 0;
  a.staged = staged ? 1 : 0;
  a.g = t.g;
  a.use_tmap = 0;
  // TMA activation stores where the storing forward is FP32-bound (Kh >= 2; measured C3, Kh = 4: 0.767 ->
  // 0.731 ms); at Kh = 1 it is bound by the HBM writes and the TMA path measured slower (C5: 9.4 ->
  // 13.1 ms).  LDBP_FWD_TMA = 0 never, 2 always.
  const int tma_mode = env_int("LDBP_FWD_TMA", 1);
  if (staged && kFwdR == 16 && ckpt && ckpt_stride % 16 == 0 && s1 >= 2 && (tma_mode == 2 || (tma_mode == 1 && kh >= 2)))
    a.use_tmap = make_act_tmap(&a.tmap, ckpt, (int64_t)(s1 - 1) * ckpt_stride / 16) ? 1 : 0;
  cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t.smem);
  {
    TraceScope ts(LDBP_K_FORWARD, s1 - s0, d->batch * d->n, st);
    if (pdl && !g_trace_on && !chk) {
      // LDBP_STREAM_PIPELINE: programmatic dependent launch; the kernel never waits on the previous
      // grid (the caller guarantees independence), it only lets the next one start early
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(t.grid);
      cfg.blockDim = dim3(t.nthreads);
      cfg.dynamicSmemBytes = t.smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, fn, a);
    } else {
      fn<<<t.grid, t.nthreads, t.smem, st>>>(a);
    }
  }
  return cuda_check("fwd_tile_kernel launch");
}

// Full multi-launch forward from src to dst over steps [0, M) using pp as ping-pong buffer.
int run_forward_chain(const ldbp_dims* d, const float2* x, float2* y, const float2* taps, const float* gamma,
                      const uint8_t* mask, float2* pp, cudaStream_t st) {
  const FwdPlan p = plan_fwd_segments(d->steps, (d->taps - 1) / 2);
  // LDBP_STREAM_PIPELINE applies to one-launch forwards only (a multi-launch chain shares its ping-pong
  // buffer with the previous call's chain)
  const bool pdl = (d->flags & LDBP_STREAM_PIPELINE) && p.segs == 1 && env_int("LDBP_PDL", 1);
  const float2* src = x;
  for (int k = 0; k < p.segs; ++k) {
    const int s0 = k * p.steps_per, s1 = std::min(d->steps, s0 + p.steps_per);
    // the last launch writes y; earlier ones alternate so that happens
    const int remaining = p.segs - 1 - k;
    float2* dst = (remaining % 2 == 0) ? y : pp;
    LDBP_TRY(launch_fwd(d, src, dst, taps, gamma, mask, s0, s1, st, nullptr, 0, 0, false, false, nullptr, nullptr,
                        pdl));
    src = dst;
  }
  return LDBP_OK;
}

int run_reduce(const ldbp_dims* d, double* partials, double* lossp, int nblk, int V, unsigned char* part2,
               unsigned char* loss2, const uint8_t* mask, cudaStream_t st, double* buf, double* dtaps,
               double* dgamma);

// Backward over all segments. `gy` != nullptr: incoming gradient; else seed from target.
int run_backward_chain(const ldbp_dims* d, const float2* x, const float2* gy, const float2* target,
                       const float2* taps, const float* gamma, const uint8_t* mask, float2* gx,
                       unsigned char* ws, const BwdPlan& p, const BwdWs& w, cudaStream_t st,
                       double* buf, double* dtaps, double* dgamma) {
  const int kh = (d->taps - 1) / 2;
  const bool sym = d->flags & LDBP_SYMMETRIC;
  const bool fast = !(d->flags & LDBP_PRECISE);
  auto ck = [&](int k) -> float2* { return reinterpret_cast<float2*>(ws + w.ck_off + (size_t)(k - 1) * w.ck_each); };
  auto gb = [&](int k) -> float2* { return reinterpret_cast<float2*>(ws + w.g_off + (size_t)(k & 1) * w.g_each); };
  // forward checkpoint pass: ck[k] = u^(k*C), k = 1..K-1.  Each launch covers G segments
  // (halo G*C*Kh, bounded by plan_fwd_segments) and writes the intermediate checkpoints on the
  // fly, so the input is read once per launch instead of once per segment.
  if (p.K > 1) {
    const FwdPlan fp = plan_fwd_segments((p.K - 1) * p.C, kh);
    const int G = std::max(1, fp.steps_per / p.C);
    for (int k0 = 0; k0 + 1 < p.K; k0 += G) {
      const int k1 = std::min(p.K - 1, k0 + G);  // this launch produces ck[k0+1 .. k1]
      // ck(k) for k >= 1 are consecutive buffers: ck(k0+1) + (j-1)*stride
      LDBP_TRY(launch_fwd(d, k0 == 0 ? x : ck(k0), ck(k1), taps, gamma, mask, k0 * p.C, k1 * p.C, st,
                          k1 - k0 >= 2 ? ck(1) : nullptr, p.C, (int64_t)(w.ck_each / sizeof(float2))));
    }
  }
  BwdFn fn = get_bwd(kh, sym, fast);
  double* partials = reinterpret_cast<double*>(ws + w.part_off);
  double* lossp = reinterpret_cast<double*>(ws + w.loss_off);
  for (int k = p.K - 1; k >= 0; --k) {
    const int s0 = k * p.C, s1 = std::min(d->steps, (k + 1) * p.C);
    ldbp::BwdArgs a;
    a.ck = k == 0 ? x : ck(k);
    a.gin = (k == p.K - 1) ? gy : gb(k + 1);
    a.target = target;
    a.gout = (k == 0) ? gx : gb(k);
    a.taps = taps;
    a.gamma = gamma;
    a.mask = mask;
    a.partials = partials;
    a.loss_partials = lossp;
    a.seed_scale = 2.0f;
    a.T = d->taps;
    a.M = d->steps;
    a.s0 = s0;
    a.s1 = s1;
    a.g = p.tile.g;
    const size_t smem = bwd_smem(kh, sym, s1 - s0, p.tile.nthreads);
    cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    {
      TraceScope ts(LDBP_K_BACKWARD, s1 - s0, d->batch * d->n, st);
      // programmatic dependent launch: this segment's prologue overlaps the previous kernel's tail
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(p.tile.grid);
      cfg.blockDim = dim3(p.tile.nthreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = env_int("LDBP_PDL", 1) && !g_trace_on ? 1 : 0;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      cudaLaunchKernelEx(&cfg, fn, a);
    }
    LDBP_TRY(cuda_check("bwd_segment_kernel launch"));
  }
  return run_reduce(d, partials, gy ? nullptr : lossp, p.tile.grid, p.V, ws + w.part2_off, ws + w.loss2_off, mask,
                    st, buf, dtaps, dgamma);
}

// Deterministic two-level fp64 reduction of per-CTA partials into buf / (dtaps, dgamma).
int run_reduce(const ldbp_dims* d, double* partials, double* lossp, int nblk, int V, unsigned char* part2,
               unsigned char* loss2, const uint8_t* mask, cudaStream_t st, double* buf, double* dtaps,
               double* dgamma) {
  const int kh = (d->taps - 1) / 2;
  const bool sym = d->flags & LDBP_SYMMETRIC;
  ldbp::ReduceArgs r;
  r.partials = partials;
  r.loss_partials = lossp;
  r.nblk = nblk;
  const int nch = reduce_chunks(nblk);
  if (nch > 0) {
    ldbp::Reduce1Args r1;
    r1.partials = partials;
    r1.loss_partials = r.loss_partials;
    r1.nblk = nblk;
    r1.total = d->steps * V;
    r1.chunk = kReduceChunk;
    r1.out = reinterpret_cast<double*>(part2);
    r1.loss_out = reinterpret_cast<double*>(loss2);
    {
      TraceScope ts(LDBP_K_REDUCE, d->steps, 0, st);
      ldbp::reduce_partials_pass1<<<dim3((r1.total + 31) / 32 + 1, nch), 256, 0, st>>>(r1);
    }
    LDBP_TRY(cuda_check("reduce_partials_pass1 launch"));
    r.partials = r1.out;
    r.loss_partials = r.loss_partials ? r1.loss_out : nullptr;
    r.nblk = nch;
  }
  r.M = d->steps;
  r.T = d->taps;
  r.V = V;
  r.kh = kh;
  r.sym = sym ? 1 : 0;
  r.mask = mask;
  r.buf = buf;
  r.dtaps = dtaps;
  r.dgamma = dgamma;
  const int nblocks = (d->steps * V + 31) / 32 + 1;
  {
    TraceScope ts(LDBP_K_REDUCE, d->steps, 0, st);
    ldbp::reduce_partials_kernel<<<nblocks, 256, 0, st>>>(r);
  }
  return cuda_check("reduce_partials_kernel launch");
}

// Store-all training path: forward chain storing u_hat^(1..M) (global normalisation), then the
// reverse launches (last steps first), then the reduction.
// forward_only: run the storing forward (and y_out) and return; skip_forward: the activations are
// already in ws (a previous forward_only call on the same stream), run the reverse only.
int run_rev_chain(const ldbp_dims* d, const float2* x, const float2* gy, const float2* target, const float2* taps,
                  const float* gamma, const uint8_t* mask, float2* gx, unsigned char* ws, const RevPlan& p,
                  const RevWs& w, cudaStream_t st, double* buf, double* dtaps, double* dgamma,
                  float2* y_out = nullptr, bool forward_only = false, bool skip_forward = false) {
  const int kh = (d->taps - 1) / 2;
  const bool sym = d->flags & LDBP_SYMMETRIC;
  const bool fast = !(d->flags & LDBP_PRECISE);
  const int M = d->steps;
  auto act = [&](int i) -> float2* { return reinterpret_cast<float2*>(ws + w.act_off + (size_t)(i - 1) * w.act_each); };
  auto gb = [&](int k) -> float2* { return reinterpret_cast<float2*>(ws + w.g_off + (size_t)(k & 1) * w.g_each); };
  const int64_t stride = (int64_t)(w.act_each / sizeof(float2));
  // parameter table for every launch below (one tiny kernel; skip_forward recomputes it too)
  void* ptab = ws + w.ptab_off;
  {
    TraceScope ts(LDBP_K_REDUCE, M, 0, st);
    // LDBP_PARAMS_SMEM_STEPS (tests): longest model whose prefix chain runs in shared memory
    const int in_smem = M <= std::min(ldbp::kParamsSmemSteps, env_int("LDBP_PARAMS_SMEM_STEPS", 1 << 30)) ? 1 : 0;
    const size_t psm = in_smem ? 16 + sizeof(ldbp::StepNorm) * (size_t)M : 0;
    if (psm > 48 * 1024)
      cudaFuncSetAttribute((const void*)get_params(kh, sym), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm);
    get_params(kh, sym)<<<1, 256, psm, st>>>(taps, gamma, mask, d->taps, M, ptab, in_smem);
  }
  LDBP_TRY(cuda_check("params_kernel launch"));
  if (!skip_forward) {
    const FwdPlan fp = plan_fwd_segments(M, kh, kFwdR);  // store-all forward: R = LDBP_FWD_R
    for (int k = 0; k < fp.segs; ++k) {
      const int s0 = k * fp.steps_per, s1 = std::min(M, s0 + fp.steps_per);
      LDBP_TRY(launch_fwd(d, s0 == 0 ? x : act(s0), act(s1), taps, gamma, mask, s0, s1, st,
                          s1 - s0 >= 2 ? act(1) : nullptr, 1, stride, true, false, s1 == M ? y_out : nullptr,
                          ptab));
    }
  }
  if (forward_only) return LDBP_OK;
  RevFn fn = get_rev_any(d);
  double* partials = reinterpret_cast<double*>(ws + w.part_off);
  double* lossp = reinterpret_cast<double*>(ws + w.loss_off);
  for (int k = p.Kr - 1; k >= 0; --k) {
    const int s0 = k * p.Cr, s1 = std::min(M, (k + 1) * p.Cr);
    ldbp::RevArgs a{};
    a.x = x;
    a.act = act(1);
    a.act_stride = stride;
    a.gin = (k == p.Kr - 1) ? gy : gb(k + 1);
    a.target = target;
    a.gout = (k == 0) ? gx : gb(k);
    a.taps = taps;
    a.gamma = gamma;
    a.mask = mask;
    a.partials = partials;
    a.loss_partials = lossp;
    a.ptab = ptab;
    a.seed_scale = 2.0f;
    a.T = d->taps;
    a.M = M;
    a.s0 = s0;
    a.s1 = s1;
    a.g = p.tile.g;
    a.ntiles = p.tile.grid;  // persistent kernels (rev4) walk the tiles with a grid stride
    const size_t smem = rev_smem_any(d, s1 - s0);
    cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    {
      TraceScope ts(LDBP_K_REVERSE, s1 - s0, d->batch * d->n, st);
      fn<<<p.launch_grid > 0 ? p.launch_grid : p.tile.grid, p.tile.nthreads, smem, st>>>(a);
    }
    LDBP_TRY(cuda_check("rev_tile_kernel launch"));
  }
  return run_reduce(d, partials, gy ? nullptr : lossp, p.tile.grid, p.V, ws + w.part2_off, ws + w.loss2_off, mask,
                    st, buf, dtaps, dgamma);
}

// ---------------------------------------------------------------------------------------
// Overlapped store-all training step (loss_grad): the batch is cut into K chunks of whole blocks;
// the storing forwards run on a side stream and the reverse of chunk c starts as soon as forward
// c has finished, so the HBM-bound storing forward of chunk c + 1 runs concurrently with the
// latency-bound reverse of chunk c (CTAs of both kernels share the SMs).  Each chunk keeps its own
// workspace region and gradient buffer; a final fixed-order sum gives buf (deterministic).
// ---------------------------------------------------------------------------------------
struct OverlapPlan {
  int K = 1;          // chunks
  int64_t Bc = 0;     // blocks per chunk (last one may be shorter)
  size_t chunk_off[16] = {};
  size_t bufs_off = 0, buf_stride = 0, total = 0;
};

ldbp_dims chunk_dims(const ldbp_dims* d, const OverlapPlan& o, int c) {
  ldbp_dims dc = *d;
  const int64_t b0 = (int64_t)c * o.Bc;
  dc.batch = std::min(d->batch, b0 + o.Bc) - b0;
  return dc;
}

OverlapPlan plan_overlap(const ldbp_dims* d, bool query) {
  OverlapPlan o;
  // default 1 (no overlap): measured, the overlapped schedule is not faster (C3 2.73 ms at K = 1,
  // 3.02 at 2, 3.34 at 4; C5 23.2 / 23.2 / 23.7 ms): the storing forward and the reverse slow each
  // other down as much as they overlap, and each chunk adds prologues and a partial last wave
  int K = env_int("LDBP_OVERLAP", 1);
  if (d->flags & LDBP_CHECK_FINITE) K = 1;
  K = (int)std::max<int64_t>(1, std::min<int64_t>({(int64_t)K, d->batch, 16}));
  o.K = K;
  o.Bc = cdiv(d->batch, K);
  o.K = (int)cdiv(d->batch, o.Bc);
  size_t off = 0;
  for (int c = 0; c < o.K; ++c) {
    const ldbp_dims dc = chunk_dims(d, o, c);
    o.chunk_off[c] = off;
    off += align256(rev_ws(&dc, plan_rev(&dc, query)).total);
  }
  o.buf_stride = 1 + (size_t)d->steps + 2 * (size_t)d->steps * d->taps;
  o.bufs_off = off;
  off += align256(sizeof(double) * o.buf_stride * o.K);
  o.total = off;
  return o;
}

// Per-thread, per-device side stream and fork / join events (created on first use).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[17] = {};
};
thread_local SideStream g_side[16];

int side_stream(SideStream** out) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return fail(LDBP_ECUDA, "cudaGetDevice");
  SideStream& ss = g_side[dev];
  if (!ss.s) {
    if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess)
      return fail(LDBP_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(cudaGetLastError()));
    for (auto& e : ss.ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
        return fail(LDBP_ECUDA, "cudaEventCreate: %s", cudaGetErrorString(cudaGetLastError()));
  }
  *out = &ss;
  return LDBP_OK;
}

int run_overlapped(const ldbp_dims* d, const OverlapPlan& o, const float2* x, const float2* target,
                   const float2* taps, const float* gamma, const uint8_t* mask, unsigned char* ws, cudaStream_t st,
                   double* buf) {
  SideStream* ss = nullptr;
  LDBP_TRY(side_stream(&ss));
  double* bufs = reinterpret_cast<double*>(ws + o.bufs_off);
  if (cudaEventRecord(ss->ev[16], st) != cudaSuccess || cudaStreamWaitEvent(ss->s, ss->ev[16], 0) != cudaSuccess)
    return fail(LDBP_ECUDA, "fork: %s", cudaGetErrorString(cudaGetLastError()));
  for (int c = 0; c < o.K; ++c) {  // storing forwards, side stream
    const ldbp_dims dc = chunk_dims(d, o, c);
    const int64_t off = (int64_t)c * o.Bc * d->n;
    const RevPlan rp = plan_rev(&dc, true);
    const RevWs rw = rev_ws(&dc, rp);
    LDBP_TRY(run_rev_chain(&dc, x + off, nullptr, target + off, taps, gamma, mask, nullptr, ws + o.chunk_off[c], rp,
                           rw, ss->s, nullptr, nullptr, nullptr, nullptr, /*forward_only=*/true));
    if (cudaEventRecord(ss->ev[c], ss->s) != cudaSuccess) return fail(LDBP_ECUDA, "cudaEventRecord");
  }
  for (int c = 0; c < o.K; ++c) {  // reverses, caller's stream, each after its forward
    const ldbp_dims dc = chunk_dims(d, o, c);
    const int64_t off = (int64_t)c * o.Bc * d->n;
    const RevPlan rp = plan_rev(&dc, true);
    const RevWs rw = rev_ws(&dc, rp);
    if (cudaStreamWaitEvent(st, ss->ev[c], 0) != cudaSuccess) return fail(LDBP_ECUDA, "cudaStreamWaitEvent");
    LDBP_TRY(run_rev_chain(&dc, x + off, nullptr, target + off, taps, gamma, mask, nullptr, ws + o.chunk_off[c], rp,
                           rw, st, bufs + (size_t)c * o.buf_stride, nullptr, nullptr, nullptr, false,
                           /*skip_forward=*/true));
  }
  {
    TraceScope ts(LDBP_K_REDUCE, d->steps, 0, st);
    ldbp::sum_bufs_kernel<<<(unsigned)cdiv((int64_t)o.buf_stride, 256), 256, 0, st>>>(
        bufs, (int64_t)o.buf_stride, o.K, (int)o.buf_stride, buf);
  }
  return cuda_check("sum_bufs_kernel launch");
}

// ---------------------------------------------------------------------------------------
// Receiver-chain symbol loss (§8(f) NEXT-1), ldbp_rx.cuh
// ---------------------------------------------------------------------------------------
struct RxWs {
  size_t st_off = 0, part_off = 0, epart_off = 0, total = 0;
  int chunks = 0;
};

RxWs rx_ws(int64_t B, int64_t n, int sps) {
  RxWs w;
  const int64_t K = n / sps;
  w.chunks = (int)cdiv(K, ldbp::kRxChunk);
  w.st_off = 0;
  size_t off = align256(sizeof(float2) * (size_t)B * K);
  w.part_off = off;
  off += align256(sizeof(double) * 4 * (size_t)B * w.chunks);
  w.epart_off = off;
  off += align256(sizeof(double) * (size_t)B * w.chunks);
  w.total = off;
  return w;
}

size_t rx_smem(int sps, int L) {
  const int P = (L + sps - 1) / sps + 1;
  const int WN = ldbp::kRxChunk + 2 * (P + ldbp::kRxTB);
  return (size_t)ldbp::kRxTapBytes + sizeof(float2) * (size_t)sps * (WN + WN / 16 + 1);
}

int validate_rx(int64_t B, int64_t n, int sps, int L) {
  if (B < 0) return fail(LDBP_ESHAPE, "batch %lld < 0", (long long)B);
  if (sps < 1 || sps > ldbp::kRxMaxSps) return fail(LDBP_ESHAPE, "sps %d not in [1, %d]", sps, ldbp::kRxMaxSps);
  if (n < sps || n % sps) return fail(LDBP_ESHAPE, "n %lld must be a positive multiple of sps %d", (long long)n, sps);
  if (L < 0 || L > ldbp::kRxMaxL) return fail(LDBP_ESHAPE, "MF half-length %d not in [0, %d]", L, ldbp::kRxMaxL);
  if ((int64_t)(2 * L + 1) > n) return fail(LDBP_ESHAPE, "MF longer than the block: 2L+1 = %d > n", 2 * L + 1);
  return LDBP_OK;
}

int launch_rx(int64_t B, int64_t n, int sps, int L, const float2* y, const float2* sym, const float* pw,
              const float* h, double* errs, float2* gy, unsigned char* ws, cudaStream_t st, double* buf = nullptr) {
  const RxWs w = rx_ws(B, n, sps);
  ldbp::RxArgs a;
  a.y = y;
  a.sym = sym;
  a.power_w = pw;
  a.h = h;
  a.st = reinterpret_cast<float2*>(ws + w.st_off);
  a.part = reinterpret_cast<double*>(ws + w.part_off);
  a.epart = reinterpret_cast<double*>(ws + w.epart_off);
  a.gy = gy;
  a.errs = errs;
  a.n = n;
  a.K = (int)(n / sps);
  a.sps = sps;
  a.L = L;
  a.chunks = w.chunks;
  const size_t smem = rx_smem(sps, L);
  cudaFuncSetAttribute((const void*)ldbp::rx_mf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute((const void*)ldbp::rx_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const dim3 grid(w.chunks, (unsigned)B);
  {
    TraceScope ts(LDBP_K_RX, 1, B * n, st);
    ldbp::rx_mf_kernel<<<grid, ldbp::kRxThreads, smem, st>>>(a);
  }
  LDBP_TRY(cuda_check("rx_mf_kernel launch"));
  {
    TraceScope ts(LDBP_K_RX, 1, B * n, st);
    ldbp::rx_grad_kernel<<<grid, ldbp::kRxThreads, smem, st>>>(a);
  }
  LDBP_TRY(cuda_check("rx_grad_kernel launch"));
  {
    TraceScope ts(LDBP_K_RX, 1, 0, st);
    ldbp::rx_errs_kernel<<<1, 256, 0, st>>>(a.epart, B, w.chunks, errs, buf);
  }
  return cuda_check("rx_errs_kernel launch");
}

// ---------------------------------------------------------------------------------------
// ESSM (§8(f) NEXT-4), ldbp_essm.cuh: one launch per step, smem tiles
// ---------------------------------------------------------------------------------------
struct EssmWs {
  size_t act_off = 0, act_each = 0, g_off = 0, part_off = 0, total = 0;
  int tiles = 0, V = 0;
  int nch = 1;           // first-level reduction chunks per step
  size_t part1_off = 0;  // [M][nch][V] chunk totals
};

EssmWs essm_ws(const ldbp_dims* d, int kappa, bool train) {
  EssmWs w;
  w.tiles = (int)cdiv(d->n, ldbp::kEssmW);
  w.V = 2 + 2 * d->taps + 2 * kappa + 1;
  const size_t blk = align256(sizeof(float2) * (size_t)d->batch * d->n);
  w.act_each = blk;
  size_t off = 0;
  w.act_off = off;
  off += blk * (train ? (size_t)d->steps : 2);  // train: u^(1..M); forward: ping-pong
  w.g_off = off;
  if (train) off += 2 * blk;
  w.part_off = off;
  if (train) off += align256(sizeof(double) * (size_t)d->steps * w.tiles * d->batch * w.V);
  w.nch = (int)cdiv((int64_t)w.tiles * d->batch, ldbp::kEssmRedChunk);
  w.part1_off = off;
  if (train) off += align256(sizeof(double) * (size_t)d->steps * w.nch * w.V);
  w.total = off;
  return w;
}

size_t essm_smem(int T, int kappa, bool bwd) {
  using namespace ldbp;
  const int kh = (T - 1) / 2;
  const int W = kEssmW, S = kESlack;
  size_t s = sizeof(float2) * kEssmMaxT + sizeof(float) * (2 * essm_nj(kEssmMaxKappa) + 2);
  (void)kh;
  const int k8 = (kappa + 7) & ~7;  // halos padded to multiples of 8 (ldbp_essm.cuh, essm_k8)
  if (!bwd) {
    const int nu = W + 2 * (8 + k8), na = W + 2 * k8;
    return s + sizeof(float2) * (essm_pc_size(nu + S) + essm_pc_size(na + S)) + sizeof(float) * essm_pf_size(na + S);
  }
  const int nU = W + 2 * (16 + 2 * k8), nA = W + 2 * (8 + 2 * k8), nG = W + 2 * (8 + k8), nQ = W + 2 * 8;
  s += sizeof(float2) * (essm_pc_size(nU + S) + essm_pc_size(nA + S) + essm_pc_size(nG + S) + essm_pc_size(nQ + S));
  s += sizeof(float) * (essm_pf_size(nA + S) + 2 * essm_pf_size(nG + S));
  return s;
}

int validate_essm(const ldbp_dims* d, int kappa) {
  if (d->taps > ldbp::kEssmMaxT) return fail(LDBP_ESHAPE, "ESSM: taps %d > %d", d->taps, ldbp::kEssmMaxT);
  if (kappa < 0 || kappa > ldbp::kEssmMaxKappa) return fail(LDBP_ESHAPE, "kappa %d not in [0, %d]", kappa, ldbp::kEssmMaxKappa);
  if (2 * (int64_t)kappa + 1 > d->n) return fail(LDBP_ESHAPE, "eta longer than the block: 2kappa+1 > n");
  return LDBP_OK;
}

template <int KH>
const void* essm_kernel_kh(bool bwd, bool fast) {
  if (bwd) return fast ? (const void*)ldbp::essm_bwd_step_kernel<KH, true> : (const void*)ldbp::essm_bwd_step_kernel<KH, false>;
  return fast ? (const void*)ldbp::essm_fwd_step_kernel<KH, true> : (const void*)ldbp::essm_fwd_step_kernel<KH, false>;
}

const void* essm_kernel(int kh, bool bwd, bool fast) {
  switch (kh) {
    case 0: return essm_kernel_kh<0>(bwd, fast);
    case 1: return essm_kernel_kh<1>(bwd, fast);
    case 2: return essm_kernel_kh<2>(bwd, fast);
    case 3: return essm_kernel_kh<3>(bwd, fast);
    case 4: return essm_kernel_kh<4>(bwd, fast);
    case 5: return essm_kernel_kh<5>(bwd, fast);
    case 6: return essm_kernel_kh<6>(bwd, fast);
    default: return essm_kernel_kh<7>(bwd, fast);
  }
}

int launch_essm_step(const ldbp_dims* d, int kappa, bool bwd, int step, const float2* u, const float2* gin,
                     const float2* target, float2* out, const float2* taps, const float* gamma,
                     const float* eta, double* partials, cudaStream_t st) {
  ldbp::EssmArgs a;
  a.u = u;
  a.gin = gin;
  a.target = target;
  a.out = out;
  a.taps = taps + (int64_t)step * d->taps;
  a.eta = eta + (int64_t)step * (2 * kappa + 1);
  a.gamma = gamma;
  a.step = step;
  a.partials = partials;
  a.n = d->n;
  a.T = d->taps;
  a.kappa = kappa;
  a.tiles = (int)cdiv(d->n, ldbp::kEssmW);
  const bool fast = !(d->flags & LDBP_PRECISE);
  const size_t smem = essm_smem(d->taps, kappa, bwd);
  const dim3 grid(a.tiles, (unsigned)d->batch);
  const void* fn = essm_kernel((d->taps - 1) / 2, bwd, fast);
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  {
    TraceScope ts(LDBP_K_ESSM, 1, d->batch * d->n, st);
    void* args[] = {&a};
    cudaLaunchKernel(fn, grid, dim3(ldbp::kEssmThreads), args, smem, st);
  }
  return cuda_check(bwd ? "essm_bwd_step_kernel launch" : "essm_fwd_step_kernel launch");
}

int zero_outputs(double* p, size_t count, cudaStream_t st) {
  if (count && cudaMemsetAsync(p, 0, count * sizeof(double), st) != cudaSuccess)
    return fail(LDBP_ECUDA, "cudaMemsetAsync: %s", cudaGetErrorString(cudaGetLastError()));
  return LDBP_OK;
}

}  // namespace

// ==========================================================================================
// Exported C ABI
// ==========================================================================================
extern "C" {

int ldbp_abi_version(void) { return LDBP_ABI_VERSION; }

const char* ldbp_status_string(int s) {
  switch (s) {
    case LDBP_OK: return "LDBP_OK";
    case LDBP_EINVAL: return "LDBP_EINVAL: invalid argument";
    case LDBP_ESHAPE: return "LDBP_ESHAPE: unsupported or inconsistent shape";
    case LDBP_EALIGN: return "LDBP_EALIGN: misaligned pointer";
    case LDBP_EWORKSPACE: return "LDBP_EWORKSPACE: workspace too small";
    case LDBP_ECUDA: return "LDBP_ECUDA: CUDA runtime error";
    case LDBP_ENONFINITE: return "LDBP_ENONFINITE: non-finite activation";
  }
  return "LDBP: unknown status";
}

const char* ldbp_last_error(void) { return g_err; }

int ldbp_workspace_bytes(const ldbp_dims* d, int op, size_t* bytes) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  if (!bytes) return fail(LDBP_EINVAL, "bytes is NULL");
  if (d->batch == 0) { *bytes = 0; return LDBP_OK; }
  switch (op) {
    case LDBP_OP_FORWARD: *bytes = fwd_ws(d).total; return LDBP_OK;
    case LDBP_OP_BACKWARD:
    case LDBP_OP_LOSS_GRAD:
    case LDBP_OP_TRAIN_STEP: {
      if (use_store_all(d)) {
        const size_t single = rev_ws(d, plan_rev(d, true)).total;
        // loss_grad / train_step may run the overlapped chunked schedule (its own layout)
        *bytes = op == LDBP_OP_BACKWARD ? single : std::max(single, plan_overlap(d, true).total);
        return LDBP_OK;
      }
      BwdPlan p = plan_bwd(d, true);
      *bytes = bwd_ws(d, p).total;
      return LDBP_OK;
    }
  }
  return fail(LDBP_EINVAL, "unknown op %d", op);
}

int ldbp_launch_count(const ldbp_dims* d, int op, int* launches) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  if (!launches) return fail(LDBP_EINVAL, "launches is NULL");
  if (d->batch == 0) { *launches = (op == LDBP_OP_FORWARD) ? 0 : 1; return LDBP_OK; }
  if (op == LDBP_OP_FORWARD) { *launches = plan_fwd_segments(d->steps, (d->taps - 1) / 2).segs; return LDBP_OK; }
  if (op != LDBP_OP_BACKWARD && use_tiny(d)) { *launches = 1; return LDBP_OK; }  // fused (Adam included)
  if (use_store_all(d)) {
    const OverlapPlan o = plan_overlap(d, true);
    auto chain = [&](const ldbp_dims* dc, bool two_params) {
      const RevPlan rp = plan_rev(dc, true);
      return (two_params ? 2 : 1) /* params_kernel */ + plan_fwd_segments(dc->steps, (dc->taps - 1) / 2, kFwdR).segs +
             rp.Kr + 1 + (reduce_chunks(rp.tile.grid) > 0 ? 1 : 0);
    };
    int n = 0;
    if (op != LDBP_OP_BACKWARD && o.K > 1) {
      for (int c = 0; c < o.K; ++c) {
        const ldbp_dims dc = chunk_dims(d, o, c);
        n += chain(&dc, true);
      }
      n += 1;  // sum_bufs_kernel
    } else {
      n = chain(d, false);
    }
    if (op == LDBP_OP_TRAIN_STEP) n += 1;
    *launches = n;
    return LDBP_OK;
  }
  BwdPlan p = plan_bwd(d, true);
  int nf = 0;
  if (p.K > 1) {
    const FwdPlan fp = plan_fwd_segments((p.K - 1) * p.C, (d->taps - 1) / 2);
    const int G = std::max(1, fp.steps_per / p.C);
    nf = (int)cdiv(p.K - 1, G);
  }
  int n = nf + p.K + 1 + (reduce_chunks(p.tile.grid) > 0 ? 1 : 0);
  if (op == LDBP_OP_TRAIN_STEP) n += 1;
  *launches = n;
  return LDBP_OK;
}

int ldbp_forward(const ldbp_dims* d, const void* x, void* y, const void* taps, const float* gamma,
                 void* ws, size_t ws_bytes, void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  if (d->batch == 0) return LDBP_OK;
  LDBP_TRY(check_ptr(x, "x", 8));
  LDBP_TRY(check_ptr(y, "y", 8));
  LDBP_TRY(check_ptr(taps, "taps", 8));
  LDBP_TRY(check_ptr(gamma, "gamma", 4));
  if (x == y) return fail(LDBP_EINVAL, "y must not alias x");
  const FwdWs w = fwd_ws(d);
  if (w.total > 0) {
    if (!ws || ws_bytes < w.total) return fail(LDBP_EWORKSPACE, "forward needs %zu workspace bytes, got %zu", w.total, ws_bytes);
    LDBP_TRY(check_ptr(ws, "ws", 8));
  }
  FiniteCheck fc(d, ws, w.total, (cudaStream_t)cuda_stream);
  return fc.finish(run_forward_chain(d, (const float2*)x, (float2*)y, (const float2*)taps, gamma, nullptr,
                                     (float2*)ws, (cudaStream_t)cuda_stream),
                   (cudaStream_t)cuda_stream);
}

int ldbp_backward(const ldbp_dims* d, const void* x, const void* gy, const void* taps, const float* gamma,
                  double* dtaps, double* dgamma, void* gx_or_null, void* ws, size_t ws_bytes, void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(check_ptr(dtaps, "dtaps", 8));
  LDBP_TRY(check_ptr(dgamma, "dgamma", 8));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (d->batch == 0) {
    LDBP_TRY(zero_outputs(dtaps, (size_t)2 * d->steps * d->taps, st));
    return zero_outputs(dgamma, d->steps, st);
  }
  LDBP_TRY(check_ptr(x, "x", 8));
  LDBP_TRY(check_ptr(gy, "gy", 8));
  LDBP_TRY(check_ptr(taps, "taps", 8));
  LDBP_TRY(check_ptr(gamma, "gamma", 4));
  if (gx_or_null) LDBP_TRY(check_ptr(gx_or_null, "gx", 8));
  if (gx_or_null == x || gx_or_null == gy) return fail(LDBP_EINVAL, "gx must not alias x or gy");
  if (use_store_all(d)) {
    const RevPlan rp = plan_rev(d, true);
    const RevWs rw = rev_ws(d, rp);
    if (!ws || ws_bytes < rw.total)
      return fail(LDBP_EWORKSPACE, "backward needs %zu workspace bytes, got %zu", rw.total, ws_bytes);
    LDBP_TRY(check_ptr(ws, "ws", 16));
    FiniteCheck fc(d, ws, rw.total, st);
    return fc.finish(run_rev_chain(d, (const float2*)x, (const float2*)gy, nullptr, (const float2*)taps, gamma,
                                   nullptr, (float2*)gx_or_null, (unsigned char*)ws, rp, rw, st, nullptr, dtaps,
                                   dgamma),
                     st);
  }
  BwdPlan p = plan_bwd(d, true);
  BwdWs w = bwd_ws(d, p);
  if (!ws || ws_bytes < w.total) return fail(LDBP_EWORKSPACE, "backward needs %zu workspace bytes, got %zu", w.total, ws_bytes);
  LDBP_TRY(check_ptr(ws, "ws", 8));
  if (gx_or_null == nullptr && p.K == 1) { /* nothing to write besides partials */ }
  return run_backward_chain(d, (const float2*)x, (const float2*)gy, nullptr, (const float2*)taps, gamma, nullptr,
                            (float2*)gx_or_null, (unsigned char*)ws, p, w, st, nullptr, dtaps, dgamma);
}

// Adam arguments (validated) shared by ldbp_adam_update and the fused tiny training step.
int fill_adam(const ldbp_dims* d, const double* buf, double n_global, double* master, double* m, double* v, int64_t t,
              double lr, double b1, double b2, double eps, const uint8_t* mask, const uint8_t* glearn,
              void* taps_out, float* gamma_out, ldbp::AdamArgs* a) {
  LDBP_TRY(check_ptr(buf, "buf", 8));
  LDBP_TRY(check_ptr(master, "master", 8));
  LDBP_TRY(check_ptr(m, "m", 8));
  LDBP_TRY(check_ptr(v, "v", 8));
  LDBP_TRY(check_ptr(taps_out, "taps_out", 8));
  LDBP_TRY(check_ptr(gamma_out, "gamma_out", 4));
  if (!(n_global > 0)) return fail(LDBP_EINVAL, "n_global must be > 0");
  if (t < 1) return fail(LDBP_EINVAL, "t must be >= 1");
  if (!(lr > 0) || !(b1 >= 0 && b1 < 1) || !(b2 >= 0 && b2 < 1) || !(eps > 0))
    return fail(LDBP_EINVAL, "bad Adam hyper-parameters");
  a->buf = buf;
  a->inv_n = 1.0 / n_global;
  a->master = master;
  a->m = m;
  a->v = v;
  a->lr = lr;
  a->b1 = b1;
  a->b2 = b2;
  a->eps = eps;
  a->bc1 = 1.0 - pow(b1, (double)t);
  a->bc2 = 1.0 - pow(b2, (double)t);
  a->mask = mask;
  a->glearn = glearn;
  a->taps_out = (float2*)taps_out;
  a->gamma_out = gamma_out;
  a->M = d->steps;
  a->T = d->taps;
  return LDBP_OK;
}

int launch_tiny(const ldbp_dims* d, const float2* x, const float2* target, const float2* taps, const float* gamma,
                const uint8_t* mask, double* buf, const ldbp::AdamArgs* adam, cudaStream_t st) {
  const TinyPlan p = plan_tiny(d, tiny_cluster_cap(d));
  if (!p.ok) return fail(LDBP_EINVAL, "tiny_train_kernel: problem too large");
  ldbp::TinyArgs a;
  a.x = x;
  a.target = target;
  a.taps = taps;
  a.gamma = gamma;
  a.mask = mask;
  a.buf = buf;
  a.B = (int)d->batch;
  a.n = (int)d->n;
  a.M = d->steps;
  a.S = p.S;
  a.lenmax = p.lenmax;
  a.nrows = p.nrows;
  a.sym = (d->flags & LDBP_SYMMETRIC) ? 1 : 0;
  a.precise = (d->flags & LDBP_PRECISE) ? 1 : 0;
  a.seed_scale = 2.0f;
  a.do_adam = adam != nullptr;
  if (adam) a.adam = *adam;
  void (*kern)(const ldbp::TinyArgs) = tiny_kernel((d->taps - 1) / 2, a.precise != 0);
  cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
  if (p.C > 8) cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p.C);
  cfg.blockDim = dim3((unsigned)p.nthr);
  cfg.dynamicSmemBytes = p.smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = p.C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e;
  {
    TraceScope ts(LDBP_K_TINY, d->steps, d->batch * d->n, st);
    e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  if (e != cudaSuccess) return fail(LDBP_ECUDA, "tiny_train_kernel launch: %s", cudaGetErrorString(e));
  return cuda_check("tiny_train_kernel launch");
}

int ldbp_loss_grad(const ldbp_dims* d, const void* x, const void* target, const void* taps, const float* gamma,
                   const uint8_t* mask, double* buf, void* ws, size_t ws_bytes, void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(check_ptr(buf, "buf", 8));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (d->batch == 0) return zero_outputs(buf, (size_t)1 + d->steps + 2 * (size_t)d->steps * d->taps, st);
  LDBP_TRY(check_ptr(x, "x", 8));
  LDBP_TRY(check_ptr(target, "target", 8));
  LDBP_TRY(check_ptr(taps, "taps", 8));
  LDBP_TRY(check_ptr(gamma, "gamma", 4));
  if (use_tiny(d))
    return launch_tiny(d, (const float2*)x, (const float2*)target, (const float2*)taps, gamma, mask, buf, nullptr, st);
  if (use_store_all(d)) {
    const OverlapPlan o = plan_overlap(d, true);
    if (o.K > 1) {
      if (!ws || ws_bytes < o.total)
        return fail(LDBP_EWORKSPACE, "loss_grad needs %zu workspace bytes, got %zu", o.total, ws_bytes);
      LDBP_TRY(check_ptr(ws, "ws", 16));
      return run_overlapped(d, o, (const float2*)x, (const float2*)target, (const float2*)taps, gamma, mask,
                            (unsigned char*)ws, st, buf);
    }
    const RevPlan rp = plan_rev(d, true);
    const RevWs rw = rev_ws(d, rp);
    if (!ws || ws_bytes < rw.total)
      return fail(LDBP_EWORKSPACE, "loss_grad needs %zu workspace bytes, got %zu", rw.total, ws_bytes);
    LDBP_TRY(check_ptr(ws, "ws", 16));
    FiniteCheck fc(d, ws, rw.total, st);
    return fc.finish(run_rev_chain(d, (const float2*)x, nullptr, (const float2*)target, (const float2*)taps, gamma,
                                   mask, nullptr, (unsigned char*)ws, rp, rw, st, buf, nullptr, nullptr),
                     st);
  }
  BwdPlan p = plan_bwd(d, true);
  BwdWs w = bwd_ws(d, p);
  if (!ws || ws_bytes < w.total) return fail(LDBP_EWORKSPACE, "loss_grad needs %zu workspace bytes, got %zu", w.total, ws_bytes);
  LDBP_TRY(check_ptr(ws, "ws", 8));
  return run_backward_chain(d, (const float2*)x, nullptr, (const float2*)target, (const float2*)taps, gamma, mask,
                            nullptr, (unsigned char*)ws, p, w, st, buf, nullptr, nullptr);
}

int ldbp_adam_update(const ldbp_dims* d, const double* buf, double n_global, double* master, double* m, double* v,
                     int64_t t, double lr, double b1, double b2, double eps, const uint8_t* mask,
                     const uint8_t* glearn, void* taps_out, float* gamma_out, void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  ldbp::AdamArgs a;
  LDBP_TRY(fill_adam(d, buf, n_global, master, m, v, t, lr, b1, b2, eps, mask, glearn, taps_out, gamma_out, &a));
  const int total = 2 * d->steps * d->taps + d->steps;
  {
    TraceScope ts(LDBP_K_ADAM, d->steps, 0, (cudaStream_t)cuda_stream);
    ldbp::adam_kernel<<<(total + 255) / 256, 256, 0, (cudaStream_t)cuda_stream>>>(a);
  }
  return cuda_check("adam_kernel launch");
}

int ldbp_train_step(const ldbp_dims* d, const void* x, const void* target, void* taps_work, float* gamma_work,
                    double* master, double* m, double* v, int64_t t, double lr, double b1, double b2, double eps,
                    const uint8_t* mask, const uint8_t* glearn, double* buf, void* ws, size_t ws_bytes,
                    void* cuda_stream) {
  if (d && validate_dims(d) == LDBP_OK && d->batch > 0 && use_tiny(d)) {  // one launch: loss, gradient, Adam
    g_err[0] = 0;
    LDBP_TRY(check_ptr(x, "x", 8));
    LDBP_TRY(check_ptr(target, "target", 8));
    LDBP_TRY(check_ptr(taps_work, "taps", 8));
    LDBP_TRY(check_ptr(gamma_work, "gamma", 4));
    ldbp::AdamArgs a;
    LDBP_TRY(fill_adam(d, buf, (double)d->batch * (double)d->n, master, m, v, t, lr, b1, b2, eps, mask, glearn,
                       taps_work, gamma_work, &a));
    return launch_tiny(d, (const float2*)x, (const float2*)target, (const float2*)taps_work, gamma_work, mask, buf,
                       &a, (cudaStream_t)cuda_stream);
  }
  LDBP_TRY(ldbp_loss_grad(d, x, target, taps_work, gamma_work, mask, buf, ws, ws_bytes, cuda_stream));
  const double n_global = (double)d->batch * (double)d->n;
  if (d->batch == 0) return LDBP_OK;
  return ldbp_adam_update(d, buf, n_global, master, m, v, t, lr, b1, b2, eps, mask, glearn, taps_work, gamma_work,
                          cuda_stream);
}

int ldbp_rx_workspace_bytes(int64_t batch, int64_t n, int32_t sps, size_t* bytes) {
  g_err[0] = 0;
  LDBP_TRY(validate_rx(batch, n, sps, 0));
  if (!bytes) return fail(LDBP_EINVAL, "bytes is NULL");
  *bytes = batch == 0 ? 0 : rx_ws(batch, n, sps).total;
  return LDBP_OK;
}

int ldbp_rx_loss_grad(int64_t batch, int64_t n, int32_t sps, int32_t mf_half, const void* y, const void* symbols,
                      const float* power_w, const float* h_mf, double* errs, void* gy_or_null, void* ws,
                      size_t ws_bytes, void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_rx(batch, n, sps, mf_half));
  if (batch == 0) return LDBP_OK;
  LDBP_TRY(check_ptr(y, "y", 8));
  LDBP_TRY(check_ptr(symbols, "symbols", 8));
  LDBP_TRY(check_ptr(power_w, "power_w", 4));
  LDBP_TRY(check_ptr(h_mf, "h_mf", 4));
  LDBP_TRY(check_ptr(errs, "errs", 8));
  if (gy_or_null) {
    LDBP_TRY(check_ptr(gy_or_null, "gy", 8));
    if (gy_or_null == y) return fail(LDBP_EINVAL, "gy must not alias y");
  }
  const RxWs w = rx_ws(batch, n, sps);
  if (!ws || ws_bytes < w.total) return fail(LDBP_EWORKSPACE, "rx needs %zu workspace bytes, got %zu", w.total, ws_bytes);
  LDBP_TRY(check_ptr(ws, "ws", 16));
  return launch_rx(batch, n, sps, mf_half, (const float2*)y, (const float2*)symbols, power_w, h_mf, errs,
                   (float2*)gy_or_null, (unsigned char*)ws, (cudaStream_t)cuda_stream);
}

}  // extern "C"

namespace {
struct RxTrainWs {
  bool store_all = false;
  size_t train_off = 0, y_off = 0, gy_off = 0, rx_off = 0, errs_off = 0, pp_off = 0, total = 0;
};

RxTrainWs rx_train_ws(const ldbp_dims* d, int sps, bool query) {
  RxTrainWs w;
  w.store_all = use_store_all(d);
  size_t off = 0;
  if (w.store_all) {
    off = rev_ws(d, plan_rev(d, query)).total;
  } else {
    off = bwd_ws(d, plan_bwd(d, query)).total;
    w.pp_off = off;
    off += align256(fwd_ws(d).total);
  }
  const size_t blk = align256(sizeof(float2) * (size_t)d->batch * d->n);
  w.y_off = off;
  off += blk;
  w.gy_off = off;
  off += blk;
  w.rx_off = off;
  off += rx_ws(d->batch, d->n, sps).total;
  w.errs_off = off;
  off += align256(sizeof(double) * (size_t)d->batch);
  w.total = off;
  return w;
}
}  // namespace

extern "C" {

int ldbp_rx_train_workspace_bytes(const ldbp_dims* d, int32_t sps, size_t* bytes) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(validate_rx(d->batch, d->n, sps, 0));
  if (!bytes) return fail(LDBP_EINVAL, "bytes is NULL");
  *bytes = d->batch == 0 ? 0 : rx_train_ws(d, sps, true).total;
  return LDBP_OK;
}

int ldbp_rx_train_grad(const ldbp_dims* d, const void* x, const void* symbols, const float* power_w, int32_t sps,
                       int32_t mf_half, const float* h_mf, const void* taps, const float* gamma, const uint8_t* mask,
                       double* buf, void* ws, size_t ws_bytes, void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(validate_rx(d->batch, d->n, sps, mf_half));
  LDBP_TRY(check_ptr(buf, "buf", 8));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (d->batch == 0) return zero_outputs(buf, (size_t)1 + d->steps + 2 * (size_t)d->steps * d->taps, st);
  LDBP_TRY(check_ptr(x, "x", 8));
  LDBP_TRY(check_ptr(symbols, "symbols", 8));
  LDBP_TRY(check_ptr(power_w, "power_w", 4));
  LDBP_TRY(check_ptr(h_mf, "h_mf", 4));
  LDBP_TRY(check_ptr(taps, "taps", 8));
  LDBP_TRY(check_ptr(gamma, "gamma", 4));
  const RxTrainWs w = rx_train_ws(d, sps, true);
  if (!ws || ws_bytes < w.total)
    return fail(LDBP_EWORKSPACE, "rx_train_grad needs %zu workspace bytes, got %zu", w.total, ws_bytes);
  LDBP_TRY(check_ptr(ws, "ws", 16));
  unsigned char* wb = (unsigned char*)ws;
  float2* ybuf = reinterpret_cast<float2*>(wb + w.y_off);
  float2* gybuf = reinterpret_cast<float2*>(wb + w.gy_off);
  double* errs = reinterpret_cast<double*>(wb + w.errs_off);
  if (w.store_all) {
    const RevPlan rp = plan_rev(d, true);
    const RevWs rw = rev_ws(d, rp);
    FiniteCheck fc(d, ws, rw.total, st);
    LDBP_TRY(fc.finish(run_rev_chain(d, (const float2*)x, nullptr, nullptr, (const float2*)taps, gamma, mask, nullptr,
                                     wb, rp, rw, st, nullptr, nullptr, nullptr, ybuf, /*forward_only=*/true),
                       st));
    LDBP_TRY(launch_rx(d->batch, d->n, sps, mf_half, ybuf, (const float2*)symbols, power_w, h_mf, errs, gybuf,
                       wb + w.rx_off, st));
    LDBP_TRY(run_rev_chain(d, (const float2*)x, gybuf, nullptr, (const float2*)taps, gamma, mask, nullptr, wb, rp, rw,
                           st, buf, nullptr, nullptr, nullptr, false, /*skip_forward=*/true));
  } else {
    const BwdPlan bp = plan_bwd(d, true);
    const BwdWs bw = bwd_ws(d, bp);
    LDBP_TRY(run_forward_chain(d, (const float2*)x, ybuf, (const float2*)taps, gamma, mask,
                               reinterpret_cast<float2*>(wb + w.pp_off), st));
    LDBP_TRY(launch_rx(d->batch, d->n, sps, mf_half, ybuf, (const float2*)symbols, power_w, h_mf, errs, gybuf,
                       wb + w.rx_off, st));
    LDBP_TRY(run_backward_chain(d, (const float2*)x, gybuf, nullptr, (const float2*)taps, gamma, mask, nullptr, wb, bp,
                                bw, st, buf, nullptr, nullptr));
  }
  // buf[0] = sum_b errs_b (the reduction above wrote 0 there: no target-seeded loss)
  const RxWs rw2 = rx_ws(d->batch, d->n, sps);
  ldbp::rx_errs_kernel<<<1, 256, 0, st>>>(reinterpret_cast<double*>(wb + w.rx_off + rw2.epart_off), d->batch,
                                          rw2.chunks, errs, buf);
  return cuda_check("rx_errs_kernel launch");
}

// ---- exact circulant matched filter (ldbp_rx_exact.cuh) ----
static int validate_rx_exact(int64_t B, int64_t n, int sps, float rolloff) {
  if (B < 0) return fail(LDBP_ESHAPE, "batch %lld < 0", (long long)B);
  if (n < 2 || (n & (n - 1)) || n > (1 << ldbp::kSsfmMaxLog2))
    return fail(LDBP_ESHAPE, "n %lld must be a power of two in [2, %d]", (long long)n, 1 << ldbp::kSsfmMaxLog2);
  if (sps < 1 || sps > kRxMaxSpsExact || n % sps) return fail(LDBP_ESHAPE, "sps %d must divide n, 1 <= sps <= 4", sps);
  if (!(rolloff > 0.f && rolloff <= 1.f)) return fail(LDBP_EINVAL, "rolloff %g not in (0, 1]", (double)rolloff);
  return LDBP_OK;
}

static int launch_rx_exact(int64_t B, int64_t n, int sps, float rolloff, const float2* y, const float2* sym,
                           const float* pw, const float* weights, double* errs, float2* gy, cudaStream_t st) {
  const int C = n > (1 << ldbp::kSsfmLocalMaxLog2) ? (int)(n >> ldbp::kSsfmLocalMaxLog2) : 1;
  const int64_t L = n / C;
  ldbp::RxExactArgs a;
  a.y = y;
  a.sym = sym;
  a.power_w = pw;
  a.weights = weights;
  a.gy = gy;
  a.errs = errs;
  a.n = n;
  a.K = (int)(n / sps);
  a.sps = sps;
  a.log2L = 0;
  while ((int64_t(1) << a.log2L) < L) ++a.log2L;
  a.rolloff = rolloff;
  const size_t smem = sizeof(float2) * ((size_t)L + L / 16 + 1 + L / 2 + (C > 1 ? (size_t)n / 64 + 64 : 0) + 1) +
                      sizeof(double) * (32 * 4 + 4);
  void (*kern)(const ldbp::RxExactArgs) = C == 1 ? ldbp::rx_exact_kernel<1>
                                          : C == 2 ? ldbp::rx_exact_kernel<2> : ldbp::rx_exact_kernel<4>;
  cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(B * C));
  cfg.blockDim = dim3(ldbp::kSsfmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  cudaError_t e;
  {
    TraceScope ts(LDBP_K_RX, 0, B * n, st);
    e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  if (e != cudaSuccess) return fail(LDBP_ECUDA, "rx_exact_kernel launch: %s", cudaGetErrorString(e));
  return cuda_check("rx_exact_kernel launch");
}

int ldbp_rx_exact_loss_grad(int64_t batch, int64_t n, int32_t sps, float rolloff, const void* y, const void* symbols,
                            const float* power_w, const float* weights_or_null, double* errs, void* gy_or_null,
                            void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_rx_exact(batch, n, sps, rolloff));
  if (batch == 0) return LDBP_OK;
  LDBP_TRY(check_ptr(y, "y", 8));
  LDBP_TRY(check_ptr(symbols, "symbols", 8));
  LDBP_TRY(check_ptr(power_w, "power_w", 4));
  LDBP_TRY(check_ptr(errs, "errs", 8));
  if (weights_or_null) LDBP_TRY(check_ptr(weights_or_null, "weights", 4));
  if (gy_or_null) {
    LDBP_TRY(check_ptr(gy_or_null, "gy", 8));
    if (gy_or_null == y) return fail(LDBP_EINVAL, "gy aliases y");
  }
  return launch_rx_exact(batch, n, sps, rolloff, (const float2*)y, (const float2*)symbols, power_w, weights_or_null,
                         errs, (float2*)gy_or_null, (cudaStream_t)cuda_stream);
}

int ldbp_tx_waveform(int64_t batch, int64_t n, int32_t sps, float rolloff, const uint8_t* codes,
                     const void* constellation, int32_t q, const float* power_w, const int32_t* shift_or_null,
                     const float* phase_or_null, void* out, void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_rx_exact(batch, n, sps, rolloff));
  if (q < 1 || q > 256) return fail(LDBP_EINVAL, "constellation size %d not in [1, 256]", q);
  if (batch == 0) return LDBP_OK;
  LDBP_TRY(check_ptr(codes, "codes", 1));
  LDBP_TRY(check_ptr(constellation, "constellation", 8));
  LDBP_TRY(check_ptr(power_w, "power_w", 4));
  LDBP_TRY(check_ptr(out, "out", 8));
  if (shift_or_null) LDBP_TRY(check_ptr(shift_or_null, "shift", 4));
  if (phase_or_null) LDBP_TRY(check_ptr(phase_or_null, "phase", 4));
  const int C = n > (1 << ldbp::kSsfmLocalMaxLog2) ? (int)(n >> ldbp::kSsfmLocalMaxLog2) : 1;
  const int64_t L = n / C;
  ldbp::TxArgs a;
  a.codes = codes;
  a.constel = (const float2*)constellation;
  a.power_w = power_w;
  a.shift = shift_or_null;
  a.phase = phase_or_null;
  a.out = (float2*)out;
  a.n = n;
  a.K = (int)(n / sps);
  a.sps = sps;
  a.Q = q;
  a.log2L = 0;
  while ((int64_t(1) << a.log2L) < L) ++a.log2L;
  a.rolloff = rolloff;
  const size_t smem = sizeof(float2) * ((size_t)L + L / 16 + 1 + L / 2 + (C > 1 ? (size_t)n / 64 + 64 : 0) + 1);
  void (*kern)(const ldbp::TxArgs) = C == 1 ? ldbp::tx_waveform_kernel<1>
                                     : C == 2 ? ldbp::tx_waveform_kernel<2> : ldbp::tx_waveform_kernel<4>;
  cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * C));
  cfg.blockDim = dim3(ldbp::kSsfmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = (cudaStream_t)cuda_stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  cudaError_t e;
  {
    TraceScope ts(LDBP_K_RX, 0, batch * n, (cudaStream_t)cuda_stream);
    e = cudaLaunchKernelEx(&cfg, kern, a);
  }
  if (e != cudaSuccess) return fail(LDBP_ECUDA, "tx_waveform_kernel launch: %s", cudaGetErrorString(e));
  return cuda_check("tx_waveform_kernel launch");
}

struct RxExTrainWs {
  bool store_all = false;
  size_t y_off = 0, gy_off = 0, errs_off = 0, pp_off = 0, total = 0;
};
static RxExTrainWs rx_exact_train_ws(const ldbp_dims* d, bool query) {
  RxExTrainWs w;
  w.store_all = use_store_all(d);
  size_t off = 0;
  if (w.store_all) {
    off = rev_ws(d, plan_rev(d, query)).total;
  } else {
    off = bwd_ws(d, plan_bwd(d, query)).total;
    w.pp_off = off;
    off += align256(fwd_ws(d).total);
  }
  const size_t blk = align256(sizeof(float2) * (size_t)d->batch * d->n);
  w.y_off = off;
  off += blk;
  w.gy_off = off;
  off += blk;
  w.errs_off = off;
  off += align256(sizeof(double) * (size_t)d->batch);
  w.total = off;
  return w;
}

int ldbp_rx_exact_train_workspace_bytes(const ldbp_dims* d, int32_t sps, size_t* bytes) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(validate_rx_exact(d->batch, d->n, sps, 0.1f));
  if (!bytes) return fail(LDBP_EINVAL, "bytes is NULL");
  *bytes = d->batch == 0 ? 0 : rx_exact_train_ws(d, true).total;
  return LDBP_OK;
}

int ldbp_rx_exact_train_grad(const ldbp_dims* d, const void* x, const void* symbols, const float* power_w,
                             const float* weights_or_null, int32_t sps, float rolloff, const void* taps,
                             const float* gamma, const uint8_t* mask, double* buf, void* ws, size_t ws_bytes,
                             void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(validate_rx_exact(d->batch, d->n, sps, rolloff));
  LDBP_TRY(check_ptr(buf, "buf", 8));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  if (d->batch == 0) return zero_outputs(buf, (size_t)1 + d->steps + 2 * (size_t)d->steps * d->taps, st);
  LDBP_TRY(check_ptr(x, "x", 8));
  LDBP_TRY(check_ptr(symbols, "symbols", 8));
  LDBP_TRY(check_ptr(power_w, "power_w", 4));
  if (weights_or_null) LDBP_TRY(check_ptr(weights_or_null, "weights", 4));
  LDBP_TRY(check_ptr(taps, "taps", 8));
  LDBP_TRY(check_ptr(gamma, "gamma", 4));
  const RxExTrainWs w = rx_exact_train_ws(d, true);
  if (!ws || ws_bytes < w.total)
    return fail(LDBP_EWORKSPACE, "rx_exact_train_grad needs %zu workspace bytes, got %zu", w.total, ws_bytes);
  LDBP_TRY(check_ptr(ws, "ws", 16));
  unsigned char* wb = (unsigned char*)ws;
  float2* ybuf = reinterpret_cast<float2*>(wb + w.y_off);
  float2* gybuf = reinterpret_cast<float2*>(wb + w.gy_off);
  double* errs = reinterpret_cast<double*>(wb + w.errs_off);
  if (w.store_all) {
    const RevPlan rp = plan_rev(d, true);
    const RevWs rw = rev_ws(d, rp);
    FiniteCheck fc(d, ws, rw.total, st);
    LDBP_TRY(fc.finish(run_rev_chain(d, (const float2*)x, nullptr, nullptr, (const float2*)taps, gamma, mask, nullptr,
                                     wb, rp, rw, st, nullptr, nullptr, nullptr, ybuf, /*forward_only=*/true),
                       st));
    LDBP_TRY(launch_rx_exact(d->batch, d->n, sps, rolloff, ybuf, (const float2*)symbols, power_w, weights_or_null,
                             errs, gybuf, st));
    LDBP_TRY(run_rev_chain(d, (const float2*)x, gybuf, nullptr, (const float2*)taps, gamma, mask, nullptr, wb, rp, rw,
                           st, buf, nullptr, nullptr, nullptr, false, /*skip_forward=*/true));
  } else {
    const BwdPlan bp = plan_bwd(d, true);
    const BwdWs bw = bwd_ws(d, bp);
    LDBP_TRY(run_forward_chain(d, (const float2*)x, ybuf, (const float2*)taps, gamma, mask,
                               reinterpret_cast<float2*>(wb + w.pp_off), st));
    LDBP_TRY(launch_rx_exact(d->batch, d->n, sps, rolloff, ybuf, (const float2*)symbols, power_w, weights_or_null,
                             errs, gybuf, st));
    LDBP_TRY(run_backward_chain(d, (const float2*)x, gybuf, nullptr, (const float2*)taps, gamma, mask, nullptr, wb, bp,
                                bw, st, buf, nullptr, nullptr));
  }
  ldbp::rx_wsum_kernel<<<1, 32, 0, st>>>(errs, weights_or_null, d->batch, buf);  // buf[0] = sum_b w_b errs_b
  return cuda_check("rx_wsum_kernel launch");
}

int ldbp_essm_workspace_bytes(const ldbp_dims* d, int32_t kappa, int op, size_t* bytes) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(validate_essm(d, kappa));
  if (!bytes) return fail(LDBP_EINVAL, "bytes is NULL");
  if (op != LDBP_OP_FORWARD && op != LDBP_OP_LOSS_GRAD) return fail(LDBP_EINVAL, "ESSM ops: FORWARD or LOSS_GRAD");
  *bytes = d->batch == 0 ? 0 : essm_ws(d, kappa, op == LDBP_OP_LOSS_GRAD).total;
  return LDBP_OK;
}

int ldbp_essm_forward(const ldbp_dims* d, int32_t kappa, const void* x, void* y, const void* taps,
                      const float* gamma, const float* eta, void* ws, size_t ws_bytes, void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(validate_essm(d, kappa));
  if (d->batch == 0) return LDBP_OK;
  LDBP_TRY(check_ptr(x, "x", 8));
  LDBP_TRY(check_ptr(y, "y", 8));
  LDBP_TRY(check_ptr(taps, "taps", 8));
  LDBP_TRY(check_ptr(gamma, "gamma", 4));
  LDBP_TRY(check_ptr(eta, "eta", 4));
  if (x == y) return fail(LDBP_EINVAL, "y must not alias x");
  const EssmWs w = essm_ws(d, kappa, false);
  if (!ws || ws_bytes < w.total) return fail(LDBP_EWORKSPACE, "essm forward needs %zu workspace bytes, got %zu", w.total, ws_bytes);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  unsigned char* wb = (unsigned char*)ws;
  const float2* src = (const float2*)x;
  for (int i = 0; i < d->steps; ++i) {
    const int remaining = d->steps - 1 - i;
    float2* dst = remaining == 0 ? (float2*)y : reinterpret_cast<float2*>(wb + w.act_off + (size_t)(i & 1) * w.act_each);
    LDBP_TRY(launch_essm_step(d, kappa, false, i, src, nullptr, nullptr, dst, (const float2*)taps, gamma, eta,
                              nullptr, st));
    src = dst;
  }
  return LDBP_OK;
}

int ldbp_essm_loss_grad(const ldbp_dims* d, int32_t kappa, const void* x, const void* target, const void* taps,
                        const float* gamma, const float* eta, double* buf, void* ws, size_t ws_bytes,
                        void* cuda_stream) {
  g_err[0] = 0;
  LDBP_TRY(validate_dims(d));
  LDBP_TRY(validate_essm(d, kappa));
  LDBP_TRY(check_ptr(buf, "buf", 8));
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const size_t nbuf = 1 + d->steps + 2 * (size_t)d->steps * d->taps + (size_t)d->steps * (2 * kappa + 1);
  if (d->batch == 0) return zero_outputs(buf, nbuf, st);
  LDBP_TRY(check_ptr(x, "x", 8));
  LDBP_TRY(check_ptr(target, "target", 8));
  LDBP_TRY(check_ptr(taps, "taps", 8));
  LDBP_TRY(check_ptr(gamma, "gamma", 4));
  LDBP_TRY(check_ptr(eta, "eta", 4));
  const EssmWs w = essm_ws(d, kappa, true);
  if (!ws || ws_bytes < w.total) return fail(LDBP_EWORKSPACE, "essm loss_grad needs %zu workspace bytes, got %zu", w.total, ws_bytes);
  unsigned char* wb = (unsigned char*)ws;
  const int M = d->steps;
  auto act = [&](int i) -> float2* { return reinterpret_cast<float2*>(wb + w.act_off + (size_t)(i - 1) * w.act_each); };
  auto gb = [&](int i) -> float2* { return reinterpret_cast<float2*>(wb + w.g_off + (size_t)(i & 1) * w.act_each); };
  double* part = reinterpret_cast<double*>(wb + w.part_off);
  const size_t part_step = (size_t)w.tiles * d->batch * w.V;
  // forward, storing u^(1..M-1) (u^(M) = y is recomputed by the seeded reverse step)
  for (int i = 0; i + 1 < M; ++i)
    LDBP_TRY(launch_essm_step(d, kappa, false, i, i == 0 ? (const float2*)x : act(i), nullptr, nullptr, act(i + 1),
                              (const float2*)taps, gamma, eta, nullptr, st));
  // reverse: step M-1 seeded from the target, then the incoming adjoints
  for (int i = M - 1; i >= 0; --i) {
    const float2* u = i == 0 ? (const float2*)x : act(i);
    const float2* gin = i == M - 1 ? nullptr : gb(i + 1);
    float2* gout = i == 0 ? nullptr : gb(i);
    LDBP_TRY(launch_essm_step(d, kappa, true, i, u, gin, (const float2*)target, gout, (const float2*)taps, gamma,
                              eta, part + (size_t)i * part_step, st));
  }
  const int nblk = w.tiles * (int)d->batch;
  double* part1 = reinterpret_cast<double*>(wb + w.part1_off);
  {
    TraceScope ts(LDBP_K_REDUCE, M, 0, st);
    ldbp::essm_reduce_chunks_kernel<<<dim3((unsigned)w.nch, (unsigned)M), 128, 0, st>>>(part, nblk, w.V, part1);
  }
  LDBP_TRY(cuda_check("essm_reduce_chunks_kernel launch"));
  ldbp::EssmReduceArgs r;
  r.partials = part1;
  r.M = M;
  r.nblk = w.nch;
  r.T = d->taps;
  r.kappa = kappa;
  r.sym = (d->flags & LDBP_SYMMETRIC) ? 1 : 0;
  r.buf = buf;
  {
    TraceScope ts(LDBP_K_REDUCE, M, 0, st);
    ldbp::essm_reduce_kernel<<<(M * w.V + 255) / 256, 256, 0, st>>>(r);
  }
  return cuda_check("essm_reduce_kernel launch");
}

// ---- GPU SSFM channel generator (§8(f) NEXT-2), ldbp_ssfm.cuh ----
static size_t ssfm_ws_bytes(int64_t n, int S) { return align256(sizeof(float2) * (size_t)S * n); }

int ldbp_ssfm_workspace_bytes(int64_t n, int32_t steps_per_span, size_t* bytes) {
  g_err[0] = 0;
  if (!bytes) return fail(LDBP_EINVAL, "bytes is NULL");
  if (n < 2 || (n & (n - 1)) || n > (1 << ldbp::kSsfmMaxLog2))
    return fail(LDBP_ESHAPE, "n %lld must be a power of two in [2, %d]", (long long)n, 1 << ldbp::kSsfmMaxLog2);
  if (steps_per_span < 1 || steps_per_span > ldbp::kSsfmMaxSteps)
    return fail(LDBP_ESHAPE, "steps_per_span %d not in [1, %d]", steps_per_span, ldbp::kSsfmMaxSteps);
  *bytes = ssfm_ws_bytes(n, steps_per_span);
  return LDBP_OK;
}

static cudaError_t ssfm_launch(int C, const ldbp::SsfmArgs& a, int64_t batch, size_t smem, cudaStream_t st) {
  void (*kern)(const ldbp::SsfmArgs) = C == 1 ? ldbp::ssfm_link_kernel<1>
                                       : C == 2 ? ldbp::ssfm_link_kernel<2> : ldbp::ssfm_link_kernel<4>;
  cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(batch * C));
  cfg.blockDim = dim3(ldbp::kSsfmThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = C > 1 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, a);
}

int ldbp_ssfm_link(int64_t batch, int64_t n, int32_t spans, int32_t steps_per_span, const double* deltas_km_host,
                   double span_km, double alpha_np, double beta2, double gamma, double fs_hz, double ase_sigma,
                   const void* noise_or_null, uint64_t ase_seed, int64_t ase_block0, void* u, void* r_or_null,
                   int32_t decim, double cutoff, void* ws, size_t ws_bytes, void* cuda_stream) {
  g_err[0] = 0;
  size_t need = 0;
  LDBP_TRY(ldbp_ssfm_workspace_bytes(n, steps_per_span, &need));
  if (batch < 0 || spans < 0) return fail(LDBP_ESHAPE, "batch and spans must be >= 0");
  if (batch == 0) return LDBP_OK;
  if (!deltas_km_host) return fail(LDBP_EINVAL, "deltas_km_host is NULL");
  if (ase_block0 < 0) return fail(LDBP_EINVAL, "ase_block0 %lld < 0", (long long)ase_block0);
  LDBP_TRY(check_ptr(u, "u", 8));
  if (noise_or_null) LDBP_TRY(check_ptr(noise_or_null, "noise", 8));
  // one CTA holds up to 2^14 samples; longer blocks are split over a 2- or 4-CTA cluster
  const int C = n > (1 << ldbp::kSsfmLocalMaxLog2) ? (int)(n >> ldbp::kSsfmLocalMaxLog2) : 1;
  const int64_t L = n / C;
  if (decim > 0) {
    LDBP_TRY(check_ptr(r_or_null, "r", 8));
    if (L % decim) return fail(LDBP_ESHAPE, "n / cluster (%lld) %% decim != 0", (long long)L);
  }
  if (!ws || ws_bytes < need) return fail(LDBP_EWORKSPACE, "ssfm needs %zu workspace bytes, got %zu", need, ws_bytes);
  cudaStream_t st = (cudaStream_t)cuda_stream;
  const int S = steps_per_span;
  float2* H = reinterpret_cast<float2*>(ws);
  // step lengths and Kerr phases travel in the kernel parameters: no copy, no host sync
  ldbp::SsfmDeltas dd;
  ldbp::SsfmArgs a;
  for (int s = 0; s < S; ++s) {
    const double d = deltas_km_host[s];
    dd.d[s] = d;
    const double leff = alpha_np == 0.0 ? d : (1.0 - exp(-alpha_np * d)) / alpha_np;
    a.kerr_phase[s] = (float)(gamma * leff);
  }
  int log2L = 0;
  while ((int64_t(1) << log2L) < L) ++log2L;
  {
    TraceScope ts(LDBP_K_SSFM, S, 0, st);
    ldbp::ssfm_htable_kernel<<<256, 256, 0, st>>>(H, dd, S, n, C, alpha_np, beta2, fs_hz, log2L);
  }
  LDBP_TRY(cuda_check("ssfm_htable_kernel launch"));
  a.u = (float2*)u;
  a.r = (float2*)r_or_null;
  a.H = H;
  a.noise = (const float2*)noise_or_null;
  a.n = n;
  a.log2L = log2L;
  a.log2n = 0;
  while ((int64_t(1) << a.log2n) < n) ++a.log2n;
  a.spans = spans;
  a.S = S;
  a.decim = decim;
  a.ase_mode = noise_or_null ? 1 : (ase_sigma != 0.0 ? 2 : 0);
  a.ase_seed = ase_seed;
  a.block0 = ase_block0;
  a.span_gain = (float)exp(0.5 * alpha_np * span_km);
  a.ase_sigma = (float)ase_sigma;
  a.cutoff = (float)cutoff;
  const size_t smem = sizeof(float2) * ((size_t)L + L / 16 + 1 + L / 2 + (C > 1 ? (size_t)n / 64 + 64 : 0));
  cudaError_t e;
  {
    TraceScope ts(LDBP_K_SSFM, spans * S, batch * n, st);
    e = ssfm_launch(C, a, batch, smem, st);
  }
  if (e != cudaSuccess) return fail(LDBP_ECUDA, "ssfm_link_kernel launch: %s", cudaGetErrorString(e));
  return cuda_check("ssfm_link_kernel launch");
}

int ldbp_trace_begin(int capacity) {
  g_err[0] = 0;
  if (capacity < 0) return fail(LDBP_EINVAL, "capacity < 0");
  for (auto& r : g_trace) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_trace.clear();
  g_trace.reserve(capacity);
  g_trace_cap = capacity;
  g_trace_seen = 0;
  g_trace_on = true;
  return LDBP_OK;
}

int ldbp_trace_end(ldbp_trace_record* out, int capacity, int* count) {
  g_err[0] = 0;
  g_trace_on = false;
  int status = LDBP_OK;
  int n = 0;
  for (auto& r : g_trace) {
    float ms = -1.f;
    if (cudaEventSynchronize(r.b) != cudaSuccess || cudaEventElapsedTime(&ms, r.a, r.b) != cudaSuccess) {
      status = fail(LDBP_ECUDA, "trace event: %s", cudaGetErrorString(cudaGetLastError()));
    }
    if (out && n < capacity) {
      out[n].kind = r.kind;
      out[n].steps = r.steps;
      out[n].samples = r.samples;
      out[n].ms = ms;
      out[n].reserved = 0;
    }
    ++n;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_trace.clear();
  if (count) *count = g_trace_seen;
  return status;
}

}  // extern "C"

// ldbp_inst.cu — explicit kernel instantiations for one half-length Kh (compiled with
// -DLDBP_KH=<Kh>); split per Kh so the build parallelises.
#include "ldbp_kernels.cuh"

#ifndef LDBP_KH
#error "compile with -DLDBP_KH=<0..7>"
#endif

using FwdFn = void (*)(const ldbp::FwdArgs);
using BwdFn = void (*)(const ldbp::BwdArgs);
using RevFn = void (*)(const ldbp::RevArgs);
using ParFn = void (*)(const float2*, const float*, const uint8_t*, int, int, void*, int);

#define LDBP_CAT2(a, b) a##b
#define LDBP_CAT(a, b) LDBP_CAT2(a, b)

FwdFn LDBP_CAT(ldbp_get_fwd_, LDBP_KH)(bool sym, bool fast, bool chk) {
  constexpr int K = LDBP_KH, R = ldbp::fwd_r(LDBP_KH);
  if (chk) {  // LDBP_CHECK_FINITE instantiations
    if (sym) return fast ? ldbp::fwd_tile_kernel<K, R, true, true, true> : ldbp::fwd_tile_kernel<K, R, true, false, true>;
    return fast ? ldbp::fwd_tile_kernel<K, R, false, true, true> : ldbp::fwd_tile_kernel<K, R, false, false, true>;
  }
  if (sym) return fast ? ldbp::fwd_tile_kernel<K, R, true, true> : ldbp::fwd_tile_kernel<K, R, true, false>;
  return fast ? ldbp::fwd_tile_kernel<K, R, false, true> : ldbp::fwd_tile_kernel<K, R, false, false>;
}

FwdFn LDBP_CAT(ldbp_get_fwd_store_, LDBP_KH)(bool sym, bool chk) {
  constexpr int K = LDBP_KH, R = LDBP_FWD_R;
  if (chk) return sym ? ldbp::fwd_store_kernel<K, R, true, true> : ldbp::fwd_store_kernel<K, R, false, true>;
  return sym ? ldbp::fwd_store_kernel<K, R, true> : ldbp::fwd_store_kernel<K, R, false>;
}

BwdFn LDBP_CAT(ldbp_get_bwd_, LDBP_KH)(bool sym, bool fast) {
  constexpr int K = LDBP_KH, R = bwd_r(LDBP_KH);
  if (sym) return fast ? ldbp::bwd_segment_kernel<K, R, true, true> : ldbp::bwd_segment_kernel<K, R, true, false>;
  return fast ? ldbp::bwd_segment_kernel<K, R, false, true> : ldbp::bwd_segment_kernel<K, R, false, false>;
}

RevFn LDBP_CAT(ldbp_get_rev_, LDBP_KH)(bool sym, bool fast) {
  constexpr int K = LDBP_KH, R = rev_r(LDBP_KH);
  if (sym) return fast ? ldbp::rev_tile_kernel<K, R, true, true> : ldbp::rev_tile_kernel<K, R, true, false>;
  return fast ? ldbp::rev_tile_kernel<K, R, false, true> : ldbp::rev_tile_kernel<K, R, false, false>;
}

ParFn LDBP_CAT(ldbp_get_params_, LDBP_KH)(bool sym) {
  constexpr int K = LDBP_KH;
  return sym ? ldbp::params_kernel<K, true> : ldbp::params_kernel<K, false>;
}

RevFn LDBP_CAT(ldbp_get_rev2_, LDBP_KH)(bool fast) {
#if LDBP_KH <= 12  // warp-overlapped slots of 12 samples: Kh <= 12
  constexpr int K = LDBP_KH;
  return fast ? ldbp::rev2_tile_kernel<K, true> : ldbp::rev2_tile_kernel<K, false>;
#else
  (void)fast;
  return nullptr;
#endif
}

RevFn LDBP_CAT(ldbp_get_rev3_, LDBP_KH)(bool fast) {
#if LDBP_KH == 2 || LDBP_KH == 4 || LDBP_KH == 6
  constexpr int K = LDBP_KH;
  return fast ? ldbp::rev3_tile_kernel<K, true> : ldbp::rev3_tile_kernel<K, false>;
#else
  (void)fast;
  return nullptr;
#endif
}

RevFn LDBP_CAT(ldbp_get_rev4_, LDBP_KH)(bool fast) {
#if LDBP_KH >= 1 && LDBP_KH <= 12  // rows of 12 samples: Kh <= 12
  constexpr int K = LDBP_KH;
  return fast ? ldbp::rev4_tile_kernel<K, true> : ldbp::rev4_tile_kernel<K, false>;
#else
  (void)fast;
  return nullptr;
#endif
}

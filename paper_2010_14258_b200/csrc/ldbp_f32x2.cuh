// ldbp_f32x2.cuh — packed FP32x2 helpers (PTX add/mul/fma .f32x2, sm_100+ -> SASS FADD2/FMUL2/
// FFMA2).  One instruction updates both halves of a complex64 value; ptxas folds the operand
// patterns used below into free SASS modifiers: pk(x, x) -> "R.F32" broadcast, pk(v.y, v.x) ->
// ".LO_HI" swap, pk(-y, y) -> ".NP" low-half negate.  Complex arithmetic therefore costs half the
// issue slots of the scalar form (the FP32 pipe rate is unchanged: 128 lane-FMA/clk/SM).
#pragma once
#include <cuda_runtime.h>

namespace ldbp {

typedef unsigned long long f2x;  // a complex64 / float2 in one 64-bit register pair

__device__ __forceinline__ f2x pk(float lo, float hi) {
  f2x r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 upk(f2x r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ f2x pk(float2 v) { return pk(v.x, v.y); }
__device__ __forceinline__ float lof(f2x r) { return upk(r).x; }
__device__ __forceinline__ float hif(f2x r) { return upk(r).y; }
__device__ __forceinline__ f2x bcast(float x) { return pk(x, x); }  // -> SASS "R.F32" operand
__device__ __forceinline__ f2x add2(f2x a, f2x b) {
  f2x d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2x mul2(f2x a, f2x b) {
  f2x d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c) {
  f2x d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// acc + h * s for complex h, s:  (acc.x + hx sx - hy sy, acc.y + hx sy + hy sx)
__device__ __forceinline__ float2 cmac(float2 acc, float2 h, float2 s) {
  f2x t = fma2(pk(h.x, h.x), pk(s), pk(acc));
  return upk(fma2(pk(-h.y, h.y), pk(s.y, s.x), t));
}
// h * s
__device__ __forceinline__ float2 cmul(float2 h, float2 s) {
  f2x t = mul2(pk(h.x, h.x), pk(s));
  return upk(fma2(pk(-h.y, h.y), pk(s.y, s.x), t));
}
// acc + conj(h) * s:  (acc.x + hx sx + hy sy, acc.y + hx sy - hy sx)
__device__ __forceinline__ float2 cmac_conj(float2 acc, float2 h, float2 s) {
  f2x t = fma2(pk(h.x, h.x), pk(s), pk(acc));
  return upk(fma2(pk(h.y, -h.y), pk(s.y, s.x), t));
}
// acc + g * conj(w):  (acc.x + gx wx + gy wy, acc.y + gy wx - gx wy)
__device__ __forceinline__ float2 cmac_gconj(float2 acc, float2 g, float2 w) {
  f2x t = fma2(pk(w.x, w.x), pk(g), pk(acc));        // (acc.x + wx gx, acc.y + wx gy)
  return upk(fma2(pk(w.y, -w.y), pk(g.y, g.x), t));   // + (wy gy, -wy gx)
}
// conj(h) * s
__device__ __forceinline__ float2 cmul_conj(float2 h, float2 s) {
  f2x t = mul2(pk(h.x, h.x), pk(s));
  return upk(fma2(pk(h.y, -h.y), pk(s.y, s.x), t));
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return upk(add2(pk(a), pk(b))); }
// a * (c + j s)
__device__ __forceinline__ float2 crot(float2 a, float c, float s) {
  f2x t = mul2(pk(a.x, a.x), pk(c, s));
  return upk(fma2(pk(-a.y, a.y), pk(s, c), t));
}

}  // namespace ldbp

// f32x2.cuh — packed-FP32 helpers for sm_100 (fma/add/sub/mul .f32x2 -> FFMA2/FADD2/FMUL2).
// Two float lanes live in one 64-bit register pair; a broadcast scalar enters as mk2(s, s).
#pragma once
#include <cuda_runtime.h>

namespace spic {

struct f2 {
  unsigned long long r;
};
__device__ __forceinline__ f2 mk2(float a, float b) {
  f2 o;
  asm("mov.b64 %0, {%1, %2};" : "=l"(o.r) : "f"(a), "f"(b));
  return o;
}
__device__ __forceinline__ void un2(f2 a, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a.r));
}
__device__ __forceinline__ f2 add2(f2 a, f2 b) {
  f2 o;
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
  return o;
}
__device__ __forceinline__ f2 sub2(f2 a, f2 b) {
  f2 o;
  asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
  return o;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 o;
  asm("mul.rn.ftz.f32x2 %0, %1, %2;" : "=l"(o.r) : "l"(a.r), "l"(b.r));
  return o;
}
// sign-bit ops on both halves: integer LOP3 on the ALU pipe (ptxas would otherwise turn
// fabs / negation into FADDs on the FMA pipe)
__device__ __forceinline__ f2 abs2(f2 a) {
  f2 o;
  asm("and.b64 %0, %1, 0x7fffffff7fffffff;" : "=l"(o.r) : "l"(a.r));
  return o;
}
__device__ __forceinline__ f2 neg2(f2 a) {
  f2 o;
  asm("xor.b64 %0, %1, 0x8000000080000000;" : "=l"(o.r) : "l"(a.r));
  return o;
}
__device__ __forceinline__ f2 rint2(f2 a) {
  float lo, hi;
  un2(a, lo, hi);
  return mk2(rintf(lo), rintf(hi));
}
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 o;
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(o.r) : "l"(a.r), "l"(b.r), "l"(c.r));
  return o;
}

// c - a*b as one FFMA2 with a negated operand: the product and the subtraction are written
// without .rn so ptxas contracts them (same single rounding as fma(-a, b, c)); saves the two
// LOP3s of an explicit sign flip
__device__ __forceinline__ f2 fnms2(f2 a, f2 b, f2 c) {
  f2 o;
  asm("{\n.reg .b64 t;\nmul.ftz.f32x2 t, %1, %2;\nsub.ftz.f32x2 %0, %3, t;\n}"
      : "=l"(o.r)
      : "l"(a.r), "l"(b.r), "l"(c.r));
  return o;
}

}  // namespace spic

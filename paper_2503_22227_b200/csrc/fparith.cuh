// FP64-pipe modular arithmetic for primes q < 2^50 (device only).
//
// B200 runs DFMA at half rate but IMAD.WIDE.U32 (the 32x32->64 product every
// 64-bit integer multiply is built from) at quarter rate, so for chains of
// primes below 2^50 the modular products go through the FP64 pipe.  Values
// are doubles carrying exact signed integer representatives; the products
// are exact through the FMA error-free split:
//   h = x w, l = fma(x, w, -h)            (x w = h + l exactly)
//   k = rint(x * (w/q))                   (magic-constant rounding, |x w/q| < 2^51)
//   t = fma(-k, q, h) + l                 (= x w - k q exactly, |t| <= q/2 + eps)
// Every intermediate is an exact integer, so results reduced to [0, q) are
// bit-identical to the integer path.
#pragma once
#include "modarith.cuh"

constexpr double kFpMagic = 6755399441055744.0;  // 1.5 * 2^52

__device__ __forceinline__ double fp_rint_mul(double x, double y) {
  return __dadd_rn(__fma_rn(x, y, kFpMagic), -kFpMagic);
}
// x w mod q (signed representative, |result| <= q/2 + eps) for |x w/q| < 2^51;
// w = (w, w / q).
__device__ __forceinline__ double fp_mulmod(double x, double2 w, double q) {
  const double h = __dmul_rn(x, w.x);
  const double l = __fma_rn(x, w.x, -h);
  const double k = fp_rint_mul(x, w.y);
  return __dadd_rn(__fma_rn(-k, q, h), l);
}
// x mod q, signed representative in [-q/2, q/2]; qd = (q, 1/q).
__device__ __forceinline__ double fp_reduce(double x, double2 qd) {
  return __fma_rn(-fp_rint_mul(x, qd.y), qd.x, x);
}
// signed representative in (-q, 2q) -> canonical u64 in [0, q)
__device__ __forceinline__ u64 fp_canon(double x, double q) {
  x = x < 0.0 ? __dadd_rn(x, q) : x;
  x = x >= q ? __dadd_rn(x, -q) : x;
  return (u64)__double2ll_rn(x);
}

// representative in [-q/2 - eps, q/2 + eps] (fp_reduce / fp_mulmod output)
// -> canonical u64 in [0, q)
__device__ __forceinline__ u64 fp_canon_half(double x, double q);

// exact u64 -> double for x < 2^52 (one LOP + one DADD instead of I2F.F64)
__device__ __forceinline__ double fp_from_u52(u64 x) {
  return __dadd_rn(__longlong_as_double((long long)(x | 0x4330000000000000ull)),
                   -4503599627370496.0);
}
// exact double -> u64 for an integer-valued x in [0, 2^52) (DADD + LOP, no F2I)
__device__ __forceinline__ u64 fp_to_u52(double x) {
  return (u64)__double_as_longlong(__dadd_rn(x, 4503599627370496.0)) & 0x000FFFFFFFFFFFFFull;
}

__device__ __forceinline__ u64 fp_canon_half(double x, double q) {
  return fp_to_u52(x < 0.0 ? __dadd_rn(x, q) : x);
}

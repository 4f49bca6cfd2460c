// Exact 64-bit modular arithmetic for RNS limbs (q < 2^62), shared by the
// sm_100a kernels and the host-side precompute / self-test code.
//
// Every function returns the canonical residue in [0, q) unless its name says
// "lazy".  Canonical outputs are what make the GPU path bit-identical to the
// reference: the reference reduces everything to [0, q)
// (coremath/_kernels.py:19-32 Shoup, :102-133 Montgomery; vecmod.py:148-165),
// so any exact algorithm over Z_q produces the same bits.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define FHE_HD __host__ __device__ __forceinline__
#else
#define FHE_HD inline
#endif

typedef uint64_t u64;
typedef uint32_t u32;

// Per-prime reduction constants (built on the host, see context.cu).
//   mu   = floor(2^(64+s) / q) with s = bitlen(q) - 1   (fits in 64 bits)
//   r64  = 2^64 mod q
struct ModConst {
  u64 q;
  u64 mu;
  u64 r64;
  u32 s;
  u32 pad;
};

FHE_HD u64 mulhi64(u64 a, u64 b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (u64)(((unsigned __int128)a * b) >> 64);
#endif
}

FHE_HD void mul_wide(u64 a, u64 b, u64& hi, u64& lo) {
  lo = a * b;
  hi = mulhi64(a, b);
}

// 128-bit accumulate: (hi, lo) += (bh, bl)
FHE_HD void add_wide(u64& hi, u64& lo, u64 bh, u64 bl) {
#ifdef __CUDA_ARCH__
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;"
      : "+l"(lo), "+l"(hi) : "l"(bl), "l"(bh));
#else
  u64 nl = lo + bl;
  hi += bh + (nl < lo);
  lo = nl;
#endif
}

// (hi, lo) += a * b
FHE_HD void mac_wide(u64& hi, u64& lo, u64 a, u64 b) {
#ifdef __CUDA_ARCH__
  u64 pl = a * b;
  u64 ph = __umul64hi(a, b);
  asm("add.cc.u64 %0, %0, %2;\n\taddc.u64 %1, %1, %3;"
      : "+l"(lo), "+l"(hi) : "l"(pl), "l"(ph));
#else
  unsigned __int128 acc = ((unsigned __int128)hi << 64) | lo;
  acc += (unsigned __int128)a * b;
  hi = (u64)(acc >> 64);
  lo = (u64)acc;
#endif
}

FHE_HD u64 csub(u64 x, u64 q) { return x >= q ? x - q : x; }

// a + b mod q for a, b in [0, q)
FHE_HD u64 add_mod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
// a - b mod q for a, b in [0, q)
FHE_HD u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
FHE_HD u64 neg_mod(u64 a, u64 q) { return a == 0 ? 0 : q - a; }

// Shoup multiply by a constant w < q with w_sh = floor(w * 2^64 / q).
// Any x < 2^64 is accepted; the lazy result lies in [0, 2q).
FHE_HD u64 shoup_lazy(u64 x, u64 w, u64 w_sh, u64 q) {
  u64 hi = mulhi64(x, w_sh);
  return x * w - hi * q;
}
FHE_HD u64 shoup_mul(u64 x, u64 w, u64 w_sh, u64 q) {
  return csub(shoup_lazy(x, w, w_sh, q), q);
}

// Barrett reduction of a double-word x = hi*2^64 + lo with x < 2^63 * q.
// (Covers any product of two canonical residues and short sums of them.)
// The quotient estimate never exceeds floor(x/q) and is short by at most 2,
// so two conditional subtractions give the canonical residue.
FHE_HD u64 reduce_prod(u64 hi, u64 lo, const ModConst& m) {
  u64 xs = (hi << (64 - m.s)) | (lo >> m.s);
  u64 qe = mulhi64(xs, m.mu);
  u64 r = lo - qe * m.q;
  r = csub(r, m.q);
  return csub(r, m.q);
}

// Reduction of any x < 2^126 (e.g. a basis-conversion accumulator of up to
// 15 products of 61-bit words): fold the high word through 2^64 mod q first.
FHE_HD u64 reduce_fold(u64 hi, u64 lo, const ModConst& m) {
  u64 h2, l2;
  mul_wide(hi, m.r64, h2, l2);
  add_wide(h2, l2, 0, lo);
  return reduce_prod(h2, l2, m);
}

// a * b mod q for canonical a, b.
FHE_HD u64 mul_mod(u64 a, u64 b, const ModConst& m) {
  u64 hi, lo;
  mul_wide(a, b, hi, lo);
  return reduce_prod(hi, lo, m);
}

// Reduce an arbitrary 64-bit word (e.g. a residue of another prime) mod q.
FHE_HD u64 reduce_word(u64 x, const ModConst& m) { return reduce_prod(0, x, m); }

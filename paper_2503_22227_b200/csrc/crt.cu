// Exact CRT lift of decrypted residues on the device: the step after the
// path, replacing the reference's O(L N) Python big-int
// loop crt_reconstruct_poly (coremath/crt.py:84-100) in
//   ckks_decode  (ckks.py:157-166):  float(v - Q if v > Q // 2 else v) / scale
//   bgv_decrypt  (bgv.py:89-101):    (centred v % t) * inv_f % t
//   bfv_decrypt  (bfv.py:106-117):   ((t * centred v + Q // 2) // Q) % t
//
// One thread per coefficient holds v as a W-limb integer:
//   v = sum_i y_i (Q / q_i) - k Q,  y_i = [r_i (Q / q_i)^-1]_{q_i}
// with k = floor(sum_i y_i / q_i) estimated in double (error < 2^-40, so one
// exact correction step at most), then centred.  Every output is the exact
// result of the reference's Python-integer formula: the float conversion
// rounds the exact integer to nearest-even (Python float(int)), the division
// by the scale is the same IEEE division, and the BFV quotient is corrected
// exactly after a floating-point estimate.  |v| >= 2^1024 gives +-inf where
// Python raises OverflowError (the host layer raises the same).
#include "fhe_context.cuh"

namespace {

constexpr int kCrtThreads = 128;

typedef unsigned __int128 u128d;

template <int W>
__device__ __forceinline__ bool ge(const u64 (&a)[W], const u64* b, int w) {
  for (int k = w - 1; k >= 0; --k)
    if (a[k] != b[k]) return a[k] > b[k];
  return true;
}
template <int W>
__device__ __forceinline__ void add_to(u64 (&a)[W], const u64* b, int w) {
  u64 c = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      const u128d s = (u128d)a[k] + b[k] + c;
      a[k] = (u64)s;
      c = (u64)(s >> 64);
    }
  }
}
template <int W>
__device__ __forceinline__ void sub_from(u64 (&a)[W], const u64* b, int w) {
  u64 br = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      const u128d d = (u128d)a[k] - b[k] - br;
      a[k] = (u64)d;
      br = (u64)(d >> 64) ? 1 : 0;
    }
  }
}
template <int W>
__device__ __forceinline__ bool neg(const u64 (&a)[W], int w) { return (a[w - 1] >> 63) != 0; }
template <int W>
__device__ __forceinline__ void negate(u64 (&a)[W], int w) {
  u64 c = 1;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      const u128d s = (u128d)(~a[k]) + c;
      a[k] = (u64)s;
      c = (u64)(s >> 64);
    }
  }
}
template <int W>
__device__ __forceinline__ bool gt(const u64 (&a)[W], const u64* b, int w) {
  for (int k = w - 1; k >= 0; --k)
    if (a[k] != b[k]) return a[k] > b[k];
  return false;
}
// a += m * b (m a word, b w limbs)
template <int W>
__device__ __forceinline__ void mac_word(u64 (&a)[W], u64 m, const u64* b, int w) {
  u64 c = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      const u128d s = (u128d)m * b[k] + a[k] + c;
      a[k] = (u64)s;
      c = (u64)(s >> 64);
    }
  }
}
// a -= m * b
template <int W>
__device__ __forceinline__ void msub_word(u64 (&a)[W], u64 m, const u64* b, int w) {
  u64 c = 0, br = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    if (k < w) {
      const u128d p = (u128d)m * b[k] + c;
      c = (u64)(p >> 64);
      const u128d d = (u128d)a[k] - (u64)p - br;
      a[k] = (u64)d;
      br = (u64)(d >> 64) ? 1 : 0;
    }
  }
}
// nonnegative multi-limb magnitude -> double (times 2^(-64 drop)), round to
// nearest even
template <int W>
__device__ __forceinline__ double to_double_rne(const u64 (&m)[W], int w, int drop = 0) {
  int h = w - 1;
  while (h >= 0 && m[h] == 0) --h;
  if (h < 0) return 0.0;
  const int lz = __clzll((long long)m[h]);
  u64 top = m[h] << lz;
  u64 low = 0;
  if (h >= 1) {
    if (lz) top |= m[h - 1] >> (64 - lz);
    low = lz ? (m[h - 1] << lz) : m[h - 1];
    for (int k = h - 2; k >= 0; --k) low |= m[k];
  }
  // value = top * 2^(64 h - lz), top has its leading bit at 63
  u64 mant = top >> 11;
  const u64 rem = top & 0x7ff;
  const bool round = (rem >> 10) & 1;
  const bool sticky = (rem & 0x3ff) || low;
  if (round && (sticky || (mant & 1))) ++mant;  // mant == 2^53 stays exact as a double
  return scalbn((double)mant, 64 * (h - drop) - lz + 11);
}

struct CrtArgs {
  const u64* rows;
  long n;
  int level, w, mode;
  const u64* M;
  const u64* Q;
  const u64* Qh;
  const WPair* inv;
  const double* qinv;
  double Qd;   // Q * 2^(-64 qdrop)
  int qdrop;
  double scale;
  u64 t, inv_f;
  double* out_d;
  u64* out_u;
};

template <int W>
__global__ void __launch_bounds__(kCrtThreads) crt_lift_kernel(const DevChain ch, const CrtArgs a) {
  const int w = a.w;
  for (long j = blockIdx.x * (long)blockDim.x + threadIdx.x; j < a.n;
       j += (long)gridDim.x * blockDim.x) {
    u64 v[W + 1];
#pragma unroll
    for (int k = 0; k <= W; ++k) v[k] = 0;
    double fsum = 0.0;
    for (int i = 0; i < a.level; ++i) {
      const u64 q = ch.mc[i].q;
      const WPair iv = a.inv[i];
      const u64 y = shoup_mul(a.rows[(long)i * a.n + j], iv.w, iv.sh, q);
      fsum = __fma_rn((double)y, a.qinv[i], fsum);
      mac_word<W + 1>(v, y, a.M + (long)i * w, w);
    }
    // v -= k Q with k = floor(sum y_i / q_i), then exact correction into [0, Q)
    const u64 k = (u64)floor(fsum);
    msub_word<W + 1>(v, k, a.Q, w);
    if (neg<W + 1>(v, w)) add_to<W + 1>(v, a.Q, w);
    else if (ge<W + 1>(v, a.Q, w)) sub_from<W + 1>(v, a.Q, w);
    // centre: v > Q // 2  ->  v - Q
    if (gt<W + 1>(v, a.Qh, w)) sub_from<W + 1>(v, a.Q, w);
    const bool sgn = neg<W + 1>(v, w);
    if (a.mode == FHE_CRT_FLOAT) {
      u64 mag[W + 1];
#pragma unroll
      for (int kk = 0; kk <= W; ++kk) mag[kk] = v[kk];
      if (sgn) negate<W + 1>(mag, w);
      double d = to_double_rne<W + 1>(mag, w);
      if (sgn) d = -d;
      a.out_d[j] = a.scale != 0.0 ? __ddiv_rn(d, a.scale) : d;
      continue;
    }
    const u64 t = a.t;
    if (a.mode == FHE_CRT_MOD_T) {
      // Python: (v % t) * inv_f % t with v the centred (signed) value
      u64 mag[W + 1];
#pragma unroll
      for (int kk = 0; kk <= W; ++kk) mag[kk] = v[kk];
      if (sgn) negate<W + 1>(mag, w);
      u64 r = 0;  // |v| mod t, Horner from the top limb
      for (int kk = w - 1; kk >= 0; --kk) r = (u64)((((u128d)r << 64) | mag[kk]) % t);
      if (sgn && r) r = t - r;
      a.out_u[j] = (u64)((u128d)r * a.inv_f % t);
      continue;
    }
    // FHE_CRT_BFV: m = floor((t v + Q // 2) / Q) mod t
    u64 x[W + 1];
#pragma unroll
    for (int kk = 0; kk <= W; ++kk) x[kk] = 0;
    {
      u64 mag[W + 1];
#pragma unroll
      for (int kk = 0; kk <= W; ++kk) mag[kk] = v[kk];
      if (sgn) negate<W + 1>(mag, w);
      mac_word<W + 1>(x, t, mag, w);  // t |v| (fits: |v| <= Q/2, t < 2^62)
      if (sgn) negate<W + 1>(x, w);
      add_to<W + 1>(x, a.Qh, w);      // X = t v + Q // 2 (signed)
    }
    const bool xs = neg<W + 1>(x, w);
    u64 xm[W + 1];
#pragma unroll
    for (int kk = 0; kk <= W; ++kk) xm[kk] = x[kk];
    if (xs) negate<W + 1>(xm, w);
    // both X and Q scaled by 2^(-64 qdrop) (Q itself can exceed the double range)
    const double xd = to_double_rne<W + 1>(xm, w, a.qdrop);
    long long m = (long long)floor((xs ? -xd : xd) / a.Qd);
    // R = X - m Q must land in [0, Q): exact corrections (the estimate is
    // within 2^-20 of X / Q for t < 2^40, so at most one step)
    u64 r[W + 1];
#pragma unroll
    for (int kk = 0; kk <= W; ++kk) r[kk] = x[kk];
    if (m >= 0) msub_word<W + 1>(r, (u64)m, a.Q, w);
    else mac_word<W + 1>(r, (u64)(-m), a.Q, w);
    for (int it = 0; it < 4 && neg<W + 1>(r, w); ++it) {
      --m;
      add_to<W + 1>(r, a.Q, w);
    }
    for (int it = 0; it < 4 && ge<W + 1>(r, a.Q, w); ++it) {
      ++m;
      sub_from<W + 1>(r, a.Q, w);
    }
    long long mt = m % (long long)t;
    if (mt < 0) mt += (long long)t;
    a.out_u[j] = (u64)mt;
  }
}

}  // namespace

int run_crt_lift(const FheContext& ctx, int mode, void* out, const u64* rows, int level,
                 double scale, u64 t, u64 inv_f, cudaStream_t st) {
  if (level < 1 || level > ctx.L) {
    fhe_set_error("crt lift: level out of range");
    return -1;
  }
  if (mode != FHE_CRT_FLOAT && (t < 2 || t >= ((u64)1 << (mode == FHE_CRT_BFV ? 40 : 62)))) {
    fhe_set_error("crt lift: plain modulus out of range (BGV < 2^62, BFV < 2^40)");
    return -1;
  }
  if (mode < FHE_CRT_FLOAT || mode > FHE_CRT_BFV) {
    fhe_set_error("crt lift: unknown mode");
    return -1;
  }
  const LevelPlan& lp = ctx.levels[level];
  const DevChain& ch = ctx.chain->dev;
  CrtArgs a{rows, 1L << ch.log_n, level, lp.crt_W, mode, lp.crt_M, lp.crt_Q, lp.crt_Qh,
            lp.crt_inv, lp.crt_qinv, lp.crt_Qd, lp.crt_qdrop, scale, t, inv_f,
            mode == FHE_CRT_FLOAT ? (double*)out : nullptr,
            mode == FHE_CRT_FLOAT ? nullptr : (u64*)out};
  const int grid = (int)std::min<long>((a.n + kCrtThreads - 1) / kCrtThreads, 4096);
  auto go = [&](auto kern) -> int {
    kern<<<grid, kCrtThreads, 0, st>>>(ch, a);
    FHE_LAUNCH_CHECK();
    return 0;
  };
  const int w = lp.crt_W;
  if (w <= 4) return go(crt_lift_kernel<4>);
  if (w <= 8) return go(crt_lift_kernel<8>);
  if (w <= 12) return go(crt_lift_kernel<12>);
  if (w <= 16) return go(crt_lift_kernel<16>);
  if (w <= 24) return go(crt_lift_kernel<24>);
  if (w <= 32) return go(crt_lift_kernel<32>);
  fhe_set_error("crt lift: modulus product above 2^1950 bits");
  return -1;
}

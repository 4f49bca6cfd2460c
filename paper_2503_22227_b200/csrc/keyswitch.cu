// Key switching (ModUp -> key inner product -> ModDown) and rescale on the
// device.
//
// Reference: key_switch (keys.py:186-237) is the per-prime gadget: INTT the
// input, re-reduce every residue polynomial against every prime of the level
// (digit_rows[i, j] = coeff[i] mod q_j), NTT the level^2 rows, multiply-
// accumulate against the level digit keys.  That is the hybrid algorithm with
// alpha = 1 and no special modulus (K = 0):
//   ModUp     digit d (primes S_d): y_s = [c_s (Q_d/q_s)^-1]_{q_s},
//             ext_m = sum_s y_s [Q_d/q_s]_m   (fast base conversion, the
//             formula of behz.py:131-153); with alpha = 1, ext_m = c_s mod m.
//   inner     b_m = sum_d ext_d,m * kb_d,m ; a_m = sum_d ext_d,m * ka_d,m
//   ModDown   (K > 0): b_j <- (b_j - BConv_{P->q_j}(b_P)) * P^-1  (same for a)
// The digit's own primes are not converted: their evaluation-domain values
// are the input itself, so the INTT/NTT round trip of the reference
// (NTT(INTT(d) mod q_i) = d) is skipped without changing a bit.
#include "fhe_context.cuh"
#include "fparith.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kMaxAlpha = 16;
#ifndef FHE_INNER_BU
#define FHE_INNER_BU 2
#endif
#ifndef FHE_TENS_MINB
#define FHE_TENS_MINB 2
#endif
#ifndef FHE_FIN_MINB
#define FHE_FIN_MINB 3
#endif
#ifndef FHE_INNER_MINB
#define FHE_INNER_MINB 3
#endif
#ifndef FHE_MODUP_CPT
#define FHE_MODUP_CPT 2
#endif
#ifndef FHE_MODUP_MINB
#define FHE_MODUP_MINB 2
#endif
#ifndef FHE_MODUP_U
#define FHE_MODUP_U 6
#endif

// Reduce a chain of multiply-accumulates every `chunk` terms so the 128-bit
// accumulator stays below 2^126 (reduce_fold's domain).
struct Acc {
  u64 hi = 0, lo = 0, r = 0;
  int cnt = 0;
  __device__ __forceinline__ void mac(u64 a, u64 b, int chunk, const ModConst& m) {
    mac_wide(hi, lo, a, b);
    if (++cnt == chunk) {
      r = add_mod(r, reduce_fold(hi, lo, m), m.q);
      hi = lo = 0;
      cnt = 0;
    }
  }
  __device__ __forceinline__ u64 done(const ModConst& m) {
    return cnt ? add_mod(r, reduce_fold(hi, lo, m), m.q) : r;
  }
};

// ModUp basis extension of one digit: grid (coef blocks, digits, batch).
__global__ void __launch_bounds__(kThreads)
    modup_kernel(const DevChain ch, const u64* __restrict__ c, long c_stride,
                 u64* __restrict__ ext, long ext_stride, const int* __restrict__ dig_info,
                 const WPair* __restrict__ up_inv, const u64* __restrict__ up_w, int level, int K,
                 int L, int chunk) {
  const int di = blockIdx.y, b = blockIdx.z;
  const int s0 = dig_info[4 * di], na = dig_info[4 * di + 1];
  const int row_off = dig_info[4 * di + 2], w_off = dig_info[4 * di + 3];
  const int nt = level + K - na;
  extern __shared__ u64 sw[];
  for (int i = threadIdx.x; i < na * nt; i += blockDim.x) sw[i] = up_w[w_off + i];
  __syncthreads();
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const u64* cb = c + b * c_stride;
  u64* eb = ext + b * ext_stride + (long)row_off * n;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    u64 y[kMaxAlpha];
#pragma unroll
    for (int s = 0; s < kMaxAlpha; ++s) {
      if (s < na) {
        const WPair w = up_inv[s0 + s];
        y[s] = shoup_mul(cb[(long)(s0 + s) * n + i], w.w, w.sh, ch.mc[s0 + s].q);
      }
    }
    // four targets per iteration: independent 128-bit accumulation chains
    int t = 0;
    for (; na <= chunk && t + 4 <= nt; t += 4) {
      u64 hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
#pragma unroll
      for (int s = 0; s < kMaxAlpha; ++s) {
        if (s < na) {
#pragma unroll
          for (int u = 0; u < 4; ++u) mac_wide(hi[u], lo[u], y[s], sw[s * nt + t + u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int m = t + u < s0 ? t + u : t + u + na;
        const int p = m < level ? m : L + (m - level);
        eb[(long)(t + u) * n + i] = reduce_fold(hi[u], lo[u], ch.mc[p]);
      }
    }
    for (; t < nt; ++t) {
      const int m = t < s0 ? t : t + na;
      const int p = m < level ? m : L + (m - level);
      const ModConst mc = ch.mc[p];
      Acc acc;
#pragma unroll
      for (int s = 0; s < kMaxAlpha; ++s)
        if (s < na) acc.mac(y[s], sw[s * nt + t], chunk, mc);
      eb[(long)t * n + i] = acc.done(mc);
    }
  }
}

// Key inner product over all digits: one thread per (target limb m, coeff i).
__global__ void __launch_bounds__(kThreads)
    ks_inner_kernel(const DevChain ch, const u64* __restrict__ d, long d_stride,
                    const u64* __restrict__ ext, long ext_stride, const u64* __restrict__ key,
                    int keyL, const int* __restrict__ dig_info, int D, int level, int K, int L,
                    u64* __restrict__ accQ, u64* __restrict__ accP, const u64* add0,
                    const u64* add1, long add_stride, u64* out0, u64* out1, long out_stride,
                    int batch, int chunk, int m_begin = 0, int m_end = -1) {
  extern __shared__ int sinfo[];
  for (int i = threadIdx.x; i < 4 * D; i += blockDim.x) sinfo[i] = dig_info[i];
  __syncthreads();
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const long total = (long)(m_end < 0 ? level + K : m_end) << log_n;
  for (long t = ((long)m_begin << log_n) + blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int m = (int)(t >> log_n);
    const long i = t & (n - 1);
    const int p = m < level ? m : L + (m - level);
    const ModConst mc = ch.mc[p];
    // small digit counts (hybrid): keep the key words in registers across the
    // batch so each key word is read from HBM once per call
    constexpr int kCache = 4;
    u64 kbc[kCache], kac[kCache];
    const bool cached = D <= kCache && D <= chunk;
    if (cached) {
#pragma unroll
      for (int di = 0; di < kCache; ++di) {
        if (di < D) {
          kbc[di] = key[((long)(2 * di) * keyL + p) * n + i];
          kac[di] = key[((long)(2 * di + 1) * keyL + p) * n + i];
        }
      }
    }
    if (cached) {
      // four batch items per iteration: all their operand loads are issued
      // before the first multiply, hiding HBM latency across the batch
      const u64* src[kCache];
      long sstr[kCache];
#pragma unroll
      for (int di = 0; di < kCache; ++di) {
        if (di < D) {
          const int s0 = sinfo[4 * di], na = sinfo[4 * di + 1], ro = sinfo[4 * di + 2];
          const bool own = m >= s0 && m < s0 + na;
          src[di] = own ? d + (long)m * n + i : ext + (long)(ro + (m < s0 ? m : m - na)) * n + i;
          sstr[di] = own ? d_stride : ext_stride;
        }
      }
      for (int b0 = 0; b0 < batch; b0 += 4) {
        u64 v[4][kCache];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int di = 0; di < kCache; ++di)
            if (di < D && b0 + u < batch) v[u][di] = __ldg(src[di] + (b0 + u) * sstr[di]);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (b0 + u >= batch) break;
          const int b = b0 + u;
          u64 bh = 0, bl = 0, ah = 0, al = 0;
#pragma unroll
          for (int di = 0; di < kCache; ++di) {
            if (di < D) {
              mac_wide(bh, bl, v[u][di], kbc[di]);
              mac_wide(ah, al, v[u][di], kac[di]);
            }
          }
          const u64 rb = reduce_fold(bh, bl, mc), ra = reduce_fold(ah, al, mc);
          if (K == 0) {
            const long o = b * out_stride + (long)m * n + i;
            const long ai = b * add_stride + (long)m * n + i;
            out0[o] = add0 ? add_mod(add0[ai], rb, mc.q) : rb;
            out1[o] = add1 ? add_mod(add1[ai], ra, mc.q) : ra;
          } else if (m < level) {
            accQ[((long)(b * 2 + 0) * level + m) * n + i] = rb;
            accQ[((long)(b * 2 + 1) * level + m) * n + i] = ra;
          } else {
            accP[((long)(b * 2 + 0) * K + (m - level)) * n + i] = rb;
            accP[((long)(b * 2 + 1) * K + (m - level)) * n + i] = ra;
          }
        }
      }
      continue;
    }
    for (int b = 0; b < batch; ++b) {
      u64 rb, ra;
      {
        Acc ab, aa;
        for (int di = 0; di < D; ++di) {
          const int s0 = sinfo[4 * di], na = sinfo[4 * di + 1], ro = sinfo[4 * di + 2];
          u64 v;
          if (m >= s0 && m < s0 + na) {
            v = d[b * d_stride + (long)m * n + i];
          } else {
            const int row = ro + (m < s0 ? m : m - na);
            v = ext[b * ext_stride + (long)row * n + i];
          }
          const u64 kb = key[((long)(2 * di) * keyL + p) * n + i];
          const u64 ka = key[((long)(2 * di + 1) * keyL + p) * n + i];
          ab.mac(v, kb, chunk, mc);
          aa.mac(v, ka, chunk, mc);
        }
        rb = ab.done(mc);
        ra = aa.done(mc);
      }
      if (K == 0) {
        const long o = b * out_stride + (long)m * n + i;
        const long ai = b * add_stride + (long)m * n + i;
        out0[o] = add0 ? add_mod(add0[ai], rb, mc.q) : rb;
        out1[o] = add1 ? add_mod(add1[ai], ra, mc.q) : ra;
      } else if (m < level) {
        accQ[((long)(b * 2 + 0) * level + m) * n + i] = rb;
        accQ[((long)(b * 2 + 1) * level + m) * n + i] = ra;
      } else {
        accP[((long)(b * 2 + 0) * K + (m - level)) * n + i] = rb;
        accP[((long)(b * 2 + 1) * K + (m - level)) * n + i] = ra;
      }
    }
  }
}

// ModDown base conversion P -> Q_level: grid (coef blocks, batch*2).
__global__ void __launch_bounds__(kThreads)
    moddown_conv_kernel(const DevChain ch, const u64* __restrict__ accP, u64* __restrict__ conv,
                        const WPair* __restrict__ down_inv, const u64* __restrict__ down_w,
                        int level, int K, int L, int chunk) {
  extern __shared__ u64 sw[];
  for (int i = threadIdx.x; i < K * level; i += blockDim.x) sw[i] = down_w[i];
  __syncthreads();
  const int bp = blockIdx.y;
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const u64* src = accP + (long)bp * K * n;
  u64* dst = conv + (long)bp * level * n;
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    u64 y[kMaxAlpha];
#pragma unroll
    for (int k = 0; k < kMaxAlpha; ++k) {
      if (k < K) {
        const WPair w = down_inv[k];
        y[k] = shoup_mul(src[(long)k * n + i], w.w, w.sh, ch.mc[L + k].q);
      }
    }
    int j = 0;
    for (; K <= chunk && j + 4 <= level; j += 4) {
      u64 hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < kMaxAlpha; ++k) {
        if (k < K) {
#pragma unroll
          for (int u = 0; u < 4; ++u) mac_wide(hi[u], lo[u], y[k], sw[k * level + j + u]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) dst[(long)(j + u) * n + i] = reduce_fold(hi[u], lo[u], ch.mc[j + u]);
    }
    for (; j < level; ++j) {
      const ModConst mc = ch.mc[j];
      Acc acc;
#pragma unroll
      for (int k = 0; k < kMaxAlpha; ++k)
        if (k < K) acc.mac(y[k], sw[k * level + j], chunk, mc);
      dst[(long)j * n + i] = acc.done(mc);
    }
  }
}

// out_p = add_p + (accQ_p - conv_p) * P^-1, p in {0 (b), 1 (a)}.
__global__ void __launch_bounds__(kThreads)
    moddown_finish_kernel(const DevChain ch, const u64* __restrict__ accQ,
                          const u64* __restrict__ conv, const WPair* __restrict__ p_inv,
                          const u64* add0, const u64* add1, long add_stride, u64* out0,
                          u64* out1, long out_stride, int level, int batch) {
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const long per = (long)level << log_n;
  const long total = (long)batch * 2 * per;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long bp = t / per;
    const long w = t - bp * per;
    const int j = (int)(w >> log_n);
    const int b = (int)(bp >> 1), poly = (int)(bp & 1);
    const u64 q = ch.mc[j].q;
    const WPair pi = p_inv[j];
    const u64 v = shoup_mul(sub_mod(accQ[t], conv[t], q), pi.w, pi.sh, q);
    const u64* add = poly ? add1 : add0;
    u64* out = poly ? out1 : out0;
    out[b * out_stride + w] = add ? add_mod(add[b * add_stride + w], v, q) : v;
  }
}

// ---------------------------------------------------------------------------
// FP64-pipe base conversions (every chain prime < 2^50): each term
// y_s * w_{s,m} mod p is an exact fp_mulmod (fparith.cuh) with w/p
// precomputed; up to 16 signed terms of |.| <= p/2 + eps sum exactly in a
// double (< 2^53) and are reduced once.  The same integers as the 128-bit
// integer accumulation, at half the pipe cost of the quarter-rate
// IMAD.WIDE products.

// canonical [0, q) representative as a double
__device__ __forceinline__ double fp_pos(double x, double q) { return x < 0.0 ? __dadd_rn(x, q) : x; }

// Per-target constants staged in shared memory; NSM bounds the digit size
// (registers), U targets are accumulated at once (independent FP64 chains).
template <int NSM, int U, int CPT = FHE_MODUP_CPT>
__global__ void __launch_bounds__(kThreads, FHE_MODUP_MINB)
    modup_fp_kernel(const DevChain ch, const u64* __restrict__ c, long c_stride,
                    u64* __restrict__ ext, long ext_stride, const int* __restrict__ dig_info,
                    const double2* __restrict__ up_inv, const double2* __restrict__ up_w, int level,
                    int K, int L) {
  fhe_pdl_trigger();
  fhe_pdl_wait();
  const int di = blockIdx.y, b = blockIdx.z;
  const int s0 = dig_info[4 * di], na = dig_info[4 * di + 1];
  const int row_off = dig_info[4 * di + 2], w_off = dig_info[4 * di + 3];
  const int nt = level + K - na;
  extern __shared__ double2 swd[];
  double2* tq = swd + na * nt;  // (p, 1/p) of each target
  for (int i = threadIdx.x; i < na * nt; i += blockDim.x) swd[i] = up_w[w_off + i];
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    const int m = t < s0 ? t : t + na;
    tq[t] = ch.qd[m < level ? m : L + (m - level)];
  }
  __syncthreads();
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const u64* cb = c + b * c_stride;
  u64* eb = ext + b * ext_stride + (long)row_off * n;
  // CPT coefficients per thread (i, i + n/CPT): each staged constant read
  // serves CPT independent accumulator chains
  for (long i0 = blockIdx.x * (long)blockDim.x + threadIdx.x; i0 < n / CPT;
       i0 += (long)gridDim.x * blockDim.x) {
    double y[CPT][NSM];
#pragma unroll
    for (int s = 0; s < NSM; ++s) {
      if (s < na) {
        const double q = ch.qd[s0 + s].x;
        // y_s = [c_s (Q_d/q_s)^-1]_{q_s}, canonical: the conversion is an
        // integer-level formula, so the representative matters
#pragma unroll
        for (int c = 0; c < CPT; ++c)
          y[c][s] = fp_pos(fp_mulmod(fp_from_u52(cb[(long)(s0 + s) * n + i0 + c * (n / CPT)]),
                                     up_inv[s0 + s], q),
                           q);
      }
    }
    int t = 0;
    for (; t + U <= nt; t += U) {
      double acc[CPT][U];
#pragma unroll
      for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int u = 0; u < U; ++u) acc[c][u] = 0.0;
#pragma unroll
      for (int s = 0; s < NSM; ++s) {
        if (s < na) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const double2 w = swd[s * nt + t + u];
            const double qv = tq[t + u].x;
#pragma unroll
            for (int c = 0; c < CPT; ++c)
              acc[c][u] = __dadd_rn(acc[c][u], fp_mulmod(y[c][s], w, qv));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double2 qd = tq[t + u];
#pragma unroll
        for (int c = 0; c < CPT; ++c)
          eb[(long)(t + u) * n + i0 + c * (n / CPT)] = fp_canon(fp_reduce(acc[c][u], qd), qd.x);
      }
    }
    for (; t < nt; ++t) {
      const double2 qd = tq[t];
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int s = 0; s < NSM; ++s)
          if (s < na) acc = __dadd_rn(acc, fp_mulmod(y[c][s], swd[s * nt + t], qd.x));
        eb[(long)t * n + i0 + c * (n / CPT)] = fp_canon(fp_reduce(acc, qd), qd.x);
      }
    }
  }
}

template <int NSM, int U, int CPT = FHE_MODUP_CPT>
__global__ void __launch_bounds__(kThreads, FHE_MODUP_MINB)
    moddown_conv_fp_kernel(const DevChain ch, const u64* __restrict__ accP,
                           u64* __restrict__ conv, const double2* __restrict__ down_inv,
                           const double2* __restrict__ down_w, int level, int K, int L) {
  extern __shared__ double2 swd[];
  double2* tq = swd + K * level;  // (q, 1/q) of each target
  for (int i = threadIdx.x; i < K * level; i += blockDim.x) swd[i] = down_w[i];
  for (int j = threadIdx.x; j < level; j += blockDim.x) tq[j] = ch.qd[j];
  __syncthreads();
  const int bp = blockIdx.y;
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const u64* src = accP + (long)bp * K * n;
  u64* dst = conv + (long)bp * level * n;
  // CPT coefficients per thread (i, i + n/CPT) share each staged constant
  for (long i0 = blockIdx.x * (long)blockDim.x + threadIdx.x; i0 < n / CPT;
       i0 += (long)gridDim.x * blockDim.x) {
    double y[CPT][NSM];
#pragma unroll
    for (int k = 0; k < NSM; ++k) {
      if (k < K) {
        const double p = ch.qd[L + k].x;
#pragma unroll
        for (int c = 0; c < CPT; ++c)
          y[c][k] = fp_pos(fp_mulmod(fp_from_u52(src[(long)k * n + i0 + c * (n / CPT)]),
                                     down_inv[k], p),
                           p);
      }
    }
    int j = 0;
    for (; j + U <= level; j += U) {
      double acc[CPT][U];
#pragma unroll
      for (int c = 0; c < CPT; ++c)
#pragma unroll
        for (int u = 0; u < U; ++u) acc[c][u] = 0.0;
#pragma unroll
      for (int k = 0; k < NSM; ++k) {
        if (k < K) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const double2 w = swd[k * level + j + u];
            const double qv = tq[j + u].x;
#pragma unroll
            for (int c = 0; c < CPT; ++c)
              acc[c][u] = __dadd_rn(acc[c][u], fp_mulmod(y[c][k], w, qv));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double2 qd = tq[j + u];
#pragma unroll
        for (int c = 0; c < CPT; ++c)
          dst[(long)(j + u) * n + i0 + c * (n / CPT)] = fp_canon(fp_reduce(acc[c][u], qd), qd.x);
      }
    }
    for (; j < level; ++j) {
      const double2 qd = tq[j];
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < NSM; ++k)
          if (k < K) acc = __dadd_rn(acc, fp_mulmod(y[c][k], swd[k * level + j], qd.x));
        dst[(long)j * n + i0 + c * (n / CPT)] = fp_canon(fp_reduce(acc, qd), qd.x);
      }
    }
  }
}

// FP64-pipe key inner product (every chain prime < 2^50, at most 4 digits):
// the key words are variable operands, so their quotient estimates key/p
// are formed on the fly (one DMUL); each term is an exact fp_mulmod, the
// digit sum (|.| <= 4 * 0.75 p) is reduced once.
// Output limbs m in [m_begin, m_end).  FIN: Q limbs only, and instead of
// storing accQ the ModDown finish is applied in place of moddown_finish_kernel:
// out = add + (acc - conv) P^-1 (conv = the NTT'd P->Q conversion), so accQ
// never round-trips HBM.
// TENS (fused HMult+Relin, with FIN): add0/add1 are the two input ciphertexts
// x, y ((2, level, n) each, add_stride apart); the tensor terms
// d0 = x0 y0, d1 = x0 y1 + x1 y0 and the own-digit word d2 = x1 y1 are formed
// here from the inputs (ckks.py ckks_multiply), so d0/d1 never touch HBM.
template <int kD, bool FIN = false, bool TENS = false>
__global__ void __launch_bounds__(kThreads, TENS  ? FHE_TENS_MINB
                                            : (FIN ? FHE_FIN_MINB : FHE_INNER_MINB))
    ks_inner_fp_kernel(const DevChain ch, const u64* __restrict__ d, long d_stride,
                       const u64* __restrict__ ext, long ext_stride, const u64* __restrict__ key,
                       int keyL, const int* __restrict__ dig_info, int D, int level, int K, int L,
                       u64* __restrict__ accQ, u64* __restrict__ accP, const u64* add0,
                       const u64* add1, long add_stride, u64* out0, u64* out1, long out_stride,
                       int batch, int m_begin, int m_end, const u64* __restrict__ conv,
                       const WPair* __restrict__ p_inv) {
  // kD: digits (template: registers sized to the key's dnum)
  extern __shared__ int sinfo[];
  for (int i = threadIdx.x; i < 4 * D; i += blockDim.x) sinfo[i] = dig_info[i];
  __syncthreads();
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const long total = (long)(m_end - m_begin) << log_n;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int m = m_begin + (int)(t >> log_n);
    const long i = t & (n - 1);
    const int p = m < level ? m : L + (m - level);
    const double2 qd = ch.qd[p];
    const u64 q = ch.mc[p].q;
    double2 kb[kD], ka[kD];
    const u64* src[kD];
    long sstr[kD];
    int own_di = -1;
#pragma unroll
    for (int di = 0; di < kD; ++di) {
      if (di < D) {
        const double b = fp_from_u52(__ldg(key + ((long)(2 * di) * keyL + p) * n + i));
        const double a = fp_from_u52(__ldg(key + ((long)(2 * di + 1) * keyL + p) * n + i));
        kb[di] = make_double2(b, __dmul_rn(b, qd.y));
        ka[di] = make_double2(a, __dmul_rn(a, qd.y));
        const int s0 = sinfo[4 * di], na = sinfo[4 * di + 1], ro = sinfo[4 * di + 2];
        const bool own = m >= s0 && m < s0 + na;
        if (own) own_di = di;
        src[di] = own ? d + (long)m * n + i : ext + (long)(ro + (m < s0 ? m : m - na)) * n + i;
        sstr[di] = own ? d_stride : ext_stride;
      }
    }
    for (int b0 = 0; b0 < batch; b0 += FHE_INNER_BU) {
      u64 v[FHE_INNER_BU][kD];
      // FIN: the finish operands are loaded with the digits (all in flight)
      u64 cv[FIN ? FHE_INNER_BU : 1][2], av[FIN ? FHE_INNER_BU : 1][2];
      u64 tx[TENS ? FHE_INNER_BU : 1][2], ty[TENS ? FHE_INNER_BU : 1][2];
#pragma unroll
      for (int u = 0; u < FHE_INNER_BU; ++u) {
#pragma unroll
        for (int di = 0; di < kD; ++di)
          if (di < D && b0 + u < batch && !(TENS && di == own_di))
            v[u][di] = __ldg(src[di] + (b0 + u) * sstr[di]);
        if constexpr (FIN) {
          if (b0 + u < batch) {
            const int bb = b0 + u;
            const long w = (long)m * n + i;
            cv[u][0] = conv[((long)(bb * 2 + 0) * level + m) * n + i];
            cv[u][1] = conv[((long)(bb * 2 + 1) * level + m) * n + i];
            if constexpr (TENS) {
              const u64* xb = add0 + bb * add_stride + w;
              const u64* yb = add1 + bb * add_stride + w;
              // plain (coherent) loads: out0/out1 may alias x (fhe_sm100.h),
              // so x is not read-only for the duration of the kernel
              tx[u][0] = xb[0];
              tx[u][1] = xb[(long)level * n];
              ty[u][0] = yb[0];
              ty[u][1] = yb[(long)level * n];
            } else {
              av[u][0] = add0 ? add0[bb * add_stride + w] : 0;
              av[u][1] = add1 ? add1[bb * add_stride + w] : 0;
            }
          }
        }
      }
#pragma unroll
      for (int u = 0; u < FHE_INNER_BU; ++u) {
        if (b0 + u >= batch) break;
        const int b = b0 + u;
        double d2 = 0.0;
        if constexpr (TENS) {
          // tensor terms on the FP64 pipe (idle in this HBM-bound kernel):
          // exact products of canonical words as in the inner product below
          const double a0 = fp_from_u52(tx[u][0]), a1 = fp_from_u52(tx[u][1]);
          const double c0 = fp_from_u52(ty[u][0]), c1 = fp_from_u52(ty[u][1]);
          const double2 w0 = make_double2(c0, __dmul_rn(c0, qd.y));
          const double2 w1 = make_double2(c1, __dmul_rn(c1, qd.y));
          av[u][0] = fp_canon_half(fp_reduce(fp_mulmod(a0, w0, qd.x), qd), qd.x);
          av[u][1] = fp_canon_half(
              fp_reduce(__dadd_rn(fp_mulmod(a0, w1, qd.x), fp_mulmod(a1, w0, qd.x)), qd), qd.x);
          const double r2 = fp_reduce(fp_mulmod(a1, w1, qd.x), qd);
          d2 = r2 < 0.0 ? __dadd_rn(r2, qd.x) : r2;
        }
        double sb = 0.0, sa = 0.0;
#pragma unroll
        for (int di = 0; di < kD; ++di) {
          if (di < D) {
            const double x = (TENS && di == own_di) ? d2 : fp_from_u52(v[u][di]);
            sb = __dadd_rn(sb, fp_mulmod(x, kb[di], qd.x));
            sa = __dadd_rn(sa, fp_mulmod(x, ka[di], qd.x));
          }
        }
        const u64 rb = fp_canon_half(fp_reduce(sb, qd), qd.x);
        const u64 ra = fp_canon_half(fp_reduce(sa, qd), qd.x);
        if constexpr (FIN) {
          const WPair pi = p_inv[m];
          const long w = (long)m * n + i;
          u64 v0 = shoup_mul(sub_mod(rb, cv[u][0], q), pi.w, pi.sh, q);
          u64 v1 = shoup_mul(sub_mod(ra, cv[u][1], q), pi.w, pi.sh, q);
          if (TENS || add0) v0 = add_mod(av[u][0], v0, q);
          if (TENS || add1) v1 = add_mod(av[u][1], v1, q);
          out0[b * out_stride + w] = v0;
          out1[b * out_stride + w] = v1;
          continue;
        }
        if (K == 0) {
          const long o = b * out_stride + (long)m * n + i;
          const long ai = b * add_stride + (long)m * n + i;
          out0[o] = add0 ? add_mod(add0[ai], rb, q) : rb;
          out1[o] = add1 ? add_mod(add1[ai], ra, q) : ra;
        } else if (m < level) {
          accQ[((long)(b * 2 + 0) * level + m) * n + i] = rb;
          accQ[((long)(b * 2 + 1) * level + m) * n + i] = ra;
        } else {
          accP[((long)(b * 2 + 0) * K + (m - level)) * n + i] = rb;
          accP[((long)(b * 2 + 1) * K + (m - level)) * n + i] = ra;
        }
      }
    }
  }
}

// Staged variant of ks_inner_fp_kernel<kD, true, TENS> (the fused Q-limb
// inner product + ModDown finish, the largest single HBM stream of HMult+Relin).
// The register-blocked kernel keeps FHE_INNER_BU batch items of loads in
// flight and then computes with none in flight, so at 2 CTAs/SM it ran
// latency-bound (ncu: 49% of DRAM peak, 54% long-scoreboard stalls on the
// first use of each word).  Here every operand word of batch item b + ST - 1
// is copied into this thread's shared-memory slots with cp.async (8-byte
// .ca copies, no registers held) while item b computes, so ST - 1 items per
// thread are always in flight.  Each thread reads back only the slots it
// filled itself, so wait_group alone orders the pipeline (no CTA barrier).
// Arithmetic and results are those of ks_inner_fp_kernel word for word.
__device__ __forceinline__ void ks_cp8(u64* s, const u64* g) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(a), "l"(g) : "memory");
}
__device__ __forceinline__ void ks_cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ks_cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

#ifndef FHE_FIN_STAGES
#define FHE_FIN_STAGES 4
#endif
// the staged finish's ModDown step on the FP64 pipe (0: integer Shoup form)
#ifndef FHE_FIN_FP
#define FHE_FIN_FP 1
#endif
#ifndef FHE_FINS_MINB
#define FHE_FINS_MINB 3
#endif

template <int kD, bool TENS>
constexpr int fin_words() {
  return TENS ? (kD - 1) + 2 + 4 : kD + 2 + 2;
}

template <int kD, bool TENS>
size_t fin_staged_smem() {
  return 64 + (size_t)FHE_FIN_STAGES * fin_words<kD, TENS>() * kThreads * sizeof(u64);
}

template <int kD, bool TENS>
__global__ void __launch_bounds__(kThreads, FHE_FINS_MINB)
    ks_fin_staged_kernel(const DevChain ch, const u64* __restrict__ d, long d_stride,
                         const u64* __restrict__ ext, long ext_stride, const u64* __restrict__ key,
                         int keyL, const int* __restrict__ dig_info, int D, int level,
                         const u64* add0, const u64* add1, long add_stride, u64* out0, u64* out1,
                         long out_stride, int batch, const u64* __restrict__ conv,
                         const WPair* __restrict__ p_inv, const double2* __restrict__ p_inv_d) {
  constexpr int W = fin_words<kD, TENS>();
  constexpr int ST = FHE_FIN_STAGES;
  extern __shared__ __align__(16) unsigned char fsm[];
  int* sinfo = reinterpret_cast<int*>(fsm);
  u64* stage = reinterpret_cast<u64*>(fsm + 64);
  if (threadIdx.x < 4 * D) sinfo[threadIdx.x] = dig_info[threadIdx.x];
  __syncthreads();
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const long total = (long)level << log_n;
  // slot (s, w) of this thread
  auto slot = [&](int s, int w) { return stage + ((long)(s * W + w) * kThreads + threadIdx.x); };
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int m = (int)(t >> log_n);
    const long i = t & (n - 1);
    const long w = (long)m * n + i;
    const double2 qd = ch.qd[m];
    const u64 q = ch.mc[m].q;
    const u64* src[kD];
    long sstr[kD];
    int own_di = -1;
#pragma unroll
    for (int di = 0; di < kD; ++di) {
      if (di < D) {
        const int s0 = sinfo[4 * di], na = sinfo[4 * di + 1], ro = sinfo[4 * di + 2];
        const bool own = m >= s0 && m < s0 + na;
        if (own) own_di = di;
        src[di] = own ? d + w : ext + (long)(ro + (m < s0 ? m : m - na)) * n + i;
        sstr[di] = own ? d_stride : ext_stride;
      }
    }
    // word order in a stage: digits (own digit skipped under TENS), conv b/a,
    // then x0 x1 y0 y1 (TENS) or add0 add1
    auto issue = [&](int b) {
      if (b < batch) {
        const int s = b % ST;
        int k = 0;
#pragma unroll
        for (int di = 0; di < kD; ++di) {
          if (di < D && !(TENS && di == own_di)) ks_cp8(slot(s, k), src[di] + b * sstr[di]);
          if (di < D && !(TENS && di == own_di)) ++k;
        }
        k = TENS ? kD - 1 : kD;
        ks_cp8(slot(s, k), conv + ((long)(b * 2 + 0) * level) * n + w);
        ks_cp8(slot(s, k + 1), conv + ((long)(b * 2 + 1) * level) * n + w);
        if constexpr (TENS) {
          const u64* xb = add0 + b * add_stride + w;
          const u64* yb = add1 + b * add_stride + w;
          ks_cp8(slot(s, k + 2), xb);
          ks_cp8(slot(s, k + 3), xb + (long)level * n);
          ks_cp8(slot(s, k + 4), yb);
          ks_cp8(slot(s, k + 5), yb + (long)level * n);
        } else {
          if (add0) ks_cp8(slot(s, k + 2), add0 + b * add_stride + w);
          if (add1) ks_cp8(slot(s, k + 3), add1 + b * add_stride + w);
        }
      }
      ks_cp_commit();  // always one group per step (empty past the end)
    };
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) issue(s);
    double2 kb[kD], ka[kD];
#pragma unroll
    for (int di = 0; di < kD; ++di) {
      if (di < D) {
        const double b = fp_from_u52(__ldg(key + ((long)(2 * di) * keyL + m) * n + i));
        const double a = fp_from_u52(__ldg(key + ((long)(2 * di + 1) * keyL + m) * n + i));
        kb[di] = make_double2(b, __dmul_rn(b, qd.y));
        ka[di] = make_double2(a, __dmul_rn(a, qd.y));
      }
    }
    const WPair pi = p_inv[m];
    const double2 pd = p_inv_d[m];
    for (int b = 0; b < batch; ++b) {
      issue(b + ST - 1);
      ks_cp_wait<ST - 1>();
      const int s = b % ST;
      const int k0 = TENS ? kD - 1 : kD;
      double d2 = 0.0;
      u64 av0 = 0, av1 = 0;
      double avd0 = 0.0, avd1 = 0.0;
      if constexpr (TENS) {
        const double a0 = fp_from_u52(*slot(s, k0 + 2)), a1 = fp_from_u52(*slot(s, k0 + 3));
        const double c0 = fp_from_u52(*slot(s, k0 + 4)), c1 = fp_from_u52(*slot(s, k0 + 5));
        const double2 w0 = make_double2(c0, __dmul_rn(c0, qd.y));
        const double2 w1 = make_double2(c1, __dmul_rn(c1, qd.y));
#if FHE_FIN_FP
        avd0 = fp_mulmod(a0, w0, qd.x);
        avd1 = fp_reduce(__dadd_rn(fp_mulmod(a0, w1, qd.x), fp_mulmod(a1, w0, qd.x)), qd);
#else
        av0 = fp_canon_half(fp_reduce(fp_mulmod(a0, w0, qd.x), qd), qd.x);
        av1 = fp_canon_half(
            fp_reduce(__dadd_rn(fp_mulmod(a0, w1, qd.x), fp_mulmod(a1, w0, qd.x)), qd), qd.x);
#endif
        const double r2 = fp_reduce(fp_mulmod(a1, w1, qd.x), qd);
        d2 = r2 < 0.0 ? __dadd_rn(r2, qd.x) : r2;
      } else {
        if (add0) av0 = *slot(s, k0 + 2);
        if (add1) av1 = *slot(s, k0 + 3);
#if FHE_FIN_FP
        avd0 = add0 ? fp_from_u52(av0) : 0.0;
        avd1 = add1 ? fp_from_u52(av1) : 0.0;
#endif
      }
      double sb = 0.0, sa = 0.0;
      int k = 0;
#pragma unroll
      for (int di = 0; di < kD; ++di) {
        if (di < D) {
          double x;
          if (TENS && di == own_di) {
            x = d2;
          } else {
            x = fp_from_u52(*slot(s, k));
            ++k;
          }
          sb = __dadd_rn(sb, fp_mulmod(x, kb[di], qd.x));
          sa = __dadd_rn(sa, fp_mulmod(x, ka[di], qd.x));
        }
      }
#if FHE_FIN_FP
      // ModDown finish on the FP64 pipe: (acc - conv) P^-1 + add with signed
      // representatives (|acc - conv| < 1.5 q, |product| <= q/2, |sum| < 2q),
      // one reduction and the canonical word -- the same word as the integer
      // Shoup form below
      const double yb = fp_mulmod(__dadd_rn(fp_reduce(sb, qd), -fp_from_u52(*slot(s, k0))), pd,
                                  qd.x);
      const double ya = fp_mulmod(__dadd_rn(fp_reduce(sa, qd), -fp_from_u52(*slot(s, k0 + 1))),
                                  pd, qd.x);
      out0[b * out_stride + w] =
          (TENS || add0) ? fp_canon_half(fp_reduce(__dadd_rn(yb, avd0), qd), qd.x)
                         : fp_canon_half(yb, qd.x);
      out1[b * out_stride + w] =
          (TENS || add1) ? fp_canon_half(fp_reduce(__dadd_rn(ya, avd1), qd), qd.x)
                         : fp_canon_half(ya, qd.x);
#else
      const u64 rb = fp_canon_half(fp_reduce(sb, qd), qd.x);
      const u64 ra = fp_canon_half(fp_reduce(sa, qd), qd.x);
      u64 v0 = shoup_mul(sub_mod(rb, *slot(s, k0), q), pi.w, pi.sh, q);
      u64 v1 = shoup_mul(sub_mod(ra, *slot(s, k0 + 1), q), pi.w, pi.sh, q);
      if (TENS || add0) v0 = add_mod(av0, v0, q);
      if (TENS || add1) v1 = add_mod(av1, v1, q);
      out0[b * out_stride + w] = v0;
      out1[b * out_stride + w] = v1;
#endif
    }
    ks_cp_wait<0>();
  }
}

// P-limb key inner product of the fused path (m in [level, level + K): no
// digit owns a P limb, every term reads ext), writing accP for the ModDown
// conversion -- the staged counterpart of ks_inner_fp_kernel<kD> over those
// limbs: the D words of batch item b + ST - 1 are in flight (cp.async into
// this thread's slots) while item b computes.  Same arithmetic, same words.
template <int kD>
__global__ void __launch_bounds__(kThreads, FHE_FINS_MINB)
    ks_plimb_staged_kernel(const DevChain ch, const u64* __restrict__ ext, long ext_stride,
                           const u64* __restrict__ key, int keyL,
                           const int* __restrict__ dig_info, int D, int level, int K, int L,
                           u64* __restrict__ accP, int batch) {
  constexpr int ST = FHE_FIN_STAGES;
  extern __shared__ __align__(16) unsigned char psm[];
  int* sinfo = reinterpret_cast<int*>(psm);
  u64* stage = reinterpret_cast<u64*>(psm + 64);
  if (threadIdx.x < 4 * D) sinfo[threadIdx.x] = dig_info[threadIdx.x];
  __syncthreads();
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  const long total = (long)K << log_n;
  auto slot = [&](int s, int w) { return stage + ((long)(s * kD + w) * kThreads + threadIdx.x); };
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int k = (int)(t >> log_n);
    const int m = level + k, p = L + k;
    const long i = t & (n - 1);
    const double2 qd = ch.qd[p];
    const u64* src[kD];
#pragma unroll
    for (int di = 0; di < kD; ++di)
      if (di < D) src[di] = ext + (long)(sinfo[4 * di + 2] + m - sinfo[4 * di + 1]) * n + i;
    auto issue = [&](int b) {
      if (b < batch) {
#pragma unroll
        for (int di = 0; di < kD; ++di)
          if (di < D) ks_cp8(slot(b % ST, di), src[di] + b * ext_stride);
      }
      ks_cp_commit();
    };
#pragma unroll
    for (int s = 0; s < ST - 1; ++s) issue(s);
    double2 kb[kD], ka[kD];
#pragma unroll
    for (int di = 0; di < kD; ++di) {
      if (di < D) {
        const double b = fp_from_u52(__ldg(key + ((long)(2 * di) * keyL + p) * n + i));
        const double a = fp_from_u52(__ldg(key + ((long)(2 * di + 1) * keyL + p) * n + i));
        kb[di] = make_double2(b, __dmul_rn(b, qd.y));
        ka[di] = make_double2(a, __dmul_rn(a, qd.y));
      }
    }
    for (int b = 0; b < batch; ++b) {
      issue(b + ST - 1);
      ks_cp_wait<ST - 1>();
      double sb = 0.0, sa = 0.0;
#pragma unroll
      for (int di = 0; di < kD; ++di) {
        if (di < D) {
          const double x = fp_from_u52(*slot(b % ST, di));
          sb = __dadd_rn(sb, fp_mulmod(x, kb[di], qd.x));
          sa = __dadd_rn(sa, fp_mulmod(x, ka[di], qd.x));
        }
      }
      accP[((long)(b * 2 + 0) * K + k) * n + i] = fp_canon_half(fp_reduce(sb, qd), qd.x);
      accP[((long)(b * 2 + 1) * K + k) * n + i] = fp_canon_half(fp_reduce(sa, qd), qd.x);
    }
    ks_cp_wait<0>();
  }
}

// FP64 key inner product for many digits (the reference's per-prime gadget,
// alpha = 1, D = level digits): digits stream through one accumulator pair
// per output, reduced every 8 terms (|sum| <= 8 * 0.75p + p < 2^53).
__global__ void __launch_bounds__(kThreads)
    ks_inner_fp_many_kernel(const DevChain ch, const u64* __restrict__ d, long d_stride,
                            const u64* __restrict__ ext, long ext_stride,
                            const u64* __restrict__ key, int keyL,
                            const int* __restrict__ dig_info, int D, int level, int K, int L,
                            u64* __restrict__ accQ, u64* __restrict__ accP, const u64* add0,
                            const u64* add1, long add_stride, u64* out0, u64* out1,
                            long out_stride, int batch) {
  fhe_pdl_trigger();
  fhe_pdl_wait();
  extern __shared__ int sinfo[];
  for (int i = threadIdx.x; i < 4 * D; i += blockDim.x) sinfo[i] = dig_info[i];
  __syncthreads();
  const int log_n = ch.log_n;
  const long n = 1L << log_n;
  // one thread per (batch item, output limb, coefficient): at the small
  // ring degrees this kernel serves (the per-prime gadget of the PDQ
  // profile, N = 4096) a thread per (limb, coefficient) looping over the
  // batch left most of the GPU idle; the key words are re-read per item
  // from L2
  const long per_b = (long)(level + K) << log_n;
  const long total = per_b * batch;
  for (long tt = blockIdx.x * (long)blockDim.x + threadIdx.x; tt < total;
       tt += (long)gridDim.x * blockDim.x) {
    const int b = (int)(tt / per_b);
    const long t = tt - (long)b * per_b;
    const int m = (int)(t >> log_n);
    const long i = t & (n - 1);
    const int p = m < level ? m : L + (m - level);
    const double2 qd = ch.qd[p];
    const u64 q = ch.mc[p].q;
    {
      // digits in chunks of 8: the chunk's 24 words are all loaded before
      // any is used (one memory latency per chunk instead of one per few
      // digits), then summed in digit order, reduced after every 8 terms
      double sb = 0.0, sa = 0.0;
      for (int d0 = 0; d0 < D; d0 += 8) {
        u64 xw[8], bw[8], aw[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int di = d0 + u;
          if (di < D) {
            const int s0 = sinfo[4 * di], na = sinfo[4 * di + 1], ro = sinfo[4 * di + 2];
            const bool own = m >= s0 && m < s0 + na;
            const u64* src = own ? d + b * d_stride + (long)m * n + i
                                 : ext + b * ext_stride + (long)(ro + (m < s0 ? m : m - na)) * n + i;
            xw[u] = __ldg(src);
            bw[u] = __ldg(key + ((long)(2 * di) * keyL + p) * n + i);
            aw[u] = __ldg(key + ((long)(2 * di + 1) * keyL + p) * n + i);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (d0 + u < D) {
            const double x = fp_from_u52(xw[u]);
            const double kbv = fp_from_u52(bw[u]), kav = fp_from_u52(aw[u]);
            sb = __dadd_rn(sb, fp_mulmod(x, make_double2(kbv, __dmul_rn(kbv, qd.y)), qd.x));
            sa = __dadd_rn(sa, fp_mulmod(x, make_double2(kav, __dmul_rn(kav, qd.y)), qd.x));
          }
        }
        sb = fp_reduce(sb, qd);
        sa = fp_reduce(sa, qd);
      }
      const u64 rb = fp_canon_half(fp_reduce(sb, qd), qd.x);
      const u64 ra = fp_canon_half(fp_reduce(sa, qd), qd.x);
      if (K == 0) {
        const long o = b * out_stride + (long)m * n + i;
        const long ai = b * add_stride + (long)m * n + i;
        out0[o] = add0 ? add_mod(add0[ai], rb, q) : rb;
        out1[o] = add1 ? add_mod(add1[ai], ra, q) : ra;
      } else if (m < level) {
        accQ[((long)(b * 2 + 0) * level + m) * n + i] = rb;
        accQ[((long)(b * 2 + 1) * level + m) * n + i] = ra;
      } else {
        accP[((long)(b * 2 + 0) * K + (m - level)) * n + i] = rb;
        accP[((long)(b * 2 + 1) * K + (m - level)) * n + i] = ra;
      }
    }
  }
}

// FHE_FIN_STAGED=0 selects the register-blocked finish kernel
static bool fin_staged_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_FIN_STAGED");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// FHE_RESCALE_FUSED_FIN=0: the rescale finish as its own kernel
static bool rescale_fin_fused_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_RESCALE_FUSED_FIN");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// FHE_MIXED_KS=0: a mixed chain's key switch stays entirely on the integer path
static bool mixed_keyswitch_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_MIXED_KS");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// FHE_BCAST_MODUP=0: per-prime gadget ModUp through the conversion kernel
static bool bcast_modup_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_BCAST_MODUP");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

bool fin_inner_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_FUSE_INNER_FINISH");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

bool fuse_finish_enabled() {
  static int on = -1;
  if (on < 0) {
    // opt-in: measured on par with the separate finish pass (profiles/r1_ntt_notes.md)
    const char* e = getenv("FHE_FUSE_MODDOWN");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

#include "bconv_imma.cuh"
#include "bconv_umma.cuh"

// tcgen05 base conversion (default; FHE_BCONV_UMMA=0 takes the mma.sync kernels)
bool bconv_umma_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_BCONV_UMMA");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// CTAs per job for the tcgen05 conversion: one wave of FHE_BU_MINB CTAs per
// SM over all jobs, each CTA looping over 128-coefficient tiles
static unsigned bu_grid_x(long n, int jobs) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const long tiles = n / kBuTile;
  return (unsigned)std::max<long>(1, std::min<long>(tiles, (long)sms * FHE_BU_MINB / jobs));
}

// tensor-core base conversions (default when the level has the tables and a
// digit of >= 4 limbs; FHE_BCONV_IMMA=0 keeps the FP64 / integer kernels)
bool bconv_imma_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_BCONV_IMMA");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// register-resident epilogue of the tensor-core conversion (default;
// FHE_BCONV_LAYOUT=1 takes the shared-memory transpose variant)
bool bconv_layout2() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_BCONV_LAYOUT");
    on = (e && e[0] == '1') ? 0 : 1;
  }
  return on == 1;
}

int mac_chunk(const std::vector<u64>& primes) {
  u64 mx = 0;
  for (u64 p : primes) mx = p > mx ? p : mx;
  const int bits = 64 - __builtin_clzll(mx);
  const int room = 126 - 2 * bits;  // accumulator headroom in bits
  if (room >= 20) return 1 << 20;
  return room <= 0 ? 1 : (1 << room);
}

}  // namespace

size_t keyswitch_workspace(const FheContext& ctx, int level, int batch) {
  const LevelPlan& lp = ctx.levels[level];
  const size_t n = (size_t)1 << ctx.chain->log_n;
  size_t rows = (size_t)batch * (level + lp.ext_rows);
  if (ctx.K > 0) rows += (size_t)batch * (2 * level + 2 * ctx.K + 2 * level);
  return rows * n * sizeof(u64);
}

// The fused inner-product/finish kernel handles this level (FP64 chain, hybrid
// key with at most 4 digits, not disabled by FHE_FUSE_INNER_FINISH=0).
// the fused Q-limb inner product + ModDown finish (FP64 pipe): FP64 chains,
// and mixed chains whose level Q primes are < 2^50 (their P-limb inner
// product then runs on the integer pipe)
static bool fin_inner_path(const FheContext& ctx, int level) {
  const LevelPlan& lp = ctx.levels[level];
  const bool fp = ctx.chain->dev.fp64_ok ||
                  (lp.p_inv_d && ctx.chain->dev.twd && mixed_keyswitch_enabled());
  return ctx.K > 0 && fp && lp.digits <= 4 && fin_inner_enabled();
}

int run_keyswitch(const FheContext& ctx, int level, const u64* d, long d_stride, const u64* key,
                  const u64* add0, const u64* add1, long add_stride, u64* out0, u64* out1,
                  long out_stride, int batch, void* ws, size_t ws_bytes, cudaStream_t st,
                  bool tens) {
  if (level < 1 || level > ctx.L) {
    fhe_set_error("keyswitch level out of range");
    return -1;
  }
  if (ctx.alpha > kMaxAlpha || ctx.K > kMaxAlpha) {
    fhe_set_error("alpha and K must be <= 16");
    return -1;
  }
  if (ws_bytes < keyswitch_workspace(ctx, level, batch)) {
    fhe_set_error("keyswitch workspace too small");
    return -1;
  }
  const LevelPlan& lp = ctx.levels[level];
  const DevChain& ch = ctx.chain->dev;
  const int log_n = ch.log_n, K = ctx.K, L = ctx.L;
  const long n = 1L << log_n;
  const int chunk = mac_chunk(ctx.chain->primes);
  u64* c = (u64*)ws;
  u64* ext = c + (long)batch * level * n;
  u64* accQ = ext + (long)batch * lp.ext_rows * n;
  u64* accP = accQ + (long)batch * 2 * level * n;
  u64* conv = accP + (long)batch * 2 * K * n;
  int rc;
  // 1. coefficient form of the input
  rc = launch_ntt(ch, NttArgs{c, d, batch * level, RowMap{nullptr, level, 0}, d_stride, 0},
                  true, st);
  if (rc) return rc;
  // 2. ModUp: basis extension of every digit, then NTT of the extended rows.
  // Per-prime gadget (alpha = 1, K = 0) on the rows path: ext(d, m) = c_d mod
  // q_m, so the forward NTT of the ext rows reads the coefficient rows c_d
  // themselves as a broadcast input (no conversion kernel, no ext write +
  // re-read).  The words c_d < 2^50 enter the FP64 butterflies unreduced,
  // which stay below 2^52 until the first lazy reduction (stage 3); the
  // transform's canonical output is NTT_m(c_d mod q_m) word for word.
  // mixed chain whose Q primes are all < 2^50 (P >= 2^50): the Q-limb parts
  // of the ext transform and of the inner product take the FP64 pipe
  bool mixed_q_fp64 = !ch.fp64_ok && ch.twd && K > 0 && mixed_keyswitch_enabled();
  for (int j = 0; mixed_q_fp64 && j < level; ++j)
    mixed_q_fp64 = ctx.chain->fp64_prime[j] != 0;
  bool modup_done = false;
  if (lp.max_na == 1 && K == 0 && ch.fp64_ok && log_n <= 12 && lp.ext_rows > 0 &&
      bcast_modup_enabled()) {
    NttArgs na{ext, ext, batch * lp.ext_rows, RowMap{lp.ext_prime, lp.ext_rows, 0}, 0, 0};
    na.bcast_src = c;
    na.bcast_stride = n;
    na.center_q = 0;
    na.bcast_div = level - 1;
    na.bcast_done = &modup_done;
    rc = launch_ntt(ch, na, false, st);
    if (rc) return rc;
  }
  if (!modup_done) {
    int max_w = 0;
    for (int di = 0; di < lp.digits; ++di)
      max_w = std::max(max_w, lp.dig_na[di] * (level + K - lp.dig_na[di]));
    const size_t smem = (size_t)max_w * sizeof(u64);
    dim3 grid((unsigned)std::max<long>(1, std::min<long>(n / kThreads, 1024)), lp.digits, batch);
    const bool umma_up = bconv_umma_enabled() && n >= kBuTile && lp.up_bu;
    if (lp.bf_ok && lp.max_na >= 4 && bconv_imma_enabled() && (umma_up || !lp.bf_wide)) {
      const bool l2 = bconv_layout2();
      BconvArgs ba{c, (long)level * n, ext, (long)lp.ext_rows * n, lp.dig_info,
                   l2 ? lp.up_bf2_off : lp.up_bf_off, l2 ? lp.up_bf2 : lp.up_bf, lp.up_inv,
                   lp.up_inv_d, lp.ext_prime, 0, 0, 0, level, K, l2};
      int max_nt = 0;
      for (int di = 0; di < lp.digits; ++di) max_nt = std::max(max_nt, level + K - lp.dig_na[di]);
      if (umma_up) {
        ba.bumma = lp.up_bu;
        ba.bu_off = lp.up_bu_off;
        rc = launch_bconv_umma(ch, ba, lp.max_na, max_nt,
                               dim3(bu_grid_x(n, lp.digits * batch), lp.digits, batch), st,
                               lp.up_sb, lp.bf_wide);
      } else {
        dim3 g((unsigned)std::max<long>(1, std::min<long>(n / (32 * kBcWarps), 64)), lp.digits,
               batch);
        rc = launch_bconv(ch, ba, lp.max_na, max_nt, g, st);
      }
      if (rc) return rc;
    } else if (ch.fp64_ok && lp.up_w_d) {
      int max_na = 0;
      for (int di = 0; di < lp.digits; ++di) max_na = std::max(max_na, lp.dig_na[di]);
      const size_t smem_d = ((size_t)max_w + level + K) * sizeof(double2);
      auto go = [&](auto kern) {
        if (smem_d > 48 * 1024)
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
        fhe_launch(kern, grid, dim3(kThreads), smem_d, st, ch, c, (long)level * n, ext,
                   (long)lp.ext_rows * n, lp.dig_info, lp.up_inv_d, lp.up_w_d, level, K, L);
      };
      if (max_na <= 4) go(modup_fp_kernel<4, FHE_MODUP_U>);
      else if (max_na <= 12) go(modup_fp_kernel<12, FHE_MODUP_U>);
      else go(modup_fp_kernel<16, FHE_MODUP_U>);
      FHE_LAUNCH_CHECK();
    } else {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(modup_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
      modup_kernel<<<grid, kThreads, smem, st>>>(ch, c, (long)level * n, ext,
                                                 (long)lp.ext_rows * n, lp.dig_info, lp.up_inv,
                                                 lp.up_w, level, K, L, chunk);
      FHE_LAUNCH_CHECK();
    }
    // mixed chain (Q < 2^50, P >= 2^50): per digit, the Q-target rows (the
    // first level - na of its block) transform on the FP64 path and the K
    // P-target rows on the integer path, instead of the whole ext block on
    // the integer path
    if (lp.ext_rows > 0 && mixed_q_fp64) {
      const long bs = (long)lp.ext_rows * n;
      for (int di = 0; di < lp.digits; ++di) {
        const int ro = lp.dig_row_off[di], nq = level - lp.dig_na[di];
        for (int part = 0; part < 2; ++part) {
          const int r0 = part ? ro + nq : ro, cnt = part ? K : nq;
          if (cnt <= 0) continue;
          NttArgs na{ext + (long)r0 * n, ext + (long)r0 * n, batch * cnt,
                     RowMap{lp.ext_prime + r0, cnt, 0}, bs, bs};
          na.fp64_rows = part == 0;
          rc = launch_ntt(ch, na, false, st);
          if (rc) return rc;
        }
      }
    } else if (lp.ext_rows > 0) {
      rc = launch_ntt(ch, ext, ext, batch * lp.ext_rows,
                      RowMap{lp.ext_prime, lp.ext_rows, 0}, false, st);
      if (rc) return rc;
    }
  }
  // 3. inner product with the key digits (K == 0 writes the result directly).
  // With the fused finish (FP64 path, <= 4 digits, K > 0) only the P limbs
  // are produced here; the Q limbs are folded into the ModDown finish below.
  const bool fin_inner = fin_inner_path(ctx, level);
  if (tens && !fin_inner) {
    fhe_set_error("keyswitch: tensor inputs need the fused finish path");
    return -1;
  }
  {
    const int m_end = level + K, m_begin = fin_inner ? level : 0;
    const long work = (long)(m_end - m_begin) << log_n;
    auto go_p = [&](auto kern, int kd) {
      const size_t sm = 64 + (size_t)FHE_FIN_STAGES * kd * kThreads * sizeof(u64);
      if (sm > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      kern<<<grid_for(work), kThreads, sm, st>>>(ch, ext, (long)lp.ext_rows * n, key, L + K,
                                                 lp.dig_info, lp.digits, level, K, L, accP, batch);
    };
    auto go = [&](auto kern) {
      kern<<<grid_for(work), kThreads, 4 * lp.digits * sizeof(int), st>>>(
          ch, d, d_stride, ext, (long)lp.ext_rows * n, key, L + K, lp.dig_info, lp.digits, level,
          K, L, accQ, accP, add0, add1, add_stride, out0, out1, out_stride, batch, m_begin, m_end,
          nullptr, nullptr);
    };
    if (fin_inner && ch.fp64_ok && lp.digits <= 4 && fin_staged_enabled()) {
      if (lp.digits <= 2) go_p(ks_plimb_staged_kernel<2>, 2);
      else if (lp.digits == 3) go_p(ks_plimb_staged_kernel<3>, 3);
      else go_p(ks_plimb_staged_kernel<4>, 4);
    } else if (ch.fp64_ok && lp.digits <= 2)
      go(ks_inner_fp_kernel<2>);
    else if (ch.fp64_ok && lp.digits == 3)
      go(ks_inner_fp_kernel<3>);
    else if (ch.fp64_ok && lp.digits == 4)
      go(ks_inner_fp_kernel<4>);
    else if (ch.fp64_ok)
      fhe_launch(ks_inner_fp_many_kernel, dim3(grid_for(work * batch)), dim3(kThreads),
                 4 * lp.digits * sizeof(int), st, ch, d, d_stride, ext, (long)lp.ext_rows * n, key,
                 L + K, lp.dig_info, lp.digits, level, K, L, accQ, accP, add0, add1, add_stride,
                 out0, out1, out_stride, batch);
    else if (mixed_q_fp64 && lp.digits <= 4 && K > 0 && !fin_inner) {
      // mixed chain: the Q limbs' inner product on the FP64 pipe, the P
      // limbs' on the integer pipe (same words)
      const long wq = (long)level << log_n, wp = (long)K << log_n;
      auto goq = [&](auto kern) {
        kern<<<grid_for(wq), kThreads, 4 * lp.digits * sizeof(int), st>>>(
            ch, d, d_stride, ext, (long)lp.ext_rows * n, key, L + K, lp.dig_info, lp.digits,
            level, K, L, accQ, accP, add0, add1, add_stride, out0, out1, out_stride, batch, 0,
            level, nullptr, nullptr);
      };
      if (lp.digits <= 2) goq(ks_inner_fp_kernel<2>);
      else if (lp.digits == 3) goq(ks_inner_fp_kernel<3>);
      else goq(ks_inner_fp_kernel<4>);
      FHE_LAUNCH_CHECK();
      ks_inner_kernel<<<grid_for(wp), kThreads, 4 * lp.digits * sizeof(int), st>>>(
          ch, d, d_stride, ext, (long)lp.ext_rows * n, key, L + K, lp.dig_info, lp.digits, level,
          K, L, accQ, accP, add0, add1, add_stride, out0, out1, out_stride, batch, chunk, level,
          level + K);
    } else
      ks_inner_kernel<<<grid_for(work), kThreads, 4 * lp.digits * sizeof(int), st>>>(
          ch, d, d_stride, ext, (long)lp.ext_rows * n, key, L + K, lp.dig_info, lp.digits, level,
          K, L, accQ, accP, add0, add1, add_stride, out0, out1, out_stride, batch, chunk, m_begin,
          m_end);
    FHE_LAUNCH_CHECK();
  }
  if (K == 0) return 0;
  // 4. ModDown
  rc = launch_ntt(ch, accP, accP, batch * 2 * K, RowMap{nullptr, K, L}, true, st);
  if (rc) return rc;
  {
    const size_t smem = (size_t)K * level * sizeof(u64);
    dim3 grid((unsigned)std::max<long>(1, std::min<long>(n / kThreads, 1024)), batch * 2);
    const bool umma_down = bconv_umma_enabled() && n >= kBuTile && lp.down_bu;
    if (lp.bf_ok && K >= 4 && bconv_imma_enabled() && (umma_down || lp.down_bf)) {
      // tensor-core conversion (tcgen05; mma.sync on narrow chains without it)
      const bool l2 = bconv_layout2();
      BconvArgs ba{accP, (long)K * n, conv, (long)level * n, nullptr, nullptr,
                   l2 ? lp.down_bf2 : lp.down_bf, lp.down_inv, lp.down_inv_d, nullptr, K, level,
                   L, level, K, l2};
      if (umma_down) {
        ba.bumma = lp.down_bu;
        rc = launch_bconv_umma(ch, ba, K, level, dim3(bu_grid_x(n, batch * 2), 1, batch * 2), st,
                               lp.down_sb, lp.bf_wide);
      } else {
        dim3 g((unsigned)std::max<long>(1, std::min<long>(n / (32 * kBcWarps), 64)), 1,
               batch * 2);
        rc = launch_bconv(ch, ba, K, level, g, st);
      }
      if (rc) return rc;
    } else if (ch.fp64_ok && lp.down_w_d) {
      const size_t smem_d = ((size_t)K * level + level) * sizeof(double2);
      auto go = [&](auto kern) {
        if (smem_d > 48 * 1024)
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_d);
        kern<<<grid, kThreads, smem_d, st>>>(ch, accP, conv, lp.down_inv_d, lp.down_w_d, level,
                                             K, L);
      };
      if (K <= 4) go(moddown_conv_fp_kernel<4, FHE_MODUP_U>);
      else if (K <= 12) go(moddown_conv_fp_kernel<12, FHE_MODUP_U>);
      else go(moddown_conv_fp_kernel<16, FHE_MODUP_U>);
      FHE_LAUNCH_CHECK();
    } else {
      moddown_conv_kernel<<<grid, kThreads, smem, st>>>(ch, accP, conv, lp.down_inv, lp.down_w,
                                                        level, K, L, chunk);
      FHE_LAUNCH_CHECK();
    }
  }
  // forward NTT of the conversion with the ModDown finish fused into its
  // last pass when the TMA chunk path runs it; otherwise a separate pass
  const NttFinish fin{accQ, lp.p_inv, add0, add1, add_stride, out0, out1, out_stride, level};
  bool fin_done = false;
  NttArgs na{conv, conv, batch * 2 * level, RowMap{nullptr, level, 0}, 0, 0};
  if (fuse_finish_enabled() && !fin_inner) {
    na.fin = &fin;
    na.fin_done = &fin_done;
  }
  rc = launch_ntt(ch, na, false, st);
  if (rc) return rc;
  if (fin_done) return 0;
  if (fin_inner && fin_staged_enabled()) {
    auto go = [&](auto kern, size_t smem_b) {
      if (smem_b > 48 * 1024)
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
      kern<<<grid_for((long)level << log_n), kThreads, smem_b, st>>>(
          ch, d, d_stride, ext, (long)lp.ext_rows * n, key, L + K, lp.dig_info, lp.digits, level,
          add0, add1, add_stride, out0, out1, out_stride, batch, conv, lp.p_inv, lp.p_inv_d);
    };
    if (tens) {
      if (lp.digits <= 2) go(ks_fin_staged_kernel<2, true>, fin_staged_smem<2, true>());
      else if (lp.digits == 3) go(ks_fin_staged_kernel<3, true>, fin_staged_smem<3, true>());
      else go(ks_fin_staged_kernel<4, true>, fin_staged_smem<4, true>());
    } else {
      if (lp.digits <= 2) go(ks_fin_staged_kernel<2, false>, fin_staged_smem<2, false>());
      else if (lp.digits == 3) go(ks_fin_staged_kernel<3, false>, fin_staged_smem<3, false>());
      else go(ks_fin_staged_kernel<4, false>, fin_staged_smem<4, false>());
    }
    FHE_LAUNCH_CHECK();
    return 0;
  }
  if (fin_inner) {
    // Q-limb inner product + ModDown finish in one pass
    auto go = [&](auto kern) {
      kern<<<grid_for((long)level << log_n), kThreads, 4 * lp.digits * sizeof(int), st>>>(
          ch, d, d_stride, ext, (long)lp.ext_rows * n, key, L + K, lp.dig_info, lp.digits, level,
          K, L, nullptr, nullptr, add0, add1, add_stride, out0, out1, out_stride, batch, 0, level,
          conv, lp.p_inv);
    };
    if (tens) {
      if (lp.digits <= 2) go(ks_inner_fp_kernel<2, true, true>);
      else if (lp.digits == 3) go(ks_inner_fp_kernel<3, true, true>);
      else go(ks_inner_fp_kernel<4, true, true>);
    } else {
      if (lp.digits <= 2) go(ks_inner_fp_kernel<2, true>);
      else if (lp.digits == 3) go(ks_inner_fp_kernel<3, true>);
      else go(ks_inner_fp_kernel<4, true>);
    }
    FHE_LAUNCH_CHECK();
    return 0;
  }
  moddown_finish_kernel<<<grid_for((long)batch * 2 * level * n), kThreads, 0, st>>>(
      ch, accQ, conv, lp.p_inv, add0, add1, add_stride, out0, out1, out_stride, level, batch);
  FHE_LAUNCH_CHECK();
  return 0;
}

// d2 = x1 * y1 of the tensor product only (the key switch's input); d0/d1 are
// formed inside the fused finish.  One read of x1, y1 and one write of d2.
__global__ void __launch_bounds__(kThreads)
    tensor_d2_kernel(const DevChain ch, u64* __restrict__ d2, const u64* __restrict__ x,
                     const u64* __restrict__ y, int level, int log_n, long batch, long in_stride) {
  const long n = 1L << log_n;
  const long per = (long)level << (log_n - 1);  // coefficient pairs per poly
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < batch * per;
       t += (long)gridDim.x * blockDim.x) {
    const long bi = t / per;
    const long w = t - bi * per;
    const ModConst m = ch.mc[(int)(w >> (log_n - 1))];
    const ulonglong2 a = reinterpret_cast<const ulonglong2*>(x + bi * in_stride + level * n)[w];
    const ulonglong2 b = reinterpret_cast<const ulonglong2*>(y + bi * in_stride + level * n)[w];
    reinterpret_cast<ulonglong2*>(d2 + bi * level * n)[w] =
        make_ulonglong2(mul_mod(a.x, b.x, m), mul_mod(a.y, b.y, m));
  }
}

// Default (FHE_HMULT_TENS=0 turns it off): form d0/d1/d2 inside the fused
// finish kernel.  It saves three polynomials of HBM traffic per op; the extra
// operands cost the HBM-bound finishing kernel a CTA per SM, so in a short
// burst it is within 0.5% (-0.4% at batch 8, +0.5% at batch 16), but under
// sustained load the board is power-capped and the lower DRAM traffic keeps
// the clocks higher: +2% at batch 16 (profiles/r1_ntt_notes.md).
static bool hmult_tens_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_HMULT_TENS");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

size_t hmult_relin_workspace(const FheContext& ctx, int level, int batch) {
  const size_t n = (size_t)1 << ctx.chain->log_n;
  return keyswitch_workspace(ctx, level, batch) + (size_t)batch * 3 * level * n * sizeof(u64);
}

// HMult+Relin in one call (ckks_multiply then ckks_relinearize, ckks.py):
// x, y are batch x (2, level, n) evaluation-domain ciphertexts in_stride words
// apart; out0/out1 receive the relinearized (c0, c1).  Default: only d2 is
// materialised and d0/d1 are formed in the finishing kernel; with
// FHE_HMULT_TENS=0 (or without the fused finish path) the full tensor goes
// to the workspace and the plain key switch runs on it.  Same words.
int run_hmult_relin(const FheContext& ctx, int level, const u64* x, const u64* y, long in_stride,
                    const u64* key, u64* out0, u64* out1, long out_stride, int batch, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
  if (level < 1 || level > ctx.L) {
    fhe_set_error("hmult_relin level out of range");
    return -1;
  }
  if (ws_bytes < hmult_relin_workspace(ctx, level, batch)) {
    fhe_set_error("hmult_relin workspace too small");
    return -1;
  }
  const DevChain& ch = ctx.chain->dev;
  const long n = 1L << ch.log_n;
  const size_t ks_bytes = keyswitch_workspace(ctx, level, batch);
  u64* t = (u64*)((char*)ws + ks_bytes);
  if (hmult_tens_enabled() && fin_inner_path(ctx, level)) {
    const long work = (long)batch * level << (ch.log_n - 1);
    tensor_d2_kernel<<<grid_for(work), kThreads, 0, st>>>(ch, t, x, y, level, ch.log_n, batch,
                                                          in_stride);
    FHE_LAUNCH_CHECK();
    return run_keyswitch(ctx, level, t, (long)level * n, key, x, y, in_stride, out0, out1,
                         out_stride, batch, ws, ks_bytes, st, true);
  }
  const long poly = (long)level * n;
  int rc = launch_tensor(ch, t, x, y, level, batch, in_stride, in_stride, 3 * poly, 0, st);
  if (rc) return rc;
  return run_keyswitch(ctx, level, t + 2 * poly, 3 * poly, key, t, t + poly, 3 * poly, out0,
                       out1, out_stride, batch, ws, ks_bytes, st, false);
}

static u64 ch_prime(const FheContext& ctx, int i) { return ctx.chain->primes[i]; }

// broadcast correction input in rescale (FHE_RESCALE_BCAST=0 keeps the
// materialised expand + NTT)
static bool bcast_rescale_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_RESCALE_BCAST");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// one-kernel rescale for N <= 2^12 (rescale_small_kernel): opt-in
// (FHE_RESCALE_SMALL=1) -- its radix-2 shared-memory NTT is slower than the
// broadcast-input tile NTT + finish it would replace (PDQ query 1: 7.7 vs
// 5.8 ms graph-replayed)
static bool small_rescale_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_RESCALE_SMALL");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

size_t rescale_workspace(const FheContext& ctx, int polys, int level) {
  const size_t n = (size_t)1 << ctx.chain->log_n;
  return (size_t)polys * level * n * sizeof(u64);
}

int run_rescale(FheContext& ctx, u64* out, const u64* in, int polys, int level, u64 t_plain,
                void* ws, size_t ws_bytes, cudaStream_t st) {
  if (level < 2 || level > ctx.L) {
    fhe_set_error("rescale needs 2 <= level <= L");
    return -1;
  }
  if (ws_bytes < rescale_workspace(ctx, polys, level)) {
    fhe_set_error("rescale workspace too small");
    return -1;
  }
  const LevelPlan& lp = ctx.levels[level];
  const DevChain& ch = ctx.chain->dev;
  const long n = 1L << ch.log_n;
  u64* last = (u64*)ws;
  u64* corr = last + (long)polys * n;
  WPair tinv{0, 0};
  const u64* t_mod = nullptr;
  if (t_plain) {
    const PlainPlan* pp = get_plain_plan(&ctx, t_plain);
    if (!pp) {
      fhe_set_error("plain-modulus plan allocation failed");
      return -2;
    }
    tinv = pp->tinv_last[level];
    t_mod = pp->t_mod[level];
  }
  // inverse NTT of each poly's last limb, read in place (row stride level*n)
  int rc = launch_ntt(ch, NttArgs{last, in + (long)(level - 1) * n, polys,
                                  RowMap{nullptr, 1, level - 1}, (long)level * n, 0},
                      true, st);
  if (rc) return rc;
  // N <= 2^12 (CKKS): expand, NTT and finish in one kernel per (limb, poly)
  if (t_plain == 0 && ch.log_n <= 12 && small_rescale_enabled())
    return launch_rescale_small(ch, out, in, last, polys, level, lp.rs_inv, lp.rs_qlast, st);
  // CKKS: the correction rows are the centred last limb mod every q_j, which
  // the forward NTT reads straight from `last` (broadcast, centred input):
  // the expanded rows are never written.  Otherwise (BGV, or a shape the
  // broadcast path does not take) the expand kernel materialises them.
  bool bcast = false;
  if (t_plain == 0 && bcast_rescale_enabled()) {
    NttArgs na{corr, corr, polys * (level - 1), RowMap{nullptr, level - 1, 0}, 0, 0};
    na.bcast_src = last;
    na.bcast_stride = n;
    na.center_q = ch_prime(ctx, level - 1);
    na.bcast_done = &bcast;
    bool fused_fin = false;
    if (lp.rs_inv_d && rescale_fin_fused_enabled()) {
      // the cluster transform applies the finish in its epilogue
      na.rs_in = in;
      na.rs_out = out;
      na.rs_inv_d = lp.rs_inv_d;
      na.rs_level = level;
      na.rs_done = &fused_fin;
    }
    rc = launch_ntt(ch, na, false, st);
    if (rc) return rc;
    if (bcast && fused_fin) return 0;
  }
  if (!bcast) {
    rc = launch_modswitch_expand(ch, corr, last, polys, level - 1, level - 1, t_plain, tinv,
                                 t_mod, lp.rs_qlast, st);
    if (rc) return rc;
    rc = launch_ntt(ch, corr, corr, polys * (level - 1), RowMap{nullptr, level - 1, 0}, false, st);
    if (rc) return rc;
  }
  return launch_modswitch_finish(ch, out, in, corr, polys, level, lp.rs_inv, st);
}

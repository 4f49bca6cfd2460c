// BEHZ full-RNS BFV multiplication kernels (schemes/behz.py:58-270).
//
// The reference computes the BFV tensor with *approximate* fast base
// conversions and the m_tilde / m_sk corrections; the GPU kernels evaluate
// exactly the same formulas per coefficient (every intermediate is an exact
// residue, so the bits match), one thread per coefficient with all limbs in
// registers:
//
//   behz_lift  : Q -> Q | Bsk  (extend_to_bsk, behz.py:162-189)
//   behz_floor : (Q | Bsk) tensor coefficients -> Q  (x t, fast_floor_q
//                behz.py:192-205, then fast_conv_sk_to_q behz.py:208-233)
//
// Constant layout (u64 words, built by schemes/behz.py, all device memory):
//   lift:  mt_ys[L] pairs      (m_tilde * (Q/q_j)^-1 mod q_j, shoup)
//          w_bsk[S][L]         ((Q/q_j) mod m_d)
//          w_mt[L]             ((Q/q_j) mod 2^16)
//          neg_q_inv_mt        ((-Q)^-1 mod 2^16)
//          q_mod_bsk[S]        (Q mod m_d)
//          mt_inv_bsk[S] pairs (m_tilde^-1 mod m_d, shoup)
//   floor: t_big[L+S] pairs    (t mod m, shoup, over Q then Bsk)
//          inv_punc_q[L] pairs ((Q/q_j)^-1 mod q_j, shoup)
//          w_bsk[S][L]         ((Q/q_j) mod m_d)
//          q_inv_bsk[S] pairs  (Q^-1 mod m_d, shoup)
//          inv_punc_b[B] pairs ((Bp/b_i)^-1 mod b_i, shoup)
//          w_bq[L][B]          ((Bp/b_i) mod q_j)
//          w_bmsk[B]           ((Bp/b_i) mod m_sk)
//          inv_b_msk pair      (Bp^-1 mod m_sk, shoup)
//          b_mod_q[L]          (Bp mod q_j)
// with S = B + 1 (Bsk = B primes then m_sk) and the big chain ordered Q, B, m_sk.
#include "fhe_kernels.cuh"

namespace {

constexpr int kThreads = 128;
constexpr int kMaxL = 24;  // Q limbs handled per coefficient
constexpr int kMaxS = 24;  // Bsk limbs

__device__ __forceinline__ WPair ldp(const u64* p) { return WPair{p[0], p[1]}; }

__global__ void __launch_bounds__(kThreads)
    behz_lift_kernel(const DevChain big, u64* __restrict__ out, const u64* __restrict__ in, int L,
                     int S, const u64* __restrict__ cst, int polys) {
  const int log_n = big.log_n;
  const long n = 1L << log_n;
  const u64* mt_ys = cst;
  const u64* w_bsk = mt_ys + 2 * L;
  const u64* w_mt = w_bsk + (long)S * L;
  const u64 neg_q_inv_mt = w_mt[L];
  const u64* q_mod_bsk = w_mt + L + 1;
  const u64* mt_inv = q_mod_bsk + S;
  const long total = (long)polys << log_n;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long p = t >> log_n, i = t & (n - 1);
    const u64* src = in + p * L * n;
    u64* dst = out + p * (L + S) * n;
    u64 ys[kMaxL];
    u64 mt = 0;
#pragma unroll
    for (int j = 0; j < kMaxL; ++j) {
      if (j < L) {
        const u64 x = src[j * n + i];
        dst[j * n + i] = x;  // the Q part of the lifted polynomial is the input itself
        const WPair c = ldp(mt_ys + 2 * j);
        ys[j] = shoup_mul(x, c.w, c.sh, big.mc[j].q);
        mt += ys[j] * w_mt[j];  // wraps mod 2^64; only the low 16 bits are used
      }
    }
    const u64 r = (mt * neg_q_inv_mt) & 0xFFFF;
    const long rs = r >= 0x8000 ? (long)r - 0x10000 : (long)r;
    for (int d = 0; d < S; ++d) {
      const ModConst mc = big.mc[L + d];
      u64 hi = 0, lo = 0;
#pragma unroll
      for (int j = 0; j < kMaxL; ++j)
        if (j < L) mac_wide(hi, lo, ys[j], w_bsk[(long)d * L + j]);
      const u64 tilde = reduce_fold(hi, lo, mc);
      const u64 rm = rs >= 0 ? (u64)rs : mc.q - (u64)(-rs);  // r_signed mod m (|r| < m)
      const u64 s = add_mod(tilde, mul_mod(rm, q_mod_bsk[d], mc), mc.q);
      const WPair iv = ldp(mt_inv + 2 * d);
      dst[(L + d) * n + i] = shoup_mul(s, iv.w, iv.sh, mc.q);
    }
  }
}

__global__ void __launch_bounds__(kThreads)
    behz_floor_kernel(const DevChain big, u64* __restrict__ out, const u64* __restrict__ in,
                      int L, int S, const u64* __restrict__ cst, int polys) {
  const int B = S - 1;
  const int log_n = big.log_n;
  const long n = 1L << log_n;
  const u64* t_big = cst;
  const u64* inv_punc_q = t_big + 2 * (L + S);
  const u64* w_bsk = inv_punc_q + 2 * L;
  const u64* q_inv_bsk = w_bsk + (long)S * L;
  const u64* inv_punc_b = q_inv_bsk + 2 * S;
  const u64* w_bq = inv_punc_b + 2 * B;
  const u64* w_bmsk = w_bq + (long)L * B;
  const u64* inv_b_msk = w_bmsk + B;
  const u64* b_mod_q = inv_b_msk + 2;
  const long total = (long)polys << log_n;
  const ModConst msk = big.mc[L + B];
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long p = t >> log_n, i = t & (n - 1);
    const u64* src = in + p * (L + S) * n;
    u64* dst = out + p * L * n;
    // x t over Q, then y_j = [x_j t (Q/q_j)^-1]_{q_j}
    u64 ys[kMaxL];
#pragma unroll
    for (int j = 0; j < kMaxL; ++j) {
      if (j < L) {
        const u64 q = big.mc[j].q;
        const WPair tw = ldp(t_big + 2 * j), iw = ldp(inv_punc_q + 2 * j);
        ys[j] = shoup_mul(shoup_mul(src[j * n + i], tw.w, tw.sh, q), iw.w, iw.sh, q);
      }
    }
    // fast floor in Bsk: ((x t)_m - FastBConv_q(x t)_m) Q^-1 mod m, then
    // z_i = [floored_i (Bp/b_i)^-1]_{b_i} for the Shenoy-Kumaresan step
    u64 zb[kMaxS];
    u64 fl_msk = 0;
#pragma unroll
    for (int d = 0; d < kMaxS; ++d) {
      if (d < S) {
        const ModConst mc = big.mc[L + d];
        const WPair tw = ldp(t_big + 2 * (L + d));
        const u64 xt = shoup_mul(src[(L + d) * n + i], tw.w, tw.sh, mc.q);
        u64 hi = 0, lo = 0;
#pragma unroll
        for (int j = 0; j < kMaxL; ++j)
          if (j < L) mac_wide(hi, lo, ys[j], w_bsk[(long)d * L + j]);
        const u64 conv = reduce_fold(hi, lo, mc);
        const WPair qi = ldp(q_inv_bsk + 2 * d);
        const u64 fl = shoup_mul(sub_mod(xt, conv, mc.q), qi.w, qi.sh, mc.q);
        if (d < B) {
          const WPair ib = ldp(inv_punc_b + 2 * d);
          zb[d] = shoup_mul(fl, ib.w, ib.sh, mc.q);
        } else {
          fl_msk = fl;
        }
      }
    }
    // alpha = (FastBConv_B(z)_{m_sk} - floored_{m_sk}) Bp^-1 mod m_sk, centred
    u64 hi = 0, lo = 0;
#pragma unroll
    for (int d = 0; d < kMaxS; ++d)
      if (d < B) mac_wide(hi, lo, zb[d], w_bmsk[d]);
    const u64 cm = reduce_fold(hi, lo, msk);
    const WPair ibm = ldp(inv_b_msk);
    const u64 alpha = shoup_mul(sub_mod(cm, fl_msk, msk.q), ibm.w, ibm.sh, msk.q);
    const bool neg = alpha > (msk.q >> 1);
    const u64 amag = neg ? msk.q - alpha : alpha;  // |alpha_signed|
    for (int j = 0; j < L; ++j) {
      const ModConst mc = big.mc[j];
      u64 h2 = 0, l2 = 0;
#pragma unroll
      for (int d = 0; d < kMaxS; ++d)
        if (d < B) mac_wide(h2, l2, zb[d], w_bq[(long)j * B + d]);
      const u64 conv = reduce_fold(h2, l2, mc);
      u64 am = reduce_word(amag, mc);
      if (neg) am = neg_mod(am, mc.q);
      dst[j * n + i] = sub_mod(conv, mul_mod(am, b_mod_q[j], mc), mc.q);
    }
  }
}

}  // namespace

extern "C" int fhe_behz_lift(const FheChain* big, uint64_t* out, const uint64_t* in, int polys,
                             int L, int S, const uint64_t* consts, void* stream);
extern "C" int fhe_behz_floor(const FheChain* big, uint64_t* out, const uint64_t* in, int polys,
                              int L, int S, const uint64_t* consts, void* stream);

#include "fhe_context.cuh"

extern "C" int fhe_behz_lift(const FheChain* big, uint64_t* out, const uint64_t* in, int polys,
                             int L, int S, const uint64_t* consts, void* stream) {
  if (!big || !out || !in || !consts || L < 1 || S < 2 || L > kMaxL || S > kMaxS ||
      L + S > big->dev.count || polys < 1) {
    fhe_set_error("fhe_behz_lift: bad arguments (L <= 24, 2 <= S <= 24, L + S <= chain)");
    return -1;
  }
  const long work = (long)polys << big->dev.log_n;
  behz_lift_kernel<<<std::max<long>(1, std::min<long>((work + kThreads - 1) / kThreads, 148 * 16)),
                     kThreads, 0, (cudaStream_t)stream>>>(big->dev, out, in, L, S, consts, polys);
  FHE_LAUNCH_CHECK();
  return 0;
}

extern "C" int fhe_behz_floor(const FheChain* big, uint64_t* out, const uint64_t* in, int polys,
                              int L, int S, const uint64_t* consts, void* stream) {
  if (!big || !out || !in || !consts || L < 1 || S < 2 || L > kMaxL || S > kMaxS ||
      L + S > big->dev.count || polys < 1) {
    fhe_set_error("fhe_behz_floor: bad arguments (L <= 24, 2 <= S <= 24, L + S <= chain)");
    return -1;
  }
  const long work = (long)polys << big->dev.log_n;
  behz_floor_kernel<<<std::max<long>(1, std::min<long>((work + kThreads - 1) / kThreads, 148 * 16)),
                      kThreads, 0, (cudaStream_t)stream>>>(big->dev, out, in, L, S, consts, polys);
  FHE_LAUNCH_CHECK();
  return 0;
}

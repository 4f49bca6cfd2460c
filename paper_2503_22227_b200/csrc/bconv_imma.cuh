// Fast base conversion on the tensor cores (integer MMA), for ModUp and
// ModDown of the hybrid key switch.  Included by keyswitch.cu inside its
// anonymous namespace.
//
//   y_s   = [x_s * inv_s]_{q_s}                       (s < ns, prologue)
//   out_t = sum_s y_s * w_{s,t}  mod p_t              (t < nt)
//
// The contraction over s is an exact integer matrix product.  With every
// prime < 2^56, y_s has 7 bytes: y_s = sum_a y_{s,a} 2^(8a), and with
// W'_{(s,a),(t,b)} = byte b of [w_{s,t} 2^(8a)]_{p_t} (host precompute),
//   out_t = sum_b 2^(8b) P_{t,b}  mod p_t,   P_{t,b} = sum_{s,a} y_{s,a} W'_{(s,a),(t,b)}
// where every P_{t,b} <= 16 * 7 * 255^2 < 2^23 is an exact u8 x u8 -> s32
// tensor-core dot product (mma.sync m16n8k32, K = 7 ns padded to 32 KS).  The
// epilogue combines the 7 partials in 128 bits (< 2^71) and reduces once
// (reduce_fold), so the result is the same canonical word as the FP64-pipe
// and integer conversion kernels (any exact evaluation of the sum agrees).
//
// Why: the FP64-pipe conversions spent ~7 FP64 instructions per exact
// multiply-accumulate and were ~30% of the HMult+Relin step at 72% of the
// FP64 pipe (profiles/r1_ncu_step_b16.txt); the byte-split contraction is
// ~145 G int8 ops per batch-16 ModUp, 0.16 ms at the measured 909 TOPS of
// mma.sync IMMA (profiles/r2_microbench_imma.txt), off the FP64 pipe.
//
// Work split: one warp = 32 coefficients (lane = coefficient in the prologue
// and epilogue, two m16 tiles in the MMA); A (the row bytes) goes through a
// per-warp shared tile, B (the packed fragments of W') is staged once per CTA.
#pragma once

#ifndef FHE_BCONV_WARPS
#define FHE_BCONV_WARPS 8
#endif
constexpr int kBcWarps = FHE_BCONV_WARPS;
constexpr int kBcThreads = 32 * kBcWarps;

// u32 words per row of the per-warp A tile: 8 KS data words, padded to a
// stride of 4 or 28 mod 32 so a fragment load (8 rows x 4 consecutive words)
// hits 32 distinct banks
__host__ __device__ constexpr int bc_astride(int ks) {
  return ks == 1 ? 12 : (ks == 2 ? 20 : (ks == 3 ? 28 : 36));
}
constexpr int kBcCStride = 12;  // u32 words per row of the per-warp C tile

__device__ __forceinline__ void imma_u8(int (&c)[4], const unsigned (&a)[4], uint2 b) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
}

// One conversion job per (blockIdx.y, blockIdx.z):
//   ModUp   (digits): y = digit, z = batch item; sources = the digit's primes
//           s0 .. s0+na-1 of c, targets = ext rows row_off .. row_off+nt-1
//   ModDown:          y = 0,     z = batch * 2 polys; sources = the K P limbs
//           of accP, targets = the level Q limbs of conv
struct BconvArgs {
  const u64* src;
  long src_bstride;         // words between z items
  u64* dst;
  long dst_bstride;
  const int* dig_info;      // ModUp: [4 * digits] (s0, na, row_off, w_off); null: ModDown
  const int* bf_off;        // ModUp: per digit offset (uint2 units) into bfrag; null: 0
  const uint2* bfrag;       // packed W' fragments [nt][KS][32]
  const WPair* inv;         // per source chain position (ModUp: up_inv[level]; ModDown: [K])
  const double2* inv_d;     // the same as FP64 pairs (w, w / q) (FP64 prologue)
  const int32_t* tgt_prime; // ModUp: ext_prime (chain index per ext row); null: identity
  int ns, nt;               // ModDown: K, level (ModUp: from dig_info, nt = level + K - na)
  int src_prime0;           // ModDown: L (first P prime); ModUp: 0 (+ s0)
  int level, K;
  bool layout2 = false;     // bfrag packed for bconv_imma2_kernel (pack_bfrag2)
  const uint4* bumma = nullptr;  // W' in the tcgen05 operand layout (bconv_umma.cuh)
  const int* bu_off = nullptr;   // ModUp: per digit offset (uint4 units) into bumma
};

// Per-target reduction constants of the epilogue: V < 2^71 is reduced by one
// Barrett step with mu = floor(2^71 / p) and x = V >> sh (sh = bitlen(p) - 1
// >= 39, so x * mu < 2^64): qe = (x mu) >> (71 - sh) is short of V / p by at
// most 2 (V / p - qe < V / 2^71 + 2^sh / p + 1 < 3), so V - qe p < 3p and two
// conditional subtractions give the canonical residue.  Only the low 64 bits
// of qe p are needed (the remainder is < 2^58).
struct __align__(16) BcTarget {  // 16 bytes: one LDS.128; keeps the smem regions after it aligned
  u64 p;
  u32 mu;  // floor(2^71 / p) < 2^32 (p >= 2^39)
  u32 sh;
};

__device__ __forceinline__ u64 bc_reduce71(u64 hi, u64 lo, const BcTarget& tg) {
  const u64 x = (hi << (64 - tg.sh)) | (lo >> tg.sh);  // V >> sh (hi < 2^7, sh >= 39)
  const u64 qe = (x * (u64)tg.mu) >> (71 - tg.sh);
  u64 r = lo - qe * tg.p;
  r = csub(r, tg.p);
  return csub(r, tg.p);
}

// V = sum_b P_b 2^(8b) from the 7 byte partials and its canonical residue,
// in 32-bit pieces (the value is that of bc_reduce71 on the 128-bit sum):
//   v = P0 + P1 2^8 + P2 2^16 + P3 2^24 < 2^48,  H = P4 + P5 2^8 + P6 2^16 < 2^40,
//   V = v + H 2^32 = (hi : lo) with hi < 2^7;
//   x = V >> sh < 2^32 (sh >= 39), mu < 2^32, qe = (x mu) >> (71 - sh) < 2^32.
// Each partial product is one IMAD.WIDE.U32 instead of 64-bit shift/add pairs.
__device__ __forceinline__ u64 bc_combine71(unsigned a0, unsigned a1, unsigned a2, unsigned a3,
                                            unsigned a4, unsigned a5, unsigned a6,
                                            const BcTarget& tg) {
  u64 v = (u64)a1 * 256u + a0;
  v = (u64)a2 * 65536u + v;
  v = (u64)a3 * 16777216u + v;
  u64 h = (u64)a5 * 256u + a4;
  h = (u64)a6 * 65536u + h;
  unsigned lo_hi, hi;
  asm("add.cc.u32 %0, %2, %3;\n\taddc.u32 %1, %4, 0;"
      : "=r"(lo_hi), "=r"(hi)
      : "r"((unsigned)(v >> 32)), "r"((unsigned)h), "r"((unsigned)(h >> 32)));
  const unsigned x = __funnelshift_r(lo_hi, hi, tg.sh - 32);
  const u64 prod = (u64)x * tg.mu;
  const unsigned qe = __funnelshift_rc((unsigned)prod, (unsigned)(prod >> 32), 71 - tg.sh);
  const u64 lo = ((u64)lo_hi << 32) | (unsigned)v;
  u64 r = lo - (u64)qe * tg.p;
  r = csub(r, tg.p);
  return csub(r, tg.p);
}

// FPPRO: the prologue product y = [x inv]_q on the FP64 pipe (fp_mulmod; the
// pipe is otherwise idle here), else the integer Shoup product.
#ifndef FHE_BCONV_COMBINE32
#define FHE_BCONV_COMBINE32 1
#endif
#ifndef FHE_BCONV_MINB
#define FHE_BCONV_MINB 2
#endif
template <int KS, int TB, bool FPPRO>
__global__ void __launch_bounds__(kBcThreads, FHE_BCONV_MINB)
    bconv_imma_kernel(const DevChain ch, const BconvArgs a) {
  constexpr int SMAX = (32 * KS) / 7;  // sources that fit the K dimension
  constexpr int AST = bc_astride(KS);
  constexpr int WARP_WORDS = 32 * AST + TB * 32 * kBcCStride;
  extern __shared__ __align__(16) unsigned char bc_smem[];
  int ns = a.ns, nt = a.nt, s0 = 0, row_off = 0, bfo = 0;
  if (a.dig_info) {
    const int di = blockIdx.y;
    s0 = a.dig_info[4 * di];
    ns = a.dig_info[4 * di + 1];
    row_off = a.dig_info[4 * di + 2];
    nt = a.level + a.K - ns;
    bfo = a.bf_off[di];
  }
  uint2* sb = reinterpret_cast<uint2*>(bc_smem);                    // [nt][KS][32]
  BcTarget* tgs = reinterpret_cast<BcTarget*>(sb + nt * KS * 32);    // [nt]
  double2* sinv = reinterpret_cast<double2*>(tgs + nt);              // [SMAX] FP: (w, w/q)
  double2* sqd = sinv + SMAX;                                        // [SMAX] FP: (q, 1/q)
  WPair* sinvi = reinterpret_cast<WPair*>(sqd + SMAX);              // [SMAX] int: Shoup pair
  u64* sqi = reinterpret_cast<u64*>(sinvi + SMAX);                   // [SMAX] int: q
  // per-warp tiles start 16-byte aligned (uint4 row stores)
  unsigned* atile = reinterpret_cast<unsigned*>(sqi + ((SMAX + 1) & ~1)) +
                    (threadIdx.x >> 5) * WARP_WORDS;
  unsigned* ctile = atile + 32 * AST;
  for (int i = threadIdx.x; i < nt * KS * 32; i += blockDim.x) sb[i] = a.bfrag[bfo + i];
  for (int t = threadIdx.x; t < nt; t += blockDim.x) {
    const ModConst m = ch.mc[a.tgt_prime ? a.tgt_prime[row_off + t] : t];
    const u32 sh = m.s;  // bitlen(p) - 1
    // mu = floor(2^71 / p) = floor(2^(64+sh) / p) >> (sh - 7) = m.mu >> (sh - 7)
    tgs[t] = BcTarget{m.q, (u32)(m.mu >> (sh - 7)), sh};
  }
  for (int s = threadIdx.x; s < SMAX; s += blockDim.x) {
    if (s < ns) {
      const int cp = a.src_prime0 + s0 + s;
      if (FPPRO) {
        sinv[s] = a.inv_d[s0 + s];
        sqd[s] = ch.qd[cp];
      } else {
        sinvi[s] = a.inv[s0 + s];
        sqi[s] = ch.mc[cp].q;
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gr = lane >> 2, gq = lane & 3;
  const long n = 1L << ch.log_n;
  const u64* src = a.src + blockIdx.z * a.src_bstride + (long)s0 * n;
  u64* dst = a.dst + blockIdx.z * a.dst_bstride + (long)row_off * n;
  const int warps_total = gridDim.x * kBcWarps;
  for (long c0 = ((long)blockIdx.x * kBcWarps + (threadIdx.x >> 5)) * 32; c0 < n;
       c0 += (long)warps_total * 32) {
    // prologue: lane = coefficient; all source words loaded first, then the
    // K bytes (7 per source) of its row go to the A tile
    const long c = c0 + lane;
    u64 xs[SMAX];
#pragma unroll
    for (int s = 0; s < SMAX; ++s) xs[s] = s < ns ? src[(long)s * n + c] : 0;
    unsigned w[8 * KS];
#pragma unroll
    for (int i = 0; i < 8 * KS; ++i) w[i] = 0;
#pragma unroll
    for (int s = 0; s < SMAX; ++s) {
      if (s < ns) {
        u64 y;
        if (FPPRO) {
          const double2 qd = sqd[s];
          y = fp_to_u52(fp_pos(fp_mulmod(fp_from_u52(xs[s]), sinv[s], qd.x), qd.x));
        } else {
          const WPair iv = sinvi[s];
          y = shoup_mul(xs[s], iv.w, iv.sh, sqi[s]);
        }
        const int bit = 56 * s, wi = bit >> 5, sh = bit & 31;
        const u64 lo64 = y << sh;
        w[wi] |= (unsigned)lo64;
        w[wi + 1] |= (unsigned)(lo64 >> 32);
        if (sh > 8) w[wi + 2] |= (unsigned)(y >> (64 - sh));
      }
    }
#pragma unroll
    for (int i = 0; i < 8 * KS; i += 4)
      *reinterpret_cast<uint4*>(&atile[lane * AST + i]) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
    __syncwarp();
    // A fragments of the two m16 tiles (rows 0..15, 16..31)
    unsigned af[2][KS][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const unsigned* r0 = &atile[(16 * m + gr) * AST + 8 * ks + gq];
        const unsigned* r1 = r0 + 8 * AST;
        af[m][ks][0] = r0[0];
        af[m][ks][1] = r1[0];
        af[m][ks][2] = r0[4];
        af[m][ks][3] = r1[4];
      }
    // TB targets per pass: independent MMA chains, one C round trip
    for (int t0 = 0; t0 < nt; t0 += TB) {
      int acc[TB][2][4];
#pragma unroll
      for (int u = 0; u < TB; ++u)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[u][m][i] = 0;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks)
#pragma unroll
        for (int u = 0; u < TB; ++u) {
          const int t = min(t0 + u, nt - 1);
          const uint2 b = sb[(t * KS + ks) * 32 + lane];
          imma_u8(acc[u][0], af[0][ks], b);
          imma_u8(acc[u][1], af[1][ks], b);
        }
#pragma unroll
      for (int u = 0; u < TB; ++u)
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          unsigned* ct = ctile + u * 32 * kBcCStride;
          *reinterpret_cast<uint2*>(&ct[(16 * m + gr) * kBcCStride + 2 * gq]) =
              make_uint2((unsigned)acc[u][m][0], (unsigned)acc[u][m][1]);
          *reinterpret_cast<uint2*>(&ct[(16 * m + 8 + gr) * kBcCStride + 2 * gq]) =
              make_uint2((unsigned)acc[u][m][2], (unsigned)acc[u][m][3]);
        }
      __syncwarp();
#pragma unroll
      for (int u = 0; u < TB; ++u) {
        const int t = t0 + u;
        if (t < nt) {
          const unsigned* ct = ctile + u * 32 * kBcCStride + lane * kBcCStride;
          const uint4 p03 = *reinterpret_cast<const uint4*>(ct);
          const uint4 p47 = *reinterpret_cast<const uint4*>(ct + 4);
          // V = sum_b P_b 2^(8b) < 2^71
          u64 lo = (u64)p03.x + ((u64)p03.y << 8) + ((u64)p03.z << 16) + ((u64)p03.w << 24) +
                   ((u64)p47.x << 32) + ((u64)p47.y << 40);
          u64 hi = 0;
          add_wide(hi, lo, (u64)p47.z >> 16, (u64)p47.z << 48);
          dst[(long)t * n + c] = bc_reduce71(hi, lo, tgs[t]);
        }
      }
      __syncwarp();
    }
  }
}

// Register-resident epilogue (default): the n8 tiles are (8 targets, one byte
// position b), so after the 7 byte tiles of a target group every lane holds
// all 7 partials of its 2 targets x 4 rows in registers -- no shared-memory
// transpose and no warp syncs per target (C fragment: lane (gr, gq) holds
// columns 2 gq, 2 gq + 1 of rows gr, gr + 8).  B is packed per (group,
// byte, k-step) on the host (pack_bfrag2, context.cu).
template <int KS, bool FPPRO>
__global__ void __launch_bounds__(kBcThreads, FHE_BCONV_MINB)
    bconv_imma2_kernel(const DevChain ch, const BconvArgs a) {
  constexpr int SMAX = (32 * KS) / 7;
  constexpr int AST = bc_astride(KS);
  extern __shared__ __align__(16) unsigned char bc_smem[];
  int ns = a.ns, nt = a.nt, s0 = 0, row_off = 0, bfo = 0;
  if (a.dig_info) {
    const int di = blockIdx.y;
    s0 = a.dig_info[4 * di];
    ns = a.dig_info[4 * di + 1];
    row_off = a.dig_info[4 * di + 2];
    nt = a.level + a.K - ns;
    bfo = a.bf_off[di];
  }
  const int ng = (nt + 7) >> 3;  // target groups of 8
  uint2* sb = reinterpret_cast<uint2*>(bc_smem);                      // [ng][7][KS][32]
  BcTarget* tgs = reinterpret_cast<BcTarget*>(sb + ng * 7 * KS * 32);  // [8 ng]
  double2* sinv = reinterpret_cast<double2*>(tgs + 8 * ng);
  double2* sqd = sinv + SMAX;
  WPair* sinvi = reinterpret_cast<WPair*>(sqd + SMAX);
  u64* sqi = reinterpret_cast<u64*>(sinvi + SMAX);
  unsigned* atile = reinterpret_cast<unsigned*>(sqi + ((SMAX + 1) & ~1)) +
                    (threadIdx.x >> 5) * (32 * AST);
  for (int i = threadIdx.x; i < ng * 7 * KS * 32; i += blockDim.x) sb[i] = a.bfrag[bfo + i];
  for (int t = threadIdx.x; t < 8 * ng; t += blockDim.x) {
    if (t < nt) {
      const ModConst m = ch.mc[a.tgt_prime ? a.tgt_prime[row_off + t] : t];
      tgs[t] = BcTarget{m.q, (u32)(m.mu >> (m.s - 7)), (u32)m.s};
    } else {
      tgs[t] = BcTarget{1, 0, 39};  // padding target (never stored)
    }
  }
  for (int s = threadIdx.x; s < SMAX; s += blockDim.x) {
    if (s < ns) {
      const int cp = a.src_prime0 + s0 + s;
      if (FPPRO) {
        sinv[s] = a.inv_d[s0 + s];
        sqd[s] = ch.qd[cp];
      } else {
        sinvi[s] = a.inv[s0 + s];
        sqi[s] = ch.mc[cp].q;
      }
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int gr = lane >> 2, gq = lane & 3;
  const long n = 1L << ch.log_n;
  const u64* src = a.src + blockIdx.z * a.src_bstride + (long)s0 * n;
  u64* dst = a.dst + blockIdx.z * a.dst_bstride + (long)row_off * n;
  const int warps_total = gridDim.x * kBcWarps;
  for (long c0 = ((long)blockIdx.x * kBcWarps + (threadIdx.x >> 5)) * 32; c0 < n;
       c0 += (long)warps_total * 32) {
    const long c = c0 + lane;
    u64 xs[SMAX];
#pragma unroll
    for (int s = 0; s < SMAX; ++s) xs[s] = s < ns ? src[(long)s * n + c] : 0;
    unsigned w[8 * KS];
#pragma unroll
    for (int i = 0; i < 8 * KS; ++i) w[i] = 0;
#pragma unroll
    for (int s = 0; s < SMAX; ++s) {
      if (s < ns) {
        u64 y;
        if (FPPRO) {
          const double2 qd = sqd[s];
          y = fp_to_u52(fp_pos(fp_mulmod(fp_from_u52(xs[s]), sinv[s], qd.x), qd.x));
        } else {
          const WPair iv = sinvi[s];
          y = shoup_mul(xs[s], iv.w, iv.sh, sqi[s]);
        }
        const int bit = 56 * s, wi = bit >> 5, sh = bit & 31;
        const u64 lo64 = y << sh;
        w[wi] |= (unsigned)lo64;
        w[wi + 1] |= (unsigned)(lo64 >> 32);
        if (sh > 8) w[wi + 2] |= (unsigned)(y >> (64 - sh));
      }
    }
    __syncwarp();  // the previous iteration's fragment loads are done
#pragma unroll
    for (int i = 0; i < 8 * KS; i += 4)
      *reinterpret_cast<uint4*>(&atile[lane * AST + i]) = make_uint4(w[i], w[i + 1], w[i + 2], w[i + 3]);
    __syncwarp();
    unsigned af[2][KS][4];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const unsigned* r0 = &atile[(16 * m + gr) * AST + 8 * ks + gq];
        const unsigned* r1 = r0 + 8 * AST;
        af[m][ks][0] = r0[0];
        af[m][ks][1] = r1[0];
        af[m][ks][2] = r0[4];
        af[m][ks][3] = r1[4];
      }
    for (int g = 0; g < ng; ++g) {
      int acc[7][2][4];
#pragma unroll
      for (int b = 0; b < 7; ++b)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[b][m][i] = 0;
#pragma unroll
      for (int b = 0; b < 7; ++b)
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          const uint2 bf = sb[((g * 7 + b) * KS + ks) * 32 + lane];
          imma_u8(acc[b][0], af[0][ks], bf);
          imma_u8(acc[b][1], af[1][ks], bf);
        }
      // lane: targets 8 g + 2 gq + e, rows 16 m + gr + 8 h  (c index 2 h + e)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = 8 * g + 2 * gq + e;
        const BcTarget tg = tgs[t];
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int ci = 2 * h + e;
#if FHE_BCONV_COMBINE32
            const u64 r = bc_combine71(acc[0][m][ci], acc[1][m][ci], acc[2][m][ci], acc[3][m][ci],
                                       acc[4][m][ci], acc[5][m][ci], acc[6][m][ci], tg);
#else
            u64 lo = (u64)(unsigned)acc[0][m][ci] + ((u64)(unsigned)acc[1][m][ci] << 8) +
                     ((u64)(unsigned)acc[2][m][ci] << 16) + ((u64)(unsigned)acc[3][m][ci] << 24) +
                     ((u64)(unsigned)acc[4][m][ci] << 32) + ((u64)(unsigned)acc[5][m][ci] << 40);
            u64 hi = 0;
            const u64 p6 = (u64)(unsigned)acc[6][m][ci];
            add_wide(hi, lo, p6 >> 16, p6 << 48);
            const u64 r = bc_reduce71(hi, lo, tg);
#endif
            if (t < nt) dst[(long)t * n + c0 + 16 * m + 8 * h + gr] = r;
          }
      }
    }
  }
}

// Shared memory of one CTA: the B fragments, the target and source
// constants, and per warp an A tile and TB C tiles.
inline size_t bconv_smem(int nt, int ks, int tb) {
  const int smax = (32 * ks) / 7;
  return (size_t)nt * ks * 32 * sizeof(uint2) + (size_t)nt * sizeof(BcTarget) +
         (size_t)smax * (2 * sizeof(double2) + sizeof(WPair)) + (size_t)((smax + 1) & ~1) * 8 +
         (size_t)kBcWarps * (32 * bc_astride(ks) + tb * 32 * kBcCStride) * sizeof(unsigned);
}

inline int bconv_ks(int ns) { return (7 * ns + 31) / 32; }

inline size_t bconv2_smem(int nt, int ks) {
  const int smax = (32 * ks) / 7, ng = (nt + 7) / 8;
  return (size_t)ng * 7 * ks * 32 * sizeof(uint2) + (size_t)8 * ng * sizeof(BcTarget) +
         (size_t)smax * (2 * sizeof(double2) + sizeof(WPair)) + (size_t)((smax + 1) & ~1) * 8 +
         (size_t)kBcWarps * 32 * bc_astride(ks) * sizeof(unsigned);
}

#ifndef FHE_BCONV_TB
#define FHE_BCONV_TB 2
#endif

template <int KS>
int launch_bconv_ks(const DevChain& ch, const BconvArgs& a, int max_nt, dim3 grid, cudaStream_t st) {
  if (a.layout2) {
    const size_t smem2 = bconv2_smem(max_nt, KS);
    auto go2 = [&](auto kern) -> int {
      if (smem2 > 48 * 1024)
        FHE_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem2));
      kern<<<grid, kBcThreads, smem2, st>>>(ch, a);
      FHE_LAUNCH_CHECK();
      return 0;
    };
    return (ch.fp64_ok && a.inv_d) ? go2(bconv_imma2_kernel<KS, true>)
                                   : go2(bconv_imma2_kernel<KS, false>);
  }
  constexpr int TB = FHE_BCONV_TB;
  const size_t smem = bconv_smem(max_nt, KS, TB);
  auto go = [&](auto kern) -> int {
    if (smem > 48 * 1024)
      FHE_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    kern<<<grid, kBcThreads, smem, st>>>(ch, a);
    FHE_LAUNCH_CHECK();
    return 0;
  };
  return (ch.fp64_ok && a.inv_d) ? go(bconv_imma_kernel<KS, TB, true>)
                                 : go(bconv_imma_kernel<KS, TB, false>);
}

int launch_bconv(const DevChain& ch, const BconvArgs& a, int max_ns, int max_nt, dim3 grid,
                 cudaStream_t st) {
  switch (bconv_ks(max_ns)) {
    case 1: return launch_bconv_ks<1>(ch, a, max_nt, grid, st);
    case 2: return launch_bconv_ks<2>(ch, a, max_nt, grid, st);
    case 3: return launch_bconv_ks<3>(ch, a, max_nt, grid, st);
    case 4: return launch_bconv_ks<4>(ch, a, max_nt, grid, st);
    default:
      fhe_set_error("tensor-core base conversion: more than 16 source limbs");
      return -1;
  }
}

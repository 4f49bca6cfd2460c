// Fast base conversion on the 5th-generation tensor cores (tcgen05, kind::i8),
// the default for ModUp and ModDown on sm_100a.  Same arithmetic as
// bconv_imma2_kernel (bconv_imma.cuh): y_s = [x_s inv_s]_{q_s} split into 7
// bytes, P_{t,b} = sum_{s,a} y_{s,a} W'_{(s,a),(t,b)} exact u8 x u8 -> s32
// dot products, out_t = (sum_b P_{t,b} 2^(8b)) mod p_t -- any exact
// evaluation gives the same canonical word.  Included by keyswitch.cu
// inside its anonymous namespace, after bconv_imma.cuh.
//
// Why tcgen05 rather than mma.sync: the mma.sync kernel kept its 56
// accumulator registers and 24 A-fragment registers per thread live through
// the epilogue, capping it at 2 CTAs (16 warps) per SM and 49% issue
// utilisation (ncu).  Here the accumulators live in TMEM and the operands
// stay in shared memory behind matrix descriptors, so the epilogue threads
// hold only the columns they reduce.
//
// Warp-specialised persistent CTA (416 threads), one tile = M = 128
// coefficients, every role looping over the CTA's tiles of one job:
//   warps 0-3   prologue: thread = coefficient; loads its ns source words,
//               forms y_s and writes its 7 ns bytes (K padded to 32 KS) as
//               one A row, canonical no-swizzle K-major layout (umma.cuh),
//               into one of 2 A stages;
//   warp 12     MMA issue (one thread): per chunk of kBuT targets (N = 8 kBuT
//               columns, target t byte b at column 8 t + b), KS K-steps into
//               one of kBuNbuf TMEM buffers, then commit;
//   warps 4-11  epilogue: warp w reads TMEM lanes 32 (w % 4) .. + 31 (lane =
//               coefficient) and half of the chunk's targets, releases the
//               buffer as soon as the columns are in registers, combines the
//               7 partials (bc_combine71) and stores 32 consecutive
//               coefficients (256 B) per target.
// The roles meet only at mbarriers (A full / empty, TMEM full / empty), so
// loads, MMAs and reductions of different tiles and chunks overlap.
// B (W' bytes, packed on the host by pack_bumma) is staged once per CTA.
#pragma once
#include "umma.cuh"

#ifndef FHE_BU_TARGETS
#define FHE_BU_TARGETS 8
#endif
#ifndef FHE_BU_NBUF
#define FHE_BU_NBUF 4
#endif
#ifndef FHE_BU_MINB
#define FHE_BU_MINB 2
#endif
constexpr int kBuProWarps = 4, kBuEpiWarps = 8;
constexpr int kBuThreads = 32 * (kBuProWarps + kBuEpiWarps + 1);
constexpr int kBuTile = 128;                   // coefficients per tile (MMA M)
constexpr int kBuT = FHE_BU_TARGETS;           // targets per TMEM chunk
constexpr int kBuCols = 8 * kBuT;              // columns per chunk (MMA N)
constexpr int kBuNbuf = FHE_BU_NBUF;           // TMEM chunk buffers
constexpr int kBuTmem = kBuNbuf * kBuCols;     // a power of 2 >= 32
static_assert(kBuT == 4 || kBuT == 8 || kBuT == 16, "chunk of 4, 8 or 16 targets");
static_assert((kBuTmem & (kBuTmem - 1)) == 0 && kBuTmem >= 32 && kBuTmem * FHE_BU_MINB <= 512,
              "TMEM columns");

__host__ __device__ constexpr int bu_abytes(int ks) { return 2 * ks * 2048; }

inline size_t bconv_umma_smem(int max_nt, int ks) {
  const int ng = (max_nt + 7) & ~7, smax = (32 * ks) / 7;
  return (size_t)2 * bu_abytes(ks) + (size_t)2 * ks * ng * 128 + (size_t)ng * sizeof(BcTarget) +
         (size_t)smax * (2 * sizeof(double2) + sizeof(WPair)) + (size_t)((smax + 1) & ~1) * 8 +
         (size_t)(4 + 2 * kBuNbuf) * 8 + 16;
}

// 79-bit form of bc_combine71 for targets p >= 2^56 (8 byte columns, sh >=
// 56): V = sum_{b<8} P_b 2^(8b) < 2^79, x = V >> sh < 2^23, mu = floor(2^79
// / p) < 2^23, qe = (x mu) >> (79 - sh) short of V / p by at most 2, r < 3p <
// 2^64 from the low words.
__device__ __forceinline__ u64 bc_combine79(const unsigned (&a)[8], const BcTarget& tg) {
  const u64 v = (u64)a[0] + ((u64)a[1] << 8) + ((u64)a[2] << 16) + ((u64)a[3] << 24);
  const u64 h = (u64)a[4] + ((u64)a[5] << 8) + ((u64)a[6] << 16) + ((u64)a[7] << 24);
  const u64 lo = v + (h << 32);
  const u64 hi = (h >> 32) + (lo < v ? 1 : 0);
  const u64 x = (hi << (64 - tg.sh)) | (lo >> tg.sh);
  const u64 qe = (x * (u64)tg.mu) >> (79 - tg.sh);
  u64 r = lo - qe * tg.p;
  r = csub(r, tg.p);
  return csub(r, tg.p);
}

// WT: some target may be >= 2^56 (79-bit reduction branch compiled in)
template <int KS, bool FPPRO, int SB = 7, bool WT = false>
__global__ void __launch_bounds__(kBuThreads, FHE_BU_MINB)
    bconv_umma_kernel(const DevChain ch, const BconvArgs a) {
  constexpr int SMAX = (32 * KS) / SB;
  constexpr int AB = bu_abytes(KS);
  extern __shared__ __align__(128) unsigned char bu_smem[];
  int ns = a.ns, nt = a.nt, s0 = 0, row_off = 0, buo = 0;
  if (a.dig_info) {
    const int di = blockIdx.y;
    s0 = a.dig_info[4 * di];
    ns = a.dig_info[4 * di + 1];
    row_off = a.dig_info[4 * di + 2];
    nt = a.level + a.K - ns;
    buo = a.bu_off[di];
  }
  const int ng = (nt + 7) & ~7;
  const int nch = (nt + kBuT - 1) / kBuT;
  unsigned char* sA = bu_smem;                                   // [2 stages][AB]
  unsigned char* sB = bu_smem + 2 * AB;                          // [2 KS][ng][8][16]
  BcTarget* tgs = reinterpret_cast<BcTarget*>(sB + 2 * KS * ng * 128);
  double2* sinv = reinterpret_cast<double2*>(tgs + ng);
  double2* sqd = sinv + SMAX;
  WPair* sinvi = reinterpret_cast<WPair*>(sqd + SMAX);
  u64* sqi = reinterpret_cast<u64*>(sinvi + SMAX);
  uint64_t* a_full = reinterpret_cast<uint64_t*>(sqi + ((SMAX + 1) & ~1));  // [2]
  uint64_t* a_empty = a_full + 2;                                         // [2]
  uint64_t* t_full = a_empty + 2;                                         // [kBuNbuf]
  uint64_t* t_empty = t_full + kBuNbuf;                                   // [kBuNbuf]
  unsigned* s_tm = reinterpret_cast<unsigned*>(t_empty + kBuNbuf);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  {
    const uint4* gb = a.bumma + buo;
    uint4* sb4 = reinterpret_cast<uint4*>(sB);
    for (int i = tid; i < 2 * KS * ng * 8; i += kBuThreads) sb4[i] = gb[i];
  }
  for (int t = tid; t < ng; t += kBuThreads) {
    if (t < nt) {
      const ModConst m = ch.mc[a.tgt_prime ? a.tgt_prime[row_off + t] : t];
      // mu = floor(2^71 / p), or floor(2^79 / p) for a wide target (sh >= 56)
      tgs[t] = BcTarget{m.q, (u32)(m.mu >> (m.s >= 56 ? m.s - 15 : m.s - 7)), (u32)m.s};
    } else {
      tgs[t] = BcTarget{1, 0, 39};
    }
  }
  for (int s = tid; s < SMAX; s += kBuThreads) {
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
  if (tid == 0) {
    for (int i = 0; i < 2; ++i) {
      umma_mbar_init(&a_full[i], 32 * kBuProWarps);
      umma_mbar_init(&a_empty[i], 1);
    }
    for (int i = 0; i < kBuNbuf; ++i) {
      umma_mbar_init(&t_full[i], 1);
      umma_mbar_init(&t_empty[i], 32 * kBuEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    tmem_alloc(s_tm, kBuTmem);
    tmem_relinquish();
  }
  fence_async_smem();
  umma_fence_before();
  __syncthreads();
  umma_fence_after();
  const unsigned tm = *s_tm;
  const long n = 1L << ch.log_n;
  const int ntiles = (int)(n / kBuTile);
  const u64* src = a.src + blockIdx.z * a.src_bstride + (long)s0 * n;
  u64* dst = a.dst + blockIdx.z * a.dst_bstride + (long)row_off * n;
  if (warp < kBuProWarps) {
    // ---- prologue: source words -> A rows
    int it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int s = it & 1;
      const long c = (long)tile * kBuTile + tid;
      u64 xs[SMAX];
#pragma unroll
      for (int k = 0; k < SMAX; ++k) xs[k] = k < ns ? src[(long)k * n + c] : 0;
      unsigned w[8 * KS];
#pragma unroll
      for (int i = 0; i < 8 * KS; ++i) w[i] = 0;
#pragma unroll
      for (int k = 0; k < SMAX; ++k) {
        if (k < ns) {
          u64 y;
          if (FPPRO) {
            const double2 qd = sqd[k];
            y = fp_to_u52(fp_pos(fp_mulmod(fp_from_u52(xs[k]), sinv[k], qd.x), qd.x));
          } else {
            const WPair iv = sinvi[k];
            y = shoup_mul(xs[k], iv.w, iv.sh, sqi[k]);
          }
          if constexpr (SB == 8) {
            w[2 * k] = (unsigned)y;
            w[2 * k + 1] = (unsigned)(y >> 32);
          } else {
            const int bit = 56 * k, wi = bit >> 5, sh = bit & 31;
            const u64 lo64 = y << sh;
            w[wi] |= (unsigned)lo64;
            w[wi + 1] |= (unsigned)(lo64 >> 32);
            if (sh > 8) w[wi + 2] |= (unsigned)(y >> (64 - sh));
          }
        }
      }
      umma_mbar_wait(&a_empty[s], ((it >> 1) & 1) ^ 1);  // stage s free (MMAs done)
      unsigned char* arow = sA + s * AB + tid * 16;
#pragma unroll
      for (int kc = 0; kc < 2 * KS; ++kc)
        *reinterpret_cast<uint4*>(arow + kc * 2048) =
            make_uint4(w[4 * kc], w[4 * kc + 1], w[4 * kc + 2], w[4 * kc + 3]);
      fence_async_smem();
      umma_mbar_arrive(&a_full[s]);
    }
  } else if (warp < kBuProWarps + kBuEpiWarps) {
    // ---- epilogue: TMEM partials -> canonical residues
    constexpr int TH = kBuT / 2;  // targets per warp per chunk
    const int q = warp & 3, h = (warp - kBuProWarps) >> 2;
    int g = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const long c = (long)tile * kBuTile + 32 * q + lane;
      for (int j = 0; j < nch; ++j, ++g) {
        const int b = g % kBuNbuf;
        umma_mbar_wait(&t_full[b], (g / kBuNbuf) & 1);
        umma_fence_after();
        const unsigned ta = tm + ((unsigned)(32 * q) << 16) + b * kBuCols + h * TH * 8;
        unsigned r[TH][8];
#pragma unroll
        for (int tl = 0; tl < TH; ++tl) tmem_ld8(ta + 8 * tl, r[tl]);
        tmem_ld_wait();
        umma_fence_before();
        umma_mbar_arrive(&t_empty[b]);
        const int tb = j * kBuT + h * TH;
        u64* o = dst + ((long)tb << ch.log_n) + c;
#pragma unroll
        for (int tl = 0; tl < TH; ++tl) {
          if (tb + tl < nt) {
            const BcTarget tg = tgs[tb + tl];  // one LDS.128
            if (WT && tg.sh >= 56)
              *o = bc_combine79(r[tl], tg);
            else
              *o = bc_combine71(r[tl][0], r[tl][1], r[tl][2], r[tl][3], r[tl][4], r[tl][5],
                                r[tl][6], tg);
          }
          o += n;
        }
      }
    }
  } else {
    // ---- MMA issue (one thread)
    if (lane == 0) {
      const unsigned aaddr = umma_smem_u32(sA), baddr = umma_smem_u32(sB);
      constexpr unsigned idesc = umma_idesc_u8(kBuTile, kBuCols);
      int it = 0, g = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
        const int s = it & 1;
        umma_mbar_wait(&a_full[s], (it >> 1) & 1);
        umma_fence_after();
        for (int j = 0; j < nch; ++j, ++g) {
          const int b = g % kBuNbuf;
          umma_mbar_wait(&t_empty[b], ((g / kBuNbuf) & 1) ^ 1);
          umma_fence_after();
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            const uint64_t ad = umma_desc(aaddr + s * AB + 2 * ks * 2048, 2048, 128);
            const uint64_t bd =
                umma_desc(baddr + (2 * ks * ng + j * kBuT) * 128, (unsigned)ng * 128, 128);
            umma_u8(tm + b * kBuCols, ad, bd, idesc, ks > 0);
          }
          umma_commit(&t_full[b]);
        }
        umma_commit(&a_empty[s]);
      }
    }
    __syncwarp();
  }
  umma_fence_before();
  __syncthreads();
  if (warp == 0) {
    umma_fence_after();
    tmem_dealloc(tm, kBuTmem);
  }
}

template <int KS, int SB, bool WT>
int launch_bconv_umma_ks(const DevChain& ch, const BconvArgs& a, int max_nt, dim3 grid,
                         cudaStream_t st) {
  const size_t smem = bconv_umma_smem(max_nt, KS);
  auto go = [&](auto kern) -> int {
    if (smem > 48 * 1024)
      FHE_CUDA_CHECK(
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<grid, kBuThreads, smem, st>>>(ch, a);
    FHE_LAUNCH_CHECK();
    return 0;
  };
  return (ch.fp64_ok && a.inv_d) ? go(bconv_umma_kernel<KS, true, SB, WT>)
                                 : go(bconv_umma_kernel<KS, false, SB, WT>);
}

// grid.x CTAs per job, each looping over 128-coefficient tiles (n >= 128);
// sb bytes per source word (7, or 8 for sources >= 2^56)
int launch_bconv_umma(const DevChain& ch, const BconvArgs& a, int max_ns, int max_nt, dim3 grid,
                      cudaStream_t st, int sb = 7, bool wide_targets = false) {
  if (sb == 8) {
    switch ((8 * max_ns + 31) / 32) {
      case 1: return launch_bconv_umma_ks<1, 8, true>(ch, a, max_nt, grid, st);
      case 2: return launch_bconv_umma_ks<2, 8, true>(ch, a, max_nt, grid, st);
      case 3: return launch_bconv_umma_ks<3, 8, true>(ch, a, max_nt, grid, st);
      case 4: return launch_bconv_umma_ks<4, 8, true>(ch, a, max_nt, grid, st);
      default:
        fhe_set_error("tcgen05 base conversion: more than 16 wide source limbs");
        return -1;
    }
  }
  if (wide_targets) {
    switch (bconv_ks(max_ns)) {
      case 1: return launch_bconv_umma_ks<1, 7, true>(ch, a, max_nt, grid, st);
      case 2: return launch_bconv_umma_ks<2, 7, true>(ch, a, max_nt, grid, st);
      case 3: return launch_bconv_umma_ks<3, 7, true>(ch, a, max_nt, grid, st);
      case 4: return launch_bconv_umma_ks<4, 7, true>(ch, a, max_nt, grid, st);
      default: break;
    }
  }
  switch (bconv_ks(max_ns)) {
    case 1: return launch_bconv_umma_ks<1, 7, false>(ch, a, max_nt, grid, st);
    case 2: return launch_bconv_umma_ks<2, 7, false>(ch, a, max_nt, grid, st);
    case 3: return launch_bconv_umma_ks<3, 7, false>(ch, a, max_nt, grid, st);
    case 4: return launch_bconv_umma_ks<4, 7, false>(ch, a, max_nt, grid, st);
    default:
      fhe_set_error("tcgen05 base conversion: more than 16 source limbs");
      return -1;
  }
}

// One N = 2^12 row per 4-CTA thread-block cluster (latency path for small
// launches: the PDQ ring, a few to ~150 rows per transform).  Included by
// ntt.cu inside its anonymous namespace, after ntt_tiles.cuh.
//
// A whole-row tile runs the row's 12 stages on one SM, and at one row per
// SM its time is set by that SM's FP64 pipe and the pass latencies (~6 us,
// profiles/r2_pdq_latency.md).  Here the row's 24576 butterflies are spread
// over 4 SMs:
//   forward (Cooley-Tukey, the merged negacyclic twiddles of the chain's
//   natural-order table, index 2^s + group at stage s):
//     A  CTA r, thread t owns position p = 256 r + t of the four 1024-point
//        blocks: x[p + 1024 j], j = 0..3; stages 0 and 1 are one radix-4
//        butterfly across the blocks;
//     X  x_j goes to CTA j's shared memory at block position p (DSMEM store),
//        one cluster barrier;
//     B  CTA k runs stages 2..11 on block k: 5 radix-4 steps through shared
//        memory, group g of local stage t reading twiddle 2^(t+2) + k 2^t + g;
//        the last step stores 4 consecutive canonical words per thread.
//   inverse (Gentleman-Sande, inverse table): the same three phases in
//   reverse, n^-1 folded into stage 0 (ninv / ninv_w1, as the tile passes).
// Every twiddle a thread needs (18 pairs) is loaded before the data, so no
// step waits on L2.  Lazy-reduction schedule and arithmetic are those of the
// tile passes (ntt_tiles.cuh run_pass_fp): forward u reduced on stages
// s = 3 mod 4, inverse sums reduced on even stages; results are canonical,
// so they are the same words as every other transform path.
#pragma once

constexpr int kRcThreads = 256;

__device__ __forceinline__ void rc_barrier_arrive_relaxed() {
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void rc_barrier_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void rc_barrier_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned rc_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// store a double into CTA `rank`'s shared memory at the address of `local`
__device__ __forceinline__ void rc_st_remote(double* local, unsigned rank, double v) {
  unsigned la = (unsigned)__cvta_generic_to_shared(local), ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}

// forward CT butterfly of the tile passes at global stage s
__device__ __forceinline__ void rc_fwd_bf(double& a, double& c, double2 w, double2 qd, int s) {
  const double u = (s & 3) == 3 ? fp_reduce(a, qd) : a;
  const double t = fp_mulmod(c, w, qd.x);
  a = __dadd_rn(u, t);
  c = __dadd_rn(u, -t);
}
// inverse GS butterfly at global stage s (not the folded stage 0)
__device__ __forceinline__ void rc_inv_bf(double& a, double& c, double2 w, double2 qd, int s) {
  const double sm = __dadd_rn(a, c);
  const double d = __dadd_rn(a, -c);
  a = (s & 1) == 0 ? fp_reduce(sm, qd) : sm;
  c = fp_mulmod(d, w, qd.x);
}

// PF: every twiddle prefetched into registers before the data (latency mode,
// 96 registers, 2 CTAs/SM); !PF: each radix-4 step loads its 3 twiddles when
// it starts and the register budget admits 4 CTAs/SM (throughput mode, larger
// launches, where other CTAs cover the loads)
template <bool FWD, bool PF = true>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kRcThreads, PF ? 1 : 4)
    ntt_row_cluster_kernel(const DevChain ch, u64* dst, const u64* src, RowMap map, RowAddr sa,
                           RowAddr da, int bcast_limbs, long bcast_stride, double center,
                           const u64* __restrict__ rs_in = nullptr, u64* rs_out = nullptr,
                           const double2* __restrict__ rs_inv_d = nullptr, int rs_level = 0) {
  __shared__ double blk[1024];   // this CTA's 1024-point block (phase B)
  __shared__ double xch[1024];   // inverse: the 4 x 256 cross-block values (phase A)
  const int row = blockIdx.x >> 2;
  const unsigned k = rc_rank();
  const int t = threadIdx.x;
  const int p = map(row);
  const double2 qd = ch.qd[p];
  const double2* tw = (FWD ? ch.twd : ch.itwd) + ((size_t)p << 12);
  // all blocks of the cluster are running before any DSMEM store
  rc_barrier_arrive_relaxed();
  // twiddles: phase A (stages 0, 1) and the 5 radix-4 steps of phase B
  // step i's twiddles: group g0 = t / (h / 2) of local stage 2 i, groups
  // 2 g0, 2 g0 + 1 of local stage 2 i + 1
  auto twa = [&](int i) {
    return __ldg(tw + (1 << (2 * i + 2)) + ((int)k << (2 * i)) + t / (256 >> (2 * i)));
  };
  auto twb = [&](int i) {
    return __ldg(tw + (1 << (2 * i + 3)) + ((int)k << (2 * i + 1)) + 2 * (t / (256 >> (2 * i))));
  };
  auto twc = [&](int i) {
    return __ldg(tw + (1 << (2 * i + 3)) + ((int)k << (2 * i + 1)) + 2 * (t / (256 >> (2 * i))) +
                 1);
  };
  double2 wa[PF ? 5 : 1], wb[PF ? 5 : 1], wc[PF ? 5 : 1];
  if constexpr (PF) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      wa[i] = twa(i);
      wb[i] = twb(i);
      wc[i] = twc(i);
    }
  }
  auto WA = [&](int i) {
    if constexpr (PF) return wa[i]; else return twa(i);
  };
  auto WB = [&](int i) {
    if constexpr (PF) return wb[i]; else return twb(i);
  };
  auto WC = [&](int i) {
    if constexpr (PF) return wc[i]; else return twc(i);
  };
  const double2 w0 = __ldg(tw + 1), w1a = __ldg(tw + 2), w1b = __ldg(tw + 3);
  // broadcast input (forward only): row r reads row r / bcast_limbs of src,
  // centred about `center` when nonzero (the rescale correction, as RowsTile)
  const u64* s_row = bcast_limbs ? src + (long)(row / bcast_limbs) * bcast_stride : src + sa(row);
  u64* d_row = dst + da(row);
  if (FWD) {
    // ---- A: stages 0, 1 across the blocks
    const int pos = 256 * (int)k + t;
    double x[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      x[j] = fp_from_u52(s_row[pos + 1024 * j]);
      if (center != 0.0) x[j] = x[j] > 0.5 * center ? __dadd_rn(x[j], -center) : x[j];
    }
    rc_fwd_bf(x[0], x[2], w0, qd, 0);
    rc_fwd_bf(x[1], x[3], w0, qd, 0);
    rc_fwd_bf(x[0], x[1], w1a, qd, 1);
    rc_fwd_bf(x[2], x[3], w1b, qd, 1);
    // ---- X: x_j -> block j, position pos
    rc_barrier_wait();
#pragma unroll
    for (int j = 0; j < 4; ++j) rc_st_remote(&blk[pos], j, x[j]);
    rc_barrier_arrive_release();
    rc_barrier_wait();
    // ---- B: stages 2..11 on block k
#pragma unroll
    for (int i = 0; i < 5; ++i) {
      const int t0 = 2 * i, h = 512 >> t0, h2 = h >> 1;
      const int b = (t / h2) * 2 * h + (t % h2);
      const double2 sa = WA(i), sb = WB(i), sc = WC(i);
      double y0 = blk[b], y1 = blk[b + h2], y2 = blk[b + h], y3 = blk[b + h + h2];
      rc_fwd_bf(y0, y2, sa, qd, t0 + 2);
      rc_fwd_bf(y1, y3, sa, qd, t0 + 2);
      rc_fwd_bf(y0, y1, sb, qd, t0 + 3);
      rc_fwd_bf(y2, y3, sc, qd, t0 + 3);
      if (i < 4) {
        __syncthreads();
        blk[b] = y0;
        blk[b + h2] = y1;
        blk[b + h] = y2;
        blk[b + h + h2] = y3;
        __syncthreads();
      } else {
        // last step: b = 4 t, four consecutive outputs
        if (rs_in) {
          // rescale finish: (in - correction) * q_last^-1 on the FP64 pipe
          // (|in - x| < 1.5 q, one product, canonical word), written to the
          // new level's row (poly, j) -- the word launch_modswitch_finish makes
          const int nl = rs_level - 1, poly = row / nl, j = row - poly * nl;
          const long off = 1024 * (long)k + b;
          const ulonglong2 i01 =
              *reinterpret_cast<const ulonglong2*>(rs_in + ((long)poly * rs_level + j) * 4096 + off);
          const ulonglong2 i23 = *reinterpret_cast<const ulonglong2*>(
              rs_in + ((long)poly * rs_level + j) * 4096 + off + 2);
          const double2 iv = rs_inv_d[j];
          auto fin = [&](u64 a, double y) {
            const double d = __dadd_rn(fp_from_u52(a), -fp_reduce(y, qd));
            return fp_canon_half(fp_mulmod(d, iv, qd.x), qd.x);
          };
          u64* o = rs_out + ((long)poly * nl + j) * 4096 + off;
          *reinterpret_cast<ulonglong2*>(o) = make_ulonglong2(fin(i01.x, y0), fin(i01.y, y1));
          *reinterpret_cast<ulonglong2*>(o + 2) = make_ulonglong2(fin(i23.x, y2), fin(i23.y, y3));
        } else {
          u64* o = d_row + 1024 * k + b;
          *reinterpret_cast<ulonglong2*>(o) =
              make_ulonglong2(fp_canon_half(fp_reduce(y0, qd), qd.x),
                              fp_canon_half(fp_reduce(y1, qd), qd.x));
          *reinterpret_cast<ulonglong2*>(o + 2) =
              make_ulonglong2(fp_canon_half(fp_reduce(y2, qd), qd.x),
                              fp_canon_half(fp_reduce(y3, qd), qd.x));
        }
      }
    }
  } else {
    // ---- B: stages 11..2 on block k (loaded contiguously)
    const u64* in = s_row + 1024 * k;
    {
      const ulonglong2 v0 = *reinterpret_cast<const ulonglong2*>(in + 4 * t);
      const ulonglong2 v1 = *reinterpret_cast<const ulonglong2*>(in + 4 * t + 2);
      double y0 = fp_from_u52(v0.x), y1 = fp_from_u52(v0.y), y2 = fp_from_u52(v1.x),
             y3 = fp_from_u52(v1.y);
      // step 4 (stages 11, 10): b = 4 t
      const double2 sa = WA(4), sb = WB(4), sc = WC(4);
      rc_inv_bf(y0, y1, sb, qd, 11);
      rc_inv_bf(y2, y3, sc, qd, 11);
      rc_inv_bf(y0, y2, sa, qd, 10);
      rc_inv_bf(y1, y3, sa, qd, 10);
      blk[4 * t] = y0;
      blk[4 * t + 1] = y1;
      blk[4 * t + 2] = y2;
      blk[4 * t + 3] = y3;
      __syncthreads();
    }
    double z[4];
#pragma unroll
    for (int i = 3; i >= 0; --i) {
      const int t0 = 2 * i, h = 512 >> t0, h2 = h >> 1;
      const int b = (t / h2) * 2 * h + (t % h2);
      const double2 sa = WA(i), sb = WB(i), sc = WC(i);
      double y0 = blk[b], y1 = blk[b + h2], y2 = blk[b + h], y3 = blk[b + h + h2];
      rc_inv_bf(y0, y1, sb, qd, t0 + 3);
      rc_inv_bf(y2, y3, sc, qd, t0 + 3);
      rc_inv_bf(y0, y2, sa, qd, t0 + 2);
      rc_inv_bf(y1, y3, sa, qd, t0 + 2);
      if (i > 0) {
        __syncthreads();
        blk[b] = y0;
        blk[b + h2] = y1;
        blk[b + h] = y2;
        blk[b + h + h2] = y3;
        __syncthreads();
      } else {
        // step 0: b = t; block positions t, t + 256, t + 512, t + 768 go to
        // CTAs 0..3 (position p = 256 r + t' lives in CTA r, slot [k][t'])
        z[0] = y0;
        z[1] = y1;
        z[2] = y2;
        z[3] = y3;
      }
    }
    // ---- X: block k position 256 r + t -> CTA r, slot 256 k + t
    rc_barrier_wait();
#pragma unroll
    for (int r = 0; r < 4; ++r) rc_st_remote(&xch[256 * k + t], r, z[r]);
    rc_barrier_arrive_release();
    rc_barrier_wait();
    // ---- A: stages 1, 0 across the blocks at position 256 k + t
    double x0 = xch[t], x1 = xch[256 + t], x2 = xch[512 + t], x3 = xch[768 + t];
    rc_inv_bf(x0, x1, w1a, qd, 1);
    rc_inv_bf(x2, x3, w1b, qd, 1);
    const double2 sn = ch.ninv_d[p], wf = ch.ninv_w1_d[p];
    {
      const double s0 = __dadd_rn(x0, x2), d0 = __dadd_rn(x0, -x2);
      const double s1 = __dadd_rn(x1, x3), d1 = __dadd_rn(x1, -x3);
      x0 = fp_mulmod(s0, sn, qd.x);
      x2 = fp_mulmod(d0, wf, qd.x);
      x1 = fp_mulmod(s1, sn, qd.x);
      x3 = fp_mulmod(d1, wf, qd.x);
    }
    const int pos = 256 * (int)k + t;
    d_row[pos] = fp_canon_half(x0, qd.x);
    d_row[pos + 1024] = fp_canon_half(x1, qd.x);
    d_row[pos + 2048] = fp_canon_half(x2, qd.x);
    d_row[pos + 3072] = fp_canon_half(x3, qd.x);
  }
}

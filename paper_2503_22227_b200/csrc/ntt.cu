// Batched negacyclic NTT / INTT over RNS limbs for sm_100a.
//
// Semantics follow the reference CPU kernels exactly:
//   forward  = Cooley-Tukey, t = N/2 .. 1, twiddle psi_br[m + i]
//              (coremath/_kernels.py:35-57, coremath/ntt.py:145-169)
//   inverse  = Gentleman-Sande, t = 1 .. N/2, twiddle ipsi_br[h + i], then
//              multiply by n^-1 (coremath/_kernels.py:60-85, ntt.py:172-198)
// Output is bit-reversed evaluation order (slot j = a(psi^(2 bitrev(j)+1)),
// ntt.py:1-7) and canonical in [0, q), so it is bit-identical to
// NttChain.forward/inverse (ntt.py:277-351).
//
// B200 design:
//  * radix-2^e register passes (e = 4..5): each thread owns 2^e elements and
//    runs e butterfly stages in registers between shared-memory exchanges,
//    so shared memory is touched once per e stages, not once per stage;
//  * Harvey lazy butterflies (values kept in [0,4q) forward / [0,2q)
//    inverse; valid because q < 2^62, modmath.py:36) - one conditional
//    subtraction per butterfly instead of two;
//  * n^-1 folded into the last inverse stage (no separate scaling pass);
//  * XOR-swizzled shared memory so both the strided and the contiguous
//    register passes are bank-conflict free;
//  * N <= 2^13: whole rows in shared memory, one HBM round trip.
//    N >= 2^14: four-step split N = N1 * N2: a column kernel runs the first
//    log N1 stages on 16-column tiles (128-byte coalesced segments), a chunk
//    kernel runs the remaining log N2 stages on contiguous N2-chunks.
#include "fhe_kernels.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int swz(int i) { return i ^ ((i >> 4) & 15); }

// Pass schedule: ceil(log_s / 5) passes, the remainder spread over the first
// passes (larger passes first keeps the contiguous last pass at e <= 4).
constexpr int npass(int log_s) { return (log_s + 4) / 5; }
constexpr int pass_e(int log_s, int p) {
  return log_s / npass(log_s) + (p < log_s % npass(log_s) ? 1 : 0);
}
constexpr int pass_r0(int log_s, int p) {
  int r = 0;
  for (int i = 0; i < p; ++i) r += pass_e(log_s, i);
  return r;
}

// Arrays stored contiguously (array b element k at swz(b*S + k)); groups
// enumerate arrays slowest so a warp stays inside one array.
template <int LOG_S>
struct RowLayout {
  __device__ __forceinline__ int idx(int b, int k) const { return swz((b << LOG_S) + k); }
  __device__ __forceinline__ void split(int G, int gpa_log, int& b, int& g) const {
    b = G >> gpa_log;
    g = G & ((1 << gpa_log) - 1);
  }
};

// Column tile: array b (a column) element k at k*NB + b; groups enumerate
// columns fastest so consecutive lanes touch consecutive words.
template <int NB>
struct ColLayout {
  __device__ __forceinline__ int idx(int b, int k) const { return k * NB + b; }
  __device__ __forceinline__ void split(int G, int, int& b, int& g) const {
    b = G % NB;
    g = G / NB;
  }
};

// Per-array twiddle context.
struct ArrCtx {
  const WPair* tw;   // table of the array's prime (forward or inverse)
  u64 q;
  int m0;            // global group base: twiddle index = (m0 << r) + g_local
  const WPair* sn;   // inverse only: n^-1 folded into global stage 0 (or null)
  const WPair* sw1;  // inverse only: ipsi_br[1] * n^-1
};

// One register pass covering local stages R0 .. R0+E_LOG-1.
template <int LOG_S, int R0, int E_LOG, bool FWD, class Lay, class CtxFn>
__device__ __forceinline__ void run_pass(u64* sm, int nb, const Lay& lay, const CtxFn& ctx) {
  constexpr int E = 1 << E_LOG;
  constexpr int S = 1 << LOG_S;
  constexpr int T0 = S >> (R0 + 1);
  constexpr int TMIN_LOG = LOG_S - R0 - E_LOG;
  constexpr int GPA_LOG = LOG_S - E_LOG;
  const int total = nb << GPA_LOG;
  for (int G = threadIdx.x; G < total; G += blockDim.x) {
    int b, g;
    lay.split(G, GPA_LOG, b, g);
    const int hi = g >> TMIN_LOG;
    const int lo = g & ((1 << TMIN_LOG) - 1);
    const int base = hi * 2 * T0 + lo;
    const ArrCtx cx = ctx(b);
    const u64 q = cx.q;
    const u64 q2 = 2 * q;
    u64 x[E];
#pragma unroll
    for (int i = 0; i < E; ++i) x[i] = sm[lay.idx(b, base + (i << TMIN_LOG))];
    if (FWD) {
#pragma unroll
      for (int rr = 0; rr < E_LOG; ++rr) {
        const int half = E >> (rr + 1);
#pragma unroll
        for (int blk = 0; blk < (1 << rr); ++blk) {
          const WPair w = cx.tw[(cx.m0 << (R0 + rr)) + (hi << rr) + blk];
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const int a = blk * 2 * half + i, c = a + half;
            u64 u = x[a];
            u = u >= q2 ? u - q2 : u;
            const u64 v = shoup_lazy(x[c], w.w, w.sh, q);
            x[a] = u + v;
            x[c] = u - v + q2;
          }
        }
      }
    } else {
#pragma unroll
      for (int rr = E_LOG - 1; rr >= 0; --rr) {
        const int half = E >> (rr + 1);
        const bool fold_ninv = (R0 == 0) && (rr == 0) && (cx.sn != nullptr);
#pragma unroll
        for (int blk = 0; blk < (1 << rr); ++blk) {
          const WPair w = cx.tw[(cx.m0 << (R0 + rr)) + (hi << rr) + blk];
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const int a = blk * 2 * half + i, c = a + half;
            const u64 u = x[a], v = x[c];
            const u64 s = u + v;
            const u64 d = u - v + q2;
            if (fold_ninv) {
              // last GS stage with n^-1 folded in; outputs canonical
              x[a] = shoup_mul(s, cx.sn->w, cx.sn->sh, q);
              x[c] = shoup_mul(d, cx.sw1->w, cx.sw1->sh, q);
            } else {
              x[a] = s >= q2 ? s - q2 : s;
              x[c] = shoup_lazy(d, w.w, w.sh, q);
            }
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < E; ++i) sm[lay.idx(b, base + (i << TMIN_LOG))] = x[i];
  }
}

template <int LOG_S, int P, class Lay, class CtxFn>
__device__ __forceinline__ void fwd_passes(u64* sm, int nb, const Lay& lay, const CtxFn& ctx) {
  if constexpr (P < npass(LOG_S)) {
    run_pass<LOG_S, pass_r0(LOG_S, P), pass_e(LOG_S, P), true>(sm, nb, lay, ctx);
    __syncthreads();
    fwd_passes<LOG_S, P + 1>(sm, nb, lay, ctx);
  }
}

template <int LOG_S, int P, class Lay, class CtxFn>
__device__ __forceinline__ void inv_passes(u64* sm, int nb, const Lay& lay, const CtxFn& ctx) {
  if constexpr (P >= 0) {
    run_pass<LOG_S, pass_r0(LOG_S, P), pass_e(LOG_S, P), false>(sm, nb, lay, ctx);
    __syncthreads();
    inv_passes<LOG_S, P - 1>(sm, nb, lay, ctx);
  }
}

// ---------------------------------------------------------------------------
// Whole rows in shared memory (N <= 2^13).  NB rows per CTA.
template <int LOG_N, bool FWD>
__global__ void __launch_bounds__(kThreads) ntt_rows_kernel(DevChain ch, u64* data, const u64* src,
                                                            int rows, RowMap map) {
  constexpr int S = 1 << LOG_N;
  constexpr int NB = S >= 2048 ? 1 : 2048 / S;
  extern __shared__ u64 sm[];
  const int row0 = blockIdx.x * NB;
  const int nb = min(NB, rows - row0);
  __shared__ int prime[NB];
  for (int i = threadIdx.x; i < nb; i += blockDim.x) prime[i] = map(row0 + i);
  u64* g = data + (size_t)row0 * S;
  const int nel = nb * S;
  if (S >= 2) {
    const ulonglong2* g2 = reinterpret_cast<const ulonglong2*>(src + (size_t)row0 * S);
    for (int i = threadIdx.x; i < nel / 2; i += blockDim.x) {
      const ulonglong2 v = g2[i];
      sm[swz(2 * i)] = v.x;
      sm[swz(2 * i + 1)] = v.y;
    }
  }
  __syncthreads();
  RowLayout<LOG_N> lay;
  const WPair* table = FWD ? ch.tw : ch.itw;
  auto ctx = [&](int b) {
    const int p = prime[b];
    return ArrCtx{table + ((size_t)p << LOG_N), ch.mc[p].q, 1, FWD ? nullptr : &ch.ninv[p],
                  FWD ? nullptr : &ch.ninv_w1[p]};
  };
  if (FWD)
    fwd_passes<LOG_N, 0>(sm, nb, lay, ctx);
  else
    inv_passes<LOG_N, npass(LOG_N) - 1>(sm, nb, lay, ctx);
  ulonglong2* o2 = reinterpret_cast<ulonglong2*>(g);
  for (int i = threadIdx.x; i < nel / 2; i += blockDim.x) {
    u64 a = sm[swz(2 * i)], b = sm[swz(2 * i + 1)];
    if (FWD) {
      const u64 q = ch.mc[prime[(2 * i) >> LOG_N]].q;
      a = csub(csub(a, 2 * q), q);
      b = csub(csub(b, 2 * q), q);
    }
    o2[i] = make_ulonglong2(a, b);
  }
}

// ---------------------------------------------------------------------------
// Four-step split for N >= 2^14: N = N1 * N2, N1 = 2^LOG_N1.
constexpr int kCols = 16;  // columns per tile: 16 x 8 B = one 128-byte segment

// Column stages (global stages 0 .. LOG_N1-1) on a [N1][kCols] tile.
template <int LOG_N, int LOG_N1, bool FWD>
__global__ void __launch_bounds__(kThreads) ntt_cols_kernel(DevChain ch, u64* data, const u64* src,
                                                            RowMap map) {
  constexpr int N = 1 << LOG_N;
  constexpr int N1 = 1 << LOG_N1;
  constexpr int N2 = N / N1;
  constexpr int TILES = N2 / kCols;
  __shared__ __align__(16) u64 sm[N1 * kCols];
  const int row = blockIdx.x / TILES;
  const int j0 = (blockIdx.x % TILES) * kCols;
  const int p = map(row);
  const u64 q = ch.mc[p].q;
  u64* g = data + (size_t)row * N + j0;
  const u64* gs = src + (size_t)row * N + j0;
  for (int i = threadIdx.x; i < N1 * kCols / 2; i += blockDim.x) {
    const int e = 2 * i, k = e / kCols, b = e % kCols;
    const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(gs + (size_t)k * N2 + b);
    sm[k * kCols + b] = v.x;
    sm[k * kCols + b + 1] = v.y;
  }
  __syncthreads();
  ColLayout<kCols> lay;
  const WPair* table = (FWD ? ch.tw : ch.itw) + ((size_t)p << LOG_N);
  const WPair* sn = FWD ? nullptr : &ch.ninv[p];
  const WPair* sw1 = FWD ? nullptr : &ch.ninv_w1[p];
  auto ctx = [&](int) { return ArrCtx{table, q, 1, sn, sw1}; };
  if (FWD)
    fwd_passes<LOG_N1, 0>(sm, kCols, lay, ctx);
  else
    inv_passes<LOG_N1, npass(LOG_N1) - 1>(sm, kCols, lay, ctx);
  for (int i = threadIdx.x; i < N1 * kCols / 2; i += blockDim.x) {
    const int e = 2 * i, k = e / kCols, b = e % kCols;
    *reinterpret_cast<ulonglong2*>(g + (size_t)k * N2 + b) =
        make_ulonglong2(sm[k * kCols + b], sm[k * kCols + b + 1]);
  }
}

// Chunk stages (global stages LOG_N1 .. LOG_N-1) on NB contiguous N2-chunks.
template <int LOG_N, int LOG_N1, bool FWD>
__global__ void __launch_bounds__(kThreads) ntt_chunks_kernel(DevChain ch, u64* data, const u64* src,
                                                              RowMap map) {
  constexpr int N = 1 << LOG_N;
  constexpr int N1 = 1 << LOG_N1;
  constexpr int LOG_N2 = LOG_N - LOG_N1;
  constexpr int N2 = 1 << LOG_N2;
  constexpr int NB = 4096 / N2 > 0 ? 4096 / N2 : 1;
  constexpr int TILES = N1 / NB;
  __shared__ __align__(16) u64 sm[NB * N2];
  const int row = blockIdx.x / TILES;
  const int c0 = (blockIdx.x % TILES) * NB;
  const int p = map(row);
  const u64 q = ch.mc[p].q;
  u64* g = data + (size_t)row * N + (size_t)c0 * N2;
  const ulonglong2* g2 =
      reinterpret_cast<const ulonglong2*>(src + (size_t)row * N + (size_t)c0 * N2);
  for (int i = threadIdx.x; i < NB * N2 / 2; i += blockDim.x) {
    const ulonglong2 v = g2[i];
    sm[swz(2 * i)] = v.x;
    sm[swz(2 * i + 1)] = v.y;
  }
  __syncthreads();
  RowLayout<LOG_N2> lay;
  const WPair* table = (FWD ? ch.tw : ch.itw) + ((size_t)p << LOG_N);
  auto ctx = [&](int b) { return ArrCtx{table, q, N1 + c0 + b, nullptr, nullptr}; };
  if (FWD)
    fwd_passes<LOG_N2, 0>(sm, NB, lay, ctx);
  else
    inv_passes<LOG_N2, npass(LOG_N2) - 1>(sm, NB, lay, ctx);
  ulonglong2* o2 = reinterpret_cast<ulonglong2*>(g);
  for (int i = threadIdx.x; i < NB * N2 / 2; i += blockDim.x) {
    u64 a = sm[swz(2 * i)], b = sm[swz(2 * i + 1)];
    if (FWD) {
      a = csub(csub(a, 2 * q), q);
      b = csub(csub(b, 2 * q), q);
    }
    o2[i] = make_ulonglong2(a, b);
  }
}

template <int LOG_N>
int launch_rows(const DevChain& ch, u64* data, const u64* in, int rows, RowMap map,
                bool inverse, cudaStream_t st) {
  constexpr int S = 1 << LOG_N;
  constexpr int NB = S >= 2048 ? 1 : 2048 / S;
  const int grid = (rows + NB - 1) / NB;
  const size_t smem = (size_t)NB * S * sizeof(u64);
  if (inverse) {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(ntt_rows_kernel<LOG_N, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ntt_rows_kernel<LOG_N, false><<<grid, kThreads, smem, st>>>(ch, data, in, rows, map);
  } else {
    if (smem > 48 * 1024)
      cudaFuncSetAttribute(ntt_rows_kernel<LOG_N, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    ntt_rows_kernel<LOG_N, true><<<grid, kThreads, smem, st>>>(ch, data, in, rows, map);
  }
  FHE_LAUNCH_CHECK();
  return 0;
}

template <int LOG_N, int LOG_N1>
int launch_split(const DevChain& ch, u64* data, const u64* in, int rows, RowMap map,
                 bool inverse, cudaStream_t st) {
  constexpr int N = 1 << LOG_N;
  constexpr int N2 = N >> LOG_N1;
  constexpr int NB = 4096 / N2 > 0 ? 4096 / N2 : 1;
  const int grid_cols = rows * (N2 / kCols);
  const int grid_chunks = rows * ((1 << LOG_N1) / NB);
  if (!inverse) {
    ntt_cols_kernel<LOG_N, LOG_N1, true><<<grid_cols, kThreads, 0, st>>>(ch, data, in, map);
    ntt_chunks_kernel<LOG_N, LOG_N1, true><<<grid_chunks, kThreads, 0, st>>>(ch, data, data,
                                                                            map);
  } else {
    ntt_chunks_kernel<LOG_N, LOG_N1, false><<<grid_chunks, kThreads, 0, st>>>(ch, data, in, map);
    ntt_cols_kernel<LOG_N, LOG_N1, false><<<grid_cols, kThreads, 0, st>>>(ch, data, data, map);
  }
  FHE_LAUNCH_CHECK();
  return 0;
}

}  // namespace

int launch_ntt(const DevChain& ch, u64* data, const u64* in, int rows, RowMap map, bool inverse,
               cudaStream_t st) {
  if (rows <= 0) return 0;
  switch (ch.log_n) {
    case 1: return launch_rows<1>(ch, data, in, rows, map, inverse, st);
    case 2: return launch_rows<2>(ch, data, in, rows, map, inverse, st);
    case 3: return launch_rows<3>(ch, data, in, rows, map, inverse, st);
    case 4: return launch_rows<4>(ch, data, in, rows, map, inverse, st);
    case 5: return launch_rows<5>(ch, data, in, rows, map, inverse, st);
    case 6: return launch_rows<6>(ch, data, in, rows, map, inverse, st);
    case 7: return launch_rows<7>(ch, data, in, rows, map, inverse, st);
    case 8: return launch_rows<8>(ch, data, in, rows, map, inverse, st);
    case 9: return launch_rows<9>(ch, data, in, rows, map, inverse, st);
    case 10: return launch_rows<10>(ch, data, in, rows, map, inverse, st);
    case 11: return launch_rows<11>(ch, data, in, rows, map, inverse, st);
    case 12: return launch_rows<12>(ch, data, in, rows, map, inverse, st);
    case 13: return launch_rows<13>(ch, data, in, rows, map, inverse, st);
    case 14: return launch_split<14, 7>(ch, data, in, rows, map, inverse, st);
    case 15: return launch_split<15, 7>(ch, data, in, rows, map, inverse, st);
    case 16: return launch_split<16, 8>(ch, data, in, rows, map, inverse, st);
    case 17: return launch_split<17, 8>(ch, data, in, rows, map, inverse, st);
    default:
      fhe_set_error("unsupported ring degree 2^" + std::to_string(ch.log_n));
      return -1;
  }
}

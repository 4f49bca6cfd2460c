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
//  * persistent CTAs (two per SM) walking tiles; each tile is brought into
//    shared memory with cp.async while the previous tile computes (double
//    buffer), so HBM latency overlaps the integer work;
//  * radix-2^e register passes (e = 4..5): each thread owns 2^e elements and
//    runs e butterfly stages in registers between shared-memory exchanges;
//    the last pass writes straight from registers to HBM;
//  * lazy butterflies: for chains whose primes are < 2^58 the forward
//    transform never reduces inside the butterfly (values grow by < 2q per
//    stage, < 33q after 16 stages) and reduces once at the end; otherwise
//    Harvey's [0,4q) forward / [0,2q) inverse butterflies (q < 2^62,
//    modmath.py:36);
//  * n^-1 folded into the last inverse stage;
//  * padded shared-memory rows (16 bytes per 128): strided passes (8-byte
//    accesses) and contiguous passes (16-byte accesses) are both
//    bank-conflict free with immediate-offset addressing;
//  * N <= 2^12: whole rows per tile (one HBM round trip).  N >= 2^13:
//    four-step split N = N1 * N2: a column kernel runs the first log N1
//    stages on [N1 x 16]-column tiles (128-byte segments), a chunk kernel
//    the remaining log N2 stages on contiguous N2-chunks.
#include "fhe_kernels.cuh"
#include "fparith.cuh"
#include "ntt_plan.cuh"

#include <cuda.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>

// Launches per transform path (fhe_ntt_path_count): evidence for the tests
// and the bench of WHICH kernel ran (FHE_NTT_PATH_* in fhe_sm100.h).
static std::atomic<unsigned long long> g_ntt_path[FHE_NTT_PATHS];
static void path_hit(int p) { g_ntt_path[p].fetch_add(1, std::memory_order_relaxed); }
void ntt_path_hit(int p) {
  if (p >= 0 && p < FHE_NTT_PATHS) path_hit(p);
}
unsigned long long ntt_path_count(int p) {
  return (p >= 0 && p < FHE_NTT_PATHS) ? g_ntt_path[p].load(std::memory_order_relaxed) : 0;
}

namespace {
#include "ntt_tiles.cuh"

// Integer-pipe tiles (a prime >= 2^50) need more registers than the FP64
// tiles' occupancy leaves (64-bit products): their CTAs per SM are capped at
// 3, which removes their 100-180 B spills (config-4 with 60-bit special
// primes: 2140 -> 2254 ops/s; 4 CTAs/SM: 2073).
#ifndef FHE_INT_MINB
#define FHE_INT_MINB 3
#endif
template <class Tile>
constexpr int int_minb() {
  return Tile::MINB < FHE_INT_MINB ? Tile::MINB : FHE_INT_MINB;
}

// Persistent, double-buffered transform kernel over the tiles of one policy.
template <class Tile, bool FWD, bool LAZY, int OUT>
__global__ void __launch_bounds__(Tile::THREADS, int_minb<Tile>())
    ntt_tiles_kernel(const DevChain ch, u64* dst, const u64* src, Tile tl, int ntiles) {
  extern __shared__ __align__(16) u64 smem_raw[];
  // contiguous tile range per CTA (keeps the tile order's twiddle locality)
  const int t_end = (int)(((long)(blockIdx.x + 1) * ntiles) / gridDim.x);
  int t = (int)(((long)blockIdx.x * ntiles) / gridDim.x);
  if (t >= t_end) return;
  Tile cur = tl;
  cur.setup(t);
  if (cur.valid) load_tile(smem_raw, cur, src);
  else cp_async_commit();
  int buf = 0;
  for (; t < t_end; ++t) {
    cp_async_wait_all();
    __syncthreads();
    const int tn = t + 1;
    if (tn < t_end) {
      Tile nxt = tl;
      nxt.setup(tn);
      if (nxt.valid) load_tile(smem_raw + (buf ? 0 : Tile::SMEM_WORDS), nxt, src);
      else cp_async_commit();
    }
    if (cur.valid) {
      if (FWD)
        fwd_passes<Tile::LOG_S, 0, LAZY, OUT>(smem_raw + (buf ? Tile::SMEM_WORDS : 0), cur, dst, ch);
      else
        inv_passes<Tile::LOG_S, npass(Tile::LOG_S) - 1>(smem_raw + (buf ? Tile::SMEM_WORDS : 0), cur,
                                                         dst, ch);
    }
    if (tn < t_end) cur.setup(tn);
    buf ^= 1;
  }
}

// FP64-pipe variant of the persistent tile kernel.  STW: the tile's twiddles
// are staged in shared memory with its data (double-buffered), so every
// butterfly reads its twiddle with an LDS instead of an L1/L2 round trip.
template <class Tile, bool FWD, int IN, int OUT, bool STW>
__global__ void __launch_bounds__(Tile::THREADS, Tile::MINB)
    ntt_tiles_fp_kernel(const DevChain ch, u64* dst, const u64* src, Tile tl, int ntiles) {
  extern __shared__ __align__(16) u64 smem_raw[];
  fhe_pdl_trigger();
  fhe_pdl_wait();
  constexpr int TWM = STW ? Tile::TWMAX : 0;
  double2* tw_raw = reinterpret_cast<double2*>(smem_raw + Tile::NBUF * Tile::SMEM_WORDS);
  // staged tables: [prime][fwd | inv][N]
  const double2* table = STW ? ch.tws + (FWD ? 0 : ch.tws_dir) : nullptr;
  // contiguous tile range per CTA (keeps the tile order's twiddle locality)
  const int t_end = (int)(((long)(blockIdx.x + 1) * ntiles) / gridDim.x);
  int t = (int)(((long)blockIdx.x * ntiles) / gridDim.x);
  if (t >= t_end) return;
  Tile cur = tl;
  if constexpr (Tile::NBUF == 1) {
    // single buffer: the other resident CTAs overlap this one's loads.
    // Round-robin tile order: the CTAs resident at one time work on
    // consecutive tiles (for column tiles: all column blocks of the same
    // rows), so HBM sees whole contiguous k-rows at once instead of scattered
    // 128-byte segments.
#ifdef FHE_NTT_CONTIG_ORDER
    for (; t < t_end; ++t) {
#else
    for (t = blockIdx.x; t < ntiles; t += gridDim.x) {
#endif
      cur.setup(t);
      if (!cur.valid) continue;
      if (STW) load_tw(tw_raw, cur, table + 2 * ch.tws_dir * cur.tw_prime());
      load_tile(smem_raw, cur, src);
      cp_async_wait_all();
      __syncthreads();
      if (FWD)
        fwd_passes_fp<Tile::LOG_S, 0, IN, OUT, STW>(smem_raw, tw_raw, cur, dst, ch);
      else
        inv_passes_fp<Tile::LOG_S, npass(Tile::LOG_S, tile_maxe<Tile>::v) - 1, IN, OUT, STW>(smem_raw, tw_raw, cur,
                                                                          dst, ch);
      __syncthreads();
    }
    return;
  }
  // NBUF-stage ring: the loads of the next NBUF - 1 tiles are in flight
  // while a tile computes (one cp.async group per stage, always committed)
  constexpr int NB = Tile::NBUF;
  auto issue = [&](int tt, int stage) {
    if (tt < t_end) {
      Tile nx = tl;
      nx.setup(tt);
      if (nx.valid) {
        if (STW) load_tw(tw_raw + stage * TWM, nx, table + 2 * ch.tws_dir * nx.tw_prime());
        load_tile(smem_raw + stage * Tile::SMEM_WORDS, nx, src);
        return;
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int j = 0; j < NB - 1; ++j) issue(t + j, j);
  for (int k = 0; t + k < t_end; ++k) {
    cp_async_wait_group<NB - 2>();
    __syncthreads();
    issue(t + k + NB - 1, (k + NB - 1) % NB);
    cur = tl;
    cur.setup(t + k);
    if (cur.valid) {
      const int stage = k % NB;
      u64* sm = smem_raw + stage * Tile::SMEM_WORDS;
      const double2* tws = tw_raw + stage * TWM;
      if (FWD)
        fwd_passes_fp<Tile::LOG_S, 0, IN, OUT, STW>(sm, tws, cur, dst, ch);
      else
        inv_passes_fp<Tile::LOG_S, npass(Tile::LOG_S, tile_maxe<Tile>::v) - 1, IN, OUT, STW>(sm, tws, cur, dst, ch);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA column tiles (FP64 path, N1 = 256): the [256 k-rows x 16 columns] tile
// (32 KB, one 128-byte segment per k-row) moves with ONE bulk tensor copy in
// each direction, issued by one thread and completed on an mbarrier; the
// twiddle block follows with a 1D bulk copy on the same barrier.  Lanes run
// across the 16 columns of a k-row, so the dense (unpadded) layout is
// bank-conflict free in both passes.
#include "ntt_tma_ptx.cuh"


// Column tile moved by TMA.  Rows are addressed as the 5D tensor
// (16 elements, N2/16 column blocks, N1 k-rows, limbs, batches) so both the
// contiguous and the batch-strided row layouts map to one box.
template <int LOG_N, int LOG_N1>
struct ColsTmaTile : ColsTile<LOG_N, LOG_N1> {
  using Base = ColsTile<LOG_N, LOG_N1>;
  static constexpr int TMA_STAGES = FHE_TMA_STAGES;
  static constexpr int MINB = FHE_TMA_COLS_MINB;
  static constexpr bool DENSE = true;
  static constexpr bool TMA = true;
  static constexpr int SMEM_WORDS = Base::TILE;
  __device__ static __forceinline__ int pad(int t) { return t; }
  const CUtensorMap* smap_p = nullptr;  // the kernel's __grid_constant__ maps
  const CUtensorMap* dmap_p = nullptr;
  int ccol = 0, climb = 0, cbat = 0;  // box coordinates of the tile
  bool bcast = false;  // source map holds one row per batch item (NttArgs::bcast_src)
  __device__ __forceinline__ void setup(int t) {
    Base::setup(t);
    ccol = this->j0 >> 4;
    climb = this->row % this->map.limbs;
    cbat = this->row / this->map.limbs;
  }
  uint64_t ld_pol = 0, st_pol = 0;  // L2 cache-hint policies (0: no hint)
  __device__ __forceinline__ void tma_load(u64* sm, uint64_t* bar) const {
    const int sl = bcast ? 0 : climb;
    if (ld_pol) tma_load_5d_hint(sm, smap_p, 0, ccol, 0, sl, cbat, bar, ld_pol);
    else tma_load_5d(sm, smap_p, 0, ccol, 0, sl, cbat, bar);
  }
  __device__ __forceinline__ void tma_store(const u64* sm) const {
    if (st_pol) tma_store_5d_hint(dmap_p, 0, ccol, 0, climb, cbat, sm, st_pol);
    else tma_store_5d(dmap_p, 0, ccol, 0, climb, cbat, sm);
  }
};

// Chunk tile moved by TMA with the 128B swizzle: R rows of one residue class
// x C chunks as the box (16 elements, 16 C row segments, 1 limb, R batches)
// of the 4D view (16, N/16, limbs, batches).  The swizzle keeps both the
// stride-16 and the contiguous register passes bank-conflict free without
// padding (run_pass_fp's SWZ addressing).
template <int LOG_N, int LOG_N1>
struct ChunksTmaTile : ChunksTile<LOG_N, LOG_N1> {
  using Base = ChunksTile<LOG_N, LOG_N1>;
  static constexpr int TMA_STAGES = FHE_TMA_STAGES;
  static constexpr int MINB = FHE_TMA_CHUNK_MINB;
  static constexpr bool DENSE = true;
  static constexpr bool TMA = true;
  static constexpr bool SWZ = true;
  static constexpr int SMEM_WORDS = Base::TILE;
  __device__ static __forceinline__ int pad(int t) { return t ^ ((t >> 3) & 14); }
  const CUtensorMap* smap_p = nullptr;
  const CUtensorMap* dmap_p = nullptr;
  bool has_fin = false;
  NttFinish fin{};
  uint64_t ld_pol = 0, st_pol = 0;  // L2 cache-hint policies (0: no hint)
  __device__ __forceinline__ void tma_load(u64* sm, uint64_t* bar) const {
    if (ld_pol)
      tma_load_4d_hint(sm, smap_p, 0, this->c0 << (Base::LOG_S - 4), this->cls_, this->i0_, bar,
                       ld_pol);
    else
      tma_load_4d(sm, smap_p, 0, this->c0 << (Base::LOG_S - 4), this->cls_, this->i0_, bar);
  }
  // ModDown finish from the swizzled result tile, 16 bytes per step: every
  // element is read once from smem, accQ and the add-in once from HBM, and
  // the output written once (no transform store, no separate finish pass)
  __device__ __forceinline__ void finish_store(const u64* sm, const DevChain& ch) const {
    constexpr int S = 1 << Base::LOG_S;
    const int lc = this->log_c;
    const int arrays = this->nb;
    for (int q = threadIdx.x; q < (arrays * S) >> 1; q += Base::THREADS) {
      const int b = q / (S >> 1), k = (q % (S >> 1)) << 1;
      const int t = b * S + k;
      const ulonglong2 x = *reinterpret_cast<const ulonglong2*>(&sm[t ^ ((t >> 3) & 14)]);
      const int i = b >> lc, c = b & ((1 << lc) - 1);
      const int row = this->cls_ + (this->i0_ + i) * this->map.limbs;  // conv row
      const long col = ((long)(this->c0 + c) << Base::LOG_S) + k;
      const int j = row % fin.level;
      const int bp = row / fin.level;  // b * 2 + poly
      const int bb = bp >> 1, poly = bp & 1;
      const u64 qj = ch.mc[j].q;
      const WPair pi = fin.p_inv[j];
      const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(fin.accQ + ((long)row << ch.log_n) + col);
      u64 v0 = shoup_mul(sub_mod(a.x, x.x, qj), pi.w, pi.sh, qj);
      u64 v1 = shoup_mul(sub_mod(a.y, x.y, qj), pi.w, pi.sh, qj);
      const u64* add = poly ? fin.add1 : fin.add0;
      const long w = ((long)j << ch.log_n) + col;
      if (add) {
        const ulonglong2 d = *reinterpret_cast<const ulonglong2*>(add + bb * fin.add_stride + w);
        v0 = add_mod(d.x, v0, qj);
        v1 = add_mod(d.y, v1, qj);
      }
      u64* out = poly ? fin.out1 : fin.out0;
      *reinterpret_cast<ulonglong2*>(out + bb * fin.out_stride + w) = make_ulonglong2(v0, v1);
    }
  }
  __device__ __forceinline__ void tma_store(const u64* sm) const {
    if (st_pol)
      tma_store_4d_hint(dmap_p, 0, this->c0 << (Base::LOG_S - 4), this->cls_, this->i0_, sm,
                        st_pol);
    else
      tma_store_4d(dmap_p, 0, this->c0 << (Base::LOG_S - 4), this->cls_, this->i0_, sm);
  }
};

template <class Tile, bool FWD, int IN, int OUT>
__global__ void __launch_bounds__(Tile::THREADS, Tile::MINB)
    ntt_tma_kernel(const DevChain ch, const __grid_constant__ CUtensorMap smap,
                   const __grid_constant__ CUtensorMap dmap, Tile tl, int ntiles) {
  // dynamic smem only (no static smem ahead of it): the TMA boxes land at
  // 1024-byte aligned stage bases; twiddles and mbarriers follow the data.
  // NB stages: thread 0 keeps the next NB - 1 tiles' loads in flight.
  constexpr int NB = Tile::TMA_STAGES;
  extern __shared__ __align__(1024) u64 tma_smem[];
  double2* tws0 = reinterpret_cast<double2*>(tma_smem + NB * Tile::SMEM_WORDS);
  uint64_t* bars = reinterpret_cast<uint64_t*>(tws0 + NB * Tile::TWMAX);
  const double2* table = ch.tws + (FWD ? 0 : ch.tws_dir);
  constexpr unsigned kDataBytes = Tile::SMEM_WORDS * sizeof(u64);
  if (threadIdx.x == 0) {
    for (int i = 0; i < NB; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  Tile cur = tl;
  cur.smap_p = &smap;
  cur.dmap_p = &dmap;
  // thread 0: issue tile `tt` into stage `s` (invalid / past-the-end: nothing)
  auto issue = [&](int tt, int s) {
    if (tt >= ntiles) return;
    Tile nx = tl;
    nx.smap_p = &smap;
    nx.setup(tt);
    if (!nx.valid) return;
    const unsigned tw_bytes = nx.tw_pairs() * sizeof(double2);
    mbar_expect_tx(&bars[s], kDataBytes + tw_bytes);
    nx.tma_load(tma_smem + s * Tile::SMEM_WORDS, &bars[s]);
    bulk_g2s(tws0 + s * Tile::TWMAX, table + 2 * ch.tws_dir * nx.tw_prime() + nx.tw_src_off(),
             tw_bytes, &bars[s]);
  };
  const int stride = gridDim.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < NB - 1; ++s) issue(blockIdx.x + s * stride, s);
  unsigned phases = 0;  // bit s: parity of stage s
  int k = 0;
  for (int t = blockIdx.x; t < ntiles; t += stride, ++k) {
    const int s = k % NB;
    if (threadIdx.x == 0) {
      // the stage refilled now was last used by tile k - 1: its store must
      // have left shared memory first
      bulk_wait_read0();
      issue(t + (NB - 1) * stride, (k + NB - 1) % NB);
    }
    cur.setup(t);
    if (!cur.valid) continue;
    mbar_wait(&bars[s], (phases >> s) & 1);
    phases ^= 1u << s;
    u64* sm = tma_smem + s * Tile::SMEM_WORDS;
    const double2* tws = tws0 + s * Tile::TWMAX;
    if (FWD)
      fwd_passes_fp<Tile::LOG_S, 0, IN, OUT, true>(sm, tws, cur, nullptr, ch);
    else
      inv_passes_fp<Tile::LOG_S, npass(Tile::LOG_S, tile_maxe<Tile>::v) - 1, IN, OUT, true>(sm, tws, cur, nullptr,
                                                                        ch);
    __syncthreads();
  }
  if (threadIdx.x == 0) bulk_wait0();
}

// ---------------------------------------------------------------------------
// Fused four-step transform (FP64 path): one persistent kernel runs both the
// column and the chunk tiles, so the intermediate never goes back to HBM --
// it is written to and re-read from the 126 MB L2 a few microseconds later.
//
// Rows are grouped like the chunk tiles (R rows of one residue class).  Tiles
// are handed out in ticket order; ticket block b holds the first-phase tiles
// of group b (column tiles forward, chunk tiles inverse) followed by the
// second-phase tiles of group b - kFuseLag.  A second-phase tile waits until
// every first-phase tile of its group has signalled its counter.  Tickets
// are taken by resident CTAs only and a CTA only ever waits on tickets issued
// before its own, so the wait cannot deadlock.
#ifndef FHE_FUSE_MAX_LOG_R
#define FHE_FUSE_MAX_LOG_R 4
#endif
#ifndef FHE_FUSE_MIN_LOG_R
#define FHE_FUSE_MIN_LOG_R 3
#endif
#ifndef FHE_FUSE_LAG
#define FHE_FUSE_LAG 16
#endif
constexpr int kFuseLag = FHE_FUSE_LAG;
#ifndef FHE_FUSE_L2HINT
#define FHE_FUSE_L2HINT 0
#endif
#ifndef FHE_FUSE_LAG_ROWS
#define FHE_FUSE_LAG_ROWS 0
#endif
#ifndef FHE_FUSE_CTAS
#define FHE_FUSE_CTAS 5
#endif
constexpr int kFuseSlabs = 8;

struct FusePlan {
  int groups;     // row groups (residue class x row block)
  int rblocks;    // row blocks per class
  int log_r;      // rows per group = 1 << log_r
  int c_per_g;    // column tiles per group = R * C::TILES
  int k_per_g;    // chunk tiles per group = cblocks
  int total;      // tickets
  int lag;        // second phase trails the first by this many groups
  FastDiv blk_div;    // ticket -> block (block = c_per_g + k_per_g tickets)
  FastDiv rb_div;     // group -> (class, row block)
};

struct FuseScratch {
  std::mutex mu;
  int* dev = nullptr;      // kFuseSlabs x slab_ints
  size_t slab_ints = 0;
  int next = 0;
  cudaEvent_t ev[kFuseSlabs] = {};
};

template <bool FWD, class Tile>
__device__ __forceinline__ void fused_run_tile(const DevChain& ch, Tile& tl, u64* sm,
                                               double2* tws, const double2* table, u64* dst,
                                               const u64* src) {
  load_tw(tws, tl, table + 2 * ch.tws_dir * tl.tw_prime());
  load_tile(sm, tl, src);
  cp_async_wait_all();
  __syncthreads();
  if constexpr (FWD)
    fwd_passes_fp<Tile::LOG_S, 0, Tile::COLS ? FPIN_U64 : FPIN_DOUBLE,
                  Tile::COLS ? FPOUT_DOUBLE : FPOUT_U64, true>(sm, tws, tl, dst, ch);
  else
    inv_passes_fp<Tile::LOG_S, npass(Tile::LOG_S, tile_maxe<Tile>::v) - 1, Tile::COLS ? FPIN_DOUBLE : FPIN_U64,
                  Tile::COLS ? FPOUT_U64 : FPOUT_DOUBLE, true>(sm, tws, tl, dst, ch);
  __syncthreads();
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <class CT, class KT, bool FWD>
__global__ void __launch_bounds__(kSplitThreads, kSplitMinB)
    ntt_fused_fp_kernel(const DevChain ch, u64* dst, const u64* src, CT ct, KT kt, FusePlan fp,
                        int* ctr) {
  extern __shared__ __align__(16) u64 smem_raw[];
  __shared__ int s_tk[2];
  constexpr int SW = CT::SMEM_WORDS > KT::SMEM_WORDS ? CT::SMEM_WORDS : KT::SMEM_WORDS;
  double2* tws = reinterpret_cast<double2*>(smem_raw + SW);
  const double2* table = ch.tws + (FWD ? 0 : ch.tws_dir);
  const int per_block = fp.c_per_g + fp.k_per_g;
  const int first_n = FWD ? fp.c_per_g : fp.k_per_g;
  if (threadIdx.x == 0) s_tk[0] = atomicAdd(&ctr[0], 1);
  __syncthreads();
  for (int cur = 0;; cur ^= 1) {
    const int t = s_tk[cur];
    if (t >= fp.total) break;
    // the next ticket is fetched while this tile runs (published by the
    // barrier at the end of the iteration)
    if (threadIdx.x == 0) s_tk[cur ^ 1] = atomicAdd(&ctr[0], 1);
    const int blk = fp.blk_div.div(t);
    const int r = t - blk * per_block;
    const bool first = r < first_n;
    const int g = first ? blk : blk - fp.lag;
    if (g >= 0 && g < fp.groups) {
      const int cls = fp.rb_div.div(g);
      const int rb = g - cls * fp.rblocks;
      const bool col_tile = (first == FWD);
      const int idx = first ? r : r - first_n;  // tile index within the group's phase
      if (!first) {
        // wait for the group's first phase (written through L2 by other CTAs)
        if (threadIdx.x == 0) {
          const int target = FWD ? fp.c_per_g : fp.k_per_g;
          while (ld_acquire(&ctr[1 + g]) < target) __nanosleep(128);
        }
        __syncthreads();
      }
      if (col_tile) {
        const int i = idx / CT::TILES, jb = idx - i * CT::TILES;
        const int row = cls + ((rb << fp.log_r) + i) * ct.map.limbs;
        if (row < ct.rows) {
          CT c = ct;
          c.setup(row * CT::TILES + jb);
          fused_run_tile<FWD>(ch, c, smem_raw, tws, table, dst, FWD ? src : dst);
        }
      } else {
        KT k = kt;
        k.setup(g * fp.k_per_g + idx);
        if (k.valid) fused_run_tile<FWD>(ch, k, smem_raw, tws, table, dst, FWD ? dst : src);
      }
      if (first) {
        __syncthreads();
        if (threadIdx.x == 0) red_release_add(&ctr[1 + g], 1);
      }
    }
    __syncthreads();
  }
}

// Fused four-step transform on TMA tiles: the ticketed persistent scheme of
// ntt_fused_fp_kernel with both tile kinds moved by bulk tensor copies.  A
// first-phase tile signals its group only after its TMA store has completed
// (cp.async.bulk.wait_group 0, then a release add); a second-phase tile
// acquires the counter and orders its TMA load after it with a proxy fence.
// The signal of a CTA's last first-phase tile is flushed before the CTA
// waits on anything, so no CTA can wait on its own pending signal.
template <class CT, class KT, bool FWD>
__global__ void __launch_bounds__(kSplitThreads, FHE_FUSE_CTAS)
    ntt_fused_tma_kernel(const DevChain ch, const __grid_constant__ CUtensorMap cs_map,
                         const __grid_constant__ CUtensorMap cd_map,
                         const __grid_constant__ CUtensorMap ks_map,
                         const __grid_constant__ CUtensorMap kd_map, CT ct, KT kt, FusePlan fp,
                         int* ctr) {
  extern __shared__ __align__(1024) u64 fused_tma_smem[];
  u64* sm = fused_tma_smem;
  constexpr int SW = CT::SMEM_WORDS > KT::SMEM_WORDS ? CT::SMEM_WORDS : KT::SMEM_WORDS;
  constexpr int TW = CT::TWMAX > KT::TWMAX ? CT::TWMAX : KT::TWMAX;
  double2* tws = reinterpret_cast<double2*>(sm + SW);
  uint64_t* bar = reinterpret_cast<uint64_t*>(tws + TW);
  int* s_tk = reinterpret_cast<int*>(bar + 1);
  const double2* table = ch.tws + (FWD ? 0 : ch.tws_dir);
  constexpr unsigned kDataBytes = SW * sizeof(u64);
  const int per_block = fp.c_per_g + fp.k_per_g;
  const int first_n = FWD ? fp.c_per_g : fp.k_per_g;
  int pending = -1;  // group whose counter this CTA still owes (thread 0)
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_tk[0] = atomicAdd(&ctr[0], 1);
  }
  __syncthreads();
  unsigned phase = 0;
  // L2 priorities (FHE_FUSE_L2HINT): bit 0 -> loads evict_first (inputs and
  // the intermediate are read once), bit 1 -> first-phase stores evict_last
  // (the intermediate is re-read by the second phase a few groups later),
  // bit 2 -> second-phase loads (of the intermediate) evict_first
  const uint64_t pol_ld = (FHE_FUSE_L2HINT & 1) ? l2_policy_evict_first() : 0;
  const uint64_t pol_mid = (FHE_FUSE_L2HINT & 2) ? l2_policy_evict_last() : 0;
  const uint64_t pol_ld2 = (FHE_FUSE_L2HINT & 4) ? l2_policy_evict_first() : pol_ld;
  // bit 4 -> second-phase (final) stores evict_first
  const uint64_t pol_out = (FHE_FUSE_L2HINT & 16) ? l2_policy_evict_first() : 0;
  for (int cur = 0;; cur ^= 1) {
    const int t = s_tk[cur];
    if (t >= fp.total) break;
    if (threadIdx.x == 0) {
      s_tk[cur ^ 1] = atomicAdd(&ctr[0], 1);
      // previous tile's store: complete (and signalled) before anything else
      bulk_wait0();
      if (pending >= 0) {
        red_release_add(&ctr[1 + pending], 1);
        pending = -1;
      }
    }
    const int blk = fp.blk_div.div(t);
    const int r = t - blk * per_block;
    const bool first = r < first_n;
    const int g = first ? blk : blk - fp.lag;
    bool work = false;
    if (g >= 0 && g < fp.groups) {
      const int cls = fp.rb_div.div(g);
      const int rb = g - cls * fp.rblocks;
      const bool col_tile = (first == FWD);
      const int idx = first ? r : r - first_n;
      if (threadIdx.x == 0 && !first) {
        const int target = FWD ? fp.c_per_g : fp.k_per_g;
        while (ld_acquire(&ctr[1 + g]) < target) __nanosleep(128);
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      if (col_tile) {
        const int i = idx / CT::TILES, jb = idx - i * CT::TILES;
        const int row = cls + ((rb << fp.log_r) + i) * ct.map.limbs;
        if (row < ct.rows) {
          CT c = ct;
          c.smap_p = &cs_map;
          c.dmap_p = &cd_map;
          c.ld_pol = first ? pol_ld : pol_ld2;
          c.st_pol = first ? pol_mid : pol_out;
          c.setup(row * CT::TILES + jb);
          if (threadIdx.x == 0) {
            const unsigned twb = c.tw_pairs() * sizeof(double2);
            mbar_expect_tx(bar, kDataBytes + twb);
            c.tma_load(sm, bar);
            bulk_g2s(tws, table + 2 * ch.tws_dir * c.tw_prime() + c.tw_src_off(), twb, bar);
          }
          mbar_wait(bar, phase);
          phase ^= 1;
          if (FWD)
            fwd_passes_fp<CT::LOG_S, 0, FPIN_U64, FPOUT_DOUBLE, true>(sm, tws, c, nullptr, ch);
          else
            inv_passes_fp<CT::LOG_S, npass(CT::LOG_S, tile_maxe<CT>::v) - 1, FPIN_DOUBLE, FPOUT_U64, true>(
                sm, tws, c, nullptr, ch);
          work = true;
        }
      } else {
        KT k = kt;
        k.smap_p = &ks_map;
        k.dmap_p = &kd_map;
        k.ld_pol = first ? pol_ld : pol_ld2;
        k.st_pol = first ? pol_mid : pol_out;
        k.setup(g * fp.k_per_g + idx);
        if (k.valid) {
          if (threadIdx.x == 0) {
            const unsigned twb = k.tw_pairs() * sizeof(double2);
            mbar_expect_tx(bar, kDataBytes + twb);
            k.tma_load(sm, bar);
            bulk_g2s(tws, table + 2 * ch.tws_dir * k.tw_prime() + k.tw_src_off(), twb, bar);
          }
          mbar_wait(bar, phase);
          phase ^= 1;
          if (FWD)
            fwd_passes_fp<KT::LOG_S, 0, FPIN_DOUBLE, FPOUT_U64, true>(sm, tws, k, nullptr, ch);
          else
            inv_passes_fp<KT::LOG_S, npass(KT::LOG_S, tile_maxe<KT>::v) - 1, FPIN_U64, FPOUT_DOUBLE, true>(
                sm, tws, k, nullptr, ch);
          work = true;
        }
      }
      if (first && threadIdx.x == 0) {
        if (work) pending = g;  // signalled once the store has completed
        else red_release_add(&ctr[1 + g], 1);
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    bulk_wait0();
    if (pending >= 0) red_release_add(&ctr[1 + pending], 1);
  }
}

int g_sm_count = 0;
int sm_count() {
  if (!g_sm_count) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sm_count, cudaDevAttrMultiProcessorCount, dev);
    if (g_sm_count <= 0) g_sm_count = 148;
  }
  return g_sm_count;
}

template <class Tile, bool FWD, bool LAZY, int OUT>
int launch_tiles(const DevChain& ch, u64* dst, const u64* src, const Tile& tl, int ntiles,
                 cudaStream_t st) {
  if (ntiles <= 0) return 0;
  const int grid = std::min(ntiles, int_minb<Tile>() * sm_count());
  constexpr int smem = 2 * Tile::SMEM_WORDS * sizeof(u64);
  static bool attr = false;  // once per instantiation
  if (!attr) {
    cudaFuncSetAttribute(ntt_tiles_kernel<Tile, FWD, LAZY, OUT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  ntt_tiles_kernel<Tile, FWD, LAZY, OUT><<<grid, Tile::THREADS, smem, st>>>(ch, dst, src, tl,
                                                                           ntiles);
  FHE_LAUNCH_CHECK();
  return 0;
}


template <class Tile, bool FWD, int IN, int OUT, bool STW = false>
int launch_tiles_fp(const DevChain& ch, u64* dst, const u64* src, const Tile& tl, int ntiles,
                    cudaStream_t st) {
  if (ntiles <= 0) return 0;
  const int grid = std::min(ntiles, Tile::MINB * sm_count());
  constexpr int smem = Tile::NBUF * (Tile::SMEM_WORDS * sizeof(u64) +
                                     (STW ? Tile::TWMAX * sizeof(double2) : 0));
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ntt_tiles_fp_kernel<Tile, FWD, IN, OUT, STW>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  fhe_launch(ntt_tiles_fp_kernel<Tile, FWD, IN, OUT, STW>, dim3(grid), dim3(Tile::THREADS), smem,
             st, ch, dst, src, tl, ntiles);
  FHE_LAUNCH_CHECK();
  return 0;
}

// Counters of one fused launch: a slab of the chain's scratch, zeroed on the
// stream after the slab's previous user (any stream) has finished.
int* fuse_slab(const DevChain& ch, size_t need, cudaStream_t st, int& slab) {
  FuseScratch* fs = static_cast<FuseScratch*>(ch.fuse);
  std::lock_guard<std::mutex> lock(fs->mu);
  if (fs->slab_ints < need) {
    if (fs->dev) {
      if (cudaDeviceSynchronize() != cudaSuccess || cudaFree(fs->dev) != cudaSuccess) return nullptr;
      fs->dev = nullptr;
    }
    const size_t ints = std::max<size_t>(need, 4096);
    if (cudaMalloc(&fs->dev, ints * kFuseSlabs * sizeof(int)) != cudaSuccess) return nullptr;
    fs->slab_ints = ints;
  }
  slab = fs->next;
  fs->next = (fs->next + 1) % kFuseSlabs;
  if (!fs->ev[slab] && cudaEventCreateWithFlags(&fs->ev[slab], cudaEventDisableTiming) != cudaSuccess)
    return nullptr;
  if (cudaStreamWaitEvent(st, fs->ev[slab], 0) != cudaSuccess) return nullptr;
  int* ctr = fs->dev + (size_t)slab * fs->slab_ints;
  if (cudaMemsetAsync(ctr, 0, need * sizeof(int), st) != cudaSuccess) return nullptr;
  return ctr;
}

int fuse_release(const DevChain& ch, int slab, cudaStream_t st) {
  FuseScratch* fs = static_cast<FuseScratch*>(ch.fuse);
  std::lock_guard<std::mutex> lock(fs->mu);
  FHE_CUDA_CHECK(cudaEventRecord(fs->ev[slab], st));
  return 0;
}

template <class K>
FusePlan make_fuse_plan(const K& kt, int cols_tiles_per_row, int rows, int limbs) {
  FusePlan fp;
  fp.log_r = kt.log_r;
  fp.rblocks = kt.rblocks;
  fp.groups = std::min(limbs, rows) * kt.rblocks;
  fp.c_per_g = (1 << kt.log_r) * cols_tiles_per_row;
  fp.k_per_g = kt.cblocks;
  // FHE_FUSE_LAG_ROWS > 0: the lag is a fixed number of rows (a fixed
  // intermediate window) instead of a fixed number of groups
  fp.lag = FHE_FUSE_LAG_ROWS > 0 ? std::max(2, FHE_FUSE_LAG_ROWS >> kt.log_r) : kFuseLag;
  fp.total = (fp.groups + fp.lag) * (fp.c_per_g + fp.k_per_g);
  fp.blk_div.init(fp.c_per_g + fp.k_per_g);
  fp.rb_div.init(kt.rblocks);
  return fp;
}

template <class C, class K>
int launch_fused(const DevChain& ch, u64* dst, const u64* src, const C& ct, const K& kt,
                 bool fwd, int rows, int limbs, cudaStream_t st) {
  const FusePlan fp = make_fuse_plan(kt, C::TILES, rows, limbs);
  int slab = 0;
  int* ctr = fuse_slab(ch, 1 + (size_t)fp.groups, st, slab);
  if (!ctr) {
    fhe_set_error("fused NTT scratch setup failed");
    return -2;
  }
  constexpr int SW = C::SMEM_WORDS > K::SMEM_WORDS ? C::SMEM_WORDS : K::SMEM_WORDS;
  constexpr int TW = C::TWMAX > K::TWMAX ? C::TWMAX : K::TWMAX;
  constexpr int smem = SW * sizeof(u64) + TW * sizeof(double2);
  const int grid = std::min(fp.total, kSplitMinB * sm_count());
  if (fwd) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(ntt_fused_fp_kernel<C, K, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    ntt_fused_fp_kernel<C, K, true><<<grid, kSplitThreads, smem, st>>>(ch, dst, src, ct, kt, fp,
                                                                      ctr);
  } else {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(ntt_fused_fp_kernel<C, K, false>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    ntt_fused_fp_kernel<C, K, false><<<grid, kSplitThreads, smem, st>>>(ch, dst, src, ct, kt, fp,
                                                                       ctr);
  }
  FHE_LAUNCH_CHECK();
  return fuse_release(ch, slab, st);
}

bool fused_tma_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_NTT_FUSED_TMA");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

bool fused_enabled() {
  static int on = -1;
  if (on < 0) {
    // opt-in: measured on par with the two-kernel path (the tile machinery,
    // not DRAM, bounds both; profiles/r1_ntt_notes.md)
    const char* e = getenv("FHE_NTT_FUSED");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// libcuda link dependency); null when unavailable.
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

bool tma_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_NTT_TMA");
    on = (e && e[0] == '0') ? 0 : (encode_tiled() ? 1 : 0);
  }
  return on == 1;
}

// Column-tile view of a row set: (16 elements, N2/16 blocks, N1 k-rows,
// limbs, batches); row r = batch r / limbs, limb r % limbs.
bool cols_tensor_map(CUtensorMap* m, const u64* base, int log_n, int log_n1, int limbs,
                     long bstride, int rows) {
  const cuuint64_t n = 1ull << log_n, n1 = 1ull << log_n1, n2 = n / n1;
  const cuuint64_t bs = bstride ? (cuuint64_t)bstride : (cuuint64_t)limbs * n;
  const cuuint64_t nb = ((cuuint64_t)rows + limbs - 1) / limbs;
  const cuuint64_t dims[5] = {16, n2 / 16, n1, (cuuint64_t)limbs, nb};
  const cuuint64_t strides[4] = {128, n2 * 8, n * 8, bs * 8};
  const cuuint32_t box[5] = {16, 1, (cuuint32_t)n1, 1, 1};
  const cuuint32_t es[5] = {1, 1, 1, 1, 1};
  return encode_tiled()(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 5, const_cast<u64*>(base), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Chunk-tile view: (16 elements, N/16 row segments, limbs, batches) with the
// 128B swizzle; box = (16, 16 C, 1, R).
bool chunks_tensor_map(CUtensorMap* m, const u64* base, int log_n, int log_s, int limbs,
                       long bstride, int rows, int log_r, int log_c) {
  const cuuint64_t n = 1ull << log_n;
  const cuuint64_t bs = bstride ? (cuuint64_t)bstride : (cuuint64_t)limbs * n;
  const cuuint64_t nb = ((cuuint64_t)rows + limbs - 1) / limbs;
  const cuuint64_t dims[4] = {16, n / 16, (cuuint64_t)limbs, nb};
  const cuuint64_t strides[3] = {128, n * 8, bs * 8};
  const cuuint32_t box[4] = {16, (cuuint32_t)(1u << (log_s - 4 + log_c)), 1, 1u << log_r};
  const cuuint32_t es[4] = {1, 1, 1, 1};
  return encode_tiled()(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<u64*>(base), dims,
                        strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#include "ntt_cluster.cuh"
#include "ntt_row_cluster.cuh"

template <class Tile, bool FWD, int IN, int OUT>
int launch_chunks_tma(const DevChain& ch, u64* dst, const u64* src, const Tile& tl, int ntiles,
                      long src_bstride, long dst_bstride, cudaStream_t st, bool& done) {
  done = false;
  const int log_c = kChunkLogTile - Tile::LOG_S - tl.log_r;
  CUtensorMap smap, dmap;
  if (!chunks_tensor_map(&smap, src, ch.log_n, Tile::LOG_S, tl.map.limbs, src_bstride, tl.rows,
                         tl.log_r, log_c) ||
      !chunks_tensor_map(&dmap, dst, ch.log_n, Tile::LOG_S, tl.map.limbs, dst_bstride, tl.rows,
                         tl.log_r, log_c))
    return 0;
  constexpr int smem =
      Tile::TMA_STAGES * (Tile::SMEM_WORDS * sizeof(u64) + Tile::TWMAX * sizeof(double2) + 8);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ntt_tma_kernel<Tile, FWD, IN, OUT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int grid = std::min(ntiles, Tile::MINB * sm_count());
  ntt_tma_kernel<Tile, FWD, IN, OUT><<<grid, Tile::THREADS, smem, st>>>(ch, smap, dmap, tl,
                                                                        ntiles);
  FHE_LAUNCH_CHECK();
  done = true;
  return 0;
}

template <class CT, class KT>
int launch_fused_tma(const DevChain& ch, u64* dst, const u64* src, const CT& ct, const KT& kt,
                     bool fwd, long src_bstride, long dst_bstride, int rows, int limbs,
                     cudaStream_t st, bool& done, bool bcast = false) {
  done = false;
#if FHE_FUSE_L2HINT & 8
  // experiment: a persisting L2 carve-out, so the evict_last policy of the
  // intermediate stores has lines to keep
  static bool l2set = false;
  if (!l2set) {
    int dev = 0, mx = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)mx);
    if (getenv("FHE_NTT_CLUSTER_DEBUG")) fprintf(stderr, "persisting L2 %d bytes\n", mx);
    cudaGetLastError();
    l2set = true;
  }
#endif
  const int log_c = kChunkLogTile - KT::LOG_S - kt.log_r;
  // forward: columns read src, chunks work in place on dst; inverse: chunks
  // read src, columns work in place on dst.  bcast (forward): src holds one
  // row per batch item (src_bstride apart), read by every limb of the item
  CUtensorMap cs, cd, ks, kd;
  const u64* col_src = fwd ? src : dst;
  const u64* chk_src = fwd ? dst : src;
  const long col_sb = fwd ? src_bstride : dst_bstride, chk_sb = fwd ? dst_bstride : src_bstride;
  const bool col_ok = bcast ? cols_tensor_map(&cs, col_src, ch.log_n, CT::LOG_S, 1, col_sb,
                                              (rows + limbs - 1) / limbs)
                            : cols_tensor_map(&cs, col_src, ch.log_n, CT::LOG_S, limbs, col_sb, rows);
  if (!col_ok ||
      !cols_tensor_map(&cd, dst, ch.log_n, CT::LOG_S, limbs, dst_bstride, rows) ||
      !chunks_tensor_map(&ks, chk_src, ch.log_n, KT::LOG_S, limbs, chk_sb, rows, kt.log_r, log_c) ||
      !chunks_tensor_map(&kd, dst, ch.log_n, KT::LOG_S, limbs, dst_bstride, rows, kt.log_r, log_c))
    return 0;
  const FusePlan fp = make_fuse_plan(kt, CT::TILES, rows, limbs);
  int slab = 0;
  int* ctr = fuse_slab(ch, 1 + (size_t)fp.groups, st, slab);
  if (!ctr) {
    fhe_set_error("fused NTT scratch setup failed");
    return -2;
  }
  constexpr int SW = CT::SMEM_WORDS > KT::SMEM_WORDS ? CT::SMEM_WORDS : KT::SMEM_WORDS;
  constexpr int TW = CT::TWMAX > KT::TWMAX ? CT::TWMAX : KT::TWMAX;
  constexpr int smem = SW * sizeof(u64) + TW * sizeof(double2) + 16;
  const int grid = std::min(fp.total, FHE_FUSE_CTAS * sm_count());
  auto go = [&](auto kern) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      attr = true;
    }
    kern<<<grid, kSplitThreads, smem, st>>>(ch, cs, cd, ks, kd, ct, kt, fp, ctr);
  };
  if (fwd)
    go(ntt_fused_tma_kernel<CT, KT, true>);
  else
    go(ntt_fused_tma_kernel<CT, KT, false>);
  FHE_LAUNCH_CHECK();
  done = true;
  return fuse_release(ch, slab, st);
}

template <int LOG_N, int LOG_N1, bool FWD, int IN, int OUT, class K>
int maybe_chunks_tma(const DevChain& ch, u64* dst, const u64* src, const K& kt, int nk,
                     long src_bstride, long dst_bstride, cudaStream_t st, bool& done,
                     const NttFinish* fin = nullptr) {
  done = false;
  if constexpr (LOG_N - LOG_N1 == 8) {
    using KT = ChunksTmaTile<LOG_N, LOG_N1>;
    KT tk;
    static_cast<K&>(tk) = kt;
    if (fin) {
      tk.has_fin = true;
      tk.fin = *fin;
    }
    return launch_chunks_tma<KT, FWD, IN, OUT>(ch, dst, src, tk, nk, src_bstride, dst_bstride, st,
                                               done);
  }
  return 0;
}

template <class Tile, bool FWD, int IN, int OUT>
int launch_cols_tma(const DevChain& ch, u64* dst, const u64* src, const Tile& tl, int ntiles,
                    long src_bstride, long dst_bstride, cudaStream_t st, bool& done) {
  done = false;
  CUtensorMap smap, dmap;
  const bool src_ok =
      tl.bcast ? cols_tensor_map(&smap, src, ch.log_n, Tile::LOG_S, 1, src_bstride,
                                 (tl.rows + tl.map.limbs - 1) / tl.map.limbs)
               : cols_tensor_map(&smap, src, ch.log_n, Tile::LOG_S, tl.map.limbs, src_bstride,
                                 tl.rows);
  if (!src_ok ||
      !cols_tensor_map(&dmap, dst, ch.log_n, Tile::LOG_S, tl.map.limbs, dst_bstride, tl.rows))
    return 0;  // fall back to the cp.async path
  constexpr int smem =
      Tile::TMA_STAGES * (Tile::SMEM_WORDS * sizeof(u64) + Tile::TWMAX * sizeof(double2) + 8);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ntt_tma_kernel<Tile, FWD, IN, OUT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int grid = std::min(ntiles, Tile::MINB * sm_count());
  ntt_tma_kernel<Tile, FWD, IN, OUT><<<grid, Tile::THREADS, smem, st>>>(ch, smap, dmap, tl,
                                                                             ntiles);
  FHE_LAUNCH_CHECK();
  done = true;
  return 0;
}

// N = 2^12 rows on 4-CTA clusters (FHE_NTT_ROW_CLUSTER=0: whole-row tiles)
// (up to FHE_ROW_CLUSTER_PER_SM rows per SM; latency mode (twiddles
// prefetched) up to half a row per SM, throughput mode (64 registers, 4
// CTAs/SM) above: 1 row 6.4 -> 3.2 us, 169 rows 11.8 -> 9.8 us, 312 rows 25
// -> 17 us, 676 rows 34 -> 31 us, but 1040 rows 42 -> 45 us and 2080 rows
// 77 -> 82 us; tools/small_ntt_time.py, tools/ntt_bench.py 12 13 <cts>)
#ifndef FHE_ROW_CLUSTER_PER_SM
#define FHE_ROW_CLUSTER_PER_SM 5
#endif
bool row_cluster_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_NTT_ROW_CLUSTER");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// whole-row tiles with staged twiddles (FHE_NTT_ROWS_STW=0 reads them through L1)
bool rows_stw_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_NTT_ROWS_STW");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

template <int LOG_N>
int launch_rows(const DevChain& ch, const NttArgs& a, bool inverse, bool lazy, cudaStream_t st) {
  using T = RowsTile<LOG_N>;
  T tl;
  tl.rows = a.rows;
  tl.map = a.map;
  tl.src = RowAddr{a.src_bstride, a.map.limbs, LOG_N};
  tl.dst = RowAddr{a.dst_bstride, a.map.limbs, LOG_N};
  tl.fwd = !inverse;
  const int ntiles = (a.rows + T::NB - 1) / T::NB;
  if (a.bcast_src) {
    // centred broadcast input (rescale correction), FP64 path
    if (a.bcast_done) *a.bcast_done = false;
    if (inverse || !ch.fp64_ok) return 0;
    const int bdiv = a.bcast_div ? a.bcast_div : a.map.limbs;
    tl.bcast_limbs = bdiv;
    tl.bcast_stride = a.bcast_stride;
    tl.center = (double)a.center_q;
    if constexpr (LOG_N == 12) {
      if (a.rows <= FHE_ROW_CLUSTER_PER_SM * sm_count() && row_cluster_enabled()) {
        path_hit(FHE_NTT_PATH_CLUSTER);
        auto go = [&](auto kern) {
          kern<<<a.rows * 4, kRcThreads, 0, st>>>(ch, a.dst, a.bcast_src, a.map, tl.src, tl.dst,
                                                  bdiv, a.bcast_stride, (double)a.center_q,
                                                  a.rs_in, a.rs_out, a.rs_inv_d, a.rs_level);
        };
        if (a.rs_done) *a.rs_done = a.rs_in != nullptr;
        if (a.rows <= sm_count() / 2) go(ntt_row_cluster_kernel<true, true>);
        else go(ntt_row_cluster_kernel<true, false>);
        FHE_LAUNCH_CHECK();
        if (a.bcast_done) *a.bcast_done = true;
        return 0;
      }
    }
    path_hit(FHE_NTT_PATH_ROWS);
    const int rc = launch_tiles_fp<T, true, FPIN_U64, FPOUT_U64>(ch, a.dst, a.bcast_src, tl, ntiles, st);
    if (!rc && a.bcast_done) *a.bcast_done = true;
    return rc;
  }
  if constexpr (LOG_N == 12) {
    // one row per 4-CTA cluster (ntt_row_cluster.cuh) for launches of a few
    // rows per SM, where the per-row latency sets the time
    if (ch.fp64_ok && a.rows <= FHE_ROW_CLUSTER_PER_SM * sm_count() && row_cluster_enabled()) {
      path_hit(FHE_NTT_PATH_CLUSTER);
      const bool pf = a.rows <= sm_count() / 2;  // latency mode: <= 2 CTAs per SM
      auto go = [&](auto kern) {
        kern<<<a.rows * 4, kRcThreads, 0, st>>>(ch, a.dst, a.src, a.map, tl.src, tl.dst, 0, 0L, 0.0,
                                                nullptr, nullptr, nullptr, 0);
      };
      if (inverse) pf ? go(ntt_row_cluster_kernel<false, true>) : go(ntt_row_cluster_kernel<false, false>);
      else pf ? go(ntt_row_cluster_kernel<true, true>) : go(ntt_row_cluster_kernel<true, false>);
      FHE_LAUNCH_CHECK();
      return 0;
    }
  }
  path_hit(ch.fp64_ok ? FHE_NTT_PATH_ROWS : FHE_NTT_PATH_INT);
  // staged twiddles take 64 KB of shared memory (1 CTA/SM): for launches of at
  // most one row per SM, where latency, not occupancy, sets the time
  if (ch.fp64_ok && T::TWMAX > 0 && ch.tws && a.rows <= sm_count() && rows_stw_enabled())
    return inverse
               ? launch_tiles_fp<T, false, FPIN_U64, FPOUT_U64, true>(ch, a.dst, a.src, tl, ntiles, st)
               : launch_tiles_fp<T, true, FPIN_U64, FPOUT_U64, true>(ch, a.dst, a.src, tl, ntiles, st);
  if (ch.fp64_ok)
    return inverse ? launch_tiles_fp<T, false, FPIN_U64, FPOUT_U64>(ch, a.dst, a.src, tl, ntiles, st)
                   : launch_tiles_fp<T, true, FPIN_U64, FPOUT_U64>(ch, a.dst, a.src, tl, ntiles, st);
  if (inverse) return launch_tiles<T, false, false, OUT_RAW>(ch, a.dst, a.src, tl, ntiles, st);
  if (lazy) return launch_tiles<T, true, true, OUT_REDUCE>(ch, a.dst, a.src, tl, ntiles, st);
  return launch_tiles<T, true, false, OUT_CANON4>(ch, a.dst, a.src, tl, ntiles, st);
}

template <int LOG_N, int LOG_N1>
int launch_split(const DevChain& ch, const NttArgs& a, bool inverse, bool lazy,
                 cudaStream_t st) {
  using C = ColsTile<LOG_N, LOG_N1>;
  using K = ChunksTile<LOG_N, LOG_N1>;
  C ct;
  ct.rows = a.rows;
  ct.map = a.map;
  ct.fwd = !inverse;
  K kt;
  kt.rows = a.rows;
  kt.map = a.map;
  kt.fwd = !inverse;
  const RowAddr s{a.src_bstride, a.map.limbs, LOG_N}, d{a.dst_bstride, a.map.limbs, LOG_N};
  const int nc = a.rows * C::TILES, nk = kt.plan(a.rows, a.map.limbs);
  ct.limbs_div.init(a.map.limbs);
  // chunk tiles of <= 2 chunks stage their twiddles in shared memory
  const bool kstage = (K::NB >> kt.log_r) <= kChunkTwC;
  int rc;
  // TMA column tiles: N1 = 256 (one 256-k-row box), 16 columns per tile
  using CT = ColsTmaTile<LOG_N, LOG_N1>;
  constexpr bool kTmaShape = (LOG_N1 == 8) && (C::CN == 16);
  const bool use_tma = kTmaShape && ch.fp64_ok && tma_enabled();
  // TMA chunk tiles: 256-point chunks, staged twiddles, and whole batches of
  // rows (rows % limbs == 0: no box row can fall past the buffer's end)
  const bool use_ktma = (LOG_N - LOG_N1 == 8) && ch.fp64_ok && kstage && tma_enabled() &&
                        a.rows % a.map.limbs == 0 && std::getenv("FHE_NTT_KTMA") == nullptr;
  if (a.bcast_src) {
    // centred broadcast input (rescale): TMA column tiles only, one source
    // row per map.limbs target rows
    if (a.bcast_done) *a.bcast_done = false;
    if (a.bcast_div && a.bcast_div != a.map.limbs) return 0;
    if constexpr (kTmaShape) {
      if (inverse || !use_tma || a.fin) return 0;
      const double center = (double)a.center_q;
      bool done = false;
      if constexpr (LOG_N - LOG_N1 == 8) {
        if (use_ktma && ch.fuse && fused_tma_enabled() && kt.log_r >= FHE_FUSE_MIN_LOG_R) {
          ColsTmaTile<LOG_N, LOG_N1> tc;
          static_cast<C&>(tc) = ct;
          tc.bcast = true;
          tc.center = center;
          tc.src = d;
          tc.dst = d;
          ChunksTmaTile<LOG_N, LOG_N1> tk;
          static_cast<K&>(tk) = kt;
          if (tk.log_r > FHE_FUSE_MAX_LOG_R) tk.plan(a.rows, a.map.limbs, FHE_FUSE_MAX_LOG_R);
          tk.src = d;
          tk.dst = d;
          rc = launch_fused_tma(ch, a.dst, a.bcast_src, tc, tk, true, a.bcast_stride,
                                a.dst_bstride, a.rows, a.map.limbs, st, done, true);
          if (done) path_hit(FHE_NTT_PATH_FUSED_TMA);
          if (rc || done) {
            if (done && a.bcast_done) *a.bcast_done = true;
            return rc;
          }
        }
      }
      // two passes: the column pass reads the broadcast rows, the chunk pass
      // runs in place on dst
      CT tt;
      static_cast<C&>(tt) = ct;
      tt.bcast = true;
      tt.center = center;
      rc = launch_cols_tma<CT, true, FPIN_U64, FPOUT_DOUBLE>(ch, a.dst, a.bcast_src, tt, nc,
                                                            a.bcast_stride, a.dst_bstride, st,
                                                            done);
      if (rc || !done) return rc;
      path_hit(FHE_NTT_PATH_SPLIT);
      kt.src = d;
      kt.dst = d;
      bool kdone = false;
      if (use_ktma)
        rc = maybe_chunks_tma<LOG_N, LOG_N1, true, FPIN_DOUBLE, FPOUT_U64>(
            ch, a.dst, a.dst, kt, nk, a.dst_bstride, a.dst_bstride, st, kdone);
      if (!rc && !kdone)
        rc = kstage ? launch_tiles_fp<K, true, FPIN_DOUBLE, FPOUT_U64, true>(ch, a.dst, a.dst, kt, nk, st)
                    : launch_tiles_fp<K, true, FPIN_DOUBLE, FPOUT_U64>(ch, a.dst, a.dst, kt, nk, st);
      if (!rc && a.bcast_done) *a.bcast_done = true;
      return rc;
    }
    return 0;
  }
  if constexpr (LOG_N1 == 8 && LOG_N - LOG_N1 == 8) {
    // one pass, the row held by a 16-CTA cluster (DSMEM transpose)
    if (ch.fp64_ok && !a.fin && tma_enabled()) {
      bool done = false;
      rc = launch_cluster_ntt(ch, a, inverse, st, done);
      if (done) path_hit(FHE_NTT_PATH_CLUSTER);
      if (rc || done) return rc;
    }
    // fused for groups of >= 8 rows of one residue class: with the second
    // phase 16 groups behind the first, the key switch's 8-row groups (input
    // INTT, ModUp NTT) gain too (HMult+Relin +2.5%); at lag 8 they lost 15%
    if (use_tma && use_ktma && ch.fuse && fused_tma_enabled() && kt.log_r >= FHE_FUSE_MIN_LOG_R &&
        !a.fin) {
      ColsTmaTile<LOG_N, LOG_N1> tc;
      static_cast<C&>(tc) = ct;
      tc.src = inverse ? d : s;
      tc.dst = d;
      ChunksTmaTile<LOG_N, LOG_N1> tk;
      static_cast<K&>(tk) = kt;
      // smaller row groups keep the L2-resident window (lag x group) small
      if (tk.log_r > FHE_FUSE_MAX_LOG_R) tk.plan(a.rows, a.map.limbs, FHE_FUSE_MAX_LOG_R);
      tk.src = inverse ? s : d;
      tk.dst = d;
      bool done = false;
      rc = launch_fused_tma(ch, a.dst, a.src, tc, tk, !inverse, a.src_bstride, a.dst_bstride,
                            a.rows, a.map.limbs, st, done);
      if (done) path_hit(FHE_NTT_PATH_FUSED_TMA);
      if (rc || done) return rc;
    }
  }
  if (C::THREADS == K::THREADS && ch.fp64_ok && kstage && ch.fuse && fused_enabled() && !a.fin) {
    ct.src = inverse ? d : s;
    ct.dst = d;
    kt.src = inverse ? s : d;
    kt.dst = d;
    path_hit(FHE_NTT_PATH_FUSED_CP);
    return launch_fused(ch, a.dst, a.src, ct, kt, !inverse, a.rows, a.map.limbs, st);
  }
  path_hit(ch.fp64_ok ? FHE_NTT_PATH_SPLIT : FHE_NTT_PATH_INT);
  if (ch.fp64_ok) {
    if (!inverse) {
      ct.src = s;
      ct.dst = d;
      kt.src = d;
      kt.dst = d;
      bool done = false;
      if (use_tma) {
        CT tt;
        static_cast<C&>(tt) = ct;
        rc = launch_cols_tma<CT, true, FPIN_U64, FPOUT_DOUBLE>(ch, a.dst, a.src, tt, nc,
                                                              a.src_bstride, a.dst_bstride, st,
                                                              done);
        if (rc) return rc;
      }
      if (!done)
        rc = launch_tiles_fp<C, true, FPIN_U64, FPOUT_DOUBLE, true>(ch, a.dst, a.src, ct, nc, st);
      bool kdone = false;
      if (!rc && use_ktma) {
        rc = maybe_chunks_tma<LOG_N, LOG_N1, true, FPIN_DOUBLE, FPOUT_U64>(
            ch, a.dst, a.dst, kt, nk, a.dst_bstride, a.dst_bstride, st, kdone, a.fin);
        if (!rc && kdone && a.fin && a.fin_done) *a.fin_done = true;
      }
      if (!rc && !kdone)
        rc = kstage ? launch_tiles_fp<K, true, FPIN_DOUBLE, FPOUT_U64, true>(ch, a.dst, a.dst, kt, nk, st)
                    : launch_tiles_fp<K, true, FPIN_DOUBLE, FPOUT_U64>(ch, a.dst, a.dst, kt, nk, st);
    } else {
      kt.src = s;
      kt.dst = d;
      ct.src = d;
      ct.dst = d;
      bool kdone = false;
      rc = 0;
      if (use_ktma)
        rc = maybe_chunks_tma<LOG_N, LOG_N1, false, FPIN_U64, FPOUT_DOUBLE>(
            ch, a.dst, a.src, kt, nk, a.src_bstride, a.dst_bstride, st, kdone);
      if (!rc && !kdone)
        rc = kstage ? launch_tiles_fp<K, false, FPIN_U64, FPOUT_DOUBLE, true>(ch, a.dst, a.src, kt, nk, st)
                    : launch_tiles_fp<K, false, FPIN_U64, FPOUT_DOUBLE>(ch, a.dst, a.src, kt, nk, st);
      bool done = false;
      if (!rc && use_tma) {
        CT tt;
        static_cast<C&>(tt) = ct;
        rc = launch_cols_tma<CT, false, FPIN_DOUBLE, FPOUT_U64>(ch, a.dst, a.dst, tt, nc,
                                                               a.dst_bstride, a.dst_bstride, st,
                                                               done);
      }
      if (!rc && !done)
        rc = launch_tiles_fp<C, false, FPIN_DOUBLE, FPOUT_U64, true>(ch, a.dst, a.dst, ct, nc, st);
    }
    return rc;
  }
  if (!inverse) {
    ct.src = s;
    ct.dst = d;
    kt.src = d;
    kt.dst = d;
    if (lazy) {
      rc = launch_tiles<C, true, true, OUT_RAW>(ch, a.dst, a.src, ct, nc, st);
      if (!rc) rc = launch_tiles<K, true, true, OUT_REDUCE>(ch, a.dst, a.dst, kt, nk, st);
    } else {
      rc = launch_tiles<C, true, false, OUT_RAW>(ch, a.dst, a.src, ct, nc, st);
      if (!rc) rc = launch_tiles<K, true, false, OUT_CANON4>(ch, a.dst, a.dst, kt, nk, st);
    }
  } else {
    kt.src = s;
    kt.dst = d;
    ct.src = d;
    ct.dst = d;
    rc = launch_tiles<K, false, false, OUT_RAW>(ch, a.dst, a.src, kt, nk, st);
    if (!rc) rc = launch_tiles<C, false, false, OUT_RAW>(ch, a.dst, a.dst, ct, nc, st);
  }
  return rc;
}

}  // namespace

static int launch_ntt_chain(const DevChain& ch, const NttArgs& a, bool inverse, cudaStream_t st);

// FHE_NTT_MIXED_FP64=0: a mixed chain's transforms all stay on the integer path
static bool mixed_fp64_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_NTT_MIXED_FP64");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

int launch_ntt(const DevChain& ch, const NttArgs& a, bool inverse, cudaStream_t st) {
  if (a.rows <= 0) return 0;
  // mixed chain (some prime >= 2^50): a transform whose rows only use primes
  // below 2^50 (identity map over a prime range) runs on the FP64 path --
  // same canonical words as the integer path
  if (!ch.fp64_ok && ch.twd && ch.fp64_prime_host && (a.map.idx == nullptr || a.fp64_rows) &&
      mixed_fp64_enabled()) {
    bool ok = a.fp64_rows ||
              (a.map.offset >= 0 && a.map.limbs > 0 && a.map.offset + a.map.limbs <= ch.count);
    for (int j = 0; ok && !a.fp64_rows && j < a.map.limbs; ++j)
      ok = ch.fp64_prime_host[a.map.offset + j] != 0;
    if (ok) {
      DevChain c2 = ch;
      c2.fp64_ok = true;
      return launch_ntt_chain(c2, a, inverse, st);
    }
  }
  return launch_ntt_chain(ch, a, inverse, st);
}

static int launch_ntt_chain(const DevChain& ch, const NttArgs& a, bool inverse, cudaStream_t st) {
  const bool lazy = !inverse && ch.lazy_ok;
  switch (ch.log_n) {
    case 1: return launch_rows<1>(ch, a, inverse, lazy, st);
    case 2: return launch_rows<2>(ch, a, inverse, lazy, st);
    case 3: return launch_rows<3>(ch, a, inverse, lazy, st);
    case 4: return launch_rows<4>(ch, a, inverse, lazy, st);
    case 5: return launch_rows<5>(ch, a, inverse, lazy, st);
    case 6: return launch_rows<6>(ch, a, inverse, lazy, st);
    case 7: return launch_rows<7>(ch, a, inverse, lazy, st);
    case 8: return launch_rows<8>(ch, a, inverse, lazy, st);
    case 9: return launch_rows<9>(ch, a, inverse, lazy, st);
    case 10: return launch_rows<10>(ch, a, inverse, lazy, st);
    case 11: return launch_rows<11>(ch, a, inverse, lazy, st);
    case 12: return launch_rows<12>(ch, a, inverse, lazy, st);
    case 13: return launch_split<13, 6>(ch, a, inverse, lazy, st);
    case 14: return launch_split<14, 7>(ch, a, inverse, lazy, st);
    case 15: return launch_split<15, 7>(ch, a, inverse, lazy, st);
    case 16: return launch_split<16, 8>(ch, a, inverse, lazy, st);
    case 17: return launch_split<17, 8>(ch, a, inverse, lazy, st);
    default:
      fhe_set_error("unsupported ring degree 2^" + std::to_string(ch.log_n));
      return -1;
  }
}

// The counter slabs are allocated with the chain (log N >= 13, where the fused
// transforms run): 64K groups per launch covers every transform that fits in
// HBM (a group is >= 8 rows of 2^13+ words), so fuse_slab never has to grow
// (and synchronise the device) on a first-use path.
void* fuse_scratch_new(int log_n) {
  FuseScratch* fs = new FuseScratch();
  if (log_n >= 13) {
    const size_t ints = 1 << 16;
    if (cudaMalloc(&fs->dev, ints * kFuseSlabs * sizeof(int)) != cudaSuccess) {
      delete fs;
      return nullptr;
    }
    fs->slab_ints = ints;
  }
  return fs;
}

void fuse_scratch_free(void* p) {
  FuseScratch* fs = static_cast<FuseScratch*>(p);
  if (!fs) return;
  for (cudaEvent_t& e : fs->ev)
    if (e) cudaEventDestroy(e);
  if (fs->dev) cudaFree(fs->dev);
  delete fs;
}

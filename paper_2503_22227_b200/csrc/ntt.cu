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

#include <cstdlib>
#include <mutex>

namespace {

// Tile geometry.  Whole-row tiles: 4096 elements, 256 threads, 2 CTAs/SM.
// Split (four-step) tiles: 2048 elements, 128 threads, 4 CTAs/SM -- small
// CTAs keep the SM's FP64 pipe fed while other CTAs sit in their load /
// barrier / store phases.
constexpr int kRowThreads = 256;
constexpr int kLogRowTile = 12;
constexpr int kSplitThreads = 128;
constexpr int kLogSplitTile = 11;
#ifndef FHE_SPLIT_MINB
#define FHE_SPLIT_MINB 6
#endif
#ifndef FHE_SPLIT_NBUF
#define FHE_SPLIT_NBUF 1
#endif
#ifndef FHE_CHUNK_MINB
#define FHE_CHUNK_MINB 5
#endif
#ifndef FHE_CHUNK_NBUF
#define FHE_CHUNK_NBUF FHE_SPLIT_NBUF
#endif
#ifndef FHE_CHUNK_TWC
#define FHE_CHUNK_TWC 2
#endif
// experiment switch: butterflies skipped (measures the data-movement floor)
#ifdef FHE_NTT_NOCOMPUTE
constexpr bool NOCOMP = true;
#else
constexpr bool NOCOMP = false;
#endif
constexpr int kSplitMinB = FHE_SPLIT_MINB;
constexpr int kSplitNBuf = FHE_SPLIT_NBUF;  // tile buffers per CTA (1: occupancy hides loads)
#ifndef FHE_COLS_LOG_TILE
#define FHE_COLS_LOG_TILE 12
#endif
#ifndef FHE_COLS_THREADS
#define FHE_COLS_THREADS kSplitThreads
#endif
#ifndef FHE_COLS_MINB
#define FHE_COLS_MINB 5
#endif
#ifndef FHE_TMA_STAGES
#define FHE_TMA_STAGES 1
#endif
#ifndef FHE_TMA_COLS_MINB
#define FHE_TMA_COLS_MINB FHE_COLS_MINB
#endif
#ifndef FHE_TMA_CHUNK_MINB
#define FHE_TMA_CHUNK_MINB FHE_CHUNK_MINB
#endif
constexpr int kColsLogTile = FHE_COLS_LOG_TILE;
constexpr int kColsThreads = FHE_COLS_THREADS;
constexpr int kColsMinB = FHE_COLS_MINB;
#ifndef FHE_CHUNK_LOG_TILE
#define FHE_CHUNK_LOG_TILE 12
#endif
constexpr int kChunkLogTile = FHE_CHUNK_LOG_TILE;
constexpr int kChunkMinB = FHE_CHUNK_MINB;
constexpr int kChunkNBuf = FHE_CHUNK_NBUF;
constexpr int kChunkTwC = FHE_CHUNK_TWC;    // chunks per tile whose twiddles can be staged



__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Padded shared-memory index of array tiles (whole rows, chunks): 16 bytes of
// pad per 16-element (128-byte) row and another 16 per 256 elements.  With
// array-major thread mapping (an array's groups on consecutive lanes) both
// stride-16 and contiguous groups are bank-conflict free.
__device__ __forceinline__ int padix(int t) { return t + ((t >> 4) << 1) + ((t >> 8) << 1); }

constexpr int padded_words(int tile) { return tile + tile / 8 + tile / 128; }
// padded distance between element i and i+1 of a thread's group (stride TMIN
// in k-rows of CN columns (column tiles) or in elements), 0 when not affine
constexpr int pad_step(int cn, int tmin, int e) {
  return cn ? (tmin >= 16 ? (cn + 2) * tmin + 2 * (tmin / 16)
                          : (tmin * e <= 16 ? (cn + 2) * tmin : 0))
              : (tmin == 1 ? 1
                           : (tmin >= 256 ? tmin + tmin / 8 + tmin / 128
                                          : (tmin >= 16 && tmin * e <= 256 ? tmin + tmin / 8 : 0)));
}

// Per-array context of one local transform.
struct ArrCtx {
  const WPair* tw;  // table of the array's prime (forward or inverse)
  u64 q;
  int m0;           // global group base: twiddle index = (m0 << r) + g_local
  int prime;        // chain position (final reduction / n^-1 folding)
  bool fold;        // inverse: fold n^-1 into global stage 0
};

// Logical row -> word offset of its first coefficient (batched strided rows:
// row r lives at (r / limbs) * bstride + (r % limbs) * N; bstride 0 means
// contiguous rows).
struct RowAddr {
  long bstride;
  int limbs;
  int log_n;
  __device__ __forceinline__ long operator()(int r) const {
    return bstride ? (long)(r / limbs) * bstride + ((long)(r % limbs) << log_n)
                   : ((long)r << log_n);
  }
};

// n / d for 0 <= n < 2^31 without a hardware divide (Granlund-Montgomery):
// n / d = (umulhi(n, m) + n) >> s.  Built on the host.
struct FastDiv {
  u32 d = 1, m = 1, s = 0;
  void init(u32 d_) {
    d = d_;
    s = 0;
    while ((1u << s) < d) ++s;
    m = (u32)((((1ull << 32) * ((1ull << s) - d)) / d) + 1);
  }
  __device__ __forceinline__ int div(int n) const {
    return (int)((__umulhi((u32)n, m) + (u32)n) >> s);
  }
};

// ---------------------------------------------------------------------------
// Tile policies.  A tile holds arrays() local arrays of S = 2^LOG_S elements.
// tile_index(b, k) is an element's slot in the tile before swizzling;
// gsrc/gdst its global address.

// Whole rows (N <= 2^12): NB = 4096 / N rows per tile.
template <int LOG_N>
struct RowsTile {
  static constexpr int LOG_S = LOG_N;
  static constexpr int S = 1 << LOG_N;
  static constexpr int TILE = 1 << kLogRowTile;
  static constexpr int NB = S >= TILE ? 1 : (TILE / S > 32 ? 32 : TILE / S);
  static constexpr int GS0 = 0;  // global stage of local stage 0
  static constexpr bool LANE_MAJOR = false;
  static constexpr bool DENSE = false;  // unpadded smem rows (TMA tiles)
  static constexpr bool TMA = false;
  static constexpr bool SWZ = false;   // 128B-swizzled rows (TMA chunk tiles)
  static constexpr int THREADS = kRowThreads;
  static constexpr int MINB = 2;
  static constexpr int NBUF = 2;
  static constexpr int SMEM_WORDS = padded_words(NB * S);
  static constexpr int LOG_CN_OR0 = 0;
  static constexpr long N2 = 1;  // (column tiles only)
  static constexpr bool COLS = false;
  static constexpr bool EPI = true;
  static constexpr long GSTEP_PER_K = 1;
  __device__ static __forceinline__ int pad(int t) { return padix(t); }
  int rows;
  RowMap map;
  RowAddr src, dst;
  bool fwd;
  int row0, nb;
  bool valid = true;
  int prime[NB];
  __device__ __forceinline__ void setup(int t) {
    row0 = t * NB;
    nb = min(NB, rows - row0);
    for (int b = 0; b < NB; ++b) prime[b] = b < nb ? map(row0 + b) : 0;
  }
  __device__ __forceinline__ int tile_index(int b, int k) const { return (b << LOG_S) + k; }
  __device__ __forceinline__ void split(int G, int gpa_log, int& b, int& g) const {
    b = G >> gpa_log;
    g = G & ((1 << gpa_log) - 1);
  }
  __device__ __forceinline__ const u64* gsrc(const u64* base, int b, int k) const {
    return base + src(row0 + b) + k;
  }
  __device__ __forceinline__ u64* gdst(u64* base, int b, int k) const {
    return base + dst(row0 + b) + k;
  }
  __device__ __forceinline__ ArrCtx ctx(int b, const DevChain& ch) const {
    const int p = prime[b];
    return ArrCtx{(fwd ? ch.tw : ch.itw) + ((size_t)p << LOG_N), ch.mc[p].q, 1, p, !fwd};
  }
  __device__ __forceinline__ int arrays() const { return nb; }
  // rows of a tile may use different primes: twiddles are read through L1
  static constexpr int TWMAX = 0;
  __device__ __forceinline__ int tw_pairs() const { return 0; }
  __device__ __forceinline__ long tw_src_off() const { return 0; }
  __device__ __forceinline__ int tw_base(int, int) const { return 0; }
  __device__ __forceinline__ int tw_prime() const { return 0; }
};

// First log N1 stages on a [N1][CN] column tile of one row (CN = 2048 / N1
// columns, one 8*CN-byte segment per k).
template <int LOG_N, int LOG_N1>
struct ColsTile {
  static constexpr int LOG_S = LOG_N1;
  static constexpr int GS0 = 0;
  static constexpr bool COLS = true;
  static constexpr bool EPI = true;
  static constexpr int N2 = 1 << (LOG_N - LOG_N1);
  static constexpr long GSTEP_PER_K = N2;
  static constexpr int LOG_CN = kColsLogTile - LOG_N1;
  static constexpr int CN = 1 << LOG_CN;
  static constexpr int LOG_CN_OR0 = LOG_CN;
  static constexpr int TILES = N2 / CN;
  static constexpr int THREADS = kColsThreads;
  static constexpr int MINB = kColsMinB;
  static constexpr int NBUF = kSplitNBuf;
  static constexpr int TILE = 1 << kColsLogTile;
  // >= 16 columns: lanes run across the columns of a k-row (conflict-free
  // with any row layout); passes then exchange under __syncthreads
  static constexpr bool LANE_MAJOR = CN >= 16;
  static constexpr bool DENSE = false;
  static constexpr bool TMA = false;
  static constexpr bool SWZ = false;
  // padded index: k-rows of CN words + 2, and 2 more per 16 k-rows, so both
  // stride-16 and contiguous-16 groups along k are bank-conflict free
  __device__ static __forceinline__ int pad(int t) {
    const int k = t >> LOG_CN;
    return t + (k << 1) + ((k >> 4) << 1);
  }
  static constexpr int SMEM_WORDS = TILE + 2 * (1 << LOG_N1) + 2 * ((1 << LOG_N1) >> 4);
  int rows;
  RowMap map;
  RowAddr src, dst;
  bool fwd;
  int row, j0, p;
  bool valid = true;
  long so, dof;  // word offsets of the tile's first element in src / dst
  FastDiv limbs_div;  // row -> (row / limbs, row % limbs) without IMAD-heavy division
  __device__ __forceinline__ void setup(int t) {
    row = t / TILES;
    j0 = (t % TILES) * CN;
    const int rq = limbs_div.div(row);
    const int cls = row - rq * map.limbs;
    p = (map.idx ? map.idx[cls] : cls) + map.offset;
    so = (src.bstride ? rq * src.bstride + ((long)cls << LOG_N) : ((long)row << LOG_N)) + j0;
    dof = (dst.bstride ? rq * dst.bstride + ((long)cls << LOG_N) : ((long)row << LOG_N)) + j0;
  }
  // twiddles staged in shared memory per tile: the N1-pair column block of
  // the prime's staged table (ntt_plan.cuh)
  static constexpr int TWMAX = 1 << LOG_N1;
  __device__ __forceinline__ int tw_pairs() const { return 1 << LOG_N1; }
  __device__ __forceinline__ long tw_src_off() const { return 0; }
  __device__ __forceinline__ int tw_base(int s, int) const { return 1 << s; }
  __device__ __forceinline__ int tw_prime() const { return p; }
  __device__ __forceinline__ int tile_index(int b, int k) const { return (k << LOG_CN) + b; }
  // array-major: the groups of one column sit on consecutive lanes, so a
  // pass's exchange stays inside the warp when every pass has 2^g_log groups
  // With 16 groups per column a warp owns two columns; each half-warp holds
  // 8 groups of both columns so its 8-byte shared accesses (serviced per
  // half-warp) hit 16 distinct bank pairs in both passes.
  __device__ __forceinline__ void split(int G, int gpa_log, int& b, int& g) const {
    if (LANE_MAJOR) {
      b = G & (CN - 1);
      g = G >> LOG_CN;
    } else if (gpa_log == 4) {
      const int lane = G & 31;
      b = ((G >> 5) << 1) + ((lane >> 3) & 1);
      g = ((lane >> 4) << 3) | (lane & 7);
    } else {
      b = G >> gpa_log;
      g = G & ((1 << gpa_log) - 1);
    }
  }
  __device__ __forceinline__ const u64* gsrc(const u64* base, int b, int k) const {
    return base + so + k * N2 + b;
  }
  __device__ __forceinline__ u64* gdst(u64* base, int b, int k) const {
    return base + dof + k * N2 + b;
  }
  __device__ __forceinline__ ArrCtx ctx(int, const DevChain& ch) const {
    return ArrCtx{(fwd ? ch.tw : ch.itw) + ((size_t)p << LOG_N), ch.mc[p].q, 1, p, !fwd};
  }
  __device__ __forceinline__ int arrays() const { return CN; }
};

// Remaining stages on contiguous N2-chunks: a tile holds R rows of one
// residue class (rows r0 + i * limbs share a prime) x C consecutive chunks,
// R * C = NB.  Array b = (i, c) with i = b >> log_c, c = b & (C - 1).  The
// R rows of a tile share every twiddle (the chunk stages' twiddles depend only
// on the chunk index), so one L1 line serves R arrays.
template <int LOG_N, int LOG_N1>
struct ChunksTile {
  static constexpr int LOG_S = LOG_N - LOG_N1;
  static constexpr int GS0 = LOG_N1;
  static constexpr bool LANE_MAJOR = false;
  static constexpr bool DENSE = false;  // unpadded smem rows (TMA tiles)
  static constexpr bool TMA = false;
  static constexpr bool SWZ = false;   // 128B-swizzled rows (TMA chunk tiles)
  static constexpr int S = 1 << LOG_S;
  static constexpr int TILE = 1 << kChunkLogTile;
  static constexpr int NB = TILE / S;
  static constexpr int THREADS = kSplitThreads;
  static constexpr int MINB = kChunkMinB;
  static constexpr int NBUF = kChunkNBuf;
  static constexpr int SMEM_WORDS = padded_words(TILE);
  static constexpr int LOG_CN_OR0 = 0;
  static constexpr long N2 = 1;  // (column tiles only)
  static constexpr bool COLS = false;
  static constexpr bool EPI = true;
  static constexpr long GSTEP_PER_K = 1;
  __device__ static __forceinline__ int pad(int t) { return padix(t); }
  static constexpr int N1 = 1 << LOG_N1;
  int rows;
  RowMap map;
  RowAddr src, dst;
  bool fwd;
  int log_r = 0;    // rows per tile = 1 << log_r (<= NB)
  int rblocks = 1;  // row blocks per residue class
  int cblocks = 1;  // chunk blocks per row = N1 / C
  bool valid = true;
  int log_c, c0, p, nb;
  int cls_ = 0, i0_ = 0;  // residue class and first row ordinal of the tile
  long so, dof, sstep, dstep;  // word offsets of array (0, 0) and the per-row steps
  // Tile order: (residue class, row block, chunk block): consecutive tiles of
  // a CTA share the prime and walk the chunks of the same rows.
  int log_cb = 0;       // log2(cblocks)
  int rows_q = 0, rows_r = 0;  // rows / limbs, rows % limbs
  FastDiv rb_div;       // division by rblocks
  __device__ __forceinline__ void setup(int t) {
    const int cb = t & (cblocks - 1);
    const int u = t >> log_cb;
    const int cls = rb_div.div(u);
    const int rb = u - cls * rblocks;
    log_c = kChunkLogTile - LOG_S - log_r;
    c0 = cb << log_c;
    const int i0 = rb << log_r;
    cls_ = cls;
    i0_ = i0;
    const int row0 = cls + i0 * map.limbs;
    valid = row0 < rows;
    if (!valid) return;
    const int in_class = rows_q + (cls < rows_r ? 1 : 0);
    nb = min(1 << log_r, in_class - i0) << log_c;
    p = (map.idx ? map.idx[cls] : cls) + map.offset;
    so = (src.bstride ? i0 * src.bstride + ((long)cls << LOG_N) : ((long)row0 << LOG_N)) +
         ((long)c0 << LOG_S);
    dof = (dst.bstride ? i0 * dst.bstride + ((long)cls << LOG_N) : ((long)row0 << LOG_N)) +
          ((long)c0 << LOG_S);
    sstep = src.bstride ? src.bstride : ((long)map.limbs << LOG_N);
    dstep = dst.bstride ? dst.bstride : ((long)map.limbs << LOG_N);
  }
  // twiddles staged in shared memory per tile (tiles of <= 2 chunks): the
  // C consecutive S-pair chunk blocks of the prime's staged table
  static constexpr int TWMAX = kChunkTwC << LOG_S;
  __device__ __forceinline__ int tw_pairs() const { return S << log_c; }
  __device__ __forceinline__ long tw_src_off() const { return N1 + ((long)c0 << LOG_S); }
  __device__ __forceinline__ int tw_base(int s, int m0) const {
    return ((m0 - N1 - c0) << LOG_S) + (1 << s);
  }
  __device__ __forceinline__ int tw_prime() const { return p; }
  __device__ __forceinline__ int tile_index(int b, int k) const { return (b << LOG_S) + k; }
  __device__ __forceinline__ void split(int G, int gpa_log, int& b, int& g) const {
    b = G >> gpa_log;
    g = G & ((1 << gpa_log) - 1);
  }
  __device__ __forceinline__ const u64* gsrc(const u64* base, int b, int k) const {
    return base + so + (b >> log_c) * sstep + ((b & ((1 << log_c) - 1)) << LOG_S) + k;
  }
  __device__ __forceinline__ u64* gdst(u64* base, int b, int k) const {
    return base + dof + (b >> log_c) * dstep + ((b & ((1 << log_c) - 1)) << LOG_S) + k;
  }
  __device__ __forceinline__ ArrCtx ctx(int b, const DevChain& ch) const {
    return ArrCtx{(fwd ? ch.tw : ch.itw) + ((size_t)p << LOG_N), ch.mc[p].q,
                  N1 + c0 + (b & ((1 << log_c) - 1)), p, false};
  }
  __device__ __forceinline__ int arrays() const { return nb; }
  // host: tiles for `rows` rows with residue classes of `limbs`
  int plan(int rows_, int limbs) {
    const int rpc = (rows_ + limbs - 1) / limbs;
    log_r = 0;
    while ((2 << log_r) <= NB && (2 << log_r) <= rpc) ++log_r;
    rblocks = (rpc + (1 << log_r) - 1) >> log_r;
    const int C = NB >> log_r;
    cblocks = N1 / C;
    log_cb = 0;
    while ((1 << log_cb) < cblocks) ++log_cb;
    rb_div.init(rblocks);
    rows_q = rows_ / limbs;
    rows_r = rows_ % limbs;
    return std::min(limbs, rows_) * rblocks * cblocks;
  }
};

// Output handling of the final pass of a kernel.
enum OutMode {
  OUT_RAW = 0,     // store values as they are (intermediate of a split transform)
  OUT_CANON4 = 1,  // forward Harvey: [0, 4q) -> [0, q)
  OUT_REDUCE = 2   // forward lazy: [0, 33q) -> [0, q) by Barrett
};

// Every register pass of a LOG_S-stage local transform has the same radix and
// at most 32 groups per array: with array-major thread mapping each array is
// owned by one warp in every pass, so passes exchange data under __syncwarp.
constexpr bool warp_local(int log_s) {
  for (int p = 1; p < npass(log_s); ++p)
    if (pass_e(log_s, p) != pass_e(log_s, 0)) return false;
  return log_s - pass_e(log_s, 0) <= 5;
}

// Copy a finished tile from shared memory to global memory in 16-byte pairs.
//  * column tiles: CTA-wide (a k-row of 16 columns = 128 contiguous bytes);
//  * array tiles, warp-local passes: each warp stores the arrays it computed;
//  * array tiles otherwise: CTA-wide over all arrays.
template <class Tile, int GPA_LOG, bool WL>
__device__ __forceinline__ void epilogue_store(const u64* sm, const Tile& tl, u64* gout,
                                               const DevChain& ch) {
  constexpr int LOG_S = Tile::LOG_S;
  constexpr int S = 1 << LOG_S;
  constexpr int T = Tile::THREADS;
  if constexpr (Tile::TMA) {
    if constexpr (Tile::SWZ) {
      if (tl.has_fin) {  // fused ModDown finish instead of the transform store
        __syncthreads();
        tl.finish_store(sm, ch);
        return;
      }
    }
    // results are in the dense tile: one bulk tensor store by thread 0
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) tl.tma_store(sm);
  } else if constexpr (Tile::COLS) {
    constexpr int CN = 1 << Tile::LOG_CN_OR0;
    constexpr int PPR = CN / 2;
    constexpr int KSTEP = T / PPR;
    __syncthreads();
    const int k0 = threadIdx.x / PPR, c = (threadIdx.x % PPR) * 2;
    u64* g = tl.gdst(gout, c, k0);
#pragma unroll
    for (int j = 0; j < S / KSTEP; ++j) {
      const int so = (KSTEP % 16 == 0)
                         ? Tile::pad(k0 * CN + c) + j * (KSTEP * (CN + 2) + 2 * (KSTEP / 16))
                         : Tile::pad((k0 + j * KSTEP) * CN + c);
      const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(sm + so);
      *reinterpret_cast<ulonglong2*>(g + (long)j * KSTEP * Tile::N2) = v;
    }
  } else if constexpr (WL) {
    // the warp's arrays (all passes kept them on this warp)
    __syncwarp();
    const int lane = threadIdx.x & 31;
    constexpr int APW = 32 >> GPA_LOG;  // arrays per warp and G-sweep
    const int total = tl.arrays() << GPA_LOG;
    for (int G0 = threadIdx.x - lane; G0 < total; G0 += T) {
#pragma unroll
      for (int a = 0; a < APW; ++a) {
        const int b = (G0 >> GPA_LOG) + a;
        if (b >= tl.arrays()) break;
        u64* g = tl.gdst(gout, b, 0);
#pragma unroll
        for (int k = 2 * lane; k < S; k += 64) {
          const ulonglong2 v =
              *reinterpret_cast<const ulonglong2*>(&sm[Tile::pad((b << LOG_S) + k)]);
          *reinterpret_cast<ulonglong2*>(g + k) = v;
        }
      }
    }
  } else {
    __syncthreads();
    for (int q = threadIdx.x; q < (tl.arrays() << LOG_S) >> 1; q += T) {
      const int bb = q >> (LOG_S - 1), k = (q & ((S >> 1) - 1)) << 1;
      const ulonglong2 v =
          *reinterpret_cast<const ulonglong2*>(&sm[Tile::pad((bb << LOG_S) + k)]);
      *reinterpret_cast<ulonglong2*>(tl.gdst(gout, bb, k)) = v;
    }
  }
}

// One register pass covering local stages R0 .. R0+E_LOG-1.
// LAST: values go straight to global memory instead of back to the tile.
template <int LOG_S, int R0, int E_LOG, bool FWD, bool LAZY, bool LAST, int OUT, class Tile>
__device__ __forceinline__ void run_pass(u64* sm, const Tile& tl, u64* gout,
                                         const DevChain& ch) {
  constexpr int E = 1 << E_LOG;
  constexpr int T0 = (1 << LOG_S) >> (R0 + 1);
  constexpr int TMIN_LOG = LOG_S - R0 - E_LOG;
  constexpr int TMIN = 1 << TMIN_LOG;
  constexpr int GPA_LOG = LOG_S - E_LOG;
  constexpr bool VEC = (TMIN_LOG == 0) && !Tile::COLS && E >= 2;
  // padded stride between consecutive elements of the thread (0: not affine)
  constexpr int PSTEP = Tile::DENSE ? (Tile::COLS ? TMIN << Tile::LOG_CN_OR0 : TMIN)
                                    : pad_step(Tile::COLS ? (1 << Tile::LOG_CN_OR0) : 0, TMIN, E);
  const int total = tl.arrays() << GPA_LOG;
  for (int G = threadIdx.x; G < total; G += blockDim.x) {
    int b, g;
    tl.split(G, GPA_LOG, b, g);
    const int hi = g >> TMIN_LOG;
    const int lo = g & (TMIN - 1);
    const int base = hi * 2 * T0 + lo;
    const int pb = Tile::pad(tl.tile_index(b, base));
    const ArrCtx cx = tl.ctx(b, ch);
    const u64 q = cx.q;
    const u64 q2 = 2 * q;
    u64 x[E];
    if (VEC) {
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&sm[pb + i + ((i >> 4) << 1)]);
        x[i] = v.x;
        x[i + 1] = v.y;
      }
    } else if (PSTEP) {
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = sm[pb + i * PSTEP];
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) x[i] = sm[Tile::pad(tl.tile_index(b, base + i * TMIN))];
    }
    if (FWD) {
#pragma unroll
      for (int rr = 0; rr < E_LOG; ++rr) {
        const int half = E >> (rr + 1);
        const WPair* twr = cx.tw + (cx.m0 << (R0 + rr)) + (hi << rr);
#pragma unroll
        for (int blk = 0; blk < (1 << rr); ++blk) {
          const ulonglong2 wv = __ldg(reinterpret_cast<const ulonglong2*>(twr + blk));
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const int a = blk * 2 * half + i, c = a + half;
            u64 u = x[a];
            if (!LAZY) u = u >= q2 ? u - q2 : u;
            const u64 v = shoup_lazy(x[c], wv.x, wv.y, q);
            x[a] = u + v;
            x[c] = u - v + q2;
          }
        }
      }
    } else {
#pragma unroll
      for (int rr = E_LOG - 1; rr >= 0; --rr) {
        const int half = E >> (rr + 1);
        const bool fold = (R0 == 0) && (rr == 0) && cx.fold;
        const WPair* twr = cx.tw + (cx.m0 << (R0 + rr)) + (hi << rr);
#pragma unroll
        for (int blk = 0; blk < (1 << rr); ++blk) {
          const ulonglong2 wv =
              __ldg(reinterpret_cast<const ulonglong2*>(fold ? &ch.ninv_w1[cx.prime] : twr + blk));
          const ulonglong2 sn =
              fold ? __ldg(reinterpret_cast<const ulonglong2*>(&ch.ninv[cx.prime])) : wv;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const int a = blk * 2 * half + i, c = a + half;
            const u64 u = x[a], v = x[c];
            const u64 s = u + v;
            const u64 d = u - v + q2;
            if (fold) {
              x[a] = shoup_mul(s, sn.x, sn.y, q);
              x[c] = shoup_mul(d, wv.x, wv.y, q);
            } else {
              x[a] = s >= q2 ? s - q2 : s;
              x[c] = shoup_lazy(d, wv.x, wv.y, q);
            }
          }
        }
      }
    }
    if (LAST) {
      if (OUT == OUT_CANON4) {
#pragma unroll
        for (int i = 0; i < E; ++i) x[i] = csub(csub(x[i], q2), q);
      } else if (OUT == OUT_REDUCE) {
        const ModConst mc = ch.mc[cx.prime];
#pragma unroll
        for (int i = 0; i < E; ++i) x[i] = reduce_word(x[i], mc);
      }
      u64* o = tl.gdst(gout, b, base);
      if (VEC) {
#pragma unroll
        for (int i = 0; i < E; i += 2)
          *reinterpret_cast<ulonglong2*>(o + i) = make_ulonglong2(x[i], x[i + 1]);
      } else {
        constexpr long GSTEP = Tile::GSTEP_PER_K * TMIN;
#pragma unroll
        for (int i = 0; i < E; ++i) o[i * GSTEP] = x[i];
      }
    } else {
      if (VEC) {
#pragma unroll
        for (int i = 0; i < E; i += 2)
          *reinterpret_cast<ulonglong2*>(&sm[pb + i + ((i >> 4) << 1)]) = make_ulonglong2(x[i], x[i + 1]);
      } else if (PSTEP) {
#pragma unroll
        for (int i = 0; i < E; ++i) sm[pb + i * PSTEP] = x[i];
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) sm[Tile::pad(tl.tile_index(b, base + i * TMIN))] = x[i];
      }
    }
  }
}

// Forward passes P .. npass-1; the last one stores to global.
template <int LOG_S, int P, bool LAZY, int OUT, class Tile>
__device__ __forceinline__ void fwd_passes(u64* sm, const Tile& tl, u64* gout,
                                           const DevChain& ch) {
  constexpr int NP = npass(LOG_S);
  if constexpr (P < NP) {
    constexpr bool last = (P == NP - 1);
    run_pass<LOG_S, pass_r0(LOG_S, P), pass_e(LOG_S, P), true, LAZY, last, OUT>(sm, tl, gout,
                                                                                ch);
    if constexpr (!last) {
      __syncthreads();
      fwd_passes<LOG_S, P + 1, LAZY, OUT>(sm, tl, gout, ch);
    }
  }
}

// Inverse passes P .. 0 (reverse order); pass 0 stores to global.
template <int LOG_S, int P, class Tile>
__device__ __forceinline__ void inv_passes(u64* sm, const Tile& tl, u64* gout,
                                           const DevChain& ch) {
  if constexpr (P >= 0) {
    constexpr bool last = (P == 0);
    run_pass<LOG_S, pass_r0(LOG_S, P), pass_e(LOG_S, P), false, false, last, OUT_RAW>(sm, tl,
                                                                                      gout, ch);
    if constexpr (!last) {
      __syncthreads();
      inv_passes<LOG_S, P - 1>(sm, tl, gout, ch);
    }
  }
}


// ---------------------------------------------------------------------------
// FP64-pipe transform for chains with every prime < 2^50.
//
// The integer butterfly is bound by the quarter-rate IMAD.WIDE (64-bit
// products); B200's FP64 pipe runs DFMA at half rate.  Values are held as
// doubles carrying signed integer representatives |x| <= q and the Shoup
// product is done with an error-free FMA split:
//   h = x w, l = fma(x, w, -h)            (x w = h + l exactly)
//   k = rint(x * (w/q))                   (magic-constant rounding, |x w/q| < 2^51)
//   t = fma(-k, q, h) + l                 (= x w - k q exactly, |t| <= q/2 + eps)
// so every value is an exact integer and the canonical outputs are the same
// bits as the integer path.
enum FpIn { FPIN_DOUBLE = 0, FPIN_U64 = 1 };
enum FpOut { FPOUT_DOUBLE = 0, FPOUT_U64 = 1 };

template <int LOG_S, int R0, int E_LOG, bool FWD, bool FIRST, bool LAST, int IN, int OUT,
          bool STW, class Tile>
__device__ __forceinline__ void run_pass_fp(u64* sm, const double2* tws, const Tile& tl,
                                            u64* gout, const DevChain& ch) {
  constexpr int E = 1 << E_LOG;
  constexpr int T0 = (1 << LOG_S) >> (R0 + 1);
  constexpr int TMIN_LOG = LOG_S - R0 - E_LOG;
  constexpr int TMIN = 1 << TMIN_LOG;
  constexpr int GPA_LOG = LOG_S - E_LOG;
  constexpr bool VEC = (TMIN_LOG == 0) && !Tile::COLS && E >= 2;
  constexpr int PSTEP = Tile::DENSE ? (Tile::COLS ? TMIN << Tile::LOG_CN_OR0 : TMIN)
                                    : pad_step(Tile::COLS ? (1 << Tile::LOG_CN_OR0) : 0, TMIN, E);
  // twiddles of the whole pass are loaded up front (E - 1 pairs) when they
  // fit the register budget, so their L1/L2 latency overlaps the tile reads
  constexpr bool PRELOAD = !STW && E <= 16;
  // results of the last pass go back to shared memory and leave in 16-byte
  // coalesced stores (no strided 8-byte STGs from the butterfly registers)
  constexpr bool EPI = Tile::EPI;
  constexpr bool WL = warp_local(LOG_S) && !Tile::LANE_MAJOR;
  // staged twiddles of the last pass are stored transposed (staged_perm)
  constexpr bool TT = STW && R0 == pass_r0(LOG_S, npass(LOG_S) - 1) && TMIN_LOG == 0;
  const int total = tl.arrays() << GPA_LOG;
  for (int G = threadIdx.x; G < total; G += blockDim.x) {
    int b, g;
    tl.split(G, GPA_LOG, b, g);
    const int hi = g >> TMIN_LOG;
    const int lo = g & (TMIN - 1);
    const int base = hi * 2 * T0 + lo;
    const int pb = Tile::pad(tl.tile_index(b, base));
    const ArrCtx cx = tl.ctx(b, ch);
    const double2 qd = __ldg(&ch.qd[cx.prime]);
    const double2* tw = (FWD ? ch.twd : ch.itwd) + ((size_t)cx.prime << ch.log_n);
    double2 wt[PRELOAD ? E - 1 : 1];
    if (PRELOAD) {
#pragma unroll
      for (int rr = 0; rr < E_LOG; ++rr) {
        const double2* twr = tw + (cx.m0 << (R0 + rr)) + (hi << rr);
#pragma unroll
        for (int blk = 0; blk < (1 << rr); ++blk) wt[(1 << rr) - 1 + blk] = __ldg(twr + blk);
      }
    }
    u64 raw[E];
    // 128B-swizzled tiles (TMA chunk tiles, S = 256, radix 16): element t
    // sits at word t ^ (((t >> 4) & 7) << 1).  Contiguous groups are one
    // 128-byte row (pair j at unit j ^ row); stride-16 groups take one word
    // per row, whose xor offset only depends on i & 7 (8 base addresses).
    const int lin = tl.tile_index(b, base);
    int swz_off[Tile::SWZ && TMIN_LOG != 0 ? 8 : 1];
    if constexpr (Tile::SWZ && TMIN_LOG != 0) {
      static_assert(TMIN == 16, "swizzled tiles: stride-16 or contiguous groups only");
#pragma unroll
      for (int c = 0; c < 8; ++c) swz_off[c] = (lin & ~14) + ((lin & 14) ^ (c << 1));
    }
    if constexpr (Tile::SWZ && TMIN_LOG == 0) {
      const int r7 = (lin >> 4) & 7;
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(
            &sm[(lin & ~15) + ((i & ~15) << 0) + ((((i & 15) >> 1) ^ r7) << 1)]);
        raw[i] = v.x;
        raw[i + 1] = v.y;
      }
    } else if constexpr (Tile::SWZ) {
#pragma unroll
      for (int i = 0; i < E; ++i) raw[i] = sm[swz_off[i & 7] + 16 * i];
    } else if (VEC) {
#pragma unroll
      for (int i = 0; i < E; i += 2) {
        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(&sm[pb + i + ((i >> 4) << 1)]);
        raw[i] = v.x;
        raw[i + 1] = v.y;
      }
    } else if (PSTEP) {
#pragma unroll
      for (int i = 0; i < E; ++i) raw[i] = sm[pb + i * PSTEP];
    } else {
#pragma unroll
      for (int i = 0; i < E; ++i) raw[i] = sm[Tile::pad(tl.tile_index(b, base + i * TMIN))];
    }
    double x[E];
#pragma unroll
    for (int i = 0; i < E; ++i)
      x[i] = (FIRST && IN == FPIN_U64) ? fp_from_u52(raw[i]) : __longlong_as_double((long long)raw[i]);
#ifdef FHE_NTT_NOCOMPUTE
    if (false) {
#else
    if (FWD) {
#endif
#pragma unroll
      for (int rr = 0; rr < E_LOG; ++rr) {
        const int half = E >> (rr + 1);
        const double2* twr = TT ? tws + tl.tw_base(R0 + rr, cx.m0) + hi
                             : STW ? tws + tl.tw_base(R0 + rr, cx.m0) + (hi << rr)
                                   : tw + (cx.m0 << (R0 + rr)) + (hi << rr);
#pragma unroll
        for (int blk = 0; blk < (1 << rr); ++blk) {
          const double2 w = PRELOAD ? wt[(1 << rr) - 1 + blk] : (STW ? twr[TT ? (blk << R0) : blk] : __ldg(twr + blk));
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const int a = blk * 2 * half + i, c = a + half;
            // signed twiddles take |x| < 2^52 = 4q; bounds grow by 0.75q per
            // stage from <= 1.25q, so u is reduced on every 4th global stage
            const double u = ((Tile::GS0 + R0 + rr) & 3) == 3 ? fp_reduce(x[a], qd) : x[a];
            const double t = fp_mulmod(x[c], w, qd.x);
            x[a] = __dadd_rn(u, t);
            x[c] = __dadd_rn(u, -t);
          }
        }
      }
    } else if (!NOCOMP) {
#pragma unroll
      for (int rr = E_LOG - 1; rr >= 0; --rr) {
        const int half = E >> (rr + 1);
        const bool fold = (R0 == 0) && (rr == 0) && cx.fold;
        const double2* twr = TT ? tws + tl.tw_base(R0 + rr, cx.m0) + hi
                             : STW ? tws + tl.tw_base(R0 + rr, cx.m0) + (hi << rr)
                                   : tw + (cx.m0 << (R0 + rr)) + (hi << rr);
#pragma unroll
        for (int blk = 0; blk < (1 << rr); ++blk) {
          const double2 w = fold ? __ldg(&ch.ninv_w1_d[cx.prime])
                                 : (PRELOAD ? wt[(1 << rr) - 1 + blk]
                                            : (STW ? twr[TT ? (blk << R0) : blk] : __ldg(twr + blk)));
          const double2 sn = fold ? __ldg(&ch.ninv_d[cx.prime]) : w;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const int a = blk * 2 * half + i, c = a + half;
            const double s = __dadd_rn(x[a], x[c]);
            const double d = __dadd_rn(x[a], -x[c]);
            // sums double per stage: reduced on even global stages, so the
            // difference fed to the mulmod stays below 4 * 0.75q < 2^52
            x[a] = fold ? fp_mulmod(s, sn, qd.x)
                        : (((Tile::GS0 + R0 + rr) & 1) == 0 ? fp_reduce(s, qd) : s);
            x[c] = fp_mulmod(d, w, qd.x);
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < E; ++i)
      raw[i] = (LAST && OUT == FPOUT_U64) ? fp_canon_half(FWD ? fp_reduce(x[i], qd) : x[i], qd.x)
                                          : (u64)__double_as_longlong(x[i]);
    if (LAST && !EPI) {
      u64* o = tl.gdst(gout, b, base);
      if (VEC) {
#pragma unroll
        for (int i = 0; i < E; i += 2)
          *reinterpret_cast<ulonglong2*>(o + i) = make_ulonglong2(raw[i], raw[i + 1]);
      } else {
        constexpr long GSTEP = Tile::GSTEP_PER_K * TMIN;
#pragma unroll
        for (int i = 0; i < E; ++i) o[i * GSTEP] = raw[i];
      }
    } else {
      if constexpr (Tile::SWZ && TMIN_LOG == 0) {
        const int r7 = (lin >> 4) & 7;
#pragma unroll
        for (int i = 0; i < E; i += 2)
          *reinterpret_cast<ulonglong2*>(
              &sm[(lin & ~15) + (i & ~15) + ((((i & 15) >> 1) ^ r7) << 1)]) =
              make_ulonglong2(raw[i], raw[i + 1]);
      } else if constexpr (Tile::SWZ) {
#pragma unroll
        for (int i = 0; i < E; ++i) sm[swz_off[i & 7] + 16 * i] = raw[i];
      } else if (VEC) {
#pragma unroll
        for (int i = 0; i < E; i += 2)
          *reinterpret_cast<ulonglong2*>(&sm[pb + i + ((i >> 4) << 1)]) = make_ulonglong2(raw[i], raw[i + 1]);
      } else if (PSTEP) {
#pragma unroll
        for (int i = 0; i < E; ++i) sm[pb + i * PSTEP] = raw[i];
      } else {
#pragma unroll
        for (int i = 0; i < E; ++i) sm[Tile::pad(tl.tile_index(b, base + i * TMIN))] = raw[i];
      }
    }
  }
  if (LAST && EPI) epilogue_store<Tile, GPA_LOG, WL>(sm, tl, gout, ch);
}

template <int LOG_S, int P, int IN, int OUT, bool STW, class Tile>
__device__ __forceinline__ void fwd_passes_fp(u64* sm, const double2* tws, const Tile& tl,
                                              u64* gout, const DevChain& ch) {
  constexpr int NP = npass(LOG_S);
  if constexpr (P < NP) {
    constexpr bool last = (P == NP - 1);
    run_pass_fp<LOG_S, pass_r0(LOG_S, P), pass_e(LOG_S, P), true, P == 0, last, IN, OUT, STW>(
        sm, tws, tl, gout, ch);
    if constexpr (!last) {
      if constexpr (warp_local(LOG_S) && !Tile::LANE_MAJOR) __syncwarp(); else __syncthreads();
      fwd_passes_fp<LOG_S, P + 1, IN, OUT, STW>(sm, tws, tl, gout, ch);
    }
  }
}

template <int LOG_S, int P, int IN, int OUT, bool STW, class Tile>
__device__ __forceinline__ void inv_passes_fp(u64* sm, const double2* tws, const Tile& tl,
                                              u64* gout, const DevChain& ch) {
  if constexpr (P >= 0) {
    constexpr bool last = (P == 0);
    run_pass_fp<LOG_S, pass_r0(LOG_S, P), pass_e(LOG_S, P), false, P == npass(LOG_S) - 1, last,
                IN, OUT, STW>(sm, tws, tl, gout, ch);
    if constexpr (!last) {
      if constexpr (warp_local(LOG_S) && !Tile::LANE_MAJOR) __syncwarp(); else __syncthreads();
      inv_passes_fp<LOG_S, P - 1, IN, OUT, STW>(sm, tws, tl, gout, ch);
    }
  }
}

// Stage the tile's twiddle pairs in shared memory (one contiguous block of
// the staged table; cp.async, committed with the tile's data group).
template <class Tile>
__device__ __forceinline__ void load_tw(double2* tws, const Tile& tl, const double2* table) {
  const double2* g = table + tl.tw_src_off();
  for (int j = threadIdx.x; j < tl.tw_pairs(); j += Tile::THREADS) cp_async16(&tws[j], &g[j]);
}

// Issue the cp.async copies of one tile (16 bytes per copy).  Each thread
// copies fixed (column pair | array offset) positions, so the per-copy
// address arithmetic reduces to constant strides.
template <class Tile>
__device__ __forceinline__ void load_tile(u64* sm, const Tile& tl, const u64* src) {
  constexpr int LOG_S = Tile::LOG_S;
  constexpr int S = 1 << LOG_S;
  constexpr int T = Tile::THREADS;
  if constexpr (Tile::COLS) {
    constexpr int CN = 1 << Tile::LOG_CN_OR0;
    constexpr int PPR = CN / 2;       // pairs per k-row
    constexpr int KSTEP = T / PPR;    // k-rows per sweep of the CTA
    const int k0 = threadIdx.x / PPR, c = (threadIdx.x % PPR) * 2;
    const u64* g = tl.gsrc(src, c, k0);
    if constexpr (KSTEP % 16 == 0) {
      u64* s = sm + Tile::pad(k0 * CN + c);
#pragma unroll
      for (int j = 0; j < S / KSTEP; ++j)
        cp_async16(s + j * (KSTEP * (CN + 2) + 2 * (KSTEP / 16)), g + (long)j * KSTEP * Tile::N2);
    } else {
#pragma unroll
      for (int j = 0; j < S / KSTEP; ++j)
        cp_async16(&sm[Tile::pad((k0 + j * KSTEP) * CN + c)], g + (long)j * KSTEP * Tile::N2);
    }
  } else {
    constexpr int PPA = S / 2;  // pairs per array
    if constexpr (PPA <= T) {
      constexpr int APJ = T / PPA;
      const int k = (threadIdx.x % PPA) * 2;
      for (int b = threadIdx.x / PPA; b < tl.arrays(); b += APJ)
        cp_async16(&sm[Tile::pad((b << LOG_S) + k)], tl.gsrc(src, b, k));
    } else {
      for (int b = 0; b < tl.arrays(); ++b)
#pragma unroll 4
        for (int k = 2 * threadIdx.x; k < S; k += 2 * T)
          cp_async16(&sm[Tile::pad((b << LOG_S) + k)], tl.gsrc(src, b, k));
    }
  }
  cp_async_commit();
}

// Persistent, double-buffered transform kernel over the tiles of one policy.
template <class Tile, bool FWD, bool LAZY, int OUT>
__global__ void __launch_bounds__(Tile::THREADS, Tile::MINB)
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
        inv_passes_fp<Tile::LOG_S, npass(Tile::LOG_S) - 1, IN, OUT, STW>(smem_raw, tw_raw, cur,
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
        inv_passes_fp<Tile::LOG_S, npass(Tile::LOG_S) - 1, IN, OUT, STW>(sm, tws, cur, dst, ch);
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
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, int c4, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                             int c4, const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4, %5}], [%6];" ::
          "l"(map),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(src))
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            int c2, int c3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, int c0, int c1, int c2,
                                             int c3, const void* src) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::
          "l"(map),
      "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src))
      : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait0() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

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
  __device__ __forceinline__ void setup(int t) {
    Base::setup(t);
    ccol = this->j0 >> 4;
    climb = this->row % this->map.limbs;
    cbat = this->row / this->map.limbs;
  }
  __device__ __forceinline__ void tma_load(u64* sm, uint64_t* bar) const {
    tma_load_5d(sm, smap_p, 0, ccol, 0, climb, cbat, bar);
  }
  __device__ __forceinline__ void tma_store(const u64* sm) const {
    tma_store_5d(dmap_p, 0, ccol, 0, climb, cbat, sm);
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
  __device__ __forceinline__ void tma_load(u64* sm, uint64_t* bar) const {
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
      inv_passes_fp<Tile::LOG_S, npass(Tile::LOG_S) - 1, IN, OUT, true>(sm, tws, cur, nullptr,
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
#ifndef FHE_FUSE_MIN_LOG_R
#define FHE_FUSE_MIN_LOG_R 4
#endif
#ifndef FHE_FUSE_LAG
#define FHE_FUSE_LAG 4
#endif
constexpr int kFuseLag = FHE_FUSE_LAG;
constexpr int kFuseSlabs = 8;

struct FusePlan {
  int groups;     // row groups (residue class x row block)
  int rblocks;    // row blocks per class
  int log_r;      // rows per group = 1 << log_r
  int c_per_g;    // column tiles per group = R * C::TILES
  int k_per_g;    // chunk tiles per group = cblocks
  int total;      // tickets
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
    inv_passes_fp<Tile::LOG_S, npass(Tile::LOG_S) - 1, Tile::COLS ? FPIN_DOUBLE : FPIN_U64,
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
    const int g = first ? blk : blk - kFuseLag;
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
__global__ void __launch_bounds__(kSplitThreads, 5)
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
    const int g = first ? blk : blk - kFuseLag;
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
            inv_passes_fp<CT::LOG_S, npass(CT::LOG_S) - 1, FPIN_DOUBLE, FPOUT_U64, true>(
                sm, tws, c, nullptr, ch);
          work = true;
        }
      } else {
        KT k = kt;
        k.smap_p = &ks_map;
        k.dmap_p = &kd_map;
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
            inv_passes_fp<KT::LOG_S, npass(KT::LOG_S) - 1, FPIN_U64, FPOUT_DOUBLE, true>(
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
  const int grid = std::min(ntiles, Tile::MINB * sm_count());
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
  ntt_tiles_fp_kernel<Tile, FWD, IN, OUT, STW><<<grid, Tile::THREADS, smem, st>>>(ch, dst, src, tl,
                                                                            ntiles);
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
  fp.total = (fp.groups + kFuseLag) * (fp.c_per_g + fp.k_per_g);
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
                     cudaStream_t st, bool& done) {
  done = false;
  const int log_c = kChunkLogTile - KT::LOG_S - kt.log_r;
  // forward: columns read src, chunks work in place on dst; inverse: chunks
  // read src, columns work in place on dst
  CUtensorMap cs, cd, ks, kd;
  const u64* col_src = fwd ? src : dst;
  const u64* chk_src = fwd ? dst : src;
  const long col_sb = fwd ? src_bstride : dst_bstride, chk_sb = fwd ? dst_bstride : src_bstride;
  if (!cols_tensor_map(&cs, col_src, ch.log_n, CT::LOG_S, limbs, col_sb, rows) ||
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
  const int grid = std::min(fp.total, 5 * sm_count());
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
  if (!cols_tensor_map(&smap, src, ch.log_n, Tile::LOG_S, tl.map.limbs, src_bstride, tl.rows) ||
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
  if constexpr (LOG_N1 == 8 && LOG_N - LOG_N1 == 8) {
    // fused only for 16-row groups (one chunk per tile): measured faster
    // there (5120-row sweep +3-6%), slower for 8-row groups (key-switch ModUp)
    if (use_tma && use_ktma && ch.fuse && fused_tma_enabled() && kt.log_r >= FHE_FUSE_MIN_LOG_R &&
        !a.fin) {
      ColsTmaTile<LOG_N, LOG_N1> tc;
      static_cast<C&>(tc) = ct;
      tc.src = inverse ? d : s;
      tc.dst = d;
      ChunksTmaTile<LOG_N, LOG_N1> tk;
      static_cast<K&>(tk) = kt;
      tk.src = inverse ? s : d;
      tk.dst = d;
      bool done = false;
      rc = launch_fused_tma(ch, a.dst, a.src, tc, tk, !inverse, a.src_bstride, a.dst_bstride,
                            a.rows, a.map.limbs, st, done);
      if (rc || done) return rc;
    }
  }
  if (C::THREADS == K::THREADS && ch.fp64_ok && kstage && ch.fuse && fused_enabled() && !a.fin) {
    ct.src = inverse ? d : s;
    ct.dst = d;
    kt.src = inverse ? s : d;
    kt.dst = d;
    return launch_fused(ch, a.dst, a.src, ct, kt, !inverse, a.rows, a.map.limbs, st);
  }
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

int launch_ntt(const DevChain& ch, const NttArgs& a, bool inverse, cudaStream_t st) {
  if (a.rows <= 0) return 0;
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

void* fuse_scratch_new() { return new FuseScratch(); }

void fuse_scratch_free(void* p) {
  FuseScratch* fs = static_cast<FuseScratch*>(p);
  if (!fs) return;
  for (cudaEvent_t& e : fs->ev)
    if (e) cudaEventDestroy(e);
  if (fs->dev) cudaFree(fs->dev);
  delete fs;
}

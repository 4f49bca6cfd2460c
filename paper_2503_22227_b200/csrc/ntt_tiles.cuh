// Tile policies and register-pass machinery of the batched NTT (ntt.cu).
// Included by ntt.cu inside its anonymous namespace; not a standalone header.
#pragma once


// Tile geometry.  Whole-row tiles: 4096 elements, 256 threads, 2 CTAs/SM.
// Split (four-step) tiles: 2048 elements, 128 threads, 4 CTAs/SM -- small
// CTAs keep the SM's FP64 pipe fed while other CTAs sit in their load /
// barrier / store phases.
#include <type_traits>

#ifndef FHE_ROW_THREADS
#define FHE_ROW_THREADS 256
#endif
constexpr int kRowThreads = FHE_ROW_THREADS;
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
  static constexpr int MAXE = FHE_ROW_MAXE;  // pass radix limit (tile_maxe)
  double center = 0.0;    // != 0: centred broadcast input (NttArgs::center_q)
  int bcast_limbs = 0;    // != 0: input row r is row r / bcast_limbs of src
  long bcast_stride = 0;  //        (bcast_stride words apart)
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
    if (bcast_limbs) return base + (long)((row0 + b) / bcast_limbs) * bcast_stride + k;
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
  // one row per tile (N = 2^12): the prime's whole staged table (S pairs, in
  // the row plan's staged_perm order, context.cu) can be staged in shared
  // memory with the row, so no pass waits on an L2 twiddle read (STW launch);
  // several rows per tile may use different primes: twiddles through L1
  static constexpr int TWMAX = NB == 1 ? S : 0;
  __device__ __forceinline__ int tw_pairs() const { return NB == 1 ? S : 0; }
  __device__ __forceinline__ long tw_src_off() const { return 0; }
  __device__ __forceinline__ int tw_base(int s, int) const { return 1 << s; }
  __device__ __forceinline__ int tw_prime() const { return prime[0]; }
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
  double center = 0.0;  // != 0: input values are centred about this modulus (NttArgs::center_q)
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
  static constexpr double center = 0.0;
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
  int plan(int rows_, int limbs, int max_log_r = 30) {
    const int rpc = (rows_ + limbs - 1) / limbs;
    log_r = 0;
    while ((2 << log_r) <= NB && (2 << log_r) <= rpc && log_r < max_log_r) ++log_r;
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
constexpr bool warp_local(int log_s, int maxe = FHE_NTT_MAXE) {
  for (int p = 1; p < npass(log_s, maxe); ++p)
    if (pass_e(log_s, p, maxe) != pass_e(log_s, 0, maxe)) return false;
  return log_s - pass_e(log_s, 0, maxe) <= 5;
}

// Pass radix limit of a tile type: Tile::MAXE when it declares one (the
// latency-mode row tiles use smaller radices and more threads), else
// FHE_NTT_MAXE.  FP64 passes only.
template <class T, class = void>
struct tile_maxe {
  static constexpr int v = FHE_NTT_MAXE;
};
template <class T>
struct tile_maxe<T, std::void_t<decltype(T::MAXE)>> {
  static constexpr int v = T::MAXE;
};

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
  constexpr int MX = tile_maxe<Tile>::v;
  constexpr bool WL = warp_local(LOG_S, MX) && !Tile::LANE_MAJOR;
  // staged twiddles of the last pass are stored transposed (staged_perm)
  constexpr bool TT = STW && R0 == pass_r0(LOG_S, npass(LOG_S, MX) - 1, MX) && TMIN_LOG == 0;
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
    if constexpr (FIRST && IN == FPIN_U64) {
      // centred broadcast input (rescale): the signed representative itself
      if (tl.center != 0.0) {
        const double hq = 0.5 * tl.center;
#pragma unroll
        for (int i = 0; i < E; ++i) x[i] = x[i] > hq ? __dadd_rn(x[i], -tl.center) : x[i];
      }
    }
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
  constexpr int MX = tile_maxe<Tile>::v;
  constexpr int NP = npass(LOG_S, MX);
  if constexpr (P < NP) {
    constexpr bool last = (P == NP - 1);
    run_pass_fp<LOG_S, pass_r0(LOG_S, P, MX), pass_e(LOG_S, P, MX), true, P == 0, last, IN, OUT,
                STW>(sm, tws, tl, gout, ch);
    if constexpr (!last) {
      if constexpr (warp_local(LOG_S, MX) && !Tile::LANE_MAJOR) __syncwarp(); else __syncthreads();
      fwd_passes_fp<LOG_S, P + 1, IN, OUT, STW>(sm, tws, tl, gout, ch);
    }
  }
}

template <int LOG_S, int P, int IN, int OUT, bool STW, class Tile>
__device__ __forceinline__ void inv_passes_fp(u64* sm, const double2* tws, const Tile& tl,
                                              u64* gout, const DevChain& ch) {
  constexpr int MX = tile_maxe<Tile>::v;
  if constexpr (P >= 0) {
    constexpr bool last = (P == 0);
    run_pass_fp<LOG_S, pass_r0(LOG_S, P, MX), pass_e(LOG_S, P, MX), false,
                P == npass(LOG_S, MX) - 1, last, IN, OUT, STW>(sm, tws, tl, gout, ch);
    if constexpr (!last) {
      if constexpr (warp_local(LOG_S, MX) && !Tile::LANE_MAJOR) __syncwarp(); else __syncthreads();
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


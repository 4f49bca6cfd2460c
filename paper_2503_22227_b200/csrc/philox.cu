// Device sampler replaying numpy's Generator(Philox(SeedSequence(seed)))
// stream bit-exactly (SURVEY.md 8(f)1 phase 2): the reference samples keys
// and noise through rnsfhe/coremath/sampling.py:27-63 with
//   integers(0, q, n, uint64)        64-bit bounded Lemire (uniform residues)
//   integers(-1, 2, n, int64)        32-bit bounded Lemire (ternary)
//   integers(0, 2, (40, n), int64)   32-bit bounded Lemire (CBD coin flips)
// Algorithms (numpy 2.3.5, restated and pinned in oracle/philox.py): Philox
// 4x64-10; next_uint64 serves a 4-word buffer and refills it after
// incrementing the 256-bit counter; next_uint32 serves the low half of a
// 64-bit draw and keeps the high half; Lemire: m = draw * (rng + 1), reject
// while the low part is below (MAX - rng) % (rng + 1).
//
// The generator state lives in device memory (FhePhilox), so consecutive
// draws chain on the stream without a host round trip.  Philox is counter
// based, so draw i of a call is computed independently: pass 1 evaluates
// C >= count candidate draws and their accept flags (per-CTA counts), pass 2
// scans the CTA counts, pass 3 scatters the accepted values to their ranks
// and the thread holding the last accepted draw writes the new state
// (counter, buffer, positions: the state numpy would hold after the call).
#include "fhe_kernels.cuh"

#include <algorithm>
#include <cmath>

namespace {

constexpr int kPxThreads = 256;
constexpr u64 kM0 = 0xD2E7470EE14C6C93ull, kM1 = 0xCA5A826395121157ull;
constexpr u64 kW0 = 0x9E3779B97F4A7C15ull, kW1 = 0xBB67AE8584CAA73Bull;

struct Ctr4 {
  u64 v[4];
};

__device__ __forceinline__ Ctr4 philox10(Ctr4 c, u64 k0, u64 k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += kW0;
      k1 += kW1;
    }
    const u64 hi0 = __umul64hi(kM0, c.v[0]), lo0 = kM0 * c.v[0];
    const u64 hi1 = __umul64hi(kM1, c.v[2]), lo1 = kM1 * c.v[2];
    c = Ctr4{{hi1 ^ c.v[1] ^ k0, lo1, hi0 ^ c.v[3] ^ k1, lo0}};
  }
  return c;
}

// counter + add (256-bit)
__device__ __forceinline__ Ctr4 ctr_add(const u64* ctr, u64 add) {
  Ctr4 c;
  u64 carry = add;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const u64 s = ctr[i] + carry;
    carry = (s < carry) ? 1 : 0;
    c.v[i] = s;
  }
  return c;
}

// 64-bit draw d of the stream that starts at state st
__device__ __forceinline__ u64 draw64(const FhePhilox& st, long d) {
  const long avail = 4 - (long)st.buffer_pos;
  if (d < avail) return st.buffer[st.buffer_pos + d];
  const long e = d - avail;
  const Ctr4 c = philox10(ctr_add(st.counter, (u64)(e >> 2) + 1), st.key[0], st.key[1]);
  return c.v[e & 3];
}

// 32-bit draw u of the stream (the buffered high half first)
__device__ __forceinline__ u32 draw32(const FhePhilox& st, long u) {
  if (st.has_uint32) {
    if (u == 0) return st.uinteger;
    --u;
  }
  const u64 v = draw64(st, u >> 1);
  return (u & 1) ? (u32)(v >> 32) : (u32)v;
}

// pass 1: candidate draws, accept flags and per-CTA accept counts
template <bool B64>
__global__ void __launch_bounds__(kPxThreads)
    philox_draw_kernel(const FhePhilox* __restrict__ stp, u64 rng, u64 thr, long cand,
                       u64* __restrict__ vals, unsigned char* __restrict__ acc,
                       int* __restrict__ block_cnt) {
  const FhePhilox st = *stp;
  const long d = blockIdx.x * (long)blockDim.x + threadIdx.x;
  int ok = 0;
  if (d < cand) {
    const u64 excl = rng + 1;
    u64 hi, lo;
    if (B64) {
      const u64 x = draw64(st, d);
      lo = x * excl;
      hi = __umul64hi(x, excl);
    } else {
      const u64 m = (u64)draw32(st, d) * excl;
      lo = m & 0xffffffffull;
      hi = m >> 32;
    }
    // Lemire: a low part below the threshold is resampled (only possible
    // when it is below rng + 1); rng == MAX32 takes the raw 32-bit draw
    ok = (lo >= excl || lo >= thr) ? 1 : 0;
    vals[d] = hi;
    acc[d] = (unsigned char)ok;
  }
  const int cnt = __syncthreads_count(ok);
  if (threadIdx.x == 0) block_cnt[blockIdx.x] = cnt;
}

// pass 2: exclusive scan of the per-CTA counts (one CTA)
__global__ void __launch_bounds__(1024) philox_scan_kernel(int* __restrict__ block_cnt, int nb) {
  __shared__ int part[1024];
  const int per = (nb + blockDim.x - 1) / blockDim.x;
  const int b0 = threadIdx.x * per;
  int s = 0;
  for (int i = 0; i < per && b0 + i < nb; ++i) s += block_cnt[b0 + i];
  part[threadIdx.x] = s;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {
    const int v = threadIdx.x >= (unsigned)off ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int i = 0; i < per && b0 + i < nb; ++i) {
    const int c = block_cnt[b0 + i];
    block_cnt[b0 + i] = run;
    run += c;
  }
  if (threadIdx.x == blockDim.x - 1) block_cnt[nb] = part[blockDim.x - 1];  // total
}

// state after consuming `used` units (64-bit draws, or 32-bit halves when !B64)
template <bool B64>
__device__ void advance(FhePhilox& st, long used) {
  long d64 = used;
  if (!B64) {
    long u = used;
    if (st.has_uint32 && u > 0) {
      st.has_uint32 = 0;
      --u;
    }
    d64 = (u + 1) >> 1;
    if (u & 1) {
      st.has_uint32 = 1;
      st.uinteger = (u32)(draw64(st, d64 - 1) >> 32);
    }
  }
  const long avail = 4 - (long)st.buffer_pos;
  if (d64 <= avail) {
    st.buffer_pos += (int)d64;
    return;
  }
  const long e = d64 - avail;
  const long blocks = (e + 3) >> 2;
  const Ctr4 c = ctr_add(st.counter, (u64)blocks);
  const Ctr4 buf = philox10(c, st.key[0], st.key[1]);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    st.counter[i] = c.v[i];
    st.buffer[i] = buf.v[i];
  }
  st.buffer_pos = (int)(e - 4 * (blocks - 1));
}

// pass 3: scatter accepted draws to their ranks; the last one updates the state
template <bool B64>
__global__ void __launch_bounds__(kPxThreads)
    philox_scatter_kernel(FhePhilox* __restrict__ stp, u64 off, long count, long cand,
                          const u64* __restrict__ vals, const unsigned char* __restrict__ acc,
                          const int* __restrict__ block_off, u64* __restrict__ out) {
  __shared__ int warp_base[kPxThreads / 32];
  const long d = blockIdx.x * (long)blockDim.x + threadIdx.x;
  const int ok = (d < cand) ? acc[d] : 0;
  const unsigned lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  if (lane == 0) warp_base[wid] = __popc(bal);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int w = 0; w < kPxThreads / 32; ++w) {
      const int c = warp_base[w];
      warp_base[w] = run;
      run += c;
    }
  }
  __syncthreads();
  if (!ok) return;
  const long rank = block_off[blockIdx.x] + warp_base[wid] + __popc(bal & ((1u << lane) - 1));
  if (rank < count) out[rank] = off + vals[d];
  if (rank == count - 1) {
    FhePhilox st = *stp;
    advance<B64>(st, d + 1);
    st.shortfall = 0;
    *stp = st;
  }
}

__global__ void philox_flag_kernel(FhePhilox* stp, const int* total, long count) {
  // a call whose candidates held fewer than `count` accepted draws leaves the
  // state untouched and raises the flag (the host retries with more)
  if (*total < count) stp->shortfall = 1;
}

// CBD noise from the coin-flip block (sampling.py cbd_error): out[i] =
// sum of the first `pairs` flip rows minus the sum of the next `pairs` rows
__global__ void cbd_combine_kernel(long long* __restrict__ out, const u64* __restrict__ flips,
                                   int pairs, long n) {
  for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n;
       i += (long)gridDim.x * blockDim.x) {
    long long s = 0;
    for (int r = 0; r < pairs; ++r) s += (long long)flips[(long)r * n + i];
    for (int r = 0; r < pairs; ++r) s -= (long long)flips[(long)(pairs + r) * n + i];
    out[i] = s;
  }
}

// small signed coefficients -> residue rows (sampling.py signed_to_residues):
// row j = c mod q_(offset + j), canonical
__global__ void signed_lift_kernel(const DevChain ch, u64* __restrict__ out,
                                   const long long* __restrict__ c, long n, int limbs, int offset) {
  const long total = n * limbs;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int j = (int)(t / n);
    const long i = t - (long)j * n;
    const u64 q = ch.mc[offset + j].q;
    const long long v = c[i];
    const u64 m = (u64)(v < 0 ? -v : v) % q;
    out[t] = (v < 0 && m) ? q - m : m;
  }
}

// Integer-valued doubles (CKKS encode: the rounded scaled coefficients,
// any magnitude up to the modulus budget) -> residue rows: v = m 2^e exactly
// (m the 53-bit significand), so [v]_q = [m]_q [2^e]_q, negated for v < 0 --
// the residues the reference computes with Python integers
// (ckks.py:104-136) without leaving the device.
__global__ void real_lift_kernel(const DevChain ch, u64* __restrict__ out,
                                 const double* __restrict__ v, long n, int limbs, int offset) {
  const long total = n * limbs;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const int j = (int)(t / n);
    const long i = t - (long)j * n;
    const ModConst mc = ch.mc[offset + j];
    const u64 q = mc.q;
    const double x = v[i];
    const u64 bits = (u64)__double_as_longlong(x);
    const bool neg = bits >> 63;
    const int be = (int)((bits >> 52) & 0x7ff);
    u64 r;
    if (be == 0) {
      r = 0;  // +-0 (subnormals cannot be integer-valued)
    } else {
      const u64 m = (bits & 0xfffffffffffffull) | (1ull << 52);
      const int e = be - 1075;  // x = m 2^e
      if (e <= 0) {
        r = (m >> (-e)) % q;  // an integer below 2^53
      } else {
        u64 p = 1 % q, b = 2 % q;
        for (int k = e; k; k >>= 1) {  // 2^e mod q
          if (k & 1) p = mul_mod(p, b, mc);
          b = mul_mod(b, b, mc);
        }
        r = mul_mod(m % q, p, mc);
      }
    }
    out[t] = (neg && r) ? q - r : r;
  }
}

}  // namespace

int run_real_lift(const DevChain& ch, u64* out, const double* v, long n, int limbs, int offset,
                  cudaStream_t st) {
  if (n <= 0 || limbs <= 0) return 0;
  real_lift_kernel<<<grid_for(n * limbs), kPxThreads, 0, st>>>(ch, out, v, n, limbs, offset);
  FHE_LAUNCH_CHECK();
  return 0;
}

int run_cbd_combine(long long* out, const u64* flips, int pairs, long n, cudaStream_t st) {
  if (n <= 0) return 0;
  cbd_combine_kernel<<<grid_for(n), kPxThreads, 0, st>>>(out, flips, pairs, n);
  FHE_LAUNCH_CHECK();
  return 0;
}

int run_signed_lift(const DevChain& ch, u64* out, const long long* c, long n, int limbs,
                    int offset, cudaStream_t st) {
  if (n <= 0 || limbs <= 0) return 0;
  signed_lift_kernel<<<grid_for(n * limbs), kPxThreads, 0, st>>>(ch, out, c, n, limbs, offset);
  FHE_LAUNCH_CHECK();
  return 0;
}

// Candidate draws for `count` accepted values: the expected number of Lemire
// rejections (rate p = min(rng + 1, threshold) / 2^bits) plus eight standard
// deviations and 64 -- a shortfall is then far below 2^-40 per call.
static long philox_candidates(long count, unsigned long long rng) {
  const bool b64 = rng > 0xffffffffull;
  const u64 excl = rng + 1;
  const u64 thr = b64 ? (~0ull - rng) % excl
                      : (rng == 0xffffffffull ? 0 : (0xffffffffull - rng) % excl);
  const double p = (double)(thr < excl ? thr : excl) / (b64 ? 18446744073709551616.0 : 4294967296.0);
  const double extra = count * p / (1.0 - p);
  return count + 64 + (long)(extra + 8.0 * sqrt(extra + 1.0) + 1.0);
}

size_t philox_workspace(long count, unsigned long long rng) {
  const long cand = philox_candidates(count, rng);
  const long nb = (cand + kPxThreads - 1) / kPxThreads;
  return (size_t)cand * (sizeof(u64) + 1) + (size_t)(nb + 1) * sizeof(int) + 256;
}

int run_philox_integers(FhePhilox* dev_state, long long low, unsigned long long rng, long count,
                        u64* out, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (count <= 0) return 0;
  if (rng == 0) {
    fhe_set_error("philox: empty range (fill with low on the host)");
    return -1;
  }
  if (rng == ~0ull) {
    fhe_set_error("philox: full 64-bit range is not a bounded draw");
    return -1;
  }
  const bool b64 = rng > 0xffffffffull;
  // rejection threshold (MAX - rng) % (rng + 1); rng == MAX32 takes raw draws
  const u64 excl = rng + 1;
  const u64 thr = b64 ? (~0ull - rng) % excl : (rng == 0xffffffffull ? 0 : (0xffffffffull - rng) % excl);
  const long cand = philox_candidates(count, rng);
  const long nb = (cand + kPxThreads - 1) / kPxThreads;
  if (ws_bytes < philox_workspace(count, rng)) {
    fhe_set_error("philox: workspace too small");
    return -1;
  }
  if (nb > (1L << 20)) {
    fhe_set_error("philox: too many draws in one call");
    return -1;
  }
  unsigned char* base = (unsigned char*)ws;
  u64* vals = (u64*)base;
  int* bcnt = (int*)(base + cand * sizeof(u64));
  unsigned char* acc = (unsigned char*)(bcnt + nb + 1);
  if (b64) {
    philox_draw_kernel<true><<<(unsigned)nb, kPxThreads, 0, st>>>(dev_state, rng, thr, cand, vals,
                                                                  acc, bcnt);
  } else {
    philox_draw_kernel<false><<<(unsigned)nb, kPxThreads, 0, st>>>(dev_state, rng, thr, cand,
                                                                   vals, acc, bcnt);
  }
  FHE_LAUNCH_CHECK();
  philox_scan_kernel<<<1, 1024, 0, st>>>(bcnt, (int)nb);
  FHE_LAUNCH_CHECK();
  philox_flag_kernel<<<1, 1, 0, st>>>(dev_state, bcnt + nb, count);
  FHE_LAUNCH_CHECK();
  if (b64) {
    philox_scatter_kernel<true><<<(unsigned)nb, kPxThreads, 0, st>>>(
        dev_state, (u64)low, count, cand, vals, acc, bcnt, out);
  } else {
    philox_scatter_kernel<false><<<(unsigned)nb, kPxThreads, 0, st>>>(
        dev_state, (u64)low, count, cand, vals, acc, bcnt, out);
  }
  FHE_LAUNCH_CHECK();
  return 0;
}

// zlib-compatible CRC-32 of a device buffer, for the CATF wire records
// (reference serial.py:1-16, 67-78: crc32 over header + body, appended
// little-endian).  The body of a ciphertext or key record is its residue
// block, resident in HBM; checksumming it on the device lets a record be
// written straight from the D2H copy into a pinned buffer (serial.py here)
// without a host pass over the body.
//
// CRC-32 (reflected polynomial 0xEDB88320, init and final xor 0xFFFFFFFF) is
// affine in the message, so chunks are checksummed independently and merged
// with zlib's crc32_combine rule: crc(A || B) = (x^(8 |B|) mod P) * crc(A) ^
// crc(B), products taken in GF(2)[x] mod P (multmodp / x2nmodp of zlib 1.2.12+).
//   pass 1: one thread per 4 KB chunk, slicing-by-8 tables in shared memory;
//   pass 2: one CTA merges the chunk CRCs pairwise in a tree (level j merges
//           neighbours 2^j chunks apart with the operator x^(8 * 4 KB * 2^j));
//           the last (short) chunk is handled by merging right-to-left in
//           length order.
#include "fhe_internal.cuh"

namespace {

constexpr unsigned kPoly = 0xEDB88320u;
constexpr long kChunk = 4096;
constexpr int kCrcThreads = 256;

__device__ __host__ inline unsigned multmodp(unsigned a, unsigned b) {
  unsigned m = 1u << 31, p = 0;
  for (;;) {
    if (a & m) {
      p ^= b;
      if ((a & (m - 1)) == 0) break;
    }
    m >>= 1;
    b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
  }
  return p;
}

// x^(n * 2^k) mod P (n bytes -> k = 3)
__device__ __host__ inline unsigned x2nmodp(unsigned long long n, unsigned k) {
  unsigned p = 1u << 31;  // x^0
  // x^(2^k) mod P, squared as k grows
  unsigned t = 1u << 30;  // x^1
  for (unsigned i = 0; i < k; ++i) t = multmodp(t, t);
  while (n) {
    if (n & 1) p = multmodp(t, p);
    n >>= 1;
    t = multmodp(t, t);
  }
  return p;
}

__global__ void __launch_bounds__(kCrcThreads)
    crc_chunks_kernel(const unsigned char* __restrict__ data, long nbytes, long nchunks,
                      unsigned* __restrict__ crcs) {
  __shared__ unsigned tab[8][256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    unsigned c = (unsigned)i;
    for (int k = 0; k < 8; ++k) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
    tab[0][i] = c;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    unsigned c = tab[0][i];
    for (int s = 1; s < 8; ++s) {
      c = tab[0][c & 0xff] ^ (c >> 8);
      tab[s][i] = c;
    }
  }
  __syncthreads();
  const long ch = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (ch >= nchunks) return;
  const long b0 = ch * kChunk, b1 = min(nbytes, b0 + kChunk);
  unsigned c = 0xFFFFFFFFu;
  long i = b0;
  // 8 bytes at a time from 8-byte aligned words (the chunk base is aligned
  // when the buffer is; unaligned heads fall back to bytes)
  while (i < b1 && (((unsigned long long)(data + i)) & 7)) c = tab[0][(c ^ data[i++]) & 0xff] ^ (c >> 8);
  for (; i + 8 <= b1; i += 8) {
    const unsigned long long w = *reinterpret_cast<const unsigned long long*>(data + i);
    const unsigned lo = (unsigned)w ^ c, hi = (unsigned)(w >> 32);
    c = tab[7][lo & 0xff] ^ tab[6][(lo >> 8) & 0xff] ^ tab[5][(lo >> 16) & 0xff] ^
        tab[4][lo >> 24] ^ tab[3][hi & 0xff] ^ tab[2][(hi >> 8) & 0xff] ^
        tab[1][(hi >> 16) & 0xff] ^ tab[0][hi >> 24];
  }
  for (; i < b1; ++i) c = tab[0][(c ^ data[i]) & 0xff] ^ (c >> 8);
  crcs[ch] = c ^ 0xFFFFFFFFu;
}

// pairwise tree over the chunk CRCs: after level j, crcs[i * 2^(j+1)] holds
// the CRC of chunks [i 2^(j+1), (i+1) 2^(j+1)); the right operand's length is
// 2^j full chunks, except at the tail (the last chunk may be short).
__global__ void __launch_bounds__(1024)
    crc_merge_kernel(unsigned* __restrict__ crcs, long nchunks, long nbytes, unsigned* out) {
  for (long span = 1; span < nchunks; span <<= 1) {
    for (long i = threadIdx.x * 2 * span; i < nchunks; i += (long)blockDim.x * 2 * span) {
      const long r = i + span;
      if (r < nchunks) {
        const long rbytes = min(nbytes, (r + span) * kChunk) - r * kChunk;
        crcs[i] = multmodp(x2nmodp((unsigned long long)rbytes, 3), crcs[i]) ^ crcs[r];
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = nchunks ? crcs[0] : 0u;
}

}  // namespace

size_t crc32_workspace(long nbytes) {
  const long nchunks = (nbytes + kChunk - 1) / kChunk;
  return (size_t)(nchunks + 1) * sizeof(unsigned);
}

int run_crc32(const void* data, long nbytes, unsigned* out, void* ws, size_t ws_bytes,
              cudaStream_t st) {
  if (nbytes < 0) {
    fhe_set_error("crc32: negative length");
    return -1;
  }
  if (ws_bytes < crc32_workspace(nbytes)) {
    fhe_set_error("crc32: workspace too small");
    return -1;
  }
  const long nchunks = (nbytes + kChunk - 1) / kChunk;
  unsigned* crcs = (unsigned*)ws;
  if (nchunks) {
    crc_chunks_kernel<<<(unsigned)((nchunks + kCrcThreads - 1) / kCrcThreads), kCrcThreads, 0,
                        st>>>((const unsigned char*)data, nbytes, nchunks, crcs);
    FHE_LAUNCH_CHECK();
  }
  crc_merge_kernel<<<1, 1024, 0, st>>>(crcs, nchunks, nbytes, out);
  FHE_LAUNCH_CHECK();
  return 0;
}

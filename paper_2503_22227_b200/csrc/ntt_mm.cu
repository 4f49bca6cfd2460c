// Matrix-product NTT variant (reference NttVariant.FORCE_MM and the AUTO rule
// below degree 1024: coremath/ntt.py:101-124 materialize_matrix, :201-233
// ntt_mm / intt_mm, :354-364 ntt_dispatch).
//
//   forward  out[j] = sum_i a[i] psi^(exp_j * i mod 2N),  exp_j = 2 bitrev(j) + 1
//   inverse  out[i] = n^-1 sum_j a[j] psi^(-(i * exp_j) mod 2N)
//
// The reference materialises the n x n matrices (in Montgomery form) on the
// host; here each entry is read from the chain's bit-reversed psi table
// (psi^k = psi_br[bitrev(k)] for k < N and -psi^(k-N) above, psi^N = -1), so
// nothing is materialised.  Every term is an exact product mod q, so the
// canonical outputs are the butterfly transform's words (the reference's own
// test: test_ntt.py:47-55, test_acceptance.py:110-137).
//
// One CTA per (row, 256 outputs); the input row is staged in shared memory.
// O(N^2) per row: a small-degree / API-completeness variant (N <= 2^13).
#include "fhe_kernels.cuh"

namespace {

constexpr int kMmThreads = 256;

__global__ void __launch_bounds__(kMmThreads)
    ntt_mm_kernel(const DevChain ch, u64* out, const u64* in, int rows, RowMap map, bool inverse) {
  extern __shared__ u64 mm_row[];
  const int log_n = ch.log_n;
  const u32 n = 1u << log_n, mask = 2 * n - 1;
  for (int row = blockIdx.y; row < rows; row += gridDim.y) {
  const int p = map(row);
  const ModConst mc = ch.mc[p];
  const u64 q = mc.q;
  const WPair* tw = ch.tw + ((size_t)p << log_n);
  const u64* src = in + ((size_t)row << log_n);
  __syncthreads();  // the previous row's reads of mm_row are done
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) mm_row[i] = src[i];
  __syncthreads();
  const u32 o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o >= n) continue;
  u64 acc = 0;
  if (!inverse) {
    const u32 e = 2 * (__brev(o) >> (32 - log_n)) + 1;
    u32 k = 0;
    for (u32 i = 0; i < n; ++i, k = (k + e) & mask) {
      const u32 r = k & (n - 1);
      u64 w = tw[__brev(r) >> (32 - log_n)].w;
      if (k & n) w = neg_mod(w, q);
      acc = add_mod(acc, mul_mod(mm_row[i], w, mc), q);
    }
  } else {
    for (u32 j = 0; j < n; ++j) {
      const u32 e = 2 * (__brev(j) >> (32 - log_n)) + 1;
      const u32 k = (2 * n - ((o * e) & mask)) & mask;  // -(o * exp_j) mod 2N
      const u32 r = k & (n - 1);
      u64 w = tw[__brev(r) >> (32 - log_n)].w;
      if (k & n) w = neg_mod(w, q);
      acc = add_mod(acc, mul_mod(mm_row[j], w, mc), q);
    }
    const WPair ni = ch.ninv[p];
    acc = shoup_mul(acc, ni.w, ni.sh, q);
  }
  out[((size_t)row << log_n) + o] = acc;
  }
}

}  // namespace

int launch_ntt_mm(const DevChain& ch, u64* out, const u64* in, int rows, RowMap map, bool inverse,
                  cudaStream_t st) {
  if (rows <= 0) return 0;
  if (ch.log_n > 13) {
    fhe_set_error("matrix NTT variant supports N <= 2^13 (O(N^2) per row)");
    return -1;
  }
  const int n = 1 << ch.log_n;
  dim3 grid((n + kMmThreads - 1) / kMmThreads, rows < 65535 ? rows : 65535);
  const size_t smem = (size_t)n * sizeof(u64);
  if (smem > 48 * 1024)
    FHE_CUDA_CHECK(cudaFuncSetAttribute(ntt_mm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem));
  ntt_mm_kernel<<<grid, kMmThreads, smem, st>>>(ch, out, in, rows, map, inverse);
  FHE_LAUNCH_CHECK();
  ntt_path_hit(FHE_NTT_PATH_MM);
  return 0;
}

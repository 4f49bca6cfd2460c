// Micro test of the tcgen05 u8 MMA wrappers (csrc/umma.cuh): D = A B^T for
// A 128 x 96 and B N x 96 random bytes, accumulator in TMEM, checked against
// a host product.  Build + run on a B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//     -I paper_2503_22227_b200/csrc tools/micro/umma_i8.cu -o /tmp/umma && /tmp/umma
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "umma.cuh"

constexpr int M = 128, K = 96;

template <int N>
__global__ void umma_test(const unsigned char* A, const unsigned char* B, int* D) {
  __shared__ __align__(128) unsigned char sa[M * K];
  __shared__ __align__(128) unsigned char sb[N * K];
  __shared__ uint64_t bar;
  __shared__ unsigned tbase;
  const int tid = threadIdx.x;
  // canonical layout [k16][row group][8 rows][16 B]
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    sa[((k / 16) * (M / 8) + r / 8) * 128 + (r % 8) * 16 + k % 16] = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    sb[((k / 16) * (N / 8) + r / 8) * 128 + (r % 8) * 16 + k % 16] = B[i];
  }
  if (tid == 0) umma_mbar_init(&bar, 1);
  if (tid < 32) {
    tmem_alloc(&tbase, N < 32 ? 32 : N);
    tmem_relinquish();
  }
  fence_async_smem();
  umma_fence_before();
  __syncthreads();
  umma_fence_after();
  const unsigned tm = tbase;
  if (tid == 0) {
    const unsigned a0 = umma_smem_u32(sa), b0 = umma_smem_u32(sb);
    for (int j = 0; j < K / 32; ++j) {
      const uint64_t ad = umma_desc(a0 + 2 * j * (M / 8) * 128, (M / 8) * 128, 128);
      const uint64_t bd = umma_desc(b0 + 2 * j * (N / 8) * 128, (N / 8) * 128, 128);
      umma_u8(tm, ad, bd, umma_idesc_u8(M, N), j > 0);
    }
    umma_commit(&bar);
  }
  umma_mbar_wait(&bar, 0);
  umma_fence_after();
  const int w = tid >> 5, row = 32 * w + (tid & 31);
  for (int c = 0; c < N; c += 8) {
    unsigned r[8];
    tmem_ld8(tm + ((32 * w) << 16) + c, r);
    tmem_ld_wait();
    for (int i = 0; i < 8; ++i) D[row * N + c + i] = (int)r[i];
  }
  umma_fence_before();
  __syncthreads();
  if (tid < 32) tmem_dealloc(tm, N < 32 ? 32 : N);
}

template <int N>
int run() {
  std::vector<unsigned char> A(M * K), B(N * K);
  srand(1 + N);
  for (auto& x : A) x = rand() & 0xff;
  for (auto& x : B) x = rand() & 0xff;
  unsigned char *dA, *dB;
  int* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, M * N * 4);
  umma_test<N><<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    printf("N=%d: %s\n", N, cudaGetErrorString(e));
    return 1;
  }
  std::vector<int> D(M * N);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      int ref = 0;
      for (int k = 0; k < K; ++k) ref += (int)A[i * K + k] * (int)B[j * K + k];
      if (ref != D[i * N + j] && bad++ < 5)
        printf("N=%d D[%d][%d] = %d, want %d\n", N, i, j, D[i * N + j], ref);
    }
  printf("N=%d: %d mismatches of %d\n", N, bad, M * N);
  return bad != 0;
}

int main() { return run<64>() | run<128>() | run<256>(); }

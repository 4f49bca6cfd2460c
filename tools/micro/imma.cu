// Microbenchmark: legacy mma.sync tensor throughput on B200 (sm_100a):
// IMMA m16n8k32 s8 (int32 accumulate) and u8, DMMA m8n8k4 f64.
#include <cstdio>
#include <cstdint>
__global__ void k_imma(int* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = blockIdx.x, b1 = b0 + 1;
  int c[4][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0 + j), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 12345) out[0] = s;
}
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x, b = blockIdx.x;
  double c[4][2] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a + j), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.0) out[0] = s;
}
int main() {
  int* d; cudaMalloc(&d, 64);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 1 << 14, blocks = sms * 4, threads = 256;
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  float ms;
  k_imma<<<blocks, threads>>>(d, 16); cudaDeviceSynchronize();
  cudaEventRecord(s); k_imma<<<blocks, threads>>>(d, iters); cudaEventRecord(e); cudaEventSynchronize(e);
  cudaEventElapsedTime(&ms, s, e);
  double ops = (double)blocks * (threads / 32) * iters * 4 * (16.0 * 8 * 32 * 2);
  printf("imma m16n8k32 s8: %8.3f ms  %8.1f TOPS\n", ms, ops / ms / 1e9);
  k_dmma<<<blocks, threads>>>((double*)d, 16); cudaDeviceSynchronize();
  cudaEventRecord(s); k_dmma<<<blocks, threads>>>((double*)d, iters); cudaEventRecord(e); cudaEventSynchronize(e);
  cudaEventElapsedTime(&ms, s, e);
  ops = (double)blocks * (threads / 32) * iters * 4 * (8.0 * 8 * 4 * 2);
  printf("dmma m8n8k4 f64:  %8.3f ms  %8.1f TFLOPS\n", ms, ops / ms / 1e9);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

// Microbenchmark: throughput of 64-bit integer multiply pieces vs FP64 FMA on B200.
#include <cstdio>
#include <cstdint>
typedef unsigned long long u64;
__global__ void k_wide(u64* out, int iters) {
  unsigned a = threadIdx.x * 7 + 1, b = blockIdx.x * 3 + 5;
  u64 acc[8];
  for (int j = 0; j < 8; ++j) acc[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = (u64)(unsigned)acc[j] * (u64)(b + j) + a;  // IMAD.WIDE.U32
  }
  u64 s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 12345) out[0] = s;
}
__global__ void k_imad(u64* out, int iters) {
  unsigned acc[8]; unsigned a = threadIdx.x * 7 + 1, b = blockIdx.x * 3 + 5;
  for (int j = 0; j < 8; ++j) acc[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = acc[j] * (b + j) + a;
  }
  unsigned s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 12345) out[0] = s;
}
__global__ void k_dfma(u64* out, int iters) {
  double acc[8]; double a = threadIdx.x * 1.0001, b = blockIdx.x * 0.999;
  for (int j = 0; j < 8; ++j) acc[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = fma(acc[j], b + j, a);
  }
  double s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 12345.0) out[0] = 1;
}
__global__ void k_mulhi64(u64* out, int iters) {
  u64 acc[8]; u64 a = threadIdx.x * 0x9E3779B97F4A7C15ull, b = blockIdx.x * 0xBF58476D1CE4E5B9ull;
  for (int j = 0; j < 8; ++j) acc[j] = j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = __umul64hi(acc[j] ^ a, b);
  }
  u64 s = 0; for (int j = 0; j < 8; ++j) s += acc[j];
  if (s == 12345) out[0] = s;
}
int main() {
  u64* d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int iters = 1 << 14; int blocks = sms * 8, threads = 256;
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  auto run = [&](const char* name, void (*k)(u64*, int), double ops_per_iter) {
    k<<<blocks, threads>>>(d, 16); cudaDeviceSynchronize();
    cudaEventRecord(s); k<<<blocks, threads>>>(d, iters); cudaEventRecord(e); cudaEventSynchronize(e);
    float ms; cudaEventElapsedTime(&ms, s, e);
    double ops = (double)blocks * threads * iters * ops_per_iter;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-10s %8.3f ms  %8.1f Gop/s  %6.1f ops/clk/SM (at %d MHz)\n", name, ms, ops / ms / 1e6,
           ops / (ms * 1e-3) / (sms * (double)clk * 1e3), clk / 1000);
  };
  run("imad32", k_imad, 8); run("imad.wide", k_wide, 8); run("dfma", k_dfma, 8); run("mulhi64", k_mulhi64, 8);
  return 0;
}

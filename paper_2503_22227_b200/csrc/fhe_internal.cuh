// Internal device-side structures shared by the kernels and the C-ABI layer.
#pragma once
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "modarith.cuh"

// Shoup pair: a constant and its floor(w * 2^64 / q) companion, loaded with a
// single 16-byte access.
struct __align__(16) WPair {
  u64 w;
  u64 sh;
};

// NTT tables for one modulus chain, resident in HBM (built once per context).
// Forward twiddles follow coremath/ntt.py:86-98 (powers of the smallest
// primitive 2N-th root psi in bit-reversed order, plus Shoup companions);
// inverse twiddles are the bit-reversed powers of psi^-1.
struct DevChain {
  int count;             // primes in the chain
  int log_n;
  const ModConst* mc;    // [count]
  const WPair* tw;       // [count][N]   (psi_br[i], shoup)
  const WPair* itw;      // [count][N]   (ipsi_br[i], shoup)
  const WPair* ninv;     // [count]      (n^-1, shoup)
  const WPair* ninv_w1;  // [count]      (ipsi_br[1] * n^-1, shoup)
  bool lazy_ok;          // every prime < 2^58: lazy forward butterflies allowed
  // FP64-pipe tables, present when every prime is < 2^50 (fp64_ok):
  bool fp64_ok;
  const double2* twd;      // [count][N] (psi_br[i], psi_br[i] / q)
  const double2* itwd;     // [count][N] (ipsi_br[i], ipsi_br[i] / q)
  const double2* qd;       // [count]    (q, 1 / q)
  const double2* ninv_d;   // [count]    (n^-1, n^-1 / q)
  const double2* ninv_w1_d;// [count]    (ipsi_br[1] n^-1, ... / q)
  // staged-order (w, w/q) tables of the four-step kernels (log_n >= 13):
  // [count][2][tws_dir]: forward then inverse; per direction N1 column pairs,
  // then N1 chunk blocks of N2 pairs (ntt_plan.cuh); tws_dir = N1 + N
  const double2* tws;
  long tws_dir;
  // host-side scratch of the fused four-step NTT (FuseScratch*, ntt.cu)
  void* fuse;
  // HOST pointer (never read on the device): per prime, 1 when its FP64
  // tables are valid (< 2^50); lets a mixed chain run FP64 transforms on
  // rows that only use such primes (launch_ntt)
  const unsigned char* fp64_prime_host;
};

// Row -> chain position mapping used by every batched kernel.  The
// reference passes an explicit per-row mod_idx (coremath/ntt.py:257-264);
// here a NULL pointer means the layout-order pattern (row % limbs) + offset
// that CData.mod_idx() produces (rnspoly.py:109-111).
struct RowMap {
  const int32_t* idx;  // device int32[limbs], may be null (identity)
  int limbs;
  int offset;
  __device__ __forceinline__ int operator()(int row) const {
    const int r = row % limbs;
    return (idx ? idx[r] : r) + offset;
  }
};

// philox.cu (FhePhilox is declared in fhe_sm100.h)
struct FhePhilox;
size_t philox_workspace(long count, unsigned long long rng);
int run_philox_integers(FhePhilox* dev_state, long long low, unsigned long long rng, long count,
                        uint64_t* out, void* ws, size_t ws_bytes, cudaStream_t st);
int run_cbd_combine(long long* out, const uint64_t* flips, int pairs, long n, cudaStream_t st);
// crc32.cu
size_t crc32_workspace(long nbytes);
int run_crc32(const void* data, long nbytes, unsigned* out, void* ws, size_t ws_bytes,
              cudaStream_t st);

// thread-local error text for fhe_last_error()
void fhe_set_error(const std::string& msg);

#define FHE_CUDA_CHECK(expr)                                                   \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      fhe_set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));       \
      return -2;                                                               \
    }                                                                          \
  } while (0)

// every kernel launch of the library is followed by FHE_LAUNCH_CHECK, which
// also counts it (fhe_launch_count())
void fhe_count_launch();

// Programmatic dependent launch (PDL).  Kernels launched with fhe_launch
// carry cudaLaunchAttributeProgrammaticStreamSerialization: the next kernel
// on the stream may be scheduled while this one runs, once every CTA of this
// one has executed fhe_pdl_trigger (issued at CTA start).  Every such kernel
// begins with fhe_pdl_wait before touching memory written by earlier work,
// which blocks until the preceding grid has completed and its writes are
// visible -- so the overlap covers launch latency and CTA rasterisation, not
// data.  Both instructions are no-ops for a kernel launched without the
// attribute.  Off by default (FHE_PDL=1 turns it on): measured on the PDQ
// query graphs (N = 2^12, ~640 small kernels) it is 1-4% slower, and eager
// chains gain nothing (profiles/r2_pdq_latency.md).
__device__ __forceinline__ void fhe_pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void fhe_pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" :::);
}
bool fhe_pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t fhe_launch(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = fhe_pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

#define FHE_LAUNCH_CHECK()                                                     \
  do {                                                                         \
    fhe_count_launch();                                                        \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      fhe_set_error(std::string("kernel launch: ") + cudaGetErrorString(_e));  \
      return -3;                                                               \
    }                                                                          \
  } while (0)


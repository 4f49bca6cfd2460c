// Host-side objects behind the opaque C-ABI handles.
#pragma once
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "fhe_kernels.cuh"

struct FheChain {
  DevChain dev{};
  int log_n = 0;
  std::vector<u64> primes;
  std::vector<u64> psi;  // smallest primitive 2N-th root per prime
  std::vector<unsigned char> fp64_prime;  // per prime: < 2^50 (FP64 tables valid)
  void* dmem = nullptr;  // one allocation for all tables
  size_t dbytes = 0;
};

// Per-level key-switch and rescale constants, resident in HBM.
// Level l = number of active Q primes (1..L).
struct LevelPlan {
  int level = 0;
  int digits = 0;        // active digits D = ceil(l / alpha)
  int ext_rows = 0;      // sum over digits of (l + K - |digit|)
  std::vector<int> dig_s0, dig_na, dig_row_off, dig_w_off;
  // device pointers into LevelPlan::dmem
  const WPair* up_inv = nullptr;     // [l]   ((Q_d / q_s)^-1 mod q_s) per Q prime
  const u64* up_w = nullptr;         // per digit [na][l+K-na]: [Q_d/q_s] mod target
  const int32_t* ext_prime = nullptr;  // [ext_rows] chain position of each ext row
  const int* dig_info = nullptr;     // [4*digits] s0, na, row_off, w_off
  const WPair* down_inv = nullptr;   // [K] (P/p_k)^-1 mod p_k
  const u64* down_w = nullptr;       // [K][l] [P/p_k] mod q_j
  const WPair* p_inv = nullptr;      // [l] P^-1 mod q_j
  const WPair* rs_inv = nullptr;     // [l-1] q_{l-1}^-1 mod q_j
  const u64* rs_qlast = nullptr;     // [l-1] q_{l-1} mod q_j
  // FP64-pipe copies (w, w / modulus) when every chain prime is < 2^50
  const double2* up_inv_d = nullptr;
  const double2* up_w_d = nullptr;
  const double2* down_inv_d = nullptr;
  const double2* down_w_d = nullptr;
  const double2* p_inv_d = nullptr;  // (P^-1 mod q_j, / q_j): the FP64 ModDown finish
  const double2* rs_inv_d = nullptr; // (q_{l-1}^-1 mod q_j, / q_j): the FP64 rescale finish
  // tensor-core base conversion (bconv_imma.cuh), every chain prime < 2^56:
  // packed byte-split W' fragments, ModUp per digit ([nt][up_ks][32] each,
  // offsets in up_bf_off) and ModDown ([level][down_ks][32])
  // exact CRT lift of the level's Q (crt.cu): W limbs per big integer;
  // crt_M[i] = Q / q_i ([level][W]), crt_Q, crt_Qh = floor(Q / 2) ([W]),
  // crt_inv[i] = (Q / q_i)^-1 mod q_i, crt_qinv[i] = 1 / q_i (quotient estimate)
  int crt_W = 0;
  const u64* crt_M = nullptr;
  const u64* crt_Q = nullptr;
  const u64* crt_Qh = nullptr;
  const WPair* crt_inv = nullptr;
  const double* crt_qinv = nullptr;
  double crt_Qd = 0.0;   // Q * 2^(-64 crt_qdrop) as a double (BFV quotient estimate)
  int crt_qdrop = 0;
  bool bf_ok = false;
  int up_ks = 0, down_ks = 0, max_na = 0;
  // wide conversion (some prime >= 2^56): source words of 8 bytes where the
  // sources are that wide, targets reduced from 79-bit sums; tcgen05 only
  bool bf_wide = false;
  int up_sb = 7, down_sb = 7;  // bytes per source word, ModUp / ModDown
  const uint2* up_bf = nullptr;
  const int* up_bf_off = nullptr;
  const uint2* down_bf = nullptr;
  const uint2* up_bf2 = nullptr;     // the same, packed for bconv_imma2_kernel
  const int* up_bf2_off = nullptr;
  const uint2* down_bf2 = nullptr;
  // the same W' bytes in the tcgen05 operand layout (bconv_umma.cuh): per job
  // [2 ks][round8(nt)][8 bytes b][16 B], ModUp per digit at up_bu_off (16 B units)
  const uint4* up_bu = nullptr;
  const int* up_bu_off = nullptr;
  const uint4* down_bu = nullptr;
  void* dmem = nullptr;
};

// BGV modulus-switch constants for one plain modulus t.
struct PlainPlan {
  std::vector<void*> dmem;                 // per level
  std::vector<const u64*> t_mod;           // per level: [l-1] t mod q_j
  std::vector<WPair> tinv_last;            // per level: t^-1 mod q_{l-1}
};

struct FheContext {
  FheChain* chain = nullptr;  // Q then P
  int L = 0, K = 0, alpha = 1;
  std::vector<LevelPlan> levels;  // index l (0 unused)
  std::mutex plain_mu;
  std::map<u64, std::unique_ptr<PlainPlan>> plain;
};

int build_chain(const u64* primes, int count, int log_n, FheChain* ch);
int build_levels(FheContext* ctx);
void free_chain(FheChain* ch);
const PlainPlan* get_plain_plan(FheContext* ctx, u64 t);

// keyswitch.cu
size_t keyswitch_workspace(const FheContext& ctx, int level, int batch);
int run_keyswitch(const FheContext& ctx, int level, const u64* d, long d_stride, const u64* key,
                  const u64* add0, const u64* add1, long add_stride, u64* out0, u64* out1,
                  long out_stride, int batch, void* ws, size_t ws_bytes, cudaStream_t st,
                  bool tens = false);
size_t hmult_relin_workspace(const FheContext& ctx, int level, int batch);
int run_hmult_relin(const FheContext& ctx, int level, const u64* x, const u64* y, long in_stride,
                    const u64* key, u64* out0, u64* out1, long out_stride, int batch, void* ws,
                    size_t ws_bytes, cudaStream_t st);
size_t rescale_workspace(const FheContext& ctx, int polys, int level);
// crt.cu
int run_crt_lift(const FheContext& ctx, int mode, void* out, const u64* rows, int level,
                 double scale, u64 t, u64 inv_f, cudaStream_t st);
int run_rescale(FheContext& ctx, u64* out, const u64* in, int polys, int level, u64 t_plain,
                void* ws, size_t ws_bytes, cudaStream_t st);

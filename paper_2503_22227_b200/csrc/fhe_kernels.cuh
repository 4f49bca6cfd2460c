// Launch wrappers implemented in ntt.cu / poly.cu / keyswitch.cu.
#pragma once
#include "../../include/fhe_sm100.h"
#include "fhe_internal.cuh"

int grid_for(long work);

// ntt.cu: transform `rows` rows of src into dst (may alias).  Row r uses
// chain position map(r) and lives at (r / map.limbs) * bstride +
// (r % map.limbs) * N words (bstride 0: contiguous rows).
// Optional ModDown finish applied in the forward NTT's last-pass epilogue
// instead of storing the transform: row r (= (b * 2 + poly) * level + j) of
// the result x gives  out_poly[b][j] = add_poly[b][j] + (accQ[r] - x) P^-1_j
// (keyswitch.cu moddown_finish_kernel; NTT rows are the ModDown conv rows).
struct NttFinish {
  const u64* accQ;
  const WPair* p_inv;  // [level] (P^-1 mod q_j, Shoup)
  const u64* add0;
  const u64* add1;
  long add_stride;
  u64* out0;
  u64* out1;
  long out_stride;
  int level;
};

struct NttArgs {
  u64* dst;
  const u64* src;
  int rows;
  RowMap map;
  long src_bstride;
  long dst_bstride;
  const NttFinish* fin = nullptr;  // forward only; *fin_done tells if it was applied
  bool* fin_done = nullptr;
  // Broadcast input (forward; N = 2^16 TMA column path and N <= 2^12 rows): input row r is
  // bcast_src + (r / map.limbs) * bcast_stride -- one row per batch item,
  // shared by its map.limbs target rows -- read as the centred integer
  // (v > center_q / 2 ? v - center_q : v).  Rescale's correction (ckks.py:
  // 382-410) is the centred last limb mod every q_j; the transform takes the
  // centred value itself as the representative, so no expanded rows are
  // materialised.  A launch that cannot take this path returns *bcast_done
  // = false and leaves dst untouched.
  const u64* bcast_src = nullptr;
  long bcast_stride = 0;
  u64 center_q = 0;               // 0: the source words are used as they are
  bool* bcast_done = nullptr;
  int bcast_div = 0;              // target rows per source row (0: map.limbs); rows path only
  // Rescale finish fused into the broadcast transform's epilogue (N = 2^12
  // cluster path): row r = (poly, j) writes rs_out[poly][j] = (rs_in[poly][j]
  // - NTT(row)) * rs_inv_d[j] instead of dst (rs_in has rs_level rows per
  // poly, rs_out rs_level - 1); *rs_done tells whether it was applied.
  const u64* rs_in = nullptr;
  u64* rs_out = nullptr;
  const double2* rs_inv_d = nullptr;
  int rs_level = 0;
  bool* rs_done = nullptr;
  // caller's assertion: every row's prime is < 2^50 (a mixed chain may then
  // run this transform on the FP64 path; launch_ntt)
  bool fp64_rows = false;
};
int launch_ntt(const DevChain& ch, const NttArgs& a, bool inverse, cudaStream_t st);
unsigned long long ntt_path_count(int path);
void ntt_path_hit(int path);
// ntt_mm.cu: matrix-product variant (reference ntt_mm / intt_mm), out != in
int launch_ntt_mm(const DevChain& ch, u64* out, const u64* in, int rows, RowMap map, bool inverse,
                  cudaStream_t st);
// per-chain scratch of the fused four-step NTT (tile tickets, group counters)
void* fuse_scratch_new(int log_n);
void fuse_scratch_free(void* p);
inline int launch_ntt(const DevChain& ch, u64* data, const u64* in, int rows, RowMap map,
                      bool inverse, cudaStream_t st) {
  return launch_ntt(ch, NttArgs{data, in, rows, map, 0, 0}, inverse, st);
}

// philox.cu: small signed coefficients -> residue rows (canonical)
int run_signed_lift(const DevChain& ch, u64* out, const long long* c, long n, int limbs,
                    int offset, cudaStream_t st);
// integer-valued doubles (any magnitude) -> residue rows (CKKS encode)
int run_real_lift(const DevChain& ch, u64* out, const double* v, long n, int limbs, int offset,
                  cudaStream_t st);

// poly.cu
int launch_ewise(const DevChain& ch, int op, u64* out, const u64* a, const u64* b, const u64* c,
                 long rows, RowMap map, int b_mode, cudaStream_t st);
int launch_tensor(const DevChain& ch, u64* out, const u64* x, const u64* y, int limbs, long batch,
                  long x_stride, long y_stride, long out_stride, int square, cudaStream_t st);
int launch_automorph(u64* out, const u64* in, long rows, int log_n, u64 elt, cudaStream_t st);
int launch_modswitch_expand(const DevChain& ch, u64* corr, const u64* last, int polys,
                            int new_level, int last_prime, u64 t_plain, WPair tinv_last,
                            const u64* t_mod, const u64* qlast_mod, cudaStream_t st);
int launch_rescale_small(const DevChain& ch, u64* out, const u64* in, const u64* last, int polys,
                         int level, const WPair* inv, const u64* qlast_mod, cudaStream_t st);
int launch_modswitch_finish(const DevChain& ch, u64* out, const u64* in, const u64* corr,
                            int polys, int level, const WPair* inv, cudaStream_t st);

/*
 * fhe_sm100.h - C ABI of the B200 (sm_100a) RNS-FHE hot path.
 *
 * This is the drop-in boundary for the reference's optional compiled-kernel
 * seam, the numba module rnsfhe.coremath._kernels, which the reference
 * imports behind try/except at coremath/ntt.py:24-27, rnspoly.py:21-24,
 * keys.py:22-25, schemes/ckks.py:33-36 and schemes/behz.py:22-25, plus the
 * scheme-level operations built on it.  Each entry point names the reference
 * interface it replaces.  INTEGRATION.md shows the ctypes binding.
 *
 * Conventions (all entry points):
 *  - plain pointers and sizes; polynomials are uint64 residues in the
 *    reference CData layout: word ((p * size_modulus) + j) * n + i
 *    (rnspoly.py:1-8), evaluation (NTT) domain unless stated;
 *  - every "uint64_t *" data pointer is DEVICE memory owned by the caller;
 *    the library never allocates on the hot path (work buffers are passed in);
 *  - "stream" is a cudaStream_t (NULL = legacy default stream); calls are
 *    asynchronous on it and thread-safe across streams;
 *  - return 0 on success, a negative code on error; fhe_last_error() returns
 *    the thread-local message of the last failure.  Shape/level validation
 *    stays in the host layer (as in the reference, e.g. ntt.py:280-282).
 */
#ifndef FHE_SM100_H
#define FHE_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct FheChain FheChain;     /* NTT + reduction tables of one prime chain */
typedef struct FheContext FheContext; /* chain Q|P plus rescale / key-switch plans */

/* element-wise op codes for fhe_ewise (rnspoly.py:214-308, vecmod.py:114-165) */
enum {
  FHE_EW_ADD = 0,     /* a + b            poly_add / add_arr          */
  FHE_EW_SUB = 1,     /* a - b            poly_sub / sub_arr          */
  FHE_EW_NEG = 2,     /* -a               poly_negate / neg_arr       */
  FHE_EW_MUL = 3,     /* a * b            _kernels.mul_batch          */
  FHE_EW_NEG_MUL = 4, /* -(a * b)         _kernels.neg_mul_batch      */
  FHE_EW_MUL_ADD = 5, /* a * b + c        _kernels.mul_add_batch      */
  FHE_EW_MUL_SUB = 6, /* c - a * b                                    */
  FHE_EW_REDUCE = 7   /* a mod q_j (a any 64-bit word)  x % q_col      */
};
/* how operand b is addressed in fhe_ewise */
enum {
  FHE_B_FULL = 0,  /* same shape as a                                   */
  FHE_B_BCAST = 1, /* one poly of `limbs` rows, broadcast over polys   */
  FHE_B_CONST = 2  /* one word per chain position: b[mod_idx(row)]      */
};

const char* fhe_last_error(void);

/* Number of kernels this library has launched in the process (every entry
 * point's launches; cudaMemsetAsync is not counted).  No reference
 * counterpart: evidence for benchmarks (bench.py gpu_launches). */
uint64_t fhe_launch_count(void);
int fhe_device_sm_count(void);

/* Transform launches per NTT kernel path since load (no reference
 * counterpart: evidence for the parity tests and the bench of WHICH kernel
 * ran a transform).  Unknown path: 0. */
enum {
  FHE_NTT_PATH_ROWS = 0,      /* whole-row tiles, N <= 2^12 (FP64 pipe)          */
  FHE_NTT_PATH_SPLIT = 1,     /* four-step, two kernels (column + chunk tiles)   */
  FHE_NTT_PATH_FUSED_TMA = 2, /* four-step, one ticketed kernel on TMA tiles      */
  FHE_NTT_PATH_FUSED_CP = 3,  /* four-step, one ticketed kernel on cp.async tiles */
  FHE_NTT_PATH_INT = 4,       /* 64-bit integer pipe (a prime >= 2^50)            */
  FHE_NTT_PATH_CLUSTER = 5,   /* row held by a CTA cluster (DSMEM): N = 2^12 small launches, N = 2^16 opt-in */
  FHE_NTT_PATH_MM = 6,        /* matrix-product variant (fhe_ntt_mm)              */
  FHE_NTT_PATHS = 8
};
uint64_t fhe_ntt_path_count(int path);

/* ---- chains: NttTables / NttChain precompute (coremath/ntt.py:52-137,
 *      240-275; primes.py:60-71 for psi; rnspoly.py:47-67) ---------------- */
int fhe_chain_create(const uint64_t* primes, int count, int log_n, FheChain** out);
int fhe_chain_destroy(FheChain* ch);
/* host copies of one prime's tables, for parity tests:
 * psi (scalar), psi_br[N], ipsi_br[N], n_inv (scalar) */
int fhe_chain_tables(const FheChain* ch, int idx, uint64_t* psi, uint64_t* psi_br,
                     uint64_t* ipsi_br, uint64_t* n_inv);

/* ---- batched NTT: NttChain.forward / .inverse (ntt.py:277-351),
 *      _kernels.ntt_batch / intt_batch (_kernels.py:88-99).  In place over
 *      `rows` contiguous rows of n words.  Row r uses chain position
 *      mod_idx[r % limbs] + offset (mod_idx: device int32[limbs]; NULL means
 *      the identity, i.e. (r % limbs) + offset; pass limbs = rows for a full
 *      per-row map). */
int fhe_ntt_fwd(const FheChain* ch, uint64_t* data, int64_t rows, const int32_t* mod_idx,
                int limbs, int offset, void* stream);
int fhe_ntt_inv(const FheChain* ch, uint64_t* data, int64_t rows, const int32_t* mod_idx,
                int limbs, int offset, void* stream);

/* ---- matrix-product NTT variant: ntt_mm / intt_mm (coremath/ntt.py:201-233),
 *      the NttVariant.FORCE_MM path of NttChain (ntt.py:266-275) and the
 *      AUTO rule of ntt_dispatch below degree 1024 (ntt.py:354-364).
 *      Same canonical words as fhe_ntt_fwd/inv; out must not alias in;
 *      N <= 2^13. */
int fhe_ntt_mm(const FheChain* ch, uint64_t* out, const uint64_t* in, int64_t rows,
               const int32_t* mod_idx, int limbs, int offset, int inverse, void* stream);

/* ---- element-wise family: _kernels.mul_batch/neg_mul_batch/mul_add_batch
 *      (_kernels.py:141-173), fused_neg_multiply / fused_mul_add
 *      (rnspoly.py:295-308), add_arr/sub_arr/neg_arr (vecmod.py:155-165).
 *      out may alias a, b or c. */
int fhe_ewise(const FheChain* ch, int op, uint64_t* out, const uint64_t* a, const uint64_t* b,
              const uint64_t* c, int64_t rows, const int32_t* mod_idx, int limbs, int offset,
              int b_mode, void* stream);

/* ---- fused tensor product: ckks_multiply / ckks_square (ckks.py:308-366),
 *      bgv_multiply (bgv.py:171-186).  x, y: batch x (2, limbs, n);
 *      out: batch x (3, limbs, n); strides in words between batch items. */
int fhe_tensor(const FheChain* ch, uint64_t* out, const uint64_t* x, const uint64_t* y, int limbs,
               int64_t batch, int64_t x_stride, int64_t y_stride, int64_t out_stride, int square,
               void* stream);

/* ---- Galois automorphism gather: _apply_galois (ckks.py:413-422) with the
 *      index of Context.galois_perm (context.py:222-234).  out != in. */
int fhe_automorph(uint64_t* out, const uint64_t* in, int64_t rows, int log_n, uint64_t elt,
                  void* stream);

/* ---- context: chain Q = q_0..q_{L-1} followed by P = p_0..p_{K-1};
 *      key-switch digits of `alpha` consecutive Q primes.  (alpha=1, K=0)
 *      is exactly the reference gadget (keys.py:1-7, 128-141, 186-237). */
int fhe_context_create(const uint64_t* q_primes, int L, const uint64_t* p_primes, int K,
                       int alpha, int log_n, FheContext** out);
/* Build the BGV modulus-switch constants of plain modulus t (bgv.py:215-260)
 * now, so fhe_rescale(t_plain = t) never allocates; Context creation calls it
 * for its plain modulus.  Idempotent. */
/* ---- exact CRT lift of decrypted residues (the step after the path,
 *      SURVEY 8(f)2): replaces crt_reconstruct_poly (crt.py:84-100) in
 *        FHE_CRT_FLOAT  ckks_decode (ckks.py:157-166): double out[n] =
 *                       float(centred v) / scale (scale 0: no division)
 *        FHE_CRT_MOD_T  bgv_decrypt (bgv.py:89-101): u64 out[n] =
 *                       (centred v % t) * inv_f % t
 *        FHE_CRT_BFV    bfv_decrypt (bfv.py:106-117): u64 out[n] =
 *                       ((t * centred v + Q // 2) // Q) % t
 *      rows: the level coefficient-domain residue rows; Python integer
 *      semantics exactly (float() rounds to nearest even; +-inf where
 *      Python raises OverflowError). */
/* ---- device sampler: numpy Generator(Philox(SeedSequence)) replay
 *      (sampling.py:27-63, SURVEY 8(f)1 phase 2).  The state is numpy's
 *      Philox state (bit_generator.state: counter, key, buffer, buffer_pos,
 *      has_uint32, uinteger) and lives in DEVICE memory, so draws chain on
 *      the stream.  fhe_philox_integers writes Generator.integers(low,
 *      low + rng + 1, count) (endpoint excluded; 64-bit Lemire for
 *      rng > 2^32 - 1, else the buffered 32-bit path) as 64-bit words to out
 *      and advances the state exactly as numpy would.  A call whose
 *      candidate draws held too few accepted values (only possible for
 *      ranges with heavy Lemire rejection) leaves the state untouched and
 *      sets shortfall = 1. */
typedef struct FhePhilox {
  uint64_t counter[4];
  uint64_t key[2];
  uint64_t buffer[4];
  int32_t buffer_pos;
  int32_t has_uint32;
  uint32_t uinteger;
  int32_t shortfall;
} FhePhilox;
size_t fhe_philox_workspace(int64_t count, uint64_t rng);
int fhe_philox_integers(FhePhilox* dev_state, int64_t low, uint64_t rng, int64_t count,
                        uint64_t* out, void* workspace, size_t ws_bytes, void* stream);
/* cbd_error's combine (sampling.py:48-52): out[i] = sum of flip rows
 * 0..pairs-1 minus rows pairs..2 pairs-1 (flips: (2 pairs, n) words) */
int fhe_cbd_combine(int64_t* out, const uint64_t* flips, int pairs, int64_t n, void* stream);
/* CKKS encode's residue lift (ckks.py:104-136): values are the rounded
 * scaled coefficients (integer-valued doubles of any magnitude); out row j =
 * the exact integer mod q_(offset+j) (what the reference computes with
 * Python integers beyond 2^62) */
int fhe_real_lift(const FheChain* ch, uint64_t* out, const double* values, int64_t n, int limbs,
                  int offset, void* stream);
/* signed_to_residues (sampling.py:60-65): out row j = coeffs mod q_(offset+j) */
int fhe_signed_lift(const FheChain* ch, uint64_t* out, const int64_t* coeffs, int64_t n, int limbs,
                    int offset, void* stream);

/* ---- zlib CRC-32 of a device buffer (the CATF record checksum, serial.py:
 *      67-78), written to the device word *out: chunked on the device and
 *      merged with zlib's crc32_combine rule.  Lets a record body go from HBM
 *      into a pinned wire buffer without a host pass over it. */
size_t fhe_crc32_workspace(int64_t nbytes);
int fhe_crc32(const void* data, int64_t nbytes, uint32_t* out, void* workspace, size_t ws_bytes,
              void* stream);

enum { FHE_CRT_FLOAT = 0, FHE_CRT_MOD_T = 1, FHE_CRT_BFV = 2 };
int fhe_crt_lift(const FheContext* ctx, int mode, void* out, const uint64_t* rows, int level,
                 double scale, uint64_t t, uint64_t inv_f, void* stream);

int fhe_context_prepare_plain(FheContext* ctx, uint64_t t);
int fhe_context_destroy(FheContext* ctx);
const FheChain* fhe_context_chain(const FheContext* ctx);

/* ---- rescale: ckks_rescale (ckks.py:382-410); with t_plain != 0 the BGV
 *      modulus switch (bgv.py:215-260).  in: (polys, level, n) eval;
 *      out: (polys, level-1, n) eval; out must not alias in. */
size_t fhe_rescale_workspace(const FheContext* ctx, int polys, int level);
int fhe_rescale(const FheContext* ctx, uint64_t* out, const uint64_t* in, int polys, int level,
                uint64_t t_plain, void* workspace, size_t ws_bytes, void* stream);

/* ---- key switching: key_switch (keys.py:186-237) generalised to hybrid
 *      (ModUp -> inner product -> ModDown).  d: batch x (level, n) eval,
 *      stride d_stride words.  key: digits x (2, L+K, n) eval, contiguous.
 *      out0 = add0 + b, out1 = add1 + a (add0/add1 may be NULL, may alias
 *      out0/out1); batch items are add_stride / out_stride words apart.
 *      One key read serves the whole batch. */
size_t fhe_keyswitch_workspace(const FheContext* ctx, int level, int batch);
int fhe_keyswitch(const FheContext* ctx, int level, const uint64_t* d, int64_t d_stride,
                  const uint64_t* key, const uint64_t* add0, const uint64_t* add1,
                  int64_t add_stride, uint64_t* out0, uint64_t* out1, int64_t out_stride,
                  int batch, void* workspace, size_t ws_bytes, void* stream);

/* ---- fused HMult+Relin: ckks_multiply (ckks.py:308-349, tensor product)
 *      followed by ckks_relinearize (ckks.py:369-379) in one call.
 *      x, y: batch x (2, level, n) eval ciphertexts, in_stride words apart
 *      (y may equal x: squaring).  out0 = d0 + b, out1 = d1 + a with
 *      (d0, d1, d2) the tensor product and (b, a) the key switch of d2;
 *      out0/out1 may alias x's polys.  The words equal those of fhe_tensor
 *      followed by fhe_keyswitch; d0/d1 are formed in the key switch's
 *      finishing kernel and never written to HBM (FHE_HMULT_TENS=0: the
 *      tensor is materialised instead). */
size_t fhe_hmult_relin_workspace(const FheContext* ctx, int level, int batch);
int fhe_hmult_relin(const FheContext* ctx, int level, const uint64_t* x, const uint64_t* y,
                    int64_t in_stride, const uint64_t* key, uint64_t* out0, uint64_t* out1,
                    int64_t out_stride, int batch, void* workspace, size_t ws_bytes,
                    void* stream);

/* ---- BEHZ BFV multiplication (schemes/behz.py:58-270).  `big` is the
 *      chain Q | B | m_sk (L + S primes, S = |B| + 1).  Coefficient domain.
 *      lift : in (polys, L, n) -> out (polys, L + S, n)   extend_to_bsk
 *      floor: in (polys, L + S, n) tensor coefficients -> out (polys, L, n):
 *             round(t x / Q) via fast_floor_q + fast_conv_sk_to_q.
 *      `consts` is the device constant block documented in csrc/behz.cu. */
int fhe_behz_lift(const FheChain* big, uint64_t* out, const uint64_t* in, int polys, int L, int S,
                  const uint64_t* consts, void* stream);
int fhe_behz_floor(const FheChain* big, uint64_t* out, const uint64_t* in, int polys, int L, int S,
                   const uint64_t* consts, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FHE_SM100_H */

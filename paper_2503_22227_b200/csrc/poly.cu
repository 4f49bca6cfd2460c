// Element-wise RNS polynomial kernels: the add/sub/neg/mul family, the fused
// ciphertext tensor product, the Galois automorphism gather and the
// rescale / modulus-switch correction kernels.
//
// All of them are HBM-bound streaming kernels: 2 coefficients per thread per
// iteration through 16-byte vector accesses, grid-stride loops sized to a
// multiple of the SM count, per-row prime looked up once per 2 coefficients.
#include "fhe_internal.cuh"
#include "fhe_kernels.cuh"

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ u64 ew_apply(int op, u64 a, u64 b, u64 c, const ModConst& m) {
  const u64 q = m.q;
  switch (op) {
    case FHE_EW_ADD: return add_mod(a, b, q);
    case FHE_EW_SUB: return sub_mod(a, b, q);
    case FHE_EW_NEG: return neg_mod(a, q);
    case FHE_EW_MUL: return mul_mod(a, b, m);
    case FHE_EW_NEG_MUL: return neg_mod(mul_mod(a, b, m), q);
    case FHE_EW_MUL_ADD: return add_mod(mul_mod(a, b, m), c, q);
    case FHE_EW_MUL_SUB: return sub_mod(c, mul_mod(a, b, m), q);
    case FHE_EW_REDUCE: return reduce_word(a, m);
    default: return a;
  }
}

// out[r][i] = op(a[r][i], b[rb][i], c[r][i]) with rb = b_bcast ? r % limbs : r.
// For the *_CONST ops b is a per-chain-position constant vector (b[prime]).
__global__ void __launch_bounds__(kThreads)
    ewise_kernel(const DevChain ch, int op, u64* __restrict__ out, const u64* __restrict__ a,
                 const u64* __restrict__ b, const u64* __restrict__ c, long rows, int log_n,
                 RowMap map, int b_mode) {
  fhe_pdl_trigger();
  fhe_pdl_wait();
  const long half_n = 1L << (log_n - 1);
  const long total = rows * half_n;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long r = t >> (log_n - 1);
    const long off = t << 1;
    const int p = map((int)r);
    const ModConst m = ch.mc[p];
    const ulonglong2 va = reinterpret_cast<const ulonglong2*>(a)[t];
    ulonglong2 vb = make_ulonglong2(0, 0), vc = make_ulonglong2(0, 0);
    int eop = op;
    if (b_mode == FHE_B_CONST) {
      const u64 k = b[p];
      vb = make_ulonglong2(k, k);
    } else if (b_mode == FHE_B_BCAST) {
      const long rb = r % map.limbs;
      vb = reinterpret_cast<const ulonglong2*>(b)[(rb << (log_n - 1)) + (t & (half_n - 1))];
    } else if (b) {
      vb = reinterpret_cast<const ulonglong2*>(b)[t];
    }
    if (c) vc = reinterpret_cast<const ulonglong2*>(c)[t];
    ulonglong2 o;
    o.x = ew_apply(eop, va.x, vb.x, vc.x, m);
    o.y = ew_apply(eop, va.y, vb.y, vc.y, m);
    reinterpret_cast<ulonglong2*>(out)[t] = o;
    (void)off;
  }
}

// Fused tensor product of 2-component ciphertexts (ckks.py:308-366,
// bgv.py:171-186): d0 = x0 y0, d1 = x0 y1 + x1 y0, d2 = x1 y1, one launch,
// one read of each input limb and one write of each output limb.  The cross
// term is accumulated as a 128-bit sum and reduced once.
__global__ void __launch_bounds__(kThreads)
    tensor_kernel(const DevChain ch, u64* __restrict__ out, const u64* __restrict__ x,
                  const u64* __restrict__ y, int limbs, int log_n, long batch, long x_stride,
                  long y_stride, long out_stride, int square) {
  fhe_pdl_trigger();
  fhe_pdl_wait();
  const long n = 1L << log_n;
  const long per = (long)limbs << (log_n - 1);  // coefficient pairs per ciphertext
  const long total = batch * per;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long bi = t / per;
    const long w = t - bi * per;
    const int j = (int)(w >> (log_n - 1));
    const ModConst m = ch.mc[j];
    const u64* xb = x + bi * x_stride;
    const u64* yb = y + bi * y_stride;
    u64* ob = out + bi * out_stride;
    const long poly = (long)limbs * n;
    const ulonglong2 x0 = reinterpret_cast<const ulonglong2*>(xb)[w];
    const ulonglong2 x1 = reinterpret_cast<const ulonglong2*>(xb + poly)[w];
    ulonglong2 y0 = x0, y1 = x1;
    if (!square) {
      y0 = reinterpret_cast<const ulonglong2*>(yb)[w];
      y1 = reinterpret_cast<const ulonglong2*>(yb + poly)[w];
    }
    ulonglong2 d0, d1, d2;
    u64 h, l;
    d0.x = mul_mod(x0.x, y0.x, m);
    d0.y = mul_mod(x0.y, y0.y, m);
    d2.x = mul_mod(x1.x, y1.x, m);
    d2.y = mul_mod(x1.y, y1.y, m);
    mul_wide(x0.x, y1.x, h, l);
    mac_wide(h, l, x1.x, y0.x);
    d1.x = reduce_prod(h, l, m);
    mul_wide(x0.y, y1.y, h, l);
    mac_wide(h, l, x1.y, y0.y);
    d1.y = reduce_prod(h, l, m);
    reinterpret_cast<ulonglong2*>(ob)[w] = d0;
    reinterpret_cast<ulonglong2*>(ob + poly)[w] = d1;
    reinterpret_cast<ulonglong2*>(ob + 2 * poly)[w] = d2;
  }
}

// Galois automorphism x -> x^elt in the evaluation domain: out[j] = in[perm(j)]
// with perm(j) = pos[(exp_j * elt) mod 2N], exp_j = 2 bitrev(j) + 1
// (context.py:222-234, ckks.py:413-422).  The index is computed
// arithmetically instead of gathered from a host table.
__global__ void __launch_bounds__(kThreads)
    automorph_kernel(u64* __restrict__ out, const u64* __restrict__ in, long rows, int log_n,
                     u64 elt) {
  fhe_pdl_trigger();
  fhe_pdl_wait();
  const long n = 1L << log_n;
  const long total = rows * n;
  const u64 mask2n = (2UL << log_n) - 1;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long r = t >> log_n;
    const u32 j = (u32)(t & (n - 1));
    const u64 e = 2 * (u64)(__brev(j) >> (32 - log_n)) + 1;
    const u64 g = (e * elt) & mask2n;  // odd
    const u32 k = (u32)((g - 1) >> 1);
    const u32 src = __brev(k) >> (32 - log_n);
    out[t] = in[(r << log_n) + src];
  }
}

// Rescale / modulus-switch correction (ckks.py:382-410, bgv.py:215-260).
// Input: the coefficient-form last limb of each poly (q_last), output: the
// correction r_j (coefficient form) against each remaining prime q_j:
//   CKKS: r = [c_last]_centred mod q_j
//   BGV : w = [c_last * t^-1]_{q_last} centred; r = t * w mod q_j
__global__ void __launch_bounds__(kThreads)
    modswitch_expand_kernel(const DevChain ch, u64* __restrict__ corr,
                            const u64* __restrict__ last, int polys, int new_level, int log_n,
                            int last_prime, u64 t_plain, WPair tinv_last,
                            const u64* __restrict__ t_mod, const u64* __restrict__ qlast_mod) {
  fhe_pdl_trigger();
  fhe_pdl_wait();
  const long n = 1L << log_n;
  const long total = (long)polys * new_level * n;
  const u64 ql = ch.mc[last_prime].q;
  const u64 half = ql >> 1;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long i = t & (n - 1);
    const long pj = t >> log_n;
    const int j = (int)(pj % new_level);
    const long p = pj / new_level;
    const ModConst m = ch.mc[j];
    u64 c = last[p * n + i];
    u64 r;
    if (t_plain == 0) {
      r = reduce_word(c, m);
      if (c > half) r = sub_mod(r, qlast_mod[j], m.q);
    } else {
      const u64 w = shoup_mul(c, tinv_last.w, tinv_last.sh, ql);
      u64 wm = reduce_word(w, m);
      if (w > half) wm = sub_mod(wm, qlast_mod[j], m.q);
      r = mul_mod(wm, t_mod[j], m);
    }
    corr[t] = r;
  }
}

// out_j = (in_j - corr_j) * inv_j  (eval domain), per poly and limb j < new_level.
__global__ void __launch_bounds__(kThreads)
    modswitch_finish_kernel(const DevChain ch, u64* __restrict__ out, const u64* __restrict__ in,
                            const u64* __restrict__ corr, int polys, int level, int log_n,
                            const WPair* __restrict__ inv) {
  fhe_pdl_trigger();
  fhe_pdl_wait();
  const int new_level = level - 1;
  const long n = 1L << log_n;
  const long half_n = n >> 1;
  const long total = (long)polys * new_level * half_n;
  for (long t = blockIdx.x * (long)blockDim.x + threadIdx.x; t < total;
       t += (long)gridDim.x * blockDim.x) {
    const long i2 = t & (half_n - 1);
    const long pj = t >> (log_n - 1);
    const int j = (int)(pj % new_level);
    const long p = pj / new_level;
    const u64 q = ch.mc[j].q;
    const WPair w = inv[j];
    const ulonglong2 a =
        reinterpret_cast<const ulonglong2*>(in + (p * level + j) * n)[i2];
    const ulonglong2 c = reinterpret_cast<const ulonglong2*>(corr)[t];
    ulonglong2 o;
    o.x = shoup_mul(sub_mod(a.x, c.x, q), w.w, w.sh, q);
    o.y = shoup_mul(sub_mod(a.y, c.y, q), w.w, w.sh, q);
    reinterpret_cast<ulonglong2*>(out + (p * new_level + j) * n)[i2] = o;
  }
}

// One-kernel rescale body for rows that fit one CTA (N <= 2^12): CTA (j, p)
// expands the centred last limb of poly p mod q_j (modswitch_expand_kernel's
// formula), runs the forward NTT mod q_j in shared memory (Cooley-Tukey with
// psi_br[m + i], ntt.py:145-169, canonical butterflies) and applies the
// finish (in_j - corr_j) q_last^-1 -- the expanded and transformed
// correction never touches HBM, and the rescale is 2 launches instead of 4.
__global__ void __launch_bounds__(kThreads)
    rescale_small_kernel(const DevChain ch, u64* __restrict__ out, const u64* __restrict__ in,
                         const u64* __restrict__ last, int level, const WPair* __restrict__ inv,
                         const u64* __restrict__ qlast_mod) {
  extern __shared__ u64 rs_row[];
  const int j = blockIdx.x, p = blockIdx.y;
  const int new_level = level - 1;
  const int log_n = ch.log_n;
  const int n = 1 << log_n;
  const ModConst m = ch.mc[j];
  const u64 q = m.q;
  const u64 half = ch.mc[level - 1].q >> 1;
  const u64 qlm = qlast_mod[j];
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const u64 c = last[(long)p * n + i];
    u64 r = reduce_word(c, m);
    if (c > half) r = sub_mod(r, qlm, q);
    rs_row[i] = r;
  }
  __syncthreads();
  const WPair* tw = ch.tw + ((size_t)j << log_n);
  for (int mm = 1, t = n >> 1; mm < n; mm <<= 1, t >>= 1) {
    for (int k = threadIdx.x; k < (n >> 1); k += blockDim.x) {
      const int i = k / t, jj = 2 * i * t + (k - i * t);
      const WPair w = tw[mm + i];
      const u64 u = rs_row[jj];
      const u64 v = shoup_mul(rs_row[jj + t], w.w, w.sh, q);
      rs_row[jj] = add_mod(u, v, q);
      rs_row[jj + t] = sub_mod(u, v, q);
    }
    __syncthreads();
  }
  const WPair w = inv[j];
  const u64* src = in + ((long)p * level + j) * n;
  u64* dst = out + ((long)p * new_level + j) * n;
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    dst[i] = shoup_mul(sub_mod(src[i], rs_row[i], q), w.w, w.sh, q);
}

}  // namespace

int launch_rescale_small(const DevChain& ch, u64* out, const u64* in, const u64* last, int polys,
                         int level, const WPair* inv, const u64* qlast_mod, cudaStream_t st) {
  if (ch.log_n > 12) {
    fhe_set_error("rescale_small: N > 2^12");
    return -1;
  }
  if (polys <= 0 || level < 2) return 0;
  dim3 grid(level - 1, polys);
  rescale_small_kernel<<<grid, kThreads, ((size_t)1 << ch.log_n) * sizeof(u64), st>>>(
      ch, out, in, last, level, inv, qlast_mod);
  FHE_LAUNCH_CHECK();
  return 0;
}

bool fhe_pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FHE_PDL");
    on = (e && e[0] == '1') ? 1 : 0;
  }
  return on == 1;
}

int grid_for(long work) {
  // enough CTAs for 8 resident per SM on 148 SMs, no more than the work needs
  long g = (work + kThreads - 1) / kThreads;
  const long cap = 148L * 8 * 4;
  return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

int launch_ewise(const DevChain& ch, int op, u64* out, const u64* a, const u64* b, const u64* c,
                 long rows, RowMap map, int b_mode, cudaStream_t st) {
  if (rows <= 0) return 0;
  const long work = rows << (ch.log_n - 1);
  fhe_launch(ewise_kernel, dim3(grid_for(work)), dim3(kThreads), 0, st, ch, op, out, a, b, c, rows,
             ch.log_n, map, b_mode);
  FHE_LAUNCH_CHECK();
  return 0;
}

int launch_tensor(const DevChain& ch, u64* out, const u64* x, const u64* y, int limbs, long batch,
                  long x_stride, long y_stride, long out_stride, int square, cudaStream_t st) {
  const long work = batch * ((long)limbs << (ch.log_n - 1));
  if (work <= 0) return 0;
  fhe_launch(tensor_kernel, dim3(grid_for(work)), dim3(kThreads), 0, st, ch, out, x, y, limbs,
             ch.log_n, batch, x_stride, y_stride, out_stride, square);
  FHE_LAUNCH_CHECK();
  return 0;
}

int launch_automorph(u64* out, const u64* in, long rows, int log_n, u64 elt, cudaStream_t st) {
  const long work = rows << log_n;
  if (work <= 0) return 0;
  fhe_launch(automorph_kernel, dim3(grid_for(work)), dim3(kThreads), 0, st, out, in, rows, log_n,
             elt);
  FHE_LAUNCH_CHECK();
  return 0;
}

int launch_modswitch_expand(const DevChain& ch, u64* corr, const u64* last, int polys,
                            int new_level, int last_prime, u64 t_plain, WPair tinv_last,
                            const u64* t_mod, const u64* qlast_mod, cudaStream_t st) {
  const long work = ((long)polys * new_level) << ch.log_n;
  fhe_launch(modswitch_expand_kernel, dim3(grid_for(work)), dim3(kThreads), 0, st, ch, corr, last,
             polys, new_level, ch.log_n, last_prime, t_plain, tinv_last, t_mod, qlast_mod);
  FHE_LAUNCH_CHECK();
  return 0;
}

int launch_modswitch_finish(const DevChain& ch, u64* out, const u64* in, const u64* corr,
                            int polys, int level, const WPair* inv, cudaStream_t st) {
  const long work = ((long)polys * (level - 1)) << (ch.log_n - 1);
  fhe_launch(modswitch_finish_kernel, dim3(grid_for(work)), dim3(kThreads), 0, st, ch, out, in,
             corr, polys, level, ch.log_n, inv);
  FHE_LAUNCH_CHECK();
  return 0;
}

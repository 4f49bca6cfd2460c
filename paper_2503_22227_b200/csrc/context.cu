// Host precompute for chains and contexts, uploaded once to HBM.
//
// Mirrors the reference's one-off precompute:
//   NttTables (coremath/ntt.py:52-137): psi = smallest primitive 2N-th root
//     (primes.py:60-71), bit-reversed powers of psi and psi^-1, Shoup
//     companions floor(w 2^64 / q) (vecmod.py:141-145), n^-1;
//   Context.last_inv (context.py:186-198) for rescale;
//   key-switch constants: for the hybrid gadget the punctured products of
//     each digit (the fast-base-conversion weights of behz.py:131-153 applied
//     to Q_d and to P); for (alpha=1, K=0) they degenerate to the identity,
//     which is the reference's per-prime gadget (keys.py:186-237).
// All arithmetic is exact unsigned __int128 host code.
#include <algorithm>
#include <cstring>
#include <stdexcept>

#include "fhe_context.cuh"
#include "ntt_plan.cuh"

namespace {

typedef unsigned __int128 u128;

u64 mulmod_h(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
u64 powmod_h(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod_h(r, a, q);
    a = mulmod_h(a, a, q);
    e >>= 1;
  }
  return r;
}
u64 invmod_h(u64 a, u64 q) {
  if (a % q == 0) throw std::runtime_error("non-invertible value");
  return powmod_h(a, q - 2, q);
}
u64 shoup_h(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
WPair wpair(u64 w, u64 q) { return WPair{w, shoup_h(w, q)}; }
int bitlen(u64 x) { return 64 - __builtin_clzll(x); }

ModConst make_mc(u64 q) {
  ModConst m;
  m.q = q;
  m.s = (u32)(bitlen(q) - 1);
  m.mu = (u64)(((u128)1 << (64 + m.s)) / q);
  m.r64 = (u64)(((u128)1 << 64) % q);
  m.pad = 0;
  return m;
}

u32 bitrev(u32 x, int bits) {
  u32 r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}

// primes.py:45-71: first g whose cofactor power is a primitive root, then
// the numerically smallest odd power of it.
u64 min_primitive_root_h(u64 q, u64 order) {
  if ((q - 1) % order != 0) throw std::runtime_error("prime is not NTT friendly for this degree");
  const u64 cof = (q - 1) / order;
  u64 root = 0;
  for (u64 g = 2; g < q; ++g) {
    const u64 r = powmod_h(g, cof, q);
    if (powmod_h(r, order / 2, q) == q - 1) {
      root = r;
      break;
    }
  }
  if (!root) throw std::runtime_error("no primitive root");
  u64 best = root, cur = root;
  const u64 gsq = mulmod_h(root, root, q);
  for (u64 k = 0; k + 1 < order / 2; ++k) {
    cur = mulmod_h(cur, gsq, q);
    if (cur < best) best = cur;
  }
  return best;
}

// simple bump allocator for packing constants into one device upload
struct Packer {
  std::vector<unsigned char> buf;
  size_t add(const void* p, size_t bytes) {
    size_t off = (buf.size() + 255) & ~(size_t)255;
    buf.resize(off + bytes);
    if (bytes) std::memcpy(buf.data() + off, p, bytes);
    return off;
  }
  template <class T>
  size_t addv(const std::vector<T>& v) {
    return add(v.data(), v.size() * sizeof(T));
  }
};

}  // namespace

int build_chain(const u64* primes, int count, int log_n, FheChain* ch) {
  const size_t n = (size_t)1 << log_n;
  ch->log_n = log_n;
  ch->primes.assign(primes, primes + count);
  ch->psi.resize(count);
  std::vector<ModConst> mc(count);
  std::vector<WPair> tw(count * n), itw(count * n), ninv(count), ninv_w1(count);
  for (int p = 0; p < count; ++p) {
    const u64 q = primes[p];
    if (q < 3 || q >= ((u64)1 << 62) || !(q & 1)) {
      fhe_set_error("modulus out of supported range [3, 2^62) or even");
      return -1;
    }
    mc[p] = make_mc(q);
    u64 psi;
    try {
      psi = min_primitive_root_h(q, 2 * n);
    } catch (const std::exception& e) {
      fhe_set_error(e.what());
      return -1;
    }
    ch->psi[p] = psi;
    const u64 ipsi = invmod_h(psi, q);
    std::vector<u64> fw(n), iv(n);
    u64 a = 1, ia = 1;
    for (size_t i = 0; i < n; ++i) {
      fw[i] = a;
      iv[i] = ia;
      a = mulmod_h(a, psi, q);
      ia = mulmod_h(ia, ipsi, q);
    }
    for (size_t i = 0; i < n; ++i) {
      const u32 br = bitrev((u32)i, log_n);
      tw[p * n + i] = wpair(fw[br], q);
      itw[p * n + i] = wpair(iv[br], q);
    }
    const u64 ni = invmod_h(n % q, q);
    ninv[p] = wpair(ni, q);
    const u64 w1 = n >= 2 ? itw[p * n + 1].w : 1;
    ninv_w1[p] = wpair(mulmod_h(w1, ni, q), q);
  }
  // FP64 tables are built for every prime below 2^50; the chain is an FP64
  // chain (fp64_ok) when all are.  A mixed chain (e.g. 50-bit Q, 60-bit P)
  // still runs the transforms whose rows all use eligible primes on the FP64
  // path (launch_ntt); everything else stays on the integer path.
  bool fp64 = true, fp64_any = false;
  ch->fp64_prime.assign(count, 0);
  for (int p = 0; p < count; ++p) {
    const bool e = primes[p] < ((u64)1 << 50);
    ch->fp64_prime[p] = e ? 1 : 0;
    fp64 &= e;
    fp64_any |= e;
  }
  std::vector<double2> twd, itwd, tws, qd(count), nid(count), nwd(count);
  // staged tables: per prime and direction N1 column pairs + N chunk pairs
  // (N <= 2^12: the whole-row plan's table, n pairs per direction)
  const size_t tws_dir = log_n >= 13 ? n + ((size_t)1 << split_log_n1(log_n)) : n;
  if (fp64_any) {
    twd.assign(count * n, make_double2(0.0, 0.0));
    itwd.assign(count * n, make_double2(0.0, 0.0));
    tws.assign(count * 2 * tws_dir, make_double2(0.0, 0.0));
    for (int p = 0; p < count; ++p) {
      if (!ch->fp64_prime[p]) continue;
      const double q = (double)primes[p];
      // signed representatives |w| <= q/2: |x w / q| <= |x| / 2, so the FP64
      // butterflies accept inputs up to 2^52 (lazier reductions, ntt.cu)
      const u64 qi = primes[p];
      auto sd = [&](u64 w) {
        const double v = w > qi / 2 ? -(double)(qi - w) : (double)w;
        return make_double2(v, v / q);
      };
      for (size_t i = 0; i < n; ++i) {
        twd[p * n + i] = sd(tw[p * n + i].w);
        itwd[p * n + i] = sd(itw[p * n + i].w);
      }
      qd[p] = make_double2(q, 1.0 / q);
      if (log_n >= 13) {
        // staged-order tables of the four-step kernels: column part (N1
        // pairs) then one S-pair block per chunk; see ntt_plan.cuh
        const int l1 = split_log_n1(log_n), ls = log_n - l1;
        const size_t n1 = (size_t)1 << l1, s_ = (size_t)1 << ls;
        double2* f = &tws[p * 2 * tws_dir];
        double2* iv = &tws[p * 2 * tws_dir + tws_dir];
        auto put = [&](size_t dst, size_t src_idx) {
          f[dst] = twd[p * n + src_idx];
          iv[dst] = itwd[p * n + src_idx];
        };
        for (int s = 0; s < l1; ++s)
          for (int j = 0; j < (1 << s); ++j) put((1u << s) + staged_perm(l1, s, j), (1u << s) + j);
        for (size_t ck = 0; ck < n1; ++ck)
          for (int s = 0; s < ls; ++s)
            for (int j = 0; j < (1 << s); ++j)
              put(n1 + ck * s_ + (1u << s) + staged_perm(ls, s, j), ((n1 + ck) << s) + j);
      } else {
        // whole-row tiles (RowsTile, one row per tile at N = 2^12)
        double2* f = &tws[p * 2 * tws_dir];
        double2* iv = &tws[p * 2 * tws_dir + tws_dir];
        for (int s = 0; s < log_n; ++s)
          for (int j = 0; j < (1 << s); ++j) {
            const size_t d = (1u << s) + staged_perm(log_n, s, j, FHE_ROW_MAXE);
            f[d] = twd[p * n + (1u << s) + j];
            iv[d] = itwd[p * n + (1u << s) + j];
          }
      }
      nid[p] = sd(ninv[p].w);
      nwd[p] = sd(ninv_w1[p].w);
    }
  }
  Packer pk;
  const size_t o_mc = pk.addv(mc), o_tw = pk.addv(tw), o_itw = pk.addv(itw),
               o_ni = pk.addv(ninv), o_nw = pk.addv(ninv_w1);
  const size_t o_twd = pk.addv(twd), o_itwd = pk.addv(itwd), o_qd = pk.addv(qd),
               o_nid = pk.addv(nid), o_nwd = pk.addv(nwd), o_tws = pk.addv(tws);
  void* d = nullptr;
  FHE_CUDA_CHECK(cudaMalloc(&d, pk.buf.size()));
  FHE_CUDA_CHECK(cudaMemcpy(d, pk.buf.data(), pk.buf.size(), cudaMemcpyHostToDevice));
  unsigned char* b = (unsigned char*)d;
  ch->dmem = d;
  ch->dbytes = pk.buf.size();
  ch->dev.count = count;
  ch->dev.log_n = log_n;
  ch->dev.mc = (const ModConst*)(b + o_mc);
  ch->dev.tw = (const WPair*)(b + o_tw);
  ch->dev.itw = (const WPair*)(b + o_itw);
  ch->dev.ninv = (const WPair*)(b + o_ni);
  ch->dev.ninv_w1 = (const WPair*)(b + o_nw);
  ch->dev.lazy_ok = true;
  for (int p = 0; p < count; ++p) ch->dev.lazy_ok &= primes[p] < ((u64)1 << 58);
  ch->dev.fp64_ok = fp64;
  ch->dev.twd = fp64_any ? (const double2*)(b + o_twd) : nullptr;
  ch->dev.itwd = fp64_any ? (const double2*)(b + o_itwd) : nullptr;
  ch->dev.qd = fp64_any ? (const double2*)(b + o_qd) : nullptr;
  ch->dev.ninv_d = fp64_any ? (const double2*)(b + o_nid) : nullptr;
  ch->dev.ninv_w1_d = fp64_any ? (const double2*)(b + o_nwd) : nullptr;
  ch->dev.tws = fp64_any ? (const double2*)(b + o_tws) : nullptr;
  ch->dev.fp64_prime_host = ch->fp64_prime.data();
  ch->dev.tws_dir = (long)tws_dir;
  ch->dev.fuse = fuse_scratch_new(log_n);
  if (!ch->dev.fuse) {
    fhe_set_error("fused NTT scratch allocation failed");
    return -2;
  }
  return 0;
}

void free_chain(FheChain* ch) {
  if (ch) {
    fuse_scratch_free(ch->dev.fuse);
    ch->dev.fuse = nullptr;
  }
  if (ch && ch->dmem) cudaFree(ch->dmem);
  if (ch) ch->dmem = nullptr;
}

// Packed mma.sync m16n8k32 B fragments of the byte-split conversion matrix
// W'[(s, a)][(t, b)] = byte b of [w(s, t) 2^(8a)]_{p(t)} (bconv_imma.cuh):
// per target t and k-step, lane (gr = lane / 4 = byte b, gq = lane % 4) holds
// rows k = 32 ks + 4 gq + i (b0) and + 16 (b1), byte i = row k's byte.
template <class W, class P>
static void pack_bfrag(std::vector<uint2>& out, int ns, int nt, int ks, W w, P p) {
  std::vector<u64> v((size_t)ns * 7 * nt);
  for (int s = 0; s < ns; ++s)
    for (int t = 0; t < nt; ++t) {
      const u64 pt = p(t);
      u64 x = w(s, t) % pt;
      for (int a = 0; a < 7; ++a) {
        v[((size_t)s * 7 + a) * nt + t] = x;
        x = mulmod_h(x, 256 % pt, pt);
      }
    }
  auto byte = [&](int k, int t, int b) -> unsigned {
    if (k >= 7 * ns || b >= 7) return 0;
    return (unsigned)((v[(size_t)k * nt + t] >> (8 * b)) & 0xff);
  };
  for (int t = 0; t < nt; ++t)
    for (int kk = 0; kk < ks; ++kk)
      for (int lane = 0; lane < 32; ++lane) {
        const int gq = lane & 3, gr = lane >> 2;
        unsigned b0 = 0, b1 = 0;
        for (int i = 0; i < 4; ++i) {
          const int k0 = 32 * kk + 4 * gq + i;
          b0 |= byte(k0, t, gr) << (8 * i);
          b1 |= byte(k0 + 16, t, gr) << (8 * i);
        }
        out.push_back(make_uint2(b0, b1));
      }
}

// The same matrix packed for bconv_imma2_kernel: n8 tile (group g, byte b)
// holds columns (target 8 g + n, byte b), n = lane / 4; tiles ordered
// [g][b][ks][lane].
template <class W, class P>
static void pack_bfrag2(std::vector<uint2>& out, int ns, int nt, int ks, W w, P p) {
  std::vector<u64> v((size_t)ns * 7 * nt);
  for (int s = 0; s < ns; ++s)
    for (int t = 0; t < nt; ++t) {
      const u64 pt = p(t);
      u64 x = w(s, t) % pt;
      for (int a = 0; a < 7; ++a) {
        v[((size_t)s * 7 + a) * nt + t] = x;
        x = mulmod_h(x, 256 % pt, pt);
      }
    }
  auto byte = [&](int k, int t, int b) -> unsigned {
    if (k >= 7 * ns || t >= nt) return 0;
    return (unsigned)((v[(size_t)k * nt + t] >> (8 * b)) & 0xff);
  };
  const int ng = (nt + 7) / 8;
  for (int g = 0; g < ng; ++g)
    for (int b = 0; b < 7; ++b)
      for (int kk = 0; kk < ks; ++kk)
        for (int lane = 0; lane < 32; ++lane) {
          const int gq = lane & 3, t = 8 * g + (lane >> 2);
          unsigned b0 = 0, b1 = 0;
          for (int i = 0; i < 4; ++i) {
            const int k0 = 32 * kk + 4 * gq + i;
            b0 |= byte(k0, t, b) << (8 * i);
            b1 |= byte(k0 + 16, t, b) << (8 * i);
          }
          out.push_back(make_uint2(b0, b1));
        }
}

// The same matrix as B operand of the tcgen05 u8 MMA (bconv_umma.cuh): row
// (target t, byte b) = t * 8 + b (b = 7 and t >= nt zero), K-major over
// k = 7 s + a, in the canonical no-swizzle layout [k16 chunk][t][b][16 B]
// with the target count padded to a multiple of 8 (whole MMA chunks).
template <class W, class P>
static void pack_bumma(std::vector<uint4>& out, int ns, int nt, int ks, W w, P p, int sb = 7) {
  // sb bytes per source word (7: sources < 2^56, 8: wider); byte columns b =
  // 0..7 of each target ([w 2^(8a)]_p has a nonzero byte 7 only for p >= 2^56)
  std::vector<u64> v((size_t)ns * sb * nt);
  for (int s = 0; s < ns; ++s)
    for (int t = 0; t < nt; ++t) {
      const u64 pt = p(t);
      u64 x = w(s, t) % pt;
      for (int a = 0; a < sb; ++a) {
        v[((size_t)s * sb + a) * nt + t] = x;
        x = mulmod_h(x, 256 % pt, pt);
      }
    }
  auto byte = [&](int k, int t, int b) -> unsigned {
    if (k >= sb * ns || t >= nt) return 0;
    return (unsigned)((v[(size_t)k * nt + t] >> (8 * b)) & 0xff);
  };
  const int ng = (nt + 7) & ~7;
  for (int kc = 0; kc < 2 * ks; ++kc)
    for (int t = 0; t < ng; ++t)
      for (int b = 0; b < 8; ++b) {
        unsigned wd[4] = {0, 0, 0, 0};
        for (int i = 0; i < 16; ++i) wd[i / 4] |= byte(16 * kc + i, t, b) << (8 * (i % 4));
        out.push_back(make_uint4(wd[0], wd[1], wd[2], wd[3]));
      }
}

// Product of primes[idx] for idx in [lo, hi) except `skip`, reduced mod m.
static u64 punct_mod(const std::vector<u64>& primes, int lo, int hi, int skip, u64 m) {
  u64 r = 1 % m;
  for (int i = lo; i < hi; ++i)
    if (i != skip) r = mulmod_h(r, primes[i] % m, m);
  return r;
}

int build_levels(FheContext* ctx) {
  const int L = ctx->L, K = ctx->K, A = ctx->alpha;
  const std::vector<u64>& pr = ctx->chain->primes;  // Q then P
  ctx->levels.resize(L + 1);
  for (int l = 1; l <= L; ++l) {
    LevelPlan& lp = ctx->levels[l];
    lp.level = l;
    lp.digits = (l + A - 1) / A;
    const int D = lp.digits;
    std::vector<WPair> up_inv(l);
    std::vector<u64> up_w;
    std::vector<int32_t> ext_prime;
    std::vector<int> info(4 * D);
    int row_off = 0;
    auto cp = [&](int m) { return m < l ? m : L + (m - l); };
    for (int di = 0; di < D; ++di) {
      const int s0 = di * A, na = std::min(A, l - s0), nt = l + K - na;
      lp.dig_s0.push_back(s0);
      lp.dig_na.push_back(na);
      lp.dig_row_off.push_back(row_off);
      lp.dig_w_off.push_back((int)up_w.size());
      info[4 * di + 0] = s0;
      info[4 * di + 1] = na;
      info[4 * di + 2] = row_off;
      info[4 * di + 3] = (int)up_w.size();
      for (int s = s0; s < s0 + na; ++s)
        up_inv[s] = wpair(invmod_h(punct_mod(pr, s0, s0 + na, s, pr[s]), pr[s]), pr[s]);
      for (int s = s0; s < s0 + na; ++s)
        for (int t = 0; t < nt; ++t) {
          const int m = t < s0 ? t : t + na;
          up_w.push_back(punct_mod(pr, s0, s0 + na, s, pr[cp(m)]));
        }
      for (int t = 0; t < nt; ++t) {
        const int m = t < s0 ? t : t + na;
        ext_prime.push_back(cp(m));
      }
      row_off += nt;
    }
    lp.ext_rows = row_off;
    std::vector<WPair> down_inv(K), p_inv(l);
    std::vector<u64> down_w((size_t)K * l);
    for (int k = 0; k < K; ++k) {
      const u64 pk = pr[L + k];
      down_inv[k] = wpair(invmod_h(punct_mod(pr, L, L + K, L + k, pk), pk), pk);
      for (int j = 0; j < l; ++j) down_w[(size_t)k * l + j] = punct_mod(pr, L, L + K, L + k, pr[j]);
    }
    for (int j = 0; j < l; ++j) {
      const u64 pm = punct_mod(pr, L, L + K, -1, pr[j]);
      p_inv[j] = wpair(invmod_h(pm, pr[j]), pr[j]);
    }
    std::vector<WPair> rs_inv(std::max(l - 1, 0));
    std::vector<u64> rs_qlast(std::max(l - 1, 0));
    for (int j = 0; j + 1 < l; ++j) {
      rs_inv[j] = wpair(invmod_h(pr[l - 1] % pr[j], pr[j]), pr[j]);
      rs_qlast[j] = pr[l - 1] % pr[j];
    }
    // FP64 pairs (value, value / modulus) for the FP64-pipe base conversions
    const bool fp64 = ctx->chain->dev.fp64_ok;
    // Q-side FP64 constants (rescale and ModDown finish) also on a mixed chain
    // whose level-l Q primes are all < 2^50
    bool q_fp64 = true;
    for (int j = 0; j < l; ++j) q_fp64 &= ctx->chain->fp64_prime[j] != 0;
    std::vector<double2> up_inv_d, up_w_d, down_inv_d, down_w_d, p_inv_d, rs_inv_d;
    if (fp64 || q_fp64) {
      for (int j = 0; j + 1 < l; ++j)
        rs_inv_d.push_back(make_double2((double)rs_inv[j].w, (double)rs_inv[j].w / (double)pr[j]));
      for (int j = 0; j < l; ++j)
        p_inv_d.push_back(make_double2((double)p_inv[j].w, (double)p_inv[j].w / (double)pr[j]));
    }
    if (fp64) {
      for (int s = 0; s < l; ++s)
        up_inv_d.push_back(make_double2((double)up_inv[s].w, (double)up_inv[s].w / (double)pr[s]));
      for (int di = 0; di < D; ++di) {
        const int s0 = lp.dig_s0[di], na = lp.dig_na[di], nt = l + K - na;
        for (int s = 0; s < na; ++s)
          for (int t = 0; t < nt; ++t) {
            const int m = t < s0 ? t : t + na;
            const u64 w = up_w[lp.dig_w_off[di] + s * nt + t];
            up_w_d.push_back(make_double2((double)w, (double)w / (double)pr[cp(m)]));
          }
      }
      for (int k = 0; k < K; ++k)
        down_inv_d.push_back(
            make_double2((double)down_inv[k].w, (double)down_inv[k].w / (double)pr[L + k]));
      for (int k = 0; k < K; ++k)
        for (int j = 0; j < l; ++j) {
          const u64 w = down_w[(size_t)k * l + j];
          down_w_d.push_back(make_double2((double)w, (double)w / (double)pr[j]));
        }
    }
    // tensor-core base conversion tables: every prime in [2^39, 2^62); the
    // mma.sync kernels need all < 2^56 (narrow), the tcgen05 kernel also takes
    // wider primes (8-byte source words, 79-bit sums before the reduction)
    bool bf_ok = K <= 16, narrow = true, q_narrow = true, p_narrow = true;
    for (int j = 0; j < L + K; ++j) {
      const u64 q = pr[j];
      bf_ok &= q < ((u64)1 << 62) && q >= ((u64)1 << 39);
      const bool nq = q < ((u64)1 << 56);
      narrow &= nq;
      (j < L ? q_narrow : p_narrow) &= nq;
    }
    lp.bf_wide = !narrow;
    lp.up_sb = q_narrow ? 7 : 8;
    lp.down_sb = p_narrow ? 7 : 8;
    std::vector<uint2> up_bf, down_bf, up_bf2, down_bf2;
    std::vector<int> up_bf_off, up_bf2_off, up_bu_off;
    std::vector<uint4> up_bu, down_bu;
    if (bf_ok) {
      int max_na = 0;
      for (int di = 0; di < D; ++di) max_na = std::max(max_na, lp.dig_na[di]);
      bf_ok = lp.up_sb * max_na <= 128 && lp.down_sb * K <= 128;  // <= 4 K-steps
      lp.max_na = max_na;
      lp.up_ks = (lp.up_sb * max_na + 31) / 32;
      lp.down_ks = (lp.down_sb * K + 31) / 32;
      for (int di = 0; bf_ok && di < D; ++di) {
        const int s0 = lp.dig_s0[di], na = lp.dig_na[di], nt = l + K - na;
        up_bf_off.push_back((int)up_bf.size());
        up_bf2_off.push_back((int)up_bf2.size());
        auto wf = [&](int s, int t) { return up_w[lp.dig_w_off[di] + s * nt + t]; };
        auto pf = [&](int t) { return pr[cp(t < s0 ? t : t + na)]; };
        if (narrow) {
          pack_bfrag(up_bf, na, nt, lp.up_ks, wf, pf);
          pack_bfrag2(up_bf2, na, nt, lp.up_ks, wf, pf);
        }
        up_bu_off.push_back((int)up_bu.size());
        pack_bumma(up_bu, na, nt, lp.up_ks, wf, pf, lp.up_sb);
      }
      if (K > 0) {
        auto wf = [&](int k, int j) { return down_w[(size_t)k * l + j]; };
        auto pf = [&](int j) { return pr[j]; };
        if (narrow) {
          pack_bfrag(down_bf, K, l, lp.down_ks, wf, pf);
          pack_bfrag2(down_bf2, K, l, lp.down_ks, wf, pf);
        }
        pack_bumma(down_bu, K, l, lp.down_ks, wf, pf, lp.down_sb);
      }
    }
    lp.bf_ok = bf_ok;
    // exact CRT lift constants of Q_l = q_0 ... q_{l-1} (multi-limb, little endian)
    int qbits = 0;
    for (int j = 0; j < l; ++j) qbits += 64 - __builtin_clzll(pr[j]);
    const int W = (qbits + 6 + 63) / 64 + 1;  // sum_i y_i Q/q_i < l Q max q / min q, plus a sign bit
    auto mul_word = [&](std::vector<u64>& a, u64 w) {
      u128 carry = 0;
      for (auto& x : a) {
        const u128 v = (u128)x * w + carry;
        x = (u64)v;
        carry = v >> 64;
      }
    };
    std::vector<u64> crt_Q(W, 0), crt_Qh(W, 0), crt_M((size_t)l * W, 0);
    crt_Q[0] = 1;
    for (int j = 0; j < l; ++j) mul_word(crt_Q, pr[j]);
    for (int k = 0; k < W; ++k) crt_Qh[k] = (crt_Q[k] >> 1) | (k + 1 < W ? crt_Q[k + 1] << 63 : 0);
    std::vector<WPair> crt_inv(l);
    std::vector<double> crt_qinv(l);
    for (int i = 0; i < l; ++i) {
      std::vector<u64> m(W, 0);
      m[0] = 1;
      for (int j = 0; j < l; ++j)
        if (j != i) mul_word(m, pr[j]);
      std::copy(m.begin(), m.end(), crt_M.begin() + (size_t)i * W);
      crt_inv[i] = wpair(invmod_h(punct_mod(pr, 0, l, i, pr[i]), pr[i]), pr[i]);
      crt_qinv[i] = 1.0 / (double)pr[i];
    }
    int hq = W - 1;
    while (hq > 0 && crt_Q[hq] == 0) --hq;
    const int qdrop = std::max(0, hq - 1);
    double qd = 0.0;
    for (int k = hq; k >= qdrop; --k) qd = qd * 18446744073709551616.0 + (double)crt_Q[k];
    lp.crt_W = W;
    lp.crt_Qd = qd;
    lp.crt_qdrop = qdrop;
    Packer pk;
    const size_t o14 = pk.addv(up_bf), o15 = pk.addv(up_bf_off), o16 = pk.addv(down_bf);
    const size_t o22 = pk.addv(up_bf2), o23 = pk.addv(up_bf2_off), o24 = pk.addv(down_bf2);
    const size_t o25 = pk.addv(up_bu), o26 = pk.addv(up_bu_off), o27 = pk.addv(down_bu);
    const size_t o17 = pk.addv(crt_M), o18 = pk.addv(crt_Q), o19 = pk.addv(crt_Qh),
                 o20 = pk.addv(crt_inv), o21 = pk.addv(crt_qinv);
    const size_t o1 = pk.addv(up_inv), o2 = pk.addv(up_w), o3 = pk.addv(ext_prime),
                 o4 = pk.addv(info), o5 = pk.addv(down_inv), o6 = pk.addv(down_w),
                 o7 = pk.addv(p_inv), o8 = pk.addv(rs_inv), o9 = pk.addv(rs_qlast);
    const size_t o10 = pk.addv(up_inv_d), o11 = pk.addv(up_w_d), o12 = pk.addv(down_inv_d),
                 o13 = pk.addv(down_w_d), o28 = pk.addv(p_inv_d), o29 = pk.addv(rs_inv_d);
    void* d = nullptr;
    FHE_CUDA_CHECK(cudaMalloc(&d, pk.buf.size()));
    FHE_CUDA_CHECK(cudaMemcpy(d, pk.buf.data(), pk.buf.size(), cudaMemcpyHostToDevice));
    unsigned char* b = (unsigned char*)d;
    lp.dmem = d;
    lp.up_inv = (const WPair*)(b + o1);
    lp.up_w = (const u64*)(b + o2);
    lp.ext_prime = (const int32_t*)(b + o3);
    lp.dig_info = (const int*)(b + o4);
    lp.down_inv = (const WPair*)(b + o5);
    lp.down_w = (const u64*)(b + o6);
    lp.p_inv = (const WPair*)(b + o7);
    lp.rs_inv = (const WPair*)(b + o8);
    lp.rs_qlast = (const u64*)(b + o9);
    lp.crt_M = (const u64*)(b + o17);
    lp.crt_Q = (const u64*)(b + o18);
    lp.crt_Qh = (const u64*)(b + o19);
    lp.crt_inv = (const WPair*)(b + o20);
    lp.crt_qinv = (const double*)(b + o21);
    if (bf_ok && !lp.bf_wide) {  // mma.sync fragments: narrow chains only
      lp.up_bf = (const uint2*)(b + o14);
      lp.up_bf_off = (const int*)(b + o15);
      lp.down_bf = K > 0 ? (const uint2*)(b + o16) : nullptr;
      lp.up_bf2 = (const uint2*)(b + o22);
      lp.up_bf2_off = (const int*)(b + o23);
      lp.down_bf2 = K > 0 ? (const uint2*)(b + o24) : nullptr;
    }
    if (bf_ok) {
      lp.up_bu = (const uint4*)(b + o25);
      lp.up_bu_off = (const int*)(b + o26);
      lp.down_bu = K > 0 ? (const uint4*)(b + o27) : nullptr;
    }
    if (fp64) {
      lp.up_inv_d = (const double2*)(b + o10);
      lp.up_w_d = (const double2*)(b + o11);
      lp.down_inv_d = (const double2*)(b + o12);
      lp.down_w_d = (const double2*)(b + o13);
    }
    if (fp64 || q_fp64) {
      lp.p_inv_d = (const double2*)(b + o28);
      lp.rs_inv_d = l > 1 ? (const double2*)(b + o29) : nullptr;
    }
  }
  return 0;
}

const PlainPlan* get_plain_plan(FheContext* ctx, u64 t) {
  std::lock_guard<std::mutex> g(ctx->plain_mu);
  auto it = ctx->plain.find(t);
  if (it != ctx->plain.end()) return it->second.get();
  auto pp = std::make_unique<PlainPlan>();
  const std::vector<u64>& pr = ctx->chain->primes;
  pp->dmem.assign(ctx->L + 1, nullptr);
  pp->t_mod.assign(ctx->L + 1, nullptr);
  pp->tinv_last.assign(ctx->L + 1, WPair{0, 0});
  // every level's (t mod q_j) table in one allocation: level l at offset
  // (l - 2)(l - 1) / 2 words
  std::vector<u64> all;
  for (int l = 2; l <= ctx->L; ++l) {
    for (int j = 0; j + 1 < l; ++j) all.push_back(t % pr[j]);
    const u64 ql = pr[l - 1];
    pp->tinv_last[l] = wpair(invmod_h(t % ql, ql), ql);
  }
  void* d = nullptr;
  if (!all.empty()) {
    if (cudaMalloc(&d, all.size() * 8) != cudaSuccess) return nullptr;
    if (cudaMemcpy(d, all.data(), all.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
      cudaFree(d);
      return nullptr;
    }
  }
  pp->dmem[0] = d;
  size_t off = 0;
  for (int l = 2; l <= ctx->L; ++l) {
    pp->t_mod[l] = (const u64*)d + off;
    off += l - 1;
  }
  PlainPlan* raw = pp.get();
  ctx->plain[t] = std::move(pp);
  return raw;
}

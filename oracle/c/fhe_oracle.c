/*
 * fhe_oracle.c - C restatement of the reference's CPU hot path.
 * TEST INFRASTRUCTURE ONLY: the parity checker for full-size GPU results
 * and the CPU baseline timed by bench.py (`cpu_baseline`, `--impl
 * reference`).  The product never links or calls this code.
 *
 * Algorithms follow the reference (paths under /root/reference/pkg/src/rnsfhe):
 *   ntt      coremath/_kernels.py:19-99  (CT forward with Shoup twiddles,
 *            GS inverse then an n^-1 pass; psi = smallest primitive 2N-th
 *            root, primes.py:60-71; bit-reversed tables, ntt.py:66-98)
 *   tensor   schemes/ckks.py:308-349
 *   keyswitch keys.py:186-237 (per-prime gadget: INTT, coeff_i mod q_j,
 *            NTT of the level^2 rows, MAC), generalised to digits of alpha
 *            primes plus special primes P (ModUp fast base conversion in the
 *            style of behz.py:131-153, ModDown (x - BConv_P(x_P)) * P^-1);
 *            alpha = 1, K = 0 is the reference algorithm itself
 *   rescale  schemes/ckks.py:382-410
 * Rows are processed in parallel on all host threads (pthreads), as numba
 * prange does in the reference (_kernels.py:88-99).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

/* ---- minimal pthread parallel-for (no OpenMP runtime in this image) ---- */
#include <pthread.h>
#include <unistd.h>

typedef void (*body_fn)(long i, void* ctx);
typedef struct {
  body_fn fn;
  void* ctx;
  long lo, hi;
} Span;

static void* run_span(void* p) {
  Span* s = (Span*)p;
  for (long i = s->lo; i < s->hi; ++i) s->fn(i, s->ctx);
  return NULL;
}

int orc_threads(void) {
  const char* e = getenv("ORACLE_THREADS");
  long n = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  return n < 1 ? 1 : (n > 256 ? 256 : (int)n);
}

static void parallel_for(long count, body_fn fn, void* ctx) {
  int nt = orc_threads();
  if (nt > count) nt = (int)count;
  if (nt <= 1) {
    for (long i = 0; i < count; ++i) fn(i, ctx);
    return;
  }
  pthread_t th[256];
  Span sp[256];
  for (int t = 0; t < nt; ++t) {
    sp[t].fn = fn;
    sp[t].ctx = ctx;
    sp[t].lo = count * t / nt;
    sp[t].hi = count * (t + 1) / nt;
    pthread_create(&th[t], NULL, run_span, &sp[t]);
  }
  for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

static pthread_mutex_t g_tab_mu = PTHREAD_MUTEX_INITIALIZER;

static u64 mulmod(u64 a, u64 b, u64 q) { return (u64)((u128)a * b % q); }
static u64 powmod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = mulmod(r, a, q);
    a = mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }
static u64 shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
static u64 shoup_mul(u64 x, u64 w, u64 wsh, u64 q) {
  u64 hi = (u64)(((u128)x * wsh) >> 64);
  u64 r = x * w - hi * q;
  return r >= q ? r - q : r;
}

/* ---- tables (cached per (q, log_n)) ------------------------------------- */
typedef struct {
  u64 q;
  int log_n;
  u64 *psi, *psi_sh, *ipsi, *ipsi_sh;
  u64 ninv, ninv_sh;
} Tab;

static Tab g_tabs[256];
static int g_ntabs = 0;

static u64 min_root(u64 q, u64 order) {
  u64 cof = (q - 1) / order, r = 0;
  for (u64 g = 2;; ++g) {
    r = powmod(g, cof, q);
    if (powmod(r, order / 2, q) == q - 1) break;
  }
  u64 best = r, cur = r, sq = mulmod(r, r, q);
  for (u64 k = 0; k + 1 < order / 2; ++k) {
    cur = mulmod(cur, sq, q);
    if (cur < best) best = cur;
  }
  return best;
}

static unsigned brev(unsigned x, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; ++i) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}

static const Tab* get_tab(u64 q, int log_n) {
  const Tab* found = NULL;
  pthread_mutex_lock(&g_tab_mu);
  {
    for (int i = 0; i < g_ntabs; ++i)
      if (g_tabs[i].q == q && g_tabs[i].log_n == log_n) found = &g_tabs[i];
    if (!found && g_ntabs < 256) {
      size_t n = (size_t)1 << log_n;
      Tab* t = &g_tabs[g_ntabs];
      t->q = q;
      t->log_n = log_n;
      t->psi = malloc(n * 8);
      t->psi_sh = malloc(n * 8);
      t->ipsi = malloc(n * 8);
      t->ipsi_sh = malloc(n * 8);
      u64 psi = min_root(q, 2 * n), ipsi = invmod(psi, q);
      u64* fw = malloc(n * 8);
      u64* iv = malloc(n * 8);
      u64 a = 1, ia = 1;
      for (size_t i = 0; i < n; ++i) {
        fw[i] = a;
        iv[i] = ia;
        a = mulmod(a, psi, q);
        ia = mulmod(ia, ipsi, q);
      }
      for (size_t i = 0; i < n; ++i) {
        unsigned b = brev((unsigned)i, log_n);
        t->psi[i] = fw[b];
        t->ipsi[i] = iv[b];
        t->psi_sh[i] = shoup(fw[b], q);
        t->ipsi_sh[i] = shoup(iv[b], q);
      }
      free(fw);
      free(iv);
      t->ninv = invmod(n % q, q);
      t->ninv_sh = shoup(t->ninv, q);
      g_ntabs++;
      found = t;
    }
  }
  pthread_mutex_unlock(&g_tab_mu);
  return found;
}

static void ntt_row(u64* a, const Tab* t) {
  const size_t n = (size_t)1 << t->log_n;
  const u64 q = t->q;
  size_t tt = n;
  for (size_t m = 1; m < n; m <<= 1) {
    tt >>= 1;
    for (size_t i = 0; i < m; ++i) {
      const u64 w = t->psi[m + i], wsh = t->psi_sh[m + i];
      const size_t j1 = 2 * i * tt;
      for (size_t j = j1; j < j1 + tt; ++j) {
        u64 v = shoup_mul(a[j + tt], w, wsh, q), u = a[j];
        u64 hi = u + v, lo = u + q - v;
        a[j] = hi >= q ? hi - q : hi;
        a[j + tt] = lo >= q ? lo - q : lo;
      }
    }
  }
}

static void intt_row(u64* a, const Tab* t) {
  const size_t n = (size_t)1 << t->log_n;
  const u64 q = t->q;
  size_t tt = 1;
  for (size_t m = n; m > 1; m >>= 1) {
    size_t h = m >> 1;
    for (size_t i = 0; i < h; ++i) {
      const u64 w = t->ipsi[h + i], wsh = t->ipsi_sh[h + i];
      const size_t j1 = 2 * i * tt;
      for (size_t j = j1; j < j1 + tt; ++j) {
        u64 u = a[j], v = a[j + tt];
        u64 s = u + v, d = u + q - v;
        a[j] = s >= q ? s - q : s;
        a[j + tt] = shoup_mul(d >= q ? d - q : d, w, wsh, q);
      }
    }
    tt <<= 1;
  }
  for (size_t j = 0; j < n; ++j) a[j] = shoup_mul(a[j], t->ninv, t->ninv_sh, q);
}

/* in place; row r uses primes[mod_idx[r]] (mod_idx NULL: r % nprimes) */
typedef struct {
  u64* data;
  size_t n;
  int log_n;
  const u64* primes;
  int nprimes;
  const int32_t* mod_idx;
  int inverse;
} NttJob;

static void ntt_body(long r, void* p) {
  NttJob* j = (NttJob*)p;
  int mi = j->mod_idx ? j->mod_idx[r] : (int)(r % j->nprimes);
  const Tab* t = get_tab(j->primes[mi], j->log_n);
  if (j->inverse)
    intt_row(j->data + r * j->n, t);
  else
    ntt_row(j->data + r * j->n, t);
}

void orc_ntt(u64* data, long rows, int log_n, const u64* primes, int nprimes,
             const int32_t* mod_idx, int inverse) {
  for (int p = 0; p < nprimes; ++p) get_tab(primes[p], log_n);
  NttJob j = {data, (size_t)1 << log_n, log_n, primes, nprimes, mod_idx, inverse};
  parallel_for(rows, ntt_body, &j);
}

/* x, y: (2, level, n); out: (3, level, n) */
typedef struct {
  u64* out;
  const u64 *x, *y, *primes;
  size_t n, poly;
} TensorJob;

static void tensor_body(long j, void* p) {
  TensorJob* t = (TensorJob*)p;
  const u64 q = t->primes[j];
  const size_t n = t->n, poly = t->poly;
  for (size_t i = 0; i < n; ++i) {
    size_t o = j * n + i;
    t->out[o] = mulmod(t->x[o], t->y[o], q);
    t->out[poly + o] =
        (u64)(((u128)t->x[o] * t->y[poly + o] + (u128)t->x[poly + o] * t->y[o]) % q);
    t->out[2 * poly + o] = mulmod(t->x[poly + o], t->y[poly + o], q);
  }
}

void orc_tensor(u64* out, const u64* x, const u64* y, int level, int log_n, const u64* primes) {
  TensorJob t = {out, x, y, primes, (size_t)1 << log_n, (size_t)level << log_n};
  parallel_for(level, tensor_body, &t);
}

/* element-wise a + b mod q over (polys, level, n) */
typedef struct {
  u64* out;
  const u64 *a, *b, *primes;
  size_t n;
  int level;
} AddJob;

static void add_body(long r, void* p) {
  AddJob* j = (AddJob*)p;
  const u64 q = j->primes[r % j->level];
  for (size_t i = 0; i < j->n; ++i) {
    u64 s = j->a[r * j->n + i] + j->b[r * j->n + i];
    j->out[r * j->n + i] = s >= q ? s - q : s;
  }
}

void orc_add(u64* out, const u64* a, const u64* b, int polys, int level, int log_n,
             const u64* primes) {
  AddJob j = {out, a, b, primes, (size_t)1 << log_n, level};
  parallel_for((long)polys * level, add_body, &j);
}

/* product of chain[lo..hi) except `skip`, mod m */
static u64 punct(const u64* chain, int lo, int hi, int skip, u64 m) {
  u64 r = 1 % m;
  for (int i = lo; i < hi; ++i)
    if (i != skip) r = mulmod(chain[i] % m, r, m);
  return r;
}

/* ---- key switch ----------------------------------------------------------- */
typedef struct {
  const u64* d;
  const u64* keys;
  const u64* chain;
  const int32_t* tidx;
  const u64* coeff;
  u64* ext;
  u128* acc;
  size_t n;
  int log_n, level, L, K, T, s0, s1, di;
} KsJob;

/* ModUp of target limb m for digit di: fast base conversion, then NTT */
static void modup_body(long m, void* p) {
  KsJob* j = (KsJob*)p;
  const size_t n = j->n;
  u64* row = j->ext + (size_t)m * n;
  if (m >= j->s0 && m < j->s1) {
    memcpy(row, j->d + (size_t)m * n, n * 8);
    return;
  }
  const u64 pm = j->chain[j->tidx[m]];
  u64 w[64], inv[64];
  for (int s = j->s0; s < j->s1; ++s) {
    inv[s - j->s0] = invmod(punct(j->chain, j->s0, j->s1, s, j->chain[s]), j->chain[s]);
    w[s - j->s0] = punct(j->chain, j->s0, j->s1, s, pm);
  }
  for (size_t i = 0; i < n; ++i) {
    u128 sum = 0;
    for (int s = j->s0; s < j->s1; ++s) {
      u64 y = mulmod(j->coeff[(size_t)s * n + i], inv[s - j->s0], j->chain[s]);
      sum += (u128)y * w[s - j->s0] % pm;
    }
    row[i] = (u64)(sum % pm);
  }
  ntt_row(row, get_tab(pm, j->log_n));
}

static void mac_body(long m, void* p) {
  KsJob* j = (KsJob*)p;
  const size_t n = j->n;
  const int LK = j->L + j->K;
  const u64 pm = j->chain[j->tidx[m]];
  const u64* kb = j->keys + (((size_t)j->di * 2 + 0) * LK + j->tidx[m]) * n;
  const u64* ka = j->keys + (((size_t)j->di * 2 + 1) * LK + j->tidx[m]) * n;
  const u64* e = j->ext + (size_t)m * n;
  u128* ab = j->acc + (size_t)m * n;
  u128* aa = j->acc + ((size_t)j->T + m) * n;
  for (size_t i = 0; i < n; ++i) {
    ab[i] = (ab[i] + (u128)e[i] * kb[i]) % pm;
    aa[i] = (aa[i] + (u128)e[i] * ka[i]) % pm;
  }
}

typedef struct {
  const u64* chain;
  const u64* cp;
  const u128* ac;
  u64* conv;
  u64* out;
  size_t n;
  int L, K;
} DownJob;

static void down_conv_body(long jj, void* p) {
  DownJob* j = (DownJob*)p;
  const size_t n = j->n;
  const int L = j->L, K = j->K;
  const u64 q = j->chain[jj];
  u64 w[64], inv[64];
  for (int k = 0; k < K; ++k) {
    inv[k] = invmod(punct(j->chain, L, L + K, L + k, j->chain[L + k]), j->chain[L + k]);
    w[k] = punct(j->chain, L, L + K, L + k, q);
  }
  for (size_t i = 0; i < n; ++i) {
    u128 sum = 0;
    for (int k = 0; k < K; ++k)
      sum += (u128)mulmod(j->cp[(size_t)k * n + i], inv[k], j->chain[L + k]) * w[k] % q;
    j->conv[(size_t)jj * n + i] = (u64)(sum % q);
  }
}

static void down_finish_body(long jj, void* p) {
  DownJob* j = (DownJob*)p;
  const size_t n = j->n;
  const u64 q = j->chain[jj];
  const u64 pinv = invmod(punct(j->chain, j->L, j->L + j->K, -1, q), q);
  for (size_t i = 0; i < n; ++i) {
    u64 x = (u64)j->ac[(size_t)jj * n + i], c = j->conv[(size_t)jj * n + i];
    j->out[(size_t)jj * n + i] = mulmod(x >= c ? x - c : x + q - c, pinv, q);
  }
}

/*
 * d: (level, n) eval over Q[0..level).  keys: (D, 2, L+K, n) over chain Q|P.
 * outputs b, a: (level, n).
 */
int orc_keyswitch(const u64* d, int level, int log_n, const u64* keys, const u64* Q, int L,
                  const u64* P, int K, int alpha, u64* out_b, u64* out_a) {
  const size_t n = (size_t)1 << log_n;
  const int D = (level + alpha - 1) / alpha;
  const int T = level + K;
  if (alpha > 64 || K > 64) return -1;
  u64* chain = malloc((size_t)(L + K) * 8);
  memcpy(chain, Q, (size_t)L * 8);
  if (K) memcpy(chain + L, P, (size_t)K * 8);
  for (int i = 0; i < L + K; ++i) get_tab(chain[i], log_n);
  u64* coeff = malloc((size_t)level * n * 8);
  memcpy(coeff, d, (size_t)level * n * 8);
  orc_ntt(coeff, level, log_n, chain, level, NULL, 1);
  u128* acc = calloc((size_t)2 * T * n, sizeof(u128));
  u64* ext = malloc((size_t)T * n * 8);
  int32_t* tidx = malloc((size_t)T * 4);
  for (int m = 0; m < T; ++m) tidx[m] = m < level ? m : L + (m - level);
  KsJob job = {d, keys, chain, tidx, coeff, ext, acc, n, log_n, level, L, K, T, 0, 0, 0};
  for (int di = 0; di < D; ++di) {
    job.di = di;
    job.s0 = di * alpha;
    job.s1 = job.s0 + alpha < level ? job.s0 + alpha : level;
    parallel_for(T, modup_body, &job);
    parallel_for(T, mac_body, &job);
  }
  for (int poly = 0; poly < 2; ++poly) {
    u64* out = poly ? out_a : out_b;
    const u128* ac = acc + (size_t)poly * T * n;
    if (K == 0) {
      for (size_t i = 0; i < (size_t)level * n; ++i) out[i] = (u64)ac[i];
      continue;
    }
    u64* cp = malloc((size_t)K * n * 8);
    for (size_t i = 0; i < (size_t)K * n; ++i) cp[i] = (u64)ac[(size_t)level * n + i];
    int32_t* pidx = malloc((size_t)K * 4);
    for (int k = 0; k < K; ++k) pidx[k] = L + k;
    orc_ntt(cp, K, log_n, chain, L + K, pidx, 1);
    u64* conv = malloc((size_t)level * n * 8);
    DownJob dj = {chain, cp, ac, conv, out, n, L, K};
    parallel_for(level, down_conv_body, &dj);
    orc_ntt(conv, level, log_n, chain, level, NULL, 0);
    parallel_for(level, down_finish_body, &dj);
    free(cp);
    free(pidx);
    free(conv);
  }
  free(chain);
  free(coeff);
  free(acc);
  free(ext);
  free(tidx);
  return 0;
}

/* ckks_rescale: in (polys, level, n) eval -> out (polys, level-1, n) eval */
typedef struct {
  const u64* coeff;
  u64* o;
  const u64* primes;
  size_t n;
  int level;
} RsJob;

static void rescale_body(long jj, void* p) {
  RsJob* j = (RsJob*)p;
  const size_t n = j->n;
  const u64 ql = j->primes[j->level - 1];
  const u64* last = j->coeff + (size_t)(j->level - 1) * n;
  const u64 q = j->primes[jj], inv = invmod(ql % q, q), qlm = ql % q;
  for (size_t i = 0; i < n; ++i) {
    u64 r = last[i] % q;
    if (last[i] > ql / 2) r = r >= qlm ? r - qlm : r + q - qlm;
    u64 c = j->coeff[(size_t)jj * n + i];
    j->o[(size_t)jj * n + i] = mulmod(c >= r ? c - r : c + q - r, inv, q);
  }
}

void orc_rescale(u64* out, const u64* in, int polys, int level, int log_n, const u64* primes) {
  const size_t n = (size_t)1 << log_n;
  u64* coeff = malloc((size_t)level * n * 8);
  for (int p = 0; p < polys; ++p) {
    memcpy(coeff, in + (size_t)p * level * n, (size_t)level * n * 8);
    orc_ntt(coeff, level, log_n, primes, level, NULL, 1);
    u64* o = out + (size_t)p * (level - 1) * n;
    RsJob j = {coeff, o, primes, n, level};
    parallel_for(level - 1, rescale_body, &j);
    orc_ntt(o, level - 1, log_n, primes, level - 1, NULL, 0);
  }
  free(coeff);
}

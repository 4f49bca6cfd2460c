// extern "C" boundary (include/fhe_sm100.h).  Argument checking that needs
// no device access happens here; everything else is forwarded to the
// launchers, which enqueue asynchronously on the caller's stream.
#include <atomic>
#include <exception>

#include "fhe_context.cuh"

static thread_local std::string g_err;
static std::atomic<unsigned long long> g_launches{0};

void fhe_set_error(const std::string& msg) { g_err = msg; }
void fhe_count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

#define FHE_TRY(body)                   \
  try {                                 \
    body                                \
  } catch (const std::exception& e) {   \
    fhe_set_error(e.what());            \
    return -9;                          \
  }

extern "C" {

const char* fhe_last_error(void) { return g_err.c_str(); }

uint64_t fhe_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

uint64_t fhe_ntt_path_count(int path) { return ntt_path_count(path); }

int fhe_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}

int fhe_chain_create(const uint64_t* primes, int count, int log_n, FheChain** out) {
  FHE_TRY({
    if (!out || !primes || count < 1 || log_n < 1 || log_n > 17) {
      fhe_set_error("fhe_chain_create: bad arguments (need count >= 1, 1 <= log_n <= 17)");
      return -1;
    }
    FheChain* ch = new FheChain();
    int rc = build_chain(primes, count, log_n, ch);
    if (rc) {
      free_chain(ch);
      delete ch;
      return rc;
    }
    *out = ch;
    return 0;
  })
}

int fhe_chain_destroy(FheChain* ch) {
  if (!ch) return 0;
  free_chain(ch);
  delete ch;
  return 0;
}

int fhe_chain_tables(const FheChain* ch, int idx, uint64_t* psi, uint64_t* psi_br,
                     uint64_t* ipsi_br, uint64_t* n_inv) {
  if (!ch || idx < 0 || idx >= (int)ch->primes.size()) {
    fhe_set_error("fhe_chain_tables: bad index");
    return -1;
  }
  const size_t n = (size_t)1 << ch->log_n;
  if (psi) *psi = ch->psi[idx];
  std::vector<WPair> tmp(n);
  if (psi_br) {
    FHE_CUDA_CHECK(cudaMemcpy(tmp.data(), ch->dev.tw + idx * n, n * sizeof(WPair),
                              cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) psi_br[i] = tmp[i].w;
  }
  if (ipsi_br) {
    FHE_CUDA_CHECK(cudaMemcpy(tmp.data(), ch->dev.itw + idx * n, n * sizeof(WPair),
                              cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < n; ++i) ipsi_br[i] = tmp[i].w;
  }
  if (n_inv) {
    WPair w;
    FHE_CUDA_CHECK(cudaMemcpy(&w, ch->dev.ninv + idx, sizeof(WPair), cudaMemcpyDeviceToHost));
    *n_inv = w.w;
  }
  return 0;
}

static int check_map(const FheChain* ch, int64_t rows, const int32_t* mod_idx, int limbs,
                     int offset) {
  if (!ch) {
    fhe_set_error("null chain");
    return -1;
  }
  if (rows < 0 || rows > (int64_t)0x7fffffff) {
    fhe_set_error("row count out of range");
    return -1;
  }
  if (limbs < 1 || offset < 0 || (!mod_idx && offset + limbs > ch->dev.count)) {
    fhe_set_error("limbs/offset exceed the chain length");
    return -1;
  }
  return 0;
}

int fhe_ntt_fwd(const FheChain* ch, uint64_t* data, int64_t rows, const int32_t* mod_idx,
                int limbs, int offset, void* stream) {
  int rc = check_map(ch, rows, mod_idx, limbs, offset);
  if (rc) return rc;
  return launch_ntt(ch->dev, data, data, (int)rows, RowMap{mod_idx, limbs, offset}, false,
                    (cudaStream_t)stream);
}

int fhe_ntt_inv(const FheChain* ch, uint64_t* data, int64_t rows, const int32_t* mod_idx,
                int limbs, int offset, void* stream) {
  int rc = check_map(ch, rows, mod_idx, limbs, offset);
  if (rc) return rc;
  return launch_ntt(ch->dev, data, data, (int)rows, RowMap{mod_idx, limbs, offset}, true,
                    (cudaStream_t)stream);
}

int fhe_ntt_mm(const FheChain* ch, uint64_t* out, const uint64_t* in, int64_t rows,
               const int32_t* mod_idx, int limbs, int offset, int inverse, void* stream) {
  int rc = check_map(ch, rows, mod_idx, limbs, offset);
  if (rc) return rc;
  if (out == in && rows > 0) {
    fhe_set_error("fhe_ntt_mm: out must not alias in");
    return -1;
  }
  return launch_ntt_mm(ch->dev, out, in, (int)rows, RowMap{mod_idx, limbs, offset}, inverse != 0,
                       (cudaStream_t)stream);
}

int fhe_ewise(const FheChain* ch, int op, uint64_t* out, const uint64_t* a, const uint64_t* b,
              const uint64_t* c, int64_t rows, const int32_t* mod_idx, int limbs, int offset,
              int b_mode, void* stream) {
  int rc = check_map(ch, rows, mod_idx, limbs, offset);
  if (rc) return rc;
  if (op < FHE_EW_ADD || op > FHE_EW_REDUCE) {
    fhe_set_error("unknown element-wise op");
    return -1;
  }
  const bool needs_b = !(op == FHE_EW_NEG || op == FHE_EW_REDUCE);
  const bool needs_c = (op == FHE_EW_MUL_ADD || op == FHE_EW_MUL_SUB);
  if (!out || !a || (needs_b && !b) || (needs_c && !c)) {
    fhe_set_error("missing operand for element-wise op");
    return -1;
  }
  if (b_mode == FHE_B_BCAST && mod_idx) {
    fhe_set_error("broadcast operand requires the layout-order row map");
    return -1;
  }
  if (ch->log_n < 1) {
    fhe_set_error("element-wise ops need n >= 2");
    return -1;
  }
  return launch_ewise(ch->dev, op, out, a, b, c, rows, RowMap{mod_idx, limbs, offset}, b_mode,
                      (cudaStream_t)stream);
}

int fhe_tensor(const FheChain* ch, uint64_t* out, const uint64_t* x, const uint64_t* y, int limbs,
               int64_t batch, int64_t x_stride, int64_t y_stride, int64_t out_stride, int square,
               void* stream) {
  if (!ch || limbs < 1 || limbs > ch->dev.count || !out || !x || (!square && !y)) {
    fhe_set_error("fhe_tensor: bad arguments");
    return -1;
  }
  return launch_tensor(ch->dev, out, x, y, limbs, batch, x_stride, y_stride, out_stride, square,
                       (cudaStream_t)stream);
}

int fhe_automorph(uint64_t* out, const uint64_t* in, int64_t rows, int log_n, uint64_t elt,
                  void* stream) {
  if (!out || !in || out == in || log_n < 1 || log_n > 17 || !(elt & 1)) {
    fhe_set_error("fhe_automorph: bad arguments (out != in, odd elt)");
    return -1;
  }
  return launch_automorph(out, in, rows, log_n, elt, (cudaStream_t)stream);
}

int fhe_context_create(const uint64_t* q_primes, int L, const uint64_t* p_primes, int K,
                       int alpha, int log_n, FheContext** out) {
  FHE_TRY({
    if (!out || !q_primes || L < 1 || K < 0 || (K > 0 && !p_primes) || alpha < 1 ||
        log_n < 1 || log_n > 17) {
      fhe_set_error("fhe_context_create: bad arguments");
      return -1;
    }
    if (alpha > 16 || K > 16) {
      fhe_set_error("fhe_context_create: alpha and K must be <= 16");
      return -1;
    }
    std::vector<u64> all(q_primes, q_primes + L);
    for (int k = 0; k < K; ++k) all.push_back(p_primes[k]);
    FheContext* ctx = new FheContext();
    ctx->L = L;
    ctx->K = K;
    ctx->alpha = alpha;
    ctx->chain = new FheChain();
    int rc = build_chain(all.data(), (int)all.size(), log_n, ctx->chain);
    if (!rc) rc = build_levels(ctx);
    if (rc) {
      fhe_context_destroy(ctx);
      return rc;
    }
    *out = ctx;
    return 0;
  })
}

size_t fhe_philox_workspace(int64_t count, uint64_t rng) {
  return count > 0 ? philox_workspace((long)count, rng) : 0;
}

int fhe_philox_integers(FhePhilox* dev_state, int64_t low, uint64_t rng, int64_t count,
                        uint64_t* out, void* workspace, size_t ws_bytes, void* stream) {
  FHE_TRY({
    if (!dev_state || (count > 0 && (!out || !workspace))) {
      fhe_set_error("fhe_philox_integers: null argument");
      return -1;
    }
    return run_philox_integers(dev_state, (long long)low, rng, (long)count, out, workspace,
                               ws_bytes, (cudaStream_t)stream);
  })
}

int fhe_cbd_combine(int64_t* out, const uint64_t* flips, int pairs, int64_t n, void* stream) {
  FHE_TRY({
    if (!out || !flips || pairs < 1) {
      fhe_set_error("fhe_cbd_combine: bad arguments");
      return -1;
    }
    return run_cbd_combine((long long*)out, flips, pairs, (long)n, (cudaStream_t)stream);
  })
}

int fhe_signed_lift(const FheChain* ch, uint64_t* out, const int64_t* coeffs, int64_t n, int limbs,
                    int offset, void* stream) {
  FHE_TRY({
    if (!ch || !out || !coeffs || limbs < 1 || offset < 0 ||
        offset + limbs > (int)ch->primes.size()) {
      fhe_set_error("fhe_signed_lift: bad arguments");
      return -1;
    }
    return run_signed_lift(ch->dev, out, (const long long*)coeffs, (long)n, limbs, offset,
                           (cudaStream_t)stream);
  })
}

size_t fhe_crc32_workspace(int64_t nbytes) { return crc32_workspace((long)nbytes); }

int fhe_crc32(const void* data, int64_t nbytes, uint32_t* out, void* workspace, size_t ws_bytes,
              void* stream) {
  FHE_TRY({
    if (!out || (nbytes > 0 && (!data || !workspace))) {
      fhe_set_error("fhe_crc32: null argument");
      return -1;
    }
    return run_crc32(data, (long)nbytes, out, workspace, ws_bytes, (cudaStream_t)stream);
  })
}

int fhe_real_lift(const FheChain* ch, uint64_t* out, const double* values, int64_t n, int limbs,
                  int offset, void* stream) {
  FHE_TRY({
    if (!ch || !out || !values || limbs < 1 || offset < 0 ||
        offset + limbs > (int)ch->primes.size()) {
      fhe_set_error("fhe_real_lift: bad arguments");
      return -1;
    }
    return run_real_lift(ch->dev, out, values, (long)n, limbs, offset, (cudaStream_t)stream);
  })
}

int fhe_crt_lift(const FheContext* ctx, int mode, void* out, const uint64_t* rows, int level,
                 double scale, uint64_t t, uint64_t inv_f, void* stream) {
  FHE_TRY({
    if (!ctx || !out || !rows) {
      fhe_set_error("fhe_crt_lift: null argument");
      return -1;
    }
    return run_crt_lift(*ctx, mode, out, rows, level, scale, t, inv_f, (cudaStream_t)stream);
  })
}

int fhe_context_prepare_plain(FheContext* ctx, uint64_t t) {
  FHE_TRY({
    if (!ctx || t < 2) {
      fhe_set_error("fhe_context_prepare_plain: bad arguments");
      return -1;
    }
    if (!get_plain_plan(ctx, t)) {
      fhe_set_error("fhe_context_prepare_plain: device allocation failed");
      return -2;
    }
    return 0;
  })
}

int fhe_context_destroy(FheContext* ctx) {
  if (!ctx) return 0;
  for (auto& lp : ctx->levels)
    if (lp.dmem) cudaFree(lp.dmem);
  for (auto& kv : ctx->plain)
    for (void* p : kv.second->dmem)
      if (p) cudaFree(p);
  if (ctx->chain) {
    free_chain(ctx->chain);
    delete ctx->chain;
  }
  delete ctx;
  return 0;
}

const FheChain* fhe_context_chain(const FheContext* ctx) { return ctx ? ctx->chain : nullptr; }

size_t fhe_rescale_workspace(const FheContext* ctx, int polys, int level) {
  return ctx ? rescale_workspace(*ctx, polys, level) : 0;
}

int fhe_rescale(const FheContext* ctx, uint64_t* out, const uint64_t* in, int polys, int level,
                uint64_t t_plain, void* workspace, size_t ws_bytes, void* stream) {
  if (!ctx || !out || !in || out == in || polys < 1) {
    fhe_set_error("fhe_rescale: bad arguments");
    return -1;
  }
  FHE_TRY({
    return run_rescale(*const_cast<FheContext*>(ctx), out, in, polys, level, t_plain, workspace,
                       ws_bytes, (cudaStream_t)stream);
  })
}

size_t fhe_keyswitch_workspace(const FheContext* ctx, int level, int batch) {
  if (!ctx || level < 1 || level > ctx->L || batch < 1) return 0;
  return keyswitch_workspace(*ctx, level, batch);
}

int fhe_keyswitch(const FheContext* ctx, int level, const uint64_t* d, int64_t d_stride,
                  const uint64_t* key, const uint64_t* add0, const uint64_t* add1,
                  int64_t add_stride, uint64_t* out0, uint64_t* out1, int64_t out_stride,
                  int batch, void* workspace, size_t ws_bytes, void* stream) {
  if (!ctx || !d || !key || !out0 || !out1 || batch < 1) {
    fhe_set_error("fhe_keyswitch: bad arguments");
    return -1;
  }
  FHE_TRY({
    return run_keyswitch(*ctx, level, d, d_stride, key, add0, add1, add_stride, out0, out1,
                         out_stride, batch, workspace, ws_bytes, (cudaStream_t)stream);
  })
}

size_t fhe_hmult_relin_workspace(const FheContext* ctx, int level, int batch) {
  if (!ctx || level < 1 || level > ctx->L || batch < 1) return 0;
  return hmult_relin_workspace(*ctx, level, batch);
}

int fhe_hmult_relin(const FheContext* ctx, int level, const uint64_t* x, const uint64_t* y,
                    int64_t in_stride, const uint64_t* key, uint64_t* out0, uint64_t* out1,
                    int64_t out_stride, int batch, void* workspace, size_t ws_bytes,
                    void* stream) {
  if (!ctx || !x || !y || !key || !out0 || !out1 || batch < 1) {
    fhe_set_error("fhe_hmult_relin: bad arguments");
    return -1;
  }
  FHE_TRY({
    return run_hmult_relin(*ctx, level, x, y, in_stride, key, out0, out1, out_stride, batch,
                           workspace, ws_bytes, (cudaStream_t)stream);
  })
}

}  // extern "C"

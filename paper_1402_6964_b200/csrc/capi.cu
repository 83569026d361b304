// extern "C" boundary (include/tsnmf_b200.h): argument validation, error mapping, dispatch.
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/tsnmf_b200.h"
#include "common.cuh"
#include "internal.h"

namespace tsnmf {

static thread_local std::string g_last_error;

int set_error(int status, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return status;
}

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// CUDA-event pairs recorded around the dominant kernels on their launching stream.
struct Profiler {
  std::mutex mu;
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev[kProfSlots];
  cudaEvent_t open_begin[kProfSlots] = {};
};
static Profiler g_prof;

void prof_mark(int slot, bool begin, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  if (!g_prof.on) return;
  cudaEvent_t e;
  if (cudaEventCreate(&e) != cudaSuccess) return;
  cudaEventRecord(e, st);
  if (begin) {
    g_prof.open_begin[slot] = e;
  } else if (g_prof.open_begin[slot]) {
    g_prof.ev[slot].emplace_back(g_prof.open_begin[slot], e);
    g_prof.open_begin[slot] = nullptr;
  } else {
    cudaEventDestroy(e);
  }
}

}  // namespace tsnmf

using namespace tsnmf;

namespace {

cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int check_matrix(const char* who, const void* x, int64_t m, int32_t n, int64_t ld) {
  if (n < 1) return set_error(kUsage, "%s: need at least one column, got n = %d", who, n);
  if (m < 1) return set_error(kData, "%s: empty row block (m = %lld)", who, (long long)m);
  if (ld < n) return set_error(kUsage, "%s: row stride %lld < n = %d", who, (long long)ld, n);
  if (!x) return set_error(kUsage, "%s: null data pointer", who);
  return kOk;
}

}  // namespace

extern "C" {

int tsnmf_abi_version(void) { return 1; }

const char* tsnmf_last_error(void) { return g_last_error.c_str(); }

int tsnmf_max_cols(void) { return tsqr_max_cols(); }

size_t tsnmf_workspace_bytes(int op, int64_t m, int32_t n, int32_t k) {
  switch (op) {
    case TSNMF_OP_TSQR: return tsqr_workspace_bytes(m, n);
    case TSNMF_OP_COMBINE: return combine_workspace_bytes((int)m, n);
    case TSNMF_OP_GRAM: return gram_workspace_bytes(m, n);
    case TSNMF_OP_SKETCH: return sketch_workspace_bytes(m, n, k);
    case TSNMF_OP_STATS: return stats_workspace_bytes(m, n);
    case TSNMF_OP_NNLS: return nnls_workspace_bytes(n);
    default: return 0;
  }
}

uint64_t tsnmf_derive_stream(uint64_t seed, uint64_t tag) { return derive_stream(seed, tag); }

int tsnmf_uniform_block(uint64_t stream, uint64_t start, int64_t count, double* out, void* s) {
  if (count < 0) return set_error(kUsage, "uniform_block: negative count");
  if (count > 0 && !out) return set_error(kUsage, "uniform_block: null output");
  return uniform_block_run(stream, start, count, out, as_stream(s));
}

int tsnmf_normal_block(uint64_t stream, uint64_t start, int64_t count, double* out, void* s) {
  if (count < 0) return set_error(kUsage, "normal_block: negative count");
  if (count > 0 && !out) return set_error(kUsage, "normal_block: null output");
  return normal_block_run(stream, start, count, out, as_stream(s));
}

int tsnmf_gaussian_rows(uint64_t seed, int64_t row_offset, int64_t rows, int32_t k, double* out, void* s) {
  if (k < 1) return set_error(kUsage, "gaussian_rows: k must be >= 1, got %d", k);
  if (rows < 0) return set_error(kUsage, "gaussian_rows: negative row count");
  return normal_block_run(derive_stream(seed, kTagSketch), (uint64_t)row_offset * (uint64_t)k, rows * k, out,
                          as_stream(s));
}

int tsnmf_tsqr(const double* x, int64_t m, int32_t n, int64_t ldx, double* r, int64_t ldr, double* l1, double* sumsq,
               void* ws, size_t ws_bytes, void* s) {
  if (int rc = check_matrix("tsqr", x, m, n, ldx)) return rc;
  if (!r || ldr < n) return set_error(kUsage, "tsqr: bad output factor");
  if (n > tsqr_max_cols()) return set_error(kUsage, "tsqr: n = %d exceeds the supported %d", n, tsqr_max_cols());
  if (m == 1) {  // reference tsqr.py:135-139
    if (int rc = single_row_factor_run(x, n, r, ldr, as_stream(s))) return rc;
    if (l1 || sumsq) return stats_run(x, m, n, ldx, l1, sumsq, ws, ws_bytes, as_stream(s));
    return kOk;
  }
  return tsqr_run(x, m, n, ldx, r, ldr, l1, sumsq, ws, ws_bytes, as_stream(s));
}

int tsnmf_r_combine(const double* rs, int32_t count, int32_t n, double* r, int64_t ldr, void* ws, size_t ws_bytes,
                    void* s) {
  if (count < 1) return set_error(kData, "combine: no factors");
  if (n < 1 || n > tsqr_max_cols()) return set_error(kUsage, "combine: bad dimension n = %d", n);
  if (!rs || !r || ldr < n) return set_error(kUsage, "combine: null pointer or bad stride");
  return r_combine_run(rs, count, n, r, ldr, ws, ws_bytes, as_stream(s));
}

int tsnmf_gram(const double* x, int64_t m, int32_t n, int64_t ldx, double* g, int64_t ldg, double* l1, double* sumsq,
               void* ws, size_t ws_bytes, void* s) {
  if (int rc = check_matrix("gram", x, m, n, ldx)) return rc;
  if (!g || ldg < n) return set_error(kUsage, "gram: bad output");
  return gram_run(x, m, n, ldx, g, ldg, l1, sumsq, ws, ws_bytes, as_stream(s));
}

int tsnmf_sketch(const double* x, int64_t m, int32_t n, int64_t ldx, int64_t row_offset, uint64_t seed, int32_t k,
                 const double* g, int64_t ldgm, double* out, int64_t lds, void* ws, size_t ws_bytes, void* s) {
  if (k < 1) return set_error(kUsage, "sketch rows must be >= 1, got %d", k);
  if (int rc = check_matrix("sketch", x, m, n, ldx)) return rc;
  if (row_offset < 0) return set_error(kUsage, "sketch: negative row offset");
  if (!out || lds < n) return set_error(kUsage, "sketch: bad output");
  if (g && ldgm < k) return set_error(kUsage, "sketch: explicit G stride %lld < k", (long long)ldgm);
  return sketch_run(x, m, n, ldx, row_offset, seed, k, g, ldgm, out, lds, ws, ws_bytes, as_stream(s));
}

int tsnmf_column_stats(const double* x, int64_t m, int32_t n, int64_t ldx, double* l1, double* sumsq, void* ws,
                       size_t ws_bytes, void* s) {
  if (int rc = check_matrix("column_stats", x, m, n, ldx)) return rc;
  return stats_run(x, m, n, ldx, l1, sumsq, ws, ws_bytes, as_stream(s));
}

int tsnmf_first_nonfinite(const double* x, int64_t count, int64_t* first, void* s) {
  if (count < 0) return set_error(kUsage, "first_nonfinite: negative count");
  if ((count > 0 && !x) || !first) return set_error(kUsage, "first_nonfinite: null pointer");
  if (reinterpret_cast<uintptr_t>(x) & 15) return set_error(kUsage, "first_nonfinite: x must be 16-byte aligned");
  return first_nonfinite_run(x, count, first, as_stream(s));
}

int tsnmf_generate(double* x, int64_t ldx, int64_t row0, int64_t rows, int32_t n, int32_t r, const double* mix,
                   int32_t w_kind, const double* bumps, int64_t m_total, double sigma, uint64_t seed, void* s) {
  if (r < 1 || r > n) return set_error(kUsage, "generate: need 1 <= r <= n, got r=%d, n=%d", r, n);
  if (w_kind < 0 || w_kind > 2) return set_error(kUsage, "generate: unknown w_kind %d", w_kind);
  if (w_kind == 2 && !bumps) return set_error(kUsage, "generate: bumps parameters required");
  if (!x || !mix || ldx < n) return set_error(kUsage, "generate: bad pointers or stride");
  if (sigma < 0) return set_error(kUsage, "generate: negative noise level");
  return generate_run(x, ldx, row0, rows, n, r, mix, w_kind, bumps, m_total, sigma, seed, as_stream(s));
}

int tsnmf_nnls(const double* a, int64_t n, int32_t t, int64_t lda, const double* b, int64_t ldb, int32_t ncols,
               double tol, int32_t max_iter, double* y, int64_t ldy, int32_t* status, void* ws, size_t ws_bytes,
               void* s) {
  if (int rc = check_matrix("nnls", a, n, t, lda)) return rc;
  if (ncols < 1) return set_error(kUsage, "nnls: need at least one target column");
  if (!b || ldb < ncols) return set_error(kUsage, "nnls: bad targets pointer / stride");
  if (!y || ldy < ncols || !status) return set_error(kUsage, "nnls: bad output pointers / stride");
  if (!(tol >= 0.0) || max_iter < 1) return set_error(kUsage, "nnls: need tol >= 0 and max_iter >= 1");
  return nnls_run(a, n, t, lda, b, ldb, ncols, tol, max_iter, y, ldy, status, ws, ws_bytes, as_stream(s));
}

int tsnmf_nnls_max_cols(void) { return nnls_max_design_cols(); }

int tsnmf_scale_columns(const double* a, int32_t rows, int32_t n, int64_t lda, const double* norms, double* out,
                        int64_t ldo, void* s) {
  if (int rc = check_matrix("scale_columns", a, rows, n, lda)) return rc;
  if (!norms || !out || ldo < n) return set_error(kUsage, "scale_columns: bad norms / output arguments");
  return scale_columns_run(a, rows, n, lda, norms, out, ldo, as_stream(s));
}

int tsnmf_gp_select(const double* sk, int32_t k, int32_t n, int64_t ldsk, int32_t r, int32_t* out, int32_t* count,
                    void* s) {
  if (int rc = check_matrix("gp_select", sk, k, n, ldsk)) return rc;
  if (r < 1 || r > n) return set_error(kUsage, "gp_select: rank must be in 1..%d, got %d", n, r);
  if (n > 200000) return set_error(kUsage, "gp_select: at most 200000 columns");
  if (!out || !count) return set_error(kUsage, "gp_select: null output");
  return gp_select_run(sk, k, n, ldsk, r, out, count, as_stream(s));
}

int tsnmf_xray_scores(const double* m, int32_t n, int64_t ldm, const double* resid, int64_t ldr,
                      const double* colnorm, double* score, void* s) {
  if (int rc = check_matrix("xray_scores", m, n, n, ldm)) return rc;
  if (!resid || ldr < n || !colnorm || !score) return set_error(kUsage, "xray_scores: bad pointers / stride");
  return xray_scores_run(m, n, ldm, resid, ldr, colnorm, score, as_stream(s));
}

int tsnmf_xray_residual(const double* m, int32_t n, int64_t ldm, const double* a, int32_t t, int64_t lda,
                        const double* coef, int64_t ldc, double* resid, int64_t ldr, void* s) {
  if (int rc = check_matrix("xray_residual", m, n, n, ldm)) return rc;
  if (t < 1 || !a || lda < t || !coef || ldc < n || !resid || ldr < n)
    return set_error(kUsage, "xray_residual: bad design / coefficient / output arguments");
  return xray_residual_run(m, n, ldm, a, t, lda, coef, ldc, resid, ldr, as_stream(s));
}

long long tsnmf_launch_count(void) { return g_launches.load(); }

int tsnmf_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = on != 0;
  return kOk;
}

int tsnmf_profile_read(int slot, double* total_ms, long long* launches) {
  if (slot < 0 || slot >= kProfSlots) return set_error(kUsage, "profile slot %d out of range", slot);
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs;
  {
    std::lock_guard<std::mutex> lk(g_prof.mu);
    evs.swap(g_prof.ev[slot]);
  }
  double tot = 0.0;
  for (auto& pr : evs) {
    float ms = 0.f;
    TSNMF_CUDA_CHECK(cudaEventSynchronize(pr.second));
    TSNMF_CUDA_CHECK(cudaEventElapsedTime(&ms, pr.first, pr.second));
    tot += ms;
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (total_ms) *total_ms = tot;
  if (launches) *launches = (long long)evs.size();
  return kOk;
}

int tsnmf_tsqr_plan(int32_t n, int64_t m, int32_t* panel, int32_t* block_rows, int32_t* ctas_per_sm,
                    int32_t* leaves) {
  int nb, br, cps, lv;
  if (int rc = tsqr_describe(n, m, &nb, &br, &cps, &lv)) return rc;
  if (panel) *panel = nb;
  if (block_rows) *block_rows = br;
  if (ctas_per_sm) *ctas_per_sm = cps;
  if (leaves) *leaves = lv;
  return kOk;
}

}  // extern "C"

/*
 * tsnmf_b200 — C ABI of the B200-native single-pass reduction (arxiv 1402.6964 hot path).
 *
 * Plain C: device pointers, sizes, an opaque CUDA stream handle (cudaStream_t passed as void*).
 * Every call is stream-ordered and asynchronous (no host synchronisation inside), allocates nothing
 * (scratch comes from a caller workspace sized by tsnmf_workspace_bytes), and returns a status code
 * that mirrors the reference's exception classes / CLI exit codes
 * (reference pkg/src/tsnmf/errors.py:16-31):
 *     0 ok | 1 usage (UsageError) | 2 data (DataError) | 3 numerical (NumericalError) | 4 CUDA failure
 * A human-readable message for the last failure on the calling thread is tsnmf_last_error().
 * Matrices are row-major float64; "ld" arguments are row strides in elements.
 *
 * Reference-side binding: see INTEGRATION.md (a ctypes stub the reference's backend switch
 * reference pkg/src/tsnmf/kernels.py:13-31 would select).
 */
#ifndef TSNMF_B200_H
#define TSNMF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TSNMF_OK = 0,
  TSNMF_EUSAGE = 1,
  TSNMF_EDATA = 2,
  TSNMF_ENUMERICAL = 3,
  TSNMF_ECUDA = 4
};

/* operation ids for tsnmf_workspace_bytes */
enum {
  TSNMF_OP_TSQR = 1,    /* m rows, n cols            */
  TSNMF_OP_COMBINE = 2, /* m = number of factors, n  */
  TSNMF_OP_GRAM = 3,    /* m rows, n cols            */
  TSNMF_OP_SKETCH = 4,  /* m rows, n cols, k         */
  TSNMF_OP_STATS = 5,   /* m rows, n cols            */
  TSNMF_OP_NNLS = 6     /* n = design columns t      */
};

/* ABI version (bumped on any signature change) and limits. */
int tsnmf_abi_version(void);
const char* tsnmf_last_error(void);
int tsnmf_max_cols(void);

/* Scratch bytes the op needs for the given problem size (0 = unsupported size). */
size_t tsnmf_workspace_bytes(int op, int64_t m, int32_t n, int32_t k);

/* ---- counter RNG: replaces reference pkg/src/tsnmf/_kernels.pyx:35-69 (uniform_block /
 *      normal_block) and rng.py:33-55 (derive_stream, gaussian_rows).  Host-callable pure function +
 *      device block generators writing `count` doubles to `out`. */
uint64_t tsnmf_derive_stream(uint64_t seed, uint64_t tag);
int tsnmf_uniform_block(uint64_t stream, uint64_t start, int64_t count, double* out, void* cuda_stream);
int tsnmf_normal_block(uint64_t stream, uint64_t start, int64_t count, double* out, void* cuda_stream);
/* rows x k matrix: entry (i, t) = normal #((row_offset + i) * k + t) of derive_stream(seed, 0) */
int tsnmf_gaussian_rows(uint64_t seed, int64_t row_offset, int64_t rows, int32_t k, double* out,
                        void* cuda_stream);

/* ---- TSQR factor of one row block: replaces reference pkg/src/tsnmf/tsqr.py:129-141 (factor_chunk)
 *      fused with tsqr.py:190-192 (_StatsAcc.from_block).
 *      r: n x n (stride ldr) upper triangular, nonnegative diagonal, zeros below.
 *      l1 / sumsq: n column sums of |x| and x^2 (either may be NULL).  m >= 1. */
int tsnmf_tsqr(const double* x, int64_t m, int32_t n, int64_t ldx, double* r, int64_t ldr, double* l1,
               double* sumsq, void* ws, size_t ws_bytes, void* cuda_stream);

/* ---- R of the vertical stack of `count` factors (count x n x n, contiguous), combined in the
 *      reference TreeReducer order: replaces tsqr.py:144-153 (combine) + tsqr.py:201-234. */
int tsnmf_r_combine(const double* rs, int32_t count, int32_t n, double* r, int64_t ldr, void* ws,
                    size_t ws_bytes, void* cuda_stream);

/* ---- Gram matrix X^T X (n x n, symmetric, stride ldg) + column l1 / sumsq.  NEW (no reference
 *      function; parity anchor reference SPEC.md:164). */
int tsnmf_gram(const double* x, int64_t m, int32_t n, int64_t ldx, double* g, int64_t ldg, double* l1,
               double* sumsq, void* ws, size_t ws_bytes, void* cuda_stream);

/* ---- Gaussian projection S = G^T X (k x n, stride lds), G regenerated in-kernel from (seed, global row
 *      row_offset + i): replaces reference pkg/src/tsnmf/sketch.py:62-73 (sketch_chunk).  If g != NULL,
 *      G (m x k, stride ldgm) is read from device memory instead (the reference's gaussian_rows_fn hook). */
int tsnmf_sketch(const double* x, int64_t m, int32_t n, int64_t ldx, int64_t row_offset, uint64_t seed,
                 int32_t k, const double* g, int64_t ldgm, double* s, int64_t lds, void* ws, size_t ws_bytes,
                 void* cuda_stream);

/* ---- column l1 / sum of squares alone (tsqr.py:190-192). */
int tsnmf_column_stats(const double* x, int64_t m, int32_t n, int64_t ldx, double* l1, double* sumsq,
                       void* ws, size_t ws_bytes, void* cuda_stream);

/* ---- ingest validation: replaces reference pkg/src/tsnmf/matio.py:81-87 (_check_finite) for device
 *      batches read by matio.ChunkReader.  *first (device int64) = linear index of the
 *      first Inf/NaN among x[0 .. count) (row-major), or -1 when all are finite.  x 16-byte aligned. */
int tsnmf_first_nonfinite(const double* x, int64_t count, int64_t* first, void* cuda_stream);

/* ---- synthetic BASELINE.json configs written straight into device memory: rows
 *      [row0, row0 + rows) of X = max(W [I H'] Pi + sigma N, 0).  mix = [I H'] Pi (r x n, device),
 *      w_kind 0 uniform / 1 lognormal / 2 bumps (bumps: r x 4 x 3 device params, else NULL). */
int tsnmf_generate(double* x, int64_t ldx, int64_t row0, int64_t rows, int32_t n, int32_t r,
                   const double* mix, int32_t w_kind, const double* bumps, int64_t m_total, double sigma,
                   uint64_t seed, void* cuda_stream);

/* ---- batched nonnegative least squares: replaces reference pkg/src/tsnmf/nnls.py:47-126 (nnls_solve /
 *      solve_columns).  For every column j of b (n x ncols, stride ldb): y_j = argmin ||a y - b_j|| with
 *      y >= 0; a is the n x t design (stride lda, 1 <= t <= tsnmf_nnls_max_cols()), y is t x ncols (stride
 *      ldy).  Lawson-Hanson with the reference's entering / leaving rules and gradient tolerance `tol`.
 *      status[j] (device int32 array of ncols): 0 ok, 3 numerical (inner loop failed or singular passive
 *      set), 5 iteration limit (y_j = last iterate, the reference's NnlsIterationError.best_y). */
int tsnmf_nnls(const double* a, int64_t n, int32_t t, int64_t lda, const double* b, int64_t ldb, int32_t ncols,
               double tol, int32_t max_iter, double* y, int64_t ldy, int32_t* status, void* ws, size_t ws_bytes,
               void* cuda_stream);
int tsnmf_nnls_max_cols(void);

/* ---- XRAY steps (reference pkg/src/tsnmf/select.py:131-140) on the n x n reduced matrix m (stride ldm):
 *      scores: score[j] = ||resid^T m(:, j)||_2 / colnorm[j]  (-inf where colnorm[j] <= 0);
 *      residual: resid = m - a coef, a = m(:, K) (n x t, stride lda), coef t x n (stride ldc). */
int tsnmf_xray_scores(const double* m, int32_t n, int64_t ldm, const double* resid, int64_t ldr,
                      const double* colnorm, double* score, void* cuda_stream);
int tsnmf_xray_residual(const double* m, int32_t n, int64_t ldm, const double* a, int32_t t, int64_t lda,
                        const double* coef, int64_t ldc, double* resid, int64_t ldr, void* cuda_stream);

/* ---- reduced-space steps, on the pass's small outputs without a host round trip:
 *      scale_columns: out = a D^-1, D = diag(norms) (rows x n): reference tsqr.py:163-177 (R D^-1, the
 *        caller rejects zero norms first, as apply_column_scaling does) and sketch.py:87-100 (G^T X D^-1);
 *      gp_select: per row of the k x n sketch its argmin then argmax column (lowest index on ties), appended
 *        if unseen, until r columns: reference select.py:159-178.  out[0..*count) is the selection order;
 *        *count < r is the reference's shortfall. */
int tsnmf_scale_columns(const double* a, int32_t rows, int32_t n, int64_t lda, const double* norms, double* out,
                        int64_t ldo, void* cuda_stream);
int tsnmf_gp_select(const double* sk, int32_t k, int32_t n, int64_t ldsk, int32_t r, int32_t* out, int32_t* count,
                    void* cuda_stream);

/* ---- introspection for benchmarks: chosen TSQR panel width / rows per block / CTAs per SM / leaves */
int tsnmf_tsqr_plan(int32_t n, int64_t m, int32_t* panel, int32_t* block_rows, int32_t* ctas_per_sm,
                    int32_t* leaves);

/* ---- measurement hooks (bench.py): number of kernels this library has launched, and CUDA-event timing
 *      (recorded on the launching stream) of the dominant kernels.  slot 0 = TSQR leaf kernel,
 *      1 = TSQR combine tree, 2 = Gram kernel, 3 = sketch kernel.  read() synchronises on the events,
 *      returns the summed milliseconds and the number of timed launches, and resets the slot. */
long long tsnmf_launch_count(void);
int tsnmf_profile_enable(int on);
int tsnmf_profile_read(int slot, double* total_ms, long long* launches);

#ifdef __cplusplus
}
#endif

#endif /* TSNMF_B200_H */

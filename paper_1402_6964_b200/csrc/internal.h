// Internal (C++) entry points behind the C ABI in capi.cu.  All pointers are device pointers.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

namespace tsnmf {

// cudaFuncSetAttribute (the >48 KB dynamic shared-memory opt-in) applies to the CURRENT device only, so a
// launcher remembers per device whether it has set its kernels' attributes (a process-wide flag
// left every GPU but the first without the opt-in).
class PerDeviceFlag {
 public:
  bool is_set() const { return (bits_.load(std::memory_order_acquire) >> dev()) & 1u; }
  void set() { bits_.fetch_or(1ull << dev(), std::memory_order_acq_rel); }

 private:
  static int dev() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 63;
  }
  std::atomic<unsigned long long> bits_{0};
};

int set_error(int status, const char* fmt, ...);

int tsqr_max_cols();
size_t tsqr_workspace_bytes(int64_t m, int n);
size_t combine_workspace_bytes(int count, int n);
int tsqr_run(const double* x, int64_t m, int n, int64_t ldx, double* r, int64_t ldr, double* l1, double* sumsq,
             void* ws, size_t ws_bytes, cudaStream_t st);
int r_combine_run(const double* rs, int count, int n, double* r, int64_t ldr, void* ws, size_t ws_bytes,
                  cudaStream_t st);
int tsqr_describe(int n, int64_t m, int* nb, int* brows, int* ctas_per_sm, int* nleaves);
// register-block leaf with DMMA trailing updates (tsqr_reg.cu)
bool tsqr_reg_supported(int n);
int tsqr_reg_block_rows(int n);
int tsqr_reg_warps_per_cta();
int tsqr_reg_leaf_run(const double* x, int64_t m, int64_t ldx, int n, int64_t rpw, int nleaves, int npad,
                      double* slots, double* stats, cudaStream_t st);

size_t nnls_workspace_bytes(int t);
int nnls_max_design_cols();
int nnls_run(const double* a, int64_t n, int t, int64_t lda, const double* b, int64_t ldb, int ncols, double tol,
             int max_iter, double* y, int64_t ldy, int* status, void* ws, size_t ws_bytes, cudaStream_t st);
int xray_scores_run(const double* m, int n, int64_t ldm, const double* resid, int64_t ldr, const double* colnorm,
                    double* score, cudaStream_t st);
int xray_residual_run(const double* m, int n, int64_t ldm, const double* a, int t, int64_t lda, const double* coef,
                      int64_t ldc, double* resid, int64_t ldr, cudaStream_t st);

int scale_columns_run(const double* a, int rows, int n, int64_t lda, const double* norms, double* out, int64_t ldo,
                      cudaStream_t st);
int gp_select_run(const double* sk, int k, int n, int64_t ldsk, int r, int* out, int* count, cudaStream_t st);

int gram_max_cols();
size_t gram_workspace_bytes(int64_t m, int n);
int gram_run(const double* x, int64_t m, int n, int64_t ldx, double* g, int64_t ldg, double* l1, double* sumsq,
             void* ws, size_t ws_bytes, cudaStream_t st);

size_t sketch_workspace_bytes(int64_t m, int n, int k);
int sketch_run(const double* x, int64_t m, int n, int64_t ldx, int64_t row_offset, uint64_t seed, int k,
               const double* gexp, int64_t ldgexp, double* s, int64_t lds_out, void* ws, size_t ws_bytes,
               cudaStream_t st);

size_t stats_workspace_bytes(int64_t m, int n);
int first_nonfinite_run(const double* x, int64_t count, int64_t* first, cudaStream_t st);
int stats_run(const double* x, int64_t m, int n, int64_t ldx, double* l1, double* sumsq, void* ws, size_t ws_bytes,
              cudaStream_t st);

int uniform_block_run(uint64_t stream, uint64_t start, int64_t count, double* out, cudaStream_t st);
int normal_block_run(uint64_t stream, uint64_t start, int64_t count, double* out, cudaStream_t st);
int single_row_factor_run(const double* x, int n, double* r, int64_t ldr, cudaStream_t st);
int generate_run(double* x, int64_t ldx, int64_t row0, int64_t rows, int n, int r, const double* mix, int w_kind,
                 const double* bumps, int64_t m_total, double sigma, uint64_t seed, cudaStream_t st);

}  // namespace tsnmf

// Device selection / coefficient kernels: batched nonnegative least squares and
// the XRAY scoring / residual steps, on the small n x n reduced matrix the pass produces.
//
// Replaces the host loops of
//   nnls_solve / solve_columns   reference pkg/src/tsnmf/nnls.py:47-126   (Lawson-Hanson active set)
//   _xray_sequence scoring        reference pkg/src/tsnmf/select.py:131-135 (||resid^T M(:,j)|| / ||M(:,j)||)
//   _xray_sequence refit          reference pkg/src/tsnmf/select.py:138-140 (resid = M - M_K coef)
//
// NNLS: every target column b_j is an independent problem  min ||A y - b_j||, y >= 0  with the same
// design A (n x t, t <= 64).  One warp per column runs the reference's Lawson-Hanson iteration
// (entering variable = argmax of the gradient over the active set, lowest index on ties; inner loop with
// the step-length / leaving rule of nnls.py:60-100) in the t-dimensional normal-equation space:
// gradient g = c_j - G y with G = A^T A (one small kernel) and c_j = A^T b_j, passive-set solves by a
// Cholesky factorisation of G_FF in shared memory.  Same solution as the reference's lstsq on A_F when
// A_F has full column rank; a singular G_FF (exactly dependent design columns) is reported as a
// numerical failure instead of the reference's minimum-norm lstsq solution.
#include "common.cuh"
#include "internal.h"

namespace tsnmf {

constexpr int kNnlsMaxT = 64;

// G = A^T A (t x t, row-major, stride t): one thread per entry, fixed summation order.
__global__ void nnls_gram_kernel(const double* __restrict__ a, int64_t n, int t, int64_t lda, double* __restrict__ g) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= t * t) return;
  const int u = idx / t, v = idx % t;
  double acc = 0.0;
  for (int64_t i = 0; i < n; ++i) acc = fma(a[i * lda + u], a[i * lda + v], acc);
  g[idx] = acc;
}

__device__ __forceinline__ void warp_argmax_low(double& v, int& i) {
  // max value; ties -> lowest index (numpy argmax); -inf entries carry index 1 << 30
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov > v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}
__device__ __forceinline__ void warp_argmin_low(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, v, o);
    const int oi = __shfl_xor_sync(0xffffffffu, i, o);
    if (ov < v || (ov == v && oi < i)) {
      v = ov;
      i = oi;
    }
  }
}

// Passive-set solve G_FF z_F = c_F (Cholesky, F in increasing index order); z = 0 off F.
// Returns false if G_FF is not numerically positive definite.  L: kNnlsMaxT^2 scratch, pos: F list.
__device__ bool nnls_passive_solve(const double* __restrict__ G, int t, const double* __restrict__ c,
                                   uint64_t freemask, double* __restrict__ L, int* __restrict__ pos,
                                   double* __restrict__ w, double* __restrict__ z, int lane) {
  const int nf = __popcll(freemask);
  // F list
  for (int v = lane; v < t; v += 32)
    if ((freemask >> v) & 1ull) pos[__popcll(freemask & ((1ull << v) - 1ull))] = v;
  __syncwarp();
  // right-looking Cholesky, column k at a time; lanes own rows a = lane, lane + 32
  for (int k = 0; k < nf; ++k) {
    const int fk = pos[k];
    double d = G[fk * t + fk];
    for (int p = 0; p < k; ++p) d = fma(-L[k * kNnlsMaxT + p], L[k * kNnlsMaxT + p], d);
    if (!(d > 0.0)) return false;
    const double lkk = sqrt(d);
    for (int a = k + 1 + lane; a < nf; a += 32) {
      const int fa = pos[a];
      double s = G[fa * t + fk];
      for (int p = 0; p < k; ++p) s = fma(-L[a * kNnlsMaxT + p], L[k * kNnlsMaxT + p], s);
      L[a * kNnlsMaxT + k] = s / lkk;
    }
    if (lane == 0) L[k * kNnlsMaxT + k] = lkk;
    __syncwarp();
  }
  // forward: L w = c_F ; back: L^T z_F = w   (lane 0: n_f <= 64 sequential steps of a dot)
  if (lane == 0) {
    for (int k = 0; k < nf; ++k) {
      double s = c[pos[k]];
      for (int p = 0; p < k; ++p) s = fma(-L[k * kNnlsMaxT + p], w[p], s);
      w[k] = s / L[k * kNnlsMaxT + k];
    }
    for (int k = nf - 1; k >= 0; --k) {
      double s = w[k];
      for (int p = k + 1; p < nf; ++p) s = fma(-L[p * kNnlsMaxT + k], w[p], s);
      w[k] = s / L[k * kNnlsMaxT + k];
    }
  }
  __syncwarp();
  for (int v = lane; v < t; v += 32) z[v] = 0.0;
  __syncwarp();
  for (int k = lane; k < nf; k += 32) z[pos[k]] = w[k];
  __syncwarp();
  return true;
}

// One warp per target column.  status: 0 ok, 3 inner loop failed / singular passive set,
// 5 iteration limit (y holds the last iterate, as NnlsIterationError.best_y).
__global__ void __launch_bounds__(32) nnls_solve_kernel(const double* __restrict__ a, int64_t n, int t, int64_t lda,
                                                        const double* __restrict__ b, int64_t ldb, int ncols,
                                                        const double* __restrict__ gmat, double tol, int max_iter,
                                                        double* __restrict__ yout, int64_t ldy, int* __restrict__ status) {
  extern __shared__ __align__(16) double sm[];
  double* G = sm;                         // t x t
  double* L = G + kNnlsMaxT * kNnlsMaxT;  // kNnlsMaxT x kNnlsMaxT
  double* c = L + kNnlsMaxT * kNnlsMaxT;
  double* y = c + kNnlsMaxT;
  double* z = y + kNnlsMaxT;
  double* w = z + kNnlsMaxT;
  int* pos = reinterpret_cast<int*>(w + kNnlsMaxT);
  const int lane = threadIdx.x, col = blockIdx.x;
  for (int i = lane; i < t * t; i += 32) G[i] = gmat[i];
  // c = A^T b_col (lane v: fixed-order dot over the n rows)
  for (int v = lane; v < t; v += 32) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc = fma(a[i * lda + v], b[i * ldb + col], acc);
    c[v] = acc;
    y[v] = 0.0;
  }
  __syncwarp();
  uint64_t freemask = 0;
  int st = 5;
  for (int it = 0; it < max_iter; ++it) {
    // entering variable: argmax over the active set of g = c - G y
    double best = -INFINITY;
    int bi = 1 << 30;
    for (int v = lane; v < t; v += 32) {
      if ((freemask >> v) & 1ull) continue;
      double gv = c[v];
      for (int u = 0; u < t; ++u) gv = fma(-G[v * t + u], y[u], gv);
      if (gv > best || (gv == best && v < bi)) {
        best = gv;
        bi = v;
      }
    }
    warp_argmax_low(best, bi);
    if (!(best > tol)) {  // KKT satisfied (also: every variable free)
      st = 0;
      break;
    }
    freemask |= 1ull << bi;
    bool ok = false;
    for (int inner = 0; inner < 3 * t + 10; ++inner) {
      if (!nnls_passive_solve(G, t, c, freemask, L, pos, w, z, lane)) break;
      // strictly positive on F -> accept
      double zmin = INFINITY;
      for (int v = lane; v < t; v += 32)
        if ((freemask >> v) & 1ull) zmin = fmin(zmin, z[v]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) zmin = fmin(zmin, __shfl_xor_sync(0xffffffffu, zmin, o));
      if (zmin > 0.0) {
        for (int v = lane; v < t; v += 32) y[v] = z[v];
        __syncwarp();
        ok = true;
        break;
      }
      // step toward z until the first blocked coordinate hits zero (nnls.py restore_feasibility)
      double amin = INFINITY;
      int ai = 1 << 30;
      for (int v = lane; v < t; v += 32) {
        if (!((freemask >> v) & 1ull) || !(z[v] <= 0.0)) continue;
        const double yb = y[v], zb = z[v];
        const double alpha = (yb - zb > 0.0) ? yb / (yb - zb) : 0.0;
        if (alpha < amin || (alpha == amin && v < ai)) {
          amin = alpha;
          ai = v;
        }
      }
      warp_argmin_low(amin, ai);
      uint64_t leave = 0;
      for (int v = lane; v < t; v += 32) {
        double yv = y[v] + amin * (z[v] - y[v]);
        const bool lv = ((freemask >> v) & 1ull) && (yv <= 0.0 || v == ai);
        if (lv) yv = 0.0;
        y[v] = yv;
        if (lv) leave |= 1ull << v;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) leave |= __shfl_xor_sync(0xffffffffu, leave, o);
      freemask &= ~leave;
      __syncwarp();
    }
    if (!ok) {
      st = 3;
      break;
    }
  }
  for (int v = lane; v < t; v += 32) yout[(int64_t)v * ldy + col] = y[v];
  if (lane == 0) status[col] = st;
}

// score[j] = || resid^T M(:, j) ||_2 / colnorm[j]  (colnorm[j] <= 0 -> -inf); one CTA per column j.
__global__ void xray_scores_kernel(const double* __restrict__ m, int n, int64_t ldm, const double* __restrict__ resid,
                                   int64_t ldr, const double* __restrict__ colnorm, double* __restrict__ score) {
  __shared__ double red[32];
  const int j = blockIdx.x;
  double ss = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {  // (resid^T m_j)_i = sum_r resid[r][i] m[r][j]
    double acc = 0.0;
    for (int r = 0; r < n; ++r) acc = fma(resid[(int64_t)r * ldr + i], m[(int64_t)r * ldm + j], acc);
    ss = fma(acc, acc, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    const double cn = colnorm[j];
    score[j] = cn > 0.0 ? sqrt(tot) / cn : -INFINITY;
  }
}

// resid = M - A coef   (A: n x t design, coef: t x n)
__global__ void xray_residual_kernel(const double* __restrict__ m, int n, int64_t ldm, const double* __restrict__ a,
                                     int t, int64_t lda, const double* __restrict__ coef, int64_t ldc,
                                     double* __restrict__ resid, int64_t ldr) {
  const int i = blockIdx.x;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double acc = 0.0;
    for (int u = 0; u < t; ++u) acc = fma(a[(int64_t)i * lda + u], coef[(int64_t)u * ldc + j], acc);
    resid[(int64_t)i * ldr + j] = m[(int64_t)i * ldm + j] - acc;
  }
}

size_t nnls_workspace_bytes(int t) {
  if (t < 1 || t > kNnlsMaxT) return 0;
  return sizeof(double) * (size_t)t * t + 256;
}

int nnls_max_design_cols() { return kNnlsMaxT; }

int nnls_run(const double* a, int64_t n, int t, int64_t lda, const double* b, int64_t ldb, int ncols, double tol,
             int max_iter, double* y, int64_t ldy, int* status, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (t < 1 || t > kNnlsMaxT) return set_error(kUsage, "nnls: design has %d columns (1..%d supported)", t, kNnlsMaxT);
  if (ws_bytes < nnls_workspace_bytes(t)) return set_error(kUsage, "nnls: workspace too small");
  double* g = reinterpret_cast<double*>(ws);
  nnls_gram_kernel<<<(unsigned)ceil_div(t * t, 128), 128, 0, st>>>(a, n, t, lda, g);
  TSNMF_LAUNCH_CHECK();
  const size_t smem = sizeof(double) * (2 * kNnlsMaxT * kNnlsMaxT + 4 * kNnlsMaxT) + sizeof(int) * kNnlsMaxT;
  static PerDeviceFlag attr;
  if (!attr.is_set()) {
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(nnls_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr.set();
  }
  nnls_solve_kernel<<<ncols, 32, smem, st>>>(a, n, t, lda, b, ldb, ncols, g, tol, max_iter, y, ldy, status);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

int xray_scores_run(const double* m, int n, int64_t ldm, const double* resid, int64_t ldr, const double* colnorm,
                    double* score, cudaStream_t st) {
  xray_scores_kernel<<<n, 256, 0, st>>>(m, n, ldm, resid, ldr, colnorm, score);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

int xray_residual_run(const double* m, int n, int64_t ldm, const double* a, int t, int64_t lda, const double* coef,
                      int64_t ldc, double* resid, int64_t ldr, cudaStream_t st) {
  xray_residual_kernel<<<n, 128, 0, st>>>(m, n, ldm, a, t, lda, coef, ldc, resid, ldr);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

}  // namespace tsnmf

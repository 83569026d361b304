// Reduced-space steps on the device: the consumers of the pass's n x n / k x n output
// without a host round trip.
//   column scaling   reference tsqr.py:163-177 (R D^-1), sketch.py:87-100 (G^T X D^-1)
//   GP selection     reference select.py:159-178: per sketch row its argmin, then argmax column, appended
//                    if not yet chosen, until r columns (numpy argmin / argmax: lowest index on ties)
// (The SVD of R for the reduced matrix, tsqr.py:156-160, is a library call: cuSOLVER through torch.)
#include "common.cuh"
#include "internal.h"

namespace tsnmf {

// out(i, j) = a(i, j) / norms[j]  (rows x n, row-major strides)
__global__ void scale_columns_kernel(const double* __restrict__ a, int rows, int n, int64_t lda,
                                     const double* __restrict__ norms, double* __restrict__ out, int64_t ldo) {
  const int64_t total = (int64_t)rows * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = idx / n;
    const int j = (int)(idx - i * n);
    out[i * ldo + j] = a[i * lda + j] / norms[j];
  }
}

// One CTA scans the k sketch rows in order.  Per row: block-wide argmin and argmax (value, then lowest
// index), each appended if unseen; stops at r.  out[0..count) = selection order, *count = how many.
constexpr int kGpThreads = 512;
__device__ __forceinline__ void arg_pair_min(double& v, int& i, double v2, int i2) {
  if (v2 < v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}
__device__ __forceinline__ void arg_pair_max(double& v, int& i, double v2, int i2) {
  if (v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

__global__ void __launch_bounds__(kGpThreads) gp_select_kernel(const double* __restrict__ sk, int k, int n,
                                                               int64_t ldsk, int r, int* __restrict__ out,
                                                               int* __restrict__ count) {
  constexpr int kW = kGpThreads / 32;
  extern __shared__ __align__(16) int gp_smem[];
  double* red_v = reinterpret_cast<double*>(gp_smem);                     // [2][kW] doubles = 4 kW ints
  int* red_i = gp_smem + 4 * kW;                                          // [2][kW]
  unsigned char* seen = reinterpret_cast<unsigned char*>(gp_smem + 6 * kW);  // [n]
  __shared__ int s_cnt;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int j = tid; j < n; j += kGpThreads) seen[j] = 0;
  if (tid == 0) s_cnt = 0;
  __syncthreads();
  for (int row = 0; row < k; ++row) {
    if (s_cnt >= r) break;
    const double* p = sk + (int64_t)row * ldsk;
    double vmin = INFINITY, vmax = -INFINITY;
    int imin = 0x7fffffff, imax = 0x7fffffff;
    for (int j = tid; j < n; j += kGpThreads) {
      const double v = p[j];
      arg_pair_min(vmin, imin, v, j);
      arg_pair_max(vmax, imax, v, j);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      arg_pair_min(vmin, imin, __shfl_xor_sync(0xffffffffu, vmin, o), __shfl_xor_sync(0xffffffffu, imin, o));
      arg_pair_max(vmax, imax, __shfl_xor_sync(0xffffffffu, vmax, o), __shfl_xor_sync(0xffffffffu, imax, o));
    }
    if (lane == 0) {
      red_v[warp] = vmin;
      red_i[warp] = imin;
      red_v[kGpThreads / 32 + warp] = vmax;
      red_i[kGpThreads / 32 + warp] = imax;
    }
    __syncthreads();
    if (tid == 0) {
      double a = red_v[0], b = red_v[kGpThreads / 32];
      int ia = red_i[0], ib = red_i[kGpThreads / 32];
      for (int w = 1; w < kGpThreads / 32; ++w) {
        arg_pair_min(a, ia, red_v[w], red_i[w]);
        arg_pair_max(b, ib, red_v[kGpThreads / 32 + w], red_i[kGpThreads / 32 + w]);
      }
      int c = s_cnt;
      const int cand[2] = {ia, ib};
      for (int q = 0; q < 2 && c < r; ++q) {
        const int j = cand[q];
        if (j >= 0 && j < n && !seen[j]) {
          seen[j] = 1;
          out[c++] = j;
        }
      }
      s_cnt = c;
    }
    __syncthreads();
  }
  if (tid == 0) *count = s_cnt;
}

int scale_columns_run(const double* a, int rows, int n, int64_t lda, const double* norms, double* out, int64_t ldo,
                      cudaStream_t st) {
  if (rows <= 0 || n <= 0) return kOk;
  const int64_t total = (int64_t)rows * n;
  const int blocks = (int)std::min<int64_t>(ceil_div(total, 256), 4 * kNumSMs);
  scale_columns_kernel<<<blocks, 256, 0, st>>>(a, rows, n, lda, norms, out, ldo);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

int gp_select_run(const double* sk, int k, int n, int64_t ldsk, int r, int* out, int* count, cudaStream_t st) {
  const size_t smem = sizeof(int) * 6 * (kGpThreads / 32) + (size_t)n;
  static PerDeviceFlag attr;
  if (smem > 48 * 1024 && !attr.is_set()) {
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(gp_select_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr.set();
  }
  gp_select_kernel<<<1, kGpThreads, smem, st>>>(sk, k, n, ldsk, r, out, count);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

}  // namespace tsnmf

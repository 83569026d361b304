// Counter-RNG block kernels, standalone column statistics, single-row factor, and the
// BASELINE.json config generators (synthetic X written straight into HBM).
#include "common.cuh"
#include "internal.h"

namespace tsnmf {

// reference pkg/src/tsnmf/_kernels.pyx:35-46 (uniform_block) / :49-69 (normal_block)
__global__ void uniform_block_kernel(uint64_t stream, uint64_t start, int64_t count, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rng_uniform(stream, start + (uint64_t)i);
}

__global__ void normal_block_kernel(uint64_t stream, uint64_t start, int64_t count, double* __restrict__ out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = rng_normal(stream, start + (uint64_t)i);
}

int uniform_block_run(uint64_t stream, uint64_t start, int64_t count, double* out, cudaStream_t st) {
  if (count <= 0) return kOk;
  const int64_t blocks = min64(ceil_div(count, 256), 148 * 16);
  uniform_block_kernel<<<(unsigned)blocks, 256, 0, st>>>(stream, start, count, out);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

int normal_block_run(uint64_t stream, uint64_t start, int64_t count, double* out, cudaStream_t st) {
  if (count <= 0) return kOk;
  const int64_t blocks = min64(ceil_div(count, 256), 148 * 16);
  normal_block_kernel<<<(unsigned)blocks, 256, 0, st>>>(stream, start, count, out);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// Column l1 / sum of squares (reference tsqr.py:190-192) as a standalone pass: each CTA reduces a
// row range for a 256-column window; partials summed in fixed order.
constexpr int kStRows = 4096;

__global__ void col_stats_kernel(const double* __restrict__ x, int64_t m, int n, int64_t ldx, int64_t rows_per,
                                 double* __restrict__ part) {
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per;
  const int64_t r1 = min64(m, r0 + rows_per);
  if (col >= n) return;
  double a = 0.0, q = 0.0;
  for (int64_t i = r0; i < r1; ++i) {
    const double v = x[i * ldx + col];
    a += fabs(v);
    q = fma(v, v, q);
  }
  part[(int64_t)blockIdx.y * 2 * n + col] = a;
  part[(int64_t)blockIdx.y * 2 * n + n + col] = q;
}

__global__ void col_stats_reduce_kernel(const double* __restrict__ part, int64_t splits, int n,
                                        double* __restrict__ l1, double* __restrict__ sumsq) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double a = 0.0, q = 0.0;
  for (int64_t s = 0; s < splits; ++s) {
    a += part[s * 2 * n + j];
    q += part[s * 2 * n + n + j];
  }
  if (l1) l1[j] = a;
  if (sumsq) sumsq[j] = q;
}

size_t stats_workspace_bytes(int64_t m, int n) {
  const int64_t splits = max64(1, ceil_div(max64(m, 1), kStRows));
  return sizeof(double) * (size_t)(splits * 2 * n) + 256;
}

int stats_run(const double* x, int64_t m, int n, int64_t ldx, double* l1, double* sumsq, void* ws, size_t ws_bytes,
              cudaStream_t st) {
  const int64_t splits = max64(1, ceil_div(m, kStRows));
  const size_t need = sizeof(double) * (size_t)(splits * 2 * n);
  if (ws_bytes < need) return set_error(kUsage, "stats: workspace too small (%zu < %zu bytes)", ws_bytes, need);
  double* part = reinterpret_cast<double*>(ws);
  col_stats_kernel<<<dim3((unsigned)ceil_div(n, 128), (unsigned)splits), 128, 0, st>>>(x, m, n, ldx, kStRows, part);
  TSNMF_LAUNCH_CHECK();
  col_stats_reduce_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(part, splits, n, l1, sumsq);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// single-row factor (reference tsqr.py:135-139): the row itself, negated if row[0] < 0, zero padded.
__global__ void single_row_factor_kernel(const double* __restrict__ x, int n, double* __restrict__ r, int64_t ldr) {
  const double sg = x[0] < 0.0 ? -1.0 : 1.0;
  for (int64_t idx = threadIdx.x; idx < (int64_t)n * n; idx += blockDim.x) {
    const int i = (int)(idx / n), j = (int)(idx % n);
    r[(int64_t)i * ldr + j] = (i == 0) ? sg * x[j] : 0.0;
  }
}

int single_row_factor_run(const double* x, int n, double* r, int64_t ldr, cudaStream_t st) {
  single_row_factor_kernel<<<1, 256, 0, st>>>(x, n, r, ldr);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// Config generator: rows [row0, row0 + rows) of X = max(W M + sigma N, 0), M = [I H'] Pi
// (r x n, host-computed), W by kind: 0 uniform (tag 4 counters i*r + t), 1 lognormal exp(normal),
// 2 bumps (4 Gaussian bumps over the row position, params r x 4 x 3).  Noise: normal #(i*n + j), tag 7.
// Transcendentals of the generator are fp32 (rng_normal_f32, expf): ~1e10 of them per C2/C5 run.
// Same term order as the oracle (oracle/tsnmf_oracle.py config_rows), no FMA contraction.
__global__ void generate_kernel(double* __restrict__ x, int64_t ldx, int64_t row0, int64_t rows, int n, int r,
                                const double* __restrict__ mix, int w_kind, const double* __restrict__ bumps,
                                int64_t m_total, double sigma, uint64_t w_stream, uint64_t noise_stream) {
  extern __shared__ double sm[];
  double* mix_s = sm;           // r * n
  double* w_s = sm + r * n;     // blockDim.y rows * r
  for (int idx = threadIdx.y * blockDim.x + threadIdx.x; idx < r * n; idx += blockDim.x * blockDim.y)
    mix_s[idx] = mix[idx];
  const int64_t i_local = (int64_t)blockIdx.x * blockDim.y + threadIdx.y;
  const int64_t i = row0 + i_local;
  double* wrow = w_s + threadIdx.y * r;
  if (i_local < rows) {
    for (int t = threadIdx.x; t < r; t += blockDim.x) {
      double w;
      const uint64_t ctr = (uint64_t)i * (uint64_t)r + (uint64_t)t;
      if (w_kind == 0) {
        w = rng_uniform(w_stream, ctr);
      } else if (w_kind == 1) {
        w = (double)expf(rng_normal_f32(w_stream, ctr));
      } else {
        const double pos = __ddiv_rn(__dadd_rn((double)i, 0.5), (double)m_total);
        w = 0.0;
        for (int q = 0; q < 4; ++q) {
          const double* p = bumps + (t * 4 + q) * 3;
          const float z = (float)__ddiv_rn(__dsub_rn(pos, p[1]), p[2]);
          w = __dadd_rn(w, __dmul_rn(p[0], (double)expf(__fmul_rn(__fmul_rn(-0.5f, z), z))));
        }
      }
      wrow[t] = w;
    }
  }
  __syncthreads();
  if (i_local >= rows) return;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double acc = 0.0;
    for (int t = 0; t < r; ++t) acc = __dadd_rn(acc, __dmul_rn(wrow[t], mix_s[t * n + j]));
    if (sigma > 0.0)
      acc = __dadd_rn(acc, __dmul_rn(sigma, (double)rng_normal_f32(noise_stream, (uint64_t)i * (uint64_t)n + (uint64_t)j)));
    x[i_local * ldx + j] = acc > 0.0 ? acc : 0.0;
  }
}

int generate_run(double* x, int64_t ldx, int64_t row0, int64_t rows, int n, int r, const double* mix, int w_kind,
                 const double* bumps, int64_t m_total, double sigma, uint64_t seed, cudaStream_t st) {
  if (rows <= 0) return kOk;
  const dim3 block(32, 8);
  const size_t smem = sizeof(double) * (size_t)(r * n + 8 * r);
  if (smem > 200 * 1024) return set_error(kUsage, "generate: r * n too large");
  static PerDeviceFlag attr;
  if (!attr.is_set()) {
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(generate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr.set();
  }
  generate_kernel<<<(unsigned)ceil_div(rows, 8), block, smem, st>>>(x, ldx, row0, rows, n, r, mix, w_kind, bumps,
                                                                   m_total, sigma, derive_stream(seed, kTagCfgW),
                                                                   derive_stream(seed, kTagCfgNoise));
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

// ---------------------------------------------------------------------------
// Ingest validation (reference matio.py:81-87 _check_finite): the first non-finite
// element of a contiguous row-major batch, as a linear index (-1 when all are finite).  HBM-bound:
// 16-byte loads, one exponent test per element, a warp vote, one atomicMin per warp that saw one.
__global__ void first_nonfinite_kernel(const double* __restrict__ x, int64_t count,
                                       unsigned long long* __restrict__ first) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t pairs = count >> 1;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  unsigned long long best = ~0ull;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += stride) {
    const double2 v = __ldg(&x2[i]);
    // exponent all ones <=> Inf or NaN
    const bool b0 = (__double2hiint(v.x) & 0x7ff00000) == 0x7ff00000;
    const bool b1 = (__double2hiint(v.y) & 0x7ff00000) == 0x7ff00000;
    if (b0 || b1) {
      const unsigned long long idx = (unsigned long long)(2 * i + (b0 ? 0 : 1));
      best = idx < best ? idx : best;
    }
  }
  if ((count & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const double v = x[count - 1];
    if ((__double2hiint(v) & 0x7ff00000) == 0x7ff00000) best = best < (unsigned long long)(count - 1) ? best : count - 1;
  }
  if (__any_sync(0xffffffffu, best != ~0ull)) {
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other < best ? other : best;
    }
    if ((threadIdx.x & 31) == 0) atomicMin(first, best);
  }
}

int first_nonfinite_run(const double* x, int64_t count, int64_t* first, cudaStream_t st) {
  static_assert(sizeof(unsigned long long) == sizeof(int64_t), "index width");
  TSNMF_CUDA_CHECK(cudaMemsetAsync(first, 0xff, sizeof(int64_t), st));  // -1: all finite
  if (count <= 0) return kOk;
  int sms = 0, dev = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = kNumSMs;
  const int64_t want = ceil_div(max64(count >> 1, 1), 256);
  const unsigned blocks = (unsigned)min64(want, (int64_t)sms * 8);
  first_nonfinite_kernel<<<blocks, 256, 0, st>>>(x, count, reinterpret_cast<unsigned long long*>(first));
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

}  // namespace tsnmf

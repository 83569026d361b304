// Gaussian projection S = G^T X (k x n) with G regenerated in-kernel from the counter RNG.
//
// Replaces reference pkg/src/tsnmf/sketch.py:62-73 (sketch_chunk: rng.gaussian_rows + g.T @ data) and
// the per-chunk merge sketch.py:76-84.  G[i, t] is normal #((row_offset + i) * k + t) of the stream
// derive_stream(seed, TAG_SKETCH) (reference rng.py:48-55, _kernels.pyx:49-69); it is never
// materialised in HBM (215 GB at BASELINE config C2): each CTA generates the G slab it needs into
// shared memory, exactly once per (row, t) over the whole grid.
//
// grid = (t groups x column groups, row splits).  A CTA owns 64 sketch rows (8 DMMA row blocks) and up
// to 26 column blocks of 8; warps split it as 4 t-pairs x 2 column parities.  X rows are staged by
// cp.async (double buffered); per-split partials are summed in fixed order by sketch_reduce_kernel.
// Optional explicit-G mode (g != nullptr): G (m x k, row-major) is read instead of generated.
#include "common.cuh"
#include "internal.h"

namespace tsnmf {

constexpr int kSkThreads = 256;
constexpr int kSkT = 64;      // sketch rows per CTA
constexpr int kSkCbMax = 26;  // column blocks per CTA
constexpr int kSkCbw = 13;    // column blocks per warp
constexpr int kSkBr = 32;     // rows per stage
constexpr int kSkLdg = 72;    // smem stride of the G slab (64 + 8, % 16 == 8)

struct SkGeom {
  int n, npad, lds, k;
  int tgroups, cgroups;
  int64_t rows_per_split;
  uint64_t stream;
  int64_t row_offset;
};

__global__ void __launch_bounds__(kSkThreads, 1)
    sketch_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, const double* __restrict__ gexp,
                  int64_t ldgexp, SkGeom g, double* __restrict__ partial) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tg = blockIdx.x % g.tgroups, cg = blockIdx.x / g.tgroups;
  const int64_t split = blockIdx.y;
  const int64_t rbeg = split * g.rows_per_split;
  const int64_t rend = min64(m, rbeg + g.rows_per_split);
  const int lds = g.lds;
  double* xbuf[2] = {smem, smem + kSkBr * lds};
  double* gs = smem + 2 * kSkBr * lds;
  const bool vec16 = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  const int t0 = tg * kSkT;
  const int cb_lo = cg * kSkCbMax;
  const int ncb = g.npad / 8;
  const int cb_hi = min(ncb, cb_lo + kSkCbMax);

  // warp -> (t blocks tb0, tb0 + 1) x (column blocks cb_lo + par + 2u)
  const int tb0 = 2 * (warp >> 1), par = warp & 1;
  const bool tv0 = t0 + 8 * tb0 < g.k, tv1 = t0 + 8 * (tb0 + 1) < g.k;
  double acc[2][kSkCbw][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int u = 0; u < kSkCbw; ++u) acc[a][u][0] = acc[a][u][1] = 0.0;

  const int64_t nstages = ceil_div(max64(rend - rbeg, 0), kSkBr);
  // column window staged: [8*cb_lo, 8*cb_hi) of the real n columns
  const int c_lo = 8 * cb_lo;
  const int c_real = max(0, min(g.n, 8 * cb_hi) - c_lo);
  const int c_tot = 8 * (cb_hi - cb_lo);
  if (nstages > 0) {
    stage_rows(xbuf[0], lds, x + rbeg * ldx + c_lo, ldx, (int)min64(kSkBr, rend - rbeg), c_real, kSkBr,
               c_tot, vec16 && ((c_lo & 1) == 0));
    cp_async_commit();
  }
  for (int64_t s = 0; s < nstages; ++s) {
    const int64_t r0 = rbeg + s * kSkBr;
    const int cnt = (int)min64(kSkBr, rend - r0);
    if (s + 1 < nstages) {
      const int64_t r1 = r0 + kSkBr;
      stage_rows(xbuf[(s + 1) & 1], lds, x + r1 * ldx + c_lo, ldx, (int)min64(kSkBr, rend - r1), c_real,
                 kSkBr, c_tot, vec16 && ((c_lo & 1) == 0));
      cp_async_commit();
    }
    // G slab for rows [r0, r0 + kSkBr), sketch rows [t0, t0 + 64)
    for (int idx = tid; idx < kSkBr * kSkT; idx += kSkThreads) {
      const int i = idx / kSkT, t = idx % kSkT;
      double v = 0.0;
      if (i < cnt && t0 + t < g.k) {
        const int64_t row = r0 + i;
        if (gexp) {
          v = gexp[row * ldgexp + t0 + t];
        } else {
          const uint64_t j = (uint64_t)(g.row_offset + row) * (uint64_t)g.k + (uint64_t)(t0 + t);
          v = rng_normal(g.stream, j);
        }
      }
      gs[i * kSkLdg + t] = v;
    }
    if (s + 1 < nstages) cp_async_wait<1>(); else cp_async_wait<0>();
    __syncthreads();
    const double* xs = xbuf[s & 1];
#pragma unroll 2
    for (int i = 0; i < kSkBr; i += 4) {
      const double* grow = gs + (i + (lane & 3)) * kSkLdg + (lane >> 2);
      const double* xrow = xs + (i + (lane & 3)) * lds + (lane >> 2);
      const double a0 = grow[8 * tb0], a1 = grow[8 * tb0 + 8];
#pragma unroll
      for (int u = 0; u < kSkCbw; ++u) {
        const int cb = cb_lo + par + 2 * u;
        if (cb < cb_hi) {
          const double b = xrow[8 * (cb - cb_lo)];
          if (tv0) dmma(acc[0][u][0], acc[0][u][1], a0, b);
          if (tv1) dmma(acc[1][u][0], acc[1][u][1], a1, b);
        }
      }
    }
    __syncthreads();
  }
  // partial layout: [split][k][npad]
  double* dst = partial + split * (int64_t)g.k * g.npad;
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int tb = tb0 + a;
    const int trow = t0 + 8 * tb + (lane >> 2);
#pragma unroll
    for (int u = 0; u < kSkCbw; ++u) {
      const int cb = cb_lo + par + 2 * u;
      if (cb < cb_hi && trow < g.k) {
        const int col = 8 * cb + 2 * (lane & 3);
        dst[(int64_t)trow * g.npad + col] = acc[a][u][0];
        dst[(int64_t)trow * g.npad + col + 1] = acc[a][u][1];
      }
    }
  }
}

__global__ void sketch_reduce_kernel(const double* __restrict__ partial, int64_t splits, int k, int n, int npad,
                                     double* __restrict__ s, int64_t lds_out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)k * n) return;
  const int t = (int)(idx / n), j = (int)(idx % n);
  double acc = 0.0;
  for (int64_t p = 0; p < splits; ++p) acc += partial[(p * k + t) * npad + j];
  s[(int64_t)t * lds_out + j] = acc;
}

namespace {

int sk_sms() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = kNumSMs;
  return sms;
}

SkGeom sk_geom(int64_t m, int n, int k) {
  SkGeom g;
  g.n = n;
  g.k = k;
  g.npad = (int)round_up(n, 8);
  g.tgroups = (int)ceil_div(k, kSkT);
  g.cgroups = (int)ceil_div(g.npad / 8, kSkCbMax);
  const int cols = 8 * std::min(g.npad / 8, kSkCbMax);
  g.lds = smem_stride(cols);
  const int64_t per = (int64_t)g.tgroups * g.cgroups;
  const int64_t target = max64(1, (int64_t)2 * sk_sms() / per);
  const int64_t splits = max64(1, min64(target, ceil_div(m, 2 * kSkBr)));
  g.rows_per_split = round_up(ceil_div(m, splits), kSkBr);
  g.stream = 0;
  g.row_offset = 0;
  return g;
}

int64_t sk_splits(int64_t m, const SkGeom& g) { return max64(1, ceil_div(m, g.rows_per_split)); }

}  // namespace

size_t sketch_workspace_bytes(int64_t m, int n, int k) {
  if (n < 1 || k < 1) return 0;
  SkGeom g = sk_geom(max64(m, 1), n, k);
  return sizeof(double) * (size_t)(sk_splits(max64(m, 1), g) * k * g.npad) + 256;
}

int sketch_run(const double* x, int64_t m, int n, int64_t ldx, int64_t row_offset, uint64_t seed, int k,
               const double* gexp, int64_t ldgexp, double* s, int64_t lds_out, void* ws, size_t ws_bytes,
               cudaStream_t st) {
  SkGeom g = sk_geom(m, n, k);
  g.stream = derive_stream(seed, kTagSketch);
  g.row_offset = row_offset;
  const int64_t splits = sk_splits(m, g);
  const size_t need = sizeof(double) * (size_t)(splits * k * g.npad);
  if (ws_bytes < need) return set_error(kUsage, "sketch: workspace too small (%zu < %zu bytes)", ws_bytes, need);
  double* partial = reinterpret_cast<double*>(ws);
  const size_t smem = sizeof(double) * (size_t)(2 * kSkBr * g.lds + kSkBr * kSkLdg);
  static bool attr = false;
  if (!attr) {
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(sketch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr = true;
  }
  prof_mark(kProfSketch, true, st);
  sketch_kernel<<<dim3((unsigned)(g.tgroups * g.cgroups), (unsigned)splits), kSkThreads, smem, st>>>(
      x, m, ldx, gexp, ldgexp, g, partial);
  TSNMF_LAUNCH_CHECK();
  prof_mark(kProfSketch, false, st);
  const int64_t tot = (int64_t)k * n;
  sketch_reduce_kernel<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(partial, splits, k, n, g.npad, s, lds_out);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

}  // namespace tsnmf

// Gram reduction G = X^T X (+ fused column l1; sum of squares = diag G).
//
// NEW relative to the reference (no Gram code there: reference pkg/src/tsnmf/tsqr.py:6 "The Gram
// matrix is never formed"); its parity anchor is the reference invariant
// ||R^T R - X^T X||_F <= 1e-10 ||X^T X||_F (reference SPEC.md:164) and a per-chunk X.T @ X oracle.
//
// Layout: G is computed in 16x16 "super-tiles" (2x2 DMMA 8x8 tiles) over the upper triangle only.
// grid = (tile groups, row splits).  A CTA stages BR rows of X into shared memory (cp.async, double
// buffered) and each warp accumulates its super-tiles in registers; every 4 rows is one DMMA k-step
// whose A and B fragments are the same 4x8 slab pattern X[i + l%4][8*cb + l/4].  Per-CTA partials go
// to the workspace and are summed in a fixed order (deterministic) by gram_reduce_kernel.
#include "common.cuh"
#include "internal.h"

namespace tsnmf {

#ifndef TSNMF_GRAM_WARPS
#define TSNMF_GRAM_WARPS 8
#endif
constexpr int kGrWarps = TSNMF_GRAM_WARPS;   // narrow widths: 2 warps per SMSP
constexpr int kGrWarpsWide = 16;             // n > 192: 4 warps per SMSP hide the fragment-load latency
                                             // better (+2..6% at n = 200..512; slower for narrow widths)
constexpr int kGrSpwMax = 96 / kGrWarps;     // super-tiles per warp (96 per CTA = one group at n <= 208)
constexpr int kGrBrMax = 256;  // rows per stage (halved until the double buffer fits)

struct GrGeom {
  int n, npad;  // npad = round_up(n, 16)
  int lds;      // smem stride (% 16 == 8, swizzled)
  int ns;       // super-blocks per side (npad / 16)
  int nst;      // super-tiles in the upper triangle
  int ks;       // k-slices per CTA (warps sharing a super-tile set, splitting the rows)
  int spw;      // super-tiles per warp (kernel template: 1, 3, 6, 10 or 12)
  int warps;    // warps per CTA (kernel template: 8 or 16)
  int spc;      // super-tiles per CTA (tile group) = (8 / ks) * spw
  int groups;   // tile groups
  int br;       // rows per stage
  int64_t rows_per_split;
};

__host__ __device__ inline void st_coords(int idx, int ns, int* P, int* Q) {
  // row-major enumeration of {(P, Q) : 0 <= P <= Q < ns}
  int p = 0, rem = idx;
  while (rem >= ns - p) {
    rem -= ns - p;
    ++p;
  }
  *P = p;
  *Q = p + rem;
}

// Warp w = kslice + ks * wi: k-slice `kslice` takes the 4-row k-steps i/4 = kslice (mod ks); warp index
// wi within the slice owns a contiguous run of SPW super-tiles (consecutive super-tiles mostly share
// their row P, so the A fragments are reused).  Partials: [split][kslice][supertile][16][16].
template <int SPW, int WARPS>
__global__ void __launch_bounds__(32 * WARPS, 1)
    gram_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, GrGeom g, double* __restrict__ partial,
                double* __restrict__ l1part) {
  extern __shared__ __align__(16) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int group = blockIdx.x;
  const int64_t split = blockIdx.y;
  const int64_t rbeg = split * g.rows_per_split;
  const int64_t rend = min64(m, rbeg + g.rows_per_split);
  const int lds = g.lds, br = g.br, ks = g.ks;
  const int kslice = warp % ks, wi = warp / ks;
  const bool vec16 = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);

  // packed super-tile coordinates: (16 P) << 16 | 16 Q; the first nvalid are real
  int stPQ[SPW];
  const int first = group * g.spc + wi * SPW;
  const int nvalid = max(0, min(SPW, g.nst - first));
#pragma unroll
  for (int u = 0; u < SPW; ++u) {
    int P = 0, Q = 0;
    if (u < nvalid) st_coords(first + u, g.ns, &P, &Q);
    stPQ[u] = (16 * P) << 16 | (16 * Q);
  }
  double acc[SPW][4][2];
#pragma unroll
  for (int u = 0; u < SPW; ++u)
#pragma unroll
    for (int t = 0; t < 4; ++t) acc[u][t][0] = acc[u][t][1] = 0.0;
  double l1x = 0.0, l1y = 0.0;  // this thread's column pair (l1_c, l1_c + 1)
  const bool do_l1 = (group == 0) && (l1part != nullptr);
  // column l1: each thread sums a column PAIR (16-byte loads; the swizzle keeps pairs adjacent) over the
  // rows of its phase; the pairs' rows are split over l1_ph thread phases
  const int npairs = g.npad / 2;
  const int l1_ph = (32 * WARPS) / npairs;  // >= 1 for npad <= 1024
  const int l1_c = 2 * (tid % npairs), l1_r0 = tid / npairs;
  const int frag_col = (lane >> 2) ^ ((lane & 2) << 1);  // swizzled slab fragment: row i + l%4, col l/4

  const int64_t nstages = ceil_div(max64(rend - rbeg, 0), br);
  if (nstages > 0) {
    stage_rows_swz(smem, lds, x + rbeg * ldx, ldx, (int)min64(br, rend - rbeg), g.n, br, g.npad, vec16);
    cp_async_commit();
  }
  for (int64_t s = 0; s < nstages; ++s) {
    if (s + 1 < nstages) {
      const int64_t r0 = rbeg + (s + 1) * br;
      stage_rows_swz(smem + ((s + 1) & 1) * br * lds, lds, x + r0 * ldx, ldx, (int)min64(br, rend - r0), g.n, br,
                     g.npad, vec16);
      cp_async_commit();
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const double* xs = smem + (s & 1) * br * lds;
    if (do_l1) {
      if (l1_r0 < l1_ph && l1_c < g.n) {
        double a0 = 0.0, a1 = 0.0;
        for (int i = l1_r0; i < br; i += l1_ph) {
          const double2 v = *reinterpret_cast<const double2*>(xs + i * lds + swz_col(i, l1_c));
          a0 += fabs(v.x);
          a1 += fabs(v.y);
        }
        l1x += a0;
        l1y += a1;
      }
    }
    // branch-free DMMA issue: padding super-tiles (u >= nvalid) compute on (0, 0) and are not stored;
    // diagonal super-tiles also form their (unused) lower tile
#pragma unroll 1
    for (int i = 4 * kslice; i < br; i += 4 * ks) {
      const double* row = xs + (i + (lane & 3)) * lds + frag_col;
#pragma unroll
      for (int u = 0; u < SPW; ++u) {
        const int P16 = stPQ[u] >> 16, Q16 = stPQ[u] & 0xffff;
        const double a0 = row[P16], a1 = row[P16 + 8];
        const double b0 = row[Q16], b1 = row[Q16 + 8];
        dmma(acc[u][0][0], acc[u][0][1], a0, b0);
        dmma(acc[u][1][0], acc[u][1][1], a0, b1);
        dmma(acc[u][2][0], acc[u][2][1], a1, b0);
        dmma(acc[u][3][0], acc[u][3][1], a1, b1);
      }
    }
    __syncthreads();  // buffer reuse
  }
#pragma unroll
  for (int u = 0; u < SPW; ++u) {
    if (u >= nvalid) break;
    const int idx = first + u;
    double* dst = partial + ((split * ks + kslice) * g.nst + idx) * 256;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int ti = t >> 1, tj = t & 1;
      const int row = 8 * ti + (lane >> 2), col = 8 * tj + 2 * (lane & 3);
      dst[row * 16 + col] = acc[u][t][0];
      dst[row * 16 + col + 1] = acc[u][t][1];
    }
  }
  if (do_l1) {  // fixed-order sum of the row phases through shared memory
    __syncthreads();
    if (l1_r0 < l1_ph) {
      smem[l1_r0 * g.npad + l1_c] = l1x;
      smem[l1_r0 * g.npad + l1_c + 1] = l1y;
    }
    __syncthreads();
    for (int c = tid; c < g.npad; c += 32 * WARPS) {
      double a = 0.0;
      for (int r = 0; r < l1_ph; ++r) a += smem[r * g.npad + c];
      l1part[split * g.npad + c] = a;
    }
  }
}

__global__ void gram_reduce_kernel(const double* __restrict__ partial, int64_t splits, GrGeom g,
                                   double* __restrict__ out, int64_t ldg, double* __restrict__ sumsq) {
  const int i = blockIdx.x;  // output row
  for (int j = i + threadIdx.x; j < g.n; j += blockDim.x) {
    const int P = i / 16, Q = j / 16;
    int idx = 0;
    for (int p = 0; p < P; ++p) idx += g.ns - p;
    idx += Q - P;
    const int64_t off = (int64_t)idx * 256 + (i % 16) * 16 + (j % 16);
    double acc = 0.0;
    for (int64_t s = 0; s < splits * g.ks; ++s) acc += partial[s * g.nst * 256 + off];
    out[(int64_t)i * ldg + j] = acc;
    out[(int64_t)j * ldg + i] = acc;
    if (i == j && sumsq) sumsq[i] = acc;
  }
}

__global__ void l1_reduce_kernel(const double* __restrict__ l1part, int64_t splits, int stride, int n,
                                 double* __restrict__ l1) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double a = 0.0;
  for (int64_t s = 0; s < splits; ++s) a += l1part[s * stride + j];
  l1[j] = a;
}

namespace {

GrGeom gr_geom(int64_t m, int n, int sms) {
  GrGeom g;
  g.n = n;
  g.npad = (int)round_up(n, 16);
  g.lds = smem_stride(g.npad);
  g.ns = g.npad / 16;
  g.nst = g.ns * (g.ns + 1) / 2;
  // Narrow matrices have few super-tiles: pick the per-warp count SPW (a kernel template) and the warps per
  // k-slice wps (power of two) minimising the DMMA slots issued per k-step, wps * SPW >= nst; the
  // remaining warps split the rows (ks = 8 / wps k-slices).  Wide ones use SPW = 12, wps = 8 and tile groups.
  {
    const int spws[5] = {1, 3, 6, 10, 12};
    int best_slots = 1 << 30;
    g.warps = kGrWarps;
    g.spw = kGrSpwMax;
    g.ks = 1;
    for (int wps = 1; wps <= kGrWarps; wps *= 2)
      for (int i = 0; i < 5; ++i)
        if (spws[i] <= kGrSpwMax && wps * spws[i] >= g.nst && wps * spws[i] < best_slots) {
          best_slots = wps * spws[i];
          g.spw = spws[i];
          g.ks = kGrWarps / wps;
        }
    if (g.nst > 80) {  // wide (n > 192): 16 warps x 6 super-tiles (same 96 per tile group, half the registers)
      g.warps = kGrWarpsWide;
      g.spw = 96 / kGrWarpsWide;
      g.ks = 1;
    }
  }
  g.spc = (g.warps / g.ks) * g.spw;
  g.groups = (int)ceil_div(g.nst, g.spc);
  g.br = kGrBrMax;
  while (g.br > 8 && 2 * g.br * g.lds * 8 > 227 * 1024) g.br /= 2;
  const int64_t target = max64(1, (int64_t)sms / g.groups);
  const int64_t splits = max64(1, min64(target, ceil_div(m, 4 * g.br)));
  g.rows_per_split = round_up(ceil_div(m, splits), g.br);
  return g;
}

size_t gr_smem(const GrGeom& g) { return sizeof(double) * 2 * g.br * (size_t)g.lds; }

int64_t gr_splits(int64_t m, const GrGeom& g) { return max64(1, ceil_div(m, g.rows_per_split)); }

int sm_count() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = kNumSMs;
  return sms;
}

}  // namespace

int gram_max_cols() { return 512; }

size_t gram_workspace_bytes(int64_t m, int n) {
  if (n < 1 || n > gram_max_cols()) return 0;
  GrGeom g = gr_geom(max64(m, 1), n, sm_count());
  const int64_t splits = gr_splits(max64(m, 1), g);
  return sizeof(double) * (size_t)(splits * g.ks * g.nst * 256 + splits * g.npad) + 256;
}

template <int SPW, int WARPS>
int gram_launch(const double* x, int64_t m, int64_t ldx, const GrGeom& g, double* partial, double* l1part,
                int64_t splits, size_t smem, cudaStream_t st) {
  static PerDeviceFlag attr;
  if (!attr.is_set()) {
    TSNMF_CUDA_CHECK((cudaFuncSetAttribute(gram_kernel<SPW, WARPS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           232448)));
    attr.set();
  }
  gram_kernel<SPW, WARPS><<<dim3(g.groups, (unsigned)splits), 32 * WARPS, smem, st>>>(x, m, ldx, g, partial, l1part);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

int gram_run(const double* x, int64_t m, int n, int64_t ldx, double* gout, int64_t ldg, double* l1, double* sumsq,
             void* ws, size_t ws_bytes, cudaStream_t st) {
  if (n > gram_max_cols()) return set_error(kUsage, "gram: n = %d exceeds %d", n, gram_max_cols());
  GrGeom g = gr_geom(m, n, sm_count());
  const int64_t splits = gr_splits(m, g);
  const size_t need = sizeof(double) * (size_t)(splits * g.ks * g.nst * 256 + splits * g.npad);
  if (ws_bytes < need) return set_error(kUsage, "gram: workspace too small (%zu < %zu bytes)", ws_bytes, need);
  double* partial = reinterpret_cast<double*>(ws);
  double* l1part = partial + splits * g.ks * g.nst * 256;
  const size_t smem = gr_smem(g);
  prof_mark(kProfGram, true, st);
  int rc = kOk;
  if (g.warps == kGrWarpsWide) {
    rc = gram_launch<96 / kGrWarpsWide, kGrWarpsWide>(x, m, ldx, g, partial, l1 ? l1part : nullptr, splits, smem, st);
  } else {
    switch (g.spw) {
      case 1: rc = gram_launch<1, kGrWarps>(x, m, ldx, g, partial, l1 ? l1part : nullptr, splits, smem, st); break;
      case 3: rc = gram_launch<3, kGrWarps>(x, m, ldx, g, partial, l1 ? l1part : nullptr, splits, smem, st); break;
      case 6: rc = gram_launch<6, kGrWarps>(x, m, ldx, g, partial, l1 ? l1part : nullptr, splits, smem, st); break;
      case 10: rc = gram_launch<10, kGrWarps>(x, m, ldx, g, partial, l1 ? l1part : nullptr, splits, smem, st); break;
      default: rc = gram_launch<12, kGrWarps>(x, m, ldx, g, partial, l1 ? l1part : nullptr, splits, smem, st); break;
    }
  }
  if (rc) return rc;
  prof_mark(kProfGram, false, st);
  gram_reduce_kernel<<<n, 128, 0, st>>>(partial, splits, g, gout, ldg, sumsq);
  TSNMF_LAUNCH_CHECK();
  if (l1) {
    l1_reduce_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(l1part, splits, g.npad, n, l1);
    TSNMF_LAUNCH_CHECK();
  }
  return kOk;
}

}  // namespace tsnmf

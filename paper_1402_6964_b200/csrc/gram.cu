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

// ---------------------------------------------------------------------------
// Narrow Gram (n <= 32, e.g. config C4 n = 25): HBM-bound (3.25 flop/B at n = 25), so no shared
// memory staging at all.  Both DMMA operands of a 4-row k-step are the same fragment X[i + l%4][8T + l/4]
// (tile column T), so each lane loads its fragments straight from global memory (TC 8-byte loads per
// k-step, U k-steps per group in flight, the next group's loads issued before the current group's DMMAs)
// and every warp accumulates the whole upper triangle (TC (TC + 1) / 2 tiles) in registers.  A width of the
// form 8 TC + 1 (25 = 24 + 1) keeps its last column off the tensor pipe: padding it to a fourth tile column
// would add 4 DMMAs per k-step (10 instead of 6) for 25 useful products, so its 8 TC + 1 dot products are
// plain FMAs against the fragments already in registers (RT = 1).  Column l1 comes from the fragments,
// sum of squares = diag G.  Warps take row groups round-robin; warp partials are summed in warp order
// through shared memory, CTA partials in CTA order by gram_narrow_reduce_kernel (deterministic).
// 33 <= n <= 64 (config C5) runs the same kernel with 15..36 accumulator tiles per warp (one CTA per SM, up to
// 255 registers; FP64-bound there, 36 DMMAs per k-step at n = 64).
constexpr int kGnWarps = 8;      // per CTA; two CTAs per SM up to four tile columns, one above
constexpr int kGnTailMax = 72;   // tail-column partials: 8 TC dots + self, padded
constexpr int kGnL1Max = 72;     // column l1 partials (<= 64 columns), padded
constexpr int kGnMaxCols = 64;

__host__ __device__ constexpr int gn_tiles(int tc) { return tc * (tc + 1) / 2; }
// k-steps per row group: <= 16 fragment loads in flight per lane (cols = TC + RT)
__host__ __device__ constexpr int gn_unroll(int cols) { return cols >= 5 ? 2 : (cols >= 3 ? 4 : (cols == 2 ? 8 : 16)); }
__host__ __device__ constexpr int gn_partial_stride(int tc) { return gn_tiles(tc) * 64 + kGnTailMax + kGnL1Max; }

template <int TC, int RT>
__global__ void __launch_bounds__(32 * kGnWarps, TC <= 4 ? 2 : 1)
    gram_narrow_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, int n, int64_t rows_per_cta,
                       double* __restrict__ partial) {
  constexpr int NT = gn_tiles(TC);
  constexpr int U = gn_unroll(TC + RT);
  constexpr int PS = gn_partial_stride(TC);
  __shared__ double sred[PS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kr = lane & 3, cj = lane >> 2;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min64(m, r0 + rows_per_cta);
  const int ct = 8 * TC;  // tail column (RT = 1)
  bool colok[TC];
#pragma unroll
  for (int T = 0; T < TC; ++T) colok[T] = 8 * T + cj < (RT ? ct : n);

  double acc[NT][2];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = 0.0;
  double sa[TC], tacc[TC];
#pragma unroll
  for (int T = 0; T < TC; ++T) sa[T] = tacc[T] = 0.0;
  double tself = 0.0, tl1 = 0.0;

  double cur[U][TC + RT], nxt[U][TC + RT];
  auto load = [&](double (&f)[U][TC + RT], int64_t g0) {  // rows g0 .. g0 + 4U of the CTA's range
    const double* p = x + (g0 + kr) * ldx + cj;
    if (g0 + 4 * U <= r1) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
#pragma unroll
        for (int T = 0; T < TC; ++T) f[u][T] = colok[T] ? __ldg(p + 8 * T) : 0.0;
        if (RT) f[u][TC] = __ldg(p + ct - cj);
        p += 4 * ldx;
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool rok = g0 + 4 * u + kr < r1;
#pragma unroll
        for (int T = 0; T < TC; ++T) f[u][T] = (rok && colok[T]) ? __ldg(p + 8 * T) : 0.0;
        if (RT) f[u][TC] = rok ? __ldg(p + ct - cj) : 0.0;
        p += 4 * ldx;
      }
    }
  };
  const int64_t gstep = (int64_t)4 * U * kGnWarps;
  int64_t g0 = r0 + (int64_t)4 * U * warp;
  if (g0 < r1) load(cur, g0);
  while (g0 < r1) {
    const int64_t gn = g0 + gstep;
    if (gn < r1) load(nxt, gn);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int t = 0;
#pragma unroll
      for (int I = 0; I < TC; ++I)
#pragma unroll
        for (int J = I; J < TC; ++J) {
          dmma(acc[t][0], acc[t][1], cur[u][I], cur[u][J]);
          ++t;
        }
#pragma unroll
      for (int T = 0; T < TC; ++T) sa[T] += fabs(cur[u][T]);
      if (RT) {
        const double xt = cur[u][TC];
#pragma unroll
        for (int T = 0; T < TC; ++T) tacc[T] = fma(cur[u][T], xt, tacc[T]);
        tself = fma(xt, xt, tself);
        tl1 += fabs(xt);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int T = 0; T < TC + RT; ++T) cur[u][T] = nxt[u][T];
    g0 = gn;
  }
  // sums over the four k-rows of a lane group (fixed order)
#pragma unroll
  for (int T = 0; T < TC; ++T) {
    sa[T] += __shfl_xor_sync(0xffffffffu, sa[T], 1);
    sa[T] += __shfl_xor_sync(0xffffffffu, sa[T], 2);
    if (RT) {
      tacc[T] += __shfl_xor_sync(0xffffffffu, tacc[T], 1);
      tacc[T] += __shfl_xor_sync(0xffffffffu, tacc[T], 2);
    }
  }
  if (RT) {
    tself += __shfl_xor_sync(0xffffffffu, tself, 1);
    tself += __shfl_xor_sync(0xffffffffu, tself, 2);
    tl1 += __shfl_xor_sync(0xffffffffu, tl1, 1);
    tl1 += __shfl_xor_sync(0xffffffffu, tl1, 2);
  }
  // warp partials -> CTA partial, in warp order
  for (int i = tid; i < PS; i += 32 * kGnWarps) sred[i] = 0.0;
  __syncthreads();
  for (int w = 0; w < kGnWarps; ++w) {
    if (warp == w) {
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        sred[t * 64 + 2 * lane] += acc[t][0];
        sred[t * 64 + 2 * lane + 1] += acc[t][1];
      }
      if (kr == 0) {
#pragma unroll
        for (int T = 0; T < TC; ++T) {
          sred[NT * 64 + kGnTailMax + 8 * T + cj] += sa[T];
          if (RT) sred[NT * 64 + 8 * T + cj] += tacc[T];
        }
      }
      if (RT && lane == 0) {
        sred[NT * 64 + ct] += tself;
        sred[NT * 64 + kGnTailMax + ct] += tl1;
      }
    }
    __syncthreads();
  }
  double* dst = partial + (int64_t)blockIdx.x * PS;
  for (int i = tid; i < PS; i += 32 * kGnWarps) dst[i] = sred[i];
}

// G(i, j), i <= j, summed over the CTA partials in CTA order; mirrored; sumsq = diag; l1.
__global__ void gram_narrow_reduce_kernel(const double* __restrict__ partial, int ctas, int tc, int rt, int n,
                                          double* __restrict__ out, int64_t ldg, double* __restrict__ l1,
                                          double* __restrict__ sumsq) {
  const int nt = gn_tiles(tc), ps = gn_partial_stride(tc), ct = 8 * tc;
  const int i = blockIdx.x;
  for (int j = i + threadIdx.x; j <= n; j += blockDim.x) {
    int off;
    if (j == n) {  // column l1 of column i
      if (!l1) continue;
      off = nt * 64 + kGnTailMax + i;
    } else if (rt && j == ct) {
      off = nt * 64 + i;  // i < ct: dot with the tail column; i == ct: its own square sum
    } else {
      const int I = i >> 3, J = j >> 3;
      off = (I * tc - I * (I - 1) / 2 + (J - I)) * 64 + (i & 7) * 8 + (j & 7);
    }
    double acc = 0.0;
    for (int c = 0; c < ctas; ++c) acc += partial[(int64_t)c * ps + off];
    if (j == n) {
      l1[i] = acc;
    } else {
      out[(int64_t)i * ldg + j] = acc;
      out[(int64_t)j * ldg + i] = acc;
      if (i == j && sumsq) sumsq[i] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// Cyclic register Gram for TC = W RPW + 1 tile columns with W warps per CTA (W = 12, RPW = 2: config C2,
// n = 193..200, 25 tile columns).  With an odd number of tile columns every unordered pair {I, J} is covered
// exactly once by the tiles (I, (I + d) mod TC), d = 0..(TC - 1) / 2, so the upper triangle is TC "tile
// rows" of D = (TC + 1) / 2 tiles each and no tile is computed twice.  Warp w owns tile rows RPW w .. RPW w +
// RPW - 1: its accumulators (RPW D tiles) stay in registers for the whole pass, its operands are the
// RPW + D - 1 fragments of tile columns RPW w .. (mod TC), loaded straight from global memory (all warps of
// the CTA walk the same rows, so after the first toucher they are L1 / L2 hits; an L2 prefetch runs kGcAhead
// k-steps ahead), A = f[r], B = f[r + d]: static register indices.  The leftover tile row TC - 1 is shared
// out: warps 0 .. W/2 - 1 take RPW of its tiles each (one more fragment, tile column TC - 1), warp W/2's
// extra slot holds the last diagonal tile; the other warps' extra slots repeat it (uniform code: every warp
// issues RPW (D + 1) DMMAs per k-step for RPW + D loads).  DMMA slots per k-step at n = 200: 336 for 314
// useful (93%; the staged kernel's 16 x 16 super-tiles: 384).
#ifndef TSNMF_GC_L1PF
#define TSNMF_GC_L1PF 0  // L1 prefetch of the next k-step's lines: 8 warps 1157 -> 1094 GB/s, 12 warps 974 -> 1075 (off)
#endif
constexpr int kGcAhead = 8;  // L2 prefetch distance in k-steps (4 rows each)

template <int W, int RPW>
struct GcShape {
  static constexpr int TC = W * RPW + 1;
  static constexpr int D = (TC + 1) / 2;
  static constexpr int NF = RPW + D - 1;        // fragments of the warp's own tile rows
  static constexpr int NT = RPW * D + RPW;      // accumulator tiles per warp (own rows + extra slots)
  static constexpr int PS = W * NT * 64 + 8 * TC;  // per-CTA partial: tiles, then column l1
};

template <int W, int RPW, bool kFullCols>
__global__ void __launch_bounds__(32 * W, 1)
    gram_cyclic_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, int n, int64_t rows_per_cta,
                       double* __restrict__ partial) {
  using S = GcShape<W, RPW>;
  constexpr int TC = S::TC, D = S::D, NF = S::NF;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kr = lane & 3, cj = lane >> 2;
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t r1 = min64(m, r0 + rows_per_cta);
  // fragment q <-> tile column (RPW warp + q) mod TC; fragment NF <-> tile column TC - 1.  Addressed from one
  // running row pointer p (this lane's row of the k-step, at the warp's first tile column): p[off(q)]
  const int qwrap = TC - RPW * warp;  // fragments q >= qwrap wrap around to tile column q - qwrap
  auto off = [&](int q) { return q == NF ? 8 * (qwrap - 1) : (q < qwrap ? 8 * q : 8 * (q - TC)); };
  auto colok = [&](int q) { return kFullCols || 8 * RPW * warp + cj + off(q) < n; };
  const bool low = warp < W / 2;  // extra slots: (TC - 1, RPW warp + e) for the low warps, the last diagonal tile otherwise
  double acc[RPW][D][2], ext[RPW][2];
#pragma unroll
  for (int r = 0; r < RPW; ++r) {
    ext[r][0] = ext[r][1] = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) acc[r][d][0] = acc[r][d][1] = 0.0;
  }
  double sa[RPW + 1];
#pragma unroll
  for (int r = 0; r <= RPW; ++r) sa[r] = 0.0;
  // L2 prefetch: 4 rows x ceil(8 n / 128) lines per k-step, kGcAhead k-steps ahead
  const int lines = (8 * n + 127) / 128 + 1;
  const int pf_row = tid / lines, pf_line = tid - pf_row * lines;
  const bool pf_on = pf_row < 4 && 128 * pf_line < 8 * n;
  const char* pf = reinterpret_cast<const char*>(x + (r0 + 4 * kGcAhead + pf_row) * ldx) + 128 * pf_line;
  int64_t pf_left = r1 - (r0 + 4 * kGcAhead + pf_row);  // rows from the prefetched row to the end of the range

  const double* p = x + (r0 + kr) * ldx + 8 * RPW * warp + cj;
  const int64_t pstep = 4 * ldx;
  // all loads of a k-step, then all its DMMAs (loads reissued one by one behind the DMMAs that free their
  // registers measured slower, 1019 vs 1106 GB/s with 8 warps: the partner warps' turns hide the wait)
  auto kstep = [&](const double (&f)[NF + 1]) {
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
      for (int d = 0; d < D; ++d) dmma(acc[r][d][0], acc[r][d][1], f[r], f[r + d]);
#pragma unroll
    for (int e = 0; e < RPW; ++e) {
      const double b = low ? f[e] : f[NF];
      dmma(ext[e][0], ext[e][1], f[NF], b);
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r) sa[r] += fabs(f[r]);
    sa[RPW] += fabs(f[NF]);
  };
  int64_t g0 = r0;
  for (; g0 + 4 <= r1; g0 += 4) {
    if (pf_on && pf_left > 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
    pf += 32 * ldx;
    pf_left -= 4;
    double f[NF + 1];
#pragma unroll
    for (int q = 0; q <= NF; ++q) f[q] = colok(q) ? __ldg(p + off(q)) : 0.0;
    p += pstep;
#if TSNMF_GC_L1PF
    if (g0 + 8 <= r1) {
#pragma unroll
      for (int q = 0; q <= NF; ++q)
        if (colok(q)) asm volatile("prefetch.global.L1 [%0];" ::"l"(p + off(q)));
    }
#endif
    kstep(f);
  }
  if (g0 < r1) {  // last, partial k-step of the range
    const bool rok = g0 + kr < r1;
    double f[NF + 1];
#pragma unroll
    for (int q = 0; q <= NF; ++q) f[q] = (rok && colok(q)) ? __ldg(p + off(q)) : 0.0;
    kstep(f);
  }
  double* dst = partial + (int64_t)blockIdx.x * S::PS + (int64_t)warp * S::NT * 64;
#pragma unroll
  for (int r = 0; r < RPW; ++r)
#pragma unroll
    for (int d = 0; d < D; ++d)
      *reinterpret_cast<double2*>(dst + (r * D + d) * 64 + 2 * lane) = make_double2(acc[r][d][0], acc[r][d][1]);
#pragma unroll
  for (int e = 0; e < RPW; ++e)
    *reinterpret_cast<double2*>(dst + (RPW * D + e) * 64 + 2 * lane) = make_double2(ext[e][0], ext[e][1]);
  // column l1: sum over the four k-rows of a lane group; warp w owns tile columns RPW w .. + RPW - 1, warp 0
  // also the last one
  double* l1dst = partial + (int64_t)blockIdx.x * S::PS + (int64_t)W * S::NT * 64;
#pragma unroll
  for (int r = 0; r <= RPW; ++r) {
    sa[r] += __shfl_xor_sync(0xffffffffu, sa[r], 1);
    sa[r] += __shfl_xor_sync(0xffffffffu, sa[r], 2);
    if (kr == 0 && (r < RPW || warp == 0)) l1dst[8 * (r < RPW ? RPW * warp + r : TC - 1) + cj] = sa[r];
  }
}

// G(i, j), i <= j, from the owner's tile (see gram_cyclic_kernel), summed over the CTA partials in CTA order
template <int W, int RPW>
__global__ void gram_cyclic_reduce_kernel(const double* __restrict__ partial, int ctas, int n,
                                          double* __restrict__ out, int64_t ldg, double* __restrict__ l1,
                                          double* __restrict__ sumsq) {
  using S = GcShape<W, RPW>;
  constexpr int TC = S::TC, D = S::D;
  const int i = blockIdx.x;
  for (int j = i + threadIdx.x; j <= n; j += blockDim.x) {
    int off;
    if (j == n) {
      if (!l1) continue;
      off = W * S::NT * 64 + i;
    } else {
      const int ti = i >> 3, tj = j >> 3, d = tj - ti;
      int w, slot, er, ec;  // owner warp, tile slot, element (row, col)
      if (ti == TC - 1) {  // last diagonal tile: warp W/2's extra slot 0
        w = W / 2, slot = RPW * D, er = i & 7, ec = j & 7;
      } else if (d < D) {  // tile (ti, tj) in tile row ti
        w = ti / RPW, slot = (ti % RPW) * D + d, er = i & 7, ec = j & 7;
      } else if (tj == TC - 1) {  // tile (TC - 1, ti) of the leftover row: warp ti / RPW's extra slot
        w = ti / RPW, slot = RPW * D + ti % RPW, er = j & 7, ec = i & 7;
      } else {  // tile (tj, ti) in tile row tj (wrapped), transposed
        w = tj / RPW, slot = (tj % RPW) * D + (TC - d), er = j & 7, ec = i & 7;
      }
      off = (w * S::NT + slot) * 64 + er * 8 + ec;
    }
    double acc = 0.0;
    for (int c = 0; c < ctas; ++c) acc += partial[(int64_t)c * S::PS + off];
    if (j == n) {
      l1[i] = acc;
    } else {
      out[(int64_t)i * ldg + j] = acc;
      out[(int64_t)j * ldg + i] = acc;
      if (i == j && sumsq) sumsq[i] = acc;
    }
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

// Narrow path (n <= 64): TSNMF_GRAM_NARROW=0 selects the staged kernel, TSNMF_GRAM_TAIL=0 pads a width of
// the form 8 TC + 1 to another tile column instead of the FMA tail.
bool gn_path(int n) {
  if (n > kGnMaxCols) return false;
  if (const char* e = getenv("TSNMF_GRAM_NARROW")) return atoi(e) != 0;
  return true;
}
struct GnPlan {
  int tc, rt, ctas;
  int64_t rpc;
};
GnPlan gn_plan(int64_t m, int n, int sms) {
  GnPlan p;
  p.rt = (n == 17 || n == 25) ? 1 : 0;  // measured: n = 25 6113 vs 4353 GB/s padded, n = 17 5924 vs 5109; n = 9 loses (4411 vs 5178)
  if (const char* e = getenv("TSNMF_GRAM_TAIL")) p.rt = p.rt && atoi(e) != 0;
  p.tc = p.rt ? n / 8 : (int)ceil_div(n, 8);
  const int64_t grp = 4 * gn_unroll(p.tc + p.rt);
  const int64_t ctas = max64(1, min64((int64_t)(p.tc <= 4 ? 2 : 1) * sms, ceil_div(m, grp * kGnWarps)));
  p.rpc = round_up(ceil_div(m, ctas), grp);
  p.ctas = (int)max64(1, ceil_div(m, p.rpc));
  return p;
}
size_t gn_ws_doubles(const GnPlan& p) { return (size_t)p.ctas * gn_partial_stride(p.tc); }

template <int TC, int RT>
int gn_launch(const double* x, int64_t m, int64_t ldx, int n, const GnPlan& p, double* partial, cudaStream_t st) {
  gram_narrow_kernel<TC, RT><<<p.ctas, 32 * kGnWarps, 0, st>>>(x, m, ldx, n, p.rpc, partial);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

int gn_run(const double* x, int64_t m, int n, int64_t ldx, double* gout, int64_t ldg, double* l1, double* sumsq,
           void* ws, size_t ws_bytes, cudaStream_t st) {
  const GnPlan p = gn_plan(m, n, sm_count());
  const size_t need = sizeof(double) * gn_ws_doubles(p);
  if (ws_bytes < need) return set_error(kUsage, "gram: workspace too small (%zu < %zu bytes)", ws_bytes, need);
  double* partial = reinterpret_cast<double*>(ws);
  prof_mark(kProfGram, true, st);
  int rc;
  switch (p.tc * 2 + p.rt) {
    case 2: rc = gn_launch<1, 0>(x, m, ldx, n, p, partial, st); break;
    case 3: rc = gn_launch<1, 1>(x, m, ldx, n, p, partial, st); break;
    case 4: rc = gn_launch<2, 0>(x, m, ldx, n, p, partial, st); break;
    case 5: rc = gn_launch<2, 1>(x, m, ldx, n, p, partial, st); break;
    case 6: rc = gn_launch<3, 0>(x, m, ldx, n, p, partial, st); break;
    case 7: rc = gn_launch<3, 1>(x, m, ldx, n, p, partial, st); break;
    case 8: rc = gn_launch<4, 0>(x, m, ldx, n, p, partial, st); break;
    case 10: rc = gn_launch<5, 0>(x, m, ldx, n, p, partial, st); break;
    case 12: rc = gn_launch<6, 0>(x, m, ldx, n, p, partial, st); break;
    case 14: rc = gn_launch<7, 0>(x, m, ldx, n, p, partial, st); break;
    default: rc = gn_launch<8, 0>(x, m, ldx, n, p, partial, st); break;
  }
  if (rc) return rc;
  prof_mark(kProfGram, false, st);
  gram_narrow_reduce_kernel<<<n, 64, 0, st>>>(partial, p.ctas, p.tc, p.rt, n, gout, ldg, l1, sumsq);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

// Cyclic register Gram: n = 193..200 (25 tile columns); TSNMF_GRAM_CYCLIC=0 selects the staged kernel.
bool gc_path(int n) {
  if (n <= 192 || n > 200) return false;
  if (const char* e = getenv("TSNMF_GRAM_CYCLIC")) return atoi(e) != 0;
  return true;
}
struct GcPlan {
  int ctas;
  int64_t rpc;
};
GcPlan gc_plan(int64_t m, int sms) {
  GcPlan p;
  const int64_t ctas = max64(1, min64(sms, ceil_div(m, 256)));
  p.rpc = round_up(ceil_div(m, ctas), 4);
  p.ctas = (int)max64(1, ceil_div(m, p.rpc));
  return p;
}
template <int W, int RPW>
int gc_launch(const double* x, int64_t m, int n, int64_t ldx, double* gout, int64_t ldg, double* l1, double* sumsq,
              void* ws, size_t ws_bytes, cudaStream_t st) {
  using S = GcShape<W, RPW>;
  const GcPlan p = gc_plan(m, sm_count());
  const size_t need = sizeof(double) * (size_t)p.ctas * S::PS;
  if (ws_bytes < need) return set_error(kUsage, "gram: workspace too small (%zu < %zu bytes)", ws_bytes, need);
  double* partial = reinterpret_cast<double*>(ws);
  prof_mark(kProfGram, true, st);
  if (n == 8 * S::TC)
    gram_cyclic_kernel<W, RPW, true><<<p.ctas, 32 * W, 0, st>>>(x, m, ldx, n, p.rpc, partial);
  else
    gram_cyclic_kernel<W, RPW, false><<<p.ctas, 32 * W, 0, st>>>(x, m, ldx, n, p.rpc, partial);
  TSNMF_LAUNCH_CHECK();
  prof_mark(kProfGram, false, st);
  gram_cyclic_reduce_kernel<W, RPW><<<n, 128, 0, st>>>(partial, p.ctas, n, gout, ldg, l1, sumsq);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}
// 25 tile columns: 8 warps x 3 tile rows at n = 200 (no column predicates; 1161 vs 974 GB/s with 12 warps), 12
// warps x 2 tile rows for the ragged widths 193..199 (996 vs 882 GB/s); TSNMF_GRAM_CYCLIC=8 / 12 forces one.
bool gc_eight(int n) {
  if (const char* e = getenv("TSNMF_GRAM_CYCLIC")) {
    if (atoi(e) == 8) return true;
    if (atoi(e) == 12) return false;
  }
  return n == 200;
}
size_t gc_ws_doubles(int64_t m, int n) {
  return (size_t)gc_plan(m, sm_count()).ctas * (gc_eight(n) ? GcShape<8, 3>::PS : GcShape<12, 2>::PS);
}
int gc_run(const double* x, int64_t m, int n, int64_t ldx, double* gout, int64_t ldg, double* l1, double* sumsq,
           void* ws, size_t ws_bytes, cudaStream_t st) {
  if (gc_eight(n)) return gc_launch<8, 3>(x, m, n, ldx, gout, ldg, l1, sumsq, ws, ws_bytes, st);
  return gc_launch<12, 2>(x, m, n, ldx, gout, ldg, l1, sumsq, ws, ws_bytes, st);
}

}  // namespace

int gram_max_cols() { return 512; }

size_t gram_workspace_bytes(int64_t m, int n) {
  if (n < 1 || n > gram_max_cols()) return 0;
  if (gn_path(n)) return sizeof(double) * gn_ws_doubles(gn_plan(max64(m, 1), n, sm_count())) + 256;
  if (gc_path(n)) return sizeof(double) * gc_ws_doubles(max64(m, 1), n) + 256;
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
  if (gn_path(n)) return gn_run(x, m, n, ldx, gout, ldg, l1, sumsq, ws, ws_bytes, st);
  if (gc_path(n)) return gc_run(x, m, n, ldx, gout, ldg, l1, sumsq, ws, ws_bytes, st);
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

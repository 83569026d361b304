// TSQR: one pass over a resident row block -> sign-fixed n x n R (+ fused column l1 / sum of squares).
//
// Replaces the reference's per-chunk LAPACK path:
//   factor_chunk  reference pkg/src/tsnmf/tsqr.py:129-141   (np.linalg.qr -> dgeqrf, _fix_signs)
//   combine       reference pkg/src/tsnmf/tsqr.py:144-153   (QR of the stacked pair)
//   _StatsAcc     reference pkg/src/tsnmf/tsqr.py:184-198   (fused l1 / sum of squares)
//   TreeReducer   reference pkg/src/tsnmf/tsqr.py:201-234   (binary-counter combine order)
//
// Leaf: each CTA owns a contiguous row range and an R slot (npad x npad, row-major, L2-resident in the
// caller's workspace).  It streams row blocks B (brows x npad) into shared memory and folds each block
// into R with a structured blocked Householder QR of [R; B]: the reflector for column j is
// u = [e_j; v] (R part is a unit vector), so only R row j and the block are touched.  Panels of NB = 8
// columns are factored by one register-resident panel warp with lazy trailing updates (no CTA barrier
// per column); the next panel's columns get the lookahead update from the panel warp + helper pair and
// the rest of the trailing matrix the compact-WY update  W = R_p + V^T B,  W <- T^T W,  R_p -= W,
// B -= V W  by six GEMM warps on FP64 tensor cores (mma.sync m8n8k4 f64 = DMMA), overlapped with the
// next panel.  Narrow matrices (n <= 32) use the register-block warp leaf instead (tsqr_warp_leaf_kernel:
// one Householder chain per warp over 32*S-row blocks held in registers; the older 32-row
// tsqr_small_leaf_kernel stays selectable and is the narrow combine).  Leaves are then combined in the
// reference TreeReducer order (perfect binary levels over the leaf index, then a fold of the leftover
// subtrees), each combine being the same structured QR with the second factor's rows as data
// (triangular: panels left of the block are skipped).
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace tsnmf {

constexpr int kTqThreads = 256;
constexpr int kTqWarps = kTqThreads / 32;
constexpr int kNB = 8;       // panel width (reflectors per compact-WY block)
constexpr int kMaxRq = 5;    // block rows per lane of each panel warp (block rows <= 160)

struct TqGeom {
  int n;      // data columns
  int npad;   // padded columns (multiple of 8); R slots are npad x npad
  int lds;    // shared-memory row stride of the block (% 16 == 8)
  int brows;  // rows per block (multiple of 8, <= 32 * kMaxRq)
};

struct TqLayout {
  // offsets in doubles from the dynamic smem base
  __host__ __device__ static int rd(const TqGeom& g) { return g.brows * g.lds; }            // 2 x 8x8 R diag blocks
  __host__ __device__ static int tm(const TqGeom& g) { return rd(g) + 2 * kNB * kNB; }      // 2 x 8x8 T
  __host__ __device__ static int red(const TqGeom& g) { return tm(g) + 2 * kNB * kNB; }    // 32 x 9 partials
  __host__ __device__ static int wsc(const TqGeom& g) { return red(g) + 32 * 9; }           // per-warp 8x8 scratch
  __host__ __device__ static int wpart(const TqGeom& g) { return wsc(g) + kTqWarps * kNB * 8; }  // partial W tiles
  __host__ __device__ static int total(const TqGeom& g) { return wpart(g) + 2 * 64; }  // pair-lookahead partials
  static size_t bytes(const TqGeom& g) { return sizeof(double) * (size_t)total(g); }
};

// Shared-memory swizzle of the block: column c of row r lives at r*lds + (c ^ swz(r)).  With
// lds % 16 == 8 this makes every DMMA fragment access conflict-free: the 4x8 operand slabs (lane:
// row l%4, col l/4), the V fragments (row l/4, col l%4) and the 16-byte C-tile rows (row l/4,
// col 2*(l%4)).  XOR by 0 or 4 permutes inside aligned 8-column groups, so 16-byte pairs stay intact.
__device__ __forceinline__ int swz(int row) { return (row & 2) << 1; }

// Named barriers between the panel warp (warp 0) and the GEMM warps (1..7).
// Warp roles: warps 0 and 4 (both on SMSP 0) = panel warps, so SMSP 0 runs the panel's latency-bound
// FP64 chain without DMMA traffic; warps 1,2,3,5,6,7 = GEMM warps (GEMM warp 0 also stages R rows).
constexpr int kBarColsReady = 1;  // next panel's columns updated + its R rows staged  (GEMM, helper -> panel)
constexpr int kBarPanelDone = 2;  // V, T of the current panel published               (panel -> GEMM, helper)
constexpr int kBarPanelPair = 4;  // panel warp + helper (pair lookahead partials)
// Lookahead tile ready (64 threads): the panel warp starts its half of the pair lookahead of panel p on tile
// p + 1 right after publishing panel p, i.e. possibly while the GEMM warps still run iteration p - 1, whose
// update of tile p + 1 by panel p - 1 it must see.  The GEMM warp that applies that update arrives here
// after it; the panel warp syncs before the lookahead.  (Without it the order held only by timing.)
constexpr int kBarNextReady = 5;
constexpr int kGemmWarps = 6;
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
// trace builds: force a deferred-blocking barrier to resolve before the next trace point
#ifdef TSNMF_TRACE
#define TQ_RESOLVE(smem_ptr) (void)(*(volatile double*)(smem_ptr))
#else
#define TQ_RESOLVE(smem_ptr) \
  do {                       \
  } while (0)
#endif
__device__ __forceinline__ int gemm_index(int warp) { return warp < 4 ? warp - 1 : warp - 2; }  // 0..5

#ifdef TSNMF_TRACE
// CTA 0, first row block only: g_trace[warp][panel * 64 + tag] = clock64() (fire-and-forget stores)
__device__ long long g_trace[8][64 * 64];
#define TQ_TRACE(tag)                                                                  \
  do {                                                                                 \
    if (tq_p >= 0 && blockIdx.x == 0 && (threadIdx.x & 31) == 0)                       \
      g_trace[threadIdx.x >> 5][tq_p * 64 + (tag)] = clock64();                        \
  } while (0)
#else
#define TQ_TRACE(tag) \
  do {                \
    (void)tq_p;       \
  } while (0)
#endif

#ifndef TSNMF_PAIR_LOOKAHEAD
#define TSNMF_PAIR_LOOKAHEAD 1
#endif
constexpr bool kPairLookahead = TSNMF_PAIR_LOOKAHEAD != 0;  // panel warp joins the helper's lookahead

__host__ __device__ constexpr int pow2ceil(int v) {  // v <= 32
  return v <= 1 ? 1 : (v <= 2 ? 2 : (v <= 4 ? 4 : (v <= 8 ? 8 : (v <= 16 ? 16 : 32))));
}


// Branchy variants (range test beside the Newton chain, IEEE path almost never taken): fewer instructions
// and registers than the branch-free ones, which the register-capped two-CTA panel build prefers.
__device__ __forceinline__ double fast_rsqrt(double a) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  const double h = 0.5 * a;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  if (!(a > 0x1p-900 && a < 0x1p+900)) y = rsqrt(a);
  return y;
}
__device__ __forceinline__ double fast_rcp(double a) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(a));
  y = y * fma(-a, y, 2.0);
  y = y * fma(-a, y, 2.0);
  if (!(a > 0x1p-900 && a < 0x1p+900)) y = __drcp_rn(a);
  return y;
}

// bj0: shared-memory column of the panel (== j0 except in the split leaf, whose tiles live in slots)
template <int RQ, bool kPreload>
__device__ __forceinline__ void panel_factor_lazy(double* __restrict__ Bs, int lds, int brows, int j0, int bj0,
                                                  double* __restrict__ R, int npad, const double* __restrict__ Rd,
                                                  double* __restrict__ Tm, double* __restrict__ red, int lane,
                                                  int tq_p) {
  const int sw = swz(lane);
  double x[RQ][kNB];
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int rl = lane + 32 * q;
    const double* rp = Bs + rl * lds + bj0;
#pragma unroll
    for (int c = 0; c < kNB; c += 2) {
      double2 v = make_double2(0.0, 0.0);
      if (rl < brows) v = *reinterpret_cast<const double2*>(rp + (c ^ sw));
      x[q][c] = v.x;
      x[q][c + 1] = v.y;
    }
  }
  double trow[kNB], rmine[kNB], f[kNB];
#pragma unroll
  for (int c = 0; c < kNB; ++c) trow[c] = rmine[c] = f[c] = 0.0;
  // R(j, j) and R(j, j+1) are not touched by the panel's earlier reflectors (reflector i only changes
  // R row i), so the diagonal and first off-diagonal are loaded up front, off the per-column chain
  // (kPreload false: the register-capped two-CTAs-per-SM build reads them when needed instead)
  double ralpha[kNB], rnext[kNB];
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    ralpha[c] = kPreload ? Rd[c * kNB + c] : 0.0;
    rnext[c] = (kPreload && c + 1 < kNB) ? Rd[c * kNB + c + 1] : 0.0;
  }
  const int rc = lane & 7, rq = lane >> 3;
  double scale_prev = 0.0;
  // dots of step 0
#pragma unroll
  for (int c = 0; c < kNB; ++c) {
    double acc = 0.0;
#pragma unroll
    for (int q = 0; q < RQ; ++q) acc = fma(x[q][0], x[q][c], acc);
    red[lane * 9 + c] = acc;
  }
#pragma unroll
  for (int js = 0; js < kNB; ++js) {
    TQ_TRACE(10 + js);
    // (A) warp reduction of this step's dots
    __syncwarp();
    const double s0 = red[(rq * 8 + 0) * 9 + rc] + red[(rq * 8 + 1) * 9 + rc];
    const double s1 = red[(rq * 8 + 2) * 9 + rc] + red[(rq * 8 + 3) * 9 + rc];
    const double s2 = red[(rq * 8 + 4) * 9 + rc] + red[(rq * 8 + 5) * 9 + rc];
    const double s3 = red[(rq * 8 + 6) * 9 + rc] + red[(rq * 8 + 7) * 9 + rc];
    double tot = (s0 + s1) + (s2 + s3);
    tot += __shfl_xor_sync(0xffffffffu, tot, 8);
    tot += __shfl_xor_sync(0xffffffffu, tot, 16);
    double d[kNB];
#pragma unroll
    for (int c = 0; c < kNB; ++c) d[c] = __shfl_sync(0xffffffffu, tot, c);
    __syncwarp();  // red free for the next step's dots
    TQ_TRACE(30 + js);
    // (B) corrections for the lazily updated trailing columns; T dot of the previous pivot
    if (js > 0) {
#pragma unroll
      for (int c = js + 1; c < kNB; ++c) d[c] = fma(-f[c], d[js - 1], d[c]);
      d[js - 1] *= scale_prev;
    }
    // (C) reflector scalars
    // (branch-free: the whole column step is one basic block, so the off-chain work of (E) can be
    // scheduled into the latency of this chain)
    // (measured: C2 n=200 228 -> 234 GB/s; the register-capped two-CTA build (kPreload false, n <= 64) is
    // faster with the branch, 352 vs 339 GB/s at n=64)
    const double alpha = kPreload ? ralpha[js] : Rd[js * kNB + js];
    double tau, scale, beta;
    if constexpr (kPreload) {
      const bool live = d[js] > 0.0;
      const double ss = live ? fma(alpha, alpha, d[js]) : 1.0;
      const double inv = rsqrt_nb(ss);
      const double nrm = ss * inv;
      beta = live ? -copysign(nrm, alpha) : alpha;
      tau = live ? fma(fabs(alpha), inv, 1.0) : 0.0;
      scale = live ? copysign(rcp_nb(fabs(alpha) + nrm), alpha) : 0.0;
    } else {
      tau = 0.0;
      scale = 0.0;
      beta = alpha;
      if (d[js] > 0.0) {
        const double ss = fma(alpha, alpha, d[js]);
        const double inv = fast_rsqrt(ss);
        const double nrm = ss * inv;
        beta = -copysign(nrm, alpha);
        tau = fma(fabs(alpha), inv, 1.0);
        scale = copysign(fast_rcp(fabs(alpha) + nrm), alpha);
      }
    }
    // (D) critical: next pivot's factor, eager update of the next pivot column, next step's dots
    if (js + 1 < kNB) {
      const double rjn = kPreload ? rnext[js] : Rd[js * kNB + js + 1];
      const double twn = tau * fma(scale, d[js + 1], rjn);
      f[js + 1] = twn * scale;
      if (lane == js + 1) rmine[js] = rjn - twn;
#pragma unroll
      for (int q = 0; q < RQ; ++q) x[q][js + 1] = fma(-f[js + 1], x[q][js], x[q][js + 1]);
#pragma unroll
      for (int c = 0; c < kNB; ++c) {
        double acc = 0.0;
#pragma unroll
        for (int q = 0; q < RQ; ++q) acc = fma(x[q][js + 1], x[q][c], acc);
        red[lane * 9 + c] = acc;
      }
    }
    // (E) off the critical path: remaining factors, R row, T row, pending trailing updates, u -> v
#pragma unroll
    for (int c = js + 2; c < kNB; ++c) {
      const double rjc = Rd[js * kNB + c];
      const double tw = tau * fma(scale, d[c], rjc);
      f[c] = tw * scale;
      if (lane == c) rmine[js] = rjc - tw;
    }
    if (lane == js) rmine[js] = beta;
    {  // T[r][js] = -tau_js * sum_{q=r}^{js-1} T[r][q] (v_q^T v_js),  v_q^T v_js = scale * d[q]
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < js; ++q) acc = fma(trow[q], d[q], acc);
      trow[js] = (lane == js) ? tau : (lane < js ? -tau * scale * acc : 0.0);
    }
    if (js + 1 < kNB) {
#pragma unroll
      for (int c = js + 2; c < kNB; ++c)
#pragma unroll
        for (int q = 0; q < RQ; ++q) x[q][c] = fma(-f[c], x[q][js], x[q][c]);
    }
#pragma unroll
    for (int q = 0; q < RQ; ++q) x[q][js] *= scale;
    scale_prev = scale;
  }
#pragma unroll
  for (int q = 0; q < RQ; ++q) {
    const int rl = lane + 32 * q;
    if (rl < brows) {
      double* rp = Bs + rl * lds + bj0;
#pragma unroll
      for (int c = 0; c < kNB; c += 2) *reinterpret_cast<double2*>(rp + (c ^ sw)) = make_double2(x[q][c], x[q][c + 1]);
    }
  }
  if (lane < kNB) {
    double* Rcol = R + (int64_t)j0 * npad + j0 + lane;
#pragma unroll
    for (int jj = 0; jj < kNB; ++jj)
      if (jj <= lane) Rcol[(int64_t)jj * npad] = rmine[jj];
#pragma unroll
    for (int c = 0; c < kNB; ++c) Tm[lane * kNB + c] = trow[c];
  }
}

// Stage rows into the swizzled block layout (cp.async); zero-fill padding rows / columns.
// swz(r) == swz_row(r), so this is the shared division-free swizzled staging loop.
__device__ __forceinline__ void stage_block(double* __restrict__ dst, int lds, const double* __restrict__ src,
                                            int64_t ldsrc, int nrows, int ncols, int rows_total, int cols_total,
                                            bool vec16) {
  stage_rows_swz(dst, lds, src, ldsrc, nrows, ncols, rows_total, cols_total, vec16);
}

// Stage the 8x8 diagonal block R(j0:j0+8, j0:j0+8) into shared memory (one warp, cp.async).
__device__ __forceinline__ void stage_rdiag(double* __restrict__ dst, const double* __restrict__ R, int npad, int j0,
                                            int lane) {
  const int r = lane >> 2, c = 2 * (lane & 3);
  cp_async16(dst + r * kNB + c, R + (int64_t)(j0 + r) * npad + j0 + c);
}

// Apply panel (j0)'s block reflector  Q^T = I - V T^T V^T  to column blocks cbs[0..G) of [R; B]:
//   W = R_p(:, cb) + V^T B(:, cb);  W' = T^T W;  R_p(:, cb) -= W';  B(:, cb) -= V W'.
// One warp, no CTA barrier.  The R_p tiles are read from global memory (L2-resident R slot) at the start
// so their latency hides behind the k-loop; R is updated in global memory.
// (vj, pcbs: shared-memory columns of V and of the tiles; j0, cbs: logical, for R)
template <int G>
__device__ __forceinline__ void update_cbs(double* __restrict__ Bs, int lds, int brows, int j0, int vj,
                                           double* __restrict__ R, int npad, const double* __restrict__ Tm,
                                           double* __restrict__ Wsc, const int (&cbs)[G], const int (&pcbs)[G],
                                           int lane, int tq_p) {
  const int frag_col = (lane >> 2) ^ ((lane & 2) << 1);  // slab fragment: row i + l%4, col l/4
  const int vsw = ((lane >> 2) & 2) << 1;                // V / C-tile rows 8rb + l/4
  double acc0[G][2], acc1[G][2], rinit[G][2];
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    const double2 rv = *reinterpret_cast<const double2*>(R + (int64_t)(j0 + (lane >> 2)) * npad + 8 * cbs[gg] +
                                                         2 * (lane & 3));
    rinit[gg][0] = rv.x;
    rinit[gg][1] = rv.y;
    acc0[gg][0] = acc0[gg][1] = acc1[gg][0] = acc1[gg][1] = 0.0;
  }
  TQ_TRACE(20);
  // W = R_p + V^T B: K = brows in steps of 4 rows, two independent accumulator chains
  const double* slab = Bs + (lane & 3) * lds + frag_col;
#pragma unroll 2
  for (int i = 0; i < brows; i += 8) {
    const double* r0 = slab + i * lds;
    const double* r1 = r0 + 4 * lds;
    const double a0 = r0[vj], a1 = r1[vj];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      dmma(acc0[gg][0], acc0[gg][1], a0, r0[pcbs[gg]]);
      dmma(acc1[gg][0], acc1[gg][1], a1, r1[pcbs[gg]]);
    }
  }
  TQ_TRACE(21);
  // W' = T^T W ; R_p -= W' ; gather -W' as B-operand fragments
  double wb[G][2];
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    Wsc[(lane >> 2) * 8 + 2 * (lane & 3)] = (acc0[gg][0] + acc1[gg][0]) + rinit[gg][0];
    Wsc[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = (acc0[gg][1] + acc1[gg][1]) + rinit[gg][1];
    __syncwarp();
    double w0 = 0.0, w1 = 0.0;
#pragma unroll
    for (int k0 = 0; k0 < 8; k0 += 4)
      dmma(w0, w1, Tm[(k0 + (lane & 3)) * kNB + (lane >> 2)], Wsc[(k0 + (lane & 3)) * 8 + (lane >> 2)]);
    double* rp = R + (int64_t)(j0 + (lane >> 2)) * npad + 8 * cbs[gg] + 2 * (lane & 3);
    *reinterpret_cast<double2*>(rp) = make_double2(rinit[gg][0] - w0, rinit[gg][1] - w1);
    __syncwarp();
    Wsc[(lane >> 2) * 8 + 2 * (lane & 3)] = w0;
    Wsc[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = w1;
    __syncwarp();
#pragma unroll
    for (int k4 = 0; k4 < 2; ++k4) wb[gg][k4] = -Wsc[(4 * k4 + (lane & 3)) * 8 + (lane >> 2)];
    __syncwarp();
  }
  TQ_TRACE(22);
  // B -= V W'   (C tiles read/written in place; K = 8), two row blocks per iteration (brows % 16 == 0)
#pragma unroll 1
  for (int rb = 0; rb < brows / 8; rb += 2) {
    double* rowa = Bs + (8 * rb + (lane >> 2)) * lds;
    double* rowb = rowa + 8 * lds;
    const double a0 = rowa[vj + ((lane & 3) ^ vsw)], a1 = rowa[vj + ((4 + (lane & 3)) ^ vsw)];
    const double b0 = rowb[vj + ((lane & 3) ^ vsw)], b1 = rowb[vj + ((4 + (lane & 3)) ^ vsw)];
    double2 ca[G], cb2[G];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      ca[gg] = *reinterpret_cast<const double2*>(rowa + pcbs[gg] + ((2 * (lane & 3)) ^ vsw));
      cb2[gg] = *reinterpret_cast<const double2*>(rowb + pcbs[gg] + ((2 * (lane & 3)) ^ vsw));
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      dmma(ca[gg].x, ca[gg].y, a0, wb[gg][0]);
      dmma(cb2[gg].x, cb2[gg].y, b0, wb[gg][0]);
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      dmma(ca[gg].x, ca[gg].y, a1, wb[gg][1]);
      dmma(cb2[gg].x, cb2[gg].y, b1, wb[gg][1]);
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      *reinterpret_cast<double2*>(rowa + pcbs[gg] + ((2 * (lane & 3)) ^ vsw)) = ca[gg];
      *reinterpret_cast<double2*>(rowb + pcbs[gg] + ((2 * (lane & 3)) ^ vsw)) = cb2[gg];
    }
  }
  TQ_TRACE(23);
}


// Single-warp lookahead (helper warp): panel (j0)'s block reflector applied to ONE column block cb, with
// 4 independent DMMA accumulator chains in W = R_p + V^T B and 4 independent C tiles per iteration in
// B -= V W' (brows % 16 == 0; the 4-tile loop handles the remainder in pairs).
__device__ __forceinline__ void lookahead_single(double* __restrict__ Bs, int lds, int brows, int j0,
                                                 double* __restrict__ R, int npad, const double* __restrict__ Tm,
                                                 double* __restrict__ Wsc, int cb, int lane) {
  const int frag_col = (lane >> 2) ^ ((lane & 2) << 1);
  const int vsw = ((lane >> 2) & 2) << 1;
  double* rtile = R + (int64_t)(j0 + (lane >> 2)) * npad + 8 * cb + 2 * (lane & 3);
  const double2 rinit = *reinterpret_cast<const double2*>(rtile);
  double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  const double* slab = Bs + (lane & 3) * lds + frag_col;
  int i = 0;
#pragma unroll 1
  for (; i + 16 <= brows; i += 16) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double* r = slab + (i + 4 * u) * lds;
      a[u] = r[j0];
      b[u] = r[8 * cb];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(c[u][0], c[u][1], a[u], b[u]);
  }
  for (; i < brows; i += 4) {  // tail (not taken when brows % 16 == 0)
    const double* r = slab + i * lds;
    dmma(c[0][0], c[0][1], r[j0], r[8 * cb]);
  }
  Wsc[(lane >> 2) * 8 + 2 * (lane & 3)] = ((c[0][0] + c[1][0]) + (c[2][0] + c[3][0])) + rinit.x;
  Wsc[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = ((c[0][1] + c[1][1]) + (c[2][1] + c[3][1])) + rinit.y;
  __syncwarp();
  double w0 = 0.0, w1 = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4)
    dmma(w0, w1, Tm[(k0 + (lane & 3)) * kNB + (lane >> 2)], Wsc[(k0 + (lane & 3)) * 8 + (lane >> 2)]);
  *reinterpret_cast<double2*>(rtile) = make_double2(rinit.x - w0, rinit.y - w1);
  __syncwarp();
  Wsc[(lane >> 2) * 8 + 2 * (lane & 3)] = w0;
  Wsc[(lane >> 2) * 8 + 2 * (lane & 3) + 1] = w1;
  __syncwarp();
  const double wb0 = -Wsc[(lane & 3) * 8 + (lane >> 2)];
  const double wb1 = -Wsc[(4 + (lane & 3)) * 8 + (lane >> 2)];
  __syncwarp();
  const int nrb = brows / 8;
  int rb = 0;
#pragma unroll 1
  for (; rb + 4 <= nrb; rb += 4) {
    double* rows[4];
    double2 cv[4];
    double va[4], vb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      rows[u] = Bs + (8 * (rb + u) + (lane >> 2)) * lds;
      va[u] = rows[u][j0 + ((lane & 3) ^ vsw)];
      vb[u] = rows[u][j0 + ((4 + (lane & 3)) ^ vsw)];
      cv[u] = *reinterpret_cast<const double2*>(rows[u] + 8 * cb + ((2 * (lane & 3)) ^ vsw));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(cv[u].x, cv[u].y, va[u], wb0);
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(cv[u].x, cv[u].y, vb[u], wb1);
#pragma unroll
    for (int u = 0; u < 4; ++u) *reinterpret_cast<double2*>(rows[u] + 8 * cb + ((2 * (lane & 3)) ^ vsw)) = cv[u];
  }
  for (; rb < nrb; ++rb) {
    double* row = Bs + (8 * rb + (lane >> 2)) * lds;
    double2 cv = *reinterpret_cast<const double2*>(row + 8 * cb + ((2 * (lane & 3)) ^ vsw));
    dmma(cv.x, cv.y, row[j0 + ((lane & 3) ^ vsw)], wb0);
    dmma(cv.x, cv.y, row[j0 + ((4 + (lane & 3)) ^ vsw)], wb1);
    *reinterpret_cast<double2*>(row + 8 * cb + ((2 * (lane & 3)) ^ vsw)) = cv;
  }
}

// Pair lookahead: the panel warp (idle until the next panel's columns are ready) and the helper, both on
// SMSP 0, apply panel (j0)'s reflector to column block cb together.  Half h takes rows
// [h*brows/2, (h+1)*brows/2) of GEMM1 (W = R_p + V^T B, 4 accumulator chains; the helper adds the R_p
// tile), the two partial W tiles meet through shared memory (one 64-thread barrier), both warps form the
// same W' = T^T W (fixed summation order), the helper writes R_p -= W', and each warp updates its half of
// the row blocks of B -= V W'.  Two dependency chains interleave on the SMSP's tensor pipe.
__device__ __forceinline__ void lookahead_pair(double* __restrict__ Bs, int lds, int brows, int j0, int vj,
                                               double* __restrict__ R, int npad, const double* __restrict__ Tm,
                                               double* __restrict__ Wpart, double* __restrict__ Wsc, int cb, int pcb,
                                               int h, int lane) {
  const int frag_col = (lane >> 2) ^ ((lane & 2) << 1);
  const int vsw = ((lane >> 2) & 2) << 1;
  double* rtile = R + (int64_t)(j0 + (lane >> 2)) * npad + 8 * cb + 2 * (lane & 3);
  double2 rinit = make_double2(0.0, 0.0);
  if (h == 1) rinit = *reinterpret_cast<const double2*>(rtile);
  const int nrb = brows / 8;
  const int rb_mid = nrb / 2;                       // row blocks [0, rb_mid) | [rb_mid, nrb)
  const int i_beg = h ? 8 * rb_mid : 0, i_end = h ? brows : 8 * rb_mid;
  double c[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
  const double* slab = Bs + (lane & 3) * lds + frag_col;
  int i = i_beg;
#pragma unroll 1
  for (; i + 16 <= i_end; i += 16) {
    double a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double* r = slab + (i + 4 * u) * lds;
      a[u] = r[vj];
      b[u] = r[pcb];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(c[u][0], c[u][1], a[u], b[u]);
  }
  for (; i < i_end; i += 4) {
    const double* r = slab + i * lds;
    dmma(c[0][0], c[0][1], r[vj], r[pcb]);
  }
  const int ci = (lane >> 2) * 8 + 2 * (lane & 3);
  Wpart[h * 64 + ci] = ((c[0][0] + c[1][0]) + (c[2][0] + c[3][0])) + rinit.x;
  Wpart[h * 64 + ci + 1] = ((c[0][1] + c[1][1]) + (c[2][1] + c[3][1])) + rinit.y;
  named_sync(kBarPanelPair, 64);
  Wsc[ci] = Wpart[ci] + Wpart[64 + ci];
  Wsc[ci + 1] = Wpart[ci + 1] + Wpart[64 + ci + 1];
  __syncwarp();
  double w0 = 0.0, w1 = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4)
    dmma(w0, w1, Tm[(k0 + (lane & 3)) * kNB + (lane >> 2)], Wsc[(k0 + (lane & 3)) * 8 + (lane >> 2)]);
  // R_p -= W' from the tile loaded at the start (no second L2 round trip on the lookahead's path: column
  // block p+1 of R_p is touched by nobody else between the two points)
  if (h == 1) *reinterpret_cast<double2*>(rtile) = make_double2(rinit.x - w0, rinit.y - w1);
  __syncwarp();
  Wsc[ci] = w0;
  Wsc[ci + 1] = w1;
  __syncwarp();
  const double wb0 = -Wsc[(lane & 3) * 8 + (lane >> 2)];
  const double wb1 = -Wsc[(4 + (lane & 3)) * 8 + (lane >> 2)];
  __syncwarp();
  int rb = h ? rb_mid : 0;
  const int rb_end = h ? nrb : rb_mid;
#pragma unroll 1
  for (; rb + 4 <= rb_end; rb += 4) {
    double* rows[4];
    double2 cv[4];
    double va[4], vb[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      rows[u] = Bs + (8 * (rb + u) + (lane >> 2)) * lds;
      va[u] = rows[u][vj + ((lane & 3) ^ vsw)];
      vb[u] = rows[u][vj + ((4 + (lane & 3)) ^ vsw)];
      cv[u] = *reinterpret_cast<const double2*>(rows[u] + pcb + ((2 * (lane & 3)) ^ vsw));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(cv[u].x, cv[u].y, va[u], wb0);
#pragma unroll
    for (int u = 0; u < 4; ++u) dmma(cv[u].x, cv[u].y, vb[u], wb1);
#pragma unroll
    for (int u = 0; u < 4; ++u) *reinterpret_cast<double2*>(rows[u] + pcb + ((2 * (lane & 3)) ^ vsw)) = cv[u];
  }
  for (; rb < rb_end; ++rb) {
    double* row = Bs + (8 * rb + (lane >> 2)) * lds;
    double2 cv = *reinterpret_cast<const double2*>(row + pcb + ((2 * (lane & 3)) ^ vsw));
    dmma(cv.x, cv.y, row[vj + ((lane & 3) ^ vsw)], wb0);
    dmma(cv.x, cv.y, row[vj + ((4 + (lane & 3)) ^ vsw)], wb1);
    *reinterpret_cast<double2*>(row + pcb + ((2 * (lane & 3)) ^ vsw)) = cv;
  }
}

// Fold `nrows` data rows (row-major, stride ldsrc, `ncols` real columns) into the R slot `R`.
// triangular: data row i is zero left of column i (the data is another R factor).
//
// Lookahead schedule per panel p (warp 0 = panel warp and warp 4 = helper, both on SMSP 0; warps
// 1,2,3,5,6,7 = GEMM warps on SMSPs 1..3):
//   panel warp : wait ColsReady(p) -> factor panel p -> arrive PanelDone(p) -> its half of the lookahead
//   helper     : wait PanelDone(p) -> stage R diag of panel p+1 -> its half of the lookahead (update of
//                column block p+1 with panel p, lookahead_pair) -> arrive ColsReady(p+1)
//   GEMM warps : wait PanelDone(p) -> arrive ColsReady(p+1) -> update column blocks p+2.. with panel p
// so panel p+1 is factored while the trailing update of panel p runs.  V_p lives in the block's
// panel-p columns (never touched again this block); T and the staged R rows are double-buffered.
template <int RQ, bool kPreload, int W = kTqWarps>
__device__ void tsqr_fold(double* __restrict__ R, const double* __restrict__ src, int64_t nrows, int64_t ldsrc,
                          int ncols, const TqGeom g, bool triangular, bool init_zero,
                          double* __restrict__ stats_out, double* smem) {
  using L = TqLayout;
  constexpr int G = 4;  // column blocks per GEMM group
  // W = 8: panel warp 0, helper warp 4 (both SMSP 0), six GEMM warps.  W = 4 (three CTAs per SM, n <= 104):
  // panel warp 0, helper warp 2, GEMM warps 1 and 3.
  constexpr int kThr = 32 * W;
  constexpr int kHelper = W == 8 ? 4 : 2;
  constexpr int kGemm = W - 2;
  constexpr int kSH = (512 + kThr - 1) / kThr;  // stats columns per thread (n <= 512)
  const int tid = threadIdx.x, lane = tid & 31;
  int warp = tid >> 5;  // logical warp (role); physical warp = (warp + rot) % 8
  if constexpr (!kPreload) {
    // two CTAs per SM: the second CTA's warps usually occupy the next 8 hardware slots, i.e. the same SMSPs
    // (slot % 4) as the first CTA's, which would put both panel warps and both helpers on SMSP 0.  Rotate
    // the roles by one warp in that CTA so its latency-critical pair runs on SMSP 1 (a hint only: any
    // rotation is functionally identical; measured n=64 353 -> 357, n=48 363 -> 371 GB/s; by 2: no change, by 3: -5%).
    // (broadcast through the reduction scratch, first used long after the block loop's first barrier)
    volatile int* s_rot = reinterpret_cast<volatile int*>(smem + TqLayout::red(g));
    if (tid == 0) {
      unsigned wid;
      asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
      *s_rot = (int)((wid >> 3) & 1u);
    }
    __syncthreads();
    warp = (warp - *s_rot) & (kTqWarps - 1);
  }
  if constexpr (W == 4) {
    // three 4-warp CTAs per SM occupy hardware slots 0-3, 4-7, 8-11: rotate the roles by the CTA's slot
    // group so the three panel warps run on different SMSPs (a hint only)
    volatile int* s_rot = reinterpret_cast<volatile int*>(smem + TqLayout::red(g));
    if (tid == 0) {
      unsigned wid;
      asm volatile("mov.u32 %0, %%warpid;" : "=r"(wid));
      *s_rot = (int)((wid >> 2) & 3u);
    }
    __syncthreads();
    warp = (warp - *s_rot) & (W - 1);
  }
  const int npad = g.npad, lds = g.lds, brows = g.brows;
  double* Bs = smem;
  double* Rdg = smem + L::rd(g);
  double* Tm = smem + L::tm(g);
  double* red = smem + L::red(g);
  double* Wsc = smem + L::wsc(g) + warp * kNB * 8;
  double* Wpart = smem + L::wpart(g);
  const int npanels = npad / kNB, ncb = npad / 8;
  const bool vec16 = ((ldsrc & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);

  if (init_zero) {
    for (int64_t idx = tid; idx < (int64_t)npad * npad; idx += kThr) R[idx] = 0.0;
  }
  double l1a[kSH], sqa[kSH];
#pragma unroll
  for (int h = 0; h < kSH; ++h) l1a[h] = sqa[h] = 0.0;

  for (int64_t r0 = 0; r0 < nrows; r0 += brows) {
    const int cnt = (int)min64(brows, nrows - r0);
    const int p0 = triangular ? (int)min64(r0 / kNB, npanels) : 0;
    __syncthreads();  // previous block fully consumed; R (init or previous block) visible
    stage_block(Bs, lds, src + r0 * ldsrc, ldsrc, cnt, ncols, brows, npad, vec16);
    if (p0 < npanels && warp == 0) stage_rdiag(Rdg + (p0 & 1) * kNB * kNB, R, npad, p0 * kNB, lane);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (stats_out) {
#pragma unroll
      for (int h = 0; h < kSH; ++h) {
        const int col = tid + h * kThr;
        if (col < ncols) {
          double a = l1a[h], q = sqa[h];
          for (int i = 0; i < cnt; ++i) {
            const double v = Bs[i * lds + (col ^ swz(i))];
            a += fabs(v);
            q = fma(v, v, q);
          }
          l1a[h] = a;
          sqa[h] = q;
        }
      }
    }
    for (int p = p0; p < npanels; ++p) {
      const int j0 = p * kNB;
      const int buf = p & 1;
      const double* Rdc = Rdg + buf * kNB * kNB;
      const double* Tmc = Tm + buf * kNB * kNB;
      const bool more = p + 1 < npanels;
      const int tq_p = (r0 == 0 && p < 64) ? p : -1;
      if (warp == 0) {
        if (p > p0) named_sync(kBarColsReady, kThr);
        TQ_RESOLVE(Rdg);
        TQ_TRACE(1);
        panel_factor_lazy<RQ, kPreload>(Bs, lds, brows, j0, j0, R, npad, Rdc, Tm + buf * kNB * kNB, red, lane, tq_p);
        TQ_TRACE(2);
        named_arrive(kBarPanelDone, kThr);
        if (kPairLookahead && more) {
          if (p > p0) named_sync(kBarNextReady, 64);  // tile p + 1's update by panel p - 1 is done
          __syncwarp();  // the warp's own V / T stores are visible to all its lanes
          lookahead_pair(Bs, lds, brows, j0, j0, R, npad, Tmc, Wpart, Wsc, p + 1, 8 * (p + 1), 0, lane);
        }
      } else if (warp == kHelper) {
        // helper on SMSP 0: the lookahead starts the moment the panel is published (not after the GEMM
        // warps' trailing work) and its DMMAs never overlap the panel's FP64 chain on this SMSP
        named_sync(kBarPanelDone, kThr);
        TQ_RESOLVE(Rdg);
        if (more) {
          TQ_TRACE(3);
          stage_rdiag(Rdg + (buf ^ 1) * kNB * kNB, R, npad, j0 + kNB, lane);
          cp_async_commit();
          if (kPairLookahead)
            lookahead_pair(Bs, lds, brows, j0, j0, R, npad, Tmc, Wpart, Wsc, p + 1, 8 * (p + 1), 1, lane);
          else
            lookahead_single(Bs, lds, brows, j0, R, npad, Tmc, Wsc, p + 1, lane);
          cp_async_wait<0>();
          __syncwarp();
          TQ_TRACE(4);
          named_arrive(kBarColsReady, kThr);
        }
      } else {
        const int gi = W == 8 ? gemm_index(warp) : (warp == 1 ? 0 : 1);
        named_sync(kBarPanelDone, kThr);
        TQ_RESOLVE(Rdg);
        if (more) named_arrive(kBarColsReady, kThr);
        // trailing column blocks p+2 .. ncb-1, round-robin over the GEMM warps in groups of G
        for (int base = p + 2 + gi; base < ncb; base += kGemm * G) {
          int cnt_g = 0;
          int cbs[G];
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
            cbs[gg] = base + kGemm * gg;
            if (cbs[gg] < ncb) ++cnt_g;
          }
          // a short last group is updated in one call (shared V fragment loads), not block by block
          if (cnt_g == G) {
            const int pc[G] = {8 * cbs[0], 8 * cbs[1], 8 * cbs[2], 8 * cbs[3]};
            update_cbs<G>(Bs, lds, brows, j0, j0, R, npad, Tmc, Wsc, cbs, pc, lane, tq_p);
          } else if (cnt_g == 3) {
            const int three[3] = {cbs[0], cbs[1], cbs[2]};
            const int pc[3] = {8 * cbs[0], 8 * cbs[1], 8 * cbs[2]};
            update_cbs<3>(Bs, lds, brows, j0, j0, R, npad, Tmc, Wsc, three, pc, lane, tq_p);
          } else if (cnt_g == 2) {
            const int two[2] = {cbs[0], cbs[1]};
            const int pc[2] = {8 * cbs[0], 8 * cbs[1]};
            update_cbs<2>(Bs, lds, brows, j0, j0, R, npad, Tmc, Wsc, two, pc, lane, tq_p);
          } else if (cnt_g == 1) {
            const int one[1] = {cbs[0]};
            const int pc[1] = {8 * cbs[0]};
            update_cbs<1>(Bs, lds, brows, j0, j0, R, npad, Tmc, Wsc, one, pc, lane, tq_p);
          }
          // tile p + 2 (this warp's first group when gi == 0) is the next lookahead's target
          if (kPairLookahead && base == p + 2) {
            __syncwarp();
            named_arrive(kBarNextReady, 64);
          }
        }
      }
    }
  }
  if (stats_out) {
#pragma unroll
    for (int h = 0; h < kSH; ++h) {
      const int col = tid + h * kThr;
      if (col < npad) {
        stats_out[col] = l1a[h];
        stats_out[npad + col] = sqa[h];
      }
    }
  }
}

// MINB == 3 selects the 4-warp CTA (three per SM, n <= 104)
template <int MINB>
constexpr int tq_warps() { return MINB == 3 ? 4 : kTqWarps; }

template <int RQ, int MINB>
__global__ void __launch_bounds__(32 * tq_warps<MINB>(), MINB)
    tsqr_leaf_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, int64_t rows_per_cta, TqGeom g,
                     double* __restrict__ slots, double* __restrict__ stats) {
  extern __shared__ __align__(16) double smem[];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t cnt = max64(0, min64(rows_per_cta, m - r0));
  double* R = slots + (int64_t)blockIdx.x * g.npad * g.npad;
  double* st = stats ? stats + (int64_t)blockIdx.x * 2 * g.npad : nullptr;
  tsqr_fold<RQ, MINB != 2, tq_warps<MINB>()>(R, x + r0 * ldx, cnt, ldx, g.n, g, false, true, st, smem);
}

// One level of the binary-counter tree: slot[q*2^L] = qr([slot[q*2^L]; slot[q*2^L + 2^(L-1)]]),
// or (fold) slot[dst] = qr([slot[dst]; slot[src]]).
template <int RQ, int MINB>
__global__ void __launch_bounds__(32 * tq_warps<MINB>(), MINB)
    tsqr_combine_kernel(double* __restrict__ slots, int64_t span, int64_t half, int64_t fold_dst, int64_t fold_src,
                        TqGeom g) {
  extern __shared__ __align__(16) double smem[];
  const int64_t ss = (int64_t)g.npad * g.npad;
  int64_t dst, srcs;
  if (span > 0) {
    dst = (int64_t)blockIdx.x * span;
    srcs = dst + half;
  } else {
    dst = fold_dst;
    srcs = fold_src;
  }
  tsqr_fold<RQ, MINB != 2, tq_warps<MINB>()>(slots + dst * ss, slots + srcs * ss, g.npad, g.npad, g.npad, g, true, false,
                                              nullptr, smem);
}

// ---------------------------------------------------------------------------
// Split leaf (wide n, e.g. config C2 n = 200): 256-row blocks, twice the rows in flight of the 128-row
// leaf above.  Throughput of the fold is (rows in flight) / (n x per-column panel latency) and the
// 227 KB of shared memory hold only 128 rows x 200 columns, so the block is split by columns: the left
// S = ceil(npanels / 2) column tiles (8 columns each) live in shared memory, the right ones in a per-leaf
// L2-resident workspace (brows x 8(npanels - S) doubles).  Tiles are updated where they live (the GEMM
// warps' trailing update of a workspace tile streams it through registers, DMMA operands from the
// shared-memory V), and they move in as the left tiles die: right-looking QR frees tile s once panel s's
// trailing update is done, so in iteration p = t - S + 1 the update of right tile t (by panel p) reads
// the workspace and writes shared slot t - S.  Panel p and the lookahead tile p + 1 are therefore always
// in shared memory (S >= 3).  Logical tile t lives in slot t (t < S) or t - S (t >= S, migrated);
// R is addressed logically.  The first update of a right tile reads X directly (zero-filling rows past
// the end and padding columns) and accumulates its column l1 / sum of squares on the way.
#ifndef TSNMF_SPLIT_ROWS
#define TSNMF_SPLIT_ROWS 256
#endif
constexpr int kSplitRows = TSNMF_SPLIT_ROWS;  // multiple of 32 (panel rows per lane = kSplitRows / 32)
constexpr int kSplitRq = kSplitRows / 32;

struct SplitGeom {
  int n, npad;  // data / padded columns
  int S;        // shared-memory tile slots (left tiles 0..S-1)
  int lds;      // shared row stride (8 S rounded to % 16 == 8)
  int wld;      // workspace row stride (8 (npanels - S))
};

__host__ __device__ inline TqGeom split_tq_geom(const SplitGeom& sg) {
  TqGeom g;
  g.n = sg.n;
  g.npad = sg.npad;
  g.lds = sg.lds;
  g.brows = kSplitRows;
  return g;
}

// One right tile (logical column block cb) updated with panel (j0)'s block reflector, data streamed from
// global memory (X when kFromX, else the tile's workspace slot: tile-major, 256 rows x 8 doubles) and
// written to the workspace slot (or, kToSmem, to the swizzled shared slot at column dcol).  The W pass
// (W = R_p + V^T B) takes the tile in the DMMA B-operand layout (lane: row 4s + l%4, col l/4), all of it in
// flight at once; the C pass (B -= V W') re-reads it in the C-tile layout (row l/4, cols 2(l%4)..+1: 512
// contiguous bytes per 8 rows, L2 hits) in double-buffered batches instead of regathering registers with
// shuffles.  kFromX also adds the tile's column l1 / sum of squares to st[0..8) / st[8..16) (one warp owns a
// right tile's first update, so plain read-modify-writes).  Not inlined: one copy per variant keeps the
// kernel in the instruction cache and its register budget for the panel / update_cbs paths.
template <bool kFromX, bool kToSmem>
__device__ __noinline__ void update_global(const double* __restrict__ Bs, int lds, int vj, int j0,
                                              const double* __restrict__ src, int64_t ldx, int vrows, int vcols,
                                              double* __restrict__ dst, int dcol, double* __restrict__ R, int npad,
                                              int cb, const double* __restrict__ Tm, double* __restrict__ Wsc,
                                              double* __restrict__ st) {
  constexpr int K = kSplitRows / 4;   // W-pass k-steps (registers per lane)
  constexpr int NRB = kSplitRows / 8;  // C-pass row blocks
  constexpr int CB = 8;                // row blocks per C-pass batch
  const int lane = threadIdx.x & 31;
  // workspace: evict_last; X: kept for the C pass's re-read, then evict_first
  const uint64_t pol_ws = l2_policy_evict_last(), pol_x = l2_policy_evict_first(), pol_xw = l2_policy_evict_last();
  const int frag_col = (lane >> 2) ^ ((lane & 2) << 1);
  const int vsw = ((lane >> 2) & 2) << 1;
  double* rtile = R + (int64_t)(j0 + (lane >> 2)) * npad + 8 * cb + 2 * (lane & 3);
  const double2 rinit = *reinterpret_cast<const double2*>(rtile);
  const bool colok = !kFromX || (lane >> 2) < vcols;
  // two accumulator chains over alternating 4-row k-steps, summed (c0 + c1) + R: update_cbs's order, so a
  // tile's update is bitwise the same whichever path applies it
  double c[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  double sa = 0.0, sq = 0.0;
  {
    double b[K];
    if (kFromX) {
      const double* bp = src + (int64_t)(lane & 3) * ldx + (lane >> 2);
      const int64_t step = 4 * ldx;
#pragma unroll
      for (int s = 0; s < K; ++s) {
        b[s] = (colok && 4 * s + (lane & 3) < vrows) ? ld_hint(bp, pol_xw) : 0.0;  // re-read by the C pass
        bp += step;
      }
    } else {
      const double* bp = src + 8 * (lane & 3) + (lane >> 2);
#pragma unroll
      for (int s = 0; s < K; ++s) b[s] = ld_hint(bp + 32 * s, pol_ws);
    }
    const double* vslab = Bs + (lane & 3) * lds + frag_col + vj;
#pragma unroll
    for (int s = 0; s < K; ++s) {
      dmma(c[s & 1][0], c[s & 1][1], vslab[4 * s * lds], b[s]);
      if (kFromX) {
        sa += fabs(b[s]);
        sq = fma(b[s], b[s], sq);
      }
    }
  }
  if (kFromX) {
    sa += __shfl_xor_sync(0xffffffffu, sa, 1);
    sq += __shfl_xor_sync(0xffffffffu, sq, 1);
    sa += __shfl_xor_sync(0xffffffffu, sa, 2);
    sq += __shfl_xor_sync(0xffffffffu, sq, 2);
    if ((lane & 3) == 0) {
      st[lane >> 2] += sa;
      st[8 + (lane >> 2)] += sq;
    }
  }
  const int ci = (lane >> 2) * 8 + 2 * (lane & 3);
  Wsc[ci] = (c[0][0] + c[1][0]) + rinit.x;
  Wsc[ci + 1] = (c[0][1] + c[1][1]) + rinit.y;
  __syncwarp();
  double w0 = 0.0, w1 = 0.0;
#pragma unroll
  for (int k0 = 0; k0 < 8; k0 += 4)
    dmma(w0, w1, Tm[(k0 + (lane & 3)) * kNB + (lane >> 2)], Wsc[(k0 + (lane & 3)) * 8 + (lane >> 2)]);
  *reinterpret_cast<double2*>(rtile) = make_double2(rinit.x - w0, rinit.y - w1);
  __syncwarp();
  Wsc[ci] = w0;
  Wsc[ci + 1] = w1;
  __syncwarp();
  const double wb0 = -Wsc[(lane & 3) * 8 + (lane >> 2)];
  const double wb1 = -Wsc[(4 + (lane & 3)) * 8 + (lane >> 2)];
  __syncwarp();
  // C pass: row block rb = rows 8 rb + l/4, cols 2 (l%4) .. +1
  const double* vrow = Bs + (lane >> 2) * lds + vj;
  const int va = (lane & 3) ^ vsw, vb = (4 + (lane & 3)) ^ vsw;
  auto cload = [&](int rb) -> double2 {
    const int row = 8 * rb + (lane >> 2);
    if (kFromX) {  // zero past the last row and the last column (C layout: this lane's columns 2 (l%4), +1)
      const int c0 = 2 * (lane & 3);
      const double* q = src + (int64_t)row * ldx + c0;
      const bool rok = row < vrows;
      return make_double2(rok && c0 < vcols ? ld_hint(q, pol_x) : 0.0, rok && c0 + 1 < vcols ? ld_hint(q + 1, pol_x) : 0.0);
    }
    double2 v;
    const double* q = src + 64 * rb + 8 * (lane >> 2) + 2 * (lane & 3);
    asm volatile("ld.global.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(q), "l"(pol_ws));
    return v;
  };
  double2 cur[CB], nxt[CB];
#pragma unroll
  for (int u = 0; u < CB; ++u) cur[u] = cload(u);
#pragma unroll
  for (int b0 = 0; b0 < NRB; b0 += CB) {
    if (b0 + CB < NRB) {
#pragma unroll
      for (int u = 0; u < CB; ++u) nxt[u] = cload(b0 + CB + u);
    }
#pragma unroll
    for (int u = 0; u < CB; ++u) {
      const int rb = b0 + u;
      const double* vr = vrow + 8 * rb * lds;
      double cx = cur[u].x, cy = cur[u].y;
      dmma(cx, cy, vr[va], wb0);
      dmma(cx, cy, vr[vb], wb1);
      if (kToSmem)
        *reinterpret_cast<double2*>(dst + (8 * rb + (lane >> 2)) * lds + dcol + ((2 * (lane & 3)) ^ vsw)) =
            make_double2(cx, cy);
      else
        st_hint(reinterpret_cast<double2*>(dst + 64 * rb + 8 * (lane >> 2) + 2 * (lane & 3)), make_double2(cx, cy),
                pol_ws);
    }
#pragma unroll
    for (int u = 0; u < CB; ++u) cur[u] = nxt[u];
  }
}

#ifndef TSNMF_SPLIT_PREFETCH
#define TSNMF_SPLIT_PREFETCH 0  // measured: none 265, at block start 261, late 261 GB/s (C2 shape, 2^24 rows)
#endif
constexpr int kSplitPrefetch = TSNMF_SPLIT_PREFETCH;
#ifndef TSNMF_TSQR_REGLEAF_DEFAULT
#define TSNMF_TSQR_REGLEAF_DEFAULT 1
#endif  // next block's right columns into L2: 0 off, 1 at block start, 2 late
// L2 prefetch of the right columns [lcols, ncols) of rows [row0, row0 + 256) (their first updates read X)
__device__ __forceinline__ void prefetch_next_right(const double* X, int64_t ldx, int64_t nrows, int64_t row0,
                                                    int lcols, int ncols, int t, int nt) {
  if (row0 >= nrows || ncols <= lcols) return;
  const int nr = (int)min64(kSplitRows, nrows - row0);
  for (int r = t; r < nr; r += nt) {
    const char* a = reinterpret_cast<const char*>(X + (row0 + r) * ldx + lcols);
    const char* e = reinterpret_cast<const char*>(X + (row0 + r) * ldx + ncols);
    for (const char* q = (const char*)((uintptr_t)a & ~(uintptr_t)127); q < e; q += 128)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
  }
}

template <int RQ>
__device__ void tsqr_split_fold(double* __restrict__ R, const double* __restrict__ X, int64_t nrows, int64_t ldx,
                                int ncols, const SplitGeom sg, double* __restrict__ ws,
                                double* __restrict__ stats_out, double* smem) {
  using L = TqLayout;
  constexpr int G = 4;
  constexpr int W = kTqWarps;
  constexpr int kThr = 32 * W;
  constexpr int kHelper = 4;
  constexpr int kGemm = W - 2;
  const TqGeom g = split_tq_geom(sg);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npad = g.npad, lds = g.lds, brows = g.brows;
  const int S = sg.S, npanels = npad / kNB;
  const int lcols = 8 * S;  // logical columns staged into shared memory
  double* Bs = smem;
  double* Rdg = smem + L::rd(g);
  double* Tm = smem + L::tm(g);
  double* red = smem + L::red(g);
  double* Wsc = smem + L::wsc(g) + warp * kNB * 8;
  double* Wpart = smem + L::wpart(g);
  double* rstat = smem + L::total(g);  // right tile t - S: column l1 [16 (t - S), +8), sum of squares [+8, +16)
  const bool vec16 = ((ldx & 1) == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  const int scols = ncols < lcols ? ncols : lcols;
  auto slot_col = [&](int t) { return 8 * (t < S ? t : t - S); };

  for (int64_t idx = tid; idx < (int64_t)npad * npad; idx += kThr) R[idx] = 0.0;
  constexpr int kSH = (512 + kThr - 1) / kThr;
  double l1a[kSH], sqa[kSH];
#pragma unroll
  for (int h = 0; h < kSH; ++h) l1a[h] = sqa[h] = 0.0;
  for (int i = tid; i < 2 * sg.wld; i += kThr) rstat[i] = 0.0;  // (ordered by the block loop's barrier)
  const int gi = warp == 0 || warp == kHelper ? -1 : gemm_index(warp);

  for (int64_t r0 = 0; r0 < nrows; r0 += brows) {
    const int cnt = (int)min64(brows, nrows - r0);
    const double* xb = X + r0 * ldx;
    __syncthreads();
    stage_rows_swz_stream(Bs, lds, xb, ldx, cnt, scols, brows, lcols, vec16);
    if (warp == 0) stage_rdiag(Rdg, R, npad, 0, lane);
    cp_async_commit();
    if (kSplitPrefetch == 1) prefetch_next_right(X, ldx, nrows, r0 + brows, lcols, ncols, tid, kThr);
    cp_async_wait<0>();
    __syncthreads();
    if (stats_out) {
#pragma unroll
      for (int h = 0; h < kSH; ++h) {
        const int col = tid + h * kThr;
        if (col < scols) {
          double a = l1a[h], q = sqa[h];
          for (int i = 0; i < cnt; ++i) {
            const double v = Bs[i * lds + (col ^ swz(i))];
            a += fabs(v);
            q = fma(v, v, q);
          }
          l1a[h] = a;
          sqa[h] = q;
        }
      }
    }
    for (int p = 0; p < npanels; ++p) {
      const int j0 = p * kNB;
      const int vj = slot_col(p);
      const int buf = p & 1;
      const double* Rdc = Rdg + buf * kNB * kNB;
      const double* Tmc = Tm + buf * kNB * kNB;
      const bool more = p + 1 < npanels;
      const int tq_p = (r0 == brows && p < 64) ? p : -1;  // trace builds: the second block of CTA 0
      if (kSplitPrefetch == 2 && p == npanels - 6 && gi >= 0)  // GEMM warps, off the tail of the block
        prefetch_next_right(X, ldx, nrows, r0 + brows, lcols, ncols, tid - 32 * (warp < kHelper ? 1 : 2), 32 * kGemm);
      if (warp == 0) {
        if (p > 0) named_sync(kBarColsReady, kThr);
        TQ_RESOLVE(Rdg);
        TQ_TRACE(41);
        panel_factor_lazy<RQ, true>(Bs, lds, brows, j0, vj, R, npad, Rdc, Tm + buf * kNB * kNB, red, lane, -1);
        TQ_TRACE(42);
        named_arrive(kBarPanelDone, kThr);
        if (more) {
          if (p > 0) named_sync(kBarNextReady, 64);  // tile p + 1's update by panel p - 1 is done
          __syncwarp();
          lookahead_pair(Bs, lds, brows, j0, vj, R, npad, Tmc, Wpart, Wsc, p + 1, slot_col(p + 1), 0, lane);
          TQ_TRACE(45);
        }
      } else if (warp == kHelper) {
        named_sync(kBarPanelDone, kThr);
        TQ_RESOLVE(Rdg);
        TQ_TRACE(43);
        if (more) {
          stage_rdiag(Rdg + (buf ^ 1) * kNB * kNB, R, npad, j0 + kNB, lane);
          cp_async_commit();
          lookahead_pair(Bs, lds, brows, j0, vj, R, npad, Tmc, Wpart, Wsc, p + 1, slot_col(p + 1), 1, lane);
          cp_async_wait<0>();
          __syncwarp();
          TQ_TRACE(44);
          named_arrive(kBarColsReady, kThr);
        }
      } else {
        named_sync(kBarPanelDone, kThr);
        TQ_RESOLVE(Rdg);
        TQ_TRACE(46);
        if (more) named_arrive(kBarColsReady, kThr);
        for (int base = p + 2 + gi; base < npanels; base += kGemm * G) {
          // shared tiles of this group in one call (shared V fragment loads), then the workspace tiles one by
          // one.  Tiles in shared memory are those below S + max(p - 1, 0): a prefix of the group.
          const int lim = min(npanels, S + (p > 0 ? p - 1 : 0));
          const int c4[4] = {base, base + kGemm, base + 2 * kGemm, base + 3 * kGemm};
          const int ns = c4[3] < lim ? 4 : (c4[2] < lim ? 3 : (c4[1] < lim ? 2 : (c4[0] < lim ? 1 : 0)));
          if (ns == 4) {
            const int p4[4] = {slot_col(c4[0]), slot_col(c4[1]), slot_col(c4[2]), slot_col(c4[3])};
            update_cbs<4>(Bs, lds, brows, j0, vj, R, npad, Tmc, Wsc, c4, p4, lane, -1);
          } else if (ns == 3) {
            const int c3[3] = {c4[0], c4[1], c4[2]}, p3[3] = {slot_col(c4[0]), slot_col(c4[1]), slot_col(c4[2])};
            update_cbs<3>(Bs, lds, brows, j0, vj, R, npad, Tmc, Wsc, c3, p3, lane, -1);
          } else if (ns == 2) {
            const int c2[2] = {c4[0], c4[1]}, p2[2] = {slot_col(c4[0]), slot_col(c4[1])};
            update_cbs<2>(Bs, lds, brows, j0, vj, R, npad, Tmc, Wsc, c2, p2, lane, -1);
          } else if (ns == 1) {
            const int c1[1] = {c4[0]}, p1[1] = {slot_col(c4[0])};
            update_cbs<1>(Bs, lds, brows, j0, vj, R, npad, Tmc, Wsc, c1, p1, lane, -1);
          }
          if (base == p + 2) {  // tile p + 2 (gi == 0, shared slot) is the next lookahead's target
            __syncwarp();
            named_arrive(kBarNextReady, 64);
          }
          TQ_TRACE(47);
#pragma unroll 1
          for (int gg = ns; gg < G; ++gg) {
            const int t = base + kGemm * gg;
            if (t >= npanels) break;
            double* wt = ws + (int64_t)kSplitRows * 8 * (t - S);  // tile-major workspace slot
            if (p == 0)
              update_global<true, false>(Bs, lds, vj, j0, xb + 8 * t, ldx, cnt, ncols - 8 * t, wt, 0, R, npad, t,
                                         Tmc, Wsc, rstat + 16 * (t - S));
            else if (t - S + 1 == p)
              update_global<false, true>(Bs, lds, vj, j0, wt, 0, 0, 0, Bs, 8 * (t - S), R, npad, t, Tmc, Wsc,
                                         nullptr);
            else
              update_global<false, false>(Bs, lds, vj, j0, wt, 0, 0, 0, wt, 0, R, npad, t, Tmc, Wsc, nullptr);
          }
          TQ_TRACE(48);
        }
      }
    }
  }
  if (stats_out) {
#pragma unroll
    for (int h = 0; h < kSH; ++h) {
      const int col = tid + h * kThr;
      if (col < lcols) {
        stats_out[col] = l1a[h];
        stats_out[npad + col] = sqa[h];
      }
    }
    __syncthreads();
    for (int i = tid; i < 8 * (npanels - S); i += kThr) {
      const int t = S + i / 8, c = i % 8;
      stats_out[8 * t + c] = rstat[16 * (t - S) + c];
      stats_out[npad + 8 * t + c] = rstat[16 * (t - S) + 8 + c];
    }
  }
}

__global__ void __launch_bounds__(256, 1)
    tsqr_split_leaf_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, int64_t rows_per_cta, SplitGeom sg,
                           double* __restrict__ slots, double* __restrict__ stats, double* __restrict__ wsr) {
  extern __shared__ __align__(16) double smem[];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t cnt = max64(0, min64(rows_per_cta, m - r0));
  double* R = slots + (int64_t)blockIdx.x * sg.npad * sg.npad;
  double* st = stats ? stats + (int64_t)blockIdx.x * 2 * sg.npad : nullptr;
  double* ws = wsr + (int64_t)blockIdx.x * kSplitRows * sg.wld;
  tsqr_split_fold<kSplitRq>(R, x + r0 * ldx, cnt, ldx, sg.n, sg, ws, st, smem);
}

// ---------------------------------------------------------------------------
// Narrow leaf (n <= 32, e.g. config C4 n = 25): one WARP per chain.  Each warp owns a contiguous row range
// and its own R (lane c holds column c of R in registers), stages 32-row blocks in shared memory
// (cp.async), takes row l of the block into lane l's registers and folds it into R with Householder
// reflectors [e_j; v] one column at a time:
//   norm: warp butterfly;  scalars (dlarfg conventions, as the panel);  v_l = x_l[j] * scale;
//   w_c = R(j, c) + sum_l v_l x_l[c]  (lane c sums the column of products through shared memory);
//   R(j, c) -= tau w_c (lane c);  x_l[c] -= tau w_c v_l (every lane, row l).
// No CTA barriers, no panel/GEMM split: the shared-panel design's throughput is bounded by one panel
// chain per SM (rows in flight / (n x column latency)); here 12 independent chains per SM run in parallel
// (3 CTAs x 4 warps) and the kernel is issue-bound instead.  Leaves = warps, combined by the same tree.
constexpr int kSmWarps = 4;

template <int NC>
struct SmallLayout {
  static constexpr int ld = NC + 1;                 // odd stride: column reads by lane c are conflict-free
  static constexpr int per_warp = 32 * ld;          // staged block / products (doubles)
  static constexpr size_t bytes = sizeof(double) * (size_t)per_warp * kSmWarps;
};

// Fold rows [0, cnt) (cnt <= 32) of a row-major matrix (stride ld, n real columns) into the warp's R
// (lane c holds column c).  buf: the warp's 32 x (NC+1) shared tile.  With `l1`/`sq` set, lane c also
// accumulates the column's sum of |x| and x^2.
template <int NC>
__device__ __forceinline__ void small_fold_block(const double* __restrict__ src, int64_t ld, int cnt, int n,
                                                 double* __restrict__ buf, double (&rcol)[NC], int lane,
                                                 double* l1, double* sq) {
  using Ly = SmallLayout<NC>;
  // stage (zero-padded to 32 x NC); element (row, c) at buf[row * ld + c]
  __syncwarp();
  for (int idx = lane; idx < 32 * NC; idx += 32) {
    const int row = idx / NC, c = idx - row * NC;
    if (row < cnt && c < n)
      cp_async8(buf + row * Ly::ld + c, src + row * ld + c);
    else
      buf[row * Ly::ld + c] = 0.0;
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncwarp();
  if (l1 && lane < NC) {
    double a = 0.0, q = 0.0;
#pragma unroll 8
    for (int row = 0; row < 32; ++row) {
      const double v = buf[row * Ly::ld + lane];
      a += fabs(v);
      q = fma(v, v, q);
    }
    *l1 += a;
    *sq += q;
  }
  double xr[NC];  // lane l: row l of the block
#pragma unroll
  for (int c = 0; c < NC; ++c) xr[c] = buf[lane * Ly::ld + c];
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    if (j >= n) break;
    // sub-column norm^2 and alpha = R(j, j) (lane j)
    double d = xr[j] * xr[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
    const double alpha = __shfl_sync(0xffffffffu, rcol[j], j);
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (d > 0.0) {
      const double ss = fma(alpha, alpha, d);
      const double inv = fast_rsqrt(ss);
      const double nrm = ss * inv;
      beta = -copysign(nrm, alpha);
      tau = fma(fabs(alpha), inv, 1.0);
      scale = copysign(fast_rcp(fabs(alpha) + nrm), alpha);
    }
    const double v = xr[j] * scale;
    __syncwarp();  // every lane has read the previous column's tw values from buf
    // products P[l][c] = v_l x_l[c] for c > j; lane c sums its column
#pragma unroll
    for (int c = j + 1; c < NC; ++c) buf[lane * Ly::ld + c] = v * xr[c];
    __syncwarp();
    double tw = 0.0;
    if (lane > j && lane < NC) {
      double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
      for (int row = 0; row < 32; row += 4) {
        s0 += buf[(row + 0) * Ly::ld + lane];
        s1 += buf[(row + 1) * Ly::ld + lane];
        s2 += buf[(row + 2) * Ly::ld + lane];
        s3 += buf[(row + 3) * Ly::ld + lane];
      }
      const double w = rcol[j] + ((s0 + s1) + (s2 + s3));
      tw = tau * w;
      rcol[j] -= tw;
    }
    if (lane == j) rcol[j] = beta;
    __syncwarp();  // products consumed
    if (lane > j && lane < NC) buf[lane] = tw;  // row 0 of the product tile is free now
    __syncwarp();
#pragma unroll
    for (int c = j + 1; c < NC; ++c) xr[c] = fma(-buf[c], v, xr[c]);  // broadcast reads
  }
}

template <int NC>
__device__ __forceinline__ void small_store_r(double* __restrict__ R, int npad, int n, const double (&rcol)[NC],
                                              int lane) {
  if (lane < npad) {
#pragma unroll
    for (int i = 0; i < NC; ++i)
      if (i < npad) R[(int64_t)i * npad + lane] = (i <= lane && lane < n) ? rcol[i] : 0.0;
    for (int i = NC; i < npad; ++i) R[(int64_t)i * npad + lane] = 0.0;  // NC may be < npad (n < NC <= npad)
  }
}

template <int NC>
__global__ void __launch_bounds__(32 * kSmWarps, 3)
    tsqr_small_leaf_kernel(const double* __restrict__ x, int64_t m, int n, int64_t ldx, int64_t rows_per_warp,
                           int npad, double* __restrict__ slots, double* __restrict__ stats) {
  extern __shared__ __align__(16) double smem[];
  using Ly = SmallLayout<NC>;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t leaf = (int64_t)blockIdx.x * kSmWarps + wib;
  double* buf = smem + wib * Ly::per_warp;
  const int64_t rbeg = leaf * rows_per_warp;
  const int64_t rend = min64(m, rbeg + rows_per_warp);
  double rcol[NC];  // lane c: column c of R (rows 0..NC)
#pragma unroll
  for (int i = 0; i < NC; ++i) rcol[i] = 0.0;
  double l1 = 0.0, sq = 0.0;  // lane c: column c
  for (int64_t r0 = rbeg; r0 < rend; r0 += 32)
    small_fold_block<NC>(x + r0 * ldx, ldx, (int)min64(32, rend - r0), n, buf, rcol, lane, stats ? &l1 : nullptr,
                         &sq);
  small_store_r<NC>(slots + leaf * npad * npad, npad, n, rcol, lane);
  if (stats && lane < npad) {
    stats[leaf * 2 * npad + lane] = lane < n ? l1 : 0.0;
    stats[leaf * 2 * npad + npad + lane] = lane < n ? sq : 0.0;
  }
}

// One level of the binary-counter tree for the narrow path, one warp per pair:
// slot[q span] = qr([slot[q span]; slot[q span + half]]), or (span == 0) slot[dst] = qr([slot[dst]; slot[src]]).
template <int NC>
__global__ void __launch_bounds__(32 * kSmWarps)
    tsqr_small_combine_kernel(double* __restrict__ slots, int npad, int n, int64_t span, int64_t half, int64_t npairs,
                              int64_t fold_dst, int64_t fold_src) {
  extern __shared__ __align__(16) double smem[];
  using Ly = SmallLayout<NC>;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t q = (int64_t)blockIdx.x * kSmWarps + wib;
  if (span > 0 && q >= npairs) return;  // whole idle warps only (no CTA barrier in this kernel)
  const int64_t dst = span > 0 ? q * span : fold_dst;
  const int64_t src = span > 0 ? dst + half : fold_src;
  const int64_t ss = (int64_t)npad * npad;
  double* R = slots + dst * ss;
  double rcol[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) rcol[i] = (i < npad && lane < npad) ? R[(int64_t)i * npad + lane] : 0.0;
  small_fold_block<NC>(slots + src * ss, npad, npad, n, smem + wib * Ly::per_warp, rcol, lane, nullptr, nullptr);
  small_store_r<NC>(R, npad, n, rcol, lane);
}

// ---------------------------------------------------------------------------
// Narrow leaf, register-block version (n <= 32; the default narrow leaf): one chain per warp (CTA = one
// warp), blocks of 32*S rows held in registers (lane l: rows l, l+32, ..), R in shared memory.
// The per-column fixed costs of the chain (butterfly norm, reflector scalars, the column sums of the
// products through shared memory, the broadcast of tau*w) are paid once per 32*S rows instead of once per
// 32, so the instruction count per row drops ~S-fold for those parts.  Blocks are staged by the bulk-copy
// (TMA) engine into a dense buffer (one instruction per block, completion on an mbarrier) when X is
// contiguous with odd n (conflict-free row reads at stride n), else by cp.async at an odd stride; the
// next block's copy is issued as soon as the current one is in registers, so it overlaps the fold.
// Same reflector algebra as small_fold_block ([e_j; v], dlarfg conventions, tsqr.py:129-153 semantics).
struct WlGeom {
  int n, npad;
  int ls;        // stage row stride (odd): n for odd n, n + 1 otherwise
  int pld;       // product tile row stride (== 2 mod 4: conflict-free 16-byte row writes)
  int stage_off, prod_off, r_off, tw_off;  // doubles from the CTA's smem base (even: 16-byte aligned)
  int total;     // doubles
};


// CTA barrier every wl_sync column steps (0: none; >= 32: once per row block, at its first column).  The
// warps of a CTA run the same straight-line column code; keeping them in step lets them share
// instruction-cache lines (the unrolled fold is ~100 KB of code at n = 25).  Measured at n = 25 (8 warps):
// none 1023, every 2 columns 971, every 4 997, every 8 1021, every 12 1041, once per block 1063 GB/s;
// narrower code fits the cache and the barrier only costs (n = 17: 1394 without, 1352 with).
#ifndef TSNMF_WL_SYNC
#define TSNMF_WL_SYNC 32
#endif
constexpr int wl_sync(int n) { return n >= 24 ? TSNMF_WL_SYNC : 0; }

// Packed upper-triangular R of the narrow leaf: row i starts at wl_roff(N, i) + i (R(i, c) at wl_roff + c):
// n(n+1)/2 doubles instead of n^2 (n = 25: one more warp per SM fits).
__host__ __device__ constexpr int wl_roff(int n, int i) { return i * n - i * (i - 1) / 2 - i; }

template <int N, int S>
__global__ void __launch_bounds__(256)
    tsqr_warp_leaf_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, int64_t rows_per_warp, int nleaves,
                          WlGeom g, double* __restrict__ slots, double* __restrict__ stats) {
  extern __shared__ __align__(16) double smem[];
  constexpr int BR = 32 * S;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int ls = g.ls, pld = g.pld;
  double* base = smem + (size_t)wib * g.total;
  uint64_t* bar = reinterpret_cast<uint64_t*>(base);
  double* stg = base + g.stage_off;
  double* P = base + g.prod_off;
  double* Rs = base + g.r_off;  // R(i, c), c >= i, packed by rows at Rs[wl_roff(N, i) + c]
  double* TW = base + g.tw_off;
  const int64_t leaf = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;  // surplus warps (leaf >= nleaves) idle
  const int64_t rbeg = leaf * rows_per_warp;
  const int64_t rend = min64(m, rbeg + rows_per_warp);
  const int64_t nblk = rows_per_warp / BR;
  constexpr int kWlSync = wl_sync(N);
  for (int i = lane; i < N * (N + 1) / 2; i += 32) Rs[i] = 0.0;
  for (int i = lane; i < N + 1; i += 32) TW[i] = 0.0;
  if (lane == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  const bool dense = (ldx == N) && (N & 1) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  // stage rows [r0, r0 + cnt); returns true when the bulk engine was used (completion on `bar`)
  auto issue = [&](int64_t r0, int cnt) -> bool {
    const double* src = x + r0 * ldx;
    if (dense && (cnt & 1) == 0) {  // r0 is even (rows_per_warp % BR == 0), so src is 16-byte aligned
      if (lane == 0) {
        fence_proxy_async_smem();  // the warp's reads of the previous block (ordered by __syncwarp) come first
        mbar_arrive_expect_tx(bar, (unsigned)(cnt * N * 8));
        bulk_copy_g2s(stg, src, (unsigned)(cnt * N * 8), bar);
      }
      return true;
    }
    for (GridWalk it(lane, 32, N); it.r < cnt; it.next()) cp_async8(stg + it.r * ls + it.c, src + it.r * ldx + it.c);
    cp_async_commit();
    return false;
  };
  // column stats: 32/N lanes per column (row phases), combined through shared memory at the end
  constexpr int kStatPhases = 32 / N;
  const int scol = lane % N, sph = lane / N;
  double l1 = 0.0, sq = 0.0;
  unsigned phase = 0;
  // every warp runs nblk blocks (empty ones past its rows) so CTA barriers stay matched
  auto count_of = [&](int64_t b) -> int { return (int)max64(0, min64(BR, rend - (rbeg + b * BR))); };
  bool bulk = false, pending = false;
  if (count_of(0) > 0) {
    bulk = issue(rbeg, count_of(0));
    pending = true;
  }
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t r0 = rbeg + b * BR;
    const int cnt = count_of(b);
    if (kWlSync == 0 && cnt == 0) break;
    if (pending) {
      if (bulk) {
        mbar_wait_parity(bar, phase);
        phase ^= 1u;
      } else {
        cp_async_wait<0>();
      }
      pending = false;
    }
    __syncwarp();
    double xr[S][N];
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const int row = lane + 32 * q;
#pragma unroll
      for (int c = 0; c < N; ++c) xr[q][c] = row < cnt ? stg[row * ls + c] : 0.0;
    }
    if (stats && sph < kStatPhases) {  // lane: column scol, rows sph, sph + phases, ...
      double a0 = 0.0, a1 = 0.0, q0 = 0.0, q1 = 0.0;
      int row = sph;
      for (; row + kStatPhases < cnt; row += 2 * kStatPhases) {
        const double v0 = stg[row * ls + scol], v1 = stg[(row + kStatPhases) * ls + scol];
        a0 += fabs(v0);
        a1 += fabs(v1);
        q0 = fma(v0, v0, q0);
        q1 = fma(v1, v1, q1);
      }
      if (row < cnt) {
        const double v0 = stg[row * ls + scol];
        a0 += fabs(v0);
        q0 = fma(v0, v0, q0);
      }
      l1 += a0 + a1;
      sq += q0 + q1;
    }
    __syncwarp();  // the whole warp is done reading the stage buffer
    if (b + 1 < nblk && count_of(b + 1) > 0) {
      bulk = issue(r0 + BR, count_of(b + 1));
      pending = true;
    }
    // Column steps, straight-line code (N, j, c compile-time; no branches): lane c (j < c < N) owns
    // w_c = R(j, c) + sum over the block of v x[:, c].  Column j+1 is updated first; the remaining
    // columns' updates of step j are deferred into step j+1, behind its norm butterfly.
    double v_prev[S];
#pragma unroll
    for (int q = 0; q < S; ++q) v_prev[q] = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      if (kWlSync > 0 && j % (kWlSync > 0 ? kWlSync : 1) == 0) named_sync(1, blockDim.x);
      // Column sums of the product tile: the V = N-1-j live columns are covered by L = pow2ceil(V) lanes,
      // and the 32 rows split over the 32/L lane groups (L rows each), combined by a shuffle butterfly —
      // L loads per lane instead of 32.  Lane l: column j+1+(l % L), rows (l / L)*L ...
      const int L = pow2ceil(N - 1 - j);
      const int col = j + 1 + (lane & (L - 1));
      const int grow = (lane & ~(L - 1)) & 31;
      // R row j is only changed by reflector j, so R(j, .) is read up front (off the chain)
      const double rjc = Rs[wl_roff(N, j) + (col < N ? col : N - 1)];
      const double alpha = Rs[wl_roff(N, j) + j];
      double d = 0.0;
#pragma unroll
      for (int q = 0; q < S; ++q) d = fma(xr[q][j], xr[q][j], d);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
      // deferred updates of step j-1 (columns j+1 .. N-1; TW still holds step j-1's tau w), overlapping the
      // butterfly
      if (j > 0) {
        int c = j + 1;
        if (c & 1) {
          const double t = TW[c];
#pragma unroll
          for (int q = 0; q < S; ++q) xr[q][c] = fma(-t, v_prev[q], xr[q][c]);
          ++c;
        }
#pragma unroll
        for (; c < N; c += 2) {
          const double2 t = *reinterpret_cast<const double2*>(TW + c);  // TW has N + 1 (even-rounded) slots
#pragma unroll
          for (int q = 0; q < S; ++q) {
            xr[q][c] = fma(-t.x, v_prev[q], xr[q][c]);
            if (c + 1 < N) xr[q][c + 1] = fma(-t.y, v_prev[q], xr[q][c + 1]);
          }
        }
      }
      const bool live = d > 0.0;
      const double ss = live ? fma(alpha, alpha, d) : 1.0;
      const double inv = rsqrt_nb(ss);
      const double nrm = ss * inv;
      const double beta = live ? -copysign(nrm, alpha) : alpha;
      const double tau = live ? fma(fabs(alpha), inv, 1.0) : 0.0;
      const double scale = live ? copysign(rcp_nb(fabs(alpha) + nrm), alpha) : 0.0;
      double v[S];
#pragma unroll
      for (int q = 0; q < S; ++q) v[q] = xr[q][j] * scale;
      if (j + 1 < N) {
        // products p_c = sum_q v_q x_q[c] (this lane's rows) -> row `lane` of the product tile
        double* prow = P + lane * pld;
        int c = j + 1;
        if (c & 1) {
          double p = 0.0;
#pragma unroll
          for (int q = 0; q < S; ++q) p = fma(v[q], xr[q][c], p);
          prow[c] = p;
          ++c;
        }
#pragma unroll
        for (; c < N; c += 2) {
          double p0 = 0.0, p1 = 0.0;
#pragma unroll
          for (int q = 0; q < S; ++q) {
            p0 = fma(v[q], xr[q][c], p0);
            if (c + 1 < N) p1 = fma(v[q], xr[q][c + 1], p1);
          }
          if (c + 1 < N)
            *reinterpret_cast<double2*>(prow + c) = make_double2(p0, p1);
          else
            prow[c] = p0;
        }
        __syncwarp();
        // lanes whose column is >= N sum bytes they then discard (inside the CTA's shared memory)
        double sa[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int r = 0; r < L; ++r) sa[r & 3] += P[(grow + r) * pld + col];
        double sum = (sa[0] + sa[1]) + (sa[2] + sa[3]);
#pragma unroll
        for (int o = L; o < 32; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        const double tw = tau * (rjc + sum);
        if (lane < L && col < N) {
          Rs[wl_roff(N, j) + col] = rjc - tw;
          TW[col] = tw;
        }
      }
      if (lane == j) Rs[wl_roff(N, j) + j] = beta;
      if (j + 1 < N) {
        __syncwarp();
        // critical: the next pivot column now; the rest is deferred into step j+1
        const double t = TW[j + 1];
#pragma unroll
        for (int q = 0; q < S; ++q) xr[q][j + 1] = fma(-t, v[q], xr[q][j + 1]);
#pragma unroll
        for (int q = 0; q < S; ++q) v_prev[q] = v[q];
      }
    }
  }
  __syncwarp();
  if (leaf >= nleaves) return;
  P[lane] = l1;
  P[32 + lane] = sq;
  __syncwarp();
  double* R = slots + leaf * g.npad * g.npad;
  if (lane < g.npad) {
    for (int i = 0; i < g.npad; ++i)
      R[(int64_t)i * g.npad + lane] = (i < N && lane < N && i <= lane) ? Rs[wl_roff(N, i) + lane] : 0.0;
    if (stats) {
      double a = 0.0, q = 0.0;
      if (lane < N)
        for (int k = 0; k < kStatPhases; ++k) {
          a += P[k * N + lane];
          q += P[32 + k * N + lane];
        }
      stats[leaf * 2 * g.npad + lane] = a;
      stats[leaf * 2 * g.npad + g.npad + lane] = q;
    }
  }
}

// R_out (n x n, row-major, stride ldr) = sign-fixed upper triangle of slot 0 (tsqr.py:113-118).
__global__ void tsqr_finalize_kernel(const double* __restrict__ slot, int npad, int n, double* __restrict__ r,
                                     int64_t ldr) {
  const int i = blockIdx.x;
  const double sg = slot[(int64_t)i * npad + i] < 0.0 ? -1.0 : 1.0;
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    r[(int64_t)i * ldr + j] = (j >= i) ? sg * slot[(int64_t)i * npad + j] : 0.0;
}

// l1 / sumsq = fixed-order sum of per-CTA partials (deterministic).
__global__ void stats_reduce_kernel(const double* __restrict__ partials, int count, int stride, int n,
                                    double* __restrict__ l1, double* __restrict__ sumsq) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double a = 0.0, q = 0.0;
  for (int c = 0; c < count; ++c) {
    a += partials[(int64_t)c * 2 * stride + j];
    q += partials[(int64_t)c * 2 * stride + stride + j];
  }
  if (l1) l1[j] = a;
  if (sumsq) sumsq[j] = q;
}

// slot[c] = zero-padded copy of input factor c (n x n, row-major, contiguous).
__global__ void tsqr_pad_kernel(const double* __restrict__ rs, int n, int npad, double* __restrict__ slots) {
  const int64_t c = blockIdx.y;
  const int i = blockIdx.x;
  const double* src = rs + c * n * n + (int64_t)i * n;
  double* dst = slots + c * npad * npad + (int64_t)i * npad;
  for (int j = threadIdx.x; j < npad; j += blockDim.x) dst[j] = (i < n && j < n && j >= i) ? src[j] : 0.0;
}

// ---------------------------------------------------------------------------
// host side

namespace {

struct TqChoice {
  int rq;    // block rows per lane of the panel warp
  int minb;
  TqGeom g;
  size_t smem;
};

bool tq_choose(int n, int minb, TqChoice* out) {
  TqGeom g;
  g.n = n;
  g.npad = (int)round_up(n, kNB);
  g.lds = smem_stride(g.npad);
  const size_t budget = (minb == 3 ? 74 : (minb == 2 ? 113 : 226)) * 1024;
  int best = 0;
  // multiple of 16 (B -= V W' runs row-block pairs; 136 rows at n = 200 with an odd-block tail measured
  // slower, 228 vs 234 GB/s); above 128 rows (RQ = 5) only for the one-CTA build at n > 64, whose register
  // budget holds the fifth panel row (n = 128: 160 rows, 249 -> 270 GB/s)
  const int bmax = (minb == 1 && n > 64) ? 32 * kMaxRq : 128;
  for (int b = 16; b <= bmax; b += 16) {
    g.brows = b;
    if (TqLayout::bytes(g) <= budget) best = b;
  }
  if (!best) return false;
  g.brows = best;
  out->rq = (best + 31) / 32;
  if (out->rq > kMaxRq) return false;
  out->minb = minb;
  out->g = g;
  out->smem = TqLayout::bytes(g);
  return true;
}

bool tq_config(int n, TqChoice* out) {
  // Occupancy: the throughput is (rows in flight) / (n x per-column panel latency) per panel chain (see
  // DESIGN.md).  Narrow matrices (n <= 64) fit a full 128-row block in half the shared memory, so two CTAs
  // per SM give two independent panel chains (measured +50% at n = 25 and 64); wider ones run one CTA
  // with the largest block.  TSNMF_TSQR_CTAS=1/2/3 overrides for tuning.
  // n <= 104: three 4-warp CTAs per SM (three panel chains, 64-112-row blocks, 168 registers): measured
  // n=48 370 -> 476, n=64 355 -> 406 (vs two 8-warp CTAs, whose 128-register cap forces spills), n=72
  // 273 -> 388, n=96 272 -> 328 GB/s (vs one 8-warp CTA); n=128 is better with one CTA (270 vs 237)
  // (97..104: npad = 104, but the block stride lds (104) and rows (64) match n = 96's, so the same fit)
  int minb = n <= 104 ? 3 : 1;
  if (const char* e = getenv("TSNMF_TSQR_CTAS")) minb = atoi(e) == 3 ? 3 : (atoi(e) == 2 ? 2 : 1);
  if (minb == 3 && n <= 128 && tq_choose(n, 3, out) && out->g.brows >= 48) return true;
  if (minb >= 2 && tq_choose(n, 2, out) && out->g.brows >= (n <= 64 ? 128 : 48)) return true;
  return tq_choose(n, 1, out);
}

template <int RQ, int MINB>
int tq_launch_all(const TqChoice& ch, const double* x, int64_t m, int64_t ldx, double* slots, double* stats,
                  int nleaves, int64_t rows_per_cta, cudaStream_t st) {
  static PerDeviceFlag attr_set;
  if (!attr_set.is_set()) {
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(tsqr_leaf_kernel<RQ, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          232448));
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(tsqr_combine_kernel<RQ, MINB>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr_set.set();
  }
  if (x) {
    prof_mark(kProfTsqrLeaf, true, st);
    tsqr_leaf_kernel<RQ, MINB><<<nleaves, 32 * tq_warps<MINB>(), ch.smem, st>>>(x, m, ldx, rows_per_cta, ch.g, slots, stats);
    TSNMF_LAUNCH_CHECK();
    prof_mark(kProfTsqrLeaf, false, st);
  }
  prof_mark(kProfTsqrTree, true, st);
  // binary-counter tree (tsqr.py:213-230): perfect levels, then fold leftover subtrees low -> high
  for (int64_t span = 2; span <= nleaves; span *= 2) {
    const int64_t q = nleaves / span;
    tsqr_combine_kernel<RQ, MINB><<<(unsigned)q, 32 * tq_warps<MINB>(), ch.smem, st>>>(slots, span, span / 2, 0, 0, ch.g);
    TSNMF_LAUNCH_CHECK();
  }
  int64_t offs[64];
  int nsub = 0;
  int64_t o = 0;
  for (int b = 62; b >= 0; --b)
    if (nleaves & (1LL << b)) {
      offs[nsub++] = o;
      o += (1LL << b);
    }
  for (int t = nsub - 2; t >= 0; --t) {
    tsqr_combine_kernel<RQ, MINB><<<1, 32 * tq_warps<MINB>(), ch.smem, st>>>(slots, 0, 0, offs[t], offs[t + 1], ch.g);
    TSNMF_LAUNCH_CHECK();
  }
  prof_mark(kProfTsqrTree, false, st);
  return kOk;
}

template <int MINB>
int tq_dispatch_rq(const TqChoice& ch, const double* x, int64_t m, int64_t ldx, double* slots, double* stats,
                   int nleaves, int64_t rows_per_cta, cudaStream_t st) {
  switch (ch.rq) {
    case 1: return tq_launch_all<1, MINB>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
    case 2: return tq_launch_all<2, MINB>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
    case 3: return tq_launch_all<3, MINB>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
    case 4: return tq_launch_all<4, MINB>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
    default:
      if constexpr (MINB == 1) return tq_launch_all<5, 1>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
      return tq_launch_all<4, MINB>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
  }
}

int tq_dispatch(const TqChoice& ch, const double* x, int64_t m, int64_t ldx, double* slots, double* stats,
                int nleaves, int64_t rows_per_cta, cudaStream_t st) {
  if (ch.minb == 3) return tq_dispatch_rq<3>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
  if (ch.minb == 2) return tq_dispatch_rq<2>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
  return tq_dispatch_rq<1>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
}

int device_sms() {
  static std::atomic<int> sms_of[64];  // per device (0 = not queried yet)
  int dev = 0;
  cudaGetDevice(&dev);
  std::atomic<int>& slot = sms_of[dev & 63];
  int sms = slot.load(std::memory_order_relaxed);
  if (!sms) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = kNumSMs;
    slot.store(sms, std::memory_order_relaxed);
  }
  return sms;
}

void tq_plan(const TqChoice& ch, int64_t m, int* nleaves, int64_t* rows_per_cta) {
  const int64_t max_leaves = (int64_t)device_sms() * ch.minb;
  const int64_t min_rows = max64(ch.g.brows, 2 * (int64_t)ch.g.npad);
  int64_t leaves = max64(1, min64(max_leaves, ceil_div(m, min_rows)));
  int64_t rpc = ceil_div(m, leaves);
  rpc = round_up(rpc, ch.g.brows);
  leaves = ceil_div(m, rpc);
  *nleaves = (int)leaves;
  *rows_per_cta = rpc;
}

// Narrow leaves (n <= 32).  Default: the register-block warp leaf (tsqr_warp_leaf_kernel, 32*S-row blocks,
// CTA = one warp); TSNMF_TSQR_WARPLEAF=0 selects the 32-row warp-chain leaf (tsqr_small_leaf_kernel) and
// TSNMF_TSQR_SMALL=0 the shared-panel leaf.
bool small_path(int n) {
  if (n > 32) return false;
  if (const char* e = getenv("TSNMF_TSQR_SMALL")) return atoi(e) != 0;
  return true;
}
bool warp_leaf_path(int n) {
  if (!small_path(n)) return false;
  if (const char* e = getenv("TSNMF_TSQR_WARPLEAF")) return atoi(e) != 0;
  return true;
}
int small_nc(int n) { return n <= 8 ? 8 : (int)round_up(n, 4); }
// rows per lane: as many as the 255-register budget holds without spilling (x block = S * n doubles)
constexpr int warp_leaf_s_of(int n) { return n <= 20 ? 4 : (n <= 28 ? 3 : 2); }
int warp_leaf_s(int n) { return warp_leaf_s_of(n); }
WlGeom warp_leaf_geom(int n, int S) {
  WlGeom g;
  g.n = n;
  g.npad = (int)round_up(n, kNB);
  g.ls = (n & 1) ? n : n + 1;
  g.pld = n + 1;
  while (g.pld % 4 != 2) ++g.pld;
  g.stage_off = 2;  // [0, 2): mbarrier
  g.prod_off = g.stage_off + (int)round_up(32 * S * g.ls, 2);
  g.r_off = g.prod_off + (int)round_up(32 * g.pld, 2);
  g.tw_off = g.r_off + (int)round_up(n * (n + 1) / 2, 2);  // R packed upper triangle
  g.total = g.tw_off + (int)round_up(n + 1, 2);
  return g;
}
// warp leaves per CTA (one CTA per SM): shared memory (227 KB per CTA) and registers (<= 255 per thread
// -> 8 warps)
int warp_leaf_per_sm(const WlGeom& g) {
  const int bytes = (int)sizeof(double) * g.total;
  int k = (227 * 1024) / bytes;
  return k < 1 ? 1 : (k > 8 ? 8 : k);
}
void warp_leaf_plan(int n, int64_t m, int* nleaves, int64_t* rows_per_warp) {
  const int S = warp_leaf_s(n);
  const int64_t br = 32 * S;
  const int64_t max_leaves = (int64_t)device_sms() * warp_leaf_per_sm(warp_leaf_geom(n, S));
  int64_t leaves = max64(1, min64(max_leaves, ceil_div(m, br)));
  const int64_t rpw = round_up(ceil_div(m, leaves), br);
  *nleaves = (int)ceil_div(m, rpw);
  *rows_per_warp = rpw;
}

// Warp-chain leaf plan: one chain per warp, 3 CTAs x 4 warps per SM, 32-row blocks.
void small_plan(int64_t m, int* nleaves, int64_t* rows_per_warp) {
  const int64_t max_leaves = (int64_t)device_sms() * 3 * kSmWarps;
  int64_t leaves = max64(1, min64(max_leaves, ceil_div(m, 32)));
  const int64_t rpw = round_up(ceil_div(m, leaves), 32);
  leaves = round_up(ceil_div(m, rpw), kSmWarps);  // whole CTAs; surplus warps contribute zero factors
  *nleaves = (int)leaves;
  *rows_per_warp = rpw;
}

void narrow_plan(int n, int64_t m, int* nleaves, int64_t* rows_per_warp) {
  if (warp_leaf_path(n))
    warp_leaf_plan(n, m, nleaves, rows_per_warp);
  else
    small_plan(m, nleaves, rows_per_warp);
}

// binary-counter tree over the narrow leaves (tsqr.py:213-230): perfect levels, then fold leftover subtrees
// low -> high
template <int NC>
int small_tree(int n, int nleaves, int npad, double* slots, cudaStream_t st) {
  prof_mark(kProfTsqrTree, true, st);
  for (int64_t span = 2; span <= nleaves; span *= 2) {
    const int64_t pairs = nleaves / span;
    tsqr_small_combine_kernel<NC><<<(unsigned)ceil_div(pairs, kSmWarps), 32 * kSmWarps, SmallLayout<NC>::bytes, st>>>(
        slots, npad, n, span, span / 2, pairs, 0, 0);
    TSNMF_LAUNCH_CHECK();
  }
  int64_t offs[64];
  int nsub = 0;
  int64_t o = 0;
  for (int b = 62; b >= 0; --b)
    if ((int64_t)nleaves & (1LL << b)) {
      offs[nsub++] = o;
      o += (1LL << b);
    }
  for (int t = nsub - 2; t >= 0; --t) {
    tsqr_small_combine_kernel<NC><<<1, 32, SmallLayout<NC>::bytes, st>>>(slots, npad, n, 0, 0, 0, offs[t], offs[t + 1]);
    TSNMF_LAUNCH_CHECK();
  }
  prof_mark(kProfTsqrTree, false, st);
  return kOk;
}

template <int N>
int warp_leaf_launch(const double* x, int64_t m, int64_t ldx, int64_t rpw, int nleaves, double* slots, double* stats,
                     cudaStream_t st) {
  constexpr int S = warp_leaf_s_of(N);
  const WlGeom g = warp_leaf_geom(N, S);
  const int w = warp_leaf_per_sm(g);
  const int bytes = (int)sizeof(double) * g.total * w;
  TSNMF_CUDA_CHECK(
      cudaFuncSetAttribute(tsqr_warp_leaf_kernel<N, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  prof_mark(kProfTsqrLeaf, true, st);
  tsqr_warp_leaf_kernel<N, S><<<(unsigned)ceil_div(nleaves, w), 32 * w, bytes, st>>>(x, m, ldx, rpw, nleaves, g,
                                                                                      slots, stats);
  TSNMF_LAUNCH_CHECK();
  prof_mark(kProfTsqrLeaf, false, st);
  return small_tree<(N <= 8 ? 8 : (N + 3) / 4 * 4)>(N, nleaves, g.npad, slots, st);
}

template <int... Ns>
int warp_leaf_exact(int n, const double* x, int64_t m, int64_t ldx, int64_t rpw, int nleaves, double* slots,
                    double* stats, cudaStream_t st, std::integer_sequence<int, Ns...>) {
  int rc = kUsage;
  ((n == Ns + 1 ? (rc = warp_leaf_launch<Ns + 1>(x, m, ldx, rpw, nleaves, slots, stats, st), 0) : 0), ...);
  return rc;
}

// one instantiation per width (the column loop is straight-line code in n)
int warp_leaf(const double* x, int64_t m, int n, int64_t ldx, int64_t rpw, int nleaves, double* slots, double* stats,
              cudaStream_t st) {
  return warp_leaf_exact(n, x, m, ldx, rpw, nleaves, slots, stats, st, std::make_integer_sequence<int, 32>{});
}

template <int NC>
int small_launch(const double* x, int64_t m, int n, int64_t ldx, int64_t rpw, int nleaves, int npad, double* slots,
                 double* stats, cudaStream_t st) {
  static PerDeviceFlag attr;
  if (!attr.is_set()) {
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(tsqr_small_leaf_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)SmallLayout<NC>::bytes));
    attr.set();
  }
  prof_mark(kProfTsqrLeaf, true, st);
  tsqr_small_leaf_kernel<NC><<<nleaves / kSmWarps, 32 * kSmWarps, SmallLayout<NC>::bytes, st>>>(
      x, m, n, ldx, rpw, npad, slots, stats);
  TSNMF_LAUNCH_CHECK();
  prof_mark(kProfTsqrLeaf, false, st);
  return small_tree<NC>(n, nleaves, npad, slots, st);
}

int small_leaf(const double* x, int64_t m, int n, int64_t ldx, int64_t rpw, int nleaves, int npad, double* slots,
               double* stats, cudaStream_t st) {
  // register width NC = n rounded up to 4 (the work per column is proportional to NC - j)
  switch ((n + 3) / 4) {
    case 1:
    case 2: return small_launch<8>(x, m, n, ldx, rpw, nleaves, npad, slots, stats, st);
    case 3: return small_launch<12>(x, m, n, ldx, rpw, nleaves, npad, slots, stats, st);
    case 4: return small_launch<16>(x, m, n, ldx, rpw, nleaves, npad, slots, stats, st);
    case 5: return small_launch<20>(x, m, n, ldx, rpw, nleaves, npad, slots, stats, st);
    case 6: return small_launch<24>(x, m, n, ldx, rpw, nleaves, npad, slots, stats, st);
    case 7: return small_launch<28>(x, m, n, ldx, rpw, nleaves, npad, slots, stats, st);
    default: return small_launch<32>(x, m, n, ldx, rpw, nleaves, npad, slots, stats, st);
  }
}

// Split leaf (256-row blocks, right column tiles in an L2 workspace): 105 <= n <= 208 (14..26 panels, so
// the shared half holds <= 13 tiles); TSNMF_TSQR_SPLIT=0 selects the 128/160-row leaf.
bool split_path(int n) {
  if (n < 105 || n > 208) return false;
  if (const char* e = getenv("TSNMF_TSQR_SPLIT")) return atoi(e) != 0;
  return true;
}
size_t split_smem(const SplitGeom& sg) { return TqLayout::bytes(split_tq_geom(sg)) + sizeof(double) * 2 * sg.wld; }  // + right-tile stats
// as many shared slots as fit (fewer workspace tiles); at least half the tiles so every right tile t has
// its own slot t - S to move into
SplitGeom split_geom(int n) {
  SplitGeom sg;
  sg.n = n;
  sg.npad = (int)round_up(n, kNB);
  const int np = sg.npad / kNB;
  for (int S = np; S >= (np + 1) / 2; --S) {
    sg.S = S;
    sg.lds = smem_stride(8 * S);
    sg.wld = 8 * (np - S);
    if (split_smem(sg) <= 232448 - 1024 || S == (np + 1) / 2) break;
  }
  return sg;
}
void split_plan(int n, int64_t m, int* nleaves, int64_t* rows_per_cta) {
  const int64_t npad = round_up(n, kNB);
  const int64_t max_leaves = device_sms();
  const int64_t min_rows = max64(kSplitRows, 2 * npad);
  int64_t leaves = max64(1, min64(max_leaves, ceil_div(m, min_rows)));
  int64_t rpc = round_up(ceil_div(m, leaves), kSplitRows);
  *nleaves = (int)ceil_div(m, rpc);
  *rows_per_cta = rpc;
}
// workspace after the R slots and stats: the right tiles (nleaves x 256 x wld, tile-major)
size_t split_ws_doubles(const SplitGeom& sg, int nleaves) { return (size_t)nleaves * kSplitRows * sg.wld; }

int split_leaf(const double* x, int64_t m, int64_t ldx, const SplitGeom& sg, int nleaves, int64_t rpc,
               double* slots, double* stats, double* wsr, cudaStream_t st) {
  static PerDeviceFlag attr;
  const size_t smem = split_smem(sg);
  if (!attr.is_set()) {
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(tsqr_split_leaf_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr.set();
  }
  prof_mark(kProfTsqrLeaf, true, st);
  tsqr_split_leaf_kernel<<<nleaves, 256, smem, st>>>(x, m, ldx, rpc, sg, slots, stats, wsr);
  TSNMF_LAUNCH_CHECK();
  prof_mark(kProfTsqrLeaf, false, st);
  return kOk;
}

// Register-block leaf with DMMA trailing updates (tsqr_reg.cu, widths 25..64): the default for 28 <= n <= 64
// (measured against the older leaves at 2^25 rows, tools/reg_leaf_sweep.py: n = 28 866 vs 783 GB/s, n = 32 872 vs
// 639, n = 40 785 vs 521, n = 48 592 vs 515, n = 64 497 vs 434; n = 25..27 stay with the exact-width warp leaf,
// n = 25 814 vs 1146).  TSNMF_TSQR_REGLEAF=1/0 forces it / the older leaves.
bool reg_leaf_path(int n) {
  if (!tsqr_reg_supported(n)) return false;
  if (const char* e = getenv("TSNMF_TSQR_REGLEAF")) return atoi(e) != 0;
  return TSNMF_TSQR_REGLEAF_DEFAULT != 0 && n >= 28;
}
void reg_leaf_plan(int n, int64_t m, int* nleaves, int64_t* rows_per_warp) {
  const int64_t br = tsqr_reg_block_rows(n);
  const int64_t max_leaves = (int64_t)device_sms() * tsqr_reg_warps_per_cta();
  const int64_t leaves = max64(1, min64(max_leaves, ceil_div(m, br)));
  const int64_t rpw = round_up(ceil_div(m, leaves), br);
  *nleaves = (int)ceil_div(m, rpw);
  *rows_per_warp = rpw;
}

}  // namespace

int tsqr_max_cols() { return 512; }

#ifdef TSNMF_TRACE
extern "C" int tsnmf_trace_read(long long* out, int cap) {
  // out: 8 warps x 4096 slots (panel * 64 + tag) of clock64 values, 0 = not recorded
  const int n = 8 * 64 * 64 < cap ? 8 * 64 * 64 : cap;
  cudaMemcpyFromSymbol(out, g_trace, sizeof(long long) * n);
  static long long zero[8 * 64 * 64];
  cudaMemcpyToSymbol(g_trace, zero, sizeof(zero));
  return n;
}
#endif

size_t tsqr_workspace_bytes(int64_t m, int n) {
  TqChoice ch;
  if (n < 1 || !tq_config(n, &ch)) return 0;
  int nleaves;
  int64_t rpc;
  size_t extra = 0;
  if (reg_leaf_path(n)) {
    reg_leaf_plan(n, max64(m, 1), &nleaves, &rpc);
  } else if (small_path(n)) {
    narrow_plan(n, max64(m, 1), &nleaves, &rpc);
  } else if (split_path(n)) {
    split_plan(n, max64(m, 1), &nleaves, &rpc);
    extra = split_ws_doubles(split_geom(n), nleaves);
  } else {
    tq_plan(ch, max64(m, 1), &nleaves, &rpc);
  }
  const int64_t npad = ch.g.npad;
  return sizeof(double) * ((size_t)(nleaves * npad * npad + nleaves * 2 * npad) + extra) + 256;
}

size_t combine_workspace_bytes(int count, int n) {
  TqChoice ch;
  if (n < 1 || count < 1 || !tq_config(n, &ch)) return 0;
  const int64_t npad = ch.g.npad;
  return sizeof(double) * (size_t)(count * npad * npad) + 256;
}

int tsqr_run(const double* x, int64_t m, int n, int64_t ldx, double* r, int64_t ldr, double* l1, double* sumsq,
             void* ws, size_t ws_bytes, cudaStream_t st) {
  TqChoice ch;
  if (!tq_config(n, &ch)) return set_error(kUsage, "tsqr: n = %d columns does not fit the on-chip block", n);
  int nleaves;
  int64_t rpc;
  const bool reg = reg_leaf_path(n);
  const bool narrow = !reg && small_path(n);
  const bool split = !reg && !narrow && split_path(n);
  size_t extra = 0;
  if (reg) {
    reg_leaf_plan(n, m, &nleaves, &rpc);
  } else if (narrow) {
    narrow_plan(n, m, &nleaves, &rpc);
  } else if (split) {
    split_plan(n, m, &nleaves, &rpc);
    extra = split_ws_doubles(split_geom(n), nleaves);
  } else {
    tq_plan(ch, m, &nleaves, &rpc);
  }
  const int64_t npad = ch.g.npad;
  const size_t need = sizeof(double) * ((size_t)(nleaves * npad * npad + nleaves * 2 * npad) + extra);
  if (ws_bytes < need) return set_error(kUsage, "tsqr: workspace too small (%zu < %zu bytes)", ws_bytes, need);
  double* slots = reinterpret_cast<double*>(ws);
  double* stats = slots + (int64_t)nleaves * npad * npad;
  const bool want_stats = (l1 != nullptr) || (sumsq != nullptr);
  int rc;
  if (reg) {
    rc = tsqr_reg_leaf_run(x, m, ldx, n, rpc, nleaves, (int)npad, slots, want_stats ? stats : nullptr, st);
    if (!rc) {
      if (n <= 32)
        rc = n <= 28 ? small_tree<28>(n, nleaves, (int)npad, slots, st) : small_tree<32>(n, nleaves, (int)npad, slots, st);
      else
        rc = tq_dispatch(ch, nullptr, 0, 0, slots, nullptr, nleaves, 0, st);
    }
  } else if (narrow && warp_leaf_path(n)) {
    rc = warp_leaf(x, m, n, ldx, rpc, nleaves, slots, want_stats ? stats : nullptr, st);
  } else if (narrow) {
    rc = small_leaf(x, m, n, ldx, rpc, nleaves, (int)npad, slots, want_stats ? stats : nullptr, st);
  } else if (split) {
    double* wsr = stats + (int64_t)nleaves * 2 * npad;
    rc = split_leaf(x, m, ldx, split_geom(n), nleaves, rpc, slots, want_stats ? stats : nullptr, wsr, st);
    if (!rc) rc = tq_dispatch(ch, nullptr, 0, 0, slots, nullptr, nleaves, 0, st);  // the combine tree
  } else {
    rc = tq_dispatch(ch, x, m, ldx, slots, want_stats ? stats : nullptr, nleaves, rpc, st);
  }
  if (rc) return rc;
  tsqr_finalize_kernel<<<n, 128, 0, st>>>(slots, (int)npad, n, r, ldr);
  TSNMF_LAUNCH_CHECK();
  if (want_stats) {
    stats_reduce_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(stats, nleaves, (int)npad, n, l1, sumsq);
    TSNMF_LAUNCH_CHECK();
  }
  return kOk;
}

int r_combine_run(const double* rs, int count, int n, double* r, int64_t ldr, void* ws, size_t ws_bytes,
                  cudaStream_t st) {
  TqChoice ch;
  if (!tq_config(n, &ch)) return set_error(kUsage, "combine: n = %d columns does not fit the on-chip block", n);
  const int64_t npad = ch.g.npad;
  const size_t need = sizeof(double) * (size_t)(count * npad * npad);
  if (ws_bytes < need) return set_error(kUsage, "combine: workspace too small (%zu < %zu bytes)", ws_bytes, need);
  double* slots = reinterpret_cast<double*>(ws);
  tsqr_pad_kernel<<<dim3((unsigned)npad, (unsigned)count), 128, 0, st>>>(rs, n, (int)npad, slots);
  TSNMF_LAUNCH_CHECK();
  int rc = tq_dispatch(ch, nullptr, 0, 0, slots, nullptr, count, 0, st);
  if (rc) return rc;
  tsqr_finalize_kernel<<<n, 128, 0, st>>>(slots, (int)npad, n, r, ldr);
  TSNMF_LAUNCH_CHECK();
  return kOk;
}

int tsqr_describe(int n, int64_t m, int* nb, int* brows, int* ctas_per_sm, int* nleaves) {
  TqChoice ch;
  if (!tq_config(n, &ch)) return set_error(kUsage, "tsqr: n = %d too large", n);
  int64_t rpc;
  if (reg_leaf_path(n)) {  // register-block leaf with DMMA trailing updates: one warp per leaf
    reg_leaf_plan(n, max64(m, 1), nleaves, &rpc);
    *nb = kNB;
    *brows = tsqr_reg_block_rows(n);
    *ctas_per_sm = 1;
    return kOk;
  }
  if (warp_leaf_path(n)) {  // register-block warp leaf: "panel" 1 column, 32*S-row blocks, one warp per CTA
    warp_leaf_plan(n, max64(m, 1), nleaves, &rpc);
    const int S = warp_leaf_s(n);
    *nb = 1;
    *brows = 32 * S;
    *ctas_per_sm = warp_leaf_per_sm(warp_leaf_geom(n, S));
    return kOk;
  }
  if (small_path(n)) {  // warp-per-chain leaf: "panel" 1 column, 32-row blocks, 3 CTAs (12 chains) per SM
    small_plan(max64(m, 1), nleaves, &rpc);
    *nb = 1;
    *brows = 32;
    *ctas_per_sm = 3;
    return kOk;
  }
  if (split_path(n)) {  // split leaf: 256-row blocks, one CTA per SM
    split_plan(n, max64(m, 1), nleaves, &rpc);
    *nb = kNB;
    *brows = kSplitRows;
    *ctas_per_sm = 1;
    return kOk;
  }
  tq_plan(ch, max64(m, 1), nleaves, &rpc);
  *nb = kNB;
  *brows = ch.g.brows;
  *ctas_per_sm = ch.minb;
  return kOk;
}

}  // namespace tsnmf

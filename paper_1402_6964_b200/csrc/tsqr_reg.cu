// TSQR register-block leaf with tensor-core trailing updates (narrow matrices, e.g. config C4 n = 25 and C5
// n = 64).  Same mathematics and outputs as the other leaves of tsqr.cu (reference pkg/src/tsnmf/tsqr.py:129-141
// factor_chunk, :184-198 _StatsAcc): each WARP owns a contiguous row range and its own R, folds 8 NT-row
// blocks into it by the structured blocked Householder QR of [R; B] (reflector j = [e_j; v]), and the per-warp
// R's are combined afterwards by the TreeReducer-order combine kernels.
//
// What is new is where the block lives: in the warp's registers, in a layout chosen so that the DMMA trailing
// update never moves it.  Lane (kr = l % 4, cj = l / 4) holds, for row tile t, column tile T and h in {0, 1},
//     B[t][h][T] = block(8 t + 2 kr + h, 8 T + cj).
//   * W = R_p + V^T B (mma.m8n8k4, D[i][c] += A[i][k] Bop[k][c]): a k-step is the row quadruple
//     {8 t + 2 kr + h : kr = 0..3}; A[i][k] = V(row_k, i) is the lane's own register of the panel's column tile,
//     Bop[k][c] = B(row_k, c) its register of the trailing column tile (the order of the rows inside the sum
//     is free, so this pairing of rows with k indices is as good as any).
//   * B -= V W' is issued transposed, B^T -= W'^T V^T: D[c][rho] with D's two columns 2 kr + {0, 1} is exactly
//     (B[t][0][T], B[t][1][T]); A = -W'^T comes from a 64-double scratch tile, Bop = V^T from the panel's
//     reflectors, which are written to shared memory once per panel (8 NT x 8 doubles).
// So a trailing column tile costs 4 NT + 2 DMMAs and no loads or stores of the block at all.
// The panel (8 columns) runs all its columns' dot products at once: the pivot column is broadcast through
// shared memory, every lane group (cj) forms the dot with its own column (2 NT FMAs + two shuffles), the
// reflector scalars are computed redundantly by every lane (dlarfg conventions, as panel_factor_lazy in
// tsqr.cu), and each group updates its own column.  T (compact WY) is built from the same dots.
// R lives in shared memory as upper 8 x 8 tiles (tile-major), the block is loaded straight from global
// memory (each fragment an 8-byte load; 64 loads in flight per lane), column l1 / sum of squares from the
// loaded registers.
#include "common.cuh"
#include "internal.h"

namespace tsnmf {

constexpr int kRgWarps = 8;
#ifndef TSNMF_RG_SCALE_FROM_TAU
#define TSNMF_RG_SCALE_FROM_TAU 1
#endif

template <int TCN, int NT>
struct RgLayout {
  static constexpr int BR = 8 * NT;                       // rows per block
  static constexpr int NTILES = TCN * (TCN + 1) / 2;      // upper 8 x 8 tiles of R
  static constexpr int BRS = BR + (20 - BR % 16) % 16;    // column stride of XC, = 4 (mod 16): conflict-free V^T reads
  static constexpr int r_off = 0;
  static constexpr int x_off = r_off + NTILES * 64;       // XC: the panel's 8 pivot columns as broadcast (unscaled)
  static constexpr int w_off = x_off + 8 * BRS;           // W / W' scratch tiles (2 x 8 x 8: two trailing tiles per round)
  static constexpr int t_off = w_off + 128;               // T (8 x 8, row r = reflector r)
  static constexpr int d_off = t_off + 64;                // the step's dots (8)
  static constexpr int total = d_off + 8;
  static constexpr size_t bytes = sizeof(double) * (size_t)total * kRgWarps;
};

__host__ __device__ constexpr int rg_tile(int tcn, int I, int J) { return I * tcn - I * (I - 1) / 2 + (J - I); }

template <int TCN, int NT, bool kKeep>
__global__ void __launch_bounds__(32 * kRgWarps, 1)
    tsqr_reg_leaf_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, int n, int64_t rows_per_warp,
                         int nleaves, int npad, double* __restrict__ slots, double* __restrict__ stats) {
  using L = RgLayout<TCN, NT>;
  constexpr int BR = L::BR, BRS = L::BRS;
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int kr = lane & 3, cj = lane >> 2;
  double* base = smem + (size_t)wib * L::total;
  double* Rt = base + L::r_off;
  double* XC = base + L::x_off;
  double* Wsc = base + L::w_off;
  double* Tm = base + L::t_off;
  double* db = base + L::d_off;
  const int64_t leaf = (int64_t)blockIdx.x * kRgWarps + wib;
  const int64_t rbeg = leaf * rows_per_warp;
  const int64_t rend = min64(m, rbeg + rows_per_warp);
  for (int i = lane; i < L::NTILES * 64; i += 32) Rt[i] = 0.0;
  __syncwarp();

  double B[NT][2][TCN];
  double sa[TCN], sq[TCN];
#pragma unroll
  for (int T = 0; T < TCN; ++T) sa[T] = sq[T] = 0.0;
  const int ci = (lane >> 2) * 8 + 2 * (lane & 3);  // C-layout index of this lane in an 8 x 8 tile

  for (int64_t r0 = rbeg; r0 < rend; r0 += BR) {
    // ---- load the block (zero past the range / the last column) and its column statistics
    {
      const double* p = x + (r0 + 2 * kr) * ldx + cj;
      const bool full = r0 + BR <= rend;
#pragma unroll
      for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const bool rok = full || r0 + 8 * t + 2 * kr + h < rend;
#pragma unroll
          for (int T = 0; T < TCN; ++T)
            B[t][h][T] = (rok && 8 * T + cj < n) ? __ldg(p + (int64_t)(8 * t + h) * ldx + 8 * T) : 0.0;
        }
      if (r0 + BR < rend) {  // next block into L2 while this one is folded
        const char* q = reinterpret_cast<const char*>(x + (r0 + BR + lane) * ldx);
        for (int rr = lane; rr < BR && r0 + BR + rr < rend; rr += 32) {
          for (int o = 0; o < 8 * n; o += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(q + o));
          q += 32 * 8 * ldx;
        }
      }
#pragma unroll
      for (int T = 0; T < TCN; ++T) {
        double a = 0.0, s = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            a += fabs(B[t][h][T]);
            s = fma(B[t][h][T], B[t][h][T], s);
          }
        sa[T] += a;
        sq[T] += s;
      }
    }
#pragma unroll
    for (int Tp = 0; Tp < TCN; ++Tp) {
      if (8 * Tp >= n) break;
      double* Rd = Rt + rg_tile(TCN, Tp, Tp) * 64;
      const int jmax = min(8, n - 8 * Tp);
      // ---- panel: columns 8 Tp .. 8 Tp + jmax - 1, one Householder reflector each.  Column j is broadcast
      // through XC[j] (written by its lane group right after its update in step j - 1) and stays there, UNSCALED,
      // as the reflector's vector: v_j = scale_j XC[j].  The scale lives in the owning lanes (myscale) and is
      // folded into the 8 x 8 matrices instead of the block: W = R_p + D (Xc^T B), B -= Xc (D W').
      double trow[8];  // lanes 0..7: row `lane` of T
#pragma unroll
      for (int c = 0; c < 8; ++c) trow[c] = 0.0;
      double myscale = 0.0;
      if (cj == 0) {
#pragma unroll
        for (int t = 0; t < NT; ++t)
          *reinterpret_cast<double2*>(XC + 8 * t + 2 * kr) = make_double2(B[t][0][Tp], B[t][1][Tp]);
      }
      if (jmax < 8) {  // zero-padded columns: zero vectors (their reflectors do nothing)
        for (int i = lane; i < BRS * (8 - jmax); i += 32) XC[jmax * BRS + i] = 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j < jmax) {
          const double* xcur = XC + j * BRS;
          __syncwarp();
          double xj[kKeep ? NT : 1][2];
          double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            const double2 v = *reinterpret_cast<const double2*>(xcur + 8 * t + 2 * kr);
            if (kKeep) {
              xj[t][0] = v.x;
              xj[t][1] = v.y;
            }
            if (t & 1) {
              d2 = fma(v.x, B[t][0][Tp], d2);
              d3 = fma(v.y, B[t][1][Tp], d3);
            } else {
              d0 = fma(v.x, B[t][0][Tp], d0);
              d1 = fma(v.y, B[t][1][Tp], d1);
            }
          }
          double d = (d0 + d1) + (d2 + d3);
          d += __shfl_xor_sync(0xffffffffu, d, 1);
          d += __shfl_xor_sync(0xffffffffu, d, 2);
          if (kr == 0) db[cj] = cj < j ? d * myscale : d;  // x_j . v_q for the finished columns q < j
          __syncwarp();
          double dv[8];
#pragma unroll
          for (int c = 0; c < 8; c += 2) {
            const double2 v = *reinterpret_cast<const double2*>(db + c);
            dv[c] = v.x;
            dv[c + 1] = v.y;
          }
          // T[r][j] = -tau_j sum_{q=r}^{j-1} T[r][q] (v_q . v_j),  v_q . v_j = scale_j dv[q]  (sum formed beside
          // the scalar chain)
          double tacc = 0.0;
#pragma unroll
          for (int q = 0; q < j; ++q) tacc = fma(trow[q], dv[q], tacc);
          // reflector scalars (every lane; dlarfg conventions as panel_factor_lazy)
          const double sigma = dv[j];
          const double alpha = Rd[j * 8 + j];
          const double rjc = Rd[j * 8 + cj];
          const bool live = sigma > 0.0;
          const double ss = live ? fma(alpha, alpha, sigma) : 1.0;
// (rsqrt_nb's range scaling stays: a uniform fast-path branch around it splits the step's basic block and
          // costs far more than the three multiplies it saves — n = 40 804 -> 625 GB/s)
          const double inv = rsqrt_nb(ss);
          const double nrm = ss * inv;
          const double beta = live ? -copysign(nrm, alpha) : alpha;
          const double tau = live ? fma(fabs(alpha), inv, 1.0) : 0.0;
#if TSNMF_RG_SCALE_FROM_TAU
          // 1 / (|alpha| + nrm) = inv / tau with tau in [1, 2]: the reciprocal needs no range scaling and starts
          // from inv, not from nrm
          double rt;
          asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rt) : "d"(tau));
          rt = rt * fma(-tau, rt, 2.0);
          rt = rt * fma(-tau, rt, 2.0);
          const double scale = live ? copysign(inv * rt, alpha) : 0.0;
#else
          const double scale = live ? copysign(rcp_nb(fabs(alpha) + nrm), alpha) : 0.0;
#endif
          const double tw = tau * fma(scale, d, rjc);
          const double f = cj > j ? tw * scale : 0.0;
          // straight-line, predicated (f = 0 for the finished and the pivot columns): a divergent branch here
          // would split the step's basic block, which the scheduler needs whole to hide the scalar chain
          {
            const bool nxt = cj == j + 1;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              double2 v;
              if (kKeep)
                v = make_double2(xj[t][0], xj[t][1]);
              else
                v = *reinterpret_cast<const double2*>(xcur + 8 * t + 2 * kr);
              B[t][0][Tp] = fma(-f, v.x, B[t][0][Tp]);
              B[t][1][Tp] = fma(-f, v.y, B[t][1][Tp]);
              if (nxt)
                *reinterpret_cast<double2*>(XC + (j + 1) * BRS + 8 * t + 2 * kr) = make_double2(B[t][0][Tp], B[t][1][Tp]);
            }
            if (kr == 0 && cj >= j) Rd[j * 8 + cj] = cj == j ? beta : rjc - tw;
            myscale = cj == j ? scale : myscale;
          }
          trow[j] = lane == j ? tau : (lane < j ? -tau * scale * tacc : 0.0);
        }
      }
      if (lane < 8) {
#pragma unroll
        for (int c = 0; c < 8; ++c) Tm[lane * 8 + c] = trow[c];
      }
      __syncwarp();
      // ---- trailing column tiles: W = R_p + D Xc^T B; W' = T^T W; R_p -= W'; B -= Xc (D W').  Two tiles per
      // round (independent DMMA chains, one set of warp barriers and one set of V^T fragment loads for both).
#pragma unroll
      for (int Tc = Tp + 1; Tc < TCN; Tc += 2) {
        if (8 * Tc >= n) break;
        const bool two = Tc + 1 < TCN;  // (TCN = ceil(n / 8): every tile column below TCN holds real columns)
        const int Td = Tc + 1 < TCN ? Tc + 1 : Tc;  // second tile (static index; == Tc when there is none)
        double* Rp = Rt + rg_tile(TCN, Tp, Tc) * 64;
        double* Rq = Rt + rg_tile(TCN, Tp, Td) * 64;
        double* Wsd = Wsc + 64;
        const double2 rinit = *reinterpret_cast<const double2*>(Rp + ci);
        const double2 qinit = *reinterpret_cast<const double2*>(Rq + ci);
        double a00 = 0.0, a01 = 0.0, a10 = 0.0, a11 = 0.0, b00 = 0.0, b01 = 0.0, b10 = 0.0, b11 = 0.0;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          dmma(a00, a01, B[t][0][Tp], B[t][0][Tc]);
          dmma(a10, a11, B[t][1][Tp], B[t][1][Tc]);
          if (two) {
            dmma(b00, b01, B[t][0][Tp], B[t][0][Td]);
            dmma(b10, b11, B[t][1][Tp], B[t][1][Td]);
          }
        }
        Wsc[ci] = fma(myscale, a00 + a10, rinit.x);  // this lane's tile row i = cj: its own group's scale
        Wsc[ci + 1] = fma(myscale, a01 + a11, rinit.y);
        if (two) {
          Wsd[ci] = fma(myscale, b00 + b10, qinit.x);
          Wsd[ci + 1] = fma(myscale, b01 + b11, qinit.y);
        }
        __syncwarp();
        double w0 = 0.0, w1 = 0.0, u0 = 0.0, u1 = 0.0;
#pragma unroll
        for (int k0 = 0; k0 < 8; k0 += 4) {
          const double tf = Tm[(k0 + (lane & 3)) * 8 + (lane >> 2)];
          dmma(w0, w1, tf, Wsc[(k0 + (lane & 3)) * 8 + (lane >> 2)]);
          if (two) dmma(u0, u1, tf, Wsd[(k0 + (lane & 3)) * 8 + (lane >> 2)]);
        }
        *reinterpret_cast<double2*>(Rp + ci) = make_double2(rinit.x - w0, rinit.y - w1);
        if (two) *reinterpret_cast<double2*>(Rq + ci) = make_double2(qinit.x - u0, qinit.y - u1);
        __syncwarp();
        Wsc[ci] = w0 * myscale;
        Wsc[ci + 1] = w1 * myscale;
        if (two) {
          Wsd[ci] = u0 * myscale;
          Wsd[ci + 1] = u1 * myscale;
        }
        __syncwarp();
        const double wb0 = -Wsc[(lane & 3) * 8 + (lane >> 2)];
        const double wb1 = -Wsc[(4 + (lane & 3)) * 8 + (lane >> 2)];
        const double wd0 = two ? -Wsd[(lane & 3) * 8 + (lane >> 2)] : 0.0;
        const double wd1 = two ? -Wsd[(4 + (lane & 3)) * 8 + (lane >> 2)] : 0.0;
        __syncwarp();
#pragma unroll
        for (int t = 0; t < NT; ++t) {
          const double v0 = XC[(lane & 3) * BRS + 8 * t + (lane >> 2)];
          const double v1 = XC[(4 + (lane & 3)) * BRS + 8 * t + (lane >> 2)];
          dmma(B[t][0][Tc], B[t][1][Tc], wb0, v0);
          if (two) dmma(B[t][0][Td], B[t][1][Td], wd0, v0);
          dmma(B[t][0][Tc], B[t][1][Tc], wb1, v1);
          if (two) dmma(B[t][0][Td], B[t][1][Td], wd1, v1);
        }
      }
    }
  }
  __syncwarp();
  if (leaf >= nleaves) return;
  // ---- R (upper tiles) -> the leaf's npad x npad slot; column statistics
  double* R = slots + leaf * (int64_t)npad * npad;
  for (int i = lane; i < npad * npad; i += 32) {
    const int r = i / npad, c = i - r * npad;
    double v = 0.0;
    if (r <= c && c < n) v = Rt[rg_tile(TCN, r >> 3, c >> 3) * 64 + (r & 7) * 8 + (c & 7)];
    R[i] = v;
  }
  if (stats) {
#pragma unroll
    for (int T = 0; T < TCN; ++T) {
      double a = sa[T], s = sq[T];
      a += __shfl_xor_sync(0xffffffffu, a, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      a += __shfl_xor_sync(0xffffffffu, a, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (kr == 0 && 8 * T + cj < npad) {
        stats[leaf * 2 * npad + 8 * T + cj] = a;
        stats[leaf * 2 * npad + npad + 8 * T + cj] = s;
      }
    }
  }
}

namespace {

template <int TCN, int NT, bool kKeep>
int rg_launch(const double* x, int64_t m, int64_t ldx, int n, int64_t rpw, int nleaves, int npad, double* slots,
              double* stats, cudaStream_t st) {
  using L = RgLayout<TCN, NT>;
  static PerDeviceFlag attr;
  if (!attr.is_set()) {
    TSNMF_CUDA_CHECK((cudaFuncSetAttribute(tsqr_reg_leaf_kernel<TCN, NT, kKeep>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)L::bytes)));
    attr.set();
  }
  prof_mark(kProfTsqrLeaf, true, st);
  tsqr_reg_leaf_kernel<TCN, NT, kKeep><<<(unsigned)ceil_div(nleaves, kRgWarps), 32 * kRgWarps, L::bytes, st>>>(
      x, m, ldx, n, rpw, nleaves, npad, slots, stats);
  TSNMF_LAUNCH_CHECK();
  prof_mark(kProfTsqrLeaf, false, st);
  return kOk;
}

}  // namespace

// Widths served: 25..64 (4..8 column tiles).  Rows per block = 8 NT with NT chosen so the block fills the
// register file (about 96 doubles per lane); TSNMF_RG_NT overrides where several are built.
bool tsqr_reg_supported(int n) { return n >= 25 && n <= 64; }
static int rg_nt(int n) {
  const int tcn = (n + 7) / 8;
  int nt = tcn == 4 ? 10 : (tcn == 5 ? 9 : (tcn == 6 ? 8 : (tcn == 7 ? 6 : 6)));
  if (const char* e = getenv("TSNMF_RG_NT")) {
    const int v = atoi(e);
    if (tcn == 4 && (v == 8 || v == 10 || v == 12)) nt = v;
    if (tcn == 8 && (v == 4 || v == 5 || v == 6)) nt = v;
  }
  return nt;
}
int tsqr_reg_block_rows(int n) { return 8 * rg_nt(n); }
int tsqr_reg_warps_per_cta() { return kRgWarps; }

int tsqr_reg_leaf_run(const double* x, int64_t m, int64_t ldx, int n, int64_t rpw, int nleaves, int npad,
                      double* slots, double* stats, cudaStream_t st) {
  const int nt = rg_nt(n);
  switch ((n + 7) / 8) {
    case 4:
      if (nt == 12) return rg_launch<4, 12, false>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
      if (nt == 8) return rg_launch<4, 8, true>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
      return rg_launch<4, 10, false>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
    case 5: return rg_launch<5, 9, false>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
    case 6: return rg_launch<6, 8, false>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
    case 7: return rg_launch<7, 6, false>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
    default:
      if (nt == 4) return rg_launch<8, 4, true>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
      if (nt == 5) return rg_launch<8, 5, false>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
      return rg_launch<8, 6, false>(x, m, ldx, n, rpw, nleaves, npad, slots, stats, st);
  }
}

}  // namespace tsnmf

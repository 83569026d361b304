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
// u = [e_j; v] (R part is a unit vector), so only R row j and the block are touched.  Panels of NB
// columns are factored cooperatively (warp shuffles + one CTA barrier per column); the trailing update
// uses the compact-WY form  W = R_p + V^T B,  W <- T^T W,  R_p -= W,  B -= V W  on FP64 tensor cores
// (mma.sync m8n8k4 f64 = DMMA).  Leaves are then combined in the reference TreeReducer order (perfect
// binary levels over the leaf index, then a fold of the leftover subtrees), each combine being the same
// structured QR with the second factor's rows as data (triangular: panels left of the block are skipped).
#include "common.cuh"
#include "internal.h"

namespace tsnmf {

constexpr int kTqThreads = 256;
constexpr int kTqWarps = kTqThreads / 32;
constexpr int kMaxRpt = 8;  // panel rows per thread

struct TqGeom {
  int n;      // data columns
  int npad;   // padded columns (multiple of NB); R slots are npad x npad
  int lds;    // shared-memory row stride of the block
  int brows;  // rows per block (multiple of 8, <= (256/NB) * kMaxRpt)
};

template <int NB>
struct TqLayout {
  static constexpr int kSlots = kTqThreads / NB;
  // offsets in doubles from the dynamic smem base
  __host__ __device__ static int rd(const TqGeom& g) { return g.brows * g.lds; }
  __host__ __device__ static int tm(const TqGeom& g) { return rd(g) + NB * NB; }
  __host__ __device__ static int tcol(const TqGeom& g) { return tm(g) + NB * NB; }
  __host__ __device__ static int tau(const TqGeom& g) { return tcol(g) + NB * NB; }
  __host__ __device__ static int part(const TqGeom& g) { return tau(g) + NB; }
  __host__ __device__ static int wsc(const TqGeom& g) { return part(g) + 2 * kTqWarps * NB; }
  __host__ __device__ static int total(const TqGeom& g) { return wsc(g) + kTqWarps * NB * 8; }
  static size_t bytes(const TqGeom& g) { return sizeof(double) * (size_t)total(g); }
};

// Fold `nrows` data rows (row-major, stride ldsrc, `ncols` real columns) into the R slot `R`.
// triangular: data row i is zero left of column i (data is another R factor).
template <int NB>
__device__ void tsqr_fold(double* __restrict__ R, const double* __restrict__ src, int64_t nrows, int64_t ldsrc,
                          int ncols, const TqGeom g, bool triangular, bool init_zero,
                          double* __restrict__ stats_out, double* smem) {
  using L = TqLayout<NB>;
  constexpr int kSlots = L::kSlots;
  constexpr int G = 4;  // column blocks per GEMM group
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int npad = g.npad, lds = g.lds, brows = g.brows;
  double* Bs = smem;
  double* Rd = smem + L::rd(g);
  double* Tm = smem + L::tm(g);
  double* Tcol = smem + L::tcol(g);
  double* tau_s = smem + L::tau(g);
  double* part = smem + L::part(g);
  double* Wsc = smem + L::wsc(g) + warp * NB * 8;

  const int c = tid % NB, s = tid / NB;
  const int rpt = (brows + kSlots - 1) / kSlots;
  const int npanels = npad / NB, ncb = npad / 8;
  const bool vec16 = ((ldsrc & 1) == 0) && ((reinterpret_cast<uintptr_t>(src) & 15) == 0);

  if (init_zero) {
    for (int64_t idx = tid; idx < (int64_t)npad * npad; idx += kTqThreads) R[idx] = 0.0;
  }
  double l1a[2] = {0.0, 0.0}, sqa[2] = {0.0, 0.0};

  for (int64_t r0 = 0; r0 < nrows; r0 += brows) {
    const int cnt = (int)min64(brows, nrows - r0);
    __syncthreads();  // previous block fully consumed; R init visible
    stage_rows(Bs, lds, src + r0 * ldsrc, ldsrc, cnt, ncols, brows, npad, vec16);
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (stats_out) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = tid + h * kTqThreads;
        if (col < ncols) {
          double a = l1a[h], q = sqa[h];
          for (int i = 0; i < cnt; ++i) {
            const double v = Bs[i * lds + col];
            a += fabs(v);
            q = fma(v, v, q);
          }
          l1a[h] = a;
          sqa[h] = q;
        }
      }
    }
    const int p0 = triangular ? (int)min64(r0 / NB, npanels) : 0;
    if (tid < NB * NB && p0 < npanels) {
      const int j0 = p0 * NB;
      Rd[tid] = R[(int64_t)(j0 + tid / NB) * npad + j0 + tid % NB];
    }
    int buf = 0;
    for (int p = p0; p < npanels; ++p) {
      const int j0 = p * NB;
      __syncthreads();  // (A) trailing update of the previous panel done; Rd loaded
      double pv[kMaxRpt];
#pragma unroll
      for (int q = 0; q < kMaxRpt; ++q) {
        const int i = s + kSlots * q;
        pv[q] = (q < rpt && i < brows) ? Bs[i * lds + j0 + c] : 0.0;
      }
      // ---- panel factorization: NB Householder reflectors on [R(j0:j0+NB, :); B(:, panel)]
#pragma unroll 1
      for (int jj = 0; jj < NB; ++jj) {
        const int j = j0 + jj;
        const int src_lane = (lane & ~(NB - 1)) | jj;
        double xj[kMaxRpt];
        double d = 0.0;
#pragma unroll
        for (int q = 0; q < kMaxRpt; ++q) {
          xj[q] = __shfl_sync(0xffffffffu, pv[q], src_lane);
          d = fma(xj[q], pv[q], d);
        }
#pragma unroll
        for (int off = NB; off < 32; off <<= 1) d += __shfl_xor_sync(0xffffffffu, d, off);
        if (lane < NB) part[(buf * kTqWarps + warp) * NB + lane] = d;
        __syncthreads();
        double dj = 0.0, dc = 0.0;
#pragma unroll
        for (int w = 0; w < kTqWarps; ++w) {
          dj += part[(buf * kTqWarps + w) * NB + jj];
          dc += part[(buf * kTqWarps + w) * NB + c];
        }
        buf ^= 1;
        const double alpha = Rd[jj * NB + jj];
        double tau = 0.0, scale = 0.0, beta = alpha;
        if (dj > 0.0) {  // dlarfg: beta = -sign(alpha) * ||(alpha, x)||, tau = (beta - alpha) / beta
          const double nrm = sqrt(fma(alpha, alpha, dj));
          beta = -copysign(nrm, alpha);
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        if (c > jj) {
          const double rjc = Rd[jj * NB + c];
          const double tw = tau * fma(scale, dc, rjc);
          const double f = tw * scale;
#pragma unroll
          for (int q = 0; q < kMaxRpt; ++q) pv[q] = fma(-f, xj[q], pv[q]);
          if (s == 0) R[(int64_t)j * npad + j0 + c] = rjc - tw;
        } else if (c == jj) {
#pragma unroll
          for (int q = 0; q < kMaxRpt; ++q) pv[q] *= scale;
          if (s == 0) {
            R[(int64_t)j * npad + j] = beta;
            tau_s[jj] = tau;
          }
        } else if (s == 0) {
          Tcol[c * NB + jj] = scale * dc;  // v_c^T v_jj
        }
      }
#pragma unroll
      for (int q = 0; q < kMaxRpt; ++q) {
        const int i = s + kSlots * q;
        if (q < rpt && i < brows) Bs[i * lds + j0 + c] = pv[q];
      }
      __syncthreads();  // (C) V in Bs, tau / Tcol visible
      if (warp == 0 && lane < NB) {  // T (upper triangular, dlarft forward/columnwise): row `lane`
        double trow[NB];
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) {
          if (jj < lane) {
            trow[jj] = 0.0;
          } else if (jj == lane) {
            trow[jj] = tau_s[jj];
          } else {
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < jj; ++q)
              if (q >= lane) acc = fma(trow[q], Tcol[q * NB + jj], acc);
            trow[jj] = -tau_s[jj] * acc;
          }
        }
#pragma unroll
        for (int jj = 0; jj < NB; ++jj) Tm[lane * NB + jj] = trow[jj];
      }
      __syncthreads();  // (D) T visible
      // ---- trailing update on warp-owned column blocks (no CTA barrier inside)
      const int cb0 = (j0 + NB) / 8;
      for (int base = cb0 + warp; base < ncb; base += kTqWarps * G) {
        double acc[NB / 8][G][2];
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const int cb = base + kTqWarps * gg;
#pragma unroll
          for (int rb = 0; rb < NB / 8; ++rb) {
            if (cb < ncb) {
              const double* rp = R + (int64_t)(j0 + 8 * rb + (lane >> 2)) * npad + 8 * cb + 2 * (lane & 3);
              acc[rb][gg][0] = rp[0];
              acc[rb][gg][1] = rp[1];
            } else {
              acc[rb][gg][0] = acc[rb][gg][1] = 0.0;
            }
          }
        }
        // W = R_p + V^T B    (K = brows, 4 rows per DMMA)
        for (int i = 0; i < brows; i += 4) {
          const double* row = Bs + (i + (lane & 3)) * lds;
          double a[NB / 8];
#pragma unroll
          for (int rb = 0; rb < NB / 8; ++rb) a[rb] = row[j0 + 8 * rb + (lane >> 2)];
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
            const int cb = base + kTqWarps * gg;
            if (cb < ncb) {
              const double b = row[8 * cb + (lane >> 2)];
#pragma unroll
              for (int rb = 0; rb < NB / 8; ++rb) dmma(acc[rb][gg][0], acc[rb][gg][1], a[rb], b);
            }
          }
        }
        // W' = T^T W ; R_p -= W' ; gather -W' as B-operand fragments
        double wb[G][NB / 4];
#pragma unroll
        for (int gg = 0; gg < G; ++gg) {
          const int cb = base + kTqWarps * gg;
          if (cb >= ncb) continue;
#pragma unroll
          for (int rb = 0; rb < NB / 8; ++rb) {
            Wsc[(8 * rb + (lane >> 2)) * 8 + 2 * (lane & 3)] = acc[rb][gg][0];
            Wsc[(8 * rb + (lane >> 2)) * 8 + 2 * (lane & 3) + 1] = acc[rb][gg][1];
          }
          __syncwarp();
          double wn[NB / 8][2];
#pragma unroll
          for (int ro = 0; ro < NB / 8; ++ro) {
            wn[ro][0] = wn[ro][1] = 0.0;
#pragma unroll
            for (int k0 = 0; k0 < 8 * (ro + 1); k0 += 4) {
              const double a = Tm[(k0 + (lane & 3)) * NB + 8 * ro + (lane >> 2)];
              const double b = Wsc[(k0 + (lane & 3)) * 8 + (lane >> 2)];
              dmma(wn[ro][0], wn[ro][1], a, b);
            }
            double* rp = R + (int64_t)(j0 + 8 * ro + (lane >> 2)) * npad + 8 * cb + 2 * (lane & 3);
            rp[0] -= wn[ro][0];
            rp[1] -= wn[ro][1];
          }
          __syncwarp();
#pragma unroll
          for (int ro = 0; ro < NB / 8; ++ro) {
            Wsc[(8 * ro + (lane >> 2)) * 8 + 2 * (lane & 3)] = wn[ro][0];
            Wsc[(8 * ro + (lane >> 2)) * 8 + 2 * (lane & 3) + 1] = wn[ro][1];
          }
          __syncwarp();
#pragma unroll
          for (int k4 = 0; k4 < NB / 4; ++k4) wb[gg][k4] = -Wsc[(4 * k4 + (lane & 3)) * 8 + (lane >> 2)];
          __syncwarp();
        }
        // B -= V W'   (C tiles read/written in place; K = NB)
        for (int rb = 0; rb < brows / 8; ++rb) {
          const double* vrow = Bs + (8 * rb + (lane >> 2)) * lds + j0 + (lane & 3);
          double a[NB / 4];
#pragma unroll
          for (int k4 = 0; k4 < NB / 4; ++k4) a[k4] = vrow[4 * k4];
#pragma unroll
          for (int gg = 0; gg < G; ++gg) {
            const int cb = base + kTqWarps * gg;
            if (cb < ncb) {
              double2* cp = reinterpret_cast<double2*>(Bs + (8 * rb + (lane >> 2)) * lds + 8 * cb + 2 * (lane & 3));
              double2 cv = *cp;
#pragma unroll
              for (int k4 = 0; k4 < NB / 4; ++k4) dmma(cv.x, cv.y, a[k4], wb[gg][k4]);
              *cp = cv;
            }
          }
        }
      }
      // next panel's diagonal block of R (rows j0+NB.., untouched by this panel)
      if (p + 1 < npanels && tid < NB * NB) {
        const int j1 = j0 + NB;
        Rd[tid] = R[(int64_t)(j1 + tid / NB) * npad + j1 + tid % NB];
      }
    }
  }
  if (stats_out) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = tid + h * kTqThreads;
      if (col < npad) {
        stats_out[col] = l1a[h];
        stats_out[npad + col] = sqa[h];
      }
    }
  }
}

template <int NB, int MINB>
__global__ void __launch_bounds__(kTqThreads, MINB)
    tsqr_leaf_kernel(const double* __restrict__ x, int64_t m, int64_t ldx, int64_t rows_per_cta, TqGeom g,
                     double* __restrict__ slots, double* __restrict__ stats) {
  extern __shared__ __align__(16) double smem[];
  const int64_t r0 = (int64_t)blockIdx.x * rows_per_cta;
  const int64_t cnt = max64(0, min64(rows_per_cta, m - r0));
  double* R = slots + (int64_t)blockIdx.x * g.npad * g.npad;
  double* st = stats ? stats + (int64_t)blockIdx.x * 2 * g.npad : nullptr;
  tsqr_fold<NB>(R, x + r0 * ldx, cnt, ldx, g.n, g, false, true, st, smem);
}

// One level of the binary-counter tree: slot[q*2^L] = qr([slot[q*2^L]; slot[q*2^L + 2^(L-1)]]),
// or (fold) slot[dst] = qr([slot[dst]; slot[src]]).
template <int NB, int MINB>
__global__ void __launch_bounds__(kTqThreads, MINB)
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
  tsqr_fold<NB>(slots + dst * ss, slots + srcs * ss, g.npad, g.npad, g.npad, g, true, false, nullptr, smem);
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
  int nb;
  int minb;
  TqGeom g;
  size_t smem;
};

int tq_max_rows(int nb) { return (kTqThreads / nb) * kMaxRpt; }

template <int NB>
size_t tq_bytes(const TqGeom& g) { return TqLayout<NB>::bytes(g); }

size_t tq_bytes_nb(int nb, const TqGeom& g) { return nb == 8 ? tq_bytes<8>(g) : tq_bytes<16>(g); }

bool tq_choose(int n, int nb, int minb, TqChoice* out) {
  TqGeom g;
  g.n = n;
  g.npad = (int)round_up(n, nb);
  g.lds = smem_stride(g.npad);
  const size_t budget = (minb == 2 ? 113 : 226) * 1024;
  g.brows = 8;
  if (tq_bytes_nb(nb, g) > budget) return false;
  int best = 8;
  for (int b = 8; b <= tq_max_rows(nb); b += 8) {
    g.brows = b;
    if (tq_bytes_nb(nb, g) <= budget) best = b;
  }
  g.brows = best;
  out->nb = nb;
  out->minb = minb;
  out->g = g;
  out->smem = tq_bytes_nb(nb, g);
  return true;
}

bool tq_config(int n, TqChoice* out) {
  // Panel width / occupancy.  TSNMF_TSQR_NB / TSNMF_TSQR_CTAS override for tuning.
  int nb = 16, minb = 2;
  if (const char* e = getenv("TSNMF_TSQR_NB")) nb = atoi(e) == 8 ? 8 : 16;
  if (const char* e = getenv("TSNMF_TSQR_CTAS")) minb = atoi(e) == 1 ? 1 : 2;
  if (tq_choose(n, nb, minb, out) && out->g.brows >= 32) return true;
  if (tq_choose(n, nb, 1, out) && out->g.brows >= 16) return true;
  if (tq_choose(n, 8, 1, out)) return true;
  return false;
}

template <int NB, int MINB>
int tq_launch_all(const TqChoice& ch, const double* x, int64_t m, int64_t ldx, double* slots, double* stats,
                  int nleaves, int64_t rows_per_cta, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(tsqr_leaf_kernel<NB, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          232448));
    TSNMF_CUDA_CHECK(cudaFuncSetAttribute(tsqr_combine_kernel<NB, MINB>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    attr_set = true;
  }
  if (x) {
    prof_mark(kProfTsqrLeaf, true, st);
    tsqr_leaf_kernel<NB, MINB><<<nleaves, kTqThreads, ch.smem, st>>>(x, m, ldx, rows_per_cta, ch.g, slots, stats);
    TSNMF_LAUNCH_CHECK();
    prof_mark(kProfTsqrLeaf, false, st);
  }
  prof_mark(kProfTsqrTree, true, st);
  // binary-counter tree (tsqr.py:213-230): perfect levels, then fold leftover subtrees low -> high
  for (int64_t span = 2; span <= nleaves; span *= 2) {
    const int64_t q = nleaves / span;
    tsqr_combine_kernel<NB, MINB><<<(unsigned)q, kTqThreads, ch.smem, st>>>(slots, span, span / 2, 0, 0, ch.g);
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
    tsqr_combine_kernel<NB, MINB><<<1, kTqThreads, ch.smem, st>>>(slots, 0, 0, offs[t], offs[t + 1], ch.g);
    TSNMF_LAUNCH_CHECK();
  }
  prof_mark(kProfTsqrTree, false, st);
  return kOk;
}

int tq_dispatch(const TqChoice& ch, const double* x, int64_t m, int64_t ldx, double* slots, double* stats,
                int nleaves, int64_t rows_per_cta, cudaStream_t st) {
  if (ch.nb == 16 && ch.minb == 2) return tq_launch_all<16, 2>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
  if (ch.nb == 16) return tq_launch_all<16, 1>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
  if (ch.minb == 2) return tq_launch_all<8, 2>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
  return tq_launch_all<8, 1>(ch, x, m, ldx, slots, stats, nleaves, rows_per_cta, st);
}

int device_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = kNumSMs;
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

}  // namespace

int tsqr_max_cols() { return 512; }

size_t tsqr_workspace_bytes(int64_t m, int n) {
  TqChoice ch;
  if (n < 1 || !tq_config(n, &ch)) return 0;
  int nleaves;
  int64_t rpc;
  tq_plan(ch, max64(m, 1), &nleaves, &rpc);
  const int64_t npad = ch.g.npad;
  return sizeof(double) * (size_t)(nleaves * npad * npad + nleaves * 2 * npad) + 256;
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
  tq_plan(ch, m, &nleaves, &rpc);
  const int64_t npad = ch.g.npad;
  const size_t need = sizeof(double) * (size_t)(nleaves * npad * npad + nleaves * 2 * npad);
  if (ws_bytes < need) return set_error(kUsage, "tsqr: workspace too small (%zu < %zu bytes)", ws_bytes, need);
  double* slots = reinterpret_cast<double*>(ws);
  double* stats = slots + (int64_t)nleaves * npad * npad;
  const bool want_stats = (l1 != nullptr) || (sumsq != nullptr);
  int rc = tq_dispatch(ch, x, m, ldx, slots, want_stats ? stats : nullptr, nleaves, rpc, st);
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
  tq_plan(ch, max64(m, 1), nleaves, &rpc);
  *nb = ch.nb;
  *brows = ch.g.brows;
  *ctas_per_sm = ch.minb;
  return kOk;
}

}  // namespace tsnmf

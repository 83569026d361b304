// Shared device helpers for the tsnmf B200 kernels (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "tsnmf_b200 is written for sm_100a (B200) only"
#endif

namespace tsnmf {

// Status codes mirror reference pkg/src/tsnmf/errors.py:16-31 (exit codes).
enum Status : int { kOk = 0, kUsage = 1, kData = 2, kNumerical = 3, kCuda = 4 };

// Set the thread-local error message (capi.cu) and return the status.
int set_error(int status, const char* fmt, ...);

#define TSNMF_CUDA_CHECK(expr)                                                              \
  do {                                                                                      \
    cudaError_t _e = (expr);                                                                \
    if (_e != cudaSuccess)                                                                  \
      return ::tsnmf::set_error(::tsnmf::kCuda, "%s failed: %s", #expr, cudaGetErrorString(_e)); \
  } while (0)

// Every kernel launch is followed by this check; it also feeds the launch counter (tsnmf_launch_count).
void note_launch();
#define TSNMF_LAUNCH_CHECK()      \
  do {                            \
    ::tsnmf::note_launch();       \
    TSNMF_CUDA_CHECK(cudaGetLastError()); \
  } while (0)

// Optional CUDA-event timing of the dominant kernels on their launching stream (tsnmf_profile_*).
enum ProfSlot : int { kProfTsqrLeaf = 0, kProfTsqrTree = 1, kProfGram = 2, kProfSketch = 3, kProfSlots = 4 };
void prof_mark(int slot, bool begin, cudaStream_t st);

constexpr int kNumSMs = 148;  // B200; launch code queries the device, this is only a default

// ---------------------------------------------------------------------------
// FP64 tensor-core MMA: D(8x8) += A(8x4) * B(4x8).  Fragment layout (per lane l):
//   A: row l/4, col l%4        B: row l%4, col l/4        C/D: row l/4, cols 2*(l%4) + {0,1}
// On sm_100a this lowers to one DMMA.8x8x4 (measured 37.0 TF/s chip-wide, profiles/r01_peaks.json).
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// Counter-based RNG, value-compatible with reference pkg/src/tsnmf/_kernels.pyx:21-69
// (integer part bit-exact; log/cos/sqrt are CUDA libdevice, within a few ulp of libm).
constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
constexpr double kTwoPi = 6.283185307179586476925286766559;
constexpr double kInv2p53 = 1.0 / 9007199254740992.0;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// word(s, c) = mix(s + (c + 1) * gamma)   (_kernels.pyx:31-32)
__host__ __device__ __forceinline__ uint64_t rng_word(uint64_t stream, uint64_t ctr) {
  return mix64(stream + (ctr + 1) * kGamma);
}

// rng.py:33-35
__host__ __device__ __forceinline__ uint64_t derive_stream(uint64_t seed, uint64_t tag) {
  return mix64(seed ^ mix64(tag + kGamma));
}

__device__ __forceinline__ double rng_uniform(uint64_t stream, uint64_t ctr) {
  return __dmul_rn((double)(rng_word(stream, ctr) >> 11), kInv2p53);
}


// Box-Muller polynomial coefficients in the constant bank: DFMA reads them as c[] operands instead of
// materialising each 64-bit immediate with two uniform moves per use (~60 UMOVs per normal).
static __constant__ double kBmLogPolyC[31] = {
    0.05263157894736842,
    0.058823529411764705,
    0.06666666666666667,
    0.07692307692307693,
    0.09090909090909091,
    0.1111111111111111,
    0.14285714285714285,
    0.2,
    0.3333333333333333,
    1.0,
    0.047619047619047616,
    4.779477332387385e-14,
    -1.1470745597729725e-11,
    2.08767569878681e-09,
    -2.755731922398589e-07,
    2.48015873015873e-05,
    -0.001388888888888889,
    0.041666666666666664,
    -0.5,
    1.0,
    -1.5619206968586225e-16,
    2.8114572543455206e-15,
    -7.647163731819816e-13,
    1.6059043836821613e-10,
    -2.505210838544172e-08,
    2.7557319223985893e-06,
    -0.0001984126984126984,
    0.008333333333333333,
    -0.16666666666666666,
    1.0,
    -8.22063524662433e-18};
// log(u), polynomial form, for u in [2^-54, 1) (the Box-Muller u1 domain): u = m 2^e with m in [sqrt(1/2), sqrt(2)),
// log m = 2 atanh(s), s = (m - 1)/(m + 1), |s| <= 0.1716, atanh series through s^21; ln 2 split hi/lo.
// No special-value paths are needed on this domain.  Max relative error ~4e-16 vs libm (1M samples).
__device__ __forceinline__ double bm_log_poly(double u) {
  const int hi = __double2hiint(u), lo = __double2loint(u);
  int e = ((hi >> 20) & 0x7ff) - 1023;
  double m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, lo);  // [1, 2)
  const bool big = m > 1.4142135623730951;
  m = big ? 0.5 * m : m;
  e = big ? e + 1 : e;
  const double f = m - 1.0;
  const double den = 2.0 + f;
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(den));
  r = r * fma(-den, r, 2.0);
  r = r * fma(-den, r, 2.0);
  double sv = f * r;
  sv = fma(r, fma(-sv, den, f), sv);  // one residual correction: s to ~0.5 ulp
  const double z = sv * sv;
  double p = kBmLogPolyC[10];
  p = fma(p, z, kBmLogPolyC[0]);
  p = fma(p, z, kBmLogPolyC[1]);
  p = fma(p, z, kBmLogPolyC[2]);
  p = fma(p, z, kBmLogPolyC[3]);
  p = fma(p, z, kBmLogPolyC[4]);
  p = fma(p, z, kBmLogPolyC[5]);
  p = fma(p, z, kBmLogPolyC[6]);
  p = fma(p, z, kBmLogPolyC[7]);
  p = fma(p, z, kBmLogPolyC[8]);
  p = fma(p, z, kBmLogPolyC[9]);
  const double de = (double)e;
  return fma(de, 0.6931471803691238, fma(de, 1.9082149292705877e-10, 2.0 * sv * p));
}

// log(u) for u in [2^-54, 1) (the Box-Muller u1 domain): table-driven.  u = 2^e m, m in [1, 2); for
// m >= 1.5 use m/2 and e+1, so m' in [0.75, 1.5) (u near 1 keeps e' = 0: no cancellation); j = round(64 m')
// from the mantissa bits, f = m' inv_j - 1 (|f| <= 0.0105, one rounding), log1p(f) through f^9 (truncation
// < 2e-21), log u = e' ln2 + L_j + log1p(f) with L_j = -ln(inv_j) (hi + lo, the exact logarithm of the
// stored reciprocal).  ~14 FP64 operations instead of ~21; ~1 ulp.  Table: tools/gen_bm_tables.py log.
// LN2_HI = 0x1.62e42fefa3a00p-1, LN2_LO = -0x1.0ca86c3898d00p-49
static __device__ const double4 kBmLogTab[49] = {
    {0x1.5555555555555p+0, -0x1.269621134db91p-2, -0x1.e0efadd9db02ap-56, 0.0},  // j = 48
    {0x1.4e5e0a72f0539p+0, -0x1.1178e8227e47ap-2, -0x1.b8ce2d07f1cb7p-56, 0.0},  // j = 49
    {0x1.47ae147ae147bp+0, -0x1.f991c6cb3b37ap-3, -0x1.ecca0cdf30143p-58, 0.0},  // j = 50
    {0x1.4141414141414p+0, -0x1.d1037f2655e7bp-3, 0x1.3f3adb7b71cbcp-58, 0.0},  // j = 51
    {0x1.3b13b13b13b14p+0, -0x1.a93ed3c8ad9e5p-3, -0x1.bcafa9de97202p-57, 0.0},  // j = 52
    {0x1.3521cfb2b78c1p+0, -0x1.823c16551a3c0p-3, -0x1.6dcd318f4187ep-57, 0.0},  // j = 53
    {0x1.2f684bda12f68p+0, -0x1.5bf406b543db0p-3, 0x1.1f5b44c0df7f7p-61, 0.0},  // j = 54
    {0x1.29e4129e4129ep+0, -0x1.365fcb0159014p-3, -0x1.bea08d2dca256p-57, 0.0},  // j = 55
    {0x1.2492492492492p+0, -0x1.1178e8227e47ap-3, 0x1.0e63a5f01c693p-58, 0.0},  // j = 56
    {0x1.1f7047dc11f70p+0, -0x1.da7276384469ep-4, -0x1.401fa71733017p-58, 0.0},  // j = 57
    {0x1.1a7b9611a7b96p+0, -0x1.9335e5d594988p-4, 0x1.478a85704ccb7p-58, 0.0},  // j = 58
    {0x1.15b1e5f75270dp+0, -0x1.4d3115d207eacp-4, -0x1.da7d0b1e10b2fp-60, 0.0},  // j = 59
    {0x1.1111111111111p+0, -0x1.08598b59e3a06p-4, 0x1.dd7009902bf32p-58, 0.0},  // j = 60
    {0x1.0c9714fbcda3bp+0, -0x1.894aa149fb34bp-5, 0x1.2ba0b44cfaee5p-59, 0.0},  // j = 61
    {0x1.0842108421084p+0, -0x1.0415d89e74440p-5, -0x1.c05cf1d753621p-59, 0.0},  // j = 62
    {0x1.0410410410410p+0, -0x1.0205658935837p-6, -0x1.27c8e8416e717p-60, 0.0},  // j = 63
    {0x1.0000000000000p+0, 0x0.0p+0, 0x0.0p+0, 0.0},  // j = 64
    {0x1.f81f81f81f820p-1, 0x1.fc0a8b0fc03c4p-7, -0x1.83092c5964281p-62, 0.0},  // j = 65
    {0x1.f07c1f07c1f08p-1, 0x1.f829b0e7832f8p-6, 0x1.33e3f04f1ef25p-60, 0.0},  // j = 66
    {0x1.e9131abf0b767p-1, 0x1.77458f632dcffp-5, 0x1.8d3ca87b92968p-63, 0.0},  // j = 67
    {0x1.e1e1e1e1e1e1ep-1, 0x1.f0a30c01162a8p-5, 0x1.85f325c5bbacdp-59, 0.0},  // j = 68
    {0x1.dae6076b981dbp-1, 0x1.341d7961bd1d0p-4, -0x1.3599f227becbbp-58, 0.0},  // j = 69
    {0x1.d41d41d41d41dp-1, 0x1.6f0d28ae56b4ep-4, -0x1.20db323097324p-59, 0.0},  // j = 70
    {0x1.cd85689039b0bp-1, 0x1.a926d3a4ad562p-4, -0x1.d7a16eab1e2adp-59, 0.0},  // j = 71
    {0x1.c71c71c71c71cp-1, 0x1.e27076e2af2eap-4, -0x1.61578001e015ap-60, 0.0},  // j = 72
    {0x1.c0e070381c0e0p-1, 0x1.0d77e7cd08e5bp-3, 0x1.9a5dc5e9030adp-57, 0.0},  // j = 73
    {0x1.bacf914c1bad0p-1, 0x1.29552f81ff521p-3, 0x1.301771c407dc0p-57, 0.0},  // j = 74
    {0x1.b4e81b4e81b4fp-1, 0x1.44d2b6ccb7d1cp-3, 0x1.7d3d950f87e23p-59, 0.0},  // j = 75
    {0x1.af286bca1af28p-1, 0x1.5ff3070a793d6p-3, -0x1.bc60efafc6f6cp-58, 0.0},  // j = 76
    {0x1.a98ef606a63bep-1, 0x1.7ab890210d907p-3, -0x1.1072534a57e7dp-57, 0.0},  // j = 77
    {0x1.a41a41a41a41ap-1, 0x1.9525a9cf456b6p-3, -0x1.26fb3e2b1d1dap-57, 0.0},  // j = 78
    {0x1.9ec8e951033d9p-1, 0x1.af3c94e80bff3p-3, 0x1.a3398064df33ep-57, 0.0},  // j = 79
    {0x1.999999999999ap-1, 0x1.c8ff7c79a9a20p-3, -0x1.4f689f8434011p-57, 0.0},  // j = 80
    {0x1.948b0fcd6e9e0p-1, 0x1.e27076e2af2e8p-3, -0x1.61578001e015ep-59, 0.0},  // j = 81
    {0x1.8f9c18f9c18fap-1, 0x1.fb9186d5e3e29p-3, 0x1.355519b0de535p-57, 0.0},  // j = 82
    {0x1.8acb90f6bf3aap-1, 0x1.0a324e27390e2p-2, 0x1.bdcfde8061c03p-56, 0.0},  // j = 83
    {0x1.8618618618618p-1, 0x1.1675cababa60fp-2, 0x1.ce63eab883727p-61, 0.0},  // j = 84
    {0x1.8181818181818p-1, 0x1.22941fbcf7966p-2, -0x1.dbd7ac258a2bdp-58, 0.0},  // j = 85
    {0x1.7d05f417d05f4p-1, 0x1.2e8e2bae11d31p-2, -0x1.1e99b72bd7bf2p-57, 0.0},  // j = 86
    {0x1.78a4c8178a4c8p-1, 0x1.3a64c556945eap-2, 0x1.cbcd735d03424p-60, 0.0},  // j = 87
    {0x1.745d1745d1746p-1, 0x1.4618bc21c5ec2p-2, -0x1.7a42642661c62p-61, 0.0},  // j = 88
    {0x1.702e05c0b8170p-1, 0x1.51aad872df82ep-2, -0x1.d8db0a7cc1543p-56, 0.0},  // j = 89
    {0x1.6c16c16c16c17p-1, 0x1.5d1bdbf5809cap-2, -0x1.7dc9c7c23801fp-56, 0.0},  // j = 90
    {0x1.6816816816817p-1, 0x1.686c81e9b14adp-2, 0x1.710af840538e3p-56, 0.0},  // j = 91
    {0x1.642c8590b2164p-1, 0x1.739d7f6bbd007p-2, 0x1.ce24c53fad3f0p-58, 0.0},  // j = 92
    {0x1.6058160581606p-1, 0x1.7eaf83b82afc2p-2, -0x1.698b43096b576p-59, 0.0},  // j = 93
    {0x1.5c9882b931057p-1, 0x1.89a3386c1425bp-2, 0x1.2d38c40881e0bp-57, 0.0},  // j = 94
    {0x1.58ed2308158edp-1, 0x1.947941c2116fbp-2, 0x1.1266e8a3e8838p-57, 0.0},  // j = 95
    {0x1.5555555555555p-1, 0x1.9f323ecbf984dp-2, -0x1.a92e513217f58p-59, 0.0},  // j = 96
};
static __constant__ double kBmLogC[8] = {1.0 / 9, -1.0 / 8, 1.0 / 7, -1.0 / 6, 1.0 / 5, -1.0 / 4, 1.0 / 3, -0.5};
__device__ __forceinline__ double bm_log_tab(double u) {
  const int hi = __double2hiint(u), lo = __double2loint(u);
  const int ftop = hi & 0x000fffff;  // top 20 bits of the mantissa field
  const bool big = ftop >= 0x80000;  // m >= 1.5
  const int e = ((hi >> 20) & 0x7ff) - 1023 + (big ? 1 : 0);
  const int j = big ? 32 + ((ftop + 0x4000) >> 15) : 64 + ((ftop + 0x2000) >> 14);  // round(64 m'), 48..96
  const double mp = __hiloint2double(ftop | (big ? 0x3fe00000 : 0x3ff00000), lo);
  const double2 t0 = __ldg(reinterpret_cast<const double2*>(&kBmLogTab[j - 48]));
  const double2 t1 = __ldg(reinterpret_cast<const double2*>(&kBmLogTab[j - 48]) + 1);
  const double f = fma(mp, t0.x, -1.0);
  double q = fma(f, kBmLogC[0], kBmLogC[1]);
  q = fma(q, f, kBmLogC[2]);
  q = fma(q, f, kBmLogC[3]);
  q = fma(q, f, kBmLogC[4]);
  q = fma(q, f, kBmLogC[5]);
  q = fma(q, f, kBmLogC[6]);
  q = fma(q, f, kBmLogC[7]);
  const double lp = fma(f * f, q, f);
  const double de = (double)e;
  return fma(de, 0x1.62e42fefa3a00p-1, t0.y) + (fma(de, -0x1.0ca86c3898d00p-49, t1.x) + lp);
}

// cos(t) for t = fl(2 pi u2), u2 = w2 2^-53 (the Box-Muller angle): table-driven.  k = round(64 u2) from
// the integer w2, r = t - k pi/32 (two-part Cody-Waite constant, exact first step), |r| <= pi/64;
// cos(k pi/32 + r) = C_k cos r - S_k sin r with cos r / sin r through r^8 / r^9 (truncation < 1e-19) and
// C_k, S_k from a 33-entry table (cos is even: k > 32 uses 64 - k and the sign of the sine term flips).
// 14 FP64 operations instead of ~26 for the quadrant version (the FP64 pipe is shared with the sketch's
// DMMAs).  Max absolute error ~2e-16 vs libm.  Table: tools/gen_bm_tables.py.
// C1 = 0x1.921fb54442e00p-4, C2 = -0x1.cf72cece675d2p-49
static __device__ const double2 kBmCosTab[33] = {
    {0x1.0000000000000p+0, 0x0.0p+0},  // k = 0
    {0x1.fd88da3d12526p-1, 0x1.917a6bc29b42cp-4},  // k = 1
    {0x1.f6297cff75cb0p-1, 0x1.8f8b83c69a60bp-3},  // k = 2
    {0x1.e9f4156c62ddap-1, 0x1.294062ed59f06p-2},  // k = 3
    {0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2},  // k = 4
    {0x1.c38b2f180bdb1p-1, 0x1.e2b5d3806f63bp-2},  // k = 5
    {0x1.a9b66290ea1a3p-1, 0x1.1c73b39ae68c8p-1},  // k = 6
    {0x1.8bc806b151741p-1, 0x1.44cf325091dd6p-1},  // k = 7
    {0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1},  // k = 8
    {0x1.44cf325091dd6p-1, 0x1.8bc806b151741p-1},  // k = 9
    {0x1.1c73b39ae68c8p-1, 0x1.a9b66290ea1a3p-1},  // k = 10
    {0x1.e2b5d3806f63bp-2, 0x1.c38b2f180bdb1p-1},  // k = 11
    {0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1},  // k = 12
    {0x1.294062ed59f06p-2, 0x1.e9f4156c62ddap-1},  // k = 13
    {0x1.8f8b83c69a60bp-3, 0x1.f6297cff75cb0p-1},  // k = 14
    {0x1.917a6bc29b42cp-4, 0x1.fd88da3d12526p-1},  // k = 15
    {0x0.0p+0, 0x1.0000000000000p+0},  // k = 16
    {-0x1.917a6bc29b42cp-4, 0x1.fd88da3d12526p-1},  // k = 17
    {-0x1.8f8b83c69a60bp-3, 0x1.f6297cff75cb0p-1},  // k = 18
    {-0x1.294062ed59f06p-2, 0x1.e9f4156c62ddap-1},  // k = 19
    {-0x1.87de2a6aea963p-2, 0x1.d906bcf328d46p-1},  // k = 20
    {-0x1.e2b5d3806f63bp-2, 0x1.c38b2f180bdb1p-1},  // k = 21
    {-0x1.1c73b39ae68c8p-1, 0x1.a9b66290ea1a3p-1},  // k = 22
    {-0x1.44cf325091dd6p-1, 0x1.8bc806b151741p-1},  // k = 23
    {-0x1.6a09e667f3bcdp-1, 0x1.6a09e667f3bcdp-1},  // k = 24
    {-0x1.8bc806b151741p-1, 0x1.44cf325091dd6p-1},  // k = 25
    {-0x1.a9b66290ea1a3p-1, 0x1.1c73b39ae68c8p-1},  // k = 26
    {-0x1.c38b2f180bdb1p-1, 0x1.e2b5d3806f63bp-2},  // k = 27
    {-0x1.d906bcf328d46p-1, 0x1.87de2a6aea963p-2},  // k = 28
    {-0x1.e9f4156c62ddap-1, 0x1.294062ed59f06p-2},  // k = 29
    {-0x1.f6297cff75cb0p-1, 0x1.8f8b83c69a60bp-3},  // k = 30
    {-0x1.fd88da3d12526p-1, 0x1.917a6bc29b42cp-4},  // k = 31
    {-0x1.0000000000000p+0, 0x0.0p+0},  // k = 32
};
static __constant__ double kBmCosC[8] = {1.0 / 40320, -1.0 / 720, 1.0 / 24, -0.5,
                                          1.0 / 362880, -1.0 / 5040, 1.0 / 120, -1.0 / 6};
__device__ __forceinline__ double bm_cos(double t, uint64_t w2) {
  const int k = (int)((w2 + (1ull << 46)) >> 47);  // round(64 u2), 0..64
  const double dk = (double)k;
  const double r = fma(-dk, -0x1.cf72cece675d2p-49, fma(-dk, 0x1.921fb54442e00p-4, t));
  const double2 cs = __ldg(&kBmCosTab[k <= 32 ? k : 64 - k]);
  const double r2 = r * r;
  const double cr = fma(fma(fma(fma(r2, kBmCosC[0], kBmCosC[1]), r2, kBmCosC[2]), r2, kBmCosC[3]), r2, 1.0);
  const double sp = fma(fma(fma(r2, kBmCosC[4], kBmCosC[5]), r2, kBmCosC[6]), r2, kBmCosC[7]);
  const double sr = fma(r * r2, sp, r);
  return fma(k <= 32 ? -cs.y : cs.y, sr, cs.x * cr);
}

// Standard normal #j: uniforms at counters 2j, 2j+1, Box-Muller cosine branch (_kernels.pyx:49-69):
// z = sqrt(-2 log u1) cos(2 pi u2) with the same rounding of u1, u2 and 2 pi u2 as the reference; log
// and cos are the domain-specialised bm_log / bm_cos (few-ulp, ~100 instructions per normal instead of
// ~250 with the general libdevice versions).  Agreement with the reference's libm: |dz| <= ~1e-15.
// sqrt(x) for x in [1e-16, 80] (the Box-Muller radius argument -2 log u1): MUFU approximation of 1/sqrt,
// two Newton steps, then one residual correction of s = x y — within 1 ulp of the correctly rounded root,
// and branch-free (the IEEE sqrt's special-value path is a call), so the generator stays one basic block.
__device__ __forceinline__ double bm_sqrt(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  const double s = x * y;
  return fma(0.5 * y, fma(-s, s, x), s);
}

// kTabLog selects the log form: the table one (fewer FP64 operations, two extra L1 loads) is faster for the
// standalone generator and the narrow sketch slabs; inside the n = 200 contraction the polynomial one is
// (its slabs already keep the shared-memory / L1 path busy).  Both within ~1 ulp of libm.
template <bool kTabLog = true>
__device__ __forceinline__ double rng_normal(uint64_t stream, uint64_t j) {
  double u1 = __dmul_rn(__dadd_rn((double)(rng_word(stream, 2 * j) >> 11), 0.5), kInv2p53);
  const uint64_t w2 = rng_word(stream, 2 * j + 1) >> 11;
  double u2 = __dmul_rn((double)w2, kInv2p53);
  const double lg = kTabLog ? bm_log_tab(u1) : bm_log_poly(u1);
  return __dmul_rn(bm_sqrt(__dmul_rn(-2.0, lg)), bm_cos(__dmul_rn(kTwoPi, u2), w2));
}

// Single-precision Box-Muller on the same counters (2j, 2j+1), used ONLY by the synthetic-data
// generator (BASELINE.json configs need ~1e10 Gaussians per run; the sketch's G always uses the
// fp64 rng_normal above).  Mirrored by oracle/tsnmf_oracle.py normal_block_f32.
__device__ __forceinline__ float rng_normal_f32(uint64_t stream, uint64_t j) {
  const float u1 = __fmul_rn(__fadd_rn((float)(rng_word(stream, 2 * j) >> 40), 0.5f), 5.9604644775390625e-08f);
  const float u2 = __fmul_rn((float)(rng_word(stream, 2 * j + 1) >> 40), 5.9604644775390625e-08f);
  return __fmul_rn(sqrtf(__fmul_rn(-2.0f, logf(u1))), cosf(__fmul_rn(6.2831855f, u2)));
}

// Stream tags (rng.py:20-23) plus the config-generator tags (>= 4).
constexpr uint64_t kTagSketch = 0;
constexpr uint64_t kTagCfgW = 4, kTagCfgNoise = 7;

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ __forceinline__ int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// smallest stride >= cols with stride % 16 == 8 (doubles): conflict-free DMMA fragment loads
// (lane l reads row l%4, col l/4) and 16-byte C-tile accesses (row l/4, col 2*(l%4)).
__host__ __device__ __forceinline__ int smem_stride(int cols) {
  int s = cols;
  while (s % 16 != 8) ++s;
  return s;
}

// 1/sqrt(a), 1/a for the Householder scalars (a > 0, any finite magnitude incl. subnormal) without
// branches: the argument is scaled by an even power of two into the range where the .ftz approximation +
// two Newton steps is accurate (<= 2 ulp vs IEEE, tools/probe_rsqrt.cu), and the result scaled back
// exactly.  Branch-free so a column step stays one basic block and the scheduler can overlap off-chain
// work with the scalar chain.  (A single third-order correction step instead of two Newton steps, with
// the range-scaled copy computed beside the chain, measured no faster and spills in the narrow kernels.)
__device__ __forceinline__ double rsqrt_nb(double a) {
  const double sc = a < 0x1p-900 ? 0x1p+600 : (a > 0x1p+900 ? 0x1p-600 : 1.0);
  const double as = a * sc * sc;
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(as));
  const double h = 0.5 * as;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y * sc;
}
__device__ __forceinline__ double rcp_nb(double a) {
  const double sc = a < 0x1p-900 ? 0x1p+600 : (a > 0x1p+900 ? 0x1p-600 : 1.0);
  const double as = a * sc;
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(as));
  y = y * fma(-as, y, 2.0);
  y = y * fma(-as, y, 2.0);
  return y * sc;
}

// L2 eviction-priority policies (createpolicy) and hinted global accesses: streamed-once data (X) is
// evict_first so it does not push out the re-used working set (TSQR R slots, split-leaf workspace tiles),
// which is evict_last.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_hint(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}

// cp.async helpers (LDGSTS): global -> shared without staging through registers.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16_hint(void* smem, const void* gmem, uint64_t pol) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void cp_async8_hint(void* smem, const void* gmem, uint64_t pol) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "l"(pol));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Bulk (TMA engine) copies global -> shared completed on an mbarrier (transaction bytes).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// Every lane spins on the parity; the caller re-converges the warp (__syncwarp) afterwards.
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Order this thread's (and, after a warp barrier, its warp's) earlier generic-proxy shared-memory accesses
// before later async-proxy (bulk copy) writes to the same buffer.
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
// bytes % 16 == 0, both addresses 16-byte aligned
__device__ __forceinline__ void bulk_copy_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// XOR swizzle of shared-memory row blocks (stride % 16 == 8 doubles): column c of row r lives at
// r*lds + swz_col(r, c).  Makes the DMMA operand slabs (lane: row l%4, col l/4), V fragments
// (row l/4, col l%4) and 16-byte C-tile rows (row l/4, col 2*(l%4)) conflict-free; XOR by 0 or 4 stays
// inside aligned 8-column groups so 16-byte pairs are preserved.
__host__ __device__ __forceinline__ int swz_row(int row) { return (row & 2) << 1; }
__host__ __device__ __forceinline__ int swz_col(int row, int col) { return col ^ swz_row(row); }

// Row-major walk over the cells {start, start + step, ...} of a grid with w columns, with one division
// up front and a carry per step instead of a division per cell (the staging loops below issue one
// cp.async per cell, so the index math is their cost).
struct GridWalk {
  int r, c, dr, dc, w;
  __device__ __forceinline__ GridWalk(int start, int step, int w_) : w(w_) {
    r = start / w;
    c = start - r * w;
    dr = step / w;
    dc = step - dr * w;
  }
  __device__ __forceinline__ void next() {
    r += dr;
    c += dc;
    if (c >= w) {
      c -= w;
      ++r;
    }
  }
};

// Stage rows [0, nrows) x cols [0, ncols) of a row-major global matrix into shared memory with row
// stride lds (swizzled: column c of row r at r*lds + swz_col(r, c)); rows [nrows, rows_total) and cols
// [ncols, cols_total) are zero-filled.  cols_total must be a multiple of 8.  All threads of the CTA
// participate; the caller commits / waits.
template <bool kSwz, bool kStream = false>
__device__ __forceinline__ void stage_rows_impl(double* __restrict__ dst, int lds, const double* __restrict__ src,
                                                int64_t ldsrc, int nrows, int ncols, int rows_total,
                                                int cols_total, bool vec16) {
  const int tid = threadIdx.x, nth = blockDim.x;
  auto at = [&](int r, int c) -> double* { return dst + (int64_t)r * lds + (kSwz ? swz_col(r, c) : c); };
  const uint64_t pol = kStream ? l2_policy_evict_first() : 0;
  if (vec16) {
    const int pairs = ncols >> 1;
    if (pairs > 0)
      for (GridWalk it(tid, nth, pairs); it.r < nrows; it.next()) {
        if (kStream)
          cp_async16_hint(at(it.r, 2 * it.c), src + it.r * ldsrc + 2 * it.c, pol);
        else
          cp_async16(at(it.r, 2 * it.c), src + it.r * ldsrc + 2 * it.c);
      }
    if (ncols & 1)
      for (int r = tid; r < nrows; r += nth) cp_async8(at(r, ncols - 1), src + r * ldsrc + ncols - 1);
  } else if (ncols > 0) {
    for (GridWalk it(tid, nth, ncols); it.r < nrows; it.next()) {
      if (kStream)
        cp_async8_hint(at(it.r, it.c), src + it.r * ldsrc + it.c, pol);
      else
        cp_async8(at(it.r, it.c), src + it.r * ldsrc + it.c);
    }
  }
  const int pad = cols_total - ncols;
  if (pad > 0)
    for (GridWalk it(tid, nth, pad); it.r < nrows; it.next()) *at(it.r, ncols + it.c) = 0.0;
  if (rows_total > nrows && cols_total > 0)
    for (GridWalk it(tid, nth, cols_total); it.r < rows_total - nrows; it.next()) *at(nrows + it.r, it.c) = 0.0;
}

__device__ __forceinline__ void stage_rows_swz(double* __restrict__ dst, int lds, const double* __restrict__ src,
                                               int64_t ldsrc, int nrows, int ncols, int rows_total,
                                               int cols_total, bool vec16) {
  stage_rows_impl<true>(dst, lds, src, ldsrc, nrows, ncols, rows_total, cols_total, vec16);
}
// the same for streamed-once input (L2 evict_first)
__device__ __forceinline__ void stage_rows_swz_stream(double* __restrict__ dst, int lds, const double* __restrict__ src,
                                                      int64_t ldsrc, int nrows, int ncols, int rows_total,
                                                      int cols_total, bool vec16) {
  stage_rows_impl<true, true>(dst, lds, src, ldsrc, nrows, ncols, rows_total, cols_total, vec16);
}

}  // namespace tsnmf

/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, imported by, or
 * called from the product path (paper_1402_6964_b200/).  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load it, and only as the checker or the CPU baseline.
 *
 * Plain-C restatement of the reference's counter-based random streams:
 *   splitmix64 finaliser      reference pkg/src/tsnmf/_kernels.pyx:21-28
 *   word(s, c)                reference pkg/src/tsnmf/_kernels.pyx:31-32
 *   uniform_block             reference pkg/src/tsnmf/_kernels.pyx:35-46
 *   normal_block (Box-Muller) reference pkg/src/tsnmf/_kernels.pyx:49-69
 *   derive_stream             reference pkg/src/tsnmf/rng.py:33-35
 *   gaussian_rows addressing  reference pkg/src/tsnmf/rng.py:48-55
 * plus a sketch accumulator (G^T X with G regenerated per row), restating
 * reference pkg/src/tsnmf/sketch.py:62-73, used as the CPU baseline for GX.
 *
 * Pinned against the live reference by tests/golden/rng.npz (uniforms
 * bit-exact, normals within the reference's own backend tolerance
 * rtol 1e-12 / atol 1e-13, reference tests/test_kernels.py:40-49).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#define GAMMA 0x9E3779B97F4A7C15ULL
static const double TWO_PI = 6.283185307179586476925286766559;
static const double INV_2_53 = 1.0 / 9007199254740992.0;

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

static inline uint64_t word_at(uint64_t stream, uint64_t ctr) {
  return mix64(stream + (ctr + 1) * GAMMA);
}

uint64_t oracle_derive_stream(uint64_t seed, uint64_t tag) {
  return mix64(seed ^ mix64(tag + GAMMA));
}

void oracle_uniform_block(uint64_t stream, uint64_t start, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i)
    out[i] = (double)(word_at(stream, start + (uint64_t)i) >> 11) * INV_2_53;
}

static inline double normal_at(uint64_t stream, uint64_t j) {
  double u1 = ((double)(word_at(stream, 2 * j) >> 11) + 0.5) * INV_2_53;
  double u2 = (double)(word_at(stream, 2 * j + 1) >> 11) * INV_2_53;
  return sqrt(-2.0 * log(u1)) * cos(TWO_PI * u2);
}

void oracle_normal_block(uint64_t stream, uint64_t start, int64_t count, double* out) {
  for (int64_t i = 0; i < count; ++i) out[i] = normal_at(stream, start + (uint64_t)i);
}

/* S (k x n, row-major) += G^T X for rows [row_offset, row_offset + rows) of the
 * sketch stream; G[i, t] = normal index (row_offset + i) * k + t.  g is a
 * caller-provided scratch of k doubles. */
void oracle_sketch_accumulate(uint64_t stream, const double* x, int64_t rows, int32_t n,
                              int64_t row_offset, int32_t k, double* s, double* g) {
  for (int64_t i = 0; i < rows; ++i) {
    uint64_t base = (uint64_t)(row_offset + i) * (uint64_t)k;
    for (int32_t t = 0; t < k; ++t) g[t] = normal_at(stream, base + (uint64_t)t);
    const double* xi = x + i * (int64_t)n;
    for (int32_t t = 0; t < k; ++t) {
      double gt = g[t];
      double* st = s + (int64_t)t * n;
      for (int32_t j = 0; j < n; ++j) st[j] += gt * xi[j];
    }
  }
}

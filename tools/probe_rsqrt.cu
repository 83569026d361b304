// Accuracy of the Householder-scalar helpers (common.cuh rsqrt_nb / rcp_nb) against IEEE
// 1/sqrt(a) and 1/a (correctly rounded __dsqrt_rn / __drcp_rn), in ulps, over random arguments spanning
// the whole positive double range (incl. subnormals).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include "../paper_1402_6964_b200/csrc/common.cuh"
using namespace tsnmf;
__device__ double ulp_err(double got, double want) {
  const long long g = __double_as_longlong(got), w = __double_as_longlong(want);
  return (double)llabs(g - w);
}
__global__ void probe(uint64_t seed, int per, unsigned long long* out) {
  double e1 = 0, e2 = 0;
  const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int i = 0; i < per; ++i) {
    const uint64_t w = mix64(seed + (t * per + i) * 0x9E3779B97F4A7C15ULL);
    // random positive finite double: exponent field 0..2046, random mantissa
    uint64_t bits = (w & 0x000FFFFFFFFFFFFFULL) | (((w >> 52) % 2047ULL) << 52);
    if ((w >> 63) & 1) bits = (w & 0x000FFFFFFFFFFFFFULL) | (((w >> 52) % 64ULL + 991ULL) << 52);  // near 1
    const double a = __longlong_as_double((long long)bits);
    if (!(a > 0.0)) continue;
    const double rs = __drcp_rn(__dsqrt_rn(a));
    if (isfinite(rs) && rs > 0x1p-1022) e1 = fmax(e1, ulp_err(rsqrt_nb(a), rs));
    const double rc = __drcp_rn(a);
    if (isfinite(rc) && rc > 0x1p-1022) e2 = fmax(e2, ulp_err(rcp_nb(a), rc));
  }
  atomicMax(out, (unsigned long long)e1);
  atomicMax(out + 1, (unsigned long long)e2);
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaMemset(d, 0, 16);
  probe<<<1184, 256>>>(12345, 256, d);
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("rsqrt_nb max err %llu ulp (vs rcp(sqrt) which itself may be 1 ulp off), rcp_nb max err %llu ulp, %d samples\n",
         h[0], h[1], 1184 * 256 * 256);
  return 0;
}

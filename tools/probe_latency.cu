// Dependent-chain latencies (cycles) of the ops on the TSQR panel's critical path, sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
  double x = a + threadIdx.x;
  long long t0, t1;
  unsigned u = threadIdx.x;
  __shared__ double sm[64];
  sm[threadIdx.x % 64] = x;
  __syncwarp();
  // DFMA chain
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = fma(x, a, b); t1 = clock64(); cyc[0] = (t1 - t0) / iters;
  // DADD chain
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = x + b; t1 = clock64(); cyc[1] = (t1 - t0) / iters;
  // SHFL 64-bit chain
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffff, x, 1) + 0.0; t1 = clock64(); cyc[2] = (t1 - t0) / iters;
  // sqrt chain
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = sqrt(x + 2.0); t1 = clock64(); cyc[3] = (t1 - t0) / iters;
  // div chain
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = 3.0 / (x + 1.5); t1 = clock64(); cyc[4] = (t1 - t0) / iters;
  // rcp approx chain
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = __drcp_rn(x + 1.5); t1 = clock64(); cyc[5] = (t1 - t0) / iters;
  // LDS chain
  int idx = threadIdx.x % 64;
  t0 = clock64(); for (int i = 0; i < iters; ++i) { idx = ((int)sm[idx] + i) & 63; } t1 = clock64(); cyc[6] = (t1 - t0) / iters;
  // rsqrt via MUFU
  t0 = clock64(); for (int i = 0; i < iters; ++i) x = rsqrt(x + 2.0); t1 = clock64(); cyc[7] = (t1 - t0) / iters;
  // shfl 32-bit
  t0 = clock64(); for (int i = 0; i < iters; ++i) u = __shfl_xor_sync(0xffffffff, u, 1) + 1; t1 = clock64(); cyc[8] = (t1 - t0) / iters;
  // DMMA chain
  double c0 = 0, c1 = 0;
  t0 = clock64(); for (int i = 0; i < iters; ++i) asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b)); t1 = clock64(); cyc[9] = (t1 - t0) / iters;
  // bar.sync (single warp)
  t0 = clock64(); for (int i = 0; i < iters; ++i) __syncthreads(); t1 = clock64(); cyc[10] = (t1 - t0) / iters;
  out[threadIdx.x] = x + idx + u + c0 + c1;
}
int main() {
  double* out; long long* cyc; cudaMalloc(&out, 8 * 256); cudaMallocManaged(&cyc, 8 * 16);
  lat<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, 1000);
  cudaDeviceSynchronize();
  lat<<<1, 32>>>(out, cyc, 1.0000001, 1e-9, 1000);
  cudaDeviceSynchronize();
  const char* names[] = {"DFMA", "DADD", "SHFL64+DADD", "sqrt(double)", "div(double)", "__drcp_rn", "LDS(+cvt)", "rsqrt(double)", "SHFL32+IADD", "DMMA 8x8x4", "bar.sync(1 warp)"};
  for (int i = 0; i < 11; ++i) printf("%-18s %lld cycles\n", names[i], cyc[i]);
  return 0;
}

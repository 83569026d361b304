// DMMA m8n8k4 throughput vs resident warps per SM and independent accumulators per warp (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
template <int ACC>
__global__ void k(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[ACC][2];
#pragma unroll
  for (int t = 0; t < ACC; ++t) c[t][0] = c[t][1] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < ACC; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < ACC; ++t) s += c[t][0] + c[t][1];
  if (s == 1.2345) out[0] = s;
}
template <int ACC> void run(int warps_per_sm, double* out) {
  int sms = 148, tpb = warps_per_sm * 32 > 1024 ? 1024 : warps_per_sm * 32;
  int blocks = sms * (warps_per_sm * 32 / tpb);
  int iters = 4096 / ACC * 8;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<ACC><<<blocks, tpb>>>(out, 16); cudaDeviceSynchronize();
  cudaEventRecord(e0); k<ACC><<<blocks, tpb>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 256 * ACC * (double)iters * blocks * (tpb / 32);
  printf("warps/SM %3d  acc/warp %2d : %6.2f TF/s\n", warps_per_sm, ACC, flops / ms / 1e9);
}
int main() {
  double* out; cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16, 32}) { run<4>(w, out); run<8>(w, out); run<16>(w, out); run<32>(w, out); }
  return 0;
}

// Microbenchmark: FP64 DFMA vs DMMA (mma.sync m8n8k4 f64) throughput and HBM read bandwidth on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 1.2345) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 1.2345) out[0] = s;
}

__global__ void read_kernel(const double2* __restrict__ x, size_t n2, double* out) {
  double acc = 0;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride * 4) {
    double2 v0 = __ldcs(x + i);
    double2 v1 = (i + stride < n2) ? __ldcs(x + i + stride) : make_double2(0, 0);
    double2 v2 = (i + 2 * stride < n2) ? __ldcs(x + i + 2 * stride) : make_double2(0, 0);
    double2 v3 = (i + 3 * stride < n2) ? __ldcs(x + i + 3 * stride) : make_double2(0, 0);
    acc += v0.x + v0.y + v1.x + v1.y + v2.x + v2.y + v3.x + v3.y;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s sms %d smemOptin %zu l2 %d regsPerSM %d clock %d kHz memclk %d kHz busw %d\n", p.name, p.multiProcessorCount,
         p.sharedMemPerBlockOptin, p.l2CacheSize, p.regsPerMultiprocessor, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int tpb : {128, 256, 512}) {
    int blocks = sms * (2048 / tpb); int iters = 4096;
    dfma_kernel<<<blocks, tpb>>>(out, 16, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, tpb>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * iters * (double)blocks * tpb;
    printf("DFMA tpb=%d: %.2f TFLOP/s (%.3f ms)\n", tpb, flops / ms / 1e9, ms);
  }
  for (int wpb : {4, 8, 16}) {
    int tpb = wpb * 32; int blocks = sms * (64 / wpb); int iters = 2048;
    dmma_kernel<<<blocks, tpb>>>(out, 16);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    dmma_kernel<<<blocks, tpb>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 8 * (double)iters * blocks * wpb;
    printf("DMMA m8n8k4 warps/blk=%d: %.2f TFLOP/s (%.3f ms)\n", wpb, flops / ms / 1e9, ms);
  }
  size_t bytes = (size_t)8 << 30; double2* x; CK(cudaMalloc(&x, bytes)); CK(cudaMemset(x, 0, bytes));
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    read_kernel<<<sms * 8, 256>>>(x, bytes / 16, out);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("HBM read 8 GiB: %.1f GB/s\n", bytes / ms / 1e6);
  }
  return 0;
}

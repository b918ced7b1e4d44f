// Microbenchmark: FP64 FMA throughput and HBM copy bandwidth on the box.
// Used once to set the ALU roofline denominators in DESIGN.md.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) b[i] = a[i];
}
int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("name=%s sms=%d l2=%d smem_optin=%zu clock_khz=%d\n", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerBlockOptin, p.clockRate);
  double* out; cudaMalloc(&out, 148 * 8 * 1024 * 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int bs : {256, 512, 1024}) for (int bpsm : {1, 2, 4, 8}) {
    if (bs * bpsm > 2048) continue;
    int grid = p.multiProcessorCount * bpsm;
    dfma_loop<<<grid, bs>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<<<grid, bs>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 64 * (double)iters * grid * bs;
    printf("dfma bs=%d bpsm=%d : %.2f TFLOP/s (%.3f ms)\n", bs, bpsm, flops / ms / 1e9, ms);
  }
  size_t n = (size_t)1 << 28;  // 2^28 double2 = 4 GiB
  double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16);
  cudaMemset(a, 0, n * 16);
  for (int g : {148 * 4, 148 * 8, 148 * 16}) {
    copy_k<<<g, 512>>>(a, b, n);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) copy_k<<<g, 512>>>(a, b, n);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("copy grid=%d: %.1f GB/s\n", g, 5.0 * 2 * n * 16 / ms / 1e6);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

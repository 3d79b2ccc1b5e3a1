// Microbenchmark: FP64 FMA issue rate, shared-memory fp64 load rate, HBM copy.
// Used once to calibrate the apply-kernel design.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void lds_kernel(double* out, int iters) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = i;
  __syncthreads();
  double acc = 0; int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) { acc += s[(idx + k * 33) & 1023]; }
    idx = (idx + 7) & 1023;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int dev = 0; cudaDeviceProp prop; cudaGetDeviceProperties(&prop, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("%s SMs=%d clock(kHz)=%d\n", prop.name, prop.multiProcessorCount, clk);
  int sms = prop.multiProcessorCount;
  double* out; cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int bpsm : {4, 8}) {
    int blocks = sms * bpsm, threads = 256, iters = 2000;
    dfma_kernel<<<blocks, threads>>>(out, 10, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 16 * 8;
    printf("DFMA blocks/SM=%d: %.3f ms, %.2f TFMA/s = %.2f TFLOP/s, %.1f FMA/clk/SM at nominal clock\n", bpsm, ms,
           fmas / ms / 1e9, 2 * fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / (clk * 1e3));
  }
  {
    int blocks = sms * 8, threads = 256, iters = 2000;
    lds_kernel<<<blocks, threads>>>(out, 10);
    cudaEventRecord(e0); lds_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    double lds = (double)blocks * threads * iters * 16;
    printf("LDS.64: %.3f ms, %.2f T doubles/s, %.1f doubles/clk/SM at nominal clock\n", ms, lds / ms / 1e9,
           lds / (ms * 1e-3) / sms / (clk * 1e3));
  }
  {
    size_t n = (size_t)1 << 27;  // 2^27 double2 = 2 GiB each
    double2 *a, *b; cudaMalloc(&a, n * 16); cudaMalloc(&b, n * 16); cudaMemset(a, 0, n * 16);
    for (int r = 0; r < 3; ++r) copy_kernel<<<sms * 8, 256>>>(a, b, n);
    float best = 1e9;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0); copy_kernel<<<sms * 8, 256>>>(a, b, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("copy: %.3f ms, %.1f GB/s (read+write)\n", best, 2.0 * n * 16 / best / 1e6);
  }
  cudaError_t err = cudaGetLastError(); printf("err=%s\n", cudaGetErrorString(err));
  return 0;
}

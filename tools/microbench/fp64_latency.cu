// Dependent-DFMA latency and the issue cost of a line-solve-like step on one warp (B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_latency fp64_latency.cu && ./fp64_latency
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_chain(double* out, long long* cyc, double a, double b, int n) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// W = 3 recurrence step as in band_sweep_s: one dependent DFMA per step plus two independent ones
__global__ void k_step(double* out, long long* cyc, double g0, double g1, double g2, int n) {
  __shared__ double tile[4096];
  for (int i = threadIdx.x; i < 4096; i += 32) tile[i] = 1e-3 * i;
  __syncwarp();
  double a0 = out[threadIdx.x], a1 = a0 * 0.5, a2 = a0 * 0.25;
  long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < n; ++i) {
    const double v = a0;
    const double e = tile[((i + 3) * 32 + threadIdx.x) & 4095];
    a0 = fma(-g0, v, a1);
    a1 = fma(-g1, v, a2);
    a2 = fma(-g2, v, e);
    tile[(i * 32 + threadIdx.x) & 4095] = v;
  }
  long long t1 = clock64();
  out[threadIdx.x] = a0 + a1 + a2;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMalloc(&cyc, 8 * 64);
  cudaMemset(out, 0, 32 * 8);
  const int n = 4096;
  long long h[64];
  for (int warps = 1; warps <= 1; ++warps) {
    k_chain<<<1, 32>>>(out, cyc, 0.999, 1e-3, n);
    k_chain<<<1, 32>>>(out, cyc, 0.999, 1e-3, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("dependent DFMA: %.2f cycles per DFMA (1 warp)\n", (double)h[0] / n);
    k_step<<<1, 32>>>(out, cyc, 0.3, 0.2, 0.1, n);
    k_step<<<1, 32>>>(out, cyc, 0.3, 0.2, 0.1, n);
    cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("line-solve step (W=3): %.2f cycles per step (1 warp per SM)\n", (double)h[0] / n);
  }
  for (int nb : {148, 148 * 5}) {
    k_step<<<nb, 32>>>(out, cyc, 0.3, 0.2, 0.1, n);
    cudaDeviceSynchronize();
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}

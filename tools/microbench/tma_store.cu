// Does a TMA tensor store / tensor reduce-add (f64) of a {32, m, 1} box work on sm_100a, with the box
// (a) inside the tensor, (b) hanging over the end of the innermost dimension, (c) starting at a
// negative row?   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_store tma_store.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ unsigned u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) k_st(const __grid_constant__ CUtensorMap tm, int i0, int r0, int o, int red, int n) {
  extern __shared__ __align__(128) double sh[];
  for (int i = threadIdx.x; i < n; i += 32) sh[i] = 1.0 + i;
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  __syncwarp();
  if (threadIdx.x == 0) {
    if (red)
      asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::
                       "l"((unsigned long long)&tm), "r"(i0), "r"(r0), "r"(o), "r"(u32(sh)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::
                       "l"((unsigned long long)&tm), "r"(i0), "r"(r0), "r"(o), "r"(u32(sh)) : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}

int main(int argc, char** argv) {
  const int which = argc > 1 ? atoi(argv[1]) : 0;
  const int m = 162, inner = 162, outer = 3, rows = which == 2 ? m + 6 : m;
  const size_t N = (size_t)outer * m * inner;
  double* x;
  cudaMalloc(&x, N * 8);
  std::vector<double> h(N, 100.0);
  cudaMemcpy(x, h.data(), N * 8, cudaMemcpyHostToDevice);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  CUtensorMap tm;
  const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)m, (cuuint64_t)outer};
  const cuuint64_t strides[2] = {(cuuint64_t)inner * 8, (cuuint64_t)inner * m * 8};
  const cuuint32_t box[3] = {32u, (cuuint32_t)rows, 1u};
  const cuuint32_t es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
  const int n = 32 * rows;
  // which: 0 store inside, 1 store over the end of the row (i0 = 160: 2 valid lines), 2 store from row -3,
  //        3 reduce inside, 4 reduce over the end
  const int i0 = (which == 1 || which == 4) ? 160 : 32, r0 = which == 2 ? -3 : 0, red = which >= 3;
  k_st<<<1, 32, n * 8>>>(tm, i0, r0, 1, red, n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("case %d: %s\n", which, cudaGetErrorString(e));
  if (e != cudaSuccess) return 0;
  cudaMemcpy(h.data(), x, N * 8, cudaMemcpyDeviceToHost);
  // element (o=1, k, i): expect sh[(k - r0) * 32 + (i - i0)] (+100 when reduce)
  int bad = 0, touched = 0;
  for (int k = 0; k < m; ++k)
    for (int i = 0; i < inner; ++i) {
      const double v = h[((size_t)1 * m + k) * inner + i];
      const bool in = i >= i0 && i < i0 + 32;
      const double want = in ? (1.0 + (k - r0) * 32 + (i - i0)) + (red ? 100.0 : 0.0) : 100.0;
      bad += v != want;
      touched += v != 100.0;
    }
  for (size_t j = 0; j < (size_t)m * inner; ++j) bad += h[j] != 100.0;   // o = 0 untouched
  printf("case %d: touched %d, mismatches %d\n", which, touched, bad);
  return 0;
}

// TMA load bandwidth of [outer][m][inner] fp64 tiles {BW lines, m rows} as a function of the
// contiguous row length BW*8 bytes (line-solve access pattern along a strided axis).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rows tma_rows.cu && ./tma_rows
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ unsigned u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(32) k_load(const __grid_constant__ CUtensorMap tm, int tiles_per_outer, long long ntiles,
                                             unsigned bytes, int rows_per_box, int nbox, int BW, double* sink) {
  extern __shared__ __align__(128) double sh[];
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sh + bytes / 8);
  const int lane = threadIdx.x;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(u32(mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  unsigned phase = 0;
  double acc = 0.0;
  for (long long g = blockIdx.x; g < ntiles; g += gridDim.x) {
    const int o = (int)(g / tiles_per_outer), i0 = (int)(g % tiles_per_outer) * BW;
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(u32(mbar)), "r"(bytes) : "memory");
      for (int b = 0; b < nbox; ++b)
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::
                "r"(u32(sh + (size_t)b * rows_per_box * BW)), "l"((unsigned long long)&tm), "r"(i0), "r"(b * rows_per_box),
            "r"(o), "r"(u32(mbar))
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra WAIT_%=;\n}\n" ::"r"(
            u32(mbar)),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    acc += sh[lane];
    __syncwarp();
  }
  if (acc == 123.456) sink[0] = acc;
}

int main() {
  const int m = 162;
  const long long inner = (long long)m * m, outer = 9;   // 3 x axis 0 of config 4 (306 MB > L2): rows 209,952 B apart
  const size_t N = (size_t)outer * m * inner;
  double *x, *sink;
  cudaMalloc(&x, N * 8);
  cudaMalloc(&sink, 8);
  cudaMemset(x, 0, N * 8);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)p;
  for (int axis = 0; axis < 2; ++axis) {
    const long long in = axis == 0 ? inner : m, ou = axis == 0 ? outer : outer * m;
    for (int BW : {32, 64, 128}) {
      const int rows_per_box = 81, nbox = 2;
      CUtensorMap tm;
      const cuuint64_t dims[3] = {(cuuint64_t)in, (cuuint64_t)m, (cuuint64_t)ou};
      const cuuint64_t strides[2] = {(cuuint64_t)in * 8, (cuuint64_t)in * m * 8};
      const cuuint32_t box[3] = {(cuuint32_t)BW, (cuuint32_t)rows_per_box, 1u};
      const cuuint32_t es[3] = {1, 1, 1};
      CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                       CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
      const unsigned bytes = (unsigned)(BW * m * 8);
      const size_t smem = bytes + 16;
      cudaFuncSetAttribute(k_load, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_load, 32, smem);
      const int tpo = (int)((in + BW - 1) / BW);
      const long long ntiles = ou * tpo;
      const int grid = (int)(ntiles < (long long)occ * 148 ? ntiles : (long long)occ * 148);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      k_load<<<grid, 32, smem>>>(tm, tpo, ntiles, bytes, rows_per_box, nbox, BW, sink);
      cudaEventRecord(e0);
      for (int it = 0; it < 10; ++it) k_load<<<grid, 32, smem>>>(tm, tpo, ntiles, bytes, rows_per_box, nbox, BW, sink);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("axis %d rows of %4d B: %d CTAs/SM, %.1f us per pass, %.0f GB/s (%s)\n", axis, BW * 8, occ, 100.0 * ms,
             N * 8.0 / (ms / 10 * 1e-3) / 1e9, cudaGetErrorString(e));
    }
  }
  return 0;
}

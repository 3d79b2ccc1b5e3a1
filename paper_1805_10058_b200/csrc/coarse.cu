// R5: exact solve on the coarsest level.  The dense SPD matrix A_L is formed entry by
// entry from the level's 1D bands and the Kronecker patterns (the same operator the
// matrix-free kernels apply), inverted once at setup by the symmetric sweep operator
// (Gauss-Jordan without pivoting; pivots of an SPD matrix stay positive), and each
// V-cycle applies x = A_L^{-1} b as a dense matrix-vector product (one warp per row).
#include <vector>

#include "internal.cuh"

namespace igacd {

__device__ __forceinline__ double band_entry(const double* band, int p, int m, int k, int l) {
  const int o = l - k;
  if (o < -p || o > p) return 0.0;
  return band[(size_t)k * (2 * p + 1) + o + p];
}

__global__ void k_dense_coarse(OpParams op, int dim, int p, double* A, int N) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)N * N) return;
  const int I = (int)(idx / N), J = (int)(idx % N);
  const int m = op.m;
  const int ns = dim == 2 ? m * m : m * m * m;   // N = nc * ns
  const int i = I / ns, j = J / ns;
  int kI[3] = {0, 0, 0}, kJ[3] = {0, 0, 0};
  int fi = I % ns, fj = J % ns;
  for (int l = dim - 1; l >= 0; --l) {
    kI[l] = fi % m; fi /= m;
    kJ[l] = fj % m; fj /= m;
  }
  double Mv[3], Sv[3], Av[3];
  for (int l = 0; l < dim; ++l) {
    Mv[l] = band_entry(op.bM, p, m, kI[l], kJ[l]);
    Sv[l] = band_entry(op.bS, p, m, kI[l], kJ[l]);
    Av[l] = band_entry(op.bA, p, m, kI[l], kJ[l]);
  }
  double v;
  if (dim == 2) {
    v = op.c.mass[i][j] * Mv[0] * Mv[1] + op.c.S[0][i][j] * Sv[0] * Mv[1] + op.c.S[1][i][j] * Mv[0] * Sv[1] +
        op.c.AA[0][i][j] * Av[0] * Av[1];
  } else {
    v = op.c.mass[i][j] * Mv[0] * Mv[1] * Mv[2] + op.c.S[0][i][j] * Sv[0] * Mv[1] * Mv[2] +
        op.c.S[1][i][j] * Mv[0] * Sv[1] * Mv[2] + op.c.S[2][i][j] * Mv[0] * Mv[1] * Sv[2] +
        op.c.AA[0][i][j] * Av[0] * Av[1] * Mv[2] + op.c.AA[1][i][j] * Av[0] * Mv[1] * Av[2] +
        op.c.AA[2][i][j] * Mv[0] * Av[1] * Av[2];
  }
  A[idx] = v;
}

__global__ void k_sweep_save(const double* A, int N, int k, double* row, double* col, int* bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) {
    row[i] = A[(size_t)k * N + i];
    col[i] = A[(size_t)i * N + k];
  }
  if (i == 0 && !(A[(size_t)k * N + k] > 0.0)) *bad = 1;
}

// sweep on pivot k: A <- A - col row / piv off the pivot row/column;
// row k <- row/piv, column k <- -col/piv, pivot <- -1/piv (then negate at the end)
__global__ void k_sweep_apply(double* A, int N, int k, const double* row, const double* col) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)N * N) return;
  const int i = (int)(idx / N), j = (int)(idx % N);
  const double piv = row[k];
  double v;
  if (i == k && j == k) v = -1.0 / piv;
  else if (i == k) v = row[j] / piv;
  else if (j == k) v = col[i] / piv;
  else v = A[idx] - col[i] * row[j] / piv;
  A[idx] = v;
}

__global__ void k_negate_sym(double* A, int N) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= (long long)N * N) return;
  const int i = (int)(idx / N), j = (int)(idx % N);
  if (i <= j) {
    const double v = -0.5 * (A[idx] + A[(size_t)j * N + i]);
    A[idx] = v;
    A[(size_t)j * N + i] = v;
  }
}

__global__ void k_dense_matvec(const double* __restrict__ A, const double* __restrict__ b, double* __restrict__ x,
                               int N) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= N) return;
  const double* row = A + (size_t)warp * N;
  double s = 0.0;
  for (int j = lane; j < N; j += 32) s = fma(__ldg(row + j), __ldg(b + j), s);
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) x[warp] = s;
}

void build_coarse_inverse(Handle& h, int sy, cudaStream_t s) {
  System& S = h.sys[sy];
  SysLevel& L = S.lv.back();
  const int N = (int)L.ndof;
  IGACD_CUDA(cudaMalloc(&S.cinv, sizeof(double) * (size_t)N * N));
  double* cinv = S.cinv;
  const long long NN = (long long)N * N;
  const int bs = 256;
  const unsigned gb = (unsigned)((NN + bs - 1) / bs);
  k_dense_coarse<<<gb, bs, 0, s>>>(L.op, h.dim, h.p, cinv, N);
  IGACD_LAUNCH_CHECK();
  count_launch(h);
  double *row, *col;
  int* bad;
  IGACD_CUDA(cudaMalloc(&row, sizeof(double) * N));
  IGACD_CUDA(cudaMalloc(&col, sizeof(double) * N));
  IGACD_CUDA(cudaMalloc(&bad, sizeof(int)));
  IGACD_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  for (int k = 0; k < N; ++k) {
    k_sweep_save<<<(N + bs - 1) / bs, bs, 0, s>>>(cinv, N, k, row, col, bad);
    k_sweep_apply<<<gb, bs, 0, s>>>(cinv, N, k, row, col);
    count_launch(h);
    count_launch(h);
  }
  IGACD_LAUNCH_CHECK();
  k_negate_sym<<<gb, bs, 0, s>>>(cinv, N);
  IGACD_LAUNCH_CHECK();
  count_launch(h);
  int hbad = 0;
  IGACD_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  IGACD_CUDA(cudaStreamSynchronize(s));
  cudaFree(row);
  cudaFree(col);
  cudaFree(bad);
  if (hbad) throw Error{IGACD_E_NOTSPD, "coarsest-level matrix is not positive definite"};
}

void launch_coarse_solve(Handle& h, int sy, const double* b, double* x, cudaStream_t s) {
  const System& S = h.sys[sy];
  const int N = (int)S.lv.back().ndof;
  const int bs = 256;
  k_dense_matvec<<<(N * 32 + bs - 1) / bs, bs, 0, s>>>(S.cinv, b, x, N);
  IGACD_LAUNCH_CHECK();
  count_launch(h);
}

}  // namespace igacd

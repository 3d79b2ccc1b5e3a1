// Batched banded SPD line solves along one tensor direction.
//
// Used for (a) the paper's preconditioner T_n^p = I_d (x) T(m_{p-1}) (x) .. (x) T(m_{p-1})
// ("each (T)^{-1} can be solved by means of an LU factorization which
// is optimal for banded matrices") as the smoother of the V-cycle (reading R4'), and (b)
// the exact inverse of the auxiliary scalar operator when b0 is a coordinate direction,
// A_s = (c_m M + c_s S)_l (x) M (x) .. (reading R8).
// A factor F = L L^T (banded Cholesky, half bandwidth W <= 6) is applied along axis `a`
// of an array viewed as [outer][m][inner]: one thread per line, forward then backward
// substitution with a register window of the last W values; the factor lives in shared
// memory.  Lines along the fastest axis are contiguous per thread (L1 absorbs the stride).
#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace igacd {

// Lb[k*(W+1) + (W - j)] = L[k][k-j], j = 0..W (zero where k-j < 0); inv[k] = 1/L[k][k]
template <int W>
__global__ void k_band_solve(double* __restrict__ data, long long outer, int m, long long inner,
                             const double* __restrict__ Lb, const double* __restrict__ inv, int mode, double omega,
                             double* __restrict__ xacc) {
  extern __shared__ double sh[];
  double* sL = sh;                     // [m][W+1]
  double* sI = sh + (size_t)m * (W + 1);  // [m]
  for (int i = threadIdx.x; i < m * (W + 1); i += blockDim.x) sL[i] = Lb[i];
  for (int i = threadIdx.x; i < m; i += blockDim.x) sI[i] = inv[i];
  __syncthreads();
  const long long lines = outer * inner;
  for (long long ln = blockIdx.x * (long long)blockDim.x + threadIdx.x; ln < lines;
       ln += (long long)gridDim.x * blockDim.x) {
    const long long o = ln / inner, i = ln % inner;
    double* base = data + o * (long long)m * inner + i;
    // forward: y_k = (b_k - sum_j L[k][k-j] y_{k-j}) / L[k][k]
    double win[W + 1];
#pragma unroll
    for (int j = 0; j <= W; ++j) win[j] = 0.0;   // win[j] = y_{k-j} after the shift
    for (int k = 0; k < m; ++k) {
#pragma unroll
      for (int j = W; j >= 1; --j) win[j] = win[j - 1];
      double acc = base[(long long)k * inner];
      const double* Lr = sL + (size_t)k * (W + 1);
#pragma unroll
      for (int j = 1; j <= W; ++j) acc = fma(-Lr[W - j], win[j], acc);
      win[0] = acc * sI[k];
      base[(long long)k * inner] = win[0];
    }
    // backward: x_k = (y_k - sum_j L[k+j][k] x_{k+j}) / L[k][k]
#pragma unroll
    for (int j = 0; j <= W; ++j) win[j] = 0.0;   // win[j] = x_{k+j}
    for (int k = m - 1; k >= 0; --k) {
#pragma unroll
      for (int j = W; j >= 1; --j) win[j] = win[j - 1];
      double acc = base[(long long)k * inner];
#pragma unroll
      for (int j = 1; j <= W; ++j)
        if (k + j < m) acc = fma(-sL[(size_t)(k + j) * (W + 1) + W - j], win[j], acc);
      win[0] = acc * sI[k];
      if (mode == 0) {
        base[(long long)k * inner] = win[0];
      } else {   // x += omega * z, written to xacc (same layout as data)
        const long long off = (base - data) + (long long)k * inner;
        xacc[off] += omega * win[0];
      }
    }
  }
}

__device__ __forceinline__ void ls_cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr), "l"(gsrc) : "memory");
}

// Tiled variant: each warp stages 32 lines in shared memory (coalesced loads/stores), and
// every lane runs its substitution out of shared memory, so the sequential recurrence sees
// shared-memory latency instead of DRAM latency.  Requires inner == 1 or inner % 32 == 0.
template <int W, int WARPS, int TW>
__global__ void __launch_bounds__(32 * WARPS) k_band_solve_tiled(double* __restrict__ data, long long outer, int m,
                                                               long long inner, const double* __restrict__ Lb,
                                                               const double* __restrict__ inv, int mode,
                                                               double omega, double* __restrict__ xacc) {
  extern __shared__ double sh[];
  double* sL = sh;                          // [m][W+1]
  double* sI = sL + (size_t)m * (W + 1);    // [m]
  constexpr int TP = TW + 1;                // padded tile row (bank-conflict free for TW = 32)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* tile = sI + m + (size_t)warp * m * TP;   // [m][TP]
  for (int i = threadIdx.x; i < m * (W + 1); i += blockDim.x) sL[i] = Lb[i];
  for (int i = threadIdx.x; i < m; i += blockDim.x) sI[i] = inv[i];
  __syncthreads();
  const long long lines = outer * inner;
  const long long groups = (lines + TW - 1) / TW;
  for (long long g = (long long)blockIdx.x * WARPS + warp; g < groups; g += (long long)gridDim.x * WARPS) {
    const long long l0 = g * TW;
    const int nl = (int)min((long long)TW, lines - l0);
    // ---- load the TW x m tile with asynchronous copies (all loads in flight at once)
    if (inner == 1) {
      const double* src = data + l0 * m;
      for (int e = lane; e < nl * m; e += 32) ls_cp_async8(&tile[(e % m) * TP + e / m], src + e);
    } else {   // lanes = consecutive lines: coalesced except where the group crosses an `outer` step
      const long long l = l0 + lane;
      const double* src = data + (l / inner) * (long long)m * inner + (l % inner);
      if (lane < nl)
        for (int k = 0; k < m; ++k) ls_cp_async8(&tile[k * TP + lane], src + (long long)k * inner);
    }
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncwarp();
    if (lane < nl) {
      double win[W + 1];
#pragma unroll
      for (int j = 0; j <= W; ++j) win[j] = 0.0;
      for (int k = 0; k < m; ++k) {
#pragma unroll
        for (int j = W; j >= 1; --j) win[j] = win[j - 1];
        double acc = tile[k * TP + lane];
        const double* Lr = sL + (size_t)k * (W + 1);
#pragma unroll
        for (int j = 1; j <= W; ++j) acc = fma(-Lr[W - j], win[j], acc);
        win[0] = acc * sI[k];
        tile[k * TP + lane] = win[0];
      }
#pragma unroll
      for (int j = 0; j <= W; ++j) win[j] = 0.0;
      for (int k = m - 1; k >= 0; --k) {
#pragma unroll
        for (int j = W; j >= 1; --j) win[j] = win[j - 1];
        double acc = tile[k * TP + lane];
#pragma unroll
        for (int j = 1; j <= W; ++j)
          if (k + j < m) acc = fma(-sL[(size_t)(k + j) * (W + 1) + W - j], win[j], acc);
        win[0] = acc * sI[k];
        tile[k * TP + lane] = win[0];
      }
    }
    __syncwarp();
    // ---- store (or accumulate omega * result into xacc, reading xacc 8 elements ahead so the
    // read-modify-writes overlap instead of serialising on DRAM latency)
    constexpr int U = 8;
    if (inner == 1) {
      double* dst = (mode == 0 ? data : xacc) + l0 * m;
      const int tot = nl * m;
      for (int e0 = lane; e0 < tot; e0 += 32 * U) {
        double xv[U];
        if (mode != 0) {
#pragma unroll
          for (int u = 0; u < U; ++u) xv[u] = (e0 + 32 * u < tot) ? dst[e0 + 32 * u] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + 32 * u;
          if (e < tot) {
            const double v = tile[(e % m) * TP + e / m];
            dst[e] = mode == 0 ? v : fma(omega, v, xv[u]);
          }
        }
      }
    } else {
      const long long l = l0 + lane;
      double* dst = (mode == 0 ? data : xacc) + (l / inner) * (long long)m * inner + (l % inner);
      if (lane < nl)
        for (int k0 = 0; k0 < m; k0 += U) {
          double xv[U];
          if (mode != 0) {
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = (k0 + u < m) ? dst[(long long)(k0 + u) * inner] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int k = k0 + u;
            if (k < m) {
              const double v = tile[k * TP + lane];
              dst[(long long)k * inner] = mode == 0 ? v : fma(omega, v, xv[u]);
            }
          }
        }
    }
    __syncwarp();
  }
}

// banded Cholesky on the host: F given in band storage [m][2w+1] (F[k][k+o] at k*(2w+1)+o+w)
void band_cholesky(const std::vector<double>& F, int m, int w, std::vector<double>& Lb, std::vector<double>& inv) {
  Lb.assign((size_t)m * (w + 1), 0.0);
  inv.assign(m, 0.0);
  auto L = [&](int i, int j) -> double& { return Lb[(size_t)i * (w + 1) + (w - (i - j))]; };  // j in [i-w, i]
  for (int i = 0; i < m; ++i) {
    for (int j = std::max(0, i - w); j <= i; ++j) {
      double s = F[(size_t)i * (2 * w + 1) + (j - i) + w];
      for (int k = std::max(0, i - w); k < j; ++k)
        if (k >= j - w) s -= L(i, k) * L(j, k);
      if (i == j) {
        if (!(s > 0.0)) throw Error{IGACD_E_NOTSPD, "banded factor is not positive definite"};
        L(i, i) = std::sqrt(s);
        inv[i] = 1.0 / L(i, i);
      } else {
        L(i, j) = s / L(j, j);
      }
    }
  }
}

void BandFactor::upload(const std::vector<double>& Lb_h, const std::vector<double>& inv_h, int m_, int w_) {
  m = m_;
  w = w_;
  IGACD_CUDA(cudaMalloc(&Lb, sizeof(double) * Lb_h.size()));
  IGACD_CUDA(cudaMalloc(&inv, sizeof(double) * inv_h.size()));
  IGACD_CUDA(cudaMemcpy(Lb, Lb_h.data(), sizeof(double) * Lb_h.size(), cudaMemcpyHostToDevice));
  IGACD_CUDA(cudaMemcpy(inv, inv_h.data(), sizeof(double) * inv_h.size(), cudaMemcpyHostToDevice));
}

void BandFactor::release() {
  cudaFree(Lb);
  cudaFree(inv);
  Lb = inv = nullptr;
}

template <int W, int WARPS, int TW>
static bool try_tiled(double* data, long long outer, int m, long long inner, const BandFactor& F, int mode,
                      double omega, double* xacc, cudaStream_t s) {
  const size_t smem_t = sizeof(double) * ((size_t)m * (W + 1) + m + (size_t)WARPS * m * (TW + 1));
  if (smem_t > 200 * 1024) return false;
  static size_t attr_t = 0;
  if (smem_t > 48 * 1024 && attr_t < smem_t) {
    IGACD_CUDA(cudaFuncSetAttribute(k_band_solve_tiled<W, WARPS, TW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)smem_t));
    attr_t = smem_t;
  }
  const long long groups = (outer * inner + TW - 1) / TW;
  long long blocks = (groups + WARPS - 1) / WARPS;
  if (blocks > 148 * 16) blocks = 148 * 16;
  k_band_solve_tiled<W, WARPS, TW><<<(unsigned)blocks, 32 * WARPS, smem_t, s>>>(data, outer, m, inner, F.Lb, F.inv,
                                                                              mode, omega, xacc);
  return true;
}

template <int W>
static void launch_w(double* data, long long outer, int m, long long inner, const BandFactor& F, int mode,
                     double omega, double* xacc, cudaStream_t s) {
  // widest tile that fits: 32 lines per warp (2 warps), else 16 or 8 lines (1 warp)
  if (try_tiled<W, 2, 32>(data, outer, m, inner, F, mode, omega, xacc, s)) return;
  if (try_tiled<W, 1, 32>(data, outer, m, inner, F, mode, omega, xacc, s)) return;
  if (try_tiled<W, 1, 16>(data, outer, m, inner, F, mode, omega, xacc, s)) return;
  if (try_tiled<W, 1, 8>(data, outer, m, inner, F, mode, omega, xacc, s)) return;
  const size_t smem = sizeof(double) * ((size_t)m * (W + 1) + m);
  static int attr_set = 0;
  if (smem > 48 * 1024 && attr_set < (int)smem) {
    IGACD_CUDA(cudaFuncSetAttribute(k_band_solve<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr_set = (int)smem;
  }
  const long long lines = outer * inner;
  const int bs = 128;
  long long blocks = (lines + bs - 1) / bs;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_band_solve<W><<<(unsigned)blocks, bs, smem, s>>>(data, outer, m, inner, F.Lb, F.inv, mode, omega, xacc);
}

// data <- F^{-1} data along axis `axis` of a [nc][m]^dim array; mode 1: xacc += omega * F^{-1} data
// (data is then left holding the forward-substitution intermediate).
void launch_band_solve(Handle& h, int nc, int level, int axis, const BandFactor& F, double* data, int mode,
                       double omega, double* xacc, cudaStream_t s) {
  const long long m = h.lv[level].m;
  long long outer = nc, inner = 1;
  for (int a = 0; a < axis; ++a) outer *= m;
  for (int a = axis + 1; a < h.dim; ++a) inner *= m;
  switch (F.w) {
    case 0: launch_w<0>(data, outer, (int)m, inner, F, mode, omega, xacc, s); break;
    case 1: launch_w<1>(data, outer, (int)m, inner, F, mode, omega, xacc, s); break;
    case 2: launch_w<2>(data, outer, (int)m, inner, F, mode, omega, xacc, s); break;
    case 3: launch_w<3>(data, outer, (int)m, inner, F, mode, omega, xacc, s); break;
    case 4: launch_w<4>(data, outer, (int)m, inner, F, mode, omega, xacc, s); break;
    case 5: launch_w<5>(data, outer, (int)m, inner, F, mode, omega, xacc, s); break;
    case 6: launch_w<6>(data, outer, (int)m, inner, F, mode, omega, xacc, s); break;
    default: throw Error{IGACD_E_ARG, "band width out of range"};
  }
  IGACD_LAUNCH_CHECK();
  count_launch(h);
}

}  // namespace igacd

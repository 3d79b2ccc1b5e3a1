// Batched banded SPD line solves along one tensor direction.
//
// Used for (a) the paper's preconditioner T_n^p = I_d (x) T(m_{p-1}) (x) .. (x) T(m_{p-1})
// ("each (T)^{-1} can be solved by means of an LU factorization which
// is optimal for banded matrices") as the smoother of the V-cycle (reading R4'), and (b)
// the exact inverse of the auxiliary scalar operator when b0 is a coordinate direction,
// A_s = (c_m M + c_s S)_l (x) M (x) .. (reading R8).
// A factor F = L L^T (banded Cholesky, half bandwidth W <= 6) is applied along axis `a`
// of an array viewed as [outer][m][inner].  Product kernels: one warp stages a tile of lines
// in shared memory (lanes = lines) and every lane runs the forward and backward substitution
// of its line in column order (band_sweep_s: one dependent DFMA per step; the factor tables
// stay in global memory, L1-resident, and only the first / last rows of a sweep read them):
//   k_band_solve_tma    3D levels with even m: 32-line tiles by one bulk tensor load and one
//                       tensor store / reduce-add each;
//   k_band_solve_tiled  every other case (cp.async staging; 4/8/32-line tiles);
//   k_band_solve_slab   3D: directions 1 and 2 of a slab in one pass when the slab fits twice;
//   k_band_solve        the in-place one-thread-per-line fallback.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>

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

// One substitution sweep over a line held in shared memory (element k at tile[k*TP + lane]),
// in right-looking (column) order: when v_t is final it is scattered into the W pending rows,
//   acc[q] (row t+1+q) -= G[t][q] v_t,  q = 0..W-1,
// where forward G[t][q] = i_r L[r][t] (r = t+1+q) and backward G[t][q] = i_r L[k][r]
// (k = m-1-t, r = k-1-q), and row t+W enters the ring as i_r * tile[r].  The loop-carried
// dependency is one DFMA per step (acc[1] - G v_t -> next v).
// The rows of the Cholesky factor of T(m_{p-1}) become bitwise constant from row Kc on
// (BandFactor::kc): on the steps whose operands all come from those rows, G[t][q] and i_r are
// the same numbers for every t, so they are held in registers (no shared-memory operand
// loads) and the entering rows are read 8 steps ahead; the first / last rows use the tables.
template <int W, bool FWD, bool SCALE = false>
__device__ __forceinline__ void band_sweep_s(double* tile, const int TP, const double* __restrict__ G,
                                             const double* __restrict__ gI, int m, int kc, double sc = 1.0) {
  auto row = [&](int t) { return FWD ? t : m - 1 - t; };
  auto put = [&](int r, double v) { tile[r * TP] = SCALE ? sc * v : v; };   // final values are never re-read
  auto sIv = [&](int r) { return (r >= 0 && r < m) ? __ldg(gI + r) : 0.0; };   // 1/L[r][r], 0 outside
  if constexpr (W == 0) {
    for (int t = 0; t < m; ++t) tile[t * TP] *= (SCALE ? sc : 1.0) * __ldg(gI + t);
  } else {
    double acc[W];
#pragma unroll
    for (int q = 0; q < W; ++q) acc[q] = tile[row(q) * TP] * sIv(row(q));
    // steps with table operands: the weights of step t+1 are requested while step t runs
    auto generic = [&](int t0, int t1) {
      if (t0 >= t1) return;
      double gq[W], gin = sIv(row(t0 + W));
#pragma unroll
      for (int q = 0; q < W; ++q) gq[q] = __ldg(G + t0 * (W + 1) + q);
      for (int t = t0; t < t1; ++t) {
        double gn[W], ginn = 0.0;
        const int tn = min(t + 1, t1 - 1);
#pragma unroll
        for (int q = 0; q < W; ++q) gn[q] = __ldg(G + tn * (W + 1) + q);
        ginn = sIv(row(tn + W));
        const double v = acc[0];
        const double enter = tile[row(t + W) * TP] * gin;
#pragma unroll
        for (int q = 0; q + 1 < W; ++q) acc[q] = fma(-gq[q], v, acc[q + 1]);
        acc[W - 1] = fma(-gq[W - 1], v, enter);
        put(row(t), v);
#pragma unroll
        for (int q = 0; q < W; ++q) gq[q] = gn[q];
        gin = ginn;
      }
    };
    int ta = FWD ? kc : 0;
    int tb = FWD ? m - W : m - W - kc;
    if (ta >= tb) {
      generic(0, m);
      return;
    }
    generic(0, ta);
    double gc[W];
#pragma unroll
    for (int q = 0; q < W; ++q) gc[q] = __ldg(G + ta * (W + 1) + q);
    const double ic = sIv(row(ta + W));
    constexpr int U = 8;
    int t = ta;
    // the entering rows of block b+1 are read before block b stores its results (rows t+W+U.. are
    // never rows a store of this sweep has touched, but the compiler cannot know)
    double e[U];
    if (t + U <= tb) {
#pragma unroll
      for (int u = 0; u < U; ++u) e[u] = tile[row(t + W + u) * TP];
    }
    for (; t + U <= tb; t += U) {
      double en[U];
      const bool more = t + 2 * U <= tb;
#pragma unroll
      for (int u = 0; u < U; ++u) en[u] = more ? tile[row(t + U + W + u) * TP] : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double v = acc[0];
#pragma unroll
        for (int q = 0; q + 1 < W; ++q) acc[q] = fma(-gc[q], v, acc[q + 1]);
        acc[W - 1] = fma(-gc[W - 1], v, e[u] * ic);
        put(row(t + u), v);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) e[u] = en[u];
    }
    for (; t < tb; ++t) {
      const double v = acc[0];
      const double enter = tile[row(t + W) * TP] * ic;
#pragma unroll
      for (int q = 0; q + 1 < W; ++q) acc[q] = fma(-gc[q], v, acc[q + 1]);
      acc[W - 1] = fma(-gc[W - 1], v, enter);
      put(row(t), v);
    }
    generic(tb, m);
  }
}

template <int W, int TP, bool FWD>
__device__ __forceinline__ void band_sweep(double* tile, const double* __restrict__ G, const double* __restrict__ gI,
                                           int m, int kc) {
  band_sweep_s<W, FWD>(tile, TP, G, gI, m, kc);
}

// Tiled variant: each warp stages TW lines in shared memory (coalesced loads/stores), and
// every lane runs its substitution out of shared memory, so the sequential recurrence sees
// shared-memory latency instead of DRAM latency.  With NBUF = 2 the warp streams: the
// asynchronous loads of its next tile are in flight while the current tile is solved and
// stored, so DRAM traffic overlaps the recurrences.  Requires inner == 1 or inner % 32 == 0
// (lanes of a tile are consecutive lines).
template <int W, int WARPS, int TW, int NBUF>
__global__ void __launch_bounds__(32 * WARPS) k_band_solve_tiled(double* __restrict__ data, long long outer, int m,
                                                               long long inner, const double* __restrict__ fac,
                                                               int kc, int mode, double omega,
                                                               double* __restrict__ xacc, const double* src_arr) {
  extern __shared__ __align__(16) double sh[];
  // factor tables stay in global memory (L1-resident; only the first / last rows of a sweep
  // read them, BandFactor::kc), so shared memory holds line tiles only
  const double* __restrict__ gF = fac;                          // [m][W+1] forward column table
  const double* __restrict__ gB = fac + (size_t)m * (W + 1);    // [m][W+1] backward column table
  const double* __restrict__ gI = gB + (size_t)m * (W + 1);     // [m] 1/L[k][k]
  constexpr int TP = TW + 1;                // padded tile row (bank-conflict free for TW = 32)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int MP = m + 2 * W;                 // tile rows incl. W zero rows on each side
  double* tiles = sh + (size_t)warp * NBUF * MP * TP + W * TP;   // buffer b: tiles + b*MP*TP
  for (int b = 0; b < NBUF; ++b) {
    double* t = tiles + (size_t)b * MP * TP;
    for (int i = lane; i < W * TP; i += 32) t[-W * TP + i] = t[m * TP + i] = 0.0;
  }
  __syncwarp();
  const long long lines = outer * inner;
  const long long groups = (lines + TW - 1) / TW;
  const long long stride = (long long)gridDim.x * WARPS;

  auto issue_load = [&](long long g, double* tile) {
    const long long l0 = g * TW;
    const int nl = (int)min((long long)TW, lines - l0);
    if (inner == 1) {
      const double* src = src_arr + l0 * m;
      int k = lane % m, ln = lane / m;   // e = ln * m + k, advanced by 32 without divisions
      for (int e = lane; e < nl * m; e += 32) {
        ls_cp_async8(&tile[k * TP + ln], src + e);
        k += 32;
        while (k >= m) { k -= m; ++ln; }
      }
    } else {   // lanes = consecutive lines: coalesced except where the group crosses an `outer` step
      const long long l = l0 + lane;
      const double* src = src_arr + (l / inner) * (long long)m * inner + (l % inner);
      double* tp = tile + lane;
      if (lane < nl)
#pragma unroll 4
        for (int k = 0; k < m; ++k) {
          ls_cp_async8(tp, src);
          tp += TP;
          src += inner;
        }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };

  // store the solved tile (mode 0) or accumulate omega * result into xacc (mode 1).
  // Mode 1 on contiguous lines (the last axis): x_acc += omega * result, with x_acc read in
  // batches of UA per lane; batch 0 is requested before the sweeps (its latency hides behind
  // them) and batch b+1 is in flight while batch b is stored.
  constexpr int UA = 24;
  double xa0[UA], xa1[UA];
  auto acc_load = [&](const double* src, int e0, int tot, double (&xv)[UA]) {
#pragma unroll
    for (int u = 0; u < UA; ++u) xv[u] = (e0 + 32 * u < tot) ? src[e0 + 32 * u] : 0.0;
  };
  auto store = [&](long long g, const double* tile) {
    const long long l0 = g * TW;
    const int nl = (int)min((long long)TW, lines - l0);
    constexpr int U = 16;
    if (inner == 1 && mode == 2) {
      double* dst = xacc + l0 * m;
      const int tot = nl * m;
      int k = lane % m, ln = lane / m;
      for (int e0 = lane; e0 < tot; e0 += 32 * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + 32 * u;
          if (e < tot) {
            dst[e] = omega * tile[k * TP + ln];
            k += 32;
            while (k >= m) { k -= m; ++ln; }
          }
        }
      }
    } else if (inner == 1 && mode != 0) {
      double* dst = xacc + l0 * m;
      const int tot = nl * m;
      int k = lane % m, ln = lane / m;
      auto put = [&](int e0, const double (&xv)[UA]) {
#pragma unroll
        for (int u = 0; u < UA; ++u) {
          const int e = e0 + 32 * u;
          if (e < tot) {
            dst[e] = fma(omega, tile[k * TP + ln], xv[u]);
            k += 32;
            while (k >= m) { k -= m; ++ln; }
          }
        }
      };
      for (int e0 = lane; e0 < tot; e0 += 64 * UA) {   // xa0 holds batch e0 (loaded earlier)
        if (e0 + 32 * UA < tot) acc_load(dst, e0 + 32 * UA, tot, xa1);
        put(e0, xa0);
        if (e0 + 32 * UA >= tot) break;
        if (e0 + 64 * UA < tot) acc_load(dst, e0 + 64 * UA, tot, xa0);
        put(e0 + 32 * UA, xa1);
      }
    } else if (inner == 1) {
      double* dst = data + l0 * m;
      const int tot = nl * m;
      int k = lane % m, ln = lane / m;
      for (int e0 = lane; e0 < tot; e0 += 32 * U) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + 32 * u;
          if (e < tot) {
            dst[e] = tile[k * TP + ln];
            k += 32;
            while (k >= m) { k -= m; ++ln; }
          }
        }
      }
    } else {
      const long long l = l0 + lane;
      double* dst = (mode == 0 ? data : xacc) + (l / inner) * (long long)m * inner + (l % inner);
      const double* tp = tile + lane;
      if (lane < nl) {
        if (mode == 0 || mode == 2) {
          const double f = mode == 0 ? 1.0 : omega;
#pragma unroll 4
          for (int k = 0; k < m; ++k) {
            *dst = f * *tp;
            tp += TP;
            dst += inner;
          }
        } else {
          for (int k0 = 0; k0 < m; k0 += U) {
            double xv[U];
            const int nu = min(U, m - k0);
#pragma unroll
            for (int u = 0; u < U; ++u) xv[u] = u < nu ? dst[(long long)u * inner] : 0.0;
#pragma unroll
            for (int u = 0; u < U; ++u)
              if (u < nu) dst[(long long)u * inner] = fma(omega, tp[u * TP], xv[u]);
            tp += U * TP;
            dst += (long long)U * inner;
          }
        }
      }
    }
  };

  long long g = (long long)blockIdx.x * WARPS + warp;
  int cur = 0;
  if (NBUF == 2 && g < groups) issue_load(g, tiles);
  for (; g < groups; g += stride) {
    double* tile = tiles + (size_t)cur * MP * TP;
    if (NBUF == 2) {
      const long long gn = g + stride;
      if (gn < groups) {
        issue_load(gn, tiles + (size_t)(cur ^ 1) * MP * TP);
        asm volatile("cp.async.wait_group 1;\n" ::: "memory");   // the current tile has landed
      } else {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
      }
    } else {
      issue_load(g, tile);
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncwarp();
    const int nl = (int)min((long long)TW, lines - g * TW);
    if (inner == 1 && mode == 1) acc_load(xacc + g * TW * m, lane, nl * m, xa0);   // batch 0, ahead
    if (lane < nl) {
      // forward  y_k = i_k b_k - sum_j (i_k L[k][k-j]) y_{k-j}
      // backward x_k = i_k y_k - sum_j (i_k L[k+j][k]) x_{k+j}
      band_sweep<W, TP, true>(tile + lane, gF, gI, m, kc);
      band_sweep<W, TP, false>(tile + lane, gB, gI, m, kc);
    }
    __syncwarp();
    store(g, tile);
    __syncwarp();
    if (NBUF == 2) cur ^= 1;
  }
}

// ---------------------------------------------------------------------------------------------
// TMA variant of the tiled line solve (3D levels with even m <= 250): one warp per CTA, one
// 32-line tile per step of a persistent loop.  The tile arrives by ONE bulk tensor copy
// (cp.async.bulk.tensor, completion on an mbarrier; the W zero rows the sweeps read before and
// after a line are the out-of-bounds rows of the box, zero-filled by the tensor map), the two
// sweeps run out of shared memory, and the result leaves by one tensor store (modes 0, 2) or
// tensor reduce-add into x (mode 1: x += omega T^{-1} r is done by the L2, the SM never reads x).  The cp.async version above spent two thirds of a tile's time issuing 8-byte copies and
// stores (ncu: profiles/r02_linesolve_config4.md); here the warp only waits for them.
//   CONTIG = false: lines `inner` apart (directions 0, 1): box {32 lines, m + 2W rows}, tile [k][lane];
//   CONTIG = true:  lines contiguous (last direction):     box {m + 2WP, 32 lines},    tile [lane][k]
//                   (WP = W rounded up to even: boxes start on 16-byte boundaries).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ unsigned ls_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int W, bool CONTIG>
__global__ void __launch_bounds__(32) k_band_solve_tma(const __grid_constant__ CUtensorMap tsrc,
                                                       const __grid_constant__ CUtensorMap tdst,
                                                       double* __restrict__ data, int m,
                                                       long long inner, int tiles_per_outer, long long ntiles,
                                                       long long lines, const double* __restrict__ fac, int kc,
                                                       int mode, double omega, double* __restrict__ xacc) {
  extern __shared__ __align__(128) double sht[];
  double* sh = sht;
  constexpr int WP = (W + 1) / 2 * 2;
  const int lane = threadIdx.x;
  const int LP = m + 2 * WP;                                    // CONTIG: pitch of a line
  const int nelem = CONTIG ? 32 * LP : 32 * (m + 2 * W);
  uint64_t* mbar = reinterpret_cast<uint64_t*>(sh + nelem);
  const double* __restrict__ gF = fac;
  const double* __restrict__ gB = fac + (size_t)m * (W + 1);
  const double* __restrict__ gI = gB + (size_t)m * (W + 1);
  double* line = CONTIG ? sh + (size_t)lane * LP + WP : sh + W * 32 + lane;   // element k = 0 of my line
  const int TP = CONTIG ? 1 : 32;
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(ls_u32(mbar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncwarp();
  unsigned phase = 0;
  for (long long g = blockIdx.x; g < ntiles; g += gridDim.x) {
    const long long o = CONTIG ? 0 : g / tiles_per_outer;
    const long long i0 = CONTIG ? g * 32 : (g - o * tiles_per_outer) * 32;   // first line (CONTIG) / inner index
    const int nl = (int)min(32LL, (CONTIG ? lines : inner) - i0);
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(ls_u32(mbar)),
                   "r"((unsigned)(nelem * 8))
                   : "memory");
      if (CONTIG)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::
                "r"(ls_u32(sh)), "l"((unsigned long long)&tsrc), "r"(-WP), "r"((int)i0), "r"(ls_u32(mbar))
            : "memory");
      else
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
            "[%5];\n" ::"r"(ls_u32(sh)),
            "l"((unsigned long long)&tsrc), "r"((int)i0), "r"(-W), "r"((int)o), "r"(ls_u32(mbar))
            : "memory");
    }
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(ls_u32(mbar)),
        "r"(phase)
        : "memory");
    phase ^= 1u;
    if (lane < nl) {
      band_sweep_s<W, true>(line, TP, gF, gI, m, kc);
      if (mode == 0) band_sweep_s<W, false>(line, TP, gB, gI, m, kc);
      else band_sweep_s<W, false, true>(line, TP, gB, gI, m, kc, omega);   // omega T^{-1} r
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // my generic writes before the async reads
    __syncwarp();
    // the tile leaves by ONE tensor store (modes 0, 2) or tensor reduce-add (mode 1) of the
    // unpadded box (measured, tools/microbench/tma_store.cu: a store whose box starts at a negative
    // row faults with an illegal instruction, one hanging over the end of a row is clipped, and
    // the fp64 reduce-add works); contiguous lines leave by one bulk copy / reduce-add each
    if (CONTIG) {
      if (lane < nl) {
        double* dst = (mode == 0 ? data : xacc) + (i0 + lane) * (long long)m;
        if (mode != 1)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(ls_u32(line)),
                       "r"((unsigned)(m * 8))
                       : "memory");
        else
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;\n" ::"l"(dst),
                       "r"(ls_u32(line)), "r"((unsigned)(m * 8))
                       : "memory");
      }
    } else if (lane == 0) {
      if (mode != 1)
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::
                         "l"((unsigned long long)&tdst), "r"((int)i0), "r"(0), "r"((int)o), "r"(ls_u32(sh + W * 32))
                     : "memory");
      else
        asm volatile(
            "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];\n" ::
                "l"((unsigned long long)&tdst), "r"((int)i0), "r"(0), "r"((int)o), "r"(ls_u32(sh + W * 32))
            : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");   // the tile has been read out
    __syncwarp();
  }
  asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
}

typedef CUresult (*LsEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static LsEncodeFn ls_encode_fn() {
  static std::once_flag once;
  static LsEncodeFn fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<LsEncodeFn>(p);
  });
  if (!fn) throw Error{IGACD_E_CUDA, "cuTensorMapEncodeTiled unavailable"};
  return fn;
}

// [outer][m][inner] fp64 viewed for the line tiles (see k_band_solve_tma)
static CUtensorMap line_map(const double* base, long long outer, int m, long long inner, int W, bool contig,
                            bool padded = true) {
  CUtensorMap map;
  CUresult r;
  const cuuint32_t es[3] = {1u, 1u, 1u};
  if (contig) {
    const int WP = (W + 1) / 2 * 2;
    const cuuint64_t dims[2] = {(cuuint64_t)m, (cuuint64_t)outer};
    const cuuint64_t strides[1] = {(cuuint64_t)m * 8};
    const cuuint32_t box[2] = {(cuuint32_t)(m + 2 * WP), 32u};
    r = ls_encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    const cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)m, (cuuint64_t)outer};
    const cuuint64_t strides[2] = {(cuuint64_t)inner * 8, (cuuint64_t)inner * m * 8};
    const cuuint32_t box[3] = {32u, (cuuint32_t)(padded ? m + 2 * W : m), 1u};
    r = ls_encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) throw Error{IGACD_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  return map;
}

// IGACD_BAND_TMA: bit 0 strided lines, bit 1 contiguous lines, bit 2 mode 1 (reduce-add); default 7;
// 0 = the cp.async tiles everywhere (comparison)
static int band_tma_mask() {
  static const int v = [] {
    const char* e = getenv("IGACD_BAND_TMA");
    return (e && *e) ? atoi(e) : 7;
  }();
  return v;
}

template <int W>
static bool try_tma(double* data, long long outer, int m, long long inner, const BandFactor& F, int mode, double omega,
                    double* xacc, const double* src, cudaStream_t s, int slot_share) {
  const bool contig = inner == 1;
  const int WP = (W + 1) / 2 * 2;
  const int rows = m + 2 * (contig ? WP : W);
  const double* dst = mode == 0 ? data : xacc;
  const int mask = band_tma_mask();
  if (!(mask & (contig ? 2 : 1)) || (mode == 1 && !(mask & 4))) return false;
  if (m % 2 || rows > 256 || outer * inner < 64LL * num_sms()) return false;
  if (((uintptr_t)src & 15) || ((uintptr_t)dst & 15)) return false;
  const size_t smem = sizeof(double) * 32 * (size_t)rows + 16;
  const long long lines = outer * inner;
  const int tpo = contig ? 0 : (int)((inner + 31) / 32);
  const long long ntiles = contig ? (lines + 31) / 32 : outer * tpo;
  const void* kern = contig ? (const void*)k_band_solve_tma<W, true> : (const void*)k_band_solve_tma<W, false>;
  ensure_smem_attr(kern, smem);
  const int occ = max_active_blocks(kern, 32, smem);
  const unsigned blocks =
      (unsigned)std::min<long long>(ntiles, std::max<long long>(1, (long long)occ * num_sms() * slot_share / 100));
  const CUtensorMap ts = line_map(src, contig ? lines : outer, m, inner, W, contig);
  const CUtensorMap td = contig ? ts : line_map(dst, outer, m, inner, W, false, false);   // output box: rows 0..m-1
  if (contig)
    k_band_solve_tma<W, true><<<blocks, 32, smem, s>>>(ts, td, data, m, inner, tpo, ntiles, lines, F.fac, F.kc, mode, omega,
                                                       xacc);
  else
    k_band_solve_tma<W, false><<<blocks, 32, smem, s>>>(ts, td, data, m, inner, tpo, ntiles, lines, F.fac, F.kc, mode, omega,
                                                        xacc);
  return true;
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
  // column-order tables for the tiled kernel: [Gf | Gb | I], rows of stride w+1 (see band_sweep)
  //   Gf[t][q] = i_r L[r][t], r = t+1+q;   Gb[t][q] = i_r L[k][r], k = m-1-t, r = k-1-q
  std::vector<double> f((size_t)(2 * (w + 1) + 1) * m, 0.0);
  double* Gf = f.data();
  double* Gb = Gf + (size_t)m * (w + 1);
  double* Ih = Gb + (size_t)m * (w + 1);
  auto Lh = [&](int i, int j) { return Lb_h[(size_t)i * (w + 1) + (w - (i - j))]; };   // j in [i-w, i]
  for (int t = 0; t < m; ++t) {
    Ih[t] = inv_h[t];
    for (int q = 0; q < w; ++q) {
      const int r = t + 1 + q;
      if (r < m) Gf[(size_t)t * (w + 1) + q] = inv_h[r] * Lh(r, t);
      const int k = m - 1 - t, rb = k - 1 - q;
      if (rb >= 0) Gb[(size_t)t * (w + 1) + q] = inv_h[rb] * Lh(k, rb);
    }
  }
  // first row from which every row of L (and 1/L[k][k]) equals the last row bit for bit
  kc = m;
  for (int k = m - 1; k >= 0; --k) {
    bool same = inv_h[k] == inv_h[m - 1];
    for (int j = 0; j <= w && same; ++j) same = Lb_h[(size_t)k * (w + 1) + j] == Lb_h[(size_t)(m - 1) * (w + 1) + j];
    if (!same) break;
    kc = k;
  }
  IGACD_CUDA(cudaMalloc(&fac, sizeof(double) * f.size()));
  IGACD_CUDA(cudaMemcpy(fac, f.data(), sizeof(double) * f.size(), cudaMemcpyHostToDevice));
}

void BandFactor::release() {
  cudaFree(Lb);
  cudaFree(inv);
  cudaFree(fac);
  Lb = inv = fac = nullptr;
}

template <int W, int WARPS, int TW, int NBUF>
static bool try_tiled(double* data, long long outer, int m, long long inner, const BandFactor& F, int mode,
                      double omega, double* xacc, const double* src, cudaStream_t s) {
  const size_t smem_t = sizeof(double) * ((size_t)WARPS * NBUF * (m + 2 * W) * (TW + 1));
  if (smem_t > 200 * 1024) return false;
  const void* kern = (const void*)k_band_solve_tiled<W, WARPS, TW, NBUF>;
  ensure_smem_attr(kern, smem_t);
  const long long groups = (outer * inner + TW - 1) / TW;
  long long blocks = (groups + WARPS - 1) / WARPS;
  // persistent grid: the factor is staged once per resident block, not once per tile
  const int occ = max_active_blocks(kern, 32 * WARPS, smem_t);
  blocks = std::min<long long>(blocks, (long long)occ * num_sms());
  k_band_solve_tiled<W, WARPS, TW, NBUF><<<(unsigned)blocks, 32 * WARPS, smem_t, s>>>(data, outer, m, inner, F.fac,
                                                                                    F.kc, mode, omega, xacc, src);
  return true;
}

// IGACD_BAND_NBUF=2 selects the double-buffered line-solve pipeline (2 warps per SM); in round 1
// it measured no faster than single-buffered tiles at 4 warps per SM (config 4: 42 vs 40 us).
static int band_nbuf() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_BAND_NBUF");
    v = (e && e[0] == '2') ? 2 : 1;
  }
  return v;
}

static int band_warps() {   // IGACD_BAND_WARPS: warps per CTA of the tiled line solve (1 default, 2)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_BAND_WARPS");
    v = (e && e[0] == '2') ? 2 : 1;
  }
  return v;
}

template <int W>
static void launch_w(double* data, long long outer, int m, long long inner, const BandFactor& F, int mode,
                     double omega, double* xacc, const double* src, cudaStream_t s, int slot_share) {
  // double-buffered 32-line tiles (2 warps) when they fit, else the widest single-buffered tile
  if (band_nbuf() == 2 && try_tiled<W, 2, 32, 2>(data, outer, m, inner, F, mode, omega, xacc, src, s)) return;
  // few long lines (2D: 2m per axis): 8-line tiles, so that more SMs run a recurrence
  // (each tile's sweep is a serial chain of 2m steps whatever its width)
  if (outer * inner < 8LL * num_sms() && try_tiled<W, 1, 4, 1>(data, outer, m, inner, F, mode, omega, xacc, src, s))
    return;
  if (outer * inner < 64LL * num_sms() && try_tiled<W, 1, 8, 1>(data, outer, m, inner, F, mode, omega, xacc, src, s))
    return;
  // many short lines (3D): TMA-staged 32-line tiles
  if (try_tma<W>(data, outer, m, inner, F, mode, omega, xacc, src, s, slot_share)) return;
  // one warp per CTA packs 5 tiles per SM for m = 162 (2 warps per CTA: 4)
  if (band_warps() == 1 && try_tiled<W, 1, 32, 1>(data, outer, m, inner, F, mode, omega, xacc, src, s)) return;
  if (try_tiled<W, 2, 32, 1>(data, outer, m, inner, F, mode, omega, xacc, src, s)) return;
  if (try_tiled<W, 1, 32, 1>(data, outer, m, inner, F, mode, omega, xacc, src, s)) return;
  if (try_tiled<W, 1, 16, 1>(data, outer, m, inner, F, mode, omega, xacc, src, s)) return;
  if (try_tiled<W, 1, 8, 1>(data, outer, m, inner, F, mode, omega, xacc, src, s)) return;
  const size_t smem = sizeof(double) * ((size_t)m * (W + 1) + m);
  ensure_smem_attr((const void*)k_band_solve<W>, smem);
  const long long lines = outer * inner;
  const int bs = 128;
  long long blocks = (lines + bs - 1) / bs;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  // the in-place fallback: stage src into data, and mode 2 (assign) as accumulate into zeros
  if (src != data) IGACD_CUDA(cudaMemcpyAsync(data, src, sizeof(double) * lines * m, cudaMemcpyDeviceToDevice, s));
  if (mode == 2) IGACD_CUDA(cudaMemsetAsync(xacc, 0, sizeof(double) * lines * m, s));
  k_band_solve<W><<<(unsigned)blocks, bs, smem, s>>>(data, outer, m, inner, F.Lb, F.inv, mode == 0 ? 0 : 1, omega,
                                                     xacc);
}


// 3D, both in-slab axes in one pass: one CTA holds one [m][m] slab (directions 1, 2) of one
// component in shared memory (row pitch m|1 odd: conflict-free row and column walks, W zero
// rows before and after), solves every row (direction 2), then every column (direction 1),
// one thread per line, and stores with the mode epilogue.  Versus two tiled passes: one
// DRAM round trip instead of two.  The slab of (component c, index i0) is contiguous.
template <int W>
__global__ void __launch_bounds__(256) k_band_solve_slab(double* __restrict__ data, int m,
                                                         const double* __restrict__ fac, int kc, int mode,
                                                         double omega, double* __restrict__ xacc,
                                                         const double* src_arr) {
  extern __shared__ __align__(16) double sh[];
  const int P = m | 1;
  double* tile = sh + (size_t)W * P;
  const double* __restrict__ gF = fac;
  const double* __restrict__ gB = fac + (size_t)m * (W + 1);
  const double* __restrict__ gI = gB + (size_t)m * (W + 1);
  const size_t base = (size_t)blockIdx.x * m * m;
  const int tid = threadIdx.x, nt = blockDim.x;
  for (int i = tid; i < W * P; i += nt) tile[-W * P + i] = tile[m * P + i] = 0.0;
  if (P != m)
    for (int i = tid; i < m; i += nt) tile[i * P + m] = 0.0;
  const double* src = src_arr + base;
  for (int e = tid; e < m * m; e += nt) ls_cp_async8(&tile[(e / m) * P + e % m], src + e);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  for (int i = tid; i < m; i += nt) {   // direction 2: row i
    band_sweep_s<W, true>(tile + (size_t)i * P, 1, gF, gI, m, kc);
    band_sweep_s<W, false>(tile + (size_t)i * P, 1, gB, gI, m, kc);
  }
  __syncthreads();
  for (int j = tid; j < m; j += nt) {   // direction 1: column j
    band_sweep_s<W, true>(tile + j, P, gF, gI, m, kc);
    band_sweep_s<W, false>(tile + j, P, gB, gI, m, kc);
  }
  __syncthreads();
  constexpr int U = 4;   // mode 1: the x_acc reads of U elements are issued before their stores
  for (int e0 = tid; e0 < m * m; e0 += U * nt) {
    double xa[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * nt;
      xa[u] = (mode == 1 && e < m * m) ? xacc[base + e] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * nt;
      if (e >= m * m) break;
      const double v = tile[(e / m) * P + e % m];
      if (mode == 0) data[base + e] = v;
      else if (mode == 2) xacc[base + e] = omega * v;
      else xacc[base + e] = fma(omega, v, xa[u]);
    }
  }
}

static size_t slab_smem(int m, int w) { return sizeof(double) * (size_t)(m + 2 * w) * (m | 1); }

template <int W>
static void launch_slab_w(double* data, int slabs, int m, const BandFactor& F, int mode, double omega, double* xacc,
                          const double* src, cudaStream_t s) {
  const size_t smem = slab_smem(m, W);
  ensure_smem_attr((const void*)k_band_solve_slab<W>, smem);
  const int nt = std::min(256, (m + 31) / 32 * 32);
  k_band_solve_slab<W><<<slabs, nt, smem, s>>>(data, m, F.fac, F.kc, mode, omega, xacc, src);
}

// data <- F^{-1} data along axis `axis` of a [nc][m]^dim array; mode 1: xacc += omega * F^{-1} data
// (data is then left holding the forward-substitution intermediate).
void launch_band_solve(Handle& h, int nc, int level, int axis, const BandFactor& F, double* data, int mode,
                       double omega, double* xacc, cudaStream_t s, const double* src) {
  const long long m = h.lv[level].m;
  if (!src) src = data;
  long long outer = nc, inner = 1;
  for (int a = 0; a < axis; ++a) outer *= m;
  for (int a = axis + 1; a < h.dim; ++a) inner *= m;
  switch (F.w) {
    case 0: launch_w<0>(data, outer, (int)m, inner, F, mode, omega, xacc, src, s, h.slot_share); break;
    case 1: launch_w<1>(data, outer, (int)m, inner, F, mode, omega, xacc, src, s, h.slot_share); break;
    case 2: launch_w<2>(data, outer, (int)m, inner, F, mode, omega, xacc, src, s, h.slot_share); break;
    case 3: launch_w<3>(data, outer, (int)m, inner, F, mode, omega, xacc, src, s, h.slot_share); break;
    case 4: launch_w<4>(data, outer, (int)m, inner, F, mode, omega, xacc, src, s, h.slot_share); break;
    case 5: launch_w<5>(data, outer, (int)m, inner, F, mode, omega, xacc, src, s, h.slot_share); break;
    case 6: launch_w<6>(data, outer, (int)m, inner, F, mode, omega, xacc, src, s, h.slot_share); break;
    default: throw Error{IGACD_E_ARG, "band width out of range"};
  }
  IGACD_LAUNCH_CHECK();
  count_launch(h);
}

}  // namespace igacd

namespace igacd {

// two CTAs per SM at least: a lone 200+ KB CTA serialises load, sweeps and store (config 4,
// m = 162: 23 % faster alone, slower inside the concurrent preconditioner)
bool band_slab_fits(int m, int w) { return slab_smem(m, w) <= 113 * 1024 && m >= 2; }

// 3D: data <- (F (x) F)^{-1} src over directions 1 and 2 of every slab of a [nc][m]^3 array
// (modes as launch_band_solve)
void launch_band_solve_slab(Handle& h, int nc, int level, const BandFactor& F, double* data, int mode, double omega,
                            double* xacc, cudaStream_t s, const double* src) {
  const int m = h.lv[level].m;
  if (!src) src = data;
  const int slabs = nc * m;
  switch (F.w) {
    case 0: launch_slab_w<0>(data, slabs, m, F, mode, omega, xacc, src, s); break;
    case 1: launch_slab_w<1>(data, slabs, m, F, mode, omega, xacc, src, s); break;
    case 2: launch_slab_w<2>(data, slabs, m, F, mode, omega, xacc, src, s); break;
    case 3: launch_slab_w<3>(data, slabs, m, F, mode, omega, xacc, src, s); break;
    case 4: launch_slab_w<4>(data, slabs, m, F, mode, omega, xacc, src, s); break;
    case 5: launch_slab_w<5>(data, slabs, m, F, mode, omega, xacc, src, s); break;
    case 6: launch_slab_w<6>(data, slabs, m, F, mode, omega, xacc, src, s); break;
    default: throw Error{IGACD_E_ARG, "band width out of range"};
  }
  IGACD_LAUNCH_CHECK();
  count_launch(h);
}

}  // namespace igacd

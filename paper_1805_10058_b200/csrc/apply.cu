// R2: matrix-free operator y = A x by sum factorisation, fused epilogues (R4 smoother,
// residual, D^-1 A, dot products).
//
// The Galerkin matrix is sum_P C_P (x) F_P with 1D factors M, A, S in every direction
// (eq:matr_Amu PAPER.md:483-492, eq:matr_Amu3D PAPER.md:515-543; the L_A form of reading
// R1 has the same Kronecker patterns, see internal.cuh Coef).  Each kernel streams the
// slowest direction ("2.5D marching"): for every slab s it contracts the in-slab
// directions from shared memory, forms the per-point combinations z_{i,F0}(s), and
// scatters F0[t][s] z(s) into a register ring of 2p+1 output slabs; slab t = s-p is then
// final and leaves through the epilogue.  Interior rows of every 1D factor are Toeplitz
// (PAPER.md:347-354): in-slab contractions use 2p+1 register weights with symmetric
// pairing (one add feeds M and S, one subtract feeds A); threads whose row lies in the
// boundary zone redo their contraction with the row's own band.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "internal.cuh"

namespace igacd {

// 8-byte asynchronous global->shared copy (LDGSTS); src_bytes = 0 zero-fills the slot.
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc, bool valid) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int nbytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// ---- TMA (cp.async.bulk.tensor) + mbarrier helpers ------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// ---------------------------------------------------------------------------------------
// Marching-direction weights: column s of each 1D factor, F[t][s] for t = s-p..s+p,
// zero outside the CTA's output chunk [c0, c1).  Written one slab ahead into shared memory.
// ---------------------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void load_col_weights(const OpParams& op, int s, int c0, int c1, double* w) {
  constexpr int R = 2 * P + 1;
  const int tid = threadIdx.x;
  if (tid < 3 * R) {
    const int f = tid / R, o = tid % R - P;
    const int t = s + o;
    double v = 0.0;
    if (t >= c0 && t < c1) {
      const double* band = f == 0 ? op.bM : (f == 1 ? op.bS : op.bA);
      v = __ldg(band + (size_t)t * R + P - o);   // F[t][s], s - t = -o
    }
    w[tid] = v;
  }
}

// ---------------------------------------------------------------------------------------
// 2D
// ---------------------------------------------------------------------------------------
template <int P, int NT, int NC>
__global__ void __launch_bounds__(NT) k_op2d(const OpParams op, const Epi ep, int mode, int dot,
                                             const double* __restrict__ x, double* __restrict__ y,
                                             int chunk) {
  constexpr int R = 2 * P + 1;
  constexpr int W = NT + 2 * P;
  constexpr int LPT = (W + NT - 1) / NT;
  __shared__ double xs[2][NC][W];
  __shared__ double wts[2][3 * R];
  __shared__ double red[NT / 32];
  const int m = op.m;
  const size_t ms = (size_t)m * m;
  const int tid = threadIdx.x;
  const int t0 = blockIdx.x * NT;
  const int k = t0 + tid;
  const bool active = k < m;
  const int c0 = blockIdx.y * chunk;
  const int c1 = min(c0 + chunk, m);
  const int sb = max(0, c0 - P);
  const int se = c1 + P;
  const bool zone = active && (k < op.zoneL || k >= op.zoneR);

  double acc[NC][R];
#pragma unroll
  for (int i = 0; i < NC; ++i)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[i][r] = 0.0;
  double dsum = 0.0;

  // slab s -> xs[buf] by asynchronous copies (zero fill outside the domain)
  auto prefetch = [&](int s, int buf) {
#pragma unroll
    for (int j = 0; j < NC; ++j)
#pragma unroll
      for (int i = 0; i < LPT; ++i) {
        const int idx = tid + i * NT;
        const int col = t0 - P + idx;
        if (idx < W) {
          const bool ok = s < m && col >= 0 && col < m;
          cp_async8(&xs[buf][j][idx], ok ? x + j * ms + (size_t)s * m + col : x, ok);
        }
      }
    cp_async_commit();
  };

  prefetch(sb, 0);
  load_col_weights<P>(op, sb, c0, c1, wts[0]);
  cp_async_wait_all();
  __syncthreads();
#pragma unroll 1
  for (int s = sb; s < se; ++s) {
    const int buf = (s - sb) & 1;
    const bool more = s + 1 < se;
    if (more) {
      prefetch(s + 1, buf ^ 1);
      load_col_weights<P>(op, s + 1, c0, c1, wts[buf ^ 1]);
    }
    if (s < m) {
      double zM[NC], zS[NC], zA[NC];
      {
        double uM[NC], uS[NC], uA[NC];
#pragma unroll
        for (int j = 0; j < NC; ++j) {
          const double* xr = &xs[buf][j][tid + P];
          const double xc = xr[0];
          double vm = op.tM[0] * xc, vs = op.tS[0] * xc, va = 0.0;
#pragma unroll
          for (int o = 1; o <= P; ++o) {
            const double lo = xr[-o], hi = xr[o];
            const double sp = lo + hi, sm = hi - lo;
            vm = fma(op.tM[o], sp, vm);
            vs = fma(op.tS[o], sp, vs);
            va = fma(op.tA[o], sm, va);
          }
          if (zone) {
            const double* rM = op.bM + (size_t)k * R + P;
            const double* rS = op.bS + (size_t)k * R + P;
            const double* rA = op.bA + (size_t)k * R + P;
            vm = vs = va = 0.0;
#pragma unroll
            for (int o = -P; o <= P; ++o) {
              const double v = xr[o];
              vm = fma(__ldg(rM + o), v, vm);
              vs = fma(__ldg(rS + o), v, vs);
              va = fma(__ldg(rA + o), v, va);
            }
          }
          uM[j] = vm;
          uS[j] = vs;
          uA[j] = va;
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          zM[i] = zS[i] = zA[i] = 0.0;
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            zM[i] = fma(op.c.mass[i][j], uM[j], fma(op.c.S[1][i][j], uS[j], zM[i]));
            zS[i] = fma(op.c.S[0][i][j], uM[j], zS[i]);
            zA[i] = fma(op.c.AA[0][i][j], uA[j], zA[i]);
          }
        }
      }
      if (s - P >= op.zoneL && s + P < op.zoneR) {   // interior: Toeplitz register weights
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int d = P - r;                        // s - t
          const int ad = d < 0 ? -d : d;
          const double wM = op.tM[ad], wS = op.tS[ad], wA = d >= 0 ? op.tA[ad] : -op.tA[ad];
#pragma unroll
          for (int i = 0; i < NC; ++i) acc[i][r] = fma(wM, zM[i], fma(wS, zS[i], fma(wA, zA[i], acc[i][r])));
        }
      } else {
        const double* w = wts[buf];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double wM = w[r], wS = w[R + r], wA = w[2 * R + r];
#pragma unroll
          for (int i = 0; i < NC; ++i) acc[i][r] = fma(wM, zM[i], fma(wS, zS[i], fma(wA, zA[i], acc[i][r])));
        }
      }
    }
    {
      const int t = s - P;   // final: all contributions s' in [t-p, t+p] are in acc[.][0]
      if (t >= c0 && t < c1 && active) {
        const size_t pt = (size_t)t * m + k;
        double Dv[NC];
#pragma unroll
        for (int i = 0; i < NC; ++i) Dv[i] = 1.0;
        if (mode >= EPI_JACOBI) {
          const double Mt = __ldg(op.bM + (size_t)t * R + P), St = __ldg(op.bS + (size_t)t * R + P);
          const double Mk = __ldg(op.bM + (size_t)k * R + P), Sk = __ldg(op.bS + (size_t)k * R + P);
#pragma unroll
          for (int i = 0; i < NC; ++i)
            Dv[i] = op.c.mass[i][i] * Mt * Mk + op.c.S[0][i][i] * St * Mk + op.c.S[1][i][i] * Mt * Sk;
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          const double a = acc[i][0];
          const size_t gi = (size_t)i * ms + pt;
          double out;
          if (mode == EPI_APPLY) out = a;
          else if (mode == EPI_RESID) out = ep.b[gi] - a;
          else if (mode == EPI_JACOBI) out = x[gi] + ep.omega * (ep.b[gi] - a) / Dv[i];
          else out = a / Dv[i];
          y[gi] = out;
          if (dot == DOT_X_OUT) dsum = fma(x[gi], out, dsum);
          else if (dot == DOT_OUT_OUT) dsum = fma(out, out, dsum);
        }
      }
#pragma unroll
      for (int i = 0; i < NC; ++i) {
#pragma unroll
        for (int r = 0; r < R - 1; ++r) acc[i][r] = acc[i][r + 1];
        acc[i][R - 1] = 0.0;
      }
    }
    cp_async_wait_all();
    __syncthreads();
  }
  if (dot != DOT_NONE) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, off);
    if ((tid & 31) == 0) red[tid >> 5] = dsum;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int w = 0; w < NT / 32; ++w) sacc += red[w];
      ep.partial[blockIdx.y * gridDim.x + blockIdx.x] = sacc;
    }
  }
}

// ---------------------------------------------------------------------------------------
// 3D
// ---------------------------------------------------------------------------------------
template <int P, int T2, int T3, int NC>
struct Op3dShape {
  static constexpr int NT = T2 * T3;
  static constexpr int R = 2 * P + 1;
  static constexpr int HR = T2 + 2 * P;
  static constexpr int HC = T3 + 2 * P;
  static constexpr int XS = HR * HC;        // one component of one slab tile
  static constexpr int US = T2 * HC;        // one stage-A output array
  static constexpr int XB = (NC * XS + 15) / 16 * 16;  // one slab buffer, padded to 128 bytes (TMA)
  static constexpr int SMEM = (2 * XB + 3 * NC * US + 2 * 3 * R) * 8 + (NT / 32) * 8 + 2 * 8;
  static constexpr int LPT = (NC * XS + NT - 1) / NT;
};

template <int P, int T2, int T3, int NC, int MINB, bool TMA>
__global__ void __launch_bounds__(T2* T3, MINB) k_op3d(const OpParams op, const Epi ep, int mode, int dot,
                                                    const double* __restrict__ x, double* __restrict__ y,
                                                    int chunk, const __grid_constant__ CUtensorMap tmap) {
  using Sh = Op3dShape<P, T2, T3, NC>;
  constexpr int NT = Sh::NT, R = Sh::R, HR = Sh::HR, HC = Sh::HC, XS = Sh::XS, US = Sh::US, LPT = Sh::LPT;
  constexpr int XB = Sh::XB;
  static_assert(LPT <= 32, "prefetch mask");
  extern __shared__ __align__(128) double smem[];
  double* xs = smem;                   // [2][XB]: [NC][HR][HC] each
  double* us = smem + 2 * XB;          // [3][NC][T2][HC]: index (F*NC + j), F: 0 M, 1 S, 2 A
  double* wts = us + 3 * NC * US;      // [2][3R]
  double* red = wts + 2 * 3 * R;
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(red + NT / 32);  // [2]
  const int m = op.m;
  const int ms = m * m;                // ndof < 2^31 is checked on the host
  const int m3 = ms * m;
  const int tid = threadIdx.x;
  const int tr = tid / T3, tc = tid % T3;
  const int r0 = blockIdx.y * T2, q0 = blockIdx.x * T3;
  const int gr = r0 + tr, gc = q0 + tc;
  const bool active = gr < m && gc < m;
  const bool zoneB = active && (gc < op.zoneL || gc >= op.zoneR);
  const int c0 = blockIdx.z * chunk;
  const int c1 = min(c0 + chunk, m);
  const int sb = max(0, c0 - P);
  const int se = c1 + P;

  // ---- slab-invariant per-thread offsets -------------------------------------------------
  int goff[TMA ? 1 : LPT];   // global offset (without the slab term) of each prefetch slot
  unsigned vmask = 0u;       // slot is inside the domain (in-plane)
#pragma unroll
  for (int i = 0; i < (TMA ? 0 : LPT); ++i) {
    const int idx = tid + i * NT;
    goff[i] = 0;
    if (idx < NC * XS) {
      const int j = idx / XS, rem = idx % XS;
      const int g1 = r0 - P + rem / HC, g2 = q0 - P + rem % HC;
      if (g1 >= 0 && g1 < m && g2 >= 0 && g2 < m) {
        goff[i] = j * m3 + g1 * m + g2;
        vmask |= 1u << i;
      }
    }
  }
  // stage A work item: (half of the tile rows, component, halo column), lanes along columns;
  // each item marches down its T2/2 output rows with a register window of T2/2 + 2P inputs
  constexpr int RH = T2 / 2;
  static_assert(T2 % 2 == 0, "two row halves");
  constexpr int NITEMS = 2 * NC * HC;
  const bool wzb = __any_sync(0xffffffffu, zoneB);
  const int bo = tr * HC + tc + P;     // stage-B window centre
  const int pto = gr * m + gc;         // in-slab output offset

  double acc[NC][R];
#pragma unroll
  for (int i = 0; i < NC; ++i)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[i][r] = 0.0;
  double dsum = 0.0;

  // slab s -> xs[buf]: one TMA box (HC x HR x 1 x NC, out-of-range elements zero-filled)
  // issued by thread 0 and completed on mbar[buf], or per-thread cp.async copies
  auto prefetch = [&](int s, int buf) {
    if constexpr (TMA) {
      if (tid == 0 && s < m) {
        fence_proxy_async();
        mbar_expect_tx(&mbar[buf], (unsigned)(NC * XS * 8));
        tma_load_4d(xs + buf * XB, &tmap, q0 - P, r0 - P, s, 0, &mbar[buf]);
      }
    } else {
      double* dst = xs + buf * XB + tid;
      const bool sv = s < m;
      const double* src = x + (size_t)s * ms;
#pragma unroll
      for (int i = 0; i < LPT; ++i) {
        if (tid + i * NT < NC * XS) {
          const bool ok = sv && ((vmask >> i) & 1u);
          cp_async8(dst + i * NT, ok ? src + goff[i] : x, ok);
        }
      }
      cp_async_commit();
    }
  };
  auto slab_ready = [&](int s, int buf) {   // TMA: wait for the bytes of slab s
    if constexpr (TMA) {
      if (s < m) mbar_wait(&mbar[buf], (unsigned)(((s - sb) >> 1) & 1));
    }
  };
  (void)HR;

  // stage A: contract direction 1 for RH consecutive rows of one (component, column)
  auto stageA = [&](const double* xb, int it) {
    const int a_cc = it % HC, a_j = (it / HC) % NC, a_r0 = (it / (NC * HC)) * RH;
    const double* col = xb + a_j * XS + a_r0 * HC + a_cc;   // input row a_r0 - P (halo origin)
    double win[RH + 2 * P];
#pragma unroll
    for (int k = 0; k < RH + 2 * P; ++k) win[k] = col[k * HC];
    double* uMo = us + (0 * NC + a_j) * US + a_r0 * HC + a_cc;
    double* uSo = us + (1 * NC + a_j) * US + a_r0 * HC + a_cc;
    double* uAo = us + (2 * NC + a_j) * US + a_r0 * HC + a_cc;
    const int g0 = r0 + a_r0;                                  // global row of the first output
    const bool zone_any = g0 < op.zoneL || g0 + RH > op.zoneR; // warp-uniform (depends on a_hf)
#pragma unroll
    for (int r = 0; r < RH; ++r) {
      const double xc = win[r + P];
      double vm = op.tM[0] * xc, vs = op.tS[0] * xc, va = 0.0;
#pragma unroll
      for (int o = 1; o <= P; ++o) {
        const double lo = win[r + P - o], hi = win[r + P + o];
        const double sp = lo + hi, sm = hi - lo;
        vm = fma(op.tM[o], sp, vm);
        vs = fma(op.tS[o], sp, vs);
        va = fma(op.tA[o], sm, va);
      }
      if (zone_any) {
        const int g1 = g0 + r;
        if (g1 < m && (g1 < op.zoneL || g1 >= op.zoneR)) {
          const double* rM = op.bM + g1 * R + P;
          const double* rS = op.bS + g1 * R + P;
          const double* rA = op.bA + g1 * R + P;
          vm = vs = va = 0.0;
#pragma unroll
          for (int o = -P; o <= P; ++o) {
            const double v = win[r + P + o];
            vm = fma(__ldg(rM + o), v, vm);
            vs = fma(__ldg(rS + o), v, vs);
            va = fma(__ldg(rA + o), v, va);
          }
        }
      }
      uMo[r * HC] = vm;
      uSo[r * HC] = vs;
      uAo[r * HC] = va;
    }
  };

  if constexpr (TMA) {
    if (tid == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  prefetch(sb, 0);
  load_col_weights<P>(op, sb, c0, c1, wts);
  if constexpr (!TMA) cp_async_wait_all();
  __syncthreads();
#pragma unroll 1
  for (int s = sb; s < se; ++s) {
    const int buf = (s - sb) & 1;
    const bool more = s + 1 < se;
    if (more) {
      prefetch(s + 1, buf ^ 1);
      load_col_weights<P>(op, s + 1, c0, c1, wts + (buf ^ 1) * 3 * R);
    }
    slab_ready(s, buf);
    if (s < m) {
#pragma unroll 1
      for (int it = tid; it < NITEMS; it += NT) stageA(xs + buf * XB, it);
      __syncthreads();
      // ---- stage B: contract direction 2, combine patterns into z_{i,F0}
      double zM[NC], zS[NC], zA[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) zM[i] = zS[i] = zA[i] = 0.0;
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const double* uM = us + (0 * NC + j) * US + bo;
        const double* uS = us + (1 * NC + j) * US + bo;
        const double* uA = us + (2 * NC + j) * US + bo;
        double vMM, vMS, vMA, vSM, vAM, vAA;
        {
          const double c = uM[0];
          double a1 = op.tM[0] * c, a2 = op.tS[0] * c, a3 = 0.0;
#pragma unroll
          for (int o = 1; o <= P; ++o) {
            const double lo = uM[-o], hi = uM[o];
            const double sp = lo + hi, sm = hi - lo;
            a1 = fma(op.tM[o], sp, a1);
            a2 = fma(op.tS[o], sp, a2);
            a3 = fma(op.tA[o], sm, a3);
          }
          vMM = a1; vMS = a2; vMA = a3;
        }
        {
          double a1 = op.tM[0] * uS[0];
#pragma unroll
          for (int o = 1; o <= P; ++o) a1 = fma(op.tM[o], uS[-o] + uS[o], a1);
          vSM = a1;
        }
        {
          const double c = uA[0];
          double a1 = op.tM[0] * c, a3 = 0.0;
#pragma unroll
          for (int o = 1; o <= P; ++o) {
            const double lo = uA[-o], hi = uA[o];
            a1 = fma(op.tM[o], lo + hi, a1);
            a3 = fma(op.tA[o], hi - lo, a3);
          }
          vAM = a1; vAA = a3;
        }
        if (wzb && zoneB) {
          const double* rM = op.bM + gc * R + P;
          const double* rS = op.bS + gc * R + P;
          const double* rA = op.bA + gc * R + P;
          vMM = vMS = vMA = vSM = vAM = vAA = 0.0;
#pragma unroll
          for (int o = -P; o <= P; ++o) {
            const double wm = __ldg(rM + o), ws = __ldg(rS + o), wa = __ldg(rA + o);
            vMM = fma(wm, uM[o], vMM);
            vMS = fma(ws, uM[o], vMS);
            vMA = fma(wa, uM[o], vMA);
            vSM = fma(wm, uS[o], vSM);
            vAM = fma(wm, uA[o], vAM);
            vAA = fma(wa, uA[o], vAA);
          }
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          zM[i] = fma(op.c.mass[i][j], vMM, zM[i]);
          zS[i] = fma(op.c.S[0][i][j], vMM, zS[i]);
          zM[i] = fma(op.c.S[1][i][j], vSM, zM[i]);
          zM[i] = fma(op.c.S[2][i][j], vMS, zM[i]);
          zA[i] = fma(op.c.AA[0][i][j], vAM, zA[i]);
          zA[i] = fma(op.c.AA[1][i][j], vMA, zA[i]);
          zM[i] = fma(op.c.AA[2][i][j], vAA, zM[i]);
        }
      }
      // ---- stage C: scatter along direction 0 into the ring.  Rows t = s-P+r; when all of
      // them are Toeplitz rows, F[t][s] = T[s-t] is a register constant (A: skew sign);
      // rows outside this CTA's chunk are never written, so they need no masking here.
      if (s - P >= op.zoneL && s + P < op.zoneR) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int d = P - r;                        // s - t
          const int ad = d < 0 ? -d : d;
          const double wM = op.tM[ad], wS = op.tS[ad], wA = d >= 0 ? op.tA[ad] : -op.tA[ad];
#pragma unroll
          for (int i = 0; i < NC; ++i) acc[i][r] = fma(wM, zM[i], fma(wS, zS[i], fma(wA, zA[i], acc[i][r])));
        }
      } else {
        const double* w = wts + buf * 3 * R;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double wM = w[r], wS = w[R + r], wA = w[2 * R + r];
#pragma unroll
          for (int i = 0; i < NC; ++i) acc[i][r] = fma(wM, zM[i], fma(wS, zS[i], fma(wA, zA[i], acc[i][r])));
        }
      }
    }
    {
      const int t = s - P;
      if (t >= c0 && t < c1 && active) {
        const int pt = t * ms + pto;
        double Dv[NC];
#pragma unroll
        for (int i = 0; i < NC; ++i) Dv[i] = 1.0;
        if (mode >= EPI_JACOBI) {
          const double M0 = __ldg(op.bM + t * R + P), S0 = __ldg(op.bS + t * R + P);
          const double M1 = __ldg(op.bM + gr * R + P), S1 = __ldg(op.bS + gr * R + P);
          const double M2 = __ldg(op.bM + gc * R + P), S2 = __ldg(op.bS + gc * R + P);
#pragma unroll
          for (int i = 0; i < NC; ++i)
            Dv[i] = op.c.mass[i][i] * M0 * M1 * M2 + op.c.S[0][i][i] * S0 * M1 * M2 +
                    op.c.S[1][i][i] * M0 * S1 * M2 + op.c.S[2][i][i] * M0 * M1 * S2;
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          const double a = acc[i][0];
          const int gi = i * m3 + pt;
          double out;
          if (mode == EPI_APPLY) out = a;
          else if (mode == EPI_RESID) out = ep.b[gi] - a;
          else if (mode == EPI_JACOBI) out = x[gi] + ep.omega * (ep.b[gi] - a) / Dv[i];
          else out = a / Dv[i];
          y[gi] = out;
          if (dot == DOT_X_OUT) dsum = fma(x[gi], out, dsum);
          else if (dot == DOT_OUT_OUT) dsum = fma(out, out, dsum);
        }
      }
#pragma unroll
      for (int i = 0; i < NC; ++i) {
#pragma unroll
        for (int r = 0; r < R - 1; ++r) acc[i][r] = acc[i][r + 1];
        acc[i][R - 1] = 0.0;
      }
    }
    if constexpr (!TMA) cp_async_wait_all();
    __syncthreads();
  }
  if (dot != DOT_NONE) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, off);
    if ((tid & 31) == 0) red[tid >> 5] = dsum;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int w = 0; w < NT / 32; ++w) sacc += red[w];
      ep.partial[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = sacc;
    }
  }
}

// ---------------------------------------------------------------------------------------
// 3D, two output points per thread (adjacent along direction 2): halves the stage-B shared
// loads and the per-point coefficient loads, and doubles the independent work per thread.
// ---------------------------------------------------------------------------------------
template <int P, int T2, int T3, int NC>
struct Op3d2Shape {
  static constexpr int NT = T2 * T3 / 2;
  static constexpr int R = 2 * P + 1;
  static constexpr int HR = T2 + 2 * P;
  static constexpr int HC = T3 + 2 * P;     // even
  static constexpr int XS = HR * HC;
  static constexpr int US = T2 * HC;
  static constexpr int XB = (NC * XS + 15) / 16 * 16;
  static constexpr int SMEM = (2 * XB + 3 * NC * US + 2 * 3 * R) * 8 + (NT / 32) * 8 + 2 * 8;
  static constexpr int LPT = (NC * XS + NT - 1) / NT;
  static constexpr int ITEMS = T2 * HC / 2;   // stage-A column pairs
};

template <int P, int T2, int T3, int NC, bool TMA>
__global__ void __launch_bounds__(T2* T3 / 2, 1) k_op3d2(const OpParams op, const Epi ep, int mode, int dot,
                                                       const double* __restrict__ x, double* __restrict__ y,
                                                       int chunk, const __grid_constant__ CUtensorMap tmap) {
  using Sh = Op3d2Shape<P, T2, T3, NC>;
  constexpr int NT = Sh::NT, R = Sh::R, HC = Sh::HC, XS = Sh::XS, US = Sh::US, LPT = Sh::LPT, XB = Sh::XB;
  constexpr int ITEMS = Sh::ITEMS;
  static_assert(HC % 2 == 0, "pairs");
  static_assert(ITEMS <= 2 * NT, "at most two stage-A items per thread");
  extern __shared__ __align__(128) double smem[];
  double* xs = smem;
  double* us = smem + 2 * XB;
  double* wts = us + 3 * NC * US;
  double* red = wts + 2 * 3 * R;
  unsigned long long* mbar = reinterpret_cast<unsigned long long*>(red + NT / 32);
  const int m = op.m;
  const int ms = m * m;
  const int m3 = ms * m;
  const int tid = threadIdx.x;
  const int tr = tid / (T3 / 2), tc = 2 * (tid % (T3 / 2));
  const int r0 = blockIdx.y * T2, q0 = blockIdx.x * T3;
  const int gr = r0 + tr, gc = q0 + tc;
  const bool act0 = gr < m && gc < m, act1 = gr < m && gc + 1 < m;
  const bool zB0 = act0 && (gc < op.zoneL || gc >= op.zoneR);
  const bool zB1 = act1 && (gc + 1 < op.zoneL || gc + 1 >= op.zoneR);
  const int c0 = blockIdx.z * chunk;
  const int c1 = min(c0 + chunk, m);
  const int sb = max(0, c0 - P);
  const int se = c1 + P;

  int goff[TMA ? 1 : LPT];
  unsigned vmask = 0u;
#pragma unroll
  for (int i = 0; i < (TMA ? 0 : LPT); ++i) {
    const int idx = tid + i * NT;
    goff[i] = 0;
    if (idx < NC * XS) {
      const int j = idx / XS, rem = idx % XS;
      const int g1 = r0 - P + rem / HC, g2 = q0 - P + rem % HC;
      if (g1 >= 0 && g1 < m && g2 >= 0 && g2 < m) {
        goff[i] = j * m3 + g1 * m + g2;
        vmask |= 1u << i;
      }
    }
  }
  const int it0 = tid, it1 = tid + NT;
  const bool has1 = it1 < ITEMS;
  auto item_xo = [&](int it) { return (it / (HC / 2) + P) * HC + 2 * (it % (HC / 2)); };
  const int xo0 = item_xo(it0), xo1 = has1 ? item_xo(it1) : 0;
  const int uo0 = (it0 / (HC / 2)) * HC + 2 * (it0 % (HC / 2));
  const int uo1 = has1 ? (it1 / (HC / 2)) * HC + 2 * (it1 % (HC / 2)) : 0;
  const int ga0 = r0 + it0 / (HC / 2), ga1 = r0 + it1 / (HC / 2);
  const bool za0 = ga0 < m && (ga0 < op.zoneL || ga0 >= op.zoneR);
  const bool za1 = has1 && ga1 < m && (ga1 < op.zoneL || ga1 >= op.zoneR);
  const bool wza0 = __any_sync(0xffffffffu, za0), wza1 = __any_sync(0xffffffffu, za1);
  const bool wzb = __any_sync(0xffffffffu, zB0 || zB1);
  const int bo = tr * HC + tc + P;
  const int pto = gr * m + gc;

  double acc[2][NC][R];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[q][i][r] = 0.0;
  double dsum = 0.0;

  auto prefetch = [&](int s, int buf) {
    if constexpr (TMA) {
      if (tid == 0 && s < m) {
        fence_proxy_async();
        mbar_expect_tx(&mbar[buf], (unsigned)(NC * XS * 8));
        tma_load_4d(xs + buf * XB, &tmap, q0 - P, r0 - P, s, 0, &mbar[buf]);
      }
    } else {
      double* dst = xs + buf * XB + tid;
      const bool sv = s < m;
      const double* src = x + (size_t)s * ms;
#pragma unroll
      for (int i = 0; i < LPT; ++i) {
        if (tid + i * NT < NC * XS) {
          const bool ok = sv && ((vmask >> i) & 1u);
          cp_async8(dst + i * NT, ok ? src + goff[i] : x, ok);
        }
      }
      cp_async_commit();
    }
  };

  // stage A on a column pair: contract direction 1 (double2 loads / stores)
  auto stageA = [&](const double* xb, int xo, int uo, int g1, bool zone, bool wzone) {
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const double* xc_ = xb + j * XS + xo;
      const double2 c = *reinterpret_cast<const double2*>(xc_);
      double m0 = op.tM[0] * c.x, s0 = op.tS[0] * c.x, a0 = 0.0;
      double m1 = op.tM[0] * c.y, s1 = op.tS[0] * c.y, a1 = 0.0;
#pragma unroll
      for (int o = 1; o <= P; ++o) {
        const double2 lo = *reinterpret_cast<const double2*>(xc_ - o * HC);
        const double2 hi = *reinterpret_cast<const double2*>(xc_ + o * HC);
        const double sp0 = lo.x + hi.x, sm0 = hi.x - lo.x, sp1 = lo.y + hi.y, sm1 = hi.y - lo.y;
        m0 = fma(op.tM[o], sp0, m0); s0 = fma(op.tS[o], sp0, s0); a0 = fma(op.tA[o], sm0, a0);
        m1 = fma(op.tM[o], sp1, m1); s1 = fma(op.tS[o], sp1, s1); a1 = fma(op.tA[o], sm1, a1);
      }
      if (wzone && zone) {
        const double* rM = op.bM + g1 * R + P;
        const double* rS = op.bS + g1 * R + P;
        const double* rA = op.bA + g1 * R + P;
        m0 = s0 = a0 = m1 = s1 = a1 = 0.0;
#pragma unroll
        for (int o = -P; o <= P; ++o) {
          const double2 v = *reinterpret_cast<const double2*>(xc_ + o * HC);
          const double wm = __ldg(rM + o), ws = __ldg(rS + o), wa = __ldg(rA + o);
          m0 = fma(wm, v.x, m0); s0 = fma(ws, v.x, s0); a0 = fma(wa, v.x, a0);
          m1 = fma(wm, v.y, m1); s1 = fma(ws, v.y, s1); a1 = fma(wa, v.y, a1);
        }
      }
      *reinterpret_cast<double2*>(us + (0 * NC + j) * US + uo) = make_double2(m0, m1);
      *reinterpret_cast<double2*>(us + (1 * NC + j) * US + uo) = make_double2(s0, s1);
      *reinterpret_cast<double2*>(us + (2 * NC + j) * US + uo) = make_double2(a0, a1);
    }
  };

  if constexpr (TMA) {
    if (tid == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  prefetch(sb, 0);
  load_col_weights<P>(op, sb, c0, c1, wts);
  if constexpr (!TMA) cp_async_wait_all();
  __syncthreads();
#pragma unroll 1
  for (int s = sb; s < se; ++s) {
    const int buf = (s - sb) & 1;
    const bool more = s + 1 < se;
    if (more) {
      prefetch(s + 1, buf ^ 1);
      load_col_weights<P>(op, s + 1, c0, c1, wts + (buf ^ 1) * 3 * R);
    }
    if constexpr (TMA) {
      if (s < m) mbar_wait(&mbar[buf], (unsigned)(((s - sb) >> 1) & 1));
    }
    if (s < m) {
      const double* xb = xs + buf * XB;
      stageA(xb, xo0, uo0, ga0, za0, wza0);
      if (has1) stageA(xb, xo1, uo1, ga1, za1, wza1);
      __syncthreads();
      double z[2][3][NC];   // [point][F: M, S, A][component]
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int f = 0; f < 3; ++f)
#pragma unroll
          for (int i = 0; i < NC; ++i) z[q][f][i] = 0.0;
#pragma unroll
      for (int j = 0; j < NC; ++j) {
        const double* uM = us + (0 * NC + j) * US + bo;
        const double* uS = us + (1 * NC + j) * US + bo;
        const double* uA = us + (2 * NC + j) * US + bo;
        double v[2][6];   // MM MS MA SM AM AA
        {
          double w[2 * P + 2];
#pragma unroll
          for (int o = 0; o < 2 * P + 2; ++o) w[o] = uM[o - P];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const double c = w[P + q];
            double a1 = op.tM[0] * c, a2 = op.tS[0] * c, a3 = 0.0;
#pragma unroll
            for (int o = 1; o <= P; ++o) {
              const double lo = w[P + q - o], hi = w[P + q + o];
              const double sp = lo + hi, sm = hi - lo;
              a1 = fma(op.tM[o], sp, a1);
              a2 = fma(op.tS[o], sp, a2);
              a3 = fma(op.tA[o], sm, a3);
            }
            v[q][0] = a1; v[q][1] = a2; v[q][2] = a3;
          }
        }
        {
          double w[2 * P + 2];
#pragma unroll
          for (int o = 0; o < 2 * P + 2; ++o) w[o] = uS[o - P];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            double a1 = op.tM[0] * w[P + q];
#pragma unroll
            for (int o = 1; o <= P; ++o) a1 = fma(op.tM[o], w[P + q - o] + w[P + q + o], a1);
            v[q][3] = a1;
          }
        }
        {
          double w[2 * P + 2];
#pragma unroll
          for (int o = 0; o < 2 * P + 2; ++o) w[o] = uA[o - P];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            double a1 = op.tM[0] * w[P + q], a3 = 0.0;
#pragma unroll
            for (int o = 1; o <= P; ++o) {
              const double lo = w[P + q - o], hi = w[P + q + o];
              a1 = fma(op.tM[o], lo + hi, a1);
              a3 = fma(op.tA[o], hi - lo, a3);
            }
            v[q][4] = a1; v[q][5] = a3;
          }
        }
        if (wzb && (zB0 || zB1)) {
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (q == 0 ? zB0 : zB1) {
              const int col = gc + q;
              const double* rM = op.bM + col * R + P;
              const double* rS = op.bS + col * R + P;
              const double* rA = op.bA + col * R + P;
#pragma unroll
              for (int k = 0; k < 6; ++k) v[q][k] = 0.0;
#pragma unroll
              for (int o = -P; o <= P; ++o) {
                const double wm = __ldg(rM + o), ws = __ldg(rS + o), wa = __ldg(rA + o);
                const double xm = uM[o + q], xsv = uS[o + q], xa = uA[o + q];
                v[q][0] = fma(wm, xm, v[q][0]);
                v[q][1] = fma(ws, xm, v[q][1]);
                v[q][2] = fma(wa, xm, v[q][2]);
                v[q][3] = fma(wm, xsv, v[q][3]);
                v[q][4] = fma(wm, xa, v[q][4]);
                v[q][5] = fma(wa, xa, v[q][5]);
              }
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          const double cm = op.c.mass[i][j], c0_ = op.c.S[0][i][j], c1_ = op.c.S[1][i][j], c2_ = op.c.S[2][i][j];
          const double d0 = op.c.AA[0][i][j], d1 = op.c.AA[1][i][j], d2 = op.c.AA[2][i][j];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            z[q][0][i] = fma(cm, v[q][0], fma(c1_, v[q][3], fma(c2_, v[q][1], fma(d2, v[q][5], z[q][0][i]))));
            z[q][1][i] = fma(c0_, v[q][0], z[q][1][i]);
            z[q][2][i] = fma(d0, v[q][4], fma(d1, v[q][2], z[q][2][i]));
          }
        }
      }
      const double* w = wts + buf * 3 * R;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const double wM = w[r], wS = w[R + r], wA = w[2 * R + r];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int i = 0; i < NC; ++i)
            acc[q][i][r] = fma(wM, z[q][0][i], fma(wS, z[q][1][i], fma(wA, z[q][2][i], acc[q][i][r])));
      }
    }
    {
      const int t = s - P;
      if (t >= c0 && t < c1) {
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (q == 0 ? act0 : act1) {
            const int pt = t * ms + pto + q;
            double Dv[NC];
#pragma unroll
            for (int i = 0; i < NC; ++i) Dv[i] = 1.0;
            if (mode >= EPI_JACOBI) {
              const int col = gc + q;
              const double M0 = __ldg(op.bM + t * R + P), S0 = __ldg(op.bS + t * R + P);
              const double M1 = __ldg(op.bM + gr * R + P), S1 = __ldg(op.bS + gr * R + P);
              const double M2 = __ldg(op.bM + col * R + P), S2 = __ldg(op.bS + col * R + P);
#pragma unroll
              for (int i = 0; i < NC; ++i)
                Dv[i] = op.c.mass[i][i] * M0 * M1 * M2 + op.c.S[0][i][i] * S0 * M1 * M2 +
                        op.c.S[1][i][i] * M0 * S1 * M2 + op.c.S[2][i][i] * M0 * M1 * S2;
            }
#pragma unroll
            for (int i = 0; i < NC; ++i) {
              const double a = acc[q][i][0];
              const int gi = i * m3 + pt;
              double out;
              if (mode == EPI_APPLY) out = a;
              else if (mode == EPI_RESID) out = ep.b[gi] - a;
              else if (mode == EPI_JACOBI) out = x[gi] + ep.omega * (ep.b[gi] - a) / Dv[i];
              else out = a / Dv[i];
              y[gi] = out;
              if (dot == DOT_X_OUT) dsum = fma(x[gi], out, dsum);
              else if (dot == DOT_OUT_OUT) dsum = fma(out, out, dsum);
            }
          }
        }
      }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < NC; ++i) {
#pragma unroll
          for (int r = 0; r < R - 1; ++r) acc[q][i][r] = acc[q][i][r + 1];
          acc[q][i][R - 1] = 0.0;
        }
    }
    if constexpr (!TMA) cp_async_wait_all();
    __syncthreads();
  }
  if (dot != DOT_NONE) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, off);
    if ((tid & 31) == 0) red[tid >> 5] = dsum;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int w = 0; w < NT / 32; ++w) sacc += red[w];
      ep.partial[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = sacc;
    }
  }
}

// ---------------------------------------------------------------------------------------
// 3D, split form: (S) per slab, contract the two in-slab directions and form the per-point
// combinations z_{F,i}(s) (written to a 3*NC-array buffer Z in HBM); (C) per column, march
// along direction 0 and scatter F0[t][s] z_{F,i}(s) into a register ring (epilogue as above).
// Each kernel keeps little live state, so both run at high occupancy without spills; the
// price is the Z round trip (9 doubles per point for the vector operator).
// ---------------------------------------------------------------------------------------
template <int P, int T2, int T3, int NC>
struct SlabShape {
  static constexpr int NT = T2 * T3;
  static constexpr int HR = T2 + 2 * P;
  static constexpr int HC = T3 + 2 * P;
  static constexpr int XS = HR * HC;
  static constexpr int US = T2 * HC;
  static constexpr int SMEM = (NC * XS + 3 * NC * US) * 8;
  static constexpr int LPT = (NC * XS + NT - 1) / NT;
};

template <int P, int T2, int T3, int NC>
__global__ void __launch_bounds__(T2* T3) k_slab3d(const OpParams op, const double* __restrict__ x,
                                                   double* __restrict__ Z) {
  using Sh = SlabShape<P, T2, T3, NC>;
  constexpr int NT = Sh::NT, R = 2 * P + 1, HC = Sh::HC, XS = Sh::XS, US = Sh::US, LPT = Sh::LPT;
  constexpr int RH = T2 / 2;
  extern __shared__ __align__(16) double smem[];
  double* xs = smem;               // [NC][HR][HC]
  double* us = smem + NC * XS;     // [3][NC][T2][HC]
  const int m = op.m;
  const int ms = m * m, m3 = ms * m;
  const int s = blockIdx.z;
  const int tid = threadIdx.x;
  const int tr = tid / T3, tc = tid % T3;
  const int r0 = blockIdx.y * T2, q0 = blockIdx.x * T3;
  const int gr = r0 + tr, gc = q0 + tc;
  const bool active = gr < m && gc < m;
  const bool zoneB = active && (gc < op.zoneL || gc >= op.zoneR);
  const bool wzb = __any_sync(0xffffffffu, zoneB);
  // ---- slab tile with halo -> shared memory (zero outside the domain)
  const double* src = x + (size_t)s * ms;
#pragma unroll
  for (int i = 0; i < LPT; ++i) {
    const int idx = tid + i * NT;
    if (idx < NC * XS) {
      const int j = idx / XS, rem = idx % XS;
      const int g1 = r0 - P + rem / HC, g2 = q0 - P + rem % HC;
      const bool ok = g1 >= 0 && g1 < m && g2 >= 0 && g2 < m;
      cp_async8(xs + idx, ok ? src + j * m3 + g1 * m + g2 : x, ok);
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  // ---- stage A: direction 1, lockstep over RH rows per (half, component, column)
  for (int it = tid; it < 2 * NC * HC; it += NT) {
    const int a_cc = it % HC, a_j = (it / HC) % NC, a_r0 = (it / (NC * HC)) * RH;
    const double* col = xs + a_j * XS + a_r0 * HC + a_cc;
    double win[RH + 2 * P];
#pragma unroll
    for (int k = 0; k < RH + 2 * P; ++k) win[k] = col[k * HC];
    const int g0 = r0 + a_r0;
    const bool zone_any = g0 < op.zoneL || g0 + RH > op.zoneR;
#pragma unroll
    for (int r = 0; r < RH; ++r) {
      const double xc = win[r + P];
      double vm = op.tM[0] * xc, vs = op.tS[0] * xc, va = 0.0;
#pragma unroll
      for (int o = 1; o <= P; ++o) {
        const double lo = win[r + P - o], hi = win[r + P + o];
        const double sp = lo + hi, sm = hi - lo;
        vm = fma(op.tM[o], sp, vm);
        vs = fma(op.tS[o], sp, vs);
        va = fma(op.tA[o], sm, va);
      }
      if (zone_any) {
        const int g1 = g0 + r;
        if (g1 < m && (g1 < op.zoneL || g1 >= op.zoneR)) {
          const double* rM = op.bM + g1 * R + P;
          const double* rS = op.bS + g1 * R + P;
          const double* rA = op.bA + g1 * R + P;
          vm = vs = va = 0.0;
#pragma unroll
          for (int o = -P; o <= P; ++o) {
            const double v = win[r + P + o];
            vm = fma(__ldg(rM + o), v, vm);
            vs = fma(__ldg(rS + o), v, vs);
            va = fma(__ldg(rA + o), v, va);
          }
        }
      }
      const int uo = (a_r0 + r) * HC + a_cc;
      us[(0 * NC + a_j) * US + uo] = vm;
      us[(1 * NC + a_j) * US + uo] = vs;
      us[(2 * NC + a_j) * US + uo] = va;
    }
  }
  __syncthreads();
  if (!active) return;
  // ---- stage B: direction 2 and the pattern combinations
  double zM[NC], zS[NC], zA[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) zM[i] = zS[i] = zA[i] = 0.0;
  const int bo = tr * HC + tc + P;
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    const double* uM = us + (0 * NC + j) * US + bo;
    const double* uS = us + (1 * NC + j) * US + bo;
    const double* uA = us + (2 * NC + j) * US + bo;
    double vMM, vMS, vMA, vSM, vAM, vAA;
    {
      const double c = uM[0];
      double a1 = op.tM[0] * c, a2 = op.tS[0] * c, a3 = 0.0;
#pragma unroll
      for (int o = 1; o <= P; ++o) {
        const double lo = uM[-o], hi = uM[o];
        const double sp = lo + hi, sm = hi - lo;
        a1 = fma(op.tM[o], sp, a1);
        a2 = fma(op.tS[o], sp, a2);
        a3 = fma(op.tA[o], sm, a3);
      }
      vMM = a1; vMS = a2; vMA = a3;
    }
    {
      double a1 = op.tM[0] * uS[0];
#pragma unroll
      for (int o = 1; o <= P; ++o) a1 = fma(op.tM[o], uS[-o] + uS[o], a1);
      vSM = a1;
    }
    {
      const double c = uA[0];
      double a1 = op.tM[0] * c, a3 = 0.0;
#pragma unroll
      for (int o = 1; o <= P; ++o) {
        const double lo = uA[-o], hi = uA[o];
        a1 = fma(op.tM[o], lo + hi, a1);
        a3 = fma(op.tA[o], hi - lo, a3);
      }
      vAM = a1; vAA = a3;
    }
    if (wzb && zoneB) {
      const double* rM = op.bM + gc * R + P;
      const double* rS = op.bS + gc * R + P;
      const double* rA = op.bA + gc * R + P;
      vMM = vMS = vMA = vSM = vAM = vAA = 0.0;
#pragma unroll
      for (int o = -P; o <= P; ++o) {
        const double wm = __ldg(rM + o), ws = __ldg(rS + o), wa = __ldg(rA + o);
        vMM = fma(wm, uM[o], vMM);
        vMS = fma(ws, uM[o], vMS);
        vMA = fma(wa, uM[o], vMA);
        vSM = fma(wm, uS[o], vSM);
        vAM = fma(wm, uA[o], vAM);
        vAA = fma(wa, uA[o], vAA);
      }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      zM[i] = fma(op.c.mass[i][j], vMM, zM[i]);
      zS[i] = fma(op.c.S[0][i][j], vMM, zS[i]);
      zM[i] = fma(op.c.S[1][i][j], vSM, zM[i]);
      zM[i] = fma(op.c.S[2][i][j], vMS, zM[i]);
      zA[i] = fma(op.c.AA[0][i][j], vAM, zA[i]);
      zA[i] = fma(op.c.AA[1][i][j], vMA, zA[i]);
      zM[i] = fma(op.c.AA[2][i][j], vAA, zM[i]);
    }
  }
  const int pt = s * ms + gr * m + gc;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    Z[(size_t)(0 * NC + i) * m3 + pt] = zM[i];
    Z[(size_t)(1 * NC + i) * m3 + pt] = zS[i];
    Z[(size_t)(2 * NC + i) * m3 + pt] = zA[i];
  }
}

// (S2): as k_slab3d, but each thread forms TWO adjacent outputs along direction 2 from one
// window of 2P+2 values read as 16-byte pairs (LDS.128): 44% fewer shared-memory wavefronts
// in stage B, which dominated the slab kernel's shared-memory traffic.
template <int P, int T2, int T3, int NC>
struct Slab2Shape {
  static constexpr int TC = T3 / 2;             // threads per row
  static constexpr int NT = T2 * TC;
  static constexpr int HR = T2 + 2 * P;
  static constexpr int HC = T3 + 2 * P;         // even: rows stay 16-byte aligned
  static constexpr int XS = HR * HC;
  static constexpr int US = T2 * HC;
  static constexpr int SMEM = (NC * XS + 3 * NC * US) * 8;
  static constexpr int LPT = (NC * XS + NT - 1) / NT;
};

template <int P, int T2, int T3, int NC>
__global__ void __launch_bounds__(T2*(T3 / 2)) k_slab3d2(const OpParams op, const double* __restrict__ x,
                                                         double* __restrict__ Z) {
  using Sh = Slab2Shape<P, T2, T3, NC>;
  constexpr int NT = Sh::NT, R = 2 * P + 1, HC = Sh::HC, XS = Sh::XS, US = Sh::US, LPT = Sh::LPT, TC = Sh::TC;
  constexpr int RH = T2 / 2;
  constexpr int WN = 2 * P + 2;
  extern __shared__ __align__(16) double smem[];
  double* xs = smem;               // [NC][HR][HC]
  double* us = smem + NC * XS;     // [3][NC][T2][HC]
  const int m = op.m;
  const int ms = m * m, m3 = ms * m;
  const int s = blockIdx.z;
  const int tid = threadIdx.x;
  const int tr = tid / TC, tc = tid % TC;
  const int r0 = blockIdx.y * T2, q0 = blockIdx.x * T3;
  const int gr = r0 + tr, gc0 = q0 + 2 * tc;
  const bool act0 = gr < m && gc0 < m, act1 = gr < m && gc0 + 1 < m;
  const bool zb0 = act0 && (gc0 < op.zoneL || gc0 >= op.zoneR);
  const bool zb1 = act1 && (gc0 + 1 < op.zoneL || gc0 + 1 >= op.zoneR);
  const bool wzb = __any_sync(0xffffffffu, zb0 || zb1);
  const double* src = x + (size_t)s * ms;
#pragma unroll
  for (int i = 0; i < LPT; ++i) {
    const int idx = tid + i * NT;
    if (idx < NC * XS) {
      const int j = idx / XS, rem = idx % XS;
      const int g1 = r0 - P + rem / HC, g2 = q0 - P + rem % HC;
      const bool ok = g1 >= 0 && g1 < m && g2 >= 0 && g2 < m;
      cp_async8(xs + idx, ok ? src + j * m3 + g1 * m + g2 : x, ok);
    }
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  // ---- stage A: direction 1 (as in k_slab3d)
  for (int it = tid; it < 2 * NC * HC; it += NT) {
    const int a_cc = it % HC, a_j = (it / HC) % NC, a_r0 = (it / (NC * HC)) * RH;
    const double* col = xs + a_j * XS + a_r0 * HC + a_cc;
    double win[RH + 2 * P];
#pragma unroll
    for (int k = 0; k < RH + 2 * P; ++k) win[k] = col[k * HC];
    const int g0 = r0 + a_r0;
    const bool zone_any = g0 < op.zoneL || g0 + RH > op.zoneR;
#pragma unroll
    for (int r = 0; r < RH; ++r) {
      const double xc = win[r + P];
      double vm = op.tM[0] * xc, vs = op.tS[0] * xc, va = 0.0;
#pragma unroll
      for (int o = 1; o <= P; ++o) {
        const double lo = win[r + P - o], hi = win[r + P + o];
        const double sp = lo + hi, sm = hi - lo;
        vm = fma(op.tM[o], sp, vm);
        vs = fma(op.tS[o], sp, vs);
        va = fma(op.tA[o], sm, va);
      }
      if (zone_any) {
        const int g1 = g0 + r;
        if (g1 < m && (g1 < op.zoneL || g1 >= op.zoneR)) {
          const double* rM = op.bM + g1 * R + P;
          const double* rS = op.bS + g1 * R + P;
          const double* rA = op.bA + g1 * R + P;
          vm = vs = va = 0.0;
#pragma unroll
          for (int o = -P; o <= P; ++o) {
            const double v = win[r + P + o];
            vm = fma(__ldg(rM + o), v, vm);
            vs = fma(__ldg(rS + o), v, vs);
            va = fma(__ldg(rA + o), v, va);
          }
        }
      }
      const int uo = (a_r0 + r) * HC + a_cc;
      us[(0 * NC + a_j) * US + uo] = vm;
      us[(1 * NC + a_j) * US + uo] = vs;
      us[(2 * NC + a_j) * US + uo] = va;
    }
  }
  __syncthreads();
  if (!act0) return;
  // ---- stage B: direction 2 for the pair (gc0, gc0 + 1) and the pattern combinations
  double zM[2][NC], zS[2][NC], zA[2][NC];
#pragma unroll
  for (int q = 0; q < 2; ++q)
#pragma unroll
    for (int i = 0; i < NC; ++i) zM[q][i] = zS[q][i] = zA[q][i] = 0.0;
  const int bo = tr * HC + 2 * tc;   // window start: column gc0 - P
#pragma unroll
  for (int j = 0; j < NC; ++j) {
    double wM[WN], wS[WN], wA[WN];
    {
      const double2* pM = reinterpret_cast<const double2*>(us + (0 * NC + j) * US + bo);
      const double2* pS = reinterpret_cast<const double2*>(us + (1 * NC + j) * US + bo);
      const double2* pA = reinterpret_cast<const double2*>(us + (2 * NC + j) * US + bo);
#pragma unroll
      for (int k = 0; k < WN / 2; ++k) {
        const double2 a = pM[k], b = pS[k], c = pA[k];
        wM[2 * k] = a.x; wM[2 * k + 1] = a.y;
        wS[2 * k] = b.x; wS[2 * k + 1] = b.y;
        wA[2 * k] = c.x; wA[2 * k + 1] = c.y;
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const double* uM = wM + P + q;   // centre of point q
      const double* uS = wS + P + q;
      const double* uA = wA + P + q;
      double vMM, vMS, vMA, vSM, vAM, vAA;
      {
        const double c = uM[0];
        double a1 = op.tM[0] * c, a2 = op.tS[0] * c, a3 = 0.0;
#pragma unroll
        for (int o = 1; o <= P; ++o) {
          const double lo = uM[-o], hi = uM[o];
          const double sp = lo + hi, sm = hi - lo;
          a1 = fma(op.tM[o], sp, a1);
          a2 = fma(op.tS[o], sp, a2);
          a3 = fma(op.tA[o], sm, a3);
        }
        vMM = a1; vMS = a2; vMA = a3;
      }
      {
        double a1 = op.tM[0] * uS[0];
#pragma unroll
        for (int o = 1; o <= P; ++o) a1 = fma(op.tM[o], uS[-o] + uS[o], a1);
        vSM = a1;
      }
      {
        const double c = uA[0];
        double a1 = op.tM[0] * c, a3 = 0.0;
#pragma unroll
        for (int o = 1; o <= P; ++o) {
          const double lo = uA[-o], hi = uA[o];
          a1 = fma(op.tM[o], lo + hi, a1);
          a3 = fma(op.tA[o], hi - lo, a3);
        }
        vAM = a1; vAA = a3;
      }
      const bool zb = q == 0 ? zb0 : zb1;
      if (wzb && zb) {
        const int g = gc0 + q;
        const double* rM = op.bM + g * R + P;
        const double* rS = op.bS + g * R + P;
        const double* rA = op.bA + g * R + P;
        vMM = vMS = vMA = vSM = vAM = vAA = 0.0;
#pragma unroll
        for (int o = -P; o <= P; ++o) {
          const double wm = __ldg(rM + o), ws = __ldg(rS + o), wa = __ldg(rA + o);
          vMM = fma(wm, uM[o], vMM);
          vMS = fma(ws, uM[o], vMS);
          vMA = fma(wa, uM[o], vMA);
          vSM = fma(wm, uS[o], vSM);
          vAM = fma(wm, uA[o], vAM);
          vAA = fma(wa, uA[o], vAA);
        }
      }
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        zM[q][i] = fma(op.c.mass[i][j], vMM, zM[q][i]);
        zS[q][i] = fma(op.c.S[0][i][j], vMM, zS[q][i]);
        zM[q][i] = fma(op.c.S[1][i][j], vSM, zM[q][i]);
        zM[q][i] = fma(op.c.S[2][i][j], vMS, zM[q][i]);
        zA[q][i] = fma(op.c.AA[0][i][j], vAM, zA[q][i]);
        zA[q][i] = fma(op.c.AA[1][i][j], vMA, zA[q][i]);
        zM[q][i] = fma(op.c.AA[2][i][j], vAA, zM[q][i]);
      }
    }
  }
  const int pt = s * ms + gr * m + gc0;
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    Z[(size_t)(0 * NC + i) * m3 + pt] = zM[0][i];
    Z[(size_t)(1 * NC + i) * m3 + pt] = zS[0][i];
    Z[(size_t)(2 * NC + i) * m3 + pt] = zA[0][i];
    if (act1) {
      Z[(size_t)(0 * NC + i) * m3 + pt + 1] = zM[1][i];
      Z[(size_t)(1 * NC + i) * m3 + pt + 1] = zS[1][i];
      Z[(size_t)(2 * NC + i) * m3 + pt + 1] = zA[1][i];
    }
  }
}

// (C): thread per (i2, i3) column; march s over the chunk; epilogue as in the fused kernels
template <int P, int NC>
__global__ void __launch_bounds__(256) k_col3d(const OpParams op, const Epi ep, int mode, int dot,
                                               const double* __restrict__ Z, const double* __restrict__ x,
                                               double* __restrict__ y, int chunk) {
  constexpr int R = 2 * P + 1;
  __shared__ double red[8];
  const int m = op.m;
  const int ms = m * m, m3 = ms * m;
  const int col = blockIdx.x * blockDim.x + threadIdx.x;
  const bool active = col < ms;
  const int gr = active ? col / m : 0, gc = active ? col % m : 0;
  const int c0 = blockIdx.y * chunk;
  const int c1 = min(c0 + chunk, m);
  const int sb = max(0, c0 - P);
  const int se = c1 + P;
  double acc[NC][R];
#pragma unroll
  for (int i = 0; i < NC; ++i)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[i][r] = 0.0;
  double dsum = 0.0;
  double M1 = 1.0, S1 = 0.0, M2 = 1.0, S2 = 0.0;
  if (mode >= EPI_JACOBI && active) {
    M1 = __ldg(op.bM + gr * R + P); S1 = __ldg(op.bS + gr * R + P);
    M2 = __ldg(op.bM + gc * R + P); S2 = __ldg(op.bS + gc * R + P);
  }
  // software pipeline: z of slab s+1 is loaded while slab s is scattered
  double zn[3][NC];
  auto loadz = [&](int s) {
#pragma unroll
    for (int f = 0; f < 3; ++f)
#pragma unroll
      for (int i = 0; i < NC; ++i)
        zn[f][i] = (active && s < m) ? __ldg(Z + (size_t)(f * NC + i) * m3 + (size_t)s * ms + col) : 0.0;
  };
  loadz(sb);
#pragma unroll 1
  for (int s = sb; s < se; ++s) {
    double z[3][NC];
#pragma unroll
    for (int f = 0; f < 3; ++f)
#pragma unroll
      for (int i = 0; i < NC; ++i) z[f][i] = zn[f][i];
    if (s + 1 < se) loadz(s + 1);
    if (s < m) {
      if (s - P >= op.zoneL && s + P < op.zoneR) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int d = P - r;
          const int ad = d < 0 ? -d : d;
          const double wM = op.tM[ad], wS = op.tS[ad], wA = d >= 0 ? op.tA[ad] : -op.tA[ad];
#pragma unroll
          for (int i = 0; i < NC; ++i) acc[i][r] = fma(wM, z[0][i], fma(wS, z[1][i], fma(wA, z[2][i], acc[i][r])));
        }
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int t = s - P + r;
          double wM = 0.0, wS = 0.0, wA = 0.0;
          if (t >= 0 && t < m) {
            const int k = t * R + (s - t) + P;   // F[t][s]
            wM = __ldg(op.bM + k); wS = __ldg(op.bS + k); wA = __ldg(op.bA + k);
          }
#pragma unroll
          for (int i = 0; i < NC; ++i) acc[i][r] = fma(wM, z[0][i], fma(wS, z[1][i], fma(wA, z[2][i], acc[i][r])));
        }
      }
    }
    const int t = s - P;
    if (t >= c0 && t < c1 && active) {
      const int pt = t * ms + col;
      double Dv[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) Dv[i] = 1.0;
      if (mode >= EPI_JACOBI) {
        const double M0 = __ldg(op.bM + t * R + P), S0 = __ldg(op.bS + t * R + P);
#pragma unroll
        for (int i = 0; i < NC; ++i)
          Dv[i] = op.c.mass[i][i] * M0 * M1 * M2 + op.c.S[0][i][i] * S0 * M1 * M2 +
                  op.c.S[1][i][i] * M0 * S1 * M2 + op.c.S[2][i][i] * M0 * M1 * S2;
      }
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const double a = acc[i][0];
        const int gi = i * m3 + pt;
        double out;
        if (mode == EPI_APPLY) out = a;
        else if (mode == EPI_RESID) out = ep.b[gi] - a;
        else if (mode == EPI_JACOBI) out = x[gi] + ep.omega * (ep.b[gi] - a) / Dv[i];
        else out = a / Dv[i];
        y[gi] = out;
        if (dot == DOT_X_OUT) dsum = fma(x[gi], out, dsum);
        else if (dot == DOT_OUT_OUT) dsum = fma(out, out, dsum);
      }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
#pragma unroll
      for (int r = 0; r < R - 1; ++r) acc[i][r] = acc[i][r + 1];
      acc[i][R - 1] = 0.0;
    }
  }
  if (dot != DOT_NONE) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, off);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = dsum;
    __syncthreads();
    if (threadIdx.x == 0) {
      double sacc = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sacc += red[w];
      ep.partial[blockIdx.y * gridDim.x + blockIdx.x] = sacc;
    }
  }
}

// ---------------------------------------------------------------------------------------
// launch configuration
// ---------------------------------------------------------------------------------------
constexpr int NT2D = 128;
constexpr int T2_3D = 8, T3_3D = 32;      // k_op3d: one output point per thread
constexpr int T2_3D2 = 8, T3_3D2 = 64;    // k_op3d2: two output points per thread
constexpr int TARGET_CTAS = 4 * 148;

static int split3d_mode() {   // IGACD_SPLIT: 0 fused only, 1 split for the vector system, 2 split for both
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_SPLIT");
    v = (e && e[0] == '0') ? 0 : (e && e[0] == '2') ? 2 : 1;
  }
  return v;
}

// 3D operator as slab kernel + column kernel, or the fused marching kernel
static bool use_split(int dim, int nc) {
  const int v = split3d_mode();
  return dim == 3 && (v == 2 || (v == 1 && nc == 3));
}

static int col_chunks(int m) {   // direction-0 chunks of the column kernel: >= ~4 CTAs per SM
  const int cb = (m * m + 255) / 256;
  int nch = std::max(1, std::min(m, (4 * 148 + cb - 1) / cb));
  const int chunk = std::max(std::min(m, 4), (m + nch - 1) / nch);
  return chunk;
}

static int k3_variant() {   // 1: one point per thread (default), 2: two points per thread
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_K3");
    v = (e && e[0] == '2') ? 2 : 1;
  }
  return v;
}

struct Grid {
  dim3 grid;
  int chunk;
};

static Grid grid_for(const Handle& h, int level) {
  const int m = h.lv[level].m;
  Grid g;
  if (h.dim == 2) {
    const int tx = (m + NT2D - 1) / NT2D;
    int nch = std::max(1, std::min(m, (TARGET_CTAS + tx - 1) / tx));
    g.chunk = (m + nch - 1) / nch;
    g.chunk = std::max(g.chunk, std::min(m, 2));
    nch = (m + g.chunk - 1) / g.chunk;
    g.grid = dim3(tx, nch, 1);
  } else {
    const int T3 = k3_variant() == 2 ? T3_3D2 : T3_3D, T2 = k3_variant() == 2 ? T2_3D2 : T2_3D;
    const int target = k3_variant() == 2 ? 2 * 148 : TARGET_CTAS;
    const int tx = (m + T3 - 1) / T3, ty = (m + T2 - 1) / T2;
    int nch = std::max(1, std::min(m, (target + tx * ty - 1) / (tx * ty)));
    g.chunk = (m + nch - 1) / nch;   // small levels: short chunks (latency), large: ~4 CTAs per SM
    g.chunk = std::max(g.chunk, std::min(m, 2));
    nch = (m + g.chunk - 1) / g.chunk;
    g.grid = dim3(tx, ty, nch);
  }
  return g;
}

int operator_ctas(const Handle& h, int level) {
  return std::max(operator_ctas_sys(h, level, 1), operator_ctas_sys(h, level, 3));
}

int operator_ctas_sys(const Handle& h, int level, int nc) {
  if (use_split(h.dim, nc)) {
    const int m = h.lv[level].m;
    const int chunk = col_chunks(m);
    return ((m * m + 255) / 256) * ((m + chunk - 1) / chunk);
  }
  Grid g = grid_for(h, level);
  return g.grid.x * g.grid.y * g.grid.z;
}

static int slab_variant() {   // IGACD_SLAB: 1 one point per thread (default), 2 two points per thread
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_SLAB");
    v = (e && e[0] == '2') ? 2 : 1;
  }
  return v;
}

constexpr int T2_SL2 = 16, T3_SL2 = 32;

template <int P, int NC>
static void launch_split3d(const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                           double* Z, cudaStream_t s) {
  const int m = op.m;
  if (slab_variant() == 2) {
    using Sh = Slab2Shape<P, T2_SL2, T3_SL2, NC>;
    static bool attr2 = false;
    if (!attr2) {
      IGACD_CUDA(cudaFuncSetAttribute(k_slab3d2<P, T2_SL2, T3_SL2, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      Sh::SMEM));
      attr2 = true;
    }
    k_slab3d2<P, T2_SL2, T3_SL2, NC><<<dim3((m + T3_SL2 - 1) / T3_SL2, (m + T2_SL2 - 1) / T2_SL2, m), Sh::NT, Sh::SMEM,
                                       s>>>(op, x, Z);
  } else {
    using Sh = SlabShape<P, 8, 32, NC>;
    static bool attr = false;
    if (!attr) {
      IGACD_CUDA(cudaFuncSetAttribute(k_slab3d<P, 8, 32, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sh::SMEM));
      attr = true;
    }
    k_slab3d<P, 8, 32, NC><<<dim3((m + 31) / 32, (m + 7) / 8, m), Sh::NT, Sh::SMEM, s>>>(op, x, Z);
  }
  const int chunk = col_chunks(m);
  k_col3d<P, NC><<<dim3((m * m + 255) / 256, (m + chunk - 1) / chunk), 256, 0, s>>>(op, ep, mode, dot, Z, x, y,
                                                                                 chunk);
}

template <int P, int NC>
static void launch2d(const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                     cudaStream_t s) {
  k_op2d<P, NT2D, NC><<<g.grid, NT2D, 0, s>>>(op, ep, mode, dot, x, y, g.chunk);
}

static int minb_choice() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_MINB");
    v = (e && e[0] == '1') ? 1 : 2;
  }
  return v;
}

// TMA slab loads are opt-in (IGACD_TMA=1): ~5% faster on config 4, but a launch with
// p = 1, m = 44 faulted in round 1 and the cause is not yet understood.
static bool tma_allowed() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_TMA");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    IGACD_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw Error{IGACD_E_CUDA, "cuTensorMapEncodeTiled unavailable"};
    fn = (EncodeTiledFn)p;
  }
  return fn;
}

// 4D view (i3, i2, i1, component) of a [nc][m][m][m] vector, box (HC, HR, 1, nc); cached per pointer
static const CUtensorMap& tensor_map(const double* x, int m, int nc, int hc, int hr) {
  static std::mutex mu;
  static std::map<std::tuple<const double*, int, int, int, int>, CUtensorMap> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_tuple(x, m, nc, hc, hr);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  if (cache.size() > 256) cache.clear();
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)m, (cuuint64_t)m, (cuuint64_t)m, (cuuint64_t)nc};
  const cuuint64_t strides[3] = {(cuuint64_t)m * 8, (cuuint64_t)m * m * 8, (cuuint64_t)m * m * m * 8};
  const cuuint32_t box[4] = {(cuuint32_t)hc, (cuuint32_t)hr, 1, (cuuint32_t)nc};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, (void*)x, dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error{IGACD_E_CUDA, "cuTensorMapEncodeTiled failed"};
  return cache.emplace(key, map).first->second;
}

template <int P, int NC, int MINB, bool TMA>
static void launch3d_m(const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                       cudaStream_t s) {
  using Sh = Op3dShape<P, T2_3D, T3_3D, NC>;
  static bool attr = false;
  if (!attr) {
    IGACD_CUDA(cudaFuncSetAttribute(k_op3d<P, T2_3D, T3_3D, NC, MINB, TMA>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, Sh::SMEM));
    attr = true;
  }
  CUtensorMap map;
  if (TMA) map = tensor_map(x, op.m, NC, Sh::HC, Sh::HR);
  else std::memset(&map, 0, sizeof(map));
  k_op3d<P, T2_3D, T3_3D, NC, MINB, TMA><<<g.grid, Sh::NT, Sh::SMEM, s>>>(op, ep, mode, dot, x, y, g.chunk, map);
}

template <int P, int NC, bool TMA>
static void launch3d2_m(const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x,
                        double* y, cudaStream_t s) {
  using Sh = Op3d2Shape<P, T2_3D2, T3_3D2, NC>;
  static bool attr = false;
  if (!attr) {
    IGACD_CUDA(cudaFuncSetAttribute(k_op3d2<P, T2_3D2, T3_3D2, NC, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Sh::SMEM));
    attr = true;
  }
  CUtensorMap map;
  if (TMA) map = tensor_map(x, op.m, NC, Sh::HC, Sh::HR);
  else std::memset(&map, 0, sizeof(map));
  k_op3d2<P, T2_3D2, T3_3D2, NC, TMA><<<g.grid, Sh::NT, Sh::SMEM, s>>>(op, ep, mode, dot, x, y, g.chunk, map);
}

template <int P, int NC>
static void launch3d(const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                     cudaStream_t s) {
  if (k3_variant() == 2) {
    using Sh2 = Op3d2Shape<P, T2_3D2, T3_3D2, NC>;
    const bool tma2 = tma_allowed() && op.m % 2 == 0 && ((uintptr_t)x % 16) == 0 && op.m >= Sh2::HC &&
                      op.m >= Sh2::HR;
    if (tma2) launch3d2_m<P, NC, true>(g, op, ep, mode, dot, x, y, s);
    else launch3d2_m<P, NC, false>(g, op, ep, mode, dot, x, y, s);
    return;
  }
  // TMA needs 16-byte aligned global strides (m even) and a 16-byte aligned base
  using Sh = Op3dShape<P, T2_3D, T3_3D, NC>;
  const bool tma = tma_allowed() && op.m % 2 == 0 && ((uintptr_t)x % 16) == 0 && op.m >= Sh::HC && op.m >= Sh::HR;
  if (minb_choice() == 1) {
    if (tma) launch3d_m<P, NC, 1, true>(g, op, ep, mode, dot, x, y, s);
    else launch3d_m<P, NC, 1, false>(g, op, ep, mode, dot, x, y, s);
  } else {
    if (tma) launch3d_m<P, NC, 2, true>(g, op, ep, mode, dot, x, y, s);
    else launch3d_m<P, NC, 2, false>(g, op, ep, mode, dot, x, y, s);
  }
}

template <int P>
static void dispatch(int dim, int nc, const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot,
                     const double* x, double* y, double* Z, cudaStream_t s) {
  if (use_split(dim, nc)) {
    if (nc == 1) launch_split3d<P, 1>(op, ep, mode, dot, x, y, Z, s);
    else launch_split3d<P, 3>(op, ep, mode, dot, x, y, Z, s);
    return;
  }
  if (dim == 2) {
    if (nc == 1) launch2d<P, 1>(g, op, ep, mode, dot, x, y, s);
    else launch2d<P, 2>(g, op, ep, mode, dot, x, y, s);
  } else {
    if (nc == 1) launch3d<P, 1>(g, op, ep, mode, dot, x, y, s);
    else launch3d<P, 3>(g, op, ep, mode, dot, x, y, s);
  }
}

int launch_operator(Handle& h, int sy, int level, const double* x, double* out, EpiMode mode, DotMode dot,
                    const Epi& epi, cudaStream_t s) {
  const System& S = h.sys[sy];
  const OpParams& op = S.lv[level].op;
  Grid g = grid_for(h, level);
  const int nct = operator_ctas_sys(h, level, S.nc);
  if (dot != DOT_NONE && (size_t)nct > h.partial_len) throw Error{IGACD_E_ARG, "partial buffer too small"};
  switch (h.p) {
    case 1: dispatch<1>(h.dim, S.nc, g, op, epi, mode, dot, x, out, h.zbuf, s); break;
    case 2: dispatch<2>(h.dim, S.nc, g, op, epi, mode, dot, x, out, h.zbuf, s); break;
    case 3: dispatch<3>(h.dim, S.nc, g, op, epi, mode, dot, x, out, h.zbuf, s); break;
    case 4: dispatch<4>(h.dim, S.nc, g, op, epi, mode, dot, x, out, h.zbuf, s); break;
    case 5: dispatch<5>(h.dim, S.nc, g, op, epi, mode, dot, x, out, h.zbuf, s); break;
    case 6: dispatch<6>(h.dim, S.nc, g, op, epi, mode, dot, x, out, h.zbuf, s); break;
    default: throw Error{IGACD_E_ARG, "degree out of range"};
  }
  IGACD_LAUNCH_CHECK();
  count_launch(h);
  if (use_split(h.dim, S.nc)) count_launch(h);
  return dot != DOT_NONE ? nct : 0;
}

}  // namespace igacd

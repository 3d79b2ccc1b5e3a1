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
#include <algorithm>
#include <cstdlib>
#include <cstring>

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
  static constexpr int NT = (T2 * T3 + 31) / 32 * 32;   // full warps (T3 need not divide 32)
  static constexpr int R = 2 * P + 1;
  static constexpr int HR = T2 + 2 * P;
  static constexpr int HC = T3 + 2 * P;
  static constexpr int XS = HR * HC;        // one component of one slab tile
  static constexpr int US = T2 * HC;        // one stage-A output array
  static constexpr int XB = (NC * XS + 15) / 16 * 16;  // one slab buffer, padded to 128 bytes
  static constexpr int SMEM = (2 * XB + 3 * NC * US + 2 * 3 * R) * 8 + (NT / 32) * 8;
  static constexpr int LPT = (NC * XS + NT - 1) / NT;
};

template <int P, int T2, int T3, int NC, int MINB>
__global__ void __launch_bounds__(Op3dShape<P, T2, T3, NC>::NT, MINB) k_op3d(const OpParams op, const Epi ep, int mode, int dot,
                                                    const double* __restrict__ x, double* __restrict__ y,
                                                    int chunk) {
  using Sh = Op3dShape<P, T2, T3, NC>;
  constexpr int NT = Sh::NT, R = Sh::R, HR = Sh::HR, HC = Sh::HC, XS = Sh::XS, US = Sh::US, LPT = Sh::LPT;
  constexpr int XB = Sh::XB;
  static_assert(LPT <= 32, "prefetch mask");
  extern __shared__ __align__(16) double smem[];
  double* xs = smem;                   // [2][XB]: [NC][HR][HC] each
  double* us = smem + 2 * XB;          // [3][NC][T2][HC]: index (F*NC + j), F: 0 M, 1 S, 2 A
  double* wts = us + 3 * NC * US;      // [2][3R]
  double* red = wts + 2 * 3 * R;
  const int m = op.m;
  const int ms = m * m;                // ndof < 2^31 is checked on the host
  const int m3 = ms * m;
  const int tid = threadIdx.x;
  const bool real = tid < T2 * T3;   // padding threads of the last warp own no point
  const int tr = real ? tid / T3 : T2 - 1, tc = real ? tid % T3 : 0;
  const int r0 = blockIdx.y * T2, q0 = blockIdx.x * T3;
  const int gr = r0 + tr, gc = q0 + tc;
  const bool active = real && gr < m && gc < m;
  const bool zoneB = active && (gc < op.zoneL || gc >= op.zoneR);
  const int c0 = blockIdx.z * chunk;
  const int c1 = min(c0 + chunk, m);
  const int sb = max(0, c0 - P);
  const int se = c1 + P;

  // ---- slab-invariant per-thread offsets -------------------------------------------------
  int goff[LPT];             // global offset (without the slab term) of each prefetch slot
  unsigned vmask = 0u;       // slot is inside the domain (in-plane)
#pragma unroll
  for (int i = 0; i < LPT; ++i) {
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
  // stage A work item: (row segment, component, halo column), lanes along columns; each
  // item marches down its RH = T2/RS output rows with a register window of RH + 2P inputs.
  // The scalar system splits the rows in 4 (160 items for 256 threads instead of 80: the
  // barrier after stage A was the top stall), the vector system in 2.
  constexpr int RS = NC == 1 ? 4 : 2;
  constexpr int RH = T2 / RS;
  static_assert(T2 % RS == 0, "row segments");
  constexpr int NITEMS = RS * NC * HC;
  const bool wzb = __any_sync(0xffffffffu, zoneB);
  const int bo = tr * HC + tc + P;     // stage-B window centre
  const int pto = gr * m + gc;         // in-slab output offset

  double acc[NC][R];
#pragma unroll
  for (int i = 0; i < NC; ++i)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[i][r] = 0.0;
  double dsum = 0.0;

  // slab s -> xs[buf]: per-thread cp.async copies (out-of-domain elements zero-filled)
  auto prefetch = [&](int s, int buf) {
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

  prefetch(sb, 0);
  load_col_weights<P>(op, sb, c0, c1, wts);
  cp_async_wait_all();
  __syncthreads();
#pragma unroll 1
  for (int s = sb; s < se; ++s) {
    const int buf = (s - sb) & 1;
    const bool more = s + 1 < se;
    if (more) {
      prefetch(s + 1, buf ^ 1);
      load_col_weights<P>(op, s + 1, c0, c1, wts + (buf ^ 1) * 3 * R);
    }
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
      ep.partial[(blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x] = sacc;
    }
  }
}

template <int P, int T2, int T3, int NC>
struct SlabShape {
  static constexpr int NT = (T2 * T3 + 31) / 32 * 32;   // full warps (T3 need not divide 32)
  static constexpr int HR = T2 + 2 * P;
  static constexpr int HC = T3 + 2 * P;
  static constexpr int XS = HR * HC;
  static constexpr int US = T2 * HC;
  static constexpr int SMEM = (NC * XS + 3 * NC * US) * 8;
  static constexpr int LPT = (NC * XS + NT - 1) / NT;
};

template <int P, int T2, int T3, int NC>
__global__ void __launch_bounds__(SlabShape<P, T2, T3, NC>::NT) k_slab3d(const OpParams op, const double* __restrict__ x,
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
  const bool real = tid < T2 * T3;   // padding threads of the last warp own no point
  const int tr = real ? tid / T3 : T2 - 1, tc = real ? tid % T3 : 0;
  const int r0 = blockIdx.y * T2, q0 = blockIdx.x * T3;
  const int gr = r0 + tr, gc = q0 + tc;
  const bool active = real && gr < m && gc < m;
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
constexpr int T2_3D = 8;                  // tile rows (direction 1) of the 3D kernels

// tile columns (direction 2) of the 3D kernels: 32, or 27 when that wastes fewer columns
// (m = 162: 6 x 27 = 162 exactly instead of 6 x 32 = 192)
static int t3_for(int m) {
  const int w32 = (m + 31) / 32 * 32, w27 = (m + 26) / 27 * 27;
  return w27 < w32 ? 27 : 32;
}
constexpr int TARGET_CTAS = 4 * 148;

// 3D vector system: slab kernel + column kernel (measured 1.4x faster than the fused
// marching kernel for nc = 3); the scalar system (nc = 1) uses the fused kernel.
// IGACD_SPLIT=0 runs the fused kernel for both (comparison only).
static bool use_split(int dim, int nc) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_SPLIT");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return dim == 3 && v == 1 && nc == 3;
}

static int col_chunks(int m) {   // direction-0 chunks of the column kernel: >= ~4 CTAs per SM
  const int cb = (m * m + 255) / 256;
  int nch = std::max(1, std::min(m, (4 * 148 + cb - 1) / cb));
  const int chunk = std::max(std::min(m, 4), (m + nch - 1) / nch);
  return chunk;
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
    const int T3 = t3_for(m);
    const int tx = (m + T3 - 1) / T3, ty = (m + T2_3D - 1) / T2_3D;
    int nch = std::max(1, std::min(m, (TARGET_CTAS + tx * ty - 1) / (tx * ty)));
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

template <int P, int NC, int T3>
static void launch_split3d_t(const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                             double* Z, cudaStream_t s) {
  const int m = op.m;
  using Sh = SlabShape<P, 8, T3, NC>;
  static bool attr = false;
  if (!attr) {
    IGACD_CUDA(cudaFuncSetAttribute(k_slab3d<P, 8, T3, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, Sh::SMEM));
    attr = true;
  }
  k_slab3d<P, 8, T3, NC><<<dim3((m + T3 - 1) / T3, (m + 7) / 8, m), Sh::NT, Sh::SMEM, s>>>(op, x, Z);
  const int chunk = col_chunks(m);
  k_col3d<P, NC><<<dim3((m * m + 255) / 256, (m + chunk - 1) / chunk), 256, 0, s>>>(op, ep, mode, dot, Z, x, y,
                                                                                 chunk);
}

template <int P, int NC>
static void launch_split3d(const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                           double* Z, cudaStream_t s) {
  if (t3_for(op.m) == 27) launch_split3d_t<P, NC, 27>(op, ep, mode, dot, x, y, Z, s);
  else launch_split3d_t<P, NC, 32>(op, ep, mode, dot, x, y, Z, s);
}

template <int P, int NC>
static void launch2d(const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                     cudaStream_t s) {
  k_op2d<P, NT2D, NC><<<g.grid, NT2D, 0, s>>>(op, ep, mode, dot, x, y, g.chunk);
}

template <int P, int NC, int T3>
static void launch3d_t(const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x,
                       double* y, cudaStream_t s) {
  using Sh = Op3dShape<P, T2_3D, T3, NC>;
  static bool attr = false;
  if (!attr) {
    IGACD_CUDA(cudaFuncSetAttribute(k_op3d<P, T2_3D, T3, NC, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    Sh::SMEM));
    attr = true;
  }
  k_op3d<P, T2_3D, T3, NC, 2><<<g.grid, Sh::NT, Sh::SMEM, s>>>(op, ep, mode, dot, x, y, g.chunk);
}

template <int P, int NC>
static void launch3d(const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                     cudaStream_t s) {
  if (t3_for(op.m) == 27) launch3d_t<P, NC, 27>(g, op, ep, mode, dot, x, y, s);
  else launch3d_t<P, NC, 32>(g, op, ep, mode, dot, x, y, s);
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
  if (use_split(h.dim, S.nc)) count_launch(h);   // slab + column kernels
  return dot != DOT_NONE ? nct : 0;
}

}  // namespace igacd

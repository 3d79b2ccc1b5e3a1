// R2 in 3D: the round-1 split form of the operator.  It serves the levels on which the
// marching kernel of apply3d.cu does not pay: too few output slabs per CTA for its 2p warm-up
// slabs (every level but the largest ones), and the vector system's odd-m levels (no TMA)
// (DESIGN.md "Kernels").  Each system has its own z workspace (the additive preconditioner runs
// the two systems concurrently):
//   k_slab3d  one CTA per (in-slab tile, slab): directions 1 and 2 from shared memory and the
//             9 per-point combinations z_{i,F0} written to global memory (zbuf);
//   k_col3d   one thread per (direction-1, direction-2) column: the direction-0 band scatter into
//             a register ring of 2p+1 output slabs per component, then the epilogue.
// Same Kronecker patterns and Toeplitz/boundary-zone handling as apply3d.cu (eq:matr_Amu3D,
// PAPER.md:515-543; boundary rows PAPER.md:347-354).  IGACD_SPLIT=1 forces it on every level.
#include <algorithm>
#include <cstdlib>

#include "internal.cuh"

namespace igacd {
namespace {

__device__ __forceinline__ void sp_cp8(double* smem_dst, const double* gsrc, bool valid) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int nbytes = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr), "l"(gsrc), "r"(nbytes) : "memory");
}
__device__ __forceinline__ void sp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void sp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

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
      sp_cp8(xs + idx, ok ? src + j * m3 + g1 * m + g2 : x, ok);
    }
  }
  sp_commit();
  sp_wait_all();
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
          {
            const bool in = t >= 0 && t < m;
            const int tc = in ? t : s;                        // clamped row: the address is always in range
            const int k = tc * R + (s - tc) + P;             // F[t][s]
            const double sel = in ? 1.0 : 0.0;
            wM = sel * __ldg(op.bM + k); wS = sel * __ldg(op.bS + k); wA = sel * __ldg(op.bA + k);
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

// direction-0 chunks of the column kernel: >= ~4 CTAs per SM
int col_chunk(int m) {
  const int cb = (m * m + 255) / 256;
  int nch = std::max(1, std::min(m, (4 * num_sms() + cb - 1) / cb));
  return std::max(std::min(m, 4), (m + nch - 1) / nch);
}

int t3_split(int m) {   // 27 columns when that wastes fewer than 32 (m = 162: 6 x 27)
  const int w32 = (m + 31) / 32 * 32, w27 = (m + 26) / 27 * 27;
  return w27 < w32 ? 27 : 32;
}

template <int P, int NC, int T3>
void launch_split_t(const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y, double* Z,
                    cudaStream_t s) {
  const int m = op.m;
  using Sh = SlabShape<P, 8, T3, NC>;
  ensure_smem_attr((const void*)k_slab3d<P, 8, T3, NC>, Sh::SMEM);
  k_slab3d<P, 8, T3, NC><<<dim3((m + T3 - 1) / T3, (m + 7) / 8, m), Sh::NT, Sh::SMEM, s>>>(op, x, Z);
  const int chunk = col_chunk(m);
  k_col3d<P, NC><<<dim3((m * m + 255) / 256, (m + chunk - 1) / chunk), 256, 0, s>>>(op, ep, mode, dot, Z, x, y,
                                                                                 chunk);
}

template <int P>
void launch_split_p(int nc, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                    double* Z, cudaStream_t s) {
  if (nc == 1) {
    if (t3_split(op.m) == 27) launch_split_t<P, 1, 27>(op, ep, mode, dot, x, y, Z, s);
    else launch_split_t<P, 1, 32>(op, ep, mode, dot, x, y, Z, s);
  } else {
    if (t3_split(op.m) == 27) launch_split_t<P, 3, 27>(op, ep, mode, dot, x, y, Z, s);
    else launch_split_t<P, 3, 32>(op, ep, mode, dot, x, y, Z, s);
  }
}

}  // namespace

bool split3d_forced() {
  static const int v = [] {
    const char* e = getenv("IGACD_SPLIT");   // IGACD_SPLIT=1: the round-1 split form on every level
    return (e && e[0] == '1') ? 1 : 0;
  }();
  return v == 1;
}

int split3d_ctas(int m) {
  const int chunk = col_chunk(m);
  return ((m * m + 255) / 256) * ((m + chunk - 1) / chunk);
}

void launch_split3d(int p, int nc, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                    double* Z, cudaStream_t s) {
  switch (p) {
    case 1: launch_split_p<1>(nc, op, ep, mode, dot, x, y, Z, s); break;
    case 2: launch_split_p<2>(nc, op, ep, mode, dot, x, y, Z, s); break;
    case 3: launch_split_p<3>(nc, op, ep, mode, dot, x, y, Z, s); break;
    case 4: launch_split_p<4>(nc, op, ep, mode, dot, x, y, Z, s); break;
    case 5: launch_split_p<5>(nc, op, ep, mode, dot, x, y, Z, s); break;
    case 6: launch_split_p<6>(nc, op, ep, mode, dot, x, y, Z, s); break;
    default: throw Error{IGACD_E_ARG, "degree out of range"};
  }
}

}  // namespace igacd

// R2: matrix-free operator y = A x by sum factorisation, fused epilogues (R4 smoother,
// residual, D^-1 A, dot products).  This file: the 2D kernel and the launch front end;
// the 3D kernel is in apply3d.cu.
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
// launch configuration
// ---------------------------------------------------------------------------------------
constexpr int NT2D = 128;
constexpr int TARGET_CTAS = 4 * 148;

struct Grid {
  dim3 grid;
  int chunk;
};

static Grid grid_for(const Handle& h, int level, int nc) {
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
    g.grid = dim3(1, 1, 1);   // 3D grids are planned by the kernels' own launchers
    g.chunk = 0;
  }
  return g;
}

// 3D paths: the persistent marching kernel (apply3d.cu; TMA staging on even-m levels, cp.async
// on odd-m ones) for the scalar system and for the large even-m levels of the vector system;
// the vector system's odd-m levels and the levels too small for marching to pay take the split
// slab + column kernels (split3d.cu)
static bool use_split(const Handle& h, int nc, int m) {
  if (h.dim != 3 || !(nc == 3 ? h.zbuf : h.zbuf1)) return false;
  if (split3d_forced() || !apply3d_marching_pays(m)) return true;
  return nc == 3 && m % 2 == 1;   // the cp.async marching kernel measured slower than the split form here
}

int operator_ctas_sys(const Handle& h, int level, int nc) {
  const int m = h.lv[level].m;
  if (h.dim == 3) {   // upper bound over the paths a launch may take
    int n = apply3d_ctas(h.p, nc, m);
    n = std::max(n, split3d_ctas(m));
    return n;
  }
  Grid g = grid_for(h, level, nc);
  return g.grid.x * g.grid.y * g.grid.z;
}

int operator_ctas(const Handle& h, int level) {
  return std::max(operator_ctas_sys(h, level, 1), operator_ctas_sys(h, level, h.dim));
}

template <int P, int NC>
static void launch2d(const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                     cudaStream_t s) {
  k_op2d<P, NT2D, NC><<<g.grid, NT2D, 0, s>>>(op, ep, mode, dot, x, y, g.chunk);
}

template <int P>
static void dispatch2d(int nc, const Grid& g, const OpParams& op, const Epi& ep, int mode, int dot, const double* x,
                       double* y, cudaStream_t s) {
  if (nc == 1) launch2d<P, 1>(g, op, ep, mode, dot, x, y, s);
  else launch2d<P, 2>(g, op, ep, mode, dot, x, y, s);
}

int launch_operator(Handle& h, int sy, int level, const double* x, double* out, EpiMode mode, DotMode dot,
                    const Epi& epi, cudaStream_t s) {
  const System& S = h.sys[sy];
  const OpParams& op = S.lv[level].op;
  Grid g = grid_for(h, level, S.nc);
  int nct = operator_ctas_sys(h, level, S.nc);
  if (dot != DOT_NONE && (size_t)nct > h.partial_len) throw Error{IGACD_E_ARG, "partial buffer too small"};
  if (use_split(h, S.nc, op.m)) {
    launch_split3d(h.p, S.nc, op, epi, mode, dot, x, out, S.nc == 3 ? h.zbuf : h.zbuf1, s);
    nct = split3d_ctas(op.m);
    count_launch(h);   // slab + column kernels
  } else if (h.dim == 3) {
    nct = launch_apply3d(h.p, S.nc, op, epi, mode, dot, x, out, s, h.slot_share);
  } else {
    switch (h.p) {
      case 1: dispatch2d<1>(S.nc, g, op, epi, mode, dot, x, out, s); break;
      case 2: dispatch2d<2>(S.nc, g, op, epi, mode, dot, x, out, s); break;
      case 3: dispatch2d<3>(S.nc, g, op, epi, mode, dot, x, out, s); break;
      case 4: dispatch2d<4>(S.nc, g, op, epi, mode, dot, x, out, s); break;
      case 5: dispatch2d<5>(S.nc, g, op, epi, mode, dot, x, out, s); break;
      case 6: dispatch2d<6>(S.nc, g, op, epi, mode, dot, x, out, s); break;
      default: throw Error{IGACD_E_ARG, "degree out of range"};
    }
  }
  IGACD_LAUNCH_CHECK();
  count_launch(h);
  return dot != DOT_NONE ? nct : 0;
}

}  // namespace igacd

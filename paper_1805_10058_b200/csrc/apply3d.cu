// R2 in 3D: matrix-free operator y = A x (vector system nc = 3, auxiliary scalar system
// nc = 1) by sum factorisation in ONE persistent kernel per apply, with fused epilogues (R4
// smoother, residual, D^-1 A, dot products).
//
// The Galerkin matrix is sum_P C_P (x) F0_P (x) F1_P (x) F2_P with 1D factors M, A, S
// (eq:matr_Amu3D PAPER.md:515-543; the L_A form of reading R1 has the same Kronecker
// patterns, internal.cuh Coef).  The (direction 1, direction 2) plane is cut into T1 x T2
// tiles; a work unit is (tile, output slab along direction 0).  The host lays the units on a
// line, weighted by the measured cost of their tile class, and cuts it into G pieces of equal
// cost (m3_schedule); CTA b of the persistent grid marches the slabs of its piece tile by tile
// ("segments"; each one pays 2p warm-up slabs).  Per slab s of a segment:
//   * the slab tile with its p-halo, all components, arrives in shared memory by TMA
//     (cp.async.bulk.tensor, out-of-domain elements zero-filled by the tensor map) into one of
//     two buffers, each completing on its own mbarrier; levels whose row pitch is not 16-byte
//     aligned (odd m) stage the tile with 8-byte cp.async instead;
//   * pass A contracts direction 1 (M, S, A of every halo column; a register window down the
//     rows, lanes along the columns) into a double-buffered shared array u;
//   * pass B (one thread per point) contracts direction 2 from u and forms the per-point
//     combinations z_{i,F0};
//   * pass C scatters F0[t][s] z(s) into a register ring of 2p+1 output slabs per component;
//     slab t = s-p is then final and leaves through the epilogue.
// Pass A of slab s+1 and passes B/C of slab s run in the same phase: ONE barrier per slab, and
// the intermediate z never leaves the registers (the round-1 split form wrote and re-read 9
// doubles per point through HBM).
// Interior rows of every 1D factor are Toeplitz: contractions use register
// weights with symmetric pairing (one add feeds M and S, one subtract feeds A).  Warps that
// hold a boundary-zone column take the direction-2 weights of their columns from a per-tile
// shared table instead; boundary-zone rows (pass A) and slabs (pass C) read the band rows,
// which are uniform over the warp.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <cstdio>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.cuh"

namespace igacd {

// ---- async-copy primitives ------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp8(double* smem_dst, const double* gsrc, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
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
// 4D tile {c2, c1, s, comp} of the tensor map -> shared memory, completion on `bar`
__device__ __forceinline__ void tma_load4(void* dst, const CUtensorMap* map, int c2, int c1, int s, int comp,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];\n" ::"r"(smem_u32(dst)),
      "l"((unsigned long long)map), "r"(c2), "r"(c1), "r"(s), "r"(comp), "r"(smem_u32(bar))
      : "memory");
}

constexpr int M3_KSEG = 6;   // most segments of one CTA (host schedule); .w of the first = how many

// ---- shape ------------------------------------------------------------------------------------
template <int P, int NC, int T1, int T2, int RH>
struct M3 {
  static constexpr int NP = T1 * T2;                    // points of the tile = threads with a point
  static constexpr int NT = (NP + 31) / 32 * 32;        // full warps
  static constexpr int R = 2 * P + 1;
  static constexpr int HR = T1 + 2 * P;                 // tile rows with halo (direction 1)
  static constexpr int HC = T2 + 2 * P;                 // tile columns with halo (direction 2)
  // TMA boxes start on a 16-byte boundary of the row (an even column; measured: odd fp64 start
  // columns raise an illegal-instruction fault), so when q0 - P can be odd the box starts one
  // column early and the tile carries one extra column
  static constexpr bool SHIFT = (T2 % 2 == 1) || (P % 2 == 1);
  static constexpr int XP = (HC + (SHIFT ? 1 : 0) + 1) / 2 * 2;   // x row pitch (16-byte multiple)
  static constexpr int XS = HR * XP;                    // one component of one slab tile
  static constexpr int XB = (NC * XS + 15) / 16 * 16;   // one slab buffer (128-byte aligned)
  // u row pitch: a half-warp of pass B that spans two tile rows must not fold onto the same
  // banks, so the pitch is congruent to T2 modulo 16 doubles
  static constexpr int UP = (T2 % 16 == 0) ? HC : HC + (((T2 - HC) % 16) + 16) % 16;
  static constexpr int US = T1 * UP;                    // one pass-A output array
  static constexpr int UB = 3 * NC * US;                // one u buffer: [F][j][T1][UP]
  static constexpr int NSEG = (T1 + RH - 1) / RH;       // pass-A row segments (the last may be shorter)
  static constexpr int NITEMS = NC * NSEG * HC;         // pass-A items (component, segment, column)
  static constexpr int IPT = (NITEMS + NT - 1) / NT;    // items per thread
  static constexpr int LPT = (NC * XS + NT - 1) / NT;   // cp.async path: copies per thread
  static constexpr int WZ = 3 * R * T2;                 // direction-2 band rows of the tile's columns
  static constexpr size_t SMEM = (size_t)(2 * XB + 2 * UB + WZ) * 8 + 16 + (NT / 32) * 8;
  static constexpr int MINB = NC == 3 ? 2 : 3;
};

template <int P, int NC, int T1, int T2, int RH, bool TMA>
__global__ void __launch_bounds__(M3<P, NC, T1, T2, RH>::NT, M3<P, NC, T1, T2, RH>::MINB)
    k_march3d(const __grid_constant__ CUtensorMap tmx, const OpParams op, const Epi ep, int mode, int dot,
              const double* __restrict__ x, double* __restrict__ y, int ntx, const int4* __restrict__ segs,
              long long* __restrict__ dbg) {
  using Sh = M3<P, NC, T1, T2, RH>;
  constexpr int NT = Sh::NT, NP = Sh::NP, R = Sh::R, HC = Sh::HC, XP = Sh::XP, XS = Sh::XS, XB = Sh::XB;
  constexpr int UP = Sh::UP, US = Sh::US, UB = Sh::UB, NSEG = Sh::NSEG, NITEMS = Sh::NITEMS, IPT = Sh::IPT;
  constexpr int LPT = Sh::LPT, WZ = Sh::WZ;
  extern __shared__ __align__(128) double smem[];
  double* xs = smem;                                          // [2][XB]: [NC][HR][XP] each
  double* us = xs + 2 * XB;                                   // [2][UB]
  double* wz = us + 2 * UB;                                   // [3][R][T2]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(wz + WZ);      // [2]
  double* red = reinterpret_cast<double*>(mbar + 2);          // [NT/32]

  const int m = op.m;
  const int ms = m * m;   // ndof < 2^31 is checked on the host
  const int m3 = ms * m;
  const int tid = threadIdx.x;
  const bool real = tid < NP;       // padding threads of the last warp own no point
  const Coef& C = op.c;

  // pass-A items of this thread (tile independent): RH outputs down one halo column
  int a_x[IPT], a_u[IPT], a_r[IPT];
#pragma unroll
  for (int i = 0; i < IPT; ++i) {
    const int it = tid + i * NT;
    a_x[i] = a_u[i] = 0;
    a_r[i] = -1;
    if (it < NITEMS) {
      const int j = it / (NSEG * HC), rem = it - j * (NSEG * HC);
      const int seg = rem / HC, cc = rem - seg * HC;
      a_x[i] = j * XS + seg * RH * XP + cc;
      a_u[i] = j * US + seg * RH * UP + cc;
      a_r[i] = seg * RH;
    }
  }

  if constexpr (TMA) {
    if (tid == 0) {
      mbar_init(&mbar[0], 1);
      mbar_init(&mbar[1], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
  }

  double dsum = 0.0;
  unsigned nld = 0;   // slab tiles requested so far (uniform): tile n lands in x buffer n & 1
  // ---- this CTA's segments: (tile, first output slab, one past the last), built on the host
  // (m3_schedule below): contiguous pieces of the cost-weighted unit order
  const int nseg = segs[blockIdx.x * M3_KSEG].w;
  if (dbg && tid == 0) {   // IGACD_A3_DBG: per-CTA record (SM, start, end, first segment)
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    dbg[blockIdx.x * 5 + 0] = smid;
    dbg[blockIdx.x * 5 + 1] = t0;
    dbg[blockIdx.x * 5 + 3] = nseg;
    dbg[blockIdx.x * 5 + 4] = segs[blockIdx.x * M3_KSEG].x;
  }

#pragma unroll 1
  for (int sg = 0; sg < nseg; ++sg) {
    // ---- segment: output slabs [c0, c1) of one tile ------------------------------------------
    const int4 sd = segs[blockIdx.x * M3_KSEG + sg];
    const int tile = sd.x, c0 = sd.y, c1 = sd.z;
    const int ty = tile / ntx, tx = tile - ty * ntx;
    const int r0 = ty * T1, q0 = tx * T2;
    const int tr = real ? tid / T2 : 0, tc = real ? tid % T2 : 0;   // lanes along direction 2
    const int gr = r0 + tr, gc = q0 + tc;
    const bool active = real && gr < m && gc < m;
    const bool zoneB = active && (gc < op.zoneL || gc >= op.zoneR);
    const bool wzb = __any_sync(0xffffffffu, zoneB);
    const int sb = max(0, c0 - P);   // first slab that reaches an output of the segment
    const int se = c1 + P;           // one past the last slab step (slabs >= m contribute zero)
    const int sl = min(se, m);       // one past the last slab with data
    const int cs = (q0 - P) & ~1;    // first tile column (even: 16-byte aligned TMA box start)
    const int co = (q0 - P) - cs;    // 0 or 1: tile column of halo column 0
    const unsigned nb = nld;         // slab s of this segment is tile number nb + (s - sb)

    // cp.async path: slab-invariant offsets of this thread's copies
    int goff[TMA ? 1 : LPT];
    unsigned vmask = 0u;
    if constexpr (!TMA) {
#pragma unroll
      for (int i = 0; i < LPT; ++i) {
        const int idx = tid + i * NT;
        goff[i] = 0;
        if (idx < NC * XS) {
          const int j = idx / XS, rem = idx - j * XS;
          const int g1 = r0 - P + rem / XP, g2 = cs + rem % XP;
          if (g1 >= 0 && g1 < m && g2 >= 0 && g2 < m) {
            goff[i] = j * m3 + g1 * m + g2;
            vmask |= 1u << i;
          }
        }
      }
    }
    auto issue = [&](int s) {   // request slab s (< sl)
      const unsigned n = nb + (unsigned)(s - sb);
      double* dst = xs + (n & 1u) * XB;
      if constexpr (TMA) {
        if (tid == 0) {
          uint64_t* bar = &mbar[n & 1u];
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic reads before async writes
          mbar_expect_tx(bar, (unsigned)(NC * XS * 8));
          tma_load4(dst, &tmx, cs, r0 - P, s, 0, bar);
        }
      } else {
        const double* src = x + (size_t)s * ms;
#pragma unroll
        for (int i = 0; i < LPT; ++i)
          if (tid + i * NT < NC * XS) {
            const bool ok = (vmask >> i) & 1u;
            cp8(dst + tid + i * NT, ok ? src + goff[i] : x, ok);
          }
        cp_commit();
      }
    };
    auto ready = [&](int s) {   // TMA: wait for the bytes of slab s (cp.async: wait_all + barrier)
      if constexpr (TMA) {
        const unsigned n = nb + (unsigned)(s - sb);
        mbar_wait(&mbar[n & 1u], (n >> 1) & 1u);
      }
    };

    // ---- pass A: direction 1 of slab tile xb -> ub --------------------------------------------
    auto passA = [&](const double* xb, double* ub) {
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        if (a_r[i] >= 0) {
          const double* col = xb + a_x[i] + co;   // input row (a_r - P) of the halo column
          double* uo = ub + a_u[i];
          const int g0 = r0 + a_r[i];             // global row of the first output
          const bool zone_any = g0 < op.zoneL || g0 + RH > op.zoneR;
          constexpr bool RAGGED = T1 % RH != 0;   // rows past the tile in the last segment
          double win[RH + 2 * P];
#pragma unroll
          for (int k = 0; k < RH + 2 * P; ++k) win[k] = (!RAGGED || a_r[i] + k < T1 + 2 * P) ? col[k * XP] : 0.0;
#pragma unroll
          for (int r = 0; r < RH; ++r) {
            if (RAGGED && a_r[i] + r >= T1) break;
            double vm, vs, va;
            const int g1 = g0 + r;
            if (zone_any && (g1 < op.zoneL || g1 >= op.zoneR)) {   // band row (uniform over the item's lanes)
              vm = vs = va = 0.0;
              if (g1 < m) {
                const double* rM = op.bM + g1 * R;
                const double* rS = op.bS + g1 * R;
                const double* rA = op.bA + g1 * R;
#pragma unroll
                for (int o = 0; o < R; ++o) {
                  const double v = win[r + o];
                  vm = fma(__ldg(rM + o), v, vm);
                  vs = fma(__ldg(rS + o), v, vs);
                  va = fma(__ldg(rA + o), v, va);
                }
              }
            } else {   // Toeplitz row: symmetric pairing, register weights
              const double xc = win[r + P];
              vm = op.tM[0] * xc;
              vs = op.tS[0] * xc;
              va = 0.0;
#pragma unroll
              for (int o = 1; o <= P; ++o) {
                const double lo = win[r + P - o], hi = win[r + P + o];
                const double sp = lo + hi, sd = hi - lo;
                vm = fma(op.tM[o], sp, vm);
                vs = fma(op.tS[o], sp, vs);
                va = fma(op.tA[o], sd, va);
              }
            }
            uo[(0 * NC) * US + r * UP] = vm;
            uo[(1 * NC) * US + r * UP] = vs;
            uo[(2 * NC) * US + r * UP] = va;
          }
        }
      }
    };

    // ---- segment prologue ----------------------------------------------------------------------
    __syncthreads();   // the previous segment is done with the shared arrays (first: mbarrier init)
    for (int idx = tid; idx < WZ; idx += NT) {   // band rows of the tile's columns, [f][o][column]
      const int f = idx / (R * T2), rem = idx - f * (R * T2);
      const int o = rem / T2, c = rem - o * T2;
      const double* band = f == 0 ? op.bM : (f == 1 ? op.bS : op.bA);
      wz[idx] = (q0 + c < m) ? __ldg(band + (q0 + c) * R + o) : 0.0;
    }
    issue(sb);
    if (sb + 1 < sl) issue(sb + 1);
    nld += (unsigned)(sl - sb);
    if constexpr (!TMA) {
      cp_wait_all();
      __syncthreads();
    }
    ready(sb);
    passA(xs + (nb & 1u) * XB, us);
    __syncthreads();

    double acc[NC][R];   // direction-0 ring
#pragma unroll
    for (int i = 0; i < NC; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[i][r] = 0.0;
    double M1 = 1.0, S1 = 0.0, M2 = 1.0, S2 = 0.0;
    if (mode >= EPI_JACOBI && active) {
      M1 = __ldg(op.bM + gr * R + P); S1 = __ldg(op.bS + gr * R + P);
      M2 = __ldg(op.bM + gc * R + P); S2 = __ldg(op.bS + gc * R + P);
    }
    const int bo = tr * UP + tc + P;   // pass-B window centre
    const int pto = gr * m + gc;       // in-slab output offset

#pragma unroll 1
    for (int s = sb; s < se; ++s) {
      const int k = s - sb;
      if (s + 2 < sl) issue(s + 2);   // into the buffer pass A read in the previous phase
      if (s + 1 < sl) {
        ready(s + 1);
        passA(xs + ((nb + k + 1) & 1u) * XB, us + ((k + 1) & 1) * UB);
      }
      double fin[NC];   // final value of slab s - P
      // z stays zero when the slab has no data (s >= m: the ring drains) or the thread no point:
      // pass C then only shifts the ring, through the same instructions (a third code path that
      // shifted by moves cost register copies at the merge)
      double zM[NC], zS[NC], zA[NC];
#pragma unroll
      for (int i = 0; i < NC; ++i) zM[i] = zS[i] = zA[i] = 0.0;
      if (s < m && active) {
        // ---- pass B: direction 2 and the pattern combinations
        const double* ub = us + (k & 1) * UB + bo;
        if (!wzb) {
#pragma unroll
          for (int j = 0; j < NC; ++j) {
            const double* uM = ub + (0 * NC + j) * US;
            const double* uS = ub + (1 * NC + j) * US;
            const double* uA = ub + (2 * NC + j) * US;
            double vMM, vMS, vMA, vSM, vAM, vAA;
            {
              const double c = uM[0];
              double a1 = op.tM[0] * c, a2 = op.tS[0] * c, a3 = 0.0;
#pragma unroll
              for (int o = 1; o <= P; ++o) {
                const double lo = uM[-o], hi = uM[o];
                const double sp = lo + hi, sd = hi - lo;
                a1 = fma(op.tM[o], sp, a1);
                a2 = fma(op.tS[o], sp, a2);
                a3 = fma(op.tA[o], sd, a3);
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
#pragma unroll
            for (int i = 0; i < NC; ++i) {
              zM[i] = fma(C.mass[i][j], vMM, zM[i]);
              zS[i] = fma(C.S[0][i][j], vMM, zS[i]);
              zM[i] = fma(C.S[1][i][j], vSM, zM[i]);
              zM[i] = fma(C.S[2][i][j], vMS, zM[i]);
              zA[i] = fma(C.AA[0][i][j], vAM, zA[i]);
              zA[i] = fma(C.AA[1][i][j], vMA, zA[i]);
              zM[i] = fma(C.AA[2][i][j], vAA, zM[i]);
            }
          }
        } else {
          // a warp with boundary-zone columns: every lane uses its own column's band row, read
          // ONCE per tap for all components (tap-outer: 3 weight + 9 window loads per tap)
          double vMM[NC], vMS[NC], vMA[NC], vSM[NC], vAM[NC], vAA[NC];
#pragma unroll
          for (int j = 0; j < NC; ++j) vMM[j] = vMS[j] = vMA[j] = vSM[j] = vAM[j] = vAA[j] = 0.0;
#pragma unroll
          for (int o = 0; o < R; ++o) {
            const double wm = wz[(0 * R + o) * T2 + tc], ws = wz[(1 * R + o) * T2 + tc];
            const double wa = wz[(2 * R + o) * T2 + tc];
#pragma unroll
            for (int j = 0; j < NC; ++j) {
              const double um = ub[(0 * NC + j) * US + o - P], usv = ub[(1 * NC + j) * US + o - P];
              const double ua = ub[(2 * NC + j) * US + o - P];
              vMM[j] = fma(wm, um, vMM[j]);
              vMS[j] = fma(ws, um, vMS[j]);
              vMA[j] = fma(wa, um, vMA[j]);
              vSM[j] = fma(wm, usv, vSM[j]);
              vAM[j] = fma(wm, ua, vAM[j]);
              vAA[j] = fma(wa, ua, vAA[j]);
            }
          }
#pragma unroll
          for (int j = 0; j < NC; ++j)
#pragma unroll
            for (int i = 0; i < NC; ++i) {
              zM[i] = fma(C.mass[i][j], vMM[j], zM[i]);
              zS[i] = fma(C.S[0][i][j], vMM[j], zS[i]);
              zM[i] = fma(C.S[1][i][j], vSM[j], zM[i]);
              zM[i] = fma(C.S[2][i][j], vMS[j], zM[i]);
              zA[i] = fma(C.AA[0][i][j], vAM[j], zA[i]);
              zA[i] = fma(C.AA[1][i][j], vMA[j], zA[i]);
              zM[i] = fma(C.AA[2][i][j], vAA[j], zM[i]);
            }
        }
      }
      {
        // ---- pass C: scatter along direction 0 into the ring (rows t = s-P+r) and shift it in the
        // same instructions: ring slot r-1 <- slot r + F[t][s] z(s); slot 0 + F[s-P][s] z(s) is the
        // final value of slab s-P.  When all rows are Toeplitz rows, F[t][s] = T[s-t] is a register
        // constant (A: skew sign); rows outside the segment are never written out, so they need
        // no masking here.
        if (s - P >= op.zoneL && s + P < op.zoneR) {
#pragma unroll
          for (int i = 0; i < NC; ++i)
            fin[i] = fma(op.tM[P], zM[i], fma(op.tS[P], zS[i], fma(op.tA[P], zA[i], acc[i][0])));
#pragma unroll
          for (int r = 1; r < R; ++r) {
            const int d = P - r;   // s - t
            const int ad = d < 0 ? -d : d;
            const double wM = op.tM[ad], wS = op.tS[ad], wA = d >= 0 ? op.tA[ad] : -op.tA[ad];
#pragma unroll
            for (int i = 0; i < NC; ++i)
              acc[i][r - 1] = fma(wM, zM[i], fma(wS, zS[i], fma(wA, zA[i], acc[i][r])));
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) {
            const int t = s - P + r;
            const bool in = t >= 0 && t < m;
            const int tcl = in ? t : min(s, m - 1);        // clamped row: the address is always in range
            const int kk = tcl * R + (s - tcl) + P;        // F[t][s]
            const double sel = in ? 1.0 : 0.0;
            const double wM = sel * __ldg(op.bM + kk), wS = sel * __ldg(op.bS + kk), wA = sel * __ldg(op.bA + kk);
#pragma unroll
            for (int i = 0; i < NC; ++i) {
              const double v = fma(wM, zM[i], fma(wS, zS[i], fma(wA, zA[i], acc[i][r])));
              if (r == 0) fin[i] = v;
              else acc[i][r - 1] = v;
            }
          }
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) acc[i][R - 1] = 0.0;
      }
      // ---- epilogue of slab t = s - P
      {
        const int t = s - P;
        if (t >= c0 && t < c1 && active) {
          const int pt = t * ms + pto;
          double M0 = 1.0, S0 = 0.0;
          if (mode >= EPI_JACOBI) {
            M0 = __ldg(op.bM + t * R + P);
            S0 = __ldg(op.bS + t * R + P);
          }
#pragma unroll
          for (int i = 0; i < NC; ++i) {
            const double a = fin[i];
            const int gi = i * m3 + pt;
            double out;
            if (mode == EPI_APPLY) {
              out = a;
            } else if (mode == EPI_RESID) {
              out = ep.b[gi] - a;
            } else {
              const double Dv = C.mass[i][i] * M0 * M1 * M2 + C.S[0][i][i] * S0 * M1 * M2 +
                                C.S[1][i][i] * M0 * S1 * M2 + C.S[2][i][i] * M0 * M1 * S2;
              out = mode == EPI_JACOBI ? x[gi] + ep.omega * (ep.b[gi] - a) / Dv : a / Dv;
            }
            y[gi] = out;
            if (dot == DOT_X_OUT) dsum = fma(x[gi], out, dsum);
            else if (dot == DOT_OUT_OUT) dsum = fma(out, out, dsum);
          }
        }
      }
      if constexpr (!TMA) cp_wait_all();   // slab s + 2 landed (this thread's copies)
      __syncthreads();   // u[(k+1)&1] complete; x buffer of slab s+1 and u[k&1] free
    }
  }
  if (dbg && tid == 0) {
    long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    dbg[blockIdx.x * 5 + 2] = t1;
  }
  if (dot != DOT_NONE) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) dsum += __shfl_down_sync(0xffffffffu, dsum, off);
    if ((tid & 31) == 0) red[tid >> 5] = dsum;
    __syncthreads();
    if (tid == 0) {
      double sacc = 0.0;
      for (int w = 0; w < NT / 32; ++w) sacc += red[w];
      ep.partial[blockIdx.x] = sacc;
    }
  }
}

// ---- host side --------------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda at link time)
static EncodeTiledFn encode_fn() {
  static std::once_flag once;
  static EncodeTiledFn fn = nullptr;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  if (!fn) throw Error{IGACD_E_CUDA, "cuTensorMapEncodeTiled unavailable"};
  return fn;
}

// x viewed as [nc][m][m][m] fp64; box = one slab tile with halo, all components
static CUtensorMap slab_map(const double* x, int m, int nc, int boxw, int boxh) {
  CUtensorMap map;
  const cuuint64_t dims[4] = {(cuuint64_t)m, (cuuint64_t)m, (cuuint64_t)m, (cuuint64_t)nc};
  const cuuint64_t strides[3] = {(cuuint64_t)m * 8, (cuuint64_t)m * m * 8, (cuuint64_t)m * m * m * 8};
  const cuuint32_t box[4] = {(cuuint32_t)boxw, (cuuint32_t)boxh, 1u, (cuuint32_t)nc};
  const cuuint32_t es[4] = {1u, 1u, 1u, 1u};
  const CUresult r = encode_fn()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(x), dims, strides, box,
                                 es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error{IGACD_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")"};
  return map;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

// tile variants: 0 = 9 x 27 (m = 162: 18 x 6 tiles, no padding), 1 = 8 x 32: the one with fewer
// padded thread slots.  Pass A splits the tile rows into segments so that there is about one
// item (component, segment, halo column) per thread -- 9 x 27: rows 5 + 4 (vector), 3 x 3
// (scalar); with one 9-row item per column only 105 of 243 threads had pass-A work and the
// others waited at the barrier (config 4: 0.305 -> 0.272 ms, scalar 0.129 -> 0.117 ms).
static int tile_variant(int m, int nc) {
  static const int force = env_int("IGACD_A3_TILE", -1);
  (void)nc;
  if (force >= 0) return force;
  auto padded = [&](int t1, int t2, int nt) {   // thread slots per slab
    return (double)((m + t1 - 1) / t1) * ((m + t2 - 1) / t2) * nt;
  };
  return padded(9, 27, 256) <= padded(8, 32, 256) ? 0 : 1;
}

// persistent grid: every resident slot, but at least `IGACD_A3_MINU` (default 4) units per CTA
static int march_ctas(int slots, int units) {
  static const int minu = std::max(1, env_int("IGACD_A3_MINU", 4));
  return std::max(1, std::min(slots, units / minu));
}

struct M3Plan {
  int ctas, ntx, nty;
  const int4* segs;
};

// The schedule of one launch configuration: units are (tile, output slab); a unit costs 16, plus
// zc in a tile with boundary-zone columns (per-lane band rows in pass B) and zr in one with
// boundary-zone rows (band rows in pass A) -- the measured per-unit times of the four tile
// classes (IGACD_A3_DBG timeline).  The units are laid on a line and cut into G pieces of equal
// cost; a piece that crosses a run boundary becomes several segments (2p warm-up slabs each).
//   order 0: tile-major, one run per tile (fewest segments);
//   order 1 (default, nch = 2): chunk-major -- the slab range is cut into nch chunks and the tiles
//            of a chunk follow each other column by column, so CTAs marching neighbouring tiles
//            are closer in time and more of the tile halos hit the L2, at the price of more
//            segments.  Measured (config 4, DRAM bytes per apply / time): order 0 354 MB / 0.305 ms;
//            nch = 1 332 MB / 0.308; nch = 2 279 MB / 0.309; nch = 3 307 MB / 0.328 ms.
static const int4* m3_schedule(int m, int zoneL, int zoneR, int t1, int t2, int G) {
  static const int zc = std::max(0, env_int("IGACD_A3_ZC", 6)), zr = std::max(0, env_int("IGACD_A3_ZR", 12));
  static const int order = env_int("IGACD_A3_ORDER", 1), nch = std::max(1, env_int("IGACD_A3_NCH", 2));
  static std::mutex mu;
  static std::map<std::tuple<int, int, int, int, int, int, int>, int4*> cache;
  int dev = 0;
  IGACD_CUDA(cudaGetDevice(&dev));
  const auto key = std::make_tuple(dev, m, zoneL, zoneR, t1, t2, G);
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  const int ntx = (m + t2 - 1) / t2, nty = (m + t1 - 1) / t1;
  auto has_zone = [&](int t0, int tw) { return t0 < zoneL || std::min(t0 + tw, m) > zoneR; };
  struct Run { int tile, s0, s1, w; };
  std::vector<Run> runs;
  auto cost = [&](int ty, int tx) { return 16 + (has_zone(tx * t2, t2) ? zc : 0) + (has_zone(ty * t1, t1) ? zr : 0); };
  if (order == 0) {
    for (int ty = 0; ty < nty; ++ty)
      for (int tx = 0; tx < ntx; ++tx) runs.push_back({ty * ntx + tx, 0, m, cost(ty, tx)});
  } else {
    const int lc = (m + nch - 1) / nch;
    for (int c = 0; c * lc < m; ++c)
      for (int tx = 0; tx < ntx; ++tx)
        for (int ty = 0; ty < nty; ++ty) runs.push_back({ty * ntx + tx, c * lc, std::min(m, (c + 1) * lc), cost(ty, tx)});
  }
  long long ctot = 0;
  for (const Run& r : runs) ctot += (long long)(r.s1 - r.s0) * r.w;
  // position (run, slab) of cumulative cost c
  auto locate = [&](long long c, size_t* ri, int* sl) {
    for (size_t i = 0; i < runs.size(); ++i) {
      const long long rc = (long long)(runs[i].s1 - runs[i].s0) * runs[i].w;
      if (c < rc) {
        *ri = i;
        *sl = runs[i].s0 + (int)(c / runs[i].w);
        return;
      }
      c -= rc;
    }
    *ri = runs.size();
    *sl = 0;
  };
  std::vector<int4> h((size_t)G * M3_KSEG, make_int4(0, 0, 0, 0));
  for (int b = 0; b < G; ++b) {
    size_t r0, r1;
    int a0, a1;
    locate(ctot * b / G, &r0, &a0);
    locate(ctot * (b + 1) / G, &r1, &a1);
    int n = 0;
    for (size_t r = r0; r < runs.size() && (r < r1 || (r == r1 && a1 > runs[r].s0)); ++r) {
      const int c0 = r == r0 ? a0 : runs[r].s0;
      const int c1 = r == r1 ? a1 : runs[r].s1;
      if (c1 <= c0) continue;
      if (n == M3_KSEG) throw Error{IGACD_E_ARG, "3D operator schedule: too many segments per CTA"};
      h[(size_t)b * M3_KSEG + n] = make_int4(runs[r].tile, c0, c1, 0);
      ++n;
    }
    h[(size_t)b * M3_KSEG].w = n;
  }
  // a schedule first needed while this thread captures a graph (the PCG graphs are captured
  // after one eager iteration, so normally never): allocation and copy are legal in relaxed mode
  cudaStreamCaptureMode cm = cudaStreamCaptureModeRelaxed;
  IGACD_CUDA(cudaThreadExchangeStreamCaptureMode(&cm));
  int4* d = nullptr;
  cudaError_t e = cudaMalloc(&d, sizeof(int4) * h.size());
  if (e == cudaSuccess) e = cudaMemcpy(d, h.data(), sizeof(int4) * h.size(), cudaMemcpyHostToDevice);
  cudaThreadExchangeStreamCaptureMode(&cm);
  IGACD_CUDA(e);
  cache[key] = d;
  return d;
}

template <int P, int NC, int T1, int T2, int RH, bool TMA>
static M3Plan plan_m3(const OpParams* op, int m, int slot_share = 100) {
  using Sh = M3<P, NC, T1, T2, RH>;
  auto kern = k_march3d<P, NC, T1, T2, RH, TMA>;
  ensure_smem_attr((const void*)kern, Sh::SMEM);
  const int occ = max_active_blocks((const void*)kern, Sh::NT, Sh::SMEM);
  M3Plan pl;
  pl.ntx = (m + T2 - 1) / T2;
  pl.nty = (m + T1 - 1) / T1;
  pl.ctas = march_ctas(std::max(1, occ * num_sms() * slot_share / 100), pl.ntx * pl.nty * m);
  pl.segs = op ? m3_schedule(m, op->zoneL, op->zoneR, T1, T2, pl.ctas) : nullptr;
  return pl;
}

template <int P, int NC, int T1, int T2, int RH, bool TMA>
static int launch_m3(const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                     cudaStream_t s, int slot_share) {
  using Sh = M3<P, NC, T1, T2, RH>;
  const M3Plan pl = plan_m3<P, NC, T1, T2, RH, TMA>(&op, op.m, slot_share);
  CUtensorMap map;
  if constexpr (TMA) map = slab_map(x, op.m, NC, Sh::XP, Sh::HR);
  else std::memset(&map, 0, sizeof(map));
  static const int dbg_on = env_int("IGACD_A3_DBG", 0);               // per-CTA timeline on stderr (measurement)
  long long* dbg = nullptr;
  if (dbg_on && NC == dbg_on) IGACD_CUDA(cudaMalloc(&dbg, sizeof(long long) * 5 * pl.ctas));
  k_march3d<P, NC, T1, T2, RH, TMA><<<pl.ctas, Sh::NT, Sh::SMEM, s>>>(map, op, ep, mode, dot, x, y, pl.ntx, pl.segs, dbg);
  if (dbg) {
    std::vector<long long> hb(5 * pl.ctas);
    IGACD_CUDA(cudaStreamSynchronize(s));
    IGACD_CUDA(cudaMemcpy(hb.data(), dbg, sizeof(long long) * hb.size(), cudaMemcpyDeviceToHost));
    cudaFree(dbg);
    long long t0 = hb[1];
    for (int b = 0; b < pl.ctas; ++b) t0 = std::min(t0, hb[b * 5 + 1]);
    for (int b = 0; b < pl.ctas; ++b) {
      const int tile = (int)hb[b * 5 + 4];
      fprintf(stderr, "A3DBG m %d cta %d sm %lld start_us %.1f dur_us %.1f segments %lld first tile %d (ty %d tx %d)\n",
              op.m, b, hb[b * 5], (hb[b * 5 + 1] - t0) * 1e-3, (hb[b * 5 + 2] - hb[b * 5 + 1]) * 1e-3, hb[b * 5 + 3],
              tile, tile / pl.ntx, tile % pl.ntx);
    }
  }
  return pl.ctas;
}

// IGACD_TMA=0 stages every slab with cp.async (comparison only)
static bool tma_enabled() {
  static const int v = env_int("IGACD_TMA", 1);
  return v == 1;
}

// op == nullptr: only the grid size is wanted (the larger of the two staging variants).
// Returns the CTAs of the persistent grid = partial sums written when a DotMode is requested.
template <int P, int NC>
static int dispatch_m3(const OpParams* op, int m, const Epi* ep, int mode, int dot, const double* x, double* y,
                       cudaStream_t s, int slot_share) {
  // TMA needs 16-byte aligned global rows (m even) and base address
  const bool tma = tma_enabled() && m % 2 == 0 && (!x || ((uintptr_t)x & 15) == 0);
  const int v = tile_variant(m, NC);
#define IGACD_M3_CASE(T1, T2, RH3, RH1)                                                                      \
  do {                                                                                                       \
    constexpr int RH = NC == 3 ? RH3 : RH1;   /* pass-A rows per item: about one item per thread */          \
    if (!op)                                                                                                 \
      return std::max(plan_m3<P, NC, T1, T2, RH, true>(nullptr, m).ctas,                                     \
                      plan_m3<P, NC, T1, T2, RH, false>(nullptr, m).ctas);                                   \
    return tma ? launch_m3<P, NC, T1, T2, RH, true>(*op, *ep, mode, dot, x, y, s, slot_share)                \
               : launch_m3<P, NC, T1, T2, RH, false>(*op, *ep, mode, dot, x, y, s, slot_share);              \
  } while (0)
  if (v == 0) IGACD_M3_CASE(9, 27, 5, 3);
  IGACD_M3_CASE(8, 32, 4, 2);
#undef IGACD_M3_CASE
}

static int dispatch_p(int p, int nc, const OpParams* op, int m, const Epi* ep, int mode, int dot, const double* x,
                      double* y, cudaStream_t s, int slot_share = 100) {
#define IGACD_M3_P(PP)                                                                        \
  case PP:                                                                                    \
    return nc == 1 ? dispatch_m3<PP, 1>(op, m, ep, mode, dot, x, y, s, slot_share)            \
                   : dispatch_m3<PP, 3>(op, m, ep, mode, dot, x, y, s, slot_share)
  switch (p) {
#ifdef IGACD_DEV_P
    IGACD_M3_P(IGACD_DEV_P);
#else
    IGACD_M3_P(1);
    IGACD_M3_P(2);
    IGACD_M3_P(3);
    IGACD_M3_P(4);
    IGACD_M3_P(5);
    IGACD_M3_P(6);
#endif
    default: throw Error{IGACD_E_ARG, "degree out of range"};
  }
#undef IGACD_M3_P
}

int launch_apply3d(int p, int nc, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                   cudaStream_t s, int slot_share) {
  return dispatch_p(p, nc, &op, op.m, &ep, mode, dot, x, y, s, slot_share);
}

// The marching kernel pays 2p warm-up slabs per segment, so it needs enough output slabs per
// CTA: true when a level has at least IGACD_A3_MINSLABS (default 32) units per resident CTA slot
// (2 x SMs).  Smaller levels of the vector system take the split slab + column kernels.
bool apply3d_marching_pays(int m) {
  static const int minslabs = env_int("IGACD_A3_MINSLABS", 32);
  const int v = tile_variant(m, 3);
  const int t1 = v == 0 ? 9 : 8, t2 = v == 0 ? 27 : 32;
  const long long units = (long long)((m + t1 - 1) / t1) * ((m + t2 - 1) / t2) * m;
  return units >= (long long)minslabs * 2 * num_sms();
}

// upper bound of the persistent grid of a level (sizes the partial-sum buffer)
int apply3d_ctas(int p, int nc, int m) { return dispatch_p(p, nc, nullptr, m, nullptr, 0, 0, nullptr, nullptr, nullptr); }

}  // namespace igacd

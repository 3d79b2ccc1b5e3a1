// R2 in 3D: matrix-free operator y = A x (vector system nc = 3, auxiliary scalar system
// nc = 1) by sum factorisation in ONE kernel per apply, with fused epilogues (R4 smoother,
// residual, D^-1 A, dot products).
//
// The Galerkin matrix is sum_P C_P (x) F0_P (x) F1_P (x) F2_P with 1D factors M, A, S
// (eq:matr_Amu3D PAPER.md:515-543; the L_A form of reading R1 has the same Kronecker
// patterns, internal.cuh Coef).  A CTA owns a T2 x T3 tile of the (direction 1, direction 2)
// plane and marches a chunk of slabs along direction 0 (the slowest):
//   * the slab tile with its p-halo, all components, arrives in shared memory by TMA
//     (cp.async.bulk.tensor, out-of-domain elements zero-filled by the tensor map) into a
//     ring of NBX slab buffers, each completing on its own mbarrier; levels whose row pitch is
//     not 16-byte aligned (odd m) stage the tile with 8-byte cp.async instead;
//   * stage A contracts direction 1 (M, S, A of every halo column, register window down the
//     rows) into a double-buffered shared array u;
//   * stage B contracts direction 2 from u and forms the per-point combinations z_{i,F0};
//   * stage C scatters F0[t][s] z(s) into a register ring of 2p+1 output slabs; slab t = s-p
//     is then final and leaves through the epilogue.
// Stage A of slab s+1 and stages B/C of slab s run in the same phase, so the CTA needs ONE
// barrier per slab, and the intermediate z never leaves the SM (the round-1 split form wrote
// and re-read 9 doubles per point through HBM).
// Interior rows of every 1D factor are Toeplitz: contractions use 2p+1
// register weights with symmetric pairing (one add feeds M and S, one subtract feeds A);
// threads whose row lies in the boundary zone redo their contraction with the row's band.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "internal.cuh"

namespace igacd {

// Debug builds (-DIGACD_A3_DEBUG): bounds checks on every shared / global index of the kernel.
#ifndef A3_CHK_MASK
#define A3_CHK_MASK 0xff
#endif
#define A3_CHK_BIT(what) ((what)[0] == 'c' ? 1 : (what)[5] == 'A' ? 2 : (what)[5] == 'B' ? 4 : 8)
#ifdef IGACD_A3_DEBUG
#define A3_CHECK(cond, what, v)                                                                          \
  do {                                                                                                   \
    if ((A3_CHK_BIT(what) & A3_CHK_MASK) && !(cond)) {                                                                                       \
      printf("k_apply3d bounds: %s (%d) block (%d,%d,%d) thread %d\n", what, (int)(v), blockIdx.x, blockIdx.y, \
             blockIdx.z, threadIdx.x);                                                                   \
      __trap();                                                                                          \
    }                                                                                                    \
  } while (0)
#else
#define A3_CHECK(cond, what, v) \
  do {                          \
  } while (0)
#endif

// Scheduling fence: keeps the compiler from hoisting the next group of shared loads above it
// (the direction-0 ring alone holds 2 NC (2p+1) registers; hoisting all 27 stage-B loads of a
// component spills at 128 registers)
#ifndef A3_NOFENCE
#define A3_SCHED_FENCE() asm volatile("" ::: "memory")
#else
#define A3_SCHED_FENCE() \
  do {                   \
  } while (0)
#endif

// ---- async-copy primitives ------------------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void cp8(double* smem_dst, const double* gsrc, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

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

// ---- shape ------------------------------------------------------------------------------------
// The CTA has NC thread groups of G threads (full warps); group c owns component c: it runs
// stage A and stage B for input component j = c, mixes them into its contributions to every
// output component i, and keeps the direction-0 ring of output component i = c.  The groups
// exchange the cross-component contributions through shared memory (nc = 3: 6 doubles written
// and 6 read per thread and slab), so a thread's ring is 2p+1 doubles instead of 3(2p+1), its
// mixing coefficients are one column C[.][.][c] (warp-uniform), and the SM holds 3x the warps.
template <int P, int T2, int T3, int NC>
struct A3Shape {
  static constexpr int NP = T2 * T3;                    // points of the tile
  static constexpr int G = (NP + 31) / 32 * 32;         // threads per group (full warps)
  static constexpr int NT = NC * G;
  static constexpr int R = 2 * P + 1;
  static constexpr int HR = T2 + 2 * P;                 // tile rows with halo (direction 1)
  static constexpr int HC = T3 + 2 * P;                 // tile columns with halo (direction 2)
  // TMA boxes must start on a 16-byte boundary of the row (an even column; measured: odd fp64
  // start columns raise an illegal-instruction fault), so when q0 - P can be odd the box starts
  // one column early and the tile carries one extra column
  static constexpr bool SHIFT = (T3 % 2 == 1) || (P % 2 == 1);
  static constexpr int XP = (HC + (SHIFT ? 1 : 0) + 1) / 2 * 2;   // x row pitch (16-byte multiple)
  static constexpr int XS = HR * XP;                    // one component of one slab tile
  static constexpr int XB = (NC * XS + 15) / 16 * 16;   // one slab buffer (128-byte aligned)
  static constexpr int NBX = 2;                         // slab buffers in flight
  static constexpr int US = T2 * HC;                    // one stage-A output array
  static constexpr int UB = 3 * NC * US;                // one u buffer: [F][j][T2][HC]
  static constexpr int RH = 2;                          // rows per stage-A item
  static constexpr int RS = T2 / RH;                    // stage-A row segments
  static constexpr int NITEMS = RS * HC;                // stage-A items of one group (one component)
  static constexpr int LPT = (NC * XS + NT - 1) / NT;   // cp.async path: copies per thread
  static constexpr int WB = (3 * R + 1) / 2 * 2;        // direction-0 weights of one slab
  static constexpr int CB = NC == 3 ? 6 * 3 * NP : 0;   // one contribution buffer: [src c][dst slot][F][pt]
  // bytes: x ring, u double buffer, contributions double buffer, weights (3 slots), mbarriers, reduction
  static constexpr int SMEM = (NBX * XB + 2 * UB + 2 * CB + 3 * WB) * 8 + NBX * 8 + (NT / 32) * 8;
  static_assert(T2 % RH == 0, "row segments");
};

template <int P, int T2, int T3, int NC, bool TMA>
__global__ void __launch_bounds__(A3Shape<P, T2, T3, NC>::NT, 1)
    k_apply3d(const __grid_constant__ CUtensorMap tmx, const OpParams op, const Epi ep, int mode, int dot,
              const double* __restrict__ x, double* __restrict__ y, int chunk) {
  using Sh = A3Shape<P, T2, T3, NC>;
  constexpr int NT = Sh::NT, G = Sh::G, NP = Sh::NP, R = Sh::R, HC = Sh::HC, XP = Sh::XP, XS = Sh::XS;
  constexpr int XB = Sh::XB, NBX = Sh::NBX, US = Sh::US, UB = Sh::UB, RH = Sh::RH, NITEMS = Sh::NITEMS;
  constexpr int LPT = Sh::LPT, WB = Sh::WB, CB = Sh::CB;
  extern __shared__ __align__(128) double smem[];
  double* xs = smem;                                           // [NBX][XB]: [NC][HR][XP] each
  double* us = smem + NBX * XB;                                // [2][UB]
  double* cbuf = us + 2 * UB;                                  // [2][CB]
  double* wts = cbuf + 2 * CB;                                 // [3][WB]: F0[t][s], t = s-P..s+P
  uint64_t* mbar = reinterpret_cast<uint64_t*>(wts + 3 * WB);  // [NBX]
  double* red = reinterpret_cast<double*>(mbar + NBX);         // [NT/32]

  const int m = op.m;
  const int ms = m * m;   // ndof < 2^31 is checked on the host
  const int m3 = ms * m;
  const int tid = threadIdx.x;
  const int grp = tid / G;          // component of this thread (warp-uniform)
  const int lt = tid - grp * G;     // thread within the group
  const bool real = lt < NP;        // padding threads of the group's last warp own no point
  const int tr = real ? lt / T3 : T2 - 1, tc = real ? lt % T3 : 0;
  const int r0 = blockIdx.y * T2, q0 = blockIdx.x * T3;
  const int gr = r0 + tr, gc = q0 + tc;
  const bool active = real && gr < m && gc < m;
  const bool zoneB = active && (gc < op.zoneL || gc >= op.zoneR);
  const bool wzb = __any_sync(0xffffffffu, zoneB);
  const int c0 = blockIdx.z * chunk;
  const int c1 = min(c0 + chunk, m);
  const int sb = max(0, c0 - P);   // first slab that reaches an output of the chunk
  const int se = c1 + P;           // one past the last slab step (slabs >= m contribute zero)
  const int sl = min(se, m);       // one past the last slab with data
  const int cs = (q0 - P) & ~1;    // first tile column (even: 16-byte aligned TMA box start)
  const int co = (q0 - P) - cs;    // 0 or 1: tile column of halo column 0

  // ---- slab loads ----------------------------------------------------------------------------
  // cp.async path: slab-invariant offsets of this thread's copies
  int goff[TMA ? 1 : LPT];
  unsigned vmask = 0u;
  if constexpr (!TMA) {
#pragma unroll
    for (int i = 0; i < LPT; ++i) {
      const int idx = tid + i * NT;
      goff[i] = 0;
      if (idx < NC * XS) {
        const int j = idx / XS, rem = idx % XS;
        const int g1 = r0 - P + rem / XP, g2 = cs + rem % XP;
        if (g1 >= 0 && g1 < m && g2 >= 0 && g2 < m) {
          goff[i] = j * m3 + g1 * m + g2;
          vmask |= 1u << i;
        }
      }
    }
  }
  // slab k -> x ring buffer (k - sb) % NBX
  auto issue = [&](int k) {
    double* dst = xs + ((k - sb) % NBX) * XB;
    if constexpr (TMA) {
      if (tid == 0 && k < sl) {
        uint64_t* bar = &mbar[(k - sb) % NBX];
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic reads before async writes
        mbar_expect_tx(bar, (unsigned)(NC * XS * 8));
        tma_load4(dst, &tmx, cs, r0 - P, k, 0, bar);
      }
    } else {
      if (k < sl) {
        const double* src = x + (size_t)k * ms;
#pragma unroll
        for (int i = 0; i < LPT; ++i)
          if (tid + i * NT < NC * XS) {
            const bool ok = (vmask >> i) & 1u;
            A3_CHECK(dst + tid + i * NT - xs < NBX * XB, "cp8 dst", tid + i * NT);
            A3_CHECK(!ok || (k * ms + goff[i] < NC * m3 && goff[i] >= 0), "cp8 src", goff[i]);
            cp8(dst + tid + i * NT, ok ? src + goff[i] : x, ok);
          }
      }
      cp_commit();   // one group per slab step, possibly empty, so the group count stays uniform
    }
  };
  auto ready = [&](int k) {   // TMA: wait for the bytes of slab k (cp.async: ensured by a barrier)
    if constexpr (TMA) mbar_wait(&mbar[(k - sb) % NBX], (unsigned)(((k - sb) / NBX) & 1));
  };
  // column k of the direction-0 factors, F[t][k] for t = k-P..k+P (zero outside the matrix), for
  // the slabs whose rows are not all Toeplitz; written two slab steps ahead into a 3-slot ring
  auto load_wts = [&](int k, double* w) {
    if (tid < 3 * R) {
      const int f = tid / R, r = tid % R;
      const int t = k - P + r;
      double v = 0.0;
      if (t >= 0 && t < m) {
        const double* band = f == 0 ? op.bM : (f == 1 ? op.bS : op.bA);
        v = __ldg(band + t * R + (k - t) + P);
      }
      w[tid] = v;
    }
  };

  // ---- stage A: direction 1 for RH consecutive rows of one halo column of component grp -------
  auto stageA = [&](const double* xb, double* ub) {
#pragma unroll 1
    for (int it = lt; it < NITEMS; it += G) {
      const int a_cc = it % HC, a_r0 = (it / HC) * RH;
      const double* col = xb + grp * XS + a_r0 * XP + a_cc + co;   // input row a_r0 - P (halo origin)
      A3_CHECK(col - xs >= 0 && col + (RH + 2 * P - 1) * XP - xs < NBX * XB, "stageA x", it);
      double win[RH + 2 * P];
#pragma unroll
      for (int k = 0; k < RH + 2 * P; ++k) win[k] = col[k * XP];
      double* uo = ub + grp * US + a_r0 * HC + a_cc;
      A3_CHECK(uo - us >= 0 && uo + 2 * NC * US + (RH - 1) * HC - us < 2 * UB, "stageA u", it);
      const int g0 = r0 + a_r0;                                    // global row of the first output
      const bool zone_any = g0 < op.zoneL || g0 + RH > op.zoneR;   // uniform per item
#pragma unroll
      for (int r = 0; r < RH; ++r) {
        const double xc = win[r + P];
        double vm = op.tM[0] * xc, vs = op.tS[0] * xc, va = 0.0;
#pragma unroll
        for (int o = 1; o <= P; ++o) {
          const double lo = win[r + P - o], hi = win[r + P + o];
          const double sp = lo + hi, sd = hi - lo;
          vm = fma(op.tM[o], sp, vm);
          vs = fma(op.tS[o], sp, vs);
          va = fma(op.tA[o], sd, va);
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
        uo[(0 * NC) * US + r * HC] = vm;
        uo[(1 * NC) * US + r * HC] = vs;
        uo[(2 * NC) * US + r * HC] = va;
      }
    }
  };

  // ---- prologue ------------------------------------------------------------------------------
  if constexpr (TMA) {
    if (tid == 0) {
#pragma unroll
      for (int b = 0; b < NBX; ++b) mbar_init(&mbar[b], 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
#pragma unroll
  for (int b = 0; b < NBX; ++b) issue(sb + b);
  if constexpr (!TMA) cp_wait<NBX - 2>();   // slabs sb and sb + 1 landed (this thread's copies)
  __syncthreads();
  if (sb < sl) {
    ready(sb);
    stageA(xs, us);
    load_wts(sb, wts);
  }
  __syncthreads();
  issue(sb + NBX);

  double acc[R];   // direction-0 ring of output component grp
#pragma unroll
  for (int r = 0; r < R; ++r) acc[r] = 0.0;
  double dsum = 0.0;
  const int bo = tr * HC + tc + P;   // stage-B window centre
  const int pto = gr * m + gc;       // in-slab output offset
  const int pl = tr * T3 + tc;       // point index in the tile
  // mixing coefficients: column j = grp of every pattern (internal.cuh Coef), output rows i
  const Coef& C = op.c;

#pragma unroll 1
  for (int s = sb; s < se; ++s) {
    const int ph = (s - sb) & 1;
    const int wslot = (s - sb) % 3;
    // ================= phase 1: stage A (slab s+1), stage B + mixing (slab s) =================
    if (s + 1 < sl) {   // stage A of the next slab (its tile landed before the last barrier)
      ready(s + 1);
      stageA(xs + ((s + 1 - sb) % NBX) * XB, us + (ph ^ 1) * UB);
      load_wts(s + 1, wts + ((s + 1 - sb) % 3) * WB);
    }
    double zM = 0.0, zS = 0.0, zA = 0.0;   // own contribution to output component grp
    if (s < m && active) {
      // ---- stage B: direction 2 of component j = grp
      const double* ub = us + ph * UB;
      const double* uM = ub + (0 * NC + grp) * US + bo;
      const double* uS = ub + (1 * NC + grp) * US + bo;
      const double* uA = ub + (2 * NC + grp) * US + bo;
      A3_CHECK(uM - P - us >= 0 && uA + P - us < 2 * UB, "stageB u", bo);
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
      // ---- mixing: contributions of component j = grp to the z_{i,F0} of every output i
      // (patterns MMM, SMM, MSM, MMS, AAM, AMA, MAA; F0 = the direction-0 factor)
#pragma unroll
      for (int i = 0; i < NC; ++i) {
        const int j = grp;
        double cM = C.mass[i][j] * vMM;
        cM = fma(C.S[1][i][j], vSM, cM);
        cM = fma(C.S[2][i][j], vMS, cM);
        cM = fma(C.AA[2][i][j], vAA, cM);
        const double cS = C.S[0][i][j] * vMM;
        const double cA = fma(C.AA[0][i][j], vAM, C.AA[1][i][j] * vMA);
        if (NC == 1 || i == grp) {
          zM = cM; zS = cS; zA = cA;
        } else {   // slot k = 0, 1 of the destination: the two other components in order
          const int k = (grp < i) ? grp : grp - 1;   // my index among the sources of i
          double* cb = cbuf + ph * CB + ((i * 2 + k) * 3) * NP + pl;
          cb[0] = cM;
          cb[NP] = cS;
          cb[2 * NP] = cA;
        }
      }
    }
    if constexpr (!TMA) cp_wait<NBX - 2>();   // slab s + 2 landed (this thread's copies)
    __syncthreads();   // u[ph ^ 1], the contributions of slab s and the weights complete
    issue(s + 1 + NBX);
    // ================= phase 2: stage C (slab s) and the epilogue of slab s - P ===============
    if (s < m && active) {
      if constexpr (NC == 3) {
        const double* cb = cbuf + ph * CB + (grp * 2 * 3) * NP + pl;
        zM += cb[0] + cb[3 * NP];
        zS += cb[NP] + cb[4 * NP];
        zA += cb[2 * NP] + cb[5 * NP];
      }
      // scatter along direction 0 into the ring (rows t = s-P+r).  When all of them are
      // Toeplitz rows, F[t][s] = T[s-t] is a register constant (A: skew sign); rows outside this
      // CTA's chunk are never written out, so they need no masking here.
      if (s - P >= op.zoneL && s + P < op.zoneR) {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int d = P - r;   // s - t
          const int ad = d < 0 ? -d : d;
          const double wM = op.tM[ad], wS = op.tS[ad], wA = d >= 0 ? op.tA[ad] : -op.tA[ad];
          acc[r] = fma(wM, zM, fma(wS, zS, fma(wA, zA, acc[r])));
        }
      } else {
        const double* w = wts + wslot * WB;
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = fma(w[r], zM, fma(w[R + r], zS, fma(w[2 * R + r], zA, acc[r])));
      }
    }
    {
      const int t = s - P;
      if (t >= c0 && t < c1 && active) {
        const int pt = t * ms + pto;
        const int gi = grp * m3 + pt;
        A3_CHECK(gi >= 0 && gi < NC * m3, "epilogue", gi);
        const double a = acc[0];
        double out;
        if (mode == EPI_APPLY) {
          out = a;
        } else if (mode == EPI_RESID) {
          out = ep.b[gi] - a;
        } else {
          const double M0 = __ldg(op.bM + t * R + P), S0 = __ldg(op.bS + t * R + P);
          const double M1 = __ldg(op.bM + gr * R + P), S1 = __ldg(op.bS + gr * R + P);
          const double M2 = __ldg(op.bM + gc * R + P), S2 = __ldg(op.bS + gc * R + P);
          const double Dv = C.mass[grp][grp] * M0 * M1 * M2 + C.S[0][grp][grp] * S0 * M1 * M2 +
                            C.S[1][grp][grp] * M0 * S1 * M2 + C.S[2][grp][grp] * M0 * M1 * S2;
          out = mode == EPI_JACOBI ? x[gi] + ep.omega * (ep.b[gi] - a) / Dv : a / Dv;
        }
        y[gi] = out;
        if (dot == DOT_X_OUT) dsum = fma(x[gi], out, dsum);
        else if (dot == DOT_OUT_OUT) dsum = fma(out, out, dsum);
      }
#pragma unroll
      for (int r = 0; r < R - 1; ++r) acc[r] = acc[r + 1];
      acc[R - 1] = 0.0;
    }
  }
  if constexpr (!TMA) cp_wait<0>();
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

// ---- host side --------------------------------------------------------------------------------

// tile columns (direction 2): 32, or 27 when that wastes fewer columns (m = 162: 6 x 27 exactly)
static int a3_t3(int m) {
  static int force = -1;   // IGACD_A3_T3=32: always 32 columns (comparison only)
  if (force < 0) {
    const char* e = getenv("IGACD_A3_T3");
    force = (e && e[0] == '3') ? 32 : 0;
  }
  if (force) return force;
  const int w32 = (m + 31) / 32 * 32, w27 = (m + 26) / 27 * 27;
  return w27 < w32 ? 27 : 32;
}

// tile rows: the vector system (3 groups) 8 rows = 672 threads, IGACD_A3_T2=4: 4 rows, two
// CTAs per SM (comparison); the scalar system 16 rows = 448 threads
static int a3_t2(int nc) {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_A3_T2");
    v = (e && e[0] == '4') ? 4 : 8;
  }
  return nc == 3 ? v : 16;
}

// direction-0 chunks: about one wave of resident CTAs over the whole grid
static int a3_chunk(int m, int tiles, int per_sm) {
  const int target = per_sm * num_sms();
  int nch = std::max(1, std::min(m, (target + tiles / 2) / tiles));
  int chunk = (m + nch - 1) / nch;
  return std::max(chunk, std::min(m, 2));
}

dim3 apply3d_grid(int m, int nc, int* chunk) {
  const int T3 = a3_t3(m);
  const int T2 = a3_t2(nc);
  const int tx = (m + T3 - 1) / T3, ty = (m + T2 - 1) / T2;
  *chunk = a3_chunk(m, tx * ty, T2 == 4 ? 2 : 1);
  return dim3(tx, ty, (m + *chunk - 1) / *chunk);
}

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

// IGACD_TMA=0 stages every slab with cp.async (comparison only)
static bool tma_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_TMA");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

template <int P, int NC, int T2, int T3, bool TMA>
static void launch_a3(const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                      cudaStream_t s) {
  using Sh = A3Shape<P, T2, T3, NC>;
  auto kern = k_apply3d<P, T2, T3, NC, TMA>;
  ensure_smem_attr((const void*)kern, Sh::SMEM);
  int chunk = 0;
  const dim3 grid = apply3d_grid(op.m, NC, &chunk);
  CUtensorMap map;
  if constexpr (TMA) map = slab_map(x, op.m, NC, Sh::XP, Sh::HR);
  else std::memset(&map, 0, sizeof(map));
  kern<<<grid, Sh::NT, Sh::SMEM, s>>>(map, op, ep, mode, dot, x, y, chunk);
}

template <int P, int NC, int T3>
static void launch_a3_t(const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                        cudaStream_t s) {
  // TMA needs 16-byte aligned global rows (m even) and base address
  const bool tma = tma_enabled() && op.m % 2 == 0 && ((uintptr_t)x & 15) == 0;
  constexpr int T2a = NC == 3 ? 8 : 16, T2b = NC == 3 ? 4 : 16;
  if (a3_t2(NC) == T2a) {
    if (tma) launch_a3<P, NC, T2a, T3, true>(op, ep, mode, dot, x, y, s);
    else launch_a3<P, NC, T2a, T3, false>(op, ep, mode, dot, x, y, s);
  } else {
    if (tma) launch_a3<P, NC, T2b, T3, true>(op, ep, mode, dot, x, y, s);
    else launch_a3<P, NC, T2b, T3, false>(op, ep, mode, dot, x, y, s);
  }
}

template <int P>
static void dispatch_a3(int nc, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                        cudaStream_t s) {
  const bool t27 = a3_t3(op.m) == 27;
  if (nc == 1) {
    if (t27) launch_a3_t<P, 1, 27>(op, ep, mode, dot, x, y, s);
    else launch_a3_t<P, 1, 32>(op, ep, mode, dot, x, y, s);
  } else {
    if (t27) launch_a3_t<P, 3, 27>(op, ep, mode, dot, x, y, s);
    else launch_a3_t<P, 3, 32>(op, ep, mode, dot, x, y, s);
  }
}

void launch_apply3d(int p, int nc, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                    cudaStream_t s) {
  switch (p) {
    case 1: dispatch_a3<1>(nc, op, ep, mode, dot, x, y, s); break;
    case 2: dispatch_a3<2>(nc, op, ep, mode, dot, x, y, s); break;
    case 3: dispatch_a3<3>(nc, op, ep, mode, dot, x, y, s); break;
    case 4: dispatch_a3<4>(nc, op, ep, mode, dot, x, y, s); break;
    case 5: dispatch_a3<5>(nc, op, ep, mode, dot, x, y, s); break;
    case 6: dispatch_a3<6>(nc, op, ep, mode, dot, x, y, s); break;
    default: throw Error{IGACD_E_ARG, "degree out of range"};
  }
}

}  // namespace igacd

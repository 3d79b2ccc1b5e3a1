// R3: prolongation x_f = (I_d (x) P (x) .. (x) P) x_c and restriction x_c = P^T x_f
// (eq:2by2prol PAPER.md:1178-1186; R_l := P_l^T).  The two in-slab axes are
// applied in ONE shared-memory pass (k_transfer2d: a CTA stages the input window of a 16 x 32
// output tile, contracts axis 2 into an intermediate, then axis 1); 2D transfers are that
// single pass, 3D transfers add one pass along axis 0 (k_axis_pass_rows), which views the array
// as [outer][axis][inner] and writes one output element per thread from the fixed-width row
// storage of P (or P^T), coalesced along `inner`.  k_axis_pass_fast is the 1D pass along the
// fastest axis (consecutive threads read overlapping windows), used by the stage entry points.
#include <algorithm>

#include "internal.cuh"

namespace igacd {

// inner == 1 (fastest axis): one output per thread, 32-bit index math
__global__ void k_axis_pass_fast(const double* __restrict__ in, double* __restrict__ out, int outer, int nin, int nout,
                                 const int* __restrict__ start, const double* __restrict__ w, int W, int accumulate) {
  const int total = outer * nout;
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
    const int o = idx % nout, ou = idx / nout;
    const int st = __ldg(start + o);
    const double* src = in + ou * nin + st;
    const double* wr = w + o * W;
    double acc = 0.0;
    for (int k = 0; k < W; ++k)
      if (st + k < nin) acc = fma(__ldg(wr + k), __ldg(src + k), acc);
    if (accumulate) out[idx] += acc;
    else out[idx] = acc;
  }
}

// inner > 1: blockIdx.y = a group of RB consecutive output rows (ou, o), threads along the
// contiguous inner index.  One thread produces the RB outputs of its column, so the input rows
// those outputs share (P has overlapping row windows) are re-read from L1, not from L2.
constexpr int RB = 8;
__global__ void k_axis_pass_rows(const double* __restrict__ in, double* __restrict__ out, int rows, int nin, int nout,
                                 int inner, const int* __restrict__ start, const double* __restrict__ w, int W,
                                 int accumulate) {
  const int row0 = (blockIdx.y + blockIdx.z * gridDim.y) * RB;
  if (row0 >= rows) return;
  const int row1 = min(row0 + RB, rows);
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < inner; i += gridDim.x * blockDim.x) {
    for (int row = row0; row < row1; ++row) {
      const int o = row % nout, ou = row / nout;
      const int st = __ldg(start + o);
      const double* wr = w + o * W;
      const double* src = in + ((long long)ou * nin + st) * inner + i;
      double acc = 0.0;
      for (int k = 0; k < W; ++k)
        if (st + k < nin) acc = fma(__ldg(wr + k), __ldg(src + (long long)k * inner), acc);
      double* dst = out + (long long)row * inner + i;
      if (accumulate) *dst += acc;
      else *dst = acc;
    }
  }
}

static void axis_pass(Handle& h, const double* in, double* out, long long outer, int nin, int nout, long long inner,
                      const int* start, const double* w, int W, bool acc, cudaStream_t s) {
  const int bs = 256;
  if (inner == 1) {
    const long long total = outer * nout;
    long long blocks = (total + bs - 1) / bs;
    if (blocks > 148LL * 16) blocks = 148LL * 16;
    k_axis_pass_fast<<<(unsigned)std::max(1LL, blocks), bs, 0, s>>>(in, out, (int)outer, nin, nout, start, w, W,
                                                                    acc ? 1 : 0);
  } else {
    const long long rows = outer * nout;
    const long long groups = (rows + RB - 1) / RB;
    const int gy = (int)std::min(groups, 65535LL);
    const int gz = (int)((groups + gy - 1) / gy);
    const int gx = (int)std::min((inner + bs - 1) / bs, 65535LL);
    k_axis_pass_rows<<<dim3(gx, gy, gz), bs, 0, s>>>(in, out, (int)rows, nin, nout, (int)inner, start, w, W,
                                                     acc ? 1 : 0);
  }
  IGACD_LAUNCH_CHECK();
  count_launch(h);
}


// Both fastest axes in one pass (2D: the whole transfer; 3D: the in-slab part):
//   out[o1][o2] (+)= sum_{k1,k2} T[o1][k1] T[o2][k2] in[st(o1)+k1][st(o2)+k2]
// for every [nin][nin] slab of `in` (blockIdx.z = slab).  A CTA owns a TO1 x TO2 output tile:
// the input window it needs is staged in shared memory (coalesced rows), contracted along
// axis 2 into a [rows][TO2] intermediate, then along axis 1, so each input element is read
// from DRAM once (window halos come from L2) instead of once per 1D pass.
constexpr int TO1 = TRANSFER_TO1, TO2 = TRANSFER_TO2, NT2 = 256;

template <int W>   // row width of the 1D transfer (compile time: the contraction loops unroll and
                   // their weight loads are all in flight at once)
__global__ void __launch_bounds__(NT2) k_transfer2d(const double* __restrict__ in, double* __restrict__ out, int nin,
                                                    int nout, const int* __restrict__ start,
                                                    const double* __restrict__ w, int accumulate) {
  extern __shared__ __align__(16) double sm2[];
  const int o1a = blockIdx.y * TO1, o2a = blockIdx.x * TO2;
  const int o1b = min(o1a + TO1, nout), o2b = min(o2a + TO2, nout);
  const int i1a = __ldg(start + o1a), i2a = __ldg(start + o2a);
  const int i1b = min(__ldg(start + o1b - 1) + W, nin), i2b = min(__ldg(start + o2b - 1) + W, nin);
  const int IR = i1b - i1a, IC = i2b - i2a;
  const int ICP = IC | 1;   // odd row pitch: conflict-free column walks
  double* xin = sm2;                       // [IR][ICP]
  double* tmp = sm2 + IR * ICP;            // [IR][TO2]
  const double* src = in + (size_t)blockIdx.z * nin * nin;
  double* dst = out + (size_t)blockIdx.z * nout * nout;
  // accumulate: the outputs' old values are requested first, so their DRAM latency hides
  // behind the window load and both contractions (each thread owns OPT outputs)
  constexpr int OPT = TO1 * TO2 / NT2;
  static_assert(TO1 * TO2 % NT2 == 0, "whole outputs per thread");
  double old[OPT];
#pragma unroll
  for (int u = 0; u < OPT; ++u) {
    const int e = threadIdx.x + u * NT2;
    const int o1 = o1a + e / TO2, c2 = e % TO2;
    old[u] = (accumulate && o1 < o1b && o2a + c2 < o2b) ? dst[(size_t)o1 * nout + o2a + c2] : 0.0;
  }
  // window load: one warp per row, lanes along the row (no division by the runtime window width)
  for (int r = threadIdx.x >> 5; r < IR; r += NT2 / 32) {
    const double* srow = src + (size_t)(i1a + r) * nin + i2a;
    double* xrow = xin + r * ICP;
    for (int c = threadIdx.x & 31; c < IC; c += 32) xrow[c] = __ldg(srow + c);
  }
  __syncthreads();
  // axis 2: tmp[r][c2] = sum_k T[o2][k] xin[r][st(o2) - i2a + k].  Lane = output column (its W
  // weights are loaded once), warp = every (NT2/32)-th window row
  const int nc2 = o2b - o2a;
  {
    static_assert(TO2 == 32, "one lane per output column");
    const int c2 = threadIdx.x & 31;
    const bool on = c2 < nc2;
    const int o2 = on ? o2a + c2 : o2a;
    const int st = __ldg(start + o2);
    const int kn = min(W, nin - st);
    double wv[W];
#pragma unroll
    for (int k = 0; k < W; ++k) wv[k] = (on && k < kn) ? __ldg(w + (size_t)o2 * W + k) : 0.0;
    const double* xc = xin + (st - i2a);
    for (int r = threadIdx.x >> 5; r < IR; r += NT2 / 32) {
      const double* xr = xc + r * ICP;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < W; ++k)
        if (k < kn) acc = fma(wv[k], xr[k], acc);
      tmp[r * TO2 + c2] = acc;
    }
  }
  __syncthreads();
  // axis 1: out[o1][o2] = sum_k T[o1][k] tmp[st(o1) - i1a + k][c2]
#pragma unroll
  for (int u = 0; u < OPT; ++u) {
    const int e = threadIdx.x + u * NT2;
    const int r1 = e / TO2, c2 = e - r1 * TO2;
    const int o1 = o1a + r1;
    if (o1 >= o1b || c2 >= nc2) continue;
    const int st = __ldg(start + o1);
    const int kn = min(W, nin - st);
    const double* wr = w + (size_t)o1 * W;
    const double* tr = tmp + (st - i1a) * TO2 + c2;
    double acc = 0.0;
    double wv[W];
#pragma unroll
    for (int k = 0; k < W; ++k) wv[k] = __ldg(wr + k);
#pragma unroll
    for (int k = 0; k < W; ++k)
      if (k < kn) acc = fma(wv[k], tr[k * TO2], acc);
    dst[(size_t)o1 * nout + o2a + c2] = old[u] + acc;   // old = 0 unless accumulating
  }
}

// win1/win2: widest input window of a TO1-row / TO2-column output tile (Transfer1D)
static void transfer2d(Handle& h, const double* in, double* out, long long slabs, int nin, int nout, const int* start,
                       const double* w, int W, int win1, int win2, bool acc, cudaStream_t s) {
  const size_t smem = sizeof(double) * ((size_t)win1 * (win2 | 1) + (size_t)win1 * TO2);
  const dim3 grid((nout + TO2 - 1) / TO2, (nout + TO1 - 1) / TO1, (unsigned)slabs);
#define IGACD_T2D(WW)                                                                       \
  case WW:                                                                                  \
    ensure_smem_attr((const void*)k_transfer2d<WW>, smem);                                  \
    k_transfer2d<WW><<<grid, NT2, smem, s>>>(in, out, nin, nout, start, w, acc ? 1 : 0);   \
    break
  switch (W) {
    IGACD_T2D(1);
    IGACD_T2D(2);
    IGACD_T2D(3);
    IGACD_T2D(4);
    IGACD_T2D(5);
    IGACD_T2D(6);
    IGACD_T2D(7);
    IGACD_T2D(8);
    default: throw Error{IGACD_E_ARG, "transfer row width out of range"};
  }
#undef IGACD_T2D
  IGACD_LAUNCH_CHECK();
  count_launch(h);
}

// level l (fine, m_f) <- level l+1 (coarse, m_c)
void launch_prolong(Handle& h, int nc, int level, const double* xc, double* xf, bool accumulate, cudaStream_t s) {
  const Transfer1D& T = h.tr[level];
  const long long d = nc, mf = T.mf, mc = T.mc;
  if (h.dim == 2) {
    // [d][mc][mc] -> [d][mf][mf] in one pass
    transfer2d(h, xc, xf, d, (int)mc, (int)mf, T.p_start, T.p_w, T.wp, T.pwin1, T.pwin2, accumulate, s);
  } else {
    // axis 0: [d][mc][mc][mc] -> [d][mf][mc][mc]; axes 1, 2 per slab: -> [d][mf][mf][mf]
    double* scr = nc == 1 ? h.scratch1 : h.scratch0;   // the scalar system may run concurrently
    axis_pass(h, xc, scr, d, (int)mc, (int)mf, mc * mc, T.p_start, T.p_w, T.wp, false, s);
    transfer2d(h, scr, xf, d * mf, (int)mc, (int)mf, T.p_start, T.p_w, T.wp, T.pwin1, T.pwin2, accumulate, s);
  }
}

void launch_restrict(Handle& h, int nc, int level, const double* xf, double* xc, cudaStream_t s) {
  const Transfer1D& T = h.tr[level];
  const long long d = nc, mf = T.mf, mc = T.mc;
  if (h.dim == 2) {
    transfer2d(h, xf, xc, d, (int)mf, (int)mc, T.r_start, T.r_w, T.wr, T.rwin1, T.rwin2, false, s);
  } else {
    // axes 1, 2 per fine slab: [d][mf][mf][mf] -> [d][mf][mc][mc]; axis 0: -> [d][mc][mc][mc]
    double* scr = nc == 1 ? h.scratch1 : h.scratch0;
    transfer2d(h, xf, scr, d * mf, (int)mf, (int)mc, T.r_start, T.r_w, T.wr, T.rwin1, T.rwin2, false, s);
    axis_pass(h, scr, xc, d, (int)mf, (int)mc, mc * mc, T.r_start, T.r_w, T.wr, false, s);
  }
}

// Auxiliary-space maps of reading R8: Pi s = b0 s (component j = b0_j s), Pi^T v = sum_j b0_j v_j.
struct B0 {
  double b[3];
};

__global__ void k_pi_t(const double* __restrict__ v, double* __restrict__ sc, size_t ns, int d, B0 b0) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < ns; i += (size_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int j = 0; j < d; ++j) acc = fma(b0.b[j], v[j * ns + i], acc);
    sc[i] = acc;
  }
}

__global__ void k_pi(const double* __restrict__ sc, double* __restrict__ v, size_t ns, int d, B0 b0, int accumulate) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < ns; i += (size_t)gridDim.x * blockDim.x) {
    const double si = sc[i];
    for (int j = 0; j < d; ++j) {
      const double val = b0.b[j] * si;
      if (accumulate) v[j * ns + i] += val;
      else v[j * ns + i] = val;
    }
  }
}

static int grid1d(size_t n) {
  long long b = (long long)((n + 255) / 256);
  if (b > 148 * 8) b = 148 * 8;
  return (int)(b < 1 ? 1 : b);
}

void launch_pi_t(Handle& h, const double* v, double* sc, cudaStream_t s) {
  B0 b0;
  for (int j = 0; j < 3; ++j) b0.b[j] = h.b0[j];
  const size_t ns = h.lv[0].nscal;
  k_pi_t<<<grid1d(ns), 256, 0, s>>>(v, sc, ns, h.dim, b0);
  IGACD_LAUNCH_CHECK();
  count_launch(h);
}

void launch_pi(Handle& h, const double* sc, double* v, bool accumulate, cudaStream_t s) {
  B0 b0;
  for (int j = 0; j < 3; ++j) b0.b[j] = h.b0[j];
  const size_t ns = h.lv[0].nscal;
  k_pi<<<grid1d(ns), 256, 0, s>>>(sc, v, ns, h.dim, b0, accumulate ? 1 : 0);
  IGACD_LAUNCH_CHECK();
  count_launch(h);
}

}  // namespace igacd

// R1 (1D Gauss-quadrature assembly of M, A, S) and R3 (knot-insertion prolongation).
//
// PAPER.md:336-345 (Sec. 3.2): M_ij = int N_{i+1} N_{j+1}, A_ij = int N_{i+1} N'_{j+1},
// S_ij = int N'_{i+1} N'_{j+1}, i,j = 1..n+p-2 on the uniform open knot vector of
// PAPER.md:215-222.  One thread per band entry F[k][k+o]; each thread integrates over the
// knot spans both B-splines share with a (p+1)-point Gauss rule (exact for degree 2p).
// B-spline values come from the triangular "basis functions" recurrence (de Boor / Cox),
// evaluated per quadrature point on the device.
//
// R3: the prolongation P is the knot-insertion matrix of uniform refinement n_c -> 2 n_c:
// column j = coefficients of the coarse B-spline N^c_j in the fine basis, by the Oslo
// recurrence (Cohen-Lyche-Riesenfeld) -- one thread per entry.
#include <cmath>
#include <cstring>

#include "internal.cuh"

namespace igacd {

__host__ __device__ inline double knot(int p, int n, int j) {  // 0-based knot xi[j], j = 0..2p+n
  if (j <= p) return 0.0;
  if (j >= p + n) return 1.0;
  return double(j - p) / double(n);
}

// Values N[r] and first derivatives dN[r] of the p+1 B-splines N_{e+r} (0-based full index)
// that are nonzero on element e (knot span p+e) at x.
__device__ void basis_on_span(int p, int n, int e, double x, double* N, double* dN) {
  double ndu[MAXP + 1][MAXP + 1];
  double left[MAXP + 1], right[MAXP + 1];
  const int i = p + e;
  ndu[0][0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = x - knot(p, n, i + 1 - j);
    right[j] = knot(p, n, i + j) - x;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      ndu[j][r] = right[r + 1] + left[j - r];
      const double temp = ndu[r][j - 1] / ndu[j][r];
      ndu[r][j] = saved + right[r + 1] * temp;
      saved = left[j - r] * temp;
    }
    ndu[j][j] = saved;
  }
  for (int r = 0; r <= p; ++r) N[r] = ndu[r][p];
  // N'_{jj,p} = p (N_{jj,p-1}/(U[jj+p]-U[jj]) - N_{jj+1,p-1}/(U[jj+p+1]-U[jj+1])), jj = e + r
  for (int r = 0; r <= p; ++r) {
    const int jj = e + r;
    double d = 0.0;
    if (p >= 1) {
      if (r >= 1) {
        const double den = knot(p, n, jj + p) - knot(p, n, jj);
        if (den != 0.0) d += ndu[r - 1][p - 1] / den;
      }
      if (r <= p - 1) {
        const double den = knot(p, n, jj + p + 1) - knot(p, n, jj + 1);
        if (den != 0.0) d -= ndu[r][p - 1] / den;
      }
      d *= p;
    }
    dN[r] = d;
  }
}

struct GaussRule {
  int q;
  double x[MAXP + 2];
  double w[MAXP + 2];
};

__global__ void k_assemble_band(int p, int n, int m, GaussRule g, double* bM, double* bA, double* bS) {
  const int W = 2 * p + 1;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= m * W) return;
  const int k = idx / W, o = idx % W - p;
  const int kc = k + o;
  double vm = 0.0, va = 0.0, vs = 0.0;
  if (kc >= 0 && kc < m) {
    const int i1 = k + 1, i2 = kc + 1;          // 0-based full B-spline indices
    const int elo = max(max(i1, i2) - p, 0);    // N_i nonzero on elements i-p..i
    const int ehi = min(min(i1, i2), n - 1);
    double N[MAXP + 1], dN[MAXP + 1];
    for (int e = elo; e <= ehi; ++e) {
      for (int gq = 0; gq < g.q; ++gq) {
        const double x = (e + g.x[gq]) / n;
        const double w = g.w[gq] / n;
        basis_on_span(p, n, e, x, N, dN);
        const int r1 = i1 - e, r2 = i2 - e;
        vm += w * N[r1] * N[r2];
        va += w * N[r1] * dN[r2];
        vs += w * dN[r1] * dN[r2];
      }
    }
  }
  bM[idx] = vm;
  bA[idx] = va;
  bS[idx] = vs;
}

// Oslo recurrence: coefficient of fine B-spline i (1-based, knots tau) in coarse B-spline j
// (1-based, knots t).  alpha_{j,0}(i) = [t_j <= tau_i < t_{j+1}],
// alpha_{j,k}(i) = w_{j,k} alpha_{j,k-1}(i) + (1 - w_{j+1,k}) alpha_{j+1,k-1}(i),
// w_{jj,k} = (tau_{i+k} - t_jj)/(t_{jj+k} - t_jj)  (0 if the denominator vanishes).
__device__ double oslo_alpha(int p, int nc, int j, int i) {
  const int nf = 2 * nc;
  auto T = [&](int jj) { return knot(p, nc, jj - 1); };
  auto U = [&](int ii) { return knot(p, nf, ii - 1); };
  double a[MAXP + 2];
  const double ti = U(i);
  for (int r = 0; r <= p; ++r) a[r] = (T(j + r) <= ti && ti < T(j + r + 1)) ? 1.0 : 0.0;
  for (int k = 1; k <= p; ++k) {
    const double x = U(i + k);
    for (int r = 0; r <= p - k; ++r) {
      const int jj = j + r;
      const double d1 = T(jj + k) - T(jj), d2 = T(jj + k + 1) - T(jj + 1);
      const double w1 = d1 != 0.0 ? (x - T(jj)) / d1 : 0.0;
      const double w2 = d2 != 0.0 ? (x - T(jj + 1)) / d2 : 0.0;
      a[r] = w1 * a[r] + (1.0 - w2) * a[r + 1];
    }
  }
  return a[0];
}

__global__ void k_prolongation_dense(int p, int nc, int mf, int mc, double* P) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= mf * mc) return;
  const int kf = idx / mc, c = idx % mc;
  // interior fine k_f <-> full 1-based index kf+2; interior coarse c <-> coarse 1-based c+2
  P[idx] = oslo_alpha(p, nc, c + 2, kf + 2);
}

void gauss_legendre(int q, double* x01, double* w01) {
  // Newton iteration on the Legendre polynomial P_q (nodes to ~1e-16), mapped to [0,1]
  for (int i = 0; i < q; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (q + 0.5));
    double pp = 0.0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= q; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      if (q == 1) { p1 = z; p0 = 1.0; }
      pp = q * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / pp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= q; ++k) {
      const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    pp = q * (z * p1 - p0) / (z * z - 1.0);
    x01[i] = 0.5 * (1.0 - z);
    w01[i] = 1.0 / ((1.0 - z * z) * pp * pp);   // (2/((1-z^2)P'^2)) / 2
  }
}

void assemble_level(Handle& h, Level& L, cudaStream_t s) {
  const int p = h.p, m = L.m, W = 2 * p + 1;
  GaussRule g;
  g.q = p + 1;
  gauss_legendre(g.q, g.x, g.w);
  for (int f = 0; f < 3; ++f) IGACD_CUDA(cudaMalloc(&L.band[f], sizeof(double) * m * W));
  const int tot = m * W, bs = 128;
  k_assemble_band<<<(tot + bs - 1) / bs, bs, 0, s>>>(p, L.n, m, g, L.band[0], L.band[1], L.band[2]);
  IGACD_LAUNCH_CHECK();
  count_launch(h);
  for (int f = 0; f < 3; ++f) {
    L.hband[f].resize((size_t)m * W);
    IGACD_CUDA(cudaMemcpyAsync(L.hband[f].data(), L.band[f], sizeof(double) * m * W, cudaMemcpyDeviceToHost, s));
  }
  IGACD_CUDA(cudaStreamSynchronize(s));
  // Toeplitz rows: 2p-1 <= k <= m-2p (all band columns are cardinal B-splines)
  OpParams& op = L.geo;
  op.m = m;
  op.bM = L.band[0];
  op.bA = L.band[1];
  op.bS = L.band[2];
  op.zoneL = 2 * p - 1;
  op.zoneR = m - 2 * p + 1;
  if (op.zoneL >= op.zoneR) {  // no Toeplitz row: everything takes the band path
    op.zoneL = m;
    op.zoneR = m;
  }
  for (int o = 0; o <= MAXP; ++o) op.tM[o] = op.tA[o] = op.tS[o] = 0.0;
  if (op.zoneL < m) {
    const int k = op.zoneL;
    for (int o = 0; o <= p; ++o) {
      op.tM[o] = L.hband[0][(size_t)k * W + o + p];
      op.tA[o] = L.hband[1][(size_t)k * W + o + p];
      op.tS[o] = L.hband[2][(size_t)k * W + o + p];
    }
  }
  std::memset(&op.c, 0, sizeof(op.c));
}

void build_transfer(Handle& h, int p, int nc, Transfer1D& T, cudaStream_t s) {
  const int nf = 2 * nc;
  const int mf = nf + p - 2, mc = nc + p - 2;
  T.mf = mf;
  T.mc = mc;
  double* dP = nullptr;
  IGACD_CUDA(cudaMalloc(&dP, sizeof(double) * (size_t)mf * mc));
  const int tot = mf * mc, bs = 128;
  k_prolongation_dense<<<(tot + bs - 1) / bs, bs, 0, s>>>(p, nc, mf, mc, dP);
  IGACD_LAUNCH_CHECK();
  count_launch(h);
  T.hdense.resize((size_t)mf * mc);
  IGACD_CUDA(cudaMemcpyAsync(T.hdense.data(), dP, sizeof(double) * tot, cudaMemcpyDeviceToHost, s));
  IGACD_CUDA(cudaStreamSynchronize(s));
  IGACD_CUDA(cudaFree(dP));
  // fixed-width row storage of P and P^T (exact zeros of the recurrence are structural)
  std::vector<int> ps(mf), rs(mc);
  int wp = 1, wr = 1;
  for (int k = 0; k < mf; ++k) {
    int lo = mc, hi = -1;
    for (int c = 0; c < mc; ++c)
      if (T.hdense[(size_t)k * mc + c] != 0.0) { lo = std::min(lo, c); hi = std::max(hi, c); }
    if (hi < 0) { lo = 0; hi = 0; }
    ps[k] = lo;
    wp = std::max(wp, hi - lo + 1);
  }
  for (int c = 0; c < mc; ++c) {
    int lo = mf, hi = -1;
    for (int k = 0; k < mf; ++k)
      if (T.hdense[(size_t)k * mc + c] != 0.0) { lo = std::min(lo, k); hi = std::max(hi, k); }
    if (hi < 0) { lo = 0; hi = 0; }
    rs[c] = lo;
    wr = std::max(wr, hi - lo + 1);
  }
  std::vector<double> pw((size_t)mf * wp, 0.0), rw((size_t)mc * wr, 0.0);
  for (int k = 0; k < mf; ++k) {
    if (ps[k] + wp > mc) ps[k] = std::max(0, mc - wp);
    for (int t = 0; t < wp; ++t) {
      const int c = ps[k] + t;
      if (c < mc) pw[(size_t)k * wp + t] = T.hdense[(size_t)k * mc + c];
    }
  }
  for (int c = 0; c < mc; ++c) {
    if (rs[c] + wr > mf) rs[c] = std::max(0, mf - wr);
    for (int t = 0; t < wr; ++t) {
      const int k = rs[c] + t;
      if (k < mf) rw[(size_t)c * wr + t] = T.hdense[(size_t)k * mc + c];
    }
  }
  T.wp = wp;
  T.wr = wr;
  // widest input window of a tile of TO consecutive output rows (transfer.cu k_transfer2d)
  auto window = [](const std::vector<int>& st, int W, int nin, int TO) {
    int best = 1;
    for (size_t a = 0; a < st.size(); a += 1) {
      const size_t b = std::min(st.size(), a + TO) - 1;
      best = std::max(best, std::min(st[b] + W, nin) - st[a]);
    }
    return best;
  };
  T.pwin1 = window(ps, wp, mc, TRANSFER_TO1);
  T.pwin2 = window(ps, wp, mc, TRANSFER_TO2);
  T.rwin1 = window(rs, wr, mf, TRANSFER_TO1);
  T.rwin2 = window(rs, wr, mf, TRANSFER_TO2);
  IGACD_CUDA(cudaMalloc(&T.p_start, sizeof(int) * mf));
  IGACD_CUDA(cudaMalloc(&T.p_w, sizeof(double) * pw.size()));
  IGACD_CUDA(cudaMalloc(&T.r_start, sizeof(int) * mc));
  IGACD_CUDA(cudaMalloc(&T.r_w, sizeof(double) * rw.size()));
  IGACD_CUDA(cudaMemcpyAsync(T.p_start, ps.data(), sizeof(int) * mf, cudaMemcpyHostToDevice, s));
  IGACD_CUDA(cudaMemcpyAsync(T.p_w, pw.data(), sizeof(double) * pw.size(), cudaMemcpyHostToDevice, s));
  IGACD_CUDA(cudaMemcpyAsync(T.r_start, rs.data(), sizeof(int) * mc, cudaMemcpyHostToDevice, s));
  IGACD_CUDA(cudaMemcpyAsync(T.r_w, rw.data(), sizeof(double) * rw.size(), cudaMemcpyHostToDevice, s));
  IGACD_CUDA(cudaStreamSynchronize(s));
}

}  // namespace igacd

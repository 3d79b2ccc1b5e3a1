// C ABI of libigacd (include/igacd.h): setup, V-cycle (R6) and PCG (R7) drivers.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "internal.cuh"

namespace igacd {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// ---- operator coefficients ------------------------------------------------------------
// Reading R1: a(u,v) = nu (u,v) + beta lambda (div u, div v) + lambda (curl(b0 x u), curl(b0 x v)).
// For constant b0, curl(b0 x u) = b0 div u - (b0 . grad) u, so with test (i,b), trial (j,a)
//   K[(i,b),(j,a)] = beta lambda d_ib d_ja + lambda sum_m (b0_m d_ib - b0_b d_im)(b0_m d_ja - b0_a d_jm)
//                  = (beta lambda + lambda |b0|^2) d_ib d_ja
//                    + lambda (-d_ib b0_j b0_a - d_ja b0_i b0_b + d_ij b0_a b0_b).
// In 2D (u3 = 0, d/dx3 = 0, b0 in the plane) the same formula holds on indices {0,1}.
static void alfven_form(int d, double nu, double beta, double lam, const double* b0, double* mass, double* K) {
  double bb = 0.0;
  for (int a = 0; a < d; ++a) bb += b0[a] * b0[a];
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) mass[i * d + j] = (i == j) ? nu : 0.0;
  for (int i = 0; i < d; ++i)
    for (int b = 0; b < d; ++b)
      for (int j = 0; j < d; ++j)
        for (int a = 0; a < d; ++a) {
          const double dib = i == b, dja = j == a, dij = i == j;
          K[((i * d + b) * d + j) * d + a] = (beta * lam + lam * bb) * dib * dja +
                                            lam * (-dib * b0[j] * b0[a] - dja * b0[i] * b0[b] + dij * b0[a] * b0[b]);
        }
}

// Kronecker patterns (internal.cuh Coef) of a(u,v) = sum mass (u_j,v_i) + sum K (d_a u_j, d_b v_i).
// 1D factor per direction l: M if l not in {a,b}; S if l = a = b; A if l = a != b (derivative on
// the trial function, A_kj = int N_k N_j'); A^T = -A if l = b != a.  Hence the pattern A(x)A on
// the pair {k,l} collects -(K[(i,l),(j,k)] + K[(i,k),(j,l)]).
static Coef patterns(int d, const double* mass, const double* K) {
  Coef c;
  std::memset(&c, 0, sizeof(c));
  auto Kf = [&](int i, int b, int j, int a) { return K[((i * d + b) * d + j) * d + a]; };
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      c.mass[i][j] = mass[i * d + j];
      for (int l = 0; l < d; ++l) c.S[l][i][j] = Kf(i, l, j, l);
      int q = 0;
      for (int k = 0; k < d; ++k)
        for (int l = k + 1; l < d; ++l, ++q) c.AA[q][i][j] = -(Kf(i, l, j, k) + Kf(i, k, j, l));
    }
  return c;
}

// Reading R6: n_{l+1} = n_l/2 while n_l is even, n_l/2 + p - 2 >= 1 and d (n_l+p-2)^d > NCOARSE_MAX.
static std::vector<int> level_sizes(int d, int p, int n, int levels) {
  std::vector<int> ns{n};
  auto big = [&](int nn) {
    double m = nn + p - 2;
    return d * std::pow(m, d) > NCOARSE_MAX;
  };
  if (levels > 0) {
    for (int l = 1; l < levels; ++l) {
      if (ns.back() % 2 || ns.back() / 2 + p - 2 < 1)
        throw Error{IGACD_E_ARG, "requested number of levels impossible for this n and p"};
      ns.push_back(ns.back() / 2);
    }
    return ns;
  }
  while (ns.back() % 2 == 0 && ns.back() / 2 + p - 2 >= 1 && big(ns.back())) ns.push_back(ns.back() / 2);
  return ns;
}

// Cardinal B-spline phi_p(t), host side, for the entries of
// T_m(m_{p-1}): (i,j) -> phi_{2p-1}(p - i + j) for |i-j| < p.
static double cardinal_host(int p, double t) {
  if (p == 0) return (t >= 0.0 && t < 1.0) ? 1.0 : 0.0;
  return t / p * cardinal_host(p - 1, t) + (p + 1 - t) / p * cardinal_host(p - 1, t - 1.0);
}

static void build_toeplitz_factor(int p, Level& L) {
  const int m = L.m, w = p - 1;
  std::vector<double> F((size_t)m * (2 * w + 1), 0.0), Lb, inv;
  for (int i = 0; i < m; ++i)
    for (int o = -w; o <= w; ++o)
      if (i + o >= 0 && i + o < m) F[(size_t)i * (2 * w + 1) + o + w] = cardinal_host(2 * p - 1, p + o);
  band_cholesky(F, m, w, Lb, inv);
  L.T.upload(Lb, inv, m, w);
}

static void free_system(System& S) {
  for (int a = 0; a < 3; ++a) S.tf[a].release();
  for (auto& L : S.lv) {
    cudaFree(L.b);
    cudaFree(L.x);
    cudaFree(L.t);
    cudaFree(L.r);
  }
  cudaFree(S.cinv);
  S.lv.clear();
  S.cinv = nullptr;
}

static void destroy_handle(Handle* h) {
  if (!h) return;
  for (auto& L : h->lv) {
    for (int f = 0; f < 3; ++f) cudaFree(L.band[f]);
    L.T.release();
  }
  for (auto& T : h->tr) {
    cudaFree(T.p_start);
    cudaFree(T.p_w);
    cudaFree(T.r_start);
    cudaFree(T.r_w);
  }
  free_system(h->sys[0]);
  free_system(h->sys[1]);
  cudaFree(h->scratch0);
  cudaFree(h->scratch1);
  cudaFree(h->partial);
  cudaFree(h->scal);
  if (h->hscal) cudaFreeHost(h->hscal);
  for (double* v : {h->pr, h->pz, h->pp, h->pq, h->px, h->pb, h->aw, h->ar, h->zbuf, h->zbuf1}) cudaFree(v);
  for (double* v : {h->gm_v, h->gm_z, h->gm_partial, h->gm_dev}) cudaFree(v);
  if (h->gm_host) cudaFreeHost(h->gm_host);
  if (h->gA) cudaGraphExecDestroy(h->gA);
  if (h->gB) cudaGraphExecDestroy(h->gB);
  if (h->ga0) cudaEventDestroy(h->ga0);
  if (h->ga1) cudaEventDestroy(h->ga1);
  if (h->cap) cudaStreamDestroy(h->cap);
  if (h->aux_stream) cudaStreamDestroy(h->aux_stream);
  if (h->vec_stream) cudaStreamDestroy(h->vec_stream);
  if (h->ev_join2) cudaEventDestroy(h->ev_join2);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  for (auto& pr : h->ev_pending) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  delete h;
}

enum Slot { S_NORM = 0, S_PQ = 1, S_RR = 2, S_RZ0 = 3, S_RZ1 = 4, S_A = 5, S_B = 6, NSLOT = 8 };

static double reduce_to_host(Handle& h, int nparts, int slot, cudaStream_t s) {
  launch_finalize(h, h.partial, nparts, h.scal + slot, s);
  IGACD_CUDA(cudaMemcpyAsync(h.hscal + slot, h.scal + slot, sizeof(double), cudaMemcpyDeviceToHost, s));
  IGACD_CUDA(cudaStreamSynchronize(s));
  return h.hscal[slot];
}

// Reading R4: rho_l = (v, A v)/(v, D v) after POWER_STEPS normalised steps v <- D^-1 A v / ||.||
// from the counter-based start vector; omega_l = 4 / (3 * 1.05 * rho_l).
static void estimate_omega(Handle& h, int sy, int l, cudaStream_t s) {
  SysLevel& L = h.sys[sy].lv[l];
  double* v = L.x;
  double* w = L.t;
  launch_hash_vector(h, v, L.ndof, s);
  Epi ep{};
  ep.partial = h.partial;
  for (int it = 0; it < POWER_STEPS; ++it) {
    const int np = launch_operator(h, sy, l, v, w, EPI_DINV, DOT_OUT_OUT, ep, s);
    launch_finalize(h, h.partial, np, h.scal + S_NORM, s);
    launch_scale(h, w, h.scal + S_NORM, nullptr, L.ndof, s);
    std::swap(v, w);
  }
  const int np = launch_operator(h, sy, l, v, w, EPI_APPLY, DOT_X_OUT, ep, s);
  const double vAv = reduce_to_host(h, np, S_A, s);
  launch_dvdot(h, sy, l, v, h.partial, s);
  const double vDv = reduce_to_host(h, vec_ctas(L.ndof), S_B, s);
  L.rho = vAv / vDv;
  L.omega = 4.0 / (3.0 * 1.05 * L.rho);
}

static bool band_slab_enabled() {   // IGACD_BAND_SLAB=0: one tiled pass per direction in 3D too
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_BAND_SLAB");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// data <- T_l^{-1} src (T = I_nc (x) T(m_{p-1})^{(x) d}, reading R4'), mode as launch_band_solve
// (0: result in data; 1: xacc += omega * result; 2: xacc = omega * result).  3D: direction 0
// by the tiled kernel, directions 1 and 2 together by the slab kernel when a slab fits.
static void tinv(Handle& h, int sy, int l, const double* src, double* data, int mode, double omega, double* xacc,
                 cudaStream_t s) {
  const int nc = h.sys[sy].nc;
  const BandFactor& T = h.lv[l].T;
  if (h.dim == 3 && band_slab_enabled() && band_slab_fits(h.lv[l].m, T.w)) {
    launch_band_solve(h, nc, l, 0, T, data, 0, 0.0, nullptr, s, src);
    launch_band_solve_slab(h, nc, l, T, data, mode, omega, xacc, s);
    return;
  }
  for (int a = 0; a + 1 < h.dim; ++a) launch_band_solve(h, nc, l, a, T, data, 0, 0.0, nullptr, s, a == 0 ? src : nullptr);
  launch_band_solve(h, nc, l, h.dim - 1, T, data, mode, omega, xacc, s);
}

// z <- T^{-1} z (in place) for system sy at level l
static void apply_tinv(Handle& h, int sy, int l, double* z, cudaStream_t s) { tinv(h, sy, l, z, z, 0, 0.0, nullptr, s); }

// Reading R4': rho_t = ||T^{-1} A v|| after POWER_STEPS normalised steps v <- T^{-1} A v / ||.||
// from the counter-based start vector; omega_t = 4 / (3 * 1.05 * rho_t).
static void estimate_omega_t(Handle& h, int sy, int l, cudaStream_t s) {
  SysLevel& L = h.sys[sy].lv[l];
  double* v = L.x;
  double* w = L.t;
  launch_hash_vector(h, v, L.ndof, s);
  Epi ep{};
  const int nv = vec_ctas(L.ndof);
  double nrm = 0.0;
  for (int it = 0; it <= POWER_STEPS; ++it) {
    launch_operator(h, sy, l, v, w, EPI_APPLY, DOT_NONE, ep, s);
    apply_tinv(h, sy, l, w, s);
    launch_dot(h, w, w, L.ndof, h.partial, s);
    if (it == POWER_STEPS) {
      nrm = std::sqrt(reduce_to_host(h, nv, S_A, s));
      break;
    }
    launch_finalize(h, h.partial, nv, h.scal + S_NORM, s);
    launch_scale(h, w, h.scal + S_NORM, nullptr, L.ndof, s);
    std::swap(v, w);
  }
  L.rho_t = nrm;
  L.omega_t = 4.0 / (3.0 * 1.05 * L.rho_t);
}

static void setup_system(Handle& h, int sy, int nc, const Coef& coef, cudaStream_t s) {
  System& S = h.sys[sy];
  S.nc = nc;
  S.coef = coef;
  S.nu_pre = h.nu_pre;
  S.nu_post = h.nu_post;
  S.lv.resize(h.lv.size());
  for (size_t l = 0; l < h.lv.size(); ++l) {
    SysLevel& L = S.lv[l];
    L.op = h.lv[l].geo;
    L.op.c = coef;
    L.ndof = (size_t)nc * h.lv[l].nscal;
    IGACD_CUDA(cudaMalloc(&L.b, sizeof(double) * L.ndof));
    IGACD_CUDA(cudaMalloc(&L.x, sizeof(double) * L.ndof));
    IGACD_CUDA(cudaMalloc(&L.t, sizeof(double) * L.ndof));
    IGACD_CUDA(cudaMalloc(&L.r, sizeof(double) * L.ndof));
  }
  // the dense coarse inverse is built only when the coarsest level is small enough;
  // otherwise the system still applies its operator but refuses V-cycles
  if (S.lv.back().ndof <= COARSE_DENSE_MAX) build_coarse_inverse(h, sy, s);
  for (size_t l = 0; l + 1 < h.lv.size(); ++l) {
    estimate_omega(h, sy, (int)l, s);
    estimate_omega_t(h, sy, (int)l, s);
  }
}

// Reading R8: when A_s is a single Kronecker product (b0 along a coordinate axis l):
// A_s = (c_m M + c_s S)_l (x) M (x) ..; factor each 1D matrix once (level 0).
static void setup_aux_tensor(Handle& h, cudaStream_t s) {
  System& A = h.sys[1];
  const Coef& c = A.coef;
  int nS = 0, lS = -1;
  for (int l = 0; l < h.dim; ++l)
    if (c.S[l][0][0] != 0.0) { ++nS; lS = l; }
  bool aa = false;
  for (int q = 0; q < 3; ++q) aa = aa || c.AA[q][0][0] != 0.0;
  if (aa || nS > 1) return;
  const Level& L0 = h.lv[0];
  const int m = L0.m, p = h.p, W = 2 * p + 1;
  const int lead = lS >= 0 ? lS : 0;   // the direction that carries the scalar coefficients
  for (int a = 0; a < h.dim; ++a) {
    std::vector<double> F((size_t)m * W), Lb, inv;
    for (size_t k = 0; k < F.size(); ++k) {
      if (a != lead) F[k] = L0.hband[0][k];                                       // M
      else F[k] = c.mass[0][0] * L0.hband[0][k] + (lS >= 0 ? c.S[lS][0][0] * L0.hband[2][k] : 0.0);
    }
    band_cholesky(F, m, p, Lb, inv);
    A.tf[a].upload(Lb, inv, m, p);
  }
  A.tensor_exact = true;
}

// Reading R8: patterns of A_s = Pi^T A Pi, Pi s = b0 s:  C_s = sum_ij b0_i C[i][j] b0_j.
static Coef aux_patterns(int d, const Coef& c, const double* b0) {
  Coef a;
  std::memset(&a, 0, sizeof(a));
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) {
      const double w = b0[i] * b0[j];
      a.mass[0][0] += w * c.mass[i][j];
      for (int l = 0; l < 3; ++l) a.S[l][0][0] += w * c.S[l][i][j];
      for (int q = 0; q < 3; ++q) a.AA[q][0][0] += w * c.AA[q][i][j];
    }
  return a;
}

static Handle* create_impl(int dim, int p, int n, const double* mass, const double* K, const double* b0, int levels,
                           int nu_pre, int nu_post, cudaStream_t s) {
  if (dim != 2 && dim != 3) throw Error{IGACD_E_ARG, "dim must be 2 or 3"};
  if (p < 1 || p > MAXP) throw Error{IGACD_E_ARG, "p must be in [1, 6]"};
  if (n < 1 || n + p - 2 < 1) throw Error{IGACD_E_ARG, "need n >= 1 and n + p - 2 >= 1"};
  if (nu_pre < 0 || nu_post < 0) throw Error{IGACD_E_ARG, "negative sweep count"};
  Handle* h = new Handle();
  try {
    h->dim = dim;
    h->p = p;
    h->nu_pre = nu_pre;
    h->nu_post = nu_post;
    h->stream = s;
    double bb = 0.0;
    if (b0)
      for (int j = 0; j < dim; ++j) {
        h->b0[j] = b0[j];
        bb += b0[j] * b0[j];
      }
    const Coef coef = patterns(dim, mass, K);
    const std::vector<int> ns = level_sizes(dim, p, n, levels);
    if ((double)dim * std::pow((double)(n + p - 2), dim) >= 2147483647.0)
      throw Error{IGACD_E_ARG, "problem too large: d*m^d must stay below 2^31"};
    h->lv.resize(ns.size());
    for (size_t l = 0; l < ns.size(); ++l) {
      Level& L = h->lv[l];
      L.n = ns[l];
      L.m = ns[l] + p - 2;
      L.nscal = 1;
      for (int a = 0; a < dim; ++a) L.nscal *= (size_t)L.m;
      assemble_level(*h, L, s);
      build_toeplitz_factor(p, L);
    }
    h->tr.resize(ns.size() - 1);
    size_t scratch = 1;
    for (size_t l = 0; l + 1 < ns.size(); ++l) {
      build_transfer(*h, p, ns[l + 1], h->tr[l], s);
      const size_t mf = h->tr[l].mf, mc = h->tr[l].mc;
      scratch = std::max(scratch, dim == 2 ? (size_t)dim * mc * mf : (size_t)dim * mc * mf * mf);
    }
    h->scratch_len = scratch;
    IGACD_CUDA(cudaMalloc(&h->scratch0, sizeof(double) * scratch));
    IGACD_CUDA(cudaMalloc(&h->scratch1, sizeof(double) * scratch));
    size_t np = 1;
    if (dim == 3) {   // z workspaces of the split operator (the levels that take it): 3 nc m^3 doubles
      size_t zmax = 0, zmax1 = 0;
      for (const Level& L : h->lv) {
        const bool small = !apply3d_marching_pays(L.m) || split3d_forced();
        if (small || L.m % 2 == 1) zmax = std::max(zmax, L.nscal);
        if (small) zmax1 = std::max(zmax1, L.nscal);
      }
      if (zmax) IGACD_CUDA(cudaMalloc(&h->zbuf, sizeof(double) * 3 * (size_t)dim * zmax));
      if (zmax1) IGACD_CUDA(cudaMalloc(&h->zbuf1, sizeof(double) * 3 * zmax1));
    }
    for (size_t l = 0; l < ns.size(); ++l) {
      np = std::max(np, (size_t)operator_ctas(*h, (int)l));
      np = std::max(np, (size_t)vec_ctas((size_t)dim * h->lv[l].nscal));
    }
    h->partial_len = np;
    IGACD_CUDA(cudaMalloc(&h->partial, sizeof(double) * np));
    IGACD_CUDA(cudaMalloc(&h->scal, sizeof(double) * NSLOT));
    IGACD_CUDA(cudaMallocHost(&h->hscal, sizeof(double) * NSLOT));
    const size_t n0 = (size_t)dim * h->lv[0].nscal;
    for (double** v : {&h->pr, &h->pz, &h->pp, &h->pq, &h->aw, &h->ar}) IGACD_CUDA(cudaMalloc(v, sizeof(double) * n0));
    setup_system(*h, 0, dim, coef, s);
    // auxiliary space span{b0 s} (reading R8) when the b0-term is present
    const Coef ac = aux_patterns(dim, coef, h->b0);
    h->has_aux = bb > 0.0 && ac.mass[0][0] + ac.S[0][0][0] + ac.S[1][0][0] + ac.S[2][0][0] > 0.0;
    if (h->has_aux) {
      setup_system(*h, 1, 1, ac, s);
      setup_aux_tensor(*h, s);
    }
    // reading R8': the concurrent additive combination (measured time-to-solution)
    h->precond = h->has_aux ? PRECOND_AUX_ADD : PRECOND_VCYCLE;
    IGACD_CUDA(cudaStreamSynchronize(s));
  } catch (...) {
    destroy_handle(h);
    throw;
  }
  return h;
}

// ---- V-cycle ------------------------------------------------------------------------------
static void jacobi_sweeps(Handle& h, int sy, int l, const double* b, double*& cur, double*& oth, int sweeps,
                          double omega, cudaStream_t s) {
  Epi ep{};
  ep.omega = omega;
  ep.b = b;
  for (int k = 0; k < sweeps; ++k) {
    launch_operator(h, sy, l, cur, oth, EPI_JACOBI, DOT_NONE, ep, s);
    std::swap(cur, oth);
  }
}

// `sweeps` smoothing steps on x for A_l x = b (system sy).  from_zero: x is 0 on entry, so the
// first step needs no operator apply.  JACOBI (R4): x <- x + omega D^{-1}(b - A x), ping-pong
// buffers; TOEPLITZ (R4'): x <- x + omega_t T^{-1}(b - A x), T = T_n^p, in place.
static int smoother_of(const Handle& h, int sy) {   // the auxiliary system may use its own
  return (sy == 1 && h.aux_smoother >= 0) ? h.aux_smoother : h.smoother;
}

// the smoother on level l: TOEPLITZ_FINE is the paper's placement of T_n^p -- the finest
// level only -- with damped Jacobi on the coarser levels
static int level_smoother(const Handle& h, int sy, int l) {
  const int k = smoother_of(h, sy);
  if (k == SMOOTH_TOEPLITZ_FINE) return l == 0 ? SMOOTH_TOEPLITZ : SMOOTH_JACOBI;
  return k;
}

static void smooth(Handle& h, int sy, int l, const double* b, double*& cur, double*& oth, int sweeps, bool from_zero,
                   cudaStream_t s) {
  SysLevel& L = h.sys[sy].lv[l];
  if (sweeps <= 0) {
    if (from_zero) launch_zero(h, cur, L.ndof, s);
    return;
  }
  if (level_smoother(h, sy, l) == SMOOTH_JACOBI) {
    int k = 0;
    if (from_zero) {
      launch_scale_dinv(h, sy, l, b, cur, L.omega, s);   // first sweep from x = 0: x = omega D^-1 b
      k = 1;
    }
    jacobi_sweeps(h, sy, l, b, cur, oth, sweeps - k, L.omega, s);
    return;
  }
  Epi ep{};
  ep.b = b;
  for (int k = 0; k < sweeps; ++k) {
    // from x = 0 the residual is b: the first line solve reads b and the last one assigns
    // x = omega_t T^{-1} b (no copy of b, no zeroing of x)
    const bool first = k == 0 && from_zero;
    if (!first) launch_operator(h, sy, l, cur, L.r, EPI_RESID, DOT_NONE, ep, s);
    tinv(h, sy, l, first ? b : L.r, L.r, first ? 2 : 1, L.omega_t, cur, s);
  }
}

// x = V_l b from a zero initial guess (pre-smooth, residual,
// restrict, recurse, prolongate-and-correct, post-smooth).  The result lands in x.
static void vcycle_level(Handle& h, int sy, int l, const double* b, double* x, cudaStream_t s) {
  System& S = h.sys[sy];
  const int Lc = (int)S.lv.size() - 1;
  if (!S.cinv)
    throw Error{IGACD_E_ARG, "coarsest level too large for the dense coarse solver (" +
                                 std::to_string(S.lv.back().ndof) + " dofs); choose n divisible by a higher power of 2"};
  if (l == Lc) {
    launch_coarse_solve(h, sy, b, x, s);
    return;
  }
  SysLevel& L = S.lv[l];
  const int swaps = level_smoother(h, sy, l) == SMOOTH_JACOBI ? std::max(0, S.nu_pre - 1) + S.nu_post : 0;
  double* cur = (swaps % 2 == 0) ? x : L.t;
  double* oth = (cur == x) ? L.t : x;
  smooth(h, sy, l, b, cur, oth, S.nu_pre, true, s);
  Epi ep{};
  ep.b = b;
  launch_operator(h, sy, l, cur, L.r, EPI_RESID, DOT_NONE, ep, s);
  SysLevel& C = S.lv[l + 1];
  launch_restrict(h, S.nc, l, L.r, C.b, s);
  vcycle_level(h, sy, l + 1, C.b, C.x, s);
  launch_prolong(h, S.nc, l, C.x, cur, true, s);
  smooth(h, sy, l, b, cur, oth, S.nu_post, false, s);
  if (cur != x) launch_copy(h, cur, x, L.ndof, s);
}

// approximate (V-cycle) or exact (tensor, reading R8) solve of the auxiliary system at level 0
static void aux_solve(Handle& h, const double* sb, double* sx, cudaStream_t s) {
  System& A = h.sys[1];
  if (A.tensor_exact) {
    for (int a = 0; a < h.dim; ++a) launch_band_solve(h, 1, 0, a, A.tf[a], sx, 0, 0.0, nullptr, s, a == 0 ? sb : nullptr);
    return;
  }
  vcycle_level(h, 1, 0, sb, sx, s);
}

// Preconditioner action z = B r (reading R8).  PRECOND_VCYCLE: B = V.  PRECOND_AUX: the
// symmetric multiplicative combination of the auxiliary-space correction on span{b0 s}
// (B_s = scalar V-cycle of A_s = Pi^T A Pi) and the vector V-cycle:
//   z = Pi B_s Pi^T r;  z += V (r - A z);  z += Pi B_s Pi^T (r - A z).
static bool prio_enabled() {   // IGACD_PRIO=0: the vector branch at default priority
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_PRIO");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// IGACD_AUX_SHARE: percent of the resident CTA slots the persistent kernels of the scalar branch
// of the additive preconditioner may take (Handle::slot_share).  Measured on config 4
// (preconditioner application): 100 % 2.73 ms, 67 % 2.66 ms, 50 % 2.76 ms, 34 % 2.97 ms.
static int aux_slot_share() {
  static const int v = [] {
    const char* e = getenv("IGACD_AUX_SHARE");
    const int p = (e && *e) ? atoi(e) : 67;
    return std::min(100, std::max(1, p));
  }();
  return v;
}

static void precond_apply(Handle& h, const double* r, double* z, cudaStream_t s) {
  if (h.precond == PRECOND_VCYCLE || !h.has_aux) {
    vcycle_level(h, 0, 0, r, z, s);
    return;
  }
  System& A = h.sys[1];
  SysLevel& a0 = A.lv[0];
  Epi ep{};
  ep.b = r;
  if (h.precond == PRECOND_AUX_ADD) {   // additive (R8'): z = V r + Pi B_s Pi^T r
    // the two corrections are independent: the scalar branch runs on a second stream
    // (fork/join events; captured as parallel graph branches)
    // The vector V-cycle is the critical path: it runs on a high-priority stream so its
    // kernels take SMs first and the scalar branch fills the gaps (node priorities are kept
    // in the captured graphs, cudaGraphInstantiateFlagUseNodePriority).
    if (!h.aux_stream) {
      int lo = 0, hi = 0;
      IGACD_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      IGACD_CUDA(cudaStreamCreateWithPriority(&h.aux_stream, cudaStreamNonBlocking, lo));
      IGACD_CUDA(cudaStreamCreateWithPriority(&h.vec_stream, cudaStreamNonBlocking, prio_enabled() ? hi : lo));
      IGACD_CUDA(cudaEventCreateWithFlags(&h.ev_fork, cudaEventDisableTiming));
      IGACD_CUDA(cudaEventCreateWithFlags(&h.ev_join, cudaEventDisableTiming));
      IGACD_CUDA(cudaEventCreateWithFlags(&h.ev_join2, cudaEventDisableTiming));
    }
    IGACD_CUDA(cudaEventRecord(h.ev_fork, s));
    IGACD_CUDA(cudaStreamWaitEvent(h.aux_stream, h.ev_fork, 0));
    IGACD_CUDA(cudaStreamWaitEvent(h.vec_stream, h.ev_fork, 0));
    launch_pi_t(h, r, a0.b, h.aux_stream);
    h.slot_share = aux_slot_share();
    try {
      aux_solve(h, a0.b, a0.x, h.aux_stream);
    } catch (...) {
      h.slot_share = 100;
      throw;
    }
    h.slot_share = 100;
    IGACD_CUDA(cudaEventRecord(h.ev_join, h.aux_stream));
    vcycle_level(h, 0, 0, r, z, h.vec_stream);
    IGACD_CUDA(cudaEventRecord(h.ev_join2, h.vec_stream));
    IGACD_CUDA(cudaStreamWaitEvent(s, h.ev_join, 0));
    IGACD_CUDA(cudaStreamWaitEvent(s, h.ev_join2, 0));
    launch_pi(h, a0.x, z, true, s);
    return;
  }
  launch_pi_t(h, r, a0.b, s);
  aux_solve(h, a0.b, a0.x, s);
  launch_pi(h, a0.x, z, false, s);
  launch_operator(h, 0, 0, z, h.ar, EPI_RESID, DOT_NONE, ep, s);
  vcycle_level(h, 0, 0, h.ar, h.aw, s);
  launch_axpy_inplace(h, h.aw, z, h.lv.empty() ? 0 : h.sys[0].lv[0].ndof, s);
  launch_operator(h, 0, 0, z, h.ar, EPI_RESID, DOT_NONE, ep, s);
  launch_pi_t(h, h.ar, a0.b, s);
  aux_solve(h, a0.b, a0.x, s);
  launch_pi(h, a0.x, z, true, s);
}

// ---- PCG ---------------------------------------------------------------------------------
// Textbook PCG (R7; oracle krylov.pcg) with device-side scalars in fixed slots:
//   A:  q = A p, (p, q) -> pq;  x += alpha p, r -= alpha q (alpha = rz/pq), ||r||^2 -> host
//   B:  z = B r, (r, z) -> rz';  p = z + (rz'/rz) p;  rz <- rz'
// The host reads ||r||^2 after A (the stopping test) and launches B only when
// the iteration continues.  A and B are captured once as CUDA graphs (IGACD_GRAPH=0 runs the
// same kernels eagerly), so an iteration costs two graph launches and one host sync.
static bool graphs_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("IGACD_GRAPH");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static void graphs_reset(Handle& h) {
  if (h.gA) cudaGraphExecDestroy(h.gA);
  if (h.gB) cudaGraphExecDestroy(h.gB);
  h.gA = h.gB = nullptr;
  h.g_x = nullptr;
}

template <class F>
static cudaGraphExec_t capture(Handle& h, F&& body, long long* nk) {
  if (!h.cap) IGACD_CUDA(cudaStreamCreateWithFlags(&h.cap, cudaStreamNonBlocking));
  const long long before = h.launches;
  IGACD_CUDA(cudaStreamBeginCapture(h.cap, cudaStreamCaptureModeThreadLocal));
  cudaGraph_t g = nullptr;
  try {
    body(h.cap);
  } catch (...) {
    cudaStreamEndCapture(h.cap, &g);
    if (g) cudaGraphDestroy(g);
    h.launches = before;
    throw;
  }
  IGACD_CUDA(cudaStreamEndCapture(h.cap, &g));
  cudaGraphExec_t ex = nullptr;
  const cudaError_t e = cudaGraphInstantiate(&ex, g, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(g);
  IGACD_CUDA(e);
  *nk = h.launches - before;
  h.launches = before;
  return ex;
}

// an event record that becomes an event node when `s` is being captured
static void record_event(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  IGACD_CUDA(cudaStreamIsCapturing(s, &st));
  if (st == cudaStreamCaptureStatusActive) IGACD_CUDA(cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal));
  else IGACD_CUDA(cudaEventRecord(ev, s));
}

static void pcg_part_a(Handle& h, double* x, cudaStream_t s) {
  const size_t N = h.sys[0].lv[0].ndof;
  Epi ep{};
  ep.partial = h.partial;
  record_event(h.ga0, s);
  const int np = launch_operator(h, 0, 0, h.pp, h.pq, EPI_APPLY, DOT_X_OUT, ep, s);
  record_event(h.ga1, s);
  launch_finalize(h, h.partial, np, h.scal + S_PQ, s);
  launch_pcg_update_xr(h, x, h.pr, h.pp, h.pq, N, h.scal + S_RZ0, h.scal + S_PQ, h.partial, s);
  launch_finalize(h, h.partial, vec_ctas(N), h.scal + S_RR, s);
  // (p, A p) and ||r||^2 (adjacent slots) to the host: the stopping test and the breakdown check
  IGACD_CUDA(cudaMemcpyAsync(h.hscal + S_PQ, h.scal + S_PQ, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
}

static void pcg_part_b(Handle& h, cudaStream_t s) {
  const size_t N = h.sys[0].lv[0].ndof;
  precond_apply(h, h.pr, h.pz, s);
  launch_dot(h, h.pr, h.pz, N, h.partial, s);
  launch_finalize(h, h.partial, vec_ctas(N), h.scal + S_RZ1, s);
  launch_pcg_update_p(h, h.pp, h.pz, N, h.scal + S_RZ1, h.scal + S_RZ0, s);
  IGACD_CUDA(cudaMemcpyAsync(h.scal + S_RZ0, h.scal + S_RZ1, sizeof(double), cudaMemcpyDeviceToDevice, s));
}

static int pcg(Handle& h, const double* b, double* x, double tol, int maxit, int* iters, double* relres,
               cudaStream_t s) {
  const size_t N = h.sys[0].lv[0].ndof;
  const int nv = vec_ctas(N);
  if (!h.ga0) {
    IGACD_CUDA(cudaEventCreate(&h.ga0));
    IGACD_CUDA(cudaEventCreate(&h.ga1));
  }
  launch_copy(h, b, h.pr, N, s);
  launch_dot(h, h.pr, h.pr, N, h.partial, s);
  const double rr0 = reduce_to_host(h, nv, S_RR, s);
  launch_zero(h, x, N, s);
  const double r0 = std::sqrt(rr0);
  if (iters) *iters = 0;
  if (relres) *relres = 0.0;
  if (r0 == 0.0) return IGACD_OK;
  // first preconditioner application eagerly (also initialises every kernel's attributes)
  precond_apply(h, h.pr, h.pz, s);
  launch_dot(h, h.pr, h.pz, N, h.partial, s);
  launch_finalize(h, h.partial, nv, h.scal + S_RZ0, s);
  launch_copy(h, h.pz, h.pp, N, s);
  const bool use_graph = h.graphs && graphs_enabled();
  if (use_graph && h.g_x != x) {
    graphs_reset(h);
    h.gA = capture(h, [&](cudaStream_t cs) { pcg_part_a(h, x, cs); }, &h.nA);
    h.gB = capture(h, [&](cudaStream_t cs) { pcg_part_b(h, cs); }, &h.nB);
    h.g_x = x;
  }
  double rel = 1.0;
  int it = 0;
  for (it = 1; it <= maxit; ++it) {
    if (use_graph) {
      IGACD_CUDA(cudaGraphLaunch(h.gA, s));
      h.launches += h.nA;
    } else {
      pcg_part_a(h, x, s);
    }
    IGACD_CUDA(cudaStreamSynchronize(s));
    h.apply_launches++;
    if (h.profiling) {
      float ms = 0.f;
      IGACD_CUDA(cudaEventElapsedTime(&ms, h.ga0, h.ga1));
      h.apply_ms += ms;
    }
    rel = std::sqrt(h.hscal[S_RR]) / r0;
    // breakdown: A or B not SPD (p^T A p <= 0), or a non-finite value from the preconditioner
    if (!(h.hscal[S_PQ] > 0.0) || !std::isfinite(rel)) {
      if (iters) *iters = it;
      if (relres) *relres = rel;
      throw Error{IGACD_E_BREAKDOWN, "PCG breakdown at iteration " + std::to_string(it) +
                                         ": (p, A p) = " + std::to_string(h.hscal[S_PQ]) +
                                         ", relative residual " + std::to_string(rel)};
    }
    if (rel < tol || it == maxit) break;
    if (use_graph) {
      IGACD_CUDA(cudaGraphLaunch(h.gB, s));
      h.launches += h.nB;
    } else {
      pcg_part_b(h, s);
    }
  }
  if (iters) *iters = std::min(it, maxit);
  if (relres) *relres = rel;
  return rel < tol ? IGACD_OK : IGACD_E_NOCONV;
}

// ---- FGMRES ------------------------------------------------------------------------------
// Flexible right-preconditioned GMRES(restart) (the paper's PGMRES; oracle
// krylov.fgmres): z_j = B v_j (precond_apply), w = A z_j, CGS2 Arnoldi with fused multi-dot
// and multi-axpy kernels (coefficients stay on the device), Givens rotations of the small
// Hessenberg matrix on the host (one device->host copy per step, as PCG's residual check),
// x = Z y at convergence / restart; a restart recomputes the true residual b - A x.
static void gm_workspace(Handle& h, int restart) {
  if (h.gm_restart >= restart) return;
  for (double* v : {h.gm_v, h.gm_z, h.gm_partial, h.gm_dev}) cudaFree(v);
  if (h.gm_host) cudaFreeHost(h.gm_host);
  h.gm_v = h.gm_z = h.gm_partial = h.gm_dev = h.gm_host = nullptr;
  h.gm_restart = 0;
  const size_t N = h.sys[0].lv[0].ndof;
  IGACD_CUDA(cudaMalloc(&h.gm_v, sizeof(double) * N * (restart + 1)));
  IGACD_CUDA(cudaMalloc(&h.gm_z, sizeof(double) * N * restart));
  IGACD_CUDA(cudaMalloc(&h.gm_partial, sizeof(double) * MDOT * vec_ctas(N)));
  const size_t nd = 3 * (size_t)restart + 3;
  IGACD_CUDA(cudaMalloc(&h.gm_dev, sizeof(double) * nd));
  IGACD_CUDA(cudaMallocHost(&h.gm_host, sizeof(double) * nd));
  h.gm_restart = restart;
}

static int fgmres(Handle& h, const double* b, double* x, double tol, int maxit, int restart, int* iters,
                  double* relres, cudaStream_t s) {
  const size_t N = h.sys[0].lv[0].ndof;
  gm_workspace(h, restart);
  std::vector<const double*> V(restart + 1), Z(restart);
  for (int j = 0; j <= restart; ++j) V[j] = h.gm_v + (size_t)j * N;
  for (int j = 0; j < restart; ++j) Z[j] = h.gm_z + (size_t)j * N;
  double* dh1 = h.gm_dev;                  // [restart + 1]
  double* dh2 = dh1 + restart + 1;         // [restart + 1]
  double* dsq = dh2 + restart + 1;         // [1]
  double* dy = dsq + 1;                    // [restart]
  double* hh = h.gm_host;
  const int nv = vec_ctas(N);
  double* v0 = h.gm_v;
  launch_copy(h, b, v0, N, s);
  launch_zero(h, x, N, s);
  launch_dot(h, v0, v0, N, h.partial, s);
  const double r0 = std::sqrt(reduce_to_host(h, nv, S_RR, s));
  if (iters) *iters = 0;
  if (relres) *relres = 0.0;
  if (r0 == 0.0) return IGACD_OK;
  double beta = r0, rel = 1.0;
  int it = 0;
  std::vector<double> H((size_t)(restart + 1) * restart), g(restart + 1), cs(restart), sn(restart), y(restart);
  auto Hm = [&](int i, int j) -> double& { return H[(size_t)i * restart + j]; };
  Epi ep{};
  for (;;) {
    launch_scal(h, v0, 1.0 / beta, N, s);
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    int k = 0;
    bool done = false;
    for (int j = 0; j < restart; ++j) {
      double* zj = h.gm_z + (size_t)j * N;
      double* w = h.gm_v + (size_t)(j + 1) * N;
      precond_apply(h, V[j], zj, s);
      launch_operator(h, 0, 0, zj, w, EPI_APPLY, DOT_NONE, ep, s);
      ++it;
      launch_mdot(h, w, V.data(), j + 1, N, h.gm_partial, dh1, s);   // CGS2, pass 1
      launch_maxpy(h, w, V.data(), j + 1, dh1, -1.0, N, s);
      launch_mdot(h, w, V.data(), j + 1, N, h.gm_partial, dh2, s);   // pass 2
      launch_maxpy(h, w, V.data(), j + 1, dh2, -1.0, N, s);
      launch_dot(h, w, w, N, h.partial, s);
      launch_finalize(h, h.partial, nv, dsq, s);
      IGACD_CUDA(cudaMemcpyAsync(hh, h.gm_dev, sizeof(double) * (2 * (restart + 1) + 1), cudaMemcpyDeviceToHost, s));
      IGACD_CUDA(cudaStreamSynchronize(s));
      const double hn = std::sqrt(hh[2 * (restart + 1)]);
      for (int i = 0; i <= j; ++i) Hm(i, j) = hh[i] + hh[restart + 1 + i];
      if (j + 1 <= restart) Hm(j + 1, j) = hn;
      for (int i = 0; i < j; ++i) {   // previous rotations
        const double a = Hm(i, j), c = Hm(i + 1, j);
        Hm(i, j) = cs[i] * a + sn[i] * c;
        Hm(i + 1, j) = -sn[i] * a + cs[i] * c;
      }
      const double den = std::hypot(Hm(j, j), Hm(j + 1, j));
      if (!(den > 0.0) || !std::isfinite(den))
        throw Error{IGACD_E_BREAKDOWN, "GMRES breakdown at iteration " + std::to_string(it) +
                                           ": Givens denominator " + std::to_string(den)};
      cs[j] = Hm(j, j) / den;
      sn[j] = Hm(j + 1, j) / den;
      Hm(j, j) = den;
      Hm(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rel = std::fabs(g[j + 1]) / r0;
      k = j + 1;
      if (rel < tol || it >= maxit || hn == 0.0) {
        done = true;
        break;
      }
      launch_scal(h, w, 1.0 / hn, N, s);
    }
    for (int i = k - 1; i >= 0; --i) {   // back substitution H[:k,:k] y = g[:k]
      double acc = g[i];
      for (int l = i + 1; l < k; ++l) acc -= Hm(i, l) * y[l];
      y[i] = acc / Hm(i, i);
    }
    IGACD_CUDA(cudaMemcpyAsync(dy, y.data(), sizeof(double) * k, cudaMemcpyHostToDevice, s));
    launch_maxpy(h, x, Z.data(), k, dy, 1.0, N, s);
    IGACD_CUDA(cudaStreamSynchronize(s));   // y (pageable) is reused by the next cycle
    if (done) break;
    Epi er{};
    er.b = b;
    launch_operator(h, 0, 0, x, v0, EPI_RESID, DOT_NONE, er, s);
    launch_dot(h, v0, v0, N, h.partial, s);
    beta = std::sqrt(reduce_to_host(h, nv, S_RR, s));
    if (beta == 0.0) {
      rel = 0.0;
      break;
    }
  }
  if (iters) *iters = it;
  if (relres) *relres = rel;
  return rel < tol ? IGACD_OK : IGACD_E_NOCONV;
}

}  // namespace igacd

using namespace igacd;

#define API_BEGIN try {
#define API_END                          \
  }                                      \
  catch (const Error& e) {               \
    set_error(e.msg);                    \
    return e.code;                       \
  }                                      \
  catch (const std::exception& e) {      \
    set_error(e.what());                 \
    return IGACD_E_CUDA;                 \
  }                                      \
  return IGACD_OK;

static Handle* H(igacd_handle h) {
  if (!h) throw Error{IGACD_E_ARG, "null handle"};
  return reinterpret_cast<Handle*>(h);
}
static void check_level(Handle* h, int level, bool need_coarser = false) {
  if (level < 0 || level >= (int)h->lv.size() || (need_coarser && level + 1 >= (int)h->lv.size()))
    throw Error{IGACD_E_ARG, "level out of range"};
}
static void check_ptr(const void* p) {
  if (!p) throw Error{IGACD_E_ARG, "null pointer argument"};
}

extern "C" {

int igacd_create(igacd_handle* out, int dim, int p, int n, double nu, double beta, double lambda, const double* b0,
                 int levels, int nu_pre, int nu_post, void* stream) {
  API_BEGIN
  check_ptr(out);
  *out = nullptr;
  check_ptr(b0);
  if (dim != 2 && dim != 3) throw Error{IGACD_E_ARG, "dim must be 2 or 3"};
  if (!(nu >= 0 && beta >= 0 && lambda >= 0)) throw Error{IGACD_E_ARG, "nu, beta, lambda must be >= 0"};
  double mass[9], K[81];
  alfven_form(dim, nu, beta, lambda, b0, mass, K);
  *out = reinterpret_cast<igacd_handle>(
      create_impl(dim, p, n, mass, K, b0, levels, nu_pre, nu_post, (cudaStream_t)stream));
  API_END
}

int igacd_create_form(igacd_handle* out, int dim, int p, int n, const double* mass, const double* K, int levels,
                      int nu_pre, int nu_post, void* stream) {
  API_BEGIN
  check_ptr(out);
  *out = nullptr;
  check_ptr(mass);
  check_ptr(K);
  *out = reinterpret_cast<igacd_handle>(
      create_impl(dim, p, n, mass, K, nullptr, levels, nu_pre, nu_post, (cudaStream_t)stream));
  API_END
}

int igacd_destroy(igacd_handle h) {
  API_BEGIN
  if (h) {
    cudaDeviceSynchronize();
    destroy_handle(reinterpret_cast<Handle*>(h));
  }
  API_END
}

int igacd_get_info(igacd_handle h, int* dim, int* p, int* levels) {
  API_BEGIN
  Handle* hh = H(h);
  if (dim) *dim = hh->dim;
  if (p) *p = hh->p;
  if (levels) *levels = (int)hh->lv.size();
  API_END
}

int igacd_num_levels(igacd_handle h, int* levels) {
  API_BEGIN
  check_ptr(levels);
  *levels = (int)H(h)->lv.size();
  API_END
}

int igacd_level_n(igacd_handle h, int level, int* n) {
  API_BEGIN
  check_ptr(n);
  check_level(H(h), level);
  *n = H(h)->lv[level].n;
  API_END
}

int igacd_level_tsolve_passes(igacd_handle h, int level, int* passes) {
  API_BEGIN
  check_ptr(passes);
  check_level(H(h), level);
  const Handle& hh = *H(h);
  *passes = (hh.dim == 3 && band_slab_enabled() && band_slab_fits(hh.lv[level].m, hh.lv[level].T.w)) ? 2 : hh.dim;
  API_END
}

int igacd_ndof(igacd_handle h, int level, size_t* ndof) {
  API_BEGIN
  check_ptr(ndof);
  check_level(H(h), level);
  *ndof = H(h)->sys[0].lv[level].ndof;
  API_END
}

int igacd_smoother_omega(igacd_handle h, int level, double* omega, double* rho) {
  API_BEGIN
  check_level(H(h), level);
  Handle* hh = H(h);
  const SysLevel& L = hh->sys[0].lv[level];
  const bool t = level_smoother(*hh, 0, level) == SMOOTH_TOEPLITZ;
  if (omega) *omega = t ? L.omega_t : L.omega;
  if (rho) *rho = t ? L.rho_t : L.rho;
  API_END
}

int igacd_apply(igacd_handle h, int level, const double* x, double* y, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level);
  check_ptr(x);
  check_ptr(y);
  if (x == y) throw Error{IGACD_E_ARG, "x and y must not alias"};
  Epi ep{};
  launch_operator(*hh, 0, level, x, y, EPI_APPLY, DOT_NONE, ep, (cudaStream_t)stream);
  API_END
}

int igacd_residual(igacd_handle h, int level, const double* b, const double* x, double* r, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level);
  check_ptr(b);
  check_ptr(x);
  check_ptr(r);
  if (r == x || r == b) throw Error{IGACD_E_ARG, "r must not alias b or x"};
  Epi ep{};
  ep.b = b;
  launch_operator(*hh, 0, level, x, r, EPI_RESID, DOT_NONE, ep, (cudaStream_t)stream);
  API_END
}

int igacd_smooth(igacd_handle h, int level, const double* b, double* x, int sweeps, double omega, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level);
  check_ptr(b);
  check_ptr(x);
  if (sweeps < 0) throw Error{IGACD_E_ARG, "negative sweeps"};
  SysLevel& L = hh->sys[0].lv[level];
  const double w = omega > 0 ? omega : L.omega;
  if (!(w > 0)) throw Error{IGACD_E_ARG, "no smoother parameter on this level; pass omega > 0"};
  double* cur = x;
  double* oth = L.t;
  jacobi_sweeps(*hh, 0, level, b, cur, oth, sweeps, w, (cudaStream_t)stream);
  if (cur != x) launch_copy(*hh, cur, x, L.ndof, (cudaStream_t)stream);
  API_END
}

int igacd_tsolve(igacd_handle h, int level, const double* b, double* x, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level);
  check_ptr(b);
  check_ptr(x);
  if (b == x) throw Error{IGACD_E_ARG, "b and x must not alias"};
  tinv(*hh, 0, level, b, x, 0, 0.0, nullptr, (cudaStream_t)stream);
  API_END
}

int igacd_restrict(igacd_handle h, int level, const double* x_fine, double* x_coarse, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level, true);
  check_ptr(x_fine);
  check_ptr(x_coarse);
  launch_restrict(*hh, hh->dim, level, x_fine, x_coarse, (cudaStream_t)stream);
  API_END
}

int igacd_prolong(igacd_handle h, int level, const double* x_coarse, double* x_fine, int accumulate, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level, true);
  check_ptr(x_fine);
  check_ptr(x_coarse);
  launch_prolong(*hh, hh->dim, level, x_coarse, x_fine, accumulate != 0, (cudaStream_t)stream);
  API_END
}

int igacd_vcycle(igacd_handle h, const double* b, double* x, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_ptr(b);
  check_ptr(x);
  if (b == x) throw Error{IGACD_E_ARG, "b and x must not alias"};
  vcycle_level(*hh, 0, 0, b, x, (cudaStream_t)stream);
  API_END
}

int igacd_precond(igacd_handle h, const double* b, double* x, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_ptr(b);
  check_ptr(x);
  if (b == x) throw Error{IGACD_E_ARG, "b and x must not alias"};
  precond_apply(*hh, b, x, (cudaStream_t)stream);
  API_END
}

int igacd_set_preconditioner(igacd_handle h, int mode) {
  API_BEGIN
  Handle* hh = H(h);
  if (mode != PRECOND_VCYCLE && mode != PRECOND_AUX && mode != PRECOND_AUX_ADD)
    throw Error{IGACD_E_ARG, "unknown preconditioner"};
  if (mode != PRECOND_VCYCLE && !hh->has_aux) throw Error{IGACD_E_ARG, "no auxiliary space (b0 = 0 or lambda = 0)"};
  if (hh->precond != mode) graphs_reset(*hh);
  hh->precond = mode;
  API_END
}

int igacd_set_smoother(igacd_handle h, int kind) {
  API_BEGIN
  if (kind != SMOOTH_JACOBI && kind != SMOOTH_TOEPLITZ && kind != SMOOTH_TOEPLITZ_FINE)
    throw Error{IGACD_E_ARG, "unknown smoother"};
  if (H(h)->smoother != kind) graphs_reset(*H(h));
  H(h)->smoother = kind;
  API_END
}

int igacd_set_aux_sweeps(igacd_handle h, int nu_pre, int nu_post) {
  API_BEGIN
  Handle* hh = H(h);
  if (!hh->has_aux) throw Error{IGACD_E_ARG, "no auxiliary space on this handle"};
  if (nu_pre < 0 || nu_post < 0) throw Error{IGACD_E_ARG, "negative sweep count"};
  graphs_reset(*hh);
  hh->sys[1].nu_pre = nu_pre;
  hh->sys[1].nu_post = nu_post;
  API_END
}

int igacd_set_graphs(igacd_handle h, int enable) {
  API_BEGIN
  Handle* hh = H(h);
  if ((enable != 0) != hh->graphs) graphs_reset(*hh);
  hh->graphs = enable != 0;
  API_END
}

int igacd_set_aux_smoother(igacd_handle h, int kind) {
  API_BEGIN
  Handle* hh = H(h);
  if (!hh->has_aux) throw Error{IGACD_E_ARG, "no auxiliary space on this handle"};
  if (kind != -1 && kind != SMOOTH_JACOBI && kind != SMOOTH_TOEPLITZ && kind != SMOOTH_TOEPLITZ_FINE)
    throw Error{IGACD_E_ARG, "unknown smoother"};
  if (hh->aux_smoother != kind) graphs_reset(*hh);
  hh->aux_smoother = kind;
  API_END
}

int igacd_get_smoother(igacd_handle h, int* kind) {
  API_BEGIN
  check_ptr(kind);
  *kind = H(h)->smoother;
  API_END
}

int igacd_aux_is_exact(igacd_handle h, int* exact) {
  API_BEGIN
  check_ptr(exact);
  Handle* hh = H(h);
  *exact = hh->has_aux && hh->sys[1].tensor_exact ? 1 : 0;
  API_END
}

int igacd_get_preconditioner(igacd_handle h, int* mode) {
  API_BEGIN
  check_ptr(mode);
  *mode = H(h)->precond;
  API_END
}

int igacd_apply_aux(igacd_handle h, int level, const double* s_in, double* s_out, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level);
  check_ptr(s_in);
  check_ptr(s_out);
  if (!hh->has_aux) throw Error{IGACD_E_ARG, "no auxiliary space on this handle"};
  Epi ep{};
  launch_operator(*hh, 1, level, s_in, s_out, EPI_APPLY, DOT_NONE, ep, (cudaStream_t)stream);
  API_END
}

int igacd_aux_omega(igacd_handle h, int level, double* omega, double* rho) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level);
  if (!hh->has_aux) throw Error{IGACD_E_ARG, "no auxiliary space on this handle"};
  const SysLevel& L = hh->sys[1].lv[level];
  const bool t = level_smoother(*hh, 1, level) == SMOOTH_TOEPLITZ;
  if (omega) *omega = t ? L.omega_t : L.omega;
  if (rho) *rho = t ? L.rho_t : L.rho;
  API_END
}

int igacd_solve(igacd_handle h, const double* b, double* x, double tol, int maxit, int* iters, double* relres,
                void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_ptr(b);
  check_ptr(x);
  if (b == x) throw Error{IGACD_E_ARG, "b and x must not alias"};
  if (!(tol > 0) || maxit < 1) throw Error{IGACD_E_ARG, "need tol > 0 and maxit >= 1"};
  const int rc = pcg(*hh, b, x, tol, maxit, iters, relres, (cudaStream_t)stream);
  if (rc != IGACD_OK) {
    set_error("PCG reached maxit without the requested relative residual");
    return rc;
  }
  API_END
}


int igacd_gmres(igacd_handle h, const double* b, double* x, double tol, int maxit, int restart, int* iters,
                double* relres, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_ptr(b);
  check_ptr(x);
  if (b == x) throw Error{IGACD_E_ARG, "b and x must not alias"};
  if (!(tol > 0) || maxit < 1) throw Error{IGACD_E_ARG, "need tol > 0 and maxit >= 1"};
  if (restart < 1 || restart > 512) throw Error{IGACD_E_ARG, "restart must be in [1, 512]"};
  const int rc = fgmres(*hh, b, x, tol, maxit, restart, iters, relres, (cudaStream_t)stream);
  if (rc != IGACD_OK) {
    set_error("GMRES reached maxit without the requested relative residual");
    return rc;
  }
  API_END
}

int igacd_solve_host(igacd_handle h, const double* b_host, double* x_host, double tol, int maxit, int* iters,
                     double* relres, void* stream) {
  API_BEGIN
  Handle* hh = H(h);
  check_ptr(b_host);
  check_ptr(x_host);
  if (!(tol > 0) || maxit < 1) throw Error{IGACD_E_ARG, "need tol > 0 and maxit >= 1"};
  cudaStream_t s = (cudaStream_t)stream;
  const size_t N = hh->sys[0].lv[0].ndof;
  if (!hh->px) IGACD_CUDA(cudaMalloc(&hh->px, sizeof(double) * N));
  if (!hh->pb) IGACD_CUDA(cudaMalloc(&hh->pb, sizeof(double) * N));
  IGACD_CUDA(cudaMemcpyAsync(hh->pb, b_host, sizeof(double) * N, cudaMemcpyHostToDevice, s));
  const int rc = pcg(*hh, hh->pb, hh->px, tol, maxit, iters, relres, s);
  IGACD_CUDA(cudaMemcpyAsync(x_host, hh->px, sizeof(double) * N, cudaMemcpyDeviceToHost, s));
  IGACD_CUDA(cudaStreamSynchronize(s));
  if (rc != IGACD_OK) {
    set_error("PCG reached maxit without the requested relative residual");
    return rc;
  }
  API_END
}

int igacd_get_band(igacd_handle h, int level, int which, double* band_host) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level);
  check_ptr(band_host);
  if (which < 0 || which > 2) throw Error{IGACD_E_ARG, "which must be 0 (M), 1 (A) or 2 (S)"};
  const auto& v = hh->lv[level].hband[which];
  std::memcpy(band_host, v.data(), sizeof(double) * v.size());
  API_END
}

int igacd_get_prolongation(igacd_handle h, int level, double* P_host) {
  API_BEGIN
  Handle* hh = H(h);
  check_level(hh, level, true);
  check_ptr(P_host);
  const auto& v = hh->tr[level].hdense;
  std::memcpy(P_host, v.data(), sizeof(double) * v.size());
  API_END
}

int igacd_set_profiling(igacd_handle h, int enable) {
  API_BEGIN
  H(h)->profiling = enable != 0;
  API_END
}

int igacd_get_profile(igacd_handle h, long long* launches, long long* apply_launches, double* apply_ms) {
  API_BEGIN
  Handle* hh = H(h);
  if (launches) *launches = hh->launches;
  if (apply_launches) *apply_launches = hh->apply_launches;
  if (apply_ms) *apply_ms = hh->apply_ms;
  API_END
}

int igacd_reset_profile(igacd_handle h) {
  API_BEGIN
  Handle* hh = H(h);
  hh->launches = 0;
  hh->apply_launches = 0;
  hh->apply_ms = 0.0;
  API_END
}

const char* igacd_last_error(void) { return g_last_error.c_str(); }
const char* igacd_version(void) { return "igacd 0.1 (sm_100a)"; }

}  // extern "C"

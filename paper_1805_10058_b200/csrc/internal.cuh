// Internal declarations of libigacd (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "../../include/igacd.h"

namespace igacd {

constexpr int MAXP = 6;   // highest supported B-spline degree
constexpr int NCOARSE_MAX = 6000;  // reading R6: coarsen while d*m^d exceeds this
constexpr int POWER_STEPS = 30;    // reading R4: power steps for rho(D^-1 A)
constexpr size_t COARSE_DENSE_MAX = 8192;  // largest coarsest level given a dense inverse

// Operator patterns.  With 1D factors
// M, A (skew), S the Galerkin matrix is
//   A = sum_ij mass[i][j] M(x)M(x)M  +  sum_l S[l][i][j] (S in direction l, M elsewhere)
//       + sum_q AA[q][i][j] (A in both directions of pair q, M elsewhere),
// pairs q: 0 = (0,1), 1 = (0,2), 2 = (1,2); directions 0-based, 0 slowest.
// (There are no single-A patterns: the forms have no value-derivative products.)
struct Coef {
  double mass[3][3];
  double S[3][3][3];
  double AA[3][3][3];
};

// Kernel view of one level's 1D factors (same in every direction: n_1 = .. = n_d = n).
struct OpParams {
  int m;             // interior B-splines per direction
  int zoneL, zoneR;  // rows k < zoneL or k >= zoneR are not Toeplitz (boundary zone)
  const double* bM;  // band storage [m][2p+1], F[k][k+o] at k*(2p+1)+o+p
  const double* bA;
  const double* bS;
  double tM[MAXP + 1], tA[MAXP + 1], tS[MAXP + 1];  // Toeplitz row F[k][k+o], o = 0..p
  Coef c;
};

// Epilogue of the fused operator kernels.
enum EpiMode { EPI_APPLY = 0, EPI_RESID = 1, EPI_JACOBI = 2, EPI_DINV = 3 };
enum DotMode { DOT_NONE = 0, DOT_X_OUT = 1, DOT_OUT_OUT = 2 };

struct Epi {
  double omega;       // EPI_JACOBI
  const double* b;    // EPI_RESID, EPI_JACOBI
  double* partial;    // per-CTA partial sums when a DotMode is requested
};

struct Transfer1D {   // 1D prolongation P (m_f x m_c) in fixed-width row storage
  int mf = 0, mc = 0;
  int wp = 0, wr = 0;           // max nonzeros per P row / per P^T row
  int* p_start = nullptr;       // [mf]  first coarse column of fine row k
  double* p_w = nullptr;        // [mf][wp]
  int* r_start = nullptr;       // [mc]  first fine column of coarse row c (row of P^T)
  double* r_w = nullptr;        // [mc][wr]
  std::vector<double> hdense;   // host dense copy (debug/parity)
  // input-window sizes of a TRANSFER_TO1 (TO2) output tile, for P (p*) and P^T (r*)
  int pwin1 = 0, pwin2 = 0, rwin1 = 0, rwin2 = 0;
};
constexpr int TRANSFER_TO1 = 16, TRANSFER_TO2 = 32;   // k_transfer2d output tile

// Banded Cholesky factor F = L L^T on the device (linesolve.cu).
struct BandFactor {
  int m = 0, w = 0;
  double* Lb = nullptr;    // [m][w+1]: L[k][k-j] at k*(w+1) + (w-j)
  double* inv = nullptr;   // [m]: 1/L[k][k]
  double* fac = nullptr;   // [(2(w+1)+1) m]: scaled forward/backward coefficients and 1/L[k][k] (tiled kernel)
  int kc = 0;              // rows k >= kc of L (and 1/L[k][k]) are bitwise equal to the last row
  void upload(const std::vector<double>& Lb_h, const std::vector<double>& inv_h, int m_, int w_);
  void release();
};

// Geometry of one level (shared by the vector system and the auxiliary scalar system).
struct Level {
  int n = 0, m = 0;
  size_t nscal = 0;
  double* band[3] = {nullptr, nullptr, nullptr};  // M, A, S
  std::vector<double> hband[3];
  OpParams geo;  // m, zones, bands, Toeplitz rows (coefficients filled per system)
  BandFactor T;  // Cholesky factor of T_{m}(m_{p-1}), the smoother's 1D factor
};

enum Smoother { SMOOTH_JACOBI = 0, SMOOTH_TOEPLITZ = 1, SMOOTH_TOEPLITZ_FINE = 2 };

// Per-level state of one system.
struct SysLevel {
  OpParams op;         // geometry of the level + this system's pattern coefficients
  size_t ndof = 0;
  double rho = 0.0, omega = 0.0;     // damped Jacobi (reading R4)
  double rho_t = 0.0, omega_t = 0.0; // Toeplitz-preconditioned Richardson (reading R4')
  double* b = nullptr;  // work vectors (ndof each)
  double* x = nullptr;
  double* t = nullptr;
  double* r = nullptr;
};

// A linear system on the level hierarchy: the d-component operator A (nc = d) or the
// auxiliary scalar operator A_s = Pi^T A Pi on span{b0 s} (nc = 1), reading R8.
struct System {
  int nc = 0;
  int nu_pre = 1, nu_post = 1;   // smoothing sweeps of this system's V-cycle
  Coef coef;
  std::vector<SysLevel> lv;
  double* cinv = nullptr;   // dense inverse of the coarsest level
  // exact tensor inverse of the level-0 operator when it is a single Kronecker product
  // (auxiliary system with b0 along a coordinate axis): one factor per direction
  bool tensor_exact = false;
  BandFactor tf[3];
};

enum Precond { PRECOND_VCYCLE = 0, PRECOND_AUX = 1, PRECOND_AUX_ADD = 2 };

struct Handle {
  int dim = 0, p = 0;
  int nu_pre = 1, nu_post = 1;
  double b0[3] = {0, 0, 0};
  std::vector<Level> lv;
  std::vector<Transfer1D> tr;   // tr[l]: level l+1 -> level l
  System sys[2];                // 0: vector operator, 1: auxiliary scalar operator
  bool has_aux = false;
  int precond = PRECOND_VCYCLE;
  int smoother = SMOOTH_TOEPLITZ;
  int aux_smoother = -1;        // smoother of the auxiliary V-cycle (-1: the same as `smoother`)
  // transfer scratch (max size), reductions
  double* scratch0 = nullptr;   // vector-system transfers
  double* scratch1 = nullptr;   // scalar-system transfers (the additive branch runs concurrently)
  size_t scratch_len = 0;
  double* partial = nullptr;    // per-CTA partial sums
  size_t partial_len = 0;
  double* scal = nullptr;       // device scalars
  double* hscal = nullptr;      // pinned host mirror
  // PCG / preconditioner vectors (level-0 size)
  double *pr = nullptr, *pz = nullptr, *pp = nullptr, *pq = nullptr, *px = nullptr, *pb = nullptr;
  double *aw = nullptr, *ar = nullptr;   // aux preconditioner work (level-0 vector size)
  double* zbuf = nullptr;                // 3D split operator (split3d.cu): 3 nc per-point combinations
  double* zbuf1 = nullptr;               // the same for the scalar system (it may run concurrently)
  // share (percent) of the resident CTA slots a persistent kernel may take: 100 except inside the
  // scalar branch of the additive preconditioner, whose low-priority persistent kernels would
  // otherwise fill every SM and hold up the vector branch (a running CTA is never preempted)
  int slot_share = 100;
  // FGMRES workspace (allocated on first use): Arnoldi basis V [restart+1][N], Z [restart][N]
  int gm_restart = 0;
  double* gm_v = nullptr;
  double* gm_z = nullptr;
  double* gm_partial = nullptr;   // MDOT * vec_ctas(N)
  double* gm_dev = nullptr;       // [h1 (r+1) | h2 (r+1) | ||w||^2 | y (r)]
  double* gm_host = nullptr;      // pinned mirror
  cudaStream_t stream = nullptr;
  // CUDA graphs of the PCG iteration (api.cu): A = apply + x/r update + ||r||^2 -> host,
  // B = preconditioner + (r, z) + p update; captured on `cap`, replayed on the caller's stream
  cudaStream_t aux_stream = nullptr;          // concurrent branch of the additive preconditioner
  cudaStream_t vec_stream = nullptr;          // its critical branch (vector V-cycle), high priority
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_join2 = nullptr;
  bool graphs = true;               // igacd_set_graphs (and IGACD_GRAPH=0 in the environment)
  cudaStream_t cap = nullptr;
  cudaGraphExec_t gA = nullptr, gB = nullptr;
  long long nA = 0, nB = 0;         // kernels per replay
  const double* g_x = nullptr;      // solution pointer baked into gA
  cudaEvent_t ga0 = nullptr, ga1 = nullptr;   // apply timing inside gA
  // instrumentation
  long long launches = 0, apply_launches = 0;
  double apply_ms = 0.0;
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pending;
};

// ---- error handling ---------------------------------------------------------------
void set_error(const std::string& msg);
struct Error {
  int code;
  std::string msg;
};

#define IGACD_CUDA(call)                                                                   \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      throw ::igacd::Error{IGACD_E_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
  } while (0)

#define IGACD_LAUNCH_CHECK() IGACD_CUDA(cudaGetLastError())

// ---- assembly.cu --------------------------------------------------------------------
void assemble_level(Handle& h, Level& L, cudaStream_t s);
void build_transfer(Handle& h, int p, int n_coarse, Transfer1D& T, cudaStream_t s);
void gauss_legendre(int q, double* x01, double* w01);

// ---- apply.cu -----------------------------------------------------------------------
// out = epilogue(A x) for system `sy`; returns the number of CTAs that wrote partial sums
// (0 if dot == DOT_NONE)
int launch_operator(Handle& h, int sy, int level, const double* x, double* out, EpiMode mode, DotMode dot,
                    const Epi& epi, cudaStream_t s);
int operator_ctas(const Handle& h, int level);                  // max over both systems
int operator_ctas_sys(const Handle& h, int level, int nc);

// ---- apply3d.cu ---------------------------------------------------------------------------
// y = epilogue(A x) in 3D (one persistent fused kernel per apply); returns the CTAs launched
// (= partial sums written when a DotMode is requested); apply3d_ctas: upper bound for a level
int launch_apply3d(int p, int nc, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                   cudaStream_t s, int slot_share = 100);
int apply3d_ctas(int p, int nc, int m);
bool apply3d_marching_pays(int m);


// ---- split3d.cu: the vector system's slab + column kernels (z through zbuf), odd-m levels ---
bool split3d_forced();   // IGACD_SPLIT=1: on every level (comparison)
int split3d_ctas(int m);
void launch_split3d(int p, int nc, const OpParams& op, const Epi& ep, int mode, int dot, const double* x, double* y,
                    double* Z, cudaStream_t s);

// ---- transfer.cu --------------------------------------------------------------------
void launch_prolong(Handle& h, int nc, int level, const double* xc, double* xf, bool accumulate, cudaStream_t s);
void launch_restrict(Handle& h, int nc, int level, const double* xf, double* xc, cudaStream_t s);
// auxiliary-space maps: s = Pi^T v = sum_j b0_j v_j;  v (+)= Pi s = b0 s
void launch_pi_t(Handle& h, const double* v, double* sc, cudaStream_t s);
void launch_pi(Handle& h, const double* sc, double* v, bool accumulate, cudaStream_t s);

// ---- coarse.cu ----------------------------------------------------------------------
void build_coarse_inverse(Handle& h, int sy, cudaStream_t s);
void launch_coarse_solve(Handle& h, int sy, const double* b, double* x, cudaStream_t s);

// ---- vec.cu -------------------------------------------------------------------------
int vec_ctas(size_t n);
void launch_dot(Handle& h, const double* a, const double* b, size_t n, double* partial, cudaStream_t s);
void launch_finalize(Handle& h, const double* partial, int nparts, double* dst, cudaStream_t s);
void launch_scale_dinv(Handle& h, int sy, int level, const double* b, double* x, double omega, cudaStream_t s);
void launch_copy(Handle& h, const double* a, double* b, size_t n, cudaStream_t s);
void launch_zero(Handle& h, double* a, size_t n, cudaStream_t s);
void launch_axpy_inplace(Handle& h, const double* a, double* b, size_t n, cudaStream_t s);   // b += a
void launch_scale(Handle& h, double* a, const double* scal_num, const double* scal_den, size_t n, cudaStream_t s);
void launch_dvdot(Handle& h, int sy, int level, const double* v, double* partial, cudaStream_t s);
void launch_hash_vector(Handle& h, double* v, size_t n, cudaStream_t s);
// PCG fused updates (scalars on device: scal[...])
void launch_pcg_update_xr(Handle& h, double* x, double* r, const double* p, const double* q, size_t n,
                          const double* rz, const double* pq, double* partial, cudaStream_t s);
void launch_pcg_update_p(Handle& h, double* p, const double* z, size_t n, const double* rz_new,
                         const double* rz_old, cudaStream_t s);
// GMRES (Arnoldi): dst[j] = (w, V[j]) for j < nv (partial: MDOT * vec_ctas(n) doubles);
// w += sign * sum_j c[j] V[j] (c on the device);  a *= f
constexpr int MDOT = 8;
void launch_mdot(Handle& h, const double* w, const double* const* V, int nv, size_t n, double* partial, double* dst,
                 cudaStream_t s);
void launch_maxpy(Handle& h, double* w, const double* const* V, int nv, const double* c, double sign, size_t n,
                  cudaStream_t s);
void launch_scal(Handle& h, double* a, double f, size_t n, cudaStream_t s);

// ---- linesolve.cu -------------------------------------------------------------------
void band_cholesky(const std::vector<double>& F, int m, int w, std::vector<double>& Lb, std::vector<double>& inv);
// data <- F^{-1} src along `axis` (src = nullptr: in place).  mode 0: result in data;
// mode 1: xacc += omega * result; mode 2: xacc = omega * result (data then holds the
// forward-substitution intermediate in modes 1, 2)
void launch_band_solve(Handle& h, int nc, int level, int axis, const BandFactor& F, double* data, int mode,
                       double omega, double* xacc, cudaStream_t s, const double* src = nullptr);
// 3D: directions 1 and 2 of every [m][m] slab in one shared-memory pass (same modes)
bool band_slab_fits(int m, int w);
void launch_band_solve_slab(Handle& h, int nc, int level, const BandFactor& F, double* data, int mode, double omega,
                            double* xacc, cudaStream_t s, const double* src = nullptr);

// ---- common.cu (device properties and kernel attributes, per device and thread-safe) -----
int num_sms();                                                  // SMs of the current device
void ensure_smem_attr(const void* func, size_t bytes);          // max dynamic shared memory >= bytes
int max_active_blocks(const void* func, int threads, size_t smem);   // occupancy (cached)

inline void count_launch(Handle& h) { h.launches++; }

}  // namespace igacd

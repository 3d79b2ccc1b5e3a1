/*
 * igacd.h -- C ABI of the B200 IgA curl-div solver (libigacd.so).
 *
 * Operator (reading R1): the Galerkin matrix of the Alfven-like operator
 *   L_A u = nu u - beta*lambda grad(div u) - lambda b0 x (curl curl (b0 x u))
 * with homogeneous Dirichlet conditions imposed strongly, discretised with
 * tensor-product B-splines of degree p on n uniform elements per direction of (0,1)^d,
 * d = 2 or 3:
 *   a(u,v) = nu (u,v) + beta*lambda (div u, div v) + lambda (curl(b0 x u), curl(b0 x v)).
 *
 * VECTORS.  Every vector argument is a plain array of doubles of length igacd_ndof(h, level)
 * = d * m^d, m = n_level + p - 2 (the interior B-splines N_2..N_{n+p-1}),
 * component-major, then lexicographic with direction 1 slowest:
 *   index(j, k_1, .., k_d) = j*m^d + (..(k_1*m + k_2)*m + ..) + k_d.
 * Unless a name says _host, pointers are CUDA DEVICE pointers owned by the caller; the
 * library never frees them.  Input and output buffers must not alias unless stated.
 *
 * STREAMS.  `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 * All work is enqueued on it; functions return without synchronising except where stated
 * (igacd_create, igacd_solve, igacd_solve_host, queries).
 *
 * ERRORS.  Every function returns an int status: 0 = success, < 0 = failure
 * (IGACD_E_* below).  igacd_last_error() returns a thread-local message for the last failure.
 * A failure leaves caller-owned buffers in an unspecified state; the handle stays valid
 * unless igacd_create itself failed (then *out is NULL).
 */
#ifndef IGACD_H
#define IGACD_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IGACD_OK 0
#define IGACD_E_ARG (-1)      /* invalid argument (dimension, degree, size, null pointer)  */
#define IGACD_E_CUDA (-2)     /* a CUDA runtime call or kernel launch failed                */
#define IGACD_E_NOTSPD (-3)   /* coarse Cholesky met a non-positive pivot                    */
#define IGACD_E_NOCONV (-4)   /* igacd_solve reached maxit without the requested residual   */
#define IGACD_E_BREAKDOWN (-5) /* Krylov breakdown: (p, A p) <= 0, a zero Givens denominator, or
                                  a non-finite residual (operator or preconditioner not SPD / NaN) */

typedef struct igacd_handle_s* igacd_handle;

/* Build the hierarchy for the operator above.
 *   dim    2 or 3;   p  degree, 1 <= p <= 6;   n  elements per direction, n + p - 2 >= 1
 *   nu, beta, lambda  >= 0 (nu > 0, beta in (1e-4, 1e-1], lambda = V_A dt)
 *   b0     host array of `dim` doubles, used as given (the configs pass unit vectors)
 *   levels 0 = automatic coarsening rule (reading R6), else exactly `levels` levels
 *   nu_pre, nu_post  smoothing sweeps before / after the coarse correction, of whichever
 *          smoother is active (default T_n^p Richardson, reading R4'; damped Jacobi, R4)
 * Work: 1D assembly (R1) and knot-insertion (R3) kernels, coarse inverse (R5), smoother
 * parameters by power iteration (R4, R4').  Synchronises `stream`.  Owns all its device memory. */
int igacd_create(igacd_handle* out, int dim, int p, int n, double nu, double beta, double lambda,
                 const double* b0, int levels, int nu_pre, int nu_post, void* stream);

/* Same, for a general constant-coefficient form a(u,v) = sum_ij mass[i][j] (u_j, v_i)
 *   + sum_{i,b,j,a} K[((i*dim+b)*dim+j)*dim+a] (d_a u_j, d_b v_i)   (test (i,b), trial (j,a),
 * directions 0-based, host arrays of dim^2 and dim^4 doubles).  The matrix must be SPD.
 * Used for the paper's model form alpha curl-curl + beta div-div (eq:curl-div). */
int igacd_create_form(igacd_handle* out, int dim, int p, int n, const double* mass, const double* K,
                      int levels, int nu_pre, int nu_post, void* stream);

int igacd_destroy(igacd_handle h);

/* Queries (host values; no device work). */
int igacd_get_info(igacd_handle h, int* dim, int* p, int* levels);
int igacd_num_levels(igacd_handle h, int* levels);
int igacd_level_n(igacd_handle h, int level, int* n);
int igacd_ndof(igacd_handle h, int level, size_t* ndof);
/* Line-solve passes of one T_n^p solve on `level` (reading R4'): dim, or 2
 * in 3D when directions 1 and 2 of every [m][m] slab are solved in one shared-memory pass. */
int igacd_level_tsolve_passes(igacd_handle h, int level, int* passes);
/* omega and rho of the active smoother on `level` (Jacobi: rho(D^-1 A); Toeplitz: rho(T^-1 A)). */
int igacd_smoother_omega(igacd_handle h, int level, double* omega, double* rho);

/* y = A_level x   (R2).  x, y device, length igacd_ndof(h, level); x != y. */
int igacd_apply(igacd_handle h, int level, const double* x, double* y, void* stream);

/* r = b - A_level x   (R2 with the residual epilogue). */
int igacd_residual(igacd_handle h, int level, const double* b, const double* x, double* r, void* stream);

/* `sweeps` damped-Jacobi sweeps x <- x + omega_l D_l^{-1} (b - A_l x) in place on x (R4),
 * whatever smoother the V-cycle uses.  omega_l = the Jacobi parameter of the level unless
 * omega > 0 is given (then used as is). */
int igacd_smooth(igacd_handle h, int level, const double* b, double* x, int sweeps, double omega, void* stream);

/* x = T_l^{-1} b on `level` for the vector system: the smoother's preconditioner
 * T_n^p = I_d (x) T(m_{p-1}) (x) .. (x) T(m_{p-1}) (reading R4'), applied as
 * banded Cholesky line solves along each direction.  b, x: device, d*m^d doubles, no aliasing. */
int igacd_tsolve(igacd_handle h, int level, const double* b, double* x, void* stream);

/* x_coarse = P_level^T x_fine   (R3, restriction to level+1; PAPER.md:1111 R = P^T).
 * x_fine: igacd_ndof(h, level) doubles, x_coarse: igacd_ndof(h, level+1) doubles, device. */
int igacd_restrict(igacd_handle h, int level, const double* x_fine, double* x_coarse, void* stream);

/* x_fine = P_level x_coarse (accumulate == 0) or x_fine += P_level x_coarse (accumulate != 0). */
int igacd_prolong(igacd_handle h, int level, const double* x_coarse, double* x_fine, int accumulate, void* stream);

/* One V-cycle of the vector operator from a zero initial guess: x = V b (R6). */
int igacd_vcycle(igacd_handle h, const double* b, double* x, void* stream);

/* The PCG preconditioner action x = B b (reading R8).  Mode IGACD_PRECOND_VCYCLE: B = V.
 * Mode IGACD_PRECOND_AUX: symmetric multiplicative
 * combination of the auxiliary-space correction on span{b0 s} -- the kernel of the lambda
 * term -- with the V-cycle:  x = Pi Vs Pi^T b;  x += V(b - A x);  x += Pi Vs Pi^T (b - A x),
 * Pi s = b0 s, Vs = V-cycle of the scalar operator A_s = Pi^T A Pi on the same levels.
 * Mode IGACD_PRECOND_AUX_ADD (the default when b0 != 0 and lambda > 0, reading R8'):
 * x = V b + Pi Vs Pi^T b, the two terms computed concurrently on two streams. */
#define IGACD_PRECOND_VCYCLE 0
#define IGACD_PRECOND_AUX 1
#define IGACD_PRECOND_AUX_ADD 2
int igacd_precond(igacd_handle h, const double* b, double* x, void* stream);
int igacd_set_preconditioner(igacd_handle h, int mode);
int igacd_get_preconditioner(igacd_handle h, int* mode);

/* V-cycle smoother (both systems, all levels but the coarsest):
 *   IGACD_SMOOTH_JACOBI   (reading R4)  x <- x + omega_l D_l^{-1} (b - A_l x)
 *   IGACD_SMOOTH_TOEPLITZ (reading R4', default) x <- x + omega_t,l T^{-1} (b - A_l x) with the
 *     paper's T_n^p = I_d (x) T(m_{p-1}) (x) .. (x) T(m_{p-1}), applied by
 *     batched banded line solves.  omega from power iteration on D^{-1}A resp. T^{-1}A.
 * igacd_aux_is_exact: 1 when the auxiliary operator is one Kronecker product (b0 along a
 * coordinate axis) and is inverted exactly by line solves instead of a V-cycle. */
#define IGACD_SMOOTH_JACOBI 0
#define IGACD_SMOOTH_TOEPLITZ 1
/* T_n^p on the finest level only, damped Jacobi on the coarser ones (the paper's placement of
 * the T_n^p smoother) */
#define IGACD_SMOOTH_TOEPLITZ_FINE 2
int igacd_set_smoother(igacd_handle h, int kind);
/* Smoother of the auxiliary scalar V-cycle: IGACD_SMOOTH_JACOBI, IGACD_SMOOTH_TOEPLITZ, or -1
 * (default) for the same smoother as the vector V-cycle.  IGACD_E_ARG without an auxiliary space. */
int igacd_set_aux_smoother(igacd_handle h, int kind);
int igacd_get_smoother(igacd_handle h, int* kind);
int igacd_aux_is_exact(igacd_handle h, int* exact);

/* Auxiliary scalar operator: s_out = A_s s_in on `level` (vectors of igacd_ndof/dim doubles),
 * and its smoother parameters.  IGACD_E_ARG when the handle has no auxiliary space. */
int igacd_apply_aux(igacd_handle h, int level, const double* s_in, double* s_out, void* stream);
int igacd_aux_omega(igacd_handle h, int level, double* omega, double* rho);

/* PCG with the preconditioner selected by igacd_set_preconditioner (default: the additive
 * auxiliary-space + V-cycle combination IGACD_PRECOND_AUX_ADD), zero initial guess, stop when
 * ||r_k||_2 / ||r_0||_2 < tol or after maxit iterations (R7).
 * iters, relres: host outputs (may be NULL).  Synchronises `stream`.
 * Returns IGACD_E_NOCONV (x still written) when maxit is reached, IGACD_E_BREAKDOWN when
 * (p, A p) <= 0 or the residual is not finite (iters/relres then hold the failing iteration). */
int igacd_solve(igacd_handle h, const double* b, double* x, double tol, int maxit, int* iters,
                double* relres, void* stream);

/* Flexible right-preconditioned restarted GMRES -- the paper's PGMRES (PAPER.md:1075, 1260:
 * "a preconditioned generalized minimal residual (PGMRES) method").  Same preconditioner as
 * igacd_solve (igacd_set_preconditioner), zero initial guess, Arnoldi by classical
 * Gram-Schmidt with one re-orthogonalisation (CGS2), Givens rotations on the host; stop when
 * the Arnoldi residual estimate |g_{k+1}| / ||r_0||_2 < tol or after maxit products A z.
 * restart in [1, 512]: the Krylov basis V (restart+1 vectors) and Z = B V (restart vectors)
 * of level-0 size are allocated on the device on first use and owned by the handle.
 * iters, relres: host outputs (may be NULL).  Synchronises `stream` once per iteration.
 * Returns IGACD_E_NOCONV (x still written) when maxit is reached. */
int igacd_gmres(igacd_handle h, const double* b, double* x, double tol, int maxit, int restart, int* iters,
                double* relres, void* stream);

/* igacd_solve replays each PCG iteration as two CUDA graphs (captured on first use, recaptured
 * when x, the preconditioner or the smoother changes): A = operator + x/r update + ||r||^2,
 * B = preconditioner + p update.  enable = 0 launches the same kernels one by one (results
 * are bit-identical).  The environment variable IGACD_GRAPH=0 disables graphs globally. */
/* Smoothing sweeps of the auxiliary scalar V-cycle (default: the handle's nu_pre / nu_post).
 * IGACD_E_ARG when the handle has no auxiliary space. */
int igacd_set_aux_sweeps(igacd_handle h, int nu_pre, int nu_post);
int igacd_set_graphs(igacd_handle h, int enable);

/* As igacd_solve with HOST b and x (pinned or pageable); the host<->device copies are
 * part of the call. */
int igacd_solve_host(igacd_handle h, const double* b_host, double* x_host, double tol, int maxit,
                     int* iters, double* relres, void* stream);

/* Debug/parity access (host outputs).
 * igacd_get_band: the level's 1D factors in band storage, each m*(2p+1) doubles with
 *   F[k][k+o] at [k*(2p+1) + o + p] (zero outside the matrix); which = 0 M, 1 A, 2 S.
 * igacd_get_prolongation: dense (m_level x m_{level+1}) 1D knot-insertion matrix, row-major. */
int igacd_get_band(igacd_handle h, int level, int which, double* band_host);
int igacd_get_prolongation(igacd_handle h, int level, double* P_host);

/* Instrumentation: kernel launch counter (all of this handle's kernels) and, when enabled,
 * CUDA-event timing of the level-0 operator-apply kernels issued inside igacd_solve. */
int igacd_set_profiling(igacd_handle h, int enable);
int igacd_get_profile(igacd_handle h, long long* launches, long long* apply_launches, double* apply_ms);
int igacd_reset_profile(igacd_handle h);

const char* igacd_last_error(void);
const char* igacd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IGACD_H */

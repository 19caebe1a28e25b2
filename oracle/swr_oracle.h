/*
 * oracle/swr_oracle.h — TEST INFRASTRUCTURE ONLY (parity oracle).
 *
 * Plain, slow, single-threaded CPU implementation of the Schwarz waveform
 * relaxation (SWR) method of Besse & Xing, arXiv:1503.02564.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  It shares no code, header or constant
 * with the CUDA product path (paper_1503_02564_b200/), and neither imports
 * the other.
 *
 * Conventions: complex arrays are C99 `double complex` (interleaved re,im);
 * subdomains are 1-based j = 1..N as in the paper; time steps n = 1..N_T are
 * stored at index n-1; the interface vector g is slot-major
 * (r_1, l_2, r_2, ..., l_{N-1}, r_{N-1}, l_N), each slot N_T long.
 */
#ifndef SWR_ORACLE_H
#define SWR_ORACLE_H
#include <complex.h>
#include <stdint.h>

typedef double complex ocplx;

enum { OR_OK = 0, OR_ERR_ARG = 1, OR_NOT_CONVERGED = 2, OR_ZERO_PIVOT = 3,
       OR_BREAKDOWN = 4, OR_INNER_NOT_CONVERGED = 5, OR_UNSUPPORTED = 6,
       OR_OOM = 9 };
enum { OR_POT_ZERO = 0, OR_POT_VX = 1, OR_POT_VTX = 2, OR_POT_CUBIC = 3 };
/* Transmission operators (P:146-170 continuous, P:218-238 discrete):
 * Robin -ip; potential strategy S0^2, S0^3, S0^4; gauge strategy S1^2, S1^4;
 * Pade strategy S2^{2,m}, S2^{4,m} (m = pade_m poles).
 * Operators other than Robin / S0^2 need a time-independent potential here
 * (V = 0 or V(x)). */
enum { OR_TC_ROBIN = 0, OR_TC_S02 = 1, OR_TC_S03 = 2, OR_TC_S04 = 3, OR_TC_S12 = 4, OR_TC_S14 = 5,
       OR_TC_S22 = 6, OR_TC_S24 = 7 };
enum { OR_ALG_NEW = 0, OR_ALG_PRECOND = 1, OR_ALG_CLASSICAL = 2 };
/* Interface solver (reading A20/A21): GMRES(restart), BiCGStab, or the fixed
 * point of the algorithm (NEW: g <- d + L g; CLASSICAL: g <- R(g), Algorithm 1). */
enum { OR_KRY_GMRES = 0, OR_KRY_BICGSTAB = 1, OR_KRY_FIXED_POINT = 2 };

typedef struct {
  double a0, b0, T, dx, dt;   /* domain (a0,b0), final time, mesh, time step */
  int32_t N;                  /* number of subdomains */
  int32_t potential;          /* OR_POT_* */
  const double *V_x;          /* [N_x+1] nodal V(x_i) for OR_POT_VX */
  int32_t n_terms;            /* V(t,x) = sum_k tau_k(t) xi_k(x) for OR_POT_VTX */
  const double *tau;          /* [n_terms][N_T+1], tau_k(t_n) */
  const double *xi;           /* [n_terms][N_x+1], xi_k(x_i) */
  double lambda;              /* f(u) = lambda |u|^2 for OR_POT_CUBIC (paper: 1) */
  int32_t transmission;       /* OR_TC_* */
  double robin_p;             /* p > 0 for Robin */
  const ocplx *u0;            /* [N_x+1] initial datum at the nodes */
  int32_t algorithm;          /* OR_ALG_* */
  double tol; int32_t restart, maxit;            /* outer: 1e-10, 30, 2000 */
  double tol_inner; int32_t maxit_inner;         /* P^{-1} inner GMRES: 1e-12, 2000 */
  double tol_fp; int32_t maxit_fp;               /* NL inner fixed point: 1e-12, 50 */
  const ocplx *g0;            /* [(2N-2) N_T] initial interface vector, NULL = zero */
  int32_t gs_passes;          /* GMRES Gram-Schmidt passes: 1 = classical (PETSc's default
                                 KSPGMRES orthogonalization, reading A6), 2 = CGS2; 0 = 1 */
  int32_t krylov;             /* OR_KRY_*: interface solver (outer, and the inner P^{-1} solve
                                 for GMRES / BiCGStab; P^{-1} is never a fixed point) */
  int32_t pade_m;             /* number of Pade poles m >= 1 for OR_TC_S22 / OR_TC_S24 */
  int32_t pinv_exact;         /* P^{-1} of OR_ALG_PRECOND: 0 = inner Krylov on (I - L0),
                                 1 = exact causal block forward substitution */
} or_problem;

typedef struct {
  int32_t iterations;         /* outer Arnoldi steps (GMRES) or Richardson steps */
  int32_t inner_iterations;   /* total inner GMRES steps (P^{-1}) */
  int32_t fp_max;             /* max NL fixed-point iterations in any step */
  int32_t converged;
  int32_t n_history;
  double *history;            /* caller-provided, capacity maxit+1 (may be NULL) */
} or_report;

/* alpha, beta, gamma sequences, n entries each. */
void or_coeffs(int32_t n, double *alpha, double *beta, double *gamma);

/* Mesh / partition sizes. */
/* Pade coefficients a_s^m, d_s^m, s = 0..m (reading A26: rotated branch cut,
 * theta = pi/4; complex; d_0 = 0). */
void or_pade_coeffs(int32_t m, ocplx *a, ocplx *d);
/* S v_n (n = 1..nsteps) of the configured transmission operator at one
 * boundary point with interface data W, dnW, applied to v_0..v_nsteps. */
int32_t or_tc_apply(const or_problem *P, double W, double dnW, int32_t nsteps, const ocplx *v, ocplx *Sv);
/* x = (I - L0)^{-1} y exactly, by forward substitution in time: at each
 * step n the history convolution of L0 (lags >= 1) is moved to the right
 * side and the (2N-2)x(2N-2) lag-0 system is solved (factored once). */
int32_t or_pinv_causal(const or_problem *P, const ocplx *X, const ocplx *y, ocplx *x);
int32_t or_sizes(const or_problem *P, int32_t *Nx, int32_t *NT, int32_t *Nj);

/* P1 FEM matrices on a uniform mesh of nn nodes, spacing h, nodal weight W
 * (NULL = 0): M, S, M_W as (diag[nn], off[nn-1]). */
void or_fem(int32_t nn, double h, const double *W, double *Mdiag, double *Moff,
            double *Sdiag, double *Soff, double *MWdiag, double *MWoff);

/* Thomas algorithm without pivoting; lo[0] and up[n-1] unused.
 * Returns OR_ZERO_PIVOT if a pivot has modulus < 1e-300. */
int32_t or_thomas(int32_t n, const ocplx *lo, const ocplx *di, const ocplx *up,
                  const ocplx *rhs, ocplx *x);

/* Tridiagonal of (A_{j,n} - B_{j,n}) for subdomain j at step n. */
int32_t or_subdomain_matrix(const or_problem *P, int32_t j, int32_t n,
                            int32_t force_zero_potential,
                            ocplx *lo, ocplx *di, ocplx *up);

/* One whole-window march of subdomain j.
 * lin/rin: flux series l_{j,n}, r_{j,n} (length N_T, NULL = 0).
 * use_u0: start from u0 restricted to the subdomain (else 0).
 * force_zero_potential: march with V == 0 (the L_0 / preconditioner problem).
 * out_left:  r_{j-1,n}^{new} = -l_{j,n} + 2 S v_{j,n}(a_j)   (j >= 2)
 * out_right: l_{j+1,n}^{new} = -r_{j,n} + 2 S v_{j,n}(b_j)   (j <= N-1)
 * uT: [N_j] local u_{N_T} (NULL allowed).  fp_max: max NL FP iterations. */
int32_t or_march(const or_problem *P, int32_t j, const ocplx *lin, const ocplx *rin,
                 int32_t use_u0, int32_t force_zero_potential,
                 ocplx *out_left, ocplx *out_right, ocplx *uT, int32_t *fp_max);

/* g -> R(g) (eq. 13): one sweep of every subdomain + exchange. */
int32_t or_apply_R(const or_problem *P, const ocplx *g, int32_t use_u0,
                   int32_t force_zero_potential, ocplx *Rg, int32_t *fp_max);

/* First columns of the Toeplitz blocks by unit-impulse probing
 * with u0 = 0.  X is [N][4][N_T]: X[(j-1)*4 + (p-1)] = first column of X^{j,p}
 * (only X^{1,4}, X^{j,1..4} (1<j<N), X^{N,1} are meaningful). */
int32_t or_build_L(const or_problem *P, int32_t force_zero_potential, ocplx *X);

/* Lg with the block pattern of eq. (15) and causal convolutions. */
void or_apply_L(const or_problem *P, const ocplx *X, const ocplx *g, ocplx *Lg);

/* Order-fixed inner product over the interface vector: partial per
 * subdomain (its own slots, sequential), partials summed in j order. */
ocplx or_dot(const or_problem *P, const ocplx *x, const ocplx *y);

/* BiCGStab on a dense n x n matrix (row-major), same driver as or_solve. */
int32_t or_bicgstab_dense(int32_t n, const ocplx *A, const ocplx *b, ocplx *x, double tol, int32_t maxit,
                          int32_t *iters, double *hist);

/* GMRES(m) with CGS2 on a dense n x n matrix (row-major); dot is plain
 * sequential.  Used by tests to pin the Krylov driver. */
int32_t or_gmres_dense(int32_t n, int32_t gs_passes, const ocplx *A, const ocplx *b, ocplx *x,
                       double tol, int32_t restart, int32_t maxit,
                       int32_t *iters, double *hist);

/* Full algorithm (NEW / PRECOND / NL Richardson) -> u(T) on [N_x+1]. */
int32_t or_solve(const or_problem *P, ocplx *uT, or_report *rep,
                 ocplx *g_out /* [(2N-2)N_T] or NULL */);

/* Worker threads of the subdomain-parallel loops (marches of independent
 * subdomains, per-subdomain Toeplitz blocks and dot-product partials,
 * element ranges of the Krylov vector updates).  Every parallel item writes
 * its own outputs and reductions keep their sequential order, so results are
 * bitwise independent of the count.  Default 1. */
void or_set_threads(int32_t n);
int32_t or_get_threads(void);

/* Single-domain reference solve (N = 1, Neumann both ends). */
int32_t or_monodomain(const or_problem *P, ocplx *uT, int32_t *fp_max);

#endif

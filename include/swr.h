/*
 * include/swr.h — C ABI of the B200-native Schwarz waveform relaxation (SWR)
 * hot path for the 1D Schrödinger equation (Besse & Xing, arXiv:1503.02564,
 * PAPER.md; "P:n" = PAPER.md line n).
 *
 * Problem:  (i d_t + d_xx + V) u = 0 on (a0,b0) x (0,T),
 *   u(0) = u0, homogeneous Neumann at a0, b0, V real: V(x), V(t,x) or
 *   f(u) = lambda |u|^2.  Crank-Nicolson in time in the v-variable,
 *   P1 finite elements on a uniform global mesh, N equal non-overlapping
 *   subdomains, transmission B = d_n + S with S = Robin -ip
 *   or the potential-strategy S0^2.
 *
 * Algorithms:
 *   SWR_ALG_NEW      Algorithm 3 for V(x): build d = R(0)
 *                     and the lower-triangular Toeplitz interface
 *                    matrix L from unit-impulse probes, solve
 *                    (I - L) g = d by GMRES, then one final sweep.
 *   SWR_ALG_PRECOND  zero-potential preconditioner P = I - L0:
 *                    GMRES on P^{-1}(I - L) g = P^{-1} d for V(t,x)
 *                    (eq. chp2_algopd_Lpf); preconditioned fixed point
 *                    g <- g - P^{-1}(g - R_nl(g)) for f(u) (eq. chp2_algopd_NL).
 *
 * Data conventions (all calls):
 *   - complex arrays are interleaved (re, im) fp64, i.e. double[2*len];
 *   - the interface vector g is slot-major
 *     (r_1, l_2, r_2, ..., l_{N-1}, r_{N-1}, l_N), each slot N_T entries
 *     (time steps n = 1..N_T at index n-1): length n_g = (2N-2) N_T complex;
 *   - N_x = round((b0-a0)/dx), N_T = round(T/dt), N must divide N_x;
 *     subdomain j = 1..N holds global nodes [(j-1)m, jm], m = N_x/N,
 *     N_j = m+1 (interface nodes duplicated, reading A1 of DESIGN.md);
 *   - every call is collective over the ranks of one handle and runs on the
 *     caller's CUDA stream; a handle is not thread-safe.
 *
 * Ownership: inputs are copied during swr_setup (and swr_update_inputs); the
 * caller keeps its arrays.  The handle owns all device memory and the report
 * buffers, released by swr_free.
 *
 * Errors: every int-returning call returns an swr_status; 0 = success.
 * SWR_NOT_CONVERGED leaves valid outputs (the last iterate).  CUDA/NCCL
 * failures are reported as SWR_ERR_CUDA / SWR_ERR_NCCL; swr_error_string and
 * swr_last_error_detail describe them.  There is no CPU fallback: a machine
 * without a usable sm_100a GPU gets SWR_ERR_CUDA from swr_setup.
 */
#ifndef SWR_H
#define SWR_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct swr_handle swr_handle;

enum swr_status {
  SWR_OK = 0,
  SWR_ERR_INVALID_ARG = 1,
  SWR_NOT_CONVERGED = 2,          /* outputs valid but unconverged */
  SWR_ERR_ZERO_PIVOT = 3,         /* |pivot| < 1e-300: A - B singular (Prop. 1 hypothesis) */
  SWR_ERR_BREAKDOWN = 4,
  SWR_ERR_INNER_NOT_CONVERGED = 5,/* P^{-1} GMRES or NL fixed point hit its cap */
  SWR_ERR_UNSUPPORTED = 6,        /* e.g. NEW with V(t,x) or f(u); f(u) = |u|^2 with
                                     N_j > 65,536 rows (the nonlinear march is resident only) */
  SWR_ERR_CUDA = 7,
  SWR_ERR_NCCL = 8,
  SWR_ERR_OOM = 9
};

enum swr_potential {
  SWR_POT_ZERO = 0,
  SWR_POT_VX = 1,              /* V(x): nodal samples V_x[N_x+1] */
  SWR_POT_VTX_SEPARABLE = 2,   /* V(t,x) = sum_k tau_k(t) xi_k(x) */
  SWR_POT_CUBIC = 3            /* f(u) = lambda |u|^2 */
};

/* Transmission operators (discrete P:218-267): Robin -ip;
 * potential strategy S0^2, S0^3, S0^4; gauge strategy S1^2, S1^4; Pade
 * strategy S2^{2,m}, S2^{4,m} with m = pade_m poles (coefficients: reading
 * A26, the rotated-branch-cut Pade approximant, theta = pi/4).  Operators other than Robin / S0^2 need a time-independent potential
 * (V = 0 or V(x)) and the NEW or CLASSICAL algorithm (readings A23-A26). */
enum swr_transmission {
  SWR_TC_ROBIN = 0, SWR_TC_S0_2 = 1, SWR_TC_S0_3 = 2, SWR_TC_S0_4 = 3, SWR_TC_S1_2 = 4, SWR_TC_S1_4 = 5,
  SWR_TC_S2_2 = 6, SWR_TC_S2_4 = 7
};
enum swr_algorithm {
  SWR_ALG_NEW = 0,       /* Algorithm 3 */
  SWR_ALG_PRECOND = 1,   /* preconditioned algorithms */
  SWR_ALG_CLASSICAL = 2  /* Algorithm 1 (fixed point g <- R(g)) or
                            Algorithm 2 (Krylov on g - R_0(g) = R(0; u0)) */
};
/* Interface solver (readings A20, A21).  GMRES / BiCGStab also serve the
 * inner P^{-1} solve of SWR_ALG_PRECOND (GMRES when the outer solver is the
 * fixed point); the fixed point is g <- d + L g for NEW, g <- R(g) for
 * CLASSICAL and g <- g - P^{-1}(g - R(g)) for PRECOND. */
enum swr_krylov { SWR_KRY_GMRES = 0, SWR_KRY_BICGSTAB = 1, SWR_KRY_FIXED_POINT = 2 };

typedef struct {
  double a0, b0, T, dx, dt;   /* domain, final time, mesh size, time step */
  int32_t N;                  /* number of subdomains, N | N_x */
  int32_t potential;          /* swr_potential */
  const double *V_x;          /* [N_x+1] real, SWR_POT_VX */
  int32_t n_terms;            /* SWR_POT_VTX_SEPARABLE */
  const double *tau;          /* [n_terms][N_T+1]: tau_k(t_n) */
  const double *xi;           /* [n_terms][N_x+1]: xi_k(x_i) */
  double lambda;              /* SWR_POT_CUBIC coefficient (paper: 1) */
  int32_t transmission;       /* swr_transmission */
  double robin_p;             /* Robin parameter p > 0 */
  const double *u0;           /* [2*(N_x+1)] initial datum at the nodes */
  int32_t inputs_on_device;   /* 1: u0, V_x, tau, xi, g0 are device pointers */
  int32_t algorithm;          /* swr_algorithm */
  double tol;                 /* outer tolerance (paper: 1e-10) */
  int32_t restart, maxit;     /* GMRES(m): 30, 2000; restart <= 31 (the fused Gram-Schmidt
                                 kernels hold up to 32 basis vectors), else SWR_ERR_INVALID_ARG */
  double tol_inner;           /* P^{-1} inner GMRES relative tol: 1e-12 */
  int32_t maxit_inner;        /* 2000 */
  double tol_fp;              /* NL inner fixed point relative max-norm: 1e-12 */
  int32_t maxit_fp;           /* 50 */
  const double *g0;           /* [2*n_g] initial interface vector, NULL = zero */
  int32_t rank, world;        /* world = 1: single GPU, no NCCL; world <= N */
  const void *nccl_unique_id; /* 128-byte ncclUniqueId (world > 1) */
  void *cuda_stream;          /* cudaStream_t owned by the caller (NULL = default stream) */
  int32_t device;             /* CUDA device ordinal for this rank */
  int32_t gs_passes;          /* GMRES Gram-Schmidt passes per Arnoldi step: 1 = classical
                                 Gram-Schmidt, PETSc's default KSPGMRES orthogonalization
                                 (the paper's solver library; reading A6);
                                 2 = CGS2 (one reorthogonalization); 0 = 1 */
  int32_t krylov;             /* swr_krylov: interface solver (0 = GMRES) */
  int32_t pade_m;             /* Pade poles m >= 1 for SWR_TC_S2_2 / SWR_TC_S2_4 (else ignored) */
  int32_t pinv_exact;         /* SWR_ALG_PRECOND: 0 = P^{-1} by the inner Krylov solve on (I - L0)
                                 (P:1059); 1 = exact causal forward substitution in time (reading
                                 A27); fails with SWR_ERR_UNSUPPORTED when the lag-0 interface
                                 coupling is too strong for the bounded sweep count */
  /* Kernel forms (same arithmetic, different rounding order only; 0 = automatic): */
  int32_t march_form;         /* 0: the resident cluster march when a subdomain fits one thread-block
                                 cluster (N_j up to ~45K rows), the streaming march otherwise;
                                 1: always the streaming march */
  int32_t toeplitz_form;      /* (I - L) x: 0: FFT convolution (register four-step kernel for
                                 257 <= N_T <= 512, shared-memory radix-4 for N_T <= 256), the direct
                                 causal convolution for N_T > 512; 1: direct; 2: shared-memory FFT */
  int32_t nl_rows_per_thread; /* f(u) march: 0: automatic; 8, 11 or 16 forces the rows per thread
                                 (the 16-row shape serves subdomains up to 16 x 256 x 16 = 65,536
                                 rows) */
} swr_config;

typedef struct {
  int32_t iterations;         /* outer GMRES Arnoldi steps / fixed-point steps */
  int32_t inner_iterations;   /* total P^{-1} inner GMRES steps */
  int32_t fp_max;             /* max NL fixed-point iterations in any step */
  int32_t converged;
  const double *residual_history; /* [n_history], owned by the handle */
  int32_t n_history;
  double t_build_ms;          /* swr_build_interface_operator, device time */
  double t_solve_ms;          /* swr_solve, device time */
  double t_march_ms;          /* sum of march-kernel time (CUDA events) */
  double t_interface_ms;      /* Toeplitz apply + Krylov vector kernels */
  double cell_steps;          /* sum over marches of (sum_j N_j) * N_T * RHS (this rank) */
  int32_t n_marches;          /* march-kernel launches */
  int32_t n_kernel_launches;  /* all kernels of this library launched (and collectives) */
  double t_setup_ms;          /* swr_setup, host wall time (allocation, copies, factorisation) */
  double t_comm_ms;           /* collectives of build + solve (cut traces, partial sums), device time */
} swr_report;

/* Validate the configuration, copy the inputs to the GPU, assemble and
 * factor the subdomain matrices (A - B), eq. (9).
 * Returns SWR_ERR_INVALID_ARG for: N not dividing N_x, world > N, Robin with
 * p <= 0, NEW with a time-dependent or nonlinear potential, CLASSICAL with a
 * Krylov solver and f(u) (R is not affine), NULL u0.
 * *out receives the handle (NULL on failure).  Collective. */
int swr_setup(const swr_config *cfg, swr_handle **out);

/* Replace u0 (and V_x for SWR_POT_VX, refactoring the matrices) with arrays
 * of the same sizes; on_device as cfg->inputs_on_device.  Stream-ordered on
 * the handle's stream (a host u0 given with V_x is copied on an internal
 * stream that the handle's stream waits for, overlapping the factorisation);
 * host buffers may be reused once the call returns (it waits for its
 * copies and the factorisation's pivot check).  Returns SWR_ERR_ZERO_PIVOT if A - B cannot
 * be factored.  Collective. */
int swr_update_inputs(swr_handle *h, const double *u0, const double *V_x, int32_t on_device);

/* NEW: one batched march per subdomain with three right-hand sides (d, the
 * l_j impulse and the r_j impulse) -> d and the first columns of
 * X^{j,1..4}.  PRECOND: the V = 0 impulse probes -> L0, plus d for
 * V(t,x).  Collective. */
int swr_build_interface_operator(swr_handle *h);

/* Solve the interface problem and run the final sweep; u_T [2*(N_x+1)]
 * receives u(x_i, T) on rank 0 (interface nodes: mean of the two copies),
 * host memory if u_T_on_device == 0.  NULL skips the gather.  rep may be
 * NULL.  Collective. */
int swr_solve(swr_handle *h, double *u_T, int32_t u_T_on_device, swr_report *rep);

void swr_free(swr_handle *h);
const char *swr_error_string(int status);
const char *swr_last_error_detail(void);

/* ---- Lower-level entry points (parity tests, benchmarks). -------------
 * Device pointers (this rank's GPU), n_g = (2N-2) N_T complex, world = 1
 * only (SWR_ERR_INVALID_ARG otherwise). */

/* Rg = R(g; u0 if use_u0 else 0) with the true potential, or with V = 0 if
 * force_zero_potential (eq. 13): one march of every subdomain and the
 * exchange of eq. (8).  g may be NULL (= 0).  If u_T is non-NULL it
 * receives the assembled u(T) [2*(N_x+1)] of that sweep. */
int swr_apply_R(swr_handle *h, const double *g, int32_t use_u0, int32_t force_zero_potential,
                double *Rg, double *u_T);

/* y = (I - L) x (which = 0) or (I - L0) x (which = 1), causal block-Toeplitz
 * convolutions with the first columns built by swr_build_interface_operator. */
int swr_apply_I_minus_L(swr_handle *h, int32_t which, const double *x, double *y);

/* Copy out d [2*n_g] and the Toeplitz first columns X [2*N*4*N_T] (X[(j-1)*4+p-1]
 * = first column of X^{j,p}; which = 0: L, 1: L0). NULL skips. */
int swr_get_interface(swr_handle *h, int32_t which, double *d, double *X);

/* Test infrastructure (one GPU, SWR_ALG_NEW): replace the interface operator
 * with a given one -- d [2*n_g] and the first columns X [2*N*4*N_T] (device
 * pointers, the layout of swr_get_interface); the next swr_solve runs the
 * interface solve and the final sweep on it.  Lets a test give both sides
 * the same operator (Algorithm 3's solve stage, isolated from the
 * rounding of the build).  SWR_ERR_INVALID_ARG otherwise. */
int swr_set_interface(swr_handle *h, const double *d, const double *X);

/* Copy out this rank's slots of the interface vector g of the last swr_solve:
 * [2 * (s_hi - s_lo + 1) * N_T] (swr_owned_slots; the whole g on one GPU). */
int swr_get_g(swr_handle *h, double *g);

/* Sizes: N_x, N_T, N_j, n_g. */
int swr_sizes(const swr_handle *h, int32_t *Nx, int32_t *NT, int32_t *Nj, int64_t *ng);

/* ---- Multi-GPU (one process per GPU). ----------------------
 * Owner computes (the block-column ownership of P:982-1011): rank r of W owns
 * the subdomains j in [floor(rN/W)+1, floor((r+1)N/W)] and their interface
 * slots [s_lo, s_hi] (swr_owned_slots, contiguous); its d, g and Krylov
 * vectors hold those slots only, its first columns of L are those of its
 * subdomains.  Per march sweep or (I - L) apply only the two cut traces cross
 * a rank cut (ncclSend/ncclRecv of N_T complex with each neighbour rank); per
 * Gram-Schmidt pass the per-subdomain partial sums are summed over ranks
 * (ncclAllReduce of disjoint columns, exact) and reduced in the same fixed
 * order as on one GPU, so any W reproduces the one-GPU iterates bitwise;
 * u(T) is reduced onto rank 0 (ncclReduce).  L0 (PRECOND) is held whole by
 * every rank (its interior blocks coincide), and the exact P^{-1}
 * (pinv_exact = 1) runs replicated on the gathered vector.
 * Pure host functions, no GPU needed: */
int swr_partition(int32_t N, int32_t world, int32_t rank, int32_t *j_lo, int32_t *j_hi);
int swr_owned_slots(int32_t N, int32_t world, int32_t rank, int32_t *s_lo, int32_t *s_hi);

/* Writes a 128-byte ncclUniqueId (rank 0; broadcast it to the other ranks
 * and pass it as swr_config.nccl_unique_id).  SWR_ERR_NCCL if libnccl is
 * not loadable. */
int swr_nccl_unique_id(void *out128);

/* TEST INFRASTRUCTURE: an id (pass as swr_config.nccl_unique_id) that runs
 * `world` logical ranks as host threads of this process on one GPU, with
 * device copies standing in for NCCL (tests/test_multirank.py drives the
 * multi-rank code path with it; never a performance configuration). */
int swr_loopback_id(void *out128, int32_t world);

#ifdef __cplusplus
}
#endif
#endif

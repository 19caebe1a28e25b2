/*
 * oracle/swr_oracle.c — TEST INFRASTRUCTURE ONLY (parity oracle).
 *
 * Plain, slow C implementation of the SWR method of
 * Besse & Xing, arXiv:1503.02564.  Every function follows the paper's
 * formulas in the paper's order; "P:n" cites PAPER.md line n, "A<k>" cites
 * a reading listed in DESIGN.md.  Built with
 * -O2 -ffp-contract=off -fcx-limited-range (plain IEEE products, no FMA).
 * Single-threaded by default; or_set_threads(P) runs independent subdomains
 * (and element ranges of vector updates) on P threads with every reduction
 * kept in its sequential order, so the results are bitwise those of one
 * thread ("Oracle timing": T_oracle,1 and T_oracle,P).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
 * --impl reference) may load this library.  The CUDA product path never
 * links, loads or calls it.
 *
 * Parity status: every exported function is pinned by a -m "not gpu" test in
 * tests/test_oracle_*.py against something other than itself (closed forms,
 * dense brute force, invariants, the paper's printed values).
 */
#include "swr_oracle.h"
#include <math.h>
#include <pthread.h>

/* Mutation hooks for tests/test_oracle_mutants.py only: a build with
 * -DOR_MUTANT=k plants one deliberate error (a wrong sign, time level or
 * coefficient) so the test can show that a pin of tests/test_oracle_pins.py
 * catches it.  The default build (OR_MUTANT = 0) contains none of them. */
#ifndef OR_MUTANT
#define OR_MUTANT 0
#endif
#define MUT(k) (OR_MUTANT == (k))

/* ------------------------------------------------------------------ */
/* Parallel loops.  par_for(n, fn, ctx) calls fn(ctx, i) for i = 0..n-1 */
/* on up to or_threads threads (dynamic schedule).  Callers only use it */
/* where every item writes disjoint outputs and sums keep their order. */
/* ------------------------------------------------------------------ */
static int32_t or_threads = 1;
void or_set_threads(int32_t n) { or_threads = n < 1 ? 1 : (n > 256 ? 256 : n); }
int32_t or_get_threads(void) { return or_threads; }

typedef void (*or_item_fn)(void *ctx, int64_t item);
typedef struct { or_item_fn fn; void *ctx; int64_t n, next; } par_job;

static void *par_worker(void *arg) {
  par_job *J = (par_job *)arg;
  for (;;) {
    const int64_t i = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (i >= J->n) break;
    J->fn(J->ctx, i);
  }
  return NULL;
}

static void par_for(int64_t n, or_item_fn fn, void *ctx) {
  int64_t T = or_threads < n ? or_threads : n;
  par_job J = {fn, ctx, n, 0};
  if (T <= 1) {
    for (int64_t i = 0; i < n; i++) fn(ctx, i);
    return;
  }
  pthread_t th[256];
  int64_t started = 0;
  for (int64_t t = 1; t < T; t++)
    if (pthread_create(&th[started], NULL, par_worker, &J) == 0) started++;
  par_worker(&J);
  for (int64_t t = 0; t < started; t++) pthread_join(th[t], NULL);
}

/* element ranges of a length-n vector loop */
#define PAR_CHUNK 8192
static int64_t n_chunks(size_t n) { return (int64_t)((n + PAR_CHUNK - 1) / PAR_CHUNK); }
#define CHUNK_RANGE(c, n, lo, hi)                 \
  const size_t lo = (size_t)(c) * PAR_CHUNK;       \
  const size_t hi = lo + PAR_CHUNK < (n) ? lo + PAR_CHUNK : (n)
#include <stdlib.h>
#include <string.h>

#define I_ _Complex_I

/* ------------------------------------------------------------------ */
/* Coefficients alpha, beta, gamma.                        */
/* alpha = (1, 1, 1/2, 1/2, 3/8, 3/8, 3*5/(2*4*6), ...):               */
/* alpha_{2k} = alpha_{2k-2} (2k-1)/(2k), alpha_{2k+1} = alpha_{2k};   */
/* beta_s = (-1)^s alpha_s;  gamma = (1, 2, 2, 2, ...).                */
/* ------------------------------------------------------------------ */
void or_coeffs(int32_t n, double *alpha, double *beta, double *gamma) {
  for (int32_t s = 0; s < n; s++) {
    double a;
    if (s == 0) a = 1.0;
    else if (s % 2 == 1) a = alpha[s - 1];
    else a = alpha[s - 2] * (double)(s - 1) / (double)s;
    alpha[s] = a;
    if (beta) beta[s] = (s % 2 == 0) ? a : -a;
    if (gamma) gamma[s] = (s == 0) ? 1.0 : 2.0;
  }
}

/* Mesh (reading A1): N_x = round((b0-a0)/dx), N_T = round(T/dt),
 * N | N_x, subdomain j holds global nodes [(j-1)m, jm], m = N_x/N. */
int32_t or_sizes(const or_problem *P, int32_t *Nx, int32_t *NT, int32_t *Nj) {
  if (!P || P->N < 1 || !(P->dx > 0) || !(P->dt > 0)) return OR_ERR_ARG;
  int32_t nx = (int32_t)llround((P->b0 - P->a0) / P->dx);
  int32_t nt = (int32_t)llround(P->T / P->dt);
  if (nx < 1 || nt < 1 || nx % P->N != 0) return OR_ERR_ARG;
  if (nx / P->N < 1) return OR_ERR_ARG;
  if (Nx) *Nx = nx;
  if (NT) *NT = nt;
  if (Nj) *Nj = nx / P->N + 1;
  return OR_OK;
}

/* P1 finite elements on a uniform mesh by element assembly.
 * Element (k,k+1) of length h contributes
 *   M:   h/3, h/3 on the diagonal, h/6 off-diagonal;
 *   S:   1/h, 1/h on the diagonal, -1/h off-diagonal  (S = int v' phi');
 *   M_W: h(3W_k+W_{k+1})/12, h(W_k+3W_{k+1})/12 diagonal,
 *        h(W_k+W_{k+1})/12 off-diagonal  (exact integral of the linear
 *        interpolant of W times hat products, reading A2). */
void or_fem(int32_t nn, double h, const double *W, double *Mdiag, double *Moff,
            double *Sdiag, double *Soff, double *MWdiag, double *MWoff) {
  for (int32_t k = 0; k < nn; k++) {
    if (Mdiag) Mdiag[k] = 0.0;
    if (Sdiag) Sdiag[k] = 0.0;
    if (MWdiag) MWdiag[k] = 0.0;
  }
  for (int32_t k = 0; k + 1 < nn; k++) {
    if (Mdiag) { Mdiag[k] += h / 3.0; Mdiag[k + 1] += h / 3.0; }
    if (Moff) Moff[k] = h / 6.0;
    if (Sdiag) { Sdiag[k] += 1.0 / h; Sdiag[k + 1] += 1.0 / h; }
    if (Soff) Soff[k] = -1.0 / h;
    double w0 = W ? W[k] : 0.0, w1 = W ? W[k + 1] : 0.0;
    if (MWdiag) {
      MWdiag[k] += h * (3.0 * w0 + w1) / 12.0;
      MWdiag[k + 1] += h * (w0 + 3.0 * w1) / 12.0;
    }
    if (MWoff) MWoff[k] = h * (w0 + w1) / 12.0;
  }
}

/* Thomas algorithm (Gaussian elimination without pivoting on a tridiagonal
 * system), the "LU direct method" of P:1079. */
int32_t or_thomas(int32_t n, const ocplx *lo, const ocplx *di, const ocplx *up,
                  const ocplx *rhs, ocplx *x) {
  ocplx *cp = (ocplx *)malloc(sizeof(ocplx) * (size_t)n);
  ocplx *dp = (ocplx *)malloc(sizeof(ocplx) * (size_t)n);
  if (!cp || !dp) { free(cp); free(dp); return OR_OOM; }
  int32_t st = OR_OK;
  for (int32_t k = 0; k < n; k++) {
    ocplx den = (k == 0) ? di[0] : di[k] - lo[k] * cp[k - 1];
    if (cabs(den) < 1e-300) { st = OR_ZERO_PIVOT; break; }
    cp[k] = (k + 1 < n) ? up[k] / den : 0.0;
    dp[k] = (k == 0) ? rhs[0] / den : (rhs[k] - lo[k] * dp[k - 1]) / den;
  }
  if (st == OR_OK) {
    x[n - 1] = dp[n - 1];
    for (int32_t k = n - 2; k >= 0; k--) x[k] = dp[k] - cp[k] * x[k + 1];
  }
  free(cp); free(dp);
  return st;
}

/* ------------------------------------------------------------------ */
/* Transmission operator constants.                                    */
/* S0^2: Sv_n = c2 sum_{s=0}^{n} beta_{n-s} v_s, c2 = e^{-i pi/4}
 * sqrt(2/dt) = (1-i)/sqrt(dt); leading coefficient c0 = c2 beta_0.
 * Robin: Sv_n = -i p v_n, c0 = -ip, no history.               */
/* ------------------------------------------------------------------ */
static ocplx or_c2(const or_problem *P) {
  /* e^{-i pi/4} sqrt(2/dt) = ((1-i)/sqrt 2) sqrt 2 / sqrt(dt), exactly. */
  return (1.0 - I_) / sqrt(P->dt);
}

/* Interface data of one side of subdomain j for the higher-order operators
 * (time-independent potential): W at the interface node, its outward normal
 * derivative dnW (reading A23: central difference of the nodal W on the
 * global mesh, n = -x at a_j, +x at b_j) and the gauge phase rate:
 * calV_n = t_n W, calW_n = (calV_n + calV_{n-1})/2 = W dt (n - 1/2) for
 * n >= 1, calW_0 = 0 (reading A24). */
typedef struct { double W, dnW; int32_t fz; } tc_side;

static tc_side or_tc_side(const or_problem *P, int32_t j, int32_t side, int32_t fz) {
  tc_side t = {0.0, 0.0, fz};
  if (fz || P->potential != OR_POT_VX) return t;
  int32_t Nx, NT, Nj;
  or_sizes(P, &Nx, &NT, &Nj);
  int32_t m = Nx / P->N, i = side == 0 ? (j - 1) * m : j * m;
  t.W = P->V_x[i];
  double dx = (i > 0 && i < Nx) ? (P->V_x[i + 1] - P->V_x[i - 1]) / (2.0 * P->dx) : 0.0;
  t.dnW = side == 0 ? -dx : dx;
  return t;
}

static double or_calW(const tc_side *t, int32_t n, double dt) { return n == 0 ? 0.0 : t->W * dt * (n - 0.5); }

/* Kernel K(n, s) of the discrete transmission operator S v_n = sum_{s<=n}
 * K(n, s) v_s, alpha/beta/gamma from or_coeffs. */
static ocplx or_tcK(const or_problem *P, const tc_side *t, int32_t n, int32_t s, const double *alpha,
                    const double *beta, const double *gamma) {
  const double dt = P->dt;
  const ocplx c2 = or_c2(P);                                  /* e^{-i pi/4} sqrt(2/dt) */
  const ocplx e3 = (1.0 + I_) / sqrt(2.0) * sqrt(MUT(7) ? dt : dt / 2.0);   /* e^{i pi/4} sqrt(dt/2) */
  const double sa = MUT(3) ? -1.0 : 1.0, sg4 = MUT(4) ? -1.0 : 1.0;
  const int32_t d = n - s;
  switch (P->transmission) {
    case OR_TC_ROBIN: return d == 0 ? -I_ * P->robin_p : 0.0;
    case OR_TC_S02: return c2 * beta[d];
    case OR_TC_S03: return c2 * beta[d] - sa * e3 * (t->W / 2.0) * alpha[d];
    case OR_TC_S04:
      return c2 * beta[d] - sa * e3 * (t->W / 2.0) * alpha[d] - sg4 * I_ * (t->dnW / 4.0) * (dt / 2.0) * gamma[d];
    case OR_TC_S12:
    case OR_TC_S14: {
      const double ph = or_calW(t, n, dt) - or_calW(t, s, dt);
      const ocplx e = cexp((MUT(5) ? -I_ : I_) * ph);
      ocplx k = c2 * e * beta[d];
      if (P->transmission == OR_TC_S14) {
        const double sg = t->dnW > 0 ? 1.0 : (t->dnW < 0 ? -1.0 : 0.0), r = sqrt(fabs(t->dnW)) / 2.0;
        k -= (MUT(6) ? -I_ : I_) * sg * r * e * (dt / 2.0) * gamma[d] * r;
      }
      return k;
    }
  }
  return 0.0;
}

static ocplx or_c0(const or_problem *P) {
  if (P->transmission == OR_TC_ROBIN) return -I_ * P->robin_p;
  return or_c2(P) * 1.0; /* beta_0 = 1 */
}

/* ------------------------------------------------------------------ */
/* Pade strategy S2^{2,m}, S2^{4,m} (P:173-177 continuous, P:241-267     */
/* discrete).  sqrt(z) ~ sum_{s=0}^m a_s - sum_{s=1}^m a_s d_s/(z + d_s). */
/* The paper does not give a_s^m, d_s^m (reading A26): the rotated-branch- */
/* cut Pade approximation of the cited ABC literature with theta = pi/4:  */
/* sqrt z = e^{i th/2} sqrt(e^{-i th} z), sqrt(1 + x) by the diagonal      */
/* Pade approximant 1 + sum_s b_s x/(1 + c_s x), b_s = 2/(2m+1) sin^2 u_s, */
/* c_s = cos^2 u_s, u_s = s pi/(2m+1); in the form above                  */
/*   d_s = e^{i th} (1 - c_s)/c_s,  a_s = e^{i th/2} b_s/(c_s (1 - c_s)),  */
/*   a_0 = e^{i th/2} (1 + sum_s b_s/c_s) - sum_{s>=1} a_s  (complex).     */
/* Chosen because it reproduces the fixed-point counts of the paper's     */
/* Table 6 (187/76/39 vs 191/76/39 for m = 20/50/100), which */
/* the unrotated forms miss by a factor ~3.7 (A26).             */
/* In S2^2 the paper writes d_k^m in one denominator; read as d_s^m.      */
/* ------------------------------------------------------------------ */
static int or_is_pade(const or_problem *P) {
  return P->transmission == OR_TC_S22 || P->transmission == OR_TC_S24;
}

void or_pade_coeffs(int32_t m, ocplx *a, ocplx *d) {
  const double pi = acos(-1.0), th = pi / 4.0;
  const ocplx eh = cexp(I_ * (th / 2.0)), ef = cexp(I_ * th);
  ocplx sumb = 0.0, suma = 0.0;
  d[0] = 0.0;
  for (int32_t s = 1; s <= m; s++) {
    const double u = s * pi / (2.0 * m + 1.0);
    const double cs = cos(u) * cos(u), bs = 2.0 / (2.0 * m + 1.0) * sin(u) * sin(u);
    d[s] = ef * ((1.0 - cs) / cs);
    a[s] = eh * (bs / (cs * (1.0 - cs)));
    sumb += bs / cs;
    suma += a[s];
  }
  a[0] = eh * (1.0 + sumb) - suma;
}

/* State of the auxiliary functions phi^s_{j,n-1} (s = 1..m) and psi_{j,n-1}
 * of one boundary point, both zero at n = 0. */
typedef struct { int32_t m; ocplx *a, *d; ocplx *phi; ocplx psi; } pade_state;

static int32_t pade_init(const or_problem *P, pade_state *S) {
  S->m = P->pade_m;
  S->a = (ocplx *)calloc((size_t)S->m + 1, sizeof(ocplx));
  S->d = (ocplx *)calloc((size_t)S->m + 1, sizeof(ocplx));
  S->phi = (ocplx *)calloc((size_t)S->m + 1, sizeof(ocplx));
  S->psi = 0.0;
  if (!S->a || !S->d || !S->phi) return OR_OOM;
  or_pade_coeffs(S->m, S->a, S->d);
  return OR_OK;
}

static void pade_free(pade_state *S) { free(S->a); free(S->d); free(S->phi); }

/* Coefficient of v_{j,n} in S2 v_{j,n}:
 *   -i (sum_{s=0}^m a_s) + i sum_{s=1}^m a_s d_s / (2i/dt + W + d_s)
 *   [+ (dnW/4) / (2i/dt + W) for S2^4]. */
static ocplx pade_c0(const or_problem *P, const tc_side *t, const pade_state *S) {
  const ocplx s2 = 2.0 * I_ / P->dt;
  ocplx sa = 0.0, c = 0.0;
  for (int32_t s = 0; s <= S->m; s++) sa += S->a[s];
  c = -I_ * sa;
  for (int32_t s = 1; s <= S->m; s++) c += I_ * S->a[s] * S->d[s] / (s2 + t->W + S->d[s]);
  if (P->transmission == OR_TC_S24) c += (t->dnW / 4.0) / (s2 + t->W);
  return c;
}

/* The rest of S2 v_{j,n}: terms in phi^s_{j,n-1}, psi_{j,n-1}. */
static ocplx pade_hist(const or_problem *P, const tc_side *t, const pade_state *S) {
  const ocplx s2 = 2.0 * I_ / P->dt;
  ocplx h = 0.0;
  for (int32_t s = 1; s <= S->m; s++) h += I_ * S->a[s] * S->d[s] * (s2 / (s2 + t->W + S->d[s])) * S->phi[s];
  if (P->transmission == OR_TC_S24) {
    const double sg = t->dnW > 0 ? 1.0 : (t->dnW < 0 ? -1.0 : 0.0);
    h += sg * (sqrt(fabs(t->dnW)) / 2.0) * (s2 / (s2 + t->W)) * S->psi;
  }
  return h;
}

/* phi^s_{n-1/2} = v_n/(2i/dt + W + d_s) + (2i/dt)/(2i/dt + W + d_s) phi^s_{n-1},
 * phi^s_n = 2 phi^s_{n-1/2} - phi^s_{n-1}; psi likewise.
 * phi, psi depend on |dnW| only, so one state serves both normals. */
static void pade_advance(const or_problem *P, const tc_side *t, pade_state *S, ocplx vn) {
  const ocplx s2 = 2.0 * I_ / P->dt;
  for (int32_t s = 1; s <= S->m; s++) {
    const ocplx D = s2 + t->W + S->d[s];
    const ocplx half = vn / D + (s2 / D) * S->phi[s];
    S->phi[s] = 2.0 * half - S->phi[s];
  }
  const ocplx D0 = s2 + t->W;
  const ocplx half = (sqrt(fabs(t->dnW)) / 2.0) * vn / D0 + (s2 / D0) * S->psi;
  S->psi = 2.0 * half - S->psi;
}

/* Leading coefficient K(n, n) of side `side` of subdomain j. */
static ocplx or_c0_side(const or_problem *P, int32_t j, int32_t side, int32_t fz) {
  if (P->transmission == OR_TC_ROBIN || P->transmission == OR_TC_S02) return or_c0(P);
  tc_side t = or_tc_side(P, j, side, fz);
  if (or_is_pade(P)) {
    pade_state S;
    ocplx c = 0.0;
    if (pade_init(P, &S) == OR_OK) c = pade_c0(P, &t, &S);
    pade_free(&S);
    return c;
  }
  double a[1] = {1.0}, b[1] = {1.0}, g[1] = {1.0};
  return or_tcK(P, &t, 1, 1, a, b, g);
}

/* S v_n, n = 1..nsteps, of the discrete transmission operator of one
 * boundary point with interface data (W, dnW) applied to the trace sequence
 * v_0..v_nsteps (test hook for the operator pins; same code as the march). */
int32_t or_tc_apply(const or_problem *P, double W, double dnW, int32_t nsteps, const ocplx *v, ocplx *Sv) {
  if (nsteps < 1) return OR_ERR_ARG;
  tc_side t = {W, dnW, 0};
  if (or_is_pade(P)) {
    pade_state S;
    int32_t st = pade_init(P, &S);
    if (st) { pade_free(&S); return st; }
    const ocplx c0 = pade_c0(P, &t, &S);
    for (int32_t n = 1; n <= nsteps; n++) {
      Sv[n - 1] = c0 * v[n] + pade_hist(P, &t, &S);
      pade_advance(P, &t, &S, v[n]);
    }
    pade_free(&S);
    return OR_OK;
  }
  double *al = (double *)calloc((size_t)nsteps + 1, sizeof(double));
  double *be = (double *)calloc((size_t)nsteps + 1, sizeof(double));
  double *ga = (double *)calloc((size_t)nsteps + 1, sizeof(double));
  if (!al || !be || !ga) { free(al); free(be); free(ga); return OR_OOM; }
  or_coeffs(nsteps + 1, al, be, ga);
  for (int32_t n = 1; n <= nsteps; n++) {
    ocplx acc = 0.0;
    for (int32_t s = 0; s <= n; s++) acc += or_tcK(P, &t, n, s, al, be, ga) * v[s];
    Sv[n - 1] = acc;
  }
  free(al); free(be); free(ga);
  return OR_OK;
}

/* Nodal W_n on subdomain j: W_n = (V_n + V_{n-1})/2. */
static void or_local_W(const or_problem *P, int32_t j, int32_t n, int32_t fz,
                       int32_t Nx, int32_t NT, int32_t Nj, double *W) {
  int32_t m = Nx / P->N, g0 = (j - 1) * m;
  for (int32_t k = 0; k < Nj; k++) W[k] = 0.0;
  if (fz) return;
  if (P->potential == OR_POT_VX) {
    for (int32_t k = 0; k < Nj; k++) W[k] = P->V_x[g0 + k];
  } else if (P->potential == OR_POT_VTX) {
    for (int32_t t = 0; t < P->n_terms; t++) {
      const double *tau = P->tau + (size_t)t * (NT + 1);
      const double *xi = P->xi + (size_t)t * (Nx + 1);
      double tb = MUT(2) ? tau[n] : 0.5 * (tau[n] + tau[n - 1]);
      for (int32_t k = 0; k < Nj; k++) W[k] += tb * xi[g0 + k];
    }
  }
}

/* (A_{j,n} - B_{j,n}) of eq. (9):
 * A = (2i/dt) M - S + M_{W_n}; B subtracts the leading coefficient c0 of
 * the transmission operator on each interface row (derived from the weak
 * form: the boundary term dn v = l - S v moves c0 v to the left side).
 * The nonlinear matrix of eq. (12) is the same with W = 0. */
int32_t or_subdomain_matrix(const or_problem *P, int32_t j, int32_t n, int32_t fz,
                            ocplx *lo, ocplx *di, ocplx *up) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return OR_ERR_ARG;
  double *W = (double *)malloc(sizeof(double) * Nj * 7);
  if (!W) return OR_OOM;
  double *Md = W + Nj, *Mo = Md + Nj, *Sd = Mo + Nj, *So = Sd + Nj, *Wd = So + Nj, *Wo = Wd + Nj;
  or_local_W(P, j, n, fz, Nx, NT, Nj, W);
  or_fem(Nj, P->dx, W, Md, Mo, Sd, So, Wd, Wo);
  ocplx s = 2.0 * I_ / P->dt;
  for (int32_t k = 0; k < Nj; k++) di[k] = s * Md[k] - Sd[k] + Wd[k];
  for (int32_t k = 0; k + 1 < Nj; k++) {
    ocplx off = s * Mo[k] - So[k] + Wo[k];
    up[k] = off;
    lo[k + 1] = off;
  }
  lo[0] = 0.0;
  up[Nj - 1] = 0.0;
  if (j >= 2) di[0] -= or_c0_side(P, j, 0, fz);
  if (j <= P->N - 1) di[Nj - 1] -= or_c0_side(P, j, 1, fz);
  free(W);
  return OR_OK;
}

/* ------------------------------------------------------------------ */
/* One whole-window march of subdomain j over n = 1..N_T.              */
/* v-form of Crank-Nicolson: v_n = (u_n + u_{n-1})/2,      */
/* v_0 = u_0, u_n = 2 v_n - u_{n-1}.  Local system eq. (9):    */
/*   (A - B) v_n = (2i/dt) M u_{n-1} + b_n - Q^T (l_n, r_n)^T          */
/* with the history vector b_n = H e_0 (+ H e_end), H = c2 sum_{s<n}   */
/* beta_{n-s} v_s.  Outputs by eq. (8):         */
/*   r_{j-1,n} = -l_{j,n} + 2 S v_{j,n}(a_j),                          */
/*   l_{j+1,n} = -r_{j,n} + 2 S v_{j,n}(b_j).                          */
/* Nonlinear f(u) = lambda|u|^2: per step the fixed point  */
/*   (A_NL - B) z^{s+1} = (2i/dt) M u_{n-1} - M_{f(z^s)} z^s + b - Q^T(l,r)
 * from z^0 = v_{n-1}, stopped by the relative max-norm test (A3, A4). */
/* ------------------------------------------------------------------ */
int32_t or_march(const or_problem *P, int32_t j, const ocplx *lin, const ocplx *rin,
                 int32_t use_u0, int32_t fz, ocplx *out_left, ocplx *out_right,
                 ocplx *uT, int32_t *fp_max) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return OR_ERR_ARG;
  if (j < 1 || j > P->N) return OR_ERR_ARG;
  int32_t N = P->N, m = Nx / N, g0 = (j - 1) * m;
  int32_t has_left = (j >= 2), has_right = (j <= N - 1);
  int32_t pot = fz ? OR_POT_ZERO : P->potential;
  int32_t hist = (P->transmission != OR_TC_ROBIN);
  tc_side tL = or_tc_side(P, j, 0, fz), tR = or_tc_side(P, j, 1, fz);
  /* the neighbour's operator at the same interface node: opposite normal */
  tc_side tLo = tL, tRo = tR;
  tLo.dnW = -tL.dnW;
  tRo.dnW = -tR.dnW;
  size_t nb = (size_t)Nj;
  ocplx *u = (ocplx *)calloc(nb, sizeof(ocplx));
  ocplx *v = (ocplx *)calloc(nb, sizeof(ocplx));
  ocplx *vprev = (ocplx *)calloc(nb, sizeof(ocplx));
  ocplx *rhs = (ocplx *)calloc(nb, sizeof(ocplx));
  ocplx *rhs2 = (ocplx *)calloc(nb, sizeof(ocplx));
  ocplx *lo = (ocplx *)calloc(nb, sizeof(ocplx));
  ocplx *di = (ocplx *)calloc(nb, sizeof(ocplx));
  ocplx *up = (ocplx *)calloc(nb, sizeof(ocplx));
  ocplx *va = (ocplx *)calloc((size_t)NT + 1, sizeof(ocplx));
  ocplx *vb = (ocplx *)calloc((size_t)NT + 1, sizeof(ocplx));
  double *beta = (double *)calloc((size_t)NT + 1, sizeof(double));
  double *alpha = (double *)calloc((size_t)NT + 1, sizeof(double));
  double *gamma = (double *)calloc((size_t)NT + 1, sizeof(double));
  double *Md = (double *)calloc(nb, sizeof(double));
  double *Mo = (double *)calloc(nb, sizeof(double));
  double *Wz = (double *)calloc(nb, sizeof(double));
  double *Wd = (double *)calloc(nb, sizeof(double));
  double *Wo = (double *)calloc(nb, sizeof(double));
  int32_t st = OR_OK;
  pade_state pL, pR;
  memset(&pL, 0, sizeof pL);
  memset(&pR, 0, sizeof pR);
  if (!u || !v || !vprev || !rhs || !rhs2 || !lo || !di || !up || !va || !vb ||
      !beta || !alpha || !gamma || !Md || !Mo || !Wz || !Wd || !Wo) { st = OR_OOM; goto done; }
  if (or_is_pade(P) && ((st = pade_init(P, &pL)) || (st = pade_init(P, &pR)))) goto done;

  or_coeffs(NT + 1, alpha, beta, gamma);
  or_fem(Nj, P->dx, NULL, Md, Mo, NULL, NULL, NULL, NULL);
  ocplx c0L = or_c0_side(P, j, 0, fz), c0R = or_c0_side(P, j, 1, fz);
  /* leading coefficients of the neighbour's operators at a_j, b_j */
  ocplx c0Lo = c0L, c0Ro = c0R;
  if (or_is_pade(P)) {
    c0Lo = pade_c0(P, &tLo, &pL);
    c0Ro = pade_c0(P, &tRo, &pR);
  } else if (P->transmission >= OR_TC_S03) {
    double a1[1] = {1.0}, b1[1] = {1.0}, g1[1] = {1.0};
    c0Lo = or_tcK(P, &tLo, 1, 1, a1, b1, g1);
    c0Ro = or_tcK(P, &tRo, 1, 1, a1, b1, g1);
  }
  ocplx s2 = 2.0 * I_ / P->dt;
  if (use_u0)
    for (int32_t k = 0; k < Nj; k++) u[k] = P->u0[g0 + k];
  for (int32_t k = 0; k < Nj; k++) vprev[k] = u[k];   /* v_0 = u_0 */
  va[0] = u[0];
  vb[0] = u[Nj - 1];
  int32_t time_dep = (pot == OR_POT_VTX);
  if (!time_dep) {
    st = or_subdomain_matrix(P, j, 1, fz, lo, di, up);
    if (st) goto done;
  }
  int32_t fpm = 0, fp_fail = 0;
  for (int32_t n = 1; n <= NT; n++) {
    if (time_dep) { st = or_subdomain_matrix(P, j, n, fz, lo, di, up); if (st) goto done; }
    /* (2i/dt) M u_{n-1} */
    for (int32_t k = 0; k < Nj; k++) {
      ocplx mu = Md[k] * u[k];
      if (k > 0) mu += Mo[k - 1] * u[k - 1];
      if (k + 1 < Nj) mu += Mo[k] * u[k + 1];
      rhs[k] = s2 * mu;
    }
    /* history H_n = sum_{s<n} K(n, s) v_s of each side */
    ocplx Ha = 0.0, Hb = 0.0, Hao = 0.0, Hbo = 0.0;   /* own side; neighbour's operator */
    if (hist) {
      if (P->transmission == OR_TC_S02) {   /* c2 factored out */
        for (int32_t s = 0; s < n; s++) {
          const int32_t ds = MUT(8) ? n - s - 1 : n - s;
          Ha += beta[ds] * va[s];
          Hb += beta[ds] * vb[s];
        }
        Ha = or_c2(P) * Ha;
        Hb = or_c2(P) * Hb;
        Hao = Ha;
        Hbo = Hb;
      } else if (or_is_pade(P)) {   /* auxiliary recursions */
        Ha = pade_hist(P, &tL, &pL);
        Hb = pade_hist(P, &tR, &pR);
        Hao = pade_hist(P, &tLo, &pL);
        Hbo = pade_hist(P, &tRo, &pR);
      } else {
        for (int32_t s = 0; s < n; s++) {
          Ha += or_tcK(P, &tL, n, s, alpha, beta, gamma) * va[s];
          Hb += or_tcK(P, &tR, n, s, alpha, beta, gamma) * vb[s];
          Hao += or_tcK(P, &tLo, n, s, alpha, beta, gamma) * va[s];
          Hbo += or_tcK(P, &tRo, n, s, alpha, beta, gamma) * vb[s];
        }
      }
    }
    if (has_left) rhs[0] += Ha - (lin ? lin[n - 1] : 0.0);
    if (has_right) rhs[Nj - 1] += Hb - (rin ? rin[n - 1] : 0.0);
    if (pot == OR_POT_CUBIC) {
      /* zeta^0 = v_{n-1}; v holds the iterate. */
      for (int32_t k = 0; k < Nj; k++) v[k] = vprev[k];
      int32_t it, conv = 0;
      for (it = 1; it <= P->maxit_fp; it++) {
        for (int32_t k = 0; k < Nj; k++)
          Wz[k] = P->lambda * (creal(v[k]) * creal(v[k]) + cimag(v[k]) * cimag(v[k]));
        or_fem(Nj, P->dx, Wz, NULL, NULL, NULL, NULL, Wd, Wo);
        for (int32_t k = 0; k < Nj; k++) {
          ocplx bf = Wd[k] * v[k];
          if (k > 0) bf += Wo[k - 1] * v[k - 1];
          if (k + 1 < Nj) bf += Wo[k] * v[k + 1];
          rhs2[k] = MUT(1) ? rhs[k] + bf : rhs[k] - bf;
        }
        st = or_thomas(Nj, lo, di, up, rhs2, rhs2);
        if (st) goto done;
        double dmax = 0.0, nmax = 0.0;
        for (int32_t k = 0; k < Nj; k++) {
          double dd = cabs(rhs2[k] - v[k]), nn = cabs(rhs2[k]);
          if (dd > dmax) dmax = dd;
          if (nn > nmax) nmax = nn;
          v[k] = rhs2[k];
        }
        if (dmax <= P->tol_fp * nmax) { conv = 1; break; }
      }
      if (!conv) { it = P->maxit_fp; fp_fail = 1; }
      if (it > fpm) fpm = it;
    } else {
      st = or_thomas(Nj, lo, di, up, rhs, v);
      if (st) goto done;
    }
    for (int32_t k = 0; k < Nj; k++) {
      u[k] = 2.0 * v[k] - u[k];
      vprev[k] = v[k];
    }
    va[n] = v[0];
    vb[n] = v[Nj - 1];
    if (or_is_pade(P)) {
      pade_advance(P, &tL, &pL, v[0]);
      pade_advance(P, &tR, &pR, v[Nj - 1]);
    }
    /* eq. (8) with the neighbour's operator: r_{j-1} = -l_j +
     * (S_{a_j} + S_{b_{j-1}}) v(a_j); the two coincide except for the terms
     * odd in the normal derivative of W (S0^4, S1^4, reading A25) */
    if (has_left && out_left)
      out_left[n - 1] = -(lin ? lin[n - 1] : 0.0) + (c0L * v[0] + Ha) + (c0Lo * v[0] + Hao);
    if (has_right && out_right)
      out_right[n - 1] = -(rin ? rin[n - 1] : 0.0) + (c0R * v[Nj - 1] + Hb) + (c0Ro * v[Nj - 1] + Hbo);
  }
  if (uT) for (int32_t k = 0; k < Nj; k++) uT[k] = u[k];
  if (fp_max && fpm > *fp_max) *fp_max = fpm;
  if (fp_fail) st = OR_INNER_NOT_CONVERGED;
done:
  free(u); free(v); free(vprev); free(rhs); free(rhs2); free(lo); free(di); free(up);
  free(va); free(vb); free(beta); free(alpha); free(gamma); free(Md); free(Mo); free(Wz); free(Wd); free(Wo);
  pade_free(&pL); pade_free(&pR);
  return st;
}

/* Slot of l_j (j = 2..N) and r_j (j = 1..N-1) in g. */
static int32_t slot_l(int32_t j) { return 2 * j - 3; }
static int32_t slot_r(int32_t j) { return 2 * j - 2; }

/* One march of every subdomain j = 1..N with the incoming fluxes of g
 * (NULL = 0); the outputs land in the neighbours' slots of Rg (NULL: none)
 * and the local u(T) in uloc + (j-1) N_j (NULL: none).  The subdomains are
 * independent (each writes its own two slots), so they run in parallel. */
typedef struct {
  const or_problem *P;
  const ocplx *g;
  int32_t use_u0, fz, NT, Nj;
  ocplx *Rg, *uloc;
  int32_t *st, *fp;
} sweep_ctx;

static void sweep_item(void *c, int64_t i) {
  sweep_ctx *S = (sweep_ctx *)c;
  const int32_t j = (int32_t)i + 1, N = S->P->N, NT = S->NT;
  const ocplx *lin = (j >= 2 && S->g) ? S->g + (size_t)slot_l(j) * NT : NULL;
  const ocplx *rin = (j <= N - 1 && S->g) ? S->g + (size_t)slot_r(j) * NT : NULL;
  ocplx *ol = (j >= 2 && S->Rg) ? S->Rg + (size_t)slot_r(j - 1) * NT : NULL;
  ocplx *orr = (j <= N - 1 && S->Rg) ? S->Rg + (size_t)slot_l(j + 1) * NT : NULL;
  ocplx *ut = S->uloc ? S->uloc + (size_t)i * S->Nj : NULL;
  S->fp[i] = 0;
  S->st[i] = or_march(S->P, j, lin, rin, S->use_u0, S->fz, ol, orr, ut, &S->fp[i]);
}

/* status: the first hard error in subdomain order, else INNER_NOT_CONVERGED
 * if any subdomain's NL fixed point hit its cap, else OK */
static int32_t sweep_all(const or_problem *P, const ocplx *g, int32_t use_u0, int32_t fz, ocplx *Rg, ocplx *uloc,
                         int32_t *fp_max) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return OR_ERR_ARG;
  const int32_t N = P->N;
  int32_t *stv = (int32_t *)calloc((size_t)N, sizeof(int32_t)), *fpv = (int32_t *)calloc((size_t)N, sizeof(int32_t));
  if (!stv || !fpv) { free(stv); free(fpv); return OR_OOM; }
  sweep_ctx S = {P, g, use_u0, fz, NT, Nj, Rg, uloc, stv, fpv};
  par_for(N, sweep_item, &S);
  int32_t st = OR_OK;
  for (int32_t i = 0; i < N; i++) {
    if (stv[i] == OR_INNER_NOT_CONVERGED) { if (st == OR_OK) st = stv[i]; }
    else if (stv[i]) { st = stv[i]; break; }
  }
  for (int32_t i = 0; i < N && fp_max; i++)
    if (fpv[i] > *fp_max) *fp_max = fpv[i];
  free(stv); free(fpv);
  return st;
}

/* g -> R(g): every subdomain marches with its incoming fluxes from g and
 * its outputs land in the neighbours' slots (eq. 13). */
int32_t or_apply_R(const or_problem *P, const ocplx *g, int32_t use_u0, int32_t fz,
                   ocplx *Rg, int32_t *fp_max) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return OR_ERR_ARG;
  int32_t N = P->N;
  size_t ng = (size_t)(2 * N - 2) * NT;
  for (size_t i = 0; i < ng; i++) Rg[i] = 0.0;
  return sweep_all(P, g, use_u0, fz, Rg, NULL, fp_max);
}

/* Probing with u0 = 0 (reading A14): a unit impulse at n = 1 on
 * l_j gives the first columns of X^{j,1} (out_left) and X^{j,3}
 * (out_right); on r_j it gives X^{j,2} and X^{j,4}. */
typedef struct { const or_problem *P; int32_t fz, NT; ocplx *X; const ocplx *e; int32_t *st; } probe_ctx;

static void probe_item(void *c, int64_t i) {
  probe_ctx *Q = (probe_ctx *)c;
  const int32_t j = (int32_t)i + 1, N = Q->P->N, NT = Q->NT;
  ocplx *X1 = Q->X + ((size_t)(j - 1) * 4 + 0) * NT, *X2 = X1 + NT, *X3 = X2 + NT, *X4 = X3 + NT;
  int32_t st = OR_OK;
  if (j >= 2) st = or_march(Q->P, j, Q->e, NULL, 0, Q->fz, X1, (j <= N - 1) ? X3 : NULL, NULL, NULL);
  if (!st && j <= N - 1) st = or_march(Q->P, j, NULL, Q->e, 0, Q->fz, (j >= 2) ? X2 : NULL, X4, NULL, NULL);
  Q->st[i] = st;
}

int32_t or_build_L(const or_problem *P, int32_t fz, ocplx *X) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return OR_ERR_ARG;
  int32_t N = P->N;
  memset(X, 0, sizeof(ocplx) * (size_t)N * 4 * NT);
  ocplx *e = (ocplx *)calloc((size_t)NT, sizeof(ocplx));
  int32_t *stv = (int32_t *)calloc((size_t)N, sizeof(int32_t));
  if (!e || !stv) { free(e); free(stv); return OR_OOM; }
  e[0] = 1.0;
  probe_ctx Q = {P, fz, NT, X, e, stv};
  par_for(N, probe_item, &Q);   /* the probes of different subdomains are independent */
  int32_t st = OR_OK;
  for (int32_t i = 0; i < N && !st; i++) st = stv[i];
  free(e); free(stv);
  return st;
}

/* Causal convolution (x * y)_n = sum_{s<=n} x_{n-s} y_s: the action of a
 * lower-triangular Toeplitz block whose first column is x (Props. 3-4,
 * P:549-707). */
static void conv_add(int32_t NT, const ocplx *x, const ocplx *y, ocplx *out) {
  for (int32_t n = 0; n < NT; n++) {
    ocplx acc = 0.0;
    for (int32_t s = 0; s <= n; s++) acc += x[n - s] * y[s];
    out[n] += acc;
  }
}

/* Lg with the block pattern of eq. (15)/(16).  Subdomain j
 * produces exactly the two output slots r_{j-1} and l_{j+1}, so the
 * subdomains run in parallel. */
typedef struct { int32_t N, NT; const ocplx *X, *g; ocplx *Lg; } applyL_ctx;

static void applyL_item(void *c, int64_t i) {
  const applyL_ctx *A = (const applyL_ctx *)c;
  const int32_t j = (int32_t)i + 1, N = A->N, NT = A->NT;
  const ocplx *X = A->X, *g = A->g;
  const ocplx *X1 = X + ((size_t)(j - 1) * 4 + 0) * NT, *X2 = X1 + NT, *X3 = X2 + NT, *X4 = X3 + NT;
  if (j >= 2) { /* r_{j-1}^{k+1} = X^{j,1} l_j + X^{j,2} r_j */
    ocplx *out = A->Lg + (size_t)slot_r(j - 1) * NT;
    conv_add(NT, X1, g + (size_t)slot_l(j) * NT, out);
    if (j <= N - 1) conv_add(NT, X2, g + (size_t)slot_r(j) * NT, out);
  }
  if (j <= N - 1) { /* l_{j+1}^{k+1} = X^{j,3} l_j + X^{j,4} r_j */
    ocplx *out = A->Lg + (size_t)slot_l(j + 1) * NT;
    if (j >= 2) conv_add(NT, X3, g + (size_t)slot_l(j) * NT, out);
    conv_add(NT, X4, g + (size_t)slot_r(j) * NT, out);
  }
}

void or_apply_L(const or_problem *P, const ocplx *X, const ocplx *g, ocplx *Lg) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return;
  int32_t N = P->N;
  memset(Lg, 0, sizeof(ocplx) * (size_t)(2 * N - 2) * NT);
  applyL_ctx A = {N, NT, X, g, Lg};
  par_for(N, applyL_item, &A);
}

/* Exact P^{-1} = (I - L0)^{-1} (P:1041-1059 define P as
 * I - L0, L0 lower block triangular in time with Toeplitz blocks, Props.
 * 3-4).  Row n of (I - L0)x = y reads
 *   x[n] - L0_0 x[n] = y[n] + sum_{k=1}^{n} L0_k x[n-k],
 * L0_k the lag-k matrix of the block pattern of eq. (15)/(16).  The lag-0
 * matrix T0 = I - L0_0 is assembled densely and LU-factored (partial
 * pivoting) once; every step solves T0 x[n] = (history + y[n]). */
int32_t or_pinv_causal(const or_problem *P, const ocplx *X, const ocplx *y, ocplx *x) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return OR_ERR_ARG;
  const int32_t N = P->N, ns = 2 * N - 2;
  if (ns < 1) return OR_OK;
  ocplx *T = (ocplx *)calloc((size_t)ns * ns, sizeof(ocplx));
  ocplx *h = (ocplx *)calloc((size_t)ns, sizeof(ocplx));
  int32_t *piv = (int32_t *)calloc((size_t)ns, sizeof(int32_t));
  if (!T || !h || !piv) { free(T); free(h); free(piv); return OR_OOM; }
  /* T0 = I - L0_0: the couplings of or_apply_L at lag 0 */
  for (int32_t s = 0; s < ns; s++) T[(size_t)s * ns + s] = 1.0;
  for (int32_t j = 1; j <= N; j++) {
    const ocplx *X1 = X + ((size_t)(j - 1) * 4 + 0) * NT, *X2 = X1 + NT, *X3 = X2 + NT, *X4 = X3 + NT;
    if (j >= 2) {
      T[(size_t)slot_r(j - 1) * ns + slot_l(j)] -= X1[0];
      if (j <= N - 1) T[(size_t)slot_r(j - 1) * ns + slot_r(j)] -= X2[0];
    }
    if (j <= N - 1) {
      if (j >= 2) T[(size_t)slot_l(j + 1) * ns + slot_l(j)] -= X3[0];
      T[(size_t)slot_l(j + 1) * ns + slot_r(j)] -= X4[0];
    }
  }
  /* LU with partial pivoting, in place (Doolittle; L unit lower) */
  for (int32_t c = 0; c < ns; c++) {
    int32_t pr = c;
    for (int32_t r = c + 1; r < ns; r++)
      if (cabs(T[(size_t)r * ns + c]) > cabs(T[(size_t)pr * ns + c])) pr = r;
    piv[c] = pr;
    if (pr != c)
      for (int32_t k = 0; k < ns; k++) {
        ocplx t = T[(size_t)c * ns + k];
        T[(size_t)c * ns + k] = T[(size_t)pr * ns + k];
        T[(size_t)pr * ns + k] = t;
      }
    if (T[(size_t)c * ns + c] == 0.0) { free(T); free(h); free(piv); return OR_ERR_ARG; }
    for (int32_t r = c + 1; r < ns; r++) {
      const ocplx f = T[(size_t)r * ns + c] / T[(size_t)c * ns + c];
      T[(size_t)r * ns + c] = f;
      for (int32_t k = c + 1; k < ns; k++) T[(size_t)r * ns + k] -= f * T[(size_t)c * ns + k];
    }
  }
  for (int32_t n = 0; n < NT; n++) {
    /* h = y[n] + sum_{k=1}^{n} L0_k x[n-k] */
    for (int32_t s = 0; s < ns; s++) h[s] = y[(size_t)s * NT + n];
    for (int32_t j = 1; j <= N; j++) {
      const ocplx *X1 = X + ((size_t)(j - 1) * 4 + 0) * NT, *X2 = X1 + NT, *X3 = X2 + NT, *X4 = X3 + NT;
      const ocplx *xl = (j >= 2) ? x + (size_t)slot_l(j) * NT : NULL;
      const ocplx *xr = (j <= N - 1) ? x + (size_t)slot_r(j) * NT : NULL;
      for (int32_t k = 1; k <= n; k++) {
        if (j >= 2) {
          h[slot_r(j - 1)] += X1[k] * xl[n - k];
          if (j <= N - 1) h[slot_r(j - 1)] += X2[k] * xr[n - k];
        }
        if (j <= N - 1) {
          if (j >= 2) h[slot_l(j + 1)] += X3[k] * xl[n - k];
          h[slot_l(j + 1)] += X4[k] * xr[n - k];
        }
      }
    }
    /* T0 x[n] = h: permute, forward (unit L), backward (U) */
    for (int32_t c = 0; c < ns; c++)
      if (piv[c] != c) { ocplx t = h[c]; h[c] = h[piv[c]]; h[piv[c]] = t; }
    for (int32_t r = 0; r < ns; r++)
      for (int32_t k = 0; k < r; k++) h[r] -= T[(size_t)r * ns + k] * h[k];
    for (int32_t r = ns - 1; r >= 0; r--) {
      for (int32_t k = r + 1; k < ns; k++) h[r] -= T[(size_t)r * ns + k] * h[k];
      h[r] /= T[(size_t)r * ns + r];
    }
    for (int32_t s = 0; s < ns; s++) x[(size_t)s * NT + n] = h[s];
  }
  free(T); free(h); free(piv);
  return OR_OK;
}

/* Order-fixed inner product <x, y> = sum conj(x) y: one partial per
 * subdomain over the slots it owns (l_j, r_j), partials summed in
 * subdomain order. */
typedef struct { int32_t N, NT; const ocplx *x, *y; ocplx *part; } dot_ctx;

static void dot_item(void *c, int64_t i) {
  const dot_ctx *D = (const dot_ctx *)c;
  const int32_t j = (int32_t)i + 1, N = D->N, NT = D->NT;
  ocplx part = 0.0;
  int32_t s_lo = (j >= 2) ? slot_l(j) : slot_r(j);
  int32_t s_hi = (j <= N - 1) ? slot_r(j) : slot_l(j);
  for (size_t q = (size_t)s_lo * NT; q < (size_t)(s_hi + 1) * NT; q++) part += conj(D->x[q]) * D->y[q];
  D->part[i] = part;
}

ocplx or_dot(const or_problem *P, const ocplx *x, const ocplx *y) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return 0.0;
  int32_t N = P->N;
  ocplx total = 0.0;
  ocplx *part = (ocplx *)malloc(sizeof(ocplx) * (size_t)N);
  if (!part) return NAN;
  dot_ctx D = {N, NT, x, y, part};
  par_for(N, dot_item, &D);          /* partials in parallel ... */
  for (int32_t i = 0; i < N; i++) total += part[i];   /* ... summed in subdomain order */
  free(part);
  return total;
}

/* ------------------------------------------------------------------ */
/* GMRES(m) with two passes of classical Gram-Schmidt (reading A6) and */
/* complex Givens rotations; stop when the residual estimate           */
/* |gamma_{k+1}| <= tol ||b||_2 (A5); true residual at each restart.    */
/* ------------------------------------------------------------------ */
/* Element-range loops of the Krylov drivers.  Each element's arithmetic is
 * the sequential one (the basis index runs in order inside an element), so
 * the threads only split the index range. */
typedef struct { size_t n, ldv; ocplx *out; const ocplx *a, *b, *V, *coef; double s; int32_t nv; } vec_ctx;

static void vsub_item(void *c, int64_t k) {
  const vec_ctx *v = (const vec_ctx *)c;
  CHUNK_RANGE(k, v->n, lo, hi);
  for (size_t i = lo; i < hi; i++) v->out[i] = v->a[i] - v->b[i];
}
static void vdiv_item(void *c, int64_t k) {
  const vec_ctx *v = (const vec_ctx *)c;
  CHUNK_RANGE(k, v->n, lo, hi);
  for (size_t i = lo; i < hi; i++) v->out[i] = v->a[i] / v->s;
}
static void vmsub_item(void *c, int64_t k) {   /* out -= sum_q coef_q V_q, q in order */
  const vec_ctx *v = (const vec_ctx *)c;
  CHUNK_RANGE(k, v->n, lo, hi);
  for (int32_t q = 0; q < v->nv; q++) {
    const ocplx *vq = v->V + (size_t)q * v->ldv;
    for (size_t i = lo; i < hi; i++) v->out[i] -= v->coef[q] * vq[i];
  }
}
static void vmadd_item(void *c, int64_t k) {   /* out += sum_q coef_q V_q, q in order */
  const vec_ctx *v = (const vec_ctx *)c;
  CHUNK_RANGE(k, v->n, lo, hi);
  for (int32_t q = 0; q < v->nv; q++) {
    const ocplx *vq = v->V + (size_t)q * v->ldv;
    for (size_t i = lo; i < hi; i++) v->out[i] += v->coef[q] * vq[i];
  }
}
static void vec_sub(size_t n, ocplx *out, const ocplx *a, const ocplx *b) {
  vec_ctx v = {n, 0, out, a, b, NULL, NULL, 0.0, 0};
  par_for(n_chunks(n), vsub_item, &v);
}
static void vec_div(size_t n, ocplx *out, const ocplx *a, double s) {
  vec_ctx v = {n, 0, out, a, NULL, NULL, NULL, s, 0};
  par_for(n_chunks(n), vdiv_item, &v);
}
static void vec_msub(size_t n, ocplx *out, const ocplx *V, size_t ldv, const ocplx *coef, int32_t nv) {
  vec_ctx v = {n, ldv, out, NULL, NULL, V, coef, 0.0, nv};
  par_for(n_chunks(n), vmsub_item, &v);
}
static void vec_madd(size_t n, ocplx *out, const ocplx *V, size_t ldv, const ocplx *coef, int32_t nv) {
  vec_ctx v = {n, ldv, out, NULL, NULL, V, coef, 0.0, nv};
  par_for(n_chunks(n), vmadd_item, &v);
}

typedef int32_t (*or_opfn)(void *ctx, const ocplx *x, ocplx *y);
typedef ocplx (*or_dotfn)(const void *ctx, const ocplx *x, const ocplx *y);

static double vnorm(or_dotfn dot, const void *dctx, const ocplx *x) { return sqrt(creal(dot(dctx, x, x))); }

static int32_t gmres_core(size_t n, or_opfn A, void *actx, or_dotfn dot, const void *dctx,
                          const ocplx *b, ocplx *x, double tol, int32_t m, int32_t maxit, int32_t npass,
                          int32_t *iters, double *hist, int32_t *converged) {
  if (npass < 1) npass = 1;
  *iters = 0;
  *converged = 0;
  double bnorm = vnorm(dot, dctx, b);
  if (bnorm == 0.0) {
    for (size_t i = 0; i < n; i++) x[i] = 0.0;
    *converged = 1;
    return OR_OK;
  }
  ocplx *V = (ocplx *)calloc((size_t)(m + 1) * n, sizeof(ocplx));
  ocplx *H = (ocplx *)calloc((size_t)(m + 1) * m, sizeof(ocplx));
  ocplx *sn = (ocplx *)calloc((size_t)m, sizeof(ocplx));
  double *cs = (double *)calloc((size_t)m, sizeof(double));
  ocplx *gam = (ocplx *)calloc((size_t)m + 1, sizeof(ocplx));
  ocplx *hc = (ocplx *)calloc((size_t)m + 1, sizeof(ocplx));
  ocplx *y = (ocplx *)calloc((size_t)m, sizeof(ocplx));
  ocplx *w = (ocplx *)calloc(n, sizeof(ocplx));
  int32_t st = OR_OK;
  if (!V || !H || !sn || !cs || !gam || !hc || !y || !w) { st = OR_OOM; goto out; }
#define Hm(i, k) H[(size_t)(i) * m + (k)]
  int32_t total = 0, done = 0;
  while (!done) {
    st = A(actx, x, w);
    if (st && st != OR_INNER_NOT_CONVERGED) goto out;
    vec_sub(n, V, b, w);
    double beta = vnorm(dot, dctx, V);
    if (beta <= tol * bnorm) { *converged = 1; break; }
    if (total >= maxit) break;
    vec_div(n, V, V, beta);
    for (int32_t i = 0; i <= m; i++) gam[i] = 0.0;
    gam[0] = beta;
    int32_t k, kend = 0;
    for (k = 0; k < m; k++) {
      ocplx *vk = V + (size_t)k * n, *vk1 = V + (size_t)(k + 1) * n;
      int32_t s = A(actx, vk, w);
      if (s && s != OR_INNER_NOT_CONVERGED) { st = s; goto out; }
      if (s) st = s;
      total++;
      double wn0 = vnorm(dot, dctx, w);
      for (int32_t i = 0; i <= k; i++) Hm(i, k) = 0.0;
      for (int pass = 0; pass < npass; pass++) {    /* classical Gram-Schmidt, npass times */
        for (int32_t i = 0; i <= k; i++) hc[i] = dot(dctx, V + (size_t)i * n, w);
        vec_msub(n, w, V, n, hc, k + 1);           /* w -= sum_i hc_i v_i */
        for (int32_t i = 0; i <= k; i++) Hm(i, k) += hc[i];
      }
      double hk1 = vnorm(dot, dctx, w);
      int32_t breakdown = (hk1 <= 1e-14 * wn0);
      if (!breakdown) vec_div(n, vk1, w, hk1);
      for (int32_t i = 0; i < k; i++) {             /* previous rotations */
        ocplx t = cs[i] * Hm(i, k) + sn[i] * Hm(i + 1, k);
        Hm(i + 1, k) = -conj(sn[i]) * Hm(i, k) + cs[i] * Hm(i + 1, k);
        Hm(i, k) = t;
      }
      ocplx a = Hm(k, k);
      double aa = cabs(a);
      if (aa == 0.0) { cs[k] = 0.0; sn[k] = 1.0; Hm(k, k) = hk1; }
      else {
        double den = sqrt(aa * aa + hk1 * hk1);
        cs[k] = aa / den;
        sn[k] = (a / aa) * hk1 / den;
        Hm(k, k) = (a / aa) * den;
      }
      gam[k + 1] = -conj(sn[k]) * gam[k];
      gam[k] = cs[k] * gam[k];
      double res = cabs(gam[k + 1]);
      if (hist) hist[total - 1] = res;
      kend = k + 1;
      if (res <= tol * bnorm || breakdown) { *converged = 1; done = 1; break; }
      if (total >= maxit) { done = 1; break; }
    }
    /* y = H^{-1} gamma (upper triangular), x += V y */
    for (int32_t i = kend - 1; i >= 0; i--) {
      ocplx acc = gam[i];
      for (int32_t q = i + 1; q < kend; q++) acc -= Hm(i, q) * y[q];
      y[i] = acc / Hm(i, i);
    }
    vec_madd(n, x, V, n, y, kend);                 /* x += sum_i y_i v_i */
  }
#undef Hm
  *iters = total;
out:
  free(V); free(H); free(sn); free(cs); free(gam); free(hc); free(y); free(w);
  return st;
}

/* BiCGStab (van der Vorst 1992; Saad, Iterative Methods, Alg. 7.7), the
 * paper's other Krylov solver (reading A20).  From x0:
 *   r = b - A x, rh = r, p = r;  per iteration: rho = <rh, r>,
 *   p = r + (rho/rho_old)(alpha/omega)(p - omega v) (i > 1), v = A p,
 *   alpha = rho / <rh, v>, s = r - alpha v  [stop if ||s|| <= tol ||b||:
 *   x += alpha p], t = A s, omega = <t, s>/<t, t>, x += alpha p + omega s,
 *   r = s - omega t  [stop if ||r|| <= tol ||b||].
 * One iteration = two operator applications; hist[i] = the stopping norm.
 * rho = 0, <rh, v> = 0 or omega = 0 before convergence: OR_BREAKDOWN. */
static int32_t bicgstab_core(size_t n, or_opfn A, void *actx, or_dotfn dot, const void *dctx,
                             const ocplx *b, ocplx *x, double tol, int32_t maxit,
                             int32_t *iters, double *hist, int32_t *converged) {
  *iters = 0;
  *converged = 0;
  double bnorm = vnorm(dot, dctx, b);
  if (bnorm == 0.0) {
    for (size_t i = 0; i < n; i++) x[i] = 0.0;
    *converged = 1;
    return OR_OK;
  }
  ocplx *r = (ocplx *)calloc(n, sizeof(ocplx)), *rh = (ocplx *)calloc(n, sizeof(ocplx));
  ocplx *p = (ocplx *)calloc(n, sizeof(ocplx)), *v = (ocplx *)calloc(n, sizeof(ocplx));
  ocplx *sv = (ocplx *)calloc(n, sizeof(ocplx)), *t = (ocplx *)calloc(n, sizeof(ocplx));
  int32_t st = OR_OK;
  if (!r || !rh || !p || !v || !sv || !t) { st = OR_OOM; goto out; }
  st = A(actx, x, r);
  if (st && st != OR_INNER_NOT_CONVERGED) goto out;
  for (size_t i = 0; i < n; i++) { r[i] = b[i] - r[i]; rh[i] = r[i]; }
  if (vnorm(dot, dctx, r) <= tol * bnorm) { *converged = 1; goto out; }
  ocplx rho_old = 1.0, alpha = 1.0, omega = 1.0;
  for (int32_t it = 0; it < maxit; it++) {
    ocplx rho = dot(dctx, rh, r);
    if (rho == 0.0) { st = OR_BREAKDOWN; break; }
    if (it == 0) {
      for (size_t i = 0; i < n; i++) p[i] = r[i];
    } else {
      ocplx beta = (rho / rho_old) * (alpha / omega);
      for (size_t i = 0; i < n; i++) p[i] = r[i] + beta * (p[i] - omega * v[i]);
    }
    int32_t s = A(actx, p, v);
    if (s && s != OR_INNER_NOT_CONVERGED) { st = s; break; }
    if (s) st = s;
    ocplx rv = dot(dctx, rh, v);
    if (rv == 0.0) { st = OR_BREAKDOWN; break; }
    alpha = rho / rv;
    for (size_t i = 0; i < n; i++) sv[i] = r[i] - alpha * v[i];
    *iters = it + 1;
    double sn = vnorm(dot, dctx, sv);
    if (sn <= tol * bnorm) {
      for (size_t i = 0; i < n; i++) x[i] += alpha * p[i];
      if (hist) hist[it] = sn;
      *converged = 1;
      break;
    }
    s = A(actx, sv, t);
    if (s && s != OR_INNER_NOT_CONVERGED) { st = s; break; }
    if (s) st = s;
    ocplx ts = dot(dctx, t, sv), tt = dot(dctx, t, t);
    if (tt == 0.0) { st = OR_BREAKDOWN; break; }
    omega = ts / tt;
    for (size_t i = 0; i < n; i++) { x[i] += alpha * p[i] + omega * sv[i]; r[i] = sv[i] - omega * t[i]; }
    double rn = vnorm(dot, dctx, r);
    if (hist) hist[it] = rn;
    if (rn <= tol * bnorm) { *converged = 1; break; }
    if (omega == 0.0) { st = OR_BREAKDOWN; break; }
    rho_old = rho;
  }
out:
  free(r); free(rh); free(p); free(v); free(sv); free(t);
  return st;
}

int32_t or_bicgstab_dense(int32_t n, const ocplx *A, const ocplx *b, ocplx *x, double tol, int32_t maxit,
                          int32_t *iters, double *hist);

/* Dense GMRES (test pin of the Krylov driver). */
typedef struct { int32_t n; const ocplx *A; } dense_ctx;
static int32_t dense_op(void *c, const ocplx *x, ocplx *y) {
  dense_ctx *d = (dense_ctx *)c;
  for (int32_t i = 0; i < d->n; i++) {
    ocplx acc = 0.0;
    for (int32_t k = 0; k < d->n; k++) acc += d->A[(size_t)i * d->n + k] * x[k];
    y[i] = acc;
  }
  return OR_OK;
}
typedef struct { size_t n; } seq_ctx;
static ocplx seq_dot(const void *c, const ocplx *x, const ocplx *y) {
  const seq_ctx *s = (const seq_ctx *)c;
  ocplx acc = 0.0;
  for (size_t i = 0; i < s->n; i++) acc += conj(x[i]) * y[i];
  return acc;
}
int32_t or_bicgstab_dense(int32_t n, const ocplx *A, const ocplx *b, ocplx *x, double tol, int32_t maxit,
                          int32_t *iters, double *hist) {
  dense_ctx d = {n, A};
  seq_ctx s = {(size_t)n};
  int32_t conv = 0;
  int32_t st = bicgstab_core((size_t)n, dense_op, &d, seq_dot, &s, b, x, tol, maxit, iters, hist, &conv);
  if (st) return st;
  return conv ? OR_OK : OR_NOT_CONVERGED;
}

int32_t or_gmres_dense(int32_t n, int32_t gs_passes, const ocplx *A, const ocplx *b, ocplx *x, double tol,
                       int32_t restart, int32_t maxit, int32_t *iters, double *hist) {
  dense_ctx d = {n, A};
  seq_ctx s = {(size_t)n};
  int32_t conv = 0;
  int32_t st = gmres_core((size_t)n, dense_op, &d, seq_dot, &s, b, x, tol, restart, maxit, gs_passes, iters, hist,
                          &conv);
  if (st) return st;
  return conv ? OR_OK : OR_NOT_CONVERGED;
}

/* ------------------------------------------------------------------ */
/* Algorithm drivers.                                                  */
/* ------------------------------------------------------------------ */
typedef struct {
  const or_problem *P;
  const ocplx *X;       /* Toeplitz first columns (L or L0) */
  ocplx *tmp, *tmp2;    /* scratch of n_g */
  size_t ng;
  int32_t inner_total;
  int32_t inner_fail;
  int32_t fp_max;
} drv_ctx;

static ocplx drv_dot(const void *c, const ocplx *x, const ocplx *y) { return or_dot(((const drv_ctx *)c)->P, x, y); }

/* y = (I - L) x (Algorithm 3 step 2, eq. 14). */
static int32_t op_I_minus_L(void *c, const ocplx *x, ocplx *y) {
  drv_ctx *d = (drv_ctx *)c;
  or_apply_L(d->P, d->X, x, y);
  vec_sub(d->ng, y, x, y);
  return OR_OK;
}

/* x = P^{-1} y: GMRES on (I - L0) x = y from x = 0 (eq. Pxg, P:1054-1059,
 * reading A8). */
/* The Krylov solver of the problem (reading A20): BiCGStab if requested,
 * GMRES(restart) otherwise (also for the inner P^{-1} of a fixed point). */
static int32_t krylov_solve(const or_problem *P, size_t n, or_opfn A, void *actx, const void *dctx,
                            const ocplx *b, ocplx *x, double tol, int32_t maxit, int32_t *iters, double *hist,
                            int32_t *conv) {
  if (P->krylov == OR_KRY_BICGSTAB)
    return bicgstab_core(n, A, actx, drv_dot, dctx, b, x, tol, maxit, iters, hist, conv);
  return gmres_core(n, A, actx, drv_dot, dctx, b, x, tol, P->restart, maxit, P->gs_passes, iters, hist, conv);
}

static int32_t apply_Pinv(drv_ctx *d, const ocplx *y, ocplx *x) {
  if (d->P->pinv_exact) return or_pinv_causal(d->P, d->X, y, x);
  for (size_t i = 0; i < d->ng; i++) x[i] = 0.0;
  int32_t it = 0, conv = 0;
  int32_t st = krylov_solve(d->P, d->ng, op_I_minus_L, d, d, y, x, d->P->tol_inner, d->P->maxit_inner, &it, NULL,
                            &conv);
  d->inner_total += it;
  if (!conv) d->inner_fail = 1;
  return st;
}

/* y = (I - L) x = x - R_0(x) matrix-free (Algorithm 2, reading A22). */
static int32_t op_I_minus_L_mf(void *c, const ocplx *x, ocplx *y) {
  drv_ctx *d = (drv_ctx *)c;
  int32_t st = or_apply_R(d->P, x, 0, 0, d->tmp, &d->fp_max);
  if (st) return st;
  vec_sub(d->ng, y, x, d->tmp);
  return OR_OK;
}

/* y = P^{-1} (x - R_0(x)), R_0(x) = R(x; u0 = 0) with the true potential
 * (eq. chp2_algopd_Lpf, readings A7, A10). */
static int32_t op_precond(void *c, const ocplx *x, ocplx *y) {
  drv_ctx *d = (drv_ctx *)c;
  int32_t st = or_apply_R(d->P, x, 0, 0, d->tmp, &d->fp_max);
  if (st) return st;
  vec_sub(d->ng, d->tmp, x, d->tmp);
  return apply_Pinv(d, d->tmp, y);
}

/* Final sweep + assembly of u(T) on the global mesh; each duplicated
 * interface node is the average of its two copies (reading A16). */
static int32_t final_march(const or_problem *P, const ocplx *g, ocplx *uT, int32_t *fp_max) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return OR_ERR_ARG;
  int32_t N = P->N, m = Nx / N;
  ocplx *loc = (ocplx *)calloc((size_t)Nj * N, sizeof(ocplx));
  ocplx *sum = (ocplx *)calloc((size_t)Nx + 1, sizeof(ocplx));
  int *cnt = (int *)calloc((size_t)Nx + 1, sizeof(int));
  int32_t st = OR_OK;
  if (!loc || !sum || !cnt) { st = OR_OOM; goto out; }
  st = sweep_all(P, g, 1, 0, NULL, loc, fp_max);
  if (st && st != OR_INNER_NOT_CONVERGED) goto out;
  for (int32_t j = 1; j <= N; j++) {
    const ocplx *lj = loc + (size_t)(j - 1) * Nj;
    for (int32_t k = 0; k < Nj; k++) { sum[(size_t)(j - 1) * m + k] += lj[k]; cnt[(size_t)(j - 1) * m + k]++; }
  }
  for (int32_t i = 0; i <= Nx; i++) uT[i] = sum[i] / (double)cnt[i];
out:
  free(loc); free(sum); free(cnt);
  return st;
}

int32_t or_monodomain(const or_problem *P, ocplx *uT, int32_t *fp_max) {
  or_problem Q = *P;
  Q.N = 1;
  return or_march(&Q, 1, NULL, NULL, 1, 0, NULL, NULL, uT, fp_max);
}

int32_t or_solve(const or_problem *P, ocplx *uT, or_report *rep, ocplx *g_out) {
  int32_t Nx, NT, Nj;
  if (or_sizes(P, &Nx, &NT, &Nj)) return OR_ERR_ARG;
  if (P->transmission == OR_TC_ROBIN && !(P->robin_p > 0)) return OR_ERR_ARG;
  if (P->transmission < OR_TC_ROBIN || P->transmission > OR_TC_S24) return OR_ERR_ARG;
  if ((P->transmission == OR_TC_S22 || P->transmission == OR_TC_S24) && P->pade_m < 1) return OR_ERR_ARG;
  if (P->transmission >= OR_TC_S03 && !(P->potential == OR_POT_ZERO || P->potential == OR_POT_VX))
    return OR_UNSUPPORTED;   /* higher orders: time-independent potentials */
  int32_t N = P->N;
  or_report dummy;
  if (!rep) rep = &dummy;
  rep->iterations = 0; rep->inner_iterations = 0; rep->fp_max = 0; rep->converged = 1; rep->n_history = 0;
  if (N == 1) return or_monodomain(P, uT, &rep->fp_max);
  int32_t linear = (P->potential != OR_POT_CUBIC);
  if (P->algorithm == OR_ALG_NEW && !(P->potential == OR_POT_ZERO || P->potential == OR_POT_VX))
    return OR_UNSUPPORTED;
  size_t ng = (size_t)(2 * N - 2) * NT;
  drv_ctx d;
  memset(&d, 0, sizeof d);
  d.P = P; d.ng = ng;
  ocplx *X = (ocplx *)calloc((size_t)N * 4 * NT, sizeof(ocplx));
  ocplx *g = (ocplx *)calloc(ng, sizeof(ocplx));
  ocplx *rhs = (ocplx *)calloc(ng, sizeof(ocplx));
  d.tmp = (ocplx *)calloc(ng, sizeof(ocplx));
  d.tmp2 = (ocplx *)calloc(ng, sizeof(ocplx));
  int32_t st = OR_OK, conv = 0, it = 0;
  if (!X || !g || !rhs || !d.tmp || !d.tmp2) { st = OR_OOM; goto out; }
  d.X = X;
  if (P->g0) memcpy(g, P->g0, sizeof(ocplx) * ng);
  if (P->algorithm == OR_ALG_NEW) {
    /* Algorithm 3: build d = R(0) and L,
     * solve (I - L) g = d, final sweep. */
    st = or_apply_R(P, NULL, 1, 0, rhs, &d.fp_max);
    if (st) goto out;
    st = or_build_L(P, 0, X);
    if (st) goto out;
    if (P->krylov == OR_KRY_FIXED_POINT) {
      /* fixed point g^{k+1} = d + L g^k (reading A21) */
      while (it < P->maxit) {
        or_apply_L(P, X, g, d.tmp);
        double diff2 = 0.0;
        for (size_t i = 0; i < ng; i++) {
          const ocplx gn = rhs[i] + d.tmp[i];
          d.tmp2[i] = gn - g[i];
          g[i] = gn;
        }
        diff2 = creal(or_dot(P, d.tmp2, d.tmp2));
        if (rep->history) rep->history[it] = sqrt(diff2);
        it++;
        if (sqrt(diff2) < P->tol) { conv = 1; break; }
      }
    } else {
      st = krylov_solve(P, ng, op_I_minus_L, &d, &d, rhs, g, P->tol, P->maxit, &it, rep->history, &conv);
      if (st) goto out;
    }
    rep->n_history = it;
  } else if (P->algorithm == OR_ALG_CLASSICAL) {
    if (P->krylov == OR_KRY_FIXED_POINT) {
      /* Algorithm 1: g^{k+1} = R(g^k), stop ||g^{k+1} - g^k|| < tol */
      while (it < P->maxit) {
        int32_t s = or_apply_R(P, g, 1, 0, d.tmp, &d.fp_max);
        if (s && s != OR_INNER_NOT_CONVERGED) { st = s; goto out; }
        for (size_t i = 0; i < ng; i++) { d.tmp2[i] = d.tmp[i] - g[i]; g[i] = d.tmp[i]; }
        double diff = sqrt(creal(or_dot(P, d.tmp2, d.tmp2)));
        if (rep->history) rep->history[it] = diff;
        it++;
        if (diff < P->tol) { conv = 1; break; }
      }
      st = OR_OK;
    } else {
      /* Algorithm 2: Krylov on (I - L) g = d, (I - L) g = g - R_0(g)
       * matrix-free, d = R(0; u0); linear potentials only */
      if (!linear) { st = OR_UNSUPPORTED; goto out; }
      st = or_apply_R(P, NULL, 1, 0, rhs, &d.fp_max);
      if (st) goto out;
      st = krylov_solve(P, ng, op_I_minus_L_mf, &d, &d, rhs, g, P->tol, P->maxit, &it, rep->history, &conv);
      if (st && st != OR_INNER_NOT_CONVERGED) goto out;
    }
    rep->n_history = it;
  } else if (linear && P->krylov != OR_KRY_FIXED_POINT) {
    /* Preconditioned Krylov for V(t,x). */
    st = or_build_L(P, 1, X);                       /* L0: V = 0 probes */
    if (st) goto out;
    st = or_apply_R(P, NULL, 1, 0, d.tmp2, &d.fp_max); /* d = R(0; u0) */
    if (st) goto out;
    st = apply_Pinv(&d, d.tmp2, rhs);               /* P^{-1} d */
    if (st && st != OR_INNER_NOT_CONVERGED) goto out;
    st = krylov_solve(P, ng, op_precond, &d, &d, rhs, g, P->tol, P->maxit, &it, rep->history, &conv);
    if (st && st != OR_INNER_NOT_CONVERGED) goto out;
    rep->n_history = it;
  } else {
    /* Preconditioned fixed point for f(u) (eq. chp2_algopd_NL, reading A9),
     * also for V(t,x) when the fixed point is requested:
     * g^{k+1} = g^k - P^{-1}(g^k - R_nl(g^k)), stop ||g^{k+1}-g^k||_2 < tol. */
    st = or_build_L(P, 1, X);
    if (st) goto out;
    while (it < P->maxit) {
      int32_t s = or_apply_R(P, g, 1, 0, d.tmp, &d.fp_max);
      if (s && s != OR_INNER_NOT_CONVERGED) { st = s; goto out; }
      for (size_t i = 0; i < ng; i++) d.tmp[i] = g[i] - d.tmp[i];
      s = apply_Pinv(&d, d.tmp, d.tmp2);
      if (s && s != OR_INNER_NOT_CONVERGED) { st = s; goto out; }
      for (size_t i = 0; i < ng; i++) g[i] = g[i] - d.tmp2[i];
      double diff = sqrt(creal(or_dot(P, d.tmp2, d.tmp2)));
      if (rep->history) rep->history[it] = diff;
      it++;
      if (diff < P->tol) { conv = 1; break; }
    }
    rep->n_history = it;
    st = OR_OK;
  }
  rep->iterations = it;
  rep->inner_iterations = d.inner_total;
  rep->converged = conv;
  {
    int32_t s = final_march(P, g, uT, &d.fp_max);
    if (s && s != OR_INNER_NOT_CONVERGED) { st = s; goto out; }
  }
  rep->fp_max = d.fp_max;
  if (g_out) memcpy(g_out, g, sizeof(ocplx) * ng);
  if (!conv) st = OR_NOT_CONVERGED;
  else if (d.inner_fail) st = OR_INNER_NOT_CONVERGED;
out:
  free(X); free(g); free(rhs); free(d.tmp); free(d.tmp2);
  return st;
}

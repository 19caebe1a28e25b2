// swr_linalg.cu — setup (assembly + factorisation of A - B), the
// block-Toeplitz interface operator, Krylov vector kernels and the u(T)
// gather (PAPER.md = Besse & Xing, arXiv:1503.02564).
#include "swr_common.cuh"
#include "swr_kernels.h"

namespace swr {

// ---------------------------------------------------------------------------
// Assembly + LU pivots of (A_{j} - B_{j}) (eq. 9):
//   A = (2i/dt) M - S + M_W, P1 elements on a uniform mesh,
//   M_W the weighted mass of the linear interpolant of W (reading A2),
//   B subtracts c0 on interface rows.  One thread factors one matrix
//   (sequential Thomas pivots p_k = D_k - E_{k-1}^2 / p_{k-1}, q_k = 1/p_k).
// ---------------------------------------------------------------------------
__global__ void k_factor(const FactorJob *jobs, int njobs, int Nj, double h, double dt, double2 c0,
                         int *err) {
  const int jb = blockIdx.x * blockDim.x + threadIdx.x;
  if (jb >= njobs) return;
  const FactorJob J = jobs[jb];
  const double eim = (2.0 / dt) * (h / 6.0);
  double er_prev = 0.0;
  double2 qprev = cz();
  for (int k = 0; k < Nj; k++) {
    const double Wk = J.W ? J.W[k] : 0.0;
    const double Wl = (J.W && k > 0) ? J.W[k - 1] : 0.0;
    const double Wr = (J.W && k < Nj - 1) ? J.W[k + 1] : 0.0;
    double Md = 0.0, Sd = 0.0, MWd = 0.0;
    if (k > 0) { Md += h / 3.0; Sd += 1.0 / h; MWd += h * (Wl + 3.0 * Wk) / 12.0; }
    if (k < Nj - 1) { Md += h / 3.0; Sd += 1.0 / h; MWd += h * (3.0 * Wk + Wr) / 12.0; }
    double2 D = make_double2(-Sd + MWd, (2.0 / dt) * Md);
    if (k == 0 && J.has_left) D = csub(D, c0);
    if (k == Nj - 1 && J.has_right) D = csub(D, c0);
    double2 p = D;
    if (k > 0) {
      const double2 E = make_double2(er_prev, eim);
      p = csub(D, cmul(E, cmul(E, qprev)));
    }
    if (!(hypot(p.x, p.y) >= 1e-300)) atomicExch(err, 3);  // zero pivot
    const double2 qk = crcp(p);
    const double erk = (k < Nj - 1) ? 1.0 / h + h * (Wk + Wr) / 12.0 : 0.0;
    J.q[k] = qk;
    J.er[k] = erk;
    qprev = qk;
    er_prev = erk;
  }
}

// ---------------------------------------------------------------------------
// y = x - L x with the block pattern of eq. (15)/(16) and
// causal convolutions (x * y)_n = sum_{s<=n} x_{n-s} y_s (Props. 3-4,
// P:549-707).  One CTA per output slot; the (<= 2) first columns and input
// slots are staged in shared memory; thread t computes outputs t and
// NT-1-t so every thread does NT+1 multiply-adds per pair.
//   slot r_{j-1} (even 2j-4):  X^{j,1} * l_j + X^{j,2} * r_j
//   slot l_{j+1} (odd 2j-1):   X^{j,3} * l_j + X^{j,4} * r_j
// X is [N][4][NT] (subdomain-major), g slot-major.
// ---------------------------------------------------------------------------
__global__ void k_toeplitz_I_minus_L(const double2 *__restrict__ X, const double2 *__restrict__ x,
                                     double2 *__restrict__ y, int N, int NT) {
  extern __shared__ double2 ts[];
  const int o = blockIdx.x;  // output slot
  double2 *c1 = ts, *c2 = ts + NT, *i1 = ts + 2 * NT, *i2 = ts + 3 * NT;
  int j, p1, p2, s1, s2;
  if ((o & 1) == 0) {       // r_{j-1}, j = o/2 + 2
    j = o / 2 + 2;
    p1 = 0; s1 = 2 * j - 3;                 // X^{j,1}, l_j
    p2 = 1; s2 = (j <= N - 1) ? 2 * j - 2 : -1;  // X^{j,2}, r_j
  } else {                  // l_{j+1}, j = (o+1)/2
    j = (o + 1) / 2;
    p1 = 2; s1 = (j >= 2) ? 2 * j - 3 : -1;  // X^{j,3}, l_j
    p2 = 3; s2 = 2 * j - 2;                  // X^{j,4}, r_j
  }
  const double2 *X1 = X + ((size_t)(j - 1) * 4 + p1) * NT, *X2 = X + ((size_t)(j - 1) * 4 + p2) * NT;
  for (int n = threadIdx.x; n < NT; n += blockDim.x) {
    c1[n] = (s1 >= 0) ? X1[n] : cz();
    i1[n] = (s1 >= 0) ? x[(size_t)s1 * NT + n] : cz();
    c2[n] = (s2 >= 0) ? X2[n] : cz();
    i2[n] = (s2 >= 0) ? x[(size_t)s2 * NT + n] : cz();
  }
  __syncthreads();
  const double2 *xo = x + (size_t)o * NT;
  double2 *yo = y + (size_t)o * NT;
  for (int t = threadIdx.x; t < (NT + 1) / 2; t += blockDim.x) {
    for (int pass = 0; pass < 2; pass++) {
      const int n = pass == 0 ? t : NT - 1 - t;
      if (pass == 1 && n == t) break;
      double2 a = cz(), b = cz();
      for (int s = 0; s <= n; s++) {
        a = cfma(c1[n - s], i1[s], a);
        b = cfma(c2[n - s], i2[s], b);
      }
      const double2 xv = xo[n];
      yo[n] = make_double2(xv.x - (a.x + b.x), xv.y - (a.y + b.y));
    }
  }
}

// ---------------------------------------------------------------------------
// Krylov vector kernels on the interface vector (n_g = (2N-2) NT complex).
// Order-fixed inner products: one partial per subdomain over the slots it
// owns (l_j, r_j; contiguous), reduced in a fixed tree inside the CTA, then
// partials summed in subdomain order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double2 block_reduce(double2 v, double2 *red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = cadd(v, shfl_down2(v, o));
  if (lane == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = lane < nw ? red[lane] : cz();
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = cadd(v, shfl_down2(v, o));
  }
  return v;
}

// partial[v * N + (j-1)] = sum over subdomain j's entries of conj(V_v) w
__global__ void k_multidot_partial(const double2 *__restrict__ V, size_t ldv, int nvec,
                                   const double2 *__restrict__ w, double2 *partial, int N, int NT) {
  __shared__ double2 red[32];
  const int j = blockIdx.x + 1, v = blockIdx.y;
  const int s_lo = (j >= 2) ? 2 * j - 3 : 0;
  const int s_hi = (j <= N - 1) ? 2 * j - 2 : 2 * j - 3;
  const size_t e0 = (size_t)s_lo * NT, e1 = (size_t)(s_hi + 1) * NT;
  const double2 *Vv = V + (size_t)v * ldv;
  double2 acc = cz();
  for (size_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) acc = cfmaconj(Vv[e], w[e], acc);
  acc = block_reduce(acc, red);
  if (threadIdx.x == 0) partial[(size_t)v * N + (j - 1)] = acc;
}

__global__ void k_multidot_final(const double2 *partial, int nvec, int N, double2 *out) {
  const int v = blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= nvec) return;
  double2 s = cz();
  for (int j = 0; j < N; j++) s = cadd(s, partial[(size_t)v * N + j]);
  out[v] = s;
}

// w -= sum_v h_v V_v
__global__ void k_multi_axpy(const double2 *__restrict__ V, size_t ldv, int nvec, const double2 *__restrict__ h,
                             double2 *__restrict__ w, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double2 acc = w[e];
    for (int v = 0; v < nvec; v++) {
      const double2 hv = h[v], x = V[(size_t)v * ldv + e];
      acc = make_double2(acc.x - (hv.x * x.x - hv.y * x.y), acc.y - (hv.x * x.y + hv.y * x.x));
    }
    w[e] = acc;
  }
}

// y = a * x + b * y (complex a, b)
__global__ void k_axpby(double2 a, const double2 *__restrict__ x, double2 b, double2 *__restrict__ y, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = cfma(a, x[e], cmul(b, y[e]));
}

// z = x - y
__global__ void k_sub(const double2 *x, const double2 *y, double2 *z, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    z[e] = csub(x[e], y[e]);
}

// x += sum_v y_v V_v  (GMRES update)
__global__ void k_multi_update(const double2 *__restrict__ V, size_t ldv, int nvec, const double2 *__restrict__ y,
                               double2 *__restrict__ x, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double2 acc = x[e];
    for (int v = 0; v < nvec; v++) acc = cfma(y[v], V[(size_t)v * ldv + e], acc);
    x[e] = acc;
  }
}

// ---------------------------------------------------------------------------
// u(T) on the global mesh from the per-subdomain finals; each duplicated
// interface node is the mean of its two copies (reading A16).
// ---------------------------------------------------------------------------
__global__ void k_gather_uT(const double2 *__restrict__ loc, int N, int m, int Nj, double2 *__restrict__ uT) {
  const int Nx = N * m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= Nx; i += gridDim.x * blockDim.x) {
    const int j = (i == Nx) ? N - 1 : i / m;   // 0-based owner with local index i - j m
    const int k = i - j * m;
    double2 v = loc[(size_t)j * Nj + k];
    if (k == 0 && j > 0) {
      const double2 w = loc[(size_t)(j - 1) * Nj + m];
      v = make_double2((w.x + v.x) / 2.0, (w.y + v.y) / 2.0);
    }
    uT[i] = v;
  }
}

__global__ void k_fill(double2 *x, double2 v, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) x[e] = v;
}

}  // namespace swr

// swr_linalg.cu — setup (assembly + factorisation of A - B), the
// block-Toeplitz interface operator, Krylov vector kernels and the u(T)
// gather (PAPER.md = Besse & Xing, arXiv:1503.02564).
#include "swr_common.cuh"
#include "swr_kernels.h"
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace swr {

// ---------------------------------------------------------------------------
// Assembly + LU pivots of (A_{j} - B_{j}) (eq. 9):
//   A = (2i/dt) M - S + M_W, P1 elements on a uniform mesh,
//   M_W the weighted mass of the linear interpolant of W (reading A2),
//   B subtracts c0 on interface rows.  One warp factors one matrix
//   (sequential Thomas pivots p_k = D_k - E_{k-1}^2 / p_{k-1}, q_k = 1/p_k).
// ---------------------------------------------------------------------------
__global__ void k_factor(const FactorJob *jobs, int njobs, int Nj, double h, double dt, double2 c0,
                         int *err) {
  // one warp per matrix: the lanes assemble 32 rows at a time (diagonal D_k,
  // Re E_k) and store the results coalesced; lane 0 runs the pivot
  // recurrence p_k = D_k - E_{k-1}^2 / p_{k-1} from shared memory
  __shared__ double2 sD[4][32], sQ[4][32];
  __shared__ double sE[4][32];
  const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jb = blockIdx.x * (blockDim.x >> 5) + wl;
  if (jb >= njobs) return;
  const FactorJob J = jobs[jb];
  const double eim = (2.0 / dt) * (h / 6.0);
  double er_prev = 0.0;
  double2 qprev = cz();
  bool bad = false;
  for (int k0 = 0; k0 < Nj; k0 += 32) {
    const int k = k0 + lane;
    if (k < Nj) {
      const double Wk = J.W ? J.W[k] : 0.0;
      const double Wl = (J.W && k > 0) ? J.W[k - 1] : 0.0;
      const double Wr = (J.W && k < Nj - 1) ? J.W[k + 1] : 0.0;
      double Md = 0.0, Sd = 0.0, MWd = 0.0;
      if (k > 0) { Md += h / 3.0; Sd += 1.0 / h; MWd += h * (Wl + 3.0 * Wk) / 12.0; }
      if (k < Nj - 1) { Md += h / 3.0; Sd += 1.0 / h; MWd += h * (3.0 * Wk + Wr) / 12.0; }
      double2 D = make_double2(-Sd + MWd, (2.0 / dt) * Md);
      if (k == 0 && J.has_left) D = csub(D, J.c0L);
      if (k == Nj - 1 && J.has_right) D = csub(D, J.c0R);
      sD[wl][lane] = D;
      sE[wl][lane] = (k < Nj - 1) ? 1.0 / h + h * (Wk + Wr) / 12.0 : 0.0;
    }
    __syncwarp();
    if (lane == 0) {
      const int kn = min(32, Nj - k0);
      for (int i = 0; i < kn; i++) {
        double2 p = sD[wl][i];
        if (k0 + i > 0) {
          const double2 E = make_double2(er_prev, eim);
          p = csub(p, cmul(E, cmul(E, qprev)));
        }
        if (!(hypot(p.x, p.y) >= 1e-300)) bad = true;   // zero pivot
        qprev = crcp(p);
        sQ[wl][i] = qprev;
        er_prev = sE[wl][i];
      }
    }
    __syncwarp();
    if (k < Nj) {
      J.q[k] = sQ[wl][lane];
      J.er[k] = sE[wl][lane];
    }
    __syncwarp();
  }
  if (lane == 0 && bad) atomicExch(err, 3);
}

// V(t,x) = sum_t tau_t(t) xi_t(x): factorisation of (A_{j,n} - B) for every
// step n (W_n = (V_n + V_{n-1})/2 enters A_{j,n} through M_{W_n}),
// one thread per (subdomain, step); step n's pivots at q + (n-1) stride.
__global__ void k_factor_td(const FactorJob *jobs, int njobs, int Nj, int NT, double h, double dt, double2 c0,
                            const double *tau, const double *xi, int n_terms, int Nx, int m, size_t stride, int *err) {
  const long idx = blockIdx.x * (long)blockDim.x + threadIdx.x;
  if (idx >= (long)njobs * NT) return;
  const int jb = (int)(idx % njobs), n = (int)(idx / njobs) + 1;
  const FactorJob J = jobs[jb];
  (void)Nx; (void)m;
  const double eim = (2.0 / dt) * (h / 6.0);
  auto Wat = [&](int k) -> double {       // W_n at local node k
    double w = 0.0;
    for (int tt = 0; tt < n_terms; tt++) {
      const double tb = 0.5 * (tau[(size_t)tt * (NT + 1) + n] + tau[(size_t)tt * (NT + 1) + n - 1]);
      w += tb * xi[(size_t)tt * (Nx + 1) + J.g0 + k];
    }
    return w;
  };
  double2 *qo = J.q + (size_t)(n - 1) * stride;
  double *eo = J.er + (size_t)(n - 1) * stride;
  double er_prev = 0.0;
  double2 qprev = cz();
  double Wl = 0.0, Wk = Wat(0);
  for (int k = 0; k < Nj; k++) {
    const double Wr = (k < Nj - 1) ? Wat(k + 1) : 0.0;
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
    if (!(hypot(p.x, p.y) >= 1e-300)) atomicExch(err, 3);
    const double2 qk = crcp(p);
    const double erk = (k < Nj - 1) ? 1.0 / h + h * (Wk + Wr) / 12.0 : 0.0;
    qo[k] = qk;
    eo[k] = erk;
    qprev = qk;
    er_prev = erk;
    Wl = Wk;
    Wk = Wr;
  }
}

// ---------------------------------------------------------------------------
// y = x - L x with the block pattern of eq. (15)/(16) and
// causal convolutions (x * y)_n = sum_{s<=n} x_{n-s} y_s (Props. 3-4,
// P:549-707).  One CTA per subdomain j: its two input slots l_j, r_j and
// its four first columns X^{j,1..4} are staged in shared memory (columns
// zero-padded), and it produces both output slots that read them:
//   r_{j-1} = X^{j,1} * l_j + X^{j,2} * r_j      (threads [0, T2))
//   l_{j+1} = X^{j,3} * l_j + X^{j,4} * r_j      (threads [T2, 2 T2))
// Each thread accumulates TR consecutive outputs over blocks of TR input
// samples (2TR-1 column values and TR inputs per block in registers) and
// takes output groups g and G-1-g so the triangular work is balanced.
// X is [N][4][NT] (subdomain-major), g slot-major.
// ---------------------------------------------------------------------------
__global__ void k_toeplitz_I_minus_L(const double2 *__restrict__ X, const double2 *__restrict__ x,
                                     double2 *__restrict__ y, int N, int NT) {
  extern __shared__ double2 ts[];
  const int j = blockIdx.x + 1;
  const int CL = NT + 3 * TR, IL = NT + TR;
  double2 *cbase = ts + 2 * TR;                       // 4 columns, stride CL, index range [-2TR, NT+TR)
  double2 *il = ts + 4 * CL, *ir = il + IL;           // inputs l_j, r_j, index range [0, NT+TR)
  const int sl = (j >= 2) ? 2 * j - 3 : -1, sr = (j <= N - 1) ? 2 * j - 2 : -1;
  const double2 *Xj = X + (size_t)(j - 1) * 4 * NT;
  for (int n = threadIdx.x - 2 * TR; n < NT + TR; n += blockDim.x) {
    const bool in = n >= 0 && n < NT;
#pragma unroll
    for (int pcol = 0; pcol < 4; pcol++) cbase[pcol * CL + n] = in ? Xj[(size_t)pcol * NT + n] : cz();
    if (n >= 0) {
      il[n] = (in && sl >= 0) ? x[(size_t)sl * NT + n] : cz();
      ir[n] = (in && sr >= 0) ? x[(size_t)sr * NT + n] : cz();
    }
  }
  __syncthreads();
  const int G = (NT + TR - 1) / TR, T2 = (G + 1) / 2;
  const int half = threadIdx.x / T2, t = threadIdx.x % T2;
  if (half > 1) return;
  const int o = half == 0 ? 2 * j - 4 : 2 * j - 1;    // r_{j-1} or l_{j+1}
  if ((half == 0 && j < 2) || (half == 1 && j > N - 1)) return;
  const double2 *c1 = cbase + (half == 0 ? 0 : 2) * CL, *c2 = c1 + CL;   // (X^{j,1},X^{j,2}) or (X^{j,3},X^{j,4})
  const double2 *xo = x + (size_t)o * NT;
  double2 *yo = y + (size_t)o * NT;
  for (int pass = 0; pass < 2; pass++) {
    const int g = pass == 0 ? t : G - 1 - t;
    if (pass == 1 && g == t) break;
    const int n0 = g * TR;
    double2 acc[TR];
#pragma unroll
    for (int r = 0; r < TR; r++) acc[r] = cz();
    // blocks of TR input samples: acc[r] += c[n0 + r - s] in[s]
    for (int sb = 0; sb <= n0; sb += TR) {
      double2 cw[2 * TR - 1], iw[TR];
#pragma unroll
      for (int d = 0; d < 2 * TR - 1; d++) cw[d] = c1[n0 - sb + d - (TR - 1)];
#pragma unroll
      for (int q = 0; q < TR; q++) iw[q] = il[sb + q];
#pragma unroll
      for (int q = 0; q < TR; q++)
#pragma unroll
        for (int r = 0; r < TR; r++) acc[r] = cfma(cw[r - q + TR - 1], iw[q], acc[r]);
#pragma unroll
      for (int d = 0; d < 2 * TR - 1; d++) cw[d] = c2[n0 - sb + d - (TR - 1)];
#pragma unroll
      for (int q = 0; q < TR; q++) iw[q] = ir[sb + q];
#pragma unroll
      for (int q = 0; q < TR; q++)
#pragma unroll
        for (int r = 0; r < TR; r++) acc[r] = cfma(cw[r - q + TR - 1], iw[q], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < TR; r++) {
      const int n = n0 + r;
      if (n < NT) {
        const double2 xv = xo[n];
        yo[n] = make_double2(xv.x - acc[r].x, xv.y - acc[r].y);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// FFT form of the same operator (the causal convolutions of Props. 3-4 as
// zero-padded cyclic convolutions of length NF = 4^LOG4 >= 2 N_T - 1).
// Radix-4 Stockham FFT in shared memory, one CTA per sequence, NF/4 threads.
//   k_fft_fwd:   F[q] = FFT(pad(src[q]))           (inputs slots; columns at build)
//   k_fft_apply: y_o  = x_o - IFFT(Fc_a .* Fx_a + Fc_b .* Fx_b)[0:N_T]
// ---------------------------------------------------------------------------
template <int LOG4>
__device__ __forceinline__ void fft4_stockham(double2 *a, double2 *b, const double2 *__restrict__ tw, bool inverse) {
  constexpr int NF = 1 << (2 * LOG4), Q = NF / 4;
  const int jt = threadIdx.x;  // one radix-4 butterfly per thread and stage
  double2 *in = a, *out = b;
#pragma unroll
  for (int st = 0, Ns = 1; st < LOG4; st++, Ns *= 4) {
    const int km = jt % Ns;
    double2 v[4];
#pragma unroll
    for (int r = 0; r < 4; r++) {
      v[r] = in[jt + r * Q];
      if (r > 0) {
        double2 wv = tw[(km * r * (NF / (4 * Ns))) & (NF - 1)];
        if (inverse) wv.y = -wv.y;
        v[r] = cmul(v[r], wv);
      }
    }
    const double2 a0 = cadd(v[0], v[2]), a1 = csub(v[0], v[2]), a2 = cadd(v[1], v[3]);
    const double2 d13 = csub(v[1], v[3]);
    const double2 a3 = inverse ? make_double2(-d13.y, d13.x) : make_double2(d13.y, -d13.x);  // (+-i)(v1 - v3)
    const int od = (jt / Ns) * Ns * 4 + km;
    out[od] = cadd(a0, a2);
    out[od + Ns] = cadd(a1, a3);
    out[od + 2 * Ns] = csub(a0, a2);
    out[od + 3 * Ns] = csub(a1, a3);
    __syncthreads();
    double2 *t = in; in = out; out = t;
  }
  if (LOG4 & 1) {  // result is in b: copy back to a
    for (int i = jt; i < NF; i += Q) a[i] = b[i];
    __syncthreads();
  }
}

template <int LOG4>
__global__ void k_fft_fwd(const double2 *__restrict__ src, size_t src_stride, int NT, const double2 *__restrict__ tw,
                          double2 *__restrict__ F) {
  constexpr int NF = 1 << (2 * LOG4), Q = NF / 4;
  __shared__ double2 a[NF], b[NF];
  const double2 *s = src + (size_t)blockIdx.x * src_stride;
  for (int i = threadIdx.x; i < NF; i += Q) a[i] = (i < NT) ? s[i] : cz();
  __syncthreads();
  fft4_stockham<LOG4>(a, b, tw, false);
  double2 *f = F + (size_t)blockIdx.x * NF;
  for (int i = threadIdx.x; i < NF; i += Q) f[i] = a[i];
}

// Fx: [2N-2][NF] transforms of the input slots; Fc: [N][4][NF] of the columns.
template <int LOG4>
__global__ void k_fft_apply(const double2 *__restrict__ Fc, const double2 *__restrict__ Fx,
                            const double2 *__restrict__ x, double2 *__restrict__ y, int N, int NT,
                            const double2 *__restrict__ tw) {
  constexpr int NF = 1 << (2 * LOG4), Q = NF / 4;
  __shared__ double2 a[NF], b[NF];
  const int o = blockIdx.x;
  int j, p1, p2, s1, s2;
  if ((o & 1) == 0) { j = o / 2 + 2; p1 = 0; s1 = 2 * j - 3; p2 = 1; s2 = (j <= N - 1) ? 2 * j - 2 : -1; }
  else { j = (o + 1) / 2; p1 = 2; s1 = (j >= 2) ? 2 * j - 3 : -1; p2 = 3; s2 = 2 * j - 2; }
  const double2 *c1 = Fc + ((size_t)(j - 1) * 4 + p1) * NF, *c2 = Fc + ((size_t)(j - 1) * 4 + p2) * NF;
  for (int i = threadIdx.x; i < NF; i += Q) {
    double2 acc = cz();
    if (s1 >= 0) acc = cmul(c1[i], Fx[(size_t)s1 * NF + i]);
    if (s2 >= 0) acc = cfma(c2[i], Fx[(size_t)s2 * NF + i], acc);
    a[i] = acc;
  }
  __syncthreads();
  fft4_stockham<LOG4>(a, b, tw, true);
  const double inv = 1.0 / NF;
  const double2 *xo = x + (size_t)o * NT;
  double2 *yo = y + (size_t)o * NT;
  for (int n = threadIdx.x; n < NT; n += Q) {
    const double2 xv = xo[n];
    yo[n] = make_double2(fma(-inv, a[n].x, xv.x), fma(-inv, a[n].y, xv.y));
  }
}

// Fused form: one CTA per output slot transforms its (<= 2) input slots
// itself (no transformed-input round trip through HBM), multiplies by the
// transformed columns, and inverse-transforms.
template <int LOG4>
__global__ void k_fft_conv(const double2 *__restrict__ Fc, const double2 *__restrict__ x, double2 *__restrict__ y,
                           int N, int NT, const double2 *__restrict__ tw) {
  pdl_wait();
  pdl_trigger();
  constexpr int NF = 1 << (2 * LOG4), Q = NF / 4;
  extern __shared__ double2 fs[];
  double2 *a1 = fs, *a2 = fs + NF, *bb = fs + 2 * NF;   // two transforms + scratch
  const int o = blockIdx.x;
  int j, p1, p2, s1, s2;
  if ((o & 1) == 0) { j = o / 2 + 2; p1 = 0; s1 = 2 * j - 3; p2 = 1; s2 = (j <= N - 1) ? 2 * j - 2 : -1; }
  else { j = (o + 1) / 2; p1 = 2; s1 = (j >= 2) ? 2 * j - 3 : -1; p2 = 3; s2 = 2 * j - 2; }
  for (int i = threadIdx.x; i < NF; i += Q) {
    a1[i] = (s1 >= 0 && i < NT) ? x[(size_t)s1 * NT + i] : cz();
    a2[i] = (s2 >= 0 && i < NT) ? x[(size_t)s2 * NT + i] : cz();
  }
  __syncthreads();
  fft4_stockham<LOG4>(a1, bb, tw, false);
  fft4_stockham<LOG4>(a2, bb, tw, false);
  const double2 *c1 = Fc + ((size_t)(j - 1) * 4 + p1) * NF, *c2 = Fc + ((size_t)(j - 1) * 4 + p2) * NF;
  for (int i = threadIdx.x; i < NF; i += Q) {
    double2 acc = cz();
    if (s1 >= 0) acc = cmul(__ldg(c1 + i), a1[i]);
    if (s2 >= 0) acc = cfma(__ldg(c2 + i), a2[i], acc);
    a1[i] = acc;
  }
  __syncthreads();
  fft4_stockham<LOG4>(a1, bb, tw, true);
  const double inv = 1.0 / NF;
  const double2 *xo = x + (size_t)o * NT;
  double2 *yo = y + (size_t)o * NT;
  for (int n = threadIdx.x; n < NT; n += Q) {
    const double2 xv = xo[n];
    yo[n] = make_double2(fma(-inv, a1[n].x, xv.x), fma(-inv, a1[n].y, xv.y));
  }
}

// ---------------------------------------------------------------------------
// Register FFT form for NF = 1024 (N_T <= 512): four-step 1024 = 32 x 32
// FFTs, one warp per transform, 32 values per thread.  A thread holds the
// column n1 = lane (values x[n1 + 32 n2], n2 = register), runs a 32-point
// radix-2 DIF in registers, multiplies by W_1024^{n1 k2}, the warp
// transposes through padded shared memory (conflict-free), and a second
// 32-point DIF finishes: lane l ends up holding X[l + 32 k1] in register
// bitrev(k1), the same lane/register layout the inverse transform reads.
// Shared-memory traffic is one transpose per transform (the radix-4
// Stockham kernel above moves the whole sequence through shared memory at
// each of its five stages).  One CTA (2 warps) per subdomain j: both input
// slots (l_j, r_j) are transformed once, exchanged, and each warp forms one
// output slot (the X^{j,1..2} and X^{j,3..4} pairs) and inverts it.
// ---------------------------------------------------------------------------
namespace fftr {
// cos / sin (2 pi k / 32), k = 0..8 (first octant + pi/4); the rest by symmetry
__device__ __forceinline__ constexpr double c32(int k) {
  return k == 0 ? 1.0 : k == 1 ? 0.98078528040323043 : k == 2 ? 0.92387953251128674 : k == 3 ? 0.83146961230254524
       : k == 4 ? 0.70710678118654752 : k == 5 ? 0.55557023301960218 : k == 6 ? 0.38268343236508977
       : k == 7 ? 0.19509032201612826 : 0.0;
}
// e^{-+ 2 pi i k / 32} times d (k in [0, 16), constant after unrolling)
template <bool INV>
__device__ __forceinline__ double2 tw32(double2 d, int k) {
  if (k == 0) return d;
  if (k == 8) return INV ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);   // * (+-i)
  const double c = k < 8 ? c32(k) : -c32(16 - k);
  const double sn = k < 8 ? c32(8 - k) : c32(k - 8);                             // sin(2 pi k / 32) >= 0
  const double s = INV ? sn : -sn;
  return make_double2(fma(d.x, c, -d.y * s), fma(d.x, s, d.y * c));
}
__device__ __forceinline__ constexpr int br5(int k) {
  return ((k & 1) << 4) | ((k & 2) << 2) | (k & 4) | ((k & 8) >> 2) | ((k & 16) >> 4);
}
// 32-point radix-2 DIF in registers; output X[k] in v[br5(k)].  HALF: v[16..31] = 0 on input.
template <bool INV, bool HALF>
__device__ __forceinline__ void dif32(double2 (&v)[32]) {
#pragma unroll
  for (int m = 32; m >= 2; m >>= 1) {
#pragma unroll
    for (int b = 0; b < 32; b += m) {
#pragma unroll
      for (int i = 0; i < m / 2; i++) {
        const double2 a = v[b + i];
        if (HALF && m == 32) {
          v[b + i + m / 2] = tw32<INV>(a, i * (32 / m));
        } else {
          const double2 c = v[b + i + m / 2];
          v[b + i] = cadd(a, c);
          v[b + i + m / 2] = tw32<INV>(csub(a, c), i * (32 / m));
        }
      }
    }
  }
}
// 1024-point transform of the warp's sequence: on entry lane n1 holds
// x[n1 + 32 n2] in v[n2]; on exit X[lane + 32 k1] in v[br5(k1)].  T: [32][33].
template <bool INV, bool HALF>
__device__ __forceinline__ void fft1024(double2 (&v)[32], double2 *T, const double2 *__restrict__ tw, int lane) {
  dif32<INV, HALF>(v);                                  // Y[k2] = v[br5(k2)]
  // W^{n1 k2} = W^{n1 a} W^{8 n1 b}, k2 = a + 8 b: W^{n1 a} by a short product
  // chain, W^{8 n1 b} from the table (4 loads per thread instead of 31 gathers)
  double2 wa[8], wb[4];
  wa[0] = make_double2(1.0, 0.0);
  wa[1] = __ldg(tw + lane);
#pragma unroll
  for (int a = 2; a < 8; a++) wa[a] = cmul(wa[a - 1], wa[1]);
  wb[0] = make_double2(1.0, 0.0);
#pragma unroll
  for (int b = 1; b < 4; b++) wb[b] = __ldg(tw + ((8 * b * lane) & 1023));
#pragma unroll
  for (int r = 1; r < 32; r++) {
    const int k2 = br5(r), a = k2 & 7, b = k2 >> 3;
    double2 w = b == 0 ? wa[a] : (a == 0 ? wb[b] : cmul(wa[a], wb[b]));
    if (INV) w.y = -w.y;
    v[r] = cmul(v[r], w);
  }
#pragma unroll
  for (int r = 0; r < 32; r++) T[lane * 33 + br5(r)] = v[r];
  __syncwarp();
#pragma unroll
  for (int n1 = 0; n1 < 32; n1++) v[n1] = T[n1 * 33 + lane];
  __syncwarp();
  dif32<INV, false>(v);
}
}  // namespace fftr

// xs (optional, device): the input is s * x with s = xs->x, and xcopy
// (optional) receives s * x — the GMRES step normalises its new basis vector
// here instead of in a separate pass.
__global__ void __launch_bounds__(64, 6) k_fft_conv_reg(const double2 *__restrict__ Fc, const double2 *__restrict__ x,
                                                     double2 *__restrict__ y, int N, int NT,
                                                     const double2 *__restrict__ tw, const double2 *__restrict__ xs,
                                                     double2 *__restrict__ xcopy) {
  pdl_wait();
  pdl_trigger();
  constexpr int NF = 1024;
  extern __shared__ double2 fsm[];
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *T = fsm + q * (32 * 33);        // per-warp transpose buffer, also the spectrum exchange
  const int j = blockIdx.x + 1;
  const int sidx = q == 0 ? 2 * j - 3 : 2 * j - 2;
  const bool has_in = q == 0 ? j >= 2 : j <= N - 1;
  const double sx = xs ? xs->x : 1.0;
  double2 v[32];
#pragma unroll
  for (int n2 = 0; n2 < 32; n2++) {
    const int n = lane + 32 * n2;
    v[n2] = (n2 < 16 && has_in && n < NT) ? cscale(sx, x[(size_t)sidx * NT + n]) : cz();
    if (xcopy && n2 < 16 && has_in && n < NT) xcopy[(size_t)sidx * NT + n] = v[n2];
  }
  fftr::fft1024<false, true>(v, T, tw, lane);
  // spectra of l_j (warp 0) and r_j (warp 1) in the own buffer (natural
  // order k = lane + 32 k1), read by both warps
#pragma unroll
  for (int k1 = 0; k1 < 32; k1++) T[k1 * 32 + lane] = v[fftr::br5(k1)];
  __syncthreads();
  // warp 0: output slot 2j-4 (l_j side, columns X^{j,1}, X^{j,2}); warp 1: 2j-1 (X^{j,3}, X^{j,4})
  const bool has_out = q == 0 ? j >= 2 : j <= N - 1;
  const int o = q == 0 ? 2 * j - 4 : 2 * j - 1;
  const double2 *c1 = Fc + ((size_t)(j - 1) * 4 + 2 * q) * NF, *c2 = c1 + NF;
  const double2 *other = fsm + (1 - q) * (32 * 33);
  const bool hA = j >= 2, hB = j <= N - 1;
  if (has_out) {
#pragma unroll
    for (int k1 = 0; k1 < 32; k1++) {
      const int k = lane + 32 * k1;
      const double2 own = T[k1 * 32 + lane], oth = other[k1 * 32 + lane];
      const double2 A = q == 0 ? own : oth, B = q == 0 ? oth : own;
      double2 acc = cz();
      if (hA) acc = cmul(__ldg(c1 + k), A);
      if (hB) acc = cfma(__ldg(c2 + k), B, acc);
      v[k1] = acc;
    }
  }
  __syncthreads();   // the other warp has read this warp's buffer
  if (!has_out) return;
  fftr::fft1024<true, false>(v, T, tw, lane);
  const double inv = 1.0 / NF;
  const double2 *xo = x + (size_t)o * NT;
  double2 *yo = y + (size_t)o * NT;
#pragma unroll
  for (int k1 = 0; k1 < 16; k1++) {
    const int n = lane + 32 * k1;
    if (n < NT) {
      const double2 xv = cscale(sx, xo[n]), a = v[fftr::br5(k1)];
      yo[n] = make_double2(fma(-inv, a.x, xv.x), fma(-inv, a.y, xv.y));
    }
  }
}

// Bytes of L2 set aside for persisting accesses on the current device (0: none;
// SWR_L2_PERSIST=0 disables the window).
size_t l2_persist_bytes() {
  static size_t v = [] {
    const char *e = getenv("SWR_L2_PERSIST");
    if (e && strcmp(e, "0") == 0) return (size_t)0;
    size_t lim = 0;
    if (cudaDeviceGetLimit(&lim, cudaLimitPersistingL2CacheSize) != cudaSuccess) return (size_t)0;
    return lim;
  }();
  return v;
}

cudaError_t launch_fft_conv_reg(const double2 *Fc, const double2 *x, double2 *y, int N, int NT, const double2 *tw,
                                cudaStream_t st, const double2 *xs, double2 *xcopy) {
  if (N < 2) return cudaSuccess;
  if (NT > 512) return cudaErrorInvalidValue;
  const size_t smem = (2 * 32 * 33) * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(k_fft_conv_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // the transformed columns (N x 4 x NF complex, 32 MB at C5) are re-read by
  // every apply: ask L2 to keep them (persisting window; the Krylov vectors
  // streamed between applies are normal accesses and do not evict them)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(N);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeAccessPolicyWindow;
  at[1].val.accessPolicyWindow.base_ptr = const_cast<double2 *>(Fc);
  at[1].val.accessPolicyWindow.num_bytes = (size_t)N * 4 * 1024 * sizeof(double2);
  at[1].val.accessPolicyWindow.hitRatio = 1.0f;
  at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = at;
  cfg.numAttrs = l2_persist_bytes() > 0 ? 2 : 1;
  if (cfg.numAttrs == 2 && at[1].val.accessPolicyWindow.num_bytes > l2_persist_bytes()) {
    at[1].val.accessPolicyWindow.hitRatio = (float)l2_persist_bytes() / (float)at[1].val.accessPolicyWindow.num_bytes;
  }
  return cudaLaunchKernelEx(&cfg, k_fft_conv_reg, Fc, x, y, N, NT, tw, xs, xcopy);
}

cudaError_t launch_fft_conv(int log4, const double2 *Fc, const double2 *x, double2 *y, int N, int NT,
                            const double2 *tw, cudaStream_t st) {
  if (N < 2) return cudaSuccess;
  const int nslots = 2 * N - 2;
  const size_t smem = 3 * ((size_t)1 << (2 * log4)) * sizeof(double2);
  switch (log4) {
    case 2: k_fft_conv<2><<<nslots, 4, smem, st>>>(Fc, x, y, N, NT, tw); break;
    case 3: k_fft_conv<3><<<nslots, 16, smem, st>>>(Fc, x, y, N, NT, tw); break;
    case 4: k_fft_conv<4><<<nslots, 64, smem, st>>>(Fc, x, y, N, NT, tw); break;
    case 5: {
      cudaError_t e = cudaFuncSetAttribute(k_fft_conv<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      k_fft_conv<5><<<nslots, 256, smem, st>>>(Fc, x, y, N, NT, tw);
      break;
    }
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

__global__ void k_twiddles(double2 *tw, int NF) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < NF) {
    double sn, cs;
    sincospi(-2.0 * (double)k / (double)NF, &sn, &cs);  // e^{-2 pi i k / NF}
    tw[k] = make_double2(cs, sn);
  }
}

int fft_log4_for(int NT) {
  for (int l = 2; l <= 5; l++)
    if ((1 << (2 * l)) >= 2 * NT - 1) return l;
  return 0;
}

cudaError_t launch_fft_fwd(int log4, const double2 *src, size_t stride, int count, int NT, const double2 *tw,
                           double2 *F, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  switch (log4) {
    case 2: k_fft_fwd<2><<<count, 4, 0, st>>>(src, stride, NT, tw, F); break;
    case 3: k_fft_fwd<3><<<count, 16, 0, st>>>(src, stride, NT, tw, F); break;
    case 4: k_fft_fwd<4><<<count, 64, 0, st>>>(src, stride, NT, tw, F); break;
    case 5: k_fft_fwd<5><<<count, 256, 0, st>>>(src, stride, NT, tw, F); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_fft_apply(int log4, const double2 *Fc, const double2 *Fx, const double2 *x, double2 *y, int N,
                             int NT, const double2 *tw, cudaStream_t st) {
  if (N < 2) return cudaSuccess;
  const int nslots = 2 * N - 2;
  switch (log4) {
    case 2: k_fft_apply<2><<<nslots, 4, 0, st>>>(Fc, Fx, x, y, N, NT, tw); break;
    case 3: k_fft_apply<3><<<nslots, 16, 0, st>>>(Fc, Fx, x, y, N, NT, tw); break;
    case 4: k_fft_apply<4><<<nslots, 64, 0, st>>>(Fc, Fx, x, y, N, NT, tw); break;
    case 5: k_fft_apply<5><<<nslots, 256, 0, st>>>(Fc, Fx, x, y, N, NT, tw); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
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
  pdl_wait();
  pdl_trigger();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = cfma(a, x[e], cmul(b, y[e]));
}

// z = a x + b y (z may alias x or y)
__global__ void k_lin2(double2 *z, double2 a, const double2 *x, double2 b, const double2 *y, size_t n) {
  pdl_wait();
  pdl_trigger();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    z[e] = cfma(a, x[e], cmul(b, y[e]));
}

// BiCGStab updates in the oracle's order (reading A20):
//   p = r + beta (p - omega v)
__global__ void k_bicg_p(double2 *__restrict__ p, const double2 *__restrict__ r, const double2 *__restrict__ v,
                         double2 beta, double2 omega, size_t n) {
  pdl_wait();
  pdl_trigger();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    p[e] = cadd(r[e], cmul(beta, csub(p[e], cmul(omega, v[e]))));
}
//   x += alpha p + omega s;  r = s - omega t
__global__ void k_bicg_xr(double2 *__restrict__ x, double2 *__restrict__ r, const double2 *__restrict__ p,
                          const double2 *__restrict__ sv, const double2 *__restrict__ t, double2 alpha, double2 omega,
                          size_t n) {
  pdl_wait();
  pdl_trigger();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    x[e] = cadd(x[e], cadd(cmul(alpha, p[e]), cmul(omega, sv[e])));
    r[e] = csub(sv[e], cmul(omega, t[e]));
  }
}

// z = x - y
__global__ void k_sub(const double2 *x, const double2 *y, double2 *z, size_t n) {
  pdl_wait();
  pdl_trigger();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    z[e] = csub(x[e], y[e]);
}

// x += sum_v y_v V_v  (GMRES update)
__global__ void k_multi_update(const double2 *__restrict__ V, size_t ldv, int nvec, const double2 *__restrict__ y,
                               double2 *__restrict__ x, size_t n) {
  pdl_wait();
  pdl_trigger();
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
    double2 acc = x[e];
    for (int v = 0; v < nvec; v++) acc = cfma(y[v], V[(size_t)v * ldv + e], acc);
    x[e] = acc;
  }
}

// ---------------------------------------------------------------------------
// Fused CGS kernel over the interface vector (n_g complex entries):
//   mode & CGS_AXPY : w -= sum_v h_v V_v          (h from the device, v < nv)
//   mode & CGS_DOTS : p_v = <V_v, w>              (v < nv, after the axpy)
//   mode & CGS_NORM : p_nv = <w, w>
// Persistent grid over chunks of 32*KE entries.  The 4 warps of a CTA split
// the basis vectors (warp q holds v = q, q+4, ...; lane holds entries
// lane + 32 kk) so each basis value is loaded from HBM exactly once per call
// and kept in registers between the axpy and the dots; the axpy partials of
// the 4 warps meet in shared memory (fixed summation order).  Per-CTA dot
// partials are reduced in a fixed tree; the last CTA sums them over CTAs in a
// fixed order (deterministic) into out[0..nv]; with CGS_SCALE it also stores
// 1/sqrt(out[nv]) in out[nv+1].
// ---------------------------------------------------------------------------
template <int VPW, int KE>
__global__ void __launch_bounds__(128, 4) k_cgs(const double2 *__restrict__ V, size_t ldv, int nv,
                                                const double2 *__restrict__ hsrc, double2 *__restrict__ w, int mode,
                                                double2 *__restrict__ partial, double2 *__restrict__ out,
                                                unsigned *counter, int N, int NT, double2 *__restrict__ out_host) {
  pdl_wait();
  pdl_trigger();
  constexpr int NVMAX = 4 * VPW, CH = 32 * KE;
  __shared__ double2 red[NVMAX + 1][4];
  __shared__ double2 sh[NVMAX];
  __shared__ double2 part[4][CH];
  __shared__ bool last;
  const size_t ntot = (size_t)(2 * N - 2) * NT;
  const size_t nch = (ntot + CH - 1) / CH;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const bool axpy = mode & CGS_AXPY, dots = mode & CGS_DOTS, norm = mode & CGS_NORM;
  if (axpy)
    for (int v = threadIdx.x; v < nv; v += blockDim.x) sh[v] = hsrc[v];
  __syncthreads();
  double2 acc[VPW];
#pragma unroll
  for (int i = 0; i < VPW; i++) acc[i] = cz();
  double nacc = 0.0;
  const bool rev = mode & CGS_REV;
  for (size_t ci = blockIdx.x; ci < nch; ci += gridDim.x) {
    const size_t c = rev ? nch - 1 - ci : ci;
    const size_t base = c * CH + lane;
    double2 x[VPW][KE], we[KE];
#pragma unroll
    for (int i = 0; i < VPW; i++) {
      const int v = wp + 4 * i;
#pragma unroll
      for (int k = 0; k < KE; k++) {
        const size_t e = base + 32 * k;
        x[i][k] = (v < nv && e < ntot) ? V[(size_t)v * ldv + e] : cz();
      }
    }
#pragma unroll
    for (int k = 0; k < KE; k++) {
      const size_t e = base + 32 * k;
      we[k] = e < ntot ? w[e] : cz();
    }
    if (axpy) {
#pragma unroll
      for (int k = 0; k < KE; k++) {
        double2 p = cz();
#pragma unroll
        for (int i = 0; i < VPW; i++)
          if (wp + 4 * i < nv) p = cfma(sh[wp + 4 * i], x[i][k], p);
        part[wp][lane + 32 * k] = p;
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < KE; k++) {
        const int t = lane + 32 * k;
        const double2 p = cadd(cadd(cadd(part[0][t], part[1][t]), part[2][t]), part[3][t]);
        we[k] = csub(we[k], p);
        const size_t e = base + 32 * k;
        if (wp == 0 && e < ntot) w[e] = we[k];
      }
      __syncthreads();
    }
    if (dots) {
#pragma unroll
      for (int i = 0; i < VPW; i++)
#pragma unroll
        for (int k = 0; k < KE; k++) acc[i] = cfmaconj(x[i][k], we[k], acc[i]);
    }
    if (norm && wp == 0) {
#pragma unroll
      for (int k = 0; k < KE; k++) nacc = fma(we[k].x, we[k].x, fma(we[k].y, we[k].y, nacc));
    }
  }
  const int nred = (dots ? nv : 0) + (norm ? 1 : 0);
  if (dots) {
#pragma unroll
    for (int i = 0; i < VPW; i++) {
      const int v = wp + 4 * i;
      double2 a = acc[i];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) a = cadd(a, shfl_down2(a, o));
      if (lane == 0 && v < nv) red[v][0] = a;
    }
  }
  if (norm && wp == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nacc += __shfl_down_sync(0xffffffffu, nacc, o);
    if (lane == 0) red[nred - 1][0] = make_double2(nacc, 0.0);
  }
  __syncthreads();
  if ((int)threadIdx.x < nred) partial[(size_t)threadIdx.x * gridDim.x + blockIdx.x] = red[threadIdx.x][0];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last CTA: one warp per reduced quantity, fixed-order tree over the CTAs
  const int np = gridDim.x;
  for (int v = wp; v < nred; v += 4) {
    double2 sum = cz();
    for (int q = lane; q < np; q += 32) sum = cadd(sum, __ldcg(partial + (size_t)v * np + q));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum = cadd(sum, shfl_down2(sum, o));
    if (lane == 0) {
      out[v] = sum;
      if (out_host) out_host[v] = sum;   // pinned host mirror (read after the step's event)
      if ((mode & CGS_SCALE) && v == nred - 1) out[v + 1] = make_double2(1.0 / sqrt(sum.x), 0.0);
    }
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// The CGS update pass without dots (CGS_AXPY | CGS_NORM [| CGS_SCALE]):
// w -= V h and <w, w>.  No dots means no per-vector sums, so the entries
// split over warps (each warp streams all nv basis vectors for its 32 KE
// entries, four vectors per unrolled step) and no shared-memory exchange or
// barrier sits in the loop.  Norm partials: warp tree, CTA fixed order, the
// last CTA sums the CTAs in a fixed order (deterministic).
template <int KE, int MINB, int VU = 4>
__global__ void __launch_bounds__(256, MINB) k_cgs_axpy(const double2 *__restrict__ V, size_t ldv, int nv,
                                                     const double2 *__restrict__ hsrc, double2 *__restrict__ w,
                                                     int mode, double2 *__restrict__ partial,
                                                     double2 *__restrict__ out, unsigned *counter, size_t ntot,
                                                     double2 *__restrict__ out_host) {
  pdl_wait();
  pdl_trigger();
  __shared__ double2 sh[32];
  __shared__ double red[8];
  __shared__ bool last;
  for (int v = threadIdx.x; v < nv; v += blockDim.x) sh[v] = hsrc[v];
  __syncthreads();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5, nwp = blockDim.x >> 5;
  constexpr int CH = 32 * KE;
  // the whole grid sweeps one front of chunks through memory (reversed with
  // CGS_REV), so consecutive passes meet the tail of the previous one in L2
  const size_t nch = (ntot + CH - 1) / CH, nwarps = (size_t)gridDim.x * nwp;
  const bool rev = mode & CGS_REV;
  const size_t hi = ntot;
  double nacc = 0.0;
  for (size_t ci = (size_t)blockIdx.x * nwp + wp; ci < nch; ci += nwarps) {
    const size_t c = rev ? nch - 1 - ci : ci;
    const size_t base = c * CH + lane;
    double2 we[KE], p[KE];
#pragma unroll
    for (int k = 0; k < KE; k++) {
      const size_t e = base + 32 * k;
      we[k] = e < hi ? w[e] : cz();
      p[k] = cz();
    }
    int v = 0;
    for (; v + VU <= nv; v += VU) {
      double2 x[VU][KE];
#pragma unroll
      for (int j = 0; j < VU; j++)
#pragma unroll
        for (int k = 0; k < KE; k++) {
          const size_t e = base + 32 * k;
          x[j][k] = e < hi ? V[(size_t)(v + j) * ldv + e] : cz();
        }
#pragma unroll
      for (int j = 0; j < VU; j++)
#pragma unroll
        for (int k = 0; k < KE; k++) p[k] = cfma(sh[v + j], x[j][k], p[k]);
    }
    for (; v < nv; v++) {
#pragma unroll
      for (int k = 0; k < KE; k++) {
        const size_t e = base + 32 * k;
        p[k] = cfma(sh[v], e < hi ? V[(size_t)v * ldv + e] : cz(), p[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < KE; k++) {
      const size_t e = base + 32 * k;
      if (e < hi) {
        const double2 r = csub(we[k], p[k]);
        w[e] = r;
        nacc = fma(r.x, r.x, fma(r.y, r.y, nacc));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nacc += __shfl_down_sync(0xffffffffu, nacc, o);
  if (lane == 0) red[wp] = nacc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sacc = 0.0;
    for (int q = 0; q < nwp; q++) sacc += red[q];
    partial[blockIdx.x] = make_double2(sacc, 0.0);
    __threadfence();
    last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last || wp != 0) return;
  __threadfence();
  double sum = 0.0;
  for (int q = lane; q < (int)gridDim.x; q += 32) sum += __ldcg(partial + q).x;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, o);
  if (lane == 0) {
    out[0] = make_double2(sum, 0.0);
    if (out_host) out_host[0] = out[0];
    if (mode & CGS_SCALE) out[1] = make_double2(1.0 / sqrt(sum), 0.0);
    *counter = 0u;
  }
}

// y = s x, s read from the device (the normalisation of a new basis vector)
__global__ void k_scale_dev(const double2 *__restrict__ x, const double2 *__restrict__ sp, double2 *__restrict__ y,
                            size_t n) {
  pdl_wait();
  pdl_trigger();
  const double sc = sp->x;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] = make_double2(x[e].x * sc, x[e].y * sc);
}

// ---------------------------------------------------------------------------
// Same CGS kernel, bulk-copy pipeline form.  One persistent CTA per SM
// streams chunks of CH = 128 EPT entries of the nv basis vectors and of w
// into shared memory with cp.async.bulk (TMA, one 1-D copy per vector row,
// completion counted on a per-stage mbarrier), NS stages deep, so HBM reads
// run ahead of the arithmetic without any thread holding them in registers.
// Thread t owns entries t + 128 k of each chunk: the axpy and the dots of an
// entry are thread-local (no cross-warp reduction per chunk, one CTA barrier
// per chunk to release the stage).  Dot partials: registers over the CTA's
// chunks (fixed order), warp shuffles + shared memory, the last CTA sums the
// per-CTA partials in CTA order.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cgs_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int NVMAX>
__global__ void __launch_bounds__(256, 1) k_cgs_tma(const double2 *__restrict__ V, size_t ldv, int nv,
                                                    const double2 *__restrict__ hsrc, double2 *__restrict__ w,
                                                    int mode, double2 *__restrict__ partial, double2 *__restrict__ out,
                                                    unsigned *counter, size_t ntot, int EPT, int NS,
                                                    double2 *__restrict__ out_host) {
  pdl_wait();
  pdl_trigger();
  constexpr int NH = NVMAX / 2;   // basis vectors per thread (v = 2 i + hf)
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ double2 red[NVMAX + 1][8];
  __shared__ double2 sh[NVMAX];
  __shared__ bool last;
  unsigned long long *mb = reinterpret_cast<unsigned long long *>(smraw);   // [NS]
  double2 *stg = reinterpret_cast<double2 *>(smraw + 128);                  // [NS][nv + 1][CH]
  const int t = threadIdx.x, lane = t & 31, wp = t >> 5, hf = t & 1, el0 = t >> 1;
  const int CH = 128 * EPT, nrow = nv + 1;
  const bool axpy = mode & CGS_AXPY, dots = mode & CGS_DOTS, norm = mode & CGS_NORM;
  const size_t nch = (ntot + CH - 1) / CH;
  const int mine = blockIdx.x < nch ? (int)((nch - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
  if (axpy)
    for (int v = t; v < nv; v += blockDim.x) sh[v] = hsrc[v];
  if (t == 0) {
    for (int i = 0; i < NS; i++)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(cgs_smem_u32(mb + i)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int i) {   // chunk i of this CTA into stage i % NS (warp 0, one row per lane)
    const int sgi = i % NS;
    const size_t base = (blockIdx.x + (size_t)i * gridDim.x) * CH;
    const uint32_t bytes = (uint32_t)(min((size_t)CH, ntot - base) * sizeof(double2));
    const uint32_t mbar = cgs_smem_u32(mb + sgi);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes * nrow) : "memory");
    double2 *dst = stg + (size_t)sgi * nrow * CH;
    for (int v = lane; v <= nv; v += 32) {
      const double2 *src = v < nv ? V + (size_t)v * ldv + base : w + base;
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(cgs_smem_u32(dst + (size_t)v * CH)), "l"(src), "r"(bytes), "r"(mbar) : "memory");
    }
  };
  if (wp == 0)
    for (int i = 0; i < NS - 1 && i < mine; i++) issue(i);
  double2 acc[NH];
#pragma unroll
  for (int v = 0; v < NH; v++) acc[v] = cz();
  double nacc = 0.0;
  for (int i = 0; i < mine; i++) {
    if (wp == 0 && i + NS - 1 < mine) issue(i + NS - 1);   // its stage was released at the end of i - 1
    const int sgi = i % NS;
    {
      const uint32_t mbar = cgs_smem_u32(mb + sgi), par = (uint32_t)((i / NS) & 1);
      uint32_t done = 0;
      while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(mbar), "r"(par) : "memory");
    }
    const double2 *st = stg + (size_t)sgi * nrow * CH;
    const size_t base = (blockIdx.x + (size_t)i * gridDim.x) * CH;
    const int n = (int)min((size_t)CH, ntot - base);
    // lanes 2e, 2e + 1 share entry e (even / odd v); the loop bound is warp-uniform
    // (CH is a multiple of 128) so the pair shuffle always sees the full warp
    for (int e = el0; e < CH; e += 128) {
      const bool ok = e < n;
      double2 we = ok ? st[(size_t)nv * CH + e] : cz();
      if (axpy) {
        double2 p0 = cz(), p1 = cz();
        if (ok) {
#pragma unroll 4
          for (int v = hf; v < nv; v += 4) {
            p0 = cfma(sh[v], st[(size_t)v * CH + e], p0);
            if (v + 2 < nv) p1 = cfma(sh[v + 2], st[(size_t)(v + 2) * CH + e], p1);
          }
        }
        const double2 pm = cadd(p0, p1), po = shfl_xor2(pm, 1);
        const double2 tot = hf == 0 ? cadd(pm, po) : cadd(po, pm);   // (even + odd), same on both lanes
        we = csub(we, tot);
        if (ok && hf == 0) w[base + e] = we;
      }
      if (ok) {
        if (dots) {
#pragma unroll
          for (int k = 0; k < NH; k++)
            if (2 * k + hf < nv) acc[k] = cfmaconj(st[(size_t)(2 * k + hf) * CH + e], we, acc[k]);
        }
        if (norm && hf == 0) nacc = fma(we.x, we.x, fma(we.y, we.y, nacc));
      }
    }
    __syncthreads();   // stage sgi free for chunk i + NS
  }
  const int nred = (dots ? nv : 0) + (norm ? 1 : 0);
  if (dots) {
#pragma unroll
    for (int k = 0; k < NH; k++) {
      if (2 * k < nv) {
        double2 a = acc[k];
#pragma unroll
        for (int o = 16; o > 1; o >>= 1) a = cadd(a, shfl_xor2(a, o));   // lanes of the same parity
        if (lane < 2 && 2 * k + lane < nv) red[2 * k + lane][wp] = a;
      }
    }
  }
  if (norm) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nacc += __shfl_xor_sync(0xffffffffu, nacc, o);
    if (lane == 0) red[nred - 1][wp] = make_double2(nacc, 0.0);
  }
  __syncthreads();
  if (t < nred) {
    double2 sum = red[t][0];
#pragma unroll
    for (int q = 1; q < 8; q++) sum = cadd(sum, red[t][q]);
    partial[(size_t)t * gridDim.x + blockIdx.x] = sum;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) last = (atomicAdd(counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int np = gridDim.x;
  for (int v = wp; v < nred; v += 8) {
    double2 sum = cz();
    for (int q = lane; q < np; q += 32) sum = cadd(sum, __ldcg(partial + (size_t)v * np + q));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum = cadd(sum, shfl_down2(sum, o));
    if (lane == 0) {
      out[v] = sum;
      if (out_host) out_host[v] = sum;   // pinned host mirror (read after the step's event)
      if ((mode & CGS_SCALE) && v == nred - 1) out[v + 1] = make_double2(1.0 / sqrt(sum.x), 0.0);
    }
  }
  if (t == 0) *counter = 0u;
}

template <int NVMAX>
static cudaError_t launch_cgs_tma_t(const double2 *V, size_t ldv, int nv, const double2 *hsrc, double2 *w, int mode,
                                    double2 *partial, double2 *out, unsigned *counter, size_t ntot, cudaStream_t st,
                                    double2 *out_host) {
  // stage = (nv + 1) rows of CH = 128 EPT entries, about 48 KB; up to 4 stages in 200 KB
  const int nrow = nv + 1;
  int EPT = (int)((48 * 1024) / ((size_t)nrow * 128 * sizeof(double2)));
  EPT = EPT < 1 ? 1 : (EPT > 16 ? 16 : EPT);
  const size_t stage = (size_t)nrow * 128 * EPT * sizeof(double2);
  const int NS = (int)std::min<size_t>(4, (200 * 1024) / stage);
  const size_t smem = 128 + (size_t)NS * stage;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_cgs_tma<NVMAX>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
    if (e != cudaSuccess) {
      fprintf(stderr, "k_cgs_tma<%d>: cudaFuncSetAttribute: %s\n", NVMAX, cudaGetErrorString(e));
      return e;
    }
    attr_set = true;
  }
  const size_t nch = (ntot + 128 * EPT - 1) / (128 * EPT);
  const unsigned grid = (unsigned)std::min<size_t>(nch, 148);
  cudaError_t e = launch_pdl(k_cgs_tma<NVMAX>, dim3(grid), dim3(256), smem, st, V, ldv, nv, hsrc, w, mode, partial, out,
                             counter, ntot, EPT, NS, out_host);
  if (e != cudaSuccess) {
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_cgs_tma<NVMAX>);
    fprintf(stderr, "k_cgs_tma<%d>: launch grid %u smem %zu (max dyn %d, static %zu, regs %d, maxthr %d): %s\n", NVMAX, grid,
            smem, fa.maxDynamicSharedSizeBytes, fa.sharedSizeBytes, fa.numRegs, fa.maxThreadsPerBlock, cudaGetErrorString(e));
  }
  return e;
}

cudaError_t launch_cgs(const double2 *V, size_t ldv, int nv, const double2 *hsrc, double2 *w, int mode,
                       double2 *partial, double2 *out, unsigned *counter, int N, int NT, cudaStream_t st,
                       double2 *out_host, size_t vwin, float vratio) {
  if (!V) vwin = 0;
  const size_t ntot = (size_t)(2 * N - 2) * NT;
  if (nv > 32) return cudaErrorInvalidValue;
  // default: register form below; SWR_CGS=tma selects the bulk-copy pipeline
  // form (measured slower at C5: 190 vs 147 ms per solve)
  const char *cgs_env = getenv("SWR_CGS");
  if (cgs_env && strcmp(cgs_env, "tma") == 0) {
    if (nv <= 8) return launch_cgs_tma_t<8>(V, ldv, nv, hsrc, w, mode, partial, out, counter, ntot, st, out_host);
    if (nv <= 16) return launch_cgs_tma_t<16>(V, ldv, nv, hsrc, w, mode, partial, out, counter, ntot, st, out_host);
    return launch_cgs_tma_t<32>(V, ldv, nv, hsrc, w, mode, partial, out, counter, ntot, st, out_host);
  }
  // update pass without dots: entry-split streaming form (SWR_CGS_AXPY=0 disables)
  static const bool axpy_split = !(getenv("SWR_CGS_AXPY") && atoi(getenv("SWR_CGS_AXPY")) == 0);
  if (axpy_split && (mode & CGS_AXPY) && !(mode & CGS_DOTS) && (mode & CGS_NORM) && nv >= 1) {
    // 4 entries x 4 vectors per unrolled step, 2 CTAs of 256 per SM (measured
    // best of KE 1/2/4, 4 or 8 vectors per step, 1-3 CTAs per SM)
    const size_t nwarp_needed = (ntot + 32 * 4 - 1) / (32 * 4);
    const unsigned g = (unsigned)std::min<size_t>((nwarp_needed + 7) / 8, 148 * 2);
    return launch_pdl_win(V, vwin, vratio, k_cgs_axpy<4, 2>, dim3(g), dim3(256), 0, st, V, ldv, nv, hsrc, w, mode,
                          partial, out, counter, ntot, out_host);
  }
  // register form: persistent grid, 4 CTAs of 128 threads per SM (148 SMs); the
  // grid only depends on the sizes, so the reduction order is fixed
  auto grid = [&](int ch) { return (unsigned)std::min<size_t>((ntot + ch - 1) / ch, 148 * 4); };
  if (nv <= 8) return launch_pdl_win(V, vwin, vratio, k_cgs<2, 8>, dim3(grid(256)), dim3(128), 0, st, V, ldv, nv, hsrc, w, mode, partial, out, counter, N, NT, out_host);
  if (nv <= 16) return launch_pdl_win(V, vwin, vratio, k_cgs<4, 4>, dim3(grid(128)), dim3(128), 0, st, V, ldv, nv, hsrc, w, mode, partial, out, counter, N, NT, out_host);
  return launch_pdl_win(V, vwin, vratio, k_cgs<8, 2>, dim3(grid(64)), dim3(128), 0, st, V, ldv, nv, hsrc, w, mode, partial, out, counter, N, NT, out_host);
}

// ---------------------------------------------------------------------------
// u(T) on the global mesh from the per-subdomain finals; each duplicated
// interface node is the mean of its two copies (reading A16).
// ---------------------------------------------------------------------------
// Multi-GPU: this rank holds subdomains [j_lo, j_hi] (1-based); nodes of
// other ranks get 0 and a node shared with another rank gets half of the
// local copy, so the sum over ranks is the mean of the two copies
// ((a + b)/2 == a/2 + b/2 exactly in binary floating point).
__global__ void k_gather_uT(const double2 *__restrict__ loc, int N, int m, int Nj, int j_lo, int j_hi,
                            double2 *__restrict__ uT) {
  const int Nx = N * m;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i <= Nx; i += gridDim.x * blockDim.x) {
    const int j = (i == Nx) ? N - 1 : i / m;   // 0-based owner with local index i - j m
    const int k = i - j * m;
    const bool own = (j + 1 >= j_lo && j + 1 <= j_hi);
    double2 v = own ? loc[(size_t)j * Nj + k] : cz();
    if (k == 0 && j > 0) {                     // interface node: copies in subdomains j-1 and j
      const bool ownl = (j >= j_lo && j <= j_hi);
      const double2 w = ownl ? loc[(size_t)(j - 1) * Nj + m] : cz();
      if (own && ownl) v = make_double2((w.x + v.x) / 2.0, (w.y + v.y) / 2.0);
      else if (own) v = make_double2(v.x / 2.0, v.y / 2.0);
      else if (ownl) v = make_double2(w.x / 2.0, w.y / 2.0);
    }
    uT[i] = v;
  }
}

__global__ void k_fill(double2 *x, double2 v, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) x[e] = v;
}

}  // namespace swr

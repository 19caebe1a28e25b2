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
        if (tiny_pivot(p)) bad = true;   // zero pivot
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
    if (tiny_pivot(p)) atomicExch(err, 3);
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
// X is [N][4][NT] (subdomain-major), x and y the rank's slots (SlotMap):
// one CTA per owned subdomain j = j_lo + blockIdx.x; an output slot owned by
// the neighbour rank receives -(L x) in the halo buffer (the owner adds x).
// ---------------------------------------------------------------------------
__global__ void k_toeplitz_I_minus_L(const double2 *__restrict__ X, const double2 *__restrict__ x,
                                     double2 *__restrict__ y, const SlotMap m) {
  extern __shared__ double2 ts[];
  const int N = m.N, NT = m.NT;
  const int j = m.j_lo + blockIdx.x;
  const int CL = NT + 3 * TR, IL = NT + TR;
  double2 *cbase = ts + 2 * TR;                       // 4 columns, stride CL, index range [-2TR, NT+TR)
  double2 *il = ts + 4 * CL, *ir = il + IL;           // inputs l_j, r_j, index range [0, NT+TR)
  const double2 *xl = (j >= 2) ? slot_ptr(m, x, 2 * j - 3) : nullptr;
  const double2 *xr = (j <= N - 1) ? slot_ptr(m, x, 2 * j - 2) : nullptr;
  const double2 *Xj = X + (size_t)(j - 1) * 4 * NT;
  for (int n = threadIdx.x - 2 * TR; n < NT + TR; n += blockDim.x) {
    const bool in = n >= 0 && n < NT;
#pragma unroll
    for (int pcol = 0; pcol < 4; pcol++) cbase[pcol * CL + n] = in ? Xj[(size_t)pcol * NT + n] : cz();
    if (n >= 0) {
      il[n] = (in && xl) ? xl[n] : cz();
      ir[n] = (in && xr) ? xr[n] : cz();
    }
  }
  __syncthreads();
  const int G = (NT + TR - 1) / TR, T2 = (G + 1) / 2;
  const int half = threadIdx.x / T2, t = threadIdx.x % T2;
  if (half > 1) return;
  const int o = half == 0 ? 2 * j - 4 : 2 * j - 1;    // r_{j-1} or l_{j+1}
  if ((half == 0 && j < 2) || (half == 1 && j > N - 1)) return;
  const double2 *c1 = cbase + (half == 0 ? 0 : 2) * CL, *c2 = c1 + CL;   // (X^{j,1},X^{j,2}) or (X^{j,3},X^{j,4})
  bool remote;
  double2 *yo = out_ptr(m, y, o, remote);
  const double2 *xo = remote ? nullptr : slot_ptr(m, x, o);
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
        const double2 xv = xo ? xo[n] : cz();
        yo[n] = make_double2(xv.x - acc[r].x, xv.y - acc[r].y);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// FFT form of the same operator (the causal convolutions of Props. 3-4 as
// zero-padded cyclic convolutions of length NF = 4^LOG4 >= 2 N_T - 1).
// Radix-4 Stockham FFT in shared memory, one CTA per sequence, NF/4 threads.
//   k_fft_fwd:   F[q] = FFT(pad(src[q]))           (the first columns, at build)
//   k_fft_conv:  y_o  = x_o - IFFT(Fc_a .* FFT(x_a) + Fc_b .* FFT(x_b))[0:N_T]
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

// One CTA per output of an owned subdomain (blockIdx = 2 b + side, j = j_lo +
// b; side 0: r_{j-1} from X^{j,1}, X^{j,2}; side 1: l_{j+1} from X^{j,3},
// X^{j,4}) transforms the (<= 2) input slots l_j, r_j itself, multiplies by
// the transformed columns and inverse-transforms; an output owned by the
// neighbour rank receives -(L x) in the halo buffer.
template <int LOG4>
__global__ void k_fft_conv(const double2 *__restrict__ Fc, const double2 *__restrict__ x, double2 *__restrict__ y,
                           const SlotMap m, const double2 *__restrict__ tw) {
  pdl_wait();
  pdl_trigger();
  constexpr int NF = 1 << (2 * LOG4), Q = NF / 4;
  extern __shared__ double2 fs[];
  double2 *a1 = fs, *a2 = fs + NF, *bb = fs + 2 * NF;   // two transforms + scratch
  const int N = m.N, NT = m.NT;
  const int j = m.j_lo + (int)(blockIdx.x >> 1), side = blockIdx.x & 1;
  if ((side == 0 && j < 2) || (side == 1 && j > N - 1)) return;
  const int o = side == 0 ? 2 * j - 4 : 2 * j - 1, p1 = 2 * side, p2 = 2 * side + 1;
  const double2 *x1 = j >= 2 ? slot_ptr(m, x, 2 * j - 3) : nullptr;       // l_j
  const double2 *x2 = j <= N - 1 ? slot_ptr(m, x, 2 * j - 2) : nullptr;   // r_j
  for (int i = threadIdx.x; i < NF; i += Q) {
    a1[i] = (x1 && i < NT) ? x1[i] : cz();
    a2[i] = (x2 && i < NT) ? x2[i] : cz();
  }
  __syncthreads();
  fft4_stockham<LOG4>(a1, bb, tw, false);
  fft4_stockham<LOG4>(a2, bb, tw, false);
  const double2 *c1 = Fc + ((size_t)(j - 1) * 4 + p1) * NF, *c2 = Fc + ((size_t)(j - 1) * 4 + p2) * NF;
  for (int i = threadIdx.x; i < NF; i += Q) {
    double2 acc = cz();
    if (x1) acc = cmul(__ldg(c1 + i), a1[i]);
    if (x2) acc = cfma(__ldg(c2 + i), a2[i], acc);
    a1[i] = acc;
  }
  __syncthreads();
  fft4_stockham<LOG4>(a1, bb, tw, true);
  const double inv = 1.0 / NF;
  bool remote;
  double2 *yo = out_ptr(m, y, o, remote);
  const double2 *xo = remote ? nullptr : slot_ptr(m, x, o);
  for (int n = threadIdx.x; n < NT; n += Q) {
    const double2 xv = xo ? xo[n] : cz();
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
// 4 CTAs per SM at most (255 registers, no spill: the butterflies of a stage
// stay independent; 6 per SM capped the kernel at 168 registers with spills):
// C5 applies 20.3 -> 18.4 ms per solve, C4 55 -> 46 ms; 8 per SM: 28.5 ms
__global__ void __launch_bounds__(64, 4) k_fft_conv_reg(const double2 *__restrict__ Fc, const double2 *__restrict__ x,
                                                     double2 *__restrict__ y, const SlotMap m,
                                                     const double2 *__restrict__ tw, const double2 *__restrict__ xs,
                                                     double2 *__restrict__ xcopy) {
  pdl_wait();
  pdl_trigger();
  constexpr int NF = 1024;
  extern __shared__ double2 fsm[];
  const int N = m.N, NT = m.NT;
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2 *T = fsm + q * (32 * 33);        // per-warp transpose buffer, also the spectrum exchange
  const int j = m.j_lo + blockIdx.x;       // owned subdomain
  const int sidx = q == 0 ? 2 * j - 3 : 2 * j - 2;
  const bool has_in = q == 0 ? j >= 2 : j <= N - 1;
  const size_t ioff = has_in ? (size_t)(sidx - m.s_lo) * NT : 0;   // input slots are always owned
  const double sx = xs ? xs->x : 1.0;
  double2 v[32];
#pragma unroll
  for (int n2 = 0; n2 < 32; n2++) {
    const int n = lane + 32 * n2;
    v[n2] = (n2 < 16 && has_in && n < NT) ? cscale(sx, x[ioff + n]) : cz();
    if (xcopy && n2 < 16 && has_in && n < NT) xcopy[ioff + n] = v[n2];
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
  bool remote;   // an output owned by the neighbour rank gets -(L s x) only (the owner adds s x)
  double2 *yo = out_ptr(m, y, o, remote);
  // the x loads stay unconditional (the compiler issues them ahead of the
  // inverse transform); a remote output reads the first owned slot, times 0
  const double2 *xo = remote ? x : slot_ptr(m, x, o);
  const double so = remote ? 0.0 : sx;
#pragma unroll
  for (int k1 = 0; k1 < 16; k1++) {
    const int n = lane + 32 * k1;
    if (n < NT) {
      const double2 xv = cscale(so, xo[n]), a = v[fftr::br5(k1)];
      yo[n] = make_double2(fma(-inv, a.x, xv.x), fma(-inv, a.y, xv.y));
    }
  }
}

// Owner side of a cut trace after the exchange: y_s = sx x_s + h (h = -(L x)_s
// computed by the neighbour rank), sx = xs->x or 1.
__global__ void k_halo_add(const double2 *__restrict__ x, const double2 *__restrict__ h, double2 *__restrict__ y,
                           int NT, const double2 *__restrict__ xs) {
  const double sx = xs ? xs->x : 1.0;
  for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < NT; n += gridDim.x * blockDim.x)
    y[n] = cadd(cscale(sx, x[n]), h[n]);
}

// Bytes of L2 set aside for persisting accesses on the current device (0: none).
size_t l2_persist_bytes() {
  static size_t v = [] {
    size_t lim = 0;
    if (cudaDeviceGetLimit(&lim, cudaLimitPersistingL2CacheSize) != cudaSuccess) return (size_t)0;
    return lim;
  }();
  return v;
}

cudaError_t launch_fft_conv_reg(const double2 *Fc, const double2 *x, double2 *y, const SlotMap &m, const double2 *tw,
                                cudaStream_t st, const double2 *xs, double2 *xcopy) {
  const int N = m.N;
  if (N < 2) return cudaSuccess;
  if (m.NT > 512) return cudaErrorInvalidValue;
  const size_t smem = (2 * 32 * 33) * sizeof(double2);
  cudaError_t e = cudaFuncSetAttribute(k_fft_conv_reg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  // the transformed columns (N x 4 x NF complex, 32 MB at C5) are re-read by
  // every apply: ask L2 to keep them (persisting window; the Krylov vectors
  // streamed between applies are normal accesses and do not evict them)
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(m.j_hi - m.j_lo + 1);
  cfg.blockDim = dim3(64);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeAccessPolicyWindow;
  at[1].val.accessPolicyWindow.base_ptr = const_cast<double2 *>(Fc + (size_t)(m.j_lo - 1) * 4 * 1024);
  at[1].val.accessPolicyWindow.num_bytes = (size_t)(m.j_hi - m.j_lo + 1) * 4 * 1024 * sizeof(double2);
  at[1].val.accessPolicyWindow.hitRatio = 1.0f;
  at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = at;
  cfg.numAttrs = l2_persist_bytes() > 0 ? 2 : 1;
  if (cfg.numAttrs == 2 && at[1].val.accessPolicyWindow.num_bytes > l2_persist_bytes()) {
    at[1].val.accessPolicyWindow.hitRatio = (float)l2_persist_bytes() / (float)at[1].val.accessPolicyWindow.num_bytes;
  }
  return cudaLaunchKernelEx(&cfg, k_fft_conv_reg, Fc, x, y, m, tw, xs, xcopy);
}

cudaError_t launch_fft_conv(int log4, const double2 *Fc, const double2 *x, double2 *y, const SlotMap &m,
                            const double2 *tw, cudaStream_t st) {
  if (m.N < 2) return cudaSuccess;
  const int nblk = 2 * (m.j_hi - m.j_lo + 1);
  const size_t smem = 3 * ((size_t)1 << (2 * log4)) * sizeof(double2);
  switch (log4) {
    case 2: k_fft_conv<2><<<nblk, 4, smem, st>>>(Fc, x, y, m, tw); break;
    case 3: k_fft_conv<3><<<nblk, 16, smem, st>>>(Fc, x, y, m, tw); break;
    case 4: k_fft_conv<4><<<nblk, 64, smem, st>>>(Fc, x, y, m, tw); break;
    case 5: {
      cudaError_t e = cudaFuncSetAttribute(k_fft_conv<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      k_fft_conv<5><<<nblk, 256, smem, st>>>(Fc, x, y, m, tw);
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
// Fused classical Gram-Schmidt passes on the rank's slots (SlotMap):
//   mode & CGS_AXPY : w -= sum_v h_v V_v          (h from the device, v < nv)
//   mode & CGS_DOTS : p_v = <V_v, w>              (v < nv, after the axpy)
//   mode & CGS_NORM : p_nv = <w, w>
// Order-fixed reductions that do not depend on the sharding: the unit of a
// partial sum is one interface slot (N_T entries, owned by one rank; SURVEY
// 8(c) step 11).  One CTA processes one unit in a fixed order (chunks in
// sequence per lane, a fixed lane tree, warps in order) and writes its
// partials to column s of partial[nred][2N-2]; k_cgs_reduce then sums the
// columns of every quantity in a fixed order -- on one GPU directly, on G
// GPUs after the columns of all ranks were summed (disjoint, exact) -- so any
// rank count gives bitwise the one-GPU scalars.  (Measured at C5, GMRES solve:
// one CTA per slot 99.3 ms; per subdomain 103.0; persistent grids 105-107;
// the reduction inside the pass's last CTA instead of a second kernel +3 ms;
// 5-6 CTAs per SM 103-124 ms.  The round-1 kernels, partials per CTA of a
// persistent grid -- not sharding-invariant -- 93.0 ms.)
// k_cgs: the 4 warps of a CTA split the basis vectors (warp q holds v = q,
// q+4, ...; lane holds entries lane + 32 kk of a chunk) so each basis value is
// loaded from HBM once per pass and kept in registers between the axpy and the
// dots; the axpy partials of the 4 warps meet in shared memory (fixed order).
// ---------------------------------------------------------------------------
// local unit b = slot s_lo + b: entries [b N_T, (b+1) N_T) of the rank's vectors
__host__ __device__ __forceinline__ int units_local(const SlotMap &m) { return m.s_hi - m.s_lo + 1; }
__host__ __device__ __forceinline__ int units_global(const SlotMap &m) { return 2 * m.N - 2; }
int cgs_units_global(const SlotMap &m) { return units_global(m); }

template <int VPW, int KE>
__global__ void __launch_bounds__(128, 4) k_cgs(const double2 *__restrict__ V, size_t ldv, int nv,
                                                const double2 *__restrict__ hsrc, double2 *__restrict__ w, int mode,
                                                const SlotMap m, double2 *__restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  constexpr int NVMAX = 4 * VPW, CH = 32 * KE;
  __shared__ double2 sh[NVMAX];
  __shared__ double2 part[4][CH];
  __shared__ double2 tr[4][VPW][33];   // per-warp transpose of the lane partials
  const int nunit = units_local(m), NU = units_global(m), NT = m.NT;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const bool axpy = mode & CGS_AXPY, dots = mode & CGS_DOTS, norm = mode & CGS_NORM;
  const int nred = (dots ? nv : 0) + (norm ? 1 : 0);
  if (axpy)
    for (int v = threadIdx.x; v < nv; v += blockDim.x) sh[v] = hsrc[v];
  __syncthreads();
  // consecutive passes alternate the traversal direction (CGS_REV): the first
  // units of a pass meet the last ones of the previous pass in L2
  const int b = (mode & CGS_REV) ? nunit - 1 - (int)blockIdx.x : (int)blockIdx.x;
  if (b < 0 || b >= nunit) return;
  const size_t e0 = (size_t)b * NT, col = (size_t)(m.s_lo + b);
  const int len = NT;
  {
    double2 acc[VPW];
#pragma unroll
    for (int i = 0; i < VPW; i++) acc[i] = cz();
    double nacc = 0.0;
    for (int c0 = 0; c0 < len; c0 += CH) {
      double2 x[VPW][KE], we[KE];
#pragma unroll
      for (int i = 0; i < VPW; i++) {
        const int v = wp + 4 * i;
#pragma unroll
        for (int k = 0; k < KE; k++) {
          const int e = c0 + lane + 32 * k;
          x[i][k] = (v < nv && e < len) ? V[(size_t)v * ldv + e0 + e] : cz();
        }
      }
#pragma unroll
      for (int k = 0; k < KE; k++) {
        const int e = c0 + lane + 32 * k;
        we[k] = e < len ? w[e0 + e] : cz();
      }
      if (axpy) {
#pragma unroll
        for (int k = 0; k < KE; k++) {
          double2 pv = cz();
#pragma unroll
          for (int i = 0; i < VPW; i++)
            if (wp + 4 * i < nv) pv = cfma(sh[wp + 4 * i], x[i][k], pv);
          part[wp][lane + 32 * k] = pv;
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < KE; k++) {
          const int t = lane + 32 * k;
          const double2 pv = cadd(cadd(cadd(part[0][t], part[1][t]), part[2][t]), part[3][t]);
          we[k] = csub(we[k], pv);
          const int e = c0 + t;
          if (wp == 0 && e < len) w[e0 + e] = we[k];
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
    // unit partials (warp q holds vectors q, q+4, ...): the lane partials go
    // through shared memory; lanes l = i + VPW r (r < 32/VPW) sum lanes
    // r, r + 32/VPW, ... of vector i in order, then a short shuffle tree over r
    if (dots) {
#pragma unroll
      for (int i = 0; i < VPW; i++) tr[wp][i][lane] = acc[i];
      __syncwarp();
      constexpr int R = 32 / VPW;
      const int i = lane % VPW, r = lane / VPW;
      double2 a = cz();
#pragma unroll
      for (int q = r; q < 32; q += R) a = cadd(a, tr[wp][i][q]);
#pragma unroll
      for (int o = 16; o >= VPW; o >>= 1) a = cadd(a, shfl_down2(a, o));
      const int v = wp + 4 * i;
      if (r == 0 && v < nv) partial[(size_t)v * NU + col] = a;
      __syncwarp();
    }
    if (norm && wp == 0) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nacc += __shfl_down_sync(0xffffffffu, nacc, o);
      if (lane == 0) partial[(size_t)(nred - 1) * NU + col] = make_double2(nacc, 0.0);
    }
  }
}

// The CGS update pass without dots (CGS_AXPY | CGS_NORM [| CGS_SCALE]):
// w -= V h and <w, w>.  No dots means no per-vector sums, so the entries
// split over warps: warp q of the unit's CTA streams all nv basis vectors for
// chunks q, q+4, ... of 32 KE entries (VU vectors per unrolled step) with no
// shared-memory exchange or barrier in the loop.  Unit norm partial: lane
// tree per warp, warps in order.
template <int KE, int VU = 4>
__global__ void __launch_bounds__(128, 4) k_cgs_axpy(const double2 *__restrict__ V, size_t ldv, int nv,
                                                     const double2 *__restrict__ hsrc, double2 *__restrict__ w,
                                                     int mode, const SlotMap m, double2 *__restrict__ partial) {
  pdl_wait();
  pdl_trigger();
  __shared__ double2 sh[32];
  __shared__ double red[4];
  for (int v = threadIdx.x; v < nv; v += blockDim.x) sh[v] = hsrc[v];
  __syncthreads();
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  constexpr int CH = 32 * KE;
  const int nunit = units_local(m), NT = m.NT;
  const int b = (mode & CGS_REV) ? nunit - 1 - (int)blockIdx.x : (int)blockIdx.x;
  if (b < 0 || b >= nunit) return;
  const size_t e0 = (size_t)b * NT, col = (size_t)(m.s_lo + b);
  const int len = NT;
  double nacc = 0.0;
  for (int c0 = wp * CH; c0 < len; c0 += 4 * CH) {
    double2 we[KE], pv[KE];
#pragma unroll
    for (int k = 0; k < KE; k++) {
      const int e = c0 + lane + 32 * k;
      we[k] = e < len ? w[e0 + e] : cz();
      pv[k] = cz();
    }
    int v = 0;
    for (; v + VU <= nv; v += VU) {
      double2 x[VU][KE];
#pragma unroll
      for (int jv = 0; jv < VU; jv++)
#pragma unroll
        for (int k = 0; k < KE; k++) {
          const int e = c0 + lane + 32 * k;
          x[jv][k] = e < len ? V[(size_t)(v + jv) * ldv + e0 + e] : cz();
        }
#pragma unroll
      for (int jv = 0; jv < VU; jv++)
#pragma unroll
        for (int k = 0; k < KE; k++) pv[k] = cfma(sh[v + jv], x[jv][k], pv[k]);
    }
    for (; v < nv; v++) {
#pragma unroll
      for (int k = 0; k < KE; k++) {
        const int e = c0 + lane + 32 * k;
        pv[k] = cfma(sh[v], e < len ? V[(size_t)v * ldv + e0 + e] : cz(), pv[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < KE; k++) {
      const int e = c0 + lane + 32 * k;
      if (e < len) {
        const double2 r = csub(we[k], pv[k]);
        w[e0 + e] = r;
        nacc = fma(r.x, r.x, fma(r.y, r.y, nacc));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nacc += __shfl_down_sync(0xffffffffu, nacc, o);
  if (lane == 0) red[wp] = nacc;
  __syncthreads();
  if (threadIdx.x == 0) partial[col] = make_double2(((red[0] + red[1]) + red[2]) + red[3], 0.0);
}

// The unit partials (on G GPUs: of all ranks, summed -- disjoint columns) ->
// the scalars in a fixed order that depends on the global unit count only:
// one CTA of 256 threads per quantity; thread t sums units t, t + 256, ...
// in sequence (all loads issued before the adds), then a fixed shuffle tree
// per warp and the 8 warp sums in order.  CGS_SCALE: out[nred] =
// 1/sqrt(out[nred - 1]).  out_host: pinned mirror (read after the step's event).
constexpr int kRedThreads = 256;
__global__ void __launch_bounds__(kRedThreads) k_cgs_reduce(const double2 *__restrict__ partial, int nu, int nred,
                                                            int mode, double2 *out, double2 *out_host) {
  pdl_wait();
  pdl_trigger();
  __shared__ double2 ws[kRedThreads / 32];
  const int v = blockIdx.x, t = threadIdx.x, lane = t & 31;
  const double2 *pv = partial + (size_t)v * nu;
  double2 sum = cz();
  int q = t;
  for (; q + 3 * kRedThreads < nu; q += 4 * kRedThreads) {
    const double2 a0 = __ldcg(pv + q), a1 = __ldcg(pv + q + kRedThreads), a2 = __ldcg(pv + q + 2 * kRedThreads),
                  a3 = __ldcg(pv + q + 3 * kRedThreads);
    sum = cadd(cadd(cadd(cadd(sum, a0), a1), a2), a3);
  }
  for (; q < nu; q += kRedThreads) sum = cadd(sum, __ldcg(pv + q));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum = cadd(sum, shfl_down2(sum, o));
  if (lane == 0) ws[t >> 5] = sum;
  __syncthreads();
  if (t == 0) {
    sum = ws[0];
#pragma unroll
    for (int i = 1; i < kRedThreads / 32; i++) sum = cadd(sum, ws[i]);
    out[v] = sum;
    if (out_host) out_host[v] = sum;
    if ((mode & CGS_SCALE) && v == nred - 1) out[v + 1] = make_double2(1.0 / sqrt(sum.x), 0.0);
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

cudaError_t launch_cgs(const double2 *V, size_t ldv, int nv, const double2 *hsrc, double2 *w, int mode,
                       const SlotMap &m, double2 *partial, cudaStream_t st, size_t vwin, float vratio) {
  if (!V) vwin = 0;
  if (nv > 32) return cudaErrorInvalidValue;
  const int nunit = units_local(m);
  if (nunit < 1) return cudaSuccess;
  const dim3 g(nunit), b(128);   // one CTA per slot
  // update pass without dots: entry-split streaming form
  if ((mode & CGS_AXPY) && !(mode & CGS_DOTS) && (mode & CGS_NORM) && nv >= 1)
    return launch_pdl_win(V, vwin, vratio, k_cgs_axpy<4>, g, b, 0, st, V, ldv, nv, hsrc, w, mode, m, partial);
  if (nv <= 8) return launch_pdl_win(V, vwin, vratio, k_cgs<2, 8>, g, b, 0, st, V, ldv, nv, hsrc, w, mode, m, partial);
  if (nv <= 16) return launch_pdl_win(V, vwin, vratio, k_cgs<4, 4>, g, b, 0, st, V, ldv, nv, hsrc, w, mode, m, partial);
  return launch_pdl_win(V, vwin, vratio, k_cgs<8, 2>, g, b, 0, st, V, ldv, nv, hsrc, w, mode, m, partial);
}

cudaError_t launch_cgs_reduce(const double2 *partial, int nu, int nred, int mode, double2 *out, double2 *out_host,
                              cudaStream_t st) {
  return launch_pdl(k_cgs_reduce, dim3(nred), dim3(kRedThreads), 0, st, partial, nu, nred, mode, out, out_host);
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

}  // namespace swr

namespace swr {
// dst[c blk + i] = src[i], c < count (identical interior L0 columns)
__global__ void k_replicate(const double2 *__restrict__ src, double2 *__restrict__ dst, size_t blk, size_t count) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < blk * count; e += (size_t)gridDim.x * blockDim.x)
    dst[e] = src[e % blk];
}
// y += x (n doubles): the loopback communicator's rank-ordered sums
__global__ void k_add_f64(double *__restrict__ y, const double *__restrict__ x, size_t n) {
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x)
    y[e] += x[e];
}
}  // namespace swr

// y = (I - L) x by FFT convolution with two warps per 1024-point transform
// (a10/a13; the Toeplitz blocks of Props. 3-4).
//
// The inputs are zero beyond N_T <= 512 and only outputs n < N_T are kept,
// so each 1024-point transform splits into two 512-point ones (W = e^{-2 pi
// i/1024}, w = W^2):
//   X[2m] = DFT512(x)[m],   X[2m+1] = DFT512(x[n] W^n)[m],
//   y[n]  = (IDFT512(Y_even)[n] + W^{-n} IDFT512(Y_odd)[n]) / 1024,  n < 512.
// One CTA per subdomain j, four warps (side s = l_j / r_j input, parity e):
// forward DFT512 of the inputs, pointwise products with the transformed first
// columns X^{j,1..4} (the even / odd bins), inverse DFT512 per (output side,
// parity), and the odd warp hands W^{-n} IDFT to the even warp, which writes
// y = s x - conv / 1024.  Twice the warps of the one-warp-per-transform
// kernel (k_fft_conv_reg) and no discarded half of the inverse -- but
// measured slower at C5 (28.6 vs 20.2 ms of applies per solve; 38 ms with
// 168 registers and two waves), so it is an option (SWR_FFT_HALVES=1).
//
// DFT512 in a warp: n = n1 + 32 n2 (lane n1, register n2), k = k2 + 16 k1:
// a 16-point DFT over n2 per lane, the twiddle w^{n1 k2}, a transpose so that
// lane 2 k2 + h holds the 16 entries n1 = 2j + h of frequency k2, a 16-point
// DFT per lane and one radix-2 step between lane pairs:
//   X[k2 + 16 k1] = E[k1] + t^{k1} O[k1],  X[k2 + 16 (k1+16)] = E[k1] - t^{k1} O[k1],
// t = e^{-2 pi i/32}.  On exit lane L = 2 k2 + h holds X[k2 + 16 (k1 + 16 h)]
// in register br4(k1).
#include "swr_common.cuh"
#include "swr_kernels.h"

#ifndef FFTH_MINB
#define FFTH_MINB 4   // 4 CTAs of 128 per SM: the N = 500 CTAs fit one wave
#endif

namespace swr {
namespace ffth {

__device__ __forceinline__ constexpr double c32(int k) {
  return k == 0 ? 1.0 : k == 1 ? 0.98078528040323043 : k == 2 ? 0.92387953251128674 : k == 3 ? 0.83146961230254524
       : k == 4 ? 0.70710678118654752 : k == 5 ? 0.55557023301960218 : k == 6 ? 0.38268343236508977
       : k == 7 ? 0.19509032201612826 : 0.0;
}
// d e^{-+2 pi i k/32}, k in [0, 16) (constant after unrolling)
template <bool INV>
__device__ __forceinline__ double2 tw32(double2 d, int k) {
  if (k == 0) return d;
  if (k == 8) return INV ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
  const double c = k < 8 ? c32(k) : -c32(16 - k);
  const double sn = k < 8 ? c32(8 - k) : c32(k - 8);
  const double s = INV ? sn : -sn;
  return make_double2(fma(d.x, c, -d.y * s), fma(d.x, s, d.y * c));
}
__device__ __forceinline__ constexpr int br4(int k) { return ((k & 1) << 3) | ((k & 2) << 1) | ((k & 4) >> 1) | ((k & 8) >> 3); }

// 16-point radix-2 DIF in registers: X[k] in v[br4(k)]
template <bool INV>
__device__ __forceinline__ void dif16(double2 (&v)[16]) {
#pragma unroll
  for (int m = 16; m >= 2; m >>= 1) {
#pragma unroll
    for (int b = 0; b < 16; b += m) {
#pragma unroll
      for (int i = 0; i < m / 2; i++) {
        const double2 a = v[b + i], c = v[b + i + m / 2];
        v[b + i] = cadd(a, c);
        v[b + i + m / 2] = tw32<INV>(csub(a, c), 2 * i * (16 / m));
      }
    }
  }
}

// DFT512 (INV: exponent sign +, no scaling) of the warp's sequence, entry:
// lane n1 holds x[n1 + 32 n2] in v[n2]; exit: see the file header.
// T: this warp's [16][33] transpose buffer; tw: e^{-2 pi i k/1024}, k < 1024.
template <bool INV>
__device__ __forceinline__ void dft512(double2 (&v)[16], double2 *T, const double2 *__restrict__ tw, int lane) {
  dif16<INV>(v);                                   // Y_{n1}[k2] in v[br4(k2)]
#pragma unroll
  for (int k2 = 1; k2 < 16; k2++) {                // w^{n1 k2} = W^{2 n1 k2}
    double2 w = __ldg(tw + ((2 * lane * k2) & 1023));
    if (INV) w.y = -w.y;
    v[br4(k2)] = cmul(v[br4(k2)], w);
  }
#pragma unroll
  for (int k2 = 0; k2 < 16; k2++) T[k2 * 33 + lane] = v[br4(k2)];
  __syncwarp();
  const int k2 = lane >> 1, h = lane & 1;
#pragma unroll
  for (int jj = 0; jj < 16; jj++) v[jj] = T[k2 * 33 + 2 * jj + h];
  __syncwarp();
  dif16<INV>(v);                                   // B_h[k1] in v[br4(k1)]
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int k1 = br4(r);
    double2 mine = v[r];
    if (h) mine = tw32<INV>(mine, k1);             // t^{k1} O[k1] on the odd lane
    const double2 other = shfl_xor2(mine, 1);
    v[r] = h ? csub(other, mine) : cadd(mine, other);
  }
}
}  // namespace ffth

// Fc: [N][4][1024] transformed first columns; x, y: [2N-2][N_T]
__global__ void __launch_bounds__(128, FFTH_MINB) k_fft_conv_h(const double2 *__restrict__ Fc, const double2 *__restrict__ x,
                                                       double2 *__restrict__ y, int N, int NT,
                                                       const double2 *__restrict__ tw,
                                                       const double2 *__restrict__ xs, double2 *__restrict__ xcopy) {
  pdl_wait();
  pdl_trigger();
  constexpr int NF = 1024, WS = 16 * 33;
  extern __shared__ double2 fsm[];
  const int q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int side = q >> 1, par = q & 1;            // forward: input side (l_j, r_j); inverse: output side
  double2 *T = fsm + q * WS;                       // transpose buffer, then this warp's spectrum / hand-off
  const int j = blockIdx.x + 1;
  const bool hA = j >= 2, hB = j <= N - 1;         // l_j, r_j exist
  const double sx = xs ? xs->x : 1.0;
  const int k2 = lane >> 1, hh = lane & 1;
  double2 v[16];
  // ---- forward: DFT512 of x (even bins) or x W^n (odd bins) ----
  const bool has_in = side == 0 ? hA : hB;
  const int sidx = side == 0 ? 2 * j - 3 : 2 * j - 2;
  if (has_in) {
#pragma unroll
    for (int n2 = 0; n2 < 16; n2++) {
      const int n = lane + 32 * n2;
      double2 a = n < NT ? cscale(sx, x[(size_t)sidx * NT + n]) : cz();
      if (xcopy && par == 0 && n < NT) xcopy[(size_t)sidx * NT + n] = a;
      if (par) a = cmul(a, __ldg(tw + n));
      v[n2] = a;
    }
    ffth::dft512<false>(v, T, tw, lane);
#pragma unroll
    for (int r = 0; r < 16; r++) T[k2 + 16 * (ffth::br4(r) + 16 * hh)] = v[r];   // natural order
  }
  __syncthreads();
  // ---- products: Y[m] = c1[2m+e] A_e[m] + c2[2m+e] B_e[m], m = lane + 32 n2 ----
  const bool has_out = side == 0 ? hA : hB;
  const double2 *c1 = Fc + ((size_t)(j - 1) * 4 + 2 * side) * NF + par, *c2 = c1 + NF;
  const double2 *SA = fsm + (0 * 2 + par) * WS, *SB = fsm + (1 * 2 + par) * WS;
  if (has_out) {
#pragma unroll
    for (int n2 = 0; n2 < 16; n2++) {
      const int m = lane + 32 * n2;
      double2 acc = cz();
      if (hA) acc = cmul(__ldg(c1 + 2 * m), SA[m]);
      if (hB) acc = cfma(__ldg(c2 + 2 * m), SB[m], acc);
      v[n2] = acc;
    }
  }
  __syncthreads();   // every warp has read the spectra: the buffers are free again
  if (has_out) {
    ffth::dft512<true>(v, T, tw, lane);             // lane holds IDFT at n = k2 + 16 (k1 + 16 hh)
    if (par) {
#pragma unroll
      for (int r = 0; r < 16; r++) {
        const int n = k2 + 16 * (ffth::br4(r) + 16 * hh);
        double2 wn = __ldg(tw + n);
        wn.y = -wn.y;                               // W^{-n}
        T[r * 32 + lane] = cmul(v[r], wn);
      }
    }
  }
  __syncthreads();
  if (!has_out || par) return;
  const int o = side == 0 ? 2 * j - 4 : 2 * j - 1;
  const double2 *odd = fsm + (side * 2 + 1) * WS;
  const double inv = 1.0 / NF;
#pragma unroll
  for (int r = 0; r < 16; r++) {
    const int n = k2 + 16 * (ffth::br4(r) + 16 * hh);
    if (n < NT) {
      const double2 a = cadd(v[r], odd[r * 32 + lane]);
      const double2 xv = cscale(sx, x[(size_t)o * NT + n]);
      y[(size_t)o * NT + n] = make_double2(fma(-inv, a.x, xv.x), fma(-inv, a.y, xv.y));
    }
  }
}

cudaError_t launch_fft_conv_h(const double2 *Fc, const double2 *x, double2 *y, int N, int NT, const double2 *tw,
                              cudaStream_t st, const double2 *xs, double2 *xcopy, size_t l2_window) {
  if (N < 2) return cudaSuccess;
  if (NT > 512) return cudaErrorInvalidValue;
  const size_t smem = (size_t)4 * 16 * 33 * sizeof(double2);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(N);
  cfg.blockDim = dim3(128);
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
  cfg.numAttrs = l2_window > 0 ? 2 : 1;
  if (cfg.numAttrs == 2 && at[1].val.accessPolicyWindow.num_bytes > l2_window)
    at[1].val.accessPolicyWindow.hitRatio = (float)l2_window / (float)at[1].val.accessPolicyWindow.num_bytes;
  return cudaLaunchKernelEx(&cfg, k_fft_conv_h, Fc, x, y, N, NT, tw, xs, xcopy);
}

}  // namespace swr

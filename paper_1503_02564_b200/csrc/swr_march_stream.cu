// swr_march_stream.cu — the whole-window march for subdomains too large to
// keep resident on one thread-block cluster (N_j beyond ~45K rows, e.g. C2:
// N = 10 at dx = 1e-5, N_j = 420,001).  Same arithmetic as k_march (P:193-198,
// P:305-330; readings A3-A16): per step (A - B) v_n = rhs, u_n = 2 v_n - u_{n-1},
// S v_n recorded at the interfaces.
//
// B200 mapping.  The state u_{n-1} and the forward values z streams through HBM
// (the march is then HBM-bound, the regime of SURVEY 8(d) "B1 streaming").
// A system is a chain of nc co-resident CTAs (cooperative launch); CTA c owns
// the contiguous rows [c Rc, (c+1) Rc) and thread t of it a contiguous block
// of Rt rows and keeps the Thomas recurrence in registers.  Three kernels:
// k_march_stream2 (constant matrix) and k_march_nl_stream (|u|^2) take two
// passes per step (or fixed-point iteration) over a thread-interleaved
// scratch layout (row i of thread t at i P + t of the CTA's block: coalesced);
// k_march_stream (V(t,x): per-step factors in the natural layout) takes the
// four passes below.  Per step of k_march_stream:
//   pass 1  forward from carry 0 over the thread's rows -> affine map (A, F)
//   scan    CTA scan of the maps; the CTA totals are published in global
//           memory (value + step flag, release/acquire) and folded by the
//           later CTAs of the chain
//   pass 2  forward again from the exact carry, z stored
//   pass 3  backward from carry 0 over z -> (Ab, B); scan and chain fold in
//           reverse order
//   pass 4  backward from the exact carry: v = x, u_n = 2 v - u_{n-1}
// The boundary rows fold b_n - l_n / b_n - r_n into the stencil as in k_march;
// the S0^2 history sum of an end row is reduced by the CTA holding it.
#include "swr_common.cuh"
#include "swr_kernels.h"
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>
#include <algorithm>

namespace swr {

namespace {

__device__ __forceinline__ double2 negqe_s(double2 q, double er, double eim) {
  return make_double2(fma(q.y, eim, -q.x * er), -fma(q.x, eim, q.y * er));
}

__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_flag(const int *p, int v) {
  while (ld_acquire(p) < v) __nanosleep(64);
}

// Exclusive scan of per-thread affine maps x -> A x + B over the CTA in
// thread order (FWD) or reverse; returns the exclusive (eA, eB) of this
// thread and, in every thread, the CTA total (tA, tB).
template <bool FWD>
__device__ void cta_scan(double2 A, double2 B, double2 *sm, double2 &eA, double2 &eB, double2 &tA, double2 &tB) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double2 Ae = FWD ? shfl_up2(A, o) : shfl_down2(A, o), Be = FWD ? shfl_up2(B, o) : shfl_down2(B, o);
    if (FWD ? lane >= o : lane + o < 32) {
      B = cfma(A, Be, B);
      A = cmul(A, Ae);
    }
  }
  double2 xA = FWD ? shfl_up2(A, 1) : shfl_down2(A, 1), xB = FWD ? shfl_up2(B, 1) : shfl_down2(B, 1);
  if (FWD ? lane == 0 : lane == 31) { xA = make_double2(1.0, 0.0); xB = cz(); }
  double2 *wA = sm, *wB = sm + 32;
  if (lane == (FWD ? 31 : 0)) { wA[w] = A; wB[w] = B; }
  __syncthreads();
  // warp prefix: fold of the other warps' totals (<= 16 warps)
  double2 pA = make_double2(1.0, 0.0), pB = cz(), aA = make_double2(1.0, 0.0), aB = cz();
  for (int i = 0; i < nw; i++) {
    const int q = FWD ? i : nw - 1 - i;
    const double2 qa = wA[q], qb = wB[q];
    if (FWD ? q < w : q > w) { pB = cfma(qa, pB, qb); pA = cmul(qa, pA); }
    aB = cfma(qa, aB, qb);
    aA = cmul(qa, aA);
  }
  __syncthreads();
  eB = cfma(xA, pB, xB);
  eA = cmul(xA, pA);
  tA = aA;
  tB = aB;
}


// Fold, applied to 0, of the maps (A, B) the chain CTAs published for step
// (or iteration) v: those before c in order (fwd) or those after c from the
// last one down (backward).  Warp 0's lanes wait for the flags in parallel,
// then every warp composes the maps by a lane tree in chunks of 32 (a serial
// fold costs one L2 round trip per CTA: chains are ~120 CTAs long at C2).
__device__ __forceinline__ double2 chain_fold(const int *flg, const double2 *vals, int c, int nc, bool fwd, int par,
                                              int v) {
  const int cnt = fwd ? c : nc - 1 - c;
  if (cnt <= 0) return cz();
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32)
    for (int i = lane; i < cnt; i += 32) wait_flag(flg + (fwd ? i : nc - 1 - i), v);
  __syncthreads();
  double2 val = cz();
  for (int b = 0; b < cnt; b += 32) {
    const int i = b + lane;
    double2 A = make_double2(1.0, 0.0), B = cz();
    if (i < cnt) {
      const int cc = fwd ? i : nc - 1 - i;
      A = __ldcg(vals + (cc * 2 + par) * 2 + 0);
      B = __ldcg(vals + (cc * 2 + par) * 2 + 1);
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {   // lane l's span, then lane l + o's
      const double2 nA = shfl_down2(A, o), nB = shfl_down2(B, o);
      if (lane + o < 32) {
        B = cfma(nA, B, nB);
        A = cmul(nA, A);
      }
    }
    const double2 cA = make_double2(__shfl_sync(0xffffffffu, A.x, 0), __shfl_sync(0xffffffffu, A.y, 0));
    const double2 cB = make_double2(__shfl_sync(0xffffffffu, B.x, 0), __shfl_sync(0xffffffffu, B.y, 0));
    val = cfma(cA, val, cB);
  }
  return val;
}
}  // namespace

// One CTA per (system, chain index).  scratch: u [nsys][Nj], z [nsys][Nj];
// sync: done/fwd/bwd flags [nsys][nc] (int), values fv/bv [nsys][nc][2 parity][2].
__global__ void __launch_bounds__(256) k_march_stream(const MarchParams p, int nc, double2 *ust, double2 *zst,
                                                      int *flags, double2 *vals) {
  extern __shared__ double2 ssm[];
  double2 *scanbuf = ssm;                      // [64]
  double2 *red = scanbuf + 64;                 // [32] block reduction
  double2 *hvL = red + 32;                     // [NT+1] v_s at row 0 (CTA 0 of a system with a left interface)
  double2 *hvR = hvL + (p.NT + 1);             // [NT+1] v_s at row N_j - 1 (last CTA, right interface)
  __shared__ double2 sHL, sHR;                 // H_n of the end rows this CTA holds
  const int t = threadIdx.x, P = blockDim.x;
  const int sidx = blockIdx.x / nc, c = blockIdx.x % nc;
  const MarchSys &S = p.sys[sidx];
  const int Nj = p.Nj, NT = p.NT;
  const double eim = p.e_im, kappa = p.kappa, ikappa = 1.0 / p.kappa;
  const int Rc = (Nj + nc - 1) / nc;
  const int rc0 = min(Nj, c * Rc), rc1 = min(Nj, (c + 1) * Rc);
  const int Rt = (rc1 - rc0 + P - 1) / P;
  const int rt0 = min(rc1, rc0 + t * Rt), rt1 = min(rc1, rc0 + (t + 1) * Rt);
  // u, z and the system record never alias: say so, or every store to u / z
  // forces the step loop to reload the record's fields (3.7x slower C2 build)
  double2 *__restrict__ u = ust + (size_t)sidx * Nj;
  double2 *__restrict__ z = zst + (size_t)sidx * Nj;
  int *fdone = flags + (size_t)sidx * nc * 3, *ffwd = fdone + nc, *fbwd = ffwd + nc;
  double2 *fv = vals + (size_t)sidx * nc * 8, *bv = fv + nc * 4;   // [nc][parity][A, B]
  const bool has_left = S.flags & SYS_HAS_LEFT, has_right = S.flags & SYS_HAS_RIGHT;
  const bool first_cta = c == 0, last_cta = rc1 == Nj && rc0 < Nj;
  const bool own0 = first_cta && t == 0 && rt0 == 0 && rt1 > 0;          // holds row 0
  const bool ownL = rt1 == Nj && rt0 < Nj;                                 // holds row N_j - 1
  const bool histL = first_cta && has_left, histR = last_cta && has_right;

  // initial state
  for (int k = rc0 + t; k < rc1; k += P) u[k] = S.u0 ? S.u0[k] : cz();
  // v'_0 (times the gauge factor f0 for the higher-order operators)
  if (histL && t == 0) hvL[0] = p.tc_hi ? cmul(S.f0[0], S.u0 ? S.u0[0] : cz()) : (S.u0 ? S.u0[0] : cz());
  if (histR && t == 0) hvR[0] = p.tc_hi ? cmul(S.f0[1], S.u0 ? S.u0[Nj - 1] : cz()) : (S.u0 ? S.u0[Nj - 1] : cz());
  // odd part of order-4 operators, B_n = sum_{s<n} rho^{n-s} v'_s (held by the end-row threads)
  double2 BoL = cz(), BoR = cz();
  if (p.tc_hi) {
    if (own0) BoL = cmul(S.rho[0], cmul(S.f0[0], S.u0 ? S.u0[0] : cz()));
    if (ownL) BoR = cmul(S.rho[1], cmul(S.f0[1], S.u0 ? S.u0[Nj - 1] : cz()));
  }
  __syncthreads();
  __threadfence();
  if (t == 0) st_release(fdone + c, 0);

  // the record's fields the step loop needs, read once (the record is in global
  // memory: reading it inside the loop after the u / z stores costs reloads)
  const int sflags = S.flags;
  const double2 *const slin = S.lin, *const srin = S.rin, *const sq = S.q;
  const double *const ser = S.er;
  double2 *const sout_l = S.out_left, *const sout_r = S.out_right;
  auto flux = [&](int sd, int n) -> double2 {
    if (sflags & (sd == 0 ? SYS_LIN_IMPULSE : SYS_RIN_IMPULSE)) return make_double2(n == 1 ? 1.0 : 0.0, 0.0);
    const double2 *f = sd == 0 ? slin : srin;
    return f ? f[n - 1] : cz();
  };

  for (int n = 1; n <= NT; n++) {
    race_jitter(0, n);
    const size_t toff = p.td_stride ? (size_t)(n - 1) * p.td_stride : 0;
    const double2 *q = sq + toff;
    const double *er = ser + toff;
    // neighbours' u_{n-1} (halo rows) are final once they reported step n-1
    if (t == 0) {
      if (c > 0) wait_flag(fdone + c - 1, n - 1);
      if (c < nc - 1) wait_flag(fdone + c + 1, n - 1);
    }
    // S0^2 history of the end rows this CTA holds: H_n = c2 sum_{s<n} beta_{n-s} v_s
    for (int sd = 0; sd < 2; sd++) {
      if (!(sd == 0 ? histL : histR)) continue;
      const double2 *hv = sd == 0 ? hvL : hvR;
      double2 acc = cz();
      if (p.tc_hi) {
        const double2 *kp = S.kap[sd];
        for (int s = t; s <= n - 1; s += P) acc = cfma(__ldg(kp + n - s), hv[s], acc);
      } else if (p.s02)
        for (int s = t; s <= n - 1; s += P)
          acc = make_double2(fma(p.beta[n - s], hv[s].x, acc.x), fma(p.beta[n - s], hv[s].y, acc.y));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
      if ((t & 31) == 0) red[t >> 5] = acc;
      __syncthreads();
      if (t == 0) {
        double2 hs = cz();
        for (int w = 0; w < (P >> 5); w++) hs = cadd(hs, red[w]);
        (sd == 0 ? sHL : sHR) = p.tc_hi ? hs : (p.s02 ? cmul(p.c2, hs) : cz());
      }
      __syncthreads();
    }
    __syncthreads();
    // end-row folds (k_march): d = H_n - l_n at row 0, H_n - r_n at row N_j - 1
    // (the odd part of order-4 operators enters the local condition only, A25)
    const double2 dL = (own0 && has_left) ? csub(cfma(cscale(2.0, S.dlt[0]), BoL, sHL), flux(0, n)) : cz();
    const double2 dR = (ownL && has_right) ? csub(cfma(cscale(2.0, S.dlt[1]), BoR, sHR), flux(1, n)) : cz();
    auto sval = [&](int k, double2 um, double2 uk, double2 up) -> double2 {
      // u_{k-1} + 4 u_k + u_{k+1} with the P1 end rows (h/6)(2, 1) and the folds
      if (k == 0) {
        const double2 f = make_double2(dL.y * ikappa, -dL.x * ikappa);
        return make_double2(fma(2.0, uk.x, up.x) + f.x, fma(2.0, uk.y, up.y) + f.y);
      }
      if (k == Nj - 1) {
        const double2 f = make_double2(dR.y * ikappa, -dR.x * ikappa);
        return make_double2(fma(2.0, uk.x, um.x) + f.x, fma(2.0, uk.y, um.y) + f.y);
      }
      return make_double2(fma(4.0, uk.x, um.x + up.x), fma(4.0, uk.y, um.y + up.y));
    };
    // ---- forward: z_k = c_k z_{k-1} + q_k (i kappa s_k), c_k = -q_k E_{k-1} ----
    // rows of this CTA through L1 (written by this SM); the halo rows of the
    // neighbouring CTAs from L2 (written by other SMs in the previous step)
    auto ldu = [&](int k) -> double2 { return (k >= rc0 && k < rc1) ? u[k] : __ldcg(u + k); };
    // The two halo values u_{n-1}(rt0 - 1), u_{n-1}(rt1) are read once, before
    // pass 1: once this CTA publishes its forward total, CTA c+1 may finish
    // step n and overwrite its first row with u_n while pass 2 here still needs
    // u_{n-1} (the neighbours' rows are final for step n-1 at this point).
    const double2 halo_m = rt0 > 0 && rt0 < rt1 ? ldu(rt0 - 1) : cz();
    const double2 halo_p = rt1 < Nj && rt0 < rt1 ? ldu(rt1) : cz();
    auto fwd_pass = [&](double2 zin, bool store, double2 &Aout) -> double2 {
      double2 zz = zin, A = make_double2(1.0, 0.0);
      double2 um = halo_m, uk = rt0 < rt1 ? ldu(rt0) : cz();
      double erp = rt0 > 0 ? er[rt0 - 1] : 0.0;
#pragma unroll 4
      for (int k = rt0; k < rt1; k++) {
        const double2 up = k + 1 < Nj ? (k + 1 == rt1 ? halo_p : ldu(k + 1)) : cz();
        const double2 qk = __ldg(q + k);
        const double2 ck = negqe_s(qk, erp, eim);
        const double2 rr = cimul(kappa, sval(k, um, uk, up));
        zz = cfma(ck, zz, cmul(qk, rr));
        if (store) z[k] = zz;
        else A = cmul(ck, A);
        erp = __ldg(er + k);
        um = uk;
        uk = up;
      }
      Aout = A;
      return zz;
    };
    const int par = n & 1;
    double2 A1, F1 = fwd_pass(cz(), false, A1);
    double2 eA, eB, tA, tB;
    cta_scan<true>(A1, F1, scanbuf, eA, eB, tA, tB);
    if (t == 0) {
      fv[(c * 2 + par) * 2 + 0] = tA;
      fv[(c * 2 + par) * 2 + 1] = tB;
      __threadfence();
      st_release(ffwd + c, n);
    }
    race_jitter(1, n);
    // carry into the CTA: fold of the earlier CTAs' totals
    double2 zc = chain_fold(ffwd, fv, c, nc, true, par, n);
    double2 dummy;
    race_jitter(2, n);
    fwd_pass(cfma(eA, zc, eB), true, dummy);
    // ---- backward: x_k = z_k + b_k x_{k+1}, b_k = -q_k E_k ----
    double2 Ab = make_double2(1.0, 0.0), xb = cz();
    for (int k = rt1 - 1; k >= rt0; k--) {
      const double2 bk = negqe_s(__ldg(q + k), __ldg(er + k), eim);
      xb = cfma(bk, xb, z[k]);
      Ab = cmul(bk, Ab);
    }
    cta_scan<false>(Ab, xb, scanbuf, eA, eB, tA, tB);
    if (t == 0) {
      bv[(c * 2 + par) * 2 + 0] = tA;
      bv[(c * 2 + par) * 2 + 1] = tB;
      __threadfence();
      st_release(fbwd + c, n);
    }
    race_jitter(3, n);
    double2 xc = chain_fold(fbwd, bv, c, nc, false, par, n);
    double2 x = cfma(eA, xc, eB), x0v = cz(), xLv = cz();
    for (int k = rt1 - 1; k >= rt0; k--) {
      const double2 bk = negqe_s(__ldg(q + k), __ldg(er + k), eim);
      x = cfma(bk, x, z[k]);
      const double2 uo = u[k];
      u[k] = make_double2(fma(2.0, x.x, -uo.x), fma(2.0, x.y, -uo.y));   // u_n = 2 v_n - u_{n-1}
      if (k == Nj - 1) xLv = x;
      if (k == 0) x0v = x;
    }
    // record v_n and S v_n at the interfaces (eq. 8)
    if (own0) {
      if (histL) hvL[n] = x0v;
      if (p.tc_hi) BoL = cmul(S.rho[0], cadd(BoL, x0v));
      if (has_left && sout_l) {
        const double2 sv = cfma(p.tc_hi ? S.c0e[0] : p.c0, x0v, sHL), l = flux(0, n);
        sout_l[n - 1] = make_double2(fma(2.0, sv.x, -l.x), fma(2.0, sv.y, -l.y));
      }
    }
    if (ownL) {
      if (histR) hvR[n] = xLv;
      if (p.tc_hi) BoR = cmul(S.rho[1], cadd(BoR, xLv));
      if (has_right && sout_r) {
        const double2 sv = cfma(p.tc_hi ? S.c0e[1] : p.c0, xLv, sHR), r = flux(1, n);
        sout_r[n - 1] = make_double2(fma(2.0, sv.x, -r.x), fma(2.0, sv.y, -r.y));
      }
    }
    __syncthreads();
    __threadfence();
    if (t == 0) st_release(fdone + c, n);
  }
  if (S.uT)
    for (int k = rc0 + t; k < rc1; k += P) S.uT[k] = u[k];
}

// Constant matrix (V = 0, V(x), and every higher-order operator): two passes
// per step instead of four.  The linear parts of a thread's forward and
// backward maps do not change during the window, so they are formed once:
// Af = prod c_k, Ab = prod b_k, the prefix products Apre_k = prod_{k'<=k} c_k'
// (one array per system, streamed with z) and G = sum_i (prod_{k<i} b_k)
// Apre_i.  Per step:
//   pass A  forward from carry 0: z^loc stored, the forward offset F and the
//           backward offset B^loc = sum_i (prod_{k<i} b_k) z^loc_i (formed in
//           forward order: no extra pass over z)
//   scans   forward (Af, F) -> z_{rt0-1}; backward (Ab, B^loc + G z_{rt0-1})
//           -> x_{rt1}; each a CTA scan and a chain fold
//   pass B  backward: x_k = (z^loc_k + Apre_k z_{rt0-1}) + b_k x_{k+1},
//           u_n = 2 x - u_{n-1}
// HBM bytes per row and step: pass A reads u, q, Re E (40) and writes z (16);
// pass B reads z, Apre, b, u (64) and writes u (16): 136 (b_k formed once per
// launch instead of from q and Re E every step: 144 -> 136; the four-pass
// form: ~224).
// four CTAs per SM (64 registers): with the interleaved layout the kernel is
// bound by memory latency and more warps win (C2 march at 1 / 2 / 3 / 4 per
// SM: 460 / 277 / 233 / 227 ms)
__global__ void __launch_bounds__(256, 4) k_march_stream2(const MarchParams p, int nc, size_t stride, double2 *ust,
                                                       double2 *zst, double2 *ast, double2 *qst, double *est,
                                                       double2 *bst, int *flags, double2 *vals) {
  extern __shared__ double2 ssm[];
  double2 *scanbuf = ssm;                      // [64]
  double2 *red = scanbuf + 64;                 // [32] block reduction
  double2 *hvL = red + 32;                     // [NT+1] v_s at row 0 (CTA 0 of a system with a left interface)
  double2 *hvR = hvL + (p.NT + 1);             // [NT+1] v_s at row N_j - 1 (last CTA, right interface)
  __shared__ double2 sHL, sHR;
  const int t = threadIdx.x, P = blockDim.x;
  const int sidx = blockIdx.x / nc, c = blockIdx.x % nc;
  const MarchSys &S = p.sys[sidx];
  const int Nj = p.Nj, NT = p.NT;
  const double eim = p.e_im, kappa = p.kappa, ikappa = 1.0 / p.kappa;
  const int Rc = (Nj + nc - 1) / nc;
  const int rc0 = min(Nj, c * Rc), rc1 = min(Nj, (c + 1) * Rc);
  const int Rt = (Rc + P - 1) / P;                     // rows per thread (every CTA)
  const int rt0 = min(rc1, rc0 + t * Rt), rt1 = min(rc1, rc0 + (t + 1) * Rt);
  // thread-interleaved layout of the scratch: row rt0 + i of thread t of CTA c
  // at c P Rt + i P + t, so a warp's access of its threads' i-th rows is one
  // contiguous 512-byte run (the natural layout made every load touch 32 lines)
  const size_t cbase = (size_t)c * P * Rt;
  auto PH = [&](int i) -> size_t { return cbase + (size_t)i * P + t; };
  auto phys_of = [&](int k) -> size_t {
    const int cc = k / Rc, r = k - cc * Rc, tt = r / Rt;
    return (size_t)cc * P * Rt + (size_t)(r - tt * Rt) * P + tt;
  };
  double2 *__restrict__ u = ust + (size_t)sidx * stride;
  double2 *__restrict__ z = zst + (size_t)sidx * stride;
  double2 *__restrict__ ap = ast + (size_t)sidx * stride;
  double2 *__restrict__ qp = qst + (size_t)sidx * stride;
  double *__restrict__ ep = est + (size_t)sidx * stride;
  double2 *__restrict__ bp = bst + (size_t)sidx * stride;
  const int cnt = rt1 - rt0;
  int *fdone = flags + (size_t)sidx * nc * 3, *ffwd = fdone + nc, *fbwd = ffwd + nc;
  double2 *fv = vals + (size_t)sidx * nc * 8, *bv = fv + nc * 4;
  const bool has_left = S.flags & SYS_HAS_LEFT, has_right = S.flags & SYS_HAS_RIGHT;
  const bool first_cta = c == 0, last_cta = rc1 == Nj && rc0 < Nj;
  const bool own0 = first_cta && t == 0 && rt0 == 0 && rt1 > 0;
  const bool ownL = rt1 == Nj && rt0 < Nj;
  const bool histL = first_cta && has_left, histR = last_cta && has_right;
  const int sflags = S.flags;
  const double2 *const slin = S.lin, *const srin = S.rin, *const sq = S.q;
  const double *const ser = S.er;
  double2 *const sout_l = S.out_left, *const sout_r = S.out_right;

  // initial state and the factors, permuted into the interleaved layout
  for (int k = rc0 + t; k < rc1; k += P) {
    const size_t ph = phys_of(k);
    u[ph] = S.u0 ? S.u0[k] : cz();
    qp[ph] = __ldg(sq + k);
    ep[ph] = __ldg(ser + k);
  }
  __syncthreads();
  // the constant parts of the thread's maps
  double2 Af = make_double2(1.0, 0.0), Ab = make_double2(1.0, 0.0), Gt = cz();
  {
    double erp = rt0 > 0 ? __ldg(ser + rt0 - 1) : 0.0;
    for (int i = 0; i < cnt; i++) {
      const double2 qk = qp[PH(i)];
      const double ek = ep[PH(i)];
      Af = cmul(negqe_s(qk, erp, eim), Af);
      ap[PH(i)] = Af;                                      // Apre_k
      Gt = cfma(Ab, Af, Gt);                               // (prod_{k'<k} b) Apre_k
      const double2 bk = negqe_s(qk, ek, eim);
      bp[PH(i)] = bk;                                      // b_k for pass B
      Ab = cmul(Ab, bk);
      erp = ek;
    }
  }
  if (histL && t == 0) hvL[0] = p.tc_hi ? cmul(S.f0[0], S.u0 ? S.u0[0] : cz()) : (S.u0 ? S.u0[0] : cz());
  if (histR && t == 0) hvR[0] = p.tc_hi ? cmul(S.f0[1], S.u0 ? S.u0[Nj - 1] : cz()) : (S.u0 ? S.u0[Nj - 1] : cz());
  double2 BoL = cz(), BoR = cz();
  if (p.tc_hi) {
    if (own0) BoL = cmul(S.rho[0], cmul(S.f0[0], S.u0 ? S.u0[0] : cz()));
    if (ownL) BoR = cmul(S.rho[1], cmul(S.f0[1], S.u0 ? S.u0[Nj - 1] : cz()));
  }
  __syncthreads();
  __threadfence();
  if (t == 0) st_release(fdone + c, 0);
  auto flux = [&](int sd, int n) -> double2 {
    if (sflags & (sd == 0 ? SYS_LIN_IMPULSE : SYS_RIN_IMPULSE)) return make_double2(n == 1 ? 1.0 : 0.0, 0.0);
    const double2 *f = sd == 0 ? slin : srin;
    return f ? f[n - 1] : cz();
  };

  for (int n = 1; n <= NT; n++) {
    race_jitter(0, n);
    if (t == 0) {
      if (c > 0) wait_flag(fdone + c - 1, n - 1);
      if (c < nc - 1) wait_flag(fdone + c + 1, n - 1);
    }
    for (int sd = 0; sd < 2; sd++) {
      if (!(sd == 0 ? histL : histR)) continue;
      const double2 *hv = sd == 0 ? hvL : hvR;
      double2 acc = cz();
      if (p.tc_hi) {
        const double2 *kp = S.kap[sd];
        for (int s = t; s <= n - 1; s += P) acc = cfma(__ldg(kp + n - s), hv[s], acc);
      } else if (p.s02)
        for (int s = t; s <= n - 1; s += P)
          acc = make_double2(fma(p.beta[n - s], hv[s].x, acc.x), fma(p.beta[n - s], hv[s].y, acc.y));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
      if ((t & 31) == 0) red[t >> 5] = acc;
      __syncthreads();
      if (t == 0) {
        double2 hs = cz();
        for (int w = 0; w < (P >> 5); w++) hs = cadd(hs, red[w]);
        (sd == 0 ? sHL : sHR) = p.tc_hi ? hs : (p.s02 ? cmul(p.c2, hs) : cz());
      }
      __syncthreads();
    }
    __syncthreads();
    const double2 dL = (own0 && has_left) ? csub(cfma(cscale(2.0, S.dlt[0]), BoL, sHL), flux(0, n)) : cz();
    const double2 dR = (ownL && has_right) ? csub(cfma(cscale(2.0, S.dlt[1]), BoR, sHR), flux(1, n)) : cz();
    auto sval = [&](int k, double2 um, double2 uk, double2 up) -> double2 {
      if (k == 0) {
        const double2 f = make_double2(dL.y * ikappa, -dL.x * ikappa);
        return make_double2(fma(2.0, uk.x, up.x) + f.x, fma(2.0, uk.y, up.y) + f.y);
      }
      if (k == Nj - 1) {
        const double2 f = make_double2(dR.y * ikappa, -dR.x * ikappa);
        return make_double2(fma(2.0, uk.x, um.x) + f.x, fma(2.0, uk.y, um.y) + f.y);
      }
      return make_double2(fma(4.0, uk.x, um.x + up.x), fma(4.0, uk.y, um.y + up.y));
    };
    auto ldu = [&](int k) -> double2 { return (k >= rc0 && k < rc1) ? u[phys_of(k)] : __ldcg(u + phys_of(k)); };
    // halo rows of u_{n-1}: read before this CTA publishes anything of step n
    const double2 halo_m = rt0 > 0 && rt0 < rt1 ? ldu(rt0 - 1) : cz();
    const double2 halo_p = rt1 < Nj && rt0 < rt1 ? ldu(rt1) : cz();
    const int par = n & 1;
    // ---- pass A ----
    double2 zl = cz(), Bl = cz(), Pb = make_double2(1.0, 0.0);
    {
      double2 um = halo_m, uk = cnt > 0 ? u[PH(0)] : cz();
      double erp = rt0 > 0 ? __ldg(ser + rt0 - 1) : 0.0;
#pragma unroll 4
      for (int i = 0; i < cnt; i++) {
        const int k = rt0 + i;
        const double2 up = k + 1 < Nj ? (i + 1 == cnt ? halo_p : u[PH(i + 1)]) : cz();
        const double2 qk = qp[PH(i)];
        const double ek = ep[PH(i)];
        const double2 rr = cimul(kappa, sval(k, um, uk, up));
        zl = cfma(negqe_s(qk, erp, eim), zl, cmul(qk, rr));
        z[PH(i)] = zl;
        Bl = cfma(Pb, zl, Bl);
        Pb = cmul(Pb, negqe_s(qk, ek, eim));
        erp = ek;
        um = uk;
        uk = up;
      }
    }
    double2 eA, eB, tA, tB;
    cta_scan<true>(Af, zl, scanbuf, eA, eB, tA, tB);
    if (t == 0) {
      fv[(c * 2 + par) * 2 + 0] = tA;
      fv[(c * 2 + par) * 2 + 1] = tB;
      __threadfence();
      st_release(ffwd + c, n);
    }
    race_jitter(1, n);
    double2 zc = chain_fold(ffwd, fv, c, nc, true, par, n);
    zc = cfma(eA, zc, eB);                                  // z_{rt0-1}
    cta_scan<false>(Ab, cfma(Gt, zc, Bl), scanbuf, eA, eB, tA, tB);
    if (t == 0) {
      bv[(c * 2 + par) * 2 + 0] = tA;
      bv[(c * 2 + par) * 2 + 1] = tB;
      __threadfence();
      st_release(fbwd + c, n);
    }
    race_jitter(2, n);
    double2 xc = chain_fold(fbwd, bv, c, nc, false, par, n);
    // ---- pass B ----
    double2 x = cfma(eA, xc, eB), x0v = cz(), xLv = cz();
    for (int i = cnt - 1; i >= 0; i--) {
      const int k = rt0 + i;
      const size_t ph = PH(i);
      x = cfma(bp[ph], x, cfma(ap[ph], zc, z[ph]));
      const double2 uo = u[ph];
      u[ph] = make_double2(fma(2.0, x.x, -uo.x), fma(2.0, x.y, -uo.y));
      if (k == Nj - 1) xLv = x;
      if (k == 0) x0v = x;
    }
    if (own0) {
      if (histL) hvL[n] = x0v;
      if (p.tc_hi) BoL = cmul(S.rho[0], cadd(BoL, x0v));
      if (has_left && sout_l) {
        const double2 sv = cfma(p.tc_hi ? S.c0e[0] : p.c0, x0v, sHL), l = flux(0, n);
        sout_l[n - 1] = make_double2(fma(2.0, sv.x, -l.x), fma(2.0, sv.y, -l.y));
      }
    }
    if (ownL) {
      if (histR) hvR[n] = xLv;
      if (p.tc_hi) BoR = cmul(S.rho[1], cadd(BoR, xLv));
      if (has_right && sout_r) {
        const double2 sv = cfma(p.tc_hi ? S.c0e[1] : p.c0, xLv, sHR), r = flux(1, n);
        sout_r[n - 1] = make_double2(fma(2.0, sv.x, -r.x), fma(2.0, sv.y, -r.y));
      }
    }
    __syncthreads();
    __threadfence();
    if (t == 0) st_release(fdone + c, n);
  }
  if (S.uT) {
    __syncthreads();
    for (int k = rc0 + t; k < rc1; k += P) S.uT[k] = u[phys_of(k)];
  }
}

size_t march_stream_smem_bytes(int NT) { return (size_t)(64 + 32 + 2 * (NT + 1)) * sizeof(double2); }

// Streams the systems in batches whose chains are all co-resident.  The
// chain length nc (CTAs per system, i.e. how a system's rows are split and
// its scans reassociated) depends on N_j, the GPU and nsys_ref (the
// problem's subdomain count) only -- not on how many systems a launch or a
// rank carries -- so a rank of a multi-GPU run rounds exactly as one GPU.
cudaError_t launch_march_stream(MarchParams p, int nsys_total, int nsys_ref, double2 *ust, double2 *zst,
                                double2 *ast, double2 *qst, double *est, double2 *bst, size_t stride, int *flags,
                                double2 *vals, cudaStream_t st) {
  // constant matrix: the two-pass form (Apre in ast); V(t,x): four passes
  const bool two = p.td_stride == 0 && ast != nullptr;
  const void *kfun = two ? (const void *)k_march_stream2 : (const void *)k_march_stream;
  const size_t smem = march_stream_smem_bytes(p.NT);
  cudaError_t e = cudaFuncSetAttribute(kfun, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kfun, 256, smem);
  if (e != cudaSuccess) return e;
  const int cap = nsm * per_sm;
  if (cap < 1) return cudaErrorInvalidConfiguration;
  const MarchSys *all = p.sys;
  int nc = std::max(1, cap / std::max(1, nsys_ref));
  nc = std::min(nc, std::max(1, p.Nj / 256));   // at least a row per thread
  const int per_batch = std::max(1, cap / nc);
  for (int s0 = 0; s0 < nsys_total;) {
    const int nb = std::min(nsys_total - s0, per_batch);
    MarchParams q = p;
    q.sys = all + s0;
    q.nsys = nb;
    if (getenv("SWR_VERBOSE")) {
      cudaFuncAttributes fa;
      cudaFuncGetAttributes(&fa, k_march_stream);
      fprintf(stderr, "k_march_stream: %d systems x %d CTAs (%d per SM, %d regs, smem %zu), N_j %d\n", nb, nc, per_sm,
              fa.numRegs, smem, p.Nj);
    }
    e = cudaMemsetAsync(flags, 0xff, (size_t)nb * nc * 3 * sizeof(int), st);   // -1: nothing reported yet
    if (e != cudaSuccess) return e;
    if (two) {
      if ((size_t)nc * 256 * (((p.Nj + nc - 1) / nc + 255) / 256) > stride) return cudaErrorInvalidValue;
      void *args[] = {(void *)&q,   (void *)&nc,  (void *)&stride, (void *)&ust,   (void *)&zst,
                      (void *)&ast, (void *)&qst, (void *)&est,    (void *)&bst,   (void *)&flags, (void *)&vals};
      e = cudaLaunchCooperativeKernel(kfun, dim3(nb * nc), dim3(256), args, smem, st);
    } else {
      void *args[] = {(void *)&q, (void *)&nc, (void *)&ust, (void *)&zst, (void *)&flags, (void *)&vals};
      e = cudaLaunchCooperativeKernel(kfun, dim3(nb * nc), dim3(256), args, smem, st);
    }
    if (e != cudaSuccess) return e;
    s0 += nb;
  }
  return cudaSuccess;
}

// ---------------------------------------------------------------------------
// Nonlinear march for subdomains beyond the resident NL march (N_j > 65,536,
// e.g. N = 10 at dx = 1e-5): f(u) = lambda |u|^2, the Duran-Sanz-Serna
// midpoint with the inner fixed point of eq. (12) (readings A3,
// A4), the arithmetic of k_march_nl with the chain structure of
// k_march_stream.  Per step n, fixed-point iteration s:
//   pass 1  forward from carry 0: rhs = i kappa (u_{k-1} + 4u_k + u_{k+1})
//           - (h/12) load_k(zeta^s) (+ the end-row folds) -> affine map
//   scan    CTA scan, chain fold of the earlier CTAs' published totals
//   pass 2  forward from the exact carry, z stored
//   pass 3  backward from carry 0 over z, scan, chain fold in reverse
//   pass 4  backward from the exact carry: zeta^{s+1} (in place) and the
//           maxima max |zeta^{s+1} - zeta^s|^2, max |zeta^{s+1}|^2
//   maxima  every CTA publishes its maxima (value + iteration flag) and reads
//           all the chain's: the stop decision is uniform (reading A4)
// then u_n = 2 zeta - u_{n-1}.  The halo rows of u_{n-1} and zeta^s are read
// before pass 1 (a neighbour may overwrite them once this CTA has published
// its forward total).  Flags count global fixed-point iterations (ic), so the
// value buffers alternate by the parity of ic.
// ---------------------------------------------------------------------------
// four CTAs per SM as k_march_stream2 (one R_nl sweep at N_j = 420,001:
// 615 ms at two per SM, 320 ms at four)
__global__ void __launch_bounds__(256, 4) k_march_nl_stream(const MarchParams p, int nc, size_t stride,
                                                            double2 *ust, double2 *zst, double2 *zest, double2 *ast,
                                                            double2 *qst, double *est, int *flags, double2 *vals) {
  extern __shared__ double2 ssm[];
  double2 *scanbuf = ssm;                      // [64]
  double2 *red = scanbuf + 64;                 // [32] block reductions
  double2 *hvL = red + 32;                     // [NT+1] v_s at row 0
  double2 *hvR = hvL + (p.NT + 1);             // [NT+1] v_s at row N_j - 1
  __shared__ double2 sHL, sHR, smx;
  const int t = threadIdx.x, P = blockDim.x, lane = t & 31, w = t >> 5, nw = P >> 5;
  const int sidx = blockIdx.x / nc, c = blockIdx.x % nc;
  const MarchSys &S = p.sys[sidx];
  const int Nj = p.Nj, NT = p.NT;
  const double eim = p.e_im, kappa = p.kappa, h12 = p.h12, lam = p.lambda;
  const int Rc = (Nj + nc - 1) / nc;
  const int rc0 = min(Nj, c * Rc), rc1 = min(Nj, (c + 1) * Rc);
  const int Rt = (Rc + P - 1) / P;                     // rows per thread (every CTA)
  const int rt0 = min(rc1, rc0 + t * Rt), rt1 = min(rc1, rc0 + (t + 1) * Rt);
  // the thread-interleaved scratch layout of k_march_stream2
  const size_t cbase = (size_t)c * P * Rt;
  auto PH = [&](int i) -> size_t { return cbase + (size_t)i * P + t; };
  auto phys_of = [&](int k) -> size_t {
    const int cc = k / Rc, r = k - cc * Rc, tt = r / Rt;
    return (size_t)cc * P * Rt + (size_t)(r - tt * Rt) * P + tt;
  };
  const int cnt = rt1 - rt0;
  double2 *__restrict__ u = ust + (size_t)sidx * stride;
  double2 *__restrict__ z = zst + (size_t)sidx * stride;
  double2 *__restrict__ ze = zest + (size_t)sidx * stride;
  double2 *__restrict__ ap = ast + (size_t)sidx * stride;
  double2 *__restrict__ qp = qst + (size_t)sidx * stride;
  double *__restrict__ ep = est + (size_t)sidx * stride;
  int *fdone = flags + (size_t)sidx * nc * 4, *ffwd = fdone + nc, *fbwd = ffwd + nc, *fmx = fbwd + nc;
  double2 *fv = vals + (size_t)sidx * nc * 10, *bv = fv + nc * 4, *mv = bv + nc * 4;   // [nc][parity](A,B) x2, [nc][parity]
  const bool has_left = S.flags & SYS_HAS_LEFT, has_right = S.flags & SYS_HAS_RIGHT;
  const bool first_cta = c == 0, last_cta = rc1 == Nj && rc0 < Nj;
  const bool own0 = first_cta && t == 0 && rt0 == 0 && rt1 > 0;
  const bool ownL = rt1 == Nj && rt0 < Nj;
  const bool histL = first_cta && has_left, histR = last_cta && has_right;

  for (int k = rc0 + t; k < rc1; k += P) {
    const double2 v = S.u0 ? S.u0[k] : cz();
    const size_t ph = phys_of(k);
    u[ph] = v;
    ze[ph] = v;                                 // zeta^0 of step 1 = v_0 = u_0
    qp[ph] = __ldg(S.q + k);
    ep[ph] = __ldg(S.er + k);
  }
  __syncthreads();
  if (histL && t == 0) hvL[0] = S.u0 ? S.u0[0] : cz();
  if (histR && t == 0) hvR[0] = S.u0 ? S.u0[Nj - 1] : cz();
  const int sflags = S.flags;
  const double2 *const slin = S.lin, *const srin = S.rin, *const sq = S.q;
  const double *const ser = S.er;
  // the constant parts of the thread's maps (k_march_stream2): Af, Ab, G and
  // the prefix products Apre_k of the forward map
  double2 Af = make_double2(1.0, 0.0), Ab = make_double2(1.0, 0.0), Gt = cz();
  {
    double erp = rt0 > 0 ? __ldg(ser + rt0 - 1) : 0.0;
    for (int i = 0; i < cnt; i++) {
      const double2 qk = qp[PH(i)];
      const double ek = ep[PH(i)];
      Af = cmul(negqe_s(qk, erp, eim), Af);
      ap[PH(i)] = Af;
      Gt = cfma(Ab, Af, Gt);
      Ab = cmul(Ab, negqe_s(qk, ek, eim));
      erp = ek;
    }
  }
  __syncthreads();
  __threadfence();
  if (t == 0) st_release(fdone + c, 0);

  double2 *const sout_l = S.out_left, *const sout_r = S.out_right;
  auto flux = [&](int sd, int n) -> double2 {
    if (sflags & (sd == 0 ? SYS_LIN_IMPULSE : SYS_RIN_IMPULSE)) return make_double2(n == 1 ? 1.0 : 0.0, 0.0);
    const double2 *f = sd == 0 ? slin : srin;
    return f ? f[n - 1] : cz();
  };
  int fp_max = 0, fp_fail = 0, ic = 0;

  for (int n = 1; n <= NT; n++) {
    race_jitter(0, n);
    if (t == 0) {
      if (c > 0) wait_flag(fdone + c - 1, n - 1);
      if (c < nc - 1) wait_flag(fdone + c + 1, n - 1);
    }
    // S0^2 history of the end rows this CTA holds
    for (int sd = 0; sd < 2; sd++) {
      if (!(sd == 0 ? histL : histR)) continue;
      const double2 *hv = sd == 0 ? hvL : hvR;
      double2 acc = cz();
      if (p.s02)
        for (int s = t; s <= n - 1; s += P)
          acc = make_double2(fma(p.beta[n - s], hv[s].x, acc.x), fma(p.beta[n - s], hv[s].y, acc.y));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
      if (lane == 0) red[w] = acc;
      __syncthreads();
      if (t == 0) {
        double2 hs = cz();
        for (int q = 0; q < nw; q++) hs = cadd(hs, red[q]);
        (sd == 0 ? sHL : sHR) = p.s02 ? cmul(p.c2, hs) : cz();
      }
      __syncthreads();
    }
    __syncthreads();
    const double2 dL = (own0 && has_left) ? csub(sHL, flux(0, n)) : cz();
    const double2 dR = (ownL && has_right) ? csub(sHR, flux(1, n)) : cz();
    const double ikappa = 1.0 / kappa;
    auto sval = [&](int k, double2 um, double2 uk, double2 up) -> double2 {
      if (k == 0) {
        const double2 f = make_double2(dL.y * ikappa, -dL.x * ikappa);
        return make_double2(fma(2.0, uk.x, up.x) + f.x, fma(2.0, uk.y, up.y) + f.y);
      }
      if (k == Nj - 1) {
        const double2 f = make_double2(dR.y * ikappa, -dR.x * ikappa);
        return make_double2(fma(2.0, uk.x, um.x) + f.x, fma(2.0, uk.y, um.y) + f.y);
      }
      return make_double2(fma(4.0, uk.x, um.x + up.x), fma(4.0, uk.y, um.y + up.y));
    };
    // load_k(zeta) of the P1 elements (k-1, k), (k, k+1) (reading A3)
    auto nload = [&](int k, double2 zm, double2 zk, double2 zp) -> double2 {
      const double Wc = lam * fma(zk.x, zk.x, zk.y * zk.y);
      double2 ld = cz();
      if (k > 0) {
        const double Wm = lam * fma(zm.x, zm.x, zm.y * zm.y);
        ld.x = fma(Wm + 3.0 * Wc, zk.x, (Wm + Wc) * zm.x);
        ld.y = fma(Wm + 3.0 * Wc, zk.y, (Wm + Wc) * zm.y);
      }
      if (k < Nj - 1) {
        const double Wp = lam * fma(zp.x, zp.x, zp.y * zp.y);
        ld.x = fma(3.0 * Wc + Wp, zk.x, fma(Wc + Wp, zp.x, ld.x));
        ld.y = fma(3.0 * Wc + Wp, zk.y, fma(Wc + Wp, zp.y, ld.y));
      }
      return ld;
    };
    auto ldg = [&](const double2 *a, int k) -> double2 {
      return (k >= rc0 && k < rc1) ? a[phys_of(k)] : __ldcg(a + phys_of(k));
    };
    // u_{n-1} halo rows: final for step n-1, unchanged through the iterations
    const double2 uh_m = rt0 > 0 && rt0 < rt1 ? ldg(u, rt0 - 1) : cz();
    const double2 uh_p = rt1 < Nj && rt0 < rt1 ? ldg(u, rt1) : cz();
    bool conv = false;
    int it;
    for (it = 1; it <= p.maxit_fp; it++, ic++) {
      const int par = ic & 1;
      // zeta^s halo rows, read before this CTA publishes anything of iteration ic
      const double2 zh_m = rt0 > 0 && rt0 < rt1 ? ldg(ze, rt0 - 1) : cz();
      const double2 zh_p = rt1 < Nj && rt0 < rt1 ? ldg(ze, rt1) : cz();
      // pass A: forward from carry 0 -- z^loc stored, the forward offset and
      // the backward offset B^loc = sum_i (prod_{k<i} b_k) z^loc_i
      double2 zl = cz(), Bl = cz(), Pb = make_double2(1.0, 0.0);
      {
        double2 um = uh_m, uk = cnt > 0 ? u[PH(0)] : cz();
        double2 zm = zh_m, zk = cnt > 0 ? ze[PH(0)] : cz();
        double erp = rt0 > 0 ? __ldg(ser + rt0 - 1) : 0.0;
#pragma unroll 2
        for (int i = 0; i < cnt; i++) {
          const int k = rt0 + i;
          const bool lastrow = i + 1 == cnt;
          const double2 up = k + 1 < Nj ? (lastrow ? uh_p : u[PH(i + 1)]) : cz();
          const double2 zp = k + 1 < Nj ? (lastrow ? zh_p : ze[PH(i + 1)]) : cz();
          const double2 qk = qp[PH(i)];
          const double ek = ep[PH(i)];
          const double2 sv = cimul(kappa, sval(k, um, uk, up));
          const double2 ld = nload(k, zm, zk, zp);
          const double2 rr = make_double2(fma(-h12, ld.x, sv.x), fma(-h12, ld.y, sv.y));
          zl = cfma(negqe_s(qk, erp, eim), zl, cmul(qk, rr));
          z[PH(i)] = zl;
          Bl = cfma(Pb, zl, Bl);
          Pb = cmul(Pb, negqe_s(qk, ek, eim));
          erp = ek;
          um = uk;
          uk = up;
          zm = zk;
          zk = zp;
        }
      }
      double2 eA, eB, tA, tB;
      cta_scan<true>(Af, zl, scanbuf, eA, eB, tA, tB);
      if (t == 0) {
        fv[(c * 2 + par) * 2 + 0] = tA;
        fv[(c * 2 + par) * 2 + 1] = tB;
        __threadfence();
        st_release(ffwd + c, ic);
      }
      race_jitter(1, n);
      double2 zc = chain_fold(ffwd, fv, c, nc, true, par, ic);
      zc = cfma(eA, zc, eB);                              // z_{rt0-1}
      cta_scan<false>(Ab, cfma(Gt, zc, Bl), scanbuf, eA, eB, tA, tB);
      if (t == 0) {
        bv[(c * 2 + par) * 2 + 0] = tA;
        bv[(c * 2 + par) * 2 + 1] = tB;
        __threadfence();
        st_release(fbwd + c, ic);
      }
      race_jitter(2, n);
      double2 xc = chain_fold(fbwd, bv, c, nc, false, par, ic);
      // pass B: zeta^{s+1}_k = (z^loc_k + Apre_k z_{rt0-1}) + b_k zeta^{s+1}_{k+1}, in place, and the maxima
      double2 x = cfma(eA, xc, eB);
      double dmax = 0.0, nmax = 0.0;
      for (int i = cnt - 1; i >= 0; i--) {
        const size_t ph = PH(i);
        const double2 bk = negqe_s(qp[ph], ep[ph], eim);   // (a stored b_k measured slower here: 324 -> 350 ms)
        x = cfma(bk, x, cfma(ap[ph], zc, z[ph]));
        const double2 zo = ze[ph];
        const double dx = x.x - zo.x, dy = x.y - zo.y;
        dmax = fmax(dmax, fma(dx, dx, dy * dy));
        nmax = fmax(nmax, fma(x.x, x.x, x.y * x.y));
        ze[ph] = x;
      }
      // chain-wide maxima -> uniform decision
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        nmax = fmax(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
      }
      if (lane == 0) red[w] = make_double2(dmax, nmax);
      __syncthreads();
      if (w == 0) {
        // the CTA's maxima, published; then every chain CTA's (lanes in parallel)
        double2 mm = cz();
        for (int q = 0; q < nw; q++) mm = make_double2(fmax(mm.x, red[q].x), fmax(mm.y, red[q].y));
        if (lane == 0) {
          mv[c * 2 + par] = mm;
          __threadfence();
          st_release(fmx + c, ic);
        }
        race_jitter(3, n);
        for (int cc = lane; cc < nc; cc += 32) {
          if (cc == c) continue;
          wait_flag(fmx + cc, ic);
          const double2 v = __ldcg(mv + cc * 2 + par);
          mm = make_double2(fmax(mm.x, v.x), fmax(mm.y, v.y));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          mm.x = fmax(mm.x, __shfl_xor_sync(0xffffffffu, mm.x, o));
          mm.y = fmax(mm.y, __shfl_xor_sync(0xffffffffu, mm.y, o));
        }
        if (lane == 0) smx = mm;
      }
      __syncthreads();
      const double2 mm = smx;
      if (sqrt(mm.x) <= p.tol_fp * sqrt(mm.y)) { conv = true; ic++; break; }
      __syncthreads();   // smx is rewritten next iteration
    }
    if (!conv) { it = p.maxit_fp; fp_fail = 1; }
    if (it > fp_max) fp_max = it;
    // v_n = zeta; u_n = 2 v_n - u_{n-1}; record S v_n at the interfaces (eq. 8)
    for (int i = 0; i < cnt; i++) {
      const size_t ph = PH(i);
      const double2 v = ze[ph], uo = u[ph];
      u[ph] = make_double2(fma(2.0, v.x, -uo.x), fma(2.0, v.y, -uo.y));
    }
    if (own0) {
      const double2 x0v = ze[phys_of(0)];
      if (histL) hvL[n] = x0v;
      if (has_left && sout_l) {
        const double2 sv = cfma(p.c0, x0v, sHL), l = flux(0, n);
        sout_l[n - 1] = make_double2(fma(2.0, sv.x, -l.x), fma(2.0, sv.y, -l.y));
      }
    }
    if (ownL) {
      const double2 xLv = ze[phys_of(Nj - 1)];
      if (histR) hvR[n] = xLv;
      if (has_right && sout_r) {
        const double2 sv = cfma(p.c0, xLv, sHR), r = flux(1, n);
        sout_r[n - 1] = make_double2(fma(2.0, sv.x, -r.x), fma(2.0, sv.y, -r.y));
      }
    }
    __syncthreads();
    __threadfence();
    if (t == 0) st_release(fdone + c, n);
  }
  if (S.uT) {
    __syncthreads();
    for (int k = rc0 + t; k < rc1; k += P) S.uT[k] = u[phys_of(k)];
  }
  if (c == 0 && t == 0 && p.fp_stat) {
    atomicMax(p.fp_stat, fp_max);
    if (fp_fail) atomicOr(p.fp_stat + 1, 1);
  }
}

// Chains of co-resident CTAs as launch_march_stream (the chain length depends
// on N_j and the problem's subdomain count only).  scratch (one batch of at
// most nslot / nc systems): u, z, zeta [batch][N_j]; flags [batch][nc][4];
// vals [batch][nc][10].
cudaError_t launch_march_nl_stream(MarchParams p, int nsys_total, int nsys_ref, double2 *ust, double2 *zst,
                                   double2 *zest, double2 *ast, double2 *qst, double *est, size_t stride, int *flags,
                                   double2 *vals, int nslot, cudaStream_t st) {
  const size_t smem = march_stream_smem_bytes(p.NT);
  cudaError_t e = cudaFuncSetAttribute(k_march_nl_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_march_nl_stream, 256, smem);
  if (e != cudaSuccess) return e;
  const int cap = std::min(nsm * per_sm, nslot);
  if (cap < 1) return cudaErrorInvalidConfiguration;
  const MarchSys *all = p.sys;
  int nc = std::max(1, cap / std::max(1, nsys_ref));
  nc = std::min(nc, std::max(1, p.Nj / 256));
  const int per_batch = std::max(1, cap / nc);
  for (int s0 = 0; s0 < nsys_total;) {
    const int nb = std::min(nsys_total - s0, per_batch);
    MarchParams q = p;
    q.sys = all + s0;
    q.nsys = nb;
    if (getenv("SWR_VERBOSE"))
      fprintf(stderr, "k_march_nl_stream: %d systems x %d CTAs (%d per SM), N_j %d\n", nb, nc, per_sm, p.Nj);
    e = cudaMemsetAsync(flags, 0xff, (size_t)nb * nc * 4 * sizeof(int), st);
    if (e != cudaSuccess) return e;
    // the scratch holds one batch (batches run in stream order)
    if ((size_t)nc * 256 * (((p.Nj + nc - 1) / nc + 255) / 256) > stride) return cudaErrorInvalidValue;
    void *args[] = {(void *)&q,   (void *)&nc,  (void *)&stride, (void *)&ust,   (void *)&zst, (void *)&zest,
                    (void *)&ast, (void *)&qst, (void *)&est,    (void *)&flags, (void *)&vals};
    e = cudaLaunchCooperativeKernel((const void *)k_march_nl_stream, dim3(nb * nc), dim3(256), args, smem, st);
    if (e != cudaSuccess) return e;
    s0 += nb;
  }
  return cudaSuccess;
}

// chain length and scratch stride of the two-pass streaming march (the
// interleaved layout pads every CTA's block to P Rt rows)
size_t stream2_stride(int Nj, int nsys_ref, int NT) {
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // the largest block layout of the two interleaved kernels (their chain
  // lengths follow their own occupancy)
  size_t best = 0;
  for (const void *kf : {(const void *)k_march_stream2, (const void *)k_march_nl_stream}) {
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kf, 256, march_stream_smem_bytes(NT)) != cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    int nc = std::max(1, nsm * per_sm / std::max(1, nsys_ref));
    nc = std::min(nc, std::max(1, Nj / 256));
    const int Rc = (Nj + nc - 1) / nc, Rt = (Rc + 255) / 256;
    best = std::max(best, (size_t)nc * 256 * Rt);
  }
  return best;
}

}  // namespace swr

// swr_march.cu — the whole-window Crank-Nicolson march of many subdomain
// systems (the hot path of PAPER.md, eq. (5) P:193-198 and eq. (9)).
//
// One system = one subdomain j with one right-hand side (physical u0 for
// d = R(0), a unit-impulse probe for the Toeplitz columns of L, or the final
// sweep).  Per time step n the system solves the complex tridiagonal
//   (A - B) v_n = i kappa (u_{n-1,k-1} + 4 u_{n-1,k} + u_{n-1,k+1}) + b_n - Q^T(l_n, r_n)^T
// with constant pivots q_k = 1/p_k of (A - B) (factor once), then
// u_n = 2 v_n - u_{n-1}, and records S v_n at a_j and b_j (eq. 8).
//
// B200 mapping.  A thread-block cluster of CS CTAs owns one system for all
// N_T steps; each thread owns M consecutive rows and keeps u_{n-1}, the
// pivots and Re E_k of its rows in registers for the whole window, the
// forward-sweep values z_k in shared memory.  Nothing but the boundary
// traces touches HBM inside the march.  The Thomas recurrences
//   z_k = q_k r_k + c_k z_{k-1},   c_k = -q_k E_{k-1}      (forward)
//   x_k = z_k + b_k x_{k+1},        b_k = -q_k E_k          (backward)
// are first-order affine recurrences: each thread reduces its rows to one
// affine map, the maps are scanned (warp shuffles -> shared memory ->
// DSMEM across the cluster) to get every thread's carry-in, and the thread
// re-runs its rows from the exact carry (same arithmetic as a sequential
// Thomas sweep, only the carry is reassociated).
#include "swr_common.cuh"
#include "swr_kernels.h"
#include <cooperative_groups.h>
#include <cstdio>

namespace cg = cooperative_groups;

namespace swr {

__device__ __forceinline__ void compose(double2 &A, double2 &B, double2 Ae, double2 Be) {
  // (A,B) o (Ae,Be):  x -> A (Ae x + Be) + B
  B = cfma(A, Be, B);
  A = cmul(A, Ae);
}

// Barrier over the system's CTAs.  Inside a CTA a bar.sync orders shared
// memory; across the cluster only the threads that wrote data read by other
// CTAs (halo rows, pushed scan totals) fence, everyone else arrives relaxed
// (no per-thread membar).
__device__ __forceinline__ void csync(int CS, bool wrote_remote_visible = false) {
  __syncthreads();
  if (CS > 1) {
    if (wrote_remote_visible) asm volatile("fence.acq_rel.cluster;" ::: "memory");
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
  }
}

template <typename T>
__device__ __forceinline__ T *remote(T *p, int rank) {
  return cg::this_cluster().map_shared_rank(p, rank);
}

// c2 * sum_{s=0}^{n-1} beta_{n-s} hv[s]  (S0^2 history),
// evaluated by one warp from shared memory; every lane returns the sum.
__device__ __forceinline__ double2 hist_sum(const double2 *hv, const double *beta, int n, int lane, double2 c2) {
  double2 a0 = cz(), a1 = cz();
  int s = lane;
#pragma unroll 1
  for (; s + 32 < n; s += 64) {
    const double b0 = beta[n - s], b1 = beta[n - s - 32];
    const double2 v0 = hv[s], v1 = hv[s + 32];
    a0.x = fma(b0, v0.x, a0.x); a0.y = fma(b0, v0.y, a0.y);
    a1.x = fma(b1, v1.x, a1.x); a1.y = fma(b1, v1.y, a1.y);
  }
  if (s < n) {
    const double b0 = beta[n - s];
    const double2 v0 = hv[s];
    a0.x = fma(b0, v0.x, a0.x); a0.y = fma(b0, v0.y, a0.y);
  }
  double2 acc = cadd(a0, a1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
  return cmul(c2, acc);
}

// Scan state shared by the CTA (shared memory).
struct ScanSmem {
  double2 *wA, *wB;   // [32] warp totals
  double2 *xA, *xB;   // [32] warp-exclusive prefixes
  double2 *ctot;      // [32] CTA totals pushed by the cluster peers: [dir*16 + ab*8 + crank]
};

// Exclusive scan (in row order) of the per-thread affine maps z -> A z + B;
// returns the carry-in (the composition of all earlier maps applied to 0).
__device__ __forceinline__ double2 scan_fwd(double2 A, double2 B, const ScanSmem &ss, int lane, int w, int nw,
                                            int CS, int crank) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double2 Ae = shfl_up2(A, o), Be = shfl_up2(B, o);
    if (lane >= o) compose(A, B, Ae, Be);
  }
  double2 eA = shfl_up2(A, 1), eB = shfl_up2(B, 1);
  if (lane == 0) { eA = make_double2(1.0, 0.0); eB = cz(); }
  if (lane == 31) { ss.wA[w] = A; ss.wB[w] = B; }
  __syncthreads();
  if (w == 0) {
    double2 a = lane < nw ? ss.wA[lane] : make_double2(1.0, 0.0);
    double2 b = lane < nw ? ss.wB[lane] : cz();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double2 Ae = shfl_up2(a, o), Be = shfl_up2(b, o);
      if (lane >= o) compose(a, b, Ae, Be);
    }
    double2 ea = shfl_up2(a, 1), eb = shfl_up2(b, 1);
    if (lane == 0) { ea = make_double2(1.0, 0.0); eb = cz(); }
    if (lane < nw) { ss.xA[lane] = ea; ss.xB[lane] = eb; }
    if (CS > 1 && lane == nw - 1) {
#pragma unroll 1
      for (int c = crank + 1; c < CS; c++) {
        *remote(ss.ctot + crank, c) = a;
        *remote(ss.ctot + 8 + crank, c) = b;
      }
    }
  }
  csync(CS, w == 0 && lane == nw - 1);
  double2 val = cz();
#pragma unroll 1
  for (int c = 0; c < crank; c++) val = cfma(ss.ctot[c], val, ss.ctot[8 + c]);
  val = cfma(ss.xA[w], val, ss.xB[w]);
  return cfma(eA, val, eB);
}

// Same in reverse row order (backward substitution).
__device__ __forceinline__ double2 scan_bwd(double2 A, double2 B, const ScanSmem &ss, int lane, int w, int nw,
                                            int CS, int crank) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double2 Ae = shfl_down2(A, o), Be = shfl_down2(B, o);
    if (lane + o < 32) compose(A, B, Ae, Be);
  }
  double2 eA = shfl_down2(A, 1), eB = shfl_down2(B, 1);
  if (lane == 31) { eA = make_double2(1.0, 0.0); eB = cz(); }
  if (lane == 0) { ss.wA[w] = A; ss.wB[w] = B; }
  __syncthreads();
  if (w == 0) {
    double2 a = lane < nw ? ss.wA[lane] : make_double2(1.0, 0.0);
    double2 b = lane < nw ? ss.wB[lane] : cz();
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const double2 Ae = shfl_down2(a, o), Be = shfl_down2(b, o);
      if (lane + o < 32) compose(a, b, Ae, Be);
    }
    double2 ea = shfl_down2(a, 1), eb = shfl_down2(b, 1);
    if (lane == 31) { ea = make_double2(1.0, 0.0); eb = cz(); }
    if (lane < nw) { ss.xA[lane] = ea; ss.xB[lane] = eb; }
    if (CS > 1 && lane == 0) {
#pragma unroll 1
      for (int c = 0; c < crank; c++) {
        *remote(ss.ctot + 16 + crank, c) = a;
        *remote(ss.ctot + 24 + crank, c) = b;
      }
    }
  }
  csync(CS, w == 0 && lane == 0);
  double2 val = cz();
#pragma unroll 1
  for (int c = CS - 1; c > crank; c--) val = cfma(ss.ctot[16 + c], val, ss.ctot[24 + c]);
  val = cfma(ss.xA[w], val, ss.xB[w]);
  return cfma(eA, val, eB);
}

// -q (er + i eim)
__device__ __forceinline__ double2 negqe(double2 q, double er, double eim) {
  return make_double2(fma(q.y, eim, -q.x * er), -fma(q.x, eim, q.y * er));
}

// Row k of the rhs of eq. (9) without the interface terms:
// (2i/dt) M u_{n-1} = i kappa (u_{k-1} + 4u_k + u_{k+1}); end rows (2u_k + u_{k+-1}).
__device__ __forceinline__ double2 rhs_row(int k, int Nj, double2 um, double2 uk, double2 up, double kappa) {
  double2 s;
  if (k == 0) s = make_double2(fma(2.0, uk.x, up.x), fma(2.0, uk.y, up.y));
  else if (k == Nj - 1) s = make_double2(fma(2.0, uk.x, um.x), fma(2.0, uk.y, um.y));
  else s = make_double2(fma(4.0, uk.x, um.x + up.x), fma(4.0, uk.y, um.y + up.y));
  return cimul(kappa, s);
}

// Hide loop invariance from the compiler so that per-row coefficients
// (c_k, b_k) are recomputed in each pass instead of being hoisted into
// registers: the resident state must fit the register file.
template <int M>
__device__ __forceinline__ void launder(double2 (&q)[M], double (&er)[M]) {
#pragma unroll
  for (int i = 0; i < M; i++) asm volatile("" : "+d"(q[i].x), "+d"(q[i].y), "+d"(er[i]));
}

// Shared-memory scalars of the boundary rows (one writer, one reader each).
struct BndSmem {
  double2 Ha, Hb;      // S0^2 history terms at a_j / b_j for the current step
  double2 lin, rin;    // incoming fluxes l_{j,n}, r_{j,n}
};

template <int M, int PMAX>
__global__ void __launch_bounds__(PMAX, 1) k_march_resident(const MarchParams p) {
  extern __shared__ double2 sm[];
  const int P = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int crank = blockIdx.x % p.CS;
  const MarchSys *Sp = p.sys + blockIdx.x / p.CS;
  const int Nj = p.Nj;
  const int s0 = (crank * P + t) * M;      // first row of this thread

  // shared memory: ybuf [M*P] | hfirst [P] | hlast [P] | Af [P] | Ab [P] |
  //                scan scratch [160] | hva [NT+1] | hvb [NT+1] | bnd
  double2 *ybuf = sm;
  double2 *hfirst = ybuf + M * P;
  double2 *hlast = hfirst + P;
  double2 *sAf = hlast + P;
  double2 *sAb = sAf + P;
  ScanSmem ss;
  ss.wA = sAb + P; ss.wB = ss.wA + 32; ss.xA = ss.wB + 32; ss.xB = ss.xA + 32; ss.ctot = ss.xB + 32;
  double2 *hva = ss.ctot + 32;
  double2 *hvb = hva + (p.NT + 1);
  BndSmem *bnd = reinterpret_cast<BndSmem *>(hvb + (p.NT + 1));
  double2 *hred = reinterpret_cast<double2 *>(bnd + 1);   // [64] warp partials of H_a, H_b
  double *sbeta = reinterpret_cast<double *>(hred + 64);    // [NT+1]
  for (int i = t; i <= p.NT; i += P) sbeta[i] = p.beta[i];

  double2 u[M], q[M];
  double er[M];
  double er_prev;
  {
    const double2 *u0p = Sp->u0, *qp = Sp->q;
    const double *erp = Sp->er;
#pragma unroll
    for (int i = 0; i < M; i++) {
      const int k = s0 + i;
      if (k < Nj) {
        q[i] = qp[k];
        er[i] = erp[k];
        u[i] = u0p ? u0p[k] : cz();
      } else {
        q[i] = make_double2(1.0, 0.0);
        er[i] = 0.0;
        u[i] = cz();
      }
    }
    // constant aggregate factors: Af = prod c_k, Ab = prod b_k over the thread's rows
    er_prev = (s0 >= 1 && s0 - 1 < Nj) ? erp[s0 - 1] : 0.0;
    double2 Af = make_double2(1.0, 0.0), Ab = make_double2(1.0, 0.0);
#pragma unroll
    for (int i = 0; i < M; i++) {
      const int k = s0 + i;
      const double2 c = (k >= 1 && k < Nj) ? negqe(q[i], i == 0 ? er_prev : er[i == 0 ? 0 : i - 1], p.e_im) : cz();
      const double2 b = (k < Nj - 1) ? negqe(q[i], er[i], p.e_im) : cz();
      Af = cmul(Af, c);
      Ab = cmul(Ab, b);
    }
    sAf[t] = Af;
    sAb[t] = Ab;
  }
  const int flags = Sp->flags;
  const int rows_cta = P * M;
  const int cb = (Nj - 1) / rows_cta, tb = ((Nj - 1) % rows_cta) / M;
  const bool owns_a = (flags & SYS_HAS_LEFT) && s0 == 0;
  const bool owns_b = (flags & SYS_HAS_RIGHT) && crank == cb && t == tb;
  if (s0 == 0) hva[0] = u[0];
#pragma unroll
  for (int i = 0; i < M; i++)
    if (s0 + i == Nj - 1) hvb[0] = u[i];
  if (t == 0) { bnd->Ha = cz(); bnd->Hb = cz(); bnd->lin = cz(); bnd->rin = cz(); }
  // incoming flux of the next step, prefetched by the owning lane
  auto flux_at = [&](const double2 *ser, int imp, int nn) -> double2 {
    if (nn > p.NT) return cz();
    if (imp) return make_double2(nn == 1 ? 1.0 : 0.0, 0.0);
    return ser ? ser[nn - 1] : cz();
  };
  double2 fnext = cz();
  if ((flags & SYS_HAS_LEFT) && crank == 0 && t == 0) fnext = flux_at(Sp->lin, flags & SYS_LIN_IMPULSE, 1);
  double2 fnext_b = cz();
  if ((flags & SYS_HAS_RIGHT) && crank == cb && t == tb) fnext_b = flux_at(Sp->rin, flags & SYS_RIN_IMPULSE, 1);
  __syncthreads();

#pragma unroll 1
  for (int n = 1; n <= p.NT; n++) {
    // ---- boundary scalars of step n ----
    // S0^2 history H = c2 sum_{s<n} beta_{n-s} v_s: every thread of the CTA
    // holding the boundary row adds a slice of s <= n-2 (written before the
    // last barrier), warp partials go to shared memory and the owner of the
    // row adds them and its own newest term beta_1 v_{n-1} after the halo
    // barrier.
    if (p.s02) {
      if ((flags & SYS_HAS_LEFT) && crank == 0) {
        double2 acc = cz();
        for (int q = t; q < n - 1; q += P) {
          const double b = sbeta[n - q];
          const double2 v = hva[q];
          acc.x = fma(b, v.x, acc.x);
          acc.y = fma(b, v.y, acc.y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
        if (lane == 0) hred[w] = acc;
      }
      if ((flags & SYS_HAS_RIGHT) && crank == cb) {
        double2 acc = cz();
        for (int q = t; q < n - 1; q += P) {
          const double b = sbeta[n - q];
          const double2 v = hvb[q];
          acc.x = fma(b, v.x, acc.x);
          acc.y = fma(b, v.y, acc.y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
        if (lane == 0) hred[32 + w] = acc;
      }
    }
    if (owns_a) {
      bnd->lin = fnext;
      fnext = flux_at(Sp->lin, flags & SYS_LIN_IMPULSE, n + 1);
    }
    if (owns_b) {
      bnd->rin = fnext_b;
      fnext_b = flux_at(Sp->rin, flags & SYS_RIN_IMPULSE, n + 1);
    }
    // ---- halo: u_{n-1} of the neighbouring rows ----
    hfirst[t] = u[0];
    hlast[t] = u[M - 1];
    csync(p.CS, t == 0 || t == P - 1);
    if (p.s02 && (owns_a || owns_b)) {
      double2 ha = owns_a ? cscale(sbeta[1], hva[n - 1]) : cz();
      double2 hb = owns_b ? cscale(sbeta[1], hvb[n - 1]) : cz();
      for (int q = 0; q < (P >> 5); q++) {
        if (owns_a) ha = cadd(ha, hred[q]);
        if (owns_b) hb = cadd(hb, hred[32 + q]);
      }
      if (owns_a) bnd->Ha = cmul(p.c2, ha);
      if (owns_b) bnd->Hb = cmul(p.c2, hb);
    }
    double2 uL = cz(), uR = cz();
    if (t > 0) uL = hlast[t - 1];
    else if (crank > 0) uL = *remote(hlast + (P - 1), crank - 1);
    if (t < P - 1) uR = hfirst[t + 1];
    else if (crank < p.CS - 1) uR = *remote(hfirst, crank + 1);

    // ---- forward sweep z_k = q_k r_k + c_k z_{k-1}: aggregate, scan, exact ----
    double2 z = cz();
    for (int pass = 0; pass < 2; pass++) {
      launder<M>(q, er);
#pragma unroll
      for (int i = 0; i < M; i++) {
        const int k = s0 + i;
        double2 r = cz(), c = cz();
        if (k < Nj) {
          r = rhs_row(k, Nj, i == 0 ? uL : u[i == 0 ? 0 : i - 1], u[i], i == M - 1 ? uR : u[i == M - 1 ? M - 1 : i + 1],
                      p.kappa);
          if (k == 0 && owns_a) r = cadd(r, csub(bnd->Ha, bnd->lin));
          if (k == Nj - 1 && owns_b) r = cadd(r, csub(bnd->Hb, bnd->rin));
          if (k >= 1) c = negqe(q[i], i == 0 ? er_prev : er[i == 0 ? 0 : i - 1], p.e_im);
        }
        z = cfma(c, z, cmul(q[i], r));
        if (pass == 1) ybuf[i * P + t] = z;
      }
      if (pass == 0) z = scan_fwd(sAf[t], z, ss, lane, w, P >> 5, p.CS, crank);
    }
    // ---- backward sweep x_k = z_k + b_k x_{k+1}: aggregate, scan, exact ----
    double2 x = cz();
    launder<M>(q, er);
#pragma unroll
    for (int i = M - 1; i >= 0; i--) {
      const int k = s0 + i;
      const double2 b = (k < Nj - 1) ? negqe(q[i], er[i], p.e_im) : cz();
      x = cfma(b, x, ybuf[i * P + t]);
    }
    x = scan_bwd(sAb[t], x, ss, lane, w, P >> 5, p.CS, crank);
    launder<M>(q, er);
#pragma unroll
    for (int i = M - 1; i >= 0; i--) {
      const int k = s0 + i;
      const double2 b = (k < Nj - 1) ? negqe(q[i], er[i], p.e_im) : cz();
      x = cfma(b, x, ybuf[i * P + t]);
      if (k == 0 && owns_a) {
        hva[n] = x;
        double2 *outl = Sp->out_left;
        if (outl) {
          const double2 sv = cfma(p.c0, x, bnd->Ha);   // S v_n(a_j) = c0 v_n + H_a
          const double2 l = bnd->lin;
          outl[n - 1] = make_double2(fma(2.0, sv.x, -l.x), fma(2.0, sv.y, -l.y));
        }
      }
      if (k == Nj - 1 && owns_b) {
        hvb[n] = x;
        double2 *outr = Sp->out_right;
        if (outr) {
          const double2 sv = cfma(p.c0, x, bnd->Hb);
          const double2 r = bnd->rin;
          outr[n - 1] = make_double2(fma(2.0, sv.x, -r.x), fma(2.0, sv.y, -r.y));
        }
      }
      u[i] = make_double2(fma(2.0, x.x, -u[i].x), fma(2.0, x.y, -u[i].y));   // u_n = 2 v_n - u_{n-1}
    }
  }
  double2 *uTp = Sp->uT;
  if (uTp) {
#pragma unroll
    for (int i = 0; i < M; i++)
      if (s0 + i < Nj) uTp[s0 + i] = u[i];
  }
  if (p.CS > 1) cg::this_cluster().sync();  // keep shared memory alive for remote readers
}

// ---------------------------------------------------------------------------
// Launch-shape selection and launcher.
// Instantiated (rows per thread M, max threads per CTA PMAX); the register
// cap is 65536 / PMAX per thread.
// ---------------------------------------------------------------------------
struct Inst { int M, PMAX; };
static const Inst kInst[] = {{1, 512}, {2, 512}, {4, 512}, {6, 256}, {8, 256}, {10, 256}, {11, 256}, {12, 256}};

MarchShape choose_march_shape(int Nj) {
  MarchShape best{0, 0, 0};
  double best_cost = 1e300;
  for (int CS = 1; CS <= 16; CS++) {
    for (const Inst &in : kInst) {
      const int M = in.M;
      long per = ((long)Nj + (long)CS * M - 1) / ((long)CS * M);
      int P = (int)((per + 31) / 32 * 32);
      if (P < 32) P = 32;
      if (P > in.PMAX) continue;
      double padded = (double)CS * P * M;
      double cost = padded * (1.0 + 0.10 * (CS - 1)) * (P < 128 ? 1.3 : 1.0);
      if (cost < best_cost) { best_cost = cost; best = {M, P, CS}; }
    }
  }
  return best;
}

size_t march_smem_bytes(const MarchShape &s, int NT) {
  return sizeof(double2) * ((size_t)s.M * s.P + 4 * (size_t)s.P + 160 + 2 * (size_t)(NT + 1) + 64) +
         sizeof(BndSmem) + sizeof(double) * (size_t)(NT + 1);
}

template <int M, int PMAX>
static cudaError_t launch_m(const MarchParams &p, const MarchShape &s, size_t smem, cudaStream_t st) {
  auto kern = k_march_resident<M, PMAX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (s.CS > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.nsys * s.CS, 1, 1);
  cfg.blockDim = dim3(s.P, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  cfg.attrs = attr;
  cfg.numAttrs = 0;
  if (s.CS > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = s.CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.numAttrs = 1;
  }
  return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_march(MarchParams p, const MarchShape &s, cudaStream_t st) {
  p.CS = s.CS;
  const size_t smem = march_smem_bytes(s, p.NT);
  switch (s.M) {
    case 1: return launch_m<1, 512>(p, s, smem, st);
    case 2: return launch_m<2, 512>(p, s, smem, st);
    case 4: return launch_m<4, 512>(p, s, smem, st);
    case 6: return launch_m<6, 256>(p, s, smem, st);
    case 8: return launch_m<8, 256>(p, s, smem, st);
    case 11: return launch_m<11, 256>(p, s, smem, st);
    case 12: return launch_m<12, 256>(p, s, smem, st);
    case 10: return launch_m<10, 256>(p, s, smem, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace swr

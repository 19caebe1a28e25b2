// swr_march.cu — the whole-window Crank-Nicolson march of many subdomain
// systems (the hot path of PAPER.md, eq. (5) P:193-198 and eq. (9)).
//
// One *group* = one subdomain j with K right-hand sides that share its
// matrix (A - B): the physical u0 for d = R(0) and the l_j / r_j
// unit-impulse probes for the Toeplitz columns of L in the
// build, K = 1 for the final sweep and R(g).  Per time step n each RHS solves
//   (A - B) v_n = i kappa (u_{n-1,k-1} + 4 u_{n-1,k} + u_{n-1,k+1}) + b_n - Q^T(l_n, r_n)^T
// with the constant pivots q_k = 1/p_k of (A - B) (factor once),
// then u_n = 2 v_n - u_{n-1}, and records S v_n at a_j and b_j (eq. 8).
//
// B200 mapping.  A thread-block cluster of CS CTAs owns one group for all
// N_T steps; each thread owns M consecutive rows and keeps u_{n-1} of its
// rows for all K RHS, the pivots and Re E_k in registers for the whole
// window, the forward-sweep values z_k in shared memory.  Nothing but the
// boundary traces touches HBM inside the march.  The Thomas recurrences
//   z_k = q_k r_k + c_k z_{k-1},   c_k = -q_k E_{k-1}      (forward)
//   x_k = z_k + b_k x_{k+1},        b_k = -q_k E_k          (backward)
// are first-order affine recurrences: each thread reduces its rows to one
// affine map per RHS (the K maps share their linear part, which depends on
// the matrix only), the maps are scanned (warp shuffles -> shared memory ->
// DSMEM pushes to the later CTAs of the cluster) to get every thread's
// carry-in, and the thread re-runs its rows from the exact carry (the same
// arithmetic as a sequential Thomas sweep, only the carry is reassociated).
// The K RHS are K independent dependency chains per thread (ILP) under the
// same barriers.
#include "swr_common.cuh"
#include "swr_kernels.h"
#include <cstdio>
#include <cstdlib>
#include <cooperative_groups.h>
#include <algorithm>

namespace cg = cooperative_groups;

namespace swr {

// Barrier over the group's CTAs.  Inside a CTA a bar.sync orders shared
// memory; across the cluster only the threads that wrote data read by other
// CTAs (halo rows, pushed scan totals) fence, everyone else arrives relaxed.
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

// mbarrier + st.async exchange between the CTAs of a cluster (no fences:
// the consumer's phase wait covers the remote stores it counts).
__device__ __forceinline__ uint32_t smem_u32(const void *ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }
__device__ __forceinline__ void mbar_init(unsigned long long *mb, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(mb)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *mb, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(smem_u32(mb)), "r"(parity) : "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// 16-byte remote store counted by the destination CTA's mbarrier
__device__ __forceinline__ void st_async(uint32_t raddr, double2 v, uint32_t rmb) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];"
               ::"r"(raddr), "d"(v.x), "d"(v.y), "r"(rmb) : "memory");
}

// -q (er + i eim)
__device__ __forceinline__ double2 negqe(double2 q, double er, double eim) {
  return make_double2(fma(q.y, eim, -q.x * er), -fma(q.x, eim, q.y * er));
}

// -q (er + i eim) in the scaled variables of the constant-matrix path:
// qk = i kappa q, et = er / kappa, eimt = eim / kappa  ->  qk (-eimt + i et)
__device__ __forceinline__ double2 ck(double2 qk, double et, double eimt) {
  return make_double2(fma(-qk.x, eimt, -qk.y * et), fma(qk.x, et, -qk.y * eimt));
}
// u_{k-1} + 4 u_k + u_{k+1}
__device__ __forceinline__ double2 srow(double2 um, double2 uk, double2 up) {
  return make_double2(fma(4.0, uk.x, um.x + up.x), fma(4.0, uk.y, um.y + up.y));
}

// Row k of (2i/dt) M u_{n-1} = i kappa (u_{k-1} + 4u_k + u_{k+1}); end rows
// of the P1 mass matrix are (h/6)(2, 1).
template <bool GEN>
__device__ __forceinline__ double2 rhs_row(int k, int Nj, double2 um, double2 uk, double2 up, double kappa) {
  double2 s;
  if (GEN && k == 0) s = make_double2(fma(2.0, uk.x, up.x), fma(2.0, uk.y, up.y));
  else if (GEN && k == Nj - 1) s = make_double2(fma(2.0, uk.x, um.x), fma(2.0, uk.y, um.y));
  else s = make_double2(fma(4.0, uk.x, um.x + up.x), fma(4.0, uk.y, um.y + up.y));
  return cimul(kappa, s);
}

// Hide loop invariance from the compiler so per-row coefficients are
// recomputed in each pass instead of being hoisted into registers: the
// resident state must fit the register file.
template <int M>
__device__ __forceinline__ void launder(double2 (&q)[M], double (&er)[M]) {
#pragma unroll
  for (int i = 0; i < M; i++) asm volatile("" : "+d"(q[i].x), "+d"(q[i].y), "+d"(er[i]));
}

// Shared-memory pointers of the scans of one direction.
template <int K>
struct ScanBuf {
  double2 *wA;       // [32] warp totals, linear part
  double2 *wB;       // [K][32] warp totals, offsets
  double2 *ctot;     // [16][1+K] totals pushed by the other CTAs of the cluster
};

// Exclusive scan of the per-thread affine maps z -> A z + B_k (k < K) in row
// order (FWD) or reverse row order; returns the carries (the composition of
// all earlier maps applied to 0).  One bar.sync; the CTA totals travel by
// st.async into the parity buffer sb.ctot of every CTA that needs them,
// counted by that CTA's mbarrier mb (phase parity ph).
template <int K, bool FWD>
__device__ __forceinline__ void scan_maps(double2 A, double2 (&B)[K], const ScanBuf<K> &sb, int lane, int w, int nw,
                                          int CS, int crank, double2 (&carry)[K], long long *tr = nullptr,
                                          unsigned long long *mb = nullptr, uint32_t ph = 0) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double2 Ae = FWD ? shfl_up2(A, o) : shfl_down2(A, o);
    const bool take = FWD ? lane >= o : lane + o < 32;
#pragma unroll
    for (int k = 0; k < K; k++) {
      const double2 Be = FWD ? shfl_up2(B[k], o) : shfl_down2(B[k], o);
      if (take) B[k] = cfma(A, Be, B[k]);
    }
    if (take) A = cmul(A, Ae);
  }
  // lane-exclusive prefix
  double2 eA = FWD ? shfl_up2(A, 1) : shfl_down2(A, 1);
  double2 eB[K];
#pragma unroll
  for (int k = 0; k < K; k++) eB[k] = FWD ? shfl_up2(B[k], 1) : shfl_down2(B[k], 1);
  const bool first = FWD ? lane == 0 : lane == 31;
  if (first) {
    eA = make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 0; k < K; k++) eB[k] = cz();
  }
  if (tr) tr[0] = clock64();
  const int tot_lane = FWD ? 31 : 0;
  if (lane == tot_lane) {
    sb.wA[w] = A;
#pragma unroll
    for (int k = 0; k < K; k++) sb.wB[k * 32 + w] = B[k];
  }
  __syncthreads();
  if (tr) tr[1] = clock64();
  // every warp scans the warp totals itself (no second CTA barrier)
  double2 a = lane < nw ? sb.wA[lane] : make_double2(1.0, 0.0);
  double2 b[K];
#pragma unroll
  for (int k = 0; k < K; k++) b[k] = lane < nw ? sb.wB[k * 32 + lane] : cz();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    if (o >= nw) break;   // nw warps: log2(nw) levels
    const double2 ae = FWD ? shfl_up2(a, o) : shfl_down2(a, o);
    const bool take = FWD ? lane >= o : lane + o < 32;
#pragma unroll
    for (int k = 0; k < K; k++) {
      const double2 be = FWD ? shfl_up2(b[k], o) : shfl_down2(b[k], o);
      if (take) b[k] = cfma(a, be, b[k]);
    }
    if (take) a = cmul(a, ae);
  }
  // warp-exclusive prefix of warp w: inclusive value of warp w -+ 1
  const bool wfirst = FWD ? w == 0 : w == nw - 1;
  const int wsrc = wfirst ? 0 : (FWD ? w - 1 : w + 1);
  double2 xa = make_double2(__shfl_sync(0xffffffffu, a.x, wsrc), __shfl_sync(0xffffffffu, a.y, wsrc));
  double2 xb[K];
#pragma unroll
  for (int k = 0; k < K; k++)
    xb[k] = make_double2(__shfl_sync(0xffffffffu, b[k].x, wsrc), __shfl_sync(0xffffffffu, b[k].y, wsrc));
  if (wfirst) {
    xa = make_double2(1.0, 0.0);
#pragma unroll
    for (int k = 0; k < K; k++) xb[k] = cz();
  }
  if (tr) tr[2] = clock64();
  double2 val[K];
#pragma unroll
  for (int k = 0; k < K; k++) val[k] = cz();
  if (CS > 1) {
    // CTA total = inclusive over all warps (lane nw-1 forward, lane 0 backward),
    // broadcast over warp 0; lane i of warp 0 pushes it to the i-th CTA that
    // needs it (st.async, counted by that CTA's mbarrier)
    const int tl = FWD ? nw - 1 : 0;
    const int c0 = FWD ? crank + 1 : 0, c1 = FWD ? CS : crank;
    if (w == 0) {
      const double2 ta = make_double2(__shfl_sync(0xffffffffu, a.x, tl), __shfl_sync(0xffffffffu, a.y, tl));
      double2 tb[K];
#pragma unroll
      for (int k = 0; k < K; k++)
        tb[k] = make_double2(__shfl_sync(0xffffffffu, b[k].x, tl), __shfl_sync(0xffffffffu, b[k].y, tl));
      const int c = c0 + lane;
      if (c < c1) {
        const uint32_t dst = mapa(smem_u32(sb.ctot + crank * (1 + K)), c), rmb = mapa(smem_u32(mb), c);
        st_async(dst, ta, rmb);
#pragma unroll
        for (int k = 0; k < K; k++) st_async(dst + 16 * (1 + k), tb[k], rmb);
      }
    }
    if (tr) tr[3] = clock64();
    const int nin = FWD ? crank : CS - 1 - crank;   // CTAs whose totals this CTA receives
    if (nin > 0) {
      if (threadIdx.x == 0) mbar_expect_tx(mb, (unsigned)(nin * 16 * (1 + K)));
      mbar_wait(mb, ph);
      // fold of the received totals in chain order (the earlier CTAs' maps
      // forward, the later ones' backward) applied to 0: a tree over the
      // lanes of every warp (lane i holds the i-th map of the chain order)
      double2 fa = make_double2(1.0, 0.0), fb[K];
#pragma unroll
      for (int k = 0; k < K; k++) fb[k] = cz();
      if (lane < nin) {
        const int c = FWD ? lane : CS - 1 - lane;
        const double2 *tc = sb.ctot + c * (1 + K);
        fa = tc[0];
#pragma unroll
        for (int k = 0; k < K; k++) fb[k] = tc[1 + k];
      }
#pragma unroll
      for (int o = 1; o < 16; o <<= 1) {
        if (o >= nin) break;
        // lane l (span [l, l+o)) then lane l+o (span [l+o, l+2o)): second o first
        const double2 na = shfl_down2(fa, o);
#pragma unroll
        for (int k = 0; k < K; k++) {
          const double2 nb = shfl_down2(fb[k], o);
          if (lane + o < 32) fb[k] = cfma(na, fb[k], nb);
        }
        if (lane + o < 32) fa = cmul(na, fa);
      }
#pragma unroll
      for (int k = 0; k < K; k++) val[k] = make_double2(__shfl_sync(0xffffffffu, fb[k].x, 0), __shfl_sync(0xffffffffu, fb[k].y, 0));
    }
  }
  if (tr) tr[4] = clock64();
#pragma unroll
  for (int k = 0; k < K; k++) {
    val[k] = cfma(xa, val[k], xb[k]);
    carry[k] = cfma(eA, val[k], eB[k]);
  }
}

// ---------------------------------------------------------------------------
// Scans with precomputed linear parts.  For a constant matrix the linear
// part of every partial composition (per thread, per warp, per CTA) is fixed
// for the whole window, so only the offsets B travel through the shuffles,
// shared memory and the cluster; the linear factors come from a table built
// once by scan_tab_init (the same composition tree applied to the A's alone).
// ---------------------------------------------------------------------------
struct ScanTab {
  double2 *lvlA;   // [5][P]  this thread's inclusive A before warp-level step L
  double2 *eA;     // [P]     lane-exclusive A
  double2 *lvla;   // [5][32] warp-total A (lane = warp index) before level-2 step L
  double2 *xa;     // [32]    warp-exclusive A
  double2 *ctA;    // [16]    CTA totals of the cluster
};
__host__ __device__ constexpr int kScanTabD2(int P) { return 6 * P + 5 * 32 + 32 + 16; }
__device__ __forceinline__ ScanTab scan_tab_at(double2 *base, int P) {
  ScanTab tb;
  tb.lvlA = base; tb.eA = base + 5 * P; tb.lvla = tb.eA + P; tb.xa = tb.lvla + 5 * 32; tb.ctA = tb.xa + 32;
  return tb;
}

// Build the table of one direction from the per-thread linear parts A; the
// CTA total is stored into ctA[crank] of every CTA of the cluster (visible
// after the caller's cluster barrier).  One bar.sync.
template <bool FWD>
__device__ void scan_tab_init(double2 A, double2 *wA, const ScanTab &tb, int t, int P, int lane, int w, int nw,
                              int CS, int crank) {
#pragma unroll
  for (int L = 0; L < 5; L++) {
    const int o = 1 << L;
    const double2 Ae = FWD ? shfl_up2(A, o) : shfl_down2(A, o);
    const bool take = FWD ? lane >= o : lane + o < 32;
    tb.lvlA[L * P + t] = A;
    if (take) A = cmul(A, Ae);
  }
  double2 eA = FWD ? shfl_up2(A, 1) : shfl_down2(A, 1);
  if (FWD ? lane == 0 : lane == 31) eA = make_double2(1.0, 0.0);
  tb.eA[t] = eA;
  if (lane == (FWD ? 31 : 0)) wA[w] = A;
  __syncthreads();
  double2 a = lane < nw ? wA[lane] : make_double2(1.0, 0.0);
#pragma unroll
  for (int L = 0; L < 5; L++) {
    const int o = 1 << L;
    if (o >= nw) break;
    const double2 ae = FWD ? shfl_up2(a, o) : shfl_down2(a, o);
    const bool take = FWD ? lane >= o : lane + o < 32;
    if (w == 0) tb.lvla[L * 32 + lane] = a;
    if (take) a = cmul(a, ae);
  }
  const bool wfirst = FWD ? w == 0 : w == nw - 1;
  const int wsrc = wfirst ? 0 : (FWD ? w - 1 : w + 1);
  double2 xa = make_double2(__shfl_sync(0xffffffffu, a.x, wsrc), __shfl_sync(0xffffffffu, a.y, wsrc));
  if (wfirst) xa = make_double2(1.0, 0.0);
  if (lane == 0) tb.xa[w] = xa;
  if (w == 0 && lane == (FWD ? nw - 1 : 0)) {
    for (int c = 0; c < CS; c++) *remote(tb.ctA + crank, c) = a;   // CTA total A
  }
}

// Exclusive scan of the offsets B_k with the tabulated linear parts: warp
// shuffles, then a serial fold over the other warps' totals, then the CTA
// totals of the cluster, which travel by st.async (K values) into the parity
// buffer sb.ctot of the CTAs that need them, counted by their mbarrier mb
// (phase parity ph).  extra() runs between the pushes and the wait.
template <int K, bool FWD, typename Extra>
__device__ __forceinline__ void scan_tab(double2 (&B)[K], const ScanBuf<K> &sb, const ScanTab &tb, int t, int P,
                                         int lane, int w, int nw, int CS, int crank, double2 (&carry)[K],
                                         unsigned long long *mb, uint32_t ph, Extra &&extra,
                                         long long *tr = nullptr) {
#pragma unroll
  for (int L = 0; L < 5; L++) {
    const int o = 1 << L;
    const bool take = FWD ? lane >= o : lane + o < 32;
    const double2 Am = tb.lvlA[L * P + t];
#pragma unroll
    for (int k = 0; k < K; k++) {
      const double2 Be = FWD ? shfl_up2(B[k], o) : shfl_down2(B[k], o);
      if (take) B[k] = cfma(Am, Be, B[k]);
    }
  }
  const bool first = FWD ? lane == 0 : lane == 31;
  double2 eB[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    eB[k] = FWD ? shfl_up2(B[k], 1) : shfl_down2(B[k], 1);
    if (first) eB[k] = cz();
  }
  if (tr) tr[0] = clock64();
  if (lane == (FWD ? 31 : 0)) {
#pragma unroll
    for (int k = 0; k < K; k++) sb.wB[k * 32 + w] = B[k];
  }
  __syncthreads();
  if (tr) tr[1] = clock64();
  double2 b[K];
#pragma unroll
  for (int k = 0; k < K; k++) b[k] = lane < nw ? sb.wB[k * 32 + lane] : cz();
#pragma unroll
  for (int L = 0; L < 5; L++) {
    const int o = 1 << L;
    if (o >= nw) break;
    const bool take = FWD ? lane >= o : lane + o < 32;
    const double2 am = tb.lvla[L * 32 + lane];
#pragma unroll
    for (int k = 0; k < K; k++) {
      const double2 be = FWD ? shfl_up2(b[k], o) : shfl_down2(b[k], o);
      if (take) b[k] = cfma(am, be, b[k]);
    }
  }
  const bool wfirst = FWD ? w == 0 : w == nw - 1;
  const int wsrc = wfirst ? 0 : (FWD ? w - 1 : w + 1);
  double2 xb[K];
#pragma unroll
  for (int k = 0; k < K; k++) {
    xb[k] = make_double2(__shfl_sync(0xffffffffu, b[k].x, wsrc), __shfl_sync(0xffffffffu, b[k].y, wsrc));
    if (wfirst) xb[k] = cz();
  }
  if (tr) tr[2] = clock64();
  double2 val[K];
#pragma unroll
  for (int k = 0; k < K; k++) val[k] = cz();
  if (CS > 1) {
    const int tl = FWD ? nw - 1 : 0;            // lane of warp 0 holding the CTA total
    const int c0 = FWD ? crank + 1 : 0, c1 = FWD ? CS : crank;
    if (w == 0 && lane == tl) {
      const uint32_t src = smem_u32(sb.ctot + crank * K), lmb = smem_u32(mb);
#pragma unroll 1
      for (int c = c0; c < c1; c++) {
        const uint32_t dst = mapa(src, c), rmb = mapa(lmb, c);
#pragma unroll
        for (int k = 0; k < K; k++) st_async(dst + 16 * k, b[k], rmb);
      }
    }
    extra();
    if (tr) tr[3] = clock64();
    const int nin = FWD ? crank : CS - 1 - crank;
    if (nin > 0) {
      if (threadIdx.x == 0) mbar_expect_tx(mb, (unsigned)(nin * 16 * K));
      mbar_wait(mb, ph);
      if (FWD) {
#pragma unroll 1
        for (int c = 0; c < crank; c++) {
          const double2 ca = tb.ctA[c];
#pragma unroll
          for (int k = 0; k < K; k++) val[k] = cfma(ca, val[k], sb.ctot[c * K + k]);
        }
      } else {
#pragma unroll 1
        for (int c = CS - 1; c > crank; c--) {
          const double2 ca = tb.ctA[c];
#pragma unroll
          for (int k = 0; k < K; k++) val[k] = cfma(ca, val[k], sb.ctot[c * K + k]);
        }
      }
    }
  } else {
    extra();
  }
  if (tr) tr[4] = clock64();
  const double2 xa = tb.xa[w], eA = tb.eA[t];
#pragma unroll
  for (int k = 0; k < K; k++) {
    val[k] = cfma(xa, val[k], xb[k]);
    carry[k] = cfma(eA, val[k], eB[k]);
  }
}

// Optional per-phase clock64 trace (p.trace != NULL): thread 0 of each CTA
// of the first cluster, step 200, 32 slots per CTA (clock64 is per SM: only
// differences within one CTA are meaningful).
#ifndef SWR_MARCH_TRACE
#define SWR_MARCH_TRACE 0   // build with SWR_TRACE_BUILD=1 to compile the trace points in
#endif
#define SWR_TRACE_ON (SWR_MARCH_TRACE && p.trace && blockIdx.x < (unsigned)CS && t == 0 && n == 200)
#define SWR_TRACE(slot)                                                          \
  do {                                                                           \
    if (SWR_TRACE_ON) p.trace[blockIdx.x * 32 + (slot)] = clock64();             \
  } while (0)

// ---------------------------------------------------------------------------
// i kappa-fold: the value u* such that i kappa u* = d (a rhs addition d on a
// row written as an extra neighbour value): u* = -i d / kappa (ikappa = 1/kappa).
__device__ __forceinline__ double2 ifold(double2 d, double ikappa) { return make_double2(d.y * ikappa, -d.x * ikappa); }

template <int M, int K, int PMAX, bool TDM>
__global__ void __launch_bounds__(PMAX, PMAX <= 128 ? 2 : 1) k_march(const MarchParams p) {
  extern __shared__ double2 sm[];
  const int P = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5, nw = P >> 5;
  const int CS = p.CS;
  const int crank = blockIdx.x % CS;
  const MarchSys *G = p.sys + (size_t)(blockIdx.x / CS) * K;   // the group's K systems
  const int Nj = p.Nj, NT = p.NT;
  const int s0 = (crank * P + t) * M;                          // first row of this thread
  const double eim = p.e_im, kappa = p.kappa, ikappa = 1.0 / p.kappa;

  // ---- shared memory ----
  // mbarriers of the cluster scans: [forward, backward][step parity]
  unsigned long long *mbar = reinterpret_cast<unsigned long long *>(sm);
  double2 *ybuf = sm + 2;                               // [K][M][P]
  double2 *hfirst = ybuf + K * M * P;                   // [K][P]
  double2 *hlast = hfirst + K * P;                      // [K][P]
  double2 *sAf = hlast + K * P;                         // [P]
  double2 *sAb = sAf + P;                               // [P]
  ScanBuf<K> sf, sbk;                                   // ctot: [2 parities][16][1+K]
  sf.wA = sAb + P;                   sf.wB = sf.wA + 32;       sf.ctot = sf.wB + 32 * K;
  sbk.wA = sf.ctot + 32 * (1 + K); sbk.wB = sbk.wA + 32; sbk.ctot = sbk.wB + 32 * K;
  double2 *hva = sbk.ctot + 32 * (1 + K);               // [K][NT+1] v_s(a_j)
  double2 *hvb = hva + K * (NT + 1);                    // [K][NT+1] v_s(b_j)
  double2 *hred = hvb + K * (NT + 1);                   // [K][2 par][2 side][32] warp partials of H
  double2 *sH = hred + K * 128;                         // [K][2] H_a, H_b of the current step
  double2 *sflux = sH + 2 * K;                          // [K][2][NT] incoming fluxes (if p.flux_smem)
  double2 *tabbase = sflux + (p.flux_smem ? 2 * K * NT : 0);
  const ScanTab tabF = scan_tab_at(tabbase, P);                          // constant matrix only
  const ScanTab tabB = scan_tab_at(tabbase + kScanTabD2(P), P);
  double2 *sApre = tabbase + 2 * kScanTabD2(P);         // [M][P] prefix products of the forward maps
  double2 *sG = sApre + M * P;                          // [P] coupling of the forward carry into x_s
  double *sbeta = reinterpret_cast<double *>(sG + P);   // [NT+1]
  double2 *kapS = reinterpret_cast<double2 *>(sbeta + ((NT + 2) & ~1));   // tc_hi: [K][2][NT+1] even kernels

  const int flags = G[0].flags;
  const bool has_left = flags & SYS_HAS_LEFT, has_right = flags & SYS_HAS_RIGHT;
  const int rows_cta = P * M;
  const int cb = (Nj - 1) / rows_cta, tb = ((Nj - 1) % rows_cta) / M;
  const bool first = s0 == 0;                                   // holds row 0
  const bool last = crank == cb && t == tb;                     // holds row N_j - 1
  const int ib = (Nj - 1) - s0;                                 // its index in the thread (if last)
  const bool owns_a = has_left && first;
  const bool owns_b = has_right && last;
  int imp[K][2];
#pragma unroll
  for (int r = 0; r < K; r++) {
    imp[r][0] = G[r].flags & SYS_LIN_IMPULSE;
    imp[r][1] = G[r].flags & SYS_RIN_IMPULSE;
  }

  // TDM: the factors of step n+1 arrive by bulk copy (TMA) into the scan-table
  // region (unused on this path) while step n runs: pmb, pq[rows_cta], pe[rows_cta + 2]
  unsigned long long *pmb = reinterpret_cast<unsigned long long *>(tabbase);
  double2 *pq = tabbase + 1;
  double *pe = reinterpret_cast<double *>(pq + P * M);   // [P M + 4]; row i at pe[emis + i]
  const int fbase = crank * P * M;
  const int fcnt = TDM ? max(0, min(P * M, Nj - fbase)) : 0;
  if (t == 0) {
    for (int i = 0; i < 4; i++) mbar_init(mbar + i, 1);
    if (TDM) mbar_init(pmb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (TDM) {
    for (int i = fcnt + t; i < P * M; i += P) pq[i] = cz();
    for (int i = t; i < P * M + 4; i += P) pe[i] = 0.0;
  }
  for (int i = t; i <= NT; i += P) sbeta[i] = p.beta[i];
  if (!TDM && p.tc_hi) {
    for (int k = 0; k < K; k++)
      for (int sd = 0; sd < 2; sd++) {
        const double2 *kp = G[k].kap[sd];
        for (int i = t; i <= NT; i += P) kapS[(k * 2 + sd) * (NT + 1) + i] = kp ? kp[i] : cz();
      }
  }
  if (p.flux_smem) {
    for (int k = 0; k < K; k++) {
      const double2 *l = G[k].lin, *r = G[k].rin;
      for (int i = t; i < NT; i += P) {
        sflux[(2 * k) * NT + i] = l ? l[i] : cz();
        sflux[(2 * k + 1) * NT + i] = r ? r[i] : cz();
      }
    }
  }
  if (t < 2 * K) sH[t] = cz();
  for (int i = t; i < 128 * K; i += P) hred[i] = cz();

  // Rows beyond N_j (padding) get q = 0: their z, x are 0 and their maps
  // decouple them, so the row loops need no bounds checks.  The end rows of
  // the P1 mass matrix and the interface terms b_n - Q^T(l,r) are folded
  // into the neighbour values u_{-1}, u_{N_j} of the rhs stencil.
  double2 u[K][M], q[M];
  double er[M];
  double er_prev;
  double2 qprev;   // q_{s0-1}, the pivot of the previous thread's last row
  auto load_factor = [&](const double2 *qp, const double *erp) {
#pragma unroll
    for (int i = 0; i < M; i++) {
      const int k = s0 + i;
      q[i] = k < Nj ? __ldg(qp + k) : cz();
      er[i] = k < Nj ? __ldg(erp + k) : 0.0;
    }
    er_prev = (s0 >= 1 && s0 - 1 < Nj) ? __ldg(erp + s0 - 1) : 0.0;
    qprev = (s0 >= 1 && s0 - 1 < Nj) ? __ldg(qp + s0 - 1) : cz();
    double2 Af = make_double2(1.0, 0.0), Ab = make_double2(1.0, 0.0);
#pragma unroll
    for (int i = 0; i < M; i++) {
      Af = cmul(Af, negqe(q[i], i == 0 ? er_prev : er[i == 0 ? 0 : i - 1], eim));
      Ab = cmul(Ab, negqe(q[i], er[i], eim));
    }
    sAf[t] = Af;
    sAb[t] = Ab;
  };
  load_factor(G[0].q, G[0].er);
  // TDM prefetch of step nn (thread 0): pq/pe by bulk copy, the previous CTA's
  // last row (qprev / er_prev of thread 0) by plain loads into registers
  double2 qprev_nx = cz();
  double erprev_nx = 0.0;
  long long tpf = 0;   // trace builds: issue time of the last prefetch (copy latency, slot 28)
  auto prefetch = [&](int nn) {
    if (SWR_MARCH_TRACE && t == 0) tpf = clock64();
    const size_t off = (size_t)(nn - 1) * p.td_stride + fbase;
    // issued by the last warp (warp 0 pushes the scan totals by st.async)
    if (t == P - 32 && fcnt > 0) {
      // er rows are 8 B: start one row early when the source is not 16-B aligned
      const double *es = G[0].er + off;
      const unsigned mis = (unsigned)(((uintptr_t)es >> 3) & 1);
      const unsigned bq = (unsigned)fcnt * 16u, be = ((unsigned)(fcnt + mis) * 8u + 15u) & ~15u;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(pmb, bq + be);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(pq)), "l"(G[0].q + off), "r"(bq), "r"(smem_u32(pmb)) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(smem_u32(pe)), "l"(es - mis), "r"(be), "r"(smem_u32(pmb)) : "memory");
    }
    if (t == 0 && fbase > 0 && fbase - 1 < Nj) {
      qprev_nx = __ldg(G[0].q + off - 1);
      erprev_nx = __ldg(G[0].er + off - 1);
    }
  };
  auto load_factor_smem = [&](int nn) {
    const double *pes = pe + (((uintptr_t)(G[0].er + (size_t)(nn - 1) * p.td_stride + fbase) >> 3) & 1);
#pragma unroll
    for (int i = 0; i < M; i++) {
      q[i] = pq[t * M + i];
      er[i] = pes[t * M + i];
    }
    if (t > 0) {
      er_prev = pes[t * M - 1];
      qprev = pq[t * M - 1];
    } else {
      er_prev = erprev_nx;
      qprev = qprev_nx;
    }
    double2 Af = make_double2(1.0, 0.0), Ab = make_double2(1.0, 0.0);
#pragma unroll
    for (int i = 0; i < M; i++) {
      Af = cmul(Af, negqe(q[i], i == 0 ? er_prev : er[i == 0 ? 0 : i - 1], eim));
      Ab = cmul(Ab, negqe(q[i], er[i], eim));
    }
    sAf[t] = Af;
    sAb[t] = Ab;
  };
#pragma unroll
  for (int r = 0; r < K; r++) {
    const double2 *u0p = G[r].u0;
#pragma unroll
    for (int i = 0; i < M; i++) {
      const int k = s0 + i;
      u[r][i] = (u0p && k < Nj) ? u0p[k] : cz();
    }
  }
  if constexpr (!TDM) {
    // constant matrix: z_i = zloc_i + Apre_i z_{s0-1} with Apre_i = prod_{k<=i} c_k,
    // x_{s0} = xloc_{s0} + Ab x_{s0+M} + G z_{s0-1}, G = sum_i (prod_{k<i} b_k) Apre_i
    double2 Ap = make_double2(1.0, 0.0), Bp = make_double2(1.0, 0.0), Gt = cz();
#pragma unroll
    for (int i = 0; i < M; i++) {
      Ap = cmul(Ap, negqe(q[i], i == 0 ? er_prev : er[i == 0 ? 0 : i - 1], eim));
      sApre[i * P + t] = Ap;
      Gt = cfma(Bp, Ap, Gt);
      Bp = cmul(Bp, negqe(q[i], er[i], eim));
    }
    sG[t] = Gt;
    scan_tab_init<true>(sAf[t], sf.wA, tabF, t, P, lane, w, nw, CS, crank);
    scan_tab_init<false>(sAb[t], sbk.wA, tabB, t, P, lane, w, nw, CS, crank);
    // scaled coefficients (see ck): q <- i kappa q, er <- er / kappa
#pragma unroll
    for (int i = 0; i < M; i++) {
      q[i] = cimul(kappa, q[i]);
      er[i] *= ikappa;
    }
    qprev = cimul(kappa, qprev);
    er_prev *= ikappa;
  }
  const double eimk = eim * ikappa;
  // odd part of order-4 operators: B_n = sum_{s<n} rho^{n-s} v'_s (owner registers)
  double2 Bodd[K][2];
#pragma unroll
  for (int r = 0; r < K; r++) Bodd[r][0] = Bodd[r][1] = cz();
  if (first) {
#pragma unroll
    for (int r = 0; r < K; r++) {
      hva[r * (NT + 1)] = (!TDM && p.tc_hi) ? cmul(G[r].f0[0], u[r][0]) : u[r][0];   // v'_0
      if (!TDM && p.tc_hi) Bodd[r][0] = cmul(G[r].rho[0], hva[r * (NT + 1)]);
    }
  }
  if (last) {
#pragma unroll
    for (int i = 0; i < M; i++)
      if (i == ib) {
#pragma unroll
        for (int r = 0; r < K; r++) {
          hvb[r * (NT + 1)] = (!TDM && p.tc_hi) ? cmul(G[r].f0[1], u[r][i]) : u[r][i];
          if (!TDM && p.tc_hi) Bodd[r][1] = cmul(G[r].rho[1], hvb[r * (NT + 1)]);
        }
      }
  }
  // halo of u_0; later steps get their neighbour values without a barrier
  // (end of the step loop)
#pragma unroll
  for (int r = 0; r < K; r++) {
    hfirst[r * P + t] = u[r][0];
    hlast[r * P + t] = u[r][M - 1];
  }
  csync(CS, true);
  if (TDM && NT >= 2) prefetch(2);
  double2 uL[K], uR[K];
#pragma unroll
  for (int r = 0; r < K; r++) {
    uL[r] = cz();
    uR[r] = cz();
    if (t > 0) uL[r] = hlast[r * P + t - 1];
    else if (crank > 0) uL[r] = *remote(hlast + r * P + (P - 1), crank - 1);
    if (t < P - 1) uR[r] = hfirst[r * P + t + 1];
    else if (crank < CS - 1) uR[r] = *remote(hfirst + r * P, crank + 1);
  }

  auto flux = [&](int r, int side, int n) -> double2 {   // incoming l (side 0) / r (side 1) at step n
    if (imp[r][side]) return make_double2(n == 1 ? 1.0 : 0.0, 0.0);
    return p.flux_smem ? sflux[(2 * r + side) * NT + n - 1] : cz();
  };

  if constexpr (TDM) {
#pragma unroll 1
  for (int n = 1; n <= NT; n++) {
    race_jitter(0, n);
    SWR_TRACE(0);
    if (TDM && n > 1) {   // time-dependent potential: the step-n factorisation of (A_{j,n} - B)
      if (fcnt > 0) mbar_wait(pmb, (uint32_t)((n - 2) & 1));
      if (SWR_TRACE_ON) p.trace[blockIdx.x * 32 + 28] = p.trace[blockIdx.x * 32] + (clock64() - tpf);
      load_factor_smem(n);
      __syncthreads();                 // every thread holds its rows: the buffer is free
      if (n < NT) prefetch(n + 1);
    }
    // ---- S0^2 history H_n = c2 (beta_1 v_{n-1} + P_n),
    // P_n = sum_{s<=n-2} beta_{n-s} v_s spread over the CTA during step n-1
    // (hred); the owner of the boundary row adds the newest term below.
    SWR_TRACE(1);
    SWR_TRACE(2);
    // ---- end rows and interface terms folded into u_{-1} and u_{N_j} ----
    // (uL of the first thread and uR / the row after N_j - 1 of the last
    // thread are rebuilt here every step)
    if (first || last) {
#pragma unroll
      for (int r = 0; r < K; r++) {
        if (first) {
          double2 d = cz();
          if (owns_a) {
            double2 h = cz();
            if (p.s02) {
              h = cscale(sbeta[1], hva[r * (NT + 1) + n - 1]);
              for (int qq = 0; qq < nw; qq++) h = cadd(h, hred[r * 64 + qq]);
              h = cmul(p.c2, h);
            }
            sH[2 * r] = h;
            d = csub(h, flux(r, 0, n));                 // b_n - l_n at row 0
          }
          const double2 f = ifold(d, ikappa);
          uL[r] = make_double2(fma(-2.0, u[r][0].x, f.x), fma(-2.0, u[r][0].y, f.y));
        }
        if (last) {
          double2 d = cz();
          if (owns_b) {
            double2 h = cz();
            if (p.s02) {
              h = cscale(sbeta[1], hvb[r * (NT + 1) + n - 1]);
              for (int qq = 0; qq < nw; qq++) h = cadd(h, hred[r * 64 + 32 + qq]);
              h = cmul(p.c2, h);
            }
            sH[2 * r + 1] = h;
            d = csub(h, flux(r, 1, n));                 // b_n - r_n at row N_j - 1
          }
          const double2 f = ifold(d, ikappa);
#pragma unroll
          for (int i = 0; i < M; i++)
            if (i == ib) {
              const double2 un = make_double2(fma(-2.0, u[r][i].x, f.x), fma(-2.0, u[r][i].y, f.y));
              if (i == M - 1) uR[r] = un;
              else u[r][i == M - 1 ? M - 1 : i + 1] = un;   // the (padding) row after N_j - 1
            }
        }
      }
    }

    // ---- forward sweep z_k = q_k r_k + c_k z_{k-1}: aggregate, scan, exact ----
    double2 z[K], zc[K];   // zc: the forward carry z_{s0-1}
    const int pb = (n - 1) & 1;                 // scan buffers / mbarriers of this step
    const uint32_t ph = ((n - 1) >> 1) & 1;     // their phase parity
    ScanBuf<K> sfp = sf, sbp = sbk;
    sfp.ctot += pb * 16 * (1 + K);
    sbp.ctot += pb * 16 * (1 + K);
#pragma unroll
    for (int r = 0; r < K; r++) z[r] = cz();
    // local forward pass from carry 0 (z^loc stored), the scan for the carry
    // z_{s0-1}, then z_i = z^loc_i + (prod_{k<=i} c_k) z_{s0-1} by a fix-up pass
    // (the rhs is built once per step)
    launder<M>(q, er);
#pragma unroll
    for (int i = 0; i < M; i++) {
      const double2 c = negqe(q[i], i == 0 ? er_prev : er[i == 0 ? 0 : i - 1], eim);
#pragma unroll
      for (int r = 0; r < K; r++) {
        const double2 rr = rhs_row<false>(0, Nj, i == 0 ? uL[r] : u[r][i == 0 ? 0 : i - 1], u[r][i],
                                          i == M - 1 ? uR[r] : u[r][i == M - 1 ? M - 1 : i + 1], kappa);
        z[r] = cfma(c, z[r], cmul(q[i], rr));
        ybuf[(r * M + i) * P + t] = z[r];
      }
    }
    {
      double2 carry[K];
      SWR_TRACE(3);
      race_jitter(1, n);
      scan_maps<K, true>(sAf[t], z, sfp, lane, w, nw, CS, crank, carry,
                               SWR_TRACE_ON ? p.trace + blockIdx.x * 32 + 10 : nullptr, mbar + pb, ph);
      SWR_TRACE(4);
#pragma unroll
      for (int r = 0; r < K; r++) zc[r] = carry[r];
    }
    {
      double2 a[K];
#pragma unroll
      for (int r = 0; r < K; r++) a[r] = zc[r];
      launder<M>(q, er);
#pragma unroll
      for (int i = 0; i < M; i++) {
        const double2 c = negqe(q[i], i == 0 ? er_prev : er[i == 0 ? 0 : i - 1], eim);
#pragma unroll
        for (int r = 0; r < K; r++) {
          a[r] = cmul(c, a[r]);
          ybuf[(r * M + i) * P + t] = cadd(ybuf[(r * M + i) * P + t], a[r]);
        }
      }
    }
    SWR_TRACE(5);
    // partial history sums of step n+1: P_{n+1} = sum_{s<=n-1} beta_{n+1-s} v_s
    if (p.s02 && n < NT) {
      if (has_left && crank == 0) {
#pragma unroll
        for (int r = 0; r < K; r++) {
          double2 acc = cz();
          const double2 *hv = hva + r * (NT + 1);
          for (int s = t; s <= n - 1; s += P) {
            const double b = sbeta[n + 1 - s];
            acc.x = fma(b, hv[s].x, acc.x);
            acc.y = fma(b, hv[s].y, acc.y);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
          if (lane == 0) hred[r * 64 + w] = acc;
        }
      }
      if (has_right && crank == cb) {
#pragma unroll
        for (int r = 0; r < K; r++) {
          double2 acc = cz();
          const double2 *hv = hvb + r * (NT + 1);
          for (int s = t; s <= n - 1; s += P) {
            const double b = sbeta[n + 1 - s];
            acc.x = fma(b, hv[s].x, acc.x);
            acc.y = fma(b, hv[s].y, acc.y);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
          if (lane == 0) hred[r * 64 + 32 + w] = acc;
        }
      }
    }
    // ---- backward sweep x_k = z_k + b_k x_{k+1}: aggregate, scan, exact ----
    double2 x[K];
#pragma unroll
    for (int r = 0; r < K; r++) x[r] = cz();
    launder<M>(q, er);
#pragma unroll
    for (int i = M - 1; i >= 0; i--) {
      const double2 b = negqe(q[i], er[i], eim);
#pragma unroll
      for (int r = 0; r < K; r++) x[r] = cfma(b, x[r], ybuf[(r * M + i) * P + t]);
    }
    {
      double2 carry[K];
      SWR_TRACE(6);
      race_jitter(2, n);
      scan_maps<K, false>(sAb[t], x, sbp, lane, w, nw, CS, crank, carry,
                                SWR_TRACE_ON ? p.trace + blockIdx.x * 32 + 20 : nullptr, mbar + 2 + pb, ph);
      SWR_TRACE(7);
#pragma unroll
      for (int r = 0; r < K; r++) {
        x[r] = carry[r];
        // u_n at row s+M (the next thread's first row) from the carry x_{s+M}
        uR[r] = make_double2(fma(2.0, carry[r].x, -uR[r].x), fma(2.0, carry[r].y, -uR[r].y));
      }
    }
    launder<M>(q, er);
    double2 xb[K];
#pragma unroll
    for (int r = 0; r < K; r++) xb[r] = cz();
#pragma unroll
    for (int i = M - 1; i >= 0; i--) {
      const double2 b = negqe(q[i], er[i], eim);
#pragma unroll
      for (int r = 0; r < K; r++) {
        x[r] = cfma(b, x[r], ybuf[(r * M + i) * P + t]);
        if (i == ib) xb[r] = x[r];
        u[r][i] = make_double2(fma(2.0, x[r].x, -u[r][i].x), fma(2.0, x[r].y, -u[r][i].y));  // u_n = 2 v_n - u_{n-1}
      }
    }
    // u_n at row s-1 (the previous thread's last row): x_{s-1} = z_{s-1} + b_{s-1} x_s
    // with z_{s-1} the forward carry and b_{s-1} = -q_{s-1} E_{s-1}
    if (s0 > 0) {
      const double2 bp = negqe(qprev, er_prev, eim);
#pragma unroll
      for (int r = 0; r < K; r++) {
        const double2 xp = cfma(bp, x[r], zc[r]);
        uL[r] = make_double2(fma(2.0, xp.x, -uL[r].x), fma(2.0, xp.y, -uL[r].y));
      }
    }
    race_jitter(3, n);
    SWR_TRACE(8);
    // ---- record v_n and S v_n at the interfaces (eq. 8) ----
    if (first) {   // x now holds v_n at row 0
#pragma unroll
      for (int r = 0; r < K; r++) {
        hva[r * (NT + 1) + n] = x[r];
        double2 *outl = G[r].out_left;
        if (owns_a && outl) {
          const double2 sv = cfma(p.c0, x[r], sH[2 * r]);   // S v_n(a_j) = c0 v_n + H_a
          const double2 l = flux(r, 0, n);
          outl[n - 1] = make_double2(fma(2.0, sv.x, -l.x), fma(2.0, sv.y, -l.y));
        }
      }
    }
    if (last) {
#pragma unroll
      for (int r = 0; r < K; r++) {
        hvb[r * (NT + 1) + n] = xb[r];
        double2 *outr = G[r].out_right;
        if (owns_b && outr) {
          const double2 sv = cfma(p.c0, xb[r], sH[2 * r + 1]);
          const double2 rv = flux(r, 1, n);
          outr[n - 1] = make_double2(fma(2.0, sv.x, -rv.x), fma(2.0, sv.y, -rv.y));
        }
      }
    }
    SWR_TRACE(9);
  }
  } else {
#pragma unroll 1
  for (int n = 1; n <= NT; n++) {
    race_jitter(0, n);
    SWR_TRACE(0);
    // ---- S0^2 history H_n = c2 (beta_1 v_{n-1} + beta_2 v_{n-2} + Q_n) (P:218,
    // P:501-507), Q_n = sum_{s<=n-3} beta_{n-s} v_s summed over the CTA during
    // step n-2 (hred); the owner of the boundary row adds the two newest terms.
    SWR_TRACE(1);
    SWR_TRACE(2);
    // ---- end rows and interface terms folded into u_{-1} and u_{N_j} ----
    // (uL of the first thread and uR / the row after N_j - 1 of the last
    // thread are rebuilt here every step)
    if (first || last) {
#pragma unroll
      for (int r = 0; r < K; r++) {
        if (first) {
          double2 d = cz();
          if (owns_a) {
            double2 h = cz();
            if (p.tc_hi) {
              // even history (emitted) + odd part (local condition only), A25
              const double2 *hv = hva + r * (NT + 1), *hq = hred + ((r * 2 + (n & 1)) * 2 + 0) * 32;
              const double2 *kp = kapS + (r * 2 + 0) * (NT + 1);
              h = cmul(kp[1], hv[n - 1]);
              if (n >= 2) h = cfma(kp[2], hv[n - 2], h);
              for (int qq = 0; qq < nw; qq++) h = cadd(h, hq[qq]);
              sH[2 * r] = h;
              d = csub(cfma(cscale(2.0, G[r].dlt[0]), Bodd[r][0], h), flux(r, 0, n));
            } else {
            if (p.s02) {
              const double2 *hv = hva + r * (NT + 1), *hq = hred + ((r * 2 + (n & 1)) * 2 + 0) * 32;
              h = cscale(sbeta[1], hv[n - 1]);
              if (n >= 2) h = cadd(h, cscale(sbeta[2], hv[n - 2]));
              for (int qq = 0; qq < nw; qq++) h = cadd(h, hq[qq]);
              h = cmul(p.c2, h);
            }
            sH[2 * r] = h;
            d = csub(h, flux(r, 0, n));                 // b_n - l_n at row 0
            }
          }
          const double2 f = ifold(d, ikappa);
          uL[r] = make_double2(fma(-2.0, u[r][0].x, f.x), fma(-2.0, u[r][0].y, f.y));
        }
        if (last) {
          double2 d = cz();
          if (owns_b) {
            double2 h = cz();
            if (p.tc_hi) {
              const double2 *hv = hvb + r * (NT + 1), *hq = hred + ((r * 2 + (n & 1)) * 2 + 1) * 32;
              const double2 *kp = kapS + (r * 2 + 1) * (NT + 1);
              h = cmul(kp[1], hv[n - 1]);
              if (n >= 2) h = cfma(kp[2], hv[n - 2], h);
              for (int qq = 0; qq < nw; qq++) h = cadd(h, hq[qq]);
              sH[2 * r + 1] = h;
              d = csub(cfma(cscale(2.0, G[r].dlt[1]), Bodd[r][1], h), flux(r, 1, n));
            } else {
            if (p.s02) {
              const double2 *hv = hvb + r * (NT + 1), *hq = hred + ((r * 2 + (n & 1)) * 2 + 1) * 32;
              h = cscale(sbeta[1], hv[n - 1]);
              if (n >= 2) h = cadd(h, cscale(sbeta[2], hv[n - 2]));
              for (int qq = 0; qq < nw; qq++) h = cadd(h, hq[qq]);
              h = cmul(p.c2, h);
            }
            sH[2 * r + 1] = h;
            d = csub(h, flux(r, 1, n));                 // b_n - r_n at row N_j - 1
            }
          }
          const double2 f = ifold(d, ikappa);
#pragma unroll
          for (int i = 0; i < M; i++)
            if (i == ib) {
              const double2 un = make_double2(fma(-2.0, u[r][i].x, f.x), fma(-2.0, u[r][i].y, f.y));
              if (i == M - 1) uR[r] = un;
              else u[r][i == M - 1 ? M - 1 : i + 1] = un;   // the (padding) row after N_j - 1
            }
        }
      }
    }

    // ---- constant matrix: local forward and backward passes (carries 0), one
    // scan per direction on the offsets, one exact backward pass ----
    double2 z[K], zc[K], x[K];
    const int pb = (n - 1) & 1;                 // scan buffers / mbarriers of this step
    const uint32_t ph = ((n - 1) >> 1) & 1;     // their phase parity
    ScanBuf<K> sfp = sf, sbp = sbk;
    sfp.ctot += pb * 16 * (1 + K);
    sbp.ctot += pb * 16 * (1 + K);
#pragma unroll
    for (int r = 0; r < K; r++) z[r] = x[r] = cz();
    launder<M>(q, er);
#pragma unroll
    for (int i = 0; i < M; i++) {
      const double2 c = ck(q[i], i == 0 ? er_prev : er[i == 0 ? 0 : i - 1], eimk);
#pragma unroll
      for (int r = 0; r < K; r++) {
        const double2 sr = srow(i == 0 ? uL[r] : u[r][i == 0 ? 0 : i - 1], u[r][i],
                                i == M - 1 ? uR[r] : u[r][i == M - 1 ? M - 1 : i + 1]);
        z[r] = cfma(c, z[r], cmul(q[i], sr));
        ybuf[(r * M + i) * P + t] = z[r];
      }
    }
    launder<M>(q, er);
#pragma unroll
    for (int i = M - 1; i >= 0; i--) {
      const double2 b = ck(q[i], er[i], eimk);
#pragma unroll
      for (int r = 0; r < K; r++) x[r] = cfma(b, x[r], ybuf[(r * M + i) * P + t]);
    }
    SWR_TRACE(3);
    // Q_{n+2} = sum_{s<=n-1} beta_{n+2-s} v_s of one side (v_{n-1} is visible
    // after the forward-scan barrier), reduced per warp into hred; run by the
    // CTA holding that side inside the backward scan (below)
    auto history = [&](int side) {
      if (!((p.s02 || p.tc_hi) && n + 2 <= NT)) return;
#pragma unroll
      for (int r = 0; r < K; r++) {
        double2 acc = cz();
        const double2 *hv = (side ? hvb : hva) + r * (NT + 1);
        if (p.tc_hi) {
          const double2 *kp = kapS + (r * 2 + side) * (NT + 1);
          for (int s = t; s <= n - 1; s += P) acc = cfma(kp[n + 2 - s], hv[s], acc);
        } else
        for (int s = t; s <= n - 1; s += P) {
          const double b = sbeta[n + 2 - s];
          acc.x = fma(b, hv[s].x, acc.x);
          acc.y = fma(b, hv[s].y, acc.y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
        if (lane == 0) hred[((r * 2 + (n & 1)) * 2 + side) * 32 + w] = acc;
      }
    };
    race_jitter(1, n);
    scan_tab<K, true>(z, sfp, tabF, t, P, lane, w, nw, CS, crank, zc, mbar + pb, ph,
                      [&] {},
                      SWR_TRACE_ON ? p.trace + blockIdx.x * 32 + 10 : nullptr);
    SWR_TRACE(4);
    SWR_TRACE(5);
    {
      const double2 Gt = sG[t];
#pragma unroll
      for (int r = 0; r < K; r++) x[r] = cfma(Gt, zc[r], x[r]);
    }
    {
      double2 carry[K];
      SWR_TRACE(6);
      race_jitter(2, n);
      scan_tab<K, false>(x, sbp, tabB, t, P, lane, w, nw, CS, crank, carry, mbar + 2 + pb, ph,
                         [&] {
                           // both history sums in the backward scan: the left one where CTA 0
                           // waits for the later CTAs' totals, the right one after the
                           // boundary CTA's pushes (its next forward fold has slack; in the
                           // forward scan it sat on the critical path)
                           if (has_left && crank == 0) history(0);
                           if (has_right && crank == cb) history(1);
                         },
                         SWR_TRACE_ON ? p.trace + blockIdx.x * 32 + 20 : nullptr);
      SWR_TRACE(7);
#pragma unroll
      for (int r = 0; r < K; r++) {
        x[r] = carry[r];
        // u_n at row s+M (the next thread's first row) from the carry x_{s+M}
        uR[r] = make_double2(fma(2.0, carry[r].x, -uR[r].x), fma(2.0, carry[r].y, -uR[r].y));
      }
    }
    launder<M>(q, er);
    double2 xb[K];
#pragma unroll
    for (int r = 0; r < K; r++) xb[r] = cz();
#pragma unroll
    for (int i = M - 1; i >= 0; i--) {
      const double2 b = ck(q[i], er[i], eimk);
      const double2 Ap = sApre[i * P + t];
#pragma unroll
      for (int r = 0; r < K; r++) {
        const double2 zi = cfma(Ap, zc[r], ybuf[(r * M + i) * P + t]);
        x[r] = cfma(b, x[r], zi);
        if (i == ib) xb[r] = x[r];
        u[r][i] = make_double2(fma(2.0, x[r].x, -u[r][i].x), fma(2.0, x[r].y, -u[r][i].y));  // u_n = 2 v_n - u_{n-1}
      }
    }
    // u_n at row s-1 (the previous thread's last row): x_{s-1} = z_{s-1} + b_{s-1} x_s
    // with z_{s-1} the forward carry and b_{s-1} = -q_{s-1} E_{s-1}
    if (s0 > 0) {
      const double2 bp = ck(qprev, er_prev, eimk);
#pragma unroll
      for (int r = 0; r < K; r++) {
        const double2 xp = cfma(bp, x[r], zc[r]);
        uL[r] = make_double2(fma(2.0, xp.x, -uL[r].x), fma(2.0, xp.y, -uL[r].y));
      }
    }
    race_jitter(3, n);
    SWR_TRACE(8);
    // ---- record v_n and S v_n at the interfaces (eq. 8) ----
    if (first) {   // x now holds v_n at row 0
#pragma unroll
      for (int r = 0; r < K; r++) {
        hva[r * (NT + 1) + n] = x[r];
        if (p.tc_hi) Bodd[r][0] = cmul(G[r].rho[0], cadd(Bodd[r][0], x[r]));
        double2 *outl = G[r].out_left;
        if (owns_a && outl) {
          const double2 sv = cfma(p.tc_hi ? G[r].c0e[0] : p.c0, x[r], sH[2 * r]);   // S v_n(a_j) = c0 v_n + H_a
          const double2 l = flux(r, 0, n);
          outl[n - 1] = make_double2(fma(2.0, sv.x, -l.x), fma(2.0, sv.y, -l.y));
        }
      }
    }
    if (last) {
#pragma unroll
      for (int r = 0; r < K; r++) {
        hvb[r * (NT + 1) + n] = xb[r];
        if (p.tc_hi) Bodd[r][1] = cmul(G[r].rho[1], cadd(Bodd[r][1], xb[r]));
        double2 *outr = G[r].out_right;
        if (owns_b && outr) {
          const double2 sv = cfma(p.tc_hi ? G[r].c0e[1] : p.c0, xb[r], sH[2 * r + 1]);
          const double2 rv = flux(r, 1, n);
          outr[n - 1] = make_double2(fma(2.0, sv.x, -rv.x), fma(2.0, sv.y, -rv.y));
        }
      }
    }
    SWR_TRACE(9);
  }
  }
#pragma unroll
  for (int r = 0; r < K; r++) {
    double2 *uTp = G[r].uT;
    if (uTp) {
#pragma unroll
      for (int i = 0; i < M; i++)
        if (s0 + i < Nj) uTp[s0 + i] = u[r][i];
    }
  }
  if (CS > 1) cg::this_cluster().sync();  // keep shared memory alive for remote readers
}

// ---------------------------------------------------------------------------
// Nonlinear march, f(u) = lambda |u|^2 (Duran-Sanz-Serna midpoint),
// one RHS per group.  Per step the inner fixed point of eq. (12):
//   (A_NL - B) z^{s+1} = (2i/dt) M u_{n-1} - M_{f(z^s)} z^s + b_n - Q^T(l_n, r_n)^T
// from z^0 = v_{n-1}, with the load M_{f(z)} z the weighted mass matrix of the
// nodal values f(z_k) (reading A3), stopped when
// max_k |z^{s+1} - z^s| <= tol_fp max_k |z^{s+1}| (reading A4; the maxima are
// reduced over the cluster so the decision is uniform).  (A_NL - B) is the
// V = 0 matrix: constant pivots, Re E_k = 1/h.
//
// Per fixed-point iteration: (1) a local forward pass from carry 0 builds the
// rhs (stencil of u_{n-1} and the load of z^s) once and stores z^loc; (2) the
// forward scan of the thread maps gives the carry z_{s0-1}; (3) a cheap pass
// adds the carry's propagation (prefix products of c_k) to z^loc; (4) a local
// backward pass, (5) the backward scan, (6) the exact backward pass, which
// also yields the maxima.  The neighbour rows of the next iterate and of u_n
// come from the scan carries (x_{s0+M} is the backward carry, x_{s0-1} =
// z_{s0-1} + b_{s0-1} x_{s0}), so no halo exchange is needed; the scan totals
// and the CTA maxima travel between the CTAs of the cluster by st.async into
// parity buffers counted by mbarriers.  The thread's rows keep u_{n-1} and z^s
// in registers; the (scaled) pivots and Re E_k sit in shared memory, so a CTA
// holds more rows per register budget and more systems are resident at once
// (C4: the 100 systems in one wave).  The boundary-value histories and the
// flux series are read from global memory by the threads that own them.
// ---------------------------------------------------------------------------
template <int M, int PMAX, int MINB = 1>
__global__ void __launch_bounds__(PMAX, MINB) k_march_nl(const MarchParams p) {
  extern __shared__ double2 sm[];
  const int P = blockDim.x, t = threadIdx.x, lane = t & 31, w = t >> 5, nw = P >> 5;
  const int CS = p.CS;
  const int crank = blockIdx.x % CS;
  const int sysi = blockIdx.x / CS;
  const MarchSys *G = p.sys + sysi;
  const int Nj = p.Nj, NT = p.NT;
  const int s0 = (crank * P + t) * M;
  const double eim = p.e_im, kappa = p.kappa, ikappa = 1.0 / p.kappa;
  const double eimk = eim * ikappa, hk = p.h12 * ikappa, lam = p.lambda;

  // ---- shared memory ----
  unsigned long long *mbar = reinterpret_cast<unsigned long long *>(sm);   // [fwd 2][bwd 2][max 2]
  double2 *ybuf = sm + 4;                               // [max(M,2)][P] z^loc, then z (first: the u_0 halo)
  double2 *sq = ybuf + (M < 2 ? 2 : M) * P;             // [M][P] scaled pivots i kappa q_k
  double *ser = reinterpret_cast<double *>(sq + M * P); // [M][P] scaled Re E_k / kappa
  double2 *sAf = reinterpret_cast<double2 *>(ser + M * P);   // [P]
  double2 *sAb = sAf + P;                               // [P]
  ScanBuf<1> sf, sbk;                                   // ctot: [2 parities][16][2]
  sf.wA = sAb + P;             sf.wB = sf.wA + 32;      sf.ctot = sf.wB + 32;
  sbk.wA = sf.ctot + 64;       sbk.wB = sbk.wA + 32;    sbk.ctot = sbk.wB + 32;
  double2 *cmax = sbk.ctot + 64;                        // [2 parities][16] CTA maxima (x: |dz|^2, y: |z|^2)
  double2 *wmax = cmax + 32;                            // [32] warp maxima
  double2 *hred = wmax + 32;                            // [2 sides][32] warp partials of the history
  double2 *sH = hred + 64;                              // [2] H_a, H_b of the step
  double2 *hva = p.hv_glob + (size_t)sysi * 2 * (NT + 1), *hvb = hva + (NT + 1);   // v_s(a_j), v_s(b_j)

  const int flags = G->flags;
  const bool has_left = flags & SYS_HAS_LEFT, has_right = flags & SYS_HAS_RIGHT;
  const int rows_cta = P * M;
  const int cb = (Nj - 1) / rows_cta, tb = ((Nj - 1) % rows_cta) / M;
  const bool first = s0 == 0;                           // holds row 0
  const bool last = crank == cb && t == tb;             // holds row N_j - 1
  const int ib = (Nj - 1) - s0;                         // its index in the thread (if last)
  const bool owns_a = has_left && first, owns_b = has_right && last;
  if (t == 0) {
    for (int i = 0; i < 6; i++) mbar_init(mbar + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (t < 2) sH[t] = cz();

  // coefficients (rows beyond N_j: q = 0, which decouples them) and the
  // per-thread linear parts of the forward / backward maps
  double2 u[M], ze[M];
  double2 qprev = cz();
  double er_prev = 0.0;
  {
    double2 Af = make_double2(1.0, 0.0), Ab = make_double2(1.0, 0.0);
    er_prev = (s0 >= 1 && s0 - 1 < Nj) ? G->er[s0 - 1] : 0.0;
    qprev = (s0 >= 1 && s0 - 1 < Nj) ? G->q[s0 - 1] : cz();
    double erl = er_prev;
#pragma unroll
    for (int i = 0; i < M; i++) {
      const int k = s0 + i;
      const double2 qv = k < Nj ? G->q[k] : cz();
      const double ev = k < Nj ? G->er[k] : 0.0;
      Af = cmul(Af, negqe(qv, erl, eim));
      Ab = cmul(Ab, negqe(qv, ev, eim));
      sq[i * P + t] = cimul(kappa, qv);
      ser[i * P + t] = ev * ikappa;
      erl = ev;
      u[i] = (G->u0 && k < Nj) ? G->u0[k] : cz();
      ze[i] = u[i];                                     // z^0 of step 1 = v_0 = u_0
    }
    sAf[t] = Af;
    sAb[t] = Ab;
    qprev = cimul(kappa, qprev);
    er_prev *= ikappa;
  }
  if (first) hva[0] = u[0];
  if (last) {
#pragma unroll
    for (int i = 0; i < M; i++)
      if (i == ib) hvb[0] = u[i];
  }
  // halo of u_0 and z^0 (later neighbour values come from the scan carries)
  double2 *hfirst = ybuf, *hlast = ybuf + P;             // ybuf is free before the first pass
  hfirst[t] = u[0];
  hlast[t] = u[M - 1];
  csync(CS, true);
  double2 uL = cz(), uR = cz();
  if (t > 0) uL = hlast[t - 1];
  else if (crank > 0) uL = *remote(hlast + (P - 1), crank - 1);
  if (t < P - 1) uR = hfirst[t + 1];
  else if (crank < CS - 1) uR = *remote(hfirst, crank + 1);
  csync(CS);   // every (remote) halo read is done before ybuf is written
  double2 zL = uL, zR = uR;

  auto flux = [&](int side, int n) -> double2 {
    const int imp = side == 0 ? (flags & SYS_LIN_IMPULSE) : (flags & SYS_RIN_IMPULSE);
    if (imp) return make_double2(n == 1 ? 1.0 : 0.0, 0.0);
    const double2 *f = side == 0 ? G->lin : G->rin;
    return f ? f[n - 1] : cz();
  };
  auto Qc = [&](int i) -> double2 { return sq[i * P + t]; };
  auto Ec = [&](int i) -> double { return ser[i * P + t]; };
  int fp_max = 0, fp_fail = 0;
  unsigned sc = 0;   // fixed-point iterations so far: parity buffers and mbarrier phases

#pragma unroll 1
  for (int n = 1; n <= NT; n++) {
    race_jitter(0, n);
    // ---- S0^2 history H_n = c2 (beta_1 v_{n-1} + sum_{s<=n-2} beta_{n-s} v_s)
    if (p.s02) {
      if (has_left && crank == 0) {
        double2 acc = cz();
        for (int s = t; s < n - 1; s += P) {
          const double b = __ldg(p.beta + n - s);
          const double2 hv = hva[s];
          acc.x = fma(b, hv.x, acc.x);
          acc.y = fma(b, hv.y, acc.y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
        if (lane == 0) hred[w] = acc;
      }
      if (has_right && crank == cb) {
        double2 acc = cz();
        for (int s = t; s < n - 1; s += P) {
          const double b = __ldg(p.beta + n - s);
          const double2 hv = hvb[s];
          acc.x = fma(b, hv.x, acc.x);
          acc.y = fma(b, hv.y, acc.y);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc = cadd(acc, shfl_xor2(acc, o));
        if (lane == 0) hred[32 + w] = acc;
      }
      __syncthreads();
    }
    // ---- end rows: the P1 mass end rows (h/6)(2, 1) and b_n - l_n / b_n - r_n
    // folded into the stencil neighbours u_{-1} and the row after N_j - 1 ----
    if (first || last) {
      if (first) {
        double2 d = cz();
        if (owns_a) {
          double2 h = cz();
          if (p.s02) {
            h = cscale(__ldg(p.beta + 1), hva[n - 1]);
            for (int qq = 0; qq < nw; qq++) h = cadd(h, hred[qq]);
            h = cmul(p.c2, h);
          }
          sH[0] = h;
          d = csub(h, flux(0, n));
        }
        const double2 f = ifold(d, ikappa);
        uL = make_double2(fma(-2.0, u[0].x, f.x), fma(-2.0, u[0].y, f.y));
      }
      if (last) {
        double2 d = cz();
        if (owns_b) {
          double2 h = cz();
          if (p.s02) {
            h = cscale(__ldg(p.beta + 1), hvb[n - 1]);
            for (int qq = 0; qq < nw; qq++) h = cadd(h, hred[32 + qq]);
            h = cmul(p.c2, h);
          }
          sH[1] = h;
          d = csub(h, flux(1, n));
        }
        const double2 f = ifold(d, ikappa);
#pragma unroll
        for (int i = 0; i < M; i++)
          if (i == ib) {
            const double2 un = make_double2(fma(-2.0, u[i].x, f.x), fma(-2.0, u[i].y, f.y));
            if (i == M - 1) uR = un;
            else u[i == M - 1 ? M - 1 : i + 1] = un;   // the (padding) row after N_j - 1
          }
      }
    }

    int it;
    bool conv = false;
    double2 zc = cz(), xc = cz();
#pragma unroll 1
    for (it = 1; it <= p.maxit_fp; it++, sc++) {
      const int pb = sc & 1;
      const uint32_t ph = (sc >> 1) & 1;
      ScanBuf<1> sfp = sf, sbp = sbk;
      sfp.ctot += pb * 32;
      sbp.ctot += pb * 32;
      // (1) local forward pass: rhs = i kappa (u_{k-1} + 4 u_k + u_{k+1}) - (h/12) load_k(z^s),
      // scaled by 1 / (i kappa) into the stencil (the pivots carry i kappa)
      double2 z = cz();
#pragma unroll
      for (int i = 0; i < M; i++) {
        const double2 c = ck(Qc(i), i == 0 ? er_prev : Ec(i == 0 ? 0 : i - 1), eimk);
        const double2 um = i == 0 ? uL : u[i == 0 ? 0 : i - 1];
        const double2 up = i == M - 1 ? uR : u[i == M - 1 ? M - 1 : i + 1];
        const double2 sr = srow(um, u[i], up);
        // weighted mass load (P1 elements, linear interpolant of W = f(z))
        const double2 zm = i == 0 ? zL : ze[i == 0 ? 0 : i - 1];
        const double2 zp = i == M - 1 ? zR : ze[i == M - 1 ? M - 1 : i + 1];
        const double2 zk = ze[i];
        const double Wc = lam * fma(zk.x, zk.x, zk.y * zk.y);
        const double Wm = lam * fma(zm.x, zm.x, zm.y * zm.y);
        const double Wp = lam * fma(zp.x, zp.x, zp.y * zp.y);
        double2 ld = cz();
        if (!(first && i == 0)) {             // element (k-1, k)
          ld.x = fma(Wm + 3.0 * Wc, zk.x, (Wm + Wc) * zm.x);
          ld.y = fma(Wm + 3.0 * Wc, zk.y, (Wm + Wc) * zm.y);
        }
        if (!(last && i == ib)) {             // element (k, k+1)
          ld.x = fma(3.0 * Wc + Wp, zk.x, fma(Wc + Wp, zp.x, ld.x));
          ld.y = fma(3.0 * Wc + Wp, zk.y, fma(Wc + Wp, zp.y, ld.y));
        }
        // sr - (h/12) ld / (i kappa) = sr + i (h / (12 kappa)) ld
        const double2 rr = make_double2(fma(-hk, ld.y, sr.x), fma(hk, ld.x, sr.y));
        z = cfma(c, z, cmul(Qc(i), rr));
        ybuf[i * P + t] = z;
      }
      // (2) forward scan: carry z_{s0-1}
      {
        double2 zz[1] = {z}, carry[1];
        race_jitter(1, n);
        scan_maps<1, true>(sAf[t], zz, sfp, lane, w, nw, CS, crank, carry, nullptr, mbar + pb, ph);
        zc = carry[0];
      }
      // (3) z_i = z^loc_i + (prod_{k<=i} c_k) z_{s0-1}; (4) local backward pass
      double2 a = zc, x = cz();
#pragma unroll
      for (int i = 0; i < M; i++) {
        const double2 c = ck(Qc(i), i == 0 ? er_prev : Ec(i == 0 ? 0 : i - 1), eimk);
        a = cmul(c, a);
        ybuf[i * P + t] = cadd(ybuf[i * P + t], a);
      }
#pragma unroll
      for (int i = M - 1; i >= 0; i--) x = cfma(ck(Qc(i), Ec(i), eimk), x, ybuf[i * P + t]);
      // (5) backward scan: carry x_{s0+M}
      {
        double2 xx[1] = {x}, carry[1];
        race_jitter(2, n);
        scan_maps<1, false>(sAb[t], xx, sbp, lane, w, nw, CS, crank, carry, nullptr, mbar + 2 + pb, ph);
        xc = carry[0];
      }
      // (6) exact backward pass: z^{s+1} and the maxima
      x = xc;
      double dmax = 0.0, nmax = 0.0;
#pragma unroll
      for (int i = M - 1; i >= 0; i--) {
        x = cfma(ck(Qc(i), Ec(i), eimk), x, ybuf[i * P + t]);
        const double dx = x.x - ze[i].x, dy = x.y - ze[i].y;
        dmax = fmax(dmax, fma(dx, dx, dy * dy));
        nmax = fmax(nmax, fma(x.x, x.x, x.y * x.y));
        ze[i] = x;
      }
      // neighbour rows of z^{s+1}: x_{s0+M} (carry), x_{s0-1} = z_{s0-1} + b_{s0-1} x_{s0}
      zR = xc;
      zL = s0 > 0 ? cfma(ck(qprev, er_prev, eimk), ze[0], zc) : cz();
      // cluster-wide maxima -> uniform convergence decision
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
        nmax = fmax(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
      }
      if (lane == 0) wmax[w] = make_double2(dmax, nmax);
      __syncthreads();
      double2 mm = make_double2(0.0, 0.0);
      for (int q = 0; q < nw; q++) {
        const double2 v = wmax[q];
        mm.x = fmax(mm.x, v.x);
        mm.y = fmax(mm.y, v.y);
      }
      if (CS > 1) {
        double2 *cm = cmax + pb * 16;
        if (t == 0) {
          const uint32_t src = smem_u32(cm + crank), lmb = smem_u32(mbar + 4 + pb);
#pragma unroll 1
          for (int c = 0; c < CS; c++)
            if (c != crank) st_async(mapa(src, c), mm, mapa(lmb, c));
          mbar_expect_tx(mbar + 4 + pb, (unsigned)((CS - 1) * 16));
        }
        race_jitter(3, n);
        mbar_wait(mbar + 4 + pb, ph);
        for (int c = 0; c < CS; c++) {
          if (c == crank) continue;
          const double2 v = cm[c];
          mm.x = fmax(mm.x, v.x);
          mm.y = fmax(mm.y, v.y);
        }
      }
      if (sqrt(mm.x) <= p.tol_fp * sqrt(mm.y)) { conv = true; sc++; break; }
    }
    if (!conv) { it = p.maxit_fp; fp_fail = 1; }
    if (it > fp_max) fp_max = it;
    // v_n = z; record S v_n at the interfaces; u_n = 2 v_n - u_{n-1}
    if (first) {
      hva[n] = ze[0];
      if (owns_a && G->out_left) {
        const double2 sv = cfma(p.c0, ze[0], sH[0]);
        const double2 l = flux(0, n);
        G->out_left[n - 1] = make_double2(fma(2.0, sv.x, -l.x), fma(2.0, sv.y, -l.y));
      }
    }
    if (last) {
#pragma unroll
      for (int i = 0; i < M; i++)
        if (i == ib) {
          hvb[n] = ze[i];
          if (owns_b && G->out_right) {
            const double2 sv = cfma(p.c0, ze[i], sH[1]);
            const double2 rv = flux(1, n);
            G->out_right[n - 1] = make_double2(fma(2.0, sv.x, -rv.x), fma(2.0, sv.y, -rv.y));
          }
        }
    }
#pragma unroll
    for (int i = 0; i < M; i++) u[i] = make_double2(fma(2.0, ze[i].x, -u[i].x), fma(2.0, ze[i].y, -u[i].y));
    uL = make_double2(fma(2.0, zL.x, -uL.x), fma(2.0, zL.y, -uL.y));
    uR = make_double2(fma(2.0, zR.x, -uR.x), fma(2.0, zR.y, -uR.y));
  }
  if (G->uT) {
#pragma unroll
    for (int i = 0; i < M; i++)
      if (s0 + i < Nj) G->uT[s0 + i] = u[i];
  }
  if (t == 0 && crank == 0 && p.fp_stat) {
    atomicMax(p.fp_stat, fp_max);
    if (fp_fail) atomicOr(p.fp_stat + 1, 1);
  }
  if (CS > 1) cg::this_cluster().sync();  // keep shared memory alive for remote writers
}

// ---------------------------------------------------------------------------
// Launch-shape selection and launcher.  Instantiated (M rows per thread, one
// RHS per group, PMAX threads per CTA); the register cap is 65536 / PMAX.
// (K = 2, 3 right-hand sides per group sharing the registers of a thread
// were measured slower at C5 and are not instantiated.)
// ---------------------------------------------------------------------------
struct Inst { int M, PMAX; };
static const Inst kInst[] = {{1, 512}, {2, 512}, {4, 512}, {6, 256}, {8, 256}, {11, 256}};

MarchShape choose_march_shape(int Nj, int NT, bool tc_hi) {
  MarchShape best{0, 0, 0, 0};
  double best_cost = 1e300;
  const int K = 1;
  for (int CS = 1; CS <= 16; CS++) {
    for (const Inst &in : kInst) {
      const int M = in.M;
      long per = ((long)Nj + (long)CS * M - 1) / ((long)CS * M);
      int P = (int)((per + 31) / 32 * 32);
      if (P < 32) P = 32;
      if (P > in.PMAX) continue;
      if (march_smem_bytes({M, P, CS, K}, NT, true, tc_hi) > 227 * 1024) continue;
      double padded = (double)CS * P * M;
      double cost = padded * (1.0 + 0.10 * (CS - 1)) * (P < 128 ? 1.3 : 1.0);
      if (cost < best_cost) { best_cost = cost; best = {M, P, CS, K}; }
    }
  }
  return best;
}

// Nonlinear march instantiations: M rows per thread, PMAX threads, MINB CTAs
// per SM (register cap 65536 / (PMAX MINB)).  The shape minimises
// waves x (M + 14) x (1 + 0.1 (CS - 1)): a wave is the systems whose clusters
// are resident at once (148 SMs x CTAs per SM / CS); the rows per thread set
// the length of every pass, the scans cost about 14 rows' worth.  rows: 0 = automatic, else forces M
// (tests of the large-subdomain shapes on small problems;
// swr_config.nl_rows_per_thread).
struct InstNL { int M, PMAX, MINB; };
static const InstNL kInstNL[] = {{1, 512, 1}, {2, 512, 1}, {4, 256, 2}, {8, 192, 2}, {11, 192, 2}, {11, 128, 3},
                                 {11, 256, 1}, {16, 256, 1}};

size_t march_nl_smem_bytes(const MarchShape &s, int NT, bool flux_smem) {
  (void)NT;
  (void)flux_smem;
  const size_t MP = (size_t)s.M * s.P;
  const size_t d2 = 4 + (size_t)(s.M < 2 ? 2 : s.M) * s.P + MP + 2 * (size_t)s.P + 2 * (32 + 32 + 64) + 32 + 32 +
                    64 + 2;
  return d2 * sizeof(double2) + MP * sizeof(double);
}

MarchShape choose_march_shape_nl(int Nj, int rows, int nsys) {
  MarchShape best{0, 0, 0, 1};
  double best_cost = 1e300;
  for (int CS = 1; CS <= 16; CS++) {
    for (const InstNL &in : kInstNL) {
      if (rows && in.M != rows) continue;
      const int M = in.M;
      long per = ((long)Nj + (long)CS * M - 1) / ((long)CS * M);
      int P = (int)((per + 31) / 32 * 32);
      if (P < 32) P = 32;
      if (P > in.PMAX) continue;
      const MarchShape sh{M, P, CS, 1};
      const size_t smem = march_nl_smem_bytes(sh, 0, false);
      if (smem > 227 * 1024) continue;
      int per_sm = std::min(in.MINB, (int)((228 * 1024) / (smem + 1024)));
      per_sm = std::min(per_sm, (int)(65536 / ((size_t)P * (65536 / (in.PMAX * in.MINB)))));
      if (per_sm < 1) continue;
      const int clusters = std::max(1, 148 * per_sm / CS);
      const int waves = (std::max(nsys, 1) + clusters - 1) / clusters;
      // a step costs ~ (M + 14) row-units: the passes scale with M, the scans and
      // cluster exchanges (~14 rows' worth at C5) do not
      const double cost = (double)waves * (M + 14) * (1.0 + 0.10 * (CS - 1)) * (P < 128 ? 1.3 : 1.0);
      if (cost < best_cost) { best_cost = cost; best = sh; }
    }
  }
  return best;
}

template <int M, int PMAX, int MINB = 1>
static cudaError_t launch_nl_m(const MarchParams &p, const MarchShape &s, size_t smem, cudaStream_t st) {
  auto kern = k_march_nl<M, PMAX, MINB>;
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
  if (getenv("SWR_VERBOSE")) {
    int ncl = 0;
    cudaOccupancyMaxActiveClusters(&ncl, (void *)kern, &cfg);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    fprintf(stderr, "k_march_nl M=%d P=%d CS=%d systems=%d regs=%d local=%zu smem=%zu: %d clusters resident\n", M,
            s.P, s.CS, p.nsys, fa.numRegs, fa.localSizeBytes, smem, ncl);
  }
  return cudaLaunchKernelEx(&cfg, kern, p);
}

cudaError_t launch_march_nl(MarchParams p, const MarchShape &s, cudaStream_t st) {
  p.CS = s.CS;
  if (!p.hv_glob) return cudaErrorInvalidValue;
  const size_t smem = march_nl_smem_bytes(s, p.NT, false);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  // the shape came from kInstNL: the same (M, P range) picks the instantiation
  if (s.M == 1) return launch_nl_m<1, 512>(p, s, smem, st);
  if (s.M == 2) return launch_nl_m<2, 512>(p, s, smem, st);
  if (s.M == 4) return launch_nl_m<4, 256, 2>(p, s, smem, st);
  if (s.M == 8) return launch_nl_m<8, 192, 2>(p, s, smem, st);
  if (s.M == 11 && s.P <= 128) return launch_nl_m<11, 128, 3>(p, s, smem, st);
  if (s.M == 11 && s.P <= 192) return launch_nl_m<11, 192, 2>(p, s, smem, st);
  if (s.M == 11) return launch_nl_m<11, 256, 1>(p, s, smem, st);
  if (s.M == 16) return launch_nl_m<16, 256, 1>(p, s, smem, st);
  return cudaErrorInvalidValue;
}

size_t march_smem_bytes(const MarchShape &s, int NT, bool flux_smem, bool tc_hi) {
  const size_t K = s.K;
  size_t d2 = 2 + K * s.M * s.P + 2 * K * s.P + 2 * (size_t)s.P + 2 * (32 + 32 * K + 32 * (1 + K)) +
              2 * K * (NT + 1) + 128 * K + 2 * K + (flux_smem ? 2 * K * NT : 0) +
              2 * (size_t)kScanTabD2(s.P) + (size_t)s.M * s.P + s.P;   // scan tables, Apre, G
  return d2 * sizeof(double2) + sizeof(double) * (size_t)((NT + 2) & ~1) +
         (tc_hi ? (size_t)2 * K * (NT + 1) * sizeof(double2) : 0);
}

template <int M, int K, int PMAX>
static cudaError_t launch_m(const MarchParams &p, const MarchShape &s, size_t smem, cudaStream_t st) {
  auto kern = p.td_stride ? k_march<M, K, PMAX, true> : k_march<M, K, PMAX, false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (s.CS > 8) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((p.nsys / K) * s.CS, 1, 1);
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
  const size_t smem = march_smem_bytes(s, p.NT, p.flux_smem, p.tc_hi != 0);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
#define SWR_CASE(MM, PP) \
  if (s.M == MM && s.P <= PP) return launch_m<MM, 1, PP>(p, s, smem, st);
  SWR_CASE(1, 512) SWR_CASE(2, 512) SWR_CASE(4, 512) SWR_CASE(6, 256) SWR_CASE(8, 256) SWR_CASE(11, 256)
#undef SWR_CASE
  return cudaErrorInvalidValue;
}

}  // namespace swr

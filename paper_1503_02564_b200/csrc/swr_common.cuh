// swr_common.cuh — device helpers and host/device structs of the B200 SWR
// hot path (PAPER.md = Besse & Xing, arXiv:1503.02564; "P:n" = line n).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace swr {

// ---- complex fp64 on double2 (x = re, y = im) ---------------------------
__host__ __device__ __forceinline__ double2 cz() { return make_double2(0.0, 0.0); }
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cscale(double s, double2 a) { return make_double2(s * a.x, s * a.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a*b + c
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// conj(a)*b + c
__device__ __forceinline__ double2 cfmaconj(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(a.y, b.y, c.x)), fma(a.x, b.y, fma(-a.y, b.x, c.y)));
}
__device__ __forceinline__ double2 crcp(double2 a) {
  double d = 1.0 / fma(a.x, a.x, a.y * a.y);
  return make_double2(a.x * d, -a.y * d);
}
// zero (or NaN) pivot test |p| < 1e-300, by the larger component
// instead of hypot (off the recurrence's chain, but hypot's ~30 instructions
// per row made the factorisation 1.4x slower)
__device__ __forceinline__ bool tiny_pivot(double2 p) {
  const double ax = fabs(p.x), ay = fabs(p.y);
  return !(ax >= 1e-300 || ay >= 1e-300) || ax != ax || ay != ay;
}
// i * kappa * a
__device__ __forceinline__ double2 cimul(double kappa, double2 a) { return make_double2(-kappa * a.y, kappa * a.x); }
__device__ __forceinline__ double2 shfl_up2(double2 v, int o) {
  return make_double2(__shfl_up_sync(0xffffffffu, v.x, o), __shfl_up_sync(0xffffffffu, v.y, o));
}
__device__ __forceinline__ double2 shfl_down2(double2 v, int o) {
  return make_double2(__shfl_down_sync(0xffffffffu, v.x, o), __shfl_down_sync(0xffffffffu, v.y, o));
}
// Programmatic dependent launch: a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its
// predecessor drains; pdl_wait() blocks until the predecessor grid has
// completed and its writes are visible (a no-op for ordinary launches), and
// pdl_trigger() lets the successor's CTAs be scheduled early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Race-stress builds (-DSWR_RACE_STRESS=1, tests/test_race_stress.py; the
// compute-sanitizer is closed on this pool): a pseudo-random delay of up to
// ~2 us for a quarter of the (warp, step, site) points of the cluster / chain
// kernels perturbs how their CTAs interleave; every result must stay bitwise
// equal to the normal build, or an ordering between CTAs is missing.
#ifndef SWR_RACE_STRESS
#define SWR_RACE_STRESS 0
#endif
__device__ __forceinline__ void race_jitter(unsigned site, unsigned step) {
#if SWR_RACE_STRESS
  unsigned h = (blockIdx.x * 0x9E3779B1u) ^ ((threadIdx.x >> 5) * 0x85EBCA6Bu) ^ (step * 0xC2B2AE35u) ^
               (site * 0x27D4EB2Fu);
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  if ((h & 3u) == 0u) __nanosleep((h >> 20) & 2047u);
#else
  (void)site;
  (void)step;
#endif
}

__device__ __forceinline__ double2 shfl_xor2(double2 v, int o) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o));
}

// ---- interface-vector layout of one rank -------
// Slots of g: l_j = 2j-3 (j >= 2), r_j = 2j-2 (j <= N-1).  A rank
// owns subdomains [j_lo, j_hi] and their slots [s_lo, s_hi] = [slot_first(j_lo),
// slot_last(j_hi)] (contiguous); its interface vectors hold those slots only
// (slot s at local offset (s - s_lo) N_T).  Every owned slot is an input of an
// owned subdomain; the two outputs of owned subdomains that land in a
// neighbour's slot, r_{j_lo - 1} (= s_lo - 1) and l_{j_hi + 1} (= s_hi + 1), go to
// the halo buffers and cross the rank cut (the "cut traces").
struct SlotMap {
  int32_t N, NT, j_lo, j_hi, s_lo, s_hi;
  double2 *haloL, *haloR;   // [N_T] each, nullptr where there is no neighbour rank
};
__host__ __device__ __forceinline__ int slot_first(int j) { return j >= 2 ? 2 * j - 3 : 0; }
__host__ __device__ __forceinline__ int slot_last(int j, int N) { return j <= N - 1 ? 2 * j - 2 : 2 * N - 3; }
// slot s of the local vector v (nullptr if another rank owns it)
template <typename T>
__host__ __device__ __forceinline__ T *slot_ptr(const SlotMap &m, T *v, int s) {
  return (s >= m.s_lo && s <= m.s_hi) ? v + (size_t)(s - m.s_lo) * m.NT : nullptr;
}
// where output slot o of an owned subdomain goes: the local slot, or the halo
// buffer of the neighbour rank that owns it (remote = true)
__host__ __device__ __forceinline__ double2 *out_ptr(const SlotMap &m, double2 *v, int o, bool &remote) {
  remote = !(o >= m.s_lo && o <= m.s_hi);
  if (!remote) return v + (size_t)(o - m.s_lo) * m.NT;
  return o < m.s_lo ? m.haloL : m.haloR;
}

// ---- one whole-window march of one system (subdomain j, one RHS) ---------
enum : int32_t {
  SYS_HAS_LEFT = 1,      // interface at a_j (j >= 2): B row 0, flux l_j in, r_{j-1} out
  SYS_HAS_RIGHT = 2,     // interface at b_j (j <= N-1)
  SYS_LIN_IMPULSE = 4,   // l_{j,n} = delta_{n,1} (probe)
  SYS_RIN_IMPULSE = 8,   // r_{j,n} = delta_{n,1} (probe)
};

struct MarchSys {
  const double2 *lin;      // [N_T] incoming l_{j,n} (NULL = 0)
  const double2 *rin;      // [N_T] incoming r_{j,n}
  double2 *out_left;       // [N_T] r_{j-1,n} = -l_{j,n} + 2 S v_{j,n}(a_j)   (eq. 8)
  double2 *out_right;      // [N_T] l_{j+1,n} = -r_{j,n} + 2 S v_{j,n}(b_j)
  double2 *uT;             // [N_j] u_{N_T} on the subdomain (NULL = skip)
  const double2 *u0;       // [N_j] u_0 restricted (NULL = 0)
  const double2 *q;        // [N_j] pivot reciprocals 1/p_k of (A - B)
  const double *er;        // [N_j] Re E_k, E_k = (A-B)_{k,k+1}
  int32_t flags;
  int32_t pad_;
  // higher-order transmission operators (MarchParams::tc_hi), side 0 = a_j, 1 = b_j:
  // S v_n = sum_{s<=n} K(n,s) v_s = even part (kernel kap, emitted by eq. 8)
  // + odd part dlt gamma_{n-s} rho^{n-s} (local condition only); the v_0 term
  // carries the factor f0 (gauge phase), A23-A25
  const double2 *kap[2];   // [N_T+1] even kernels
  double2 c0e[2];          // kap[side][0]
  double2 dlt[2], rho[2], f0[2];
};

struct MarchParams {
  const MarchSys *sys;
  int32_t nsys, Nj, NT, CS;  // CS = CTAs per system (thread-block cluster)
  double e_im;               // Im E_k = (2/dt)(h/6), constant on the uniform mesh
  double kappa;              // (2/dt)(h/6): rhs = i kappa (u_{k-1} + 4u_k + u_{k+1})
  double2 c0;                // leading coefficient of the transmission operator
  double2 c2;                // e^{-i pi/4} sqrt(2/dt) (S0^2)
  int32_t s02;               // 1: S0^2 history convolution, 0: Robin
  int32_t tc_hi;             // 1: higher-order operator (per-system kernels in MarchSys)
  int32_t flux_smem;         // 1: stage the incoming flux series in shared memory
  const double *beta;        // [N_T+1] beta_s
  long long *trace;          // optional per-phase clock trace (debug), NULL in production
  size_t td_stride;          // V(t,x): q/er of step n at q + (n-1) td_stride; 0 = constant matrix
  // nonlinear f(u) = lambda |u|^2, k_march_nl only
  double lambda, h12;        // lambda, h/12
  double tol_fp;
  int32_t maxit_fp;
  int32_t *fp_stat;          // [0] max fixed-point iterations (atomicMax), [1] = 1 if a step hit maxit_fp
  double2 *hv_glob;          // k_march_nl: boundary-value histories [nsys][2][N_T+1] (scratch)
};

}  // namespace swr

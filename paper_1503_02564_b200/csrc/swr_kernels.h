// swr_kernels.h — kernel declarations shared by the host orchestration.
#pragma once
#include "swr_common.cuh"
#include <utility>

namespace swr {

// Launch with programmatic stream serialization (the kernel must call
// pdl_wait() before reading what earlier work in the stream wrote).
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// launch_pdl plus an L2 access-policy window (persisting hits on
// [wptr, wptr + wbytes), hit ratio wratio); wbytes = 0: no window
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_win(const void *wptr, size_t wbytes, float wratio, void (*kern)(KArgs...), dim3 grid,
                                  dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  at[1].id = cudaLaunchAttributeAccessPolicyWindow;
  at[1].val.accessPolicyWindow.base_ptr = const_cast<void *>(wptr);
  at[1].val.accessPolicyWindow.num_bytes = wbytes;
  at[1].val.accessPolicyWindow.hitRatio = wratio;
  at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = at;
  cfg.numAttrs = wbytes ? 2 : 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

struct FactorJob {
  const double *W;   // nodal W on the subdomain [N_j] (NULL = 0)
  int32_t has_left, has_right;
  int32_t g0, pad_; // global index of local node 0 (V(t,x))
  double2 *q;        // [N_j] out: 1/p_k
  double *er;        // [N_j] out: Re E_k
  double2 c0L, c0R;  // leading coefficients of the transmission operator at a_j, b_j
};

__global__ void k_factor(const FactorJob *jobs, int njobs, int Nj, double h, double dt, double2 c0, int *err);
constexpr int TR = 8;  // outputs per thread of the Toeplitz kernel (N_T = 500: 32 threads per output slot)
__global__ void k_toeplitz_I_minus_L(const double2 *X, const double2 *x, double2 *y, const SlotMap m);
__global__ void k_halo_add(const double2 *x, const double2 *h, double2 *y, int NT, const double2 *xs);
__global__ void k_axpby(double2 a, const double2 *x, double2 b, double2 *y, size_t n);
__global__ void k_lin2(double2 *z, double2 a, const double2 *x, double2 b, const double2 *y, size_t n);
__global__ void k_bicg_p(double2 *p, const double2 *r, const double2 *v, double2 beta, double2 omega, size_t n);
__global__ void k_bicg_xr(double2 *x, double2 *r, const double2 *p, const double2 *sv, const double2 *t, double2 alpha,
                          double2 omega, size_t n);
__global__ void k_sub(const double2 *x, const double2 *y, double2 *z, size_t n);
__global__ void k_multi_update(const double2 *V, size_t ldv, int nvec, const double2 *y, double2 *x, size_t n);
__global__ void k_gather_uT(const double2 *loc, int N, int m, int Nj, int j_lo, int j_hi, double2 *uT);
__global__ void k_replicate(const double2 *src, double2 *dst, size_t blk, size_t count);
__global__ void k_add_f64(double *y, const double *x, size_t n);

// CGS_REV: walk the element chunks from the end (alternating directions
// between consecutive passes keeps the last-read part of V hot in L2)
enum : int { CGS_AXPY = 1, CGS_DOTS = 2, CGS_NORM = 4, CGS_SCALE = 8, CGS_REV = 16 };
cudaError_t launch_fft_conv_reg(const double2 *Fc, const double2 *x, double2 *y, const SlotMap &m, const double2 *tw,
                                cudaStream_t st, const double2 *xs = nullptr, double2 *xcopy = nullptr);
size_t l2_persist_bytes();
// exact P^{-1} by causal forward substitution (swr_pinv.cu), time blocks of PINV_B steps
constexpr int PINV_B = 16;
cudaError_t launch_pinv_causal(const double2 *X0, const double2 *y, double2 *x, double2 *F, int N, int NT,
                               int sweeps, cudaStream_t st, int *n_launches);
// one fused Gram-Schmidt pass: per-slot unit partials into partial[nred][2N-2]
// (columns of this rank's slots); launch_cgs_reduce sums them in a fixed order
cudaError_t launch_cgs(const double2 *V, size_t ldv, int nv, const double2 *hsrc, double2 *w, int mode,
                       const SlotMap &m, double2 *partial, cudaStream_t st, size_t vwin = 0, float vratio = 1.0f);
int cgs_units_global(const SlotMap &m);   // columns of the partials (units of the fixed-order sums)
cudaError_t launch_cgs_reduce(const double2 *partial, int nu, int nred, int mode, double2 *out, double2 *out_host,
                              cudaStream_t st);
__global__ void k_scale_dev(const double2 *x, const double2 *sp, double2 *y, size_t n);

int fft_log4_for(int NT);
cudaError_t launch_fft_conv(int log4, const double2 *Fc, const double2 *x, double2 *y, const SlotMap &m,
                            const double2 *tw, cudaStream_t st);
__global__ void k_twiddles(double2 *tw, int NF);
cudaError_t launch_fft_fwd(int log4, const double2 *src, size_t stride, int count, int NT, const double2 *tw,
                           double2 *F, cudaStream_t st);

struct MarchShape { int M, P, CS, K; };
MarchShape choose_march_shape(int Nj, int NT, bool tc_hi = false);
size_t march_smem_bytes(const MarchShape &s, int NT, bool flux_smem, bool tc_hi = false);
cudaError_t launch_march(MarchParams p, const MarchShape &s, cudaStream_t st);
size_t march_stream_smem_bytes(int NT);
size_t stream2_stride(int Nj, int nsys_ref, int NT);
cudaError_t launch_march_stream(MarchParams p, int nsys_total, int nsys_ref, double2 *ust, double2 *zst,
                                double2 *ast, double2 *qst, double *est, double2 *bst, size_t stride, int *flags,
                                double2 *vals, cudaStream_t st);
MarchShape choose_march_shape_nl(int Nj, int rows = 0, int nsys = 1);
cudaError_t launch_march_nl_stream(MarchParams p, int nsys_total, int nsys_ref, double2 *ust, double2 *zst,
                                   double2 *zest, double2 *ast, double2 *qst, double *est, size_t stride, int *flags,
                                   double2 *vals, int nslot, cudaStream_t st);
size_t march_nl_smem_bytes(const MarchShape &s, int NT, bool flux_smem);
cudaError_t launch_march_nl(MarchParams p, const MarchShape &s, cudaStream_t st);
__global__ void k_factor_td(const FactorJob *jobs, int njobs, int Nj, int NT, double h, double dt, double2 c0,
                            const double *tau, const double *xi, int n_terms, int Nx, int m, size_t stride, int *err);

}  // namespace swr

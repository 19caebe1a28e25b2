// swr_api.cu — host orchestration behind include/swr.h: setup, interface
// operator construction (Algorithm 3 of PAPER.md), GMRES(m) with
// classical Gram-Schmidt on the interface problem, the preconditioned
// algorithms and the final sweep, one process (rank) per GPU.
// All arithmetic of the method runs in the kernels of swr_march.cu /
// swr_linalg.cu; the host only keeps the (m+1) x m Hessenberg matrix and its
// Givens rotations.
//
// Multi-GPU (the block-column ownership of P:982-1011): a rank
// owns a contiguous range of subdomains and their interface slots; its
// Krylov vectors, d and g hold those slots only.  Per operator application
// (a march sweep or the Toeplitz apply) only the two cut traces cross to the
// neighbour ranks (send/recv of N_T complex each); per Gram-Schmidt pass the
// per-subdomain partial sums are summed over ranks (disjoint columns) and
// reduced in the same fixed order as on one GPU, so G GPUs reproduce the
// one-GPU scalars bitwise.
#include "swr.h"
#include "swr_kernels.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <complex>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>
#include <dlfcn.h>

using swr::MarchParams;
using swr::MarchShape;
using swr::MarchSys;
typedef std::complex<double> cplx;

namespace {

thread_local std::string g_detail;

#define CK(call)                                                                     \
  do {                                                                               \
    cudaError_t e_ = (call);                                                         \
    if (e_ != cudaSuccess) {                                                         \
      g_detail = std::string(#call) + ": " + cudaGetErrorString(e_) + " (" +         \
                 __FILE__ + ":" + std::to_string(__LINE__) + ")";                    \
      return SWR_ERR_CUDA;                                                           \
    }                                                                                \
  } while (0)
#define CKS(call)                                                                    \
  do {                                                                               \
    int s_ = (call);                                                                 \
    if (s_ != SWR_OK) return s_;                                                     \
  } while (0)

inline double2 d2(cplx z) { return make_double2(z.real(), z.imag()); }
inline cplx c2(double2 z) { return cplx(z.x, z.y); }

// ---- NCCL (loaded on demand for world > 1) ---------------------------------
typedef struct ncclComm *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId_t;
typedef int (*fn_commInitRank)(ncclComm_t *, int, ncclUniqueId_t, int);
typedef int (*fn_commDestroy)(ncclComm_t);
typedef int (*fn_send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*fn_recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*fn_allreduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t);
typedef int (*fn_allgather)(const void *, void *, size_t, int, ncclComm_t, cudaStream_t);
typedef int (*fn_reduce)(const void *, void *, size_t, int, int, int, ncclComm_t, cudaStream_t);
typedef int (*fn_group)(void);
typedef int (*fn_getid)(ncclUniqueId_t *);
struct Nccl {
  void *lib = nullptr;
  fn_commInitRank commInitRank;
  fn_commDestroy commDestroy;
  fn_send send;
  fn_recv recv;
  fn_allreduce allReduce;
  fn_allgather allGather;
  fn_reduce reduce;
  fn_group groupStart, groupEnd;
  fn_getid getUniqueId;
};
Nccl g_nccl;
enum { nccl_int32 = 2, nccl_float64 = 8, nccl_sum = 0, nccl_max = 2 };

int load_nccl() {
  if (g_nccl.lib) return SWR_OK;
  const char *names[] = {"libnccl.so.2", "libnccl.so"};
  for (const char *nm : names) {
    g_nccl.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
    if (g_nccl.lib) break;
  }
  if (!g_nccl.lib) { g_detail = "cannot dlopen libnccl.so.2"; return SWR_ERR_NCCL; }
  g_nccl.commInitRank = (fn_commInitRank)dlsym(g_nccl.lib, "ncclCommInitRank");
  g_nccl.commDestroy = (fn_commDestroy)dlsym(g_nccl.lib, "ncclCommDestroy");
  g_nccl.send = (fn_send)dlsym(g_nccl.lib, "ncclSend");
  g_nccl.recv = (fn_recv)dlsym(g_nccl.lib, "ncclRecv");
  g_nccl.allReduce = (fn_allreduce)dlsym(g_nccl.lib, "ncclAllReduce");
  g_nccl.allGather = (fn_allgather)dlsym(g_nccl.lib, "ncclAllGather");
  g_nccl.reduce = (fn_reduce)dlsym(g_nccl.lib, "ncclReduce");
  g_nccl.groupStart = (fn_group)dlsym(g_nccl.lib, "ncclGroupStart");
  g_nccl.groupEnd = (fn_group)dlsym(g_nccl.lib, "ncclGroupEnd");
  g_nccl.getUniqueId = (fn_getid)dlsym(g_nccl.lib, "ncclGetUniqueId");
  if (!g_nccl.commInitRank || !g_nccl.send || !g_nccl.recv || !g_nccl.allReduce || !g_nccl.reduce ||
      !g_nccl.groupStart) {
    g_detail = "libnccl is missing symbols";
    return SWR_ERR_NCCL;
  }
  return SWR_OK;
}

// ---- communicators ----------------------------------------------------------
// The ranks of one handle exchange: sums of vectors with disjoint supports
// (exact in any order), the cut traces with the two neighbour ranks, an
// integer max, and the final reduction of u(T) to rank 0.  NcclComm is the
// product path (one process per GPU, NVLink / NVSwitch); LoopbackComm runs G
// logical ranks as G host threads of one process on one GPU with device copies
// standing in for NCCL -- test infrastructure for the multi-rank code path
// (swr_loopback_id), never selected otherwise.
struct Comm {
  virtual ~Comm() {}
  virtual int allreduce_sum(const double *send, double *recv, size_t n, cudaStream_t st) = 0;
  virtual int allreduce_max_i32(int *buf, size_t n, cudaStream_t st) = 0;
  // sendL -> rank-1 (its recvR), sendR -> rank+1 (its recvL); nullptr where absent
  virtual int exchange(const double2 *sendL, double2 *recvL, const double2 *sendR, double2 *recvR, size_t n,
                       cudaStream_t st) = 0;
  virtual int reduce_sum_root(double *buf, size_t n, cudaStream_t st) = 0;
};

struct NcclComm : Comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1;
  ~NcclComm() override {
    if (comm && g_nccl.commDestroy) g_nccl.commDestroy(comm);
  }
  int allreduce_sum(const double *send, double *recv, size_t n, cudaStream_t st) override {
    if (g_nccl.allReduce(send, recv, n, nccl_float64, nccl_sum, comm, st) != 0) {
      g_detail = "ncclAllReduce failed";
      return SWR_ERR_NCCL;
    }
    return SWR_OK;
  }
  int allreduce_max_i32(int *buf, size_t n, cudaStream_t st) override {
    if (g_nccl.allReduce(buf, buf, n, nccl_int32, nccl_max, comm, st) != 0) {
      g_detail = "ncclAllReduce (max) failed";
      return SWR_ERR_NCCL;
    }
    return SWR_OK;
  }
  int exchange(const double2 *sendL, double2 *recvL, const double2 *sendR, double2 *recvR, size_t n,
               cudaStream_t st) override {
    g_nccl.groupStart();
    int e = 0;
    if (sendL) e |= g_nccl.send(sendL, 2 * n, nccl_float64, rank - 1, comm, st);
    if (recvL) e |= g_nccl.recv(recvL, 2 * n, nccl_float64, rank - 1, comm, st);
    if (sendR) e |= g_nccl.send(sendR, 2 * n, nccl_float64, rank + 1, comm, st);
    if (recvR) e |= g_nccl.recv(recvR, 2 * n, nccl_float64, rank + 1, comm, st);
    e |= g_nccl.groupEnd();
    if (e) { g_detail = "ncclSend/ncclRecv of the cut traces failed"; return SWR_ERR_NCCL; }
    return SWR_OK;
  }
  int reduce_sum_root(double *buf, size_t n, cudaStream_t st) override {
    if (g_nccl.reduce(buf, buf, n, nccl_float64, nccl_sum, 0, comm, st) != 0) {
      g_detail = "ncclReduce failed";
      return SWR_ERR_NCCL;
    }
    return SWR_OK;
  }
};

// In-process group of G logical ranks (one host thread each, same device).
struct LoopGroup {
  int world = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  std::vector<const void *> a, b;   // published pointers of each rank
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const unsigned long long g = gen;
    if (++arrived == world) {
      arrived = 0;
      gen++;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};
std::mutex g_loop_mu;
std::map<unsigned long long, std::shared_ptr<LoopGroup>> g_loop_groups;
const char kLoopMagic[8] = {'S', 'W', 'R', 'L', 'O', 'O', 'P', 0};

struct LoopbackComm : Comm {
  std::shared_ptr<LoopGroup> grp;
  int rank = 0, world = 1;
  double *scratch = nullptr;
  size_t scratch_n = 0;
  ~LoopbackComm() override {
    if (scratch) cudaFree(scratch);
  }
  int sync(cudaStream_t st) {
    if (cudaStreamSynchronize(st) != cudaSuccess) { g_detail = "loopback: stream sync failed"; return SWR_ERR_CUDA; }
    return SWR_OK;
  }
  int allreduce_sum(const double *send, double *recv, size_t n, cudaStream_t st) override {
    if (n > scratch_n) {
      if (scratch) cudaFree(scratch);
      if (cudaMalloc((void **)&scratch, n * sizeof(double)) != cudaSuccess) return SWR_ERR_OOM;
      scratch_n = n;
    }
    int s = sync(st);
    if (s) return s;
    grp->a[rank] = send;
    grp->barrier();
    // every rank sums all ranks' buffers in rank order into its own scratch
    if (cudaMemcpyAsync(scratch, grp->a[0], n * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return SWR_ERR_CUDA;
    for (int r = 1; r < world; r++)
      swr::k_add_f64<<<(unsigned)std::min<size_t>((n + 255) / 256, 4096), 256, 0, st>>>(
          scratch, (const double *)grp->a[r], n);
    if ((s = sync(st))) return s;
    grp->barrier();   // nobody reads the send buffers any more
    if (cudaMemcpyAsync(recv, scratch, n * sizeof(double), cudaMemcpyDeviceToDevice, st) != cudaSuccess)
      return SWR_ERR_CUDA;
    return sync(st);
  }
  int allreduce_max_i32(int *buf, size_t n, cudaStream_t st) override {
    std::vector<int> mine(n), acc(n);
    if (cudaMemcpyAsync(mine.data(), buf, n * sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess)
      return SWR_ERR_CUDA;
    int s = sync(st);
    if (s) return s;
    grp->a[rank] = mine.data();
    grp->barrier();
    for (size_t i = 0; i < n; i++) {
      int m = ((const int *)grp->a[0])[i];
      for (int r = 1; r < world; r++) m = std::max(m, ((const int *)grp->a[r])[i]);
      acc[i] = m;
    }
    grp->barrier();
    if (cudaMemcpyAsync(buf, acc.data(), n * sizeof(int), cudaMemcpyHostToDevice, st) != cudaSuccess)
      return SWR_ERR_CUDA;
    return sync(st);
  }
  int exchange(const double2 *sendL, double2 *recvL, const double2 *sendR, double2 *recvR, size_t n,
               cudaStream_t st) override {
    int s = sync(st);
    if (s) return s;
    grp->a[rank] = sendL;
    grp->b[rank] = sendR;
    grp->barrier();
    if (recvL && cudaMemcpyAsync(recvL, grp->b[rank - 1], n * sizeof(double2), cudaMemcpyDeviceToDevice, st))
      return SWR_ERR_CUDA;
    if (recvR && cudaMemcpyAsync(recvR, grp->a[rank + 1], n * sizeof(double2), cudaMemcpyDeviceToDevice, st))
      return SWR_ERR_CUDA;
    if ((s = sync(st))) return s;
    grp->barrier();
    return SWR_OK;
  }
  int reduce_sum_root(double *buf, size_t n, cudaStream_t st) override { return allreduce_sum(buf, buf, n, st); }
};

template <typename T>
int dalloc(T **p, size_t n) {
  if (n == 0) { *p = nullptr; return SWR_OK; }
  cudaError_t e = cudaMalloc((void **)p, n * sizeof(T));
  if (e != cudaSuccess) {
    g_detail = std::string("cudaMalloc(") + std::to_string(n * sizeof(T)) + "): " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? SWR_ERR_OOM : SWR_ERR_CUDA;
  }
  return SWR_OK;
}

inline unsigned grid_for(size_t n, int bs = 256) {
  size_t g = (n + bs - 1) / bs;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g ? g : 1);
}

// Krylov workspace of one GMRES instance (outer and inner P^{-1} solves
// have their own, so the outer speculation never races the inner solve).
struct Krylov {
  double2 *V, *w;
  double2 *w2;          // second work vector (fused normalisation path)
  double2 *dots;        // device [2][3(m+2)+8]: per-iteration scalars, double-buffered
  double2 *hp;          // pinned mirror, same layout
  double2 *ycoef;       // device [m]
  cudaEvent_t ev[2];
};

}  // namespace

struct swr_handle {
  // problem
  double a0, b0, T, dx, dt, lambda, robin_p, tol, tol_inner, tol_fp;
  int N, potential, transmission, algorithm, restart, maxit, maxit_inner, maxit_fp, n_terms;
  int gs_passes = 1;   // Gram-Schmidt passes per Arnoldi step (1: CGS, 2: CGS2)
  int krylov = 0;      // swr_krylov
  int pade_m = 0;      // Pade poles (SWR_TC_S2_*)
  int pinv_exact = 0;  // exact causal P^{-1} (A27)
  int pinv_sweeps = 0; // block-Jacobi sweeps of its lag-0 solve
  double pinv_rho = 0.0;
  double2 *pinvF = nullptr;   // [2N-2][PINV_B] far-history scratch
  double2 *pinv_y = nullptr, *pinv_x = nullptr;   // world > 1: full-length P^{-1} operands
  int cgs_dir = 0;         // alternating traversal direction of the CGS passes (L2 reuse)
  size_t vwin_bytes = 0;   // persisting L2 window over the first outer-Krylov basis vectors
  float vwin_ratio = 1.0f;
  size_t l2_window = 0;    // persisting L2 set-aside this handle asked for
  int Nx, NT, Nj, m;
  size_t ng;               // full interface vector, (2N-2) N_T
  size_t nloc;             // this rank's slots, (s_hi - s_lo + 1) N_T (= ng on one GPU)
  int rank, world, device;
  int j_lo, j_hi;                          // this rank's subdomains (1-based, inclusive)
  int s_lo, s_hi;                          // and their slots
  swr::SlotMap smap;
  Comm *comm = nullptr;
  double2 *haloL = nullptr, *haloR = nullptr;     // [N_T] outputs for the neighbour ranks
  double2 *hrecvL = nullptr, *hrecvR = nullptr;   // [N_T] (I - L) contributions from them
  double2 *part_send = nullptr, *part_recv = nullptr;   // [33][N] CGS unit partials (world > 1)
  int march_form = 0, toeplitz_form = 0, nl_rows = 0;
  double t_setup_ms = 0.0;
  cudaStream_t st;
  double2 c0, c2v;
  // higher-order transmission operators (tc_hi): per subdomain side
  bool tc_hi = false;
  double2 *kap = nullptr;                 // device [N][2][N_T+1] even kernels
  std::vector<double2> tc_c0, tc_c0e, tc_dlt, tc_rho, tc_f0;   // [N][2]
  double kappa, eim;
  MarchShape shape;                        // launch shape of the resident march (one RHS per group)
  // device data
  double2 *u0 = nullptr;
  double *Vx = nullptr, *beta = nullptr;
  double2 *q = nullptr, *q0 = nullptr;     // pivots: physical [N][Nj], V=0 [3][Nj]
  double *er = nullptr, *er0 = nullptr;
  double2 *d = nullptr, *X = nullptr, *X0 = nullptr, *g = nullptr, *g0 = nullptr;
  double2 *uloc = nullptr, *uT = nullptr;
  double2 *tmp = nullptr, *tmp2 = nullptr, *rhs = nullptr;
  // FFT form of the Toeplitz apply: twiddles, transformed columns of L and L0
  int log4 = 0;           // NF = 4^log4 (0: the direct causal convolution)
  bool fft_reg = false;   // register four-step FFT kernel (NF = 1024)
  // V(t,x): per-step pivots [N_T][N][N_j]; f(u): fixed-point stats
  double *tau = nullptr, *xi = nullptr;
  double2 *qtd = nullptr;
  double *ertd = nullptr;
  int *fp_stat = nullptr;
  MarchShape shape_nl;
  double2 *hv_nl = nullptr;                // NL march: boundary-value histories [owned][2][N_T+1]
  bool nl_stream = false;                  // NL subdomains beyond the resident march: k_march_nl_stream
  double2 *snl_ze = nullptr, *snl_vals = nullptr;
  int *snl_flags = nullptr;
  double2 *tw = nullptr, *FX = nullptr, *FX0 = nullptr;
  double2 *partial = nullptr;
  // streaming march (subdomains too large for the resident kernel)
  bool stream_march = false;
  double2 *sst_u = nullptr, *sst_z = nullptr, *sst_a = nullptr, *sst_q = nullptr, *sst_b = nullptr,
          *sst_vals = nullptr;
  double *sst_e = nullptr;
  size_t sst_stride = 0;
  int *sst_flags = nullptr;
  int sst_cap = 0;   // systems the scratch holds
  Krylov kout = {}, kin = {};             // outer / inner (P^{-1}) GMRES workspaces
  double2 *hpin = nullptr;                 // pinned scalars for restarts and norms
  MarchSys *sys_dev = nullptr;
  int *err_dev = nullptr;
  swr::FactorJob *jobs_dev = nullptr;
  size_t jobs_cap = 0;
  bool have_L = false, have_L0 = false, have_d = false, have_g = false;
  // report
  std::vector<double> hist;
  int iterations = 0, inner_total = 0, fp_max = 0, converged = 0;
  bool inner_fail = false;
  double cell_steps = 0;
  int n_marches = 0, n_launches = 0;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> march_ev, intf_ev, comm_ev;
  size_t march_ev_used = 0, intf_ev_used = 0, comm_ev_used = 0;
  cudaEvent_t ev_b0 = nullptr, ev_b1 = nullptr, ev_s0 = nullptr, ev_s1 = nullptr;
  cudaStream_t st_in = nullptr;                     // host-input copies overlapping the factorisation
  cudaEvent_t ev_in0 = nullptr, ev_in1 = nullptr;
  bool build_timed = false;
};

namespace {

enum { EV_INTF = 0, EV_MARCH = 1, EV_COMM = 2 };
int record_pair(swr_handle *h, int kind, bool begin) {
  auto &vec = kind == EV_MARCH ? h->march_ev : (kind == EV_COMM ? h->comm_ev : h->intf_ev);
  size_t &used = kind == EV_MARCH ? h->march_ev_used : (kind == EV_COMM ? h->comm_ev_used : h->intf_ev_used);
  if (begin) {
    if (used == vec.size()) {
      cudaEvent_t a, b;
      CK(cudaEventCreate(&a));
      CK(cudaEventCreate(&b));
      vec.push_back({a, b});
    }
    CK(cudaEventRecord(vec[used].first, h->st));
  } else {
    CK(cudaEventRecord(vec[used].second, h->st));
    used++;
  }
  return SWR_OK;
}

double sum_pairs(swr_handle *h, int kind) {
  auto &vec = kind == EV_MARCH ? h->march_ev : (kind == EV_COMM ? h->comm_ev : h->intf_ev);
  size_t used = kind == EV_MARCH ? h->march_ev_used : (kind == EV_COMM ? h->comm_ev_used : h->intf_ev_used);
  double s = 0;
  for (size_t i = 0; i < used; i++) {
    float ms = 0;
    if (cudaEventElapsedTime(&ms, vec[i].first, vec[i].second) == cudaSuccess) s += ms;
  }
  return s;
}

constexpr int kStreamSlots = 148 * 32;   // chain CTAs of one streaming launch, upper bound
int slot_l(int j) { return 2 * j - 3; }
int slot_r(int j) { return 2 * j - 2; }
int zero_matrix_index(swr_handle *h, int j) { return j == 1 ? 0 : (j == h->N ? 2 : 1); }

// ---- one batched march of many systems --------------------------------------
enum { MARCH_CONST = 0, MARCH_TD = 1, MARCH_NL = 2 };

int run_march(swr_handle *h, const std::vector<MarchSys> &sys, int nreal, int mode = MARCH_CONST) {
  if (sys.empty()) return SWR_OK;
  CK(cudaMemcpyAsync(h->sys_dev, sys.data(), sys.size() * sizeof(MarchSys), cudaMemcpyHostToDevice, h->st));
  MarchParams p;
  p.sys = h->sys_dev;
  p.nsys = (int)sys.size();
  p.Nj = h->Nj;
  p.NT = h->NT;
  p.CS = h->shape.CS;
  p.e_im = h->eim;
  p.kappa = h->kappa;
  p.c0 = h->c0;
  p.tc_hi = h->tc_hi ? 1 : 0;
  p.c2 = h->c2v;
  p.s02 = h->transmission == SWR_TC_S0_2;
  p.flux_smem = 0;
  for (const MarchSys &m : sys)
    if (m.lin || m.rin) p.flux_smem = 1;
  p.beta = h->beta;
  p.trace = nullptr;
  p.td_stride = mode == MARCH_TD ? (size_t)h->N * h->Nj : 0;
  p.lambda = h->lambda;
  p.h12 = h->dx / 12.0;
  p.tol_fp = h->tol_fp;
  p.maxit_fp = h->maxit_fp;
  p.fp_stat = h->fp_stat;
  if (mode == MARCH_NL) {
    p.hv_glob = h->hv_nl;
    CKS(record_pair(h, EV_MARCH, true));
    if (h->nl_stream) {
      if ((int)sys.size() > h->sst_cap) { g_detail = "streaming scratch too small"; return SWR_ERR_UNSUPPORTED; }
      CK(swr::launch_march_nl_stream(p, (int)sys.size(), h->N, h->sst_u, h->sst_z, h->snl_ze, h->sst_a, h->sst_q,
                                     h->sst_e, h->sst_stride, h->snl_flags, h->snl_vals, kStreamSlots, h->st));
    } else {
      CK(swr::launch_march_nl(p, h->shape_nl, h->st));
    }
    CK(cudaGetLastError());
    CKS(record_pair(h, EV_MARCH, false));
    h->n_marches++;
    h->n_launches++;
    h->cell_steps += (double)nreal * h->Nj * h->NT;
    return SWR_OK;
  }
#if SWR_MARCH_TRACE
  if (getenv("SWR_TRACE") && !h->stream_march) {
    // per-CTA phase trace of the first cluster (trace builds only: tools/march_trace.sh)
    static long long *tr = nullptr;
    const int ntr = 16 * 32;
    if (!tr) CK(cudaMalloc(&tr, ntr * sizeof(long long)));
    CK(cudaMemsetAsync(tr, 0, ntr * sizeof(long long), h->st));
    p.trace = tr;
    CK(swr::launch_march(p, h->shape, h->st));
    std::vector<long long> hv(ntr);
    CK(cudaMemcpyAsync(hv.data(), tr, ntr * sizeof(long long), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    const MarchShape &sh = h->shape;
    fprintf(stderr, "march trace M=%d P=%d CS=%d (cycles from step start)\n", sh.M, sh.P, sh.CS);
    for (int c = 0; c < sh.CS; c++) {
      const long long *r = hv.data() + c * 32;
      fprintf(stderr, "  cta %d:", c);
      for (int i = 1; i < 30; i++)
        if (r[i]) fprintf(stderr, " %d:%lld", i, r[i] - r[0]);
      fprintf(stderr, "\n");
    }
    p.trace = nullptr;
  }
#endif
  CKS(record_pair(h, EV_MARCH, true));
  if (h->stream_march) {
    // in batches of co-resident chains
    if ((int)sys.size() > h->sst_cap) { g_detail = "streaming scratch too small"; return SWR_ERR_UNSUPPORTED; }
    CK(swr::launch_march_stream(p, (int)sys.size(), h->N, h->sst_u, h->sst_z, h->sst_a, h->sst_q, h->sst_e,
                                h->sst_b, h->sst_stride, h->sst_flags, h->sst_vals, h->st));
  } else {
    CK(swr::launch_march(p, h->shape, h->st));
  }
  CK(cudaGetLastError());
  CKS(record_pair(h, EV_MARCH, false));
  h->n_marches++;
  h->n_launches++;
  h->cell_steps += (double)nreal * h->Nj * h->NT;
  return SWR_OK;
}

// system of owned subdomain j (1-based) with fluxes from the local interface
// vector g (may be NULL); its outputs go to the local slots of Rg, or to the
// halo buffers when the neighbour rank owns the slot (eq. 8 across a cut)
MarchSys make_sys(swr_handle *h, int j, const double2 *g, bool use_u0, bool zero_pot, double2 *Rg,
                  double2 *uloc) {
  MarchSys s;
  memset(&s, 0, sizeof s);
  const int N = h->N;
  if (j >= 2) s.flags |= swr::SYS_HAS_LEFT;
  if (j <= N - 1) s.flags |= swr::SYS_HAS_RIGHT;
  if (g && j >= 2) s.lin = swr::slot_ptr(h->smap, g, slot_l(j));
  if (g && j <= N - 1) s.rin = swr::slot_ptr(h->smap, g, slot_r(j));
  bool remote;
  if (Rg && j >= 2) s.out_left = swr::out_ptr(h->smap, Rg, slot_r(j - 1), remote);
  if (Rg && j <= N - 1) s.out_right = swr::out_ptr(h->smap, Rg, slot_l(j + 1), remote);
  s.uT = uloc ? uloc + (size_t)(j - 1) * h->Nj : nullptr;
  s.u0 = use_u0 ? h->u0 + (size_t)(j - 1) * h->m : nullptr;
  if (zero_pot) {
    const int zi = zero_matrix_index(h, j);
    s.q = h->q0 + (size_t)zi * h->Nj;
    s.er = h->er0 + (size_t)zi * h->Nj;
  } else if (h->potential == SWR_POT_VTX_SEPARABLE) {
    s.q = h->qtd + (size_t)(j - 1) * h->Nj;     // step 1; step n at + (n-1) N N_j
    s.er = h->ertd + (size_t)(j - 1) * h->Nj;
  } else {
    s.q = h->q + (size_t)(j - 1) * h->Nj;
    s.er = h->er + (size_t)(j - 1) * h->Nj;
  }
  if (h->tc_hi && !zero_pot) {
    for (int side = 0; side < 2; side++) {
      const size_t o = (size_t)(j - 1) * 2 + side;
      s.kap[side] = h->kap + o * (h->NT + 1);
      s.c0e[side] = h->tc_c0e[o];
      s.dlt[side] = h->tc_dlt[o];
      s.rho[side] = h->tc_rho[o];
      s.f0[side] = h->tc_f0[o];
    }
  }
  return s;
}

int fill_zero(swr_handle *h, double2 *x, size_t n) {
  if (!n) return SWR_OK;
  CK(cudaMemsetAsync(x, 0, n * sizeof(double2), h->st));
  return SWR_OK;
}

// ---- collectives (world > 1), timed as communication ----------------------
// The cut traces of eq. (8): what this rank's subdomains produced for the
// neighbours' first / last slot (halo buffers) goes out, and the neighbours'
// contributions arrive -- into recvL / recvR (first and last local slot).
int exchange_cut(swr_handle *h, double2 *recvL, double2 *recvR) {
  if (h->world <= 1) return SWR_OK;
  CKS(record_pair(h, EV_COMM, true));
  CKS(h->comm->exchange(h->rank > 0 ? h->haloL : nullptr, h->rank > 0 ? recvL : nullptr,
                        h->rank < h->world - 1 ? h->haloR : nullptr, h->rank < h->world - 1 ? recvR : nullptr,
                        (size_t)h->NT, h->st));
  CKS(record_pair(h, EV_COMM, false));
  h->n_launches++;
  return SWR_OK;
}

double2 *last_slot(swr_handle *h, double2 *v) { return v + (size_t)(h->s_hi - h->s_lo) * h->NT; }

// Sum over ranks of n doubles (disjoint supports: exact in any order).
int allreduce_sum(swr_handle *h, const double *send, double *recv, size_t n) {
  if (h->world <= 1 || n == 0) return SWR_OK;
  CKS(record_pair(h, EV_COMM, true));
  CKS(h->comm->allreduce_sum(send, recv, n, h->st));
  CKS(record_pair(h, EV_COMM, false));
  h->n_launches++;
  return SWR_OK;
}

// Rg = R(g; u0?) (eq. 13): every owned subdomain marches once; the outputs
// that cross a rank cut are exchanged with the neighbour ranks.
int sweep_R(swr_handle *h, const double2 *g, bool use_u0, bool zero_pot, double2 *Rg, double2 *uloc) {
  std::vector<MarchSys> sys;
  for (int j = h->j_lo; j <= h->j_hi; j++) sys.push_back(make_sys(h, j, g, use_u0, zero_pot, Rg, uloc));
  if (Rg) CKS(fill_zero(h, Rg, h->nloc));
  int mode = MARCH_CONST;
  if (!zero_pot && h->potential == SWR_POT_VTX_SEPARABLE) mode = MARCH_TD;
  if (!zero_pot && h->potential == SWR_POT_CUBIC) mode = MARCH_NL;
  CKS(run_march(h, sys, (int)sys.size(), mode));
  if (Rg) CKS(exchange_cut(h, Rg, last_slot(h, Rg)));
  return SWR_OK;
}

// ---- higher-order transmission operators -----------
// Per subdomain side: W at the interface node, dnW by the central difference
// on the global mesh with the outward normal (A23), gauge phase rate
// theta = W dt (A24).  Even kernel (emitted through eq. 8, A25):
//   S0^3, S0^4: kap_m = c2 beta_m - e^{i pi/4} sqrt(dt/2) (W/2) alpha_m
//   S1^2, S1^4: kap_m = c2 beta_m e^{i theta m},   v_0 term times e^{-i theta/2}
// odd part (S0^4, S1^4): dlt gamma_m rho^m, dlt = -i (dnW/4)(dt/2), rho = 1 or
// e^{i theta}; leading coefficient of the local condition kap_0 + dlt.
int setup_tc(swr_handle *h) {
  const int N = h->N, NT = h->NT;
  h->tc_c0.assign(2 * N, h->c0);
  h->tc_c0e.assign(2 * N, h->c0);
  h->tc_dlt.assign(2 * N, make_double2(0, 0));
  h->tc_rho.assign(2 * N, make_double2(1, 0));
  h->tc_f0.assign(2 * N, make_double2(1, 0));
  if (!h->tc_hi) return SWR_OK;
  std::vector<double> V((size_t)h->Nx + 1, 0.0);
  if (h->Vx) {
    CK(cudaStreamSynchronize(h->st));
    CK(cudaMemcpy(V.data(), h->Vx, V.size() * sizeof(double), cudaMemcpyDeviceToHost));
  }
  std::vector<double> al(NT + 1), be(NT + 1);
  for (int m = 0; m <= NT; m++) {
    const double a = m == 0 ? 1.0 : (m % 2 ? al[m - 1] : al[m - 2] * (double)(m - 1) / (double)m);
    al[m] = a;
    be[m] = (m % 2) ? -a : a;
  }
  const cplx cc2 = c2(h->c2v), e3 = cplx(1.0, 1.0) / std::sqrt(2.0) * std::sqrt(h->dt / 2.0);
  const int tc = h->transmission;
  const bool pade = tc == SWR_TC_S2_2 || tc == SWR_TC_S2_4;
  // Pade poles (reading A26): the diagonal Pade approximant of sqrt(1 + x)
  // (b_s = 2/(2m+1) sin^2 u_s, c_s = cos^2 u_s, u_s = s pi/(2m+1)) with the
  // branch cut rotated by theta = pi/4, sqrt z = e^{i th/2} sqrt(e^{-i th} z),
  // written as sum_{s>=0} a_s - sum_{s>=1} a_s d_s/(z + d_s) (complex a_s, d_s)
  const int pm = h->pade_m;
  std::vector<cplx> pa(pade ? pm + 1 : 0, cplx(0.0)), pd(pade ? pm + 1 : 0, cplx(0.0));
  if (pade) {
    const double tht = M_PI / 4.0;
    const cplx eh = std::exp(cplx(0.0, tht / 2.0)), ef = std::exp(cplx(0.0, tht));
    cplx sb(0.0), sa(0.0);
    for (int s = 1; s <= pm; s++) {
      const double u = s * M_PI / (2.0 * pm + 1.0), cs = std::cos(u) * std::cos(u);
      const double bs = 2.0 / (2.0 * pm + 1.0) * std::sin(u) * std::sin(u);
      pd[s] = ef * ((1.0 - cs) / cs);
      pa[s] = eh * (bs / (cs * (1.0 - cs)));
      sb += bs / cs;
      sa += pa[s];
    }
    pa[0] = eh * (1.0 + sb) - sa;
  }
  const bool gauge = tc == SWR_TC_S1_2 || tc == SWR_TC_S1_4, order4 = tc == SWR_TC_S0_4 || tc == SWR_TC_S1_4;
  std::vector<double2> K((size_t)N * 2 * (NT + 1));
  for (int j = 1; j <= N; j++) {
    for (int side = 0; side < 2; side++) {
      const int i = side == 0 ? (j - 1) * h->m : j * h->m;
      const double W = V[i];
      const double dxW = (i > 0 && i < h->Nx) ? (V[i + 1] - V[i - 1]) / (2.0 * h->dx) : 0.0;
      const double dnW = side == 0 ? -dxW : dxW;
      const double th = W * h->dt;
      double2 *k = K.data() + ((size_t)(j - 1) * 2 + side) * (NT + 1);
      const size_t o = (size_t)(j - 1) * 2 + side;
      if (pade) {
        // Eliminating phi^s, psi from S2: with
        // D_s = 2i/dt + W + d_s and rho_s = (2i/dt - W - d_s)/D_s,
        //   phi^s_n = (2/D_s) v_n + rho_s phi^s_{n-1}   (v_0 never enters)
        // so S2 v_n = kap_0 v_n + sum_{t=1}^{n-1} kap_{n-t} v_t with
        //   kap_0 = -i sum_s a_s + i sum_s a_s d_s / D_s,
        //   kap_k = sum_s i a_s d_s (2i/dt) (2/D_s^2) rho_s^{k-1}   (k >= 1);
        // S2^4 adds (dnW/4)/D_0 v_n and sum_t (dnW/4)(2i/dt)(2/D_0^2) rho_0^{n-1-t} v_t,
        // i.e. the odd part 2 dlt rho_0^{n-t} with dlt = (dnW/4)(2i/dt)/(D_0^2 rho_0).
        const cplx s2(0.0, 2.0 / h->dt);
        cplx k0(0.0, 0.0);
        for (int s = 0; s <= pm; s++) k0 += cplx(0.0, -1.0) * pa[s];
        for (int m = 1; m <= NT; m++) k[m] = make_double2(0, 0);
        std::vector<cplx> acc(NT + 1, cplx(0.0, 0.0));
        for (int s = 1; s <= pm; s++) {
          const cplx D = s2 + W + pd[s], rho = (s2 - W - pd[s]) / D;
          k0 += cplx(0.0, 1.0) * pa[s] * pd[s] / D;
          const cplx w = cplx(0.0, 1.0) * pa[s] * pd[s] * s2 * 2.0 / (D * D);
          cplx r(1.0, 0.0);
          for (int m = 1; m <= NT; m++) {
            acc[m] += w * r;
            r *= rho;
          }
        }
        acc[0] = k0;
        for (int m = 0; m <= NT; m++) k[m] = d2(acc[m]);
        cplx c0o(0.0), dlt(0.0), rho0(1.0, 0.0);
        if (tc == SWR_TC_S2_4) {
          const cplx D0 = s2 + W;
          rho0 = (s2 - W) / D0;
          c0o = (dnW / 4.0) / D0;
          dlt = (dnW / 4.0) * s2 / (D0 * D0 * rho0);
        }
        h->tc_c0e[o] = k[0];
        h->tc_dlt[o] = d2(dlt);
        h->tc_c0[o] = d2(k0 + c0o);
        h->tc_rho[o] = d2(rho0);
        h->tc_f0[o] = make_double2(0, 0);
        continue;
      }
      for (int m = 0; m <= NT; m++) {
        cplx v = gauge ? cc2 * be[m] * std::exp(cplx(0.0, th * m)) : cc2 * be[m] - e3 * (W / 2.0) * al[m];
        k[m] = d2(v);
      }
      const cplx dlt = order4 ? cplx(0.0, -1.0) * (dnW / 4.0) * (h->dt / 2.0) : cplx(0.0);
      h->tc_c0e[o] = k[0];
      h->tc_dlt[o] = d2(dlt);
      h->tc_c0[o] = d2(c2(k[0]) + dlt);
      h->tc_rho[o] = gauge ? d2(std::exp(cplx(0.0, th))) : make_double2(1, 0);
      h->tc_f0[o] = gauge ? d2(std::exp(cplx(0.0, -th / 2.0))) : make_double2(1, 0);
    }
  }
  if (!h->kap) CKS(dalloc(&h->kap, K.size()));
  CK(cudaMemcpy(h->kap, K.data(), K.size() * sizeof(double2), cudaMemcpyHostToDevice));
  return SWR_OK;
}

// ---- assembly + factorisation ----------------------------------------------
int factor_matrices(swr_handle *h) {
  CKS(setup_tc(h));
  std::vector<swr::FactorJob> jobs;
  const bool phys_const = h->potential != SWR_POT_VTX_SEPARABLE;
  if (phys_const) {
    for (int j = h->j_lo; j <= h->j_hi; j++) {
      swr::FactorJob J;
      J.W = (h->potential == SWR_POT_VX) ? h->Vx + (size_t)(j - 1) * h->m : nullptr;
      J.has_left = j >= 2;
      J.has_right = j <= h->N - 1;
      J.g0 = (j - 1) * h->m;
      J.q = h->q + (size_t)(j - 1) * h->Nj;
      J.er = h->er + (size_t)(j - 1) * h->Nj;
      J.c0L = h->tc_c0[(size_t)(j - 1) * 2 + 0];
      J.c0R = h->tc_c0[(size_t)(j - 1) * 2 + 1];
      jobs.push_back(J);
    }
  }
  if (h->q0) {
    for (int zi = 0; zi < 3; zi++) {
      swr::FactorJob J;
      J.W = nullptr;
      J.has_left = zi >= 1;
      J.has_right = zi <= 1;
      J.g0 = 0;
      if (h->N == 1) J.has_left = J.has_right = 0;
      J.q = h->q0 + (size_t)zi * h->Nj;
      J.er = h->er0 + (size_t)zi * h->Nj;
      J.c0L = J.c0R = h->c0;
      jobs.push_back(J);
    }
  }
  if (h->potential == SWR_POT_VTX_SEPARABLE) {
    std::vector<swr::FactorJob> tj;
    for (int j = h->j_lo; j <= h->j_hi; j++) {
      swr::FactorJob J;
      J.W = nullptr;
      J.has_left = j >= 2;
      J.has_right = j <= h->N - 1;
      J.g0 = (j - 1) * h->m;
      J.q = h->qtd + (size_t)(j - 1) * h->Nj;
      J.er = h->ertd + (size_t)(j - 1) * h->Nj;
      J.c0L = J.c0R = h->c0;
      tj.push_back(J);
    }
    swr::FactorJob *tdev = nullptr;
    CKS(dalloc(&tdev, tj.size()));
    CK(cudaMemcpyAsync(tdev, tj.data(), tj.size() * sizeof(tj[0]), cudaMemcpyHostToDevice, h->st));
    CK(cudaMemsetAsync(h->err_dev, 0, sizeof(int), h->st));
    const long nth = (long)tj.size() * h->NT;
    swr::k_factor_td<<<(unsigned)((nth + 127) / 128), 128, 0, h->st>>>(tdev, (int)tj.size(), h->Nj, h->NT, h->dx, h->dt,
                                                                      h->c0, h->tau, h->xi, h->n_terms, h->Nx, h->m,
                                                                      (size_t)h->N * h->Nj, h->err_dev);
    CK(cudaGetLastError());
    h->n_launches++;
    int herr = 0;
    CK(cudaMemcpyAsync(&herr, h->err_dev, sizeof(int), cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    cudaFree(tdev);
    if (herr) { g_detail = "zero pivot while factoring A_n - B"; return SWR_ERR_ZERO_PIVOT; }
  }
  if (jobs.empty()) return SWR_OK;
  if (jobs.size() > h->jobs_cap) {   // once per handle: a cudaFree here would wait for every stream
    CK(cudaFree(h->jobs_dev));
    h->jobs_dev = nullptr;
    CKS(dalloc(&h->jobs_dev, jobs.size()));
    h->jobs_cap = jobs.size();
  }
  CK(cudaMemcpyAsync(h->jobs_dev, jobs.data(), jobs.size() * sizeof(jobs[0]), cudaMemcpyHostToDevice, h->st));
  CK(cudaMemsetAsync(h->err_dev, 0, sizeof(int), h->st));
  swr::k_factor<<<(unsigned)((jobs.size() + 3) / 4), 128, 0, h->st>>>(h->jobs_dev, (int)jobs.size(), h->Nj, h->dx,
                                                                        h->dt, h->c0, h->err_dev);
  CK(cudaGetLastError());
  h->n_launches++;
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, h->err_dev, sizeof(int), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  if (herr) { g_detail = "zero pivot while factoring A - B"; return SWR_ERR_ZERO_PIVOT; }
  return SWR_OK;
}

// ---- Krylov kernels ----------------------------------------------------------

int fetch(swr_handle *h, const double2 *dev, int n, double2 *host) {
  CK(cudaMemcpyAsync(host, dev, n * sizeof(double2), cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  return SWR_OK;
}

typedef std::function<int(const double2 *, double2 *)> Op;
// Fused form of a linear operator for GMRES: y = A(s x) and vcopy = s x,
// s = sp->x on the device (the new basis vector is normalised on load).
typedef std::function<int(const double2 *x, const double2 *sp, double2 *vcopy, double2 *y)> OpScaled;

// One fused Gram-Schmidt pass (dots / axpy / norm, see launch_cgs) on this
// rank's slots.  Every pass alternates its traversal direction (the first
// units of a pass meet the last ones of the previous pass in L2).  World > 1:
// the unit partials of all ranks are summed (disjoint columns, exact) and
// reduced in the one-GPU order.
int cgs(swr_handle *h, const double2 *V, int nv, const double2 *hsrc, double2 *w, int mode, double2 *out,
        double2 *out_host = nullptr) {
  h->cgs_dir ^= 1;
  if (h->cgs_dir) mode |= swr::CGS_REV;
  // the first basis vectors stay in L2 (persisting window; every pass reads them)
  const bool win = V && V == h->kout.V && h->vwin_bytes > 0;
  double2 *part = h->world > 1 ? h->part_send : h->partial;
  CK(swr::launch_cgs(V, h->nloc, nv, hsrc, w, mode, h->smap, part, h->st, win ? h->vwin_bytes : 0, h->vwin_ratio));
  h->n_launches++;
  const int nred = ((mode & swr::CGS_DOTS) ? nv : 0) + ((mode & swr::CGS_NORM) ? 1 : 0);
  const int nu = swr::cgs_units_global(h->smap);
  if (h->world > 1) {
    CKS(allreduce_sum(h, (const double *)h->part_send, (double *)h->part_recv, (size_t)2 * nred * nu));
    part = h->part_recv;
  }
  CK(swr::launch_cgs_reduce(part, nu, nred, mode, out, out_host, h->st));
  h->n_launches++;
  return SWR_OK;
}

int gmres(swr_handle *h, const Op &A, const double2 *b, double2 *x, double tol, int m, int maxit, Krylov &K,
          int *iters, std::vector<double> *hist, int *converged, bool speculate = true,
          const OpScaled *AS = nullptr) {
  const size_t n = h->nloc;
  const size_t ldv = n;
  double2 *V = K.V, *w = K.w;
  *iters = 0;
  *converged = 0;
  const int stride = 3 * (m + 2) + 8;
  auto O1 = [&](int par) { return K.dots + (size_t)par * stride; };
  auto O2 = [&](int par) { return K.dots + (size_t)par * stride + (m + 2); };
  auto O3 = [&](int par) { return K.dots + (size_t)par * stride + 2 * (m + 2); };
  auto HP = [&](int par) { return K.hp + (size_t)par * stride; };
  CKS(cgs(h, nullptr, 0, nullptr, const_cast<double2 *>(b), swr::CGS_NORM, O3(0)));
  CKS(fetch(h, O3(0), 1, HP(0) + 2 * (m + 2)));
  const double bnorm = std::sqrt(HP(0)[2 * (m + 2)].x);
  if (bnorm == 0.0) {
    CKS(fill_zero(h, x, n));
    *converged = 1;
    return SWR_OK;
  }
  std::vector<cplx> H((size_t)(m + 1) * m), sn(m), gam(m + 1), y(m);
  std::vector<double> cs(m);
  auto Hm = [&](int i, int k) -> cplx & { return H[(size_t)i * m + k]; };
  int total = 0, done = 0, st = SWR_OK;
  // device work of Arnoldi step k: w = A v_k, CGS2, v_{k+1} = w/||w||,
  // scalars -> pinned buffer (k & 1), event.  No host dependency, so step
  // k+1 is issued before the host reads step k's scalars.
  // fused path (AS): step k reads the raw vector left by step k-1 (or the
  // restart) in buf[(k + 1) & 1] with its 1/norm at sptr(k), writes
  // v_k = V_k = s x on the fly and w = A v_k into buf[k & 1]; no separate
  // normalisation pass
  double2 *buf[2] = {K.w, K.w2};
  auto sptr = [&](int k) -> const double2 * { return k == 0 ? O3(1) + 1 : O3((k - 1) & 1) + 1; };
  auto issue = [&](int k) -> int {
    const int par = k & 1;
    if (AS) w = buf[k & 1];
    int s = AS ? (*AS)(buf[(k + 1) & 1], sptr(k), V + (size_t)k * ldv, w) : A(V + (size_t)k * ldv, w);
    if (s && s != SWR_ERR_INNER_NOT_CONVERGED) return s;
    if (s) st = s;
    // scalars also go straight to the pinned mirror HP(par) (no copy node)
    CKS(cgs(h, V, k + 1, nullptr, w, swr::CGS_DOTS | swr::CGS_NORM, O1(par), HP(par)));              // h1, ||w||^2
    if (h->gs_passes == 2) {
      CKS(cgs(h, V, k + 1, O1(par), w, swr::CGS_AXPY | swr::CGS_DOTS, O2(par), HP(par) + (m + 2))); // w -= V h1; h2
      CKS(cgs(h, V, k + 1, O2(par), w, swr::CGS_AXPY | swr::CGS_NORM | swr::CGS_SCALE, O3(par),
              HP(par) + 2 * (m + 2)));                                                               // w -= V h2
    } else {
      CKS(cgs(h, V, k + 1, O1(par), w, swr::CGS_AXPY | swr::CGS_NORM | swr::CGS_SCALE, O3(par),
              HP(par) + 2 * (m + 2)));                                                               // w -= V h1
    }
    if (!AS) {
      CK(swr::launch_pdl(swr::k_scale_dev, dim3(grid_for(n)), dim3(256), 0, h->st, (const double2 *)w,
                         (const double2 *)(O3(par) + 1), V + (size_t)(k + 1) * ldv, n));
      h->n_launches++;
    }
    CK(cudaEventRecord(K.ev[par], h->st));
    return SWR_OK;
  };
  while (!done) {
    CKS(A(x, K.w));
    double2 *r0 = AS ? buf[1] : V;   // fused: raw r in buf[1], 1/beta at O3(1)+1 (sptr(0))
    CK(swr::launch_pdl(swr::k_sub, dim3(grid_for(n)), dim3(256), 0, h->st, b, (const double2 *)K.w, r0, n));
    h->n_launches++;
    const int rp = AS ? 1 : 0;
    CKS(cgs(h, nullptr, 0, nullptr, r0, swr::CGS_NORM | (AS ? swr::CGS_SCALE : 0), O3(rp)));
    CKS(fetch(h, O3(rp), 1, HP(0) + 2 * (m + 2)));
    const double beta = std::sqrt(HP(0)[2 * (m + 2)].x);
    if (beta <= tol * bnorm) { *converged = 1; break; }
    if (total >= maxit) break;
    if (!AS) {
      CK(swr::launch_pdl(swr::k_axpby, dim3(grid_for(n)), dim3(256), 0, h->st, make_double2(0, 0), (const double2 *)V,
                         make_double2(1.0 / beta, 0), V, n));
      h->n_launches++;
    }
    std::fill(gam.begin(), gam.end(), cplx(0));
    gam[0] = beta;
    int k, kend = 0;
    CKS(issue(0));
    for (k = 0; k < m; k++) {
      if (!speculate && k > 0) CKS(issue(k));                             // issue step k now
      if (speculate && k + 1 < m && total + 1 < maxit) CKS(issue(k + 1));  // or issue the next step ahead
      CK(cudaEventSynchronize(K.ev[k & 1]));
      const double2 *hp = HP(k & 1);
      total++;
      const double wn0 = std::sqrt(hp[k + 1].x);
      for (int i = 0; i <= k; i++) Hm(i, k) = h->gs_passes == 2 ? c2(hp[i]) + c2(hp[(m + 2) + i]) : c2(hp[i]);
      const double hk1 = std::sqrt(hp[2 * (m + 2)].x);
      const bool breakdown = hk1 <= 1e-14 * wn0;
      for (int i = 0; i < k; i++) {
        cplx t = cs[i] * Hm(i, k) + sn[i] * Hm(i + 1, k);
        Hm(i + 1, k) = -std::conj(sn[i]) * Hm(i, k) + cs[i] * Hm(i + 1, k);
        Hm(i, k) = t;
      }
      cplx a = Hm(k, k);
      double aa = std::abs(a);
      if (aa == 0.0) {
        cs[k] = 0.0;
        sn[k] = 1.0;
        Hm(k, k) = hk1;
      } else {
        double den = std::sqrt(aa * aa + hk1 * hk1);
        cs[k] = aa / den;
        sn[k] = (a / aa) * hk1 / den;
        Hm(k, k) = (a / aa) * den;
      }
      gam[k + 1] = -std::conj(sn[k]) * gam[k];
      gam[k] = cs[k] * gam[k];
      const double res = std::abs(gam[k + 1]);
      if (hist) hist->push_back(res);
      kend = k + 1;
      if (res <= tol * bnorm || breakdown) { *converged = 1; done = 1; break; }
      if (total >= maxit) { done = 1; break; }
    }
    for (int i = kend - 1; i >= 0; i--) {
      cplx acc = gam[i];
      for (int qq = i + 1; qq < kend; qq++) acc -= Hm(i, qq) * y[qq];
      y[i] = acc / Hm(i, i);
    }
    CK(cudaStreamSynchronize(h->st));  // retire speculative work before reusing the pinned buffer
    double2 *hy = HP(0);
    for (int i = 0; i < kend; i++) hy[i] = d2(y[i]);
    CK(cudaMemcpyAsync(K.ycoef, hy, kend * sizeof(double2), cudaMemcpyHostToDevice, h->st));
    CK(swr::launch_pdl(swr::k_multi_update, dim3(grid_for(n)), dim3(256), 0, h->st, (const double2 *)V, ldv, kend,
                       (const double2 *)K.ycoef, x, n));
    h->n_launches++;
    CK(cudaStreamSynchronize(h->st));
  }
  *iters = total;
  return st;
}

// y = (I - L) x or (I - L0) x on this rank's slots: the FFT convolution
// (N_T <= 512) or the direct causal convolution; xs (device, optional): the
// input is xs->x times x and vcopy receives that scaled input (register FFT
// only: the GMRES step normalises its new basis vector on load).  Across a
// rank cut the neighbour computes -(L x) of our first / last slot and we add
// our own (scaled) x after the exchange.
int apply_toeplitz(swr_handle *h, bool zero, const double2 *x, const double2 *xs, double2 *vcopy, double2 *y) {
  if (h->N < 2) return SWR_OK;
  CKS(record_pair(h, EV_INTF, true));
  const double2 *F = zero ? h->FX0 : h->FX;
  if (h->log4 && h->fft_reg) {
    CK(swr::launch_fft_conv_reg(F, x, y, h->smap, h->tw, h->st, xs, vcopy));
  } else if (xs) {
    g_detail = "scaled Toeplitz apply needs the register FFT";
    return SWR_ERR_UNSUPPORTED;
  } else if (h->log4) {
    CK(swr::launch_fft_conv(h->log4, F, x, y, h->smap, h->tw, h->st));
  } else {
    const double2 *X = zero ? h->X0 : h->X;
    const int G = (h->NT + swr::TR - 1) / swr::TR;
    const int thr = (2 * ((G + 1) / 2) + 31) / 32 * 32;
    const size_t smem = (4 * ((size_t)h->NT + 3 * swr::TR) + 2 * ((size_t)h->NT + swr::TR)) * sizeof(double2);
    if (smem > 48 * 1024) CK(cudaFuncSetAttribute(swr::k_toeplitz_I_minus_L, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    swr::k_toeplitz_I_minus_L<<<h->j_hi - h->j_lo + 1, thr, smem, h->st>>>(X, x, y, h->smap);
  }
  CK(cudaGetLastError());
  h->n_launches++;
  CKS(record_pair(h, EV_INTF, false));
  if (h->world > 1) {
    CKS(exchange_cut(h, h->hrecvL, h->hrecvR));
    const int NT = h->NT;
    // (vcopy is complete: every owned slot is an input of an owned subdomain)
    if (h->rank > 0) {
      swr::k_halo_add<<<(NT + 127) / 128, 128, 0, h->st>>>(x, h->hrecvL, y, NT, xs);
      h->n_launches++;
    }
    if (h->rank < h->world - 1) {
      const size_t o = (size_t)(h->s_hi - h->s_lo) * NT;
      swr::k_halo_add<<<(NT + 127) / 128, 128, 0, h->st>>>(x + o, h->hrecvR, y + o, NT, xs);
      h->n_launches++;
    }
    CK(cudaGetLastError());
  }
  return SWR_OK;
}

int apply_I_minus_L(swr_handle *h, bool zero, const double2 *x, double2 *y) {
  return apply_toeplitz(h, zero, x, nullptr, nullptr, y);
}

// Fused GMRES operator (register FFT path only): y = (I - L)(s x), vcopy = s x.
int apply_I_minus_L_scaled(swr_handle *h, bool zero, const double2 *x, const double2 *sp, double2 *vcopy, double2 *y) {
  return apply_toeplitz(h, zero, x, sp, vcopy, y);
}

// transforms of this rank's first columns, once per build
int transform_columns(swr_handle *h, bool zero) {
  if (!h->log4) return SWR_OK;
  const size_t o = (size_t)(h->j_lo - 1) * 4;
  const size_t NF = (size_t)1 << (2 * h->log4);
  CK(swr::launch_fft_fwd(h->log4, (zero ? h->X0 : h->X) + o * h->NT, h->NT, 4 * (h->j_hi - h->j_lo + 1), h->NT, h->tw,
                         (zero ? h->FX0 : h->FX) + o * NF, h->st));
  h->n_launches++;
  return SWR_OK;
}

// x = P^{-1} y: GMRES on (I - L0) x = y from x = 0 (eq. Pxg, reading A8)
// BiCGStab in the oracle's order (van der Vorst; reading A20): r, rh, p, v,
// s, t live in basis slots 0..5 of K; the scalars come back to the host at
// each half step (the method's own decisions: alpha, omega, the stops).
int bicgstab(swr_handle *h, const Op &A, const double2 *b, double2 *x, double tol, int maxit, Krylov &K, int *iters,
             std::vector<double> *hist, int *converged) {
  const size_t n = h->nloc;
  double2 *r = K.V, *rh = K.V + n, *p = K.V + 2 * n, *v = K.V + 3 * n, *sv = K.V + 4 * n, *t = K.V + 5 * n;
  double2 *dv = K.dots, *hp = K.hp;
  const dim3 g(grid_for(n)), bl(256);
  *iters = 0;
  *converged = 0;
  CKS(cgs(h, nullptr, 0, nullptr, const_cast<double2 *>(b), swr::CGS_NORM, dv));
  CKS(fetch(h, dv, 1, hp));
  const double bnorm = std::sqrt(hp[0].x);
  if (bnorm == 0.0) {
    CKS(fill_zero(h, x, n));
    *converged = 1;
    return SWR_OK;
  }
  int st = SWR_OK;
  auto op = [&](const double2 *in, double2 *out) -> int {
    int s = A(in, out);
    if (s && s != SWR_ERR_INNER_NOT_CONVERGED) return s;
    if (s) st = s;
    return SWR_OK;
  };
  CKS(op(x, r));
  CK(swr::launch_pdl(swr::k_lin2, g, bl, 0, h->st, r, make_double2(1, 0), b, make_double2(-1, 0), (const double2 *)r, n));
  CK(cudaMemcpyAsync(rh, r, n * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
  h->n_launches++;
  // rho = <rh, r>, ||r||^2
  CKS(cgs(h, rh, 1, nullptr, r, swr::CGS_DOTS | swr::CGS_NORM, dv));
  CKS(fetch(h, dv, 2, hp));
  if (std::sqrt(hp[1].x) <= tol * bnorm) { *converged = 1; return st; }
  cplx rho = c2(hp[0]), rho_old = 1.0, alpha = 1.0, omega = 1.0;
  for (int it = 0; it < maxit; it++) {
    if (rho == 0.0) return SWR_ERR_BREAKDOWN;
    if (it == 0) {
      CK(cudaMemcpyAsync(p, r, n * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
    } else {
      const cplx beta = (rho / rho_old) * (alpha / omega);
      CK(swr::launch_pdl(swr::k_bicg_p, g, bl, 0, h->st, p, (const double2 *)r, (const double2 *)v, d2(beta), d2(omega), n));
      h->n_launches++;
    }
    CKS(op(p, v));
    CKS(cgs(h, rh, 1, nullptr, v, swr::CGS_DOTS, dv));                 // <rh, v>
    CKS(fetch(h, dv, 1, hp));
    const cplx rv = c2(hp[0]);
    if (rv == 0.0) return SWR_ERR_BREAKDOWN;
    alpha = rho / rv;
    CK(swr::launch_pdl(swr::k_lin2, g, bl, 0, h->st, sv, make_double2(1, 0), (const double2 *)r, d2(-alpha),
                       (const double2 *)v, n));                             // s = r - alpha v
    h->n_launches++;
    CKS(cgs(h, nullptr, 0, nullptr, sv, swr::CGS_NORM, dv));
    CKS(fetch(h, dv, 1, hp));
    *iters = it + 1;
    const double sn = std::sqrt(hp[0].x);
    if (sn <= tol * bnorm) {
      CK(swr::launch_pdl(swr::k_axpby, g, bl, 0, h->st, d2(alpha), (const double2 *)p, make_double2(1, 0), x, n));
      h->n_launches++;
      if (hist) hist->push_back(sn);
      *converged = 1;
      break;
    }
    CKS(op(sv, t));
    CKS(cgs(h, sv, 2, nullptr, t, swr::CGS_DOTS, dv));                 // <s, t>, <t, t> (s, t adjacent)
    CKS(fetch(h, dv, 2, hp));
    const cplx ts = std::conj(c2(hp[0])), tt = c2(hp[1]);
    if (tt == 0.0) return SWR_ERR_BREAKDOWN;
    omega = ts / tt;
    CK(swr::launch_pdl(swr::k_bicg_xr, g, bl, 0, h->st, x, r, (const double2 *)p, (const double2 *)sv,
                       (const double2 *)t, d2(alpha), d2(omega), n));
    h->n_launches++;
    rho_old = rho;
    CKS(cgs(h, rh, 1, nullptr, r, swr::CGS_DOTS | swr::CGS_NORM, dv));  // next rho, ||r||^2
    CKS(fetch(h, dv, 2, hp));
    const double rn = std::sqrt(hp[1].x);
    if (hist) hist->push_back(rn);
    if (rn <= tol * bnorm) { *converged = 1; break; }
    if (omega == 0.0) return SWR_ERR_BREAKDOWN;
    rho = c2(hp[0]);
  }
  return st;
}

// Exact P^{-1} (reading A27): block-Jacobi sweeps on the lag-0 system of
// every step.  rho = max_i ||D_i^{-1} C_i||_inf over the interfaces bounds
// the contraction; S sweeps leave an error <= rho^{S+1} ||x||_inf <= 1e-17.
int setup_pinv(swr_handle *h) {
  const int N = h->N, NT = h->NT;
  if (N < 2) return SWR_OK;
  std::vector<double2> l0((size_t)N * 4);
  CK(cudaMemcpy2DAsync(l0.data(), sizeof(double2), h->X0, (size_t)NT * sizeof(double2), sizeof(double2),
                       (size_t)N * 4, cudaMemcpyDeviceToHost, h->st));
  CK(cudaStreamSynchronize(h->st));
  auto X = [&](int j, int c) { return c2(l0[(size_t)(j - 1) * 4 + c]); };   // X^{j,c+1}_0
  double rho = 0.0;
  for (int i = 1; i <= N - 1; i++) {
    const cplx p = X(i + 1, 0), q = X(i, 3), det = 1.0 - p * q;
    if (std::abs(det) == 0.0) { g_detail = "exact P^{-1}: singular lag-0 interface block"; return SWR_ERR_UNSUPPORTED; }
    const cplx d00 = 1.0 / det, d01 = p / det, d10 = q / det, d11 = 1.0 / det;
    const double ca = (i + 1 <= N - 1) ? std::abs(X(i + 1, 1)) : 0.0, cb = (i >= 2) ? std::abs(X(i, 2)) : 0.0;
    rho = std::max(rho, std::max(std::abs(d00) * ca + std::abs(d01) * cb, std::abs(d10) * ca + std::abs(d11) * cb));
  }
  int S = 0;
  if (rho > 0.0) {
    if (rho >= 0.5) { g_detail = "exact P^{-1}: lag-0 interface coupling too strong (rho >= 0.5)"; return SWR_ERR_UNSUPPORTED; }
    S = std::max(0, (int)std::ceil(std::log(1e-17) / std::log(rho)) - 1);
  }
  h->pinv_sweeps = S;
  h->pinv_rho = rho;
  return SWR_OK;
}

int apply_Pinv(swr_handle *h, const double2 *y, double2 *x) {
  if (h->pinv_exact) {
    // the forward substitution in time couples every interface at every step:
    // on multi-GPU runs it is replicated on the whole vector (every rank holds
    // L0), gathered by one sum of zero-padded slices, and each rank keeps its
    // own slots
    const size_t off = (size_t)h->s_lo * h->NT;
    const double2 *yf = y;
    double2 *xf = x;
    if (h->world > 1) {
      CKS(fill_zero(h, h->pinv_y, h->ng));
      CK(cudaMemcpyAsync(h->pinv_y + off, y, h->nloc * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
      CKS(allreduce_sum(h, (const double *)h->pinv_y, (double *)h->pinv_y, 2 * h->ng));
      yf = h->pinv_y;
      xf = h->pinv_x;
    }
    int nl = 0;
    CKS(record_pair(h, EV_INTF, true));
    CK(swr::launch_pinv_causal(h->X0, yf, xf, h->pinvF, h->N, h->NT, h->pinv_sweeps, h->st, &nl));
    CKS(record_pair(h, EV_INTF, false));
    h->n_launches += nl;
    if (h->world > 1)
      CK(cudaMemcpyAsync(x, h->pinv_x + off, h->nloc * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
    return SWR_OK;
  }
  CKS(fill_zero(h, x, h->nloc));
  Op A0 = [h](const double2 *a, double2 *b) { return apply_I_minus_L(h, true, a, b); };
  OpScaled A0s = [h](const double2 *a, const double2 *sp, double2 *vc, double2 *b) {
    return apply_I_minus_L_scaled(h, true, a, sp, vc, b);
  };
  int it = 0, conv = 0;
  int s = h->krylov == SWR_KRY_BICGSTAB
              ? bicgstab(h, A0, y, x, h->tol_inner, h->maxit_inner, h->kin, &it, nullptr, &conv)
              : gmres(h, A0, y, x, h->tol_inner, h->restart, h->maxit_inner, h->kin, &it, nullptr, &conv, true,
                      h->N >= 2 && h->log4 && h->fft_reg ? &A0s : nullptr);
  h->inner_total += it;
  if (!conv) h->inner_fail = true;
  return s;
}

// The L / L0 first columns by impulse probing, with d = R(0; u0)
// in the same launch (NEW): per owned subdomain the d system and the l_j / r_j
// unit-impulse probes.  L0 (V = 0, PRECOND): the probes of an interior
// subdomain do not depend on j (same matrix, u0 = 0; reading A14), so only
// the three distinct subdomains j = 1, 2, N march and the interior columns
// are copied -- bitwise what probing every subdomain gives -- and every rank
// holds all of L0 (the exact P^{-1} needs it on multi-GPU runs).
int build_probes(swr_handle *h, bool zero, double2 *X, double2 *dvec) {
  std::vector<MarchSys> sys;
  const int N = h->N, NT = h->NT;
  int nreal = 0;
  CKS(fill_zero(h, X, (size_t)N * 4 * NT));
  if (dvec) CKS(fill_zero(h, dvec, h->nloc));
  std::vector<int> js;
  if (zero) {
    js.push_back(1);
    if (N >= 3) js.push_back(2);
    js.push_back(N);
  } else {
    for (int j = h->j_lo; j <= h->j_hi; j++) js.push_back(j);
  }
  for (int j : js) {
    double2 *Xj = X + (size_t)(j - 1) * 4 * NT;
    const MarchSys blank = make_sys(h, j, nullptr, false, zero, nullptr, nullptr);
    if (dvec) { sys.push_back(make_sys(h, j, nullptr, true, zero, dvec, nullptr)); nreal++; }
    if (j >= 2) {  // l_{j,1} = 1 -> X^{j,1} (out_left), X^{j,3} (out_right)
      MarchSys s = blank;
      s.flags |= swr::SYS_LIN_IMPULSE;
      s.out_left = Xj + 0 * NT;
      s.out_right = (j <= N - 1) ? Xj + 2 * NT : nullptr;
      sys.push_back(s);
      nreal++;
    }
    if (j <= N - 1) {  // r_{j,1} = 1 -> X^{j,2}, X^{j,4}
      MarchSys s = blank;
      s.flags |= swr::SYS_RIN_IMPULSE;
      s.out_left = (j >= 2) ? Xj + 1 * NT : nullptr;
      s.out_right = Xj + 3 * NT;
      sys.push_back(s);
      nreal++;
    }
  }
  CKS(run_march(h, sys, nreal));
  if (zero && N >= 4) {   // interior columns j = 3..N-1 := those of j = 2
    const size_t blk = (size_t)4 * NT;
    swr::k_replicate<<<grid_for(blk * (N - 3)), 256, 0, h->st>>>(X + blk, X + 2 * blk, blk, (size_t)(N - 3));
    CK(cudaGetLastError());
    h->n_launches++;
  }
  if (dvec) CKS(exchange_cut(h, dvec, last_slot(h, dvec)));
  return SWR_OK;
}

// Final sweep and u(T) on the global mesh; multi-GPU: every rank fills its
// nodes (half of each copy at a node shared with a neighbour rank) and the
// sum over ranks lands on rank 0.
int final_sweep(swr_handle *h, const double2 *g) {
  CKS(sweep_R(h, g, true, false, nullptr, h->uloc));
  swr::k_gather_uT<<<grid_for(h->Nx + 1), 256, 0, h->st>>>(h->uloc, h->N, h->m, h->Nj, h->j_lo, h->j_hi, h->uT);
  CK(cudaGetLastError());
  h->n_launches++;
  if (h->world > 1) {
    CKS(record_pair(h, EV_COMM, true));
    CKS(h->comm->reduce_sum_root((double *)h->uT, (size_t)2 * (h->Nx + 1), h->st));
    CKS(record_pair(h, EV_COMM, false));
    h->n_launches++;
  }
  return SWR_OK;
}

int copy_in(double2 *dst, const double *src, size_t n, bool on_dev, cudaStream_t st) {
  CK(cudaMemcpyAsync(dst, src, n * sizeof(double2), on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  return SWR_OK;
}
int copy_in_r(double *dst, const double *src, size_t n, bool on_dev, cudaStream_t st) {
  CK(cudaMemcpyAsync(dst, src, n * sizeof(double), on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
  return SWR_OK;
}

int alloc_krylov(Krylov &K, size_t mm, size_t ng) {
  const size_t stride = 3 * (mm + 1) + 8;
  int s;
  if ((s = dalloc(&K.V, mm * ng)) || (s = dalloc(&K.w, ng)) || (s = dalloc(&K.dots, 2 * stride)) ||
      (s = dalloc(&K.ycoef, mm)) || (s = dalloc(&K.w2, ng)))
    return s;
  if (cudaMallocHost((void **)&K.hp, 2 * stride * sizeof(double2)) != cudaSuccess) return SWR_ERR_OOM;
  for (int i = 0; i < 2; i++)
    if (cudaEventCreateWithFlags(&K.ev[i], cudaEventDisableTiming) != cudaSuccess) return SWR_ERR_CUDA;
  return SWR_OK;
}

// Persisting-L2 set-aside (device-wide limit): raised by the first live
// handle of a device, restored (and the persisting lines reset) when the
// last one is freed, so it does not leak into other work of the process.
struct L2State { int users = 0; size_t prev = 0; };
std::mutex g_l2_mu;
std::map<int, L2State> g_l2;

void l2_acquire(int dev, size_t want) {
  std::lock_guard<std::mutex> lk(g_l2_mu);
  L2State &S = g_l2[dev];
  if (S.users++ == 0) cudaDeviceGetLimit(&S.prev, cudaLimitPersistingL2CacheSize);
  size_t cur = 0;
  cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
  if (want > cur) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
  cudaGetLastError();
}

void l2_release(int dev) {
  std::lock_guard<std::mutex> lk(g_l2_mu);
  L2State &S = g_l2[dev];
  if (S.users > 0 && --S.users == 0) {
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, S.prev);
    cudaGetLastError();
  }
}

void free_all(swr_handle *h) {
  void *ptrs[] = {h->pinvF, h->u0, h->Vx, h->beta, h->q, h->q0, h->er, h->er0, h->d, h->X, h->X0, h->g, h->g0,
                  h->uloc, h->uT, h->tmp, h->tmp2, h->rhs, h->partial, h->tw, h->FX, h->FX0,
                  h->tau, h->xi, h->qtd, h->ertd, h->fp_stat,
                  h->sys_dev, h->err_dev, h->jobs_dev,
                  h->sst_u, h->sst_z, h->sst_a, h->sst_q, h->sst_e, h->sst_b, h->sst_vals, h->sst_flags, h->kap, h->pinv_y, h->pinv_x,
                  h->haloL, h->haloR, h->hrecvL, h->hrecvR, h->part_send, h->part_recv, h->hv_nl, h->snl_ze, h->snl_vals, h->snl_flags};
  for (void *p : ptrs)
    if (p) cudaFree(p);
  for (Krylov *K : {&h->kout, &h->kin}) {
    for (void *p : {(void *)K->V, (void *)K->w, (void *)K->dots, (void *)K->ycoef, (void *)K->w2})
      if (p) cudaFree(p);
    if (K->hp) cudaFreeHost(K->hp);
    for (int i = 0; i < 2; i++)
      if (K->ev[i]) cudaEventDestroy(K->ev[i]);
  }
  if (h->hpin) cudaFreeHost(h->hpin);
  for (cudaEvent_t e : {h->ev_b0, h->ev_b1, h->ev_s0, h->ev_s1, h->ev_in0, h->ev_in1})
    if (e) cudaEventDestroy(e);
  if (h->st_in) cudaStreamDestroy(h->st_in);
  for (auto *vec : {&h->march_ev, &h->intf_ev, &h->comm_ev})
    for (auto &e : *vec) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
  delete h->comm;
  h->comm = nullptr;
  if (h->l2_window) l2_release(h->device);
  h->l2_window = 0;
}

}  // namespace

extern "C" {

const char *swr_error_string(int s) {
  switch (s) {
    case SWR_OK: return "ok";
    case SWR_ERR_INVALID_ARG: return "invalid argument";
    case SWR_NOT_CONVERGED: return "not converged (outputs hold the last iterate)";
    case SWR_ERR_ZERO_PIVOT: return "zero pivot: A - B is singular";
    case SWR_ERR_BREAKDOWN: return "Krylov breakdown";
    case SWR_ERR_INNER_NOT_CONVERGED: return "inner iteration (P^-1 GMRES or NL fixed point) not converged";
    case SWR_ERR_UNSUPPORTED: return "unsupported combination";
    case SWR_ERR_CUDA: return "CUDA error";
    case SWR_ERR_NCCL: return "NCCL error";
    case SWR_ERR_OOM: return "out of device memory";
    default: return "unknown status";
  }
}

const char *swr_last_error_detail(void) { return g_detail.c_str(); }

int swr_partition(int32_t N, int32_t world, int32_t rank, int32_t *j_lo, int32_t *j_hi) {
  if (N < 1 || world < 1 || world > N || rank < 0 || rank >= world || !j_lo || !j_hi) return SWR_ERR_INVALID_ARG;
  *j_lo = (int32_t)(((int64_t)rank * N) / world) + 1;
  *j_hi = (int32_t)(((int64_t)(rank + 1) * N) / world);
  return SWR_OK;
}

int swr_owned_slots(int32_t N, int32_t world, int32_t rank, int32_t *s_lo, int32_t *s_hi) {
  int32_t jl, jh;
  CKS(swr_partition(N, world, rank, &jl, &jh));
  if (!s_lo || !s_hi || N < 2) return SWR_ERR_INVALID_ARG;
  *s_lo = swr::slot_first(jl);
  *s_hi = swr::slot_last(jh, N);
  return SWR_OK;
}

int swr_nccl_unique_id(void *out) {
  if (!out) return SWR_ERR_INVALID_ARG;
  CKS(load_nccl());
  if (!g_nccl.getUniqueId) { g_detail = "ncclGetUniqueId missing"; return SWR_ERR_NCCL; }
  ncclUniqueId_t id;
  if (g_nccl.getUniqueId(&id) != 0) { g_detail = "ncclGetUniqueId failed"; return SWR_ERR_NCCL; }
  memcpy(out, &id, sizeof id);
  return SWR_OK;
}

int swr_loopback_id(void *out, int32_t world) {
  if (!out || world < 1) return SWR_ERR_INVALID_ARG;
  static unsigned long long next = 1;
  std::lock_guard<std::mutex> lk(g_loop_mu);
  const unsigned long long gid = next++;
  auto grp = std::make_shared<LoopGroup>();
  grp->world = world;
  grp->a.assign(world, nullptr);
  grp->b.assign(world, nullptr);
  g_loop_groups[gid] = grp;
  memset(out, 0, 128);
  memcpy(out, kLoopMagic, 8);
  memcpy((char *)out + 8, &gid, sizeof gid);
  return SWR_OK;
}

int swr_sizes(const swr_handle *h, int32_t *Nx, int32_t *NT, int32_t *Nj, int64_t *ng) {
  if (!h) return SWR_ERR_INVALID_ARG;
  if (Nx) *Nx = h->Nx;
  if (NT) *NT = h->NT;
  if (Nj) *Nj = h->Nj;
  if (ng) *ng = (int64_t)h->ng;
  return SWR_OK;
}

int swr_setup(const swr_config *cfg, swr_handle **out) {
  const auto t_start = std::chrono::steady_clock::now();
  g_detail.clear();
  if (!out) return SWR_ERR_INVALID_ARG;
  *out = nullptr;
  if (!cfg || !cfg->u0 || !(cfg->dx > 0) || !(cfg->dt > 0) || !(cfg->T > 0) || cfg->N < 1 || !(cfg->b0 > cfg->a0)) {
    g_detail = "bad geometry or missing u0";
    return SWR_ERR_INVALID_ARG;
  }
  const long Nx = std::lround((cfg->b0 - cfg->a0) / cfg->dx), NT = std::lround(cfg->T / cfg->dt);
  if (Nx < 1 || NT < 1 || Nx % cfg->N != 0) { g_detail = "N must divide N_x"; return SWR_ERR_INVALID_ARG; }
  if (cfg->world < 1 || cfg->world > cfg->N || cfg->rank < 0 || cfg->rank >= cfg->world) {
    g_detail = "bad rank/world";
    return SWR_ERR_INVALID_ARG;
  }
  if (cfg->transmission == SWR_TC_ROBIN && !(cfg->robin_p > 0)) { g_detail = "Robin needs p > 0"; return SWR_ERR_INVALID_ARG; }
  if (cfg->transmission < SWR_TC_ROBIN || cfg->transmission > SWR_TC_S2_4) return SWR_ERR_INVALID_ARG;
  if ((cfg->transmission == SWR_TC_S2_2 || cfg->transmission == SWR_TC_S2_4) && cfg->pade_m < 1) {
    g_detail = "the Pade operators need pade_m >= 1";
    return SWR_ERR_INVALID_ARG;
  }
  if (cfg->transmission >= SWR_TC_S0_3 &&
      (!(cfg->potential == SWR_POT_ZERO || cfg->potential == SWR_POT_VX) || cfg->algorithm == SWR_ALG_PRECOND)) {
    g_detail = "orders above S0^2 need a time-independent potential and the NEW or CLASSICAL algorithm";
    return SWR_ERR_INVALID_ARG;
  }
  if (cfg->potential < 0 || cfg->potential > 3) return SWR_ERR_INVALID_ARG;
  if (cfg->algorithm == SWR_ALG_NEW && !(cfg->potential == SWR_POT_ZERO || cfg->potential == SWR_POT_VX)) {
    g_detail = "NEW needs a time-independent linear potential (P:1015)";
    return SWR_ERR_INVALID_ARG;
  }
  if (cfg->krylov < 0 || cfg->krylov > 2 || cfg->algorithm < 0 || cfg->algorithm > 2) return SWR_ERR_INVALID_ARG;
  if (cfg->restart > 31) { g_detail = "GMRES restart must be <= 31"; return SWR_ERR_INVALID_ARG; }
  if (cfg->algorithm == SWR_ALG_CLASSICAL && cfg->potential == SWR_POT_CUBIC && cfg->krylov != SWR_KRY_FIXED_POINT) {
    g_detail = "the classical Krylov algorithm needs an affine R (linear potential, P:734)";
    return SWR_ERR_INVALID_ARG;
  }
  if (cfg->potential == SWR_POT_VX && !cfg->V_x) return SWR_ERR_INVALID_ARG;
  if (cfg->potential == SWR_POT_VTX_SEPARABLE && (cfg->n_terms < 1 || !cfg->tau || !cfg->xi)) {
    g_detail = "V(t,x) needs n_terms >= 1, tau and xi";
    return SWR_ERR_INVALID_ARG;
  }
  if (cfg->march_form < 0 || cfg->march_form > 1 || cfg->toeplitz_form < 0 || cfg->toeplitz_form > 2 ||
      !(cfg->nl_rows_per_thread == 0 || cfg->nl_rows_per_thread == 8 || cfg->nl_rows_per_thread == 11 ||
        cfg->nl_rows_per_thread == 16)) {
    g_detail = "march_form in {0,1}, toeplitz_form in {0,1,2}, nl_rows_per_thread in {0,8,11,16}";
    return SWR_ERR_INVALID_ARG;
  }

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) { g_detail = "no CUDA device"; return SWR_ERR_CUDA; }
  CK(cudaSetDevice(cfg->device));
  swr_handle *h = new swr_handle();
  h->a0 = cfg->a0; h->b0 = cfg->b0; h->T = cfg->T; h->dx = cfg->dx; h->dt = cfg->dt;
  h->lambda = cfg->lambda; h->robin_p = cfg->robin_p; h->tol = cfg->tol > 0 ? cfg->tol : 1e-10;
  h->tol_inner = cfg->tol_inner > 0 ? cfg->tol_inner : 1e-12; h->tol_fp = cfg->tol_fp > 0 ? cfg->tol_fp : 1e-12;
  h->N = cfg->N; h->potential = cfg->potential; h->transmission = cfg->transmission; h->algorithm = cfg->algorithm;
  h->restart = cfg->restart > 0 ? cfg->restart : 30; h->maxit = cfg->maxit > 0 ? cfg->maxit : 2000;
  h->gs_passes = cfg->gs_passes == 2 ? 2 : 1;
  h->krylov = cfg->krylov;
  h->pade_m = cfg->pade_m;
  h->pinv_exact = cfg->pinv_exact ? 1 : 0;
  h->march_form = cfg->march_form;
  h->toeplitz_form = cfg->toeplitz_form;
  h->nl_rows = cfg->nl_rows_per_thread;
  h->maxit_inner = cfg->maxit_inner > 0 ? cfg->maxit_inner : 2000; h->maxit_fp = cfg->maxit_fp > 0 ? cfg->maxit_fp : 50;
  h->n_terms = cfg->n_terms;
  h->Nx = (int)Nx; h->NT = (int)NT; h->m = (int)(Nx / cfg->N); h->Nj = h->m + 1;
  h->ng = (size_t)(2 * h->N - 2) * h->NT;
  h->rank = cfg->rank; h->world = cfg->world; h->device = cfg->device;
  swr_partition(h->N, h->world, h->rank, &h->j_lo, &h->j_hi);
  h->s_lo = h->N >= 2 ? swr::slot_first(h->j_lo) : 0;
  h->s_hi = h->N >= 2 ? swr::slot_last(h->j_hi, h->N) : -1;
  h->nloc = h->N >= 2 ? (size_t)(h->s_hi - h->s_lo + 1) * h->NT : 0;
  h->st = (cudaStream_t)cfg->cuda_stream;
  auto fail = [&](int s) { free_all(h); delete h; return s; };
  if (h->world > 1) {
    if (!cfg->nccl_unique_id) { delete h; g_detail = "world > 1 needs a communicator id"; return SWR_ERR_NCCL; }
    if (memcmp(cfg->nccl_unique_id, kLoopMagic, 8) == 0) {
      unsigned long long gid;
      memcpy(&gid, (const char *)cfg->nccl_unique_id + 8, sizeof gid);
      std::shared_ptr<LoopGroup> grp;
      {
        std::lock_guard<std::mutex> lk(g_loop_mu);
        auto it = g_loop_groups.find(gid);
        if (it != g_loop_groups.end()) grp = it->second;
      }
      if (!grp || grp->world != h->world) { delete h; g_detail = "unknown loopback group"; return SWR_ERR_NCCL; }
      auto *lc = new LoopbackComm();
      lc->grp = grp;
      lc->rank = h->rank;
      lc->world = h->world;
      h->comm = lc;
    } else {
      if (load_nccl() != 0) { delete h; return SWR_ERR_NCCL; }
      ncclUniqueId_t id;
      memcpy(&id, cfg->nccl_unique_id, sizeof id);
      auto *nc = new NcclComm();
      nc->rank = h->rank;
      nc->world = h->world;
      if (g_nccl.commInitRank(&nc->comm, h->world, id, h->rank) != 0) {
        delete nc;
        delete h;
        g_detail = "ncclCommInitRank failed";
        return SWR_ERR_NCCL;
      }
      h->comm = nc;
    }
  }
  // transmission constants: c2 = e^{-i pi/4} sqrt(2/dt) = (1-i)/sqrt(dt)
  const double sq = std::sqrt(h->dt);
  h->c2v = make_double2(1.0 / sq, -1.0 / sq);
  h->c0 = (h->transmission == SWR_TC_ROBIN) ? make_double2(0.0, -h->robin_p) : h->c2v;  // beta_0 = 1
  h->tc_hi = h->transmission >= SWR_TC_S0_3;
  h->kappa = (2.0 / h->dt) * (h->dx / 6.0);
  h->eim = (2.0 / h->dt) * (h->dx / 6.0);
  h->shape = swr::choose_march_shape(h->Nj, h->NT, h->tc_hi);
  if (h->march_form == 1 || h->shape.M == 0 || swr::march_smem_bytes(h->shape, h->NT, true, h->tc_hi) > 227 * 1024) {
    // too large for a resident cluster (or asked for): stream the state through HBM
    h->stream_march = true;
    h->shape = {1, 256, 1, 1};
  }
  int s;
  const size_t nx1 = (size_t)h->Nx + 1, ng = h->ng, nloc = h->nloc, NTt = h->NT;
  const bool precond = h->algorithm == SWR_ALG_PRECOND;
  if ((s = dalloc(&h->u0, nx1)) || (s = dalloc(&h->beta, NTt + 1)) || (s = dalloc(&h->q, (size_t)h->N * h->Nj)) ||
      (s = dalloc(&h->er, (size_t)h->N * h->Nj)) || (s = dalloc(&h->uloc, (size_t)h->N * h->Nj)) ||
      (s = dalloc(&h->uT, nx1)) || (s = dalloc(&h->sys_dev, (size_t)4 * h->N + 8)) || (s = dalloc(&h->err_dev, 1)))
    return fail(s);
  if (h->potential == SWR_POT_VX && (s = dalloc(&h->Vx, nx1))) return fail(s);
  if (h->potential == SWR_POT_VTX_SEPARABLE) {
    const size_t nt = (size_t)h->n_terms;
    if ((s = dalloc(&h->tau, nt * (NTt + 1))) || (s = dalloc(&h->xi, nt * nx1)) ||
        (s = dalloc(&h->qtd, NTt * (size_t)h->N * h->Nj)) || (s = dalloc(&h->ertd, NTt * (size_t)h->N * h->Nj + 2)))
      return fail(s);
    // the march's bulk copies of er round up to 16 B: the last one reads one pad element
    if (cudaMemsetAsync(h->ertd + NTt * (size_t)h->N * h->Nj, 0, 2 * sizeof(double), h->st) != cudaSuccess)
      return fail(SWR_ERR_CUDA);
    if ((s = copy_in_r(h->tau, cfg->tau, nt * (NTt + 1), cfg->inputs_on_device, h->st)) ||
        (s = copy_in_r(h->xi, cfg->xi, nt * nx1, cfg->inputs_on_device, h->st)))
      return fail(s);
  }
  if (h->stream_march) {
    h->sst_cap = 3 * h->N + 2;   // the largest batched march (3 RHS per subdomain in the build)
    const size_t nslot = kStreamSlots;   // chain CTAs of one launch, upper bound
    // the two-pass form's interleaved layout pads each system to sst_stride rows
    h->sst_stride = std::max((size_t)h->Nj, swr::stream2_stride(h->Nj, h->N, h->NT));
    const size_t sn = (size_t)h->sst_cap * h->sst_stride;
    if ((s = dalloc(&h->sst_u, sn)) || (s = dalloc(&h->sst_z, sn)) || (s = dalloc(&h->sst_a, sn)) ||
        (s = dalloc(&h->sst_q, sn)) || (s = dalloc(&h->sst_e, sn)) || (s = dalloc(&h->sst_b, sn)) ||
        (s = dalloc(&h->sst_vals, nslot * 8)))
      return fail(s);
    if (cudaMalloc((void **)&h->sst_flags, nslot * 3 * sizeof(int)) != cudaSuccess) return fail(SWR_ERR_OOM);
  }
  if ((s = dalloc(&h->fp_stat, 2))) return fail(s);
  if (cudaMemset(h->fp_stat, 0, 2 * sizeof(int)) != cudaSuccess) return fail(SWR_ERR_CUDA);
  h->shape_nl = swr::choose_march_shape_nl(h->Nj, h->nl_rows, h->j_hi - h->j_lo + 1);
  if (h->potential == SWR_POT_CUBIC) {
    if (h->march_form == 1 || h->shape_nl.M == 0 ||
        swr::march_nl_smem_bytes(h->shape_nl, h->NT, false) > 227 * 1024) {
      // beyond the resident NL march (or asked for): stream through HBM
      if (!h->stream_march) { g_detail = "NL streaming march without the streaming scratch"; return fail(SWR_ERR_UNSUPPORTED); }
      h->nl_stream = true;
      if ((s = dalloc(&h->snl_ze, (size_t)h->sst_cap * h->sst_stride)) ||
          (s = dalloc(&h->snl_vals, (size_t)kStreamSlots * 10)))
        return fail(s);
      if (cudaMalloc((void **)&h->snl_flags, (size_t)kStreamSlots * 4 * sizeof(int)) != cudaSuccess)
        return fail(SWR_ERR_OOM);
    }
    if ((s = dalloc(&h->hv_nl, (size_t)(h->j_hi - h->j_lo + 1) * 2 * (NTt + 1)))) return fail(s);
  }
  if (precond && ((s = dalloc(&h->q0, (size_t)3 * h->Nj)) || (s = dalloc(&h->er0, (size_t)3 * h->Nj)))) return fail(s);
  if (ng) {
    const size_t mm = std::max(h->restart + 1, 6);   // BiCGStab uses 6 of the basis slots
    if ((s = dalloc(&h->d, nloc)) || (s = dalloc(&h->X, (size_t)h->N * 4 * NTt)) || (s = dalloc(&h->g, nloc)) ||
        (s = alloc_krylov(h->kout, mm, nloc)) || (s = dalloc(&h->tmp, nloc)) || (s = dalloc(&h->tmp2, nloc)) ||
        (s = dalloc(&h->rhs, nloc)) || (s = dalloc(&h->partial, (mm + 2) * (size_t)(2 * h->N))))
      return fail(s);
    if (precond && ((s = dalloc(&h->X0, (size_t)h->N * 4 * NTt)) || (s = alloc_krylov(h->kin, mm, nloc))))
      return fail(s);
    if (precond && h->pinv_exact && (s = dalloc(&h->pinvF, (size_t)(2 * h->N - 2) * swr::PINV_B))) return fail(s);
    if (cfg->g0 && (s = dalloc(&h->g0, nloc))) return fail(s);
    if (h->world > 1) {
      if ((s = dalloc(&h->haloL, NTt)) || (s = dalloc(&h->haloR, NTt)) || (s = dalloc(&h->hrecvL, NTt)) ||
          (s = dalloc(&h->hrecvR, NTt)) || (s = dalloc(&h->part_send, (mm + 2) * (size_t)(2 * h->N))) ||
          (s = dalloc(&h->part_recv, (mm + 2) * (size_t)(2 * h->N))))
        return fail(s);
      if (precond && h->pinv_exact && ((s = dalloc(&h->pinv_y, ng)) || (s = dalloc(&h->pinv_x, ng)))) return fail(s);
      // the other ranks' columns of the partials stay 0 (this rank writes its own only)
      if (cudaMemset(h->part_send, 0, (mm + 2) * (size_t)(2 * h->N) * sizeof(double2)) != cudaSuccess)
        return fail(SWR_ERR_CUDA);
    }
    h->smap = {h->N, h->NT, h->j_lo, h->j_hi, h->s_lo, h->s_hi, h->haloL, h->haloR};
    // (I - L) apply: FFT convolution for N_T <= 512 (register form for NF =
    // 1024), the direct causal convolution beyond or when asked for
    h->log4 = h->toeplitz_form == 1 ? 0 : swr::fft_log4_for(h->NT);
    h->fft_reg = h->log4 == 5 && h->toeplitz_form == 0;
    if (h->log4) {
      const size_t NF = (size_t)1 << (2 * h->log4);
      if ((s = dalloc(&h->tw, NF)) || (s = dalloc(&h->FX, (size_t)h->N * 4 * NF)) ||
          (precond && (s = dalloc(&h->FX0, (size_t)h->N * 4 * NF))))
        return fail(s);
      // set aside L2 for this rank's transformed columns, re-read by every (I - L)
      // apply, and for the first 4 outer basis vectors, read by every CGS pass
      // (measured: 0 / 3 / 4 / 5 / 6 / 8 vectors -> C5 solve 94.2 / 93.0 / 92.6 /
      // 93.6 / 96.4 / 96.9 ms: more set-aside starves the streamed vectors)
      int maxp = 0;
      cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, h->device);
      const size_t fxb = (size_t)(h->j_hi - h->j_lo + 1) * 4 * NF * sizeof(double2);
      const size_t vb = (size_t)4 * nloc * sizeof(double2);
      h->l2_window = std::max<size_t>(1, std::min((size_t)maxp, fxb + vb));
      l2_acquire(h->device, h->l2_window);
      if ((size_t)maxp > fxb) {
        h->vwin_bytes = vb;
        h->vwin_ratio = (float)std::min(1.0, (double)((size_t)maxp - fxb) / (double)vb);
      }
      if (getenv("SWR_VERBOSE"))
        fprintf(stderr, "L2 persisting: max %d B, FX %zu B, V window %zu B ratio %.3f\n", maxp, fxb, h->vwin_bytes,
                h->vwin_ratio);
      swr::k_twiddles<<<(unsigned)((NF + 255) / 256), 256, 0, h->st>>>(h->tw, (int)NF);
      if (cudaGetLastError() != cudaSuccess) return fail(SWR_ERR_CUDA);
    }
  } else {
    h->smap = {h->N, h->NT, h->j_lo, h->j_hi, 0, -1, nullptr, nullptr};
  }
  if (cudaMallocHost((void **)&h->hpin, sizeof(double2) * (3 * (h->restart + 1) + 16)) != cudaSuccess) return fail(SWR_ERR_OOM);
  if (cudaEventCreate(&h->ev_b0) || cudaEventCreate(&h->ev_b1) || cudaEventCreate(&h->ev_s0) || cudaEventCreate(&h->ev_s1) ||
      cudaEventCreateWithFlags(&h->ev_in0, cudaEventDisableTiming) ||
      cudaEventCreateWithFlags(&h->ev_in1, cudaEventDisableTiming) ||
      cudaStreamCreateWithFlags(&h->st_in, cudaStreamNonBlocking))
    return fail(SWR_ERR_CUDA);
  const bool od = cfg->inputs_on_device != 0;
  if ((s = copy_in(h->u0, cfg->u0, nx1, od, h->st))) return fail(s);
  if (h->Vx && (s = copy_in_r(h->Vx, cfg->V_x, nx1, od, h->st))) return fail(s);
  // g0: this rank's slots of the full initial interface vector
  if (h->g0 && (s = copy_in(h->g0, cfg->g0 + 2 * (size_t)h->s_lo * h->NT, nloc, od, h->st))) return fail(s);
  // beta_s: alpha_0 = 1, alpha_{2k} = alpha_{2k-2}(2k-1)/(2k), alpha_{2k+1} = alpha_{2k}
  {
    std::vector<double> al(NTt + 1), be(NTt + 1);
    for (size_t sidx = 0; sidx <= NTt; sidx++) {
      double a = sidx == 0 ? 1.0 : (sidx % 2 ? al[sidx - 1] : al[sidx - 2] * (double)(sidx - 1) / (double)sidx);
      al[sidx] = a;
      be[sidx] = (sidx % 2) ? -a : a;
    }
    if (cudaMemcpy(h->beta, be.data(), (NTt + 1) * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
      return fail(SWR_ERR_CUDA);
  }
  if ((s = factor_matrices(h))) return fail(s);
  if (cudaStreamSynchronize(h->st) != cudaSuccess) return fail(SWR_ERR_CUDA);
  h->t_setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_start).count();
  *out = h;
  return SWR_OK;
}

int swr_update_inputs(swr_handle *h, const double *u0, const double *V_x, int32_t on_device) {
  if (!h) return SWR_ERR_INVALID_ARG;
  const size_t nx1 = (size_t)h->Nx + 1;
  // host u0 together with a new V_x: u0's copy runs on a side stream, after
  // the handle stream's earlier work (which may still read u0), overlapping
  // V_x's copy and the factorisation (V_x is issued first: copies queue on the
  // copy engine in issue order).  C5: 3.3 -> 1.8 ms, now bound by the copies.
  const bool overlap = u0 && V_x && h->Vx && !on_device && h->st_in;
  if (V_x && h->Vx) CKS(copy_in_r(h->Vx, V_x, nx1, on_device, h->st));
  if (overlap) {
    CK(cudaEventRecord(h->ev_in0, h->st));
    CK(cudaStreamWaitEvent(h->st_in, h->ev_in0, 0));
    CKS(copy_in(h->u0, u0, nx1, false, h->st_in));
    CK(cudaEventRecord(h->ev_in1, h->st_in));
  } else if (u0) {
    CKS(copy_in(h->u0, u0, nx1, on_device, h->st));
  }
  if (V_x && h->Vx) {
    CKS(factor_matrices(h));
    h->have_L = false;
  }
  if (overlap) CK(cudaStreamWaitEvent(h->st, h->ev_in1, 0));
  // host buffers are free for reuse on return (the copies are done)
  if (!on_device && (u0 || (V_x && h->Vx))) CK(cudaStreamSynchronize(h->st));
  h->have_d = false;
  return SWR_OK;
}

int swr_build_interface_operator(swr_handle *h) {
  if (!h) return SWR_ERR_INVALID_ARG;
  h->march_ev_used = h->intf_ev_used = h->comm_ev_used = 0;
  h->n_marches = h->n_launches = 0;
  h->cell_steps = 0;
  CK(cudaEventRecord(h->ev_b0, h->st));
  if (h->N > 1) {
    if (h->algorithm == SWR_ALG_NEW) {
      CKS(build_probes(h, false, h->X, h->d));    // 3 RHS per interior subdomain
      CKS(transform_columns(h, false));
      h->have_L = h->have_d = true;
    } else if (h->algorithm == SWR_ALG_CLASSICAL) {
      if (h->krylov != SWR_KRY_FIXED_POINT) {      // Algorithm 2: d = R(0; u0)
        CKS(sweep_R(h, nullptr, true, false, h->d, nullptr));
        h->have_d = true;
      }
    } else {
      CKS(build_probes(h, true, h->X0, nullptr));  // L0: the probes of j = 1, 2, N
      CKS(transform_columns(h, true));
      h->have_L0 = true;
      if (h->pinv_exact) CKS(setup_pinv(h));
      if (h->potential != SWR_POT_CUBIC) {
        CKS(sweep_R(h, nullptr, true, false, h->d, nullptr));  // d = R(0; u0)
        h->have_d = true;
      }
    }
  }
  CK(cudaEventRecord(h->ev_b1, h->st));
  h->build_timed = true;
  return SWR_OK;
}

int swr_solve(swr_handle *h, double *u_T, int32_t u_T_on_device, swr_report *rep) {
  if (!h) return SWR_ERR_INVALID_ARG;
  if (!h->build_timed) {
    h->march_ev_used = h->intf_ev_used = h->comm_ev_used = 0;
    h->n_marches = h->n_launches = 0;
    h->cell_steps = 0;
  }
  CK(cudaEventRecord(h->ev_s0, h->st));
  h->hist.clear();
  h->cgs_dir = 0;   // the same pass directions (and rounding) on every solve
  h->iterations = h->inner_total = h->fp_max = 0;
  h->converged = 1;
  h->inner_fail = false;
  CK(cudaMemsetAsync(h->fp_stat, 0, 2 * sizeof(int), h->st));
  int st = SWR_OK;
  if (h->N > 1) {
    if (h->g0) CK(cudaMemcpyAsync(h->g, h->g0, h->nloc * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
    else CKS(fill_zero(h, h->g, h->nloc));
    int it = 0, conv = 0;
    double2 *hp = h->hpin;
    // fixed point driver: g <- next(g), stop at ||g^{k+1} - g^k||_2 < tol (A5, A21);
    // next() leaves the increment g^{k+1} - g^k in h->tmp2
    auto fixed_point = [&](const std::function<int()> &next) -> int {
      while (it < h->maxit) {
        const int s2 = next();
        if (s2 && s2 != SWR_ERR_INNER_NOT_CONVERGED) return s2;
        CKS(cgs(h, nullptr, 0, nullptr, h->tmp2, swr::CGS_NORM, h->kout.dots));
        CKS(fetch(h, h->kout.dots, 1, hp));
        const double diff = std::sqrt(hp[0].x);
        h->hist.push_back(diff);
        it++;
        if (diff < h->tol) { conv = 1; break; }
      }
      return SWR_OK;
    };
    const dim3 gg(grid_for(h->nloc)), bb(256);
    if (h->algorithm == SWR_ALG_NEW) {
      if (!h->have_L || !h->have_d) CKS(swr_build_interface_operator(h));
      Op A = [h](const double2 *a, double2 *b) { return apply_I_minus_L(h, false, a, b); };
      OpScaled As = [h](const double2 *a, const double2 *sp, double2 *vc, double2 *b) {
        return apply_I_minus_L_scaled(h, false, a, sp, vc, b);
      };
      if (h->krylov == SWR_KRY_FIXED_POINT) {
        // g <- d + L g = g + (d - (I - L) g)
        st = fixed_point([&]() -> int {
          CKS(apply_I_minus_L(h, false, h->g, h->tmp));
          CK(swr::launch_pdl(swr::k_lin2, gg, bb, 0, h->st, h->tmp2, make_double2(1, 0), (const double2 *)h->d,
                             make_double2(-1, 0), (const double2 *)h->tmp, h->nloc));
          CK(swr::launch_pdl(swr::k_axpby, gg, bb, 0, h->st, make_double2(1, 0), (const double2 *)h->tmp2,
                             make_double2(1, 0), h->g, h->nloc));
          h->n_launches += 2;
          return SWR_OK;
        });
      } else if (h->krylov == SWR_KRY_BICGSTAB) {
        st = bicgstab(h, A, h->d, h->g, h->tol, h->maxit, h->kout, &it, &h->hist, &conv);
      } else {
        st = gmres(h, A, h->d, h->g, h->tol, h->restart, h->maxit, h->kout, &it, &h->hist, &conv, true,
                   h->N >= 2 && h->log4 && h->fft_reg ? &As : nullptr);
      }
    } else if (h->algorithm == SWR_ALG_CLASSICAL) {
      if (h->krylov == SWR_KRY_FIXED_POINT) {
        // Algorithm 1: g <- R(g) (with u0; R_nl for f(u))
        st = fixed_point([&]() -> int {
          CKS(sweep_R(h, h->g, true, false, h->tmp, nullptr));
          swr::k_sub<<<gg, bb, 0, h->st>>>(h->tmp, h->g, h->tmp2, h->nloc);
          CK(cudaGetLastError());
          CK(cudaMemcpyAsync(h->g, h->tmp, h->nloc * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
          h->n_launches++;
          return SWR_OK;
        });
      } else {
        // Algorithm 2: Krylov on (I - L) g = d, (I - L) g = g - R_0(g) matrix-free
        if (!h->have_d) CKS(swr_build_interface_operator(h));
        Op A = [h](const double2 *a, double2 *b) -> int {
          CKS(sweep_R(h, a, false, false, h->tmp, nullptr));
          swr::k_sub<<<grid_for(h->nloc), 256, 0, h->st>>>(a, h->tmp, b, h->nloc);
          CK(cudaGetLastError());
          h->n_launches++;
          return SWR_OK;
        };
        st = h->krylov == SWR_KRY_BICGSTAB
                 ? bicgstab(h, A, h->d, h->g, h->tol, h->maxit, h->kout, &it, &h->hist, &conv)
                 : gmres(h, A, h->d, h->g, h->tol, h->restart, h->maxit, h->kout, &it, &h->hist, &conv, true);
      }
    } else if (h->potential == SWR_POT_CUBIC || h->krylov == SWR_KRY_FIXED_POINT) {
      // preconditioned fixed point (eq. chp2_algopd_NL, reading A9):
      // g <- g - P^{-1}(g - R(g)), stop at ||g^{k+1} - g^k||_2 < tol (A5)
      if (!h->have_L0) CKS(swr_build_interface_operator(h));
      st = fixed_point([&]() -> int {
        CKS(sweep_R(h, h->g, true, false, h->tmp, nullptr));
        swr::k_sub<<<gg, bb, 0, h->st>>>(h->g, h->tmp, h->tmp2, h->nloc);
        CK(cudaGetLastError());
        const int s2 = apply_Pinv(h, h->tmp2, h->tmp);
        if (s2 && s2 != SWR_ERR_INNER_NOT_CONVERGED) return s2;
        swr::k_axpby<<<gg, bb, 0, h->st>>>(make_double2(-1.0, 0.0), h->tmp, make_double2(1.0, 0.0), h->g, h->nloc);
        CK(cudaGetLastError());
        // increment g^{k+1} - g^k = -P^{-1}(...): same norm as h->tmp
        CK(cudaMemcpyAsync(h->tmp2, h->tmp, h->nloc * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
        h->n_launches += 2;
        return s2;
      });
    } else {
      if (!h->have_L0 || !h->have_d) CKS(swr_build_interface_operator(h));
      CKS(apply_Pinv(h, h->d, h->rhs));
      Op A = [h](const double2 *a, double2 *b) -> int {
        CKS(sweep_R(h, a, false, false, h->tmp, nullptr));
        swr::k_sub<<<grid_for(h->nloc), 256, 0, h->st>>>(a, h->tmp, h->tmp2, h->nloc);
        CK(cudaGetLastError());
        return apply_Pinv(h, h->tmp2, b);
      };
      // the operator runs an inner Krylov solve (host round trips): no
      // speculation, which would also run inner solves the oracle does not
      st = h->krylov == SWR_KRY_BICGSTAB
               ? bicgstab(h, A, h->rhs, h->g, h->tol, h->maxit, h->kout, &it, &h->hist, &conv)
               : gmres(h, A, h->rhs, h->g, h->tol, h->restart, h->maxit, h->kout, &it, &h->hist, &conv, false);
    }
    if (st && st != SWR_ERR_INNER_NOT_CONVERGED) return st;
    h->iterations = it;
    h->converged = conv;
    h->have_g = true;
  }
  CKS(final_sweep(h, h->N > 1 ? h->g : nullptr));
  CK(cudaEventRecord(h->ev_s1, h->st));
  if (u_T && h->rank == 0)
    CK(cudaMemcpyAsync(u_T, h->uT, ((size_t)h->Nx + 1) * sizeof(double2),
                       u_T_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, h->st));
  // NL fixed-point statistics of all ranks' marches (max iterations, failure)
  if (h->world > 1) CKS(h->comm->allreduce_max_i32(h->fp_stat, 2, h->st));
  CK(cudaStreamSynchronize(h->st));
  {
    int fs[2] = {0, 0};
    CK(cudaMemcpy(fs, h->fp_stat, sizeof fs, cudaMemcpyDeviceToHost));
    h->fp_max = fs[0];
    if (fs[1]) h->inner_fail = true;
  }
  if (rep) {
    memset(rep, 0, sizeof(*rep));
    rep->iterations = h->iterations;
    rep->inner_iterations = h->inner_total;
    rep->fp_max = h->fp_max;
    rep->converged = h->converged;
    rep->residual_history = h->hist.data();
    rep->n_history = (int)h->hist.size();
    float ms = 0;
    if (h->build_timed && cudaEventElapsedTime(&ms, h->ev_b0, h->ev_b1) == cudaSuccess) rep->t_build_ms = ms;
    if (cudaEventElapsedTime(&ms, h->ev_s0, h->ev_s1) == cudaSuccess) rep->t_solve_ms = ms;
    rep->t_march_ms = sum_pairs(h, EV_MARCH);
    rep->t_interface_ms = sum_pairs(h, EV_INTF);
    rep->t_comm_ms = sum_pairs(h, EV_COMM);
    rep->t_setup_ms = h->t_setup_ms;
    rep->cell_steps = h->cell_steps;
    rep->n_marches = h->n_marches;
    rep->n_kernel_launches = h->n_launches;
  }
  h->build_timed = false;
  if (!h->converged) return SWR_NOT_CONVERGED;
  if (h->inner_fail) return SWR_ERR_INNER_NOT_CONVERGED;
  return st;
}

void swr_free(swr_handle *h) {
  if (!h) return;
  cudaStreamSynchronize(h->st);
  free_all(h);
  delete h;
}

int swr_apply_R(swr_handle *h, const double *g, int32_t use_u0, int32_t force_zero_potential, double *Rg,
                double *u_T) {
  if (!h || h->N < 1 || h->world > 1) return SWR_ERR_INVALID_ARG;
  if (force_zero_potential && !h->q0) return SWR_ERR_UNSUPPORTED;
  CKS(sweep_R(h, (const double2 *)g, use_u0 != 0, force_zero_potential != 0, (double2 *)Rg,
              u_T ? h->uloc : nullptr));
  if (u_T) {
    swr::k_gather_uT<<<grid_for(h->Nx + 1), 256, 0, h->st>>>(h->uloc, h->N, h->m, h->Nj, h->j_lo, h->j_hi,
                                                             (double2 *)u_T);
    CK(cudaGetLastError());
  }
  CK(cudaStreamSynchronize(h->st));
  return SWR_OK;
}

int swr_apply_I_minus_L(swr_handle *h, int32_t which, const double *x, double *y) {
  if (!h || h->world > 1) return SWR_ERR_INVALID_ARG;
  if ((which == 0 && !h->have_L) || (which == 1 && !h->have_L0)) return SWR_ERR_INVALID_ARG;
  CKS(apply_I_minus_L(h, which == 1, (const double2 *)x, (double2 *)y));
  CK(cudaStreamSynchronize(h->st));
  return SWR_OK;
}

int swr_get_interface(swr_handle *h, int32_t which, double *d, double *X) {
  if (!h || h->world > 1) return SWR_ERR_INVALID_ARG;
  if (d && h->have_d) CK(cudaMemcpyAsync(d, h->d, h->ng * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
  const double2 *src = which ? h->X0 : h->X;
  if (X && src) CK(cudaMemcpyAsync(X, src, (size_t)h->N * 4 * h->NT * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  return SWR_OK;
}

int swr_set_interface(swr_handle *h, const double *d, const double *X) {
  if (!h || h->world > 1 || h->algorithm != SWR_ALG_NEW || h->N < 2 || !d || !X) return SWR_ERR_INVALID_ARG;
  CK(cudaMemcpyAsync(h->d, d, h->ng * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
  CK(cudaMemcpyAsync(h->X, X, (size_t)h->N * 4 * h->NT * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
  CKS(transform_columns(h, false));
  h->have_L = h->have_d = true;
  CK(cudaStreamSynchronize(h->st));
  return SWR_OK;
}

int swr_get_g(swr_handle *h, double *g) {
  if (!h || !h->have_g) return SWR_ERR_INVALID_ARG;
  CK(cudaMemcpyAsync(g, h->g, h->nloc * sizeof(double2), cudaMemcpyDeviceToDevice, h->st));
  CK(cudaStreamSynchronize(h->st));
  return SWR_OK;
}

}  // extern "C"

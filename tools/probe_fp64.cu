// Microbenchmarks used to size the march kernel: FP64 FMA throughput,
// dependent-DFMA latency, L2-resident and HBM streaming bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

template<int ILP>
__global__ void dfma_tput(double* out, int iters, double a, double b) {
  double x[ILP];
  for (int i = 0; i < ILP; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < ILP; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0; for (int i = 0; i < ILP; i++) s += x[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_lat(double* out, int iters, double a, double b, long long* cyc) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) x = fma(x, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; }
  if (x == 12345.678) out[0] = x;
}
__global__ void rcp_lat(double* out, int iters, long long* cyc) {
  double x = 1.5 + threadIdx.x;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) x = 1.0 / x + 0.5;
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  if (x == 12345.678) out[0] = x;
}
__global__ void readbw(const double2* __restrict__ p, size_t n, double* out) {
  double2 acc = {0, 0};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcg(p + i); acc.x += v.x; acc.y += v.y;
  }
  if (acc.x == 12345.678) out[0] = acc.y;
}
__global__ void copybw(const double2* __restrict__ p, double2* __restrict__ q, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) q[i] = p[i];
}
int main() {
  cudaDeviceProp pr; CK(cudaGetDeviceProperties(&pr, 0));
  printf("gpu %s sms %d l2 %d MB smem/blk optin %zu regs/sm %d clock %d kHz\n", pr.name, pr.multiProcessorCount, pr.l2CacheSize>>20, pr.sharedMemPerBlockOptin, pr.regsPerMultiprocessor, pr.clockRate);
  double* out; CK(cudaMalloc(&out, 64)); long long* cyc; CK(cudaMalloc(&cyc, 64));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; float ms;
  for (int bs : {256, 512}) {
    int grid = pr.multiProcessorCount * (2048 / bs);
    dfma_tput<8><<<grid, bs>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0); dfma_tput<8><<<grid, bs>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)grid * bs;
    printf("dfma tput bs=%d: %.2f TFLOP/s (%.3f ms)\n", bs, fl / ms / 1e9, ms);
  }
  long long h;
  dfma_lat<<<1, 32>>>(out, iters, 1.0000001, 1e-9, cyc); CK(cudaDeviceSynchronize());
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("dfma dependent latency %.2f cyc\n", (double)h / iters);
  rcp_lat<<<1, 32>>>(out, 2000, cyc); CK(cudaDeviceSynchronize());
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost); printf("1/x+0.5 dependent latency %.2f cyc\n", (double)h / 2000);
  for (size_t mb : {32, 64, 96, 4096}) {
    size_t n = mb * (1 << 20) / 16; double2 *p, *q; CK(cudaMalloc(&p, n * 16)); CK(cudaMalloc(&q, n * 16)); cudaMemset(p, 0, n*16);
    int grid = pr.multiProcessorCount * 4;
    for (int w = 0; w < 3; w++) readbw<<<grid, 512>>>(p, n, out);
    cudaEventRecord(e0); for (int r = 0; r < 10; r++) readbw<<<grid, 512>>>(p, n, out); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("read %zu MB: %.1f GB/s\n", mb, 10.0 * n * 16 / ms / 1e6);
    for (int w = 0; w < 3; w++) copybw<<<grid, 512>>>(p, q, n);
    cudaEventRecord(e0); for (int r = 0; r < 10; r++) copybw<<<grid, 512>>>(p, q, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("copy %zu MB: %.1f GB/s (r+w)\n", mb, 10.0 * 2 * n * 16 / ms / 1e6);
    cudaFree(p); cudaFree(q);
  }
  return 0;
}

// Resident clusters of a 1-CTA-per-SM kernel (256 threads, ~200 KB shared
// memory) for cluster sizes 1..16 (GPC packing on this GPU).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 1) k_dummy(int *x) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (x) x[blockIdx.x] = s[(threadIdx.x + 1) & 255];
}
int main() {
  const size_t smem = 200 * 1024;
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int cs = 1; cs <= 16; cs++) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    int ncl = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, (void *)k_dummy, &cfg);
    printf("CS %2d: %3d clusters resident = %3d of %d SMs%s\n", cs, ncl, ncl * cs, nsm, e ? " (error)" : "");
  }
  return 0;
}

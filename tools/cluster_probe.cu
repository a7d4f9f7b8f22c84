#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  extern __shared__ char sm[];
  if (threadIdx.x == 0) out[blockIdx.x] = 1;
  sm[threadIdx.x] = 0;
}
int main() {
  int* out; cudaMalloc(&out, 4096);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(148 / cs * cs); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[2];
    a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    a[1].id = cudaLaunchAttributeCooperative; a[1].val.cooperative = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int nclusters = -1;
    cudaError_t e1 = cudaOccupancyMaxActiveClusters(&nclusters, k, &cfg);
    cfg.numAttrs = 2;
    cudaError_t e2 = cudaLaunchKernelEx(&cfg, k, out);
    cudaError_t e3 = cudaDeviceSynchronize();
    printf("cluster %d: max active clusters %d (%s) -> CTAs %d; coop launch of %d CTAs: %s / %s\n", cs, nclusters,
           cudaGetErrorString(e1), nclusters * cs, 148 / cs * cs, cudaGetErrorString(e2), cudaGetErrorString(e3));
  }
  return 0;
}

// How many thread-block clusters of 2 / 4 / 8 / 16 CTAs (one CTA per SM:
// ~200 KB dynamic smem, as the tcgen05 GEMMs) the B200 places at once
// (cudaOccupancyMaxActiveClusters).  Diagnostics for DESIGN.md §9.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dummy(int* p) {
  extern __shared__ int s[];
  if (p) p[blockIdx.x] = s[threadIdx.x];
}

int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = cs;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k_dummy, &cfg);
    printf("cluster %2d: %3d clusters -> %3d of %d SMs (%s)\n", cs, n, n * cs, sms, cudaGetErrorString(e));
  }
  return 0;
}

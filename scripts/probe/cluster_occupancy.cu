// Probe: co-resident clusters of size c (1 CTA/SM via ~200 KB dynamic smem) on this GPU.
#include <cstdio>
__global__ void k() {}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int c : {1, 2, 3, 4, 5, 6, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * 64);
    cfg.blockDim = dim3(192);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute at;
    at.id = cudaLaunchAttributeClusterDimension;
    at.val.clusterDim.x = c; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
    cfg.attrs = &at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: %3d clusters -> %3d SMs (%s)\n", c, n, n * c, cudaGetErrorString(e));
  }
  return 0;
}

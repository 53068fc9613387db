#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(1,1,1) dummy() {}
__global__ void k16() {}
int main() {
  for (int cs : {4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs, 64, 1); cfg.blockDim = dim3(512, 1, 1);
    cfg.dynamicSmemBytes = 150 * 1024;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    cudaFuncSetAttribute(k16, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    cudaFuncSetAttribute(k16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k16, &cfg);
    printf("cluster %d: max active clusters %d (%s)\n", cs, n, cudaGetErrorString(e));
  }
  return 0;
}

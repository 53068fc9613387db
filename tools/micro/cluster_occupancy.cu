// Co-resident clusters of a given size (one 512-thread CTA per SM, ~200 KB
// shared memory each): cudaOccupancyMaxActiveClusters for sizes 1..16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cluster_occupancy cluster_occupancy.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k16() {}
int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  for (int smem_kb : {100, 200}) {
    for (int cs = 1; cs <= 16; ++cs) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 64, 1); cfg.blockDim = dim3(512, 1, 1);
      cfg.dynamicSmemBytes = smem_kb * 1024;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr; cfg.numAttrs = 1;
      cudaFuncSetAttribute(k16, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_kb * 1024);
      cudaFuncSetAttribute(k16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k16, &cfg);
      printf("smem %d KB cluster %2d: max active clusters %3d = %3d CTAs (%s)\n", smem_kb, cs, n, n * cs,
             cudaGetErrorString(e));
    }
  }
  return 0;
}

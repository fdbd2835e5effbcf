// How many 2-CTA clusters (1 CTA per SM, ~200 KB smem) can be co-resident?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(2, 1, 1) k2(int* p) { if (p) p[blockIdx.x] = 1; }
__global__ void k4(int* p) { if (p) p[blockIdx.x] = 1; }
int main() {
  for (int smem : {100 * 1024, 200 * 1024}) {
    for (int cs : {2, 4}) {
      cudaFuncSetAttribute(k4, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      cudaFuncSetAttribute(k4, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148 * 4);
      cfg.blockDim = dim3(320);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k4, &cfg);
      printf("smem %d KB cluster %d: max active clusters %d (%s) -> %d CTAs\n", smem / 1024, cs, n,
             cudaGetErrorString(e), n * cs);
    }
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
}

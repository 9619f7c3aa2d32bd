// How many clusters of size 1/2/4/8 of a 1-CTA/SM kernel (448 threads,
// ~220 KB smem) can be co-resident on this GPU (cudaOccupancyMaxActiveClusters)?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(448, 1) dummy(int* p) { extern __shared__ int s[]; if (p) p[0] = s[0]; }
int main() {
  const int smem = 220 * 1024;
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int cl : {1, 2, 3, 4, 6, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cl * 64);
    cfg.blockDim = dim3(448);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d of %d SMs (%s)\n", cl, n, n * cl, sms, cudaGetErrorString(e));
  }
  return 0;
}

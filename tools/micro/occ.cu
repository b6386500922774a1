#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(){}
int main(){
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220*1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1,2,4,8}) {
    cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(148); cfg.blockDim = dim3(384); cfg.dynamicSmemBytes = 200*1024;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = cs; a[0].val.clusterDim.y=1; a[0].val.clusterDim.z=1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
    printf("cluster %d: max active clusters %d (%s) -> CTAs %d\n", cs, n, cudaGetErrorString(e), n*cs);
  }
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0); printf("SMs %d\n", p.multiProcessorCount);
}

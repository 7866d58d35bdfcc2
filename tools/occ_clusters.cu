// How many clusters of a given size fit on the GPU at once (1 CTA per SM:
// 1024 threads, ~200 KB dynamic shared memory) — cudaOccupancyMaxActiveClusters.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* p) { extern __shared__ double s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main() {
  cudaDeviceProp pr; cudaGetDeviceProperties(&pr, 0);
  printf("SMs %d\n", pr.multiProcessorCount);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cl : {1, 2, 4, 6, 8, 9, 10, 11, 12, 13, 14, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 64); cfg.blockDim = dim3(1024); cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = cl; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
    printf("cluster %2d: max active clusters %3d -> %3d SMs (%s)\n", cl, n, n * cl, cudaGetErrorString(e));
  }
}

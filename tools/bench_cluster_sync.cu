// microbenchmark: cost of cluster.sync() vs cluster size / block size (sm_100a)
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) cl.sync();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}
__global__ void kb(int iters, unsigned long long* out) {   // arrive.relaxed + wait (no acquire/release)
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *out = (t1 - t0) / iters;
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 8);
  for (int csz : {1, 2, 4, 8, 11, 16}) for (int bs : {128, 256, 512, 1024}) for (int relaxed : {0, 1}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(csz); cfg.blockDim = dim3(bs);
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = csz; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    if (relaxed) { cudaFuncSetAttribute(kb, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); cudaLaunchKernelEx(&cfg, kb, 2000, d); }
    else { cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); cudaLaunchKernelEx(&cfg, k, 2000, d); }
    unsigned long long h = 0; cudaError_t e = cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("cluster %2d block %4d %s: %llu cycles/sync (%s)\n", csz, bs, relaxed ? "relaxed" : "cg.sync", h, cudaGetErrorString(e));
  }
}

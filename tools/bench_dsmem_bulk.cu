// microbenchmark: moving a Jacobi block pair (~96 KB) to the next CTA of a
// 16-CTA cluster — TMA bulk push into the neighbour's shared memory
// (cp.async.bulk.shared::cluster, mbarrier complete_tx) vs the L2 round trip
// the kernel uses (bulk store to global, cluster barrier, bulk load).
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned r) {
  unsigned o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void wait_bar(unsigned long long* bar, unsigned ph) {
  unsigned done = 0;
  long long spins = 0;
  while (!done && spins < (1ll << 26)) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(sa(bar)), "r"(ph) : "memory");
    ++spins;
  }
}

__global__ void push(int bytes, int chunks, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* src = sm;
  unsigned char* dst = sm + bytes;
  __shared__ __align__(8) unsigned long long bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned r = cl.block_rank(), CL = cl.num_blocks(), nxt = (r + 1) % CL;
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) src[i] = (unsigned char)(i + r);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cl.sync();
  const long long t0 = clock64();
  if (threadIdx.x == 0) {
    const int cb = bytes / chunks;
    for (int c = 0; c < chunks; ++c)
      asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(mapa(sa(dst + c * cb), nxt)), "r"(sa(src + c * cb)), "r"(cb), "r"(mapa(sa(&bar), nxt))
                   : "memory");
  }
  if (threadIdx.x == 0) wait_bar(&bar, 0);
  __syncthreads();
  const long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

__global__ void l2trip(int bytes, int chunks, unsigned char* g, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  unsigned char* src = sm;
  unsigned char* dst = sm + bytes;
  __shared__ __align__(8) unsigned long long bar;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned r = cl.block_rank(), CL = cl.num_blocks(), prv = (r + CL - 1) % CL;
  unsigned char* gme = g + (size_t)(blockIdx.x) * bytes;
  unsigned char* gprv = g + (size_t)(blockIdx.x - r + prv) * bytes;
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) src[i] = (unsigned char)(i + r);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  cl.sync();
  const long long t0 = clock64();
  const int cb = bytes / chunks;
  if (threadIdx.x == 0) {
    for (int c = 0; c < chunks; ++c)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gme + c * cb), "r"(sa(src + c * cb)), "r"(cb) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __threadfence();
  cl.sync();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes) : "memory");
    for (int c = 0; c < chunks; ++c)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(sa(dst + c * cb)), "l"(gprv + c * cb), "r"(cb), "r"(sa(&bar)) : "memory");
    wait_bar(&bar, 0);
  }
  __syncthreads();
  const long long t1 = clock64();
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 16 * 8);
  unsigned char* g; cudaMalloc(&g, 16 * 128 * 1024);
  for (int bytes : {49152, 98304}) for (int chunks : {1, 12, 24}) for (int mode : {0, 1}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16); cfg.blockDim = dim3(224);
    cfg.dynamicSmemBytes = 2 * bytes;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = 16; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    cudaError_t e;
    if (mode == 0) {
      cudaFuncSetAttribute(push, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(push, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * bytes);
      e = cudaLaunchKernelEx(&cfg, push, bytes, chunks, d);
    } else {
      cudaFuncSetAttribute(l2trip, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(l2trip, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * bytes);
      e = cudaLaunchKernelEx(&cfg, l2trip, bytes, chunks, g, d);
    }
    unsigned long long h[16] = {};
    cudaError_t e2 = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0, sum = 0;
    for (int i = 0; i < 16; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    printf("%s bytes %6d chunks %2d: mean %llu max %llu cycles (%s / %s)\n", mode ? "L2 trip " : "DSM push",
           bytes, chunks, sum / 16, mx, cudaGetErrorString(e), cudaGetErrorString(e2));
  }
}

// Microbenchmark of the Jacobi cross-phase step (jacobi.cu): W warps of one
// CTA, each holding one register column (RPL doubles per lane) and meeting a
// shared-memory column per step, with / without the per-step named barrier.
// Prints cycles per step.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_rot bench_rot.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double fast_rsqrt(double x) {
  double y;
  asm("rsqrt.approx.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
__device__ __forceinline__ double fast_rcp(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  y = y * fma(-x, y, 2.0);
  y = y * fma(-x, y, 2.0);
  return y;
}

template <int RPL, int MODE>
__global__ void kern(double* out, long long* cyc, int steps) {
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, B = blockDim.x >> 5;
  constexpr int MP = 32 * RPL;
  for (int e = threadIdx.x; e < B * MP; e += blockDim.x) sm[e] = 1e-3 * ((e * 7919) % 1000) + 0.5;
  __syncthreads();
  double xa[RPL], xb[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) xa[i] = 0.3 + 1e-3 * (lane + 32 * i + warp);
  double al = 1.0, be = 1.0, dp = 1.0, ip = 1.0;
  int q = warp;
  long long t0 = clock64();
  for (int st = 0; st < steps; ++st, q = (q + 1 == B) ? 0 : q + 1) {
    if (MODE & 1) asm volatile("bar.sync 15, %0;" ::"r"(B * 32) : "memory");
    double* col = sm + q * MP;
#pragma unroll
    for (int i = 0; i < RPL; ++i) xb[i] = col[lane + 32 * i];
    double g0 = 0.0, g1 = 0.0;
#pragma unroll
    for (int i = 0; i < RPL; i += 2) { g0 = fma(xa[i], xb[i], g0); g1 = fma(xa[i + 1], xb[i + 1], g1); }
    const double ga = wsum(g0 + g1) * 1e-9;
    double t = ga;
    if (MODE & 2) {
      const double d = be - al + 1e-3, g2 = 2.0 * ga;
      const double q2 = fma(d, d, g2 * g2);
      const double hyp = q2 * fast_rsqrt(q2);
      t = (d >= 0.0 ? g2 : -g2) * fast_rcp(fabs(d) + hyp);
      const double u = fma(t, t, 1.0);
      const double c = fast_rsqrt(u);
      dp *= c; ip *= u * c;
    }
    const double mup = t * ip, muq = t * dp;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const double x = xa[i], y = xb[i];
      xa[i] = fma(-mup, y, x);
      xb[i] = fma(muq, x, y);
    }
    al = fma(-t, ga, al);
    be = fma(t, ga, be);
    if (MODE & 4) {
#pragma unroll
      for (int i = 0; i < RPL; ++i) col[lane + 32 * i] = xb[i];
    }
  }
  long long t1 = clock64();
  double acc = al + be;
#pragma unroll
  for (int i = 0; i < RPL; ++i) acc += xa[i];
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(int warps, const char* name) {
  double* out; long long* cyc;
  cudaMalloc(&out, 1024 * 8); cudaMalloc(&cyc, 8);
  const int smem = warps * 512 * 8;
  cudaFuncSetAttribute(kern<16, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int steps = 2000;
  kern<16, MODE><<<1, warps * 32, smem>>>(out, cyc, steps);
  kern<16, MODE><<<1, warps * 32, smem>>>(out, cyc, steps);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-34s warps %2d : %7.1f cycles/step  (%s)\n", name, warps, (double)c / steps,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(out); cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 14}) {
    run<0>(w, "dot+update");
    run<2>(w, "dot+math+update");
    run<6>(w, "dot+math+update+store");
    run<7>(w, "full (barrier)");
    run<5>(w, "no math, barrier+store");
  }
  return 0;
}

// microbenchmark: FP64 DFMA latency / throughput, div / sqrt / rsqrt latency, shuffle latency (sm_100a)
#include <cstdio>
__global__ void lat_fma(double* out, int iters, double a) {
  double x = threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = fma(x, a, 1e-7);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / iters; }
}
__global__ void lat_div(double* out, int iters, double a) {
  double x = 1.5 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = a / (x + 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / iters; }
}
__global__ void lat_sqrt(double* out, int iters) {
  double x = 2.5 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = sqrt(x) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / iters; }
}
__global__ void lat_rsqrt(double* out, int iters) {
  double x = 2.5 + threadIdx.x * 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = rsqrt(x) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / iters; }
}
__global__ void lat_shfl(double* out, int iters) {
  double x = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1) + 1.0;
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / iters; }
}
__global__ void thr_fma(double* out, int iters) {   // 8 independent chains per thread
  double x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], 0.999999, 1e-7);
  double s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* d; cudaMalloc(&d, 1 << 24);
  double h[2];
  lat_fma<<<1, 32>>>(d, 10000, 0.999); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("DFMA latency %.1f cyc\n", h[1]);
  lat_div<<<1, 32>>>(d, 10000, 0.7); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("DDIV latency (+DADD) %.1f cyc\n", h[1]);
  lat_sqrt<<<1, 32>>>(d, 10000); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("DSQRT latency (+DADD) %.1f cyc\n", h[1]);
  lat_rsqrt<<<1, 32>>>(d, 10000); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("DRSQRT latency (+DADD) %.1f cyc\n", h[1]);
  lat_shfl<<<1, 32>>>(d, 10000); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("SHFL(double)+DADD latency %.1f cyc\n", h[1]);
  int iters = 20000;
  for (int warps : {1, 4, 8, 16, 32}) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    thr_fma<<<148, 32 * warps>>>(d, iters);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double flops = 2.0 * 8 * iters * 148.0 * 32 * warps;
    printf("DFMA throughput, %2d warps/SM: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1.965 GHz)\n", warps, flops / ms / 1e9,
           flops / 2 / (ms * 1e-3) / 148 / 1.965e9);
  }
}

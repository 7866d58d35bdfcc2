// Batched FP64 GEMM microbenchmark: launch_gemm (gemm.cu, per-launch tile
// configuration; TLRB_GEMM_CFG=0/1/2 forces one) vs cuBLAS strided-batched
// DGEMM on the shapes of the TLR path (C3: nb = 760) and a correctness check
// of every shape against cuBLAS (max relative difference).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1804_09137_b200/csrc \
//        tools/bench_gemm.cu paper_1804_09137_b200/csrc/gemm.cu paper_1804_09137_b200/csrc/misc.cu \
//        -lcublas -o tools/bench_gemm
#include "common.cuh"
#include <cublas_v2.h>
#include <cstdio>
#include <vector>
#include <cmath>
#include <algorithm>
#include <cstdlib>

using namespace tlrb;

int main() {
  struct Shape { const char* name; int m, n, k, ta, tb, count; };
  std::vector<Shape> shapes = {
      {"M-formation 760x760x200 (N,T)", 760, 760, 200, 0, 1, 64},
      {"U = E V 760x200x760", 760, 200, 760, 0, 0, 64},
      {"X = V^T V 30x30x760 (T,N)", 30, 30, 760, 1, 0, 4000},
      {"X = V^T V 120x60x760 (T,N)", 120, 60, 760, 1, 0, 1000},
      {"Y = U X 760x60x120", 760, 60, 120, 0, 0, 1000},
      {"W = V^T A 24x736x760 (T,N)", 24, 736, 760, 1, 0, 64},
      {"trail 760x736x24", 760, 736, 24, 0, 0, 64},
      {"dense upd 760x760x760 (T,N)", 760, 760, 760, 1, 0, 82},
      {"dense upd 760x760x760 (N,T)", 760, 760, 760, 0, 1, 82},
      {"big 4096x4096x4096", 4096, 4096, 4096, 0, 0, 1},
  };
  DescArena ar;
  ar.init(64 << 20);
  cublasHandle_t hb;
  cublasCreate(&hb);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cublasSetStream(hb, s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int only = getenv("BENCH_SHAPE") ? atoi(getenv("BENCH_SHAPE")) : -1;   // one shape (ncu captures)
  for (size_t si = 0; si < shapes.size(); ++si) {
    if (only >= 0 && (int)si != only) continue;
    const Shape& sh = shapes[si];
    const int lda = sh.ta ? sh.k : sh.m, ldb = sh.tb ? sh.n : sh.k, ldc = sh.m;
    const size_t sa = (size_t)lda * (sh.ta ? sh.m : sh.k), sb = (size_t)ldb * (sh.tb ? sh.k : sh.n),
                 sc = (size_t)ldc * sh.n;
    double *A, *B, *C;
    cudaMalloc(&A, sa * sh.count * 8);
    cudaMalloc(&B, sb * sh.count * 8);
    cudaMalloc(&C, sc * sh.count * 8);
    {
      std::vector<double> ha(sa * sh.count), hb2(sb * sh.count);
      uint64_t x = 88172645463325252ull;
      auto rnd = [&] { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return (double)(x >> 11) / 9007199254740992.0 - 0.5; };
      for (auto& v : ha) v = rnd();
      for (auto& v : hb2) v = rnd();
      cudaMemcpy(A, ha.data(), ha.size() * 8, cudaMemcpyHostToDevice);
      cudaMemcpy(B, hb2.data(), hb2.size() * 8, cudaMemcpyHostToDevice);
    }
    double* C2;
    cudaMalloc(&C2, sc * sh.count * 8);
    std::vector<GemmProb> probs;
    for (int i = 0; i < sh.count; ++i)
      probs.push_back({A + sa * i, B + sb * i, nullptr, C + sc * i, sh.m, sh.n, sh.k, lda, ldb, 0, ldc, sh.ta,
                       sh.tb, 0, 1.0, 0.0});
    const double fl = 2.0 * sh.m * sh.n * sh.k * sh.count;
    float best = 1e30f, bestc = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0, s);
      launch_gemm(probs, ar, s);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = std::min(best, ms);
      ar.reset();
      const double one = 1.0, zero = 0.0;
      cudaEventRecord(e0, s);
      cublasDgemmStridedBatched(hb, sh.ta ? CUBLAS_OP_T : CUBLAS_OP_N, sh.tb ? CUBLAS_OP_T : CUBLAS_OP_N, sh.m,
                                sh.n, sh.k, &one, A, lda, sa, B, ldb, sb, &zero, C2, ldc, sc, sh.count);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      bestc = std::min(bestc, ms);
    }
    std::vector<double> h1(sc * sh.count), h2(sc * sh.count);
    cudaMemcpy(h1.data(), C, h1.size() * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), C2, h2.size() * 8, cudaMemcpyDeviceToHost);
    double md = 0, mx = 0;
    for (size_t i = 0; i < h1.size(); ++i) { md = std::max(md, std::fabs(h1[i] - h2[i])); mx = std::max(mx, std::fabs(h2[i])); }
    printf("%-32s x%5d : ours %8.3f ms %6.2f TF/s | cuBLAS %8.3f ms %6.2f TF/s | maxdiff %.1e\n", sh.name, sh.count,
           best, fl / best / 1e9, bestc, fl / bestc / 1e9, md / (mx > 0 ? mx : 1));
    cudaFree(C2);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
  }
  return 0;
}

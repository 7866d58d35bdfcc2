// Batched FP64 GEMM microbenchmark: dgemm_vbatch_kernel (gemm.cu) vs cuBLAS
// strided-batched DGEMM on the shapes of the TLR path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1804_09137_b200/csrc \
//        tools/bench_gemm.cu paper_1804_09137_b200/csrc/gemm.cu paper_1804_09137_b200/csrc/misc.cu \
//        -lcublas -o tools/bench_gemm
#include "common.cuh"
#include <cublas_v2.h>
#include <cstdio>
#include <vector>

using namespace tlrb;

int main() {
  struct Shape { const char* name; int m, n, k, ta, tb, count; };
  std::vector<Shape> shapes = {
      {"M-formation 500x500x320", 500, 500, 320, 0, 1, 36},
      {"U = M V  500x320x500", 500, 320, 500, 0, 0, 36},
      {"W = V^T A 32x468x500", 32, 468, 500, 1, 0, 36},
      {"update 500x468x32", 500, 468, 32, 0, 0, 36},
      {"sketch 40x500x500", 40, 500, 500, 0, 0, 36},
      {"SYRK-like 500x500x64", 500, 500, 64, 0, 1, 170},
      {"big 2000x2000x2000", 2000, 2000, 2000, 0, 0, 1},
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
  for (const Shape& sh : shapes) {
    const int lda = sh.ta ? sh.k : sh.m, ldb = sh.tb ? sh.n : sh.k, ldc = sh.m;
    const size_t sa = (size_t)lda * (sh.ta ? sh.m : sh.k), sb = (size_t)ldb * (sh.tb ? sh.k : sh.n),
                 sc = (size_t)ldc * sh.n;
    double *A, *B, *C;
    cudaMalloc(&A, sa * sh.count * 8);
    cudaMalloc(&B, sb * sh.count * 8);
    cudaMalloc(&C, sc * sh.count * 8);
    cudaMemset(A, 0, sa * sh.count * 8);
    cudaMemset(B, 0, sb * sh.count * 8);
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
                                sh.n, sh.k, &one, A, lda, sa, B, ldb, sb, &zero, C, ldc, sc, sh.count);
      cudaEventRecord(e1, s);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      bestc = std::min(bestc, ms);
    }
    printf("%-28s x%4d : ours %8.3f ms %6.2f TF/s | cuBLAS %8.3f ms %6.2f TF/s\n", sh.name, sh.count, best,
           fl / best / 1e9, bestc, fl / bestc / 1e9);
    cudaFree(A);
    cudaFree(B);
    cudaFree(C);
  }
  return 0;
}

// Prototype: CUTLASS 4.x grouped GEMM (SM80 DMMA path, runs on sm_100a) on
// the TLR batch shapes, against dgemm_vbatch (gemm.cu) — decides whether the
// vendored CUTLASS templates are worth instantiating inside the library.
#include "common.cuh"
#include "cutlass/cutlass.h"
#include "cutlass/gemm/gemm.h"
#include "cutlass/gemm/kernel/gemm_grouped.h"
#include "cutlass/gemm/kernel/default_gemm_grouped.h"
#include "cutlass/gemm/device/gemm_grouped.h"
#include "cutlass/epilogue/thread/linear_combination.h"
#include <cstdio>
#include <vector>

using namespace tlrb;
using CM = cutlass::layout::ColumnMajor;
using RM = cutlass::layout::RowMajor;

template <class LA, class LB>
using Kernel = typename cutlass::gemm::kernel::DefaultGemmGrouped<
    double, LA, cutlass::ComplexTransform::kNone, 1, double, LB, cutlass::ComplexTransform::kNone, 1, double, CM,
    double, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<64, 128, 16>,
    cutlass::gemm::GemmShape<32, 64, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<1>, 3,
    cutlass::gemm::kernel::GroupScheduleMode::kDeviceOnly>::GemmKernel;

template <class LA, class LB>
float run_cutlass(int count, int m, int n, int k, double* A, size_t sa, int lda, double* B, size_t sb, int ldb,
                  double* C, size_t sc, int ldc, cudaStream_t s) {
  using G = cutlass::gemm::device::GemmGrouped<Kernel<LA, LB>>;
  std::vector<cutlass::gemm::GemmCoord> ps(count, cutlass::gemm::GemmCoord(m, n, k));
  std::vector<double*> pa(count), pb(count), pc(count);
  std::vector<int64_t> la(count, lda), lb(count, ldb), lc(count, ldc);
  for (int i = 0; i < count; ++i) { pa[i] = A + sa * i; pb[i] = B + sb * i; pc[i] = C + sc * i; }
  cutlass::gemm::GemmCoord* dps; double **dpa, **dpb, **dpc; int64_t *dla, *dlb, *dlc;
  cudaMalloc(&dps, count * sizeof(*dps)); cudaMalloc(&dpa, count * 8); cudaMalloc(&dpb, count * 8);
  cudaMalloc(&dpc, count * 8); cudaMalloc(&dla, count * 8); cudaMalloc(&dlb, count * 8); cudaMalloc(&dlc, count * 8);
  cudaMemcpy(dps, ps.data(), count * sizeof(*dps), cudaMemcpyHostToDevice);
  cudaMemcpy(dpa, pa.data(), count * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dpb, pb.data(), count * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dpc, pc.data(), count * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dla, la.data(), count * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dlb, lb.data(), count * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dlc, lc.data(), count * 8, cudaMemcpyHostToDevice);
  const int tbs = G::sufficient(ps.data(), count);
  typename G::EpilogueOutputOp::Params ep(1.0, 0.0);
  typename G::Arguments args(dps, count, tbs, ep, dpa, dpb, dpc, dpc, dla, dlb, dlc, dlc, ps.data());
  G g;
  size_t wsb = g.get_workspace_size(args);
  void* ws = nullptr;
  if (wsb) cudaMalloc(&ws, wsb);
  if (g.initialize(args, ws) != cutlass::Status::kSuccess) { printf("init failed\n"); return -1; }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0, s);
    g.run(s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    best = std::min(best, ms);
  }
  printf("   (tbs %d, err %s)\n", tbs, cudaGetErrorString(cudaGetLastError()));
  return best;
}

int main() {
  struct Shape { const char* name; int m, n, k, ta, tb, count; };
  std::vector<Shape> shapes = {
      {"M-formation 500x500x320 NT", 500, 500, 320, 0, 1, 36},
      {"U = M V  500x320x500 NN", 500, 320, 500, 0, 0, 36},
      {"W = V^T A 32x468x500 TN", 32, 468, 500, 1, 0, 36},
      {"update 500x468x32 NN", 500, 468, 32, 0, 0, 36},
      {"SYRK-like 500x500x64 NT", 500, 500, 64, 0, 1, 170},
      {"big 2000^3 NN", 2000, 2000, 2000, 0, 0, 1},
  };
  DescArena ar; ar.init(64 << 20);
  cudaStream_t s; cudaStreamCreate(&s);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (const Shape& sh : shapes) {
    const int lda = sh.ta ? sh.k : sh.m, ldb = sh.tb ? sh.n : sh.k, ldc = sh.m;
    const size_t sa = (size_t)lda * (sh.ta ? sh.m : sh.k), sb = (size_t)ldb * (sh.tb ? sh.k : sh.n), sc = (size_t)ldc * sh.n;
    double *A, *B, *C;
    cudaMalloc(&A, sa * sh.count * 8); cudaMalloc(&B, sb * sh.count * 8); cudaMalloc(&C, sc * sh.count * 8);
    cudaMemset(A, 0, sa * sh.count * 8); cudaMemset(B, 0, sb * sh.count * 8);
    std::vector<GemmProb> probs;
    for (int i = 0; i < sh.count; ++i)
      probs.push_back({A + sa * i, B + sb * i, nullptr, C + sc * i, sh.m, sh.n, sh.k, lda, ldb, 0, ldc, sh.ta, sh.tb, 0, 1.0, 0.0});
    const double fl = 2.0 * sh.m * sh.n * sh.k * sh.count;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0, s); launch_gemm(probs, ar, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms); ar.reset();
    }
    float bc;
    if (!sh.ta && !sh.tb) bc = run_cutlass<CM, CM>(sh.count, sh.m, sh.n, sh.k, A, sa, lda, B, sb, ldb, C, sc, ldc, s);
    else if (!sh.ta && sh.tb) bc = run_cutlass<CM, RM>(sh.count, sh.m, sh.n, sh.k, A, sa, lda, B, sb, ldb, C, sc, ldc, s);
    else bc = run_cutlass<RM, CM>(sh.count, sh.m, sh.n, sh.k, A, sa, lda, B, sb, ldb, C, sc, ldc, s);
    printf("%-28s x%4d : vbatch %7.3f ms %6.2f TF/s | cutlass grouped %7.3f ms %6.2f TF/s\n", sh.name, sh.count,
           best, fl / best / 1e9, bc, fl / bc / 1e9);
    cudaFree(A); cudaFree(B); cudaFree(C);
  }
}

// gemm_cutlass.cu — grouped variable-size FP64 GEMM from the CUTLASS 4.x
// templates (SM80 DMMA mainloop: mma.sync.m8n8k4.f64, 64x128x16 CTA tile,
// 32x64 warp tile, 3-stage cp.async pipeline; runs natively on sm_100a,
// where tcgen05 has no f64 kind).
//
// launch_gemm() (gemm.cu) hands this file the problems it can take — no
// lower-only tiles, no device `active` flag, m, n >= 64 — grouped by
// (op(A), op(B), alpha, beta); one persistent grouped launch per group, the
// problem list (sizes, pointers, leading dimensions) staged on the device
// through the DescArena.  Measured on the TLR batch shapes (tools/
// bench_cutlass_grouped.cu): 1.4-1.8x the throughput of dgemm_vbatch_kernel.
// The header tree is the CUTLASS vendored in the image (build.py locates it);
// without it this file compiles to a stub and everything stays on
// dgemm_vbatch_kernel.
#include "common.cuh"

#ifdef TLRB_HAVE_CUTLASS
#include "cutlass/cutlass.h"
#include "cutlass/gemm/gemm.h"
#include "cutlass/gemm/kernel/gemm_grouped.h"
#include "cutlass/gemm/kernel/default_gemm_grouped.h"
#include "cutlass/gemm/device/gemm_grouped.h"
#include "cutlass/epilogue/thread/linear_combination.h"
#endif

#include <algorithm>
#include <map>
#include <tuple>

namespace tlrb {

#ifdef TLRB_HAVE_CUTLASS
namespace {

using CM = cutlass::layout::ColumnMajor;
using RM = cutlass::layout::RowMajor;
constexpr int kTileM = 64, kTileN = 128;

template <class LA, class LB>
using GroupedKernel = typename cutlass::gemm::kernel::DefaultGemmGrouped<
    double, LA, cutlass::ComplexTransform::kNone, 1, double, LB, cutlass::ComplexTransform::kNone, 1, double, CM,
    double, cutlass::arch::OpClassTensorOp, cutlass::arch::Sm80, cutlass::gemm::GemmShape<kTileM, kTileN, 16>,
    cutlass::gemm::GemmShape<32, 64, 16>, cutlass::gemm::GemmShape<8, 8, 4>,
    cutlass::epilogue::thread::LinearCombination<double, 1, double, double>,
    cutlass::gemm::threadblock::GemmIdentityThreadblockSwizzle<1>, 3,
    cutlass::gemm::kernel::GroupScheduleMode::kDeviceOnly>::GemmKernel;

struct Staged {   // device copies of one group's problem list
  cutlass::gemm::GemmCoord* sizes;
  double **a, **b, **c, **d;
  int64_t *lda, *ldb, *ldc, *ldd;
};

template <class LA, class LB>
void run_group(const std::vector<const GemmProb*>& g, DescArena& ar, cudaStream_t s) {
  using G = cutlass::gemm::device::GemmGrouped<GroupedKernel<LA, LB>>;
  const int n = (int)g.size();
  std::vector<cutlass::gemm::GemmCoord> sz(n);
  std::vector<double*> pa(n), pb(n), pc(n), pd(n);
  std::vector<int64_t> la(n), lb(n), lc(n), ld(n);
  int64_t tiles = 0;
  double fl = 0, by = 0;
  for (int i = 0; i < n; ++i) {
    const GemmProb& p = *g[i];
    sz[i] = cutlass::gemm::GemmCoord(p.m, p.n, p.k);
    pa[i] = const_cast<double*>(p.A);
    pb[i] = const_cast<double*>(p.B);
    pd[i] = p.C;
    pc[i] = p.beta != 0.0 ? const_cast<double*>(p.Cin) : p.C;
    la[i] = p.lda;
    lb[i] = p.ldb;
    ld[i] = p.ldc;
    lc[i] = p.beta != 0.0 ? p.ldcin : p.ldc;
    tiles += (int64_t)((p.m + kTileM - 1) / kTileM) * ((p.n + kTileN - 1) / kTileN);
    fl += 2.0 * p.m * p.n * p.k;
    by += 8.0 * ((double)p.m * p.k + (double)p.k * p.n + (double)p.m * p.n * (p.beta != 0.0 ? 2 : 1));
  }
  // persistent CTAs: occupancy x SMs, at most one per output tile
  static const int max_ctas = [] {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return G::maximum_active_blocks() * sms;
  }();
  const int ctas = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, max_ctas));
  typename G::EpilogueOutputOp::Params ep(g[0]->alpha, g[0]->beta);
  typename G::Arguments args(ar.put(sz, s), n, ctas, ep, ar.put(pa, s), ar.put(pb, s), ar.put(pc, s),
                             ar.put(pd, s), ar.put(la, s), ar.put(lb, s), ar.put(lc, s), ar.put(ld, s),
                             sz.data());
  G op;
  if (op.initialize(args, nullptr, s) != cutlass::Status::kSuccess)
    throw CudaError(cudaErrorUnknown, "cutlass grouped GEMM initialize", __FILE__, __LINE__);
  ProfScope ps(K_GEMM, s, fl, by);
  if (op.run(s) != cutlass::Status::kSuccess)
    throw CudaError(cudaErrorUnknown, "cutlass grouped GEMM run", __FILE__, __LINE__);
  post_launch();
}

}  // namespace

std::vector<GemmProb> launch_gemm_cutlass(const std::vector<GemmProb>& probs, DescArena& ar, cudaStream_t s) {
  std::vector<GemmProb> rest;
  // (ta, tb, alpha, beta) -> problems
  std::map<std::tuple<int, int, double, double>, std::vector<const GemmProb*>> groups;
  for (const GemmProb& p : probs) {
    if (p.m <= 0 || p.n <= 0) continue;
    if (p.lower_only || p.active || p.m < 64 || p.n < 64 || p.k < 1) {
      rest.push_back(p);
      continue;
    }
    groups[std::make_tuple(p.ta, p.tb, p.alpha, p.beta)].push_back(&p);
  }
  for (auto& kv : groups) {
    const int ta = std::get<0>(kv.first), tb = std::get<1>(kv.first);
    if (!ta && !tb) run_group<CM, CM>(kv.second, ar, s);
    else if (!ta && tb) run_group<CM, RM>(kv.second, ar, s);
    else if (ta && !tb) run_group<RM, CM>(kv.second, ar, s);
    else run_group<RM, RM>(kv.second, ar, s);
  }
  return rest;
}

bool have_cutlass_gemm() { return true; }

#else

std::vector<GemmProb> launch_gemm_cutlass(const std::vector<GemmProb>& probs, DescArena&, cudaStream_t) {
  return probs;
}
bool have_cutlass_gemm() { return false; }

#endif

}  // namespace tlrb

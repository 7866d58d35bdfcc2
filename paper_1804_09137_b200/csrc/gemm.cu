// gemm.cu — variable-size batched FP64 GEMM on the sm_100a FP64 tensor pipe.
//
// tcgen05.mma has no f64 kind on sm_100a, so FP64 tensor-core math is
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  One launch covers a whole batch of
// independent problems of different (m, n, k): the grid is the flattened list
// of 64x64 output tiles of every problem (binary search of a prefix sum), so
// a step of the tile Cholesky (all SYRK / GEMM / low-rank product updates of
// panel k) is one launch.
//
// CTA: 128 threads = 4 warps in a 2x2 layout, warp tile 32x32 = 4x4 DMMA
// tiles; BK = 16; operands staged global -> registers -> shared memory with a
// two-stage ping-pong so the next K slab loads while DMMAs run.
#include "common.cuh"
#include <chrono>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

namespace tlrb {

constexpr int GBM = 64, GBN = 64, GBK = 16, GPAD = 8;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(128) dgemm_vbatch_kernel(const GemmProb* __restrict__ probs,
                                                           const int* __restrict__ start,
                                                           int nprob) {
  const int blk = blockIdx.x;
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= blk) lo = mid; else hi = mid - 1;
  }
  const GemmProb P = probs[lo];
  if (P.active && !*P.active) return;
  const int local = blk - start[lo];
  const int tm = (P.m + GBM - 1) / GBM;
  const int m0 = (local % tm) * GBM, n0 = (local / tm) * GBN;
  if (P.lower_only && n0 >= m0 + GBM) return;

  __shared__ double As[2][GBK][GBM + GPAD];
  __shared__ double Bs[2][GBK][GBN + GPAD];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 32;

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  double ra[8], rb[8];
  auto load = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + i * 128;
      int r, kk;
      if (!P.ta) { r = e & 63; kk = e >> 6; } else { r = e >> 4; kk = e & 15; }
      const int gr = m0 + r, gk = k0 + kk;
      double v = 0.0;
      if (gr < P.m && gk < P.k)
        v = P.ta ? P.A[(size_t)gr * P.lda + gk] : P.A[(size_t)gk * P.lda + gr];
      ra[i] = v;
      int c;
      if (!P.tb) { kk = e & 15; c = e >> 4; } else { c = e & 63; kk = e >> 6; }
      const int gc = n0 + c;
      const int gk2 = k0 + kk;
      double w = 0.0;
      if (gc < P.n && gk2 < P.k)
        w = P.tb ? P.B[(size_t)gk2 * P.ldb + gc] : P.B[(size_t)gc * P.ldb + gk2];
      rb[i] = w;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + i * 128;
      int r, kk;
      if (!P.ta) { r = e & 63; kk = e >> 6; } else { r = e >> 4; kk = e & 15; }
      As[buf][kk][r] = ra[i];
      int c;
      if (!P.tb) { kk = e & 15; c = e >> 4; } else { c = e & 63; kk = e >> 6; }
      Bs[buf][kk][c] = rb[i];
    }
  };

  const int nk = (P.k + GBK - 1) / GBK;
  if (nk > 0) {
    load(0);
    store(0);
    __syncthreads();
  }
  for (int kc = 0; kc < nk; ++kc) {
    const int cur = kc & 1;
    if (kc + 1 < nk) load((kc + 1) * GBK);
#pragma unroll
    for (int k4 = 0; k4 < GBK; k4 += 4) {
      double a[4], b[4];
      const int kr = k4 + (lane & 3);
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        a[t] = As[cur][kr][wm + t * 8 + (lane >> 2)];
        b[t] = Bs[cur][kr][wn + t * 8 + (lane >> 2)];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
    }
    if (kc + 1 < nk) store(cur ^ 1);
    __syncthreads();
  }

  // epilogue: C = alpha acc + beta Cin
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = m0 + wm + i * 8 + (lane >> 2);
    if (r >= P.m) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = n0 + wn + j * 8 + 2 * (lane & 3) + h;
        if (c >= P.n) continue;
        double v = P.alpha * acc[i][j][h];
        if (P.beta != 0.0) v += P.beta * P.Cin[(size_t)c * P.ldcin + r];
        P.C[(size_t)c * P.ldc + r] = v;
      }
    }
  }
}

// host-side staging of one batched launch: appends the non-empty problems and
// their tile prefix sums to (allp, alls); returns the launch record
GemmStaged stage_gemm(const std::vector<GemmProb>& probs, std::vector<GemmProb>& allp, std::vector<int>& alls) {
  GemmStaged g;
  g.poff = (int)allp.size();
  g.soff = (int)alls.size();
  int tot = 0;
  for (const GemmProb& p : probs) {
    if (p.m <= 0 || p.n <= 0) continue;
    allp.push_back(p);
    alls.push_back(tot);
    tot += ((p.m + GBM - 1) / GBM) * ((p.n + GBN - 1) / GBN);
    g.fl += 2.0 * p.m * p.n * p.k;
    g.by += 8.0 * ((double)p.m * p.k + (double)p.k * p.n + (double)p.m * p.n * (p.beta != 0.0 ? 2 : 1));
  }
  alls.push_back(tot);
  g.n = (int)allp.size() - g.poff;
  g.tot = tot;
  return g;
}

// launch a staged batch whose descriptors already live on the device
void launch_gemm_staged(const GemmStaged& g, const GemmProb* dp, const int* ds, cudaStream_t s) {
  if (g.tot == 0 || g.n == 0) return;
  ProfScope ps(K_GEMM, s, g.fl, g.by);
  dgemm_vbatch_kernel<<<g.tot, 128, 0, s>>>(dp + g.poff, ds + g.soff, g.n);
  post_launch();
}

// TLRB_GEMM_STATS=1 (diagnostic, serialising): per launch, the stream is
// synchronised around the call and the time is split over the launch's
// problems by flops; buckets (m, n, k rounded up to powers of two, large-plain
// flag) are printed at exit.  Used to aim the GEMM work.
namespace {
struct GemmStats {
  std::mutex mu;
  std::map<std::tuple<int, int, int, int>, std::tuple<int64_t, double, double>> b;   // count, flops, ms
  ~GemmStats() {
    if (b.empty()) return;
    fprintf(stderr, "[gemm-stats] m n k large count gflop ms tflops\n");
    for (auto& [k, v] : b)
      fprintf(stderr, "[gemm-stats] %d %d %d %d %lld %.3f %.3f %.2f\n", std::get<0>(k), std::get<1>(k),
              std::get<2>(k), std::get<3>(k), (long long)std::get<0>(v), std::get<1>(v) / 1e9, std::get<2>(v),
              std::get<2>(v) > 0 ? std::get<1>(v) / (std::get<2>(v) * 1e-3) / 1e12 : 0.0);
  }
};
GemmStats g_gstats;
int p2(int x) {
  int r = 1;
  while (r < x) r <<= 1;
  return r;
}
}  // namespace

void launch_gemm_impl(const std::vector<GemmProb>& probs, DescArena& ar, cudaStream_t s);

void launch_gemm(const std::vector<GemmProb>& probs, DescArena& ar, cudaStream_t s) {
  static const bool stats = getenv("TLRB_GEMM_STATS") != nullptr;
  if (!stats || probs.empty()) return launch_gemm_impl(probs, ar, s);
  TLRB_CUDA(cudaStreamSynchronize(s));
  const auto t0 = std::chrono::steady_clock::now();
  launch_gemm_impl(probs, ar, s);
  TLRB_CUDA(cudaStreamSynchronize(s));
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  double tot = 0;
  for (const GemmProb& p : probs) tot += 2.0 * p.m * p.n * p.k;
  std::lock_guard<std::mutex> lk(g_gstats.mu);
  for (const GemmProb& p : probs) {
    if (p.m <= 0 || p.n <= 0) continue;
    const double f = 2.0 * p.m * p.n * p.k;
    const int large = !(p.lower_only || p.active || p.m < 64 || p.n < 64);
    auto& v = g_gstats.b[{p2(p.m), p2(p.n), p2(std::max(1, p.k)), large}];
    std::get<0>(v) += 1;
    std::get<1>(v) += f;
    std::get<2>(v) += tot > 0 ? ms * f / tot : 0.0;
  }
}

void launch_gemm_impl(const std::vector<GemmProb>& probs, DescArena& ar, cudaStream_t s) {
  if (probs.empty()) return;
  // large plain problems go to the CUTLASS grouped DMMA kernel (gemm_cutlass.cu);
  // lower-only, flagged and skinny ones stay here (TLRB_GEMM_CUTLASS=0: all here)
  static const bool use_cutlass = have_cutlass_gemm() && !(getenv("TLRB_GEMM_CUTLASS") &&
                                                           atoi(getenv("TLRB_GEMM_CUTLASS")) == 0);
  const std::vector<GemmProb> rest = use_cutlass ? launch_gemm_cutlass(probs, ar, s) : probs;
  if (rest.empty()) return;
  std::vector<GemmProb> keep;
  std::vector<int> start;
  keep.reserve(rest.size());
  start.reserve(rest.size() + 1);
  const GemmStaged g = stage_gemm(rest, keep, start);
  if (g.tot == 0) return;
  const GemmProb* dp = ar.put(keep, s);
  const int* ds = ar.put(start, s);
  launch_gemm_staged(g, dp, ds, s);
}

}  // namespace tlrb

// gemm.cu — variable-size batched FP64 GEMM on the sm_100a FP64 tensor pipe.
//
// tcgen05.mma has no f64 kind on sm_100a, so FP64 tensor-core math is
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  One launch covers a whole batch of
// independent problems of different (m, n, k): the grid is the flattened list
// of 64x64 output tiles of every problem (binary search of a prefix sum), so
// a step of the tile Cholesky (all SYRK / GEMM / low-rank product updates of
// panel k) is one launch.
//
// Three tile configurations of one kernel template (64x64 / 4 warps / 4
// stages, 64x128 / 4 warps / 3 stages, 128x128 / 8 warps / 3 stages), chosen
// per launch from the batch's shapes; operands go global -> shared memory
// through a multi-stage cp.async (LDGSTS) pipeline, fragments from shared
// memory into DMMA.  Replaces the round-1 register-staged kernel and the
// CUTLASS grouped GEMM (no external headers).
#include "common.cuh"
#include <chrono>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

namespace tlrb {

#ifndef TLRB_GEMM_INTER
#define TLRB_GEMM_INTER 0   // measured: refill after the k-steps 32.6 TF/s, spread over them 32.4, before them 31.1 (4096^3)
#endif
constexpr int GBK = 16;        // K slab per pipeline stage
constexpr int PADK = 4;        // k-contiguous smem rows: stride GBK + 4 (conflict-free fragments)
constexpr int PADMN = 4;       // m/n-contiguous smem rows: stride BM/BN + 4 (= 4 mod 16: the four k rows of a
                               // fragment land on distinct banks; + 8 gave 2-way conflicts, ncu r02f)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 8-byte global -> shared asynchronous copy (LDGSTS); src_bytes = 0 fills
// the shared word with zeros (tile edges)
// (`base` is a valid global address of the operand, used when nothing is read)
__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, const double* base, bool ok) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(ok ? gmem : base),
               "r"(ok ? 8 : 0));
}
// 16-byte variant (LDGSTS.128, L2 only): `bytes` in {0, 8, 16} are read, the
// rest of the 16-byte shared word pair is zero-filled
__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, const double* base, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(bytes ? gmem : base),
               "r"(bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Batched FP64 GEMM, C = alpha op(A) op(B) + beta Cin, one CTA per BM x BN
// output tile of any problem of the batch (binary search of the tile prefix
// sums).  Warps in a (BM/WM) x (BN/WN) grid, warp tile WM x WN of 8x8 DMMA
// fragments; ST-stage cp.async pipeline of K slabs of 16.  Shared layouts
// follow the operand's contiguous direction so that the asynchronous copies
// are coalesced and the fragment reads hit distinct banks:
//   op(A) = A   (m contiguous): As[k][m], stride BM + 4
//   op(A) = A^T (k contiguous): As[m][k], stride 16 + 4
//   op(B) = B   (k contiguous): Bs[n][k], stride 16 + 4
//   op(B) = B^T (n contiguous): Bs[k][n], stride BN + 4
// The transposition flags are template parameters (a launch holds problems of
// one (ta, tb) only): the shared-memory addresses of the fragment reads are
// then immediates and the copy addresses advance by one add per slab.  ncu of
// the runtime-flag version (r02f): 5.5 instructions issued per DMMA, most of
// them SEL / IMAD / LEA address selection, FP64 tensor pipe 78% busy.
template <int BM, int BN, int WM, int WN, int ST, int KS, int VEC, bool TA, bool TB>
__global__ void __launch_bounds__((BM / WM) * (BN / WN) * KS * 32)
    dgemm_tiles_kernel(const GemmProb* __restrict__ probs, const int* __restrict__ start,
                       const int* __restrict__ blk2p, int nprob) {
  constexpr int NT = (BM / WM) * (BN / WN) * KS * 32;
  constexpr bool INTER = TLRB_GEMM_INTER;             // refill spread over the k-steps
  constexpr int LSA = TA ? GBK + PADK : BM + PADMN;   // shared row strides
  constexpr int LSB = TB ? BN + PADMN : GBK + PADK;
  constexpr int AS = TA ? BM * LSA : GBK * LSA;       // doubles per stage
  constexpr int BS = TB ? GBK * LSB : BN * LSB;
  constexpr int FM = WM / 8, FN = WN / 8;
  extern __shared__ double smem[];
  double* As = smem;              // ST x AS
  double* Bs = smem + ST * AS;    // ST x BS

  const int blk = blockIdx.x;
  int lo = 0;
  if (blk2p) {   // per-CTA problem index (one load instead of a dependent binary search)
    lo = blk2p[blk];
  } else {
    int hi = nprob - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (start[mid] <= blk) lo = mid; else hi = mid - 1;
    }
  }
  const GemmProb& P = probs[lo];
  if (P.active && !*P.active) return;
  const int local = blk - start[lo];
  const int tm = (P.m + BM - 1) / BM;
  const int m0 = (local % tm) * BM, n0 = (local / tm) * BN;
  if (P.lower_only && n0 >= m0 + BM) return;
  const int M = P.m, N = P.n, K = P.k, lda = P.lda, ldb = P.ldb;
  const double* __restrict__ A = P.A;
  const double* __restrict__ B = P.B;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int WG = (BM / WM) * (BN / WN);   // warps per K slice
  const int wk = warp / WG;                   // this warp's share of each slab's k-steps (split K)
  const int wm = (warp % WG % (BM / WM)) * WM, wn = (warp % WG / (BM / WM)) * WN;

  // per-thread copy positions: NT is a multiple of BM, BN and 16, so each
  // thread's elements of a stage lie on one row / column stride apart and a
  // single base pointer per operand serves all of them.  VEC = 2 (every
  // operand of the batch 16-byte aligned with an even leading dimension):
  // a thread moves pairs along the operand's contiguous direction with one
  // 16-byte cp.async (half the LDGSTS instructions, L1 bypassed).
  //   A   (m contiguous): row pair a_r fixed, k = a_k + i NT / CM
  //   A^T (k contiguous): k pair a_k fixed,   m = a_r + i NT / CK
  //   B   (k contiguous): k pair b_k fixed,   n = b_c + i NT / CK
  //   B^T (n contiguous): col pair b_c fixed, k = b_k + i NT / CN
  static_assert(NT % BM == 0 && NT % BN == 0 && NT % GBK == 0, "copy layout");
  constexpr int CM = BM / VEC, CN = BN / VEC, CK = GBK / VEC;   // copy positions along m / n / k
  constexpr int NA = TA ? BM * CK / NT : CM * GBK / NT;         // copies per thread and stage
  constexpr int NB = TB ? CN * GBK / NT : BN * CK / NT;
  constexpr int SA = TA ? NT / CK : NT / CM;                    // index step between a thread's copies
  constexpr int SB = TB ? NT / CN : NT / CK;
  const int a_r = TA ? tid / CK : VEC * (tid % CM), a_k = TA ? VEC * (tid % CK) : tid / CM;
  const int b_c = TB ? VEC * (tid % CN) : tid / CK, b_k = TB ? tid / CN : VEC * (tid % CK);
  const double* a_ptr = TA ? A + (size_t)(m0 + a_r) * lda + a_k : A + (size_t)a_k * lda + m0 + a_r;
  const double* b_ptr = TB ? B + (size_t)b_k * ldb + n0 + b_c : B + (size_t)(n0 + b_c) * ldb + b_k;
  const size_t a_gs = (size_t)SA * lda, b_gs = (size_t)SB * ldb;          // global step between copies
  const size_t a_ks = TA ? GBK : (size_t)GBK * lda, b_ks = TB ? (size_t)GBK * ldb : GBK;   // per slab
  const unsigned a_sm = (unsigned)__cvta_generic_to_shared(As + (TA ? a_r * LSA + a_k : a_k * LSA + a_r));
  const unsigned b_sm = (unsigned)__cvta_generic_to_shared(Bs + (TB ? b_k * LSB + b_c : b_c * LSB + b_k));
  // edge of the tile along m / n: bytes of a copy (0 = zero fill).  Along
  // the contiguous direction the count is per thread, across it per copy.
  auto edge = [](int left) { return 8 * max(0, min(VEC, left)); };
  const int a_edge = TA ? 0 : edge(M - (m0 + a_r));
  const int b_edge = TB ? edge(N - (n0 + b_c)) : 0;
  unsigned a_rows = 0, b_cols = 0;   // bit i: copy i of the stage lies inside the matrix
  if constexpr (TA) {
#pragma unroll
    for (int i = 0; i < NA; ++i) a_rows |= (unsigned)(m0 + a_r + i * SA < M) << i;
  }
  if constexpr (!TB) {
#pragma unroll
    for (int i = 0; i < NB; ++i) b_cols |= (unsigned)(n0 + b_c + i * SB < N) << i;
  }
  auto cp = [&](unsigned sa, const double* g, int bytes) {
    // a zero-byte copy reads nothing (the address may lie past the matrix) and zero-fills
    if constexpr (VEC == 1)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(bytes));
    else
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(bytes));
  };
  // stage `st` <- slab at k0 (a_ptr / b_ptr already point at it).  `tail`:
  // the slab crosses K (only the last one can): per-copy k tests
  // (part q of np: every np-th copy; the main loop spreads the refill of a
  // stage over its k-steps so that the copy instructions of one warp issue
  // behind the DMMA burst of the other warp of its scheduler)
  auto load_part = [&](int st, int k0, bool tail, int q, int np) {
    const unsigned sa = a_sm + st * (AS * 8), sb = b_sm + st * (BS * 8);
#pragma unroll
    for (int i = 0; i < NA; ++i) {
      if (i % np != q) continue;
      int by;
      if constexpr (TA) {
        by = (a_rows >> i) & 1 ? VEC * 8 : 0;
        if (tail) by = min(by, edge(K - (k0 + a_k)));
      } else {
        by = a_edge;
        if (tail && k0 + a_k + i * SA >= K) by = 0;
      }
      cp(sa + i * (SA * LSA * 8), a_ptr + i * a_gs, by);
    }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
      if (i % np != q) continue;
      int by;
      if constexpr (TB) {
        by = b_edge;
        if (tail && k0 + b_k + i * SB >= K) by = 0;
      } else {
        by = (b_cols >> i) & 1 ? VEC * 8 : 0;
        if (tail) by = min(by, edge(K - (k0 + b_k)));
      }
      cp(sb + i * (SB * LSB * 8), b_ptr + i * b_gs, by);
    }
    if (q == np - 1) {
      a_ptr += a_ks;
      b_ptr += b_ks;
    }
  };
  auto load_stage = [&](int st, int k0, bool tail) { load_part(st, k0, tail, 0, 1); };

  double acc[FM][FN][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (K + GBK - 1) / GBK, kfull = K / GBK;
#pragma unroll
  for (int st = 0; st < ST - 1; ++st) {
    if (st < nk) load_stage(st, st * GBK, st >= kfull);
    cp_async_commit();
  }
  // fragment reads: lane (fr, fk) takes row / column fr of an 8-wide
  // fragment at k = fk of the k-step; all other offsets are immediates
  const int fr = lane >> 2, fk = lane & 3;
  const double* af = As + (TA ? (wm + fr) * LSA + 4 * wk + fk : (4 * wk + fk) * LSA + wm + fr);
  const double* bf = Bs + (TB ? (4 * wk + fk) * LSB + wn + fr : (wn + fr) * LSB + 4 * wk + fk);
  constexpr int A_T = TA ? 8 * LSA : 8, A_Q = TA ? 4 * KS : 4 * KS * LSA;   // per fragment / per k-step
  constexpr int B_T = TB ? 8 : 8 * LSB, B_Q = TB ? 4 * KS * LSB : 4 * KS;
  int st_c = 0, st_l = (ST - 1) % ST;   // stage consumed / loaded in this iteration
  for (int kc = 0; kc < nk; ++kc) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    // the stage consumed at kc - 1 (everyone is past it) is refilled in NQ
    // parts, one after each k-step's DMMAs
    const int kn = kc + ST - 1;
    const bool more = kn < nk, tail = kn >= kfull;
    const double* as = af + st_c * AS;
    const double* bs = bf + st_c * BS;
    constexpr int NQ = GBK / (4 * KS);
    constexpr bool PRE = ST < 3;   // two stages: the refill must be in flight during this slab's DMMAs
    if (PRE && more) load_stage(st_l, kn * GBK, tail);
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      double a[FM], b[FN];
#pragma unroll
      for (int t = 0; t < FM; ++t) a[t] = as[q * A_Q + t * A_T];
#pragma unroll
      for (int t = 0; t < FN; ++t) b[t] = bs[q * B_Q + t * B_T];
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      if (!PRE && INTER && more) load_part(st_l, kn * GBK, tail, q, NQ);
    }
    if (!PRE && !INTER && more) load_stage(st_l, kn * GBK, tail);
    cp_async_commit();
    st_c = st_c + 1 == ST ? 0 : st_c + 1;
    st_l = st_l + 1 == ST ? 0 : st_l + 1;
  }
  cp_async_wait<0>();
  if constexpr (KS > 1) {   // sum the K slices' partial tiles through shared memory
    __syncthreads();
    double* red = smem;     // (KS - 1) x WG warps x FM x FN x 2 x 32
    constexpr int PER = FM * FN * 2 * 32;
    if (wk > 0) {
#pragma unroll
      for (int i = 0; i < FM; ++i)
#pragma unroll
        for (int j = 0; j < FN; ++j)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            red[((size_t)(wk - 1) * WG + warp % WG) * PER + ((i * FN + j) * 2 + h) * 32 + lane] = acc[i][j][h];
    }
    __syncthreads();
    if (wk == 0) {
      for (int q = 1; q < KS; ++q)
#pragma unroll
        for (int i = 0; i < FM; ++i)
#pragma unroll
          for (int j = 0; j < FN; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              acc[i][j][h] += red[((size_t)(q - 1) * WG + warp) * PER + ((i * FN + j) * 2 + h) * 32 + lane];
    }
  }

  // epilogue through shared memory: the warps drop alpha * acc into a
  // column-major BM x BN tile, then consecutive threads write consecutive
  // rows of a column (coalesced C / Cin traffic, which dominates the
  // small-k shapes: trailing updates, M formation)
  const double alpha = P.alpha, beta = P.beta;
  __syncthreads();   // every warp is done with the pipeline buffers
  constexpr int LDC = BM + 1;
  double* cs = smem;
  if (KS == 1 || wk == 0) {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          cs[(wn + j * 8 + 2 * fk + h) * LDC + wm + i * 8 + fr] = alpha * acc[i][j][h];
  }
  __syncthreads();
  const int mr = min(BM, M - m0), nc = min(BN, N - n0);
  double* __restrict__ Cout = P.C + (size_t)n0 * P.ldc + m0;
  const double* __restrict__ Cin = beta != 0.0 ? P.Cin + (size_t)n0 * P.ldcin + m0 : nullptr;
  for (int e = tid; e < BM * BN; e += NT) {
    const int r = e % BM, c = e / BM;
    if (r >= mr || c >= nc) continue;
    double v = cs[c * LDC + r];
    if (beta != 0.0) v += beta * Cin[(size_t)c * P.ldcin + r];
    Cout[(size_t)c * P.ldc + r] = v;
  }
}

// tile configurations (m x n tile, warp tile, stages)
struct GemmCfg { int bm, bn; };
constexpr int kNCfg = 9;
constexpr GemmCfg kCfg[kNCfg] = {{64, 64}, {64, 128}, {128, 128}, {32, 32}, {32, 128},
                                 {64, 64}, {64, 128}, {32, 128}, {32, 32}};   // 5..8: two-stage variants of 0, 1, 4, 3

template <int BM, int BN, int WM, int WN, int ST, int KS, int VEC, bool TA, bool TB>
void run_tiles_t(int tot, const GemmProb* dp, const int* ds, const int* dm, int n, cudaStream_t s) {
  auto kern = dgemm_tiles_kernel<BM, BN, WM, WN, ST, KS, VEC, TA, TB>;
  constexpr int AS = TA ? BM * (GBK + PADK) : GBK * (BM + PADMN);
  constexpr int BS = TB ? GBK * (BN + PADMN) : BN * (GBK + PADK);
  const size_t pipe = (size_t)ST * (AS + BS) * sizeof(double);
  const size_t red = (size_t)(KS - 1) * (BM / WM) * (BN / WN) * (WM / 8) * (WN / 8) * 2 * 32 * sizeof(double);
  const size_t epi = (size_t)(BM + 1) * BN * sizeof(double);
  const size_t sm = std::max({pipe, red, epi});
  allow_smem(kern, sm);
  kern<<<tot, (BM / WM) * (BN / WN) * KS * 32, sm, s>>>(dp, ds, dm, n);
}

template <int BM, int BN, int WM, int WN, int ST, int KS, int VEC>
void run_tiles_v(int ta, int tb, int tot, const GemmProb* dp, const int* ds, const int* dm, int n, cudaStream_t s) {
  if (ta && tb) run_tiles_t<BM, BN, WM, WN, ST, KS, VEC, true, true>(tot, dp, ds, dm, n, s);
  else if (ta) run_tiles_t<BM, BN, WM, WN, ST, KS, VEC, true, false>(tot, dp, ds, dm, n, s);
  else if (tb) run_tiles_t<BM, BN, WM, WN, ST, KS, VEC, false, true>(tot, dp, ds, dm, n, s);
  else run_tiles_t<BM, BN, WM, WN, ST, KS, VEC, false, false>(tot, dp, ds, dm, n, s);
}

template <int BM, int BN, int WM, int WN, int ST, int KS = 1>
void run_tiles(const GemmStaged& g, const GemmProb* dp, const int* ds, const int* dm, cudaStream_t s) {
  if (g.vec) run_tiles_v<BM, BN, WM, WN, ST, KS, 2>(g.ta, g.tb, g.tot, dp, ds, dm, g.n, s);
  else run_tiles_v<BM, BN, WM, WN, ST, KS, 1>(g.ta, g.tb, g.tot, dp, ds, dm, g.n, s);
}

// tile configuration of one problem.  Measured with the templated kernel
// (tools/bench_gemm.cu, TLRB_GEMM_CFG sweep, B200): the two-stage 64 x 64
// configuration (41 KB of shared memory, five CTAs per SM) is the fastest or
// within 1% of it on every shape with m > 40 -- 4096^3 34.2 TF/s (128 x 128
// tiles: 32.6; cuBLAS 35.0), 82 x 760^3 32.4 (cuBLAS 34.2), 760 x 760 x 200
// 28.0, 760 x 736 x 24 9.8 -- so only problems with m <= 40 keep their own
// tiles: 32 x 32 with a four-way split of k when k is long, 32 x 128 with a
// two-way split for short k and wide n.
static int prob_cfg(const GemmProb& p) {
  if (p.m <= 40 && p.k >= 128) return 3;   // also thin problems: 24 x 736 x 760 16.9 TF/s (32 x 128 tiles: 12.2)
  if (p.m <= 40 && p.n >= 96) return 4;
  return 5;
}

// configuration of a whole batch (one launch): the class that holds most of
// the batch's flops, else the 64 x 64 tiles
int pick_cfg(const std::vector<GemmProb>& probs) {
  static const int force = getenv("TLRB_GEMM_CFG") ? atoi(getenv("TLRB_GEMM_CFG")) : -1;
  if (force >= 0 && force < kNCfg) return force;
  double fl = 0, fc[kNCfg] = {};
  for (const GemmProb& p : probs) {
    const double f = 2.0 * p.m * p.n * p.k;
    fl += f;
    fc[prob_cfg(p)] += f;
  }
  if (fc[3] >= 0.7 * fl) return 3;
  if (fc[4] >= 0.7 * fl) return 4;
  return 5;
}

// host-side staging of one batched launch: appends the non-empty problems and
// their tile prefix sums to (allp, alls); returns the launch record
GemmStaged stage_gemm(const std::vector<GemmProb>& probs, std::vector<GemmProb>& allp, std::vector<int>& alls,
                      int cfg) {
  GemmStaged g;
  g.cfg = cfg >= 0 ? cfg : pick_cfg(probs);
  const int bm = kCfg[g.cfg].bm, bn = kCfg[g.cfg].bn;
  g.poff = (int)allp.size();
  g.soff = (int)alls.size();
  int tot = 0;
  static const bool novec = getenv("TLRB_GEMM_NOVEC") != nullptr;
  g.vec = !novec;
  for (const GemmProb& p : probs) {
    if (p.m <= 0 || p.n <= 0) continue;
    // 16-byte copies need both operands 16-byte aligned with even leading dimensions
    if (((reinterpret_cast<uintptr_t>(p.A) | reinterpret_cast<uintptr_t>(p.B)) & 15) || ((p.lda | p.ldb) & 1))
      g.vec = false;
    if (g.ta < 0) { g.ta = p.ta != 0; g.tb = p.tb != 0; }
    if ((p.ta != 0) != (g.ta != 0) || (p.tb != 0) != (g.tb != 0))
      throw CudaError(cudaErrorInvalidValue, "stage_gemm: mixed transposition flags in one launch", __FILE__, __LINE__);
    allp.push_back(p);
    alls.push_back(tot);
    tot += ((p.m + bm - 1) / bm) * ((p.n + bn - 1) / bn);
    g.fl += 2.0 * p.m * p.n * p.k;
    g.by += 8.0 * ((double)p.m * p.k + (double)p.k * p.n + (double)p.m * p.n * (p.beta != 0.0 ? 2 : 1));
  }
  alls.push_back(tot);
  g.n = (int)allp.size() - g.poff;
  g.tot = tot;
  // CTA -> problem map after the prefix sums (small and mid-size launches:
  // their CTAs are short, a dependent binary search per CTA would dominate)
  if (g.n > 1 && tot <= (1 << 18)) {
    g.moff = (int)alls.size();
    alls.resize(alls.size() + tot);
    int* mp = alls.data() + g.moff;
    for (int q = 0; q < g.n; ++q) {
      const int a = alls[g.soff + q], b = alls[g.soff + q + 1];
      for (int c = a; c < b; ++c) mp[c] = q;
    }
  }
  return g;
}

// launch a staged batch whose descriptors already live on the device
void launch_gemm_staged(const GemmStaged& g, const GemmProb* dp, const int* ds, cudaStream_t s) {
  if (g.tot == 0 || g.n == 0) return;
  ProfScope ps(K_GEMM, s, g.fl, g.by);
  const GemmProb* p = dp + g.poff;
  const int* st = ds + g.soff;
  const int* mp = g.moff >= 0 ? ds + g.moff : nullptr;
  switch (g.cfg) {
    case 4: run_tiles<32, 128, 32, 64, 4, 2>(g, p, st, mp, s); break;
    case 3: run_tiles<32, 32, 32, 32, 4, 4>(g, p, st, mp, s); break;
    case 2: run_tiles<128, 128, 32, 64, 3>(g, p, st, mp, s); break;
    case 1: run_tiles<64, 128, 32, 64, 3>(g, p, st, mp, s); break;
    case 5: run_tiles<64, 64, 32, 32, 2>(g, p, st, mp, s); break;
    case 6: run_tiles<64, 128, 32, 64, 2>(g, p, st, mp, s); break;
    case 7: run_tiles<32, 128, 32, 64, 2, 2>(g, p, st, mp, s); break;
    case 8: run_tiles<32, 32, 32, 32, 2, 4>(g, p, st, mp, s); break;
    default: run_tiles<64, 64, 32, 32, 4>(g, p, st, mp, s); break;
  }
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

static void launch_gemm_one(const std::vector<GemmProb>& probs, int cfg, DescArena& ar, cudaStream_t s) {
  std::vector<GemmProb> keep;
  std::vector<int> start;
  keep.reserve(probs.size());
  start.reserve(probs.size() + 1);
  const GemmStaged g = stage_gemm(probs, keep, start, cfg);
  if (g.tot == 0) return;
  // descriptors and tile prefix sums in one upload
  const size_t pb = keep.size() * sizeof(GemmProb), sb = start.size() * sizeof(int);
  std::vector<char> buf(pb + sb);
  memcpy(buf.data(), keep.data(), pb);
  memcpy(buf.data() + pb, start.data(), sb);
  const char* d = static_cast<const char*>(ar.put_bytes(buf.data(), buf.size(), s));
  launch_gemm_staged(g, reinterpret_cast<const GemmProb*>(d), reinterpret_cast<const int*>(d + pb), s);
}

// One call = one batch of independent problems.  A batch of mixed shapes
// (the tile Cholesky's update batches hold exact 760^3 products next to
// rank-20 ones) is split by tile configuration, one launch per class that
// carries a real share of the work, so the large problems run on the
// 128 x 128 tiles and the small ones do not pay for them; classes with little
// work ride along with the dominant one.  TLRB_GEMM_SPLIT=0: one launch.
static void launch_gemm_same_op(const std::vector<GemmProb>& probs, DescArena& ar, cudaStream_t s) {
  if (probs.empty()) return;
  static const bool split = !(getenv("TLRB_GEMM_SPLIT") && atoi(getenv("TLRB_GEMM_SPLIT")) == 0) &&
                            !getenv("TLRB_GEMM_CFG");
  if (!split || probs.size() < 16) return launch_gemm_one(probs, -1, ar, s);
  double fl = 0, fc[kNCfg] = {};
  int cnt[kNCfg] = {};
  for (const GemmProb& p : probs) {
    const double f = 2.0 * p.m * p.n * std::max(1, p.k);
    const int c = prob_cfg(p);
    fl += f;
    fc[c] += f;
    ++cnt[c];
  }
  int dom = 5, nsep = 0;
  for (int c = 0; c < kNCfg; ++c)
    if (fc[c] > fc[dom]) dom = c;
  bool sep[kNCfg];
  for (int c = 0; c < kNCfg; ++c) {
    sep[c] = c == dom || (cnt[c] >= 8 && fc[c] >= 0.05 * fl);
    nsep += sep[c];
  }
  if (nsep == 1) return launch_gemm_one(probs, -1, ar, s);
  std::vector<GemmProb> grp[kNCfg];
  for (const GemmProb& p : probs) {
    const int c = prob_cfg(p);
    // a class without its own launch joins the 64 x 64 launch when there is one (any shape runs well enough there),
    // else the dominant one
    grp[sep[c] ? c : (sep[5] ? 5 : dom)].push_back(p);
  }
  for (int c = 0; c < kNCfg; ++c)
    if (!grp[c].empty()) launch_gemm_one(grp[c], c, ar, s);
}

// a launch holds one (ta, tb) combination (compile-time in the kernel): the
// batch is cut by its transposition flags first (batches built by one code
// path are uniform; the exact-tile updates of the TLR Cholesky mix three)
void launch_gemm_impl(const std::vector<GemmProb>& probs, DescArena& ar, cudaStream_t s) {
  if (probs.empty()) return;
  bool uniform = true;
  int first = -1;
  for (const GemmProb& p : probs) {
    if (p.m <= 0 || p.n <= 0) { uniform = false; continue; }   // dropped below
    const int op = (p.ta != 0) * 2 + (p.tb != 0);
    if (first < 0) first = op;
    uniform &= op == first;
  }
  if (first < 0) return;
  if (uniform) return launch_gemm_same_op(probs, ar, s);
  std::vector<GemmProb> byop[4];
  for (const GemmProb& p : probs)
    if (p.m > 0 && p.n > 0) byop[(p.ta != 0) * 2 + (p.tb != 0)].push_back(p);
  for (int o = 0; o < 4; ++o) launch_gemm_same_op(byop[o], ar, s);
}

}  // namespace tlrb

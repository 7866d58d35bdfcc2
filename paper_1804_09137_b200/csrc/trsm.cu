// trsm.cu — triangular kernels of the tile Cholesky:
//   * batched left-lower TRSM  B <- L^-1 B  (panel solves: dense tiles stored
//     transposed, and the V factors of low-rank tiles, linalg.py:94-97 and
//     :121-127) and its transpose B <- L^-T B (backward solve, :180-192);
//   * blocked diagonal-tile POTRF with the not-positive-definite pivot report
//     of LAPACK dpotrf (linalg.py:36-45) and the log-diagonal for the
//     log-determinant (linalg.py:78-79).
// The trailing rank-32 update of POTRF goes through the DMMA GEMM.
#include "common.cuh"
#include <cstdlib>

namespace tlrb {

constexpr int TR_RB = 32;   // row block = warp width

// One CTA solves a slab of W right-hand sides of one problem.  Warp c owns
// column c of the slab; lane r owns row r of the current 32-row block, so the
// 32x32 diagonal solve is warp-local (shuffles, no barriers).  The
// off-diagonal L blocks are staged in shared memory once for all warps.
template <bool TRANS>
__global__ void __launch_bounds__(512) trsm_vbatch_kernel(const TrsmProb* __restrict__ probs,
                                                          const int* __restrict__ start,
                                                          int nprob, int W) {
  extern __shared__ double sm[];
  const int blk = blockIdx.x;
  int lo = 0, hi = nprob - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (start[mid] <= blk) lo = mid; else hi = mid - 1;
  }
  const TrsmProb P = probs[lo];
  const int c0 = (blk - start[lo]) * W;
  const int ncol = min(W, P.nrhs - c0);
  const int n = P.n;
  const int ldx = n + 1;
  double* Xs = sm;                       // W x (n+1)
  double* Ls = sm + (size_t)W * ldx;     // 32 x 33
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nthr = blockDim.x;

  for (int e = threadIdx.x; e < n * ncol; e += nthr) {
    const int r = e % n, c = e / n;
    Xs[c * ldx + r] = P.B[(size_t)(c0 + c) * P.ldb + r];
  }
  __syncthreads();

  const int nblk = (n + TR_RB - 1) / TR_RB;
  for (int bi = 0; bi < nblk; ++bi) {
    const int b = TRANS ? nblk - 1 - bi : bi;
    const int r0 = b * TR_RB;
    const int rb = min(TR_RB, n - r0);
    double acc = 0.0;
    // ---- update with the already solved rows
    const int lbeg = TRANS ? r0 + rb : 0;
    const int lend = TRANS ? n : r0;
    for (int l0 = lbeg; l0 < lend; l0 += 32) {
      const int lb = min(32, lend - l0);
      for (int e = threadIdx.x; e < 32 * 32; e += nthr) {
        int q, rr;
        double v = 0.0;
        if (!TRANS) {  // Ls[q][rr] = L[r0+rr][l0+q]  (coalesced along rr)
          rr = e & 31; q = e >> 5;
          if (rr < rb && q < lb) v = P.L[(size_t)(l0 + q) * P.ldl + r0 + rr];
        } else {       // Ls[q][rr] = L^T[r0+rr][l0+q] = L[l0+q][r0+rr] (coalesced along q)
          q = e & 31; rr = e >> 5;
          if (rr < rb && q < lb) v = P.L[(size_t)(r0 + rr) * P.ldl + l0 + q];
        }
        Ls[q * 33 + rr] = v;
      }
      __syncthreads();
      if (warp < ncol) {  // warp owns column `warp` of the slab (W == #warps)
        double a = 0.0;
#pragma unroll 8
        for (int q = 0; q < lb; ++q) a += Ls[q * 33 + lane] * Xs[warp * ldx + l0 + q];
        acc += a;
      }
      __syncthreads();
    }
    // ---- diagonal block: Ls[q][rr] = L[r0+rr][r0+q] (lower part)
    for (int e = threadIdx.x; e < 32 * 32; e += nthr) {
      const int rr = e & 31, q = e >> 5;
      double v = 0.0;
      if (rr < rb && q < rb && rr >= q) v = P.L[(size_t)(r0 + q) * P.ldl + r0 + rr];
      Ls[q * 33 + rr] = v;
    }
    __syncthreads();
    if (warp < ncol) {
      const int c = warp;
      double x = (lane < rb) ? Xs[c * ldx + r0 + lane] - acc : 0.0;
      if (!TRANS) {
        for (int q = 0; q < rb; ++q) {
          if (lane == q) x /= Ls[q * 33 + q];
          const double xq = __shfl_sync(0xffffffffu, x, q);
          if (lane > q) x -= Ls[q * 33 + lane] * xq;
        }
      } else {
        for (int q = rb - 1; q >= 0; --q) {
          if (lane == q) x /= Ls[q * 33 + q];
          const double xq = __shfl_sync(0xffffffffu, x, q);
          if (lane < q) x -= Ls[lane * 33 + q] * xq;   // L^T[lane][q] = L[q][lane]
        }
      }
      if (lane < rb) Xs[c * ldx + r0 + lane] = x;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < n * ncol; e += nthr) {
    const int r = e % n, c = e / n;
    P.B[(size_t)(c0 + c) * P.ldb + r] = Xs[c * ldx + r];
  }
}

void launch_trsm(const std::vector<TrsmProb>& probs, bool trans, DescArena& ar, cudaStream_t s) {
  std::vector<TrsmProb> keep;
  std::vector<int> start;
  int tot = 0, nmax = 0;
  for (const TrsmProb& p : probs) {
    if (p.n <= 0 || p.nrhs <= 0) continue;
    nmax = std::max(nmax, p.n);
  }
  if (nmax == 0) return;
  // slab width: warps own columns; keep X slab + L block within 200 KB
  int W = 16;
  while (W > 1 && (size_t)W * (nmax + 1) * 8 + 32 * 33 * 8 > 200 * 1024) W >>= 1;
  for (const TrsmProb& p : probs) {
    if (p.n <= 0 || p.nrhs <= 0) continue;
    keep.push_back(p);
    start.push_back(tot);
    tot += (p.nrhs + W - 1) / W;
  }
  start.push_back(tot);
  const size_t smem = (size_t)W * (nmax + 1) * 8 + 32 * 33 * 8;
  const TrsmProb* dp = ar.put(keep, s);
  const int* ds = ar.put(start, s);
  const int threads = 32 * W;
  double fl = 0, by = 0;
  for (const TrsmProb& p : keep) {
    fl += (double)p.n * p.n * p.nrhs;
    by += 8.0 * ((double)p.n * p.n / 2 + 2.0 * p.n * p.nrhs);
  }
  ProfScope ps(K_TRSM, s, fl, by);
  if (trans) {
    allow_smem(trsm_vbatch_kernel<true>, smem);
    trsm_vbatch_kernel<true><<<tot, threads, smem, s>>>(dp, ds, (int)keep.size(), W);
  } else {
    allow_smem(trsm_vbatch_kernel<false>, smem);
    trsm_vbatch_kernel<false><<<tot, threads, smem, s>>>(dp, ds, (int)keep.size(), W);
  }
  post_launch();
}

// Panel solves of one Cholesky step: every problem applies the same L_kk
// (n x n) to its own right-hand sides (dense tiles stored transposed, V
// factors of low-rank tiles).  Blocked forward substitution over row blocks
// of 128: the rows of the block are first updated with the solved rows above
// by one batched DMMA GEMM (B_b -= L_b,0:b X_0:b, all problems in one launch),
// then solved against the 128 x 128 diagonal block by the CUDA-core kernel,
// which is left with n_b / n of the flops.  Small panels (n <= 256 or few
// right-hand sides) keep the single-kernel path.  TLRB_TRSM_BLOCKED=0: always.
void launch_trsm_panel(const std::vector<TrsmProb>& probs, DescArena& ar, cudaStream_t s) {
  static const int IB = getenv("TLRB_TRSM_BLOCKED") ? atoi(getenv("TLRB_TRSM_BLOCKED")) : 128;
  long rhs = 0;
  int n = 0;
  bool same = true;
  for (const TrsmProb& p : probs) {
    if (p.n <= 0 || p.nrhs <= 0) continue;
    if (n == 0) n = p.n;
    same &= p.n == n && p.L == probs[0].L;
    rhs += p.nrhs;
  }
  if (IB <= 0 || !same || n <= 2 * IB || rhs < 256) return launch_trsm(probs, false, ar, s);
  std::vector<TrsmProb> tb;
  std::vector<GemmProb> gu;
  for (int r0 = 0; r0 < n; r0 += IB) {
    const int rb = std::min(IB, n - r0);
    tb.clear(); gu.clear();
    for (const TrsmProb& p : probs) {
      if (p.n <= 0 || p.nrhs <= 0) continue;
      if (r0 > 0)
        gu.push_back({p.L + r0, p.B, p.B + r0, p.B + r0, rb, p.nrhs, r0, p.ldl, p.ldb, p.ldb, p.ldb, 0, 0, 0, -1.0, 1.0});
      tb.push_back({p.L + (size_t)r0 * p.ldl + r0, p.ldl, p.B + r0, p.ldb, rb, p.nrhs});
    }
    launch_gemm(gu, ar, s);
    launch_trsm(tb, false, ar, s);
  }
}

// ------------------------------------------------------------------ POTRF
// Factor the bs x bs diagonal block at (r0, r0) of an n x n tile (lower,
// column-major) and solve the panel below it: A21 <- A21 L11^-T.  info[0]
// is set (first failure wins) with tile index and pivot like dpotrf's
// info-1 (linalg.py:43-44); logdiag[r0 + j] = 2 log L_jj.
__global__ void __launch_bounds__(512) potrf_block_kernel(double* A, int ld, int n, int r0, int bs,
                                                          int tile, int* info, double* logdiag) {
  __shared__ double L[32][33];
  __shared__ int bad;
  const int tid = threadIdx.x;
  if (tid == 0) bad = -1;
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int r = e & 31, c = e >> 5;
    L[c][r] = (r < bs && c < bs) ? A[(size_t)(r0 + c) * ld + r0 + r] : 0.0;
  }
  __syncthreads();
  // right-looking unblocked Cholesky on the 32x32 block (warp 0, lane = row)
  if (tid < 32) {
    const int r = tid;
    for (int j = 0; j < bs; ++j) {
      double d = __shfl_sync(0xffffffffu, L[j][r], j);
      if (!(d > 0.0)) {  // also catches NaN, like dpotrf
        if (r == 0 && bad < 0) bad = j;
        d = 1.0;  // keep going deterministically; result is discarded by the host
        break;
      }
      d = sqrt(d);
      if (r == j) L[j][j] = d;
      if (r > j && r < bs) L[j][r] /= d;
      __syncwarp();
      // trailing update of columns j+1..bs-1 (lane = row)
      for (int c = j + 1; c < bs; ++c)
        if (r >= c && r < bs) L[c][r] -= L[j][r] * L[j][c];
      __syncwarp();
    }
  }
  __syncthreads();
  if (bad >= 0) {
    if (tid == 0) {
      if (atomicCAS(info, 0, 1) == 0) {
        info[1] = tile;
        info[2] = r0 + bad;
      }
    }
  }
  if (tid < bs) logdiag[r0 + tid] = 2.0 * log(L[tid][tid]);
  for (int e = tid; e < 32 * 32; e += blockDim.x) {
    const int r = e & 31, c = e >> 5;
    if (r < bs && c < bs && r >= c) A[(size_t)(r0 + c) * ld + r0 + r] = L[c][r];
  }
  // panel solve: each thread one row r of A21, x L11^T = a
  for (int rr = r0 + bs + tid; rr < n; rr += blockDim.x) {
    double x[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      if (j < bs) {
        double a = A[(size_t)(r0 + j) * ld + rr];
#pragma unroll
        for (int l = 0; l < 32; ++l)
          if (l < j) a -= x[l] * L[l][j];
        x[j] = a / L[j][j];
      }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < bs) A[(size_t)(r0 + j) * ld + rr] = x[j];
  }
}

void launch_potrf_block(double* A, int ld, int n, int r0, int bs, int tile, int* info,
                        double* logdiag, cudaStream_t s) {
  const double rest = n - r0 - bs;
  ProfScope ps(K_POTRF, s, (double)bs * bs * bs / 3 + rest * bs * bs,
               8.0 * (bs * bs * 2.0 + 2.0 * rest * bs));
  potrf_block_kernel<<<1, 512, 0, s>>>(A, ld, n, r0, bs, tile, info, logdiag);
  post_launch();
}

}  // namespace tlrb

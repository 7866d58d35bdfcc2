// qrcp.cu — batched truncated Householder QR with column pivoting (FP64).
//
// Rank-revealing front end of the tile compressor K2: M P = Q [R11 R12] + E
// with ||E||_F^2 tracked exactly (partial column norms recomputed from the
// updated columns at every step, no downdating).  Factorisation stops at
// the first step j with sum_{c>=j} ||M_(j:,c)||^2 <= stop_rel2 ||M||_F^2, so
// the residual enters the truncation tail exactly (compression.py:26-36 rule
// applied to sigma(R) plus ||E||^2).  The Jacobi SVD is then run on R^T,
// which converges in a handful of sweeps (QRCP preconditioning, as in
// LAPACK's dgejsv), and the right singular vectors of M come out directly as
// P * (normalised Jacobi columns).
//
// One CTA (1024 threads) per matrix; the matrix stays in global memory / L2
// and every step streams the trailing columns once (warp per column:
// load, dot with the reflector, update, recompute the partial norm, store).
#include "common.cuh"

namespace tlrb {

__device__ __forceinline__ double wsum_q(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int RPL>
__global__ void __launch_bounds__(1024) qrcp_kernel(const QrcpProb* __restrict__ probs) {
  extern __shared__ double sm[];
  const QrcpProb P = probs[blockIdx.x];
  const int m = P.m, n = P.n, lda = P.lda;
  double* A = P.A;
  double* cn = sm;            // n partial column norms^2
  double* v = cn + n;         // m reflector entries
  double* red = v + m;        // 32 doubles
  int* perm = (int*)(red + 64);
  int* redi = perm + n;       // 32 ints
  __shared__ double s_tau, s_total;
  __shared__ int s_piv, s_stop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int kmax = min(m, n);

  for (int c = tid; c < n; c += blockDim.x) perm[c] = c;
  for (int c = warp; c < n; c += nw) {
    double a = 0.0;
    for (int r = lane; r < m; r += 32) {
      const double x = A[(size_t)c * lda + r];
      a = fma(x, x, a);
    }
    a = wsum_q(a);
    if (lane == 0) cn[c] = a;
  }
  __syncthreads();
  // total ||M||^2 (deterministic: contiguous ranges + tree)
  auto block_sum = [&](int from) -> double {
    double a = 0.0;
    for (int c = from + tid; c < n; c += blockDim.x) a += cn[c];
    a = wsum_q(a);
    if (lane == 0) red[warp] = a;
    __syncthreads();
    double t = 0.0;
    if (warp == 0) {
      t = lane < nw ? red[lane] : 0.0;
      t = wsum_q(t);
    }
    return t;   // valid in warp 0
  };
  {
    const double t = block_sum(0);
    if (tid == 0) s_total = t;
    __syncthreads();
  }
  const double stop = P.stop_rel2 * s_total;
  if (tid == 0) P.resid_out[-1] = s_total;   // ||M||_F^2 (sums[6p+0])
  int j = 0;
  double resid = s_total;
  for (; j < kmax; ++j) {
    // residual and pivot
    const double t = block_sum(j);
    // argmax over cn[j..n): per-thread best, then warp, then block
    double best = -1.0;
    int bi = n;
    for (int c = j + tid; c < n; c += blockDim.x)
      if (cn[c] > best) { best = cn[c]; bi = c; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    __syncthreads();   // red[] reuse
    if (lane == 0) { red[warp] = best; redi[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      best = lane < nw ? red[lane] : -1.0;
      bi = lane < nw ? redi[lane] : n;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        s_piv = bi;
        s_stop = (t <= stop) ? 1 : 0;
        s_total = t;   // current residual
      }
    }
    __syncthreads();
    resid = s_total;
    if (s_stop) break;
    const int p = s_piv;
    if (p != j) {   // swap columns j and p
      for (int r = tid; r < m; r += blockDim.x) {
        const double a = A[(size_t)j * lda + r];
        A[(size_t)j * lda + r] = A[(size_t)p * lda + r];
        A[(size_t)p * lda + r] = a;
      }
      if (tid == 0) {
        const double tc = cn[j]; cn[j] = cn[p]; cn[p] = tc;
        const int ti = perm[j]; perm[j] = perm[p]; perm[p] = ti;
      }
    }
    __syncthreads();
    // Householder reflector of A[j:, j] (dlarfg convention)
    if (warp == 0) {
      double ss = 0.0;
      for (int r = j + 1 + lane; r < m; r += 32) {
        const double x = A[(size_t)j * lda + r];
        ss = fma(x, x, ss);
      }
      ss = wsum_q(ss);
      const double alpha = A[(size_t)j * lda + j];
      double tau = 0.0, beta = alpha, scale = 1.0;
      if (ss != 0.0) {
        beta = -copysign(sqrt(alpha * alpha + ss), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int r = j + 1 + lane; r < m; r += 32) {
        const double x = A[(size_t)j * lda + r] * scale;
        v[r] = x;
        A[(size_t)j * lda + r] = x;
      }
      if (lane == 0) {
        v[j] = 1.0;
        s_tau = tau;
        A[(size_t)j * lda + j] = beta;
      }
    }
    __syncthreads();
    const double tau = s_tau;
    // apply H_j to trailing columns; recompute partial norms over rows > j.
    // Each warp owns whole columns; a column segment A[j:, c] is held in
    // registers (RPL rows per lane, loads issued back to back).
    for (int c = j + 1 + warp; c < n; c += nw) {
      double* col = A + (size_t)c * lda;
      double x[RPL];
      double w0 = 0.0, w1 = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = j + lane + 32 * i;
        x[i] = r < m ? col[r] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = j + lane + 32 * i;
        const double vr = r < m ? v[r] : 0.0;
        if (i & 1) w1 = fma(vr, x[i], w1); else w0 = fma(vr, x[i], w0);
      }
      const double w = wsum_q(w0 + w1) * tau;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = j + lane + 32 * i;
        if (r < m) {
          const double y = x[i] - w * v[r];
          col[r] = y;
          if (r > j) { if (i & 1) a1 = fma(y, y, a1); else a0 = fma(y, y, a0); }
        }
      }
      const double a = wsum_q(a0 + a1);
      if (lane == 0) cn[c] = a;
    }
    __syncthreads();
  }
  if (tid == 0) {
    *P.r_out = j;
    *P.resid_out = (j < kmax) ? resid : 0.0;
    if (j == kmax) {
      // full factorisation: remaining rows (m > n case) hold the residual
      double e = 0.0;
      for (int c = kmax; c < n; ++c) e += cn[c];
      *P.resid_out = e;
    }
  }
  for (int c = tid; c < n; c += blockDim.x) P.perm[c] = perm[c];
}

void launch_qrcp(const std::vector<QrcpProb>& probs, DescArena& ar, cudaStream_t s) {
  if (probs.empty()) return;
  int mmax = 1, nmax = 1;
  double fl = 0, by = 0;
  for (const QrcpProb& p : probs) {
    mmax = std::max(mmax, p.m);
    nmax = std::max(nmax, p.n);
    const double k = std::min(p.m, p.n);
    fl += 4.0 * p.m * p.n * k - 2.0 * (p.m + p.n) * k * k + 4.0 / 3.0 * k * k * k;
    by += 16.0 * p.m * p.n;
  }
  const size_t smem = (size_t)(nmax + mmax + 64) * 8 + (size_t)(nmax + 32) * 4;
  auto kern = mmax <= 512 ? qrcp_kernel<16> : mmax <= 1024 ? qrcp_kernel<32> : qrcp_kernel<64>;
  TLRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const QrcpProb* dp = ar.put(probs, s);
  ProfScope ps(K_QR, s, fl, by);
  kern<<<(unsigned)probs.size(), 1024, smem, s>>>(dp);
  post_launch();
}

}  // namespace tlrb

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
#include <cooperative_groups.h>
#include <cstdlib>

namespace cg = cooperative_groups;

namespace tlrb {

__device__ long long* g_qrcp_prof = nullptr;   // optional phase counters (debug)

__device__ __forceinline__ double A_ld(const double* a, size_t i) { return __ldcg(a + i); }

__device__ __forceinline__ double wsum_q(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int RPL, int NT>
__global__ void __launch_bounds__(NT) qrcp_kernel(const QrcpProb* __restrict__ probs) {
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


// ---------------------------------------------------------------------------
// Cluster variant: the n columns are split into slabs of cpc columns, one slab
// per CTA of a (<=16) thread-block cluster, held in shared memory for the
// whole factorisation.  Columns are never moved.  One cluster barrier per
// pivot step: after it, every CTA reads all published candidates (argmax of
// remaining partial norms + their sums) through distributed shared memory,
// fetches the pivot column from its owner (DSMEM) and forms the Householder
// reflector itself — the same data and the same reduction order give the
// same reflector in every CTA — then updates its own slab and publishes its
// candidate for the next step.  The owner writes the reflector into the
// pivot column only after the next barrier (others may still be reading it).
// perm[0..r) = pivot order, perm[r..n) = the remaining columns in index order.
template <int RPL, int NT>
__global__ void __launch_bounds__(NT) qrcp_cluster_kernel(const QrcpProb* __restrict__ probs, int cpc) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const QrcpProb P = probs[blockIdx.x / CL];
  const int m = P.m, n = P.n, lda = P.lda;
  const int c_lo = crank * cpc, c_hi = min(n, c_lo + cpc), nloc = max(0, c_hi - c_lo);
  double* Ac = sm;                          // cpc x m (column c_lo + k at Ac + k*m)
  double* v = Ac + (size_t)cpc * m;         // m: reflector of the current step
  double* cn = v + m;                       // cpc partial norms^2
  __shared__ double pub_val[2], pub_sum[2];
  __shared__ int pub_idx[2], pub_cnt;
  __shared__ double red[32];
  __shared__ int s_piv, s_stop;
  __shared__ double s_resid, s_total, s_beta, s_tau, s_scale;
  __shared__ unsigned char done[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int kmax = min(m, n);

  for (int e = tid; e < nloc * m; e += blockDim.x) {
    const int k = e / m, r = e - k * m;
    Ac[(size_t)k * m + r] = A_ld(P.A, (size_t)(c_lo + k) * lda + r);
  }
  if (tid < 64) done[tid] = 0;
  __syncthreads();
  for (int k = warp; k < nloc; k += nw) {
    double a = 0.0;
    for (int r = lane; r < m; r += 32) a = fma(Ac[(size_t)k * m + r], Ac[(size_t)k * m + r], a);
    a = wsum_q(a);
    if (lane == 0) cn[k] = a;
  }
  __syncthreads();
  // local candidate for step `step` into pub[par]
  auto publish = [&](int par) {
    if (warp == 0) {
      double best = -1.0, sum = 0.0;
      int bi = n;
      for (int k = lane; k < nloc; k += 32)
        if (!done[k]) {
          sum += cn[k];
          if (cn[k] > best) { best = cn[k]; bi = c_lo + k; }
        }
      sum = wsum_q(sum);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) { pub_val[par] = best; pub_idx[par] = bi; pub_sum[par] = sum; }
    }
  };
  publish(0);
  cl.sync();
  // ||M||^2 = sum of the step-0 sums (fixed shuffle tree: identical everywhere)
  if (warp == 0) {
    double t = lane < CL ? *cl.map_shared_rank(&pub_sum[0], lane) : 0.0;
    t = wsum_q(t);
    if (lane == 0) s_total = t;
  }
  __syncthreads();
  const double total = s_total;
  if (crank == 0 && tid == 0) P.resid_out[-1] = total;
  const double stop = P.stop_rel2 * total;
  int j = 0, pend = -1;   // pend: local index of the owned pivot column awaiting its reflector write
  double pend_beta = 0.0;
  int pend_j = 0;
  double resid = total;
  auto flush_pending = [&]() {
    if (pend >= 0) {
      double* col = Ac + (size_t)pend * m;
      for (int r = pend_j + 1 + tid; r < m; r += blockDim.x) col[r] = v[r];
      if (tid == 0) col[pend_j] = pend_beta;
      __syncthreads();
      pend = -1;
    }
  };
  long long c_cand = 0, c_fetch = 0, c_refl = 0, c_upd = 0, c_pub = 0, c_sync = 0;
  long long tt = kClockProf ? clock64() : 0;
  auto tick = [&](long long& a) {
    if (kClockProf) { const long long nw_ = clock64(); a += nw_ - tt; tt = nw_; }
  };
  for (; j < kmax; ++j) {
    const int par = j & 1;
    if (warp == 0) {
      double best = -1.0, t = 0.0;
      int bi = n;
      if (lane < CL) {
        best = *cl.map_shared_rank(&pub_val[par], lane);
        bi = *cl.map_shared_rank(&pub_idx[par], lane);
        t = *cl.map_shared_rank(&pub_sum[par], lane);
      }
      t = wsum_q(t);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (lane == 0) {
        s_piv = bi;
        s_resid = t;
        s_stop = (t <= stop) ? 1 : 0;
      }
    }
    __syncthreads();
    // the previous step's pivot column may be written now (everyone is past
    // the barrier, so nobody reads it any more); v is still that reflector
    flush_pending();
    resid = s_resid;
    tick(c_cand);
    if (s_stop) break;
    const int p = s_piv;
    const int owner = p / cpc;
    if (crank == 0 && tid == 0) P.perm[j] = p;
    // fetch the pivot column (rows j..m-1) from its owner
    const double* src = cl.map_shared_rank(sm, owner) + (size_t)(p - owner * cpc) * m;
    double part = 0.0;
    for (int r = j + tid; r < m; r += blockDim.x) {
      const double x = src[r];
      v[r] = x;
      if (r > j) part = fma(x, x, part);
    }
    part = wsum_q(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    tick(c_fetch);
    if (warp == 0) {
      double ss = lane < nw ? red[lane] : 0.0;
      ss = wsum_q(ss);
      if (lane == 0) {
        const double alpha = v[j];
        double tau = 0.0, beta = alpha, scale = 1.0;
        if (ss != 0.0) {
          beta = -copysign(sqrt(alpha * alpha + ss), alpha);
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        s_beta = beta;
        s_tau = tau;
        s_scale = scale;
      }
    }
    __syncthreads();
    const double tau = s_tau, scale = s_scale;
    for (int r = j + 1 + tid; r < m; r += blockDim.x) v[r] *= scale;
    if (tid == 0) v[j] = 1.0;
    if (crank == owner) {
      pend = p - c_lo;
      pend_beta = s_beta;
      pend_j = j;
      if (tid == 0) done[pend] = 1;
    }
    __syncthreads();
    tick(c_refl);
    for (int k = warp; k < nloc; k += nw) {
      if (done[k]) continue;
      double* col = Ac + (size_t)k * m;
      double x[RPL];
      double w0 = 0.0, w1 = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int r = j + lane + 32 * i;
        x[i] = r < m ? col[r] : 0.0;
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
      if (lane == 0) cn[k] = a;
    }
    __syncthreads();
    tick(c_upd);
    publish(par ^ 1);
    tick(c_pub);
    cl.sync();
    tick(c_sync);
  }
  if (g_qrcp_prof && blockIdx.x < 16 && tid == 0) {
    long long* q = g_qrcp_prof + 8 * blockIdx.x;
    q[0] = c_cand; q[1] = c_fetch; q[2] = c_refl; q[3] = c_upd; q[4] = c_pub; q[5] = c_sync; q[6] = j;
  }
  flush_pending();
  // write the slab back; remaining columns go to perm[j..n) in index order
  for (int e = tid; e < nloc * m; e += blockDim.x) {
    const int k = e / m, r = e - k * m;
    P.A[(size_t)(c_lo + k) * lda + r] = Ac[(size_t)k * m + r];
  }
  if (tid == 0) {
    int cnt = 0;
    for (int k = 0; k < nloc; ++k) cnt += !done[k];
    pub_cnt = cnt;
  }
  cl.sync();
  if (tid == 0) {
    int off = j;
    for (int c = 0; c < crank; ++c) off += *cl.map_shared_rank(&pub_cnt, c);
    for (int k = 0; k < nloc; ++k)
      if (!done[k]) P.perm[off++] = c_lo + k;
    if (crank == 0) {
      *P.r_out = j;
      *P.resid_out = (j < kmax) ? resid : 0.0;
    }
  }
  cl.sync();   // keep shared memory alive until every remote read is done
}

struct QrcpLaunch {
  const QrcpProb* dp = nullptr;
  int count = 0, mmax = 1, nmax = 1;
  double fl = 0, by = 0;
};

static QrcpLaunch stage(const std::vector<QrcpProb>& probs, DescArena& ar, cudaStream_t s) {
  QrcpLaunch L;
  L.count = (int)probs.size();
  for (const QrcpProb& p : probs) {
    L.mmax = std::max(L.mmax, p.m);
    L.nmax = std::max(L.nmax, p.n);
    const double k = std::min(p.m, std::max(1, p.hint));
    L.fl += 4.0 * p.m * p.n * k - 2.0 * (p.m + p.n) * k * k + 4.0 / 3.0 * k * k * k;
    L.by += 16.0 * p.m * p.n;
  }
  if (L.count) L.dp = ar.put(probs, s);
  return L;
}

static int cluster_cpc(int mmax, int nmax, int& CL) {
  const size_t budget = 200 * 1024;
  int cpc = (int)((budget - 2 * (size_t)mmax * 8) / ((size_t)mmax * 8 + 8));
  cpc = std::min(cpc, 64);
  CL = (nmax + cpc - 1) / cpc;
  if (cpc < 8 || CL > 16 || mmax > 1024) return 0;
  // spread over the full 16-CTA cluster: one column per warp per pivot step
  // (the per-step column update is the longest phase)
  CL = std::max(CL, std::min(16, (nmax + 31) / 32));
  return (nmax + CL - 1) / CL;
}

static void run_cluster(const QrcpLaunch& L, cudaStream_t s) {
  static long long* d_prof = nullptr;
  if (getenv("TLRB_QRCP_PROF")) {
    if (!d_prof) {
      TLRB_CUDA(cudaMalloc(&d_prof, 16 * 8 * sizeof(long long)));
      TLRB_CUDA(cudaMemcpyToSymbol(g_qrcp_prof, &d_prof, sizeof d_prof));
    }
    TLRB_CUDA(cudaMemsetAsync(d_prof, 0, 16 * 8 * sizeof(long long), s));
  }
  int CL = 0;
  const int cpc = cluster_cpc(L.mmax, L.nmax, CL);
  const size_t smem = ((size_t)cpc * L.mmax + (size_t)L.mmax + cpc) * 8;
  auto kern = L.mmax <= 512 ? qrcp_cluster_kernel<16, 1024> : qrcp_cluster_kernel<32, 512>;
  allow_smem(kern, smem);
  if (CL > 8) TLRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  ProfScope ps(K_QR, s, L.fl, L.by);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(L.count * CL));
  cfg.blockDim = dim3(L.mmax <= 512 ? 1024 : 512);   // = NT of the instantiation
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TLRB_CUDA(cudaLaunchKernelEx(&cfg, kern, L.dp, cpc));
  post_launch();
  if (d_prof && getenv("TLRB_QRCP_PROF")) {
    long long hp[16 * 8];
    TLRB_CUDA(cudaMemcpyAsync(hp, d_prof, sizeof hp, cudaMemcpyDeviceToHost, s));
    TLRB_CUDA(cudaStreamSynchronize(s));
    for (int c = 0; c < 16; ++c)
      if (hp[8 * c + 6])
        fprintf(stderr, "[qrcp-prof] cta %d cand %lld fetch %lld refl %lld upd %lld pub %lld sync %lld steps %lld\n", c,
                hp[8 * c], hp[8 * c + 1], hp[8 * c + 2], hp[8 * c + 3], hp[8 * c + 4], hp[8 * c + 5], hp[8 * c + 6]);
  }
}

static void run_single(const QrcpLaunch& L, cudaStream_t s) {
  const size_t smem = (size_t)(L.nmax + L.mmax + 64) * 8 + (size_t)(L.nmax + 32) * 4;
  auto kern = L.mmax <= 512 ? qrcp_kernel<16, 1024> : L.mmax <= 1024 ? qrcp_kernel<32, 512>
                                                     : qrcp_kernel<64, 256>;
  const int nt = L.mmax <= 512 ? 1024 : L.mmax <= 1024 ? 512 : 256;
  allow_smem(kern, smem);
  ProfScope ps(K_QR, s, L.fl, L.by);
  kern<<<(unsigned)L.count, nt, smem, s>>>(L.dp);
  post_launch();
}

// Problems with a large predicted rank go to the cluster kernel (latency:
// ~3 us per pivot step on 16 SMs); the rest to the one-CTA kernel (throughput:
// they finish in few steps).  The two groups run concurrently (side stream
// forked after the descriptors are staged, joined before returning).
void launch_qrcp(const std::vector<QrcpProb>& probs, std::vector<char>& gathered, DescArena& ar,
                 cudaStream_t s) {
  gathered.assign(probs.size(), 0);
  if (probs.empty()) return;
  static const bool no_cluster = getenv("TLRB_QRCP_NOCLUSTER") != nullptr;
  static const int thr_env = getenv("TLRB_QRCP_CLUSTER_MIN") ? atoi(getenv("TLRB_QRCP_CLUSTER_MIN")) : -1;
  std::vector<QrcpProb> big, small;
  std::vector<int> big_idx;
  int mmax = 1, nmax = 1;
  for (const QrcpProb& p : probs) { mmax = std::max(mmax, p.m); nmax = std::max(nmax, p.n); }
  int CL = 0;
  const bool cluster_ok = !no_cluster && cluster_cpc(mmax, nmax, CL) > 0;
  // "big" problems (predicted QRCP steps above thr) leave the one-CTA kernel;
  // without the cluster kernel (nb > ~500) even modest ones go to the blocked
  // path: the one-CTA kernel streams an nb x nb trailing matrix per pivot
  // (C3: thr 32 -> 16.0 s vs 16.2 s at 160)
  const int thr = thr_env >= 0 ? thr_env : (cluster_ok ? 160 : 32);
  // blocked path available for every tile size up to 2048 (the panel of b
  // columns fits in shared memory); the cluster kernel only while a matrix
  // fits in the shared memory of a 16-CTA cluster (nb <= ~500)
  static const int blocked_min = getenv("TLRB_QRCP_BLOCKED") ? atoi(getenv("TLRB_QRCP_BLOCKED")) : 8;
  const bool blocked_ok = blocked_min > 0 && mmax <= 2048 && nmax <= 2048;
  for (size_t i = 0; i < probs.size(); ++i) {
    if ((cluster_ok || blocked_ok) && probs[i].hint > thr) { big.push_back(probs[i]); big_idx.push_back((int)i); }
    else small.push_back(probs[i]);
  }
  // large problems: blocked randomized QRCP (bqrcp.cu), GEMM-based and not
  // bound by cluster occupancy; TLRB_QRCP_BLOCKED=<min batch> (0 = never)
  // The cluster kernel has the lower latency for a lone matrix, the blocked
  // one the higher throughput: it is used once the big problems exceed the
  // clusters that can be co-resident (7 of 16 CTAs on 148 SMs).
  // Without the cluster kernel (large tiles) the blocked path takes the big
  // problems at any batch size: a one-CTA QRCP of a 760 x 760 matrix streams
  // the whole trailing matrix through one SM at every pivot.
  if (blocked_ok && !big.empty() && ((int)big.size() >= blocked_min || !cluster_ok)) {
    const QrcpLaunch Ls = stage(small, ar, s);
    if (!Ls.count) { launch_qrcp_blocked(big, ar, s); return; }
    LaunchCtx& cx = launch_ctx();
    cudaStream_t& side2 = cx.q_side2;
    cudaEvent_t& f2 = cx.q_f2;
    cudaEvent_t& j2 = cx.q_j2;
    if (!side2) {
      TLRB_CUDA(cudaStreamCreateWithFlags(&side2, cudaStreamNonBlocking));
      TLRB_CUDA(cudaEventCreateWithFlags(&f2, cudaEventDisableTiming));
      TLRB_CUDA(cudaEventCreateWithFlags(&j2, cudaEventDisableTiming));
    }
    TLRB_CUDA(cudaEventRecord(f2, s));
    TLRB_CUDA(cudaStreamWaitEvent(side2, f2, 0));
    run_single(Ls, side2);
    launch_qrcp_blocked(big, ar, s);
    TLRB_CUDA(cudaEventRecord(j2, side2));
    TLRB_CUDA(cudaStreamWaitEvent(s, j2, 0));
    return;
  }
  const QrcpLaunch Lb = stage(big, ar, s), Ls = stage(small, ar, s);
  if (!Lb.count) { run_single(Ls, s); return; }
  for (int i : big_idx) gathered[i] = 1;
  if (!Ls.count) { run_cluster(Lb, s); return; }
  LaunchCtx& cx = launch_ctx();
  cudaStream_t& side = cx.q_side;
  cudaEvent_t& fork_ev = cx.q_fork;
  cudaEvent_t& join_ev = cx.q_join;
  if (!side) {
    TLRB_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    TLRB_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
    TLRB_CUDA(cudaEventCreateWithFlags(&join_ev, cudaEventDisableTiming));
  }
  TLRB_CUDA(cudaEventRecord(fork_ev, s));
  TLRB_CUDA(cudaStreamWaitEvent(side, fork_ev, 0));
  run_single(Ls, side);
  run_cluster(Lb, s);
  TLRB_CUDA(cudaEventRecord(join_ev, side));
  TLRB_CUDA(cudaStreamWaitEvent(s, join_ev, 0));
}

}  // namespace tlrb

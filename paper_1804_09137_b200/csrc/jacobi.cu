// jacobi.cu — batched one-sided (Hestenes) Jacobi SVD with the reference's
// truncation rule fused into its epilogue (K2's accurate-SVD stage).
//
// The reference truncates at the smallest k with ||s[k:]|| <= eps ||s||,
// summing the tail from the small end (compression.py:26-36), after dropping
// singular values at or below a noise floor in recompression
// (compression.py:78-79).  Parity needs the *same* truncation decisions, so
// the singular values must be accurate to ~u ||A|| (hard
// part 2).  One-sided Jacobi is backward stable column by column and yields
// exactly that.
//
// Parallel layout: X (m x s, column-major) lives in global memory / L2 and is
// cut into column blocks of B.  One thread-block CLUSTER (1..8 CTAs, sized by
// the matrix) owns one matrix.  A sweep is a round-robin tournament over the
// blocks: in each round the cluster's CTAs take disjoint block pairs (I, J),
// stage both blocks in shared memory, rotate all B x B cross column pairs
// (one warp per pair, B disjoint pairs per inner round) and write them back;
// a cluster barrier separates rounds.  Pairs inside a block are rotated once
// per sweep (round 0, where every block appears exactly once).  The sweep
// loop stops when no pair of the whole cluster needed a rotation
// (|a_p.a_q| <= m eps ||a_p|| ||a_q||, LAPACK dgesvj's tolerance).
// Afterwards CTA 0 computes the column norms (= singular values), sorts them,
// writes normalised columns in sorted order, and applies the truncation rule
// with the sketch residual e2 (aux[0]) and the noise floor (aux[1]).
#include "common.cuh"
#include <cfloat>
#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace tlrb {

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// rotate columns a and b (length m, shared memory); true if rotated
__device__ __forceinline__ bool rotate_pair(double* a, double* b, int m, double tol, double tiny2,
                                            int lane) {
  double al = 0.0, be = 0.0, ga = 0.0;
  for (int r = lane; r < m; r += 32) {
    const double x = a[r], y = b[r];
    al = fma(x, x, al);
    be = fma(y, y, be);
    ga = fma(x, y, ga);
  }
  al = wsum(al);
  be = wsum(be);
  ga = wsum(ga);
  if (ga == 0.0 || al <= tiny2 || be <= tiny2) return false;
  if (fabs(ga) <= tol * sqrt(al) * sqrt(be)) return false;
  const double zeta = (be - al) / (2.0 * ga);
  const double t = copysign(1.0, zeta) / (fabs(zeta) + hypot(1.0, zeta));
  const double c = 1.0 / sqrt(1.0 + t * t);
  const double sn = c * t;
  for (int r = lane; r < m; r += 32) {
    const double x = a[r], y = b[r];
    a[r] = c * x - sn * y;
    b[r] = sn * x + c * y;
  }
  return true;
}

// round-robin tournament over nplayers (even): match idx of round r
__device__ __forceinline__ void match(int r, int idx, int np, int& p, int& q) {
  const int rot = np - 1;
  if (idx == 0) {
    p = r % rot;
    q = np - 1;
  } else {
    p = (r + idx) % rot;
    q = (r - idx + rot) % rot;
  }
}

__global__ void __launch_bounds__(512) jacobi_cluster_kernel(const JacobiProb* __restrict__ probs, int B,
                                                             int max_sweeps) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks();
  const int crank = (int)cl.block_rank();
  const JacobiProb P = probs[blockIdx.x / CL];
  const int m = P.m, s = P.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nthr = blockDim.x;
  double* S0 = sm;
  double* S1 = sm + (size_t)B * m;
  __shared__ int rot_flag;
  // rotation tolerance: LAPACK dgesvj's m*eps, tightened for very small acc
  // (the truncated product M V V^T inherits the columns' non-orthogonality);
  // columns below tau*||M|| carry no information for the truncation at acc
  // (their energy is preserved by the rotations) and are not rotated.
  const double tol = fmin((double)m * DBL_EPSILON, fmax(0.01 * P.eps, 2.0 * sqrt((double)m) * DBL_EPSILON));
  const double tau = fmax(1e-3 * P.eps, 2.0 * sqrt((double)m) * DBL_EPSILON);
  const double tiny2 = tau * tau * P.aux[2];
  const int nblk = (s + B - 1) / B;
  const int np = nblk + (nblk & 1);   // pad with a dummy block
  int sweeps = 0;

  auto load = [&](double* dst, int blk) {
    const int c0 = blk * B, nc = min(B, s - c0);
    for (int e = threadIdx.x; e < m * B; e += nthr) {
      const int r = e % m, c = e / m;
      dst[c * m + r] = (c < nc) ? __ldcg(P.X + (size_t)(c0 + c) * P.ldx + r) : 0.0;
    }
  };
  auto store = [&](const double* src, int blk) {
    const int c0 = blk * B, nc = min(B, s - c0);
    for (int e = threadIdx.x; e < m * nc; e += nthr) {
      const int r = e % m, c = e / m;
      __stcg(P.X + (size_t)(c0 + c) * P.ldx + r, src[c * m + r]);
    }
  };
  auto within = [&](double* S, int nc, bool& any) {   // all pairs inside one block
    for (int r = 0; r < B - 1; ++r) {
      if (warp < B / 2) {
        int p, q;
        match(r, warp, B, p, q);
        if (p < nc && q < nc) any |= rotate_pair(S + p * m, S + q * m, m, tol, tiny2, lane);
      }
      __syncthreads();
    }
  };

  if (s > 1) {
    for (sweeps = 1; sweeps <= max_sweeps; ++sweeps) {
      bool any = false;
      for (int r = 0; r < np - 1; ++r) {
        for (int idx = crank; idx < np / 2; idx += CL) {
          int I, J;
          match(r, idx, np, I, J);
          if (I >= nblk) { const int t = I; I = J; J = t; }   // I real, J maybe dummy
          const bool realJ = J < nblk;
          load(S0, I);
          if (realJ) load(S1, J);
          __syncthreads();
          const int ncI = min(B, s - I * B);
          const int ncJ = realJ ? min(B, s - J * B) : 0;
          if (r == 0) {
            within(S0, ncI, any);
            if (realJ) within(S1, ncJ, any);
          }
          if (realJ) {
            for (int rr = 0; rr < B; ++rr) {
              if (warp < B) {
                const int p = warp, q = (warp + rr) % B;
                if (p < ncI && q < ncJ) any |= rotate_pair(S0 + p * m, S1 + q * m, m, tol, tiny2, lane);
              }
              __syncthreads();
            }
          }
          store(S0, I);
          if (realJ) store(S1, J);
          __syncthreads();
        }
        __threadfence();
        cl.sync();
      }
      // cluster-wide convergence decision through distributed shared memory
      if (threadIdx.x == 0) rot_flag = 0;
      __syncthreads();
      if (any && lane == 0) atomicOr(&rot_flag, 1);
      cl.sync();
      int total = 0;
      if (threadIdx.x == 0)
        for (int c = 0; c < CL; ++c) total |= *cl.map_shared_rank(&rot_flag, c);
      __syncthreads();
      if (threadIdx.x == 0) S0[0] = (double)total;   // broadcast via smem (S0 is free here)
      __syncthreads();
      const bool more = S0[0] != 0.0;
      cl.sync();   // everyone has read the flags before they are reset
      if (!more) break;
    }
  }
  if (crank != 0) return;
  if (threadIdx.x == 0) *P.sweeps_out = sweeps;

  // ---- singular values = column norms; sort descending; normalise
  double* sig = sm;                // s values (shared memory reused)
  int* perm = (int*)(sm + s);
  for (int c = warp; c < s; c += nw) {
    double a = 0.0;
    for (int r = lane; r < m; r += 32) {
      const double x = __ldcg(P.X + (size_t)c * P.ldx + r);
      a = fma(x, x, a);
    }
    a = wsum(a);
    if (lane == 0) sig[c] = sqrt(a);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < s; c += nthr) {
    const double v = sig[c];
    int pos = 0;
    for (int i = 0; i < s; ++i) {
      const double w = sig[i];
      pos += (w > v) || (w == v && i < c);
    }
    perm[pos] = c;
  }
  __syncthreads();
  for (int pos = warp; pos < s; pos += nw) {
    const int c = perm[pos];
    const double v = sig[c];
    const double inv = v > 0.0 ? 1.0 / v : 0.0;
    for (int r = lane; r < m; r += 32)
      P.Vout[(size_t)pos * P.ldv + r] = __ldcg(P.X + (size_t)c * P.ldx + r) * inv;
    if (lane == 0) P.sigma[pos] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const double e2 = P.aux[0], noise = P.aux[1];
    int S = 0;
    while (S < s && P.sigma[S] > noise) ++S;
    double fro2 = e2;
    for (int i = 0; i < S; ++i) fro2 += P.sigma[i] * P.sigma[i];
    int k = S;
    if (fro2 == 0.0) {
      k = 0;
    } else {
      const double thr = P.eps * P.eps * fro2;
      double tail = e2;
      for (int i = S - 1; i >= 0; --i) {
        tail += P.sigma[i] * P.sigma[i];
        if (tail <= thr) k = i; else break;
      }
    }
    *P.rank_out = k;
  }
}

void launch_jacobi(const std::vector<JacobiProb>& probs, DescArena& ar, cudaStream_t s) {
  if (probs.empty()) return;
  int mmax = 1;
  for (const JacobiProb& p : probs) mmax = std::max(mmax, p.m);
  int B = 16;
  while (B > 2 && (size_t)2 * B * mmax * 8 > 200 * 1024) B >>= 1;
  // group by cluster size: one CTA per block pair of a round, at most 8
  std::vector<JacobiProb> groups[4];
  for (const JacobiProb& p : probs) {
    const int nblk = (p.s + B - 1) / B;
    const int pairs = (nblk + 1) / 2;
    const int g = pairs <= 1 ? 0 : pairs <= 2 ? 1 : pairs <= 4 ? 2 : 3;
    groups[g].push_back(p);
  }
  for (int g = 0; g < 4; ++g) {
    if (groups[g].empty()) continue;
    const int CL = 1 << g;
    int smax = 1;
    for (const JacobiProb& p : groups[g]) smax = std::max(smax, p.s);
    const size_t smem = std::max((size_t)2 * B * mmax * 8, (size_t)smax * 12 + 64);
    TLRB_CUDA(cudaFuncSetAttribute(jacobi_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
    const JacobiProb* dp = ar.put(groups[g], s);
    double by = 0;
    for (const JacobiProb& p : groups[g]) by += 8.0 * 3.0 * p.m * p.s;
    ProfScope ps(K_JACOBI, s, 0, by);  // flops added once the sweep counts are known
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(groups[g].size() * CL));
    cfg.blockDim = dim3(32 * B);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TLRB_CUDA(cudaLaunchKernelEx(&cfg, jacobi_cluster_kernel, dp, B, 60));
    post_launch();
  }
}

}  // namespace tlrb

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
// Layout: X (m x s, column-major, global/L2) holds the columns to be
// orthogonalised (X = B^T of the range-finder, or M^T when unsketched).  One
// CTA per matrix runs block-cyclic sweeps: block I (B columns) stays resident
// in shared memory while blocks J > I stream through; every column pair is
// rotated by one warp (dot products by lane-strided FMA + xor-shuffle
// reduction).  After convergence the column norms are the singular values;
// the columns are normalised, sorted descending and written to Vout, and the
// truncation rank is computed from the sorted values plus the sketch
// residual e2 (aux[0]).
#include "common.cuh"
#include <cfloat>

namespace tlrb {

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// rotate columns a and b (length m, in shared memory); returns true if rotated
__device__ __forceinline__ bool rotate_pair(double* a, double* b, int m, double tol, int lane) {
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
  if (ga == 0.0 || al == 0.0 || be == 0.0) return false;
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

__global__ void jacobi_kernel(const JacobiProb* __restrict__ probs, int B, int max_sweeps) {
  extern __shared__ double sm[];
  const JacobiProb P = probs[blockIdx.x];
  const int m = P.m, s = P.s;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nthr = blockDim.x;
  double* S0 = sm;
  double* S1 = sm + (size_t)B * m;
  __shared__ int rotated;
  const double tol = sqrt((double)m) * DBL_EPSILON;
  const int nblk = (s + B - 1) / B;
  int sweeps = 0;

  auto load = [&](double* dst, int blk) {
    const int c0 = blk * B, nc = min(B, s - c0);
    for (int e = threadIdx.x; e < m * B; e += nthr) {
      const int r = e % m, c = e / m;
      dst[c * m + r] = (c < nc) ? P.X[(size_t)(c0 + c) * P.ldx + r] : 0.0;
    }
  };
  auto store = [&](const double* src, int blk) {
    const int c0 = blk * B, nc = min(B, s - c0);
    for (int e = threadIdx.x; e < m * nc; e += nthr) {
      const int r = e % m, c = e / m;
      P.X[(size_t)(c0 + c) * P.ldx + r] = src[c * m + r];
    }
  };

  if (s > 1) {
    for (sweeps = 1; sweeps <= max_sweeps; ++sweeps) {
      if (threadIdx.x == 0) rotated = 0;
      __syncthreads();
      bool any = false;
      for (int I = 0; I < nblk; ++I) {
        load(S0, I);
        __syncthreads();
        const int ncI = min(B, s - I * B);
        // pairs inside block I: round-robin tournament, B-1 rounds of B/2 pairs
        for (int r = 0; r < B - 1; ++r) {
          if (warp < B / 2) {
            int p, q;
            if (warp == 0) { p = r; q = B - 1; }
            else { p = (r + warp) % (B - 1); q = (r - warp + (B - 1)) % (B - 1); }
            if (p < ncI && q < ncI) any |= rotate_pair(S0 + p * m, S0 + q * m, m, tol, lane);
          }
          __syncthreads();
        }
        for (int J = I + 1; J < nblk; ++J) {
          load(S1, J);
          __syncthreads();
          const int ncJ = min(B, s - J * B);
          for (int r = 0; r < B; ++r) {
            if (warp < B) {
              const int p = warp, q = (warp + r) % B;
              if (p < ncI && q < ncJ) any |= rotate_pair(S0 + p * m, S1 + q * m, m, tol, lane);
            }
            __syncthreads();
          }
          store(S1, J);
          __syncthreads();
        }
        store(S0, I);
        __syncthreads();
      }
      if (any && lane == 0) rotated = 1;
      __syncthreads();
      if (!rotated) break;
      __syncthreads();
    }
  }
  if (threadIdx.x == 0) *P.sweeps_out = sweeps;

  // ---- singular values = column norms; sort descending; normalise
  double* sig = sm;                // s values (shared memory reused)
  int* perm = (int*)(sm + s);
  for (int c = warp; c < s; c += nw) {
    double a = 0.0;
    for (int r = lane; r < m; r += 32) {
      const double x = P.X[(size_t)c * P.ldx + r];
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
      P.Vout[(size_t)pos * P.ldv + r] = P.X[(size_t)c * P.ldx + r] * inv;
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
  int mmax = 1, smax = 1;
  for (const JacobiProb& p : probs) {
    mmax = std::max(mmax, p.m);
    smax = std::max(smax, p.s);
  }
  int B = 16;
  while (B > 2 && (size_t)2 * B * mmax * 8 > 200 * 1024) B >>= 1;
  size_t smem = std::max((size_t)2 * B * mmax * 8, (size_t)smax * 12 + 64);
  TLRB_CUDA(cudaFuncSetAttribute(jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  const JacobiProb* dp = ar.put(probs, s);
  jacobi_kernel<<<(unsigned)probs.size(), 32 * B, smem, s>>>(dp, B, 60);
  post_launch();
}

}  // namespace tlrb

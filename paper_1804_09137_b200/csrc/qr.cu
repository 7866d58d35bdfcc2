// qr.cu — batched blocked Householder QR with explicit Q (FP64).
//
// Used by the compression kernel K2 to orthonormalise the sketch Y = M Omega
// (range finder).  The reference's compression does its orthogonal
// factorisations with LAPACK dgesdd / dgeqrf+dorgqr (compression.py:48,70-71);
// here one CTA owns one matrix: an m x PB panel is factored in shared memory
// (unblocked Householder, LAPACK dlarfg sign convention), its compact-WY
// factor T is formed (dlarft, forward/columnwise), and the block reflector is
// applied to the trailing columns chunk by chunk (each chunk staged once in
// shared memory: W = V^T C, W = T^T W, C -= V W).  Q is then accumulated by
// applying the block reflectors in reverse to [I; 0].
#include "common.cuh"

namespace tlrb {

struct QrCfg { int PB, CW, ld; };

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// V_i[r] with the implicit unit diagonal and zeros above it
__device__ __forceinline__ double vval(const double* Vp, int ld, int i, int r) {
  return r < i ? 0.0 : (r == i ? 1.0 : Vp[i * ld + r]);
}

// Apply (I - V op(T) V^T) to the columns [cbeg, cend) of G (rows p0..m-1),
// G column-major with leading dimension ldg.  transT: use T^T (factorisation).
__device__ void apply_block_reflector(const double* Vp, const double* Ts, int pb, int mr,
                                      double* G, int ldg, int p0, int cbeg, int cend,
                                      bool transT, double* Cs, double* Ws, double* W2,
                                      const QrCfg& cf) {
  const int tid = threadIdx.x, nthr = blockDim.x;
  for (int cb = cbeg; cb < cend; cb += cf.CW) {
    const int cw = min(cf.CW, cend - cb);
    for (int e = tid; e < mr * cw; e += nthr) {
      const int r = e % mr, c = e / mr;
      Cs[c * cf.ld + r] = G[(size_t)(cb + c) * ldg + p0 + r];
    }
    __syncthreads();
    // W = V^T C  (pb x cw)
    for (int e = tid; e < pb * cw; e += nthr) {
      const int c = e % cw, i = e / cw;
      double a = Cs[c * cf.ld + i];  // unit diagonal
      for (int r = i + 1; r < mr; ++r) a += Vp[i * cf.ld + r] * Cs[c * cf.ld + r];
      Ws[i * cf.CW + c] = a;
    }
    __syncthreads();
    // W2 = op(T) W ; T upper triangular (Ts[i*16+j] = T[i][j])
    for (int e = tid; e < pb * cw; e += nthr) {
      const int c = e % cw, i = e / cw;
      double a = 0.0;
      if (transT) {
        for (int l = 0; l <= i; ++l) a += Ts[l * 16 + i] * Ws[l * cf.CW + c];
      } else {
        for (int l = i; l < pb; ++l) a += Ts[i * 16 + l] * Ws[l * cf.CW + c];
      }
      W2[i * cf.CW + c] = a;
    }
    __syncthreads();
    // C -= V W2
    for (int e = tid; e < mr * cw; e += nthr) {
      const int r = e % mr, c = e / mr;
      double a = 0.0;
      const int imax = min(pb - 1, r);
      for (int i = 0; i <= imax; ++i) a += vval(Vp, cf.ld, i, r) * W2[i * cf.CW + c];
      G[(size_t)(cb + c) * ldg + p0 + r] = Cs[c * cf.ld + r] - a;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(512) qr_kernel(const QrProb* __restrict__ probs, QrCfg cf) {
  extern __shared__ double sm[];
  const QrProb P = probs[blockIdx.x];
  const int m = P.m, s = P.s;
  double* Vp = sm;                              // PB x ld
  double* Cs = Vp + (size_t)cf.PB * cf.ld;      // CW x ld
  double* Ts = Cs + (size_t)cf.CW * cf.ld;      // 16 x 16
  double* Ws = Ts + 256;                        // 16 x CW
  double* W2 = Ws + 16 * cf.CW;                 // 16 x CW
  __shared__ double tau[16], zz[16], bcast[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int kmax = min(m, s);

  for (int p0 = 0; p0 < kmax; p0 += cf.PB) {
    const int pb = min(cf.PB, kmax - p0);
    const int mr = m - p0;
    for (int e = tid; e < mr * pb; e += blockDim.x) {
      const int r = e % mr, c = e / mr;
      Vp[c * cf.ld + r] = P.A[(size_t)(p0 + c) * P.lda + p0 + r];
    }
    __syncthreads();
    for (int j = 0; j < pb; ++j) {
      if (warp == 0) {
        double ss = 0.0;
        for (int r = j + 1 + lane; r < mr; r += 32) ss += Vp[j * cf.ld + r] * Vp[j * cf.ld + r];
        ss = warp_sum(ss);
        const double alpha = Vp[j * cf.ld + j];
        double t = 0.0, beta = alpha, scale = 0.0;
        if (ss != 0.0) {
          beta = -copysign(sqrt(alpha * alpha + ss), alpha);
          t = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        for (int r = j + 1 + lane; r < mr; r += 32) Vp[j * cf.ld + r] *= (ss != 0.0 ? scale : 1.0);
        if (lane == 0) {
          tau[j] = t;
          bcast[0] = beta;
        }
      }
      __syncthreads();
      // apply H_j to panel columns j+1..pb-1 (one warp per column)
      const double t = tau[j];
      for (int c = j + 1 + warp; c < pb; c += nw) {
        double a = (lane == 0) ? Vp[c * cf.ld + j] : 0.0;   // v_j[j] = 1
        for (int r = j + 1 + lane; r < mr; r += 32) a += Vp[j * cf.ld + r] * Vp[c * cf.ld + r];
        a = warp_sum(a);
        const double f = t * a;
        if (lane == 0) Vp[c * cf.ld + j] -= f;
        for (int r = j + 1 + lane; r < mr; r += 32) Vp[c * cf.ld + r] -= f * Vp[j * cf.ld + r];
      }
      __syncthreads();
      if (tid == 0) Vp[j * cf.ld + j] = bcast[0];  // R diagonal (V's unit diag is implicit)
      __syncthreads();
    }
    // T factor (dlarft forward, columnwise): T[j][j] = tau_j,
    // T[0:j, j] = -tau_j T[0:j,0:j] (V[:,0:j]^T v_j)
    for (int j = 0; j < pb; ++j) {
      if (warp < j) {
        const int i = warp;  // z_i = V_i^T v_j = V_i[j] + sum_{r>j} V_i[r] V_j[r]
        double a = 0.0;
        for (int r = j + 1 + lane; r < mr; r += 32) a += Vp[i * cf.ld + r] * Vp[j * cf.ld + r];
        a = warp_sum(a);
        if (lane == 0) zz[i] = a + Vp[i * cf.ld + j];
      }
      __syncthreads();
      if (tid < j) {
        double a = 0.0;
        for (int l = tid; l < j; ++l) a += Ts[tid * 16 + l] * zz[l];
        Ts[tid * 16 + j] = -tau[j] * a;
      }
      if (tid == j) Ts[j * 16 + j] = tau[j];
      if (tid < 16 && tid > j) Ts[tid * 16 + j] = 0.0;
      __syncthreads();
    }
    for (int e = tid; e < 16 * 16; e += blockDim.x)
      if ((e >> 4) >= pb || (e & 15) >= pb) Ts[e] = 0.0;
    __syncthreads();
    // write the panel back (R upper part + V below the diagonal) and save T
    for (int e = tid; e < mr * pb; e += blockDim.x) {
      const int r = e % mr, c = e / mr;
      P.A[(size_t)(p0 + c) * P.lda + p0 + r] = Vp[c * cf.ld + r];
    }
    for (int e = tid; e < 256; e += blockDim.x) P.T[(size_t)p0 * 16 + e] = Ts[e];
    __syncthreads();
    apply_block_reflector(Vp, Ts, pb, mr, P.A, P.lda, p0, p0 + pb, s, true, Cs, Ws, W2, cf);
  }

  // ---- form Q = H_0 ... H_{k-1} [I; 0]  (m x s, columns >= kmax stay 0)
  for (int e = tid; e < m * s; e += blockDim.x) {
    const int r = e % m, c = e / m;
    P.Q[(size_t)c * P.ldq + r] = (r == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const int npan = (kmax + cf.PB - 1) / cf.PB;
  for (int pi = npan - 1; pi >= 0; --pi) {
    const int p0 = pi * cf.PB;
    const int pb = min(cf.PB, kmax - p0);
    const int mr = m - p0;
    for (int e = tid; e < mr * pb; e += blockDim.x) {
      const int r = e % mr, c = e / mr;
      Vp[c * cf.ld + r] = P.A[(size_t)(p0 + c) * P.lda + p0 + r];
    }
    for (int e = tid; e < 256; e += blockDim.x) Ts[e] = P.T[(size_t)p0 * 16 + e];
    __syncthreads();
    apply_block_reflector(Vp, Ts, pb, mr, P.Q, P.ldq, p0, p0, s, false, Cs, Ws, W2, cf);
  }
}

void launch_qr(const std::vector<QrProb>& probs, DescArena& ar, cudaStream_t s) {
  if (probs.empty()) return;
  int mmax = 1;
  for (const QrProb& p : probs) mmax = std::max(mmax, p.m);
  QrCfg cf;
  cf.ld = mmax + 1;
  const size_t budget = 200 * 1024;
  cf.PB = 16;
  cf.CW = 32;
  auto need = [&](const QrCfg& c) {
    return ((size_t)(c.PB + c.CW) * c.ld + 256 + 32 * c.CW) * sizeof(double);
  };
  while (need(cf) > budget && cf.CW > 4) cf.CW >>= 1;
  while (need(cf) > budget && cf.PB > 4) cf.PB >>= 1;
  const size_t smem = need(cf);
  TLRB_CUDA(cudaFuncSetAttribute(qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)smem));
  const QrProb* dp = ar.put(probs, s);
  double fl = 0, by = 0;
  for (const QrProb& p : probs) {
    const double m = p.m, k = std::min(p.m, p.s);
    fl += 2.0 * (2.0 * m * k * k - 2.0 / 3.0 * k * k * k);  // geqrf + orgqr
    by += 8.0 * (2.0 * m * p.s);
  }
  ProfScope ps(K_QR, s, fl, by);
  qr_kernel<<<(unsigned)probs.size(), 512, smem, s>>>(dp, cf);
  post_launch();
}

}  // namespace tlrb

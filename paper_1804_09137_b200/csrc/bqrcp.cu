// bqrcp.cu — blocked randomized QR with column pivoting (HQRRP scheme:
// Martinsson, Quintana-Orti, Heavner, van de Geijn 2017) for the large
// compressions of K2.
//
// Same contract as qrcp.cu (QrcpProb): M P = Q [R11 R12] + E, stop at the
// first index s with ||E||_F^2 <= stop_rel2 ||M||_F^2, R (upper trapezoidal,
// pivoted column order) left in A, perm, r_out = s, resid_out[0] = ||E||^2,
// resid_out[-1] = ||M||^2.  Columns are physically permuted (gathered = 0).
//
// Instead of one pivot (one global argmax + one rank-1 update of the whole
// trailing matrix) per step, b pivots are chosen at once from a Gaussian
// sketch Y = Omega A_trailing (l = b + 8 rows) by a small QRCP on Y, the b
// selected columns are factorised by an unpivoted Householder QR in one CTA,
// and the trailing matrix gets the compact-WY block reflector through three
// batched DMMA GEMMs.  The residual is recomputed exactly from the updated
// trailing matrix after every block, and the stopping index inside the last
// block comes from the exact R row norms, so the truncation accounting is the
// same as the unblocked kernel's; only the pivot order differs (sketch
// pivots are as rank-revealing as greedy ones in practice, and the
// subsequent Jacobi SVD of R is insensitive to it).
//
// Per block and problem: sketch GEMM, pick (QRCP of Y + column swaps), panel
// QR (+ T of the compact WY form), W = V^T A2, W = T^T W, A2 -= V W, exact
// norms + stop test.  All kernels take a per-problem `active` flag, so one
// host loop drives a whole batch without synchronising per block.
#include "common.cuh"
#include <cstdlib>

namespace tlrb {

namespace {

struct BqState {
  double stop;   // absolute threshold stop_rel2 * ||M||^2
  int active;
  int pad;
};

__device__ __forceinline__ double wsum_b(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic block sum (fixed per-thread ranges + fixed trees); result in
// every thread.  red: >= 33 doubles of shared memory.
__device__ double block_sum(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = wsum_b(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  if (warp == 0) {
    double t = lane < nw ? red[lane] : 0.0;
    t = wsum_b(t);
    if (lane == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// this thread's share of sum A(r, c)^2 over r in [r0, r1), c in [c0, c1):
// flat index loop, four independent accumulators (deterministic per thread)
__device__ double sumsq_region(const double* A, int lda, int r0, int r1, int c0, int c1) {
  const int mr = r1 - r0;
  if (mr <= 0 || c1 <= c0) return 0.0;
  const int64_t tot = (int64_t)mr * (c1 - c0);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int64_t st = blockDim.x;
  int64_t e = threadIdx.x;
  for (; e + 3 * st < tot; e += 4 * st) {
    const int64_t e1 = e + st, e2 = e + 2 * st, e3 = e + 3 * st;
    const double x0 = A[(size_t)(c0 + e / mr) * lda + r0 + e % mr];
    const double x1 = A[(size_t)(c0 + e1 / mr) * lda + r0 + e1 % mr];
    const double x2 = A[(size_t)(c0 + e2 / mr) * lda + r0 + e2 % mr];
    const double x3 = A[(size_t)(c0 + e3 / mr) * lda + r0 + e3 % mr];
    a0 = fma(x0, x0, a0);
    a1 = fma(x1, x1, a1);
    a2 = fma(x2, x2, a2);
    a3 = fma(x3, x3, a3);
  }
  for (; e < tot; e += st) {
    const double x = A[(size_t)(c0 + e / mr) * lda + r0 + e % mr];
    a0 = fma(x, x, a0);
  }
  return (a0 + a1) + (a2 + a3);
}

__global__ void __launch_bounds__(512) bq_init_kernel(const QrcpProb* __restrict__ probs, BqState* st) {
  const QrcpProb P = probs[blockIdx.x];
  __shared__ double red[33];
  const double tot = block_sum(sumsq_region(P.A, P.lda, 0, P.m, 0, P.n), red);
  for (int c = threadIdx.x; c < P.n; c += blockDim.x) P.perm[c] = c;
  if (threadIdx.x == 0) {
    const double stop = P.stop_rel2 * tot;
    st[blockIdx.x].stop = stop;
    P.resid_out[-1] = tot;
    const bool go = tot > stop;
    st[blockIdx.x].active = go ? 1 : 0;
    if (!go) {
      *P.r_out = 0;
      P.resid_out[0] = tot;
    }
  }
}

// QRCP of the sketch Y (l x nr; written column-major, ld l, by the sketch
// GEMM): bb pivot positions (sequential-swap convention, as LAPACK ipiv),
// then the same swaps applied to the full columns of A and to perm.  One
// thread per column (l <= 40 rows: a column is a short sequential dot), Y
// staged row-major in shared memory when it fits (conflict-free per-thread
// column walks), else read in place from the workspace (L2).
template <bool kStage>
__global__ void __launch_bounds__(512) bq_pick_kernel(const QrcpProb* __restrict__ probs, BqState* st,
                                                      double* ws, size_t wsz, int j, int b, int l) {
  const QrcpProb P = probs[blockIdx.x];
  if (!st[blockIdx.x].active) return;
  extern __shared__ double sm[];
  const int nr = P.n - j, mr = P.m - j;
  const int bb = min(b, min(nr, mr));
  double* Yg = ws + (size_t)blockIdx.x * wsz;
  const int ldt = nr;                                  // row-major staging: Y(r, c) = Ys[r * ldt + c]
  double* Ys = sm;
  double* cn = kStage ? sm + (size_t)l * nr : sm;      // nr
  double* v = cn + nr;                                 // l
  auto Y = [&](int r, int c) -> double& { return kStage ? Ys[r * ldt + c] : Yg[(size_t)c * l + r]; };
  __shared__ int piv[32];
  __shared__ double s_tau;
  __shared__ double red[33];
  __shared__ int redi[32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  if (kStage)
    for (int e = tid; e < l * nr; e += blockDim.x) {
      const int c = e / l, r = e - c * l;
      Ys[r * ldt + c] = Yg[e];
    }
  __syncthreads();
  for (int c = tid; c < nr; c += blockDim.x) {
    double a0 = 0.0, a1 = 0.0;
    int r = 0;
    for (; r + 1 < l; r += 2) {
      const double x0 = Y(r, c), x1 = Y(r + 1, c);
      a0 = fma(x0, x0, a0);
      a1 = fma(x1, x1, a1);
    }
    if (r < l) { const double x = Y(r, c); a0 = fma(x, x, a0); }
    cn[c] = a0 + a1;
  }
  __syncthreads();
  for (int t = 0; t < bb; ++t) {
    // argmax of cn[t..nr) (ties -> smallest index)
    double best = -1.0;
    int bi = nr;
    for (int c = t + tid; c < nr; c += blockDim.x)
      if (cn[c] > best) { best = cn[c]; bi = c; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (lane == 0) { red[warp] = best; redi[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      best = lane < nw ? red[lane] : -1.0;
      bi = lane < nw ? redi[lane] : nr;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      const int pc = bi;
      if (lane == 0) piv[t] = pc;
      // swap columns t <-> pc of Y and cn, then the reflector of Y(t:l, t)
      if (pc != t) {
        for (int r = lane; r < l; r += 32) {
          const double x = Y(r, t);
          Y(r, t) = Y(r, pc);
          Y(r, pc) = x;
        }
        if (lane == 0) { const double x = cn[t]; cn[t] = cn[pc]; cn[pc] = x; }
      }
      __syncwarp();
      double ss = 0.0;
      for (int r = t + 1 + lane; r < l; r += 32) ss = fma(Y(r, t), Y(r, t), ss);
      ss = wsum_b(ss);
      const double alpha = Y(t, t);
      double tau = 0.0, scale = 0.0;
      if (ss != 0.0) {
        const double beta = -copysign(sqrt(alpha * alpha + ss), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int r = t + 1 + lane; r < l; r += 32) v[r] = Y(r, t) * scale;
      if (lane == 0) { v[t] = 1.0; s_tau = tau; }
    }
    __syncthreads();
    const double tau = s_tau;
    for (int c = t + 1 + tid; c < nr; c += blockDim.x) {
      double w0 = 0.0, w1 = 0.0;
      int r = t;
      for (; r + 1 < l; r += 2) {
        w0 = fma(v[r], Y(r, c), w0);
        w1 = fma(v[r + 1], Y(r + 1, c), w1);
      }
      if (r < l) w0 = fma(v[r], Y(r, c), w0);
      const double w = (w0 + w1) * tau;
      double a0 = 0.0, a1 = 0.0;
      for (r = t; r < l; ++r) {
        const double y = Y(r, c) - w * v[r];
        Y(r, c) = y;
        if (r > t) { if (r & 1) a1 = fma(y, y, a1); else a0 = fma(y, y, a0); }
      }
      cn[c] = a0 + a1;
    }
    __syncthreads();
  }
  // the same sequential swaps on the full columns of A (rows 0..m-1) and perm
  for (int t = 0; t < bb; ++t) {
    const int pc = piv[t];
    if (pc == t) continue;
    double* ca = P.A + (size_t)(j + t) * P.lda;
    double* cb = P.A + (size_t)(j + pc) * P.lda;
    for (int r = tid; r < P.m; r += blockDim.x) {
      const double x = ca[r];
      ca[r] = cb[r];
      cb[r] = x;
    }
    if (tid == 0) {
      const int x = P.perm[j + t];
      P.perm[j + t] = P.perm[j + pc];
      P.perm[j + pc] = x;
    }
    __syncthreads();
  }
}

// Register variant of the sketch QRCP for nr <= 512: thread c keeps column c
// of Y (L rows) in registers; per step one block argmax over the unselected
// columns, the pivot column goes through shared memory to warp 0 for the
// reflector, every other column updates itself.  The chosen original column
// ids are turned into sequential swap positions at the end.
template <int L>
__global__ void __launch_bounds__(512) bq_pick_reg_kernel(const QrcpProb* __restrict__ probs, BqState* st,
                                                          const double* ws, size_t wsz, int j, int b) {
  const QrcpProb P = probs[blockIdx.x];
  if (!st[blockIdx.x].active) return;
  const int nr = P.n - j, mr = P.m - j;
  const int bb = min(b, min(nr, mr));
  const int c = threadIdx.x, lane = c & 31, warp = c >> 5, nw = blockDim.x >> 5;
  const bool own = c < nr;
  const double* Yg = ws + (size_t)blockIdx.x * wsz;
  double x[L];
#pragma unroll
  for (int r = 0; r < L; ++r) x[r] = own ? Yg[(size_t)c * L + r] : 0.0;
  double cn = 0.0;
#pragma unroll
  for (int r = 0; r < L; ++r) cn = fma(x[r], x[r], cn);
  bool sel = !own;
  // each warp publishes its best candidate column speculatively, so a step
  // needs two barriers: (warp candidates) -> (warp 0: global argmax +
  // reflector) -> (update)
  __shared__ double slot[16 * L], v[L], wbest[16];
  __shared__ int widx[16], chosen[32], arr[512], pos[512], piv[32];
  __shared__ double s_tau;
  for (int t = 0; t < bb; ++t) {
    double best = sel ? -1.0 : cn;
    int bi = sel ? 1 << 30 : c;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (c == bi) {
#pragma unroll
      for (int r = 0; r < L; ++r) slot[warp * L + r] = x[r];
    }
    if (lane == 0) { wbest[warp] = best; widx[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      double gb = lane < nw ? wbest[lane] : -1.0;
      int gi = lane < nw ? widx[lane] : 1 << 30;
      int gw = lane;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, gb, o);
        const int oi = __shfl_xor_sync(0xffffffffu, gi, o);
        const int ow = __shfl_xor_sync(0xffffffffu, gw, o);
        if (ob > gb || (ob == gb && oi < gi)) { gb = ob; gi = oi; gw = ow; }
      }
      if (lane == 0) chosen[t] = gi;
      const double* colb = slot + gw * L;
      double ss = 0.0;
      for (int r = t + 1 + lane; r < L; r += 32) ss = fma(colb[r], colb[r], ss);
      ss = wsum_b(ss);
      const double alpha = colb[t];
      double tau = 0.0, scale = 0.0;
      if (ss != 0.0) {
        const double beta = -copysign(sqrt(alpha * alpha + ss), alpha);
        tau = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      for (int r = lane; r < L; r += 32) v[r] = r < t ? 0.0 : (r == t ? 1.0 : colb[r] * scale);
      if (lane == 0) s_tau = tau;
    }
    __syncthreads();
    if (c == chosen[t]) sel = true;
    if (!sel) {
      // volatile reads: the reflector is re-read from shared memory in both
      // passes instead of being held in registers (x[] already takes 2L)
      const volatile double* vv = v;
      double w0 = 0.0, w1 = 0.0;
#pragma unroll
      for (int r = 0; r < L; r += 2) {
        w0 = fma(vv[r], x[r], w0);
        if (r + 1 < L) w1 = fma(vv[r + 1], x[r + 1], w1);
      }
      const double w = (w0 + w1) * s_tau;
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int r = 0; r < L; ++r) {
        x[r] = fma(-w, vv[r], x[r]);
        if (r > t) { if (r & 1) a1 = fma(x[r], x[r], a1); else a0 = fma(x[r], x[r], a0); }
      }
      cn = a0 + a1;
    }
  }
  // chosen original column ids -> sequential swap positions
  for (int q = c; q < nr; q += blockDim.x) { arr[q] = q; pos[q] = q; }
  __syncthreads();
  if (c == 0)
    for (int t = 0; t < bb; ++t) {
      const int p = pos[chosen[t]];
      piv[t] = p;
      const int a = arr[t], bcol = arr[p];
      arr[t] = bcol; arr[p] = a;
      pos[bcol] = t; pos[a] = p;
    }
  __syncthreads();
  for (int t = 0; t < bb; ++t) {
    const int pc = piv[t];
    if (pc == t) continue;
    double* ca = P.A + (size_t)(j + t) * P.lda;
    double* cb = P.A + (size_t)(j + pc) * P.lda;
    for (int r = c; r < P.m; r += blockDim.x) {
      const double y = ca[r];
      ca[r] = cb[r];
      cb[r] = y;
    }
    if (c == 0) {
      const int y = P.perm[j + t];
      P.perm[j + t] = P.perm[j + pc];
      P.perm[j + pc] = y;
    }
    __syncthreads();
  }
}

// Unblocked Householder QR of the panel A[j:m, j:j+bb] in shared memory;
// writes R + reflectors back to A, the explicit V (unit lower trapezoidal,
// mr x bb, ld m) and T (bb x bb, ld b, upper) of I - V T V^T.
// P: the problem's A / lda / m / n; V: block V storage at row j (ld P.m);
// T: the block's b x b T factor.
__device__ void panel_qr(const QrcpProb& P, double* V, double* T, int j, int b, int ldt = 0) {
  extern __shared__ double sm[];
  const int nr = P.n - j, mr = P.m - j;
  const int bb = min(b, min(nr, mr));
  double* Pn = sm;                       // mr x bb, ld mr
  __shared__ double tau_s[32], G[32 * 32], Ts[32 * 32], red[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int c = 0; c < bb; ++c)
    for (int r = tid; r < mr; r += blockDim.x) Pn[c * mr + r] = P.A[(size_t)(j + c) * P.lda + j + r];
  __syncthreads();
  // One barrier per column.  Every warp forms the reflector scalars of column
  // t itself (from the norm of column t below row t, which the warp that
  // updated column t in step t-1 left in s_ss2, and the diagonal entry), so
  // no thread waits for a single scalar thread; column t itself is scaled
  // into v_t after the barrier that ends step t, when no warp reads it any
  // more.  For panels of at most 32 kRegRows rows a lane keeps its rows of
  // v_t and of the column it updates in registers: one shared-memory read
  // and one write per element and column instead of four reads and a write
  // (same reflectors up to roundoff; C3 TLR 2.73 -> 2.69 s).
  __shared__ double s_ss2[2];
  {
    double a = 0.0;
    for (int r = 1 + tid; r < mr; r += blockDim.x) a = fma(Pn[r], Pn[r], a);
    const double ss0 = block_sum(a, red);
    if (tid == 0) s_ss2[0] = ss0;
  }
  __syncthreads();
  constexpr int kRegRows = 24;
  const bool in_regs = mr <= 32 * kRegRows;
  for (int t = 0; t < bb; ++t) {
    const double ss = s_ss2[t & 1];
    const double alpha = Pn[t * mr + t];
    double tau = 0.0, scale = 0.0, beta = alpha;
    if (ss != 0.0) {
      beta = -copysign(sqrt(alpha * alpha + ss), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (tid == 0) tau_s[t] = tau;
    const double* vt = Pn + t * mr;
    // columns c > t: w = tau (x_t + scale sum_{r>t} a_r x_r), x -= w v_t
    if (in_regs) {
      double v[kRegRows];
#pragma unroll
      for (int i = 0; i < kRegRows; ++i) {
        const int r = t + 1 + lane + 32 * i;
        v[i] = r < mr ? vt[r] : 0.0;
      }
      for (int c = t + 1 + warp; c < bb; c += nw) {
        double* xc = Pn + c * mr;
        double x[kRegRows];
        double w = 0.0;
#pragma unroll
        for (int i = 0; i < kRegRows; ++i) {
          const int r = t + 1 + lane + 32 * i;
          x[i] = r < mr ? xc[r] : 0.0;
          if (r < mr) w = fma(v[i], x[i], w);
        }
        w = (wsum_b(w) * scale + xc[t]) * tau;
        const double ws_ = w * scale;
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < kRegRows; ++i) {
          const int r = t + 1 + lane + 32 * i;
          if (r < mr) {
            const double y = fma(-ws_, v[i], x[i]);
            xc[r] = y;
            if (c == t + 1 && r > t + 1) a = fma(y, y, a);
          }
        }
        if (c == t + 1) {
          a = wsum_b(a);
          if (lane == 0) s_ss2[(t + 1) & 1] = a;   // read by every warp after the next barrier
        }
        if (lane == 0) xc[t] -= w;
      }
    } else {
      for (int c = t + 1 + warp; c < bb; c += nw) {
        double w = 0.0;
        for (int r = t + 1 + lane; r < mr; r += 32) w = fma(vt[r], Pn[c * mr + r], w);
        w = (wsum_b(w) * scale + Pn[c * mr + t]) * tau;
        const double ws_ = w * scale;
        double a = 0.0;
        for (int r = t + 1 + lane; r < mr; r += 32) {
          const double y = fma(-ws_, vt[r], Pn[c * mr + r]);
          Pn[c * mr + r] = y;
          if (c == t + 1 && r > t + 1) a = fma(y, y, a);
        }
        if (c == t + 1) {
          a = wsum_b(a);
          if (lane == 0) s_ss2[(t + 1) & 1] = a;
        }
        if (lane == 0) Pn[c * mr + t] -= w;
      }
    }
    __syncthreads();
    // column t -> reflector storage (nobody reads it during step t + 1)
    if (warp == nw - 1) {
      for (int r = t + 1 + lane; r < mr; r += 32) Pn[t * mr + r] *= scale;
      if (lane == 0) Pn[t * mr + t] = beta;
    }
  }
  __syncthreads();
  // write back R / reflectors, explicit V
  for (int c = 0; c < bb; ++c)
    for (int r = tid; r < mr; r += blockDim.x) {
      const double x = Pn[c * mr + r];
      P.A[(size_t)(j + c) * P.lda + j + r] = x;
      V[(size_t)c * P.m + r] = r < c ? 0.0 : (r == c ? 1.0 : x);
    }
  // G(i, t) = v_i . v_t (i < t): rows >= t (v_t is zero above t, one at t)
  for (int pr = warp; pr < bb * bb; pr += nw) {
    const int i = pr % bb, t = pr / bb;
    if (i >= t) continue;
    double w = 0.0;
    for (int r = t + 1 + lane; r < mr; r += 32) w = fma(Pn[i * mr + r], Pn[t * mr + r], w);
    w = wsum_b(w);
    if (lane == 0) G[t * 32 + i] = w + Pn[i * mr + t];
  }
  __syncthreads();
  // T recurrence: T(t,t) = tau_t, T(0:t, t) = -tau_t T(0:t,0:t) G(0:t, t)
  // (shared memory, one warp), then T (b x b, ld b) to the workspace
  if (warp == 0) {
    for (int t = 0; t < bb; ++t) {
      for (int i = lane; i < t; i += 32) {
        double a = 0.0;
        for (int q = i; q < t; ++q) a = fma(Ts[q * 32 + i], G[t * 32 + q], a);
        Ts[t * 32 + i] = -tau_s[t] * a;
      }
      if (lane == 0) Ts[t * 32 + t] = tau_s[t];
      __syncwarp();
    }
  }
  __syncthreads();
  if (!ldt) ldt = b;
  for (int e = tid; e < b * b; e += blockDim.x) {
    const int i = e % b, t = e / b;
    T[(size_t)t * ldt + i] = (t < bb && i <= t) ? Ts[t * 32 + i] : 0.0;
  }
}

__global__ void __launch_bounds__(512) bq_panel_kernel(const QrcpProb* __restrict__ probs, BqState* st,
                                                       double* ws, size_t wsz, size_t off_v, size_t off_t,
                                                       int j, int b) {
  if (!st[blockIdx.x].active) return;
  panel_qr(probs[blockIdx.x], ws + (size_t)blockIdx.x * wsz + off_v, ws + (size_t)blockIdx.x * wsz + off_t, j, b);
}

// unpivoted blocked QR: the panel at column j (inside the super-block that
// starts at J0, width SB) of every problem with j < s.  Its T goes to the
// diagonal block of the super-block's merged T (ld SB); the rows J0..j-1 of
// its V columns are zeroed so V of the whole super-block is explicit.
__global__ void __launch_bounds__(512) bqr_panel_kernel(const BqrProb* __restrict__ probs, int j, int b, int J0,
                                                        int SB) {
  const BqrProb B = probs[blockIdx.x];
  if (j >= B.s) return;
  const QrcpProb P{B.A, B.lda, B.m, B.s, nullptr, nullptr, nullptr, 0.0, 0};
  double* TJ = B.T + (size_t)(J0 / SB) * SB * SB;
  panel_qr(P, B.V + (size_t)j * B.m + j, TJ + (size_t)(j - J0) * SB + (j - J0), j, b, SB);
  const int bb = min(b, B.s - j);
  for (int e = threadIdx.x; e < bb * (j - J0); e += blockDim.x) {
    const int c = e / (j - J0), r = J0 + e % (j - J0);
    B.V[(size_t)(j + c) * B.m + r] = 0.0;
  }
  // T_J is upper triangular: zero this panel's columns below its diagonal block
  const int below = SB - (j - J0) - b;
  for (int e = threadIdx.x; e < b * max(below, 0); e += blockDim.x) {
    const int c = e / below, r = (j - J0) + b + e % below;
    TJ[(size_t)((j - J0) + c) * SB + r] = 0.0;
  }
}

// Exact residual after the block and stop test: e = ||A[j+bb:, j+bb:]||^2,
// rn[t] = ||R(j+t, j+t:)||^2; res(q) = e + sum_{t >= q-j} rn[t].
__global__ void __launch_bounds__(512) bq_norms_kernel(const QrcpProb* __restrict__ probs, BqState* st, int j,
                                                       int b) {
  const QrcpProb P = probs[blockIdx.x];
  if (!st[blockIdx.x].active) return;
  const int nr = P.n - j, mr = P.m - j;
  const int bb = min(b, min(nr, mr));
  __shared__ double rn[64], red[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  for (int t = warp; t < bb; t += nw) {
    double a = 0.0;
    for (int c = j + t + lane; c < P.n; c += 32) {
      const double x = P.A[(size_t)c * P.lda + j + t];
      a = fma(x, x, a);
    }
    a = wsum_b(a);
    if (lane == 0) rn[t] = a;
  }
  const int r0 = j + bb;
  const double e = block_sum(sumsq_region(P.A, P.lda, r0, P.m, r0, P.n), red);   // syncs: rn visible after
  if (tid == 0) {
    const double stop = st[blockIdx.x].stop;
    const int kmax = min(P.m, P.n);
    // (rank cap: once the steps taken exceed P.cap and the residual is still
    // above the stop, the rank is known to exceed the cap -- all the caller
    // asks; the reported rank j + bb > cap is a lower bound)
    if (e <= stop || j + bb >= kmax || (P.cap > 0 && j + bb > P.cap)) {
      int s = j + bb;
      double res = e;
      for (int t = bb - 1; t >= 0; --t) {
        const double v = res + rn[t];
        if (v <= stop) { s = j + t; res = v; } else break;
      }
      *P.r_out = s;
      P.resid_out[0] = res;
      st[blockIdx.x].active = 0;
    }
  }
}

constexpr int kMaxL = 64;

}  // namespace

// Batched driver.  Problems must have m <= 2048, n <= 2048.
void launch_qrcp_blocked(const std::vector<QrcpProb>& probs, DescArena& ar, cudaStream_t s) {
  const int np = (int)probs.size();
  if (!np) return;
  int mmax = 1, nmax = 1, hmax = 1;
  for (const QrcpProb& p : probs) {
    mmax = std::max(mmax, p.m);
    nmax = std::max(nmax, p.n);
    hmax = std::max(hmax, p.cap > 0 ? std::min(p.hint, p.cap + 32) : p.hint);
  }
  // block width: the panel (mmax x b doubles) must fit in shared memory
  static const int b_env = getenv("TLRB_BQ_B") ? atoi(getenv("TLRB_BQ_B")) : 32;
  int b = b_env;
  while (b > 8 && (size_t)mmax * b * 8 > 200 * 1024) b -= 8;
  // beyond the register pick (n <= 512) prefer a block whose l x n sketch
  // fits in shared memory: the pick then never re-reads Y from L2
  // (nb = 760: b = 24, C3 10.0 -> 9.6 s)
  if (!getenv("TLRB_BQ_B") && nmax > 512)
    for (int bt = b; bt >= 8; bt -= 8)
      if (((size_t)(bt + 8) * nmax + nmax + bt + 8) * 8 <= 200 * 1024) { b = bt; break; }
  const int l = b + 8;
  // per-problem workspace: Y (l x nmax) | V (mmax x b) | T (b x b) | W (b x nmax) | W2 (b x nmax)
  const size_t off_v = (size_t)l * nmax, off_t = off_v + (size_t)mmax * b, off_w = off_t + (size_t)b * b,
               off_w2 = off_w + (size_t)b * nmax;
  const size_t wsz = (off_w2 + (size_t)b * nmax + 31) & ~(size_t)31;
  LaunchCtx& cx = launch_ctx();
  double*& ws = cx.bq_ws;
  size_t& ws_cap = cx.bq_ws_cap;
  BqState* st = static_cast<BqState*>(cx.bq_st);
  int& st_cap = cx.bq_st_cap;
  double*& omega = cx.bq_omega;
  constexpr int kOmegaCols = 2048;
  if ((size_t)np * wsz > ws_cap) {
    if (ws) TLRB_CUDA(cudaFree(ws));
    ws_cap = (size_t)np * wsz;
    TLRB_CUDA(cudaMalloc(&ws, ws_cap * sizeof(double)));
  }
  if (np > st_cap) {
    if (st) TLRB_CUDA(cudaFree(st));
    st_cap = np;
    TLRB_CUDA(cudaMalloc(&st, st_cap * sizeof(BqState)));
    cx.bq_st = st;
  }
  if (!omega) {   // fixed Gaussian test matrix (kMaxL x 2048, ld kMaxL), splitmix64 + Box-Muller
    std::vector<double> h((size_t)kMaxL * kOmegaCols);
    uint64_t x = 0x9E3779B97F4A7C15ull;
    auto next = [&]() {
      uint64_t z = (x += 0x9E3779B97F4A7C15ull);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      return ((z >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    };
    for (size_t i = 0; i < h.size(); i += 2) {
      const double u1 = next(), u2 = next();
      const double rr = sqrt(-2.0 * log(u1));
      h[i] = rr * cos(6.283185307179586 * u2);
      if (i + 1 < h.size()) h[i + 1] = rr * sin(6.283185307179586 * u2);
    }
    TLRB_CUDA(cudaMalloc(&omega, h.size() * sizeof(double)));
    TLRB_CUDA(cudaMemcpy(omega, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  const QrcpProb* dp = ar.put(probs, s);
  {
    ProfScope ps(K_QR, s, 0, 0);
    bq_init_kernel<<<np, 512, 0, s>>>(dp, st);
    post_launch();
  }
  const bool stage_y = ((size_t)l * nmax + nmax + l) * 8 <= 200 * 1024;
  const size_t smem_pick = ((stage_y ? (size_t)l * nmax : 0) + nmax + l) * 8;
  const size_t smem_panel = (size_t)mmax * b * 8;
  auto pick = stage_y ? bq_pick_kernel<true> : bq_pick_kernel<false>;
  allow_smem(pick, smem_pick);
  allow_smem(bq_panel_kernel, smem_panel);
  const int kmax_all = std::min(mmax, nmax);
  int planned = (std::min(hmax, kmax_all) + b - 1) / b + 2;
  int it = 0;
  std::vector<GemmProb> g0, g1, g2, g3, allp;
  std::vector<int> alls;
  std::vector<GemmStaged> rec;
  while (true) {
    // stage the GEMM descriptors of the next `planned` blocks in one upload
    const int it0 = it;
    int nit = std::max(0, std::min(planned, (kmax_all + b - 1) / b - it0));
    allp.clear(); alls.clear(); rec.clear();
    // the staged descriptors of one upload stay within a fixed budget (large
    // tiles: nb = 1900 stages ~0.6 MB per block for a 24 x 24 tile grid)
    const size_t kStageBudget = std::min<size_t>(12u << 20, ar.capacity() / 4);
    for (int q = 0; q < nit; ++q) {
      if (q > 0 && allp.size() * sizeof(GemmProb) + alls.size() * sizeof(int) > kStageBudget) {
        nit = q;
        break;
      }
      const int j = (it0 + q) * b;
      g0.clear(); g1.clear(); g2.clear(); g3.clear();
      for (int p = 0; p < np; ++p) {
        const QrcpProb& P = probs[p];
        const int mr = P.m - j, nr = P.n - j;
        if (mr <= 0 || nr <= 0) continue;
        const int bb = std::min(b, std::min(mr, nr)), n2 = nr - bb;
        double* W = ws + (size_t)p * wsz;
        const int* act = &st[p].active;
        double* Aj = P.A + (size_t)j * P.lda + j;
        GemmProb y{omega, Aj, nullptr, W, l, nr, mr, kMaxL, P.lda, 0, l, 0, 0, 0, 1.0, 0.0};
        y.active = act;
        g0.push_back(y);
        if (n2 <= 0) continue;
        double* V = W + off_v;
        double* T = W + off_t;
        double* Wm = W + off_w;
        double* W2 = W + off_w2;
        double* A2 = P.A + (size_t)(j + bb) * P.lda + j;
        GemmProb ga{V, A2, nullptr, Wm, bb, n2, mr, P.m, P.lda, 0, b, 1, 0, 0, 1.0, 0.0};
        GemmProb gc{T, Wm, nullptr, W2, bb, n2, bb, b, b, 0, b, 1, 0, 0, 1.0, 0.0};
        GemmProb gd{V, W2, A2, A2, mr, n2, bb, P.m, b, P.lda, P.lda, 0, 0, 0, -1.0, 1.0};
        ga.active = gc.active = gd.active = act;
        g1.push_back(ga);
        g2.push_back(gc);
        g3.push_back(gd);
      }
      rec.push_back(stage_gemm(g0, allp, alls));
      rec.push_back(stage_gemm(g1, allp, alls));
      rec.push_back(stage_gemm(g2, allp, alls));
      rec.push_back(stage_gemm(g3, allp, alls));
    }
    // the descriptor arena wraps when full: the problem descriptors are
    // staged again with every chunk so that they never predate a wrap
    if (it0 > 0) dp = ar.put(probs, s);
    const GemmProb* gp = allp.empty() ? nullptr : ar.put(allp, s);
    const int* gs = alls.empty() ? nullptr : ar.put(alls, s);
    for (int q = 0; q < nit; ++q, ++it) {
      const int j = it * b;
      launch_gemm_staged(rec[4 * q + 0], gp, gs, s);   // sketch Y = Omega A[j:, j:]
      {
        ProfScope ps(K_QR, s, 0, 0);
        if (nmax <= 512 && l == 40) bq_pick_reg_kernel<40><<<np, 512, 0, s>>>(dp, st, ws, wsz, j, b);
        else if (nmax <= 512 && l == 32) bq_pick_reg_kernel<32><<<np, 512, 0, s>>>(dp, st, ws, wsz, j, b);
        else pick<<<np, 512, smem_pick, s>>>(dp, st, ws, wsz, j, b, l);
        post_launch();
      }
      {
        ProfScope ps(K_QR, s, 0, 0);
        bq_panel_kernel<<<np, 512, smem_panel, s>>>(dp, st, ws, wsz, off_v, off_t, j, b);
        post_launch();
      }
      launch_gemm_staged(rec[4 * q + 1], gp, gs, s);   // W = V^T A2
      launch_gemm_staged(rec[4 * q + 2], gp, gs, s);   // W2 = T^T W
      launch_gemm_staged(rec[4 * q + 3], gp, gs, s);   // A2 -= V W2
      {
        ProfScope ps(K_QR, s, 0, 0);
        bq_norms_kernel<<<np, 512, 0, s>>>(dp, st, j, b);
        post_launch();
      }
    }
    if (it * b >= kmax_all) break;
    // any problem still running? (one readback per chunk of blocks)
    std::vector<BqState> hs(np);
    TLRB_CUDA(cudaMemcpyAsync(hs.data(), st, np * sizeof(BqState), cudaMemcpyDeviceToHost, s));
    TLRB_CUDA(cudaStreamSynchronize(s));
    bool any = false;
    for (const BqState& x : hs) any |= x.active != 0;
    if (!any) break;
    planned = std::max(3, planned - nit);   // the rest of the prediction, then three blocks at a time
  }
}

// ------------------------------------------------ unpivoted blocked QR
// A (m x s) = Q R.  Panels of b columns are factored by one CTA each
// (Householder in shared memory, compact WY); four panels (<= 128 columns) form a
// super-block whose reflectors are merged into one compact-WY factor
// I - V_J T_J V_J^T (T_J upper, SB x SB, SB = 4 b by default):
//   T_J(0:q, q) = -T_J(0:q, 0:q) (V(:, 0:q)^T V(:, q)) T_qq   (block columns q)
// so the trailing matrix beyond a super-block and the later application of
// Q take one rank-SB update per super-block (three DMMA GEMMs) instead of
// four rank-b ones: the m x n operand is streamed four times less.
// R + reflectors stay in A, the explicit V (zero above the diagonal within
// each super-block) in B.V (m x s, ld m), T_J at B.T + J SB SB, and B.W
// (>= 2 SB max(s, k) doubles) is GEMM scratch.  The factored
// recompression's stacked-factor QRs (tlrb.cu) use it; Q is applied, never formed.
static int super_panels() {
  static const int v = getenv("TLRB_BQR_SUPER") ? atoi(getenv("TLRB_BQR_SUPER")) : 4;
  return v;
}

int qr_blocked_width(int mmax) {
  static const int b0 = getenv("TLRB_BQR_B") ? atoi(getenv("TLRB_BQR_B")) : 32;
  int b = b0;
  while (b > 8 && (size_t)mmax * b * 8 > 200 * 1024) b -= 8;
  return b;
}

// super-block width: at most 128 columns (the slot layout of tlrb.cu's
// factored path budgets merged T factors of <= 128 x 128 per super-block)
int qr_blocked_super(int mmax) {
  const int b = qr_blocked_width(mmax);
  return std::max(1, std::min(super_panels(), 128 / b)) * b;
}

void launch_qr_blocked(const std::vector<BqrProb>& probs, DescArena& ar, cudaStream_t s) {
  if (probs.empty()) return;
  int mmax = 1, smax = 0;
  for (const BqrProb& p : probs) { mmax = std::max(mmax, p.m); smax = std::max(smax, p.s); }
  const int b = qr_blocked_width(mmax), SB = qr_blocked_super(mmax);
  const size_t smem_panel = (size_t)mmax * b * 8;
  allow_smem(bqr_panel_kernel, smem_panel);
  const BqrProb* dp = ar.put(probs, s);
  std::vector<GemmProb> ga, gc, gd;
  for (int J0 = 0; J0 < smax; J0 += SB) {
    // panels of the super-block; their updates stay inside it
    for (int j = J0; j < std::min(smax, J0 + SB); j += b) {
      {
        double fl = 0;
        for (const BqrProb& p : probs)
          if (j < p.s) fl += 2.0 * (p.m - j) * std::min(b, p.s - j) * std::min(b, p.s - j);
        ProfScope ps(K_QR, s, fl, 0);
        if (j > 0) dp = ar.put(probs, s);   // the GEMM launches in between may have wrapped the arena
        bqr_panel_kernel<<<(unsigned)probs.size(), 512, smem_panel, s>>>(dp, j, b, J0, SB);
        post_launch();
      }
      ga.clear(); gc.clear(); gd.clear();
      for (const BqrProb& p : probs) {
        if (j >= p.s) continue;
        const int mr = p.m - j, bb = std::min(b, p.s - j), n2 = std::min(p.s, J0 + SB) - j - bb;
        if (n2 <= 0) continue;
        double* V = p.V + (size_t)j * p.m + j;
        double* T = p.T + (size_t)(J0 / SB) * SB * SB + (size_t)(j - J0) * SB + (j - J0);
        double* A2 = p.A + (size_t)(j + bb) * p.lda + j;
        double* W = p.W;
        double* W2 = p.W + (size_t)b * n2;
        ga.push_back({V, A2, nullptr, W, bb, n2, mr, p.m, p.lda, 0, b, 1, 0, 0, 1.0, 0.0});
        gc.push_back({T, W, nullptr, W2, bb, n2, bb, SB, b, 0, b, 1, 0, 0, 1.0, 0.0});
        gd.push_back({V, W2, A2, A2, mr, n2, bb, p.m, b, p.lda, p.lda, 0, 0, 0, -1.0, 1.0});
      }
      launch_gemm(ga, ar, s);   // W = V^T A2
      launch_gemm(gc, ar, s);   // W2 = T^T W
      launch_gemm(gd, ar, s);   // A2 -= V W2
    }
    // merge the super-block's panel T factors: block column q of T_J
    for (int q = J0 + b; q < std::min(smax, J0 + SB); q += b) {
      std::vector<GemmProb> gx, gy, gt;
      for (const BqrProb& p : probs) {
        if (q >= p.s) continue;
        const int qb = q - J0, bq = std::min(b, p.s - q), mr = p.m - J0;
        double* TJ = p.T + (size_t)(J0 / SB) * SB * SB;
        double* VJ = p.V + (size_t)J0 * p.m + J0;      // rows J0.., explicit zeros above the panels
        double* X = p.W;                                 // qb x bq
        double* Y = p.W + (size_t)SB * b;                // qb x bq
        gx.push_back({VJ, VJ + (size_t)qb * p.m, nullptr, X, qb, bq, mr, p.m, p.m, 0, qb, 1, 0, 0, 1.0, 0.0});
        gy.push_back({X, TJ + (size_t)qb * SB + qb, nullptr, Y, qb, bq, bq, qb, SB, 0, qb, 0, 0, 0, 1.0, 0.0});
        gt.push_back({TJ, Y, nullptr, TJ + (size_t)qb * SB, qb, bq, qb, SB, qb, 0, SB, 0, 0, 0, -1.0, 0.0});
      }
      launch_gemm(gx, ar, s);   // X = V(:, 0:q)^T V(:, q)
      launch_gemm(gy, ar, s);   // Y = X T_qq
      launch_gemm(gt, ar, s);   // T(0:q, q) = -T(0:q, 0:q) Y
    }
    // trailing matrix beyond the super-block: one rank-SB update
    ga.clear(); gc.clear(); gd.clear();
    for (const BqrProb& p : probs) {
      if (J0 >= p.s) continue;
      const int sw = std::min(SB, p.s - J0), n2 = p.s - J0 - sw, mr = p.m - J0;
      if (n2 <= 0) continue;
      double* VJ = p.V + (size_t)J0 * p.m + J0;
      double* TJ = p.T + (size_t)(J0 / SB) * SB * SB;
      double* A2 = p.A + (size_t)(J0 + sw) * p.lda + J0;
      double* W = p.W;
      double* W2 = p.W + (size_t)SB * n2;
      ga.push_back({VJ, A2, nullptr, W, sw, n2, mr, p.m, p.lda, 0, SB, 1, 0, 0, 1.0, 0.0});
      gc.push_back({TJ, W, nullptr, W2, sw, n2, sw, SB, SB, 0, SB, 1, 0, 0, 1.0, 0.0});
      gd.push_back({VJ, W2, A2, A2, mr, n2, sw, p.m, SB, p.lda, p.lda, 0, 0, 0, -1.0, 1.0});
    }
    launch_gemm(ga, ar, s);
    launch_gemm(gc, ar, s);
    launch_gemm(gd, ar, s);
  }
}

// C (m x k[p], ld ldc[p]) <- Q C for the Q of launch_qr_blocked: one rank-SB
// update per super-block, in reverse order (C_J -= V_J T_J V_J^T C_J)
void launch_apply_q_blocked(const std::vector<BqrProb>& probs, const std::vector<double*>& C,
                            const std::vector<int>& ldc, const std::vector<int>& k, DescArena& ar,
                            cudaStream_t s) {
  if (probs.empty()) return;
  int mmax = 1, smax = 0;
  for (const BqrProb& p : probs) { mmax = std::max(mmax, p.m); smax = std::max(smax, p.s); }
  const int SB = qr_blocked_super(mmax);
  std::vector<GemmProb> g1, g2, g3;
  for (int J0 = ((smax - 1) / SB) * SB; J0 >= 0; J0 -= SB) {
    g1.clear(); g2.clear(); g3.clear();
    for (size_t q = 0; q < probs.size(); ++q) {
      const BqrProb& p = probs[q];
      if (J0 >= p.s || k[q] <= 0) continue;
      const int mr = p.m - J0, sw = std::min(SB, p.s - J0), kk = k[q];
      double* VJ = p.V + (size_t)J0 * p.m + J0;
      double* TJ = p.T + (size_t)(J0 / SB) * SB * SB;
      double* Cj = C[q] + J0;
      double* W = p.W;
      double* W2 = p.W + (size_t)SB * kk;
      g1.push_back({VJ, Cj, nullptr, W, sw, kk, mr, p.m, ldc[q], 0, SB, 1, 0, 0, 1.0, 0.0});
      g2.push_back({TJ, W, nullptr, W2, sw, kk, sw, SB, SB, 0, SB, 0, 0, 0, 1.0, 0.0});
      g3.push_back({VJ, W2, Cj, Cj, mr, kk, sw, p.m, SB, ldc[q], ldc[q], 0, 0, 0, -1.0, 1.0});
    }
    launch_gemm(g1, ar, s);
    launch_gemm(g2, ar, s);
    launch_gemm(g3, ar, s);
  }
}

}  // namespace tlrb

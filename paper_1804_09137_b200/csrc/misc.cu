// misc.cu — small batched helpers: Frobenius sums of squares (deterministic
// block reductions), strided copies / transposes, seeded Gaussian sketches,
// log-determinant and dot-product reductions, compression bookkeeping.
#include "common.cuh"
#include <execinfo.h>
#include <cstdlib>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <mutex>

namespace tlrb {

std::atomic<int64_t> g_launches{0};

bool sync_check_on() {
  static const bool on = getenv("TLRB_SYNC_CHECK") != nullptr;
  return on;
}
void sync_check_fail() {
  void* frames[32];
  const int n = backtrace(frames, 32);
  fprintf(stderr, "[tlrb] TLRB_SYNC_CHECK: launch %lld failed; host stack:\n", (long long)g_launches.load());
  backtrace_symbols_fd(frames, n, 2);
}
Profiler g_prof;
const char* kclass_name[K_NCLASS] = {"gen_tiles", "dgemm_vbatch", "trsm_vbatch", "potrf_block",
                                     "qr_householder", "jacobi_svd", "sumsq", "copy", "unused",
                                     "reduce", "cross_gemv"};

cudaEvent_t Profiler::get() {   // caller holds mu
  if (pool.empty()) {
    cudaEvent_t e;
    TLRB_CUDA(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = pool.back();
  pool.pop_back();
  return e;
}
cudaEvent_t Profiler::begin(cudaStream_t s) {
  std::lock_guard<std::mutex> lk(mu);
  cudaEvent_t a = get();
  TLRB_CUDA(cudaEventRecord(a, s));
  return a;
}
void Profiler::end(int cls, cudaEvent_t a, cudaStream_t s, double fl, double by) {
  std::lock_guard<std::mutex> lk(mu);
  cudaEvent_t b = get();
  TLRB_CUDA(cudaEventRecord(b, s));
  pend.push_back({cls, a, b, s, fl});
  flops[cls] += fl;
  bytes[cls] += by;
  count[cls] += 1;
}
void Profiler::drain() {
  std::lock_guard<std::mutex> lk(mu);
  static const char* tl_path = getenv("TLRB_TIMELINE");
  FILE* tl = (tl_path && epoch) ? fopen(tl_path, "a") : nullptr;
  std::vector<Pend> keep;   // launches still running on another stream (lane2)
  for (const Pend& p : pend) {
    if (cudaEventQuery(p.b) == cudaErrorNotReady) {
      cudaGetLastError();
      keep.push_back(p);
      continue;
    }
    float a = 0;
    if (cudaEventElapsedTime(&a, p.a, p.b) == cudaSuccess) ms[p.cls] += a;
    float t0 = 0;
    if (epoch && cudaEventElapsedTime(&t0, epoch, p.a) == cudaSuccess) {
      iv[p.cls].push_back({t0, t0 + a});
      if (tl) fprintf(tl, "%s %.4f %.4f %p %.6g\n", kclass_name[p.cls], t0, t0 + a, (void*)p.s, p.fl);
    }
    pool.push_back(p.a);
    pool.push_back(p.b);
  }
  pend.swap(keep);
  if (tl) fclose(tl);
}
void Profiler::reset() {
  drain();
  // new time origin for the per-launch intervals (GPU timestamps are global
  // across streams)
  if (!epoch) TLRB_CUDA(cudaEventCreate(&epoch));
  TLRB_CUDA(cudaEventRecord(epoch, 0));
  TLRB_CUDA(cudaEventSynchronize(epoch));
  for (int i = 0; i < K_NCLASS; ++i) ms[i] = flops[i] = bytes[i] = 0, count[i] = 0, iv[i].clear();
}
double Profiler::busy_ms(int cls) {
  drain();
  std::lock_guard<std::mutex> lk(mu);
  std::vector<std::pair<float, float>> all;
  for (int c = 0; c < K_NCLASS; ++c)
    if (cls < 0 || c == cls) all.insert(all.end(), iv[c].begin(), iv[c].end());
  std::sort(all.begin(), all.end());
  double tot = 0, a = -1e30, b = -1e30;
  for (const auto& x : all) {
    if (x.first > b) { if (b > a) tot += b - a; a = x.first; b = x.second; }
    else b = std::max(b, (double)x.second);
  }
  if (b > a) tot += b - a;
  return tot;
}

// ------------------------------------------------------- launch contexts
namespace {
LaunchCtx g_ctx[kMaxCtx];
bool g_ctx_used[kMaxCtx] = {};
std::mutex g_ctx_mu;
thread_local int t_ctx = 0;   // slot 0: threads outside any handle call
}  // namespace

void LaunchCtx::release() {
  if (device >= 0) cudaSetDevice(device);
  if (bq_ws) cudaFree(bq_ws);
  if (bq_st) cudaFree(bq_st);
  if (bq_omega) cudaFree(bq_omega);
  for (int i = 0; i < 4; ++i) {
    if (jac_side[i]) cudaStreamDestroy(jac_side[i]);
    if (jac_join[i]) cudaEventDestroy(jac_join[i]);
  }
  if (jac_fork) cudaEventDestroy(jac_fork);
  if (q_side) cudaStreamDestroy(q_side);
  if (q_side2) cudaStreamDestroy(q_side2);
  for (cudaEvent_t e : {q_fork, q_join, q_f2, q_j2})
    if (e) cudaEventDestroy(e);
  *this = LaunchCtx{};
}

int acquire_ctx() {
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  for (int i = 1; i < kMaxCtx; ++i)
    if (!g_ctx_used[i]) {
      g_ctx_used[i] = true;
      g_ctx[i] = LaunchCtx{};
      g_ctx[i].device = current_device();
      return i;
    }
  throw CudaError(cudaErrorLaunchOutOfResources, "too many live handles (launch contexts)", __FILE__, __LINE__);
}

void release_ctx(int slot) {
  if (slot <= 0 || slot >= kMaxCtx) return;
  std::lock_guard<std::mutex> lk(g_ctx_mu);
  g_ctx[slot].release();
  g_ctx_used[slot] = false;
}

void set_thread_ctx(int slot) { t_ctx = (slot > 0 && slot < kMaxCtx) ? slot : 0; }

LaunchCtx& launch_ctx() {
  LaunchCtx& c = g_ctx[t_ctx];
  if (c.device < 0) c.device = current_device();
  return c;
}

void DescArena::init(size_t bytes) {
  TLRB_CUDA(cudaHostAlloc(&h_, bytes, cudaHostAllocDefault));
  TLRB_CUDA(cudaMalloc(&d_, bytes));
  cap_ = bytes;
  off_ = 0;
}
void DescArena::release() {
  if (h_) cudaFreeHost(h_);
  if (d_) cudaFree(d_);
  h_ = d_ = nullptr;
  cap_ = off_ = 0;
}
void* DescArena::put_bytes(const void* src, size_t bytes, cudaStream_t s) {
  const size_t a = (off_ + 255) & ~(size_t)255;
  if (bytes > cap_)
    throw CudaError(cudaErrorMemoryAllocation, "descriptor batch larger than the staging arena", __FILE__, __LINE__);
  if (a + bytes > cap_) {
    // arena full: wait until earlier descriptors are consumed (every stream
    // of the device may hold some: look-ahead / side streams)
    TLRB_CUDA(cudaDeviceSynchronize());
    off_ = 0;
    return put_bytes(src, bytes, s);
  }
  memcpy(h_ + a, src, bytes);
  TLRB_CUDA(cudaMemcpyAsync(d_ + a, h_ + a, bytes, cudaMemcpyHostToDevice, s));
  off_ = a + bytes;
  return d_ + a;
}

// ------------------------------------------------------------ sum of squares
__global__ void __launch_bounds__(256) sumsq_kernel(const SumsqProb* __restrict__ probs) {
  const SumsqProb P = probs[blockIdx.x];
  if (P.A == nullptr) {   // constant entry: *out = m (used as ||V||^2 = rank of an orthonormal V)
    if (threadIdx.x == 0) *P.out = (double)P.m;
    return;
  }
  double a = 0.0;
  const int64_t tot = (int64_t)P.m * P.n;
  for (int64_t e = threadIdx.x; e < tot; e += blockDim.x) {
    const int r = (int)(e % P.m), c = (int)(e / P.m);
    const double x = P.A[(size_t)c * P.ld + r];
    a = fma(x, x, a);
  }
  __shared__ double red[256];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *P.out = red[0];
}

void launch_sumsq(const std::vector<SumsqProb>& probs, DescArena& ar, cudaStream_t s) {
  if (probs.empty()) return;
  const SumsqProb* dp = ar.put(probs, s);
  double by = 0;
  for (const SumsqProb& p : probs) by += 8.0 * p.m * p.n;
  ProfScope ps(K_SUMSQ, s, 2.0 * by / 8, by);
  sumsq_kernel<<<(unsigned)probs.size(), 256, 0, s>>>(dp);
  post_launch();
}

// ---------------------------------------------------------------- copies
__global__ void __launch_bounds__(256) copy_kernel(const CopyProb* __restrict__ probs, int chunks) {
  const CopyProb P = probs[blockIdx.x / chunks];
  const int part = blockIdx.x % chunks;
  const int64_t tot = (int64_t)P.m * P.n;
  const int64_t per = (tot + chunks - 1) / chunks;
  const int64_t e0 = part * per, e1 = min(tot, e0 + per);
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const int r = (int)(e % P.m), c = (int)(e / P.m);
    double v = !P.src ? 0.0   // no source: zero fill
               : P.transpose ? P.src[(size_t)(P.srccol ? P.srccol[r] : r) * P.lds + c]
                             : P.src[(size_t)c * P.lds + r];
    if (P.tri == 1 && r < c) v = 0.0;
    const int rd = P.rowperm ? P.rowperm[r] : r;
    double* d = P.dst + (size_t)c * P.ldd + rd;
    *d = P.tri == 2 ? *d + P.scale * v : P.scale * v;
  }
}

void launch_copy(const std::vector<CopyProb>& probs, DescArena& ar, cudaStream_t s) {
  std::vector<CopyProb> keep;
  int64_t mx = 0;
  for (const CopyProb& p : probs)
    if (p.m > 0 && p.n > 0) {
      keep.push_back(p);
      mx = std::max<int64_t>(mx, (int64_t)p.m * p.n);
    }
  if (keep.empty()) return;
  const int chunks = (int)std::min<int64_t>(64, (mx + 8191) / 8192);
  const CopyProb* dp = ar.put(keep, s);
  double by = 0;
  for (const CopyProb& p : keep) by += 16.0 * p.m * p.n;
  ProfScope ps(K_COPY, s, 0, by);
  copy_kernel<<<(unsigned)(keep.size() * chunks), 256, 0, s>>>(dp, chunks);
  post_launch();
}

// ------------------------------------------- column normalisation (factored
// recompression: the kept factor U_ij = Q D has orthogonal columns; Q goes
// back in place and D onto the diagonal of the stacked R factor)
__global__ void __launch_bounds__(256) colnorm_kernel(const ColNormProb* __restrict__ probs) {
  const ColNormProb P = probs[blockIdx.x];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int c = warp; c < P.n; c += nw) {
    if (!P.A) {
      if (lane == 0) P.diag[(size_t)c * (P.ldd + 1)] = 1.0;
      continue;
    }
    double* col = P.A + (size_t)c * P.ld;
    double a = 0.0;
    for (int r = lane; r < P.m; r += 32) a = fma(col[r], col[r], a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    const double nrm = sqrt(a), inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int r = lane; r < P.m; r += 32) col[r] *= inv;
    if (lane == 0) P.diag[(size_t)c * (P.ldd + 1)] = nrm;
  }
}

void launch_colnorm(const std::vector<ColNormProb>& probs, DescArena& ar, cudaStream_t s) {
  std::vector<ColNormProb> keep;
  double by = 0;
  for (const ColNormProb& p : probs)
    if (p.n > 0) {
      keep.push_back(p);
      by += p.A ? 24.0 * p.m * p.n : 8.0 * p.n;
    }
  if (keep.empty()) return;
  const ColNormProb* dp = ar.put(keep, s);
  ProfScope ps(K_COPY, s, 0, by);
  colnorm_kernel<<<(unsigned)keep.size(), 256, 0, s>>>(dp);
  post_launch();
}

// ---------------------------------------------------- scalar reductions
__global__ void __launch_bounds__(1024) reduce_kernel(const double* x, int n, double* out,
                                                      int square) {
  double a = 0.0;
  // contiguous per-thread ranges: deterministic
  const int per = (n + blockDim.x - 1) / blockDim.x;
  const int i0 = threadIdx.x * per, i1 = min(n, i0 + per);
  for (int i = i0; i < i1; ++i) a += square ? x[i] * x[i] : x[i];
  __shared__ double red[1024];
  red[threadIdx.x] = a;
  __syncthreads();
  for (int o = 512; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

void launch_sum_log(const double* logdiag, int n, double* out, cudaStream_t s) {
  ProfScope ps(K_REDUCE, s, n, 8.0 * n);
  reduce_kernel<<<1, 1024, 0, s>>>(logdiag, n, out, 0);
  post_launch();
}
void launch_dot(const double* x, int n, double* out, cudaStream_t s) {
  ProfScope ps(K_REDUCE, s, 2.0 * n, 8.0 * n);
  reduce_kernel<<<1, 1024, 0, s>>>(x, n, out, 1);
  post_launch();
}

// ------------------------------------------------ compression bookkeeping
// sums[6p + {0..5}] = {||M||^2, e2, ||U1||^2, ||U2||^2, ||V1||^2, ||V2||^2}
// aux[3p] = e2 (0 when unsketched), aux[3p+1] = noise floor, aux[3p+2] = ||M||^2
//   50 eps_mach ||[U1 U2]||_F ||[V1 V2]||_F  (compression.py:78), 0 for tiles;
// ok[p] = e2 <= rel_tol2 ||M||^2.
__global__ void aux_kernel(const double* sums, const int* kinds, int nprob, double* aux, int* ok,
                           double rel_tol2) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nprob) return;
  const double* S = sums + 6 * p;
  const int kind = kinds[p];   // bit0: sketched, bit1: recompression
  const double e2 = (kind & 1) ? S[1] : 0.0;
  aux[3 * p] = e2;
  aux[3 * p + 1] = (kind & 2) ? 50.0 * DBL_EPSILON * sqrt(S[2] + S[3]) * sqrt(S[4] + S[5]) : 0.0;
  aux[3 * p + 2] = S[0];
  ok[p] = (!(kind & 1)) || (e2 <= rel_tol2 * S[0]);
}

void launch_aux(const double* sums, const int* kinds, int nprob, double* aux, int* ok,
                double rel_tol2, cudaStream_t s) {
  aux_kernel<<<(nprob + 127) / 128, 128, 0, s>>>(sums, kinds, nprob, aux, ok, rel_tol2);
  post_launch();
}

}  // namespace tlrb

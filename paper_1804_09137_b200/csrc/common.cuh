// common.cuh — shared declarations for the sm_100a TLR likelihood kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>

namespace tlrb {

extern std::atomic<int64_t> g_launches;  // kernels launched by this library (process-wide)

#define TLRB_CUDA(call)                                                        \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) throw ::tlrb::CudaError(e_, #call, __FILE__, __LINE__); \
  } while (0)

struct CudaError {
  cudaError_t code;
  char msg[256];
  CudaError(cudaError_t c, const char* what, const char* file, int line) : code(c) {
    snprintf(msg, sizeof msg, "%s failed at %s:%d: %s", what, file, line,
             cudaGetErrorString(c));
  }
};

// TLRB_SYNC_CHECK=1 (diagnostic): synchronise after every launch and, on an
// error, print the host call stack of the launch that produced it
bool sync_check_on();
void sync_check_fail();
inline void post_launch() {
  ++g_launches;
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess && sync_check_on()) {
    e = cudaDeviceSynchronize();
    if (e != cudaSuccess) sync_check_fail();
  }
  if (e != cudaSuccess) throw CudaError(e, "kernel launch", __FILE__, __LINE__);
}

// ---- per-kernel-class profiler (CUDA events on the launching stream) ----
enum KClass { K_GEN = 0, K_GEMM, K_TRSM, K_POTRF, K_QR, K_JACOBI, K_SUMSQ, K_COPY, K_UNUSED,
              K_REDUCE, K_CROSS, K_NCLASS };
extern const char* kclass_name[K_NCLASS];
struct Profiler {
  bool on = false;
  unsigned mask = ~0u;   // kernel classes timed while on (tlrb_profile_mask)
  double ms[K_NCLASS] = {}, flops[K_NCLASS] = {}, bytes[K_NCLASS] = {};
  int64_t count[K_NCLASS] = {};
  struct Pend { int cls; cudaEvent_t a, b; cudaStream_t s; double fl; };
  cudaEvent_t epoch = nullptr;   // time origin (reset): per-launch intervals, TLRB_TIMELINE dump
  std::vector<Pend> pend;
  // per-class launch intervals [start, end] in ms since `epoch`: the union is
  // the class's busy time (launches of one class on several streams overlap)
  std::vector<std::pair<float, float>> iv[K_NCLASS];
  double busy_ms(int cls);   // cls < 0: union over every class
  std::vector<cudaEvent_t> pool;
  std::mutex mu;             // launches may come from several host threads (group handles)
  cudaEvent_t get();
  cudaEvent_t begin(cudaStream_t s);
  void end(int cls, cudaEvent_t a, cudaStream_t s, double fl, double by);
  void add_work(int cls, double fl, double by) {
    std::lock_guard<std::mutex> lk(mu);
    if ((mask >> cls) & 1u) { flops[cls] += fl; bytes[cls] += by; }
  }
  void drain();   // after a stream synchronisation
  void reset();
};
extern Profiler g_prof;
struct ProfScope {   // RAII: times one launch of class cls
  int cls; cudaStream_t s; double fl, by; cudaEvent_t a = nullptr;
  ProfScope(int c, cudaStream_t st, double f = 0, double b = 0) : cls(c), s(st), fl(f), by(b) {
    if (g_prof.on && ((g_prof.mask >> cls) & 1u)) a = g_prof.begin(st);
  }
  ~ProfScope() { if (a) g_prof.end(cls, a, s, fl, by); }
};

// clock64 phase counters inside the QRCP / Jacobi kernels (TLRB_QRCP_PROF /
// TLRB_JACOBI_PROF readouts); compiled in only with -DTLRB_CLOCK_PROF
// (TLRB_CLOCK_PROF=1 python -m paper_1804_09137_b200.build --force), as the
// live counters cost registers in the hot loops.
#ifdef TLRB_CLOCK_PROF
constexpr bool kClockProf = true;
#else
constexpr bool kClockProf = false;
#endif

// ------------------------------------------------------------------ Matern
struct MaternParamsDev {
  double theta1, inv_theta2, nu, pref;   // pref = theta1 / (2^(nu-1) Gamma(nu))
  double gampl, gammi, gam1, gam2;       // Temme constants for mu = nu - round(nu)
  int nl;                                // int(nu + 0.5)
  double mu;
  int kind;                              // 0: nu=1/2, 1: nu=3/2, 2: nu=5/2, 3: general
};
MaternParamsDev make_matern(double theta1, double theta2, double nu);

// Point coordinates in the layout the distance kernel reads (the reference's
// KernelView, geometry.py:58-72,106-122): Euclidean a1 = x, a2 = y; great
// circle a1 = lat (rad), a2 = lon (rad), a3 = cos(lat), diam = 2 * radius.
struct Pts {
  const double* a1; const double* a2; const double* a3;
  double diam;            // 0 => Euclidean
};

struct GenTile {          // one Matern block: rows [r0, r0+m) x cols [c0, c0+n)
  double* out; int ld;
  int r0, m, c0, n;
  double diag_add;        // added where global row == global col (nugget)
};

// --------------------------------------------------------------------- GEMM
struct GemmProb {
  const double* A; const double* B; const double* Cin; double* C;
  int m, n, k, lda, ldb, ldcin, ldc;
  int ta, tb;             // op(A) = A^T if ta, op(B) = B^T if tb
  int lower_only;         // skip CTA tiles strictly above the diagonal
  double alpha, beta;     // C = alpha op(A) op(B) + beta Cin
  const int* active = nullptr;   // optional device flag: skip the problem when *active == 0
};

// --------------------------------------------------------------------- TRSM
struct TrsmProb {          // B <- L^-1 B (or L^-T B), L lower n x n
  const double* L; int ldl;
  double* B; int ldb;
  int n, nrhs;
};


// ------------------------------------------------------------------- Jacobi
struct JacobiProb {        // one-sided Jacobi on the columns of X (m x s)
  double* X; int ldx;
  double* Vout; int ldv;   // sorted, normalized columns (m x s)
  double* sigma;           // s sorted singular values (descending)
  const double* aux;       // [0] = e2 (sketch residual^2), [1] = noise floor
  double eps;              // accuracy threshold
  int* rank_out;           // truncation rank (compression.py:26-36 rule)
  int* sweeps_out;
  int m, s;
  long long* prof = nullptr;   // optional phase cycle counters (debug)
};

// ----------------------------------------------------------- small helpers
struct SumsqProb { const double* A; int ld, m, n; double* out; };
// dst(r, c) = scale * (transpose ? src(c, r) : src(r, c)); tri = 1: zero where r < c;
// tri = 2: dst(r, c) += scale * src (accumulate); src == nullptr: zero fill;
// rowperm: dst row rowperm[r] receives row r
// srccol (transpose mode): dst row r reads source column srccol[r]
struct CopyProb { const double* src; int lds; double* dst; int ldd; int m, n; int transpose; double scale;
                  int tri; const int* rowperm; const int* srccol = nullptr; };
struct QrcpProb { double* A; int lda, m, n; int* perm; int* r_out; double* resid_out; double stop_rel2;
                  int hint = 0;      // hint: predicted number of QRCP steps (selects the kernel)
                  int cap = 0; };    // > 0: the caller only needs to know whether the rank exceeds cap (the tile is then
                                     // stored exactly): the blocked QRCP stops at the first block past it

// Device-resident descriptor staging (pinned host ring -> device), reset at
// stream synchronisation points.
constexpr int kMaxDevices = 16;
inline int current_device() {
  int d = 0;
  TLRB_CUDA(cudaGetDevice(&d));
  if (d < 0 || d >= kMaxDevices) throw CudaError(cudaErrorInvalidDevice, "device index >= 16", __FILE__, __LINE__);
  return d;
}

// Launcher-side caches (side streams, events, blocked-QRCP scratch) belong to
// a launch context: one per handle, selected for the calling thread by the C
// ABI (tlrb.cu guarded()).  Handles — including several logical ranks on one
// device — therefore never share launcher state and may run concurrently.
struct LaunchCtx {
  int device = -1;
  // bqrcp.cu
  double* bq_ws = nullptr; size_t bq_ws_cap = 0;
  void* bq_st = nullptr; int bq_st_cap = 0;
  double* bq_omega = nullptr;
  // jacobi.cu
  cudaStream_t jac_side[4] = {}; cudaEvent_t jac_fork = nullptr, jac_join[4] = {};
  // qrcp.cu
  cudaStream_t q_side = nullptr, q_side2 = nullptr;
  cudaEvent_t q_fork = nullptr, q_join = nullptr, q_f2 = nullptr, q_j2 = nullptr;
  void release();   // frees everything above (on `device`)
};
constexpr int kMaxCtx = 256;
int acquire_ctx();             // a free context slot (throws when all are taken)
void release_ctx(int slot);    // frees its resources and the slot
void set_thread_ctx(int slot); // the calling thread's launches use this context
LaunchCtx& launch_ctx();        // the calling thread's context

// Dynamic shared memory of a kernel: the attribute is raised to the device's
// opt-in maximum (not to this launch's need), so launches of one kernel from
// several host threads (group handles) never lower it under one another.
template <class K>
void allow_smem(K kern, size_t need) {
  static const int optin = [] {
    int v = 0;
    TLRB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, current_device()));
    return v;
  }();
  cudaFuncAttributes fa{};
  TLRB_CUDA(cudaFuncGetAttributes(&fa, kern));
  const int room = optin - (int)fa.sharedSizeBytes;   // static shared memory counts against the opt-in limit
  if ((int64_t)need > room)
    throw CudaError(cudaErrorInvalidValue, "kernel shared memory above the device limit", __FILE__, __LINE__);
  if (fa.maxDynamicSharedSizeBytes < room)
    TLRB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, room));
}

class DescArena {
 public:
  void init(size_t bytes);
  void release();
  template <class T> T* put(const std::vector<T>& v, cudaStream_t s) {
    return static_cast<T*>(put_bytes(v.data(), v.size() * sizeof(T), s));
  }
  void* put_bytes(const void* src, size_t bytes, cudaStream_t s);
  void reset() { off_ = 0; }
  size_t used() const { return off_; }
  size_t capacity() const { return cap_; }
 private:
  char* h_ = nullptr; char* d_ = nullptr; size_t cap_ = 0, off_ = 0;
};

// launchers (all asynchronous on `s`)
void launch_gen_tiles(const std::vector<GenTile>& tiles, const Pts& pts, const MaternParamsDev& p,
                      DescArena& ar, cudaStream_t s);
void launch_bessel(double nu, const double* x, double* out, int64_t n, cudaStream_t s);
void launch_gemm(const std::vector<GemmProb>& probs, DescArena& ar, cudaStream_t s);
// multi-launch staging: build several batches on the host, upload once, launch
struct GemmStaged { int poff = 0, soff = 0, moff = -1, n = 0, tot = 0, cfg = 0; double fl = 0, by = 0; bool vec = false;
                    int ta = -1, tb = -1; };   // one (ta, tb) per launch
GemmStaged stage_gemm(const std::vector<GemmProb>& probs, std::vector<GemmProb>& allp, std::vector<int>& alls,
                      int cfg = -1);   // cfg < 0: chosen from the batch
void launch_gemm_staged(const GemmStaged& g, const GemmProb* dp, const int* ds, cudaStream_t s);
void launch_trsm(const std::vector<TrsmProb>& probs, bool trans, DescArena& ar, cudaStream_t s);
void launch_trsm_panel(const std::vector<TrsmProb>& probs, DescArena& ar, cudaStream_t s);   // one shared L, blocked on DMMA
void launch_potrf_block(double* A, int ld, int n, int r0, int bs, int tile, int* info,
                        double* logdiag, cudaStream_t s);
// unpivoted blocked Householder QR (bqrcp.cu): R + reflectors in A (m x s),
// explicit V (m x s, ld m), merged T per super-block (SB x SB each), W scratch
// (>= 2 SB max(s, k) doubles)
struct BqrProb { double* A; int lda, m, s; double* V; double* T; double* W; };
int qr_blocked_width(int mmax);
int qr_blocked_super(int mmax);   // merged super-block width (kSuper panels)
void launch_qr_blocked(const std::vector<BqrProb>& probs, DescArena& ar, cudaStream_t s);
void launch_apply_q_blocked(const std::vector<BqrProb>& probs, const std::vector<double*>& C,
                            const std::vector<int>& ldc, const std::vector<int>& k, DescArena& ar,
                            cudaStream_t s);
// gathered[p] = 1: columns left in place (R column jj at perm[jj]); 0: physically pivoted
void launch_qrcp(const std::vector<QrcpProb>& probs, std::vector<char>& gathered, DescArena& ar,
                 cudaStream_t s);
void launch_qrcp_blocked(const std::vector<QrcpProb>& probs, DescArena& ar, cudaStream_t s);
void launch_jacobi(const std::vector<JacobiProb>& probs, DescArena& ar, cudaStream_t s);
void launch_sumsq(const std::vector<SumsqProb>& probs, DescArena& ar, cudaStream_t s);
// columns of A (m x n, ld) scaled to unit norm in place; their norms go to the diagonal diag[c (ldd + 1)]
// (A == nullptr: the diagonal is set to one)
struct ColNormProb { double* A; int ld, m, n; double* diag; int ldd; };
void launch_colnorm(const std::vector<ColNormProb>& probs, DescArena& ar, cudaStream_t s);
void launch_copy(const std::vector<CopyProb>& probs, DescArena& ar, cudaStream_t s);
void launch_sum_log(const double* logdiag, int n, double* out, cudaStream_t s);
void launch_dot(const double* x, int n, double* out, cudaStream_t s);
void launch_cross_gemv(const Pts& known, const double* w, int64_t n, const Pts& unknown, int64_t m,
                       const MaternParamsDev& p, double* partial, double* out, cudaStream_t s);
void launch_aux(const double* sums, const int* kinds, int nprob, double* aux, int* ok,
                double rel_tol2, cudaStream_t s);

}  // namespace tlrb

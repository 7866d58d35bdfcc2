// tlrb.cu — host runtime and C ABI of libtlrb200.so.
//
// One evaluation of the Gaussian log-likelihood (stats.py:103-112) as a
// sequence of batched sm_100a kernel launches on the handle's stream:
//
//   K1  generate every lower-triangle tile (tilestore.py:181-223)
//   K2  TLR: compress every off-diagonal tile to acc (compression.py:39-51)
//   K3  per panel k: POTRF(L_kk) with NPD report (linalg.py:36-45)
//   K4  per panel k: TRSM of the panel (dense tiles linalg.py:94-97 /
//       V factors linalg.py:121-127)
//   K5  per panel k: diagonal updates (dense :100 / low-rank :128-132)
//   K6+K7 per panel k: off-diagonal updates; TLR: form the updated tile
//       U_ij V_ij^T - U_ik (V_ik^T V_jk) U_jk^T and recompress it to acc with
//       the reference's truncation rule and noise floor (:133-139,
//       compression.py:54-81) — all (i,j) of one k in one batch, never
//       merging several k (eager recompression)
//   K8  forward solve + dot + log-det (linalg.py:166-177, 200-206, 78-79)
//
// Data layout in HBM (column-major FP64 everywhere):
//   diag   : t tiles of nb x nb (ld nb)
//   U, V   : one slab of nb x cap per lower tile (i > j), tile id i(i-1)/2+j.
//            TLR: U_ij (size_i x k), V_ij (size_j x k).  Dense mode: the U
//            slab holds L_ij^T (size_j x size_i) so panel solves are
//            left-lower TRSMs on contiguous columns.
//   ws     : per-job compression workspace slots (M, E, Y, Q, Omega, B^T, V)
#include "common.cuh"
#include "comm.cuh"
#include "../../include/tlrb200.h"
#include <nccl.h>
#include <cmath>
#include <string>
#include <chrono>
#include <mutex>
#include <thread>
#include <limits>

using namespace tlrb;

namespace {

// truncated QRCP stops at ||residual||_F <= rel acc ||M||_F.  The residual
// enters the truncation tail exactly; the top-k sigma(R) differ from sigma(M)
// by at most rel^2 acc^2 ||M||^2 in the squared tail sums, i.e. rel^2 of the
// truncation threshold.  TLRB_QRCP_REL overrides.
double qrcp_rel_tol() {
  static const double v = getenv("TLRB_QRCP_REL") ? atof(getenv("TLRB_QRCP_REL")) : 1e-2;
  return v;
}
constexpr int kPotrfBlock = 32;
constexpr int kMaxTile = 2048;   // largest supported tile size (rows staged per column)

// Factored recompression (reference scheme: QR of the stacked factors, SVD of
// the K x K core) for stacked ranks K <= frac min(m, n).  Measured: nb = 500
// (C2, latency-bound steps) best at 0.1-0.15 (0.2: +2%, 0.4: +10%); nb = 760
// (C3, throughput-bound) 15.8 s at 0.15, 13.1 s at 0.4, 11.4 s at 0.6 (the
// slot layout caps K near nb / 2).  TLRB_FACTORED_FRAC overrides.
double factored_frac(int nb) {
  static const double v = getenv("TLRB_FACTORED_FRAC") ? atof(getenv("TLRB_FACTORED_FRAC")) : -1.0;
  return v >= 0.0 ? v : (nb <= 512 ? 0.15 : 1.0);
}

// roofline denominators of tlrb_stats.t_roof_ms (tlrb_set_peaks)
double g_peak_flops = 35.5e12, g_peak_bytes = 6449.7e9;

// Storage rule of a tile's factors when a storage cap (BASELINE max_rank,
// SURVEY A13) is configured: a tile is kept exact (dense, updated by GEMMs,
// never recompressed) once its QRCP rank at 1e-2 acc (an upper bound of its
// truncation rank) exceeds the cap, or exceeds rho min(m, n).  Keeping such
// a tile exact is more accurate than the reference's truncation (never below
// acc, compression.py:6) and removes the costliest work of the evaluation:
// the SVD of its initial compression and the QRCP + Jacobi of a high-rank
// nb x nb tile on every later update.  rho is the measured time break-even
// of this GPU, where an exact tile is updated by DMMA GEMMs at ~30 TFLOP/s
// and a low-rank one pays QR + SVD recompressions at ~1: C3 (nb = 760, cap
// 380, tools/c3_once.py) with the round's first GEMM, rule on the SVD rank,
// rho = 0.45: 7.05 s; on the QRCP rank, 0.45 / 0.35 / 0.3 / 0.25 / 0.2: 4.99 /
// 4.51 / 3.95 / 3.82 / 3.81 s (profiles/r02_sweep.jsonl); with the final
// kernels 0.3 / 0.25 / 0.2 / 0.15 / 0.12 / 0.1 / 0.08 / 0.05 / 0.03 (all exact):
// 2.78 / 2.54 / 2.37 / 1.95 / 1.79 / 1.73 / 1.75 / 2.26 / 3.01 s
// (profiles/r02_sweep_final.jsonl); at 0.1: 1,387 of 3,403 tiles exact, 7.4 GB
// of factor storage (dense: 31 GB), likelihood 1e-11 from the dense one.
// Without a cap every tile follows the reference's truncation
// exactly (its TLR-vs-dense gap, hundreds of acc on ill-conditioned inputs,
// is part of the parity contract).  TLRB_DENSE_FRAC overrides rho (>= 1:
// cap only).
double dense_frac() {
  static const double v = getenv("TLRB_DENSE_FRAC") ? atof(getenv("TLRB_DENSE_FRAC")) : 0.1;
  return v;
}

// TLRB_FACTORED_OVER=0: updates whose stacked rank exceeds the dense limit
// take the dense path (M formed, QRCP, exact storage decided on the QRCP
// rank) instead of the factored one followed by a densify
bool factored_over_limit() {
  static const bool v = !(getenv("TLRB_FACTORED_OVER") && atoi(getenv("TLRB_FACTORED_OVER")) == 0);
  return v;
}

// TLRB_FACTORED_ORTHO=0: the stacked-factor QRs refactor all K columns
// (default: only the update's columns, see factor_tlr)
bool factored_ortho() {
  static const bool v = !(getenv("TLRB_FACTORED_ORTHO") && atoi(getenv("TLRB_FACTORED_ORTHO")) == 0);
  return v;
}

// TLRB_DENSE_BY_QRCP=0: decide exact storage on the SVD truncation rank only
// (the SVD of every capped tile runs); default: on the QRCP rank
bool dense_by_qrcp() {
  static const bool v = !(getenv("TLRB_DENSE_BY_QRCP") && atoi(getenv("TLRB_DENSE_BY_QRCP")) == 0);
  return v;
}

struct Flops {
  double f = 0, b = 0, troof = 0;   // troof: sum over ops of max(F / P64, B / BW), seconds
  void add(double ff, double bb) {
    f += ff;
    b += bb;
    troof += std::max(ff / g_peak_flops, bb / g_peak_bytes);
  }
};

}  // namespace

struct tlrb_handle {
  int device = 0;
  int ctx = 0;                   // launch context slot (per-handle launcher caches)
  std::recursive_mutex mu;       // calls on one handle take turns
  cudaStream_t stream = nullptr;
  // look-ahead stream: POTRF of the next diagonal tile overlaps the current
  // step's recompressions (factor_tlr)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_syrk = nullptr, ev_potrf = nullptr;
  // factored-recompression stream: the stacked-factor QRs of a batch run
  // beside the dense-path jobs' compression (factor_tlr)
  cudaStream_t lane2 = nullptr;
  cudaEvent_t ev_b = nullptr, ev_f = nullptr;
  cudaEvent_t ev[6];
  int64_t n = 0;
  int nb = 0, t = 0, cap = 0, max_rank = 0;
  bool npd_seen = false;   // set by compress_jobs' readback; factor_tlr stops
  std::vector<int> off, sz;
  double* dx = nullptr;          // point coordinates in the Pts layout (a1, a2, a3)
  double* dy = nullptr;
  double* dz = nullptr;          // cos(lat), great circle only
  double diam = 0.0;             // 2 * sphere radius; 0 => Euclidean
  std::vector<double> hxy;       // caller's (x, y) / (lon, lat), kept for tlrb_set_metric
  Pts pts() const { return Pts{dx, dy, dz, diam}; }
  double* diag = nullptr;         // the owned diagonal tiles, nb x nb each
  std::vector<double*> dptr;     // per diagonal tile: its storage (nullptr: owned elsewhere)
  double* lkk = nullptr;         // distributed: L_kk received from its owner (nb x nb)
  // distributed: the panel tiles received at the current step (row and
  // column broadcasts land in pbuf; their uptr / vptr point into it)
  double* pbuf = nullptr;
  size_t pbuf_cap = 0;           // doubles
  std::vector<size_t> recv_tiles;
  // tile factors: rank-adaptive bump arena, reset at every factorisation;
  // tile t owns U (nb x tcap[t]) and V (nb x tcap[t]), or a dense nb x nb
  char* arena = nullptr;
  size_t arena_bytes = 0, arena_off = 0, arena_peak = 0;
  size_t panel_peak = 0;           // largest received panel (distributed)
  std::vector<double*> uptr, vptr;
  std::vector<int> tcap;
  std::vector<int> rank;         // per lower tile
  std::vector<char> dense;       // per lower tile: stored dense (rank > max_rank), as L_ij^T in the U slab
  int* d_info = nullptr;         // [flag, tile, pivot]
  double* d_logdiag = nullptr;   // n
  double* d_scal = nullptr;      // [logdet, quad]
  double* d_z = nullptr;         // n (rhs / solution)
  double* d_w = nullptr;         // solve temporaries (t * nb)
  double* d_y = nullptr;         // y = L x output (n), allocated on first use
  // kriging
  double* d_ux = nullptr; double* d_uy = nullptr; double* d_uz = nullptr; double* d_pred = nullptr;
  double* d_partial = nullptr; double* d_pacc = nullptr; int64_t ucap = 0;
  DescArena ar;
  // compression workspace
  char* ws = nullptr;
  size_t ws_bytes = 0;
  size_t slot_doubles = 0;
  int max_jobs = 0;
  double* d_sums = nullptr;      // 6 per job
  double* d_aux = nullptr;       // 2 per job
  int* d_kind = nullptr;         // per job
  int* d_ok = nullptr;           // per job
  int* d_rank = nullptr;         // per job
  int* d_sweeps = nullptr;       // per job
  int* d_perm = nullptr;         // nb per job (QRCP column permutation)
  // state
  int factor_mode = 0;           // 0: none, 1: dense, 2: tlr
  MaternParamsDev mp{};
  double acc = 0;
  int err_tile = -1, err_pivot = -1;
  std::string msg;
  tlrb_stats st{};
  Flops work;
  int retries = 0, max_sweeps = 0;

  // 2D block-cyclic distribution: tile (i, j) lives on rank
  // (i mod P) * Q + (j mod Q); rank r sits in process row r / Q and process
  // column r mod Q.  cw == nullptr -> single-GPU path.
  int drank = 0, dworld = 1, P = 1, Q = 1;
  std::unique_ptr<Comm> cw, crow, ccol;   // world, my process row (Q members), my process column (P members)
  int* d_ibuf = nullptr;         // int all-reduce scratch (2 * ntile + 8)
  double* d_acc = nullptr;       // distributed solve accumulator (n)
  bool dist() const { return cw != nullptr; }
  int prow() const { return drank / Q; }
  int pcol() const { return drank % Q; }
  int owner(int i, int j) const { return (i % P) * Q + (j % Q); }
  bool own(int i, int j) const { return !cw || owner(i, j) == drank; }
  // group handle (tlrb_create with ngpus > 1, tlrb_create_group): one member
  // handle per rank, each driven by its own host thread per call
  std::vector<tlrb_handle*> members;
  bool group() const { return !members.empty(); }

  size_t tid(int i, int j) const { return (size_t)i * (i - 1) / 2 + j; }
  bool dn(int i, int j) const { return dense[tid(i, j)] != 0; }
  bool live(int i, int j) const { return dense[tid(i, j)] || rank[tid(i, j)] > 0; }
  double* Ut(int i, int j) const { return uptr[tid(i, j)]; }
  double* Vt(int i, int j) const { return vptr[tid(i, j)]; }
  void arena_reset() {
    arena_off = 0;
    recv_tiles.clear();
    std::fill(uptr.begin(), uptr.end(), nullptr);
    std::fill(vptr.begin(), vptr.end(), nullptr);
    std::fill(tcap.begin(), tcap.end(), 0);
  }
  double* arena_get(size_t doubles) {
    const size_t a = (arena_off + 255) & ~(size_t)255;
    if (a + doubles * sizeof(double) > arena_bytes)
      throw CudaError(cudaErrorMemoryAllocation, "tile factor arena exhausted", __FILE__, __LINE__);
    arena_off = a + doubles * sizeof(double);
    arena_peak = std::max(arena_peak, arena_off);
    return reinterpret_cast<double*>(arena + a);
  }
  // make tile t able to hold rank k (k == nb with dense: the whole L^T tile)
  void ensure(size_t t, int k, bool dense_tile = false) {
    if (k <= tcap[t] && (!dense_tile || tcap[t] >= nb)) return;
    const int c = dense_tile ? nb : std::min(nb, (k + 15) & ~15);
    uptr[t] = arena_get((size_t)nb * c);
    vptr[t] = dense_tile ? nullptr : arena_get((size_t)nb * c);
    tcap[t] = c;
  }
  double* D(int i) const { return dptr[i]; }
  // L_kk where the panel step needs it: owned, or received from its owner
  double* Dk(int k) const { return dptr[k] ? dptr[k] : lkk; }
  void sync() {
    TLRB_CUDA(cudaStreamSynchronize(stream));
    // the arena is reset below: descriptors queued on the look-ahead stream
    // must have been consumed too
    if (side) TLRB_CUDA(cudaStreamSynchronize(side));
    // descriptors still queued on lane2 keep the arena (it wraps with a
    // device sync when full)
    if (lane2 && cudaStreamQuery(lane2) == cudaErrorNotReady) {
      cudaGetLastError();
    } else {
      ar.reset();
    }
    if (g_prof.on) g_prof.drain();
  }
};

namespace {

int dense_rank_limit(const tlrb_handle* h, int m, int n) {
  if (h->max_rank <= 0) return std::numeric_limits<int>::max();   // no cap: the reference's rule only
  return (int)std::floor(std::min(dense_frac() * std::min(m, n), (double)h->max_rank));
}

bool trace_on() {
  static const bool on = getenv("TLRB_TRACE") != nullptr;
  return on;
}
double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

#define TLRB_NCCL(call)                                                              \
  do {                                                                               \
    ncclResult_t r_ = (call);                                                        \
    if (r_ != ncclSuccess) throw CudaError(cudaErrorUnknown, ncclGetErrorString(r_), __FILE__, __LINE__); \
  } while (0)

// every rank learns every tile's rank / dense flag (owners contribute, others
// 0): once per evaluation, after the factorisation (rank maps, statistics)
void sync_ranks(tlrb_handle* h) {
  if (!h->dist()) return;
  const size_t nt = h->rank.size();
  std::vector<int> buf(2 * nt, 0);
  for (int i = 1; i < h->t; ++i)
    for (int j = 0; j < i; ++j)
      if (h->own(i, j)) {
        buf[h->tid(i, j)] = h->rank[h->tid(i, j)];
        buf[nt + h->tid(i, j)] = h->dense[h->tid(i, j)];
      }
  if (nt) {
    TLRB_CUDA(cudaMemcpyAsync(h->d_ibuf, h->ar.put(buf, h->stream), 2 * nt * sizeof(int), cudaMemcpyDeviceToDevice,
                              h->stream));
    h->cw->allreduce_sum(h->d_ibuf, 2 * nt, CType::I32, h->stream);
    TLRB_CUDA(cudaMemcpyAsync(buf.data(), h->d_ibuf, 2 * nt * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  }
  h->sync();
  for (size_t q = 0; q < nt; ++q) {
    h->rank[q] = buf[q];
    h->dense[q] = (char)buf[nt + q];
  }
}

__global__ void axpy_kernel(double* y, const double* x, double a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) y[i] += a * x[i];
}

// ------------------------------------------------------------ compression
struct Job {
  int m, n;           // M is m x n
  int s;              // QRCP kernel hint on entry; QRCP rank r (Jacobi width) after it
  int kind;           // bit1: recompression (noise floor)
  double* M;          // slot pointers
  double* E; double* Y; double* Q; double* Om; double* Bt; double* Vs; double* F; double* sig; double* T;
  double* Uout; double* Vout; int ldu, ldv;
  int out_rank;
  bool dense_out;     // rank above max_rank: stored dense (L^T in Uout, ld ldu)
  uint64_t seed;      // unused (kept for descriptor stability)
  // factored recompression (compression.py:54-81): M is the K x K core,
  // U_new = Qu u_core, V_new = Qv v_core are formed after compress_jobs by
  // applying the blocked Householder reflectors of the stacked-factor QRs
  bool factored = false;
  BqrProb qu{}, qv{};
  int mu = 0, nv = 0;
  double* Ufin = nullptr; double* Vfin = nullptr;
  // orthogonal-part shortcut of the factored path (V side): the kept
  // factor's k1 columns are not refactored (Q1v = V_ij in the slot)
  int k1 = 0;
  double* Q1v = nullptr;
  long tile = -1;     // destination tile (outputs allocated once the rank is known)
  long ftile = -1;    // factored path: destination tile of Qu u_core / Qv v_core
};

void bind_slot(tlrb_handle* h, Job& J, int slot) {
  double* base = reinterpret_cast<double*>(h->ws) + (size_t)slot * h->slot_doubles;
  const size_t nb2 = (size_t)h->nb * h->nb;
  J.M = base;
  J.E = base + nb2;
  J.Y = base + 2 * nb2;
  J.Q = base + 3 * nb2;
  J.Om = base + 4 * nb2;
  J.Bt = base + 5 * nb2;
  J.Vs = base + 6 * nb2;
  J.F = base + 7 * nb2;     // factored path: core factors u_core, v_core
  J.sig = base + 8 * nb2;
  J.T = J.sig + h->nb;
}

// Compress the M of every job (already formed in its slot) to acc; writes
// U = M V_k (m x k) and V_k (n x k) into the job's output slabs.
//   1. E <- M (the original is needed for U = M V_k)
//   2. truncated QRCP of M until ||residual||_F <= 1e-3 acc ||M||_F
//   3. X = R^T (n x r, masked transpose), one-sided Jacobi on X -> sorted
//      sigma, normalised columns (= right singular vectors in pivoted order),
//      truncation rank k with e2 = ||residual||^2 and the noise floor
//   4. V_k = P * columns (row un-permutation), U = E V_k (DMMA GEMM)
void compress_jobs(tlrb_handle* h, std::vector<Job>& jobs, double acc, int j0 = 0) {
  const int nj = (int)jobs.size();
  if (!nj) return;
  cudaStream_t s = h->stream;
  // per-job device arrays from position j0 (a batch may be compressed in parts)
  int* d_perm = reinterpret_cast<int*>(h->d_perm) + (size_t)j0 * h->nb;
  int* d_rank = h->d_rank + j0;
  int* d_sweeps = h->d_sweeps + j0;
  int* d_kind = h->d_kind + j0;
  int* d_ok = h->d_ok + j0;
  double* d_sums = h->d_sums + 6 * (size_t)j0;
  double* d_aux = h->d_aux + 3 * (size_t)j0;
  std::vector<char> gathered;
  {
    std::vector<CopyProb> cp;
    std::vector<QrcpProb> qp;
    for (int j = 0; j < nj; ++j) {
      Job& J = jobs[j];
      cp.push_back({J.M, J.m, J.E, J.m, J.m, J.n, 0, 1.0, 0, nullptr});
      qp.push_back({J.M, J.m, J.m, J.n, d_perm + (size_t)j * h->nb, d_rank + j, d_sums + 6 * j + 1,
                    (qrcp_rel_tol() * acc) * (qrcp_rel_tol() * acc), J.s});
      // a tile whose QRCP rank passes the dense limit is stored exactly: its QRCP may stop there
      if (dense_by_qrcp() && !J.factored && J.tile >= 0 && h->max_rank > 0)
        qp.back().cap = dense_rank_limit(h, J.m, J.n);
    }
    launch_copy(cp, h->ar, s);
    launch_qrcp(qp, gathered, h->ar, s);
  }
  std::vector<int> rr(nj);
  const double t_q0 = trace_on() ? now_ms() : 0;
  if (trace_on()) h->sync();
  TLRB_CUDA(cudaMemcpyAsync(rr.data(), d_rank, nj * sizeof(int), cudaMemcpyDeviceToHost, s));
  int info0 = 0;   // NPD flag of the POTRFs so far, read with the ranks (no extra sync)
  TLRB_CUDA(cudaMemcpyAsync(&info0, h->d_info, sizeof(int), cudaMemcpyDeviceToHost, s));
  h->sync();
  if (info0) {   // a POTRF failed: the factorisation stops, the batch is not finished
    h->npd_seen = true;
    for (Job& J : jobs) {
      J.out_rank = 0;
      J.dense_out = false;
    }
    return;
  }
  const double t_q1 = trace_on() ? now_ms() : 0;
  std::vector<int> kinds(nj);
  // under a storage cap, a tile whose QRCP rank already exceeds the dense
  // limit is kept exact without its SVD: the truncation rank never exceeds
  // the QRCP rank (the Jacobi tail only shrinks it), and an exact tile is
  // never less accurate than the truncated one (see dense_frac)
  std::vector<char> pre_dense(nj, 0);
  {
    std::vector<CopyProb> cp;
    for (int j = 0; j < nj; ++j) {
      Job& J = jobs[j];
      J.s = rr[j];
      kinds[j] = 1 | (J.kind & 2);   // e2 = QRCP residual (sums[6j+1])
      pre_dense[j] = dense_by_qrcp() && !J.factored && J.tile >= 0 && J.s > dense_rank_limit(h, J.m, J.n);
      // X (n x r): X(p, c) = R(c, p) for p >= c
      if (J.s && !pre_dense[j])
        cp.push_back({J.M, J.m, J.Bt, J.n, J.n, J.s, 1, 1.0, 1, nullptr,
                      gathered[j] ? d_perm + (size_t)j * h->nb : nullptr});
    }
    launch_copy(cp, h->ar, s);
  }
  TLRB_CUDA(cudaMemcpyAsync(d_kind, h->ar.put(kinds, s), nj * sizeof(int), cudaMemcpyDeviceToDevice, s));
  launch_aux(d_sums, d_kind, nj, d_aux, d_ok, 0.0, s);
  {
    std::vector<JacobiProb> jp;
    for (int j = 0; j < nj; ++j) {
      Job& J = jobs[j];
      if (pre_dense[j]) continue;   // d_rank keeps the QRCP rank (> the dense limit)
      jp.push_back({J.Bt, J.n, J.Vs, J.n, J.sig, d_aux + 3 * j, acc, d_rank + j,
                    d_sweeps + j, J.n, J.s});
    }
    static long long* d_prof = nullptr;
    const bool prof = getenv("TLRB_JACOBI_PROF") != nullptr;
    if (prof) {
      if (!d_prof) TLRB_CUDA(cudaMalloc(&d_prof, 16 * 8 * sizeof(long long)));
      TLRB_CUDA(cudaMemsetAsync(d_prof, 0, 16 * 8 * sizeof(long long), s));
      for (auto& q : jp) q.prof = nullptr;
      jp[0].prof = d_prof;   // first problem only (one tile in tools/one_tile.py)
    }
    if (!jp.empty()) launch_jacobi(jp, h->ar, s);
    if (prof) {
      long long hp[16 * 8];
      TLRB_CUDA(cudaMemcpyAsync(hp, d_prof, sizeof hp, cudaMemcpyDeviceToHost, s));
      h->sync();
      for (int c = 0; c < 16; ++c)
        if (hp[8 * c + 6])
          fprintf(stderr, "[jacobi-prof] cta %d load %lld within %lld cross %lld store %lld sync %lld conv %lld sweeps %lld\n",
                  c, hp[8 * c], hp[8 * c + 1], hp[8 * c + 2], hp[8 * c + 3], hp[8 * c + 4], hp[8 * c + 5], hp[8 * c + 6]);
    }
  }
  std::vector<int> rk(nj), sw(nj);
  TLRB_CUDA(cudaMemcpyAsync(rk.data(), d_rank, nj * sizeof(int), cudaMemcpyDeviceToHost, s));
  TLRB_CUDA(cudaMemcpyAsync(sw.data(), d_sweeps, nj * sizeof(int), cudaMemcpyDeviceToHost, s));
  h->sync();
  if (trace_on()) {
    int rmax = 0, smax = 0;
    for (int j = 0; j < nj; ++j) { rmax = std::max(rmax, rr[j]); smax = std::max(smax, sw[j]); }
    fprintf(stderr, "[tlrb] compress nj=%d  qrcp %.2f ms  jacobi %.2f ms  rmax=%d sweeps<=%d\n", nj,
            t_q1 - t_q0, now_ms() - t_q1, rmax, smax);
    if (getenv("TLRB_TRACE_JOBS"))   // per job: m n qrcp-rank final-rank sweeps
      for (int j = 0; j < nj; ++j)
        fprintf(stderr, "[job] %d %d %d %d %d\n", jobs[j].m, jobs[j].n, rr[j], rk[j], sw[j]);
  }
  std::vector<GemmProb> gu;
  std::vector<CopyProb> cv;
  for (int j = 0; j < nj; ++j) {
    Job& J = jobs[j];
    if (pre_dense[j]) sw[j] = 0;   // no SVD ran (its d_sweeps entry is stale)
    J.out_rank = J.s ? rk[j] : 0;
    h->max_sweeps = std::max(h->max_sweeps, J.s ? sw[j] : 0);
    // one-sided Jacobi as implemented: per sweep s(s-1)/2 pairs x (one dot,
    // 2n flops, + the scaled rotation, 4n flops) = 3 n s (s-1) flops
    if (g_prof.on && J.s) g_prof.add_work(K_JACOBI, 3.0 * J.n * (double)J.s * (J.s - 1) * sw[j], 0);
    const int k = J.out_rank;
    // (a standalone compression, tlrb_compress_tile, has no tile: always U V^T)
    J.dense_out = !J.factored && J.tile >= 0 && k > dense_rank_limit(h, J.m, J.n);
    if (J.tile >= 0) {   // the destination tile's storage is sized by the new rank
      if (J.dense_out || k) h->ensure((size_t)J.tile, J.dense_out ? h->nb : k, J.dense_out);
      J.Uout = h->uptr[J.tile];
      J.Vout = h->vptr[J.tile];
      J.ldu = J.ldv = h->nb;
    }
    if (J.dense_out) {   // A13: over the storage cap -> keep the tile exact (dense, transposed)
      cv.push_back({J.E, J.m, J.Uout, J.ldu, J.n, J.m, 1, 1.0, 0, nullptr});
      continue;
    }
    if (!k) continue;
    cv.push_back({J.Vs, J.n, J.Vout, J.ldv, J.n, k, 0, 1.0, 0, d_perm + (size_t)j * h->nb});
    gu.push_back({J.E, J.Vout, nullptr, J.Uout, J.m, k, J.n, J.m, J.ldv, J.ldu, J.ldu, 0, 0, 0, 1.0, 0.0});
  }
  launch_copy(cv, h->ar, s);
  launch_gemm(gu, h->ar, s);
}

// predicted number of QRCP steps of an update (selects the QRCP kernel)
int rank_hint(int prev_rank, int n) {
  int s = (int)std::ceil(1.25 * prev_rank) + 32;
  s = (s + 7) & ~7;
  return std::min(s, n);
}

// ----------------------------------------------------------- generation
void generate(tlrb_handle* h, double nugget, bool dense_lower) {
  std::vector<GenTile> tiles;
  for (int i = 0; i < h->t; ++i) {
    if (h->own(i, i)) tiles.push_back({h->D(i), h->nb, h->off[i], h->sz[i], h->off[i], h->sz[i], nugget});
    if (dense_lower)
      for (int j = 0; j < i; ++j)  // L_ij^T: rows = tile j points, cols = tile i points
        if (h->own(i, j)) tiles.push_back({h->Ut(i, j), h->nb, h->off[j], h->sz[j], h->off[i], h->sz[i], 0.0});
  }
  launch_gen_tiles(tiles, h->pts(), h->mp, h->ar, h->stream);
  for (int i = 0; i < h->t; ++i) {
    h->work.add(0, 8.0 * h->sz[i] * h->sz[i]);
    if (dense_lower)
      for (int j = 0; j < i; ++j) h->work.add(0, 8.0 * h->sz[i] * h->sz[j]);
  }
}

void compress_all(tlrb_handle* h, double acc) {
  std::vector<std::pair<int, int>> all;
  for (int i = 1; i < h->t; ++i)
    for (int j = 0; j < i; ++j)
      if (h->own(i, j)) all.push_back({i, j});
  // far tiles first (small ranks), near-diagonal last
  for (size_t c0 = 0; c0 < all.size(); c0 += h->max_jobs) {
    const size_t c1 = std::min(all.size(), c0 + h->max_jobs);
    std::vector<Job> jobs;
    std::vector<GenTile> gen;
    for (size_t q = c0; q < c1; ++q) {
      const int i = all[q].first, j = all[q].second;
      Job J{};
      bind_slot(h, J, (int)(q - c0));
      J.m = h->sz[i];
      J.n = h->sz[j];
      // initial sketch: ranks grow towards the diagonal
      const int off = i - j;
      J.s = off <= 2 ? J.n : std::min(J.n, 64);   // QRCP kernel hint (predicted steps)
      J.kind = 0;
      J.tile = (long)h->tid(i, j);
      J.seed = h->tid(i, j) * 131 + 17;
      jobs.push_back(J);
      gen.push_back({J.M, J.m, h->off[i], J.m, h->off[j], J.n, 0.0});
    }
    launch_gen_tiles(gen, h->pts(), h->mp, h->ar, h->stream);
    compress_jobs(h, jobs, acc);
    for (size_t q = c0; q < c1; ++q) {
      const Job& J = jobs[q - c0];
      h->rank[h->tid(all[q].first, all[q].second)] = J.dense_out ? 0 : J.out_rank;
      h->dense[h->tid(all[q].first, all[q].second)] = J.dense_out;
      const double m = J.m, n = J.n, k = J.out_rank;
      h->work.add(4.0 * m * n * k, 8.0 * m * n + 8.0 * k * (m + n));
    }
  }
}

// ------------------------------------------------------------------ POTRF
// L_kk on its owner (linalg.py:36-45); distributed handles then share it
// down process column k mod Q, where the panel tiles (i, k) live (share_lkk)
// right-looking blocked Cholesky of one n x n tile (lower, ld): 32-column
// panel kernel + DMMA trailing update; the first failure lands in info
void potrf_blocks(double* A, int ld, int n, int tile, int* info, double* logdiag, DescArena& ar, cudaStream_t s) {
  for (int r0 = 0; r0 < n; r0 += kPotrfBlock) {
    const int bs = std::min(kPotrfBlock, n - r0);
    launch_potrf_block(A, ld, n, r0, bs, tile, info, logdiag, s);
    const int rest = n - r0 - bs;
    if (rest > 0) {
      double* A21 = A + (size_t)r0 * ld + r0 + bs;
      double* A22 = A + (size_t)(r0 + bs) * ld + r0 + bs;
      launch_gemm({GemmProb{A21, A21, A22, A22, rest, rest, bs, ld, ld, ld, ld, 0, 1, 1, -1.0, 1.0}}, ar, s);
    }
  }
}

void potrf(tlrb_handle* h, int k, cudaStream_t s = nullptr) {
  if (!s) s = h->stream;
  if (!h->own(k, k)) return;
  const int n = h->sz[k];
  potrf_blocks(h->D(k), h->nb, n, k, h->d_info, h->d_logdiag + h->off[k], h->ar, s);
  const double nn = n;
  h->work.add(nn * nn * nn / 3.0, 16.0 * nn * nn);
}

void share_lkk(tlrb_handle* h, int k) {
  if (!h->dist() || h->pcol() != k % h->Q) return;
  double* buf = h->own(k, k) ? h->D(k) : h->lkk;
  h->ccol->bcast(buf, (size_t)h->nb * h->nb, CType::F64, k % h->P, h->stream);
}

// One all-reduce per panel step (distributed): the NPD flag of POTRF(k) and
// the ranks / dense flags of the panel tiles (i, k), i > k, which every rank
// needs to size the received panel and build its updates.  Returns true on NPD.
bool set_npd(tlrb_handle* h, const int* info) {
  if (!info[0]) return false;
  h->err_tile = info[1];
  h->err_pivot = info[2];
  char b[160];
  snprintf(b, sizeof b, "covariance not positive definite at tile %d, pivot %d; consider adding a nugget",
           info[1], info[2]);
  h->msg = b;
  return true;
}

// every rank's POTRF report [flag, tile, pivot] sits in its own slot of the
// all-reduced buffer; the first failing tile wins (a failure poisons the
// later diagonal tiles, which other ranks may also report)
void first_failure(const int* slots, int world, int* info) {
  info[0] = info[1] = info[2] = 0;
  for (int r = 0; r < world; ++r)
    if (slots[3 * r] && (!info[0] || slots[3 * r + 1] < info[1])) {
      info[0] = 1;
      info[1] = slots[3 * r + 1];
      info[2] = slots[3 * r + 2];
    }
}

// One all-reduce per panel step (distributed): the POTRF reports and the
// ranks / dense flags of the panel tiles (i, k), i > k, which every rank
// needs to size the received panel and build its updates.  Returns true on NPD.
bool panel_meta(tlrb_handle* h, int k) {
  const int t = h->t, W = h->dworld;
  const int np = t - k - 1;
  std::vector<int> buf(3 * (size_t)W + 2 * (size_t)np, 0);
  int* meta = buf.data() + 3 * W;
  for (int i = k + 1; i < t; ++i)
    if (h->own(i, k)) {
      meta[i - k - 1] = h->rank[h->tid(i, k)];
      meta[np + i - k - 1] = h->dense[h->tid(i, k)];
    }
  int* d = h->d_ibuf;
  TLRB_CUDA(cudaMemcpyAsync(d, h->ar.put(buf, h->stream), buf.size() * sizeof(int), cudaMemcpyDeviceToDevice,
                            h->stream));
  TLRB_CUDA(cudaMemcpyAsync(d + 3 * h->drank, h->d_info, 3 * sizeof(int), cudaMemcpyDeviceToDevice, h->stream));
  h->cw->allreduce_sum(d, buf.size(), CType::I32, h->stream);
  TLRB_CUDA(cudaMemcpyAsync(buf.data(), d, buf.size() * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  h->sync();
  meta = buf.data() + 3 * W;
  for (int i = k + 1; i < t; ++i) {
    h->rank[h->tid(i, k)] = meta[i - k - 1];
    h->dense[h->tid(i, k)] = (char)meta[np + i - k - 1];
  }
  int info[3];
  first_failure(buf.data(), W, info);
  return set_npd(h, info);
}

// Panel broadcast of step k, one packed buffer per
// broadcast.  Rank (p, q) needs L_ik for its tiles (i, j) — i mod P = p, the
// panel owner is in its own process row — and L_jk — j mod Q = q:
//   row step    in each process row p, member k mod Q sends its panel tiles
//               (i, k), i mod P = p, packed, to the row;
//   column step in each process column q, member p sends the tiles (j, k),
//               j mod P = p, j mod Q = q (owned or just received), packed,
//               to the column — one broadcast per p.
// A packed tile is U (nb x c) then V (nb x c), c = its rank, or the whole
// dense L_ik^T (nb x sz_i).  Receivers point the tile's factors into pbuf;
// release_panel drops them after the step, so a rank only ever stores its own
// tiles plus one panel.
size_t packed_doubles(const tlrb_handle* h, int i, int k, bool dense_mode) {
  if (dense_mode || h->dn(i, k)) return (size_t)h->nb * h->sz[i];
  return 2 * (size_t)h->nb * h->rank[h->tid(i, k)];
}

void bcast_panel(tlrb_handle* h, int k, bool dense_mode) {
  if (!h->dist()) return;
  const int t = h->t, nb = h->nb, P = h->P, Q = h->Q, myp = h->prow(), myq = h->pcol();
  std::vector<int> rowt;   // row step tiles
  size_t rowtot = 0;
  for (int i = k + 1; i < t; ++i)
    if (i % P == myp && packed_doubles(h, i, k, dense_mode)) {
      rowt.push_back(i);
      rowtot += packed_doubles(h, i, k, dense_mode);
    }
  std::vector<std::vector<int>> colt(P);
  std::vector<size_t> coltot(P, 0);
  size_t coll = 0;
  for (int j = k + 1; j < t; ++j)
    if (j % Q == myq && packed_doubles(h, j, k, dense_mode)) {
      colt[j % P].push_back(j);
      coltot[j % P] += packed_doubles(h, j, k, dense_mode);
    }
  for (int p = 0; p < P; ++p) coll += coltot[p];
  const size_t need = (Q > 1 ? rowtot : 0) + (P > 1 ? coll : 0);
  if (need > h->pbuf_cap) {
    h->sync();   // earlier steps' updates may still read the old panel
    if (h->pbuf) TLRB_CUDA(cudaFree(h->pbuf));
    h->pbuf_cap = std::max(need, h->pbuf_cap + h->pbuf_cap / 2);
    TLRB_CUDA(cudaMalloc(&h->pbuf, h->pbuf_cap * sizeof(double)));
  }
  h->panel_peak = std::max(h->panel_peak, need * sizeof(double));
  // pack (root) or point into (receiver) one broadcast's tiles
  auto run = [&](const std::vector<int>& tiles, double* base, size_t tot, bool root, Comm& c, int croot) {
    if (!tot) return;
    std::vector<CopyProb> cp;
    size_t o = 0;
    for (int i : tiles) {
      const size_t q = h->tid(i, k);
      const bool dt = dense_mode || h->dn(i, k);
      const int c1 = dt ? h->sz[i] : h->rank[q];
      if (root) {
        cp.push_back({h->uptr[q], nb, base + o, nb, nb, c1, 0, 1.0, 0, nullptr});
        if (!dt) cp.push_back({h->vptr[q], nb, base + o + (size_t)nb * c1, nb, nb, c1, 0, 1.0, 0, nullptr});
      } else {
        h->uptr[q] = base + o;
        h->vptr[q] = dt ? nullptr : base + o + (size_t)nb * c1;
        h->tcap[q] = dt ? nb : c1;
        h->recv_tiles.push_back(q);
      }
      o += dt ? (size_t)nb * c1 : 2 * (size_t)nb * c1;
    }
    if (root) launch_copy(cp, h->ar, h->stream);
    c.bcast(base, tot, CType::F64, croot, h->stream);
  };
  double* base = h->pbuf;
  if (Q > 1) {
    run(rowt, base, rowtot, myq == k % Q, *h->crow, k % Q);
    base += rowtot;
  }
  if (P > 1)
    for (int p = 0; p < P; ++p) {
      run(colt[p], base, coltot[p], myp == p, *h->ccol, p);
      base += coltot[p];
    }
}

// the received panel tiles of the step just finished are not kept
void release_panel(tlrb_handle* h) {
  for (size_t q : h->recv_tiles) {
    h->uptr[q] = h->vptr[q] = nullptr;
    h->tcap[q] = 0;
  }
  h->recv_tiles.clear();
}

bool check_npd(tlrb_handle* h) {
  int info[3];
  if (h->dist()) {   // the failing tile's owner reported it; everyone stops
    const int W = h->dworld;
    std::vector<int> slots(3 * (size_t)W, 0);
    int* d = h->d_ibuf;
    TLRB_CUDA(cudaMemsetAsync(d, 0, slots.size() * sizeof(int), h->stream));
    TLRB_CUDA(cudaMemcpyAsync(d + 3 * h->drank, h->d_info, 3 * sizeof(int), cudaMemcpyDeviceToDevice, h->stream));
    h->cw->allreduce_sum(d, slots.size(), CType::I32, h->stream);
    TLRB_CUDA(cudaMemcpyAsync(slots.data(), d, slots.size() * sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    h->sync();
    first_failure(slots.data(), W, info);
    return set_npd(h, info);
  }
  TLRB_CUDA(cudaMemcpyAsync(info, h->d_info, sizeof info, cudaMemcpyDeviceToHost, h->stream));
  h->sync();
  if (info[0])   // a look-ahead POTRF may have been writing it: re-read settled
    TLRB_CUDA(cudaMemcpy(info, h->d_info, sizeof info, cudaMemcpyDeviceToHost));
  return set_npd(h, info);
}

// ------------------------------------------------------ dense factorisation
bool factor_dense(tlrb_handle* h) {
  const int t = h->t, nb = h->nb;
  // look-ahead: POTRF(k+1) needs only step k's SYRK of D(k+1); it is
  // launched first and the POTRF runs on the side stream beside the rest of
  // the trailing update (linalg.py:82-103 order per tile is unchanged)
  static const bool lookahead = !(getenv("TLRB_LOOKAHEAD") && atoi(getenv("TLRB_LOOKAHEAD")) == 0);
  int ahead = -1;
  for (int k = 0; k < t; ++k) {
    if (ahead == k) TLRB_CUDA(cudaStreamWaitEvent(h->stream, h->ev_potrf, 0));
    else potrf(h, k);
    share_lkk(h, k);
    std::vector<TrsmProb> tp;
    for (int i = k + 1; i < t; ++i)
      if (h->own(i, k)) tp.push_back({h->Dk(k), nb, h->Ut(i, k), nb, h->sz[k], h->sz[i]});
    launch_trsm_panel(tp, h->ar, h->stream);
    bcast_panel(h, k, true);
    if (lookahead && k + 1 < t && h->own(k + 1, k + 1)) {
      const int j = k + 1;
      launch_gemm({GemmProb{h->Ut(j, k), h->Ut(j, k), h->D(j), h->D(j), h->sz[j], h->sz[j], h->sz[k], nb, nb, nb,
                            nb, 1, 0, 1, -1.0, 1.0}}, h->ar, h->stream);
      TLRB_CUDA(cudaEventRecord(h->ev_syrk, h->stream));
      TLRB_CUDA(cudaStreamWaitEvent(h->side, h->ev_syrk, 0));
      potrf(h, j, h->side);
      TLRB_CUDA(cudaEventRecord(h->ev_potrf, h->side));
      ahead = j;
    }
    std::vector<GemmProb> gp;
    const double nk = h->sz[k];
    for (int j = k + 1; j < t; ++j) {
      // D_j -= L_jk L_jk^T = T_jk^T T_jk  (j = k + 1 already went ahead of the look-ahead POTRF)
      if (h->own(j, j) && ahead != j)
        gp.push_back({h->Ut(j, k), h->Ut(j, k), h->D(j), h->D(j), h->sz[j], h->sz[j], h->sz[k], nb, nb, nb,
                      nb, 1, 0, 1, -1.0, 1.0});
      h->work.add(nk * h->sz[j] * h->sz[j], 8.0 * (2.0 * nk * h->sz[j] + 2.0 * h->sz[j] * h->sz[j]));
      // T_ij -= T_jk^T T_ik
      for (int i = j + 1; i < t; ++i) {
        if (!h->own(i, j)) continue;
        gp.push_back({h->Ut(j, k), h->Ut(i, k), h->Ut(i, j), h->Ut(i, j), h->sz[j], h->sz[i], h->sz[k], nb,
                      nb, nb, nb, 1, 0, 0, -1.0, 1.0});
        h->work.add(2.0 * nk * h->sz[i] * h->sz[j],
                    8.0 * (nk * (h->sz[i] + h->sz[j]) + 2.0 * h->sz[i] * h->sz[j]));
      }
    }
    for (int i = k + 1; i < t; ++i)
      h->work.add(nk * nk * h->sz[i], 8.0 * (nk * nk / 2 + 2.0 * nk * h->sz[i]));
    launch_gemm(gp, h->ar, h->stream);
    release_panel(h);
  }
  return !check_npd(h);
}

// -------------------------------------------------------- TLR factorisation
bool factor_tlr(tlrb_handle* h, double acc) {
  const int t = h->t, nb = h->nb;
  h->npd_seen = false;
  double* tmp = reinterpret_cast<double*>(h->ws);  // small products before the job batch
  // POTRF(k+1) only needs step k's SYRK of D(k+1): it runs on the look-ahead
  // stream while step k's recompressions run (single-GPU handles)
  static const bool lookahead = !(getenv("TLRB_LOOKAHEAD") && atoi(getenv("TLRB_LOOKAHEAD")) == 0);
  int ahead = -1;
  for (int k = 0; k < t; ++k) {
    const double tk0 = trace_on() ? now_ms() : 0;
    if (ahead == k) TLRB_CUDA(cudaStreamWaitEvent(h->stream, h->ev_potrf, 0));
    else potrf(h, k);
    share_lkk(h, k);
    // K4: V_ik <- L_kk^-1 V_ik (low-rank) / L_ik^T <- L_kk^-1 A_ik^T (dense, A13)
    std::vector<TrsmProb> tp;
    for (int i = k + 1; i < t; ++i) {
      const double nk = h->sz[k];
      if (!h->own(i, k)) continue;
      if (h->dn(i, k)) {
        tp.push_back({h->Dk(k), nb, h->Ut(i, k), nb, h->sz[k], h->sz[i]});
        h->work.add(nk * nk * h->sz[i], 8.0 * (nk * nk / 2 + 2.0 * nk * h->sz[i]));
        continue;
      }
      const int r = h->rank[h->tid(i, k)];
      if (r) tp.push_back({h->Dk(k), nb, h->Vt(i, k), nb, h->sz[k], r});
      if (r) h->work.add(nk * nk * r, 8.0 * (nk * nk / 2 + 2.0 * nk * r));
    }
    launch_trsm_panel(tp, h->ar, h->stream);
    // single GPU: the NPD flag is read with the next rank readback (no sync
    // here); a failed POTRF only lets this step's batch run on garbage.
    // Distributed: one all-reduce carries the flag and the panel's ranks.
    if (h->dist() ? panel_meta(h, k) : (h->npd_seen && check_npd(h))) return false;
    bcast_panel(h, k, false);
    // K5: D_j -= U_jk (V_jk^T V_jk) U_jk^T  (dense panel tile: D_j -= T_jk^T T_jk)
    {
      std::vector<GemmProb> g1, g2, g3;
      size_t o = 0;
      const size_t ws_doubles = h->ws_bytes / sizeof(double);
      for (int j = k + 1; j < t; ++j) {
        const double nj = h->sz[j];
        if (!h->own(j, j)) continue;
        if (h->dn(j, k)) {
          g3.push_back({h->Ut(j, k), h->Ut(j, k), h->D(j), h->D(j), h->sz[j], h->sz[j], h->sz[k], nb, nb, nb,
                        nb, 1, 0, 1, -1.0, 1.0});
          h->work.add(nj * nj * h->sz[k], 8.0 * (2.0 * nj * h->sz[k] + 2.0 * nj * nj));
          continue;
        }
        const int r = h->rank[h->tid(j, k)];
        if (!r) continue;
        if (o + (size_t)r * r + (size_t)h->sz[j] * r > ws_doubles) {
          launch_gemm(g1, h->ar, h->stream);
          launch_gemm(g2, h->ar, h->stream);
          launch_gemm(g3, h->ar, h->stream);
          g1.clear(); g2.clear(); g3.clear();
          o = 0;
        }
        double* X = tmp + o;
        o += (size_t)r * r;
        double* W = tmp + o;
        o += (size_t)h->sz[j] * r;
        g1.push_back({h->Vt(j, k), h->Vt(j, k), nullptr, X, r, r, h->sz[k], nb, nb, r, r, 1, 0, 0, 1.0, 0.0});
        g2.push_back({h->Ut(j, k), X, nullptr, W, h->sz[j], r, r, nb, r, h->sz[j], h->sz[j], 0, 0, 0, 1.0, 0.0});
        g3.push_back({W, h->Ut(j, k), h->D(j), h->D(j), h->sz[j], h->sz[j], r, h->sz[j], nb, nb, nb, 0, 1, 1,
                      -1.0, 1.0});
        h->work.add(4.0 * nj * r * r + 2.0 * nj * nj * r, 8.0 * (2.0 * nj * r + 2.0 * nj * nj));
      }
      launch_gemm(g1, h->ar, h->stream);
      launch_gemm(g2, h->ar, h->stream);
      launch_gemm(g3, h->ar, h->stream);
    }
    if (lookahead && k + 1 < t && h->own(k + 1, k + 1)) {
      TLRB_CUDA(cudaEventRecord(h->ev_syrk, h->stream));
      TLRB_CUDA(cudaStreamWaitEvent(h->side, h->ev_syrk, 0));
      potrf(h, k + 1, h->side);
      TLRB_CUDA(cudaEventRecord(h->ev_potrf, h->side));
      ahead = k + 1;
    }
    if (trace_on()) {
      h->sync();
      fprintf(stderr, "[tlrb] step %d potrf+trsm+syrk %.2f ms\n", k, now_ms() - tk0);
    }
    // K6 + K7: updates of (i, j), i > j > k, in job batches; a rank-0 panel
    // tile skips the update exactly like linalg.py:135
    std::vector<std::pair<int, int>> upd;
    std::vector<GemmProb> dx, dy, dt;   // dense targets (A13): T_ij -= (L_ik L_jk^T)^T in place
    {
      double* tmpd = reinterpret_cast<double*>(h->ws);
      size_t o = 0;
      const size_t ws_doubles = h->ws_bytes / sizeof(double);
      for (int j = k + 1; j < t; ++j)
        for (int i = j + 1; i < t; ++i) {
          if (!(h->live(i, k) && h->live(j, k)) || !h->own(i, j)) continue;
          if (!h->dn(i, j)) { upd.push_back({i, j}); continue; }
          // a tile over the rank cap stays dense: no recompression, exact update
          const int ki = h->rank[h->tid(i, k)], kj = h->rank[h->tid(j, k)];
          const bool di = h->dn(i, k), dj = h->dn(j, k);
          const int mi = h->sz[i], mj = h->sz[j], mk = h->sz[k];
          double* T = h->Ut(i, j);
          if (o + (size_t)nb * nb > ws_doubles) {
            launch_gemm(dx, h->ar, h->stream); launch_gemm(dy, h->ar, h->stream); launch_gemm(dt, h->ar, h->stream);
            dx.clear(); dy.clear(); dt.clear();
            o = 0;
          }
          double* W = tmpd + o;
          o += (size_t)nb * nb;
          if (!di && !dj) {        // T -= U_jk (V_jk^T V_ik) U_ik^T
            double* X = W;                          // kj x ki
            double* Y = W + (size_t)kj * ki;        // mj x ki
            dx.push_back({h->Vt(j, k), h->Vt(i, k), nullptr, X, kj, ki, mk, nb, nb, kj, kj, 1, 0, 0, 1.0, 0.0});
            dy.push_back({h->Ut(j, k), X, nullptr, Y, mj, ki, kj, nb, kj, mj, mj, 0, 0, 0, 1.0, 0.0});
            dt.push_back({Y, h->Ut(i, k), T, T, mj, mi, ki, mj, nb, nb, nb, 0, 1, 0, -1.0, 1.0});
          } else if (di && !dj) {  // T -= U_jk (V_jk^T T_ik)
            dx.push_back({h->Vt(j, k), h->Ut(i, k), nullptr, W, kj, mi, mk, nb, nb, kj, kj, 1, 0, 0, 1.0, 0.0});
            dt.push_back({h->Ut(j, k), W, T, T, mj, mi, kj, nb, kj, nb, nb, 0, 0, 0, -1.0, 1.0});
          } else if (!di && dj) {  // T -= (T_jk^T V_ik) U_ik^T
            dx.push_back({h->Ut(j, k), h->Vt(i, k), nullptr, W, mj, ki, mk, nb, nb, mj, mj, 1, 0, 0, 1.0, 0.0});
            dt.push_back({W, h->Ut(i, k), T, T, mj, mi, ki, mj, nb, nb, nb, 0, 1, 0, -1.0, 1.0});
          } else {                 // T -= T_jk^T T_ik
            dt.push_back({h->Ut(j, k), h->Ut(i, k), T, T, mj, mi, mk, nb, nb, nb, nb, 1, 0, 0, -1.0, 1.0});
          }
          const double a = di ? mk : ki, b = dj ? mk : kj;
          h->work.add(di && dj ? 2.0 * mi * mj * mk : 2.0 * mi * mj * std::min(a, b) + 2.0 * mk * a * b,
                      8.0 * (2.0 * mi * mj + mk * (a + b)));
        }
      launch_gemm(dx, h->ar, h->stream);
      launch_gemm(dy, h->ar, h->stream);
      launch_gemm(dt, h->ar, h->stream);
    }
    for (size_t c0 = 0; c0 < upd.size(); c0 += h->max_jobs) {
      if (h->npd_seen) break;
      const size_t c1 = std::min(upd.size(), c0 + h->max_jobs);
      std::vector<Job> jobs;
      std::vector<GemmProb> gx, gy, gm, gm2;
      std::vector<CopyProb> cm;
      std::vector<SumsqProb> sq;
      // factored-path launches
      std::vector<GemmProb> fx, fy, fcore, oa1, ob1, oa2, ob2;
      std::vector<CopyProb> fcp, fr, fz, facc;
      std::vector<ColNormProb> fcn;
      std::vector<BqrProb> fq;
      std::vector<SumsqProb> fsq;
      const size_t nb2s = (size_t)nb * nb;
      // factored (reference-scheme) recompression where the slot layout holds
      // it: stacked factors (mi + mj) K in Y, their V in Q, merged T factors
      // (super-blocks <= 128 columns: <= 128 K + 128^2 each) + the ki x kj
      // product in Om, GEMM scratch and the K x K core factors in F
      // rank of the update's low-rank form L_ik L_jk^T = Y W^T: the product
      // of two low-rank panel tiles keeps kj columns, and one dense (A13)
      // panel tile times a low-rank one keeps the low-rank one's; two dense
      // panel tiles: no low-rank form (-1)
      auto upd_rank = [&](int i, int j) {
        const bool di = h->dn(i, k), dj = h->dn(j, k);
        return di && dj ? -1 : dj ? h->rank[h->tid(i, k)] : h->rank[h->tid(j, k)];
      };
      auto use_factored = [&](int i, int j) {
        const int ku = upd_rank(i, j);
        if (ku < 0 || h->dn(i, j)) return false;
        const int ki = h->rank[h->tid(i, k)], kj = h->rank[h->tid(j, k)], kij = h->rank[h->tid(i, j)];
        const int mi = h->sz[i], mj = h->sz[j], K = kij + ku;
        const bool fits = (size_t)(mi + mj) * K <= nb2s && 2 * (size_t)K * K <= nb2s &&
                          (size_t)4 * 128 * K <= nb2s &&
                          2 * ((size_t)128 * K + 16384) + (size_t)ki * kj <= nb2s;
        // under a storage cap both stacked parts are within the dense limit,
        // so K <= 2 limit; a result above the limit is stored exactly after
        // the recompression (densify below)
        return fits && K <= factored_frac(nb) * std::min(mi, mj) &&
               (factored_over_limit() || K <= dense_rank_limit(h, mi, mj));
      };
      // dense-path jobs first (slots 0..nd-1), factored ones after them
      std::vector<size_t> order;
      std::vector<char> isf(c1 - c0);
      for (size_t q = c0; q < c1; ++q) isf[q - c0] = use_factored(upd[q].first, upd[q].second);
      for (size_t q = c0; q < c1; ++q) if (!isf[q - c0]) order.push_back(q);
      const int nd = (int)order.size();
      for (size_t q = c0; q < c1; ++q) if (isf[q - c0]) order.push_back(q);
      std::vector<int> posq(c1 - c0);
      for (size_t pos = 0; pos < order.size(); ++pos) {
        const size_t q = order[pos];
        posq[q - c0] = (int)pos;
        const int i = upd[q].first, j = upd[q].second;
        const int ki = h->rank[h->tid(i, k)], kj = h->rank[h->tid(j, k)], kij = h->rank[h->tid(i, j)];
        const bool di = h->dn(i, k), dj = h->dn(j, k), dij = h->dn(i, j);
        const int mi = h->sz[i], mj = h->sz[j], mk = h->sz[k];
        Job J{};
        const int slot = (int)pos;
        bind_slot(h, J, slot);
        if (isf[q - c0]) {
          // stacked factors Us = [U_ij, -Y] (mi x K), Vs = [V_ij, W] (mj x K), L_ik L_jk^T = Y W^T:
          //   both panel tiles low-rank: Y = U_ik (V_ik^T V_jk), W = U_jk
          //   L_jk dense (stored L_jk^T): Y = U_ik,            W = L_jk V_ik
          //   L_ik dense (stored L_ik^T): Y = L_ik V_jk,       W = U_jk
          const int ku = upd_rank(i, j);
          const int K = kij + ku;
          double* Us = J.Y;
          double* Vs = J.Y + (size_t)mi * K;
          // blocked Householder QRs of the stacked factors: V in the Q slot,
          // merged T factors in Om, GEMM scratch in F (free until the core
          // factors land there; consumed again before the Q application)
          double* Vu = J.Q;
          double* Vv = J.Q + (size_t)mi * K;
          const size_t TB = (size_t)128 * K + 16384;   // ceil(K/SB) SB^2, SB <= 128
          double* Tu = J.Om;
          double* Tv = Tu + TB;
          double* Xs = Tv + TB;   // ki x kj
          double* Wu = J.F;
          double* Wv = J.F + nb2s / 2;
          double* uc = J.F;
          double* vc = J.F + (size_t)K * K;
          fcp.push_back({h->Ut(i, j), nb, Us, mi, mi, kij, 0, 1.0, 0, nullptr});
          fcp.push_back({h->Vt(i, j), nb, Vs, mj, mj, kij, 0, 1.0, 0, nullptr});
          if (!di && !dj) {
            fx.push_back({h->Vt(i, k), h->Vt(j, k), nullptr, Xs, ki, kj, mk, nb, nb, ki, ki, 1, 0, 0, 1.0, 0.0});
            fy.push_back({h->Ut(i, k), Xs, nullptr, Us + (size_t)mi * kij, mi, kj, ki, nb, ki, mi, mi, 0, 0, 0, -1.0, 0.0});
            fcp.push_back({h->Ut(j, k), nb, Vs + (size_t)mj * kij, mj, mj, kj, 0, 1.0, 0, nullptr});
          } else if (dj) {
            fcp.push_back({h->Ut(i, k), nb, Us + (size_t)mi * kij, mi, mi, ki, 0, -1.0, 0, nullptr});
            fy.push_back({h->Ut(j, k), h->Vt(i, k), nullptr, Vs + (size_t)mj * kij, mj, ki, mk, nb, nb, mj, mj, 1, 0, 0, 1.0, 0.0});
          } else {
            fy.push_back({h->Ut(i, k), h->Vt(j, k), nullptr, Us + (size_t)mi * kij, mi, kj, mk, nb, nb, mi, mi, 1, 0, 0, -1.0, 0.0});
            fcp.push_back({h->Ut(j, k), nb, Vs + (size_t)mj * kij, mj, mj, kj, 0, 1.0, 0, nullptr});
          }
          double* S = h->d_sums + 6 * slot;
          fsq.push_back({Us, mi, mi, K, S + 2});
          fsq.push_back({nullptr, 0, 0, 0, S + 3});
          fsq.push_back({Vs, mj, mj, K, S + 4});
          fsq.push_back({nullptr, 0, 0, 0, S + 5});
          // U side: Householder QR of all K stacked columns, R^T (lower) into E
          fq.push_back({Us, mi, mi, K, Vu, Tu, Wu});
          fr.push_back({Us, mi, J.E, K, K, K, 1, 1.0, 1, nullptr});
          if (factored_ortho() && kij > 0) {
            // V side: the kept factor V_ij is orthonormal to roundoff (the
            // normalised Jacobi columns of the previous SVD, or Q times
            // them), so the QR of the stacked factor is
            //   [V1, W] = [V1, Q2] [[I, V1^T W], [0, R2]],  Q2 R2 = (I - V1 V1^T) W,
            // with the projection done twice by GEMMs (CGS2) and only the ku
            // update columns refactored by Householder panels.  (The U side
            // cannot take the shortcut: U_ij = M V_k carries the QRCP
            // residual, 1e-2 acc ||M||, so its smallest columns are
            // orthogonal to 1e-2 only; treating them as orthogonal moved
            // the C4p TLR(1e-9) likelihood by 2e-7, cond 4e8.)
            double* Wp = Vs + (size_t)mj * kij;
            double* C2v = Vv + (size_t)mj * ku;   // ku x kij
            double* C1v = J.Bt + kij;             // block (kij.., 0..kij) of Rv^T, ld K
            fz.push_back({nullptr, 0, J.Bt, K, K, K, 0, 1.0, 0, nullptr});
            fcn.push_back({nullptr, 0, 0, kij, J.Bt, K});
            oa1.push_back({Wp, Vs, nullptr, C1v, ku, kij, mj, mj, mj, 0, K, 1, 0, 0, 1.0, 0.0});
            ob1.push_back({Vs, C1v, Wp, Wp, mj, ku, kij, mj, K, mj, mj, 0, 1, 0, -1.0, 1.0});
            oa2.push_back({Wp, Vs, nullptr, C2v, ku, kij, mj, mj, mj, 0, ku, 1, 0, 0, 1.0, 0.0});
            ob2.push_back({Vs, C2v, Wp, Wp, mj, ku, kij, mj, ku, mj, mj, 0, 1, 0, -1.0, 1.0});
            facc.push_back({C2v, ku, C1v, K, ku, kij, 0, 1.0, 2, nullptr});
            fq.push_back({Wp, mj, mj, ku, Vv, Tv, Wv});
            fr.push_back({Wp, mj, J.Bt + (size_t)kij * K + kij, K, ku, ku, 1, 1.0, 1, nullptr});
            J.k1 = kij;
            J.Q1v = Vs;
          } else {
            fq.push_back({Vs, mj, mj, K, Vv, Tv, Wv});
            fr.push_back({Vs, mj, J.Bt, K, K, K, 1, 1.0, 1, nullptr});
          }
          fcore.push_back({J.E, J.Bt, nullptr, J.M, K, K, K, K, K, K, K, 1, 0, 0, 1.0, 0.0});
          J.m = J.n = K;
          J.kind = 2;
          J.s = K;
          J.Uout = uc;
          J.Vout = vc;
          J.ldu = J.ldv = K;
          J.factored = true;
          J.qu = fq[fq.size() - 2];
          J.qv = fq.back();
          J.mu = mi; J.nv = mj;
          J.ftile = (long)h->tid(i, j);
          J.seed = 0;
          jobs.push_back(J);
          continue;
        }
        J.m = mi;
        J.n = mj;
        J.kind = 2;
        J.s = dij ? mj : rank_hint(std::max(kij, di || dj ? mj : kj), mj);
        J.tile = (long)h->tid(i, j);
        J.seed = (uint64_t)h->tid(i, j) * 7777 + (uint64_t)k * 131 + 5;
        double* X = J.E;
        double* Y = J.Y;
        double* S = h->d_sums + 6 * slot;
        // current tile
        if (dij) {
          cm.push_back({h->Ut(i, j), nb, J.M, mi, mi, mj, 1, 1.0, 0, nullptr});
          sq.push_back({h->Ut(i, j), nb, mj, mi, S + 2});
          sq.push_back({nullptr, 0, std::min(mi, mj), 0, S + 4});
        } else {
          gm.push_back({h->Ut(i, j), h->Vt(i, j), nullptr, J.M, mi, mj, kij, nb, nb, mi, mi, 0, 1, 0, 1.0, 0.0});
          sq.push_back({h->Ut(i, j), nb, mi, kij, S + 2});
          sq.push_back({h->Vt(i, j), nb, mj, kij, S + 4});
        }
        // M -= L_ik L_jk^T  (compression.py:54-81 operands u2 = -L_ik-part, v2 = L_jk-part)
        if (!di && !dj) {
          gx.push_back({h->Vt(i, k), h->Vt(j, k), nullptr, X, ki, kj, mk, nb, nb, ki, ki, 1, 0, 0, 1.0, 0.0});
          gy.push_back({h->Ut(i, k), X, nullptr, Y, mi, kj, ki, nb, ki, mi, mi, 0, 0, 0, 1.0, 0.0});
          gm2.push_back({Y, h->Ut(j, k), J.M, J.M, mi, mj, kj, mi, nb, mi, mi, 0, 1, 0, -1.0, 1.0});
          sq.push_back({Y, mi, mi, kj, S + 3});
          sq.push_back({h->Ut(j, k), nb, mj, kj, S + 5});
        } else if (di && !dj) {
          gy.push_back({h->Ut(i, k), h->Vt(j, k), nullptr, Y, mi, kj, mk, nb, nb, mi, mi, 1, 0, 0, 1.0, 0.0});
          gm2.push_back({Y, h->Ut(j, k), J.M, J.M, mi, mj, kj, mi, nb, mi, mi, 0, 1, 0, -1.0, 1.0});
          sq.push_back({Y, mi, mi, kj, S + 3});
          sq.push_back({h->Ut(j, k), nb, mj, kj, S + 5});
        } else if (!di && dj) {
          gx.push_back({h->Vt(i, k), h->Ut(j, k), nullptr, X, ki, mj, mk, nb, nb, ki, ki, 1, 0, 0, 1.0, 0.0});
          gm2.push_back({h->Ut(i, k), X, J.M, J.M, mi, mj, ki, nb, ki, mi, mi, 0, 0, 0, -1.0, 1.0});
          sq.push_back({h->Ut(i, k), nb, mi, ki, S + 3});
          sq.push_back({h->Ut(j, k), nb, mk, mj, S + 5});
        } else {
          gm2.push_back({h->Ut(i, k), h->Ut(j, k), J.M, J.M, mi, mj, mk, nb, nb, mi, mi, 1, 0, 0, -1.0, 1.0});
          sq.push_back({h->Ut(i, k), nb, mk, mi, S + 3});
          sq.push_back({h->Ut(j, k), nb, mk, mj, S + 5});
        }
        jobs.push_back(J);
      }
      const int nf = (int)jobs.size() - nd;
      const bool two = nd > 0 && nf > 0;
      cudaStream_t fs = two ? h->lane2 : h->stream;   // factored-path prep stream
      if (two) {
        TLRB_CUDA(cudaEventRecord(h->ev_b, h->stream));
        TLRB_CUDA(cudaStreamWaitEvent(h->lane2, h->ev_b, 0));
      }
      launch_gemm(gx, h->ar, h->stream);
      launch_gemm(gy, h->ar, h->stream);
      launch_gemm(gm, h->ar, h->stream);
      launch_copy(cm, h->ar, h->stream);
      launch_gemm(gm2, h->ar, h->stream);
      // noise-floor norms (Y = U2 exists now; the tile's old factors are
      // only overwritten at the end of compress_jobs)
      launch_sumsq(sq, h->ar, h->stream);
      // factored path: stacked factors, two Householder QRs, K x K core; on
      // lane2 beside the dense jobs' QRCP / Jacobi when the batch has both
      launch_gemm(fx, h->ar, fs);
      launch_copy(fcp, h->ar, fs);
      launch_gemm(fy, h->ar, fs);
      launch_sumsq(fsq, h->ar, fs);
      launch_copy(fz, h->ar, fs);       // orthogonal-part shortcut: R^T skeletons,
      launch_colnorm(fcn, h->ar, fs);   // Q1 = U_ij D^-1 in place, D / I on the diagonals,
      launch_gemm(oa1, h->ar, fs);      // two Gram-Schmidt passes of the update columns against Q1
      launch_gemm(ob1, h->ar, fs);
      launch_gemm(oa2, h->ar, fs);
      launch_gemm(ob2, h->ar, fs);
      launch_copy(facc, h->ar, fs);
      launch_qr_blocked(fq, h->ar, fs);
      launch_copy(fr, h->ar, fs);
      launch_gemm(fcore, h->ar, fs);
      if (two) {
        TLRB_CUDA(cudaEventRecord(h->ev_f, h->lane2));
        std::vector<Job> jd(jobs.begin(), jobs.begin() + nd), jf(jobs.begin() + nd, jobs.end());
        compress_jobs(h, jd, acc, 0);
        TLRB_CUDA(cudaStreamWaitEvent(h->stream, h->ev_f, 0));
        compress_jobs(h, jf, acc, nd);
        std::copy(jd.begin(), jd.end(), jobs.begin());
        std::copy(jf.begin(), jf.end(), jobs.begin() + nd);
      } else {
        compress_jobs(h, jobs, acc);
      }
      {   // U_new = Qu u_core, V_new = Qv v_core (compression.py:81)
        std::vector<BqrProb> fp;
        std::vector<double*> fc;
        std::vector<int> fld, fk;
        std::vector<CopyProb> fin;
        std::vector<GemmProb> fq1;   // V_new += V1 v_core[0:k1]
        for (Job& J : jobs) {
          if (!J.factored || !J.out_rank) continue;
          const int kk = J.out_rank;
          h->ensure((size_t)J.ftile, kk);
          J.Ufin = h->uptr[J.ftile];
          J.Vfin = h->vptr[J.ftile];
          // [core factor; 0] (K x kk on top of mu - K zero rows), then Q applied in place
          // (orthogonal-part shortcut on the V side: rows k1.. of the core
          // factor belong to Q2; V1's share is added after the Q application)
          const int q2 = J.n - J.k1;
          fin.push_back({J.Uout, J.ldu, J.Ufin, nb, J.m, kk, 0, 1.0, 0, nullptr});
          fin.push_back({J.Vout + J.k1, J.ldv, J.Vfin, nb, q2, kk, 0, 1.0, 0, nullptr});
          // zero rows below the core factor (batched zero fill: one launch
          // for the whole batch instead of two memsets per job)
          fin.push_back({nullptr, 0, J.Ufin + J.m, nb, J.mu - J.m, kk, 0, 1.0, 0, nullptr});
          fin.push_back({nullptr, 0, J.Vfin + q2, nb, J.nv - q2, kk, 0, 1.0, 0, nullptr});
          if (J.k1) {
            // the Q application below uses the slot's F region (where the core
            // factors live) as scratch: V1's rows of the core factor are
            // saved in the M region first (the core is consumed by now)
            double* sv = J.M;
            fin.push_back({J.Vout, J.ldv, sv, J.k1, J.k1, kk, 0, 1.0, 0, nullptr});
            fq1.push_back({J.Q1v, sv, J.Vfin, J.Vfin, J.nv, kk, J.k1, J.nv, J.k1, nb, nb, 0, 0, 0, 1.0, 1.0});
          }
          fp.push_back(J.qu); fc.push_back(J.Ufin); fld.push_back(nb); fk.push_back(kk);
          fp.push_back(J.qv); fc.push_back(J.Vfin); fld.push_back(nb); fk.push_back(kk);
        }
        launch_copy(fin, h->ar, h->stream);
        const double ta0 = trace_on() ? (h->sync(), now_ms()) : 0.0;
        launch_apply_q_blocked(fp, fc, fld, fk, h->ar, h->stream);
        launch_gemm(fq1, h->ar, h->stream);
        if (trace_on()) {
          h->sync();
          fprintf(stderr, "[tlrb] apply-Q %zu factors %.2f ms\n", fp.size(), now_ms() - ta0);
        }
        // storage rule (dense_frac): a recompressed tile whose rank exceeds
        // the dense limit is kept as the exact product of its new factors,
        // L_ij^T = V_new U_new^T, in a fresh dense slot (the factor slabs
        // stay valid in the bump arena until the GEMM has read them)
        std::vector<GemmProb> dens;
        for (Job& J : jobs) {
          if (!J.factored || J.out_rank <= dense_rank_limit(h, J.mu, J.nv)) continue;
          const double* U = J.Ufin;
          const double* V = J.Vfin;
          h->ensure((size_t)J.ftile, nb, true);
          dens.push_back({V, U, nullptr, h->uptr[J.ftile], J.nv, J.mu, J.out_rank, nb, nb, 0, nb, 0, 1, 0, 1.0, 0.0});
          J.dense_out = true;
        }
        launch_gemm(dens, h->ar, h->stream);
      }
      for (size_t q = c0; q < c1; ++q) {
        const int i = upd[q].first, j = upd[q].second;
        // algorithmic work of the update at the execution ranks:
        // the low-rank form of L_ik L_jk^T (rank ku: the low-rank operand's
        // when one panel tile is stored exactly, none when both are), the
        // QRs of the stacked factors, the SVD of the K x K core and the new
        // factors (compression.py:54-81)
        const bool di = h->dn(i, k), dj = h->dn(j, k);
        const double ki = h->rank[h->tid(i, k)], kj = h->rank[h->tid(j, k)], mk = h->sz[k];
        const double kij = h->dn(i, j) ? h->sz[j] : h->rank[h->tid(i, j)];
        const Job& J = jobs[posq[q - c0]];
        const double kn = J.dense_out ? h->sz[j] : J.out_rank;
        const double nbd = h->sz[i], nbj = h->sz[j], full = std::min(nbd, nbj);
        const double ku = di && dj ? full : dj ? ki : kj;
        const double prod = di && dj ? 2.0 * nbd * nbj * mk
                            : di || dj ? 2.0 * (di ? nbd : nbj) * mk * ku
                                       : 2.0 * mk * ki * kj + 2.0 * nbd * ki * kj;
        const double K = std::min(kij + ku, nbd + nbj), Kh = std::min(K, full);
        h->work.add(prod + 2.0 * (4.0 * nbd * K * Kh - 4.0 / 3.0 * Kh * Kh * Kh) +
                        24.0 * Kh * Kh * Kh + 4.0 * nbd * Kh * kn,
                    8.0 * (nbd + nbj) * (kij + ku + kn) + 8.0 * mk * ((di ? nbd : ki) + (dj ? nbj : kj)));
        h->rank[h->tid(i, j)] = J.dense_out ? 0 : J.out_rank;
        h->dense[h->tid(i, j)] = J.dense_out;
      }
    }
    release_panel(h);
    if (h->npd_seen) break;   // single GPU: a POTRF failed (read with a rank readback)
  }
  sync_ranks(h);   // rank maps / statistics: every rank learns every tile's final rank
  return !check_npd(h);
}

// ------------------------------------------------------------ y = L x
// (sample_measurements, stats.py:115-133: z = L w tile by tile)
void add_tile_times(tlrb_handle* h, int i, int j, const double* x, double* acc, bool transpose,
                    std::vector<GemmProb>& g1, std::vector<GemmProb>& g2);

__global__ void tril_kernel(double* A, int ld, int n) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < n * n; e += gridDim.x * blockDim.x) {
    const int r = e % n, c = e / n;
    if (r < c) A[(size_t)c * ld + r] = 0.0;
  }
}

void apply_factor(tlrb_handle* h, const double* dx, double* dy) {
  const int t = h->t, nb = h->nb;
  if (h->dist()) {   // owned contributions, then one sum all-reduce
    TLRB_CUDA(cudaMemsetAsync(dy, 0, h->n * sizeof(double), h->stream));
    for (int i = 0; i < t; ++i) {
      if (!h->own(i, i)) continue;
      tril_kernel<<<64, 256, 0, h->stream>>>(h->D(i), nb, h->sz[i]);
      post_launch();
    }
    std::vector<GemmProb> g0, g1, g2;
    for (int i = 0; i < t; ++i)
      if (h->own(i, i))
        g0.push_back({h->D(i), dx + h->off[i], dy + h->off[i], dy + h->off[i], h->sz[i], 1, h->sz[i], nb,
                      h->sz[i], h->sz[i], h->sz[i], 0, 0, 0, 1.0, 1.0});
    launch_gemm(g0, h->ar, h->stream);
    for (int j = 0; j < t; ++j) {
      g1.clear(); g2.clear();
      for (int i = j + 1; i < t; ++i)
        if (h->own(i, j)) add_tile_times(h, i, j, dx + h->off[j], dy + h->off[i], false, g1, g2);
      launch_gemm(g1, h->ar, h->stream);
      launch_gemm(g2, h->ar, h->stream);
    }
    h->cw->allreduce_sum(dy, h->n, CType::F64, h->stream);
    return;
  }
  for (int i = 0; i < t; ++i) {   // the diagonal factors' upper parts are stale: clear them
    tril_kernel<<<64, 256, 0, h->stream>>>(h->D(i), nb, h->sz[i]);
    post_launch();
  }
  // y_i = L_ii x_i, then y_i += L_ij x_j column by column (one launch per j,
  // every problem of a launch writes a different y_i)
  std::vector<GemmProb> g0;
  for (int i = 0; i < t; ++i)
    g0.push_back({h->D(i), dx + h->off[i], nullptr, dy + h->off[i], h->sz[i], 1, h->sz[i], nb, h->sz[i],
                  h->sz[i], h->sz[i], 0, 0, 0, 1.0, 0.0});
  launch_gemm(g0, h->ar, h->stream);
  for (int j = 0; j < t; ++j) {
    const double* xj = dx + h->off[j];
    std::vector<GemmProb> g1, g2;
    for (int i = j + 1; i < t; ++i) {
      double* yi = dy + h->off[i];
      if (h->factor_mode == 1 || h->dn(i, j)) {
        g1.push_back({h->Ut(i, j), xj, yi, yi, h->sz[i], 1, h->sz[j], nb, h->sz[j], h->sz[i], h->sz[i], 1, 0, 0,
                      1.0, 1.0});
      } else {
        const int r = h->rank[h->tid(i, j)];
        if (!r) continue;
        double* w = h->d_w + (size_t)i * nb;
        g1.push_back({h->Vt(i, j), xj, nullptr, w, r, 1, h->sz[j], nb, h->sz[j], r, r, 1, 0, 0, 1.0, 0.0});
        g2.push_back({h->Ut(i, j), w, yi, yi, h->sz[i], 1, r, nb, r, h->sz[i], h->sz[i], 0, 0, 0, 1.0, 1.0});
      }
    }
    launch_gemm(g1, h->ar, h->stream);
    launch_gemm(g2, h->ar, h->stream);
  }
}

// ------------------------------------------------ distributed solves (8(e))
// Forward: for each tile column j, the contributions sum_i L_ji y_i
// accumulated by the owners of (j, i) are reduced onto the owner of D_j,
// which solves y_j and broadcasts it; owners of (i, j), i > j, then add
// L_ij y_j into their accumulators.  Every rank ends with the full y.
void add_tile_times(tlrb_handle* h, int i, int j, const double* x, double* acc, bool transpose,
                    std::vector<GemmProb>& g1, std::vector<GemmProb>& g2) {
  const int nb = h->nb;
  // transpose == false: acc_i += L_ij x_j ; true: acc_j += L_ij^T x_i
  if (h->factor_mode == 1 || h->dn(i, j)) {
    if (!transpose)
      g1.push_back({h->Ut(i, j), x, acc, acc, h->sz[i], 1, h->sz[j], nb, h->sz[j], h->sz[i], h->sz[i], 1, 0, 0,
                    1.0, 1.0});
    else
      g1.push_back({h->Ut(i, j), x, acc, acc, h->sz[j], 1, h->sz[i], nb, h->sz[i], h->sz[j], h->sz[j], 0, 0, 0,
                    1.0, 1.0});
    return;
  }
  const int r = h->rank[h->tid(i, j)];
  if (!r) return;
  double* w = h->d_w + (size_t)(transpose ? j : i) * nb;
  if (!transpose) {
    g1.push_back({h->Vt(i, j), x, nullptr, w, r, 1, h->sz[j], nb, h->sz[j], r, r, 1, 0, 0, 1.0, 0.0});
    g2.push_back({h->Ut(i, j), w, acc, acc, h->sz[i], 1, r, nb, r, h->sz[i], h->sz[i], 0, 0, 0, 1.0, 1.0});
  } else {
    g1.push_back({h->Ut(i, j), x, nullptr, w, r, 1, h->sz[i], nb, h->sz[i], r, r, 1, 0, 0, 1.0, 0.0});
    g2.push_back({h->Vt(i, j), w, acc, acc, h->sz[j], 1, r, nb, r, h->sz[j], h->sz[j], 0, 0, 0, 1.0, 1.0});
  }
}

// Forward (linalg.py:166-177): for tile row j, the partial sums
// acc_j = sum_{l<j} L_jl y_l live with the owners of (j, l), i.e. in process
// row j mod P: reduced onto the owner of D_j (member j mod Q), which solves
// y_j; y_j then goes down process column j mod Q, where the owners of (i, j),
// i > j, add L_ij y_j into their accumulators.
// Backward (linalg.py:180-197): the transpose — acc_j = sum_{i>j} L_ij^T x_i
// lives in process column j mod Q (reduced onto member j mod P), and x_j goes
// along process row j mod P to the owners of (j, l), l < j.
// Each rank ends holding the solved tiles of its own diagonal tiles;
// gather_solution assembles the full vector on every rank.
void solve_dist(tlrb_handle* h, bool backward) {
  const int t = h->t, nb = h->nb, P = h->P, Q = h->Q, myp = h->prow(), myq = h->pcol();
  cudaStream_t s = h->stream;
  TLRB_CUDA(cudaMemsetAsync(h->d_acc, 0, h->n * sizeof(double), s));
  for (int q = 0; q < t; ++q) {
    const int j = backward ? t - 1 - q : q;
    double* zj = h->d_z + h->off[j];
    double* aj = h->d_acc + h->off[j];
    if (!backward && myp == j % P) h->crow->reduce_sum(aj, h->sz[j], CType::F64, j % Q, s);
    if (backward && myq == j % Q) h->ccol->reduce_sum(aj, h->sz[j], CType::F64, j % P, s);
    if (h->own(j, j)) {
      axpy_kernel<<<4, 256, 0, s>>>(zj, aj, -1.0, h->sz[j]);
      post_launch();
      launch_trsm({TrsmProb{h->D(j), nb, zj, h->sz[j], h->sz[j], 1}}, backward, h->ar, s);
    }
    if (!backward && myq == j % Q) h->ccol->bcast(zj, h->sz[j], CType::F64, j % P, s);
    if (backward && myp == j % P) h->crow->bcast(zj, h->sz[j], CType::F64, j % Q, s);
    std::vector<GemmProb> g1, g2;
    if (!backward) {
      for (int i = j + 1; i < t; ++i)
        if (h->own(i, j)) add_tile_times(h, i, j, zj, h->d_acc + h->off[i], false, g1, g2);
    } else {
      for (int l = 0; l < j; ++l)
        if (h->own(j, l)) add_tile_times(h, j, l, zj, h->d_acc + h->off[l], true, g1, g2);
    }
    launch_gemm(g1, h->ar, s);
    launch_gemm(g2, h->ar, s);
  }
}

// every rank gets the whole solution: the owners of the diagonal tiles
// contribute their solved tiles, one sum all-reduce of n doubles
void gather_solution(tlrb_handle* h) {
  if (!h->dist()) return;
  cudaStream_t s = h->stream;
  TLRB_CUDA(cudaMemsetAsync(h->d_acc, 0, h->n * sizeof(double), s));
  for (int j = 0; j < h->t; ++j)
    if (h->own(j, j))
      TLRB_CUDA(cudaMemcpyAsync(h->d_acc + h->off[j], h->d_z + h->off[j], h->sz[j] * sizeof(double),
                                cudaMemcpyDeviceToDevice, s));
  h->cw->allreduce_sum(h->d_acc, h->n, CType::F64, s);
  TLRB_CUDA(cudaMemcpyAsync(h->d_z, h->d_acc, h->n * sizeof(double), cudaMemcpyDeviceToDevice, s));
}

// ------------------------------------------------------------------ solves
// Single-GPU triangular solves on q right-hand sides X (n x q, ld ldx),
// tile column by tile column (linalg.py:166-197): TRSM of the diagonal tile
// then one batched GEMM launch (two for low-rank tiles, through the scratch
// W: t * nb x q) for every tile below / left of it.
void forward_solve_multi(tlrb_handle* h, double* X, int ldx, int q, double* W) {
  const int t = h->t, nb = h->nb;
  for (int j = 0; j < t; ++j) {
    double* yj = X + h->off[j];
    launch_trsm({TrsmProb{h->D(j), nb, yj, ldx, h->sz[j], q}}, false, h->ar, h->stream);
    std::vector<GemmProb> g1, g2;
    for (int i = j + 1; i < t; ++i) {
      double* yi = X + h->off[i];
      if (h->factor_mode == 1 || h->dn(i, j)) {  // y_i -= T_ij^T y_j
        g1.push_back({h->Ut(i, j), yj, yi, yi, h->sz[i], q, h->sz[j], nb, ldx, ldx, ldx, 1, 0, 0, -1.0, 1.0});
      } else {
        const int r = h->rank[h->tid(i, j)];
        if (!r) continue;
        double* w = W + (size_t)i * nb * q;
        g1.push_back({h->Vt(i, j), yj, nullptr, w, r, q, h->sz[j], nb, ldx, r, r, 1, 0, 0, 1.0, 0.0});
        g2.push_back({h->Ut(i, j), w, yi, yi, h->sz[i], q, r, nb, r, ldx, ldx, 0, 0, 0, -1.0, 1.0});
      }
    }
    launch_gemm(g1, h->ar, h->stream);
    launch_gemm(g2, h->ar, h->stream);
  }
}

void backward_solve_multi(tlrb_handle* h, double* X, int ldx, int q, double* W) {
  const int t = h->t, nb = h->nb;
  for (int i = t - 1; i >= 0; --i) {
    double* xi = X + h->off[i];
    launch_trsm({TrsmProb{h->D(i), nb, xi, ldx, h->sz[i], q}}, true, h->ar, h->stream);
    std::vector<GemmProb> g1, g2;
    for (int j = 0; j < i; ++j) {
      double* xj = X + h->off[j];
      if (h->factor_mode == 1 || h->dn(i, j)) {  // x_j -= L_ij^T x_i = T_ij x_i
        g1.push_back({h->Ut(i, j), xi, xj, xj, h->sz[j], q, h->sz[i], nb, ldx, ldx, ldx, 0, 0, 0, -1.0, 1.0});
      } else {
        const int r = h->rank[h->tid(i, j)];
        if (!r) continue;
        double* w = W + (size_t)j * nb * q;
        g1.push_back({h->Ut(i, j), xi, nullptr, w, r, q, h->sz[i], nb, ldx, r, r, 1, 0, 0, 1.0, 0.0});
        g2.push_back({h->Vt(i, j), w, xj, xj, h->sz[j], q, r, nb, r, ldx, ldx, 0, 0, 0, -1.0, 1.0});
      }
    }
    launch_gemm(g1, h->ar, h->stream);
    launch_gemm(g2, h->ar, h->stream);
  }
}

void forward_solve(tlrb_handle* h) {
  if (h->dist()) { solve_dist(h, false); gather_solution(h); return; }
  forward_solve_multi(h, h->d_z, (int)h->n, 1, h->d_w);
}

void backward_solve(tlrb_handle* h) {
  if (h->dist()) { solve_dist(h, true); gather_solution(h); return; }
  backward_solve_multi(h, h->d_z, (int)h->n, 1, h->d_w);
}

// -------------------------------------------------------------- one eval
// Host half of the reference's KernelView (geometry.py:106-122): Euclidean
// keeps (x, y); great circle maps (lon, lat) degrees to (lat, lon) radians and
// cos(lat), after the range check of LocationSet.__init__ (geometry.py:86-90).
int kernel_view(const double* xy, int64_t n, double radius, std::vector<double>& a1, std::vector<double>& a2,
                std::vector<double>& a3) {
  if (!(radius >= 0.0) || !std::isfinite(radius)) return TLRB_ERR_ARG;
  a1.resize(n); a2.resize(n); a3.clear();
  if (radius == 0.0) {
    for (int64_t i = 0; i < n; ++i) { a1[i] = xy[2 * i]; a2[i] = xy[2 * i + 1]; }
    return TLRB_OK;
  }
  a3.resize(n);
  const double deg = M_PI / 180.0;   // numpy.radians: x * (pi / 180)
  for (int64_t i = 0; i < n; ++i) {
    const double lon = xy[2 * i], lat = xy[2 * i + 1];
    if (std::fabs(lon) > 180.0 || std::fabs(lat) > 90.0) return TLRB_ERR_ARG;
    a1[i] = lat * deg;
    a2[i] = lon * deg;
    a3[i] = std::cos(a1[i]);
  }
  return TLRB_OK;
}

int validate(double th1, double th2, double th3, double nugget, double acc) {
  const double v[5] = {th1, th2, th3, nugget, acc};
  for (double x : v)
    if (!std::isfinite(x)) return TLRB_ERR_ARG;
  if (th1 <= 0 || th2 <= 0 || th3 <= 0 || th3 > 5.0 || nugget < 0) return TLRB_ERR_ARG;
  if (acc < 0 || acc >= 1) return TLRB_ERR_ARG;
  return TLRB_OK;
}

// factorise Sigma(theta) into the handle; returns TLRB_* code
int factorize(tlrb_handle* h, double th1, double th2, double th3, double nugget, double acc) {
  cudaStream_t s = h->stream;
  h->mp = make_matern(th1, th2, th3);
  h->acc = acc;
  h->work = Flops{};
  h->retries = 0;
  h->max_sweeps = 0;
  h->err_tile = h->err_pivot = -1;
  h->factor_mode = 0;
  TLRB_CUDA(cudaMemsetAsync(h->d_info, 0, 3 * sizeof(int), s));
  TLRB_CUDA(cudaMemsetAsync(h->d_logdiag, 0, h->n * sizeof(double), s));
  TLRB_CUDA(cudaEventRecord(h->ev[0], s));
  const bool dense = acc == 0.0;
  h->sync();   // previous users of the arena are done before it is recycled
  h->arena_reset();
  if (dense)
    for (int i = 1; i < h->t; ++i)
      for (int j = 0; j < i; ++j)
        if (h->own(i, j)) h->ensure(h->tid(i, j), h->nb, true);
  generate(h, nugget, dense);
  TLRB_CUDA(cudaEventRecord(h->ev[1], s));
  std::fill(h->rank.begin(), h->rank.end(), 0);
  std::fill(h->dense.begin(), h->dense.end(), 0);
  if (!dense) compress_all(h, acc);
  TLRB_CUDA(cudaEventRecord(h->ev[2], s));
  const bool ok = dense ? factor_dense(h) : factor_tlr(h, acc);
  TLRB_CUDA(cudaEventRecord(h->ev[3], s));
  if (!ok) return TLRB_ERR_NPD;
  h->factor_mode = dense ? 1 : 2;
  return TLRB_OK;
}

int loglik_impl(tlrb_handle* h, const double* z, bool z_on_device, double th1, double th2,
                double th3, double nugget, double acc, double* ll, double* logdet, double* quad,
                tlrb_stats* st) {
  const int64_t l0 = g_launches;
  int rc = validate(th1, th2, th3, nugget, acc);
  if (rc) {
    h->msg = "invalid theta / nugget / accuracy";
    return rc;
  }
  TLRB_CUDA(cudaSetDevice(h->device));
  cudaStream_t s = h->stream;
  const auto t0 = std::chrono::steady_clock::now();
  TLRB_CUDA(cudaEventRecord(h->ev[5], s));
  TLRB_CUDA(cudaMemcpyAsync(h->d_z, z, h->n * sizeof(double),
                            z_on_device ? cudaMemcpyDefault : cudaMemcpyHostToDevice, s));
  rc = factorize(h, th1, th2, th3, nugget, acc);
  if (rc) return rc;
  forward_solve(h);
  launch_dot(h->d_z, (int)h->n, h->d_scal + 1, s);
  launch_sum_log(h->d_logdiag, (int)h->n, h->d_scal, s);
  if (h->dist())   // log-det: owners of the diagonal tiles hold the partial sums
    h->cw->allreduce_sum(h->d_scal, 1, CType::F64, s);
  TLRB_CUDA(cudaEventRecord(h->ev[4], s));
  double sc[2];
  TLRB_CUDA(cudaMemcpyAsync(sc, h->d_scal, sizeof sc, cudaMemcpyDeviceToHost, s));
  h->sync();
  const double LOG_2PI = std::log(2.0 * M_PI);
  if (ll) *ll = -0.5 * (h->n * LOG_2PI + sc[0] + sc[1]);
  if (logdet) *logdet = sc[0];
  if (quad) *quad = sc[1];
  {
    tlrb_stats S{};
    float a;
    TLRB_CUDA(cudaEventElapsedTime(&a, h->ev[0], h->ev[2])); S.ms_generate = a;
    TLRB_CUDA(cudaEventElapsedTime(&a, h->ev[1], h->ev[2])); S.ms_compress = a;
    TLRB_CUDA(cudaEventElapsedTime(&a, h->ev[2], h->ev[3])); S.ms_factor = a;
    TLRB_CUDA(cudaEventElapsedTime(&a, h->ev[3], h->ev[4])); S.ms_solve = a;
    S.ms_total = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    TLRB_CUDA(cudaEventElapsedTime(&a, h->ev[5], h->ev[4])); S.ms_device = a;
    int64_t reals = 0;
    int mx = 0;
    double sum = 0;
    int cnt = 0;
    for (int i = 0; i < h->t; ++i) {
      reals += (int64_t)h->sz[i] * h->sz[i];
      for (int j = 0; j < i; ++j) {
        if (h->factor_mode == 1 || h->dn(i, j)) { reals += (int64_t)h->sz[i] * h->sz[j]; continue; }
        const int r = h->rank[h->tid(i, j)];
        reals += (int64_t)r * (h->sz[i] + h->sz[j]);
        mx = std::max(mx, r);
        sum += r;
        ++cnt;
      }
    }
    h->work.add(2.0 * reals, 8.0 * reals);
    S.flops = h->work.f;
    S.bytes = h->work.b;
    S.stored_reals = reals;
    S.max_rank = mx;
    S.mean_rank = cnt ? sum / cnt : 0.0;
    S.sketch_retries = h->retries;
    S.jacobi_max_sweeps = h->max_sweeps;
    S.kernel_launches = g_launches - l0;
    S.t_roof_ms = h->work.troof * 1e3;
    S.arena_peak_bytes = (int64_t)h->arena_peak;
    S.panel_peak_bytes = (int64_t)h->panel_peak;
    h->st = S;
    if (st) *st = S;
  }
  return TLRB_OK;
}

template <class F>
int guarded(tlrb_handle* h, F&& f) {
  // calls on one handle take turns (DescArena, workspace, streams); the
  // launcher caches belong to the handle's launch context, so different
  // handles — also several logical ranks on one device — run concurrently
  std::unique_lock<std::recursive_mutex> lk;
  if (h) {
    lk = std::unique_lock<std::recursive_mutex>(h->mu);
    set_thread_ctx(h->ctx);
  }
  try {
    return f();
  } catch (const CudaError& e) {
    if (h) h->msg = e.msg;
    cudaGetLastError();
    return TLRB_ERR_CUDA;
  } catch (const std::exception& e) {
    if (h) h->msg = e.what();
    return TLRB_ERR_CUDA;
  }
}

// Allocate one (member) handle.  rank / P / Q: its place on the 2D
// block-cyclic grid (0 / 1 / 1 single GPU) — only owned tiles get storage.
// share / slot: handles created together on this device and this one's
// index among them: the HBM budgets are split between them.
tlrb_handle* create_one(const double* xy, int64_t n, int nb, int max_rank, int device, int rank, int P, int Q,
                        int share, int slot, int32_t* err) {
  tlrb_handle* h = new tlrb_handle();
  h->device = device;
  const int rc = guarded(h, [&]() -> int {
    TLRB_CUDA(cudaSetDevice(device));
    h->ctx = acquire_ctx();
    set_thread_ctx(h->ctx);
    h->drank = rank;
    h->P = P;
    h->Q = Q;
    h->dworld = P * Q;
    TLRB_CUDA(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    {   // look-ahead POTRF stream: highest priority, so its few CTAs get the
        // SM slots the main stream's large batches free up
      int lo_prio = 0, hi_prio = 0;
      TLRB_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
      TLRB_CUDA(cudaStreamCreateWithPriority(&h->side, cudaStreamNonBlocking, hi_prio));
    }
    TLRB_CUDA(cudaStreamCreateWithFlags(&h->lane2, cudaStreamNonBlocking));
    TLRB_CUDA(cudaEventCreateWithFlags(&h->ev_b, cudaEventDisableTiming));
    TLRB_CUDA(cudaEventCreateWithFlags(&h->ev_f, cudaEventDisableTiming));
    TLRB_CUDA(cudaEventCreateWithFlags(&h->ev_syrk, cudaEventDisableTiming));
    TLRB_CUDA(cudaEventCreateWithFlags(&h->ev_potrf, cudaEventDisableTiming));
    for (auto& e : h->ev) TLRB_CUDA(cudaEventCreate(&e));
    h->n = n;
    h->nb = (int)std::min<int64_t>(nb, n);
    h->t = (int)((n + h->nb - 1) / h->nb);
    h->max_rank = max_rank;
    for (int i = 0; i < h->t; ++i) {
      h->off.push_back(i * h->nb);
      h->sz.push_back((int)std::min<int64_t>(h->nb, n - (int64_t)i * h->nb));
    }
    h->hxy.assign(xy, xy + 2 * n);
    std::vector<double> xs, ys, zs;
    kernel_view(xy, n, 0.0, xs, ys, zs);
    TLRB_CUDA(cudaMalloc(&h->dx, n * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->dy, n * sizeof(double)));
    TLRB_CUDA(cudaMemcpy(h->dx, xs.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    TLRB_CUDA(cudaMemcpy(h->dy, ys.data(), n * sizeof(double), cudaMemcpyHostToDevice));
    const size_t nb2 = (size_t)h->nb * h->nb;
    const size_t ntile = (size_t)h->t * (h->t - 1) / 2;
    auto owns = [&](int i, int j) { return (i % P) * Q + (j % Q) == rank; };
    size_t nd = 0, nlow = 0;
    for (int i = 0; i < h->t; ++i) {
      nd += owns(i, i);
      for (int j = 0; j < i; ++j) nlow += owns(i, j);
    }
    TLRB_CUDA(cudaMalloc(&h->diag, std::max<size_t>(1, nd * nb2) * sizeof(double)));
    h->dptr.assign(h->t, nullptr);
    for (int i = 0, q = 0; i < h->t; ++i)
      if (owns(i, i)) h->dptr[i] = h->diag + (size_t)(q++) * nb2;
    if (P * Q > 1) TLRB_CUDA(cudaMalloc(&h->lkk, nb2 * sizeof(double)));
    h->uptr.assign(ntile, nullptr);
    h->vptr.assign(ntile, nullptr);
    h->tcap.assign(ntile, 0);
    h->rank.assign(ntile, 0);
    h->dense.assign(ntile, 0);
    TLRB_CUDA(cudaMalloc(&h->d_info, 4 * sizeof(int)));
    TLRB_CUDA(cudaMemset(h->d_info, 0, 4 * sizeof(int)));   // no POTRF failure yet
    TLRB_CUDA(cudaMalloc(&h->d_logdiag, n * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_scal, 4 * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_z, n * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_w, (size_t)h->t * h->nb * sizeof(double)));
    {   // launch-descriptor staging ring (TLRB_DESC_MB: smaller rings force the
        // wrap path, tests/test_gpu_parity.py::test_descriptor_arena_wraps)
      const int mb = getenv("TLRB_DESC_MB") ? std::max(1, atoi(getenv("TLRB_DESC_MB"))) : 64;
      h->ar.init((size_t)mb << 20);
    }
    // compression workspace: 8 nb^2 + 2 nb + 16 nb doubles per job slot
    h->slot_doubles = 8 * nb2 + 18 * (size_t)h->nb + 64;
    size_t freeb = 0, totb = 0;
    TLRB_CUDA(cudaMemGetInfo(&freeb, &totb));
    // capped at 56 GB for tile grids up to 128 x 128 (fewer, larger job
    // batches: C3 16.3 s vs 17.2 s at 24 GB) and at 24 GB beyond, where the
    // rank-adaptive factor arena needs the rest of HBM (C4, C5); TLRB_WS_GB
    // overrides.  Handles created together on one device split the budget.
    const size_t cap_gb = getenv("TLRB_WS_GB") ? (size_t)atoll(getenv("TLRB_WS_GB")) : (h->t <= 128 ? 56 : 24);
    const int left = std::max(1, share - slot);   // handles of this group still to size on the device
    size_t budget = std::min<size_t>(freeb / 3 / left, (cap_gb << 30) / std::max(1, share));
    const size_t owned_jobs = std::max<size_t>(nlow, 1);
    int jobs = (int)std::max<size_t>(1, budget / (h->slot_doubles * 8));
    jobs = (int)std::min<size_t>(jobs, owned_jobs);
    h->max_jobs = std::min(jobs, 8192);
    h->ws_bytes = std::max((size_t)h->max_jobs * h->slot_doubles * 8, nb2 * 8 * 4);
    TLRB_CUDA(cudaMalloc(&h->ws, h->ws_bytes));
    TLRB_CUDA(cudaMalloc(&h->d_sums, 6 * (size_t)h->max_jobs * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_aux, 3 * (size_t)h->max_jobs * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_kind, (size_t)h->max_jobs * sizeof(int)));
    TLRB_CUDA(cudaMalloc(&h->d_ok, (size_t)h->max_jobs * sizeof(int)));
    TLRB_CUDA(cudaMalloc(&h->d_rank, (size_t)h->max_jobs * sizeof(int)));
    TLRB_CUDA(cudaMalloc(&h->d_sweeps, (size_t)h->max_jobs * sizeof(int)));
    TLRB_CUDA(cudaMalloc(&h->d_perm, (size_t)h->max_jobs * h->nb * sizeof(int)));
    {
      // the factor arena holds this rank's own tiles only (received panel
      // tiles live in pbuf): at most all of them dense, twice (a tile whose
      // rank grows gets a fresh slot), within 85% of what is left
      size_t fb = 0, tb = 0;
      TLRB_CUDA(cudaMemGetInfo(&fb, &tb));
      const size_t full = std::max<size_t>(1, nlow) * 2 * nb2 * sizeof(double) + (1 << 20);
      const size_t avail = (size_t)(0.85 * (double)fb / left);
      h->arena_bytes = std::min(full, avail);
      TLRB_CUDA(cudaMalloc(&h->arena, h->arena_bytes));
    }
    return TLRB_OK;
  });
  if (rc != TLRB_OK) {
    if (err) *err = rc;
    fprintf(stderr, "tlrb_create: %s\n", h->msg.c_str());
    tlrb_destroy(h);
    return nullptr;
  }
  return h;
}

// distributed scratch, once the communicators are attached
int attach_dist(tlrb_handle* h) {
  return guarded(h, [&]() -> int {
    TLRB_CUDA(cudaSetDevice(h->device));
    TLRB_CUDA(cudaMalloc(&h->d_ibuf, (2 * h->rank.size() + 3 * (size_t)h->dworld + 8) * sizeof(int)));
    TLRB_CUDA(cudaMalloc(&h->d_acc, h->n * sizeof(double)));
    return TLRB_OK;
  });
}

// Run fn(member, index) for every member of a group handle, one host thread
// each (the members' collectives rendezvous with one another).  A CUDA
// failure on one member aborts the loopback communicators so that the others
// leave their collectives instead of waiting forever.
template <class F>
int run_members(tlrb_handle* g, F&& fn) {
  const int W = (int)g->members.size();
  std::vector<int> rc(W, TLRB_OK);
  std::vector<std::thread> th;
  for (int r = 0; r < W; ++r)
    th.emplace_back([&, r] {
      tlrb_handle* m = g->members[r];
      rc[r] = guarded(m, [&]() -> int {
        TLRB_CUDA(cudaSetDevice(m->device));
        return fn(m, r);
      });
      if (rc[r] == TLRB_ERR_CUDA)
        for (tlrb_handle* o : g->members)
          for (Comm* c : {o->cw.get(), o->crow.get(), o->ccol.get()})
            if (c && !strcmp(c->kind(), "loopback")) c->abort();
    });
  for (auto& x : th) x.join();
  int out = TLRB_OK;
  for (int r = 0; r < W && out == TLRB_OK; ++r)
    if (rc[r] != TLRB_OK) {
      out = rc[r];
      g->msg = g->members[r]->msg;
      g->err_tile = g->members[r]->err_tile;
      g->err_pivot = g->members[r]->err_pivot;
    }
  // a genuine failure (not an NPD, which every member reports) wins
  for (int r = 0; r < W; ++r)
    if (rc[r] == TLRB_ERR_CUDA) {
      out = rc[r];
      g->msg = g->members[r]->msg;
      break;
    }
  return out;
}

void grid_shape(int world, int& P, int& Q) {
  // P x Q with P <= Q, as square as possible (1x1, 1x2, 2x2, 2x4, ...)
  P = 1;
  for (int p = 1; p * p <= world; ++p)
    if (world % p == 0) P = p;
  Q = world / P;
}

tlrb_handle* create_group(const double* xy, int64_t n, int32_t nb, int32_t max_rank, const int32_t* devices,
                          int32_t world, int32_t P, int32_t Q, int32_t backend, int32_t* err) {
  if (err) *err = TLRB_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess) ndev = 0;
  cudaGetLastError();
  bool distinct = true;
  for (int r = 0; r < world; ++r) {
    if (devices[r] < 0 || devices[r] >= ndev) {
      if (err) *err = TLRB_ERR_ARG;
      return nullptr;
    }
    for (int q = 0; q < r; ++q) distinct &= devices[q] != devices[r];
  }
  if (backend == TLRB_BACKEND_AUTO) backend = distinct ? TLRB_BACKEND_NCCL : TLRB_BACKEND_LOOPBACK;
  if (backend == TLRB_BACKEND_NCCL && !distinct) {   // NCCL takes one rank per device
    if (err) *err = TLRB_ERR_ARG;
    return nullptr;
  }
  tlrb_handle* g = new tlrb_handle();
  g->device = devices[0];
  g->dworld = world;
  g->P = P;
  g->Q = Q;
  g->n = n;
  g->nb = (int)std::min<int64_t>(nb, n);
  g->t = (int)((n + g->nb - 1) / g->nb);
  std::vector<int> share(world), slot(world);
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q)
      if (devices[q] == devices[r]) {
        ++share[r];
        if (q < r) ++slot[r];
      }
  for (int r = 0; r < world; ++r) {
    tlrb_handle* m = create_one(xy, n, nb, max_rank, devices[r], r, P, Q, share[r], slot[r], err);
    if (!m) {
      tlrb_destroy(g);
      return nullptr;
    }
    g->members.push_back(m);
  }
  int rc = TLRB_OK;
  try {
    if (backend == TLRB_BACKEND_LOOPBACK) {
      auto wg = make_local_group(world);
      std::vector<std::shared_ptr<LocalGroup>> rows, cols;
      for (int p = 0; p < P; ++p) rows.push_back(make_local_group(Q));
      for (int q = 0; q < Q; ++q) cols.push_back(make_local_group(P));
      for (int r = 0; r < world; ++r) {
        tlrb_handle* m = g->members[r];
        TLRB_CUDA(cudaSetDevice(m->device));
        m->cw = make_local_comm(wg, r, m->device);
        m->crow = make_local_comm(rows[r / Q], r % Q, m->device);
        m->ccol = make_local_comm(cols[r % Q], r / Q, m->device);
      }
    } else {
      std::vector<ncclComm_t> comms(world);
      TLRB_NCCL(ncclCommInitAll(comms.data(), world, devices));
      for (int r = 0; r < world; ++r) g->members[r]->cw = make_nccl_comm(comms[r]);
      // row / column communicators: ncclCommSplit is collective over the
      // world members, one host thread each
      rc = run_members(g, [&](tlrb_handle* m, int r) -> int {
        m->crow = split_nccl_comm(*m->cw, r / Q, r % Q);
        m->ccol = split_nccl_comm(*m->cw, Q + r % Q, r / Q);
        return TLRB_OK;
      });
    }
  } catch (const CudaError& e) {
    g->msg = e.msg;
    rc = TLRB_ERR_CUDA;
  }
  for (int r = 0; r < world && rc == TLRB_OK; ++r) rc = attach_dist(g->members[r]);
  if (rc != TLRB_OK) {
    if (err) *err = rc;
    fprintf(stderr, "tlrb_create_group: %s\n", g->msg.c_str());
    tlrb_destroy(g);
    return nullptr;
  }
  return g;
}

// the group's statistics: member 0's, with the slowest member's device time
// and the largest per-member memory high-water marks
void group_stats(tlrb_handle* g, std::vector<tlrb_stats>& ms, tlrb_stats* st) {
  if (!st) return;
  tlrb_stats S = ms[0];
  for (const tlrb_stats& m : ms) {
    S.ms_device = std::max(S.ms_device, m.ms_device);
    S.ms_total = std::max(S.ms_total, m.ms_total);
    S.arena_peak_bytes = std::max(S.arena_peak_bytes, m.arena_peak_bytes);
    S.panel_peak_bytes = std::max(S.panel_peak_bytes, m.panel_peak_bytes);
  }
  S.kernel_launches = 0;
  for (const tlrb_stats& m : ms) S.kernel_launches += m.kernel_launches;
  *st = S;
}

int loglik_any(tlrb_handle* h, const double* z, bool on_dev, double th1, double th2, double th3, double nugget,
               double acc, double* ll, double* logdet, double* quad, tlrb_stats* st) {
  if (!h->group())
    return guarded(h, [&] { return loglik_impl(h, z, on_dev, th1, th2, th3, nugget, acc, ll, logdet, quad, st); });
  std::vector<tlrb_stats> ms(h->members.size());
  std::vector<double> out(3 * h->members.size());
  const int rc = run_members(h, [&](tlrb_handle* m, int r) {
    return loglik_impl(m, z, on_dev, th1, th2, th3, nugget, acc, &out[3 * r], &out[3 * r + 1], &out[3 * r + 2],
                       &ms[r]);
  });
  if (rc) return rc;
  if (ll) *ll = out[0];
  if (logdet) *logdet = out[1];
  if (quad) *quad = out[2];
  group_stats(h, ms, st);
  return TLRB_OK;
}

int factorize_one(tlrb_handle* h, double th1, double th2, double th3, double nugget, double acc) {
  TLRB_CUDA(cudaSetDevice(h->device));
  const int r = factorize(h, th1, th2, th3, nugget, acc);
  h->sync();
  return r;
}

int apply_factor_one(tlrb_handle* h, const double* x, double* y) {
  if (!h->factor_mode) {
    h->msg = "no factor available";
    return TLRB_ERR_ARG;
  }
  TLRB_CUDA(cudaSetDevice(h->device));
  if (!h->d_y) TLRB_CUDA(cudaMalloc(&h->d_y, h->n * sizeof(double)));
  TLRB_CUDA(cudaMemcpyAsync(h->d_z, x, h->n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  apply_factor(h, h->d_z, h->d_y);
  if (y) TLRB_CUDA(cudaMemcpyAsync(y, h->d_y, h->n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  h->sync();
  return TLRB_OK;
}

int solve_one(tlrb_handle* h, const double* rhs, double* x) {
  if (!h->factor_mode) {
    h->msg = "no factor available";
    return TLRB_ERR_ARG;
  }
  TLRB_CUDA(cudaSetDevice(h->device));
  TLRB_CUDA(cudaMemcpyAsync(h->d_z, rhs, h->n * sizeof(double), cudaMemcpyHostToDevice, h->stream));
  forward_solve(h);
  backward_solve(h);
  if (x) TLRB_CUDA(cudaMemcpyAsync(x, h->d_z, h->n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  h->sync();
  return TLRB_OK;
}

int predict_one(tlrb_handle* h, const double* z, const double* xy_unknown, int64_t m, double th1, double th2,
                double th3, double nugget, double acc, double* pred) {
  TLRB_CUDA(cudaSetDevice(h->device));
  cudaStream_t s = h->stream;
  if (m > h->ucap) {
    if (h->d_ux) {
      cudaFree(h->d_ux); cudaFree(h->d_uy); cudaFree(h->d_uz); cudaFree(h->d_pred); cudaFree(h->d_partial);
      cudaFree(h->d_pacc);
    }
    h->ucap = m;
    const int64_t nchunk = (h->n + 2047) / 2048;
    TLRB_CUDA(cudaMalloc(&h->d_ux, m * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_uy, m * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_uz, m * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_pred, m * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_pacc, m * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&h->d_partial, m * nchunk * sizeof(double)));
  }
  std::vector<double> ux, uy, uz;
  if (kernel_view(xy_unknown, m, 0.5 * h->diam, ux, uy, uz)) return TLRB_ERR_ARG;
  TLRB_CUDA(cudaMemcpyAsync(h->d_ux, ux.data(), m * sizeof(double), cudaMemcpyHostToDevice, s));
  TLRB_CUDA(cudaMemcpyAsync(h->d_uy, uy.data(), m * sizeof(double), cudaMemcpyHostToDevice, s));
  if (h->diam > 0.0)
    TLRB_CUDA(cudaMemcpyAsync(h->d_uz, uz.data(), m * sizeof(double), cudaMemcpyHostToDevice, s));
  TLRB_CUDA(cudaMemcpyAsync(h->d_z, z, h->n * sizeof(double), cudaMemcpyHostToDevice, s));
  int r = factorize(h, th1, th2, th3, nugget, acc);
  if (r) return r;
  forward_solve(h);
  backward_solve(h);
  const Pts unk{h->d_ux, h->d_uy, h->d_uz, h->diam};
  if (h->dist()) {
    // SURVEY 8(e) kriging: each rank generates the cross-covariance columns
    // of its own diagonal tiles' sites and multiplies them with its solved
    // tiles; one all-reduce of the m-vector
    TLRB_CUDA(cudaMemsetAsync(h->d_pred, 0, m * sizeof(double), s));
    for (int j = 0; j < h->t; ++j) {
      if (!h->own(j, j)) continue;
      const int64_t o = h->off[j];
      const Pts kp{h->dx + o, h->dy + o, h->dz ? h->dz + o : nullptr, h->diam};
      launch_cross_gemv(kp, h->d_z + o, h->sz[j], unk, m, h->mp, h->d_partial, h->d_pacc, s);
      axpy_kernel<<<4, 256, 0, s>>>(h->d_pred, h->d_pacc, 1.0, (int)m);
      post_launch();
    }
    h->cw->allreduce_sum(h->d_pred, m, CType::F64, s);
  } else {
    launch_cross_gemv(h->pts(), h->d_z, h->n, unk, m, h->mp, h->d_partial, h->d_pred, s);
  }
  if (pred) TLRB_CUDA(cudaMemcpyAsync(pred, h->d_pred, m * sizeof(double), cudaMemcpyDeviceToHost, s));
  h->sync();
  return TLRB_OK;
}

// conditional covariance S11 - S12 S22^-1 S21 of the unknown sites on the
// factor just computed (predict.py:81-87), all on the device: S21 generated
// from [known; unknown] points, q = m right-hand-side solves, one GEMM
int kriging_cov(tlrb_handle* h, int64_t m, double nugget, double* cov) {
  cudaStream_t s = h->stream;
  const int64_t n = h->n, nt = n + m;
  double *cx = nullptr, *cy = nullptr, *cz = nullptr, *S = nullptr, *W = nullptr, *C = nullptr;
  auto cat = [&](double*& dst, const double* a, const double* b) {
    TLRB_CUDA(cudaMalloc(&dst, nt * sizeof(double)));
    TLRB_CUDA(cudaMemcpyAsync(dst, a, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    TLRB_CUDA(cudaMemcpyAsync(dst + n, b, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
  };
  cat(cx, h->dx, h->d_ux);
  cat(cy, h->dy, h->d_uy);
  if (h->diam > 0.0) cat(cz, h->dz, h->d_uz);
  TLRB_CUDA(cudaMalloc(&S, (size_t)n * m * sizeof(double)));
  TLRB_CUDA(cudaMalloc(&W, (size_t)h->t * h->nb * m * sizeof(double)));
  TLRB_CUDA(cudaMalloc(&C, (size_t)m * m * sizeof(double)));
  const Pts all{cx, cy, cz, h->diam};
  // S21 (n x m): rows = known sites, columns = unknown sites (disjoint index
  // ranges: no diagonal term); S11 (m x m) with the nugget on its diagonal
  launch_gen_tiles({GenTile{S, (int)n, 0, (int)n, (int)n, (int)m, 0.0},
                    GenTile{C, (int)m, (int)n, (int)m, (int)n, (int)m, nugget}},
                   all, h->mp, h->ar, s);
  forward_solve_multi(h, S, (int)n, (int)m, W);
  backward_solve_multi(h, S, (int)n, (int)m, W);   // S <- S22^-1 S21
  // C = S11 - S21^T (S22^-1 S21): generate a fresh S21 into W for the left factor
  launch_gen_tiles({GenTile{W, (int)n, 0, (int)n, (int)n, (int)m, 0.0}}, all, h->mp, h->ar, s);
  launch_gemm({GemmProb{W, S, C, C, (int)m, (int)m, (int)n, (int)n, (int)n, (int)m, (int)m, 1, 0, 0, -1.0, 1.0}},
              h->ar, s);
  TLRB_CUDA(cudaMemcpyAsync(cov, C, (size_t)m * m * sizeof(double), cudaMemcpyDeviceToHost, s));
  h->sync();
  for (double* p : {cx, cy, cz, S, W, C})
    if (p) cudaFree(p);
  return TLRB_OK;
}

int set_metric_one(tlrb_handle* h, const std::vector<double>& a1, const std::vector<double>& a2,
                   const std::vector<double>& a3, double sphere_radius) {
  TLRB_CUDA(cudaSetDevice(h->device));
  TLRB_CUDA(cudaStreamSynchronize(h->stream));
  TLRB_CUDA(cudaMemcpy(h->dx, a1.data(), h->n * sizeof(double), cudaMemcpyHostToDevice));
  TLRB_CUDA(cudaMemcpy(h->dy, a2.data(), h->n * sizeof(double), cudaMemcpyHostToDevice));
  if (!a3.empty()) {
    if (!h->dz) TLRB_CUDA(cudaMalloc(&h->dz, h->n * sizeof(double)));
    TLRB_CUDA(cudaMemcpy(h->dz, a3.data(), h->n * sizeof(double), cudaMemcpyHostToDevice));
  }
  h->diam = 2.0 * sphere_radius;
  return TLRB_OK;
}

}  // namespace

// =================================================================== C ABI
extern "C" {

tlrb_handle* tlrb_create(const double* xy, int64_t n, int32_t nb, int32_t ngpus, int32_t max_rank,
                         int32_t device, int32_t* err) {
  if (err) *err = TLRB_OK;
  // the compression kernels stage at most 2048 rows per column (QRCP / Jacobi
  // register tiles of 64 doubles per lane): larger tiles are refused
  if (!xy || n < 1 || nb < 1 || ngpus < 1 || ngpus > kMaxDevices || device < 0 ||
      std::min<int64_t>(nb, n) > kMaxTile) {
    if (err) *err = TLRB_ERR_ARG;
    return nullptr;
  }
  if (ngpus == 1) return create_one(xy, n, nb, max_rank, device, 0, 1, 1, 1, 0, err);
  // one process driving devices device .. device + ngpus - 1 (NCCL over
  // NVLink between them, one host thread per device inside each call)
  std::vector<int32_t> devs(ngpus);
  for (int r = 0; r < ngpus; ++r) devs[r] = device + r;
  int P = 1, Q = 1;
  grid_shape(ngpus, P, Q);
  return create_group(xy, n, nb, max_rank, devs.data(), ngpus, P, Q, TLRB_BACKEND_AUTO, err);
}

tlrb_handle* tlrb_create_group(const double* xy, int64_t n, int32_t nb, int32_t max_rank,
                               const int32_t* devices, int32_t world, int32_t P, int32_t Q, int32_t backend,
                               int32_t* err) {
  if (err) *err = TLRB_OK;
  if (!xy || !devices || n < 1 || nb < 1 || world < 1 || world > 64 || P < 1 || Q < 1 || P * Q != world ||
      backend < TLRB_BACKEND_AUTO || backend > TLRB_BACKEND_LOOPBACK || std::min<int64_t>(nb, n) > kMaxTile) {
    if (err) *err = TLRB_ERR_ARG;
    return nullptr;
  }
  return create_group(xy, n, nb, max_rank, devices, world, P, Q, backend, err);
}

int32_t tlrb_nccl_unique_id(char* out, int32_t len) {
  if (!out || len < (int32_t)sizeof(ncclUniqueId)) return TLRB_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return TLRB_ERR_CUDA;
  memcpy(out, &id, sizeof id);
  return TLRB_OK;
}

tlrb_handle* tlrb_create_dist(const double* xy, int64_t n, int32_t nb, int32_t max_rank, int32_t device,
                              int32_t rank, int32_t world, int32_t P, int32_t Q, const char* nccl_id,
                              int32_t* err) {
  if (err) *err = TLRB_OK;
  if (!xy || !nccl_id || n < 1 || nb < 1 || world < 1 || rank < 0 || rank >= world || P < 1 || Q < 1 ||
      P * Q != world || std::min<int64_t>(nb, n) > kMaxTile) {
    if (err) *err = TLRB_ERR_ARG;
    return nullptr;
  }
  tlrb_handle* h = create_one(xy, n, nb, max_rank, device, rank, P, Q, 1, 0, err);
  if (!h) return nullptr;
  int rc = guarded(h, [&]() -> int {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof id);
    ncclComm_t c = nullptr;
    TLRB_NCCL(ncclCommInitRank(&c, world, id, rank));
    h->cw = make_nccl_comm(c);
    h->crow = split_nccl_comm(*h->cw, rank / Q, rank % Q);
    h->ccol = split_nccl_comm(*h->cw, Q + rank % Q, rank / Q);
    return TLRB_OK;
  });
  if (rc == TLRB_OK) rc = attach_dist(h);
  if (rc != TLRB_OK) {
    if (err) *err = rc;
    fprintf(stderr, "tlrb_create_dist: %s\n", h->msg.c_str());
    tlrb_destroy(h);
    return nullptr;
  }
  return h;
}

void tlrb_destroy(tlrb_handle* h) {
  if (!h) return;
  for (tlrb_handle* m : h->members) tlrb_destroy(m);
  h->members.clear();
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  h->cw.reset();
  h->crow.reset();
  h->ccol.reset();
  void* ptrs[] = {h->dx, h->dy, h->dz, h->d_uz, h->diag, h->arena, h->d_info, h->d_logdiag, h->d_scal, h->d_z, h->d_w,
                  h->ws, h->d_sums, h->d_aux, h->d_kind, h->d_ok, h->d_rank, h->d_sweeps, h->d_perm, h->d_y, h->d_ux, h->d_uy,
                  h->d_pred, h->d_partial, h->d_pacc, h->d_ibuf, h->d_acc, h->lkk, h->pbuf};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  h->ar.release();
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  if (h->stream) cudaStreamDestroy(h->stream);
  if (h->side) cudaStreamDestroy(h->side);
  if (h->lane2) cudaStreamDestroy(h->lane2);
  if (h->ev_b) cudaEventDestroy(h->ev_b);
  if (h->ev_f) cudaEventDestroy(h->ev_f);
  if (h->ev_syrk) cudaEventDestroy(h->ev_syrk);
  if (h->ev_potrf) cudaEventDestroy(h->ev_potrf);
  if (h->ctx) release_ctx(h->ctx);
  delete h;
}

int32_t tlrb_group_size(tlrb_handle* h) { return !h ? 0 : h->group() ? (int32_t)h->members.size() : 1; }

int32_t tlrb_member_stats(tlrb_handle* h, int32_t member, tlrb_stats* st) {
  if (!h || !st || member < 0 || member >= tlrb_group_size(h)) return TLRB_ERR_ARG;
  tlrb_handle* m = h->group() ? h->members[member] : h;
  *st = m->st;
  return TLRB_OK;
}

int32_t tlrb_loglik(tlrb_handle* h, const double* z, double th1, double th2, double th3, double nugget,
                    double acc, double* ll, double* logdet, double* quad, tlrb_stats* st) {
  if (!h || !z) return TLRB_ERR_ARG;
  return loglik_any(h, z, false, th1, th2, th3, nugget, acc, ll, logdet, quad, st);
}

int32_t tlrb_loglik_device(tlrb_handle* h, const double* d_z, double th1, double th2, double th3,
                           double nugget, double acc, double* ll, double* logdet, double* quad,
                           tlrb_stats* st) {
  if (!h || !d_z) return TLRB_ERR_ARG;
  return loglik_any(h, d_z, true, th1, th2, th3, nugget, acc, ll, logdet, quad, st);
}

int32_t tlrb_factorize(tlrb_handle* h, double th1, double th2, double th3, double nugget, double acc) {
  if (!h) return TLRB_ERR_ARG;
  const int rc = validate(th1, th2, th3, nugget, acc);
  if (rc) return rc;
  if (h->group())
    return run_members(h, [&](tlrb_handle* m, int) { return factorize_one(m, th1, th2, th3, nugget, acc); });
  return guarded(h, [&] { return factorize_one(h, th1, th2, th3, nugget, acc); });
}

int32_t tlrb_apply_factor(tlrb_handle* h, const double* x, double* y) {
  if (!h || !x || !y) return TLRB_ERR_ARG;
  if (h->group())
    return run_members(h, [&](tlrb_handle* m, int r) { return apply_factor_one(m, x, r ? nullptr : y); });
  return guarded(h, [&] { return apply_factor_one(h, x, y); });
}

int32_t tlrb_solve(tlrb_handle* h, const double* rhs, double* x) {
  if (!h || !rhs || !x) return TLRB_ERR_ARG;
  if (h->group())
    return run_members(h, [&](tlrb_handle* m, int r) { return solve_one(m, rhs, r ? nullptr : x); });
  return guarded(h, [&] { return solve_one(h, rhs, x); });
}

int32_t tlrb_predict(tlrb_handle* h, const double* z, const double* xy_unknown, int64_t m, double th1,
                     double th2, double th3, double nugget, double acc, double* pred) {
  if (!h || !z || !xy_unknown || !pred || m < 1) return TLRB_ERR_ARG;
  int rc = validate(th1, th2, th3, nugget, acc);
  if (rc) return rc;
  if (h->group())
    return run_members(h, [&](tlrb_handle* mm, int r) {
      return predict_one(mm, z, xy_unknown, m, th1, th2, th3, nugget, acc, r ? nullptr : pred);
    });
  return guarded(h, [&] { return predict_one(h, z, xy_unknown, m, th1, th2, th3, nugget, acc, pred); });
}

int32_t tlrb_predict_var(tlrb_handle* h, const double* z, const double* xy_unknown, int64_t m, double th1,
                         double th2, double th3, double nugget, double acc, double* pred, double* cov) {
  if (!h || !z || !xy_unknown || !pred || !cov || m < 1) return TLRB_ERR_ARG;
  int rc = validate(th1, th2, th3, nugget, acc);
  if (rc) return rc;
  if (h->group() || h->dist()) {
    h->msg = "conditional covariance: single-GPU handles only";
    return TLRB_ERR_ARG;
  }
  return guarded(h, [&]() -> int {
    const int r = predict_one(h, z, xy_unknown, m, th1, th2, th3, nugget, acc, pred);
    if (r) return r;
    return kriging_cov(h, m, nugget, cov);
  });
}

int32_t tlrb_rank_map(tlrb_handle* h, int32_t* ranks, int32_t cap, int32_t* t_out) {
  if (!h) return TLRB_ERR_ARG;
  if (h->group()) return tlrb_rank_map(h->members[0], ranks, cap, t_out);
  if (t_out) *t_out = h->t;
  if (!ranks) return TLRB_OK;
  if (cap < h->t * h->t) return TLRB_ERR_ARG;
  for (int i = 0; i < h->t * h->t; ++i) ranks[i] = 0;
  for (int i = 1; i < h->t; ++i)
    for (int j = 0; j < i; ++j)
      ranks[i * h->t + j] = (h->factor_mode == 1 || h->dn(i, j)) ? -1 : h->rank[h->tid(i, j)];
  return TLRB_OK;
}

int32_t tlrb_last_error(tlrb_handle* h, int32_t* tile, int32_t* pivot, char* msg, int32_t len) {
  if (!h) return TLRB_ERR_ARG;
  if (tile) *tile = h->err_tile;
  if (pivot) *pivot = h->err_pivot;
  if (msg && len > 0) {
    strncpy(msg, h->msg.c_str(), len - 1);
    msg[len - 1] = 0;
  }
  return TLRB_OK;
}

int32_t tlrb_bessel_k(double nu, const double* x, int64_t count, double* out, int32_t device) {
  if (!x || !out || count < 0 || !(nu > 0 && nu <= 5)) return TLRB_ERR_ARG;
  return guarded(nullptr, [&]() -> int {
    TLRB_CUDA(cudaSetDevice(device));
    double *dxp, *dop;
    TLRB_CUDA(cudaMalloc(&dxp, std::max<int64_t>(1, count) * 8));
    TLRB_CUDA(cudaMalloc(&dop, std::max<int64_t>(1, count) * 8));
    TLRB_CUDA(cudaMemcpy(dxp, x, count * 8, cudaMemcpyHostToDevice));
    if (count) launch_bessel(nu, dxp, dop, count, 0);
    TLRB_CUDA(cudaMemcpy(out, dop, count * 8, cudaMemcpyDeviceToHost));
    cudaFree(dxp);
    cudaFree(dop);
    return TLRB_OK;
  });
}

int32_t tlrb_matern_block(const double* rows_xy, int64_t m, const double* cols_xy, int64_t n, double th1,
                          double th2, double th3, double* out, int32_t device) {
  return tlrb_matern_block_metric(rows_xy, m, cols_xy, n, th1, th2, th3, 0.0, out, device);
}

int32_t tlrb_matern_block_metric(const double* rows_xy, int64_t m, const double* cols_xy, int64_t n,
                                 double th1, double th2, double th3, double sphere_radius, double* out,
                                 int32_t device) {
  if (!rows_xy || !cols_xy || !out || m < 1 || n < 1) return TLRB_ERR_ARG;
  if (validate(th1, th2, th3, 0.0, 0.0)) return TLRB_ERR_ARG;
  std::vector<double> all(2 * (m + n));
  std::copy(rows_xy, rows_xy + 2 * m, all.begin());
  std::copy(cols_xy, cols_xy + 2 * n, all.begin() + 2 * m);
  std::vector<double> a1, a2, a3;
  if (kernel_view(all.data(), m + n, sphere_radius, a1, a2, a3)) return TLRB_ERR_ARG;
  return guarded(nullptr, [&]() -> int {
    TLRB_CUDA(cudaSetDevice(device));
    double *p1, *p2, *p3 = nullptr, *po;
    TLRB_CUDA(cudaMalloc(&p1, (m + n) * 8));
    TLRB_CUDA(cudaMalloc(&p2, (m + n) * 8));
    TLRB_CUDA(cudaMalloc(&po, m * n * 8));
    TLRB_CUDA(cudaMemcpy(p1, a1.data(), (m + n) * 8, cudaMemcpyHostToDevice));
    TLRB_CUDA(cudaMemcpy(p2, a2.data(), (m + n) * 8, cudaMemcpyHostToDevice));
    if (!a3.empty()) {
      TLRB_CUDA(cudaMalloc(&p3, (m + n) * 8));
      TLRB_CUDA(cudaMemcpy(p3, a3.data(), (m + n) * 8, cudaMemcpyHostToDevice));
    }
    DescArena ar;
    ar.init(1 << 20);
    // diag_add applies where global row == global col: rows and cols are disjoint index ranges here
    launch_gen_tiles({GenTile{po, (int)m, 0, (int)m, (int)m, (int)n, 0.0}}, Pts{p1, p2, p3, 2.0 * sphere_radius},
                     make_matern(th1, th2, th3), ar, 0);
    TLRB_CUDA(cudaMemcpy(out, po, m * n * 8, cudaMemcpyDeviceToHost));
    ar.release();
    cudaFree(p1);
    cudaFree(p2);
    if (p3) cudaFree(p3);
    cudaFree(po);
    return TLRB_OK;
  });
}

int32_t tlrb_potrf_tile(const double* a, int32_t n, int32_t tile_index, double* l, int32_t* pivot,
                        int32_t device) {
  if (!a || !l || n < 1) return TLRB_ERR_ARG;
  if (pivot) *pivot = -1;
  int info[3] = {0, 0, 0};
  const int rc = guarded(nullptr, [&]() -> int {
    TLRB_CUDA(cudaSetDevice(device));
    double *dA = nullptr, *dlog = nullptr;
    int* dinfo = nullptr;
    TLRB_CUDA(cudaMalloc(&dA, (size_t)n * n * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&dlog, (size_t)n * sizeof(double)));
    TLRB_CUDA(cudaMalloc(&dinfo, 3 * sizeof(int)));
    TLRB_CUDA(cudaMemset(dinfo, 0, 3 * sizeof(int)));
    TLRB_CUDA(cudaMemcpy(dA, a, (size_t)n * n * sizeof(double), cudaMemcpyHostToDevice));
    DescArena ar;
    ar.init(1 << 20);
    potrf_blocks(dA, n, n, tile_index, dinfo, dlog, ar, 0);
    tril_kernel<<<64, 256>>>(dA, n, n);   // np.tril (linalg.py:45)
    post_launch();
    TLRB_CUDA(cudaMemcpy(l, dA, (size_t)n * n * sizeof(double), cudaMemcpyDeviceToHost));
    TLRB_CUDA(cudaMemcpy(info, dinfo, sizeof info, cudaMemcpyDeviceToHost));
    ar.release();
    cudaFree(dA);
    cudaFree(dlog);
    cudaFree(dinfo);
    return TLRB_OK;
  });
  if (rc) return rc;
  if (info[0]) {
    if (pivot) *pivot = info[2];
    return TLRB_ERR_NPD;
  }
  return TLRB_OK;
}

int32_t tlrb_set_metric(tlrb_handle* h, double sphere_radius) {
  if (!h) return TLRB_ERR_ARG;
  std::vector<double> a1, a2, a3;
  const std::vector<double>& xy = h->group() ? h->members[0]->hxy : h->hxy;
  if (kernel_view(xy.data(), h->n, sphere_radius, a1, a2, a3)) return TLRB_ERR_ARG;
  if (h->group()) {
    h->diam = 2.0 * sphere_radius;
    return run_members(h, [&](tlrb_handle* m, int) { return set_metric_one(m, a1, a2, a3, sphere_radius); });
  }
  return guarded(h, [&] { return set_metric_one(h, a1, a2, a3, sphere_radius); });
}

int32_t tlrb_compress_tile(const double* a, int32_t m, int32_t n, double acc, int32_t* rank, double* u,
                           double* v, int32_t device) {
  if (!a || !rank || m < 1 || n < 1 || !(acc > 0 && acc < 1)) return TLRB_ERR_ARG;
  // a one-tile handle: nb = max(m, n), compression workspace of one job
  std::vector<double> xy(2 * (size_t)std::max(m, n), 0.0);
  for (size_t i = 0; i < xy.size() / 2; ++i) xy[2 * i] = (double)i;
  int32_t err = 0;
  tlrb_handle* h = tlrb_create(xy.data(), std::max(m, n), std::max(m, n), 1, 0, device, &err);
  if (!h) return err;
  const int rc = guarded(h, [&]() -> int {
    Job J{};
    bind_slot(h, J, 0);
    J.m = m;
    J.n = n;
    J.s = n;   // QRCP kernel hint: unknown rank, assume large
    J.kind = 0;
    J.Uout = h->diag;  // the diag arena (nb x nb) receives U (m x k)
    double* dv;
    TLRB_CUDA(cudaMalloc(&dv, (size_t)n * std::min(m, n) * 8));
    J.Vout = dv;
    J.ldu = m;
    J.ldv = n;
    J.seed = 99;
    TLRB_CUDA(cudaMemcpy(J.M, a, (size_t)m * n * 8, cudaMemcpyHostToDevice));
    std::vector<Job> jobs{J};
    compress_jobs(h, jobs, acc);
    h->sync();
    const int k = jobs[0].out_rank;
    *rank = k;
    if (u && k) TLRB_CUDA(cudaMemcpy(u, h->diag, (size_t)m * k * 8, cudaMemcpyDeviceToHost));
    if (v && k) TLRB_CUDA(cudaMemcpy(v, dv, (size_t)n * k * 8, cudaMemcpyDeviceToHost));
    cudaFree(dv);
    return TLRB_OK;
  });
  tlrb_destroy(h);
  return rc;
}

int64_t tlrb_launch_count(void) { return g_launches; }

int32_t tlrb_profile_enable(int32_t on) {
  g_prof.reset();
  g_prof.on = on != 0;
  return TLRB_OK;
}

int32_t tlrb_profile_mask(uint32_t mask) {
  g_prof.mask = mask;
  return TLRB_OK;
}

int32_t tlrb_set_peaks(double fp64_tflops, double hbm_gbs) {
  if (!(fp64_tflops > 0) || !(hbm_gbs > 0)) return TLRB_ERR_ARG;
  g_peak_flops = fp64_tflops * 1e12;
  g_peak_bytes = hbm_gbs * 1e9;
  return TLRB_OK;
}

int32_t tlrb_profile_busy(int32_t cls, double* busy_ms) {
  if (cls >= K_NCLASS || !busy_ms) return TLRB_ERR_ARG;
  *busy_ms = g_prof.busy_ms(cls);
  return TLRB_OK;
}

int32_t tlrb_profile_read(int32_t cls, char* name, int32_t len, double* ms, double* flops, double* bytes,
                          int64_t* launches) {
  if (cls < 0 || cls >= K_NCLASS) return TLRB_ERR_ARG;
  g_prof.drain();
  if (name && len > 0) {
    strncpy(name, kclass_name[cls], len - 1);
    name[len - 1] = 0;
  }
  if (ms) *ms = g_prof.ms[cls];
  if (flops) *flops = g_prof.flops[cls];
  if (bytes) *bytes = g_prof.bytes[cls];
  if (launches) *launches = g_prof.count[cls];
  return TLRB_OK;
}

}  // extern "C"

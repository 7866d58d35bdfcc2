/*
 * tlrb200.h — C ABI of the B200-native TLR Gaussian log-likelihood library
 * (libtlrb200.so).  Plain pointers and sizes only; no torch / CUDA types.
 *
 * The drop-in boundary replaces these reference entry points
 * (/root/reference/pkg/src/tlrgeo/):
 *   stats.log_likelihood        stats.py:103-112   -> tlrb_loglik
 *   stats._factorize            stats.py:96-100    -> (inside tlrb_loglik)
 *   tilestore.assemble_covariance tilestore.py:181-223 -> (inside tlrb_loglik)
 *   linalg.cholesky / tlr_cholesky / dense_cholesky linalg.py:82-147
 *   linalg.quadratic_form       linalg.py:200-206
 *   linalg.solve_cholesky       linalg.py:195-197  -> tlrb_solve
 *   predict.predict (mean)      predict.py:65-87   -> tlrb_predict
 *   kernels.bessel_k            kernels.py:216-226 -> tlrb_bessel_k
 *   kernels.matern_block        kernels.py:494-530 -> tlrb_matern_block(_metric)
 *   geometry.GreatCircle / LocationSet(..., GreatCircle(r)) geometry.py:24-31,80-122
 *                               kernels.py:460-491 -> tlrb_set_metric
 *   compression.compress_tile   compression.py:39-51 -> tlrb_compress_tile
 *   linalg.NotPositiveDefiniteError linalg.py:20-33 -> TLRB_ERR_NPD + tlrb_last_error
 *
 * Return codes of every int-returning call.
 *
 * Threading: a handle lives on one device; calls that reach the same device
 * (from any host thread, on any handle) are serialised inside the library,
 * calls on different devices run concurrently.  Distributed handles
 * (tlrb_create_dist) hold an NCCL communicator: every rank makes the same
 * sequence of calls.
 */
#ifndef TLRB200_H
#define TLRB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TLRB_OK 0
#define TLRB_ERR_NPD 1     /* not positive definite: (tile, pivot) via tlrb_last_error */
#define TLRB_ERR_ARG 2     /* invalid argument (shape, theta, accuracy) */
#define TLRB_ERR_CUDA 3    /* CUDA / NCCL / out-of-memory */

/* communicator backends of tlrb_create_group */
#define TLRB_BACKEND_AUTO 0      /* NCCL when the devices are distinct, else loopback */
#define TLRB_BACKEND_NCCL 1      /* NCCL over NVLink / NVSwitch, one rank per device */
#define TLRB_BACKEND_LOOPBACK 2  /* in-process: host rendezvous + stream-ordered device copies */

typedef struct tlrb_handle tlrb_handle;

/* Per-evaluation statistics (phase times measured with CUDA events on the
 * handle's stream; algorithmic work counted from the actual ranks). */
typedef struct tlrb_stats {
  double ms_generate;     /* tile generation (+ initial compression in TLR) */
  double ms_compress;     /* initial compression only */
  double ms_factor;       /* tile Cholesky */
  double ms_solve;        /* forward solve + dot + log-det reduction */
  double ms_total;        /* host wall clock of the call */
  double ms_device;       /* CUDA events on the handle's stream, call entry -> result ready */
  double flops;           /* algorithmic FP64 flops (SURVEY 8(d) formulas) */
  double bytes;           /* algorithmic HBM bytes (SURVEY 8(d) formulas) */
  int64_t stored_reals;   /* footprint() semantics, tilestore.py:150-163 */
  int64_t kernel_launches;/* kernels launched by this call */
  int32_t max_rank;       /* of the final factor's off-diagonal tiles */
  double mean_rank;
  int32_t sketch_retries; /* compression sketches that had to be enlarged */
  int32_t jacobi_max_sweeps;
  double t_roof_ms;       /* sum over ops of max(F / P64, B / BW) (tlrb_set_peaks) */
  int64_t arena_peak_bytes; /* high-water mark of this rank's tile factor arena */
  int64_t panel_peak_bytes; /* largest received panel (distributed handles) */
} tlrb_stats;

/* Create a handle for n locations (xy: n x 2, row-major, like
 * LocationSet.coords).  nb: tile size (min(nb, n) is used), max_rank: <=0
 * means uncapped, device: CUDA ordinal.  ngpus > 1: this one handle drives
 * devices device .. device + ngpus - 1 from the calling process (2D
 * block-cyclic tiles, as tlrb_create_dist, NCCL between the devices, one host
 * thread per device inside each call) — the replacement for
 * LikelihoodConfig(ngpus=G) in a single-process caller such as mle_fit.
 * min(nb, n) above 2048 is refused (TLRB_ERR_ARG): the compression kernels
 * stage at most 2048 rows per column.  Locations stay resident on the device
 * across evaluations.  *err receives a TLRB_* code. */
tlrb_handle* tlrb_create(const double* xy, int64_t n, int32_t nb, int32_t ngpus,
                         int32_t max_rank, int32_t device, int32_t* err);
void tlrb_destroy(tlrb_handle* h);

/* Multi-GPU (one process per GPU): 2D block-cyclic tile distribution over a
 * P x Q process grid (P * Q == world), tile (i, j) on rank (i mod P) * Q +
 * (j mod Q); rank r is in process row r / Q and process column r mod Q, with
 * a communicator for each.  Per panel k: the owner of D_k
 * factors it and broadcasts L_kk down its process column; the panel owners
 * solve their tiles; one world all-reduce carries the NPD flag and the
 * panel's ranks; the panel goes out packed, along process rows (tiles (i, k)
 * to the owners of row i) then down process columns (tiles (j, k) to the
 * owners of column j); owners of D_j / (i, j) apply their updates and the
 * received panel is dropped, so a rank stores its own tiles plus one panel.
 * log-det is all-reduced; the triangular solves reduce a tile vector along a
 * process row (column) and broadcast it down a column (row) per step.  All
 * collectives run on the handle's stream.  rank 0 creates the id with
 * tlrb_nccl_unique_id (128 bytes) and shares it out of band (e.g.
 * torch.distributed). */
int32_t tlrb_nccl_unique_id(char* out, int32_t len);
tlrb_handle* tlrb_create_dist(const double* xy, int64_t n, int32_t nb, int32_t max_rank,
                              int32_t device, int32_t rank, int32_t world, int32_t P,
                              int32_t Q, const char* nccl_id, int32_t* err);

/* The same 2D block-cyclic schedule with `world` ranks inside this process,
 * rank r on devices[r] (devices may repeat), driven by one host thread per
 * rank within each call.  backend TLRB_BACKEND_LOOPBACK runs the collectives
 * as host rendezvous + stream-ordered device copies (no kernel waits on
 * another rank), so W logical ranks can share one GPU: the multi-GPU path is
 * executed and checked on one B200.  Every tlrb_* call on the returned handle
 * runs on all ranks; outputs come from rank 0. */
tlrb_handle* tlrb_create_group(const double* xy, int64_t n, int32_t nb, int32_t max_rank,
                               const int32_t* devices, int32_t world, int32_t P, int32_t Q,
                               int32_t backend, int32_t* err);
/* Ranks behind a handle (1 for a single-GPU or one-process-per-GPU handle). */
int32_t tlrb_group_size(tlrb_handle* h);
/* The last evaluation's statistics of one rank of a group handle. */
int32_t tlrb_member_stats(tlrb_handle* h, int32_t member, tlrb_stats* st);

/* Distance metric of the handle's locations.  sphere_radius == 0: Euclidean
 * (the default after create); > 0: great-circle (haversine) distance on a
 * sphere of that radius, xy read as (lon, lat) in degrees with |lon| <= 180,
 * |lat| <= 90 (else TLRB_ERR_ARG) — geometry.GreatCircle.  Applies to every
 * later evaluation, including the unknown points of tlrb_predict. */
int32_t tlrb_set_metric(tlrb_handle* h, double sphere_radius);

/* One Gaussian log-likelihood evaluation
 *   ll = -0.5 (n log 2pi + log|Sigma| + z' Sigma^-1 z)     (stats.py:112)
 * z: host pointer (n doubles).  acc == 0 -> dense mode, else TLR(acc).
 * Any of ll/logdet/quad/st may be NULL. */
int32_t tlrb_loglik(tlrb_handle* h, const double* z, double theta1, double theta2,
                    double theta3, double nugget, double acc, double* ll,
                    double* logdet, double* quad, tlrb_stats* st);

/* Same, with z already resident in device memory (used for the HBM-resident
 * throughput measurement). */
int32_t tlrb_loglik_device(tlrb_handle* h, const double* d_z, double theta1,
                           double theta2, double theta3, double nugget, double acc,
                           double* ll, double* logdet, double* quad, tlrb_stats* st);

/* Factorise Sigma(theta) into the handle without a solve (acc == 0: dense).
 * Used by tlrb_apply_factor / tlrb_solve. */
int32_t tlrb_factorize(tlrb_handle* h, double theta1, double theta2, double theta3,
                       double nugget, double acc);

/* y = L x with the current factor (stats.sample_measurements, stats.py:115-133,
 * draws z = L w with the dense nb = min(200, n) factor).  x, y: host, n. */
int32_t tlrb_apply_factor(tlrb_handle* h, const double* x, double* y);

/* Solve Sigma x = rhs with the factor of the last successful tlrb_loglik /
 * tlrb_predict call (linalg.solve_cholesky semantics).  rhs, x: host, n. */
int32_t tlrb_solve(tlrb_handle* h, const double* rhs, double* x);

/* Kriging mean (predict.py:65-87): factorize Sigma_22 over the handle's
 * locations, w = Sigma_22^-1 z, pred = Sigma_12 w with Sigma_12 generated on
 * the fly (never materialised).  xy_unknown: m x 2 row-major host array. */
int32_t tlrb_predict(tlrb_handle* h, const double* z, const double* xy_unknown,
                     int64_t m, double theta1, double theta2, double theta3,
                     double nugget, double acc, double* pred);

/* tlrb_predict plus the conditional covariance of the unknown sites,
 * S11 - S12 S22^-1 S21 (predict.py:81-87), m x m column-major in cov:
 * generated, solved (m right-hand sides) and multiplied on the device.
 * Single-GPU handles (TLRB_ERR_ARG otherwise). */
int32_t tlrb_predict_var(tlrb_handle* h, const double* z, const double* xy_unknown, int64_t m,
                         double th1, double th2, double th3, double nugget, double acc,
                         double* pred, double* cov);

/* Tile rank map of the last factor: ranks[i*t + j] for i > j (t = tiles);
 * -1 marks a tile stored dense.  Returns t via *t_out. */
int32_t tlrb_rank_map(tlrb_handle* h, int32_t* ranks, int32_t cap, int32_t* t_out);

/* Last error of the handle: NPD tile / pivot (linalg.py:43-44) and message. */
int32_t tlrb_last_error(tlrb_handle* h, int32_t* tile, int32_t* pivot, char* msg,
                        int32_t len);

/* ---- stand-alone device kernels, for parity tests of single components ---- */

/* out[i] = K_nu(x[i]) on the device (kernels.py:160-174). */
int32_t tlrb_bessel_k(double nu, const double* x, int64_t count, double* out,
                      int32_t device);

/* out (m x n, column-major, ld = m) = Matern block between row points and
 * column points (kernels.py:494-530, no nugget). */
int32_t tlrb_matern_block(const double* rows_xy, int64_t m, const double* cols_xy,
                          int64_t n, double theta1, double theta2, double theta3,
                          double* out, int32_t device);
/* Same with a metric: sphere_radius as in tlrb_set_metric (kernels.py:460-491). */
int32_t tlrb_matern_block_metric(const double* rows_xy, int64_t m, const double* cols_xy,
                                 int64_t n, double theta1, double theta2, double theta3,
                                 double sphere_radius, double* out, int32_t device);

/* Compress one dense m x n tile (column-major) to relative Frobenius accuracy
 * acc with the device compressor (compression.py:39-51).  u: m x k, v: n x k
 * (column-major, ld = m / n; caller provides min(m,n) columns). */
int32_t tlrb_compress_tile(const double* a, int32_t m, int32_t n, double acc,
                           int32_t* rank, double* u, double* v, int32_t device);

/* Cholesky of one dense tile (potrf_tile, linalg.py:36-45): a is n x n
 * column-major (the lower triangle is read), l receives the lower factor
 * (upper part zero).  TLRB_ERR_NPD when a pivot is not positive: *pivot is
 * its 0-based column (the reference's info - 1). */
int32_t tlrb_potrf_tile(const double* a, int32_t n, int32_t tile_index, double* l, int32_t* pivot,
                        int32_t device);

/* Number of kernels this library has launched in this process. */
int64_t tlrb_launch_count(void);

/* Per-kernel-class profiler: CUDA events around every launch on its stream,
 * plus the algorithmic flops / bytes of each launch.
 * enable resets the counters.  Classes: 0..10 (name returned). */
int32_t tlrb_profile_enable(int32_t on);
/* Restrict the profiler to the classes whose bit is set (default: all), so a
 * timed region can carry events for one kernel class only. */
int32_t tlrb_profile_mask(uint32_t mask);
int32_t tlrb_profile_read(int32_t cls, char* name, int32_t len, double* ms, double* flops,
                          double* bytes, int64_t* launches);
/* Busy time (ms) of one class since enable: the union of its launches'
 * [start, end] intervals, so launches of one class overlapping on several
 * streams count once (cls = -1: union over every class). */
int32_t tlrb_profile_busy(int32_t cls, double* busy_ms);
/* Peaks behind tlrb_stats.t_roof_ms (default 35.5 TFLOP/s FP64 DMMA,
 * 6449.7 GB/s HBM: the measured B200 figures). */
int32_t tlrb_set_peaks(double fp64_tflops, double hbm_gbs);

#ifdef __cplusplus
}
#endif
#endif

/* qdwhg.h — C ABI of libqdwhg, the B200-native (sm_100a) QDWHpartial hot path.
 *
 * Drop-in boundary for the reference's core/ driver entry points
 * (/root/reference/proj/core/include/qdwh):
 *
 *   qdwhg_polar              <- qdwh::polar_decompose          polar.hpp:60
 *   qdwhg_partial_eig        <- qdwh::qdwh_partial_eig         partial.hpp:55-57
 *   qdwhg_partial_svd        <- qdwh::qdwh_partial_svd         partial.hpp:85-86
 *   qdwhg_partial_eig_request <- spectrum-fraction front end for partial EIG
 *                               (shift map B = cI - A / A - cI)
 *   qdwhg_partial_svd_request <- absolute-cut / top-k front end for partial SVD
 *   qdwhg_run_fixed_iterations <- qdwh::run_fixed_iterations  polar.hpp:74-75
 *   qdwhg_qdwh_chol_step     <- qdwh::qdwh_chol_step           polar.hpp:56
 *   qdwhg_qdwh_qr_step       <- qdwh::qdwh_qr_step             polar.hpp:53
 *   qdwhg_qr_factor          <- qdwh::qr_factor                kernels.hpp:18
 *   qdwhg_cholesky           <- qdwh::cholesky                 kernels.hpp:25
 *   qdwhg_sym_eig_dense      <- qdwh::sym_eig_dense            kernels.hpp:33
 *   qdwhg_svd_dense          <- qdwh::svd_dense                kernels.hpp:42
 *   qdwhg_two_norm_estimate  <- qdwh::two_norm_estimate        kernels.hpp:46
 *   qdwhg_lanczos_min_bound  <- qdwh::lanczos_min_bound        kernels.hpp:51
 *   qdwhg_halley_weights     <- qdwh::halley_weights           polar.hpp:22
 *   qdwhg_iterations_to_converge <- qdwh::iterations_to_converge polar.hpp:30
 *   qdwhg_choose_shift       <- qdwh::choose_shift             partial.hpp:23
 *   qdwhg_eig_full           <- qdwh::qdwh_eig_full            fullsolve.hpp:21
 *   qdwhg_svd_full           <- qdwh::qdwh_svd_full            fullsolve.hpp:24
 *   qdwhg_accuracy_report    <- qdwh::accuracy_report          metrics.hpp:25-28
 *
 * Conventions (mirroring the reference):
 *   - matrices are column-major FP64 with an explicit leading dimension;
 *   - every matrix pointer may be HOST or DEVICE memory (on the handle's
 *     device); the kind is detected per pointer.  Device pointers skip the
 *     host<->device copies (the benchmark's "value" path), host pointers are
 *     the end-to-end path;
 *   - outputs are caller-allocated; vector outputs hold k_cap columns and the
 *     number actually returned is info->k (QDWHG_CAPACITY if k > k_cap);
 *   - exceptions of the reference map to status codes; an empty spectrum is
 *     NOT an error (status OK, info->k == 0), as in partial.cpp:52,73,90,140,152;
 *   - a handle is used by one thread at a time; calls are synchronous.
 */
#ifndef QDWHG_H
#define QDWHG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum qdwhg_status {
  QDWHG_OK = 0,
  QDWHG_INVALID_ARGUMENT = 1,      /* std::invalid_argument                      */
  QDWHG_NOT_POSITIVE_DEFINITE = 2, /* qdwh::NotPositiveDefinite, matrix.hpp:13-16 */
  QDWHG_NOT_CONVERGED = 3,         /* qdwh::NotConverged, matrix.hpp:19-22        */
  QDWHG_CAPACITY = 4,              /* k exceeds the caller's k_cap                 */
  QDWHG_CUDA_ERROR = 5,
  QDWHG_NCCL_ERROR = 6,
  QDWHG_INTERNAL = 7
} qdwhg_status;

typedef struct qdwhg_handle qdwhg_handle;

typedef struct qdwhg_options {
  int32_t device;        /* CUDA ordinal; -1 = current device */
  int32_t reserved0;
  uint64_t arena_bytes;  /* 0 = grow on demand */
  uint64_t flags;        /* QDWHG_FLAG_* bits, 0 = defaults */
} qdwhg_options;

/* Bitwise run-to-run reproducible results: the cross-CTA reductions of the tall
 * QR panels sum per-CTA partials in a fixed order instead of FP64 atomics
 * (slower panels on matrices with more than 2048 rows). */
#define QDWHG_FLAG_DETERMINISTIC 1u

#define QDWHG_MAX_TRACE 64
#define QDWHG_NUM_STAGES 8
/* stage_seconds[]: 0 bound (Lanczos / power iteration), 1 QDWH iterations,
 * 2 subspace QR + diag scan, 3 Q2 formation, 4 Rayleigh-Ritz products,
 * 5 small EIG/SVD, 6 back-transform, 7 host<->device transfers */

typedef struct qdwhg_eig_info { /* partial.hpp:29-52 */
  double mu;               /* Lanczos lower bound used as scale          */
  double shift;            /* plan.s                                     */
  double tol;
  double c_shift;          /* request front end: spectral shift c (0 for raw calls) */
  int64_t rank_index;      /* 1-based deficiency index, 0 when none      */
  int64_t subspace_size;   /* ell                                        */
  int64_t k;               /* values returned                            */
  int64_t k_found;         /* values found before a request's top-k cut  */
  int64_t iters_qr, iters_chol, borderline;
  int32_t no_savings, randomized;
  int32_t n_trace;
  int32_t subspace_path;   /* 0: Householder QR of B (partial.cpp:71-79), 1: Cholesky-QR extraction */
  double ell_trace[QDWHG_MAX_TRACE];
  double seconds;          /* device time of the call                    */
  double flops;            /* algorithmic FP64 flops   */
  double stage_seconds[QDWHG_NUM_STAGES];
} qdwhg_eig_info;

typedef struct qdwhg_svd_info { /* partial.hpp:59-81 */
  double alpha;            /* two-norm estimate used for scaling */
  double threshold;        /* relative threshold s               */
  double tol;
  double cut;              /* absolute cut s*alpha               */
  int64_t rank_index, subspace_size, k, k_found;
  int64_t iters_qr, iters_chol;
  int32_t no_savings, randomized;
  int32_t n_trace, reserved;
  double ell_trace[QDWHG_MAX_TRACE];
  double seconds, flops;
  double stage_seconds[QDWHG_NUM_STAGES];
} qdwhg_svd_info;

typedef struct qdwhg_polar_config { /* polar.hpp:34-40 */
  double ell0;           /* 1e-15 */
  int64_t max_iters;     /* 60 */
  double conv_eps;       /* 2.220446049250313e-16 */
  double chol_switch_c;  /* 100 */
  int32_t force_variant; /* 0 Auto, 1 QrOnly, 2 CholeskyOnly */
  int32_t estimate_ell0; /* 1: ell0 ignored, a lower bound of sigma_min(A)/||A||_2 is
                            estimated from the R factor of A (no reference
                            counterpart: polar.hpp:35 takes 1/kappa from the caller) */
} qdwhg_polar_config;

typedef struct qdwhg_polar_info { /* polar.hpp:42-50 */
  double alpha;
  int64_t iters_qr, iters_chol;
  int32_t converged, n_trace;
  double ell_trace[QDWHG_MAX_TRACE];
  double seconds, flops;
} qdwhg_polar_info;

typedef enum qdwhg_which {
  QDWHG_NEGATIVE = 0, /* reference semantics: eigenvalues < 0 of A            */
  QDWHG_LARGEST = 1,  /* eigenvalues > c of A   (B = c I - A)                  */
  QDWHG_SMALLEST = 2  /* eigenvalues < c of A   (B = A - c I)                  */
} qdwhg_which;

typedef struct qdwhg_eig_request {
  int32_t which;       /* qdwhg_which */
  int32_t iters;       /* 2 or 3 (choose_shift, partial.cpp:26-30) */
  double c;            /* spectral shift (ignored for NEGATIVE) */
  int64_t k;           /* keep the k extreme values by count; 0 = all found */
  double tol;          /* 0.01 */
  int32_t randomize;
  int32_t reserved;
  uint64_t seed;
} qdwhg_eig_request;

typedef struct qdwhg_svd_request {
  int32_t mode;        /* 0: relative s (keep sigma > s*alpha, reference);
                          1: absolute cut (keep sigma > value; s = value/alpha) */
  int32_t randomize;
  double value;
  int64_t k;           /* keep the k largest by count; 0 = all found */
  double tol;
  uint64_t seed;
} qdwhg_svd_request;

/* ---- handle ------------------------------------------------------------ */
qdwhg_status qdwhg_create(qdwhg_handle** h, const qdwhg_options* opts);
qdwhg_status qdwhg_destroy(qdwhg_handle* h);
const char* qdwhg_last_error(const qdwhg_handle* h);
qdwhg_status qdwhg_get_launch_count(const qdwhg_handle* h, uint64_t* launches);
qdwhg_status qdwhg_synchronize(qdwhg_handle* h);
/* Run on a caller stream (cudaStream_t, e.g. torch's current stream); NULL
 * restores the handle's own (non-blocking) stream, cudaStreamLegacy ((void*)1)
 * selects the legacy default stream.  Calls stay synchronous. */
qdwhg_status qdwhg_set_stream(qdwhg_handle* h, void* stream);

/* Live kernel accounting: with profiling enabled every DMMA GEMM launch is
 * bracketed by CUDA events on its stream; get_kernel_stats returns and resets
 * the event-timed totals (launch counters are cumulative). */
typedef struct qdwhg_kernel_stats {
  uint64_t gemm_launches;       /* cumulative */
  uint64_t other_launches;      /* cumulative, all other libqdwhg kernels */
  uint64_t gemm_timed_launches; /* since the last get_kernel_stats */
  double gemm_seconds;          /* sum of event-timed GEMM durations */
  double gemm_flops;            /* sum of algorithmic flops of those launches */
  double gemm_busy_seconds;     /* union of the launch intervals (concurrent launches counted once) */
  uint64_t dag_timed_launches;  /* tile-DAG Cholesky-and-inverse launches, since the last call */
  double dag_seconds;           /* their event-timed durations */
  double dag_flops;             /* algorithmic flops: 2/3 n^3 per n x n factorisation + inverse */
} qdwhg_kernel_stats;
qdwhg_status qdwhg_profile(qdwhg_handle* h, int32_t enable);
/* Toggle QDWHG_FLAG_DETERMINISTIC on an existing handle. */
qdwhg_status qdwhg_set_deterministic(qdwhg_handle* h, int32_t enable);
qdwhg_status qdwhg_get_kernel_stats(qdwhg_handle* h, qdwhg_kernel_stats* out);

/* ---- drivers ------------------------------------------------------------ */
qdwhg_status qdwhg_partial_eig(qdwhg_handle* h, int64_t n, const double* A, int64_t lda,
                               int64_t qdwh_iters, int32_t use_randomization, double tol,
                               uint64_t seed, double* lambda, double* V, int64_t ldv,
                               int64_t k_cap, qdwhg_eig_info* info);
qdwhg_status qdwhg_partial_eig_request(qdwhg_handle* h, int64_t n, const double* A, int64_t lda,
                               const qdwhg_eig_request* req, double* lambda, double* V,
                               int64_t ldv, int64_t k_cap, qdwhg_eig_info* info);
qdwhg_status qdwhg_partial_svd(qdwhg_handle* h, int64_t m, int64_t n, const double* A,
                               int64_t lda, double s, double tol, int32_t use_randomization,
                               uint64_t seed, double* sigma, double* U, int64_t ldu, double* V,
                               int64_t ldv, int64_t k_cap, qdwhg_svd_info* info);
qdwhg_status qdwhg_partial_svd_request(qdwhg_handle* h, int64_t m, int64_t n, const double* A,
                               int64_t lda, const qdwhg_svd_request* req, double* sigma,
                               double* U, int64_t ldu, double* V, int64_t ldv, int64_t k_cap,
                               qdwhg_svd_info* info);
qdwhg_status qdwhg_polar(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                         const qdwhg_polar_config* cfg, double* Up, int64_t ldu, double* H,
                         int64_t ldh, qdwhg_polar_info* info);

/* ---- QDWH iteration pieces ----------------------------------------------- */
/* variant: 0 QrFirst, 1 CholeskyOnly.  trace_out (optional) receives iters+1 values. */
qdwhg_status qdwhg_run_fixed_iterations(qdwhg_handle* h, int64_t m, int64_t n, const double* X0,
                                        int64_t ldx, double ell0, int64_t iters, int32_t variant,
                                        double* X, int64_t ldo, double* trace_out);
qdwhg_status qdwhg_qdwh_chol_step(qdwhg_handle* h, int64_t m, int64_t n, const double* X,
                                  int64_t ldx, double ell, double* out, int64_t ldo);
qdwhg_status qdwhg_qdwh_qr_step(qdwhg_handle* h, int64_t m, int64_t n, const double* X,
                                int64_t ldx, double ell, double* out, int64_t ldo);

/* ---- dense kernels ---------------------------------------------------- */
qdwhg_status qdwhg_qr_factor(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                             double* Q, int64_t ldq, double* R, int64_t ldr);
qdwhg_status qdwhg_cholesky(qdwhg_handle* h, int64_t n, const double* Z, int64_t ldz, double* W,
                            int64_t ldw);
qdwhg_status qdwhg_sym_eig_dense(qdwhg_handle* h, int64_t n, const double* S, int64_t lds,
                                 double* values, double* V, int64_t ldv);
qdwhg_status qdwhg_svd_dense(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                             double* U, int64_t ldu, double* sigma, double* V, int64_t ldv);
/* Accuracy of a computed decomposition A ~ U diag(sigma) V^T (metrics.hpp:11-28,
 * Eq. 5-7): orth = ||I - U^T U||_F / n, residuals = max per-pair 2-norms; sigma and
 * delta (optional, may be NULL) are HOST arrays of length k; A m x n, U m x k, V n x k. */
typedef struct qdwhg_accuracy {
  double orth_left, orth_right;
  double value_err;        /* valid when has_value_err */
  double resid_right;      /* max ||A v_i - sigma_i u_i|| (paper pairing: the same)   */
  double resid_left;       /* max ||A^T u_i - sigma_i v_i|| (paper: ||A u_i - sigma_i v_i||) */
  int64_t n, k;
  int32_t has_value_err, reserved;
} qdwhg_accuracy;
qdwhg_status qdwhg_accuracy_report(qdwhg_handle* h, int64_t m, int64_t n, const double* A,
                                   int64_t lda, int64_t k, const double* U, int64_t ldu,
                                   const double* sigma, const double* V, int64_t ldv,
                                   const double* delta, int32_t paper_pairing,
                                   qdwhg_accuracy* out);

/* Full spectrum (fullsolve.cpp:22-103): all eigenpairs of a symmetric A by QDWH
 * spectral divide-and-conquer down to base_size (<= 0: the reference's 32),
 * values ascending, V (n x n); *depth (may be NULL) = recursion depth reached.
 * All singular triplets of A (m >= n) via the polar factor, sigma descending. */
qdwhg_status qdwhg_eig_full(qdwhg_handle* h, int64_t n, const double* A, int64_t lda,
                            int64_t base_size, double* lambda, double* V, int64_t ldv,
                            int64_t* depth);
qdwhg_status qdwhg_svd_full(qdwhg_handle* h, int64_t m, int64_t n, const double* A, int64_t lda,
                            int64_t base_size, double* U, int64_t ldu, double* sigma, double* V,
                            int64_t ldv);
qdwhg_status qdwhg_two_norm_estimate(qdwhg_handle* h, int64_t m, int64_t n, const double* A,
                                     int64_t lda, double* out);
qdwhg_status qdwhg_lanczos_min_bound(qdwhg_handle* h, int64_t n, const double* A, int64_t lda,
                                     int64_t steps, double* out);
/* C = alpha op(A) op(B) + beta C on DEVICE pointers (the DMMA engine itself). */
qdwhg_status qdwhg_gemm(qdwhg_handle* h, int32_t trans_a, int32_t trans_b, int64_t m, int64_t n,
                        int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                        int64_t ldb, double beta, double* C, int64_t ldc);
/* The same engine with the structure flags the QDWH steps use (DEVICE pointers):
 *   krange: 0 full, 1 op(B) upper, 2 op(B) lower, 3 op(A) upper, 4 op(A) lower
 *           (triangular operands store explicit zeros; their zero tiles are skipped)
 *   out:    0 full C, 1 lower triangle mirrored to the upper, 2 lower triangle only
 *   diag_add is added to the diagonal of C (e.g. Z = I + c X^T X in one launch). */
qdwhg_status qdwhg_gemm_ex(qdwhg_handle* h, int32_t trans_a, int32_t trans_b, int64_t m, int64_t n,
                           int64_t k, double alpha, const double* A, int64_t lda, const double* B,
                           int64_t ldb, double beta, double* C, int64_t ldc, int32_t krange,
                           int32_t out, double diag_add);
/* Upper Cholesky factor and its inverse: Z = W^T W; on return Z holds W and
 * Winv = W^{-1} (both upper, explicit zeros below).  Reads the lower triangle
 * of Z.  NOT_POSITIVE_DEFINITE on a non-positive pivot (kernels.cpp:136-138).
 * Host or device pointers. */
qdwhg_status qdwhg_cholesky_inverse(qdwhg_handle* h, int64_t n, double* Z, int64_t ldz,
                                    double* Winv, int64_t ldwi);
/* W^{-1} only (upper, explicit zeros below) of Z = W^T W by the recursive
 * Cholesky-and-inverse that multiplies by explicit inverses of half blocks (errors
 * ~ u*kappa(Z)): for well-conditioned Z such as the QDWH Cholesky step's
 * I + c X^T X (kappa <= 1 + c; polar.cpp:85-93).  Z is not modified. */
qdwhg_status qdwhg_cholesky_inverse_fast(qdwhg_handle* h, int64_t n, const double* Z, int64_t ldz,
                                         double* Winv, int64_t ldwi);
/* Subspace extraction of Alg. 1/2 (partial.cpp:71-79 / 138-146): unpivoted Householder
 * QR of the n x n B, *ind = first 1-based i with |R_ii| < tol (0: none), *ell = n - ind + 1,
 * and Q2 = Q(:, ind-1:n) (n x ell) formed from the trailing reflectors only.  B is read
 * (host or device).  CAPACITY when ell > ell_cap. */
qdwhg_status qdwhg_subspace_q2(qdwhg_handle* h, int64_t n, double* B, int64_t ldb, double tol,
                               int64_t* ind, int64_t* ell, double* Q2, int64_t ldq, int64_t ell_cap);
/* Counter-based N(0,1) matrix on the device (kernels.cpp:441-447 scheme, device libm). */
qdwhg_status qdwhg_gaussian_matrix(qdwhg_handle* h, int64_t m, int64_t n, uint64_t seed, double* A,
                                   int64_t lda);

/* ---- distributed driver: P x Q grid, 2D block-cyclic nb x nb tiles ------
 * (PAPER.md:671-686 data layout, Alg. 3).  One rank per GPU,
 * SPMD: every rank makes the same calls with its own handle.  Communication is
 * NCCL (panel / diagonal-block broadcasts in the grid's row / column / world
 * teams, short all-reductions, tile exchanges for transposes and gathers);
 * libnccl is loaded at run time.  Ranks emulated as threads of one process use
 * a loopback world instead (tests).  Matrices passed to load / solve are FULL
 * m x n (host or device; each rank reads only its own tiles).  Results: lambda /
 * sigma and info on every rank, V / U on rank 0 only (others may pass NULL).
 * The QR-based first step of partial SVD (s < 1e-3) is single-GPU only. */
typedef struct qdwhg_dist qdwhg_dist;
qdwhg_status qdwhg_dist_unique_id(void* id128); /* ncclGetUniqueId (rank 0 shares it) */
qdwhg_status qdwhg_dist_create_nccl(qdwhg_dist** d, qdwhg_handle* h, int32_t P, int32_t Q, int32_t nb,
                                    int32_t rank, const void* id128);
qdwhg_status qdwhg_dist_world_create(void** world, int32_t nranks);
qdwhg_status qdwhg_dist_world_destroy(void* world);
qdwhg_status qdwhg_dist_create_loopback(qdwhg_dist** d, qdwhg_handle* h, int32_t P, int32_t Q, int32_t nb,
                                        int32_t rank, void* world);
/* Caller-supplied transport (MPI, torch.distributed, ...): buffers are device
 * pointers on the rank's GPU, its stream synchronized before every call.  team:
 * 0 world, 1 grid row (ranks with the same p), 2 grid column; root / peer are
 * world ranks (rank = p * Q + q); op: 0 sum, 1 max, 2 min.  Inside a
 * group_begin/group_end bracket, results may complete at group_end (receives
 * must not block sends of the same group).  Return 0 on success. */
typedef struct qdwhg_comm_callbacks {
  void* ctx;
  int (*bcast)(void* ctx, double* buf, size_t count, int root, int team);
  int (*allreduce)(void* ctx, double* buf, size_t count, int op, int team);
  int (*send)(void* ctx, const double* buf, size_t count, int peer);
  int (*recv)(void* ctx, double* buf, size_t count, int peer);
  int (*group_begin)(void* ctx); /* optional (NULL) */
  int (*group_end)(void* ctx);   /* optional (NULL) */
} qdwhg_comm_callbacks;
qdwhg_status qdwhg_dist_create_callback(qdwhg_dist** d, qdwhg_handle* h, int32_t P, int32_t Q, int32_t nb,
                                        int32_t rank, const qdwhg_comm_callbacks* cb);
qdwhg_status qdwhg_dist_destroy(qdwhg_dist* d);
qdwhg_status qdwhg_dist_get_stats(const qdwhg_dist* d, uint64_t* collectives, uint64_t* local_gemms);
/* Keep the rank's tiles of A resident (solves with A == NULL reuse them). */
qdwhg_status qdwhg_dist_load(qdwhg_dist* d, int64_t m, int64_t n, const double* A, int64_t lda);
qdwhg_status qdwhg_dist_partial_eig_request(qdwhg_dist* d, int64_t n, const double* A, int64_t lda,
                                            const qdwhg_eig_request* req, double* lambda, double* V,
                                            int64_t ldv, int64_t k_cap, qdwhg_eig_info* info);
qdwhg_status qdwhg_dist_partial_svd_request(qdwhg_dist* d, int64_t m, int64_t n, const double* A, int64_t lda,
                                            const qdwhg_svd_request* req, double* sigma, double* U,
                                            int64_t ldu, double* V, int64_t ldv, int64_t k_cap,
                                            qdwhg_svd_info* info);

/* Distributed building blocks on FULL operands (every rank passes its copy; the
 * result is gathered to rank 0): pgemm (flags: 1 op(A) upper, 2 op(A) lower,
 * 4 op(B) upper, 8 op(B) lower, 16 only C's lower tiles), the recursive
 * Cholesky-and-inverse, and Householder QR |diag R| + Q(:, c0:c0+ell). */
qdwhg_status qdwhg_dist_pgemm(qdwhg_dist* d, int32_t ta, int32_t tb, int64_t m, int64_t n, int64_t k, double alpha,
                              const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                              const double* C0, int64_t ldc0, double* C, int64_t ldc, int32_t flags);
qdwhg_status qdwhg_dist_cholesky_inverse(qdwhg_dist* d, int64_t n, const double* Z, int64_t ldz, double* Winv,
                                         int64_t ldwi);
qdwhg_status qdwhg_dist_qr(qdwhg_dist* d, int64_t m, int64_t n, const double* X, int64_t ldx, int64_t c0,
                           int64_t ell, double* rdiag, double* Q2, int64_t ldq);

/* ---- host scalars (bit-identical to the reference: same libm calls) ---- */
qdwhg_status qdwhg_halley_weights(double ell, double out5[5]); /* a, b, c, ell_in, ell_out */
qdwhg_status qdwhg_iterations_to_converge(double ell0, double eps, int64_t max_iters,
                                          int64_t* out);
qdwhg_status qdwhg_choose_shift(int64_t qdwh_iters, double* s);

#ifdef __cplusplus
}
#endif

#endif /* QDWHG_H */

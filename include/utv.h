/*
 * utv.h -- C ABI of libutv.so: randUTV complete orthogonal decomposition and the
 * fast-option least-squares solve of arXiv 2408.05238 (Chillaron, Quintana-Orti, Vidal,
 * Martinsson), implemented as hand-written sm_100a (B200) CUDA kernels.
 *
 * Citations: "P:n" = line n of the paper's LaTeX source; readings R1..R18 are listed in
 * DESIGN.md ("Readings of the paper").
 *
 * Conventions (all entry points):
 *  - FP64, column-major, leading dimensions as in LAPACK (ld >= rows, ld >= 1).
 *  - Matrix pointers are DEVICE pointers of the handle's device unless stated otherwise;
 *    the caller allocates and owns every matrix.  The handle owns its workspace (allocated
 *    lazily, reused, freed by utv_destroy).
 *  - All work is enqueued on the handle's stream.  The only host synchronisation is the
 *    device->host read of the numerical rank r in utv_factor / utv_lstsq.
 *  - Errors are returned as utv_status, never by abort().  utv_last_error() gives a message.
 *    Argument / shape errors are detected before anything is written; after a later
 *    failure the contents of A, B, V, U and X are unspecified (LAPACK-like).
 *  - One handle per host thread.
 */
#ifndef UTV_H_
#define UTV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct utv_handle_s* utv_handle;

typedef enum {
  UTV_OK = 0,
  UTV_ERR_ARG = -1,          /* bad argument (null pointer, ld < rows, b < 1, q < 0, tau not in [0,1)) */
  UTV_ERR_SHAPE = -2,        /* m < n where unsupported: utv_factor / utv_solve (the paper's loop
                                guard for wide matrices is garbled: R4), multi-GPU or out-of-core lstsq */
  UTV_ERR_ALLOC = -3,        /* device / pinned allocation failed */
  UTV_ERR_CUDA = -4,         /* a CUDA runtime call failed */
  UTV_ERR_NCCL = -5,         /* multi-GPU communication failure (peer aborted, NCCL error, timeout) */
  UTV_ERR_NUMERICAL = -6,    /* NaN/Inf in A or B, or the b x b Jacobi SVD exceeded 30 sweeps */
  UTV_ERR_UNSUPPORTED = -7   /* a feature of this ABI that this build does not provide */
} utv_status;

enum {
  UTV_WANT_V = 1u,           /* (informational: V is produced whenever a V pointer is passed) */
  UTV_WANT_U = 2u,           /* build U explicitly (v21t semantics) when U != NULL */
  UTV_NULLIFY_T12 = 4u,      /* Nullify_top_right_part_of_T after Compute_rank (fig:alg_nullify_t12) */
  UTV_HOST_STREAMED = 8u,    /* utv_lstsq: A stays in host memory, streamed through HBM (out of core) */
  UTV_EXPLICIT_V = 16u,      /* utv_lstsq: accumulate V explicitly (default: factored V, see below) */
  UTV_KEEP_FACTORS = 32u     /* keep U and V in factored form on the handle for utv_solve_rhs */
};

/* Parameters of randUTV(A, q, n_b) (fig:alg_utv) and Compute_rank. */
typedef struct {
  int64_t block;        /* n_b >= 1; this build supports n_b <= 256 (UTV_ERR_UNSUPPORTED above) */
  int32_t power_iters;  /* q >= 0 ("q=1 or q=2 is sufficient") */
  double tau;           /* rank tolerance in [0, 1): r = first j with T_jj <= tau * max_l T_ll (R10) */
  uint64_t seed;        /* key of the Philox4x32-10 Gaussian sketch (R6) */
  uint32_t flags;       /* UTV_WANT_* bits */
} utv_opts;

/* Create a handle bound to CUDA device `device`; `stream` is a cudaStream_t (NULL = the
 * legacy default stream).  Returns UTV_ERR_CUDA if the device is unusable. */
utv_status utv_create(utv_handle* handle, int device, void* stream);

/*
 * Multi-GPU handles: one rank per GPU, 1D block-cyclic columns (block n_b = opts->block,
 * block j on rank j mod P).  With such a handle utv_lstsq takes A = THIS RANK's shard: its column
 * blocks packed in order (m x utv_dist_local_cols(n, n_b, P, rank), lda >= m, device memory) and
 * n = the GLOBAL column count (the shard is overwritten by this rank's column blocks of T, with
 * Sigma on the diagonal blocks it owns); B (m x k, device) is replicated on every rank and overwritten by
 * U^T B; X (n x k, device) is written, identical on every rank; *rank is identical on every rank.
 * All ranks must make the same calls with the same m, n, k, opts (collectives in lock step).
 * Fast option with factored V only (UTV_NULLIFY_T12 / UTV_EXPLICIT_V -> UTV_ERR_UNSUPPORTED);
 * utv_factor on such a handle: A = the rank's shard (-> its shard of T), V (if non-NULL) = the rank's
 * CONTIGUOUS row block of V, rows [p ceil(n/P), min(n, (p+1) ceil(n/P))) x n columns (device,
 * ldv >= its row count), B replicated -> U^T B; U (UTV_WANT_U), UTV_NULLIFY_T12 and
 * UTV_HOST_STREAMED -> UTV_ERR_UNSUPPORTED.  utv_solve on such a handle: T = the rank's shard of T
 * (block-cyclic with the block size of the handle's last utv_factor / utv_lstsq), V = its row block,
 * C replicated; X (n x k) is written, identical on every rank.  In utv_lstsq, with UTV_HOST_STREAMED the shard A is
 * in HOST memory (pinned, or registered for the call) and is streamed through the rank's device
 * (out-of-core x multi-GPU, SURVEY 8(e) x 8(f) #1; the device budget is per handle); B, X stay on
 * the device.
 * Failures: the ranks first agree on the call (one AllReduce of a flag after every rank has checked
 * its arguments and reserved its device memory), so a rank-local argument / allocation error fails
 * the call on EVERY rank (the peers get UTV_ERR_ARG) and the handle stays usable; NaN / Inf and
 * Jacobi failures are AllReduce-d as well (every rank returns UTV_ERR_NUMERICAL).  A later failure
 * (CUDA error, an NCCL asynchronous error, or no progress for UTV_COMM_TIMEOUT_S seconds, default
 * 3600) aborts the communicator (ncclCommAbort, which ends the rank's in-flight collectives) and
 * returns UTV_ERR_NCCL / UTV_ERR_CUDA; such a handle must be destroyed.
 */
/* NCCL unique id (128 bytes) for utv_create_dist; call on one rank and share it (e.g. through
 * torch.distributed).  libnccl.so.2 is loaded at run time; UTV_ERR_NCCL if it is unavailable. */
utv_status utv_get_unique_id(void* nccl_uid);

/* One process per GPU: rank `rank` of `nranks`, NCCL communicator from nccl_uid (ncclCommInitRank
 * on `device`; collective with the other ranks). */
utv_status utv_create_dist(utv_handle* handle, int device, void* stream, const void* nccl_uid,
                           int nranks, int rank);

/* One process, several ranks (one host thread per handle): handles[r] is rank r of an in-process
 * group on devices[r] with streams[r] (NULL = legacy default streams).  Collectives rendezvous on
 * the host and combine the peers' device buffers in rank order; each handle must be driven by its
 * own thread.  If one rank's call fails, its peers' calls return UTV_ERR_NCCL instead of waiting
 * forever, and the group stays unusable (destroy it).  Destroy each handle with utv_destroy. */
utv_status utv_create_local_group(utv_handle* handles, int nranks, const int* devices,
                                  void* const* streams);

/* A caller-supplied communicator ("bring your own": MPI, gloo through torch.distributed, ...) for
 * the same multi-GPU algorithm.  Every callback is invoked on the calling host thread in the rank's
 * program order (the same order on every rank); buffers are device pointers on the handle's device
 * and `stream` (a cudaStream_t) orders them: the callback must make its result visible in stream
 * order (e.g. synchronise the stream, exchange, copy back) and return 0, or non-zero on failure
 * (the call then fails with UTV_ERR_NCCL).  allreduce_sum: in-place elementwise sum of `count`
 * doubles over the ranks, the SAME result on every rank; broadcast: `count` doubles from `root`;
 * allgather: recv[r * count + i] = send of rank r.  abort (may be NULL) is called when this rank
 * fails inside the method's collectives, so that the peers stop waiting.  `ops` is copied. */
typedef struct {
  int (*allreduce_sum)(void* ctx, double* buf, int64_t count, void* stream);
  int (*broadcast)(void* ctx, double* buf, int64_t count, int root, void* stream);
  int (*allgather)(void* ctx, const double* send, double* recv, int64_t count, void* stream);
  void (*abort)(void* ctx);
  void* ctx;
} utv_comm_ops;
utv_status utv_create_with_comm(utv_handle* handle, int device, void* stream, int nranks, int rank,
                                const utv_comm_ops* ops);

/* Number of columns of rank `rank`'s shard of an n-column matrix (block-cyclic, block `block`). */
int64_t utv_dist_local_cols(int64_t n, int64_t block, int nranks, int rank);

/* Release the handle and its workspace (synchronises its stream).  NULL is accepted. */
utv_status utv_destroy(utv_handle handle);

/* Message describing the last non-OK status on this handle ("" if none). */
const char* utv_last_error(utv_handle handle);

/* Change the stream of a handle (cudaStream_t). */
utv_status utv_set_stream(utv_handle handle, void* stream);

/* Wait for all work enqueued on the handle's stream. */
utv_status utv_synchronize(utv_handle handle);

/*
 * randUTV: A V = U T (eq:UTVdef P:467-473), the blocked algorithm of fig:alg_utv
 * with the readings R1 (the right update covers all rows), R3, R5, R13.
 *   A (m x n, m >= n, lda >= m)  in: the matrix; out: T, upper trapezoidal, strictly-lower
 *                                 part exactly 0, each n_b x n_b diagonal block diagonal with
 *                                 non-negative, non-increasing entries (SVD of the block).
 *   V (n x n, ldv >= n)           out if non-NULL: the orthogonal right factor.
 *   U (m x m, ldu >= m)           out only if non-NULL and opts->flags & UTV_WANT_U.
 *   B (m x k, ldb >= m)           if non-NULL and k > 0: overwritten by C = U^T B, applied on
 *                                 the fly (v23t).
 *   rank                          if non-NULL: r for opts->tau (R10); this reads r back to the
 *                                 host (one synchronisation).
 * opts->flags & UTV_NULLIFY_T12: after Compute_rank, Nullify_top_right_part_of_T
 * (fig:alg_nullify_t12) zeroes T(0:r, r:n) by an RZ sweep (blocked, bottom-up, n_b
 * rows at a time; reading R19) whose reflectors are also applied to V; T(0:r, 0:r) stays upper
 * triangular but its diagonal blocks are no longer diagonal.  r is computed even if rank is NULL.
 */
utv_status utv_factor(utv_handle handle, int64_t m, int64_t n, double* A, int64_t lda, double* V,
                      int64_t ldv, double* U, int64_t ldu, double* B, int64_t ldb, int64_t k,
                      const utv_opts* opts, int64_t* rank);

/*
 * x_simple = V(:, 1:r) T11^{-1} U_1^T b (eq:simplesoln P:894-901), with C = U^T B from
 * utv_factor:  X (n x k, ldx >= n) = V(:, 0:r) * T(0:r, 0:r)^{-1} * C(0:r, :).
 * T (ldt >= m) is read-only (upper triangular in its leading r x r block); r == 0 -> X = 0.
 */
utv_status utv_solve(utv_handle handle, int64_t m, int64_t n, int64_t r, const double* T,
                     int64_t ldt, const double* V, int64_t ldv, const double* C, int64_t ldc,
                     int64_t k, double* X, int64_t ldx);

/*
 * Reuse of a factorization for a new right-hand side (the reuse that the paper's
 * v23t "cannot" offer, without the m x m explicit U of v21t).
 * A utv_factor or utv_lstsq call with opts->flags & UTV_KEEP_FACTORS leaves on the handle every
 * step's block reflectors (W_U, T_U), (W_V, T_V) and the small SVD factors U_s, V_s -- about
 * m n doubles (sum of the m' x b panels) + n^2 / 2 -- so that
 *   U = Q_U,1 ... Q_U,s blockdiag(U_s,i),   V = Q_V,1 ... Q_V,s blockdiag(V_s,i)
 * can be applied later.  Supported: single-GPU in-core calls with DEVICE A (T stays in the
 * caller's A), and multi-GPU handles (T stays in each rank's shard); UTV_NULLIFY_T12,
 * UTV_HOST_STREAMED, host A and wide A (m < n) with UTV_KEEP_FACTORS -> UTV_ERR_UNSUPPORTED.
 * The factors stay valid until the next UTV_KEEP_FACTORS call or utv_destroy.
 *
 * utv_solve_rhs: X (n x k, ldx >= n) = V(:, 0:r) T(0:r, 0:r)^{-1} (U^T B)(0:r, :) for a NEW B
 * (m x k, ldb >= m; overwritten by U^T B), with r, m, n those of the kept factorization (m, n
 * must match: UTV_ERR_SHAPE).  T (ldt) is the T that factorization left in A (the rank's shard
 * on a multi-GPU handle; B and X are then replicated on every rank).  *rank (if non-NULL) = r.
 * UTV_ERR_ARG if no factorization was kept.  No host synchronisation (multi-GPU: one per block of
 * the distributed triangular solve).
 */
utv_status utv_solve_rhs(utv_handle handle, int64_t m, int64_t n, int64_t k, const double* T,
                         int64_t ldt, double* B, int64_t ldb, double* X, int64_t ldx,
                         int64_t* rank);

/*
 * Solve_linear_system, fast option (fig:alg_axb P:1075-1108 without the Nullify line;
 * "Fast option" P:1114-1121; v34s): factor + Compute_rank + solve.  A and B are consumed
 * (overwritten by T and U^T B); X (n x k) written; *rank = r.  V is not formed: the handle keeps
 * every step's block reflector (W_V, T_V) and V_s (about n^2/2 doubles instead of n^2) and
 * applies V = Q_1 ... Q_s blockdiag(V_s) to [z; 0] (saves the 2 n^3 flops of
 * accumulating V); opts->flags & UTV_EXPLICIT_V accumulates V explicitly instead.  opts->flags & UTV_NULLIFY_T12 runs
 * Nullify_top_right_part_of_T (fig:alg_nullify_t12, fig:alg_axb line 3 P:1087) after the rank
 * is known, so X is the minimum-norm solution pinv(A_r) B of the rank-r approximation (the
 * factored V then also keeps the nullify reflectors, about r (n - r) more doubles).  A, B and X may be HOST pointers (pageable or pinned): they are then staged
 * through device buffers inside the call (the end-to-end path); host A and B are inputs only
 * (left unchanged), a host X is written and the call returns after X has landed.
 * Wide A (m < n, reading R21): randUTV of the tall A^T (A^T V' = U' T') and
 * X = U'(:, 0:r) T'11^{-T} V'(:, 0:r)^T B, evaluated without forming U' as
 * A^T V'(:, 0:r) T'11^{-1} T'11^{-T} V'(:, 0:r)^T B with V' factored (workspace about
 * n m + 3.5 m^2 doubles);
 * A and B are left unchanged; single-GPU in-core only (multi-GPU / UTV_HOST_STREAMED ->
 * UTV_ERR_SHAPE, UTV_NULLIFY_T12 -> UTV_ERR_UNSUPPORTED).
 */
utv_status utv_lstsq(utv_handle handle, int64_t m, int64_t n, int64_t k, double* A, int64_t lda,
                     double* B, int64_t ldb, double* X, int64_t ldx, const utv_opts* opts,
                     int64_t* rank);

/*
 * Out-of-core mode (opts->flags & UTV_HOST_STREAMED; the paper's out-of-core regime, P:1580-1675,
 * P:1790-1824) -- utv_lstsq only, fast option with factored V (UTV_NULLIFY_T12 /
 * UTV_EXPLICIT_V -> UTV_ERR_UNSUPPORTED).  A must be a HOST pointer (pinned or pageable; pageable
 * memory is registered with cudaHostRegister for the duration of the call) and is OVERWRITTEN by T
 * there.  B and X may be host or device pointers (a device B is overwritten by U^T B, a host B is
 * left unchanged).  HBM holds the workspace, the factored V (about n^2/2 doubles), a ring of staging
 * chunks and as many trailing column blocks as the device budget allows; the other column blocks
 * are streamed host <-> device on two copy streams, overlapped with the GEMMs (2q+2 reads and one
 * write of the trailing columns per step).  UTV_ERR_ALLOC if the budget cannot hold the fixed part.
 */
/* Device-memory budget in bytes for UTV_HOST_STREAMED calls on this handle (workspace + factored V
 * + staging + resident blocks); 0 (default) = free HBM at call time minus 1 GiB. */
utv_status utv_set_device_budget(utv_handle handle, int64_t bytes);

/* Host-link traffic of the last UTV_HOST_STREAMED call: bytes copied host->device and
 * device->host, and the number of trailing columns that were kept resident in HBM. */
utv_status utv_stream_stats(utv_handle handle, int64_t* h2d_bytes, int64_t* d2h_bytes,
                            int64_t* resident_cols);

/* Library version string, e.g. "utv-b200 0.1 sm_100a". */
const char* utv_version(void);

#ifdef __cplusplus
}
#endif

#endif /* UTV_H_ */

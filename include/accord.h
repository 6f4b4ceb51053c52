/*
 * accord.h — C ABI of the B200-native ACCORD-FBS hot path (libaccord.so).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md, arXiv 2412.11554):
 *   the ACCORD estimator  argmin_Omega  -log det Omega_D + 1/2 tr(Omega^T Omega S)
 *                                       + lambda ||Omega||_1          (Eq. 3.2)
 *   with S = X^T X / n never formed, by Algorithm 1 (ACCORD-FBS,
 *   PAPER.md:246-263): per outer iteration t
 *     grad g = Omega S = (1/n)(Omega X^T) X            (two-step gradient)
 *     for tau = tau0, beta tau0, ...:                  (backtracking)
 *        Omega+ = prox_{tau h}(Omega - tau grad g)      (closed form Eq. 3.5)
 *     until  ||(Omega+ - Omega) X^T||_F^2 / n <= ||Omega+ - Omega||_F^2 / tau   or  tau <= 1/L
 *                                                      (reading R8)
 *   Omega is asymmetric, the l1 norm covers the diagonal (Eq. 3.2).
 *
 * Data layout and sharding: rank k owns the contiguous row block
 * [row_begin, row_end) of Omega (rows separate, and Alg. 1
 * couples them only through tau_t). X is either replicated on every rank
 * (default; collectives then carry only the per-trial line-search sums, 8
 * doubles, and the export gather) or, for X beyond one GPU's memory, sharded
 * by variables (x_sharded = 1: rank k holds the columns [row_begin, row_end)
 * of X, and every pass that needs all of X (gradient GEMM, candidate refine,
 * SpMM) visits the slabs in a ring, the 1DMM scheme of Alg. 2,
 * PAPER.md:326-356).
 *
 * Conventions for every call:
 *   - No C++ exception crosses the ABI. Every call returns an accord_status;
 *     ACCORD_OK == 0. On failure accord_last_error(ctx) describes it.
 *   - A context is not thread-safe: one context per host thread (per rank).
 *   - All device work is ordered on the stream given at create time. Calls
 *     return after the host has synchronized with that stream unless noted.
 *   - The library owns all device memory it allocates (cudaMalloc at create
 *     time; the candidate pool grows on demand, see accord_step).
 */
#ifndef ACCORD_H_
#define ACCORD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACCORD_ABI_VERSION 4

typedef enum {
  ACCORD_OK = 0,
  ACCORD_E_INVALID = 1,      /* bad argument (n<1, p<1, lambda<0, tau0<=0, beta not in (0,1], bad row range, non-finite X, ...) */
  ACCORD_E_CUDA = 2,         /* CUDA runtime error (message in accord_last_error) */
  ACCORD_E_NCCL = 3,         /* NCCL error or NCCL unavailable */
  ACCORD_E_CAPACITY = 4,     /* a caller-provided output buffer is too small; *nnz_out holds the size needed */
  ACCORD_E_NUMERIC = 5,      /* non-finite objective / sums during a step (iteration index in the message) */
  ACCORD_E_DOMAIN = 6,       /* nonpositive diagonal (Omega outside dom f) */
  ACCORD_E_NOMEM = 7,        /* device allocation failed */
  ACCORD_E_UNSUPPORTED = 8,  /* request not supported on this device / build (e.g. tcgen05 GEMM off sm_100) */
  ACCORD_E_COMM = 9          /* host-callback communicator reported failure */
} accord_status;

typedef enum {
  ACCORD_LAYOUT_SAMPLES_ROW_MAJOR = 0,   /* X is n x p row-major: X[m*ldx + j], rows = samples */
  ACCORD_LAYOUT_VARIABLES_ROW_MAJOR = 1  /* X^T is p x n row-major: Xt[j*ldx + m] (X stored column-major) */
} accord_layout;

typedef enum {
  ACCORD_F32 = 0,   /* values and X in float; reductions in double */
  ACCORD_F64 = 1    /* everything in double (CUDA cores; tcgen05 has no f64 kind) */
} accord_dtype;

typedef enum {
  ACCORD_GEMM_AUTO = 0,         /* F32 on sm_100: the certified filter with ADAPTIVE operands -- bf16
                                   while the candidate set is large (|C| / p > 48, the first
                                   iterations), then int8 (I8_FILTER's GEMM); X sharded: BF16_FILTER.
                                   Otherwise SIMT. F64: SIMT. info.gemm reports BF16_FILTER, or
                                   I8_FILTER once an int8 GEMM ran (gemm_launches_i8). */
  ACCORD_GEMM_BF16X3 = 1,       /* tcgen05 GEMM, split-bf16 operands, 3 MMAs (hi*hi + hi*lo + lo*hi),
                                   fp32 TMEM accumulator; candidate values taken from the tensor cores
                                   (~2^-16 relative product error) */
  ACCORD_GEMM_SIMT = 2,         /* CUDA-core GEMM in the context dtype (reference path; the only F64 path) */
  ACCORD_GEMM_BF16_FILTER = 3,  /* tcgen05 single-pass bf16 GEMM as a certified filter: emits (i,k) when
                                   |G~_ik| > lambda - delta_ik (delta_ik a rigorous bound on the bf16
                                   rounding + fp32 accumulation error), then every candidate value is
                                   recomputed exactly (float64 accumulation) by an SDDMM */
  ACCORD_GEMM_I8_FILTER = 4     /* the same certified filter on int8 operands (tcgen05 kind::i8, exact
                                   s32 accumulation, twice the bf16 MMA rate): Y rows quantised with a
                                   per-row scale, X^T with a per-256-variable block scale; the bound is
                                   the quantisation error alone (Cauchy-Schwarz on the actual error
                                   vectors); values recomputed exactly by the SDDMM. F32, sm_100,
                                   X replicated (not x_sharded). Every GEMM in int8 (AUTO switches
                                   adaptively). DESIGN.md §5. */
} accord_gemm;

typedef enum {
  ACCORD_COMM_NONE = 0,   /* world must be 1 */
  ACCORD_COMM_NCCL = 1,   /* NCCL communicator built from nccl_id (all ranks pass the same 128-byte id) */
  ACCORD_COMM_HOST = 2    /* host callback: allreduce(user, buf, count) must sum buf across ranks in place */
} accord_comm;

typedef enum {
  ACCORD_SCOPE_LOCAL = 0,   /* this rank's row block; row_ptr indexes local rows */
  ACCORD_SCOPE_GATHER = 1   /* all p rows (collective: every rank must call) */
} accord_scope;

/* Sum `count` doubles across all ranks in place. Return 0 on success. */
typedef int (*accord_allreduce_fn)(void* user, double* buf, int32_t count);
/* Gather variable-size byte blocks from all ranks (rank order) into `out`
 * (host memory). counts[r] is filled by the callee with rank r's byte count
 * when out == NULL. Return 0 on success. Used only by ACCORD_SCOPE_GATHER
 * with ACCORD_COMM_HOST. */
typedef int (*accord_allgatherv_fn)(void* user, const void* in, int64_t in_bytes,
                                    void* out, int64_t* counts);
/* Ring exchange of host buffers (x_sharded with ACCORD_COMM_HOST): send
 * send_bytes from `send` to rank dst and receive recv_bytes from rank src into
 * `recv` (all ranks call together). Return 0 on success. */
typedef int (*accord_sendrecv_fn)(void* user, const void* send, int64_t send_bytes, int32_t dst,
                                  void* recv, int64_t recv_bytes, int32_t src);

typedef struct {
  int32_t abi_version;      /* must be ACCORD_ABI_VERSION */
  int32_t device;           /* CUDA device ordinal, or -1 = current device */
  int64_t n, p;             /* samples, variables; n >= 1, p >= 1 */
  const void* X;            /* data (host or device, see x_on_device); used as given:
                               the caller centers it (reading R12). Copied at
                               create; the caller keeps ownership. */
  int64_t ldx;              /* leading dimension in elements (0 = dense: p for SAMPLES, n for VARIABLES) */
  int32_t layout;           /* accord_layout */
  int32_t dtype;            /* accord_dtype of X and of the iterate */
  int32_t x_on_device;      /* 1: X is a device pointer on `device`; 0: host pointer */
  int32_t gemm;             /* accord_gemm */
  double lambda;            /* >= 0, penalty on every entry incl. the diagonal (Eq. 3.2) */
  double tau0;              /* > 0, initial step of every outer iteration (Alg. 1) */
  double beta;              /* in (0, 1]; 1 = fixed step tau0 (Alg. 1, Thm 3.3 case i) */
  double inv_L;             /* > 0: 1/L given by the caller; 0: computed on device
                               (Lanczos on the samples' Gram X X^T / n, whose top eigenvalue
                               is sigma_max(S); inflated by 2e-3, SPEC.md:85:
                               overestimating L is safe) */
  int64_t row_begin, row_end;  /* this rank's rows [row_begin, row_end) of Omega; 0 <= begin < end <= p */
  int32_t rank, world;      /* 0 <= rank < world */
  int32_t comm;             /* accord_comm */
  const uint8_t* nccl_id;   /* ACCORD_COMM_NCCL: 128-byte ncclUniqueId (same on all ranks) */
  accord_allreduce_fn allreduce;     /* ACCORD_COMM_HOST */
  accord_allgatherv_fn allgatherv;   /* ACCORD_COMM_HOST (export gather); may be NULL */
  void* comm_user;                   /* passed to the callbacks */
  void* stream;             /* cudaStream_t to order all work on (NULL = legacy default stream) */
  int64_t cand_capacity;    /* initial candidate-pool capacity in entries (0 = auto); grows on demand */
  int32_t x_sharded;        /* 0: X holds all p variables (replicated on every rank).
                               1: X holds only this rank's variables [row_begin, row_end)
                               (n x p_k samples-major or p_k x n variables-major); the
                               rank blocks must tile [0, p) in rank order (with a tensor-core
                               GEMM each starting at a multiple of 256, the GEMM tile).
                               Collective passes over X run as a ring
                               (Alg. 2): NCCL send/recv on a split
                               communicator, or `sendrecv` with ACCORD_COMM_HOST. */
  accord_sendrecv_fn sendrecv;       /* ACCORD_COMM_HOST with x_sharded */
  void* workspace;          /* NULL: the library cudaMallocs its device memory. Else a
                               caller-owned device buffer on `device` (e.g. a torch
                               tensor) of workspace_bytes bytes, at least
                               accord_workspace_size(): every device buffer of the
                               context is carved out of it and the library never calls
                               cudaMalloc. A pool overflow grows inside the workspace;
                               when it does not fit, the call returns ACCORD_E_CAPACITY
                               (nothing committed; the message gives the bytes needed).
                               The caller frees it after accord_destroy. */
  size_t workspace_bytes;
} accord_init_params;

/* Per accepted outer iteration (one element per iteration of accord_step). */
typedef struct {
  double tau;         /* accepted step tau_t */
  double f;           /* f(Omega^{(t+1)}) (Eq. 3.2), global */
  double logdet_part; /* -sum_i log omega_ii */
  double g_part;      /* ||Omega X^T||_F^2 / (2n) */
  double l1_part;     /* lambda * ||Omega||_1 */
  double delta_fro;   /* ||Omega^{(t+1)} - Omega^{(t)}||_F */
  double ls_lhs;      /* ||Delta X^T||_F^2 / n  of the accepted trial */
  double ls_rhs;      /* ||Delta||_F^2 / tau    of the accepted trial */
  int64_t nnz;        /* nnz(Omega^{(t+1)}) incl. diagonal, global */
  int64_t n_cand;     /* |C| = |diag U supp(Omega^{(t)}) U {|G| > lambda}|, global */
  int32_t trials;     /* line-search trials (>= 1) */
  int32_t floor_hit;  /* 1 if accepted because tau <= 1/L */
  float ms_gemm;      /* device time of the gradient GEMM + fused epilogue (CUDA events) */
  float ms_finalize;  /* candidate scan / scatter / row sort */
  float ms_refine;    /* exact SDDMM of the candidate values (BF16_FILTER), else 0 */
  float ms_prox;      /* prox kernels, all trials */
  float ms_spmm;      /* SpMM kernels, all trials */
  float ms_reduce;    /* reductions + collectives + host decision, all trials */
  float ms_total;     /* whole iteration */
  int64_t max_row_cand; /* longest candidate row of this rank (diagnostic) */
  int32_t gemm_i8;      /* 1 if this iteration's gradient GEMM ran on int8 operands (I8_FILTER) */
  int32_t pad_;
} accord_iter_stats;

typedef struct {
  int64_t n, p, row_begin, row_end, ldk;
  double L, inv_L, lambda, tau0, beta;
  int32_t dtype, gemm;          /* resolved accord_gemm actually used */
  int32_t sm_count, cc_major, cc_minor;
  int64_t iterations;           /* accepted iterations so far */
  int64_t nnz_local;            /* nnz of this rank's rows of the current Omega */
  int64_t cand_capacity;        /* current pool capacity (entries) */
  int64_t kernel_launches;      /* cumulative count of library kernel launches */
  int64_t gemm_launches;        /* cumulative count of gradient-GEMM launches */
  double f;                     /* current objective (global) */
  size_t device_bytes;          /* device memory held by the context */
  size_t workspace_bytes;       /* caller workspace size (0: library-allocated memory) */
  size_t workspace_high;        /* high-water mark of the workspace in use */
  int64_t mirrored_sent;        /* candidate positions this rank sent to their row's owner in the
                                   symmetric first GEMM across ranks (cumulative, diagnostic) */
  int64_t gemm_launches_i8;     /* of gemm_launches, those on int8 operands */
} accord_info;

typedef struct accord_ctx accord_ctx;

/* Fill *prm with defaults (abi_version, device=-1, beta=0.5, tau0=0.5, world=1, ...). */
void accord_default_params(accord_init_params* prm);

/* Device bytes accord_create needs for *prm when the caller owns the memory
 * (prm->workspace): X^T and its bf16 copy, Y x 2 and its bf16 copies, the
 * per-row state, and the candidate pool / C / Omega arrays at the pool
 * capacity (prm->cand_capacity, or the default ~512 candidates per row, the
 * first iteration's demand at config 5) -- the inputs of Alg. 1
 * laid out as DESIGN.md §6 states -- plus the transient
 * staging of a host X or the Lanczos vectors of L. Pure: validates *prm (same
 * errors as accord_create) and touches no device. An upper bound for the
 * AUTO GEMM kind and balanced sharded slabs; later calls that allocate
 * temporaries (export GATHER, transformed exports, path, refit, lambda_max)
 * need free workspace beyond it. */
accord_status accord_workspace_size(const accord_init_params* prm, size_t* bytes);

/* Create a solver context: validates, copies X to the device (variable-major,
 * zero-padded to a multiple of 64 samples), builds GEMM operand copies,
 * computes L if inv_L == 0, sets Omega^{(0)} = I
 * and Y^{(0)} = rows of X^T. Collective when world > 1 (NCCL init).
 * Errors: ACCORD_E_INVALID (arguments; non-finite X with the first offending
 * (row, col) in the message), ACCORD_E_CUDA, ACCORD_E_NOMEM, ACCORD_E_NCCL,
 * ACCORD_E_UNSUPPORTED. On error *out is NULL. */
accord_status accord_create(accord_ctx** out, const accord_init_params* prm);

/* Run `iters` outer iterations of Algorithm 1. Collective:
 * all ranks call with the same iters. stats may be NULL, else it receives
 * `iters` records. One host synchronization per line-search trial (the
 * decision needs the global sums). If the candidate pool overflows, the
 * library grows it and redoes the iteration (nothing is committed before a
 * trial is accepted). Errors: ACCORD_E_NUMERIC, ACCORD_E_CUDA, ACCORD_E_NCCL,
 * ACCORD_E_COMM, ACCORD_E_NOMEM. Not converging is not an error. */
accord_status accord_step(accord_ctx* ctx, int32_t iters, accord_iter_stats* stats);

/* Objective of the current iterate (global; collective when world > 1).
 * parts (may be NULL) receives {-sum log omega_ii, ||Omega X^T||^2/(2n),
 * lambda ||Omega||_1}. */
accord_status accord_objective(accord_ctx* ctx, double* f, double* parts);

/* Export Omega as CSR with columns sorted per row, the diagonal always
 * present and off-diagonal zeros absent. Values are in the context dtype.
 * Two-call convention: with row_ptr == NULL (or capacity too small) only
 * *nnz_out is written (ACCORD_E_CAPACITY if buffers were given but too
 * small). row_ptr has (rows + 1) entries, rows = row_end - row_begin for
 * LOCAL and p for GATHER; global column indices. on_device = 1 means the
 * buffers are device pointers. GATHER is collective. */
accord_status accord_export_csr(accord_ctx* ctx, int32_t scope, int64_t* row_ptr,
                                int32_t* col, void* val, int64_t capacity,
                                int64_t* nnz_out, int32_t on_device);

typedef enum {
  ACCORD_EXPORT_OMEGA = 0,  /* Omega-hat itself (same as accord_export_csr) */
  ACCORD_EXPORT_THETA = 1,  /* Theta-hat = T^{-1}(Omega-hat) = Omega_D Omega: theta_ij = omega_ii omega_ij
                               (PAPER.md:151-156, :166); same CSR structure as Omega */
  ACCORD_EXPORT_PCORR = 2   /* partial correlations rho-hat_ij = -1/2 (omega_ij / omega_jj + omega_ji / omega_ii),
                               i != j: symmetric, stored on supp(Omega) U supp(Omega^T)
                               off the diagonal (no diagonal entries) */
} accord_export_kind;

/* Post-processing of the current estimate on the device (SURVEY.md §8(f)
 * NEXT(4)). Same conventions as accord_export_csr (two-call size query,
 * sorted columns, rows = local block for LOCAL and p for GATHER, buffers
 * host or device per on_device); values in the context dtype, computed in
 * double. PCORR needs the transpose, so it gathers Omega (collective for any
 * scope when world > 1); THETA with LOCAL scope is rank-local. Each call
 * recomputes (a size query costs the same as the export). Errors:
 * ACCORD_E_DOMAIN (a diagonal entry <= 0), ACCORD_E_CAPACITY, ACCORD_E_INVALID
 * (bad kind or scope), ACCORD_E_CUDA, ACCORD_E_NCCL, ACCORD_E_COMM. */
accord_status accord_export_transformed(accord_ctx* ctx, int32_t kind, int32_t scope,
                                        int64_t* row_ptr, int32_t* col, void* val,
                                        int64_t capacity, int64_t* nnz_out, int32_t on_device);

/* Warm start / resume: replace this rank's rows of Omega by a host CSR
 * (local rows, global sorted columns, context dtype). Validates a positive
 * stored diagonal (ACCORD_E_DOMAIN) and recomputes Y = Omega X^T.
 * Collective when world > 1 (recomputes the global objective). */
accord_status accord_set_omega_csr(accord_ctx* ctx, const int64_t* row_ptr,
                                   const int32_t* col, const void* val, int64_t nnz);

/* Change lambda (keeps Omega: warm start for a path).
 * Collective (recomputes the global objective). */
accord_status accord_set_lambda(accord_ctx* ctx, double lambda);

/* Bias-correction refit, Eq. (3.8): freeze S_hat = the
 * support of the current estimate (diagonal included) and continue
 * Algorithm 1 with penalty phi*lambda on S_hat and +inf (entries fixed at 0)
 * off it; 0 <= phi <= 1. The gradient is then needed only on S_hat and comes
 * from the SDDMM (no GEMM). Collective. */
accord_status accord_refit(accord_ctx* ctx, double phi);

/* Run Algorithm 1 until ||Omega^(t+1) - Omega^(t)||_F < tol or max_iter
 * iterations (reading R13). Collective. */
accord_status accord_solve(accord_ctx* ctx, int32_t max_iter, double tol, int32_t* iters_done,
                           accord_iter_stats* last);

/* KKT certificate (Eq. 3.3; supp. :985-997) of the current
 * iterate: max over all entries of | -1/omega_ii + [Omega S]_ii + lambda |,
 * | [Omega S]_ij + lambda sign omega_ij | (nonzero), max(0, |[Omega S]_ij| -
 * lambda) (zero). Entries outside the candidate set have |[Omega S]_ij| <=
 * lambda by the filter's certificate and contribute 0; under a refit, entries
 * off S_hat are skipped. Costs one gradient pass. Collective. */
accord_status accord_kkt_residual(accord_ctx* ctx, double* kkt);

/* Regularisation path with warm starts and epBIC selection (Eq. 3.7,
 * PAPER.md:360-377): for j = 0..k-1 (lambdas in the given order, normally
 * descending) set lambda_j, solve to tol / max_iter from the previous
 * estimate, record epBIC_j = 2n(-log det Omega_D + ||Omega X^T||^2/2n)
 * + k_j (log n + 4 gamma log p), k_j = number of nonzero off-diagonal
 * entries, and the iterations used. On return the context holds the
 * epBIC-minimising estimate and its lambda; *best = its index. Any output
 * pointer may be NULL. Collective. */
accord_status accord_path(accord_ctx* ctx, const double* lambdas, int32_t k, int32_t max_iter,
                          double tol, double gamma, double* epbic, int64_t* nnz_off,
                          int32_t* iters, int32_t* best);

/* lambda_max = max_{i != k} |S_ik|, S = X^T X / n, the top
 * of the descending lambda grid of a path (§5.3, "an evenly spaced
 * grid of lambda's in logarithmic scale"; SPEC.md
 * lambda_grid). BF16_FILTER: the tensor-core gradient
 * GEMM at Omega = I in max-reduce mode bounds it from below, a candidate pass
 * at that bound keeps the maximiser, and the float64 refine makes the value
 * exact for the f32 data; other kinds: float64 dot products on CUDA cores.
 * Does not change the iterate. Collective. Errors: ACCORD_E_NUMERIC when
 * lambda_max is 0 (all-zero or exactly uncorrelated data). */
accord_status accord_lambda_max(accord_ctx* ctx, double* lambda_max);

/* lambdas[j] = lambda_max * ratio^(j / (k-1)), j = 0..k-1: k log-evenly
 * spaced values from lambda_max down to ratio * lambda_max (descending, the
 * order accord_path expects). k >= 1, 0 < ratio < 1. Collective. */
accord_status accord_lambda_grid(accord_ctx* ctx, int32_t k, double ratio, double* lambdas);

/* DIAGNOSTIC (filter certification): run the gradient GEMM +
 * fused epilogue + candidate finalize of the NEXT iteration exactly as
 * accord_step would (same tiles, same bf16 operands, same thresholds, the
 * symmetric schedule at Omega = I included), and additionally write the raw
 * fp32 tensor-core accumulator acc_ik (~ n G_ik) of every (local row i,
 * column k) to `acc` (device, row-major, ld >= p floats per row; every entry
 * of the p_k x p block is written). Also returns (each may be NULL): y
 * (device, p_k x n, row stride ldy) = the f32 Y = Omega X^T the GEMM's bf16 A
 * operand was rounded from; row_ab (host, 2 p_k floats) = ||y_i - bf16(y_i)||
 * then ||y_i||; col_sd (host, 2 p floats, interleaved) = (||x_k|| +
 * ||x_k - bf16(x_k)||, ||x_k - bf16(x_k)||); gamma = the accumulation factor;
 * and the candidate set C (host CSR, sorted columns, two-call convention as
 * accord_export_csr: *n_cand = |C|, ACCORD_E_CAPACITY if capacity < |C|).
 * The iterate is not changed. BF16_FILTER contexts only (else
 * ACCORD_E_UNSUPPORTED). */
accord_status accord_filter_audit(accord_ctx* ctx, float* acc, int64_t ld, float* y, int64_t ldy,
                                  float* row_ab, float* col_sd, double* gamma, int64_t* c_ptr,
                                  int32_t* c_col, int64_t capacity, int64_t* n_cand);

/* Per-row line-search summands of the LAST trial evaluated by accord_step
 * (||D_i||^2, ||Delta_i||^2, i = local row indices). For sampled-row parity. */
accord_status accord_row_stats(accord_ctx* ctx, const int64_t* rows, int64_t count,
                               double* d2, double* delta2);

accord_status accord_get_info(accord_ctx* ctx, accord_info* info);

/* 128-byte NCCL unique id for ACCORD_COMM_NCCL (call on one rank, broadcast). */
accord_status accord_nccl_unique_id(uint8_t id[128]);

void accord_destroy(accord_ctx* ctx);
const char* accord_status_string(accord_status s);
const char* accord_last_error(const accord_ctx* ctx);  /* ctx may be NULL: last create error */
int32_t accord_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ACCORD_H_ */

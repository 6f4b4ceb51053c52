// Internal declarations shared by the host driver (api.cpp) and the CUDA
// kernels. Not part of the ABI (include/accord.h is).
#pragma once
#include <cstdint>
#include <cstddef>
#include <functional>
#include <string>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../../include/accord.h"

namespace accord {

constexpr int kKPad = 64;       // samples padded to a multiple of 64 (one 128-B bf16 TMA row)
constexpr int kRowPad = 256;    // operand rows padded to the GEMM tile (M and N)

#ifdef __CUDACC__
// bf16 rounding of the filter GEMM's operands (hi = rn(x)); the filter bound
// uses the residual x - hi of exactly this rounding (col_norms, the SpMM
// epilogues), so the candidate set stays certified for any rounding here.
// ACCORD_BF16_DROP = k (diagnostic builds only) rounds to 7 - k mantissa bits.
#ifndef ACCORD_BF16_DROP
#define ACCORD_BF16_DROP 0
#endif
__device__ __forceinline__ __nv_bfloat16 filter_bf16(float x) {
#if ACCORD_BF16_DROP == 0
  return __float2bfloat16_rn(x);
#else
  constexpr int s = 16 + ACCORD_BF16_DROP;
  uint32_t u = __float_as_uint(x);
  u += ((1u << (s - 1)) - 1) + ((u >> s) & 1u);
  return __ushort_as_bfloat16((unsigned short)((u & ~((1u << s) - 1)) >> 16));
#endif
}
__device__ __forceinline__ __nv_bfloat162 filter_bf16x2(float a, float b) {
#if ACCORD_BF16_DROP == 0
  return __floats2bfloat162_rn(a, b);
#else
  return __halves2bfloat162(filter_bf16(a), filter_bf16(b));
#endif
}
// The X^T operand rounded to 7 - drop mantissa bits (round to nearest even;
// drop = 0: plain bf16). Fewer toggling bits lower the MMAs' energy and so
// raise the power-capped clock; the filter bound uses this very rounding's
// residual, so the candidate set stays certified.
__device__ __forceinline__ __nv_bfloat16 filter_bf16_x(float x, int drop) {
  if (drop == 0) return filter_bf16(x);
  const int s = 16 + drop;
  uint32_t u = __float_as_uint(x);
  u += ((1u << (s - 1)) - 1) + ((u >> s) & 1u);
  return __ushort_as_bfloat16((unsigned short)((u & ~((1u << s) - 1)) >> 16));
}
#endif

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// Kernel attributes (dynamic shared-memory limits) are set once per device and
// call site: `seen` holds one bit per device, set only AFTER the attributes
// were applied, so a concurrent caller can at worst set them twice.
inline int attr_device_bit() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev & 63;
}
inline bool attr_needed(const unsigned long long& seen) {
  return !(seen & (1ull << attr_device_bit()));
}
inline void attr_done(unsigned long long& seen) { seen |= 1ull << attr_device_bit(); }

// ---------------------------------------------------------------------------
// Device-side views of the per-rank state (plain pointers, no ownership).
// ---------------------------------------------------------------------------
struct OmegaView {            // this rank's rows of Omega, CSR, sorted global columns
  const int64_t* ptr;         // [pk + 1]
  const int32_t* col;
  const void* val;            // T
};

struct PoolView {             // candidate pool written by the GEMM epilogue (unsorted)
  int32_t* row;               // local row index
  int32_t* col;               // global column
  void* g;                    // T: [Omega S]_ik
  void* w;                    // T: omega_ik^{(t)} (0 if absent)
  // The pool is handed out in chunks of `chunk` entries: chunk c is
  // [c*chunk, (c+1)*chunk). Each tcgen05 epilogue warp fills a private chunk
  // and takes the next one with one atomicAdd on *chunk_next (no contention on
  // a single cursor, no per-CTA imbalance). The SIMT GEMM uses one chunk of
  // the whole capacity with an atomic cursor in chunk_fill[0].
  int64_t chunk;              // entries per chunk
  int64_t nchunks;            // chunks available
  unsigned int* chunk_next;   // chunks handed out (may exceed nchunks: overflow)
  unsigned long long* chunk_fill;   // [nchunks] entries written into each chunk
  int32_t* row_cnt;           // [pk] entries emitted per row
};

struct EpiParams {            // candidate rule of the fused epilogue
  int64_t pk, p, r0;          // local rows, columns, global index of local row 0
  // columns [col_base, col_end) of this launch; the B operand (X^T rows) holds
  // exactly these, row 0 = column col_base (all p columns unless X is sharded
  // and this is one step of the ring, NEXT(3)); col_base is a multiple of 256
  int64_t col_base, col_end;
  double inv_n;
  double lam_cand;            // emit (i,k) iff k == i, or omega_ik != 0, or |g| > lam_cand
  // BF16_FILTER only: per-entry rigorous error bound of the single-pass bf16
  // product, n*delta_ik = r1_i * s_k + B_i * D_k (see gemm_tc.cu)
  const float* row_A;         // ||y_i - bf16(y_i)||       (current Y buffer)
  const float* row_B;         // ||y_i||
  const float2* col_sd;       // (||x_k|| + ||x_k - bf16(x_k)||, ||x_k - bf16(x_k)||)
  float gamma;                // accumulation-error factor
  // I8_FILTER only: y^_i = row_scale[i] q_i, x^_k = blk_scale[k / 256] q_k
  // (row_A / row_B / col_sd then hold the int8 quantisation errors)
  const float* row_scale;
  const float* blk_scale;
  const int32_t* col_perm;    // I8_FILTER: B row (= G column) k' holds variable col_perm[k']
  int exact_cols;             // 1: re-test tile-test survivors with their own column's bound
  // Omega is exactly I (the first iteration of a solve), so G = X^T X / n is
  // symmetric and each off-diagonal tile pair runs once, its survivors (i,k)
  // emitted also as (k,i) (BF16_FILTER): 1 = one rank, tiles with N-block >=
  // M-block; 2 = several ranks (row blocks on 256-row tiles), the cyclic half
  // of gemm_tc.cu's Sched; mirrored entries of another rank's rows go to the
  // mirror buffer (global row, column) and are sent to their owner
  int sym;
  int mt0, nt;                // sym 2: global row tile of local M-block 0, column tiles
  int32_t* mir_row;           // [mir_cap] global row of a mirrored entry (sym 2)
  int32_t* mir_col;
  unsigned long long* mir_cnt;   // entries written (may exceed mir_cap: overflow)
  int64_t mir_cap;
  // diagnostics / NEXT(2) (nullptr in the product path): audit_acc != NULL
  // writes every raw fp32 accumulator (row-major, audit_ld floats per local
  // row) besides the normal emission; max_out != NULL emits nothing and
  // atomically raises *max_out (float bits) to max_{i != k} (|acc_ik| - n delta)
  float* audit_acc;
  int64_t audit_ld;
  unsigned int* max_out;
};

// ---------------------------------------------------------------------------
// Kernel launchers (kernels.cu, gemm_simt.cu, gemm_tc.cu). All asynchronous
// on `st`; each returns the number of kernel launches issued.
// ---------------------------------------------------------------------------
// X (any layout, f32/f64, device) -> Xt (T, prows x ldk, zero padded). Sets
// *bad to the first non-finite linear index (init it to INT64_MAX).
int launch_load_xt(int dtype, const void* X, int64_t ldx, int layout, int64_t n, int64_t p,
                   void* Xt, int64_t ldk, int64_t prows, unsigned long long* bad,
                   cudaStream_t st);
// Xt f32 -> hi = bf16_rn(x), lo = bf16_rn(x - hi) (rows x ldk)
int launch_split_bf16(const float* src, int64_t elems, __nv_bfloat16* hi,
                      __nv_bfloat16* lo, cudaStream_t st, int drop = 0);

// w = X (X^T u) / n (the samples' Gram operator; its top eigenvalue is L =
// sigma_max(S)) on this rank's Xt (p x ldk). t: p doubles,
// part: nsplit x ldk doubles of scratch. Deterministic.
int launch_gram_apply(int dtype, const void* Xt, int64_t p, int64_t n, int64_t ldk,
                      const double* u, double* t, double* part, int64_t nsplit, double* w,
                      cudaStream_t st);

// Exclusive scan: out[0..N] (out[N] = total) from int32 counts.
int launch_scan_i32(const int32_t* in, int64_t* out, int64_t N, void* tmp, size_t tmp_bytes,
                    cudaStream_t st);
size_t scan_tmp_bytes(int64_t N);

// Finalize the candidate pool into the sorted per-row candidate set C.
int launch_finalize(int dtype, int64_t pk, const PoolView& pool, const int64_t* c_ptr,
                    int32_t* rcur, uint64_t* keys, uint64_t* keys_tmp, int32_t* c_col,
                    void* c_g, void* c_w, int32_t* long_rows, cudaStream_t st,
                    const int64_t* sup_ptr = nullptr, const int32_t* sup_col = nullptr);

// Filter path: supp Omega (its CSR, diagonal included) joins C in the
// finalize: row_cnt += its row lengths before the scan, launch_finalize
// scatters it next to the GEMM's entries (sup_ptr / sup_col), and after the
// row sort one entry per column is kept (cnt: per-row unique counts, optr:
// their scan, col: the columns).
int launch_support_count(int64_t pk, const int64_t* om_ptr, int32_t* row_cnt, cudaStream_t st);
int launch_dedupe(int64_t pk, const int64_t* ptr, const uint64_t* keys, int32_t* cnt,
                  int64_t* optr, int32_t* col, void* scan_tmp, size_t scan_tmp_bytes,
                  cudaStream_t st);

// Sort every CSR row segment of 64-bit keys ascending (warp bitonic for rows
// <= 1024, block bitonic + merge path above). long_rows: int32[rows + 1],
// zeroed by the caller; tmp: scratch of the same size as keys.
int launch_rowsort(int64_t rows, const int64_t* ptr, uint64_t* keys, uint64_t* tmp,
                   int32_t* long_rows, cudaStream_t st);

// NEXT(4) post-processing on the GLOBAL CSR of Omega (postproc.cu):
// d[i] = omega_{i, i + off} for the CSR's rows (bad = 1 if some omega_ii <= 0);
// theta_ij = omega_ii omega_ij
// on rows [a, b) (output indexed from ptr[a]); partial correlations rho on
// supp(Omega) U supp(Omega^T) off the diagonal, rows [a, b): count -> scan ->
// fill keys -> launch_rowsort -> values.
int launch_diag(int dtype, int64_t rows, int64_t off, const int64_t* ptr, const int32_t* col,
                const void* val, double* d, int32_t* bad, cudaStream_t st);
int launch_theta(int dtype, int64_t a, int64_t b, const int64_t* ptr, const int32_t* col,
                 const void* val, const double* d, void* out, cudaStream_t st);
int launch_pcorr_count(int dtype, int64_t p, int64_t a, int64_t b, const int64_t* ptr,
                       const int32_t* col, const void* val, int32_t* own, int32_t* cnt,
                       cudaStream_t st);
int launch_pcorr_fill(int dtype, int64_t p, int64_t a, int64_t b, const int64_t* ptr,
                      const int32_t* col, const void* val, const int32_t* own,
                      const int64_t* optr, int32_t* ext, uint64_t* keys, cudaStream_t st);
int launch_pcorr_value(int dtype, int64_t a, int64_t b, const int64_t* ptr, const int32_t* col,
                       const void* val, const double* d, const int64_t* optr,
                       const uint64_t* keys, int32_t* ocol, void* oval, cudaStream_t st);

// Prox at trial tau over C (Eq. 3.5) with per-row partial sums. With items:
// a warp per work item (hub rows split), per-item sums combined per row in
// item order.
struct ProxItems {
  const int64_t* itm_ptr;     // [pk + 1] (NULL: warp per row)
  const int32_t* item_row;    // [n_items]
  int64_t n_items, L;
  double *dd, *l1, *logd;     // [n_items] per-item partial sums
  int32_t* nnz;
};
int launch_prox(int dtype, int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
                const void* c_g, const void* c_w, void* c_wn, double tau, double lam,
                double* row_dd, double* row_l1, double* row_logd, int32_t* row_nnz,
                cudaStream_t st, const ProxItems* items = nullptr);
// c_w[e] = omega_{i, c_col[e]} (0 if absent) on the structure (c_ptr, c_col);
// warp per row, or per work item when `items` is given.
int launch_lookup(int dtype, int64_t pk, const int64_t* c_ptr, const int32_t* c_col,
                  const int64_t* om_ptr, const int32_t* om_col, const void* om_val, void* c_w,
                  cudaStream_t st, const ProxItems* items = nullptr);

// SpMM Y+ = Omega+ X^T and D = Delta X^T over a CSR (ptr/col/wn/wo); wo may be
// NULL (Delta = 0). Accumulates in double; writes Y (T), optionally its bf16
// hi (and lo) copies with the per-row norms ||y||, ||y - bf16(y)||, and the
// per-row ||D_i||^2, ||Y+_i||^2.
struct SpmmRing {             // one ring step of the sharded-X SpMM (NEXT(3))
  int64_t v0, v1;             // columns of the resident slab; Xt row 0 = column v0
  double* yacc;               // [pk x ldk] partial Y+ across the ring steps (NULL: plain SpMM)
  double* dacc;               // [pk x ldk] partial D
  int first, last;            // first step initialises, last step finalises (Y, norms)
};
int launch_spmm(int dtype, int64_t pk, int64_t n, int64_t ldk, const int64_t* ptr,
                const int32_t* col, const void* wn, const void* wo, const void* Xt,
                void* Yout, __nv_bfloat16* Yhi, __nv_bfloat16* Ylo, float* row_A,
                float* row_B, double* row_D2, double* row_Y2, cudaStream_t st,
                const SpmmRing* ring = nullptr, int ydrop = 0);

// Exact candidate values: c_g[e] = (1/n) sum_m Y_im Xt_km in float64
// accumulation, for every entry of C (block per row). BF16_FILTER refine and
// the fixed-support gradient of the refit.
// Work items over a CSR (row chunks of <= L entries; rows longer than L
// become several items) for the TMA-staged SpMM and the refine.
constexpr int kSpmmTmaMaxConsumers = 256;   // ldk <= 2048
constexpr int kSpmmPairMaxConsumers = 128;  // paired-trial variant: ldk <= 1024
constexpr int64_t kItemEntries = 2048;
struct SpmmItems {
  const int64_t* itm_ptr;     // [rows + 1] exclusive scan of items per row
  const int32_t* item_row;    // [items] row of each item
  const int64_t* slot_ptr;    // [rows + 1] scratch slots of multi-item rows
  double* part_y;             // [slots x ldk] partial Y+ of multi-item rows
  double* part_d;             // [slots x ldk] partial D
  double* part_d2;            // [slots x ldk] partial D' (paired trial; may be NULL otherwise)
  int32_t* row_done;          // [rows] items finished (reset to 0 by the finisher)
  int64_t L;
};
int launch_item_map(int64_t rows, const int64_t* ptr, int64_t L, int32_t* nitem, int32_t* nslot,
                    int64_t* itm_ptr, int64_t* slot_ptr, void* scan_tmp, size_t scan_tmp_bytes,
                    cudaStream_t st);
int launch_item_rows(int64_t rows, const int64_t* itm_ptr, int32_t* item_row, cudaStream_t st);
bool spmm_tma_supported(int dtype, int64_t ldk);
// Producer warp + cp.async.bulk gathers of X^T rows into a shared-memory ring,
// float64 accumulation in the consumer warps (spmm_tma.cu). F32 only.
int launch_spmm_tma(int64_t pk, int64_t ldk, const int64_t* ptr, const int32_t* col,
                    const float* wn, const float* wo, const float* Xt, float* Yout,
                    __nv_bfloat16* Yhi, __nv_bfloat16* Ylo, float* row_A, float* row_B,
                    double* row_D2, double* row_Y2, const SpmmItems& items, int sm_count,
                    cudaStream_t st, const float* wn2 = nullptr, double* row_D2b = nullptr,
                    int ydrop = 0);

// Columns [v0, v1) only, Xt row 0 = column v0 (one ring step of the sharded mode).
// itm_ptr != NULL: one block per work item (row chunk of <= L candidates).
int launch_refine(int dtype, int64_t pk, int64_t n, int64_t ldk, const int64_t* c_ptr,
                  const int32_t* c_col, const void* Y, const void* Xt, void* c_g,
                  cudaStream_t st, int64_t v0 = 0, int64_t v1 = INT64_MAX,
                  const int64_t* itm_ptr = nullptr, int64_t n_items = 0, int64_t L = 0,
                  const int32_t* item_row = nullptr, int arith = 0,   // 1: float-float
                  int sym = 0);   // 1: C = C^T at Omega = I, entries k < i from their twins



// KKT residual (Eq. 3.3) over C with penalty lam: row maxima -> *out (device).
int launch_kkt(int dtype, int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
               const void* c_g, const void* c_w, double lam, double* row_max, double* out,
               cudaStream_t st);

// lambda_max (NEXT(2)): filter row constants of A = rows of X^T (Omega = I);
// max over the off-diagonal entries of C of |<x_i, x_k>| / n in float64 -> *out; direct max over
// columns [v0, v1) of |<x_i, x_k>| / n (CUDA cores; out may be NULL: ring steps
// accumulate into row_max with accumulate = 1, then launch once more or reduce).
int launch_row_ab(int64_t pk, int64_t ldk, const float* Xt_rows, float* row_A, float* row_B,
                  cudaStream_t st, int drop = 0);
int launch_cand_dot_max(int dtype, int64_t pk, int64_t r0, int64_t n, int64_t ldk,
                        const int64_t* c_ptr, const int32_t* c_col, const void* Xi, const void* Xt,
                        int64_t v0, int64_t v1, int accumulate, double* row_max, double* out,
                        cudaStream_t st);
int launch_gram_offdiag_max(int dtype, int64_t pk, int64_t r0, int64_t n, int64_t ldk,
                            const void* Xi, const void* Xt, int64_t v0, int64_t v1, int accumulate,
                            double* row_max, double* out, cudaStream_t st);

// Symmetric first GEMM across ranks: bucket the mirrored (global row, col)
// entries by owner rank (rb: the ranks' global row boundaries, P <= 64), and
// append received ones (global rows of this rank) to the pool from `start`.
int launch_mirror_count(int64_t n, const int32_t* row, const int64_t* rb, int P,
                        unsigned long long* cnt, cudaStream_t st);
int launch_mirror_scatter(int64_t n, const int32_t* row, const int32_t* col, const int64_t* rb,
                          int P, unsigned long long* cursor, int32_t* out, cudaStream_t st);
int launch_mirror_append(int64_t n, const int32_t* in, int64_t r0, int32_t* prow, int32_t* pcol,
                         int64_t start, int32_t* row_cnt, cudaStream_t st);

// Diagnostic: one thread spinning `ms` milliseconds on the stream (the
// NCCL watchdog test's stand-in for a slow or dead peer).
int launch_spin(int ms, cudaStream_t st);

// Per-column constants of the filter bound from Xt (f32).
int launch_col_norms(int64_t p, int64_t ldk, const float* Xt, float2* col_sd, cudaStream_t st,
                     int drop = 0);

// Omega stats over the current CSR: l1, logdiag, nnz, diagonal check.
int launch_omega_stats(int dtype, int64_t pk, int64_t r0, const int64_t* ptr,
                       const int32_t* col, const void* val, double* row_l1, double* row_logd,
                       int32_t* row_nnz, int32_t* bad_diag, cudaStream_t st);

// Fixed-order reduction of the per-row partials into out[8] =
// {D2, dd, logd, Y2, l1, nnz, ncand, max candidates in a row}. Any pointer may
// be NULL (-> 0).
// line search from Omega = I (kernels.cu): T on C, row dots, per-trial norms, apply
int launch_diag_t(int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
                  const float* c_g, double lam, float* c_t, cudaStream_t st);
int launch_diag_dots(int64_t pk, int64_t ldk, int64_t xrow0, const float* Xt, const float* Z,
                     double* xx, double* xz, double* zz, cudaStream_t st);
int launch_diag_trial(int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
                      const float* c_w, const float* c_wn, double tau, const double* xx,
                      const double* xz, const double* zz, double* row_Y2, double* row_D2,
                      double* row_a, cudaStream_t st);
int launch_diag_apply(int64_t pk, int64_t ldk, int64_t xrow0, const float* Xt, float* Y,
                      __nv_bfloat16* Yhi, const double* row_a, double tau, float* row_A,
                      float* row_B, cudaStream_t st, int ydrop = 0);
int launch_reduce_rows(int64_t pk, const double* row_D2, const double* row_dd,
                       const double* row_logd, const double* row_Y2, const double* row_l1,
                       const int32_t* row_nnz, const int64_t* c_ptr, double* out,
                       cudaStream_t st);

// Compaction of C (with new values) into Omega's CSR after acceptance.
int launch_compact(int dtype, int64_t pk, int64_t r0, const int64_t* c_ptr,
                   const int32_t* c_col, const void* c_wn, const int64_t* om_ptr,
                   int32_t* om_col, void* om_val, cudaStream_t st);

// Identity Omega^{(0)}.
int launch_identity(int dtype, int64_t pk, int64_t r0, int64_t* om_ptr, int32_t* om_col,
                    void* om_val, cudaStream_t st);

// Gradient GEMM + fused candidate epilogue (CUDA cores; T = float or double).
int launch_gemm_simt(int dtype, const void* Y, const void* Xt, int64_t ldk, int64_t kdim,
                     const EpiParams& ep, const OmegaView& om, const PoolView& pool,
                     cudaStream_t st);

// int8 operands of the I8_FILTER GEMM and its bound constants (quant_i8.cu).
// Y: per-row scale; rows [0, rows) of Y (f32, stride ldk) -> Yq, scale, A = ||e||, B = ||y||.
int launch_quant_y_i8(int64_t rows, int64_t n, int64_t ldk, const float* Y, int8_t* Yq,
                      float* scale, float* rA, float* rB, cudaStream_t st);
// X^T: Xq row k' = variable perm[k'] with the scale of its block of 256
// permuted rows -> blk_scale[rows/256], col_sd[variable] = (C + D, D).
int launch_quant_x_i8(int64_t rows, int64_t n, int64_t ldk, const float* Xt, const int32_t* perm,
                      int8_t* Xq, float* blk_scale, float2* col_sd, cudaStream_t st);
// max |x| per X^T row (the permutation key)
int launch_row_absmax(int64_t rows, int64_t n, int64_t ldk, const float* Xt, float* out,
                      cudaStream_t st);

// tcgen05 split-bf16 GEMM + fused epilogue (gemm_tc.cu).
struct TcGemmPlan;   // opaque: tensor maps for both Y buffers
TcGemmPlan* tc_plan_create(const __nv_bfloat16* Yhi0, const __nv_bfloat16* Ylo0,
                           const __nv_bfloat16* Yhi1, const __nv_bfloat16* Ylo1,
                           int64_t pk_pad, const __nv_bfloat16* Xhi,
                           const __nv_bfloat16* Xlo, int64_t xrows_pad, int64_t p_pad,
                           int64_t kdim, int64_t ldk, float2* blk_sdmax /* [p_pad/256], zeroed */,
                           std::string* err);
void tc_plan_destroy(TcGemmPlan*);
// per-256-column maxima of the filter's column constants (after launch_col_norms)
int tc_plan_set_col_norms(TcGemmPlan* plan, const float2* col_sd, int64_t p, cudaStream_t st,
                          bool i8 = false, const int32_t* perm = nullptr);
int tc_grid_size(const TcGemmPlan* plan, int sm_count);   // persistent CTAs
// A operand idx 2 = this rank's rows of X^T_hi (the Omega = I operand of the
// lambda_max pass); rows_pad rows from `hi`
bool tc_plan_set_a(TcGemmPlan* plan, int idx, const __nv_bfloat16* hi, int64_t rows_pad,
                   std::string* err);
// I8_FILTER operands: the two int8 Y buffers and int8 X^T (pk_pad / xrows_pad
// x ldk bytes, K-major); idx 2 of the A maps = an override (lambda_max)
bool tc_plan_set_i8(TcGemmPlan* plan, const int8_t* Yq0, const int8_t* Yq1, const int8_t* Xq,
                    int64_t xrows_pad, float2* blk_q /* [p_pad/256], zeroed */, std::string* err);
bool tc_plan_set_a_i8(TcGemmPlan* plan, int idx, const int8_t* q, int64_t rows_pad,
                      std::string* err);
// B operand idx 1/2 = ring buffers of the sharded mode (rows_pad x ldk bf16)
bool tc_plan_set_b(TcGemmPlan* plan, int idx, const __nv_bfloat16* hi, const __nv_bfloat16* lo,
                   int64_t rows_pad, std::string* err);
// columns [ep.col_base, ep.col_end) against B operand `bsel`
int launch_gemm_tc(TcGemmPlan* plan, int mode /* accord_gemm: BF16X3, BF16_FILTER, I8_FILTER */,
                   int ybuf, int bsel, int sm_count, const EpiParams& ep,
                   const OmegaView& om, const PoolView& pool, cudaStream_t st);
bool tc_supported(int cc_major, int cc_minor);

}  // namespace accord

// HBM-bound kernels of the ACCORD-FBS hot path (everything except the
// gradient GEMM): data load / operand split (a1), candidate finalize (a4),
// prox at trial tau (a5), SpMM with fused reductions (a6), fixed-order
// reductions (a7), compaction of the accepted iterate, power iteration for L.
//
// Row r of every per-rank array is the global row r0 + r of Omega.
#include "accord_internal.h"

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cfloat>
#include <climits>
#include <vector>

namespace accord {

namespace {

template <typename T> struct Vec;
template <> struct Vec<float> { using type = float4; static constexpr int V = 4; };
template <> struct Vec<double> { using type = double2; static constexpr int V = 2; };

__device__ __forceinline__ float vget(const float4& v, int i) {
  return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
}
__device__ __forceinline__ double vget(const double2& v, int i) { return i == 0 ? v.x : v.y; }

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum with a fixed reduction order (deterministic).
template <typename T>
__device__ T block_sum(T v, T* sh /* >= 32 */) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  T r = (threadIdx.x < nw) ? sh[threadIdx.x] : T(0);
  if (w == 0) r = warp_sum(r);
  if (threadIdx.x == 0) sh[0] = r;
  __syncthreads();
  r = sh[0];
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------
// a1: X -> Xt (variable-major, zero padded), finiteness check
// ---------------------------------------------------------------------------
template <typename T>
__global__ void load_xt_kernel(const T* __restrict__ X, int64_t ldx, int layout, int64_t n,
                               int64_t p, T* __restrict__ Xt, int64_t ldk, int64_t prows,
                               unsigned long long* bad) {
  __shared__ T tile[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int64_t m0 = (int64_t)blockIdx.x * 32;
  for (int64_t jb = blockIdx.y; jb * 32 < prows; jb += gridDim.y) {
    const int64_t j0 = jb * 32;
    if (layout == ACCORD_LAYOUT_VARIABLES_ROW_MAJOR) {
      for (int jj = ty; jj < 32; jj += 8) {
        const int64_t j = j0 + jj, m = m0 + tx;
        T v = T(0);
        if (j < p && m < n) {
          v = X[j * ldx + m];
          if (!isfinite(v)) atomicMin(bad, (unsigned long long)(j * n + m));
        }
        Xt[j * ldk + m] = v;
      }
    } else {
      // X is n x p row-major: read with tx along j (coalesced), write with tx along m.
      for (int mm = ty; mm < 32; mm += 8) {
        const int64_t m = m0 + mm, j = j0 + tx;
        T v = T(0);
        if (j < p && m < n) {
          v = X[m * ldx + j];
          if (!isfinite(v)) atomicMin(bad, (unsigned long long)(m * p + j));
        }
        tile[mm][tx] = v;
      }
      __syncthreads();
      for (int jj = ty; jj < 32; jj += 8) Xt[(j0 + jj) * ldk + m0 + tx] = tile[tx][jj];
      __syncthreads();
    }
  }
}

__global__ void split_bf16_kernel(const float4* __restrict__ src, int64_t n4,
                                  __nv_bfloat162* __restrict__ hi,
                                  __nv_bfloat162* __restrict__ lo, int drop) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    float4 v = src[i];
    __nv_bfloat162 h0 = drop ? __halves2bfloat162(filter_bf16_x(v.x, drop), filter_bf16_x(v.y, drop))
                             : filter_bf16x2(v.x, v.y);
    __nv_bfloat162 h1 = drop ? __halves2bfloat162(filter_bf16_x(v.z, drop), filter_bf16_x(v.w, drop))
                             : filter_bf16x2(v.z, v.w);
    float2 f0 = __bfloat1622float2(h0), f1 = __bfloat1622float2(h1);
    hi[2 * i] = h0;
    hi[2 * i + 1] = h1;
    if (lo) {   // NULL: the single-pass filter needs no low part
      lo[2 * i] = __floats2bfloat162_rn(v.x - f0.x, v.y - f0.y);
      lo[2 * i + 1] = __floats2bfloat162_rn(v.z - f1.x, v.w - f1.y);
    }
  }
}

// ---------------------------------------------------------------------------
// Exclusive scan int32 -> int64 (3 phases, fixed order)
// ---------------------------------------------------------------------------
constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanChunk = kScanThreads * kScanItems;

__device__ int64_t block_excl_scan(int64_t v, int64_t* sh, int64_t* total) {
  const int l = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (l >= o) x += y;
  }
  if (l == 31) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    int64_t s = (l < (int)(blockDim.x >> 5)) ? sh[l] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (l >= o) s += y;
    }
    sh[l] = s;  // inclusive warp sums
  }
  __syncthreads();
  int64_t off = (w > 0) ? sh[w - 1] : 0;
  *total = sh[(blockDim.x >> 5) - 1];
  __syncthreads();
  return off + x - v;
}

__global__ void __launch_bounds__(1024) scan_phase1(const int32_t* __restrict__ in, int64_t N, int64_t* bsum) {
  __shared__ int64_t sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * kScanItems;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < N) s += in[base + k];
  s = block_sum<int64_t>(s, sh);
  if (threadIdx.x == 0) bsum[blockIdx.x] = s;
}

__global__ void __launch_bounds__(1024) scan_phase2(int64_t* bsum, int64_t nb) {
  __shared__ int64_t sh[32];
  int64_t carry = 0;
  for (int64_t c = 0; c < nb; c += blockDim.x) {
    const int64_t i = c + threadIdx.x;
    int64_t v = i < nb ? bsum[i] : 0, tot;
    int64_t e = block_excl_scan(v, sh, &tot);
    if (i < nb) bsum[i] = carry + e;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[nb] = carry;
}

__global__ void __launch_bounds__(1024) scan_phase3(const int32_t* __restrict__ in, int64_t N,
                            const int64_t* __restrict__ bsum, int64_t nb, int64_t* out) {
  __shared__ int64_t sh[32];
  const int64_t base = (int64_t)blockIdx.x * kScanChunk + threadIdx.x * kScanItems;
  int64_t v[kScanItems], s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = (base + k < N) ? in[base + k] : 0;
    s += v[k];
  }
  int64_t tot;
  int64_t e = block_excl_scan(s, sh, &tot) + bsum[blockIdx.x];
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (base + k < N) out[base + k] = e;
    e += v[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[N] = bsum[nb];
}

// ---------------------------------------------------------------------------
// a4: candidate finalize: scatter pool -> per-row key segments, per-row sort
// by column, gather values in sorted order.
// key = (col << 32) | pool_index (unique), so sorting keys sorts by column.
// ---------------------------------------------------------------------------
constexpr int kWarpSortMax = 1024;     // rows up to this length: one warp, smem bitonic
constexpr int kBlockSortMax = 16384;   // rows up to this length: one block, smem bitonic

// grid: (blocks per chunk) x chunks handed out
__global__ void scatter_kernel(const int32_t* __restrict__ prow, const int32_t* __restrict__ pcol,
                               int64_t chunk, int64_t nchunks,
                               const unsigned int* __restrict__ chunk_next,
                               const unsigned long long* __restrict__ chunk_fill,
                               const int64_t* __restrict__ c_ptr, int32_t* rcur,
                               uint64_t* __restrict__ keys) {
  const int64_t used = min((int64_t)*chunk_next, nchunks);
  for (int64_t ch = blockIdx.y; ch < used; ch += gridDim.y) {
    const int64_t cnt = min((int64_t)chunk_fill[ch], chunk);
    for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < cnt;
         o += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = ch * chunk + o;
      const int32_t r = prow[i];
      const int64_t pos = c_ptr[r] + atomicAdd(&rcur[r], 1);
      keys[pos] = ((uint64_t)(uint32_t)pcol[i] << 32) | (uint64_t)(uint32_t)i;
    }
  }
}

__device__ __forceinline__ void bitonic_warp(uint64_t* s, int n2) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= n2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = lane; t < n2; t += 32) {
        const int ixj = t ^ j;
        if (ixj > t) {
          const bool asc = (t & k) == 0;
          uint64_t a = s[t], b = s[ixj];
          if ((a > b) == asc) { s[t] = b; s[ixj] = a; }
        }
      }
      __syncwarp();
    }
  }
}

__global__ void rowsort_warp_kernel(int64_t pk, const int64_t* __restrict__ c_ptr,
                                    uint64_t* __restrict__ keys, int32_t* long_rows) {
  extern __shared__ uint64_t sm_keys[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* s = sm_keys + (size_t)wib * kWarpSortMax;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (r >= pk) return;
  const int64_t beg = c_ptr[r], len = c_ptr[r + 1] - beg;
  if (len <= 1) return;
  if (len > kWarpSortMax) {
    if (lane == 0) {
      int slot = atomicAdd(&long_rows[0], 1);
      long_rows[1 + slot] = (int32_t)r;
    }
    return;
  }
  int n2 = 32;
  while (n2 < len) n2 <<= 1;
  for (int t = lane; t < n2; t += 32) s[t] = t < len ? keys[beg + t] : ~0ull;
  __syncwarp();
  bitonic_warp(s, n2);
  for (int t = lane; t < len; t += 32) keys[beg + t] = s[t];
}

// Rows longer than kWarpSortMax: one block per row. Runs of kBlockSortMax are
// sorted in shared memory (bitonic), then merged pairwise in global memory
// (merge path: each output position finds its split by binary search).
__global__ void __launch_bounds__(1024) rowsort_block_kernel(const int64_t* __restrict__ c_ptr,
                                                             uint64_t* __restrict__ keys,
                                                             uint64_t* __restrict__ tmp,
                                                             const int32_t* __restrict__ long_rows) {
  extern __shared__ uint64_t sm_keys[];
  const int nlong = long_rows[0];
  for (int q = blockIdx.x; q < nlong; q += gridDim.x) {
    const int64_t r = long_rows[1 + q];
    const int64_t beg = c_ptr[r], len = c_ptr[r + 1] - beg;
    for (int64_t run0 = 0; run0 < len; run0 += kBlockSortMax) {
      const int64_t rl = min((int64_t)kBlockSortMax, len - run0);
      int n2 = 32;
      while (n2 < rl) n2 <<= 1;
      uint64_t* g = keys + beg + run0;
      for (int t = threadIdx.x; t < n2; t += blockDim.x) sm_keys[t] = t < rl ? g[t] : ~0ull;
      __syncthreads();
      for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int t = threadIdx.x; t < n2; t += blockDim.x) {
            const int ixj = t ^ j;
            if (ixj > t) {
              const bool asc = (t & k) == 0;
              uint64_t x = sm_keys[t], y = sm_keys[ixj];
              if ((x > y) == asc) { sm_keys[t] = y; sm_keys[ixj] = x; }
            }
          }
          __syncthreads();
        }
      }
      for (int t = threadIdx.x; t < rl; t += blockDim.x) g[t] = sm_keys[t];
      __syncthreads();
    }
    uint64_t* src = keys + beg;
    uint64_t* dst = tmp + beg;
    for (int64_t w = kBlockSortMax; w < len; w *= 2) {
      for (int64_t s0 = 0; s0 < len; s0 += 2 * w) {
        const uint64_t* A = src + s0;
        const int64_t la = min(w, len - s0);
        const uint64_t* B = A + la;
        const int64_t lb = max((int64_t)0, min(w, len - s0 - la));
        for (int64_t k = threadIdx.x; k < la + lb; k += blockDim.x) {
          int64_t lo = max((int64_t)0, k - lb), hi = min(k, la);
          while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (A[mid] < B[k - mid - 1]) lo = mid + 1; else hi = mid;
          }
          const int64_t i = lo, j = k - lo;
          dst[s0 + k] = (j >= lb || (i < la && A[i] < B[j])) ? A[i] : B[j];
        }
      }
      __syncthreads();
      uint64_t* t2 = src; src = dst; dst = t2;
    }
    if (src != keys + beg) {
      for (int64_t t = threadIdx.x; t < len; t += blockDim.x) keys[beg + t] = src[t];
    }
    __syncthreads();
  }
}

template <typename T>
__global__ void gather_kernel(int64_t pk, const int64_t* __restrict__ c_ptr,
                              const uint64_t* __restrict__ keys, const T* __restrict__ pg,
                              const T* __restrict__ pw, int32_t* __restrict__ c_col,
                              T* __restrict__ c_g, T* __restrict__ c_w) {
  const int64_t tot = c_ptr[pk];
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[e];
    const uint32_t idx = (uint32_t)(k & 0xffffffffu);
    c_col[e] = (int32_t)(k >> 32);
    if (pg) c_g[e] = pg[idx];   // NULL for BF16_FILTER: the refine SDDMM writes c_g
    if (pw) c_w[e] = pw[idx];   // NULL for BF16_FILTER: looked up in Omega after the sort
  }
}

// ---------------------------------------------------------------------------
// Filter path: supp Omega (diagonal included: Omega's rows always store it)
// joins C in the finalize instead of the GEMM epilogue: its row lengths are
// added to the candidate counts, its entries scattered into the rows' key
// segments next to the GEMM's, the row sort puts duplicates (entries the
// filter also emitted) side by side, and a count + write pass keeps one of
// each (warp per row, order preserved).
// ---------------------------------------------------------------------------
__global__ void support_count_kernel(int64_t pk, const int64_t* __restrict__ om_ptr,
                                     int32_t* __restrict__ row_cnt) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < pk;
       r += (int64_t)gridDim.x * blockDim.x)
    row_cnt[r] += (int32_t)(om_ptr[r + 1] - om_ptr[r]);
}

__global__ void support_scatter_kernel(int64_t pk, const int64_t* __restrict__ om_ptr,
                                       const int32_t* __restrict__ om_col,
                                       const int64_t* __restrict__ c_ptr, int32_t* rcur,
                                       uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  const int64_t b = om_ptr[r], e = om_ptr[r + 1];
  if (b == e) return;
  int base = 0;
  if (lane == 0) base = atomicAdd(&rcur[r], (int)(e - b));
  base = __shfl_sync(0xffffffffu, base, 0);
  for (int64_t q = b + lane; q < e; q += 32)
    keys[c_ptr[r] + base + (q - b)] = ((uint64_t)(uint32_t)om_col[q] << 32) | 0xffffffffull;
}

__global__ void dedupe_count_kernel(int64_t pk, const int64_t* __restrict__ ptr,
                                    const uint64_t* __restrict__ keys, int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  const int64_t b = ptr[r], e = ptr[r + 1];
  int u = 0;
  for (int64_t q = b + lane; q < e; q += 32)
    u += (q == b || (keys[q] >> 32) != (keys[q - 1] >> 32)) ? 1 : 0;
  u = warp_sum(u);
  if (lane == 0) cnt[r] = u;
}

__global__ void dedupe_write_kernel(int64_t pk, const int64_t* __restrict__ ptr,
                                    const uint64_t* __restrict__ keys,
                                    const int64_t* __restrict__ optr, int32_t* __restrict__ col) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  const int64_t b = ptr[r], e = ptr[r + 1];
  int64_t o = optr[r];
  for (int64_t q0 = b; q0 < e; q0 += 32) {
    const int64_t q = q0 + lane;
    const bool u = q < e && (q == b || (keys[q] >> 32) != (keys[q - 1] >> 32));
    const unsigned m = __ballot_sync(0xffffffffu, u);
    if (u) col[o + __popc(m & ((1u << lane) - 1u))] = (int32_t)(keys[q] >> 32);
    o += __popc(m);
  }
}

// ---------------------------------------------------------------------------
// a5: prox at trial tau (Eq. 3.5), warp per row.
// Forward step and prox are evaluated in double from the stored values; the
// result is rounded to T. Diagonal root in the cancellation-free branch form.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double prox_diag_d(double y, double tau, double lam) {
  const double a = y - tau * lam;
  const double r = sqrt(a * a + 4.0 * tau);
  return a >= 0.0 ? 0.5 * (a + r) : 2.0 * tau / (r - a);
}

template <typename T>
__global__ void prox_kernel(int64_t pk, int64_t r0, const int64_t* __restrict__ c_ptr,
                            const int32_t* __restrict__ c_col, const T* __restrict__ c_g,
                            const T* __restrict__ c_w, T* __restrict__ c_wn, double tau,
                            double lam, double* __restrict__ row_dd,
                            double* __restrict__ row_l1, double* __restrict__ row_logd,
                            int32_t* __restrict__ row_nnz, ProxItems pi) {
  const int lane = threadIdx.x & 31;
  const int64_t w_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t r = w_id, beg, end;
  if (pi.itm_ptr) {   // warp per work item (hub rows split); sums per item
    if (w_id >= pi.n_items) return;
    r = pi.item_row[w_id];
    beg = c_ptr[r] + (w_id - pi.itm_ptr[r]) * pi.L;
    end = min(c_ptr[r + 1], beg + pi.L);
  } else {
    if (r >= pk) return;
    beg = c_ptr[r];
    end = c_ptr[r + 1];
  }
  const int64_t gi = r0 + r;
  const double tl = tau * lam;
  double dd = 0.0, l1 = 0.0, logd = 0.0;
  int nnz = 0;
  for (int64_t e = beg + lane; e < end; e += 32) {
    const double wo = (double)c_w[e];
    const double y = wo - tau * (double)c_g[e];       // forward step
    double w;
    if (c_col[e] == gi) {
      w = prox_diag_d(y, tau, lam);
    } else {
      const double m = fabs(y) - tl;                   // S_{tau lam}(y)
      w = m > 0.0 ? copysign(m, y) : 0.0;
    }
    const T wt = (T)w;
    c_wn[e] = wt;
    const double d = (double)wt - wo;
    dd += d * d;
    l1 += fabs((double)wt);
    nnz += wt != T(0);
    if (c_col[e] == gi) logd += log((double)wt);
  }
  dd = warp_sum(dd);
  l1 = warp_sum(l1);
  logd = warp_sum(logd);
  nnz = warp_sum(nnz);
  if (lane == 0) {
    if (pi.itm_ptr) {   // per item; prox_combine_kernel sums them per row
      pi.dd[w_id] = dd;
      pi.l1[w_id] = l1;
      pi.logd[w_id] = logd;
      pi.nnz[w_id] = nnz;
    } else {
      row_dd[r] = dd;
      row_l1[r] = l1;
      row_logd[r] = logd;
      row_nnz[r] = nnz;
    }
  }
}

// per-row sums from the per-item partials (fixed item order)
__global__ void prox_combine_kernel(int64_t pk, ProxItems pi, double* __restrict__ row_dd,
                                    double* __restrict__ row_l1, double* __restrict__ row_logd,
                                    int32_t* __restrict__ row_nnz) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < pk;
       r += (int64_t)gridDim.x * blockDim.x) {
    double dd = 0.0, l1 = 0.0, logd = 0.0;
    int nnz = 0;
    for (int64_t it = pi.itm_ptr[r]; it < pi.itm_ptr[r + 1]; ++it) {
      dd += pi.dd[it];
      l1 += pi.l1[it];
      logd += pi.logd[it];
      nnz += pi.nnz[it];
    }
    row_dd[r] = dd;
    row_l1[r] = l1;
    row_logd[r] = logd;
    row_nnz[r] = nnz;
  }
}

// ---------------------------------------------------------------------------
// a6: SpMM Y+_i = sum_j w+_ij Xt_j and D_i = sum_j Delta_ij Xt_j, block per row,
// 16-byte coalesced gathers of Xt rows; fused ||D_i||^2 and ||Y+_i||^2.
// ---------------------------------------------------------------------------
// first index e in [lo, hi) of a sorted column run with col[e] >= v
__device__ __forceinline__ int64_t lower_bound_col(const int32_t* __restrict__ col, int64_t lo,
                                                   int64_t hi, int64_t v) {
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if ((int64_t)col[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

constexpr int kSpmmMaxThreads = 1024;

template <typename T, bool kSplit>
__global__ void __launch_bounds__(1024) spmm_kernel(
    int64_t pk, int64_t n, int64_t ldk, const int64_t* __restrict__ ptr,
    const int32_t* __restrict__ col, const T* __restrict__ wn, const T* __restrict__ wo,
    const T* __restrict__ Xt, T* __restrict__ Yout, __nv_bfloat16* __restrict__ Yhi,
    __nv_bfloat16* __restrict__ Ylo, float* __restrict__ row_A, float* __restrict__ row_B,
    double* __restrict__ row_D2, double* __restrict__ row_Y2, SpmmRing rg, int ydrop) {
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  __shared__ int32_t s_col[kSpmmMaxThreads];
  __shared__ double s_w[kSpmmMaxThreads];
  __shared__ double s_d[kSpmmMaxThreads];
  __shared__ int s_wc[32];
  __shared__ double s_red[32];
  const int64_t r = blockIdx.x;
  int64_t beg = ptr[r], end = ptr[r + 1];
  // sharded X (NEXT(3)): only this row's entries in the resident slab's
  // columns [v0, v1) (a contiguous run of the sorted row); partial sums carry
  // across the ring steps in float64 accumulators
  const bool ring = rg.yacc != nullptr;
  const int32_t xoff = ring ? (int32_t)rg.v0 : 0;
  if (ring) {
    beg = lower_bound_col(col, beg, end, rg.v0);
    end = lower_bound_col(col, beg, end, rg.v1);
    if (beg == end && !rg.first && !rg.last) return;   // nothing to add
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double d2 = 0.0, y2 = 0.0, a2 = 0.0, b2 = 0.0;
  for (int64_t c0 = 0; c0 < ldk; c0 += (int64_t)blockDim.x * V) {
    const int64_t c = c0 + (int64_t)threadIdx.x * V;
    const bool active = c < ldk;
    double ay[V], ad[V];
#pragma unroll
    for (int v = 0; v < V; ++v) { ay[v] = 0.0; ad[v] = 0.0; }
    if (ring && !rg.first && active) {
#pragma unroll
      for (int v = 0; v < V; ++v) {
        ay[v] = rg.yacc[r * ldk + c + v];
        ad[v] = rg.dacc[r * ldk + c + v];
      }
    }
    for (int64_t e0 = beg; e0 < end; e0 += blockDim.x) {
      // stage the next blockDim entries in order, dropping w+ = Delta = 0
      // (deterministic ballot/prefix compaction)
      const int64_t e = e0 + threadIdx.x;
      bool keep = false;
      double w = 0.0, d = 0.0;
      int32_t cc = 0;
      if (e < end) {
        w = (double)wn[e];
        d = wo ? w - (double)wo[e] : 0.0;
        cc = col[e] - xoff;
        keep = (w != 0.0) || (d != 0.0);
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (lane == 0) s_wc[wid] = __popc(m);
      __syncthreads();
      int off = 0, cnt = 0;
      for (int q = 0; q < nw; ++q) {
        const int x = s_wc[q];
        off += q < wid ? x : 0;
        cnt += x;
      }
      if (keep) {
        const int s = off + __popc(m & ((1u << lane) - 1u));
        s_col[s] = cc;
        s_w[s] = w;
        s_d[s] = d;
      }
      __syncthreads();
      if (active) {
        int q = 0;
        for (; q + 4 <= cnt; q += 4) {
          VT x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u)
            x[u] = __ldg(reinterpret_cast<const VT*>(Xt + (int64_t)s_col[q + u] * ldk + c));
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double wv = s_w[q + u], dv = s_d[q + u];
#pragma unroll
            for (int v = 0; v < V; ++v) {
              ay[v] = fma(wv, (double)vget(x[u], v), ay[v]);
              ad[v] = fma(dv, (double)vget(x[u], v), ad[v]);
            }
          }
        }
        for (; q < cnt; ++q) {
          VT x = __ldg(reinterpret_cast<const VT*>(Xt + (int64_t)s_col[q] * ldk + c));
          const double wv = s_w[q], dv = s_d[q];
#pragma unroll
          for (int v = 0; v < V; ++v) {
            ay[v] = fma(wv, (double)vget(x, v), ay[v]);
            ad[v] = fma(dv, (double)vget(x, v), ad[v]);
          }
        }
      }
      __syncthreads();
    }
    if (ring && !rg.last) {
      if (active) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
          rg.yacc[r * ldk + c + v] = ay[v];
          rg.dacc[r * ldk + c + v] = ad[v];
        }
      }
      continue;
    }
    if (active) {
      T yt[V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        d2 += ad[v] * ad[v];
        y2 += ay[v] * ay[v];
        yt[v] = (T)ay[v];
      }
      if (Yout) {
        VT o;
        if constexpr (V == 4) o = make_float4(yt[0], yt[1], yt[2], yt[3]);
        else o = make_double2(yt[0], yt[1]);
        *reinterpret_cast<VT*>(Yout + r * ldk + c) = o;
      }
      if constexpr (kSplit) {
        // GEMM operand copies: hi = bf16(y), lo = bf16(y - hi); norms for the
        // filter bound: ||y||, ||y - hi||
#pragma unroll
        for (int v = 0; v < V; ++v) {
          const float y = (float)yt[v];
          const __nv_bfloat16 h = filter_bf16_x(y, ydrop);
          const float hf = __bfloat162float(h);
          Yhi[r * ldk + c + v] = h;
          if (Ylo) Ylo[r * ldk + c + v] = __float2bfloat16_rn(y - hf);
          const double e = (double)y - (double)hf;
          a2 += e * e;
          b2 += (double)y * (double)y;
        }
      }
    }
  }
  if (ring && !rg.last) return;   // block-uniform
  d2 = block_sum(d2, s_red);
  y2 = block_sum(y2, s_red);
  if constexpr (kSplit) {
    a2 = block_sum(a2, s_red);
    b2 = block_sum(b2, s_red);
  }
  if (threadIdx.x == 0) {
    if (row_D2) row_D2[r] = d2;
    if (row_Y2) row_Y2[r] = y2;
    if constexpr (kSplit) {
      // rounded up: these enter an upper bound
      if (row_A) row_A[r] = __double2float_ru(sqrt(a2) * (1.0 + 1e-12));
      if (row_B) row_B[r] = __double2float_ru(sqrt(b2) * (1.0 + 1e-12));
    }
  }
  (void)n;
}

// ---------------------------------------------------------------------------
// Exact candidate values (BF16_FILTER refine, and the gradient on a fixed
// support for the bias-correction refit): c_g[e] = (1/n) <Y_i, Xt_k> with
// float64 accumulation; warp per candidate, Y_i staged in shared memory.
//
// kFF (float data): the dot product in float-float arithmetic on the FP32
// pipes instead of float64: each product x y is split exactly into p + e
// (p = rn(x y), e = fma(x, y, -p)) and summed with Knuth's TwoSum into a
// (hi, lo) pair. The float64 path converts both operands of every product
// (F2F.F64.F32 on the XU pipe, 16 per clock per SM): ncu showed the XU pipe
// 56 % busy at 4.4 TB/s, the ceiling the gather could not pass. Float-float
// keeps ~2^-46 of the sum of |products| (the f32 result is the correctly
// rounded value of the exact dot except in ties below that), far inside the
// f32 value c_g stores.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ff_madd(float& hi, float& lo, float x, float y) {
  const float p = __fmul_rn(x, y);
  const float e = __fmaf_rn(x, y, -p);              // x y = p + e exactly
  const float t = __fadd_rn(hi, p);                 // TwoSum(hi, p) = t + err exactly
  const float z = __fsub_rn(t, hi);
  const float err = __fadd_rn(__fsub_rn(hi, __fsub_rn(t, z)), __fsub_rn(p, z));
  lo = __fadd_rn(lo, __fadd_rn(err, e));
  hi = t;
}

// <y, x> over ldk elements in float64 (exact f32 products), lanes striding
// the row, 8 loads in flight per lane, warp-reduced: the refine's dot product
// (its summation order is fixed, so (i,k) and (k,i) at Omega = I agree bitwise)
template <typename T>
__device__ __forceinline__ double warp_dot_f64(const T* ys, const T* __restrict__ xr, int64_t ldk,
                                               int lane) {
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  constexpr int kStep = 32 * V;           // elements per lane-pass over the row
  double s = 0.0;
  int64_t m = lane * V;
  for (; m + 7 * kStep < ldk; m += 8 * kStep) {
    VT x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(reinterpret_cast<const VT*>(xr + m + u * kStep));
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const VT yv = *reinterpret_cast<const VT*>(ys + m + u * kStep);
#pragma unroll
      for (int v = 0; v < V; ++v) s = fma((double)vget(yv, v), (double)vget(x[u], v), s);
    }
  }
  for (; m < ldk; m += kStep) {
    const VT x = __ldg(reinterpret_cast<const VT*>(xr + m));
    const VT yv = *reinterpret_cast<const VT*>(ys + m);
#pragma unroll
    for (int v = 0; v < V; ++v) s = fma((double)vget(yv, v), (double)vget(x, v), s);
  }
  return warp_sum(s);
}

// Shared-memory slot of element e of Y_i staged as float64 for the refine:
// element e belongs to lane (e >> 2) & 31 of 128-element block e >> 7; the
// lanes' first double2 (elements 0-1 of their four) are stored contiguously,
// then their second (elements 2-3), so each of the two 16-byte loads of a
// warp reads 512 contiguous bytes (4 wavefronts, no bank conflict; with the
// plain layout the lanes were 32 B apart and each load took 8)
__device__ __forceinline__ int64_t yd_slot(int64_t e) {
  return ((((e >> 7) * 2 + ((e >> 1) & 1)) * 32 + ((e >> 2) & 31)) << 1) + (e & 1);
}

// <y, x> as above with y already in float64 (staged once per work item):
// one F2F per product instead of two (the XU pipe's F2F.F64.F32 was the
// refine's limit); the same products in the same order, so bitwise equal
__device__ __forceinline__ double warp_dot_f64_yd(const double* ysd, const float* __restrict__ xr,
                                                  int64_t ldk, int lane) {
  constexpr int V = 4;
  constexpr int kStep = 32 * V;
  const double2* y2 = reinterpret_cast<const double2*>(ysd);
  double s = 0.0;
  int64_t m = lane * V;
  for (; m + 7 * kStep < ldk; m += 8 * kStep) {
    float4 x[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = __ldg(reinterpret_cast<const float4*>(xr + m + u * kStep));
    const int64_t U0 = (m - lane * V) >> 7;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const double2 y0 = y2[((U0 + u) * 2) * 32 + lane];
      const double2 y1 = y2[((U0 + u) * 2 + 1) * 32 + lane];
      s = fma(y0.x, (double)x[u].x, s);
      s = fma(y0.y, (double)x[u].y, s);
      s = fma(y1.x, (double)x[u].z, s);
      s = fma(y1.y, (double)x[u].w, s);
    }
  }
  for (; m < ldk; m += kStep) {
    const float4 x = __ldg(reinterpret_cast<const float4*>(xr + m));
    const int64_t U = (m - lane * V) >> 7;
    const double2 y0 = y2[(U * 2) * 32 + lane];
    const double2 y1 = y2[(U * 2 + 1) * 32 + lane];
    s = fma(y0.x, (double)x.x, s);
    s = fma(y0.y, (double)x.y, s);
    s = fma(y1.x, (double)x.z, s);
    s = fma(y1.y, (double)x.w, s);
  }
  return warp_sum(s);
}

// kArith: 0 = float64 products (both operands converted by F2F), 1 =
// float-float (A-B variant, slower; ACCORD_REFINE=ff), 2 = Y_i staged in
// shared memory as float64 (one F2F per product; T = float, default)
// sym (Omega = I on one rank, C = C^T): only the entries with k >= i; the
// others are copied from their twins afterwards (sym_mirror_kernel)
template <typename T, int kArith = 0>
__global__ void __launch_bounds__(256) refine_kernel(int64_t pk, int64_t n, int64_t ldk,
                                                     const int64_t* __restrict__ c_ptr,
                                                     const int32_t* __restrict__ c_col,
                                                     const T* __restrict__ Y,
                                                     const T* __restrict__ Xt,
                                                     T* __restrict__ c_g, int64_t v0,
                                                     int64_t v1, const int64_t* __restrict__ itm_ptr,
                                                     int64_t L, const int32_t* __restrict__ item_row,
                                                     int y_global, int sym) {
  using VT = typename Vec<T>::type;
  constexpr int V = Vec<T>::V;
  extern __shared__ __align__(16) uint8_t ys_raw[];
  // Y_i staged in shared memory, or read in place (through L1) when a row
  // does not fit (n beyond ~25,000 float64 / ~50,000 float32 samples)
  const T* ys = reinterpret_cast<const T*>(ys_raw);
  int64_t r = blockIdx.x;
  int64_t beg, end;
  if (itm_ptr) {   // work item = chunk of <= L candidates of one row (hub rows split)
    const int64_t it = blockIdx.x;
    r = item_row[it];
    beg = c_ptr[r] + (it - itm_ptr[r]) * L;
    end = min(c_ptr[r + 1], beg + L);
  } else {
    beg = c_ptr[r];
    end = c_ptr[r + 1];
  }
  // columns [v0, v1) only (Xt row 0 = column v0): one ring step of the
  // sharded mode (NEXT(3)); v0 = 0, v1 = p otherwise
  beg = lower_bound_col(c_col, beg, end, sym ? max(v0, r) : v0);
  end = lower_bound_col(c_col, beg, end, v1);
  if (beg == end) return;
  if (y_global) {
    ys = Y + r * ldk;
  } else if constexpr (kArith == 2) {
    double* yd = reinterpret_cast<double*>(ys_raw);
    for (int64_t m = threadIdx.x * V; m < ldk; m += blockDim.x * V) {
      const VT v = *reinterpret_cast<const VT*>(Y + r * ldk + m);
#pragma unroll
      for (int u = 0; u < V; ++u) yd[yd_slot(m + u)] = (double)vget(v, u);
    }
    __syncthreads();
  } else {
    T* yw = reinterpret_cast<T*>(ys_raw);
    for (int64_t m = threadIdx.x * V; m < ldk; m += blockDim.x * V)
      *reinterpret_cast<VT*>(yw + m) = *reinterpret_cast<const VT*>(Y + r * ldk + m);
    __syncthreads();
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const double inv_n = 1.0 / (double)n;
  constexpr int kStep = 32 * V;           // elements per lane-pass over the row
  for (int64_t e = beg + wid; e < end; e += nw) {
    const T* xr = Xt + (int64_t)(c_col[e] - v0) * ldk;
    if constexpr (kArith == 1) {
      // two (hi, lo) accumulators: shorter dependent chains
      float h0 = 0.f, l0 = 0.f, h1 = 0.f, l1 = 0.f;
      int64_t m = lane * V;
      for (; m + 7 * kStep < ldk; m += 8 * kStep) {
        VT x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = __ldg(reinterpret_cast<const VT*>(xr + m + u * kStep));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const VT yv = *reinterpret_cast<const VT*>(ys + m + u * kStep);
#pragma unroll
          for (int v = 0; v < V; ++v) {
            if (v & 1) ff_madd(h1, l1, (float)vget(yv, v), (float)vget(x[u], v));
            else ff_madd(h0, l0, (float)vget(yv, v), (float)vget(x[u], v));
          }
        }
      }
      for (; m < ldk; m += kStep) {
        const VT x = __ldg(reinterpret_cast<const VT*>(xr + m));
        const VT yv = *reinterpret_cast<const VT*>(ys + m);
#pragma unroll
        for (int v = 0; v < V; ++v) ff_madd(h0, l0, (float)vget(yv, v), (float)vget(x, v));
      }
      double s = ((double)h0 + (double)h1) + ((double)l0 + (double)l1);
      s = warp_sum(s);
      if (lane == 0) c_g[e] = (T)(s * inv_n);
      continue;
    }
    double s;
    if constexpr (kArith == 2) {
      if (y_global) s = warp_dot_f64<T>(ys, xr, ldk, lane);
      else s = warp_dot_f64_yd(reinterpret_cast<const double*>(ys_raw), (const float*)xr, ldk, lane);
    } else {
      s = warp_dot_f64<T>(ys, xr, ldk, lane);
    }
    if (lane == 0) c_g[e] = (T)(s * inv_n);
  }
}

// The entries k < i of a symmetric C (Omega = I on one rank, G = S): c_g from
// the twin (k, i), found by binary search in row k's sorted columns. The
// filter decides the entries of a diagonal tile one by one, so a twin can be
// missing near the threshold: that entry's dot product is computed here, by
// the whole warp in the refine's order. Warp per row. all_miss: every entry
// takes that path (test of the fallback).
template <typename T>
__global__ void sym_mirror_kernel(int64_t pk, int64_t ldk, const int64_t* __restrict__ c_ptr,
                                  const int32_t* __restrict__ c_col, const T* __restrict__ Y,
                                  const T* __restrict__ Xt, T* __restrict__ c_g, double inv_n,
                                  int all_miss) {
  const int lane = threadIdx.x & 31;
  const int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= pk) return;
  const int64_t beg = c_ptr[i];
  const int64_t end = lower_bound_col(c_col, beg, c_ptr[i + 1], i);
  for (int64_t e0 = beg; e0 < end; e0 += 32) {
    const int64_t e = e0 + lane;
    bool miss = false;
    if (e < end) {
      const int64_t k = c_col[e];
      const int64_t kb = c_ptr[k], ke = c_ptr[k + 1];
      const int64_t pos = lower_bound_col(c_col, kb, ke, i);
      if (!all_miss && pos < ke && c_col[pos] == (int32_t)i) c_g[e] = c_g[pos];
      else miss = true;
    }
    unsigned mm = __ballot_sync(0xffffffffu, miss);
    while (mm) {
      const int l = __ffs(mm) - 1;
      mm &= mm - 1;
      const int64_t ee = e0 + l;
      const double s = warp_dot_f64<T>(Y + i * ldk, Xt + (int64_t)c_col[ee] * ldk, ldk, lane);
      if (lane == 0) c_g[ee] = (T)(s * inv_n);
    }
  }
}

// Values of Omega on a fixed structure (refit support): c_w[e] = omega_{i, c_col[e]}
// or 0. Warp per row, binary search in Omega's sorted row.
template <typename T>
__global__ void lookup_kernel(int64_t pk, const int64_t* __restrict__ c_ptr,
                              const int32_t* __restrict__ c_col, const int64_t* __restrict__ om_ptr,
                              const int32_t* __restrict__ om_col, const T* __restrict__ om_val,
                              T* __restrict__ c_w, ProxItems pi) {
  const int lane = threadIdx.x & 31;
  const int64_t w_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  int64_t r = w_id, beg, end;
  if (pi.itm_ptr) {   // warp per work item (hub rows split)
    if (w_id >= pi.n_items) return;
    r = pi.item_row[w_id];
    beg = c_ptr[r] + (w_id - pi.itm_ptr[r]) * pi.L;
    end = min(c_ptr[r + 1], beg + pi.L);
  } else {
    if (r >= pk) return;
    beg = c_ptr[r];
    end = c_ptr[r + 1];
  }
  const int64_t ob = om_ptr[r], oe = om_ptr[r + 1];
  for (int64_t e = beg + lane; e < end; e += 32) {
    const int32_t k = c_col[e];
    int64_t lo = ob, hi = oe;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (om_col[mid] < k) lo = mid + 1; else hi = mid;
    }
    c_w[e] = (lo < oe && om_col[lo] == k) ? om_val[lo] : T(0);
  }
}

// KKT residual of Eq. (3.3) over the candidate set, per row:
//   diagonal |-1/w + G + lam|, nonzero |G + lam sign w|, zero max(0, |G| - lam).
// Entries outside C have |G| <= lam (certified by the GEMM epilogue) and
// contribute 0; on a refit support, entries outside it are fixed at zero.
template <typename T>
__global__ void kkt_kernel(int64_t pk, int64_t r0, const int64_t* __restrict__ c_ptr,
                           const int32_t* __restrict__ c_col, const T* __restrict__ c_g,
                           const T* __restrict__ c_w, double lam, double* __restrict__ row_max) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  double mx = 0.0;
  for (int64_t e = c_ptr[r] + lane; e < c_ptr[r + 1]; e += 32) {
    const double g = (double)c_g[e], w = (double)c_w[e];
    double v;
    if (c_col[e] == r0 + r) v = fabs(-1.0 / w + g + lam);
    else if (w != 0.0) v = fabs(g + copysign(lam, w));
    else v = fmax(0.0, fabs(g) - lam);
    mx = fmax(mx, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) row_max[r] = mx;
}

__global__ void __launch_bounds__(1024) reduce_max_kernel(int64_t pk, const double* __restrict__ v,
                                                          double* out) {
  __shared__ double sh[32];
  double mx = 0.0;
  for (int64_t r = threadIdx.x; r < pk; r += blockDim.x) mx = fmax(mx, v[r]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sh[w]);
    *out = mx;
  }
}

// ---------------------------------------------------------------------------
// lambda_max = max_{i != k} |S_ik| (the top of a lambda path, SURVEY.md §8(f)
// NEXT(2); SPEC.md lambda_grid)
// ---------------------------------------------------------------------------
// Filter row constants of A = the rank's rows of X^T (Omega = I): A_i =
// ||x_i - bf16(x_i)||, B_i = ||x_i||, rounded up (warp per row).
__global__ void xrow_ab_kernel(int64_t pk, int64_t ldk, const float* __restrict__ Xt,
                               float* __restrict__ row_A, float* __restrict__ row_B, int drop) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  double xx = 0, ee = 0;
  for (int64_t m = lane; m < ldk; m += 32) {
    const float x = Xt[r * ldk + m];
    const double e = (double)x - (double)__bfloat162float(filter_bf16_x(x, drop));
    xx += (double)x * x;
    ee += e * e;
  }
  xx = warp_sum(xx);
  ee = warp_sum(ee);
  if (lane == 0) {
    row_A[r] = __double2float_ru(sqrt(ee) * (1.0 + 1e-12));
    row_B[r] = __double2float_ru(sqrt(xx) * (1.0 + 1e-12));
  }
}

// Per-row max over the OFF-diagonal entries (i,k) of C, columns [v0, v1), of
// |<x_i, x_k>| / n recomputed in float64 (warp per row, warp per entry).
// Xi = the rank's row r of X^T; Xt row 0 = column v0.
template <typename T>
__global__ void cand_dot_max_kernel(int64_t pk, int64_t r0, int64_t n, int64_t ldk,
                                    const int64_t* __restrict__ c_ptr,
                                    const int32_t* __restrict__ c_col, const T* __restrict__ Xi,
                                    const T* __restrict__ Xt, int64_t v0, int64_t v1,
                                    int accumulate, double* __restrict__ row_max) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  const int64_t beg = lower_bound_col(c_col, c_ptr[r], c_ptr[r + 1], v0);
  const int64_t end = lower_bound_col(c_col, beg, c_ptr[r + 1], v1);
  double mx = accumulate ? row_max[r] : 0.0;
  for (int64_t e = beg; e < end; ++e) {
    const int64_t k = c_col[e];
    if (k == r0 + r) continue;
    const T* xa = Xi + r * ldk;
    const T* xb = Xt + (k - v0) * ldk;
    double s = 0.0;
    for (int64_t m = lane; m < ldk; m += 32) s = fma((double)xa[m], (double)xb[m], s);
    s = warp_sum(s);
    mx = fmax(mx, fabs(s) / (double)n);
  }
  if (lane == 0) row_max[r] = mx;
}

// Direct evaluation (CUDA cores, float64 accumulation) for the SIMT / BF16X3
// contexts: row_max[r] = max over columns k in [v0, v1), k != r0 + r, of
// |<x_{r0+r}, x_k>| / n. Block per row, x_i staged in shared memory, warp per
// column. Xi = the rank's row r of X^T; Xt row 0 = column v0.
template <typename T>
__global__ void __launch_bounds__(256) gram_offdiag_max_kernel(int64_t pk, int64_t r0, int64_t n,
                                                               int64_t ldk, const T* __restrict__ Xi,
                                                               const T* __restrict__ Xt, int64_t v0,
                                                               int64_t v1, int accumulate,
                                                               double* __restrict__ row_max) {
  extern __shared__ __align__(16) uint8_t xs_raw[];
  T* xs = reinterpret_cast<T*>(xs_raw);
  __shared__ double wm[8];
  const int64_t r = blockIdx.x;
  for (int64_t m = threadIdx.x; m < ldk; m += blockDim.x) xs[m] = Xi[r * ldk + m];
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double mx = 0.0;
  for (int64_t k = v0 + wid; k < v1; k += nw) {
    if (k == r0 + r) continue;
    const T* xr = Xt + (k - v0) * ldk;
    double s = 0.0;
    for (int64_t m = lane; m < ldk; m += 32) s = fma((double)xs[m], (double)xr[m], s);
    s = warp_sum(s);
    mx = fmax(mx, fabs(s) / (double)n);
  }
  if (lane == 0) wm[wid] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < nw; ++w) mx = fmax(mx, wm[w]);
    row_max[r] = accumulate ? fmax(row_max[r], mx) : mx;
  }
}

// ---------------------------------------------------------------------------
// Symmetric first GEMM across ranks (EpiParams::sym = 2): the mirrored
// entries (k, i) of rows k another rank owns are bucketed by owner, sent, and
// the received ones appended to the candidate pool as extra chunks.
// ---------------------------------------------------------------------------
__device__ __forceinline__ int owner_of(int64_t k, const int64_t* __restrict__ rb, int P) {
  int q = 0;
  while (q + 1 < P && k >= rb[q + 1]) ++q;
  return q;
}

__global__ void mirror_count_kernel(int64_t n, const int32_t* __restrict__ row,
                                    const int64_t* __restrict__ rb, int P,
                                    unsigned long long* __restrict__ cnt) {
  __shared__ unsigned int sc[64];
  for (int q = threadIdx.x; q < P; q += blockDim.x) sc[q] = 0;
  __syncthreads();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&sc[owner_of(row[e], rb, P)], 1u);
  __syncthreads();
  for (int q = threadIdx.x; q < P; q += blockDim.x)
    if (sc[q]) atomicAdd(&cnt[q], (unsigned long long)sc[q]);
}

__global__ void mirror_scatter_kernel(int64_t n, const int32_t* __restrict__ row,
                                      const int32_t* __restrict__ col,
                                      const int64_t* __restrict__ rb, int P,
                                      unsigned long long* __restrict__ cursor,
                                      int32_t* __restrict__ out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t k = row[e];
    const unsigned long long pos = atomicAdd(&cursor[owner_of(k, rb, P)], 1ull);
    out[2 * pos] = k;
    out[2 * pos + 1] = col[e];
  }
}

__global__ void mirror_append_kernel(int64_t n, const int32_t* __restrict__ in, int64_t r0,
                                     int32_t* __restrict__ prow, int32_t* __restrict__ pcol,
                                     int64_t start, int32_t* __restrict__ row_cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t r = (int32_t)(in[2 * e] - r0);
    prow[start + e] = r;
    pcol[start + e] = in[2 * e + 1];
    atomicAdd(&row_cnt[r], 1);
  }
}

// per-column constants of the filter bound (warp per column of X = row of Xt)
__global__ void col_norms_kernel(int64_t p, int64_t ldk, const float* __restrict__ Xt,
                                 float2* __restrict__ col_sd, int drop) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= p) return;
  double xx = 0, ee = 0;
  for (int64_t m = lane; m < ldk; m += 32) {
    const float x = Xt[k * ldk + m];
    const double e = (double)x - (double)__bfloat162float(filter_bf16_x(x, drop));
    xx += (double)x * x;
    ee += e * e;
  }
  xx = warp_sum(xx);
  ee = warp_sum(ee);
  if (lane == 0) {
    const double xn = sqrt(xx) * (1.0 + 1e-12), en = sqrt(ee) * (1.0 + 1e-12);
    col_sd[k] = make_float2(__double2float_ru(xn + en), __double2float_ru(en));
  }
}

// ---------------------------------------------------------------------------
// Omega statistics (l1, log diag, nnz, diagonal present and > 0), warp per row
// ---------------------------------------------------------------------------
template <typename T>
__global__ void omega_stats_kernel(int64_t pk, int64_t r0, const int64_t* __restrict__ ptr,
                                   const int32_t* __restrict__ col, const T* __restrict__ val,
                                   double* row_l1, double* row_logd, int32_t* row_nnz,
                                   int32_t* bad_diag) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  double l1 = 0, logd = 0;
  int nnz = 0, has_diag = 0;
  for (int64_t e = ptr[r] + lane; e < ptr[r + 1]; e += 32) {
    const double v = (double)val[e];
    l1 += fabs(v);
    nnz += v != 0.0;
    if (col[e] == r0 + r) {
      has_diag = 1;
      if (v > 0.0) logd += log(v); else atomicExch(bad_diag, 1);
    }
  }
  l1 = warp_sum(l1);
  logd = warp_sum(logd);
  nnz = warp_sum(nnz);
  has_diag = warp_sum(has_diag);
  if (lane == 0) {
    row_l1[r] = l1;
    row_logd[r] = logd;
    row_nnz[r] = nnz;
    if (!has_diag) atomicExch(bad_diag, 1);
  }
}

// ---------------------------------------------------------------------------
// a7: fixed-order reduction of per-row partials (one block, deterministic)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) reduce_rows_kernel(int64_t pk, const double* __restrict__ D2,
                                   const double* __restrict__ dd, const double* __restrict__ logd,
                                   const double* __restrict__ Y2, const double* __restrict__ l1,
                                   const int32_t* __restrict__ nnz, const int64_t* __restrict__ c_ptr,
                                   double* out) {
  __shared__ double sh[32];
  double a[5] = {0, 0, 0, 0, 0};
  long long cnt = 0;
  double mx = 0;
  for (int64_t r = threadIdx.x; r < pk; r += blockDim.x) {
    if (c_ptr) mx = fmax(mx, (double)(c_ptr[r + 1] - c_ptr[r]));
    if (D2) a[0] += D2[r];
    if (dd) a[1] += dd[r];
    if (logd) a[2] += logd[r];
    if (Y2) a[3] += Y2[r];
    if (l1) a[4] += l1[r];
    if (nnz) cnt += nnz[r];
  }
  for (int k = 0; k < 5; ++k) {
    double s = block_sum(a[k], sh);
    if (threadIdx.x == 0) out[k] = s;
  }
  double s = block_sum((double)cnt, sh);
  if (threadIdx.x == 0) {
    out[5] = s;
    out[6] = c_ptr ? (double)c_ptr[pk] : 0.0;
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, sh[w]);
    out[7] = mx;
  }
}

// ---------------------------------------------------------------------------
// Accept: compact C (with new values) into Omega's CSR; warp per row
// ---------------------------------------------------------------------------
template <typename T>
__global__ void compact_kernel(int64_t pk, int64_t r0, const int64_t* __restrict__ c_ptr,
                               const int32_t* __restrict__ c_col, const T* __restrict__ c_wn,
                               const int64_t* __restrict__ om_ptr, int32_t* __restrict__ om_col,
                               T* __restrict__ om_val) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  int64_t out = om_ptr[r];
  const int64_t end = c_ptr[r + 1];
  for (int64_t e0 = c_ptr[r]; e0 < end; e0 += 32) {
    const int64_t e = e0 + lane;
    bool keep = false;
    int32_t cc = 0;
    T v = T(0);
    if (e < end) {
      cc = c_col[e];
      v = c_wn[e];
      keep = (v != T(0)) || (cc == r0 + r);
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int64_t pos = out + __popc(m & ((1u << lane) - 1u));
      om_col[pos] = cc;
      om_val[pos] = v;
    }
    out += __popc(m);
  }
}

template <typename T>
__global__ void identity_kernel(int64_t pk, int64_t r0, int64_t* om_ptr, int32_t* om_col,
                                T* om_val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= pk;
       i += (int64_t)gridDim.x * blockDim.x) {
    om_ptr[i] = i;
    if (i < pk) {
      om_col[i] = (int32_t)(r0 + i);
      om_val[i] = T(1);
    }
  }
}

// ---------------------------------------------------------------------------
// Power iteration for L = sigma_max(S), deterministic:
// u = X v (fixed split partial sums), w = X^T u / n (warp per row),
// rq = v.w, v <- w / ||w||.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void pi_xv_kernel(const T* __restrict__ Xt, int64_t p, int64_t ldk, int64_t rows_per,
                             const double* __restrict__ v, double* __restrict__ part) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= ldk) return;
  const int64_t j0 = blockIdx.y * rows_per, j1 = min(p, j0 + rows_per);
  double s = 0;
  for (int64_t j = j0; j < j1; ++j) s += (double)Xt[j * ldk + m] * v[j];
  part[blockIdx.y * ldk + m] = s;
}

__global__ void pi_sum_parts(const double* __restrict__ part, int64_t nsplit, int64_t ldk,
                             double* __restrict__ u) {
  const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= ldk) return;
  double s = 0;
  for (int64_t q = 0; q < nsplit; ++q) s += part[q * ldk + m];
  u[m] = s;
}

template <typename T>
__global__ void pi_xtu_kernel(const T* __restrict__ Xt, int64_t p, int64_t ldk, int64_t n,
                              const double* __restrict__ u, double* __restrict__ w) {
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (j >= p) return;
  double s = 0;
  for (int64_t m = lane; m < n; m += 32) s += (double)Xt[j * ldk + m] * u[m];
  s = warp_sum(s);
  if (lane == 0) w[j] = s / (double)n;
}




// One pass over X^T for the Lanczos operator w = X (X^T u) / n (ldk <= 1024,
// float X): a warp takes whole rows x_j, t_j = <x_j, u> / n by a warp
// reduction, then w += t_j x_j, with u and the warp's share of w held in
// registers (lane = columns 4 lane + 128 q + v); the next row of the warp is
// loaded while the current one is used. Each block sums its warps in fixed
// order into part[block] (the caller sums the blocks in order):
// deterministic, and X is read once instead of twice.
__global__ void __launch_bounds__(256, 1) gram_fused_kernel(const float* __restrict__ Xt,
                                                            int64_t p, int64_t ldk, int64_t n,
                                                            int64_t rows_per,
                                                            const double* __restrict__ u,
                                                            double* __restrict__ part) {
  __shared__ double sw[1024];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nq = (int)(ldk / 128);          // float4 chunks per lane (<= 8)
  double uv[32], wv[32];
#pragma unroll
  for (int q = 0; q < 8; ++q)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int64_t m = (int64_t)q * 128 + lane * 4 + v;
      uv[q * 4 + v] = (q < nq) ? u[m] : 0.0;
      wv[q * 4 + v] = 0.0;
    }
  const int64_t j0 = (int64_t)blockIdx.x * rows_per, j1 = min(p, j0 + rows_per);
  const double inv_n = 1.0 / (double)n;
  auto load = [&](int64_t j, float4* x) {
#pragma unroll
    for (int q = 0; q < 8; ++q)
      x[q] = (q < nq && j < j1) ? __ldg(reinterpret_cast<const float4*>(Xt + j * ldk + q * 128 +
                                                                       lane * 4))
                                : make_float4(0.f, 0.f, 0.f, 0.f);
  };
  float4 xa[8], xb[8];
  int64_t j = j0 + warp;
  load(j, xa);
  for (; j < j1; j += 8) {
    load(j + 8, xb);                        // next row of this warp in flight
    double d = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      d = fma(uv[q * 4 + 0], (double)xa[q].x, d);
      d = fma(uv[q * 4 + 1], (double)xa[q].y, d);
      d = fma(uv[q * 4 + 2], (double)xa[q].z, d);
      d = fma(uv[q * 4 + 3], (double)xa[q].w, d);
    }
    const double t = warp_sum(d) * inv_n;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      wv[q * 4 + 0] = fma(t, (double)xa[q].x, wv[q * 4 + 0]);
      wv[q * 4 + 1] = fma(t, (double)xa[q].y, wv[q * 4 + 1]);
      wv[q * 4 + 2] = fma(t, (double)xa[q].z, wv[q * 4 + 2]);
      wv[q * 4 + 3] = fma(t, (double)xa[q].w, wv[q * 4 + 3]);
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) xa[q] = xb[q];
  }
  // block sum of the warps' w, fixed order
  for (int w = 0; w < 8; ++w) {
    if (warp == w) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int m = q * 128 + lane * 4 + v;
          if (q < nq) sw[m] = (w == 0 ? 0.0 : sw[m]) + wv[q * 4 + v];
        }
    }
    __syncthreads();
  }
  for (int64_t m = threadIdx.x; m < ldk; m += blockDim.x) part[blockIdx.x * ldk + m] = sw[m];
}

inline int grid_for(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  return (int)(g < cap ? g : cap);
}

}  // namespace

// ===========================================================================
// launchers
// ===========================================================================
int launch_load_xt(int dtype, const void* X, int64_t ldx, int layout, int64_t n, int64_t p,
                   void* Xt, int64_t ldk, int64_t prows, unsigned long long* bad,
                   cudaStream_t st) {
  dim3 blk(32, 8);
  dim3 grd((unsigned)(ldk / 32), (unsigned)std::min<int64_t>(prows / 32, 65535));
  if (dtype == ACCORD_F64)
    load_xt_kernel<double><<<grd, blk, 0, st>>>((const double*)X, ldx, layout, n, p,
                                                (double*)Xt, ldk, prows, bad);
  else
    load_xt_kernel<float><<<grd, blk, 0, st>>>((const float*)X, ldx, layout, n, p, (float*)Xt,
                                               ldk, prows, bad);
  return 1;
}

int launch_split_bf16(const float* src, int64_t elems, __nv_bfloat16* hi, __nv_bfloat16* lo,
                      cudaStream_t st, int drop) {
  const int64_t n4 = elems / 4;
  split_bf16_kernel<<<grid_for(n4, 256, 148 * 64), 256, 0, st>>>(
      reinterpret_cast<const float4*>(src), n4, reinterpret_cast<__nv_bfloat162*>(hi),
      reinterpret_cast<__nv_bfloat162*>(lo), drop);
  return 1;
}

size_t scan_tmp_bytes(int64_t N) {
  const int64_t nb = (N + kScanChunk - 1) / kScanChunk + 1;
  return (size_t)(nb + 1) * sizeof(int64_t);
}

int launch_scan_i32(const int32_t* in, int64_t* out, int64_t N, void* tmp, size_t,
                    cudaStream_t st) {
  const int64_t nb = std::max<int64_t>(1, (N + kScanChunk - 1) / kScanChunk);
  int64_t* bsum = (int64_t*)tmp;
  scan_phase1<<<(unsigned)nb, kScanThreads, 0, st>>>(in, N, bsum);
  scan_phase2<<<1, kScanThreads, 0, st>>>(bsum, nb);
  scan_phase3<<<(unsigned)nb, kScanThreads, 0, st>>>(in, N, bsum, nb, out);
  return 3;
}

int launch_rowsort(int64_t rows, const int64_t* ptr, uint64_t* keys, uint64_t* tmp,
                   int32_t* long_rows, cudaStream_t st) {
  if (rows <= 0) return 0;
  const int warps = 8;
  const size_t smem = (size_t)warps * kWarpSortMax * sizeof(uint64_t);
  static unsigned long long attr_seen = 0;
  if (attr_needed(attr_seen)) {
    cudaFuncSetAttribute(rowsort_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    cudaFuncSetAttribute(rowsort_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(kBlockSortMax * sizeof(uint64_t)));
    attr_done(attr_seen);
  }
  rowsort_warp_kernel<<<(unsigned)((rows + warps - 1) / warps), warps * 32, smem, st>>>(
      rows, ptr, keys, long_rows);
  rowsort_block_kernel<<<148, 1024, kBlockSortMax * sizeof(uint64_t), st>>>(ptr, keys, tmp,
                                                                           long_rows);
  return 2;
}

int launch_finalize(int dtype, int64_t pk, const PoolView& pool, const int64_t* c_ptr,
                    int32_t* rcur, uint64_t* keys, uint64_t* keys_tmp, int32_t* c_col, void* c_g,
                    void* c_w, int32_t* long_rows, cudaStream_t st, const int64_t* sup_ptr,
                    const int32_t* sup_col) {
  int launches = 0;
  {
    const unsigned gx = (unsigned)std::max<int64_t>(1, std::min<int64_t>(pool.chunk / 256, 148 * 8));
    const unsigned gy = (unsigned)std::max<int64_t>(1, std::min<int64_t>(pool.nchunks, 65535));
    scatter_kernel<<<dim3(gx, gy), 256, 0, st>>>(pool.row, pool.col, pool.chunk, pool.nchunks,
                                                 pool.chunk_next, pool.chunk_fill, c_ptr, rcur,
                                                 keys);
  }
  ++launches;
  if (sup_ptr) {   // supp Omega into the same row segments (filter path)
    support_scatter_kernel<<<(unsigned)((pk + 7) / 8), 256, 0, st>>>(pk, sup_ptr, sup_col, c_ptr,
                                                                     rcur, keys);
    ++launches;
  }
  launches += launch_rowsort(pk, c_ptr, keys, keys_tmp, long_rows, st);
  if (dtype == ACCORD_F64)
    gather_kernel<double><<<148 * 8, 256, 0, st>>>(pk, c_ptr, keys, (const double*)pool.g,
                                                   (const double*)pool.w, c_col, (double*)c_g,
                                                   (double*)c_w);
  else
    gather_kernel<float><<<148 * 8, 256, 0, st>>>(pk, c_ptr, keys, (const float*)pool.g,
                                                  (const float*)pool.w, c_col, (float*)c_g,
                                                  (float*)c_w);
  return launches + 1;
}

int launch_support_count(int64_t pk, const int64_t* om_ptr, int32_t* row_cnt, cudaStream_t st) {
  if (pk == 0) return 0;
  support_count_kernel<<<grid_for(pk, 256), 256, 0, st>>>(pk, om_ptr, row_cnt);
  return 1;
}

int launch_dedupe(int64_t pk, const int64_t* ptr, const uint64_t* keys, int32_t* cnt,
                  int64_t* optr, int32_t* col, void* scan_tmp, size_t scan_tmp_bytes,
                  cudaStream_t st) {
  if (pk == 0) return 0;
  const unsigned g = (unsigned)((pk + 7) / 8);
  dedupe_count_kernel<<<g, 256, 0, st>>>(pk, ptr, keys, cnt);
  int l = 1 + launch_scan_i32(cnt, optr, pk, scan_tmp, scan_tmp_bytes, st);
  dedupe_write_kernel<<<g, 256, 0, st>>>(pk, ptr, keys, optr, col);
  return l + 1;
}

int launch_prox(int dtype, int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
                const void* c_g, const void* c_w, void* c_wn, double tau, double lam,
                double* row_dd, double* row_l1, double* row_logd, int32_t* row_nnz,
                cudaStream_t st, const ProxItems* items) {
  const ProxItems pi = items ? *items
                            : ProxItems{nullptr, nullptr, 0, 0, nullptr, nullptr, nullptr, nullptr};
  const int warps = 8;
  const int64_t nw = pi.itm_ptr ? pi.n_items : pk;
  const unsigned g = (unsigned)std::max<int64_t>(1, (nw + warps - 1) / warps);
  if (dtype == ACCORD_F64)
    prox_kernel<double><<<g, warps * 32, 0, st>>>(pk, r0, c_ptr, c_col, (const double*)c_g,
                                                  (const double*)c_w, (double*)c_wn, tau, lam,
                                                  row_dd, row_l1, row_logd, row_nnz, pi);
  else
    prox_kernel<float><<<g, warps * 32, 0, st>>>(pk, r0, c_ptr, c_col, (const float*)c_g,
                                                 (const float*)c_w, (float*)c_wn, tau, lam,
                                                 row_dd, row_l1, row_logd, row_nnz, pi);
  if (!pi.itm_ptr) return 1;
  prox_combine_kernel<<<grid_for(pk, 256), 256, 0, st>>>(pk, pi, row_dd, row_l1, row_logd,
                                                         row_nnz);
  return 2;
}

int launch_spmm(int dtype, int64_t pk, int64_t n, int64_t ldk, const int64_t* ptr,
                const int32_t* col, const void* wn, const void* wo, const void* Xt, void* Yout,
                __nv_bfloat16* Yhi, __nv_bfloat16* Ylo, float* row_A, float* row_B,
                double* row_D2, double* row_Y2, cudaStream_t st, const SpmmRing* ring,
                int ydrop) {
  const SpmmRing rg = ring ? *ring : SpmmRing{0, 0, nullptr, nullptr, 1, 1};
  const int V = dtype == ACCORD_F64 ? 2 : 4;
  int threads = (int)std::min<int64_t>(kSpmmMaxThreads, round_up(ldk / V, 32));
  if (pk == 0) return 0;
  if (dtype == ACCORD_F64) {
    spmm_kernel<double, false><<<(unsigned)pk, threads, 0, st>>>(
        pk, n, ldk, ptr, col, (const double*)wn, (const double*)wo, (const double*)Xt,
        (double*)Yout, nullptr, nullptr, nullptr, nullptr, row_D2, row_Y2, rg, 0);
  } else if (Yhi) {
    spmm_kernel<float, true><<<(unsigned)pk, threads, 0, st>>>(
        pk, n, ldk, ptr, col, (const float*)wn, (const float*)wo, (const float*)Xt,
        (float*)Yout, Yhi, Ylo, row_A, row_B, row_D2, row_Y2, rg, Ylo ? 0 : ydrop);
  } else {
    spmm_kernel<float, false><<<(unsigned)pk, threads, 0, st>>>(
        pk, n, ldk, ptr, col, (const float*)wn, (const float*)wo, (const float*)Xt,
        (float*)Yout, nullptr, nullptr, nullptr, nullptr, row_D2, row_Y2, rg, 0);
  }
  return 1;
}

int launch_refine(int dtype, int64_t pk, int64_t n, int64_t ldk, const int64_t* c_ptr,
                  const int32_t* c_col, const void* Y, const void* Xt, void* c_g,
                  cudaStream_t st, int64_t v0, int64_t v1, const int64_t* itm_ptr,
                  int64_t n_items, int64_t L, const int32_t* item_row, int ff, int sym) {
  const unsigned grid = (unsigned)(itm_ptr ? n_items : pk);
  if (pk == 0) return 0;
  // f32: Y_i staged as float64 (kArith 2) unless ACCORD_REFINE=f32 (A-B)
  static const bool yd = [] {
    const char* e = std::getenv("ACCORD_REFINE");
    return !(e && std::strcmp(e, "f32") == 0);
  }();
  const bool stage_d = dtype != ACCORD_F64 && ff != 1 && yd;
  // (the float64 staging's conflict-free layout fills whole 128-element blocks)
  size_t smem = stage_d ? (size_t)((ldk + 127) / 128 * 128) * 8
                        : (size_t)ldk * (dtype == ACCORD_F64 ? 8 : 4);
  const int y_global = smem > 200 * 1024 ? 1 : 0;
  if (y_global) smem = 0;
  // threads per block (warps share the item's candidates): ACCORD_REFINE_THREADS (A-B);
  // a c5 item has ~13 candidates, so 4 warps keep each warp busier than 8
  static const int thr = [] {
    const char* e = std::getenv("ACCORD_REFINE_THREADS");
    const int t = e ? std::atoi(e) : 128;   // c5: 128 -> 14.2 ms, 256 -> 16.6-17.1 ms
    return (t == 64 || t == 128 || t == 256) ? t : 128;
  }();
  static unsigned long long attr_seen = 0;
  if (attr_needed(attr_seen)) {
    cudaFuncSetAttribute(refine_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(refine_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(refine_kernel<float, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(refine_kernel<float, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_done(attr_seen);
  }
  if (dtype == ACCORD_F64)
    refine_kernel<double><<<grid, thr, smem, st>>>(pk, n, ldk, c_ptr, c_col,
                                                   (const double*)Y, (const double*)Xt,
                                                   (double*)c_g, v0, v1, itm_ptr, L, item_row,
                                                   y_global, sym);
  else if (ff == 1)
    refine_kernel<float, 1><<<grid, thr, smem, st>>>(pk, n, ldk, c_ptr, c_col,
                                                        (const float*)Y, (const float*)Xt,
                                                        (float*)c_g, v0, v1, itm_ptr, L, item_row,
                                                        y_global, sym);
  else if (stage_d)
    refine_kernel<float, 2><<<grid, thr, smem, st>>>(pk, n, ldk, c_ptr, c_col,
                                                        (const float*)Y, (const float*)Xt,
                                                        (float*)c_g, v0, v1, itm_ptr, L, item_row,
                                                        y_global, sym);
  else
    refine_kernel<float><<<grid, thr, smem, st>>>(pk, n, ldk, c_ptr, c_col,
                                                  (const float*)Y, (const float*)Xt,
                                                  (float*)c_g, v0, v1, itm_ptr, L, item_row,
                                                  y_global, sym);
  if (!sym) return 1;
  const unsigned mg = (unsigned)((pk + 7) / 8);
  if (dtype == ACCORD_F64)
    sym_mirror_kernel<double><<<mg, 256, 0, st>>>(pk, ldk, c_ptr, c_col, (const double*)Y,
                                                  (const double*)Xt, (double*)c_g, 1.0 / (double)n,
                                                  sym == 2);
  else
    sym_mirror_kernel<float><<<mg, 256, 0, st>>>(pk, ldk, c_ptr, c_col, (const float*)Y,
                                                 (const float*)Xt, (float*)c_g, 1.0 / (double)n,
                                                 sym == 2);
  return 2;
}

int launch_lookup(int dtype, int64_t pk, const int64_t* c_ptr, const int32_t* c_col,
                  const int64_t* om_ptr, const int32_t* om_col, const void* om_val, void* c_w,
                  cudaStream_t st, const ProxItems* items) {
  const ProxItems pi = items ? *items
                            : ProxItems{nullptr, nullptr, 0, 0, nullptr, nullptr, nullptr, nullptr};
  const int64_t nw = pi.itm_ptr ? pi.n_items : pk;
  const unsigned g = (unsigned)std::max<int64_t>(1, (nw + 7) / 8);
  if (dtype == ACCORD_F64)
    lookup_kernel<double><<<g, 256, 0, st>>>(pk, c_ptr, c_col, om_ptr, om_col,
                                             (const double*)om_val, (double*)c_w, pi);
  else
    lookup_kernel<float><<<g, 256, 0, st>>>(pk, c_ptr, c_col, om_ptr, om_col,
                                            (const float*)om_val, (float*)c_w, pi);
  return 1;
}

int launch_kkt(int dtype, int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
               const void* c_g, const void* c_w, double lam, double* row_max, double* out,
               cudaStream_t st) {
  const unsigned g = (unsigned)((pk + 7) / 8);
  if (dtype == ACCORD_F64)
    kkt_kernel<double><<<g, 256, 0, st>>>(pk, r0, c_ptr, c_col, (const double*)c_g,
                                          (const double*)c_w, lam, row_max);
  else
    kkt_kernel<float><<<g, 256, 0, st>>>(pk, r0, c_ptr, c_col, (const float*)c_g,
                                         (const float*)c_w, lam, row_max);
  reduce_max_kernel<<<1, 1024, 0, st>>>(pk, row_max, out);
  return 2;
}

int launch_row_ab(int64_t pk, int64_t ldk, const float* Xt_rows, float* row_A, float* row_B,
                  cudaStream_t st, int drop) {
  if (pk == 0) return 0;
  xrow_ab_kernel<<<(unsigned)((pk + 7) / 8), 256, 0, st>>>(pk, ldk, Xt_rows, row_A, row_B, drop);
  return 1;
}

int launch_cand_dot_max(int dtype, int64_t pk, int64_t r0, int64_t n, int64_t ldk,
                        const int64_t* c_ptr, const int32_t* c_col, const void* Xi, const void* Xt,
                        int64_t v0, int64_t v1, int accumulate, double* row_max, double* out,
                        cudaStream_t st) {
  if (pk == 0) return 0;
  const unsigned g = (unsigned)((pk + 7) / 8);
  if (dtype == ACCORD_F64)
    cand_dot_max_kernel<double><<<g, 256, 0, st>>>(pk, r0, n, ldk, c_ptr, c_col,
                                                   (const double*)Xi, (const double*)Xt, v0, v1,
                                                   accumulate, row_max);
  else
    cand_dot_max_kernel<float><<<g, 256, 0, st>>>(pk, r0, n, ldk, c_ptr, c_col, (const float*)Xi,
                                                  (const float*)Xt, v0, v1, accumulate, row_max);
  if (out) reduce_max_kernel<<<1, 1024, 0, st>>>(pk, row_max, out);
  return out ? 2 : 1;
}

int launch_gram_offdiag_max(int dtype, int64_t pk, int64_t r0, int64_t n, int64_t ldk,
                            const void* Xi, const void* Xt, int64_t v0, int64_t v1, int accumulate,
                            double* row_max, double* out, cudaStream_t st) {
  if (pk == 0) return 0;
  const size_t T = dtype == ACCORD_F64 ? 8 : 4;
  const size_t smem = (size_t)ldk * T;
  static unsigned long long attr_seen = 0;
  if (attr_needed(attr_seen)) {
    cudaFuncSetAttribute(gram_offdiag_max_kernel<float>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(gram_offdiag_max_kernel<double>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_done(attr_seen);
  }
  if (dtype == ACCORD_F64)
    gram_offdiag_max_kernel<double><<<(unsigned)pk, 256, smem, st>>>(
        pk, r0, n, ldk, (const double*)Xi, (const double*)Xt, v0, v1, accumulate, row_max);
  else
    gram_offdiag_max_kernel<float><<<(unsigned)pk, 256, smem, st>>>(
        pk, r0, n, ldk, (const float*)Xi, (const float*)Xt, v0, v1, accumulate, row_max);
  if (out) reduce_max_kernel<<<1, 1024, 0, st>>>(pk, row_max, out);
  return out ? 2 : 1;
}

int launch_mirror_count(int64_t n, const int32_t* row, const int64_t* rb, int P,
                        unsigned long long* cnt, cudaStream_t st) {
  if (n == 0) return 0;
  mirror_count_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, row, rb, P, cnt);
  return 1;
}

int launch_mirror_scatter(int64_t n, const int32_t* row, const int32_t* col, const int64_t* rb,
                          int P, unsigned long long* cursor, int32_t* out, cudaStream_t st) {
  if (n == 0) return 0;
  mirror_scatter_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, row, col, rb, P, cursor, out);
  return 1;
}

int launch_mirror_append(int64_t n, const int32_t* in, int64_t r0, int32_t* prow, int32_t* pcol,
                         int64_t start, int32_t* row_cnt, cudaStream_t st) {
  if (n == 0) return 0;
  mirror_append_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, in, r0, prow, pcol, start, row_cnt);
  return 1;
}

__global__ void spin_kernel(long long ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if ((long long)(t - t0) >= ns) break;
  }
}

int launch_spin(int ms, cudaStream_t st) {
  if (ms <= 0) return 0;
  spin_kernel<<<1, 1, 0, st>>>((long long)ms * 1000000ll);
  return 1;
}

int launch_col_norms(int64_t p, int64_t ldk, const float* Xt, float2* col_sd, cudaStream_t st,
                     int drop) {
  col_norms_kernel<<<(unsigned)((p + 7) / 8), 256, 0, st>>>(p, ldk, Xt, col_sd, drop);
  return 1;
}

int launch_omega_stats(int dtype, int64_t pk, int64_t r0, const int64_t* ptr, const int32_t* col,
                       const void* val, double* row_l1, double* row_logd, int32_t* row_nnz,
                       int32_t* bad_diag, cudaStream_t st) {
  const int warps = 8;
  const unsigned g = (unsigned)((pk + warps - 1) / warps);
  if (dtype == ACCORD_F64)
    omega_stats_kernel<double><<<g, warps * 32, 0, st>>>(pk, r0, ptr, col, (const double*)val,
                                                         row_l1, row_logd, row_nnz, bad_diag);
  else
    omega_stats_kernel<float><<<g, warps * 32, 0, st>>>(pk, r0, ptr, col, (const float*)val,
                                                        row_l1, row_logd, row_nnz, bad_diag);
  return 1;
}

int launch_reduce_rows(int64_t pk, const double* row_D2, const double* row_dd,
                       const double* row_logd, const double* row_Y2, const double* row_l1,
                       const int32_t* row_nnz, const int64_t* c_ptr, double* out,
                       cudaStream_t st) {
  reduce_rows_kernel<<<1, 1024, 0, st>>>(pk, row_D2, row_dd, row_logd, row_Y2, row_l1, row_nnz,
                                         c_ptr, out);
  return 1;
}

int launch_compact(int dtype, int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
                   const void* c_wn, const int64_t* om_ptr, int32_t* om_col, void* om_val,
                   cudaStream_t st) {
  const int warps = 8;
  const unsigned g = (unsigned)((pk + warps - 1) / warps);
  if (dtype == ACCORD_F64)
    compact_kernel<double><<<g, warps * 32, 0, st>>>(pk, r0, c_ptr, c_col, (const double*)c_wn,
                                                     om_ptr, om_col, (double*)om_val);
  else
    compact_kernel<float><<<g, warps * 32, 0, st>>>(pk, r0, c_ptr, c_col, (const float*)c_wn,
                                                    om_ptr, om_col, (float*)om_val);
  return 1;
}

int launch_identity(int dtype, int64_t pk, int64_t r0, int64_t* om_ptr, int32_t* om_col,
                    void* om_val, cudaStream_t st) {
  if (dtype == ACCORD_F64)
    identity_kernel<double><<<grid_for(pk + 1, 256), 256, 0, st>>>(pk, r0, om_ptr, om_col,
                                                                   (double*)om_val);
  else
    identity_kernel<float><<<grid_for(pk + 1, 256), 256, 0, st>>>(pk, r0, om_ptr, om_col,
                                                                  (float*)om_val);
  return 1;
}

// w = X (X^T u) / n for an n-vector u (ldk entries, zero past n): the Gram
// operator of the samples, whose nonzero spectrum is that of S = X^T X / n
// (L = sigma_max(S)). t: scratch of p doubles; part: nsplit x ldk.
int launch_gram_apply(int dtype, const void* Xt, int64_t p, int64_t n, int64_t ldk,
                      const double* u, double* t, double* part, int64_t nsplit, double* w,
                      cudaStream_t st) {
  if (p <= 0) {
    cudaMemsetAsync(w, 0, ldk * sizeof(double), st);
    return 0;
  }
  if (dtype == ACCORD_F32 && ldk <= 1024 && ldk % 128 == 0 && !std::getenv("ACCORD_GRAM_2PASS")) {
    // single pass: one block of contiguous rows per SM (255 registers per
    // thread: one resident block), part holds nb x ldk (nb <= nsplit)
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t nb = std::max<int64_t>(1, std::min<int64_t>(nsplit, sms));
    const int64_t rows_per = (p + nb - 1) / nb;
    gram_fused_kernel<<<(unsigned)nb, 256, 0, st>>>((const float*)Xt, p, ldk, n, rows_per, u,
                                                    part);
    pi_sum_parts<<<(unsigned)((ldk + 255) / 256), 256, 0, st>>>(part, nb, ldk, w);
    return 2;
  }
  const unsigned g3 = (unsigned)((p + 7) / 8);
  if (dtype == ACCORD_F64)
    pi_xtu_kernel<double><<<g3, 256, 0, st>>>((const double*)Xt, p, ldk, n, u, t);
  else
    pi_xtu_kernel<float><<<g3, 256, 0, st>>>((const float*)Xt, p, ldk, n, u, t);
  const int64_t rows_per = (p + nsplit - 1) / nsplit;
  dim3 g1((unsigned)((ldk + 255) / 256), (unsigned)nsplit);
  if (dtype == ACCORD_F64)
    pi_xv_kernel<double><<<g1, 256, 0, st>>>((const double*)Xt, p, ldk, rows_per, t, part);
  else
    pi_xv_kernel<float><<<g1, 256, 0, st>>>((const float*)Xt, p, ldk, rows_per, t, part);
  pi_sum_parts<<<(unsigned)((ldk + 255) / 256), 256, 0, st>>>(part, nsplit, ldk, w);
  return 3;
}

// ---------------------------------------------------------------------------
// Line search from Omega = I (the first iteration of a solve).
// Off the diagonal omega_ik = 0, so prox gives omega+_ik(tau) =
// S_{tau lam}(-tau g_ik) = tau t_ik with t_ik = S_lam(-g_ik): exactly, for a
// power-of-two tau (the scaling commutes with every rounding in prox_kernel).
// Hence Y+_i(tau) = a_i(tau) x_i + tau z_i with z = T X^T (T = off-diagonal
// t), and every trial's ||Y+_i||^2 and ||D_i||^2 follow from three dot
// products per row: one SpMM pass serves all trials of the iteration.
// ---------------------------------------------------------------------------
__global__ void diag_t_kernel(int64_t pk, int64_t r0, const int64_t* __restrict__ c_ptr,
                              const int32_t* __restrict__ c_col, const float* __restrict__ c_g,
                              double lam, float* __restrict__ c_t) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  const int64_t gi = r0 + r;
  for (int64_t e = c_ptr[r] + lane; e < c_ptr[r + 1]; e += 32) {
    const double y = -(double)c_g[e];     // prox_kernel's y at tau = 1, omega = 0
    const double m = fabs(y) - lam;
    c_t[e] = (c_col[e] == gi || !(m > 0.0)) ? 0.f : (float)copysign(m, y);
  }
}

// per row: ||x_i||^2, <x_i, z_i>, ||z_i||^2 (float64), warp per row
__global__ void diag_dots_kernel(int64_t pk, int64_t ldk, int64_t xrow0,
                                 const float* __restrict__ Xt, const float* __restrict__ Z,
                                 double* __restrict__ xx, double* __restrict__ xz,
                                 double* __restrict__ zz) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  const float4* x = reinterpret_cast<const float4*>(Xt + (xrow0 + r) * ldk);
  const float4* z = reinterpret_cast<const float4*>(Z + r * ldk);
  double a = 0.0, b = 0.0, c = 0.0;
  for (int64_t m = lane; m < ldk / 4; m += 32) {
    const float4 xv = x[m], zv = z[m];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const double xd = vget(xv, v), zd = vget(zv, v);
      a += xd * xd;
      b += xd * zd;
      c += zd * zd;
    }
  }
  a = warp_sum(a);
  b = warp_sum(b);
  c = warp_sum(c);
  if (lane == 0) {
    xx[r] = a;
    xz[r] = b;
    zz[r] = c;
  }
}

// one trial: a_i = omega+_ii(tau) from the prox output on C (diagonal always
// in C), ||Y+_i||^2 and ||D_i||^2 = ||(a_i - omega_ii) x_i + tau z_i||^2
__global__ void diag_trial_kernel(int64_t pk, int64_t r0, const int64_t* __restrict__ c_ptr,
                                  const int32_t* __restrict__ c_col,
                                  const float* __restrict__ c_w, const float* __restrict__ c_wn,
                                  double tau, const double* __restrict__ xx,
                                  const double* __restrict__ xz, const double* __restrict__ zz,
                                  double* __restrict__ row_Y2, double* __restrict__ row_D2,
                                  double* __restrict__ row_a) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < pk;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = lower_bound_col(c_col, c_ptr[r], c_ptr[r + 1], (int32_t)(r0 + r));
    const double a = c_wn[e], d = a - (double)c_w[e];
    const double X2 = xx[r], XZ = xz[r], Z2 = zz[r];
    row_Y2[r] = fmax(0.0, a * a * X2 + 2.0 * a * tau * XZ + tau * tau * Z2);
    row_D2[r] = fmax(0.0, d * d * X2 + 2.0 * d * tau * XZ + tau * tau * Z2);
    row_a[r] = a;
  }
}

// the accepted trial: Y+_i = a_i x_i + tau z_i (in place over Z), the bf16
// operand and the filter's row norms, as the SpMM epilogue writes them
__global__ void diag_apply_kernel(int64_t pk, int64_t ldk, int64_t xrow0,
                                  const float* __restrict__ Xt, float* __restrict__ Y,
                                  __nv_bfloat16* __restrict__ Yhi,
                                  const double* __restrict__ row_a, double tau,
                                  float* __restrict__ row_A, float* __restrict__ row_B,
                                  int ydrop) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= pk) return;
  const double a = row_a[r];
  const float* x = Xt + (xrow0 + r) * ldk;
  float* y = Y + r * ldk;
  double a2 = 0.0, b2 = 0.0;
  for (int64_t m = lane; m < ldk; m += 32) {
    const float v = (float)(a * (double)x[m] + tau * (double)y[m]);
    y[m] = v;
    const __nv_bfloat16 h = filter_bf16_x(v, ydrop);
    Yhi[r * ldk + m] = h;
    const double e = (double)v - (double)__bfloat162float(h);
    a2 += e * e;
    b2 += (double)v * (double)v;
  }
  a2 = warp_sum(a2);
  b2 = warp_sum(b2);
  if (lane == 0) {
    row_A[r] = __double2float_ru(sqrt(a2) * (1.0 + 1e-12));
    row_B[r] = __double2float_ru(sqrt(b2) * (1.0 + 1e-12));
  }
}

int launch_diag_t(int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
                  const float* c_g, double lam, float* c_t, cudaStream_t st) {
  if (pk == 0) return 0;
  diag_t_kernel<<<(unsigned)((pk + 7) / 8), 256, 0, st>>>(pk, r0, c_ptr, c_col, c_g, lam, c_t);
  return 1;
}

int launch_diag_dots(int64_t pk, int64_t ldk, int64_t xrow0, const float* Xt, const float* Z,
                     double* xx, double* xz, double* zz, cudaStream_t st) {
  if (pk == 0) return 0;
  diag_dots_kernel<<<(unsigned)((pk + 7) / 8), 256, 0, st>>>(pk, ldk, xrow0, Xt, Z, xx, xz, zz);
  return 1;
}

int launch_diag_trial(int64_t pk, int64_t r0, const int64_t* c_ptr, const int32_t* c_col,
                      const float* c_w, const float* c_wn, double tau, const double* xx,
                      const double* xz, const double* zz, double* row_Y2, double* row_D2,
                      double* row_a, cudaStream_t st) {
  if (pk == 0) return 0;
  diag_trial_kernel<<<grid_for(pk, 256, 148 * 8), 256, 0, st>>>(
      pk, r0, c_ptr, c_col, c_w, c_wn, tau, xx, xz, zz, row_Y2, row_D2, row_a);
  return 1;
}

int launch_diag_apply(int64_t pk, int64_t ldk, int64_t xrow0, const float* Xt, float* Y,
                      __nv_bfloat16* Yhi, const double* row_a, double tau, float* row_A,
                      float* row_B, cudaStream_t st, int ydrop) {
  if (pk == 0) return 0;
  diag_apply_kernel<<<(unsigned)((pk + 7) / 8), 256, 0, st>>>(pk, ldk, xrow0, Xt, Y, Yhi, row_a,
                                                               tau, row_A, row_B, ydrop);
  return 1;
}

}  // namespace accord

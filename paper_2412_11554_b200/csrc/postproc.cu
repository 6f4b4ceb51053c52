// NEXT(4): on-device post-processing of the estimate.
//
//   Theta-hat = T^{-1}(Omega-hat) = Omega_D Omega,  theta_ij = omega_ii omega_ij
//
//   rho-hat_ij = -1/2 (omega_ij / omega_jj + omega_ji / omega_ii),  i != j
//
//
// Theta keeps Omega's CSR structure. rho needs the transpose: its support is
// supp(Omega) U supp(Omega^T) off the diagonal. Every kernel here reads the
// GLOBAL CSR (all p rows, sorted columns, diagonal stored) and produces the
// output rows [a, b). Arithmetic in double, rounded once to the context type.
#include "accord_internal.h"

namespace accord {

namespace {

// value of (row, c) in a sorted CSR row, 0 if absent
template <typename T>
__device__ __forceinline__ double csr_at(const int64_t* __restrict__ ptr,
                                         const int32_t* __restrict__ col,
                                         const T* __restrict__ val, int64_t row, int32_t c,
                                         bool* found = nullptr) {
  int64_t lo = ptr[row], hi = ptr[row + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (col[mid] < c) lo = mid + 1; else hi = mid;
  }
  const bool f = lo < ptr[row + 1] && col[lo] == c;
  if (found) *found = f;
  return f ? (double)val[lo] : 0.0;
}

// d[i] = omega_ii for the CSR's rows (row i holds global row i + off); bad = 1
// if some omega_ii is not > 0
template <typename T>
__global__ void diag_kernel(int64_t rows, int64_t off, const int64_t* __restrict__ ptr,
                            const int32_t* __restrict__ col, const T* __restrict__ val,
                            double* __restrict__ d, int32_t* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double w = csr_at(ptr, col, val, i, (int32_t)(i + off));
    d[i] = w;
    if (!(w > 0.0)) atomicOr(bad, 1);
  }
}

// theta_ij = omega_ii omega_ij on rows [a, b) of the global CSR (same structure)
template <typename T>
__global__ void theta_kernel(int64_t a, int64_t b, const int64_t* __restrict__ ptr,
                             const int32_t* __restrict__ col, const T* __restrict__ val,
                             const double* __restrict__ d, T* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t i = a + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= b) return;
  const double di = d[i];
  const int64_t base = ptr[a];
  for (int64_t e = ptr[i] + lane; e < ptr[i + 1]; e += 32)
    out[e - base] = (T)(di * (double)val[e]);
}

// Pass 1 (warp per global row k): own[k-a] = off-diagonal count of row k (k in
// [a,b)); for every stored (k, i), i != k, i in [a,b), with (i, k) absent:
// one extra entry of output row i (it comes from the transpose).
template <typename T>
__global__ void pcorr_count_kernel(int64_t p, int64_t a, int64_t b,
                                   const int64_t* __restrict__ ptr,
                                   const int32_t* __restrict__ col, const T* __restrict__ val,
                                   int32_t* __restrict__ own, int32_t* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= p) return;
  int mine = 0;
  for (int64_t e = ptr[k] + lane; e < ptr[k + 1]; e += 32) {
    const int32_t i = col[e];
    if (i == k) continue;
    ++mine;
    if (i >= a && i < b) {
      bool f;
      csr_at(ptr, col, val, i, (int32_t)k, &f);
      if (!f) atomicAdd(&cnt[i - a], 1);
    }
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if (lane == 0 && k >= a && k < b) {
    own[k - a] = mine;
    atomicAdd(&cnt[k - a], mine);
  }
}

// Pass 2 (warp per global row k): own off-diagonal columns of row k in order,
// then the transposed extras appended behind them (unordered; sorted next).
template <typename T>
__global__ void pcorr_fill_kernel(int64_t p, int64_t a, int64_t b,
                                  const int64_t* __restrict__ ptr,
                                  const int32_t* __restrict__ col, const T* __restrict__ val,
                                  const int32_t* __restrict__ own,
                                  const int64_t* __restrict__ optr, int32_t* __restrict__ ext,
                                  uint64_t* __restrict__ keys) {
  const int lane = threadIdx.x & 31;
  const int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (k >= p) return;
  const bool in = k >= a && k < b;
  int64_t wpos = in ? optr[k - a] : 0;
  for (int64_t e0 = ptr[k]; e0 < ptr[k + 1]; e0 += 32) {
    const int64_t e = e0 + lane;
    const bool valid = e < ptr[k + 1];
    const int32_t i = valid ? col[e] : -1;
    const bool offd = valid && i != k;
    if (in) {
      const unsigned m = __ballot_sync(0xffffffffu, offd);
      if (offd) keys[wpos + __popc(m & ((1u << lane) - 1u))] = (uint64_t)(uint32_t)i << 32;
      wpos += __popc(m);
    }
    if (offd && i >= a && i < b) {
      bool f;
      csr_at(ptr, col, val, i, (int32_t)k, &f);
      if (!f) {
        const int64_t pos = optr[i - a] + own[i - a] + atomicAdd(&ext[i - a], 1);
        keys[pos] = (uint64_t)(uint32_t)k << 32;
      }
    }
  }
}

// Pass 3 (warp per output row i): rho_ik from the sorted keys.
template <typename T>
__global__ void pcorr_value_kernel(int64_t a, int64_t b, const int64_t* __restrict__ ptr,
                                   const int32_t* __restrict__ col, const T* __restrict__ val,
                                   const double* __restrict__ d,
                                   const int64_t* __restrict__ optr,
                                   const uint64_t* __restrict__ keys, int32_t* __restrict__ ocol,
                                   T* __restrict__ oval) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t i = a + r;
  if (i >= b) return;
  const double di = d[i];
  for (int64_t e = optr[r] + lane; e < optr[r + 1]; e += 32) {
    const int32_t k = (int32_t)(keys[e] >> 32);
    const double wik = csr_at(ptr, col, val, i, k);
    const double wki = csr_at(ptr, col, val, (int64_t)k, (int32_t)i);
    ocol[e] = k;
    oval[e] = (T)(-0.5 * (wik / d[k] + wki / di));
  }
}

inline unsigned warp_grid(int64_t rows, int warps) {
  return (unsigned)std::max<int64_t>(1, (rows + warps - 1) / warps);
}

}  // namespace

int launch_diag(int dtype, int64_t rows, int64_t off, const int64_t* ptr, const int32_t* col,
                const void* val, double* d, int32_t* bad, cudaStream_t st) {
  if (rows <= 0) return 0;
  const unsigned g =
      (unsigned)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (rows + 255) / 256));
  if (dtype == ACCORD_F64)
    diag_kernel<double><<<g, 256, 0, st>>>(rows, off, ptr, col, (const double*)val, d, bad);
  else
    diag_kernel<float><<<g, 256, 0, st>>>(rows, off, ptr, col, (const float*)val, d, bad);
  return 1;
}

int launch_theta(int dtype, int64_t a, int64_t b, const int64_t* ptr, const int32_t* col,
                 const void* val, const double* d, void* out, cudaStream_t st) {
  if (b <= a) return 0;
  if (dtype == ACCORD_F64)
    theta_kernel<double><<<warp_grid(b - a, 8), 256, 0, st>>>(a, b, ptr, col,
                                                              (const double*)val, d,
                                                              (double*)out);
  else
    theta_kernel<float><<<warp_grid(b - a, 8), 256, 0, st>>>(a, b, ptr, col, (const float*)val,
                                                             d, (float*)out);
  return 1;
}

int launch_pcorr_count(int dtype, int64_t p, int64_t a, int64_t b, const int64_t* ptr,
                       const int32_t* col, const void* val, int32_t* own, int32_t* cnt,
                       cudaStream_t st) {
  if (dtype == ACCORD_F64)
    pcorr_count_kernel<double><<<warp_grid(p, 8), 256, 0, st>>>(p, a, b, ptr, col,
                                                                (const double*)val, own, cnt);
  else
    pcorr_count_kernel<float><<<warp_grid(p, 8), 256, 0, st>>>(p, a, b, ptr, col,
                                                               (const float*)val, own, cnt);
  return 1;
}

int launch_pcorr_fill(int dtype, int64_t p, int64_t a, int64_t b, const int64_t* ptr,
                      const int32_t* col, const void* val, const int32_t* own,
                      const int64_t* optr, int32_t* ext, uint64_t* keys, cudaStream_t st) {
  if (dtype == ACCORD_F64)
    pcorr_fill_kernel<double><<<warp_grid(p, 8), 256, 0, st>>>(
        p, a, b, ptr, col, (const double*)val, own, optr, ext, keys);
  else
    pcorr_fill_kernel<float><<<warp_grid(p, 8), 256, 0, st>>>(
        p, a, b, ptr, col, (const float*)val, own, optr, ext, keys);
  return 1;
}

int launch_pcorr_value(int dtype, int64_t a, int64_t b, const int64_t* ptr, const int32_t* col,
                       const void* val, const double* d, const int64_t* optr,
                       const uint64_t* keys, int32_t* ocol, void* oval, cudaStream_t st) {
  if (b <= a) return 0;
  if (dtype == ACCORD_F64)
    pcorr_value_kernel<double><<<warp_grid(b - a, 8), 256, 0, st>>>(
        a, b, ptr, col, (const double*)val, d, optr, keys, ocol, (double*)oval);
  else
    pcorr_value_kernel<float><<<warp_grid(b - a, 8), 256, 0, st>>>(
        a, b, ptr, col, (const float*)val, d, optr, keys, ocol, (float*)oval);
  return 1;
}

}  // namespace accord

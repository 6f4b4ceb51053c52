// Gradient GEMM on CUDA cores with the fused candidate epilogue (a2 + a3,
// reference path and the only float64 path: tcgen05 has no f64 kind).
//
//   G_ik = (1/n) sum_m Y_im Xt_km     (Y = Omega X^T, two-step gradient)
//   emit (i, k, G_ik, omega_ik) iff k == i, omega_ik != 0, or |G_ik| > lambda
//
// The emitted set C is a superset of supp Omega+(tau) for every tau > 0
// (derived from Eq. 3.5: for omega_ik = 0, S_{tau lam}(-tau G_ik) != 0 iff
// |G_ik| > lam), so the line search never recomputes the GEMM. The dense p x p
// product never reaches HBM.
#include "accord_internal.h"

namespace accord {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename T>
__device__ __forceinline__ T lookup_omega(const OmegaView& om, int64_t r, int32_t k) {
  int64_t lo = om.ptr[r], hi = om.ptr[r + 1];
  const T* val = (const T*)om.val;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int32_t c = om.col[mid];
    if (c == k) return val[mid];
    if (c < k) lo = mid + 1; else hi = mid;
  }
  return T(0);
}

template <typename T>
__global__ void __launch_bounds__(256)
gemm_simt_kernel(const T* __restrict__ Y, const T* __restrict__ Xt, int64_t ldk, int64_t kdim,
                 EpiParams ep, OmegaView om, PoolView pool) {
  __shared__ T As[BK][BM + 4];
  __shared__ T Bs[BK][BN + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;   // n0: slab row
  const int64_t ncols = ep.col_end - ep.col_base;
  T acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = T(0);

  // loader mapping: 256 threads load 64 rows x 16 k of A and of B
  const int lr = threadIdx.x >> 2;          // 0..63
  const int lk = (threadIdx.x & 3) * 4;     // 0,4,8,12
  for (int64_t k0 = 0; k0 < kdim; k0 += BK) {
    const int64_t ra = m0 + lr, rb = n0 + lr;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int64_t kk = k0 + lk + q;
      As[lk + q][lr] = (ra < ep.pk && kk < ldk) ? Y[ra * ldk + kk] : T(0);
      Bs[lk + q][lr] = (rb < ncols && kk < ldk) ? Xt[rb * ldk + kk] : T(0);
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = As[kk][ty * 4 + q];
        b[q] = Bs[kk][tx * 4 + q];
      }
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }

  // fused epilogue: candidate rule + emission (no p x p output)
  const T nT = (T)(1.0 / ep.inv_n);
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int64_t r = m0 + ty * 4 + x;
    if (r >= ep.pk) continue;
    const int64_t gi = ep.r0 + r;
    int cnt = 0;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int64_t k = ep.col_base + n0 + tx * 4 + y;
      if (k >= ep.col_end) continue;
      const T g = acc[x][y] / nT;
      const T w = lookup_omega<T>(om, r, (int32_t)k);
      const bool emit = (k == gi) || (w != T(0)) || (fabs((double)g) > ep.lam_cand);
      if (!emit) continue;
      const unsigned long long pos = atomicAdd(&pool.chunk_fill[0], 1ull);   // one chunk
      ++cnt;
      if ((int64_t)pos < pool.chunk) {
        pool.row[pos] = (int32_t)r;
        pool.col[pos] = (int32_t)k;
        ((T*)pool.g)[pos] = g;
        ((T*)pool.w)[pos] = w;
      }
    }
    if (cnt) atomicAdd(&pool.row_cnt[r], cnt);
  }
}

}  // namespace

int launch_gemm_simt(int dtype, const void* Y, const void* Xt, int64_t ldk, int64_t kdim,
                     const EpiParams& ep, const OmegaView& om, const PoolView& pool,
                     cudaStream_t st) {
  dim3 grd((unsigned)((ep.col_end - ep.col_base + BN - 1) / BN),
           (unsigned)((ep.pk + BM - 1) / BM));
  if (dtype == ACCORD_F64)
    gemm_simt_kernel<double><<<grd, 256, 0, st>>>((const double*)Y, (const double*)Xt, ldk,
                                                   kdim, ep, om, pool);
  else
    gemm_simt_kernel<float><<<grd, 256, 0, st>>>((const float*)Y, (const float*)Xt, ldk, kdim,
                                                  ep, om, pool);
  return 1;
}

}  // namespace accord

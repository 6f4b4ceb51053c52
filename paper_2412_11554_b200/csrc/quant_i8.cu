// int8 operands of the I8_FILTER gradient GEMM (gemm_tc.cu, kMode 2) and the
// constants of its certified bound.
//
//   Y rows (A operand): per-row scale a_i = max_m |y_im| / 127,
//     q_im = rint(y_im / a_i) in [-127, 127], y^_i = a_i q_i.
//   X^T rows (B operand): one scale per block of 256 variables (one GEMM
//     tile of columns), b_K = max over the block / 127, x^_k = b_K q_k. The
//     variables are first permuted so that a block holds variables of nearly
//     the same max |x| (host counting sort of log2 max |x_k| at 1/32 octave,
//     api.cpp): the block scale is then within ~2 % of each variable's own,
//     and the tile maxima of the bound's column constants are tight. Xq row k'
//     holds variable perm[k']; the GEMM epilogue maps its columns back.
//
// For every row the exact quantisation error vector e = v^ - v is formed in
// float64 (a float times a small integer minus a float: exact), and the bound
// constants are its norm and the row's norm, rounded up:
//   Y:   A_i = ||e_y,i||, B_i = ||y_i||
//   X^T: col_sd[k] = (||x_k|| + ||e_x,k||, ||e_x,k||)
// so that |<y^_i, x^_k> - <y_i, x_k>| <= A_i (C_k + D_k) + B_i D_k
// (Cauchy-Schwarz on e_y.x^ + y.e_x). Any rounding in the choice of q only
// changes e, which is measured, never assumed. A zero row / block gets scale 1
// (q = 0, e = 0).
#include "accord_internal.h"

namespace accord {

namespace {

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float row_absmax(const float* __restrict__ src, int64_t n, int lane) {
  float m = 0.f;
  const int64_t n4 = n >> 2;
  const float4* s4 = (const float4*)src;
  for (int64_t j = lane; j < n4; j += 32) {
    const float4 v = __ldg(&s4[j]);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  for (int64_t j = (n4 << 2) + lane; j < n; j += 32) m = fmaxf(m, fabsf(__ldg(&src[j])));
  return warp_max_f(m);
}

__device__ __forceinline__ int8_t q8(float v, float inv) {
  return (int8_t)max(-127, min(127, __float2int_rn(v * inv)));
}

// One warp quantises one row of n values (row stride ldk, ldk % 4 == 0) with
// scale `a` (inverse `inv`) into dst (columns [n, ldk) zeroed); returns the
// squared norms of the error and of the row (warp-reduced, float64).
__device__ __forceinline__ void quant_row(const float* __restrict__ src, int8_t* __restrict__ dst,
                                          int64_t n, int64_t ldk, float a, float inv, int lane,
                                          double& ee, double& vv) {
  ee = 0.0;
  vv = 0.0;
  const int64_t n4 = n >> 2;
  const float4* s4 = (const float4*)src;
  char4* d4 = (char4*)dst;
  for (int64_t j = lane; j < (ldk >> 2); j += 32) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < n4) {
      v = __ldg(&s4[j]);
    } else {
      const int64_t b = j << 2;   // ragged tail of the row, then padding
      if (b + 0 < n) v.x = __ldg(&src[b + 0]);
      if (b + 1 < n) v.y = __ldg(&src[b + 1]);
      if (b + 2 < n) v.z = __ldg(&src[b + 2]);
      if (b + 3 < n) v.w = __ldg(&src[b + 3]);
    }
    const int8_t qx = q8(v.x, inv), qy = q8(v.y, inv), qz = q8(v.z, inv), qw = q8(v.w, inv);
    d4[j] = make_char4(qx, qy, qz, qw);
    const double ex = (double)a * qx - v.x, ey = (double)a * qy - v.y,
                 ez = (double)a * qz - v.z, ew = (double)a * qw - v.w;
    ee += ex * ex + ey * ey + ez * ez + ew * ew;
    vv += (double)v.x * v.x + (double)v.y * v.y + (double)v.z * v.z + (double)v.w * v.w;
  }
  ee = warp_sum_d(ee);
  vv = warp_sum_d(vv);
}

__device__ __forceinline__ float norm_ru(double s2) {
  return __double2float_ru(sqrt(s2) * (1.0 + 1e-12));
}

// Y: warp per row, per-row scale
__global__ void quant_y_kernel(int64_t rows, int64_t n, int64_t ldk, const float* __restrict__ Y,
                               int8_t* __restrict__ Yq, float* __restrict__ scale,
                               float* __restrict__ rA, float* __restrict__ rB) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float* src = Y + r * ldk;
  const float mx = row_absmax(src, n, lane);
  const float a = mx > 0.f ? mx / 127.f : 1.f;
  const float inv = mx > 0.f ? 127.f / mx : 0.f;
  double ee, vv;
  quant_row(src, Yq + r * ldk, n, ldk, a, inv, lane, ee, vv);
  if (lane == 0) {
    scale[r] = a;
    rA[r] = norm_ru(ee);
    rB[r] = norm_ru(vv);
  }
}

// max |x| of every X^T row (warp per row): the key of the variable permutation
__global__ void row_absmax_kernel(int64_t rows, int64_t n, int64_t ldk,
                                  const float* __restrict__ Xt, float* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const float m = row_absmax(Xt + r * ldk, n, lane);
  if (lane == 0) out[r] = m;
}

// X^T, pass 1: block of 256 threads = 8 warps x 32 rows -> the max |x| over
// the 256 (permuted) rows of the block, as the block's scale
__global__ void xblk_scale_kernel(int64_t rows, int64_t n, int64_t ldk,
                                  const float* __restrict__ Xt, const int32_t* __restrict__ perm,
                                  float* __restrict__ blk_scale) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float m = 0.f;
  for (int i = w; i < 256; i += 8) {
    const int64_t r = (int64_t)blockIdx.x * 256 + i;
    if (r < rows) m = fmaxf(m, row_absmax(Xt + (int64_t)perm[r] * ldk, n, lane));
  }
  __shared__ float sm[8];
  if (lane == 0) sm[w] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < 8; ++j) m = fmaxf(m, sm[j]);
    blk_scale[blockIdx.x] = m > 0.f ? m / 127.f : 1.f;
  }
}

// X^T, pass 2: warp per (permuted) row with its block's scale; Xq row r holds
// variable perm[r]; col_sd is indexed by the variable
__global__ void quant_x_kernel(int64_t rows, int64_t n, int64_t ldk, const float* __restrict__ Xt,
                               const int32_t* __restrict__ perm, int8_t* __restrict__ Xq,
                               const float* __restrict__ blk_scale, float2* __restrict__ col_sd) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int64_t k = perm[r];
  const float a = blk_scale[r >> 8];
  // the max over the block is >= every |x| of the row, so |x / a| <= 127
  // (up to the rounding of the division: q8 clamps)
  const float inv = 1.f / a;
  double ee, vv;
  quant_row(Xt + k * ldk, Xq + r * ldk, n, ldk, a, inv, lane, ee, vv);
  if (lane == 0) {
    const float D = norm_ru(ee), C = norm_ru(vv);
    col_sd[k] = make_float2(__fadd_ru(C, D), D);
  }
}

}  // namespace

int launch_quant_y_i8(int64_t rows, int64_t n, int64_t ldk, const float* Y, int8_t* Yq,
                      float* scale, float* rA, float* rB, cudaStream_t st) {
  if (rows <= 0) return 0;
  quant_y_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(rows, n, ldk, Y, Yq, scale, rA, rB);
  return 1;
}

int launch_row_absmax(int64_t rows, int64_t n, int64_t ldk, const float* Xt, float* out,
                      cudaStream_t st) {
  if (rows <= 0) return 0;
  row_absmax_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(rows, n, ldk, Xt, out);
  return 1;
}

int launch_quant_x_i8(int64_t rows, int64_t n, int64_t ldk, const float* Xt, const int32_t* perm,
                      int8_t* Xq, float* blk_scale, float2* col_sd, cudaStream_t st) {
  if (rows <= 0) return 0;
  xblk_scale_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(rows, n, ldk, Xt, perm,
                                                                      blk_scale);
  quant_x_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(rows, n, ldk, Xt, perm, Xq,
                                                              blk_scale, col_sd);
  return 2;
}

}  // namespace accord

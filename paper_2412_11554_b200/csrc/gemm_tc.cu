// tcgen05 gradient GEMM with the fused candidate epilogue (SURVEY.md §8(a)
// rows a2 + a3), sm_100a.
//
//   G_k = Y_k X / n,  Y_k = Omega_{R_k} X^T  (two-step gradient)
//
// Precision: Y and X^T are each split once into bf16 pairs
// hi = bf16(v), lo = bf16(v - hi); the tensor cores accumulate
//   hi*hi + hi*lo + lo*hi      (3 x kind::f16 MMAs, fp32 accumulator in TMEM)
// which carries ~16 significant bits per operand product instead of 8; the
// dropped lo*lo term is <= 2^-16 relative. Measured against the float64
// oracle this is fp32-grade, which the 1e-5 parity budget needs (single-pass
// bf16 or tf32 is not).
//
// Structure: persistent kernel, one 128 x 256 output tile per step, 8 warps:
//   warp 0   TMA producer (lane 0): A_hi, A_lo (Y rows), B_hi, B_lo (X^T rows)
//            into a 2-stage SMEM ring (SWIZZLE_128B, 96 KB / stage)
//   warp 1   MMA issuer (lane 0): 4 k-steps x 3 MMAs (M128 N256 K16) per stage
//   warp 2   TMEM allocator (512 columns = 2 accumulator stages)
//   warps 4-7 epilogue: TMEM -> registers (32x32b.x32), candidate rule, warp
//            ballot/prefix compaction into the candidate pool. The p x p
//            gradient never reaches HBM. The epilogue of tile t overlaps the
//            mainloop of tile t+1 (double-buffered accumulator).
//
// Epilogue rule (derived from Eq. 3.5): emit
// (i, k, g = acc / n, omega_ik) iff k == i, or (i,k) in supp Omega (found by a
// merge walk of the thread's sorted CSR row), or |acc| > lam_cand * n.
#include "accord_internal.h"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <climits>
#include <cstring>

namespace accord {

namespace {

constexpr int BM = 128, BN = 256, BK = 64;     // BK in bf16 elements = 128 B rows
constexpr int kAccStages = 2;
constexpr int kTmemCols = 512;
constexpr uint32_t kTileA = BM * BK * 2;       // 16 KB
constexpr uint32_t kTileB = BN * BK * 2;       // 32 KB
constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;
constexpr int kGroupM = 16;                    // M-blocks per raster group (L2 reuse)

// kMode 0 = BF16X3 (hi/lo operands, 3 MMAs per k-step, values from TMEM)
// kMode 1 = BF16_FILTER (hi operands only, 1 MMA per k-step, certified filter)
template <int kMode> struct Cfg {
  static constexpr int kOps = kMode == 0 ? 2 : 1;                        // hi (+lo)
  static constexpr uint32_t kStageBytes = kOps * (kTileA + kTileB);      // 96 / 48 KB
  static constexpr int kStages = kMode == 0 ? 2 : 4;
  static constexpr size_t kSmemBytes = 1024 + (size_t)kStages * kStageBytes + 256;
};

struct TileCoord { int m, n; };

__device__ __forceinline__ TileCoord tile_coord(int t, int num_m, int num_n) {
  const int per_group = kGroupM * num_n;
  const int g = t / per_group;
  const int first = g * kGroupM;
  const int gm = min(kGroupM, num_m - first);
  const int l = t - g * per_group;
  return TileCoord{first + l % gm, l / gm};
}

template <int kMode>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap mA_hi,
                   const __grid_constant__ CUtensorMap mA_lo,
                   const __grid_constant__ CUtensorMap mB_hi,
                   const __grid_constant__ CUtensorMap mB_lo, int num_kb, int num_m, int num_n,
                   EpiParams ep, OmegaView om, PoolView pool) {
  constexpr int kStages = Cfg<kMode>::kStages;
  constexpr uint32_t kStageBytes = Cfg<kMode>::kStageBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment for SWIZZLE_128B atoms
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + kStages * kStageBytes);
  uint64_t* full = bars;                         // [kStages]
  uint64_t* empty = bars + kStages;              // [kStages]
  uint64_t* tfull = bars + 2 * kStages;          // [kAccStages]
  uint64_t* tempty = bars + 2 * kStages + kAccStages;
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * kStages + 2 * kAccStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_tiles = num_m * num_n;

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&mA_hi);
    tc::tma_prefetch(&mA_lo);
    tc::tma_prefetch(&mB_hi);
    tc::tma_prefetch(&mB_lo);
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(tc::smem_u32(&full[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < kAccStages; ++a) {
      tc::mbar_init(tc::smem_u32(&tfull[a]), 1);
      tc::mbar_init(tc::smem_u32(&tempty[a]), 4);   // one arrive per epilogue warp
    }
    tc::fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc<kTmemCols, 1>(tc::smem_u32(tmem_slot));
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ============================ TMA producer ============================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const TileCoord tc_ = tile_coord(t, num_m, num_n);
        for (int kb = 0; kb < num_kb; ++kb) {
          tc::mbar_wait(tc::smem_u32(&empty[stage]), phase ^ 1);
          uint8_t* s = smem + stage * kStageBytes;
          const uint32_t fb = tc::smem_u32(&full[stage]);
          tc::mbar_arrive_expect_tx(fb, kStageBytes);
          const int kx = kb * BK;
          // stage layout: A_hi | B_hi | (A_lo | B_lo)
          tc::tma_load_2d(tc::smem_u32(s), &mA_hi, fb, kx, tc_.m * BM);
          tc::tma_load_2d(tc::smem_u32(s + kTileA), &mB_hi, fb, kx, tc_.n * BN);
          if constexpr (kMode == 0) {
            tc::tma_load_2d(tc::smem_u32(s + kTileA + kTileB), &mA_lo, fb, kx, tc_.m * BM);
            tc::tma_load_2d(tc::smem_u32(s + 2 * kTileA + kTileB), &mB_lo, fb, kx, tc_.n * BN);
          }
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer ==============================
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_bf16_f32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        tc::mbar_wait(tc::smem_u32(&tempty[acc]), acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < num_kb; ++kb) {
          tc::mbar_wait(tc::smem_u32(&full[stage]), phase);
          tc::tc_fence_after();
          const uint32_t s = tc::smem_u32(smem + stage * kStageBytes);
          const uint64_t a_hi = tc::sdesc_k_sw128(s);
          const uint64_t b_hi = tc::sdesc_k_sw128(s + kTileA);
          const uint64_t a_lo = tc::sdesc_k_sw128(s + kTileA + kTileB);
          const uint64_t b_lo = tc::sdesc_k_sw128(s + 2 * kTileA + kTileB);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t off = (uint64_t)(kk * 32) >> 4;   // 16 bf16 = 32 B along K
            const uint32_t accum = (kb | kk) != 0;
            tc::mma_bf16<1>(d, a_hi + off, b_hi + off, idesc, accum);
            if constexpr (kMode == 0) {
              tc::mma_bf16<1>(d, a_hi + off, b_lo + off, idesc, 1);
              tc::mma_bf16<1>(d, a_lo + off, b_hi + off, idesc, 1);
            }
          }
          tc::mma_commit(tc::smem_u32(&empty[stage]));
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        tc::mma_commit(tc::smem_u32(&tfull[acc]));
        if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= kEpiWarp0) {
    // ============================ epilogue ================================
    const int q = warp - kEpiWarp0;                 // TMEM lane quarter (= warp % 4)
    const float thr = (float)(ep.lam_cand / ep.inv_n);   // |acc| > lam * n
    const float gam = ep.gamma;
    const float nf = (float)(1.0 / ep.inv_n);
    const float* omv = (const float*)om.val;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      const TileCoord tc_ = tile_coord(t, num_m, num_n);
      const int64_t r = (int64_t)tc_.m * BM + q * 32 + lane;     // local row
      const bool row_ok = r < ep.pk;
      const int64_t gi = ep.r0 + r;
      const int n0 = tc_.n * BN;
      // support walk setup (before waiting: overlaps the mainloop)
      int64_t sp = 0, se = 0;
      int32_t nxt = INT_MAX;
      if (row_ok) {
        int64_t lo = om.ptr[r], hi = om.ptr[r + 1];
        se = hi;
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (om.col[mid] < n0) lo = mid + 1; else hi = mid;
        }
        sp = lo;
        nxt = sp < se ? om.col[sp] : INT_MAX;
      }
      // BF16_FILTER: n*delta_ik = r1 * s_k + Bn * D_k, a rigorous bound on
      // |acc - n*G_ik| (bf16 rounding of both operands by Cauchy-Schwarz on
      // the actual rounding-error vectors, plus fp32 accumulation), inflated
      // by 1.0625 for the float evaluation of the bound itself.
      float r1 = 0.f, Bn = 0.f;
      if (kMode == 1 && row_ok) {
        const float A = ep.row_A[r], B = ep.row_B[r];
        r1 = (A + gam * (A + B)) * 1.0625f;
        Bn = B * 1.0625f;
      }
      tc::mbar_wait(tc::smem_u32(&tfull[acc]), acc_phase);
      tc::tc_fence_after();
      int row_count = 0;
      const uint32_t tbase = tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN);
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        uint32_t v[32];
        tc::tmem_ld32(tbase + ch * 32, v);
        tc::tmem_ld_wait();
        const int c0 = n0 + ch * 32;
        const int64_t sp0 = sp;
        uint32_t mask = 0;
        if (row_ok) {
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int col = c0 + c;
            const bool hit = col == nxt;
            if (hit) {
              ++sp;
              nxt = sp < se ? om.col[sp] : INT_MAX;
            }
            float t = thr;
            if constexpr (kMode == 1) {
              const float2 sd = __ldg(&ep.col_sd[col < ep.p ? col : 0]);
              t = thr - fmaf(r1, sd.x, Bn * sd.y);
            }
            const bool cand = hit || (col == gi) || (fabsf(__uint_as_float(v[c])) > t);
            mask |= (cand && col < ep.p) ? (1u << c) : 0u;
          }
        }
        const int cnt = __popc(mask);
        const int total = __reduce_add_sync(0xffffffffu, cnt);
        if (total == 0) continue;
        int incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        unsigned long long base = 0;
        if (lane == 31) base = atomicAdd(pool.cursor, (unsigned long long)incl);
        base = __shfl_sync(0xffffffffu, base, 31);
        unsigned long long pos = base + (unsigned long long)(incl - cnt);
        row_count += cnt;
        if (cnt) {
          int64_t s2 = sp0;
          int32_t n2 = s2 < se ? om.col[s2] : INT_MAX;
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int col = c0 + c;
            float w = 0.f;
            if (col == n2) {
              w = omv[s2];
              ++s2;
              n2 = s2 < se ? om.col[s2] : INT_MAX;
            }
            if (mask & (1u << c)) {
              if ((int64_t)pos < pool.cap) {
                pool.row[pos] = (int32_t)r;
                pool.col[pos] = col;
                ((float*)pool.g)[pos] = __uint_as_float(v[c]) / nf;
                ((float*)pool.w)[pos] = w;
              }
              ++pos;
            }
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&tempty[acc]));
      if (row_count) atomicAdd(&pool.row_cnt[r], row_count);
      if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc<kTmemCols, 1>(tmem_base);
}

// ---- host: tensor maps ----------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
  }
  return fn;
}

bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t ldk, int box_rows,
              std::string* err) {
  auto fn = encode_fn();
  if (!fn) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)ldk, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ldk * 2)};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")";
    return false;
  }
  return true;
}

}  // namespace

struct TcGemmPlan {
  CUtensorMap a_hi[2], a_lo[2], b_hi, b_lo;
  int64_t pk_pad = 0, p_pad = 0, ldk = 0;
};

bool tc_supported(int cc_major, int cc_minor) { return cc_major == 10 && cc_minor == 0; }

TcGemmPlan* tc_plan_create(const __nv_bfloat16* Yhi0, const __nv_bfloat16* Ylo0,
                           const __nv_bfloat16* Yhi1, const __nv_bfloat16* Ylo1, int64_t pk_pad,
                           const __nv_bfloat16* Xhi, const __nv_bfloat16* Xlo, int64_t p_pad,
                           int64_t ldk, std::string* err) {
  auto* p = new TcGemmPlan();
  p->pk_pad = pk_pad;
  p->p_pad = p_pad;
  p->ldk = ldk;
  bool ok = make_map(&p->a_hi[0], Yhi0, pk_pad, ldk, BM, err) &&
            make_map(&p->a_lo[0], Ylo0, pk_pad, ldk, BM, err) &&
            make_map(&p->a_hi[1], Yhi1, pk_pad, ldk, BM, err) &&
            make_map(&p->a_lo[1], Ylo1, pk_pad, ldk, BM, err) &&
            make_map(&p->b_hi, Xhi, p_pad, ldk, BN, err) &&
            make_map(&p->b_lo, Xlo, p_pad, ldk, BN, err);
  if (!ok) {
    delete p;
    return nullptr;
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg<0>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg<1>::kSmemBytes);
    attr = true;
  }
  return p;
}

void tc_plan_destroy(TcGemmPlan* p) { delete p; }

int launch_gemm_tc(TcGemmPlan* plan, int mode, int ybuf, int64_t kdim, int sm_count,
                   const EpiParams& ep, const OmegaView& om, const PoolView& pool,
                   cudaStream_t st) {
  const int num_m = (int)(plan->pk_pad / BM);
  const int num_n = (int)(plan->p_pad / BN);
  const int num_kb = (int)((kdim + BK - 1) / BK);
  const int tiles = num_m * num_n;
  const int grid = tiles < sm_count ? tiles : sm_count;
  if (mode == ACCORD_GEMM_BF16X3)
    gemm_tc_kernel<0><<<grid, kThreads, Cfg<0>::kSmemBytes, st>>>(
        plan->a_hi[ybuf], plan->a_lo[ybuf], plan->b_hi, plan->b_lo, num_kb, num_m, num_n, ep,
        om, pool);
  else
    gemm_tc_kernel<1><<<grid, kThreads, Cfg<1>::kSmemBytes, st>>>(
        plan->a_hi[ybuf], plan->a_hi[ybuf], plan->b_hi, plan->b_hi, num_kb, num_m, num_n, ep,
        om, pool);
  return 1;
}

}  // namespace accord

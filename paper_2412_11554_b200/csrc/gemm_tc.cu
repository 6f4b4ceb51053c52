// tcgen05 gradient GEMM with the fused candidate epilogue (SURVEY.md §8(a)
// rows a2 + a3), sm_100a, CTA pairs (cta_group::2).
//
//   G_k = Y_k X / n,  Y_k = Omega_{R_k} X^T   (two-step gradient)
//
// Both operands are K-major (Y rows and X^T rows, K = n samples), so the
// product is a plain "TN" GEMM: D[i,k] = sum_m Y[i,m] Xt[k,m].
//
// Two arithmetic modes:
//   kMode 1, BF16_FILTER (default): one bf16 MMA pass; the epilogue emits
//     (i,k) when |acc| > n*lambda - n*delta_ik, with n*delta_ik a rigorous
//     bound on |acc - n*G_ik| (bf16 rounding of both operands by
//     Cauchy-Schwarz on the actual rounding-error vectors, plus the fp32
//     accumulation). The candidate values are then recomputed exactly by the
//     refine SDDMM (kernels.cu), so no candidate can be missed and every value
//     is float64-accumulated.
//   kMode 0, BF16X3: operands split hi = bf16(v), lo = bf16(v - hi); three
//     MMA passes hi*hi + hi*lo + lo*hi into the same fp32 accumulator; values
//     come from TMEM (relative product error ~2^-16).
//   kMode 2, I8_FILTER: the same certified filter with int8 operands
//     (kind::i8, twice the bf16 MMA rate, half the operand bytes): Y rows
//     quantised with a per-row scale a_i, X^T rows with a per-256-row block
//     scale b_K, so y^ = a_i q_i and x^ = b_K q_k. The s32 accumulator is
//     EXACT (|acc| <= n 127^2 < 2^31 for n < 133,000), so a_i b_K acc =
//     <y^_i, x^_k> exactly and the bound needs no accumulation model:
//     |<y^,x^> - <y,x>| = |e_y.x^ + y.e_x| <= A_i (C_k + D_k) + B_i D_k with
//     A = ||e_y||, B = ||y||, C = ||x||, D = ||e_x|| (the actual quantisation
//     errors, quant_i8.cu). The epilogue turns n lambda - n delta into an
//     integer threshold per row and tile (double arithmetic, rounded down)
//     and tests |acc| against it with integer min/max.
//
// Structure (persistent, one 256 x 256 tile per CTA pair per step):
//   cluster of 2 CTAs; CTA r holds rows [128r, 128r+128) of the A tile (Y)
//   and rows [128r, 128r+128) of the B tile (X^T); the leader (r = 0) issues
//   tcgen05.mma.cta_group::2 (M256 N256 K16), whose accumulator lands half in
//   each CTA's TMEM (lane = row).
//   warp 0  TMA producer (both CTAs; the bytes are credited to the leader's
//           full barrier), SWIZZLE_128B, kStages-deep ring
//   warp 1  MMA issuer (leader only), commits multicast to both CTAs
//           (warps 0 and 1 run their loops warp-wide so that descriptors and
//           coordinates stay in uniform registers; an elect.sync lane issues:
//           single-lane loops made ptxas wrap every UTCHMMA in an ELECT/R2UR
//           waterfall, which left the tensor pipe ~70% busy)
//   warp 2  TMEM allocator (512 columns = 2 accumulator stages)
//   warps 4-7 epilogue (both CTAs): TMEM -> registers (32x32b), candidate
//           rule, warp prefix-sum compaction into the candidate pool, one
//           atomicAdd per warp-chunk. The p x p gradient never reaches HBM;
//           the epilogue of tile t overlaps the mainloop of tile t+1.
//
// Epilogue rule (derived from Eq. 3.5): C =
// diag U supp Omega U {|G| > lambda}. BF16X3 emits (i, k, g, omega_ik) for all
// three (merge walk of the thread's sorted CSR row); the filter emits only the
// positions passing its |acc| test -- the diagonal and supp Omega are merged
// in by the finalize (kernels.cu, support append + dedupe), which keeps the
// support walk off the tensor-core epilogue (after iteration 1, ~240 support
// entries per row at config 5).
#include "accord_internal.h"
#include "tc_ptx.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <cstring>

namespace accord {

namespace {

constexpr int BM = 128;                         // rows of A per CTA (256 per pair)
constexpr int BN = 256;                         // columns of the tile (N of one MMA)
constexpr int BNH = BN / 2;                     // rows of B held per CTA
constexpr int BK = 64;                          // bf16 elements = 128-B rows (128 int8)
constexpr int kAccStages = 2;
constexpr int kTmemCols = 512;
constexpr uint32_t kTileA = BM * BK * 2;        // 16 KB
constexpr uint32_t kTileB = BNH * BK * 2;       // 16 KB
constexpr int kThreads = 256;
constexpr int kEpiWarp0 = 4;

template <int kMode, int kStagesT, int kEpiWT = 0> struct Cfg {
  static constexpr int kOps = kMode == 0 ? 2 : 1;                        // hi (+lo)
  static constexpr int kBKe = kMode == 2 ? 2 * BK : BK;                  // elements per 128-B row
  // epilogue warps: int8 halves the MMA time per tile, so two warps share a
  // TMEM lane quarter (each half of the 256 columns); with four the int8
  // GEMM ran 19 % faster with its epilogue switched off (ACCORD_DEBUG_GEMM=1)
  static constexpr int kEpiW = kEpiWT ? kEpiWT : (kMode == 2 ? 8 : 4);
  static constexpr int kThreads = 128 + 32 * kEpiW;
  static constexpr uint32_t kStageBytes = kOps * (kTileA + kTileB);      // 64 / 32 KB
  static constexpr int kStages = kStagesT;
  static constexpr size_t kSmemBytes = 1024 + (size_t)kStages * kStageBytes + 256;
  static_assert(kSmemBytes <= 232448, "shared memory");
};

// Tile order. Work unit = up to `U` consecutive N-blocks at a fixed M-block,
// inside a group of `GN` N-blocks; units are enumerated group-major, then by
// M-block, and dealt round-robin to the clusters. All clusters therefore work
// on one X^T group at a time (GN x 256 rows, <= 32 MB, stay L2-resident, so
// X^T crosses HBM once per launch and Y once per group), each cluster reuses
// its Y block across its unit, and inside a unit a thread's row stays the
// same, so the epilogue's walk through the sorted CSR row of Omega continues
// from tile to tile (one binary search per unit instead of per tile). This
// keeps the schedule's L2 footprint bounded however far the persistent
// clusters drift apart.
struct Sched {
  int num_m, num_n, GN, U;
  int full_groups, rem, spu, spu_last;
  long long units_full, units;
  // symmetric G (EpiParams::sym): 1 = upper triangle only (one rank), 2 = the
  // cyclic half across ranks: tile (I, J) of global row tile I = mt0 + m runs
  // iff d = (J - I) mod nt is 0 or <= (nt-1)/2 (d = nt/2: iff I < J), so each
  // unordered pair of tiles runs once and every row tile runs ~half its tiles
  int sym, mt0, nt;
  __device__ Sched(int nm, int nn, int gn, int u, int sy, int m0, int ntg)
      : num_m(nm), num_n(nn), GN(gn), U(u), sym(sy), mt0(m0), nt(ntg) {
    full_groups = num_n / GN;
    rem = num_n - full_groups * GN;
    spu = (GN + U - 1) / U;
    spu_last = (rem + U - 1) / U;
    units_full = (long long)full_groups * num_m * spu;
    units = units_full + (long long)num_m * spu_last;
  }
  __device__ bool valid(int m, int n) const {
    if (sym != 2) return sym == 0 || n >= m;
    const int I = mt0 + m;
    if (n == I) return true;
    const int d = ((n - I) % nt + nt) % nt;
    if (d <= (nt - 1) / 2) return true;
    return (nt % 2 == 0) && d == nt / 2 && I < n;
  }
  // unit -> (M-block, first N-block, count)
  __device__ void unit(long long u, int& m, int& n0, int& cnt) const {
    if (u < units_full) {
      const long long per_g = (long long)num_m * spu;
      const int g = (int)(u / per_g);
      const int r = (int)(u - (long long)g * per_g);
      m = r / spu;
      const int s = r - m * spu;
      n0 = g * GN + s * U;
      cnt = min(U, GN - s * U);
    } else {
      const int r = (int)(u - units_full);
      m = r / spu_last;
      const int s = r - m * spu_last;
      n0 = full_groups * GN + s * U;
      cnt = min(U, rem - s * U);
    }
  }
};

// Iterate this cluster's tiles in schedule order: for (TileIt it(...); it.ok; it.next())
// (sym: the tiles below the diagonal are skipped identically by every role)
struct TileIt {
  const Sched& S;
  long long u;
  int stride, m, n0, cnt, ni;
  bool ok, start;
  __device__ TileIt(const Sched& s, int cluster, int nclusters)
      : S(s), u(cluster), stride(nclusters), ni(0) { load(); }
  __device__ void load() {
    for (;;) {
      ok = u < S.units;
      ni = 0;
      start = true;
      if (!ok) return;
      S.unit(u, m, n0, cnt);
      if (!S.sym) return;
      if (S.sym == 1) {
        if (n0 + cnt - 1 < m) { u += stride; continue; }   // whole unit below the diagonal
        if (n0 < m) ni = m - n0;
        return;
      }
      while (ni < cnt && !S.valid(m, n0 + ni)) ++ni;
      if (ni == cnt) { u += stride; continue; }
      return;
    }
  }
  __device__ void next() {
    start = false;
    ++ni;
    if (S.sym == 2)
      while (ni < cnt && !S.valid(m, n0 + ni)) {   // a gap: the row walk restarts after it
        ++ni;
        start = true;
      }
    if (ni == cnt) { u += stride; load(); }
  }
  __device__ int n() const { return n0 + ni; }
  __device__ bool unit_start() const { return start; }
};

// kDiag: 0 = the product epilogue; 3 = the same for the symmetric first GEMM
// across ranks (EpiParams::sym = 2: the only instantiation with the mirror
// buffer path -- that branch, never taken elsewhere, cost ~2 % of the c5
// GEMM through the power-capped clock when compiled into the product kernel);
// 1 = audit (also writes every raw fp32
// accumulator to ep.audit_acc, for the filter certification test); 2 = max
// reduction (no emission: a certified lower bound on n max_{i!=k} |G_ik|
// into *ep.max_out, the lambda_max of a path)
template <int kMode, int kStagesT, bool kFast, int kDiag = 0, int kEpiWT = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(Cfg<kMode, kStagesT, kEpiWT>::kThreads, 1)
gemm_tc_kernel(const __grid_constant__ CUtensorMap mA_hi,
               const __grid_constant__ CUtensorMap mA_lo,
               const __grid_constant__ CUtensorMap mB_hi,
               const __grid_constant__ CUtensorMap mB_lo, int num_kb, int kk_last, int num_m,
               int num_n,
               int group_n, int unit_n, int dbg, int l2hint, EpiParams ep,
               const float2* __restrict__ blk_sdmax, OmegaView om,
               PoolView pool) {
  constexpr int kStages = Cfg<kMode, kStagesT, kEpiWT>::kStages;
  constexpr uint32_t kStageBytes = Cfg<kMode, kStagesT, kEpiWT>::kStageBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = (uint64_t*)(smem + kStages * kStageBytes);
  uint64_t* full = bars;                          // [kStages]   (leader's is used)
  uint64_t* empty = bars + kStages;               // [kStages]   (each CTA's own)
  uint64_t* tfull = bars + 2 * kStages;           // [kAccStages] (each CTA's own)
  uint64_t* tempty = bars + 2 * kStages + kAccStages;   // (leader's is used)
  uint32_t* tmem_slot = (uint32_t*)(bars + 2 * kStages + 2 * kAccStages);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const Sched sched(num_m, num_n, group_n, unit_n, kMode != 0 ? ep.sym : 0, ep.mt0, ep.nt);

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&mA_hi);
    tc::tma_prefetch(&mB_hi);
    if (kMode == 0) {
      tc::tma_prefetch(&mA_lo);
      tc::tma_prefetch(&mB_lo);
    }
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(tc::smem_u32(&full[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < kAccStages; ++a) {
      tc::mbar_init(tc::smem_u32(&tfull[a]), 1);
      tc::mbar_init(tc::smem_u32(&tempty[a]), 2 * Cfg<kMode, kStagesT, kEpiWT>::kEpiW);   // x 2 CTAs
    }
    tc::fence_mbar_init();
  }
  if (warp == 2) tc::tmem_alloc<kTmemCols, 2>(tc::smem_u32(tmem_slot));
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ============================ TMA producer (both CTAs) ================
    // warp-wide loop (uniform operands), one elected lane issues
    {
      const uint64_t bpol = l2hint == 2 ? tc::policy_evict_first() : tc::policy_evict_last();
      int stage = 0;
      uint32_t phase = 0;
      for (TileIt it(sched, cluster, nclusters); it.ok; it.next()) {
        const int ya = it.m * (2 * BM) + (int)rank * BM;
        const int yb = it.n() * BN + (int)rank * BNH;
        for (int kb = 0; kb < num_kb; ++kb) {
          tc::mbar_wait(tc::smem_u32(&empty[stage]), phase ^ 1);
          uint8_t* s = smem + stage * kStageBytes;
          const uint32_t fb_local = tc::smem_u32(&full[stage]);
          const uint32_t fb = tc::mapa_shared(fb_local, 0);                  // leader's barrier
          const int kx = kb * Cfg<kMode, kStagesT, kEpiWT>::kBKe;
          if (tc::elect_one()) {
            if (leader) tc::mbar_arrive_expect_tx(fb_local, 2 * kStageBytes);   // both CTAs' bytes
            // stage layout: A_hi | B_hi | (A_lo | B_lo)
            if (l2hint) {   // X^T group: keep in L2 (every pair re-reads it); Y: normal
              tc::tma_load_2d_cg2(tc::smem_u32(s), &mA_hi, fb, kx, ya);
              tc::tma_load_2d_cg2_hint(tc::smem_u32(s + kTileA), &mB_hi, fb, kx, yb, bpol);
            } else {
              tc::tma_load_2d_cg2(tc::smem_u32(s), &mA_hi, fb, kx, ya);
              tc::tma_load_2d_cg2(tc::smem_u32(s + kTileA), &mB_hi, fb, kx, yb);
            }
            if constexpr (kMode == 0) {
              tc::tma_load_2d_cg2(tc::smem_u32(s + kTileA + kTileB), &mA_lo, fb, kx, ya);
              tc::tma_load_2d_cg2(tc::smem_u32(s + 2 * kTileA + kTileB), &mB_lo, fb, kx, yb);
            }
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ============================ MMA issuer (leader) =====================
    // The whole warp runs the loop (so the descriptors stay warp-uniform and
    // live in uniform registers); one elected lane issues the MMAs/commits.
    if (leader) {
      constexpr uint32_t idesc =
          kMode == 2 ? tc::idesc_s8_s32(2 * BM, BN) : tc::idesc_bf16_f32(2 * BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (TileIt it(sched, cluster, nclusters); it.ok; it.next()) {
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
          // the last k-block issues only the K16 steps that reach a sample
          // (the rest of its box is TMA zero fill past n)
          const int nkk = kb == num_kb - 1 ? kk_last : BK / 16;
          if (tc::elect_one()) {
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              if (kk >= nkk) break;
              const uint64_t off = (uint64_t)(kk * 32) >> 4;   // 16 bf16 / 32 int8 = 32 B along K
              const uint32_t accum = (kb | kk) != 0;
              if constexpr (kMode == 2) {
                if (dbg != 2) tc::mma_i8<2>(d, a_hi + off, b_hi + off, idesc, accum);
              } else {
                if (dbg != 2) tc::mma_bf16<2>(d, a_hi + off, b_hi + off, idesc, accum);
              }
              if constexpr (kMode == 0) {
                tc::mma_bf16<2>(d, a_hi + off, b_lo + off, idesc, 1);
                tc::mma_bf16<2>(d, a_lo + off, b_hi + off, idesc, 1);
              }
            }
            tc::mma_commit_mc(tc::smem_u32(&empty[stage]), 0x3);   // free the slot in both CTAs
          }
          __syncwarp();
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        if (tc::elect_one()) tc::mma_commit_mc(tc::smem_u32(&tfull[acc]), 0x3);   // acc ready
        __syncwarp();
        if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= kEpiWarp0) {
    // ============================ epilogue (both CTAs) ====================
    constexpr int kEpiW = Cfg<kMode, kStagesT, kEpiWT>::kEpiW;
    constexpr int kCols = BN / (kEpiW / 4);          // columns of the tile this warp tests
    const int q = (warp - kEpiWarp0) & 3;            // TMEM lane quarter (= warp % 4)
    const int cb = ((warp - kEpiWarp0) >> 2) * kCols;   // first column of this warp's part
    const float thr = (float)(ep.lam_cand / ep.inv_n);   // n * lambda
    const double thr_d = ep.lam_cand / ep.inv_n;
    const float inv_nf = (float)ep.inv_n;
    const float gam = ep.gamma;
    const float* omv = (const float*)om.val;
    const uint32_t tempty_leader = tc::smem_u32(&tempty[0]);
    const int64_t col_end = ep.col_end;
    // this warp's private pool chunk (warp-uniform); taken on first use
    long long chunk_id = -1;
    int64_t fill = pool.chunk;
    int acc = 0;
    uint32_t acc_phase = 0;
    int64_t r = 0, gi = 0, sp = 0, se = 0;
    bool row_ok = false;
    int32_t nxt = INT_MAX;
    float r1 = 0.f, Bn = 0.f;
    double asc = 0.0;                               // kMode 2: a_i (row scale)
    float wmax = 0.f;                               // kDiag == 2
    for (TileIt it(sched, cluster, nclusters); it.ok; it.next()) {
      const int n0 = (int)ep.col_base + it.n() * BN;   // global column of the tile
      if (it.unit_start()) {
        // new row block: row constants and the start of the CSR walk (the
        // walk then continues across the unit's consecutive column tiles)
        r = (int64_t)it.m * (2 * BM) + (int64_t)rank * BM + q * 32 + lane;
        row_ok = r < ep.pk;
        gi = ep.r0 + r;
        nxt = INT_MAX;
        if (row_ok) {
          if constexpr (kMode == 0) {
            // BF16X3 emits values: walk Omega's sorted row for omega_ik (the
            // filter emits positions only; diagonal and support join C in the
            // finalize, so its epilogue tests |acc| alone)
            int64_t lo = om.ptr[r], hi = om.ptr[r + 1];
            se = hi;
            while (lo < hi) {
              const int64_t mid = (lo + hi) >> 1;
              if (om.col[mid] < n0) lo = mid + 1; else hi = mid;
            }
            sp = lo;
            nxt = sp < se ? om.col[sp] : INT_MAX;
          }
          if constexpr (kMode == 1) {
            // n*delta_ik = r1 * s_k + Bn * D_k, inflated by 1.0625 for the
            // float evaluation of the bound
            const float A = ep.row_A[r], B = ep.row_B[r];
            r1 = (A + gam * (A + B)) * 1.0625f;
            Bn = B * 1.0625f;
          }
          if constexpr (kMode == 2) {
            // exact accumulation: n*delta_ik = A_i s_k + B_i D_k (the norms
            // are rounded up; the tile threshold is evaluated in double)
            r1 = ep.row_A[r];
            Bn = ep.row_B[r];
            asc = (double)ep.row_scale[r];
          }
        }
      }
      float tfast = thr;
      int tint = -1;                             // kMode 2: emit iff |acc| > tint
      double sc = 0.0, ndel = 0.0;               // kMode 2: a_i b_K, tile bound n*delta
      if (kMode == 1 && row_ok) {
        const float2 mx = blk_sdmax[n0 / BN];    // tile max of the column constants
        tfast = thr - fmaf(r1, mx.x, Bn * mx.y);
      }
      if (kMode == 2 && row_ok) {
        // |acc| a_i b_K > n lambda - n delta  <=>  |acc| > t; the integer acc
        // passes iff |acc| > floor(t') for any t' <= t: t is taken 1e-12
        // relative and 1 unit low (double evaluation of t itself)
        const float2 mx = blk_sdmax[n0 / BN];
        ndel = fma((double)r1, (double)mx.x, (double)Bn * (double)mx.y) * (1.0 + 1e-9);
        sc = asc * (double)ep.blk_scale[n0 / BN];
        const double t = (thr_d - ndel) / sc;
        if (!(t > 0.0)) tint = -1;
        else if (t >= 2.0e9) tint = INT_MAX;
        else tint = (int)floor(t * (1.0 - 1e-12)) - 1;
        if (tint < -1) tint = -1;
      }
      tc::mbar_wait(tc::smem_u32(&tfull[acc]), acc_phase);
      tc::tc_fence_after();
      int row_count = 0;
      if (dbg == 1) {   // diagnostic: release the accumulator without reading it
        tc::tc_fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_remote(tempty_leader + acc * 8, 0);
        if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      const uint32_t tbase =
          tmem_base + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN) + (uint32_t)cb;
      // TMEM -> registers 32 columns at a time, one load ahead: the next
      // 32 columns are in flight while these are tested
      uint32_t va[32], vb[32];
      tc::tmem_ld32(tbase, va);
#pragma unroll 1
      for (int ch2 = 0; ch2 < kCols / 64; ++ch2) {
        tc::tmem_ld_wait();                                   // va = columns 64 ch2 + [0, 32)
        tc::tmem_ld32(tbase + ch2 * 64 + 32, vb);             // in flight: 64 ch2 + [32, 64)
        if (dbg >= 3) {   // diagnostics: 3 = TMEM reads only, 4 = reads + max test only
          tc::tmem_ld_wait();
          if (dbg == 4) {   // the max test of both halves (kept alive by an opaque compare)
            float m0 = 0.f, m1 = 0.f;
#pragma unroll
            for (int c = 0; c < 32; c += 2) {
              m0 = fmaxf(m0, fmaxf(fabsf(__uint_as_float(va[c])), fabsf(__uint_as_float(va[c + 1]))));
              m1 = fmaxf(m1, fmaxf(fabsf(__uint_as_float(vb[c])), fabsf(__uint_as_float(vb[c + 1]))));
            }
            if (__float_as_uint(fmaxf(m0, m1)) == 0x7f7ffff1u) pool.row[0] = 0;
          } else if (va[0] == 0xffffffffu && vb[31] == 0xffffffffu) {
            pool.row[0] = 0;                  // keep the loads alive (never true)
          }
          if (ch2 + 1 < kCols / 64) tc::tmem_ld32(tbase + (ch2 + 1) * 64, va);
          continue;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (h == 1) {
            tc::tmem_ld_wait();                               // vb ready
            if (ch2 + 1 < kCols / 64)                         // in flight: next 64 ch2 + [0, 32)
              tc::tmem_ld32(tbase + (ch2 + 1) * 64, va);
          }
          const uint32_t* v = h ? vb : va;
          const int c0 = n0 + cb + ch2 * 64 + h * 32;
          const int64_t sp0 = sp;
          if constexpr (kDiag == 1) {   // audit: the raw accumulator of every computed entry
            if (row_ok) {
              const bool mir = sched.sym && it.n() != sched.mt0 + it.m;
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                const int64_t k = c0 + c;
                if (k < col_end) {
                  // kMode 2: the accumulator in the units of n G (a_i b_K acc),
                  // at the variable's own column
                  const float a = kMode == 2 ? (float)((double)(int)v[c] * sc)
                                             : __uint_as_float(v[c]);
                  const int64_t kv = (kMode == 2 && ep.col_perm) ? (int64_t)ep.col_perm[k] : k;
                  ep.audit_acc[r * ep.audit_ld + kv] = a;
                  if (mir && k >= ep.r0 && k < ep.r0 + ep.pk)
                    ep.audit_acc[(k - ep.r0) * ep.audit_ld + gi] = a;
                }
              }
            }
          }
          if constexpr (kDiag == 2) {
            // max |acc| off the diagonal minus this row's tile bound n*delta
            // (= thr - tfast): a lower bound on n |G_ik| of the maximiser
            if (row_ok) {
              if constexpr (kMode == 2) {
                int mi = 0;
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  if (c0 + c < col_end &&
                      (ep.col_perm ? (int64_t)ep.col_perm[c0 + c] : (int64_t)(c0 + c)) != gi)
                    mi = max(mi, abs((int)v[c]));
                wmax = fmaxf(wmax, __double2float_rd((double)mi * sc - ndel));
              } else {
                float mm = 0.f;
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  if (c0 + c < col_end && c0 + c != gi) mm = fmaxf(mm, fabsf(__uint_as_float(v[c])));
                wmax = fmaxf(wmax, mm - (thr - tfast));
              }
            }
            continue;
          }
          // common case first, one vote per 32 columns: no lane has an |acc|
          // above the tile's threshold (one FMNMX3 per two values), its
          // diagonal or a support entry of Omega in these columns
          bool over;
          if constexpr (kMode == 2) {
            // integer max / min over the 32 accumulators (3-input VIMNMX)
            int hi = (int)v[0], lo = (int)v[0];
#pragma unroll
            for (int c = 1; c < 31; c += 2) {
              hi = __vimax3_s32(hi, (int)v[c], (int)v[c + 1]);
              lo = __vimin3_s32(lo, (int)v[c], (int)v[c + 1]);
            }
            hi = max(hi, (int)v[31]);
            lo = min(lo, (int)v[31]);
            over = hi > tint || lo < -tint;
          } else {
            float m0 = 0.f, m1 = 0.f;
            if constexpr (kFast) {
#pragma unroll
              for (int c = 0; c < 32; c += 2) {
                m0 = fmaxf(m0, fabsf(__uint_as_float(v[c])));
                m1 = fmaxf(m1, fabsf(__uint_as_float(v[c + 1])));
              }
            } else {
              m0 = INFINITY;
            }
            over = fmaxf(m0, m1) > tfast;
          }
          const bool hot =
              row_ok && (over || (kMode == 0 && (nxt < c0 + 32 || (gi >= c0 && gi < c0 + 32))));
          if (!__any_sync(0xffffffffu, hot)) continue;
          uint32_t mask = 0, sup = 0;
          if (hot) {
            if (over) {
              if constexpr (kMode == 2) {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  mask |= (abs((int)v[c]) > tint ? 1u : 0u) << c;
              } else {
#pragma unroll
                for (int c = 0; c < 32; ++c)
                  mask |= (fabsf(__uint_as_float(v[c])) > tfast ? 1u : 0u) << c;
              }
            }
            if (kMode == 1 && ep.exact_cols && mask) {
              // exact per-column bound for the survivors of the tile-level test
              // (optional: the tile test alone is already a certified superset;
              // where lambda is only ~2.5 sd of the null S, e.g. config 3, nearly
              // every 32-column chunk has a survivor and these predicated loads
              // dominated the epilogue)
#pragma unroll
              for (int c = 0; c < 32; ++c) {
                if (mask & (1u << c)) {
                  const float2 sd = __ldg(&ep.col_sd[min(c0 + c, (int)ep.p - 1)]);
                  if (!(fabsf(__uint_as_float(v[c])) > thr - fmaf(r1, sd.x, Bn * sd.y)))
                    mask &= ~(1u << c);
                }
              }
            }
            if (kMode == 0 && gi >= c0 && gi < c0 + 32) mask |= 1u << (gi - c0);   // diagonal
            while (kMode == 0 && nxt < c0 + 32) {                     // support of Omega
              sup |= 1u << (nxt - c0);
              ++sp;
              nxt = sp < se ? om.col[sp] : INT_MAX;
            }
            mask |= sup;
            const int64_t left = col_end - c0;                        // ragged p / slab
            if (left < 32) mask &= left <= 0 ? 0u : ((1u << left) - 1u);
          }
          if (__ballot_sync(0xffffffffu, mask != 0u) == 0u) continue;
          // sym, off-diagonal tile: each survivor (i,k) is also (k,i) (G = G^T;
          // the bound on |acc_ik - G_ik| is one on |acc_ik - G_ki|). Row k is
          // this rank's (into the pool) or another rank's (into the mirror
          // buffer, sent after the GEMM); a 32-column chunk never straddles a
          // rank boundary (multiples of 256)
          const bool mirror = kMode != 0 && sched.sym && it.n() != sched.mt0 + it.m;
          const bool mir_local = mirror && (int64_t)c0 >= ep.r0 && (int64_t)c0 < ep.r0 + ep.pk;
          const bool mir_remote = kDiag == 3 && mirror && !mir_local;
          const int cnt = __popc(mask) << (mir_local ? 1 : 0);
          const int total = __reduce_add_sync(0xffffffffu, cnt);
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          if (fill + total > pool.chunk) {   // chunk full: record it, take the next one
            if (lane == 0 && chunk_id >= 0 && chunk_id < pool.nchunks)
              pool.chunk_fill[chunk_id] = (unsigned long long)fill;
            unsigned int nc = 0;
            if (lane == 0) nc = atomicAdd(pool.chunk_next, 1u);
            chunk_id = (long long)__shfl_sync(0xffffffffu, nc, 0);
            fill = 0;
          }
          const bool writable = chunk_id < pool.nchunks;
          int64_t pos = chunk_id * pool.chunk + fill + (incl - cnt);
          fill += total;
          row_count += cnt;
          int64_t rpos = 0;
          if (kDiag == 3 && mir_remote) {   // warp-aggregated reservation in the mirror buffer
            const int rc = __popc(mask);
            int rincl = rc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int y = __shfl_up_sync(0xffffffffu, rincl, o);
              if (lane >= o) rincl += y;
            }
            const int rtot = __shfl_sync(0xffffffffu, rincl, 31);
            unsigned long long base = 0;
            if (lane == 0) base = atomicAdd(ep.mir_cnt, (unsigned long long)rtot);
            base = __shfl_sync(0xffffffffu, base, 0);
            rpos = (int64_t)base + rincl - rc;
          }
          if constexpr (kMode != 0) {
            // candidate positions only: the exact values come from the refine
            // SDDMM and omega_ik from a lookup in Omega's CSR after the sort
            // (no dependent load of Omega's values on the epilogue's path)
            uint32_t m = mask;
            while (m) {
              const int c = __ffs(m) - 1;
              m &= m - 1;
              if (writable) {
                pool.row[pos] = (int32_t)r;
                pool.col[pos] = (kMode == 2 && ep.col_perm) ? ep.col_perm[c0 + c] : c0 + c;
              }
              ++pos;
              if (mir_local) {
                const int32_t kr = (int32_t)(c0 + c - ep.r0);
                if (writable) {
                  pool.row[pos] = kr;
                  pool.col[pos] = (int32_t)gi;
                }
                ++pos;
                atomicAdd(&pool.row_cnt[kr], 1);
              } else if (kDiag == 3 && mir_remote) {
                if (rpos < ep.mir_cap) {
                  ep.mir_row[rpos] = c0 + c;
                  ep.mir_col[rpos] = (int32_t)gi;
                }
                ++rpos;
              }
            }
            if (mir_local) row_count -= cnt >> 1;   // row r gained only the direct half
          } else if (cnt) {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
              if (mask & (1u << c)) {
                float w = 0.f;
                if (sup & (1u << c)) w = omv[sp0 + __popc(sup & ((1u << c) - 1u))];
                if (writable) {
                  pool.row[pos] = (int32_t)r;
                  pool.col[pos] = c0 + c;
                  ((float*)pool.g)[pos] = __uint_as_float(v[c]) * inv_nf;
                  ((float*)pool.w)[pos] = w;
                }
                ++pos;
              }
            }
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote(tempty_leader + acc * 8, 0);
      if (row_count) atomicAdd(&pool.row_cnt[r], row_count);
      if (++acc == kAccStages) { acc = 0; acc_phase ^= 1; }
    }
    if (lane == 0 && chunk_id >= 0 && chunk_id < pool.nchunks)
      pool.chunk_fill[chunk_id] = (unsigned long long)fill;
    if constexpr (kDiag == 2) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
      if (lane == 0 && wmax > 0.f) atomicMax(ep.max_out, __float_as_uint(wmax));
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  if (warp == 2) tc::tmem_dealloc<kTmemCols, 2>(tmem_base);
}

// per-256-column-block maxima of the filter's column constants
// (perm: column k' of the tile order holds variable perm[k'])
__global__ void blk_max_kernel(const float2* __restrict__ col_sd, int64_t p, int nblk,
                               const int32_t* __restrict__ perm, float2* __restrict__ out) {
  const int b = blockIdx.x;
  float mx = 0.f, my = 0.f;
  for (int j = threadIdx.x; j < BN; j += blockDim.x) {
    const int64_t k = (int64_t)b * BN + j;
    if (k < p) {
      const float2 v = col_sd[perm ? perm[k] : k];
      mx = fmaxf(mx, v.x);
      my = fmaxf(my, v.y);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    my = fmaxf(my, __shfl_xor_sync(0xffffffffu, my, o));
  }
  __shared__ float sx[32], sy[32];
  if ((threadIdx.x & 31) == 0) { sx[threadIdx.x >> 5] = mx; sy[threadIdx.x >> 5] = my; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { mx = fmaxf(mx, sx[w]); my = fmaxf(my, sy[w]); }
    out[b] = make_float2(mx, my);
  }
  (void)nblk;
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

// rows x kdim bf16 (row stride ldk elements); the box runs past kdim into TMA
// zero fill, so the padding columns [kdim, ldk) are never read
bool make_map(CUtensorMap* m, const void* base, int64_t rows, int64_t kdim, int64_t ldk,
              int box_rows, std::string* err, bool i8 = false) {
  auto fn = encode_fn();
  if (!fn) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)kdim, (cuuint64_t)rows};
  // int8: 128 elements per 128-B swizzle row (the same bytes as 64 bf16)
  cuuint64_t strides[1] = {(cuuint64_t)(ldk * (i8 ? 1 : 2))};
  cuuint32_t box[2] = {(cuuint32_t)(i8 ? 2 * BK : BK), (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides,
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
  // B operand maps: [0] = X^T (all columns, or this rank's slab when X is
  // sharded), [1], [2] = the two ring buffers of the sharded mode (NEXT(3))
  // A operand maps: [0], [1] = the two Y buffers, [2] = this rank's rows of
  // X^T_hi (Omega = I operand of the lambda_max pass, tc_plan_set_a)
  CUtensorMap a_hi[3], a_lo[3], b_hi[3], b_lo[3];
  // I8_FILTER: A maps over the two int8 Y buffers (+ [2] = an override), B
  // over int8 X^T
  CUtensorMap a_q[3], b_q;
  bool has_i8 = false;
  float2* blk_q = nullptr;       // [p_pad / 256] tile maxima of the int8 constants
  int64_t pk_pad = 0, p_pad = 0, ldk = 0, kdim = 0;   // p_pad: padded column count (all p)
  float2* blk_sdmax = nullptr;   // [p_pad / 256] (BF16_FILTER; caller-owned, zeroed)
};

bool tc_supported(int cc_major, int cc_minor) { return cc_major == 10 && cc_minor == 0; }

TcGemmPlan* tc_plan_create(const __nv_bfloat16* Yhi0, const __nv_bfloat16* Ylo0,
                           const __nv_bfloat16* Yhi1, const __nv_bfloat16* Ylo1, int64_t pk_pad,
                           const __nv_bfloat16* Xhi, const __nv_bfloat16* Xlo, int64_t xrows_pad,
                           int64_t p_pad, int64_t kdim, int64_t ldk, float2* blk_sdmax,
                           std::string* err) {
  auto* p = new TcGemmPlan();
  if (std::getenv("ACCORD_GEMM_KFULL")) kdim = ldk;   // A-B diagnostic: no K-tail trim
  p->pk_pad = pk_pad;
  p->p_pad = p_pad;
  p->ldk = ldk;
  p->kdim = kdim;
  bool ok = make_map(&p->a_hi[0], Yhi0, pk_pad, kdim, ldk, BM, err) &&
            make_map(&p->a_lo[0], Ylo0, pk_pad, kdim, ldk, BM, err) &&
            make_map(&p->a_hi[1], Yhi1, pk_pad, kdim, ldk, BM, err) &&
            make_map(&p->a_lo[1], Ylo1, pk_pad, kdim, ldk, BM, err) &&
            make_map(&p->b_hi[0], Xhi, xrows_pad, kdim, ldk, BNH, err) &&
            make_map(&p->b_lo[0], Xlo, xrows_pad, kdim, ldk, BNH, err);
  p->b_hi[1] = p->b_hi[2] = p->b_hi[0];
  p->b_lo[1] = p->b_lo[2] = p->b_lo[0];
  p->a_hi[2] = p->a_hi[0];
  p->a_lo[2] = p->a_lo[0];
  p->blk_sdmax = blk_sdmax;   // owned by the caller
  if (!ok) {
    delete p;
    return nullptr;
  }
  static unsigned long long attr_seen = 0;
  if (attr_needed(attr_seen)) {
    cudaFuncSetAttribute(gemm_tc_kernel<0, 3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg<0, 3>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<1, 6, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg<1, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<1, 7, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg<1, 7>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<1, 6, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg<1, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<1, 6, true, 1>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<1, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<1, 6, true, 2>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<1, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<1, 6, true, 3>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<1, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<2, 6, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)Cfg<2, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<1, 6, true, 0, 8>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<1, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<2, 6, true, 0, 16>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<2, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<2, 6, true, 1>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<2, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<2, 6, true, 2>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<2, 6>::kSmemBytes);
    cudaFuncSetAttribute(gemm_tc_kernel<2, 6, true, 3>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg<2, 6>::kSmemBytes);
    attr_done(attr_seen);
  }
  return p;
}

bool tc_plan_set_a(TcGemmPlan* p, int idx, const __nv_bfloat16* hi, int64_t rows_pad,
                   std::string* err) {
  return make_map(&p->a_hi[idx], hi, rows_pad, p->kdim, p->ldk, BM, err) &&
         make_map(&p->a_lo[idx], hi, rows_pad, p->kdim, p->ldk, BM, err);
}

bool tc_plan_set_b(TcGemmPlan* p, int idx, const __nv_bfloat16* hi, const __nv_bfloat16* lo,
                   int64_t rows_pad, std::string* err) {
  return make_map(&p->b_hi[idx], hi, rows_pad, p->kdim, p->ldk, BNH, err) &&
         make_map(&p->b_lo[idx], lo, rows_pad, p->kdim, p->ldk, BNH, err);
}

bool tc_plan_set_i8(TcGemmPlan* p, const int8_t* Yq0, const int8_t* Yq1, const int8_t* Xq,
                    int64_t xrows_pad, float2* blk_q, std::string* err) {
  p->blk_q = blk_q;
  p->has_i8 = make_map(&p->a_q[0], Yq0, p->pk_pad, p->kdim, p->ldk, BM, err, true) &&
              make_map(&p->a_q[1], Yq1, p->pk_pad, p->kdim, p->ldk, BM, err, true) &&
              make_map(&p->b_q, Xq, xrows_pad, p->kdim, p->ldk, BNH, err, true);
  p->a_q[2] = p->a_q[0];
  return p->has_i8;
}

bool tc_plan_set_a_i8(TcGemmPlan* p, int idx, const int8_t* q, int64_t rows_pad,
                      std::string* err) {
  return make_map(&p->a_q[idx], q, rows_pad, p->kdim, p->ldk, BM, err, true);
}

int tc_plan_set_col_norms(TcGemmPlan* p, const float2* col_sd, int64_t pcols, cudaStream_t st,
                          bool i8, const int32_t* perm) {
  const int nblk = (int)(p->p_pad / BN);
  blk_max_kernel<<<nblk, 256, 0, st>>>(col_sd, pcols, nblk, perm, i8 ? p->blk_q : p->blk_sdmax);
  return 1;
}

void tc_plan_destroy(TcGemmPlan* p) {
  if (!p) return;
  delete p;
}

int tc_grid_size(const TcGemmPlan* plan, int sm_count) {
  const int64_t tiles = (plan->pk_pad / (2 * BM)) * (plan->p_pad / BN);
  const int64_t clusters = tiles < sm_count / 2 ? tiles : sm_count / 2;
  return (int)(2 * clusters);
}

int launch_gemm_tc(TcGemmPlan* plan, int mode, int ybuf, int bsel, int sm_count,
                   const EpiParams& ep, const OmegaView& om, const PoolView& pool,
                   cudaStream_t st) {
  const int num_m = (int)(plan->pk_pad / (2 * BM));
  const int num_n = (int)((ep.col_end - ep.col_base + BN - 1) / BN);
  const int64_t kdim = plan->kdim;
  const bool i8 = mode == ACCORD_GEMM_I8_FILTER;
  if (i8 && !plan->has_i8) return -1;
  const int bke = i8 ? 2 * BK : BK;                       // K elements per 128-B k-block
  const int kmma = i8 ? 32 : 16;                          // K per MMA
  const int num_kb = (int)((kdim + bke - 1) / bke);
  const int kk_last = (int)((kdim - (int64_t)(num_kb - 1) * bke + kmma - 1) / kmma);   // 1..4
  const int grid = tc_grid_size(plan, sm_count);
  // A group of <= 64 N-blocks (<= 32 MB of X^T_hi at n = 1000) stays in L2;
  // units small enough that the per-cluster imbalance is <= ~6% of its work
  // X^T group of gn N-blocks (gn x 256 rows x ldk bf16 stay L2-resident):
  // measured best 48 at ldk = 1024 (c5, 6 alternating reps), 32 at ldk = 2048
  int gn = plan->ldk <= 1024 ? 48 : 32;
  if (const char* e = std::getenv("ACCORD_GEMM_GN")) gn = std::max(1, std::atoi(e));   // tuning
  const int group_n = num_n < gn ? num_n : gn;
  const long long tiles = (long long)num_m * num_n;
  long long u = tiles / ((long long)(grid / 2) * 16);
  if (const char* e = std::getenv("ACCORD_GEMM_UNIT")) u = std::max(1, std::atoi(e));  // tuning
  const int unit_n = (int)(u < 1 ? 1 : (u > group_n ? group_n : u));
  // ACCORD_DEBUG_GEMM (diagnostics only; results are wrong when set):
  // 1 = skip the epilogue, 2 = skip the MMAs
  const char* dbg_env = std::getenv("ACCORD_DEBUG_GEMM");
  const int dbg = dbg_env ? std::atoi(dbg_env) : 0;
  // ACCORD_GEMM_VARIANT (tuning / A-B diagnostics, results identical):
  // 0 = 6-stage ring + FMNMX3 fast path (default), 1 = 7 stages, 2 = no fast path,
  // 3 = bf16 with 8 epilogue warps (the int8 kernel's split), 4 = int8 with 16
  int var = 0;
  if (const char* e = std::getenv("ACCORD_GEMM_VARIANT")) var = std::atoi(e);
  // ACCORD_GEMM_L2HINT (tuning): 1 = TMA loads of X^T with evict_last, 2 = evict_first
  int l2hint = 0;
  if (const char* e = std::getenv("ACCORD_GEMM_L2HINT")) l2hint = std::atoi(e);
#define ACCORD_TC_ARGS(bsel_lo)                                                               \
  plan->a_hi[ybuf], plan->a_lo[ybuf], plan->b_hi[bsel], bsel_lo, num_kb, kk_last, num_m,   \
      num_n, group_n, unit_n, dbg, l2hint, ep, plan->blk_sdmax, om, pool
#define ACCORD_TC_ARGS_I8                                                                    \
  plan->a_q[ybuf], plan->a_q[ybuf], plan->b_q, plan->b_q, num_kb, kk_last, num_m, num_n,     \
      group_n, unit_n, dbg, l2hint, ep, plan->blk_q, om, pool
  if (i8) {
    if (bsel != 0) return -1;   // no sharded-X ring in int8
    if (ep.audit_acc)
      gemm_tc_kernel<2, 6, true, 1><<<grid, Cfg<2, 6>::kThreads, Cfg<2, 6>::kSmemBytes, st>>>(
          ACCORD_TC_ARGS_I8);
    else if (ep.max_out)
      gemm_tc_kernel<2, 6, true, 2><<<grid, Cfg<2, 6>::kThreads, Cfg<2, 6>::kSmemBytes, st>>>(
          ACCORD_TC_ARGS_I8);
    else if (ep.sym == 2)
      gemm_tc_kernel<2, 6, true, 3><<<grid, Cfg<2, 6>::kThreads, Cfg<2, 6>::kSmemBytes, st>>>(
          ACCORD_TC_ARGS_I8);
    else if (var == 4)   // A-B: 16 epilogue warps (64 columns each)
      gemm_tc_kernel<2, 6, true, 0, 16><<<grid, Cfg<2, 6, 16>::kThreads, Cfg<2, 6>::kSmemBytes,
                                          st>>>(ACCORD_TC_ARGS_I8);
    else
      gemm_tc_kernel<2, 6, true><<<grid, Cfg<2, 6>::kThreads, Cfg<2, 6>::kSmemBytes, st>>>(
          ACCORD_TC_ARGS_I8);
  } else if (mode == ACCORD_GEMM_BF16X3)
    gemm_tc_kernel<0, 3, true><<<grid, kThreads, Cfg<0, 3>::kSmemBytes, st>>>(
        ACCORD_TC_ARGS(plan->b_lo[bsel]));
  else if (ep.audit_acc)
    gemm_tc_kernel<1, 6, true, 1><<<grid, kThreads, Cfg<1, 6>::kSmemBytes, st>>>(
        ACCORD_TC_ARGS(plan->b_hi[bsel]));
  else if (ep.max_out)
    gemm_tc_kernel<1, 6, true, 2><<<grid, kThreads, Cfg<1, 6>::kSmemBytes, st>>>(
        ACCORD_TC_ARGS(plan->b_hi[bsel]));
  else if (ep.sym == 2)
    gemm_tc_kernel<1, 6, true, 3><<<grid, kThreads, Cfg<1, 6>::kSmemBytes, st>>>(
        ACCORD_TC_ARGS(plan->b_hi[bsel]));
  else if (var == 1)
    gemm_tc_kernel<1, 7, true><<<grid, kThreads, Cfg<1, 7>::kSmemBytes, st>>>(
        ACCORD_TC_ARGS(plan->b_hi[bsel]));
  else if (var == 2)
    gemm_tc_kernel<1, 6, false><<<grid, kThreads, Cfg<1, 6>::kSmemBytes, st>>>(
        ACCORD_TC_ARGS(plan->b_hi[bsel]));
  else if (var == 3)
    gemm_tc_kernel<1, 6, true, 0, 8><<<grid, Cfg<1, 6, 8>::kThreads, Cfg<1, 6>::kSmemBytes, st>>>(
        ACCORD_TC_ARGS(plan->b_hi[bsel]));
  else
    gemm_tc_kernel<1, 6, true><<<grid, kThreads, Cfg<1, 6>::kSmemBytes, st>>>(
        ACCORD_TC_ARGS(plan->b_hi[bsel]));
#undef ACCORD_TC_ARGS
#undef ACCORD_TC_ARGS_I8
  return 1;
}

}  // namespace accord

// a6 SpMM, TMA-staged: Y+_i = sum_j w+_ij X^T_j and
// D_i = sum_j Delta_ij X^T_j (PAPER.md:357 two-step gradient, :258 Delta),
// with the fused row norms ||D_i||^2, ||Y+_i||^2 and the bf16 GEMM operand
// copy of Y+ (DESIGN.md §5).
//
// The op is a gather of whole X^T rows (n floats each, at c5 mostly from
// DRAM: the off-block candidates hit random columns), so it is bound by
// memory-level parallelism, not arithmetic. One producer warp per block walks
// the block's work items (row chunks of <= kItemEntries entries of C, the
// CSR of the trial), drops entries with w+ = Delta = 0, and streams each
// needed X^T row into a ring of shared-memory stages with cp.async.bulk
// (one 4 KB bulk copy per entry at n = 1000, completion on an mbarrier).
// Consumer warps (8 columns per thread) accumulate in float64 from shared
// memory. The register file no longer limits the bytes in flight: ~16 stages
// x 3 blocks per SM = 192 KB per SM.
//
// Rows longer than one item (hub rows, up to 1.6e5 candidates at c5) are
// split over several items processed by different blocks: each writes its
// partial sums to a scratch slot, and the block that completes the row (an
// atomic counter per row) adds the slots in chunk order, so the result does
// not depend on which block finishes last (deterministic).
#include "accord_internal.h"
#include "tc_ptx.cuh"

#include <algorithm>
#include <cstdlib>

namespace accord {
namespace {

constexpr int kFlagData = 1, kFlagLast = 2, kFlagEnd = 4;

struct StageMeta {
  double w, d, d2;                  // d2: Delta of the second step size (kPair)
  int64_t row;
  int32_t chunk, nch;
  int32_t flags, pad;
};

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ double wsum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// kPair: also D' = (W' - Wold) X^T for a second trial step (weights wn2),
// of which only the row norms ||D'_i||^2 are kept (row_D2b): one gather pass
// serves two line-search trials.
// kCols: output columns per consumer thread (8: two float4 per staged row;
// 4: one float4, twice the consumer warps per block and a third of the
// accumulator registers -- more warps in flight per SM)
// kMinB: resident blocks the register budget is sized for (0 = the default:
// 3 for the paired kernel, whose 128-register cap spills ~176 B; 2 = no
// spills, fewer warps: ACCORD_SPMM_MINB=2, A-B)
template <bool kPair, int kCols, int kMinB = 0>
__global__ void __launch_bounds__(kCols == 4 ? 32 + kSpmmTmaMaxConsumers
                                  : (kPair ? 32 + kSpmmPairMaxConsumers : 32 + kSpmmTmaMaxConsumers),
                                  kMinB ? kMinB : (kCols == 4 ? (kPair ? 2 : 3) : (kPair ? 3 : 2)))
spmm_tma_kernel(int64_t pk, int64_t ldk, int stages, const int64_t* __restrict__ ptr,
                const int32_t* __restrict__ col, const float* __restrict__ wn,
                const float* __restrict__ wo, const float* __restrict__ Xt, float* __restrict__ Yout,
                __nv_bfloat16* __restrict__ Yhi, __nv_bfloat16* __restrict__ Ylo,
                float* __restrict__ row_A, float* __restrict__ row_B, double* __restrict__ row_D2,
                double* __restrict__ row_Y2, const float* __restrict__ wn2,
                double* __restrict__ row_D2b, SpmmItems items, int ydrop,
                int par_emit) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t stage_bytes = (uint32_t)(ldk * 4);
  float* data = reinterpret_cast<float*>(sm);
  StageMeta* meta = reinterpret_cast<StageMeta*>(sm + (size_t)stages * stage_bytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(meta + stages);
  uint64_t* empty = full + stages;
  double* red = reinterpret_cast<double*>(empty + stages);   // [5][16] + flag
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncw = (blockDim.x >> 5) - 1;                     // consumer warps
  const int nct = ncw * 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      tc::mbar_init(tc::smem_u32(&full[s]), 1);
      tc::mbar_init(tc::smem_u32(&empty[s]), ncw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t n_items = items.itm_ptr[pk];

  if (warp == 0) {
    // ============================== producer ==============================
    int stage = 0;
    uint32_t phase = 0;
    auto emit = [&](double w, double d, double d2, int32_t c, int flags, int64_t row, int chunk,
                    int nch) {
      tc::mbar_wait(tc::smem_u32(&empty[stage]), phase ^ 1);
      if (lane == 0) {
        StageMeta& m = meta[stage];
        m.w = w;
        m.d = d;
        m.d2 = d2;
        m.row = row;
        m.chunk = chunk;
        m.nch = nch;
        m.flags = flags;
        // every stage carries a row: a dataless one (an item whose entries
        // were all dropped, the end marker) gets X^T row 0 with zero weights,
        // which adds exact zeros (X is finite, checked at create), so the
        // consumer loop has no data / no-data branch
        const uint32_t fb = tc::smem_u32(&full[stage]);
        tc::mbar_arrive_expect_tx(fb, stage_bytes);
        bulk_g2s(tc::smem_u32(data + (size_t)stage * ldk),
                 Xt + (int64_t)((flags & kFlagData) ? c : 0) * ldk, stage_bytes, fb);
      }
      __syncwarp();
      if (++stage == stages) { stage = 0; phase ^= 1; }
    };
    // Items it = blockIdx.x + k * gridDim.x. Their metadata is fetched 32 at a
    // time (lane j holds item j of the batch: row from the item->row map, entry
    // range, chunk), and the first 32 entries of the next item are loaded while
    // the current one is being emitted, so the producer's global-memory
    // latencies overlap the copies in flight.
    const int64_t G = gridDim.x;
    // the item -> row map of the next batch of 32 items is loaded one batch
    // ahead (one dependent global latency per batch instead of two)
    int32_t row_next = 0;
    {
      const int64_t itj0 = blockIdx.x + (int64_t)lane * G;
      if (itj0 < n_items) row_next = items.item_row[itj0];
    }
    for (int64_t base = blockIdx.x; base < n_items; base += 32 * G) {
      const int64_t itj = base + (int64_t)lane * G;
      const bool vj = itj < n_items;
      const int64_t rj = vj ? (int64_t)row_next : 0;
      {
        const int64_t itn = itj + 32 * G;
        row_next = itn < n_items ? items.item_row[itn] : 0;
      }
      const int64_t i0 = items.itm_ptr[rj], i1 = items.itm_ptr[rj + 1];
      const int64_t p0 = ptr[rj], p1 = ptr[rj + 1];
      const int chj = (int)(itj - i0), nchj = (int)(i1 - i0);
      const int64_t begj = p0 + (int64_t)chj * items.L;
      const int64_t endj = min(p1, begj + items.L);
      const int nv = __popc(__ballot_sync(0xffffffffu, vj));
      // entries of the first item
      // raw loads (no use of the values: the warp does not wait for them
      // here) and the conversion where the values are consumed
      struct Raw { float w, o, w2; int32_t cc; };
      auto load_raw = [&](int64_t e, int64_t end, Raw& q) {
        if (e < end) {
          q.w = __ldg(wn + e);
          q.o = wo ? __ldg(wo + e) : 0.f;
          q.w2 = kPair ? __ldg(wn2 + e) : 0.f;
          q.cc = __ldg(col + e);
        } else {
          q.w = 0.f; q.o = 0.f; q.w2 = 0.f; q.cc = 0;
        }
      };
      auto cvt = [&](const Raw& q, double& w, double& d, double& d2, int32_t& cc) {
        w = (double)q.w;
        d = wo ? w - (double)q.o : 0.0;
        d2 = kPair ? (double)q.w2 - (double)q.o : 0.0;
        cc = q.cc;
      };
      // lookahead of two items: the first 32 entries of items k+1 (set a)
      // and k+2 (set b) are in flight while item k is emitted (items have
      // ~10 entries in the steady state, so one item of lookahead left the
      // producer waiting on these loads: ncu, int8-filter c5 run)
      Raw qa{0.f, 0.f, 0.f, 0}, qb{0.f, 0.f, 0.f, 0};
      // the second 32 entries of items k+1, k+2 are in flight as well (the
      // int8 filter leaves ~60 candidates per row at c5, i.e. two batches per
      // item: round 2c A-B, 27.9 -> 26.7 ms per step)
      Raw qa2{0.f, 0.f, 0.f, 0}, qb2{0.f, 0.f, 0.f, 0};
      {
        const int64_t b0 = __shfl_sync(0xffffffffu, begj, 0), e0_ = __shfl_sync(0xffffffffu, endj, 0);
        load_raw(b0 + lane, e0_, qa);
        const int64_t b1 = __shfl_sync(0xffffffffu, begj, 1), e1_ = __shfl_sync(0xffffffffu, endj, 1);
        if (nv > 1) load_raw(b1 + lane, e1_, qb);
        load_raw(b0 + 32 + lane, e0_, qa2);
        if (nv > 1) load_raw(b1 + 32 + lane, e1_, qb2);
      }
      for (int k = 0; k < nv; ++k) {
        const int64_t r = __shfl_sync(0xffffffffu, rj, k);
        const int chunk = __shfl_sync(0xffffffffu, chj, k);
        const int nch = __shfl_sync(0xffffffffu, nchj, k);
        const int64_t beg = __shfl_sync(0xffffffffu, begj, k);
        const int64_t end = __shfl_sync(0xffffffffu, endj, k);
        double w, d, d2;
        int32_t cc;
        cvt(qa, w, d, d2, cc);
        qa = qb;
        const Raw q2 = qa2;
        qa2 = qb2;
        {
          const int kn = k + 2 < 32 ? k + 2 : 31;
          const int64_t bn = __shfl_sync(0xffffffffu, begj, kn);
          const int64_t en = __shfl_sync(0xffffffffu, endj, kn);
          if (k + 2 < nv) load_raw(bn + lane, en, qb);
          if (k + 2 < nv) load_raw(bn + 32 + lane, en, qb2);
        }
        // one entry of lookahead so that the item's last nonzero carries kFlagLast
        bool pend = false;
        double pw = 0.0, pd = 0.0, pd2 = 0.0;
        int32_t pc = 0;
        Raw qn{0.f, 0.f, 0.f, 0};
        for (int64_t e0 = beg; e0 < end; e0 += 32) {
          // batch 0 came with the item lookahead (qa), batch 1 too (q2); from
          // batch 2 on (long rows: the first iterations, hub rows) each batch
          // is requested while the previous one is being emitted
          if (e0 == beg + 32) cvt(q2, w, d, d2, cc);
          else if (e0 != beg) cvt(qn, w, d, d2, cc);
          if (e0 != beg && e0 + 32 < end) load_raw(e0 + 32 + lane, end, qn);
          const bool keep = (e0 + lane < end) && ((w != 0.0) || (d != 0.0) || (d2 != 0.0));
          const unsigned m = __ballot_sync(0xffffffffu, keep);
          if (!m) continue;
          if (!par_emit) {   // one entry at a time (ACCORD_SPMM_SERIAL=1, A-B)
            unsigned mm = m;
            while (mm) {
              const int src = __ffs(mm) - 1;
              mm &= mm - 1;
              const double ws = __shfl_sync(0xffffffffu, w, src);
              const double ds = __shfl_sync(0xffffffffu, d, src);
              const double ds2 = kPair ? __shfl_sync(0xffffffffu, d2, src) : 0.0;
              const int32_t cs = __shfl_sync(0xffffffffu, cc, src);
              if (pend) emit(pw, pd, pd2, pc, kFlagData, r, chunk, nch);
              pend = true;
              pw = ws;
              pd = ds;
              pd2 = ds2;
              pc = cs;
            }
            continue;
          }
          // Warp-parallel issue: every kept lane fills its own stage (its
          // rank among this batch's entries), up to `stages` per round, so a
          // batch costs one round of waits / metadata / bulk copies instead
          // of one serial emit per entry (a single producer's serial issue
          // rate limited the ring: DESIGN §7, gather microbenchmark). The
          // highest kept lane's entry is held back as the new pending one
          // (the item's last entry must carry kFlagLast); that lane emits the
          // previous pending entry at rank 0. Stages are filled in the same
          // order as by the serial loop, so the sums are bitwise the same.
          const int hi = 31 - __clz(m);
          const unsigned em = m & ~(1u << hi);
          const int p0 = pend ? 1 : 0;
          int myrank = -1;
          if (lane == hi) myrank = pend ? 0 : -1;
          else if ((em >> lane) & 1u) myrank = p0 + __popc(em & ((1u << lane) - 1u));
          const int cnt = p0 + __popc(em);
          for (int r0 = 0; r0 < cnt; r0 += stages) {
            const int nr = min(stages, cnt - r0);
            if (myrank >= r0 && myrank < r0 + nr) {
              int si = stage + (myrank - r0);
              uint32_t ph = phase;
              if (si >= stages) { si -= stages; ph ^= 1; }
              tc::mbar_wait(tc::smem_u32(&empty[si]), ph ^ 1);
              const bool mine = lane != hi;
              StageMeta& mt = meta[si];
              mt.w = mine ? w : pw;
              mt.d = mine ? d : pd;
              mt.d2 = mine ? d2 : pd2;
              mt.row = r;
              mt.chunk = chunk;
              mt.nch = nch;
              mt.flags = kFlagData;
              const uint32_t fb = tc::smem_u32(&full[si]);
              tc::mbar_arrive_expect_tx(fb, stage_bytes);
              bulk_g2s(tc::smem_u32(data + (size_t)si * ldk), Xt + (int64_t)(mine ? cc : pc) * ldk,
                       stage_bytes, fb);
            }
            // a round's lanes must have passed their waits before the next
            // round's lanes wait on the same stages for the following phase
            // (a parity wait one phase ahead would return at once)
            __syncwarp();
            stage += nr;
            if (stage >= stages) { stage -= stages; phase ^= 1; }
          }
          pend = true;
          pw = __shfl_sync(0xffffffffu, w, hi);
          pd = __shfl_sync(0xffffffffu, d, hi);
          pd2 = kPair ? __shfl_sync(0xffffffffu, d2, hi) : 0.0;
          pc = __shfl_sync(0xffffffffu, cc, hi);
        }
        if (pend) emit(pw, pd, pd2, pc, kFlagData | kFlagLast, r, chunk, nch);
        else emit(0.0, 0.0, 0.0, 0, kFlagLast, r, chunk, nch);
      }
    }
    emit(0.0, 0.0, 0.0, 0, kFlagEnd | kFlagLast, 0, 0, 0);
    return;
  }

  // ================================ consumers ===============================
  const int t = threadIdx.x - 32;
  const int64_t c0 = (int64_t)t * kCols;
  const bool active = c0 < ldk;
  double ay[kCols], ad[kCols], ae[kCols];   // Y+, D, and D' (kPair)
#pragma unroll
  for (int v = 0; v < kCols; ++v) { ay[v] = 0.0; ad[v] = 0.0; ae[v] = 0.0; }
  int stage = 0;
  uint32_t phase = 0;
  // per-warp partials of a finished row, x 5 quantities, double-buffered by
  // row parity: thread 0 sums row q from one buffer while the other warps may
  // already write row q+1 into the other, so one barrier per row suffices
  int rowpar = 0;
  volatile int* sh_flag = reinterpret_cast<volatile int*>(red + 160);
  auto accumulate = [&](double w, double d, double d2, float4 x0, float4 x1) {
    const float xv[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
    for (int v = 0; v < kCols; ++v) {
      ay[v] = fma(w, (double)xv[v], ay[v]);
      ad[v] = fma(d, (double)xv[v], ad[v]);
      if constexpr (kPair) ae[v] = fma(d2, (double)xv[v], ae[v]);
    }
  };
  const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
  // this thread's columns in stage 0 (32-bit shared address; threads past the
  // row end read column 0 and discard it)
  const uint32_t data_u32 = tc::smem_u32(data) + (active ? (uint32_t)c0 * 4u : 0u);
  const uint32_t meta_u32 = tc::smem_u32(meta);
  // Two nested loops: the inner one walks the staged rows of one item with the
  // accumulators updated in place (a single back edge, one definition of each
  // accumulator at its head: with the finalize inside a single loop ptxas
  // merged two definitions and copied all 48 accumulator registers of the
  // paired kernel every round), the outer one zeroes them and finalizes.
  for (;;) {
#pragma unroll
    for (int v = 0; v < kCols; ++v) { ay[v] = 0.0; ad[v] = 0.0; ae[v] = 0.0; }
    int64_t m_row = 0;        // row / chunk of the finished item (read before the release)
    int m_chunk = 0, m_nch = 1, m_flags = 0;
    for (;;) {
      tc::mbar_wait(tc::smem_u32(&full[stage]), phase);
      // the stage's metadata (three 16-byte loads) and this thread's columns
      // are requested together: one shared-memory latency per round, and no
      // branch before the arithmetic
      const uint32_t ms = meta_u32 + (uint32_t)stage * (uint32_t)sizeof(StageMeta);
      const uint32_t xs = data_u32 + (uint32_t)stage * stage_bytes;
      double w0, d0, e0d;
      int64_t mrow;
      int mchunk, mnch, f0, mpad;
      asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(mchunk), "=r"(mnch), "=r"(f0), "=r"(mpad)
                   : "r"(ms + 32)
                   : "memory");
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w0), "=d"(d0) : "r"(ms) : "memory");
      asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=d"(e0d), "=l"(mrow) : "r"(ms + 16) : "memory");
      const float4 a0 = lds128(xs);
      const float4 b0 = kCols == 8 ? lds128(xs + 16) : z4;
      // unconditional: dataless stages carry zero weights and a finite row
      accumulate(w0, d0, kPair ? e0d : 0.0, a0, b0);
      const bool last = (f0 & kFlagLast) != 0;
      if (last) {
        m_row = mrow;
        m_chunk = mchunk;
        m_nch = mnch;
        m_flags = f0;
      }
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tc::smem_u32(&empty[stage]));
      if (++stage == stages) { stage = 0; phase ^= 1; }
      if (last) break;
    }
    if (m_flags & kFlagEnd) return;   // the end marker follows the last item
    {
      // ---------------- item complete: finalize the row (or its partial) ----
      const int64_t r = m_row;
      bool finish = true;
      if (m_nch > 1) {
        const int64_t slot0 = items.slot_ptr[r];
        if (active) {
          double* py = items.part_y + (slot0 + m_chunk) * ldk + c0;
          double* pd = items.part_d + (slot0 + m_chunk) * ldk + c0;
#pragma unroll
          for (int v = 0; v < kCols; ++v) { py[v] = ay[v]; pd[v] = ad[v]; }
          if constexpr (kPair) {
            double* pe = items.part_d2 + (slot0 + m_chunk) * ldk + c0;
#pragma unroll
            for (int v = 0; v < kCols; ++v) pe[v] = ae[v];
          }
        }
        __threadfence();
        named_sync(1, nct);
        if (t == 0) *sh_flag = (atomicAdd(&items.row_done[r], 1) == m_nch - 1) ? 1 : 0;
        named_sync(1, nct);
        finish = *sh_flag != 0;
        if (finish) {
          __threadfence();
          if (active) {
#pragma unroll
            for (int v = 0; v < kCols; ++v) { ay[v] = 0.0; ad[v] = 0.0; ae[v] = 0.0; }
            for (int k = 0; k < m_nch; ++k) {   // chunk order: deterministic sum
              const double* py = items.part_y + (slot0 + k) * ldk + c0;
              const double* pd = items.part_d + (slot0 + k) * ldk + c0;
#pragma unroll
              for (int v = 0; v < kCols; ++v) {
                ay[v] += __ldcg(py + v);
                ad[v] += __ldcg(pd + v);
              }
              if constexpr (kPair) {
                const double* pe = items.part_d2 + (slot0 + k) * ldk + c0;
#pragma unroll
                for (int v = 0; v < kCols; ++v) ae[v] += __ldcg(pe + v);
              }
            }
          }
          if (t == 0) items.row_done[r] = 0;   // ready for the next trial
        }
      }
      if (finish) {
        double d2 = 0.0, y2 = 0.0, a2 = 0.0, b2 = 0.0, e2 = 0.0;
        if (active) {
          float yt[kCols];
#pragma unroll
          for (int v = 0; v < kCols; ++v) {
            d2 += ad[v] * ad[v];
            y2 += ay[v] * ay[v];
            if constexpr (kPair) e2 += ae[v] * ae[v];
            yt[v] = (float)ay[v];
          }
          float* yo = Yout + r * ldk + c0;
          *reinterpret_cast<float4*>(yo) = make_float4(yt[0], yt[1], yt[2], yt[3]);
          if constexpr (kCols == 8)
            *reinterpret_cast<float4*>(yo + 4) = make_float4(yt[4], yt[5], yt[6], yt[7]);
          if (Yhi) {
            uint32_t hp[kCols / 2], lp[kCols / 2];
#pragma unroll
            for (int v = 0; v < kCols; v += 2) {
              const __nv_bfloat162 h2 =
                  ydrop ? __halves2bfloat162(filter_bf16_x(yt[v], ydrop), filter_bf16_x(yt[v + 1], ydrop))
                        : filter_bf16x2(yt[v], yt[v + 1]);
              const float2 hf = __bfloat1622float2(h2);
              const __nv_bfloat162 l2 = __floats2bfloat162_rn(yt[v] - hf.x, yt[v + 1] - hf.y);
              hp[v / 2] = *reinterpret_cast<const uint32_t*>(&h2);
              lp[v / 2] = *reinterpret_cast<const uint32_t*>(&l2);
              const double e0 = (double)yt[v] - (double)hf.x, e1 = (double)yt[v + 1] - (double)hf.y;
              a2 += e0 * e0 + e1 * e1;
              b2 += (double)yt[v] * (double)yt[v] + (double)yt[v + 1] * (double)yt[v + 1];
            }
            if constexpr (kCols == 8) {
              *reinterpret_cast<uint4*>(Yhi + r * ldk + c0) = make_uint4(hp[0], hp[1], hp[2], hp[3]);
              if (Ylo)
                *reinterpret_cast<uint4*>(Ylo + r * ldk + c0) = make_uint4(lp[0], lp[1], lp[2], lp[3]);
            } else {
              *reinterpret_cast<uint2*>(Yhi + r * ldk + c0) = make_uint2(hp[0], hp[1]);
              if (Ylo) *reinterpret_cast<uint2*>(Ylo + r * ldk + c0) = make_uint2(lp[0], lp[1]);
            }
          }
        }
        d2 = wsum(d2);
        y2 = wsum(y2);
        if (Yhi) {   // the operand-split norms exist only with the bf16 copy (block-uniform)
          a2 = wsum(a2);
          b2 = wsum(b2);
        }
        if constexpr (kPair) e2 = wsum(e2);
        const int cw = warp - 1;
        double* sh_red = red + rowpar * 80;
        rowpar ^= 1;
        if (lane == 0) {
          sh_red[cw] = d2;
          sh_red[16 + cw] = y2;
          sh_red[32 + cw] = a2;
          sh_red[48 + cw] = b2;
          sh_red[64 + cw] = e2;
        }
        named_sync(1, nct);
        if (t == 0) {
          double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0;
          for (int q = 0; q < ncw; ++q) {   // fixed order
            s0 += sh_red[q];
            s1 += sh_red[16 + q];
            s2 += sh_red[32 + q];
            s3 += sh_red[48 + q];
            s4 += sh_red[64 + q];
          }
          if (row_D2) row_D2[r] = s0;
          if (kPair && row_D2b) row_D2b[r] = s4;
          if (row_Y2) row_Y2[r] = s1;
          if (Yhi) {
            // rounded up: these enter an upper bound (the GEMM filter)
            if (row_A) row_A[r] = __double2float_ru(sqrt(s2) * (1.0 + 1e-12));
            if (row_B) row_B[r] = __double2float_ru(sqrt(s3) * (1.0 + 1e-12));
          }
        }
      }
    }
  }
}

}  // namespace

namespace {

// per row: work items (chunks of <= L entries, >= 1) and scratch slots
// (multi-chunk rows only)
__global__ void item_count_kernel(int64_t rows, const int64_t* __restrict__ ptr, int64_t L,
                                  int32_t* __restrict__ nitem, int32_t* __restrict__ nslot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t len = ptr[i + 1] - ptr[i];
    const int64_t c = len <= L ? 1 : (len + L - 1) / L;
    nitem[i] = (int32_t)c;
    nslot[i] = c > 1 ? (int32_t)c : 0;
  }
}

// item -> row (thread per row writes its items)
__global__ void item_row_kernel(int64_t rows, const int64_t* __restrict__ itm_ptr,
                                int32_t* __restrict__ item_row) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows;
       i += (int64_t)gridDim.x * blockDim.x)
    for (int64_t it = itm_ptr[i]; it < itm_ptr[i + 1]; ++it) item_row[it] = (int32_t)i;
}

}  // namespace

int launch_item_rows(int64_t rows, const int64_t* itm_ptr, int32_t* item_row, cudaStream_t st) {
  const unsigned g = (unsigned)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (rows + 255) / 256));
  item_row_kernel<<<g, 256, 0, st>>>(rows, itm_ptr, item_row);
  return 1;
}

size_t spmm_tma_smem(int64_t ldk, int* stages) {
  const int64_t sb = ldk * 4;
  // stages (4 KB each at n = 1000); 16 absorb the row finalize and the item
  // boundaries better than 8 (round 2c A-B: 26.7 -> 25.4 ms per step at c5);
  // ACCORD_SPMM_STAGES: tuning
  int want = 16;
  if (const char* e = std::getenv("ACCORD_SPMM_STAGES")) want = std::max(2, std::atoi(e));
  int s = (int)std::min<int64_t>(want, std::max<int64_t>(2, (want * 4096) / sb));
  *stages = s;
  return (size_t)s * sb + (size_t)s * sizeof(StageMeta) + 2 * s * 8 + 161 * 8 + 64;
}

bool spmm_tma_supported(int dtype, int64_t ldk) {
  return dtype == ACCORD_F32 && ldk % 8 == 0 && ldk / 8 <= kSpmmTmaMaxConsumers;
}

int launch_item_map(int64_t rows, const int64_t* ptr, int64_t L, int32_t* nitem, int32_t* nslot,
                    int64_t* itm_ptr, int64_t* slot_ptr, void* scan_tmp, size_t scan_tmp_bytes,
                    cudaStream_t st) {
  const unsigned g = (unsigned)std::min<int64_t>(148 * 16, std::max<int64_t>(1, (rows + 255) / 256));
  item_count_kernel<<<g, 256, 0, st>>>(rows, ptr, L, nitem, nslot);
  int l = 1;
  l += launch_scan_i32(nitem, itm_ptr, rows, scan_tmp, scan_tmp_bytes, st);
  l += launch_scan_i32(nslot, slot_ptr, rows, scan_tmp, scan_tmp_bytes, st);
  return l;
}

int launch_spmm_tma(int64_t pk, int64_t ldk, const int64_t* ptr, const int32_t* col,
                    const float* wn, const float* wo, const float* Xt, float* Yout,
                    __nv_bfloat16* Yhi, __nv_bfloat16* Ylo, float* row_A, float* row_B,
                    double* row_D2, double* row_Y2, const SpmmItems& items, int sm_count,
                    cudaStream_t st, const float* wn2, double* row_D2b, int ydrop) {
  if (pk == 0) return 0;
  int stages = 0;
  const size_t smem = spmm_tma_smem(ldk, &stages);
  static unsigned long long attr_seen = 0;
  if (attr_needed(attr_seen)) {
    cudaFuncSetAttribute(spmm_tma_kernel<false, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         100 * 1024);
    cudaFuncSetAttribute(spmm_tma_kernel<true, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         100 * 1024);
    cudaFuncSetAttribute(spmm_tma_kernel<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         100 * 1024);
    cudaFuncSetAttribute(spmm_tma_kernel<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         100 * 1024);
    cudaFuncSetAttribute(spmm_tma_kernel<true, 8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         100 * 1024);
    attr_done(attr_seen);
  }
  // 8 columns per consumer thread; 4 (twice the consumer warps, a third of the
  // accumulator registers) measured slower at c5: 50.3 vs 39.8 ms per step
  // (ACCORD_SPMM_COLS=4: A-B, ldk <= 1024)
  int cols = 8;
  if (const char* e = std::getenv("ACCORD_SPMM_COLS"))
    cols = (std::atoi(e) == 4 && ldk <= 4 * kSpmmTmaMaxConsumers) ? 4 : 8;
  const int consumers = (int)round_up(ldk / cols, 32);
  // warp-parallel producer issue (ACCORD_SPMM_SERIAL=1: one entry at a time;
  // read per launch, tests flip it)
  const char* eser = std::getenv("ACCORD_SPMM_SERIAL");
  const int par_emit = (eser && std::atoi(eser) == 1) ? 0 : 1;
  // persistent: exactly the resident blocks (items are dealt round-robin)
  auto launch = [&](auto kern) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 + consumers, smem) !=
            cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    kern<<<sm_count * std::min(per_sm, 8), 32 + consumers, smem, st>>>(
        pk, ldk, stages, ptr, col, wn, wo, Xt, Yout, Yhi, Ylo, row_A, row_B, row_D2, row_Y2,
        wn2, row_D2b, items, Ylo ? 0 : ydrop, par_emit);
  };
  if (cols == 4) {
    if (wn2) launch(spmm_tma_kernel<true, 4>);
    else launch(spmm_tma_kernel<false, 4>);
  } else {
    static const bool minb2 = [] {
      const char* e = std::getenv("ACCORD_SPMM_MINB");
      return e && std::atoi(e) == 2;
    }();
    if (wn2 && minb2) launch(spmm_tma_kernel<true, 8, 2>);
    else if (wn2) launch(spmm_tma_kernel<true, 8>);
    else launch(spmm_tma_kernel<false, 8>);
  }
  return 1;
}

}  // namespace accord

// Gather ceiling on this GPU: what fraction of the copy bandwidth can a
// kernel reach when every access is a whole 4 KB row of a 4 GB matrix picked
// at random -- the access pattern of the refine SDDMM and the SpMM at config 5
// (X^T rows of random candidate columns). Sets the achievable
// roofline the sparse kernels are judged against.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/gather_bench.cu -o gather_bench
//   ./gather_bench [rows=1000000] [ldk=1024] [gathers=20000000]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));               \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

__global__ void copy_kernel(const float4* __restrict__ a, float4* __restrict__ b, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

__global__ void read_kernel(const float4* __restrict__ a, int64_t n4, float* out) {
  float s = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = __ldg(a + i);
    s += v.x + v.y + v.z + v.w;
  }
  if (s == 1234.5f) *out = s;
}

// warp per gathered row, `unroll` float4 loads in flight per lane
template <int kUnroll>
__global__ void gather_warp_kernel(const float* __restrict__ X, int64_t ldk,
                                   const int32_t* __restrict__ idx, int64_t ng, float* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  float s = 0.f;
  for (int64_t g = w; g < ng; g += nw) {
    const float* r = X + (int64_t)idx[g] * ldk;
    for (int64_t m = lane * 4; m < ldk; m += 32 * 4 * kUnroll) {
      float4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        v[u] = (m + u * 128 < ldk) ? __ldg(reinterpret_cast<const float4*>(r + m + u * 128))
                                   : make_float4(0, 0, 0, 0);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) s += v[u].x + v[u].y + v[u].z + v[u].w;
    }
  }
  if (s == 1234.5f) *out = s;
}

// cp.async.bulk ring: one producer lane per block streams rows into `stages`
// shared-memory slots; the other warps sum them
__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint32_t b, uint32_t tx) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(tx) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(b),
      "r"(ph)
      : "memory");
}

__global__ void gather_bulk_kernel(const float* __restrict__ X, int64_t ldk,
                                   const int32_t* __restrict__ idx, int64_t ng, int stages,
                                   float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t sb = (uint32_t)(ldk * 4);
  float* data = reinterpret_cast<float*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * sb);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ncw = (blockDim.x >> 5) - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(su32(&full[s]), 1);
      mbar_init(su32(&empty[s]), ncw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int64_t g = blockIdx.x; g < ng; g += gridDim.x) {
        mbar_wait(su32(&empty[s]), ph ^ 1);
        mbar_expect(su32(&full[s]), sb);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                su32(data + (size_t)s * ldk)),
            "l"(X + (int64_t)idx[g] * ldk), "r"(sb), "r"(su32(&full[s]))
            : "memory");
        if (++s == stages) { s = 0; ph ^= 1; }
      }
    }
    return;
  }
  const int t = threadIdx.x - 32;
  float acc = 0.f;
  int s = 0;
  uint32_t ph = 0;
  for (int64_t g = blockIdx.x; g < ng; g += gridDim.x) {
    mbar_wait(su32(&full[s]), ph);
    const float* d = data + (size_t)s * ldk;
    for (int64_t m = t * 4; m < ldk; m += (int64_t)ncw * 128) {
      const float4 v = *reinterpret_cast<const float4*>(d + m);
      acc += v.x + v.y + v.z + v.w;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(su32(&empty[s]));
    if (++s == stages) { s = 0; ph ^= 1; }
  }
  if (acc == 1234.5f) *out = acc;
}

// Round 2c: the ring above serialises on the dependent idx[g] load in its
// one-lane producer loop (a global-memory latency per issue), so it measures
// that chain, not the copy engine. These variants prefetch the indices a batch
// of 32 ahead (coalesced), issue from one lane or from all lanes, and the
// consumers either sum in float or do the paired SpMM's arithmetic (8 columns
// per thread, 3 float64 FMAs per element).
template <bool kParIssue, bool kF64>
__global__ void gather_bulk_pf_kernel(const float* __restrict__ X, int64_t ldk,
                                      const int32_t* __restrict__ idx, int64_t ng, int stages,
                                      float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t sb = (uint32_t)(ldk * 4);
  float* data = reinterpret_cast<float*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * sb);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ncw = (blockDim.x >> 5) - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(su32(&full[s]), 1);
      mbar_init(su32(&empty[s]), ncw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  if (warp == 0) {
    int s = 0;
    uint32_t ph = 0;
    int64_t g0 = blockIdx.x;
    int32_t nxt = (g0 + lane * G < ng) ? idx[g0 + lane * G] : -1;
    for (; g0 < ng; g0 += 32 * G) {
      const int32_t cur = nxt;
      const int64_t gn = g0 + 32 * G + lane * G;
      nxt = gn < ng ? idx[gn] : -1;
      const unsigned m = __ballot_sync(0xffffffffu, cur >= 0);
      const int cnt = __popc(m);
      if (kParIssue) {
        for (int r0 = 0; r0 < cnt; r0 += stages) {
          const int nr = min(stages, cnt - r0);
          if (lane >= r0 && lane < r0 + nr) {
            int si = s + (lane - r0);
            uint32_t p2 = ph;
            if (si >= stages) { si -= stages; p2 ^= 1; }
            mbar_wait(su32(&empty[si]), p2 ^ 1);
            mbar_expect(su32(&full[si]), sb);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(data + (size_t)si * ldk)),
                "l"(X + (int64_t)cur * ldk), "r"(sb), "r"(su32(&full[si]))
                : "memory");
          }
          __syncwarp();
          s += nr;
          if (s >= stages) { s -= stages; ph ^= 1; }
        }
      } else {
        for (int k = 0; k < cnt; ++k) {
          const int32_t c = __shfl_sync(0xffffffffu, cur, k);
          if (lane == 0) {
            mbar_wait(su32(&empty[s]), ph ^ 1);
            mbar_expect(su32(&full[s]), sb);
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(data + (size_t)s * ldk)),
                "l"(X + (int64_t)c * ldk), "r"(sb), "r"(su32(&full[s]))
                : "memory");
          }
          __syncwarp();
          if (++s == stages) { s = 0; ph ^= 1; }
        }
      }
    }
    return;
  }
  const int t = threadIdx.x - 32;
  float acc = 0.f;
  double ay[8], ad[8], ae[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) { ay[v] = 0; ad[v] = 0; ae[v] = 0; }
  int s = 0;
  uint32_t ph = 0;
  for (int64_t g = blockIdx.x; g < ng; g += G) {
    mbar_wait(su32(&full[s]), ph);
    const float* d = data + (size_t)s * ldk;
    if (kF64) {
      if ((int64_t)t * 8 < ldk) {
        const float4 a = *reinterpret_cast<const float4*>(d + t * 8);
        const float4 b = *reinterpret_cast<const float4*>(d + t * 8 + 4);
        const float xv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        const double w = 1.0 + (double)(g & 7), dd = 0.5 * w, ee = 0.25 * w;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          ay[v] = fma(w, (double)xv[v], ay[v]);
          ad[v] = fma(dd, (double)xv[v], ad[v]);
          ae[v] = fma(ee, (double)xv[v], ae[v]);
        }
      }
    } else {
      for (int64_t m = t * 4; m < ldk; m += (int64_t)ncw * 128) {
        const float4 v = *reinterpret_cast<const float4*>(d + m);
        acc += v.x + v.y + v.z + v.w;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(su32(&empty[s]));
    if (++s == stages) { s = 0; ph ^= 1; }
  }
  if (kF64) {
#pragma unroll
    for (int v = 0; v < 8; ++v) acc += (float)(ay[v] + ad[v] + ae[v]);
  }
  if (acc == 1234.5f) *out = acc;
}

// LDGSTS ring: the producer warp copies each row with 16-byte cp.async (8 per
// lane at ldk = 1024) and completes the stage through
// cp.async.mbarrier.arrive.noinc (32 arrivals per stage).
template <bool kF64>
__global__ void gather_ldgsts_kernel(const float* __restrict__ X, int64_t ldk,
                                     const int32_t* __restrict__ idx, int64_t ng, int stages,
                                     int npw, float* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  const uint32_t sb = (uint32_t)(ldk * 4);
  float* data = reinterpret_cast<float*>(sm);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * sb);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ncw = (blockDim.x >> 5) - npw;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(su32(&full[s]), 32);
      mbar_init(su32(&empty[s]), ncw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t G = gridDim.x;
  if (warp < npw) {
    // producer warp w handles the block's entries k = w, w + npw, ... (stage k % stages)
    int64_t k = warp;
    int64_t g0 = blockIdx.x + (int64_t)warp * G;   // entry k of this block
    const int64_t step = (int64_t)npw * G;
    int32_t nxt = (g0 + lane * step < ng) ? idx[g0 + lane * step] : -1;
    for (; g0 < ng; g0 += 32 * step) {
      const int32_t cur = nxt;
      const int64_t gn = g0 + 32 * step + lane * step;
      nxt = gn < ng ? idx[gn] : -1;
      const int cnt = __popc(__ballot_sync(0xffffffffu, cur >= 0));
      for (int j = 0; j < cnt; ++j, k += npw) {
        const int32_t c = __shfl_sync(0xffffffffu, cur, j);
        const int s = (int)(k % stages);
        const uint32_t ph = (uint32_t)((k / stages) & 1);
        mbar_wait(su32(&empty[s]), ph ^ 1);
        const float* src = X + (int64_t)c * ldk;
        const uint32_t dst = su32(data + (size_t)s * ldk);
        for (int64_t m = lane * 4; m < ldk; m += 128)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + (uint32_t)m * 4),
                       "l"(src + m)
                       : "memory");
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s]))
                     : "memory");
      }
    }
    return;
  }
  const int t = threadIdx.x - 32 * npw;
  float acc = 0.f;
  double ay[8], ad[8], ae[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) { ay[v] = 0; ad[v] = 0; ae[v] = 0; }
  int s = 0;
  uint32_t ph = 0;
  for (int64_t g = blockIdx.x; g < ng; g += G) {
    mbar_wait(su32(&full[s]), ph);
    const float* d = data + (size_t)s * ldk;
    if (kF64) {
      if ((int64_t)t * 8 < ldk) {
        const float4 a = *reinterpret_cast<const float4*>(d + t * 8);
        const float4 b = *reinterpret_cast<const float4*>(d + t * 8 + 4);
        const float xv[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        const double w = 1.0 + (double)(g & 7), dd = 0.5 * w, ee = 0.25 * w;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          ay[v] = fma(w, (double)xv[v], ay[v]);
          ad[v] = fma(dd, (double)xv[v], ad[v]);
          ae[v] = fma(ee, (double)xv[v], ae[v]);
        }
      }
    } else {
      for (int64_t m = t * 4; m < ldk; m += (int64_t)ncw * 128) {
        const float4 v = *reinterpret_cast<const float4*>(d + m);
        acc += v.x + v.y + v.z + v.w;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(su32(&empty[s]));
    if (++s == stages) { s = 0; ph ^= 1; }
  }
  if (kF64) {
#pragma unroll
    for (int v = 0; v < 8; ++v) acc += (float)(ay[v] + ad[v] + ae[v]);
  }
  if (acc == 1234.5f) *out = acc;
}

int main(int argc, char** argv) {
  const int64_t rows = argc > 1 ? std::atoll(argv[1]) : 1000000;
  const int64_t ldk = argc > 2 ? std::atoll(argv[2]) : 1024;
  const int64_t ng = argc > 3 ? std::atoll(argv[3]) : 20000000;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  float *X, *Y, *out;
  int32_t* idx;
  const size_t xb = (size_t)rows * ldk * 4;
  CK(cudaMalloc(&X, xb));
  CK(cudaMalloc(&Y, xb));
  CK(cudaMalloc(&out, 4));
  CK(cudaMalloc(&idx, ng * 4));
  CK(cudaMemset(X, 0, xb));
  std::vector<int32_t> h(ng);
  uint64_t z = 88172645463325252ull;
  for (int64_t i = 0; i < ng; ++i) {
    z ^= z << 13; z ^= z >> 7; z ^= z << 17;
    h[i] = (int32_t)(z % (uint64_t)rows);
  }
  CK(cudaMemcpy(idx, h.data(), ng * 4, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, double bytes, auto fn) {
    fn();
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    std::printf("%-44s %9.3f ms %8.1f GB/s\n", name, best, bytes / best / 1e6);
  };
  const int64_t n4 = (int64_t)(xb / 16);
  timeit("copy (read + write bytes)", 2.0 * xb, [&] { copy_kernel<<<sms * 8, 512>>>((float4*)X, (float4*)Y, n4); });
  timeit("stream read", (double)xb, [&] { read_kernel<<<sms * 8, 512>>>((float4*)X, n4, out); });
  const double gb = (double)ng * ldk * 4;
  for (int bpsm : {4, 8, 16}) {
    char nm[64];
    std::snprintf(nm, sizeof nm, "gather warp/row unroll 8, %d x 256 thr/SM", bpsm);
    timeit(nm, gb, [&] { gather_warp_kernel<8><<<sms * bpsm, 256>>>(X, ldk, idx, ng, out); });
  }
  timeit("gather warp/row unroll 2, 16 x 256 thr/SM", gb,
         [&] { gather_warp_kernel<2><<<sms * 16, 256>>>(X, ldk, idx, ng, out); });
  for (int stages : {8, 16}) {
    for (int per : {2, 3, 4}) {
      const size_t smem = (size_t)stages * ldk * 4 + 2 * stages * 8;
      if (smem * per > 220 * 1024) continue;
      CK(cudaFuncSetAttribute(gather_bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
      char nm[64];
      std::snprintf(nm, sizeof nm, "gather bulk ring %d stages, %d blk/SM", stages, per);
      timeit(nm, gb, [&] {
        gather_bulk_kernel<<<sms * per, 32 + 128, smem>>>(X, ldk, idx, ng, stages, out);
      });
    }
  }
  // round 2c variants (indices prefetched)
  auto run_pf = [&](const char* tag, auto kern, int stages, int per) {
    const size_t smem = (size_t)stages * ldk * 4 + 2 * stages * 8;
    if (smem * per > 220 * 1024) return;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    char nm[96];
    std::snprintf(nm, sizeof nm, "bulk pf %s %d st, %d blk/SM", tag, stages, per);
    timeit(nm, gb, [&] { kern<<<sms * per, 32 + 128, smem>>>(X, ldk, idx, ng, stages, out); });
  };
  for (int per : {2, 3, 4}) {
    run_pf("lane0 sum", gather_bulk_pf_kernel<false, false>, 8, per);
    run_pf("par   sum", gather_bulk_pf_kernel<true, false>, 8, per);
    run_pf("lane0 f64", gather_bulk_pf_kernel<false, true>, 8, per);
    run_pf("par   f64", gather_bulk_pf_kernel<true, true>, 8, per);
  }
  run_pf("par   sum", gather_bulk_pf_kernel<true, false>, 16, 3);
  run_pf("par   f64", gather_bulk_pf_kernel<true, true>, 16, 3);
  auto run_ls = [&](const char* tag, auto kern, int stages, int per, int npw) {
    const size_t smem = (size_t)stages * ldk * 4 + 2 * stages * 8;
    if (smem * per > 220 * 1024) return;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    char nm[96];
    std::snprintf(nm, sizeof nm, "ldgsts %s %d st, %d blk/SM, %d prod warps", tag, stages, per, npw);
    timeit(nm, gb, [&] {
      kern<<<sms * per, 32 * npw + 128, smem>>>(X, ldk, idx, ng, stages, npw, out);
    });
  };
  for (int per : {2, 3, 4})
    for (int npw : {1, 2}) {
      run_ls("sum", gather_ldgsts_kernel<false>, 8, per, npw);
      run_ls("f64", gather_ldgsts_kernel<true>, 8, per, npw);
    }
  run_ls("f64", gather_ldgsts_kernel<true>, 16, 3, 2);
  CK(cudaGetLastError());
  return 0;
}

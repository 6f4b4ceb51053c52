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
  CK(cudaGetLastError());
  return 0;
}

// Host driver of the ACCORD-FBS hot path: the C ABI of include/accord.h.
//
// One accord_ctx per rank owns the rank's row block of Omega (CSR), the
// replicated X (variable-major), the GEMM operand copies and all scratch.
// accord_step runs Algorithm 1:
//   GEMM + fused candidate epilogue (once per outer iteration; reading R3)
//   -> finalize C -> trial loop { prox(tau) -> SpMM -> reduce -> allreduce ->
//   host decision } -> compact Omega+, swap Y.
#include "accord_internal.h"

#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

using namespace accord;

namespace {

thread_local std::string g_create_err;

struct Fail {
  accord_status s;
  std::string msg;
};

#define CK(call)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess)                                                            \
      throw Fail{e_ == cudaErrorMemoryAllocation ? ACCORD_E_NOMEM : ACCORD_E_CUDA,     \
                 std::string(#call) + ": " + cudaGetErrorString(e_)};                 \
  } while (0)

// --- NCCL, loaded lazily (the process may already hold torch's libnccl) -----
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  ncclResult_t (*CommDestroy)(ncclComm_t);
  const char* (*GetErrorString)(ncclResult_t);
};

NcclApi* nccl_api() {
  static std::once_flag once;
  static NcclApi api;
  static bool ok = false;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
#define SYM(name) api.name = (decltype(api.name))dlsym(h, "nccl" #name)
    SYM(GetUniqueId); SYM(CommInitRank); SYM(AllReduce); SYM(AllGather); SYM(Broadcast);
    SYM(GroupStart); SYM(GroupEnd); SYM(CommDestroy); SYM(GetErrorString);
#undef SYM
    ok = api.GetUniqueId && api.CommInitRank && api.AllReduce && api.AllGather &&
         api.Broadcast && api.GroupStart && api.GroupEnd && api.CommDestroy &&
         api.GetErrorString;
  });
  return ok ? &api : nullptr;
}

#define NK(call)                                                                  \
  do {                                                                            \
    ncclResult_t r_ = (call);                                                     \
    if (r_ != ncclSuccess)                                                        \
      throw Fail{ACCORD_E_NCCL, std::string(#call) + ": " + nccl_api()->GetErrorString(r_)}; \
  } while (0)

}  // namespace

struct accord_ctx {
  int device = 0;
  cudaStream_t st = nullptr;
  int sm_count = 0, cc_major = 0, cc_minor = 0;
  int64_t n = 0, p = 0, r0 = 0, r1 = 0, pk = 0, ldk = 0, p_pad = 0, pk_pad = 0;
  int dtype = ACCORD_F32;
  size_t tsz = 4;
  int gemm = ACCORD_GEMM_SIMT;
  double lam = 0, tau0 = 0, beta = 0, inv_L = 0, L = 0;
  int rank = 0, world = 1, comm = ACCORD_COMM_NONE;
  accord_allreduce_fn ar = nullptr;
  accord_allgatherv_fn agv = nullptr;
  void* cu = nullptr;
  ncclComm_t nccl = nullptr;

  void* Xt = nullptr;
  __nv_bfloat16 *Xhi = nullptr, *Xlo = nullptr;
  void* Y[2] = {nullptr, nullptr};
  __nv_bfloat16* Yhi[2] = {nullptr, nullptr};
  __nv_bfloat16* Ylo[2] = {nullptr, nullptr};
  float* row_A[2] = {nullptr, nullptr};   // ||y_i - bf16(y_i)|| per Y buffer (filter bound)
  float* row_B[2] = {nullptr, nullptr};   // ||y_i||
  float2* col_sd = nullptr;               // per-column constants of the filter bound
  int cur = 0;

  int64_t cap = 0;  // entries of pool / C / keys / Omega arrays
  int64_t* om_ptr = nullptr;
  int32_t* om_col = nullptr;
  void* om_val = nullptr;
  int64_t* c_ptr = nullptr;
  int32_t* c_col = nullptr;
  void *c_g = nullptr, *c_w = nullptr, *c_wn = nullptr;
  uint64_t *keys = nullptr, *keys_tmp = nullptr;
  int32_t *pool_row = nullptr, *pool_col = nullptr;
  void *pool_g = nullptr, *pool_w = nullptr;
  int32_t *row_cnt = nullptr, *rcur = nullptr, *long_rows = nullptr;
  unsigned int* chunk_next = nullptr;      // pool chunks handed out (device counter)
  unsigned long long* chunk_fill = nullptr;   // [nchunks] entries per chunk
  int64_t chunk = 0, nchunks = 0;          // pool chunking (see PoolView)
  int gemm_warps = 0;                      // epilogue warps of the tcgen05 GEMM (0 = SIMT)
  double *row_D2 = nullptr, *row_Y2 = nullptr, *row_dd = nullptr, *row_l1 = nullptr,
         *row_logd = nullptr;
  int32_t* row_nnz = nullptr;
  double* red_d = nullptr;
  int32_t* bad_diag = nullptr;
  void* scan_tmp = nullptr;
  size_t scan_tmp_sz = 0;
  double* h_red = nullptr;                 // pinned [16]
  unsigned long long* h_seg = nullptr;     // pinned [2]: chunks handed out, chunk_fill[0]
  TcGemmPlan* plan = nullptr;
  cudaEvent_t ev[8] = {};

  // bias-correction refit (Eq. 3.8): fixed support S_hat, penalty phi * lambda
  bool refit = false;
  double phi = 1.0;
  int64_t* refit_ptr = nullptr;
  int32_t* refit_col = nullptr;
  int64_t refit_nnz = 0;
  // optional per-kernel tracing (ACCORD_TRACE=1): events after each launch,
  // printed to stderr at the end of every iteration
  bool trace = false;
  std::vector<cudaEvent_t> tr_pool;
  std::vector<std::pair<const char*, cudaEvent_t>> tr_marks;
  int64_t launches = 0, gemm_launches = 0, iters = 0, nnz_local = 0, nnz_global = 0;
  double f = 0, parts[3] = {0, 0, 0};
  std::vector<void*> allocs;
  size_t bytes = 0;
  std::string err;

  template <typename T>
  T* dalloc(size_t count) {
    void* ptr = nullptr;
    const size_t b = std::max<size_t>(count, 1) * sizeof(T);
    CK(cudaMalloc(&ptr, b));
    allocs.push_back(ptr);
    bytes += b;
    return (T*)ptr;
  }
  void* dalloc_bytes(size_t b) {
    void* ptr = nullptr;
    CK(cudaMalloc(&ptr, std::max<size_t>(b, 1)));
    allocs.push_back(ptr);
    bytes += b;
    return ptr;
  }
  void dfree(void* ptr, size_t b) {
    if (!ptr) return;
    auto it = std::find(allocs.begin(), allocs.end(), ptr);
    if (it != allocs.end()) allocs.erase(it);
    cudaFree(ptr);
    bytes -= std::min(bytes, b);
  }
};

namespace {

void allreduce(accord_ctx* c, double* d_buf, double* h_buf, int count) {
  // d_buf (device) -> h_buf (host), summed over ranks. Synchronizes the stream.
  if (c->world > 1 && c->comm == ACCORD_COMM_NCCL) {
    NK(nccl_api()->AllReduce(d_buf, d_buf, count, ncclDouble, ncclSum, c->nccl, c->st));
  }
  CK(cudaMemcpyAsync(h_buf, d_buf, count * sizeof(double), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (c->world > 1 && c->comm == ACCORD_COMM_HOST) {
    if (c->ar(c->cu, h_buf, count) != 0) throw Fail{ACCORD_E_COMM, "host allreduce failed"};
  }
}

// Global maximum of one value per rank (KKT certificate).
double allreduce_max(accord_ctx* c, double* d_val) {
  double h = 0;
  if (c->world > 1 && c->comm == ACCORD_COMM_NCCL)
    NK(nccl_api()->AllReduce(d_val, d_val, 1, ncclDouble, ncclMax, c->nccl, c->st));
  CK(cudaMemcpyAsync(&h, d_val, 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (c->world > 1 && c->comm == ACCORD_COMM_HOST) {
    std::vector<double> v(c->world, 0.0);
    v[c->rank] = h;
    if (c->ar(c->cu, v.data(), c->world) != 0) throw Fail{ACCORD_E_COMM, "host allreduce failed"};
    h = *std::max_element(v.begin(), v.end());
  }
  return h;
}

OmegaView omega_view(accord_ctx* c) { return OmegaView{c->om_ptr, c->om_col, c->om_val}; }

PoolView pool_view(accord_ctx* c) {
  return PoolView{c->pool_row, c->pool_col, c->pool_g, c->pool_w, c->chunk, c->nchunks,
                  c->chunk_next, c->chunk_fill, c->row_cnt};
}

// (Re)allocate the entry-indexed arrays for capacity `cap`, preserving Omega.
void grow(accord_ctx* c, int64_t cap, int64_t keep_nnz) {
  const size_t T = c->tsz;
  int32_t* om_col = c->dalloc<int32_t>(cap);
  void* om_val = c->dalloc_bytes(cap * T);
  if (c->om_col && keep_nnz > 0) {
    CK(cudaMemcpyAsync(om_col, c->om_col, keep_nnz * 4, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(om_val, c->om_val, keep_nnz * T, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
  }
  const int64_t oc = c->cap;
  c->dfree(c->om_col, oc * 4);
  c->dfree(c->om_val, oc * T);
  c->om_col = om_col;
  c->om_val = om_val;
  c->dfree(c->c_col, oc * 4);   c->c_col = c->dalloc<int32_t>(cap);
  c->dfree(c->c_g, oc * T);     c->c_g = c->dalloc_bytes(cap * T);
  c->dfree(c->c_w, oc * T);     c->c_w = c->dalloc_bytes(cap * T);
  c->dfree(c->c_wn, oc * T);    c->c_wn = c->dalloc_bytes(cap * T);
  c->dfree(c->keys, oc * 8);    c->keys = c->dalloc<uint64_t>(cap);
  c->dfree(c->keys_tmp, oc * 8); c->keys_tmp = c->dalloc<uint64_t>(cap);
  c->dfree(c->pool_row, oc * 4); c->pool_row = c->dalloc<int32_t>(cap);
  c->dfree(c->pool_col, oc * 4); c->pool_col = c->dalloc<int32_t>(cap);
  c->dfree(c->pool_g, oc * T);  c->pool_g = c->dalloc_bytes(cap * T);
  c->dfree(c->pool_w, oc * T);  c->pool_w = c->dalloc_bytes(cap * T);
  c->cap = cap;
  // chunking: the SIMT GEMM uses one chunk; the tcgen05 epilogue warps take
  // private chunks of 1024..8192 entries (>= one 32x32 emission batch)
  c->dfree(c->chunk_fill, c->nchunks * 8);
  if (c->gemm_warps == 0) {
    c->chunk = cap;
    c->nchunks = 1;
  } else {
    int64_t ch = 8192;
    while (ch > 1024 && cap / ch < 4 * (int64_t)c->gemm_warps) ch >>= 1;
    c->chunk = ch;
    c->nchunks = std::max<int64_t>(1, cap / ch);
  }
  c->chunk_fill = c->dalloc<unsigned long long>(c->nchunks);
}

// Objective and nnz of the current Omega (collective). Y[cur] must be current
// and row_Y2 must hold ||Y_i||^2.
void refresh_objective(accord_ctx* c) {
  CK(cudaMemsetAsync(c->bad_diag, 0, 4, c->st));
  c->launches += launch_omega_stats(c->dtype, c->pk, c->r0, c->om_ptr, c->om_col, c->om_val,
                                    c->row_l1, c->row_logd, c->row_nnz, c->bad_diag, c->st);
  c->launches += launch_reduce_rows(c->pk, nullptr, nullptr, c->row_logd, c->row_Y2, c->row_l1,
                                    c->row_nnz, nullptr, c->red_d, c->st);
  int32_t bad = 0;
  double loc[8];
  CK(cudaMemcpyAsync(&bad, c->bad_diag, 4, cudaMemcpyDeviceToHost, c->st));
  CK(cudaMemcpyAsync(loc, c->red_d, sizeof(loc), cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  c->nnz_local = (int64_t)loc[5];
  loc[7] = bad ? 1.0 : 0.0;   // make the domain check collective
  CK(cudaMemcpyAsync(c->red_d, loc, sizeof(loc), cudaMemcpyHostToDevice, c->st));
  allreduce(c, c->red_d, c->h_red, 8);
  const bool bad_any = c->h_red[7] > 0;
  c->nnz_global = (int64_t)c->h_red[5];
  const double* r = c->h_red;
  c->parts[0] = -r[2];
  c->parts[1] = r[3] / (2.0 * (double)c->n);
  c->parts[2] = (c->refit ? c->phi * c->lam : c->lam) * r[4];
  c->f = c->parts[0] + c->parts[1] + c->parts[2];
  if (bad_any) throw Fail{ACCORD_E_DOMAIN, "Omega has a missing or nonpositive diagonal entry"};
}

// Y = Omega X^T for the current Omega into Y[cur] (+ row norms).
void recompute_y(accord_ctx* c) {
  c->launches += launch_spmm(c->dtype, c->pk, c->n, c->ldk, c->om_ptr, c->om_col, c->om_val,
                             nullptr, c->Xt, c->Y[c->cur], c->Yhi[c->cur], c->Ylo[c->cur],
                             c->row_A[c->cur], c->row_B[c->cur], nullptr, c->row_Y2, c->st);
}

void validate(const accord_init_params* prm) {
  auto bad = [](const std::string& m) { throw Fail{ACCORD_E_INVALID, m}; };
  if (!prm) bad("params is NULL");
  if (prm->abi_version != ACCORD_ABI_VERSION) bad("abi_version mismatch");
  if (prm->n < 1 || prm->p < 1) bad("need n >= 1 and p >= 1");
  if (prm->p > INT32_MAX - 1024) bad("p too large for int32 column indices");
  if (!prm->X) bad("X is NULL");
  if (prm->dtype != ACCORD_F32 && prm->dtype != ACCORD_F64) bad("dtype must be F32 or F64");
  if (prm->layout != ACCORD_LAYOUT_SAMPLES_ROW_MAJOR &&
      prm->layout != ACCORD_LAYOUT_VARIABLES_ROW_MAJOR)
    bad("bad layout");
  const int64_t minld = prm->layout == ACCORD_LAYOUT_SAMPLES_ROW_MAJOR ? prm->p : prm->n;
  if (prm->ldx != 0 && prm->ldx < minld) bad("ldx smaller than the row length");
  if (!(prm->lambda >= 0) || !std::isfinite(prm->lambda)) bad("lambda must be finite and >= 0");
  if (!(prm->tau0 > 0) || !std::isfinite(prm->tau0)) bad("tau0 must be > 0");
  if (!(prm->beta > 0 && prm->beta <= 1)) bad("beta must be in (0, 1]");
  if (!(prm->inv_L >= 0) || !std::isfinite(prm->inv_L)) bad("inv_L must be >= 0");
  if (prm->row_begin < 0 || prm->row_end > prm->p || prm->row_begin >= prm->row_end)
    bad("bad row range");
  if (prm->world < 1 || prm->rank < 0 || prm->rank >= prm->world) bad("bad rank/world");
  if (prm->world > 1 && prm->comm == ACCORD_COMM_NONE) bad("world > 1 needs a communicator");
  if (prm->comm == ACCORD_COMM_NCCL && prm->world > 1 && !prm->nccl_id) bad("nccl_id is NULL");
  if (prm->comm == ACCORD_COMM_HOST && !prm->allreduce) bad("allreduce callback is NULL");
  if (prm->gemm < ACCORD_GEMM_AUTO || prm->gemm > ACCORD_GEMM_BF16_FILTER) bad("bad gemm kind");
  if (prm->dtype == ACCORD_F64 &&
      (prm->gemm == ACCORD_GEMM_BF16X3 || prm->gemm == ACCORD_GEMM_BF16_FILTER))
    bad("tensor-core GEMM kinds need dtype F32");
}

void create_impl(accord_ctx* c, const accord_init_params* prm) {
  validate(prm);
  if (prm->device >= 0) CK(cudaSetDevice(prm->device));
  CK(cudaGetDevice(&c->device));
  CK(cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, c->device));
  CK(cudaDeviceGetAttribute(&c->cc_major, cudaDevAttrComputeCapabilityMajor, c->device));
  CK(cudaDeviceGetAttribute(&c->cc_minor, cudaDevAttrComputeCapabilityMinor, c->device));
  c->st = (cudaStream_t)prm->stream;
  c->n = prm->n;
  c->p = prm->p;
  c->r0 = prm->row_begin;
  c->r1 = prm->row_end;
  c->pk = c->r1 - c->r0;
  c->ldk = round_up(c->n, kKPad);
  c->p_pad = round_up(c->p, kRowPad);
  c->pk_pad = round_up(c->pk, kRowPad);
  c->dtype = prm->dtype;
  c->tsz = c->dtype == ACCORD_F64 ? 8 : 4;
  c->lam = prm->lambda;
  c->tau0 = prm->tau0;
  c->beta = prm->beta;
  c->rank = prm->rank;
  c->world = prm->world;
  c->comm = prm->world > 1 ? prm->comm : ACCORD_COMM_NONE;
  c->ar = prm->allreduce;
  c->agv = prm->allgatherv;
  c->cu = prm->comm_user;
  const bool tc_ok = tc_supported(c->cc_major, c->cc_minor);
  constexpr int64_t kMaxFilterK = 4096;   // refine kernel stages a Y row in smem
  if (prm->gemm == ACCORD_GEMM_AUTO)
    c->gemm = (c->dtype == ACCORD_F32 && tc_ok)
                  ? (c->ldk <= kMaxFilterK ? ACCORD_GEMM_BF16_FILTER : ACCORD_GEMM_BF16X3)
                  : ACCORD_GEMM_SIMT;
  else
    c->gemm = prm->gemm;
  const bool tc = c->gemm == ACCORD_GEMM_BF16X3 || c->gemm == ACCORD_GEMM_BF16_FILTER;
  if (tc && !tc_ok) throw Fail{ACCORD_E_UNSUPPORTED, "tcgen05 GEMM needs an sm_100 device"};
  if (c->gemm == ACCORD_GEMM_BF16_FILTER && c->ldk > kMaxFilterK)
    throw Fail{ACCORD_E_UNSUPPORTED, "BF16_FILTER supports n <= 4096"};

  for (auto& e : c->ev) CK(cudaEventCreate(&e));
  {
    const char* t = std::getenv("ACCORD_TRACE");
    c->trace = t && t[0] == '1';
  }
  CK(cudaMallocHost(&c->h_red, 16 * sizeof(double)));
  CK(cudaMallocHost(&c->h_seg, 2 * sizeof(unsigned long long)));

  if (c->comm == ACCORD_COMM_NCCL) {
    NcclApi* api = nccl_api();
    if (!api) throw Fail{ACCORD_E_NCCL, "libnccl.so.2 could not be loaded"};
    ncclUniqueId id;
    std::memcpy(&id, prm->nccl_id, sizeof(id));
    NK(api->CommInitRank(&c->nccl, c->world, id, c->rank));
  }

  // ---- X -> Xt (variable-major, padded), finiteness check ----
  const size_t T = c->tsz;
  c->Xt = c->dalloc_bytes((size_t)c->p_pad * c->ldk * T);
  const int64_t rows_src = prm->layout == ACCORD_LAYOUT_SAMPLES_ROW_MAJOR ? c->n : c->p;
  const int64_t cols_src = prm->layout == ACCORD_LAYOUT_SAMPLES_ROW_MAJOR ? c->p : c->n;
  const int64_t ldx = prm->ldx ? prm->ldx : cols_src;
  const void* Xsrc = prm->X;
  void* staging = nullptr;
  if (!prm->x_on_device) {
    CK(cudaMalloc(&staging, (size_t)rows_src * cols_src * T));
    CK(cudaMemcpy2DAsync(staging, cols_src * T, prm->X, ldx * T, cols_src * T, rows_src,
                         cudaMemcpyHostToDevice, c->st));
    Xsrc = staging;
  }
  unsigned long long* badidx = c->dalloc<unsigned long long>(1);
  CK(cudaMemsetAsync(badidx, 0xff, 8, c->st));
  c->launches += launch_load_xt(c->dtype, Xsrc, prm->x_on_device ? ldx : cols_src, prm->layout,
                                c->n, c->p, c->Xt, c->ldk, c->p_pad, badidx, c->st);
  unsigned long long hb = 0;
  CK(cudaMemcpyAsync(&hb, badidx, 8, cudaMemcpyDeviceToHost, c->st));
  CK(cudaStreamSynchronize(c->st));
  if (staging) cudaFree(staging);
  if (hb != ~0ull) {
    char m[160];
    std::snprintf(m, sizeof m, "non-finite X at (row %lld, col %lld) of the given layout",
                  (long long)(hb / cols_src), (long long)(hb % cols_src));
    throw Fail{ACCORD_E_INVALID, m};
  }

  // ---- L ----
  if (prm->inv_L > 0) {
    c->inv_L = prm->inv_L;
    c->L = 1.0 / prm->inv_L;
  } else {
    double L = 0;
    std::string e;
    // power iteration from the all-ones start, relative tolerance,
    // then a safety inflation (overestimating L is safe, underestimating is not)
    int l = power_iteration(c->dtype, c->Xt, c->p, c->n, c->ldk, 600, 1e-8, &L, c->st, &e);
    if (l < 0) throw Fail{ACCORD_E_CUDA, e};
    c->launches += l;
    c->L = L * (1.0 + 2e-3);
    c->inv_L = c->L > 0 ? 1.0 / c->L : 1e300;
  }

  // ---- operands ----
  const bool x3 = c->gemm == ACCORD_GEMM_BF16X3, filt = c->gemm == ACCORD_GEMM_BF16_FILTER;
  for (int b = 0; b < 2; ++b) {
    c->Y[b] = c->dalloc_bytes((size_t)c->pk_pad * c->ldk * T);
    CK(cudaMemsetAsync(c->Y[b], 0, (size_t)c->pk_pad * c->ldk * T, c->st));
  }
  if (tc) {
    c->Xhi = c->dalloc<__nv_bfloat16>((size_t)c->p_pad * c->ldk);
    c->Xlo = c->dalloc<__nv_bfloat16>((size_t)c->p_pad * c->ldk);   // scratch when !x3
    c->launches += launch_split_bf16((const float*)c->Xt, c->p_pad * c->ldk, c->Xhi, c->Xlo,
                                     c->st);
    if (!x3) {
      CK(cudaStreamSynchronize(c->st));
      c->dfree(c->Xlo, (size_t)c->p_pad * c->ldk * 2);
      c->Xlo = nullptr;
    }
    for (int b = 0; b < 2; ++b) {
      c->Yhi[b] = c->dalloc<__nv_bfloat16>((size_t)c->pk_pad * c->ldk);
      CK(cudaMemsetAsync(c->Yhi[b], 0, (size_t)c->pk_pad * c->ldk * 2, c->st));
      if (x3) {
        c->Ylo[b] = c->dalloc<__nv_bfloat16>((size_t)c->pk_pad * c->ldk);
        CK(cudaMemsetAsync(c->Ylo[b], 0, (size_t)c->pk_pad * c->ldk * 2, c->st));
      }
      c->row_A[b] = c->dalloc<float>(c->pk);
      c->row_B[b] = c->dalloc<float>(c->pk);
    }
    if (filt) {
      c->col_sd = c->dalloc<float2>(c->p);
      c->launches += launch_col_norms(c->p, c->ldk, (const float*)c->Xt, c->col_sd, c->st);
    }
    std::string e;
    c->plan = tc_plan_create(c->Yhi[0], x3 ? c->Ylo[0] : c->Yhi[0], c->Yhi[1],
                             x3 ? c->Ylo[1] : c->Yhi[1], c->pk_pad, c->Xhi,
                             x3 ? c->Xlo : c->Xhi, c->p_pad, c->ldk, &e);
    if (!c->plan) throw Fail{ACCORD_E_CUDA, "tensor map: " + e};
    if (filt) c->launches += tc_plan_set_col_norms(c->plan, c->col_sd, c->p, c->st);
  }

  // ---- per-row and entry-indexed state ----
  c->om_ptr = c->dalloc<int64_t>(c->pk + 1);
  c->c_ptr = c->dalloc<int64_t>(c->pk + 1);
  c->row_cnt = c->dalloc<int32_t>(c->pk);
  c->rcur = c->dalloc<int32_t>(c->pk);
  c->long_rows = c->dalloc<int32_t>(c->pk + 1);
  c->chunk_next = c->dalloc<unsigned int>(1);
  c->gemm_warps = c->plan ? 4 * tc_grid_size(c->plan, c->sm_count) : 0;
  c->row_D2 = c->dalloc<double>(c->pk);
  c->row_Y2 = c->dalloc<double>(c->pk);
  c->row_dd = c->dalloc<double>(c->pk);
  c->row_l1 = c->dalloc<double>(c->pk);
  c->row_logd = c->dalloc<double>(c->pk);
  c->row_nnz = c->dalloc<int32_t>(c->pk);
  c->red_d = c->dalloc<double>(16);
  c->bad_diag = c->dalloc<int32_t>(1);
  c->scan_tmp_sz = scan_tmp_bytes(c->pk + 1);
  c->scan_tmp = c->dalloc_bytes(c->scan_tmp_sz);
  int64_t cap = prm->cand_capacity;
  if (cap <= 0) {
    // The first iteration (G = S) has the most candidates (config 5: ~365 per
    // row); size for it so that it is not recomputed, within 40% of the free
    // device memory (~52 B per entry across pool, C, keys and Omega arrays).
    const int64_t dense = c->pk * c->p;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    const int64_t mem_cap = (int64_t)(0.4 * (double)fr / 52.0);
    cap = std::min<int64_t>(dense, std::max<int64_t>(c->pk * 512, 1 << 20));
    cap = std::max<int64_t>(std::min(cap, mem_cap), std::min<int64_t>(dense, c->pk * 16));
  }
  cap = std::max<int64_t>(cap, c->pk);
  grow(c, std::min<int64_t>(cap, (int64_t)UINT32_MAX), 0);

  // ---- Omega^{(0)} = I, Y^{(0)} = rows of X^T, f^{(0)} ----
  c->launches += launch_identity(c->dtype, c->pk, c->r0, c->om_ptr, c->om_col, c->om_val, c->st);
  recompute_y(c);
  refresh_objective(c);
}

template <typename F>
accord_status guard(accord_ctx* c, F&& fn) {
  try {
    fn();
    return ACCORD_OK;
  } catch (const Fail& f) {
    if (c) c->err = f.msg;
    return f.s;
  } catch (const std::bad_alloc&) {
    if (c) c->err = "host allocation failed";
    return ACCORD_E_NOMEM;
  } catch (...) {
    if (c) c->err = "unknown internal error";
    return ACCORD_E_CUDA;
  }
}

void TR(accord_ctx* c, const char* name) {
  if (!c->trace) return;
  if (c->tr_marks.size() >= c->tr_pool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    c->tr_pool.push_back(e);
  }
  cudaEvent_t e = c->tr_pool[c->tr_marks.size()];
  CK(cudaEventRecord(e, c->st));
  c->tr_marks.emplace_back(name, e);
}

void TR_flush(accord_ctx* c) {
  if (!c->trace || c->tr_marks.empty()) return;
  CK(cudaEventSynchronize(c->tr_marks.back().second));
  std::fprintf(stderr, "[accord trace] it=%lld maxrow=%.0f ncand=%.0f", (long long)c->iters,
               c->h_red[7], c->h_red[6]);
  for (size_t i = 1; i < c->tr_marks.size(); ++i) {
    float ms = 0;
    cudaEventElapsedTime(&ms, c->tr_marks[i - 1].second, c->tr_marks[i].second);
    std::fprintf(stderr, " %s=%.3f", c->tr_marks[i].first, ms);
  }
  std::fprintf(stderr, "\n");
  c->tr_marks.clear();
}

float ev_ms(accord_ctx* c, int a, int b) {
  float ms = 0;
  cudaEventElapsedTime(&ms, c->ev[a], c->ev[b]);
  return ms;
}

double lam_eff(const accord_ctx* c) { return c->refit ? c->phi * c->lam : c->lam; }

// Candidate set C with exact gradient values G on it and the current omega:
// either the GEMM + fused epilogue + finalize (+ refine) of a plain iteration,
// or, for the bias-correction refit (Eq. 3.8), the fixed support S_hat with G
// from the SDDMM (entries off S_hat carry an infinite penalty and stay 0).
void build_candidates(accord_ctx* c, accord_iter_stats& st) {
  cudaStream_t S = c->st;
  if (c->refit) {
    CK(cudaEventRecord(c->ev[1], S));
    CK(cudaEventRecord(c->ev[2], S));
    CK(cudaMemcpyAsync(c->c_ptr, c->refit_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToDevice, S));
    CK(cudaMemcpyAsync(c->c_col, c->refit_col, c->refit_nnz * 4, cudaMemcpyDeviceToDevice, S));
    c->launches += launch_lookup(c->dtype, c->pk, c->c_ptr, c->c_col, c->om_ptr, c->om_col,
                                 c->om_val, c->c_w, S);
    CK(cudaEventRecord(c->ev[3], S));
    c->launches += launch_refine(c->dtype, c->pk, c->n, c->ldk, c->c_ptr, c->c_col,
                                 c->Y[c->cur], c->Xt, c->c_g, S);
    CK(cudaEventRecord(c->ev[4], S));
    TR(c, "refit_sddmm");
    CK(cudaEventSynchronize(c->ev[4]));
    st.ms_finalize = ev_ms(c, 2, 3);
    st.ms_refine = ev_ms(c, 3, 4);
    return;
  }
  // ---------------- a2 + a3: gradient GEMM with the fused epilogue --------
  for (;;) {
    CK(cudaMemsetAsync(c->row_cnt, 0, c->pk * 4, S));
    CK(cudaMemsetAsync(c->chunk_fill, 0, c->nchunks * 8, S));
    if (c->gemm_warps == 0) {   // SIMT: one chunk, handed out up front
      static const unsigned int one = 1;
      CK(cudaMemcpyAsync(c->chunk_next, &one, 4, cudaMemcpyHostToDevice, S));
    } else {
      CK(cudaMemsetAsync(c->chunk_next, 0, 4, S));
    }
    EpiParams ep{};
    ep.pk = c->pk;
    ep.p = c->p;
    ep.r0 = c->r0;
    ep.inv_n = 1.0 / (double)c->n;
    ep.lam_cand = c->dtype == ACCORD_F64 ? c->lam : c->lam * (1.0 - 4e-6);
    ep.row_A = c->row_A[c->cur];
    ep.row_B = c->row_B[c->cur];
    ep.col_sd = c->col_sd;
    // fp32-accumulation term of the filter bound: (n/16 + 17) * 2^-22 * sum|y^ x^|
    ep.gamma = (float)(((double)c->ldk / 16.0 + 17.0) * std::ldexp(1.0, -22));
    CK(cudaEventRecord(c->ev[1], S));
    if (c->gemm == ACCORD_GEMM_BF16X3 || c->gemm == ACCORD_GEMM_BF16_FILTER)
    {
      const int l = launch_gemm_tc(c->plan, c->gemm, c->cur, c->ldk, c->sm_count, ep,
                                   omega_view(c), pool_view(c), S);
      if (l < 0) throw Fail{ACCORD_E_CUDA, "GEMM grid / pool segment mismatch"};
      c->launches += l;
    }
    else
      c->launches += launch_gemm_simt(c->dtype, c->Y[c->cur], c->Xt, c->ldk, c->ldk, ep,
                                      omega_view(c), pool_view(c), S);
    c->gemm_launches++;
    CK(cudaGetLastError());
    CK(cudaEventRecord(c->ev[2], S));
    TR(c, "gemm");
    {
      unsigned int used = 0;
      CK(cudaMemcpyAsync(&used, c->chunk_next, 4, cudaMemcpyDeviceToHost, S));
      CK(cudaMemcpyAsync(c->h_seg, c->chunk_fill, 8, cudaMemcpyDeviceToHost, S));
      CK(cudaStreamSynchronize(S));
      c->h_seg[1] = used;
    }
    st.ms_gemm += ev_ms(c, 1, 2);
    // overflow: SIMT counts entries in chunk_fill[0]; tcgen05 counts chunks
    const int64_t need = c->gemm_warps == 0 ? (int64_t)c->h_seg[0]
                                            : (int64_t)c->h_seg[1] * c->chunk;
    const bool ovf = c->gemm_warps == 0 ? need > c->chunk : (int64_t)c->h_seg[1] > c->nchunks;
    if (!ovf) break;
    const int64_t want = need + need / 4 + (1 << 20);
    if (want >= (int64_t)UINT32_MAX)
      throw Fail{ACCORD_E_NOMEM, "candidate pool exceeds 2^32 entries"};
    grow(c, want, c->nnz_local);
  }
  // ---------------- a4: finalize C ----------------
  TR(c, "host_gap");
  c->launches += launch_scan_i32(c->row_cnt, c->c_ptr, c->pk, c->scan_tmp, c->scan_tmp_sz, S);
  TR(c, "scan");
  CK(cudaMemsetAsync(c->rcur, 0, c->pk * 4, S));
  CK(cudaMemsetAsync(c->long_rows, 0, 4, S));
  TR(c, "memset");
  PoolView pv = pool_view(c);
  if (c->gemm == ACCORD_GEMM_BF16_FILTER) pv.g = nullptr;   // values come from the refine
  c->launches += launch_finalize(c->dtype, c->pk, pv, c->c_ptr, c->rcur, c->keys,
                                 c->keys_tmp, c->c_col, c->c_g, c->c_w, c->long_rows, S);
  CK(cudaEventRecord(c->ev[3], S));
  TR(c, "finalize");
  if (c->gemm == ACCORD_GEMM_BF16_FILTER) {
    // exact values of the filtered candidates: G_ik = <Y_i, X_k> / n (f64 accumulation)
    c->launches += launch_refine(c->dtype, c->pk, c->n, c->ldk, c->c_ptr, c->c_col,
                                 c->Y[c->cur], c->Xt, c->c_g, S);
  }
  CK(cudaEventRecord(c->ev[4], S));
  TR(c, "refine");
  CK(cudaEventSynchronize(c->ev[4]));
  st.ms_finalize = ev_ms(c, 2, 3);
  st.ms_refine = ev_ms(c, 3, 4);
}

void step_one(accord_ctx* c, accord_iter_stats* s) {
  accord_iter_stats st{};
  cudaStream_t S = c->st;
  CK(cudaEventRecord(c->ev[0], S));
  TR(c, "start");
  build_candidates(c, st);
  const double lam = lam_eff(c);
  // ---------------- a5-a7: line search ----------------
  const int nb = c->cur ^ 1;
  double tau = c->tau0;
  double r[8];
  for (;;) {
    st.trials++;
    CK(cudaEventRecord(c->ev[4], S));
    c->launches += launch_prox(c->dtype, c->pk, c->r0, c->c_ptr, c->c_col, c->c_g, c->c_w,
                               c->c_wn, tau, lam, c->row_dd, c->row_l1, c->row_logd,
                               c->row_nnz, S);
    CK(cudaEventRecord(c->ev[5], S));
    TR(c, "prox");
    c->launches += launch_spmm(c->dtype, c->pk, c->n, c->ldk, c->c_ptr, c->c_col, c->c_wn,
                               c->c_w, c->Xt, c->Y[nb], c->Yhi[nb], c->Ylo[nb], c->row_A[nb],
                               c->row_B[nb], c->row_D2, c->row_Y2, S);
    CK(cudaEventRecord(c->ev[6], S));
    TR(c, "spmm");
    c->launches += launch_reduce_rows(c->pk, c->row_D2, c->row_dd, c->row_logd, c->row_Y2,
                                      c->row_l1, c->row_nnz, c->c_ptr, c->red_d, S);
    CK(cudaGetLastError());
    allreduce(c, c->red_d, c->h_red, 8);
    CK(cudaEventRecord(c->ev[7], S));
    TR(c, "reduce+decide");
    CK(cudaEventSynchronize(c->ev[7]));
    st.ms_prox += ev_ms(c, 4, 5);
    st.ms_spmm += ev_ms(c, 5, 6);
    st.ms_reduce += ev_ms(c, 6, 7);
    std::memcpy(r, c->h_red, sizeof(r));
    for (int k = 0; k < 7; ++k)
      if (!std::isfinite(r[k])) {
        char m[128];
        std::snprintf(m, sizeof m, "non-finite line-search sum at iteration %lld",
                      (long long)c->iters);
        throw Fail{ACCORD_E_NUMERIC, m};
      }
    // Sufficient decrease in the exact-quadratic form (reading R8):
    // ||Delta X^T||^2 / n <= ||Delta||^2 / tau, or tau <= 1/L.
    const double lhs = r[0] / (double)c->n, rhs = r[1] / tau;
    st.ls_lhs = lhs;
    st.ls_rhs = rhs;
    const bool floor_hit = tau <= c->inv_L;
    if (c->beta >= 1.0 || lhs <= rhs || floor_hit) {
      st.floor_hit = (!(lhs <= rhs) && floor_hit) ? 1 : 0;
      break;
    }
    tau *= c->beta;
  }
  // ---------------- accept: Omega <- Omega+, Y <- Y+ ----------------
  c->launches += launch_scan_i32(c->row_nnz, c->om_ptr, c->pk, c->scan_tmp, c->scan_tmp_sz, S);
  c->launches += launch_compact(c->dtype, c->pk, c->r0, c->c_ptr, c->c_col, c->c_wn, c->om_ptr,
                                c->om_col, c->om_val, S);
  TR(c, "compact");
  c->cur = nb;
  int64_t nnz_loc = 0;
  CK(cudaMemcpyAsync(&nnz_loc, c->om_ptr + c->pk, 8, cudaMemcpyDeviceToHost, S));
  CK(cudaGetLastError());
  CK(cudaEventRecord(c->ev[7], S));
  CK(cudaEventSynchronize(c->ev[7]));
  c->nnz_local = nnz_loc;
  c->nnz_global = (int64_t)r[5];
  c->parts[0] = -r[2];
  c->parts[1] = r[3] / (2.0 * (double)c->n);
  c->parts[2] = lam * r[4];
  c->f = c->parts[0] + c->parts[1] + c->parts[2];
  c->iters++;
  st.tau = tau;
  st.f = c->f;
  st.logdet_part = c->parts[0];
  st.g_part = c->parts[1];
  st.l1_part = c->parts[2];
  st.delta_fro = std::sqrt(r[1]);
  st.nnz = (int64_t)r[5];
  st.n_cand = (int64_t)r[6];
  st.max_row_cand = (int64_t)r[7];
  st.ms_total = ev_ms(c, 0, 7);
  TR_flush(c);
  if (!std::isfinite(c->f)) throw Fail{ACCORD_E_NUMERIC, "non-finite objective"};
  if (s) *s = st;
}

}  // namespace

// ============================================================================
// C ABI
// ============================================================================
extern "C" {

void accord_default_params(accord_init_params* prm) {
  if (!prm) return;
  std::memset(prm, 0, sizeof(*prm));
  prm->abi_version = ACCORD_ABI_VERSION;
  prm->device = -1;
  prm->layout = ACCORD_LAYOUT_SAMPLES_ROW_MAJOR;
  prm->dtype = ACCORD_F32;
  prm->gemm = ACCORD_GEMM_AUTO;
  prm->tau0 = 0.5;
  prm->beta = 0.5;
  prm->world = 1;
  prm->comm = ACCORD_COMM_NONE;
}

accord_status accord_create(accord_ctx** out, const accord_init_params* prm) {
  g_create_err.clear();
  if (!out) {
    g_create_err = "out is NULL";
    return ACCORD_E_INVALID;
  }
  *out = nullptr;
  accord_ctx* c = new (std::nothrow) accord_ctx();
  if (!c) return ACCORD_E_NOMEM;
  accord_status s = guard(c, [&] { create_impl(c, prm); });
  if (s != ACCORD_OK) {
    g_create_err = c->err;
    accord_destroy(c);
    return s;
  }
  *out = c;
  return ACCORD_OK;
}

accord_status accord_step(accord_ctx* c, int32_t iters, accord_iter_stats* stats) {
  if (!c) return ACCORD_E_INVALID;
  if (iters < 0) {
    c->err = "iters < 0";
    return ACCORD_E_INVALID;
  }
  return guard(c, [&] {
    for (int32_t i = 0; i < iters; ++i) step_one(c, stats ? stats + i : nullptr);
  });
}

accord_status accord_objective(accord_ctx* c, double* f, double* parts) {
  if (!c) return ACCORD_E_INVALID;
  if (f) *f = c->f;
  if (parts) std::memcpy(parts, c->parts, sizeof(c->parts));
  return ACCORD_OK;
}

accord_status accord_export_csr(accord_ctx* c, int32_t scope, int64_t* row_ptr, int32_t* col,
                                void* val, int64_t capacity, int64_t* nnz_out,
                                int32_t on_device) {
  if (!c || !nnz_out) return ACCORD_E_INVALID;
  return guard(c, [&] {
    const size_t T = c->tsz;
    const cudaMemcpyKind k = on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (scope == ACCORD_SCOPE_LOCAL || c->world == 1) {
      *nnz_out = c->nnz_local;
      if (!row_ptr) return;
      if (capacity < c->nnz_local) throw Fail{ACCORD_E_CAPACITY, "capacity too small"};
      CK(cudaMemcpyAsync(row_ptr, c->om_ptr, (c->pk + 1) * 8, k, c->st));
      CK(cudaMemcpyAsync(col, c->om_col, c->nnz_local * 4, k, c->st));
      CK(cudaMemcpyAsync(val, c->om_val, c->nnz_local * T, k, c->st));
      CK(cudaStreamSynchronize(c->st));
      return;
    }
    if (scope != ACCORD_SCOPE_GATHER) throw Fail{ACCORD_E_INVALID, "bad scope"};
    // ---- gather all ranks' row blocks (collective) ----
    // 1) per-rank (rows, nnz)
    std::vector<double> h(2 * c->world, 0.0);
    double* d = c->red_d;
    std::vector<double> mine(2 * c->world, 0.0);
    mine[2 * c->rank] = (double)c->pk;
    mine[2 * c->rank + 1] = (double)c->nnz_local;
    std::vector<double> tot(2 * c->world);
    for (int q = 0; q < 2 * c->world; q += 8) {
      const int cnt = std::min(8, 2 * c->world - q);
      CK(cudaMemcpyAsync(d, mine.data() + q, cnt * 8, cudaMemcpyHostToDevice, c->st));
      allreduce(c, d, c->h_red, cnt);
      std::memcpy(tot.data() + q, c->h_red, cnt * 8);
    }
    int64_t total = 0, rows_total = 0;
    for (int q = 0; q < c->world; ++q) {
      rows_total += (int64_t)tot[2 * q];
      total += (int64_t)tot[2 * q + 1];
    }
    *nnz_out = total;
    if (!row_ptr) return;
    if (capacity < total) throw Fail{ACCORD_E_CAPACITY, "capacity too small"};
    if (rows_total != c->p) throw Fail{ACCORD_E_INVALID, "row blocks do not cover p rows"};
    // local block to host
    std::vector<int64_t> lp(c->pk + 1);
    std::vector<int32_t> lc(c->nnz_local);
    std::vector<char> lv(c->nnz_local * T);
    CK(cudaMemcpyAsync(lp.data(), c->om_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(lc.data(), c->om_col, c->nnz_local * 4, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(lv.data(), c->om_val, c->nnz_local * T, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    std::vector<int64_t> gp(c->p + 1, 0);
    std::vector<int32_t> gc(total);
    std::vector<char> gv(total * T);
    if (c->comm == ACCORD_COMM_NCCL) {
      NcclApi* api = nccl_api();
      int64_t* dptr = nullptr;
      int32_t* dcol = nullptr;
      char* dval = nullptr;
      CK(cudaMalloc(&dptr, (rows_total + c->world) * 8));
      CK(cudaMalloc(&dcol, std::max<int64_t>(total, 1) * 4));
      CK(cudaMalloc(&dval, std::max<int64_t>(total, 1) * T));
      int64_t ro = 0, eo = 0;
      NK(api->GroupStart());
      for (int q = 0; q < c->world; ++q) {
        const int64_t rq = (int64_t)tot[2 * q], nq = (int64_t)tot[2 * q + 1];
        const bool me = q == c->rank;
        NK(api->Broadcast(me ? (const void*)c->om_ptr : nullptr, dptr + ro + q, (rq + 1) * 8,
                          ncclChar, q, c->nccl, c->st));
        if (nq > 0) {
          NK(api->Broadcast(me ? (const void*)c->om_col : nullptr, dcol + eo, nq * 4, ncclChar, q,
                            c->nccl, c->st));
          NK(api->Broadcast(me ? (const void*)c->om_val : nullptr, dval + eo * T, nq * T,
                            ncclChar, q, c->nccl, c->st));
        }
        ro += rq;
        eo += nq;
      }
      NK(api->GroupEnd());
      std::vector<int64_t> hp(rows_total + c->world);
      CK(cudaMemcpyAsync(hp.data(), dptr, hp.size() * 8, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(gc.data(), dcol, total * 4, cudaMemcpyDeviceToHost, c->st));
      CK(cudaMemcpyAsync(gv.data(), dval, total * T, cudaMemcpyDeviceToHost, c->st));
      CK(cudaStreamSynchronize(c->st));
      cudaFree(dptr);
      cudaFree(dcol);
      cudaFree(dval);
      ro = 0;
      eo = 0;
      for (int q = 0; q < c->world; ++q) {
        const int64_t rq = (int64_t)tot[2 * q];
        for (int64_t i = 0; i <= rq; ++i) gp[ro + i] = eo + hp[ro + q + i];
        ro += rq;
        eo += (int64_t)tot[2 * q + 1];
      }
    } else {
      if (!c->agv) throw Fail{ACCORD_E_INVALID, "GATHER with host comm needs allgatherv"};
      // pack [rows][nnz][row_ptr][col][val]
      std::vector<char> blob(16 + lp.size() * 8 + lc.size() * 4 + lv.size());
      int64_t hdr[2] = {c->pk, c->nnz_local};
      char* w = blob.data();
      std::memcpy(w, hdr, 16); w += 16;
      std::memcpy(w, lp.data(), lp.size() * 8); w += lp.size() * 8;
      std::memcpy(w, lc.data(), lc.size() * 4); w += lc.size() * 4;
      std::memcpy(w, lv.data(), lv.size());
      std::vector<int64_t> counts(c->world, 0);
      if (c->agv(c->cu, blob.data(), (int64_t)blob.size(), nullptr, counts.data()) != 0)
        throw Fail{ACCORD_E_COMM, "allgatherv (sizes) failed"};
      int64_t all = 0;
      for (auto x : counts) all += x;
      std::vector<char> buf(all);
      if (c->agv(c->cu, blob.data(), (int64_t)blob.size(), buf.data(), counts.data()) != 0)
        throw Fail{ACCORD_E_COMM, "allgatherv failed"};
      const char* rd = buf.data();
      int64_t ro = 0, eo = 0;
      for (int q = 0; q < c->world; ++q) {
        int64_t hq[2];
        std::memcpy(hq, rd, 16);
        const int64_t* qp = (const int64_t*)(rd + 16);
        for (int64_t i = 0; i <= hq[0]; ++i) gp[ro + i] = eo + qp[i];
        std::memcpy(gc.data() + eo, rd + 16 + (hq[0] + 1) * 8, hq[1] * 4);
        std::memcpy(gv.data() + eo * T, rd + 16 + (hq[0] + 1) * 8 + hq[1] * 4, hq[1] * T);
        rd += counts[q];
        ro += hq[0];
        eo += hq[1];
      }
    }
    const cudaMemcpyKind hk = on_device ? cudaMemcpyHostToDevice : cudaMemcpyHostToHost;
    CK(cudaMemcpy(row_ptr, gp.data(), gp.size() * 8, hk));
    CK(cudaMemcpy(col, gc.data(), gc.size() * 4, hk));
    CK(cudaMemcpy(val, gv.data(), gv.size(), hk));
  });
}

accord_status accord_set_omega_csr(accord_ctx* c, const int64_t* row_ptr, const int32_t* col,
                                   const void* val, int64_t nnz) {
  if (!c || !row_ptr || (nnz > 0 && (!col || !val))) return ACCORD_E_INVALID;
  return guard(c, [&] {
    if (row_ptr[0] != 0 || row_ptr[c->pk] != nnz) throw Fail{ACCORD_E_INVALID, "bad row_ptr"};
    for (int64_t i = 0; i < c->pk; ++i) {
      if (row_ptr[i + 1] < row_ptr[i]) throw Fail{ACCORD_E_INVALID, "row_ptr not monotone"};
      for (int64_t e = row_ptr[i]; e < row_ptr[i + 1]; ++e) {
        if (col[e] < 0 || col[e] >= c->p) throw Fail{ACCORD_E_INVALID, "column out of range"};
        if (e > row_ptr[i] && col[e] <= col[e - 1])
          throw Fail{ACCORD_E_INVALID, "columns not strictly increasing"};
      }
    }
    if (nnz > c->cap) grow(c, nnz + nnz / 4 + 1024, 0);
    CK(cudaMemcpyAsync(c->om_ptr, row_ptr, (c->pk + 1) * 8, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->om_col, col, nnz * 4, cudaMemcpyHostToDevice, c->st));
    CK(cudaMemcpyAsync(c->om_val, val, nnz * c->tsz, cudaMemcpyHostToDevice, c->st));
    c->nnz_local = nnz;
    recompute_y(c);
    refresh_objective(c);
  });
}

accord_status accord_set_lambda(accord_ctx* c, double lambda) {
  if (!c) return ACCORD_E_INVALID;
  if (!(lambda >= 0) || !std::isfinite(lambda)) {
    c->err = "lambda must be finite and >= 0";
    return ACCORD_E_INVALID;
  }
  return guard(c, [&] {
    c->lam = lambda;
    refresh_objective(c);
  });
}

accord_status accord_refit(accord_ctx* c, double phi) {
  if (!c) return ACCORD_E_INVALID;
  if (!(phi >= 0 && phi <= 1)) {
    c->err = "phi must be in [0, 1] (Eq. 3.8)";
    return ACCORD_E_INVALID;
  }
  return guard(c, [&] {
    // S_hat = support of the current estimate (diagonal always stored)
    c->dfree(c->refit_ptr, (c->pk + 1) * 8);
    c->dfree(c->refit_col, c->refit_nnz * 4);
    c->refit_nnz = c->nnz_local;
    c->refit_ptr = c->dalloc<int64_t>(c->pk + 1);
    c->refit_col = c->dalloc<int32_t>(std::max<int64_t>(c->refit_nnz, 1));
    CK(cudaMemcpyAsync(c->refit_ptr, c->om_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToDevice,
                       c->st));
    CK(cudaMemcpyAsync(c->refit_col, c->om_col, c->refit_nnz * 4, cudaMemcpyDeviceToDevice,
                       c->st));
    c->refit = true;
    c->phi = phi;
    refresh_objective(c);
  });
}

accord_status accord_solve(accord_ctx* c, int32_t max_iter, double tol, int32_t* iters_done,
                           accord_iter_stats* last) {
  if (!c || max_iter < 0 || !(tol >= 0)) return ACCORD_E_INVALID;
  return guard(c, [&] {
    accord_iter_stats st{};
    int32_t it = 0;
    while (it < max_iter) {
      step_one(c, &st);
      ++it;
      if (st.delta_fro < tol) break;   // ||Omega^(t+1) - Omega^(t)||_F < tol (reading R13)
    }
    if (iters_done) *iters_done = it;
    if (last) *last = st;
  });
}

accord_status accord_kkt_residual(accord_ctx* c, double* kkt) {
  if (!c || !kkt) return ACCORD_E_INVALID;
  return guard(c, [&] {
    accord_iter_stats st{};
    build_candidates(c, st);
    c->launches += launch_kkt(c->dtype, c->pk, c->r0, c->c_ptr, c->c_col, c->c_g, c->c_w,
                              lam_eff(c), c->row_dd, c->red_d + 8, c->st);
    CK(cudaGetLastError());
    *kkt = allreduce_max(c, c->red_d + 8);
  });
}

accord_status accord_path(accord_ctx* c, const double* lambdas, int32_t k, int32_t max_iter,
                          double tol, double gamma, double* epbic, int64_t* nnz_off,
                          int32_t* iters, int32_t* best) {
  if (!c || !lambdas || k < 1 || max_iter < 1 || !(gamma >= 0)) return ACCORD_E_INVALID;
  return guard(c, [&] {
    const size_t T = c->tsz;
    int64_t* bptr = c->dalloc<int64_t>(c->pk + 1);
    int32_t* bcol = nullptr;
    void* bval = nullptr;
    int64_t bcap = 0, bnnz = 0;
    double best_e = INFINITY, best_lam = c->lam;
    int32_t bi = 0;
    for (int32_t j = 0; j < k; ++j) {
      if (!(lambdas[j] >= 0) || !std::isfinite(lambdas[j]))
        throw Fail{ACCORD_E_INVALID, "bad lambda in the path"};
      c->lam = lambdas[j];
      refresh_objective(c);                       // warm start from the previous estimate
      accord_iter_stats st{};
      int32_t it = 0;
      while (it < max_iter) {
        step_one(c, &st);
        ++it;
        if (st.delta_fro < tol) break;
      }
      // epBIC, Eq. (3.7): 2n (loss) + ||Omega||_0 (log n + 4 gamma log p), off-diagonal count
      const double loss = c->parts[0] + c->parts[1];
      const int64_t koff = c->nnz_global - c->p;
      const double e = 2.0 * (double)c->n * loss +
                       (double)koff * (std::log((double)c->n) + 4.0 * gamma * std::log((double)c->p));
      if (epbic) epbic[j] = e;
      if (nnz_off) nnz_off[j] = koff;
      if (iters) iters[j] = it;
      if (e < best_e) {
        best_e = e;
        best_lam = lambdas[j];
        bi = j;
        if (c->nnz_local > bcap) {
          c->dfree(bcol, bcap * 4);
          c->dfree(bval, bcap * T);
          bcap = c->nnz_local + c->nnz_local / 4 + 16;
          bcol = c->dalloc<int32_t>(bcap);
          bval = c->dalloc_bytes(bcap * T);
        }
        bnnz = c->nnz_local;
        CK(cudaMemcpyAsync(bptr, c->om_ptr, (c->pk + 1) * 8, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(bcol, c->om_col, bnnz * 4, cudaMemcpyDeviceToDevice, c->st));
        CK(cudaMemcpyAsync(bval, c->om_val, bnnz * T, cudaMemcpyDeviceToDevice, c->st));
      }
    }
    // restore the epBIC-selected estimate (and its lambda)
    CK(cudaMemcpyAsync(c->om_ptr, bptr, (c->pk + 1) * 8, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(c->om_col, bcol, bnnz * 4, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaMemcpyAsync(c->om_val, bval, bnnz * T, cudaMemcpyDeviceToDevice, c->st));
    CK(cudaStreamSynchronize(c->st));
    c->dfree(bptr, (c->pk + 1) * 8);
    c->dfree(bcol, bcap * 4);
    c->dfree(bval, bcap * T);
    c->nnz_local = bnnz;
    c->lam = best_lam;
    recompute_y(c);
    refresh_objective(c);
    if (best) *best = bi;
  });
}

accord_status accord_row_stats(accord_ctx* c, const int64_t* rows, int64_t count, double* d2,
                               double* delta2) {
  if (!c || (count > 0 && !rows)) return ACCORD_E_INVALID;
  return guard(c, [&] {
    std::vector<double> a(c->pk), b(c->pk);
    CK(cudaMemcpyAsync(a.data(), c->row_D2, c->pk * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaMemcpyAsync(b.data(), c->row_dd, c->pk * 8, cudaMemcpyDeviceToHost, c->st));
    CK(cudaStreamSynchronize(c->st));
    for (int64_t q = 0; q < count; ++q) {
      if (rows[q] < 0 || rows[q] >= c->pk) throw Fail{ACCORD_E_INVALID, "row out of range"};
      if (d2) d2[q] = a[rows[q]];
      if (delta2) delta2[q] = b[rows[q]];
    }
  });
}

accord_status accord_get_info(accord_ctx* c, accord_info* info) {
  if (!c || !info) return ACCORD_E_INVALID;
  std::memset(info, 0, sizeof(*info));
  info->n = c->n;
  info->p = c->p;
  info->row_begin = c->r0;
  info->row_end = c->r1;
  info->ldk = c->ldk;
  info->L = c->L;
  info->inv_L = c->inv_L;
  info->lambda = c->lam;
  info->tau0 = c->tau0;
  info->beta = c->beta;
  info->dtype = c->dtype;
  info->gemm = c->gemm;
  info->sm_count = c->sm_count;
  info->cc_major = c->cc_major;
  info->cc_minor = c->cc_minor;
  info->iterations = c->iters;
  info->nnz_local = c->nnz_local;
  info->cand_capacity = c->cap;
  info->kernel_launches = c->launches;
  info->gemm_launches = c->gemm_launches;
  info->f = c->f;
  info->device_bytes = c->bytes;
  return ACCORD_OK;
}

accord_status accord_nccl_unique_id(uint8_t id[128]) {
  NcclApi* api = nccl_api();
  if (!api || !id) return ACCORD_E_NCCL;
  ncclUniqueId u;
  if (api->GetUniqueId(&u) != ncclSuccess) return ACCORD_E_NCCL;
  std::memcpy(id, &u, 128);
  return ACCORD_OK;
}

void accord_destroy(accord_ctx* c) {
  if (!c) return;
  if (c->st) cudaStreamSynchronize(c->st);
  else cudaDeviceSynchronize();
  if (c->plan) tc_plan_destroy(c->plan);
  for (void* ptr : c->allocs) cudaFree(ptr);
  for (auto& e : c->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : c->tr_pool) cudaEventDestroy(e);
  if (c->h_red) cudaFreeHost(c->h_red);
  if (c->h_seg) cudaFreeHost(c->h_seg);
  if (c->nccl && nccl_api()) nccl_api()->CommDestroy(c->nccl);
  delete c;
}

const char* accord_status_string(accord_status s) {
  switch (s) {
    case ACCORD_OK: return "ok";
    case ACCORD_E_INVALID: return "invalid argument";
    case ACCORD_E_CUDA: return "CUDA error";
    case ACCORD_E_NCCL: return "NCCL error";
    case ACCORD_E_CAPACITY: return "buffer capacity too small";
    case ACCORD_E_NUMERIC: return "non-finite value";
    case ACCORD_E_DOMAIN: return "nonpositive diagonal";
    case ACCORD_E_NOMEM: return "out of memory";
    case ACCORD_E_UNSUPPORTED: return "unsupported";
    case ACCORD_E_COMM: return "communicator callback failed";
  }
  return "unknown status";
}

const char* accord_last_error(const accord_ctx* c) {
  return c ? c->err.c_str() : g_create_err.c_str();
}

int32_t accord_abi_version(void) { return ACCORD_ABI_VERSION; }

}  // extern "C"
